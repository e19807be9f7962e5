// Library plumbing: version, status strings, last-error text, the device
// error word (integer divide by zero, reference simulator.py:63-65) and the
// launch counter used for the bench's `gpu_launches` accounting.
#include "common.cuh"

#include <mutex>
#include <stdlib.h>
#include <string.h>

namespace spmd {

static thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int* device_error_word() {
  // One word per device, allocated lazily on first use.
  static std::mutex mu;
  static int* words[64] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!words[dev]) {
    int* p = nullptr;
    if (cudaMalloc(&p, sizeof(int)) != cudaSuccess) {
      set_error("cudaMalloc(error word) failed");
      return nullptr;
    }
    cudaMemset(p, 0, sizeof(int));
    cudaDeviceSynchronize();
    words[dev] = p;
  }
  return words[dev];
}

static std::atomic<int> g_sm_limit{0};

int sm_budget() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int lim = g_sm_limit.load();
  int n = (lim > 0 && lim < sms) ? lim : sms;
  return n < 2 ? 2 : (n & ~1);   // even: CTA pairs
}

struct OptDef {
  const char* name;
  const char* env;
  int64_t def;
};
static const OptDef kOpts[OPT_COUNT] = {
    {"gemm_mode", "SPMD_GEMM_MODE", 3},
    {"gemm_group", "SPMD_GEMM_GROUP", 0},
    {"gemm_raster_n", "SPMD_GEMM_RASTER", 0},
    {"gemm_hint", "SPMD_GEMM_HINT", 0},
    {"gemm_store_hint", "SPMD_GEMM_STORE_HINT", 0},
    {"gemm_epi_direct", "SPMD_GEMM_EPI", 0},
    {"scatter_epi_direct", "SPMD_SCATTER_EPI", 0},
    {"attn_mode", "SPMD_ATTN_MODE", 2},
    {"attn_kt", "SPMD_ATTN_KT", 0},
    {"conv_mode", "SPMD_CONV_MODE", 2},
    {"conv_wres", "SPMD_CONV_WRES", 1},
    {"conv_taps", "SPMD_CONV_TAPS", 1},
    {"nccl_max_ctas", "SPMD_NCCL_MAX_CTAS", 0},
    {"peer_timeout_ms", "SPMD_PEER_TIMEOUT_MS", 20000},
    {"peer_serial_pulls", "SPMD_PEER_SERIAL_PULLS", 0},
    {"f32_dot_tc", "SPMD_F32_DOT_TC", 1},
    {"gemm_persistent", "SPMD_GEMM_PERSISTENT", 1},
    {"gemm_dynamic", "SPMD_GEMM_DYNAMIC", 1},
};
static std::atomic<int64_t> g_opts[OPT_COUNT];
static std::once_flag g_opts_once;

// Environment spellings kept from the per-kernel getenv()s they replace.
static int64_t parse_env(int id, const char* e) {
  if (!strcmp(e, "1sm")) return 1;
  if (!strcmp(e, "2sm")) return 2;
  if (!strcmp(e, "wide")) return 3;
  if (!strcmp(e, "direct")) return 1;
  if (id == OPT_GEMM_RASTER_N) return !strcmp(e, "n") ? 1 : atoll(e);
  if (id == OPT_GEMM_MODE || id == OPT_ATTN_MODE || id == OPT_CONV_MODE) {
    const int64_t v = atoll(e);
    return v > 0 ? v : kOpts[id].def;
  }
  return atoll(e);
}

static void init_options() {
  std::call_once(g_opts_once, [] {
    for (int i = 0; i < OPT_COUNT; ++i) {
      const char* e = getenv(kOpts[i].env);
      g_opts[i].store(e && *e ? parse_env(i, e) : kOpts[i].def);
    }
    // seconds spelling of the peer timeout
    const char* t = getenv("SPMD_PEER_TIMEOUT_S");
    if (t && *t && !getenv("SPMD_PEER_TIMEOUT_MS"))
      g_opts[OPT_PEER_TIMEOUT_MS].store((int64_t)(atof(t) * 1000.0));
  });
}

int64_t option(int id) {
  init_options();
  return (id >= 0 && id < OPT_COUNT) ? g_opts[id].load(std::memory_order_relaxed) : 0;
}

static int find_option(const char* name) {
  for (int i = 0; name && i < OPT_COUNT; ++i)
    if (!strcmp(kOpts[i].name, name)) return i;
  return -1;
}

int set_smem_attr(const void* kernel, int bytes, std::atomic<uint64_t>* done_mask) {
  int dev = 0;
  SPMD_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done_mask->load() & bit) return SPMD_OK;
  SPMD_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done_mask->fetch_or(bit);
  return SPMD_OK;
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_set_option(const char* name, int64_t value) {
  init_options();
  const int i = find_option(name);
  if (i < 0) {
    set_error(std::string("unknown option: ") + (name ? name : "(null)"));
    return SPMD_ERR_INVALID;
  }
  g_opts[i].store(value);
  return SPMD_OK;
}

extern "C" int spmd_get_option(const char* name, int64_t* value) {
  const int i = find_option(name);
  if (i < 0 || !value) {
    set_error(std::string("unknown option: ") + (name ? name : "(null)"));
    return SPMD_ERR_INVALID;
  }
  *value = option(i);
  return SPMD_OK;
}

extern "C" int spmd_set_sm_limit(int sms) {
  g_sm_limit.store(sms > 0 ? sms : 0);
  return SPMD_OK;
}

extern "C" const char* spmd_version(void) { return "spmd_b200 0.1.0 (sm_100a)"; }

extern "C" const char* spmd_status_string(int status) {
  switch (status) {
    case SPMD_OK: return "ok";
    case SPMD_ERR_INVALID: return "invalid argument";
    case SPMD_ERR_SHAPE: return "shape mismatch";
    case SPMD_ERR_SUBGROUP: return "subgroup mismatch";
    case SPMD_ERR_DIV_ZERO: return "integer division by zero";
    case SPMD_ERR_CUDA: return "CUDA error";
    case SPMD_ERR_NCCL: return "NCCL error";
    case SPMD_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

extern "C" const char* spmd_last_error(void) { return g_last_error.c_str(); }

extern "C" int64_t spmd_launch_count(void) { return g_launches.load(); }

extern "C" int spmd_check_device_errors(void* stream) {
  int* w = device_error_word();
  if (!w) return SPMD_ERR_CUDA;
  int host = 0;
  cudaStream_t s = as_stream(stream);
  SPMD_CUDA_TRY(cudaMemcpyAsync(&host, w, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPMD_CUDA_TRY(cudaStreamSynchronize(s));
  if (host) {
    SPMD_CUDA_TRY(cudaMemsetAsync(w, 0, sizeof(int), s));
    SPMD_CUDA_TRY(cudaStreamSynchronize(s));
    if (host & 1) {
      set_error("integer division by zero");
      return SPMD_ERR_DIV_ZERO;
    }
    if (host & 2) {
      set_error("peer barrier timed out (a rank did not reach the fused collective)");
      return SPMD_ERR_NCCL;
    }
  }
  return SPMD_OK;
}
