// Library plumbing: version, status strings, last-error text, the device
// error word (integer divide by zero, reference simulator.py:63-65) and the
// launch counter used for the bench's `gpu_launches` accounting.
#include "common.cuh"

#include <mutex>

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

}  // namespace spmd

using namespace spmd;

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
