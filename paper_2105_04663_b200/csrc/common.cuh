// Shared helpers for the sm_100a kernels behind include/spmd_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <atomic>
#include <string>

#include "../../include/spmd_b200.h"

namespace spmd {

// ---------------------------------------------------------------------------
// status / error plumbing
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
extern std::atomic<int64_t> g_launches;
// Device error word (cudaMalloc'd int on the current device): bit 0 =
// integer division by zero.  Kernels that can fault receive it as a pointer.
int* device_error_word();
// SMs the persistent tensor-core kernels may occupy (spmd_set_sm_limit):
// leaves room for NCCL kernels to co-reside when collectives overlap GEMMs.
int sm_budget();

// Runtime tuning options (spmd_set_option / spmd_get_option).  Each starts
// from its SPMD_* environment variable (read once, at first use) and is read
// again at every launch, so a process can switch kernel variants (tests force
// every GEMM path this way) without restarting.
enum Option : int {
  OPT_GEMM_MODE = 0,        // 1: 1-CTA tiles, 2: 256x256 CTA pairs, 3: 256x512 wide pairs
  OPT_GEMM_GROUP,           // M-tiles per raster group (0: kernel default)
  OPT_GEMM_RASTER_N,        // 1: raster along N inside a group
  OPT_GEMM_HINT,            // L2 cache hint of the operand loads
  OPT_GEMM_STORE_HINT,      // 1: evict-first output stores
  OPT_GEMM_EPI_DIRECT,      // 1: st.global epilogue instead of TMA stores
  OPT_SCATTER_EPI_DIRECT,   // 1: st.global peer stores in the reduce-scatter epilogue
  OPT_ATTN_MODE,            // 1: 1-CTA attention, 2: CTA pairs
  OPT_ATTN_KT,              // key tile (0: per head dim)
  OPT_CONV_MODE,            // 1: 1-CTA conv, 2: CTA pairs
  OPT_CONV_WRES,            // 1: weights resident in smem
  OPT_CONV_TAPS,            // 1: one input box feeds the 3 kw taps
  OPT_NCCL_MAX_CTAS,        // NCCL maxCTAs at communicator creation (0: NCCL default)
  OPT_PEER_TIMEOUT_MS,      // peer barrier timeout
  OPT_PEER_SERIAL_PULLS,    // 1: staged gathers pull members one after another
  OPT_F32_DOT_TC,           // 1: large f32 Dots on the tensor cores (3xTF32)
  OPT_GEMM_PERSISTENT,      // 1: one CTA pair per 2 SMs walks the tiles; 0: one pair per tile
  OPT_GEMM_DYNAMIC,         // 1: persistent wide GEMM takes tiles from a global counter
  OPT_COUNT
};
int64_t option(int id);
// cudaFuncAttributeMaxDynamicSharedMemorySize once per (kernel, device):
// the attribute is per device, so a process driving two GPUs sets it twice.
int set_smem_attr(const void* kernel, int bytes, std::atomic<uint64_t>* done_mask);

// Reduce-scatter epilogue target of the tcgen05 GEMM (peer.cu): column chunk
// j of the output goes to dst[j] (group position j's peer heap), slot
// parity * par_slots + pos.
struct GemmScatter {
  int gsize, pos;
  void* dst[8];
  const uint32_t* epoch;
  // rows != 0: all-to-all mode -- output ROW chunks of `rchunk` rows go to
  // group member row / rchunk, slot slot_base + batch of nslots (no reduce)
  int rows;
  int64_t rchunk;
  int slot_base, nslots;
  // Slots per parity buffer: parity p of the landing zone starts at slot
  // p * par_slots (peer.cu fused_parity: a fixed byte stride for all ops).
  int par_slots;
};
// Implemented in gemm_tcgen05.cu: returns SPMD_ERR_UNSUPPORTED when the
// layout cannot be expressed with TMA descriptors (or, with `sc`, when the
// scattered dim is not the whole GEMM N).
int dot_tcgen05(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
                const spmd_dot_dims& dd, int64_t nparts, cudaStream_t s,
                const GemmScatter* sc = nullptr, const void* resid = nullptr);
// Implemented in gemm_tf32x3.cu: large f32 Dots as a 3xTF32 tcgen05 GEMM;
// SPMD_ERR_UNSUPPORTED for small / untileable ones (SIMT fp64 path then).
// lhs_hi / lhs_lo: the lhs already split (K-major, the lhs's own dense
// layout; spmd_local_all_gather_split) -- only the rhs is split here.
int dot_tf32x3(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
               const spmd_dot_dims& dd, int64_t nparts, cudaStream_t s,
               const float* lhs_hi = nullptr, const float* lhs_lo = nullptr,
               const float* rhs_hi = nullptr, const float* rhs_lo = nullptr);

#define SPMD_CHECK_ARG(cond, msg)                  \
  do {                                             \
    if (!(cond)) {                                 \
      ::spmd::set_error(msg);                      \
      return SPMD_ERR_INVALID;                     \
    }                                              \
  } while (0)

#define SPMD_CUDA_TRY(expr)                                                 \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      ::spmd::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      return SPMD_ERR_CUDA;                                                 \
    }                                                                       \
  } while (0)

inline int launched(cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("kernel launch: ") + cudaGetErrorString(e));
    return SPMD_ERR_CUDA;
  }
  (void)s;
  return SPMD_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// shapes
// ---------------------------------------------------------------------------
inline int64_t numel(const spmd_tensor& t) {
  int64_t n = 1;
  for (int i = 0; i < t.rank; ++i) n *= t.dims[i];
  return n;
}

inline int elem_size(int dtype) {
  switch (dtype) {
    case SPMD_F32: case SPMD_S32: case SPMD_U32: return 4;
    case SPMD_PRED: return 1;
    case SPMD_BF16: return 2;
  }
  return 0;
}

struct Shape8 {
  int rank;
  int64_t d[SPMD_MAX_RANK];
};

inline Shape8 shape_of(const spmd_tensor& t) {
  Shape8 s;
  s.rank = t.rank;
  for (int i = 0; i < SPMD_MAX_RANK; ++i) s.d[i] = i < t.rank ? t.dims[i] : 1;
  return s;
}

inline void row_strides(const Shape8& s, int64_t* st) {
  int64_t acc = 1;
  for (int i = s.rank - 1; i >= 0; --i) {
    st[i] = acc;
    acc *= s.d[i];
  }
}

// Grid for a grid-stride loop over n work items.
inline unsigned grid_for(int64_t n, int block, int per_thread = 1) {
  int64_t b = (n + (int64_t)block * per_thread - 1) / ((int64_t)block * per_thread);
  if (b < 1) b = 1;
  const int64_t cap = 148LL * 32;   // 148 SMs x enough resident blocks
  return (unsigned)(b < cap ? b : cap);
}

// ---------------------------------------------------------------------------
// element types
// ---------------------------------------------------------------------------
typedef __nv_bfloat16 bf16;

template <typename T> struct Compute { typedef T type; };
template <> struct Compute<bf16> { typedef float type; };

template <typename T> __device__ __forceinline__ typename Compute<T>::type ld(const T& v) { return v; }
template <> __device__ __forceinline__ float ld<bf16>(const bf16& v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T st(typename Compute<T>::type v) { return v; }
template <> __device__ __forceinline__ bf16 st<bf16>(float v) { return __float2bfloat16_rn(v); }

#define SPMD_DISPATCH(DT, T, ...)                                  \
  switch (DT) {                                                    \
    case SPMD_F32: { typedef float T; __VA_ARGS__; break; }        \
    case SPMD_S32: { typedef int32_t T; __VA_ARGS__; break; }      \
    case SPMD_U32: { typedef uint32_t T; __VA_ARGS__; break; }     \
    case SPMD_PRED: { typedef uint8_t T; __VA_ARGS__; break; }     \
    case SPMD_BF16: { typedef bf16 T; __VA_ARGS__; break; }        \
    default: set_error("bad dtype"); return SPMD_ERR_INVALID;     \
  }

// Dispatch on element byte size only (pure data movement).
#define SPMD_DISPATCH_BYTES(DT, T, ...)                            \
  switch (elem_size(DT)) {                                         \
    case 4: { typedef uint32_t T; __VA_ARGS__; break; }            \
    case 2: { typedef uint16_t T; __VA_ARGS__; break; }            \
    case 1: { typedef uint8_t T; __VA_ARGS__; break; }             \
    default: set_error("bad dtype"); return SPMD_ERR_INVALID;     \
  }

// NaN-propagating max/min (numpy semantics).
template <typename T> __device__ __forceinline__ T vmax(T a, T b) { return a > b ? a : b; }
template <typename T> __device__ __forceinline__ T vmin(T a, T b) { return a < b ? a : b; }
template <> __device__ __forceinline__ float vmax<float>(float a, float b) {
  return (a > b || a != a) ? a : b;
}
template <> __device__ __forceinline__ float vmin<float>(float a, float b) {
  return (a < b || a != a) ? a : b;
}

// Wrapping integer arithmetic (numpy int32 semantics).
template <typename T> __device__ __forceinline__ T wadd(T a, T b) { return a + b; }
template <typename T> __device__ __forceinline__ T wsub(T a, T b) { return a - b; }
template <typename T> __device__ __forceinline__ T wmul(T a, T b) { return a * b; }
template <> __device__ __forceinline__ int32_t wadd<int32_t>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}
template <> __device__ __forceinline__ int32_t wsub<int32_t>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a - (uint32_t)b);
}
template <> __device__ __forceinline__ int32_t wmul<int32_t>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a * (uint32_t)b);
}
template <> __device__ __forceinline__ uint8_t wadd<uint8_t>(uint8_t a, uint8_t b) { return a | b; }
template <> __device__ __forceinline__ uint8_t wmul<uint8_t>(uint8_t a, uint8_t b) { return a & b; }
template <> __device__ __forceinline__ uint8_t wsub<uint8_t>(uint8_t a, uint8_t b) { return a ^ b; }

// Reduction combiner.
template <typename C>
__device__ __forceinline__ C combine(int kind, C a, C b) {
  switch (kind) {
    case SPMD_SUM: return wadd<C>(a, b);
    case SPMD_MAX: return vmax<C>(a, b);
    case SPMD_MIN: return vmin<C>(a, b);
    default: return wmul<C>(a, b);
  }
}

// Unravel a linear index into coordinates (row-major).
template <typename I>
__device__ __forceinline__ void unravel(I idx, const Shape8& s, I* c) {
#pragma unroll
  for (int i = SPMD_MAX_RANK - 1; i >= 0; --i) {
    if (i < s.rank) {
      I di = (I)s.d[i];
      c[i] = idx % di;
      idx /= di;
    } else {
      c[i] = 0;
    }
  }
}

// Affine strided copy between two views (datamove.cu).
struct CopyArgs {
  int rank;
  int64_t shape[SPMD_MAX_RANK];
  int64_t sst[SPMD_MAX_RANK];
  int64_t dst[SPMD_MAX_RANK];
  int64_t sbase, dbase;        // element offsets
  int64_t spart, dpart;        // per-partition element strides
  int64_t n;                   // elements per partition
  // dynamic (per-partition) base: base += clamp(start[d][p], 0, dmax[d]) * dmul[d]
  int ndyn;
  const int32_t* dyn_start[SPMD_MAX_RANK];
  int64_t dyn_max[SPMD_MAX_RANK];
  int64_t dyn_mul[SPMD_MAX_RANK];
  int dyn_on_dst;
  // 1: every thread ends with __threadfence_system() -- the destination is a
  // peer's heap (NVLink stores) and a peer barrier follows (peer.cu)
  int fence_sys;
  // ReLU on the copied elements' bits (fused Transpose -> ReLU): 1 IEEE
  // float (f32 / bf16: negative or -0 -> +0, NaN kept, as UnaryF's vmax), 2
  // signed int
  int relu;
};

// 3xTF32 operand split: hi = x rounded to tf32, lo = x - hi (exact in f32;
// 0 for non-finite x), so hi + lo == x.  Shared by the GEMM's split passes
// and the loopback all-gather that writes the split directly.
__device__ __forceinline__ void split_tf32(float v, float& h, float& l) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v));
  h = __uint_as_float(u);
  l = isfinite(v) ? v - h : 0.f;
}

template <typename T>
__device__ __forceinline__ T relu_bits(T b, int mode) {
  constexpr int BITS = 8 * sizeof(T);
  if (BITS != 16 && BITS != 32) return b;
  const T sign = (T)((T)1 << (BITS - 1));
  if (!(b & sign)) return b;
  if (mode == 2) return (T)0;
  const T mag = (T)(b & (T)~sign);
  const T inf = BITS == 16 ? (T)0x7f80 : (T)0x7f800000u;
  return mag > inf ? b : (T)0;          // NaN stays
}

int launch_copy(const void* src, void* dst, int dtype, CopyArgs a, int64_t nparts,
                cudaStream_t s);

// Row-chunk streaming (HBM-bound data movement with long contiguous rows):
// a block owns 256 x ROW_U 16-byte vectors of one row, so the per-row index
// math (unravel, clamps, predicates) runs once per block instead of once per
// vector -- the per-vector 64-bit div / mod of the generic kernels made them
// instruction-bound at 79-86% of HBM bandwidth on C5's 2 MB rows.
constexpr int ROW_U = 4;
constexpr int64_t ROW_MIN_VECS = 2048;   // rows shorter than this use the generic kernels
inline unsigned row_grid(int64_t rows, int64_t chunks) {
  const int64_t b = rows * chunks;
  const int64_t cap = 148LL * 16;
  return (unsigned)(b < 1 ? 1 : (b < cap ? b : cap));
}
int launch_fill(void* out, const void* value, int dtype, int64_t n, int64_t nparts,
                cudaStream_t s);

}  // namespace spmd
