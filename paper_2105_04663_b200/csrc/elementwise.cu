// Sources and elementwise ops (reference simulator.py:161-198).
// HBM-bound: 16-byte vectorised grid-stride loops over the partition-stacked
// buffers; numpy semantics (wrapping ints, NaN-propagating max, IEEE divide,
// C-truncating int divide with a device error flag on division by zero).
#include "common.cuh"

#include <math.h>
#include <string.h>

namespace spmd {

template <typename T, int V>
struct alignas(sizeof(T) * V) Vec {
  T v[V];
};

template <typename T>
constexpr int vec_width() { return 16 / sizeof(T) > 0 ? 16 / sizeof(T) : 1; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------------------
// sources
// ---------------------------------------------------------------------------
template <typename T, typename I>
__global__ void iota_kernel(T* out, I total, I inner, I len) {
  for (I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    I v = (i / inner) % len;
    out[i] = st<T>((typename Compute<T>::type)v);
  }
}

__global__ void partition_id_kernel(int32_t* out, int64_t nparts, int32_t first) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nparts) out[i] = first + (int32_t)i;
}

template <typename T>
__global__ void tile_kernel(const T* __restrict__ src, T* __restrict__ out, int64_t n,
                            int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[i % n];
}

// ---------------------------------------------------------------------------
// elementwise functors
// ---------------------------------------------------------------------------
template <typename T>
struct UnaryF {
  int op;
  __device__ __forceinline__ T operator()(T x) const {
    typedef typename Compute<T>::type C;
    C a = ld<T>(x);
    C r;
    if (op == SPMD_NEGATE) {
      r = wsub<C>((C)0, a);
    } else if (op == SPMD_EXP) {
      r = (C)expf((float)a);
    } else {
      r = vmax<C>(a, (C)0);
    }
    return st<T>(r);
  }
};

template <>
struct UnaryF<int32_t> {
  int op;
  __device__ __forceinline__ int32_t operator()(int32_t a) const {
    if (op == SPMD_NEGATE) return wsub<int32_t>(0, a);
    if (op == SPMD_EXP) return (int32_t)exp((double)a);
    return a > 0 ? a : 0;
  }
};

__device__ __forceinline__ float bdiv(float a, float b, int*) { return a / b; }
__device__ __forceinline__ int32_t bdiv(int32_t a, int32_t b, int* err) {
  if (b == 0) {
    atomicOr(err, 1);
    return 0;
  }
  return (int32_t)((int64_t)a / (int64_t)b);   // C truncation toward zero
}
__device__ __forceinline__ uint32_t bdiv(uint32_t a, uint32_t b, int* err) {
  if (b == 0) {
    atomicOr(err, 1);
    return 0;
  }
  return a / b;
}
__device__ __forceinline__ uint8_t bdiv(uint8_t a, uint8_t b, int* err) {
  if (b == 0) {
    atomicOr(err, 1);
    return 0;
  }
  return a / b;
}

template <typename T>
struct BinaryF {
  int op, cmp;
  int* err;
  __device__ __forceinline__ T operator()(T x, T y) const {
    typedef typename Compute<T>::type C;
    C a = ld<T>(x), b = ld<T>(y);
    switch (op) {
      case SPMD_ADD: return st<T>(wadd<C>(a, b));
      case SPMD_MULTIPLY: return st<T>(wmul<C>(a, b));
      case SPMD_MAXIMUM: return st<T>(vmax<C>(a, b));
      case SPMD_SUBTRACT: return st<T>(wsub<C>(a, b));
      default: return st<T>(bdiv(a, b, err));
    }
  }
};

template <typename T>
struct CompareF {
  int cmp;
  __device__ __forceinline__ uint8_t operator()(T x, T y) const {
    typedef typename Compute<T>::type C;
    C a = ld<T>(x), b = ld<T>(y);
    switch (cmp) {
      case SPMD_EQ: return a == b;
      case SPMD_NE: return a != b;
      case SPMD_LT: return a < b;
      case SPMD_LE: return a <= b;
      case SPMD_GT: return a > b;
      default: return a >= b;
    }
  }
};

// ---------------------------------------------------------------------------
// vectorised drivers
// ---------------------------------------------------------------------------
template <typename T, typename R, int V, typename F>
__global__ void map1_kernel(const T* __restrict__ a, R* __restrict__ out, int64_t n, F f) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = n / V;
  for (int64_t i = tid; i < nv; i += step) {
    Vec<T, V> x = reinterpret_cast<const Vec<T, V>*>(a)[i];
    Vec<R, V> r;
#pragma unroll
    for (int j = 0; j < V; ++j) r.v[j] = f(x.v[j]);
    reinterpret_cast<Vec<R, V>*>(out)[i] = r;
  }
  for (int64_t i = nv * V + tid; i < n; i += step) out[i] = f(a[i]);
}

template <typename T, typename R, int V, typename F>
__global__ void map2_kernel(const T* __restrict__ a, const T* __restrict__ b, R* __restrict__ out,
                            int64_t n, F f) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = n / V;
  for (int64_t i = tid; i < nv; i += step) {
    Vec<T, V> x = reinterpret_cast<const Vec<T, V>*>(a)[i];
    Vec<T, V> y = reinterpret_cast<const Vec<T, V>*>(b)[i];
    Vec<R, V> r;
#pragma unroll
    for (int j = 0; j < V; ++j) r.v[j] = f(x.v[j], y.v[j]);
    reinterpret_cast<Vec<R, V>*>(out)[i] = r;
  }
  for (int64_t i = nv * V + tid; i < n; i += step) out[i] = f(a[i], b[i]);
}

template <typename T, int V>
__global__ void select_kernel(const uint8_t* __restrict__ p, const T* __restrict__ a,
                              const T* __restrict__ b, T* __restrict__ out, int64_t n) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += step) out[i] = p[i] ? a[i] : b[i];
}

template <typename TI, typename TO>
__global__ void convert_kernel(const TI* __restrict__ in, TO* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = st<TO>((typename Compute<TO>::type)ld<TI>(in[i]));
  }
}

template <typename T, typename R, typename F>
int launch_map1(const void* a, void* out, int64_t n, F f, cudaStream_t s) {
  constexpr int V = vec_width<T>() < vec_width<R>() ? vec_width<T>() : vec_width<R>();
  if (aligned16(a) && aligned16(out))
    map1_kernel<T, R, V><<<grid_for(n, 256, V * 2), 256, 0, s>>>((const T*)a, (R*)out, n, f);
  else
    map1_kernel<T, R, 1><<<grid_for(n, 256, 4), 256, 0, s>>>((const T*)a, (R*)out, n, f);
  return launched(s);
}

template <typename T, typename R, typename F>
int launch_map2(const void* a, const void* b, void* out, int64_t n, F f, cudaStream_t s) {
  constexpr int V = vec_width<T>() < vec_width<R>() ? vec_width<T>() : vec_width<R>();
  if (aligned16(a) && aligned16(b) && aligned16(out))
    map2_kernel<T, R, V><<<grid_for(n, 256, V * 2), 256, 0, s>>>((const T*)a, (const T*)b,
                                                                  (R*)out, n, f);
  else
    map2_kernel<T, R, 1><<<grid_for(n, 256, 4), 256, 0, s>>>((const T*)a, (const T*)b,
                                                             (R*)out, n, f);
  return launched(s);
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_iota(spmd_tensor out, int axis, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(axis >= 0 && axis < out.rank, "iota axis out of range");
  int64_t n = numel(out), total = n * nparts;
  if (total == 0) return SPMD_OK;
  int64_t inner = 1;
  for (int i = axis + 1; i < out.rank; ++i) inner *= out.dims[i];
  cudaStream_t s = as_stream(stream);
  const bool small = total < ((int64_t)1 << 31);
  SPMD_DISPATCH(out.dtype, T, {
    if (small)
      iota_kernel<T, uint32_t><<<grid_for(total, 256, 4), 256, 0, s>>>(
          (T*)out.data, (uint32_t)total, (uint32_t)inner, (uint32_t)out.dims[axis]);
    else
      iota_kernel<T, uint64_t><<<grid_for(total, 256, 4), 256, 0, s>>>(
          (T*)out.data, (uint64_t)total, (uint64_t)inner, (uint64_t)out.dims[axis]);
  });
  return launched(s);
}

extern "C" int spmd_partition_id(spmd_tensor out, int64_t nparts, int32_t first_id,
                                 void* stream) {
  SPMD_CHECK_ARG(out.dtype == SPMD_S32 && out.rank == 0, "partition-id must be s32[]");
  cudaStream_t s = as_stream(stream);
  partition_id_kernel<<<(unsigned)((nparts + 127) / 128), 128, 0, s>>>((int32_t*)out.data, nparts,
                                                                       first_id);
  return launched(s);
}

extern "C" int spmd_constant(spmd_tensor lit, spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(lit.dtype == out.dtype && numel(lit) == numel(out), "constant shape mismatch");
  int64_t n = numel(out);
  if (n == 0 || nparts == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  size_t bytes = (size_t)n * elem_size(out.dtype);
  SPMD_CUDA_TRY(cudaMemcpyAsync(out.data, lit.data, bytes, cudaMemcpyHostToDevice, s));
  if (nparts > 1) {
    SPMD_DISPATCH_BYTES(out.dtype, T,
                        tile_kernel<T><<<grid_for(n * nparts, 256, 4), 256, 0, s>>>(
                            (const T*)out.data, (T*)out.data + n, n, n * (nparts - 1)));
    return launched(s);
  }
  return SPMD_OK;
}

extern "C" int spmd_unary(int op, spmd_tensor in, spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && numel(in) == numel(out), "unary shape mismatch");
  SPMD_CHECK_ARG(op >= 0 && op <= 2, "bad unary op");
  int64_t n = numel(in) * nparts;
  if (n == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  SPMD_DISPATCH(in.dtype, T, return launch_map1<T, T>(in.data, out.data, n, UnaryF<T>{op}, s));
  return SPMD_OK;
}

extern "C" int spmd_binary(int op, int cmp, spmd_tensor a, spmd_tensor b, spmd_tensor out,
                           int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(a.dtype == b.dtype && numel(a) == numel(b) && numel(a) == numel(out),
                 "binary shape mismatch");
  int64_t n = numel(a) * nparts;
  if (n == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  if (op == SPMD_COMPARE) {
    SPMD_CHECK_ARG(out.dtype == SPMD_PRED, "compare output must be pred");
    SPMD_DISPATCH(a.dtype, T,
                  return launch_map2<T, uint8_t>(a.data, b.data, out.data, n, CompareF<T>{cmp}, s));
  }
  SPMD_CHECK_ARG(out.dtype == a.dtype, "binary dtype mismatch");
  SPMD_CHECK_ARG(op >= 0 && op <= 4, "bad binary op");
  int* err = device_error_word();
  if (!err) return SPMD_ERR_CUDA;
  SPMD_DISPATCH(a.dtype, T,
                return launch_map2<T, T>(a.data, b.data, out.data, n, BinaryF<T>{op, cmp, err}, s));
  return SPMD_OK;
}

extern "C" int spmd_select(spmd_tensor pred, spmd_tensor a, spmd_tensor b, spmd_tensor out,
                           int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(pred.dtype == SPMD_PRED && a.dtype == b.dtype && a.dtype == out.dtype,
                 "select dtype mismatch");
  int64_t n = numel(out) * nparts;
  SPMD_CHECK_ARG(numel(pred) * nparts == n && numel(a) * nparts == n, "select shape mismatch");
  if (n == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  SPMD_DISPATCH_BYTES(a.dtype, T,
                      select_kernel<T, 1><<<grid_for(n, 256, 4), 256, 0, s>>>(
                          (const uint8_t*)pred.data, (const T*)a.data, (const T*)b.data,
                          (T*)out.data, n));
  return launched(s);
}

extern "C" int spmd_convert(spmd_tensor in, spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(numel(in) == numel(out), "convert shape mismatch");
  int64_t n = numel(in) * nparts;
  if (n == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  if (in.dtype == SPMD_F32 && out.dtype == SPMD_BF16) {
    convert_kernel<float, bf16><<<grid_for(n, 256, 4), 256, 0, s>>>((const float*)in.data,
                                                                    (bf16*)out.data, n);
  } else if (in.dtype == SPMD_BF16 && out.dtype == SPMD_F32) {
    convert_kernel<bf16, float><<<grid_for(n, 256, 4), 256, 0, s>>>((const bf16*)in.data,
                                                                    (float*)out.data, n);
  } else {
    set_error("unsupported conversion");
    return SPMD_ERR_UNSUPPORTED;
  }
  return launched(s);
}

// ReLU backward: out = h > 0 ? g : 0 -- the compare / broadcast-zero / select
// chain of the training graph in one pass (16-byte vectors for bf16/f32).
template <typename T, int V>
__global__ void relu_bwd_kernel(const T* __restrict__ h, const T* __restrict__ g,
                                T* __restrict__ out, int64_t n) {
  const int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (V == 1) {
      out[i] = ld<T>(h[i]) > 0.f ? g[i] : st<T>(0.f);
    } else {
      const uint4 hv = __ldcs(reinterpret_cast<const uint4*>(h) + i);
      const uint4 gv = __ldcs(reinterpret_cast<const uint4*>(g) + i);
      uint4 ov;
      const T* hh = reinterpret_cast<const T*>(&hv);
      const T* gg = reinterpret_cast<const T*>(&gv);
      T* oo = reinterpret_cast<T*>(&ov);
#pragma unroll
      for (int j = 0; j < V; ++j) oo[j] = ld<T>(hh[j]) > 0.f ? gg[j] : st<T>(0.f);
      __stcs(reinterpret_cast<uint4*>(out) + i, ov);
    }
  }
}

extern "C" int spmd_relu_backward(spmd_tensor h, spmd_tensor g, spmd_tensor out, int64_t nparts,
                                  void* stream) {
  SPMD_CHECK_ARG(h.dtype == g.dtype && h.dtype == out.dtype &&
                     (h.dtype == SPMD_BF16 || h.dtype == SPMD_F32) && numel(h) == numel(g) &&
                     numel(h) == numel(out),
                 "relu backward expects bf16/f32 h, g, out of one shape");
  const int64_t n = numel(h) * nparts;
  if (n == 0) return SPMD_OK;
  const int V = 16 / elem_size(h.dtype);
  cudaStream_t s = as_stream(stream);
  if (n % V || (reinterpret_cast<uintptr_t>(h.data) & 15) ||
      (reinterpret_cast<uintptr_t>(g.data) & 15) || (reinterpret_cast<uintptr_t>(out.data) & 15)) {
    if (h.dtype == SPMD_BF16)
      relu_bwd_kernel<bf16, 1><<<grid_for(n, 256), 256, 0, s>>>(
          (const bf16*)h.data, (const bf16*)g.data, (bf16*)out.data, n);
    else
      relu_bwd_kernel<float, 1><<<grid_for(n, 256), 256, 0, s>>>(
          (const float*)h.data, (const float*)g.data, (float*)out.data, n);
    return launched(s);
  }
  if (h.dtype == SPMD_BF16)
    relu_bwd_kernel<bf16, 8><<<grid_for(n / 8, 256), 256, 0, s>>>(
        (const bf16*)h.data, (const bf16*)g.data, (bf16*)out.data, n);
  else
    relu_bwd_kernel<float, 4><<<grid_for(n / 4, 256), 256, 0, s>>>(
        (const float*)h.data, (const float*)g.data, (float*)out.data, n);
  return launched(s);
}
