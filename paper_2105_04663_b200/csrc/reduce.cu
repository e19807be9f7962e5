// Reductions (reference simulator.py:242-257) and the fused row softmax.
//
// out[kept] = init (+) reduce_{reduced dims} in[...]; integer reductions wrap
// exactly like numpy; float reductions accumulate in fp32 (bf16 in fp32).
// Two schedules, both coalesced:
//  * the innermost input dim is reduced -> one warp per output element,
//    lanes stride along the contiguous run, shuffle tree at the end;
//  * the innermost input dim is kept -> one thread per output element,
//    threads of a warp read adjacent addresses at every reduction step.
#include "common.cuh"

#include <string.h>

namespace spmd {

struct ReduceArgs {
  int nk, nr;                        // kept / reduced dim counts
  int64_t kshape[SPMD_MAX_RANK], kst[SPMD_MAX_RANK];
  int64_t rshape[SPMD_MAX_RANK], rst[SPMD_MAX_RANK];
  int64_t nout, nred, in_part;       // per-partition sizes
  int kind;
};

template <typename I>
__device__ __forceinline__ int64_t offset_of(I idx, int n, const int64_t* shape,
                                             const int64_t* st) {
  int64_t off = 0;
#pragma unroll
  for (int k = SPMD_MAX_RANK - 1; k >= 0; --k) {
    if (k < n) {
      I d = (I)shape[k];
      off += (int64_t)(idx % d) * st[k];
      idx /= d;
    }
  }
  return off;
}

template <typename C>
__device__ __forceinline__ C identity(int kind);
template <> __device__ __forceinline__ float identity<float>(int kind) {
  return kind == SPMD_SUM ? 0.f : kind == SPMD_PROD ? 1.f : kind == SPMD_MAX ? -INFINITY : INFINITY;
}
template <> __device__ __forceinline__ int32_t identity<int32_t>(int kind) {
  return kind == SPMD_SUM ? 0 : kind == SPMD_PROD ? 1 : kind == SPMD_MAX ? INT32_MIN : INT32_MAX;
}
template <> __device__ __forceinline__ uint32_t identity<uint32_t>(int kind) {
  return kind == SPMD_SUM ? 0u : kind == SPMD_PROD ? 1u : kind == SPMD_MAX ? 0u : 0xffffffffu;
}
template <> __device__ __forceinline__ uint8_t identity<uint8_t>(int kind) {
  return kind == SPMD_SUM ? 0 : kind == SPMD_PROD ? 1 : kind == SPMD_MAX ? 0 : 1;
}

template <typename T>
__device__ __forceinline__ typename Compute<T>::type shfl_combine(int kind,
                                                                  typename Compute<T>::type v) {
  typedef typename Compute<T>::type C;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    C w = __shfl_xor_sync(0xffffffffu, v, o);
    v = combine<C>(kind, v, w);
  }
  return v;
}

template <typename T>
__global__ void reduce_warp_kernel(const T* __restrict__ in, const T* __restrict__ init,
                                   T* __restrict__ out, ReduceArgs a, int64_t nparts) {
  typedef typename Compute<T>::type C;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = a.nout * nparts;
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += warps) {
    int64_t p = w / a.nout, o = w - p * a.nout;
    const T* base = in + p * a.in_part + offset_of<int64_t>(o, a.nk, a.kshape, a.kst);
    C acc = identity<C>(a.kind);
    for (int64_t r = lane; r < a.nred; r += 32)
      acc = combine<C>(a.kind, acc, ld<T>(base[offset_of<int64_t>(r, a.nr, a.rshape, a.rst)]));
    acc = shfl_combine<T>(a.kind, acc);
    if (lane == 0) out[w] = st<T>(combine<C>(a.kind, acc, ld<T>(init[p])));
  }
}

template <typename T>
__global__ void reduce_thread_kernel(const T* __restrict__ in, const T* __restrict__ init,
                                     T* __restrict__ out, ReduceArgs a, int64_t nparts) {
  typedef typename Compute<T>::type C;
  const int64_t total = a.nout * nparts;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = w / a.nout, o = w - p * a.nout;
    const T* base = in + p * a.in_part + offset_of<int64_t>(o, a.nk, a.kshape, a.kst);
    C acc = identity<C>(a.kind);
    for (int64_t r = 0; r < a.nred; ++r)
      acc = combine<C>(a.kind, acc, ld<T>(base[offset_of<int64_t>(r, a.nr, a.rshape, a.rst)]));
    out[w] = st<T>(combine<C>(a.kind, acc, ld<T>(init[p])));
  }
}

// Float reduction of a contiguous trailing run (the reduced dims are the
// innermost ones): one warp per output, 16-byte loads, fp32 accumulation.
template <typename T>
__global__ void __launch_bounds__(256) reduce_rows_vec_kernel(const T* __restrict__ in,
                                                             const T* __restrict__ init,
                                                             T* __restrict__ out, int64_t rows,
                                                             int64_t L, int64_t rows_per_part,
                                                             int kind) {
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const uint4* x = reinterpret_cast<const uint4*>(in + row * L);
    float acc = identity<float>(kind);
    for (int64_t c = lane; c < L / V; c += 32) {
      const uint4 w = __ldcs(x + c);
      const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
      for (int j = 0; j < V; ++j) acc = combine<float>(kind, acc, ld<T>(e[j]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = combine<float>(kind, acc, __shfl_xor_sync(~0u, acc, o));
    if (lane == 0) out[row] = st<T>(combine<float>(kind, acc, ld<T>(init[row / rows_per_part])));
  }
}

// Row softmax over a contiguous last dim of length L: one warp per row, the
// row held in registers when L <= 32*32, else three streaming passes.
template <typename T, int PER_LANE>
__global__ void softmax_rows_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t rows,
                                    int64_t L) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const T* x = in + row * L;
    T* y = out + row * L;
    float m = -INFINITY;
    if (PER_LANE > 0) {
      float v[PER_LANE > 0 ? PER_LANE : 1];
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j) {
        int64_t c = lane + 32 * j;
        v[j] = c < L ? ld<T>(x[c]) : -INFINITY;
        m = vmax<float>(m, v[j]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = vmax<float>(m, __shfl_xor_sync(0xffffffffu, m, o));
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j) {
        int64_t c = lane + 32 * j;
        v[j] = c < L ? expf(v[j] - m) : 0.f;
        s += v[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j) {
        int64_t c = lane + 32 * j;
        if (c < L) y[c] = st<T>(v[j] / s);
      }
    } else {
      for (int64_t c = lane; c < L; c += 32) m = vmax<float>(m, ld<T>(x[c]));
      for (int o = 16; o > 0; o >>= 1) m = vmax<float>(m, __shfl_xor_sync(0xffffffffu, m, o));
      float s = 0.f;
      for (int64_t c = lane; c < L; c += 32) s += expf(ld<T>(x[c]) - m);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      for (int64_t c = lane; c < L; c += 32) y[c] = st<T>(expf(ld<T>(x[c]) - m) / s);
    }
  }
}

// Vectorised row softmax for contiguous rows with L % 8 == 0 and
// L <= 256 * CH: each lane owns CH 16-byte chunks (8 bf16 each) of its row,
// the row never leaves registers, exp is ex2.approx on log2e-prescaled
// inputs and the normalisation is one reciprocal.  One HBM read + one write
// per element.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int CH>
__global__ void __launch_bounds__(256, 4)
    softmax_rows_bf16_vec(const bf16* __restrict__ in, bf16* __restrict__ out, int64_t rows,
                          int L) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const float LOG2E = 1.4426950408889634f;
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const uint4* x = reinterpret_cast<const uint4*>(in + row * L);
    uint4* y = reinterpret_cast<uint4*>(out + row * L);
    const int nch = L >> 3;
    uint4 raw[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      int c = lane + 32 * i;
      raw[i] = c < nch ? __ldcs(x + c) : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u,
                                                      0xff80ff80u);   // -inf
    }
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        m = vmax<float>(m, vmax<float>(f.x, f.y));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = vmax<float>(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float mb = (m == -INFINITY) ? 0.f : m * LOG2E;
    float v[CH][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        v[i][2 * j] = fast_exp2(fmaf(f.x, LOG2E, -mb));
        v[i][2 * j + 1] = fast_exp2(fmaf(f.y, LOG2E, -mb));
        s += v[i][2 * j] + v[i][2 * j + 1];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float r = 1.f / s;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      int c = lane + 32 * i;
      if (c < nch) {
        uint4 o4;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o4);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          h[j] = __floats2bfloat162_rn(v[i][2 * j] * r, v[i][2 * j + 1] * r);
        __stcs(y + c, o4);
      }
    }
  }
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_reduce(spmd_tensor in, spmd_tensor init, spmd_tensor out, const int32_t* dims,
                           int ndims, int kind, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && init.dtype == in.dtype && init.rank == 0,
                 "reduce dtype mismatch");
  SPMD_CHECK_ARG(kind >= 0 && kind <= 3, "bad reduce kind");
  bool red[SPMD_MAX_RANK] = {false};
  for (int i = 0; i < ndims; ++i) {
    SPMD_CHECK_ARG(dims[i] >= 0 && dims[i] < in.rank, "reduce dim out of range");
    red[dims[i]] = true;
  }
  ReduceArgs a;
  memset(&a, 0, sizeof(a));
  a.kind = kind;
  int64_t st_[SPMD_MAX_RANK];
  int64_t acc = 1;
  for (int k = in.rank - 1; k >= 0; --k) {
    st_[k] = acc;
    acc *= in.dims[k];
  }
  a.in_part = acc;
  a.nout = a.nred = 1;
  for (int k = 0; k < in.rank; ++k) {
    if (red[k]) {
      a.rshape[a.nr] = in.dims[k];
      a.rst[a.nr++] = st_[k];
      a.nred *= in.dims[k];
    } else {
      a.kshape[a.nk] = in.dims[k];
      a.kst[a.nk++] = st_[k];
      a.nout *= in.dims[k];
    }
  }
  SPMD_CHECK_ARG(a.nout == numel(out), "reduce output shape mismatch");
  if (a.nout * nparts == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  const bool inner_reduced = in.rank > 0 && red[in.rank - 1];
  // reduced dims == a contiguous trailing run -> rows of length nred
  bool trailing = inner_reduced;
  for (int k = 0; k < in.rank; ++k) trailing = trailing && (red[k] == (k >= in.rank - ndims));
  if (trailing && (in.dtype == SPMD_BF16 || in.dtype == SPMD_F32)) {
    const int V = 16 / elem_size(in.dtype);
    if (a.nred % V == 0 && (reinterpret_cast<uintptr_t>(in.data) & 15) == 0) {
      const int64_t rows = a.nout * nparts;
      if (in.dtype == SPMD_BF16)
        reduce_rows_vec_kernel<bf16><<<grid_for(rows * 32, 256), 256, 0, s>>>(
            (const bf16*)in.data, (const bf16*)init.data, (bf16*)out.data, rows, a.nred, a.nout,
            kind);
      else
        reduce_rows_vec_kernel<float><<<grid_for(rows * 32, 256), 256, 0, s>>>(
            (const float*)in.data, (const float*)init.data, (float*)out.data, rows, a.nred,
            a.nout, kind);
      return launched(s);
    }
  }
  SPMD_DISPATCH(in.dtype, T, {
    if (inner_reduced || a.nout * nparts < 148 * 64) {
      int64_t warps = a.nout * nparts;
      reduce_warp_kernel<T><<<grid_for(warps * 32, 256), 256, 0, s>>>(
          (const T*)in.data, (const T*)init.data, (T*)out.data, a, nparts);
    } else {
      reduce_thread_kernel<T><<<grid_for(a.nout * nparts, 256), 256, 0, s>>>(
          (const T*)in.data, (const T*)init.data, (T*)out.data, a, nparts);
    }
  });
  return launched(s);
}

// Softmax backward over rows: out = p * (dp - sum_row(dp * p)), bf16 rows in
// registers (one warp per row, 16-byte loads), fp32 row sum -- the
// multiply / reduce / broadcast / subtract / multiply chain of the training
// graph in one pass (reads p and dp once, writes out once).
template <int CH>
__global__ void __launch_bounds__(256, 4)
    softmax_bwd_rows_bf16(const bf16* __restrict__ p, const bf16* __restrict__ dp,
                          bf16* __restrict__ out, int64_t rows, int L) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const uint4* pp = reinterpret_cast<const uint4*>(p + row * L);
    const uint4* gg = reinterpret_cast<const uint4*>(dp + row * L);
    uint4* y = reinterpret_cast<uint4*>(out + row * L);
    const int nch = L >> 3;
    uint4 rp[CH], rg[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = lane + 32 * i;
      rp[i] = c < nch ? __ldcs(pp + c) : make_uint4(0, 0, 0, 0);
      rg[i] = c < nch ? __ldcs(gg + c) : make_uint4(0, 0, 0, 0);
    }
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&rp[i]);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&rg[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fa = __bfloat1622float2(a[j]), fb = __bfloat1622float2(b[j]);
        sum = fmaf(fa.x, fb.x, fmaf(fa.y, fb.y, sum));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = lane + 32 * i;
      if (c >= nch) continue;
      const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&rp[i]);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&rg[i]);
      uint4 o;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fa = __bfloat1622float2(a[j]), fb = __bfloat1622float2(b[j]);
        h[j] = __floats2bfloat162_rn(fa.x * (fb.x - sum), fa.y * (fb.y - sum));
      }
      __stcs(y + c, o);
    }
  }
}

// Any row length / alignment / float dtype: warp per row, two passes.
template <typename T>
__global__ void softmax_bwd_rows_kernel(const T* __restrict__ p, const T* __restrict__ dp,
                                        T* __restrict__ out, int64_t rows, int64_t L) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const T* a = p + row * L;
    const T* b = dp + row * L;
    float sum = 0.f;
    for (int64_t i = lane; i < L; i += 32) sum = fmaf(ld<T>(a[i]), ld<T>(b[i]), sum);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    for (int64_t i = lane; i < L; i += 32) out[row * L + i] = st<T>(ld<T>(a[i]) * (ld<T>(b[i]) - sum));
  }
}

extern "C" int spmd_softmax_backward_lastdim(spmd_tensor p, spmd_tensor dp, spmd_tensor out,
                                             int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(p.dtype == dp.dtype && p.dtype == out.dtype &&
                     (p.dtype == SPMD_BF16 || p.dtype == SPMD_F32) && p.rank >= 1 &&
                     numel(p) == numel(dp) && numel(p) == numel(out),
                 "softmax backward expects bf16/f32 p, dp, out of one shape");
  const int64_t L = p.dims[p.rank - 1];
  const int64_t rows = L ? numel(p) / L * nparts : 0;
  if (rows == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  if (p.dtype == SPMD_F32 || L % 8 || L > 1024 || (reinterpret_cast<uintptr_t>(p.data) & 15) ||
      (reinterpret_cast<uintptr_t>(dp.data) & 15) || (reinterpret_cast<uintptr_t>(out.data) & 15)) {
    const unsigned grid = grid_for(rows * 32, 256);
    if (p.dtype == SPMD_F32)
      softmax_bwd_rows_kernel<float><<<grid, 256, 0, s>>>((const float*)p.data,
                                                          (const float*)dp.data,
                                                          (float*)out.data, rows, L);
    else
      softmax_bwd_rows_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)p.data, (const bf16*)dp.data,
                                                         (bf16*)out.data, rows, L);
    return launched(s);
  }
  const unsigned grid = grid_for(rows * 32, 256);
  const bf16 *a = (const bf16*)p.data, *b = (const bf16*)dp.data;
  bf16* o = (bf16*)out.data;
  if (L <= 256)
    softmax_bwd_rows_bf16<1><<<grid, 256, 0, s>>>(a, b, o, rows, (int)L);
  else if (L <= 512)
    softmax_bwd_rows_bf16<2><<<grid, 256, 0, s>>>(a, b, o, rows, (int)L);
  else
    softmax_bwd_rows_bf16<4><<<grid, 256, 0, s>>>(a, b, o, rows, (int)L);
  return launched(s);
}

extern "C" int spmd_softmax_lastdim(spmd_tensor in, spmd_tensor out, int64_t nparts,
                                    void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && (in.dtype == SPMD_F32 || in.dtype == SPMD_BF16) &&
                     in.rank >= 1 && numel(in) == numel(out),
                 "softmax expects f32/bf16 with rank >= 1");
  int64_t L = in.dims[in.rank - 1];
  int64_t rows = L ? numel(in) / L * nparts : 0;
  if (rows == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  unsigned grid = grid_for(rows * 32, 256);
  if (in.dtype == SPMD_BF16 && L % 8 == 0 && L <= 256 * 4 &&
      (reinterpret_cast<uintptr_t>(in.data) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out.data) & 15) == 0) {
    if (L <= 256)
      softmax_rows_bf16_vec<1><<<grid, 256, 0, s>>>((const bf16*)in.data, (bf16*)out.data, rows,
                                                    (int)L);
    else if (L <= 512)
      softmax_rows_bf16_vec<2><<<grid, 256, 0, s>>>((const bf16*)in.data, (bf16*)out.data, rows,
                                                    (int)L);
    else
      softmax_rows_bf16_vec<4><<<grid, 256, 0, s>>>((const bf16*)in.data, (bf16*)out.data, rows,
                                                    (int)L);
    return launched(s);
  }
#define SOFTMAX_LAUNCH(T)                                                                        \
  if (L <= 32 * 8)                                                                               \
    softmax_rows_kernel<T, 8><<<grid, 256, 0, s>>>((const T*)in.data, (T*)out.data, rows, L);   \
  else if (L <= 32 * 32)                                                                         \
    softmax_rows_kernel<T, 32><<<grid, 256, 0, s>>>((const T*)in.data, (T*)out.data, rows, L);  \
  else                                                                                           \
    softmax_rows_kernel<T, 0><<<grid, 256, 0, s>>>((const T*)in.data, (T*)out.data, rows, L);
  if (in.dtype == SPMD_F32) {
    SOFTMAX_LAUNCH(float)
  } else {
    SOFTMAX_LAUNCH(bf16)
  }
#undef SOFTMAX_LAUNCH
  return launched(s);
}
