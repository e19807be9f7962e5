// Data-movement ops (reference simulator.py:199-241, 278-300): broadcast,
// transpose, reverse, pad, slice, dynamic-slice, dynamic-update-slice, concat,
// rotate, shift.
//
// Every one of them is an *affine* copy between two strided views
//   dst[dbase(p) + sum_d c_d * dstride_d] = src[sbase(p) + sum_d c_d * sstride_d]
// (negative strides for reverse, stride*(interior+1) for pad, a per-partition
// clamped base for dynamic slices), optionally preceded by a per-partition
// scalar fill.  The host side merges dims that are contiguous in both views
// and drops unit dims, so most copies run with 1-3 dims of index math; when
// the innermost dim is unit-stride on both sides and 16-byte aligned the
// kernel moves 16 bytes per thread.  Pure HBM-bound work.
#include "common.cuh"

#include <string.h>

namespace spmd {


// SPLAT: the innermost dim broadcasts one source element (source stride 0);
// each 16-byte output group repeats it.
template <typename T, typename I, int V, bool SPLAT = false>
__global__ void strided_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, CopyArgs a,
                                    int64_t nparts) {
  const I per = (I)(a.n / V);
  const I total = per * (I)nparts;
  // Per-partition dynamic base offsets (clamped starts), computed once per
  // block instead of re-reading the start scalars for every element.
  __shared__ int64_t dyn_off[SPMD_MAX_PARTS];
  if (a.ndyn) {
    for (int p = threadIdx.x; p < nparts && p < SPMD_MAX_PARTS; p += blockDim.x) {
      int64_t off = 0;
      for (int k = 0; k < a.ndyn; ++k) {
        int64_t s0 = a.dyn_start[k][p];
        s0 = s0 < 0 ? 0 : (s0 > a.dyn_max[k] ? a.dyn_max[k] : s0);
        off += s0 * a.dyn_mul[k];
      }
      dyn_off[p] = off;
    }
    __syncthreads();
  }
  for (I idx = blockIdx.x * (I)blockDim.x + threadIdx.x; idx < total;
       idx += (I)gridDim.x * blockDim.x) {
    I p = idx / per;
    I r = (idx - p * per) * V;
    int64_t so = a.sbase + (int64_t)p * a.spart;
    int64_t d0 = a.dbase + (int64_t)p * a.dpart;
#pragma unroll
    for (int k = SPMD_MAX_RANK - 1; k >= 0; --k) {
      if (k < a.rank) {
        I dk = (I)a.shape[k];
        I c = r % dk;
        r /= dk;
        so += (int64_t)c * a.sst[k];
        d0 += (int64_t)c * a.dst[k];
      }
    }
    if (a.ndyn) {
      const int64_t off = dyn_off[p];
      if (a.dyn_on_dst) d0 += off; else so += off;
    }
    if (V == 1) {
      dst[d0] = a.relu ? relu_bits<T>(src[so], a.relu) : src[so];
    } else if (SPLAT) {
      const T v = src[so];
      T f[V];
#pragma unroll
      for (int j = 0; j < V; ++j) f[j] = v;
      *reinterpret_cast<uint4*>(dst + d0) = *reinterpret_cast<uint4*>(f);
    } else if (a.relu) {
      uint4 w = *reinterpret_cast<const uint4*>(src + so);
      T* e = reinterpret_cast<T*>(&w);
#pragma unroll
      for (int j = 0; j < V; ++j) e[j] = relu_bits<T>(e[j], a.relu);
      *reinterpret_cast<uint4*>(dst + d0) = w;
    } else {
      *reinterpret_cast<uint4*>(dst + d0) = *reinterpret_cast<const uint4*>(src + so);
    }
  }
  if (a.fence_sys) __threadfence_system();
}

// Row-chunk variant of strided_copy_kernel for a contiguous innermost dim of
// >= ROW_MIN_VECS vectors: rows = nparts x (outer dims); each block handles
// 256 x ROW_U vectors of one row with ROW_U independent loads in flight.
template <typename T>
__global__ void __launch_bounds__(256) row_copy_kernel(const T* __restrict__ src,
                                                       T* __restrict__ dst, CopyArgs a,
                                                       int64_t nparts, int64_t chunks) {
  constexpr int V = 16 / sizeof(T);
  const int r = a.rank - 1;                    // dim r is the row (contiguous on both sides)
  const int64_t per_row = a.shape[r] / V;
  int64_t rows_per_part = 1;
  for (int k = 0; k < r; ++k) rows_per_part *= a.shape[k];
  const int64_t rows = rows_per_part * nparts;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks, chunk = b - row * chunks;
    const int64_t p = row / rows_per_part;
    int64_t q = row - p * rows_per_part;
    int64_t so = a.sbase + p * a.spart, d0 = a.dbase + p * a.dpart;
    for (int k = r - 1; k >= 0; --k) {
      const int64_t c = q % a.shape[k];
      q /= a.shape[k];
      so += c * a.sst[k];
      d0 += c * a.dst[k];
    }
    for (int k = 0; k < a.ndyn; ++k) {
      int64_t s0 = a.dyn_start[k][p];
      s0 = s0 < 0 ? 0 : (s0 > a.dyn_max[k] ? a.dyn_max[k] : s0);
      if (a.dyn_on_dst) d0 += s0 * a.dyn_mul[k]; else so += s0 * a.dyn_mul[k];
    }
    const uint4* s4 = reinterpret_cast<const uint4*>(src + so);
    uint4* d4 = reinterpret_cast<uint4*>(dst + d0);
    const int64_t v0 = chunk * (256 * ROW_U) + threadIdx.x;
    uint4 v[ROW_U];
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) v[u] = __ldcs(s4 + v0 + u * 256);
    if (a.relu) {
#pragma unroll
      for (int u = 0; u < ROW_U; ++u) {
        T* e = reinterpret_cast<T*>(&v[u]);
#pragma unroll
        for (int j = 0; j < V; ++j) e[j] = relu_bits<T>(e[j], a.relu);
      }
    }
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) __stcs(d4 + v0 + u * 256, v[u]);
  }
  if (a.fence_sys) __threadfence_system();
}

// dst[dbase + p*dpart + i] = src[sbase + p*spart] for i < n, 16 bytes per store.
template <typename T>
__global__ void splat_kernel(const T* __restrict__ src, T* __restrict__ dst, CopyArgs a,
                             int64_t nparts) {
  constexpr int V = 16 / sizeof(T);
  const int64_t per = a.n / V, total = per * nparts;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / per;
    const T v = src[a.sbase + p * a.spart];
    T f[V];
#pragma unroll
    for (int j = 0; j < V; ++j) f[j] = v;
    *reinterpret_cast<uint4*>(dst + a.dbase + p * a.dpart + (i - p * per) * V) =
        *reinterpret_cast<uint4*>(f);
  }
}

template <typename T, int V>
__global__ void fill_kernel(T* __restrict__ out, const T* __restrict__ value, int64_t n,
                            int64_t nparts) {
  const int64_t per = n / V, total = per * nparts;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = value[i / per];
    if (V == 1) {
      out[i] = v;
    } else {
      T f[V];
#pragma unroll
      for (int j = 0; j < V; ++j) f[j] = v;
      *reinterpret_cast<uint4*>(out + i * V) = *reinterpret_cast<uint4*>(f);
    }
  }
}

// Edge padding without interior padding, in ONE pass: every output element
// (or 16-byte group of the last dim) either reads its source element or takes
// the partition's pad value.  Reads the input once and writes the output once
// (the fill+copy formulation writes the interior twice).
struct PadArgs {
  int rank;
  int64_t od[SPMD_MAX_RANK];   // output dims (last in units of V)
  int64_t id[SPMD_MAX_RANK];   // input dims (last in units of V)
  int64_t low[SPMD_MAX_RANK];  // low padding (last in units of V)
  int64_t ist[SPMD_MAX_RANK];  // input strides in elements
  int64_t spart, dpart, per;   // per-partition elements in/out; V-groups out
};

template <typename T, typename I, int V>
__global__ void pad_gather_kernel(const T* __restrict__ src, const T* __restrict__ value,
                                  T* __restrict__ dst, PadArgs a, int64_t nparts) {
  const I per = (I)a.per;
  const I total = per * (I)nparts;
  for (I idx = blockIdx.x * (I)blockDim.x + threadIdx.x; idx < total;
       idx += (I)gridDim.x * blockDim.x) {
    const I p = idx / per;
    I r = idx - p * per;
    int64_t so = 0;
    bool inside = true;
#pragma unroll
    for (int k = SPMD_MAX_RANK - 1; k >= 0; --k) {
      if (k < a.rank) {
        const I dk = (I)a.od[k];
        const int64_t c = (int64_t)(r % dk) - a.low[k];
        r /= dk;
        inside = inside && c >= 0 && c < a.id[k];
        so += c * a.ist[k];
      }
    }
    T* out = dst + (int64_t)p * a.dpart + (int64_t)(idx - p * per) * V;
    if (V == 1) {
      *out = inside ? src[(int64_t)p * a.spart + so] : value[p];
    } else if (inside) {
      *reinterpret_cast<uint4*>(out) =
          *reinterpret_cast<const uint4*>(src + (int64_t)p * a.spart + so * V);
    } else {
      const T v = value[p];
      T f[V];
#pragma unroll
      for (int j = 0; j < V; ++j) f[j] = v;
      *reinterpret_cast<uint4*>(out) = *reinterpret_cast<uint4*>(f);
    }
  }
}

// Row-chunk variant of pad_gather_kernel: every output row (all dims but the
// last) is decided once per block; the last dim may carry its own low / high
// padding (vector units).
template <typename T>
__global__ void __launch_bounds__(256) pad_rows_kernel(const T* __restrict__ src,
                                                       const T* __restrict__ value,
                                                       T* __restrict__ dst, PadArgs a,
                                                       int64_t nparts, int64_t chunks) {
  constexpr int V = 16 / sizeof(T);
  const int r = a.rank - 1;
  const int64_t per_row = a.od[r];            // output vectors per row
  int64_t rows_per_part = 1;
  for (int k = 0; k < r; ++k) rows_per_part *= a.od[k];
  const int64_t rows = rows_per_part * nparts;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks, chunk = b - row * chunks;
    const int64_t p = row / rows_per_part;
    int64_t q = row - p * rows_per_part;
    int64_t so = 0;
    bool inside = true;
    for (int k = r - 1; k >= 0; --k) {
      const int64_t c = q % a.od[k] - a.low[k];
      q /= a.od[k];
      inside = inside && c >= 0 && c < a.id[k];
      so += c * a.ist[k];
    }
    T f[V];
    const T pv = value[p];
#pragma unroll
    for (int j = 0; j < V; ++j) f[j] = pv;
    const uint4 fill = *reinterpret_cast<uint4*>(f);
    const uint4* s4 = reinterpret_cast<const uint4*>(src + p * a.spart) + so;
    uint4* d4 = reinterpret_cast<uint4*>(dst + p * a.dpart) + (row - p * rows_per_part) * per_row;
    const int64_t v0 = chunk * (256 * ROW_U) + threadIdx.x;
    uint4 v[ROW_U];
#pragma unroll
    for (int u = 0; u < ROW_U; ++u) {
      const int64_t c = v0 + u * 256 - a.low[r];
      v[u] = (inside && c >= 0 && c < a.id[r]) ? __ldcs(s4 + c) : fill;
    }
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) __stcs(d4 + v0 + u * 256, v[u]);
  }
}

// Merge dims contiguous in both views; drop unit dims.
static void canonicalize(CopyArgs& a) {
  int64_t sh[SPMD_MAX_RANK], ss[SPMD_MAX_RANK], ds[SPMD_MAX_RANK];
  int r = 0;
  for (int k = 0; k < a.rank; ++k) {
    if (a.shape[k] == 1) continue;
    if (r > 0 && ss[r - 1] == a.sst[k] * a.shape[k] && ds[r - 1] == a.dst[k] * a.shape[k]) {
      sh[r - 1] *= a.shape[k];
      ss[r - 1] = a.sst[k];
      ds[r - 1] = a.dst[k];
      continue;
    }
    sh[r] = a.shape[k];
    ss[r] = a.sst[k];
    ds[r] = a.dst[k];
    ++r;
  }
  a.rank = r;
  for (int k = 0; k < r; ++k) {
    a.shape[k] = sh[k];
    a.sst[k] = ss[k];
    a.dst[k] = ds[k];
  }
}

int launch_copy(const void* src, void* dst, int dtype, CopyArgs a, int64_t nparts,
                cudaStream_t s) {
  a.n = 1;
  for (int k = 0; k < a.rank; ++k) a.n *= a.shape[k];
  if (a.n == 0 || nparts == 0) return SPMD_OK;
  SPMD_CHECK_ARG(a.ndyn == 0 || nparts <= SPMD_MAX_PARTS, "too many partitions for dynamic offsets");
  canonicalize(a);
  const int es = elem_size(dtype);
  // 16-byte vector path: innermost dim unit-stride on both sides, all offsets
  // and strides multiples of the vector width, pointers aligned.
  const int V = 16 / es;
  // Scalar broadcast (every source stride 0, contiguous destination): splat.
  if (a.rank == 1 && a.sst[0] == 0 && a.dst[0] == 1 && a.ndyn == 0 && a.n % V == 0 &&
      (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && a.dbase % V == 0 && a.dpart % V == 0) {
    const int64_t work = a.n / V * nparts;
    SPMD_DISPATCH_BYTES(dtype, T,
                        splat_kernel<T><<<grid_for(work, 256, 2), 256, 0, s>>>(
                            (const T*)src, (T*)dst, a, nparts));
    return launched(s);
  }
  bool dyn_aligned = true;
  for (int k = 0; k < a.ndyn; ++k) dyn_aligned = dyn_aligned && a.dyn_mul[k] % V == 0;
  bool vec = a.rank >= 1 && a.sst[a.rank - 1] == 1 && a.dst[a.rank - 1] == 1 &&
             a.shape[a.rank - 1] % V == 0 && dyn_aligned &&
             (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
             (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && a.sbase % V == 0 &&
             a.dbase % V == 0 && a.spart % V == 0 && a.dpart % V == 0;
  for (int k = 0; vec && k < a.rank - 1; ++k) vec = a.sst[k] % V == 0 && a.dst[k] % V == 0;
  // Innermost dim broadcasts (source stride 0): splat 16-byte groups.
  bool splat = !vec && a.rank >= 1 && a.sst[a.rank - 1] == 0 && a.dst[a.rank - 1] == 1 &&
               a.shape[a.rank - 1] % V == 0 && a.ndyn == 0 &&
               (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && a.dbase % V == 0 &&
               a.dpart % V == 0;
  for (int k = 0; splat && k < a.rank - 1; ++k) splat = a.dst[k] % V == 0;
  if (splat) {
    const int64_t w = a.n / V * nparts;
    const bool sm = a.n * nparts < (int64_t)1 << 31;
    SPMD_DISPATCH_BYTES(dtype, T, {
      if (sm)
        strided_copy_kernel<T, uint32_t, 16 / sizeof(T), true><<<grid_for(w, 256), 256, 0, s>>>(
            (const T*)src, (T*)dst, a, nparts);
      else
        strided_copy_kernel<T, uint64_t, 16 / sizeof(T), true><<<grid_for(w, 256), 256, 0, s>>>(
            (const T*)src, (T*)dst, a, nparts);
    });
    return launched(s);
  }
  if (vec && a.shape[a.rank - 1] / V >= ROW_MIN_VECS) {
    const int64_t chunks = (a.shape[a.rank - 1] / V + 256 * ROW_U - 1) / (256 * ROW_U);
    int64_t rows = nparts;
    for (int k = 0; k < a.rank - 1; ++k) rows *= a.shape[k];
    SPMD_DISPATCH_BYTES(dtype, T,
                        row_copy_kernel<T><<<row_grid(rows, chunks), 256, 0, s>>>(
                            (const T*)src, (T*)dst, a, nparts, chunks));
    return launched(s);
  }
  // The kernel walks groups of V consecutive last-dim elements (element-unit
  // index math is unchanged; each group is contiguous on both sides).
  const int64_t work = (vec ? a.n / V : a.n) * nparts;
  const bool small = a.n * nparts < (int64_t)1 << 31;
  SPMD_DISPATCH_BYTES(dtype, T, {
    if (vec) {
      if (small)
        strided_copy_kernel<T, uint32_t, 16 / sizeof(T)><<<grid_for(work, 256), 256, 0, s>>>(
            (const T*)src, (T*)dst, a, nparts);
      else
        strided_copy_kernel<T, uint64_t, 16 / sizeof(T)><<<grid_for(work, 256), 256, 0, s>>>(
            (const T*)src, (T*)dst, a, nparts);
    } else {
      if (small)
        strided_copy_kernel<T, uint32_t, 1><<<grid_for(work, 256, 2), 256, 0, s>>>(
            (const T*)src, (T*)dst, a, nparts);
      else
        strided_copy_kernel<T, uint64_t, 1><<<grid_for(work, 256, 2), 256, 0, s>>>(
            (const T*)src, (T*)dst, a, nparts);
    }
  });
  return launched(s);
}

int launch_fill(void* out, const void* value, int dtype, int64_t n, int64_t nparts,
                cudaStream_t s) {
  if (n == 0 || nparts == 0) return SPMD_OK;
  const int V = 16 / elem_size(dtype);
  const bool vec = n % V == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  SPMD_DISPATCH_BYTES(dtype, T, {
    if (vec)
      fill_kernel<T, 16 / sizeof(T)><<<grid_for(n / V * nparts, 256), 256, 0, s>>>(
          (T*)out, (const T*)value, n, nparts);
    else
      fill_kernel<T, 1><<<grid_for(n * nparts, 256, 4), 256, 0, s>>>(
          (T*)out, (const T*)value, n, nparts);
  });
  return launched(s);
}

static CopyArgs base_args(const spmd_tensor& shape_src) {
  CopyArgs a;
  memset(&a, 0, sizeof(a));
  a.rank = shape_src.rank;
  for (int k = 0; k < a.rank; ++k) a.shape[k] = shape_src.dims[k];
  return a;
}

static void contiguous_strides(const spmd_tensor& t, int64_t* st) {
  int64_t acc = 1;
  for (int k = t.rank - 1; k >= 0; --k) {
    st[k] = acc;
    acc *= t.dims[k];
  }
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_broadcast(spmd_tensor in, spmd_tensor out, const int32_t* bdims,
                              int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype, "broadcast dtype mismatch");
  int64_t ist[SPMD_MAX_RANK];
  contiguous_strides(in, ist);
  CopyArgs a = base_args(out);
  contiguous_strides(out, a.dst);
  for (int k = 0; k < out.rank; ++k) a.sst[k] = 0;
  for (int i = 0; i < in.rank; ++i) {
    SPMD_CHECK_ARG(bdims[i] >= 0 && bdims[i] < out.rank && out.dims[bdims[i]] == in.dims[i],
                   "broadcast dims mismatch");
    a.sst[bdims[i]] = ist[i];
  }
  a.spart = numel(in);
  a.dpart = numel(out);
  return launch_copy(in.data, out.data, out.dtype, a, nparts, as_stream(stream));
}

static int transpose_impl(const spmd_tensor& in, const spmd_tensor& out, const int32_t* perm,
                          int relu, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && in.rank == out.rank, "transpose mismatch");
  int64_t ist[SPMD_MAX_RANK];
  contiguous_strides(in, ist);
  CopyArgs a = base_args(out);
  contiguous_strides(out, a.dst);
  for (int j = 0; j < out.rank; ++j) {
    SPMD_CHECK_ARG(out.dims[j] == in.dims[perm[j]], "transpose dims mismatch");
    a.sst[j] = ist[perm[j]];
  }
  a.spart = a.dpart = numel(in);
  a.relu = relu;
  return launch_copy(in.data, out.data, out.dtype, a, nparts, as_stream(stream));
}

extern "C" int spmd_transpose(spmd_tensor in, spmd_tensor out, const int32_t* perm,
                              int64_t nparts, void* stream) {
  return transpose_impl(in, out, perm, 0, nparts, stream);
}

// Transpose -> ReLU in one pass (the MoE layer's reshard annotations: the
// dispatched tokens and the expert outputs are transposed, then ReLU'd).
extern "C" int spmd_transpose_relu(spmd_tensor in, spmd_tensor out, const int32_t* perm,
                                   int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == SPMD_F32 || in.dtype == SPMD_BF16 || in.dtype == SPMD_S32,
                 "transpose_relu: f32 / bf16 / s32");
  return transpose_impl(in, out, perm, in.dtype == SPMD_S32 ? 2 : 1, nparts, stream);
}

extern "C" int spmd_reverse(spmd_tensor in, spmd_tensor out, const int32_t* dims, int ndims,
                            int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && numel(in) == numel(out), "reverse mismatch");
  CopyArgs a = base_args(out);
  contiguous_strides(in, a.sst);
  contiguous_strides(out, a.dst);
  for (int i = 0; i < ndims; ++i) {
    int d = dims[i];
    SPMD_CHECK_ARG(d >= 0 && d < in.rank, "reverse dim out of range");
    if (in.dims[d] == 0) continue;
    a.sbase += (in.dims[d] - 1) * a.sst[d];
    a.sst[d] = -a.sst[d];
  }
  a.spart = a.dpart = numel(in);
  return launch_copy(in.data, out.data, out.dtype, a, nparts, as_stream(stream));
}

static int pad_edges(const spmd_tensor& in, const spmd_tensor& value, const spmd_tensor& out,
                     const int64_t* low, const int64_t* high, int64_t nparts, cudaStream_t s) {
  PadArgs a;
  memset(&a, 0, sizeof(a));
  // Merge runs of dims that carry no padding into their left neighbour's
  // stride walk: only dims with padding (and the last dim) need coordinates.
  int r = 0;
  for (int k = 0; k < in.rank; ++k) {
    SPMD_CHECK_ARG(low[k] >= 0 && high[k] >= 0, "negative padding");
    SPMD_CHECK_ARG(out.dims[k] == in.dims[k] + low[k] + high[k], "pad output shape mismatch");
    if (r > 0 && low[k] == 0 && high[k] == 0 && a.low[r - 1] == 0 && a.od[r - 1] == a.id[r - 1]) {
      a.od[r - 1] *= out.dims[k];
      a.id[r - 1] *= in.dims[k];
      continue;
    }
    a.od[r] = out.dims[k];
    a.id[r] = in.dims[k];
    a.low[r] = low[k];
    ++r;
  }
  a.rank = r;
  int64_t acc = 1;
  for (int k = r - 1; k >= 0; --k) {
    a.ist[k] = acc;
    acc *= a.id[k];
  }
  a.spart = numel(in);
  a.dpart = numel(out);
  const int V = 16 / elem_size(out.dtype);
  const bool vec = a.id[r - 1] % V == 0 && a.low[r - 1] % V == 0 && a.od[r - 1] % V == 0 &&
                   (reinterpret_cast<uintptr_t>(in.data) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(out.data) & 15) == 0;
  if (vec) {
    a.id[r - 1] /= V;
    a.od[r - 1] /= V;
    a.low[r - 1] /= V;
    for (int k = 0; k < r - 1; ++k) a.ist[k] /= V;
  }
  a.per = a.dpart / (vec ? V : 1);
  if (vec && a.od[r - 1] >= ROW_MIN_VECS) {
    const int64_t chunks = (a.od[r - 1] + 256 * ROW_U - 1) / (256 * ROW_U);
    int64_t rows = nparts;
    for (int k = 0; k < r - 1; ++k) rows *= a.od[k];
    SPMD_DISPATCH_BYTES(out.dtype, T,
                        pad_rows_kernel<T><<<row_grid(rows, chunks), 256, 0, s>>>(
                            (const T*)in.data, (const T*)value.data, (T*)out.data, a, nparts,
                            chunks));
    return launched(s);
  }
  const int64_t work = a.per * nparts;
  const bool small = work < (int64_t)1 << 31;
  SPMD_DISPATCH_BYTES(out.dtype, T, {
    const T* src = (const T*)in.data;
    const T* val = (const T*)value.data;
    T* dst = (T*)out.data;
    if (vec) {
      if (small)
        pad_gather_kernel<T, uint32_t, 16 / sizeof(T)><<<grid_for(work, 256), 256, 0, s>>>(
            src, val, dst, a, nparts);
      else
        pad_gather_kernel<T, uint64_t, 16 / sizeof(T)><<<grid_for(work, 256), 256, 0, s>>>(
            src, val, dst, a, nparts);
    } else {
      if (small)
        pad_gather_kernel<T, uint32_t, 1><<<grid_for(work, 256, 2), 256, 0, s>>>(
            src, val, dst, a, nparts);
      else
        pad_gather_kernel<T, uint64_t, 1><<<grid_for(work, 256, 2), 256, 0, s>>>(
            src, val, dst, a, nparts);
    }
  });
  return launched(s);
}

extern "C" int spmd_pad(spmd_tensor in, spmd_tensor value, spmd_tensor out, const int64_t* low,
                        const int64_t* high, const int64_t* interior, int64_t nparts,
                        void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && value.dtype == in.dtype && value.rank == 0,
                 "pad dtype mismatch");
  cudaStream_t s = as_stream(stream);
  bool edge_only = in.rank == out.rank && in.rank > 0;
  for (int k = 0; k < in.rank; ++k) edge_only = edge_only && interior[k] == 0;
  if (edge_only && numel(in) > 0 && numel(out) > 0) return pad_edges(in, value, out, low, high,
                                                                     nparts, s);
  int rc = launch_fill(out.data, value.data, out.dtype, numel(out), nparts, s);
  if (rc) return rc;
  CopyArgs a = base_args(in);
  contiguous_strides(in, a.sst);
  int64_t ost[SPMD_MAX_RANK];
  contiguous_strides(out, ost);
  for (int k = 0; k < in.rank; ++k) {
    SPMD_CHECK_ARG(low[k] >= 0 && high[k] >= 0 && interior[k] >= 0, "negative padding");
    int64_t n = in.dims[k];
    SPMD_CHECK_ARG(out.dims[k] == n + (n > 0 ? n - 1 : 0) * interior[k] + low[k] + high[k],
                   "pad output shape mismatch");
    a.dst[k] = ost[k] * (interior[k] + 1);
    a.dbase += low[k] * ost[k];
  }
  a.spart = numel(in);
  a.dpart = numel(out);
  return launch_copy(in.data, out.data, out.dtype, a, nparts, s);
}

extern "C" int spmd_slice(spmd_tensor in, spmd_tensor out, const int64_t* starts,
                          const int64_t* strides, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && in.rank == out.rank, "slice mismatch");
  int64_t ist[SPMD_MAX_RANK];
  contiguous_strides(in, ist);
  CopyArgs a = base_args(out);
  contiguous_strides(out, a.dst);
  for (int k = 0; k < in.rank; ++k) {
    SPMD_CHECK_ARG(strides[k] >= 1, "slice stride must be >= 1");
    a.sst[k] = ist[k] * strides[k];
    a.sbase += starts[k] * ist[k];
  }
  a.spart = numel(in);
  a.dpart = numel(out);
  return launch_copy(in.data, out.data, out.dtype, a, nparts, as_stream(stream));
}

extern "C" int spmd_dynamic_slice(spmd_tensor in, const spmd_tensor* starts, spmd_tensor out,
                                  int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && in.rank == out.rank, "dynamic-slice mismatch");
  CopyArgs a = base_args(out);
  contiguous_strides(in, a.sst);
  contiguous_strides(out, a.dst);
  for (int k = 0; k < in.rank; ++k) {
    SPMD_CHECK_ARG(starts[k].dtype == SPMD_S32 || starts[k].dtype == SPMD_U32,
                   "dynamic-slice index must be s32/u32");
    SPMD_CHECK_ARG(out.dims[k] <= in.dims[k], "dynamic-slice size exceeds operand");
    if (out.dims[k] == in.dims[k]) continue;  // start clamps to 0: static
    a.dyn_start[a.ndyn] = (const int32_t*)starts[k].data;
    a.dyn_max[a.ndyn] = in.dims[k] - out.dims[k];
    a.dyn_mul[a.ndyn] = a.sst[k];
    a.ndyn++;
  }
  a.spart = numel(in);
  a.dpart = numel(out);
  return launch_copy(in.data, out.data, out.dtype, a, nparts, as_stream(stream));
}

extern "C" int spmd_dynamic_update_slice(spmd_tensor in, spmd_tensor upd, const spmd_tensor* starts,
                                         spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && upd.dtype == in.dtype && in.rank == upd.rank,
                 "dynamic-update-slice mismatch");
  cudaStream_t s = as_stream(stream);
  if (out.data != in.data)
    SPMD_CUDA_TRY(cudaMemcpyAsync(out.data, in.data,
                                  (size_t)numel(in) * nparts * elem_size(in.dtype),
                                  cudaMemcpyDeviceToDevice, s));
  CopyArgs a = base_args(upd);
  contiguous_strides(upd, a.sst);
  contiguous_strides(out, a.dst);
  a.dyn_on_dst = 1;
  for (int k = 0; k < in.rank; ++k) {
    SPMD_CHECK_ARG(upd.dims[k] <= in.dims[k], "update larger than operand");
    if (upd.dims[k] == in.dims[k]) continue;  // start clamps to 0: static
    a.dyn_start[a.ndyn] = (const int32_t*)starts[k].data;
    a.dyn_max[a.ndyn] = in.dims[k] - upd.dims[k];
    a.dyn_mul[a.ndyn] = a.dst[k];
    a.ndyn++;
  }
  a.spart = numel(upd);
  a.dpart = numel(out);
  return launch_copy(upd.data, out.data, out.dtype, a, nparts, s);
}

extern "C" int spmd_concat(const spmd_tensor* ins, int n, int axis, spmd_tensor out,
                           int64_t nparts, void* stream) {
  cudaStream_t s = as_stream(stream);
  int64_t off = 0;
  int64_t ost[SPMD_MAX_RANK];
  contiguous_strides(out, ost);
  for (int i = 0; i < n; ++i) {
    const spmd_tensor& t = ins[i];
    SPMD_CHECK_ARG(t.dtype == out.dtype && t.rank == out.rank, "concat mismatch");
    CopyArgs a = base_args(t);
    contiguous_strides(t, a.sst);
    for (int k = 0; k < t.rank; ++k) a.dst[k] = ost[k];
    a.dbase = off * ost[axis];
    a.spart = numel(t);
    a.dpart = numel(out);
    int rc = launch_copy(t.data, out.data, out.dtype, a, nparts, s);
    if (rc) return rc;
    off += t.dims[axis];
  }
  SPMD_CHECK_ARG(off == out.dims[axis], "concat output size mismatch");
  return SPMD_OK;
}

extern "C" int spmd_rotate(spmd_tensor in, spmd_tensor out, int dim, int64_t amount,
                           int64_t nparts, void* stream) {
  // out[o] = in[(o + amount) mod n]  (np.roll(x, -amount), simulator.py:278-279)
  SPMD_CHECK_ARG(in.dtype == out.dtype && dim >= 0 && dim < in.rank, "rotate mismatch");
  cudaStream_t s = as_stream(stream);
  int64_t n = in.dims[dim];
  if (n == 0) return SPMD_OK;
  int64_t k = ((amount % n) + n) % n;
  int64_t st[SPMD_MAX_RANK];
  contiguous_strides(in, st);
  for (int piece = 0; piece < 2; ++piece) {
    int64_t len = piece == 0 ? n - k : k;
    if (len == 0) continue;
    CopyArgs a = base_args(in);
    a.shape[dim] = len;
    for (int d = 0; d < in.rank; ++d) a.sst[d] = a.dst[d] = st[d];
    a.sbase = (piece == 0 ? k : 0) * st[dim];
    a.dbase = (piece == 0 ? 0 : n - k) * st[dim];
    a.spart = a.dpart = numel(in);
    int rc = launch_copy(in.data, out.data, out.dtype, a, nparts, s);
    if (rc) return rc;
  }
  return SPMD_OK;
}

extern "C" int spmd_shift(spmd_tensor in, spmd_tensor fill, spmd_tensor out, int dim,
                          int64_t amount, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && fill.dtype == in.dtype && dim >= 0 && dim < in.rank,
                 "shift mismatch");
  cudaStream_t s = as_stream(stream);
  int rc = launch_fill(out.data, fill.data, out.dtype, numel(out), nparts, s);
  if (rc) return rc;
  int64_t n = in.dims[dim];
  int64_t k = amount >= 0 ? amount : -amount;
  if (k >= n) return SPMD_OK;
  int64_t st[SPMD_MAX_RANK];
  contiguous_strides(in, st);
  CopyArgs a = base_args(in);
  a.shape[dim] = n - k;
  for (int d = 0; d < in.rank; ++d) a.sst[d] = a.dst[d] = st[d];
  if (amount >= 0) a.dbase = amount * st[dim];
  else a.sbase = k * st[dim];
  a.spart = a.dpart = numel(in);
  return launch_copy(in.data, out.data, out.dtype, a, nparts, s);
}
