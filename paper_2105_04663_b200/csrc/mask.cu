// Fused uneven-shard / halo-window range mask (one HBM pass).
//
// The partitioner masks padding and out-of-range halo elements with the op
// chain of select_range (reference partitioner.py:205-228):
//   g    = iota(dims, axis) + offset[partition]
//   out  = select(g < high, val, fill)           [then select(g >= low, out, fill)]
// which is 7-9 full-tensor kernels when executed op by op.  The executor
// recognises the chain and calls this kernel instead: the predicate depends
// only on the axis coordinate, so the tensor is walked as
// [P, outer, n_axis, inner] with 16-byte vectors along `inner`.
#include "common.cuh"

#include <string.h>

namespace spmd {

template <typename T, int V>
__global__ void mask_range_kernel(const T* __restrict__ in, T* __restrict__ out,
                                  const int32_t* __restrict__ offset, const T* __restrict__ fill,
                                  int64_t outer, int64_t n_axis, int64_t inner, int64_t nparts,
                                  int64_t low, int64_t high) {
  const int64_t per_row = inner / V;                 // vectors per (outer, axis) row
  const int64_t per_part = outer * n_axis * per_row;
  const int64_t total = per_part * nparts;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / per_part;
    const int64_t r = i - p * per_part;
    const int64_t a = (r / per_row) % n_axis;
    const int64_t gidx = a + offset[p];
    const bool keep = gidx < high && gidx >= low;
    if (V == 1) {
      out[i] = keep ? in[i] : fill[p];
    } else {
      uint4 v;
      if (keep) {
        v = reinterpret_cast<const uint4*>(in)[i];
      } else {
        T f[V];
#pragma unroll
        for (int j = 0; j < V; ++j) f[j] = fill[p];
        v = *reinterpret_cast<uint4*>(f);
      }
      reinterpret_cast<uint4*>(out)[i] = v;
    }
  }
}

// Row-chunk variant: rows = [P, outer, n_axis], each `inner` contiguous;
// the predicate is decided once per block.
template <typename T>
__global__ void __launch_bounds__(256) mask_rows_kernel(const T* __restrict__ in,
                                                        T* __restrict__ out,
                                                        const int32_t* __restrict__ offset,
                                                        const T* __restrict__ fill,
                                                        int64_t outer, int64_t n_axis,
                                                        int64_t inner, int64_t nparts,
                                                        int64_t low, int64_t high,
                                                        int64_t chunks) {
  constexpr int V = 16 / sizeof(T);
  const int64_t per_row = inner / V;
  const int64_t rows_per_part = outer * n_axis;
  const int64_t rows = rows_per_part * nparts;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks, chunk = b - row * chunks;
    const int64_t p = row / rows_per_part;
    const int64_t gidx = (row - p * rows_per_part) % n_axis + offset[p];
    const bool keep = gidx < high && gidx >= low;
    T f[V];
    const T fv = fill[p];
#pragma unroll
    for (int j = 0; j < V; ++j) f[j] = fv;
    const uint4 fillv = *reinterpret_cast<uint4*>(f);
    const uint4* s4 = reinterpret_cast<const uint4*>(in) + row * per_row;
    uint4* d4 = reinterpret_cast<uint4*>(out) + row * per_row;
    const int64_t v0 = chunk * (256 * ROW_U) + threadIdx.x;
    uint4 v[ROW_U];
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      v[u] = (keep && v0 + u * 256 < per_row) ? __ldcs(s4 + v0 + u * 256) : fillv;
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) __stcs(d4 + v0 + u * 256, v[u]);
  }
}

// Halo window (exchange_and_slice, reference formatting.py:109-182): the
// per-device window = DS(mask(concat(left_halo, shard, right_halo)), start)
// read straight from the three pieces in one pass.
struct HaloArgs {
  const void* piece[3];
  int64_t len[3];          // piece extents along the axis
  int npieces;
  int64_t outer, inner, buf_len, window;
  const int32_t* start;    // per-partition dynamic-slice start (clamped)
  int has_mask, has_low;
  const int32_t* offset;   // per-partition global offset of buffer position 0
  const void* fill;
  int64_t low, high;
};

template <typename T, int V>
__global__ void halo_window_kernel(T* __restrict__ out, HaloArgs a, int64_t nparts) {
  const int64_t per_row = a.inner / V;
  const int64_t per_part = a.outer * a.window * per_row;
  const int64_t total = per_part * nparts;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / per_part;
    int64_t r = idx - p * per_part;
    const int64_t v = r % per_row;
    r /= per_row;
    const int64_t i = r % a.window;
    const int64_t o = r / a.window;
    int64_t s0 = a.start[p];
    s0 = s0 < 0 ? 0 : (s0 > a.buf_len - a.window ? a.buf_len - a.window : s0);
    const int64_t j = s0 + i;
    bool keep = true;
    if (a.has_mask) {
      const int64_t g = j + a.offset[p];
      keep = g < a.high && (!a.has_low || g >= a.low);
    }
    T* dst = out + idx * V;
    if (!keep) {
      const T f = reinterpret_cast<const T*>(a.fill)[p];
#pragma unroll
      for (int q = 0; q < V; ++q) dst[q] = f;
      continue;
    }
    int k = 0;
    int64_t jj = j;
    while (k < a.npieces - 1 && jj >= a.len[k]) {
      jj -= a.len[k];
      ++k;
    }
    const T* src = reinterpret_cast<const T*>(a.piece[k]) +
                   ((p * a.outer + o) * a.len[k] + jj) * a.inner + v * V;
    if (V == 1) {
      dst[0] = src[0];
    } else {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    }
  }
}

// Row-uniform variant for long rows (inner >= one block's worth of vectors):
// each block owns a chunk of one output row (partition p, outer o, window row
// i), so the clamp / mask / piece lookup runs once per block and every thread
// keeps U independent 16-byte loads in flight.
template <typename T, int U>
__global__ void __launch_bounds__(256) halo_rows_kernel(T* __restrict__ out, HaloArgs a,
                                                        int64_t nparts, int64_t chunks) {
  constexpr int V = 16 / sizeof(T);
  const int64_t per_row = a.inner / V;
  const int64_t rows = nparts * a.outer * a.window;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks;
    const int64_t v0 = (b - row * chunks) * (256 * U) + threadIdx.x;
    const int64_t p = row / (a.outer * a.window);
    const int64_t rr = row - p * a.outer * a.window;
    const int64_t o = rr / a.window, i = rr - o * a.window;
    int64_t s0 = a.start[p];
    s0 = s0 < 0 ? 0 : (s0 > a.buf_len - a.window ? a.buf_len - a.window : s0);
    const int64_t j = s0 + i;
    bool keep = true;
    if (a.has_mask) {
      const int64_t g = j + a.offset[p];
      keep = g < a.high && (!a.has_low || g >= a.low);
    }
    uint4* dst = reinterpret_cast<uint4*>(out) + row * per_row;
    if (!keep) {
      const T f = reinterpret_cast<const T*>(a.fill)[p];
      T fv[V];
#pragma unroll
      for (int q = 0; q < V; ++q) fv[q] = f;
      const uint4 w = *reinterpret_cast<uint4*>(fv);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v0 + u * 256 < per_row) dst[v0 + u * 256] = w;
      continue;
    }
    int k = 0;
    int64_t jj = j;
    while (k < a.npieces - 1 && jj >= a.len[k]) {
      jj -= a.len[k];
      ++k;
    }
    const uint4* src = reinterpret_cast<const uint4*>(
        reinterpret_cast<const T*>(a.piece[k]) + ((p * a.outer + o) * a.len[k] + jj) * a.inner);
    uint4 reg[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 256 < per_row) reg[u] = __ldcs(src + v0 + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 256 < per_row) __stcs(dst + v0 + u * 256, reg[u]);
  }
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_halo_window(const spmd_tensor* pieces, int npieces, int axis,
                                spmd_tensor start, int has_mask, spmd_tensor offset,
                                spmd_tensor fill, int64_t low, int64_t high, int has_low,
                                spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(npieces >= 1 && npieces <= 3 && axis >= 0 && axis < out.rank,
                 "halo_window arguments");
  SPMD_CHECK_ARG(start.dtype == SPMD_S32 && start.rank == 0, "halo_window start");
  HaloArgs a;
  memset(&a, 0, sizeof(a));
  a.npieces = npieces;
  a.outer = a.inner = 1;
  for (int d = 0; d < axis; ++d) a.outer *= out.dims[d];
  for (int d = axis + 1; d < out.rank; ++d) a.inner *= out.dims[d];
  a.window = out.dims[axis];
  for (int k = 0; k < npieces; ++k) {
    SPMD_CHECK_ARG(pieces[k].dtype == out.dtype && pieces[k].rank == out.rank,
                   "halo_window piece mismatch");
    a.piece[k] = pieces[k].data;
    a.len[k] = pieces[k].dims[axis];
    a.buf_len += a.len[k];
  }
  SPMD_CHECK_ARG(a.window <= a.buf_len, "halo_window larger than buffer");
  a.start = (const int32_t*)start.data;
  a.has_mask = has_mask;
  if (has_mask) {
    SPMD_CHECK_ARG(offset.dtype == SPMD_S32 && fill.dtype == out.dtype, "halo_window mask");
    a.offset = (const int32_t*)offset.data;
    a.fill = fill.data;
    a.low = low;
    a.high = high;
    a.has_low = has_low;
  }
  const int64_t n = a.outer * a.window * a.inner * nparts;
  if (n == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  const int V = 16 / elem_size(out.dtype);
  bool vec = a.inner % V == 0 && (reinterpret_cast<uintptr_t>(out.data) & 15) == 0;
  for (int k = 0; k < npieces; ++k) vec = vec && (reinterpret_cast<uintptr_t>(a.piece[k]) & 15) == 0;
  if (vec && a.inner / V >= 1024) {
    const int64_t chunks = (a.inner / V + 1023) / 1024;
    const int64_t blocks = a.outer * a.window * nparts * chunks;
    const int64_t grid = blocks < 148LL * 8 ? blocks : 148LL * 8;  // 8 x 256 threads per SM
    SPMD_DISPATCH_BYTES(out.dtype, T,
                        halo_rows_kernel<T, 4><<<grid, 256, 0, s>>>((T*)out.data, a, nparts,
                                                                   chunks));
    return launched(s);
  }
  SPMD_DISPATCH_BYTES(out.dtype, T, {
    if (vec)
      halo_window_kernel<T, 16 / sizeof(T)><<<grid_for(n / V, 256), 256, 0, s>>>((T*)out.data, a,
                                                                                nparts);
    else
      halo_window_kernel<T, 1><<<grid_for(n, 256, 2), 256, 0, s>>>((T*)out.data, a, nparts);
  });
  return launched(s);
}

// out = (low <= iota_axis + offset[p] < high) ? in : fill[p]; has_low=0 drops
// the lower bound (low = INT64_MIN).
extern "C" int spmd_mask_range(spmd_tensor in, spmd_tensor offset, spmd_tensor fill,
                               spmd_tensor out, int axis, int64_t low, int64_t high, int has_low,
                               int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && fill.dtype == in.dtype && numel(in) == numel(out),
                 "mask_range mismatch");
  SPMD_CHECK_ARG(offset.dtype == SPMD_S32 && offset.rank == 0 && fill.rank == 0,
                 "mask_range offset/fill must be per-partition scalars");
  SPMD_CHECK_ARG(axis >= 0 && axis < in.rank, "mask_range axis");
  int64_t outer = 1, inner = 1;
  for (int i = 0; i < axis; ++i) outer *= in.dims[i];
  for (int i = axis + 1; i < in.rank; ++i) inner *= in.dims[i];
  const int64_t n = in.dims[axis];
  if (outer * n * inner * nparts == 0) return SPMD_OK;
  if (!has_low) low = INT64_MIN;
  cudaStream_t s = as_stream(stream);
  const int es = elem_size(in.dtype);
  const int V = 16 / es;
  const bool vec = inner % V == 0 && (reinterpret_cast<uintptr_t>(in.data) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(out.data) & 15) == 0;
  if (vec && inner / V >= ROW_MIN_VECS) {
    const int64_t chunks = (inner / V + 256 * ROW_U - 1) / (256 * ROW_U);
    SPMD_DISPATCH_BYTES(in.dtype, T,
                        mask_rows_kernel<T><<<row_grid(outer * n * nparts, chunks), 256, 0, s>>>(
                            (const T*)in.data, (T*)out.data, (const int32_t*)offset.data,
                            (const T*)fill.data, outer, n, inner, nparts, low, high, chunks));
    return launched(s);
  }
  SPMD_DISPATCH_BYTES(in.dtype, T, {
    if (vec)
      mask_range_kernel<T, 16 / sizeof(T)><<<grid_for(outer * n * inner * nparts / V, 256), 256, 0,
                                             s>>>((const T*)in.data, (T*)out.data,
                                                  (const int32_t*)offset.data, (const T*)fill.data,
                                                  outer, n, inner, nparts, low, high);
    else
      mask_range_kernel<T, 1><<<grid_for(outer * n * inner * nparts, 256, 2), 256, 0, s>>>(
          (const T*)in.data, (T*)out.data, (const int32_t*)offset.data, (const T*)fill.data, outer,
          n, inner, nparts, low, high);
  });
  return launched(s);
}
