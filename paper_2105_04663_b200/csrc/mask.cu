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

}  // namespace spmd

using namespace spmd;

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
