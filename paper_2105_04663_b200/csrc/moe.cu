// GShard-style MoE routing and dispatch/combine permutations (config C3).
//
// The reference consumes a given one-hot dispatch tensor through a dense Dot
// (tests/test_acceptance.py:326-349); gating is out of its scope.
// The slot rule is pinned by paper_2105_04663_b200/moe.py::route_top1:
//   expert(b,s) = argmax_e logits (first max), slot(b,s) = number of earlier
//   tokens of row b routed to the same expert (exclusive prefix count),
//   dropped when slot >= capacity; gate = softmax prob of the chosen expert.
//
// route:    one warp per (partition, batch row); tokens in chunks of 32 lanes.
//           __match_any_sync groups lanes by expert -> in-chunk rank by popc of
//           the lower-lane mask; per-expert running counts live in shared
//           memory (the scan carry).  Integer results are bit-exact.
// dispatch: expert buffers [E, C, M] filled by row gathers (16-B vector
//           copies, one warp per token row), empty slots zeroed -- equal to
//           Dot(dispatch_onehot, x).
// combine:  out[b,s,:] = gate * y[b, e, slot, :] (or 0 when dropped) --
//           equal to Dot(combine_weights, y) for one-hot routing.
#include "common.cuh"

namespace spmd {

constexpr int MOE_MAX_E = 256;

template <typename T>
__global__ void moe_route_kernel(const T* __restrict__ logits, int32_t* __restrict__ expert,
                                 int32_t* __restrict__ slot, float* __restrict__ gate,
                                 int64_t rows, int S, int E, int capacity) {
  __shared__ int counts[8][MOE_MAX_E];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t row = blockIdx.x * 8 + w; row < rows; row += (int64_t)gridDim.x * 8) {
    for (int e = lane; e < E; e += 32) counts[w][e] = 0;
    __syncwarp();
    for (int s0 = 0; s0 < S; s0 += 32) {
      const int s = s0 + lane;
      int best = -1;
      float m = -INFINITY, denom = 0.f;
      if (s < S) {
        const T* l = logits + (row * S + s) * (int64_t)E;
        for (int e = 0; e < E; ++e) {
          float v = ld<T>(l[e]);
          if (best < 0 || v > m) {
            m = v;
            best = e;
          }
        }
        for (int e = 0; e < E; ++e) denom += expf(ld<T>(l[e]) - m);
      }
      const unsigned same = __match_any_sync(0xffffffffu, best);
      const int rank = __popc(same & ((1u << lane) - 1));
      int base = (best >= 0) ? counts[w][best] : 0;
      __syncwarp();
      if (best >= 0) {
        const int sl = base + rank;
        expert[row * S + s] = best;
        slot[row * S + s] = sl;
        gate[row * S + s] = 1.f / denom;   // exp(m - m) / sum
        if (rank == 0) counts[w][best] = base + __popc(same);
      }
      __syncwarp();
    }
    (void)capacity;
  }
}

template <int V>
__global__ void moe_dispatch_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ expert,
                                    const int32_t* __restrict__ slot, uint16_t* __restrict__ out,
                                    int64_t tokens, int S, int E, int C, int M) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < tokens;
       t += warps) {
    const int sl = slot[t];
    if (sl >= C) continue;   // dropped (capacity)
    const int64_t row = t / S;   // (partition, batch) row
    const int e = expert[t];
    const uint4* src = reinterpret_cast<const uint4*>(x + t * (int64_t)M);
    uint4* dst = reinterpret_cast<uint4*>(out + ((row * E + e) * (int64_t)C + sl) * M);
    for (int i = lane; i < M / V; i += 32) dst[i] = __ldcs(src + i);
  }
}

__global__ void moe_combine_kernel(const bf16* __restrict__ y, const int32_t* __restrict__ expert,
                                   const int32_t* __restrict__ slot, const float* __restrict__ gate,
                                   bf16* __restrict__ out, int64_t tokens, int S, int E, int C,
                                   int M) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < tokens;
       t += warps) {
    const int sl = slot[t];
    uint4* dst = reinterpret_cast<uint4*>(out + t * (int64_t)M);
    if (sl >= C) {
      for (int i = lane; i < M / 8; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const int64_t row = t / S;
    // bf16 combine weights (what the reference graph's bf16 combine tensor
    // holds): g*y is then exact in fp32 and rounds once, bit-identical to
    // Dot(combine, y) with one nonzero per token.
    const float g = __bfloat162float(__float2bfloat16_rn(gate[t]));
    const uint4* src =
        reinterpret_cast<const uint4*>(y + ((row * E + expert[t]) * (int64_t)C + sl) * M);
    for (int i = lane; i < M / 8; i += 32) {
      uint4 v = __ldcs(src + i);
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        h[j] = __floats2bfloat162_rn(f.x * g, f.y * g);
      }
      dst[i] = v;
    }
  }
}

template <typename T>
__global__ void moe_masks_kernel(const int32_t* __restrict__ expert, const int32_t* __restrict__ slot,
                                 const float* __restrict__ gate, T* __restrict__ dispatch,
                                 T* __restrict__ combine, int64_t tokens, int E, int C) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tokens;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int sl = slot[t];
    if (sl < C) {
      const int64_t o = (t * E + expert[t]) * (int64_t)C + sl;
      dispatch[o] = st<T>(1.f);
      combine[o] = st<T>(gate[t]);
    }
  }
}

}  // namespace spmd

using namespace spmd;

// logits [P, B, S, E] (f32 or bf16) -> expert/slot s32 [P, B, S], gate f32 [P, B, S].
extern "C" int spmd_moe_route(spmd_tensor logits, int capacity, spmd_tensor expert,
                              spmd_tensor slot, spmd_tensor gate, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(logits.rank == 3 && (logits.dtype == SPMD_F32 || logits.dtype == SPMD_BF16),
                 "moe route expects logits [B, S, E] f32/bf16");
  SPMD_CHECK_ARG(expert.dtype == SPMD_S32 && slot.dtype == SPMD_S32 && gate.dtype == SPMD_F32,
                 "moe route output dtypes");
  const int S = (int)logits.dims[1], E = (int)logits.dims[2];
  SPMD_CHECK_ARG(E <= MOE_MAX_E, "too many experts");
  const int64_t rows = logits.dims[0] * nparts;
  if (rows * S == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  unsigned grid = (unsigned)((rows + 7) / 8);
  if (logits.dtype == SPMD_F32)
    moe_route_kernel<float><<<grid, 256, 0, s>>>((const float*)logits.data, (int32_t*)expert.data,
                                                 (int32_t*)slot.data, (float*)gate.data, rows, S,
                                                 E, capacity);
  else
    moe_route_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)logits.data, (int32_t*)expert.data,
                                                (int32_t*)slot.data, (float*)gate.data, rows, S,
                                                E, capacity);
  return launched(s);
}

// x [P, B, S, M] bf16 -> out [P, B, E, C, M] bf16 (zero-filled empty slots).
extern "C" int spmd_moe_dispatch(spmd_tensor x, spmd_tensor expert, spmd_tensor slot,
                                 spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(x.dtype == SPMD_BF16 && out.dtype == SPMD_BF16 && x.rank == 3 && out.rank == 4,
                 "moe dispatch expects bf16 x [B,S,M] -> [B,E,C,M]");
  const int S = (int)x.dims[1], M = (int)x.dims[2];
  const int E = (int)out.dims[1], C = (int)out.dims[2];
  SPMD_CHECK_ARG(out.dims[0] == x.dims[0] && out.dims[3] == M && M % 8 == 0, "moe dispatch shape");
  cudaStream_t s = as_stream(stream);
  SPMD_CUDA_TRY(cudaMemsetAsync(out.data, 0, (size_t)numel(out) * nparts * 2, s));
  const int64_t tokens = x.dims[0] * S * nparts;
  if (tokens == 0) return SPMD_OK;
  moe_dispatch_kernel<8><<<grid_for(tokens * 32, 256), 256, 0, s>>>(
      (const uint16_t*)x.data, (const int32_t*)expert.data, (const int32_t*)slot.data,
      (uint16_t*)out.data, tokens, S, E, C, M);
  return launched(s);
}

// y [P, B, E, C, M] bf16 -> out [P, B, S, M] bf16.
extern "C" int spmd_moe_combine(spmd_tensor y, spmd_tensor expert, spmd_tensor slot,
                                spmd_tensor gate, spmd_tensor out, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(y.dtype == SPMD_BF16 && out.dtype == SPMD_BF16 && y.rank == 4 && out.rank == 3,
                 "moe combine expects bf16 y [B,E,C,M] -> [B,S,M]");
  const int S = (int)out.dims[1], M = (int)out.dims[2];
  const int E = (int)y.dims[1], C = (int)y.dims[2];
  SPMD_CHECK_ARG(M % 8 == 0 && y.dims[3] == M, "moe combine shape");
  const int64_t tokens = out.dims[0] * S * nparts;
  if (tokens == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  moe_combine_kernel<<<grid_for(tokens * 32, 256), 256, 0, s>>>(
      (const bf16*)y.data, (const int32_t*)expert.data, (const int32_t*)slot.data,
      (const float*)gate.data, (bf16*)out.data, tokens, S, E, C, M);
  return launched(s);
}

// Dense one-hot masks [P, B, S, E, C] (dispatch = 1, combine = gate) from a
// routing -- the tensors the reference's MoE graph consumes.
extern "C" int spmd_moe_masks(spmd_tensor expert, spmd_tensor slot, spmd_tensor gate,
                              spmd_tensor dispatch, spmd_tensor combine, int64_t nparts,
                              void* stream) {
  SPMD_CHECK_ARG(dispatch.rank == 4 && dispatch.dtype == combine.dtype, "moe masks shape");
  const int E = (int)dispatch.dims[2], C = (int)dispatch.dims[3];
  const int64_t tokens = dispatch.dims[0] * dispatch.dims[1] * nparts;
  cudaStream_t s = as_stream(stream);
  const size_t bytes = (size_t)numel(dispatch) * nparts * elem_size(dispatch.dtype);
  SPMD_CUDA_TRY(cudaMemsetAsync(dispatch.data, 0, bytes, s));
  SPMD_CUDA_TRY(cudaMemsetAsync(combine.data, 0, bytes, s));
  if (tokens == 0) return SPMD_OK;
  if (dispatch.dtype == SPMD_F32)
    moe_masks_kernel<float><<<grid_for(tokens, 256), 256, 0, s>>>(
        (const int32_t*)expert.data, (const int32_t*)slot.data, (const float*)gate.data,
        (float*)dispatch.data, (float*)combine.data, tokens, E, C);
  else
    moe_masks_kernel<bf16><<<grid_for(tokens, 256), 256, 0, s>>>(
        (const int32_t*)expert.data, (const int32_t*)slot.data, (const float*)gate.data,
        (bf16*)dispatch.data, (bf16*)combine.data, tokens, E, C);
  return launched(s);
}
