// GShard-style MoE routing and dispatch/combine permutations (config C3).
//
// The reference consumes a given one-hot dispatch tensor through a dense Dot
// (tests/test_acceptance.py:326-349); gating is out of its scope.
// The rule is pinned by paper_2105_04663_b200/moe.py::route_topk (GShard
// Top2Gating order): choice c of a token is the first max of its logits over
// the experts not chosen yet; slots are assigned choice by choice -- every
// first choice of a batch row before any second choice -- as the number of
// earlier tokens of the row with the same expert at this choice plus the
// kept (capacity-truncated) slots of that expert from earlier choices; a
// slot >= capacity is dropped.  Gates: top-1 the softmax probability,
// top-k the chosen probabilities renormalised to sum to one.
//
// route:    one warp per (partition, batch row); tokens in chunks of 32 lanes.
//           __match_any_sync groups lanes by expert -> in-chunk rank by popc of
//           the lower-lane mask; per-expert running counts live in shared
//           memory (the scan carry).  One scan pass per choice.  Integer
//           results are bit-exact.
// dispatch: expert buffers [E, C, M] filled by row gathers (16-B vector
//           copies, one warp per kept (token, choice)), empty slots zeroed --
//           equal to Dot(dispatch_mask, x) (one nonzero term per output).
// combine:  out[b,s,:] = sum_c gate_c * y[b, e_c, slot_c, :] accumulated in
//           fp64 and rounded once to f32 then bf16 -- equal to
//           Dot(combine_mask, y) as the reference evaluates it (f64
//           accumulation, simulator.py:258-275).
// Layouts: expert / slot s32 and gate f32 [.., B, S, K] (K = 1: [.., B, S]).
#include "common.cuh"

namespace spmd {

constexpr int MOE_MAX_E = 256;
constexpr int MOE_MAX_K = 4;

template <typename T>
__global__ void moe_route_kernel(const T* __restrict__ logits, int32_t* __restrict__ expert,
                                 int32_t* __restrict__ slot, float* __restrict__ gate,
                                 int64_t rows, int S, int E, int K, int capacity) {
  __shared__ int counts[8][MOE_MAX_E];   // this choice's running counts
  __shared__ int kept[8][MOE_MAX_E];     // kept slots of earlier choices
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t row = blockIdx.x * 8 + w; row < rows; row += (int64_t)gridDim.x * 8) {
    for (int e = lane; e < E; e += 32) kept[w][e] = 0;
    // choices of this lane's tokens are recomputed per pass from the logits
    // (K <= 4 passes over an [S, E] row: E <= 256 floats per token)
    for (int c = 0; c < K; ++c) {
      for (int e = lane; e < E; e += 32) counts[w][e] = kept[w][e];
      __syncwarp();
      for (int s0 = 0; s0 < S; s0 += 32) {
        const int s = s0 + lane;
        int pick = -1;
        if (s < S) {
          const T* l = logits + (row * S + s) * (int64_t)E;
          const int32_t* prev = expert + (row * S + s) * (int64_t)K;
          float m = -INFINITY;
          for (int e = 0; e < E; ++e) {
            bool taken = false;
            for (int j = 0; j < c; ++j) taken |= prev[j] == e;
            const float v = ld<T>(l[e]);
            if (!taken && (pick < 0 || v > m)) {
              m = v;
              pick = e;
            }
          }
        }
        const unsigned same = __match_any_sync(0xffffffffu, pick);
        const int rank = __popc(same & ((1u << lane) - 1));
        const int base = (pick >= 0) ? counts[w][pick] : 0;
        __syncwarp();
        if (pick >= 0) {
          expert[(row * S + s) * (int64_t)K + c] = pick;
          slot[(row * S + s) * (int64_t)K + c] = base + rank;
          if (rank == 0) counts[w][pick] = base + __popc(same);
        }
        __syncwarp();
      }
      // kept slots after this choice: min(total assigned, capacity)
      for (int e = lane; e < E; e += 32) kept[w][e] = min(counts[w][e], capacity);
      __syncwarp();
    }
    // gates: softmax over all experts; top-k renormalised over the choices
    for (int s = lane; s < S; s += 32) {
      const T* l = logits + (row * S + s) * (int64_t)E;
      float m = -INFINITY;
      for (int e = 0; e < E; ++e) m = fmaxf(m, ld<T>(l[e]));
      float denom = 0.f;
      for (int e = 0; e < E; ++e) denom += expf(ld<T>(l[e]) - m);
      const int64_t o = (row * S + s) * (int64_t)K;
      if (K == 1) {
        gate[o] = expf(ld<T>(l[expert[o]]) - m) / denom;
      } else {
        float pk[MOE_MAX_K], tot = 0.f;
        for (int c = 0; c < K; ++c) {
          pk[c] = expf(ld<T>(l[expert[o + c]]) - m) / denom;
          tot += pk[c];
        }
        for (int c = 0; c < K; ++c) gate[o + c] = pk[c] / tot;
      }
    }
    __syncwarp();
  }
}

// One warp per (token, choice) assignment a = t * K + c.  flags (the
// executor folds the MoE layer's Transpose(1,0,2,3) -> ReLU chain into the
// gather): MOE_EBCM writes [P][E][B][C][M] instead of [P][B][E][C][M],
// MOE_RELU applies ReLU to the copied values.
enum { MOE_EBCM = 1, MOE_RELU = 2 };

__device__ __forceinline__ int64_t moe_row(int flags, int64_t row, int e, int sl, int B, int E,
                                           int C) {
  if (!(flags & MOE_EBCM)) return (row * E + e) * (int64_t)C + sl;
  const int64_t p = row / B, b = row - p * B;
  return ((p * E + e) * (int64_t)B + b) * C + sl;
}

template <int V>
__global__ void moe_dispatch_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ expert,
                                    const int32_t* __restrict__ slot, uint16_t* __restrict__ out,
                                    int64_t assigns, int K, int S, int B, int E, int C, int M,
                                    int flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t a = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); a < assigns;
       a += warps) {
    const int sl = slot[a];
    if (sl >= C) continue;   // dropped (capacity)
    const int64_t t = a / K;
    const int64_t row = t / S;   // (partition, batch) row
    const int e = expert[a];
    const uint4* src = reinterpret_cast<const uint4*>(x + t * (int64_t)M);
    uint4* dst = reinterpret_cast<uint4*>(out + moe_row(flags, row, e, sl, B, E, C) * M);
    // 4 independent 16-byte loads in flight per lane (one row is M/V vectors)
    const int nv = M / V;
    for (int i0 = lane; i0 < nv; i0 += 128) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + 32 * u < nv) v[u] = __ldcs(src + i0 + 32 * u);
      if (flags & MOE_RELU) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint16_t* h = reinterpret_cast<uint16_t*>(&v[u]);
#pragma unroll
          for (int q = 0; q < 8; ++q) h[q] = relu_bits<uint16_t>(h[q], 1);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + 32 * u < nv) dst[i0 + 32 * u] = v[u];
    }
  }
}

// One warp per token: out = sum over kept choices of gate_c * y[e_c, slot_c].
// The gate is rounded to bf16 first (what the graph's bf16 combine tensor
// holds); each product of two bf16 values is exact in fp64 and the sum of
// <= K of them is rounded once to f32 and then to bf16 -- the value the
// oracle's f64 Dot(combine, y) produces (one nonzero term per choice).
__global__ void moe_combine_kernel(const bf16* __restrict__ y, const int32_t* __restrict__ expert,
                                   const int32_t* __restrict__ slot, const float* __restrict__ gate,
                                   bf16* __restrict__ out, int64_t tokens, int K, int S, int B,
                                   int E, int C, int M, int flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < tokens;
       t += warps) {
    const int64_t row = t / S;
    const uint4* src[MOE_MAX_K];
    double g[MOE_MAX_K];
    int n = 0;
    for (int c = 0; c < K; ++c) {
      const int sl = slot[t * K + c];
      if (sl >= C) continue;
      src[n] = reinterpret_cast<const uint4*>(
          y + moe_row(flags, row, expert[t * K + c], sl, B, E, C) * M);
      g[n++] = (double)__bfloat162float(__float2bfloat16_rn(gate[t * K + c]));
    }
    uint4* dst = reinterpret_cast<uint4*>(out + t * (int64_t)M);
    for (int i = lane; i < M / 8; i += 32) {
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int j = 0; j < n; ++j) {
        uint4 v = __ldcs(src[j] + i);
        if (flags & MOE_RELU) {
          uint16_t* r = reinterpret_cast<uint16_t*>(&v);
#pragma unroll
          for (int q = 0; q < 8; ++q) r[q] = relu_bits<uint16_t>(r[q], 1);
        }
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h[q]);
          acc[2 * q] = fma(g[j], (double)f.x, acc[2 * q]);
          acc[2 * q + 1] = fma(g[j], (double)f.y, acc[2 * q + 1]);
        }
      }
      uint4 o;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        oh[q] = __floats2bfloat162_rn((float)acc[2 * q], (float)acc[2 * q + 1]);
      dst[i] = o;
    }
  }
}

template <typename T>
__global__ void moe_masks_kernel(const int32_t* __restrict__ expert, const int32_t* __restrict__ slot,
                                 const float* __restrict__ gate, T* __restrict__ dispatch,
                                 T* __restrict__ combine, int64_t assigns, int K, int E, int C) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < assigns;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int sl = slot[a];
    if (sl < C) {
      const int64_t o = ((a / K) * E + expert[a]) * (int64_t)C + sl;
      dispatch[o] = st<T>(1.f);
      combine[o] = st<T>(gate[a]);
    }
  }
}

}  // namespace spmd

using namespace spmd;

// Choices per token of a routing tensor [.., B, S] (K = 1) or [.., B, S, K],
// given the rank of the per-token tensor it routes (tokens_rank: 2 for
// [B, S], i.e. x [B, S, M] minus the feature dim).
static int routing_k(const spmd_tensor& r, int tokens_rank) {
  if (r.rank == tokens_rank) return 1;
  if (r.rank == tokens_rank + 1 && r.dims[r.rank - 1] >= 1 && r.dims[r.rank - 1] <= MOE_MAX_K)
    return (int)r.dims[r.rank - 1];
  return 0;
}

// logits [P, B, S, E] (f32 or bf16) -> expert/slot s32, gate f32 [P, B, S(, K)].
extern "C" int spmd_moe_route(spmd_tensor logits, int capacity, spmd_tensor expert,
                              spmd_tensor slot, spmd_tensor gate, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(logits.rank == 3 && (logits.dtype == SPMD_F32 || logits.dtype == SPMD_BF16),
                 "moe route expects logits [B, S, E] f32/bf16");
  SPMD_CHECK_ARG(expert.dtype == SPMD_S32 && slot.dtype == SPMD_S32 && gate.dtype == SPMD_F32,
                 "moe route output dtypes");
  const int S = (int)logits.dims[1], E = (int)logits.dims[2];
  const int K = routing_k(expert, 2);
  SPMD_CHECK_ARG(K >= 1 && K <= E && routing_k(slot, 2) == K && routing_k(gate, 2) == K &&
                     expert.dims[0] == logits.dims[0] && expert.dims[1] == S,
                 "moe route outputs must be [B, S] or [B, S, k] with 1 <= k <= min(E, 4)");
  SPMD_CHECK_ARG(E <= MOE_MAX_E && capacity >= 0, "too many experts / bad capacity");
  const int64_t rows = logits.dims[0] * nparts;
  if (rows * S == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  unsigned grid = (unsigned)((rows + 7) / 8);
  if (logits.dtype == SPMD_F32)
    moe_route_kernel<float><<<grid, 256, 0, s>>>((const float*)logits.data, (int32_t*)expert.data,
                                                 (int32_t*)slot.data, (float*)gate.data, rows, S,
                                                 E, K, capacity);
  else
    moe_route_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)logits.data, (int32_t*)expert.data,
                                                (int32_t*)slot.data, (float*)gate.data, rows, S,
                                                E, K, capacity);
  return launched(s);
}

// x [P, B, S, M] bf16 -> out [P, B, E, C, M] bf16 (zero-filled empty slots).
// x [P, B, S, M] -> out [P, B, E, C, M] (flags & MOE_EBCM: [P, E, B, C, M]).
extern "C" int spmd_moe_dispatch_ex(spmd_tensor x, spmd_tensor expert, spmd_tensor slot,
                                    spmd_tensor out, int flags, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(x.dtype == SPMD_BF16 && out.dtype == SPMD_BF16 && x.rank == 3 && out.rank == 4,
                 "moe dispatch expects bf16 x [B,S,M] -> [B,E,C,M] / [E,B,C,M]");
  SPMD_CHECK_ARG(flags >= 0 && flags <= 3, "moe dispatch flags");
  const int ebcm = flags & MOE_EBCM;
  const int B = (int)x.dims[0], S = (int)x.dims[1], M = (int)x.dims[2];
  const int E = (int)out.dims[ebcm ? 0 : 1], C = (int)out.dims[2];
  const int K = routing_k(expert, 2);
  SPMD_CHECK_ARG(out.dims[ebcm ? 1 : 0] == B && out.dims[3] == M && M % 8 == 0 && K >= 1 &&
                     routing_k(slot, 2) == K,
                 "moe dispatch shape");
  cudaStream_t s = as_stream(stream);
  SPMD_CUDA_TRY(cudaMemsetAsync(out.data, 0, (size_t)numel(out) * nparts * 2, s));
  const int64_t assigns = x.dims[0] * S * nparts * K;
  if (assigns == 0) return SPMD_OK;
  moe_dispatch_kernel<8><<<grid_for(assigns * 32, 256), 256, 0, s>>>(
      (const uint16_t*)x.data, (const int32_t*)expert.data, (const int32_t*)slot.data,
      (uint16_t*)out.data, assigns, K, S, B, E, C, M, flags);
  return launched(s);
}

extern "C" int spmd_moe_dispatch(spmd_tensor x, spmd_tensor expert, spmd_tensor slot,
                                 spmd_tensor out, int64_t nparts, void* stream) {
  return spmd_moe_dispatch_ex(x, expert, slot, out, 0, nparts, stream);
}

// y [P, B, E, C, M] (flags & MOE_EBCM: [P, E, B, C, M]) bf16 -> out [P, B, S, M] bf16.
extern "C" int spmd_moe_combine_ex(spmd_tensor y, spmd_tensor expert, spmd_tensor slot,
                                   spmd_tensor gate, spmd_tensor out, int flags, int64_t nparts,
                                   void* stream) {
  SPMD_CHECK_ARG(y.dtype == SPMD_BF16 && out.dtype == SPMD_BF16 && y.rank == 4 && out.rank == 3,
                 "moe combine expects bf16 y [B,E,C,M] / [E,B,C,M] -> [B,S,M]");
  SPMD_CHECK_ARG(flags >= 0 && flags <= 3, "moe combine flags");
  const int ebcm = flags & MOE_EBCM;
  const int B = (int)out.dims[0], S = (int)out.dims[1], M = (int)out.dims[2];
  const int E = (int)y.dims[ebcm ? 0 : 1], C = (int)y.dims[2];
  const int K = routing_k(expert, 2);
  SPMD_CHECK_ARG(M % 8 == 0 && y.dims[3] == M && y.dims[ebcm ? 1 : 0] == B && K >= 1 &&
                     routing_k(slot, 2) == K && routing_k(gate, 2) == K,
                 "moe combine shape");
  const int64_t tokens = out.dims[0] * S * nparts;
  if (tokens == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  moe_combine_kernel<<<grid_for(tokens * 32, 256), 256, 0, s>>>(
      (const bf16*)y.data, (const int32_t*)expert.data, (const int32_t*)slot.data,
      (const float*)gate.data, (bf16*)out.data, tokens, K, S, B, E, C, M, flags);
  return launched(s);
}

extern "C" int spmd_moe_combine(spmd_tensor y, spmd_tensor expert, spmd_tensor slot,
                                spmd_tensor gate, spmd_tensor out, int64_t nparts, void* stream) {
  return spmd_moe_combine_ex(y, expert, slot, gate, out, 0, nparts, stream);
}

// Dense masks [P, B, S, E, C] (dispatch = 1 at every kept choice, combine =
// its gate) from a routing -- the tensors the reference's MoE graph consumes.
extern "C" int spmd_moe_masks(spmd_tensor expert, spmd_tensor slot, spmd_tensor gate,
                              spmd_tensor dispatch, spmd_tensor combine, int64_t nparts,
                              void* stream) {
  SPMD_CHECK_ARG(dispatch.rank == 4 && dispatch.dtype == combine.dtype, "moe masks shape");
  const int E = (int)dispatch.dims[2], C = (int)dispatch.dims[3];
  const int K = routing_k(expert, 2);
  SPMD_CHECK_ARG(K >= 1 && routing_k(slot, 2) == K && routing_k(gate, 2) == K,
                 "moe masks routing shape");
  const int64_t assigns = dispatch.dims[0] * dispatch.dims[1] * nparts * K;
  cudaStream_t s = as_stream(stream);
  const size_t bytes = (size_t)numel(dispatch) * nparts * elem_size(dispatch.dtype);
  SPMD_CUDA_TRY(cudaMemsetAsync(dispatch.data, 0, bytes, s));
  SPMD_CUDA_TRY(cudaMemsetAsync(combine.data, 0, bytes, s));
  if (assigns == 0) return SPMD_OK;
  if (dispatch.dtype == SPMD_F32)
    moe_masks_kernel<float><<<grid_for(assigns, 256), 256, 0, s>>>(
        (const int32_t*)expert.data, (const int32_t*)slot.data, (const float*)gate.data,
        (float*)dispatch.data, (float*)combine.data, assigns, K, E, C);
  else
    moe_masks_kernel<bf16><<<grid_for(assigns, 256), 256, 0, s>>>(
        (const int32_t*)expert.data, (const int32_t*)slot.data, (const float*)gate.data,
        (bf16*)dispatch.data, (bf16*)combine.data, assigns, K, E, C);
  return launched(s);
}
