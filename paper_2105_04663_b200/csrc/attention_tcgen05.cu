// Fused attention on tcgen05: replaces the op chain
//   logits = Dot(q, k)  [B,N,S,T]  ->  softmax over T  ->  ctx = Dot(probs, v)
// of the partitioned Transformer layer (the executor recognises the chain),
// never materialising the [B,N,S,T] logits/probabilities in HBM.
//
// One CTA per (128 query rows, head, batch); online softmax over 64-key tiles:
//   warp 0     TMA producer: Q once (D/64 boxes), K_j/V_j into a 2-slot ring
//   warp 1     MMA issuer:   S_j = Q K_j^T -> TMEM (double-buffered S),
//                            O += P_j V_j  -> TMEM (O: D fp32 columns)
//   warp 2     TMEM allocator
//   warps 4-7  softmax/correction: row max/sum in fp32 (one row per thread),
//              P_j (bf16) written to shared memory in the UMMA SW128 K-major
//              layout, O rescaled in TMEM when the running max moves, final
//              O / l -> bf16 staged in shared memory -> TMA bulk store.
// Layouts: q [B,S,N,D], k/v [B,T,N,D] (the QKV projection outputs), out
// [B,N,S,D] (the ctx Dot's output) -- all read/written with 4-D tensor maps,
// the partition stack folded into B.  Numerics: exp2 on log2e-scaled fp32,
// fp32 accumulation, P rounded to bf16 for the PV MMA.
#include "tcgen05.cuh"

#include <string.h>

namespace spmd {

template <int D>
struct AttnSmem {
  static constexpr int Q_BYTES = 128 * D * 2;
  static constexpr int KV_TILE = 64 * D * 2;            // one K or V tile
  static constexpr int SLOT = 2 * KV_TILE;              // K + V
  static constexpr int P_BYTES = 128 * 64 * 2;          // one P buffer (2 used)
  static constexpr int Q_OFF = 0;
  static constexpr int KV_OFF = Q_BYTES;
  static constexpr int P_OFF = KV_OFF + 2 * SLOT;
  static constexpr int BAR_OFF = P_OFF + 2 * P_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

struct AttnShape {
  int S, T, N, Bp;     // Bp = partitions * batch
  float scale_log2e;   // softmax scale * log2(e)
  // output for direct stores (persistent kernel): element strides of a
  // query row, a head and a batch (the [B,S,N,D] or [B,N,S,D] layout)
  bf16* out;
  int64_t o_row, o_head, o_batch;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (FFMA2 / FADD2, sm_100): the softmax warps are
// issue-bound, and the scale and the row sum halve their instruction count
// (+1.2-1.5% best-of-4 same-box, profiles/r2_attn_ab_f2.log).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int D>
__global__ void __launch_bounds__(256, 1)
    attention_tcgen05(const __grid_constant__ CUtensorMap map_q,
                      const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v,
                      const __grid_constant__ CUtensorMap map_o, AttnShape g) {
  typedef AttnSmem<D> L;
  constexpr int DC = D / 64;                  // 64-wide D chunks
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;     // [2]
  uint64_t* kv_empty = bars + 3;    // [2]
  uint64_t* s_full = bars + 5;      // [2]
  uint64_t* s_free = bars + 7;      // [2]
  uint64_t* p_full = bars + 9;      // [2] per P buffer
  uint64_t* pv_done = bars + 11;    // [2] per P buffer
  uint32_t* tmem_slot = (uint32_t*)(bars + 13);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int st = blockIdx.x % ((g.S + 127) / 128);
  const int rest = blockIdx.x / ((g.S + 127) / 128);
  const int n = rest % g.N, b = rest / g.N;
  const int nT = (g.T + 63) / 64;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: O [0, 256); S double-buffered [256, 512).  TP: P(t)
  // overwrites the first 64 columns of S(t)'s buffer (packed bf16) -- the
  // next S UMMA into that buffer is issued after PV(t) by the same thread,
  // and tcgen05.mma operations from one thread execute in issue order
  const uint32_t O_COL = 0, S_COL = 256;   // S buffers at 256 and 320

  uint8_t* sq = smem + L::Q_OFF;
  uint8_t* skv = smem + L::KV_OFF;
  uint8_t* sp = smem + L::P_OFF;

  if (warp == 0 && lane == 0) {
    // ---------------- producer ----------------
    mbar_expect_tx(q_full, L::Q_BYTES);
#pragma unroll
    for (int c = 0; c < DC; ++c) tma_load_4d(sq + c * 16384, &map_q, q_full, c * 64, st * 128, n, b);
    for (int j = 0; j < nT; ++j) {
      const int slot = j & 1;
      mbar_wait(&kv_empty[slot], ((j >> 1) & 1) ^ 1);
      uint8_t* kk = skv + slot * L::SLOT;
      uint8_t* vv = kk + L::KV_TILE;
      mbar_expect_tx(&kv_full[slot], L::SLOT);
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        tma_load_4d(kk + c * 8192, &map_k, &kv_full[slot], c * 64, j * 64, n, b);
        tma_load_4d(vv + c * 8192, &map_v, &kv_full[slot], c * 64, j * 64, n, b);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc_s = make_idesc(128, 64, 0, 0);
    const uint32_t idesc_o = make_idesc(128, D, 0, 1);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int slot = j & 1;
      mbar_wait(&kv_full[slot], (j >> 1) & 1);
      if (j >= 2) mbar_wait(&s_free[slot], ((j >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t qa = smem_u32(sq), ka = smem_u32(skv + slot * L::SLOT);
#pragma unroll
      for (int c = 0; c < DC; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma(tmem + S_COL + slot * 64, make_desc(qa + c * 16384 + k * 32, 16, 1024),
                 make_desc(ka + c * 8192 + k * 32, 16, 1024), idesc_s, (c | k) != 0);
      tc_commit(&s_full[slot]);
    };
    auto issue_pv = [&](int j) {
      const int slot = j & 1;           // K/V slot == P buffer index
      mbar_wait(&p_full[slot], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t pa = smem_u32(sp + slot * L::P_BYTES);
      const uint32_t va = smem_u32(skv + slot * L::SLOT + L::KV_TILE);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma(tmem + O_COL, make_desc(pa + k * 32, 16, 1024),
               make_desc(va + k * 2048, 8192, 1024), idesc_o, (j | k) != 0);
      tc_commit(&pv_done[slot]);
      tc_commit(&kv_empty[slot]);
    };
    issue_s(0);
    for (int j = 1; j < nT; ++j) {
      issue_s(j);
      issue_pv(j - 1);
    }
    issue_pv(nT - 1);
  } else if (warp >= 4) {
    // ---------------- softmax / correction / epilogue ----------------
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const int srow = st * 128 + row;
    (void)srow;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nT; ++j) {
      const int slot = j & 1;
      mbar_wait(&s_full[slot], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32(tmem + lane_base + S_COL + slot * 64, r0);
      tmem_ld32(tmem + lane_base + S_COL + slot * 64 + 32, r1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[slot]);
      float s[64];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        s[i] = __uint_as_float(r0[i]) * g.scale_log2e;
        s[32 + i] = __uint_as_float(r1[i]) * g.scale_log2e;
      }
      const int valid = g.T - j * 64;          // mask keys beyond T
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (i >= valid) s[i] = -INFINITY;
        mx = fmaxf(mx, s[i]);
      }
      // Conditional rescaling (log2 domain): keep the reference max m unless
      // this tile exceeds it by more than 2^8; exp2(s - m) then stays <= 256
      // and the final O / l is unchanged mathematically.
      float alpha = 1.f;
      bool resc = false;
      if (m == -INFINITY) {
        m = mx;                                  // first finite max: nothing in O yet
      } else if (mx > m + 8.f) {
        alpha = ex2(m - mx);
        m = mx;
        resc = true;
      }
      const float mb = m == -INFINITY ? 0.f : m;
      float rs = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        s[i] = ex2(s[i] - mb);
        rs += s[i];
      }
      l = l * alpha + rs;
      const int pb = j & 1;
      // P buffer pb was last read by PV_{j-2}.
      if (j >= 2) mbar_wait(&pv_done[pb], ((j >> 1) - 1) & 1);
      // O rescale needs every earlier PV (PV_{j-1}) complete.
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
        mbar_wait(&pv_done[pb ^ 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_base + O_COL + c, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tmem + lane_base + O_COL + c, o);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      // P_j (bf16) -> smem, SW128 K-major rows of 64 keys.
      uint8_t* prow = sp + pb * L::P_BYTES + row * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint4 v;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int t = 0; t < 4; ++t) h[t] = __floats2bfloat162_rn(s[q * 8 + 2 * t], s[q * 8 + 2 * t + 1]);
        *reinterpret_cast<uint4*>(prow + ((q ^ (row & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
    }
    // Final: O / l -> bf16 -> smem (Q area, SW128 chunks) -> TMA store.
    mbar_wait(&pv_done[(nT - 1) & 1], ((nT - 1) >> 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + O_COL + c, o);
      uint8_t* orow = sq + (c / 64) * 16384 + row * 128;
      const int qbase = (c % 64) / 8;          // 16-B chunk index within the 128-B row
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          h[t] = __floats2bfloat162_rn(__uint_as_float(o[q * 8 + 2 * t]) * inv,
                                       __uint_as_float(o[q * 8 + 2 * t + 1]) * inv);
        *reinterpret_cast<uint4*>(orow + (((qbase + q) ^ (row & 7)) << 4)) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 128) {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        asm volatile(
            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::
                "l"(reinterpret_cast<uint64_t>(&map_o)),
            "r"(smem_u32(sq + c * 16384)), "r"(c * 64), "r"(st * 128), "r"(n), "r"(b)
            : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      bulk_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2, UMMA M=256): the pair owns 256 query rows
// (128 per CTA) and splits every K tile by keys (32 per CTA) and every V tile
// by head-dim columns (D/2 per CTA), so each K/V byte crosses L2->SMEM once
// per 256 query rows -- the single-CTA kernel is L2-bandwidth bound at D=256.
// Leader CTA issues the MMAs; S and O land in each CTA's own TMEM half;
// softmax/P/correction/store run in both CTAs on their own rows.
// ---------------------------------------------------------------------------
template <int D>
struct Attn2Smem {
  static constexpr int Q_BYTES = 128 * D * 2;           // own 128 rows
  static constexpr int K_HALF = 32 * D * 2;             // 32 keys x D
  static constexpr int V_HALF = 64 * (D / 2) * 2;       // 64 keys x D/2
  static constexpr int SLOT = K_HALF + V_HALF;
  static constexpr int STAGES = 3;
  static constexpr int P_BYTES = 128 * 64 * 2;
  static constexpr int KV_OFF = Q_BYTES;
  static constexpr int P_OFF = KV_OFF + STAGES * SLOT;
  static constexpr int BAR_OFF = P_OFF + 2 * P_BYTES;
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;
};

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    attention_tcgen05_2sm(const __grid_constant__ CUtensorMap map_q,
                          const __grid_constant__ CUtensorMap map_k,
                          const __grid_constant__ CUtensorMap map_v,
                          const __grid_constant__ CUtensorMap map_o, AttnShape g) {
  typedef Attn2Smem<D> L;
  constexpr int DC = D / 64, NS = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;            // [NS] leader
  uint64_t* kv_empty = kv_full + NS;       // [NS] both (multicast)
  uint64_t* s_full = kv_empty + NS;        // [2] both (multicast)
  uint64_t* s_free = s_full + 2;           // [2] leader, 8 arrivals
  uint64_t* p_full = s_free + 2;           // [2] leader, 8 arrivals
  uint64_t* pv_done = p_full + 2;          // [2] both (multicast)
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nSt = (g.S + 255) / 256;
  const int cl = blockIdx.x >> 1;
  const int st = cl % nSt;
  const int rest = cl / nSt;
  const int n = rest % g.N, b = rest / g.N;
  const int nT = (g.T + 63) / 64;
  const int row0 = st * 256 + rank * 128;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: O [0, 256); S double-buffered [256, 512).  TP: P(t)
  // overwrites the first 64 columns of S(t)'s buffer (packed bf16) -- the
  // next S UMMA into that buffer is issued after PV(t) by the same thread,
  // and tcgen05.mma operations from one thread execute in issue order
  const uint32_t O_COL = 0, S_COL = 256;
  uint8_t* sq = smem;
  uint8_t* skv = smem + L::KV_OFF;
  uint8_t* sp = smem + L::P_OFF;

  if (warp == 0 && lane == 0) {
    if (leader) mbar_expect_tx(q_full, 2 * L::Q_BYTES);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      tma_load_4d_2sm(sq + c * 16384, &map_q, q_full, c * 64, row0, n, b);
    for (int j = 0; j < nT; ++j) {
      const int slot = j % NS;
      mbar_wait(&kv_empty[slot], ((j / NS) & 1) ^ 1);
      uint8_t* kk = skv + slot * L::SLOT;
      uint8_t* vv = kk + L::K_HALF;
      if (leader) mbar_expect_tx(&kv_full[slot], 2 * L::SLOT);
#pragma unroll
      for (int c = 0; c < DC; ++c)
        tma_load_4d_2sm(kk + c * 4096, &map_k, &kv_full[slot], c * 64, j * 64 + rank * 32, n, b);
#pragma unroll
      for (int c = 0; c < DC / 2; ++c)
        tma_load_4d_2sm(vv + c * 8192, &map_v, &kv_full[slot], rank * (D / 2) + c * 64, j * 64, n,
                        b);
    }
  } else if (warp == 1 && lane == 0 && leader) {
    const uint32_t idesc_s = make_idesc(256, 64, 0, 0);
    const uint32_t idesc_o = make_idesc(256, D, 0, 1);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int slot = j % NS, sb = j & 1;
      mbar_wait(&kv_full[slot], (j / NS) & 1);
      if (j >= 2) mbar_wait(&s_free[sb], ((j >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t qa = smem_u32(sq), ka = smem_u32(skv + slot * L::SLOT);
#pragma unroll
      for (int c = 0; c < DC; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_2sm(tmem + S_COL + sb * 64, make_desc(qa + c * 16384 + k * 32, 16, 1024),
                    make_desc(ka + c * 4096 + k * 32, 16, 1024), idesc_s, (c | k) != 0);
      tc_commit_2sm_mc(&s_full[sb]);
    };
    auto issue_pv = [&](int j) {
      const int slot = j % NS, pb = j & 1;
      mbar_wait(&p_full[pb], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t pa = smem_u32(sp + pb * L::P_BYTES);
      const uint32_t va = smem_u32(skv + slot * L::SLOT + L::K_HALF);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma_2sm(tmem + O_COL, make_desc(pa + k * 32, 16, 1024),
                  make_desc(va + k * 2048, 8192, 1024), idesc_o, (j | k) != 0);
      tc_commit_2sm_mc(&pv_done[pb]);
      tc_commit_2sm_mc(&kv_empty[slot]);
    };
    issue_s(0);
    for (int j = 1; j < nT; ++j) {
      issue_s(j);
      issue_pv(j - 1);
    }
    issue_pv(nT - 1);
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nT; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32_nowait(tmem + lane_base + S_COL + sb * 64, r0);
      tmem_ld32_nowait(tmem + lane_base + S_COL + sb * 64 + 32, r1);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&s_free[sb]);
      float s[64];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        s[i] = __uint_as_float(r0[i]) * g.scale_log2e;
        s[32 + i] = __uint_as_float(r1[i]) * g.scale_log2e;
      }
      const int valid = g.T - j * 64;
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (i >= valid) s[i] = -INFINITY;
        mx = fmaxf(mx, s[i]);
      }
      float alpha = 1.f;
      bool resc = false;
      if (m == -INFINITY) {
        m = mx;
      } else if (mx > m + 8.f) {
        alpha = ex2(m - mx);
        m = mx;
        resc = true;
      }
      const float mb = m == -INFINITY ? 0.f : m;
      float rs = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        s[i] = ex2(s[i] - mb);
        rs += s[i];
      }
      l = l * alpha + rs;
      const int pb = j & 1;
      if (j >= 2) mbar_wait(&pv_done[pb], ((j >> 1) - 1) & 1);
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
        mbar_wait(&pv_done[pb ^ 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_base + O_COL + c, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tmem + lane_base + O_COL + c, o);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      uint8_t* prow = sp + pb * L::P_BYTES + row * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint4 v;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int t = 0; t < 4; ++t) h[t] = __floats2bfloat162_rn(s[q * 8 + 2 * t], s[q * 8 + 2 * t + 1]);
        *reinterpret_cast<uint4*>(prow + ((q ^ (row & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&p_full[pb]);
    }
    mbar_wait(&pv_done[(nT - 1) & 1], ((nT - 1) >> 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + O_COL + c, o);
      uint8_t* orow = sq + (c / 64) * 16384 + row * 128;
      const int qbase = (c % 64) / 8;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          h[t] = __floats2bfloat162_rn(__uint_as_float(o[q * 8 + 2 * t]) * inv,
                                       __uint_as_float(o[q * 8 + 2 * t + 1]) * inv);
        *reinterpret_cast<uint4*>(orow + (((qbase + q) ^ (row & 7)) << 4)) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 128) {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        asm volatile(
            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::
                "l"(reinterpret_cast<uint64_t>(&map_o)),
            "r"(smem_u32(sq + c * 16384)), "r"(c * 64), "r"(row0), "r"(n), "r"(b)
            : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      bulk_wait_all();
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// 4-D bf16 map with SW128: dims (D, rows, heads, batch) with element strides.
static bool encode4(CUtensorMap* map, void* base, int64_t d, int64_t rows, int64_t heads,
                    int64_t batch, int64_t st_row, int64_t st_head, int64_t st_batch,
                    int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)rows, (cuuint64_t)heads, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)st_row * 2, (cuuint64_t)st_head * 2,
                           (cuuint64_t)st_batch * 2};
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16) return false;
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int D>
static int launch_attention(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                            const CUtensorMap& mo, AttnShape g, cudaStream_t s) {
  typedef AttnSmem<D> L;
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)attention_tcgen05<D>, L::TOTAL, &attr_done)) return rc;
  const int64_t grid = (int64_t)((g.S + 127) / 128) * g.N * g.Bp;
  attention_tcgen05<D><<<(unsigned)grid, 256, L::TOTAL, s>>>(mq, mk, mv, mo, g);
  return launched(s);
}

// ---------------------------------------------------------------------------
// 128-key tiles for the CTA pair: S = Q.K^T per tile is one N=128 UMMA chain
// (64 keys per CTA), PV has K=128, and the per-key barrier / issue overheads
// halve.  P is single-buffered (32 KB): the softmax keeps its 128 values in
// registers while PV(j-1) drains, then writes P(j).  TMEM: O [0, D), S double
// buffer at 256 and 384.  SPMD_ATTN_KT=64 selects the 64-key kernel.
// ---------------------------------------------------------------------------
template <int D>
struct Attn2SmemK128 {
  static constexpr int Q_BYTES = 128 * D * 2;           // own 128 rows
  static constexpr int K_HALF = 64 * D * 2;             // 64 keys x D
  static constexpr int V_HALF = 128 * (D / 2) * 2;      // 128 keys x D/2
  static constexpr int SLOT = K_HALF + V_HALF;
  static constexpr int STAGES = D >= 256 ? 2 : 3;
  static constexpr int P_BYTES = 128 * 128 * 2;         // 128 rows x 128 keys
  static constexpr int KV_OFF = Q_BYTES;
  static constexpr int P_OFF = KV_OFF + STAGES * SLOT;
  static constexpr int BAR_OFF = P_OFF + P_BYTES;
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;
};

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    attention_tcgen05_2sm_k128(const __grid_constant__ CUtensorMap map_q,
                               const __grid_constant__ CUtensorMap map_k,
                               const __grid_constant__ CUtensorMap map_v,
                               const __grid_constant__ CUtensorMap map_o, AttnShape g) {
  typedef Attn2SmemK128<D> L;
  constexpr int DC = D / 64, NS = L::STAGES, KT = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;            // [NS] leader
  uint64_t* kv_empty = kv_full + NS;       // [NS] both (multicast)
  uint64_t* s_full = kv_empty + NS;        // [2] both (multicast)
  uint64_t* s_free = s_full + 2;           // [2] leader, 8 arrivals
  uint64_t* p_full = s_free + 2;           // [1] leader, 8 arrivals
  uint64_t* pv_done = p_full + 1;          // [1] both (multicast)
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nSt = (g.S + 255) / 256;
  const int cl = blockIdx.x >> 1;
  const int st = cl % nSt;
  const int rest = cl / nSt;
  const int n = rest % g.N, b = rest / g.N;
  const int nT = (g.T + KT - 1) / KT;
  const int row0 = st * 256 + rank * 128;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
    }
    mbar_init(p_full, 8);
    mbar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: O [0, 256); S double-buffered [256, 512).  TP: P(t)
  // overwrites the first 64 columns of S(t)'s buffer (packed bf16) -- the
  // next S UMMA into that buffer is issued after PV(t) by the same thread,
  // and tcgen05.mma operations from one thread execute in issue order
  const uint32_t O_COL = 0, S_COL = 256;
  uint8_t* sq = smem;
  uint8_t* skv = smem + L::KV_OFF;
  uint8_t* sp = smem + L::P_OFF;

  if (warp == 0 && lane == 0) {
    if (leader) mbar_expect_tx(q_full, 2 * L::Q_BYTES);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      tma_load_4d_2sm(sq + c * 16384, &map_q, q_full, c * 64, row0, n, b);
    for (int j = 0; j < nT; ++j) {
      const int slot = j % NS;
      mbar_wait(&kv_empty[slot], ((j / NS) & 1) ^ 1);
      uint8_t* kk = skv + slot * L::SLOT;
      uint8_t* vv = kk + L::K_HALF;
      if (leader) mbar_expect_tx(&kv_full[slot], 2 * L::SLOT);
      // K: this CTA's 64 keys, D in 64-wide chunks of 64 rows x 128 B
#pragma unroll
      for (int c = 0; c < DC; ++c)
        tma_load_4d_2sm(kk + c * 8192, &map_k, &kv_full[slot], c * 64, j * KT + rank * 64, n, b);
      // V: all 128 keys, this CTA's D/2 columns, chunks of 128 rows x 128 B
#pragma unroll
      for (int c = 0; c < DC / 2; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          tma_load_4d_2sm(vv + c * 16384 + h * 8192, &map_v, &kv_full[slot],
                          rank * (D / 2) + c * 64, j * KT + h * 64, n, b);
    }
  } else if (warp == 1 && lane == 0 && leader) {
    const uint32_t idesc_s = make_idesc(256, KT, 0, 0);
    const uint32_t idesc_o = make_idesc(256, D, 0, 1);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int slot = j % NS, sb = j & 1;
      mbar_wait(&kv_full[slot], (j / NS) & 1);
      if (j >= 2) mbar_wait(&s_free[sb], ((j >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t qa = smem_u32(sq), ka = smem_u32(skv + slot * L::SLOT);
#pragma unroll
      for (int c = 0; c < DC; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_2sm(tmem + S_COL + sb * KT, make_desc(qa + c * 16384 + k * 32, 16, 1024),
                     make_desc(ka + c * 8192 + k * 32, 16, 1024), idesc_s, (c | k) != 0);
      tc_commit_2sm_mc(&s_full[sb]);
    };
    auto issue_pv = [&](int j) {
      const int slot = j % NS;
      mbar_wait(p_full, j & 1);
      tc_fence_after();
      const uint32_t pa = smem_u32(sp);
      const uint32_t va = smem_u32(skv + slot * L::SLOT + L::K_HALF);
#pragma unroll
      for (int k = 0; k < KT / 16; ++k)
        tc_mma_2sm(tmem + O_COL, make_desc(pa + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                   make_desc(va + k * 2048, 16384, 1024), idesc_o, (j | k) != 0);
      tc_commit_2sm_mc(pv_done);
      tc_commit_2sm_mc(&kv_empty[slot]);
    };
    issue_s(0);
    for (int j = 1; j < nT; ++j) {
      issue_s(j);
      issue_pv(j - 1);
    }
    issue_pv(nT - 1);
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nT; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      float s[KT];
      {
        uint32_t r[4][32];
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld32_nowait(tmem + lane_base + S_COL + sb * KT + q * 32, r[q]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 32; ++i) s[q * 32 + i] = __uint_as_float(r[q][i]) * g.scale_log2e;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&s_free[sb]);
      const int valid = g.T - j * KT;
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        if (i >= valid) s[i] = -INFINITY;
        mx = fmaxf(mx, s[i]);
      }
      float alpha = 1.f;
      bool resc = false;
      if (m == -INFINITY) {
        m = mx;
      } else if (mx > m + 8.f) {
        alpha = ex2(m - mx);
        m = mx;
        resc = true;
      }
      const float mb = m == -INFINITY ? 0.f : m;
      float rs = 0.f;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        s[i] = ex2(s[i] - mb);
        rs += s[i];
      }
      l = l * alpha + rs;
      // P is single-buffered and O may need rescaling: PV(j-1) must be done
      if (j >= 1) mbar_wait(pv_done, (j - 1) & 1);
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_base + O_COL + c, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tmem + lane_base + O_COL + c, o);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int a = 0; a < 2; ++a) {          // two 64-key SW128 atoms
        uint8_t* prow = sp + a * 16384 + row * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint4 v;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
          for (int t = 0; t < 4; ++t)
            h[t] = __floats2bfloat162_rn(s[a * 64 + q * 8 + 2 * t], s[a * 64 + q * 8 + 2 * t + 1]);
          *reinterpret_cast<uint4*>(prow + ((q ^ (row & 7)) << 4)) = v;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(p_full);
    }
    mbar_wait(pv_done, (nT - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + O_COL + c, o);
      uint8_t* orow = sq + (c / 64) * 16384 + row * 128;
      const int qbase = (c % 64) / 8;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          h[t] = __floats2bfloat162_rn(__uint_as_float(o[q * 8 + 2 * t]) * inv,
                                       __uint_as_float(o[q * 8 + 2 * t + 1]) * inv);
        *reinterpret_cast<uint4*>(orow + (((qbase + q) ^ (row & 7)) << 4)) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 128) {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        asm volatile(
            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::
                "l"(reinterpret_cast<uint64_t>(&map_o)),
            "r"(smem_u32(sq + c * 16384)), "r"(c * 64), "r"(row0), "r"(n), "r"(b)
            : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      bulk_wait_all();
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int D>
static int launch_attention_2sm_k128(const CUtensorMap& mq, const CUtensorMap& mk,
                                     const CUtensorMap& mv, const CUtensorMap& mo, AttnShape g,
                                     cudaStream_t s) {
  typedef Attn2SmemK128<D> L;
  static_assert(L::TOTAL <= 232448, "attention k128 smem");
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)attention_tcgen05_2sm_k128<D>, L::TOTAL, &attr_done)) return rc;
  const int64_t grid = 2 * (int64_t)((g.S + 255) / 256) * g.N * g.Bp;
  attention_tcgen05_2sm_k128<D><<<(unsigned)grid, 256, L::TOTAL, s>>>(mq, mk, mv, mo, g);
  return launched(s);
}

template <int D>
static int launch_attention_2sm(const CUtensorMap& mq, const CUtensorMap& mk,
                                const CUtensorMap& mv, const CUtensorMap& mo, AttnShape g,
                                cudaStream_t s) {
  typedef Attn2Smem<D> L;
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)attention_tcgen05_2sm<D>, L::TOTAL, &attr_done)) return rc;
  const int64_t grid = 2 * (int64_t)((g.S + 255) / 256) * g.N * g.Bp;
  attention_tcgen05_2sm<D><<<(unsigned)grid, 256, L::TOTAL, s>>>(mq, mk, mv, mo, g);
  return launched(s);
}

// ---------------------------------------------------------------------------
// Persistent CTA-pair attention with two softmax warps per TMEM lane quarter
// (the default for D = 128 / 256).  Same data split as the 128-key-tile
// kernel above (pair = 256 query rows; K tiles split by keys, V tiles by
// head-dim halves), but:
//  * persistent: one CTA pair per two SMs walks (q-tile, head, batch) work
//    items; the Q buffer is released as soon as the item's last S MMA has
//    completed, so the next item's Q load and first S MMAs overlap this
//    item's last softmax and its epilogue (the O accumulator is only
//    overwritten by the next item's first PV MMA, which waits for P, i.e.
//    after the epilogue has read O out of TMEM);
//  * 8 softmax warps (2 per SMSP): warp (quarter q, half h) owns rows
//    32q..32q+31 and keys 64h..64h+63 of every 128-key tile, so two
//    independent instruction streams per SMSP hide the MUFU / TMEM-load /
//    barrier latencies the 4-warp kernel stalls on (ncu r1: 29% tensor-pipe
//    active).  The two warps of a quarter exchange their partial row max
//    through shared memory (named barrier per quarter pair) so both scale
//    their half of P by the same running max; row sums stay per warp and are
//    added in the epilogue;
//  * row max / row sum as 8-way trees, scale folded into one FFMA per exp2;
//  * separate K and V rings (a K slot frees after its S MMA, a V slot after
//    its PV MMA), K loaded one tile ahead of V;
//  * O drained after the NEXT item's first tile has been softmaxed (the
//    final-PV wait overlaps it), each softmax warp staging its own rows in
//    its own slice of the P buffer and storing them with TMA.
// Warps: 0 TMA producer, 1 MMA issuer (leader CTA), 2 TMEM allocator,
// 3 idle, 4-11 softmax / correction / epilogue.
// ---------------------------------------------------------------------------
template <int D>
struct AttnPSmem {
  static constexpr int Q_BYTES = 128 * D * 2;           // own 128 rows
  static constexpr int K_HALF = 64 * D * 2;             // own 64 keys x D
  static constexpr int V_HALF = 128 * (D / 2) * 2;      // 128 keys x own D/2
  static constexpr int STAGES = D >= 256 ? 2 : 4;       // per ring (K ring, V ring)
  static constexpr int P_BYTES = 128 * 128 * 2;         // 128 rows x 128 keys
  static constexpr int K_OFF = Q_BYTES;
  static constexpr int V_OFF = K_OFF + STAGES * K_HALF;
  static constexpr int P_OFF = V_OFF + STAGES * V_HALF;
  static constexpr int RED_OFF = P_OFF + P_BYTES;       // [2 halves][128 rows] f32
  static constexpr int BAR_OFF = RED_OFF + 1024;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// TP = true: P goes from the softmax warps into tensor memory over S
// (tcgen05.st, packed bf16) and the PV UMMA reads A from TMEM, so the
// P smem buffer is only the O drain's staging area.  That lets the softmax
// warps hand P(t) of a new item to the MMA warp BEFORE draining the previous
// item's O, and the drain releases O's columns (o_free) as soon as they are
// in registers -- the first PV of the next item no longer waits for the O
// stores.  TP = false: P staged in shared memory (SS UMMA).
template <int D, bool TP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attention_tcgen05_2sm_pp(const __grid_constant__ CUtensorMap map_q,
                             const __grid_constant__ CUtensorMap map_k,
                             const __grid_constant__ CUtensorMap map_v,
                             const __grid_constant__ CUtensorMap map_o, AttnShape g) {
  typedef AttnPSmem<D> L;
  constexpr int DC = D / 64, NS = L::STAGES, KT = 128, DH = D / 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + L::BAR_OFF);
  // Q per 64-column chunk c (the S UMMAs' K steps): at an item boundary
  // chunk c of the next Q loads as soon as the last S UMMA's chunk-c steps
  // are done, and the next item's first S starts on chunk 0 while the rest
  // streams in (one barrier for all of Q: -1.5% at the C2 shape, best of
  // 4 same-box rounds, profiles/r2_attn_ab_qchunk.log)
  uint64_t* q_full = bars + 0;             // [DC] leader, 1 arrival + tx
  uint64_t* q_empty = q_full + DC;         // [DC] both (multicast commit)
  // K and V have separate rings: a K slot frees when its S MMA completes, a
  // V slot when its PV MMA does, so K(j+2) streams in while PV(j) still runs
  // (one shared K+V ring of 2 slots waited for PV(j) -- ncu: the MMA warp
  // starved on the loads 27% of the time)
  uint64_t* k_full = q_empty + DC;        // [NS] leader
  uint64_t* k_empty = k_full + NS;         // [NS] both (multicast)
  uint64_t* v_full = k_empty + NS;         // [NS] leader
  uint64_t* v_empty = v_full + NS;         // [NS] both (multicast)
  uint64_t* s_full = v_empty + NS;         // [2] both (multicast)
  uint64_t* s_free = s_full + 2;           // [2] leader, 16 arrivals
  uint64_t* p_full = s_free + 2;           // [1] leader, 16 arrivals
  uint64_t* pv_done = p_full + 1;          // [1] both (multicast)
  uint64_t* o_free = pv_done + 1;          // [1] leader, 16 arrivals (TP: O drained to registers)
  uint32_t* tmem_slot = (uint32_t*)(o_free + 1);
  float* red = (float*)(smem + L::RED_OFF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nSt = (g.S + 255) / 256;
  const int items = nSt * g.N * g.Bp;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nT = (g.T + KT - 1) / KT;

  if (threadIdx.x == 0) {
    for (int c = 0; c < DC; ++c) {
      mbar_init(&q_full[c], 1);
      mbar_init(&q_empty[c], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 16);
    }
    mbar_init(p_full, 16);
    mbar_init(pv_done, 1);
    mbar_init(o_free, 16);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: O [0, 256); S double-buffered [256, 512).  TP: P(t)
  // overwrites the first 64 columns of S(t)'s buffer (packed bf16) -- the
  // next S UMMA into that buffer is issued after PV(t) by the same thread,
  // and tcgen05.mma operations from one thread execute in issue order
  const uint32_t O_COL = 0, S_COL = 256;
  uint8_t* sq = smem;
  uint8_t* sk = smem + L::K_OFF;
  uint8_t* sv = smem + L::V_OFF;
  uint8_t* sp = smem + L::P_OFF;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    // Flat order over this pair's tiles t: [Q(item) at an item's first
    // tile], K(t), then V(t-1) -- K runs one tile ahead of V, matching the
    // MMA order S(t+1) before PV(t).  K(t) goes first: its slot frees when
    // S(t-2) completes, V(t-1)'s only when PV(t-3) does (one UMMA group
    // later), so waiting for the V slot first delayed every K load
    // (same-box A/B: +0.3..1.2% median, profiles/r2_attn_ab_kfirst.log).
    const int my_items = cl < items ? (items - cl + ncl - 1) / ncl : 0;
    const int G = my_items * nT;
    int item = cl, j = 0, it = 0;          // coordinates of tile t
    int pn = 0, pb = 0, pj = 0;            // coordinates of tile t - 1
    auto load_v = [&](int tv) {            // V(tv) at the coordinates (pn, pb, pj)
      const int slot = tv % NS;
      mbar_wait(&v_empty[slot], ((tv / NS) & 1) ^ 1);
      uint8_t* vv = sv + slot * L::V_HALF;
      if (leader) mbar_expect_tx(&v_full[slot], 2 * L::V_HALF);
#pragma unroll
      for (int c = 0; c < DC / 2; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          tma_load_4d_2sm(vv + c * 16384 + h * 8192, &map_v, &v_full[slot],
                          (int)rank * DH + c * 64, pj * KT + h * 64, pn, pb);
    };
    for (int t = 0; t <= G; ++t) {
      if (t == G) {
        if (t >= 1) load_v(t - 1);
        break;
      }
      const int st = item % nSt, rest = item / nSt;
      const int n = rest % g.N, b = rest / g.N;
      if (j == 0) {
#pragma unroll 1
        for (int c = 0; c < DC; ++c) {
          if (it > 0) mbar_wait(&q_empty[c], (it - 1) & 1);
          if (leader) mbar_expect_tx(&q_full[c], 2 * (L::Q_BYTES / DC));
          tma_load_4d_2sm(sq + c * 16384, &map_q, &q_full[c], c * 64, st * 256 + (int)rank * 128,
                          n, b);
        }
        // Q is read once, from HBM: pull the next item's Q into L2 now, so
        // its load at the item boundary (after this item's last S MMA frees
        // the Q buffer) is an L2 hit and the tensor pipe does not idle on it
        const int nx = item + ncl;
        if (nx < items) {
          const int nst = nx % nSt, nrest = nx / nSt;
#pragma unroll
          for (int c = 0; c < DC; ++c)
            asm volatile(
                "cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(
                    reinterpret_cast<uint64_t>(&map_q)),
                "r"(c * 64), "r"(nst * 256 + (int)rank * 128), "r"(nrest % g.N), "r"(nrest / g.N)
                : "memory");
        }
      }
      const int slot = t % NS;
      mbar_wait(&k_empty[slot], ((t / NS) & 1) ^ 1);
      uint8_t* kk = sk + slot * L::K_HALF;
      if (leader) mbar_expect_tx(&k_full[slot], 2 * L::K_HALF);
#pragma unroll
      for (int c = 0; c < DC; ++c)
        tma_load_4d_2sm(kk + c * 8192, &map_k, &k_full[slot], c * 64, j * KT + (int)rank * 64, n,
                        b);
      if (t >= 1) load_v(t - 1);
      pn = n, pb = b, pj = j;
      if (++j == nT) {
        j = 0;
        item += ncl;
        ++it;
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (flat sequence over this pair's tiles) ----------------
    // The whole warp runs the loop (uniform control flow, so descriptors and
    // counters live in uniform registers); one elected lane issues.  An S
    // MMA here is only 64 tensor cycles, so per-MMA issue cost matters:
    // descriptors are precomputed and advanced by constants.
    const uint32_t idesc_s = make_idesc(256, KT, 0, 0);
    const uint32_t idesc_o = make_idesc(256, D, 0, 1);
    const int my_items = cl < items ? (items - cl + ncl - 1) / ncl : 0;
    const int G = my_items * nT;
    const uint64_t qd0 = make_desc(smem_u32(sq), 16, 1024);
    const uint64_t kd0 = make_desc(smem_u32(sk), 16, 1024);
    const uint64_t vd0 = make_desc(smem_u32(sv), 16384, 1024);
    const uint64_t pd0 = make_desc(smem_u32(sp), 16, 1024);
    constexpr uint32_t K16 = L::K_HALF >> 4, V16 = L::V_HALF >> 4;
    // S side counters (tile gs = 0, 1, ...) and PV side counters
    int s_j = 0, s_slot = 0, s_item = 0;
    uint32_t s_kvph = 0;
    int p_j = 0, p_slot = 0, p_item = 0;
    uint32_t p_vph = 0;
    auto issue_s = [&](int gi) {
      const int sb = gi & 1;
      mbar_wait(&k_full[s_slot], s_kvph);
      if (gi >= 2) mbar_wait(&s_free[sb], ((gi >> 1) - 1) & 1);
      const uint64_t kd = kd0 + (uint64_t)(s_slot * K16);
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        if (s_j == 0) mbar_wait(&q_full[c], s_item & 1);   // the item's first S: chunk by chunk
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_2sm(tmem + S_COL + sb * KT, qd0 + (uint64_t)((c * 16384 + k * 32) >> 4),
                       kd + (uint64_t)((c * 8192 + k * 32) >> 4), idesc_s, (c | k) != 0);
          // Q chunk c is free once the item's last S has used it
          if (s_j == nT - 1) tc_commit_2sm_mc(&q_empty[c]);
        }
        __syncwarp();
      }
      if (elect_one()) {
        tc_commit_2sm_mc(&s_full[sb]);
        tc_commit_2sm_mc(&k_empty[s_slot]);
      }
      __syncwarp();
      if (++s_slot == NS) {
        s_slot = 0;
        s_kvph ^= 1;
      }
      if (++s_j == nT) {
        s_j = 0;
        ++s_item;
      }
    };
    auto issue_pv = [&](int gi) {
      mbar_wait(&v_full[p_slot], p_vph);
      mbar_wait(p_full, gi & 1);
      // TP: the first PV of an item overwrites O -- wait until the previous
      // item's O is out of TMEM (in the softmax warps' registers)
      if (TP && p_j == 0 && p_item > 0) mbar_wait(o_free, (p_item - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t vd = vd0 + (uint64_t)(p_slot * V16);
        const uint32_t pa = tmem + S_COL + (uint32_t)((gi & 1) * KT);
#pragma unroll
        for (int k = 0; k < KT / 16; ++k) {
          if (TP)
            tc_mma_2sm_ts(tmem + O_COL, pa + (uint32_t)(k * 8), vd + (uint64_t)((k * 2048) >> 4),
                          idesc_o, (p_j | k) != 0);
          else
            tc_mma_2sm(tmem + O_COL, pd0 + (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4),
                       vd + (uint64_t)((k * 2048) >> 4), idesc_o, (p_j | k) != 0);
        }
        tc_commit_2sm_mc(pv_done);
        tc_commit_2sm_mc(&v_empty[p_slot]);
      }
      __syncwarp();
      if (++p_slot == NS) {
        p_slot = 0;
        p_vph ^= 1;
      }
      if (++p_j == nT) {
        p_j = 0;
        ++p_item;
      }
    };
    if (G > 0) {
      issue_s(0);
      // (issuing an item's last PV before the next item's first S -- whose
      // Q is still loading -- measured 5% slower: the new item's softmax
      // pipeline then starts later; profiles/r2_attn_ab_pvfirst.log)
      for (int gi = 1; gi < G; ++gi) {
        issue_s(gi);
        issue_pv(gi - 1);
      }
      issue_pv(G - 1);
    }
  } else if (warp >= 4) {
    // ---------------- softmax / correction / epilogue ----------------
    const int qd = warp & 3, h = (warp - 4) >> 2;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const int pair_bar = 1 + qd;          // the two warps of this lane quarter
    float* my_red = red + h * 128 + row;
    const float* other_red = red + (1 - h) * 128 + row;
    const float c = g.scale_log2e;        // > 0 (host-checked)
    // Flat loop over this pair's tiles.  At an item boundary the next item's
    // first tile is softmaxed BEFORE waiting for the previous item's last PV
    // and draining its O (ncu: the softmax warps spent 27% of their time in
    // the drain -- the final-PV wait, barriers and the smem/TMA store path).
    // O is written straight from registers to global memory (each thread one
    // row, its half of the head dim: 16-byte stores), so the drain needs no
    // shared memory, no named barriers and does not hold the P buffer.
    const int my_items = cl < items ? (items - cl + ncl - 1) / ncl : 0;
    const int G = my_items * nT;
    int item = cl, j = 0;
    int cst = 0, cn = 0, cb = 0;          // current item (query tile, head, batch)
    float m = -INFINITY, l = 0.f;         // running max (raw logits), this half's row sum
    // Drain of a finished item's O: each warp stages its 32 rows x 64
    // columns (one round of its half of the head dim) in the SW128 layout,
    // in exactly the 4 KB of the P buffer it writes P into (atom h, rows
    // 32q..32q+31) -- no other warp touches that region, so the drain needs
    // no cross-warp barrier -- and one lane stores the box with TMA (per-row
    // 16-byte global stores measured ~20% of the softmax warps' time: one
    // L1 transaction per lane).
    auto drain = [&](float lsum, int st_, int n_, int b_) {
      *my_red = lsum;
      named_sync(pair_bar, 64);
      const float lt = lsum + *other_red;
      named_sync(pair_bar, 64);
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      uint8_t* stage = sp + h * 16384 + qd * 4096;
      uint8_t* srow = stage + lane * 128;
#pragma unroll 1
      for (int rd = 0; rd < DH / 64; ++rd) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_base + O_COL + h * DH + rd * 64 + half * 32, o);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 v;
            __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              hv[u] = __floats2bfloat162_rn(__uint_as_float(o[q * 8 + 2 * u]) * inv,
                                            __uint_as_float(o[q * 8 + 2 * u + 1]) * inv);
            *reinterpret_cast<uint4*>(srow + (((half * 4 + q) ^ (row & 7)) << 4)) = v;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], "
              "[%1];" ::"l"(reinterpret_cast<uint64_t>(&map_o)),
              "r"(smem_u32(stage)), "r"(h * DH + rd * 64),
              "r"(st_ * 256 + (int)rank * 128 + qd * 32), "r"(n_), "r"(b_)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
      }
    };
    // TP drain: all of this thread's O columns (its row, its half of the head
    // dim) into registers first, release O (o_free), then normalise and
    // store through this warp's 4 KB staging slice, 64 columns per TMA box.
    auto drain_tp = [&](float lsum, int st_, int n_, int b_, bool release) {
      constexpr int NQ = DH / 32;
      uint32_t o[NQ][32];
#pragma unroll
      for (int q = 0; q < NQ; ++q) tmem_ld32_nowait(tmem + lane_base + O_COL + h * DH + q * 32, o[q]);
      *my_red = lsum;
      named_sync(pair_bar, 64);
      const float lt = lsum + *other_red;
      named_sync(pair_bar, 64);
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      tmem_wait_ld();
      if (release) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(o_free);
      }
      uint8_t* stage = sp + h * 16384 + qd * 4096;
      uint8_t* srow = stage + lane * 128;
#pragma unroll
      for (int rd = 0; rd < DH / 64; ++rd) {
        // the staging slice is free once the previous box's store has read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int half = 0; half < 2; ++half)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 v;
            __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              hv[u] = __floats2bfloat162_rn(__uint_as_float(o[rd * 2 + half][q * 8 + 2 * u]) * inv,
                                            __uint_as_float(o[rd * 2 + half][q * 8 + 2 * u + 1]) * inv);
            *reinterpret_cast<uint4*>(srow + (((half * 4 + q) ^ (row & 7)) << 4)) = v;
          }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], "
              "[%1];" ::"l"(reinterpret_cast<uint64_t>(&map_o)),
              "r"(smem_u32(stage)), "r"(h * DH + rd * 64),
              "r"(st_ * 256 + (int)rank * 128 + qd * 32), "r"(n_), "r"(b_)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    };
    for (int t = 0; t < G; ++t) {
      float l_prev = 0.f;
      int pst = cst, pn = cn, pb = cb;
      if (j == 0) {
        const int rest = item / nSt;
        cst = item % nSt, cn = rest % g.N, cb = rest / g.N;
        l_prev = l;
        m = -INFINITY;
        l = 0.f;
      }
      const int sb = t & 1;
      mbar_wait(&s_full[sb], (t >> 1) & 1);
      tc_fence_after();
      float s[64];
      {
        uint32_t r[2][32];
        tmem_ld32_nowait(tmem + lane_base + S_COL + sb * KT + h * 64, r[0]);
        tmem_ld32_nowait(tmem + lane_base + S_COL + sb * KT + h * 64 + 32, r[1]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int i = 0; i < 32; ++i) s[q * 32 + i] = __uint_as_float(r[q][i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&s_free[sb]);
      const int valid = g.T - j * KT - h * 64;
      if (valid < 64) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (i >= valid) s[i] = -INFINITY;
      }
      float t8[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) t8[a] = s[a];
#pragma unroll
      for (int i = 8; i < 64; ++i) t8[i & 7] = fmaxf(t8[i & 7], s[i]);
      float pm = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                       fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7])));
      *my_red = pm;
      named_sync(pair_bar, 64);
      const float mx = fmaxf(pm, *other_red);
      named_sync(pair_bar, 64);          // red is rewritten next tile
      float alpha = 1.f;
      bool resc = false;
      if (m == -INFINITY) {
        m = mx;
      } else if ((mx - m) * c > 8.f) {    // rescale only when the max grows by > 2^8
        alpha = ex2((m - mx) * c);
        m = mx;
        resc = true;
      }
      const float nmc = m == -INFINITY ? 0.f : -m * c;
      {
        const uint64_t c2 = f2pack(c, c), n2 = f2pack(nmc, nmc);
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float a, b;
          f2unpack(ffma2(f2pack(s[i], s[i + 1]), c2, n2), a, b);
          s[i] = ex2(a);
          s[i + 1] = ex2(b);
        }
        uint64_t t4[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) t4[a] = f2pack(s[2 * a], s[2 * a + 1]);
#pragma unroll
        for (int i = 8; i < 64; i += 2)
          t4[(i >> 1) & 3] = fadd2(t4[(i >> 1) & 3], f2pack(s[i], s[i + 1]));
        t4[0] = fadd2(t4[0], t4[1]);
        t4[2] = fadd2(t4[2], t4[3]);
        t4[0] = fadd2(t4[0], t4[2]);
        float lo, hi;
        f2unpack(t4[0], lo, hi);
        l = l * alpha + (lo + hi);
      }
      if (TP) {
        // PV(t-1) landed: needed by an O rescale / drain, and waited on every
        // tile so this warp never falls two phases behind pv_done (a parity
        // wait cannot tell phase k from k-2: skipping the wait on tiles
        // without a rescale let a later rescale pass early now and then)
        if (t >= 1) mbar_wait(pv_done, (t - 1) & 1);
        if (j > 0 && __any_sync(0xffffffffu, resc)) {
          tc_fence_after();
#pragma unroll 1
          for (int cc = 0; cc < DH; cc += 32) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_base + O_COL + h * DH + cc, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tmem + lane_base + O_COL + h * DH + cc, o);
          }
        }
        // P(t) into TMEM over S(t): both warps of this lane quarter finished
        // reading S(t) before the max-exchange barriers above
        {
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(s[2 * i], s[2 * i + 1]);
            pk[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          tmem_st32(tmem + lane_base + S_COL + sb * KT + h * 32, pk);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(p_full);
        if (j == 0 && t > 0) {
          tc_fence_after();
          drain_tp(l_prev, pst, pn, pb, true);   // the previous item's O
        }
      } else {
        // P is single-buffered and O may need rescaling / draining: PV(t-1) done
        if (t >= 1) mbar_wait(pv_done, (t - 1) & 1);
        if (j == 0 && t > 0) {
          tc_fence_after();
          drain(l_prev, pst, pn, pb);       // previous item's O, before PV(t) overwrites it
        }
        if (j > 0 && __any_sync(0xffffffffu, resc)) {
          tc_fence_after();
  #pragma unroll 1
          for (int cc = 0; cc < DH; cc += 32) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_base + O_COL + h * DH + cc, o);
  #pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tmem + lane_base + O_COL + h * DH + cc, o);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        uint8_t* prow = sp + h * 16384 + row * 128;   // SW128 atom h = keys 64h..64h+63
  #pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint4 v;
          __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
  #pragma unroll
          for (int u = 0; u < 4; ++u)
            hv[u] = __floats2bfloat162_rn(s[q * 8 + 2 * u], s[q * 8 + 2 * u + 1]);
          *reinterpret_cast<uint4*>(prow + ((q ^ (row & 7)) << 4)) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(p_full);
      }
      if (++j == nT) {
        j = 0;
        item += ncl;
      }
    }
    if (G > 0) {
      mbar_wait(pv_done, (G - 1) & 1);
      tc_fence_after();
      if (TP)
        drain_tp(l, cst, cn, cb, false);
      else
        drain(l, cst, cn, cb);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int D, bool TP>
static int launch_attention_2sm_pp(const CUtensorMap& mq, const CUtensorMap& mk,
                                   const CUtensorMap& mv, const CUtensorMap& mo, AttnShape g,
                                   cudaStream_t s) {
  typedef AttnPSmem<D> L;
  static_assert(L::TOTAL <= 232448, "persistent attention smem");
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)attention_tcgen05_2sm_pp<D, TP>, L::TOTAL, &attr_done))
    return rc;
  const int64_t items = (int64_t)((g.S + 255) / 256) * g.N * g.Bp;
  const int pairs = sm_budget() / 2;
  const int64_t clusters = items < pairs ? items : pairs;
  attention_tcgen05_2sm_pp<D, TP><<<(unsigned)(2 * clusters), 384, L::TOTAL, s>>>(mq, mk, mv, mo,
                                                                                 g);
  return launched(s);
}

}  // namespace spmd

using namespace spmd;

// q [B,S,N,D], k/v [B,T,N,D] -> out [B,N,S,D] = softmax(scale * q.k^T) . v
extern "C" int spmd_attention_layout(spmd_tensor q, spmd_tensor k, spmd_tensor v,
                                     spmd_tensor out, float scale, int out_bsnd, int64_t nparts,
                                     void* stream) {
  SPMD_CHECK_ARG(q.dtype == SPMD_BF16 && k.dtype == SPMD_BF16 && v.dtype == SPMD_BF16 &&
                     out.dtype == SPMD_BF16 && q.rank == 4 && k.rank == 4 && v.rank == 4 &&
                     out.rank == 4,
                 "attention expects bf16 q[B,S,N,D], k/v[B,T,N,D], out[B,N,S,D] or [B,S,N,D]");
  const int64_t B = q.dims[0], S = q.dims[1], N = q.dims[2], D = q.dims[3], T = k.dims[1];
  const int64_t od1 = out_bsnd ? S : N, od2 = out_bsnd ? N : S;
  SPMD_CHECK_ARG(k.dims[0] == B && k.dims[2] == N && k.dims[3] == D && v.dims[0] == B &&
                     v.dims[1] == T && v.dims[2] == N && v.dims[3] == D && out.dims[0] == B &&
                     out.dims[1] == od1 && out.dims[2] == od2 && out.dims[3] == D,
                 "attention shape mismatch");
  if (!(D == 64 || D == 128 || D == 256)) return SPMD_ERR_UNSUPPORTED;
  const int64_t Bp = B * nparts;
  CUtensorMap mq, mk, mv, mo;
  bool ok = encode4(&mq, q.data, D, S, N, Bp, N * D, D, S * N * D, 128) &&
            encode4(&mk, k.data, D, T, N, Bp, N * D, D, T * N * D, 64) &&
            encode4(&mv, v.data, D, T, N, Bp, N * D, D, T * N * D, 64) &&
            (out_bsnd ? encode4(&mo, out.data, D, S, N, Bp, N * D, D, S * N * D, 128)
                      : encode4(&mo, out.data, D, S, N, Bp, D, S * D, N * S * D, 128));
  if (!ok) return SPMD_ERR_UNSUPPORTED;
  AttnShape g;
  g.S = (int)S;
  g.T = (int)T;
  g.N = (int)N;
  g.Bp = (int)Bp;
  g.scale_log2e = scale * 1.4426950408889634f;
  g.out = (bf16*)out.data;
  g.o_row = out_bsnd ? N * D : D;
  g.o_head = out_bsnd ? D : S * D;
  g.o_batch = S * N * D;
  cudaStream_t s = as_stream(stream);
  const int mode = option(OPT_ATTN_MODE) == 1 ? 1 : 2;
  // key tile: 128 for D=128 (549 vs 469 TF/s at T=1024), 64 for D=256 (equal at
  // T=1024, 993 vs 955 TF/s at T=4096: 3 K/V stages fit) -- profiles/r1_attention_kt.jsonl
  // option attn_kt: 0 = the persistent kernel with P in tensor memory
  // (default; same-box A/B, median of 8 rotated rounds: C2 shape +6%,
  // T=4096 +7%, D=128 +4%: profiles/r2_attn_ab_tp.log); 1 = the persistent
  // kernel with P in shared memory; 64 / 128 = the round-1 non-persistent
  // kernels with that key tile
  const int kt = (int)option(OPT_ATTN_KT);
  if (mode == 2 && D >= 128 && (kt == 0 || kt == 1) && scale > 0.f) {
    // persistent CTA pairs, 8 softmax warps, 128-key tiles (default); each
    // softmax warp stores its own 32-row output boxes
    CUtensorMap mo32;
    if (out_bsnd ? encode4(&mo32, out.data, D, S, N, Bp, N * D, D, S * N * D, 32)
                 : encode4(&mo32, out.data, D, S, N, Bp, D, S * D, N * S * D, 32)) {
      if (kt == 0) {
        if (D == 128) return launch_attention_2sm_pp<128, true>(mq, mk, mv, mo32, g, s);
        return launch_attention_2sm_pp<256, true>(mq, mk, mv, mo32, g, s);
      }
      if (D == 128) return launch_attention_2sm_pp<128, false>(mq, mk, mv, mo32, g, s);
      return launch_attention_2sm_pp<256, false>(mq, mk, mv, mo32, g, s);
    }
  }
  if (mode == 2 && D >= 128 && kt == 128) {
    // 128-key tiles: K boxes of 64 rows (mk), V boxes of 64 rows (mv)
    if (D == 128) return launch_attention_2sm_k128<128>(mq, mk, mv, mo, g, s);
    return launch_attention_2sm_k128<256>(mq, mk, mv, mo, g, s);
  }
  if (mode == 2 && D >= 128 && kt != 128) {
    CUtensorMap mk2;   // K split by keys: 32-row boxes
    if (encode4(&mk2, k.data, D, T, N, Bp, N * D, D, T * N * D, 32)) {
      if (D == 128) return launch_attention_2sm<128>(mq, mk2, mv, mo, g, s);
      return launch_attention_2sm<256>(mq, mk2, mv, mo, g, s);
    }
  }
  if (D == 64) return launch_attention<64>(mq, mk, mv, mo, g, s);
  if (D == 128) return launch_attention<128>(mq, mk, mv, mo, g, s);
  return launch_attention<256>(mq, mk, mv, mo, g, s);
}

// out[B,N,S,D] (the logits->softmax->ctx Dot chain's output layout).
extern "C" int spmd_attention(spmd_tensor q, spmd_tensor k, spmd_tensor v, spmd_tensor out,
                              float scale, int64_t nparts, void* stream) {
  return spmd_attention_layout(q, k, v, out, scale, 0, nparts, stream);
}
