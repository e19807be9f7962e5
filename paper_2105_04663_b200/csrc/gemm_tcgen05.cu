// BF16 generalised dot on 5th-gen tensor cores (sm_100a): TMA -> swizzled
// smem ring -> tcgen05.mma (fp32 accumulators in TMEM) -> tcgen05.ld epilogue.
//
// Replaces the reference's float64 einsum (simulator.py:258-275) for BF16.
// out[b, m, n] = sum_k A[b, m, k] * B[b, n, k] where A/B are views of the
// Dot operands: batch dims (<= 3, incl. the partition stack) and one merged
// M / N / K dim each.  Each operand may be K-major (K contiguous) or MN-major
// (M or N contiguous) -- both are native UMMA smem layouts, so weights stored
// [K, N] (x @ W) and activations stored [.., K] feed the tensor cores without
// any transpose pass.
//
// Kernel structure (persistent, one CTA per SM, 256 threads):
//   warp 0      TMA producer: kStages-deep ring of (A, B) tiles, mbarrier
//               expect-tx completion.
//   warp 1      MMA issuer: one elected thread issues BK/16 tcgen05.mma per
//               stage into a double-buffered TMEM accumulator (2 x BN cols),
//               tcgen05.commit frees smem stages / signals the epilogue.
//   warp 2      TMEM allocator (alloc/relinquish/dealloc).
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> fp32 regs -> (relu) -> bf16 ->
//               global; overlaps the next tile's MMAs via the second buffer.
// Tile 128 x BN x 64, BN in {128, 256}; SWIZZLE_128B everywhere.
#include "tcgen05.cuh"

#include <mutex>

#include <cuda.h>
#include <string.h>

namespace spmd {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int EPI_WARP0 = 4;

struct GemmShape {
  // wide kernel: non-null -> dynamic tile order (tile_ring_*): a global
  // counter hands out tiles first come, first served
  int* tile_counter;
  int M, N, K;
  int nb[3];            // batch extents (innermost first in tensor-map order)
  int mt, nt;           // tile counts
  int64_t tiles;
  int64_t out_batch_stride;   // elements between consecutive flat batches
  int a_mn, b_mn;
  int relu;
  int tma_store;        // epilogue through the bulk-tensor store path
  int group;            // rasterisation group size (tiles of the grouped dim)
  int raster_n;         // 0: group M-tiles and sweep N; 1: group N-tiles and sweep M
  int hint;             // 0 none, 1: A evict_last / B evict_first, 2: the reverse
  // Reduce-scatter epilogue (peer.cu): output column chunk j (sc_chunk wide)
  // goes to group position j's peer heap, slot sc_pos, buffer parity
  // (epoch + 1) & 1 -- P2P stores over NVLink, tile by tile.
  // Parity p starts at slot p * sc_par (peer.cu: a fixed stride for every
  // fused op, so consecutive ops of different sizes never overlap).
  int scatter, sc_g, sc_pos, sc_par;
  int64_t sc_chunk, sc_slot;
  bf16* sc_dst[8];
  const uint32_t* sc_epoch;
  int sc_tma;           // scatter through per-destination bulk-tensor store maps
  int store_hint;       // 1: output stores with an L2 evict_first policy
  int sc_rows;          // all-to-all (row-chunk) scatter, wide kernel only
  int64_t sc_rchunk;
  int sc_slot_base, sc_nslots;
  // wide kernel, plain store epilogue: C = A.B + resid (same [nbat][M][N]
  // layout as C), added in fp32 before the one rounding (spmd_dot_add)
  const bf16* resid;
};

// Per-destination store maps of the reduce-scatter epilogue: rank j's heap as
// (chunk cols, rows, 2 parities x gsize slots).
struct ScatterMaps {
  CUtensorMap m[8];
};

template <int BN, int STAGES>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 1024;        // 4 warps x 2 x 2 KB staging
  static constexpr int TOTAL = EPI_OFF + 8 * EPI_STAGE_BYTES + 1024;   // + align slack
};

__device__ __forceinline__ void tile_coords(const GemmShape& g, int64_t t, int& b, int& m, int& n) {
  const int64_t per = (int64_t)g.mt * g.nt;
  b = (int)(t / per);
  int r = (int)(t - (int64_t)b * per);
  // Grouped rasterisation: G tiles of one dim sweep the other dim together,
  // so one operand's group stays L2-resident while the other streams.
  const int G = g.group;
  const int ga = g.raster_n ? g.nt : g.mt;   // grouped dim extent
  const int gb = g.raster_n ? g.mt : g.nt;   // swept dim extent
  int group = r / (G * gb);
  int first = group * G;
  int gs = ga - first < G ? ga - first : G;
  int rr = r - group * G * gb;
  int x = first + rr % gs, y = rr / gs;
  m = g.raster_n ? y : x;
  n = g.raster_n ? x : y;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_c, bf16* __restrict__ out,
                      GemmShape g) {
  typedef Smem<BN, STAGES> L;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);   // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  const int kblocks = (g.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      int b, m, n;
      tile_coords(g, t, b, m, n);
      const int b0 = b % g.nb[0], b1 = (b / g.nb[0]) % g.nb[1], b2 = b / (g.nb[0] * g.nb[1]);
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        uint8_t* sb = sa + L::A_BYTES;
        mbar_expect_tx(&full[s], L::STAGE_BYTES);
        const int k0 = kb * BK;
        if (!g.a_mn) {
          tma_load_5d(sa, &map_a, &full[s], k0, m * BM, b0, b1, b2);
        } else {
#pragma unroll
          for (int c = 0; c < BM / 64; ++c)
            tma_load_5d(sa + c * (BK * 128), &map_a, &full[s], m * BM + c * 64, k0, b0, b1, b2);
        }
        if (!g.b_mn) {
          tma_load_5d(sb, &map_b, &full[s], k0, n * BN, b0, b1, b2);
        } else {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_5d(sb + c * (BK * 128), &map_b, &full[s], n * BN + c * 64, k0, b0, b1, b2);
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc(BM, BN, g.a_mn, g.b_mn);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * BN;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
        const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // K advance of 16 elements: +32 B inside a K-major 128 B row, or
          // +2 atoms (16 K-rows x 128 B) in an MN-major tile.
          const uint64_t ad = g.a_mn ? make_desc(sa + k * 2048, BK * 128, 1024)
                                     : make_desc(sa + k * 32, 16, 1024);
          const uint64_t bd = g.b_mn ? make_desc(sb + k * 2048, BK * 128, 1024)
                                     : make_desc(sb + k * 32, 16, 1024);
          tc_mma(d_tmem, ad, bd, idesc, (kb | k) != 0);
        }
        tc_commit(&empty[s]);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      tc_commit(&tfull[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ---------------- epilogue ----------------
    const int ew = warp - EPI_WARP0;          // == warp % 4 -> TMEM lanes 32*ew..
    uint8_t* epi = smem + L::EPI_OFF + ew * 2 * EPI_STAGE_BYTES;
    int chunk = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      int b, m, n;
      tile_coords(g, t, b, m, n);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int row = m * BM + ew * 32 + lane;
      bf16* orow = out + (int64_t)b * g.out_batch_stride + (int64_t)row * g.N;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + acc * BN + c0, r);
        const int col = n * BN + c0;
        if (g.tma_store) {
          if (col < g.N)
            epi_store_chunk(&map_c, epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu, col,
                            m * BM + ew * 32, b, lane);
        } else if (row < g.M && col < g.N) {
          __align__(16) bf16 v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float f = __uint_as_float(r[j]);
            if (g.relu) f = f > 0.f ? f : 0.f;
            v[j] = __float2bfloat16_rn(f);
          }
          if (col + 32 <= g.N && (g.N & 7) == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(orow + col + 8 * j) = reinterpret_cast<uint4*>(v)[j];
          } else {
            for (int j = 0; j < 32 && col + j < g.N; ++j) orow[col + j] = v[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): a CTA pair computes a 256 x 256 tile with
// UMMA M=256.  Each CTA stages its 128-row half of A and its 128-row half
// of B (N split) in its own smem; the leader CTA issues the MMAs, which read
// both CTAs' smem and write each CTA's own TMEM half.  Per-SM smem operand
// traffic halves versus the 1-CTA kernel -- the condition for feeding the
// tensor cores at full rate.
//   * TMA: .cta_group::2 loads complete on the LEADER's full barrier (peer
//     bit masked); the leader arms it with both CTAs' bytes.
//   * MMA commit multicasts to both CTAs' empty / tmem-full barriers.
//   * Epilogue warps of both CTAs release the leader's tmem-empty barrier
//     with remote (mapa) arrives.
// ---------------------------------------------------------------------------
constexpr int BM2 = 256, BN2 = 256, HALF = 128;

template <int STAGES>
struct Smem2 {
  static constexpr int A_BYTES = HALF * BK * 2;
  static constexpr int B_BYTES = HALF * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 1024;
  static constexpr int TOTAL = EPI_OFF + 8 * EPI_STAGE_BYTES + 1024;
};

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_bf16_tcgen05_2sm(const __grid_constant__ CUtensorMap map_a,
                          const __grid_constant__ CUtensorMap map_b,
                          const __grid_constant__ CUtensorMap map_c, bf16* __restrict__ out,
                          GemmShape g, const __grid_constant__ ScatterMaps smaps) {
  typedef Smem2<STAGES> L;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);   // 4 epilogue warps x 2 CTAs
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
  const int kblocks = (g.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    int s = 0;
    uint32_t ph = 0;
    uint64_t pol_last, pol_first;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    const int hint = g.hint != 0;
    const uint64_t pa = g.hint == 1 ? pol_last : pol_first;
    const uint64_t pb = g.hint == 1 ? pol_first : pol_last;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int b, m, n;
      tile_coords(g, t, b, m, n);
      const int b0 = b % g.nb[0], b1 = (b / g.nb[0]) % g.nb[1], b2 = b / (g.nb[0] * g.nb[1]);
      const int mrow = m * BM2 + rank * HALF, nrow = n * BN2 + rank * HALF;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        uint8_t* sb = sa + L::A_BYTES;
        if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
        const int k0 = kb * BK;
        if (!g.a_mn) {
          load_2sm(sa, &map_a, &full[s], k0, mrow, b0, b1, b2, hint, pa);
        } else {
#pragma unroll
          for (int c = 0; c < HALF / 64; ++c)
            load_2sm(sa + c * (BK * 128), &map_a, &full[s], mrow + c * 64, k0, b0, b1, b2, hint,
                     pa);
        }
        if (!g.b_mn) {
          load_2sm(sb, &map_b, &full[s], k0, nrow, b0, b1, b2, hint, pb);
        } else {
#pragma unroll
          for (int c = 0; c < HALF / 64; ++c)
            load_2sm(sb + c * (BK * 128), &map_b, &full[s], nrow + c * 64, k0, b0, b1, b2, hint,
                     pb);
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    const uint32_t idesc = make_idesc(BM2, BN2, g.a_mn, g.b_mn);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * BN2;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
        const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = g.a_mn ? make_desc(sa + k * 2048, BK * 128, 1024)
                                     : make_desc(sa + k * 32, 16, 1024);
          const uint64_t bd = g.b_mn ? make_desc(sb + k * 2048, BK * 128, 1024)
                                     : make_desc(sb + k * 32, 16, 1024);
          tc_mma_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0);
        }
        tc_commit_2sm_mc(&empty[s]);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      tc_commit_2sm_mc(&tfull[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ---------------- epilogue (both CTAs, own TMEM half) ----------------
    const int ew = warp - EPI_WARP0;
    uint8_t* epi = smem + L::EPI_OFF + ew * 2 * EPI_STAGE_BYTES;
    uint64_t store_pol = 0;
    if (g.store_hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(store_pol));
    const int par = g.scatter ? (int)((*(volatile const uint32_t*)g.sc_epoch + 1) & 1) : 0;
    const int64_t par_off = (int64_t)par * g.sc_par * g.sc_slot;
    int chunk = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int b, m, n;
      tile_coords(g, t, b, m, n);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int row = m * BM2 + rank * HALF + ew * 32 + lane;
      bf16* orow = out + (int64_t)b * g.out_batch_stride + (int64_t)row * g.N;
#pragma unroll 1
      for (int c0 = 0; c0 < BN2; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + acc * BN2 + c0, r);
        const int col = n * BN2 + c0;
        if (g.tma_store) {
          if (col < g.N)
            epi_store_chunk(&map_c, epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu, col,
                            m * BM2 + rank * HALF + ew * 32, b, lane, store_pol);
        } else if (g.scatter && g.sc_tma) {
          if (col < g.N) {
            const int j = (int)(col / g.sc_chunk);
            epi_store_chunk(&smaps.m[j], epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu,
                            (int)(col - j * g.sc_chunk), m * BM2 + rank * HALF + ew * 32,
                            par * g.sc_par + g.sc_pos, lane);
          }
        } else if (g.scatter) {
          if (row < g.M && col < g.N) {
            __align__(16) bf16 v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float f = __uint_as_float(r[j]);
              if (g.relu) f = f > 0.f ? f : 0.f;
              v[j] = __float2bfloat16_rn(f);
            }
            const int j = (int)(col / g.sc_chunk);
            const int64_t lc = col - j * g.sc_chunk;
            bf16* d = g.sc_dst[j] + par_off + g.sc_pos * g.sc_slot + (int64_t)row * g.sc_chunk + lc;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              reinterpret_cast<uint4*>(d)[q] = reinterpret_cast<uint4*>(v)[q];
          }
        } else if (row < g.M && col < g.N) {
          __align__(16) bf16 v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float f = __uint_as_float(r[j]);
            if (g.relu) f = f > 0.f ? f : 0.f;
            v[j] = __float2bfloat16_rn(f);
          }
          if (col + 32 <= g.N && (g.N & 7) == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(orow + col + 8 * j) = reinterpret_cast<uint4*>(v)[j];
          } else {
            for (int j = 0; j < 32 && col + j < g.N; ++j) orow[col + j] = v[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();
    // Peer stores globally visible before the completion signal (peer.cu).
    if (g.scatter) __threadfence_system();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// Wide CTA-pair variant: 256 x 512 pair tiles (two N=256 UMMAs per k-step
// into all 512 TMEM columns).  Per CTA and k-block: A 128 x 64 + B 256 x 64
// -> operand bytes per FLOP 25% lower than 256 x 256 and half the L2 reads
// of A per output; measured on the C2 FFN shapes: L2 traffic 171 -> ~96 GB,
// the layout cuBLAS picks for these shapes.  The accumulator fills TMEM, so
// tiles cannot double-buffer it: 8 epilogue warps (384 threads) drain it,
// two per TMEM lane quarter, each half the columns.
// ---------------------------------------------------------------------------
constexpr int WBN = 512;          // pair tile N
constexpr int WHALF_N = 256;      // N per UMMA

// ---------------------------------------------------------------------------
// Dynamic tile order for the persistent wide kernel.  A static round-robin
// (pair c takes tiles c, c+74, ...) lets the 74 pairs drift apart over ~110
// tiles, so the tiles in flight spread far beyond one raster group and L2
// reuse collapses: ncu on the C2 FFN-in GEMM measured 22-35 GB of DRAM reads
// (cuBLAS 12.5 GB) and, under the 1 kW power cap, ~7% lower SM clocks.  A
// non-persistent launch (the hardware hands tiles out in order) cut the
// DRAM reads to 13.5 GB but loses the epilogue/mainloop overlap.  Here the
// leader CTA's producer thread takes the next tile from a global counter and
// publishes it through a small ring (tile id in both CTAs' shared memory,
// mbarriers) to its peer producer, the MMA warp and the 16 epilogue warps:
// tiles are consumed in global order, the kernel stays persistent.
// ---------------------------------------------------------------------------
constexpr int TILE_RING = 4;
constexpr int TILE_RING_CONSUMERS = 1 + 1 + 16;   // peer producer, MMA warp, 2 x 8 epilogue warps

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}

// arrive on the barrier at the same smem offset in cluster CTA `cta`
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n.reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

__device__ __forceinline__ void st_cluster_u32(uint32_t* p, uint32_t cta, uint32_t v) {
  asm volatile(
      "{\n.reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "st.shared::cluster.u32 [ra], %2;\n}" ::"r"(smem_u32(p)),
      "r"(cta), "r"(v)
      : "memory");
}

// Scheduler side (leader producer): fetch the next tile and publish it in
// slot i % TILE_RING of both CTAs.  Returns the tile (>= g.tiles: done).
__device__ __forceinline__ int64_t ring_publish(const GemmShape& g, int32_t* ids, uint64_t* rfull,
                                                uint64_t* rempty, int i) {
  const int slot = i % TILE_RING;
  mbar_wait_cluster(&rempty[slot], ((i / TILE_RING) & 1) ^ 1);
  int t = atomicAdd(g.tile_counter, 1);
  if (t > g.tiles) t = (int)g.tiles;
  ids[slot] = t;
  st_cluster_u32((uint32_t*)&ids[slot], 1, (uint32_t)t);
  mbar_arrive_cta(&rfull[slot], 0);
  mbar_arrive_cta(&rfull[slot], 1);
  return t;
}

// Consumer side: the tile of slot i % TILE_RING; `notify` = this thread
// releases the slot (one arrival on the leader's ring-empty barrier).
__device__ __forceinline__ int64_t ring_take(int32_t* ids, uint64_t* rfull, uint64_t* rempty,
                                             int i, bool notify) {
  const int slot = i % TILE_RING;
  mbar_wait_cluster(&rfull[slot], (i / TILE_RING) & 1);
  const int64_t t = *(volatile int32_t*)&ids[slot];
  if (notify) mbar_arrive_cta(&rempty[slot], 0);
  return t;
}

// Lane `lane` of an epilogue warp holds row row0 + lane, columns [col, col + 32)
// of the tile in r[] (fp32 bits): add the residual's bf16 values in fp32.
__device__ __forceinline__ void add_resid_chunk(const GemmShape& g, int b, int row0, int col,
                                                int lane, uint32_t (&r)[32]) {
  const int row = row0 + lane;
  if (row >= g.M) return;
  const bf16* src = g.resid + (int64_t)b * g.out_batch_stride + (int64_t)row * g.N + col;
  if (col + 32 <= g.N && (((uintptr_t)src) & 15) == 0) {
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcs(reinterpret_cast<const uint4*>(src) + q);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      r[2 * i] = __float_as_uint(__uint_as_float(r[2 * i]) + f.x);
      r[2 * i + 1] = __float_as_uint(__uint_as_float(r[2 * i + 1]) + f.y);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (col + i < g.N) r[i] = __float_as_uint(__uint_as_float(r[i]) + __bfloat162float(src[i]));
  }
}

template <int STAGES>
struct SmemW {
  static constexpr int A_BYTES = HALF * BK * 2;              // 16 KB
  static constexpr int B_BYTES = 2 * HALF * BK * 2;          // 32 KB: 2 x 128 rows
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 1024;
  static constexpr int TOTAL = EPI_OFF + 16 * EPI_STAGE_BYTES + 1024;
};

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    gemm_bf16_tcgen05_2sm_wide(const __grid_constant__ CUtensorMap map_a,
                               const __grid_constant__ CUtensorMap map_b,
                               const __grid_constant__ CUtensorMap map_c, GemmShape g,
                               const __grid_constant__ ScatterMaps smaps) {
  typedef SmemW<STAGES> L;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint64_t* rfull = tempty + 1;            // [TILE_RING] tile-id ring (dynamic order)
  uint64_t* rempty = rfull + TILE_RING;    // [TILE_RING] leader only
  int32_t* ring_ids = (int32_t*)(rempty + TILE_RING);
  uint32_t* tmem_slot = (uint32_t*)(ring_ids + TILE_RING);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const bool dyn = g.tile_counter != nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < TILE_RING; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], TILE_RING_CONSUMERS);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 16);   // 8 epilogue warps x 2 CTAs
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
  const int kblocks = (g.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    int s = 0;
    uint32_t ph = 0;
    uint64_t pol_last, pol_first;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    const int hint = g.hint != 0;
    const uint64_t pa = g.hint == 1 ? pol_last : pol_first;
    const uint64_t pb = g.hint == 1 ? pol_first : pol_last;
    for (int64_t it = 0, t = cluster;; ++it) {
      if (dyn)
        t = leader ? ring_publish(g, ring_ids, rfull, rempty, (int)it)
                   : ring_take(ring_ids, rfull, rempty, (int)it, true);
      else if (it > 0)
        t += nclusters;
      if (t >= g.tiles) break;
      int b, m, n;
      tile_coords(g, t, b, m, n);
      const int b0 = b % g.nb[0], b1 = (b / g.nb[0]) % g.nb[1], b2 = b / (g.nb[0] * g.nb[1]);
      const int mrow = m * BM2 + rank * HALF;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        uint8_t* sb = sa + L::A_BYTES;
        if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
        const int k0 = kb * BK;
        if (!g.a_mn) {
          load_2sm(sa, &map_a, &full[s], k0, mrow, b0, b1, b2, hint, pa);
        } else {
#pragma unroll
          for (int c = 0; c < HALF / 64; ++c)
            load_2sm(sa + c * (BK * 128), &map_a, &full[s], mrow + c * 64, k0, b0, b1, b2, hint,
                     pa);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {   // UMMA j covers pair-tile cols [256j, 256j+256)
          const int nrow = n * WBN + j * WHALF_N + rank * HALF;
          uint8_t* sbj = sb + j * (HALF * BK * 2);
          if (!g.b_mn) {
            load_2sm(sbj, &map_b, &full[s], k0, nrow, b0, b1, b2, hint, pb);
          } else {
#pragma unroll
            for (int c = 0; c < HALF / 64; ++c)
              load_2sm(sbj + c * (BK * 128), &map_b, &full[s], nrow + c * 64, k0, b0, b1, b2,
                       hint, pb);
          }
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    // Descriptors are precomputed and advanced by constant offsets (the
    // 14-bit start field is addr >> 4; smem < 256 KB never carries out of
    // it).  Running the loop on the whole warp with one elected issuer (the
    // conv kernel's scheme, where a UMMA is only 64 tensor cycles) measured
    // no gain here (UMMA 256x256x16 = 128 cycles): -9% .. +2% per shape,
    // C2 step within noise (profiles/r2_gemm_ab_mmawarp.log).
    const uint32_t idesc = make_idesc(BM2, WHALF_N, g.a_mn, g.b_mn);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t a0 = g.a_mn ? make_desc(s0, BK * 128, 1024) : make_desc(s0, 16, 1024);
    const uint64_t b0 = g.b_mn ? make_desc(s0 + L::A_BYTES, BK * 128, 1024)
                               : make_desc(s0 + L::A_BYTES, 16, 1024);
    const uint32_t ka = g.a_mn ? (2048 >> 4) : (32 >> 4), kb16 = g.b_mn ? (2048 >> 4) : (32 >> 4);
    constexpr uint32_t STAGE16 = L::STAGE_BYTES >> 4, BJ16 = (HALF * BK * 2) >> 4;
    int s = 0;
    uint32_t ph = 0;
    uint32_t acc_ph = 0;
    for (int64_t it = 0, t = cluster;; ++it) {
      if (dyn)
        t = ring_take(ring_ids, rfull, rempty, (int)it, true);
      else if (it > 0)
        t += nclusters;
      if (t >= g.tiles) break;
      mbar_wait(tempty, acc_ph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        {
          const uint64_t ad = a0 + (uint64_t)(s * STAGE16), bd = b0 + (uint64_t)(s * STAGE16);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tc_mma_2sm(tmem + j * WHALF_N, ad + (uint64_t)(k * ka),
                         bd + (uint64_t)(j * BJ16 + k * kb16), idesc, (kb | k) != 0);
          }
          tc_commit_2sm_mc(&empty[s]);
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      tc_commit_2sm_mc(tfull);
      acc_ph ^= 1;
    }
  } else if (warp >= EPI_WARP0) {
    // ---------------- epilogue: 8 warps, (lane quarter, column half) ----------------
    const int ew = warp - EPI_WARP0;              // 0..7
    const int quarter = warp & 3, half = ew >> 2;
    uint8_t* epi = smem + L::EPI_OFF + ew * 2 * EPI_STAGE_BYTES;
    uint64_t store_pol = 0;
    if (g.store_hint)
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(store_pol));
    // reduce-scatter epilogue (peer.cu): parity buffer of this epoch
    const int par = g.scatter ? (int)((*(volatile const uint32_t*)g.sc_epoch + 1) & 1) : 0;
    int chunk = 0;
    uint32_t acc_ph = 0;
    for (int64_t it = 0, t = cluster;; ++it) {
      if (dyn) {
        t = ring_take(ring_ids, rfull, rempty, (int)it, false);
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&rempty[(int)it % TILE_RING], 0);
      } else if (it > 0) {
        t += nclusters;
      }
      if (t >= g.tiles) break;
      int b, m, n;
      tile_coords(g, t, b, m, n);
      mbar_wait(tfull, acc_ph);
      tc_fence_after();
      const int row0 = m * BM2 + rank * HALF + quarter * 32;
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + half * WHALF_N;
      // software-pipelined drain: chunk c+1's TMEM load is in flight while
      // chunk c is converted and stored
      uint32_t ra[32], rb[32];
      tmem_ld32_nowait(tbase, ra);
      tmem_wait_ld();
#pragma unroll 1
      for (int c0 = 0; c0 < WHALF_N; c0 += 32) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = ra[i];
        if (c0 + 32 < WHALF_N) tmem_ld32_nowait(tbase + c0 + 32, rb);
        const int col = n * WBN + half * WHALF_N + c0;
        if (col >= g.N) {
          // past N: nothing to store (keep the load pipeline in step)
        } else if (g.scatter && g.sc_rows) {
          if (row0 < g.M) {
            const int j = (int)(row0 / g.sc_rchunk);
            epi_store_chunk(&smaps.m[j], epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu, col,
                            (int)(row0 - j * g.sc_rchunk),
                            par * g.sc_par + g.sc_slot_base + b, lane);
          }
        } else if (g.scatter) {
          const int j = (int)(col / g.sc_chunk);
          epi_store_chunk(&smaps.m[j], epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu,
                          (int)(col - j * g.sc_chunk), row0, par * g.sc_par + g.sc_pos, lane);
        } else {
          if (g.resid) add_resid_chunk(g, b, row0, col, lane, r);
          epi_store_chunk(&map_c, epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu, col, row0,
                          b, lane, store_pol);
        }
        if (c0 + 32 < WHALF_N) {
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ra[i] = rb[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(tempty);
      acc_ph ^= 1;
    }
    if (lane == 0) bulk_wait_all();
    // peer stores globally visible before the completion signal (peer.cu)
    if (g.scatter) __threadfence_system();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// host side: operand views -> tensor maps
// ---------------------------------------------------------------------------
struct DimRef {
  int64_t size;
  int64_t st;
};

// Merge a list of (size, stride) dims (outer->inner order) into one dim.
static bool merge_dims(const DimRef* d, int n, DimRef* out) {
  int64_t size = 1, st = 0;
  bool first = true;
  for (int i = n - 1; i >= 0; --i) {
    if (d[i].size == 1) continue;
    if (first) {
      size = d[i].size;
      st = d[i].st;
      first = false;
    } else {
      if (d[i].st != st * size) return false;
      size *= d[i].size;
    }
  }
  out->size = size;
  out->st = first ? 1 : st;
  return true;
}

template <int BN, int STAGES>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                       bf16* out, GemmShape g,
                       cudaStream_t s) {
  typedef Smem<BN, STAGES> L;
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)gemm_bf16_tcgen05<BN, STAGES>, L::TOTAL, &attr_done)) return rc;
  const int sms = sm_budget();
  int64_t grid = g.tiles < sms ? g.tiles : sms;
  gemm_bf16_tcgen05<BN, STAGES><<<(unsigned)grid, 256, L::TOTAL, s>>>(ma, mb, mc, out, g);
  return launched(s);
}

template <int STAGES>
static int launch_gemm_2sm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                           bf16* out, GemmShape g, const ScatterMaps& smaps,
                           cudaStream_t s) {
  typedef Smem2<STAGES> L;
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)gemm_bf16_tcgen05_2sm<STAGES>, L::TOTAL, &attr_done)) return rc;
  const int sms = sm_budget();
  int64_t clusters = g.tiles < sms / 2 || !option(OPT_GEMM_PERSISTENT) ? g.tiles : sms / 2;
  gemm_bf16_tcgen05_2sm<STAGES><<<(unsigned)(2 * clusters), 256, L::TOTAL, s>>>(ma, mb, mc, out,
                                                                                    g, smaps);
  return launched(s);
}

// Per-launch tile counters of the dynamic schedule: a ring of 256 counters
// per device (128 bytes apart), each zeroed on the stream right before its
// launch (a memset node under graph capture), so launches in flight never
// share one.
static int* next_tile_counter(cudaStream_t s) {
  static std::mutex mu;
  static int* bufs[64] = {nullptr};
  static unsigned next[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  int* p;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!bufs[dev] && cudaMalloc(&bufs[dev], 256 * 128) != cudaSuccess) {
      bufs[dev] = nullptr;
      return nullptr;
    }
    p = bufs[dev] + (next[dev]++ % 256) * 32;
  }
  if (cudaMemsetAsync(p, 0, sizeof(int), s) != cudaSuccess) return nullptr;
  return p;
}

template <int STAGES>
static int launch_gemm_2sm_wide(const CUtensorMap& ma, const CUtensorMap& mb,
                                const CUtensorMap& mc, GemmShape g, const ScatterMaps& smaps,
                                cudaStream_t s) {
  typedef SmemW<STAGES> L;
  static_assert(L::TOTAL <= 232448, "wide GEMM smem");
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)gemm_bf16_tcgen05_2sm_wide<STAGES>, L::TOTAL, &attr_done)) return rc;
  const int sms = sm_budget();
  int64_t clusters = g.tiles < sms / 2 || !option(OPT_GEMM_PERSISTENT) ? g.tiles : sms / 2;
  g.tile_counter = nullptr;
  if (option(OPT_GEMM_DYNAMIC) && clusters < g.tiles) {
    g.tile_counter = next_tile_counter(s);
    if (!g.tile_counter) {
      set_error("tile counter allocation failed");
      return SPMD_ERR_CUDA;
    }
  }
  gemm_bf16_tcgen05_2sm_wide<STAGES><<<(unsigned)(2 * clusters), 384, L::TOTAL, s>>>(ma, mb, mc,
                                                                                     g, smaps);
  return launched(s);
}

static int gemm_mode() { return (int)option(OPT_GEMM_MODE); }

// Dot dimension numbers -> one (batch x M x N x K) GEMM over the operands'
// own layouts (no transposes): M / N / K each merge into one strided dim,
// up to 3 batch dims (the partition stack included) become tensor-map dims.
// Shared by the bf16 kernels and the 3xTF32 f32 kernel (gemm_tf32x3.cu).
int gemm_layout(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
                const spmd_dot_dims& dd, int64_t nparts, GemmLayout* L) {
  int64_t ls[SPMD_MAX_RANK], rs[SPMD_MAX_RANK];
  {
    int64_t a = 1;
    for (int k = lhs.rank - 1; k >= 0; --k) ls[k] = a, a *= lhs.dims[k];
    a = 1;
    for (int k = rhs.rank - 1; k >= 0; --k) rs[k] = a, a *= rhs.dims[k];
  }
  bool lu[SPMD_MAX_RANK] = {false}, ru[SPMD_MAX_RANK] = {false};
  DimRef lb[SPMD_MAX_RANK + 1], rb[SPMD_MAX_RANK + 1], lk[SPMD_MAX_RANK], rk[SPMD_MAX_RANK];
  DimRef lm[SPMD_MAX_RANK], rn[SPMD_MAX_RANK];
  int nb = 0, nk = 0, nm = 0, nn = 0;
  int64_t Bsz = 1;
  for (int i = 0; i < dd.n_batch; ++i) {
    int l = dd.lhs_batch[i], r = dd.rhs_batch[i];
    lu[l] = ru[r] = true;
    if (lhs.dims[l] == 1) continue;
    lb[nb] = {lhs.dims[l], ls[l]};
    rb[nb++] = {rhs.dims[r], rs[r]};
    Bsz *= lhs.dims[l];
  }
  for (int i = 0; i < dd.n_contract; ++i) {
    int l = dd.lhs_contracting[i], r = dd.rhs_contracting[i];
    lu[l] = ru[r] = true;
    lk[nk] = {lhs.dims[l], ls[l]};
    rk[nk++] = {rhs.dims[r], rs[r]};
  }
  for (int d = 0; d < lhs.rank; ++d)
    if (!lu[d]) lm[nm++] = {lhs.dims[d], ls[d]};
  for (int d = 0; d < rhs.rank; ++d)
    if (!ru[d]) rn[nn++] = {rhs.dims[d], rs[d]};
  DimRef M, N, K, K2;
  if (!merge_dims(lm, nm, &M) || !merge_dims(rn, nn, &N) || !merge_dims(lk, nk, &K) ||
      !merge_dims(rk, nk, &K2))
    return SPMD_ERR_UNSUPPORTED;
  if (K.size != K2.size || M.size * N.size * Bsz != numel(out)) return SPMD_ERR_UNSUPPORTED;
  // Partition stack as an extra (outermost) batch dim.
  if (nparts > 1) {
    // shift batch dims to make room for the partition dim at the front
    for (int i = nb; i > 0; --i) lb[i] = lb[i - 1], rb[i] = rb[i - 1];
    lb[0] = {nparts, numel(lhs)};
    rb[0] = {nparts, numel(rhs)};
    ++nb;
  }
  if (nb > 3) return SPMD_ERR_UNSUPPORTED;
  const int a_mn = M.st == 1 && K.st != 1;
  const int b_mn = N.st == 1 && K2.st != 1 ? 1 : 0;
  if (!a_mn && K.st != 1) return SPMD_ERR_UNSUPPORTED;
  const int b_k = K2.st == 1;
  if (!b_mn && !b_k) return SPMD_ERR_UNSUPPORTED;

  L->nbatch = nb;
  L->M = (int)M.size;
  L->N = (int)N.size;
  L->K = (int)K.size;
  L->a_mn = a_mn;
  L->b_mn = b_mn;
  // tensor-map batch dims: innermost first
  OperandView& va = L->va;
  OperandView& vb = L->vb;
  for (int i = 0; i < 3; ++i) {
    int src = nb - 1 - i;   // innermost batch dim first
    va.size[2 + i] = src >= 0 ? lb[src].size : 1;
    va.stride[2 + i] = src >= 0 ? lb[src].st : 1;
    vb.size[2 + i] = src >= 0 ? rb[src].size : 1;
    vb.stride[2 + i] = src >= 0 ? rb[src].st : 1;
    L->nb[i] = (int)(src >= 0 ? lb[src].size : 1);
  }
  // give unit dims a harmless stride (tensor maps need 16B multiples)
  for (int i = 2; i < 5; ++i) {
    if (va.size[i] == 1) va.stride[i] = va.stride[i - 1] ? 8 : 8;
    if (vb.size[i] == 1) vb.stride[i] = 8;
  }
  if (!a_mn) {
    va.size[0] = K.size, va.stride[0] = 1, va.size[1] = M.size, va.stride[1] = M.st;
  } else {
    va.size[0] = M.size, va.stride[0] = 1, va.size[1] = K.size, va.stride[1] = K.st;
  }
  if (!b_mn) {
    vb.size[0] = K2.size, vb.stride[0] = 1, vb.size[1] = N.size, vb.stride[1] = N.st;
  } else {
    vb.size[0] = N.size, vb.stride[0] = 1, vb.size[1] = K2.size, vb.stride[1] = K2.st;
  }
  return SPMD_OK;
}

int dot_tcgen05(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
                const spmd_dot_dims& dd, int64_t nparts, cudaStream_t s, const GemmScatter* sc,
                const void* resid) {
  if (lhs.dtype != SPMD_BF16) return SPMD_ERR_UNSUPPORTED;
  GemmLayout lay;
  if (int rc = gemm_layout(lhs, rhs, out, dd, nparts, &lay)) return rc;
  if (lay.M < 64 || lay.N < 64 || lay.K < 16) return SPMD_ERR_UNSUPPORTED;
  const int a_mn = lay.a_mn, b_mn = lay.b_mn;
  const OperandView& va = lay.va;
  const OperandView& vb = lay.vb;
  GemmShape g;
  memset(&g, 0, sizeof(g));
  g.M = lay.M;
  g.N = lay.N;
  g.K = lay.K;
  g.a_mn = a_mn;
  g.b_mn = b_mn;
  g.relu = dd.epilogue == 1;
  g.resid = (const bf16*)resid;
  if (resid && (sc || g.relu || (reinterpret_cast<uintptr_t>(resid) & 15))) return SPMD_ERR_UNSUPPORTED;
  const int group_opt = (int)option(OPT_GEMM_GROUP);   // 0: per-kernel default
  g.group = group_opt > 0 ? group_opt : 8;
  g.raster_n = (int)option(OPT_GEMM_RASTER_N);
  g.hint = (int)option(OPT_GEMM_HINT);
  g.store_hint = (int)option(OPT_GEMM_STORE_HINT);
  for (int i = 0; i < 3; ++i) g.nb[i] = lay.nb[i];
  g.out_batch_stride = (int64_t)g.M * g.N;
  CUtensorMap ma, mb, mc;
  ScatterMaps smaps;
  memset(&smaps, 0, sizeof(smaps));
  // Bulk-tensor store epilogue whenever the output rows are 16-byte aligned.
  {
    const int64_t nbat = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];
    const int direct = (int)option(OPT_GEMM_EPI_DIRECT);
    g.tma_store = !direct && (g.N % 8 == 0) &&
                  encode_store_map(&mc, out.data, g.N, g.M, g.N, nbat, g.out_batch_stride);
    if (!g.tma_store) memset(&mc, 0, sizeof(mc));
  }
  if (sc && sc->rows) {
    // All-to-all epilogue (wide kernel): one batch dim (the concat dim), the
    // split dim = the leading GEMM row dim, whole row chunks per member.
    const int64_t nbat = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];
    // rchunk 0: reduce-scatter on the leading row dim -> M / gsize rows each
    const int64_t rchunk = sc->rchunk ? sc->rchunk : (int64_t)g.M / (sc->gsize ? sc->gsize : 1);
    if ((int64_t)g.M < 256 || (int64_t)g.N < 512 || gemm_mode() != 3 ||
        sc->gsize < 1 || sc->gsize > 8 || rchunk % 32 != 0 ||
        rchunk * sc->gsize != (int64_t)g.M || nbat * sc->gsize != sc->nslots)
      return SPMD_ERR_UNSUPPORTED;
    g.tma_store = 0;
    g.scatter = 1;
    g.sc_rows = 1;
    g.sc_g = sc->gsize;
    g.sc_pos = sc->pos;
    g.sc_rchunk = rchunk;
    g.sc_slot_base = sc->slot_base;
    g.sc_nslots = sc->nslots;
    g.sc_par = sc->par_slots;
    g.sc_epoch = sc->epoch;
    g.sc_tma = sc->par_slots >= sc->nslots;
    for (int j = 0; g.sc_tma && j < sc->gsize; ++j)
      g.sc_tma = encode_store_map(&smaps.m[j], sc->dst[j], (int64_t)g.N, rchunk, (int64_t)g.N,
                                  sc->par_slots + sc->nslots, rchunk * (int64_t)g.N);
    if (!g.sc_tma) return SPMD_ERR_UNSUPPORTED;
  } else if (sc) {
    // Reduce-scatter epilogue: 2-CTA kernel, no batch dims, the scattered
    // dim is the last output dim == the whole GEMM N.
    if ((int64_t)g.M < 256 || (int64_t)g.N < 256 || lay.nbatch != 0 || (int64_t)g.N != out.dims[out.rank - 1] ||
        sc->gsize < 1 || sc->gsize > 8 || (int64_t)g.N % sc->gsize != 0 ||
        ((int64_t)g.N / sc->gsize) % 32 != 0)
      return SPMD_ERR_UNSUPPORTED;
    g.tma_store = 0;
    g.scatter = 1;
    g.sc_g = sc->gsize;
    g.sc_pos = sc->pos;
    g.sc_chunk = (int64_t)g.N / sc->gsize;
    g.sc_slot = (int64_t)g.M * g.sc_chunk;
    if (sc->par_slots < sc->gsize) return SPMD_ERR_UNSUPPORTED;
    g.sc_par = sc->par_slots;
    for (int j = 0; j < sc->gsize; ++j) g.sc_dst[j] = (bf16*)sc->dst[j];
    g.sc_epoch = sc->epoch;
    g.sc_tma = !option(OPT_SCATTER_EPI_DIRECT);
    for (int j = 0; g.sc_tma && j < sc->gsize; ++j)
      g.sc_tma = encode_store_map(&smaps.m[j], sc->dst[j], g.sc_chunk, (int64_t)g.M, g.sc_chunk,
                                  sc->par_slots + sc->gsize, g.sc_slot);
  }
  if (gemm_mode() == 3 && (sc ? g.sc_tma : g.tma_store) && (int64_t)g.M >= 256 && (int64_t)g.N >= 512) {
    // wide pair tiles (256 x 512); the store epilogue is TMA-only
    bool okw = a_mn ? encode(&ma, lhs.data, va, 64, BK) : encode(&ma, lhs.data, va, BK, HALF);
    okw = okw && (b_mn ? encode(&mb, rhs.data, vb, 64, BK) : encode(&mb, rhs.data, vb, BK, HALF));
    if (okw) {
      // Raster groups of 8 M-tiles under the dynamic tile order (ncu on
      // FFN-in, profiles/r2_gemm_dyn_raster_ncu.csv: DRAM reads 12.5 GB vs
      // 14.6 at 16 and 19.4 at 4, SM clock 1.43 vs 1.41 / 1.41 GHz under the
      // power cap).  The round-1 static order preferred 16.
      if (group_opt <= 0) g.group = option(OPT_GEMM_DYNAMIC) ? 8 : 16;
      g.mt = (g.M + BM2 - 1) / BM2;
      g.nt = (g.N + WBN - 1) / WBN;
      g.tiles = (int64_t)g.mt * g.nt * g.nb[0] * g.nb[1] * g.nb[2];
      return launch_gemm_2sm_wide<4>(ma, mb, mc, g, smaps, s);
    }
  }
  if (g.resid) return SPMD_ERR_UNSUPPORTED;   // residual epilogue: wide kernel only
  if ((gemm_mode() >= 2 || sc) && (int64_t)g.M >= 256 && (int64_t)g.N >= 256) {
    // 2-CTA path: per-CTA boxes are 128 rows of A and 128 rows of B.
    bool ok2 = a_mn ? encode(&ma, lhs.data, va, 64, BK) : encode(&ma, lhs.data, va, BK, HALF);
    ok2 = ok2 && (b_mn ? encode(&mb, rhs.data, vb, 64, BK) : encode(&mb, rhs.data, vb, BK, HALF));
    if (!ok2) return SPMD_ERR_UNSUPPORTED;
    g.mt = (g.M + BM2 - 1) / BM2;
    g.nt = (g.N + BN2 - 1) / BN2;
    g.tiles = (int64_t)g.mt * g.nt * g.nb[0] * g.nb[1] * g.nb[2];
    return launch_gemm_2sm<6>(ma, mb, mc, (bf16*)out.data, g, smaps, s);
  }
  const int BNsel = (int64_t)g.N >= 256 ? 256 : 128;
  bool ok = a_mn ? encode(&ma, lhs.data, va, 64, BK) : encode(&ma, lhs.data, va, BK, BM);
  ok = ok && (b_mn ? encode(&mb, rhs.data, vb, 64, BK) : encode(&mb, rhs.data, vb, BK, BNsel));
  if (!ok) return SPMD_ERR_UNSUPPORTED;
  g.mt = (g.M + BM - 1) / BM;
  g.nt = (g.N + BNsel - 1) / BNsel;
  g.tiles = (int64_t)g.mt * g.nt * g.nb[0] * g.nb[1] * g.nb[2];
  g.out_batch_stride = (int64_t)g.M * g.N;
  if (BNsel == 256) return launch_gemm<256, 4>(ma, mb, mc, (bf16*)out.data, g, s);
  return launch_gemm<128, 6>(ma, mb, mc, (bf16*)out.data, g, s);
}

}  // namespace spmd

// Direct entry point for benchmarking the GEMM alone: C[M,N] = A[M,K] . B[K,N]
// (row-major, A K-major, B MN-major), all bf16.
extern "C" int spmd_gemm_bf16(const void* a, const void* b, void* c, int64_t M, int64_t N,
                              int64_t K, int relu, void* stream) {
  spmd_tensor ta, tb, tc;
  memset(&ta, 0, sizeof(ta));
  memset(&tb, 0, sizeof(tb));
  memset(&tc, 0, sizeof(tc));
  ta.data = const_cast<void*>(a), ta.dtype = SPMD_BF16, ta.rank = 2, ta.dims[0] = M, ta.dims[1] = K;
  tb.data = const_cast<void*>(b), tb.dtype = SPMD_BF16, tb.rank = 2, tb.dims[0] = K, tb.dims[1] = N;
  tc.data = c, tc.dtype = SPMD_BF16, tc.rank = 2, tc.dims[0] = M, tc.dims[1] = N;
  spmd_dot_dims dd;
  memset(&dd, 0, sizeof(dd));
  dd.n_contract = 1;
  dd.lhs_contracting[0] = 1;
  dd.rhs_contracting[0] = 0;
  dd.epilogue = relu;
  return spmd::dot_tcgen05(ta, tb, tc, dd, 1, spmd::as_stream(stream));
}
