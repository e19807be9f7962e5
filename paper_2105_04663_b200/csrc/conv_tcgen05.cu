// Implicit-GEMM convolution on tcgen05 for NHWC bf16 (config C4), replacing
// the reference's per-output-position tensordot (simulator.py:121-154).
//
// GEMM view: M = output pixels (tiles of 128 consecutive wo in one (n, ho)
// row), N = Cout, K = (kh, kw, cin) in blocks of 64 channels.  For K-block
// (kh, kw, c0) the A tile is the input box {64 ch x 128 px} at
// (c0, wo0 + kw - pad_w, ho + kh - pad_h, n): TMA's out-of-bounds zero fill
// IS the convolution padding (and the masked halo rows of a spatially
// partitioned input are already explicit), so no im2col buffer and no
// boundary code.  B = HWIO weights, MN-major (Cout contiguous).  Same
// warp-specialised pipeline as the 1-CTA GEMM: TMA producer, single-thread
// MMA issuer, double-buffered TMEM accumulators, 4 epilogue warps (fused ReLU).
// Supported: 2 spatial dims, stride 1, no dilation, Cin % 64 == 0,
// Cout % 64 == 0; anything else returns SPMD_ERR_UNSUPPORTED (direct kernel).
#include "tcgen05.cuh"

#include <string.h>

namespace spmd {

constexpr int CBM = 128, CBK = 64;

struct ConvShape {
  int N, Ho, Wo, Cin, Cout, KH, KW, pad_h, pad_w;
  int nwb, nt, cin_blocks, kblocks;
  int64_t tiles;
  int relu;
  int tma_store;
  // Halo-window input (spmd_halo_convolution): the conv input rows are the
  // window DS(mask(concat(pieces)), start) along H, read straight from the
  // pieces (map_x, map_x1, map_x2); masked rows load out of bounds = zeros.
  int win, npieces, has_mask, has_low;
  int len[3];                  // piece extents along H
  int buf_len, win_rows, nparts;
  const int32_t* start;        // per-partition window start (clamped)
  const int32_t* offset;       // per-partition global row of buffer row 0
  int64_t low, high;
};

// Window row h (start s0, global offset off) -> (piece, row in piece);
// row -1 = masked / outside the window.
__device__ __forceinline__ int window_row(const ConvShape& g, int s0, int off, int h,
                                          int& piece) {
  piece = 0;
  if (h < 0 || h >= g.win_rows) return -1;
  int r = s0 + h;
  if (g.has_mask) {
    const int64_t gl = (int64_t)r + off;
    if (!(gl < g.high && (!g.has_low || gl >= g.low))) return -1;
  }
  while (piece < g.npieces - 1 && r >= g.len[piece]) {
    r -= g.len[piece];
    ++piece;
  }
  return r;
}

template <int BN, int STAGES>
struct ConvSmem {
  static constexpr int A_BYTES = CBM * CBK * 2;
  static constexpr int B_BYTES = BN * CBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 1024;
  static constexpr int TOTAL = EPI_OFF + 8 * EPI_STAGE_BYTES + 1024;
};

__device__ __forceinline__ void conv_tile(const ConvShape& g, int64_t t64, int& pn, int& ho, int& wb,
                                          int& ct) {
  // 32-bit index math (the host keeps tiles < 2^31): 64-bit division by a
  // runtime value is a long call sequence per tile on the producer and
  // epilogue paths (C4 layer at N=4 shapes: 0.447 -> 0.430 ms,
  // scripts/halo_part_bench.py)
  uint32_t t = (uint32_t)t64;
  ct = (int)(t % (uint32_t)g.nt);
  t /= (uint32_t)g.nt;
  wb = (int)(t % (uint32_t)g.nwb);
  t /= (uint32_t)g.nwb;
  ho = (int)(t % (uint32_t)g.Ho);
  pn = (int)(t / (uint32_t)g.Ho);
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    conv_bf16_tcgen05(const __grid_constant__ CUtensorMap map_x,
                      const __grid_constant__ CUtensorMap map_w,
                      const __grid_constant__ CUtensorMap map_o, bf16* __restrict__ out,
                      ConvShape g, const __grid_constant__ CUtensorMap map_x1,
                      const __grid_constant__ CUtensorMap map_x2) {
  typedef ConvSmem<BN, STAGES> L;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // halo-window input: per-partition clamped start / offset, read once
  __shared__ int win_s0[SPMD_MAX_PARTS], win_off[SPMD_MAX_PARTS];
  if (g.win) {
    for (int p = threadIdx.x; p < g.nparts && p < SPMD_MAX_PARTS; p += blockDim.x) {
      int s0 = g.start[p];
      win_s0[p] = s0 < 0 ? 0 : (s0 > g.buf_len - g.win_rows ? g.buf_len - g.win_rows : s0);
      win_off[p] = g.has_mask ? g.offset[p] : 0;
    }
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
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

  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      int pn, ho, wb, ct;
      conv_tile(g, t, pn, ho, wb, ct);
      const int n = pn % g.N, p = pn / g.N;
      int row_kh = -1, row_r = 0, row_piece = 0;   // window row of the current kh
      for (int kb = 0; kb < g.kblocks; ++kb) {
        const int tap = kb / g.cin_blocks, cb = kb - tap * g.cin_blocks;
        const int kh = tap / g.KW, kw = tap - kh * g.KW;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        uint8_t* sb = sa + L::A_BYTES;
        mbar_expect_tx(&full[s], L::STAGE_BYTES);
        if (!g.win) {
          tma_load_5d(sa, &map_x, &full[s], cb * CBK, wb * CBM + kw - g.pad_w, ho + kh - g.pad_h,
                      n, p);
        } else {
          if (kh != row_kh) {
            row_kh = kh;
            row_r = window_row(g, win_s0[p], win_off[p], ho + kh - g.pad_h, row_piece);
          }
          const CUtensorMap* mp = row_piece == 0 ? &map_x : (row_piece == 1 ? &map_x1 : &map_x2);
          tma_load_5d(sa, mp, &full[s], cb * CBK, wb * CBM + kw - g.pad_w, row_r, n, p);
        }
#pragma unroll
        for (int c = 0; c < BN / 64; ++c)
          tma_load_5d(sb + c * (CBK * 128), &map_w, &full[s], ct * BN + c * 64, cb * CBK, kw, kh,
                      p);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = make_idesc(CBM, BN, 0, 1);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * BN;
      for (int kb = 0; kb < g.kblocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
        const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < CBK / 16; ++k)
          tc_mma(d_tmem, make_desc(sa + k * 32, 16, 1024), make_desc(sb + k * 2048, CBK * 128, 1024),
                 idesc, (kb | k) != 0);
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
  } else if (warp >= 4) {
    const int ew = warp - 4;
    uint8_t* epi = smem + L::EPI_OFF + ew * 2 * EPI_STAGE_BYTES;
    int chunk = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      int pn, ho, wb, ct;
      conv_tile(g, t, pn, ho, wb, ct);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int wo = wb * CBM + ew * 32 + lane;
      bf16* orow = out + (((int64_t)pn * g.Ho + ho) * g.Wo + wo) * g.Cout;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + acc * BN + c0, r);
        const int col = ct * BN + c0;
        if (g.tma_store) {
          epi_store_chunk(&map_o, epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu, col,
                          wb * CBM + ew * 32, pn * g.Ho + ho, lane);
        } else if (wo < g.Wo && col < g.Cout) {
          __align__(16) bf16 v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float f = __uint_as_float(r[j]);
            if (g.relu) f = f > 0.f ? f : 0.f;
            v[j] = __float2bfloat16_rn(f);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(orow + col + 8 * j) = reinterpret_cast<uint4*>(v)[j];
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
// CTA-pair variant for Cout = 128 (cta_group::2, UMMA 256 x 128): the pair
// owns 256 consecutive output pixels of one (n, ho) row; each CTA stages its
// 128 pixels of the input box and 64 of the 128 output channels of the
// weights, so per-SM operand smem traffic per MMA drops by a third versus
// the 1-CTA 128 x 128 tile (which is smem-bandwidth bound at Cout = 128).
// ---------------------------------------------------------------------------
constexpr int CHALF = 64;   // Cout per CTA

// WRES: this CTA's half of the weights (kblocks x 8 KB) stays resident in
// smem for the whole kernel (loaded once); only input boxes stream.
// TAPS > 0 (resident weights only): one input box of 128 + TAPS - 1 pixels per
// (kh, cin block) feeds all TAPS horizontal taps through UMMA descriptors
// whose start is shifted by whole 128-byte rows -- 3x fewer input bytes.
template <int STAGES, int WRES, int TAPS = 0>
struct Conv2Smem {
  static constexpr int A_ROWS = TAPS ? CBM + TAPS - 1 : CBM;
  static constexpr int A_TX = A_ROWS * CBK * 2;                  // bytes per box
  static constexpr int A_BYTES = (A_TX + 1023) / 1024 * 1024;     // 1 KB aligned stages
  static constexpr int B_BYTES = CHALF * CBK * 2;     // 64 cout x 64 ch
  static constexpr int STAGE_BYTES = A_BYTES + (WRES ? 0 : B_BYTES);
  static constexpr int W_OFF = STAGES * STAGE_BYTES;  // resident weights (WRES kblocks)
  static constexpr int BAR_OFF = W_OFF + WRES * B_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 1024;
  static constexpr int TOTAL = EPI_OFF + 8 * EPI_STAGE_BYTES + 1024;
};

template <int STAGES, int WRES, int TAPS = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    conv_bf16_tcgen05_2sm(const __grid_constant__ CUtensorMap map_x,
                          const __grid_constant__ CUtensorMap map_w,
                          const __grid_constant__ CUtensorMap map_o, ConvShape g,
                          const __grid_constant__ CUtensorMap map_x1,
                          const __grid_constant__ CUtensorMap map_x2) {
  typedef Conv2Smem<STAGES, WRES, TAPS> L;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* wfull = tempty + 2;
  uint32_t* tmem_slot = (uint32_t*)(wfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  __shared__ int win_s0[SPMD_MAX_PARTS], win_off[SPMD_MAX_PARTS];
  if (g.win) {
    for (int p = threadIdx.x; p < g.nparts && p < SPMD_MAX_PARTS; p += blockDim.x) {
      int s0 = g.start[p];
      win_s0[p] = s0 < 0 ? 0 : (s0 > g.buf_len - g.win_rows ? g.buf_len - g.win_rows : s0);
      win_off[p] = g.has_mask ? g.offset[p] : 0;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);   // 4 epilogue warps x 2 CTAs
    }
    mbar_init(wfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    if (WRES) {
      // whole weight half once (single output-channel tile, one partition
      // of weights: both guaranteed by the host)
      if (leader) mbar_expect_tx(wfull, 2 * WRES * L::B_BYTES);
      for (int kb = 0; kb < WRES; ++kb) {
        const int tap = kb / g.cin_blocks, cb = kb - tap * g.cin_blocks;
        const int kh = tap / g.KW, kw = tap - kh * g.KW;
        tma_load_5d_2sm(smem + L::W_OFF + kb * L::B_BYTES, &map_w, wfull, rank * CHALF, cb * CBK,
                        kw, kh, 0);
      }
    }
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int pn, ho, wb, ct;
      conv_tile(g, t, pn, ho, wb, ct);
      const int n = pn % g.N, p = pn / g.N;
      const int w0 = wb * 2 * CBM + rank * CBM;
      int row_kh = -1, row_r = 0, row_piece = 0;
      const int nstage = TAPS ? g.KH * g.cin_blocks : g.kblocks;
      for (int kb = 0; kb < nstage; ++kb) {
        // TAPS: stage = (kh, cb), the box covers every kw; else stage = tap
        const int tap = TAPS ? (kb / g.cin_blocks) * g.KW : kb / g.cin_blocks;
        const int cb = kb % g.cin_blocks;
        const int kh = tap / g.KW, kw = TAPS ? 0 : tap - kh * g.KW;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        uint8_t* sb = sa + L::A_BYTES;
        if (leader) mbar_expect_tx(&full[s], 2 * (L::A_TX + (WRES ? 0 : L::B_BYTES)));
        (void)sb;
        if (!g.win) {
          tma_load_5d_2sm(sa, &map_x, &full[s], cb * CBK, w0 + kw - g.pad_w, ho + kh - g.pad_h,
                          n, p);
        } else {
          if (kh != row_kh) {
            row_kh = kh;
            row_r = window_row(g, win_s0[p], win_off[p], ho + kh - g.pad_h, row_piece);
          }
          const CUtensorMap* mp = row_piece == 0 ? &map_x : (row_piece == 1 ? &map_x1 : &map_x2);
          tma_load_5d_2sm(sa, mp, &full[s], cb * CBK, w0 + kw - g.pad_w, row_r, n, p);
        }
        if (!WRES)
          tma_load_5d_2sm(sb, &map_w, &full[s], ct * 2 * CHALF + rank * CHALF, cb * CBK, kw, kh,
                          p);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && leader) {
    // The whole warp runs the loop (uniform control flow: descriptors and
    // counters in uniform registers), one elected lane issues.  A conv MMA
    // (UMMA 256 x 128 x 16) is only 64 tensor cycles, so the per-MMA issue
    // cost is on the critical path (ncu: tensor pipe 62% active): the
    // descriptors are precomputed and advanced by constant offsets.
    const uint32_t idesc = make_idesc(2 * CBM, 2 * CHALF, 0, 1);
    const uint64_t a0 = make_desc(smem_u32(smem), 16, 1024);
    const uint64_t w0d = make_desc(smem_u32(smem + L::W_OFF), CBK * 128, 1024);
    constexpr uint32_t STAGE16 = L::STAGE_BYTES >> 4, B16 = L::B_BYTES >> 4, A16 = L::A_BYTES >> 4;
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    if (WRES) {
      mbar_wait(wfull, 0);
      tc_fence_after();
    }
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * 2 * CHALF;
      const int nstage = TAPS ? g.KH * g.cin_blocks : g.kblocks;
      int kh = 0, cb = 0;
      for (int kb = 0; kb < nstage; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = a0 + (uint64_t)(s * STAGE16);
          if (TAPS) {
#pragma unroll
            for (int kw = 0; kw < TAPS; ++kw) {
              const uint64_t bd = w0d + (uint64_t)(((kh * g.KW + kw) * g.cin_blocks + cb) * B16);
#pragma unroll
              for (int k = 0; k < CBK / 16; ++k)
                tc_mma_2sm(d_tmem, ad + (uint64_t)((kw * 128 + k * 32) >> 4),
                           bd + (uint64_t)((k * 2048) >> 4), idesc, (kb | kw | k) != 0);
            }
          } else {
            const uint64_t bd = WRES ? w0d + (uint64_t)(kb * B16)
                                     : make_desc(smem_u32(smem + s * L::STAGE_BYTES) + A16 * 16,
                                                 CBK * 128, 1024);
#pragma unroll
            for (int k = 0; k < CBK / 16; ++k)
              tc_mma_2sm(d_tmem, ad + (uint64_t)((k * 32) >> 4),
                         bd + (uint64_t)((k * 2048) >> 4), idesc, (kb | k) != 0);
          }
          tc_commit_2sm_mc(&empty[s]);
        }
        __syncwarp();
        if (++cb == g.cin_blocks) {
          cb = 0;
          ++kh;
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) tc_commit_2sm_mc(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    uint8_t* epi = smem + L::EPI_OFF + ew * 2 * EPI_STAGE_BYTES;
    int chunk = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int pn, ho, wb, ct;
      conv_tile(g, t, pn, ho, wb, ct);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < 2 * CHALF; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + acc * 2 * CHALF + c0, r);
        epi_store_chunk(&map_o, epi + (chunk++ & 1) * EPI_STAGE_BYTES, r, g.relu,
                        ct * 2 * CHALF + c0, wb * 2 * CBM + rank * CBM + ew * 32,
                        pn * g.Ho + ho, lane);
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
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int STAGES, int WRES, int TAPS = 0>
static int launch_conv_2sm(const CUtensorMap& mx, const CUtensorMap& mw, const CUtensorMap& mo,
                           ConvShape g, const CUtensorMap& mx1, const CUtensorMap& mx2,
                           cudaStream_t s) {
  typedef Conv2Smem<STAGES, WRES, TAPS> L;
  static_assert(L::TOTAL <= 232448, "conv 2-CTA smem");
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)conv_bf16_tcgen05_2sm<STAGES, WRES, TAPS>, L::TOTAL, &attr_done)) return rc;
  const int sms = sm_budget();
  const int64_t clusters = g.tiles < sms / 2 ? g.tiles : sms / 2;
  conv_bf16_tcgen05_2sm<STAGES, WRES, TAPS><<<(unsigned)(2 * clusters), 256, L::TOTAL, s>>>(
      mx, mw, mo, g, mx1, mx2);
  return launched(s);
}

static int conv_mode() { return option(OPT_CONV_MODE) == 1 ? 1 : 2; }

template <int BN, int STAGES>
static int launch_conv(const CUtensorMap& mx, const CUtensorMap& mw, const CUtensorMap& mo,
                       bf16* out, ConvShape g, const CUtensorMap& mx1, const CUtensorMap& mx2,
                       cudaStream_t s) {
  typedef ConvSmem<BN, STAGES> L;
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)conv_bf16_tcgen05<BN, STAGES>, L::TOTAL, &attr_done)) return rc;
  const int sms = sm_budget();
  int64_t grid = g.tiles < sms ? g.tiles : sms;
  conv_bf16_tcgen05<BN, STAGES><<<(unsigned)grid, 256, L::TOTAL, s>>>(mx, mw, mo, out, g, mx1,
                                                                       mx2);
  return launched(s);
}

struct ConvWindow {
  const spmd_tensor* pieces;
  int npieces, has_mask, has_low;
  const int32_t* start;
  const int32_t* offset;
  int64_t low, high;
};

int conv_tcgen05(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
                 const spmd_conv_dims& cd, int64_t nparts, cudaStream_t s,
                 const ConvWindow* win = nullptr) {
  if (lhs.dtype != SPMD_BF16 || cd.n_spatial != 2 || lhs.rank != 4) return SPMD_ERR_UNSUPPORTED;
  // NHWC / HWIO / NHWC only.
  if (!(cd.lhs_batch == 0 && cd.lhs_spatial[0] == 1 && cd.lhs_spatial[1] == 2 &&
        cd.lhs_feature == 3 && cd.rhs_spatial[0] == 0 && cd.rhs_spatial[1] == 1 &&
        cd.rhs_in_feature == 2 && cd.rhs_out_feature == 3 && cd.out_batch == 0 &&
        cd.out_spatial[0] == 1 && cd.out_spatial[1] == 2 && cd.out_feature == 3))
    return SPMD_ERR_UNSUPPORTED;
  for (int i = 0; i < 2; ++i)
    if (cd.stride[i] != 1 || cd.base_dilation[i] != 1 || cd.window_dilation[i] != 1)
      return SPMD_ERR_UNSUPPORTED;
  ConvShape g;
  memset(&g, 0, sizeof(g));
  g.N = (int)lhs.dims[0];
  const int H = (int)lhs.dims[1], W = (int)lhs.dims[2];
  g.Cin = (int)lhs.dims[3];
  g.KH = (int)rhs.dims[0];
  g.KW = (int)rhs.dims[1];
  g.Cout = (int)rhs.dims[3];
  g.Ho = (int)out.dims[1];
  g.Wo = (int)out.dims[2];
  g.pad_h = cd.pad_low[0];
  g.pad_w = cd.pad_low[1];
  if (g.Cin % 64 || g.Cout % 64 || g.Wo < 64) return SPMD_ERR_UNSUPPORTED;
  const int BN = g.Cout % 256 == 0 ? 256 : 128;
  if (g.Cout % BN) return SPMD_ERR_UNSUPPORTED;
  OperandView vx, vw;
  vx.size[0] = g.Cin, vx.stride[0] = 1;
  vx.size[1] = W, vx.stride[1] = g.Cin;
  vx.size[2] = H, vx.stride[2] = (int64_t)W * g.Cin;
  vx.size[3] = g.N, vx.stride[3] = (int64_t)H * W * g.Cin;
  vx.size[4] = nparts, vx.stride[4] = numel(lhs);
  vw.size[0] = g.Cout, vw.stride[0] = 1;
  vw.size[1] = g.Cin, vw.stride[1] = g.Cout;
  vw.size[2] = g.KW, vw.stride[2] = (int64_t)g.Cin * g.Cout;
  vw.size[3] = g.KH, vw.stride[3] = (int64_t)g.KW * g.Cin * g.Cout;
  vw.size[4] = nparts, vw.stride[4] = numel(rhs);
  if (nparts == 1) vx.stride[4] = vw.stride[4] = 8;
  CUtensorMap mx, mw, mx1, mx2;
  memset(&mx1, 0, sizeof(mx1));
  memset(&mx2, 0, sizeof(mx2));
  if (!encode(&mw, rhs.data, vw, 64, CBK)) return SPMD_ERR_UNSUPPORTED;
  // input map(s) with `rows`-pixel boxes (CBM, or CBM + KW - 1 for tap reuse)
  auto encode_inputs = [&](int rows) -> bool {
    if (!win) return encode(&mx, lhs.data, vx, CBK, rows);
    CUtensorMap* maps[3] = {&mx, &mx1, &mx2};
    for (int k = 0; k < win->npieces; ++k) {
      const spmd_tensor& pc = win->pieces[k];
      OperandView vp = vx;
      vp.size[2] = pc.dims[1];
      vp.stride[3] = pc.dims[1] * W * g.Cin;
      vp.stride[4] = nparts == 1 ? 8 : numel(pc);
      if (!encode(maps[k], pc.data, vp, CBK, rows)) return false;
    }
    return true;
  };
  if (win) {
    // one map per piece: [nparts][N][len_k][W][Cin]
    g.win = 1;
    g.npieces = win->npieces;
    g.has_mask = win->has_mask;
    g.has_low = win->has_low;
    g.start = win->start;
    g.offset = win->offset;
    g.low = win->low;
    g.high = win->high;
    g.win_rows = H;
    g.nparts = (int)nparts;
    if (nparts > SPMD_MAX_PARTS) return SPMD_ERR_UNSUPPORTED;
    for (int k = 0; k < win->npieces; ++k) {
      const spmd_tensor& pc = win->pieces[k];
      if (pc.dtype != SPMD_BF16 || pc.rank != 4 || pc.dims[0] != g.N || pc.dims[2] != W ||
          pc.dims[3] != g.Cin)
        return SPMD_ERR_UNSUPPORTED;
      g.len[k] = (int)pc.dims[1];
      g.buf_len += g.len[k];
    }
    if (g.buf_len < H) return SPMD_ERR_UNSUPPORTED;
  }
  if (!encode_inputs(CBM)) return SPMD_ERR_UNSUPPORTED;
  g.nwb = (g.Wo + CBM - 1) / CBM;
  g.nt = g.Cout / BN;
  g.cin_blocks = g.Cin / CBK;
  g.kblocks = g.KH * g.KW * g.cin_blocks;
  g.tiles = (int64_t)nparts * g.N * g.Ho * g.nwb * g.nt;
  if (g.tiles >= ((int64_t)1 << 31)) return SPMD_ERR_UNSUPPORTED;   // conv_tile's 32-bit math
  g.relu = cd.epilogue == 1;
  CUtensorMap mo;
  g.tma_store = encode_store_map(&mo, out.data, g.Cout, g.Wo, g.Cout, nparts * g.N * g.Ho,
                                 (int64_t)g.Wo * g.Cout);
  if (!g.tma_store) memset(&mo, 0, sizeof(mo));
  if (BN == 128 && g.tma_store && conv_mode() == 2 && g.Wo >= 2 * CBM) {
    // CTA pairs: tiles of 256 pixels, weights boxed 64 output channels per CTA
    CUtensorMap mw2;
    if (encode(&mw2, rhs.data, vw, CHALF, CBK)) {
      g.nwb = (g.Wo + 2 * CBM - 1) / (2 * CBM);
      g.tiles = (int64_t)nparts * g.N * g.Ho * g.nwb * g.nt;
      // 3x3 x 128 input channels: weights resident in smem (one weight set)
      const int64_t wres = option(OPT_CONV_WRES), taps = option(OPT_CONV_TAPS);
      if (wres && taps && g.kblocks == 18 && g.KW == 3 && g.nt == 1 && nparts == 1) {
        if (encode_inputs(CBM + 2)) return launch_conv_2sm<3, 18, 3>(mx, mw2, mo, g, mx1, mx2, s);
        // restore the 128-pixel boxes the other kernels expect
        if (!encode_inputs(CBM)) return SPMD_ERR_UNSUPPORTED;
      }
      if (wres && g.kblocks == 18 && g.nt == 1 && nparts == 1)
        return launch_conv_2sm<4, 18>(mx, mw2, mo, g, mx1, mx2, s);
      return launch_conv_2sm<7, 0>(mx, mw2, mo, g, mx1, mx2, s);
    }
  }
  if (BN == 256) return launch_conv<256, 4>(mx, mw, mo, (bf16*)out.data, g, mx1, mx2, s);
  return launch_conv<128, 6>(mx, mw, mo, (bf16*)out.data, g, mx1, mx2, s);
}

}  // namespace spmd

using namespace spmd;

// Convolution whose input is a halo window along H: window =
// DS(mask(concat(pieces)), start) (reference formatting.py:109-182 feeding
// handle_convolution :494-540), read by the conv's TMA loads straight from
// the pieces -- no window buffer in HBM.  `window` carries the window shape
// (its data is not read).  Masked rows read as zeros, so the caller's mask
// fill must be 0.  SPMD_ERR_UNSUPPORTED when the conv does not qualify.
extern "C" int spmd_halo_convolution(const spmd_tensor* pieces, int npieces, int axis,
                                     spmd_tensor start, int has_mask, spmd_tensor offset,
                                     int64_t low, int64_t high, int has_low, spmd_tensor window,
                                     spmd_tensor rhs, spmd_tensor out, const spmd_conv_dims* cd,
                                     int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(npieces >= 1 && npieces <= 3 && cd, "halo_convolution arguments");
  SPMD_CHECK_ARG(start.dtype == SPMD_S32 && (!has_mask || offset.dtype == SPMD_S32),
                 "halo_convolution start/offset must be s32");
  if (axis != 1 || window.rank != 4 || cd->lhs_spatial[0] != 1) return SPMD_ERR_UNSUPPORTED;
  ConvWindow w;
  w.pieces = pieces;
  w.npieces = npieces;
  w.has_mask = has_mask;
  w.has_low = has_low;
  w.start = (const int32_t*)start.data;
  w.offset = has_mask ? (const int32_t*)offset.data : nullptr;
  w.low = low;
  w.high = high;
  if (numel(out) * nparts == 0) return SPMD_OK;
  return conv_tcgen05(window, rhs, out, *cd, nparts, as_stream(stream), &w);
}
