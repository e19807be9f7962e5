// f32 Dot on the tensor cores: 3xTF32 split GEMM (config C1, the f32 einsum
// BSM,MH->BSH; reference simulator.py:258-275 evaluates it as a float64
// einsum rounded once to float32).
//
// Every f32 operand x is split into x_hi = tf32(x) (round to nearest) and
// x_lo = x - x_hi (exact in f32; the tensor core reads it as tf32 again),
// and the product is accumulated as
//     A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi          (fp32 in TMEM)
// dropping only A_lo.B_lo (~2^-22 relative).  The products run as
// tcgen05.mma kind::tf32 (UMMA 256x256x8 per CTA pair); the result matches
// the f64 reference to ~1e-6 normwise (the test bound is the reference's own
// default tolerance, 1e-4).  Against the SIMT fp64 path (contract.cu) this is
// the tensor-core rate: 3 tf32 MMAs per fp32 product at 1.1 PF/s dense.
//
// Both operands are fed K-major: an MN-major operand (the C1 weight w[M,H]
// contracting M) is transposed by the split pass.
// Structure = the 2-CTA bf16 GEMM (gemm_tcgen05.cu) with fp32 elements:
// 128-byte rows hold 32 K elements, a k-block stages A_hi, A_lo, B_hi, B_lo
// (16 KB each per CTA), the leader issues 4 K-steps x 3 products; 4
// epilogue warps per CTA drain their 32 TMEM lanes as fp32 rows.
// The hi / lo operands are produced by one HBM pass (split_tf32_kernel) into
// stream-ordered scratch (cudaMallocAsync, graph-capturable).
#include "tcgen05.cuh"

#include <string.h>

namespace spmd {

constexpr int TBK = 32;                  // fp32 K elements per 128-byte row
constexpr int TBM = 256, TBN = 256, THALF = 128;

template <int STAGES>
struct SmemT {
  static constexpr int OP_BYTES = THALF * TBK * 4;          // 16 KB: one of A_hi/A_lo/B_hi/B_lo
  static constexpr int STAGE_BYTES = 4 * OP_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

struct TShape {
  int M, N, K;
  int nb[3];
  int mt, nt, group;
  int64_t tiles;
  float* out;
  int64_t out_batch;     // elements between batches (M * N)
};

__device__ __forceinline__ void tc_mma_2sm_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Instruction descriptor: kind::tf32, tf32 x tf32 -> f32.
__host__ __device__ constexpr uint32_t make_idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void ttile_coords(const TShape& g, int64_t t, int& b, int& m, int& n) {
  const int64_t per = (int64_t)g.mt * g.nt;
  b = (int)(t / per);
  const int r = (int)(t - (int64_t)b * per);
  const int G = g.group;
  const int group = r / (G * g.nt);
  const int first = group * G;
  const int gs = g.mt - first < G ? g.mt - first : G;
  const int rr = r - group * G * g.nt;
  m = first + rr % gs;
  n = rr / gs;
}

__device__ __forceinline__ void split1(float v, float& h, float& l) { split_tf32(v, h, l); }

// K-major operand: elementwise split, 16-byte vectors (scalar tail / when
// misaligned).
__global__ void split_tf32_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t n) {
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) |
                     reinterpret_cast<uintptr_t>(lo)) & 15) == 0;
  const int64_t nv = vec ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
    float4 h, l;
    split1(v.x, h.x, l.x);
    split1(v.y, h.y, l.y);
    split1(v.z, h.z, l.z);
    split1(v.w, h.w, l.w);
    reinterpret_cast<float4*>(hi)[i] = h;
    reinterpret_cast<float4*>(lo)[i] = l;
  }
  for (int64_t i = nv * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    split1(x[i], hi[i], lo[i]);
}

// MN-major operand (MN contiguous, K strided) -> K-major dense hi / lo copies
// [batch][MN][K] through a 32x32 shared-memory tile (coalesced both ways).
// Measured: with the MN-major SW128 descriptors that serve the bf16 GEMM, a
// kind::tf32 MMA returned an all-zero result for an MN-major B (K-major B
// exact), so both operands are fed K-major.
struct SplitView {
  int64_t mn, k, st_k;              // MN extent (stride 1), K extent and stride
  int64_t bsize[3], bstride[3];     // batch dims (innermost first)
};

// 64 x 64 tiles, 256 threads: 16-byte loads along MN and 16-byte stores
// along K (the 32 x 32 / 4-byte version ran at 3.1 TB/s on C1's weight).
__global__ void __launch_bounds__(256) split_tf32_transpose_kernel(const float* __restrict__ x,
                                                                   SplitView v,
                                                                   float* __restrict__ hi,
                                                                   float* __restrict__ lo) {
  __shared__ float tile[64][65];
  const int64_t b = blockIdx.z;
  int64_t boff = 0, r = b;
  for (int i = 0; i < 3; ++i) {
    boff += (r % v.bsize[i]) * v.bstride[i];
    r /= v.bsize[i];
  }
  const int64_t mn0 = (int64_t)blockIdx.x * 64, k0 = (int64_t)blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 16 x 16
  const bool vec_in = (v.mn & 3) == 0 && (v.st_k & 3) == 0 && (boff & 3) == 0 &&
                      (reinterpret_cast<uintptr_t>(x) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kk = ty + 16 * i;
    const int64_t k = k0 + kk, mn = mn0 + 4 * tx;
    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < v.k) {
      const float* src = x + boff + k * v.st_k + mn;
      if (vec_in && mn + 3 < v.mn) {
        f = __ldcs(reinterpret_cast<const float4*>(src));
      } else {
        if (mn < v.mn) f.x = src[0];
        if (mn + 1 < v.mn) f.y = src[1];
        if (mn + 2 < v.mn) f.z = src[2];
        if (mn + 3 < v.mn) f.w = src[3];
      }
    }
    tile[kk][4 * tx] = f.x;
    tile[kk][4 * tx + 1] = f.y;
    tile[kk][4 * tx + 2] = f.z;
    tile[kk][4 * tx + 3] = f.w;
  }
  __syncthreads();
  const bool vec_out = (v.k & 3) == 0 && (reinterpret_cast<uintptr_t>(hi) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(lo) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int mm = ty + 16 * i;
    const int64_t mn = mn0 + mm, k = k0 + 4 * tx;
    if (mn >= v.mn) continue;
    float val[4], h4[4], l4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      val[j] = tile[4 * tx + j][mm];
      uint32_t h;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(val[j]));
      h4[j] = __uint_as_float(h);
      l4[j] = isfinite(val[j]) ? val[j] - h4[j] : 0.f;
    }
    const int64_t o = (b * v.mn + mn) * v.k + k;
    if (vec_out && k + 3 < v.k) {
      *reinterpret_cast<float4*>(hi + o) = make_float4(h4[0], h4[1], h4[2], h4[3]);
      *reinterpret_cast<float4*>(lo + o) = make_float4(l4[0], l4[1], l4[2], l4[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (k + j < v.k) {
          hi[o + j] = h4[j];
          lo[o + j] = l4[j];
        }
    }
  }
}

// Loopback all-gather along K of an MN-major [K_local][MN] operand fused with
// its 3xTF32 split and transpose: partition p's output is the K-major hi / lo
// [MN][gs * K_local] with K rows [j * K_local, (j + 1) * K_local) taken from
// group member j's shard.  64 x 64 tiles as split_tf32_transpose_kernel.
struct GatherK {
  int64_t k_local, mn;
  int gs;
  int8_t src[SPMD_MAX_PARTS][8];   // [p][j]: partition holding K block j of p's gather
};

__global__ void __launch_bounds__(256) gather_split_transpose_kernel(const float* __restrict__ x,
                                                                    GatherK g,
                                                                    float* __restrict__ hi,
                                                                    float* __restrict__ lo) {
  __shared__ float tile[64][65];
  const int p = blockIdx.z;
  const int64_t K = g.k_local * g.gs;
  const int64_t mn0 = (int64_t)blockIdx.x * 64, k0 = (int64_t)blockIdx.y * 64;
  const int j = (int)(k0 / g.k_local);          // k_local % 64 == 0: one member per tile
  const float* src = x + (int64_t)g.src[p][j] * g.k_local * g.mn + (k0 - j * g.k_local) * g.mn;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kk = ty + 16 * i;
    const int64_t mn = mn0 + 4 * tx;
    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
    if (mn + 3 < g.mn) f = __ldcs(reinterpret_cast<const float4*>(src + kk * g.mn + mn));
    tile[kk][4 * tx] = f.x;
    tile[kk][4 * tx + 1] = f.y;
    tile[kk][4 * tx + 2] = f.z;
    tile[kk][4 * tx + 3] = f.w;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int mm = ty + 16 * i;
    const int64_t mn = mn0 + mm, k = k0 + 4 * tx;
    if (mn >= g.mn) continue;
    float4 h, l;
    split_tf32(tile[4 * tx][mm], h.x, l.x);
    split_tf32(tile[4 * tx + 1][mm], h.y, l.y);
    split_tf32(tile[4 * tx + 2][mm], h.z, l.z);
    split_tf32(tile[4 * tx + 3][mm], h.w, l.w);
    const int64_t o = ((int64_t)p * g.mn + mn) * K + k;
    *reinterpret_cast<float4*>(hi + o) = h;
    *reinterpret_cast<float4*>(lo + o) = l;
  }
}

// Split one operand into hi / lo K-major copies at `hi`, `lo` (each sized for
// the operand's own layout when it is K-major, else dense [batch][MN][K]) and
// rewrite `view` to describe them.
// The dense K-major view [b2][b1][b0][MN][K] an MN-major operand is split
// into (split_tf32_transpose_kernel's output layout).
static OperandView kmajor_view(const OperandView& mnv) {
  OperandView kv;
  kv.size[0] = mnv.size[1], kv.stride[0] = 1;
  kv.size[1] = mnv.size[0], kv.stride[1] = mnv.size[1];
  int64_t st = mnv.size[0] * mnv.size[1];
  for (int i = 0; i < 3; ++i) {
    kv.size[2 + i] = mnv.size[2 + i];
    kv.stride[2 + i] = mnv.size[2 + i] > 1 ? st : 8;
    st *= mnv.size[2 + i];
  }
  return kv;
}

static int split_operand(const float* src, int64_t n, OperandView* view, int mn_major, float* hi,
                         float* lo, cudaStream_t s) {
  if (!mn_major) {
    split_tf32_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(src, hi, lo, n);
    return launched(s);
  }
  SplitView v;
  v.mn = view->size[0];
  v.k = view->size[1];
  v.st_k = view->stride[1];
  int64_t nb = 1;
  for (int i = 0; i < 3; ++i) {
    v.bsize[i] = view->size[2 + i];
    v.bstride[i] = view->stride[2 + i];
    nb *= v.bsize[i];
  }
  if (nb > 65535) return SPMD_ERR_UNSUPPORTED;
  dim3 grid((unsigned)((v.mn + 63) / 64), (unsigned)((v.k + 63) / 64), (unsigned)nb);
  split_tf32_transpose_kernel<<<grid, 256, 0, s>>>(src, v, hi, lo);
  OperandView kv = kmajor_view(*view);
  *view = kv;
  return launched(s);
}

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_f32_3xtf32_2sm(const __grid_constant__ CUtensorMap map_ah,
                        const __grid_constant__ CUtensorMap map_al,
                        const __grid_constant__ CUtensorMap map_bh,
                        const __grid_constant__ CUtensorMap map_bl, TShape g) {
  typedef SmemT<STAGES> L;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  const int kblocks = (g.K + TBK - 1) / TBK;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int b, m, n;
      ttile_coords(g, t, b, m, n);
      const int b0 = b % g.nb[0], b1 = (b / g.nb[0]) % g.nb[1], b2 = b / (g.nb[0] * g.nb[1]);
      const int mrow = m * TBM + rank * THALF, nrow = n * TBN + rank * THALF;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * L::STAGE_BYTES;
        if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
        const int k0 = kb * TBK;
        const CUtensorMap* ma[2] = {&map_ah, &map_al};
        const CUtensorMap* mb[2] = {&map_bh, &map_bl};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          tma_load_5d_2sm(st + p * L::OP_BYTES, ma[p], &full[s], k0, mrow, b0, b1, b2);
          tma_load_5d_2sm(st + (2 + p) * L::OP_BYTES, mb[p], &full[s], k0, nrow, b0, b1, b2);
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader CTA, whole warp, one elected lane) ----------------
    const uint32_t idesc = make_idesc_tf32(TBM, TBN, 0, 0);
    // K-major: a K-step of 8 fp32 is 32 bytes inside the 128-byte row
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * TBN;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        uint32_t pred;
        asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}"
                     : "=r"(pred));
        if (pred) {
          const uint32_t st = smem_u32(smem + s * L::STAGE_BYTES);
          const uint32_t ah = st, al = st + L::OP_BYTES;
          const uint32_t bh = st + 2 * L::OP_BYTES, bl = st + 3 * L::OP_BYTES;
#pragma unroll
          for (int k = 0; k < TBK / 8; ++k) {
            const uint64_t dah = make_desc(ah + k * 32, 16, 1024);
            const uint64_t dal = make_desc(al + k * 32, 16, 1024);
            const uint64_t dbh = make_desc(bh + k * 32, 16, 1024);
            const uint64_t dbl = make_desc(bl + k * 32, 16, 1024);
            // small terms first, then the leading product
            tc_mma_2sm_tf32(d_tmem, dal, dbh, idesc, (kb | k) != 0);
            tc_mma_2sm_tf32(d_tmem, dah, dbl, idesc, 1);
            tc_mma_2sm_tf32(d_tmem, dah, dbh, idesc, 1);
          }
          tc_commit_2sm_mc(&empty[s]);
          if (kb == kblocks - 1) tc_commit_2sm_mc(&tfull[acc]);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 4 warps per CTA, own TMEM lane quarter ----------------
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int b, m, n;
      ttile_coords(g, t, b, m, n);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int row = m * TBM + rank * THALF + ew * 32 + lane;
      float* orow = g.out + (int64_t)b * g.out_batch + (int64_t)row * g.N;
      const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + acc * TBN;
#pragma unroll 1
      for (int c0 = 0; c0 < TBN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c0, r);
        const int col = n * TBN + c0;
        if (row < g.M && col < g.N) {
          if (col + 32 <= g.N && (g.N & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4*>(orow + col)[j] =
                  make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                              __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          } else {
            for (int j = 0; j < 32 && col + j < g.N; ++j) orow[col + j] = __uint_as_float(r[j]);
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
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Wide variant: 256 x 512 pair tiles (two N=256 halves per K step, the whole
// TMEM as one accumulator, 8 epilogue warps), 2 stages of A_hi/A_lo/B_hi/B_lo
// = 96 KB per CTA.  L2 -> SM bytes per MMA cycle fall from 42 B/clk/SM (the
// 256 x 256 kernel: 64 KB per 1536 cycles, at the L2 cap) to 31.
template <int STAGES>
struct SmemTW {
  static constexpr int A_BYTES = THALF * TBK * 4;           // 16 KB
  static constexpr int B_BYTES = 2 * THALF * TBK * 4;       // 32 KB: two N=256 halves
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    gemm_f32_3xtf32_2sm_wide(const __grid_constant__ CUtensorMap map_ah,
                             const __grid_constant__ CUtensorMap map_al,
                             const __grid_constant__ CUtensorMap map_bh,
                             const __grid_constant__ CUtensorMap map_bl, TShape g) {
  typedef SmemTW<STAGES> L;
  constexpr int WN = 512, HN = 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
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
  const int kblocks = (g.K + TBK - 1) / TBK;

  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int b, m, n;
      ttile_coords(g, t, b, m, n);
      const int b0 = b % g.nb[0], b1 = (b / g.nb[0]) % g.nb[1], b2 = b / (g.nb[0] * g.nb[1]);
      const int mrow = m * TBM + rank * THALF;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * L::STAGE_BYTES;
        if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
        const int k0 = kb * TBK;
        tma_load_5d_2sm(st, &map_ah, &full[s], k0, mrow, b0, b1, b2);
        tma_load_5d_2sm(st + L::A_BYTES, &map_al, &full[s], k0, mrow, b0, b1, b2);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int nrow = n * WN + j * HN + rank * THALF;
          tma_load_5d_2sm(st + 2 * L::A_BYTES + j * (L::B_BYTES / 2), &map_bh, &full[s], k0, nrow,
                          b0, b1, b2);
          tma_load_5d_2sm(st + 2 * L::A_BYTES + L::B_BYTES + j * (L::B_BYTES / 2), &map_bl,
                          &full[s], k0, nrow, b0, b1, b2);
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1 && leader) {
    const uint32_t idesc = make_idesc_tf32(TBM, HN, 0, 0);
    int s = 0;
    uint32_t ph = 0, acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      mbar_wait(tempty, acc_ph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        uint32_t pred;
        asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}"
                     : "=r"(pred));
        if (pred) {
          const uint32_t st = smem_u32(smem + s * L::STAGE_BYTES);
          const uint32_t ah = st, al = st + L::A_BYTES;
          const uint32_t bh = st + 2 * L::A_BYTES, bl = bh + L::B_BYTES;
#pragma unroll
          for (int k = 0; k < TBK / 8; ++k) {
            const uint64_t dah = make_desc(ah + k * 32, 16, 1024);
            const uint64_t dal = make_desc(al + k * 32, 16, 1024);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint64_t dbh = make_desc(bh + j * (L::B_BYTES / 2) + k * 32, 16, 1024);
              const uint64_t dbl = make_desc(bl + j * (L::B_BYTES / 2) + k * 32, 16, 1024);
              const uint32_t d = tmem + j * HN;
              tc_mma_2sm_tf32(d, dal, dbh, idesc, (kb | k) != 0);
              tc_mma_2sm_tf32(d, dah, dbl, idesc, 1);
              tc_mma_2sm_tf32(d, dah, dbh, idesc, 1);
            }
          }
          tc_commit_2sm_mc(&empty[s]);
          if (kb == kblocks - 1) tc_commit_2sm_mc(tfull);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      acc_ph ^= 1;
    }
  } else if (warp >= 4) {
    // 8 epilogue warps: (TMEM lane quarter, column half)
    const int ew = warp - 4, quarter = warp & 3, half = ew >> 2;
    uint32_t acc_ph = 0;
    for (int64_t t = cluster; t < g.tiles; t += nclusters) {
      int b, m, n;
      ttile_coords(g, t, b, m, n);
      mbar_wait(tfull, acc_ph);
      tc_fence_after();
      const int row = m * TBM + rank * THALF + quarter * 32 + lane;
      float* orow = g.out + (int64_t)b * g.out_batch + (int64_t)row * g.N;
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + half * HN;
#pragma unroll 1
      for (int c0 = 0; c0 < HN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c0, r);
        const int col = n * WN + half * HN + c0;
        if (row < g.M && col < g.N) {
          if (col + 32 <= g.N && (g.N & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4*>(orow + col)[j] =
                  make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                              __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          } else {
            for (int j = 0; j < 32 && col + j < g.N; ++j) orow[col + j] = __uint_as_float(r[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(tempty);
      acc_ph ^= 1;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// 5-D fp32 tensor map over an OperandView (element strides), 128B swizzle.
static bool encode_f32(CUtensorMap* map, void* base, const OperandView& v, int box_inner,
                       int box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) dims[i] = (cuuint64_t)v.size[i];
  for (int i = 1; i < 5; ++i) {
    strides[i - 1] = (cuuint64_t)(v.stride[i] * 4);
    if (strides[i - 1] % 16 != 0 || strides[i - 1] >= ((cuuint64_t)1 << 40)) return false;
  }
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// The hi / lo scratch comes from the device's stream-ordered pool.  Its
// default release threshold (0) hands freed memory back to the driver at
// every synchronisation, so each call re-mapped ~GBs (measured: 3xTF32 calls
// in a fresh process at 60-130 instead of ~240 TF/s); keep it cached.
static void keep_pool_memory() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  const uint64_t bit = 1ull << dev;
  if (done.load() & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.fetch_or(bit);
}

// f32 Dot -> 3xTF32 tcgen05 GEMM; SPMD_ERR_UNSUPPORTED when the layout or the
// size does not qualify (the caller then runs the SIMT fp64 kernel).
int dot_tf32x3(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
               const spmd_dot_dims& dd, int64_t nparts, cudaStream_t s, const float* lhs_hi,
               const float* lhs_lo, const float* rhs_hi, const float* rhs_lo) {
  if (lhs.dtype != SPMD_F32 || !option(OPT_F32_DOT_TC) || dd.epilogue != 0)
    return SPMD_ERR_UNSUPPORTED;
  GemmLayout lay;
  if (gemm_layout(lhs, rhs, out, dd, nparts, &lay) != SPMD_OK) return SPMD_ERR_UNSUPPORTED;
  // small Dots (the parity-sized golden cases) stay on the exact fp64 path
  if (lay.M < 256 || lay.N < 256 || lay.K < 64) return SPMD_ERR_UNSUPPORTED;
  const bool presplit = lhs_hi != nullptr;
  if (presplit && (lay.a_mn || !lhs_lo || ((reinterpret_cast<uintptr_t>(lhs_hi) |
                                            reinterpret_cast<uintptr_t>(lhs_lo)) & 15)))
    return SPMD_ERR_UNSUPPORTED;
  const bool presplit_b = rhs_hi != nullptr;
  if (presplit_b && (!rhs_lo || ((reinterpret_cast<uintptr_t>(rhs_hi) |
                                  reinterpret_cast<uintptr_t>(rhs_lo)) & 15)))
    return SPMD_ERR_UNSUPPORTED;
  const int64_t na = presplit ? 0 : numel(lhs) * nparts;
  const int64_t nb = presplit_b ? 0 : numel(rhs) * nparts;
  // each of the four split copies starts 16-byte aligned (vector stores, TMA)
  const int64_t na4 = (na + 3) & ~(int64_t)3, nb4 = (nb + 3) & ~(int64_t)3;
  keep_pool_memory();
  float* scratch = nullptr;
  if (cudaMallocAsync((void**)&scratch, (size_t)(2 * (na4 + nb4)) * 4, s) != cudaSuccess) {
    cudaGetLastError();
    return SPMD_ERR_UNSUPPORTED;
  }
  // an MN-major operand's dense transpose is never larger than its buffer
  // (the view covers a sub-box of it), so the same scratch sizes hold
  float *ah = scratch, *al = scratch + na4, *bh = scratch + 2 * na4, *bl = bh + nb4;
  OperandView va = lay.va, vb = lay.vb;
  int rc = SPMD_OK;
  if (presplit) {
    ah = const_cast<float*>(lhs_hi);
    al = const_cast<float*>(lhs_lo);
  } else {
    rc = split_operand((const float*)lhs.data, na, &va, lay.a_mn, ah, al, s);
  }
  if (rc == SPMD_OK && presplit_b) {
    // the K-major halves split_operand would have written (MN-major rhs:
    // dense [batch][N][K]; K-major rhs: its own layout)
    bh = const_cast<float*>(rhs_hi);
    bl = const_cast<float*>(rhs_lo);
    if (lay.b_mn) vb = kmajor_view(vb);
  } else if (rc == SPMD_OK) {
    rc = split_operand((const float*)rhs.data, nb, &vb, lay.b_mn, bh, bl, s);
  }
  if (rc != SPMD_OK) {
    cudaFreeAsync(scratch, s);
    return rc;
  }
  CUtensorMap mah, mal, mbh, mbl;
  bool ok = encode_f32(&mah, ah, va, TBK, THALF) && encode_f32(&mal, al, va, TBK, THALF) &&
            encode_f32(&mbh, bh, vb, TBK, THALF) && encode_f32(&mbl, bl, vb, TBK, THALF);
  if (!ok) {
    cudaFreeAsync(scratch, s);
    return SPMD_ERR_UNSUPPORTED;
  }
  TShape g;
  memset(&g, 0, sizeof(g));
  g.M = lay.M;
  g.N = lay.N;
  g.K = lay.K;
  for (int i = 0; i < 3; ++i) g.nb[i] = lay.nb[i];
  g.group = 8;
  g.out = (float*)out.data;
  g.out_batch = (int64_t)g.M * g.N;
  const int sms = sm_budget();
  // 256 x 512 tiles move fewer L2 bytes per MMA, 256 x 256 tiles quantise
  // better over the 74 CTA pairs: take the wide tile unless its last wave is
  // emptier (measured at C1's 8192 x 4096 x 4096: 256 tiles = 3.5 waves, wide
  // 241 vs 266 TF/s; 8192^3: wide 278 vs 275)
  const int64_t nbt = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];
  const int64_t t_wide = (int64_t)((g.M + TBM - 1) / TBM) * ((g.N + 511) / 512) * nbt;
  const int64_t t_sq = (int64_t)((g.M + TBM - 1) / TBM) * ((g.N + TBN - 1) / TBN) * nbt;
  const int64_t pairs = sms / 2;
  auto wave_eff = [&](int64_t t) { return (double)t / (double)(((t + pairs - 1) / pairs) * pairs); };
  if (g.N >= 512 && option(OPT_GEMM_MODE) == 3 && wave_eff(t_wide) >= wave_eff(t_sq) - 0.02) {
    g.mt = (g.M + TBM - 1) / TBM;
    g.nt = (g.N + 511) / 512;
    g.tiles = (int64_t)g.mt * g.nt * g.nb[0] * g.nb[1] * g.nb[2];
    typedef SmemTW<2> LW;
    static_assert(LW::TOTAL <= 232448, "3xTF32 wide GEMM smem");
    static std::atomic<uint64_t> attr_w{0};
    if (int rc = set_smem_attr((const void*)gemm_f32_3xtf32_2sm_wide<2>, LW::TOTAL, &attr_w))
      return rc;
    const int64_t clusters = g.tiles < sms / 2 ? g.tiles : sms / 2;
    gemm_f32_3xtf32_2sm_wide<2><<<(unsigned)(2 * clusters), 384, LW::TOTAL, s>>>(mah, mal, mbh,
                                                                               mbl, g);
    rc = launched(s);
    cudaFreeAsync(scratch, s);
    return rc;
  }
  g.mt = (g.M + TBM - 1) / TBM;
  g.nt = (g.N + TBN - 1) / TBN;
  g.tiles = (int64_t)g.mt * g.nt * g.nb[0] * g.nb[1] * g.nb[2];
  typedef SmemT<3> L;
  static_assert(L::TOTAL <= 232448, "3xTF32 GEMM smem");
  static std::atomic<uint64_t> attr_done{0};
  if (int rc = set_smem_attr((const void*)gemm_f32_3xtf32_2sm<3>, L::TOTAL, &attr_done)) return rc;
  const int64_t clusters = g.tiles < sms / 2 ? g.tiles : sms / 2;
  gemm_f32_3xtf32_2sm<3><<<(unsigned)(2 * clusters), 256, L::TOTAL, s>>>(mah, mal, mbh, mbl, g);
  rc = launched(s);
  cudaFreeAsync(scratch, s);
  return rc;
}

}  // namespace spmd

using namespace spmd;

// Loopback all-gather along dim 0 of an f32 [K_local, N] operand (per
// partition) written as the tf32 hi / lo halves of its K-major transpose
// [N, K] -- the rhs layout spmd_dot_f32_presplit takes for an MN-major rhs.
// SPMD_ERR_UNSUPPORTED unless K_local % 64 == 0 and N % 4 == 0.
extern "C" int spmd_local_all_gather_split_t(spmd_tensor in, spmd_tensor hi, spmd_tensor lo,
                                             const int32_t* groups, int ngroups, int gsize,
                                             int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == SPMD_F32 && hi.dtype == SPMD_F32 && lo.dtype == SPMD_F32 &&
                     in.rank == 2 && hi.rank == 2 && lo.rank == 2,
                 "all-gather split-transpose expects f32 [K_local, N] -> [N, K]");
  const int64_t kl = in.dims[0], N = in.dims[1];
  SPMD_CHECK_ARG(hi.dims[0] == N && hi.dims[1] == kl * gsize && lo.dims[0] == N &&
                     lo.dims[1] == kl * gsize,
                 "all-gather split-transpose output shape");
  if (kl % 64 || N % 4 || gsize > 8 || nparts > SPMD_MAX_PARTS || nparts > 65535 ||
      ngroups * gsize != nparts ||
      ((reinterpret_cast<uintptr_t>(in.data) | reinterpret_cast<uintptr_t>(hi.data) |
        reinterpret_cast<uintptr_t>(lo.data)) & 15))
    return SPMD_ERR_UNSUPPORTED;
  GatherK g;
  memset(&g, -1, sizeof(g));
  g.k_local = kl;
  g.mn = N;
  g.gs = gsize;
  for (int i = 0; i < ngroups * gsize; ++i) {
    const int d = groups[i];
    SPMD_CHECK_ARG(d >= 0 && d < nparts, "subgroups do not partition the devices");
    const int grp = i / gsize;
    for (int j = 0; j < gsize; ++j) g.src[d][j] = (int8_t)groups[grp * gsize + j];
  }
  if (numel(hi) * nparts == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)(kl * gsize / 64), (unsigned)nparts);
  gather_split_transpose_kernel<<<grid, 256, 0, s>>>((const float*)in.data, g, (float*)hi.data,
                                                     (float*)lo.data);
  return launched(s);
}
