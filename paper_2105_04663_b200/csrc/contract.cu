// Generalised dot (einsum) and convolution (reference simulator.py:258-277,
// 121-154).
//
// BF16 dots with a TMA-describable layout go to the tcgen05/TMEM GEMM
// (gemm_tcgen05.cu), large F32 dots to the 3xTF32 tcgen05 GEMM
// (gemm_tf32x3.cu).  Everything else -- small F32 (fp64 accumulation, one
// rounding, as the reference's float64 einsum), S32/U32 (int64 accumulation,
// wrap on the final cast, exact), and odd-layout BF16 -- runs the tiled SIMT
// kernel below, which addresses operands through arbitrary batch / free /
// contracting dim lists so no transposes are materialised.
#include "common.cuh"

#include <string.h>

namespace spmd {

struct DimList {
  int n;
  int64_t shape[SPMD_MAX_RANK];
  int64_t st_l[SPMD_MAX_RANK];   // stride in lhs (or input)
  int64_t st_r[SPMD_MAX_RANK];   // stride in rhs
};

struct DotArgs {
  DimList batch, m, n, k;   // m: lhs-free (st_l), n: rhs-free (st_r), k: both
  int64_t B, M, N, K;
  int64_t lhs_part, rhs_part, out_part;
  int epilogue;
};

__device__ __forceinline__ int64_t off_l(int64_t idx, const DimList& d) {
  int64_t o = 0;
  for (int i = d.n - 1; i >= 0; --i) {
    int64_t c = idx % d.shape[i];
    idx /= d.shape[i];
    o += c * d.st_l[i];
  }
  return o;
}
__device__ __forceinline__ int64_t off_r(int64_t idx, const DimList& d) {
  int64_t o = 0;
  for (int i = d.n - 1; i >= 0; --i) {
    int64_t c = idx % d.shape[i];
    idx /= d.shape[i];
    o += c * d.st_r[i];
  }
  return o;
}

template <typename T> struct Acc { typedef float type; };
template <> struct Acc<float> { typedef double type; };
template <> struct Acc<int32_t> { typedef int64_t type; };
template <> struct Acc<uint32_t> { typedef int64_t type; };

template <typename A> __device__ __forceinline__ A to_acc(float v) { return (A)v; }

template <typename T, typename A>
__device__ __forceinline__ T from_acc(A v) { return st<T>((typename Compute<T>::type)v); }
template <> __device__ __forceinline__ int32_t from_acc<int32_t, int64_t>(int64_t v) {
  return (int32_t)(uint32_t)(uint64_t)v;
}
template <> __device__ __forceinline__ uint32_t from_acc<uint32_t, int64_t>(int64_t v) {
  return (uint32_t)(uint64_t)v;
}

constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
__global__ void __launch_bounds__(256) dot_simt_kernel(const T* __restrict__ lhs,
                                                       const T* __restrict__ rhs,
                                                       T* __restrict__ out, DotArgs a,
                                                       int64_t nbatch_total) {
  typedef typename Acc<T>::type A;
  __shared__ A sa[TK][TM + 1];
  __shared__ A sb[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.y * TM, n0 = (int64_t)blockIdx.x * TN;
  for (int64_t z = blockIdx.z; z < nbatch_total; z += gridDim.z) {
    const int64_t p = z / a.B, b = z - p * a.B;
    const T* L = lhs + p * a.lhs_part + off_l(b, a.batch);
    const T* R = rhs + p * a.rhs_part + off_r(b, a.batch);
    A acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    for (int64_t k0 = 0; k0 < a.K; k0 += TK) {
      for (int e = threadIdx.x; e < TK * TM; e += 256) {
        int kk = e / TM, mm = e % TM;
        int64_t gm = m0 + mm, gk = k0 + kk;
        sa[kk][mm] = (gm < a.M && gk < a.K)
                         ? (A)ld<T>(L[off_l(gm, a.m) + off_l(gk, a.k)]) : (A)0;
        int64_t gn = n0 + mm;
        sb[kk][mm] = (gn < a.N && gk < a.K)
                         ? (A)ld<T>(R[off_r(gn, a.n) + off_r(gk, a.k)]) : (A)0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        A av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = sa[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = sb[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
      }
      __syncthreads();
    }
    T* O = out + p * a.out_part + b * a.M * a.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t gm = m0 + ty + 16 * i;
      if (gm >= a.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t gn = n0 + tx + 16 * j;
        if (gn >= a.N) continue;
        A v = acc[i][j];
        if (a.epilogue == 1 && v < (A)0) v = 0;
        O[gm * a.N + gn] = from_acc<T, A>(v);
      }
    }
  }
}

static void strides_of(const spmd_tensor& t, int64_t* st) {
  int64_t acc = 1;
  for (int k = t.rank - 1; k >= 0; --k) {
    st[k] = acc;
    acc *= t.dims[k];
  }
}


// ---------------------------------------------------------------------------
// direct convolution (parity path; B200 implicit GEMM is in conv_tcgen05.cu)
// ---------------------------------------------------------------------------
struct ConvArgs {
  int nsp;
  int64_t B, Cin, Cout;
  int64_t in_sp[SPMD_MAX_RANK], out_sp[SPMD_MAX_RANK], win[SPMD_MAX_RANK];
  int64_t l_st_b, l_st_c, l_st_sp[SPMD_MAX_RANK];
  int64_t r_st_o, r_st_i, r_st_sp[SPMD_MAX_RANK];
  int64_t o_st_b, o_st_c, o_st_sp[SPMD_MAX_RANK];
  int64_t stride[SPMD_MAX_RANK], pad_lo[SPMD_MAX_RANK], bd[SPMD_MAX_RANK], wd[SPMD_MAX_RANK];
  int64_t lhs_part, rhs_part, out_part, nout;
  int relu;
};

template <typename T>
__global__ void conv_direct_kernel(const T* __restrict__ lhs, const T* __restrict__ rhs,
                                   T* __restrict__ out, ConvArgs a, int64_t nparts) {
  typedef typename Acc<T>::type A;
  const int64_t total = a.nout * nparts;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = idx / a.nout, r = idx - p * a.nout;
    // canonical output order: [b, o, spatial...]
    int64_t osp[SPMD_MAX_RANK];
    for (int i = a.nsp - 1; i >= 0; --i) {
      osp[i] = r % a.out_sp[i];
      r /= a.out_sp[i];
    }
    int64_t o = r % a.Cout;
    int64_t b = r / a.Cout;
    const T* L = lhs + p * a.lhs_part + b * a.l_st_b;
    const T* R = rhs + p * a.rhs_part + o * a.r_st_o;
    int64_t nwin = 1;
    for (int i = 0; i < a.nsp; ++i) nwin *= a.win[i];
    A acc = 0;
    for (int64_t w = 0; w < nwin; ++w) {
      int64_t rem = w, loff = 0, roff = 0;
      bool valid = true;
      for (int i = a.nsp - 1; i >= 0; --i) {
        int64_t q = rem % a.win[i];
        rem /= a.win[i];
        int64_t pos = osp[i] * a.stride[i] - a.pad_lo[i] + q * a.wd[i];  // dilated coords
        if (pos < 0 || pos % a.bd[i] != 0) { valid = false; break; }
        int64_t src = pos / a.bd[i];
        if (src >= a.in_sp[i]) { valid = false; break; }
        loff += src * a.l_st_sp[i];
        roff += q * a.r_st_sp[i];
      }
      if (!valid) continue;
      for (int64_t c = 0; c < a.Cin; ++c)
        acc += (A)ld<T>(L[loff + c * a.l_st_c]) * (A)ld<T>(R[roff + c * a.r_st_i]);
    }
    int64_t ooff = p * a.out_part + b * a.o_st_b + o * a.o_st_c;
    for (int i = 0; i < a.nsp; ++i) ooff += osp[i] * a.o_st_sp[i];
    if (a.relu && acc < (A)0) acc = 0;
    out[ooff] = from_acc<T, A>(acc);
  }
}

// Implemented in conv_tcgen05.cu (NHWC bf16 implicit GEMM).
struct ConvWindow;
int conv_tcgen05(const spmd_tensor& lhs, const spmd_tensor& rhs, const spmd_tensor& out,
                 const spmd_conv_dims& cd, int64_t nparts, cudaStream_t s, const ConvWindow* win);

}  // namespace spmd

using namespace spmd;

// f32 Dot with operands that arrive already split into their tf32 hi / lo
// halves (spmd_local_all_gather_split / _split_t): `lhs` / `rhs` give the
// shapes (their data is read only when that operand is not pre-split, i.e.
// its hi.data is NULL); a pre-split lhs is in its own (K-major) layout, a
// pre-split MN-major rhs in the dense K-major [batch][N][K] transpose.
// SPMD_ERR_UNSUPPORTED when the 3xTF32 path does not apply (the caller then
// forms the operands as hi + lo -- exact -- and runs spmd_dot).
extern "C" int spmd_dot_f32_presplit(spmd_tensor lhs, spmd_tensor lhs_hi, spmd_tensor lhs_lo,
                                     spmd_tensor rhs, spmd_tensor rhs_hi, spmd_tensor rhs_lo,
                                     spmd_tensor out, const spmd_dot_dims* dd, int64_t nparts,
                                     void* stream) {
  SPMD_CHECK_ARG(lhs.dtype == SPMD_F32 && rhs.dtype == SPMD_F32 && out.dtype == SPMD_F32,
                 "dot_f32_presplit expects f32");
  if (numel(out) * nparts == 0) return SPMD_OK;
  return dot_tf32x3(lhs, rhs, out, *dd, nparts, as_stream(stream), (const float*)lhs_hi.data,
                    (const float*)lhs_lo.data, (const float*)rhs_hi.data,
                    (const float*)rhs_lo.data);
}

// out = Dot(lhs, rhs) + resid (bf16, the Dot's output shape): the residual
// add of a Transformer layer folded into the GEMM epilogue (one fp32 add
// before the single rounding).  SPMD_ERR_UNSUPPORTED when the GEMM does not
// take the wide tcgen05 kernel -- the caller then runs spmd_dot + the add.
extern "C" int spmd_dot_add(spmd_tensor lhs, spmd_tensor rhs, spmd_tensor resid, spmd_tensor out,
                            const spmd_dot_dims* dd, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(lhs.dtype == SPMD_BF16 && rhs.dtype == SPMD_BF16 && out.dtype == SPMD_BF16 &&
                     resid.dtype == SPMD_BF16 && numel(resid) == numel(out) &&
                     resid.rank == out.rank,
                 "dot_add expects bf16 operands and a residual of the output's shape");
  for (int i = 0; i < out.rank; ++i)
    SPMD_CHECK_ARG(resid.dims[i] == out.dims[i], "dot_add residual shape");
  if (numel(out) * nparts == 0) return SPMD_OK;
  return dot_tcgen05(lhs, rhs, out, *dd, nparts, as_stream(stream), nullptr, resid.data);
}

extern "C" int spmd_dot(spmd_tensor lhs, spmd_tensor rhs, spmd_tensor out, const spmd_dot_dims* dd,
                        int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(lhs.dtype == rhs.dtype && lhs.dtype == out.dtype, "dot dtype mismatch");
  SPMD_CHECK_ARG(lhs.dtype != SPMD_PRED, "pred dot unsupported");
  cudaStream_t s = as_stream(stream);
  if (numel(out) * nparts == 0) return SPMD_OK;
  if (lhs.dtype == SPMD_BF16) {
    int rc = dot_tcgen05(lhs, rhs, out, *dd, nparts, s);
    if (rc != SPMD_ERR_UNSUPPORTED) return rc;
  }
  if (lhs.dtype == SPMD_F32) {
    int rc = dot_tf32x3(lhs, rhs, out, *dd, nparts, s);
    if (rc != SPMD_ERR_UNSUPPORTED) return rc;
  }
  int64_t ls[SPMD_MAX_RANK], rs[SPMD_MAX_RANK];
  strides_of(lhs, ls);
  strides_of(rhs, rs);
  DotArgs a;
  memset(&a, 0, sizeof(a));
  bool lused[SPMD_MAX_RANK] = {false}, rused[SPMD_MAX_RANK] = {false};
  a.B = a.M = a.N = a.K = 1;
  for (int i = 0; i < dd->n_batch; ++i) {
    int l = dd->lhs_batch[i], r = dd->rhs_batch[i];
    SPMD_CHECK_ARG(lhs.dims[l] == rhs.dims[r], "dot batch size mismatch");
    a.batch.shape[a.batch.n] = lhs.dims[l];
    a.batch.st_l[a.batch.n] = ls[l];
    a.batch.st_r[a.batch.n++] = rs[r];
    a.B *= lhs.dims[l];
    lused[l] = rused[r] = true;
  }
  for (int i = 0; i < dd->n_contract; ++i) {
    int l = dd->lhs_contracting[i], r = dd->rhs_contracting[i];
    SPMD_CHECK_ARG(lhs.dims[l] == rhs.dims[r], "dot contracting size mismatch");
    a.k.shape[a.k.n] = lhs.dims[l];
    a.k.st_l[a.k.n] = ls[l];
    a.k.st_r[a.k.n++] = rs[r];
    a.K *= lhs.dims[l];
    lused[l] = rused[r] = true;
  }
  for (int d = 0; d < lhs.rank; ++d)
    if (!lused[d]) {
      a.m.shape[a.m.n] = lhs.dims[d];
      a.m.st_l[a.m.n++] = ls[d];
      a.M *= lhs.dims[d];
    }
  for (int d = 0; d < rhs.rank; ++d)
    if (!rused[d]) {
      a.n.shape[a.n.n] = rhs.dims[d];
      a.n.st_r[a.n.n++] = rs[d];
      a.N *= rhs.dims[d];
    }
  SPMD_CHECK_ARG(a.B * a.M * a.N == numel(out), "dot output shape mismatch");
  a.lhs_part = numel(lhs);
  a.rhs_part = numel(rhs);
  a.out_part = numel(out);
  a.epilogue = dd->epilogue;
  int64_t zb = a.B * nparts;
  dim3 grid((unsigned)((a.N + TN - 1) / TN), (unsigned)((a.M + TM - 1) / TM),
            (unsigned)(zb < 65535 ? zb : 65535));
  SPMD_CHECK_ARG(grid.y <= 65535, "dot M too large for the SIMT path");
  switch (lhs.dtype) {
    case SPMD_F32:
      dot_simt_kernel<float><<<grid, 256, 0, s>>>((const float*)lhs.data, (const float*)rhs.data,
                                                  (float*)out.data, a, zb);
      break;
    case SPMD_S32:
      dot_simt_kernel<int32_t><<<grid, 256, 0, s>>>((const int32_t*)lhs.data,
                                                    (const int32_t*)rhs.data,
                                                    (int32_t*)out.data, a, zb);
      break;
    case SPMD_U32:
      dot_simt_kernel<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)lhs.data,
                                                     (const uint32_t*)rhs.data,
                                                     (uint32_t*)out.data, a, zb);
      break;
    case SPMD_BF16:
      dot_simt_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)lhs.data, (const bf16*)rhs.data,
                                                 (bf16*)out.data, a, zb);
      break;
    default:
      set_error("bad dot dtype");
      return SPMD_ERR_INVALID;
  }
  return launched(s);
}

extern "C" int spmd_convolution(spmd_tensor lhs, spmd_tensor rhs, spmd_tensor out,
                                const spmd_conv_dims* cd, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(lhs.dtype == rhs.dtype && lhs.dtype == out.dtype, "conv dtype mismatch");
  cudaStream_t s = as_stream(stream);
  if (numel(out) * nparts == 0) return SPMD_OK;
  if (lhs.dtype == SPMD_BF16) {
    int rc = conv_tcgen05(lhs, rhs, out, *cd, nparts, s, nullptr);
    if (rc != SPMD_ERR_UNSUPPORTED) return rc;
  }
  int64_t ls[SPMD_MAX_RANK], rs[SPMD_MAX_RANK], os[SPMD_MAX_RANK];
  strides_of(lhs, ls);
  strides_of(rhs, rs);
  strides_of(out, os);
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.nsp = cd->n_spatial;
  a.B = lhs.dims[cd->lhs_batch];
  a.Cin = lhs.dims[cd->lhs_feature];
  a.Cout = rhs.dims[cd->rhs_out_feature];
  SPMD_CHECK_ARG(rhs.dims[cd->rhs_in_feature] == a.Cin, "conv feature mismatch");
  a.l_st_b = ls[cd->lhs_batch];
  a.l_st_c = ls[cd->lhs_feature];
  a.r_st_o = rs[cd->rhs_out_feature];
  a.r_st_i = rs[cd->rhs_in_feature];
  a.o_st_b = os[cd->out_batch];
  a.o_st_c = os[cd->out_feature];
  for (int i = 0; i < a.nsp; ++i) {
    a.in_sp[i] = lhs.dims[cd->lhs_spatial[i]];
    a.out_sp[i] = out.dims[cd->out_spatial[i]];
    a.win[i] = rhs.dims[cd->rhs_spatial[i]];
    SPMD_CHECK_ARG(a.win[i] == cd->size[i], "window size mismatch");
    a.l_st_sp[i] = ls[cd->lhs_spatial[i]];
    a.r_st_sp[i] = rs[cd->rhs_spatial[i]];
    a.o_st_sp[i] = os[cd->out_spatial[i]];
    a.stride[i] = cd->stride[i];
    a.pad_lo[i] = cd->pad_low[i];
    a.bd[i] = cd->base_dilation[i];
    a.wd[i] = cd->window_dilation[i];
  }
  a.lhs_part = numel(lhs);
  a.rhs_part = numel(rhs);
  a.out_part = numel(out);
  a.nout = numel(out);
  a.relu = cd->epilogue == 1;
  int64_t total = a.nout * nparts;
  switch (lhs.dtype) {
    case SPMD_F32:
      conv_direct_kernel<float><<<grid_for(total, 128), 128, 0, s>>>(
          (const float*)lhs.data, (const float*)rhs.data, (float*)out.data, a, nparts);
      break;
    case SPMD_S32:
      conv_direct_kernel<int32_t><<<grid_for(total, 128), 128, 0, s>>>(
          (const int32_t*)lhs.data, (const int32_t*)rhs.data, (int32_t*)out.data, a, nparts);
      break;
    case SPMD_U32:
      conv_direct_kernel<uint32_t><<<grid_for(total, 128), 128, 0, s>>>(
          (const uint32_t*)lhs.data, (const uint32_t*)rhs.data, (uint32_t*)out.data, a, nparts);
      break;
    case SPMD_BF16:
      conv_direct_kernel<bf16><<<grid_for(total, 128), 128, 0, s>>>(
          (const bf16*)lhs.data, (const bf16*)rhs.data, (bf16*)out.data, a, nparts);
      break;
    default:
      set_error("bad conv dtype");
      return SPMD_ERR_INVALID;
  }
  return launched(s);
}
