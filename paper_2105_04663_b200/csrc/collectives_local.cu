// Loopback collectives: all partitions of a simulated mesh resident on ONE
// GPU (partition-stacked buffers).  Exact reference semantics
// (simulator.py:333-390): all-gather concatenates in subgroup order;
// all-reduce / reduce-scatter fold serially in subgroup order (so float
// results are bit-identical to the reference, not just within tolerance);
// all-to-all splits evenly and concatenates in group order; collective-permute
// zero-fills non-targets.  NCCL refuses two ranks on one GPU, so this is the
// comm backend for single-GPU parity runs -- still GPU-only.
#include "common.cuh"

#include <string.h>

namespace spmd {

struct GroupTab {
  int P, gsize;
  int8_t gid[SPMD_MAX_PARTS];
  int8_t gpos[SPMD_MAX_PARTS];
  int8_t members[SPMD_MAX_PARTS];   // [ngroups][gsize]
};

static int make_groups(const int32_t* groups, int ngroups, int gsize, int64_t nparts,
                       GroupTab& g) {
  if (nparts > SPMD_MAX_PARTS || ngroups * gsize != nparts) {
    set_error("subgroups do not partition the devices");
    return SPMD_ERR_SUBGROUP;
  }
  memset(&g, -1, sizeof(g));
  g.P = (int)nparts;
  g.gsize = gsize;
  for (int i = 0; i < ngroups * gsize; ++i) {
    int d = groups[i];
    if (d < 0 || d >= nparts || g.gid[d] != -1) {
      set_error("subgroups do not partition the devices");
      return SPMD_ERR_SUBGROUP;
    }
    g.gid[d] = (int8_t)(i / gsize);
    g.gpos[d] = (int8_t)(i % gsize);
    g.members[i] = (int8_t)d;
  }
  return SPMD_OK;
}

struct View {
  int rank;
  int64_t d[SPMD_MAX_RANK];
};

static View view_of(const spmd_tensor& t) {
  View v;
  v.rank = t.rank;
  for (int i = 0; i < SPMD_MAX_RANK; ++i) v.d[i] = i < t.rank ? t.dims[i] : 1;
  return v;
}

__device__ __forceinline__ void unravel_v(int64_t r, const View& v, int64_t* c) {
  for (int i = v.rank - 1; i >= 0; --i) {
    c[i] = r % v.d[i];
    r /= v.d[i];
  }
}
__device__ __forceinline__ int64_t ravel_v(const int64_t* c, const View& v) {
  int64_t o = 0;
  for (int i = 0; i < v.rank; ++i) o = o * v.d[i] + c[i];
  return o;
}

enum { K_AG = 0, K_A2A = 1, K_CP = 2 };

struct MoveArgs {
  int kind;
  View in, out, piece;
  int dim, split, concat;
  int8_t src_of[SPMD_MAX_PARTS];   // collective-permute: source partition or -1
};

template <typename T>
__global__ void local_move_kernel(const T* __restrict__ in, T* __restrict__ out, MoveArgs a,
                                  GroupTab g, int64_t n_out, int64_t n_in) {
  const int64_t total = n_out * g.P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int p = (int)(idx / n_out);
    int64_t r = idx - (int64_t)p * n_out;
    int64_t c[SPMD_MAX_RANK];
    unravel_v(r, a.out, c);
    int src;
    if (a.kind == K_CP) {
      src = a.src_of[p];
      if (src < 0) {
        out[idx] = T(0);
        continue;
      }
    } else if (a.kind == K_AG) {
      int64_t nd = a.in.d[a.dim];
      int j = (int)(c[a.dim] / nd);
      c[a.dim] -= j * nd;
      src = g.members[g.gid[p] * g.gsize + j];
    } else {   // all-to-all
      int64_t pc = a.piece.d[a.concat];
      int j = (int)(c[a.concat] / pc);
      c[a.concat] -= j * pc;
      c[a.split] += (int64_t)g.gpos[p] * a.piece.d[a.split];
      src = g.members[g.gid[p] * g.gsize + j];
    }
    out[idx] = in[(int64_t)src * n_in + ravel_v(c, a.in)];
  }
}

template <typename T>
__global__ void local_reduce_kernel(const T* __restrict__ in, T* __restrict__ out, View vin,
                                    View vout, int dim, int scatter, int kind, GroupTab g,
                                    int64_t n_out, int64_t n_in) {
  typedef typename Compute<T>::type C;
  const int64_t total = n_out * g.P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int p = (int)(idx / n_out);
    int64_t r = idx - (int64_t)p * n_out;
    int64_t c[SPMD_MAX_RANK];
    unravel_v(r, vout, c);
    if (scatter) c[dim] += (int64_t)g.gpos[p] * vout.d[dim];
    int64_t off = ravel_v(c, vin);
    const int8_t* mem = g.members + g.gid[p] * g.gsize;
    C acc = ld<T>(in[(int64_t)mem[0] * n_in + off]);
    for (int j = 1; j < g.gsize; ++j)   // serial fold in group order
      acc = combine<C>(kind, acc, ld<T>(in[(int64_t)mem[j] * n_in + off]));
    out[idx] = st<T>(acc);
  }
}

// Row form of a move: every (partition p, piece j, outer index o) is one
// contiguous run of L elements on both sides,
//   dst = out + p*n_out + sum_k o_k*dstr[k] + j*dst_j
//   src = in + src_p*n_in + sum_k o_k*sstr[k] + gpos[p]*src_pos
// with src_p the group member j of p's group (all-gather / all-to-all) or
// p's permute source (-1: zero fill).  Blocks own 256 x ROW_U 16-byte
// vectors of one run, so the index math runs once per block (the element
// kernel above decodes up to 8 dims per element: ~0.9 TB/s on C1's gathers).
struct RowMove {
  int kind, outer_rank, G;
  int64_t oshape[SPMD_MAX_RANK], sstr[SPMD_MAX_RANK], dstr[SPMD_MAX_RANK];
  int64_t L, dst_j, src_pos, n_in, n_out, outer;
};

template <typename T>
__global__ void __launch_bounds__(256) local_rows_kernel(const T* __restrict__ in,
                                                         T* __restrict__ out, RowMove r,
                                                         MoveArgs a, GroupTab g, int64_t chunks) {
  constexpr int V = 16 / sizeof(T);
  const int64_t per_row = r.L / V;
  const int64_t rows = (int64_t)g.P * r.G * r.outer;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks, chunk = b - row * chunks;
    const int p = (int)(row / (r.G * r.outer));
    int64_t q = row - (int64_t)p * r.G * r.outer;
    const int j = (int)(q / r.outer);
    q -= (int64_t)j * r.outer;
    int64_t so = 0, d0 = (int64_t)p * r.n_out + (int64_t)j * r.dst_j;
    for (int k = r.outer_rank - 1; k >= 0; --k) {
      const int64_t c = q % r.oshape[k];
      q /= r.oshape[k];
      so += c * r.sstr[k];
      d0 += c * r.dstr[k];
    }
    int src;
    if (r.kind == K_CP) {
      src = a.src_of[p];
    } else {
      src = g.members[g.gid[p] * g.gsize + j];
      if (r.kind == K_A2A) so += (int64_t)g.gpos[p] * r.src_pos;
    }
    uint4* d4 = reinterpret_cast<uint4*>(out + d0);
    const int64_t v0 = chunk * (256 * ROW_U) + threadIdx.x;
    if (src < 0) {
#pragma unroll
      for (int u = 0; u < ROW_U; ++u)
        if (v0 + u * 256 < per_row) __stcs(d4 + v0 + u * 256, make_uint4(0, 0, 0, 0));
      continue;
    }
    const uint4* s4 = reinterpret_cast<const uint4*>(in + (int64_t)src * r.n_in + so);
    uint4 v[ROW_U];
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) v[u] = __ldcs(s4 + v0 + u * 256);
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) __stcs(d4 + v0 + u * 256, v[u]);
  }
}

// The all-gather of an f32 3xTF32 GEMM operand written as its tf32 hi / lo
// halves (split_tf32) instead of f32: the GEMM then skips its split pass
// (one HBM read + write of the gathered operand less).
__global__ void __launch_bounds__(256) local_rows_split_kernel(const float* __restrict__ in,
                                                               float* __restrict__ hi,
                                                               float* __restrict__ lo,
                                                               RowMove r, GroupTab g,
                                                               int64_t chunks) {
  const int64_t per_row = r.L / 4;
  const int64_t rows = (int64_t)g.P * r.G * r.outer;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks, chunk = b - row * chunks;
    const int p = (int)(row / (r.G * r.outer));
    int64_t q = row - (int64_t)p * r.G * r.outer;
    const int j = (int)(q / r.outer);
    q -= (int64_t)j * r.outer;
    int64_t so = 0, d0 = (int64_t)p * r.n_out + (int64_t)j * r.dst_j;
    for (int k = r.outer_rank - 1; k >= 0; --k) {
      const int64_t c = q % r.oshape[k];
      q /= r.oshape[k];
      so += c * r.sstr[k];
      d0 += c * r.dstr[k];
    }
    const int src = g.members[g.gid[p] * g.gsize + j];
    const float4* s4 = reinterpret_cast<const float4*>(in + (int64_t)src * r.n_in + so);
    float4* h4 = reinterpret_cast<float4*>(hi + d0);
    float4* l4 = reinterpret_cast<float4*>(lo + d0);
    const int64_t v0 = chunk * (256 * ROW_U) + threadIdx.x;
    float4 v[ROW_U];
#pragma unroll
    for (int u = 0; u < ROW_U; ++u)
      if (v0 + u * 256 < per_row) v[u] = __ldcs(s4 + v0 + u * 256);
#pragma unroll
    for (int u = 0; u < ROW_U; ++u) {
      if (v0 + u * 256 >= per_row) continue;
      float4 h, l;
      split_tf32(v[u].x, h.x, l.x);
      split_tf32(v[u].y, h.y, l.y);
      split_tf32(v[u].z, h.z, l.z);
      split_tf32(v[u].w, h.w, l.w);
      h4[v0 + u * 256] = h;
      l4[v0 + u * 256] = l;
    }
  }
}

// Row form of the move described by `a`, or false when the runs are too
// short / misaligned for it (the element kernel then runs).
static bool row_move(const spmd_tensor& in, const spmd_tensor& out, const MoveArgs& a,
                     int G, RowMove& r) {
  const int es = elem_size(in.dtype);
  const int V = 16 / es;
  memset(&r, 0, sizeof(r));
  r.kind = a.kind;
  r.G = G;
  r.n_in = numel(in);
  r.n_out = numel(out);
  int64_t ist[SPMD_MAX_RANK], ost[SPMD_MAX_RANK];
  int64_t acc = 1;
  for (int k = in.rank - 1; k >= 0; --k) { ist[k] = acc; acc *= in.dims[k]; }
  acc = 1;
  for (int k = out.rank - 1; k >= 0; --k) { ost[k] = acc; acc *= out.dims[k]; }
  int t;   // the run covers dims t.. of the piece
  int64_t piece[SPMD_MAX_RANK];
  for (int k = 0; k < in.rank; ++k) piece[k] = in.dims[k];
  if (a.kind == K_CP) {
    t = 0;
    r.G = 1;
  } else if (a.kind == K_AG) {
    t = a.dim;
    r.dst_j = in.dims[a.dim] * ost[a.dim];
  } else {
    piece[a.split] /= G;
    t = a.split > a.concat ? a.split : a.concat;
    r.src_pos = piece[a.split] * ist[a.split];
    r.dst_j = piece[a.concat] * ost[a.concat];
  }
  if (in.rank == 0) return false;
  r.L = 1;
  for (int k = t; k < in.rank; ++k) r.L *= piece[k];
  r.outer_rank = t;
  r.outer = 1;
  for (int k = 0; k < t; ++k) {
    r.oshape[k] = piece[k];
    r.sstr[k] = ist[k];
    r.dstr[k] = ost[k];
    r.outer *= piece[k];
  }
  return r.L % V == 0 && r.L / V >= 512 && (reinterpret_cast<uintptr_t>(in.data) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(out.data) & 15) == 0;
}

template <typename T>
static int launch_move(const spmd_tensor& in, const spmd_tensor& out, MoveArgs& a, GroupTab& g,
                       cudaStream_t s) {
  int64_t n_out = numel(out), n_in = numel(in);
  if (n_out * g.P == 0) return SPMD_OK;
  RowMove r;
  if (row_move(in, out, a, g.gsize, r)) {
    constexpr int V = 16 / sizeof(T);
    const int64_t chunks = (r.L / V + 256 * ROW_U - 1) / (256 * ROW_U);
    const int64_t rows = (int64_t)g.P * r.G * r.outer;
    local_rows_kernel<T><<<row_grid(rows, chunks), 256, 0, s>>>((const T*)in.data, (T*)out.data,
                                                                r, a, g, chunks);
    return launched(s);
  }
  local_move_kernel<T><<<grid_for(n_out * g.P, 256, 2), 256, 0, s>>>((const T*)in.data,
                                                                     (T*)out.data, a, g, n_out,
                                                                     n_in);
  return launched(s);
}

// Row form of the loopback all-reduce / reduce-scatter: run (p, o) of L
// elements, out = fold over p's group members j (serial, group order -- the
// element kernel's order, so the bits are the same) of in[m_j] at
// o*sstr + gpos[p]*src_pos.
template <typename T>
__global__ void __launch_bounds__(256) local_rows_reduce_kernel(const T* __restrict__ in,
                                                                T* __restrict__ out, RowMove r,
                                                                int kind, GroupTab g,
                                                                int64_t chunks) {
  typedef typename Compute<T>::type C;
  constexpr int V = 16 / sizeof(T);
  const int64_t per_row = r.L / V;
  const int64_t rows = (int64_t)g.P * r.outer;
  for (int64_t b = blockIdx.x; b < rows * chunks; b += gridDim.x) {
    const int64_t row = b / chunks, chunk = b - row * chunks;
    const int p = (int)(row / r.outer);
    int64_t q = row - (int64_t)p * r.outer;
    int64_t so = (int64_t)g.gpos[p] * r.src_pos, d0 = (int64_t)p * r.n_out;
    for (int k = r.outer_rank - 1; k >= 0; --k) {
      const int64_t c = q % r.oshape[k];
      q /= r.oshape[k];
      so += c * r.sstr[k];
      d0 += c * r.dstr[k];
    }
    const int8_t* mem = g.members + g.gid[p] * g.gsize;
    const int64_t v0 = chunk * (256 * ROW_U) + threadIdx.x;
#pragma unroll 1
    for (int u = 0; u < ROW_U; ++u) {
      const int64_t vi = v0 + u * 256;
      if (vi >= per_row) break;
      C acc[V];
      uint4 w = __ldcs(reinterpret_cast<const uint4*>(in + (int64_t)mem[0] * r.n_in + so) + vi);
      const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = ld<T>(e[i]);
      for (int j = 1; j < g.gsize; ++j) {
        w = __ldcs(reinterpret_cast<const uint4*>(in + (int64_t)mem[j] * r.n_in + so) + vi);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = combine<C>(kind, acc[i], ld<T>(e[i]));
      }
      T o[V];
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = st<T>(acc[i]);
      __stcs(reinterpret_cast<uint4*>(out + d0) + vi, *reinterpret_cast<const uint4*>(o));
    }
  }
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_local_all_gather(spmd_tensor in, spmd_tensor out, int dim,
                                     const int32_t* groups, int ngroups, int gsize,
                                     int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && dim >= 0 && dim < in.rank, "all-gather mismatch");
  SPMD_CHECK_ARG(out.dims[dim] == in.dims[dim] * gsize, "all-gather output shape mismatch");
  GroupTab g;
  int rc = make_groups(groups, ngroups, gsize, nparts, g);
  if (rc) return rc;
  MoveArgs a;
  memset(&a, 0, sizeof(a));
  a.kind = K_AG;
  a.in = view_of(in);
  a.out = view_of(out);
  a.dim = dim;
  SPMD_DISPATCH_BYTES(in.dtype, T, return launch_move<T>(in, out, a, g, as_stream(stream)));
  return SPMD_OK;
}

// spmd_local_all_gather of an f32 tensor written as tf32 hi / lo halves (each
// with the gathered shape), for spmd_dot_f32_presplit.  SPMD_ERR_UNSUPPORTED
// when the runs are too short for the row kernel.
extern "C" int spmd_local_all_gather_split(spmd_tensor in, spmd_tensor hi, spmd_tensor lo,
                                           int dim, const int32_t* groups, int ngroups,
                                           int gsize, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == SPMD_F32 && hi.dtype == SPMD_F32 && lo.dtype == SPMD_F32 &&
                     dim >= 0 && dim < in.rank && numel(hi) == numel(lo),
                 "all-gather split expects f32");
  SPMD_CHECK_ARG(hi.dims[dim] == in.dims[dim] * gsize, "all-gather output shape mismatch");
  GroupTab g;
  int rc = make_groups(groups, ngroups, gsize, nparts, g);
  if (rc) return rc;
  MoveArgs a;
  memset(&a, 0, sizeof(a));
  a.kind = K_AG;
  a.in = view_of(in);
  a.out = view_of(hi);
  a.dim = dim;
  RowMove r;
  if (!row_move(in, hi, a, gsize, r) ||
      ((reinterpret_cast<uintptr_t>(hi.data) | reinterpret_cast<uintptr_t>(lo.data)) & 15))
    return SPMD_ERR_UNSUPPORTED;
  if (numel(hi) * nparts == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  const int64_t chunks = (r.L / 4 + 256 * ROW_U - 1) / (256 * ROW_U);
  const int64_t rows = (int64_t)g.P * r.G * r.outer;
  local_rows_split_kernel<<<row_grid(rows, chunks), 256, 0, s>>>(
      (const float*)in.data, (float*)hi.data, (float*)lo.data, r, g, chunks);
  return launched(s);
}

extern "C" int spmd_local_all_to_all(spmd_tensor in, spmd_tensor out, int split_dim,
                                     int concat_dim, const int32_t* groups, int ngroups,
                                     int gsize, int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype, "all-to-all dtype mismatch");
  SPMD_CHECK_ARG(in.dims[split_dim] % gsize == 0, "all-to-all split dim not divisible");
  GroupTab g;
  int rc = make_groups(groups, ngroups, gsize, nparts, g);
  if (rc) return rc;
  MoveArgs a;
  memset(&a, 0, sizeof(a));
  a.kind = K_A2A;
  a.in = view_of(in);
  a.out = view_of(out);
  a.piece = a.in;
  a.piece.d[split_dim] /= gsize;
  a.split = split_dim;
  a.concat = concat_dim;
  SPMD_DISPATCH_BYTES(in.dtype, T, return launch_move<T>(in, out, a, g, as_stream(stream)));
  return SPMD_OK;
}

extern "C" int spmd_local_collective_permute(spmd_tensor in, spmd_tensor out,
                                             const int32_t* pairs, int npairs, int64_t nparts,
                                             void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && numel(in) == numel(out), "permute mismatch");
  SPMD_CHECK_ARG(nparts <= SPMD_MAX_PARTS, "too many partitions");
  MoveArgs a;
  memset(&a, 0, sizeof(a));
  memset(a.src_of, -1, sizeof(a.src_of));
  bool src_seen[SPMD_MAX_PARTS] = {false};
  for (int i = 0; i < npairs; ++i) {
    int sdev = pairs[2 * i], tdev = pairs[2 * i + 1];
    if (sdev < 0 || sdev >= nparts || tdev < 0 || tdev >= nparts || a.src_of[tdev] != -1 ||
        src_seen[sdev]) {
      set_error("collective-permute pairs must have distinct sources and distinct targets");
      return SPMD_ERR_SUBGROUP;
    }
    a.src_of[tdev] = (int8_t)sdev;
    src_seen[sdev] = true;
  }
  a.kind = K_CP;
  a.in = view_of(in);
  a.out = view_of(out);
  GroupTab g;
  memset(&g, 0, sizeof(g));
  g.P = (int)nparts;
  g.gsize = 1;
  SPMD_DISPATCH_BYTES(in.dtype, T, return launch_move<T>(in, out, a, g, as_stream(stream)));
  return SPMD_OK;
}

static int local_reduce(spmd_tensor in, spmd_tensor out, int dim, int scatter, int kind,
                        const int32_t* groups, int ngroups, int gsize, int64_t nparts,
                        void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype, "reduction dtype mismatch");
  SPMD_CHECK_ARG(kind >= 0 && kind <= 3, "bad reduce kind");
  GroupTab g;
  int rc = make_groups(groups, ngroups, gsize, nparts, g);
  if (rc) return rc;
  int64_t n_out = numel(out), n_in = numel(in);
  if (n_out * nparts == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  View vin = view_of(in), vout = view_of(out);
  // row form: runs of L contiguous elements (all of it for an all-reduce;
  // the scattered piece of dims dim.. for a reduce-scatter)
  RowMove r;
  memset(&r, 0, sizeof(r));
  r.n_in = n_in;
  r.n_out = n_out;
  r.G = 1;
  const int t = scatter ? dim : 0;
  int64_t ist = 1, ost = 1;
  r.L = 1;
  for (int k = out.rank - 1; k >= t; --k) r.L *= out.dims[k];
  for (int k = in.rank - 1; k >= 0; --k) {
    if (k < t) {
      r.oshape[k] = out.dims[k];
      r.sstr[k] = ist;
      r.dstr[k] = ost;
    }
    ist *= in.dims[k];
    ost *= out.dims[k];
  }
  r.outer_rank = t;
  r.outer = 1;
  for (int k = 0; k < t; ++k) r.outer *= out.dims[k];
  r.src_pos = scatter ? r.L : 0;
  const int V = 16 / elem_size(in.dtype);
  const bool rows_ok = r.L % V == 0 && r.L / V >= 512 &&
                       ((reinterpret_cast<uintptr_t>(in.data) |
                         reinterpret_cast<uintptr_t>(out.data)) & 15) == 0;
  if (rows_ok) {
    const int64_t chunks = (r.L / V + 256 * ROW_U - 1) / (256 * ROW_U);
    const int64_t rows = nparts * r.outer;
    SPMD_DISPATCH(in.dtype, T,
                  local_rows_reduce_kernel<T><<<row_grid(rows, chunks), 256, 0, s>>>(
                      (const T*)in.data, (T*)out.data, r, kind, g, chunks));
    return launched(s);
  }
  SPMD_DISPATCH(in.dtype, T,
                local_reduce_kernel<T><<<grid_for(n_out * nparts, 256, 2), 256, 0, s>>>(
                    (const T*)in.data, (T*)out.data, vin, vout, dim, scatter, kind, g, n_out,
                    n_in));
  return launched(s);
}

extern "C" int spmd_local_all_reduce(spmd_tensor in, spmd_tensor out, int kind,
                                     const int32_t* groups, int ngroups, int gsize,
                                     int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(numel(in) == numel(out), "all-reduce shape mismatch");
  return local_reduce(in, out, 0, 0, kind, groups, ngroups, gsize, nparts, stream);
}

extern "C" int spmd_local_reduce_scatter(spmd_tensor in, spmd_tensor out, int dim, int kind,
                                         const int32_t* groups, int ngroups, int gsize,
                                         int64_t nparts, void* stream) {
  SPMD_CHECK_ARG(dim >= 0 && dim < in.rank && in.dims[dim] == out.dims[dim] * gsize,
                 "reduce-scatter shape mismatch");
  return local_reduce(in, out, dim, 1, kind, groups, ngroups, gsize, nparts, stream);
}
