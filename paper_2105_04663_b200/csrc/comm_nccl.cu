// NCCL collectives for one-process-per-GPU execution over NVLink/NVSwitch
// (replaces reference simulator.py:333-390 across real devices).
//
// * Subgroups: one communicator per distinct subgroup partition, created with
//   ncclCommSplit(color = group index, key = position in the group) so that
//   NCCL rank order == the emitted group order (all-gather / reduce-scatter /
//   all-to-all piece order follows it).  Cached by the flattened group table.
// * Non-leading-dim all-gather / reduce-scatter / all-to-all pack or unpack
//   through the caller's workspace with the affine copy kernel; leading-dim
//   (outer extent 1) collectives run in place with no extra HBM pass.
// * collective-permute: grouped ncclSend/ncclRecv on the world communicator;
//   devices that are not a target receive zeros (reference :345-350).
// Reductions run in NCCL's order, so float results match the reference
// within tolerance (integers exactly).
#include "comm.cuh"

#include <string.h>

namespace spmd {

static bool nccl_type(int dtype, ncclDataType_t* t) {
  switch (dtype) {
    case SPMD_F32: *t = ncclFloat32; return true;
    case SPMD_S32: *t = ncclInt32; return true;
    case SPMD_U32: *t = ncclUint32; return true;
    case SPMD_PRED: *t = ncclUint8; return true;
    case SPMD_BF16: *t = ncclBfloat16; return true;
  }
  return false;
}

static ncclRedOp_t nccl_op(int kind) {
  switch (kind) {
    case SPMD_SUM: return ncclSum;
    case SPMD_MAX: return ncclMax;
    case SPMD_MIN: return ncclMin;
    default: return ncclProd;
  }
}

int group_position(const spmd_comm* c, const int32_t* groups, int ngroups, int gsize, int* group,
                   int* pos) {
  if (ngroups * gsize != c->nranks) {
    set_error("subgroups do not partition the ranks");
    return SPMD_ERR_SUBGROUP;
  }
  std::vector<int> seen(c->nranks, 0);
  *group = *pos = -1;
  for (int i = 0; i < ngroups * gsize; ++i) {
    if (groups[i] < 0 || groups[i] >= c->nranks || seen[groups[i]]++) {
      set_error("subgroups do not partition the ranks");
      return SPMD_ERR_SUBGROUP;
    }
    if (groups[i] == c->rank) {
      *group = i / gsize;
      *pos = i % gsize;
    }
  }
  return SPMD_OK;
}

// Sub-communicator for a subgroup partition; *pos = my position in my group.
static int subcomm(spmd_comm* c, const int32_t* groups, int ngroups, int gsize, ncclComm_t* out,
                   int* pos) {
  if (ngroups * gsize != c->nranks) {
    set_error("subgroups do not partition the ranks");
    return SPMD_ERR_SUBGROUP;
  }
  // Key = (group size, flattened groups): ((0,2),(1,3)) and ((0,2,1,3),)
  // flatten identically but are different partitions.
  std::vector<int32_t> key(1, gsize);
  key.insert(key.end(), groups, groups + ngroups * gsize);
  int color = -1, k = -1;
  std::vector<int> seen(c->nranks, 0);
  for (int i = 0; i < ngroups * gsize; ++i) {
    if (groups[i] < 0 || groups[i] >= c->nranks || seen[groups[i]]++) {
      set_error("subgroups do not partition the ranks");
      return SPMD_ERR_SUBGROUP;
    }
    if (groups[i] == c->rank) {
      color = i / gsize;
      k = i % gsize;
    }
  }
  *pos = k;
  bool identity = ngroups == 1;
  for (int i = 0; identity && i < gsize; ++i) identity = groups[i] == i;
  if (identity) {
    *out = c->world;
    return SPMD_OK;
  }
  auto it = c->splits.find(key);
  if (it != c->splits.end()) {
    *out = it->second;
    return SPMD_OK;
  }
  ncclComm_t nc;
  NCCL_TRY(ncclCommSplit(c->world, color, k, &nc, nullptr));
  c->splits[key] = nc;
  *out = nc;
  return SPMD_OK;
}

static void split3(const spmd_tensor& t, int dim, int64_t* outer, int64_t* mid, int64_t* inner) {
  *outer = *inner = 1;
  for (int i = 0; i < dim; ++i) *outer *= t.dims[i];
  for (int i = dim + 1; i < t.rank; ++i) *inner *= t.dims[i];
  *mid = t.dims[dim];
}

// dst[o][j][i][in] <-> src[j][o][i][in] style 4-D block moves.
static int block_move(const void* src, void* dst, int dtype, int64_t G, int64_t outer,
                      int64_t mid, int64_t inner, bool to_grouped, cudaStream_t s) {
  CopyArgs a;
  memset(&a, 0, sizeof(a));
  a.rank = 4;
  a.shape[0] = G;
  a.shape[1] = outer;
  a.shape[2] = mid;
  a.shape[3] = inner;
  // grouped layout [G][outer][mid][inner]; interleaved layout [outer][G*mid][inner]
  int64_t g_st[4] = {outer * mid * inner, mid * inner, inner, 1};
  int64_t i_st[4] = {mid * inner, G * mid * inner, inner, 1};
  for (int k = 0; k < 4; ++k) {
    a.sst[k] = to_grouped ? i_st[k] : g_st[k];
    a.dst[k] = to_grouped ? g_st[k] : i_st[k];
  }
  a.spart = a.dpart = 0;
  return launch_copy(src, dst, dtype, a, 1, s);
}

static int need_ws(spmd_comm* c, int64_t bytes) {
  if (c->ws_bytes < bytes) {
    set_error("collective workspace too small (spmd_comm_set_workspace)");
    return SPMD_ERR_INVALID;
  }
  return SPMD_OK;
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_comm_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

extern "C" int spmd_comm_get_unique_id(void* id_out) {
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return SPMD_OK;
}

extern "C" int spmd_comm_init(spmd_comm** comm, int nranks, int rank, const void* unique_id) {
  spmd_comm* c = new spmd_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  // Optional CTA cap so NCCL kernels fit beside persistent GEMMs
  // (SPMD_NCCL_MAX_CTAS; sub-communicators inherit the config).
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  const int max_ctas = (int)option(OPT_NCCL_MAX_CTAS);
  if (max_ctas > 0) {
    cfg.maxCTAs = max_ctas;
    cfg.minCTAs = cfg.maxCTAs < 4 ? cfg.maxCTAs : 4;
  }
  ncclResult_t r = ncclCommInitRankConfig(&c->world, nranks, id, rank, &cfg);
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    delete c;
    return SPMD_ERR_NCCL;
  }
  *comm = c;
  return SPMD_OK;
}

extern "C" int spmd_comm_destroy(spmd_comm* c) {
  if (!c) return SPMD_OK;
  for (auto& row : c->fork)
    for (auto& st : row)
      if (st) cudaStreamDestroy(st);
  for (auto& row : c->fork_ev)
    for (auto& ev : row)
      if (ev) cudaEventDestroy(ev);
  for (auto& kv : c->splits) ncclCommDestroy(kv.second);
  ncclCommDestroy(c->world);
  delete c;
  return SPMD_OK;
}

extern "C" int spmd_comm_set_workspace(spmd_comm* c, void* ptr, int64_t bytes) {
  c->ws = (char*)ptr;
  c->ws_bytes = bytes;
  return SPMD_OK;
}

extern "C" int spmd_all_gather(spmd_comm* c, spmd_tensor in, spmd_tensor out, int dim,
                               const int32_t* groups, int ngroups, int gsize, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && dim >= 0 && dim < in.rank &&
                     out.dims[dim] == in.dims[dim] * gsize,
                 "all-gather shape mismatch");
  ncclComm_t nc;
  int pos;
  int rc = subcomm(c, groups, ngroups, gsize, &nc, &pos);
  if (rc) return rc;
  ncclDataType_t t;
  nccl_type(in.dtype, &t);
  cudaStream_t s = as_stream(stream);
  int64_t outer, mid, inner;
  split3(in, dim, &outer, &mid, &inner);
  int64_t n = numel(in);
  if (outer == 1) {
    NCCL_TRY(ncclAllGather(in.data, out.data, (size_t)n, t, nc, s));
    return SPMD_OK;
  }
  int64_t bytes = n * gsize * elem_size(in.dtype);
  if ((rc = need_ws(c, bytes))) return rc;
  NCCL_TRY(ncclAllGather(in.data, c->ws, (size_t)n, t, nc, s));
  return block_move(c->ws, out.data, in.dtype, gsize, outer, mid, inner, false, s);
}

extern "C" int spmd_all_reduce(spmd_comm* c, spmd_tensor in, spmd_tensor out, int kind,
                               const int32_t* groups, int ngroups, int gsize, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && numel(in) == numel(out), "all-reduce mismatch");
  ncclComm_t nc;
  int pos;
  int rc = subcomm(c, groups, ngroups, gsize, &nc, &pos);
  if (rc) return rc;
  ncclDataType_t t;
  nccl_type(in.dtype, &t);
  NCCL_TRY(ncclAllReduce(in.data, out.data, (size_t)numel(in), t, nccl_op(kind), nc,
                         as_stream(stream)));
  return SPMD_OK;
}

extern "C" int spmd_reduce_scatter(spmd_comm* c, spmd_tensor in, spmd_tensor out, int dim,
                                   int kind, const int32_t* groups, int ngroups, int gsize,
                                   void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && dim >= 0 && dim < in.rank &&
                     in.dims[dim] == out.dims[dim] * gsize,
                 "reduce-scatter shape mismatch");
  ncclComm_t nc;
  int pos;
  int rc = subcomm(c, groups, ngroups, gsize, &nc, &pos);
  if (rc) return rc;
  ncclDataType_t t;
  nccl_type(in.dtype, &t);
  cudaStream_t s = as_stream(stream);
  int64_t outer, mid, inner;
  split3(out, dim, &outer, &mid, &inner);
  int64_t n = numel(out);
  if (outer == 1) {
    NCCL_TRY(ncclReduceScatter(in.data, out.data, (size_t)n, t, nccl_op(kind), nc, s));
    return SPMD_OK;
  }
  if ((rc = need_ws(c, numel(in) * elem_size(in.dtype)))) return rc;
  rc = block_move(in.data, c->ws, in.dtype, gsize, outer, mid, inner, true, s);
  if (rc) return rc;
  NCCL_TRY(ncclReduceScatter(c->ws, out.data, (size_t)n, t, nccl_op(kind), nc, s));
  return SPMD_OK;
}

extern "C" int spmd_all_to_all(spmd_comm* c, spmd_tensor in, spmd_tensor out, int split_dim,
                               int concat_dim, const int32_t* groups, int ngroups, int gsize,
                               void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && in.dims[split_dim] % gsize == 0,
                 "all-to-all shape mismatch");
  ncclComm_t nc;
  int pos;
  int rc = subcomm(c, groups, ngroups, gsize, &nc, &pos);
  if (rc) return rc;
  ncclDataType_t t;
  nccl_type(in.dtype, &t);
  cudaStream_t s = as_stream(stream);
  const int64_t n = numel(in), piece = n / gsize, es = elem_size(in.dtype);
  // send layout: [G][piece] with piece j = slice j along split_dim.
  int64_t so, sm, si;
  split3(in, split_dim, &so, &sm, &si);
  const bool send_direct = so == 1;
  // recv layout: [G][piece'] where out = concat_j recv[j] along concat_dim.
  spmd_tensor pshape = in;
  pshape.dims[split_dim] /= gsize;
  int64_t co, cm, ci;
  split3(pshape, concat_dim, &co, &cm, &ci);
  const bool recv_direct = co == 1;
  int64_t need = (send_direct ? 0 : n) + (recv_direct ? 0 : n);
  if ((rc = need_ws(c, need * es))) return rc;
  const void* sendbuf = in.data;
  char* ws = c->ws;
  if (!send_direct) {
    rc = block_move(in.data, ws, in.dtype, gsize, so, sm / gsize, si, true, s);
    if (rc) return rc;
    sendbuf = ws;
    ws += n * es;
  }
  void* recvbuf = recv_direct ? out.data : (void*)ws;
  NCCL_TRY(ncclAlltoAll(sendbuf, recvbuf, (size_t)piece, t, nc, s));
  if (!recv_direct) return block_move(recvbuf, out.data, in.dtype, gsize, co, cm, ci, false, s);
  return SPMD_OK;
}

extern "C" int spmd_collective_permute(spmd_comm* c, spmd_tensor in, spmd_tensor out,
                                       const int32_t* pairs, int npairs, void* stream) {
  SPMD_CHECK_ARG(in.dtype == out.dtype && numel(in) == numel(out), "permute mismatch");
  cudaStream_t s = as_stream(stream);
  int send_to = -1, recv_from = -1;
  std::vector<int> src_seen(c->nranks, 0), dst_seen(c->nranks, 0);
  for (int i = 0; i < npairs; ++i) {
    int a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a < 0 || b < 0 || a >= c->nranks || b >= c->nranks || src_seen[a]++ || dst_seen[b]++) {
      set_error("collective-permute pairs must have distinct sources and distinct targets");
      return SPMD_ERR_SUBGROUP;
    }
    if (a == c->rank) send_to = b;
    if (b == c->rank) recv_from = a;
  }
  ncclDataType_t t;
  nccl_type(in.dtype, &t);
  const size_t n = (size_t)numel(in);
  const size_t bytes = n * elem_size(in.dtype);
  if (recv_from < 0) SPMD_CUDA_TRY(cudaMemsetAsync(out.data, 0, bytes, s));
  if (send_to == c->rank && recv_from == c->rank) {
    if (out.data != in.data)
      SPMD_CUDA_TRY(cudaMemcpyAsync(out.data, in.data, bytes, cudaMemcpyDeviceToDevice, s));
    return SPMD_OK;
  }
  NCCL_TRY(ncclGroupStart());
  if (send_to >= 0 && send_to != c->rank) NCCL_TRY(ncclSend(in.data, n, t, send_to, c->world, s));
  if (recv_from >= 0 && recv_from != c->rank)
    NCCL_TRY(ncclRecv(out.data, n, t, recv_from, c->world, s));
  NCCL_TRY(ncclGroupEnd());
  if (send_to == c->rank)   // self pair with a foreign receive cannot happen (distinct targets)
    SPMD_CUDA_TRY(cudaMemcpyAsync(out.data, in.data, bytes, cudaMemcpyDeviceToDevice, s));
  return SPMD_OK;
}
