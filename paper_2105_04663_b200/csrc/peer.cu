// Peer-memory fused Dot -> reduce-scatter over NVLink / NVSwitch.
//
// The partitioner emits Dot followed by ReduceScatter whenever the dot's
// contracting dim is sharded and an output dim takes the reduced sharding
// (reference partitioner.py:751-759; C2's out-projection and FFN-out).  The
// unfused path writes the full partial product to HBM and then runs an NCCL
// reduce-scatter that cannot start before the last GEMM tile.  Here the GEMM
// epilogue itself stores every output tile into the heap of the rank that
// owns its column chunk (P2P stores through the CUDA-IPC mapping), so the
// transfer overlaps the math tile by tile; a one-block barrier and an
// HBM-bound slot reduction finish the collective.
//
// Heap (per rank, same size everywhere, opened by every other rank):
//   control page: per barrier channel c (one per issuing stream, so ranks
//                 agree on the order of barriers within a channel): u32 epoch
//                 at [256c]; u32 flag[q] at [256c + 64 + q] = last epoch that
//                 rank q has completed (written remotely by q)
//   data:         [0, 3H): the fused-op landing zone (H = fused_half,
//                 spmd_comm_reserve_fused): parity p of an op whose unit
//                 (slot / row) is u bytes starts at unit p * ceil(H / u), so
//                 parity 0 of every op lies in [0, H) and parity 1 in
//                 [H, 3H) -- consecutive fused ops of different sizes never
//                 overlap across parities;
//                 caller-assigned offsets >= 3H: all-gather staging slots,
//                 collective-permute landing slots.
// Epochs live in device memory, so the sequence is CUDA-graph replay safe:
// the GEMM reads parity (epoch + 1) & 1, the barrier kernel increments the
// epoch, publishes it to every rank and waits for every rank's flag.  Waiting
// on ALL ranks (not only the group) keeps the parity buffers safe when
// consecutive fused ops use different subgroups: rank q can only write
// parity p again after this rank has passed the barrier of the op in between,
// which follows this rank's reduction of parity p in stream order.
#include "comm.cuh"

#include <string.h>

namespace spmd {

constexpr int64_t CTRL_BYTES = 4096;
constexpr int CHANNEL_WORDS = 256;    // per barrier channel: epoch, pad, flags[64 + q]
constexpr int NUM_CHANNELS = 4;
constexpr int FLAG0 = 64;
constexpr int ERR_PEER_TIMEOUT = 2;   // device error word bit

struct PeerFlags {
  uint32_t* remote[SPMD_MAX_PARTS];   // &flag[rank] in rank q's control page
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One block: bump the epoch, publish it to every rank, wait for every rank.
__global__ void peer_barrier_kernel(uint32_t* ctrl, PeerFlags pf, int nranks, int rank,
                                    long long timeout_cycles, int* err) {
  __shared__ uint32_t e;
  if (threadIdx.x == 0) {
    e = ctrl[0] + 1;
    ctrl[0] = e;
    __threadfence_system();
  }
  __syncthreads();
  const uint32_t ep = e;
  for (int q = threadIdx.x; q < nranks; q += blockDim.x)
    if (q != rank) st_release_sys(pf.remote[q], ep);
  for (int q = threadIdx.x; q < nranks; q += blockDim.x) {
    if (q == rank) continue;
    const long long t0 = clock64();
    while ((int32_t)(ld_acquire_sys(&ctrl[FLAG0 + q]) - ep) < 0) {
      if (clock64() - t0 > timeout_cycles) {
        atomicOr(err, ERR_PEER_TIMEOUT);
        break;
      }
      __nanosleep(64);
    }
  }
}

// out[i] = sum_j slot_j[i] (fp32 accumulation in group-position order).
__global__ void peer_slot_reduce_kernel(const bf16* __restrict__ data, bf16* __restrict__ out,
                                        const uint32_t* ctrl, int G, int64_t slot,
                                        int64_t par_slots, int64_t nvec,
                                        const bf16* __restrict__ resid) {
  const int64_t par = (int64_t)(*(volatile const uint32_t*)ctrl & 1);
  const bf16* base = data + par * par_slots * slot;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < G; ++j) {
      uint4 w = __ldcs(reinterpret_cast<const uint4*>(base + j * slot) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(h[q]);
        acc[2 * q] += f.x;
        acc[2 * q + 1] += f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) oh[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
    if (resid) {
      // the layer's residual Add, with the unfused path's roundings (the
      // reduce-scatter result in bf16, then the Add in f32 and one rounding)
      const uint4 rw = __ldcs(reinterpret_cast<const uint4*>(resid) + i);
      const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rw);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 a = __bfloat1622float2(oh[q]), b = __bfloat1622float2(rh[q]);
        oh[q] = __floats2bfloat162_rn(a.x + b.x, a.y + b.y);
      }
    }
    reinterpret_cast<uint4*>(out)[i] = o;
  }
}

static long long timeout_cycles();

// Barrier on channel `ch` (stream-ordered, one block).
static int peer_barrier(spmd_comm* c, int ch, cudaStream_t s) {
  PeerFlags pf;
  memset(&pf, 0, sizeof(pf));
  for (int q = 0; q < c->nranks; ++q)
    pf.remote[q] = (uint32_t*)c->peer[q] + ch * CHANNEL_WORDS + FLAG0 + c->rank;
  int* err = device_error_word();
  if (!err) return SPMD_ERR_CUDA;
  peer_barrier_kernel<<<1, 64, 0, s>>>((uint32_t*)c->heap + ch * CHANNEL_WORDS, pf, c->nranks,
                                       c->rank, timeout_cycles(), err);
  return launched(s);
}

// SM pull engine of the all-gather: dst[r][j][v] = src_j[r][v] in 16-byte
// vectors, 4 independent NVLink loads in flight per thread.
struct PullArgs {
  const uint4* src[8];
  int G;
  int64_t outer, w16;   // rows of my piece, 16-byte vectors per row
};

__global__ void __launch_bounds__(512) peer_pull_kernel(PullArgs a, uint4* __restrict__ dst) {
  const int64_t per = a.outer * a.w16;
  const int64_t total = per * a.G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < total;
       base += 4 * stride) {
    uint4 v[4];
    int64_t d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t idx = base + u * stride;
      d[u] = -1;
      if (idx < total) {
        const int j = (int)(idx / per);
        const int64_t rv = idx - j * per;
        const int64_t r = rv / a.w16, c = rv - r * a.w16;
        v[u] = __ldcs(a.src[j] + rv);
        d[u] = (r * a.G + j) * a.w16 + c;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (d[u] >= 0) __stcs(dst + d[u], v[u]);
  }
}

// out[i] = parity buffer (epoch & 1) of the all-to-all landing zone.
__global__ void peer_parity_copy_kernel(const uint4* __restrict__ data, uint4* __restrict__ out,
                                        const uint32_t* ctrl, int64_t par16, int64_t n16) {
  const int64_t par = (int64_t)(*(volatile const uint32_t*)ctrl & 1);
  const uint4* src = data + par * par16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldcs(src + i);
}

static void close_peers(spmd_comm* c) {
  for (int q = 0; q < c->nranks; ++q)
    if (q != c->rank && c->peer[q]) cudaIpcCloseMemHandle(c->peer[q]);
  if (c->heap) cudaFree(c->heap);
  memset(c->peer, 0, sizeof(c->peer));
  c->heap = nullptr;
  c->heap_bytes = 0;
}

// Units per parity of a fused op that lands `units` units of `unit_bytes`
// per parity: ceil(H / unit).  Fails when the reserved region is too small.
static int fused_parity(const spmd_comm* c, int64_t unit_bytes, int64_t units,
                        int64_t* par_units) {
  const int64_t h = c->fused_half;
  if (h <= 0 || unit_bytes <= 0 || units * unit_bytes > h || 3 * h > c->heap_bytes) {
    set_error("peer heap fused region too small for this op (spmd_comm_reserve_fused)");
    return SPMD_ERR_INVALID;
  }
  *par_units = (h + unit_bytes - 1) / unit_bytes;
  return SPMD_OK;
}

static int check_slot(const spmd_comm* c, int64_t off, int64_t bytes, const char* what) {
  if (off < 3 * c->fused_half || off % 256 != 0 || off + bytes > c->heap_bytes) {
    set_error(std::string(what) + ": slot outside the heap or inside the fused region");
    return SPMD_ERR_INVALID;
  }
  return SPMD_OK;
}

static long long timeout_cycles() {
  return (long long)option(OPT_PEER_TIMEOUT_MS) * 2000000LL;   // clock64 at <= 2 GHz
}

}  // namespace spmd

using namespace spmd;

extern "C" int spmd_comm_enable_peer(spmd_comm* c, int64_t bytes, void* stream) {
  SPMD_CHECK_ARG(c && bytes >= 0, "enable_peer arguments");
  SPMD_CHECK_ARG(c->nranks <= SPMD_MAX_PARTS && c->nranks <= CHANNEL_WORDS - FLAG0,
                 "too many ranks for the peer heap");
  if (c->heap && c->heap_bytes >= bytes) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  // Collective: every rank reallocates and re-exchanges together.
  SPMD_CUDA_TRY(cudaDeviceSynchronize());
  close_peers(c);
  bytes = (bytes + 4095) & ~(int64_t)4095;
  SPMD_CUDA_TRY(cudaMalloc(&c->heap, CTRL_BYTES + bytes));
  SPMD_CUDA_TRY(cudaMemset(c->heap, 0, CTRL_BYTES));
  cudaIpcMemHandle_t h;
  SPMD_CUDA_TRY(cudaIpcGetMemHandle(&h, c->heap));
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* dev = nullptr;
  SPMD_CUDA_TRY(cudaMalloc(&dev, hb * c->nranks));
  SPMD_CUDA_TRY(cudaMemcpy(dev + hb * c->rank, &h, hb, cudaMemcpyHostToDevice));
  ncclResult_t r = ncclAllGather(dev + hb * c->rank, dev, hb, ncclUint8, c->world, s);
  if (r != ncclSuccess) {
    cudaFree(dev);
    set_error(std::string("peer handle exchange: ") + ncclGetErrorString(r));
    return SPMD_ERR_NCCL;
  }
  std::vector<cudaIpcMemHandle_t> all(c->nranks);
  SPMD_CUDA_TRY(cudaStreamSynchronize(s));
  SPMD_CUDA_TRY(cudaMemcpy(all.data(), dev, hb * c->nranks, cudaMemcpyDeviceToHost));
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->peer[q] = c->heap;
      continue;
    }
    void* p = nullptr;
    SPMD_CUDA_TRY(cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess));
    c->peer[q] = (char*)p;
  }
  c->heap_bytes = bytes;
  // Everyone has mapped everyone before the first remote store.
  r = ncclAllReduce(dev, dev, 1, ncclUint8, ncclSum, c->world, s);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(dev);
  if (r != ncclSuccess) {
    set_error(std::string("peer barrier: ") + ncclGetErrorString(r));
    return SPMD_ERR_NCCL;
  }
  SPMD_CUDA_TRY(e);
  return SPMD_OK;
}

extern "C" int64_t spmd_comm_peer_bytes(spmd_comm* c) { return c ? c->heap_bytes : 0; }

extern "C" int spmd_comm_reserve_fused(spmd_comm* c, int64_t half_bytes) {
  SPMD_CHECK_ARG(c && half_bytes >= 0, "reserve_fused arguments");
  half_bytes = (half_bytes + 4095) & ~(int64_t)4095;
  if (half_bytes > c->fused_half) c->fused_half = half_bytes;
  return SPMD_OK;
}

extern "C" int64_t spmd_comm_fused_half(spmd_comm* c) { return c ? c->fused_half : 0; }

static int dot_reduce_scatter(spmd_comm* c, spmd_tensor lhs, spmd_tensor rhs,
                              const bf16* resid, spmd_tensor out, const spmd_dot_dims* dd,
                              int dim, const int32_t* groups, int ngroups, int gsize,
                              void* stream) {
  SPMD_CHECK_ARG(c && dd, "dot_reduce_scatter arguments");
  SPMD_CHECK_ARG(lhs.dtype == SPMD_BF16 && rhs.dtype == SPMD_BF16 && out.dtype == SPMD_BF16,
                 "dot_reduce_scatter is bf16");
  SPMD_CHECK_ARG(out.rank >= 1 && (dim == out.rank - 1 || (dim == 0 && out.rank >= 2)),
                 "dot_reduce_scatter scatters the last dim or the leading (row) dim");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int grp, pos;
  int rc = group_position(c, groups, ngroups, gsize, &grp, &pos);
  if (rc) return rc;
  SPMD_CHECK_ARG(gsize <= 8, "dot_reduce_scatter group size <= 8");
  const int64_t slot = numel(out);
  int64_t par_slots = 0;
  if ((rc = fused_parity(c, slot * 2, gsize, &par_slots))) return rc;
  SPMD_CHECK_ARG(slot % 8 == 0, "dot_reduce_scatter shard must be a multiple of 8 elements");
  cudaStream_t s = as_stream(stream);
  spmd_tensor full = out;
  full.dims[dim] *= gsize;
  full.data = nullptr;
  GemmScatter sc;
  memset(&sc, 0, sizeof(sc));
  sc.gsize = gsize;
  sc.pos = pos;
  for (int j = 0; j < gsize; ++j) sc.dst[j] = c->peer[groups[grp * gsize + j]] + CTRL_BYTES;
  sc.epoch = (const uint32_t*)c->heap;
  sc.par_slots = (int)par_slots;
  if (dim == 0 && out.rank >= 2 && dim != out.rank - 1) {
    // split on the leading output dim = GEMM rows (no batch dims): member j
    // gets rows [j * R/G, (j+1) * R/G) into slot `pos` (wide kernel)
    sc.rows = 1;
    sc.rchunk = 0;   // M / gsize
    sc.slot_base = pos;
    sc.nslots = gsize;
  }
  rc = dot_tcgen05(lhs, rhs, full, *dd, 1, s, &sc);
  if (rc) return rc;
  if ((rc = peer_barrier(c, 0, s))) return rc;
  const int64_t nvec = slot / 8;
  peer_slot_reduce_kernel<<<grid_for(nvec, 256), 256, 0, s>>>(
      (const bf16*)(c->heap + CTRL_BYTES), (bf16*)out.data, (const uint32_t*)c->heap, gsize, slot,
      par_slots, nvec, resid);
  return launched(s);
}

extern "C" int spmd_dot_reduce_scatter(spmd_comm* c, spmd_tensor lhs, spmd_tensor rhs,
                                       spmd_tensor out, const spmd_dot_dims* dd, int dim,
                                       const int32_t* groups, int ngroups, int gsize,
                                       void* stream) {
  return dot_reduce_scatter(c, lhs, rhs, nullptr, out, dd, dim, groups, ngroups, gsize, stream);
}

// The same with the layer's residual Add folded into the slot reduce:
// out = reduce_scatter(dot) + resid (resid has out's shape), rounded exactly
// as the unfused reduce-scatter followed by the Add.
extern "C" int spmd_dot_reduce_scatter_add(spmd_comm* c, spmd_tensor lhs, spmd_tensor rhs,
                                           spmd_tensor resid, spmd_tensor out,
                                           const spmd_dot_dims* dd, int dim,
                                           const int32_t* groups, int ngroups, int gsize,
                                           void* stream) {
  SPMD_CHECK_ARG(resid.dtype == SPMD_BF16 && numel(resid) == numel(out) &&
                     (reinterpret_cast<uintptr_t>(resid.data) & 15) == 0,
                 "dot_reduce_scatter_add residual");
  return dot_reduce_scatter(c, lhs, rhs, (const bf16*)resid.data, out, dd, dim, groups, ngroups,
                            gsize, stream);
}

// All-gather through the peer heap: stage my shard at `heap_offset`, barrier,
// pull every group member's staged shard with copy-engine 2-D copies (no SMs
// taken from concurrently running GEMMs), barrier (so the staging slot may be
// rewritten by the next call).  Piece order = group order (reference
// simulator.py:353-359).
extern "C" int spmd_peer_all_gather(spmd_comm* c, spmd_tensor in, spmd_tensor out, int dim,
                                    const int32_t* groups, int ngroups, int gsize,
                                    int64_t heap_offset, int channel, int engine, void* stream) {
  SPMD_CHECK_ARG(c && in.dtype == out.dtype && dim >= 0 && dim < in.rank &&
                     out.dims[dim] == in.dims[dim] * gsize,
                 "peer all-gather shape mismatch");
  SPMD_CHECK_ARG(channel >= 0 && channel < NUM_CHANNELS, "peer barrier channel");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int grp, pos;
  int rc = group_position(c, groups, ngroups, gsize, &grp, &pos);
  if (rc) return rc;
  const int64_t es = elem_size(in.dtype);
  const int64_t bytes = numel(in) * es;
  if ((rc = check_slot(c, heap_offset, bytes, "peer all-gather staging"))) return rc;
  if (bytes == 0) return SPMD_OK;
  cudaStream_t s = as_stream(stream);
  int64_t outer = 1;
  for (int i = 0; i < dim; ++i) outer *= in.dims[i];
  const int64_t w = bytes / outer;   // one contiguous run of my piece
  const bool staged = engine == 4;   // pieces staged + barrier passed by the caller
  if (!staged) {
    SPMD_CUDA_TRY(cudaMemcpyAsync(c->heap + CTRL_BYTES + heap_offset, in.data, bytes,
                                  cudaMemcpyDeviceToDevice, s));
    if ((rc = peer_barrier(c, channel, s))) return rc;
  }
  // engine 1: SM pull over the whole GPU (critical path); 3: background SM
  // pull, 32 CTAs that co-reside beside a persistent GEMM (like NCCL's)
  const bool sm = (engine == 1 || engine == 3) && gsize <= 8 && w % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(in.data) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(out.data) & 15) == 0;
  if (sm) {
    PullArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.G = gsize;
    pa.outer = outer;
    pa.w16 = w / 16;
    for (int j = 0; j < gsize; ++j) {
      const int q = groups[grp * gsize + j];
      pa.src[j] = (const uint4*)(q == c->rank ? (const char*)in.data
                                              : c->peer[q] + CTRL_BYTES + heap_offset);
    }
    const int64_t work = (bytes / 16) * gsize;
    int64_t grid = (work + 4 * 512 - 1) / (4 * 512);
    const int64_t cap = engine == 3 ? 32 : 148 * 4;
    if (grid > cap) grid = cap;
    peer_pull_kernel<<<(unsigned)grid, 512, 0, s>>>(pa, (uint4*)out.data);
    if ((rc = launched(s))) return rc;
    return peer_barrier(c, channel, s);
  }
  // Staged gathers of more than two members pull every member's piece on its
  // own forked stream (event fork/join, graph-capturable), so the copy
  // engines read the peers concurrently instead of one after another.
  const bool fork = staged && gsize > 2 && !option(OPT_PEER_SERIAL_PULLS);
  cudaEvent_t* fev = c->fork_ev[channel];
  if (fork) {
    for (int j = 0; j <= gsize; ++j)
      if (!fev[j]) SPMD_CUDA_TRY(cudaEventCreateWithFlags(&fev[j], cudaEventDisableTiming));
    for (int j = 0; j < gsize; ++j)
      if (!c->fork[channel][j])
        SPMD_CUDA_TRY(cudaStreamCreateWithFlags(&c->fork[channel][j], cudaStreamNonBlocking));
    SPMD_CUDA_TRY(cudaEventRecord(fev[gsize], s));
  }
  for (int j = 0; j < gsize; ++j) {
    const int q = groups[grp * gsize + j];
    const char* src = q == c->rank ? (const char*)in.data : c->peer[q] + CTRL_BYTES + heap_offset;
    char* dst = (char*)out.data + j * w;
    cudaStream_t sj = s;
    if (fork) {
      sj = c->fork[channel][j];
      SPMD_CUDA_TRY(cudaStreamWaitEvent(sj, fev[gsize], 0));
    }
    if (outer == 1)
      SPMD_CUDA_TRY(cudaMemcpyAsync(dst, src, w, cudaMemcpyDeviceToDevice, sj));
    else
      SPMD_CUDA_TRY(cudaMemcpy2DAsync(dst, gsize * w, src, w, w, outer, cudaMemcpyDeviceToDevice,
                                      sj));
    if (fork) {
      SPMD_CUDA_TRY(cudaEventRecord(fev[j], sj));
      SPMD_CUDA_TRY(cudaStreamWaitEvent(s, fev[j], 0));
    }
  }
  return staged ? SPMD_OK : peer_barrier(c, channel, s);
}

extern "C" int spmd_peer_stage(spmd_comm* c, spmd_tensor in, int64_t heap_offset, void* stream) {
  SPMD_CHECK_ARG(c, "peer stage arguments");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  const int64_t bytes = numel(in) * elem_size(in.dtype);
  if (int rc = check_slot(c, heap_offset, bytes, "peer stage")) return rc;
  if (bytes == 0) return SPMD_OK;
  SPMD_CUDA_TRY(cudaMemcpyAsync(c->heap + CTRL_BYTES + heap_offset, in.data, bytes,
                                cudaMemcpyDeviceToDevice, as_stream(stream)));
  return SPMD_OK;
}

extern "C" int spmd_peer_barrier(spmd_comm* c, int channel, void* stream) {
  SPMD_CHECK_ARG(c && channel >= 0 && channel < NUM_CHANNELS, "peer barrier channel");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  return peer_barrier(c, channel, as_stream(stream));
}

// out = all-to-all(split_dim = 1, concat_dim = 0)(dot(lhs, rhs)) for a dot
// with one batch dim (the output's dim 0) -- the expert FFN-out einsum
// followed by the GShard combine all-to-all (C3; reference partitioner.py
// _try_all_to_all :283-318, simulator.py:372-390).  The wide GEMM's epilogue
// stores every 32-row output chunk into the heap of the member that owns its
// row block (rows = the flattened free dims, split on the leading one), in
// slot pos * batch + b of the concat dim, overlapping the exchange with the
// math; a barrier and one copy out of this epoch's parity buffer finish it.
extern "C" int spmd_dot_all_to_all(spmd_comm* c, spmd_tensor lhs, spmd_tensor rhs,
                                   spmd_tensor out, const spmd_dot_dims* dd, int split_dim,
                                   int concat_dim, const int32_t* groups, int ngroups, int gsize,
                                   void* stream) {
  SPMD_CHECK_ARG(c && dd, "dot_all_to_all arguments");
  SPMD_CHECK_ARG(lhs.dtype == SPMD_BF16 && rhs.dtype == SPMD_BF16 && out.dtype == SPMD_BF16,
                 "dot_all_to_all is bf16");
  if (split_dim != 1 || concat_dim != 0 || out.rank < 3 || dd->n_batch != 1 ||
      dd->lhs_batch[0] != 0 || dd->rhs_batch[0] != 0)
    return SPMD_ERR_UNSUPPORTED;
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int grp, pos;
  int rc = group_position(c, groups, ngroups, gsize, &grp, &pos);
  if (rc) return rc;
  SPMD_CHECK_ARG(gsize <= 8 && out.dims[0] % gsize == 0, "dot_all_to_all group");
  // dot output [batch, d1 * gsize, d2...] (pre-exchange); out = [batch * gsize, d1, d2...]
  spmd_tensor full = out;
  full.dims[0] = out.dims[0] / gsize;
  full.dims[1] = out.dims[1] * gsize;
  full.data = nullptr;
  const int64_t n = numel(out);
  SPMD_CHECK_ARG(n % 8 == 0, "dot_all_to_all size");
  int64_t rows_per_batch = 1;   // GEMM rows of one batch (the flattened free dims)
  for (int d = 1; d < out.rank - 1; ++d) rows_per_batch *= full.dims[d];
  SPMD_CHECK_ARG(rows_per_batch % gsize == 0, "dot_all_to_all split");
  // one slot = one member's row chunk of one batch: n / out.dims[0] elements
  const int64_t slot = n / out.dims[0];
  int64_t par_slots = 0;
  if ((rc = fused_parity(c, slot * 2, out.dims[0], &par_slots))) return rc;
  GemmScatter sc;
  memset(&sc, 0, sizeof(sc));
  sc.gsize = gsize;
  sc.pos = pos;
  for (int j = 0; j < gsize; ++j) sc.dst[j] = c->peer[groups[grp * gsize + j]] + CTRL_BYTES;
  sc.epoch = (const uint32_t*)c->heap;
  sc.rows = 1;
  sc.rchunk = rows_per_batch / gsize;
  sc.slot_base = pos * (int)full.dims[0];
  sc.nslots = (int)out.dims[0];
  sc.par_slots = (int)par_slots;
  cudaStream_t s = as_stream(stream);
  rc = dot_tcgen05(lhs, rhs, full, *dd, 1, s, &sc);
  if (rc) return rc;
  if ((rc = peer_barrier(c, 0, s))) return rc;
  const int64_t n16 = n / 8;
  peer_parity_copy_kernel<<<grid_for(n16, 256), 256, 0, s>>>(
      (const uint4*)(c->heap + CTRL_BYTES), (uint4*)out.data, (const uint32_t*)c->heap,
      par_slots * slot / 8, n16);
  return launched(s);
}

// ---------------------------------------------------------------------------
// Fused GShard dispatch + all-to-all (C3): x [B_loc, S, M] routed by
// (expert, slot) -> every member j receives rows [pos*B_loc + b, e_loc, c, :]
// for its experts e = j*E_loc + e_loc, written straight into its heap
// (16-byte NVLink stores, empty slots as zeros, so no receiver-side clear).
// ---------------------------------------------------------------------------
// Routing [B, S, K] (moe.cu layout) -> inv[(b * E + e) * C + slot] = s for
// every kept (token, choice); empty slots stay -1.
__global__ void moe_inverse_kernel(const int32_t* __restrict__ expert,
                                   const int32_t* __restrict__ slot, int32_t* __restrict__ inv,
                                   int64_t assigns, int K, int S, int E, int C) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < assigns;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int sl = slot[a];
    const int64_t t = a / K;
    if (sl < C) inv[((t / S) * E + expert[a]) * (int64_t)C + sl] = (int32_t)(t % S);
  }
}

struct DispatchPush {
  uint4* dst[8];      // member j's landing zone (data start of its heap)
  int G, pos, Bl, S, E, El, C;
  int64_t m16;        // 16-byte vectors per row
  int64_t par_rows;   // rows per parity (fused_parity: parity p starts at row p * par_rows)
};

__global__ void __launch_bounds__(256) moe_dispatch_push_kernel(const uint4* __restrict__ x,
                                                                const int32_t* __restrict__ inv,
                                                                DispatchPush a,
                                                                const uint32_t* ctrl) {
  const int64_t par = (int64_t)((*(volatile const uint32_t*)ctrl + 1) & 1);
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)a.G * a.Bl * a.El * a.C;   // (j, b, e_loc, c)
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < rows;
       w += warps) {
    int64_t r = w;
    const int c = (int)(r % a.C);
    r /= a.C;
    const int el = (int)(r % a.El);
    r /= a.El;
    const int b = (int)(r % a.Bl);
    const int j = (int)(r / a.Bl);
    const int s = inv[((int64_t)b * a.E + j * a.El + el) * a.C + c];
    const int64_t drow = par * a.par_rows +
                         (((int64_t)(a.pos * a.Bl + b) * a.El + el) * a.C + c);
    uint4* dst = a.dst[j] + drow * a.m16;
    if (s < 0) {
      for (int64_t i = lane; i < a.m16; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
    } else {
      const uint4* src = x + ((int64_t)b * a.S + s) * a.m16;
      for (int64_t i = lane; i < a.m16; i += 32) dst[i] = __ldcs(src + i);
    }
  }
  __threadfence_system();   // peer stores visible before the barrier signal
}

// x [B_loc, S, M] bf16, expert/slot s32 [B_loc, S] (spmd_moe_route) ->
// out [B_loc * G, E / G, C, M] = all-to-all(split 1, concat 0)(dispatch(x)).
extern "C" int spmd_moe_dispatch_all_to_all(spmd_comm* c, spmd_tensor x, spmd_tensor expert,
                                            spmd_tensor slot, spmd_tensor out,
                                            spmd_tensor index_scratch, const int32_t* groups,
                                            int ngroups, int gsize, void* stream) {
  SPMD_CHECK_ARG(c && x.dtype == SPMD_BF16 && out.dtype == SPMD_BF16 && x.rank == 3 &&
                     out.rank == 4 && expert.dtype == SPMD_S32 && slot.dtype == SPMD_S32,
                 "moe dispatch all-to-all expects bf16 x [B,S,M] -> [B*G, E/G, C, M]");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int grp, pos;
  int rc = group_position(c, groups, ngroups, gsize, &grp, &pos);
  if (rc) return rc;
  const int Bl = (int)x.dims[0], S = (int)x.dims[1], M = (int)x.dims[2];
  const int El = (int)out.dims[1], C = (int)out.dims[2], E = El * gsize;
  // routing [B, S] (top-1) or [B, S, K]
  const int K = expert.rank == 3 ? (int)expert.dims[2] : 1;
  SPMD_CHECK_ARG(expert.rank >= 2 && expert.rank <= 3 && slot.rank == expert.rank &&
                     expert.dims[0] == Bl && expert.dims[1] == S && K >= 1 && K <= 4,
                 "moe dispatch all-to-all routing shape");
  SPMD_CHECK_ARG(gsize <= 8 && out.dims[0] == (int64_t)Bl * gsize && out.dims[3] == M &&
                     M % 8 == 0,
                 "moe dispatch all-to-all shape");
  const int64_t n = numel(out);
  int64_t par_rows = 0;
  if ((rc = fused_parity(c, (int64_t)M * 2, n / M, &par_rows))) return rc;
  const int64_t inv_bytes = (int64_t)Bl * E * C * 4;
  SPMD_CHECK_ARG(index_scratch.data && index_scratch.dtype == SPMD_S32 &&
                     numel(index_scratch) * 4 >= inv_bytes,
                 "moe dispatch all-to-all: index scratch must hold B*E*C s32");
  cudaStream_t s = as_stream(stream);
  int32_t* inv = (int32_t*)index_scratch.data;
  SPMD_CUDA_TRY(cudaMemsetAsync(inv, 0xff, inv_bytes, s));   // -1: empty slot
  const int64_t tokens = (int64_t)Bl * S;
  moe_inverse_kernel<<<grid_for(tokens * K, 256), 256, 0, s>>>(
      (const int32_t*)expert.data, (const int32_t*)slot.data, inv, tokens * K, K, S, E, C);
  if ((rc = launched(s))) return rc;
  DispatchPush a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < gsize; ++j)
    a.dst[j] = (uint4*)(c->peer[groups[grp * gsize + j]] + CTRL_BYTES);
  a.G = gsize, a.pos = pos, a.Bl = Bl, a.S = S, a.E = E, a.El = El, a.C = C;
  a.m16 = M / 8;
  a.par_rows = par_rows;
  const int64_t rows = (int64_t)gsize * Bl * El * C;
  moe_dispatch_push_kernel<<<grid_for(rows * 32, 256), 256, 0, s>>>(
      (const uint4*)x.data, inv, a, (const uint32_t*)c->heap);
  if ((rc = launched(s))) return rc;
  if ((rc = peer_barrier(c, 0, s))) return rc;
  const int64_t n16 = n / 8;
  peer_parity_copy_kernel<<<grid_for(n16, 256), 256, 0, s>>>(
      (const uint4*)(c->heap + CTRL_BYTES), (uint4*)out.data, (const uint32_t*)c->heap,
      par_rows * (M / 8), n16);
  return launched(s);
}

// ---------------------------------------------------------------------------
// Push-based all-to-all / all-gather through the peer heap (C5 resharding,
// reference simulator.py:353-359, 382-387; partitioner.py:283-318).  Every
// rank writes each member's piece of its input straight into that member's
// landing zone at `heap_offset` -- in the member's final output layout, so
// the strided send side needs no pack pass -- with 16-byte NVLink stores
// (the affine copy kernel with a trailing system fence), then one barrier.
// The landing zone then IS the output: the executor hands out a view of it
// (`out.data == NULL`), or it is copied to `out`.  Zones stay stable until a
// later barrier (the executor closes each step with one).
// ---------------------------------------------------------------------------
static void row_major(const spmd_tensor& t, int64_t* st) {
  int64_t acc = 1;
  for (int k = t.rank - 1; k >= 0; --k) {
    st[k] = acc;
    acc *= t.dims[k];
  }
}

// One launch pushes all G pieces: chunk c of the flattened (piece, element)
// space goes to destination c % G, so the NVLink stores to the peers and the
// local copy of this rank's own piece run concurrently (G sequential copies
// measured 544 GB/s per GPU at G = 2).  Index math as the affine copy kernel
// (datamove.cu): pieces share shape and strides, differ in source offset and
// destination pointer.
struct PushArgs {
  int rank;
  int64_t shape[SPMD_MAX_RANK], sst[SPMD_MAX_RANK], dst[SPMD_MAX_RANK];
  int64_t n;                  // elements per piece (a multiple of V when vectorised)
  int64_t sbase[8];           // source offset of piece j
  int64_t dbase;              // destination offset (same in every member's zone)
  char* out[8];               // member j's landing zone
  int G;
};

template <typename T, int V>
__device__ __forceinline__ void push_offsets(const PushArgs& a, int j, int64_t v, int64_t& so,
                                             int64_t& d0) {
  int64_t r = v * V;
  so = a.sbase[j];
  d0 = a.dbase;
#pragma unroll
  for (int k = SPMD_MAX_RANK - 1; k >= 0; --k) {
    if (k < a.rank) {
      const int64_t ck = r % a.shape[k];
      r /= a.shape[k];
      so += ck * a.sst[k];
      d0 += ck * a.dst[k];
    }
  }
}

// U vectors per thread per chunk (chunk = 256 * U vectors of one piece):
// the U loads are all issued before the U NVLink stores.
template <typename T, int V, int U>
__global__ void __launch_bounds__(256) peer_push_kernel(const T* __restrict__ src, PushArgs a) {
  const int64_t per = a.n / V;                       // vectors per piece
  const int64_t chunks = (per + 256 * U - 1) / (256 * U);
  const int64_t total = chunks * a.G;
  for (int64_t c = blockIdx.x; c < total; c += gridDim.x) {
    const int j = (int)(c % a.G);
    const int64_t v0 = (c / a.G) * (256 * U) + threadIdx.x;
    T* dst = reinterpret_cast<T*>(a.out[j]);
    if (V == 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 256;
        if (v >= per) break;
        int64_t so, d0;
        push_offsets<T, V>(a, j, v, so, d0);
        dst[d0] = src[so];
      }
    } else {
      uint4 val[U];
      int64_t dof[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 256;
        dof[u] = -1;
        if (v < per) {
          int64_t so;
          push_offsets<T, V>(a, j, v, so, dof[u]);
          val[u] = __ldcs(reinterpret_cast<const uint4*>(src + so));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (dof[u] >= 0) *reinterpret_cast<uint4*>(dst + dof[u]) = val[u];
    }
  }
  __threadfence_system();   // peer stores visible before the barrier signal
}

// in: this rank's operand; zone_shape: one member's output shape.  piece j of
// `in` (index j of `sdim` split G ways, or the whole input when sdim < 0)
// lands at index pos of `cdim` (split G ways) in member j's zone.
static int peer_push(spmd_comm* c, const spmd_tensor& in, const spmd_tensor& zone_shape,
                     int sdim, int cdim, const int32_t* members, int gsize, int pos,
                     int64_t heap_offset, cudaStream_t s) {
  SPMD_CHECK_ARG(gsize >= 1 && gsize <= 8, "peer push group size <= 8");
  int64_t ist[SPMD_MAX_RANK], ost[SPMD_MAX_RANK];
  row_major(in, ist);
  row_major(zone_shape, ost);
  spmd_tensor piece = in;
  if (sdim >= 0) piece.dims[sdim] /= gsize;
  // merge dims contiguous in both views (fewer div/mods per element)
  PushArgs a;
  memset(&a, 0, sizeof(a));
  int r = 0;
  for (int k = 0; k < in.rank; ++k) {
    if (piece.dims[k] == 1) continue;
    if (r > 0 && a.sst[r - 1] == ist[k] * piece.dims[k] && a.dst[r - 1] == ost[k] * piece.dims[k]) {
      a.shape[r - 1] *= piece.dims[k];
      a.sst[r - 1] = ist[k];
      a.dst[r - 1] = ost[k];
      continue;
    }
    a.shape[r] = piece.dims[k];
    a.sst[r] = ist[k];
    a.dst[r] = ost[k];
    ++r;
  }
  a.rank = r;
  a.n = numel(piece);
  if (a.n == 0) return SPMD_OK;
  a.G = gsize;
  a.dbase = (int64_t)pos * piece.dims[cdim] * ost[cdim];
  for (int j = 0; j < gsize; ++j) {
    a.sbase[j] = sdim >= 0 ? (int64_t)j * piece.dims[sdim] * ist[sdim] : 0;
    a.out[j] = c->peer[members[j]] + CTRL_BYTES + heap_offset;
  }
  const int es = elem_size(in.dtype);
  const int V = 16 / es;
  bool vec = r >= 1 && a.sst[r - 1] == 1 && a.dst[r - 1] == 1 && a.shape[r - 1] % V == 0 &&
             a.dbase % V == 0 && (reinterpret_cast<uintptr_t>(in.data) & 15) == 0 &&
             (heap_offset & 15) == 0;
  for (int k = 0; vec && k < r - 1; ++k) vec = a.sst[k] % V == 0 && a.dst[k] % V == 0;
  for (int j = 0; vec && j < gsize; ++j) vec = a.sbase[j] % V == 0;
  const int64_t vecs = vec ? a.n / V : a.n;
  // 4 vectors per thread per chunk (loads before stores).  Grid cap by size
  // (scripts/push_size_probe.py, profiles/r2_push_ilp*_probe.log): 8 blocks
  // per SM for pushes under 256 MB (33.5 MB piece 0.069 vs 0.083 ms with 16;
  // the C2 2x2 step-start pair 0.154 vs 0.182), 16 above (536 MB piece:
  // 669 vs 650 GB/s).
  constexpr int PU = 4;
  int64_t grid = ((vecs + 256 * PU - 1) / (256 * PU)) * gsize;
  const int64_t cap = a.n * elem_size(in.dtype) * gsize >= (256LL << 20) ? 148LL * 16 : 148LL * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  SPMD_DISPATCH_BYTES(in.dtype, T, {
    if (vec)
      peer_push_kernel<T, 16 / sizeof(T), PU><<<(unsigned)grid, 256, 0, s>>>((const T*)in.data,
                                                                              a);
    else
      peer_push_kernel<T, 1, PU><<<(unsigned)grid, 256, 0, s>>>((const T*)in.data, a);
  });
  return launched(s);
}

static int finish_zone(spmd_comm* c, const spmd_tensor& out, int64_t heap_offset, int64_t bytes,
                       cudaStream_t s) {
  if (out.data && bytes)
    SPMD_CUDA_TRY(cudaMemcpyAsync(out.data, c->heap + CTRL_BYTES + heap_offset, bytes,
                                  cudaMemcpyDeviceToDevice, s));
  return SPMD_OK;
}

extern "C" int spmd_peer_all_to_all(spmd_comm* c, spmd_tensor in, spmd_tensor out,
                                    int split_dim, int concat_dim, const int32_t* groups,
                                    int ngroups, int gsize, int64_t heap_offset, int channel,
                                    void* stream) {
  SPMD_CHECK_ARG(c && in.dtype == out.dtype && in.rank == out.rank && split_dim >= 0 &&
                     split_dim < in.rank && concat_dim >= 0 && concat_dim < in.rank &&
                     in.dims[split_dim] % gsize == 0,
                 "peer all-to-all arguments");
  SPMD_CHECK_ARG(channel >= 0 && channel < NUM_CHANNELS, "peer barrier channel");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int grp, pos;
  int rc = group_position(c, groups, ngroups, gsize, &grp, &pos);
  if (rc) return rc;
  for (int k = 0; k < in.rank; ++k) {
    int64_t want = in.dims[k];
    if (k == split_dim) want /= gsize;
    if (k == concat_dim) want *= gsize;
    SPMD_CHECK_ARG(out.dims[k] == want, "peer all-to-all output shape");
  }
  const int64_t bytes = numel(out) * elem_size(out.dtype);
  if ((rc = check_slot(c, heap_offset, bytes, "peer all-to-all landing"))) return rc;
  cudaStream_t s = as_stream(stream);
  if ((rc = peer_push(c, in, out, split_dim, concat_dim, groups + grp * gsize, gsize, pos,
                      heap_offset, s)))
    return rc;
  if ((rc = peer_barrier(c, channel, s))) return rc;
  return finish_zone(c, out, heap_offset, bytes, s);
}

extern "C" int spmd_peer_push_all_gather(spmd_comm* c, spmd_tensor in, spmd_tensor out, int dim,
                                         const int32_t* groups, int ngroups, int gsize,
                                         int64_t heap_offset, int channel, void* stream) {
  SPMD_CHECK_ARG(c && in.dtype == out.dtype && in.rank == out.rank && dim >= 0 &&
                     dim < in.rank && out.dims[dim] == in.dims[dim] * gsize,
                 "peer all-gather arguments");
  SPMD_CHECK_ARG(channel >= 0 && channel < NUM_CHANNELS, "peer barrier channel");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int grp, pos;
  int rc = group_position(c, groups, ngroups, gsize, &grp, &pos);
  if (rc) return rc;
  const int64_t bytes = numel(out) * elem_size(out.dtype);
  if ((rc = check_slot(c, heap_offset, bytes, "peer all-gather landing"))) return rc;
  cudaStream_t s = as_stream(stream);
  if ((rc = peer_push(c, in, out, -1, dim, groups + grp * gsize, gsize, pos, heap_offset, s)))
    return rc;
  if ((rc = peer_barrier(c, channel, s))) return rc;
  return finish_zone(c, out, heap_offset, bytes, s);
}

// Device address of this rank's heap data at `offset` (the landing zone the
// push collectives leave their result in).
extern "C" void* spmd_comm_heap_ptr(spmd_comm* c, int64_t offset) {
  if (!c || !c->heap || offset < 0 || offset > c->heap_bytes) return nullptr;
  return c->heap + CTRL_BYTES + offset;
}

// Collective-permute through the peer heap (reference simulator.py:372-390:
// each target receives its source's buffer, non-targets are zero-filled):
// the sender's copy engine writes `in` straight into the target's heap slot
// at `heap_offset`, one barrier, then the receiver copies the slot out.
// Latency ~ two copy-engine launches + one barrier instead of NCCL's
// send/recv protocol (the halo exchange of a conv layer is ~2 MB).
static int peer_permute(spmd_comm* c, const char* src, int64_t rows, int64_t width,
                        int64_t pitch, spmd_tensor out, const int32_t* pairs, int npairs,
                        int64_t heap_offset, int channel, cudaStream_t s);

extern "C" int spmd_peer_collective_permute(spmd_comm* c, spmd_tensor in, spmd_tensor out,
                                            const int32_t* pairs, int npairs,
                                            int64_t heap_offset, int channel, void* stream) {
  SPMD_CHECK_ARG(c && in.dtype == out.dtype && numel(in) == numel(out), "permute mismatch");
  const int64_t bytes = numel(in) * elem_size(in.dtype);
  return peer_permute(c, (const char*)in.data, 1, bytes, bytes, out, pairs, npairs, heap_offset,
                      channel, as_stream(stream));
}

// Same, the sent buffer being the slice [start, start + out.dims[axis]) of
// `src` along `axis` with every other dim whole (the halo slab of a
// spatially partitioned conv): one 2-D copy-engine write of the slab rows
// straight from the producer's output, no slice kernel.
extern "C" int spmd_peer_slice_collective_permute(spmd_comm* c, spmd_tensor src, int axis,
                                                  int64_t start, spmd_tensor out,
                                                  const int32_t* pairs, int npairs,
                                                  int64_t heap_offset, int channel,
                                                  void* stream) {
  SPMD_CHECK_ARG(c && src.dtype == out.dtype && src.rank == out.rank && axis >= 0 &&
                     axis < src.rank && start >= 0 && start + out.dims[axis] <= src.dims[axis],
                 "slice permute mismatch");
  int64_t outer = 1, inner = elem_size(src.dtype);
  for (int d = 0; d < src.rank; ++d) {
    if (d != axis) SPMD_CHECK_ARG(src.dims[d] == out.dims[d], "slice permute: only `axis` is sliced");
    if (d < axis) outer *= src.dims[d];
    if (d > axis) inner *= src.dims[d];
  }
  return peer_permute(c, (const char*)src.data + start * inner, outer, out.dims[axis] * inner,
                      src.dims[axis] * inner, out, pairs, npairs, heap_offset, channel,
                      as_stream(stream));
}

static int peer_permute(spmd_comm* c, const char* src, int64_t rows, int64_t width,
                        int64_t pitch, spmd_tensor out, const int32_t* pairs, int npairs,
                        int64_t heap_offset, int channel, cudaStream_t s) {
  SPMD_CHECK_ARG(channel >= 0 && channel < NUM_CHANNELS, "peer barrier channel");
  if (!c->heap) {
    set_error("peer heap not enabled (spmd_comm_enable_peer)");
    return SPMD_ERR_INVALID;
  }
  int send_to = -1, recv_from = -1;
  std::vector<int> src_seen(c->nranks, 0), dst_seen(c->nranks, 0);
  for (int i = 0; i < npairs; ++i) {
    const int a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a < 0 || b < 0 || a >= c->nranks || b >= c->nranks || src_seen[a]++ || dst_seen[b]++) {
      set_error("collective-permute pairs must have distinct sources and distinct targets");
      return SPMD_ERR_SUBGROUP;
    }
    if (a == c->rank) send_to = b;
    if (b == c->rank) recv_from = a;
  }
  const int64_t bytes = rows * width;
  SPMD_CHECK_ARG(bytes == numel(out) * elem_size(out.dtype), "permute mismatch");
  if (int rc = check_slot(c, heap_offset, bytes, "peer permute landing")) return rc;
  if (send_to >= 0 && bytes) {
    char* dst = c->peer[send_to] + CTRL_BYTES + heap_offset;
    if (rows == 1)
      SPMD_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
    else
      SPMD_CUDA_TRY(cudaMemcpy2DAsync(dst, width, src, pitch, width, rows,
                                      cudaMemcpyDeviceToDevice, s));
  }
  int rc = peer_barrier(c, channel, s);
  if (rc) return rc;
  if (recv_from < 0)
    SPMD_CUDA_TRY(cudaMemsetAsync(out.data, 0, bytes, s));
  else if (bytes)
    SPMD_CUDA_TRY(cudaMemcpyAsync(out.data, c->heap + CTRL_BYTES + heap_offset, bytes,
                                  cudaMemcpyDeviceToDevice, s));
  return SPMD_OK;
}
