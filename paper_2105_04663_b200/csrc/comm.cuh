// The communicator handle behind `spmd_comm*` (shared by the NCCL
// collectives and the peer-memory fused kernels).
#pragma once

#include "common.cuh"

#include <nccl.h>

#include <map>
#include <vector>

struct spmd_comm {
  ncclComm_t world;
  int nranks, rank;
  std::map<std::vector<int32_t>, ncclComm_t> splits;
  char* ws = nullptr;
  int64_t ws_bytes = 0;
  // Peer-memory heap (CUDA IPC, one per rank, same size everywhere):
  // [control page | data].  peer[q] = rank q's heap mapped into this
  // process (peer[rank] = heap).  See peer.cu.
  char* heap = nullptr;
  int64_t heap_bytes = 0;   // data bytes (excluding the control page)
  // Fused-op landing zone: parity p of every fused dot -> reduce-scatter /
  // all-to-all and of the MoE dispatch push starts at the first whole unit
  // (slot or row) at or past p * fused_half, so the two parities of ANY two
  // ops are disjoint ([0, half) vs [half, 3 * half)).  Staging / landing
  // slots of the peer gathers and permutes live at offsets >= 3 * half.
  int64_t fused_half = 0;
  char* peer[SPMD_MAX_PARTS] = {nullptr};
  // Fork streams/events for per-member parallel copy-engine pulls of
  // pre-staged gathers, one set per barrier channel (created lazily).
  cudaStream_t fork[4][SPMD_MAX_PARTS] = {};
  cudaEvent_t fork_ev[4][SPMD_MAX_PARTS + 1] = {};
};

namespace spmd {

#define NCCL_TRY(expr)                                                              \
  do {                                                                              \
    ncclResult_t _r = (expr);                                                       \
    if (_r != ncclSuccess) {                                                        \
      set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));                \
      return SPMD_ERR_NCCL;                                                         \
    }                                                                               \
  } while (0)

// Subgroup table -> (my group index, my position); validates that the groups
// partition the ranks (reference simulator.py:322-330).
int group_position(const spmd_comm* c, const int32_t* groups, int ngroups, int gsize, int* group,
                   int* pos);
}  // namespace spmd
