/*
 * spmd_b200.h -- C ABI of the B200-native GSPMD partitioned-execution hot path.
 *
 * The reference (minispmd, pure Python/NumPy) executes a partitioned program
 * with `evaluate_spmd` (minispmd/simulator.py:393-426), dispatching every
 * instruction to `evaluate_instruction` (simulator.py:157-301) and every
 * collective to `_collective` (simulator.py:333-390).  This library replaces
 * both: one entry point per instruction family, plain pointers and sizes, no
 * torch types.  A ctypes binding of exactly these symbols is what a
 * maintainer would add to the reference.
 *
 * Conventions
 *  - Every tensor is dense row-major and *partition-stacked*: the buffer holds
 *    `nparts` consecutive per-partition tensors of shape dims[0..rank).  With
 *    one process per GPU nparts == 1 and the partition id is the rank; on one
 *    GPU simulating an N-device mesh nparts == N (reference lockstep
 *    semantics, simulator.py:412-425).
 *  - Scalars consumed per partition (pad value, reduce init, dynamic-slice
 *    start indices) are rank-0 tensors, i.e. `nparts` values.
 *  - All calls are asynchronous on the caller's `cudaStream_t` (passed as
 *    void*).  Status codes are returned synchronously for argument errors;
 *    device-side faults (integer divide by zero, simulator.py:63-69) set a
 *    device error word read back by spmd_check_device_errors().
 *  - The library never frees caller memory.
 */
#ifndef SPMD_B200_H_
#define SPMD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMD_MAX_RANK 8
#define SPMD_MAX_PARTS 64

/* IR dtypes (reference ir.py:19-23 plus BF16). */
typedef enum {
  SPMD_F32 = 0, SPMD_S32 = 1, SPMD_U32 = 2, SPMD_PRED = 3, SPMD_BF16 = 4
} spmd_dtype;

/* Status codes.  The Python shim maps them onto the reference's exception
 * classes (simulator.py:33-42, sharding.py:27-58, partitioner.py:44-53). */
typedef enum {
  SPMD_OK = 0,
  SPMD_ERR_INVALID = 1,      /* bad argument                     -> EvalError */
  SPMD_ERR_SHAPE = 2,        /* inconsistent shapes              -> EvalError */
  SPMD_ERR_SUBGROUP = 3,     /* groups/pairs do not partition    -> SubgroupMismatch */
  SPMD_ERR_DIV_ZERO = 4,     /* integer division by zero         -> DivideByZero */
  SPMD_ERR_CUDA = 5,
  SPMD_ERR_NCCL = 6,
  SPMD_ERR_UNSUPPORTED = 7
} spmd_status;

typedef struct {
  void* data;
  int32_t dtype;   /* spmd_dtype */
  int32_t rank;    /* per-partition rank, <= SPMD_MAX_RANK */
  int64_t dims[SPMD_MAX_RANK];
} spmd_tensor;

/* Opcodes of the elementwise families (values of ir.Op order). */
typedef enum { SPMD_NEGATE = 0, SPMD_EXP = 1, SPMD_RELU = 2 } spmd_unary_op;
typedef enum {
  SPMD_ADD = 0, SPMD_MULTIPLY = 1, SPMD_MAXIMUM = 2, SPMD_SUBTRACT = 3,
  SPMD_DIVIDE = 4, SPMD_COMPARE = 5
} spmd_binary_op;
typedef enum { SPMD_EQ = 0, SPMD_NE = 1, SPMD_LT = 2, SPMD_LE = 3, SPMD_GT = 4, SPMD_GE = 5 } spmd_cmp;
typedef enum { SPMD_SUM = 0, SPMD_MAX = 1, SPMD_MIN = 2, SPMD_PROD = 3 } spmd_reduce_kind;

/* ---- library ------------------------------------------------------------ */
const char* spmd_version(void);
const char* spmd_status_string(int status);
const char* spmd_last_error(void);
/* Reads and clears the device error word; returns SPMD_ERR_DIV_ZERO if an
 * integer division by zero happened since the last call. Synchronises stream. */
int spmd_check_device_errors(void* stream);
/* Number of kernels this library has launched (for launch accounting). */
int64_t spmd_launch_count(void);
/* Cap the SMs used by the persistent tensor-core kernels (0 = all), leaving
 * room for collective kernels that overlap them. */
int spmd_set_sm_limit(int sms);
/* Runtime tuning options, read at every launch (each starts from its SPMD_*
 * environment variable): "gemm_mode" (1: 1-CTA, 2: 256x256 CTA pairs,
 * 3: 256x512 wide pairs), "gemm_group", "gemm_raster_n", "gemm_hint",
 * "gemm_store_hint", "gemm_epi_direct", "scatter_epi_direct", "attn_mode",
 * "attn_kt", "conv_mode", "conv_wres", "conv_taps", "nccl_max_ctas",
 * "peer_timeout_ms", "peer_serial_pulls", "f32_dot_tc" (large f32 Dots as 3xTF32
 * tensor-core GEMMs, default 1).  Unknown names -> SPMD_ERR_INVALID.
 * Not part of the reference interface (tuning and variant selection). */
int spmd_set_option(const char* name, int64_t value);
int spmd_get_option(const char* name, int64_t* value);
/* C[M,N] = A[M,K] . B[K,N] (+ReLU if relu), row-major bf16, A K-major and B
 * MN-major: the tcgen05 GEMM alone, for micro-benchmarks (the Dot of
 * simulator.py:258-275 without the dimension-number plumbing). */
int spmd_gemm_bf16(const void* a, const void* b, void* c, int64_t M, int64_t N, int64_t K,
                   int relu, void* stream);

/* ---- sources (simulator.py:161-172) ---------------------------------------- */
int spmd_iota(spmd_tensor out, int axis, int64_t nparts, void* stream);
int spmd_partition_id(spmd_tensor out, int64_t nparts, int32_t first_id, void* stream);
/* Broadcast one host literal (rank `lit.rank`, `lit.data` on the HOST) to all
 * partitions of `out`. */
int spmd_constant(spmd_tensor lit_host, spmd_tensor out, int64_t nparts, void* stream);

/* ---- elementwise (simulator.py:173-198) ------------------------------------ */
int spmd_unary(int op, spmd_tensor in, spmd_tensor out, int64_t nparts, void* stream);
int spmd_binary(int op, int cmp, spmd_tensor a, spmd_tensor b, spmd_tensor out,
                int64_t nparts, void* stream);
int spmd_select(spmd_tensor pred, spmd_tensor on_true, spmd_tensor on_false,
                spmd_tensor out, int64_t nparts, void* stream);
/* dtype conversion (host I/O helper; not an IR op). */
int spmd_convert(spmd_tensor in, spmd_tensor out, int64_t nparts, void* stream);

/* ---- data movement (simulator.py:199-241, 278-300) ------------------------- */
int spmd_broadcast(spmd_tensor in, spmd_tensor out, const int32_t* broadcast_dims,
                   int64_t nparts, void* stream);
int spmd_transpose(spmd_tensor in, spmd_tensor out, const int32_t* perm,
                   int64_t nparts, void* stream);
/* Transpose -> ReLU (numpy maximum(x, 0): -0 -> +0, NaN kept) in one pass. */
int spmd_transpose_relu(spmd_tensor in, spmd_tensor out, const int32_t* perm, int64_t nparts,
                        void* stream);
int spmd_reverse(spmd_tensor in, spmd_tensor out, const int32_t* dims, int ndims,
                 int64_t nparts, void* stream);
int spmd_pad(spmd_tensor in, spmd_tensor value, spmd_tensor out, const int64_t* low,
             const int64_t* high, const int64_t* interior, int64_t nparts, void* stream);
int spmd_slice(spmd_tensor in, spmd_tensor out, const int64_t* starts,
               const int64_t* strides, int64_t nparts, void* stream);
/* Start indices are clamped to [0, dim - size] (XLA semantics, simulator.py:227). */
int spmd_dynamic_slice(spmd_tensor in, const spmd_tensor* starts, spmd_tensor out,
                       int64_t nparts, void* stream);
int spmd_dynamic_update_slice(spmd_tensor in, spmd_tensor update,
                              const spmd_tensor* starts, spmd_tensor out,
                              int64_t nparts, void* stream);
int spmd_concat(const spmd_tensor* ins, int n, int axis, spmd_tensor out,
                int64_t nparts, void* stream);
int spmd_rotate(spmd_tensor in, spmd_tensor out, int dim, int64_t amount,
                int64_t nparts, void* stream);
int spmd_shift(spmd_tensor in, spmd_tensor fill, spmd_tensor out, int dim,
               int64_t amount, int64_t nparts, void* stream);

/* ---- reductions (simulator.py:242-257) ------------------------------------- */
int spmd_reduce(spmd_tensor in, spmd_tensor init, spmd_tensor out, const int32_t* dims,
                int ndims, int kind, int64_t nparts, void* stream);

/* ---- contractions (simulator.py:258-277) ------------------------------------
 * Generalised dot: out[batch, lhs_free, rhs_free] = sum_k lhs*rhs.  BF16 runs on
 * tcgen05 tensor cores (fp32 TMEM accumulation).  F32: Dots with M, N >= 256
 * and K >= 64 run as a 3xTF32 tcgen05 GEMM (hi*hi + hi*lo + lo*hi, ~1e-6
 * normwise vs the f64 reference; option "f32_dot_tc" = 0 disables), smaller
 * ones accumulate in fp64; integers accumulate in int64 (as the reference),
 * rounding once. */
typedef struct {
  int32_t n_batch, n_contract;
  int32_t lhs_batch[SPMD_MAX_RANK], rhs_batch[SPMD_MAX_RANK];
  int32_t lhs_contracting[SPMD_MAX_RANK], rhs_contracting[SPMD_MAX_RANK];
  int32_t epilogue;      /* 0 none, 1 relu (fused; executor-level fusion) */
} spmd_dot_dims;
int spmd_dot(spmd_tensor lhs, spmd_tensor rhs, spmd_tensor out, const spmd_dot_dims* dd,
             int64_t nparts, void* stream);
/* f32 Dot with operands given as their tf32 hi / lo halves
 * (spmd_local_all_gather_split / _split_t; hi.data NULL = not pre-split, then
 * the operand tensor's data is split here): the 3xTF32 GEMM without those
 * split passes.  A pre-split MN-major rhs is in the K-major [batch][N][K]
 * layout.  SPMD_ERR_UNSUPPORTED when the 3xTF32 path does not apply (operand =
 * hi + lo exactly; run spmd_dot). */
int spmd_dot_f32_presplit(spmd_tensor lhs, spmd_tensor lhs_hi, spmd_tensor lhs_lo,
                          spmd_tensor rhs, spmd_tensor rhs_hi, spmd_tensor rhs_lo,
                          spmd_tensor out, const spmd_dot_dims* dd, int64_t nparts,
                          void* stream);
/* out = Dot(lhs, rhs) + resid (bf16; resid has the output's shape): the
 * layer's residual Add (simulator.py:173-198) folded into the GEMM epilogue,
 * one fp32 add before the single rounding.  SPMD_ERR_UNSUPPORTED when the
 * wide tcgen05 GEMM does not apply (run spmd_dot and the Add instead). */
int spmd_dot_add(spmd_tensor lhs, spmd_tensor rhs, spmd_tensor resid, spmd_tensor out,
                 const spmd_dot_dims* dd, int64_t nparts, void* stream);

typedef struct {
  int32_t lhs_batch, lhs_feature, rhs_in_feature, rhs_out_feature, out_batch, out_feature;
  int32_t n_spatial;
  int32_t lhs_spatial[SPMD_MAX_RANK], rhs_spatial[SPMD_MAX_RANK], out_spatial[SPMD_MAX_RANK];
  int32_t size[SPMD_MAX_RANK], stride[SPMD_MAX_RANK], pad_low[SPMD_MAX_RANK],
          pad_high[SPMD_MAX_RANK], base_dilation[SPMD_MAX_RANK], window_dilation[SPMD_MAX_RANK];
  int32_t epilogue;      /* 0 none, 1 relu (fused; executor-level fusion) */
} spmd_conv_dims;
int spmd_convolution(spmd_tensor lhs, spmd_tensor rhs, spmd_tensor out,
                     const spmd_conv_dims* cd, int64_t nparts, void* stream);

/* ---- fused kernels selected by the executor (same semantics as the op chain) */
/* Uneven-shard / halo range mask (partitioner select_range chain,
 * reference partitioner.py:205-228): out = (low <= iota_axis + offset[p] < high)
 * ? in : fill[p]; offset s32 and fill are per-partition scalars. */
int spmd_mask_range(spmd_tensor in, spmd_tensor offset, spmd_tensor fill, spmd_tensor out,
                    int axis, int64_t low, int64_t high, int has_low, int64_t nparts,
                    void* stream);
/* Halo window (reference formatting.py:109-182): out = dynamic_slice(
 * mask(concat(pieces[0..n), axis)), start[p] on axis) in one pass; the mask
 * (optional) is the range mask above on buffer positions. */
int spmd_halo_window(const spmd_tensor* pieces, int npieces, int axis, spmd_tensor start,
                     int has_mask, spmd_tensor offset, spmd_tensor fill, int64_t low,
                     int64_t high, int has_low, spmd_tensor out, int64_t nparts, void* stream);
/* Fused attention (executor fusion of Dot(q,k) -> softmax -> Dot(p,v)):
 * q [B,S,N,D], k/v [B,T,N,D] bf16 -> out [B,N,S,D] = softmax(scale q.k^T) v,
 * D in {64,128,256}; tcgen05 with S/O accumulators in TMEM. */
int spmd_attention(spmd_tensor q, spmd_tensor k, spmd_tensor v, spmd_tensor out, float scale,
                   int64_t nparts, void* stream);
/* Same, output layout selectable: out_bsnd = 1 writes out[B,S,N,D] (the
 * transposed context the out-projection consumes, App. A ctx_t) straight from
 * the epilogue's TMA store. */
int spmd_attention_layout(spmd_tensor q, spmd_tensor k, spmd_tensor v, spmd_tensor out,
                          float scale, int out_bsnd, int64_t nparts, void* stream);
/* Row softmax over the last dim: out = exp(x - max) / sum(exp(x - max)). */
int spmd_softmax_lastdim(spmd_tensor in, spmd_tensor out, int64_t nparts, void* stream);
/* Softmax backward over the last dim (bf16 or f32; 16-byte vector path for
 * bf16 rows of L % 8 == 0, L <= 1024): out = p * (dp - sum_last(dp * p)) --
 * the training graph's multiply/reduce/broadcast/subtract/multiply chain
 * (reference simulator.py:173-198 elementwise, :242-257 reduce) in one pass,
 * fp32 row sum. */
int spmd_softmax_backward_lastdim(spmd_tensor p, spmd_tensor dp, spmd_tensor out,
                                  int64_t nparts, void* stream);
/* ReLU backward: out = h > 0 ? g : 0 (compare GT + select over broadcast
 * zeros in the reference graph), bf16 or f32. */
int spmd_relu_backward(spmd_tensor h, spmd_tensor g, spmd_tensor out, int64_t nparts,
                       void* stream);

/* ---- GShard MoE routing + dispatch/combine permutations (config C3) ---------
 * The reference consumes a given one-hot dispatch tensor through a dense Dot
 * (tests/test_acceptance.py:326-349); these kernels produce it (route), and
 * replace the one-hot Dots by exact gathers (dispatch/combine). */
/* logits [B,S,E] f32/bf16 -> expert, slot s32 [B,S] and gate f32 [B,S] */
int spmd_moe_route(spmd_tensor logits, int capacity, spmd_tensor expert, spmd_tensor slot,
                   spmd_tensor gate, int64_t nparts, void* stream);
/* x [B,S,M] bf16 -> expert buffers [B,E,C,M] (== Dot(dispatch_onehot, x)) */
int spmd_moe_dispatch(spmd_tensor x, spmd_tensor expert, spmd_tensor slot, spmd_tensor out,
                      int64_t nparts, void* stream);
/* y [B,E,C,M] bf16 -> out [B,S,M] (== Dot(combine_weights, y)) */
int spmd_moe_combine(spmd_tensor y, spmd_tensor expert, spmd_tensor slot, spmd_tensor gate,
                     spmd_tensor out, int64_t nparts, void* stream);
/* The same gathers with the MoE layer's Transpose(1,0,2,3) -> ReLU annotation
 * chain folded in (workloads.moe_layer): flags bit 0 = the expert-side tensor
 * is [E,B,C,M] (dispatch writes it, combine reads it), bit 1 = ReLU on the
 * copied / read values (numpy maximum(x, 0)). */
int spmd_moe_dispatch_ex(spmd_tensor x, spmd_tensor expert, spmd_tensor slot, spmd_tensor out,
                         int flags, int64_t nparts, void* stream);
int spmd_moe_combine_ex(spmd_tensor y, spmd_tensor expert, spmd_tensor slot, spmd_tensor gate,
                        spmd_tensor out, int flags, int64_t nparts, void* stream);
/* dense dispatch / combine masks [B,S,E,C] from a routing */
int spmd_moe_masks(spmd_tensor expert, spmd_tensor slot, spmd_tensor gate,
                   spmd_tensor dispatch, spmd_tensor combine, int64_t nparts, void* stream);

/* ---- loopback collectives: all partitions resident on this GPU ---------------
 * (simulator.py:333-390 semantics; groups is a flat [ngroups*gsize] table in
 * group order; reductions fold serially in group order, so integer and float
 * results are bit-identical to the reference). */
int spmd_local_all_gather(spmd_tensor in, spmd_tensor out, int dim, const int32_t* groups,
                          int ngroups, int gsize, int64_t nparts, void* stream);
/* The same all-gather of an f32 operand written as its tf32 hi / lo halves
 * (hi = tf32(x), lo = x - hi): feeds spmd_dot_f32_presplit, which then skips
 * its split pass.  SPMD_ERR_UNSUPPORTED for runs too short for the row kernel. */
int spmd_local_all_gather_split(spmd_tensor in, spmd_tensor hi, spmd_tensor lo, int dim,
                                const int32_t* groups, int ngroups, int gsize, int64_t nparts,
                                void* stream);
/* All-gather along dim 0 of an f32 [K_local, N] operand written as the tf32
 * hi / lo halves of its K-major transpose [N, gsize * K_local] (the layout
 * spmd_dot_f32_presplit takes for an MN-major rhs).  SPMD_ERR_UNSUPPORTED
 * unless K_local % 64 == 0 and N % 4 == 0. */
int spmd_local_all_gather_split_t(spmd_tensor in, spmd_tensor hi, spmd_tensor lo,
                                  const int32_t* groups, int ngroups, int gsize, int64_t nparts,
                                  void* stream);
int spmd_local_all_reduce(spmd_tensor in, spmd_tensor out, int kind, const int32_t* groups,
                          int ngroups, int gsize, int64_t nparts, void* stream);
int spmd_local_reduce_scatter(spmd_tensor in, spmd_tensor out, int dim, int kind,
                              const int32_t* groups, int ngroups, int gsize,
                              int64_t nparts, void* stream);
int spmd_local_all_to_all(spmd_tensor in, spmd_tensor out, int split_dim, int concat_dim,
                          const int32_t* groups, int ngroups, int gsize, int64_t nparts,
                          void* stream);
/* pairs: flat [npairs*2] (source, target); non-targets receive zeros. */
int spmd_local_collective_permute(spmd_tensor in, spmd_tensor out, const int32_t* pairs,
                                  int npairs, int64_t nparts, void* stream);

/* Convolution whose input is a halo window along H (dim 1):
 * window = DS(mask(concat(pieces)), start), the window assembly of
 * exchange_and_slice (reference formatting.py:109-182) feeding
 * handle_convolution (:494-540).  The conv's TMA loads read each window row
 * straight from its piece -- no window buffer in HBM.  Masked rows
 * (global row + offset outside [low, high)) read as zeros: the mask's fill
 * must be 0.  `window` gives the window shape only (data unused).
 * SPMD_ERR_UNSUPPORTED when the conv does not qualify (spmd_halo_window +
 * spmd_convolution then). */
int spmd_halo_convolution(const spmd_tensor* pieces, int npieces, int axis, spmd_tensor start,
                          int has_mask, spmd_tensor offset, int64_t low, int64_t high,
                          int has_low, spmd_tensor window, spmd_tensor rhs, spmd_tensor out,
                          const spmd_conv_dims* dims, int64_t nparts, void* stream);

/* ---- NCCL collectives: one process per GPU over NVLink/NVSwitch -------------- */
typedef struct spmd_comm spmd_comm;
int spmd_comm_id_bytes(void);
int spmd_comm_get_unique_id(void* id_out);
int spmd_comm_init(spmd_comm** comm, int nranks, int rank, const void* unique_id);
int spmd_comm_destroy(spmd_comm* comm);
/* Scratch used for pack/unpack of non-leading-dim collectives (device memory
 * owned by the caller, >= 2x the largest collective buffer). */
int spmd_comm_set_workspace(spmd_comm* comm, void* ptr, int64_t bytes);
int spmd_all_gather(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int dim,
                    const int32_t* groups, int ngroups, int gsize, void* stream);
int spmd_all_reduce(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int kind,
                    const int32_t* groups, int ngroups, int gsize, void* stream);
int spmd_reduce_scatter(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int dim, int kind,
                        const int32_t* groups, int ngroups, int gsize, void* stream);
int spmd_all_to_all(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int split_dim,
                    int concat_dim, const int32_t* groups, int ngroups, int gsize,
                    void* stream);
int spmd_collective_permute(spmd_comm* comm, spmd_tensor in, spmd_tensor out,
                            const int32_t* pairs, int npairs, void* stream);

/* ---- Peer-memory fused collectives (CUDA IPC over NVLink/NVSwitch) -----------
 * Collective: every rank allocates a `bytes` heap and maps every other rank's.
 * Growing re-exchanges (all ranks must call with the same size). */
int spmd_comm_enable_peer(spmd_comm* comm, int64_t bytes, void* stream);
int64_t spmd_comm_peer_bytes(spmd_comm* comm);
/* Reserve the fused-op landing zone [0, 3H) of the heap (grows only; H is
 * rounded up to 4 KiB).  H must be >= the per-parity bytes of every fused op
 * below (gsize * numel(out) * 2 for a dot -> reduce-scatter, numel(out) * 2
 * for the all-to-all ones).  Parity p of an op with unit (slot / row) u
 * starts at unit p * ceil(H / u): both parities of ANY two ops are disjoint,
 * so back-to-back fused ops of different sizes never overwrite a buffer a
 * peer is still reducing.  All ranks reserve the same H, before enable_peer
 * sizes the heap to >= 3H + the staging slots (offsets >= 3H). */
int spmd_comm_reserve_fused(spmd_comm* comm, int64_t half_bytes);
int64_t spmd_comm_fused_half(spmd_comm* comm);
/* out = reduce-scatter(sum, dim)(dot(lhs, rhs)) in one tcgen05 GEMM whose
 * epilogue stores each output tile straight into the owning rank's heap
 * (replaces the Dot + ReduceScatter pair emitted by reference
 * partitioner.py:751-759 and executed by simulator.py:258-275, 360-371).
 * bf16; `dim` must be the last output dim and come from the rhs free dim
 * (or the leading row dim of a dot without batch dims); needs
 * spmd_comm_reserve_fused(>= 2 * gsize * numel(out)).  SPMD_ERR_UNSUPPORTED
 * when the GEMM layout does not qualify (use spmd_dot + spmd_reduce_scatter). */
int spmd_dot_reduce_scatter(spmd_comm* comm, spmd_tensor lhs, spmd_tensor rhs, spmd_tensor out,
                            const spmd_dot_dims* dims, int dim, const int32_t* groups,
                            int ngroups, int gsize, void* stream);
/* ... with the layer's residual Add (simulator.py:173-198) folded into the
 * reduce: out = reduce_scatter(dot(lhs, rhs)) + resid, rounded as the unfused
 * pair (bit-identical to spmd_dot_reduce_scatter followed by the Add). */
int spmd_dot_reduce_scatter_add(spmd_comm* comm, spmd_tensor lhs, spmd_tensor rhs,
                                spmd_tensor resid, spmd_tensor out, const spmd_dot_dims* dims,
                                int dim, const int32_t* groups, int ngroups, int gsize,
                                void* stream);
/* out = all-to-all(split 1, concat 0)(dot(lhs, rhs)) for a dot with one
 * batch dim (output dim 0): the expert FFN-out einsum + GShard combine
 * all-to-all (C3).  The GEMM epilogue stores each output row chunk into the
 * owning member's heap (slot pos * batch + b), then a barrier and one copy.
 * bf16; needs spmd_comm_reserve_fused(>= 2 * numel(out)); SPMD_ERR_UNSUPPORTED when
 * the layout does not qualify (spmd_dot + spmd_all_to_all then). */
int spmd_dot_all_to_all(spmd_comm* comm, spmd_tensor lhs, spmd_tensor rhs, spmd_tensor out,
                        const spmd_dot_dims* dims, int split_dim, int concat_dim,
                        const int32_t* groups, int ngroups, int gsize, void* stream);
/* x [B,S,M] bf16 routed by expert/slot s32 [B,S] (spmd_moe_route) -> out
 * [B*G, E/G, C, M] = all-to-all(split 1, concat 0)(dispatch(x)): every row is
 * pushed straight into the owning member's heap (empty capacity slots as
 * zeros), barrier, one copy.  `index_scratch`: caller-owned s32 of >= B*E*C
 * elements (the (batch, expert, slot) -> token table; stream-ordered with
 * this call only).  Needs spmd_comm_reserve_fused(>= 2 * numel(out)). */
int spmd_moe_dispatch_all_to_all(spmd_comm* comm, spmd_tensor x, spmd_tensor expert,
                                 spmd_tensor slot, spmd_tensor out, spmd_tensor index_scratch,
                                 const int32_t* groups, int ngroups, int gsize, void* stream);
/* All-gather through the peer heap (reference simulator.py:353-359 piece
 * order): stage `in` at heap data offset `heap_offset` (256-aligned, caller
 * assigned, >= 3 * fused_half and disjoint from other live all-gathers), barrier, pull every member's piece with copy-engine copies,
 * barrier.  `channel` (0..3): one per issuing stream -- all ranks must issue
 * the calls of a channel in the same order.  `engine`: 0 = copy engines (no
 * SMs: for gathers hidden under GEMMs), 1 = SM pull kernel (16-byte NVLink
 * loads, whole GPU: for gathers on the critical path), 3 = SM pull with 32
 * CTAs (background, co-resident beside a persistent GEMM), 4 = pre-staged:
 * every member already staged its piece with spmd_peer_stage and passed a
 * spmd_peer_barrier since, and none overwrites it before a later barrier --
 * only the copy-engine pulls are issued (no kernel, so the gather never waits
 * for SMs a persistent GEMM holds). */
int spmd_peer_all_gather(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int dim,
                         const int32_t* groups, int ngroups, int gsize, int64_t heap_offset,
                         int channel, int engine, void* stream);
/* Stage `in` at heap data offset `heap_offset` (copy engine) for engine-4
 * gathers: the executor stages every parameter (weight) gather of a step at
 * the step start, then one barrier; another barrier at the step end keeps
 * the slots stable until every member has pulled. */
int spmd_peer_stage(spmd_comm* comm, spmd_tensor in, int64_t heap_offset, void* stream);
/* Collective-permute through the peer heap (reference simulator.py:372-390;
 * non-targets zero-filled): the sender's copy engine writes `in` into the
 * target's heap slot at `heap_offset` (uniform layout, caller assigned),
 * barrier on `channel`, the receiver copies its slot to `out`.  Callers keep
 * the slot live until a later barrier (the executor closes each step with
 * one). */
int spmd_peer_collective_permute(spmd_comm* comm, spmd_tensor in, spmd_tensor out,
                                 const int32_t* pairs, int npairs, int64_t heap_offset,
                                 int channel, void* stream);
/* Same, the sent buffer being the slice [start, start + out.dims[axis]) of
 * `src` along `axis`, every other dim whole (a halo slab): one 2-D
 * copy-engine write from the producer's output, no slice kernel. */
int spmd_peer_slice_collective_permute(spmd_comm* comm, spmd_tensor src, int axis, int64_t start,
                                       spmd_tensor out, const int32_t* pairs, int npairs,
                                       int64_t heap_offset, int channel, void* stream);
/* Push-based all-to-all (reference simulator.py:382-387 semantics: piece j
 * of `in` split along split_dim goes to group member j, concatenated along
 * concat_dim in group order): every rank writes each member's piece straight
 * into that member's landing zone at heap data offset `heap_offset` (>= 3 *
 * fused_half, 256-aligned, same on every rank, sized numel(out)), already in
 * the member's output layout -- no pack / unpack pass -- then one barrier on
 * `channel`.  out.data == NULL: the zone (spmd_comm_heap_ptr) is the result,
 * valid until the zone is reused after a later barrier; else it is copied
 * to out. */
int spmd_peer_all_to_all(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int split_dim,
                         int concat_dim, const int32_t* groups, int ngroups, int gsize,
                         int64_t heap_offset, int channel, void* stream);
/* Push-based all-gather along `dim` (simulator.py:353-359 piece order): every
 * rank writes its shard into slot `pos` of every member's landing zone, one
 * barrier; out.data == NULL as for spmd_peer_all_to_all. */
int spmd_peer_push_all_gather(spmd_comm* comm, spmd_tensor in, spmd_tensor out, int dim,
                              const int32_t* groups, int ngroups, int gsize,
                              int64_t heap_offset, int channel, void* stream);
/* Device address of this rank's heap data at `offset` (NULL if outside). */
void* spmd_comm_heap_ptr(spmd_comm* comm, int64_t offset);
/* Device-side barrier of all ranks on `channel` (epoch flags in the peer
 * heap control page; graph-replay safe; times out into the device error
 * word). */
int spmd_peer_barrier(spmd_comm* comm, int channel, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPMD_B200_H_ */
