"""B200 executor for partitioned SPMD programs.

Replaces the reference's lockstep NumPy interpreter ``evaluate_spmd``
(``minispmd/simulator.py:393-426``): every instruction of the per-device
program is dispatched to one C-ABI entry point (``include/spmd_b200.h``),
which launches hand-written sm_100a kernels on the current CUDA stream;
collectives go to NCCL (one process per GPU) or, when one GPU simulates the
whole mesh, to loopback kernels with the reference's exact semantics.

Values live on the device *partition-stacked*: a per-device value of shape
``dims`` is a tensor ``[P, *dims]`` where ``P`` is the number of partitions
this process executes (``P = N`` for a simulated mesh on one GPU, ``P = 1``
with one process per GPU).  Reshape is a free view of that layout.

Executor-level fusions (``fuse=True``, default off for bit-level parity
runs) replace op chains by single kernels with identical semantics:
  * reduce-max / broadcast / subtract / exp / reduce-sum / broadcast /
    divide over the last dim  ->  one row-softmax kernel;
  * dot followed only by relu ->  relu in the GEMM epilogue.

Public functions ``evaluate_single`` / ``evaluate_spmd`` /
``verify_equivalence`` keep the reference signatures
(``simulator.py:304, 393, 438``) and raise the reference's exception classes.
"""

from __future__ import annotations

import ctypes
import dataclasses
from typing import Mapping, Optional, Sequence

import numpy as np

from . import _capi as C
from . import knobs as _knobs
from .ir import (COLLECTIVES, ELEMENTWISE_BINARY, ELEMENTWISE_UNARY,
                 CompareDirection, DType, Graph, Instruction, Op, ReduceKind,
                 Shape, np_dtype)


class EvalError(Exception):
    pass


class DivideByZero(EvalError):
    pass


class SubgroupMismatch(EvalError):
    pass


def _torch():
    import torch
    return torch


def torch_dtype(dt: DType):
    t = _torch()
    return {DType.F32: t.float32, DType.S32: t.int32, DType.U32: t.int32,
            DType.PRED: t.uint8, DType.BF16: t.bfloat16}[dt]


_UNARY = {Op.NEGATE: 0, Op.EXP: 1, Op.RELU: 2}
_BINARY = {Op.ADD: 0, Op.MULTIPLY: 1, Op.MAXIMUM: 2, Op.SUBTRACT: 3,
           Op.DIVIDE: 4, Op.COMPARE: 5}
_CMP = {CompareDirection.EQ: 0, CompareDirection.NE: 1, CompareDirection.LT: 2,
        CompareDirection.LE: 3, CompareDirection.GT: 4, CompareDirection.GE: 5}
_KIND = {ReduceKind.SUM: 0, ReduceKind.MAX: 1, ReduceKind.MIN: 2, ReduceKind.PROD: 3}


def desc(t, shape: Shape) -> C.SpmdTensor:
    """Descriptor of a partition-stacked tensor holding per-partition ``shape``."""
    d = C.SpmdTensor()
    d.data = t.data_ptr()
    d.dtype = C.DTYPE_CODE[shape.dtype]
    d.rank = shape.rank
    for i, n in enumerate(shape.dims):
        d.dims[i] = n
    return d


def _groups_arg(subgroups):
    flat = [d for g in subgroups for d in g]
    sizes = {len(g) for g in subgroups}
    if len(sizes) != 1:
        raise SubgroupMismatch(f"subgroups {subgroups} have unequal sizes")
    return C.i32_array(flat), len(subgroups), sizes.pop()


class NcclComm:
    """Per-process NCCL communicator (world + cached subgroup splits)."""

    def __init__(self, rank: int, world: int, unique_id: Optional[bytes] = None):
        lib = C.lib()
        self.rank, self.world = rank, world
        n = lib.spmd_comm_id_bytes()
        if unique_id is None:
            buf = ctypes.create_string_buffer(n)
            C.check(lib.spmd_comm_get_unique_id(buf), "spmd_comm_get_unique_id")
            unique_id = buf.raw
        self.unique_id = unique_id
        self.handle = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(unique_id, n)
        C.check(lib.spmd_comm_init(ctypes.byref(self.handle), world, rank, idbuf),
                "spmd_comm_init")
        self._ws = None

    @staticmethod
    def from_torch_distributed():
        """Create with the rank/world of ``torch.distributed`` (unique id
        broadcast through its store)."""
        torch = _torch()
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [NcclComm._new_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return NcclComm(rank, world, obj[0])

    @staticmethod
    def _new_id() -> bytes:
        lib = C.lib()
        buf = ctypes.create_string_buffer(lib.spmd_comm_id_bytes())
        C.check(lib.spmd_comm_get_unique_id(buf), "spmd_comm_get_unique_id")
        return buf.raw

    def ensure_workspace(self, nbytes: int, device) -> None:
        torch = _torch()
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            C.check(C.lib().spmd_comm_set_workspace(self.handle, self._ws.data_ptr(),
                                                    self._ws.numel()),
                    "spmd_comm_set_workspace")

    def heap_view(self, offset: int, dims, dtype, device):
        """A tensor aliasing this rank's peer heap at data offset ``offset``
        (the landing zone of a push collective); valid while the heap lives
        and until the zone is rewritten (after a later barrier)."""
        torch = _torch()
        lib = C.lib()
        ptr = lib.spmd_comm_heap_ptr(self.handle, int(offset))
        if not ptr:
            raise EvalError(f"peer heap offset {offset} outside the heap")
        nbytes = int(np.prod(dims)) * dtype.itemsize

        class _Zone:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                        "data": (int(ptr), False), "version": 3}
        raw = torch.as_tensor(_Zone(), device=device)
        return raw.view(torch_dtype(dtype)).view(tuple(dims))

    def reserve_fused(self, half_bytes: int) -> int:
        """Grow the fused-op landing zone to >= ``half_bytes`` per parity
        (peer.cu fused_parity); returns the communicator's H.  Every rank
        compiles the same program, so every rank reserves the same H."""
        lib = C.lib()
        C.check(lib.spmd_comm_reserve_fused(self.handle, int(half_bytes)),
                "spmd_comm_reserve_fused")
        return int(lib.spmd_comm_fused_half(self.handle))

    def ensure_peer(self, nbytes: int, device) -> None:
        """Collective: allocate / grow the CUDA-IPC peer heap used by the
        fused dot -> reduce-scatter kernels (every rank, same size)."""
        torch = _torch()
        lib = C.lib()
        if lib.spmd_comm_peer_bytes(self.handle) >= nbytes:
            return
        s = torch.cuda.current_stream(device).cuda_stream
        C.check(lib.spmd_comm_enable_peer(self.handle, int(nbytes), s), "spmd_comm_enable_peer")

    def close(self):
        if self.handle:
            C.lib().spmd_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()


@dataclasses.dataclass
class Routing:
    """A GShard top-k routing on the device, per local partition:
    ``expert``/``slot`` s32 and ``gate`` f32 of shape ``[P, B, S]`` (top-1)
    or ``[P, B, S, k]`` (slot >= capacity = dropped) -- what
    ``spmd_moe_route`` produces (rule pinned by ``moe.route_topk``).

    Declaring a routing PINS the dispatch / combine masks: the executor's
    dispatch and combine run as gathers driven by these tensors and never
    read the mask parameters' values, so the masks passed to ``run`` must be
    the ones this routing produces (``spmd_moe_masks``).  The tensors are read
    at every run, so updating them in place re-routes the next step."""
    expert: object
    slot: object
    gate: object


@dataclasses.dataclass
class _Step:
    ins: Instruction
    fn: object              # callable(env, stream) -> tensor
    frees: tuple = ()
    ops: tuple = ()         # value ids read
    coll: bool = False      # runs on a comm stream when overlapping
    lane: int = 0           # 0 compute stream, k >= 1: comm stream k - 1
    after: tuple = ()       # extra value ids to wait for (just-in-time prefetch)


class Executor:
    """Compiled per-process runner of one SpmdProgram."""

    def __init__(self, program, nparts: Optional[int] = None, device=None,
                 comm: Optional[NcclComm] = None, partition_base: int = 0,
                 fuse: bool = False, overlap: Optional[bool] = None,
                 routing: Optional[Mapping[int, "Routing"]] = None,
                 knobs: Optional[Mapping[str, object]] = None):
        torch = _torch()
        self.lib = C.lib()
        # plan knobs (knobs.py): environment / overrides, read once here
        self._knobs = _knobs.resolve(knobs)
        # Collectives on a dedicated stream, hoisted to issue as soon as
        # their operands exist (weight all-gathers prefetch under GEMMs).
        self.overlap = (comm is not None) if overlap is None else overlap
        self.program = program
        self.graph: Graph = program.graph
        self.P = int(nparts if nparts is not None else program.num_partitions)
        self.comm = comm
        self.base = partition_base
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.by_id = self.graph.by_id
        self.params = self.graph.parameters
        self.fuse = fuse
        self._consts: dict[str, object] = {}
        self._fused_skip: set[str] = set()
        self._fused: dict[str, object] = {}
        self.routing = dict(routing or {})
        if self.routing:
            self._plan_moe_routing()
        if fuse:
            self._plan_fusions()
        self.steps = self._compile()
        self.comm_stream = None
        self.comm_streams = []
        if self.overlap:
            self.steps = self._hoist_collectives(self.steps)
            prio = int(self._knob("SPMD_COMM_PRIORITY"))
            self.comm_stream = torch.cuda.Stream(device=self.device, priority=prio)
            self.comm_streams = [self.comm_stream]
        if comm is not None:
            comm.ensure_workspace(self._workspace_bytes(), self.device)
            peer = self._peer_bytes()
            self._peer_bytes_used = peer
            if peer:
                comm.ensure_peer(peer, self.device)
        else:
            self._peer_ag = {}
            self._peer_cp = {}
            self._peer_a2a = {}
            self._peer_agp = {}
            self._peer_bytes_used = 0
            self._fused_half = 0
        self._peer_engine = self._plan_peer_engines()
        self._staged_exposed: list = []
        self._act_staged: set = set()
        self._staged = self._plan_staged_gathers()
        if comm is not None:
            self._add_param_push_zones()
        if self.comm_streams:
            self.steps = self._jit_prefetch(self.steps)
        self._sm_limit = self._plan_sm_limit()
        self._assign_lanes()
        self._lane_of = {st.cuda_stream: k + 1 for k, st in enumerate(self.comm_streams)}


    def _knob(self, name: str) -> str:
        return self._knobs[name]
    def _plan_staged_gathers(self) -> dict:
        """Peer all-gathers of parameters (the weight gathers, GSPMD's
        2-D-finalized weight AG over X) -> pre-staged copy-engine pulls
        (engine 4): every weight shard is staged into the peer heap at the
        step start, one barrier follows, and each gather is then only
        copy-engine reads of the members' slots -- no barrier kernel that
        would wait for the SMs a persistent GEMM holds.  A barrier at the
        step end keeps the slots until every member has pulled.
        Returns {all-gather id: parameter index}.  SPMD_PEER_STAGE=0
        disables it."""
        if not self.comm_streams or self._knob("SPMD_PEER_STAGE") == "0":
            return {}
        pids = [p.id for p in self.params]
        staged = {}
        wide = self._knob("SPMD_PEER_STAGE_WIDE") == "1"
        # exposed parameter gathers: pushed from the parameter itself
        # (peer_push_kernel, 661 / 677 GB/s per GPU at N=2 / 4 vs 463 / 342
        # for staged pulls: profiles/r2_bench_n{2,4}_final.log) unless
        # SPMD_PEER_AG_PUSH_PARAMS=0
        push_params = self._knob("SPMD_PEER_AG_PUSH") != "0" and \
            self._knob("SPMD_PEER_AG_PUSH_PARAMS") != "0"
        # activation staging measured slower (profiles/r1_c2_n4_ab_stage_act.log)
        act = self._knob("SPMD_PEER_STAGE_ACT") == "1"
        for aid in self._peer_ag:
            src = self.by_id[self.by_id[aid].operands[0]]
            if src.opcode != Op.PARAMETER:
                if act:
                    # activation gathers: staged on the compute stream right
                    # after the producer (copy + barrier while no GEMM runs),
                    # then copy-engine pulls on the critical lane
                    self._act_staged.add(aid)
                    self._peer_engine[aid] = 4
                continue
            if push_params and self._peer_engine.get(aid, -1) not in (0, 3):
                continue                          # exposed: push engine (1 / -1)
            if wide and self._peer_engine.get(aid, -1) < 0:
                self._peer_engine[aid] = 1        # exposed NCCL gather -> staged pulls too
            if self._peer_engine.get(aid, -1) >= 0:
                staged[aid] = pids.index(src.id)
                if self._peer_engine[aid] not in (0, 3):
                    self._staged_exposed.append(aid)
                self._peer_engine[aid] = 4
        return staged

    def _add_param_push_zones(self) -> None:
        """Parameter all-gathers left on the critical path (engine 1 / -1:
        not staged, _plan_staged_gathers) -- C5's replicate reshard, a
        step's first x / weight gathers -- get a push landing zone after the
        heap regions _peer_bytes laid out; every member pushes its shard
        straight from the parameter (spmd_peer_push_all_gather)."""
        if self._knob("SPMD_PEER_AG_PUSH") == "0" or \
                self._knob("SPMD_PEER_AG_PUSH_PARAMS") == "0":
            return
        pids = {p.id for p in self.params}
        off = self._peer_bytes_used
        for ins in self.graph.instructions:
            if ins.opcode == Op.ALL_GATHER and ins.id not in self._fused_skip and \
                    ins.id not in self._peer_agp and ins.operands[0] in pids and \
                    self._peer_engine.get(ins.id, 0) in (1, -1):
                self._peer_agp[ins.id] = off
                off += (ins.shape.nbytes + 4095) // 4096 * 4096
        if off != self._peer_bytes_used:
            self._peer_bytes_used = off
            self.comm.ensure_peer(off, self.device)

    def _stage_phases(self) -> list:
        """Staging order: exposed gathers' shards, then the rest
        (SPMD_STAGE_PHASES=1: one phase)."""
        if self._knob("SPMD_STAGE_PHASES") == "1":
            return [list(self._staged)]
        first = [a for a in self._staged if a in self._staged_exposed]
        rest = [a for a in self._staged if a not in self._staged_exposed]
        return [p for p in (first, rest) if p]

    def _plan_sm_limit(self) -> int:
        """GEMM/conv SM budget while this executor runs (0 = every SM).

        The persistent tcgen05 GEMM holds every SM (one CTA with the whole
        register file each), so a kernel queued on a comm lane -- the peer
        barrier that brackets every copy-engine gather, or an NCCL kernel --
        cannot start until the GEMM ends: a 256 MB pair gather under GEMMs
        took 5.7 ms instead of 0.9 ms (profiles/r1_gather_under_gemm.jsonl).
        With overlapped collectives the GEMM leaves SPMD_COMM_SMS SMs to
        them (default 2; 0 when the weight gathers are pre-staged and need
        no kernel, since a reserved pair costs a GEMM whose tile count is a
        multiple of 74 pairs up to one extra tile round)."""
        if not self.comm_streams or self.comm is None or \
                not any(st.coll for st in self.steps):
            return 0
        reserve = int((self._knob("SPMD_COMM_SMS") or ("0" if self._staged else "2")))
        if reserve <= 0:
            return 0
        sms = _torch().cuda.get_device_properties(self.device).multi_processor_count
        return max(2, sms - reserve)

    def _jit_prefetch(self, steps: list) -> list:
        """Background prefetch gathers (peer engines 0/3) move from "as early
        as the operands exist" to just before the heavy compute step
        SPMD_PREFETCH_DEPTH GEMMs ahead of their first consumer, and start only
        when that GEMM can start.  They no longer pile up at the start of the
        step, where they compete for NVLink with the critical gathers (at C2
        2x2 the first critical gather took 0.50 instead of ~0.17 ms,
        profiles/r1_timeline_c2_n4_wide.log).  SPMD_PREFETCH=asap keeps the
        hoisted order."""
        if self._knob("SPMD_PREFETCH") == "asap":
            return steps
        # GEMMs ahead: 2 measured best at C2 2x2 (15.28 ms vs 15.76 for 1 and
        # 15.56-16.81 for as-soon-as-possible, profiles/r1_c2_n4_ab_wide_lanes_engines.log)
        depth = max(1, int(self._knob("SPMD_PREFETCH_DEPTH")))
        heavy_ops = (Op.DOT, Op.CONVOLUTION)
        heavy_fused = ("dot_relu", "conv_relu", "attention", "dot_rs", "dot_a2a", "halo_conv",
                       "dot_add", "dot_rs_add")

        def heavy(st):
            f = self._fused.get(st.ins.id)
            return not st.coll and (st.ins.opcode in heavy_ops or
                                    (f is not None and f[0] in heavy_fused))
        order = list(steps)
        for g in [st for st in order if st.coll and self._peer_engine.get(st.ins.id, -1) in (0, 3)]:
            i = order.index(g)
            first = next((k for k in range(i + 1, len(order)) if g.ins.id in order[k].ops), None)
            if first is None:
                continue
            hs = [k for k in range(first - 1, i, -1) if heavy(order[k])][:depth]
            h = hs[-1] if hs else None
            if h is None or h <= i + 1:
                continue
            # start when the GEMM it rides under can start: wait for that
            # GEMM's operands too
            g.after = tuple(o for o in order[h].ops if o not in g.ops)
            order.pop(i)
            order.insert(h - 1, g)     # h shifted down by one after the pop
        last_use = {}
        for k, st in enumerate(order):
            for o in st.ops:
                last_use[o] = k
        keep = set(self.graph.outputs)
        for k, st in enumerate(order):
            st.frees = tuple(o for o in set(st.ops) if last_use.get(o) == k and o not in keep)
        return order

    def _assign_lanes(self) -> None:
        """Collectives on comm lanes.  Lane 1 carries only the background
        prefetch gathers (peer copy-engine / background SM-pull engines: a
        GEMM hides them) and the pre-staged weight gathers (copy-engine reads
        only, in program order after the staging barrier, so the first one
        overlaps the activation gather on lane 2); everything on the critical
        path -- exposed peer
        gathers and every NCCL call (one stream, so NCCL's per-communicator
        order is the same on all ranks) -- takes lane 2 with its own barrier
        channel, so it never queues behind a prefetch.  At C2 N=4 the res1
        gather otherwise waited 1.6 ms behind the w_out prefetch
        (profiles/r1_timeline_c2_n4_wide.log).  SPMD_COMM_LANES=1: one lane;
        =2: alternate all peer gathers (measured slower); default "critical".
        """
        if not self.comm_streams:
            return
        mode = self._knob("SPMD_COMM_LANES")
        nxt = 0
        npush = ncp = 0
        pids = {p.id for p in self.params}
        for st in self.steps:
            if not st.coll:
                continue
            st.lane = 1
            eng = self._peer_engine.get(st.ins.id, -1)
            if mode == "2" and eng >= 0:
                st.lane = 1 + nxt
                nxt = (nxt + 1) % 2
            elif mode == "critical" and st.ins.id in self._act_staged:
                st.lane = 2
            elif mode == "critical" and eng == 4 and st.ins.id in self._staged_exposed:
                # exposed staged gathers wait only for the first staging phase;
                # they alternate lanes 2 and 3, so e.g. the x and w_q pulls
                # before the first GEMM run on two copy engines at once (one
                # lane serialised them: 0.29 + 0.32 ms exposed at 2x2,
                # profiles/r2_timeline_c2_2x2.log).  SPMD_STAGE_PHASES=1:
                # alternate lanes 2 and 1 (round 1)
                k = self._staged_exposed.index(st.ins.id) % 2
                if self._knob("SPMD_STAGE_PHASES") == "1":
                    st.lane = 2 - k
                else:
                    st.lane = 2 + (k if self._knob("SPMD_EXPOSED_SPLIT") != "0" else 0)
            elif mode == "critical" and eng in (1, -1) and st.ins.id in self._peer_agp and \
                    self.by_id[st.ins.id].operands[0] in pids:
                # exposed parameter gathers on the push engine (the step's
                # first x and w_q gathers): lanes 2 and 3 alternate so they
                # run at once (one lane serialised them: 0.35 + 0.32 ms before
                # the first GEMM at 2x2, profiles/r2_timeline_c2_n4_push.log;
                # concurrent: first GEMM 0.12 ms earlier in the eager
                # timeline, r2_timeline_c2_n4_lanes.log; graph-replayed step
                # within noise, 13.67 vs 13.71 ms: r2_ab_exposed_split_push.log)
                st.lane = 2 + (npush % 2 if self._knob("SPMD_EXPOSED_SPLIT") != "0"
                               else 0)
                npush += 1
            elif mode == "critical" and st.ins.opcode == Op.COLLECTIVE_PERMUTE and \
                    st.ins.id in self._peer_cp:
                # halo exchanges: a conv layer's left and right slab permutes
                # go out on lanes 2 and 3 at once (one lane ran them back to
                # back, ~0.03 ms each per layer at C4 N=4:
                # profiles/r2_timeline_c4_n4.log)
                st.lane = 2 + (ncp % 2 if self._knob("SPMD_EXPOSED_SPLIT") != "0"
                               else 0)
                ncp += 1
            elif mode == "critical" and eng not in (0, 3, 4):
                st.lane = 2
        torch = _torch()
        for lane in (2, 3):
            if any(st.lane >= lane for st in self.steps if st.coll) and \
                    len(self.comm_streams) < lane:
                self.comm_streams.append(torch.cuda.Stream(device=self.device,
                                                           priority=self.comm_stream.priority))

    def _shape(self, vid: str) -> Shape:
        return self.by_id[vid].shape

    def _alloc(self, shape: Shape):
        torch = _torch()
        return torch.empty((self.P,) + shape.dims, dtype=torch_dtype(shape.dtype),
                           device=self.device)

    def _peer_bytes(self) -> int:
        """Peer heap: [0, 3H) the fused-op landing zone (H = per-parity bytes
        of the largest fused dot -> reduce-scatter / all-to-all / MoE
        dispatch, reserved on the communicator so every executor sharing it
        uses the same parity stride: peer.cu fused_parity), then one staging
        slot per peer all-gather and one landing slot per peer permute
        (offsets recorded in ``self._peer_ag`` / ``self._peer_cp``)."""
        half = 0
        for spec in self._fused.values():
            if spec[0] in ("dot_rs", "dot_rs_add"):
                rs = spec[2]
                half = max(half, rs.shape.num_elements * len(rs.attrs["subgroups"][0]) *
                           rs.shape.dtype.itemsize)
            elif spec[0] == "dot_a2a":
                half = max(half, spec[2].shape.num_elements * spec[2].shape.dtype.itemsize)
            elif spec[0] == "moe_dispatch_a2a":
                half = max(half, spec[3].shape.num_elements * spec[3].shape.dtype.itemsize)
        if self.comm is not None:
            half = self.comm.reserve_fused(half)
        self._fused_half = half
        off = 3 * half
        self._peer_ag = {}
        if self._knob("SPMD_PEER_AG") != "0":
            for ins in self.graph.instructions:
                if ins.opcode == Op.ALL_GATHER and ins.id not in self._fused_skip:
                    self._peer_ag[ins.id] = off
                    nb = self._shape(ins.operands[0]).num_elements * ins.shape.dtype.itemsize
                    off += (nb + 4095) // 4096 * 4096
        # push all-gathers: gathers of computed values (parameters are
        # pre-staged) get a landing zone holding the whole output; every
        # member pushes its shard into every zone.  Used for the gathers on
        # the critical path (engine 1 / NCCL), where SMs are free: 652 vs 475
        # (pull) vs 467 (NCCL) GB/s per GPU at N=2 (profiles/r2_bench_n2.log);
        # gathers hidden under a GEMM keep the copy engines.
        # (parameter gathers left on the critical path get theirs later,
        # _add_param_push_zones, once the engines are planned)
        self._peer_agp = {}
        if self._knob("SPMD_PEER_AG_PUSH") != "0":
            pids = {p.id for p in self.params}
            for ins in self.graph.instructions:
                if ins.opcode == Op.ALL_GATHER and ins.id not in self._fused_skip and \
                        ins.operands[0] not in pids:
                    self._peer_agp[ins.id] = off
                    off += (ins.shape.nbytes + 4095) // 4096 * 4096
        # all-to-alls (C5 resharding; MoE exchanges not fused into a GEMM):
        # one landing zone each, holding this rank's output -- every member
        # pushes its piece there (spmd_peer_all_to_all), and the zone is the
        # value the consumers read
        self._peer_a2a = {}
        if self._knob("SPMD_PEER_A2A") != "0":
            for ins in self.graph.instructions:
                if ins.opcode == Op.ALL_TO_ALL and ins.id not in self._fused_skip and \
                        ins.id not in self._fused:
                    self._peer_a2a[ins.id] = off
                    off += (ins.shape.nbytes + 4095) // 4096 * 4096
        # collective-permutes (halo exchanges, pipeline shifts): one landing
        # slot each, written by the source rank's copy engine
        self._peer_cp = {}
        if self._knob("SPMD_PEER_CP") != "0":
            for ins in self.graph.instructions:
                if ins.opcode == Op.COLLECTIVE_PERMUTE and ins.id not in self._fused_skip:
                    self._peer_cp[ins.id] = off
                    nb = ins.shape.num_elements * ins.shape.dtype.itemsize
                    off += (nb + 4095) // 4096 * 4096
        return off

    def _plan_peer_engines(self) -> dict:
        """Copy engines (0) for peer all-gathers that a GEMM hides on the
        compute stream (no SMs taken from it); for the ones on the critical
        path (no dot / convolution issued between the gather and its first
        consumer) the SM pull kernel (1) for pairs and NCCL (-1) for larger
        groups, where its NVLink-multicast all-gather out-runs point-to-point
        pulls (profiles/r1_peer_ag_bench_n4.jsonl).  SPMD_PEER_AG_ENGINE=ce|sm
        forces one."""
        force = self._knob("SPMD_PEER_AG_ENGINE")
        # hidden gathers: copy engines (0), background SM pull (3) or NCCL (-1)
        hidden_mode = self._knob("SPMD_PEER_HIDDEN_ENGINE")
        heavy_ops = (Op.DOT, Op.CONVOLUTION)
        heavy_fused = ("dot_relu", "conv_relu", "attention", "dot_rs", "dot_a2a", "dot_add",
                       "dot_rs_add")
        eng = {}
        order = self.steps
        for i, st in enumerate(order):
            if st.ins.id not in self._peer_ag:
                continue
            if force in ("ce", "sm"):
                eng[st.ins.id] = 0 if force == "ce" else 1
                continue
            hidden = False
            if self.comm_stream is not None:
                for nxt in order[i + 1:]:
                    if st.ins.id in nxt.ops:
                        break
                    f = self._fused.get(nxt.ins.id)
                    if not nxt.coll and (nxt.ins.opcode in heavy_ops or
                                         (f is not None and f[0] in heavy_fused)):
                        hidden = True
                        break
            gs = len(st.ins.attrs["subgroups"][0])
            if hidden:
                # copy engines move contiguous pieces well; a gather along an
                # inner dim is a 2-D copy of many short rows (slow on the
                # copy engines): "mixed" sends those to the background SM pull
                leading = all(d == 1 for d in self._shape(st.ins.operands[0]).dims[
                    :st.ins.attrs["dim"]])
                eng[st.ins.id] = {"ce": 0, "sm": 3, "nccl": -1}.get(
                    hidden_mode, 0 if leading else 3)
            else:
                eng[st.ins.id] = 1 if gs <= 2 else -1
        return eng

    def _workspace_bytes(self) -> int:
        need = 0
        for ins in self.graph.instructions:
            if ins.opcode in COLLECTIVES and ins.opcode != Op.COLLECTIVE_PERMUTE:
                src = self._shape(ins.operands[0])
                n = max(src.num_elements, ins.shape.num_elements)
                need = max(need, 2 * n * ins.shape.dtype.itemsize)
        return need

    # ------------------------------------------------------------------
    # fusion planning
    # ------------------------------------------------------------------
    def _users(self):
        users: dict[str, list[str]] = {}
        for ins in self.graph.instructions:
            for o in ins.operands:
                users.setdefault(o, []).append(ins.id)
        return users

    def _plan_fusions(self):
        users = self._users()
        outs = set(self.graph.outputs)
        by = self.by_id

        def only_user(vid, op):
            u = users.get(vid, [])
            return len(u) == 1 and by[u[0]].opcode == op and vid not in outs

        def const_value(vid):
            c = by[vid]
            if c.opcode != Op.CONSTANT:
                return None
            lit = np.asarray(c.attrs["literal"])
            return float(lit) if lit.size == 1 else None

        for ins in self.graph.instructions:
            # softmax: e=exp(x - bcast(max(x))); e / bcast(sum(e))
            if ins.opcode == Op.REDUCE and ins.attrs["kind"] == ReduceKind.MAX \
                    and ins.shape.dtype.is_float:
                x = ins.operands[0]
                xs = self._shape(x)
                if tuple(ins.attrs["dims"]) != (xs.rank - 1,) or const_value(ins.operands[1]) != -np.inf:
                    continue
                if not only_user(ins.id, Op.BROADCAST):
                    continue
                mxb = by[users[ins.id][0]]
                if tuple(mxb.attrs["broadcast_dims"]) != tuple(range(xs.rank - 1)):
                    continue
                if not only_user(mxb.id, Op.SUBTRACT):
                    continue
                sub = by[users[mxb.id][0]]
                if sub.operands != (x, mxb.id) or not only_user(sub.id, Op.EXP):
                    continue
                e = by[users[sub.id][0]]
                eu = users.get(e.id, [])
                if len(eu) != 2 or e.id in outs:
                    continue
                red = [by[u] for u in eu if by[u].opcode == Op.REDUCE]
                div = [by[u] for u in eu if by[u].opcode == Op.DIVIDE]
                if len(red) != 1 or len(div) != 1:
                    continue
                red, div = red[0], div[0]
                if red.attrs["kind"] != ReduceKind.SUM or tuple(red.attrs["dims"]) != (xs.rank - 1,) \
                        or red.operands[0] != e.id or const_value(red.operands[1]) != 0.0:
                    continue
                if not only_user(red.id, Op.BROADCAST):
                    continue
                denb = by[users[red.id][0]]
                if tuple(denb.attrs["broadcast_dims"]) != tuple(range(xs.rank - 1)):
                    continue
                if div.operands != (e.id, denb.id) or len(users.get(denb.id, [])) != 1:
                    continue
                for vid in (ins.id, mxb.id, sub.id, e.id, red.id, denb.id):
                    self._fused_skip.add(vid)
                self._fused[div.id] = ("softmax", x)
            # partitioner select_range chain -> one range-mask kernel
            if ins.opcode == Op.SELECT and ins.id not in self._fused_skip:
                m = self._match_range_mask(ins, users, outs)
                if m is not None:
                    result, skip, spec = m
                    self._fused_skip.update(skip)
                    self._fused[result] = spec
                    continue
            # dot / convolution -> relu epilogue
            if ins.opcode in (Op.DOT, Op.CONVOLUTION) and only_user(ins.id, Op.RELU) \
                    and ins.shape.dtype == DType.BF16 and ins.id not in self._fused:
                relu = by[users[ins.id][0]]
                self._fused_skip.add(ins.id)
                self._fused[relu.id] = ("dot_relu" if ins.opcode == Op.DOT else "conv_relu", ins)
            # transpose -> relu: one pass (the MoE layer's reshard annotations)
            if ins.opcode == Op.TRANSPOSE and only_user(ins.id, Op.RELU) and \
                    ins.shape.dtype in (DType.F32, DType.BF16, DType.S32) and \
                    ins.id not in self._fused and ins.id not in self._fused_skip and \
                    self._knob("SPMD_TRANSPOSE_RELU") != "0":
                relu = by[users[ins.id][0]]
                src = self._fused.get(ins.operands[0])
                if relu.id in self._fused:
                    pass
                elif src is not None and src[0] == "moe_dispatch" and len(src) == 3 and \
                        tuple(ins.attrs["permutation"]) == (1, 0, 2, 3) and \
                        only_user(ins.operands[0], Op.TRANSPOSE):
                    # dispatch -> Transpose(1,0,2,3) -> ReLU: the gather writes
                    # [E,B,C,M] rows with the ReLU applied (no extra pass)
                    self._fused_skip.update((ins.operands[0], ins.id))
                    del self._fused[ins.operands[0]]
                    self._fused[relu.id] = ("moe_dispatch", src[1], src[2], 3)
                else:
                    self._fused_skip.add(ins.id)
                    self._fused[relu.id] = ("transpose_relu", ins)
            # loopback all-gathers -> f32 Dot: a gathered lhs (K-major) comes
            # as tf32 hi / lo halves, a gathered 2-D rhs [K, N] (along K) as the
            # halves of its K-major transpose; the 3xTF32 GEMM skips those
            # split passes
            if ins.opcode == Op.DOT and self.comm is None and ins.shape.dtype == DType.F32 and \
                    ins.id not in self._fused and ins.id not in self._fused_skip and \
                    ins.operands[0] != ins.operands[1] and \
                    self._knob("SPMD_AG_SPLIT") != "0":
                def gathered(vid):
                    a = by[vid]
                    return a if a.opcode == Op.ALL_GATHER and a.shape.dtype == DType.F32 and \
                        only_user(vid, Op.DOT) and vid not in self._fused_skip else None
                lag, rag = gathered(ins.operands[0]), gathered(ins.operands[1])
                at = ins.attrs
                if rag is not None and not (rag.shape.rank == 2 and rag.attrs["dim"] == 0 and
                                            not at["rhs_batch"] and
                                            tuple(at["rhs_contracting"]) == (0,)):
                    rag = None
                if lag is not None or rag is not None:
                    for a in (lag, rag):
                        if a is not None:
                            self._fused_skip.add(a.id)
                    self._fused[ins.id] = ("ag_split_dot", lag, rag, ins)
            # dot -> residual add: the add runs in the GEMM epilogue (fp32,
            # one rounding); falls back to dot + add if the wide GEMM does
            # not take it
            if ins.opcode == Op.ADD and ins.shape.dtype == DType.BF16 and \
                    ins.id not in self._fused and \
                    self._knob("SPMD_DOT_ADD") != "0":
                for k in (0, 1):
                    d, r = ins.operands[k], ins.operands[1 - k]
                    dot = by[d]
                    if dot.opcode == Op.DOT and dot.shape == ins.shape and \
                            by[r].shape == ins.shape and d != r and \
                            only_user(d, Op.ADD) and d not in self._fused and \
                            d not in self._fused_skip:
                        self._fused_skip.add(d)
                        self._fused[ins.id] = ("dot_add", dot, r)
                        break
        # Transpose(1,0,2,3) -> ReLU -> combine gather: the gather reads the
        # [E,B,C,M] expert outputs and applies the ReLU itself
        for cid, spec in list(self._fused.items()):
            if spec[0] != "moe_combine" or len(spec) != 3:
                continue
            tr = self._fused.get(spec[1])
            if tr is None or tr[0] != "transpose_relu" or spec[1] in outs or \
                    tuple(tr[1].attrs["permutation"]) != (1, 0, 2, 3) or \
                    len(users.get(spec[1], [])) != 1:
                continue
            self._fused_skip.add(spec[1])
            del self._fused[spec[1]]
            self._fused[cid] = ("moe_combine", tr[1].operands[0], spec[2], 3)
        self._plan_backward(users, outs, only_user, const_value)
        self._plan_halo_windows(users, outs)
        self._plan_halo_convs(users, outs)
        self._plan_attention(users, outs)
        self._plan_dot_reduce_scatter(users, outs)
        self._plan_rs_residual_adds(users, outs)
        self._plan_slice_permutes(users, outs)

    def _plan_rs_residual_adds(self, users, outs):
        """Fused dot -> reduce-scatter whose only user is the layer's residual
        Add: the add runs in the reduce-scatter's slot reduce
        (spmd_dot_reduce_scatter_add, same roundings as unfused).
        SPMD_RS_ADD=0 disables it."""
        if self._knob("SPMD_RS_ADD") == "0":
            return
        by = self.by_id
        for add in self.graph.instructions:
            if add.opcode != Op.ADD or add.shape.dtype != DType.BF16 or add.id in self._fused:
                continue
            for k in (0, 1):
                rsid, r = add.operands[k], add.operands[1 - k]
                spec = self._fused.get(rsid)
                if spec is None or spec[0] != "dot_rs" or rsid in outs or r == rsid or \
                        len(users.get(rsid, [])) != 1 or by[r].shape != add.shape:
                    continue
                del self._fused[rsid]
                self._fused_skip.add(rsid)
                self._fused[add.id] = ("dot_rs_add", spec[1], spec[2], r)
                break

    def _plan_backward(self, users, outs, only_user, const_value):
        """Training-step backward chains (workloads.transformer_train_step):

        * softmax backward ``p * (dp - bcast(sum_t(dp * p)))`` -> one row
          kernel (spmd_softmax_backward_lastdim), bf16/f32, full rows local;
        * ReLU backward ``select(h > bcast(0), g, bcast(0))`` -> one
          elementwise kernel (spmd_relu_backward).  When ``h`` is a bf16 DOT
          whose other user is its forward RELU, the DOT takes the ReLU
          epilogue and the mask reads ``relu(h) > 0`` (the same predicate,
          NaN included) so ``h`` is never written.
        SPMD_BWD_FUSION=0 disables both."""
        if self._knob("SPMD_BWD_FUSION") == "0":
            return
        by = self.by_id

        def zero_bcast(vid):
            z = by.get(vid)
            return z is not None and z.opcode == Op.BROADCAST and \
                tuple(z.attrs["broadcast_dims"]) == () and const_value(z.operands[0]) == 0.0

        taken = lambda vid: vid in self._fused or vid in self._fused_skip
        for ins in self.graph.instructions:
            if ins.opcode == Op.REDUCE and ins.attrs["kind"] == ReduceKind.SUM \
                    and ins.shape.dtype in (DType.BF16, DType.F32) and not taken(ins.id):
                pdp = by[ins.operands[0]]
                rank = pdp.shape.rank
                if pdp.opcode != Op.MULTIPLY or tuple(ins.attrs["dims"]) != (rank - 1,) \
                        or const_value(ins.operands[1]) != 0.0 or not only_user(pdp.id, Op.REDUCE) \
                        or not only_user(ins.id, Op.BROADCAST) or taken(pdp.id):
                    continue
                spb = by[users[ins.id][0]]
                if tuple(spb.attrs["broadcast_dims"]) != tuple(range(rank - 1)) \
                        or not only_user(spb.id, Op.SUBTRACT):
                    continue
                sub = by[users[spb.id][0]]
                dp = sub.operands[0]
                if sub.operands[1] != spb.id or dp not in pdp.operands \
                        or not only_user(sub.id, Op.MULTIPLY):
                    continue
                p = pdp.operands[1] if pdp.operands[0] == dp else pdp.operands[0]
                mul = by[users[sub.id][0]]
                if sorted(mul.operands) != sorted((p, sub.id)) or p == dp or taken(mul.id) \
                        or self._shape(p) != self._shape(dp):
                    continue
                self._fused_skip.update((pdp.id, ins.id, spb.id, sub.id))
                self._fused[mul.id] = ("softmax_bwd", p, dp)
            elif ins.opcode == Op.SELECT and not taken(ins.id):
                pred, g, z = ins.operands
                cmp = by[pred]
                if cmp.opcode != Op.COMPARE or cmp.attrs["direction"].name != "GT" \
                        or not only_user(pred, Op.SELECT) or not zero_bcast(z) \
                        or not zero_bcast(cmp.operands[1]) or taken(pred):
                    continue
                h = by[cmp.operands[0]]
                if h.shape.dtype not in (DType.BF16, DType.F32) or self._shape(g) != h.shape:
                    continue
                skip = {pred}
                for zid in {z, cmp.operands[1]}:
                    if zid not in outs and all(u in (pred, ins.id) for u in users[zid]):
                        skip.add(zid)
                src = h.id
                hu = [by[u] for u in users.get(h.id, [])]
                if h.opcode == Op.DOT and h.shape.dtype == DType.BF16 and h.id not in outs \
                        and not taken(h.id) and len(hu) == 2 \
                        and {u.opcode for u in hu} == {Op.RELU, Op.COMPARE}:
                    relu = next(u for u in hu if u.opcode == Op.RELU)
                    if not taken(relu.id):
                        self._fused_skip.add(h.id)
                        self._fused[relu.id] = ("dot_relu", h)
                        src = relu.id
                self._fused_skip.update(skip)
                self._fused[ins.id] = ("relu_bwd", src, g)

    def _plan_slice_permutes(self, users, outs):
        """Slice (one dim, stride 1) -> CollectivePermute, the slice's only
        user: the halo slab of a spatially partitioned conv
        (formatting.py:54-182 exchange_and_slice).  With a multi-process
        communicator the peer permute writes the slab rows straight from the
        sliced tensor (spmd_peer_slice_collective_permute)."""
        if self.comm is None or self.P != 1 or self._knob("SPMD_PEER_CP") == "0":
            return
        by = self.by_id
        for cp in self.graph.instructions:
            if cp.opcode != Op.COLLECTIVE_PERMUTE or cp.id in self._fused:
                continue
            sl = by[cp.operands[0]]
            if sl.opcode != Op.SLICE or sl.id in outs or users.get(sl.id) != [cp.id] \
                    or sl.id in self._fused or sl.id in self._fused_skip:
                continue
            src = self._shape(sl.operands[0])
            a = sl.attrs
            cut = [d for d in range(src.rank)
                   if (a["starts"][d], a["limits"][d]) != (0, src.dims[d])]
            if len(cut) != 1 or any(x != 1 for x in a["strides"]):
                continue
            self._fused_skip.add(sl.id)
            self._fused[cp.id] = ("slice_cp", sl, cp, cut[0])

    def _conv_tc_eligible(self, conv) -> bool:
        """The NHWC/HWIO bf16 shapes conv_tcgen05 takes (conv_tcgen05.cu)."""
        cd, win = conv.attrs["conv_dims"], conv.attrs["window"]
        ls, rs = self._shape(conv.operands[0]), self._shape(conv.operands[1])
        if ls.dtype != DType.BF16 or ls.rank != 4 or len(win) != 2:
            return False
        layout = (cd.lhs_batch, tuple(cd.lhs_spatial), cd.lhs_feature, tuple(cd.rhs_spatial),
                  cd.rhs_in_feature, cd.rhs_out_feature, cd.out_batch, tuple(cd.out_spatial),
                  cd.out_feature)
        if layout != (0, (1, 2), 3, (0, 1), 2, 3, 0, (1, 2), 3):
            return False
        if any(w.stride != 1 or w.base_dilation != 1 or w.window_dilation != 1 for w in win):
            return False
        # Cout tiles of 128 or 256 channels (conv_tcgen05.cu BN)
        return ls.dims[3] % 64 == 0 and rs.dims[3] % 128 == 0 and conv.shape.dims[2] >= 64

    def _plan_halo_convs(self, users, outs):
        """Halo window along H whose only user is a tcgen05-eligible conv ->
        the conv reads the window rows straight from the halo pieces (no
        window buffer; unpack bytes 0 when fused into the conv
        loader).  Needs a zero mask fill (masked rows load as TMA zeros).
        SPMD_HALO_CONV=0 disables it."""
        if self._knob("SPMD_HALO_CONV") == "0":
            return
        by = self.by_id
        for ds_id, spec in list(self._fused.items()):
            if spec[0] != "halo" or ds_id in outs:
                continue
            _, pieces, axis, start, mask = spec
            u = users.get(ds_id, [])
            if len(u) != 1 or by[u[0]].opcode != Op.CONVOLUTION:
                continue
            conv = by[u[0]]
            if conv.operands[0] != ds_id or axis != 1 or not self._conv_tc_eligible(conv):
                continue
            if mask is not None:
                fill = by.get(mask[3])
                lit = np.asarray(fill.attrs["literal"]) if fill is not None and \
                    fill.opcode == Op.CONSTANT else None
                if lit is None or lit.size != 1 or float(lit) != 0.0:
                    continue
            relu = [k for k, v in self._fused.items() if v[0] == "conv_relu" and v[1] is conv]
            del self._fused[ds_id]
            self._fused_skip.add(ds_id)
            entry = ("halo_conv", conv, 1 if relu else 0, spec, ds_id)
            if relu:
                self._fused[relu[0]] = entry
            else:
                self._fused[conv.id] = entry

    def _plan_moe_routing(self):
        """GShard dispatch / combine einsums over a declared one-hot routing
        (``routing[param_index] = Routing(expert, slot, gate)``) run as the
        gather kernels of moe.cu.  Every dispatch output element has a single
        nonzero term and every combine output at most k (one per choice), so
        the results equal the dense Dot as the reference evaluates it
        (tests/test_acceptance.py:326-349 consumes the same masks through a
        Dot; f64 accumulation, simulator.py:258-275).  The mask parameters'
        values are not read (see ``Routing``)."""
        pidx = {p.id: p.attrs["index"] for p in self.params}
        for ins in self.graph.instructions:
            if ins.opcode != Op.DOT or ins.shape.dtype != DType.BF16:
                continue
            mask, other = ins.operands
            if pidx.get(mask) not in self.routing:
                continue
            a = ins.attrs
            dims = (tuple(a["lhs_batch"]), tuple(a["rhs_batch"]), tuple(a["lhs_contracting"]),
                    tuple(a["rhs_contracting"]))
            if dims == ((0,), (0,), (1,), (1,)) and self._shape(other).rank == 3:
                self._fused[ins.id] = ("moe_dispatch", other, pidx[mask])
            elif dims == ((0,), (0,), (2, 3), (1, 2)) and self._shape(other).rank == 4:
                self._fused[ins.id] = ("moe_combine", other, pidx[mask])

    def _plan_dot_reduce_scatter(self, users, outs):
        """Dot whose only user is a sum reduce-scatter of its last dim (the
        rhs free dim) -> one GEMM with a peer-store epilogue (peer.cu).  Only
        with a multi-process communicator; SPMD_PEER_FUSION=0 disables."""
        if self.comm is None or self._knob("SPMD_PEER_FUSION") == "0":
            return
        by = self.by_id
        for rs in self.graph.instructions:
            if rs.opcode != Op.REDUCE_SCATTER or rs.attrs["kind"] != ReduceKind.SUM:
                continue
            d = by.get(rs.operands[0])
            if d is None or d.opcode != Op.DOT or d.id in outs or d.id in self._fused_skip \
                    or users.get(d.id, []) != [rs.id] or d.shape.dtype != DType.BF16:
                continue
            groups = rs.attrs["subgroups"]
            gs = len(groups[0])
            if any(len(g) != gs for g in groups) or gs > 8:
                continue
            a = d.attrs
            ls, rsh = self._shape(d.operands[0]), self._shape(d.operands[1])
            if a["lhs_batch"] or a["rhs_batch"]:
                continue
            lfree = [k for k in range(ls.rank) if k not in a["lhs_contracting"]]
            rfree = [k for k in range(rsh.rank) if k not in a["rhs_contracting"]]
            m = int(np.prod([ls.dims[k] for k in lfree]))
            n = int(np.prod([rsh.dims[k] for k in rfree]))
            if rs.attrs["dim"] == d.shape.rank - 1:
                # column split: the last output dim is the whole GEMM N
                if [rsh.dims[k] for k in rfree if rsh.dims[k] != 1] != [d.shape.dims[-1]]:
                    continue
                if m < 256 or n < 256 or n % gs or (n // gs) % 32:
                    continue
            elif rs.attrs["dim"] == 0 and lfree and d.shape.rank >= 2:
                # row split (wide GEMM): the leading output dim leads the rows
                if m < 256 or n < 512 or m % gs or (m // gs) % 32 or \
                        d.shape.dims[0] % gs:
                    continue
            else:
                continue
            self._fused_skip.add(d.id)
            self._fused[rs.id] = ("dot_rs", d, rs)
        # routed dispatch -> all-to-all(split 1, concat 0): push rows into the
        # owners' heaps (peer.cu spmd_moe_dispatch_all_to_all)
        for a2a in self.graph.instructions:
            if a2a.opcode != Op.ALL_TO_ALL or a2a.attrs["split_dim"] != 1 or \
                    a2a.attrs["concat_dim"] != 0:
                continue
            spec = self._fused.get(a2a.operands[0])
            if spec is None or spec[0] != "moe_dispatch" or a2a.operands[0] in outs or \
                    users.get(a2a.operands[0], []) != [a2a.id]:
                continue
            groups = a2a.attrs["subgroups"]
            if any(len(g) != len(groups[0]) for g in groups) or len(groups[0]) > 8:
                continue
            self._fused_skip.add(a2a.operands[0])
            self._fused[a2a.id] = ("moe_dispatch_a2a", spec[1], spec[2], a2a)
        # Dot (one batch dim) -> all-to-all(split 1, concat 0): the expert
        # FFN-out einsum + GShard combine exchange (C3) -> wide GEMM with a
        # row-scatter epilogue (peer.cu spmd_dot_all_to_all).
        for a2a in self.graph.instructions:
            if a2a.opcode != Op.ALL_TO_ALL or a2a.attrs["split_dim"] != 1 or \
                    a2a.attrs["concat_dim"] != 0:
                continue
            d = by.get(a2a.operands[0])
            if d is None or d.opcode != Op.DOT or d.id in outs or d.id in self._fused_skip \
                    or d.id in self._fused or users.get(d.id, []) != [a2a.id] \
                    or d.shape.dtype != DType.BF16 or d.shape.rank < 3:
                continue
            at = d.attrs
            if tuple(at["lhs_batch"]) != (0,) or tuple(at["rhs_batch"]) != (0,):
                continue
            groups = a2a.attrs["subgroups"]
            gs = len(groups[0])
            if any(len(g) != gs for g in groups) or gs > 8:
                continue
            rsh = self._shape(d.operands[1])
            rfree = [k for k in range(rsh.rank) if k not in at["rhs_contracting"] and k != 0]
            if [rsh.dims[k] for k in rfree if rsh.dims[k] != 1] != [d.shape.dims[-1]]:
                continue
            rows = int(np.prod(d.shape.dims[1:-1]))
            if d.shape.dims[-1] < 512 or rows < 256 or d.shape.dims[1] % gs or \
                    (rows // gs) % 32:
                continue
            self._fused_skip.add(d.id)
            self._fused[a2a.id] = ("dot_a2a", d, a2a)

    def _plan_attention(self, users, outs):
        """Dot(q,k) -> fused softmax -> Dot(probs, v) with the Transformer
        layouts q/k/v [B,S|T,N,D], logits [B,N,S,T], ctx [B,N,S,D] -> one
        flash-attention kernel (tcgen05; no logits in HBM)."""
        if self._knob("SPMD_FUSED_ATTENTION") == "0":
            return
        by = self.by_id
        for div_id, spec in list(self._fused.items()):
            if spec[0] != "softmax" or div_id in outs:
                continue
            logits = by[spec[1]]
            if logits.opcode != Op.DOT or logits.shape.dtype != DType.BF16:
                continue
            a = logits.attrs
            if (tuple(a["lhs_batch"]), tuple(a["rhs_batch"]), tuple(a["lhs_contracting"]),
                    tuple(a["rhs_contracting"])) != ((0, 2), (0, 2), (3,), (3,)):
                continue
            u = users.get(div_id, [])
            if len(u) != 1 or by[u[0]].opcode != Op.DOT:
                continue
            ctx = by[u[0]]
            c = ctx.attrs
            if ctx.operands[0] != div_id or (tuple(c["lhs_batch"]), tuple(c["rhs_batch"]),
                                             tuple(c["lhs_contracting"]),
                                             tuple(c["rhs_contracting"])) != \
                    ((0, 1), (0, 2), (3,), (1,)):
                continue
            if any(x != spec[1] and x not in self._fused_skip
                   for x in users.get(logits.id, [])) or logits.id in outs:
                continue
            q, k = logits.operands
            v = ctx.operands[1]
            qs, ks, vs = self._shape(q), self._shape(k), self._shape(v)
            if qs.rank != 4 or ks.dims != vs.dims or qs.dims[3] not in (64, 128, 256):
                continue
            self._fused_skip.update({logits.id, div_id})
            # ctx -> transpose(0,2,1,3) (App. A ctx_t): the kernel stores
            # [B,S,N,D] directly
            cu = users.get(ctx.id, [])
            tr = by[cu[0]] if len(cu) == 1 else None
            if tr is not None and ctx.id not in outs and tr.opcode == Op.TRANSPOSE and \
                    tuple(tr.attrs["permutation"]) == (0, 2, 1, 3):
                self._fused_skip.add(ctx.id)
                self._fused[tr.id] = ("attention", q, k, v, 1)
            else:
                self._fused[ctx.id] = ("attention", q, k, v, 0)

    def _plan_halo_windows(self, users, outs):
        """dynamic-slice(mask(concat(left, shard, right))) -> one halo-window
        pass (the window assembly of exchange_and_slice, reference
        formatting.py:109-182)."""
        by = self.by_id
        for ds in self.graph.instructions:
            if ds.opcode != Op.DYNAMIC_SLICE or ds.id in self._fused_skip:
                continue
            src = ds.operands[0]
            mask = self._fused.get(src)
            if mask is not None and mask[0] != "mask":
                continue
            cat_id = mask[1] if mask is not None else src
            cat = by.get(cat_id)
            if cat is None or cat.opcode != Op.CONCAT or len(cat.operands) > 3:
                continue
            axis = cat.attrs["dim"]
            if mask is not None and mask[4] != axis:
                continue
            consumer = src if mask is not None else ds.id
            if cat_id in outs or any(u != consumer and u not in self._fused_skip
                                     for u in users.get(cat_id, [])):
                continue
            if mask is not None and (src in outs or users.get(src, []) != [ds.id]):
                continue
            starts = ds.operands[1:]
            ok = True
            for d in range(ds.shape.rank):
                if d == axis:
                    continue
                c = by.get(starts[d])
                lit = np.asarray(c.attrs["literal"]) if c is not None and \
                    c.opcode == Op.CONSTANT else None
                if lit is None or lit.size != 1 or int(lit) != 0 or \
                        ds.attrs["sizes"][d] != cat.shape.dims[d]:
                    ok = False
                    break
            if not ok:
                continue
            self._fused_skip.add(cat_id)
            if mask is not None:
                self._fused_skip.add(src)
            self._fused[ds.id] = ("halo", tuple(cat.operands), axis, starts[axis], mask)

    def _match_range_mask(self, sel: Instruction, users, outs):
        """Recognise select(iota+off < high, val, bcast(fill)) [then
        select(iota+off >= low, ., same fill)] as emitted by the partitioner's
        select_range (reference partitioner.py:212-228)."""
        by = self.by_id

        def get(i):
            return by.get(i)

        def scalar_bcast(i):
            b = get(i)
            if b is None or b.opcode != Op.BROADCAST or tuple(b.attrs["broadcast_dims"]) != ():
                return None
            return b

        def const_int(i):
            c = get(i)
            if c is None or c.opcode != Op.CONSTANT:
                return None
            lit = np.asarray(c.attrs["literal"])
            return int(lit) if lit.size == 1 else None

        def parse_cmp(pred_id, direction):
            pred = get(pred_id)
            if pred is None or pred.opcode != Op.COMPARE or pred.attrs["direction"] != direction:
                return None
            gidx, bc = get(pred.operands[0]), scalar_bcast(pred.operands[1])
            if gidx is None or bc is None or gidx.opcode != Op.ADD:
                return None
            bound = const_int(bc.operands[0])
            if bound is None:
                return None
            return pred, gidx, bc, bound

        if sel.id in outs:
            return None
        lt = parse_cmp(sel.operands[0], CompareDirection.LT)
        if lt is None:
            return None
        pred_lt, gidx, bc_hi, high = lt
        iota, boff = get(gidx.operands[0]), scalar_bcast(gidx.operands[1])
        if iota is None or iota.opcode != Op.IOTA or boff is None:
            return None
        if iota.shape.dims != sel.shape.dims or boff.shape.dtype != DType.S32:
            return None
        fill = scalar_bcast(sel.operands[2])
        if fill is None:
            return None
        val = sel.operands[1]
        chain = [iota.id, boff.id, gidx.id, bc_hi.id, pred_lt.id, fill.id]
        result, low, has_low = sel, 0, False
        su = users.get(sel.id, [])
        if len(su) == 1 and get(su[0]).opcode == Op.SELECT:
            outer = get(su[0])
            ge = parse_cmp(outer.operands[0], CompareDirection.GE)
            if ge is not None and ge[1].id == gidx.id and outer.operands[1] == sel.id \
                    and outer.operands[2] == fill.id:
                chain += [sel.id, ge[0].id, ge[2].id]
                result, low, has_low = outer, ge[3], True
        allowed = set(chain) | {result.id}
        for vid in chain:
            if vid in outs or any(u not in allowed for u in users.get(vid, [])):
                return None
        spec = ("mask", val, boff.operands[0], fill.operands[0], iota.attrs["iota_dimension"],
                low, high, has_low)
        return result.id, chain, spec

    # ------------------------------------------------------------------
    # compilation: one closure per instruction
    # ------------------------------------------------------------------
    def _compile(self) -> list[_Step]:
        last_use: dict[str, int] = {}
        instrs = [i for i in self.graph.instructions if i.id not in self._fused_skip]
        for k, ins in enumerate(instrs):
            for o in self._operands_of(ins):
                last_use[o] = k
        keep = set(self.graph.outputs)
        steps = []
        for k, ins in enumerate(instrs):
            fn = self._make_step(ins)
            ops = tuple(self._operands_of(ins))
            frees = tuple(o for o in set(ops) if last_use.get(o) == k and o not in keep)
            fused = self._fused.get(ins.id)
            coll = ins.opcode in COLLECTIVES and not (
                fused and fused[0] in ("dot_rs", "dot_a2a", "moe_dispatch_a2a"))
            steps.append(_Step(ins, fn, frees, ops, coll))
        return steps

    def _hoist_collectives(self, steps: list) -> list:
        """Issue order with every collective moved up to right after its last
        operand producer (per-stream order is issue order, so this is what
        lets weight all-gathers run under earlier GEMMs)."""
        pending = [s for s in steps if s.coll]
        order, issued = [], set()

        def flush():
            progress = True
            while progress:
                progress = False
                for s in list(pending):
                    if all(o in issued for o in s.ops):
                        order.append(s)
                        issued.add(s.ins.id)
                        pending.remove(s)
                        progress = True

        flush()
        for s in steps:
            if s.coll:
                continue
            order.append(s)
            issued.add(s.ins.id)
            flush()
        order += pending
        last_use = {}
        for k, s in enumerate(order):
            for o in s.ops:
                last_use[o] = k
        keep = set(self.graph.outputs)
        for k, s in enumerate(order):
            s.frees = tuple(o for o in set(s.ops) if last_use.get(o) == k and o not in keep)
        return order

    def _operands_of(self, ins: Instruction):
        f = self._fused.get(ins.id)
        if f is None:
            return ins.operands
        if f[0] == "softmax":
            return (f[1],)
        if f[0] in ("softmax_bwd", "relu_bwd"):
            return (f[1], f[2])
        if f[0] == "slice_cp":
            return (f[1].operands[0],)
        if f[0] == "mask":
            return (f[1], f[2], f[3])
        if f[0] == "attention":
            return f[1:4]
        if f[0] == "halo":
            mask = f[4]
            return tuple(f[1]) + (f[3],) + ((mask[2], mask[3]) if mask is not None else ())
        if f[0] in ("moe_dispatch", "moe_combine", "moe_dispatch_a2a"):
            return (f[1],)
        if f[0] == "dot_rs_add":
            return tuple(f[1].operands) + (f[3],)
        if f[0] == "ag_split_dot":
            lag, rag, dot = f[1], f[2], f[3]
            return (lag.operands[0] if lag is not None else dot.operands[0],
                    rag.operands[0] if rag is not None else dot.operands[1])
        if f[0] == "dot_add":
            return tuple(f[1].operands) + (f[2],)
        if f[0] == "halo_conv":
            _, conv, _, (_, pieces, _, start, mask), _ = f
            return tuple(pieces) + (start,) + ((mask[2],) if mask is not None else ()) + \
                (conv.operands[1],)
        return f[1].operands   # dot_relu / conv_relu / dot_rs: the producer's operands

    def _make_step(self, ins: Instruction):
        lib = self.lib
        op = ins.opcode
        P = self.P
        shp = ins.shape
        f = self._fused.get(ins.id)
        if f is not None and f[0] == "softmax":
            x = f[1]
            xs = self._shape(x)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_softmax_lastdim(desc(env[x], xs), desc(out, shp), P, s),
                        "spmd_softmax_lastdim")
                return out
            return run
        if f is not None and f[0] == "slice_cp":
            _, sl, cp, axis = f
            x, xsh = sl.operands[0], self._shape(sl.operands[0])
            start = sl.attrs["starts"][axis]
            pairs = (ctypes.c_int32 * max(1, 2 * len(cp.attrs["pairs"])))(
                *[v for pr in cp.attrs["pairs"] for v in pr])
            npairs = len(cp.attrs["pairs"])
            comm = self.comm

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_peer_slice_collective_permute(
                    comm.handle, desc(env[x], xsh), axis, start, desc(out, shp), pairs, npairs,
                    self._peer_cp[cp.id], self._lane_of.get(s, 0), s), "collective-permute")
                return out
            return run
        if f is not None and f[0] in ("softmax_bwd", "relu_bwd"):
            _, a, b = f
            ash, bsh = self._shape(a), self._shape(b)
            fn = lib.spmd_softmax_backward_lastdim if f[0] == "softmax_bwd" \
                else lib.spmd_relu_backward

            def run(env, s):
                out = self._alloc(shp)
                C.check(fn(desc(env[a], ash), desc(env[b], bsh), desc(out, shp), P, s), f[0])
                return out
            return run
        if f is not None and f[0] == "ag_split_dot":
            return self._ag_split_dot_step(f[1], f[2], f[3], shp)
        if f is not None and f[0] == "dot_add":
            dot, res = f[1], f[2]
            a, b = dot.operands
            ash, bsh = self._shape(a), self._shape(b)
            dd = self._dot_dims(dot)
            ref = ctypes.byref(dd)

            def run(env, s):
                out = self._alloc(shp)
                rc = lib.spmd_dot_add(desc(env[a], ash), desc(env[b], bsh), desc(env[res], shp),
                                      desc(out, shp), ref, P, s)
                if rc == C.ERR_UNSUPPORTED:
                    # not a wide-GEMM shape: the Dot, then the Add in place
                    C.check(lib.spmd_dot(desc(env[a], ash), desc(env[b], bsh), desc(out, shp),
                                         ref, P, s), "dot")
                    C.check(lib.spmd_binary(_BINARY[Op.ADD], 0, desc(out, shp),
                                            desc(env[res], shp), desc(out, shp), P, s), "add")
                else:
                    C.check(rc, "dot_add")
                return out
            return run
        if f is not None and f[0] == "transpose_relu":
            tr = f[1]
            src = tr.operands[0]
            ssh = self._shape(src)
            perm = C.i32_array(tr.attrs["permutation"])

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_transpose_relu(desc(env[src], ssh), desc(out, shp), perm, P, s),
                        "transpose_relu")
                return out
            return run
        if f is not None and f[0] == "dot_relu":
            return self._dot_step(f[1], shp, epilogue=1)
        if f is not None and f[0] == "conv_relu":
            return self._conv_step(f[1], epilogue=1)
        if f is not None and f[0] == "halo_conv":
            return self._halo_conv_step(*f[1:])
        if f is not None and f[0] == "dot_rs_add":
            return self._dot_rs_step(f[1], f[2], resid=f[3])
        if f is not None and f[0] == "dot_rs":
            return self._dot_rs_step(f[1], f[2])
        if f is not None and f[0] == "dot_a2a":
            return self._dot_a2a_step(f[1], f[2])
        if f is not None and f[0] == "moe_dispatch_a2a":
            _, x, ridx, a2a = f
            xsh, r = self._shape(x), self.routing[ridx]
            ish = Shape(tuple(r.expert.shape[1:]), DType.S32)
            groups, ng, gs = _groups_arg(a2a.attrs["subgroups"])
            comm = self.comm
            # (batch, expert, slot) -> token table, private to this op
            nidx = shp.dims[0] * shp.dims[1] * shp.dims[2]
            idx = _torch().empty((nidx,), dtype=_torch().int32, device=self.device)
            idx_sh = Shape((nidx,), DType.S32)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_moe_dispatch_all_to_all(comm.handle, desc(env[x], xsh),
                                                         desc(r.expert, ish), desc(r.slot, ish),
                                                         desc(out, shp), desc(idx, idx_sh),
                                                         groups, ng, gs, s),
                        "moe_dispatch_all_to_all")
                return out
            return run
        if f is not None and f[0] in ("moe_dispatch", "moe_combine"):
            x, ridx = f[1], f[2]
            flags = f[3] if len(f) > 3 else 0     # moe.cu MOE_EBCM | MOE_RELU
            xsh = self._shape(x)
            r = self.routing[ridx]
            ish = Shape(tuple(r.expert.shape[1:]), DType.S32)
            gsh = Shape(tuple(r.gate.shape[1:]), DType.F32)

            def run(env, s):
                out = self._alloc(shp)
                if f[0] == "moe_dispatch":
                    rc = lib.spmd_moe_dispatch_ex(desc(env[x], xsh), desc(r.expert, ish),
                                                  desc(r.slot, ish), desc(out, shp), flags, P, s)
                else:
                    rc = lib.spmd_moe_combine_ex(desc(env[x], xsh), desc(r.expert, ish),
                                                 desc(r.slot, ish), desc(r.gate, gsh),
                                                 desc(out, shp), flags, P, s)
                C.check(rc, f[0])
                return out
            return run
        if f is not None and f[0] == "attention":
            _, q, k, v, bsnd = f
            qs, ks, vs = self._shape(q), self._shape(k), self._shape(v)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_attention_layout(desc(env[q], qs), desc(env[k], ks),
                                                  desc(env[v], vs), desc(out, shp), 1.0, bsnd, P,
                                                  s), "attention")
                return out
            return run
        if f is not None and f[0] == "halo":
            _, pieces, axis, start, mask = f
            psh = [self._shape(x) for x in pieces]
            ssh = self._shape(start)
            if mask is not None:
                _, _, off, fill, _, low, high, has_low = mask
                osh, fsh = self._shape(off), self._shape(fill)

            def run(env, s):
                out = self._alloc(shp)
                arr = (C.SpmdTensor * len(pieces))(*[desc(env[x], sh)
                                                     for x, sh in zip(pieces, psh)])
                if mask is None:
                    dummy = desc(env[start], ssh)
                    rc = lib.spmd_halo_window(arr, len(pieces), axis, desc(env[start], ssh), 0,
                                              dummy, dummy, 0, 0, 0, desc(out, shp), P, s)
                else:
                    rc = lib.spmd_halo_window(arr, len(pieces), axis, desc(env[start], ssh), 1,
                                              desc(env[off], osh), desc(env[fill], fsh), low,
                                              high, int(has_low), desc(out, shp), P, s)
                C.check(rc, "halo_window")
                return out
            return run
        if f is not None and f[0] == "mask":
            _, val, off, fill, axis, low, high, has_low = f
            vsh, osh, fsh = self._shape(val), self._shape(off), self._shape(fill)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_mask_range(desc(env[val], vsh), desc(env[off], osh),
                                            desc(env[fill], fsh), desc(out, shp), axis, low,
                                            high, int(has_low), P, s), "mask_range")
                return out
            return run

        if op == Op.PARAMETER:
            idx = [p.id for p in self.params].index(ins.id)
            return lambda env, s: env["__inputs__"][idx]
        if op == Op.CONSTANT:
            return lambda env, s: self._constant(ins)
        if op == Op.IOTA:
            axis = ins.attrs["iota_dimension"]

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_iota(desc(out, shp), axis, P, s), "spmd_iota")
                return out
            return run
        if op == Op.PARTITION_ID:
            base = self.base

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_partition_id(desc(out, shp), P, base, s), "spmd_partition_id")
                return out
            return run
        if op in ELEMENTWISE_UNARY:
            code = _UNARY[op]
            a = ins.operands[0]

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_unary(code, desc(env[a], shp), desc(out, shp), P, s), op.value)
                return out
            return run
        if op in ELEMENTWISE_BINARY:
            code = _BINARY[op]
            cmp = _CMP[ins.attrs["direction"]] if op == Op.COMPARE else 0
            a, b = ins.operands
            ish = self._shape(a)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_binary(code, cmp, desc(env[a], ish), desc(env[b], ish),
                                        desc(out, shp), P, s), op.value)
                return out
            return run
        if op == Op.SELECT:
            p_, a, b = ins.operands
            psh = self._shape(p_)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_select(desc(env[p_], psh), desc(env[a], shp),
                                        desc(env[b], shp), desc(out, shp), P, s), "select")
                return out
            return run
        if op == Op.BROADCAST:
            a = ins.operands[0]
            ash = self._shape(a)
            bd = C.i32_array(ins.attrs["broadcast_dims"])

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_broadcast(desc(env[a], ash), desc(out, shp), bd, P, s),
                        "broadcast")
                return out
            return run
        if op == Op.RESHAPE:
            a = ins.operands[0]
            return lambda env, s: env[a].reshape((P,) + shp.dims)
        if op == Op.TRANSPOSE:
            a = ins.operands[0]
            ash = self._shape(a)
            perm = C.i32_array(ins.attrs["permutation"])

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_transpose(desc(env[a], ash), desc(out, shp), perm, P, s),
                        "transpose")
                return out
            return run
        if op == Op.REVERSE:
            a = ins.operands[0]
            dims = list(ins.attrs["dims"])
            arr = C.i32_array(dims)

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_reverse(desc(env[a], shp), desc(out, shp), arr, len(dims), P, s),
                        "reverse")
                return out
            return run
        if op == Op.PAD:
            a, v = ins.operands
            ash, vsh = self._shape(a), self._shape(v)
            lo, hi, it = (C.i64_array(ins.attrs[k]) for k in ("low", "high", "interior"))

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_pad(desc(env[a], ash), desc(env[v], vsh), desc(out, shp),
                                     lo, hi, it, P, s), "pad")
                return out
            return run
        if op == Op.SLICE:
            a = ins.operands[0]
            ash = self._shape(a)
            st, sd = C.i64_array(ins.attrs["starts"]), C.i64_array(ins.attrs["strides"])

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_slice(desc(env[a], ash), desc(out, shp), st, sd, P, s), "slice")
                return out
            return run
        if op in (Op.DYNAMIC_SLICE, Op.DYNAMIC_UPDATE_SLICE):
            a = ins.operands[0]
            ash = self._shape(a)
            upd = ins.operands[1] if op == Op.DYNAMIC_UPDATE_SLICE else None
            first = 2 if upd else 1
            starts = ins.operands[first:]
            ssh = [self._shape(x) for x in starts]
            ush = self._shape(upd) if upd else None

            def run(env, s):
                out = self._alloc(shp)
                arr = (C.SpmdTensor * max(1, len(starts)))(
                    *[desc(env[x], sh) for x, sh in zip(starts, ssh)])
                if upd is None:
                    C.check(lib.spmd_dynamic_slice(desc(env[a], ash), arr, desc(out, shp), P, s),
                            "dynamic-slice")
                else:
                    C.check(lib.spmd_dynamic_update_slice(desc(env[a], ash), desc(env[upd], ush),
                                                          arr, desc(out, shp), P, s),
                            "dynamic-update-slice")
                return out
            return run
        if op == Op.CONCAT:
            ops = ins.operands
            shs = [self._shape(x) for x in ops]
            axis = ins.attrs["dim"]

            def run(env, s):
                out = self._alloc(shp)
                arr = (C.SpmdTensor * max(1, len(ops)))(
                    *[desc(env[x], sh) for x, sh in zip(ops, shs)])
                C.check(lib.spmd_concat(arr, len(ops), axis, desc(out, shp), P, s), "concat")
                return out
            return run
        if op == Op.REDUCE:
            a, init = ins.operands
            ash, ish = self._shape(a), self._shape(init)
            dims = list(ins.attrs["dims"])
            arr = C.i32_array(dims)
            kind = _KIND[ins.attrs["kind"]]

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_reduce(desc(env[a], ash), desc(env[init], ish), desc(out, shp),
                                        arr, len(dims), kind, P, s), "reduce")
                return out
            return run
        if op == Op.DOT:
            return self._dot_step(ins, shp, epilogue=0)
        if op == Op.CONVOLUTION:
            return self._conv_step(ins)
        if op == Op.ROTATE:
            a = ins.operands[0]
            dim, amt = ins.attrs["dim"], ins.attrs["amount"]

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_rotate(desc(env[a], shp), desc(out, shp), dim, amt, P, s),
                        "rotate")
                return out
            return run
        if op == Op.SHIFT:
            a, fill = ins.operands
            fsh = self._shape(fill)
            dim, amt = ins.attrs["dim"], ins.attrs["amount"]

            def run(env, s):
                out = self._alloc(shp)
                C.check(lib.spmd_shift(desc(env[a], shp), desc(env[fill], fsh), desc(out, shp),
                                       dim, amt, P, s), "shift")
                return out
            return run
        if op in COLLECTIVES:
            return self._collective_step(ins)
        raise EvalError(f"cannot evaluate opcode {op.value}")

    def _dot_step(self, ins, shp, epilogue):
        lib, P = self.lib, self.P
        a, b = ins.operands
        ash, bsh = self._shape(a), self._shape(b)
        dd = C.SpmdDotDims()
        at = ins.attrs
        dd.n_batch = len(at["lhs_batch"])
        dd.n_contract = len(at["lhs_contracting"])
        for i, (x, y) in enumerate(zip(at["lhs_batch"], at["rhs_batch"])):
            dd.lhs_batch[i], dd.rhs_batch[i] = x, y
        for i, (x, y) in enumerate(zip(at["lhs_contracting"], at["rhs_contracting"])):
            dd.lhs_contracting[i], dd.rhs_contracting[i] = x, y
        dd.epilogue = epilogue
        ref = ctypes.byref(dd)

        def run(env, s):
            out = self._alloc(shp)
            C.check(lib.spmd_dot(desc(env[a], ash), desc(env[b], bsh), desc(out, shp), ref, P, s),
                    "dot")
            return out
        return run

    def _ag_split_dot_step(self, lag, rag, dot, shp):
        """Loopback all-gather(s) -> f32 Dot (_plan_fusions): the gathers write
        the operands' tf32 hi / lo halves (spmd_local_all_gather_split /
        _split_t) and spmd_dot_f32_presplit skips those splits.  Any step
        that does not apply falls back to the plain gather / Dot (hi + lo is
        the gathered value exactly)."""
        lib, P = self.lib, self.P
        dd = self._dot_dims(dot)
        ref = ctypes.byref(dd)
        ash, bsh = self._shape(dot.operands[0]), self._shape(dot.operands[1])
        a_src = lag.operands[0] if lag is not None else dot.operands[0]
        b_src = rag.operands[0] if rag is not None else dot.operands[1]
        a_ssh, b_ssh = self._shape(a_src), self._shape(b_src)
        ga = _groups_arg(lag.attrs["subgroups"]) if lag is not None else None
        gb = _groups_arg(rag.attrs["subgroups"]) if rag is not None else None
        bt = Shape((bsh.dims[1], bsh.dims[0]), DType.F32) if rag is not None else None
        t10 = C.i32_array((1, 0))

        def gather(ag, gr, src, ssh, osh, env, s):
            out = self._alloc(osh)
            C.check(lib.spmd_local_all_gather(desc(env[src], ssh), desc(out, osh),
                                              ag.attrs["dim"], gr[0], gr[1], gr[2], P, s),
                    "all-gather")
            return out

        def shape_only(sh):
            t = C.SpmdTensor()
            t.dtype, t.rank = C.DTYPE_CODE[DType.F32], sh.rank
            for i, d in enumerate(sh.dims):
                t.dims[i] = d
            return t

        def run(env, s):
            out = self._alloc(shp)
            a_full = b_full = None
            a_hl = b_hl = (C.SpmdTensor(), C.SpmdTensor())
            # (the four halves stay referenced until the Dot is enqueued)
            ahi = alo = bhi = blo = None
            if lag is not None:
                ahi, alo = self._alloc(ash), self._alloc(ash)
                rc = lib.spmd_local_all_gather_split(desc(env[a_src], a_ssh), desc(ahi, ash),
                                                     desc(alo, ash), lag.attrs["dim"], ga[0],
                                                     ga[1], ga[2], P, s)
                if rc == C.ERR_UNSUPPORTED:
                    a_full = gather(lag, ga, a_src, a_ssh, ash, env, s)
                else:
                    C.check(rc, "all-gather split")
                    a_hl = (desc(ahi, ash), desc(alo, ash))
            else:
                a_full = env[a_src]
            if rag is not None:
                bhi, blo = self._alloc(bt), self._alloc(bt)
                rc = lib.spmd_local_all_gather_split_t(desc(env[b_src], b_ssh), desc(bhi, bt),
                                                       desc(blo, bt), gb[0], gb[1], gb[2], P, s)
                if rc == C.ERR_UNSUPPORTED:
                    b_full = gather(rag, gb, b_src, b_ssh, bsh, env, s)
                else:
                    C.check(rc, "all-gather split-transpose")
                    b_hl = (desc(bhi, bt), desc(blo, bt))
            else:
                b_full = env[b_src]
            a_d = desc(a_full, ash) if a_full is not None else shape_only(ash)
            b_d = desc(b_full, bsh) if b_full is not None else shape_only(bsh)
            rc = lib.spmd_dot_f32_presplit(a_d, a_hl[0], a_hl[1], b_d, b_hl[0], b_hl[1],
                                           desc(out, shp), ref, P, s)
            if rc == C.ERR_UNSUPPORTED:
                # rebuild the gathered operands exactly (hi + lo; the rhs
                # halves are transposed) and run the plain Dot
                if a_full is None:
                    a_full = self._alloc(ash)
                    C.check(lib.spmd_binary(_BINARY[Op.ADD], 0, a_hl[0], a_hl[1],
                                            desc(a_full, ash), P, s), "add")
                if b_full is None:
                    t = self._alloc(bt)
                    C.check(lib.spmd_binary(_BINARY[Op.ADD], 0, b_hl[0], b_hl[1], desc(t, bt),
                                            P, s), "add")
                    b_full = self._alloc(bsh)
                    C.check(lib.spmd_transpose(desc(t, bt), desc(b_full, bsh), t10, P, s),
                            "transpose")
                C.check(lib.spmd_dot(desc(a_full, ash), desc(b_full, bsh), desc(out, shp), ref,
                                     P, s), "dot")
            else:
                C.check(rc, "dot_f32_presplit")
            return out
        return run

    def _dot_dims(self, ins, epilogue=0):
        dd = C.SpmdDotDims()
        at = ins.attrs
        dd.n_batch = len(at["lhs_batch"])
        dd.n_contract = len(at["lhs_contracting"])
        for i, (x, y) in enumerate(zip(at["lhs_batch"], at["rhs_batch"])):
            dd.lhs_batch[i], dd.rhs_batch[i] = x, y
        for i, (x, y) in enumerate(zip(at["lhs_contracting"], at["rhs_contracting"])):
            dd.lhs_contracting[i], dd.rhs_contracting[i] = x, y
        dd.epilogue = epilogue
        return dd

    def _dot_a2a_step(self, dot, a2a):
        lib, comm = self.lib, self.comm
        a, b = dot.operands
        ash, bsh, shp = self._shape(a), self._shape(b), a2a.shape
        dd = self._dot_dims(dot)
        ref = ctypes.byref(dd)
        groups, ng, gs = _groups_arg(a2a.attrs["subgroups"])

        def run(env, s):
            out = self._alloc(shp)
            C.check(lib.spmd_dot_all_to_all(comm.handle, desc(env[a], ash), desc(env[b], bsh),
                                            desc(out, shp), ref, 1, 0, groups, ng, gs, s),
                    "dot_all_to_all")
            return out
        return run

    def _dot_rs_step(self, dot, rs, resid=None):
        lib, comm = self.lib, self.comm
        a, b = dot.operands
        ash, bsh, shp = self._shape(a), self._shape(b), rs.shape
        dd = self._dot_dims(dot)
        ref = ctypes.byref(dd)
        groups, ng, gs = _groups_arg(rs.attrs["subgroups"])
        dim = rs.attrs["dim"]

        def run(env, s):
            out = self._alloc(shp)
            if resid is None:
                C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(env[a], ash),
                                                    desc(env[b], bsh), desc(out, shp), ref, dim,
                                                    groups, ng, gs, s), "dot_reduce_scatter")
            else:
                C.check(lib.spmd_dot_reduce_scatter_add(comm.handle, desc(env[a], ash),
                                                        desc(env[b], bsh),
                                                        desc(env[resid], shp), desc(out, shp),
                                                        ref, dim, groups, ng, gs, s),
                        "dot_reduce_scatter_add")
            return out
        return run

    def _conv_dims(self, ins, epilogue=0):
        cd = ins.attrs["conv_dims"]
        c = C.SpmdConvDims()
        c.lhs_batch, c.lhs_feature = cd.lhs_batch, cd.lhs_feature
        c.rhs_in_feature, c.rhs_out_feature = cd.rhs_in_feature, cd.rhs_out_feature
        c.out_batch, c.out_feature = cd.out_batch, cd.out_feature
        c.n_spatial = len(cd.lhs_spatial)
        for i, w in enumerate(ins.attrs["window"]):
            c.lhs_spatial[i], c.rhs_spatial[i] = cd.lhs_spatial[i], cd.rhs_spatial[i]
            c.out_spatial[i] = cd.out_spatial[i]
            c.size[i], c.stride[i] = w.size, w.stride
            c.pad_low[i], c.pad_high[i] = w.padding_low, w.padding_high
            c.base_dilation[i], c.window_dilation[i] = w.base_dilation, w.window_dilation
        c.epilogue = epilogue
        return c

    def _halo_conv_step(self, conv, epilogue, halo, window_id):
        lib, P = self.lib, self.P
        _, pieces, axis, start, mask = halo
        psh = [self._shape(x) for x in pieces]
        ssh = self._shape(start)
        wsh, rsh, osh = self._shape(window_id), self._shape(conv.operands[1]), conv.shape
        rhs = conv.operands[1]
        c = self._conv_dims(conv, epilogue)
        ref = ctypes.byref(c)
        if mask is not None:
            _, _, off, _, _, low, high, has_low = mask
            offsh = self._shape(off)

        def run(env, s):
            out = self._alloc(osh)
            arr = (C.SpmdTensor * len(pieces))(*[desc(env[x], sh) for x, sh in zip(pieces, psh)])
            st = desc(env[start], ssh)
            win = C.SpmdTensor()
            win.dtype, win.rank = C.DTYPE_CODE[wsh.dtype], wsh.rank
            for i, d in enumerate(wsh.dims):
                win.dims[i] = d
            if mask is None:
                rc = lib.spmd_halo_convolution(arr, len(pieces), axis, st, 0, st, 0, 0, 0, win,
                                               desc(env[rhs], rsh), desc(out, osh), ref, P, s)
            else:
                rc = lib.spmd_halo_convolution(arr, len(pieces), axis, st, 1,
                                               desc(env[off], offsh), low, high, int(has_low),
                                               win, desc(env[rhs], rsh), desc(out, osh), ref, P,
                                               s)
            C.check(rc, "halo_convolution")
            return out
        return run

    def _conv_step(self, ins, epilogue=0):
        lib, P = self.lib, self.P
        a, b = ins.operands
        ash, bsh, shp = self._shape(a), self._shape(b), ins.shape
        cd = ins.attrs["conv_dims"]
        win = ins.attrs["window"]
        c = C.SpmdConvDims()
        c.lhs_batch, c.lhs_feature = cd.lhs_batch, cd.lhs_feature
        c.rhs_in_feature, c.rhs_out_feature = cd.rhs_in_feature, cd.rhs_out_feature
        c.out_batch, c.out_feature = cd.out_batch, cd.out_feature
        c.n_spatial = len(cd.lhs_spatial)
        for i, w in enumerate(win):
            c.lhs_spatial[i], c.rhs_spatial[i] = cd.lhs_spatial[i], cd.rhs_spatial[i]
            c.out_spatial[i] = cd.out_spatial[i]
            c.size[i], c.stride[i] = w.size, w.stride
            c.pad_low[i], c.pad_high[i] = w.padding_low, w.padding_high
            c.base_dilation[i], c.window_dilation[i] = w.base_dilation, w.window_dilation
        c.epilogue = epilogue
        ref = ctypes.byref(c)

        def run(env, s):
            out = self._alloc(shp)
            C.check(lib.spmd_convolution(desc(env[a], ash), desc(env[b], bsh), desc(out, shp),
                                         ref, P, s), "convolution")
            return out
        return run

    def _collective_step(self, ins):
        lib, P = self.lib, self.P
        op, shp = ins.opcode, ins.shape
        a = ins.operands[0]
        ash = self._shape(a)
        at = ins.attrs
        comm = self.comm
        if op == Op.COLLECTIVE_PERMUTE:
            flat = [x for pr in at["pairs"] for x in pr]
            pairs = C.i32_array(flat)
            npairs = len(at["pairs"])

            def run(env, s):
                out = self._alloc(shp)
                if comm is None:
                    C.check(lib.spmd_local_collective_permute(desc(env[a], ash), desc(out, shp),
                                                              pairs, npairs, P, s),
                            "collective-permute")
                elif ins.id in self._peer_cp:
                    C.check(lib.spmd_peer_collective_permute(
                        comm.handle, desc(env[a], ash), desc(out, shp), pairs, npairs,
                        self._peer_cp[ins.id], self._lane_of.get(s, 0), s), "collective-permute")
                else:
                    C.check(lib.spmd_collective_permute(comm.handle, desc(env[a], ash),
                                                        desc(out, shp), pairs, npairs, s),
                            "collective-permute")
                return out
            return run
        groups, ng, gs = _groups_arg(at["subgroups"])
        if comm is None and ng * gs != P:
            raise SubgroupMismatch(f"subgroups {at['subgroups']} do not partition "
                                   f"{P} devices")

        def run(env, s):
            out = self._alloc(shp)
            x, y = desc(env[a], ash), desc(out, shp)
            if op == Op.ALL_GATHER and self._peer_engine.get(ins.id, -1) >= 0:
                # one barrier channel per issuing stream
                ch = self._lane_of.get(s, 0)
                if ins.id in self._act_staged:
                    # stage + barrier on the compute stream (issued in program
                    # order right after the producer), pulls on this lane
                    torch = _torch()
                    cs = torch.cuda.current_stream(self.device)
                    lane = torch.cuda.ExternalStream(s, device=self.device)
                    ready = torch.cuda.Event()     # x may come from another lane
                    ready.record(lane)
                    cs.wait_event(ready)
                    C.check(lib.spmd_peer_stage(comm.handle, x, self._peer_ag[ins.id],
                                                cs.cuda_stream), "peer_stage")
                    C.check(lib.spmd_peer_barrier(comm.handle, 0, cs.cuda_stream),
                            "peer_barrier")
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    lane.wait_event(ev)
                rc = lib.spmd_peer_all_gather(comm.handle, x, y, at["dim"], groups, ng, gs,
                                              self._peer_ag[ins.id], ch,
                                              self._peer_engine.get(ins.id, 1), s)
            elif op == Op.ALL_GATHER:
                rc = lib.spmd_local_all_gather(x, y, at["dim"], groups, ng, gs, P, s) \
                    if comm is None else \
                    lib.spmd_all_gather(comm.handle, x, y, at["dim"], groups, ng, gs, s)
            elif op == Op.ALL_REDUCE:
                k = _KIND[at["kind"]]
                rc = lib.spmd_local_all_reduce(x, y, k, groups, ng, gs, P, s) \
                    if comm is None else \
                    lib.spmd_all_reduce(comm.handle, x, y, k, groups, ng, gs, s)
            elif op == Op.REDUCE_SCATTER:
                k = _KIND[at["kind"]]
                rc = lib.spmd_local_reduce_scatter(x, y, at["dim"], k, groups, ng, gs, P, s) \
                    if comm is None else \
                    lib.spmd_reduce_scatter(comm.handle, x, y, at["dim"], k, groups, ng, gs, s)
            else:
                rc = lib.spmd_local_all_to_all(x, y, at["split_dim"], at["concat_dim"], groups,
                                               ng, gs, P, s) \
                    if comm is None else \
                    lib.spmd_all_to_all(comm.handle, x, y, at["split_dim"], at["concat_dim"],
                                        groups, ng, gs, s)
            C.check(rc, op.value)
            return out

        if op in (Op.ALL_TO_ALL, Op.ALL_GATHER) and comm is not None:
            # peer landing zones are assigned after compilation (_peer_bytes):
            # choose the engine at run time
            keep_copy = ins.id in self.graph.outputs   # outputs outlive the step
            zone = {}
            def run_a2a(env, s):
                zones = self._peer_a2a if op == Op.ALL_TO_ALL else self._peer_agp
                if ins.id not in zones or (op == Op.ALL_GATHER and
                                           self._peer_engine.get(ins.id, -1) not in (1, -1)):
                    return run(env, s)
                off = zones[ins.id]
                x = desc(env[a], ash)
                if keep_copy:
                    out = self._alloc(shp)
                    y = desc(out, shp)
                else:
                    # the heap may have been re-allocated (grown) since the
                    # last run: re-derive the view from its current address
                    ptr = lib.spmd_comm_heap_ptr(comm.handle, off)
                    if zone.get("ptr") != ptr:
                        zone["ptr"] = ptr
                        zone["t"] = comm.heap_view(off, (1,) + shp.dims, shp.dtype, self.device)
                    out = zone["t"]
                    y = desc(out, shp)
                    y.data = None                # the landing zone is the result
                if op == Op.ALL_TO_ALL:
                    rc = lib.spmd_peer_all_to_all(comm.handle, x, y, at["split_dim"],
                                                  at["concat_dim"], groups, ng, gs, off,
                                                  self._lane_of.get(s, 0), s)
                else:
                    rc = lib.spmd_peer_push_all_gather(comm.handle, x, y, at["dim"], groups, ng,
                                                       gs, off, self._lane_of.get(s, 0), s)
                C.check(rc, op.value)
                return out
            return run_a2a
        return run

    def _constant(self, ins: Instruction):
        t = self._consts.get(ins.id)
        if t is None:
            t = upload_stacked([np.asarray(ins.attrs["literal"])] * self.P, ins.shape,
                               self.device, self.lib)
            self._consts[ins.id] = t
        return t

    # ------------------------------------------------------------------
    def run(self, inputs: Sequence, stream=None, keep: Optional[set] = None) -> list:
        """Execute on stacked device inputs ``[P, *param_dims]``; returns the
        stacked device outputs.  ``keep``: extra value ids to retain
        (returned via ``self.last_env``)."""
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        if len(inputs) != len(self.params):
            raise EvalError(f"expected {len(self.params)} inputs, got {len(inputs)}")
        if self.comm is not None and self._peer_bytes_used and \
                self.lib.spmd_comm_fused_half(self.comm.handle) != self._fused_half:
            raise EvalError("the communicator's fused peer region grew after this executor "
                            "was compiled (its staging slots would overlap it): rebuild the "
                            "Executor")
        env = {"__inputs__": list(inputs)}
        keep = keep or set()
        self.lib.spmd_set_sm_limit(self._sm_limit)   # process-wide; captured into graphs
        if self.comm_stream is None:
            for step in self.steps:
                env[step.ins.id] = step.fn(env, s)
                for vid in step.frees:
                    if vid not in keep:
                        env.pop(vid, None)
            if self._peer_cp or self._peer_a2a or self._peer_agp:
                # landing slots are read before any rank writes them again
                C.check(self.lib.spmd_peer_barrier(self.comm.handle, 0, s), "peer_barrier")
        else:
            self._run_two_streams(env, keep)
        if self._peer_bytes_used and not torch.cuda.is_current_stream_capturing():
            # a peer barrier that timed out only sets the device error word:
            # surface it here (graph replays: the caller checks after them)
            C.check(self.lib.spmd_check_device_errors(
                torch.cuda.current_stream(self.device).cuda_stream), "peer barrier")
        self.last_env = env if keep else None
        return [env[o] for o in self.graph.outputs]

    def _run_two_streams(self, env: dict, keep: set) -> None:
        """Compute on the current stream, collectives on the comm lanes;
        cross-stream values are ordered with events, and tensors touched by a
        comm stream are recorded on it so the caching allocator never
        recycles them early."""
        torch = _torch()
        compute = torch.cuda.current_stream(self.device)
        streams = [compute] + self.comm_streams
        for st in self.comm_streams:
            st.wait_stream(compute)               # inputs / fork for graph capture
        staged_ev: dict = {}
        if self._staged:
            # parameter shards -> peer heap slots, each phase closed by one
            # barrier on lane 1: the exposed gathers' shards first (their
            # pulls start after a small copy), then the rest
            st = self.comm_streams[0]
            for phase in self._stage_phases():
                for aid in phase:
                    t = env["__inputs__"][self._staged[aid]]
                    C.check(self.lib.spmd_peer_stage(
                        self.comm.handle, desc(t, self._shape(self.by_id[aid].operands[0])),
                        self._peer_ag[aid], st.cuda_stream), "peer_stage")
                    t.record_stream(st)
                C.check(self.lib.spmd_peer_barrier(self.comm.handle,
                                                   self._lane_of[st.cuda_stream],
                                                   st.cuda_stream), "peer_barrier")
                ev = torch.cuda.Event()
                ev.record(st)
                staged_ev.update({aid: ev for aid in phase})
        staged_waited: set = set()                # (lane, event id) pairs issued
        lane_of: dict[str, int] = {}
        events: dict[str, object] = {}
        for step in self.steps:
            lane = step.lane if step.coll else 0
            stream = streams[lane]
            ev = staged_ev.get(step.ins.id)
            if ev is not None and lane != 1 and (lane, id(ev)) not in staged_waited:
                stream.wait_event(ev)             # lane 1 is ordered after it already
                staged_waited.add((lane, id(ev)))
            for o in tuple(step.ops) + tuple(step.after):
                if o not in lane_of and o not in env:
                    continue
                src = lane_of.get(o, 0)
                if src == lane:
                    continue
                ev = events.get(o)
                if ev is None:
                    # produced on the compute stream: a marker recorded now
                    # covers it (the producer was issued earlier)
                    ev = torch.cuda.Event()
                    ev.record(streams[src])
                    events[o] = ev
                stream.wait_event(ev)
            if lane:
                # lane outputs and temporaries come from the lane's own
                # allocator pool: a block the compute stream freed while its
                # readers are still queued is never handed to a lane kernel
                with torch.cuda.stream(stream):
                    out = step.fn(env, stream.cuda_stream)
            else:
                out = step.fn(env, stream.cuda_stream)
            env[step.ins.id] = out
            lane_of[step.ins.id] = lane
            if lane:
                for o in step.ops:
                    t = env.get(o)
                    if t is not None and hasattr(t, "record_stream"):
                        t.record_stream(stream)
                # consumers run on the compute stream (or other lanes): the
                # block is recycled only after their uses complete
                out.record_stream(compute)
                ev = torch.cuda.Event()
                ev.record(stream)
                events[step.ins.id] = ev
            for vid in step.frees:
                if vid not in keep:
                    env.pop(vid, None)
        for st in self.comm_streams:
            compute.wait_stream(st)               # join
        if self._staged or self._act_staged or self._peer_cp or self._peer_a2a or \
                self._peer_agp:
            # every member has read the staged / landing slots before any
            # rank writes them again
            st = self.comm_streams[0]
            C.check(self.lib.spmd_peer_barrier(self.comm.handle, self._lane_of[st.cuda_stream],
                                               compute.cuda_stream), "peer_barrier")

    def timeline(self, inputs, graph: bool = False, replays: int = 5) -> list[dict]:
        """Run with CUDA events around every step on the stream it is issued
        to; returns [{id, op, stream, start_ms, end_ms}] relative to the
        first event (diagnostics: compute-stream gaps = exposed comm).
        ``graph``: the events become external event-record nodes of a
        captured CUDA graph (cudaEventRecordExternal) and the times are those
        of the last of ``replays`` back-to-back replays -- the timed step of
        bench.py, not the eager run."""
        torch = _torch()
        marks = []
        orig = [s.fn for s in self.steps]
        compute = torch.cuda.current_stream(self.device)
        if graph:
            rt = ctypes.CDLL("libcudart.so.12")

            def event():
                e = ctypes.c_void_p()
                assert rt.cudaEventCreate(ctypes.byref(e)) == 0
                return e

            def record(e, st):
                assert rt.cudaEventRecordWithFlags(e, ctypes.c_void_p(st.cuda_stream), 1) == 0

            def elapsed(a, b):
                ms = ctypes.c_float()
                assert rt.cudaEventElapsedTime(ctypes.byref(ms), a, b) == 0
                return ms.value
        else:
            def event():
                return torch.cuda.Event(enable_timing=True)

            def record(e, st):
                e.record(st)

            def elapsed(a, b):
                return a.elapsed_time(b)

        def wrap(step, fn):
            def run(env, s):
                cur = torch.cuda.current_stream(self.device)
                st = self.comm_streams[step.lane - 1] if (step.coll and step.lane) else cur
                e0, e1 = event(), event()
                record(e0, st)
                out = fn(env, s)
                record(e1, st)
                marks.append((step.ins.id, step.ins.opcode.value,
                              f"comm{step.lane}" if st is not cur else "compute", e0, e1))
                return out
            return run

        if graph:
            self.run(inputs)
            torch.cuda.synchronize(self.device)
        for s, f in zip(self.steps, orig):
            s.fn = wrap(s, f)
        try:
            t0 = event()
            if graph:
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream(device=self.device)
                cap.wait_stream(compute)
                with torch.cuda.graph(g, stream=cap):
                    record(t0, cap)
                    self.run(inputs)
                torch.cuda.synchronize(self.device)
                for _ in range(replays):
                    g.replay()
            else:
                record(t0, compute)
                self.run(inputs)
            torch.cuda.synchronize(self.device)
        finally:
            for s, f in zip(self.steps, orig):
                s.fn = f
        return [{"id": i, "op": o, "stream": st, "start_ms": elapsed(t0, a),
                 "end_ms": elapsed(t0, b)} for i, o, st, a, b in marks]

    def capture(self, inputs):
        """Capture one execution into a CUDA graph (after an eager warm-up
        run that materialises constants, communicators and kernel attributes).
        Returns ``(graph, outputs)``; ``graph.replay()`` re-runs the step on the
        same static input/output buffers."""
        torch = _torch()
        self.run(inputs)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=self.device)
        cap.wait_stream(torch.cuda.current_stream(self.device))
        n0 = self.lib.spmd_launch_count()
        with torch.cuda.graph(g, stream=cap):
            outs = self.run(inputs)
        self.launches_per_replay = self.lib.spmd_launch_count() - n0
        torch.cuda.synchronize(self.device)
        return g, outs

    def check_errors(self, stream=None) -> None:
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        C.check(self.lib.spmd_check_device_errors(s), "device")


# ---------------------------------------------------------------------------
# host <-> device
# ---------------------------------------------------------------------------

def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round to nearest even; NaN stays
    a quiet NaN (the device conversion __float2bfloat16_rn)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r = np.where(nan, ((u >> 16) | 0x40).astype(np.uint16), r)
    return r


def upload_stacked(arrays: Sequence[np.ndarray], shape: Shape, device, lib=None):
    """Stack per-partition host arrays into one device tensor ``[P, *dims]``."""
    torch = _torch()
    lib = lib or C.lib()
    P = len(arrays)
    if shape.dtype == DType.BF16:
        # round on the host (nearest-even, as the device convert) and ship
        # 2 bytes per element
        host = np.stack([np.asarray(a, dtype=np.float32).reshape(shape.dims) for a in arrays])
        bits = torch.from_numpy(np.ascontiguousarray(bf16_bits(host)).view(np.int16))
        return bits.to(device).view(torch.bfloat16)
    host = np.stack([np.asarray(a, dtype=np_dtype(shape.dtype)).reshape(shape.dims)
                     for a in arrays])
    if shape.dtype == DType.U32:
        host = host.view(np.int32)
    elif shape.dtype == DType.PRED:
        host = host.astype(np.uint8)
    return torch.from_numpy(np.ascontiguousarray(host)).to(device)


def download_stacked(t, shape: Shape, lib=None) -> list[np.ndarray]:
    """Device ``[P, *dims]`` -> list of per-partition host arrays (bf16 as
    float32)."""
    torch = _torch()
    lib = lib or C.lib()
    if shape.dtype == DType.BF16:
        # 2 bytes per element over PCIe, widened exactly on the host
        bits = t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        host = (bits.astype(np.uint32) << 16).view(np.float32)
    else:
        host = t.cpu().numpy()
        if shape.dtype == DType.U32:
            host = host.view(np.uint32)
        elif shape.dtype == DType.PRED:
            host = host.astype(np.bool_)
    return [host[p] for p in range(host.shape[0])]


# ---------------------------------------------------------------------------
# reference-compatible entry points
# ---------------------------------------------------------------------------

class _Compiled:
    """One compiled program behind the reference-signature entry points:
    the Executor, and from the second call on a CUDA graph of the whole
    step over static input buffers (each call then costs the uploads, one
    replay and the downloads -- no per-op host overhead, no recompilation)."""

    def __init__(self, program, n, dev, fuse):
        self.ex = Executor(program, nparts=n, device=dev, fuse=fuse)
        self.calls = 0
        self.graph = None
        self.static_in = None
        self.static_out = None


_COMPILED: dict = {}          # (id(program), fuse, device) -> (weakref, _Compiled)


def _compiled(program, n, dev, fuse) -> _Compiled:
    import weakref
    key = (id(program), bool(fuse), str(dev))
    hit = _COMPILED.get(key)
    if hit is not None and hit[0]() is program:
        return hit[1]
    entry = _Compiled(program, n, dev, fuse)
    try:
        ref = weakref.ref(program, lambda _r, k=key: _COMPILED.pop(k, None))
    except TypeError:         # not weak-referenceable: cache by identity only
        ref = (lambda p=program: p)
    _COMPILED[key] = (ref, entry)
    return entry


def evaluate_spmd(program, per_device_inputs: Mapping[int, Sequence[np.ndarray]],
                  fuse: bool = False, device=None) -> dict[int, list[np.ndarray]]:
    """Lockstep-equivalent evaluation of ``program`` on a simulated mesh of
    ``program.num_partitions`` partitions stacked on one B200
    (reference ``simulator.py:393-426``).  The compiled executor is cached
    per program; repeated calls replay a captured CUDA graph."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", 0)
    n = program.num_partitions
    params = program.graph.parameters
    for d in range(n):
        if len(per_device_inputs[d]) != len(params):
            raise EvalError(f"device {d}: expected {len(params)} inputs")
    entry = _compiled(program, n, dev, fuse)
    ex = entry.ex
    stacked = [upload_stacked([per_device_inputs[d][k] for d in range(n)], p.shape, dev)
               for k, p in enumerate(params)]
    with torch.cuda.device(dev):
        entry.calls += 1
        if entry.graph is None and entry.calls >= 2 and ex.comm is None:
            try:
                entry.static_in = [t.clone() for t in stacked]
                entry.graph, entry.static_out = ex.capture(entry.static_in)
            except Exception:     # noqa: BLE001 -- capture-incompatible program: stay eager
                entry.graph, entry.static_in = None, None
        if entry.graph is not None:
            for dst, src in zip(entry.static_in, stacked):
                dst.copy_(src)
            entry.graph.replay()
            outs = entry.static_out
        else:
            outs = ex.run(stacked)
        ex.check_errors()
    host = [download_stacked(o, program.graph.instr(oid).shape)
            for o, oid in zip(outs, program.graph.outputs)]
    return {d: [h[d] for h in host] for d in range(n)}


def evaluate_single(graph: Graph, inputs: Sequence[np.ndarray], fuse: bool = False,
                    device=None) -> list[np.ndarray]:
    """Single-device evaluation of an unpartitioned graph on one B200
    (reference ``simulator.py:304-319``; rejects SPMD-only opcodes)."""
    from .partitioner import SpmdProgram
    for ins in graph.instructions:
        if ins.opcode in COLLECTIVES or ins.opcode == Op.PARTITION_ID:
            raise EvalError(f"{ins.id}: {ins.opcode.value} is SPMD-only")
    if len(inputs) != len(graph.parameters):
        raise EvalError(f"expected {len(graph.parameters)} inputs, got {len(inputs)}")
    prog = SpmdProgram(graph, 1, {}, (), ())
    return evaluate_spmd(prog, {0: list(inputs)}, fuse=fuse, device=device)[0]


@dataclasses.dataclass
class EquivalenceReport:
    passed: bool
    max_abs_error: float
    max_rel_error: float
    collective_counts: dict[str, int]
    details: list[str] = dataclasses.field(default_factory=list)


def verify_equivalence(graph: Graph, annotated_graph: Graph, num_devices: int,
                       inputs: Sequence[np.ndarray], tolerance: float = 1e-4,
                       pad_value=0, plan: str = "reference",
                       fuse: bool = False) -> EquivalenceReport:
    """Partition, run on the B200 (simulated mesh), reassemble, and compare
    with the single-device B200 run (reference ``simulator.py:438-490``;
    metric: max|err| / max(max|expected|, 1) <= tolerance; ints exact)."""
    from .partitioner import partition
    from .sharding import assemble_data, shard_data
    expected = evaluate_single(graph, inputs, fuse=fuse)
    program = partition(annotated_graph, num_devices, plan=plan)
    devices = list(range(num_devices))
    per_dev: dict[int, list] = {d: [] for d in devices}
    for p, val in zip(annotated_graph.parameters, inputs):
        arr = np.asarray(val, dtype=np_dtype(p.shape.dtype)).reshape(p.shape.dims)
        shards = shard_data(arr, p.sharding, pad_value=pad_value, devices=devices)
        for d in devices:
            per_dev[d].append(shards[d])
    results = evaluate_spmd(program, per_dev, fuse=fuse)
    max_abs = max_rel = 0.0
    passed = True
    details = []
    for i, oid in enumerate(graph.outputs):
        shape = graph.instr(oid).shape
        actual = assemble_data({d: results[d][i] for d in devices},
                               program.output_shardings[i], shape,
                               rtol=max(tolerance, 1e-6))
        exp = expected[i]
        if shape.dtype.is_float:
            a64, e64 = np.asarray(actual, np.float64), np.asarray(exp, np.float64)
            err = float(np.max(np.abs(a64 - e64))) if e64.size else 0.0
            scale = float(np.max(np.abs(e64))) if e64.size else 0.0
            rel = err / max(scale, 1.0)
            max_abs, max_rel = max(max_abs, err), max(max_rel, rel)
            if rel > tolerance:       # NaN compares false, as in the reference
                passed = False
                details.append(f"output {oid}: rel error {rel} > {tolerance}")
        elif not np.array_equal(actual, exp):
            passed = False
            diff = np.max(np.abs(actual.astype(np.int64) - exp.astype(np.int64)))
            max_abs = max(max_abs, float(diff))
            details.append(f"output {oid}: integer mismatch")
    counts: dict[str, int] = {}
    for ins in program.graph.instructions:
        if ins.opcode in COLLECTIVES:
            counts[ins.opcode.value] = counts.get(ins.opcode.value, 0) + 1
    return EquivalenceReport(passed, max_abs, max_rel, counts, details)
