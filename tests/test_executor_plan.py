"""Executor planning on CPU (no kernels launched): fusion-group matching,
the peer-heap layout and the all-gather engine policy.  The executor is built
with a stand-in communicator; nothing here touches a GPU."""

import os

import pytest

from paper_2105_04663_b200 import partition, propagate
from paper_2105_04663_b200.executor import Executor
from paper_2105_04663_b200.ir import DType, Op
from paper_2105_04663_b200.workloads import transformer_layer


class FakeComm:
    handle = None
    peer = 0
    half = 0

    def ensure_workspace(self, nbytes, device):
        pass

    def reserve_fused(self, half_bytes):
        # spmd_comm_reserve_fused: grows only, 4 KiB granules
        self.half = max(self.half, (int(half_bytes) + 4095) // 4096 * 4096)
        return self.half

    def ensure_peer(self, nbytes, device):
        self.peer = nbytes


def _layer(mesh, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        world = mesh[0] * mesh[1]
        g, _ = transformer_layer(mesh, B=4, S=256, M=1024, N=8, D=64, H=4096, dtype=DType.BF16,
                                 with_inputs=False)
        ann, _ = propagate(g)
        prog = partition(ann, world, plan="fast")
        comm = FakeComm()
        ex = Executor(prog, nparts=1, device="cpu", comm=comm, partition_base=0, fuse=True,
                      overlap=False)
        return ex, comm
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("mesh", [(1, 2), (2, 2), (1, 4), (2, 4)])
def test_dot_reduce_scatter_fusion_matches_the_two_output_projections(mesh):
    ex, comm = _layer(mesh)
    rs = {k: v for k, v in ex._fused.items() if v[0] in ("dot_rs", "dot_rs_add")}
    assert len(rs) == 2   # attention out-projection and FFN-out (2-D finalized)
    for rid, (kind, dot, r, *resid) in rs.items():
        assert r.opcode == Op.REDUCE_SCATTER and dot.opcode == Op.DOT
        assert r.attrs["dim"] == dot.shape.rank - 1 and r.operands[0] == dot.id
        assert dot.id in ex._fused_skip
        step = next(s for s in ex.steps if s.ins.id == rid)
        assert not step.coll   # runs on the compute stream
        # both are the layer's residual adds: the add runs in the RS reduce
        assert kind == "dot_rs_add" and r.id in ex._fused_skip
        assert step.ops == tuple(dot.operands) + tuple(resid)
    # other fusions still planned
    kinds = {v[0] for v in ex._fused.values()}
    assert {"softmax", "attention", "dot_relu"} <= kinds


def test_peer_fusion_can_be_disabled():
    ex, _ = _layer((2, 2), SPMD_PEER_FUSION="0", SPMD_PEER_AG="0")
    assert not any(v[0] in ("dot_rs", "dot_rs_add") for v in ex._fused.values())
    assert ex._peer_ag == {} and ex._peer_engine == {}
    assert sum(1 for s in ex.steps if s.coll and s.ins.opcode == Op.REDUCE_SCATTER) == 2


def test_no_peer_fusion_without_a_communicator():
    g, _ = transformer_layer((2, 2), B=4, S=256, M=1024, N=8, D=64, H=4096, dtype=DType.BF16,
                             with_inputs=False)
    ann, _ = propagate(g)
    prog = partition(ann, 4, plan="fast")
    ex = Executor(prog, nparts=4, device="cpu", fuse=True, overlap=False)
    assert not any(v[0] in ("dot_rs", "dot_rs_add") for v in ex._fused.values())
    assert ex._peer_ag == {}


@pytest.mark.parametrize("mesh", [(2, 2), (2, 4)])
def test_peer_heap_layout_is_disjoint_and_aligned(mesh):
    ex, comm = _layer(mesh)
    rs_bytes = max(2 * r.shape.num_elements * len(r.attrs["subgroups"][0]) * 2
                   for _, _, r, *_ in (v for v in ex._fused.values()
                                       if v[0] in ("dot_rs", "dot_rs_add")))
    spans = []
    for aid, off in ex._peer_ag.items():
        ins = ex.by_id[aid]
        nb = ex._shape(ins.operands[0]).num_elements * ins.shape.dtype.itemsize
        assert off % 4096 == 0 and off >= rs_bytes
        spans.append((off, off + nb))
    spans.sort()
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 <= b0
    assert comm.peer >= spans[-1][1]
    all_gathers = [i.id for i in ex.graph.instructions if i.opcode == Op.ALL_GATHER]
    assert sorted(ex._peer_ag) == sorted(all_gathers)


def test_engine_policy_under_overlap():
    """Hoisted order: gathers with a GEMM between them and their consumer ride
    the copy engines; exposed pair gathers use the SM pull; exposed 4-way
    gathers stay on NCCL."""
    for mesh in [(2, 2), (2, 4)]:
        ex, _ = _layer(mesh)
        ex.steps = ex._hoist_collectives(ex.steps)
        ex.comm_stream = object()           # as if overlapping
        eng = ex._plan_peer_engines()
        order = [s.ins.id for s in ex.steps]
        for aid, e in eng.items():
            ins = ex.by_id[aid]
            gs = len(ins.attrs["subgroups"][0])
            i = order.index(aid)
            first_use = next(k for k in range(i + 1, len(order))
                             if aid in ex.steps[k].ops)
            between = ex.steps[i + 1:first_use]
            hidden = any(not s.coll and (s.ins.opcode == Op.DOT or
                                         (ex._fused.get(s.ins.id) or ("",))[0] in
                                         ("dot_relu", "attention", "dot_rs", "dot_rs_add"))
                         for s in between)
            assert e == (0 if hidden else (1 if gs <= 2 else -1)), (mesh, aid)
        # the weight gathers of the later projections are hidden, the first
        # activation gather is not
        assert 0 in eng.values() and any(v != 0 for v in eng.values())


@pytest.mark.parametrize("mesh", [(2, 2), (2, 4)])
def test_training_step_gradient_reduce_scatters_all_fuse(mesh):
    """Every weight-gradient reduce-scatter of the training step becomes a
    fused GEMM epilogue: column splits (last dim) and row splits (dim 0,
    dW[M, ...] split on M, wide kernel)."""
    from paper_2105_04663_b200.workloads import transformer_train_step
    g = transformer_train_step(mesh, dtype=DType.BF16, B=16, S=1024, M=8192, N=128, D=256,
                               H=65536)
    prog = partition(propagate(g)[0], mesh[0] * mesh[1], plan="fast")
    comm = FakeComm()
    ex = Executor(prog, nparts=1, device="cpu", comm=comm, partition_base=0, fuse=True,
                  overlap=False)
    rs = [i for i in prog.graph.instructions if i.opcode == Op.REDUCE_SCATTER]
    fused = {k: v for k, v in ex._fused.items() if v[0] in ("dot_rs", "dot_rs_add")}
    assert len(rs) == 12 and len(fused) == 12
    dims = {v[2].attrs["dim"] for v in fused.values()}
    assert 0 in dims and any(d > 0 for d in dims)
    assert comm.peer > 0
    _check_fused_parity_layout(ex, comm)


def _check_fused_parity_layout(ex, comm):
    """peer.cu fused_parity: parity p of a fused op with unit u bytes (slot /
    row) and n units per parity starts at unit p * ceil(H / u).  Parity 0 of
    EVERY op must lie in [0, H) and parity 1 in [H, 3H), so back-to-back
    fused ops of different sizes (the training step's 67M -> 268M -> 67M
    element reduce-scatters) never write into the buffer a peer is still
    reducing; staging / landing slots start at or after 3H."""
    H = comm.half
    assert H > 0 and ex._fused_half == H
    sizes = set()
    for kind, *spec in ex._fused.values():
        if kind in ("dot_rs", "dot_rs_add"):
            rs = spec[1]
            u, n = rs.shape.nbytes, len(rs.attrs["subgroups"][0])
        elif kind == "dot_a2a":
            a2a = spec[1]
            u, n = a2a.shape.nbytes // a2a.shape.dims[0], a2a.shape.dims[0]
        elif kind == "moe_dispatch_a2a":
            sh = spec[2].shape
            u, n = sh.dims[-1] * sh.dtype.itemsize, sh.num_elements // sh.dims[-1]
        else:
            continue
        sizes.add(u * n)
        k = -(-H // u)
        p0, p1 = (0, n * u), (k * u, k * u + n * u)
        assert p0[1] <= H <= p1[0] and p1[1] <= 3 * H, (kind, u, n, H)
    assert len(sizes) > 1          # the case the fixed stride exists for
    slots = list(ex._peer_ag.values()) + list(ex._peer_cp.values())
    assert all(off >= 3 * H for off in slots)


class _Arr:
    def __init__(self, *shape):
        self.shape = shape


@pytest.mark.parametrize("routed", [False, True])
def test_moe_all_to_alls_fuse(routed):
    """C3 over 4: the expert FFN-out einsum + combine all-to-all fuse into the
    GEMM's row-scatter epilogue; the dispatch exchange fuses with the dense
    dispatch einsum, or -- under a declared routing -- with the dispatch
    gather (rows pushed into the owners' heaps)."""
    from paper_2105_04663_b200.executor import Routing
    from paper_2105_04663_b200.workloads import moe_layer
    g, _ = moe_layer(4, E=8, B=64, S=512, C=160, M=4096, H=16384, dtype=DType.BF16,
                     with_inputs=False)
    ann, _ = propagate(g)
    prog = partition(ann, 4, plan="fast")
    routing = None
    if routed:
        r = Routing(_Arr(1, 16, 512), _Arr(1, 16, 512), _Arr(1, 16, 512))
        idx = {p.id: p.attrs["index"] for p in ann.parameters}
        routing = {idx["dispatch"]: r, idx["combine"]: r}
    ex = Executor(prog, nparts=1, device="cpu", comm=FakeComm(), partition_base=0, fuse=True,
                  overlap=False, routing=routing)
    kinds = sorted(v[0] for k, v in ex._fused.items() if k not in ex._fused_skip)
    a2a = [i.id for i in prog.graph.instructions if i.opcode == Op.ALL_TO_ALL]
    assert len(a2a) == 2
    if routed:
        assert ex._fused[a2a[0]][0] == "moe_dispatch_a2a" and ex._fused[a2a[1]][0] == "dot_a2a"
        assert "moe_combine" in kinds
    else:
        assert [ex._fused[x][0] for x in a2a] == ["dot_a2a", "dot_a2a"]
    assert not any(s.coll for s in ex.steps if s.ins.id in a2a)


@pytest.mark.parametrize("mesh", [(1, 1), (2, 2), (2, 4)])
def test_training_step_backward_chains_fuse(mesh):
    """Softmax backward (multiply/reduce/broadcast/subtract/multiply) and ReLU
    backward (compare/select over broadcast zeros) each become one kernel;
    the FFN-in GEMM takes the ReLU epilogue and the mask reads relu(h)."""
    from paper_2105_04663_b200.workloads import transformer_train_step
    g = transformer_train_step(mesh, dtype=DType.BF16, B=16, S=1024, M=8192, N=128, D=256,
                               H=65536)
    prog = partition(propagate(g)[0], mesh[0] * mesh[1], plan="fast")
    ex = Executor(prog, nparts=1, device="cpu", comm=FakeComm(), partition_base=0, fuse=True,
                  overlap=False)
    by = ex.by_id
    sb = [v for v in ex._fused.values() if v[0] == "softmax_bwd"]
    rb = [v for v in ex._fused.values() if v[0] == "relu_bwd"]
    assert len(sb) == 1 and len(rb) == 1
    assert by[sb[0][1]].opcode == Op.DIVIDE          # probs
    relu = by[rb[0][1]]
    assert relu.opcode == Op.RELU and ex._fused[relu.id][0] == "dot_relu"
    skipped = {by[i].opcode for i in ex._fused_skip}
    assert {Op.COMPARE, Op.SUBTRACT, Op.REDUCE, Op.BROADCAST, Op.MULTIPLY} <= skipped
    assert not any(s.ins.opcode in (Op.COMPARE, Op.SUBTRACT) for s in ex.steps)


def test_backward_fusion_can_be_disabled():
    ex, _ = _layer((2, 2))
    from paper_2105_04663_b200.workloads import transformer_train_step
    os.environ["SPMD_BWD_FUSION"] = "0"
    try:
        g = transformer_train_step((2, 2), dtype=DType.BF16, B=4, S=256, M=256, N=4, D=64, H=512)
        prog = partition(propagate(g)[0], 4, plan="fast")
        ex = Executor(prog, nparts=1, device="cpu", comm=FakeComm(), partition_base=0, fuse=True,
                      overlap=False)
    finally:
        os.environ.pop("SPMD_BWD_FUSION")
    assert not any(v[0] in ("softmax_bwd", "relu_bwd") for v in ex._fused.values())


@pytest.mark.parametrize("push_params", ["1", "0"])
@pytest.mark.parametrize("mesh", [(2, 2), (1, 4), (2, 4)])
def test_parameter_gathers_are_prestaged(mesh, push_params):
    """Overlapped runs stage the parameter all-gathers a GEMM hides (weights)
    into the peer heap at the step start: engine 4 (copy-engine pulls only).
    The exposed ones (the step's first gathers) are pushed straight from the
    parameter (engine 1 / -1, push zone) -- unless SPMD_PEER_AG_PUSH_PARAMS=0,
    which stages every one.  Activation gathers keep their engine unless
    SPMD_PEER_STAGE_ACT."""
    os.environ["SPMD_PEER_AG_PUSH_PARAMS"] = push_params
    try:
        ex, _ = _layer(mesh)
        ex.steps = ex._hoist_collectives(ex.steps)
        ex.comm_stream = object()
        ex.comm_streams = [ex.comm_stream]
        ex._peer_engine = ex._plan_peer_engines()
        planned = dict(ex._peer_engine)
        ex._staged_exposed, ex._act_staged = [], set()
        staged = ex._plan_staged_gathers()
        # (the executor was built without overlap: drop the parameter push
        # zones planned then and re-plan them for the overlapped engines)
        pset = {p.id for p in ex.params}
        ex._peer_agp = {k: v for k, v in ex._peer_agp.items()
                        if ex.by_id[k].operands[0] not in pset}
        ex._add_param_push_zones()
    finally:
        os.environ.pop("SPMD_PEER_AG_PUSH_PARAMS")
    pids = [p.id for p in ex.params]
    pushed = 0
    for aid in ex._peer_ag:
        src = ex.by_id[ex.by_id[aid].operands[0]]
        if src.opcode == Op.PARAMETER:
            if push_params == "1" and planned.get(aid, -1) not in (0, 3):
                assert aid not in staged and ex._peer_engine[aid] in (1, -1)
                assert aid in ex._peer_agp
                pushed += 1
            else:
                assert staged[aid] == pids.index(src.id) and ex._peer_engine[aid] == 4
                assert aid not in ex._peer_agp
        else:
            assert aid not in staged and ex._peer_engine[aid] != 4
    if push_params == "1":
        assert pushed >= 1          # the step's first gathers are exposed
    if mesh[0] > 1:          # weights gathered over the data axis
        assert len(staged) + pushed >= 6
    assert not ex._act_staged


def test_prestaging_can_be_disabled():
    os.environ["SPMD_PEER_STAGE"] = "0"
    try:
        ex, _ = _layer((2, 2))
        ex.comm_streams = [object()]
        assert ex._plan_staged_gathers() == {}
    finally:
        os.environ.pop("SPMD_PEER_STAGE")


def test_halo_slab_slices_fuse_into_the_peer_permute():
    """C4 over 4: every halo slab (slice of one dim -> collective-permute)
    becomes one peer permute reading the slab rows from the conv output."""
    from paper_2105_04663_b200.workloads import conv_stack
    g, _ = conv_stack((4,), N=8, H=64, W=64, C=128, layers=2, with_inputs=False)
    prog = partition(propagate(g)[0], 4, plan="fast")
    ex = Executor(prog, nparts=1, device="cpu", comm=FakeComm(), partition_base=0, fuse=True,
                  overlap=False)
    cps = [i for i in prog.graph.instructions if i.opcode == Op.COLLECTIVE_PERMUTE]
    assert len(cps) == 4
    for cp in cps:
        kind, sl, cp2, axis = ex._fused[cp.id]
        assert kind == "slice_cp" and cp2 is cp and axis == 1 and sl.id in ex._fused_skip
        assert cp.id in ex._peer_cp
    assert not any(s.ins.opcode == Op.SLICE for s in ex.steps)
