"""The fast (minimal-reshard) planner keeps every per-op sharding of the
reference plan and must compute the same function: execute its programs with
the CPU oracle on every golden case and compare the assembled outputs with
the reference's single-device results (f32 1e-4 normwise, ints exact)."""

import numpy as np
import pytest

from oracle import evaluator as O
from paper_2105_04663_b200 import collective_stats, partition, propagate
from paper_2105_04663_b200.sharding import assemble_data, shard_data

import golden_io as G

CASES = [(k, c["name"]) for k in G.KINDS for c in G.cases(k) if "expected" in c]


def _case(kind, name):
    return next(c for c in G.cases(kind) if c["name"] == name)


@pytest.mark.parametrize("kind,name", CASES)
def test_fast_plan_equivalent(kind, name):
    case = _case(kind, name)
    g = G.graph(case)
    ann, _ = propagate(g)
    n = case["num_devices"]
    prog = partition(ann, n, plan="fast")
    assert [s.format() for s in prog.output_shardings] == case["output_shardings"]
    devices = list(range(n))
    per = {d: [] for d in devices}
    for p, x in zip(ann.parameters, G.inputs(case)):
        sh = shard_data(x, p.sharding, devices=devices)
        for d in devices:
            per[d].append(sh[d])
    res = O.evaluate_spmd(prog, per)
    for i, oid in enumerate(g.outputs):
        shape = g.instr(oid).shape
        full = assemble_data({d: res[d][i] for d in devices}, prog.output_shardings[i], shape,
                             rtol=1e-4)
        want = G.expected(case)[i]
        if shape.dtype.is_float:
            _, rel = O.rel_error(full, want)
            assert not rel > 1e-4, rel
        else:
            np.testing.assert_array_equal(full, want)


def test_fast_plan_moves_less_data():
    """On the 2x4 transformer layer the fast plan is the GSPMD-proper set:
    activation AG over Y, weight AG over X, RS over Y (8 AG + 2 RS)."""
    case = G.case_by_name("c2_2x4")
    ann, _ = propagate(G.graph(case))
    ref = collective_stats(partition(ann, 8))
    fast = collective_stats(partition(ann, 8, plan="fast"))
    assert fast["counts"] == {"all-gather": 8, "reduce-scatter": 2}
    assert fast["total_bytes"] < ref["total_bytes"] / 4


def _feature_conv(mesh_dims, Co, dtype):
    from paper_2105_04663_b200.ir import ConvDims, DType, GraphBuilder, Op, Shape, WindowDim
    from paper_2105_04663_b200.sharding import DeviceMesh, mesh_split
    mesh = DeviceMesh.default(*mesh_dims)
    b = GraphBuilder("featconv", mesh)
    N, H, W, Ci = 2, 8, 6, 4
    cd = ConvDims(lhs_batch=0, lhs_feature=3, lhs_spatial=(1, 2), rhs_in_feature=2,
                  rhs_out_feature=3, rhs_spatial=(0, 1), out_batch=0, out_feature=3,
                  out_spatial=(1, 2))
    win = (WindowDim(3, 1, 1, 1), WindowDim(3, 1, 1, 1))
    x = b.parameter(Shape((N, H, W, Ci), dtype), sharding=mesh_split(4, mesh, [-1, 0, -1, -1]),
                    id="x")
    w = b.parameter(Shape((3, 3, Ci, Co), dtype), sharding=mesh_split(4, mesh, [-1, -1, -1, 1]),
                    id="w")
    y = b.add(Op.CONVOLUTION, [x, w], {"conv_dims": cd, "window": win},
              sharding=mesh_split(4, mesh, [-1, 0, -1, 1]), id="y")
    g = b.build([y])
    rng = np.random.default_rng(Co)
    ins = [rng.integers(-4, 5, (N, H, W, Ci)).astype(np.int32),
           rng.integers(-4, 5, (3, 3, Ci, Co)).astype(np.int32)]
    if dtype == DType.F32:
        ins = [i.astype(np.float32) for i in ins]
    return g, ins


@pytest.mark.parametrize("Co", [8, 6, 7])
def test_fast_plan_partitions_conv_output_features(Co):
    """Feature-dim conv partitioning (the reference forces
    the weights replicated, formatting.py:507): with the output tiled on its
    feature dim, the fast plan tiles the weights' output-feature dim the same
    way -- the only collectives left are the halo permutes -- and the result
    equals the single-device oracle exactly (int32 conv), even (Co=8) and
    uneven (Co=6, 7 over 2) channel counts."""
    from paper_2105_04663_b200.ir import DType, Op
    g, ins = _feature_conv((2, 2), Co, DType.S32)
    ann, _ = propagate(g)
    want = O.evaluate_single(g, ins)[0]
    for plan in ("reference", "fast"):
        prog = partition(ann, 4, plan=plan)
        kinds = {i.opcode for i in prog.graph.instructions}
        if plan == "fast":
            colls = {i.opcode for i in prog.graph.instructions
                     if i.opcode in (Op.ALL_GATHER, Op.ALL_REDUCE, Op.ALL_TO_ALL,
                                     Op.REDUCE_SCATTER)}
            assert not colls, colls
            conv = next(i for i in prog.graph.instructions if i.opcode == Op.CONVOLUTION)
            assert conv.shape.dims[3] == -(-Co // 2)        # half the filters per device
        devices = list(range(4))
        per = {d: [] for d in devices}
        for p, x in zip(ann.parameters, ins):
            sh = shard_data(x, p.sharding, devices=devices)
            for d in devices:
                per[d].append(sh[d])
        res = O.evaluate_spmd(prog, per)
        full = assemble_data({d: res[d][0] for d in devices}, prog.output_shardings[0],
                             g.instr(g.outputs[0]).shape)
        np.testing.assert_array_equal(full, want)
