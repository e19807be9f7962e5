"""GPU parity: the CUDA path (through the C ABI) against the reference.

* Every golden case: execute the REFERENCE's own SPMD program on the B200
  (loopback collectives, all partitions on one GPU) with the reference's
  per-device inputs and compare every device's outputs with the reference
  evaluator's: integers bit-exact, f32 within 1e-5 normwise (Dot/Conv
  accumulate in fp64 like the reference; only float reductions re-associate).
* ``verify_equivalence`` through the public API for the named configs
  (reference tolerance 1e-4), with both planners and with fusions on.
* Known-answer collective cases and error semantics.
"""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

CASES = [(k, c["name"]) for k in G.KINDS for c in G.cases(k) if "spmd" in c]
NAMED = [c["name"] for k in ("named", "c5w") for c in G.cases(k) if "spmd" in c]


def _case(kind, name):
    return next(c for c in G.cases(kind) if c["name"] == name)


def _close(got, want, dtype_is_float, tol=1e-5):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    if not dtype_is_float:
        np.testing.assert_array_equal(got, want)
        return
    g64, w64 = got.astype(np.float64), want.astype(np.float64)
    finite = np.isfinite(w64)
    np.testing.assert_array_equal(np.isnan(g64), np.isnan(w64))
    np.testing.assert_array_equal(g64[~finite & ~np.isnan(w64)], w64[~finite & ~np.isnan(w64)])
    if finite.any():
        err = np.max(np.abs(g64[finite] - w64[finite]))
        scale = max(1.0, np.max(np.abs(w64[finite])))
        assert err / scale <= tol, (err, scale)


@pytest.mark.parametrize("kind,name", CASES)
def test_reference_program_on_b200(kind, name):
    from paper_2105_04663_b200.executor import evaluate_spmd
    from paper_2105_04663_b200.partitioner import SpmdProgram
    from paper_2105_04663_b200.sharding import Sharding, shard_data
    case = _case(kind, name)
    prog_graph = G.program(case)
    n = case["num_devices"]
    prog = SpmdProgram(prog_graph, n, {}, (), ())
    devices = list(range(n))
    per_dev = {d: [] for d in devices}
    for s, x in zip(case["param_shardings"], G.inputs(case)):
        sh = shard_data(x, Sharding.parse(s), devices=devices)
        for d in devices:
            per_dev[d].append(sh[d])
    got = evaluate_spmd(prog, per_dev)
    want = G.spmd_outputs(case)
    for d in devices:
        for oid, x, y in zip(prog_graph.outputs, got[d], want[d]):
            _close(x, y, prog_graph.instr(oid).shape.dtype.is_float)


@pytest.mark.parametrize("name", NAMED)
@pytest.mark.parametrize("plan,fuse", [("reference", False), ("fast", True)])
def test_verify_equivalence_named(name, plan, fuse):
    from paper_2105_04663_b200 import propagate, verify_equivalence
    case = G.case_by_name(name)
    g = G.graph(case)
    annotated, _ = propagate(g)
    rep = verify_equivalence(g, annotated, case["num_devices"], G.inputs(case),
                             plan=plan, fuse=fuse)
    assert rep.passed, rep.details
    if plan == "reference":
        assert rep.collective_counts == case["verify"]["counts"]


@pytest.mark.parametrize("kind,name", CASES)
def test_fast_plan_two_streams_on_b200(kind, name):
    """Fast plan + fusions + comm-stream overlap (loopback collectives on a
    second stream, CUDA-graph captured) against the reference's outputs."""
    import torch
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor, download_stacked, upload_stacked
    from paper_2105_04663_b200.sharding import assemble_data, shard_data
    case = _case(kind, name)
    g = G.graph(case)
    ann, _ = propagate(g)
    n = case["num_devices"]
    prog = partition(ann, n, plan="fast")
    dev = torch.device("cuda", 0)
    stacked = []
    for p_src, x, p in zip(ann.parameters, G.inputs(case), prog.graph.parameters):
        sh = shard_data(x, p_src.sharding, devices=range(n))
        stacked.append(upload_stacked([sh[d] for d in range(n)], p.shape, dev))
    ex = Executor(prog, nparts=n, device=dev, fuse=True, overlap=True)
    graph, outs = ex.capture(stacked)
    graph.replay()
    torch.cuda.synchronize()
    for i, oid in enumerate(g.outputs):
        shape = g.instr(oid).shape
        per = download_stacked(outs[i], prog.graph.instr(prog.graph.outputs[i]).shape)
        full = assemble_data({d: per[d] for d in range(n)}, prog.output_shardings[i], shape,
                             rtol=1e-5)
        _close(full, G.expected(case)[i], shape.dtype.is_float, tol=1e-4)


def test_single_device_matches_reference_oracle():
    from paper_2105_04663_b200 import evaluate_single
    for c in G.cases("named"):
        if "expected" not in c:
            continue
        g = G.graph(c)
        for oid, got, want in zip(g.outputs, evaluate_single(g, G.inputs(c)), G.expected(c)):
            _close(got, want, g.instr(oid).shape.dtype.is_float, tol=1e-5)


def test_collective_known_answers():
    from paper_2105_04663_b200.executor import evaluate_spmd
    from paper_2105_04663_b200.ir import Graph, Instruction, Op, Shape, DType, instruction_from_json
    from paper_2105_04663_b200.partitioner import SpmdProgram
    a = G.arrays()
    for k, c in enumerate(G.cases("extra")["collectives"]):
        # (the recorded "shape" attr is informational; the reference evaluator
        # ignores it -- take the true output shape from the recorded result)
        out_shape = list(a[f"coll{k}/out{c['devices'][0]}"].shape)
        ins = instruction_from_json({"id": "c", "op": c["op"], "operands": ["x"],
                                     "attrs": c["attrs"], "shape": [out_shape, c["dtype"]]})
        x_in = a[f"coll{k}/in0"]
        dt = DType(c["dtype"])
        p = Instruction("x", Op.PARAMETER, (), {"index": 0, "shape": Shape(x_in.shape, dt)},
                        Shape(x_in.shape, dt))
        g = Graph("coll", (p, ins), ("c",))
        n = len(c["devices"])
        got = evaluate_spmd(SpmdProgram(g, n, {}, (), ()),
                            {d: [a[f"coll{k}/in{d}"]] for d in c["devices"]})
        for d in c["devices"]:
            # loopback reductions fold in group order: bit-exact even for f32
            np.testing.assert_array_equal(got[d][0], a[f"coll{k}/out{d}"])


def test_divide_by_zero_and_subgroup_errors():
    from paper_2105_04663_b200 import GraphBuilder, Op, Shape, DType
    from paper_2105_04663_b200.executor import DivideByZero, SubgroupMismatch, evaluate_single, \
        evaluate_spmd
    from paper_2105_04663_b200.ir import Graph, Instruction
    from paper_2105_04663_b200.partitioner import SpmdProgram
    b = GraphBuilder("g")
    x = b.parameter(Shape((4,), DType.S32))
    y = b.parameter(Shape((4,), DType.S32))
    q = b.add(Op.DIVIDE, [x, y])
    g = b.build([q])
    out = evaluate_single(g, [np.array([7, -7, 7, -7], np.int32), np.array([2, 2, -2, -2], np.int32)])
    assert out[0].tolist() == [3, -3, -3, 3]
    with pytest.raises(DivideByZero):
        evaluate_single(g, [np.array([1, 1, 1, 1], np.int32), np.array([1, 0, 1, 1], np.int32)])
    p = Instruction("x", Op.PARAMETER, (), {"index": 0, "shape": Shape((1,), DType.S32)},
                    Shape((1,), DType.S32))
    cp = Instruction("c", Op.COLLECTIVE_PERMUTE, ("x",), {"pairs": ((0, 1), (1, 1))},
                     Shape((1,), DType.S32))
    with pytest.raises(SubgroupMismatch):
        evaluate_spmd(SpmdProgram(Graph("g", (p, cp), ("c",)), 2, {}, (), ()),
                      {0: [np.array([1], np.int32)], 1: [np.array([2], np.int32)]})
