"""Zero-extent edge cases on the B200 path vs the CPU oracle (simulator.py
semantics, restated in oracle/evaluator.py): empty operands of Dot / Reduce /
Pad / Slice / Concat / elementwise ops, a contraction over an empty dim
(zeros), a reduction over an empty dim (the identity of each kind,
simulator.py:80-90), and collectives of empty shards on a simulated mesh.
C5's 7-over-8 layout (last shard with 0 valid rows) is in the golden set;
these are the degenerate shapes around it."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(g, ins):
    from oracle import evaluator as O
    from paper_2105_04663_b200.executor import evaluate_single
    got = evaluate_single(g, ins)
    want = O.evaluate_single(g, ins)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a.shape == b.shape, (a.shape, b.shape)
        np.testing.assert_array_equal(a, b)


def test_dot_with_empty_rows_and_empty_contraction():
    from paper_2105_04663_b200 import GraphBuilder, Op, Shape, DType
    b = GraphBuilder("g")
    x = b.parameter(Shape((0, 4), DType.F32))
    y = b.parameter(Shape((4, 3), DType.F32))
    u = b.parameter(Shape((2, 0), DType.F32))
    v = b.parameter(Shape((0, 5), DType.F32))
    dd = {"lhs_batch": (), "rhs_batch": (), "lhs_contracting": (1,), "rhs_contracting": (0,)}
    d0 = b.add(Op.DOT, [x, y], dict(dd))
    d1 = b.add(Op.DOT, [u, v], dict(dd))        # K = 0: all zeros
    g = b.build([d0, d1])
    _check(g, [np.zeros((0, 4), np.float32), np.ones((4, 3), np.float32),
               np.zeros((2, 0), np.float32), np.zeros((0, 5), np.float32)])


@pytest.mark.parametrize("kind", ["sum", "max", "min", "prod"])
@pytest.mark.parametrize("dt", ["f32", "s32"])
def test_reduce_over_an_empty_dim_gives_the_identity(kind, dt):
    """sum / prod: the identity, as the reference (np.add / np.multiply
    .reduce).  max / min: the reference has no result -- numpy's
    maximum / minimum .reduce raise on a zero-size axis (simulator.py:72-77)
    -- and the B200 path returns the kind's identity (the value
    simulator.py:80-90 reduce_identity defines, XLA's semantics): a
    documented, strictly more lenient divergence."""
    from paper_2105_04663_b200 import GraphBuilder, Op, Shape, DType
    from paper_2105_04663_b200.ir import ReduceKind
    dtype = DType.F32 if dt == "f32" else DType.S32
    npdt = np.float32 if dt == "f32" else np.int32
    ident = {"sum": 0, "prod": 1,
             "max": -np.inf if dt == "f32" else np.iinfo(np.int32).min,
             "min": np.inf if dt == "f32" else np.iinfo(np.int32).max}[kind]
    b = GraphBuilder("g")
    z = b.parameter(Shape((5, 0), dtype))
    init = b.constant(npdt(ident), Shape((), dtype))
    r = b.add(Op.REDUCE, [z, init], {"kind": ReduceKind(kind), "dims": (1,)})
    g = b.build([r])
    if kind in ("sum", "prod"):
        _check(g, [np.zeros((5, 0), npdt)])
        return
    from oracle import evaluator as O
    from paper_2105_04663_b200.executor import evaluate_single
    with pytest.raises(ValueError):
        O.evaluate_single(g, [np.zeros((5, 0), npdt)])
    got = evaluate_single(g, [np.zeros((5, 0), npdt)])[0]
    np.testing.assert_array_equal(got, np.full((5,), ident, npdt))


def test_data_formatting_of_empty_and_to_empty():
    from paper_2105_04663_b200 import GraphBuilder, Op, Shape, DType
    b = GraphBuilder("g")
    x = b.parameter(Shape((0, 3), DType.F32))
    w = b.parameter(Shape((4, 3), DType.F32))
    pv = b.constant(np.float32(7), Shape((), DType.F32))
    p = b.add(Op.PAD, [x, pv], {"low": (1, 0), "high": (2, 0), "interior": (0, 0)})
    s = b.add(Op.SLICE, [w, ], {"starts": (2, 0), "limits": (2, 3), "strides": (1, 1)})
    c = b.add(Op.CONCAT, [x, w], {"dim": 0})
    e = b.add(Op.NEGATE, [x])
    g = b.build([p, s, c, e])
    _check(g, [np.zeros((0, 3), np.float32),
               np.arange(12, dtype=np.float32).reshape(4, 3)])


@pytest.mark.parametrize("op", ["all-gather", "all-to-all", "all-reduce", "collective-permute"])
def test_collectives_of_empty_shards(op):
    from oracle import evaluator as O
    from paper_2105_04663_b200.executor import evaluate_spmd
    from paper_2105_04663_b200.ir import DType, Graph, Instruction, Op, Shape, ReduceKind
    from paper_2105_04663_b200.partitioner import SpmdProgram
    n = 4
    groups = ((0, 1, 2, 3),)
    shp = Shape((0, 8), DType.F32)
    attrs = {"all-gather": {"dim": 0, "subgroups": groups},
             "all-to-all": {"split_dim": 1, "concat_dim": 0, "subgroups": groups},
             "all-reduce": {"kind": ReduceKind.SUM, "subgroups": groups},
             "collective-permute": {"pairs": ((0, 1), (1, 2))}}[op]
    out = {"all-gather": (0, 8), "all-to-all": (0, 2), "all-reduce": (0, 8),
           "collective-permute": (0, 8)}[op]
    p = Instruction("x", Op.PARAMETER, (), {"index": 0, "shape": shp}, shp)
    ins = Instruction("c", Op(op), ("x",), attrs, Shape(out, DType.F32))
    g = Graph("coll", (p, ins), ("c",))
    per = {d: np.zeros((0, 8), np.float32) for d in range(n)}
    got = evaluate_spmd(SpmdProgram(g, n, {}, (), ()), {d: [per[d]] for d in range(n)})
    want = O.collective(ins, per, list(range(n)))
    for d in range(n):
        assert got[d][0].shape == want[d].shape
