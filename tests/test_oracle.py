"""Pin the CPU oracle (``oracle/evaluator.py``) to the reference: run the
oracle on the reference's own SPMD programs and inputs and require the
reference's recorded outputs bit-for-bit (single-device oracle, every
device's SPMD result, and the collective known-answer cases)."""

import numpy as np
import pytest

from oracle import evaluator as O
from paper_2105_04663_b200.ir import DType, Instruction, Op, Shape, instruction_from_json
from paper_2105_04663_b200.partitioner import SpmdProgram

import golden_io as G

CASES = [(k, c["name"]) for k in G.KINDS for c in G.cases(k) if "expected" in c]


def _case(kind, name):
    return next(c for c in G.cases(kind) if c["name"] == name)


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("kind,name", CASES)
def test_oracle_matches_reference(kind, name):
    case = _case(kind, name)
    g = G.graph(case)
    ins = G.inputs(case)
    for got, want in zip(O.evaluate_single(g, ins), G.expected(case)):
        _same(got, want)
    prog = SpmdProgram(G.program(case), case["num_devices"], {}, (), ())
    a = G.arrays()
    per_dev = {}
    from paper_2105_04663_b200.sharding import Sharding, shard_data
    shardings = [Sharding.parse(s) for s in case["param_shardings"]]
    devices = list(range(case["num_devices"]))
    for d in devices:
        per_dev[d] = []
    for s, x in zip(shardings, ins):
        sh = shard_data(x, s, devices=devices)
        for d in devices:
            per_dev[d].append(sh[d])
    got = O.evaluate_spmd(prog, per_dev)
    for d, outs in G.spmd_outputs(case).items():
        for x, y in zip(got[d], outs):
            _same(x, y)


def test_collective_known_answers():
    a = G.arrays()
    for k, c in enumerate(G.cases("extra")["collectives"]):
        ins = instruction_from_json({"id": "c", "op": c["op"], "operands": ["x"],
                                     "attrs": c["attrs"],
                                     "shape": [c["shape"], c["dtype"]]})
        per = {d: a[f"coll{k}/in{d}"] for d in c["devices"]}
        got = O.collective(ins, per, c["devices"])
        for d in c["devices"]:
            _same(got[d], a[f"coll{k}/out{d}"])


def test_reference_known_answers():
    # minispmd tests/test_simulator.py:38-107 (known answers restated).
    def run(op, args, attrs, shape):
        ins = Instruction("t", op, tuple(f"a{i}" for i in range(len(args))), attrs, shape)
        return O.eval_instruction(ins, [np.asarray(x) for x in args])
    i32 = lambda v: np.array(v, dtype=np.int32)
    assert run(Op.DIVIDE, [i32([7, -7, 7, -7]), i32([2, 2, -2, -2])], {},
               Shape((4,), DType.S32)).tolist() == [3, -3, -3, 3]
    with pytest.raises(O.OracleDivideByZero):
        run(Op.DIVIDE, [i32([1]), i32([0])], {}, Shape((1,), DType.S32))
    assert run(Op.PAD, [np.array([1, 2, 3], np.float32), np.float32(9)],
               {"low": (1,), "high": (1,), "interior": (1,)},
               Shape((7,))).tolist() == [9, 1, 9, 2, 9, 3, 9]
    assert run(Op.DYNAMIC_SLICE, [np.arange(5, dtype=np.int32), np.int32(4)],
               {"sizes": (3,)}, Shape((3,), DType.S32)).tolist() == [2, 3, 4]
    assert run(Op.ROTATE, [np.arange(6, dtype=np.int32)], {"dim": 0, "amount": 2},
               Shape((6,), DType.S32)).tolist() == [2, 3, 4, 5, 0, 1]
    assert run(Op.SHIFT, [np.arange(6, dtype=np.int32), np.int32(-1)],
               {"dim": 0, "amount": -2}, Shape((6,), DType.S32)).tolist() == [2, 3, 4, 5, -1, -1]
    assert run(Op.SHIFT, [np.arange(6, dtype=np.int32), np.int32(-1)],
               {"dim": 0, "amount": 2}, Shape((6,), DType.S32)).tolist() == [-1, -1, 0, 1, 2, 3]


def test_bf16_rounding():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 65504.0, np.inf], np.float32)
    y = O.to_bf16(x)
    assert y[0] == 1.0 and y[1] == 1.0          # tie -> even
    assert y[2] == np.float32(1.0078125)
    assert np.isinf(y[5])
    assert (y.view(np.uint32) & 0xFFFF).max() == 0
