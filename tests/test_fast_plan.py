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
