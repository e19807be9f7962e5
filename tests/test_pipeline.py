"""Shifting-buffer pipelines (reference pipeline.py; tests/test_pipeline.py).

* The builder reproduces the reference's graphs exactly (JSON of the golden
  pipeline cases recorded by running the reference, tests/golden/make_golden.py);
  the generic host-parity / oracle / GPU-parity suites then cover their
  propagation, SPMD programs and outputs like every other golden case.
* Bubble accounting known answers (reference tests/test_pipeline.py:39-61).
* Functional equivalence with a sequential stage loop, on the oracle.
* Lowering: the sharded stage shift becomes collective-permutes, never an
  all-gather of the state.
"""

import os
import sys
from fractions import Fraction

import numpy as np
import pytest

import golden_io as G

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))

from paper_2105_04663_b200 import partition, propagate  # noqa: E402
from paper_2105_04663_b200.ir import Op, Shape, graph_to_json  # noqa: E402
from paper_2105_04663_b200.partitioner import collective_stats  # noqa: E402
from paper_2105_04663_b200.pipeline import (PipelineConfig, ShapeMismatch,  # noqa: E402
                                            bubble_stats, build_pipeline, schedule_slots)
from paper_2105_04663_b200.sharding import DeviceMesh, Sharding, mesh_split  # noqa: E402

PIPE_CASES = [c for c in G.cases("named") if "pipeline" in c]


def _body(kind):
    def add(b, x, ws):
        return b.add(Op.ADD, [x, ws[0]])

    def dot(b, x, ws):
        y = b.add(Op.DOT, [x, ws[0]], {"lhs_batch": (0,), "rhs_batch": (0,),
                                        "lhs_contracting": (2,), "rhs_contracting": (1,)})
        return b.add(Op.ADD, [x, y])
    return add if kind == "add" else dot


def _rebuild(case):
    p = case["pipeline"]
    L, R, sdims, kind = p["L"], p["R"], tuple(p["state_dims"]), p["body"]
    mesh = DeviceMesh.default(case["num_devices"])
    cfg = PipelineConfig(L, p["M"], p["schedule"], R)
    wdims = (sdims[-1], sdims[-1]) if kind == "dot" else sdims
    lead = (L,) if p["schedule"] == "gpipe" else (L, R)
    st_sh = mesh_split(1 + len(sdims), mesh, [0] + [-1] * len(sdims))
    w_sh = mesh_split(len(lead) + len(wdims), mesh, [0] + [-1] * (len(lead) + len(wdims) - 1))
    return cfg, build_pipeline(cfg, mesh, sdims, _body(kind), [Shape(wdims)],
                               input_sharding=Sharding.replicated(), state_sharding=st_sh,
                               weight_shardings=[w_sh])


def test_golden_pipelines_present():
    assert len(PIPE_CASES) == 5
    assert {c["pipeline"]["schedule"] for c in PIPE_CASES} == {"gpipe", "circular"}


@pytest.mark.parametrize("case", PIPE_CASES, ids=lambda c: c["name"])
def test_builder_reproduces_reference_graph(case):
    cfg, g = _rebuild(case)
    assert graph_to_json(g) == case["graph"]
    assert bubble_stats(cfg).to_json() == case["pipeline"]["bubble"]


class TestBubbleStats:
    def test_gpipe_formula(self):
        st = bubble_stats(PipelineConfig(4, 16))
        assert st.total_iterations == 19
        assert st.bubble_ratio == Fraction(3, 19)
        assert st.padded_applications == 12

    def test_single_stage_has_no_bubble(self):
        assert bubble_stats(PipelineConfig(1, 5)).bubble_ratio == 0

    def test_l8_m32(self):
        assert bubble_stats(PipelineConfig(8, 32)).bubble_ratio == Fraction(7, 39)

    def test_circular_beats_gpipe_at_equal_depth(self):
        assert bubble_stats(PipelineConfig(8, 32, "circular", 2)).bubble_ratio < \
            bubble_stats(PipelineConfig(16, 32)).bubble_ratio

    def test_json(self):
        j = bubble_stats(PipelineConfig(4, 16)).to_json()
        assert j["bubble_ratio"] == [3, 19] and j["total_iterations"] == 19

    def test_every_microbatch_visits_every_stage_once_per_lap(self):
        for cfg in (PipelineConfig(3, 5), PipelineConfig(3, 7, "circular", 2)):
            seen = {}
            for row in schedule_slots(cfg):
                for s, (m, r) in row.items():
                    seen.setdefault((m, r), []).append(s)
            assert len(seen) == cfg.num_microbatches * cfg.layers_per_device
            assert all(v == list(range(cfg.num_stages)) for v in seen.values())

    def test_config_validation(self):
        for bad in (dict(num_stages=0, num_microbatches=1),
                    dict(num_stages=2, num_microbatches=2, schedule="1f1b"),
                    dict(num_stages=2, num_microbatches=2, layers_per_device=2)):
            with pytest.raises(ValueError):
                PipelineConfig(**bad)


def _sequential(cfg, inputs, w):
    outs = []
    for x in inputs:
        v = x.astype(np.float64)
        for r in range(cfg.layers_per_device):
            for s in range(cfg.num_stages):
                v = v + (w[s] if cfg.schedule == "gpipe" else w[s, r])
        outs.append(v)
    return outs


class TestFunctionalEquivalence:
    """On the oracle (test infrastructure), like reference tests/test_pipeline.py:64-96."""

    @pytest.mark.parametrize("L", [1, 2, 4])
    @pytest.mark.parametrize("M", [1, 2, 8])
    def test_gpipe(self, L, M):
        from oracle import evaluator as O
        cfg = PipelineConfig(L, M)
        g = build_pipeline(cfg, None, (3,), _body("add"), [Shape((3,))])
        rng = np.random.default_rng(L * 10 + M)
        xs = [rng.standard_normal(3).astype(np.float32) for _ in range(M)]
        w = rng.standard_normal((L, 3)).astype(np.float32)
        for got, want in zip(O.evaluate_single(g, xs + [w]), _sequential(cfg, xs, w)):
            np.testing.assert_allclose(got, want, rtol=1e-5)

    @pytest.mark.parametrize("L,M,R", [(2, 2, 2), (2, 4, 2), (4, 8, 2), (3, 5, 3)])
    def test_circular(self, L, M, R):
        from oracle import evaluator as O
        cfg = PipelineConfig(L, M, "circular", R)
        g = build_pipeline(cfg, None, (3,), _body("add"), [Shape((3,))])
        rng = np.random.default_rng(7)
        xs = [rng.standard_normal(3).astype(np.float32) for _ in range(M)]
        w = rng.standard_normal((L, R, 3)).astype(np.float32)
        for got, want in zip(O.evaluate_single(g, xs + [w]), _sequential(cfg, xs, w)):
            np.testing.assert_allclose(got, want, rtol=1e-5)

    def test_body_must_keep_the_buffer_shape(self):
        def bad(b, x, ws):
            return b.add(Op.SLICE, [x], {"starts": (0, 0), "limits": (2, 2), "strides": (1, 1)})
        with pytest.raises(ShapeMismatch):
            build_pipeline(PipelineConfig(2, 2), None, (3,), bad, [Shape((3,))])


def test_shift_lowers_to_collective_permute():
    """reference tests/test_pipeline.py:99-122"""
    mesh = DeviceMesh.default(4)
    cfg = PipelineConfig(4, 8)
    sh = mesh_split(2, mesh, [0, -1])
    g = build_pipeline(cfg, mesh, (6,), _body("add"), [Shape((6,))],
                       input_sharding=Sharding.replicated(), state_sharding=sh,
                       weight_shardings=[sh])
    ann, _ = propagate(g)
    prog = partition(ann, 4)
    assert collective_stats(prog)["counts"].get("collective-permute", 0) >= cfg.num_microbatches
    rev = {e: logical for logical, emitted in prog.mapping.items() for e in emitted}
    for ins in prog.graph.instructions:
        if ins.opcode == Op.ALL_GATHER:
            assert not rev.get(ins.id, "").startswith(("shift", "state", "padded", "select"))
