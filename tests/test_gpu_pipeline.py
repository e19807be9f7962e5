"""Shifting-buffer pipelines executed on the B200 (reference pipeline.py +
simulator.py): the stage-sharded buffer moves by collective-permute, the
stage body is a stage-batched tcgen05 GEMM.  The golden pipeline programs
(recorded from the reference) are covered by tests/test_gpu_parity.py like
every other golden case; these tests add bf16 GEMM bodies at GEMM-sized
shapes, both planners, fusions, against the single-device B200 run and a
float64 sequential loop."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _graph(schedule, L, M, R, rows, width):
    from paper_2105_04663_b200 import DType, Op, Shape
    from paper_2105_04663_b200.pipeline import PipelineConfig, build_pipeline
    from paper_2105_04663_b200.sharding import DeviceMesh, Sharding, mesh_split

    def body(b, x, ws):
        y = b.add(Op.DOT, [x, ws[0]], {"lhs_batch": (0,), "rhs_batch": (0,),
                                        "lhs_contracting": (2,), "rhs_contracting": (1,)})
        return b.add(Op.ADD, [x, y])

    mesh = DeviceMesh.default(L)
    cfg = PipelineConfig(L, M, schedule, R)
    lead = (L,) if schedule == "gpipe" else (L, R)
    st = mesh_split(3, mesh, [0, -1, -1])
    wsh = mesh_split(len(lead) + 2, mesh, [0] + [-1] * (len(lead) + 1))
    g = build_pipeline(cfg, mesh, (rows, width), body, [Shape((width, width), DType.BF16)],
                       dtype=DType.BF16, input_sharding=Sharding.replicated(),
                       state_sharding=st, weight_shardings=[wsh])
    rng = np.random.default_rng(L + M + R)
    xs = [rng.standard_normal((rows, width)).astype(np.float32) for _ in range(M)]
    w = (rng.standard_normal(lead + (width, width)) / (2 * np.sqrt(width))).astype(np.float32)
    return cfg, g, xs, w


def _bf16(a):
    import torch
    return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy()


@pytest.mark.parametrize("schedule,L,M,R", [("gpipe", 4, 6, 1), ("circular", 2, 4, 2)])
@pytest.mark.parametrize("plan,fuse", [("reference", False), ("fast", True)])
def test_pipeline_with_gemm_body_on_b200(schedule, L, M, R, plan, fuse):
    from paper_2105_04663_b200 import propagate, verify_equivalence
    from paper_2105_04663_b200.executor import evaluate_single
    cfg, g, xs, w = _graph(schedule, L, M, R, rows=256, width=256)
    ann, _ = propagate(g)
    rep = verify_equivalence(g, ann, L, xs + [w], tolerance=2e-2, plan=plan, fuse=fuse)
    assert rep.passed, rep.details
    assert rep.collective_counts.get("collective-permute", 0) >= M
    # and the single-device B200 run matches a float64 sequential stage loop
    got = evaluate_single(g, xs + [w])
    wb = _bf16(w).astype(np.float64)
    for m, x in enumerate(xs):
        v = _bf16(x).astype(np.float64)
        for r in range(R):
            for s in range(L):
                ws = wb[s] if schedule == "gpipe" else wb[s, r]
                v = _bf16(v + _bf16(v @ ws))
        err = np.max(np.abs(got[m] - v)) / max(1.0, np.max(np.abs(v)))
        assert err < 2e-2, (m, err)
