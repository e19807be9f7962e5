"""MoE routing / dispatch / combine kernels (config C3) on the B200.

* routing (warp match-any scans, one pass per choice): expert and slot
  bit-exact with the pinned host rule ``moe.route_topk`` (GShard top-1 and
  top-2 order, capacity drop); gates within 1e-6 relative;
* dense masks bit-exact with ``moe.route_masks`` (the tensors the reference's
  MoE graph consumes);
* dispatch / combine gathers bit-exact with the CPU oracle's Dot on the same
  bf16 data -- the reference semantics (f64 accumulation, one rounding,
  simulator.py:258-275) of ``Dot(dispatch, x)`` / ``Dot(combine, y)``
  (tests/test_acceptance.py:326-349), rounded to bf16.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(x, dtype):
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import Shape
    return desc(x, Shape(tuple(x.shape[1:]), dtype))


def _route(logits_np, C, k=1):
    import torch
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200.ir import DType
    B, S, E = logits_np.shape
    lg = torch.from_numpy(logits_np).cuda().unsqueeze(0)
    shape = (1, B, S) if k == 1 else (1, B, S, k)
    ex = torch.empty(shape, dtype=torch.int32, device="cuda")
    sl = torch.empty_like(ex)
    gt = torch.empty(shape, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    C_.check(C_.lib().spmd_moe_route(_t(lg, DType.F32), C, _t(ex, DType.S32), _t(sl, DType.S32),
                                     _t(gt, DType.F32), 1, st), "route")
    return ex, sl, gt


def _oracle_dot(lhs, rhs, lb, rb, lc, rc):
    """The CPU oracle's Dot (reference simulator.py:258-275) on float32
    arrays holding bf16 values."""
    from oracle import evaluator as O
    from paper_2105_04663_b200.ir import DType, GraphBuilder, Op, Shape
    from paper_2105_04663_b200.sharding import DeviceMesh
    b = GraphBuilder("dot", DeviceMesh.default(1))
    x = b.parameter(Shape(lhs.shape, DType.F32), id="l")
    y = b.parameter(Shape(rhs.shape, DType.F32), id="r")
    d = b.add(Op.DOT, [x, y], {"lhs_batch": lb, "rhs_batch": rb, "lhs_contracting": lc,
                               "rhs_contracting": rc}, id="d")
    return O.evaluate_single(b.build([d]), [lhs, rhs])[0]


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("B,S,E,C", [(4, 64, 8, 10), (8, 512, 8, 160), (2, 100, 64, 3),
                                     (8, 512, 8, 40)])
def test_route_matches_pinned_rule(B, S, E, C, k):
    """C3's B8 S512 E8 C160 included (k=2: C = ceil(1.25 * 2 * 512 / 8));
    C=40 forces second choices to be dropped."""
    import torch
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.moe import route_masks, route_topk
    rng = np.random.default_rng(B * S + E + k)
    logits = rng.standard_normal((B, S, E)).astype(np.float32)
    ex, sl, gt = _route(logits, C, k)
    e_h, s_h, g_h = route_topk(logits, k, C)
    if k == 1:
        e_h, s_h, g_h = e_h[..., 0], s_h[..., 0], g_h[..., 0]
    np.testing.assert_array_equal(ex[0].cpu().numpy(), e_h)
    np.testing.assert_array_equal(sl[0].cpu().numpy(), s_h)
    np.testing.assert_allclose(gt[0].cpu().numpy(), g_h, rtol=1e-6)
    # dense masks
    d = torch.empty((1, B, S, E, C), dtype=torch.float32, device="cuda")
    c = torch.empty_like(d)
    C_.check(C_.lib().spmd_moe_masks(_t(ex, DType.S32), _t(sl, DType.S32), _t(gt, DType.F32),
                                     _t(d, DType.F32), _t(c, DType.F32), 1,
                                     torch.cuda.current_stream().cuda_stream), "masks")
    disp, comb = route_masks(logits, C, k)
    np.testing.assert_array_equal(d[0].cpu().numpy(), disp)
    np.testing.assert_allclose(c[0].cpu().numpy(), comb, rtol=1e-6)


@pytest.mark.parametrize("k,B,S,E,C,M", [(1, 4, 256, 8, 40, 512), (2, 8, 512, 8, 160, 256),
                                         (2, 4, 128, 8, 20, 128)])
def test_dispatch_combine_equal_oracle_dots(k, B, S, E, C, M):
    """Gather dispatch / weighted-gather combine vs the oracle's
    Dot(dispatch [B,S,E,C], x [B,S,M]) and Dot(combine [B,S,E,C], y
    [B,E,C,M]) on the same bf16 values: bit-exact after the bf16 rounding."""
    import torch
    from oracle import evaluator as O
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200.ir import DType
    rng = np.random.default_rng(7 + k)
    logits = rng.standard_normal((B, S, E)).astype(np.float32)
    ex, sl, gt = _route(logits, C, k)
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn((1, B, S, M), device="cuda").bfloat16()
    disp = torch.empty((1, B, S, E, C), dtype=torch.bfloat16, device="cuda")
    comb = torch.empty_like(disp)
    C_.check(C_.lib().spmd_moe_masks(_t(ex, DType.S32), _t(sl, DType.S32), _t(gt, DType.F32),
                                     _t(disp, DType.BF16), _t(comb, DType.BF16), 1, st), "masks")
    buf = torch.empty((1, B, E, C, M), dtype=torch.bfloat16, device="cuda")
    C_.check(C_.lib().spmd_moe_dispatch(_t(x, DType.BF16), _t(ex, DType.S32), _t(sl, DType.S32),
                                        _t(buf, DType.BF16), 1, st), "dispatch")
    y = torch.randn((1, B, E, C, M), device="cuda").bfloat16()
    out = torch.empty((1, B, S, M), dtype=torch.bfloat16, device="cuda")
    C_.check(C_.lib().spmd_moe_combine(_t(y, DType.BF16), _t(ex, DType.S32), _t(sl, DType.S32),
                                       _t(gt, DType.F32), _t(out, DType.BF16), 1, st), "combine")
    torch.cuda.synchronize()
    f32 = lambda t: t[0].float().cpu().numpy()
    want_d = _oracle_dot(f32(disp), f32(x), (0,), (0,), (1,), (1,))
    np.testing.assert_array_equal(f32(buf), O.to_bf16(want_d))
    want_c = _oracle_dot(f32(comb), f32(y), (0,), (0,), (2, 3), (1, 2))
    np.testing.assert_array_equal(f32(out), O.to_bf16(want_c))
    if k == 2:
        s_np = sl[0].cpu().numpy()
        assert (s_np[..., 1] < C).any()          # second choices kept
        if C * E < k * S:
            assert (s_np >= C).any()             # and some dropped


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_executor_routing_equals_dense_masks(n, k):
    """The partitioned C3 layer (loopback mesh of n) with a declared routing:
    dispatch/combine Dots run as the gather kernels and the output is
    bit-identical to the same program consuming the dense one-hot masks."""
    import torch
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor, Routing, upload_stacked
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.sharding import shard_data
    from paper_2105_04663_b200.workloads import moe_layer
    E, B, S, C, M, H = 8, 8, 64, 16, 128, 256
    g, ins = moe_layer(n, E=E, B=B, S=S, C=C, M=M, H=H, dtype=DType.BF16)
    ann, _ = propagate(g)
    prog = partition(ann, n, plan="fast")
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    Bl = B // n
    rng = np.random.default_rng(n)
    logits = torch.from_numpy(rng.standard_normal((n, Bl, S, E)).astype(np.float32)).cuda()
    shape = (n, Bl, S) if k == 1 else (n, Bl, S, k)
    ex = torch.empty(shape, dtype=torch.int32, device="cuda")
    sl, gt = torch.empty_like(ex), torch.empty(shape, dtype=torch.float32, device="cuda")
    C_.check(C_.lib().spmd_moe_route(_t(logits, DType.F32), C, _t(ex, DType.S32),
                                     _t(sl, DType.S32), _t(gt, DType.F32), n, st), "route")
    disp = torch.empty((n, Bl, S, E, C), dtype=torch.bfloat16, device="cuda")
    comb = torch.empty_like(disp)
    C_.check(C_.lib().spmd_moe_masks(_t(ex, DType.S32), _t(sl, DType.S32), _t(gt, DType.F32),
                                     _t(disp, DType.BF16), _t(comb, DType.BF16), n, st), "masks")
    names = [p.id for p in ann.parameters]
    stacked = []
    for p_src, x, p in zip(ann.parameters, ins, prog.graph.parameters):
        stacked.append(upload_stacked([shard_data(x, p_src.sharding, devices=range(n))[d]
                                       for d in range(n)], p.shape, dev))
    stacked[names.index("dispatch")] = disp
    stacked[names.index("combine")] = comb
    idx = {p.id: p.attrs["index"] for p in ann.parameters}
    r = Routing(ex, sl, gt)
    routed = Executor(prog, nparts=n, device=dev, fuse=True,
                      routing={idx["dispatch"]: r, idx["combine"]: r})
    kinds = sorted(v[0] for v in routed._fused.values() if v[0].startswith("moe_"))
    assert kinds == ["moe_combine", "moe_dispatch"]
    if n == 1:   # the Transpose(1,0,2,3) -> ReLU chains fold into both gathers
        flags = {v[0]: (v[3] if len(v) > 3 else 0) for v in routed._fused.values()
                 if v[0].startswith("moe_")}
        assert flags == {"moe_dispatch": 3, "moe_combine": 3}, flags
    dense = Executor(prog, nparts=n, device=dev, fuse=True)
    a = routed.run(stacked)[0]
    b = dense.run(stacked)[0]
    torch.cuda.synchronize()
    if k == 1:   # one nonzero term per output element on both paths
        assert torch.equal(a, b)
    else:        # combine: the dense GEMM sums k terms in fp32, the gather in fp64
        err = (a.float() - b.float()).abs().max().item() / max(1.0, b.float().abs().max().item())
        assert err < 2 ** -8, err
