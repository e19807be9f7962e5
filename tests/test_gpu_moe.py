"""MoE routing / dispatch / combine kernels (config C3) on the B200.

* routing (warp match-any scans): expert and slot bit-exact with the pinned
  host rule ``moe.route_assign``; gate within 1e-6 relative.
* dense masks bit-exact with ``moe.route_top1`` (the tensors the reference's
  MoE graph consumes);
* dispatch / combine gathers bit-identical to the reference-semantics dense
  Dots ``Dot(dispatch, x)`` / ``Dot(combine, y)`` executed by the tcgen05
  GEMM on the same bf16 data.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(x, dtype):
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import Shape
    return desc(x, Shape(tuple(x.shape[1:]), dtype))


def _route(logits_np, C):
    import torch
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200.ir import DType
    B, S, E = logits_np.shape
    lg = torch.from_numpy(logits_np).cuda().unsqueeze(0)
    ex = torch.empty((1, B, S), dtype=torch.int32, device="cuda")
    sl = torch.empty_like(ex)
    gt = torch.empty((1, B, S), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    C_.check(C_.lib().spmd_moe_route(_t(lg, DType.F32), C, _t(ex, DType.S32), _t(sl, DType.S32),
                                     _t(gt, DType.F32), 1, st), "route")
    return ex, sl, gt


@pytest.mark.parametrize("B,S,E,C", [(4, 64, 8, 10), (8, 512, 8, 160), (2, 100, 64, 3)])
def test_route_matches_pinned_rule(B, S, E, C):
    from paper_2105_04663_b200.moe import route_assign, route_top1
    rng = np.random.default_rng(B * S + E)
    logits = rng.standard_normal((B, S, E)).astype(np.float32)
    ex, sl, gt = _route(logits, C)
    e_h, s_h, g_h = route_assign(logits)
    np.testing.assert_array_equal(ex[0].cpu().numpy(), e_h)
    np.testing.assert_array_equal(sl[0].cpu().numpy(), s_h)
    np.testing.assert_allclose(gt[0].cpu().numpy(), g_h, rtol=1e-6)
    # dense masks
    import torch
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200.ir import DType
    d = torch.empty((1, B, S, E, C), dtype=torch.float32, device="cuda")
    c = torch.empty_like(d)
    C_.check(C_.lib().spmd_moe_masks(_t(ex, DType.S32), _t(sl, DType.S32), _t(gt, DType.F32),
                                     _t(d, DType.F32), _t(c, DType.F32), 1,
                                     torch.cuda.current_stream().cuda_stream), "masks")
    disp, comb = route_top1(logits, C)
    np.testing.assert_array_equal(d[0].cpu().numpy(), disp)
    np.testing.assert_allclose(c[0].cpu().numpy(), comb, rtol=1e-6)


def test_dispatch_combine_equal_dense_dots():
    import torch
    from paper_2105_04663_b200 import _capi as C_
    from paper_2105_04663_b200.ir import DType
    B, S, E, C, M = 4, 256, 8, 40, 512
    rng = np.random.default_rng(7)
    logits = rng.standard_normal((B, S, E)).astype(np.float32)
    ex, sl, gt = _route(logits, C)
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn((1, B, S, M), device="cuda").bfloat16()
    disp = torch.empty((1, B, S, E, C), dtype=torch.bfloat16, device="cuda")
    comb = torch.empty_like(disp)
    C_.check(C_.lib().spmd_moe_masks(_t(ex, DType.S32), _t(sl, DType.S32), _t(gt, DType.F32),
                                     _t(disp, DType.BF16), _t(comb, DType.BF16), 1, st), "masks")
    buf = torch.empty((1, B, E, C, M), dtype=torch.bfloat16, device="cuda")
    C_.check(C_.lib().spmd_moe_dispatch(_t(x, DType.BF16), _t(ex, DType.S32), _t(sl, DType.S32),
                                        _t(buf, DType.BF16), 1, st), "dispatch")
    # reference semantics: Dot(dispatch [B,S,E,C], x [B,S,M]) batch b, contract s
    dd = C_.SpmdDotDims()
    dd.n_batch, dd.n_contract = 1, 1
    dd.lhs_batch[0] = dd.rhs_batch[0] = 0
    dd.lhs_contracting[0] = dd.rhs_contracting[0] = 1
    ref = torch.empty((1, B, E, C, M), dtype=torch.bfloat16, device="cuda")
    C_.check(C_.lib().spmd_dot(_t(disp, DType.BF16), _t(x, DType.BF16), _t(ref, DType.BF16),
                               ctypes.byref(dd), 1, st), "dot")
    torch.cuda.synchronize()
    assert torch.equal(buf, ref)
    y = torch.randn((1, B, E, C, M), device="cuda").bfloat16()
    out = torch.empty((1, B, S, M), dtype=torch.bfloat16, device="cuda")
    C_.check(C_.lib().spmd_moe_combine(_t(y, DType.BF16), _t(ex, DType.S32), _t(sl, DType.S32),
                                       _t(gt, DType.F32), _t(out, DType.BF16), 1, st), "combine")
    dd2 = C_.SpmdDotDims()
    dd2.n_batch, dd2.n_contract = 1, 2
    dd2.lhs_batch[0] = dd2.rhs_batch[0] = 0
    dd2.lhs_contracting[0], dd2.lhs_contracting[1] = 2, 3
    dd2.rhs_contracting[0], dd2.rhs_contracting[1] = 1, 2
    ref2 = torch.empty((1, B, S, M), dtype=torch.bfloat16, device="cuda")
    C_.check(C_.lib().spmd_dot(_t(comb, DType.BF16), _t(y, DType.BF16), _t(ref2, DType.BF16),
                               ctypes.byref(dd2), 1, st), "dot")
    torch.cuda.synchronize()
    assert torch.equal(out, ref2)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_executor_routing_equals_dense_masks(n):
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
    ex = torch.empty((n, Bl, S), dtype=torch.int32, device="cuda")
    sl, gt = torch.empty_like(ex), torch.empty((n, Bl, S), dtype=torch.float32, device="cuda")
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
    dense = Executor(prog, nparts=n, device=dev, fuse=True)
    a = routed.run(stacked)[0]
    b = dense.run(stacked)[0]
    torch.cuda.synchronize()
    assert torch.equal(a, b)
