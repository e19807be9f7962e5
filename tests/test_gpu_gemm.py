"""tcgen05 GEMM and bf16 paths vs a plain PyTorch fp32 reference.

BF16 tolerance: inputs are bf16 (exact in fp32), the kernel accumulates in
fp32 in TMEM and rounds the output once to bf16, so the normwise error
max|out - ref| / max|ref| is bounded by ~2^-8 (bf16 output rounding) plus
fp32 accumulation-order noise: we require <= 8e-3 (SURVEY 8(c) proposal).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BF16_TOL = 8e-3


def _dot(lhs, rhs, lb, rb, lc, rc, nparts=1, relu=False):
    import ctypes
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape, infer_shape, Op
    lsh = Shape(tuple(lhs.shape[1:]), DType.BF16)
    rsh = Shape(tuple(rhs.shape[1:]), DType.BF16)
    attrs = {"lhs_batch": lb, "rhs_batch": rb, "lhs_contracting": lc, "rhs_contracting": rc}
    osh = infer_shape(Op.DOT, [lsh, rsh], attrs)
    out = torch.empty((nparts,) + osh.dims, dtype=torch.bfloat16, device="cuda")
    dd = C.SpmdDotDims()
    dd.n_batch, dd.n_contract = len(lb), len(lc)
    for i, (x, y) in enumerate(zip(lb, rb)):
        dd.lhs_batch[i], dd.rhs_batch[i] = x, y
    for i, (x, y) in enumerate(zip(lc, rc)):
        dd.lhs_contracting[i], dd.rhs_contracting[i] = x, y
    dd.epilogue = int(relu)
    C.check(C.lib().spmd_dot(desc(lhs, lsh), desc(rhs, rsh), desc(out, osh), ctypes.byref(dd),
                             nparts, torch.cuda.current_stream().cuda_stream), "dot")
    torch.cuda.synchronize()
    return out


def _ref(lhs, rhs, spec):
    import torch
    return torch.einsum(spec, lhs.float(), rhs.float())


def _err(a, b):
    a, b = a.float(), b.float()
    return (a - b).abs().max().item() / max(1.0, b.abs().max().item())


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (1000, 300, 200),
                                   (64, 64, 16), (512, 128, 4096), (2048, 2048, 512)])
def test_plain_gemm_mn_major_b(M, N, K):
    """x[M,K] @ w[K,N]: A K-major, B MN-major (the weight layout)."""
    import torch
    torch.manual_seed(0)
    a = torch.randn(1, M, K, device="cuda").bfloat16()
    b = (torch.randn(1, K, N, device="cuda") / K ** 0.5).bfloat16()
    out = _dot(a, b, (), (), (1,), (0,))
    assert _err(out[0], a[0].float() @ b[0].float()) < BF16_TOL


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (384, 640, 128), (130, 70, 48)])
def test_gemm_k_major_b(M, N, K):
    """q[M,K] . k[N,K]^T: both K-major (attention logits layout)."""
    import torch
    torch.manual_seed(1)
    a = torch.randn(1, M, K, device="cuda").bfloat16()
    b = torch.randn(1, N, K, device="cuda").bfloat16()
    out = _dot(a, b, (), (), (1,), (1,))
    assert _err(out[0], a[0].float() @ b[0].float().T) < BF16_TOL


def test_gemm_mn_major_a():
    """A stored [K, M] (M contiguous)."""
    import torch
    torch.manual_seed(2)
    a = torch.randn(1, 192, 320, device="cuda").bfloat16()     # [K, M]
    b = torch.randn(1, 192, 256, device="cuda").bfloat16()     # [K, N]
    out = _dot(a, b, (), (), (0,), (0,))
    assert _err(out[0], a[0].float().T @ b[0].float()) < BF16_TOL


def test_batched_attention_layouts():
    """logits = q[B,S,N,D] . k[B,T,N,D] over (B,N); ctx = p[B,N,S,T] . v[B,T,N,D]."""
    import torch
    torch.manual_seed(3)
    B, S, N, D = 2, 256, 4, 128
    q = torch.randn(1, B, S, N, D, device="cuda").bfloat16()
    k = torch.randn(1, B, S, N, D, device="cuda").bfloat16()
    logits = _dot(q, k, (0, 2), (0, 2), (3,), (3,))
    ref = torch.einsum("bsnd,btnd->bnst", q[0].float(), k[0].float())
    assert logits.shape[1:] == (B, N, S, S)
    assert _err(logits[0], ref) < BF16_TOL
    p = torch.softmax(ref, -1).bfloat16().unsqueeze(0)
    v = torch.randn(1, B, S, N, D, device="cuda").bfloat16()
    ctx = _dot(p, v, (0, 1), (0, 2), (3,), (1,))
    ref2 = torch.einsum("bnst,btnd->bnsd", p[0].float(), v[0].float())
    assert _err(ctx[0], ref2) < BF16_TOL


def test_partition_stacked_and_relu():
    import torch
    torch.manual_seed(4)
    P, M, K, N = 4, 256, 128, 384
    a = torch.randn(P, M, K, device="cuda").bfloat16()
    b = torch.randn(P, K, N, device="cuda").bfloat16()
    out = _dot(a, b, (), (), (1,), (0,), nparts=P, relu=True)
    ref = torch.relu(torch.bmm(a.float(), b.float()))
    assert _err(out, ref) < BF16_TOL


def test_out_projection_two_contracting_dims():
    """ctx_t[B,S,N,D] . wo[N,D,M] contracting (N,D) (merged K)."""
    import torch
    torch.manual_seed(5)
    x = torch.randn(1, 2, 128, 4, 64, device="cuda").bfloat16()
    w = (torch.randn(1, 4, 64, 256, device="cuda") / 16).bfloat16()
    out = _dot(x, w, (), (), (2, 3), (0, 1))
    ref = torch.einsum("bsnd,ndm->bsm", x[0].float(), w[0].float())
    assert _err(out[0], ref) < BF16_TOL


def test_bf16_transformer_layer_small():
    """Full attention+FFN layer in bf16 on a simulated 2x4 mesh (fast plan,
    fused softmax) vs the CPU oracle on bf16-rounded inputs; 2e-2 normwise."""
    import golden_io as G
    from oracle import evaluator as O
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import evaluate_spmd
    from paper_2105_04663_b200.workloads import transformer_layer
    from paper_2105_04663_b200.sharding import assemble_data, shard_data
    g, ins = transformer_layer((2, 4), B=4, S=64, M=256, N=8, D=64, H=512, seed=0)
    ann, _ = propagate(g)
    prog = partition(ann, 8, plan="fast")
    devices = list(range(8))
    per = {d: [] for d in devices}
    for p, x in zip(ann.parameters, ins):
        sh = shard_data(O.to_bf16(x), p.sharding, devices=devices)
        for d in devices:
            per[d].append(sh[d])
    res = evaluate_spmd(prog, per, fuse=True)
    out = assemble_data({d: res[d][0] for d in devices}, prog.output_shardings[0],
                        g.instr(g.outputs[0]).shape, rtol=5e-2)
    want = O.evaluate_single(g, [O.to_bf16(x) for x in ins])[0]
    err, rel = O.rel_error(out, want)
    assert rel < 2e-2, rel
