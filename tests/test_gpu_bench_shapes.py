"""Parity at the benchmarked shapes (the configurations bench.py times).

The small-shape tests elsewhere give every CTA pair at most one output tile.
Here the kernels run at the C2 / C4 paper dims, where the persistent tile
loop, the TMEM accumulator phase flips and the multi-group rasterisation are
all exercised (~55 tiles per CTA pair for the FFN GEMMs), for every GEMM
variant, against plain PyTorch fp32 references (TF32 off) of the same bf16
inputs -- the Dot semantics of reference simulator.py:258-277 (accumulate
wide, round once).

Tolerances (normwise max|err| / max(1, max|ref|), reference metric
simulator.py:471-479): 8e-3 for one bf16-output contraction, 2e-2 for the
full bf16 layer.
"""

import ctypes

import pytest

pytestmark = pytest.mark.gpu

BF16_TOL = 8e-3
LAYER_TOL = 2e-2


@pytest.fixture(autouse=True)
def _no_tf32():
    import torch
    old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old
    torch.cuda.empty_cache()


def _err(a, b):
    a, b = a.float(), b.float()
    return (a - b).abs().max().item() / max(1.0, b.abs().max().item())


def _gemm(a, b, relu=False):
    """C[M,N] = A[M,K] . B[K,N] through spmd_dot (the executor's call)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    M, K = a.shape
    N = b.shape[1]
    out = torch.empty((1, M, N), dtype=torch.bfloat16, device="cuda")
    dd = C.SpmdDotDims()
    dd.n_contract = 1
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 1, 0
    dd.epilogue = int(relu)
    C.check(C.lib().spmd_dot(desc(a, Shape((M, K), DType.BF16)), desc(b, Shape((K, N), DType.BF16)),
                             desc(out, Shape((M, N), DType.BF16)), ctypes.byref(dd), 1,
                             torch.cuda.current_stream().cuda_stream), "dot")
    return out[0]


def _sampled_rows(M, group_rows=16 * 256, block=256):
    """One 256-row block from every raster group (16 M-tiles of 256 rows),
    at a different offset inside each group, plus the last block."""
    starts = []
    for gi, g0 in enumerate(range(0, M, group_rows)):
        span = min(group_rows, M - g0)
        off = ((gi * 5 + 3) * block) % max(block, span - block + 1)
        starts.append(g0 + off // block * block)
    starts.append(M - block)
    return sorted(set(starts))


# C2 per-GPU GEMMs at N=1 (T = B*S = 16384 tokens): FFN-in, FFN-out, the
# Q/K/V projection (N*D = 32768) and the out-projection (K = N*D).
C2_SHAPES = [(16384, 65536, 8192), (16384, 8192, 65536), (16384, 32768, 8192),
             (16384, 8192, 32768)]


@pytest.mark.parametrize("M,N,K", C2_SHAPES)
def test_c2_gemm_at_paper_dims(M, N, K):
    """Default (wide 256x512 CTA-pair) kernel at the exact C2 shapes: every
    raster group sampled, all columns, vs fp32."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    b = (torch.randn((K, N), generator=g, device="cuda") / K ** 0.5).bfloat16()
    relu = N == 65536   # FFN-in carries the fused ReLU epilogue in the layer
    out = _gemm(a, b, relu=relu)
    torch.cuda.synchronize()
    bf = b.float()
    worst = 0.0
    for r0 in _sampled_rows(M):
        ref = a[r0:r0 + 256].float() @ bf
        if relu:
            ref = torch.relu(ref)
        worst = max(worst, _err(out[r0:r0 + 256], ref))
    assert worst < BF16_TOL, worst
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_every_gemm_variant_with_many_tiles_per_cta(mode):
    """Each variant (1: 1-CTA 128x256, 2: 256x256 pairs, 3: wide 256x512
    pairs) on a shape with >= 4 tiles per CTA (pair), fully checked."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    M, N, K = 4096, 16384, 1024     # wide: 16 x 32 = 512 tiles over 74 pairs
    g = torch.Generator(device="cuda").manual_seed(mode)
    a = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    b = (torch.randn((K, N), generator=g, device="cuda") / K ** 0.5).bfloat16()
    with C.option("gemm_mode", mode):
        out = _gemm(a, b)
        torch.cuda.synchronize()
    ref = a.float() @ b.float()
    assert _err(out, ref) < BF16_TOL


@pytest.mark.parametrize("group", [1, 3, 16])
def test_gemm_raster_groups_partial_last_group(group):
    """Raster groups that do not divide the M tiles (a partial last group)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    M, N, K = 256 * 21, 512 * 9, 512
    g = torch.Generator(device="cuda").manual_seed(group)
    a = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    b = (torch.randn((K, N), generator=g, device="cuda") / K ** 0.5).bfloat16()
    with C.option("gemm_group", group):
        out = _gemm(a, b)
        torch.cuda.synchronize()
    assert _err(out, a.float() @ b.float()) < BF16_TOL


def _layer_ref(xs):
    """fp32 torch evaluation of workloads.transformer_layer (App. A op chain)
    on the same bf16 inputs."""
    import torch
    x, wq, wk, wv, wo, wi, wt = (t[0].float() for t in xs)
    q = torch.einsum("bsm,mnd->bsnd", x, wq)
    k = torch.einsum("bsm,mnd->bsnd", x, wk)
    v = torch.einsum("bsm,mnd->bsnd", x, wv)
    logits = torch.einsum("bsnd,btnd->bnst", q, k)
    del q, k
    probs = torch.softmax(logits, dim=-1)
    del logits
    ctx = torch.einsum("bnst,btnd->bnsd", probs, v)
    del probs, v
    attn = torch.einsum("bsnd,ndm->bsm", ctx.permute(0, 2, 1, 3), wo)
    res1 = attn + x
    h = torch.relu(res1 @ wi)
    return h @ wt + res1


def test_c2_fused_layer_at_paper_dims_b1():
    """The benchmarked C2 layer (M=8192, N=128, D=256, H=65536, S=1024) with
    B=1, through Executor(fuse=True) -- tcgen05 GEMMs with the ReLU
    epilogue, the fused flash attention storing the transposed context --
    vs an fp32 evaluation of the same bf16 inputs."""
    import numpy as np
    import torch
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.workloads import transformer_layer
    dims = dict(B=1, S=1024, M=8192, N=128, D=256, H=65536)
    g, _ = transformer_layer((1, 1), dtype=DType.BF16, with_inputs=False, **dims)
    ann, _ = propagate(g)
    prog = partition(ann, 1, plan="fast")
    fan = [1, dims["M"], dims["M"], dims["M"], dims["N"] * dims["D"], dims["M"], dims["H"]]
    gen = torch.Generator(device="cuda").manual_seed(7)
    xs = [(torch.randn((1,) + p.shape.dims, generator=gen, device="cuda") /
           np.sqrt(f)).bfloat16() for p, f in zip(prog.graph.parameters, fan)]
    ex = Executor(prog, nparts=1, fuse=True)
    fused = {v[0] for v in ex._fused.values()}
    assert "attention" in " ".join(fused) and "dot_relu" in fused, fused
    out = ex.run(xs)[0]
    torch.cuda.synchronize()
    ref = _layer_ref(xs)
    err = _err(out[0], ref)
    assert err < LAYER_TOL, err
    # the CUDA-graph replay of the same step gives the same bits
    graph, gouts = ex.capture(xs)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(gouts[0], out)


def _conv(x, w, relu=False):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    N, H, W, Ci = x.shape
    Co = w.shape[3]
    out = torch.empty((1, N, H, W, Co), dtype=torch.bfloat16, device="cuda")
    cd = C.SpmdConvDims()
    cd.lhs_batch, cd.lhs_feature, cd.rhs_in_feature, cd.rhs_out_feature = 0, 3, 2, 3
    cd.out_batch, cd.out_feature, cd.n_spatial = 0, 3, 2
    for i, (ls, rs, os_) in enumerate([(1, 0, 1), (2, 1, 2)]):
        cd.lhs_spatial[i], cd.rhs_spatial[i], cd.out_spatial[i] = ls, rs, os_
        cd.size[i], cd.stride[i] = 3, 1
        cd.pad_low[i] = cd.pad_high[i] = 1
        cd.base_dilation[i] = cd.window_dilation[i] = 1
    cd.epilogue = int(relu)
    C.check(C.lib().spmd_convolution(desc(x, Shape((N, H, W, Ci), DType.BF16)),
                                     desc(w, Shape((3, 3, Ci, Co), DType.BF16)),
                                     desc(out, Shape((N, H, W, Co), DType.BF16)),
                                     ctypes.byref(cd), 1, torch.cuda.current_stream().cuda_stream),
            "conv")
    return out[0]


@pytest.mark.parametrize("taps,wres", [(1, 1), (0, 1), (0, 0)])
def test_c4_conv_at_paper_dims(taps, wres):
    """C4 layer: 3x3 / stride 1 / pad 1, Cin = Cout = 128, 1024 x 1024 NHWC,
    fused ReLU, N = 2 (8192 pair tiles).  taps=1: the shipped tap-reuse
    kernel <3,18,3>; taps=0: resident weights <4,18>; wres=0: streamed
    weights <7,0>."""
    import torch
    import torch.nn.functional as F
    from paper_2105_04663_b200 import _capi as C
    g = torch.Generator(device="cuda").manual_seed(11 + taps + 2 * wres)
    x = torch.randn((2, 1024, 1024, 128), generator=g, device="cuda").bfloat16()
    w = (torch.randn((3, 3, 128, 128), generator=g, device="cuda") / (9 * 128) ** 0.5).bfloat16()
    with C.option("conv_taps", taps), C.option("conv_wres", wres):
        out = _conv(x, w, relu=True)
        torch.cuda.synchronize()
    ref = torch.relu(F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(3, 2, 0, 1),
                              padding=1)).permute(0, 2, 3, 1)
    assert _err(out, ref) < BF16_TOL


@pytest.mark.parametrize("M,N,K", [(16384, 8192, 65536 // 8), (2048, 1024, 512), (300, 520, 256)])
def test_dot_add_epilogue(M, N, K):
    """spmd_dot_add: C = A.B + R with the add in the wide GEMM's epilogue
    (fp32, one rounding) vs fp32 torch; shapes the wide kernel does not take
    report SPMD_ERR_UNSUPPORTED (the executor then runs Dot + Add)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    b = (torch.randn((K, N), generator=g, device="cuda") / K ** 0.5).bfloat16()
    r = torch.randn((M, N), generator=g, device="cuda").bfloat16()
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    dd = C.SpmdDotDims()
    dd.n_contract = 1
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 1, 0
    bf = DType.BF16
    rc = C.lib().spmd_dot_add(desc(a, Shape((M, K), bf)), desc(b, Shape((K, N), bf)),
                              desc(r, Shape((M, N), bf)), desc(out, Shape((M, N), bf)),
                              ctypes.byref(dd), 1, torch.cuda.current_stream().cuda_stream)
    if M < 256 or N < 512:
        assert rc == C.ERR_UNSUPPORTED
        return
    C.check(rc, "dot_add")
    torch.cuda.synchronize()
    ref = a.float() @ b.float() + r.float()
    assert _err(out, ref) < BF16_TOL
