"""The C2 layer at the paper's dims (M=8192, N=128, D=256, H=65536, S=1024;
B=4 so every data axis divides it) partitioned for the scaling run's meshes
-- (1,2), (2,2), (1,4), (2,4) (the N=8 north star), (4,2), (1,8) -- and
executed on ONE B200 as a simulated mesh (all partitions stacked, loopback
collectives), fast plan with the fused kernels.  Each partition's shard of
the output is checked against an fp32 torch evaluation of the same bf16
global inputs (normwise <= 2e-2, the bf16-layer tolerance).

The multi-process runs (tests/test_gpu_multirank.py, scripts/) cover NCCL
and the peer engines at 2 and 4 GPUs; this pins the partitioned programs
of the 8-way meshes at full size, where only shard shapes differ from the
golden small-dim cases.
"""

import pytest

pytestmark = pytest.mark.gpu

LAYER_TOL = 2e-2
DIMS = dict(B=4, S=1024, M=8192, N=128, D=256, H=65536)


def _layer_ref(x, wq, wk, wv, wo, wi, wt):
    import torch
    x, wq, wk, wv, wo, wi, wt = (t.float() for t in (x, wq, wk, wv, wo, wi, wt))
    q = torch.einsum("bsm,mnd->bsnd", x, wq)
    k = torch.einsum("bsm,mnd->bsnd", x, wk)
    v = torch.einsum("bsm,mnd->bsnd", x, wv)
    probs = torch.softmax(torch.einsum("bsnd,btnd->bnst", q, k), dim=-1)
    del q, k
    ctx = torch.einsum("bnst,btnd->bnsd", probs, v)
    del probs, v
    res1 = torch.einsum("bsnd,ndm->bsm", ctx.permute(0, 2, 1, 3), wo) + x
    return torch.relu(res1 @ wi) @ wt + res1


def _tile(t, sharding, dev):
    """Device `dev`'s shard of global tensor t (even tilings only)."""
    from paper_2105_04663_b200.ir import DType, Shape
    from paper_2105_04663_b200.sharding import shard_offset, shard_shape
    if sharding.is_replicated:
        return t
    full = Shape(tuple(t.shape), DType.BF16)
    per = shard_shape(full, sharding).dims
    sl = tuple(slice(shard_offset(full, sharding, dev, k), shard_offset(full, sharding, dev, k)
                     + per[k]) for k in range(t.dim()))
    return t[sl]


@pytest.fixture(scope="module")
def layer():
    import torch
    g = torch.Generator(device="cuda").manual_seed(11)
    B, S, M, N, D, H = (DIMS[k] for k in "BSMNDH")
    r = lambda *s, fan: (torch.randn(s, generator=g, device="cuda") / fan ** 0.5).bfloat16()
    xs = [r(B, S, M, fan=1), r(M, N, D, fan=M), r(M, N, D, fan=M), r(M, N, D, fan=M),
          r(N, D, M, fan=N * D), r(M, H, fan=M), r(H, M, fan=H)]
    ref = _layer_ref(*xs)
    torch.cuda.synchronize()
    yield xs, ref
    del xs, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mesh", [(1, 2), (2, 2), (1, 4), (2, 4), (4, 2), (1, 8)])
def test_c2_layer_paper_dims_on_simulated_mesh(layer, mesh):
    import torch
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.workloads import transformer_layer
    xs, ref = layer
    P = mesh[0] * mesh[1]
    g, _ = transformer_layer(mesh, dtype=DType.BF16, with_inputs=False, **DIMS)
    ann, _ = propagate(g)
    prog = partition(ann, P, plan="fast")
    stacked = [torch.stack([_tile(x, p.sharding, d).contiguous() for d in range(P)])
               for x, p in zip(xs, ann.parameters)]
    ex = Executor(prog, nparts=P, fuse=True)
    out = ex.run(stacked)[0]
    torch.cuda.synchronize()
    ex.check_errors()
    osh = prog.output_shardings[0]
    scale = max(1.0, ref.abs().max().item())
    for d in range(P):
        want = _tile(ref, osh, d)
        err = (out[d].float() - want).abs().max().item() / scale
        assert err < LAYER_TOL, (mesh, d, err)
    del ex, out, stacked
    torch.cuda.empty_cache()
