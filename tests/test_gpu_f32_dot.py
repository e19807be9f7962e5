"""f32 Dot on the tensor cores (3xTF32 tcgen05 GEMM, gemm_tf32x3.cu) --
config C1's einsum BSM,MH->BSH.

The reference evaluates an f32 Dot as a float64 einsum rounded once to f32
(simulator.py:258-275).  3xTF32 keeps hi*hi + hi*lo + lo*hi of the split
operands; the per-product error is ~2^-22, but the tensor core's fp32
accumulation does not round every partial sum to nearest, so the normwise
error grows with K: measured 6e-7 at K=64, 1.9e-6 at K=256, ~1e-5 at
K=4096.  The bound is the reference's own default tolerance for C1,
1e-4 (verify_equivalence).  The test also checks that the
tensor-core path ran, against the exact SIMT fp64 kernel (option
f32_dot_tc = 0).
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _dot(a, b, lc, rc, nparts=1):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Op, Shape, infer_shape
    lsh = Shape(tuple(a.shape[1:]), DType.F32)
    rsh = Shape(tuple(b.shape[1:]), DType.F32)
    attrs = {"lhs_batch": (), "rhs_batch": (), "lhs_contracting": lc, "rhs_contracting": rc}
    osh = infer_shape(Op.DOT, [lsh, rsh], attrs)
    out = torch.empty((nparts,) + osh.dims, dtype=torch.float32, device="cuda")
    dd = C.SpmdDotDims()
    dd.n_contract = len(lc)
    for i, (x, y) in enumerate(zip(lc, rc)):
        dd.lhs_contracting[i], dd.rhs_contracting[i] = x, y
    C.check(C.lib().spmd_dot(desc(a, lsh), desc(b, rsh), desc(out, osh), ctypes.byref(dd), nparts,
                             torch.cuda.current_stream().cuda_stream), "dot")
    torch.cuda.synchronize()
    return out


def _err(a, b):
    a, b = a.double(), b.double()
    return (a - b).abs().max().item() / max(1.0, b.abs().max().item())


@pytest.mark.parametrize("mode", [3, 2])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (1024, 768, 512), (4096, 4096, 4096),
                                   (300, 520, 1000), (2048, 256, 8192), (2304, 3072, 2048),
                                   (4096, 8192, 1024)])
def test_f32_dot_3xtf32_vs_float64(M, N, K, mode):
    """x[M,K] . w[K,N] (B MN-major, the C1 weight layout), partial tiles and
    long K included; gemm_mode 3: 256 x 512 pair tiles when N >= 512 and the
    waves quantise as well (else 256 x 256), 2: always 256 x 256."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn((1, M, K), generator=g, device="cuda")
    b = torch.randn((1, K, N), generator=g, device="cuda") / K ** 0.5
    with C.option("gemm_mode", mode):
        out = _dot(a, b, (1,), (0,))
    ref = a[0].double() @ b[0].double()
    err = _err(out[0], ref)
    assert err < TOL, err
    with C.option("f32_dot_tc", 0):
        exact = _dot(a, b, (1,), (0,))
    assert _err(exact[0], ref) < 1e-7
    # the tensor-core result is not the fp64 SIMT one bit for bit
    assert not torch.equal(out, exact)


def test_f32_dot_k_major_b_and_partitions():
    """q[M,K] . k[N,K]^T (both K-major) over a stack of 3 partitions."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn((3, 512, 384), generator=g, device="cuda")
    b = torch.randn((3, 640, 384), generator=g, device="cuda")
    out = _dot(a, b, (1,), (1,), nparts=3)
    for p in range(3):
        ref = a[p].double() @ b[p].double().T
        assert _err(out[p], ref) < TOL


def test_c1_einsum_on_simulated_2x2_mesh_vs_oracle():
    """C1 (BSM,MH->BSH, x [X,-,Y], w [X,Y]) at B=16 S=256 M=1024 H=1024 on a
    simulated 2x2 mesh (reference plan: all-gathers + local Dots of 2048 x
    512 x 1024 on the tensor cores) vs the CPU oracle's float64 einsum."""
    from oracle import evaluator as O
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import evaluate_spmd
    from paper_2105_04663_b200.sharding import assemble_data, shard_data
    from paper_2105_04663_b200.workloads import einsum_c1
    g, ins = einsum_c1((2, 2), B=16, S=256, M=1024, H=1024, seed=3)
    ann, _ = propagate(g)
    prog = partition(ann, 4)
    devices = list(range(4))
    per = {d: [] for d in devices}
    for p, x in zip(ann.parameters, ins):
        sh = shard_data(x, p.sharding, devices=devices)
        for d in devices:
            per[d].append(sh[d])
    res = evaluate_spmd(prog, per)
    out = assemble_data({d: res[d][0] for d in devices}, prog.output_shardings[0],
                        g.instr(g.outputs[0]).shape, rtol=1e-4)
    want = O.evaluate_single(g, ins)[0]
    _, rel = O.rel_error(out, want)
    assert rel < 1e-4, rel


def test_c1_fused_gather_split_vs_oracle():
    """The executor's fused path for C1 (fuse=True): the loopback all-gather
    of x writes tf32 hi / lo halves and the 3xTF32 GEMM skips its lhs split
    (spmd_local_all_gather_split + spmd_dot_f32_presplit).  M=4096 so the
    gathered rows are long enough for the row kernel; vs the oracle's float64
    einsum and vs the unfused path."""
    import numpy as np
    from oracle import evaluator as O
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor, evaluate_spmd
    from paper_2105_04663_b200.sharding import assemble_data, shard_data
    from paper_2105_04663_b200.workloads import einsum_c1
    g, ins = einsum_c1((2, 2), B=4, S=256, M=4096, H=1024, seed=5)
    ann, _ = propagate(g)
    prog = partition(ann, 4, plan="fast")
    ex = Executor(prog, nparts=4, fuse=True)
    assert any(v[0] == "ag_split_dot" for v in ex._fused.values())
    devices = list(range(4))
    per = {d: [] for d in devices}
    for p, x in zip(ann.parameters, ins):
        sh = shard_data(x, p.sharding, devices=devices)
        for d in devices:
            per[d].append(sh[d])
    fused = evaluate_spmd(prog, per, fuse=True)
    plain = evaluate_spmd(prog, per, fuse=False)
    out = assemble_data({d: fused[d][0] for d in devices}, prog.output_shardings[0],
                        g.instr(g.outputs[0]).shape, rtol=1e-4)
    want = O.evaluate_single(g, ins)[0]
    _, rel = O.rel_error(out, want)
    assert rel < 1e-4, rel
    for d in devices:   # the split is the same either way: identical GEMM inputs
        np.testing.assert_array_equal(fused[d][0], plain[d][0])
