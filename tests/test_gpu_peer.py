"""Peer-memory collectives (peer.cu) on one GPU: a world-of-one NCCL
communicator still allocates / maps the CUDA-IPC heap and runs the real
kernels -- the scatter epilogue of the tcgen05 GEMM (both parity buffers),
the epoch barrier and the slot reduction; the all-gather staging + copy-engine
and SM-pull engines.  Multi-GPU parity of the same paths against NCCL is
scripts/peer_fusion_check.py and scripts/multi_gpu_check.py
(profiles/r1_peer_fusion_n{2,4}.log)."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    import torch
    from paper_2105_04663_b200.executor import NcclComm
    c = NcclComm(0, 1)
    c.reserve_fused(2 << 20)       # fused landing zone [0, 6 MiB); slots above it
    c.ensure_peer(64 << 20, torch.device("cuda", 0))
    yield c
    c.close()


def _dd():
    from paper_2105_04663_b200 import _capi as C
    dd = C.SpmdDotDims()
    dd.n_contract = 1
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 1, 0
    return dd


@pytest.mark.parametrize("M,K,N", [(256, 128, 256), (384, 640, 1024)])
def test_dot_reduce_scatter_world_of_one(comm, M, K, N):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    garr, ng, gs = _groups_arg([[0]])
    dd = _dd()
    ash, bsh, osh = (Shape((M, K), DType.BF16), Shape((K, N), DType.BF16),
                     Shape((M, N), DType.BF16))
    for it in range(3):   # consecutive epochs alternate the parity buffers
        torch.manual_seed(it)
        a = torch.randn((1, M, K), device="cuda").bfloat16()
        b = (torch.randn((1, K, N), device="cuda") * 0.05).bfloat16()
        fused = torch.empty((1, M, N), device="cuda", dtype=torch.bfloat16)
        plain = torch.empty_like(fused)
        C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(a, ash), desc(b, bsh),
                                            desc(fused, osh), ctypes.byref(dd), 1, garr, ng, gs,
                                            s), "dot_reduce_scatter")
        C.check(lib.spmd_dot(desc(a, ash), desc(b, bsh), desc(plain, osh), ctypes.byref(dd), 1,
                             s), "dot")
        torch.cuda.synchronize()
        C.check(lib.spmd_check_device_errors(s), "device")
        assert torch.equal(fused, plain)
        ref = (a[0].float() @ b[0].float())
        err = (fused[0].float() - ref).abs().max().item() / max(1.0, ref.abs().max().item())
        assert err < 1e-2, err


def test_dot_reduce_scatter_rejects_bad_layouts(comm):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import EvalError, _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    garr, ng, gs = _groups_arg([[0]])
    a = torch.zeros((1, 256, 64), device="cuda", dtype=torch.bfloat16)
    b = torch.zeros((1, 64, 256), device="cuda", dtype=torch.bfloat16)
    o = torch.zeros((1, 256, 256), device="cuda", dtype=torch.bfloat16)
    sh = Shape((256, 256), DType.BF16)
    with pytest.raises(EvalError):   # not the last output dim
        C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(a, Shape((256, 64), DType.BF16)),
                                            desc(b, Shape((64, 256), DType.BF16)), desc(o, sh),
                                            ctypes.byref(_dd()), 0, garr, ng, gs, s), "rs")


@pytest.mark.parametrize("engine", [0, 1, 3, 4])
@pytest.mark.parametrize("dim", [0, 1])
def test_peer_all_gather_world_of_one(comm, engine, dim):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    garr, ng, gs = _groups_arg([[0]])
    x = torch.randn((1, 48, 80), device="cuda")
    y = torch.empty_like(x)
    sh = Shape((48, 80), DType.F32)
    for ch in (0, 1):
        y.zero_()
        if engine == 4:     # pre-staged: stage + barrier first (executor step start)
            C.check(lib.spmd_peer_stage(comm.handle, desc(x, sh), 8 << 20, s), "stage")
            C.check(lib.spmd_peer_barrier(comm.handle, ch, s), "barrier")
        C.check(lib.spmd_peer_all_gather(comm.handle, desc(x, sh), desc(y, sh), dim, garr, ng, gs,
                                         8 << 20, ch, engine, s), "peer_all_gather")
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    C.check(lib.spmd_check_device_errors(s), "device")


def test_dot_all_to_all_world_of_one(comm):
    """Expert-FFN einsum [E,B,C,H] x [E,H,M] with the row-scatter epilogue:
    with one member the all-to-all is the identity, so the result equals the
    plain tcgen05 dot bit for bit (both parity buffers exercised)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    garr, ng, gs = _groups_arg([[0]])
    E, B, Cc, H, M = 2, 8, 64, 256, 512
    dd = C.SpmdDotDims()
    dd.n_batch, dd.n_contract = 1, 1
    dd.lhs_batch[0] = dd.rhs_batch[0] = 0
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 3, 1
    ash, bsh = Shape((E, B, Cc, H), DType.BF16), Shape((E, H, M), DType.BF16)
    osh = Shape((E, B, Cc, M), DType.BF16)
    for it in range(3):
        torch.manual_seed(10 + it)
        a = torch.randn((1, E, B, Cc, H), device="cuda").bfloat16()
        b = (torch.randn((1, E, H, M), device="cuda") * 0.05).bfloat16()
        fused = torch.empty((1, E, B, Cc, M), device="cuda", dtype=torch.bfloat16)
        plain = torch.empty_like(fused)
        C.check(lib.spmd_dot_all_to_all(comm.handle, desc(a, ash), desc(b, bsh), desc(fused, osh),
                                        ctypes.byref(dd), 1, 0, garr, ng, gs, s), "dot_a2a")
        C.check(lib.spmd_dot(desc(a, ash), desc(b, bsh), desc(plain, osh), ctypes.byref(dd), 1,
                             s), "dot")
        torch.cuda.synchronize()
        C.check(lib.spmd_check_device_errors(s), "device")
        assert torch.equal(fused, plain)


def test_dot_reduce_scatter_rows_world_of_one(comm):
    """Reduce-scatter on the leading (row) output dim -- the weight-gradient
    case dW[M,N,D] = x^T.dy split on M -- through the row-scatter epilogue:
    with one member it equals the plain dot bit for bit."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    garr, ng, gs = _groups_arg([[0]])
    T, M, N, D = 256, 256, 8, 64   # x [T, M], dy [T, N, D] -> dW [M, N, D]
    dd = C.SpmdDotDims()
    dd.n_contract = 1
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 0, 0
    ash, bsh = Shape((T, M), DType.BF16), Shape((T, N, D), DType.BF16)
    osh = Shape((M, N, D), DType.BF16)
    for it in range(2):
        torch.manual_seed(20 + it)
        a = torch.randn((1, T, M), device="cuda").bfloat16()
        b = (torch.randn((1, T, N, D), device="cuda") * 0.05).bfloat16()
        fused = torch.empty((1, M, N, D), device="cuda", dtype=torch.bfloat16)
        plain = torch.empty_like(fused)
        C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(a, ash), desc(b, bsh),
                                            desc(fused, osh), ctypes.byref(dd), 0, garr, ng, gs,
                                            s), "dot_rs_rows")
        C.check(lib.spmd_dot(desc(a, ash), desc(b, bsh), desc(plain, osh), ctypes.byref(dd), 1,
                             s), "dot")
        torch.cuda.synchronize()
        C.check(lib.spmd_check_device_errors(s), "device")
        assert torch.equal(fused, plain)


@pytest.mark.parametrize("pairs", [[(0, 0)], []])
def test_peer_collective_permute_world_of_one(comm, pairs):
    """Self pair: out == in through the heap slot; no pair: zero-filled."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    x = torch.randn((1, 3, 1000), device="cuda")
    y = torch.full_like(x, 7.0)
    sh = Shape((3, 1000), DType.F32)
    flat = [v for p in pairs for v in p]
    arr = (ctypes.c_int32 * max(1, len(flat)))(*flat)
    for ch in (0, 2):
        C.check(lib.spmd_peer_collective_permute(comm.handle, desc(x, sh), desc(y, sh), arr,
                                                 len(pairs), 16 << 20, ch, s), "peer_cp")
        torch.cuda.synchronize()
        assert torch.equal(y, x if pairs else torch.zeros_like(x))
    C.check(lib.spmd_check_device_errors(s), "device")


def test_peer_slots_inside_the_fused_region_are_rejected(comm):
    """Staging / landing slots below 3 * fused_half would alias the fused
    ops' parity buffers: refused with EvalError (peer.cu check_slot)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import EvalError, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    x = torch.randn((1, 1024), device="cuda")
    with pytest.raises(EvalError):
        C.check(lib.spmd_peer_stage(comm.handle, desc(x, Shape((1024,), DType.F32)), 1 << 20, s),
                "stage")


def test_fused_ops_of_different_sizes_back_to_back(comm):
    """Consecutive fused dot -> reduce-scatters of different sizes (the
    training step's pattern) alternate parities at the fixed stride and stay
    bit-equal to the plain dot."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
    garr, ng, gs = _groups_arg([[0]])
    dd = _dd()
    outs = []
    for it, (M, K, N) in enumerate([(256, 128, 1024), (512, 256, 1536), (256, 64, 512),
                                    (768, 128, 1024)]):
        torch.manual_seed(40 + it)
        a = torch.randn((1, M, K), device="cuda").bfloat16()
        b = (torch.randn((1, K, N), device="cuda") * 0.05).bfloat16()
        ash, bsh, osh = (Shape((M, K), DType.BF16), Shape((K, N), DType.BF16),
                         Shape((M, N), DType.BF16))
        fused = torch.empty((1, M, N), device="cuda", dtype=torch.bfloat16)
        plain = torch.empty_like(fused)
        C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(a, ash), desc(b, bsh),
                                            desc(fused, osh), ctypes.byref(dd), 1, garr, ng, gs,
                                            s), "dot_reduce_scatter")
        C.check(lib.spmd_dot(desc(a, ash), desc(b, bsh), desc(plain, osh), ctypes.byref(dd), 1,
                             s), "dot")
        outs.append((fused, plain))
    torch.cuda.synchronize()
    C.check(lib.spmd_check_device_errors(s), "device")
    for fused, plain in outs:
        assert torch.equal(fused, plain)
