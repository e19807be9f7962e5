"""Loopback collectives (collectives_local.cu) on runs long enough for the
row kernel (>= 512 16-byte vectors per contiguous run) and on short runs
(element kernel), vs the CPU oracle's collective semantics
(oracle.evaluator.collective = reference simulator.py:333-390): all-gather
concatenates in subgroup order, all-to-all splits evenly and concatenates
in group order, collective-permute zero-fills non-targets.  Copies only, so
bit-exact for every dtype.  These are the simulated-mesh collectives of the
C1 bench config (2x2 on one GPU)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GROUPS4 = [((0, 1), (2, 3)), ((0, 2), (1, 3)), ((3, 1, 0, 2),)]


def _run(op, attrs, per, out_dims, dtype):
    from oracle import evaluator as O
    from paper_2105_04663_b200.executor import evaluate_spmd
    from paper_2105_04663_b200.ir import Graph, Instruction, Op, Shape
    from paper_2105_04663_b200.partitioner import SpmdProgram
    n = len(per)
    shp = Shape(per[0].shape, dtype)
    p = Instruction("x", Op.PARAMETER, (), {"index": 0, "shape": shp}, shp)
    ins = Instruction("c", op, ("x",), attrs, Shape(tuple(out_dims), dtype))
    g = Graph("coll", (p, ins), ("c",))
    got = evaluate_spmd(SpmdProgram(g, n, {}, (), ()), {d: [per[d]] for d in range(n)})
    want = O.collective(ins, per, list(range(n)))
    for d in range(n):
        np.testing.assert_array_equal(got[d][0], want[d])


def _inputs(dims, dtype, n=4, seed=0):
    from paper_2105_04663_b200.ir import DType
    rng = np.random.default_rng(seed)
    if dtype == DType.F32:
        return {d: rng.standard_normal(dims).astype(np.float32) for d in range(n)}
    if dtype == DType.PRED:
        return {d: rng.integers(0, 2, dims).astype(bool) for d in range(n)}
    if dtype == DType.S32:
        return {d: rng.integers(-2**31, 2**31 - 1, dims).astype(np.int32) for d in range(n)}
    # bf16: bf16-representable f32 values (the executor uploads bf16 as 2 bytes)
    x = {d: rng.standard_normal(dims).astype(np.float32) for d in range(n)}
    return {d: (v.view(np.uint32) & 0xFFFF0000).view(np.float32) for d, v in x.items()}


@pytest.mark.parametrize("groups", GROUPS4)
@pytest.mark.parametrize("dims,dim,dt", [
    ((2, 3, 4096), 0, "f32"), ((2, 3, 4096), 1, "f32"), ((2, 3, 4096), 2, "f32"),
    ((5, 8192), 1, "bf16"), ((3, 16384), 0, "pred"), ((4, 2048), 1, "s32"),
    ((2, 3, 12), 1, "f32"),                         # short runs: element kernel
])
def test_local_all_gather_long_runs(groups, dims, dim, dt):
    from paper_2105_04663_b200.ir import DType, Op
    dtype = {"f32": DType.F32, "bf16": DType.BF16, "pred": DType.PRED, "s32": DType.S32}[dt]
    gsize = len(groups[0])
    out = list(dims)
    out[dim] *= gsize
    _run(Op.ALL_GATHER, {"dim": dim, "subgroups": groups}, _inputs(dims, dtype), out, dtype)


@pytest.mark.parametrize("groups", GROUPS4)
@pytest.mark.parametrize("dims,split,concat,dt", [
    ((8, 4096), 0, 1, "f32"), ((8, 4096), 1, 0, "f32"), ((8, 4096), 0, 0, "f32"),
    ((4, 6, 8192), 2, 1, "bf16"), ((4, 6, 8192), 0, 2, "bf16"), ((4, 2, 16384), 0, 0, "pred"),
    ((4, 12), 0, 1, "f32"),                         # short runs: element kernel
])
def test_local_all_to_all_long_runs(groups, dims, split, concat, dt):
    from paper_2105_04663_b200.ir import DType, Op
    dtype = {"f32": DType.F32, "bf16": DType.BF16, "pred": DType.PRED}[dt]
    gsize = len(groups[0])
    out = list(dims)
    out[split] //= gsize
    out[concat] *= gsize
    _run(Op.ALL_TO_ALL, {"split_dim": split, "concat_dim": concat, "subgroups": groups},
         _inputs(dims, dtype), out, dtype)


@pytest.mark.parametrize("pairs", [((0, 1), (1, 2), (2, 3), (3, 0)), ((0, 2), (3, 1)),
                                   ((1, 1),)])
@pytest.mark.parametrize("dims", [(4, 4096), (3, 5)])
def test_local_collective_permute_long_runs(pairs, dims):
    from paper_2105_04663_b200.ir import DType, Op
    _run(Op.COLLECTIVE_PERMUTE, {"pairs": pairs}, _inputs(dims, DType.F32), dims, DType.F32)


@pytest.mark.parametrize("groups", GROUPS4)
@pytest.mark.parametrize("kind", ["sum", "max", "min", "prod"])
@pytest.mark.parametrize("dims,dt", [((2, 8192), "f32"), ((4096,), "s32"), ((3, 5), "f32")])
def test_local_all_reduce_long_runs(groups, kind, dims, dt):
    """Serial fold in group order: bit-exact for f32 too (oracle folds the
    same way with numpy)."""
    from paper_2105_04663_b200.ir import DType, Op, ReduceKind
    dtype = {"f32": DType.F32, "s32": DType.S32}[dt]
    per = _inputs(dims, dtype)
    if dtype == DType.S32:      # keep sums / products inside int32
        per = {d: (v % 7).astype(np.int32) for d, v in per.items()}
    _run(Op.ALL_REDUCE, {"kind": ReduceKind(kind), "subgroups": groups}, per, dims, dtype)


@pytest.mark.parametrize("groups", GROUPS4)
@pytest.mark.parametrize("dims,dim", [((8, 4096), 0), ((2, 16384), 1), ((4, 8, 4096), 1),
                                      ((4, 12), 1)])
def test_local_reduce_scatter_long_runs(groups, dims, dim):
    from paper_2105_04663_b200.ir import DType, Op, ReduceKind
    gsize = len(groups[0])
    out = list(dims)
    out[dim] //= gsize
    _run(Op.REDUCE_SCATTER, {"kind": ReduceKind.SUM, "dim": dim, "subgroups": groups},
         _inputs(dims, DType.F32), out, DType.F32)


def test_local_all_reduce_bf16_max_exact():
    from paper_2105_04663_b200.ir import DType, Op, ReduceKind
    _run(Op.ALL_REDUCE, {"kind": ReduceKind.MAX, "subgroups": GROUPS4[0]},
         _inputs((2, 8192), DType.BF16), (2, 8192), DType.BF16)


@pytest.mark.parametrize("groups", [((0, 1), (2, 3)), ((0, 2), (1, 3))])
def test_local_all_gather_split_halves(groups):
    """spmd_local_all_gather_split / _split_t: hi + lo == the gathered value
    exactly, hi is the tf32 rounding of it; _split_t writes the K-major
    transpose."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    P, f32 = 4, DType.F32
    g = torch.Generator(device="cuda").manual_seed(9)
    flat = [d for grp in groups for d in grp]
    st = torch.cuda.current_stream().cuda_stream
    # lhs: [2, 3, 2048] per partition gathered along the last dim
    x = torch.randn((P, 2, 3, 2048), generator=g, device="cuda")
    hi = torch.empty((P, 2, 3, 4096), device="cuda")
    lo = torch.empty_like(hi)
    C.check(C.lib().spmd_local_all_gather_split(desc(x, Shape((2, 3, 2048), f32)),
                                                desc(hi, Shape((2, 3, 4096), f32)),
                                                desc(lo, Shape((2, 3, 4096), f32)), 2,
                                                C.i32_array(flat), len(groups), 2, P, st), "split")
    # rhs: [K_local=128, N=96] per partition gathered along K, K-major transpose out
    w = torch.randn((P, 128, 96), generator=g, device="cuda")
    thi = torch.empty((P, 96, 256), device="cuda")
    tlo = torch.empty_like(thi)
    C.check(C.lib().spmd_local_all_gather_split_t(desc(w, Shape((128, 96), f32)),
                                                  desc(thi, Shape((96, 256), f32)),
                                                  desc(tlo, Shape((96, 256), f32)),
                                                  C.i32_array(flat), len(groups), 2, P, st),
            "split_t")
    torch.cuda.synchronize()
    for p in range(P):
        grp = next(gr for gr in groups if p in gr)
        full = torch.cat([x[m] for m in grp], dim=-1)
        assert torch.equal(hi[p] + lo[p], full)
        assert torch.equal(hi[p], (hi[p].view(torch.int32) & ~0x1FFF).view(torch.float32))
        wfull = torch.cat([w[m] for m in grp], dim=0).t()
        assert torch.equal(thi[p] + tlo[p], wfull)
