"""C5 at its full sizes: X[n0, D1], n0 in {1000, 1001, 999},
D1 in {4096, 65536, 524288}, f32 and bf16, dim-0 sharded over 8 partitions
(simulated 8-way mesh on one B200, loopback collectives), resharded to
dim 1 (all-to-all; padded all-to-all for the uneven n0), to replicated
(all-gather + slice), or reduced over dim 0 with the uneven last shard
masked by the reduction identity (partitioner.py:236-247, 571-624).

Both planners, through the Executor on device-resident inputs.  Checks are
on the device against torch restatements of the same global ops: the copy
paths are bit-exact; the reductions use integer-valued inputs so the f32
sum is exact in any order, and bf16 (8-bit mantissa) uses values in
{-1, 0, 1} whose partial and total sums stay below 256 in magnitude, so
every rounding is exact as well.  Max is exact by construction.  The
padded rows of the uneven last shard must not leak into any result: the
shards are padded with NaN (not the reference's 0) so a missing mask shows.
"""

import pytest

pytestmark = pytest.mark.gpu

KINDS = ["a2a", "repl", "reduce_max", "reduce_sum"]
CASES = [(n0, d1) for d1 in (4096, 65536) for n0 in (1000, 1001, 999)] + \
        [(1001, 524288), (1000, 524288)]


def _stack_shards(x, parts):
    """[n0, D1] -> [parts, ceil(n0/parts), D1], tail padded with NaN."""
    import torch
    n0 = x.shape[0]
    per = -(-n0 // parts)
    out = torch.full((parts * per,) + tuple(x.shape[1:]), float("nan"), dtype=x.dtype,
                     device=x.device)
    out[:n0] = x
    return out.view((parts, per) + tuple(x.shape[1:]))


def _check_output(out, want, sharding, parts):
    """Every partition's shard of ``out`` equals its tile of the global
    ``want`` (valid region; replicas all checked)."""
    import torch
    from paper_2105_04663_b200.ir import DType, Shape
    from paper_2105_04663_b200.sharding import shard_offset, shard_shape
    full = Shape(tuple(want.shape), DType.F32)
    per = shard_shape(full, sharding).dims
    for d in range(parts):
        sl = []
        for k, n in enumerate(want.shape):
            o = shard_offset(full, sharding, d, k)
            sl.append(slice(min(o, n), min(o + per[k], n)))
        tile = want[tuple(sl)]
        got = out[d][tuple(slice(0, s) for s in tile.shape)]
        assert torch.equal(got, tile), (d, (got.float() - tile.float()).abs().max().item())


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n0,d1", CASES)
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_c5_full_size_simulated_8way(kind, n0, d1, dt):
    import torch
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.workloads import uneven
    dtype = DType.F32 if dt == "f32" else DType.BF16
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    parts = 8
    g, _ = uneven(n0, d1, kind, parts=parts, dtype=dtype, with_inputs=False)
    ann, _ = propagate(g)
    gen = torch.Generator(device="cuda").manual_seed(n0 + d1)
    hi = 5 if dt == "f32" else 2
    x = torch.randint(-hi + 1, hi, (n0, d1), generator=gen, device="cuda").to(tdt)
    if kind == "a2a" or kind == "repl":
        want = -x
    elif kind == "reduce_max":
        want = x.max(dim=0).values
    else:
        want = x.float().sum(dim=0).to(tdt)
    stacked = _stack_shards(x, parts)
    for plan in ("reference", "fast"):
        prog = partition(ann, parts, plan=plan)
        ex = Executor(prog, nparts=parts)
        out = ex.run([stacked])[0]
        torch.cuda.synchronize()
        ex.check_errors()
        _check_output(out, want, prog.output_shardings[0], parts)
        del ex, out
        torch.cuda.empty_cache()
