"""Pad (single-pass edge gather and fill+copy interior path) and dynamic
slice / update-slice kernels vs numpy (reference simulator.py pad /
dynamic-slice semantics: starts clamped into [0, operand - size]).
Bit-exact: pure data movement."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_TORCH = {"f32": "float32", "s32": "int32", "pred": "bool"}


def _dev(arr):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


def _pad(x, values, low, high, interior, dt):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import Shape
    P = x.shape[0]
    dims = x.shape[1:]
    od = tuple(n + (n - 1) * it + lo + hi if n else lo + hi
               for n, lo, hi, it in zip(dims, low, high, interior))
    xt = _dev(x)
    vt = _dev(values)
    out = torch.empty((P,) + od, dtype=xt.dtype, device="cuda")
    C.check(C.lib().spmd_pad(desc(xt, Shape(dims, dt)), desc(vt, Shape((), dt)),
                             desc(out, Shape(od, dt)), C.i64_array(low), C.i64_array(high),
                             C.i64_array(interior), P, torch.cuda.current_stream().cuda_stream),
            "pad")
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _np_pad(x, v, low, high, interior):
    dims = x.shape
    od = tuple(n + (n - 1) * it + lo + hi for n, lo, hi, it in zip(dims, low, high, interior))
    out = np.full(od, v, dtype=x.dtype)
    idx = tuple(slice(lo, lo + (n - 1) * (it + 1) + 1, it + 1)
                for n, lo, it in zip(dims, low, interior))
    out[idx] = x
    return out


@pytest.mark.parametrize("dims,low,high,interior,dt", [
    ((1001, 64), (0, 0), (7, 0), (0, 0), "f32"),          # C5 localize: vector path
    ((5, 6, 8), (1, 0, 4), (2, 0, 4), (0, 0, 0), "f32"),  # merged middle dim, vec last
    ((5, 7), (1, 3), (0, 2), (0, 0), "f32"),              # misaligned: scalar path
    ((3, 4, 32), (0, 1, 16), (2, 0, 0), (0, 0, 0), "pred"),
    ((4, 9), (2, 1), (1, 0), (1, 2), "s32"),              # interior: fill+copy path
    ((16,), (0,), (0,), (0,), "s32"),                     # no-op pad
    ((9, 12288), (0, 0), (7, 0), (0, 0), "f32"),          # row-chunk kernel (3072 vectors)
    ((6, 8200), (1, 8), (2, 0), (0, 0), "f32"),           # row-chunk kernel, padded rows
    ((5, 16388), (0, 4), (1, 4), (0, 0), "s32"),          # row-chunk, partial last chunk
])
def test_pad_matches_numpy(dims, low, high, interior, dt):
    from paper_2105_04663_b200.ir import DType
    dtype = {"f32": DType.F32, "s32": DType.S32, "pred": DType.PRED}[dt]
    rng = np.random.default_rng(len(dims) + sum(low))
    P = 3
    if dt == "pred":
        x = rng.random((P,) + dims) < 0.5
        vals = np.array([True, False, True])
    else:
        x = rng.standard_normal((P,) + dims).astype(_TORCH[dt]) * 100
        vals = np.array([-1.5, 2.0, 7.0]).astype(_TORCH[dt])
    got = _pad(x, vals, low, high, interior, dtype)
    for p in range(P):
        np.testing.assert_array_equal(got[p], _np_pad(x[p], vals[p], low, high, interior))


@pytest.mark.parametrize("W", [64, 12292])    # generic / row-chunk copy kernel
@pytest.mark.parametrize("update", [False, True])
def test_dynamic_slice_clamped_per_partition(update, W):
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    P, R, r = 4, 40, 9
    rng = np.random.default_rng(5)
    x = rng.standard_normal((P, R, W)).astype(np.float32)
    starts0 = np.array([-3, 5, 31, 100], dtype=np.int32)   # clamp low / mid / edge / high
    s0 = _dev(starts0)
    s1 = _dev(np.array([0, 0, 0, 0], dtype=np.int32))
    sh_s = Shape((), DType.S32)
    starts = (C.SpmdTensor * 2)(desc(s0, sh_s), desc(s1, sh_s))
    st = torch.cuda.current_stream().cuda_stream
    xt = _dev(x)
    clamp = np.clip(starts0, 0, R - r)
    if not update:
        out = torch.empty((P, r, W), device="cuda")
        C.check(C.lib().spmd_dynamic_slice(desc(xt, Shape((R, W), DType.F32)), starts,
                                           desc(out, Shape((r, W), DType.F32)), P, st), "ds")
        got = out.cpu().numpy()
        for p in range(P):
            np.testing.assert_array_equal(got[p], x[p, clamp[p]:clamp[p] + r])
    else:
        u = rng.standard_normal((P, r, W)).astype(np.float32)
        ut = _dev(u)
        out = torch.empty_like(xt)
        C.check(C.lib().spmd_dynamic_update_slice(
            desc(xt, Shape((R, W), DType.F32)), desc(ut, Shape((r, W), DType.F32)), starts,
            desc(out, Shape((R, W), DType.F32)), P, st), "dus")
        got = out.cpu().numpy()
        for p in range(P):
            want = x[p].copy()
            want[clamp[p]:clamp[p] + r] = u[p]
            np.testing.assert_array_equal(got[p], want)


@pytest.mark.parametrize("inner", [8192 + 512, 12])   # row-uniform kernel / element kernel
def test_halo_window_matches_numpy(inner):
    """window = DS(mask(concat(left, shard, right)), start) in one pass
    (reference formatting.py:109-182 exchange_and_slice)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    P, outer, c = 4, 3, 6
    rng = np.random.default_rng(inner)
    lh = rng.standard_normal((P, outer, 1, inner)).astype(np.float32)
    val = rng.standard_normal((P, outer, c, inner)).astype(np.float32)
    rh = rng.standard_normal((P, outer, 2, inner)).astype(np.float32)
    starts = np.array([0, 1, 3, 9], dtype=np.int32)      # last clamps to buf_len - window
    offsets = np.array([-1, 5, 11, 17], dtype=np.int32)  # global row of buffer position 0
    fills = np.array([-1.0, -2.0, -3.0, -4.0], dtype=np.float32)
    low, high, window = 0, 20, c + 1
    f32, s32 = DType.F32, DType.S32
    ts = [_dev(a) for a in (lh, val, rh)]
    pieces = (C.SpmdTensor * 3)(*[desc(t, Shape(t.shape[1:], f32)) for t in ts])
    st_t, off_t, fill_t = _dev(starts), _dev(offsets), _dev(fills)
    out = torch.empty((P, outer, window, inner), device="cuda")
    C.check(C.lib().spmd_halo_window(pieces, 3, 1, desc(st_t, Shape((), s32)), 1,
                                     desc(off_t, Shape((), s32)), desc(fill_t, Shape((), f32)),
                                     low, high, 1, desc(out, Shape((outer, window, inner), f32)),
                                     P, torch.cuda.current_stream().cuda_stream), "halo")
    got = out.cpu().numpy()
    for p in range(P):
        buf = np.concatenate([lh[p], val[p], rh[p]], axis=1)
        s0 = int(np.clip(starts[p], 0, buf.shape[1] - window))
        g = np.arange(buf.shape[1]) + offsets[p]
        keep = (g >= low) & (g < high)
        masked = np.where(keep[None, :, None], buf, fills[p])
        np.testing.assert_array_equal(got[p], masked[:, s0:s0 + window])


@pytest.mark.parametrize("inner", [8, 16384 + 36])      # element kernel / row-chunk kernel
def test_mask_range_matches_select_chain(inner):
    """spmd_mask_range = select(low <= iota + offset[p] < high, x, fill[p])
    (reference partitioner.py:205-247 select_range / mask_uneven)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    P, outer, n = 3, 2, 13
    rng = np.random.default_rng(inner)
    x = rng.standard_normal((P, outer, n, inner)).astype(np.float32)
    offs = np.array([0, 10, 27], dtype=np.int32)
    fills = np.array([-1.0, 0.0, np.inf], dtype=np.float32)
    low, high = 3, 30
    out = torch.empty((P, outer, n, inner), device="cuda")
    sh = Shape((outer, n, inner), DType.F32)
    xt, ot, ft = _dev(x), _dev(offs), _dev(fills)      # keep the buffers alive
    C.check(C.lib().spmd_mask_range(desc(xt, sh), desc(ot, Shape((), DType.S32)),
                                     desc(ft, Shape((), DType.F32)), desc(out, sh), 1,
                                     low, high, 1, P, torch.cuda.current_stream().cuda_stream),
            "mask_range")
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for p in range(P):
        g = np.arange(n) + offs[p]
        keep = ((g >= low) & (g < high))[None, :, None]
        np.testing.assert_array_equal(got[p], np.where(keep, x[p], fills[p]))


@pytest.mark.parametrize("dims,perm,dt", [
    ((4, 6, 8, 16), (1, 0, 2, 3), "bf16"),      # the MoE annotation transposes: vector path
    ((4, 6, 8, 16), (1, 0, 2, 3), "f32"),
    ((5, 7, 3), (2, 0, 1), "f32"),              # last dim moves: scalar path
    ((3, 4, 16400), (1, 0, 2), "bf16"),         # row-chunk kernel (2050 vectors per row)
    ((6, 10), (1, 0), "s32"),
])
def test_transpose_relu_matches_numpy(dims, perm, dt):
    """spmd_transpose_relu == numpy maximum(transpose(x), 0) bit for bit,
    with -0.0, NaN, +-inf and (ints) INT_MIN in the data."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    rng = np.random.default_rng(len(dims) + sum(dims))
    if dt == "s32":
        x = rng.integers(-50, 50, dims).astype(np.int32)
        x.flat[0] = np.iinfo(np.int32).min
        t = torch.from_numpy(x).cuda()
        dtype = DType.S32
    else:
        x = rng.standard_normal(dims).astype(np.float32)
        x.flat[:4] = [-0.0, np.nan, -np.inf, np.inf]
        t = torch.from_numpy(x).cuda()
        if dt == "bf16":
            t = t.bfloat16()
            x = t.float().cpu().numpy()
        dtype = DType.BF16 if dt == "bf16" else DType.F32
    odims = tuple(dims[p] for p in perm)
    out = torch.empty(odims, dtype=t.dtype, device="cuda")
    C.check(C.lib().spmd_transpose_relu(desc(t, Shape(dims, dtype)), desc(out, Shape(odims, dtype)),
                                        C.i32_array(perm), 1,
                                        torch.cuda.current_stream().cuda_stream), "transpose_relu")
    torch.cuda.synchronize()
    want = np.maximum(np.transpose(x, perm), 0)
    got = out.float().cpu().numpy() if dt == "bf16" else out.cpu().numpy()
    np.testing.assert_array_equal(got, want.astype(got.dtype))
    if dt != "s32":
        assert not np.signbit(got[np.transpose(x, perm) == 0]).any()   # -0 -> +0
