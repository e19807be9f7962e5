"""Micro-benchmarks of the hot kernels at the C2 (paper-dims, 1 GPU) shapes.

    python scripts/kernel_bench.py [gemm|softmax|all]

Times each kernel with CUDA events on the launching stream after warm-up and
prints one JSON line per case (TFLOP/s or GB/s).
"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Op, Shape, infer_shape  # noqa: E402


def timeit(fn, reps=10, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def dot_case(name, lshape, rshape, lb, rb, lc, rc):
    lib = C.lib()
    lsh, rsh = Shape(lshape, DType.BF16), Shape(rshape, DType.BF16)
    attrs = {"lhs_batch": lb, "rhs_batch": rb, "lhs_contracting": lc, "rhs_contracting": rc}
    osh = infer_shape(Op.DOT, [lsh, rsh], attrs)
    a = torch.randn((1,) + lshape, device="cuda", dtype=torch.bfloat16)
    b = torch.randn((1,) + rshape, device="cuda", dtype=torch.bfloat16) * 0.01
    o = torch.empty((1,) + osh.dims, device="cuda", dtype=torch.bfloat16)
    dd = C.SpmdDotDims()
    dd.n_batch, dd.n_contract = len(lb), len(lc)
    for i, (x, y) in enumerate(zip(lb, rb)):
        dd.lhs_batch[i], dd.rhs_batch[i] = x, y
    for i, (x, y) in enumerate(zip(lc, rc)):
        dd.lhs_contracting[i], dd.rhs_contracting[i] = x, y
    da, db, do = desc(a, lsh), desc(b, rsh), desc(o, osh)
    st = torch.cuda.current_stream().cuda_stream

    def fn():
        C.check(lib.spmd_dot(da, db, do, ctypes.byref(dd), 1, st), "dot")
    ms = timeit(fn)
    k = 1
    for d in lc:
        k *= lshape[d]
    flops = 2.0 * osh.num_elements * k
    print(json.dumps({"kernel": "gemm_bf16_tcgen05", "case": name, "ms": ms,
                      "tflops": flops / ms / 1e9}), flush=True)


def gemms():
    B, S, M, N, D, H = 16, 1024, 8192, 128, 256, 65536
    dot_case("qkv x[B,S,M].w[M,N,D]", (B, S, M), (M, N, D), (), (), (2,), (0,))
    dot_case("logits q.k", (B, S, N, D), (B, S, N, D), (0, 2), (0, 2), (3,), (3,))
    dot_case("ctx p.v", (B, N, S, S), (B, S, N, D), (0, 1), (0, 2), (3,), (1,))
    dot_case("out ctx_t.wo", (B, S, N, D), (N, D, M), (), (), (2, 3), (0, 1))
    dot_case("ffn_in res.wi", (B, S, M), (M, H), (), (), (2,), (0,))
    dot_case("ffn_out act.wt", (B, S, H), (H, M), (), (), (2,), (0,))
    dot_case("square 8192", (8192, 8192), (8192, 8192), (), (), (1,), (0,))


def softmax():
    lib = C.lib()
    shp = Shape((16, 128, 1024, 1024), DType.BF16)
    x = torch.randn((1,) + shp.dims, device="cuda", dtype=torch.bfloat16)
    y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    dx, dy = desc(x, shp), desc(y, shp)
    ms = timeit(lambda: C.check(lib.spmd_softmax_lastdim(dx, dy, 1, st), "softmax"))
    ref = torch.softmax(x[0, 0, 0].float(), -1)
    err = (y[0, 0, 0].float() - ref).abs().max().item()
    print(json.dumps({"kernel": "softmax_rows_bf16_vec", "ms": ms,
                      "gbs": 2 * x.numel() * 2 / ms / 1e6, "max_err": err}), flush=True)


def datamove():
    """HBM-bound kernels at C4/C5 sizes: GB/s = (bytes read + written) / time."""
    lib = C.lib()
    st = torch.cuda.current_stream().cuda_stream
    bf = DType.BF16
    # C4 halo window: 8-way H-sharded [8,128,1024,128] shard + 1-row halos ->
    # masked window [8,130,1024,128] in one pass.
    N, c, W, Ch = 8, 128, 1024, 128
    val = torch.randn((1, N, c, W, Ch), device="cuda", dtype=torch.bfloat16)
    lh = torch.randn((1, N, 1, W, Ch), device="cuda", dtype=torch.bfloat16)
    rh = torch.randn_like(lh)
    out = torch.empty((1, N, c + 2, W, Ch), device="cuda", dtype=torch.bfloat16)
    start = torch.zeros((1,), dtype=torch.int32, device="cuda")
    off = torch.full((1,), 3 * 128 - 1, dtype=torch.int32, device="cuda")
    fill = torch.zeros((1,), dtype=torch.bfloat16, device="cuda")
    pieces = (C.SpmdTensor * 3)(desc(lh, Shape((N, 1, W, Ch), bf)),
                                desc(val, Shape((N, c, W, Ch), bf)),
                                desc(rh, Shape((N, 1, W, Ch), bf)))
    sh_s = Shape((), DType.S32)
    ms = timeit(lambda: C.check(lib.spmd_halo_window(
        pieces, 3, 1, desc(start, sh_s), 1, desc(off, sh_s), desc(fill, Shape((), bf)), 0, 1024,
        1, desc(out, Shape((N, c + 2, W, Ch), bf)), 1, st), "halo"))
    by = (val.numel() + 2 * lh.numel() + out.numel()) * 2
    print(json.dumps({"kernel": "halo_rows_kernel", "case": "C4 [8,128+2,1024,128] bf16",
                      "ms": ms, "gbs": by / ms / 1e6}), flush=True)
    # C5 uneven mask: [1001 -> 126 rows/shard, 524288] f32 range mask on the last shard.
    rows, D1 = 126, 524288
    x = torch.randn((1, rows, D1), device="cuda")
    y = torch.empty_like(x)
    off = torch.full((1,), 7 * 126, dtype=torch.int32, device="cuda")
    fill = torch.full((1,), float("-inf"), device="cuda")
    f32 = DType.F32
    ms = timeit(lambda: C.check(lib.spmd_mask_range(
        desc(x, Shape((rows, D1), f32)), desc(off, sh_s), desc(fill, Shape((), f32)),
        desc(y, Shape((rows, D1), f32)), 0, 0, 1001, 0, 1, st), "mask"))
    print(json.dumps({"kernel": "mask_range_kernel", "case": "C5 [126,524288] f32",
                      "ms": ms, "gbs": 2 * x.numel() * 4 / ms / 1e6}), flush=True)
    # C5 padded layout: pad [1001,524288] -> [1008,524288] f32 (localize).
    x = torch.randn((1, 1001, D1), device="cuda")
    y = torch.empty((1, 1008, D1), device="cuda")
    z = torch.zeros((1,), device="cuda")
    lo, hi, it = C.i64_array([0, 0]), C.i64_array([7, 0]), C.i64_array([0, 0])
    ms = timeit(lambda: C.check(lib.spmd_pad(desc(x, Shape((1001, D1), f32)), desc(z, Shape((), f32)),
                                             desc(y, Shape((1008, D1), f32)), lo, hi, it, 1, st),
                                "pad"))
    print(json.dumps({"kernel": "pad_gather_kernel (pad)", "case": "C5 [1001->1008,524288] f32",
                      "ms": ms, "gbs": (x.numel() + y.numel()) * 4 / ms / 1e6}), flush=True)
    # dynamic-slice of the local shard out of the padded full value.
    s0 = torch.full((1,), 126 * 3, dtype=torch.int32, device="cuda")
    s1 = torch.zeros((1,), dtype=torch.int32, device="cuda")
    y2 = torch.empty((1, 126, D1), device="cuda")
    starts = (C.SpmdTensor * 2)(desc(s0, sh_s), desc(s1, sh_s))
    ms = timeit(lambda: C.check(lib.spmd_dynamic_slice(desc(y, Shape((1008, D1), f32)), starts,
                                                       desc(y2, Shape((126, D1), f32)), 1, st),
                                "ds"))
    print(json.dumps({"kernel": "strided_copy_kernel (dynamic-slice)",
                      "case": "C5 [1008,524288] -> [126,524288] f32", "ms": ms,
                      "gbs": 2 * y2.numel() * 4 / ms / 1e6}), flush=True)
    # C2 transpose ctx [16,128,1024,256] -> [16,1024,128,256] bf16.
    a = torch.randn((1, 16, 128, 1024, 256), device="cuda", dtype=torch.bfloat16)
    b = torch.empty((1, 16, 1024, 128, 256), device="cuda", dtype=torch.bfloat16)
    perm = C.i32_array([0, 2, 1, 3])
    ms = timeit(lambda: C.check(lib.spmd_transpose(desc(a, Shape((16, 128, 1024, 256), bf)),
                                                   desc(b, Shape((16, 1024, 128, 256), bf)), perm,
                                                   1, st), "tr"))
    print(json.dumps({"kernel": "strided_copy_kernel (transpose)",
                      "case": "C2 ctx [16,128,1024,256] bf16", "ms": ms,
                      "gbs": 2 * a.numel() * 2 / ms / 1e6}), flush=True)


def attention():
    lib = C.lib()
    B, S, N, D = 16, 1024, 128, 256
    q = torch.randn((1, B, S, N, D), device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    o = torch.empty((1, B, N, S, D), device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    qd = desc(q, Shape((B, S, N, D), DType.BF16))
    kd = desc(k, Shape((B, S, N, D), DType.BF16))
    vd = desc(v, Shape((B, S, N, D), DType.BF16))
    od = desc(o, Shape((B, N, S, D), DType.BF16))
    ms = timeit(lambda: C.check(lib.spmd_attention(qd, kd, vd, od, 0.0625, 1, st), "attn"))
    flops = 4.0 * B * N * S * S * D
    print(json.dumps({"kernel": "attention_tcgen05", "case": "C2 attention B16 S1024 N128 D256",
                      "ms": ms, "tflops": flops / ms / 1e9}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("datamove", "all"):
        datamove()
    if what in ("attention", "all"):
        attention()
    if what in ("softmax", "all"):
        softmax()
    if what in ("gemm", "all"):
        gemms()
