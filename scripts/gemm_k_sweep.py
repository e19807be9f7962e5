"""Per-tile fixed cost of the persistent GEMMs: time C[M,N] = A[M,K] . B[K,N]
(bf16, spmd_gemm_bf16) for a sweep of K at fixed M, N and fit
t = tiles_per_pair * (t_fixed + kblocks * t_kblock).  t_fixed is what each
tile pays outside its main loop (accumulator drain not overlapped, tile
hand-off); compared across gemm_mode 2 (256 x 256, double-buffered TMEM)
and 3 (256 x 512, single accumulator).

    python scripts/gemm_k_sweep.py [M N]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402


def t(fn, reps=10):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


M, N = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16384, 65536)
st = torch.cuda.current_stream().cuda_stream
Ks = [256, 512, 1024, 2048, 4096, 8192]
for mode, bn in ((3, 512), (2, 256)):
    pairs = 74
    tiles = (M // 256) * (N // bn)
    tpp = tiles / pairs
    xs, ys = [], []
    for K in Ks:
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        with C.option("gemm_mode", mode):
            ms = min(t(lambda: C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(),
                                                             c.data_ptr(), M, N, K, 0, st), "g"))
                     for _ in range(3))
        us_per_tile = ms * 1e3 / tpp
        xs.append(K // 64)
        ys.append(us_per_tile)
        print(json.dumps({"mode": mode, "M": M, "N": N, "K": K, "ms": round(ms, 4),
                          "tflops": round(2.0 * M * N * K / ms / 1e9, 1),
                          "us_per_tile": round(us_per_tile, 3)}), flush=True)
        del a, b, c
    slope, icpt = np.polyfit(xs, ys, 1)
    print(json.dumps({"mode": mode, "fit_us_per_kblock": round(slope, 4),
                      "fit_us_fixed_per_tile": round(icpt, 3),
                      "fixed_share_at_K8192": round(icpt / (icpt + 128 * slope), 4)}), flush=True)
