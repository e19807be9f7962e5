"""Wide tcgen05 GEMM rasterisation sweep on a C2 shape (default FFN-in
16384 x 65536 x 8192): time per (gemm_group, gemm_raster_n) setting,
interleaved rounds on the same box.  Under ncu (`--ncu`: one launch per
setting, no timing loop) the launch list carries each setting's DRAM bytes.

    python scripts/gemm_raster.py [M N K] [--ncu]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
M, N, K = (int(v) for v in args[:3]) if len(args) >= 3 else (16384, 65536, 8192)
ncu = "--ncu" in sys.argv
# (gemm_group, gemm_raster_n, gemm_hint, gemm_store_hint)
settings = [(g, r, 0, 0) for r in (0, 1) for g in (4, 8, 16, 32)]
if "--hints" in sys.argv:
    settings = [(16, 0, h, sh) for h in (0, 1, 2) for sh in (0, 1)]
st = torch.cuda.current_stream().cuda_stream
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)


def run():
    C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, st), "g")


best = {}
for rnd in range(1 if ncu else 3):
    for g, r, h, sh in settings:
        with C.option("gemm_group", g), C.option("gemm_raster_n", r), C.option("gemm_hint", h), \
                C.option("gemm_store_hint", sh):
            if ncu:
                run()
                torch.cuda.synchronize()
                continue
            run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            best[(g, r, h, sh)] = min(best.get((g, r, h, sh), 1e9), ms)
for (g, r, h, sh), ms in sorted(best.items()):
    print(json.dumps({"M": M, "N": N, "K": K, "group": g, "raster_n": r, "hint": h,
                      "store_hint": sh, "ms": round(ms, 3),
                      "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}), flush=True)
