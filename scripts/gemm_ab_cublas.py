"""Same-box A/B of one GEMM shape: ours (spmd_gemm_bf16, current options)
vs cuBLAS (torch.matmul), alternating R rounds of 5 launches each so power /
clock drift hits both; prints every round and the medians.

    python scripts/gemm_ab_cublas.py [M N K] [rounds]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402

args = [int(a) for a in sys.argv[1:]]
M, N, K = args[:3] if len(args) >= 3 else (16384, 65536, 8192)
R = args[3] if len(args) >= 4 else 8
st = torch.cuda.current_stream().cuda_stream
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ours = lambda: C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K,
                                              0, st), "g")
cub = lambda: torch.matmul(a, b, out=c)


def t(fn, reps=5):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


f = 2.0 * M * N * K
res = {"ours": [], "cublas": []}
for r in range(R):
    for name, fn in (("ours", ours), ("cublas", cub)) if r % 2 == 0 else (("cublas", cub), ("ours", ours)):
        res[name].append(f / t(fn) / 1e9)
print(json.dumps({"M": M, "N": N, "K": K, "ours_tflops": [round(x, 1) for x in res["ours"]],
                  "cublas_tflops": [round(x, 1) for x in res["cublas"]],
                  "ours_median": round(statistics.median(res["ours"]), 1),
                  "cublas_median": round(statistics.median(res["cublas"]), 1)}))
