"""Time our GEMM on given shapes (env knobs picked up by the library)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
st = torch.cuda.current_stream().cuda_stream
env = {k: v for k, v in os.environ.items() if k.startswith("SPMD_GEMM")}
SHAPES = [(16384, 65536, 8192), (16384, 8192, 65536), (16384, 32768, 8192), (16384, 8192, 32768),
          (8192, 16384, 8192), (8192, 8192, 16384)]
for M, N, K in SHAPES:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, st), "g")
    for _ in range(2): f()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(5): f()
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 5)
    print(json.dumps({"M": M, "N": N, "K": K, "env": env, "tflops": round(2 * M * N * K / best / 1e9, 1)}), flush=True)
    del a, b, c
