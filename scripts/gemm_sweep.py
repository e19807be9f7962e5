"""Time one GEMM shape (bf16 x[M,K] @ w[K,N]) with CUDA events; prints ms and TFLOP/s.
Used with SPMD_GEMM_* environment knobs for rasterisation / cache-policy sweeps."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
M, N, K = (int(x) for x in sys.argv[1:4])
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
f = lambda: C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, st), "gemm")
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(json.dumps({"M": M, "N": N, "K": K, "env": {k: v for k, v in os.environ.items() if k.startswith("SPMD_GEMM")}, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}))
