"""One launch each of our GEMM and cuBLAS on one shape (for ncu A/B)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 65536, 8192)))
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, st), "g")
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
print("ok")
