"""Run one bf16 tcgen05 GEMM shape a few times (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 8192, 8192)))
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0,
                                   torch.cuda.current_stream().cuda_stream), "gemm")
torch.cuda.synchronize()
ref = (a[:256].float() @ b.float())
print("err", ((c[:256].float() - ref).abs().max() / ref.abs().max()).item())
