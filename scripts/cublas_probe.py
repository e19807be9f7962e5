"""cuBLAS (torch.matmul) bf16 on the C2 FFN-in shape, launched for an ncu
capture (the cuBLAS side of profiles/r2_cublas_ffn_ncu_raw.csv)."""
import torch
M,N,K=16384,65536,8192
a=torch.randn(M,K,device="cuda",dtype=torch.bfloat16); b=torch.randn(K,N,device="cuda",dtype=torch.bfloat16)*0.01
c=torch.empty(M,N,device="cuda",dtype=torch.bfloat16)
for _ in range(2): torch.matmul(a,b,out=c)
torch.cuda.synchronize()
