"""Our tcgen05 GEMM vs cuBLAS (torch.matmul) on the same box, interleaved
rounds so power-cap drift hits both alike.  C = A[M,K] . B[K,N] bf16."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C

def t(fn, reps=10):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2): fn()
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(reps): fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

shapes = [(8192, 8192, 8192), (16384, 32768, 8192), (16384, 8192, 32768), (16384, 65536, 8192),
          (16384, 8192, 65536), (8192, 16384, 8192), (8192, 8192, 16384)]
st = torch.cuda.current_stream().cuda_stream
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) * 0.01
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    c_ref = torch.empty_like(c)
    ours = lambda: C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, st), "g")
    cub = lambda: torch.matmul(a, b, out=c_ref)
    res = {"ours": [], "cublas": []}
    for _ in range(3):
        res["ours"].append(t(ours)); res["cublas"].append(t(cub))
    f = 2.0 * M * N * K
    # both results against each other (bf16 outputs, fp32 accumulation in
    # different orders): normwise <= 8e-3
    err = ((c.float() - c_ref.float()).abs().max() / c_ref.float().abs().max().clamp(min=1)).item()
    assert err < 8e-3, (M, N, K, err)
    print(json.dumps({"M": M, "N": N, "K": K, "max_rel_vs_cublas": err,
                      "ours_tflops": round(f / min(res["ours"]) / 1e9, 1),
                      "cublas_tflops": round(f / min(res["cublas"]) / 1e9, 1)}), flush=True)
    del a, b, c
