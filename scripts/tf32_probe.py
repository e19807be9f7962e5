"""3xTF32 GEMM (spmd_dot f32) vs cuBLAS TF32 (torch.matmul, allow_tf32) at
the C1 per-partition shape; prints TF/s of both (cuBLAS = 1 tf32 product per
f32 product, ours = 3)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 8192, 8192)
a = torch.randn((1, M, K), device="cuda")
b = torch.randn((1, K, N), device="cuda") / K ** 0.5
out = torch.empty((1, M, N), device="cuda")
dd = C.SpmdDotDims()
dd.n_contract = 1
dd.lhs_contracting[0], dd.rhs_contracting[0] = 1, 0
st = torch.cuda.current_stream().cuda_stream
ours = lambda: C.check(C.lib().spmd_dot(desc(a, Shape((M, K), DType.F32)),
                                        desc(b, Shape((K, N), DType.F32)),
                                        desc(out, Shape((M, N), DType.F32)), ctypes.byref(dd), 1,
                                        st), "dot")
torch.backends.cuda.matmul.allow_tf32 = True
ref = torch.empty((M, N), device="cuda")
cub = lambda: torch.matmul(a[0], b[0], out=ref)


def t(fn, reps=10):
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
res = {"ours_3xtf32": [], "cublas_tf32": []}
for _ in range(3):
    res["ours_3xtf32"].append(f / t(ours) / 1e9)
    res["cublas_tf32"].append(f / t(cub) / 1e9)
print(json.dumps({"M": M, "N": N, "K": K, **{k: round(max(v), 1) for k, v in res.items()}}))
