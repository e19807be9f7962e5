"""Transpose [16,32,1024,256] bf16 -> [16,1024,32,256] (the training step's
ctx / dq / dk / dv layout changes) through spmd_transpose: GB/s, row kernel vs
the per-vector kernel, and exactness vs torch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
from paper_2105_04663_b200.executor import desc
from paper_2105_04663_b200.ir import DType, Shape
lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
x = torch.randn(1, 16, 32, 1024, 256, device="cuda").to(torch.bfloat16)
y = torch.empty(1, 16, 1024, 32, 256, device="cuda", dtype=torch.bfloat16)
import ctypes
perm = (ctypes.c_int32 * 4)(0, 2, 1, 3)
def run():
    C.check(lib.spmd_transpose(desc(x, Shape((16, 32, 1024, 256), DType.BF16)),
                               desc(y, Shape((16, 1024, 32, 256), DType.BF16)), perm, 1, s), "t")
run(); torch.cuda.synchronize()
assert torch.equal(y[0], x[0].permute(0, 2, 1, 3)), "mismatch"
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"rows={'off' if os.environ.get('SPMD_COPY_NO_ROWS') else 'on'}: {ms:.3f} ms, {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
