"""One launch each of the training-step backward kernels at C2 sizes (for ncu):
softmax backward [16*128*1024, 1024] bf16, ReLU backward [16*1024, 65536] bf16."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
from paper_2105_04663_b200.executor import desc
from paper_2105_04663_b200.ir import DType, Shape
lib, s = C.lib(), torch.cuda.current_stream().cuda_stream
R, L = 16 * 128 * 1024, 1024
p = torch.softmax(torch.randn(R, L, device="cuda", dtype=torch.bfloat16), -1)
dp = torch.randn(R, L, device="cuda", dtype=torch.bfloat16)
out = torch.empty_like(p)
sh = Shape((R, L), DType.BF16)
h = torch.randn(16 * 1024, 65536, device="cuda", dtype=torch.bfloat16)
g = torch.randn_like(h)
o2 = torch.empty_like(h)
sh2 = Shape((16 * 1024, 65536), DType.BF16)
for _ in range(2):
    C.check(lib.spmd_softmax_backward_lastdim(desc(p, sh), desc(dp, sh), desc(out, sh), 1, s), "sbwd")
    C.check(lib.spmd_relu_backward(desc(h, sh2), desc(g, sh2), desc(o2, sh2), 1, s), "rbwd")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in [("softmax_bwd", lambda: lib.spmd_softmax_backward_lastdim(desc(p, sh), desc(dp, sh), desc(out, sh), 1, s), 3 * R * L * 2),
                         ("relu_bwd", lambda: lib.spmd_relu_backward(desc(h, sh2), desc(g, sh2), desc(o2, sh2), 1, s), 3 * h.numel() * 2)]:
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms, {nbytes / ms / 1e6:.0f} GB/s algorithmic")
