"""Run the C4 conv layer (NHWC [8,1024,1024,128] x HWIO [3,3,128,128], pad 1,
ReLU) a few times through spmd_convolution (for ncu captures)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
from paper_2105_04663_b200.executor import desc
from paper_2105_04663_b200.ir import DType, Shape
N, H, W, Ci, Co = 8, 1024, 1024, 128, 128
x = torch.randn((1, N, H, W, Ci), device="cuda", dtype=torch.bfloat16)
w = torch.randn((1, 3, 3, Ci, Co), device="cuda", dtype=torch.bfloat16) * 0.03
y = torch.empty((1, N, H, W, Co), device="cuda", dtype=torch.bfloat16)
c = C.SpmdConvDims()
c.lhs_batch, c.lhs_feature, c.rhs_in_feature, c.rhs_out_feature = 0, 3, 2, 3
c.out_batch, c.out_feature, c.n_spatial = 0, 3, 2
for i in range(2):
    c.lhs_spatial[i], c.rhs_spatial[i], c.out_spatial[i] = 1 + i, i, 1 + i
    c.size[i], c.stride[i], c.pad_low[i], c.pad_high[i] = 3, 1, 1, 1
    c.base_dilation[i] = c.window_dilation[i] = 1
c.epilogue = 1
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    C.check(C.lib().spmd_convolution(desc(x, Shape((N, H, W, Ci), DType.BF16)),
                                     desc(w, Shape((3, 3, Ci, Co), DType.BF16)),
                                     desc(y, Shape((N, H, W, Co), DType.BF16)), ctypes.byref(c), 1,
                                     st), "conv")
torch.cuda.synchronize()
print("ok")
