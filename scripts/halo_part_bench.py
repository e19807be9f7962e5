"""Time spmd_halo_convolution at the C4 per-GPU shape at N=4 (window of
1 + 256 + 1 rows of [8, *, 1024, 128] bf16, 3x3 conv, ReLU).

    python scripts/halo_part_bench.py

Round 2 also tried splitting this conv into a shard-only launch (issued
while the halo permutes are in flight) plus a boundary-tile launch: bit-
identical, but 0.446 + 0.058 ms against 0.430 ms for one launch -- more
than the ~0.035 ms per layer of permute it would hide -- so it was not kept.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402

N, H, W, Ci, Co = 8, 256, 1024, 128, 128
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
bf = DType.BF16
top = torch.randn(1, N, 1, W, Ci, device=dev).bfloat16()
mid = torch.randn(1, N, H, W, Ci, device=dev).bfloat16()
bot = torch.randn(1, N, 1, W, Ci, device=dev).bfloat16()
w = (torch.randn(1, 3, 3, Ci, Co, device=dev) / 34).bfloat16()
start = torch.zeros(1, dtype=torch.int32, device=dev)
pieces = (C.SpmdTensor * 3)(desc(top, Shape((N, 1, W, Ci), bf)), desc(mid, Shape((N, H, W, Ci), bf)),
                            desc(bot, Shape((N, 1, W, Ci), bf)))
win = C.SpmdTensor()
win.dtype, win.rank = C.DTYPE_CODE[bf], 4
for i, d in enumerate((N, H + 2, W, Ci)):
    win.dims[i] = d
cd = C.SpmdConvDims()
cd.lhs_batch, cd.lhs_feature, cd.rhs_in_feature, cd.rhs_out_feature = 0, 3, 2, 3
cd.out_batch, cd.out_feature, cd.n_spatial = 0, 3, 2
for i, (ls, rs, os_) in enumerate([(1, 0, 1), (2, 1, 2)]):
    cd.lhs_spatial[i], cd.rhs_spatial[i], cd.out_spatial[i] = ls, rs, os_
    cd.size[i], cd.stride[i] = 3, 1
    cd.pad_low[i] = cd.pad_high[i] = 0 if i == 0 else 1
    cd.base_dilation[i] = cd.window_dilation[i] = 1
cd.epilogue = 1
ssh = Shape((), DType.S32)
out = torch.zeros(1, N, H, W, Co, device=dev).bfloat16()


def run():
    C.check(C.lib().spmd_halo_convolution(
        pieces, 3, 1, desc(start, ssh), 0, desc(start, ssh), 0, 0, 0, win,
        desc(w, Shape((3, 3, Ci, Co), bf)), desc(out, Shape((N, H, W, Co), bf)),
        ctypes.byref(cd), 1, st), "halo_conv")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(run)
print(json.dumps({"ms": ms, "tflops": 2.0 * N * H * W * Ci * Co * 9 / ms / 1e9}))
