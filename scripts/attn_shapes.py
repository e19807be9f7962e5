"""Attention kernel variants at the C2 shapes and vs key length.

    python scripts/attn_shapes.py

For each kernel variant (option attn_kt: 0 = persistent 8-softmax-warp
kernel with P in tensor memory, 1 = the same with P in shared memory,
64 / 128 = the round-1 non-persistent kernels) times
spmd_attention with CUDA events (10 launches after 3 warm-ups) and checks
one head against an fp32 torch reference.  One JSON line per case.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
cases = [(16, 1024, 1024, 128, 256), (4, 1024, 4096, 128, 256), (1, 1024, 16384, 128, 256),
         (16, 1024, 1024, 128, 128)]
if len(sys.argv) > 1 and sys.argv[1] == "c2":
    cases = cases[:1]
for B, S, T, N, D in cases:
    q = torch.randn((1, B, S, N, D), device="cuda", dtype=torch.bfloat16)
    k = torch.randn((1, B, T, N, D), device="cuda", dtype=torch.bfloat16)
    v = torch.randn_like(k)
    o = torch.empty((1, B, N, S, D), device="cuda", dtype=torch.bfloat16)
    scale = 1.0 / D ** 0.5
    f = lambda: C.check(C.lib().spmd_attention(desc(q, Shape((B, S, N, D), DType.BF16)),
                                               desc(k, Shape((B, T, N, D), DType.BF16)),
                                               desc(v, Shape((B, T, N, D), DType.BF16)),
                                               desc(o, Shape((B, N, S, D), DType.BF16)), scale, 1,
                                               st), "a")
    for kt in (0, 1, 64, 128):
        with C.option("attn_kt", kt):
            for _ in range(3):
                f()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        bb, nn = B - 1, N - 1
        ref = torch.softmax(q[0, bb, :, nn].float() @ k[0, bb, :, nn].float().T * scale, -1) @ \
            v[0, bb, :, nn].float()
        err = (o[0, bb, nn].float() - ref).abs().max().item() / max(1.0, ref.abs().max().item())
        print(json.dumps({"B": B, "S": S, "T": T, "N": N, "D": D, "attn_kt": kt,
                          "ms": round(ms, 4), "tflops": round(4.0 * B * N * S * T * D / ms / 1e9, 1),
                          "err_last_head": err}), flush=True)
    del q, k, v, o
