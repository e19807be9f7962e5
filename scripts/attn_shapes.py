"""Attention throughput vs key length at fixed FLOPs (per-tile overhead probe)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_04663_b200 import _capi as C
from paper_2105_04663_b200.executor import desc
from paper_2105_04663_b200.ir import DType, Shape
st = torch.cuda.current_stream().cuda_stream
for B, S, T, N, D in [(16, 1024, 1024, 128, 256), (4, 1024, 4096, 128, 256), (1, 1024, 16384, 128, 256),
                      (16, 1024, 1024, 128, 128), (4, 1024, 4096, 128, 128)]:
    q = torch.randn((1, B, S, N, D), device="cuda", dtype=torch.bfloat16)
    k = torch.randn((1, B, T, N, D), device="cuda", dtype=torch.bfloat16)
    v = torch.randn_like(k)
    o = torch.empty((1, B, N, S, D), device="cuda", dtype=torch.bfloat16)
    f = lambda: C.check(C.lib().spmd_attention(desc(q, Shape((B, S, N, D), DType.BF16)),
                                               desc(k, Shape((B, T, N, D), DType.BF16)),
                                               desc(v, Shape((B, T, N, D), DType.BF16)),
                                               desc(o, Shape((B, N, S, D), DType.BF16)), 0.0625, 1, st), "a")
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"B": B, "S": S, "T": T, "N": N, "D": D, "kt": os.environ.get("SPMD_ATTN_KT", "128"), "ms": round(ms, 3),
                      "tflops": round(4.0 * B * N * S * T * D / ms / 1e9, 1)}), flush=True)
    del q, k, v, o
