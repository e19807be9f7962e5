"""Same-box A/B of persistent-attention options at the C2 shape (or a given
B S T N D), interleaved rounds so power-cap drift hits every arm alike.

    python scripts/attn_ab.py [--opt NAME V0 V1] [B S T N D]

Arms: attn_kt 0 (P in tensor memory, default) and 1 (P in shared memory);
both run the same arithmetic, so their outputs must be bit-identical.
(profiles/r2_attn_ab.log also holds a since-removed MMA-order option.)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402

argv = sys.argv[1:]
opt, vals = "attn_kt", [0, 1]
if argv[:1] == ["--opt"]:
    opt, vals, argv = argv[1], [int(argv[2]), int(argv[3])], argv[4:]
B, S, T, N, D = (int(x) for x in argv[:5]) if len(argv) >= 5 else (16, 1024, 1024, 128, 256)
st = torch.cuda.current_stream().cuda_stream
q = torch.randn((1, B, S, N, D), device="cuda", dtype=torch.bfloat16)
k = torch.randn((1, B, T, N, D), device="cuda", dtype=torch.bfloat16)
v = torch.randn_like(k)
arms = vals
outs = {a: torch.empty((1, B, N, S, D), device="cuda", dtype=torch.bfloat16) for a in arms}


def run(a):
    with C.option(opt, a):
        C.check(C.lib().spmd_attention(desc(q, Shape((B, S, N, D), DType.BF16)),
                                       desc(k, Shape((B, T, N, D), DType.BF16)),
                                       desc(v, Shape((B, T, N, D), DType.BF16)),
                                       desc(outs[a], Shape((B, N, S, D), DType.BF16)),
                                       D ** -0.5, 1, st), "attention")


def timed(a, reps=20):
    for _ in range(3):
        run(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        run(a)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {a: [] for a in arms}
for r in range(8):
    # rotate the arm order every round: clocks drift under the power cap
    for a in arms[r % len(arms):] + arms[:r % len(arms)]:
        res[a].append(timed(a))
assert torch.equal(outs[arms[0]], outs[arms[1]])
f = 4.0 * B * N * S * T * D
for a in arms:
    ms = min(res[a])
    med = sorted(res[a])[len(res[a]) // 2]
    print(json.dumps({"B": B, "S": S, "T": T, "N": N, "D": D, opt: a,
                      "ms": round(ms, 4),
                      "tflops": round(f / ms / 1e9, 1), "tflops_median": round(f / med / 1e9, 1),
                      "ms_all": [round(x, 4) for x in res[a]]}), flush=True)
