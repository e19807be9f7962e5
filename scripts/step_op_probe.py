"""Time single steps of the C2 executor program in isolation (the step's own
function on the step's own operands, 10 back-to-back calls) beside the same
GEMM shape through spmd_gemm_bf16 -- separates a slow layout / kernel path
from in-step context (clocks, L2).

    python scripts/step_op_probe.py [op ids ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench as B  # noqa: E402
from paper_2105_04663_b200 import _capi as C  # noqa: E402

dev = torch.device("cuda", 0)
run = B._Run("c2", 1, 0, dev, None)
ex = run.ex
ids = sys.argv[1:] or [s.ins.id for s in ex.steps if s.ins.opcode.value in ("dot", "add", "relu")]
keep = set()
for s in ex.steps:
    if s.ins.id in ids:
        keep |= set(s.ops)
ex.run(run.inputs, keep=keep)
env = {"__inputs__": run.inputs}
env.update({k: v for k, v in ex.last_env.items() if k in keep})
st = torch.cuda.current_stream(dev)


def t(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for s in ex.steps:
    if s.ins.id not in ids:
        continue
    ms = t(lambda: s.fn(env, st.cuda_stream))
    print(f"{s.ins.id:14s} {s.ins.opcode.value:8s} {ms:7.3f} ms  ops={s.ops}", flush=True)
for M, N, K in ((16384, 32768, 8192), (16384, 65536, 8192), (16384, 8192, 65536),
                (16384, 8192, 32768)):
    a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    b = torch.randn(K, N, device=dev, dtype=torch.bfloat16) * 0.01
    c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ms = t(lambda: C.check(C.lib().spmd_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N,
                                                  K, 0, st.cuda_stream), "gemm"))
    print(f"gemm {M}x{N}x{K}: {ms:7.3f} ms  {2.0 * M * N * K / ms / 1e9:7.1f} TF/s", flush=True)
    del a, b, c
