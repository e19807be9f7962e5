"""Per-op timeline of a bench workload on N GPUs (torchrun), rank 0 prints the
compute/comm stream intervals and the compute-stream idle gaps.  Built
exactly like bench.py's timed step (bench._Run: same program, fusions,
overlap and, for C3, the declared routing); CUDA events around every step
-- eager run, or with GRAPH=1 external event nodes inside the captured graph
(the last of 5 back-to-back replays: bench.py's timed step).

    [GRAPH=1] CFG=c2|c3|c4|c2train torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/timeline.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2105_04663_b200.executor import NcclComm  # noqa: E402

rank, world, local = B._dist_env()
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
comm = NcclComm.from_torch_distributed() if world > 1 else None
run = B._Run(os.environ.get("CFG", "c2"), world, rank, dev, comm)
ex, inputs = run.ex, run.inputs
for _ in range(3):
    ex.run(inputs)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
tl = ex.timeline(inputs, graph=os.environ.get("GRAPH") == "1")
if rank == 0:
    comp = sorted([t for t in tl if t["stream"] == "compute"], key=lambda t: t["start_ms"])
    busy = sum(t["end_ms"] - t["start_ms"] for t in comp)
    end = max(t["end_ms"] for t in tl)
    for t in sorted(tl, key=lambda t: t["start_ms"]):
        print("%-8s %-20s %-22s %8.3f %8.3f  %7.3f" % (t["stream"], t["id"], t["op"],
                                                     t["start_ms"], t["end_ms"],
                                                     t["end_ms"] - t["start_ms"]))
    print("total %.3f ms, compute busy %.3f ms" % (end, busy))
if world > 1 and os.environ.get("ALL_RANKS") == "1":
    # every rank's first steps (start-of-step skew between ranks)
    head = [(t["stream"], t["id"], t["start_ms"], t["end_ms"])
            for t in sorted(tl, key=lambda t: t["start_ms"])[:14]]
    heads = [None] * world if rank == 0 else None
    dist.gather_object(head, heads, dst=0)
    if rank == 0:
        for r, h in enumerate(heads):
            print(f"rank {r}: " + "  ".join(f"{i}@{a:.3f}-{b:.3f}" for st, i, a, b in h
                                            if not i.startswith(("parameter", "constant"))))
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
