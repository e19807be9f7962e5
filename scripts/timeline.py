"""Per-op timeline of the C2 layer on N GPUs (torchrun), rank 0 prints the
compute/comm stream intervals and the compute-stream idle gaps."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import bench as B
from paper_2105_04663_b200 import partition, propagate
from paper_2105_04663_b200.executor import Executor, NcclComm
rank, world, local = B._dist_env()
torch.cuda.set_device(local); dev = torch.device("cuda", local)
if world > 1: dist.init_process_group("nccl", device_id=dev)
mesh, g, dims, flops, fan, _ = B._workload(os.environ.get("CFG", "c2"), world)
ann, _ = propagate(g); prog = partition(ann, world, plan="fast")
comm = NcclComm.from_torch_distributed() if world > 1 else None
ex = Executor(prog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True)
inputs = [B._rand_like_shard(p.shape, dev, 0.01, 1) for p in prog.graph.parameters]
for _ in range(3): ex.run(inputs)
torch.cuda.synchronize()
if world > 1: dist.barrier()
tl = ex.timeline(inputs)
if rank == 0:
    comp = sorted([t for t in tl if t["stream"] == "compute"], key=lambda t: t["start_ms"])
    busy = sum(t["end_ms"] - t["start_ms"] for t in comp)
    end = max(t["end_ms"] for t in tl)
    for t in sorted(tl, key=lambda t: t["start_ms"]):
        print("%-8s %-20s %-22s %8.3f %8.3f  %7.3f" % (t["stream"], t["id"], t["op"], t["start_ms"], t["end_ms"], t["end_ms"] - t["start_ms"]))
    print("total %.3f ms, compute busy %.3f ms" % (end, busy))
if world > 1: dist.barrier(); dist.destroy_process_group()
