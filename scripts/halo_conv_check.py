"""Halo-window conv fusion under NCCL (one process per GPU): the C4 conv
stack with the conv reading its halo pieces directly equals the
materialised-window path bit for bit on every rank; then the C4 paper-dims
step time with and without the fusion (CUDA graph replay, max over ranks).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/halo_conv_check.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2105_04663_b200 import partition, propagate  # noqa: E402
from paper_2105_04663_b200.executor import Executor, NcclComm  # noqa: E402
from paper_2105_04663_b200.ir import DType  # noqa: E402
from paper_2105_04663_b200.workloads import conv_stack  # noqa: E402


def build(world, dims, fused, comm, rank, dev):
    os.environ["SPMD_HALO_CONV"] = "1" if fused else "0"
    g, _ = conv_stack((world,), (-1, 0, -1, -1), dtype=DType.BF16, with_inputs=False, **dims)
    prog = partition(propagate(g)[0], world, plan="fast")
    ex = Executor(prog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True)
    xs = [B._rand_like_shard(p.shape, dev, 0.05, 7 + k) for k, p in enumerate(prog.graph.parameters)]
    return ex, xs


def main():
    rank, world, local = B._dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = NcclComm.from_torch_distributed()
    small = dict(N=2, H=32 * world, W=256, C=128, layers=3)
    (ea, xa), (eb, xb) = (build(world, small, f, comm, rank, dev) for f in (True, False))
    same = bool(torch.equal(ea.run(xa)[0], eb.run(xb)[0]))
    flags = [None] * world
    dist.all_gather_object(flags, same)
    if rank == 0:
        print(json.dumps({"section": "equal", "world": world, "ranks_equal": flags}), flush=True)
    for fused in (True, False):
        ex, xs = build(world, dict(B.C4), fused, comm, rank, dev)
        graph, _ = ex.capture(xs)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / 10], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"section": "c4_perf", "world": world, "halo_conv": fused,
                              "ms_per_step": ms.item()}), flush=True)
        del graph, ex, xs
        torch.cuda.empty_cache()
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0 if all(flags) else 1


if __name__ == "__main__":
    sys.exit(main())
