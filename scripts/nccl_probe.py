"""Probe the NCCL collective path (C ABI) with permuted / split subgroups.

    torchrun --nproc-per-node 4 scripts/nccl_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import NcclComm, desc, _groups_arg  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    comm = NcclComm.from_torch_distributed()
    comm.ensure_workspace(1 << 20, dev)
    lib = C.lib()
    s = torch.cuda.current_stream().cuda_stream
    lines = []
    perms = [tuple(range(world)), tuple([0, 2, 1, 3][:world]) if world == 4 else (1, 0),
             tuple(reversed(range(world)))]
    for groups in [(p,) for p in perms] + ([((0, 1), (2, 3)), ((0, 2), (1, 3))] if world == 4 else []):
        g, ng, gs = _groups_arg(groups)
        x = torch.full((1, 2), float(rank + 1), device=dev)
        y = torch.empty((1, 2 * gs), device=dev)
        C.check(lib.spmd_all_gather(comm.handle, desc(x, Shape((2,), DType.F32)),
                                    desc(y, Shape((2 * gs,), DType.F32)), 0, g, ng, gs, s), "ag")
        z = torch.empty((1, 2), device=dev)
        C.check(lib.spmd_all_reduce(comm.handle, desc(x, Shape((2,), DType.F32)),
                                    desc(z, Shape((2,), DType.F32)), 0, g, ng, gs, s), "ar")
        torch.cuda.synchronize()
        lines.append(f"groups={groups} ag={y[0].tolist()} ar={z[0].tolist()}")
    out = [None] * world
    dist.all_gather_object(out, lines)
    if rank == 0:
        for r, ls in enumerate(out):
            for l in ls:
                print(f"rank{r} {l}")
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
