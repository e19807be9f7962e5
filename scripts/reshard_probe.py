"""C5 reshard at N>1: the executor's all-to-all step vs the raw engine call
(bench.py's `reshard` and `reshard.engines`), each section run twice in one
process to separate order / warm-up effects from the path itself.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/reshard_probe.py
"""
import json
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
dist.init_process_group("nccl", device_id=dev)
comm = NcclComm.from_torch_distributed()
for rep in range(2):
    r = B._reshard(world, rank, dev, comm, dist.barrier)
    if rank == 0:
        print(json.dumps({"rep": rep, **{k: round(v["bus_gbs_per_gpu"], 1) if "bus_gbs_per_gpu" in v
                                         else {e: round(x["bus_gbs_per_gpu"], 1) for e, x in v.items()}
                                         for k, v in r.items()}}), flush=True)
dist.barrier()
dist.destroy_process_group()
