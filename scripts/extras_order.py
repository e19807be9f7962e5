"""Does a config's step time depend on what ran before it in the same
process (shared communicator / peer heap)?  Times the configs named on the
command line in that order with bench.py's harness.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/extras_order.py c3 c2 c3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import NcclComm  # noqa: E402

rank, world, local = B._dist_env()
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = NcclComm.from_torch_distributed()


def barrier():
    dist.barrier()


for cfg in sys.argv[1:]:
    # "c2@1x4": the C2 layer on the (1, 4) mesh (bench.py's N=4 alternative)
    name, _, m = cfg.partition("@")
    mesh = tuple(int(v) for v in m.split("x")) if m else None
    run = B._Run(name, world, rank, dev, comm, mesh=mesh)
    torch.cuda.synchronize()
    __import__("time").sleep(float(os.environ.get("SETTLE", "0")))
    ms, *_ = B._time_steps(run, int(os.environ.get("STEPS", "10")), 3, False, barrier, world, dev)
    heap = C.lib().spmd_comm_peer_bytes(comm.handle) if hasattr(C.lib(), "spmd_comm_peer_bytes") \
        else -1
    half = C.lib().spmd_comm_fused_half(comm.handle)
    if rank == 0:
        print(f"{cfg}: {ms:.3f} ms  peer heap {heap / 2**20:.0f} MiB  fused half {half / 2**20:.0f} MiB",
              flush=True)
    del run
    torch.cuda.empty_cache()
dist.barrier()
dist.destroy_process_group()
