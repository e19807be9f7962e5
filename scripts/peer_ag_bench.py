"""All-gather engines over NVLink: NCCL vs peer heap (copy engine / SM pull).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/peer_ag_bench.py

Times each variant with CUDA events (max over ranks) on leading-dim and
last-dim gathers; prints bus GB/s = out_bytes * (G-1)/G / t (nccl-tests
convention) per line on rank 0.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import NcclComm, _groups_arg, desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = NcclComm.from_torch_distributed()
    lib = C.lib()
    s = torch.cuda.current_stream().cuda_stream
    comm.ensure_peer(512 << 20, dev)
    comm.ensure_workspace(2 << 30, dev)
    partitions = {"all": [list(range(world))]}
    if world == 4:
        partitions["pairs"] = [[0, 1], [2, 3]]
    for pname, groups in partitions.items():
        gs = len(groups[0])
        garr, ng, gsz = _groups_arg(groups)
        for mb in (16, 64, 256):
            rows = 8192
            cols = mb * (1 << 20) // 2 // rows
            for dim in (0, 1):
                ish = Shape((rows, cols), DType.BF16)
                osh = Shape((rows * gs, cols) if dim == 0 else (rows, cols * gs), DType.BF16)
                x = torch.randn((1, rows, cols), device=dev).bfloat16()
                y = torch.empty((1,) + osh.dims, device=dev, dtype=torch.bfloat16)
                variants = {
                    "nccl": lambda: lib.spmd_all_gather(comm.handle, desc(x, ish), desc(y, osh),
                                                        dim, garr, ng, gsz, s),
                    "peer_ce": lambda: lib.spmd_peer_all_gather(comm.handle, desc(x, ish),
                                                                desc(y, osh), dim, garr, ng,
                                                                gsz, 0, 0, 0, s),
                    "peer_sm": lambda: lib.spmd_peer_all_gather(comm.handle, desc(x, ish),
                                                                desc(y, osh), dim, garr, ng,
                                                                gsz, 0, 0, 1, s),
                }
                ref = None
                for name, fn in variants.items():
                    for _ in range(3):
                        C.check(fn(), name)
                    torch.cuda.synchronize()
                    if ref is None:
                        ref = y.clone()
                    else:
                        assert torch.equal(ref, y), name
                    dist.barrier()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(10):
                        C.check(fn(), name)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = torch.tensor([e0.elapsed_time(e1) / 10], device=dev)
                    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
                    if rank == 0:
                        out_b = y.numel() * 2
                        print(json.dumps({"groups": pname, "gsize": gs, "in_mb": mb, "dim": dim,
                                          "engine": name, "ms": round(ms.item(), 4),
                                          "bus_gbs": round(out_b * (gs - 1) / gs / ms.item() / 1e6,
                                                           1)}), flush=True)
                del x, y
    C.check(lib.spmd_check_device_errors(s), "device")
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
