"""Push all-gather time vs piece size (fixed cost vs bandwidth): pieces of
[rows, cols] bf16 gathered over pairs of ranks along dim 0 (contiguous
pieces, like a weight gather) and along dim 1 (strided rows, like C2's x
gather), each call = push kernel + peer barrier, max over ranks.

    torchrun --nproc-per-node 2|4 --master-addr 127.0.0.1 scripts/push_size_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200.executor import NcclComm, _groups_arg, desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402

rank, world, local = B._dist_env()
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = NcclComm.from_torch_distributed()
lib = C.lib()
s = torch.cuda.current_stream(dev).cuda_stream
groups, ng, gs = _groups_arg([list(range(g, g + 2)) for g in range(0, world, 2)])
off = 3 * int(lib.spmd_comm_fused_half(comm.handle)) + 4096
comm.ensure_peer(off + (1 << 31), dev)
for mb in (2, 8, 33.5, 134, 536):
    rows = int(mb * 2**20 / 2 / 4096)
    x = torch.randn((1, rows, 4096), device=dev).to(torch.bfloat16)
    res = {"piece_MB": mb}
    for dim in (0, 1):
        osh = Shape((rows * 2, 4096) if dim == 0 else (rows, 8192), DType.BF16)
        zone = desc(torch.empty(0, device=dev), osh)
        zone.data = None
        def fn():
            C.check(lib.spmd_peer_push_all_gather(
                comm.handle, desc(x, Shape((rows, 4096), DType.BF16)), zone, dim, groups,
                ng, gs, off, 0, s), "push")
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / 20], device=dev, dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        res[f"dim{dim}_ms"] = round(float(ms), 4)
        res[f"dim{dim}_GBs"] = round(x.numel() * 2 / (float(ms) * 1e-3) / 1e9, 1)
    if rank == 0:
        print(json.dumps(res), flush=True)
    del x
# The C2 step's start on the 2x2 mesh: x over Y pairs and w_q over X pairs
# pushed at once on two streams (33.5 MB pieces), optionally after a 4 GB
# sweep (cold L2 / TLBs as after a step's GEMMs); only the pushes are timed.
if world == 4:
    gy, ngy, gsy = _groups_arg([[0, 1], [2, 3]])
    gx, ngx, gsx = _groups_arg([[0, 2], [1, 3]])
    rows = int(33.5 * 2**20 / 2 / 4096)
    xa = torch.randn((1, rows, 4096), device=dev).to(torch.bfloat16)
    xb = torch.randn((1, rows, 4096), device=dev).to(torch.bfloat16)
    za = desc(torch.empty(0, device=dev), Shape((rows, 8192), DType.BF16))
    zb = desc(torch.empty(0, device=dev), Shape((rows * 2, 4096), DType.BF16))
    za.data = zb.data = None
    off2 = off + rows * 8192 * 2 + (1 << 20)
    sweep = torch.empty(2 * 2**30, dtype=torch.uint8, device=dev)
    sweep2 = torch.empty_like(sweep)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream(dev)
    for cold in (0, 1):
        for both in (0, 1):
            tot = 0.0
            for it in range(12):
                if cold:
                    sweep2.copy_(sweep)
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cur)
                s1.wait_stream(cur)
                s2.wait_stream(cur)
                C.check(lib.spmd_peer_push_all_gather(
                    comm.handle, desc(xa, Shape((rows, 4096), DType.BF16)), za, 1, gy, ngy, gsy,
                    off, 2, s1.cuda_stream), "push y")
                if both:
                    C.check(lib.spmd_peer_push_all_gather(
                        comm.handle, desc(xb, Shape((rows, 4096), DType.BF16)), zb, 0, gx, ngx,
                        gsx, off2, 3, s2.cuda_stream), "push x")
                cur.wait_stream(s1)
                cur.wait_stream(s2)
                e1.record(cur)
                torch.cuda.synchronize()
                if it >= 2:
                    tot += e0.elapsed_time(e1)
            ms = torch.tensor([tot / 10], device=dev, dtype=torch.float64)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"section": "c2_start", "cold": cold, "both": both,
                                  "ms": round(float(ms), 4)}), flush=True)
C.check(lib.spmd_check_device_errors(s), "errors")
dist.barrier()
dist.destroy_process_group()
