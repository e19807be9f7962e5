"""Fused dot -> reduce-scatter over peer memory vs spmd_dot + NCCL
reduce-scatter, one process per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/peer_fusion_check.py [--perf]

1. Direct ABI: random bf16 GEMMs, several epochs in a row (parity buffers),
   alternating subgroup partitions (consecutive fused ops over different
   groups), compared with the unfused dot + NCCL reduce-scatter (fp32-accumulated
   sums of bf16 partials: normwise 1e-2).
2. Transformer layer (fast plan, fusions) with and without the peer fusion.
3. --perf: C2 paper-dims step time (CUDA graph replay, max over ranks) with and
   without the peer fusion.
Prints one JSON line per section on rank 0; exit 1 on any failure.
"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2105_04663_b200 import _capi as C  # noqa: E402
from paper_2105_04663_b200 import partition, propagate  # noqa: E402
from paper_2105_04663_b200.executor import Executor, NcclComm, _groups_arg, desc  # noqa: E402
from paper_2105_04663_b200.ir import DType, Shape  # noqa: E402
from paper_2105_04663_b200.sharding import shard_data  # noqa: E402
from paper_2105_04663_b200.workloads import transformer_flops, transformer_layer  # noqa: E402


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / b.abs().max().clamp(min=1.0)).item()


def direct_abi(comm, rank, world, dev):
    """Fused dot -> reduce-scatter vs dot + NCCL reduce-scatter.  The fused
    ops run back to back with NO host sync and alternate sizes and subgroups
    (the training step's pattern): a peer that passed op k's barrier writes
    op k+1's tiles while this rank may still reduce op k, which the fixed
    parity stride (peer.cu fused_parity) must keep apart."""
    lib = C.lib()
    s = torch.cuda.current_stream().cuda_stream
    partitions = [[list(range(world))]]
    if world >= 4:
        partitions.append([[0, 1], [2, 3]] if world == 4 else
                          [list(range(i, i + world // 2)) for i in (0, world // 2)])
        partitions.append([[r for r in range(world) if r % 2 == k] for k in (0, 1)])
    K, N = 768, 1024
    sizes = [512, 2048, 256, 1024, 2048, 512, 256, 1536]
    comm.reserve_fused(max(sizes) * N * 2)
    comm.ensure_peer(3 * max(sizes) * N * 2 + (1 << 20), dev)
    comm.ensure_workspace(4 * max(sizes) * N, dev)
    dd = C.SpmdDotDims()
    dd.n_contract = 1
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 1, 0
    runs = []
    for it, M in enumerate(sizes):
        groups = partitions[it % len(partitions)]
        gs = len(groups[0])
        garr, ng, gsz = _groups_arg(groups)
        g = torch.Generator(device=dev).manual_seed(1000 * it + rank)
        a = torch.randn((1, M, K), device=dev, generator=g).bfloat16()
        b = (torch.randn((1, K, N), device=dev, generator=g) * 0.05).bfloat16()
        ash, bsh = Shape((M, K), DType.BF16), Shape((K, N), DType.BF16)
        osh = Shape((M, N // gs), DType.BF16)
        fused = torch.empty((1, M, N // gs), device=dev, dtype=torch.bfloat16)
        C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(a, ash), desc(b, bsh),
                                            desc(fused, osh), ctypes.byref(dd), 1, garr, ng, gsz,
                                            s), "dot_reduce_scatter")
        runs.append((a, b, ash, bsh, osh, fused, garr, ng, gsz, M))
    errs = []
    for a, b, ash, bsh, osh, fused, garr, ng, gsz, M in runs:
        full = torch.empty((1, M, N), device=dev, dtype=torch.bfloat16)
        C.check(lib.spmd_dot(desc(a, ash), desc(b, bsh), desc(full, Shape((M, N), DType.BF16)),
                             ctypes.byref(dd), 1, s), "dot")
        ref = torch.empty_like(fused)
        C.check(lib.spmd_reduce_scatter(comm.handle, desc(full, Shape((M, N), DType.BF16)),
                                        desc(ref, osh), 1, 0, garr, ng, gsz, s), "rs")
        torch.cuda.synchronize()
        C.check(lib.spmd_check_device_errors(s), "device")
        errs.append(rel(fused, ref))
    return errs


def direct_abi_rows(comm, rank, world, dev):
    """Row-split reduce-scatter (weight-gradient shape dW[M,N,D] = x^T.dy
    split on M) vs dot + NCCL reduce-scatter on dim 0."""
    lib = C.lib()
    s = torch.cuda.current_stream().cuda_stream
    T, M, N, D = 512, 256 * world, 8, 128
    garr, ng, gsz = _groups_arg([list(range(world))])
    dd = C.SpmdDotDims()
    dd.n_contract = 1
    dd.lhs_contracting[0], dd.rhs_contracting[0] = 0, 0
    errs = []
    comm.reserve_fused(M * N * D * 2)
    comm.ensure_peer(3 * M * N * D * 2 + (1 << 20), dev)
    for it in range(3):
        g = torch.Generator(device=dev).manual_seed(77 * it + rank)
        a = torch.randn((1, T, M), device=dev, generator=g).bfloat16()
        b = (torch.randn((1, T, N, D), device=dev, generator=g) * 0.05).bfloat16()
        ash, bsh = Shape((T, M), DType.BF16), Shape((T, N, D), DType.BF16)
        osh = Shape((M // world, N, D), DType.BF16)
        fused = torch.empty((1, M // world, N, D), device=dev, dtype=torch.bfloat16)
        C.check(lib.spmd_dot_reduce_scatter(comm.handle, desc(a, ash), desc(b, bsh),
                                            desc(fused, osh), ctypes.byref(dd), 0, garr, ng, gsz,
                                            s), "dot_rs_rows")
        full = torch.empty((1, M, N, D), device=dev, dtype=torch.bfloat16)
        C.check(lib.spmd_dot(desc(a, ash), desc(b, bsh), desc(full, Shape((M, N, D), DType.BF16)),
                             ctypes.byref(dd), 1, s), "dot")
        ref = torch.empty_like(fused)
        comm.ensure_workspace(4 * M * N * D, dev)
        C.check(lib.spmd_reduce_scatter(comm.handle, desc(full, Shape((M, N, D), DType.BF16)),
                                        desc(ref, osh), 0, 0, garr, ng, gsz, s), "rs")
        torch.cuda.synchronize()
        C.check(lib.spmd_check_device_errors(s), "device")
        errs.append(rel(fused, ref))
    return errs


def layer(comm, rank, world, dev, mesh, dims, fused_rs, env=None):
    os.environ["SPMD_PEER_FUSION"] = "1" if fused_rs else "0"
    for k in ("SPMD_PEER_AG", "SPMD_PEER_AG_ENGINE"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    big = dims["M"] >= 4096
    g, ins = transformer_layer(mesh, dtype=DType.BF16, with_inputs=not big, **dims)
    ann, _ = propagate(g)
    prog = partition(ann, world, plan="fast")
    stacked = []
    gen = torch.Generator(device=dev).manual_seed(rank)
    for k, p in enumerate(prog.graph.parameters):
        if big:   # synthetic shard of the paper-dims layer, made on the device
            t = torch.randn((1,) + p.shape.dims, device=dev, generator=gen) * 0.02
        else:
            piece = shard_data(ins[k], ann.parameters[k].sharding, devices=range(world))[rank]
            t = torch.from_numpy(np.ascontiguousarray(piece, dtype=np.float32)).to(dev)
        stacked.append(t.to(torch.bfloat16).reshape((1,) + p.shape.dims))
    ex = Executor(prog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True)
    n_rs = sum(1 for v in ex._fused.values() if v[0] in ("dot_rs", "dot_rs_add"))
    return ex, stacked, n_rs


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = NcclComm.from_torch_distributed()
    failed = []

    errs = direct_abi(comm, rank, world, dev) + direct_abi_rows(comm, rank, world, dev)
    allerrs = [None] * world
    dist.all_gather_object(allerrs, errs)
    worst = max(max(e) for e in allerrs)
    if rank == 0:
        print(json.dumps({"section": "direct_abi", "world": world, "max_rel": worst}), flush=True)
    if not worst < 1e-2:
        failed.append("direct_abi")

    mesh = (1, world) if world <= 2 else (2, world // 2)
    small = dict(B=4, S=256, M=1024, N=8, D=64, H=4096)
    meshes = [mesh] + ([(1, world)] if world > 2 else [])
    for lm in meshes:
        for eng in ("auto", "ce", "sm"):
            ex1, x1, n1 = layer(comm, rank, world, dev, lm, small, True,
                                {"SPMD_PEER_AG_ENGINE": eng})
            ex0, x0, n0 = layer(comm, rank, world, dev, lm, small, False, {"SPMD_PEER_AG": "0"})
            a = ex1.run(x1)[0]
            b = ex0.run(x0)[0]
            torch.cuda.synchronize()
            e = rel(a, b)
            es = [None] * world
            dist.all_gather_object(es, e)
            if rank == 0:
                print(json.dumps({"section": "layer_small", "mesh": lm, "engine": eng,
                                  "fused_dot_rs": n1, "unfused_dot_rs": n0,
                                  "peer_all_gathers": sum(1 for v in ex1._peer_engine.values()
                                                          if v >= 0),
                                  "max_rel": max(es)}), flush=True)
            if not (max(es) < 2e-2 and n1 > 0 and n0 == 0):
                failed.append(f"layer_small{lm}:{eng}")
            del ex1, ex0, x1, x0

    # residual Add inside the reduce-scatter's slot reduce (dot_rs_add) vs
    # the reduce-scatter then the Add: same roundings, so bit-identical
    for lm in meshes:
        ex1, x1, n1 = layer(comm, rank, world, dev, lm, small, True, {"SPMD_RS_ADD": "1"})
        ex0, x0, _ = layer(comm, rank, world, dev, lm, small, True, {"SPMD_RS_ADD": "0"})
        n_add = sum(1 for v in ex1._fused.values() if v[0] == "dot_rs_add")
        a = ex1.run(x1)[0]
        b = ex0.run(x0)[0]
        torch.cuda.synchronize()
        same = bool(torch.equal(a, b))
        alls = [None] * world
        dist.all_gather_object(alls, same)
        if rank == 0:
            print(json.dumps({"section": "rs_add_bitwise", "mesh": lm, "dot_rs_add": n_add,
                              "bit_identical_all_ranks": all(alls)}), flush=True)
        if not (all(alls) and n_add == 2):
            failed.append(f"rs_add_bitwise{lm}")
        os.environ.pop("SPMD_RS_ADD", None)
        del ex1, ex0, x1, x0

    # training step (forward + backward): all weight-gradient reduce-scatters
    # fused (row and column splits) vs NCCL
    from paper_2105_04663_b200.workloads import train_step_inputs, transformer_train_step
    tdims = dict(B=4, S=256, M=1024, N=8, D=64, H=2048)
    res = {}
    for fusedflag in (True, False):
        os.environ["SPMD_PEER_FUSION"] = "1" if fusedflag else "0"
        tg = transformer_train_step(mesh, dtype=DType.BF16, **tdims)
        tann, _ = propagate(tg)
        tprog = partition(tann, world, plan="fast")
        tins = train_step_inputs(**tdims, seed=5)
        txs = []
        for k, p in enumerate(tprog.graph.parameters):
            piece = shard_data(tins[k], tann.parameters[k].sharding, devices=range(world))[rank]
            t = torch.from_numpy(np.ascontiguousarray(piece, dtype=np.float32)).to(dev)
            txs.append(t.to(torch.bfloat16).reshape((1,) + p.shape.dims))
        tex = Executor(tprog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True)
        n_fused = sum(1 for v in tex._fused.values() if v[0] in ("dot_rs", "dot_rs_add"))
        res[fusedflag] = ([o.float() for o in tex.run(txs)], n_fused)
    torch.cuda.synchronize()
    terr = max(rel(a, b) for a, b in zip(res[True][0], res[False][0]))
    tall = [None] * world
    dist.all_gather_object(tall, terr)
    if rank == 0:
        print(json.dumps({"section": "train_step", "mesh": mesh, "fused_dot_rs": res[True][1],
                          "unfused": res[False][1], "max_rel": max(tall)}), flush=True)
    if not (max(tall) < 2e-2 and res[True][1] >= 6 and res[False][1] == 0):
        failed.append("train_step")
    os.environ.pop("SPMD_PEER_FUSION", None)

    # MoE layer: expert FFN-out einsum + combine all-to-all fused over peer
    # memory (and the dense dispatch einsum + all-to-all) vs NCCL
    from paper_2105_04663_b200.workloads import moe_layer
    outs = {}
    for fused in (True, False):
        os.environ["SPMD_PEER_FUSION"] = "1" if fused else "0"
        g, ins = moe_layer(world, E=8, B=8, S=64, C=64, M=512, H=1024, dtype=DType.BF16)
        ann, _ = propagate(g)
        prog = partition(ann, world, plan="fast")
        xs = []
        for k, p in enumerate(prog.graph.parameters):
            piece = shard_data(ins[k], ann.parameters[k].sharding, devices=range(world))[rank]
            t = torch.from_numpy(np.ascontiguousarray(piece, dtype=np.float32)).to(dev)
            xs.append(t.to(torch.bfloat16).reshape((1,) + p.shape.dims))
        ex = Executor(prog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True)
        n_a2a = sum(1 for v in ex._fused.values() if v[0] == "dot_a2a")
        outs[fused] = (ex.run(xs)[0], n_a2a)
    torch.cuda.synchronize()
    same = bool(torch.equal(outs[True][0], outs[False][0]))
    flags = [None] * world
    dist.all_gather_object(flags, same)
    if rank == 0:
        print(json.dumps({"section": "moe_dot_a2a", "fused_dot_a2a": outs[True][1],
                          "unfused": outs[False][1], "ranks_equal": flags}), flush=True)
    if not (all(flags) and outs[True][1] > 0 and outs[False][1] == 0):
        failed.append("moe_dot_a2a")
    os.environ.pop("SPMD_PEER_FUSION", None)

    # routed MoE: dispatch pushed straight into the experts' owners' heaps
    # (spmd_moe_dispatch_all_to_all) + fused FFN-out/combine exchange, vs the
    # same routing with NCCL all-to-alls
    from paper_2105_04663_b200.executor import Routing
    E, Bg, S_, Cc, M_, H_ = 8, 8, 64, 32, 512, 1024
    Bl = Bg // world
    st = torch.cuda.current_stream().cuda_stream
    gen = torch.Generator(device=dev).manual_seed(100 + rank)
    logits = torch.randn((1, Bl, S_, E), device=dev, generator=gen)
    ex_t = torch.empty((1, Bl, S_), dtype=torch.int32, device=dev)
    sl_t, gt_t = torch.empty_like(ex_t), torch.empty((1, Bl, S_), dtype=torch.float32, device=dev)
    lib = C.lib()
    f32, s32, bf = DType.F32, DType.S32, DType.BF16
    C.check(lib.spmd_moe_route(desc(logits, Shape((Bl, S_, E), f32)), Cc,
                               desc(ex_t, Shape((Bl, S_), s32)), desc(sl_t, Shape((Bl, S_), s32)),
                               desc(gt_t, Shape((Bl, S_), f32)), 1, st), "route")
    outs = {}
    for fused in (True, False):
        os.environ["SPMD_PEER_FUSION"] = "1" if fused else "0"
        g, ins = moe_layer(world, E=E, B=Bg, S=S_, C=Cc, M=M_, H=H_, dtype=DType.BF16)
        ann, _ = propagate(g)
        prog = partition(ann, world, plan="fast")
        xs = []
        for k, p in enumerate(prog.graph.parameters):
            piece = shard_data(ins[k], ann.parameters[k].sharding, devices=range(world))[rank]
            t = torch.from_numpy(np.ascontiguousarray(piece, dtype=np.float32)).to(dev)
            xs.append(t.to(torch.bfloat16).reshape((1,) + p.shape.dims))
        names = [p.id for p in ann.parameters]
        msh = Shape((Bl, S_, E, Cc), bf)
        C.check(lib.spmd_moe_masks(desc(ex_t, Shape((Bl, S_), s32)), desc(sl_t, Shape((Bl, S_), s32)),
                                   desc(gt_t, Shape((Bl, S_), f32)),
                                   desc(xs[names.index("dispatch")], msh),
                                   desc(xs[names.index("combine")], msh), 1, st), "masks")
        idx = {p.id: p.attrs["index"] for p in ann.parameters}
        r = Routing(ex_t, sl_t, gt_t)
        ex = Executor(prog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True,
                      routing={idx["dispatch"]: r, idx["combine"]: r})
        kinds = sorted(v[0] for v in ex._fused.values())
        outs[fused] = (ex.run(xs)[0], kinds)
    torch.cuda.synchronize()
    same = bool(torch.equal(outs[True][0], outs[False][0]))
    flags = [None] * world
    dist.all_gather_object(flags, same)
    if rank == 0:
        print(json.dumps({"section": "moe_routed", "fused": outs[True][1],
                          "unfused": outs[False][1], "ranks_equal": flags}), flush=True)
    if not (all(flags) and "moe_dispatch_a2a" in outs[True][1]):
        failed.append("moe_routed")
    os.environ.pop("SPMD_PEER_FUSION", None)

    if "--perf" in sys.argv:
        dims = dict(B=16, S=1024, M=8192, N=128, D=256, H=65536)
        flops = transformer_flops(**dims)
        variants = [("peer (auto engines)", True, {}),
                    ("peer, copy engines only", True, {"SPMD_PEER_AG_ENGINE": "ce"}),
                    ("peer, SM pulls only", True, {"SPMD_PEER_AG_ENGINE": "sm"}),
                    ("nccl only", False, {"SPMD_PEER_AG": "0"})]
        for name, fused, env in variants:
            ex, xs, n = layer(comm, rank, world, dev, mesh, dims, fused, env)
            graph, outs = ex.capture(xs)
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
            C.check(C.lib().spmd_check_device_errors(torch.cuda.current_stream().cuda_stream),
                    "device")
            if rank == 0:
                print(json.dumps({"section": "c2_perf", "mesh": mesh, "variant": name,
                                  "fused_dot_rs": n, "ms_per_step": ms.item(),
                                  "tflops_per_gpu": flops / world / ms.item() / 1e9}), flush=True)
            del graph, outs, ex, xs
            torch.cuda.empty_cache()

    flags = [None] * world
    dist.all_gather_object(flags, failed)
    rc = 0
    if rank == 0:
        allf = sorted({f for fl in flags for f in fl})
        print(json.dumps({"world": world, "failed": allf}), flush=True)
        rc = 1 if allf else 0
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
