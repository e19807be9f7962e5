"""Multi-GPU parity through NCCL (one process per GPU).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/multi_gpu_check.py

For every golden case whose device count equals the world size, each rank
runs the REFERENCE's SPMD program for its own partition id with NCCL
collectives and compares its outputs with the reference evaluator's outputs
for that device (ints exact, f32 1e-5 normwise).  Then the fast plan with
fusions is checked end to end (outputs gathered to rank 0 and assembled).
Prints one summary JSON line on rank 0; exit code 1 on any failure.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import golden_io as G  # noqa: E402
from paper_2105_04663_b200 import partition, propagate  # noqa: E402
from paper_2105_04663_b200.executor import (Executor, NcclComm, download_stacked,  # noqa: E402
                                            upload_stacked)
from paper_2105_04663_b200.partitioner import SpmdProgram  # noqa: E402
from paper_2105_04663_b200.sharding import Sharding, assemble_data, shard_data  # noqa: E402


def close(got, want, is_float, tol=1e-5):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    if got.shape != want.shape:
        return False
    if not is_float:
        return bool(np.array_equal(got, want))
    fin = np.isfinite(want)
    if not np.array_equal(np.isnan(got), np.isnan(want)):
        return False
    if not fin.any():
        return True
    err = np.max(np.abs(got[fin] - want[fin]))
    return err / max(1.0, np.max(np.abs(want[fin]))) <= tol


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = NcclComm.from_torch_distributed()
    results = {}
    cases = [c for kind in G.KINDS for c in G.cases(kind)
             if c.get("num_devices") == world and "spmd" in c]
    for case in cases:
        prog_graph = G.program(case)
        prog = SpmdProgram(prog_graph, world, {}, (), ())
        shardings = [Sharding.parse(s) for s in case["param_shardings"]]
        my_in = []
        for s, x, p in zip(shardings, G.inputs(case), prog_graph.parameters):
            my_in.append(upload_stacked([shard_data(x, s, devices=range(world))[rank]],
                                        p.shape, dev))
        ex = Executor(prog, nparts=1, device=dev, comm=comm, partition_base=rank)
        outs = ex.run(my_in)
        torch.cuda.synchronize()
        want = G.spmd_outputs(case)[rank]
        ok = True
        for oid, o, w in zip(prog_graph.outputs, outs, want):
            got = download_stacked(o, prog_graph.instr(oid).shape)[0]
            ok &= close(got, w, prog_graph.instr(oid).shape.dtype.is_float)
        results["ref:" + case["name"]] = ok
        # fast plan + fusions, assembled on rank 0
        g = G.graph(case)
        ann, _ = propagate(g)
        fprog = partition(ann, world, plan="fast")
        fin = []
        for p_src, x, p in zip(ann.parameters, G.inputs(case), fprog.graph.parameters):
            fin.append(upload_stacked([shard_data(x, p_src.sharding, devices=range(world))[rank]],
                                      p.shape, dev))
        fex = Executor(fprog, nparts=1, device=dev, comm=comm, partition_base=rank, fuse=True)
        fouts = [download_stacked(o, fprog.graph.instr(oid).shape)[0]
                 for o, oid in zip(fex.run(fin), fprog.graph.outputs)]
        gathered = [None] * world
        dist.all_gather_object(gathered, fouts)
        if rank == 0:
            ok = True
            try:
                for i, oid in enumerate(g.outputs):
                    shape = g.instr(oid).shape
                    full = assemble_data({d: gathered[d][i] for d in range(world)},
                                         fprog.output_shardings[i], shape, rtol=1e-4)
                    ok &= close(full, G.expected(case)[i], shape.dtype.is_float, tol=1e-4)
            except Exception as e:   # report, keep going
                print(f"[{case['name']}] {type(e).__name__}: {e}", flush=True)
                ok = False
            results["fast:" + case["name"]] = ok
    torch.cuda.synchronize()
    flags = [None] * world
    dist.all_gather_object(flags, results)
    rc = 0
    if rank == 0:
        merged = {}
        for r in flags:
            for k, v in r.items():
                merged[k] = merged.get(k, True) and v
        failed = sorted(k for k, v in merged.items() if not v)
        print(json.dumps({"world": world, "cases": len(merged), "failed": failed}), flush=True)
        rc = 1 if failed else 0
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
