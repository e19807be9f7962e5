"""The N>1 host path on CPU with real processes (gloo, world_size 2, 4 and 8).

Each rank does what a GPU rank does in bench.py / scripts/multi_gpu_check.py:
partitions the same annotated graph (both planners), takes partition id =
rank, builds its own parameter shards, executes its per-device program
(local ops with the CPU oracle -- test infrastructure -- and every
collective as a real inter-process exchange over gloo, group/pair order as
emitted), then the outputs are gathered and assembled on rank 0 and compared
with the reference's recorded single-device results.  This pins the
cross-process consistency of partitioning, subgroup ordering, the
partition-id convention and per-rank input sharding / output assembly.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

# C5 (uneven dims over 2 / 4 shards): every reshard kind crosses the process
# boundary, including the fast plan's padded all-to-all for 1001 / 999
C5W_2 = ["c5w2_%s_%s" % (k, d) for k in ("a2a", "repl", "reduce_max", "reduce_sum")
         for d in ("1000x16", "1001x16", "999x16", "16x1001")]
C5W_4 = [n.replace("c5w2", "c5w4") for n in C5W_2]
CASES_2 = ["priority_fig4", "acc5_reshape", "shift_8_1_0_2", "c2_1x2", "c3_moe_2",
           "c4_conv_2"] + C5W_2
CASES_4 = ["c1_8x16x32x24", "ffw_final", "ffw_attempt", "acc7_moe", "c3_moe_4", "c4_conv_4",
           "acc5_pad", "acc5_reverse", "acc5_slice", "rotate_8_3_4", "c2_2x2", "rand25",
           "rand110"] + C5W_4
# the 8-device configs the scaling run's N=8 executes (C2 2x4 / 4x2 / 1x8,
# C3 8 experts, C4 8 shards and 2x4, C5 over 8, the C2 training step)
CASES_8 = ["c2_2x4", "c2_4x2", "c2_1x8", "c3_moe_8", "c4_conv_8", "c4_conv_2x4",
           "c5_a2a_1001x16", "c5_repl_999x16", "c5_reduce_sum_16x1001", "c2_train_2x4",
           "pipe_gpipe_L8_M8_add", "rand13"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, names, q):
    try:
        _work(rank, world, port, names, q)
    except Exception as e:          # never leave the parent waiting
        q.put([f"rank {rank}: {type(e).__name__}: {e}"])
        raise


def _work(rank, world, port, names, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist
    import golden_io as G
    from oracle import evaluator as O
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.ir import COLLECTIVES, Op
    from paper_2105_04663_b200.sharding import assemble_data, shard_data
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    failures = []
    for name in names:
        case = G.case_by_name(name)
        assert case["num_devices"] == world
        g = G.graph(case)
        ann, _ = propagate(g)
        for plan in ("reference", "fast"):
            prog = partition(ann, world, plan=plan)
            env = {}
            for p_src, x, p in zip(ann.parameters, G.inputs(case), prog.graph.parameters):
                env[p.id] = O.cast(shard_data(x, p_src.sharding, devices=range(world))[rank],
                                   p.shape)
            for ins in prog.graph.instructions:
                if ins.opcode == Op.PARAMETER:
                    continue
                if ins.opcode in COLLECTIVES:
                    mine = env[ins.operands[0]]
                    allv = [None] * world
                    dist.all_gather_object(allv, mine)
                    res = O.collective(ins, dict(enumerate(allv)), list(range(world)))
                    env[ins.id] = O.cast(res[rank], ins.shape)
                else:
                    env[ins.id] = O.cast(O.eval_instruction(
                        ins, [env[o] for o in ins.operands], partition_id=rank), ins.shape)
            outs = [env[o] for o in prog.graph.outputs]
            gathered = [None] * world
            dist.all_gather_object(gathered, outs)
            if rank == 0:
                for i, oid in enumerate(g.outputs):
                    shape = g.instr(oid).shape
                    full = assemble_data({d: gathered[d][i] for d in range(world)},
                                         prog.output_shardings[i], shape, rtol=1e-4)
                    want = G.expected(case)[i]
                    if shape.dtype.is_float:
                        _, rel = O.rel_error(full, want)
                        ok = not rel > 1e-4
                    else:
                        ok = np.array_equal(full, want)
                    if not ok:
                        failures.append(f"{name}/{plan}/{oid}")
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(failures)


@pytest.mark.parametrize("world,names", [(2, CASES_2), (4, CASES_4), (8, CASES_8)])
def test_multiprocess_partitioned_execution(world, names):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, q)) for r in range(world)]
    for p in procs:
        p.start()
    failures = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert failures == []
