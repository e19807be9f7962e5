#!/usr/bin/env python
"""Benchmark: 2-D (data x model) sharded Transformer layer (BASELINE configs[1])
through the B200 partitioned-execution path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (config C2, paper Table-2 dims): M=8192, H=65536,
N=128 heads, D=256, S=1024, global batch B=16, bf16, synthetic random data
generated on the device.  Mesh per GPU count: 1 (1,1), 2 (1,2), 4 (2,2),
8 (2,4) as (X=data, Y=model); annotations per PAPER.md:679.  One step =
one forward pass of the layer: propagate -> partition (fast plan, done once)
-> per-rank executor (tcgen05 GEMMs, fused softmax, NCCL collectives).
Total work is fixed as N grows ("scaling": "strong").

`value` = aggregate layer TFLOP/s over all GPUs (algorithmic FLOPs
2T(3MND+NDM+2MH)+4BNS^2D per step / step time, max over ranks);
`tflops_per_gpu` and `mfu` are the per-GPU views of the same number.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sharded Transformer layer TFLOP/s/GPU & MFU at 1/2/4/8 B200; reshard GB/s"
# (X=data, Y=model): (1,1), (1,2), (2,2) and the
# north-star 2x4.  At N=4 the line also carries the 1x4 mesh under
# configs.c2_mesh_1x4 (no data axis, so no per-step weight gathers).
MESHES = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
if os.environ.get("SPMD_BENCH_MESH"):   # e.g. "1x4": override the (X=data, Y=model) mesh
    _x, _y = (int(v) for v in os.environ["SPMD_BENCH_MESH"].split("x"))
    MESHES[_x * _y] = (_x, _y)
PAPER = dict(B=16, S=1024, M=8192, N=128, D=256, H=65536)
SPEC_BF16_TFLOPS = 2250.0
TF32_SPEC_TFLOPS = 1100.0      # B200_PROFILING.md dense tf32


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("bf16_tflops", 1590.0), p.get("bf16_tflops_sustained", 1400.0), \
            p.get("hbm_gbs", 6650.0), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _cpu_baseline(mesh, steps=1, B=4):
    """Reference executor restated on the CPU (oracle port, single-threaded
    float64 einsum like the reference) on a bounded sample of the C2 graph:
    same annotations/mesh, dims M=1024 N=16 D=64 H=8192 S=256 and B=4
    (BASELINE.md section 4)."""
    import numpy as np
    from oracle import evaluator as O
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.sharding import shard_data
    from paper_2105_04663_b200.workloads import transformer_flops, transformer_layer
    dims = dict(B=max(B, mesh[0]), S=256, M=1024, N=16, D=64, H=8192)
    g, ins = transformer_layer(mesh, dtype=DType.F32, seed=1, **dims)
    ann, _ = propagate(g)
    n = mesh[0] * mesh[1]
    prog = partition(ann, n)
    devices = list(range(n))
    per = {d: [] for d in devices}
    for p, x in zip(ann.parameters, ins):
        sh = shard_data(x, p.sharding, devices=devices)
        for d in devices:
            per[d].append(sh[d])
    best = None
    for _ in range(steps):
        t0 = time.perf_counter()
        O.evaluate_spmd(prog, per)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    flops = transformer_flops(**dims)
    host = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    # the Dot path (np.einsum without optimize = c_einsum, as the reference's
    # simulator.py:268) runs on one thread whatever the host offers
    cores = 1
    sample = ("oracle evaluate_spmd of the C2 layer graph, mesh %s, B=%d S=256 M=1024 N=16 "
              "D=64 H=8192 f32 (%.3g FLOP/step); single-threaded c_einsum Dot like the "
              "reference, host has %d cores" % (mesh, dims["B"], flops, host))
    return flops / best / 1e12, best, cores, sample


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    mesh = MESHES[args.gpus]
    vals = []
    for i in range(args.warmup + args.steps):
        # untimed warm-up steps run the B=1 sample (same graph, imports and
        # caches warmed); every timed step is one B=4 sample (~9 s)
        v, t, cores, sample = _cpu_baseline(mesh, B=1 if i < args.warmup else 4)
        if i >= args.warmup:
            vals.append((v, t))
    v = sorted(x[0] for x in vals)[len(vals) // 2]
    t = sorted(x[1] for x in vals)[len(vals) // 2]
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 transformer layer (attention+FFN), paper dims",
                       "dims": dict(PAPER), "mesh": list(mesh),
                       "parallelism": "dp%dxmp%d" % mesh, "global_batch": PAPER["B"],
                       "seq_len": PAPER["S"],
                       "cpu_sample": "each step times a bounded sample of the workload, "
                                     "see cpu_baseline.sample"},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _rand_like_shard(shape, device, scale, seed, nparts=1):
    import torch
    from paper_2105_04663_b200.executor import torch_dtype
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    t = torch.randn((nparts,) + tuple(shape.dims), generator=gen, device=device,
                    dtype=torch.float32)
    return (t * scale).to(torch_dtype(shape.dtype))


def _traffic_for(top, prog):
    """dram read+write bytes per launch of the top GEMM from the committed ncu
    --set full capture (profiles/*_top_kernel_traffic.json) when the shape
    matches; else None."""
    import glob
    try:
        from paper_2105_04663_b200.ir import Op, dot_dim_lists
        if top.opcode != Op.DOT:
            return None
        a = prog.graph.instr(top.operands[0]).shape
        b = prog.graph.instr(top.operands[1]).shape
        lb, rb, lc, rc, lf, rf = dot_dim_lists(top.attrs, a.rank, b.rank)
        prod = lambda s, ds: int(__import__("math").prod(s.dims[d] for d in ds))
        mnk = [prod(a, lb + lf), prod(b, rf), prod(a, lc)]
        # newest round first
        for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_top_kernel_traffic.json")),
                         reverse=True):
            with open(fn) as f:
                t = json.load(f)
            if list(t["shape_mnk"]) == mnk:
                return t["dram_bytes_read"] + t["dram_bytes_write"]
    except Exception:
        return None
    return None


C1 = dict(B=16, S=1024, M=8192, H=8192)
C3 = dict(E=8, B=64, S=512, C=160, M=4096, H=16384, k=2)
C4 = dict(N=8, H=1024, W=1024, C=128, layers=4)


def _workload(config, world, scale=1.0, mesh=None):
    """(mesh, graph, dims, flops/step, fan-in per parameter, description)."""
    from paper_2105_04663_b200.ir import DType
    from paper_2105_04663_b200.workloads import (conv_stack, moe_layer, transformer_flops,
                                                 transformer_layer)
    if config == "c2":
        mesh = mesh or MESHES[world]
        dims = dict(PAPER)
        if scale != 1.0:
            dims["B"] = max(mesh[0], int(dims["B"] * scale))
        g, _ = transformer_layer(mesh, dtype=DType.BF16, with_inputs=False, **dims)
        fan = {"wq": dims["M"], "wk": dims["M"], "wv": dims["M"], "wo": dims["N"] * dims["D"],
               "wi": dims["M"], "wt": dims["H"]}
        return mesh, g, dims, transformer_flops(**dims), fan, \
            "C2 transformer layer (attention+FFN), paper dims"
    if config == "c2train":
        from paper_2105_04663_b200.workloads import transformer_train_flops, transformer_train_step
        mesh = mesh or MESHES[world]
        dims = dict(PAPER)
        if scale != 1.0:
            dims["B"] = max(mesh[0], int(dims["B"] * scale))
        g = transformer_train_step(mesh, dtype=DType.BF16, **dims)
        fan = {"wq": dims["M"], "wk": dims["M"], "wv": dims["M"], "wo": dims["N"] * dims["D"],
               "wi": dims["M"], "wt": dims["H"], "g": dims["B"] * dims["S"]}
        return mesh, g, dims, transformer_train_flops(**dims), fan, \
            "C2 training step (forward + backward layer, weight gradients reduce-scattered), " \
            "paper dims"
    if config == "c1":
        from paper_2105_04663_b200.workloads import einsum_c1
        d = dict(C1)
        g, _ = einsum_c1((2, 2), dtype=DType.F32, with_inputs=False, **d)
        flops = 2.0 * d["B"] * d["S"] * d["M"] * d["H"]
        return (2, 2), g, d, flops, {"w": d["M"]}, \
            "C1 2-D sharded einsum BSM,MH->BSH f32 (3xTF32 tensor cores), 2x2 mesh"
    if config == "c3":
        d = dict(C3)
        g, _ = moe_layer(world, dtype=DType.BF16, with_inputs=False,
                         **{k: v for k, v in d.items() if k != "k"})
        flops = 4.0 * d["E"] * d["B"] * d["C"] * d["M"] * d["H"]
        return (world,), g, d, flops, {"wi": d["M"], "wo": d["H"]}, \
            "C3 GShard MoE FFN (top-2 routing, capacity C=160 = 1.25*2*S/E), expert GEMM FLOPs"
    if config == "c4":
        d = dict(C4)
        g, _ = conv_stack((world,), (-1, 0, -1, -1), dtype=DType.BF16, with_inputs=False, **d)
        flops = d["layers"] * 2.0 * d["N"] * d["H"] * d["W"] * d["C"] * d["C"] * 9
        return (world,), g, d, flops, {f"w{i}": 9 * d["C"] for i in range(d["layers"])}, \
            "C4 spatially partitioned 3x3 conv stack (NHWC, H-sharded, halo via collective-permute)"
    raise SystemExit(f"unknown config {config}")


def _moe_masks(inputs, names, dims, dev, seed, k=2):
    """Replace the dispatch/combine parameters with real GShard top-k
    routings of random gating logits (on-device router, then dense masks)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    di, ci = names.index("dispatch"), names.index("combine")
    Bl, S, E, Cap = inputs[di].shape[1:]
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    logits = torch.randn((1, Bl, S, E), generator=gen, device=dev)
    ex = torch.empty((1, Bl, S, k), dtype=torch.int32, device=dev)
    sl = torch.empty_like(ex)
    gt = torch.empty((1, Bl, S, k), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    lib = C.lib()
    rsh = lambda dt: Shape((Bl, S, k), dt)
    C.check(lib.spmd_moe_route(desc(logits, Shape((Bl, S, E), DType.F32)), Cap,
                               desc(ex, rsh(DType.S32)), desc(sl, rsh(DType.S32)),
                               desc(gt, rsh(DType.F32)), 1, st), "route")
    msh = Shape((Bl, S, E, Cap), DType.BF16)
    C.check(lib.spmd_moe_masks(desc(ex, rsh(DType.S32)), desc(sl, rsh(DType.S32)),
                               desc(gt, rsh(DType.F32)), desc(inputs[di], msh),
                               desc(inputs[ci], msh), 1, st), "masks")
    return ex, sl, gt


class _Run:
    """One workload compiled for this rank: program, executor, inputs."""

    def __init__(self, config, world, rank, dev, comm, mesh=None, scale=1.0, overlap=True):
        import numpy as np
        from paper_2105_04663_b200 import partition, propagate
        from paper_2105_04663_b200.executor import Executor, Routing
        self.config = config
        self.mesh, g, self.dims, self.flops, fan, self.wdesc = _workload(config, world, scale,
                                                                          mesh)
        ann, _ = propagate(g)
        # C1's 2x2 mesh is simulated on one GPU (4 partitions, loopback
        # collectives) unless 4 ranks run it
        parts = self.mesh[0] * self.mesh[1] if config == "c1" else world
        self.nparts = parts // world
        self.prog = partition(ann, parts, plan="fast")
        # Synthetic local shards, generated on the device (weights ~ N(0, 1/fan_in);
        # MoE dispatch/combine masks from the on-device router).
        src_params = {p.attrs["index"]: p.id for p in ann.parameters}
        self.inputs = []
        for p in self.prog.graph.parameters:
            name = src_params[p.attrs["index"]]
            self.inputs.append(_rand_like_shard(p.shape, dev, 1.0 / np.sqrt(fan.get(name, 1)),
                                                seed=1000 * rank + p.attrs["index"],
                                                nparts=self.nparts))
        self.routing = None
        if config == "c3":
            # On-device GShard top-2 router -> masks (the reference graph's
            # inputs) and the routing itself: the dispatch / combine einsums then
            # run as the gather kernels (equal to the dense Dots).
            names = [src_params[p.attrs["index"]] for p in self.prog.graph.parameters]
            r = Routing(*_moe_masks(self.inputs, names, self.dims, dev, seed=rank,
                                    k=self.dims["k"]))
            idx = {name: p.attrs["index"] for p, name in zip(self.prog.graph.parameters, names)}
            self.routing = {idx["dispatch"]: r, idx["combine"]: r}
        self.ex = Executor(self.prog, nparts=self.nparts, device=dev, comm=comm,
                           partition_base=rank * self.nparts, fuse=True,
                           overlap=(world > 1 and overlap), routing=self.routing)


def _time_steps(run, steps, warmup, eager, barrier, world, dev):
    """W warm-up steps: one eager run (materialises constants, NCCL
    sub-communicators, kernel attributes), capture of the whole step into one
    CUDA graph (compute + comm streams), W-1 warm replays (the first replays
    after another config ran in the process were measured slow: peer-heap
    pages first touched over NVLink); then K timed replays between barriers.
    Eager mode: W eager warm-up runs.  Returns (ms max over ranks, step fn,
    graph, outs, launches/step)."""
    import torch
    import torch.distributed as dist
    ex, inputs = run.ex, run.inputs
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(1, warmup - 1) if eager else 1):
        ex.run(inputs)
    torch.cuda.synchronize()
    ex.check_errors()
    barrier()
    if eager:
        graph = outs = None
        launches = None

        def step():
            return ex.run(inputs)
    else:
        graph, outs = ex.capture(inputs)
        launches = ex.launches_per_replay

        def step():
            graph.replay()
            return outs
    for _ in range(1 if eager else max(1, warmup - 1)):
        step()
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ex.check_errors()      # a peer barrier that timed out inside the replays
    t = torch.tensor([ev0.elapsed_time(ev1) / steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), step, graph, outs, launches


def _dot_flops(prog, ins):
    import numpy as np
    from paper_2105_04663_b200.ir import Op, dot_dim_lists
    a = prog.graph.instr(ins.operands[0]).shape
    bsh = prog.graph.instr(ins.operands[1]).shape
    if ins.opcode == Op.CONVOLUTION:
        cd = ins.attrs["conv_dims"]
        k = a.dims[cd.lhs_feature] * int(np.prod([bsh.dims[d] for d in cd.rhs_spatial]))
        return 2.0 * ins.shape.num_elements * k
    lb, rb, lc, rc, lf, rf = dot_dim_lists(ins.attrs, a.rank, bsh.rank)
    k = int(np.prod([a.dims[d] for d in lc]))
    return 2.0 * ins.shape.num_elements * k


def _top_kernel(run, dev, burst, sustained, peak_src, reps=20):
    """The dominant tensor-core kernel of the step (the largest Dot / Conv by
    FLOPs), launched alone `reps` times on the stream the executor uses,
    timed with CUDA events: the roofline entry of the JSON line."""
    import torch
    from paper_2105_04663_b200.ir import DType, Op
    prog, ex = run.prog, run.ex
    stream = torch.cuda.current_stream(dev)
    dots = [i for i in prog.graph.instructions if i.opcode in (Op.DOT, Op.CONVOLUTION)]
    top = max(dots, key=lambda i: _dot_flops(prog, i))
    kname = "conv_bf16_tcgen05" if top.opcode == Op.CONVOLUTION else "gemm_bf16_tcgen05"
    top_step = next(s for s in ex.steps if s.ins.id == top.id or
                    (ex._fused.get(s.ins.id) or (None, None))[1] is top)
    env = {"__inputs__": run.inputs}
    keep = set(top_step.ops)
    ex.run(run.inputs, keep=keep)
    env.update({k: v for k, v in ex.last_env.items() if k in keep})
    for _ in range(3):
        top_step.fn(env, stream.cuda_stream)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(reps):
        top_step.fn(env, stream.cuda_stream)
    k1.record(stream)
    torch.cuda.synchronize()
    kms = k0.elapsed_time(k1) / reps
    fl = _dot_flops(prog, top) * run.nparts
    achieved = fl / (kms * 1e-3) / 1e12
    if top.shape.dtype == DType.F32:
        # 3xTF32: three tf32 MMAs per f32 product.  MEASURED_PEAKS.json has no
        # tf32 number, so the tf32 peak is measured here: cuBLAS TF32 on 8192^3
        # (burst, best of 10), divided by 3; the spec (1.1 PF/s dense) also given
        tf32 = _cublas_tf32_tflops(dev)
        peak = tf32 / 3.0
        return {"bound": "tensor", "kernel": "gemm_f32_3xtf32_2sm (%s)" % top.id,
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s (f32 products)",
                "frac": achieved / peak, "frac_vs_spec": achieved / (TF32_SPEC_TFLOPS / 3.0),
                "peak_source": "cuBLAS TF32 8192^3 measured in this run (%.0f TF/s) / 3 MMAs "
                               "per f32 product" % tf32,
                "ms_per_launch": kms, "flops_per_launch": fl}
    return {"bound": "tensor", "kernel": "%s (%s)" % (kname, top.id), "achieved": achieved,
            "peak": burst, "unit": "TFLOP/s", "frac": achieved / burst,
            "peak_source": peak_src + " burst (kernel timed alone)",
            "frac_sustained": achieved / sustained, "traffic": _traffic_for(top, prog),
            "ms_per_launch": kms, "flops_per_launch": fl}


def _cublas_tf32_tflops(dev, n=8192, reps=10):
    """Dense TF32 rate of cuBLAS on this box (burst): the measured tf32 peak."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn((n, n), device=dev)
        b = torch.randn((n, n), device=dev)
        c = torch.empty((n, n), device=dev)
        best = None
        for _ in range(3):
            torch.matmul(a, b, out=c)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            best = ms if best is None else min(best, ms)
        del a, b, c
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def _extra_config(config, world, rank, dev, comm, barrier, steps, warmup, burst, sustained,
                  peak_src):
    """A compact summary of another BASELINE config, same harness: step time
    (CUDA-graph replay, max over ranks), TFLOP/s, MFU and the roofline of its
    dominant kernel."""
    import torch
    run = _Run(config, world, rank, dev, comm)
    # let the power controller recover from the previous config: right after
    # the C2 layer the first C3 replays ran ~20% slow at N=4 (clock transient
    # under the power cap; a 1 s pause removes it, scripts/extras_order.py)
    torch.cuda.synchronize()
    time.sleep(1.0)
    ms, _, graph, outs, launches = _time_steps(run, steps, warmup, False, barrier, world, dev)
    tf = run.flops / (ms * 1e-3) / 1e12
    roof = _top_kernel(run, dev, burst, sustained, peak_src, reps=10)
    out = {"workload": run.wdesc, "dims": run.dims, "mesh": list(run.mesh), "ms_per_step": ms,
           "tflops": tf, "tflops_per_gpu": tf / world, "gpu_launches_per_step": launches,
           "roofline": {k: roof[k] for k in ("kernel", "achieved", "peak", "unit", "frac",
                                             "frac_sustained", "frac_vs_spec", "ms_per_launch",
                                             "peak_source")
                        if k in roof}}
    if config == "c1":
        out["dtype"] = "f32 (3xTF32 split on tcgen05 kind::tf32)"
        if run.nparts > 1:
            out["mesh_simulated_on_one_gpu"] = True
    else:
        out["mfu_vs_spec_2250"] = tf / world / SPEC_BF16_TFLOPS
    del run, graph, outs
    torch.cuda.empty_cache()
    return out


def _c5_hbm(dev, hbm, peak_src):
    """C5's HBM-bound kernels at the 8-way uneven layout ([1001, D1] over 8
    shards of ceil(1001/8) = 126 rows): the localize pad 1001 -> 1008 rows
    (partitioner.py:379-408), the dynamic-slice of one shard out of it, and
    the select_range mask of the last shard (partitioner.py:236-247) -- for
    f32 and bf16 at D1 = 524288 and f32 at D1 = 65536.
    Achieved = bytes read + written / kernel time (CUDA events, 10 launches)."""
    import torch
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib, st = C.lib(), torch.cuda.current_stream(dev).cuda_stream
    s32 = DType.S32
    rows = 126
    sc = Shape((), s32)

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    res = {}
    for D1, dt in ((524288, DType.F32), (524288, DType.BF16), (65536, DType.F32)):
        tdt = torch.float32 if dt == DType.F32 else torch.bfloat16
        es = 4 if dt == DType.F32 else 2
        tag = "%dx%d_%s" % (rows, D1, dt.value)
        x = torch.randn((1, 1001, D1), device=dev).to(tdt)
        y = torch.empty((1, 1008, D1), device=dev, dtype=tdt)
        z = torch.zeros((1,), device=dev, dtype=tdt)
        lo, hi, it = C.i64_array([0, 0]), C.i64_array([7, 0]), C.i64_array([0, 0])
        ms = timed(lambda: C.check(lib.spmd_pad(desc(x, Shape((1001, D1), dt)),
                                                desc(z, Shape((), dt)),
                                                desc(y, Shape((1008, D1), dt)), lo, hi, it, 1,
                                                st), "pad"))
        res["pad_1001_to_1008x%d_%s" % (D1, dt.value)] = (ms, (x.numel() + y.numel()) * es)
        s0 = torch.full((1,), rows * 7, dtype=torch.int32, device=dev)
        s1 = torch.zeros((1,), dtype=torch.int32, device=dev)
        y2 = torch.empty((1, rows, D1), device=dev, dtype=tdt)
        starts = (C.SpmdTensor * 2)(desc(s0, sc), desc(s1, sc))
        ms = timed(lambda: C.check(lib.spmd_dynamic_slice(desc(y, Shape((1008, D1), dt)), starts,
                                                          desc(y2, Shape((rows, D1), dt)), 1,
                                                          st), "dynamic_slice"))
        res["dynamic_slice_1008_to_" + tag] = (ms, 2 * y2.numel() * es)
        off = torch.full((1,), 7 * rows, dtype=torch.int32, device=dev)
        fill = torch.full((1,), float("-inf"), device=dev, dtype=tdt)
        y3 = torch.empty_like(y2)
        ms = timed(lambda: C.check(lib.spmd_mask_range(
            desc(y2, Shape((rows, D1), dt)), desc(off, sc), desc(fill, Shape((), dt)),
            desc(y3, Shape((rows, D1), dt)), 0, 0, 1001, 0, 1, st), "mask_range"))
        res["mask_range_" + tag] = (ms, 2 * y2.numel() * es)
        del x, y, y2, y3
        torch.cuda.empty_cache()
    return {"bound": "hbm", "peak_gbs": hbm, "peak_source": peak_src + " copy bandwidth",
            "kernels": {k: {"ms": ms, "bytes": b, "gbs": b / (ms * 1e-3) / 1e9,
                            "frac": b / (ms * 1e-3) / 1e9 / hbm} for k, (ms, b) in res.items()}}


def _reshard(world, rank, dev, comm, barrier):
    """C5 reshard GB/s at N > 1: [n0, 524288] f32 dim-0 -> dim-1 (all-to-all,
    padded for 1001) and -> replicated (all-gather), nccl-tests bus bytes."""
    import torch
    import torch.distributed as dist
    from paper_2105_04663_b200 import partition, propagate
    from paper_2105_04663_b200.executor import Executor
    from paper_2105_04663_b200.ir import DType, Op
    from paper_2105_04663_b200.workloads import uneven
    stream = torch.cuda.current_stream(dev)
    reshard = {}
    D1 = 65536 * 8
    for n0, kind in ((1000, "a2a"), (1001, "a2a"), (1001, "repl")):
        gg, _ = uneven(n0=n0, n1=D1, kind=kind, parts=world, dtype=DType.F32, with_inputs=False)
        ga, _ = propagate(gg)
        rp = partition(ga, world, plan="fast")
        rex = Executor(rp, nparts=1, device=dev, comm=comm, partition_base=rank, overlap=False)
        rin = [torch.randn((1,) + rp.graph.parameters[0].shape.dims, device=dev)]
        coll = next(s for s in rex.steps if s.coll)
        keep = set(coll.ops)
        rex.run(rin, keep=keep)
        renv = {"__inputs__": rin}
        renv.update({k: v for k, v in rex.last_env.items() if k in keep})
        for _ in range(3):
            coll.fn(renv, stream.cuda_stream)
        torch.cuda.synchronize()
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(10):
            coll.fn(renv, stream.cuda_stream)
        r1.record(stream)
        torch.cuda.synchronize()
        rms = torch.tensor([r0.elapsed_time(r1) / 10], device=dev, dtype=torch.float64)
        dist.all_reduce(rms, op=dist.ReduceOp.MAX)
        rms = float(rms.item())
        src = rp.graph.instr(coll.ins.operands[0]).shape
        if coll.ins.opcode == Op.ALL_GATHER:
            bus = coll.ins.shape.nbytes * (world - 1) / world
        else:
            bus = src.nbytes * (world - 1) / world
        reshard[f"{kind}_{n0}x{D1}_f32"] = {
            "collective": coll.ins.opcode.value, "ms": rms,
            "bus_gbs_per_gpu": bus / (rms * 1e-3) / 1e9,
            "frac_of_nvlink_900": bus / (rms * 1e-3) / 1e9 / 900.0}
        del rex, rin, renv
    torch.cuda.empty_cache()
    reshard["engines"] = _reshard_engines(world, dev, comm, barrier)
    return reshard


def _reshard_engines(world, dev, comm, barrier):
    """The same C5 transitions ([1008, 524288] f32, the padded 1001 rows)
    through each engine of the C ABI, bus GB/s per GPU (max over ranks):
    NCCL (pack + ncclAllToAll / ncclAllGather), the peer pull all-gather
    (16-byte NVLink loads) and the push collectives (16-byte NVLink stores
    straight into the members' landing zones, no pack pass)."""
    import torch
    import torch.distributed as dist
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200.executor import _groups_arg, desc
    from paper_2105_04663_b200.ir import DType, Shape
    lib = C.lib()
    s = torch.cuda.current_stream(dev).cuda_stream
    D1, rows = 524288, -(-1008 // world)
    G = world
    groups, ng, gs = _groups_arg([list(range(world))])
    x = torch.randn((1, rows, D1), device=dev)
    ag_out = torch.empty((1, rows * G, D1), device=dev)
    a2a_out = torch.empty((1, rows * G, D1 // G), device=dev)
    xs = desc(x, Shape((rows, D1), DType.F32))
    ag_sh, a2a_sh = Shape((rows * G, D1), DType.F32), Shape((rows * G, D1 // G), DType.F32)
    comm.ensure_workspace(2 * x.numel() * 4 * G, dev)
    off = 3 * int(lib.spmd_comm_fused_half(comm.handle)) + 4096
    comm.ensure_peer(off + ag_out.numel() * 4 + (1 << 20), dev)
    zone_ag = desc(ag_out, ag_sh)
    zone_ag.data = None
    zone_a2a = desc(a2a_out, a2a_sh)
    zone_a2a.data = None
    variants = {
        "all-gather/nccl": lambda: lib.spmd_all_gather(comm.handle, xs, desc(ag_out, ag_sh), 0,
                                                       groups, ng, gs, s),
        "all-gather/peer-pull": lambda: lib.spmd_peer_all_gather(
            comm.handle, xs, desc(ag_out, ag_sh), 0, groups, ng, gs, off, 0, 1, s),
        "all-gather/peer-push": lambda: lib.spmd_peer_push_all_gather(
            comm.handle, xs, zone_ag, 0, groups, ng, gs, off, 0, s),
        "all-to-all/nccl": lambda: lib.spmd_all_to_all(comm.handle, xs, desc(a2a_out, a2a_sh), 1,
                                                       0, groups, ng, gs, s),
        "all-to-all/peer-push": lambda: lib.spmd_peer_all_to_all(
            comm.handle, xs, zone_a2a, 1, 0, groups, ng, gs, off, 0, s),
    }
    out = {}
    for name, fn in variants.items():
        for _ in range(3):
            C.check(fn(), name)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            C.check(fn(), name)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / 10], device=dev, dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms.item())
        bus = (ag_out.numel() if name.startswith("all-gather") else x.numel()) * 4 * (G - 1) / G
        out[name] = {"ms": ms, "bus_gbs_per_gpu": bus / (ms * 1e-3) / 1e9}
    C.check(lib.spmd_check_device_errors(s), "reshard engines")
    del x, ag_out, a2a_out
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c2train", "c3", "c4"])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the other configs' summaries (C3/C4/C5, extra mesh)")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph")
    ap.add_argument("--no-overlap", action="store_true", help="collectives on the compute stream")
    ap.add_argument("--scale", type=float, default=1.0,
                    help="shrink B (testing only; the reported config is the paper's)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2105_04663_b200 import _capi as C
    from paper_2105_04663_b200 import collective_stats
    from paper_2105_04663_b200.executor import NcclComm

    rank, world, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = NcclComm.from_torch_distributed() if world > 1 else None

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    run = _Run(args.config, world, rank, dev, comm, scale=args.scale,
               overlap=not args.no_overlap)
    prog, ex, inputs, flops = run.prog, run.ex, run.inputs, run.flops
    stream = torch.cuda.current_stream(dev)

    sampler = ClockSampler(local)
    sampler.start()
    launches0 = C.lib().spmd_launch_count()
    ms, step, graph, graph_outs, launches_per_step = _time_steps(
        run, args.steps, args.warmup, args.eager, barrier, world, dev)
    launches = C.lib().spmd_launch_count() - launches0
    if launches_per_step is not None:
        launches = launches_per_step * args.steps
    clocks = sampler.stop()
    value = flops / (ms * 1e-3) / 1e12
    out = step()
    torch.cuda.synchronize()

    # ---- e2e: host (pinned) activation in, host result out, every step ----
    # Every step uploads its activation from pinned host memory and reads its
    # result back.  With CUDA graphs the copies are pipelined: two captured
    # steps on two activation/output buffer sets alternate, step k+1's upload
    # and step k-1's download run on copy streams under step k's compute.
    e2e = None
    if not args.no_e2e:
        x_host = torch.empty(inputs[0].shape, dtype=inputs[0].dtype, pin_memory=True)
        x_host.copy_(inputs[0].cpu())
        out_host = [torch.empty(out[0].shape, dtype=out[0].dtype, pin_memory=True)
                    for _ in range(2)]
        if args.eager:
            dev_inputs = list(inputs)

            def run_e2e(nsteps):
                for _ in range(nsteps):
                    dev_inputs[0].copy_(x_host, non_blocking=True)
                    o = ex.run(dev_inputs)
                    out_host[0].copy_(o[0], non_blocking=True)
        else:
            inputs_b = [inputs[0].clone()] + list(inputs[1:])
            graph_b, outs_b = ex.capture(inputs_b)
            sets = [(inputs, graph, graph_outs), (inputs_b, graph_b, outs_b)]
            copy_in = torch.cuda.Stream(device=dev)
            copy_out = torch.cuda.Stream(device=dev)

            def run_e2e(nsteps):
                done = [None, None]      # step finished reading its activation
                drained = [None, None]   # its result copied out
                last = None
                for k in range(nsteps):
                    b = k % 2
                    ins, gph, gouts = sets[b]
                    if done[b] is not None:
                        copy_in.wait_event(done[b])
                    with torch.cuda.stream(copy_in):
                        ins[0].copy_(x_host, non_blocking=True)
                    up = torch.cuda.Event()
                    up.record(copy_in)
                    stream.wait_event(up)
                    if drained[b] is not None:
                        stream.wait_event(drained[b])
                    gph.replay()
                    done[b] = torch.cuda.Event()
                    done[b].record(stream)
                    copy_out.wait_event(done[b])
                    with torch.cuda.stream(copy_out):
                        out_host[b].copy_(gouts[0], non_blocking=True)
                    drained[b] = last = torch.cuda.Event()
                    last.record(copy_out)
                stream.wait_event(last)
        run_e2e(2)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_e2e(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1) / args.steps
        t = torch.tensor([ems], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
        e2e = {"value": flops / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": ems,
               "h2d_bytes_per_step": int(x_host.numel() * x_host.element_size() * world),
               "d2h_bytes_per_step": int(out_host[0].numel() * out_host[0].element_size() * world),
               "copies": "serial" if args.eager else
               "pipelined (2 captured steps, copy streams)"}
        if not args.eager:
            del graph_b, outs_b, sets

    # ---- roofline of the dominant kernel: the largest tcgen05 GEMM ----
    burst, sustained, hbm, peak_src = _peaks()
    print(f"[bench] step {ms:.2f} ms  ({value:.1f} TFLOP/s aggregate)", file=sys.stderr)
    roofline = _top_kernel(run, dev, burst, sustained, peak_src)
    stats = collective_stats(prog)
    mesh, dims, wdesc, routing = run.mesh, run.dims, run.wdesc, run.routing
    del run, ex, graph, graph_outs, step, out, inputs
    torch.cuda.empty_cache()

    # ---- the other BASELINE configs, same harness (driver-visible) ----
    configs = None
    if not args.no_extras and args.config == "c2":
        configs = {}
        if world == 4:
            # BASELINE's 2x2 is the headline at N=4; the 1x4 mesh (no data
            # axis: no weight gathers) as the alternative layout
            alt = _Run("c2", world, rank, dev, comm, mesh=(1, 4))
            torch.cuda.synchronize()
            time.sleep(1.0)                  # see _extra_config
            ams, _, ag, ao, _ = _time_steps(alt, args.steps, args.warmup, False, barrier, world,
                                            dev)
            configs["c2_mesh_1x4"] = {"mesh": [1, 4], "ms_per_step": ams,
                                      "tflops": alt.flops / (ams * 1e-3) / 1e12}
            del alt, ag, ao
            torch.cuda.empty_cache()
        # C1 last: its 3xTF32 scratch pool keeps its memory (keep_pool_memory)
        for cfg in ("c3", "c4", "c1") if world in (1, 4) else ("c3", "c4"):
            configs[cfg] = _extra_config(cfg, world, rank, dev, comm, barrier,
                                         max(5, args.steps // 2), args.warmup, burst, sustained,
                                         peak_src)
        if rank == 0:
            configs["c5_hbm"] = _c5_hbm(dev, hbm, peak_src)
        barrier()

    # ---- reshard GB/s (config C5) at N > 1 ----
    reshard = None
    if world > 1 and args.config == "c2":
        # settle after the tensor-core configs: run straight after C1 the
        # all-to-all measured 549 GB/s/GPU at N=4, 650 on its own
        # (scripts/reshard_probe.py, profiles/r2_reshard_probe_n4.log)
        torch.cuda.synchronize()
        time.sleep(1.0)
        reshard = _reshard(world, rank, dev, comm, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == "c2":
        # ~20 s of CPU work: the best of 2 samples of ~9 s each (B=4)
        v, tcpu, cores, sample = _cpu_baseline(mesh, steps=2)
        sample += ", best of 2 timed samples"
        cpu = {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port",
               "sample": sample, "seconds_per_sample": tcpu}

    if rank == 0:
        per_gpu = value / world
        cfg = {"workload": wdesc, "dims": dims, "mesh": list(mesh),
               "parallelism": ("dp%dxmp%d" % mesh) if args.config in ("c1", "c2", "c2train") else
               ("expert%d" % world if args.config == "c3" else "spatial%d" % world),
               "plan": "fast", "l2": "inputs larger than L2 (weights+activations)",
               "collectives_per_step": stats["counts"]}
        if routing:
            cfg["dispatch_combine"] = "moe.cu gather kernels over the on-device top-2 " \
                "routing (equal to the dense Dots)"
        if args.config in ("c2", "c2train"):
            cfg.update(global_batch=dims["B"], seq_len=dims["S"])
        line = {
            "metric": METRIC if args.config == "c2" else
            f"{args.config} throughput (TFLOP/s) at 1/2/4/8 B200",
            "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if args.config == "c1" else "bf16", "data": "synthetic",
            "config": cfg,
            "tflops_per_gpu": per_gpu,
            "mfu": {"vs_spec_2250": per_gpu / SPEC_BF16_TFLOPS,
                    "vs_measured_sustained": per_gpu / sustained},
            "roofline": roofline,
            "reshard": reshard,
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "cpu_baseline": cpu,
            "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
