"""Generate golden fixtures by running the REFERENCE (minispmd) itself.

Run in the build container (the reference is not on the GPU box):

    cp -r /root/reference/pkg /tmp/refpkg        # never write into /root/reference
    PYTHONPATH=/tmp/refpkg/src:. python tests/golden/make_golden.py

Writes ``tests/golden/{random,named}.json.gz`` and ``*.npz``:

* ``random``: ``minispmd.testing.random_graph`` seeds 0..239 (the reference's
  acceptance-1 suite, ``tests/test_acceptance.py:55-71``): the user-annotated
  graph, the reference's propagation result (per-op sharding strings,
  iteration count, change log), the reference's SPMD program (every emitted
  instruction), ``collective_stats``, and the reference evaluator's outputs
  (single-device oracle and per-device SPMD results).
* ``named``: hand-built graphs covering the BASELINE configs C1-C5 at small
  dims, the acceptance fixtures (priority Fig-4, 2-D FFW, conv halo grid,
  data formatting, MoE all-to-all), halo specs, and the reference's own
  known-answer op/collective tests, and shifting-buffer pipelines (gpipe and
  circular schedules, reference pipeline.py) with their bubble accounting.
* C2 training steps (forward + backward layer, weight gradients
  reduce-scattered into the weights' shardings) on 1x2 / 2x2 / 2x4 meshes.
* ``textir``: the reference's ``print_graph`` text of every golden graph,
  its propagated form and its SPMD program, and the ``ParseError``
  line/column/message for a set of malformed inputs.

Everything is converted to this package's JSON graph format
(``paper_2105_04663_b200.ir.graph_to_json``) so that tests never need the
reference at run time.
"""

from __future__ import annotations

import gzip
import io
import json
import os
import sys

import numpy as np

import minispmd as R
from minispmd import formatting as RF
from minispmd import simulator as RS
from minispmd.testing import random_graph

from paper_2105_04663_b200 import ir as M
from paper_2105_04663_b200.sharding import DeviceMesh, Sharding

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# reference object -> this package's objects
# ---------------------------------------------------------------------------

def conv_attr(v):
    if isinstance(v, R.Shape):
        return M.Shape(v.dims, M.DType(v.dtype.value))
    if isinstance(v, R.ReduceKind):
        return M.ReduceKind(v.value)
    if isinstance(v, R.CompareDirection):
        return M.CompareDirection(v.value)
    if isinstance(v, R.ConvDims):
        return M.ConvDims(**v.__dict__)
    if isinstance(v, R.WindowDim):
        return M.WindowDim(**v.__dict__)
    if isinstance(v, tuple):
        return tuple(conv_attr(x) for x in v)
    if isinstance(v, list):
        return tuple(conv_attr(x) for x in v)
    return v


def conv_ins(ins):
    s = ins.sharding
    return M.Instruction(
        ins.id, M.Op(ins.opcode.value), tuple(ins.operands),
        {k: conv_attr(v) for k, v in ins.attrs.items()},
        M.Shape(ins.shape.dims, M.DType(ins.shape.dtype.value)),
        None if s is None else Sharding.parse(s.format()))


def conv_graph(g):
    mesh = None if g.mesh is None else DeviceMesh(g.mesh.mesh_dims, g.mesh.device_ids)
    return M.Graph(g.name, tuple(conv_ins(i) for i in g.instructions),
                   tuple(g.outputs), mesh)


def gjson(g):
    return M.graph_to_json(conv_graph(g))


# ---------------------------------------------------------------------------
# one case: propagate + partition + evaluate with the reference
# ---------------------------------------------------------------------------

REF_GRAPHS = {}   # name -> (reference graph, num_devices), for the text-IR fixtures


def run_case(name, graph, inputs, num_devices, arrays, evaluate=True):
    REF_GRAPHS[name] = (graph, num_devices)
    annotated, rep = R.propagate(graph)
    case = {"name": name, "num_devices": num_devices, "graph": gjson(graph),
            "propagation": {"iterations": rep.iterations,
                            "final": rep.final_shardings,
                            "changes": [c.to_json() for c in rep.changes]}}
    try:
        prog = R.partition(annotated, num_devices)
    except Exception as e:  # record unsupported configurations too
        case["partition_error"] = type(e).__name__
        return case
    case["program"] = gjson(prog.graph)
    case["param_shardings"] = [s.format() for s in prog.param_shardings]
    case["output_shardings"] = [s.format() for s in prog.output_shardings]
    case["stats"] = R.collective_stats(prog)
    case["inputs"] = []
    for k, x in enumerate(inputs):
        key = f"{name}/in{k}"
        arrays[key] = np.asarray(x)
        case["inputs"].append(key)
    if not evaluate:
        return case
    exp = RS.evaluate_single(graph, inputs)
    case["expected"] = []
    for k, x in enumerate(exp):
        key = f"{name}/exp{k}"
        arrays[key] = np.asarray(x)
        case["expected"].append(key)
    devices = list(range(num_devices))
    per_dev = {d: [] for d in devices}
    for p, val in zip(annotated.parameters, inputs):
        shards = R.shard_data(np.asarray(val), p.sharding, devices=devices)
        for d in devices:
            per_dev[d].append(shards[d])
    res = RS.evaluate_spmd(prog, per_dev)
    case["spmd"] = {}
    for d in devices:
        keys = []
        for k, x in enumerate(res[d]):
            key = f"{name}/d{d}/out{k}"
            arrays[key] = np.asarray(x)
            keys.append(key)
        case["spmd"][str(d)] = keys
    vr = RS.verify_equivalence(graph, annotated, num_devices, list(inputs))
    case["verify"] = {"passed": vr.passed, "max_abs": vr.max_abs_error,
                      "max_rel": vr.max_rel_error, "counts": vr.collective_counts}
    return case


# ---------------------------------------------------------------------------
# named graphs (built with the reference API)
# ---------------------------------------------------------------------------

def _dot(b, x, w, lb, rb, lc, rc, sharding=None, id=None):
    return b.add(R.Op.DOT, [x, w], {"lhs_batch": lb, "rhs_batch": rb,
                                    "lhs_contracting": lc, "rhs_contracting": rc},
                 sharding=sharding, id=id)


def named_cases():
    rng = np.random.default_rng(1234)
    out = []

    def f32(*dims):
        return rng.standard_normal(dims).astype(np.float32)

    def ints(*dims):
        return rng.integers(-4, 5, dims).astype(np.int32)

    # C1: BSM,MH->BSH on 2x2 (BASELINE configs[0]); two sizes.
    for (B, S, Md, H) in ((4, 6, 8, 12), (8, 16, 32, 24)):
        mesh = R.DeviceMesh.default(2, 2)
        b = R.GraphBuilder("c1", mesh)
        x = b.parameter(R.Shape((B, S, Md)), sharding=R.mesh_split(3, mesh, [0, -1, 1]), id="x")
        w = b.parameter(R.Shape((Md, H)), sharding=R.mesh_split(2, mesh, [0, 1]), id="w")
        y = _dot(b, x, w, (), (), (2,), (0,), id="y")
        out.append((f"c1_{B}x{S}x{Md}x{H}", b.build([y]), [f32(B, S, Md), f32(Md, H)], 4))

    # Acceptance 3: 2-D FFW finalized / attempt 1.
    for tag, xm, wm, om in (("final", [0, 1], [1, 0], [0, 1]),
                            ("attempt", [-1, 1], [1, 0], [-1, 0])):
        mesh = R.DeviceMesh.default(2, 2)
        b = R.GraphBuilder("ffw", mesh)
        x = b.parameter(R.Shape((8, 8)), sharding=R.mesh_split(2, mesh, xm))
        w = b.parameter(R.Shape((8, 8)), sharding=R.mesh_split(2, mesh, wm))
        y = _dot(b, x, w, (), (), (1,), (0,), sharding=R.mesh_split(2, mesh, om))
        out.append((f"ffw_{tag}", b.build([y]), [f32(8, 8), f32(8, 8)], 4))

    # Priority fixture (Fig. 4).
    mesh = R.DeviceMesh.default(2)
    b = R.GraphBuilder("fixture", mesh)
    u = b.parameter(R.Shape((8,)), sharding=R.mesh_split(1, mesh, [0]), id="u")
    r = b.parameter(R.Shape((8, 6)), sharding=R.mesh_split(2, mesh, [-1, 0]), id="r")
    bc = b.add(R.Op.BROADCAST, [u], {"out_dims": (8, 6), "broadcast_dims": (0,)}, id="b")
    y = b.add(R.Op.ADD, [bc, r], id="y")
    out.append(("priority_fig4", b.build([y]), [f32(8), f32(8, 6)], 2))

    # C2: transformer layer (attention + FFN), small dims, meshes of 1/2/4/8.
    for mesh_dims in ((1, 1), (1, 2), (2, 2), (2, 4), (4, 2), (1, 8)):
        g, ins = transformer_layer(mesh_dims, B=4, S=8, M=16, N=8, D=4, H=32, rng=rng)
        out.append(("c2_%dx%d" % mesh_dims, g, ins, mesh_dims[0] * mesh_dims[1]))

    # C3: GShard MoE FFN, expert-sharded over 8 (dispatch via one-hot Dot).
    for n in (2, 4, 8):
        g, ins = moe_layer(n, E=8, B=8, S=8, C=4, M=8, H=16, rng=rng)
        out.append((f"c3_moe_{n}", g, ins, n))

    # C4: spatially partitioned 3x3 conv stack (NHWC), H or (H,W) sharded.
    for mesh_dims, mapping in (((2,), [-1, 0, -1, -1]), ((4,), [-1, 0, -1, -1]),
                               ((8,), [-1, 0, -1, -1]), ((2, 4), [-1, 0, 1, -1])):
        g, ins = conv_stack(mesh_dims, mapping, N=2, H=16, W=16, C=4, layers=2, rng=rng)
        out.append(("c4_conv_" + "x".join(map(str, mesh_dims)), g, ins,
                    int(np.prod(mesh_dims))))

    # C5: uneven partitioning: dim 1000 (even over 8!) / 1001 / 999 over 8.
    for n0, n1 in ((1000, 16), (1001, 16), (999, 16), (16, 1001)):
        for kind in ("a2a", "repl", "reduce_max", "reduce_sum"):
            g, ins = uneven_case(n0, n1, kind, rng)
            out.append((f"c5_{kind}_{n0}x{n1}", g, ins, 8))

    # Acceptance 4: the 72-config conv halo grid (int32, exact).
    n = 16
    for size in (2, 3, 5):
        for stride in (1, 2):
            for pad_mode in ("valid", "same"):
                for bd in (1, 2, 3):
                    if pad_mode == "valid":
                        pl = ph = 0
                    else:
                        nd = (n - 1) * bd + 1
                        m_out = -(-nd // stride)
                        tot = max((m_out - 1) * stride + size - nd, 0)
                        pl, ph = tot // 2, tot - tot // 2
                    w = R.WindowDim(size=size, stride=stride, padding_low=pl,
                                    padding_high=ph, base_dilation=bd)
                    for parts in (2, 4):
                        mesh = R.DeviceMesh.default(parts)
                        b = R.GraphBuilder("conv", mesh)
                        cd = R.ConvDims(0, 1, (2,), 0, 1, (2,), 0, 1, (2,))
                        x = b.parameter(R.Shape((2, 3, n), R.DType.S32),
                                        sharding=R.mesh_split(3, mesh, [-1, -1, 0]))
                        k = b.parameter(R.Shape((3, 4, size), R.DType.S32),
                                        sharding=R.Sharding.replicated())
                        y = b.add(R.Op.CONVOLUTION, [x, k], {"conv_dims": cd, "window": (w,)})
                        out.append((f"acc4_{size}_{stride}_{pad_mode}_{bd}_{parts}",
                                    b.build([y]), [ints(2, 3, n), ints(3, 4, size)], parts))

    # Acceptance 5: data formatting, exact ints.
    mesh2, mesh4 = R.DeviceMesh.default(2), R.DeviceMesh.default(4)
    b = R.GraphBuilder("rs", mesh2)
    x = b.parameter(R.Shape((3, 2), R.DType.S32), sharding=R.mesh_split(2, mesh2, [0, -1]))
    y = b.add(R.Op.RESHAPE, [x], {"out_dims": (6,)}, sharding=R.mesh_split(1, mesh2, [0]))
    out.append(("acc5_reshape", b.build([y]), [np.arange(6, dtype=np.int32).reshape(3, 2)], 2))
    b = R.GraphBuilder("rev", mesh4)
    x = b.parameter(R.Shape((11,), R.DType.S32), sharding=R.mesh_split(1, mesh4, [0]))
    y = b.add(R.Op.REVERSE, [x], {"dims": (0,)}, sharding=R.mesh_split(1, mesh4, [0]))
    out.append(("acc5_reverse", b.build([y]), [np.arange(11, dtype=np.int32)], 4))
    b = R.GraphBuilder("pad", mesh4)
    x = b.parameter(R.Shape((10,), R.DType.S32), sharding=R.mesh_split(1, mesh4, [0]))
    c = b.constant(np.int32(-7), R.Shape((), R.DType.S32))
    y = b.add(R.Op.PAD, [x, c], {"low": (3,), "high": (2,), "interior": (1,)},
              sharding=R.mesh_split(1, mesh4, [0]))
    out.append(("acc5_pad", b.build([y]), [np.arange(10, dtype=np.int32)], 4))
    b = R.GraphBuilder("slc", mesh4)
    x = b.parameter(R.Shape((13,), R.DType.S32), sharding=R.mesh_split(1, mesh4, [0]))
    y = b.add(R.Op.SLICE, [x], {"starts": (2,), "limits": (12,), "strides": (2,)},
              sharding=R.mesh_split(1, mesh4, [0]))
    out.append(("acc5_slice", b.build([y]), [np.arange(13, dtype=np.int32)], 4))

    # Acceptance 7: expert-parallel einsum -> all-to-all.
    mesh = R.DeviceMesh.default(4)
    b = R.GraphBuilder("moe", mesh)
    x = b.parameter(R.Shape((4, 8, 2, 6)), sharding=R.mesh_split(4, mesh, [-1, 0, -1, -1]))
    h = b.add(R.Op.RELU, [x], sharding=R.mesh_split(4, mesh, [-1, 0, -1, -1]))
    w = b.parameter(R.Shape((4, 6, 5)), sharding=R.mesh_split(3, mesh, [0, -1, -1]))
    y = _dot(b, h, w, (0,), (0,), (3,), (1,), sharding=R.mesh_split(4, mesh, [0, -1, -1, -1]))
    out.append(("acc7_moe", b.build([y]), [f32(4, 8, 2, 6), f32(4, 6, 5)], 4))

    # Rotate / shift lowering (reference tests/test_formatting.py:186-237).
    for n_, k_, parts in ((8, 2, 4), (8, 3, 4), (12, 4, 4), (8, 4, 2)):
        mesh = R.DeviceMesh.default(parts)
        b = R.GraphBuilder("rot", mesh)
        x = b.parameter(R.Shape((n_, 3)), sharding=R.mesh_split(2, mesh, [0, -1]))
        a_ = b.add(R.Op.SLICE, [x], {"starts": (k_, 0), "limits": (n_, 3), "strides": (1, 1)})
        c_ = b.add(R.Op.SLICE, [x], {"starts": (0, 0), "limits": (k_, 3), "strides": (1, 1)})
        y = b.add(R.Op.CONCAT, [a_, c_], {"dim": 0}, sharding=R.mesh_split(2, mesh, [0, -1]))
        out.append((f"rotate_{n_}_{k_}_{parts}", b.build([y]), [f32(n_, 3)], parts))
    for n_, lo, hi, parts, fill in ((8, 2, 0, 4, 0.0), (8, 0, 2, 4, 0.0), (8, 3, 0, 4, 1.5),
                                    (8, 1, 0, 2, -2.0)):
        mesh = R.DeviceMesh.default(parts)
        b = R.GraphBuilder("shift", mesh)
        x = b.parameter(R.Shape((n_,)), sharding=R.mesh_split(1, mesh, [0]))
        cst = b.constant(np.float32(fill), R.Shape(()))
        pd = b.add(R.Op.PAD, [x, cst], {"low": (lo,), "high": (hi,), "interior": (0,)})
        y = b.add(R.Op.SLICE, [pd], {"starts": (hi,), "limits": (hi + n_,), "strides": (1,)},
                  sharding=R.mesh_split(1, mesh, [0]))
        out.append((f"shift_{n_}_{lo}_{hi}_{parts}", b.build([y]), [f32(n_)], parts))
    return out


def transformer_layer(mesh_dims, B, S, M, N, D, H, rng, dtype=None):
    """Attention + FFN, 2-D finalized annotations: x [X,-,Y],
    Wq/k/v [X,Y,-], Wo [Y,-,X], W_in [X,Y], W_out [Y,X]."""
    mesh = R.DeviceMesh.default(*mesh_dims)
    ms = lambda r, m: R.mesh_split(r, mesh, m)
    b = R.GraphBuilder("transformer", mesh)
    x = b.parameter(R.Shape((B, S, M)), sharding=ms(3, [0, -1, 1]), id="x")
    wq = b.parameter(R.Shape((M, N, D)), sharding=ms(3, [0, 1, -1]), id="wq")
    wk = b.parameter(R.Shape((M, N, D)), sharding=ms(3, [0, 1, -1]), id="wk")
    wv = b.parameter(R.Shape((M, N, D)), sharding=ms(3, [0, 1, -1]), id="wv")
    wo = b.parameter(R.Shape((N, D, M)), sharding=ms(3, [1, -1, 0]), id="wo")
    wi = b.parameter(R.Shape((M, H)), sharding=ms(2, [0, 1]), id="wi")
    wt = b.parameter(R.Shape((H, M)), sharding=ms(2, [1, 0]), id="wt")
    q = _dot(b, x, wq, (), (), (2,), (0,), id="q")          # [B,S,N,D]
    k = _dot(b, x, wk, (), (), (2,), (0,), id="k")
    v = _dot(b, x, wv, (), (), (2,), (0,), id="v")
    logits = _dot(b, q, k, (0, 2), (0, 2), (3,), (3,), id="logits")   # [B,N,S,T]
    ninf = b.constant(np.float32(-np.inf), R.Shape(()), id="ninf")
    zero = b.constant(np.float32(0), R.Shape(()), id="zero")
    mx = b.add(R.Op.REDUCE, [logits, ninf], {"kind": R.ReduceKind.MAX, "dims": (3,)}, id="mx")
    mxb = b.add(R.Op.BROADCAST, [mx], {"out_dims": (B, N, S, S), "broadcast_dims": (0, 1, 2)},
                id="mxb")
    sh = b.add(R.Op.SUBTRACT, [logits, mxb], id="shifted")
    e = b.add(R.Op.EXP, [sh], id="e")
    den = b.add(R.Op.REDUCE, [e, zero], {"kind": R.ReduceKind.SUM, "dims": (3,)}, id="den")
    denb = b.add(R.Op.BROADCAST, [den], {"out_dims": (B, N, S, S), "broadcast_dims": (0, 1, 2)},
                 id="denb")
    probs = b.add(R.Op.DIVIDE, [e, denb], id="probs")
    ctx = _dot(b, probs, v, (0, 1), (0, 2), (3,), (1,), id="ctx")   # [B,N,S,D]
    ctx_t = b.add(R.Op.TRANSPOSE, [ctx], {"permutation": (0, 2, 1, 3)}, id="ctx_t")
    attn = _dot(b, ctx_t, wo, (), (), (2, 3), (0, 1), id="attn_out")   # [B,S,M]
    res1 = b.add(R.Op.ADD, [attn, x], id="res1")
    h = _dot(b, res1, wi, (), (), (2,), (0,), id="h")
    act = b.add(R.Op.RELU, [h], id="act")
    ffn = _dot(b, act, wt, (), (), (2,), (0,), id="ffn_out")
    out = b.add(R.Op.ADD, [ffn, res1], id="out")
    g = b.build([out])
    sc = lambda *d: (rng.standard_normal(d) / np.sqrt(d[0])).astype(np.float32)
    ins = [rng.standard_normal((B, S, M)).astype(np.float32), sc(M, N, D), sc(M, N, D),
           sc(M, N, D), (rng.standard_normal((N, D, M)) / np.sqrt(N * D)).astype(np.float32),
           sc(M, H), sc(H, M)]
    return g, ins


def moe_layer(n, E, B, S, C, M, H, rng):
    """GShard MoE FFN: dispatch one-hot [B,S,E,C] x tokens [B,S,M] ->
    [B,E,C,M] (B-sharded) -> transpose [E,B,C,M] (E-sharded: all-to-all) ->
    expert FFN -> back to B (all-to-all) -> combine."""
    mesh = R.DeviceMesh.default(n)
    ms = lambda r, m: R.mesh_split(r, mesh, m)
    b = R.GraphBuilder("moe", mesh)
    x = b.parameter(R.Shape((B, S, M)), sharding=ms(3, [0, -1, -1]), id="x")
    disp = b.parameter(R.Shape((B, S, E, C)), sharding=ms(4, [0, -1, -1, -1]), id="dispatch")
    comb = b.parameter(R.Shape((B, S, E, C)), sharding=ms(4, [0, -1, -1, -1]), id="combine")
    wi = b.parameter(R.Shape((E, M, H)), sharding=ms(3, [0, -1, -1]), id="wi")
    wo = b.parameter(R.Shape((E, H, M)), sharding=ms(3, [0, -1, -1]), id="wo")
    dsp = _dot(b, disp, x, (0,), (0,), (1,), (1,), sharding=ms(4, [0, -1, -1, -1]),
               id="dispatched")                                            # [B,E,C,M]
    ebcm = b.add(R.Op.TRANSPOSE, [dsp], {"permutation": (1, 0, 2, 3)}, id="ebcm_b")
    ebcm_e = b.add(R.Op.RELU, [ebcm], sharding=ms(4, [0, -1, -1, -1]), id="ebcm_e")
    h = _dot(b, ebcm_e, wi, (0,), (0,), (3,), (1,), sharding=ms(4, [0, -1, -1, -1]),
             id="h")                                                       # [E,B,C,H]
    a = b.add(R.Op.RELU, [h], id="a")
    y = _dot(b, a, wo, (0,), (0,), (3,), (1,), sharding=ms(4, [0, -1, -1, -1]),
             id="y")                                                       # [E,B,C,M]
    yb = b.add(R.Op.TRANSPOSE, [y], {"permutation": (1, 0, 2, 3)}, id="ebcm_bsh")
    yb2 = b.add(R.Op.RELU, [yb], sharding=ms(4, [0, -1, -1, -1]), id="ybe")
    out = _dot(b, comb, yb2, (0,), (0,), (2, 3), (1, 2), id="out")         # [B,S,M]
    g = b.build([out])
    # Top-1 routing with capacity: one-hot masks.
    disp_v = np.zeros((B, S, E, C), np.float32)
    for bb in range(B):
        fill = [0] * E
        for ss in range(S):
            e_ = int(rng.integers(E))
            if fill[e_] < C:
                disp_v[bb, ss, e_, fill[e_]] = 1.0
                fill[e_] += 1
    comb_v = disp_v * rng.uniform(0.2, 1.0, (B, S, 1, 1)).astype(np.float32)
    ins = [rng.standard_normal((B, S, M)).astype(np.float32), disp_v, comb_v,
           (rng.standard_normal((E, M, H)) / np.sqrt(M)).astype(np.float32),
           (rng.standard_normal((E, H, M)) / np.sqrt(H)).astype(np.float32)]
    return g, ins


def conv_stack(mesh_dims, mapping, N, H, W, C, layers, rng):
    mesh = R.DeviceMesh.default(*mesh_dims)
    b = R.GraphBuilder("convstack", mesh)
    cd = R.ConvDims(lhs_batch=0, lhs_feature=3, lhs_spatial=(1, 2), rhs_in_feature=2,
                    rhs_out_feature=3, rhs_spatial=(0, 1), out_batch=0, out_feature=3,
                    out_spatial=(1, 2))
    win = (R.WindowDim(3, 1, 1, 1), R.WindowDim(3, 1, 1, 1))
    x = b.parameter(R.Shape((N, H, W, C)), sharding=R.mesh_split(4, mesh, mapping), id="x")
    ws = [b.parameter(R.Shape((3, 3, C, C)), sharding=R.Sharding.replicated(), id=f"w{i}")
          for i in range(layers)]
    cur = x
    for i in range(layers):
        y = b.add(R.Op.CONVOLUTION, [cur, ws[i]], {"conv_dims": cd, "window": win}, id=f"conv{i}")
        cur = b.add(R.Op.RELU, [y], id=f"relu{i}")
    g = b.build([cur])
    ins = [rng.standard_normal((N, H, W, C)).astype(np.float32)] + \
          [(rng.standard_normal((3, 3, C, C)) / np.sqrt(9 * C)).astype(np.float32)
           for _ in range(layers)]
    return g, ins


def uneven_case(n0, n1, kind, rng, parts=8):
    mesh = R.DeviceMesh.default(parts)
    b = R.GraphBuilder("uneven", mesh)
    x = b.parameter(R.Shape((n0, n1)), sharding=R.mesh_split(2, mesh, [0, -1]), id="x")
    if kind == "a2a":
        y = b.add(R.Op.NEGATE, [x], sharding=R.mesh_split(2, mesh, [-1, 0]), id="y")
    elif kind == "repl":
        y = b.add(R.Op.NEGATE, [x], sharding=R.Sharding.replicated(), id="y")
    else:
        rk = R.ReduceKind.MAX if kind == "reduce_max" else R.ReduceKind.SUM
        init = b.constant(np.float32(-np.inf if rk == R.ReduceKind.MAX else 0),
                          R.Shape(()), id="init")
        y = b.add(R.Op.REDUCE, [x, init], {"kind": rk, "dims": (0,)}, id="y")
    return b.build([y]), [rng.standard_normal((n0, n1)).astype(np.float32)]


def halo_specs():
    cases = [(1024, 2, dict(size=3, padding_low=1, padding_high=1), 1024),
             (1024, 4, dict(size=3, padding_low=1, padding_high=1), 1024),
             (1024, 8, dict(size=3, padding_low=1, padding_high=1), 1024),
             (1024, 8, dict(size=5, padding_low=2, padding_high=2), 1024),
             (1024, 8, dict(size=3, stride=2, padding_low=1, padding_high=1), 512),
             (16, 4, dict(size=2, padding_low=1, padding_high=1), 17),
             (12, 4, dict(size=3, padding_low=1, padding_high=1, base_dilation=2), 23),
             (10, 2, dict(size=3, stride=2, padding_low=2, padding_high=1, base_dilation=3), 15),
             (15, 4, dict(size=2, stride=2, padding_low=0, padding_high=1, base_dilation=2), 15)]
    out = []
    for n, t, w, m in cases:
        wd = R.WindowDim(**w)
        m = wd.output_size(n)
        s = RF.conv_halo_spec(n, t, wd, m)
        out.append({"n": n, "t": t, "window": w, "m": m, "spec": s.__dict__})
    return out


def collective_known_answers(arrays):
    """Per-device in/out of the reference's own collective known-answer tests
    plus randomized cases (dtype s32/f32, groups of 2..8)."""
    rng = np.random.default_rng(77)
    cases = []

    def add(op, attrs, shape_out, per_dev, dtype):
        ins = R.Instruction(id="c", opcode=op, operands=("x",), attrs=attrs,
                            shape=R.Shape(shape_out, dtype), sharding=None)
        res = RS._collective(ins, per_dev, sorted(per_dev))
        k = len(cases)
        for d, v in per_dev.items():
            arrays[f"coll{k}/in{d}"] = v
            arrays[f"coll{k}/out{d}"] = res[d]
        cases.append({"op": op.value, "attrs": M.instruction_to_json(conv_ins(ins))["attrs"],
                      "shape": list(shape_out), "dtype": dtype.value,
                      "devices": sorted(per_dev)})

    for n in (2, 4, 8):
        devs = list(range(n))
        for dtype in (R.DType.S32, R.DType.F32):
            mk = (lambda *s: rng.integers(-9, 10, s).astype(np.int32)) if dtype == R.DType.S32 \
                else (lambda *s: rng.standard_normal(s).astype(np.float32))
            for gs in sorted({g for g in (2, n // 2, n) if g >= 2 and n % g == 0}):
                perm = [int(v) for v in rng.permutation(n)]
                groups = tuple(tuple(perm[i:i + gs]) for i in range(0, n, gs))
                data = {d: mk(gs * 2, 3) for d in devs}
                for kind in (R.ReduceKind.SUM, R.ReduceKind.MAX, R.ReduceKind.MIN):
                    add(R.Op.ALL_REDUCE, {"kind": kind, "subgroups": groups}, (gs * 2, 3),
                        data, dtype)
                    add(R.Op.REDUCE_SCATTER, {"kind": kind, "dim": 0, "subgroups": groups},
                        (2, 3), data, dtype)
                for dim in (0, 1):
                    add(R.Op.ALL_GATHER, {"dim": dim, "subgroups": groups},
                        (gs * 4, 3) if dim == 0 else (gs * 2, 3 * gs), data, dtype)
                add(R.Op.ALL_TO_ALL, {"split_dim": 0, "concat_dim": 1, "subgroups": groups},
                    (2, 3 * gs), data, dtype)
                add(R.Op.ALL_TO_ALL, {"split_dim": 0, "concat_dim": 0, "subgroups": groups},
                    (gs * 2, 3), data, dtype)
            pairs = tuple(sorted((d, (d + 1) % n) for d in devs if d != n - 1))
            add(R.Op.COLLECTIVE_PERMUTE, {"pairs": pairs}, (4, 3), {d: mk(4, 3) for d in devs},
                dtype)
    return cases


# ---------------------------------------------------------------------------
# pipelines (reference pipeline.py): configs recorded so the test rebuilds
# the same graph with this package's builder
# ---------------------------------------------------------------------------

PIPELINES = [
    # name, L, M, schedule, R, state_dims, body, devices
    ("pipe_gpipe_L4_M8_add", 4, 8, "gpipe", 1, (6,), "add", 4),
    ("pipe_gpipe_L2_M3_dot", 2, 3, "gpipe", 1, (4, 8), "dot", 2),
    ("pipe_circ_L4_M8_R2_add", 4, 8, "circular", 2, (6,), "add", 4),
    ("pipe_circ_L2_M4_R2_dot", 2, 4, "circular", 2, (4, 8), "dot", 2),
    ("pipe_gpipe_L8_M8_add", 8, 8, "gpipe", 1, (16,), "add", 8),
]


def pipeline_body(ops, kind):
    """Stage bodies shared by the generator (reference Op) and the tests
    (this package's Op): x + w, or x + x.w (batched over the stage dim)."""
    def add(b, x, ws):
        return b.add(ops.ADD, [x, ws[0]])

    def dot(b, x, ws):
        y = b.add(ops.DOT, [x, ws[0]], {"lhs_batch": (0,), "rhs_batch": (0,),
                                         "lhs_contracting": (2,), "rhs_contracting": (1,)})
        return b.add(ops.ADD, [x, y])
    return add if kind == "add" else dot


def pipeline_weight_dims(state_dims, kind):
    return (state_dims[-1], state_dims[-1]) if kind == "dot" else tuple(state_dims)


def pipeline_cases(arrays):
    from minispmd import pipeline as RP
    out = []
    for name, L, Mb, sched, Rr, sdims, kind, nd in PIPELINES:
        rng = np.random.default_rng(L * 100 + Mb * 10 + Rr)
        mesh = R.DeviceMesh.default(nd)
        cfg = RP.PipelineConfig(L, Mb, sched, Rr)
        wdims = pipeline_weight_dims(sdims, kind)
        lead = (L,) if sched == "gpipe" else (L, Rr)
        st_sh = R.mesh_split(1 + len(sdims), mesh, [0] + [-1] * len(sdims))
        w_sh = R.mesh_split(len(lead) + len(wdims), mesh, [0] + [-1] * (len(lead) + len(wdims) - 1))
        g = RP.build_pipeline(cfg, mesh, sdims, pipeline_body(R.Op, kind), [R.Shape(wdims)],
                              input_sharding=R.Sharding.replicated(), state_sharding=st_sh,
                              weight_shardings=[w_sh])
        scale = 0.25 if kind == "dot" else 1.0
        ins = [rng.standard_normal(sdims).astype(np.float32) for _ in range(Mb)]
        ins.append((rng.standard_normal(lead + wdims) * scale).astype(np.float32))
        case = run_case(name, g, ins, nd, arrays)
        case["pipeline"] = {"L": L, "M": Mb, "schedule": sched, "R": Rr,
                            "state_dims": list(sdims), "body": kind,
                            "bubble": RP.bubble_stats(cfg).to_json()}
        out.append(case)
    return out


# ---------------------------------------------------------------------------
# text IR (reference textir.py): printouts of every golden graph / program and
# ParseError positions for malformed inputs
# ---------------------------------------------------------------------------

BAD_TEXTS = [
    "graph @g {\n  %x = f32[8 parameter(0)\n  return %x\n}",
    "%x = f32[8] parameter(0), sharding={devices=[2]0,0}",
    "%y = f32[8] relu(%x)",
    "graph @g {\n  %x = f32[8] parameter(0)\n  %y = f32[9] relu(%x)\n  return %y\n}",
    "graph @g {\n  %x = q32[8] parameter(0)\n  return %x\n}",
    "graph @g {\n  %x = f32[8] frobnicate(%x)\n  return %x\n}",
    "graph @g {\n  %x = f32[8] parameter()\n  return %x\n}",
    "graph @g {\n  %c = f32[2] constant()\n  return %c\n}",
    "graph @g {\n  %c = f32[2] constant(), literal=[1.0,2.0,3.0]\n  return %c\n}",
    "%x = f32[8] parameter(0), sharding={devices=[2,2]0,1,2,3}",
    "%x = f32[8] parameter(0) $",
    "graph @g {\n  %x = f32[8] parameter(0), sharding={devices=[2]0,1\n",
    "graph @g {\n  %a = f32[4] parameter(0)\n  %b = f32[4] compare(%a, %a), direction=XX\n"
    "  return %b\n}",
    "graph @g {\n  %a = f32[4] parameter(0)\n  %z = f32[] constant(), literal=0.0\n"
    "  %r = f32[] reduce(%a, %z), kind=avg, dims=[0]\n  return %r\n}",
    "graph @g {\n  %x = f32[8] parameter(0)\n  %y = f32[8] negate(%x)\n}",
    "",
    "graph @g (mesh=[2,2]) {\n  %x = f32[4,4] parameter(0), sharding={devices=[2,2]0,1,2,3}\n"
    "  return %x\n} trailing",
    "graph @g {\n  %x = f32[4] parameter(1.5)\n  return %x\n}",
]


def textir_fixtures():
    from minispmd import textir as RT
    out = {"graphs": {}, "errors": []}
    for name, (g, n) in REF_GRAPHS.items():
        entry = {"graph": RT.print_graph(g)}
        ann, _ = R.propagate(g)
        entry["annotated"] = RT.print_graph(ann)
        try:
            entry["program"] = RT.print_graph(R.partition(ann, n).graph)
        except Exception:   # noqa: BLE001 -- unsupported configurations have no program
            pass
        out["graphs"][name] = entry
    for text in BAD_TEXTS:
        try:
            RT.parse_graph(text)
            out["errors"].append({"text": text, "error": None})
        except RT.ParseError as e:
            out["errors"].append({"text": text, "error": "ParseError", "line": e.line,
                                  "column": e.column, "message": str(e)})
        except Exception as e:   # noqa: BLE001 -- record what the reference raises
            out["errors"].append({"text": text, "error": type(e).__name__, "message": str(e)})
    return out


# ---------------------------------------------------------------------------
# C2 training step (forward + backward), built by this package's workload
# function with the REFERENCE IR (api=minispmd): same graph, reference run
# ---------------------------------------------------------------------------

TRAIN_MESHES = [(1, 2), (2, 2), (2, 4)]
TRAIN_DIMS = dict(B=4, S=8, M=16, N=8, D=4, H=32)


def train_cases(arrays):
    from paper_2105_04663_b200.workloads import train_step_inputs, transformer_train_step
    out = []
    for mesh in TRAIN_MESHES:
        g = transformer_train_step(mesh, api=R, **TRAIN_DIMS)
        ins = train_step_inputs(**TRAIN_DIMS, seed=sum(mesh))
        name = "c2_train_%dx%d" % mesh
        case = run_case(name, g, ins, mesh[0] * mesh[1], arrays)
        case["train"] = {"mesh": list(mesh), "dims": TRAIN_DIMS, "seed": sum(mesh)}
        out.append(case)
    return out


def c5_world_cases(arrays):
    """C5 at world sizes 2 and 4 (the 8-device C5 cases cannot run one
    process per GPU on a 2/4-GPU box): uneven dims 1000/1001/999 (and a
    1001-wide second dim) over 2 and 4 shards, each reshard kind."""
    rng = np.random.default_rng(5005)
    out = []
    for parts in (2, 4):
        for n0, n1 in ((1000, 16), (1001, 16), (999, 16), (16, 1001)):
            for kind in ("a2a", "repl", "reduce_max", "reduce_sum"):
                g, ins = uneven_case(n0, n1, kind, rng, parts=parts)
                out.append(run_case(f"c5w{parts}_{kind}_{n0}x{n1}", g, ins, parts, arrays))
    return out


def write_c5w():
    arrays = {}
    cases = c5_world_cases(arrays)
    with gzip.open(os.path.join(HERE, "c5w.json.gz"), "wt") as f:
        json.dump(cases, f, sort_keys=True)
    buf = io.BytesIO()
    np.savez_compressed(buf, **arrays)
    with open(os.path.join(HERE, "c5w_arrays.npz"), "wb") as f:
        f.write(buf.getvalue())
    print("c5w cases:", len(cases), "arrays:", len(arrays))


def main():
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "c5w":
        return write_c5w()
    arrays = {}
    rand = []
    for seed in range(240):
        rng = np.random.default_rng(seed)
        nd = [2, 4, 8][int(rng.integers(3))]
        g, inputs = random_graph(rng, nd)
        rand.append(run_case(f"rand{seed}", g, inputs, nd, arrays))
    named = [run_case(name, g, ins, n, arrays) for name, g, ins, n in named_cases()]
    named += pipeline_cases(arrays)
    named += train_cases(arrays)
    extra = {"halo_specs": halo_specs(), "collectives": collective_known_answers(arrays)}
    textir = textir_fixtures()
    for fname, obj in (("random.json.gz", rand), ("named.json.gz", named),
                       ("extra.json.gz", extra), ("textir.json.gz", textir)):
        with gzip.open(os.path.join(HERE, fname), "wt") as f:
            json.dump(obj, f, sort_keys=True)
    buf = io.BytesIO()
    np.savez_compressed(buf, **arrays)
    with open(os.path.join(HERE, "arrays.npz"), "wb") as f:
        f.write(buf.getvalue())
    print("cases:", len(rand), len(named), "arrays:", len(arrays))
    write_c5w()


if __name__ == "__main__":
    sys.exit(main())
