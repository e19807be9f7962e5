"""Annotated graphs of the BASELINE configurations (C1-C5), built with this
package's IR.  Shapes and annotations follow SURVEY.md 8(d) / PAPER.md:679
("2D finalized" sharding); the same constructions, built with the reference
API, produce the golden fixtures in ``tests/golden/make_golden.py``.

Each builder returns ``(graph, inputs)``: an annotated graph whose user
annotations are only on parameters and a few anchors (propagation completes
the rest), and seeded synthetic host inputs (N(0,1) activations, N(0,1/fan_in)
weights).  With ``dtype=BF16`` the inputs are returned as float32 holding
bf16-rounded values.
"""

from __future__ import annotations

import numpy as np

from .ir import ConvDims, DType, GraphBuilder, Op, ReduceKind, Shape, WindowDim
from .sharding import DeviceMesh, Sharding, mesh_split


def _bf16(x: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = (((u + ((u >> 16) & 1) + 0x7FFF) >> 16) << 16).astype(np.uint32)
    return r.view(np.float32)


def _dot(b, x, w, lb, rb, lc, rc, sharding=None, id=None):
    return b.add(Op.DOT, [x, w], {"lhs_batch": lb, "rhs_batch": rb,
                                  "lhs_contracting": lc, "rhs_contracting": rc},
                 sharding=sharding, id=id)


def einsum_c1(mesh_dims=(2, 2), B=4, S=6, M=8, H=12, dtype=DType.F32, seed=0,
              with_inputs=True):
    """C1: y[B,S,H] = x[B,S,M] . w[M,H]; x [X,-,Y], w [X,Y] (BASELINE configs[0])."""
    mesh = DeviceMesh.default(*mesh_dims)
    b = GraphBuilder("einsum_bsm_mh", mesh)
    x = b.parameter(Shape((B, S, M), dtype), sharding=mesh_split(3, mesh, [0, -1, 1]), id="x")
    w = b.parameter(Shape((M, H), dtype), sharding=mesh_split(2, mesh, [0, 1]), id="w")
    y = _dot(b, x, w, (), (), (2,), (0,), id="y")
    g = b.build([y])
    if not with_inputs:
        return g, None
    rng = np.random.default_rng(seed)
    ins = [rng.standard_normal((B, S, M)).astype(np.float32),
           (rng.standard_normal((M, H)) / np.sqrt(M)).astype(np.float32)]
    return g, [_bf16(i) for i in ins] if dtype == DType.BF16 else ins


def transformer_layer(mesh_dims=(2, 4), B=16, S=1024, M=8192, N=128, D=256, H=65536,
                      dtype=DType.BF16, seed=0, with_inputs=True):
    """C2: attention + FFN with 2-D finalized sharding (mesh X=data, Y=model):
    x [X,-,Y], Wq/k/v [X,Y,-], Wo [Y,-,X], W_in [X,Y], W_out [Y,X]."""
    mesh = DeviceMesh.default(*mesh_dims)
    ms = lambda r, m: mesh_split(r, mesh, m)
    b = GraphBuilder("transformer", mesh)
    x = b.parameter(Shape((B, S, M), dtype), sharding=ms(3, [0, -1, 1]), id="x")
    wq = b.parameter(Shape((M, N, D), dtype), sharding=ms(3, [0, 1, -1]), id="wq")
    wk = b.parameter(Shape((M, N, D), dtype), sharding=ms(3, [0, 1, -1]), id="wk")
    wv = b.parameter(Shape((M, N, D), dtype), sharding=ms(3, [0, 1, -1]), id="wv")
    wo = b.parameter(Shape((N, D, M), dtype), sharding=ms(3, [1, -1, 0]), id="wo")
    wi = b.parameter(Shape((M, H), dtype), sharding=ms(2, [0, 1]), id="wi")
    wt = b.parameter(Shape((H, M), dtype), sharding=ms(2, [1, 0]), id="wt")
    q = _dot(b, x, wq, (), (), (2,), (0,), id="q")
    k = _dot(b, x, wk, (), (), (2,), (0,), id="k")
    v = _dot(b, x, wv, (), (), (2,), (0,), id="v")
    logits = _dot(b, q, k, (0, 2), (0, 2), (3,), (3,), id="logits")
    ninf = b.constant(np.float32(-np.inf), Shape((), dtype), id="ninf")
    zero = b.constant(np.float32(0), Shape((), dtype), id="zero")
    mx = b.add(Op.REDUCE, [logits, ninf], {"kind": ReduceKind.MAX, "dims": (3,)}, id="mx")
    mxb = b.add(Op.BROADCAST, [mx], {"out_dims": (B, N, S, S), "broadcast_dims": (0, 1, 2)},
                id="mxb")
    sh = b.add(Op.SUBTRACT, [logits, mxb], id="shifted")
    e = b.add(Op.EXP, [sh], id="e")
    den = b.add(Op.REDUCE, [e, zero], {"kind": ReduceKind.SUM, "dims": (3,)}, id="den")
    denb = b.add(Op.BROADCAST, [den], {"out_dims": (B, N, S, S), "broadcast_dims": (0, 1, 2)},
                 id="denb")
    probs = b.add(Op.DIVIDE, [e, denb], id="probs")
    ctx = _dot(b, probs, v, (0, 1), (0, 2), (3,), (1,), id="ctx")
    ctx_t = b.add(Op.TRANSPOSE, [ctx], {"permutation": (0, 2, 1, 3)}, id="ctx_t")
    attn = _dot(b, ctx_t, wo, (), (), (2, 3), (0, 1), id="attn_out")
    res1 = b.add(Op.ADD, [attn, x], id="res1")
    h = _dot(b, res1, wi, (), (), (2,), (0,), id="h")
    act = b.add(Op.RELU, [h], id="act")
    ffn = _dot(b, act, wt, (), (), (2,), (0,), id="ffn_out")
    out = b.add(Op.ADD, [ffn, res1], id="out")
    g = b.build([out])
    if not with_inputs:
        return g, None
    rng = np.random.default_rng(seed)
    f = lambda *d: rng.standard_normal(d).astype(np.float32)
    ins = [f(B, S, M), f(M, N, D) / np.sqrt(M), f(M, N, D) / np.sqrt(M),
           f(M, N, D) / np.sqrt(M), f(N, D, M) / np.sqrt(N * D), f(M, H) / np.sqrt(M),
           f(H, M) / np.sqrt(H)]
    ins = [np.asarray(i, np.float32) for i in ins]
    return g, [_bf16(i) for i in ins] if dtype == DType.BF16 else ins


def transformer_train_step(mesh_dims=(2, 4), B=16, S=1024, M=8192, N=128, D=256, H=65536,
                           dtype=None, api=None):
    """C2 training step: the forward layer plus its backward pass, as plain
    dataflow (the paper's real workload).  ``api`` is the
    package whose IR builds the graph -- this one, or the reference
    ``minispmd`` for the golden fixtures (same names, same graph).

    Inputs: x, the seven weights and the upstream gradient g = dL/d(out).
    Outputs: out, dx and the seven weight gradients.  Only x, g and the
    weights are annotated (2-D finalized) plus the weight
    gradients, pinned to their weights' shardings: the gradient of every
    weight is reduced over the data axis X, which the partitioner emits as a
    reduce-scatter into the weight's shard -- GSPMD weight-update sharding.
    """
    import sys
    api = api or sys.modules[__package__]
    Op, Shape, RK, CD = api.Op, api.Shape, api.ReduceKind, api.CompareDirection
    dtype = dtype or api.DType.F32
    mesh = api.DeviceMesh.default(*mesh_dims)
    ms = lambda r, m: api.mesh_split(r, mesh, m)
    b = api.GraphBuilder("transformer_train", mesh)

    def dot(x, w, lb, rb, lc, rc, id, sharding=None):
        return b.add(Op.DOT, [x, w], {"lhs_batch": lb, "rhs_batch": rb,
                                      "lhs_contracting": lc, "rhs_contracting": rc},
                     sharding=sharding, id=id)

    def tr(x, id):
        return b.add(Op.TRANSPOSE, [x], {"permutation": (0, 2, 1, 3)}, id=id)

    act_sh, qkv_sh, wo_sh, wi_sh, wt_sh = (ms(3, [0, -1, 1]), ms(3, [0, 1, -1]),
                                           ms(3, [1, -1, 0]), ms(2, [0, 1]), ms(2, [1, 0]))
    x = b.parameter(Shape((B, S, M), dtype), sharding=act_sh, id="x")
    wq = b.parameter(Shape((M, N, D), dtype), sharding=qkv_sh, id="wq")
    wk = b.parameter(Shape((M, N, D), dtype), sharding=qkv_sh, id="wk")
    wv = b.parameter(Shape((M, N, D), dtype), sharding=qkv_sh, id="wv")
    wo = b.parameter(Shape((N, D, M), dtype), sharding=wo_sh, id="wo")
    wi = b.parameter(Shape((M, H), dtype), sharding=wi_sh, id="wi")
    wt = b.parameter(Shape((H, M), dtype), sharding=wt_sh, id="wt")
    g = b.parameter(Shape((B, S, M), dtype), sharding=act_sh, id="g")
    # ---- forward (as transformer_layer) ----
    q = dot(x, wq, (), (), (2,), (0,), "q")
    k = dot(x, wk, (), (), (2,), (0,), "k")
    v = dot(x, wv, (), (), (2,), (0,), "v")
    logits = dot(q, k, (0, 2), (0, 2), (3,), (3,), "logits")
    ninf = b.constant(np.float32(-np.inf), Shape((), dtype), id="ninf")
    zero = b.constant(np.float32(0), Shape((), dtype), id="zero")
    full = (B, N, S, S)
    mx = b.add(Op.REDUCE, [logits, ninf], {"kind": RK.MAX, "dims": (3,)}, id="mx")
    mxb = b.add(Op.BROADCAST, [mx], {"out_dims": full, "broadcast_dims": (0, 1, 2)}, id="mxb")
    e = b.add(Op.EXP, [b.add(Op.SUBTRACT, [logits, mxb], id="shifted")], id="e")
    den = b.add(Op.REDUCE, [e, zero], {"kind": RK.SUM, "dims": (3,)}, id="den")
    denb = b.add(Op.BROADCAST, [den], {"out_dims": full, "broadcast_dims": (0, 1, 2)},
                 id="denb")
    probs = b.add(Op.DIVIDE, [e, denb], id="probs")
    ctx = dot(probs, v, (0, 1), (0, 2), (3,), (1,), "ctx")
    ctx_t = tr(ctx, "ctx_t")
    attn = dot(ctx_t, wo, (), (), (2, 3), (0, 1), "attn_out")
    res1 = b.add(Op.ADD, [attn, x], id="res1")
    h = dot(res1, wi, (), (), (2,), (0,), "h")
    act = b.add(Op.RELU, [h], id="act")
    ffn = dot(act, wt, (), (), (2,), (0,), "ffn_out")
    out = b.add(Op.ADD, [ffn, res1], id="out")
    # ---- backward ----
    d_wt = dot(act, g, (), (), (0, 1), (0, 1), "d_wt", sharding=wt_sh)
    dact = dot(g, wt, (), (), (2,), (1,), "dact")
    zb = b.add(Op.BROADCAST, [zero], {"out_dims": (B, S, H), "broadcast_dims": ()}, id="zero_bsh")
    live = b.add(Op.COMPARE, [h, zb], {"direction": CD.GT}, id="relu_mask")
    dh = b.add(Op.SELECT, [live, dact, zb], id="dh")
    d_wi = dot(res1, dh, (), (), (0, 1), (0, 1), "d_wi", sharding=wi_sh)
    dres1 = b.add(Op.ADD, [g, dot(dh, wi, (), (), (2,), (1,), "dres1_ffn")], id="dres1")
    d_wo = dot(ctx_t, dres1, (), (), (0, 1), (0, 1), "d_wo", sharding=wo_sh)
    dctx = tr(dot(dres1, wo, (), (), (2,), (2,), "dctx_t"), "dctx")
    dprobs = dot(dctx, v, (0, 1), (0, 2), (3,), (3,), "dprobs")
    dv = tr(dot(probs, dctx, (0, 1), (0, 1), (2,), (2,), "dv_t"), "dv")
    # softmax: dlogits = p * (dp - sum_t(dp * p))
    pdp = b.add(Op.MULTIPLY, [dprobs, probs], id="pdp")
    spdp = b.add(Op.REDUCE, [pdp, zero], {"kind": RK.SUM, "dims": (3,)}, id="spdp")
    spdpb = b.add(Op.BROADCAST, [spdp], {"out_dims": full, "broadcast_dims": (0, 1, 2)},
                  id="spdpb")
    dlogits = b.add(Op.MULTIPLY, [probs, b.add(Op.SUBTRACT, [dprobs, spdpb], id="dcentered")],
                    id="dlogits")
    dq = tr(dot(dlogits, k, (0, 1), (0, 2), (3,), (1,), "dq_t"), "dq")
    dk = tr(dot(dlogits, q, (0, 1), (0, 2), (2,), (1,), "dk_t"), "dk")
    d_wq = dot(x, dq, (), (), (0, 1), (0, 1), "d_wq", sharding=qkv_sh)
    d_wk = dot(x, dk, (), (), (0, 1), (0, 1), "d_wk", sharding=qkv_sh)
    d_wv = dot(x, dv, (), (), (0, 1), (0, 1), "d_wv", sharding=qkv_sh)
    dxq = dot(dq, wq, (), (), (2, 3), (1, 2), "dx_q")
    dxk = dot(dk, wk, (), (), (2, 3), (1, 2), "dx_k")
    dxv = dot(dv, wv, (), (), (2, 3), (1, 2), "dx_v")
    dx = b.add(Op.ADD, [b.add(Op.ADD, [b.add(Op.ADD, [dres1, dxq], id="dx1"), dxk], id="dx2"),
                        dxv], id="dx")
    return b.build([out, dx, d_wq, d_wk, d_wv, d_wo, d_wi, d_wt])


def train_step_inputs(B, S, M, N, D, H, seed=0):
    """Host inputs of ``transformer_train_step`` (x, weights ~ N(0, 1/fan_in), g)."""
    rng = np.random.default_rng(seed)
    f = lambda *d: rng.standard_normal(d).astype(np.float32)
    return [f(B, S, M), f(M, N, D) / np.sqrt(M), f(M, N, D) / np.sqrt(M), f(M, N, D) / np.sqrt(M),
            f(N, D, M) / np.sqrt(N * D), f(M, H) / np.sqrt(M), f(H, M) / np.sqrt(H),
            f(B, S, M) / np.sqrt(B * S)]


def transformer_train_flops(B, S, M, N, D, H) -> float:
    """Forward + backward GEMM FLOPs: every forward contraction has two
    backward ones of the same size (data and weight/operand gradients)."""
    return 3.0 * transformer_flops(B, S, M, N, D, H)


def transformer_flops(B, S, M, N, D, H) -> float:
    """Algorithmic forward FLOPs of one layer (softmax/elementwise excluded),
    SURVEY 8(d): 2T(3MND + NDM + 2MH) + 4 B N S^2 D."""
    T = B * S
    return 2.0 * T * (3 * M * N * D + N * D * M + 2 * M * H) + 4.0 * B * N * S * S * D


def moe_layer(n, E=8, B=8, S=8, C=4, M=8, H=16, dtype=DType.F32, seed=0, with_inputs=True,
              top_k=1):
    """C3: GShard MoE FFN; dispatch [B,S,E,C] one-hot x tokens -> [B,E,C,M]
    (B-sharded) -> transpose [E,B,C,M] (E-sharded, all-to-all) -> expert FFN ->
    all-to-all back -> combine.  Inputs: masks of a GShard top-``top_k``
    routing of seeded gating logits (moe.route_masks)."""
    mesh = DeviceMesh.default(n)
    ms = lambda r, m: mesh_split(r, mesh, m)
    b = GraphBuilder("moe", mesh)
    x = b.parameter(Shape((B, S, M), dtype), sharding=ms(3, [0, -1, -1]), id="x")
    disp = b.parameter(Shape((B, S, E, C), dtype), sharding=ms(4, [0, -1, -1, -1]), id="dispatch")
    comb = b.parameter(Shape((B, S, E, C), dtype), sharding=ms(4, [0, -1, -1, -1]), id="combine")
    wi = b.parameter(Shape((E, M, H), dtype), sharding=ms(3, [0, -1, -1]), id="wi")
    wo = b.parameter(Shape((E, H, M), dtype), sharding=ms(3, [0, -1, -1]), id="wo")
    # GShard annotations on the einsum outputs: dispatch result batch-sharded,
    # expert FFN expert-sharded (the reshard between them is the all-to-all).
    dsp = _dot(b, disp, x, (0,), (0,), (1,), (1,), sharding=ms(4, [0, -1, -1, -1]),
               id="dispatched")
    ebcm = b.add(Op.TRANSPOSE, [dsp], {"permutation": (1, 0, 2, 3)}, id="ebcm_b")
    ebcm_e = b.add(Op.RELU, [ebcm], sharding=ms(4, [0, -1, -1, -1]), id="ebcm_e")
    h = _dot(b, ebcm_e, wi, (0,), (0,), (3,), (1,), sharding=ms(4, [0, -1, -1, -1]), id="h")
    a = b.add(Op.RELU, [h], id="a")
    y = _dot(b, a, wo, (0,), (0,), (3,), (1,), sharding=ms(4, [0, -1, -1, -1]), id="y")
    yb = b.add(Op.TRANSPOSE, [y], {"permutation": (1, 0, 2, 3)}, id="ebcm_bsh")
    yb2 = b.add(Op.RELU, [yb], sharding=ms(4, [0, -1, -1, -1]), id="ybe")
    out = _dot(b, comb, yb2, (0,), (0,), (2, 3), (1, 2), id="out")
    g = b.build([out])
    if not with_inputs:
        return g, None
    rng = np.random.default_rng(seed)
    from .moe import route_masks
    logits = rng.standard_normal((B, S, E)).astype(np.float32)
    disp_v, comb_v = route_masks(logits, C, top_k)
    ins = [rng.standard_normal((B, S, M)).astype(np.float32), disp_v, comb_v,
           (rng.standard_normal((E, M, H)) / np.sqrt(M)).astype(np.float32),
           (rng.standard_normal((E, H, M)) / np.sqrt(H)).astype(np.float32)]
    return g, [_bf16(i) for i in ins] if dtype == DType.BF16 else ins


def conv_stack(mesh_dims=(8,), mapping=(-1, 0, -1, -1), N=8, H=1024, W=1024, C=128, layers=4,
               dtype=DType.BF16, seed=0, with_inputs=True):
    """C4: NHWC 3x3/stride 1/pad 1 conv + ReLU stack, spatially partitioned;
    weights HWIO replicated (reference forces it, formatting.py:507)."""
    mesh = DeviceMesh.default(*mesh_dims)
    b = GraphBuilder("convstack", mesh)
    cd = ConvDims(lhs_batch=0, lhs_feature=3, lhs_spatial=(1, 2), rhs_in_feature=2,
                  rhs_out_feature=3, rhs_spatial=(0, 1), out_batch=0, out_feature=3,
                  out_spatial=(1, 2))
    win = (WindowDim(3, 1, 1, 1), WindowDim(3, 1, 1, 1))
    x = b.parameter(Shape((N, H, W, C), dtype), sharding=mesh_split(4, mesh, list(mapping)),
                    id="x")
    ws = [b.parameter(Shape((3, 3, C, C), dtype), sharding=Sharding.replicated(), id=f"w{i}")
          for i in range(layers)]
    cur = x
    for i in range(layers):
        y = b.add(Op.CONVOLUTION, [cur, ws[i]], {"conv_dims": cd, "window": win}, id=f"conv{i}")
        cur = b.add(Op.RELU, [y], id=f"relu{i}")
    g = b.build([cur])
    if not with_inputs:
        return g, None
    rng = np.random.default_rng(seed)
    ins = [rng.standard_normal((N, H, W, C)).astype(np.float32)] + \
          [(rng.standard_normal((3, 3, C, C)) / np.sqrt(9 * C)).astype(np.float32)
           for _ in range(layers)]
    return g, [_bf16(i) for i in ins] if dtype == DType.BF16 else ins


def uneven(n0=1001, n1=4096, kind="a2a", parts=8, dtype=DType.F32, seed=0, with_inputs=True):
    """C5: [n0, n1] dim-0 sharded over ``parts``; reshard to dim 1 ("a2a"),
    to replicated ("repl"), or masked reduce over dim 0 ("reduce_max"/"reduce_sum")."""
    mesh = DeviceMesh.default(parts)
    b = GraphBuilder("uneven", mesh)
    x = b.parameter(Shape((n0, n1), dtype), sharding=mesh_split(2, mesh, [0, -1]), id="x")
    if kind == "a2a":
        y = b.add(Op.NEGATE, [x], sharding=mesh_split(2, mesh, [-1, 0]), id="y")
    elif kind == "repl":
        y = b.add(Op.NEGATE, [x], sharding=Sharding.replicated(), id="y")
    else:
        rk = ReduceKind.MAX if kind == "reduce_max" else ReduceKind.SUM
        init = b.constant(np.float32(-np.inf if rk == ReduceKind.MAX else 0), Shape((), dtype),
                          id="init")
        y = b.add(Op.REDUCE, [x, init], {"kind": rk, "dims": (0,)}, id="y")
    g = b.build([y])
    if not with_inputs:
        return g, None
    rng = np.random.default_rng(seed)
    ins = [rng.standard_normal((n0, n1)).astype(np.float32)]
    return g, [_bf16(i) for i in ins] if dtype == DType.BF16 else ins
