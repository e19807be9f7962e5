"""Sharding completion (GSPMD auto-completion) over a dataflow graph.

Behavioural contract: ``minispmd/propagation.py`` (reference).  The result --
every instruction's final sharding and the change log -- is bit-identical
with the reference; golden fixtures in ``tests/golden`` pin it.

Algorithm (reference ``propagate`` ``propagation.py:420-491``): refinement-only
updates (``_State.try_update`` ``:393-417``) iterate to a fixed point.  Each
iteration visits priority tiers 0..4 and, *per tier*, runs a forward sweep in
program order followed by a backward sweep in reverse order
(``:445-478``; SPEC.md's "all forward then all backward" is not what the code
does).  Tier membership (``:163-194``):

====  ==================================  ===============================
tier  forward                             backward
====  ==================================  ===============================
0     elementwise + select                elementwise + select
1     reduce, transpose, reverse          reduce, transpose, reverse, broadcast
2     dot, convolution                    dot, convolution
3     reshape, pad, slice, concat, d-s    reshape, pad, slice, concat, d-s
4     broadcast                           --
====  ==================================  ===============================

The B200 build organises the per-opcode rules as two tables of small
functions (one forward, one backward) instead of two if-chains.
"""

from __future__ import annotations

import dataclasses
from typing import Callable, Optional, Sequence

from .ir import (ELEMENTWISE_BINARY, ELEMENTWISE_UNARY, ConvDims, Graph,
                 Instruction, Op, dot_dim_lists)
from .sharding import Sharding, merge_shardings


class ConflictingUserAnnotations(Exception):
    """Two user annotations pin one value to incompatible shardings."""


@dataclasses.dataclass
class Change:
    iteration: int
    instruction: str
    old: Optional[str]
    new: str
    rule: str
    direction: str

    def to_json(self) -> dict:
        return dataclasses.asdict(self)


@dataclasses.dataclass
class PropagationReport:
    iterations: int
    final_shardings: dict[str, str]
    changes: list[Change]

    def to_json(self) -> dict:
        return {"iterations": self.iterations,
                "final_shardings": dict(self.final_shardings),
                "changes": [c.to_json() for c in self.changes]}


# ---------------------------------------------------------------------------
# Operand-dim -> result-dim correspondences
# ---------------------------------------------------------------------------

def dot_operand_map(ins: Instruction, k: int, operand_rank: int) -> dict[int, int]:
    """Operand ``k`` dims -> Dot result dims [batch, lhs-free, rhs-free]
    (reference ``propagation.py:67-89``); contracting dims are absent."""
    attrs = ins.attrs
    batch = list(attrs["lhs_batch"] if k == 0 else attrs["rhs_batch"])
    contr = list(attrs["lhs_contracting"] if k == 0 else attrs["rhs_contracting"])
    free = [d for d in range(operand_rank) if d not in batch and d not in contr]
    base = len(batch)
    if k == 1:
        base += ins.shape.rank - len(batch) - len(free)   # lhs-free count
    m = {d: pos for pos, d in enumerate(batch)}
    m.update({d: base + pos for pos, d in enumerate(free)})
    return m


def conv_operand_map(ins: Instruction, k: int) -> dict[int, int]:
    """Convolution operand dims -> result dims (reference ``:92-99``)."""
    cd: ConvDims = ins.attrs["conv_dims"]
    if k == 1:
        return {cd.rhs_out_feature: cd.out_feature}
    m = {cd.lhs_batch: cd.out_batch}
    m.update(zip(cd.lhs_spatial, cd.out_spatial))
    return m


def reshape_groups(in_dims: Sequence[int],
                   out_dims: Sequence[int]) -> list[tuple[list[int], list[int]]]:
    """Greedy pairing of input/output dim runs with equal element counts,
    trailing size-1 dims absorbed (reference ``propagation.py:102-134``)."""
    n_in, n_out = len(in_dims), len(out_dims)

    def size(dims, n, k):
        return dims[k] if k < n else 1

    groups = []
    i = j = 0
    while i < n_in or j < n_out:
        gi, gj = [i], [j]
        pi, pj = size(in_dims, n_in, i), size(out_dims, n_out, j)
        while pi != pj:
            if pi < pj:
                i += 1
                gi.append(i)
                pi *= in_dims[i]
            else:
                j += 1
                gj.append(j)
                pj *= out_dims[j]
        while i + 1 < n_in and in_dims[i + 1] == 1:
            i += 1
            gi.append(i)
        while j + 1 < n_out and out_dims[j + 1] == 1:
            j += 1
            gj.append(j)
        groups.append(([d for d in gi if d < n_in], [d for d in gj if d < n_out]))
        i += 1
        j += 1
    return groups


def reshape_dim_map(s: Sharding, in_dims: Sequence[int],
                    out_dims: Sequence[int]) -> dict[int, int]:
    """Lead-dim correspondences of a reshape that a tiling survives: exact
    1:1 dims, or lead dims both divisible by the lead tiling
    (reference ``:137-152``)."""
    m: dict[int, int] = {}
    for gin, gout in reshape_groups(in_dims, out_dims):
        if not (gin and gout):
            continue
        a, b = gin[0], gout[0]
        if len(gin) == 1 and len(gout) == 1 and in_dims[a] == out_dims[b]:
            m[a] = b
            continue
        t = s.tiles(a)
        if t > 1 and in_dims[a] % t == 0 and out_dims[b] % t == 0:
            m[a] = b
    return m


def untouched_dims_map(ins: Instruction, operand_dims: Sequence[int]) -> dict[int, int]:
    """Identity map over the dims a slice-like op leaves intact
    (reference ``:197-221``)."""
    a = ins.attrs
    rank = len(operand_dims)
    op = ins.opcode
    if op == Op.SLICE:
        ok = lambda d: (a["starts"][d] == 0 and a["limits"][d] == operand_dims[d]
                        and a["strides"][d] == 1)
    elif op == Op.PAD:
        ok = lambda d: a["low"][d] == 0 and a["high"][d] == 0 and a["interior"][d] == 0
    elif op == Op.CONCAT:
        ok = lambda d: d != a["dim"]
    elif op == Op.DYNAMIC_SLICE:
        ok = lambda d: a["sizes"][d] == operand_dims[d]
    else:
        ok = lambda d: True
    return {d: d for d in range(rank) if ok(d)}


# ---------------------------------------------------------------------------
# Rule tables
# ---------------------------------------------------------------------------

_ELEMENTWISE = ELEMENTWISE_UNARY | ELEMENTWISE_BINARY | {Op.SELECT}
_SLICE_LIKE = (Op.SLICE, Op.PAD, Op.CONCAT, Op.DYNAMIC_SLICE)

FORWARD_TIER: dict[Op, int] = {}
BACKWARD_TIER: dict[Op, int] = {}
for _op in _ELEMENTWISE:
    FORWARD_TIER[_op] = BACKWARD_TIER[_op] = 0
for _op in (Op.REDUCE, Op.TRANSPOSE, Op.REVERSE):
    FORWARD_TIER[_op] = BACKWARD_TIER[_op] = 1
BACKWARD_TIER[Op.BROADCAST] = 1
for _op in (Op.DOT, Op.CONVOLUTION):
    FORWARD_TIER[_op] = BACKWARD_TIER[_op] = 2
for _op in (Op.RESHAPE,) + _SLICE_LIKE:
    FORWARD_TIER[_op] = BACKWARD_TIER[_op] = 3
FORWARD_TIER[Op.BROADCAST] = 4


def _tiled(s: Optional[Sharding]) -> bool:
    return s is not None and not s.is_replicated


def _fold(candidates) -> Optional[Sharding]:
    """First candidate wins; later ones refine it when mergeable."""
    acc = None
    for c in candidates:
        if acc is None:
            acc = c
        else:
            acc = merge_shardings(acc, c) or acc
    return acc


def _nonrepl(c: Optional[Sharding]) -> Optional[Sharding]:
    return None if c is None or c.is_replicated else c


def _fwd_elementwise(ins, shs, shapes):
    return _fold(s for s in shs if _tiled(s))


def _fwd_broadcast(ins, shs, shapes):
    s = shs[0]
    if not _tiled(s):
        return None
    bd = tuple(ins.attrs["broadcast_dims"])
    return s.project(dict(enumerate(bd)), ins.shape.rank)


def _fwd_transpose(ins, shs, shapes):
    s = shs[0]
    if not _tiled(s):
        return None
    perm = tuple(ins.attrs["permutation"])
    return s.project({p: j for j, p in enumerate(perm)}, ins.shape.rank)


def _fwd_reverse(ins, shs, shapes):
    return shs[0] if _tiled(shs[0]) else None


def _kept_map(ins, operand_rank):
    rd = set(ins.attrs["dims"])
    return {d: pos for pos, d in enumerate(d for d in range(operand_rank)
                                           if d not in rd)}


def _fwd_reduce(ins, shs, shapes):
    s = shs[0]
    if not _tiled(s):
        return None
    return s.project(_kept_map(ins, shapes[0].rank), ins.shape.rank)


def _fwd_slice_like(ins, shs, shapes):
    n = len(shs) if ins.opcode == Op.CONCAT else 1
    cands = (_nonrepl(shs[k].project(untouched_dims_map(ins, shapes[k].dims),
                                     ins.shape.rank))
             for k in range(n) if _tiled(shs[k]))
    return _fold(c for c in cands if c is not None)


def _fwd_reshape(ins, shs, shapes):
    s = shs[0]
    if not _tiled(s):
        return None
    m = reshape_dim_map(s, shapes[0].dims, ins.shape.dims)
    return _nonrepl(s.project(m, ins.shape.rank)) if m else None


def _fwd_contraction(mapper):
    def rule(ins, shs, shapes):
        cands = (_nonrepl(shs[k].project(mapper(ins, k, shapes[k].rank),
                                         ins.shape.rank))
                 for k in (0, 1) if _tiled(shs[k]))
        return _fold(c for c in cands if c is not None)
    return rule


FORWARD_RULES: dict[Op, Callable] = {
    Op.BROADCAST: _fwd_broadcast,
    Op.TRANSPOSE: _fwd_transpose,
    Op.REVERSE: _fwd_reverse,
    Op.REDUCE: _fwd_reduce,
    Op.RESHAPE: _fwd_reshape,
    Op.DOT: _fwd_contraction(dot_operand_map),
    Op.CONVOLUTION: _fwd_contraction(lambda ins, k, r: conv_operand_map(ins, k)),
}
FORWARD_RULES.update({o: _fwd_elementwise for o in _ELEMENTWISE})
FORWARD_RULES.update({o: _fwd_slice_like for o in _SLICE_LIKE})


def _pull(s: Sharding, fwd_map: dict[int, int], operand_rank: int):
    """Invert an operand->result map and project the result sharding back."""
    return _nonrepl(s.project({r: o for o, r in fwd_map.items()}, operand_rank))


def _bwd_same(ins, s, k, shape):
    return s


def _bwd_broadcast(ins, s, k, shape):
    bd = tuple(ins.attrs["broadcast_dims"])
    return _pull(s, dict(enumerate(bd)), shape.rank)


def _bwd_transpose(ins, s, k, shape):
    perm = tuple(ins.attrs["permutation"])
    return _pull(s, {p: j for j, p in enumerate(perm)}, shape.rank)


def _bwd_reduce(ins, s, k, shape):
    return _pull(s, _kept_map(ins, shape.rank), shape.rank) if k == 0 else None


def _bwd_slice_like(ins, s, k, shape):
    if k != 0 and ins.opcode in (Op.PAD, Op.DYNAMIC_SLICE):
        return None
    if shape.rank != ins.shape.rank:
        return None
    return _pull(s, untouched_dims_map(ins, shape.dims), shape.rank)


def _bwd_reshape(ins, s, k, shape):
    m = reshape_dim_map(s, ins.shape.dims, shape.dims)
    return _nonrepl(s.project(m, shape.rank)) if m else None


def _bwd_dot(ins, s, k, shape):
    return _pull(s, dot_operand_map(ins, k, shape.rank), shape.rank) \
        if k in (0, 1) else None


def _bwd_conv(ins, s, k, shape):
    return _pull(s, conv_operand_map(ins, k), shape.rank) if k in (0, 1) else None


BACKWARD_RULES: dict[Op, Callable] = {
    Op.BROADCAST: _bwd_broadcast,
    Op.TRANSPOSE: _bwd_transpose,
    Op.REVERSE: _bwd_same,
    Op.REDUCE: _bwd_reduce,
    Op.RESHAPE: _bwd_reshape,
    Op.DOT: _bwd_dot,
    Op.CONVOLUTION: _bwd_conv,
}
BACKWARD_RULES.update({o: _bwd_same for o in _ELEMENTWISE})
BACKWARD_RULES.update({o: _bwd_slice_like for o in _SLICE_LIKE})


def infer_forward(ins: Instruction, operand_shardings, operand_ranks,
                  operand_dims) -> Optional[Sharding]:
    """Candidate result sharding from operand shardings (reference ``:224-315``)."""
    rule = FORWARD_RULES.get(ins.opcode)
    if rule is None:
        return None
    from .ir import Shape
    shapes = [Shape(tuple(d)) for d in operand_dims]
    return rule(ins, list(operand_shardings), shapes)


def infer_backward(ins: Instruction, result_sharding, k: int, operand_rank: int,
                   operand_dims) -> Optional[Sharding]:
    """Candidate sharding for operand ``k`` (reference ``:318-360``)."""
    if not _tiled(result_sharding):
        return None
    rule = BACKWARD_RULES.get(ins.opcode)
    if rule is None:
        return None
    from .ir import Shape
    return rule(ins, result_sharding, k, Shape(tuple(operand_dims)))


# ---------------------------------------------------------------------------
# Fixed-point driver
# ---------------------------------------------------------------------------

def _same_placement(a: Sharding, b: Sharding, dims, devices) -> bool:
    for d in dims:
        t = a.tiles(d)
        if t != b.tiles(d):
            return False
        if t > 1 and any(a.coord(dev, d) != b.coord(dev, d) for dev in devices):
            return False
    return True


class _Completion:
    """Working shardings plus the user annotations that constrain them."""

    def __init__(self, graph: Graph):
        self.current: dict[str, Optional[Sharding]] = {}
        self.pinned: dict[str, Sharding] = {}
        for ins in graph.instructions:
            if ins.sharding is None:
                self.current[ins.id] = None
            else:
                self.pinned[ins.id] = ins.sharding
                self.current[ins.id] = ins.sharding.clear_unspecified()

    def offer(self, ins_id: str, cand: Optional[Sharding], rank: int):
        """Refine ``ins_id`` with ``cand``; returns (old, new) on change."""
        if cand is None or cand.is_replicated:
            return None
        cand = cand.clear_unspecified()
        if cand.data_rank != rank:
            return None
        old = self.current[ins_id]
        if old is None:
            new = cand
        else:
            new = merge_shardings(old, cand)
            if new is None or new == old:
                return None
        pin = self.pinned.get(ins_id)
        if pin is not None:
            fixed = [d for d in range(rank) if d not in pin.unspecified_dims]
            base = pin.clear_unspecified()
            devs = new.devices if base.is_replicated else base.devices
            if not _same_placement(base, new, fixed, devs):
                return None
        self.current[ins_id] = new
        return old, new


def propagate(graph: Graph, use_priorities: bool = True,
              max_iterations: Optional[int] = None):
    """Complete shardings over ``graph``; returns ``(annotated, report)``.

    ``use_priorities=False`` runs every rule in one tier (plain topological
    order) -- the regression mode the reference keeps to show why tiers exist.
    """
    st = _Completion(graph)
    by_id = graph.by_id
    order = list(graph.instructions)
    limit = max_iterations or max(10, 10 * len(order))
    tiers = (0, 1, 2, 3, 4) if use_priorities else (None,)
    log: list[Change] = []
    it = 0

    def record(iteration, target, upd, ins, direction):
        old, new = upd
        log.append(Change(iteration, target, old.format() if old else None,
                          new.format(), ins.opcode.value, direction))

    while it < limit:
        it += 1
        progress = False
        for tier in tiers:
            for ins in order:
                t = FORWARD_TIER.get(ins.opcode)
                if t is None or (tier is not None and t != tier):
                    continue
                ops = [by_id[o] for o in ins.operands]
                cand = FORWARD_RULES[ins.opcode](
                    ins, [st.current[o.id] for o in ops], [o.shape for o in ops])
                upd = st.offer(ins.id, cand, ins.shape.rank)
                if upd:
                    progress = True
                    record(it, ins.id, upd, ins, "forward")
            for ins in reversed(order):
                t = BACKWARD_TIER.get(ins.opcode)
                if t is None or (tier is not None and t != tier):
                    continue
                res = st.current[ins.id]
                if res is None or res.is_replicated:
                    continue
                rule = BACKWARD_RULES[ins.opcode]
                for k, oid in enumerate(ins.operands):
                    opnd = by_id[oid]
                    upd = st.offer(oid, rule(ins, res, k, opnd.shape),
                                   opnd.shape.rank)
                    if upd:
                        progress = True
                        record(it, oid, upd, ins, "backward")
        if not progress:
            break

    annotated, final = [], {}
    for ins in order:
        s = (st.current[ins.id] or Sharding.replicated()).clear_unspecified()
        annotated.append(ins.with_sharding(s))
        final[ins.id] = s.format()
    return (Graph(graph.name, tuple(annotated), graph.outputs, graph.mesh),
            PropagationReport(it, final, log))
