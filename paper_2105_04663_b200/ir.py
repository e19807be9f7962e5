"""Static-shape SSA tensor IR consumed by propagation, partitioning and the
B200 executor.

Behavioural contract: ``minispmd/ir.py`` (reference).  Differences by design:

* ``DType.BF16`` is added (reference ``ir.py:19-23`` has F32/S32/U32/PRED
  only).  It is the compute dtype of the large B200 workloads; its host-side
  numpy image is float32 holding bf16-rounded values.
* Shape inference is a per-opcode rule table instead of an if-chain
  (reference ``infer_shape`` ``ir.py:221-412``); the rules, results and the
  ``IncompatibleShapes`` exception are the same.
* Graphs serialise to/from plain JSON (``graph_to_json``/``graph_from_json``)
  so golden fixtures produced from the reference can travel to the GPU box
  without the reference package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import TYPE_CHECKING, Callable, Optional, Sequence

import numpy as np

if TYPE_CHECKING:  # pragma: no cover
    from .sharding import DeviceMesh, Sharding


class DType(Enum):
    F32 = "f32"
    S32 = "s32"
    U32 = "u32"
    PRED = "pred"
    BF16 = "bf16"

    @property
    def is_integer(self) -> bool:
        return self in (DType.S32, DType.U32)

    @property
    def is_float(self) -> bool:
        return self in (DType.F32, DType.BF16)

    @property
    def itemsize(self) -> int:
        return _ITEMSIZE[self]


_ITEMSIZE = {DType.F32: 4, DType.S32: 4, DType.U32: 4, DType.PRED: 1,
             DType.BF16: 2}


def np_dtype(dtype: DType):
    """Host numpy type of an IR dtype (bf16 is carried as float32)."""
    return {DType.F32: np.float32, DType.S32: np.int32, DType.U32: np.uint32,
            DType.PRED: np.bool_, DType.BF16: np.float32}[dtype]


@dataclass(frozen=True)
class Shape:
    dims: tuple[int, ...]
    dtype: DType = DType.F32

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        if min(dims, default=0) < 0:
            raise ValueError(f"negative dimension in shape {dims}")
        object.__setattr__(self, "dims", dims)

    @property
    def rank(self) -> int:
        return len(self.dims)

    @property
    def num_elements(self) -> int:
        return math.prod(self.dims)

    @property
    def nbytes(self) -> int:
        return self.num_elements * self.dtype.itemsize

    def __str__(self) -> str:
        return "%s[%s]" % (self.dtype.value, ",".join(map(str, self.dims)))


class Op(Enum):
    PARAMETER = "parameter"
    CONSTANT = "constant"
    IOTA = "iota"
    PARTITION_ID = "partition-id"
    NEGATE = "negate"
    EXP = "exp"
    RELU = "relu"
    ADD = "add"
    MULTIPLY = "multiply"
    MAXIMUM = "maximum"
    SUBTRACT = "subtract"
    DIVIDE = "divide"
    COMPARE = "compare"
    SELECT = "select"
    BROADCAST = "broadcast"
    RESHAPE = "reshape"
    TRANSPOSE = "transpose"
    REVERSE = "reverse"
    PAD = "pad"
    SLICE = "slice"
    DYNAMIC_SLICE = "dynamic-slice"
    DYNAMIC_UPDATE_SLICE = "dynamic-update-slice"
    CONCAT = "concat"
    REDUCE = "reduce"
    DOT = "dot"
    CONVOLUTION = "convolution"
    ROTATE = "rotate"
    SHIFT = "shift"
    ALL_REDUCE = "all-reduce"
    ALL_GATHER = "all-gather"
    REDUCE_SCATTER = "reduce-scatter"
    ALL_TO_ALL = "all-to-all"
    COLLECTIVE_PERMUTE = "collective-permute"


ELEMENTWISE_UNARY = frozenset({Op.NEGATE, Op.EXP, Op.RELU})
ELEMENTWISE_BINARY = frozenset(
    {Op.ADD, Op.MULTIPLY, Op.MAXIMUM, Op.SUBTRACT, Op.DIVIDE, Op.COMPARE})
COLLECTIVES = frozenset({Op.ALL_REDUCE, Op.ALL_GATHER, Op.REDUCE_SCATTER,
                         Op.ALL_TO_ALL, Op.COLLECTIVE_PERMUTE})


class ReduceKind(Enum):
    SUM = "sum"
    MAX = "max"
    MIN = "min"
    PROD = "prod"


class CompareDirection(Enum):
    EQ = "eq"
    NE = "ne"
    LT = "lt"
    LE = "le"
    GT = "gt"
    GE = "ge"


@dataclass(frozen=True)
class WindowDim:
    """One spatial dim of a convolution window (reference ``ir.py:118-146``)."""

    size: int
    stride: int = 1
    padding_low: int = 0
    padding_high: int = 0
    base_dilation: int = 1
    window_dilation: int = 1

    def __post_init__(self):
        if min(self.size, self.stride) < 1:
            raise ValueError("window size and stride must be >= 1")
        if min(self.base_dilation, self.window_dilation) < 1:
            raise ValueError("dilation factors must be >= 1")
        if min(self.padding_low, self.padding_high) < 0:
            raise ValueError("padding must be >= 0")

    @property
    def effective_window(self) -> int:
        return self.window_dilation * (self.size - 1) + 1

    def dilated_base(self, n: int) -> int:
        return 0 if n <= 0 else self.base_dilation * (n - 1) + 1

    def output_size(self, n: int) -> int:
        span = self.dilated_base(n) + self.padding_low + self.padding_high
        return (span - self.effective_window) // self.stride + 1


@dataclass(frozen=True)
class ConvDims:
    lhs_batch: int
    lhs_feature: int
    lhs_spatial: tuple[int, ...]
    rhs_in_feature: int
    rhs_out_feature: int
    rhs_spatial: tuple[int, ...]
    out_batch: int
    out_feature: int
    out_spatial: tuple[int, ...]


class IncompatibleShapes(Exception):
    pass


@dataclass(frozen=True, eq=False)
class Instruction:
    id: str
    opcode: Op
    operands: tuple[str, ...] = ()
    attrs: dict = field(default_factory=dict)
    shape: Shape = Shape((), DType.F32)
    sharding: Optional["Sharding"] = None

    def with_sharding(self, sharding) -> "Instruction":
        return replace(self, sharding=sharding)


@dataclass(frozen=True, eq=False)
class Graph:
    name: str
    instructions: tuple[Instruction, ...]
    outputs: tuple[str, ...]
    mesh: Optional["DeviceMesh"] = None

    def __post_init__(self):
        object.__setattr__(self, "instructions", tuple(self.instructions))
        object.__setattr__(self, "outputs", tuple(self.outputs))

    def instr(self, id: str) -> Instruction:
        for ins in self.instructions:
            if ins.id == id:
                return ins
        raise KeyError(id)

    @property
    def by_id(self) -> dict[str, Instruction]:
        return {ins.id: ins for ins in self.instructions}

    @property
    def parameters(self) -> tuple[Instruction, ...]:
        return tuple(sorted((i for i in self.instructions
                             if i.opcode == Op.PARAMETER),
                            key=lambda i: i.attrs["index"]))


# ---------------------------------------------------------------------------
# Shape rules (one function per opcode family)
# ---------------------------------------------------------------------------

def _fail(msg: str):
    raise IncompatibleShapes(msg)


def _rule_declared(op, shapes, attrs):
    return attrs["shape"]


def _rule_iota(op, shapes, attrs):
    shape = attrs["shape"]
    if not 0 <= attrs["iota_dimension"] < shape.rank:
        _fail("iota dimension out of range")
    return shape


def _rule_partition_id(op, shapes, attrs):
    return Shape((), DType.S32)


def _rule_same_as_first(op, shapes, attrs):
    return shapes[0]


def _rule_elementwise(op, shapes, attrs):
    first = shapes[0]
    for other in shapes[1:]:
        if other.dims != first.dims:
            _fail(f"{op.value}: operand dims {other.dims} != {first.dims}")
        if other.dtype != first.dtype:
            _fail(f"{op.value}: operand dtypes differ")
    return Shape(first.dims, DType.PRED) if op == Op.COMPARE else first


def _rule_select(op, shapes, attrs):
    pred, a, b = shapes
    if pred.dtype != DType.PRED:
        _fail("select predicate must be pred")
    if pred.dims != a.dims or a != b:
        _fail("select operand shapes must match")
    return a


def _rule_broadcast(op, shapes, attrs):
    src = shapes[0]
    out_dims = tuple(attrs["out_dims"])
    bdims = tuple(attrs["broadcast_dims"])
    if len(bdims) != src.rank:
        _fail("broadcast_dims must map every operand dim")
    for k, d in enumerate(bdims):
        if not (0 <= d < len(out_dims)) or out_dims[d] != src.dims[k]:
            _fail("broadcast dim mismatch")
    if list(bdims) != sorted(set(bdims)):
        _fail("broadcast_dims must be strictly increasing")
    return Shape(out_dims, src.dtype)


def _rule_reshape(op, shapes, attrs):
    out_dims = tuple(attrs["out_dims"])
    if math.prod(out_dims) != shapes[0].num_elements:
        _fail("reshape element count mismatch")
    return Shape(out_dims, shapes[0].dtype)


def _rule_transpose(op, shapes, attrs):
    perm = tuple(attrs["permutation"])
    src = shapes[0]
    if sorted(perm) != list(range(src.rank)):
        _fail("invalid permutation")
    return Shape(tuple(src.dims[p] for p in perm), src.dtype)


def _rule_reverse(op, shapes, attrs):
    src = shapes[0]
    if any(not 0 <= d < src.rank for d in attrs["dims"]):
        _fail("reverse dim out of range")
    return src


def _rule_pad(op, shapes, attrs):
    src, value = shapes
    if value.rank != 0 or value.dtype != src.dtype:
        _fail("pad value must be a scalar of the same dtype")
    lo, hi, it = attrs["low"], attrs["high"], attrs["interior"]
    if not len(lo) == len(hi) == len(it) == src.rank:
        _fail("pad config rank mismatch")
    out = []
    for n, a, b, c in zip(src.dims, lo, hi, it):
        if min(a, b, c) < 0:
            _fail("negative padding not supported")
        out.append(n + max(n - 1, 0) * c + a + b)
    return Shape(tuple(out), src.dtype)


def _rule_slice(op, shapes, attrs):
    src = shapes[0]
    out = []
    for n, b, e, s in zip(src.dims, attrs["starts"], attrs["limits"],
                          attrs["strides"]):
        if s < 1 or not (0 <= b <= e <= n):
            _fail("invalid slice bounds")
        out.append(-(-(e - b) // s))
    return Shape(tuple(out), src.dtype)


def _rule_dynamic_slice(op, shapes, attrs):
    src = shapes[0]
    sizes = tuple(attrs["sizes"])
    if len(sizes) != src.rank or len(shapes) != src.rank + 1:
        _fail("dynamic-slice arity mismatch")
    if any(s.rank != 0 or not s.dtype.is_integer for s in shapes[1:]):
        _fail("dynamic-slice indices must be integer scalars")
    if any(not 0 <= z <= n for z, n in zip(sizes, src.dims)):
        _fail("dynamic-slice size exceeds operand")
    return Shape(sizes, src.dtype)


def _rule_dynamic_update_slice(op, shapes, attrs):
    src, upd = shapes[0], shapes[1]
    if upd.rank != src.rank or upd.dtype != src.dtype:
        _fail("dynamic-update-slice operand mismatch")
    if any(u > n for u, n in zip(upd.dims, src.dims)):
        _fail("update larger than operand")
    if len(shapes) != src.rank + 2:
        _fail("dynamic-update-slice arity mismatch")
    return src


def _rule_concat(op, shapes, attrs):
    axis = attrs["dim"]
    first = shapes[0]
    total = 0
    for s in shapes:
        if s.rank != first.rank or s.dtype != first.dtype:
            _fail("concat rank/dtype mismatch")
        if any(s.dims[i] != first.dims[i] for i in range(s.rank) if i != axis):
            _fail("concat non-concat dim mismatch")
        total += s.dims[axis]
    dims = list(first.dims)
    dims[axis] = total
    return Shape(tuple(dims), first.dtype)


def _rule_reduce(op, shapes, attrs):
    src, init = shapes
    rdims = set(attrs["dims"])
    if init.rank != 0 or init.dtype != src.dtype:
        _fail("reduce init must be scalar of operand dtype")
    if any(not 0 <= d < src.rank for d in rdims):
        _fail("reduce dim out of range")
    return Shape(tuple(n for i, n in enumerate(src.dims) if i not in rdims),
                 src.dtype)


def dot_dim_lists(attrs, lhs_rank: int, rhs_rank: int):
    """(lb, rb, lc, rc, lfree, rfree) of a Dot; result dims are
    [batch..., lhs-free..., rhs-free...] (reference ``ir.py:353-358``)."""
    lb, rb = list(attrs["lhs_batch"]), list(attrs["rhs_batch"])
    lc, rc = list(attrs["lhs_contracting"]), list(attrs["rhs_contracting"])
    lfree = [d for d in range(lhs_rank) if d not in lb and d not in lc]
    rfree = [d for d in range(rhs_rank) if d not in rb and d not in rc]
    return lb, rb, lc, rc, lfree, rfree


def _rule_dot(op, shapes, attrs):
    lhs, rhs = shapes
    if lhs.dtype != rhs.dtype:
        _fail("dot dtype mismatch")
    lb, rb, lc, rc, lfree, rfree = dot_dim_lists(attrs, lhs.rank, rhs.rank)
    if len(lb) != len(rb) or len(lc) != len(rc):
        _fail("dot dim list length mismatch")
    if any(lhs.dims[a] != rhs.dims[b] for a, b in zip(lb + lc, rb + rc)):
        _fail("dot batch/contracting size mismatch")
    dims = [lhs.dims[d] for d in lb + lfree] + [rhs.dims[d] for d in rfree]
    return Shape(tuple(dims), lhs.dtype)


def _rule_convolution(op, shapes, attrs):
    lhs, rhs = shapes
    cd: ConvDims = attrs["conv_dims"]
    window = tuple(attrs["window"])
    if lhs.dtype != rhs.dtype:
        _fail("convolution dtype mismatch")
    if len(window) != len(cd.lhs_spatial):
        _fail("window config rank mismatch")
    if lhs.dims[cd.lhs_feature] != rhs.dims[cd.rhs_in_feature]:
        _fail("convolution feature size mismatch")
    out = [0] * lhs.rank
    out[cd.out_batch] = lhs.dims[cd.lhs_batch]
    out[cd.out_feature] = rhs.dims[cd.rhs_out_feature]
    for od, ld, rd, w in zip(cd.out_spatial, cd.lhs_spatial, cd.rhs_spatial,
                             window):
        if rhs.dims[rd] != w.size:
            _fail("window size disagrees with rhs spatial dim")
        n = w.output_size(lhs.dims[ld])
        if n <= 0:
            _fail("non-positive convolution output size")
        out[od] = n
    return Shape(tuple(out), lhs.dtype)


def _group_factor(attrs) -> int:
    return len(attrs["subgroups"][0])


def _rule_all_gather(op, shapes, attrs):
    dims = list(shapes[0].dims)
    dims[attrs["dim"]] *= _group_factor(attrs)
    return Shape(tuple(dims), shapes[0].dtype)


def _rule_reduce_scatter(op, shapes, attrs):
    dims = list(shapes[0].dims)
    f = _group_factor(attrs)
    if dims[attrs["dim"]] % f:
        _fail("reduce-scatter dim not divisible by group size")
    dims[attrs["dim"]] //= f
    return Shape(tuple(dims), shapes[0].dtype)


def _rule_all_to_all(op, shapes, attrs):
    dims = list(shapes[0].dims)
    f = _group_factor(attrs)
    if dims[attrs["split_dim"]] % f:
        _fail("all-to-all split dim not divisible")
    dims[attrs["split_dim"]] //= f
    dims[attrs["concat_dim"]] *= f
    return Shape(tuple(dims), shapes[0].dtype)


_SHAPE_RULES: dict[Op, Callable] = {
    Op.PARAMETER: _rule_declared,
    Op.CONSTANT: _rule_declared,
    Op.IOTA: _rule_iota,
    Op.PARTITION_ID: _rule_partition_id,
    Op.SELECT: _rule_select,
    Op.BROADCAST: _rule_broadcast,
    Op.RESHAPE: _rule_reshape,
    Op.TRANSPOSE: _rule_transpose,
    Op.REVERSE: _rule_reverse,
    Op.PAD: _rule_pad,
    Op.SLICE: _rule_slice,
    Op.DYNAMIC_SLICE: _rule_dynamic_slice,
    Op.DYNAMIC_UPDATE_SLICE: _rule_dynamic_update_slice,
    Op.CONCAT: _rule_concat,
    Op.REDUCE: _rule_reduce,
    Op.DOT: _rule_dot,
    Op.CONVOLUTION: _rule_convolution,
    Op.ROTATE: _rule_same_as_first,
    Op.SHIFT: _rule_same_as_first,
    Op.ALL_REDUCE: _rule_same_as_first,
    Op.COLLECTIVE_PERMUTE: _rule_same_as_first,
    Op.ALL_GATHER: _rule_all_gather,
    Op.REDUCE_SCATTER: _rule_reduce_scatter,
    Op.ALL_TO_ALL: _rule_all_to_all,
}
_SHAPE_RULES.update({o: _rule_same_as_first for o in ELEMENTWISE_UNARY})
_SHAPE_RULES.update({o: _rule_elementwise for o in ELEMENTWISE_BINARY})


def infer_shape(opcode: Op, operand_shapes: Sequence[Shape], attrs: dict) -> Shape:
    """Output shape of ``opcode`` or :class:`IncompatibleShapes`."""
    rule = _SHAPE_RULES.get(opcode)
    if rule is None:
        _fail(f"unknown opcode {opcode}")
    return rule(opcode, list(operand_shapes), attrs)


_FIXED_ARITY = {Op.PARAMETER: 0, Op.CONSTANT: 0, Op.IOTA: 0,
                Op.PARTITION_ID: 0, Op.SELECT: 3, Op.PAD: 2, Op.REDUCE: 2,
                Op.DOT: 2, Op.CONVOLUTION: 2, Op.SHIFT: 2}
_FIXED_ARITY.update({o: 1 for o in ELEMENTWISE_UNARY})
_FIXED_ARITY.update({o: 2 for o in ELEMENTWISE_BINARY})


def validate_graph(graph: Graph) -> list[str]:
    """Diagnostics for every violated invariant (reference ``ir.py:429-465``)."""
    problems: list[str] = []
    defined: dict[str, Instruction] = {}
    for ins in graph.instructions:
        if ins.id in defined:
            problems.append(f"{ins.id}: duplicate definition")
            continue
        problems += [f"{ins.id}: use-before-def of {o}"
                     for o in ins.operands if o not in defined]
        arity = _FIXED_ARITY.get(ins.opcode)
        if arity is not None and len(ins.operands) != arity:
            problems.append(f"{ins.id}: wrong operand count for "
                            f"{ins.opcode.value}")
        elif all(o in defined for o in ins.operands):
            try:
                want = infer_shape(ins.opcode,
                                   [defined[o].shape for o in ins.operands],
                                   ins.attrs)
                if want != ins.shape:
                    problems.append(f"{ins.id}: shape mismatch: declared "
                                    f"{ins.shape}, inferred {want}")
            except IncompatibleShapes as e:
                problems.append(f"{ins.id}: shape mismatch: {e}")
        s = ins.sharding
        if s is not None and s.tile_dims is not None \
                and s.data_rank != ins.shape.rank:
            problems.append(f"{ins.id}: sharding rank does not match shape rank")
        defined[ins.id] = ins
    problems += [f"output {o} is not defined" for o in graph.outputs
                 if o not in defined]
    return problems


class GraphBuilder:
    """Builds a valid Graph; ids default to ``<opcode>.<counter>``."""

    def __init__(self, name: str = "main", mesh=None):
        self.name = name
        self.mesh = mesh
        self._instrs: list[Instruction] = []
        self._index: dict[str, Instruction] = {}
        self._count = 0
        self._param_count = 0

    def shape_of(self, id: str) -> Shape:
        return self._index[id].shape

    def add(self, opcode: Op, operands: Sequence[str] = (),
            attrs: Optional[dict] = None, sharding=None,
            id: Optional[str] = None) -> str:
        attrs = dict(attrs or {})
        shape = infer_shape(opcode, [self._index[o].shape for o in operands],
                            attrs)
        if id is None:
            self._count += 1
            id = "%s.%d" % (opcode.value.replace("-", "_"), self._count)
        ins = Instruction(id, opcode, tuple(operands), attrs, shape, sharding)
        self._instrs.append(ins)
        self._index[id] = ins
        return id

    def set_sharding(self, id: str, sharding) -> None:
        """Attach an annotation to an already-added instruction."""
        for k, ins in enumerate(self._instrs):
            if ins.id == id:
                self._instrs[k] = self._index[id] = ins.with_sharding(sharding)
                return
        raise KeyError(id)

    def parameter(self, shape: Shape, sharding=None, id=None) -> str:
        idx = self._param_count
        self._param_count += 1
        return self.add(Op.PARAMETER, attrs={"index": idx, "shape": shape},
                        sharding=sharding, id=id)

    def constant(self, literal, shape: Shape, sharding=None, id=None) -> str:
        return self.add(Op.CONSTANT, attrs={"literal": literal, "shape": shape},
                        sharding=sharding, id=id)

    def build(self, outputs: Sequence[str]) -> Graph:
        g = Graph(self.name, tuple(self._instrs), tuple(outputs), self.mesh)
        problems = validate_graph(g)
        if problems:
            raise ValueError("invalid graph: " + "; ".join(problems))
        return g


# ---------------------------------------------------------------------------
# JSON serialisation (fixtures; not part of the reference API)
# ---------------------------------------------------------------------------

def _attr_to_json(key, v):
    if isinstance(v, Shape):
        return {"__shape__": [list(v.dims), v.dtype.value]}
    if isinstance(v, (ReduceKind, CompareDirection)):
        return {"__enum__": [type(v).__name__, v.value]}
    if isinstance(v, ConvDims):
        return {"__convdims__": {k: (list(x) if isinstance(x, tuple) else x)
                                 for k, x in v.__dict__.items()}}
    if key == "window":
        return {"__window__": [w.__dict__ for w in v]}
    if key == "literal":
        arr = np.asarray(v)
        lst = arr.astype(np.float64).tolist() if arr.dtype.kind == "f" \
            else arr.tolist()
        return {"__literal__": [list(arr.shape), str(arr.dtype), lst]}
    if isinstance(v, tuple):
        return [_attr_to_json(None, x) for x in v]
    if isinstance(v, (np.integer,)):
        return int(v)
    return v


def _attr_from_json(key, v):
    if isinstance(v, dict):
        if "__shape__" in v:
            dims, dt = v["__shape__"]
            return Shape(tuple(dims), DType(dt))
        if "__enum__" in v:
            cls, val = v["__enum__"]
            return {"ReduceKind": ReduceKind,
                    "CompareDirection": CompareDirection}[cls](val)
        if "__convdims__" in v:
            d = v["__convdims__"]
            return ConvDims(**{k: (tuple(x) if isinstance(x, list) else x)
                               for k, x in d.items()})
        if "__window__" in v:
            return tuple(WindowDim(**w) for w in v["__window__"])
        if "__literal__" in v:
            shape, dt, lst = v["__literal__"]
            return np.asarray(lst, dtype=np.dtype(dt)).reshape(shape)
    if isinstance(v, list):
        return tuple(_attr_from_json(None, x) if not isinstance(x, list)
                     else tuple(_attr_from_json(None, y) for y in x)
                     for x in v)
    return v


def instruction_to_json(ins: Instruction) -> dict:
    d = {"id": ins.id, "op": ins.opcode.value, "operands": list(ins.operands),
         "attrs": {k: _attr_to_json(k, v) for k, v in sorted(ins.attrs.items())},
         "shape": [list(ins.shape.dims), ins.shape.dtype.value]}
    if ins.sharding is not None:
        d["sharding"] = ins.sharding.format()
    return d


def instruction_from_json(d: dict) -> Instruction:
    from .sharding import Sharding
    attrs = {k: _attr_from_json(k, v) for k, v in d["attrs"].items()}
    s = d.get("sharding")
    return Instruction(d["id"], Op(d["op"]), tuple(d["operands"]), attrs,
                       Shape(tuple(d["shape"][0]), DType(d["shape"][1])),
                       Sharding.parse(s) if s is not None else None)


def graph_to_json(g: Graph) -> dict:
    out = {"name": g.name, "outputs": list(g.outputs),
           "instructions": [instruction_to_json(i) for i in g.instructions]}
    if g.mesh is not None:
        out["mesh"] = [list(g.mesh.mesh_dims), list(g.mesh.device_ids)]
    return out


def graph_from_json(d: dict) -> Graph:
    from .sharding import DeviceMesh
    mesh = DeviceMesh(tuple(d["mesh"][0]), tuple(d["mesh"][1])) \
        if "mesh" in d else None
    return Graph(d["name"], tuple(instruction_from_json(i)
                                  for i in d["instructions"]),
                 tuple(d["outputs"]), mesh)
