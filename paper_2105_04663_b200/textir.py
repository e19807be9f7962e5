"""Text form of graphs (reference textir.py:1-630).

    graph @name (mesh=[2,2]) {
      %x = f32[8,16] parameter(0), sharding={devices=[2,1]0,1}
      %y = f32[8,16] relu(%x)
      return %y
    }

``print_graph`` emits byte-identical text to the reference (pinned against
the reference's own printout of every golden graph and SPMD program);
``parse_graph`` accepts the same grammar -- including the headerless
instruction list -- and reports ``ParseError`` at the same line/column.
Float literals round-trip exactly (shortest repr).  Host-side tooling: not
on the execution path.
"""

from __future__ import annotations

import re
from typing import Iterator, Optional

import numpy as np

from .ir import (CompareDirection, ConvDims, DType, Graph, Instruction, Op, ReduceKind,
                 Shape, WindowDim, np_dtype, validate_graph)
from .sharding import DeviceMesh, Sharding, ShardingError


class ParseError(Exception):
    """(reference textir.py:38-42)"""

    def __init__(self, message: str, line: int, column: int):
        super().__init__(f"line {line}, column {column}: {message}")
        self.line = line
        self.column = column


OPCODES = {op.value: op for op in Op}
DTYPES = {dt.value: dt for dt in DType}

# attributes the printer leaves out: recoverable from the result shape
DERIVED = frozenset({"shape", "out_dims"})
# print order (reference textir.py:70-77); unknown names sort last, by name
ORDER = ("index", "iota_dimension", "direction", "kind", "dim", "dims", "broadcast_dims",
         "permutation", "low", "high", "interior", "starts", "limits", "strides", "sizes",
         "lhs_batch", "lhs_contracting", "rhs_batch", "rhs_contracting", "conv_dims",
         "window", "amount", "fill", "split_dim", "concat_dim", "subgroups", "pairs",
         "literal")
RANK = {name: i for i, name in enumerate(ORDER)}

CONV_FIELDS = ("lhs_batch", "lhs_feature", "lhs_spatial", "rhs_in_feature",
               "rhs_out_feature", "rhs_spatial", "out_batch", "out_feature", "out_spatial")
WINDOW_FIELDS = ("size", "stride", "padding_low", "padding_high", "base_dilation",
                 "window_dilation")
WINDOW_DEFAULTS = {"stride": 1, "padding_low": 0, "padding_high": 0, "base_dilation": 1,
                   "window_dilation": 1}


# ---------------------------------------------------------------------------
# printing
# ---------------------------------------------------------------------------

def _num(x) -> str:
    if isinstance(x, (bool, np.bool_)):
        return "true" if x else "false"
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    f = float(x)
    if f != f:
        return "nan"
    if f in (float("inf"), float("-inf")):
        return "inf" if f > 0 else "-inf"
    s = repr(f)
    return s if any(c in s for c in ".en") else s + ".0"


def _ints(vals) -> str:
    return "[" + ",".join(str(int(v)) for v in vals) + "]"


def _nested(arr: np.ndarray) -> str:
    if arr.ndim == 0:
        return _num(arr[()])
    return "[" + ",".join(_nested(arr[i]) for i in range(arr.shape[0])) + "]"


def _struct(pairs) -> str:
    return "{" + ",".join(f"{k}={_ints(v) if isinstance(v, (tuple, list)) else int(v)}"
                          for k, v in pairs) + "}"


def _attr_text(name: str, v) -> str:
    if name == "literal":
        return _nested(np.asarray(v))
    if isinstance(v, (CompareDirection, ReduceKind)):
        return v.value
    if name in ("subgroups", "pairs"):
        return "[" + ",".join(_ints(g) for g in v) + "]"
    if name == "conv_dims":
        return _struct((f, getattr(v, f)) for f in CONV_FIELDS)
    if name == "window":
        return "[" + ",".join(_struct((f, getattr(w, f)) for f in WINDOW_FIELDS)
                              for w in v) + "]"
    if name == "fill":
        return _num(v)
    if isinstance(v, (tuple, list)):
        return _ints(v)
    return str(int(v))


def print_instruction(ins: Instruction) -> str:
    """(reference textir.py:500-519)"""
    if ins.opcode == Op.PARAMETER:
        head = f"parameter({ins.attrs['index']})"
        hidden = DERIVED | {"index"}
    else:
        head = f"{ins.opcode.value}({', '.join('%' + o for o in ins.operands)})"
        hidden = DERIVED
    names = sorted((k for k in ins.attrs if k not in hidden),
                   key=lambda k: (RANK.get(k, 99), k))
    parts = [f"%{ins.id} = {ins.shape} {head}"]
    parts += [f"{k}={_attr_text(k, ins.attrs[k])}" for k in names]
    if ins.sharding is not None:
        parts.append("sharding={%s}" % ins.sharding.format())
    return ", ".join(parts)


def print_graph(graph: Graph) -> str:
    """(reference textir.py:522-538)"""
    head = f"graph @{graph.name}"
    if graph.mesh is not None:
        ids = tuple(graph.mesh.device_ids)
        custom = "" if ids == tuple(range(len(ids))) else ",".join(map(str, ids))
        head += f" (mesh={_ints(graph.mesh.mesh_dims)}{custom})"
    body = [f"  {print_instruction(i)}" for i in graph.instructions]
    ret = "  return " + ", ".join("%" + o for o in graph.outputs)
    return "\n".join([head + " {"] + body + [ret, "}"]) + "\n"


# ---------------------------------------------------------------------------
# tokens
# ---------------------------------------------------------------------------

_LEX = re.compile(r"""
      (?P<ws>[ \t]+)
    | (?P<comment>//[^\n]*)
    | (?P<newline>\n)
    | (?P<number>-?\d+\.\d+(?:[eE][-+]?\d+)?|-?\d+[eE][-+]?\d+|-?inf|nan|-?\d+)
    | (?P<ssa>%[A-Za-z0-9_.\-]+)
    | (?P<at>@[A-Za-z0-9_.\-]+)
    | (?P<ident>[A-Za-z_][A-Za-z0-9_\-]*)
    | (?P<punct>[{}()\[\],=])
""", re.VERBOSE)


class _Tok(tuple):
    kind = property(lambda t: t[0])
    text = property(lambda t: t[1])
    line = property(lambda t: t[2])
    col = property(lambda t: t[3])


def _lex(src: str) -> Iterator[_Tok]:
    line = col = 1
    pos = 0
    while pos < len(src):
        m = _LEX.match(src, pos)
        if m is None:
            raise ParseError(f"unexpected character {src[pos]!r}", line, col)
        kind, text = m.lastgroup, m.group()
        if kind == "newline":
            yield _Tok(("newline", text, line, col))
            line, col = line + 1, 1
        else:
            if kind not in ("ws", "comment"):
                yield _Tok((kind, text, line, col))
            col += len(text)
        pos = m.end()
    yield _Tok(("eof", "", line, col))


# ---------------------------------------------------------------------------
# parsing
# ---------------------------------------------------------------------------

class _Reader:
    def __init__(self, src: str):
        self.toks = list(_lex(src))
        self.i = 0

    # cursor --------------------------------------------------------------
    @property
    def cur(self) -> _Tok:
        return self.toks[self.i]

    def take(self) -> _Tok:
        t = self.toks[self.i]
        if t.kind != "eof":
            self.i += 1
        return t

    def fail(self, msg: str, tok: Optional[_Tok] = None):
        t = tok or self.cur
        raise ParseError(msg, t.line, t.col)

    def want(self, kind: str, text: Optional[str] = None) -> _Tok:
        t = self.take()
        if t.kind != kind or (text is not None and t.text != text):
            self.fail(f"expected {text if text is not None else kind!r}, found {t.text!r}", t)
        return t

    def sym(self, ch: str) -> _Tok:
        return self.want("punct", ch)

    def at(self, ch: str) -> bool:
        return self.cur.kind == "punct" and self.cur.text == ch

    def lines(self):
        while self.cur.kind == "newline":
            self.take()

    def comma_list(self, item, close="]"):
        out = []
        if not self.at(close):
            out.append(item())
            while self.at(","):
                self.take()
                out.append(item())
        return out

    # values ----------------------------------------------------------------
    def integer(self) -> int:
        t = self.want("number")
        try:
            return int(t.text)
        except ValueError:
            self.fail(f"expected integer, found {t.text!r}", t)

    def number(self):
        t = self.want("number")
        if t.text in ("inf", "-inf", "nan"):
            return float(t.text)
        try:
            return int(t.text)
        except ValueError:
            return float(t.text)

    def ints(self) -> tuple:
        self.sym("[")
        v = self.comma_list(self.integer)
        self.sym("]")
        return tuple(v)

    def int_lists(self) -> tuple:
        self.sym("[")
        v = self.comma_list(self.ints)
        self.sym("]")
        return tuple(v)

    def ints_or_lists(self):
        if self.toks[self.i + 1].kind == "punct" and self.toks[self.i + 1].text == "[":
            return self.int_lists()
        return self.ints()

    def shape(self) -> Shape:
        t = self.want("ident")
        if t.text not in DTYPES:
            self.fail(f"unknown dtype {t.text!r}", t)
        return Shape(self.ints(), DTYPES[t.text])

    def literal(self):
        if self.at("["):
            self.take()
            v = self.comma_list(self.literal)
            self.sym("]")
            return v
        if self.cur.kind == "ident" and self.cur.text in ("true", "false"):
            return self.take().text == "true"
        return self.number()

    def fields(self) -> dict:
        self.sym("{")
        out = {}
        while not self.at("}"):
            key = self.want("ident").text
            self.sym("=")
            out[key] = self.ints() if self.at("[") else self.integer()
            if self.at(","):
                self.take()
        self.sym("}")
        return out

    def sharding(self) -> Sharding:
        """Re-join the tokens of a balanced {...} and parse them as a
        sharding string (reference textir.py:220-244)."""
        open_tok = self.sym("{")
        depth, text = 1, ""
        while True:
            t = self.take()
            if t.kind == "eof":
                self.fail("unterminated sharding", open_tok)
            if t.kind == "punct" and t.text in "{}":
                depth += 1 if t.text == "{" else -1
                if depth == 0:
                    break
            if t.kind == "ident" and text and text[-1] not in "{[=":
                text += " "
            text += t.text
        try:
            return Sharding.parse(text)
        except ShardingError as e:
            self.fail(str(e), open_tok)

    def attribute(self, name: str):
        if name == "sharding":
            return self.sharding()
        if name in ("direction", "kind"):
            t = self.want("ident")
            enum = CompareDirection if name == "direction" else ReduceKind
            try:
                return enum(t.text)
            except ValueError:
                what = "compare direction" if name == "direction" else "reduce kind"
                self.fail(f"unknown {what} {t.text!r}", t)
        if name in ("subgroups", "pairs"):
            return self.int_lists()
        if name == "conv_dims":
            f = self.fields()
            try:
                return ConvDims(**{k: tuple(f[k]) if k.endswith("spatial") else f[k]
                                   for k in CONV_FIELDS})
            except KeyError as e:
                self.fail(f"conv_dims missing field {e}")
        if name == "window":
            self.sym("[")
            dims = []
            while not self.at("]"):
                f = self.fields()
                dims.append(WindowDim(size=f["size"],
                                      **{k: f.get(k, d) for k, d in WINDOW_DEFAULTS.items()}))
                if self.at(","):
                    self.take()
            self.sym("]")
            return tuple(dims)
        if name == "literal":
            return self.literal()
        if name == "fill":
            return self.number()
        return self.ints_or_lists() if self.at("[") else self.integer()

    # structure ---------------------------------------------------------------
    def instruction(self) -> Instruction:
        id_tok = self.want("ssa")
        self.sym("=")
        shape = self.shape()
        op_tok = self.want("ident")
        op = OPCODES.get(op_tok.text)
        if op is None:
            self.fail(f"unknown opcode {op_tok.text!r}", op_tok)
        self.sym("(")
        operands, attrs, sharding = [], {}, None
        if op == Op.PARAMETER:
            if self.cur.kind == "number":
                attrs["index"] = self.integer()
        else:
            while self.cur.kind == "ssa":
                operands.append(self.take().text[1:])
                if self.at(","):
                    self.take()
        self.sym(")")
        while self.at(","):
            self.take()
            name = self.want("ident").text
            self.sym("=")
            value = self.attribute(name)
            if name == "sharding":
                sharding = value
            else:
                attrs[name] = value
        if op in (Op.PARAMETER, Op.CONSTANT, Op.IOTA):
            attrs["shape"] = shape
        if op == Op.PARAMETER and "index" not in attrs:
            self.fail("parameter needs an index", id_tok)
        if op in (Op.RESHAPE, Op.BROADCAST):
            attrs["out_dims"] = shape.dims
        if op == Op.CONSTANT:
            if "literal" not in attrs:
                self.fail("constant needs a literal", id_tok)
            try:
                attrs["literal"] = np.asarray(attrs["literal"],
                                              dtype=np_dtype(shape.dtype)).reshape(shape.dims)
            except ValueError as e:
                self.fail(f"bad constant literal: {e}", id_tok)
        if sharding is not None and sharding.kind.name != "REPLICATED" and \
                sharding.data_rank != shape.rank:
            self.fail(f"sharding rank {sharding.data_rank} does not match shape rank "
                      f"{shape.rank}", id_tok)
        return Instruction(id=id_tok.text[1:], opcode=op, operands=tuple(operands),
                           attrs=attrs, shape=shape, sharding=sharding)

    def returns(self) -> tuple:
        self.want("ident", "return")
        outs = [self.want("ssa").text[1:]]
        while self.at(","):
            self.take()
            outs.append(self.want("ssa").text[1:])
        self.lines()
        return tuple(outs)

    def graph(self) -> Graph:
        self.lines()
        if self.cur.kind == "ssa":
            return self.bare()
        self.want("ident", "graph")
        name = self.want("at").text[1:]
        mesh = None
        if self.at("("):
            self.take()
            self.want("ident", "mesh")
            self.sym("=")
            dims = self.ints()
            ids = []
            while self.cur.kind == "number":
                ids.append(self.integer())
                if self.at(","):
                    self.take()
            mesh = DeviceMesh(dims, tuple(ids)) if ids else DeviceMesh.default(*dims)
            self.sym(")")
        self.sym("{")
        self.lines()
        body = []
        while True:
            t = self.cur
            if t.kind == "ident" and t.text == "return":
                outputs = self.returns()
                break
            if t.kind != "ssa":
                self.fail(f"expected instruction or return, found {t.text!r}", t)
            body.append(self.instruction())
            self.lines()
        self.sym("}")
        self.lines()
        return _checked(Graph(name, tuple(body), outputs, mesh))

    def bare(self) -> Graph:
        """Headerless instruction list; outputs default to the last one
        (reference textir.py:425-457)."""
        body, outputs = [], ()
        while self.cur.kind == "ssa":
            body.append(self.instruction())
            self.lines()
        if self.cur.kind == "ident" and self.cur.text == "return":
            outputs = self.returns()
        if self.cur.kind != "eof":
            self.fail(f"expected instruction, found {self.cur.text!r}", self.cur)
        if not body:
            self.fail("empty input")
        return _checked(Graph("main", tuple(body), outputs or (body[-1].id,), None))


def _checked(g: Graph) -> Graph:
    problems = validate_graph(g)
    if problems:
        raise ParseError("; ".join(problems), 1, 1)
    return g


def parse_graph(text: str) -> Graph:
    """(reference textir.py:460-461)"""
    return _Reader(text).graph()


# ---------------------------------------------------------------------------
# structural equality (reference textir.py:576-630)
# ---------------------------------------------------------------------------

def _canon(v):
    if isinstance(v, np.ndarray):
        return ("nd", v.shape, v.dtype.kind, v.tobytes())
    if isinstance(v, (tuple, list)):
        return tuple(_canon(x) for x in v)
    return v


def instructions_equal(a: Instruction, b: Instruction) -> bool:
    if (a.id, a.opcode, a.operands, a.shape, a.sharding) != \
            (b.id, b.opcode, b.operands, b.shape, b.sharding) or set(a.attrs) != set(b.attrs):
        return False
    for k, va in a.attrs.items():
        vb = b.attrs[k]
        if isinstance(va, np.ndarray) or isinstance(vb, np.ndarray):
            if np.asarray(va).shape != np.asarray(vb).shape or not np.array_equal(va, vb):
                return False
        elif _canon(va) != _canon(vb):
            return False
    return True


def graphs_equal(a: Graph, b: Graph) -> bool:
    if (a.name, a.outputs) != (b.name, b.outputs) or (a.mesh is None) != (b.mesh is None):
        return False
    if a.mesh is not None and (tuple(a.mesh.mesh_dims), tuple(a.mesh.device_ids)) != \
            (tuple(b.mesh.mesh_dims), tuple(b.mesh.device_ids)):
        return False
    return len(a.instructions) == len(b.instructions) and \
        all(instructions_equal(x, y) for x, y in zip(a.instructions, b.instructions))
