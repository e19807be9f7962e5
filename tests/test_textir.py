"""Text IR (reference textir.py, tests/test_textir.py).

Pinned against the reference's own printout (tests/golden/textir.json.gz) of
every golden graph (240 random + 124 named), its propagated form and its SPMD
program: ``print_graph`` is byte-identical, ``parse_graph`` inverts it
structurally, and malformed inputs fail with the reference's ParseError line,
column and message."""

import numpy as np
import pytest

import golden_io as G
from paper_2105_04663_b200 import propagate
from paper_2105_04663_b200.ir import (ConvDims, DType, GraphBuilder, Op, ReduceKind, Shape,
                                      WindowDim)
from paper_2105_04663_b200.partitioner import partition
from paper_2105_04663_b200.sharding import DeviceMesh, mesh_split
from paper_2105_04663_b200.textir import ParseError, graphs_equal, parse_graph, print_graph

TEXT = G.textir()
CASES = [(kind, c) for kind in ("random", "named") for c in G.cases(kind)]


def _ids(kc):
    return kc[1]["name"]


@pytest.mark.parametrize("kc", CASES, ids=_ids)
def test_print_matches_reference(kc):
    kind, case = kc
    ref = TEXT["graphs"][case["name"]]
    g = G.graph(case)
    assert print_graph(g) == ref["graph"]
    ann, _ = propagate(g)
    assert print_graph(ann) == ref["annotated"]
    if "program" in case:
        assert print_graph(partition(ann, case["num_devices"]).graph) == ref["program"]
        assert print_graph(G.program(case)) == ref["program"]


@pytest.mark.parametrize("kc", CASES, ids=_ids)
def test_parse_inverts_print(kc):
    _, case = kc
    for key in ("graph", "annotated", "program"):
        text = TEXT["graphs"][case["name"]].get(key)
        if text is None:
            continue
        g = parse_graph(text)
        assert print_graph(g) == text
    g0 = G.graph(case)
    assert graphs_equal(parse_graph(print_graph(g0)), g0)


@pytest.mark.parametrize("i", range(len(TEXT["errors"])))
def test_parse_errors_match_reference(i):
    e = TEXT["errors"][i]
    if e["error"] is None:
        parse_graph(e["text"])
        return
    with pytest.raises(ParseError) as got:
        parse_graph(e["text"])
    assert (got.value.line, got.value.column, str(got.value)) == \
        (e["line"], e["column"], e["message"])


# -- reference tests/test_textir.py restated -----------------------------------

def _round_trip(g):
    text = print_graph(g)
    back = parse_graph(text)
    assert graphs_equal(g, back), text
    assert print_graph(back) == text
    return text


def test_minimal():
    b = GraphBuilder("g")
    x = b.parameter(Shape((8,)))
    _round_trip(b.build([b.add(Op.RELU, [x])]))


def test_shardings_and_mesh():
    mesh = DeviceMesh.default(2, 2)
    b = GraphBuilder("g", mesh)
    x = b.parameter(Shape((8, 8)), sharding=mesh_split(2, mesh, [0, 1]))
    y = b.add(Op.EXP, [x], sharding=mesh_split(2, mesh, [-1, 0]))
    text = _round_trip(b.build([y]))
    assert "mesh=[2,2]" in text and "last_tile_dim_replicate" in text


def test_custom_mesh_order_round_trips():
    mesh = DeviceMesh((2, 2), (3, 1, 2, 0))
    b = GraphBuilder("g", mesh)
    x = b.parameter(Shape((4, 4)), sharding=mesh_split(2, mesh, [0, 1]))
    text = _round_trip(b.build([x]))
    assert text.startswith("graph @g (mesh=[2,2]3,1,2,0) {")


def test_unspecified_dims():
    mesh = DeviceMesh.default(2)
    b = GraphBuilder("g", mesh)
    x = b.parameter(Shape((4, 4)), sharding=mesh_split(2, mesh, [0, -1]).with_unspecified([1]))
    _round_trip(b.build([x]))


def test_all_attr_kinds():
    b = GraphBuilder("g")
    x = b.parameter(Shape((2, 3, 16)))
    k = b.parameter(Shape((3, 4, 3)))
    cd = ConvDims(lhs_batch=0, lhs_feature=1, lhs_spatial=(2,), rhs_in_feature=0,
                  rhs_out_feature=1, rhs_spatial=(2,), out_batch=0, out_feature=1,
                  out_spatial=(2,))
    w = WindowDim(size=3, stride=2, padding_low=1, padding_high=0, base_dilation=2,
                  window_dilation=1)
    c = b.add(Op.CONVOLUTION, [x, k], {"conv_dims": cd, "window": (w,)})
    z = b.constant(np.float32(0), Shape((), DType.F32))
    _round_trip(b.build([b.add(Op.REDUCE, [c, z], {"kind": ReduceKind.SUM, "dims": (0, 2)})]))


def test_float_literals_exact():
    b = GraphBuilder("g")
    lit = np.array([0.1, -1.5, 3e-8, float("inf")], dtype=np.float32)
    c = b.constant(lit, Shape((4,), DType.F32))
    back = parse_graph(print_graph(b.build([c])))
    np.testing.assert_array_equal(back.instr(c).attrs["literal"], lit)


def test_collectives_and_multiple_outputs():
    b = GraphBuilder("g")
    x = b.parameter(Shape((4,)))
    ar = b.add(Op.ALL_REDUCE, [x], {"kind": ReduceKind.SUM, "subgroups": ((0, 1), (2, 3))})
    cp = b.add(Op.COLLECTIVE_PERMUTE, [ar], {"pairs": ((0, 1), (1, 0))})
    _round_trip(b.build([cp, b.add(Op.NEGATE, [x])]))


def test_bare_instruction_list():
    g = parse_graph("%x = f32[8] parameter(0), sharding={devices=[2]0,1}")
    assert g.instr("x").opcode == Op.PARAMETER and g.outputs == ("x",)
    assert g.instr("x").sharding.tiles(0) == 2


def test_print_is_stable():
    mesh = DeviceMesh.default(4)
    b = GraphBuilder("g", mesh)
    x = b.parameter(Shape((12,)), sharding=mesh_split(1, mesh, [0]))
    c = b.constant(np.float32(1), Shape((), DType.F32))
    g = b.build([b.add(Op.PAD, [x, c], {"low": (2,), "high": (1,), "interior": (1,)})])
    assert print_graph(g) == print_graph(g) == print_graph(parse_graph(print_graph(g)))
