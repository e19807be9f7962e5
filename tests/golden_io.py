"""Loader for the golden fixtures produced by ``tests/golden/make_golden.py``
(which runs the reference).  Pure data: no reference import at test time."""

import functools
import gzip
import json
import os

import numpy as np

from paper_2105_04663_b200.ir import graph_from_json

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(None)
def cases(kind: str):
    with gzip.open(os.path.join(HERE, f"{kind}.json.gz"), "rt") as f:
        return json.load(f)


@functools.lru_cache(None)
def arrays():
    out = dict(np.load(os.path.join(HERE, "arrays.npz")))
    out.update(np.load(os.path.join(HERE, "c5w_arrays.npz")))   # C5 over 2 / 4 shards
    return out


# case kinds holding reference-run graphs, programs and outputs
KINDS = ("named", "random", "c5w")


def case_by_name(name):
    for kind in KINDS:
        for c in cases(kind):
            if c["name"] == name:
                return c
    raise KeyError(name)


def graph(case):
    return graph_from_json(case["graph"])


def program(case):
    return graph_from_json(case["program"])


def inputs(case):
    a = arrays()
    return [a[k] for k in case["inputs"]]


def expected(case):
    a = arrays()
    return [a[k] for k in case["expected"]]


def spmd_outputs(case):
    a = arrays()
    return {int(d): [a[k] for k in keys] for d, keys in case["spmd"].items()}


def textir():
    """Reference print_graph texts and ParseError positions (make_golden.py)."""
    with gzip.open(os.path.join(HERE, "textir.json.gz"), "rt") as f:
        return json.load(f)
