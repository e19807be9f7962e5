"""PartitionContext (recursive device grouping) vs the reference
(partitioner.py:95-138), on the seeded nestings recorded by
tests/golden/make_context_golden.py."""

import json
import os

import pytest

from paper_2105_04663_b200.partitioner import PartitionContext

with open(os.path.join(os.path.dirname(__file__), "golden", "context.json")) as f:
    CASES = json.load(f)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c['n']}_{len(c['steps'])}")
def test_matches_reference(case):
    ctx = PartitionContext.root(case["n"])
    assert ctx.num_logical == case["n"] and ctx.parent is None
    for st in case["steps"]:
        assert ctx.physical_subgroups(st["query"]) == st["physical"]
        parent, ctx = ctx, ctx.child(st["merge"])
        assert ctx.parent is parent
        assert ctx.device_groups == st["groups"] and ctx.num_logical == st["num_logical"]


def test_nested_axes_of_a_2x4_mesh():
    """Rows of a 2x4 mesh as the outer grouping: an all-gather over the
    inner (4-way) logical axis runs once per row."""
    root = PartitionContext.root(8)
    rows = root.child([[0, 1, 2, 3], [4, 5, 6, 7]])
    assert rows.physical_subgroups([[0, 1]]) == [[0, 4], [1, 5], [2, 6], [3, 7]]
    cols = root.child([[0, 4], [1, 5], [2, 6], [3, 7]])
    assert cols.physical_subgroups([[0, 1, 2, 3]]) == [[0, 1, 2, 3], [4, 5, 6, 7]]


def test_ragged_groups_raise_like_the_reference():
    ctx = PartitionContext([[0, 1], [2]])
    with pytest.raises(IndexError):
        ctx.physical_subgroups([[0, 1]])
