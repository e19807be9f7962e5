"""The pinned GShard routing rule (moe.route_topk), on hand-checked cases.

Gating is out of the reference's scope (it consumes a given
dispatch tensor through a Dot, tests/test_acceptance.py:326-349), so the
rule is restated from GShard's Top2Gating (Lepikhin et al. 2020, Alg. 1):
first choices take slots before second choices, a second choice's slot
starts after the expert's capacity-truncated first-choice count.
"""

import numpy as np

from paper_2105_04663_b200.moe import route_assign, route_masks, route_topk


def _logits(rows):
    return np.asarray(rows, np.float32)[None]


def test_top2_order_and_capacity():
    # 4 tokens, 3 experts; first choices: 0, 0, 1, 0; second: 1, 2, 0, 2
    lg = _logits([[3, 2, 0], [3, 0, 1], [1, 4, 0], [5, 0, 2]])
    e, s, g = route_topk(lg, 2, capacity=2)
    np.testing.assert_array_equal(e[0], [[0, 1], [0, 2], [1, 0], [0, 2]])
    # expert 0 first choices: tokens 0, 1, 3 -> slots 0, 1, 2 (token 3 dropped)
    # expert 1: first choice of token 2 -> 0; second choice of token 0 -> 0 + 1
    # expert 2: second choices of tokens 1, 3 -> 0, 1
    # expert 0 second choice (token 2): after min(3, C=2) kept firsts -> 2 (dropped)
    np.testing.assert_array_equal(s[0], [[0, 1], [1, 0], [0, 2], [2, 1]])
    np.testing.assert_allclose(g.sum(-1), 1.0, rtol=1e-6)
    d, c = route_masks(lg, 2, 2)
    assert d.sum() == 6                       # 8 choices, 2 dropped
    assert d[0, 3, 0].sum() == 0 and d[0, 3, 2, 1] == 1
    np.testing.assert_allclose(c[0, 0, 1, 1], g[0, 0, 1], rtol=1e-7)


def test_ties_take_the_first_maximum():
    lg = _logits([[1, 1, 1], [0, 2, 2]])
    e, s, _ = route_topk(lg, 2, capacity=4)
    np.testing.assert_array_equal(e[0], [[0, 1], [1, 2]])


def test_top1_matches_route_assign_and_slots_are_prefix_counts():
    rng = np.random.default_rng(0)
    lg = rng.standard_normal((3, 50, 4)).astype(np.float32)
    e1, s1, g1 = route_topk(lg, 1, capacity=7)
    e, s, g = route_assign(lg)
    np.testing.assert_array_equal(e1[..., 0], e)
    np.testing.assert_array_equal(s1[..., 0], s)
    for b in range(3):
        for t in range(50):
            assert s[b, t] == np.sum(e[b, :t] == e[b, t])


def test_second_choice_slots_follow_first_choice_counts():
    rng = np.random.default_rng(1)
    lg = rng.standard_normal((2, 64, 8)).astype(np.float32)
    C = 12
    e, s, _ = route_topk(lg, 2, capacity=C)
    for b in range(2):
        for x in range(8):
            first = min(int(np.sum(e[b, :, 0] == x)), C)
            sec = np.nonzero(e[b, :, 1] == x)[0]
            np.testing.assert_array_equal(s[b, sec, 1], first + np.arange(len(sec)))
