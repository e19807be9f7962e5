"""GShard-style top-k routing with expert capacity (host-side slot rules).

The reference consumes a *given* dispatch tensor through a dense Dot
(``tests/test_acceptance.py:326-349``); gating is out of its scope
(SPEC.md:8), so slot assignment is pinned here: tokens are visited in
(batch, sequence) order, each token's expert slot is the running count of
earlier tokens of the same batch row routed to that expert (an exclusive
prefix sum of the one-hot assignment), and tokens beyond capacity ``C`` are
dropped.  The device kernels (``csrc/moe.cu``) implement the same rule with
warp-level scans; tests check them bit-exact against this function.
"""

from __future__ import annotations

import numpy as np


def route_assign(logits: np.ndarray):
    """logits [B, S, E] -> (expert [B,S] int32, slot [B,S] int32, gate [B,S]
    float32): first-max argmax, exclusive per-(row, expert) prefix count,
    softmax probability of the chosen expert."""
    B, S, E = logits.shape
    logits = np.asarray(logits, np.float32)
    z = logits - logits.max(-1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(-1, keepdims=True)
    expert = logits.argmax(-1)
    onehot = np.eye(E, dtype=np.int64)[expert]                 # [B, S, E]
    pos = np.cumsum(onehot, axis=1) - onehot                   # exclusive scan over S
    slot = (pos * onehot).sum(-1)                              # [B, S]
    gate = np.take_along_axis(p, expert[..., None], -1)[..., 0].astype(np.float32)
    return expert.astype(np.int32), slot.astype(np.int32), gate


def route_top1(logits: np.ndarray, capacity: int):
    """logits [B, S, E] -> (dispatch, combine) one-hot masks [B, S, E, C].

    combine carries the softmax gate probability of the chosen expert."""
    B, S, E = logits.shape
    expert, slot, _ = route_assign(logits)
    z = logits - logits.max(-1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(-1, keepdims=True)
    keep = slot < capacity
    dispatch = np.zeros((B, S, E, capacity), np.float32)
    bi, si = np.nonzero(keep)
    dispatch[bi, si, expert[bi, si], slot[bi, si]] = 1.0
    gate = np.take_along_axis(p, expert[..., None], -1)[..., 0].astype(np.float32)
    combine = dispatch * gate[:, :, None, None]
    return dispatch, combine.astype(np.float32)
