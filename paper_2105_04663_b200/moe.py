"""GShard-style top-k routing with expert capacity (host-side slot rules).

The reference consumes a *given* dispatch tensor through a dense Dot
(``tests/test_acceptance.py:326-349``); gating is out of its scope
(SPEC.md:8), so the routing rule is pinned here and the device kernels
(``csrc/moe.cu``) are checked bit-exact against it:

* choice 1 of a token is the first maximum of its logits; choice k > 1 is the
  first maximum over the experts not chosen yet (GShard Top2Gating,
  Lepikhin et al. 2020, Algorithm 1: ``index_2 = argmax(logits * (1 - mask_1))``);
* slots are assigned choice by choice (GShard order: every first choice of a
  group before any second choice).  Within choice k, tokens are visited in
  sequence order inside their batch row (the GShard group); a token's slot is
  the number of earlier tokens of the row that picked the same expert as
  their k-th choice, plus the kept (capacity-truncated) slots of that expert
  from choices 1..k-1 (``position_in_expert_2 = cumsum(mask_2) - mask_2 +
  sum(mask_1)`` with ``mask_1`` already truncated to capacity);
* a choice whose slot is >= capacity C is dropped (its dispatch row stays
  empty and it contributes nothing to the combine);
* gates: top-1 keeps the softmax probability of the chosen expert; top-k
  (k >= 2) renormalises the chosen probabilities to sum to one
  (``gate_k = p_k / sum_j p_j``).  GShard's random second-expert dispatch is
  not used: routing here is deterministic, so it can be pinned bit-exactly.

Layouts: ``expert``/``slot`` int32 and ``gate`` float32 of shape ``[B, S]``
(top-1) or ``[B, S, k]``.
"""

from __future__ import annotations

import numpy as np


def _softmax(logits: np.ndarray) -> np.ndarray:
    z = logits - logits.max(-1, keepdims=True)
    p = np.exp(z)
    return p / p.sum(-1, keepdims=True)


def route_topk(logits: np.ndarray, k: int, capacity: int):
    """logits [B, S, E] -> (expert, slot, gate), each [B, S, k] (int32,
    int32, float32).  ``slot >= capacity`` marks a dropped choice."""
    B, S, E = logits.shape
    if not 1 <= k <= min(E, 4):
        raise ValueError(f"top-k routing needs 1 <= k <= min(E, 4), got k={k}, E={E}")
    logits = np.asarray(logits, np.float32)
    p = _softmax(logits)
    expert = np.zeros((B, S, k), np.int64)
    slot = np.zeros((B, S, k), np.int64)
    taken = np.zeros((B, S, E), bool)
    kept = np.zeros((B, E), np.int64)          # kept slots of earlier choices
    for c in range(k):
        masked = np.where(taken, -np.inf, logits)
        e = masked.argmax(-1)                   # first maximum
        onehot = np.eye(E, dtype=np.int64)[e]   # [B, S, E]
        pos = np.cumsum(onehot, axis=1) - onehot + kept[:, None, :]
        expert[..., c] = e
        slot[..., c] = (pos * onehot).sum(-1)
        taken |= onehot.astype(bool)
        kept = np.minimum(kept + onehot.sum(1), capacity)
    gate = np.take_along_axis(p, expert, -1).astype(np.float32)
    if k > 1:
        gate = (gate / gate.sum(-1, keepdims=True, dtype=np.float32)).astype(np.float32)
    return expert.astype(np.int32), slot.astype(np.int32), gate


def route_assign(logits: np.ndarray):
    """Top-1: logits [B, S, E] -> (expert [B,S] int32, slot [B,S] int32, gate
    [B,S] float32): first-max argmax, exclusive per-(row, expert) prefix count,
    softmax probability of the chosen expert."""
    B, S, E = logits.shape
    e, s, g = route_topk(logits, 1, capacity=S + 1)
    return e[..., 0], s[..., 0], g[..., 0]


def route_masks(logits: np.ndarray, capacity: int, k: int = 1):
    """logits [B, S, E] -> (dispatch, combine) masks [B, S, E, C]: dispatch
    holds 1 at every kept (expert, slot) of a token, combine its gate."""
    B, S, E = logits.shape
    expert, slot, gate = route_topk(logits, k, capacity)
    dispatch = np.zeros((B, S, E, capacity), np.float32)
    combine = np.zeros((B, S, E, capacity), np.float32)
    bi, si, ci = np.nonzero(slot < capacity)
    dispatch[bi, si, expert[bi, si, ci], slot[bi, si, ci]] = 1.0
    combine[bi, si, expert[bi, si, ci], slot[bi, si, ci]] = gate[bi, si, ci]
    return dispatch, combine


def route_top1(logits: np.ndarray, capacity: int):
    """logits [B, S, E] -> (dispatch, combine) one-hot masks [B, S, E, C];
    combine carries the softmax gate probability of the chosen expert."""
    return route_masks(logits, capacity, 1)


def route_top2(logits: np.ndarray, capacity: int):
    """GShard top-2 masks [B, S, E, C] (combine = renormalised gates)."""
    return route_masks(logits, capacity, 2)
