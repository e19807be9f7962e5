"""Pipeline parallelism as plain dataflow (reference pipeline.py:1-319).

GSPMD expresses a pipeline without a scheduler: the activations of all ``L``
stages live in ONE buffer with a leading stage dim; every unrolled iteration
moves the buffer one stage along and applies the (stage-batched) body.  With
the stage dim sharded over the mesh, the partitioner turns that move into a
collective-permute between neighbours (``halo.detect_and_rotate``,
reference formatting.py:689-792) -- the paper's Sec. 3.3 pipelining.

* ``gpipe``: microbatch m enters stage 0 at iteration m and leaves stage L-1
  at iteration m+L-1 (pad-left-then-slice shift, the last stage falls off).
* ``circular``: each device owns ``R`` layers round-robin; the buffer
  wraps from the last stage back to the first (a rotate) and every
  microbatch makes ``R`` laps.  Per-stage weights are picked per iteration
  by the lap each stage is on.

The emitted instruction stream (ids, order, attributes) is the reference's,
so the partitioned programs are identical (tests/test_pipeline.py against
golden programs recorded from the reference).
"""

from __future__ import annotations

import dataclasses
from fractions import Fraction
from typing import Callable, Optional, Sequence

import numpy as np

from .ir import CompareDirection, DType, Graph, GraphBuilder, Op, Shape, np_dtype
from .sharding import DeviceMesh, Sharding


class ShapeMismatch(Exception):
    """The stage body changed the buffer shape (reference pipeline.py:36-37)."""


# body(builder, buffer_id [L, *state], weight_ids [L, *w] each) -> new buffer id
StageBody = Callable[[GraphBuilder, str, Sequence[str]], str]

SCHEDULES = ("gpipe", "circular")


@dataclasses.dataclass(frozen=True)
class PipelineConfig:
    """(reference pipeline.py:47-69)"""

    num_stages: int
    num_microbatches: int
    schedule: str = "gpipe"
    layers_per_device: int = 1

    def __post_init__(self):
        if min(self.num_stages, self.num_microbatches) < 1:
            raise ValueError("num_stages and num_microbatches must be >= 1")
        if self.schedule not in SCHEDULES:
            raise ValueError(f"unknown schedule {self.schedule!r}")
        if self.layers_per_device < 1:
            raise ValueError("layers_per_device must be >= 1")
        if self.schedule == "gpipe" and self.layers_per_device != 1:
            raise ValueError("gpipe schedule uses exactly one layer per stage")

    @property
    def total_layers(self) -> int:
        return self.num_stages * self.layers_per_device


@dataclasses.dataclass(frozen=True)
class BubbleStats:
    """Useful vs padded stage applications (reference pipeline.py:71-99)."""

    total_iterations: int
    useful_applications: int
    padded_applications: int

    @property
    def total_applications(self) -> int:
        return self.useful_applications + self.padded_applications

    @property
    def bubble_ratio(self) -> Fraction:
        total = self.total_applications
        return Fraction(self.padded_applications, total) if total else Fraction(0)

    def to_json(self) -> dict:
        r = self.bubble_ratio
        return {"total_iterations": self.total_iterations,
                "useful_applications": self.useful_applications,
                "padded_applications": self.padded_applications,
                "bubble_ratio": [r.numerator, r.denominator],
                "bubble_ratio_float": float(r)}


def schedule_slots(cfg: PipelineConfig) -> list[dict[int, tuple[int, int]]]:
    """Per iteration: {stage: (microbatch, lap)} for the occupied slots
    (reference pipeline.py:102-120).  Microbatches are issued in groups of L;
    inside a group, lap r of microbatch m enters stage 0 at
    ``group*L*R + r*L + (m mod L)``."""
    L, R = cfg.num_stages, cfg.layers_per_device
    starts = []
    for m in range(cfg.num_microbatches):
        grp, pos = divmod(m, L)
        starts += [(grp * L * R + lap * L + pos, m, lap) for lap in range(R)]
    n_iter = 1 + max(t for t, _, _ in starts) + L - 1
    slots: list[dict[int, tuple[int, int]]] = [{} for _ in range(n_iter)]
    for t, m, lap in starts:
        for stage in range(L):
            slots[t + stage][stage] = (m, lap)
    return slots


def bubble_stats(cfg: PipelineConfig) -> BubbleStats:
    """(reference pipeline.py:123-132)"""
    slots = schedule_slots(cfg)
    useful = sum(map(len, slots))
    return BubbleStats(len(slots), useful, len(slots) * cfg.num_stages - useful)


class _Emitter:
    """Emits the pipeline's instructions in the reference's order."""

    def __init__(self, b: GraphBuilder, cfg: PipelineConfig, state: Shape):
        self.b, self.cfg, self.state = b, cfg, state
        self.L, self.R = cfg.num_stages, cfg.layers_per_device
        self.rank = state.rank
        self.tail = (0,) * (self.rank - 1)

    def _slice(self, src, lo0, hi0, id):
        return self.b.add(Op.SLICE, [src],
                          {"starts": (lo0,) + self.tail,
                           "limits": (hi0,) + self.state.dims[1:],
                           "strides": (1,) * self.rank}, id=id)

    def stage0_mask(self) -> str:
        """broadcast(iota(L) == 0) over the buffer (pipeline.py:185-197)."""
        b, L = self.b, self.L
        ids = b.add(Op.IOTA, [], {"shape": Shape((L,), DType.S32), "iota_dimension": 0},
                    id="stage_ids")
        z = b.constant(np.int32(0), Shape((), DType.S32), id="zero_s32")
        zv = b.add(Op.BROADCAST, [z], {"out_dims": (L,), "broadcast_dims": ()}, id="zero_vec")
        eq = b.add(Op.COMPARE, [ids, zv], {"direction": CompareDirection.EQ}, id="first_stage")
        return b.add(Op.BROADCAST, [eq], {"out_dims": self.state.dims, "broadcast_dims": (0,)},
                     id="first_stage_mask")

    def advance(self, buf: str, fill: str, i: int) -> str:
        """Move every stage's activation to the next stage (pipeline.py:207-230)."""
        L = self.L
        if L == 1:
            return buf
        if self.cfg.schedule == "circular":
            last = self._slice(buf, L - 1, L, f"wrap{i}")
            rest = self._slice(buf, 0, L - 1, f"head{i}")
            return self.b.add(Op.CONCAT, [last, rest], {"dim": 0}, id=f"shift{i}")
        padded = self.b.add(Op.PAD, [buf, fill],
                            {"low": (1,) + self.tail, "high": (0,) * self.rank,
                             "interior": (0,) * self.rank}, id=f"padded{i}")
        return self._slice(padded, 0, L, f"shift{i}")

    def inject(self, buf: str, mask: str, micro: str, i: int) -> str:
        """Stage 0 takes the entering microbatch (pipeline.py:232-241)."""
        inp = self.b.add(Op.BROADCAST, [micro],
                         {"out_dims": self.state.dims,
                          "broadcast_dims": tuple(range(1, self.rank))}, id=f"inp{i}")
        return self.b.add(Op.SELECT, [mask, inp, buf], id=f"select{i}")

    def lap_weights(self, weights, wshapes, row, i):
        """Circular schedule: per stage, the weight of the lap it is on --
        select chains against the per-iteration lap vector
        (pipeline.py:265-306)."""
        b, L, R = self.b, self.L, self.R
        laps = np.asarray([row.get(s, (0, 0))[1] for s in range(L)], dtype=np.int32)
        lap_vec = b.add(Op.CONSTANT, [], {"literal": laps, "shape": Shape((L,), DType.S32)},
                        id=f"rounds{i}")
        picked = []
        for k, (w, ws) in enumerate(zip(weights, wshapes)):
            per_stage = (L,) + tuple(ws.dims)
            cur = None
            for r in range(R):
                piece = b.add(Op.SLICE, [w],
                              {"starts": (0, r) + (0,) * ws.rank,
                               "limits": (L, r + 1) + tuple(ws.dims),
                               "strides": (1,) * (ws.rank + 2)}, id=f"w{k}_r{r}_i{i}")
                flat = b.add(Op.RESHAPE, [piece], {"out_dims": per_stage},
                             id=f"w{k}_r{r}f_i{i}")
                if cur is None:
                    cur = flat
                    continue
                rv = b.add(Op.CONSTANT, [],
                           {"literal": np.full((L,), r, dtype=np.int32),
                            "shape": Shape((L,), DType.S32)}, id=f"rc{k}_{r}_i{i}")
                on_r = b.add(Op.COMPARE, [lap_vec, rv], {"direction": CompareDirection.EQ},
                             id=f"isr{k}_{r}_i{i}")
                m = b.add(Op.BROADCAST, [on_r], {"out_dims": per_stage, "broadcast_dims": (0,)},
                          id=f"wm{k}_{r}_i{i}")
                cur = b.add(Op.SELECT, [m, flat, cur], id=f"wsel{k}_{r}_i{i}")
            picked.append(cur)
        return picked


def build_pipeline(cfg: PipelineConfig, mesh: Optional[DeviceMesh], state_dims: Sequence[int],
                   body: StageBody, weight_shapes: Sequence[Shape] = (),
                   dtype: DType = DType.F32, input_sharding: Optional[Sharding] = None,
                   state_sharding: Optional[Sharding] = None,
                   weight_shardings: Optional[Sequence[Optional[Sharding]]] = None,
                   name: str = "pipeline") -> Graph:
    """Unrolled shifting-buffer pipeline (reference pipeline.py:135-262).

    Parameters: one ``state_dims`` tensor per microbatch, then the weights
    with a leading ``(L,)`` (gpipe) or ``(L, R)`` (circular) dim.  Outputs:
    each microbatch's last-stage result, in microbatch order."""
    L, M, R = cfg.num_stages, cfg.num_microbatches, cfg.layers_per_device
    state = Shape((L,) + tuple(state_dims), dtype)
    wshards = list(weight_shardings) if weight_shardings is not None else \
        [None] * len(weight_shapes)
    b = GraphBuilder(name, mesh)
    micro = [b.parameter(Shape(tuple(state_dims), dtype), sharding=input_sharding,
                         id=f"microbatch{m}") for m in range(M)]
    lead = (L,) if cfg.schedule == "gpipe" else (L, R)
    weights = [b.parameter(Shape(lead + tuple(ws.dims), ws.dtype), sharding=sh, id=f"weight{k}")
               for k, (ws, sh) in enumerate(zip(weight_shapes, wshards))]
    em = _Emitter(b, cfg, state)
    mask = em.stage0_mask()
    fill = b.constant(np.zeros((), dtype=np_dtype(dtype)), Shape((), dtype), id="state_fill")
    buf = b.add(Op.BROADCAST, [fill], {"out_dims": state.dims, "broadcast_dims": ()},
                id="state_init")
    outputs: list[Optional[str]] = [None] * M
    for i, row in enumerate(schedule_slots(cfg)):
        buf = em.advance(buf, fill, i)
        entering = [m for s, (m, lap) in row.items() if s == 0 and lap == 0]
        if entering:
            buf = em.inject(buf, mask, micro[entering[0]], i)
        ws = em.lap_weights(weights, weight_shapes, row, i) if cfg.schedule == "circular" \
            else weights
        buf = body(b, buf, ws)
        got = b.shape_of(buf)
        if got != state:
            raise ShapeMismatch(f"stage body produced {got}, expected {state}")
        if state_sharding is not None:   # identity reshape = annotation point
            buf = b.add(Op.RESHAPE, [buf], {"out_dims": state.dims}, sharding=state_sharding,
                        id=f"state{i}")
        leaving = [m for s, (m, lap) in row.items() if s == L - 1 and lap == R - 1]
        if leaving:
            m = leaving[0]
            last = em._slice(buf, L - 1, L, f"last{i}")
            outputs[m] = b.add(Op.RESHAPE, [last], {"out_dims": tuple(state_dims)}, id=f"out{m}")
    assert all(o is not None for o in outputs)
    return b.build(outputs)
