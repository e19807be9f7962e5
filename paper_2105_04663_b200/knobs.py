"""Executor plan knobs: one registry, read once per Executor.

Every fusion / engine / lane choice the executor makes at plan time can be
switched off or forced for A/B measurements (scripts/ab_bench.sh) and for
tests.  Each knob's default is the measured best (DESIGN.md cites the A/B);
the environment variable of the same name overrides it, and
``Executor(..., knobs={"SPMD_RS_ADD": "0"})`` overrides both for one
executor.  The kernel-side variants (GEMM tile shape, attention key tile,
...) are separate: ``spmd_set_option`` in the C library (``_capi.option``).
"""

import os
from typing import Mapping, Optional

# name -> (default, meaning)
KNOBS: dict[str, tuple[str, str]] = {
    # fusions (_plan_fusions and friends)
    "SPMD_FUSED_ATTENTION": ("1", "Dot -> softmax chain -> Dot as one attention kernel"),
    "SPMD_TRANSPOSE_RELU": ("1", "Transpose -> ReLU in one pass (MoE reshard chains)"),
    "SPMD_AG_SPLIT": ("1", "loopback all-gathers of an f32 Dot write the 3xTF32 halves"),
    "SPMD_DOT_ADD": ("1", "residual Add in the GEMM epilogue"),
    "SPMD_RS_ADD": ("1", "residual Add in the peer reduce-scatter's slot reduce"),
    "SPMD_BWD_FUSION": ("1", "softmax-backward and ReLU-backward chains as one kernel each"),
    "SPMD_HALO_CONV": ("1", "halo window read in place by the convolution"),
    "SPMD_PEER_FUSION": ("1", "Dot -> reduce-scatter / all-to-all in the GEMM epilogue"),
    # peer-memory collective engines
    "SPMD_PEER_AG": ("1", "parameter all-gathers through staged peer-heap slots"),
    "SPMD_PEER_AG_PUSH": ("1", "critical-path all-gathers pushed into landing zones"),
    "SPMD_PEER_AG_PUSH_PARAMS": ("1", "exposed parameter gathers pushed too, not staged"),
    "SPMD_PEER_A2A": ("1", "all-to-alls pushed into landing zones"),
    "SPMD_PEER_CP": ("1", "collective-permutes through peer-heap slots"),
    "SPMD_PEER_AG_ENGINE": ("auto", "engine of exposed staged gathers: auto | ce | sm"),
    "SPMD_PEER_HIDDEN_ENGINE": ("ce", "engine of gathers hidden under GEMMs: ce | sm"),
    "SPMD_PEER_STAGE": ("1", "stage parameter shards once per step"),
    "SPMD_PEER_STAGE_WIDE": ("1", "stage every parameter gather, not only hidden ones"),
    "SPMD_PEER_STAGE_ACT": ("0", "stage activation gathers too"),
    "SPMD_STAGE_PHASES": ("2", "staging barriers per step: 1 | 2 (exposed shards first)"),
    # streams and scheduling
    "SPMD_COMM_LANES": ("critical", "comm lane assignment: critical | single"),
    "SPMD_EXPOSED_SPLIT": ("1", "exposed collectives alternate over two lanes"),
    "SPMD_COMM_PRIORITY": ("0", "CUDA stream priority of the comm lanes"),
    "SPMD_COMM_SMS": ("", "SMs kept free of persistent kernels (empty: 0 when staged, else 2)"),
    "SPMD_PREFETCH": ("jit", "collective hoisting: jit | asap"),
    "SPMD_PREFETCH_DEPTH": ("2", "GEMMs a hoisted gather may run ahead of its consumer"),
}


def resolve(overrides: Optional[Mapping[str, object]] = None) -> dict[str, str]:
    """Snapshot of every knob: override > environment > default."""
    out = {}
    for name, (default, _) in KNOBS.items():
        out[name] = os.environ.get(name, default)
    for name, v in (overrides or {}).items():
        if name not in KNOBS:
            raise KeyError(f"unknown executor knob {name!r}")
        out[name] = str(v)
    return out
