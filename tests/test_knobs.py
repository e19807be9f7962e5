"""Executor plan knobs (knobs.py): every knob the executor reads is
registered with a default, read once per Executor, and an explicit
``knobs=`` override beats the environment.  CPU only (stand-in comm)."""

import os
import re

import pytest

from paper_2105_04663_b200 import knobs, partition, propagate
from paper_2105_04663_b200.executor import Executor
from paper_2105_04663_b200.ir import DType
from paper_2105_04663_b200.workloads import transformer_layer

from test_executor_plan import FakeComm

HERE = os.path.dirname(os.path.abspath(__file__))
EXECUTOR = os.path.join(HERE, "..", "paper_2105_04663_b200", "executor.py")


def test_every_knob_the_executor_reads_is_registered():
    src = open(EXECUTOR).read()
    used = set(re.findall(r'_knob\("(SPMD_[A-Z0-9_]+)"\)', src))
    assert used and used <= set(knobs.KNOBS), used - set(knobs.KNOBS)
    assert "os.environ" not in src     # no plan-time environment reads outside the registry
    assert used == set(knobs.KNOBS), set(knobs.KNOBS) - used   # no dead knobs


def test_resolve_precedence(monkeypatch):
    monkeypatch.delenv("SPMD_RS_ADD", raising=False)
    assert knobs.resolve()["SPMD_RS_ADD"] == "1"
    monkeypatch.setenv("SPMD_RS_ADD", "0")
    assert knobs.resolve()["SPMD_RS_ADD"] == "0"
    assert knobs.resolve({"SPMD_RS_ADD": 1})["SPMD_RS_ADD"] == "1"
    with pytest.raises(KeyError):
        knobs.resolve({"SPMD_NO_SUCH_KNOB": "1"})


def _executor(**kw):
    g, _ = transformer_layer((1, 2), B=4, S=256, M=1024, N=8, D=64, H=4096, dtype=DType.BF16,
                             with_inputs=False)
    ann, _ = propagate(g)
    prog = partition(ann, 2, plan="fast")
    return Executor(prog, nparts=1, device="cpu", comm=FakeComm(), partition_base=0, fuse=True,
                    overlap=False, **kw)


@pytest.mark.parametrize("rs_add", ["0", "1"])
def test_override_switches_a_fusion(rs_add):
    ex = _executor(knobs={"SPMD_RS_ADD": rs_add})
    kinds = [v[0] for v in ex._fused.values()]
    assert kinds.count("dot_rs_add") == (2 if rs_add == "1" else 0)
    assert kinds.count("dot_rs") == (0 if rs_add == "1" else 2)


def test_knobs_are_read_once_per_executor(monkeypatch):
    monkeypatch.setenv("SPMD_FUSED_ATTENTION", "0")
    ex = _executor()
    monkeypatch.setenv("SPMD_FUSED_ATTENTION", "1")
    assert ex._knob("SPMD_FUSED_ATTENTION") == "0"
    assert "attention" not in {v[0] for v in ex._fused.values()}
