"""Command line (paper_2105_04663_b200.cli) vs the reference ``minispmd``
command, recorded by tests/golden/make_cli_golden.py.

* propagate / partition / stats / pipeline and every error path: exit code,
  stdout, stderr and every artefact written are byte-identical.
* run / verify execute on the B200 (``-m gpu``): exit code, the printed
  output ids and shapes equal, values within the reference's 1e-4 metric
  (integers exact), and ``verify`` prints the same PASS line and collective
  counts.
* The reference's own tests/test_cli.py, restated.
"""

import gzip
import io
import json
import os
import re
import sys

import numpy as np
import pytest

from paper_2105_04663_b200.cli import main

HERE = os.path.dirname(os.path.abspath(__file__))
with gzip.open(os.path.join(HERE, "golden", "cli.json.gz"), "rt") as _f:
    RECORDS = json.load(_f)


def _executes(r):
    return r["argv"][0] in ("run", "verify") and r["code"] in (0, 1)


HOST = [r for r in RECORDS if not _executes(r)]
DEVICE = [r for r in RECORDS if _executes(r)]


def _id(r):
    return " ".join(r["argv"])[:80]


def _invoke(argv, files, tmp_path, monkeypatch, capsys):
    monkeypatch.chdir(tmp_path)
    monkeypatch.setattr(sys, "stdin", io.StringIO(""))
    for name, text in files.items():
        (tmp_path / name).write_text(text)
    capsys.readouterr()
    try:
        code = main(argv)
    except SystemExit as e:
        code = e.code
    cap = capsys.readouterr()
    wrote = {p.name: p.read_text() for p in sorted(tmp_path.iterdir()) if p.name not in files}
    return code, cap.out, cap.err, wrote


@pytest.mark.parametrize("rec", HOST, ids=_id)
def test_matches_reference_command(rec, tmp_path, monkeypatch, capsys):
    code, out, err, wrote = _invoke(rec["argv"], rec["files"], tmp_path, monkeypatch, capsys)
    assert code == rec["code"]
    assert out == rec["stdout"]
    assert err == rec["stderr"]
    assert wrote == rec["wrote"]


def test_fixture_covers_every_subcommand_and_exit_code():
    assert {r["argv"][0] for r in RECORDS} == {"propagate", "partition", "stats", "pipeline",
                                              "run", "verify"}
    assert {r["code"] for r in HOST} == {0, 2, 3}
    assert {r["code"] for r in DEVICE} == {0, 1} and len(DEVICE) >= 14


_NUM = re.compile(r"-?(?:\d+\.\d*|\d+)(?:e[-+]?\d+)?|True|False|nan|inf")


def _values(text):
    """``%id = array`` blocks -> (ids, list of number tokens per block)."""
    blocks = re.split(r"^%(\S+) = ", text, flags=re.M)[1:]
    ids, vals = blocks[0::2], []
    for body in blocks[1::2]:
        toks = _NUM.findall(body)
        vals.append([1.0 if t == "True" else 0.0 if t == "False" else float(t) for t in toks])
    return ids, vals


@pytest.mark.gpu
@pytest.mark.parametrize("rec", DEVICE, ids=_id)
def test_run_and_verify_on_b200(rec, tmp_path, monkeypatch, capsys):
    code, out, err, wrote = _invoke(rec["argv"], rec["files"], tmp_path, monkeypatch, capsys)
    assert code == rec["code"] and wrote == rec["wrote"]
    if rec["argv"][0] == "verify":
        tail = lambda s: (re.search(r"collectives=.*", s).group(0),
                          [_NUM.sub("#", x) for x in s.splitlines()[1:]])
        assert tail(out) == tail(rec["stdout"])
        return
    ids, got = _values(out)
    rids, want = _values(rec["stdout"])
    assert ids == rids
    for g, w in zip(got, want):
        g, w = np.array(g), np.array(w)
        assert g.shape == w.shape
        # printed with numpy's 8 significant digits: the reference metric
        assert np.max(np.abs(g - w), initial=0.0) <= 1e-4 * max(1.0, np.max(np.abs(w), initial=0))


# -- reference tests/test_cli.py restated --------------------------------------

FFW = next(r["files"]["ffw.txt"] for r in RECORDS if "ffw.txt" in r["files"])


@pytest.fixture
def ffw(tmp_path):
    p = tmp_path / "ffw.txt"
    p.write_text(FFW)
    return p


def test_propagate_annotates_all(ffw, capsys):
    assert main(["propagate", str(ffw)]) == 0
    assert capsys.readouterr().out.count("sharding=") >= 3


def test_propagate_trace_artifact(ffw, tmp_path):
    assert main(["propagate", str(ffw), "--trace"]) == 0
    trace = json.loads((tmp_path / "ffw.trace.json").read_text())
    assert "changes" in trace and "iterations" in trace


def test_partition_artifacts(ffw, tmp_path):
    assert main(["partition", str(ffw), "--devices", "4", "--dot"]) == 0
    assert (tmp_path / "ffw.spmd.txt").exists()
    stats = json.loads((tmp_path / "ffw.stats.json").read_text())
    assert "collective_counts" in stats and "sent_bytes" in stats
    dot = (tmp_path / "ffw.dot").read_text()
    assert dot.startswith("digraph") and "orange" in dot


def test_stats_keys(ffw, capsys):
    assert main(["stats", str(ffw), "--devices", "4"]) == 0
    assert set(json.loads(capsys.readouterr().out)) == {
        "collective_counts", "exchanged_bytes", "total_exchanged_bytes", "sent_bytes"}


def test_pipeline_bubble_ratio(capsys):
    assert main(["pipeline", "--stages", "4", "--microbatches", "16"]) == 0
    out = capsys.readouterr().out
    assert json.loads(out[out.rindex("\n{") + 1:])["bubble_ratio"] == [3, 19]


def test_exit_codes(tmp_path, capsys):
    assert main(["propagate", str(tmp_path / "missing.txt")]) == 2
    p = tmp_path / "bad.txt"
    p.write_text("graph @g {\n  %x = f32[8 parameter(0)\n  return %x\n}")
    assert main(["propagate", str(p)]) == 2
    assert "line 2" in capsys.readouterr().err
    assert main(["pipeline", "--stages", "2", "--microbatches", "4", "--schedule", "zigzag"]) == 2


def test_module_entry_point():
    import subprocess
    r = subprocess.run([sys.executable, "-m", "paper_2105_04663_b200", "pipeline", "--stages",
                        "2", "--microbatches", "2"], capture_output=True, text=True,
                       cwd=os.path.dirname(HERE), timeout=300)
    assert r.returncode == 0 and '"bubble_ratio"' in r.stdout
