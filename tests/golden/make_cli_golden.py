"""Record the reference command line's behaviour -> ``tests/golden/cli.json.gz``.

Run in the build container (the reference never travels to the GPU box)::

    cp -r /root/reference/pkg /tmp/refpkg        # never write into /root/reference
    PYTHONPATH=/tmp/refpkg/src:/root/repo python tests/golden/make_cli_golden.py

Inputs are the reference-printed graph texts already pinned in
``textir.json.gz`` (named cases + every 6th random case) plus the reference
test-suite graphs (``tests/test_cli.py``).  Every invocation runs
``minispmd.cli.main(argv)`` in a scratch directory holding ``<name>.txt``
and records exit code, stdout, stderr and every file it wrote.  ``run`` and
``verify`` are recorded too; their numbers come from the reference's f64
evaluator and are compared numerically by the GPU tests.
"""

from __future__ import annotations

import contextlib
import gzip
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))

FFW = """\
graph @ffw (mesh=[2,2]) {
  %x = f32[8,8] parameter(0), sharding={devices=[2,2]0,1,2,3}
  %w = f32[8,8] parameter(1), sharding={devices=[2,2]0,2,1,3}
  %y = f32[8,8] dot(%x, %w), lhs_batch=[], rhs_batch=[], lhs_contracting=[1], rhs_contracting=[0], sharding={devices=[2,2]0,1,2,3}
  return %y
}
"""

REPLICATED = """\
graph @r {
  %x = f32[4] parameter(0)
  %y = f32[4] relu(%x)
  return %y
}
"""

INTS = """\
graph @ints (mesh=[4]) {
  %a = s32[8,6] parameter(0), sharding={devices=[4,1]0,1,2,3}
  %b = s32[8,6] parameter(1)
  %c = s32[8,6] multiply(%a, %b)
  %z = s32[] constant(), literal=0
  %s = s32[6] reduce(%c, %z), kind=sum, dims=[0]
  %m = pred[8,6] compare(%a, %b), direction=gt
  return %s, %m
}
"""

UNEVEN = """\
graph @uneven (mesh=[4]) {
  %x = f32[10,3] parameter(0), sharding={devices=[4,1]0,1,2,3}
  %z = f32[] constant(), literal=0.0
  %s = f32[3] reduce(%x, %z), kind=sum, dims=[0]
  return %s
}
"""

BAD = {
    "parse_error": "graph @g {\n  %x = f32[8 parameter(0)\n  return %x\n}",
    "dup_device": "%x = f32[8] parameter(0), sharding={devices=[2]0,0}",
    "bare": "%x = f32[8] parameter(0), sharding={devices=[2]0,1}",
    "use_before_def": "graph @g {\n  %y = f32[4] relu(%x)\n  %x = f32[4] parameter(0)\n"
                      "  return %y\n}",
    "bad_shape": "graph @g {\n  %x = f32[4] parameter(0)\n  %y = f32[5] relu(%x)\n"
                 "  return %y\n}",
    "conflict": "graph @g (mesh=[2]) {\n  %x = f32[4,4] parameter(0), sharding={devices=[2,1]0,1}\n"
                "  %y = f32[4,4] relu(%x), sharding={devices=[1,2]0,1}\n  return %y\n}",
}


def _invoke(main, argv, files):
    with tempfile.TemporaryDirectory() as tmp:
        cwd = os.getcwd()
        os.chdir(tmp)
        try:
            for name, text in files.items():
                with open(name, "w") as f:
                    f.write(text)
            out, err = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
                try:
                    code = main(argv)
                except SystemExit as e:      # argparse usage errors
                    code = e.code
            wrote = {}
            for name in sorted(os.listdir(tmp)):
                if name not in files:
                    with open(name) as f:
                        wrote[name] = f.read()
        finally:
            os.chdir(cwd)
    return {"argv": argv, "files": files, "code": code, "stdout": out.getvalue(),
            "stderr": err.getvalue(), "wrote": wrote}


def _collective_text():
    """A graph that already holds a collective (partition refuses it: exit 3)."""
    import minispmd as R
    from minispmd.textir import print_graph
    mesh = R.DeviceMesh.default(2)
    b = R.GraphBuilder("coll", mesh)
    x = b.parameter(R.Shape((4,)), sharding=R.mesh_split(1, mesh, [-1]))
    y = b.add(R.Op.ALL_REDUCE, [x], {"kind": R.ReduceKind.SUM, "subgroups": ((0, 1),)})
    return print_graph(b.build([y]))


FEATURE_CONV = """\
graph @fconv (mesh=[2]) {
  %x = f32[2,4,16] parameter(0), sharding={devices=[1,2,1]0,1}
  %k = f32[4,4,3] parameter(1), sharding={replicated}
  %y = f32[2,4,16] convolution(%x, %k), conv_dims={lhs_batch=0,lhs_feature=1,lhs_spatial=[2],rhs_in_feature=0,rhs_out_feature=1,rhs_spatial=[2],out_batch=0,out_feature=1,out_spatial=[2]}, window=[{size=3,stride=1,padding_low=1,padding_high=1,base_dilation=1,window_dilation=1}], sharding={devices=[1,2,1]0,1}
  return %y
}
"""


def invocations():
    with gzip.open(os.path.join(HERE, "textir.json.gz"), "rt") as f:
        texts = json.load(f)["graphs"]
    with gzip.open(os.path.join(HERE, "named.json.gz"), "rt") as f:
        ndev = {c["name"]: c["num_devices"] for c in json.load(f)}
    with gzip.open(os.path.join(HERE, "random.json.gz"), "rt") as f:
        ndev.update({c["name"]: c["num_devices"] for c in json.load(f)})
    graphs = {"ffw": (FFW, 4), "r": (REPLICATED, 4), "ints": (INTS, 4), "uneven": (UNEVEN, 4)}
    for name, entry in texts.items():
        if name.startswith("rand") and int(name[4:]) % 6:
            continue
        graphs[name] = (entry["graph"], ndev[name])
    inv = []
    for name, (text, n) in graphs.items():
        files = {f"{name}.txt": text}
        src = f"{name}.txt"
        inv.append((["propagate", src, "--trace", "--dot"], files))
        inv.append((["partition", src, "--devices", str(n), "--dot"], files))
        inv.append((["stats", src, "--devices", str(n)], files))
        if name in ("ffw", "r", "ints", "uneven", "c1_acceptance", "c5_uneven_1001"):
            inv.append((["propagate", src, "--no-priorities", "-o", "np.spmd.txt"], files))
            inv.append((["partition", "-", "--devices", str(n)], {}))   # stdin: empty
    # small graphs the GPU tests run through run / verify
    for name in ("ffw", "r", "ints", "uneven"):
        text, n = graphs[name]
        files = {f"{name}.txt": text}
        inv.append((["run", f"{name}.txt"], files))
        inv.append((["run", f"{name}.txt", "--devices", str(n), "--seed", "3"], files))
        inv.append((["verify", f"{name}.txt", "--devices", str(n)], files))
    inv.append((["verify", "ffw.txt", "--devices", "4", "--tol", "-1"], {"ffw.txt": FFW}))
    inv.append((["run", "fconv.txt", "--devices", "2"], {"fconv.txt": FEATURE_CONV}))
    inv.append((["verify", "fconv.txt", "--devices", "2"], {"fconv.txt": FEATURE_CONV}))
    inv.append((["run", "r.txt", "--inputs", "in.json"],
                {"r.txt": REPLICATED, "in.json": "[[1.0, -2.0, 3.0, -4.0]]"}))
    inv.append((["run", "r.txt", "--inputs", "in.json"],
                {"r.txt": REPLICATED, "in.json": "[[1.0, -2.0]]"}))
    inv.append((["run", "r.txt", "--inputs", "in.json"], {"r.txt": REPLICATED, "in.json": "[1,"}))
    inv.append((["run", "r.txt", "--inputs", "in.json"], {"r.txt": REPLICATED, "in.json": "[]"}))
    for sched, s, m, dims in [("gpipe", 4, 16, ["4"]), ("circular:2", 2, 4, ["4"]),
                              ("circular", 2, 4, ["2", "3"]), ("gpipe", 1, 1, []),
                              ("circular:3", 4, 8, ["8"]), ("zigzag", 2, 4, ["4"]),
                              ("circular:x", 2, 4, ["4"]), ("gpipe", 0, 4, ["4"]),
                              ("circular:2", 4, 3, ["4"])]:
        argv = ["pipeline", "--stages", str(s), "--microbatches", str(m), "--schedule", sched]
        if dims:
            argv += ["--state-dims"] + dims
        inv.append((argv, {}))
    inv.append((["pipeline", "--stages", "2", "--microbatches", "4", "-o", "pp", "--dot"], {}))
    inv.append((["propagate", "no-such-file.txt"], {}))
    for name, text in list(BAD.items()) + [("coll", _collective_text()),
                                           ("fconv", FEATURE_CONV)]:
        inv.append((["propagate", f"{name}.txt"], {f"{name}.txt": text}))
        inv.append((["partition", f"{name}.txt", "--devices", "2"], {f"{name}.txt": text}))
    return inv


def main():
    from minispmd.cli import main as ref_main
    rec = [_invoke(ref_main, argv, files) for argv, files in invocations()]
    with gzip.open(os.path.join(HERE, "cli.json.gz"), "wt") as f:
        json.dump(rec, f, sort_keys=True)
    codes = {}
    for r in rec:
        codes[r["code"]] = codes.get(r["code"], 0) + 1
    print("invocations:", len(rec), "exit codes:", codes)


if __name__ == "__main__":
    sys.exit(main())
