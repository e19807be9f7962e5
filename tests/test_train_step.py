"""C2 training step (forward + backward layer).

* The graph built with this package's IR equals the one the reference built
  for the golden fixtures (same function, ``api=minispmd``); the generic
  host-parity / oracle / GPU suites then cover its propagation, SPMD programs
  and outputs like every other golden case.
* The hand-written backward is the gradient: oracle vs float64 torch autograd.
* GSPMD weight-update sharding: every weight gradient leaves the partitioned
  program in its weight's sharding, produced by a reduce-scatter over the
  data axis (both planners).
"""

import numpy as np
import pytest

import golden_io as G
from paper_2105_04663_b200 import Op, partition, propagate
from paper_2105_04663_b200.ir import graph_to_json
from paper_2105_04663_b200.workloads import (train_step_inputs, transformer_flops,
                                             transformer_train_flops, transformer_train_step)

CASES = [c for c in G.cases("named") if "train" in c]
WEIGHTS = ("wq", "wk", "wv", "wo", "wi", "wt")


def test_golden_train_cases_present():
    assert [tuple(c["train"]["mesh"]) for c in CASES] == [(1, 2), (2, 2), (2, 4)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_builder_matches_reference_graph(case):
    g = transformer_train_step(tuple(case["train"]["mesh"]), **case["train"]["dims"])
    assert graph_to_json(g) == case["graph"]


def test_backward_is_the_gradient():
    torch = pytest.importorskip("torch")
    from oracle import evaluator as O
    dims = dict(B=2, S=8, M=16, N=4, D=4, H=32)
    ins = train_step_inputs(**dims, seed=3)
    got = O.evaluate_single(transformer_train_step((1, 1), **dims), ins)
    t = [torch.tensor(a, dtype=torch.float64, requires_grad=True) for a in ins[:7]]
    x, wq, wk, wv, wo, wi, wt = t
    q, k, v = (torch.einsum("bsm,mnd->bsnd", x, w) for w in (wq, wk, wv))
    p = torch.softmax(torch.einsum("bsnd,btnd->bnst", q, k), -1)
    ctx = torch.einsum("bnst,btnd->bnsd", p, v).permute(0, 2, 1, 3)
    res1 = torch.einsum("bsnd,ndm->bsm", ctx, wo) + x
    out = torch.einsum("bsh,hm->bsm", torch.relu(torch.einsum("bsm,mh->bsh", res1, wi)),
                       wt) + res1
    (out * torch.tensor(ins[7], dtype=torch.float64)).sum().backward()
    want = [out.detach()] + [a.grad for a in t]
    for a, b in zip(got, want):
        b = b.numpy()
        assert np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))) < 1e-5


@pytest.mark.parametrize("mesh", [(1, 2), (2, 2), (2, 4)])
@pytest.mark.parametrize("plan", ["reference", "fast"])
def test_weight_gradients_are_reduce_scattered_into_weight_shards(mesh, plan):
    g = transformer_train_step(mesh, B=4, S=8, M=16, N=8, D=4, H=32)
    ann, _ = propagate(g)
    prog = partition(ann, mesh[0] * mesh[1], plan=plan)
    params = {p.id: p.sharding for p in ann.parameters}
    # outputs: out, dx, d_wq, d_wk, d_wv, d_wo, d_wi, d_wt
    for w, s in zip(WEIGHTS, prog.output_shardings[2:]):
        assert s == params[w], (w, s.format(), params[w].format())
    assert prog.output_shardings[1] == params["x"]
    n_rs = sum(1 for i in prog.graph.instructions if i.opcode == Op.REDUCE_SCATTER)
    assert n_rs >= 6 if mesh[0] > 1 else n_rs >= 1


def test_train_flops_are_three_forwards():
    d = dict(B=16, S=1024, M=8192, N=128, D=256, H=65536)
    assert transformer_train_flops(**d) == 3 * transformer_flops(**d)
