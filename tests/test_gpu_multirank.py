"""Multi-rank parity on a multi-GPU box (skipped with fewer than 2 GPUs).

One process per GPU (torchrun, NCCL + the CUDA-IPC peer heap):

* ``scripts/multi_gpu_check.py``: every golden case whose device count equals
  the world size runs the reference's SPMD program per rank with NCCL
  collectives against the reference's recorded per-device outputs (ints
  exact, f32 1e-5), then the fast plan with fusions end to end -- including
  the world-2/4 uneven (C5) cases.
* ``scripts/peer_fusion_check.py``: fused dot -> reduce-scatter issued back
  to back with different sizes and subgroups and no host sync (the fixed
  parity stride), row-split reduce-scatters, the layer / training step /
  MoE layer with peer fusions vs NCCL only.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _torchrun(script, n, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29561", os.path.join(ROOT, script)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    sys.stdout.write(r.stdout[-4000:])
    sys.stderr.write(r.stderr[-4000:])
    return r.returncode


@pytest.mark.parametrize("n", [2, 4])
def test_multi_gpu_golden_parity(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun("scripts/multi_gpu_check.py", n) == 0


@pytest.mark.parametrize("n", [2, 4])
def test_peer_fusion_parity(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun("scripts/peer_fusion_check.py", n) == 0
