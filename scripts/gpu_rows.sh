#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python scripts/transpose_once.py; SPMD_COPY_NO_ROWS=1 timeout 120 python scripts/transpose_once.py
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for v in "" "SPMD_COPY_NO_ROWS=1" "" "SPMD_COPY_NO_ROWS=1"; do
  env $v timeout 600 python bench.py --config c2train --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rows_ab.log 2>&1
  grep "^{" gpurun_out/rows_ab.log | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c2train [$v]', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
