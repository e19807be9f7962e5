#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/l_b1.log 2>&1; echo b1=$?
grep "^{" gpurun_out/l_b1.log | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['mfu']['vs_spec_2250'],3), d['clocks'], d['cpu_baseline'])"
