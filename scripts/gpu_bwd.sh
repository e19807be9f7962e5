#!/bin/bash
# Backward fusions: kernel + executor parity, train-step golden cases, c2train A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/bwd_tests.log 2>&1; echo "train tests rc=$?" >> gpurun_out/bwd_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k train >> gpurun_out/bwd_tests.log 2>&1; echo "parity rc=$?" >> gpurun_out/bwd_tests.log
for v in 0 1; do
  SPMD_BWD_FUSION=$v timeout 400 python bench.py --config c2train --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bwd_c2train_$v.json 2> gpurun_out/bwd_c2train_$v.err
done
tail -4 gpurun_out/bwd_tests.log
for v in 0 1; do grep "^{" gpurun_out/bwd_c2train_$v.json | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('bwd=$v', d['ms_per_step'], round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'], d['gpu_launches'], d['e2e']['value'])"; done
