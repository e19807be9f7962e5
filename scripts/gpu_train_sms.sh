#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for v in "SPMD_COMM_SMS=2" "SPMD_COMM_SMS=0" "SPMD_COMM_SMS=2" "SPMD_COMM_SMS=0"; do
  i=$((i+1))
  env $v $T4 --master-port 297$((10+i)) bench.py --gpus 4 --config c2train --no-e2e --no-cpu-baseline > gpurun_out/ts_ab_$i.log 2>&1
  grep "^{" gpurun_out/ts_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('c2train n4 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ts_ab_$i.log
done 2>&1 | tee gpurun_out/ts_summary.txt
