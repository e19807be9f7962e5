#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/st_m2.log 2>&1; echo m2=$?; tail -1 gpurun_out/st_m2.log
i=0
for v in "" "SPMD_PEER_STAGE=0" "" "SPMD_PEER_STAGE=0"; do
  i=$((i+1))
  env $v $T2 --master-port 2970$i bench.py --gpus 2 --no-e2e --no-cpu-baseline > gpurun_out/stn2_ab_$i.log 2>&1
  grep "^{" gpurun_out/stn2_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('n2 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/stn2_ab_$i.log
done
