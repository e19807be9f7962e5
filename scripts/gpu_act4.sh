#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for v in "SPMD_PEER_STAGE_ACT=1" "SPMD_PEER_STAGE_ACT=0" "SPMD_PEER_STAGE_ACT=1" "SPMD_PEER_STAGE_ACT=0" "SPMD_PEER_STAGE_ACT=1" "SPMD_PEER_STAGE_ACT=0"; do
  i=$((i+1))
  env SPMD_BENCH_MESH=1x4 $v $T4 --master-port 297$((10+i)) bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/a4_ab_$i.log 2>&1
  grep "^{" gpurun_out/a4_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('1x4 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/a4_ab_$i.log
done 2>&1 | tee gpurun_out/a4_summary.txt
