#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/ph_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/ph_m4.log | cut -c1-300
i=0
for m in 2x2 1x4; do
for v in "SPMD_STAGE_PHASES=2" "SPMD_STAGE_PHASES=1" "SPMD_STAGE_PHASES=2" "SPMD_STAGE_PHASES=1" "SPMD_STAGE_PHASES=2" "SPMD_STAGE_PHASES=1"; do
  i=$((i+1))
  env SPMD_BENCH_MESH=$m $v $T4 --master-port 297$((10+i)) bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/ph_ab_$i.log 2>&1
  grep "^{" gpurun_out/ph_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$m [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ph_ab_$i.log
done; done 2>&1 | tee gpurun_out/ph_summary.txt
