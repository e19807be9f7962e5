#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/sc_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/sc_m4.log | cut -c1-300
$T2 --master-port 29795 scripts/multi_gpu_check.py > gpurun_out/sc_m2.log 2>&1; echo m2=$?; tail -1 gpurun_out/sc_m2.log | cut -c1-300
CUDA_VISIBLE_DEVICES=0,1 $T2 --master-port 29796 scripts/halo_conv_check.py > gpurun_out/sc_halo2.log 2>&1; echo halo2=$?; tail -2 gpurun_out/sc_halo2.log | cut -c1-300
i=0
for v in "" "SPMD_PEER_CP=0" "" "SPMD_PEER_CP=0"; do
  i=$((i+1))
  env $v $T4 --master-port 297$((10+i)) bench.py --gpus 4 --config c4 --no-e2e --no-cpu-baseline > gpurun_out/sc_ab_$i.log 2>&1
  grep "^{" gpurun_out/sc_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('c4 n4 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sc_ab_$i.log
done 2>&1 | tee gpurun_out/sc_summary.txt
