#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_peer.py -q -x 2>&1 | tail -2
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/cp_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/cp_m4.log | cut -c1-300
$T2 --master-port 29795 scripts/multi_gpu_check.py > gpurun_out/cp_m2.log 2>&1; echo m2=$?; tail -1 gpurun_out/cp_m2.log | cut -c1-300
$T4 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/cp_peer4.log 2>&1; echo peer4=$?; grep '"failed"' gpurun_out/cp_peer4.log | cut -c1-200
i=0
for v in "SPMD_PEER_CP=1" "SPMD_PEER_CP=0" "SPMD_PEER_CP=1" "SPMD_PEER_CP=0" "SPMD_PEER_CP=1" "SPMD_PEER_CP=0"; do
  i=$((i+1))
  env $v $T4 --master-port 297$((10+i)) bench.py --gpus 4 --config c4 --no-e2e --no-cpu-baseline > gpurun_out/cp_ab_$i.log 2>&1
  grep "^{" gpurun_out/cp_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('c4 n4 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/cp_ab_$i.log
done 2>&1 | tee gpurun_out/cp_summary.txt
for v in "SPMD_PEER_CP=1" "SPMD_PEER_CP=0"; do
  env $v $T2 --master-port 29731 bench.py --gpus 2 --config c4 --no-e2e --no-cpu-baseline > gpurun_out/cp_n2.log 2>&1
  grep "^{" gpurun_out/cp_n2.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('c4 n2 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" | tee -a gpurun_out/cp_summary.txt
done
