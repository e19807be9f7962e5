#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for v in "SPMD_PEER_STAGE_WIDE=1" "SPMD_PEER_STAGE_WIDE=0" "SPMD_PEER_STAGE_WIDE=1" "SPMD_PEER_STAGE_WIDE=0" "SPMD_PEER_STAGE_WIDE=1" "SPMD_PEER_STAGE_WIDE=0"; do
  i=$((i+1))
  env SPMD_BENCH_MESH=1x4 $v $T4 --master-port 2970$i bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/sw_ab_$i.log 2>&1
  grep "^{" gpurun_out/sw_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('1x4 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw_ab_$i.log
done
SPMD_PEER_STAGE_WIDE=1 SPMD_BENCH_MESH=1x4 CFG=c2 $T4 --master-port 29688 scripts/timeline.py > gpurun_out/tl_sw.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_sw.log | tail -24
SPMD_PEER_STAGE_WIDE=1 $T4 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/sw_peer4.log 2>&1; echo peer4=$?; grep '"failed"' gpurun_out/sw_peer4.log | cut -c1-300
