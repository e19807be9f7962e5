#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/fk_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/fk_m4.log | cut -c1-300
$T4 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/fk_peer4.log 2>&1; echo peer4=$?; grep '"failed"' gpurun_out/fk_peer4.log | cut -c1-300
i=0
for v in "SPMD_PEER_SERIAL_PULLS=0" "SPMD_PEER_SERIAL_PULLS=1" "SPMD_PEER_SERIAL_PULLS=0" "SPMD_PEER_SERIAL_PULLS=1" "SPMD_PEER_SERIAL_PULLS=0" "SPMD_PEER_SERIAL_PULLS=1"; do
  i=$((i+1))
  env SPMD_BENCH_MESH=1x4 $v $T4 --master-port 297$((10+i)) bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/fk_ab_$i.log 2>&1
  grep "^{" gpurun_out/fk_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('1x4 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/fk_ab_$i.log
done 2>&1 | tee gpurun_out/fk_summary.txt
SPMD_BENCH_MESH=1x4 CFG=c2 $T4 --master-port 29688 scripts/timeline.py > gpurun_out/tl_fk.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_fk.log | tail -22 | head -12
