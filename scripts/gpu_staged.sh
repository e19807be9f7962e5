#!/bin/bash
# Pre-staged weight gathers: parity at N=4, then C2 2x2 A/B (staged / not staged / staged+reserve).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/st_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/st_m4.log
$T4 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/st_peer4.log 2>&1; echo peer4=$?; grep '"failed"' gpurun_out/st_peer4.log | cut -c1-300
i=0
for v in "" "SPMD_PEER_STAGE=0" "SPMD_COMM_SMS=2" "" "SPMD_PEER_STAGE=0" "SPMD_COMM_SMS=2"; do
  i=$((i+1))
  env SPMD_BENCH_MESH=2x2 $v $T4 --master-port 2970$i bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/st_ab_$i.log 2>&1
  grep "^{" gpurun_out/st_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('2x2 [$v]', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/st_ab_$i.log
done
SPMD_BENCH_MESH=2x2 CFG=c2 $T4 --master-port 29688 scripts/timeline.py > gpurun_out/tl_staged.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_staged.log | tail -28
