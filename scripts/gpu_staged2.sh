#!/bin/bash
# Staged gathers, lane placement: C2 2x2 and 1x4 at N=4, N=2 check, parity.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/st2_peer4.log 2>&1; echo peer4=$?; grep '"failed"' gpurun_out/st2_peer4.log | cut -c1-300
i=0
for m in 2x2 1x4 2x2 1x4; do
  i=$((i+1))
  env SPMD_BENCH_MESH=$m $T4 --master-port 2970$i bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/st2_ab_$i.log 2>&1
  grep "^{" gpurun_out/st2_ab_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$m', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/st2_ab_$i.log
done
SPMD_BENCH_MESH=2x2 CFG=c2 $T4 --master-port 29688 scripts/timeline.py > gpurun_out/tl_staged2.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_staged2.log | tail -28
