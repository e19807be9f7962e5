#!/bin/bash
# C2 N=4 A/B: GEMM SM reservation for the comm lanes (SPMD_COMM_SMS), 2x2 and 1x4 meshes.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for mesh in 2x2 1x4; do
for r in 0 2 4 0 2 4; do
  i=$((i+1))
  SPMD_BENCH_MESH=$mesh SPMD_COMM_SMS=$r $T4 --master-port 2967$((i%10)) bench.py --gpus 4 --no-e2e --no-cpu-baseline > gpurun_out/absms_$i.log 2>&1
  grep "^{" gpurun_out/absms_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$mesh reserve=$r', round(d['ms_per_step'],3), round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/absms_$i.log
done; done 2>&1 | tee gpurun_out/absms_summary.txt
