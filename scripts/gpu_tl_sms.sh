#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 2 0; do
SPMD_BENCH_MESH=2x2 SPMD_COMM_SMS=$r CFG=c2 $T4 --master-port 2968$r scripts/timeline.py > gpurun_out/tl_sms$r.log 2>&1
echo "== reserve $r"; grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_sms$r.log | tail -28
done
