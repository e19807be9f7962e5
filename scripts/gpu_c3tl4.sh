#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CFG=c3 $T4 --master-port 29688 scripts/timeline.py > gpurun_out/tl_c3_n4.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_c3_n4.log | tail -40
