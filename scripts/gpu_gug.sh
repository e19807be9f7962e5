#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GEMM_RESERVE=0,2,4 GATHER_KINDS=ce,sm_bg timeout 400 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/gather_under_gemm.py 2>&1 | grep "^{\|Error\|error" | tee gpurun_out/gug_n2_ce_reserve.jsonl
