#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/p4_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/p4_m4.log | cut -c1-400
SPMD_PEER_STAGE_ACT=1 $T4 --master-port 29793 scripts/multi_gpu_check.py > gpurun_out/p4_m4_act.log 2>&1; echo m4act=$?; tail -1 gpurun_out/p4_m4_act.log | cut -c1-400
SPMD_PEER_STAGE=0 $T4 --master-port 29794 scripts/multi_gpu_check.py > gpurun_out/p4_m4_nostage.log 2>&1; echo m4nostage=$?; tail -1 gpurun_out/p4_m4_nostage.log | cut -c1-400
$T2 --master-port 29795 scripts/multi_gpu_check.py > gpurun_out/p4_m2.log 2>&1; echo m2=$?; tail -1 gpurun_out/p4_m2.log | cut -c1-400
