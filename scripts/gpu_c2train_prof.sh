#!/bin/bash
# c2train launch list (per-kernel durations, one step) for the kernel breakdown.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--config c2train --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/c2t_plain.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c2t_launches.csv python bench.py $ARGS > gpurun_out/c2t_ncu.log 2>&1; echo list=$?
