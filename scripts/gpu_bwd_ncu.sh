#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/bwd_kernels_once.py > gpurun_out/bwdk.log 2>&1; echo plain=$?; cat gpurun_out/bwdk.log
timeout 900 ncu --set full --clock-control none -k regex:"softmax_bwd|relu_bwd" -c 2 -o gpurun_out/bwd_kernels python scripts/bwd_kernels_once.py > gpurun_out/bwd_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/bwd_kernels.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/bwd_kernels_raw.csv 2>&1
cat gpurun_out/bwd_kernels_raw.csv | cut -c1-400 | head -8
