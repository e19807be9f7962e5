cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"
timeout 120 python scripts/conv_once.py > gpurun_out/conv_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 1 -c 1 -o gpurun_out/conv2sm_full python scripts/conv_once.py > gpurun_out/ncu_conv.log 2>&1; echo conv=$?
timeout 300 python scripts/kernel_bench.py attention > gpurun_out/attn_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention -s 3 -c 1 -o gpurun_out/attn_full python scripts/kernel_bench.py attention > gpurun_out/ncu_attn.log 2>&1; echo attn=$?
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r1b.csv python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1; echo list=$?
for r in conv2sm_full attn_full; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; done
ls -la gpurun_out/*.ncu-rep
