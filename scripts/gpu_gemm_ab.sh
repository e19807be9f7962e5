cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
timeout 120 python scripts/gemm_ab_once.py > gpurun_out/ab_once.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:"gemm|nvjet|sm100|cutlass|xmma" -s 2 -c 2 --csv python scripts/gemm_ab_once.py > gpurun_out/gemm_ab_ncu.csv 2>&1; echo ncu=$?
timeout 120 python scripts/gemm_ab_once.py 8192 8192 8192 > /dev/null 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:"gemm|nvjet|sm100|cutlass|xmma" -s 2 -c 2 --csv python scripts/gemm_ab_once.py 8192 8192 8192 > gpurun_out/gemm_ab_ncu_sq.csv 2>&1; echo ncu2=$?
