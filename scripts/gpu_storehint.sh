cd $GRAFT_REPO_ROOT
for h in 0 1; do
  SPMD_GEMM_STORE_HINT=$h timeout 300 python scripts/kernel_bench.py gemm > gpurun_out/sh_$h.log 2>&1; echo kb$h=$?
done
for h in 0 1; do
  SPMD_GEMM_STORE_HINT=$h timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_bf16 -s 2 -c 1 --csv python scripts/gemm_once.py 16384 65536 8192 > gpurun_out/sh_ncu_$h.csv 2>&1; echo ncu$h=$?
done
paste gpurun_out/sh_0.log gpurun_out/sh_1.log | cut -c1-250
grep -h "dram__\|lts__\|gpu__time\|cycles_elapsed" gpurun_out/sh_ncu_*.csv | cut -d, -f13- 
