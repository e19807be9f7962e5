set -x
# conv tap-reuse kernel at C4 dims (1 launch, 2nd launch of the c4 bench's conv)
bash scripts/ncu_top.sh r2_conv_taps conv_bf16_tcgen05_2sm 2 python bench.py --config c4 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-e2e
# wide GEMM FFN-in (spmd_gemm_bf16)
bash scripts/ncu_top.sh r2_gemm_wide_ffn gemm_bf16_tcgen05_2sm_wide 1 python scripts/gemm_raster.py 16384 65536 8192 --ncu
# MoE route / dispatch / combine (top-2) in the C3 step
ncu --set full --clock-control none -k regex:moe_ --launch-count 3 -o gpurun_out/r2_moe python bench.py --config c3 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/r2_moe.log 2>&1
ncu -i gpurun_out/r2_moe.ncu-rep --page raw --csv > gpurun_out/r2_moe_raw.csv 2>&1
python scripts/gemm_vs_cublas.py > gpurun_out/r2_gemm_vs_cublas.log 2>&1
ls gpurun_out | grep r2_ | tail -20
