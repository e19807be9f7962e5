cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 300 python scripts/kernel_bench.py gemm > gpurun_out/ab_tma_$i.log 2>&1
SPMD_GEMM_EPI=direct timeout 300 python scripts/kernel_bench.py gemm > gpurun_out/ab_direct_$i.log 2>&1
done
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv > gpurun_out/ab_smi.txt
