cd $GRAFT_REPO_ROOT
timeout 180 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm2.log 2>&1; echo gemm=$?
timeout 180 python scripts/kernel_bench.py gemm > gpurun_out/kbench_2sm.log 2>&1; echo k2=$?
SPMD_GEMM_MODE=1sm timeout 180 python scripts/kernel_bench.py gemm > gpurun_out/kbench_1sm.log 2>&1; echo k1=$?
