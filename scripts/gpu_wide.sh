cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention.py -q -x > gpurun_out/wide_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/wide_tests.log
timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/wide_vs.log 2>&1; echo vs=$?; cat gpurun_out/wide_vs.log
SPMD_GEMM_MODE=2sm timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/wide_vs_old.log 2>&1; echo old=$?; cat gpurun_out/wide_vs_old.log
