cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py tests/test_gpu_moe.py -q -x > gpurun_out/tmastore_tests.log 2>&1; echo tests=$?
timeout 300 python scripts/kernel_bench.py gemm > gpurun_out/kbench_tmastore.log 2>&1; echo kb=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1_tmastore.log 2>&1; echo b=$?
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_n1b.log 2>&1; echo c4=$?
