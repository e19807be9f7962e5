cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention.py tests/test_gpu_peer.py tests/test_gpu_parity.py -q -x > gpurun_out/tl_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/tl_tests.log
timeout 300 python scripts/kernel_bench.py attention > gpurun_out/tl_attn.log 2>&1; cat gpurun_out/tl_attn.log
timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/tl_vs.log 2>&1; cat gpurun_out/tl_vs.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/tl_b1.log 2>&1
grep "^{" gpurun_out/tl_b1.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"
