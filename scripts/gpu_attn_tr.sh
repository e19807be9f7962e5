cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_parity.py -q -x > gpurun_out/at_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/at_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/at_b1.log 2>&1; echo b1=$?
grep "^{" gpurun_out/at_b1.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], round(d['tflops_per_gpu'],1), d['mfu'], d['clocks'], d['gpu_launches'])"
