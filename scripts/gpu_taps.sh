cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -q -x > gpurun_out/taps_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/taps_tests.log
for t in 1 0 1 0; do
SPMD_CONV_TAPS=$t timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/taps_$t.log 2>&1
grep "^{" gpurun_out/taps_$t.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('taps=$t', d['ms_per_step'], round(d['tflops_per_gpu'],1), d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
