cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_parity.py -q -x -k "conv" > gpurun_out/cv_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/cv_tests.log
for m in 2sm 1sm 2sm; do
SPMD_CONV_MODE=$m timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/cv_$m.log 2>&1; echo $m=$?
grep "^{" gpurun_out/cv_$m.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$m', d['ms_per_step'], d['tflops_per_gpu'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"
done
