cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -q > gpurun_out/taps2_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/taps2_tests.log
for t in 1 0 1; do
SPMD_CONV_TAPS=$t timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/taps2_$t.log 2>&1
grep "^{" gpurun_out/taps2_$t.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('taps=$t', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 scripts/halo_conv_check.py > gpurun_out/taps2_hc2.log 2>&1; echo hc2=$?; grep "^{" gpurun_out/taps2_hc2.log
