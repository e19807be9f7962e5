cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/moe_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/moe_tests.log
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/c3_n1.log 2>&1; echo c3=$?
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29611 bench.py --gpus 4 --config c3 --no-e2e > gpurun_out/c3_n4.log 2>&1; echo c3n4=$?
for f in c3_n1 c3_n4; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['ms_per_step'], d['tflops_per_gpu'], d['config'].get('dispatch_combine','dense'), d['clocks'])"; done
grep -i "Traceback\|Error" gpurun_out/c3_n*.log | head -5
