cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "train" > gpurun_out/train_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/train_tests.log
timeout 900 python bench.py --config c2train --no-cpu-baseline > gpurun_out/train_n1.log 2>&1; echo b1=$?
grep "^{" gpurun_out/train_n1.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['ms_per_step'], d['tflops_per_gpu'], d['mfu'], d['clocks'], d['config']['collectives_per_step'])"
tail -5 gpurun_out/train_n1.log | grep -i "error\|Trace" 
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29601 bench.py --gpus 4 --config c2train --no-e2e > gpurun_out/train_n4.log 2>&1; echo b4=$?
grep "^{" gpurun_out/train_n4.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['ms_per_step'], d['tflops_per_gpu'], d['mfu'], d['clocks'], d['config']['collectives_per_step'])"
grep -i "error\|Trace" gpurun_out/train_n4.log | head -5
