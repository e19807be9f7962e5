cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29761 bench.py --gpus 4 --no-e2e > gpurun_out/n4now.log 2>&1
grep "^{" gpurun_out/n4now.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"
$T4 --master-port 29762 scripts/timeline.py > gpurun_out/tl4_now.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl4_now.log | tail -30
