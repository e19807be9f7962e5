#!/bin/bash
# Final validation after the last changes: smoke, -m gpu suite, N=1 benches (GPU 0),
# then N=2 / N=4 C2 + C4 + C2 train.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/f3_gpu.log 2>&1; echo gpu=$?; tail -1 gpurun_out/f3_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/f3_n1_c2.log 2>&1; echo n1=$?
$T4 --master-port 29801 bench.py --gpus 4 > gpurun_out/f3_n4_c2.log 2>&1; echo n4=$?
SPMD_BENCH_MESH=2x2 $T4 --master-port 29802 bench.py --gpus 4 > gpurun_out/f3_n4_c2_2x2.log 2>&1; echo n4_2x2=$?
$T2 --master-port 29803 bench.py --gpus 2 > gpurun_out/f3_n2_c2.log 2>&1; echo n2=$?
$T4 --master-port 29804 bench.py --gpus 4 --config c4 > gpurun_out/f3_n4_c4.log 2>&1; echo n4c4=$?
$T4 --master-port 29805 bench.py --gpus 4 --config c2train > gpurun_out/f3_n4_c2train.log 2>&1; echo n4c2train=$?
for f in gpurun_out/f3_n*.log; do grep "^{" $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$f'.split('/')[-1], d['n_gpus'], d['config'].get('mesh'), round(d['ms_per_step'],2), round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'], d['clocks'].get('reasons'), round(d['e2e']['ms_per_step'],2), d['gpu_launches'])"; done
