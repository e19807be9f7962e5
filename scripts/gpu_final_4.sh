#!/bin/bash
# Round-end multi-GPU benches: N=4 and N=2, every config (+ C2 on the 2x2 mesh).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for c in c2 c2train c3 c4; do
  i=$((i+1))
  $T4 --master-port 2980$i bench.py --gpus 4 --config $c > gpurun_out/f4_n4_$c.log 2>&1; echo n4_$c=$?
  $T2 --master-port 2981$i bench.py --gpus 2 --config $c > gpurun_out/f4_n2_$c.log 2>&1; echo n2_$c=$?
done
SPMD_BENCH_MESH=2x2 $T4 --master-port 29820 bench.py --gpus 4 > gpurun_out/f4_n4_c2_2x2.log 2>&1; echo n4_c2_2x2=$?
SPMD_BENCH_MESH=2x2 $T4 --master-port 29821 bench.py --gpus 4 --config c2train > gpurun_out/f4_n4_c2train_2x2.log 2>&1; echo n4_c2train_2x2=$?
$T4 --master-port 29822 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > gpurun_out/f4_n4_ref.log 2>&1; echo n4_ref=$?
for f in gpurun_out/f4_n*_c*.log; do grep "^{" $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$f'.split('/')[-1], d['n_gpus'], d['config'].get('mesh'), round(d['ms_per_step'],2), round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'], d['clocks'].get('reasons'), round(d['e2e']['ms_per_step'],2), d.get('reshard', {}) and list(d['reshard'].items())[:2])"; done
