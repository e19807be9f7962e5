#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/lc_peer2.log 2>&1; echo peer2=$?; grep '"failed"' gpurun_out/lc_peer2.log | cut -c1-200
$T4 --master-port 29793 scripts/halo_conv_check.py > gpurun_out/lc_halo4.log 2>&1; echo halo4=$?; grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/lc_halo4.log | tail -4 | cut -c1-250
$T4 --master-port 29794 bench.py --gpus 4 --config c3 > gpurun_out/lc_c3.log 2>&1; echo c3=$?
$T2 --master-port 29795 bench.py --gpus 2 --config c2train > gpurun_out/lc_c2train2.log 2>&1; echo c2train2=$?
for f in gpurun_out/lc_c3.log gpurun_out/lc_c2train2.log; do grep "^{" $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$f'.split('/')[-1], d['n_gpus'], round(d['ms_per_step'],2), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"; done
