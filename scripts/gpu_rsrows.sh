cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/rr_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/rr_tests.log
for n in 2 4; do
timeout 1200 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2974$n scripts/peer_fusion_check.py > gpurun_out/rr_check$n.log 2>&1; echo check$n=$?; grep "direct\|train\|failed" gpurun_out/rr_check$n.log | tail -3; grep -i "Traceback\|Error" gpurun_out/rr_check$n.log | head -3
done
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for F in 1 0; do
SPMD_PEER_FUSION=$F $T4 --master-port 29750 bench.py --gpus 4 --config c2train --no-e2e > gpurun_out/rr_train_$F.log 2>&1; echo tr$F=$?
grep "^{" gpurun_out/rr_train_$F.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('fusion=$F', d['ms_per_step'], round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done
