cd $GRAFT_REPO_ROOT
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29545 scripts/peer_fusion_check.py > gpurun_out/peer4c.log 2>&1; echo peer4=$?
grep "^{" gpurun_out/peer4c.log; grep -i "Traceback\|Error" gpurun_out/peer4c.log | head -5
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29546 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench2_peer.log 2>&1; echo bench2=$?
grep "^{" gpurun_out/bench2_peer.log | cut -c1-700
