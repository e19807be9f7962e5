cd $GRAFT_REPO_ROOT
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29541 scripts/peer_fusion_check.py --perf > gpurun_out/peer4.log 2>&1; echo peer4=$?
grep -v "^W1\|\*\*\*\|OMP_NUM" gpurun_out/peer4.log | tail -8
#$T --master-port 29543 scripts/multi_gpu_check.py > gpurun_out/multi4_peer.log 2>&1; echo multi4=$?
#tail -2 gpurun_out/multi4_peer.log
$T --master-port 29542 scripts/timeline.py > gpurun_out/tl4_peer.log 2>&1; echo tl=$?
grep -v "^W1\|\*\*\*\|OMP_NUM" gpurun_out/tl4_peer.log | tail -40
