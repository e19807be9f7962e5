cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_peer.py -q > gpurun_out/peer_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/peer_tests.log
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29543 scripts/multi_gpu_check.py > gpurun_out/multi4_peer.log 2>&1; echo multi4=$?
tail -1 gpurun_out/multi4_peer.log
$T --master-port 29541 scripts/peer_fusion_check.py --perf > gpurun_out/peer4.log 2>&1; echo peer4=$?
grep "^{" gpurun_out/peer4.log
$T --master-port 29544 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench4_peer.log 2>&1; echo bench4=$?
grep "^{" gpurun_out/bench4_peer.log | cut -c1-900
