cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_peer.py tests/test_gpu_gemm.py -q -x > gpurun_out/w4_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/w4_tests.log
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29651 scripts/peer_fusion_check.py > gpurun_out/w4_peer.log 2>&1; echo peer=$?; grep "^{" gpurun_out/w4_peer.log | cut -c1-200
$T4 --master-port 29652 scripts/multi_gpu_check.py > gpurun_out/w4_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/w4_m4.log
$T4 --master-port 29653 bench.py --gpus 4 > gpurun_out/w4_b4.log 2>&1; echo b4=$?
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29654 bench.py --gpus 2 > gpurun_out/w4_b2.log 2>&1; echo b2=$?
for f in w4_b4 w4_b2; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['ms_per_step'], d['tflops_per_gpu'], d['mfu'], d['clocks'], d['e2e']['ms_per_step'])"; done
