cd $GRAFT_REPO_ROOT
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29571 scripts/peer_fusion_check.py > gpurun_out/lanes_check.log 2>&1; echo check=$?; grep "^{" gpurun_out/lanes_check.log | tail -3
for L in 2 1 2; do
SPMD_COMM_LANES=$L $T --master-port 2958$L bench.py --gpus 4 --no-e2e > gpurun_out/lanes_b$L.log 2>&1; echo b$L=$?
grep "^{" gpurun_out/lanes_b$L.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('lanes', $L, d['ms_per_step'], d['tflops_per_gpu'], d['clocks'])"
done
$T --master-port 29579 scripts/timeline.py > gpurun_out/tl4_lanes.log 2>&1; echo tl=$?
grep -v "^W1\|\*\*\*\|OMP_NUM" gpurun_out/tl4_lanes.log | head -16; tail -1 gpurun_out/tl4_lanes.log
