cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29691 scripts/peer_fusion_check.py > gpurun_out/l4c_check.log 2>&1; echo check=$?; grep '"failed"' gpurun_out/l4c_check.log
$T4 --master-port 29692 scripts/multi_gpu_check.py > gpurun_out/l4c_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/l4c_m4.log
for c in c3 c4; do $T4 --master-port 2969$((3+${#c})) bench.py --gpus 4 --config $c --no-e2e > gpurun_out/l4c_$c.log 2>&1; echo $c=$?; grep "^{" gpurun_out/l4c_$c.log | cut -c1-160; done
i=0
for L in critical 1 critical 1; do
  i=$((i+1))
  SPMD_COMM_LANES=$L $T4 --master-port 2970$i bench.py --gpus 4 --no-e2e > gpurun_out/l4c_$i.log 2>&1
  grep "^{" gpurun_out/l4c_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('lanes=$L', d['ms_per_step'], round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done
