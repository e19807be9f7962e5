cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29671 scripts/peer_fusion_check.py > gpurun_out/l4b_check.log 2>&1; echo check=$?; grep '"failed"' gpurun_out/l4b_check.log
i=0
for L in critical 1 critical 1; do
  i=$((i+1))
  SPMD_COMM_LANES=$L $T4 --master-port 2967$((i+1)) bench.py --gpus 4 --no-e2e > gpurun_out/l4b_$i.log 2>&1
  grep "^{" gpurun_out/l4b_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('lanes=$L', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"
done
$T4 --master-port 29679 scripts/timeline.py > gpurun_out/tl4_crit.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl4_crit.log | tail -22
