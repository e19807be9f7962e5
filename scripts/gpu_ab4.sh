cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for m in 3 2 3 2; do
  i=$((i+1))
  if [ $m = 2 ]; then E="SPMD_GEMM_MODE=2sm"; else E="SPMD_GEMM_MODE=wide"; fi
  env $E $T4 --master-port 2966$i bench.py --gpus 4 --no-e2e > gpurun_out/ab4_$i.log 2>&1
  grep "^{" gpurun_out/ab4_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('mode$m', d['ms_per_step'], round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done
CFG=c2 $T4 --master-port 29669 scripts/timeline.py > gpurun_out/tl4_wide.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl4_wide.log | tail -30
