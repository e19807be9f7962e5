cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29841 scripts/peer_fusion_check.py > gpurun_out/jit_check.log 2>&1; echo check=$?; grep '"failed"' gpurun_out/jit_check.log
for P in jit asap jit asap; do
SPMD_BENCH_MESH=2x2 SPMD_PREFETCH=$P $T4 --master-port 29842 bench.py --gpus 4 --no-e2e > gpurun_out/jit_$P.log 2>&1
grep "^{" gpurun_out/jit_$P.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('prefetch=$P', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"
done
SPMD_BENCH_MESH=2x2 $T4 --master-port 29843 scripts/timeline.py > gpurun_out/tl4_jit.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl4_jit.log | grep "all_gather\|dot\|reduce\|relu\|transpose\|total"
