cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 1 2; do for H in ce sm nccl; do
SPMD_BENCH_MESH=2x2 SPMD_PEER_HIDDEN_ENGINE=$H $T4 --master-port 29851 bench.py --gpus 4 --no-e2e > gpurun_out/jit2_$H.log 2>&1
grep "^{" gpurun_out/jit2_$H.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('jit hidden=$H', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"
done; done
SPMD_BENCH_MESH=2x2 SPMD_PEER_HIDDEN_ENGINE=sm $T4 --master-port 29853 scripts/timeline.py > gpurun_out/tl4_jit_sm.log 2>&1
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl4_jit_sm.log | grep "all_gather\|dot\|reduce\|relu\|transpose\|total"
