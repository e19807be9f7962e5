cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for m in 1x4 2x2 1x4 2x2; do
SPMD_BENCH_MESH=$m $T4 --master-port 29820 bench.py --gpus 4 --no-e2e > gpurun_out/mesh_$m.log 2>&1
grep "^{" gpurun_out/mesh_$m.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('mesh=$m', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['config']['collectives_per_step'], d['clocks']['sm_mhz'])"
done
