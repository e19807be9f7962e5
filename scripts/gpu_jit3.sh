cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 1 2; do for D in 1 2 asap; do
if [ $D = asap ]; then E="SPMD_PREFETCH=asap"; else E="SPMD_PREFETCH_DEPTH=$D"; fi
env SPMD_BENCH_MESH=2x2 $E $T4 --master-port 29861 bench.py --gpus 4 --no-e2e > gpurun_out/jit3_$D.log 2>&1
grep "^{" gpurun_out/jit3_$D.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('depth=$D', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'])"
done; done
