cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rg_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/rg_gpu.log 2>&1; echo gpu=$?; tail -1 gpurun_out/rg_gpu.log
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T2 --master-port 29641 scripts/multi_gpu_check.py > gpurun_out/rg_m2.log 2>&1; echo m2=$?; tail -1 gpurun_out/rg_m2.log
$T4 --master-port 29642 scripts/multi_gpu_check.py > gpurun_out/rg_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/rg_m4.log
timeout 600 python bench.py > gpurun_out/rg_b1.log 2>&1; echo b1=$?
$T4 --master-port 29643 bench.py --gpus 4 > gpurun_out/rg_b4.log 2>&1; echo b4=$?
$T2 --master-port 29644 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/rg_ref2.log 2>&1; echo ref2=$?
for f in rg_b1 rg_b4 rg_ref2; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('impl','ours'), d['n_gpus'], d['ms_per_step'], d.get('tflops_per_gpu'), d.get('mfu'), d.get('clocks'), (d.get('e2e') or {}).get('ms_per_step'))"; done
