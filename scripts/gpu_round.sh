cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo gpu=$?
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo b1=$?
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29661 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1; echo b2=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_n1.log 2>&1; echo ref=$?
