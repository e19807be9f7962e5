cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_moe.py -q > gpurun_out/moe.log 2>&1; echo moe=$?
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_reshard.log 2>&1; echo b2=$?
