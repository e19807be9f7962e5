cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo gpu=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3_n1.log 2>&1; echo c3=$?
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3_n2.log 2>&1; echo c3n2=$?
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 scripts/multi_gpu_check.py > gpurun_out/multi2.log 2>&1; echo multi=$?
