cd $GRAFT_REPO_ROOT
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29511 scripts/multi_gpu_check.py > gpurun_out/multi2.log 2>&1; echo multi=$?
$T --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_graph.log 2>&1; echo b1=$?
$T --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-overlap > gpurun_out/bench_n2_nooverlap.log 2>&1; echo b2=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1_graph.log 2>&1; echo b3=$?
