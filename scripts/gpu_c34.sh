cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_n1.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3_n1.log 2>&1; echo c3=$?
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29551 bench.py --gpus 2 --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_n2.log 2>&1; echo c4n2=$?
$T --master-port 29552 bench.py --gpus 2 --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3_n2.log 2>&1; echo c3n2=$?
