cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py -q -x -k "two_streams or verify_equivalence or partitioned" > gpurun_out/halo_tests.log 2>&1; echo t=$?
timeout 300 python scripts/c4_local_profile.py 2 > gpurun_out/c4prof.log 2>&1; echo prof=$?
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29571 bench.py --gpus 2 --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_n2.log 2>&1; echo c4n2=$?
