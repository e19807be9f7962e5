cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -q -x > gpurun_out/pipe_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/pipe_tests.log
grep -c "pipe_" gpurun_out/pipe_tests.log
T="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29591 scripts/multi_gpu_check.py > gpurun_out/pipe_multi4.log 2>&1; echo multi4=$?; tail -1 gpurun_out/pipe_multi4.log
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29592 scripts/multi_gpu_check.py > gpurun_out/pipe_multi2.log 2>&1; echo multi2=$?; tail -1 gpurun_out/pipe_multi2.log
