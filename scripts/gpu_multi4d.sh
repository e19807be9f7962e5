cd $GRAFT_REPO_ROOT
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29531 scripts/nccl_probe.py > gpurun_out/probe4.log 2>&1; echo probe=$?
$T --master-port 29521 scripts/multi_gpu_check.py > gpurun_out/multi4.log 2>&1; echo multi=$?
