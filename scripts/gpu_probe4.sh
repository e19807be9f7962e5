cd $GRAFT_REPO_ROOT
timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 scripts/nccl_probe.py > gpurun_out/probe4.log 2>&1; echo probe=$?
