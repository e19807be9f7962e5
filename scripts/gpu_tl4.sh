cd $GRAFT_REPO_ROOT
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 scripts/timeline.py > gpurun_out/tl4.log 2>&1; echo tl=$?
