cd $GRAFT_REPO_ROOT
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 scripts/peer_ag_bench.py > gpurun_out/agbench4.log 2>&1; echo ag=$?
grep "^{" gpurun_out/agbench4.log; grep -i "error\|Traceback" gpurun_out/agbench4.log | head
