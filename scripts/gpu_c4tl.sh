cd $GRAFT_REPO_ROOT
CFG=c4 timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 scripts/timeline.py > gpurun_out/tl_c4_n2.log 2>&1; echo tl=$?
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_c4_n2.log | tail -45
