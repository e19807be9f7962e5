cd $GRAFT_REPO_ROOT
CFG=c3 timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 scripts/timeline.py > gpurun_out/tl_c3_n4.log 2>&1; echo tl=$?
grep -v "^W1\|\*\*\*\|OMP_NUM\|NCCL version" gpurun_out/tl_c3_n4.log | tail -30
