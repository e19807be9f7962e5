cd $GRAFT_REPO_ROOT
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 8 16 32; do
SPMD_COMM_SMS=$r $T --master-port 2962$r scripts/timeline.py > gpurun_out/tl4_sm$r.log 2>&1; echo tl$r=$?
done
