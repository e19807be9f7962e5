cd $GRAFT_REPO_ROOT
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
SPMD_COMM_SMS=16 $T --master-port 29631 scripts/timeline.py > gpurun_out/tl4_a.log 2>&1; echo a=$?
SPMD_COMM_SMS=16 SPMD_COMM_PRIORITY=-1 $T --master-port 29632 scripts/timeline.py > gpurun_out/tl4_b.log 2>&1; echo b=$?
SPMD_COMM_SMS=32 SPMD_COMM_PRIORITY=-1 NCCL_PROTO=Simple $T --master-port 29633 scripts/timeline.py > gpurun_out/tl4_c.log 2>&1; echo c=$?
NCCL_MAX_NCHANNELS=8 SPMD_COMM_SMS=16 $T --master-port 29634 scripts/timeline.py > gpurun_out/tl4_d.log 2>&1; echo d=$?
