cd $GRAFT_REPO_ROOT
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
A="bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e"
i=0
for cfg in "SPMD_COMM_SMS=0" "SPMD_COMM_SMS=32 SPMD_COMM_PRIORITY=-1 NCCL_PROTO=Simple" "SPMD_COMM_SMS=24 SPMD_COMM_PRIORITY=-1 NCCL_PROTO=Simple" "SPMD_COMM_SMS=48 SPMD_COMM_PRIORITY=-1 NCCL_PROTO=Simple" "SPMD_COMM_SMS=0 SPMD_COMM_PRIORITY=-1 NCCL_PROTO=Simple" "SPMD_COMM_SMS=32 SPMD_COMM_PRIORITY=-1"; do
i=$((i+1))
env $cfg $T --master-port 2964$i $A > gpurun_out/b4env_$i.log 2>&1
echo "$i [$cfg] $(grep -m1 -o 'step [0-9.]* ms' gpurun_out/b4env_$i.log)"
done
