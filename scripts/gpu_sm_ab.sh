cd $GRAFT_REPO_ROOT
T="timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
A="bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e"
$T --master-port 29601 $A > gpurun_out/sm_base.log 2>&1; echo base=$?
SPMD_COMM_SMS=16 SPMD_NCCL_MAX_CTAS=16 $T --master-port 29602 $A > gpurun_out/sm_16.log 2>&1; echo s16=$?
SPMD_COMM_SMS=8 SPMD_NCCL_MAX_CTAS=8 $T --master-port 29603 $A > gpurun_out/sm_8.log 2>&1; echo s8=$?
SPMD_NCCL_MAX_CTAS=8 $T --master-port 29604 $A > gpurun_out/sm_nccl8.log 2>&1; echo n8=$?
$T --master-port 29605 $A --no-overlap > gpurun_out/sm_nooverlap.log 2>&1; echo no=$?
