cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/topo.log 2>&1
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/peer_fusion_check.py --perf > gpurun_out/peer2.log 2>&1; echo peer2=$?
grep -v "^W1\|\*\*\*\|OMP_NUM" gpurun_out/peer2.log | tail -20
