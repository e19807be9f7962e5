cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x > gpurun_out/hc_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/hc_tests.log
for n in 2 4; do
timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n scripts/halo_conv_check.py > gpurun_out/hc_n$n.log 2>&1; echo hc$n=$?
grep "^{" gpurun_out/hc_n$n.log; grep -i "Traceback\|Error" gpurun_out/hc_n$n.log | head -3
done
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29639 bench.py --gpus 2 --config c4 --no-e2e > gpurun_out/c4b_n2.log 2>&1; echo b2=$?
grep "^{" gpurun_out/c4b_n2.log | cut -c1-300
