cd $GRAFT_REPO_ROOT
for m in 0 1 2; do
SPMD_CONV_SHIFT_MODE=$m timeout 300 python -m pytest tests/test_gpu_conv.py -q -k "test_conv_tcgen05" > gpurun_out/shift_$m.log 2>&1; echo mode$m=$?; tail -1 gpurun_out/shift_$m.log; grep "where 0\.\|assert 0\." gpurun_out/shift_$m.log | head -3 | cut -c1-120
done
