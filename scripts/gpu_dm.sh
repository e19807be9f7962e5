cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_datamove.py tests/test_gpu_parity.py -x -q > gpurun_out/dm_parity.log 2>&1; echo parity=$?
timeout 300 python scripts/kernel_bench.py datamove > gpurun_out/kb_dm.log 2>&1; echo kb=$?
tail -3 gpurun_out/dm_parity.log; cat gpurun_out/kb_dm.log
