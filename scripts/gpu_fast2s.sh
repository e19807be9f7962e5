cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k two_streams > gpurun_out/fast2s.log 2>&1; echo fast2s=$?
