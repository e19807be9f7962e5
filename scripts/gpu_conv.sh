cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -q -x > gpurun_out/conv.log 2>&1; echo conv=$?
