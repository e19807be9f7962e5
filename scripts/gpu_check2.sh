cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/parity.log 2>&1; echo parity=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.log 2>&1; echo bench=$?
