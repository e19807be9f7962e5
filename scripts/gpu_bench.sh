cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.log 2>&1; echo bench=$?
