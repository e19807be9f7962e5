cd $GRAFT_REPO_ROOT
timeout 300 python scripts/kernel_bench.py all > gpurun_out/kbench.log 2>&1; echo kbench=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; echo bench=$?
