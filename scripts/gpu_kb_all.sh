cd $GRAFT_REPO_ROOT
timeout 600 python scripts/kernel_bench.py all > gpurun_out/kb_all.log 2>&1; echo kb=$?
