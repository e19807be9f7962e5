cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo gpu=$?; tail -2 gpurun_out/gpu_all.log
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo b1=$?
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3_n1.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_c4_n1.log 2>&1; echo c4=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_n1.log 2>&1; echo ref=$?
for f in bench_n1 bench_c3_n1 bench_c4_n1 bench_ref_n1; do grep "^{" gpurun_out/$f.log | cut -c1-400; done
