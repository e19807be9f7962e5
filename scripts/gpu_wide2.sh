cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/w2_gpu.log 2>&1; echo gpu=$?; tail -1 gpurun_out/w2_gpu.log
timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/w2_vs.log 2>&1; cat gpurun_out/w2_vs.log
for m in 3 2 3; do
  if [ $m = 2 ]; then E="SPMD_GEMM_MODE=2sm"; else E=""; fi
  env $E timeout 600 python bench.py --no-cpu-baseline > gpurun_out/w2_b1_$m.log 2>&1
  grep "^{" gpurun_out/w2_b1_$m.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('mode$m', d['ms_per_step'], d['tflops_per_gpu'], d['mfu'], d['clocks'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
done
