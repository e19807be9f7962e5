#!/bin/bash
# Round-end validation on one GPU: smoke, the -m gpu suite, N=1 benches.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/f1_gpu.log 2>&1; echo gpu=$?; tail -2 gpurun_out/f1_gpu.log
timeout 600 python bench.py > gpurun_out/f1_b1.log 2>&1; echo b1=$?
for c in c2train c3 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/f1_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f1_ref.log 2>&1; echo ref=$?; grep "^{" gpurun_out/f1_ref.log | cut -c1-300
for f in f1_b1 f1_c2train f1_c3 f1_c4; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$f', round(d['ms_per_step'],2), round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'], d['clocks'].get('reasons'), d['roofline']['frac'], d['gpu_launches'], round(d['e2e']['value'],1))"; done
