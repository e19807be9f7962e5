cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fa_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/fa_gpu.log 2>&1; echo gpu=$?; tail -1 gpurun_out/fa_gpu.log
timeout 600 python bench.py > gpurun_out/fa_b1.log 2>&1; echo b1=$?
for c in c2train c3 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/fa_$c.log 2>&1; echo $c=$?; done
timeout 120 python scripts/gemm_once.py 16384 65536 8192 > gpurun_out/fa_gemm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 -o gpurun_out/gemm_wide_full python scripts/gemm_once.py 16384 65536 8192 > gpurun_out/fa_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/gemm_wide_full.ncu-rep --page raw --csv > gpurun_out/gemm_wide_full_raw.csv 2>/dev/null
ncu -i gpurun_out/gemm_wide_full.ncu-rep --page details --csv > gpurun_out/gemm_wide_full_details.csv 2>/dev/null
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/fa_launches.csv python bench.py $ARGS > gpurun_out/fa_ncu_list.log 2>&1; echo list=$?
for f in fa_b1 fa_c2train fa_c3 fa_c4; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$f', d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'], d['roofline']['frac'], d['gpu_launches'])"; done
