cd $GRAFT_REPO_ROOT
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r1.csv python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1; echo list=$?
timeout 120 python scripts/gemm_once.py 16384 65536 8192 > gpurun_out/gemm_ffn.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 -o gpurun_out/gemm_ffn_full python scripts/gemm_once.py 16384 65536 8192 > gpurun_out/ncu_full.log 2>&1; echo full=$?
