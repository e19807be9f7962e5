cd $GRAFT_REPO_ROOT
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu.log 2>&1; echo ncu=$?
