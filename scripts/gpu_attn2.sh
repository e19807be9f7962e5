cd $GRAFT_REPO_ROOT
timeout 300 python scripts/kernel_bench.py attention > gpurun_out/kb_attn.log 2>&1; echo kb=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_n1_attn.log 2>&1; echo b1=$?
SPMD_FUSED_ATTENTION=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_n1_noattn.log 2>&1; echo b0=$?
