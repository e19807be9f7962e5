cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/k128_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/k128_tests.log
for kt in 128 64 128 64; do
SPMD_ATTN_KT=$kt timeout 300 python scripts/kernel_bench.py attention 2>&1 | grep "^{" | sed "s/^/kt=$kt /"
done
