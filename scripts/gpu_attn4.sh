cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/attn.log 2>&1; echo attn=$?
timeout 300 python scripts/kernel_bench.py attention > gpurun_out/kb_attn.log 2>&1; echo kb=$?
SPMD_ATTN_MODE=1sm timeout 300 python scripts/kernel_bench.py attention >> gpurun_out/kb_attn.log 2>&1; echo kb1=$?
