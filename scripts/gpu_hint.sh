cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for cfg in "SPMD_GEMM_HINT=0" "SPMD_GEMM_HINT=1" "SPMD_GEMM_STORE_HINT=1" "SPMD_GEMM_HINT=1 SPMD_GEMM_STORE_HINT=1" "SPMD_GEMM_HINT=2"; do
    env $cfg timeout 300 python scripts/gemm_env_sweep.py 2>&1 | grep "^{" | python -c "
import sys, json
v = [json.loads(l)['tflops'] for l in sys.stdin]
print('$cfg', v, round(sum(v)/len(v),1))"
  done
done
