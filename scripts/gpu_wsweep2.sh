cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for cfg in "SPMD_GEMM_GROUP=8" "SPMD_GEMM_GROUP=16" "SPMD_GEMM_GROUP=12"; do
    env $cfg timeout 300 python scripts/gemm_env_sweep.py 2>&1 | grep "^{" | python -c "
import sys, json
v = [json.loads(l)['tflops'] for l in sys.stdin]
print('$cfg', v, round(sum(v)/len(v),1))"
  done
done
