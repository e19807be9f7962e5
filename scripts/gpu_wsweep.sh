cd $GRAFT_REPO_ROOT
for cfg in "" "SPMD_GEMM_GROUP=4" "SPMD_GEMM_GROUP=16" "SPMD_GEMM_RASTER=n" "SPMD_GEMM_RASTER=n SPMD_GEMM_GROUP=4" "SPMD_GEMM_GROUP=2" "SPMD_GEMM_RASTER=n SPMD_GEMM_GROUP=16" ""; do
  env $cfg timeout 300 python scripts/gemm_env_sweep.py 2>&1 | grep "^{"
done
timeout 300 python -c "
import torch, time
for M,N,K in [(16384,65536,8192),(16384,8192,65536)]:
    a=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); b=torch.randn(K,N,device='cuda',dtype=torch.bfloat16)
    for _ in range(2): torch.matmul(a,b)
    best=1e9
    for _ in range(3):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); torch.cuda.synchronize(); e0.record()
        for _ in range(5): torch.matmul(a,b)
        e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1)/5)
    print('cublas', M,N,K, round(2*M*N*K/best/1e9,1))
"
