cd $GRAFT_REPO_ROOT
S="timeout 120 python scripts/gemm_sweep.py"
for shape in "16384 65536 8192" "16384 8192 65536" "16384 32768 8192"; do
  $S $shape
  SPMD_GEMM_GROUP=4 $S $shape
  SPMD_GEMM_GROUP=16 $S $shape
  SPMD_GEMM_GROUP=32 $S $shape
  SPMD_GEMM_RASTER=n $S $shape
  SPMD_GEMM_RASTER=n SPMD_GEMM_GROUP=16 $S $shape
  SPMD_GEMM_HINT=1 $S $shape
  SPMD_GEMM_HINT=2 $S $shape
  SPMD_GEMM_HINT=1 SPMD_GEMM_GROUP=16 $S $shape
  $S $shape
done > gpurun_out/sweep.jsonl 2>&1
echo done
