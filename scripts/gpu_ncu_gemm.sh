cd $GRAFT_REPO_ROOT
timeout 120 python scripts/gemm_once.py > gpurun_out/gemm_once.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 -o gpurun_out/gemm_2sm python scripts/gemm_once.py > gpurun_out/ncu_gemm.log 2>&1; echo ncu=$?
