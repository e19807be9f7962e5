cd $GRAFT_REPO_ROOT
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 300 python -m pytest tests/test_gpu_gemm.py -q > gpurun_out/gemm.log 2>&1; echo gemm=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity.log 2>&1; echo parity=$?
