cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T4 --master-port 29871 scripts/multi_gpu_check.py > gpurun_out/v_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/v_m4.log
$T2 --master-port 29872 scripts/multi_gpu_check.py > gpurun_out/v_m2.log 2>&1; echo m2=$?; tail -1 gpurun_out/v_m2.log
$T4 --master-port 29873 scripts/peer_fusion_check.py > gpurun_out/v_p4.log 2>&1; echo p4=$?; grep '"failed"' gpurun_out/v_p4.log
$T2 --master-port 29874 scripts/peer_fusion_check.py > gpurun_out/v_p2.log 2>&1; echo p2=$?; grep '"failed"' gpurun_out/v_p2.log
$T4 --master-port 29875 bench.py --gpus 4 > gpurun_out/v_b4.log 2>&1; echo b4=$?
grep "^{" gpurun_out/v_b4.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['config']['mesh'], d['ms_per_step'], round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['e2e']['ms_per_step'])"
