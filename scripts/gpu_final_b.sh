cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T2="timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T4 --master-port 29791 scripts/multi_gpu_check.py > gpurun_out/fb_m4.log 2>&1; echo m4=$?; tail -1 gpurun_out/fb_m4.log
$T4 --master-port 29792 scripts/peer_fusion_check.py > gpurun_out/fb_peer4.log 2>&1; echo peer4=$?; grep '"failed"' gpurun_out/fb_peer4.log
i=0
for c in c2 c2train c3 c4; do
  i=$((i+1))
  $T4 --master-port 2980$i bench.py --gpus 4 --config $c > gpurun_out/fb_n4_$c.log 2>&1; echo n4_$c=$?
  $T2 --master-port 2981$i bench.py --gpus 2 --config $c > gpurun_out/fb_n2_$c.log 2>&1; echo n2_$c=$?
done
for f in gpurun_out/fb_n*_c*.log; do grep "^{" $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$f'.split('/')[-1], d['n_gpus'], round(d['ms_per_step'],2), round(d['tflops_per_gpu'],1), round(d['mfu']['vs_spec_2250'],3), d['clocks']['sm_mhz'], round(d['e2e']['ms_per_step'],2))"; done
