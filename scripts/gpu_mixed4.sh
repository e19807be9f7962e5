cd $GRAFT_REPO_ROOT
T4="timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for r in 1 2; do for H in ce mixed sm; do
  i=$((i+1))
  SPMD_PEER_HIDDEN_ENGINE=$H $T4 --master-port 2977$i bench.py --gpus 4 --no-e2e > gpurun_out/mx_$i.log 2>&1
  grep "^{" gpurun_out/mx_$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('hidden=$H', d['ms_per_step'], round(d['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done; done
