cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e2e_n1.log 2>&1; echo b1=$?
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/e2e_n2.log 2>&1; echo b2=$?
for f in e2e_n1 e2e_n2; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['ms_per_step'], d['e2e'], d['clocks'])"; done
grep -i "error\|Traceback" gpurun_out/e2e_n*.log | head
