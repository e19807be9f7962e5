cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -x -m gpu > gpurun_out/gpu_all2.log 2>&1; echo gpu=$?; tail -2 gpurun_out/gpu_all2.log
CFG=c2train timeout 900 python scripts/timeline.py > gpurun_out/tl_train_n1b.log 2>&1; echo tl=$?
python - <<'PY'
import collections
rows = []
for l in open("gpurun_out/tl_train_n1b.log"):
    p = l.split()
    if len(p) >= 6 and p[0] in ("compute", "comm1"):
        rows.append((p[1], p[2], float(p[5])))
agg = collections.defaultdict(float)
for i, op, ms in rows: agg[op] += ms
tot = sum(agg.values())
for op, ms in sorted(agg.items(), key=lambda t: -t[1]): print("%-18s %8.2f ms %5.1f%%" % (op, ms, 100 * ms / tot))
PY
timeout 900 python bench.py --config c2train --no-cpu-baseline > gpurun_out/train_n1b.log 2>&1; echo b1=$?
grep "^{" gpurun_out/train_n1b.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['ms_per_step'], d['tflops_per_gpu'], d['mfu'], d['clocks'])"
