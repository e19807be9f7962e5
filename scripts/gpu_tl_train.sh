cd $GRAFT_REPO_ROOT
CFG=c2train timeout 900 python scripts/timeline.py > gpurun_out/tl_train_n1.log 2>&1; echo tl=$?
python - <<'PY'
import re, collections
rows = []
for l in open("gpurun_out/tl_train_n1.log"):
    p = l.split()
    if len(p) >= 6 and p[0] in ("compute", "comm1"):
        rows.append((p[1], p[2], float(p[5])))
agg = collections.defaultdict(float)
for i, op, ms in rows: agg[op] += ms
tot = sum(agg.values())
for op, ms in sorted(agg.items(), key=lambda t: -t[1]): print("%-18s %8.2f ms %5.1f%%" % (op, ms, 100 * ms / tot))
for i, op, ms in sorted(rows, key=lambda t: -t[2])[:25]: print("   %-16s %-14s %7.3f" % (i, op, ms))
PY
tail -1 gpurun_out/tl_train_n1.log
