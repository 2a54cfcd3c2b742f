cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ep8_launches.csv python tools/fused_timeline.py --nc0 64 --g0 4 --pairs 0 > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(l for l in open('gpurun_out/ep8_launches.csv') if not l.startswith('==')))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    if 'comet' in r[ki]: d[r[ki].split('(')[0]].append(float(r[vi].replace(',',''))/1000)
for k,v in d.items(): print(f"{k:50s} n={len(v):4d} mean={sum(v)/len(v):8.1f}us min={min(v):8.1f} max={max(v):8.1f}")
PY
