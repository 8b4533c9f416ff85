# Per-launch durations of the fin_lab variants (ncu, no cache control: the
# L2 state each variant sees is the one fin_lab.py prepared).
LAB_MODES=${LAB_MODES:-hot} ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file gpurun_out/fin_lab_ncu.csv python scripts/fin_lab.py > gpurun_out/fin_lab_ncu.log 2>&1
python - <<'PY'
import csv, collections
lines = open("gpurun_out/fin_lab_ncu.csv").read().split("\n")
i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i:]))
h = rows[0]
ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
d = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) > vi and r[vi]:
        d[(r[ki].split("(")[0][:50], r[gi])].append(float(r[vi].replace(",", "")))
for k, v in d.items():
    if len(v) < 5:
        continue
    v = sorted(v)
    print(f"{k[0]:50s} {k[1]:14s} n={len(v):4d} med={v[len(v)//2]/1e3:8.2f}us min={v[0]/1e3:8.2f}")
PY
