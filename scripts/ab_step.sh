# Median per-kernel durations of the headline step's two kernels (and the
# fused variant's) over 10 flushed steps; see scripts/prof_step.py.
for v in "" fused; do
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none \
    -k "regex:tile_pool|tile_finalize" --csv python scripts/prof_step.py $v 2>/dev/null | python -c "
import csv, sys, statistics, collections
rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h = rows[0]; ki, vi = h.index('Kernel Name'), h.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split('(')[0].split('<')[0].split()[-1]].append(float(r[vi].replace(',', '')))
print('$v' or 'f32', {k: round(statistics.median(v[2:]) / 1e3, 2) for k, v in d.items()})
"
done
