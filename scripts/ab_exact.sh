#!/bin/bash
# Per-kernel median durations of the exact-mode step at S (scripts/prof_exact.py
# under ncu, --cache-control none: every launch cold), for A/B of exact layouts.
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none \
    -k "regex:pool_ivl|pool_exact|to_nhwc" --csv python scripts/prof_exact.py $1 2>/dev/null | python -c "
import csv, sys, statistics, collections
rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h = rows[0]; ki, vi = h.index('Kernel Name'), h.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split('(')[0]].append(float(r[vi].replace(',', '')))
print('exact $1', {k: round(statistics.median(v) / 1e3, 2) for k, v in d.items()})
"
