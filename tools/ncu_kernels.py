"""Per-kernel mean / max duration from an `ncu --metrics gpu__time_duration.sum --csv` log."""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
ix = {h: i for i, h in enumerate(rows[0])}
d = defaultdict(list)
for r in rows[1:]:
    try:
        d[r[ix["Kernel Name"]][:60]].append(float(r[ix["Metric Value"]]))
    except (ValueError, IndexError):
        pass
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):4d} mean={sum(v)/len(v)/1e3:8.1f} us max={max(v)/1e3:8.1f} sum={sum(v)/1e6:8.2f} ms {100*sum(v)/tot:5.1f}%")
