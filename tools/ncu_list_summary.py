"""Per-kernel summary of an ncu launch list with gpu__time_duration.sum and
dram__bytes_{read,write}.sum (tools/r02_ncu.sh): launches, serialised time,
share, DRAM bytes and the achieved DRAM GB/s of each kernel.
    python tools/ncu_list_summary.py launches.csv [--md]"""
import csv
import sys
from collections import defaultdict

import gzip
_p = sys.argv[1]
lines = (gzip.open(_p, "rt") if _p.endswith(".gz") else open(_p)).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
ix = {h: i for i, h in enumerate(rows[0])}
scale_t = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
scale_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "bytes": 1.0}
agg = defaultdict(lambda: {"n": 0, "ms": 0.0, "rd": 0.0, "wr": 0.0, "max": 0.0})
for r in rows[1:]:
    try:
        name = r[ix["Kernel Name"]].replace("void ", "").replace("tlrb::", "").replace("(anonymous namespace)::", "")
        name = name.split("(")[0]
        m, u, v = r[ix["Metric Name"]], r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
    except (ValueError, IndexError):
        continue
    a = agg[name]
    if m == "gpu__time_duration.sum":
        a["n"] += 1
        a["ms"] += v * scale_t[u]
        a["max"] = max(a["max"], v * scale_t[u])
    elif m == "dram__bytes_read.sum":
        a["rd"] += v * scale_b[u]
    elif m == "dram__bytes_write.sum":
        a["wr"] += v * scale_b[u]
tot = sum(a["ms"] for a in agg.values())
md = "--md" in sys.argv
if md:
    print("| kernel | launches | ms (serialised) | share | mean us | DRAM read GB | DRAM write GB | DRAM GB/s |")
    print("|---|---|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
    gbs = (a["rd"] + a["wr"]) / 1e9 / (a["ms"] * 1e-3) if a["ms"] else 0.0
    if md:
        print(f"| `{k[:64]}` | {a['n']} | {a['ms']:.1f} | {100 * a['ms'] / tot:.1f}% | {1e3 * a['ms'] / a['n']:.1f} | "
              f"{a['rd'] / 1e9:.2f} | {a['wr'] / 1e9:.2f} | {gbs:.0f} |")
    else:
        print(f"{k[:56]:56s} n={a['n']:6d} ms={a['ms']:9.1f} {100 * a['ms'] / tot:5.1f}% mean={1e3 * a['ms'] / a['n']:8.1f}us "
              f"max={a['max']:7.2f}ms rd={a['rd'] / 1e9:8.2f}GB wr={a['wr'] / 1e9:8.2f}GB {gbs:7.0f} GB/s")
print(f"total {tot:.1f} ms over {sum(a['n'] for a in agg.values())} launches")
