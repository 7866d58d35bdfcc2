"""Aggregate an ncu --page source --csv (SASS) dump: stall totals and the
hottest instructions.   python tools/ncu_src.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {s: 0 for s in stalls}
allsum = 0
for r in data:
    try:
        allsum += int(r[samp])
    except ValueError:
        continue
    for s in stalls:
        tot[s] += int(r[ix[s]] or 0)
print("samples", allsum)
for s, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {s:28s} {v:8d} {100*v/max(1,allsum):5.1f}%")
print("hottest:")
best = sorted(range(len(data)), key=lambda i: -int(data[i][samp] or 0))[:top]
for i in sorted(best):
    r = data[i]
    st = sorted(((int(r[ix[s]] or 0), s) for s in stalls), reverse=True)[:2]
    print(f"{i:5d} {int(r[samp]):6d}  {r[1].strip()[:60]:60s} {st[0][1][6:]}:{st[0][0]} {st[1][1][6:]}:{st[1][0]}")
