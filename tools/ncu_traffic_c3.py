"""profiles/ncu_traffic_c3.json: DRAM bytes per launch of every bench kernel
class at C3, from the ncu launch list of one evaluation (tools/r02_ncu.sh:
dram__bytes_read.sum + dram__bytes_write.sum of every launch, cold cache,
serialised).  bench.py reports the dominant class's figure as
`roofline.traffic`.
    python tools/ncu_traffic_c3.py gpurun_out/r02_launches_c3.csv.gz"""
import csv
import gzip
import json
import sys
from collections import defaultdict
from pathlib import Path

CLASSES = [("dgemm_tiles", "dgemm_vbatch"), ("jacobi_cluster", "jacobi_svd"), ("qrcp_", "qr_householder"),
           ("bq_", "qr_householder"), ("bqr_", "qr_householder"), ("gen_tiles", "gen_tiles"),
           ("trsm_vbatch", "trsm_vbatch"), ("potrf_block", "potrf_block"), ("sumsq", "sumsq"),
           ("copy_kernel", "copy"), ("colnorm", "copy"), ("reduce_kernel", "reduce")]
p = sys.argv[1]
lines = (gzip.open(p, "rt") if p.endswith(".gz") else open(p)).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
ix = {h: i for i, h in enumerate(rows[0])}
sb = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
st = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}
agg = defaultdict(lambda: {"bytes": 0.0, "launches": 0, "s": 0.0})
for r in rows[1:]:
    try:
        name, m, u, v = r[ix["Kernel Name"]], r[ix["Metric Name"]], r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
    except (ValueError, IndexError):
        continue
    cls = next((c for key, c in CLASSES if key in name), None)
    if cls is None:
        continue
    a = agg[cls]
    if m == "gpu__time_duration.sum":
        a["launches"] += 1
        a["s"] += v * st[u]
    elif m.startswith("dram__bytes"):
        a["bytes"] += v * sb[u]
out = {c: {"dram_bytes_per_launch": a["bytes"] / max(1, a["launches"]), "launches": a["launches"],
           "dram_gbs_during_kernel": a["bytes"] / 1e9 / a["s"] if a["s"] else 0.0,
           "source": "profiles/r02_launches_c3.csv.gz: ncu dram__bytes_read.sum + dram__bytes_write.sum over every launch "
                     "of one C3 evaluation (cold cache, serialised)"} for c, a in agg.items()}
Path(__file__).resolve().parents[1].joinpath("profiles", "ncu_traffic_c3.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out, indent=1))
