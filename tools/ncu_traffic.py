"""DRAM traffic per launch of the bench's dominant kernel class from an ncu
metrics CSV (dram__bytes_read.sum + dram__bytes_write.sum, one row per metric
and launch) -> profiles/ncu_traffic.json, read by bench.py for roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/ev_jacobi_dram.csv jacobi_svd
"""
import collections
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main():
    path, cls = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hi]
    ii, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    launches = [d for d in per.values() if "dram__bytes_read.sum" in d]
    tot = sum(d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0) for d in launches)
    dur = sum(d.get("gpu__time_duration.sum", 0.0) for d in launches)
    out_p = ROOT / "profiles" / "ncu_traffic.json"
    out = json.loads(out_p.read_text()) if out_p.exists() else {}
    out[cls] = {"dram_bytes_per_launch": tot / len(launches), "launches": len(launches),
                "dram_gbs_during_kernel": tot / dur / 1e9 if dur else None,
                "source": f"{Path(path).name}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                          "over every launch of the bench's timed step (cold cache, serialised)"}
    out_p.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out[cls], indent=1))


if __name__ == "__main__":
    main()
