"""Summarise ncu outputs into profiles/<round>_summary.md (text evidence).

  python profiles/summarize.py r01 <launches.csv> <report.ncu-rep> [...]
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[mi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | ms (cold, serialised) | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k[:70]}` | {c} | {t:.2f} | {100 * t / tot:.1f}% |")
    return "\n".join(out), tot


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__cluster_dim_x", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        out.append(f"**{name}**  ")
        for w in WANT:
            if w in h:
                i = h.index(w)
                out.append(f"- `{w}` = {r[i]} {u[i]}")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    tag, csvp, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    tab, tot = launches(csvp)
    md = [f"# ncu summary {tag}", "", f"Launch list: `{csvp}` (total {tot:.1f} ms, "
          "ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache serialised launches: "
          "compare shares, not absolutes)", "", tab, ""]
    for rp in reps:
        md += [f"## `{rp}` (--set full)", "", report(rp), ""]
    open(f"profiles/{tag}_summary.md", "w").write("\n".join(md))
    print("\n".join(md))
