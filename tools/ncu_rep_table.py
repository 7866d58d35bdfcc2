"""Key counters of every launch in ncu --set full reports, one markdown row
per launch (pipe utilisation, issue rate, occupancy, DRAM / L2 traffic):
    python tools/ncu_rep_table.py a.ncu-rep b.ncu-rep ..."""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "time"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"), ("launch__cluster_dim_x", "cluster"),
        ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thr %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts")]


def fnum(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main():
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " | DRAM GB/s |")
    print("|---" * (len(COLS) + 2) + "|")
    for path in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        h, u = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("tlrb::", "")
            name = name.replace("(anonymous namespace)::", "")
            cells, t_s, byt = [], None, 0.0
            for key, _ in COLS:
                if key not in h:
                    cells.append("-")
                    continue
                i = h.index(key)
                v, unit = fnum(r[i]), u[i]
                if v is None:
                    cells.append(r[i])
                    continue
                if key == "gpu__time_duration.sum":
                    sc = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
                          "second": 1.0}[unit]
                    t_s = v * sc
                    cells.append(f"{t_s * 1e6:.1f} us")
                elif key.startswith("dram__bytes"):
                    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                    byt += v * sc
                    cells.append(f"{v * sc / 1e6:.2f} MB")
                else:
                    cells.append(f"{v:.1f}" if v != int(v) else f"{int(v)}")
            gbs = f"{byt / t_s / 1e9:.0f}" if t_s else "-"
            print(f"| `{name[:48]}` | " + " | ".join(cells) + f" | {gbs} |")


if __name__ == "__main__":
    main()
