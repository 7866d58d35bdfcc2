"""Assemble profiles/r02_summary.md from the evidence run's outputs
(gpurun_out/: launch list, --set full reports, bench line):
    python tools/make_r02_summary.py > profiles/r02_summary.md"""
import glob
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "gpurun_out"
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
bench = json.loads((G / "r02_bench_c3.json").read_text().strip().splitlines()[-1])


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout


print("# ncu summary, round 2 (C3: n = 62,500, nb = 760, TLR 1e-7, cap 380; one B200)\n")
print(f"Peaks: HBM {peaks.get('hbm_gbs', 6553.3)} GB/s (MEASURED_PEAKS.json); FP64 tensor (DMMA) "
      f"{bench['fp64_peak_tflops_measured']:.1f} TFLOP/s (cuBLAS DGEMM 8192^3, measured inside the bench run; "
      "MEASURED_PEAKS.json has no FP64 figure).  Bench line of the same tree: `profiles/r02_bench_c3.json` "
      f"({bench['value']:.3f} s per evaluation, e2e {bench['e2e']['value']:.3f} s).\n")
print("## Launch list of one evaluation\n")
print("`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` on "
      "`python tools/trace_cfg.py C3 --no-warm` (`tools/r02_ncu.sh`; raw list: `profiles/r02_launches_c3.csv.gz`). "
      "Launches are serialised and cold-cache under ncu: compare shares, not absolutes.\n")
_csv = G / "r02_launches_c3.csv.gz"
print(run("tools/ncu_list_summary.py", str(_csv if _csv.exists() else G / "r02_launches_c3.csv"), "--md"))
print("\n## Counters per kernel class (`ncu --set full`, launches past the first steps)\n")
_cnt = G / "r02_counters.md"
reps = sorted(glob.glob(str(G / "r02_full_*.ncu-rep")))
print(_cnt.read_text() if _cnt.exists() else run("tools/ncu_rep_table.py", *reps))
_gb = ROOT / "profiles" / "r02_counters_gemmbench.md"
if _gb.exists():
    print("\nThe in-evaluation captures above land on small GEMM launches (look-ahead SYRK, K x K products); the "
          "large-launch behaviour of the same kernel, `ncu --set full` on `tools/bench_gemm` (760 x 760 x 200 batch of 64, "
          "82 x 760^3 batch, 4096^3):\n")
    print(_gb.read_text())
print("\nGEMM microbenchmark (`tools/bench_gemm`, ours vs cuBLAS on the TLR shapes): `profiles/r02_gemm_bench.txt`.\n")
notes = ROOT / "profiles" / "r02_summary_notes.md"
if notes.exists():
    print(notes.read_text())
