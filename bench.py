#!/usr/bin/env python
"""Benchmark: seconds per TLR Gaussian log-likelihood evaluation (BASELINE.json).

Workload (BASELINE.json configs[1], "C2"): n = 10,000 jittered 100x100 grid
(generate_locations(10000, 0)), Matern theta = (1.0, 0.1, 0.5), nb = 500, FP64,
TLR accuracy 1e-9 (headline) with 1e-7 / 1e-5 / dense as variants.  z is the
reference's own seeded field sample_measurements(locs, theta, 1), committed
as a golden fixture (tests/golden/z_big.npz); synthetic data, no dataset.

One step = one complete likelihood evaluation (tile generation, TLR
compression, TLR Cholesky with recompression, log-det, forward solve, dot).
  value : device time (CUDA events on the library's stream) with z and the
          locations resident in HBM (tlrb_loglik_device); L2 flushed before
          every step (256 MB write) — the tile working set (~0.8 GB) also
          exceeds the 126 MB L2.
  e2e   : the public API log_likelihood(locs, z_host, p, cfg) timed on the
          host: H2D of z + evaluation + D2H of the result.
N > 1: one process per GPU, tiles 2D block-cyclic over a P x Q grid with NCCL
panel broadcasts (tlrb_create_dist); value = max-over-ranks device time of the
shared evaluation (strong scaling).

JSON extras: `roofline` (dominant kernel class, measured live; `traffic`
from profiles/ncu_traffic.json), `step_roofline` (whole
evaluation, algorithmic flops / bytes against the measured peaks), `kernels`
(per-class breakdown of one profiled warm-up step), `variants` (dense /
1e-7 / 1e-5 with their parity), `parity`, `phases_ms`, `work`.

`--impl reference` times the CPU oracle port (oracle/, a restatement of the
reference pinned to its goldens) on the host cores with a bounded stratified
sample per step (oracle/cpu_baseline.py).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

THETA = (1.0, 0.1, 0.5)
N_POINTS, NB = 10_000, 500
METRIC = "s per TLR log-likelihood eval"
REF_LL = {  # reference values (tests/golden/loglik_big.json)
    "dense": -2792.8552885992976,
    "tlr:1e-09": -2792.8552965835443,
    "tlr:1e-07": -2792.8531515364302,
    "tlr:1e-05": -2792.9884456292575,
}


def h_grid(world):
    from paper_1804_09137_b200.dist import grid_shape
    p, q = grid_shape(world)
    return f"{p}x{q}"


def load_z():
    p = ROOT / "tests" / "golden" / "z_big.npz"
    if p.exists():
        return np.load(p)["C2"]
    # fall back to the oracle's own seeded sample (pinned to the reference)
    from oracle import tlr_oracle as orc
    return orc.sample_measurements(orc.generate_locations(N_POINTS, 0), THETA, 1)


def mode_key(acc):
    return "dense" if not acc else f"tlr:{acc:.0e}".replace("e-0", "e-0")


def ref_key(acc):
    return "dense" if not acc else "tlr:" + f"{acc:g}".replace("e-0", "e-0")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for k, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


def fp64_peak_tflops(torch):
    """cuBLAS DGEMM 8192^3 (FP64 DMMA), best of 5 — MEASURED_PEAKS.json has no
    FP64 figure."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    best = 0.0
    for _ in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = max(best, 2 * 8192 ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


def traffic_for(kernel: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(kernel)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
        return v
    return None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import cpu_baseline as cb
    from oracle import tlr_oracle as orc
    xy = orc.generate_locations(N_POINTS, 0)
    z = load_z()
    times = []
    desc = ""
    for it in range(args.warmup + args.steps):
        est, desc = cb.estimate_eval_seconds(xy, z, THETA, NB, args.acc)
        if it >= args.warmup:
            times.append(est)
    v = float(np.median(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seeded)",
        "config": {"workload": f"C2 n={N_POINTS} nb={NB} theta={THETA} {mode_key(args.acc)}",
                   "n": N_POINTS, "nb": NB, "acc": args.acc},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cb.host_threads(), "kind": "port",
                         "sample": desc},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--acc", type=float, default=1e-9)
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1804_09137_b200 as tb
    from paper_1804_09137_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    locs = tb.generate_locations(N_POINTS, 0)
    z = load_z()
    p = tb.MaternParams(*THETA)
    if world > 1:   # 2D block-cyclic tiles over all ranks (NCCL), SURVEY 8(e)
        h = tb.api.distributed_handle(locs.coords, NB, 0, device=local)
    else:
        h = tb.Handle(locs.coords, NB, device=local)
    dz = torch.from_numpy(z).to("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def one(acc):
        flush.random_(0, 255)   # evict L2 (256 MB > 126 MB)
        torch.cuda.synchronize()
        return h.loglik_device(dz.data_ptr(), p, acc)

    for _ in range(max(0, args.warmup - 1)):
        one(args.acc)
    # last warm-up step: every kernel class under per-launch CUDA events ->
    # the per-class breakdown and the dominant class (outside the timed region)
    _lib.profile_enable(True)
    one(args.acc)
    barrier()
    prof_all = _lib.profile_read()
    dom_name = max(prof_all.items(), key=lambda kv: kv[1]["ms"])[0]
    # timed region: events only around the dominant class's launches (a few
    # dozen per step), so the roofline is measured live at ~zero overhead
    _lib.profile_enable(True, classes=[dom_name])
    l0 = tb.launch_count()
    step_ms, lls, stats = [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            barrier()
            ll, ld, q = one(args.acc)
            st = h.last_stats
            stats.append(st)
            step_ms.append(allmax(st["ms_device"]))
            lls.append(ll)
        barrier()
    launches = (tb.launch_count() - l0) // max(1, args.steps)
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    ms = float(np.median(step_ms))
    value_s = ms * 1e-3   # one evaluation shared by all ranks (strong scaling)

    # e2e through the public API (host z in, host float out)
    e2e = []
    cfg = (tb.LikelihoodConfig(mode="tlr", accuracy=args.acc, nb=NB, ngpus=world) if args.acc
           else tb.LikelihoodConfig(nb=NB, ngpus=world))
    tb.log_likelihood(locs, z, p, cfg)
    for _ in range(args.steps):
        flush.random_(0, 255)
        barrier()
        t0 = time.perf_counter()
        ll_e = tb.log_likelihood(locs, z, p, cfg)
        e2e.append(allmax(time.perf_counter() - t0))
    e2e_s = float(np.median(e2e))

    # variants (other accuracies / dense): every rank takes part, since a
    # distributed handle runs NCCL collectives inside each evaluation
    var = None
    if not args.no_variants:
        var = {}
        for acc in ([0.0, 1e-7, 1e-5] if args.acc else [1e-9, 1e-7, 1e-5]):
            if acc == args.acc:
                continue
            one(acc)
            tt = []
            for _ in range(2):
                ll_v, _, _ = one(acc)
                tt.append(allmax(h.last_stats["ms_device"]))
            r = REF_LL.get(ref_key(acc))
            var[mode_key(acc)] = {"s": float(np.median(tt)) * 1e-3, "ll": ll_v, "ref_ll": r,
                                  "rel": abs(ll_v - r) / abs(r) if r else None,
                                  "max_rank": h.last_stats["max_rank"]}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peaks = measured_peaks()
    p64 = fp64_peak_tflops(torch)
    # dominant kernel class (from the all-class warm-up step), timed inside the timed region
    name, d = dom_name, prof[dom_name]
    per_launch_s = d["ms"] * 1e-3 / max(1, d["launches"])
    flops_bound = d["flops"] > 0 and (d["flops"] / (p64 * 1e12)) >= (d["bytes"] / (peaks["hbm_gbs"] * 1e9))
    if flops_bound:
        achieved = d["flops"] / max(1, d["launches"]) / per_launch_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": p64, "unit": "TFLOP/s",
                "frac": achieved / p64, "peak_source": "measured cuBLAS DGEMM 8192^3 (FP64) in bench.py"}
    else:
        achieved = d["bytes"] / max(1, d["launches"]) / per_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if peaks.get("fallback") else "")}
    roof["kernel"] = name
    roof["share_of_step"] = d["ms"] / (ms * args.steps)
    roof["note"] = ("dominant class timed with per-launch CUDA events inside the timed region; "
                    "algorithmic flops per SURVEY 8(d) / as implemented (Jacobi: 3 n s(s-1) per sweep)")
    roof["launches_per_step"] = d["launches"] / args.steps
    roof["traffic"] = traffic_for(name)
    kernels = {k: {"ms_per_step": v["ms"], "launches_per_step": v["launches"],
                   "gflop_per_step": v["flops"] / 1e9, "gb_per_step": v["bytes"] / 1e9}
               for k, v in prof_all.items() if v["launches"]}   # one profiled warm-up step
    st = stats[-1]
    ref = REF_LL.get(ref_key(args.acc))
    line = {
        "metric": METRIC, "value": value_s, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator generate_locations(10000,0); z = reference "
                "sample_measurements(locs, theta, 1) fixture)",
        "config": {"workload": f"C2 n={N_POINTS} nb={NB} theta={THETA} {mode_key(args.acc)}",
                   "n": N_POINTS, "nb": NB, "acc": args.acc,
                   "l2": "flushed before every step (256 MB write); tile working set > L2",
                   "parallelism": (f"2D block-cyclic tiles P x Q = {h_grid(world)} over NCCL"
                                   if world > 1 else "1 GPU")},
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * N_POINTS, "d2h_bytes_per_step": 24},
        "gpu_launches": int(launches),
        "roofline": roof,
        "parity": {"ll": lls[-1], "ref_ll": ref,
                   "rel": (abs(lls[-1] - ref) / abs(ref)) if ref else None,
                   "tol": max(1e-8, 10 * args.acc) if args.acc else 1e-10,
                   "e2e_ll": ll_e},
        "phases_ms": {"generate+compress": st["ms_generate"], "compress": st["ms_compress"],
                      "factor": st["ms_factor"], "solve": st["ms_solve"]},
        "work": {"gflop": st["flops"] / 1e9, "gb": st["bytes"] / 1e9, "max_rank": st["max_rank"],
                 "mean_rank": st["mean_rank"], "sketch_retries": st["sketch_retries"],
                 "jacobi_max_sweeps": st["jacobi_max_sweeps"], "stored_reals": st["stored_reals"]},
        "kernels": kernels,
        "fp64_peak_tflops_measured": p64,
        # whole-evaluation roofline from the algorithmic work
        # counted per op at execution ranks (min flops / bytes; the op sum of
        # max(F/P64, B/BW) is bounded below by this max of the totals)
        "step_roofline": {
            "t_roof_s": max(st["flops"] / (p64 * 1e12), st["bytes"] / (peaks["hbm_gbs"] * 1e9)),
            "frac": max(st["flops"] / (p64 * 1e12), st["bytes"] / (peaks["hbm_gbs"] * 1e9)) / value_s,
            "gflop": st["flops"] / 1e9, "gb": st["bytes"] / 1e9,
            "note": "algorithmic FP64 flops / HBM bytes of the whole evaluation (gen, compression, "
                    "TLR Cholesky, solve; rank 0's counted work) against the measured DGEMM peak and MEASURED_PEAKS hbm_gbs"},
    }
    clk_s = clk.summary()
    if clk_s:
        line["clocks"] = clk_s
    if var is not None:
        line["variants"] = var
    if not args.no_cpu:
        # in a fresh interpreter (no torch / CUDA runtime threads next to the
        # BLAS pool), the same way the --impl reference arm runs
        code = ("import json, sys; sys.path.insert(0, %r); import bench; "
                "from oracle import cpu_baseline as cb; from oracle import tlr_oracle as orc; "
                "est, desc = cb.estimate_eval_seconds(orc.generate_locations(bench.N_POINTS, 0), bench.load_z(), "
                "bench.THETA, bench.NB, %r); print(json.dumps([est, desc, cb.host_threads()]))"
                % (str(Path(__file__).resolve().parent), args.acc))
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True)
        est, desc, cores = json.loads(out.stdout.strip().splitlines()[-1])
        line["cpu_baseline"] = {"value": est, "unit": "s", "cores": cores, "kind": "port", "sample": desc}
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
