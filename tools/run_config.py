"""Run one BASELINE config end to end on the device and print a JSON line:
locations (reference generator), z = sample_measurements on the device
(stats.py:115-133 semantics), one TLR (and optionally dense) log-likelihood,
and kriging of m held-out sites (predict.holdout_experiment index draw,
predict.py:114-119).

    python tools/run_config.py C3 [--dense] [--repeats 3]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1804_09137_b200 as tb  # noqa: E402

CONFIGS = {
    "C1": dict(n=1600, theta=(1.0, 0.1, 0.5), nb=400, acc=1e-9, max_rank=200, m=0),
    "C2": dict(n=10_000, theta=(1.0, 0.1, 0.5), nb=500, acc=1e-9, max_rank=None, m=0),
    "C3": dict(n=62_500, theta=(1.0, 0.03, 0.5), nb=760, acc=1e-7, max_rank=380, m=100),
    "C4": dict(n=250_000, theta=(1.0, 0.1, 1.0), nb=1000, acc=1e-7, max_rank=None, m=0),
    "C5": dict(n=1_000_000, theta=(1.0, 0.03, 0.5), nb=1900, acc=1e-5, max_rank=500, m=1000),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--repeats", type=int, default=2)
    ap.add_argument("--z-normal", action="store_true",
                    help="z = default_rng(1).standard_normal(n) (timing only; C4/C5 cannot be "
                         "sampled densely on one GPU)")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    out = {"config": a.config, **{k: v for k, v in c.items()}}
    locs = tb.generate_locations(c["n"], 0)
    p = tb.MaternParams(*c["theta"])
    t0 = time.perf_counter()
    z = (np.random.default_rng(1).standard_normal(c["n"]) if a.z_normal
         else tb.sample_measurements(locs, p, 1))
    out["sample_s"] = time.perf_counter() - t0
    out["z"] = "standard normal (timing only)" if a.z_normal else "sample_measurements(locs, theta, 1)"
    cfg = tb.LikelihoodConfig(mode="tlr", accuracy=c["acc"], nb=c["nb"], max_rank=c["max_rank"])
    ts = []
    for _ in range(a.repeats):
        t0 = time.perf_counter()
        ll, ld, q, st = tb.log_likelihood_parts(locs, z, p, cfg)
        ts.append(time.perf_counter() - t0)
    out.update(tlr_ll=ll, tlr_logdet=ld, tlr_quad=q, tlr_s=min(ts), tlr_device_ms=st["ms_device"],
               max_rank=st["max_rank"], mean_rank=st["mean_rank"], stored_reals=st["stored_reals"],
               launches=st["kernel_launches"], jacobi_max_sweeps=st["jacobi_max_sweeps"],
               phases_ms={k: st[k] for k in ("ms_generate", "ms_compress", "ms_factor", "ms_solve")})
    h = tb.api._handle_for(locs.coords, c["nb"], c["max_rank"], 1)
    rm = h.rank_map()
    out["dense_tiles"] = int((np.tril(rm, -1) == -1).sum())
    if a.dense:
        t0 = time.perf_counter()
        lld = tb.log_likelihood(locs, z, p, tb.LikelihoodConfig(nb=c["nb"]))
        out.update(dense_ll=lld, dense_s=time.perf_counter() - t0,
                   tlr_vs_dense=abs(ll - lld) / abs(lld))
    if c["m"]:
        rng = np.random.default_rng(2)
        idx = np.sort(rng.choice(c["n"], size=c["m"], replace=False))
        mask = np.zeros(c["n"], bool)
        mask[idx] = True
        kn, un = tb.LocationSet(locs.coords[~mask]), tb.LocationSet(locs.coords[mask])
        t0 = time.perf_counter()
        pred = tb.predict(tb.PredictionProblem(kn, z[~mask], un, p, "tlr", c["acc"], c["nb"],
                                               max_rank=c["max_rank"]))
        out.update(kriging_s=time.perf_counter() - t0,
                   kriging_mse=float(np.mean((pred - z[mask]) ** 2)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
