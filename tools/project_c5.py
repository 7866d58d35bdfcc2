"""C5 (n = 1,000,000, nb = 1900, theta = (1, 0.03, 0.5), TLR 1e-5, max rank
500) projected from measured leading blocks on one B200.

The full C5 factor does not fit one GPU (dense band at tile offsets 1-3 over
the cap plus ~138,600 low-rank tiles: ~210 GB).  The leading L x L tile block
of Sigma (the first 1900 L generator points) is factorised by exactly the
computation the full factorisation performs on tiles i < L, and its tile
geometry per offset is the full problem's (the row-major grid is
translation invariant along x), so its evaluation time T(L) is measured for a
few L and fitted with T = a L^2 + b L^3 (generation / compression ~ L^2
tiles, updates ~ L^3); the fit is extrapolated to L = 527.  The cubic term
over-counts (far-offset updates of the full problem have small ranks), so the
projection is an upper bound.  z is standard normal (ranks and work do not
depend on z).

    python tools/project_c5.py --lead 24 48 72 > c5.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_09137_b200 as tb  # noqa: E402

N, NB, THETA, ACC, CAP = 1_000_000, 1900, (1.0, 0.03, 0.5), 1e-5, 500
T_FULL = -(-N // NB)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lead", type=int, nargs="*", default=[24, 48, 72])
    ap.add_argument("--repeats", type=int, default=2)
    a = ap.parse_args()
    full = tb.generate_locations(N, 0).coords
    p = tb.MaternParams(*THETA)
    runs = []
    for L in a.lead:
        xy = np.ascontiguousarray(full[: L * NB])
        z = np.random.default_rng(1).standard_normal(len(xy))
        h = tb.Handle(xy, NB, CAP)
        ts = []
        for _ in range(a.repeats):
            t0 = time.perf_counter()
            ll = h.loglik(z, p, ACC)[0]
            ts.append(time.perf_counter() - t0)
        st = h.last_stats
        rm = h.rank_map()
        low = np.tril(rm, -1)
        r = {"L": L, "points": len(xy), "s": min(ts), "ll": ll, "device_ms": st["ms_device"],
             "phases_ms": {k: st[k] for k in ("ms_generate", "ms_compress", "ms_factor", "ms_solve")},
             "max_rank": st["max_rank"], "mean_rank": st["mean_rank"], "dense_tiles": int((low == -1).sum()),
             "arena_peak_gb": st["arena_peak_bytes"] / 1e9, "stored_gb": st["stored_reals"] * 8 / 1e9,
             "launches": st["kernel_launches"], "gflop": st["flops"] / 1e9}
        runs.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
        h.close()
        del h
    Ls = np.array([r["L"] for r in runs], float)
    Ts = np.array([r["s"] for r in runs])
    coef, *_ = np.linalg.lstsq(np.stack([Ls ** 2, Ls ** 3], 1), Ts, rcond=None)
    t1 = float(coef[0] * T_FULL ** 2 + coef[1] * T_FULL ** 3)
    # stored memory of the full factor: per-offset storage of the largest
    # block, extended to the full tile grid
    out = {"config": "C5", "n": N, "nb": NB, "acc": ACC, "max_rank": CAP, "tiles": T_FULL, "runs": runs,
           "fit": {"a_L2": float(coef[0]), "b_L3": float(coef[1])},
           "projected_s_per_eval_1gpu": t1,
           "projected_s_per_eval_8gpu_ideal": t1 / 8,
           "projected_20_eval_mle_8gpu_ideal_h": 20 * t1 / 8 / 3600,
           "note": ("upper bound: T(L) = a L^2 + b L^3 fitted on leading blocks, extrapolated to L = 527; "
                    "8-GPU figure assumes ideal strong scaling of the 2D block-cyclic schedule")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
