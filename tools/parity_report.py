"""Parity report: device log-likelihood vs the reference goldens for every
committed case (tests/golden).  Writes a markdown table to stdout."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1804_09137_b200 as tb  # noqa: E402

G = ROOT / "tests" / "golden"


def cases():
    lik = json.loads((G / "loglik.json").read_text())
    lik.update(json.loads((G / "loglik_big.json").read_text()))
    z = dict(np.load(G / "z.npz"))
    z.update(dict(np.load(G / "z_big.npz")))
    for name, e in lik.items():
        yield name, tb.generate_locations(e["n"], e["loc_seed"]), z[name], e
    pat = json.loads((G / "patches.json").read_text())
    zp = np.load(G / "z_patches.npz")
    for name, e in pat.items():
        full = tb.generate_locations(e["parent_n"], 0).coords
        sel = (full[:, 0] < e["edge"]) & (full[:, 1] < e["edge"])
        yield name, tb.LocationSet(full[sel]), zp[name], e


print("| case | n | nb | theta | mode | reference ll | B200 ll | rel. diff | tolerance | B200 s | max rank |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for name, locs, z, e in cases():
    p = tb.MaternParams(*e["theta"])
    for mode, r in e["modes"].items():
        acc = None if mode == "dense" else float(mode.split(":")[1])
        cfg = tb.LikelihoodConfig(nb=e["nb"]) if acc is None else \
            tb.LikelihoodConfig(mode="tlr", accuracy=acc, nb=e["nb"])
        tb.log_likelihood_parts(locs, z, p, cfg)
        t0 = time.perf_counter()
        ll, ld, q, st = tb.log_likelihood_parts(locs, z, p, cfg)
        dt = time.perf_counter() - t0
        rel = abs(ll - r["ll"]) / abs(r["ll"])
        tol = 1e-10 if acc is None else max(1e-8, 10 * acc)
        print(f"| {name} | {len(locs)} | {e['nb']} | {tuple(e['theta'])} | {mode} | {r['ll']:.12f} | "
              f"{ll:.12f} | {rel:.2e} | {tol:.0e} | {dt:.3f} | {st['max_rank'] if acc else '-'} |", flush=True)
