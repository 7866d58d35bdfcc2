"""Generate golden fixtures by running the UNMODIFIED reference (`tlrgeo`).

Run here (the container that has /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_goldens.py [--big]

Outputs (committed, small): tests/golden/*.npz / *.json.  Nothing on the GPU
box imports the reference; tests and bench read only these files.
Reference call sites used (all /root/reference/pkg/src/tlrgeo/):
  geometry.generate_locations (geometry.py:186-206)
  kernels.bessel_k / matern_block (kernels.py:216-226, 494-530)
  tilestore.assemble_covariance + dump_tiles (tilestore.py:181-223, 138-147)
  stats.sample_measurements / log_likelihood (stats.py:103-133)
  linalg.dense_cholesky / tlr_cholesky / solve_cholesky (linalg.py:82-197)
  predict.predict (predict.py:65-87)
"""
import io
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

import tlrgeo
from tlrgeo import (LikelihoodConfig, LocationSet, MaternParams, PredictionProblem,
                    TileGrid, assemble_covariance, bessel_k, dense_cholesky,
                    generate_locations, log_likelihood, predict, sample_measurements,
                    solve_cholesky, tlr_cholesky)
from tlrgeo import kernels, compression

OUT = Path(__file__).resolve().parent


def ll_parts(locs, z, p, mode, acc, nb):
    n = len(locs)
    grid = TileGrid(n, min(nb, n))
    cov = assemble_covariance(locs, p, grid, mode, acc)
    from tlrgeo import linalg
    f = linalg.cholesky(cov)
    quad = linalg.quadratic_form(f, z)
    ll = -0.5 * (n * math.log(2 * math.pi) + f.log_det + quad)
    ranks = None
    if mode == "tlr":
        ranks = {f"{i},{j}": int(cov.lower[(i, j)].rank) for (i, j) in cov.lower}
        franks = {f"{i},{j}": int(f.lower[(i, j)].rank) for (i, j) in f.lower}
    else:
        franks = None
    return dict(ll=ll, log_det=f.log_det, quad=quad, init_ranks=ranks, factor_ranks=franks)


def main(big: bool):
    t_start = time.time()
    # ---- special functions -------------------------------------------------
    nus = [0.1, 0.3, 0.5, 0.8, 1.0, 1.5, 1.7, 2.3, 2.5, 3.7, 5.0]
    xs = [1e-8, 1e-4, 0.01, 0.1, 0.5, 1.0, 1.99, 2.0, 2.01, 5.0, 20.0, 50.0, 300.0]
    kv = np.array([[bessel_k(nu, x) for x in xs] for nu in nus])
    np.savez(OUT / "bessel.npz", nus=np.array(nus), xs=np.array(xs), kv=kv)

    # ---- locations ---------------------------------------------------------
    loc_cases = {}
    for n, seed in [(1, 0), (7, 3), (64, 0), (1600, 0), (10000, 0)]:
        c = generate_locations(n, seed).coords
        loc_cases[f"{n}_{seed}"] = c
    np.savez(OUT / "locations.npz", **loc_cases)

    # ---- covariance tiles (exact and profile) ------------------------------
    tiles = {}
    for (n, seed, th) in [(64, 0, (1.0, 0.1, 0.5)), (300, 2, (1.3, 0.05, 1.7)),
                          (300, 2, (0.7, 0.2, 2.5))]:
        locs = generate_locations(n, seed)
        p = MaternParams(*th, nugget=0.01)
        key = f"{n}_{seed}_{th[2]}"
        tiles[key + "_exact"] = assemble_covariance(locs, p, TileGrid(n, n), "dense",
                                                    profile="never").diag[0]
        tiles[key + "_auto"] = assemble_covariance(locs, p, TileGrid(n, n), "dense",
                                                   profile="auto").diag[0]
    np.savez(OUT / "tiles.npz", **tiles)

    # ---- compression of individual tiles -----------------------------------
    comp = {}
    locs = generate_locations(1600, 0)
    p = MaternParams(1.0, 0.1, 0.5)
    view = [locs.kernel_view(i * 400, (i + 1) * 400) for i in range(4)]
    for (i, j) in [(1, 0), (2, 0), (3, 0), (3, 2)]:
        blk = kernels.matern_block(view[i], view[j], p, None)
        comp[f"tile_{i}_{j}"] = blk
        for eps in (1e-5, 1e-7, 1e-9, 1e-12):
            lr = compression.compress_tile(blk, eps)
            comp[f"rank_{i}_{j}_{eps:g}"] = np.array(lr.rank)
            comp[f"err_{i}_{j}_{eps:g}"] = np.array(np.linalg.norm(blk - lr.to_dense()))
    np.savez(OUT / "compression.npz", **comp)

    # ---- likelihood goldens ------------------------------------------------
    lik = {}
    small = [
        # (name, n, loc_seed, theta, z_seed, nb, modes)
        ("s120", 120, 33, (1.0, 0.1, 0.5), 1, 40, [("dense", None), ("tlr", 1e-9), ("tlr", 1e-7)]),
        ("s300", 300, 8, (1.0, 0.1, 0.5), 5, 75, [("dense", None), ("tlr", 1e-9)]),
        ("s300nu", 300, 8, (1.0, 0.1, 1.0), 5, 64, [("dense", None), ("tlr", 1e-9), ("tlr", 1e-5)]),
        ("s500r", 500, 3, (1.5, 0.05, 0.8, 0.01), 2, 96, [("dense", None), ("tlr", 1e-7)]),
        ("C1", 1600, 0, (1.0, 0.1, 0.5), 1, 400, [("dense", None), ("tlr", 1e-9), ("tlr", 1e-7), ("tlr", 1e-5)]),
    ]
    if big:
        small.append(("C2", 10000, 0, (1.0, 0.1, 0.5), 1, 500,
                      [("dense", None), ("tlr", 1e-9), ("tlr", 1e-7), ("tlr", 1e-5)]))
    zs = {}
    for name, n, lseed, th, zseed, nb, modes in small:
        locs = generate_locations(n, lseed)
        p = MaternParams(*th)
        z = sample_measurements(locs, p, zseed)
        zs[name] = z
        entry = dict(n=n, loc_seed=lseed, theta=list(th), z_seed=zseed, nb=nb, modes={})
        for mode, acc in modes:
            t0 = time.time()
            r = ll_parts(locs, z, p, mode, acc, nb)
            # cross-check against the public entry point
            cfg = LikelihoodConfig(mode=mode, accuracy=acc, nb=nb, nugget=p.nugget)
            r["ll_public"] = log_likelihood(locs, z, p, cfg)
            r["seconds"] = time.time() - t0
            entry["modes"]["dense" if mode == "dense" else f"tlr:{acc:g}"] = r
            print(name, mode, acc, r["ll"], f"{r['seconds']:.1f}s", flush=True)
        lik[name] = entry
    np.savez(OUT / ("z_big.npz" if big else "z.npz"), **zs)
    with open(OUT / ("loglik_big.json" if big else "loglik.json"), "w") as fh:
        json.dump(lik, fh, indent=1)

    if not big:
        # ---- solves (test_linalg.py:143-155 style) -------------------------
        sol = {}
        for n, nb, eps in [(120, 40, 1e-9), (150, 32, 1e-7), (200, 64, 1e-12)]:
            locs = generate_locations(n, 33)
            p = MaternParams(1.0, 0.1, 0.5)
            rhs = np.random.default_rng(1).standard_normal(n)
            d = dense_cholesky(assemble_covariance(locs, p, TileGrid(n, nb), "dense"))
            t = tlr_cholesky(assemble_covariance(locs, p, TileGrid(n, nb), "tlr", eps))
            sol[f"{n}_{nb}_{eps:g}_rhs"] = rhs
            sol[f"{n}_{nb}_{eps:g}_dense_x"] = solve_cholesky(d, rhs)
            sol[f"{n}_{nb}_{eps:g}_tlr_x"] = solve_cholesky(t, rhs)
            sol[f"{n}_{nb}_{eps:g}_dense_logdet"] = np.array(d.log_det)
            sol[f"{n}_{nb}_{eps:g}_tlr_logdet"] = np.array(t.log_det)
        np.savez(OUT / "solves.npz", **sol)

        # ---- kriging (predict.py:65-87) ------------------------------------
        kr = {}
        theta = MaternParams(1.0, 0.1, 0.5)
        locs = generate_locations(320, 4)
        z = sample_measurements(locs, theta, 5)
        known = LocationSet(locs.coords[:300], locs.metric)
        unknown = LocationSet(locs.coords[300:], locs.metric)
        kr["known"] = known.coords
        kr["unknown"] = unknown.coords
        kr["z"] = z[:300]
        kr["dense_nb100"] = predict(PredictionProblem(known, z[:300], unknown, theta, nb=100))
        kr["tlr9_nb100"] = predict(PredictionProblem(known, z[:300], unknown, theta, "tlr", 1e-9, 100))
        # exact interpolation case (test_predict.py:30-37)
        locs2 = generate_locations(320, 12)
        z2 = sample_measurements(locs2, theta, 7)
        kr["interp_locs"] = locs2.coords
        kr["interp_z"] = z2
        # C1 holdout (predict.py:100-127 index draw) m=100, seed 2
        locs3 = generate_locations(1600, 0)
        z3 = sample_measurements(locs3, theta, 1)
        rng = np.random.default_rng(2)
        idx = np.sort(rng.choice(1600, size=100, replace=False))
        mask = np.zeros(1600, bool)
        mask[idx] = True
        kn = LocationSet(locs3.coords[~mask]); un = LocationSet(locs3.coords[mask])
        kr["c1_holdout_idx"] = idx
        kr["c1_dense"] = predict(PredictionProblem(kn, z3[~mask], un, theta, "dense", None, 400))
        kr["c1_tlr9"] = predict(PredictionProblem(kn, z3[~mask], un, theta, "tlr", 1e-9, 400))
        np.savez(OUT / "kriging.npz", **kr)
    print("done in", time.time() - t_start)


if __name__ == "__main__":
    main("--big" in sys.argv)
