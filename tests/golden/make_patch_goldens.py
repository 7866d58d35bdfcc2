"""Geometry-matched 10K-point patch goldens, from the
UNMODIFIED reference.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_patch_goldens.py

Each patch takes the full generator's points with x < e and y < e in their
original order (a 100x100 jittered sub-grid, n = 10,000) at the parent
config's theta / nb / acc; z = sample_measurements(patch, theta, 1).
Writes tests/golden/patches.json and tests/golden/z_patches.npz.
"""
import json
import math
import time
from pathlib import Path

import numpy as np

from tlrgeo import (LocationSet, MaternParams, TileGrid, assemble_covariance, generate_locations,
                    sample_measurements)
from tlrgeo import linalg

OUT = Path(__file__).resolve().parent
PATCHES = [
    # name, parent n, edge, theta, nb, accs
    ("C3p", 62_500, 0.4, (1.0, 0.03, 0.5), 760, [1e-7]),
    ("C4p", 250_000, 0.2, (1.0, 0.1, 1.0), 1000, [1e-7, 1e-9]),
    ("C5p", 1_000_000, 0.1, (1.0, 0.03, 0.5), 1900, [1e-5]),
]


def main():
    out, zs = {}, {}
    for name, parent, e, th, nb, accs in PATCHES:
        full = generate_locations(parent, 0).coords
        sel = (full[:, 0] < e) & (full[:, 1] < e)
        locs = LocationSet(full[sel])
        n = len(locs)
        p = MaternParams(*th)
        t0 = time.time()
        z = sample_measurements(locs, p, 1)
        zs[name] = z
        entry = {"parent_n": parent, "edge": e, "n": n, "theta": list(th), "nb": nb, "modes": {}}
        for mode, acc in [("dense", None)] + [("tlr", a) for a in accs]:
            t1 = time.time()
            grid = TileGrid(n, min(nb, n))
            cov = assemble_covariance(locs, p, grid, mode, acc)
            f = linalg.cholesky(cov)
            quad = linalg.quadratic_form(f, z)
            ll = -0.5 * (n * math.log(2 * math.pi) + f.log_det + quad)
            key = "dense" if mode == "dense" else f"tlr:{acc:g}"
            r = {"ll": ll, "log_det": f.log_det, "quad": quad, "seconds": time.time() - t1}
            if mode == "tlr":
                r["factor_ranks"] = {f"{i},{j}": int(f.lower[(i, j)].rank) for (i, j) in f.lower}
            entry["modes"][key] = r
            print(name, key, ll, f"{time.time() - t1:.1f}s", flush=True)
        out[name] = entry
        np.savez(OUT / "z_patches.npz", **zs)
        (OUT / "patches.json").write_text(json.dumps(out, indent=1))
    print("done")


if __name__ == "__main__":
    main()
