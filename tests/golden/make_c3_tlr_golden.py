"""Full C3 TLR(1e-7) golden from the UNMODIFIED reference (slow: ~5 h on 8
host cores, SURVEY.md 8(c) "C3 TLR: one long run, done once").  Uses the z
of make_c3_golden.py (tests/golden/z_c3.npz) and the reference's own
assemble_covariance / cholesky / quadratic_form at nb = 760, acc = 1e-7 (the
reference has no max-rank cap; ours stores over-cap tiles exactly, which
never truncates below acc).  Writes tests/golden/c3_tlr.json.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c3_tlr_golden.py
"""
import json
import math
import time
from pathlib import Path

import numpy as np

from tlrgeo import MaternParams, TileGrid, assemble_covariance, generate_locations
from tlrgeo import linalg

OUT = Path(__file__).resolve().parent
locs = generate_locations(62_500, 0)
p = MaternParams(1.0, 0.03, 0.5)
z = np.load(OUT / "z_c3.npz")["C3"]
t1 = time.time()
cov = assemble_covariance(locs, p, TileGrid(62_500, 760), "tlr", 1e-7)
t_asm = time.time() - t1
init_ranks = {f"{i},{j}": int(cov.lower[(i, j)].rank) for (i, j) in cov.lower}
print("assembled", t_asm, flush=True)
f = linalg.cholesky(cov)
quad = linalg.quadratic_form(f, z)
ll = -0.5 * (62_500 * math.log(2 * math.pi) + f.log_det + quad)
(OUT / "c3_tlr.json").write_text(json.dumps({"C3": {
    "n": 62500, "theta": [1.0, 0.03, 0.5], "nb": 760, "acc": 1e-7,
    "ll": ll, "log_det": f.log_det, "quad": quad, "seconds": time.time() - t1,
    "assemble_seconds": t_asm,
    "initial_ranks": init_ranks,
    "factor_ranks": {f"{i},{j}": int(f.lower[(i, j)].rank) for (i, j) in f.lower}}}))
print("tlr", ll, time.time() - t1, flush=True)
