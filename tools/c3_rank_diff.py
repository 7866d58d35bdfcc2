"""C3 TLR(1e-7), uncapped: factor rank map against the reference golden (tests/golden/c3_tlr.json)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1804_09137_b200 as tb  # noqa: E402

e = json.loads((ROOT / "tests/golden/c3_tlr.json").read_text())["C3"]
locs = tb.generate_locations(e["n"], 0)
z = np.load(ROOT / "tests/golden/z_c3.npz")["C3"]
h = tb.Handle(locs.coords, e["nb"])
ll, ld, q = h.loglik(z, tb.MaternParams(*e["theta"]), e["acc"])
rm = h.rank_map()
print("ll", ll, "ref", e["ll"], "rel", abs(ll - e["ll"]) / abs(e["ll"]), "stats", h.last_stats["ms_device"])
rows = []
for k, r in e["factor_ranks"].items():
    i, j = map(int, k.split(","))
    rows.append((i, j, r, int(rm[i, j])))
d = np.array([a[3] - a[2] for a in rows])
print("tiles", len(d), "equal", int((d == 0).sum()), "within 1", int((abs(d) <= 1).sum()), "within 4", int((abs(d) <= 4).sum()),
      "max", int(abs(d).max()))
for a in sorted(rows, key=lambda a: -abs(a[3] - a[2]))[:25]:
    print(a)
