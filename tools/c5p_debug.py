"""C5p patch (nb=1900) TLR evaluation for debugging: python tools/c5p_debug.py [acc]"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_09137_b200 as tb  # noqa: E402
acc = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-5
full = tb.generate_locations(1_000_000, 0).coords
m = (full[:, 0] < 0.1) & (full[:, 1] < 0.1)
locs = tb.LocationSet(full[m])
z = np.random.default_rng(1).standard_normal(len(locs))
print(len(locs), tb.log_likelihood(locs, z, tb.MaternParams(1.0, 0.03, 0.5),
                                   tb.LikelihoodConfig(mode="tlr", accuracy=acc, nb=1900)))
