"""One warm TLR evaluation of a BASELINE config for TLRB_TRACE runs (z is
standard normal: tile ranks and the work do not depend on z):
    TLRB_TRACE=1 python tools/trace_cfg.py C3 2> trace.log
--dense: the dense (no compression) evaluation instead."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_09137_b200 as tb  # noqa: E402
from tools.run_config import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1]]
warm = "--no-warm" not in sys.argv
locs = tb.generate_locations(c["n"], 0)
z = np.random.default_rng(1).standard_normal(c["n"])
h = tb.Handle(locs.coords, c["nb"], max_rank=c["max_rank"] or 0)
p = tb.MaternParams(*c["theta"])
acc = None if "--dense" in sys.argv else c["acc"]
if warm:
    h.loglik(z, p, acc)
print("---- warm", file=sys.stderr, flush=True)
prof = "--profile" in sys.argv   # per-kernel-class event times (serialising)
if prof:
    from paper_1804_09137_b200 import _lib
    _lib.profile_enable(True)
t0 = time.perf_counter()
ll = h.loglik(z, p, acc)
print(f"ll {ll[0]!r}  wall {time.perf_counter() - t0:.3f} s  stats {h.last_stats}")
if prof:
    for k, v in sorted(_lib.profile_read().items(), key=lambda kv: -kv[1]["ms"]):
        print(f"  {k:16s} {v['ms']:10.1f} ms  {v['launches']:7d} launches  "
              f"{v['flops'] / 1e9:10.1f} GF  {v['bytes'] / 1e9:8.2f} GB")
