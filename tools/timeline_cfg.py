"""Kernel timeline of one warm TLR evaluation (TLRB_TIMELINE dump of the
per-launch CUDA events): busy/idle time, per-class union, time buckets.
    python tools/timeline_cfg.py C3 [acc] [--bucket MS]"""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
path = os.path.join(tempfile.gettempdir(), "tlrb_timeline.txt")
os.environ["TLRB_TIMELINE"] = path
import paper_1804_09137_b200 as tb  # noqa: E402
from paper_1804_09137_b200 import _lib  # noqa: E402

from tools.run_config import CONFIGS  # noqa: E402

argv = sys.argv[1:]
if "--bucket" in argv:
    del argv[argv.index("--bucket"):argv.index("--bucket") + 2]
args = [a for a in argv if not a.startswith("--")]
cfg = CONFIGS[args[0] if args else "C2"]
acc = float(args[1]) if len(args) > 1 else cfg["acc"]
B = float(sys.argv[sys.argv.index("--bucket") + 1]) if "--bucket" in sys.argv else 10.0
locs = tb.generate_locations(cfg["n"], 0)
z = np.random.default_rng(1).standard_normal(cfg["n"])
h = tb.Handle(locs.coords, cfg["nb"], max_rank=cfg["max_rank"] or 0)
p = tb.MaternParams(*cfg["theta"])
h.loglik(z, p, acc)
if os.path.exists(path):
    os.remove(path)
_lib.profile_enable(True)
h.loglik(z, p, acc)
_lib.profile_read()
rows = [ln.split() for ln in open(path)]
ev = sorted((float(a), float(b), c) for c, a, b, *_ in rows)
t0 = ev[0][0]
end = max(b for _, b, _ in ev)


def union(iv):
    tot, cur_a, cur_b = 0.0, None, None
    for a, b in sorted(iv):
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                tot += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    if cur_b is not None:
        tot += cur_b - cur_a
    return tot


busy = union([(a, b) for a, b, _ in ev])
print(f"span {end - t0:.1f} ms  busy(any kernel) {busy:.1f} ms  idle {end - t0 - busy:.1f} ms  launches {len(ev)}")
for c in sorted({c for _, _, c in ev}):
    iv = [(a, b) for a, b, cc in ev if cc == c]
    print(f"  {c:16s} union {union(iv):8.1f} ms  sum {sum(b - a for a, b in iv):8.1f} ms  n {len(iv)}")
# buckets: fraction of time each class is active
nb = int((end - t0) / B) + 1
cls = sorted({c for _, _, c in ev})
print("bucket(ms) " + " ".join(f"{c[:6]:>6s}" for c in cls) + "  idle")
for k in range(nb):
    lo, hi = t0 + k * B, t0 + (k + 1) * B
    fr = []
    for c in cls:
        iv = [(max(a, lo), min(b, hi)) for a, b, cc in ev if cc == c and b > lo and a < hi]
        fr.append(union(iv) / B)
    anyiv = [(max(a, lo), min(b, hi)) for a, b, _ in ev if b > lo and a < hi]
    print(f"{k * B:8.0f}   " + " ".join(f"{f:6.2f}" for f in fr) + f"  {1 - union(anyiv) / B:5.2f}")
# GEMM launches: achieved TFLOP/s distribution (weighted by time)
g = [(float(b) - float(a), float(r[4])) for r in rows for (c, a, b) in [(r[0], r[1], r[2])] if c == "dgemm_vbatch" and len(r) > 4]
if g:
    import collections
    bins = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for dt, fl in g:
        tf = fl / (dt * 1e-3) / 1e12 if dt > 0 else 0.0
        k = "<0.5" if tf < 0.5 else "<2" if tf < 2 else "<5" if tf < 5 else "<10" if tf < 10 else "<20" if tf < 20 else ">=20"
        bins[k][0] += dt; bins[k][1] += fl; bins[k][2] += 1
    print("GEMM launches by achieved TFLOP/s: bucket  ms  GFLOP  launches")
    for k in ("<0.5", "<2", "<5", "<10", "<20", ">=20"):
        if k in bins:
            v = bins[k]
            print(f"  {k:5s} {v[0]:8.2f} {v[1] / 1e9:9.2f} {v[2]:6d}")
# optional window listing: TL_WINDOW="t0,t1" (ms relative to the first launch)
win = os.environ.get("TL_WINDOW")
if win:
    lo, hi = (float(v) for v in win.split(","))
    print(f"launches in [{lo}, {hi}] ms:")
    for r in sorted(rows, key=lambda r: float(r[1])):
        a, b = float(r[1]) - t0, float(r[2]) - t0
        if b >= lo and a <= hi:
            print(f"  {a:9.3f} {b:9.3f} {1e3 * (b - a):8.1f} us  {r[0]:15s} {r[3][-6:]}  {float(r[4]) / 1e9 if len(r) > 4 else 0:8.3f} GF")
