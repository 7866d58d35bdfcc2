"""CSV ingestion goldens from the UNMODIFIED reference (dataio.py:141-221):
a set of input files (tests/golden/dataio/*.csv) and what the reference's
loaders return for each (arrays, or the error class + message with the
temporary path replaced by <path>).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_dataio_goldens.py
"""
import json
from pathlib import Path

import numpy as np

from tlrgeo import Dataset, GreatCircle, LocationSet
from tlrgeo import dataio

OUT = Path(__file__).resolve().parent / "dataio"
OUT.mkdir(exist_ok=True)
rng = np.random.default_rng(5)

files = {
    "plain.csv": "x,y,value\n0.1,0.2,1.5\n0.3,0.4,2.5\n0.5,0.6,3.5\n",
    "missing.csv": "x,y,value\n0.1,0.2,1.5\n0.3,0.4,NA\n0.5,0.6,\n\n0.7,0.8,2.0\n",
    "dups.csv": "x,y,value\n0.5,0.5,1\n0.1,0.2,1.0\n0.3,0.4,2.0\n0.5,0.5,7\n0.1,0.2,3.0\n",
    "malformed.csv": "x,y,value\n0.1,0.2,1.0\nbogus,0.4,2.0\n",
    "short.csv": "x,y,value\n0.1,0.2,1.0\n0.3,0.4\n",
    "allna.csv": "x,y,value\n0.1,0.2,NA\n",
    "header.csv": "a,b,c\n1,2,3\n",
    "header_case.csv": " X , Y ,Value\n1,2,3\n2,3,4\n",
    "empty.csv": "",
    "gcd.csv": "lon,lat,value\n10,20,1.0\n11,21,2.0\n-179.5,-89,3\n",
    "gcd_range.csv": "lon,lat,value\n10,20,1.0\n181,21,2.0\n",
    "nonfinite.csv": "x,y,value\n0.1,0.2,inf\n",
}
c = rng.uniform(-5, 7, (137, 2))
v = rng.standard_normal(137) * 1e-7
files["random.csv"] = "x,y,value\n" + "".join(f"{format(a, '.17g')},{format(b, '.17g')},{format(w, '.17g')}\n"
                                            for (a, b), w in zip(c, v))
for name, text in files.items():
    (OUT / name).write_text(text, encoding="utf-8")

expect = {}
for name in files:
    metric = GreatCircle() if name.startswith("gcd") else None
    for policy in ("drop", "strict"):
        key = f"{name}:{policy}"
        try:
            ds = dataio.load_dataset(OUT / name, *( [metric] if metric else []), missing_policy=policy)
            expect[key] = {"coords": ds.locations.coords.tolist(), "values": ds.values.tolist()}
        except Exception as e:
            expect[key] = {"error": type(e).__name__, "msg": str(e).replace(str(OUT / name), "<path>")}
ds = dataio.load_dataset(OUT / "random.csv")
for r, cc in [(1, 1), (2, 2), (4, 2), (3, 3), (2, 3)]:
    expect[f"partition:{r}x{cc}"] = [
        {"coords": g.locations.coords.tolist(), "values": g.values.tolist(),
         "provenance": g.provenance.replace(str(OUT / "random.csv"), "<path>")}
        for g in dataio.partition_regions(ds, r, cc)]
dataio.save_dataset(OUT / "random_saved.csv.out", ds)
expect["saved_random"] = (OUT / "random_saved.csv.out").read_text()
(OUT / "random_saved.csv.out").unlink()
locs = LocationSet(np.array([[10.0, 20.0], [11.0, 21.0]]), GreatCircle())
tmp = OUT / "tmp.out"
dataio.save_locations(tmp, locs)
expect["saved_gcd_locations"] = tmp.read_text()
dataio.save_predictions(tmp, locs, np.array([0.5, -1.25]), np.array([1.0 / 3, 2.0]))
expect["saved_predictions"] = tmp.read_text()
tmp.unlink()
(OUT / "expected.json").write_text(json.dumps(expect, indent=0))
print(len(expect), "cases")
