"""CSV ingestion against the reference's own outputs on the
same files (tests/golden/make_dataio_goldens.py) plus the reference test
suite's round-trip properties (tests/test_dataio.py of the reference).  CPU."""
import json

import numpy as np
import pytest

from conftest import GOLD
from paper_1804_09137_b200 import dataio
from paper_1804_09137_b200.api import GreatCircle, LocationSet

D = GOLD / "dataio"
EXPECT = json.loads((D / "expected.json").read_text())
LOAD_CASES = sorted(k for k in EXPECT if k.endswith((":drop", ":strict")))


@pytest.mark.parametrize("key", LOAD_CASES)
def test_load_dataset_matches_reference(key):
    name, policy = key.split(":")
    metric = GreatCircle() if name.startswith("gcd") else None
    want = EXPECT[key]
    if "error" in want:
        with pytest.raises(Exception) as exc:
            dataio.load_dataset(D / name, metric, missing_policy=policy)
        assert type(exc.value).__name__ == want["error"]
        assert str(exc.value).replace(str(D / name), "<path>") == want["msg"]
    else:
        ds = dataio.load_dataset(D / name, metric, missing_policy=policy)
        assert np.array_equal(ds.locations.coords, np.array(want["coords"]))
        assert np.array_equal(ds.values, np.array(want["values"]))
        assert ds.provenance == str(D / name)


@pytest.mark.parametrize("grid", ["1x1", "2x2", "4x2", "3x3", "2x3"])
def test_partition_matches_reference(grid):
    r, c = map(int, grid.split("x"))
    ds = dataio.load_dataset(D / "random.csv")
    got = dataio.partition_regions(ds, r, c)
    want = EXPECT[f"partition:{grid}"]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert np.array_equal(g.locations.coords, np.array(w["coords"]))
        assert np.array_equal(g.values, np.array(w["values"]))
        assert g.provenance.replace(str(D / "random.csv"), "<path>") == w["provenance"]
    assert sum(len(g.locations) for g in got) == len(ds.locations)


def test_writers_byte_identical_to_reference(tmp_path):
    ds = dataio.load_dataset(D / "random.csv")
    dataio.save_dataset(tmp_path / "a.csv", ds)
    assert (tmp_path / "a.csv").read_text() == EXPECT["saved_random"]
    locs = LocationSet(np.array([[10.0, 20.0], [11.0, 21.0]]), GreatCircle())
    dataio.save_locations(tmp_path / "l.csv", locs)
    assert (tmp_path / "l.csv").read_text() == EXPECT["saved_gcd_locations"]
    dataio.save_predictions(tmp_path / "p.csv", locs, np.array([0.5, -1.25]), np.array([1.0 / 3, 2.0]))
    assert (tmp_path / "p.csv").read_text() == EXPECT["saved_predictions"]


def test_round_trips_bitwise(tmp_path):
    rng = np.random.default_rng(3)
    coords, vals = rng.uniform(0, 1, (25, 2)), rng.standard_normal(25) * 1e-7
    ds = dataio.Dataset(LocationSet(coords), vals, provenance="t")
    dataio.save_dataset(tmp_path / "d.csv", ds)
    back = dataio.load_dataset(tmp_path / "d.csv")
    assert np.array_equal(back.locations.coords, coords) and np.array_equal(back.values, vals)
    dataio.save_dataset(tmp_path / "d2.csv", back)
    assert (tmp_path / "d.csv").read_bytes() == (tmp_path / "d2.csv").read_bytes()
    assert b"\r" not in (tmp_path / "d.csv").read_bytes()
    dataio.save_values(tmp_path / "v.csv", vals)
    assert np.array_equal(dataio.load_values(tmp_path / "v.csv"), vals)
    locs = LocationSet(rng.uniform(-10, 10, (12, 2)))
    dataio.save_locations(tmp_path / "l.csv", locs)
    assert np.array_equal(dataio.load_locations(tmp_path / "l.csv").coords, locs.coords)
    with pytest.raises(dataio.DataError, match="header"):
        dataio.load_locations(tmp_path / "l.csv", GreatCircle())
    pred, truth = rng.standard_normal(12), rng.standard_normal(12)
    dataio.save_predictions(tmp_path / "p.csv", locs, pred, truth)
    c, p, t = dataio.load_predictions(tmp_path / "p.csv")
    assert np.array_equal(c, locs.coords) and np.array_equal(p, pred) and np.array_equal(t, truth)
    dataio.save_predictions(tmp_path / "p.csv", locs, pred)
    assert dataio.load_predictions(tmp_path / "p.csv")[2] is None


def test_trace_format(tmp_path):
    from paper_1804_09137_b200.mle import TraceEntry

    trace = [TraceEntry(0, (1.0, 0.1, 0.5), -12.5, 0.01), TraceEntry(1, (1.1, 0.2, 0.6), -11.0, 0.02)]
    dataio.save_trace(tmp_path / "t.csv", trace)
    lines = (tmp_path / "t.csv").read_text().strip().split("\n")
    assert lines[0] == "iter,theta1,theta2,theta3,loglik,seconds"
    assert lines[1].startswith("0,1,") and len(lines) == 3


def test_invalid_arguments():
    ds = dataio.load_dataset(D / "plain.csv")
    with pytest.raises(ValueError):
        dataio.partition_regions(ds, 0, 2)
    with pytest.raises(ValueError, match="policy"):
        dataio.load_dataset(D / "plain.csv", missing_policy="fill")
