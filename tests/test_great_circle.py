"""Great-circle metric: haversine distance on (lon, lat)
degrees, reference geometry.py:24-31,80-122 and kernels.py:460-491.

Fixtures: tests/golden/make_gcd_goldens.py (unmodified reference, n = 600
points in a 14 x 16 degree box, theta = (1, 300 km, 0.5), nb = 150).
CPU tests pin the oracle and the host-side validation; `gpu` tests run the
device path through the C ABI (tlrb_set_metric / tlrb_matern_block_metric).
"""
import json
from dataclasses import dataclass

import numpy as np
import pytest

from conftest import GOLD
from oracle import tlr_oracle as orc

R = 6371.0
TH = (1.0, 300.0, 0.5)


@pytest.fixture(scope="module")
def g():
    d = dict(np.load(GOLD / "gcd.npz"))
    d["meta"] = json.loads((GOLD / "gcd.json").read_text())
    return d


# ----------------------------------------------------------------- CPU: oracle
def test_oracle_tile_matches_reference(g):
    c = g["coords"][:64]
    np.testing.assert_allclose(orc.matern_block(c, c, TH, R), g["tile"], rtol=1e-13, atol=1e-15)


def test_oracle_distance_properties():
    # haversine: symmetric, zero on the diagonal, antipodes at pi * R
    pts = np.array([[0.0, 0.0], [180.0, 0.0], [10.0, 45.0], [-170.0, -45.0]])
    d = orc.distance_block(pts, pts, R)
    np.testing.assert_allclose(d, d.T, rtol=1e-15, atol=0)
    assert np.all(np.diag(d) == 0.0)
    assert d[0, 1] == pytest.approx(np.pi * R, rel=1e-14)
    assert d[2, 3] == pytest.approx(np.pi * R, rel=1e-7)   # antipodal pair, a clamps to 1


@pytest.mark.parametrize("mode", ["dense", "tlr:1e-07", "tlr:1e-09"])
def test_oracle_loglik_matches_reference(g, mode):
    acc = None if mode == "dense" else float(mode.split(":")[1])
    ll = orc.log_likelihood(g["coords"], g["z"], TH, 150, acc, R)[0]
    ref = g["meta"]["modes"][mode]["ll"]
    # the reference evaluates through its spline profile at n >= 256
    assert abs(ll - ref) <= 1e-11 * abs(ref)


def test_oracle_kriging_matches_reference(g):
    c = g["coords"]
    p = orc.predict(c[:560], g["z"][:560], c[560:], TH, 150, None, R)
    np.testing.assert_allclose(p, g["pred"], rtol=0, atol=1e-10)


# ------------------------------------------------------------ CPU: host logic
def test_location_set_validation():
    import paper_1804_09137_b200 as tb

    with pytest.raises(ValueError, match="great-circle"):
        tb.LocationSet([[181.0, 0.0], [0.0, 0.0]], tb.GreatCircle())
    with pytest.raises(ValueError, match="great-circle"):
        tb.LocationSet([[0.0, -90.5], [0.0, 0.0]], tb.GreatCircle(100.0))
    with pytest.raises(ValueError, match="radius"):
        tb.GreatCircle(0.0)
    with pytest.raises(ValueError, match="radius"):
        tb.GreatCircle(float("inf"))
    ok = tb.LocationSet([[180.0, 90.0], [-180.0, -90.0]], tb.GreatCircle())
    assert len(ok) == 2 and tb.api._radius_of(ok) == R


def test_metric_duck_typing_and_mismatch():
    """Reference metric objects are accepted by class name; known / unknown
    sets with different metrics are rejected like predict.py:30-32."""
    import paper_1804_09137_b200 as tb

    @dataclass(frozen=True)
    class GreatCircle:          # stands in for tlrgeo.geometry.GreatCircle
        radius: float = 1000.0

    assert tb.api.sphere_radius(GreatCircle()) == 1000.0
    assert tb.api.sphere_radius(tb.Euclidean()) == 0.0
    assert tb.api.sphere_radius(None) == 0.0
    known = tb.LocationSet([[0.0, 0.0], [1.0, 1.0]], tb.GreatCircle())
    unknown = tb.LocationSet([[0.5, 0.5]])
    with pytest.raises(ValueError, match="different metrics"):
        tb.PredictionProblem(known, np.zeros(2), unknown, tb.MaternParams(*TH))


# ----------------------------------------------------------------- GPU parity
@pytest.mark.gpu
def test_matern_block_device(tb, g):
    c = g["coords"][:64]
    a = tb.matern_block(c, c, tb.MaternParams(*TH), R)
    np.testing.assert_allclose(a, g["tile"], rtol=1e-12, atol=1e-15)
    # rectangular, rows != cols, against the oracle
    c = g["coords"]
    a = tb.matern_block(c[:100], c[100:250], tb.MaternParams(0.7, 500.0, 1.7), R)
    np.testing.assert_allclose(a, orc.matern_block(c[:100], c[100:250], (0.7, 500.0, 1.7), R),
                               rtol=1e-12, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["dense", "tlr:1e-07", "tlr:1e-09"])
def test_loglik_device(tb, g, mode):
    acc = None if mode == "dense" else float(mode.split(":")[1])
    locs = tb.LocationSet(g["coords"], tb.GreatCircle())
    cfg = tb.LikelihoodConfig(mode="dense" if acc is None else "tlr", accuracy=acc, nb=150)
    ll = tb.log_likelihood(locs, g["z"], tb.MaternParams(*TH), cfg)
    ref = g["meta"]["modes"][mode]["ll"]
    tol = 1e-10 if acc is None else max(1e-8, 10 * acc)
    assert abs(ll - ref) <= tol * abs(ref), (ll, ref)


@pytest.mark.gpu
def test_euclidean_handle_unchanged_by_metric_api(tb, g):
    """The same coordinates read as planar points give a different (Euclidean)
    likelihood, equal to the oracle's: the metric is per handle."""
    c = g["coords"]
    th = (1.0, 3.0, 0.5)
    ll = tb.log_likelihood(tb.LocationSet(c), g["z"], tb.MaternParams(*th),
                           tb.LikelihoodConfig(mode="dense", nb=150))
    ref = orc.log_likelihood(c, g["z"], th, 150)[0]
    assert abs(ll - ref) <= 1e-10 * abs(ref)


@pytest.mark.gpu
def test_sample_measurements_device(tb, g):
    z = tb.sample_measurements(tb.LocationSet(g["coords"], tb.GreatCircle()), tb.MaternParams(*TH), 1)
    np.testing.assert_allclose(z, g["z"], rtol=0, atol=1e-10)


@pytest.mark.gpu
def test_kriging_device(tb, g):
    c = g["coords"]
    known = tb.LocationSet(c[:560], tb.GreatCircle())
    unknown = tb.LocationSet(c[560:], tb.GreatCircle())
    pred = tb.predict(tb.PredictionProblem(known, g["z"][:560], unknown, tb.MaternParams(*TH), nb=150))
    np.testing.assert_allclose(pred, g["pred"], rtol=0, atol=1e-9)
    # TLR kriging against the oracle's TLR kriging at the same accuracy
    pt = tb.predict(tb.PredictionProblem(known, g["z"][:560], unknown, tb.MaternParams(*TH),
                                         mode="tlr", accuracy=1e-9, nb=150))
    po = orc.predict(c[:560], g["z"][:560], c[560:], TH, 150, 1e-9, R)
    assert np.abs(pt - po).max() <= 1e-7 * np.abs(po).max()


@pytest.mark.gpu
def test_set_metric_rejects_bad_coordinates(tb):
    xy = np.array([[0.0, 0.0], [200.0, 10.0]])
    with pytest.raises(ValueError):
        tb.Handle(xy, 2, radius=R)
    with pytest.raises(ValueError):
        tb.matern_block(xy, xy, tb.MaternParams(*TH), R)
