"""Pin the CPU oracle (oracle/tlr_oracle.py) against fixtures produced by the
unmodified reference (tests/golden/make_goldens.py).  CPU only."""
import math

import numpy as np
import pytest

from conftest import GOLD
from oracle import tlr_oracle as orc


def test_bessel_matches_reference():
    g = np.load(GOLD / "bessel.npz")
    for i, nu in enumerate(g["nus"]):
        got = orc.bessel_k(float(nu), g["xs"])
        np.testing.assert_allclose(got, g["kv"][i], rtol=1e-13, atol=0)


def test_bessel_frozen_values():
    # tests/oracles.py:29-31 of the reference
    assert orc.bessel_k(1.0, 1.0)[0] == pytest.approx(0.60190723019723457, rel=1e-13)
    assert orc.bessel_k(0.5, 2.0)[0] == pytest.approx(0.11993777196806145, rel=1e-13)
    assert orc.bessel_k(1.5, 1.0)[0] == pytest.approx(0.92213700889578912, rel=1e-13)


def test_locations_match_reference():
    g = np.load(GOLD / "locations.npz")
    for key in g.files:
        n, seed = map(int, key.split("_"))
        np.testing.assert_array_equal(orc.generate_locations(n, seed), g[key])


def test_tiles_match_reference():
    g = np.load(GOLD / "tiles.npz")
    for key in [k for k in g.files if k.endswith("_exact")]:
        n, seed, nu = key.split("_")[:3]
        th = {"0.5": (1.0, 0.1, 0.5), "1.7": (1.3, 0.05, 1.7), "2.5": (0.7, 0.2, 2.5)}[nu]
        xy = orc.generate_locations(int(n), int(seed))
        a = orc.matern_block(xy, xy, th)
        a[np.diag_indices_from(a)] += 0.01
        np.testing.assert_allclose(a, g[key], rtol=1e-14, atol=1e-15)
        # the reference's spline profile stays within 1e-12 of exact
        np.testing.assert_allclose(a, g[key.replace("_exact", "_auto")], rtol=0, atol=2e-12 * th[0])


def test_compression_ranks_match_reference():
    g = np.load(GOLD / "compression.npz")
    for i, j in [(1, 0), (2, 0), (3, 0), (3, 2)]:
        tile = g[f"tile_{i}_{j}"]
        for eps in (1e-5, 1e-7, 1e-9, 1e-12):
            u, v = orc.compress_tile(tile, eps)
            assert u.shape[1] == int(g[f"rank_{i}_{j}_{eps:g}"])
            err = np.linalg.norm(tile - u @ v.T)
            assert err <= eps * np.linalg.norm(tile)


def test_truncation_rank_edge_cases():
    assert orc.truncation_rank(np.zeros(0), 1e-3) == 0
    assert orc.truncation_rank(np.zeros(5), 1e-3) == 0
    assert orc.truncation_rank(np.array([1.0, 0.0]), 1e-3) == 1
    assert orc.truncation_rank(np.array([1.0, 1.0]), 1e-3) == 2


@pytest.mark.parametrize("name", ["s120", "s300", "s300nu", "s500r", "C1"])
def test_loglik_matches_reference(gold, name):
    e = gold["loglik"][name]
    th = tuple(e["theta"])
    xy = orc.generate_locations(e["n"], e["loc_seed"])
    z = gold["z"][name]
    np.testing.assert_allclose(orc.sample_measurements(xy, th, e["z_seed"]), z, rtol=1e-9,
                               atol=1e-10)
    for mode, r in e["modes"].items():
        acc = None if mode == "dense" else float(mode.split(":")[1])
        ll, ld, q = orc.log_likelihood(xy, z, th, e["nb"], acc)
        tol = 1e-10 if acc is None else max(1e-8, 10 * acc) * 1e-2
        assert abs(ll - r["ll"]) <= tol * abs(r["ll"]), (name, mode, ll, r["ll"])


def test_solves_match_reference():
    g = np.load(GOLD / "solves.npz")
    for n, nb, eps in [(120, 40, 1e-9), (150, 32, 1e-7), (200, 64, 1e-12)]:
        key = f"{n}_{nb}_{eps:g}"
        xy = orc.generate_locations(n, 33)
        th = (1.0, 0.1, 0.5)
        rhs = g[key + "_rhs"]
        for acc, tag in ((None, "dense"), (eps, "tlr")):
            D, L, ld = orc.cholesky(*orc.assemble(xy, th, nb, acc), acc)
            x = orc.backward_solve(D, L, n, nb, orc.forward_solve(D, L, n, nb, rhs))
            ref = g[f"{key}_{tag}_x"]
            assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)
            assert ld == pytest.approx(float(g[f"{key}_{tag}_logdet"]), rel=1e-11)


def test_kriging_matches_reference():
    g = np.load(GOLD / "kriging.npz")
    th = (1.0, 0.1, 0.5)
    pred = orc.predict(g["known"], g["z"], g["unknown"], th, 100)
    np.testing.assert_allclose(pred, g["dense_nb100"], rtol=1e-9, atol=1e-12)
    pred = orc.predict(g["known"], g["z"], g["unknown"], th, 100, 1e-9)
    np.testing.assert_allclose(pred, g["tlr9_nb100"], rtol=1e-7, atol=1e-9)


def test_npd_raises():
    xy = orc.generate_locations(120, 3)
    with pytest.raises(orc.NotPositiveDefiniteError):
        orc.log_likelihood(xy, np.zeros(120), (1.0, 2.0, 4.9), 48, None)
