"""The reference's own pinning tests, restated on the
device path: every call goes through libtlrb200.so.  Each test cites the
reference test it mirrors; tolerances are the reference's."""
import math

import numpy as np
import pytest

from conftest import GOLD
from oracle import tlr_oracle as orc

pytestmark = pytest.mark.gpu

EPS_GRID = (1e-5, 1e-7, 1e-9, 1e-12)   # test_acceptance.py:40


def test_potrf_tile_not_positive_definite_pivot(tb):
    """test_linalg.py:59-64: eye(5) with a[3,3] = -1 fails at pivot 3 of the
    given tile, with the reference's message."""
    a = np.eye(5)
    a[3, 3] = -1.0
    with pytest.raises(tb.NotPositiveDefiniteError) as exc:
        tb.potrf_tile(a, tile_index=7)
    assert exc.value.pivot_index == 3 and exc.value.tile_index == 7
    assert "nugget" in str(exc.value)


def test_potrf_tile_factor(tb):
    """test_linalg.py:40-57: [[4,2],[2,5]] -> [[2,0],[1,2]]; a random SPD
    tile: ||L L^T - A|| / ||A|| <= 1e-13, positive diagonal, lower."""
    np.testing.assert_allclose(tb.potrf_tile(np.array([[4.0, 2.0], [2.0, 5.0]])), [[2.0, 0.0], [1.0, 2.0]],
                               rtol=1e-15)
    rng = np.random.default_rng(20240817)
    b = rng.standard_normal((70, 70))
    a = b @ b.T + 70 * np.eye(70)
    el = tb.potrf_tile(a)
    assert np.linalg.norm(el @ el.T - a) / np.linalg.norm(a) <= 1e-13
    assert (np.diag(el) > 0).all() and np.array_equal(el, np.tril(el))


def test_npd_tile_and_pivot_vs_reference(tb):
    """test_linalg.py:121-127 case (smooth long-range kernel, no nugget):
    the device stops at the reference's tile and pivot (linalg.py:43-44)."""
    locs = tb.generate_locations(120, 3)
    p = tb.MaternParams(1.0, 2.0, 4.9)
    with pytest.raises(tb.NotPositiveDefiniteError) as exc:
        tb.log_likelihood(locs, np.zeros(120), p, tb.LikelihoodConfig(nb=48))
    with pytest.raises(orc.NotPositiveDefiniteError) as ref:
        orc.log_likelihood(locs.coords, np.zeros(120), (1.0, 2.0, 4.9), 48, None)
    assert (exc.value.tile_index, exc.value.pivot_index) == (ref.value.tile_index, ref.value.pivot_index)


def test_tlr_permutation_invariance(tb):
    """test_stats.py:245-256: permuting the sites moves the TLR(1e-9)
    likelihood by at most 100 eps."""
    n, eps = 200, 1e-9
    locs = tb.generate_locations(n, 14)
    p = tb.MaternParams(1.0, 0.1, 0.5)
    z = tb.sample_measurements(locs, p, 3)
    perm = np.random.default_rng(20240817).permutation(n)
    cfg = tb.LikelihoodConfig(mode="tlr", accuracy=eps, nb=64)
    ll1 = tb.log_likelihood(locs, z, p, cfg)
    ll2 = tb.log_likelihood(tb.LocationSet(locs.coords[perm]), z[perm], p, cfg)
    assert abs(ll2 - ll1) / abs(ll1) <= 100 * eps


def test_compression_contract_1000_tiles(tb):
    """test_acceptance.py:91-119: 1000 random tiles (Gaussian, low rank plus
    noise, smooth kernel-like) x 4 thresholds: ||A - U V^T||_F <= eps ||A||_F
    and the rank is monotone in the accuracy."""
    rng = np.random.default_rng(314159)
    worst = 0.0
    for i in range(1000):
        m = int(rng.integers(16, 65))
        n = int(rng.integers(16, 65))
        kind = i % 3
        if kind == 0:
            tile = rng.standard_normal((m, n))
        elif kind == 1:
            k = int(rng.integers(1, 8))
            tile = (rng.standard_normal((m, k)) @ rng.standard_normal((k, n))
                    + 10.0 ** rng.uniform(-12, -3) * rng.standard_normal((m, n)))
        else:
            x = rng.uniform(0, 1, m)[:, None]
            y = rng.uniform(2, 3, n)[None, :]
            tile = np.exp(-np.abs(x - y) / rng.uniform(0.05, 2.0))
        norm = np.linalg.norm(tile)
        prev = 0
        for eps in EPS_GRID:
            u, v = tb.compress_tile(tile, eps)
            err = np.linalg.norm(tile - u @ v.T)
            assert err <= eps * norm, (i, eps, err / norm)
            worst = max(worst, err / (eps * norm))
            assert u.shape[1] >= prev, (i, eps)
            prev = u.shape[1]
    assert worst <= 1.0


def test_likelihood_error_monotone_in_accuracy(tb):
    """test_acceptance.py:153-167: n = 1600, dense at nb = 200 vs TLR at
    nb = 400 over the accuracy grid: the relative likelihood error decreases
    monotonically."""
    n = 1600
    p = tb.MaternParams(1.0, 0.1, 0.5)
    locs = tb.generate_locations(n, 42)
    z = tb.sample_measurements(locs, p, 43)
    ll_d = tb.log_likelihood(locs, z, p, tb.LikelihoodConfig(nb=200))
    errs = []
    for eps in EPS_GRID:
        ll_t = tb.log_likelihood(locs, z, p, tb.LikelihoodConfig(mode="tlr", accuracy=eps, nb=400))
        errs.append(abs(ll_t - ll_d) / abs(ll_d))
    for a, b in zip(errs, errs[1:]):
        assert b <= a, errs


def test_tlr_factorization_residual(tb):
    """test_linalg.py:157-165: n = 160, nb = 48, eps = 1e-9.  The reference
    bounds ||L L^T - A_tlr||_F <= 50 eps ||A_tlr||_F against its compressed
    input; the device factor is checked against the exact covariance, which
    the compression moves by at most eps ||Sigma||_F: bound 51 eps."""
    n, nb, eps = 160, 48, 1e-9
    locs = tb.generate_locations(n, 4)
    p = tb.MaternParams(1.0, 0.1, 0.5)
    h = tb.Handle(locs.coords, nb)
    try:
        h.factorize(p, eps)
        el = np.stack([h.apply_factor(col) for col in np.eye(n)], axis=1)   # L e_j
    finally:
        h.close()
    sigma = tb.matern_block(locs.coords, locs.coords, p)
    assert np.allclose(el, np.tril(el))
    assert np.linalg.norm(el @ el.T - sigma) / np.linalg.norm(sigma) <= 51 * eps


@pytest.mark.parametrize("n,nb,eps", [(120, 40, 1e-9), (150, 32, 1e-7), (200, 64, 1e-12)])
def test_tlr_against_dense(tb, n, nb, eps):
    """test_linalg.py:143-155: TLR log-det within 100 eps of dense, solve
    within 1000 eps."""
    locs = tb.generate_locations(n, 33)
    p = tb.MaternParams(1.0, 0.1, 0.5)
    h = tb.Handle(locs.coords, nb)
    rhs = np.random.default_rng(1).standard_normal(n)
    try:
        _, ld_d, _ = h.loglik(rhs, p, None)
        xd = h.solve(rhs)
        _, ld_t, _ = h.loglik(rhs, p, eps)
        xt = h.solve(rhs)
    finally:
        h.close()
    assert ld_t == pytest.approx(ld_d, rel=100 * eps)
    assert np.linalg.norm(xt - xd) / np.linalg.norm(xd) <= 1000 * eps


def test_c3p_kriging_vs_reference(tb):
    """C3p kriging (tests/golden/make_c3p_kriging_golden.py, the unmodified
    reference's predict on the C3 patch, 50 held-out sites, nb = 760):
    dense within 1e-10 relative (2-norm), TLR(1e-9) / TLR(1e-7) within
    max(1e-8, 10 acc) of the reference TLR at the same accuracy."""
    import json
    path = GOLD / "c3p_kriging.npz"
    if not path.exists():
        pytest.skip("C3p kriging golden not generated")
    g = np.load(path)
    d = json.loads((GOLD / "patches.json").read_text())["C3p"]
    full = tb.generate_locations(d["parent_n"], 0).coords
    sel = (full[:, 0] < d["edge"]) & (full[:, 1] < d["edge"])
    xy = full[sel]
    z = np.load(GOLD / "z_patches.npz")["C3p"]
    mask = np.zeros(len(xy), bool)
    mask[g["idx"]] = True
    kn, un = tb.LocationSet(xy[~mask]), tb.LocationSet(xy[mask])
    p = tb.MaternParams(*d["theta"])
    for key, mode, acc in (("dense", "dense", None), ("tlr_1e-9", "tlr", 1e-9), ("tlr_1e-7", "tlr", 1e-7)):
        pred = tb.predict(tb.PredictionProblem(kn, z[~mask], un, p, mode, acc, 760))
        ref = g[key]
        rel = np.linalg.norm(pred - ref) / np.linalg.norm(ref)
        tol = 1e-10 if acc is None else max(1e-8, 10 * acc)
        assert rel <= tol, (key, rel)
