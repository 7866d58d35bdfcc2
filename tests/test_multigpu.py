"""The product's 2D block-cyclic multi-GPU path, executed on
one B200: `world` logical ranks in one process (tlrb_create_group with the
loopback communicator — host rendezvous + stream-ordered device copies, no
kernel waits on another rank), each rank owning only its tiles plus one
received panel.  The same libtlrb200 code as the NCCL path runs (packed row /
column panel broadcasts, the per-step panel metadata all-reduce, row / column
reduces and broadcasts in the solves); only the Comm backend differs.

Parity: world W equals world 1 (ll within 1e-12 relative, identical rank
maps), and both match the reference goldens (linalg.py:106-140 per-step
dependencies are the same on every grid)."""
import numpy as np
import pytest

from conftest import GOLD

pytestmark = pytest.mark.gpu

GRIDS = [(2, 1, 2), (4, 2, 2), (8, 2, 4)]   # world, P, Q


def _c1(gold, tb):
    e = gold["loglik"]["C1"]
    return e, tb.generate_locations(e["n"], e["loc_seed"]).coords, gold["z"]["C1"]


def _c2(gold, tb):
    e = gold["loglik"]["C2"]
    return e, tb.generate_locations(e["n"], e["loc_seed"]).coords, gold["z"]["C2"]


def _c3p(tb):
    import json
    d = json.loads((GOLD / "patches.json").read_text())
    e = d["C3p"]
    full = tb.generate_locations(e["parent_n"], 0).coords
    sel = (full[:, 0] < e["edge"]) & (full[:, 1] < e["edge"])
    return e, full[sel], np.load(GOLD / "z_patches.npz")["C3p"]


def _compare(tb, xy, nb, z, p, accs, world, P, Q, max_rank=0, ref=None):
    single = tb.Handle(xy, nb, max_rank)
    group = tb.api.group_handle(xy, nb, world, max_rank, P=P, Q=Q)
    assert group.world == world
    try:
        for acc in accs:
            a = single.loglik(z, p, acc)
            rm1 = single.rank_map()
            b = group.loglik(z, p, acc)
            rmw = group.rank_map()
            # ll to 1e-12; log-det / quadratic form to 1e-11 (the distributed
            # solve and reductions sum in another order)
            assert abs(b[0] - a[0]) <= 1e-12 * abs(a[0]), (world, acc, b, a)
            np.testing.assert_allclose(b[1:], a[1:], rtol=1e-11, atol=0, err_msg=f"world {world} acc {acc}")
            np.testing.assert_array_equal(rmw, rm1)
            if ref is not None:
                key = "dense" if acc is None else f"tlr:{acc:g}"
                r = ref[key]["ll"]
                tol = 1e-10 if acc is None else max(1e-8, 10 * acc)
                assert abs(b[0] - r) <= tol * abs(r), (world, key, b[0], r)
    finally:
        group.close()
        single.close()


@pytest.mark.parametrize("world,P,Q", GRIDS)
def test_group_c1_equals_world1(tb, gold, world, P, Q):
    e, xy, z = _c1(gold, tb)
    _compare(tb, xy, e["nb"], z, tb.MaternParams(*e["theta"]), (None, 1e-9, 1e-7), world, P, Q,
             ref=e["modes"])


@pytest.mark.parametrize("world,P,Q", GRIDS)
def test_group_c2_equals_world1(tb, gold, world, P, Q):
    e, xy, z = _c2(gold, tb)
    _compare(tb, xy, e["nb"], z, tb.MaternParams(*e["theta"]), (None, 1e-9), world, P, Q, ref=e["modes"])


@pytest.mark.parametrize("world,P,Q", GRIDS)
def test_group_c3p_equals_world1(tb, world, P, Q):
    """nb = 760 with the C3 storage cap (380): dense (A13) panel tiles travel
    in the packed panels beside low-rank ones."""
    e, xy, z = _c3p(tb)
    _compare(tb, xy, e["nb"], z, tb.MaternParams(*e["theta"]), (1e-7,), world, P, Q, max_rank=200,
             ref=None)


@pytest.mark.parametrize("world,P,Q", [(4, 2, 2), (3, 1, 3), (6, 2, 3)])
def test_group_solves_predict_sampling(tb, gold, world, P, Q):
    """Distributed forward / backward solves (row / column reduces and
    broadcasts), z = L w and kriging through a group handle equal world 1."""
    e, xy, z = _c1(gold, tb)
    p = tb.MaternParams(*e["theta"])
    single = tb.Handle(xy, e["nb"])
    group = tb.api.group_handle(xy, e["nb"], world, P=P, Q=Q)
    x = np.random.default_rng(0).standard_normal(e["n"])
    unk = np.random.default_rng(5).uniform(0, 1, (7, 2))
    try:
        for acc in (None, 1e-9):
            single.factorize(p, acc)
            group.factorize(p, acc)
            np.testing.assert_allclose(group.solve(x), single.solve(x), rtol=1e-10, atol=1e-10)
            # y = L x: the distributed sum adds the owners' tile products in
            # another order (all-reduce), so agreement is to roundoff
            np.testing.assert_allclose(group.apply_factor(x), single.apply_factor(x), rtol=1e-10, atol=1e-11)
            np.testing.assert_allclose(group.predict(z, unk, p, acc), single.predict(z, unk, p, acc),
                                       rtol=1e-10, atol=1e-12)
    finally:
        group.close()
        single.close()


@pytest.mark.parametrize("acc", [None, 1e-9])
def test_group_npd_same_tile_and_pivot(tb, acc):
    """A non-positive-definite covariance (test_linalg.py:121-127: smooth
    long-range kernel, no nugget) stops every rank at the same panel with the
    same (tile, pivot) as one GPU (linalg.py:36-45); the group handle stays
    usable afterwards."""
    xy = tb.generate_locations(120, 3).coords
    p = tb.MaternParams(1.0, 2.0, 4.9)
    single = tb.Handle(xy, 48)
    group = tb.api.group_handle(xy, 48, 3, P=1, Q=3)
    try:
        with pytest.raises(tb.NotPositiveDefiniteError) as e1:
            single.loglik(np.zeros(120), p, acc)
        with pytest.raises(tb.NotPositiveDefiniteError) as e2:
            group.loglik(np.zeros(120), p, acc)
        assert (e2.value.tile_index, e2.value.pivot_index) == (e1.value.tile_index, e1.value.pivot_index)
        ok = tb.MaternParams(1.0, 0.1, 0.5)
        np.testing.assert_allclose(group.loglik(np.ones(120), ok, acc), single.loglik(np.ones(120), ok, acc),
                                   rtol=1e-12)
    finally:
        group.close()
        single.close()


def test_group_memory_scales(tb, gold):
    """Each rank stores only its own tiles (arena) plus one received panel:
    the largest per-rank factor arena at world 4 is well below world 1's."""
    e, xy, z = _c2(gold, tb)
    p = tb.MaternParams(*e["theta"])
    single = tb.Handle(xy, e["nb"])
    group = tb.api.group_handle(xy, e["nb"], 4)
    try:
        single.loglik(z, p, 1e-9)
        group.loglik(z, p, 1e-9)
        a1 = single.last_stats["arena_peak_bytes"]
        per = [group.member_stats(r)["arena_peak_bytes"] for r in range(4)]
        assert max(per) <= 0.45 * a1, (a1, per)
        assert group.last_stats["panel_peak_bytes"] > 0
    finally:
        group.close()
        single.close()


def test_ngpus_single_process_api(tb, gold):
    """LikelihoodConfig(ngpus=G) from one process: with one visible GPU the
    request for two devices is refused as an invalid argument (no silent
    single-GPU fallback)."""
    import torch
    e, xy, z = _c1(gold, tb)
    cfg = tb.LikelihoodConfig(mode="tlr", accuracy=1e-9, nb=e["nb"], ngpus=2)
    locs = tb.LocationSet(xy)
    if torch.cuda.device_count() >= 2:
        ll = tb.log_likelihood(locs, z, tb.MaternParams(*e["theta"]), cfg)
        r = e["modes"]["tlr:1e-09"]["ll"]
        assert abs(ll - r) <= 1e-8 * abs(r)
    else:
        with pytest.raises(ValueError):
            tb.log_likelihood(locs, z, tb.MaternParams(*e["theta"]), cfg)
