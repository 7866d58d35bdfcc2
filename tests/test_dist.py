"""Multi-process (gloo, CPU) tests of the 2D block-cyclic schedule
(paper_1804_09137_b200/dist.py, the same schedule libtlrb200's
tlrb_create_dist runs with NCCL).  Tile arithmetic: the CPU oracle."""
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401
from oracle import tlr_oracle as orc
from paper_1804_09137_b200.dist import BlockCyclic, dist_loglik, grid_shape

N, NB, THETA = 600, 100, (1.0, 0.1, 0.5)


class OracleOps:
    def __init__(self, xy, acc):
        self.xy, self.acc = xy, acc
        self.b = orc.tile_bounds(xy.shape[0], NB)

    def _blk(self, i, j):
        (a, b), (c, d) = self.b[i], self.b[j]
        return orc.matern_block(self.xy[a:b], self.xy[c:d], THETA)

    def gen_diag(self, i):
        return self._blk(i, i)

    def gen_lower(self, i, j):
        blk = self._blk(i, j)
        return orc.compress_tile(blk, self.acc) if self.acc else blk

    def potrf(self, D, k):
        return orc.potrf_tile(D, k)

    def logdet_tile(self, L):
        return 2.0 * float(np.sum(np.log(np.diag(L))))

    def panel_solve(self, L, tile):
        if self.acc:
            u, v = tile
            return (u, sla.solve_triangular(L, v, lower=True)) if u.shape[1] else tile
        return sla.solve_triangular(L, tile.T, lower=True).T

    def syrk(self, D, tile):
        if self.acc:
            u, v = tile
            return D - (u @ (v.T @ v)) @ u.T if u.shape[1] else D
        return D - tile @ tile.T

    def update(self, tij, tik, tjk):
        if self.acc:
            (u0, v0), (ui, vi), (uj, vj) = tij, tik, tjk
            if ui.shape[1] == 0 or uj.shape[1] == 0:
                return tij
            return orc.recompress(u0, v0, -(ui @ (vi.T @ vj)), uj, self.acc)
        return tij - tik @ tjk.T

    def times(self, tile, x):
        if self.acc:
            u, v = tile
            return u @ (v.T @ x) if u.shape[1] else np.zeros(u.shape[0])
        return tile @ x

    def trsv(self, L, b):
        return sla.solve_triangular(L, b, lower=True)


class GlooGroup:
    """One communicator (world, a process row or a process column) over a
    gloo group; members are numbered by their position in `ranks`."""

    def __init__(self, ranks, group):
        self.ranks, self.group = list(ranks), group

    def bcast(self, obj, root):
        box = [obj]
        dist.broadcast_object_list(box, src=self.ranks[root], group=self.group)
        return box[0]

    def reduce_sum(self, vec, root):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64))
        dist.reduce(t, dst=self.ranks[root], op=dist.ReduceOp.SUM, group=self.group)
        return t.numpy()

    def allreduce_sum(self, vec):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64))
        dist.all_reduce(t, group=self.group)
        return t.numpy()


class GlooComm:
    """World + process-row + process-column communicators of a P x Q grid
    (every rank creates every group, in the same order)."""

    def __init__(self, P, Q):
        self.rank = dist.get_rank()
        world = P * Q
        self.world = GlooGroup(range(world), None)
        rows = [[p * Q + q for q in range(Q)] for p in range(P)]
        cols = [[p * Q + q for p in range(P)] for q in range(Q)]
        rg = [dist.new_group(r) for r in rows]
        cg = [dist.new_group(c) for c in cols]
        p, q = self.rank // Q, self.rank % Q
        self.row = GlooGroup(rows[p], rg[p])
        self.col = GlooGroup(cols[q], cg[q])


def _worker(rank, world, port, acc, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    xy = orc.generate_locations(N, 5)
    z = np.random.default_rng(3).standard_normal(N)
    P, Q = grid_shape(world)
    ll, ld, q = dist_loglik(N, -(-N // NB), orc.tile_bounds(N, NB), z, OracleOps(xy, acc), GlooComm(P, Q),
                            BlockCyclic(P, Q), acc)
    out[rank] = (ll, ld, q)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("acc", [None, 1e-7])
def test_block_cyclic_matches_single_process(world, acc):
    port = 29500 + world * 7 + (0 if acc is None else 3)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, acc, out), nprocs=world, join=True)
        res = dict(out)
    xy = orc.generate_locations(N, 5)
    z = np.random.default_rng(3).standard_normal(N)
    want = orc.log_likelihood(xy, z, THETA, NB, acc)
    for r in range(world):
        ll, ld, q = res[r]
        assert ll == pytest.approx(want[0], rel=1e-12)
        assert ld == pytest.approx(want[1], rel=1e-12)
        assert q == pytest.approx(want[2], rel=1e-12)


def test_layout_balance_and_messages():
    lay = BlockCyclic(*grid_shape(8))
    assert (lay.P, lay.Q) == (2, 4)
    cnt = lay.balance(83)            # C3 tile grid
    assert max(cnt) / min(cnt) < 1.3   # lower-triangle block-cyclic: diagonal ranks carry more
    msgs = lay.step_messages(5, 83)
    assert msgs[0] == ("col", 5 % 4, 5 % 2, ((5, 5),))
    # every panel tile reaches the owners of its tile row (row step) and of
    # its tile column (column step)
    row_tiles = {tl for c, _, _, ts in msgs if c == "row" for tl in ts}
    assert row_tiles == {(i, 5) for i in range(6, 83)}
    col_msgs = [(q, p, ts) for c, q, p, ts in msgs[1:] if c == "col"]
    assert {tl for _, _, ts in col_msgs for tl in ts} == {(j, 5) for j in range(6, 83)}
    for q, p, ts in col_msgs:
        assert all(j % 4 == q and j % 2 == p for j, _ in ts)
    # one packed message per process row and per non-empty (column, root row):
    # with P = 2 | Q = 4, j mod 4 fixes j mod 2, so 4 column messages
    assert len(msgs) == 1 + 2 + 4
    seen = set()
    for i in range(20):
        for j in range(i + 1):
            seen.add(lay.owner(i, j))
    assert seen == set(range(8))
