"""2D block-cyclic multi-GPU schedule of the TLR Cholesky.

The production path lives in libtlrb200.so (tlrb.cu: `bcast_panel`,
`panel_meta`, `share_lkk`, `solve_dist`, `gather_solution`) and runs over
either NCCL (`tlrb_create_dist`, one process per GPU; `tlrb_create` with
ngpus > 1) or the in-process loopback communicator (`tlrb_create_group`, the
GPU tests run it with up to 8 ranks on one B200, tests/test_multigpu.py).
This module states the same schedule in Python so that the host logic can be
exercised on CPU with torch.distributed/gloo (tests/test_dist.py), with the
per-tile arithmetic supplied by the caller (`ops`); it never computes on the
CPU by itself and the product never routes through it.

Ownership: tile (i, j), i >= j, lives on rank (i mod P) * Q + (j mod Q); rank
r is in process row r // Q and process column r % Q, each with its own
communicator.  Per panel k (right-looking, eager recompression,
linalg.py:106-140):
  1. owner(k,k): L_kk = potrf(D_k); L_kk down process column k mod Q (the
     panel owners)
  2. panel owners: solve their tiles (i, k)
  3. one world all-reduce: NPD flag + the panel tiles' ranks (sizes)
  4. row step: in process row p, member k mod Q broadcasts the packed tiles
     (i, k), i mod P = p, to the row (they feed the owners of rows i)
  5. column step: in process column q, member p broadcasts the packed tiles
     (j, k), j mod P = p, j mod Q = q, to the column (owners of columns j)
  6. owner(j,j): D_j -= L_jk L_jk^T ;  owner(i,j): tile(i,j) updated
  7. the received panel is dropped
Forward solve: per tile row j, the owners' partial sums are reduced along
process row j mod P onto owner(j,j), which solves y_j and broadcasts it down
process column j mod Q; the full y is then assembled with one all-reduce.
log|Sigma| and ||y||^2: all-reduce.
"""
from __future__ import annotations

import math


def grid_shape(world: int) -> tuple[int, int]:
    """P x Q with P <= Q, P * Q = world, as square as possible (1x1, 1x2, 2x2, 2x4)."""
    p = int(math.isqrt(world))
    while world % p:
        p -= 1
    return p, world // p


class BlockCyclic:
    def __init__(self, P: int, Q: int):
        self.P, self.Q = P, Q
        self.world = P * Q

    def owner(self, i: int, j: int) -> int:
        return (i % self.P) * self.Q + (j % self.Q)

    def tiles_of(self, rank: int, t: int):
        return [(i, j) for i in range(t) for j in range(i + 1) if self.owner(i, j) == rank]

    def balance(self, t: int) -> list[int]:
        """Lower-triangle tile count per rank (load balance of the layout)."""
        cnt = [0] * self.world
        for i in range(t):
            for j in range(i + 1):
                cnt[self.owner(i, j)] += 1
        return cnt

    def row_of(self, rank: int) -> int:
        return rank // self.Q

    def col_of(self, rank: int) -> int:
        return rank % self.Q

    def step_messages(self, k: int, t: int) -> list[tuple[str, int, int, tuple]]:
        """Broadcasts of panel step k as (communicator, index, root member,
        tiles): L_kk down process column k mod Q, one packed panel per
        process row (root: column k mod Q), then per process column q one
        packed panel per root row p."""
        P, Q = self.P, self.Q
        msgs = [("col", k % Q, k % P, ((k, k),))]
        if Q > 1:
            for p in range(P):
                tiles = tuple((i, k) for i in range(k + 1, t) if i % P == p)
                if tiles:
                    msgs.append(("row", p, k % Q, tiles))
        if P > 1:
            for q in range(Q):
                for p in range(P):
                    tiles = tuple((j, k) for j in range(k + 1, t) if j % Q == q and j % P == p)
                    if tiles:
                        msgs.append(("col", q, p, tiles))
        return msgs


def dist_loglik(n: int, t: int, bounds, z, ops, comm, layout: BlockCyclic, acc):
    """Distributed log-likelihood with caller-supplied tile ops.

    ops: gen_diag(i) -> D; gen_lower(i, j) -> tile; potrf(D, k) -> L (or
         None when not positive definite); logdet_tile(L) -> float;
         panel_solve(L, tile) -> tile; syrk(D, tile) -> D;
         update(tile_ij, tile_ik, tile_jk) -> tile; times(tile, x) -> L_ij x;
         trsv(L, b) -> L^-1 b
    comm: .world / .row / .col, each with bcast(obj, root_member) -> obj,
          reduce_sum(vec, root_member) -> vec (valid on the root) and
          allreduce_sum(vec) -> vec; members are numbered as in libtlrb200
          (row: by process column, column: by process row).
    Returns (ll, logdet, quad), or raises RuntimeError on every rank when a
    diagonal tile is not positive definite.
    """
    import numpy as np

    P, Q = layout.P, layout.Q
    me = comm.rank
    myp, myq = layout.row_of(me), layout.col_of(me)
    D, T = {}, {}
    for i in range(t):
        if layout.owner(i, i) == me:
            D[i] = ops.gen_diag(i)
        for j in range(i):
            if layout.owner(i, j) == me:
                T[(i, j)] = ops.gen_lower(i, j)
    logdet = 0.0
    for k in range(t):
        # 1. POTRF on the owner, L_kk down process column k mod Q
        L, bad = None, 0.0
        if layout.owner(k, k) == me:
            L = ops.potrf(D[k], k)
            if L is None:
                bad = 1.0
            else:
                logdet += ops.logdet_tile(L)
                D[k] = L
        if myq == k % Q:
            L = comm.col.bcast(L, k % P)
        # 2. panel solves on the owners
        for i in range(k + 1, t):
            if layout.owner(i, k) == me and L is not None:
                T[(i, k)] = ops.panel_solve(L, T[(i, k)])
        # 3. NPD flag (+ panel sizes, implicit here) on the world
        if comm.world.allreduce_sum(np.array([bad]))[0] > 0:
            raise RuntimeError(f"not positive definite at tile {k}")
        # 4. row step: tiles (i, k), i mod P = myp, from member k mod Q
        have = {i: T[(i, k)] for i in range(k + 1, t) if layout.owner(i, k) == me}
        if Q > 1:
            pack = have if myq == k % Q else None
            pack = comm.row.bcast(pack, k % Q)
            have.update(pack)
        # 5. column step: per root row p, tiles (j, k), j mod P = p, j mod Q = myq
        if P > 1:
            for p in range(P):
                pack = ({j: have[j] for j in range(k + 1, t) if j % Q == myq and j % P == p}
                        if myp == p else None)
                have.update(comm.col.bcast(pack, p))
        # 6. updates of the owned tiles
        for j in range(k + 1, t):
            if layout.owner(j, j) == me:
                D[j] = ops.syrk(D[j], have[j])
            for i in range(j + 1, t):
                if layout.owner(i, j) == me:
                    T[(i, j)] = ops.update(T[(i, j)], have[i], have[j])
        # 7. the received panel goes out of scope here
    logdet = float(comm.world.allreduce_sum(np.array([logdet]))[0])
    # forward solve: reduce along process rows, broadcast down process columns
    y = np.array(z, dtype=float, copy=True)
    acc_vec = np.zeros(n)
    for j in range(t):
        c0, c1 = bounds[j]
        part = acc_vec[c0:c1].copy()
        if myp == j % P:
            part = comm.row.reduce_sum(part, j % Q)
        yj = ops.trsv(D[j], y[c0:c1] - part) if layout.owner(j, j) == me else None
        if myq == j % Q:
            yj = comm.col.bcast(yj, j % P)
            y[c0:c1] = yj
        for i in range(j + 1, t):
            if layout.owner(i, j) == me:
                a0, a1 = bounds[i]
                acc_vec[a0:a1] += ops.times(T[(i, j)], yj)
    # every rank assembles y from the owners of the diagonal tiles
    full = np.zeros(n)
    for j in range(t):
        if layout.owner(j, j) == me:
            c0, c1 = bounds[j]
            full[c0:c1] = y[c0:c1]
    y = comm.world.allreduce_sum(full)
    quad = float(y @ y)
    return -0.5 * (n * math.log(2 * math.pi) + logdet + quad), logdet, quad
