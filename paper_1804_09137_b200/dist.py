"""2D block-cyclic multi-GPU schedule of the TLR Cholesky.

The production path lives in libtlrb200.so (`tlrb_create_dist`: NCCL
broadcasts / reduces on the handle's stream, one process per GPU).  This
module holds the same schedule in Python so that it can be exercised on CPU
with torch.distributed/gloo (tests/test_dist.py), with the per-tile
arithmetic supplied by the caller (`ops`); it never computes on the CPU by
itself and the product never routes through it.

Ownership: tile (i, j), i >= j, lives on rank (i mod P) * Q + (j mod Q).
Per panel k (right-looking, eager recompression, linalg.py:106-140):
  1. owner(k,k): L_kk = potrf(D_k)           -> broadcast L_kk to all
  2. owners of (i,k): panel solve            -> broadcast tile (i,k) to all
  3. owner(j,j): D_j -= L_jk L_jk^T ;  owner(i,j): tile(i,j) updated/recompressed
  4. tile ranks all-reduced (owners contribute)
Forward solve: per column j, reduce the owners' partial sums onto owner(j,j),
which solves y_j and broadcasts it.  log|Sigma| and ||y||^2: all-reduce.
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

    def step_messages(self, k: int, t: int) -> list[tuple[str, tuple[int, int], int]]:
        """Broadcasts of panel step k: ("L", (k,k), root) then ("panel", (i,k), root)."""
        msgs = [("L", (k, k), self.owner(k, k))]
        msgs += [("panel", (i, k), self.owner(i, k)) for i in range(k + 1, t)]
        return msgs


def dist_loglik(n: int, t: int, bounds, z, ops, comm, layout: BlockCyclic, acc):
    """Distributed log-likelihood with caller-supplied tile ops.

    ops: gen_diag(i) -> D; gen_lower(i, j) -> tile; potrf(D, k) -> L;
         logdet_tile(L) -> float; panel_solve(L, tile) -> tile;
         syrk(D, tile) -> D; update(tile_ij, tile_ik, tile_jk) -> tile;
         times(tile, x) -> L_ij x (vector); trsv(L, b) -> L^-1 b
    comm: rank, bcast(obj, root) -> obj, reduce_sum(vec, root) -> vec (valid on root),
          allreduce_sum(float) -> float
    """
    r = comm.rank
    D, T = {}, {}
    for i in range(t):
        if layout.owner(i, i) == r:
            D[i] = ops.gen_diag(i)
        for j in range(i):
            if layout.owner(i, j) == r:
                T[(i, j)] = ops.gen_lower(i, j)
    logdet = 0.0
    Lk = {}
    for k in range(t):
        root = layout.owner(k, k)
        L = ops.potrf(D[k], k) if root == r else None
        if root == r:
            logdet += ops.logdet_tile(L)
            D[k] = L
        L = comm.bcast(L, root)
        Lk[k] = L
        panel = {}
        for i in range(k + 1, t):
            own = layout.owner(i, k)
            tile = ops.panel_solve(L, T[(i, k)]) if own == r else None
            if own == r:
                T[(i, k)] = tile
            panel[i] = comm.bcast(tile, own)
        for j in range(k + 1, t):
            if layout.owner(j, j) == r:
                D[j] = ops.syrk(D[j], panel[j])
            for i in range(j + 1, t):
                if layout.owner(i, j) == r:
                    T[(i, j)] = ops.update(T[(i, j)], panel[i], panel[j])
    logdet = comm.allreduce_sum(logdet)
    # forward solve (column-oriented, reduce + broadcast per tile column)
    import numpy as np
    y = np.array(z, dtype=float, copy=True)
    acc_vec = np.zeros(n)
    for j in range(t):
        c0, c1 = bounds[j]
        root = layout.owner(j, j)
        part = comm.reduce_sum(acc_vec[c0:c1].copy(), root)
        yj = ops.trsv(Lk[j], y[c0:c1] - part) if root == r else None
        yj = comm.bcast(yj, root)
        y[c0:c1] = yj
        for i in range(j + 1, t):
            if layout.owner(i, j) == r:
                a0, a1 = bounds[i]
                acc_vec[a0:a1] += ops.times(T[(i, j)], yj)
    quad = float(y @ y)
    return -0.5 * (n * math.log(2 * math.pi) + logdet + quad), logdet, quad
