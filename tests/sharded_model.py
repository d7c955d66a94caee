"""Host (numpy) model of libisvd's row-sharded mode -- TEST INFRASTRUCTURE.

It restates, step by step, what isvd_engine_set_shard makes the CUDA engine
do (csrc/engine.cu, gram_svd.cu, guard.cu), with the cross-rank sums done by
a caller-supplied ``allreduce`` (torch.distributed gloo in
tests/test_sharded_model_gloo.py), so the sharding algorithm itself -- which
sums travel, what is replicated, who stores appended rows -- is checked on
CPU against the unsharded reference restatement (oracle/):

  init      G = sum_r A_r^T A_r; G = Vg diag(lam) Vg^T; B_r = A_r Vg[:, :w];
            two CholeskyQR + core-SVD passes with sum_r B_r^T B_r
  row       replicated projection on V, core SVD, V rotation; every shard
            rotates its U block; the last shard stores the new row
  column    p = sum_r U_r^T y_r (+ ||y||^2), z_r = y_r - U_r p,
            rho^2 = sum_r ||z_r||^2; replicated core; local U rotation
  rank-1    U[i, :] and A[i, j] from the owning shard (summed); replicated
  signs     per-column (max |u|, global row, sign) gathered by a sum
"""

from __future__ import annotations

import numpy as np

from oracle import core_svd_lapack


def _canon(u_blk, vt, row0, allreduce, rank, world):
    w = u_blk.shape[1]
    pk = np.zeros((world, w, 3))
    if u_blk.shape[0]:
        lead = np.argmax(np.abs(u_blk), axis=0)
        pk[rank, :, 0] = np.abs(u_blk[lead, np.arange(w)])
        pk[rank, :, 1] = row0 + lead
        pk[rank, :, 2] = np.sign(u_blk[lead, np.arange(w)])
    else:
        pk[rank, :, 0] = -1.0
    pk = allreduce(pk)
    for c in range(w):
        best = max(range(world), key=lambda t: (pk[t, c, 0], -pk[t, c, 1]))
        if pk[best, c, 2] < 0:
            u_blk[:, c] *= -1.0
            vt[c, :] *= -1.0


def _cholqr_svd(u_blk, s, v, allreduce):
    """reortho_apply with a row-sharded U (guard.cu)."""
    ru = np.linalg.cholesky(allreduce(u_blk.T @ u_blk)).T
    rv = np.linalg.cholesky(v.T @ v).T
    uk, s2, vkt = core_svd_lapack((ru * s) @ rv.T)
    return u_blk @ np.linalg.solve(ru, uk), s2, v @ np.linalg.solve(rv, vkt.T)


class ShardModel:
    def __init__(self, a_blk, k, m_global, row0, rank, world, allreduce, tol=1e-10):
        self.ar, self.rank, self.world = allreduce, rank, world
        self.row0, self.m_global, self.tol = row0, m_global, tol
        self.owner = rank == world - 1
        self.a = np.array(a_blk, dtype=np.float64)
        self.k = k
        self.sq = float(allreduce(np.array([np.sum(self.a * self.a)]))[0])
        n = self.a.shape[1]
        w = min(k, m_global, n)
        g = allreduce(self.a.T @ self.a)
        lam, vg = np.linalg.eigh(g)
        order = np.argsort(lam)[::-1]
        vg = vg[:, order[:w]]
        u, s, v = self.a @ vg, np.ones(w), vg
        for _ in range(2):
            u, s, v = _cholqr_svd(u, s, v, allreduce)
        self.u, self.s, self.vt = u, s, v.T.copy()
        _canon(self.u, self.vt, row0, allreduce, rank, world)

    def row_append(self, x):
        n = self.vt.shape[1]
        r = self.s.size
        keep = min(r + 1, self.k, self.m_global + 1, n)
        p = self.vt @ x
        z = x - self.vt.T @ p
        rho = float(np.linalg.norm(z))
        core = np.zeros((r + 1, r + 1))
        core[np.arange(r), np.arange(r)] = self.s
        core[r, :r] = p
        inj = np.zeros(n)
        if rho > self.tol:
            core[r, r] = rho
            inj = z / rho
        uk, s2, vkt = core_svd_lapack(core)
        self.u = self.u @ uk[:r, :keep]
        if self.owner:
            self.u = np.vstack([self.u, uk[r, :keep]])
            self.a = np.vstack([self.a, x])
        self.vt = vkt[:keep, :r] @ self.vt + np.outer(vkt[:keep, r], inj)
        self.s = s2[:keep].copy()
        self.sq += float(x @ x)
        self.m_global += 1
        _canon(self.u, self.vt, self.row0, self.ar, self.rank, self.world)

    def col_append(self, y):
        ml = self.u.shape[0]
        yl = y[self.row0:self.row0 + ml]
        r = self.s.size
        n = self.vt.shape[1]
        keep = min(r + 1, self.k, self.m_global, n + 1)
        pv = self.ar(np.concatenate([self.u.T @ yl, [yl @ yl]]))
        p, yy = pv[:r], pv[r]
        z = yl - self.u @ p
        rho = float(np.sqrt(self.ar(np.array([z @ z]))[0]))
        core = np.zeros((r + 1, r + 1))
        core[np.arange(r), np.arange(r)] = self.s
        core[r, :r] = p
        inj = np.zeros(ml)
        if rho > self.tol:
            core[r, r] = rho
            inj = z / rho
        uk, s2, vkt = core_svd_lapack(core)  # transpose trick: U <-> V roles
        v = self.vt.T
        v_new = np.vstack([v @ uk[:r, :keep], uk[r, :keep]])
        self.u = self.u @ vkt[:keep, :r].T + np.outer(inj, vkt[:keep, r])
        self.vt = v_new.T.copy()
        self.s = s2[:keep].copy()
        self.a = np.hstack([self.a, yl[:, None]])
        self.sq += float(yy)
        _canon(self.u, self.vt, self.row0, self.ar, self.rank, self.world)

    def rank_one_update(self, i, j, delta):
        r = self.s.size
        il = i - self.row0
        vec = np.zeros(r + 1)
        if 0 <= il < self.u.shape[0]:
            vec[:r] = self.u[il]
            vec[r] = self.a[il, j]
            self.a[il, j] += delta
        vec = self.ar(vec)
        core = np.diag(self.s) + delta * np.outer(vec[:r], self.vt[:, j])
        uk, s2, vkt = core_svd_lapack(core)
        self.u = self.u @ uk
        self.vt = vkt @ self.vt
        self.s = s2.copy()
        self.sq += 2.0 * delta * vec[r] + delta * delta
        _canon(self.u, self.vt, self.row0, self.ar, self.rank, self.world)
