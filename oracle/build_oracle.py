"""CPU ORACLE for HODLR assembly -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module, as the checker of the device builder
(``paper_2208_06290_b200.construct`` / ``hodlr_build_*``).  It restates, in
numpy and without copying code:

* ``contour_default`` and the Laplace double-layer entry oracle with log
  completion                                    problems.py:133-217
* adaptive cross approximation with rook pivoting, real fp64, tol = 0 and a
  rank cap (the path ``compress(rows, cols, CompressionConfig(tol=0,
  max_rank=r, method="aca_rook_pivot"))`` takes)  compress.py:87-170, 173-200
* SPEC assemble: exact leaf blocks, one compressed block per orientation of
  every sibling pair, A(I_a, I_b) = U_a V_b^T

Parity pin: ``tests/golden/make_build_golden.py`` assembles the same operators
by calling the reference's own ``hodlr.compress.compress`` and
``hodlr.problems.laplace_dl_oracle`` (imported read-only from
/root/reference) block by block and asserts this restatement reproduces D, U
and V BIT-FOR-BIT; those outputs are committed as ``tests/golden/build_*.npz``.
"""

from __future__ import annotations

import math

import numpy as np

ROOK_SWEEPS = 4  # compress.py _ROOK_SWEEPS


def contour(n: int, amplitude: float = 0.3, lobes: int = 5):
    """Nodes, exterior normals, curvature and trapezoid weights of the star
    contour r(t) = 1 + amplitude cos(lobes t) (problems.py:133-156)."""
    t = 2.0 * np.pi * np.arange(n) / n
    rr = 1.0 + amplitude * np.cos(lobes * t)
    d1 = -amplitude * lobes * np.sin(lobes * t)
    d2 = -amplitude * lobes * lobes * np.cos(lobes * t)
    c, s = np.cos(t), np.sin(t)
    tx, ty = d1 * c - rr * s, d1 * s + rr * c
    sp = np.hypot(tx, ty)
    xy = np.stack([rr * c, rr * s], axis=1)
    nrm = np.stack([ty / sp, -tx / sp], axis=1)
    kappa = (rr * rr + 2.0 * d1 * d1 - rr * d2) / sp**3
    return xy, nrm, kappa, sp * (2.0 * np.pi / n)


class LaplaceDL:
    """A_ij = (d(x_i, y_j) + logterm_i) w_j + delta_ij / 2 (problems.py:158-217)."""

    def __init__(self, n: int, amplitude: float = 0.3, lobes: int = 5, z=(0.0, 0.0)):
        self.xy, self.nrm, kappa, self.w = contour(n, amplitude, lobes)
        dz = self.xy - np.asarray(z, dtype=np.float64)
        self.logt = -np.log(np.hypot(dz[:, 0], dz[:, 1])) / (2.0 * np.pi)
        self.diag = -kappa / (4.0 * np.pi)

    def __call__(self, i, j):
        i, j = np.asarray(i), np.asarray(j)
        eq = i == j
        d = self.xy[i] - self.xy[j]
        r2 = np.sum(d * d, axis=-1)
        num = np.sum(self.nrm[j] * d, axis=-1)
        k = np.where(eq, self.diag[np.broadcast_to(i, r2.shape)], num / (2.0 * np.pi * np.where(eq, 1.0, r2)))
        return (k + self.logt[i]) * self.w[j] + 0.5 * eq


class Gaussian:
    """exp(-|p_i - p_j|^2 / h^2) + lam delta_ij on (dim, n) points (BASELINE
    cfg1 / cfg3 operators; not in the reference package, so parity for this
    oracle is against this restatement only)."""

    def __init__(self, pts, h: float = 0.1, lam: float = 1.0):
        self.P = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).T)  # (n, dim)
        self.h2 = h * h
        self.lam = lam

    def __call__(self, i, j):
        i, j = np.asarray(i), np.asarray(j)
        d = self.P[i] - self.P[j]
        return np.exp(-(np.sum(d * d, axis=-1) / self.h2)) + self.lam * (i == j)


class Dense:
    def __init__(self, A):
        self.A = np.asarray(A, dtype=np.float64)

    def __call__(self, i, j):
        return self.A[i, j]


def aca_rook(entry, r0: int, c0: int, nr: int, nc: int, kmax: int):
    """Crosses (u, w) of A(r0:r0+nr, c0:c0+nc) ~ u w^T, at most kmax of them
    (compress.py:87-170 with tol = 0, rook pivoting, real data)."""
    rows, cols = np.arange(r0, r0 + nr), np.arange(c0, c0 + nc)
    us, ws = [], []
    ur, uc = np.zeros(nr, dtype=bool), np.zeros(nc, dtype=bool)

    def res_row(i):
        v = np.asarray(entry(rows[i], cols), dtype=np.float64)
        for u, w in zip(us, ws):
            v = v - u[i] * w
        return v

    def res_col(j):
        v = np.asarray(entry(rows, cols[j]), dtype=np.float64)
        for u, w in zip(us, ws):
            v = v - w[j] * u
        return v

    def masked(v, used):
        return np.where(used, 0.0, np.abs(v))

    prop = None
    while len(us) < min(nr, nc, kmax):
        i, row = None, None
        if prop is not None and not ur[prop]:
            v = res_row(prop)
            if masked(v, uc).max() > 0.0:
                i, row = prop, v
        if row is None:
            for cand in np.flatnonzero(~ur):
                v = res_row(cand)
                if masked(v, uc).max() > 0.0:
                    i, row = int(cand), v
                    break
                ur[cand] = True
        if row is None:
            break
        j = int(masked(row, uc).argmax())
        col = res_col(j)
        for _ in range(ROOK_SWEEPS):
            cm = masked(col, ur)
            i2 = int(cm.argmax())
            if cm[i2] <= abs(row[j]):
                break
            i, row = i2, res_row(i2)
            j2 = int(masked(row, uc).argmax())
            if j2 == j:
                break
            j, col = j2, res_col(j2)
        piv = row[j]
        if piv == 0:
            ur[i] = True
            continue
        us.append(col / piv)
        ws.append(row)
        ur[i] = uc[j] = True
        cm = masked(col, ur)
        prop = int(cm.argmax()) if cm.max() > 0.0 else None
    return us, ws


def assemble(entry, n: int, m: int, r: int):
    """Flat D (leaf a at a m^2, column-major), U and V (N x rL, ld N) of the
    rank-r HODLR approximation of the oracle."""
    L = int(round(math.log2(n // m)))
    D = np.empty((1 << L) * m * m)
    for a in range(1 << L):
        idx = np.arange(a * m, (a + 1) * m)
        D[a * m * m : (a + 1) * m * m] = np.asarray(entry(idx[:, None], idx[None, :]), dtype=np.float64).ravel(order="F")
    U = np.zeros(n * r * L)
    V = np.zeros(n * r * L)
    for lv in range(1, L + 1):
        nl = n >> lv
        for p in range(1 << (lv - 1)):
            for o in range(2):
                ra, cb = (2 * p + o) * nl, (2 * p + 1 - o) * nl
                us, ws = aca_rook(entry, ra, cb, nl, nl, r)
                for l, (u, w) in enumerate(zip(us, ws)):
                    c = ((lv - 1) * r + l) * n
                    U[c + ra : c + ra + nl] = u
                    V[c + cb : c + cb + nl] = w
    return D, U, V
