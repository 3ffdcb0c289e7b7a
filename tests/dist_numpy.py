"""Numpy compute backend for the sharded schedule (paper_2208_06290_b200.distributed)
-- TEST INFRASTRUCTURE: lets the host-side schedule (partitioning, packing,
all-reduces) run on CPU with gloo.  Every kernel is the oracle's restatement
of the reference kernels (oracle/hodlr_oracle.py), applied to the rank's rows.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import hodlr_oracle as orc


@dataclass
class NpState:
    shard: object
    D: np.ndarray
    Y: np.ndarray
    V: np.ndarray
    dpiv: object = None
    K: dict = field(default_factory=dict)   # level -> (npar_global, 2r, 2r) LU stacks (global indices)
    kperm: dict = field(default_factory=dict)
    kswaps: dict = field(default_factory=dict)
    ksing: dict = field(default_factory=dict)  # level -> set of global parents flagged singular


def _col(buf, n, j0, ncols):
    """(n, ncols) column-major view of columns [j0, j0+ncols) of an n-row slab."""
    return buf.reshape(-1, n)[j0 : j0 + ncols].T


class NumpyBackend:
    def zeros(self, n):
        return np.zeros(n)

    def singular_flags(self, st):
        sh = st.shard
        L, nleaf = sh.L, 1 << sh.L
        f = np.zeros(2 * nleaf - 1)
        a = sh.row0 // sh.m
        for i in np.flatnonzero(st.dpiv.singular):
            f[a + int(i)] = 1.0
        for lv, ps in st.ksing.items():
            for p in ps:
                f[nleaf + (1 << lv) - 1 + p] = 1.0
        return f

    def raise_if_singular(self, st, flags):
        from paper_2208_06290_b200.distributed import raise_singular_from_flags

        raise_singular_from_flags(flags, st.shard.L)

    def factor_init(self, sh):
        return NpState(sh, np.array(sh.D, dtype=np.float64), np.array(sh.U, dtype=np.float64),
                       np.array(sh.V, dtype=np.float64))

    # level lv: children at lv+1 with nc rows; local parents start at global index p0
    def _k_factor(self, st, lv, tw_par, p_glob0):
        """tw_par: (npar, 2r, ncol) stacked [W|T] of the local parents (row half = child)."""
        r = st.shard.r
        npar = tw_par.shape[0]
        K = np.zeros((npar, 2 * r, 2 * r))
        K[:, :r, :r] = tw_par[:, :r, r * lv :]
        K[:, r:, r:] = tw_par[:, r:, r * lv :]
        K[:, :r, r:] = np.eye(r)
        K[:, r:, :r] = np.eye(r)
        flat = np.ascontiguousarray(K.transpose(0, 2, 1)).reshape(-1)  # column-major blocks
        stack = orc.sview(flat, 0, 4 * r * r, npar, 2 * r, 2 * r, 2 * r)
        piv = orc.lu_factor(stack)
        st.ksing.setdefault(lv, set()).update(p_glob0 + int(i) for i in np.flatnonzero(piv.singular))
        for i in range(npar):
            st.K.setdefault(lv, {})[p_glob0 + i] = np.array(stack[i])
            st.kperm.setdefault(lv, {})[p_glob0 + i] = piv.perm[i].copy()
            st.kswaps.setdefault(lv, {})[p_glob0 + i] = piv.swaps[i].copy()
        return stack, piv.perm

    def factor_local(self, st, p):
        sh = st.shard
        n, m, r, L, nl = sh.n_loc, sh.m, sh.r, sh.L, sh.n_loc // sh.m
        dst = orc.sview(st.D, 0, m * m, nl, m, m, m)
        st.dpiv = orc.lu_factor(dst)
        if L == 0:
            return np.zeros(0)
        yst = orc.sview(st.Y, 0, m, nl, m, r * L, n)
        orc.lu_solve(dst, st.dpiv.perm, yst)
        for lv in range(L - 1, p - 1, -1):
            nc = sh.n >> (lv + 1)
            nch = n // nc
            npar = nch // 2
            ncol = r * (lv + 1)
            tw = np.stack([_col(st.V, n, lv * r, r)[c * nc : (c + 1) * nc].T @ _col(st.Y, n, 0, ncol)[c * nc : (c + 1) * nc]
                           for c in range(nch)])
            tw_par = tw.reshape(npar, 2 * r, ncol)
            stack, perm = self._k_factor(st, lv, tw_par, sh.row0 // (2 * nc))
            if lv == 0:
                break
            wc = r * lv
            for q in range(npar):
                W = tw_par[q, :, :wc].copy()
                orc.lu_solve(stack[q : q + 1], perm[q : q + 1], W[None])
                for h in range(2):
                    c = 2 * q + h
                    rows = slice(c * nc, (c + 1) * nc)
                    Yc = _col(st.Y, n, lv * r, r)[rows]
                    _col(st.Y, n, 0, wc)[rows] -= Yc @ W[h * r : (h + 1) * r]
        if p == 0:
            return np.zeros(0)
        # [W|T] of this rank's level-p node (children of level p-1): r x r p
        return (_col(st.V, n, (p - 1) * r, r).T @ _col(st.Y, n, 0, r * p)).T.reshape(-1)

    def factor_top(self, st, lv, tw_all):
        sh = st.shard
        n, r = sh.n_loc, sh.r
        ncol = r * (lv + 1)
        npar = 1 << lv
        tw_par = tw_all.reshape(npar, ncol, 2 * r).transpose(0, 2, 1)
        stack, perm = self._k_factor(st, lv, tw_par, 0)
        if lv == 0:
            return np.zeros(0)
        nc = sh.n >> (lv + 1)
        pidx, half = sh.row0 // (2 * nc), (sh.row0 // nc) & 1
        wc = r * lv
        W = tw_par[pidx, :, :wc].copy()
        orc.lu_solve(stack[pidx : pidx + 1], perm[pidx : pidx + 1], W[None])
        _col(st.Y, n, 0, wc)[:] -= _col(st.Y, n, lv * r, r) @ W[half * r : (half + 1) * r]
        return (_col(st.V, n, (lv - 1) * r, r).T @ _col(st.Y, n, 0, wc)).T.reshape(-1)

    def solve_local(self, st, x, nrhs, p):
        sh = st.shard
        n, m, r, L, nl = sh.n_loc, sh.m, sh.r, sh.L, sh.n_loc // sh.m
        X = x.reshape(nrhs, n).T  # view, column-major
        dst = orc.sview(st.D, 0, m * m, nl, m, m, m)
        xs = orc.sview(x, 0, m, nl, m, nrhs, n)
        orc.lu_solve(dst, st.dpiv.perm, xs)
        for lv in range(L - 1, p - 1, -1):
            nc = sh.n >> (lv + 1)
            npar = n // nc // 2
            p0 = sh.row0 // (2 * nc)
            for q in range(npar):
                w = np.vstack([_col(st.V, n, lv * r, r)[(2 * q + h) * nc : (2 * q + h + 1) * nc].T
                               @ X[(2 * q + h) * nc : (2 * q + h + 1) * nc] for h in range(2)])
                orc.lu_solve(st.K[lv][p0 + q][None], st.kperm[lv][p0 + q][None], w[None])
                for h in range(2):
                    rows = slice((2 * q + h) * nc, (2 * q + h + 1) * nc)
                    X[rows] -= _col(st.Y, n, lv * r, r)[rows] @ w[h * r : (h + 1) * r]
        if p == 0:
            return np.zeros(0)
        return (_col(st.V, n, (p - 1) * r, r).T @ X).T.reshape(-1)

    def solve_top(self, st, lv, w_all, x, nrhs):
        sh = st.shard
        n, r = sh.n_loc, sh.r
        X = x.reshape(nrhs, n).T
        nc = sh.n >> (lv + 1)
        pidx, half = sh.row0 // (2 * nc), (sh.row0 // nc) & 1
        w = w_all.reshape(1 << lv, nrhs, 2 * r)[pidx].T.copy()
        orc.lu_solve(st.K[lv][pidx][None], st.kperm[lv][pidx][None], w[None])
        X -= _col(st.Y, n, lv * r, r) @ w[half * r : (half + 1) * r]
        if lv == 0:
            return np.zeros(0)
        return (_col(st.V, n, (lv - 1) * r, r).T @ X).T.reshape(-1)
