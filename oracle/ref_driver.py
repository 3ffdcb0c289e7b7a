"""Alg. 3/4 driven through the REFERENCE's own batched kernels -- TEST / BASELINE
INFRASTRUCTURE ONLY (tests/, bench.py --impl reference / cpu_baseline).

The reference package implements the batched kernel layer
(pkg/src/hodlr/backend.py) but not factorize/solve, so this
module is the SPEC recipe (SURVEY.md
Appendix B) issuing only the reference's public kernels:
``BlockRef`` (backend.py:48), ``batched_gemm`` (:320),
``batched_lu_factor_inplace`` (:481), ``batched_lu_solve_inplace`` (:570),
with its executors (:175-232).  ``scratch`` is always None (the reference's
shared-scratch race).

The reference is imported read-only from ``baseline/_ref`` (pip-installed
copy, travels to the GPU box) or ``/root/reference/pkg/src``.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

_ROOT = Path(__file__).resolve().parent.parent
for cand in (_ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "hodlr" / "backend.py").exists():
        if str(cand) not in sys.path:
            sys.path.insert(0, str(cand))
        break

try:  # noqa: E402
    from hodlr.backend import (  # type: ignore
        SERIAL,
        BlockRef,
        ThreadedExecutor,
        batched_gemm,
        batched_lu_factor_inplace,
        batched_lu_solve_inplace,
    )

    AVAILABLE = True
except Exception:  # pragma: no cover - reference not present
    AVAILABLE = False


def executor(threads: int):
    return SERIAL if threads <= 1 else ThreadedExecutor(threads)


def _level_ranks(r, L, ranks):
    rk = [r] * L if ranks is None else [int(x) for x in ranks]
    c = [0]
    for k in rk:
        c.append(c[-1] + k)
    return rk, c  # rank of level l' = rk[l'-1], its first column c[l'-1]; c[L] = total


def ref_factorize(D, Y, V, n, m, r, L, ex=None, ranks=None):
    """Appendix-B recipe through the reference kernels; returns pivots + K.
    ``ranks``: per-level ranks (level l' at ranks[l'-1], panels padded per level)."""
    ex = ex or SERIAL
    rk, cc = _level_ranks(r, L, ranks)
    nleaf = 1 << L
    drefs = [BlockRef(D, a * m * m, m, m, m) for a in range(nleaf)]
    dpiv, _ = batched_lu_factor_inplace(drefs, executor=ex)
    assert not dpiv.singular
    if L > 0 and cc[L]:
        batched_lu_solve_inplace(drefs, dpiv, [BlockRef(Y, a * m, m, cc[L], n) for a in range(nleaf)], executor=ex)
    Ks, kpivs = [None] * L, [None] * L
    for lv in range(L - 1, -1, -1):
        nch, npar, nc = 1 << (lv + 1), 1 << lv, n >> (lv + 1)
        r, c1 = rk[lv], cc[lv]  # rank / first column of level lv + 1
        ncol = c1 + r
        if r == 0:
            Ks[lv], kpivs[lv] = np.zeros(0), None
            continue
        tw = np.zeros(nch * r * ncol)
        batched_gemm(
            [
                (
                    BlockRef(V, c1 * n + c * nc, nc, r, n),
                    BlockRef(Y, c * nc, nc, ncol, n),
                    BlockRef(tw, c * r * ncol, r, ncol, r),
                )
                for c in range(nch)
            ],
            transpose_a="conj_transpose",
            executor=ex,
        )
        K = np.zeros(npar * 4 * r * r)
        for p in range(npar):
            kb = BlockRef(K, p * 4 * r * r, 2 * r, 2 * r, 2 * r).view()
            kb[:r, :r] = BlockRef(tw, 2 * p * r * ncol + c1 * r, r, r, r).view()
            kb[r:, r:] = BlockRef(tw, (2 * p + 1) * r * ncol + c1 * r, r, r, r).view()
            kb[:r, r:] = np.eye(r)
            kb[r:, :r] = np.eye(r)
        krefs = [BlockRef(K, p * 4 * r * r, 2 * r, 2 * r, 2 * r) for p in range(npar)]
        kpiv, _ = batched_lu_factor_inplace(krefs, executor=ex)
        assert not kpiv.singular
        Ks[lv], kpivs[lv] = K, kpiv
        if lv == 0 or c1 == 0:
            continue
        wc = c1
        W = np.zeros(npar * 2 * r * wc)
        for c in range(nch):
            BlockRef(W, (c // 2) * 2 * r * wc + (c % 2) * r, r, wc, 2 * r).view()[...] = BlockRef(
                tw, c * r * ncol, r, wc, r
            ).view()
        batched_lu_solve_inplace(krefs, kpiv, [BlockRef(W, p * 2 * r * wc, 2 * r, wc, 2 * r) for p in range(npar)], executor=ex)
        batched_gemm(
            [
                (
                    BlockRef(Y, c1 * n + c * nc, nc, r, n),
                    BlockRef(W, (c // 2) * 2 * r * wc + (c % 2) * r, r, wc, 2 * r),
                    BlockRef(Y, c * nc, nc, wc, n),
                )
                for c in range(nch)
            ],
            alpha=-1.0,
            beta=1.0,
            executor=ex,
        )
    return dpiv, Ks, kpivs


def ref_solve(D, dpiv, Y, V, Ks, kpivs, b, n, m, r, L, ex=None, ranks=None):
    ex = ex or SERIAL
    rk, cc = _level_ranks(r, L, ranks)
    nrhs = b.shape[1]
    x = np.asfortranarray(b).ravel(order="F").copy()
    nleaf = 1 << L
    drefs = [BlockRef(D, a * m * m, m, m, m) for a in range(nleaf)]
    batched_lu_solve_inplace(drefs, dpiv, [BlockRef(x, a * m, m, nrhs, n) for a in range(nleaf)], executor=ex)
    for lv in range(L - 1, -1, -1):
        nch, npar, nc = 1 << (lv + 1), 1 << lv, n >> (lv + 1)
        r, c1 = rk[lv], cc[lv]
        if r == 0:
            continue
        w = np.zeros(npar * 2 * r * nrhs)
        wref = lambda c, r=r: BlockRef(w, (c // 2) * 2 * r * nrhs + (c % 2) * r, r, nrhs, 2 * r)  # noqa: E731
        batched_gemm(
            [(BlockRef(V, c1 * n + c * nc, nc, r, n), BlockRef(x, c * nc, nc, nrhs, n), wref(c)) for c in range(nch)],
            transpose_a="conj_transpose",
            executor=ex,
        )
        krefs = [BlockRef(Ks[lv], p * 4 * r * r, 2 * r, 2 * r, 2 * r) for p in range(npar)]
        batched_lu_solve_inplace(krefs, kpivs[lv], [BlockRef(w, p * 2 * r * nrhs, 2 * r, nrhs, 2 * r) for p in range(npar)], executor=ex)
        batched_gemm(
            [(BlockRef(Y, c1 * n + c * nc, nc, r, n), wref(c), BlockRef(x, c * nc, nc, nrhs, n)) for c in range(nch)],
            alpha=-1.0,
            beta=1.0,
            executor=ex,
        )
    return x.reshape(nrhs, n).T.copy()


def ref_assemble(entry, n: int, m: int, r: int):
    """HODLR of the n x n matrix entry(i, j) assembled by the reference's own
    ``compress`` (compress.py:173-200, CompressionConfig(tol=0, max_rank=r,
    method="aca_rook_pivot")) on both orientations of every sibling block
    (SPEC.md:163-171); leaves materialised exactly.  Flat D, U, V (SPEC layout)."""
    import math

    from hodlr.compress import CompressionConfig, compress  # type: ignore
    from hodlr.tree import IndexRange  # type: ignore

    L = int(round(math.log2(n // m)))
    D = np.empty((1 << L) * m * m)
    for a in range(1 << L):
        idx = np.arange(a * m, (a + 1) * m)
        D[a * m * m : (a + 1) * m * m] = np.asarray(entry(idx[:, None], idx[None, :])).ravel(order="F")
    U, V = np.zeros(n * r * L), np.zeros(n * r * L)
    cfg = CompressionConfig(tol=0.0, max_rank=r, method="aca_rook_pivot")
    for lv in range(1, L + 1):
        nl = n >> lv
        for p in range(1 << (lv - 1)):
            for o in range(2):
                ra, cb = (2 * p + o) * nl, (2 * p + 1 - o) * nl
                f = compress(entry, IndexRange(ra, ra + nl), IndexRange(cb, cb + nl), cfg)
                for l in range(f.rank):
                    c = ((lv - 1) * r + l) * n
                    U[c + ra : c + ra + nl] = f.u[:, l]
                    V[c + cb : c + cb + nl] = np.conj(f.v[:, l])
    return D, U, V


def ref_assemble_laplace(n_total: int, n: int, m: int, r: int):
    """The leading n x n diagonal block of the cfg2 operator
    (``laplace_dl_oracle(contour_default(n_total))``, problems.py:133-217)
    assembled by the reference's own ``compress`` (see :func:`ref_assemble`)."""
    from hodlr.problems import contour_default, laplace_dl_oracle  # type: ignore

    return ref_assemble(laplace_dl_oracle(contour_default(n_total)), n, m, r)
