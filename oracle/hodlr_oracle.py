"""CPU ORACLE for the HODLR factorize/solve hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / the timed CPU baseline.  The product package
``paper_2208_06290_b200`` never imports it; its GPU path fails loudly when the
CUDA library is missing.

What it restates (no code copied; same arithmetic, same buffer views):

* the reference batched kernel layer ``pkg/src/hodlr/backend.py``
  - block views on flat column-major buffers      backend.py:48-89, 114-144
  - GEMM ``c <- alpha op(a) b + beta c``           backend.py:282-303
  - right-looking partial-pivot LU (+ guard)      backend.py:444-478
  - pivot-gather + unit-L / U substitution         backend.py:546-567
  - flop conventions                              backend.py:240-251
* the level-wise factorization / solve drivers the reference only specifies
  (Alg. 3/4) in the SPEC column-major layout
  (SPEC.md:147-160), following SURVEY.md Appendix B: leaf getrf, leaf getrs of
  all Y-panel rows, then per level [W|T] = V_c^T Y(I_c, 0:r(l+1)), K_p
  assembly [[T_2p, I], [I, T_2p+1]], K getrf, K getrs(W), Y update.

Parity pin: ``tests/golden/make_golden.py`` runs the same recipe through the
reference's own public kernels (``hodlr.backend`` imported read-only from
/root/reference) and asserts this oracle reproduces every buffer BIT-FOR-BIT;
the resulting vectors are committed under ``tests/golden/``.  The SPEC worked
examples are also pinned by the tests.

Layout (uniform rank r, N = m 2^L):
  D    flat, leaf a at offset a*m*m, column-major m x m
  Y/U  flat N x rL column-major slab, ld = N; level l' in 1..L holds
       columns [(l'-1) r, l' r)  (Fig. 3)
  V    same as Y
  K[l] flat, parent p at offset p*(2r)^2, column-major 2r x 2r
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import as_strided

# ---------------------------------------------------------------------------
# views (backend.py:76-83 BlockRef.view, :114-144 as_stack)
# ---------------------------------------------------------------------------


def bview(buf: np.ndarray, off: int, rows: int, cols: int, ld: int) -> np.ndarray:
    """Writable (rows, cols) column-major view of ``buf[off + i + j*ld]``."""
    it = buf.itemsize
    return as_strided(buf[off:], shape=(rows, cols), strides=(it, ld * it))


def sview(buf, off, step, nb, rows, cols, ld) -> np.ndarray:
    """(nb, rows, cols) stack of equally spaced blocks; one block -> stride 0."""
    it = buf.itemsize
    bstride = 0 if nb == 1 else step * it
    return as_strided(buf[off:], shape=(nb, rows, cols), strides=(bstride, it, ld * it))


# ---------------------------------------------------------------------------
# flop conventions (backend.py:240-251)
# ---------------------------------------------------------------------------


def gemm_flops(m, k, n):
    return 2 * m * k * n


def lu_factor_flops(s):
    return s * (s - 1) // 2 + s * (s - 1) * (2 * s - 1) // 3


def lu_solve_flops(s, ncols):
    return 2 * s * s * ncols


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------


def gemm_into(a, b, c, alpha=1.0, beta=0.0, conj_a=False):
    """c <- alpha op(a) b + beta c; the product is rounded before combining.

    backend.py:282-303: alpha=1,beta=0 writes matmul straight into c;
    otherwise tmp = matmul, then (c*beta) +/- tmp as separate ufuncs.
    """
    if conj_a:
        a = a.swapaxes(-1, -2)
        if np.iscomplexobj(a):
            a = a.conj()
    if alpha == 1 and beta == 0:
        np.matmul(a, b, out=c)
        return
    prod = np.matmul(a, b)
    if beta == 0:
        np.multiply(prod, alpha, out=c)
        return
    if beta != 1:
        np.multiply(c, beta, out=c)
    if alpha == 1:
        np.add(c, prod, out=c)
    elif alpha == -1:
        np.subtract(c, prod, out=c)
    else:
        prod *= alpha
        np.add(c, prod, out=c)


@dataclass
class Pivots:
    """LAPACK-style swaps, final row permutation, singular flags (backend.py:419-441)."""

    swaps: np.ndarray
    perm: np.ndarray
    singular: np.ndarray  # bool per block

    def sign(self) -> np.ndarray:
        k = np.arange(self.swaps.shape[1])
        odd = ((self.swaps != k).sum(axis=1) % 2) == 1
        return np.where(odd, -1.0, 1.0)


def lu_factor(stack: np.ndarray) -> Pivots:
    """In-place right-looking partial-pivot LU of a (B, s, s) stack.

    Restates backend.py:444-478: step k picks the FIRST max |a[k:, k]|
    (numpy argmax), swaps whole rows k <-> p, flags the block singular when
    |pivot| <= eps*s*max|original column k|, divides the sub-column by the
    pivot (a zero pivot divides by one), then subtracts the separately
    rounded outer product l*u from the trailing block.
    """
    nb, s = stack.shape[0], stack.shape[1]
    swaps = np.zeros((nb, s), dtype=np.int64)
    sing = np.zeros(nb, dtype=bool)
    if nb == 0 or s == 0:
        return Pivots(swaps, swaps.copy(), sing)
    eps = np.finfo(stack.dtype).eps
    colmax = np.abs(stack).max(axis=1)
    rows = np.arange(nb)
    perm = np.repeat(np.arange(s, dtype=np.int64)[None, :], nb, axis=0)
    for k in range(s):
        p = k + np.abs(stack[:, k:, k]).argmax(axis=1)
        swaps[:, k] = p
        row_k = stack[rows, k, :].copy()
        stack[rows, k, :] = stack[rows, p, :]
        stack[rows, p, :] = row_k
        pk = perm[rows, k].copy()
        perm[rows, k] = perm[rows, p]
        perm[rows, p] = pk
        piv = stack[:, k, k]
        sing |= np.abs(piv) <= eps * s * colmax[:, k]
        if k + 1 < s:
            div = np.where(piv == 0, np.ones((), dtype=stack.dtype), piv)
            stack[:, k + 1 :, k] /= div[:, None]
            outer = stack[:, k + 1 :, k : k + 1] * stack[:, k : k + 1, k + 1 :]
            stack[:, k + 1 :, k + 1 :] -= outer
    return Pivots(swaps, perm, sing)


def lu_solve(lu: np.ndarray, perm: np.ndarray, rhs: np.ndarray) -> None:
    """In-place P^T-gather, unit-lower forward and upper backward substitution.

    Restates backend.py:546-567 (rhs (..., B, s, c); each row update is one
    small matmul of the already-solved rows; the diagonal is a true divide).
    """
    s = lu.shape[-1]
    if s == 0 or rhs.size == 0:
        return
    idx = perm.reshape((1,) * (rhs.ndim - 3) + perm.shape + (1,))
    idx = np.broadcast_to(idx, rhs.shape[:-2] + (s, rhs.shape[-1]))
    rhs[...] = np.take_along_axis(rhs, idx, axis=-2)
    for i in range(1, s):
        rhs[..., i, :] -= np.matmul(lu[..., i : i + 1, :i], rhs[..., :i, :])[..., 0, :]
    for i in range(s - 1, -1, -1):
        if i + 1 < s:
            rhs[..., i, :] -= np.matmul(lu[..., i : i + 1, i + 1 :], rhs[..., i + 1 :, :])[..., 0, :]
        rhs[..., i, :] /= lu[..., i, i][..., None]


def _chunks(nitems: int, threads: int, body) -> None:
    """Contiguous chunking over a thread pool (backend.py:188-215 semantics)."""
    if nitems <= 0:
        return
    k = max(1, min(threads, nitems))
    if k == 1:
        body(0, nitems)
        return
    bounds = [nitems * i // k for i in range(k + 1)]
    with ThreadPoolExecutor(max_workers=k) as pool:
        futs = [pool.submit(body, bounds[i], bounds[i + 1]) for i in range(k) if bounds[i] < bounds[i + 1]]
        for f in futs:
            f.result()


# ---------------------------------------------------------------------------
# HODLR layout, generator, dense reconstruction
# ---------------------------------------------------------------------------


@dataclass
class Layout:
    """N = m 2^L rows; rank r at every level, or per-level ``ranks`` (level
    l' = 1..L at ranks[l'-1], SPEC.md:147-160 ragged panels padded per level):
    level l' then owns slab columns [c(l'), c(l') + rk(l'))."""

    n: int
    m: int
    r: int
    ranks: tuple | None = None

    @property
    def L(self) -> int:
        return int(round(math.log2(self.n // self.m)))

    def rk(self, lp: int) -> int:
        return self.r if self.ranks is None else int(self.ranks[lp - 1])

    def c(self, lp: int) -> int:
        return (lp - 1) * self.r if self.ranks is None else int(sum(self.ranks[: lp - 1]))

    @property
    def C(self) -> int:
        return self.c(self.L + 1)

    def __post_init__(self):
        if self.n % self.m or (self.n // self.m) & (self.n // self.m - 1):
            raise ValueError("oracle layout needs N = m * 2^L")
        if self.ranks is not None:
            self.ranks = tuple(int(x) for x in self.ranks)
            if len(self.ranks) != self.L:
                raise ValueError("per-level ranks: one per level 1..L")


@dataclass
class HodlrData:
    lay: Layout
    D: np.ndarray  # flat 2^L m^2
    U: np.ndarray  # flat N rL (overwritten by Y in factorize)
    V: np.ndarray  # flat N rL

    def copy(self) -> "HodlrData":
        return HodlrData(self.lay, self.D.copy(), self.U.copy(), self.V.copy())


def make_exact_hodlr(n: int, m: int, r: int, seed: int = 0, s: float = 1.0, dtype=np.float64,
                     ranks=None) -> HodlrData:
    """Seeded exact uniform-rank HODLR (SURVEY.md §8d stand-in generator).

    D_a = N(0,1)/sqrt(m) + 4 I; level-l U entries N(0, s^2/n_l), V entries
    N(0, 1/n_l) with n_l = N/2^l rows per node.  s=1: trivial K pivots;
    s=16: most K pivots are real partial-pivot choices.
    """
    lay = Layout(n, m, r if ranks is None else max(ranks, default=0), ranks)
    L = lay.L
    rng = np.random.default_rng(seed)
    nleaf = 1 << L
    D = rng.standard_normal(nleaf * m * m) / math.sqrt(m)
    diag = (np.arange(nleaf)[:, None] * m * m + np.arange(m)[None, :] * (m + 1)).ravel()
    D[diag] += 4.0
    U = rng.standard_normal(n * lay.C)
    V = rng.standard_normal(n * lay.C)
    for lv in range(1, L + 1):
        nl = n >> lv
        sl = slice(lay.c(lv) * n, (lay.c(lv) + lay.rk(lv)) * n)
        U[sl] *= s / math.sqrt(nl)
        V[sl] *= 1.0 / math.sqrt(nl)
    return HodlrData(lay, D.astype(dtype), U.astype(dtype), V.astype(dtype))


def dense(h: HodlrData) -> np.ndarray:
    """Exact dense expansion: leaf blocks + U_a V_b^T / U_b V_a^T per sibling pair."""
    lay = h.lay
    n, m, r, L = lay.n, lay.m, lay.r, lay.L
    A = np.zeros((n, n), dtype=h.D.dtype)
    for a in range(1 << L):
        A[a * m : (a + 1) * m, a * m : (a + 1) * m] = bview(h.D, a * m * m, m, m, m)
    for lv in range(1, L + 1):
        nl = n >> lv
        r, c0 = lay.rk(lv), lay.c(lv) * n
        for k in range(1 << (lv - 1)):
            ia, ib = 2 * k * nl, (2 * k + 1) * nl
            Ua = bview(h.U, c0 + ia, nl, r, n)
            Ub = bview(h.U, c0 + ib, nl, r, n)
            Va = bview(h.V, c0 + ia, nl, r, n)
            Vb = bview(h.V, c0 + ib, nl, r, n)
            A[ia : ia + nl, ib : ib + nl] = Ua @ Vb.T
            A[ib : ib + nl, ia : ia + nl] = Ub @ Va.T
    return A


def matvec(h: HodlrData, x: np.ndarray) -> np.ndarray:
    """A x block-wise (SPEC.md:183-191 [OP] matvec):
    y(I_a) = D_a x(I_a) + sum_l' U_c (V_sib^T x_sib) over the sibling pairs,
    without forming A.  x: (N,) or (N, k)."""
    lay = h.lay
    n, m, r, L = lay.n, lay.m, lay.r, lay.L
    X = np.asarray(x, dtype=h.D.dtype).reshape(n, -1)
    Dm = h.D.reshape(1 << L, m, m).transpose(0, 2, 1)  # block a row-major (column-major storage)
    y = np.einsum("aij,ajk->aik", Dm, X.reshape(1 << L, m, -1)).reshape(n, -1)
    for lv in range(1, L + 1):
        nl = n >> lv
        r, c0 = lay.rk(lv), lay.c(lv) * n
        U = h.U[c0 : c0 + r * n].reshape(r, n).T.reshape(1 << (lv - 1), 2, nl, r)
        V = h.V[c0 : c0 + r * n].reshape(r, n).T.reshape(1 << (lv - 1), 2, nl, r)
        w = np.einsum("pcir,pcik->pcrk", V, X.reshape(1 << (lv - 1), 2, nl, -1))  # V_c^T x_c
        y += np.einsum("pcir,pcrk->pcik", U, w[:, ::-1]).reshape(n, -1)  # child 0 gets U_0 w_1
    return y.reshape(np.shape(x))


# ---------------------------------------------------------------------------
# factorize / solve drivers (PAPER Alg. 3/4)
# ---------------------------------------------------------------------------


@dataclass
class Factorization:
    lay: Layout
    D: np.ndarray
    Y: np.ndarray
    V: np.ndarray
    dpiv: Pivots
    K: list = field(default_factory=list)  # K[l] flat, l = 0..L-1
    kpiv: list = field(default_factory=list)
    flops: dict = field(default_factory=dict)


def factorize(h: HodlrData, threads: int = 1) -> Factorization:
    """Alg. 3 over flat buffers; consumes ``h`` (Y overwrites U in place)."""
    lay = h.lay
    n, m, r, L = lay.n, lay.m, lay.r, lay.L
    D, Y, V = h.D, h.U, h.V
    nleaf = 1 << L
    fl = {"leaf_getrf": 0, "leaf_getrs": 0, "tw_gemm": 0, "k_getrf": 0, "k_getrs": 0, "update_gemm": 0}

    # (1) leaf getrf  (Alg.3 l.2)
    dst = sview(D, 0, m * m, nleaf, m, m, m)
    sw = np.zeros((nleaf, m), np.int64)
    pm = np.zeros((nleaf, m), np.int64)
    sg = np.zeros(nleaf, bool)

    def f_body(lo, hi):
        p = lu_factor(dst[lo:hi])
        sw[lo:hi], pm[lo:hi], sg[lo:hi] = p.swaps, p.perm, p.singular

    _chunks(nleaf, threads, f_body)
    dpiv = Pivots(sw, pm, sg)
    fl["leaf_getrf"] = lu_factor_flops(m) * nleaf
    fact = Factorization(lay, D, Y, V, dpiv, flops=fl)
    if sg.any():
        raise SingularError("leaf", L, np.flatnonzero(sg).tolist())

    # (2) leaf getrs on all Y rows (Alg.3 l.3)
    if L > 0:
        yst = sview(Y, 0, m, nleaf, m, lay.C, n)
        _chunks(nleaf, threads, lambda lo, hi: lu_solve(dst[lo:hi], pm[lo:hi], yst[lo:hi]))
        fl["leaf_getrs"] = lu_solve_flops(m, lay.C) * nleaf

    # (3) levels
    for lv in range(L - 1, -1, -1):
        nch = 1 << (lv + 1)
        npar = 1 << lv
        nc = n >> (lv + 1)
        r = lay.rk(lv + 1)  # rank of the children (level lv + 1)
        c1 = lay.c(lv + 1)  # their panel's first column = the columns of levels 1..lv
        ncol = c1 + r
        if r == 0:  # rank-0 level: empty K blocks, no update
            fact.K.insert(0, np.zeros(0, dtype=Y.dtype))
            fact.kpiv.insert(0, Pivots(np.zeros((npar, 0), np.int64), np.zeros((npar, 0), np.int64),
                                       np.zeros(npar, bool)))
            continue
        tw = np.zeros(nch * r * ncol, dtype=Y.dtype)
        va = sview(V, c1 * n, nc, nch, nc, r, n)
        yb = sview(Y, 0, nc, nch, nc, ncol, n)
        tc = sview(tw, 0, r * ncol, nch, r, ncol, r)
        _chunks(nch, threads, lambda lo, hi: gemm_into(va[lo:hi], yb[lo:hi], tc[lo:hi], conj_a=True))
        fl["tw_gemm"] += gemm_flops(r, nc, ncol) * nch

        K = np.zeros(npar * 4 * r * r, dtype=Y.dtype)
        for p in range(npar):
            kb = bview(K, p * 4 * r * r, 2 * r, 2 * r, 2 * r)
            kb[:r, :r] = bview(tw, 2 * p * r * ncol + c1 * r, r, r, r)
            kb[r:, r:] = bview(tw, (2 * p + 1) * r * ncol + c1 * r, r, r, r)
            kb[:r, r:] = np.eye(r)
            kb[r:, :r] = np.eye(r)
        kst = sview(K, 0, 4 * r * r, npar, 2 * r, 2 * r, 2 * r)
        ksw = np.zeros((npar, 2 * r), np.int64)
        kpm = np.zeros((npar, 2 * r), np.int64)
        ksg = np.zeros(npar, bool)

        def k_body(lo, hi):
            p = lu_factor(kst[lo:hi])
            ksw[lo:hi], kpm[lo:hi], ksg[lo:hi] = p.swaps, p.perm, p.singular

        _chunks(npar, threads, k_body)
        fl["k_getrf"] += lu_factor_flops(2 * r) * npar
        fact.K.insert(0, K)
        fact.kpiv.insert(0, Pivots(ksw, kpm, ksg))
        if ksg.any():
            raise SingularError("K", lv, np.flatnonzero(ksg).tolist())
        if lv == 0 or c1 == 0:
            continue
        wcols = c1
        W = np.zeros(npar * 2 * r * wcols, dtype=Y.dtype)
        for c in range(nch):
            bview(W, (c // 2) * 2 * r * wcols + (c % 2) * r, r, wcols, 2 * r)[...] = bview(
                tw, c * r * ncol, r, wcols, r
            )
        wst = sview(W, 0, 2 * r * wcols, npar, 2 * r, wcols, 2 * r)
        _chunks(npar, threads, lambda lo, hi: lu_solve(kst[lo:hi], kpm[lo:hi], wst[lo:hi]))
        fl["k_getrs"] += lu_solve_flops(2 * r, wcols) * npar

        # update: W operand offsets alternate -> reference generic per-item path
        def u_body(lo, hi):
            for c in range(lo, hi):
                a = bview(Y, c1 * n + c * nc, nc, r, n)[None]
                b = bview(W, (c // 2) * 2 * r * wcols + (c % 2) * r, r, wcols, 2 * r)[None]
                cc = bview(Y, c * nc, nc, wcols, n)[None]
                gemm_into(a, b, cc, alpha=-1.0, beta=1.0)

        _chunks(nch, threads, u_body)
        fl["update_gemm"] += gemm_flops(nc, r, wcols) * nch
    return fact


def solve(fact: Factorization, b: np.ndarray, threads: int = 1) -> np.ndarray:
    """Alg. 4; b is (N,) or (N, nrhs) and is not modified."""
    lay = fact.lay
    n, m, r, L = lay.n, lay.m, lay.r, lay.L
    vec = b.ndim == 1
    bb = b.reshape(n, -1)
    nrhs = bb.shape[1]
    x = np.asfortranarray(bb).ravel(order="F").copy()
    nleaf = 1 << L
    dst = sview(fact.D, 0, m * m, nleaf, m, m, m)
    xst = sview(x, 0, m, nleaf, m, nrhs, n)
    _chunks(nleaf, threads, lambda lo, hi: lu_solve(dst[lo:hi], fact.dpiv.perm[lo:hi], xst[lo:hi]))
    for lv in range(L - 1, -1, -1):
        nch, npar, nc = 1 << (lv + 1), 1 << lv, n >> (lv + 1)
        r, c1 = lay.rk(lv + 1), lay.c(lv + 1)
        if r == 0:
            continue
        w = np.zeros(npar * 2 * r * nrhs, dtype=x.dtype)

        def w_body(lo, hi):
            for c in range(lo, hi):
                gemm_into(
                    bview(fact.V, c1 * n + c * nc, nc, r, n)[None],
                    bview(x, c * nc, nc, nrhs, n)[None],
                    bview(w, (c // 2) * 2 * r * nrhs + (c % 2) * r, r, nrhs, 2 * r)[None],
                    conj_a=True,
                )

        _chunks(nch, threads, w_body)
        kst = sview(fact.K[lv], 0, 4 * r * r, npar, 2 * r, 2 * r, 2 * r)
        wst = sview(w, 0, 2 * r * nrhs, npar, 2 * r, nrhs, 2 * r)
        _chunks(npar, threads, lambda lo, hi: lu_solve(kst[lo:hi], fact.kpiv[lv].perm[lo:hi], wst[lo:hi]))

        def x_body(lo, hi):
            for c in range(lo, hi):
                gemm_into(
                    bview(fact.Y, c1 * n + c * nc, nc, r, n)[None],
                    bview(w, (c // 2) * 2 * r * nrhs + (c % 2) * r, r, nrhs, 2 * r)[None],
                    bview(x, c * nc, nc, nrhs, n)[None],
                    alpha=-1.0,
                    beta=1.0,
                )

        _chunks(nch, threads, x_body)
    out = x.reshape(nrhs, n).T
    return out[:, 0].copy() if vec else np.ascontiguousarray(out)


def logdet(fact: Factorization):
    """(log|det A|, sign) from leaf and K LU diagonals.

    det(I + Z X^*) = det(I + X^* Z) (Sylvester) = det(K_p) (-1)^{r r}
    because K_p is I + X^* Z with its two block columns exchanged.
    """
    lay = fact.lay
    m, r, L = lay.m, lay.r, lay.L
    nleaf = 1 << L
    dd = np.stack([np.diagonal(bview(fact.D, a * m * m, m, m, m)) for a in range(nleaf)])
    logabs = float(np.log(np.abs(dd)).sum())
    sign = float(np.prod(fact.dpiv.sign()) * np.prod(np.sign(dd)))
    for lv in range(L):
        npar = 1 << lv
        r = lay.rk(lv + 1)
        if r == 0:
            continue
        kd = np.stack([np.diagonal(bview(fact.K[lv], p * 4 * r * r, 2 * r, 2 * r, 2 * r)) for p in range(npar)])
        logabs += float(np.log(np.abs(kd)).sum())
        sign *= float(np.prod(fact.kpiv[lv].sign()) * np.prod(np.sign(kd)))
        if (r * r) % 2 == 1:
            sign *= (-1.0) ** npar
    return logabs, sign


def factor_flops(n: int, m: int, r: int) -> int:
    """Closed-form factor flops (equals the counters above)."""
    L = int(round(math.log2(n // m)))
    t = lu_factor_flops(m) * (1 << L) + lu_solve_flops(m, r * L) * (1 << L)
    for lv in range(L):
        nc = n >> (lv + 1)
        t += gemm_flops(r, nc, r * (lv + 1)) * (1 << (lv + 1))
        t += lu_factor_flops(2 * r) * (1 << lv)
        if lv > 0:
            t += lu_solve_flops(2 * r, r * lv) * (1 << lv)
            t += gemm_flops(nc, r, r * lv) * (1 << (lv + 1))
    return t


def solve_flops(n: int, m: int, r: int, nrhs: int = 1) -> int:
    """Closed-form solve flops: 2mN + 4rNL + 8r^2(2^L - 1) per rhs column."""
    L = int(round(math.log2(n // m)))
    return nrhs * (2 * m * n + 4 * r * n * L + 8 * r * r * ((1 << L) - 1))


class SingularError(RuntimeError):
    def __init__(self, what, level, nodes):
        self.what, self.level, self.nodes = what, level, list(nodes)
        super().__init__(f"singular {what} block at level {level}, node(s) {self.nodes}")
