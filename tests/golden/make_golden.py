"""Generate the golden vectors that pin the CPU oracle to the reference.

Runs ONLY in the build container (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The HODLR factorization/solve recipe of SURVEY.md Appendix B (PAPER.md
Alg. 3/4) is driven here *through the reference's own public
kernels* -- ``hodlr.backend.BlockRef``, ``batched_lu_factor_inplace``,
``batched_lu_solve_inplace``, ``batched_gemm`` (backend.py:48, 320, 481, 570)
-- with the serial executor and ``scratch=None``.  The same inputs are then run
through ``oracle/hodlr_oracle.py`` and every output buffer is asserted to be
BIT-IDENTICAL.  The reference outputs are written to ``tests/golden/*.npz`` so
the GPU box (which has no /root/reference) can check the oracle and the CUDA
path against them.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from hodlr.backend import (  # noqa: E402  (reference, read-only)
    BlockRef,
    batched_gemm,
    batched_lu_factor_inplace,
    batched_lu_solve_inplace,
)

from oracle import hodlr_oracle as orc  # noqa: E402

CASES = [
    # name, N, m, r, s(U scale), seed, nrhs
    ("n256_m16_r4_s1", 256, 16, 4, 1.0, 11, 3),
    ("n512_m32_r8_s16", 512, 32, 8, 16.0, 12, 2),
    ("n1024_m64_r16_s16", 1024, 64, 16, 16.0, 13, 1),
    ("n512_m16_r32_s16", 512, 16, 32, 16.0, 14, 2),
]


def ref_factorize(D, Y, V, n, m, r, L):
    """Appendix-B recipe through the reference kernels; returns pivots + K."""
    nleaf = 1 << L
    drefs = [BlockRef(D, a * m * m, m, m, m) for a in range(nleaf)]
    dpiv, _ = batched_lu_factor_inplace(drefs)
    assert not dpiv.singular
    if L > 0:
        batched_lu_solve_inplace(drefs, dpiv, [BlockRef(Y, a * m, m, r * L, n) for a in range(nleaf)])
    Ks, kpivs = [None] * L, [None] * L
    for lv in range(L - 1, -1, -1):
        nch, npar, nc, ncol = 1 << (lv + 1), 1 << lv, n >> (lv + 1), r * (lv + 1)
        tw = np.zeros(nch * r * ncol)
        batched_gemm(
            [
                (
                    BlockRef(V, lv * r * n + c * nc, nc, r, n),
                    BlockRef(Y, c * nc, nc, ncol, n),
                    BlockRef(tw, c * r * ncol, r, ncol, r),
                )
                for c in range(nch)
            ],
            transpose_a="conj_transpose",
        )
        K = np.zeros(npar * 4 * r * r)
        for p in range(npar):
            kb = BlockRef(K, p * 4 * r * r, 2 * r, 2 * r, 2 * r).view()
            kb[:r, :r] = BlockRef(tw, 2 * p * r * ncol + lv * r * r, r, r, r).view()
            kb[r:, r:] = BlockRef(tw, (2 * p + 1) * r * ncol + lv * r * r, r, r, r).view()
            kb[:r, r:] = np.eye(r)
            kb[r:, :r] = np.eye(r)
        krefs = [BlockRef(K, p * 4 * r * r, 2 * r, 2 * r, 2 * r) for p in range(npar)]
        kpiv, _ = batched_lu_factor_inplace(krefs)
        assert not kpiv.singular
        Ks[lv], kpivs[lv] = K, kpiv
        if lv == 0:
            continue
        wc = r * lv
        W = np.zeros(npar * 2 * r * wc)
        for c in range(nch):
            BlockRef(W, (c // 2) * 2 * r * wc + (c % 2) * r, r, wc, 2 * r).view()[...] = BlockRef(
                tw, c * r * ncol, r, wc, r
            ).view()
        batched_lu_solve_inplace(krefs, kpiv, [BlockRef(W, p * 2 * r * wc, 2 * r, wc, 2 * r) for p in range(npar)])
        batched_gemm(
            [
                (
                    BlockRef(Y, lv * r * n + c * nc, nc, r, n),
                    BlockRef(W, (c // 2) * 2 * r * wc + (c % 2) * r, r, wc, 2 * r),
                    BlockRef(Y, c * nc, nc, wc, n),
                )
                for c in range(nch)
            ],
            alpha=-1.0,
            beta=1.0,
        )
    return dpiv, Ks, kpivs


def ref_solve(D, dpiv, Y, V, Ks, kpivs, b, n, m, r, L):
    nrhs = b.shape[1]
    x = np.asfortranarray(b).ravel(order="F").copy()
    nleaf = 1 << L
    drefs = [BlockRef(D, a * m * m, m, m, m) for a in range(nleaf)]
    batched_lu_solve_inplace(drefs, dpiv, [BlockRef(x, a * m, m, nrhs, n) for a in range(nleaf)])
    for lv in range(L - 1, -1, -1):
        nch, npar, nc = 1 << (lv + 1), 1 << lv, n >> (lv + 1)
        w = np.zeros(npar * 2 * r * nrhs)
        wref = lambda c: BlockRef(w, (c // 2) * 2 * r * nrhs + (c % 2) * r, r, nrhs, 2 * r)  # noqa: E731
        batched_gemm(
            [(BlockRef(V, lv * r * n + c * nc, nc, r, n), BlockRef(x, c * nc, nc, nrhs, n), wref(c)) for c in range(nch)],
            transpose_a="conj_transpose",
        )
        krefs = [BlockRef(Ks[lv], p * 4 * r * r, 2 * r, 2 * r, 2 * r) for p in range(npar)]
        batched_lu_solve_inplace(krefs, kpivs[lv], [BlockRef(w, p * 2 * r * nrhs, 2 * r, nrhs, 2 * r) for p in range(npar)])
        batched_gemm(
            [(BlockRef(Y, lv * r * n + c * nc, nc, r, n), wref(c), BlockRef(x, c * nc, nc, nrhs, n)) for c in range(nch)],
            alpha=-1.0,
            beta=1.0,
        )
    return x.reshape(nrhs, n).T.copy()


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    for name, n, m, r, s, seed, nrhs in CASES:
        h = orc.make_exact_hodlr(n, m, r, seed=seed, s=s)
        L = h.lay.L
        in_digest = digest(h.D, h.U, h.V)
        b = np.random.default_rng(seed + 1000).standard_normal((n, nrhs))
        A = orc.dense(h)

        # reference kernels
        D, Y, V = h.D.copy(), h.U.copy(), h.V.copy()
        dpiv, Ks, kpivs = ref_factorize(D, Y, V, n, m, r, L)
        x = ref_solve(D, dpiv, Y, V, Ks, kpivs, b, n, m, r, L)

        # oracle restatement must be bit-identical
        fo = orc.factorize(h.copy())
        assert fo.D.tobytes() == D.tobytes(), name
        assert fo.Y.tobytes() == Y.tobytes(), name
        assert np.array_equal(fo.dpiv.perm, dpiv.perm) and np.array_equal(fo.dpiv.swaps, dpiv.swaps)
        for lv in range(L):
            assert fo.K[lv].tobytes() == Ks[lv].tobytes(), (name, lv)
            assert np.array_equal(fo.kpiv[lv].swaps, kpivs[lv].swaps), (name, lv)
        xo = orc.solve(fo, b)
        assert xo.tobytes() == x.tobytes(), name
        # the recipe solves the HODLR system
        xd = np.linalg.solve(A, b)
        err = np.linalg.norm(x - xd) / np.linalg.norm(xd)
        assert err < 1e-11, (name, err)
        la, sg = orc.logdet(fo)
        sd, ld = np.linalg.slogdet(A)
        assert abs(la - ld) <= 1e-9 * max(1.0, abs(ld)) and sg == sd, (name, la, ld, sg, sd)
        nontrivial = int(sum((kp.swaps[:, :r] != (np.arange(r) + r)).sum() for kp in kpivs))
        np.savez_compressed(
            HERE / f"{name}.npz",
            n=n, m=m, r=r, s=s, seed=seed, nrhs=nrhs, input_sha256=in_digest,
            D_lu=D, d_swaps=dpiv.swaps, d_perm=dpiv.perm, Y=Y,
            K=np.concatenate(Ks), k_swaps=np.concatenate([kp.swaps for kp in kpivs]),
            k_perm=np.concatenate([kp.perm for kp in kpivs]),
            b=b, x=x, logdet=la, logdet_sign=sg, dense_err=err,
        )
        print(f"{name}: L={L} oracle==reference bitwise; dense err {err:.2e}; "
              f"logdet {la:.6f} ({sg:+.0f}); nontrivial K pivots {nontrivial}")

    # SPEC 2x2 worked example: [[2,1],[1,2]], tree(2,1)
    D = np.array([2.0, 2.0]); U = np.array([1.0, 1.0]); V = np.array([1.0, 1.0])
    dpiv, Ks, kpivs = ref_factorize(D, U, V, 2, 1, 1, 1)
    assert U.tolist() == [0.5, 0.5] and Ks[0].reshape(2, 2).T.tolist() is not None
    x = ref_solve(D, dpiv, U, V, Ks, kpivs, np.array([[3.0], [3.0]]), 2, 1, 1, 1)
    print("spec 2x2: Y", U.tolist(), "K(LU)", Ks[0].tolist(), "kswaps", kpivs[0].swaps.tolist(), "x", x.ravel().tolist())
    np.savez_compressed(HERE / "spec_2x2.npz", Y=U, K_lu=Ks[0], k_swaps=kpivs[0].swaps, x=x)


if __name__ == "__main__":
    main()
