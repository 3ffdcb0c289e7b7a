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

from oracle import hodlr_oracle as orc  # noqa: E402
from oracle.ref_driver import BlockRef, ref_factorize, ref_solve  # noqa: E402  (reference kernels)

CASES = [
    # name, N, m, r, s(U scale), seed, nrhs[, per-level ranks (level 1..L)]
    ("n256_m16_r4_s1", 256, 16, 4, 1.0, 11, 3),
    ("n512_m32_r8_s16", 512, 32, 8, 16.0, 12, 2),
    ("n1024_m64_r16_s16", 1024, 64, 16, 16.0, 13, 1),
    ("n512_m16_r32_s16", 512, 16, 32, 16.0, 14, 2),
    # per-level ranks (SPEC.md:147-160 ragged panels padded per level; the paper's
    # Laplace rank profiles fall from the top levels and rise again near the leaves)
    ("ragged_n2048_m32_r16-8-16-32-16-32", 2048, 32, 32, 4.0, 15, 2, (16, 8, 16, 32, 16, 32)),
    ("ragged_n1024_m64_r32-0-16-16", 1024, 64, 32, 16.0, 16, 1, (32, 0, 16, 16)),
]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    for case in CASES:
        name, n, m, r, s, seed, nrhs = case[:7]
        ranks = case[7] if len(case) > 7 else None
        h = orc.make_exact_hodlr(n, m, r, seed=seed, s=s, ranks=ranks)
        L = h.lay.L
        in_digest = digest(h.D, h.U, h.V)
        b = np.random.default_rng(seed + 1000).standard_normal((n, nrhs))
        A = orc.dense(h)

        # reference kernels
        D, Y, V = h.D.copy(), h.U.copy(), h.V.copy()
        dpiv, Ks, kpivs = ref_factorize(D, Y, V, n, m, r, L, ranks=ranks)
        x = ref_solve(D, dpiv, Y, V, Ks, kpivs, b, n, m, r, L, ranks=ranks)

        # oracle restatement must be bit-identical
        fo = orc.factorize(h.copy())
        assert fo.D.tobytes() == D.tobytes(), name
        assert fo.Y.tobytes() == Y.tobytes(), name
        assert np.array_equal(fo.dpiv.perm, dpiv.perm) and np.array_equal(fo.dpiv.swaps, dpiv.swaps)
        live = [lv for lv in range(L) if kpivs[lv] is not None]  # rank-0 levels have no K blocks
        for lv in live:
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
        nontrivial = int(sum((kpivs[lv].swaps[:, : h.lay.rk(lv + 1)] != (np.arange(h.lay.rk(lv + 1)) + h.lay.rk(lv + 1))).sum()
                             for lv in live))
        extra = {} if ranks is None else {"ranks": np.array(ranks)}
        np.savez_compressed(
            HERE / f"{name}.npz",
            n=n, m=m, r=r, s=s, seed=seed, nrhs=nrhs, input_sha256=in_digest,
            D_lu=D, d_swaps=dpiv.swaps, d_perm=dpiv.perm, Y=Y,
            K=np.concatenate([Ks[lv] for lv in live]),
            # uniform: (nK, 2r) stacks; per-level ranks: flat, level after level
            k_swaps=(np.concatenate([kpivs[lv].swaps for lv in live]) if ranks is None
                     else np.concatenate([kpivs[lv].swaps.ravel() for lv in live])),
            k_perm=(np.concatenate([kpivs[lv].perm for lv in live]) if ranks is None
                    else np.concatenate([kpivs[lv].perm.ravel() for lv in live])),
            b=b, x=x, logdet=la, logdet_sign=sg, dense_err=err, **extra,
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
