"""Golden vectors for HODLR assembly (device builder vs the reference's ACA).

Runs ONLY in the build container (needs /root/reference, read-only):

    python tests/golden/make_build_golden.py

Each case assembles a HODLR operator by calling the reference's own
``hodlr.compress.compress`` (compress.py:173-200) with
``CompressionConfig(tol=0, max_rank=r, method="aca_rook_pivot")`` on both
orientations of every sibling block, and its own entry oracles
(``hodlr.problems.laplace_dl_oracle(contour_default(n))``, problems.py:133-217,
or a dense matrix).  ``oracle/build_oracle.py`` must reproduce D, U, V
BIT-FOR-BIT; the reference outputs go to ``tests/golden/build_*.npz`` for the
GPU tests (the GPU box has no /root/reference).
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from hodlr.compress import CompressionConfig, compress  # noqa: E402  (reference)
from hodlr.problems import contour_default, laplace_dl_oracle  # noqa: E402  (reference)
from hodlr.tree import IndexRange  # noqa: E402  (reference)
from oracle import build_oracle as bo  # noqa: E402


def ref_assemble(entry, n, m, r):
    L = int(round(math.log2(n // m)))
    D = np.empty((1 << L) * m * m)
    for a in range(1 << L):
        idx = np.arange(a * m, (a + 1) * m)
        D[a * m * m : (a + 1) * m * m] = np.asarray(entry(idx[:, None], idx[None, :]), dtype=np.float64).ravel(order="F")
    U, V = np.zeros(n * r * L), np.zeros(n * r * L)
    cfg = CompressionConfig(tol=0.0, max_rank=r, method="aca_rook_pivot")
    ranks = []
    for lv in range(1, L + 1):
        nl = n >> lv
        for p in range(1 << (lv - 1)):
            for o in range(2):
                ra, cb = (2 * p + o) * nl, (2 * p + 1 - o) * nl
                f = compress(entry, IndexRange(ra, ra + nl), IndexRange(cb, cb + nl), cfg)
                ranks.append(f.rank)
                for l in range(f.rank):
                    c = ((lv - 1) * r + l) * n
                    U[c + ra : c + ra + nl] = f.u[:, l]
                    V[c + cb : c + cb + nl] = np.conj(f.v[:, l])
    return D, U, V, np.array(ranks)


def smooth_dense(n, seed):
    rng = np.random.default_rng(seed)
    x = np.sort(rng.uniform(-1.0, 1.0, n))
    A = 1.0 / (1.0 + 25.0 * (x[:, None] - x[None, :]) ** 2)
    return A + 2.0 * np.eye(n)


CASES = [
    # name, kind, n, m, r
    ("build_laplace_n1024_m64_r8", "laplace", 1024, 64, 8),
    ("build_laplace_n2048_m32_r16", "laplace", 2048, 32, 16),
    ("build_dense_spec2x2", "spec2x2", 2, 1, 1),
    ("build_dense_identity_n64_m16_r4", "identity", 64, 16, 4),
    ("build_dense_smooth_n256_m16_r6", "smooth", 256, 16, 6),
    # exact rank-1 off-diagonal blocks with power-of-two entries: the residual
    # becomes exactly zero after one cross, so the zero-row scan runs to the end
    ("build_dense_rank1_n128_m16_r3", "rank1", 128, 16, 3),
]


def main():
    for name, kind, n, m, r in CASES:
        if kind == "laplace":
            ref_entry = laplace_dl_oracle(contour_default(n))
            my_entry = bo.LaplaceDL(n)
            A = None
        else:
            A = {"spec2x2": np.array([[2.0, 1.0], [1.0, 2.0]]), "identity": np.eye(n),
                 "smooth": smooth_dense(n, 5) if kind == "smooth" else None,
                 "rank1": np.outer(2.0 ** (np.arange(n) % 3), 2.0 ** ((7 * np.arange(n)) % 3)) + 8.0 * np.eye(n)}[kind]
            ref_entry = lambda i, j, A=A: A[i, j]  # noqa: E731
            my_entry = bo.Dense(A)
        D, U, V, ranks = ref_assemble(ref_entry, n, m, r)
        D2, U2, V2 = bo.assemble(my_entry, n, m, r)
        assert D.tobytes() == D2.tobytes(), name
        assert U.tobytes() == U2.tobytes(), name
        assert V.tobytes() == V2.tobytes(), name
        out = dict(n=n, m=m, r=r, kind=kind, D=D, U=U, V=V, ranks=ranks)
        if A is not None:
            out["A"] = A
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, "ranks", np.bincount(ranks).nonzero()[0].tolist(), "ok")


if __name__ == "__main__":
    main()
