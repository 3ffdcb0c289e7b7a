"""GPU: BASELINE cfg4 -- GMRES on the Schur-complement surrogate operator
(fp64 HODLR, rank 32) preconditioned by a low-accuracy rank-8 fp32 HODLR
factorization of the same kernel; the device builder for the surrogate kernel."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2208_06290_b200 as hb  # noqa: E402


def test_schur_surrogate_builder_matches_the_kernel():
    # leaves exact; off-diagonal blocks of a 2-D separator plane need ranks that grow toward
    # the top levels, so the HODLR error falls with the rank (the cfg4 preconditioning regime)
    n, m = 1 << 12, 64
    errs = {}
    for r in (8, 32, 64):
        h = hb.schur_surrogate_hodlr(n, m, r, sigma=0.1)
        P = hb.separator_grid(n, h.L)
        A = h.reconstruct_dense().cpu().numpy()
        d2 = (P[0][:, None] - P[0][None, :]) ** 2 + (P[1][:, None] - P[1][None, :]) ** 2
        with np.errstate(divide="ignore"):
            S = -1.0 / (np.pi * d2 ** 1.5)
        np.fill_diagonal(S, 2.8754826265883277 + 0.1)
        assert np.array_equal(np.diag(A), np.diag(S))
        errs[r] = np.linalg.norm(A - S) / np.linalg.norm(S)
    assert errs[64] < errs[32] < errs[8] < 0.2, errs
    assert errs[64] < 1e-2, errs
    assert np.all(np.linalg.eigvalsh((S + S.T) / 2) > 0)  # SPD surrogate


def test_gmres_with_fp32_rank8_preconditioner_converges():
    n, m = 1 << 13, 64
    op = hb.schur_surrogate_hodlr(n, m, 32, sigma=0.1)
    p8 = hb.schur_surrogate_hodlr(n, m, 8, sigma=0.1)
    prec = hb.factorize(hb.HodlrMatrix(p8.tree, 8, p8.D.float(), p8.U.float(), p8.V.float()))
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    res = hb.gmres_hodlr(op, prec, b, tol=1e-10, restart=30)
    assert res.converged and res.true_relres <= 1e-10, (res.true_relres, res.iterations)
    # the direct fp64 solve of the same operator agrees
    x_direct = hb.solve(hb.factorize(op.clone()), b)
    assert float(torch.linalg.norm(res.x - x_direct) / torch.linalg.norm(x_direct)) < 1e-8
    plain = hb.gmres(op.matvec, b, tol=1e-10, restart=30, maxiter=res.iterations)
    assert not plain.converged or plain.iterations >= res.iterations  # the preconditioner pays
