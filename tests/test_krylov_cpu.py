"""CPU: the device GMRES driver (paper_2208_06290_b200/krylov.py) on torch CPU
tensors with dense operators -- convergence, restarts, right preconditioning."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2208_06290_b200.krylov import gmres  # noqa: E402


def _problem(n=200, seed=0):
    rng = np.random.default_rng(seed)
    A = np.eye(n) * 4 + rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    return torch.from_numpy(A), torch.from_numpy(b), np.linalg.solve(A, b)


def test_unpreconditioned_converges_to_the_dense_solution():
    A, b, x_ref = _problem()
    res = gmres(lambda v: A @ v, b, tol=1e-12, restart=60, maxiter=200)
    assert res.converged and res.true_relres <= 1e-12
    assert np.linalg.norm(res.x.numpy() - x_ref) / np.linalg.norm(x_ref) < 1e-10


def test_restarted_gmres_with_an_inexact_preconditioner():
    A, b, x_ref = _problem(seed=1)
    # preconditioner: the inverse of a perturbed operator (as a low-accuracy fp32 HODLR would be)
    Ap = A.numpy() + 1e-3 * np.random.default_rng(2).standard_normal(A.shape)
    Minv = torch.from_numpy(np.linalg.inv(Ap).astype(np.float32))
    res = gmres(lambda v: A @ v, b, precond=lambda v: (Minv @ v.float()).double(), tol=1e-11, restart=3,
                maxiter=50)
    assert res.converged and res.iterations <= 12, res.iterations
    assert res.restarts >= 1
    assert np.linalg.norm(res.x.numpy() - x_ref) / np.linalg.norm(x_ref) < 1e-9
    assert res.history == sorted(res.history, reverse=True) or res.restarts > 0


def test_zero_rhs_and_argument_errors():
    A, _, _ = _problem(n=20)
    res = gmres(lambda v: A @ v, torch.zeros(20, dtype=torch.float64))
    assert res.converged and res.iterations == 0 and float(res.x.abs().max()) == 0.0
    with pytest.raises(ValueError):
        gmres(lambda v: A @ v, torch.ones(20, dtype=torch.float64), restart=0)
