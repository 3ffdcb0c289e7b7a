"""Preconditioned restarted GMRES on the device (BASELINE cfg4: a low-accuracy
fp32 HODLR factorization preconditioning an fp64 operator inside GMRES).

The reference has no Krylov layer (SPEC.md:416, 493 list iterative solvers as
non-goals; its only refinement is SPEC.md:392-400 ``solve_with_refinement``);
this is the SURVEY §8(f) "next" row that puts the HODLR solve to work as the
paper's preconditioner use case.  Right preconditioning: GMRES on A M^-1 y = b,
x = M^-1 y, so the monitored residual is the true ||b - A x||.  Arnoldi with
classical Gram-Schmidt applied twice (CGS2: two V^T w GEMVs per step, stable
like MGS, two launches instead of j), Givens rotations on the (tiny)
Hessenberg matrix on the host.

``matvec`` / ``precond`` are callables on torch tensors (device or host), so
the same code runs the HODLR matvec (``HodlrMatrix.matvec``) and the fp32
HODLR solve (``solve`` of a float32 factorization, cast in and out).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field


@dataclass
class GmresResult:
    x: "object"
    converged: bool
    iterations: int            # total Arnoldi steps (matvec + precond applications)
    restarts: int
    history: list = field(default_factory=list)  # relative residual after each step (Arnoldi estimate)
    true_relres: float = float("nan")            # ||b - A x|| / ||b|| recomputed at the end


def gmres(matvec, b, precond=None, tol: float = 1e-10, restart: int = 30, maxiter: int = 300,
          x0=None) -> GmresResult:
    """Right-preconditioned GMRES(restart).  Stops when the Arnoldi residual
    estimate drops below ``tol * ||b||`` (then verifies with a true residual;
    a restart continues if it does not hold) or after ``maxiter`` steps."""
    import torch

    if restart < 1 or maxiter < 1:
        raise ValueError("restart and maxiter must be >= 1")
    b = b.reshape(-1)
    n = b.numel()
    dt = b.dtype
    M = precond or (lambda v: v)
    nb = float(torch.linalg.norm(b))
    x = torch.zeros_like(b) if x0 is None else x0.reshape(-1).to(dtype=dt).clone()
    if nb == 0.0:
        return GmresResult(torch.zeros_like(b), True, 0, 0, [0.0], 0.0)
    hist, steps, restarts = [], 0, 0
    V = torch.empty(restart + 1, n, dtype=dt, device=b.device)
    while True:
        r = b - matvec(x) if (x0 is not None or steps) else b.clone()
        beta = float(torch.linalg.norm(r))
        if beta <= tol * nb or steps >= maxiter:
            rel = beta / nb
            return GmresResult(x, beta <= tol * nb, steps, restarts, hist, rel)
        V[0] = r / beta
        H = torch.zeros(restart + 1, restart, dtype=torch.float64)
        cs, sn = [0.0] * restart, [0.0] * restart
        g = [0.0] * (restart + 1)
        g[0] = beta
        Z = []  # preconditioned directions M^-1 v_j (kept: x += Z y)
        k = 0
        for j in range(restart):
            z = M(V[j])
            Z.append(z)
            w = matvec(z)
            # CGS2: h = V^T w twice
            h1 = V[: j + 1] @ w
            w = w - V[: j + 1].T @ h1
            h2 = V[: j + 1] @ w
            w = w - V[: j + 1].T @ h2
            hcol = (h1 + h2).double().cpu()
            hn = float(torch.linalg.norm(w))
            H[: j + 1, j] = hcol
            H[j + 1, j] = hn
            # apply previous rotations, then the new one
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            a, c = float(H[j, j]), float(H[j + 1, j])
            den = math.hypot(a, c)
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (a / den, c / den)
            H[j, j] = cs[j] * a + sn[j] * c
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            steps += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / nb)
            if abs(g[j + 1]) <= tol * nb or steps >= maxiter or hn == 0.0:
                break
            V[j + 1] = w / hn
        # y = H[:k, :k]^-1 g[:k] (upper triangular), x += Z y
        y = torch.linalg.solve_triangular(H[:k, :k], torch.tensor(g[:k], dtype=torch.float64).reshape(-1, 1),
                                          upper=True).reshape(-1)
        for i in range(k):
            x = x + float(y[i]) * Z[i]
        restarts += 1


def gmres_hodlr(op, prec, b, tol: float = 1e-10, restart: int = 30, maxiter: int = 300) -> GmresResult:
    """GMRES on a HODLR operator ``op`` (HodlrMatrix, its device matvec) right-
    preconditioned by the solve of a HODLR factorization ``prec`` (typically a
    low-rank fp32 factorization of the same operator, BASELINE cfg4).  ``b``
    (N,) torch on op's device; the preconditioner runs in its own dtype."""
    from .hodlr import solve

    dt = op.D.dtype
    pdt = prec.D.dtype

    def precond(v):
        return solve(prec, v.to(pdt)).to(dt)

    return gmres(op.matvec, b.to(dt), precond=precond, tol=tol, restart=restart, maxiter=maxiter)
