"""Golden fixtures for the BASELINE operators: the reference's own factorize /
solve outputs on the exact inputs the GPU path factors.

    # build container (reference compress(), CPU only):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cfg_golden.py laplace
    # GPU box (the cfg1 operator is assembled by the device builder, whose exp()
    # differs from libm's in the last bit, so its inputs only exist there):
    python tests/golden/make_cfg_golden.py cfg1

* ``cfg2_laplace_sub14.npz`` -- the leading 2^14-row subtree (leaf 64, rank 32)
  of the cfg2 operator ``laplace_dl_oracle(contour_default(2^20))``, z = 0,
  compressed by the reference's own ``compress()`` (ACA rook, tol 0, max rank
  32; oracle/ref_driver.py ``ref_assemble_laplace``).  The device builder
  reproduces these inputs bit for bit (tests/test_gpu_build.py), which the
  parity test re-checks through ``in_sha``.
* ``cfg1_gaussian_n16384.npz`` -- BASELINE cfg1: exp(-|x-y|^2 / h^2) + I
  (h = 0.1) on 2^14 kd-ordered xorshift64* points in [0,1]^2, leaf 64, rank
  32, assembled on the device (``hb.gaussian_hodlr``); ``in_sha`` pins the
  device-assembled inputs.

Factorize / solve run through the reference's batched kernels
(``hodlr.backend``: ``batched_lu_factor_inplace``, ``batched_lu_solve_inplace``,
``batched_gemm``; oracle/ref_driver.py, the SPEC Alg. 3/4 recipe).  Stored:
the input digest, the rhs, x, leaf / K swaps (bit-exact gates) and random
sketches of Y and of the K LU factors (G^T Y, K_b g) -- the full 32 MB Y slab
does not fit a fixture; the parity test also compares full Y / K against the
oracle run live on the same inputs.
"""

from __future__ import annotations

import hashlib
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

N, M, R = 1 << 14, 64, 32
SKETCH_SEED = 20240
RHS_SEED = 4242


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sketches(Y, Kcat, n, r, L):
    """(r L) x 4 sketch of the Y slab and (nK) x 2 sketch of the K LU blocks."""
    rng = np.random.default_rng(SKETCH_SEED)
    G = rng.standard_normal((n, 4))
    g = rng.standard_normal((4 * r * r, 2))
    ys = Y.reshape(r * L, n) @ G
    ks = Kcat.reshape(-1, 4 * r * r) @ g
    return ys, ks


def run_reference(D, U, V, n, m, r, b):
    from oracle import ref_driver as rd

    assert rd.AVAILABLE, "the reference package (baseline/_ref or /root/reference/pkg/src) is required"
    L = int(round(math.log2(n // m)))
    D, Y, V = D.copy(), U.copy(), V.copy()
    ex = rd.executor(8)
    dpiv, Ks, kpivs = rd.ref_factorize(D, Y, V, n, m, r, L, ex)
    x = rd.ref_solve(D, dpiv, Y, V, Ks, kpivs, b, n, m, r, L, ex)
    Kcat = np.concatenate([Ks[lv] for lv in range(L)])
    ys, ks = sketches(Y, Kcat, n, r, L)
    return dict(
        x=x, d_swaps=dpiv.swaps.astype(np.int8), k_swaps=np.concatenate([kpivs[lv].swaps for lv in range(L)]).astype(np.int8),
        y_sketch=ys, k_sketch=ks, d_lu_sha=digest(D),
    )


def save(name, n, m, r, D, U, V, extra):
    b = np.random.default_rng(RHS_SEED).standard_normal((n, 1))
    out = run_reference(D, U, V, n, m, r, b)
    np.savez_compressed(HERE / name, n=n, m=m, r=r, in_sha=digest(D, U, V), b=b, sketch_seed=SKETCH_SEED, **out,
                        **extra)
    print("wrote", HERE / name, "x[:3] =", out["x"][:3, 0])


def laplace():
    from oracle import ref_driver as rd

    D, U, V = rd.ref_assemble_laplace(1 << 20, N, M, R)
    save("cfg2_laplace_sub14.npz", N, M, R, D, U, V, dict(kind="laplace_sub", n_total=1 << 20))


def cfg1():
    import torch

    import paper_2208_06290_b200 as hb

    h = hb.gaussian_hodlr(N, M, R, dim=2, h=0.1, lam=1.0)
    torch.cuda.synchronize()
    D, U, V = (t.cpu().numpy() for t in (h.D, h.U, h.V))
    save("cfg1_gaussian_n16384.npz", N, M, R, D, U, V, dict(kind="gaussian2d", h=0.1, lam=1.0, seed=0))
    out = REPO / "gpurun_out"
    if out.is_dir():
        import shutil

        shutil.copy(HERE / "cfg1_gaussian_n16384.npz", out / "cfg1_gaussian_n16384.npz")


if __name__ == "__main__":
    {"laplace": laplace, "cfg1": cfg1}[sys.argv[1]]()
