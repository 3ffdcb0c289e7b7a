"""GPU parity on the BASELINE operators themselves (BASELINE.json configs[0] /
configs[1]): the device factorization vs the REFERENCE's own factorize/solve
outputs on the same inputs (tests/golden/make_cfg_golden.py), and vs the oracle
run live on those inputs for the full Y slab and K factors.

Gates (north_star): leaf / K pivots bit-exact, leaf LU bit-exact, x / Y / K
within 1e-10 relative (fp64)."""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2208_06290_b200 as hb  # noqa: E402
from oracle import hodlr_oracle as orc  # noqa: E402
from tests.conftest import record_parity  # noqa: E402
from tests.golden.make_cfg_golden import digest, sketches  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden"
TOL = 1e-10


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def subtree(h, n_sub):
    """Leading n_sub-row subtree of a device HODLR (numpy D, U, V; SPEC layout)."""
    m, r, L, n = h.m, h.rank, h.L, h.n
    Ls = int(round(math.log2(n_sub // m)))
    D = h.D[: (n_sub // m) * m * m].cpu().numpy()
    U = h.U.view(L, r, n)[L - Ls :, :, :n_sub].contiguous().view(-1).cpu().numpy()
    V = h.V.view(L, r, n)[L - Ls :, :, :n_sub].contiguous().view(-1).cpu().numpy()
    return D, U, V


def check_against_reference(name, g, D, U, V):
    n, m, r = int(g["n"]), int(g["m"]), int(g["r"])
    L = int(round(math.log2(n // m)))
    assert digest(D, U, V) == str(g["in_sha"]), "inputs differ from the fixture's"
    f = hb.factorize(hb.HodlrMatrix.from_buffers(n, m, r, D, U, V))
    # bit-exact: leaf LU factors, leaf and K pivots
    assert digest(f.D.cpu().numpy()) == str(g["d_lu_sha"])
    assert np.array_equal(f.dswaps.cpu().numpy().reshape(-1, m), g["d_swaps"])
    assert np.array_equal(f.kswaps.cpu().numpy().reshape(-1, 2 * r), g["k_swaps"])
    x = hb.solve(f, g["b"])
    Y, K = f.Y.cpu().numpy(), f.K.cpu().numpy()
    ys, ks = sketches(Y, K, n, r, L)
    ex, eys, eks = rel(x, g["x"]), rel(ys, g["y_sketch"]), rel(ks, g["k_sketch"])
    # full Y / K vs the oracle on the same inputs (bit-identical to the reference kernels)
    fo = orc.factorize(orc.HodlrData(orc.Layout(n, m, r), D.copy(), U.copy(), V.copy()), threads=8)
    assert np.array_equal(orc.solve(fo, g["b"], threads=8), g["x"])  # the oracle reproduces the reference here
    ey, ek = rel(Y, fo.Y), rel(K, np.concatenate(fo.K))
    hm = hb.HodlrMatrix.from_buffers(n, m, r, D, U, V)
    bt = torch.from_numpy(g["b"]).cuda()
    relres = float(torch.linalg.norm(hm.matvec(torch.from_numpy(x).cuda()) - bt) / torch.linalg.norm(bt))
    record_parity(name, x=ex, y=ey, k=ek, y_sketch=eys, k_sketch=eks, relres=relres, gate_x=TOL)
    assert ex <= TOL and ey <= TOL and ek <= TOL and eys <= TOL and eks <= TOL, (ex, ey, ek, eys, eks)
    assert relres <= 1e-13


def test_cfg2_laplace_subtree_vs_reference():
    # the leading 2^14-row subtree of the bench workload (cfg2 operator at N = 2^20), device-assembled
    g = np.load(GOLDEN / "cfg2_laplace_sub14.npz")
    h = hb.laplace_dl_hodlr(int(g["n_total"]), int(g["m"]), int(g["r"]))
    D, U, V = subtree(h, int(g["n"]))
    del h
    torch.cuda.empty_cache()
    check_against_reference("baseline/cfg2_laplace_sub14", g, D, U, V)


def test_cfg1_gaussian_vs_reference():
    # BASELINE cfg1: Gaussian kernel on 2^14 2-D points, leaf 64, rank 32, device-assembled
    p = GOLDEN / "cfg1_gaussian_n16384.npz"
    if not p.exists():
        pytest.skip("fixture not generated (python tests/golden/make_cfg_golden.py cfg1 on a GPU box)")
    g = np.load(p)
    h = hb.gaussian_hodlr(int(g["n"]), int(g["m"]), int(g["r"]), dim=2, h=float(g["h"]), lam=float(g["lam"]),
                          seed=int(g["seed"]))
    D, U, V = (t.cpu().numpy() for t in (h.D, h.U, h.V))
    check_against_reference("baseline/cfg1_gaussian_n16384", g, D, U, V)
