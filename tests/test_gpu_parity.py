"""GPU parity: the sm_100a path vs the CPU oracle and the reference golden vectors.

Bars (BASELINE.json north_star): leaf/K pivot indices bit-exact, leaf LU
factors bit-exact (the kernel replays the reference's IEEE op order), Y / K /
x within 1e-10 relative (fp64) of the oracle, which is itself bit-identical to
the reference kernels (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import hodlr_oracle as orc  # noqa: E402
import paper_2208_06290_b200 as hb  # noqa: E402
from tests.conftest import record_parity  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden"
TOL = 1e-10  # fp64 solution / factor agreement (north_star)
SENS_MULT = 4.0  # hard-pivoting (s = 16) inputs only: gate = max(TOL, 4 x the oracle's own 1-ulp sensitivity)


def gate(s: float, sens: float) -> float:
    """North-star 1e-10 for well-conditioned inputs (U scale s <= 4); for the
    s = 16 stress regime (cond ~2e4, ~80 % real K pivot choices) any
    non-OpenBLAS summation order moves Y / x by the oracle's own 1-ulp
    sensitivity, so the gate is max(1e-10, 4 x that sensitivity)."""
    return TOL if s <= 4 else max(TOL, SENS_MULT * sens)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_gpu(h: orc.HodlrData) -> hb.HodlrMatrix:
    return hb.HodlrMatrix.from_buffers(h.lay.n, h.lay.m, h.lay.r, h.D, h.U, h.V)


def golden_cases():
    return sorted(p for p in GOLDEN.glob("n*.npz"))


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.stem)
def test_golden_factor_and_solve(path):
    g = np.load(path)
    n, m, r = int(g["n"]), int(g["m"]), int(g["r"])
    h = orc.make_exact_hodlr(n, m, r, seed=int(g["seed"]), s=float(g["s"]))
    f = hb.factorize(to_gpu(h))
    L = f.L
    # leaf LU: factors and pivots bit-exact
    assert np.array_equal(f.D.cpu().numpy(), g["D_lu"])
    assert np.array_equal(f.dperm.cpu().numpy().reshape(-1, m), g["d_perm"])
    assert np.array_equal(f.dswaps.cpu().numpy().reshape(-1, m), g["d_swaps"])
    # K pivots bit-exact, Y and K factors to tolerance
    assert np.array_equal(f.kswaps.cpu().numpy().reshape(-1, 2 * r), g["k_swaps"])
    assert np.array_equal(f.kperm.cpu().numpy().reshape(-1, 2 * r), g["k_perm"])
    _, sy, sx = oracle_sensitivity(h, g["b"])
    s = float(g["s"])
    x = hb.solve(f, g["b"])
    ey, ek, ex = rel(f.Y.cpu().numpy(), g["Y"]), rel(f.K.cpu().numpy(), g["K"]), rel(x, g["x"])
    record_parity(f"golden/{path.stem}", y=ey, k=ek, x=ex, gate_y=gate(s, sy), gate_x=gate(s, sx), sens_y=sy, sens_x=sx)
    assert ey <= gate(s, sy)
    assert ek <= gate(s, sy)
    assert ex <= gate(s, sx)
    la, sg = hb.logdet(f)
    assert sg == float(g["logdet_sign"])
    assert abs(la - float(g["logdet"])) <= 1e-10 * abs(float(g["logdet"]))
    assert L == int(round(math.log2(n // m)))


def test_spec_2x2_worked_example():
    # [[2,1],[1,2]], tree(2,1)
    h = hb.HodlrMatrix.from_buffers(2, 1, 1, np.array([2.0, 2.0]), np.array([1.0, 1.0]), np.array([1.0, 1.0]))
    f = hb.factorize(h)
    assert f.Y.cpu().tolist() == [0.5, 0.5]
    g = np.load(GOLDEN / "spec_2x2.npz")
    assert f.K.cpu().numpy().tolist() == g["K_lu"].tolist()
    x = hb.solve(f, np.array([3.0, 3.0]))
    assert np.allclose(x, [1.0, 1.0], rtol=0, atol=1e-15)
    la, sg = hb.logdet(f)
    assert abs(la - math.log(3.0)) < 1e-15 and sg == 1.0


def test_identity_hodlr_solves_to_b():
    n, m, r = 256, 32, 4
    L = 3
    D = np.zeros((1 << L) * m * m)
    for a in range(1 << L):
        D[a * m * m + np.arange(m) * (m + 1)] = 1.0
    U = np.zeros(n * r * L)
    V = np.zeros(n * r * L)
    f = hb.factorize(hb.HodlrMatrix.from_buffers(n, m, r, D, U, V))
    b = np.random.default_rng(0).standard_normal(n)
    assert np.array_equal(hb.solve(f, b), b)
    assert hb.logdet(f) == (0.0, 1.0)


def oracle_sensitivity(h, b):
    """Relative change of the oracle's Y and x when U is perturbed by ~1 ulp.

    Any implementation that is not bit-identical to OpenBLAS (different GEMM
    summation order) can only agree with the oracle to about this level, so the
    1e-10 gate is applied as max(1e-10, 4 x sensitivity) on the hard-pivoting
    s = 16 inputs only (their K blocks amplify rounding); s <= 4 uses 1e-10.
    """
    f1 = orc.factorize(h.copy(), threads=8)
    h2 = h.copy()
    h2.U *= 1 + 1e-16 * np.random.default_rng(0).standard_normal(h2.U.size)
    f2 = orc.factorize(h2, threads=8)
    sy = rel(f2.Y, f1.Y)
    sx = rel(orc.solve(f2, b, threads=8), orc.solve(f1, b, threads=8))
    return f1, sy, sx


@pytest.mark.parametrize(
    "n,m,r,s",
    [(1 << 14, 64, 32, 4.0), (1 << 14, 64, 32, 16.0), (1 << 13, 64, 16, 1.0), (1 << 12, 32, 8, 16.0),
     (1 << 11, 16, 32, 16.0), (1 << 12, 64, 64, 2.0), (1 << 14, 64, 64, 16.0), (1 << 13, 32, 32, 4.0),
     (1 << 13, 32, 16, 16.0)],
)
def test_random_vs_oracle(n, m, r, s):
    h = orc.make_exact_hodlr(n, m, r, seed=n + r, s=s)
    b = np.random.default_rng(1).standard_normal((n, 2))
    fo, sy, sx = oracle_sensitivity(h, b)
    f = hb.factorize(to_gpu(h))
    # bit-exact: leaf factors, leaf pivots, K pivots
    assert np.array_equal(f.D.cpu().numpy(), fo.D)
    assert np.array_equal(f.dperm.cpu().numpy().reshape(-1, m), fo.dpiv.perm)
    ks = f.kswaps.cpu().numpy().reshape(-1, 2 * r)
    assert np.array_equal(ks, np.concatenate([kp.swaps for kp in fo.kpiv]))
    x = hb.solve(f, b)
    ey, ek = rel(f.Y.cpu().numpy(), fo.Y), rel(f.K.cpu().numpy(), np.concatenate(fo.K))
    ex = rel(x, orc.solve(fo, b, threads=8))
    record_parity(f"random/n{n}_m{m}_r{r}_s{s:g}", y=ey, k=ek, x=ex, gate_y=gate(s, sy), gate_x=gate(s, sx),
                  sens_y=sy, sens_x=sx)
    assert ey <= gate(s, sy)
    assert ek <= gate(s, sy)
    assert ex <= gate(s, sx)
    # relative residual against the HODLR operator itself, vs the oracle's own
    hm = to_gpu(h)
    bt = torch.from_numpy(b).cuda()

    def relres(xx):
        return float(torch.linalg.norm(hm.matvec(torch.from_numpy(xx).cuda()) - bt) / torch.linalg.norm(bt))

    assert relres(x) <= max(1e-12, 4 * relres(orc.solve(fo, b, threads=8)))


@pytest.mark.parametrize("nrhs", [5, 12, 16, 20, 27, 40, 64, 72, 131, 257])
@pytest.mark.parametrize("r", [16, 32, 64])
def test_multi_rhs_columns_bitwise_equal_single(nrhs, r):
    # column j of a blocked solve == single-vector solve, bit for bit
    # (<= 24/32 columns: the warp-specialized TMA solve step; more: the shared-panel
    # kernels; rank 32 with >= 128 columns: level_update6 in solve mode for the
    # leading 16-group blocks + the shared-panel kernel for the rest)
    n, m = 1 << 13, 64
    h = hb.random_hodlr(n, m, r, seed=3, s=16.0)
    f = hb.factorize(h)
    B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    X = hb.solve(f, B)
    for j in range(nrhs):
        xj = hb.solve(f, B[:, j].contiguous())
        assert torch.equal(X[:, j], xj), j


def test_solve_does_not_mutate_b_and_is_linear():
    n, m, r = 1 << 12, 64, 16
    f = hb.factorize(hb.random_hodlr(n, m, r, seed=4))
    g = torch.Generator("cuda").manual_seed(5)
    b1 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    b2 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    keep = b1.clone()
    x1, x2 = hb.solve(f, b1), hb.solve(f, b2)
    assert torch.equal(b1, keep)
    x12 = hb.solve(f, 2.0 * b1 - 3.0 * b2)
    assert float(torch.linalg.norm(x12 - (2 * x1 - 3 * x2)) / torch.linalg.norm(x12)) < 1e-12


def test_factorize_deterministic_run_to_run():
    n, m, r = 1 << 14, 64, 32
    h1 = hb.random_hodlr(n, m, r, seed=9, s=16.0)
    h2 = h1.clone()
    f1, f2 = hb.factorize(h1), hb.factorize(h2)
    assert torch.equal(f1.Y, f2.Y) and torch.equal(f1.K, f2.K) and torch.equal(f1.kswaps, f2.kswaps)


def test_single_leaf_tree():
    # L = 0: the whole matrix is one dense leaf block
    n = m = 48
    rng = np.random.default_rng(6)
    D = rng.standard_normal(m * m) + 8 * np.eye(m).ravel()
    f = hb.factorize(hb.HodlrMatrix.from_buffers(n, m, 4, D, np.zeros(0), np.zeros(0)))
    b = rng.standard_normal(n)
    x = hb.solve(f, b)
    A = D.reshape(m, m).T
    assert rel(x, np.linalg.solve(A, b)) < 1e-13


def test_singular_leaf_raises_with_level_and_node():
    n, m, r = 256, 32, 4
    h = orc.make_exact_hodlr(n, m, r, seed=1)
    h.D[3 * m * m : 4 * m * m] = 0.0  # leaf 3 is the zero matrix
    with pytest.raises(hb.HodlrSingularError, match=r"leaf block at level 3, node\(s\) \[3\]"):
        hb.factorize(to_gpu(h))


@pytest.mark.parametrize("n,m,r", [(1 << 13, 64, 8), (1 << 12, 32, 16)])
def test_fp32_preconditioner_path_vs_oracle(n, m, r):
    # cfg4 path (rank-8 fp32 HODLR): bit-exact fp32 leaf LU + pivots, <= 1e-4 elsewhere (north star)
    h = orc.make_exact_hodlr(n, m, r, seed=n + r, s=1.0, dtype=np.float32)
    b = np.random.default_rng(2).standard_normal((n, 3)).astype(np.float32)
    fo = orc.factorize(h.copy(), threads=8)
    f = hb.factorize(to_gpu(h))
    assert f.D.dtype == torch.float32
    assert np.array_equal(f.D.cpu().numpy(), fo.D)
    assert np.array_equal(f.dperm.cpu().numpy().reshape(-1, m), fo.dpiv.perm)
    ks = f.kswaps.cpu().numpy().reshape(-1, 2 * r)
    assert np.array_equal(ks, np.concatenate([kp.swaps for kp in fo.kpiv]))
    x = hb.solve(f, b)
    assert x.dtype == np.float32
    ey, ex = rel(f.Y.cpu().numpy(), fo.Y), rel(x, orc.solve(fo, b, threads=8))
    record_parity(f"fp32/n{n}_m{m}_r{r}", y=ey, x=ex, gate_x=1e-4)
    assert ey <= 1e-4
    assert ex <= 1e-4


def test_fp32_multi_rhs_columns_bitwise_equal_single():
    n, m, r = 1 << 13, 64, 8
    h = hb.random_hodlr(n, m, r, seed=5, s=1.0, dtype=torch.float32)
    f = hb.factorize(h)
    B = torch.randn(n, 20, dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    X = hb.solve(f, B)
    for j in (0, 7, 19):
        assert torch.equal(X[:, j], hb.solve(f, B[:, j].contiguous())), j
    for k in (2, 3, 6):  # the 2- / 4- / 8-column level kernels and the warp getrs
        assert torch.equal(X[:, :k], hb.solve(f, B[:, :k].contiguous())), k


def test_factorize_from_host_equals_device_path():
    # streamed-upload factorization == factorize(from_buffers(...)) bit for bit
    n, m, r = 1 << 13, 64, 32
    h = orc.make_exact_hodlr(n, m, r, seed=21, s=4.0)
    f1 = hb.factorize(to_gpu(h))
    Dh, Uh, Vh = (torch.from_numpy(x).pin_memory() for x in (h.D, h.U, h.V))
    f2 = hb.factorize_from_host(n, m, r, Dh, Uh, Vh)
    for name in ("D", "Y", "K", "kswaps", "dperm"):
        assert torch.equal(getattr(f1, name), getattr(f2, name)), name
    b = np.random.default_rng(3).standard_normal(n)
    assert np.array_equal(hb.solve(f1, b), hb.solve(f2, b))


@pytest.mark.parametrize("pinned_d", [False, True])
def test_factorize_from_host_pageable_equals_device_path(pinned_d):
    # pageable (numpy) inputs stream through the pinned staging ring (369 MB
    # slabs: several 64 MB chunks, the 4-slot ring wraps) while a second host
    # thread enqueues the factorization; also mixed pinned / pageable inputs
    n, m, r = 1 << 17, 64, 32
    h = hb.random_hodlr(n, m, r, seed=5, s=4.0)
    Dn, Un, Vn = (x.cpu().numpy().copy() for x in (h.D, h.U, h.V))
    f1 = hb.factorize(h.clone())
    Dh = torch.from_numpy(Dn).pin_memory() if pinned_d else Dn
    f2 = hb.factorize_from_host(n, m, r, Dh, Un, Vn)
    del Dn, Un, Vn  # the call returns once the host buffers have been consumed
    for name in ("D", "Y", "K", "kswaps", "dperm"):
        assert torch.equal(getattr(f1, name), getattr(f2, name)), name


@pytest.mark.parametrize("nrhs", [1, 3, 20])
def test_solve_graph_replay_bitwise_equals_eager(nrhs):
    # the CUDA-graph solve (captured once per (nrhs, stream), replayed) == the eager launches
    n, m, r = 1 << 13, 64, 32
    f = hb.factorize(hb.random_hodlr(n, m, r, seed=31, s=4.0))
    g = torch.Generator("cuda").manual_seed(7)
    for _ in range(3):  # first call captures, later calls replay with new right-hand sides
        B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda", generator=g)
        keep = B.clone()
        xg = hb.solve(f, B, graph=True)
        xe = hb.solve(f, B, graph=False)
        assert torch.equal(xg, xe)
        assert torch.equal(B, keep)


def test_factor_plan_refactor_bitwise_equals_factorize():
    # FactorPlan: eager factorization + captured graph; refactor() after loading new entries
    n, m, r = 1 << 13, 64, 32
    h1 = hb.random_hodlr(n, m, r, seed=41, s=16.0)
    h2 = hb.random_hodlr(n, m, r, seed=42, s=16.0)
    plan = hb.FactorPlan(h1.clone())
    for h in (h1, h2, h1):
        plan.load(h.D, h.U, h.V)
        fp = plan.refactor()
        fr = hb.factorize(h.clone())
        for name in ("D", "Y", "K", "kswaps", "dperm", "Dinv", "Kinv"):
            assert torch.equal(getattr(fp, name), getattr(fr, name)), name
        b = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
        assert torch.equal(hb.solve(fp, b), hb.solve(fr, b))


def test_factor_plan_raises_on_singular_refactor():
    n, m, r = 1 << 10, 32, 8
    h = hb.random_hodlr(n, m, r, seed=5)
    plan = hb.FactorPlan(h.clone())
    D = h.D.clone()
    D[5 * m * m : 6 * m * m] = 0.0
    plan.load(D, h.U, h.V)
    with pytest.raises(hb.HodlrSingularError, match=r"leaf block at level 5, node\(s\) \[5\]"):
        plan.refactor()


def test_ragged_level_panels_vs_oracle_on_the_padded_layout():
    # SPEC.md:147-160 ragged panels (per-node ranks 0..24, scattered column offsets) ingested by
    # HodlrMatrix.from_level_panels (zero-pad to rank 32, the fused-kernel rank): K pivots bit-exact
    # vs the oracle on the same padded layout, x within 1e-10, and the ragged dense matrix solved
    from tests.test_ragged_cpu import ragged

    n, m, L = 1 << 12, 64, 6
    D, ups, vps, A = ragged(n, m, L, seed=5, width=32, kmax=24)
    h = hb.HodlrMatrix.from_level_panels(n, m, D, ups, vps, per_level=False)
    assert h.rank == 32 and h.ranks is None
    r, U, V = hb.pad_level_panels(n, m, ups, vps)
    fo = orc.factorize(orc.HodlrData(orc.Layout(n, m, r), D.copy(), U, V))
    f = hb.factorize(h)
    assert np.array_equal(f.kswaps.cpu().numpy().reshape(-1, 2 * r), np.concatenate([p.swaps for p in fo.kpiv]))
    b = np.random.default_rng(2).standard_normal(n)
    x = hb.solve(f, b)
    ex = rel(x, orc.solve(fo, b.reshape(-1, 1))[:, 0])
    record_parity("ragged/n4096_m64_kmax24_pad32", x=ex, gate_x=TOL)
    assert ex <= TOL
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
