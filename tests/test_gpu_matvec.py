"""GPU: hodlr_matvec against the oracle.

Bars: fp64 within 1e-13 relative of the oracle's dense product;
fp32 within 1e-5; the SPEC known answers exactly; every column of a
multi-RHS product bit-identical to the single-vector product (the per-column
summation order depends only on the shape); the scalar-load path (m % 4 != 0
or misaligned slabs) equal to the vector path's answer within rounding.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import hodlr_oracle as orc  # noqa: E402
import paper_2208_06290_b200 as hb  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_gpu(h, dtype=None):
    hm = hb.HodlrMatrix.from_buffers(h.lay.n, h.lay.m, h.lay.r, h.D, h.U, h.V)
    if dtype is not None:
        hm = hb.HodlrMatrix(hm.tree, hm.rank, hm.D.to(dtype), hm.U.to(dtype), hm.V.to(dtype))
    return hm


def test_spec_known_answers():
    h = orc.HodlrData(orc.Layout(2, 1, 1), np.array([2.0, 2.0]), np.array([1.0, 1.0]), np.array([1.0, 1.0]))
    assert hb.HodlrMatrix.from_buffers(2, 1, 1, h.D, h.U, h.V).matvec(np.array([1.0, 1.0])).tolist() == [3.0, 3.0]
    n, m, r, L = 1024, 64, 8, 4
    eye = hb.HodlrMatrix.from_buffers(n, m, r, np.tile(np.eye(m).ravel(), 1 << L), np.zeros(n * r * L),
                                      np.zeros(n * r * L))
    x = np.random.default_rng(0).standard_normal(n)
    assert np.array_equal(eye.matvec(x), x)


@pytest.mark.parametrize("n,m,r", [(1024, 64, 8), (4096, 32, 16), (2048, 64, 32), (1536, 48, 8), (768, 6, 4),
                                   (512, 16, 1), (64, 64, 8), (8192, 16, 4)])
@pytest.mark.parametrize("nrhs", [1, 3, 11])
def test_matvec_vs_dense(n, m, r, nrhs):
    h = orc.make_exact_hodlr(n, m, r, seed=n + m + r, s=8.0)
    X = np.random.default_rng(nrhs).standard_normal((n, nrhs) if nrhs > 1 else n)
    y = to_gpu(h).matvec(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = orc.dense(h) @ X if n <= 4096 else orc.matvec(h, X)
    assert rel(y, ref) <= 1e-13


def test_matvec_columns_bitwise():
    h = orc.make_exact_hodlr(1 << 14, 64, 16, seed=7, s=4.0)
    hm = to_gpu(h)
    X = torch.randn(1 << 14, 13, dtype=torch.float64, device="cuda")
    Y = hm.matvec(X)
    for k in (0, 4, 8, 12):
        assert torch.equal(Y[:, k], hm.matvec(X[:, k].contiguous()))
    assert torch.equal(Y[:, :5], hm.matvec(X[:, :5].contiguous()))


def test_matvec_scalar_path_matches_vector_path():
    # a 1-scalar-offset view of the slabs forces the scalar-load kernels
    n, m, r = 4096, 64, 8
    h = orc.make_exact_hodlr(n, m, r, seed=11, s=2.0)
    hm = to_gpu(h)
    L = hm.L

    def shifted(t):
        buf = torch.empty(t.numel() + 1, dtype=t.dtype, device=t.device)
        buf[1:] = t
        return buf[1:]

    hs = hb.HodlrMatrix(hm.tree, r, shifted(hm.D), shifted(hm.U), shifted(hm.V))
    assert hs.V.data_ptr() % 32 != 0
    x = torch.randn(n, 2, dtype=torch.float64, device="cuda")
    assert rel(hs.matvec(x).cpu(), hm.matvec(x).cpu()) <= 1e-15
    assert L == 6


def test_matvec_fp32():
    n, m, r = 1 << 13, 64, 8
    h = orc.make_exact_hodlr(n, m, r, seed=3, s=4.0)
    x = np.random.default_rng(3).standard_normal((n, 2))
    y = to_gpu(h, torch.float32).matvec(torch.from_numpy(x).float().cuda()).double().cpu().numpy()
    assert rel(y, orc.matvec(h, x)) <= 1e-5


def test_matvec_large_linearity_and_solve_roundtrip():
    # cfg2-scale shape (N = 2^18 here to keep the test short): A (x1 + x2) = A x1 + A x2 within
    # rounding, and A (A^-1 b) = b to the solve's residual
    n, m, r = 1 << 18, 64, 32
    h = orc.make_exact_hodlr(n, m, r, seed=5, s=1.0)
    hm = to_gpu(h)
    g = torch.Generator(device="cuda").manual_seed(0)
    x1 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x2 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    lhs = hm.matvec(x1 + x2)
    assert float(torch.linalg.norm(lhs - hm.matvec(x1) - hm.matvec(x2)) / torch.linalg.norm(lhs)) <= 1e-14
    ref = orc.matvec(h, (x1 + x2).cpu().numpy())
    assert rel(lhs.cpu().numpy(), ref) <= 1e-13
    f = hb.factorize(hm.clone())
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x = hb.solve(f, b)
    assert float(torch.linalg.norm(hm.matvec(x) - b) / torch.linalg.norm(b)) <= 1e-12


def test_matvec_errors():
    h = orc.make_exact_hodlr(1024, 64, 8, seed=1)
    hm = to_gpu(h)
    with pytest.raises(ValueError):
        hm.matvec(torch.zeros(1000, dtype=torch.float64, device="cuda"))


def test_refinement_spec_examples():
    n, m, r = 4096, 64, 16
    h = orc.make_exact_hodlr(n, m, r, seed=21, s=2.0)
    hm = to_gpu(h)
    f = hb.factorize(hm.clone())
    # b = 0 -> x = 0 immediately
    res = hb.solve_with_refinement(f, hm, np.zeros(n))
    assert res.iterations == 0 and not res.x.any()
    # exact factorization: converged after the first solve (relres at rounding level), at most
    # the two stall iterations follow and do not improve materially
    b = np.random.default_rng(1).standard_normal(n)
    res = hb.solve_with_refinement(f, hm, b, max_iters=5)
    assert res.history[0] <= 1e-13 and min(res.history) <= res.history[0]
    assert rel(orc.dense(h) @ res.x, b) <= 1e-13 and not res.diverged


def test_refinement_fp32_preconditioner_reaches_fp64():
    # cfg4-style: fp32 factorization as the preconditioner, fp64 operator for the residual
    n, m, r = 1 << 16, 64, 8
    h = orc.make_exact_hodlr(n, m, r, seed=4, s=4.0)
    h64 = to_gpu(h)
    f32 = hb.factorize(to_gpu(h, torch.float32))
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    res = hb.solve_with_refinement(f32, h64, b, max_iters=8)
    hist = res.history
    assert hist[0] > 1e-8  # fp32 accuracy after the first solve
    assert all(hist[k + 1] < hist[k] for k in range(3))  # monotone for >= 3 iterations
    assert min(hist) <= 1e-13 and not res.diverged
    assert float(torch.linalg.norm(h64.matvec(res.x) - b) / torch.linalg.norm(b)) == pytest.approx(min(hist))


def test_concurrent_solves_on_two_streams():
    # solve is safe to call concurrently on one factorization with
    # distinct right-hand sides (per-stream workspaces)
    n, m, r = 1 << 15, 64, 32
    f = hb.factorize(hb.random_hodlr(n, m, r, seed=9))
    g = torch.Generator(device="cuda").manual_seed(3)
    b1 = torch.randn(n, 3, dtype=torch.float64, device="cuda", generator=g)
    b2 = torch.randn(n, 3, dtype=torch.float64, device="cuda", generator=g)
    x1_ref, x2_ref = hb.solve(f, b1), hb.solve(f, b2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        x1 = hb.solve(f, b1, stream=s1)
        x2 = hb.solve(f, b2, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(x1, x1_ref) and torch.equal(x2, x2_ref)


def test_dump_load_roundtrip_matrix_and_factorization(tmp_path):
    # SPEC.md:215 binary format: the reloaded matrix / factorization are bit-identical and
    # the reloaded factorization solves without refactoring (factor once, solve many)
    n, m, r = 1 << 12, 64, 16
    h = hb.random_hodlr(n, m, r, seed=12, s=4.0)
    hb.dump(h, tmp_path / "h.hodlr")
    h2 = hb.load(tmp_path / "h.hodlr")
    assert torch.equal(h.D, h2.D) and torch.equal(h.U, h2.U) and torch.equal(h.V, h2.V)
    f = hb.factorize(h.clone())
    hb.dump(f, tmp_path / "f.hodlr")
    f2 = hb.load(tmp_path / "f.hodlr")
    b = torch.randn(n, 3, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    assert torch.equal(hb.solve(f, b), hb.solve(f2, b))
    assert hb.logdet(f) == hb.logdet(f2)
    h32 = hb.random_hodlr(n, m, 8, seed=3, dtype=torch.float32)
    f32 = hb.factorize(h32)
    hb.dump(f32, tmp_path / "f32.hodlr")
    assert torch.equal(hb.solve(f32, b.float()), hb.solve(hb.load(tmp_path / "f32.hodlr"), b.float()))


def test_hodlr_bench_cli_cells(tmp_path):
    # SPEC.md:537-574 harness on the device: records, the 14 CSV columns, and byte-identical
    # output (timing columns excluded) for identical config + seed
    from paper_2208_06290_b200 import cli

    cfg = tmp_path / "cells.txt"
    cfg.write_text("[cell]\nproblem=laplace\nn=4096\nrank=16\nruns=2\n[cell]\nproblem=standin\nn=4096\nrank=16\n"
                   "precision=single\nruns=2\n")
    outs = []
    for k in range(2):
        out = tmp_path / f"r{k}.csv"
        assert cli.main(["--config", str(cfg), "--out", str(out), "--seed", "3"]) == 0
        recs = cli.parse_results(out.read_text(), "csv")
        assert [r["problem"] for r in recs] == ["laplace", "standin"]
        assert recs[0]["relres"] < 1e-13 and recs[1]["relres"] < 1e-5
        assert recs[0]["ranks"] == "/".join(["16"] * 6)
        for r in recs:
            r.pop("t_f_seconds"), r.pop("t_s_seconds")
        outs.append(recs)
    assert outs[0] == outs[1]
