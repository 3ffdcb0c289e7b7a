"""The reference's batched-kernel tests (pkg/tests/test_backend.py) run against
the sm_100a executor.  LU factors/pivots must be bit-identical to the oracle's
restatement of backend.py:444-478; GEMM/solve values agree to rounding
(different summation order from OpenBLAS)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import hodlr_oracle as orc  # noqa: E402
from paper_2208_06290_b200 import (  # noqa: E402
    BlockBatch,
    BlockRef,
    SingularBlockError,
    batched_gemm,
    batched_lu_factor_inplace,
    batched_lu_solve_inplace,
    gemm_stacks,
    grouped_gemm_large,
    lu_solve_stacks,
)


def make_block(arr):
    a = np.asarray(arr)
    buf = np.asfortranarray(a).ravel(order="F").copy()
    return BlockRef(buf, 0, a.shape[0], a.shape[1], a.shape[0])


def test_gemm_one_by_one():  # test_backend.py:73-76
    a, b, c = make_block([[2.0]]), make_block([[3.0]]), make_block([[0.0]])
    batched_gemm([(a, b, c)])
    assert c.view()[0, 0] == 6.0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gemm_batch_matches_sequential(dtype):  # :87-98 (relaxed to rounding)
    rng = np.random.default_rng(7)
    items, refs = [], []
    for _ in range(8):
        a, b = rng.standard_normal((16, 16)).astype(dtype), rng.standard_normal((16, 16)).astype(dtype)
        items.append((make_block(a), make_block(b), make_block(np.zeros((16, 16), dtype=dtype))))
        refs.append(a @ b)
    batched_gemm(items)
    tol = 1e-14 if dtype == np.float64 else 2e-5
    for (_, _, c), want in zip(items, refs):
        assert c.view().dtype == dtype
        np.testing.assert_allclose(c.view(), want, rtol=tol, atol=tol)


def test_gemm_fp32_conj_transpose_long_k_split():
    # fp32 transA with a long reduction (the fixed-order split-K path)
    rng = np.random.default_rng(8)
    a = rng.standard_normal((4096, 8)).astype(np.float32)
    b = rng.standard_normal((4096, 24)).astype(np.float32)
    c = make_block(np.zeros((8, 24), dtype=np.float32))
    batched_gemm([(make_block(a), make_block(b), c)], transpose_a="conj_transpose")
    want = a.astype(np.float64).T @ b.astype(np.float64)
    assert np.abs(c.view() - want).max() <= 1e-4 * np.abs(want).max()


def test_gemm_accumulate_and_alpha_beta():  # :101-110
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal((5, 4)), rng.standard_normal((4, 6))
    c0 = rng.standard_normal((5, 6))
    c = make_block(c0)
    batched_gemm([(make_block(a), make_block(b), c)], alpha=-1.0, beta=1.0)
    assert np.allclose(c.view(), c0 - a @ b, atol=1e-14)
    c2 = make_block(c0)
    batched_gemm([(make_block(a), make_block(b), c2)], alpha=0.5, beta=2.0)
    assert np.allclose(c2.view(), 2.0 * c0 + 0.5 * (a @ b), atol=1e-14)


def test_gemm_conj_transpose_real_and_long_k():
    rng = np.random.default_rng(19)
    a = rng.standard_normal((70000, 32))  # long K exercises the split-K tree
    b = rng.standard_normal((70000, 40))
    c = make_block(np.zeros((32, 40)))
    batched_gemm([(make_block(a), make_block(b), c)], transpose_a="conj_transpose")
    np.testing.assert_allclose(c.view(), a.T @ b, rtol=1e-12, atol=1e-11)


def test_gemm_strided_fast_path_equals_generic():  # :134-158
    rng = np.random.default_rng(11)
    B, m, k, n = 6, 9, 5, 7
    abuf, bbuf = rng.standard_normal(B * m * k), rng.standard_normal(B * k * n)
    c1, c2 = np.zeros(B * m * n), np.zeros(B * m * n)
    mk = lambda cb: [  # noqa: E731
        (BlockRef(abuf, i * m * k, m, k, m), BlockRef(bbuf, i * k * n, k, n, k), BlockRef(cb, i * m * n, m, n, m))
        for i in range(B)
    ]
    batched_gemm(BlockBatch(mk(c1)))
    sh = mk(c2)
    batched_gemm([sh[i] for i in (3, 0, 5, 1, 4, 2)])
    assert c1.tobytes() == c2.tobytes()


def test_gemm_device_buffers_and_paired_layout():
    # paired-child offsets (b//2)*hi + (b%2)*lo, as in the level GEMMs
    rng = np.random.default_rng(2)
    r, nc, ncol, nch = 8, 64, 24, 8
    V = torch.from_numpy(rng.standard_normal(nch * nc * r)).cuda()
    Y = torch.from_numpy(rng.standard_normal(nch * nc * ncol)).cuda()
    TW = torch.zeros((nch // 2) * 2 * r * ncol, dtype=torch.float64, device="cuda")
    N = nch * nc
    items = [
        (BlockRef(V, c * nc, nc, r, N), BlockRef(Y, c * nc, nc, ncol, N),
         BlockRef(TW, (c // 2) * 2 * r * ncol + (c % 2) * r, r, ncol, 2 * r))
        for c in range(nch)
    ]
    batched_gemm(items, transpose_a="conj_transpose")
    Vn, Yn, T = V.cpu().numpy(), Y.cpu().numpy(), TW.cpu().numpy()
    for c in range(nch):
        want = orc.bview(Vn, c * nc, nc, r, N).T @ orc.bview(Yn, c * nc, nc, ncol, N)
        got = orc.bview(T, (c // 2) * 2 * r * ncol + (c % 2) * r, r, ncol, 2 * r)
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)


def test_gemm_stacks_and_grouped():  # :182-201, :227-253
    rng = np.random.default_rng(17)
    a, b = rng.standard_normal((5, 8, 3)), rng.standard_normal((5, 3, 4))
    c = np.zeros((5, 8, 4))
    gemm_stacks(a, b, c)
    np.testing.assert_allclose(c, a @ b, rtol=1e-14, atol=1e-14)
    a2, b2 = rng.standard_normal((512, 8)), rng.standard_normal((8, 512))
    c1, c2 = make_block(np.zeros((512, 512))), make_block(np.zeros((512, 512)))
    batched_gemm([(make_block(a2), make_block(b2), c1)])
    grouped_gemm_large([(make_block(a2), make_block(b2), c2)], inner_threads=4)
    assert c1.view().tobytes() == c2.view().tobytes()


def test_lu_known_answers():  # :261-275
    b = make_block([[2.0]])
    piv, _ = batched_lu_factor_inplace([b])
    assert b.view()[0, 0] == 2.0 and piv.swaps.tolist() == [[0]] and not piv.singular
    p = make_block(np.array([[0.0, 1.0], [1.0, 0.0]]))
    piv, _ = batched_lu_factor_inplace([p])
    assert piv.swaps[0].tolist() == [1, 1]
    assert np.array_equal(p.view(), np.eye(2))
    assert piv.sign()[0] == -1.0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("s,nb", [(16, 12), (32, 12), (64, 12), (128, 12), (64, 2053)])
def test_lu_nonfinite_and_degenerate_blocks_bit_exact(s, nb, dtype):
    # NaN wins the pivot search (np.argmax), +-inf, exact ties, zero columns, duplicate
    # rows (singular flags) -- factors (NaN-aware), pivots and flags as the reference;
    # nb > 2048: the full-wave register-row kernel (blocks in lockstep per CTA, ragged tail)
    rng = np.random.default_rng(s)
    base = rng.standard_normal((nb, s, s))
    base[0, 3, 0] = np.nan
    base[1, :, 2] = 0.0
    base[2, 5, :] = base[2, 1, :]
    base[3, 2, 1] = np.inf
    base[4, 7, 0] = -np.inf
    base[5] = np.round(base[5])  # many exact ties
    base[6, :, :] = 0.0  # all-zero block
    base[7, 4, 4] = np.nan
    base[8] *= 1e-300 if dtype == np.float64 else 1e-37  # tiny values (subnormal multipliers)
    base[9, :, 0] = base[9, 0, 0]  # every candidate ties on the first pivot
    flat = np.ascontiguousarray(base.transpose(0, 2, 1)).astype(dtype).ravel()  # column-major blocks
    buf = flat.copy()
    with np.errstate(all="ignore"):
        piv, _ = batched_lu_factor_inplace([BlockRef(buf, i * s * s, s, s, s) for i in range(nb)])
        ref = flat.copy()
        p = orc.lu_factor(orc.sview(ref, 0, s * s, nb, s, s, s))
    assert np.array_equal(buf, ref, equal_nan=True)
    assert np.array_equal(piv.swaps, p.swaps) and np.array_equal(piv.perm, p.perm)
    assert sorted(piv.singular) == sorted(np.flatnonzero(p.singular).tolist())


@pytest.mark.parametrize("s,nb", [(64, 512), (64, 296), (64, 1), (64, 4099), (32, 300), (32, 148), (16, 1000), (128, 40), (128, 300), (7, 33)])
def test_lu_bit_exact_vs_reference_order(s, nb):
    rng = np.random.default_rng(s * 1000 + nb)
    base = rng.standard_normal(nb * s * s)
    base[: s * s] = np.round(base[: s * s])  # ties in pivot search for block 0
    buf = base.copy()
    piv, fl = batched_lu_factor_inplace([BlockRef(buf, i * s * s, s, s, s) for i in range(nb)])
    ref = base.copy()
    p = orc.lu_factor(orc.sview(ref, 0, s * s, nb, s, s, s))
    assert buf.tobytes() == ref.tobytes()
    assert np.array_equal(piv.swaps, p.swaps) and np.array_equal(piv.perm, p.perm)
    assert fl == orc.lu_factor_flops(s) * nb


def test_lu_bit_exact_fp32():
    rng = np.random.default_rng(5)
    s, nb = 64, 256
    base = rng.standard_normal(nb * s * s).astype(np.float32)
    buf = base.copy()
    piv, _ = batched_lu_factor_inplace([BlockRef(buf, i * s * s, s, s, s) for i in range(nb)])
    ref = base.copy()
    p = orc.lu_factor(orc.sview(ref, 0, s * s, nb, s, s, s))
    assert buf.tobytes() == ref.tobytes() and np.array_equal(piv.swaps, p.swaps)


def test_lu_singular_flagged_and_solve_refuses():  # :294-301
    good = make_block(np.eye(2))
    bad = make_block(np.array([[1.0, 2.0], [2.0, 4.0]]))
    piv, _ = batched_lu_factor_inplace([good, bad])
    assert piv.singular == [1]
    with pytest.raises(SingularBlockError, match=r"index \[1\]"):
        batched_lu_solve_inplace([good, bad], piv, [make_block(np.ones((2, 1))), make_block(np.ones((2, 1)))])


def test_lu_solve_identity_and_diagonal():  # :304-315
    ident = make_block(np.eye(3))
    pivi, _ = batched_lu_factor_inplace([ident])
    rhs = make_block(np.array([[1.0], [2.0], [3.0]]))
    batched_lu_solve_inplace([ident], pivi, [rhs])
    assert rhs.view()[:, 0].tolist() == [1.0, 2.0, 3.0]
    diag = make_block(np.diag([2.0, 4.0]))
    pivd, _ = batched_lu_factor_inplace([diag])
    r2 = make_block(np.array([[2.0], [4.0]]))
    batched_lu_solve_inplace([diag], pivd, [r2])
    assert r2.view()[:, 0].tolist() == [1.0, 1.0]


def test_lu_solve_matches_dense():  # :318-333
    rng = np.random.default_rng(41)
    mats = [rng.standard_normal((24, 24)) + 24 * np.eye(24) for _ in range(5)]
    rhss = [rng.standard_normal((24, 3)) for _ in range(5)]
    blocks = [make_block(m) for m in mats]
    rblocks = [make_block(r) for r in rhss]
    piv, _ = batched_lu_factor_inplace(blocks)
    fl = batched_lu_solve_inplace(blocks, piv, rblocks)
    assert fl == 5 * 2 * 24 * 24 * 3
    for m, r, rb in zip(mats, rhss, rblocks):
        want = np.linalg.solve(m, r)
        assert np.linalg.norm(rb.view() - want) / np.linalg.norm(want) <= 1e-13


def test_lu_solve_stacks_multicolumn():  # :373-391
    rng = np.random.default_rng(53)
    B, s, c = 4, 8, 3
    mats = rng.standard_normal((B, s, s)) + s * np.eye(s)
    blocks = [make_block(mats[i].copy()) for i in range(B)]
    piv, _ = batched_lu_factor_inplace(blocks)
    lu_stack = np.stack([blocks[i].view().copy() for i in range(B)])
    rhs = rng.standard_normal((c, B, s, 1))
    got = rhs.copy()
    lu_solve_stacks(lu_stack, piv.perm, got)
    single = rhs.copy()
    for j in range(c):
        lu_solve_stacks(lu_stack, piv.perm, single[j])
    assert got.tobytes() == single.tobytes()
    for j in range(c):
        for b in range(B):
            want = np.linalg.solve(mats[b], rhs[j, b])
            assert np.linalg.norm(got[j, b] - want) <= 1e-12 * np.linalg.norm(want)
