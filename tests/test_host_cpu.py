"""CPU-only checks of the host layer: the tree, the reference-mirror API's
validation/error conventions, and that the C-ABI library loads and exports
every symbol include/hodlr_b200.h declares (no compute without a GPU)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import _lib
from paper_2208_06290_b200.tree import ClusterTree, IndexRange, build_tree, sibling_pairs

ROOT = Path(__file__).resolve().parent.parent


def ranges(level):
    return [(r.start, r.end) for r in level]


# ---- tree (reference pkg/tests/test_tree.py semantics) ----

def test_index_range():
    assert len(IndexRange(3, 7)) == 4
    for a, b in ((5, 5), (-1, 2)):
        with pytest.raises(ValueError):
            IndexRange(a, b)


def test_spec_tree_examples():
    assert ranges(build_tree(400, 100).leaves) == [(0, 100), (100, 200), (200, 300), (300, 400)]
    t = build_tree(7, 8)
    assert t.depth == 0 and ranges(t.leaves) == [(0, 7)]
    t = build_tree(5, 3)
    assert t.depth == 1 and ranges(t.leaves) == [(0, 3), (3, 5)]
    assert build_tree(5, 1).depth == 2 and build_tree(1, 1).depth == 0


@pytest.mark.parametrize("n", [1, 2, 5, 7, 64, 100, 257, 1000, 1024])
@pytest.mark.parametrize("leaf", [1, 3, 16, 64])
def test_partition_child_sum(n, leaf):
    t = build_tree(n, leaf)
    for ell, level in enumerate(t.levels):
        assert len(level) == 2**ell
        pos = 0
        for r in level:
            assert r.start == pos
            pos = r.end
        assert pos == n
    for ell in range(t.depth):
        for k, parent in enumerate(t.levels[ell]):
            a, b = t.children(ell, k)
            assert (a.start, b.end, a.end) == (parent.start, parent.end, b.start)
    assert max(t.leaf_sizes) - min(t.leaf_sizes) <= 1


def test_sibling_pairs_and_errors():
    t = build_tree(400, 100)
    assert [(ranges([a])[0], ranges([b])[0]) for a, b in sibling_pairs(t, 2)] == [
        ((0, 100), (100, 200)), ((200, 300), (300, 400))]
    with pytest.raises(ValueError):
        sibling_pairs(build_tree(7, 8), 1)
    with pytest.raises(ValueError):
        ClusterTree(4, 3)
    assert ClusterTree(8, 2) == build_tree(8, 2)


# ---- API validation (raised before any device work) ----

def make_block(arr):
    a = np.asarray(arr)
    return hb.BlockRef(np.asfortranarray(a).ravel(order="F").copy(), 0, a.shape[0], a.shape[1], a.shape[0])


def test_blockref_bounds_and_view():
    buf = np.arange(12, dtype=float)
    v = hb.BlockRef(buf, 2, 3, 2, 5).view()
    assert v.shape == (3, 2) and v[0, 1] == 7 and v[2, 1] == 9
    with pytest.raises(ValueError):
        hb.BlockRef(np.zeros(10), 4, 3, 2, 5)


def test_as_stack():
    buf = np.arange(48, dtype=float)
    st = hb.as_stack([hb.BlockRef(buf, 16 * i, 4, 4, 4) for i in range(3)])
    assert st.shape == (3, 4, 4) and st[2, 1, 2] == 41.0
    assert hb.as_stack([hb.BlockRef(buf, 0, 4, 4, 4), hb.BlockRef(buf, 16, 4, 3, 4)]) is None


def test_gemm_shape_and_overlap_errors():
    a, b = make_block(np.zeros((3, 2))), make_block(np.zeros((2, 2)))
    with pytest.raises(ValueError, match="batch index 1"):
        hb.batched_gemm([(a, b, make_block(np.zeros((3, 2)))), (a, b, make_block(np.zeros((2, 2))))])
    buf = np.zeros(64)
    e, o = make_block(np.eye(4)), make_block(np.ones((4, 4)))
    with pytest.raises(ValueError, match="overlap"):
        hb.batched_gemm([(e, o, hb.BlockRef(buf, 0, 4, 4, 8)), (e, o, hb.BlockRef(buf, 2, 4, 4, 8))])
    with pytest.raises(ValueError, match="unsupported transpose_a"):
        hb.batched_gemm([], transpose_a="t")
    assert hb.batched_gemm([]) == 0 and hb.grouped_gemm_large([]) == 0


def test_lu_validation_errors():
    with pytest.raises(ValueError, match="not square"):
        hb.batched_lu_factor_inplace([make_block(np.zeros((2, 3)))])
    with pytest.raises(ValueError, match="share one size"):
        hb.batched_lu_factor_inplace([make_block(np.eye(2)), make_block(np.eye(3))])
    piv = hb.LuPivots(np.zeros((1, 2), np.int64), np.zeros((1, 2), np.int64), [0])
    with pytest.raises(hb.SingularBlockError, match=r"index \[0\]"):
        hb.batched_lu_solve_inplace([make_block(np.eye(2))], piv, [make_block(np.ones((2, 1)))])
    piv = hb.LuPivots(np.zeros((1, 2), np.int64), np.zeros((1, 2), np.int64))
    with pytest.raises(ValueError, match="differ in length"):
        hb.batched_lu_solve_inplace([make_block(np.eye(2))], piv, [])
    assert hb.batched_lu_factor_inplace([])[1] == 0


def test_parse_executor():
    assert hb.parse_executor("serial") is hb.SERIAL
    assert hb.parse_executor("threads:3").threads == 3
    with pytest.raises(ValueError):
        hb.parse_executor("gpu")


def test_flop_report_matches_closed_form():
    from oracle import hodlr_oracle as orc
    for n, m, r in ((1 << 14, 64, 32), (1 << 20, 64, 32), (4096, 64, 8)):
        assert hb.flop_report(n, m, r)["total"] == orc.factor_flops(n, m, r)
        assert hb.solve_flops(n, m, r, 3) == orc.solve_flops(n, m, r, 3)


# ---- native library: loads and exports the header's symbols ----

def header_symbols():
    txt = (ROOT / "include" / "hodlr_b200.h").read_text()
    return sorted(set(re.findall(r"\b(hodlr_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"
    assert b"sm_100a" in lib.hodlr_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_queries_without_gpu():
    lib = _lib.load()
    d = _lib.Desc(1 << 20, 64, 32, 14, _lib.F64)
    assert lib.hodlr_factorize_workspace(ctypes.byref(d)) > 0
    bad = _lib.Desc(1000, 64, 32, 4, _lib.F64)
    assert lib.hodlr_factorize_workspace(ctypes.byref(bad)) == 0


def test_product_path_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.HodlrNativeError):
        hb.HodlrMatrix.from_buffers(128, 16, 2, np.zeros(8 * 256), np.zeros(128 * 6), np.zeros(128 * 6))


def test_per_level_rank_descriptors_without_gpu():
    # hodlr_desc.ranks: workspace sizing, validation (max must equal r; fp32 takes one rank),
    # and the per-level flop counters vs the oracle's instrumented counts
    from oracle import hodlr_oracle as orc

    lib = _lib.load()
    ranks = (16, 32, 0, 16, 32, 64)
    d = _lib.make_desc(4096, 64, 64, 6, _lib.F64, ranks)
    assert lib.hodlr_factorize_workspace(ctypes.byref(d)) > 0
    assert lib.hodlr_solve_workspace(ctypes.byref(d), 3) > 0
    assert lib.hodlr_matvec_workspace(ctypes.byref(d), 3) > 0
    assert lib.hodlr_factorize_workspace(ctypes.byref(_lib.make_desc(4096, 64, 32, 6, _lib.F64, ranks))) == 0
    assert lib.hodlr_factorize_workspace(ctypes.byref(_lib.make_desc(4096, 64, 64, 6, _lib.F32, ranks))) == 0
    assert lib.hodlr_build_workspace(ctypes.byref(d)) == 0  # the builders take one rank
    h = orc.make_exact_hodlr(4096, 64, 64, seed=2, ranks=ranks)
    f = orc.factorize(h)
    rep = hb.flop_report(4096, 64, 64, ranks=ranks)
    for k in ("leaf_getrf", "leaf_getrs", "tw_gemm", "k_getrf", "k_getrs", "update_gemm"):
        assert rep[k] == f.flops[k], k
