"""CPU: the assembly oracle against the reference's own ACA (golden vectors),
and the product's host-side contour geometry against the oracle."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import build_oracle as bo

GOLDEN = Path(__file__).resolve().parent / "golden"


def cases():
    return sorted(GOLDEN.glob("build_*.npz"))


@pytest.mark.parametrize("path", cases(), ids=lambda p: p.stem)
def test_build_oracle_reproduces_reference_bitwise(path):
    g = np.load(path)
    n, m, r, kind = int(g["n"]), int(g["m"]), int(g["r"]), str(g["kind"])
    entry = bo.LaplaceDL(n) if kind == "laplace" else bo.Dense(g["A"])
    D, U, V = bo.assemble(entry, n, m, r)
    assert D.tobytes() == g["D"].tobytes()
    assert U.tobytes() == g["U"].tobytes()
    assert V.tobytes() == g["V"].tobytes()


def test_spec_assemble_examples():
    # identity -> rank-0 off-diagonals, identity leaves; [[2,1],[1,2]] -> U = V = [1]
    g = np.load(GOLDEN / "build_dense_spec2x2.npz")
    assert g["D"].tolist() == [2.0, 2.0] and g["U"].tolist() == [1.0, 1.0] and g["V"].tolist() == [1.0, 1.0]
    g = np.load(GOLDEN / "build_dense_identity_n64_m16_r4.npz")
    assert not g["U"].any() and not g["V"].any() and not g["ranks"].any()


def test_product_geometry_matches_oracle_bitwise():
    from paper_2208_06290_b200.construct import laplace_dl_geometry

    n = 4096
    geom = laplace_dl_geometry(n)
    ref = bo.LaplaceDL(n)
    assert geom[0].tobytes() == ref.xy[:, 0].tobytes() and geom[1].tobytes() == ref.xy[:, 1].tobytes()
    assert geom[2].tobytes() == ref.nrm[:, 0].tobytes() and geom[3].tobytes() == ref.nrm[:, 1].tobytes()
    assert geom[4].tobytes() == ref.w.tobytes()
    assert geom[5].tobytes() == ref.logt.tobytes() and geom[6].tobytes() == ref.diag.tobytes()


def test_laplace_hodlr_approximates_the_operator():
    # the rank-r HODLR of the cfg2 operator: error vs the exact dense matrix falls with r
    n, m = 512, 32
    ent = bo.LaplaceDL(n)
    idx = np.arange(n)
    A = ent(idx[:, None], idx[None, :])
    errs = []
    for r in (4, 8, 16):
        D, U, V = bo.assemble(ent, n, m, r)
        from oracle import hodlr_oracle as orc

        h = orc.HodlrData(orc.Layout(n, m, r), D, U, V)
        errs.append(np.linalg.norm(orc.dense(h) - A) / np.linalg.norm(A))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-3  # sibling blocks touch: slow decay
