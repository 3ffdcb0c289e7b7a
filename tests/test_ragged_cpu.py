"""CPU: ragged LevelPanel ingestion -> the
engine's uniform slabs, zero-padded per node.  The padded matrix
equals the ragged one entry for entry, and the oracle factorization of the
padded layout (K blocks with zero-padded T parts) solves it."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import hodlr_oracle as orc
from paper_2208_06290_b200.hodlr import LevelPanel, pad_level_panels


def ragged(n, m, L, seed, width=8, kmax=6):
    rng = np.random.default_rng(seed)
    D = (rng.standard_normal((1 << L) * m * m) / np.sqrt(m)).reshape(1 << L, m, m)
    D += 4 * np.eye(m)
    A = np.zeros((n, n))
    for a in range(1 << L):
        A[a * m : (a + 1) * m, a * m : (a + 1) * m] = D[a].T  # column-major storage of block a
    ups, vps = [], []
    for lv in range(1, L + 1):
        nl = n >> lv
        ks = rng.integers(0, kmax + 1, size=1 << (lv - 1))
        nr_u = np.repeat(ks, 2)  # both orientations of a sibling pair share its rank
        nr_v = nr_u.copy()
        off_u = rng.integers(0, width - kmax + 1, size=1 << lv)
        off_v = rng.integers(0, width - kmax + 1, size=1 << lv)
        Up = rng.standard_normal((width, n)) / np.sqrt(nl)
        Vp = rng.standard_normal((width, n)) / np.sqrt(nl)
        for p in range(1 << (lv - 1)):
            for o in range(2):
                a, b = 2 * p + o, 2 * p + 1 - o
                k = nr_u[a]
                Ua = Up[off_u[a] : off_u[a] + k, a * nl : (a + 1) * nl]
                Vb = Vp[off_v[b] : off_v[b] + k, b * nl : (b + 1) * nl]
                A[a * nl : (a + 1) * nl, b * nl : (b + 1) * nl] = Ua.T @ Vb
        ups.append(LevelPanel(lv, Up.reshape(-1), off_u, nr_u))
        vps.append(LevelPanel(lv, Vp.reshape(-1), off_v, nr_v))
    return D.reshape(-1), ups, vps, A


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_padded_layout_reproduces_the_ragged_matrix_and_solves(seed):
    n, m, L = 512, 32, 4
    D, ups, vps, A = ragged(n, m, L, seed)
    r, U, V = pad_level_panels(n, m, ups, vps, round_rank=False)
    assert r == max(int(p.node_ranks.max()) for p in ups)
    h = orc.HodlrData(orc.Layout(n, m, r), D.copy(), U, V)
    assert np.allclose(orc.dense(h), A, rtol=0, atol=1e-13)
    f = orc.factorize(h.copy())
    b = np.random.default_rng(9).standard_normal((n, 1))
    x = orc.solve(f, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
    # rounding the rank up to a fused-kernel size pads further and changes nothing
    r16, U16, V16 = pad_level_panels(n, m, ups, vps)
    assert r16 == 16 or r16 == r
    h16 = orc.HodlrData(orc.Layout(n, m, r16), D.copy(), U16, V16)
    assert np.allclose(orc.dense(h16), A, rtol=0, atol=1e-13)


def test_ragged_errors():
    n, m, L = 128, 32, 2
    D, ups, vps, _ = ragged(n, m, L, 3)
    with pytest.raises(ValueError, match="one u and one v panel per level"):
        pad_level_panels(n, m, ups[:1], vps)
    bad = LevelPanel(2, vps[1].data, vps[1].col_offsets, vps[1].node_ranks + 1)
    with pytest.raises(ValueError, match="equal column counts"):
        pad_level_panels(n, m, ups, [vps[0], bad])
    with pytest.raises(ValueError, match="rank 1 < the largest node rank"):
        pad_level_panels(n, m, ups, vps, rank=1)
