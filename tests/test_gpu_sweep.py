"""GPU: a seeded sweep over shapes the fused and generic paths dispatch on --
leaf m, rank r, depth L, pivoting regime s, nrhs -- against the CPU oracle
(leaf / K pivots bit-exact; x within 1e-10 of the oracle for s = 1, within
max(1e-10, 4 x the oracle's own 1-ulp sensitivity) for the hard-pivoting
s = 16 regime; relres within 4x of the oracle's own residual)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import hodlr_oracle as orc  # noqa: E402
import paper_2208_06290_b200 as hb  # noqa: E402
from tests.conftest import record_parity  # noqa: E402


def _cases():
    rng = np.random.default_rng(2024)
    out = []
    for k in range(16):
        m = int(rng.choice([16, 32, 64]))
        r = int(rng.choice([4, 8, 16, 32, 64]))
        L = int(rng.integers(1, 6))
        if 2 * r > (m << L) // 2:  # keep the coarsest blocks at least rank-wide
            r = max(4, ((m << L) // 4) // 8 * 8) if ((m << L) // 4) >= 8 else 4
        s = float(rng.choice([1.0, 16.0]))
        nrhs = int(rng.choice([1, 3, 9, 17]))
        out.append((m, r, L, s, nrhs, 100 + k))
    return out


@pytest.mark.parametrize("m,r,L,s,nrhs,seed", _cases())
def test_sweep_against_oracle(m, r, L, s, nrhs, seed):
    n = m << L
    h = orc.make_exact_hodlr(n, m, r, seed=seed, s=s)
    b = np.random.default_rng(seed).standard_normal((n, nrhs))
    fo = orc.factorize(h.copy())
    xo = orc.solve(fo, b)
    hm = hb.HodlrMatrix.from_buffers(n, m, r, h.D, h.U, h.V)
    f = hb.factorize(hm.clone())
    x = hb.solve(f, b)
    assert np.array_equal(f.dperm.cpu().numpy().reshape(-1, m), fo.dpiv.perm)
    if L > 0:
        assert np.array_equal(f.kswaps.cpu().numpy()[: ((1 << L) - 1) * 2 * r].reshape(-1, 2 * r),
                              np.concatenate([p.swaps for p in fo.kpiv]))
    rel = np.linalg.norm(x - xo) / np.linalg.norm(xo)
    if s <= 4:
        gate, sens = 1e-10, None
    else:  # the oracle's own change under a 1-ulp perturbation of U
        h2 = h.copy()
        h2.U *= 1 + 1e-16 * np.random.default_rng(0).standard_normal(h2.U.size)
        xo2 = orc.solve(orc.factorize(h2), b)
        sens = np.linalg.norm(xo2 - xo) / np.linalg.norm(xo)
        gate = max(1e-10, 4 * sens)
    record_parity(f"sweep/m{m}_r{r}_L{L}_s{s:g}_nrhs{nrhs}", x=rel, gate_x=gate, sens_x=sens)
    assert rel <= gate, (rel, gate)
    bt = torch.from_numpy(b).cuda()

    def relres(xx):
        return float(torch.linalg.norm(hm.matvec(torch.from_numpy(xx).cuda()) - bt) / torch.linalg.norm(bt))

    # the s = 16 regime is ill-conditioned: measure against the oracle's own residual
    assert relres(x) <= max(1e-12, 4 * relres(xo)), (relres(x), relres(xo))


@pytest.mark.parametrize("m,r,L,nrhs", [(64, 8, 5, 1), (64, 8, 3, 9), (32, 8, 4, 3), (64, 16, 4, 2), (32, 4, 5, 1),
                                        (16, 8, 4, 5)])
def test_sweep_fp32_against_oracle(m, r, L, nrhs):
    # fp32 (cfg4 preconditioner path): fused r = 8 / m = 64 kernels and the generic fp32 path
    n = m << L
    h = orc.make_exact_hodlr(n, m, r, seed=n + r, s=1.0, dtype=np.float32)
    b = np.random.default_rng(5).standard_normal((n, nrhs)).astype(np.float32)
    fo = orc.factorize(h.copy())
    xo = orc.solve(fo, b)
    f = hb.factorize(hb.HodlrMatrix.from_buffers(n, m, r, h.D, h.U, h.V))
    assert f.D.dtype == torch.float32
    assert np.array_equal(f.dperm.cpu().numpy().reshape(-1, m), fo.dpiv.perm)
    x = hb.solve(f, b)
    rel = np.linalg.norm(x.astype(np.float64) - xo) / np.linalg.norm(xo)
    record_parity(f"sweep_fp32/m{m}_r{r}_L{L}_nrhs{nrhs}", x=rel, gate_x=1e-4)
    assert rel <= 1e-4, rel
