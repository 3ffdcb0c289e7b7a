"""GPU: the sharded schedule (hodlr_*_local / hodlr_*_top + per-level sum
all-reduce) on one device, P shards driven in lockstep, against the
single-GPU factorization and solve."""

from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2208_06290_b200 as hb  # noqa: E402
from paper_2208_06290_b200 import distributed as dd  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("n,m,r", [(1 << 14, 64, 32), (1 << 13, 64, 16)])
def test_sharded_matches_single_gpu(world, n, m, r):
    h = hb.random_hodlr(n, m, r, seed=11, s=2.0)
    shards = [dd.make_shard(h, g, world) for g in range(world)]
    f = hb.factorize(h.clone())
    be = dd.GpuBackend()
    states = dd.run_lockstep([dd.factorize_steps(s, be) for s in shards])
    L, n_loc = h.L, n // world
    Yref = f.Y.view(r * L, n)
    for g, st in enumerate(states):
        Yg = st.bufs["Y"].view(r * L, n_loc)
        yo = Yref[:, g * n_loc : (g + 1) * n_loc]
        assert float((Yg - yo).abs().max() / yo.abs().max()) < 1e-12
        # K pivots of every level this rank factored agree with the single-GPU run
        kinfo_all = st.bufs["kinfo"]
        assert int(kinfo_all.sum()) == 0
    # top-level K blocks (factored redundantly on every rank) match exactly in pivots
    nk = (1 << world.bit_length() - 1) - 1
    for st in states:
        assert torch.equal(st.bufs["kswaps"][: nk * 2 * r], f.kswaps[: nk * 2 * r])
    g = torch.Generator("cuda").manual_seed(4)
    b = torch.randn(n, 3, dtype=torch.float64, device="cuda", generator=g)
    x = hb.solve(f, b)
    xs = [b[g * n_loc : (g + 1) * n_loc].t().contiguous().reshape(-1) for g in range(world)]
    dd.run_lockstep([dd.solve_steps(st, st.shard, be, xg, 3) for st, xg in zip(states, xs)])
    xd = torch.cat([xg.view(3, n_loc).t() for xg in xs])
    assert float((xd - x).norm() / x.norm()) < 1e-12
