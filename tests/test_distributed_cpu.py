"""CPU: the sharded (multi-GPU) schedule's host logic -- partitioning, packing
and the per-top-level sum all-reduces -- driven with the numpy (oracle)
backend, in lockstep (world 1..8) and over real gloo process groups (world_size 2 and 4)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import hodlr_oracle as orc
from paper_2208_06290_b200 import distributed as dd
from tests.dist_numpy import NumpyBackend


def np_shard(h, rank, world):
    lay = h.lay
    n, m, r, L = lay.n, lay.m, lay.r, lay.L
    n_loc, row0 = n // world, rank * (n // world)
    D = h.D[(row0 // m) * m * m : (row0 + n_loc) // m * m * m].copy()
    return dd.Shard(n, m, r, rank, world, D, dd.slice_rows(np, h.U, n, r * L, row0, n_loc),
                    dd.slice_rows(np, h.V, n, r * L, row0, n_loc))


def check_against_oracle(h, states, xs, b, world):
    lay = h.lay
    n, m, r, L = lay.n, lay.m, lay.r, lay.L
    fo = orc.factorize(h.copy())
    xo = orc.solve(fo, b)
    n_loc = n // world
    for g, st in enumerate(states):
        yo = fo.Y.reshape(r * L, n)[:, g * n_loc : (g + 1) * n_loc]
        assert np.allclose(st.Y.reshape(r * L, n_loc), yo, rtol=0, atol=1e-12 * np.abs(yo).max())
        for lv in range(L):
            for p, sw in st.kswaps.get(lv, {}).items():
                assert np.array_equal(sw, fo.kpiv[lv].swaps[p]), (g, lv, p)
        xg = xs[g].reshape(-1, n_loc).T
        assert np.allclose(xg, xo.reshape(n, -1)[g * n_loc : (g + 1) * n_loc], rtol=0, atol=1e-12 * np.abs(xo).max())


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_lockstep_schedule_matches_oracle(world):
    n, m, r = 2048, 32, 8
    h = orc.make_exact_hodlr(n, m, r, seed=5, s=2.0)  # well conditioned: partial-sum order is the only difference
    be = NumpyBackend()
    shards = [np_shard(h, g, world) for g in range(world)]
    states = dd.run_lockstep([dd.factorize_steps(s, be) for s in shards])
    b = np.random.default_rng(3).standard_normal((n, 2))
    n_loc = n // world
    xs = [np.asfortranarray(b[g * n_loc : (g + 1) * n_loc]).ravel(order="F").copy() for g in range(world)]
    dd.run_lockstep([dd.solve_steps(st, st.shard, be, x, 2) for st, x in zip(states, xs)])
    check_against_oracle(h, states, xs, b, world)


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, r = 1024, 32, 8
        h = orc.make_exact_hodlr(n, m, r, seed=9, s=4.0)
        sh = np_shard(h, rank, world)
        be = NumpyBackend()

        def all_reduce(buf):
            dist.all_reduce(torch.from_numpy(buf), op=dist.ReduceOp.SUM)

        st = dd.run(dd.factorize_steps(sh, be), all_reduce)
        b = np.random.default_rng(1).standard_normal((n, 1))
        n_loc = n // world
        x = b[rank * n_loc : (rank + 1) * n_loc, 0].copy()
        dd.run(dd.solve_steps(st, sh, be, x, 1), all_reduce)
        np.savez(out.format(rank=rank), Y=st.Y, x=x,
                 kswaps=np.array([[lv, p] + list(sw) for lv, d in st.kswaps.items() for p, sw in d.items()]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_world_matches_oracle(tmp_path, world):
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "rank{rank}.npz")
    mp.start_processes(_gloo_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    n, m, r = 1024, 32, 8
    h = orc.make_exact_hodlr(n, m, r, seed=9, s=4.0)
    b = np.random.default_rng(1).standard_normal((n, 1))
    fo = orc.factorize(h.copy())
    xo = orc.solve(fo, b)
    n_loc = n // world
    L = h.lay.L
    for g in range(world):
        d = np.load(out.format(rank=g))
        yo = fo.Y.reshape(r * L, n)[:, g * n_loc : (g + 1) * n_loc]
        assert np.allclose(d["Y"].reshape(r * L, n_loc), yo, rtol=0, atol=1e-12 * np.abs(yo).max())
        assert np.allclose(d["x"], xo[g * n_loc : (g + 1) * n_loc, 0], rtol=0, atol=1e-12 * np.abs(xo).max())
        for row in d["kswaps"]:
            lv, p, sw = int(row[0]), int(row[1]), row[2:]
            assert np.array_equal(sw, fo.kpiv[lv].swaps[p])
