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


def _gloo_singular_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2208_06290_b200.hodlr import HodlrSingularError

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, r = 512, 32, 4
        h = orc.make_exact_hodlr(n, m, r, seed=3, s=1.0)
        h.D[13 * m * m : 14 * m * m] = 0.0  # leaf 13 (owned by rank 1 of 2) is singular
        sh = np_shard(h, rank, world)

        def all_reduce(buf):
            dist.all_reduce(torch.from_numpy(buf), op=dist.ReduceOp.SUM)

        try:
            dd.run(dd.factorize_steps(sh, NumpyBackend()), all_reduce)
            msg = "no error"
        except HodlrSingularError as e:
            msg = str(e)
        with open(out.format(rank=rank), "w") as fh:
            fh.write(msg)
    finally:
        dist.destroy_process_group()


def test_gloo_singular_leaf_raises_on_every_rank(tmp_path):
    # a singular leaf on one rank makes ALL ranks raise with level and node
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "sing{rank}.txt")
    mp.start_processes(_gloo_singular_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    for g in range(2):
        with open(out.format(rank=g)) as fh:
            assert fh.read() == "singular leaf block at level 4, node(s) [13]"


def test_lockstep_singular_k_block_reported():
    # zero leaves on both halves -> K singular is impossible to provoke portably; check the
    # flag decoder directly on a synthetic flag vector (level 2, node 1)
    from paper_2208_06290_b200.distributed import raise_singular_from_flags
    from paper_2208_06290_b200.hodlr import HodlrSingularError

    L = 3
    flags = np.zeros(2 * (1 << L) - 1)
    flags[(1 << L) + 3 + 1] = 2.0  # K level 2 starts at 2^2 - 1 = 3
    with pytest.raises(HodlrSingularError, match=r"K block at level 2, node\(s\) \[1\]"):
        raise_singular_from_flags(flags, L)
    raise_singular_from_flags(np.zeros(2 * (1 << L) - 1), L)  # clean: no raise
