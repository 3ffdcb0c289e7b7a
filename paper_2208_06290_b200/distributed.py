"""Subtree-sharded factorize / solve over P = 2^p ranks.

Rank g owns the rows of level-p node g (N/P consecutive rows): its leaves'
diagonal blocks and its rows of every U / V panel.  Levels l >= p are purely
local (the whole level-l node lives on one rank).  For each top level l < p,
every rank contributes the partial [W|T] (factorization) or w (solve) of its
rows, ONE sum all-reduce of the packed 2^(l+1)-children buffer makes them
complete everywhere, every rank factors the 2^l K blocks of that level
redundantly (tiny) and updates its own rows.  Communication: p all-reduces of
2^(l+1) r x r(l+1) (resp. r x nrhs) scalars -- latency-bound, independent of N.

The schedule is written once as a generator that yields each buffer to be
all-reduced; `run` drives it with a real communicator (NCCL through
torch.distributed) and `run_lockstep` drives P shards in one process (one GPU,
used by the tests).  The compute backend is pluggable: `GpuBackend` calls the
sm_100a library (include/hodlr_b200.h, hodlr_*_local / hodlr_*_top); the CPU
tests inject a numpy backend built on the oracle to check this host logic with
gloo.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

from . import _lib


@dataclass
class Shard:
    """One rank's rows of an N = m 2^L HODLR matrix (reference layout, ld n_loc)."""

    n: int
    m: int
    r: int
    rank: int
    world: int
    D: object  # local leaves, flat (n_loc/m) m^2
    U: object  # n_loc x rL column-major (becomes Y)
    V: object  # n_loc x rL column-major

    @property
    def L(self) -> int:
        return int(round(math.log2(self.n // self.m)))

    @property
    def p(self) -> int:
        return int(round(math.log2(self.world)))

    @property
    def n_loc(self) -> int:
        return self.n // self.world

    @property
    def row0(self) -> int:
        return self.rank * self.n_loc


def slice_rows(xp, buf, n, ncols, row0, n_loc):
    """Rows [row0, row0+n_loc) of an n x ncols column-major flat buffer (copy)."""
    if ncols == 0:
        return buf[:0].clone() if hasattr(buf, "clone") else buf[:0].copy()
    v = buf.reshape(ncols, n)[:, row0 : row0 + n_loc]
    return v.reshape(-1).clone() if hasattr(v, "clone") else v.reshape(-1).copy()


def make_shard(h, rank: int, world: int) -> Shard:
    """Split a global HodlrMatrix (torch) into rank `rank`'s shard."""
    n, m, r, L = h.n, h.m, h.rank, h.L
    if world & (world - 1) or world > (1 << L):
        raise ValueError(f"world size {world} must be a power of two <= 2^L")
    n_loc = n // world
    row0 = rank * n_loc
    nl = n_loc // m
    D = h.D[(row0 // m) * m * m : (row0 // m + nl) * m * m].clone()
    return Shard(n, m, r, rank, world, D, slice_rows(None, h.U, n, r * L, row0, n_loc),
                 slice_rows(None, h.V, n, r * L, row0, n_loc))


# ---------------------------------------------------------------------------
# the schedule (backend-independent host logic)
# ---------------------------------------------------------------------------


def _pack(backend, contrib, q, lv, ncols, r):
    """Place node q's r x ncols contribution (ld r) in the packed buffer of all
    2^(lv+1) level-(lv+1) nodes (paired per parent: 2r x ncols, ld 2r)."""
    buf = backend.zeros((1 << lv) * 2 * r * ncols)
    view = buf.reshape(1 << lv, ncols, 2 * r)
    view[q >> 1, :, (q & 1) * r : (q & 1) * r + r] = contrib.reshape(ncols, r)
    return buf


def factorize_steps(shard: Shard, backend):
    """Generator: yields buffers to sum-all-reduce; returns the factor state."""
    st = backend.factor_init(shard)
    p, r, n = shard.p, shard.r, shard.n
    contrib = backend.factor_local(st, p)  # [W|T] of this rank's level-p node (p > 0)
    for lv in range(p - 1, -1, -1):
        q = shard.row0 // (n >> (lv + 1))  # this rank's level-(lv+1) node
        buf = _pack(backend, contrib, q, lv, r * (lv + 1), r)
        buf = yield buf
        contrib = backend.factor_top(st, lv, buf)
    return st


def solve_steps(state, shard: Shard, backend, x_local, nrhs: int):
    """Generator for the sharded solve; x_local (n_loc x nrhs, column-major) in place."""
    p, r, n = shard.p, shard.r, shard.n
    contrib = backend.solve_local(state, x_local, nrhs, p)
    for lv in range(p - 1, -1, -1):
        q = shard.row0 // (n >> (lv + 1))
        buf = _pack(backend, contrib, q, lv, nrhs, r)
        buf = yield buf
        contrib = backend.solve_top(state, lv, buf, x_local, nrhs)
    return x_local


def run(gen, all_reduce):
    """Drive one rank's schedule with a real communicator."""
    try:
        buf = next(gen)
        while True:
            all_reduce(buf)
            buf = gen.send(buf)
    except StopIteration as e:
        return e.value


def _copy(x):
    return x.clone() if hasattr(x, "clone") else x.copy()


def run_lockstep(gens):
    """Drive P ranks' schedules in one process; the all-reduce is a fixed-order sum."""
    results = [None] * len(gens)
    bufs = []
    for i, g in enumerate(gens):
        try:
            bufs.append(next(g))
        except StopIteration as e:
            results[i] = e.value
            bufs.append(None)
    while any(b is not None for b in bufs):
        total = None
        for b in bufs:
            if b is not None:
                total = _copy(b) if total is None else total + b
        for i, b in enumerate(bufs):
            if b is None:
                continue
            try:
                bufs[i] = gens[i].send(_copy(total))
            except StopIteration as e:
                results[i] = e.value
                bufs[i] = None
    return results


def torch_all_reduce(buf):
    import torch.distributed as dist

    dist.all_reduce(buf, op=dist.ReduceOp.SUM)


# ---------------------------------------------------------------------------
# GPU backend (C ABI)
# ---------------------------------------------------------------------------


@dataclass
class GpuShardFactor:
    shard: Shard
    desc: object
    fac: object
    bufs: dict = field(default_factory=dict)
    ws: object = None
    wsb: int = 0


class GpuBackend:
    """hodlr_factorize_local / _top and hodlr_solve_local / _top on the rank's GPU."""

    def __init__(self, device="cuda"):
        self.torch = _lib.require_cuda()
        self.lib = _lib.load()
        self.device = device

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def factor_init(self, sh: Shard) -> GpuShardFactor:
        torch = self.torch
        dev = self.device
        n, m, r, L = sh.n, sh.m, sh.r, sh.L
        nl = sh.n_loc // m
        nk = (1 << L) - 1
        i32 = dict(dtype=torch.int32, device=dev)
        b = dict(
            D=sh.D, Dinv=torch.empty_like(sh.D), Y=sh.U, V=sh.V,
            # K blocks of other ranks' deep parents are never written nor read here:
            # no zero-fill (it would be a 1 GB memset per factorization at cfg2)
            K=torch.empty(max(nk, 1) * 4 * r * r, dtype=torch.float64, device=dev),
            Kinv=torch.empty(max(nk, 1) * 4 * r * r, dtype=torch.float64, device=dev),
            dswaps=torch.empty(nl * m, **i32), dperm=torch.empty(nl * m, **i32), dinfo=torch.zeros(nl, **i32),
            kswaps=torch.empty(max(nk, 1) * 2 * r, **i32), kperm=torch.empty(max(nk, 1) * 2 * r, **i32),
            kinfo=torch.zeros(max(nk, 1), **i32),
        )
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        fac = _lib.Factors(*(p(b[k]) for k in ("D", "Dinv", "Y", "V", "K", "Kinv", "dswaps", "dperm", "dinfo",
                                               "kswaps", "kperm", "kinfo")))
        desc = _lib.Desc(n, m, r, L, _lib.F64)
        st = GpuShardFactor(sh, desc, fac, b)
        st.wsb = self.lib.hodlr_factorize_local_workspace(C.byref(desc), sh.n_loc)
        st.ws = torch.empty(max(st.wsb, 1), dtype=torch.uint8, device=dev)
        return st

    def factor_local(self, st: GpuShardFactor, p: int):
        sh = st.shard
        out = self.zeros(sh.r * sh.r * max(p, 1))
        _lib.check(self.lib.hodlr_factorize_local(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, p, C.c_void_p(out.data_ptr()),
            C.c_void_p(st.ws.data_ptr()), st.wsb, self._stream()), "hodlr_factorize_local")
        return out

    def factor_top(self, st: GpuShardFactor, lv: int, tw_all):
        sh = st.shard
        out = self.zeros(sh.r * sh.r * max(lv, 1))
        _lib.check(self.lib.hodlr_factorize_top(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, lv, C.c_void_p(tw_all.data_ptr()),
            C.c_void_p(out.data_ptr()), C.c_void_p(st.ws.data_ptr()), st.wsb, self._stream()), "hodlr_factorize_top")
        return out

    def _solve_ws(self, st, nrhs):
        wsb = self.lib.hodlr_solve_workspace(C.byref(st.desc), nrhs)
        key = ("solve_ws", nrhs)
        if key not in st.bufs:
            st.bufs[key] = self.torch.empty(max(wsb, 1), dtype=self.torch.uint8, device=self.device)
        return st.bufs[key], wsb

    def solve_local(self, st: GpuShardFactor, x, nrhs: int, p: int):
        sh = st.shard
        ws, wsb = self._solve_ws(st, nrhs)
        out = self.zeros(sh.r * nrhs)
        _lib.check(self.lib.hodlr_solve_local(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, p, C.c_void_p(x.data_ptr()), sh.n_loc, nrhs,
            C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), wsb, self._stream()), "hodlr_solve_local")
        return out

    def solve_top(self, st: GpuShardFactor, lv: int, w_all, x, nrhs: int):
        sh = st.shard
        ws, wsb = self._solve_ws(st, nrhs)
        out = self.zeros(sh.r * nrhs)
        _lib.check(self.lib.hodlr_solve_top(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, lv, C.c_void_p(w_all.data_ptr()),
            C.c_void_p(out.data_ptr()), C.c_void_p(x.data_ptr()), sh.n_loc, nrhs, C.c_void_p(ws.data_ptr()), wsb,
            self._stream()), "hodlr_solve_top")
        return out


def factorize_sharded(shard: Shard, all_reduce=torch_all_reduce, backend=None):
    """One rank's part of the sharded factorization (call on every rank)."""
    backend = backend or GpuBackend()
    return run(factorize_steps(shard, backend), all_reduce)


def solve_sharded(state, x_local, nrhs: int = 1, all_reduce=torch_all_reduce, backend=None):
    """One rank's part of the sharded solve; x_local (n_loc x nrhs, column-major) in place."""
    backend = backend or GpuBackend()
    return run(solve_steps(state, state.shard, backend, x_local, nrhs), all_reduce)
