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
    """Split a global HodlrMatrix (torch, float64) into rank `rank`'s shard.

    The row-sharded entry points (``hodlr_*_local`` / ``hodlr_*_top``) are
    fp64-only, so anything else is rejected here rather than reinterpreted."""
    import torch

    n, m, r, L = h.n, h.m, h.rank, h.L
    if getattr(h, "ranks", None) is not None:
        raise ValueError("the row-sharded path takes one rank per matrix (per-level ranks: single GPU)")
    if world < 1 or world & (world - 1) or world > (1 << L):
        raise ValueError(f"world size {world} must be a power of two <= 2^L")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    for name in ("D", "U", "V"):
        t = getattr(h, name)
        if t.dtype != torch.float64:
            raise TypeError(f"sharded factorization is fp64-only ({name} is {t.dtype})")
    n_loc = n // world
    row0 = rank * n_loc
    nl = n_loc // m
    D = h.D[(row0 // m) * m * m : (row0 // m + nl) * m * m].clone()
    return Shard(n, m, r, rank, world, D, slice_rows(None, h.U, n, r * L, row0, n_loc),
                 slice_rows(None, h.V, n, r * L, row0, n_loc))


def make_shard_like(sh: Shard) -> Shard:
    """A second shard with the same geometry and (copied) buffers: the working
    copy the factorization consumes, restored from ``sh`` between runs."""
    return Shard(sh.n, sh.m, sh.r, sh.rank, sh.world, sh.D.clone(), sh.U.clone(), sh.V)


def check_shard_buffers(sh: Shard) -> None:
    """fp64, contiguous, exactly the local sizes (the C ABI trusts them)."""
    import torch

    n_loc, m, r, L = sh.n_loc, sh.m, sh.r, sh.L
    want = {"D": (n_loc // m) * m * m, "U": n_loc * r * L, "V": n_loc * r * L}
    for name, size in want.items():
        t = getattr(sh, name)
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"shard {name} must be a torch tensor (got {type(t).__name__})")
        if t.dtype != torch.float64:
            raise TypeError(f"shard {name} must be float64 (got {t.dtype})")
        if not t.is_contiguous() or t.numel() != size:
            raise ValueError(f"shard {name} must be contiguous with {size} entries (got {t.numel()})")


# ---------------------------------------------------------------------------
# the schedule (backend-independent host logic)
# ---------------------------------------------------------------------------


def _pack(backend, st, contrib, q, lv, ncols, r):
    """Place node q's r x ncols contribution (ld r) in the packed buffer of all
    2^(lv+1) level-(lv+1) nodes (paired per parent: 2r x ncols, ld 2r).  The
    buffer is the rank state's reusable per-(level, ncols) one, zeroed in place."""
    size = (1 << lv) * 2 * r * ncols
    if hasattr(backend, "pack_buffer"):
        buf = backend.pack_buffer(st, ("pack", lv, ncols), size)
    else:
        buf = backend.zeros(size)
    view = buf.reshape(1 << lv, ncols, 2 * r)
    view[q >> 1, :, (q & 1) * r : (q & 1) * r + r] = contrib.reshape(ncols, r)
    return buf


def factorize_steps(shard: Shard, backend, check: bool = True):
    """Generator: yields buffers to sum-all-reduce; returns the factor state.

    The last buffer yielded carries the singular-block flags of every rank
    (leaf and K blocks it factored), so all ranks raise together
    (:class:`~paper_2208_06290_b200.hodlr.HodlrSingularError`)."""
    st = backend.factor_init(shard)
    p, r, n = shard.p, shard.r, shard.n
    contrib = backend.factor_local(st, p)  # [W|T] of this rank's level-p node (p > 0)
    for lv in range(p - 1, -1, -1):
        q = shard.row0 // (n >> (lv + 1))  # this rank's level-(lv+1) node
        buf = _pack(backend, st, contrib, q, lv, r * (lv + 1), r)
        buf = yield buf
        contrib = backend.factor_top(st, lv, buf)
    flags = backend.singular_flags(st) if (check and hasattr(backend, "singular_flags")) else None
    if flags is not None:
        flags = yield flags
        backend.raise_if_singular(st, flags)
    return st


def solve_steps(state, shard: Shard, backend, x_local, nrhs: int):
    """Generator for the sharded solve; x_local (n_loc x nrhs, column-major) in place."""
    p, r, n = shard.p, shard.r, shard.n
    contrib = backend.solve_local(state, x_local, nrhs, p)
    for lv in range(p - 1, -1, -1):
        q = shard.row0 // (n >> (lv + 1))
        buf = _pack(backend, state, contrib, q, lv, nrhs, r)
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


def raise_singular_from_flags(flags, L: int) -> None:
    """Raise HodlrSingularError (level, nodes) from the all-reduced flag vector
    [leaf flags (2^L) | K flags (2^L - 1, level l at 2^l - 1)] -- the same
    report as the single-GPU factorize."""
    import numpy as np

    from .hodlr import HodlrSingularError

    flags = np.asarray(flags)
    nleaf = 1 << L
    bad = np.flatnonzero(flags[:nleaf] > 0)
    if bad.size:
        raise HodlrSingularError("leaf", L, bad.tolist())
    kf = flags[nleaf:]
    for lv in range(L):
        seg = kf[(1 << lv) - 1 : (2 << lv) - 1]
        if (seg > 0).any():
            raise HodlrSingularError("K", lv, np.flatnonzero(seg > 0).tolist())


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
        self._ws = {}

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def factor_init(self, sh: Shard) -> GpuShardFactor:
        torch = self.torch
        dev = self.device
        check_shard_buffers(sh)
        n, m, r, L = sh.n, sh.m, sh.r, sh.L
        nl = sh.n_loc // m
        nk = (1 << L) - 1
        inv = lambda nb, s: max(nb * int(self.lib.hodlr_inv_elems(s)), 1)  # noqa: E731
        i32 = dict(dtype=torch.int32, device=dev)
        b = dict(
            D=sh.D, Dinv=torch.empty(inv(nl, m), dtype=torch.float64, device=dev), Y=sh.U, V=sh.V,
            # K blocks of other ranks' deep parents are never written nor read here:
            # no zero-fill (it would be a 1 GB memset per factorization at cfg2)
            K=torch.empty(max(nk, 1) * 4 * r * r, dtype=torch.float64, device=dev),
            Kinv=torch.empty(inv(max(nk, 1), 2 * r), dtype=torch.float64, device=dev),
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
        ws = self._ws.get((sh.rank, sh.world, st.wsb))  # one workspace per shard, reused across factorizations
        if ws is None:
            ws = self._ws[(sh.rank, sh.world, st.wsb)] = torch.empty(max(st.wsb, 1), dtype=torch.uint8, device=dev)
        st.ws = ws
        return st

    def pack_buffer(self, st: GpuShardFactor, key, n, dtype=None, zero=True):
        """Reusable device buffers of one rank's state (all-reduce packs, outputs),
        allocated once per (key, size) and zeroed in place on reuse."""
        dtype = dtype or self.torch.float64
        key = ("_cache",) + tuple(key)
        buf = st.bufs.get(key)
        if buf is None or buf.numel() != n or buf.dtype != dtype:
            buf = self.torch.zeros(n, dtype=dtype, device=self.device)
            st.bufs[key] = buf
        elif zero:
            buf.zero_()
        return buf

    def singular_flags(self, st: GpuShardFactor):
        """[leaf flags of all 2^L leaves | K flags of all 2^L - 1 blocks], this
        rank's entries filled (sum-all-reduced by the schedule)."""
        sh = st.shard
        nleaf, nl = 1 << sh.L, sh.n_loc // sh.m
        f = self.pack_buffer(st, ("flags",), 2 * nleaf - 1)
        a = sh.row0 // sh.m
        f[a : a + nl] = st.bufs["dinfo"].to(self.torch.float64)
        if sh.L:
            f[nleaf:] = st.bufs["kinfo"][: nleaf - 1].to(self.torch.float64)
        return f

    def raise_if_singular(self, st: GpuShardFactor, flags) -> None:
        raise_singular_from_flags(flags.cpu().numpy(), st.shard.L)

    def factor_local(self, st: GpuShardFactor, p: int):
        sh = st.shard
        out = self.pack_buffer(st, ("tw_out",), sh.r * sh.r * max(p, 1), zero=False)
        _lib.check(self.lib.hodlr_factorize_local(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, p, C.c_void_p(out.data_ptr()),
            C.c_void_p(st.ws.data_ptr()), st.wsb, self._stream()), "hodlr_factorize_local")
        return out

    def factor_top(self, st: GpuShardFactor, lv: int, tw_all):
        sh = st.shard
        out = self.pack_buffer(st, ("tw_out", lv), sh.r * sh.r * max(lv, 1), zero=False)
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

    def _check_x(self, st: GpuShardFactor, x, nrhs: int):
        torch = self.torch
        want = st.shard.n_loc * nrhs
        if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 or not x.is_cuda:
            raise TypeError("x_local must be a float64 CUDA tensor (the sharded solve is fp64-only)")
        if not x.is_contiguous() or x.numel() != want:
            raise ValueError(f"x_local must be contiguous with n_loc * nrhs = {want} entries (got {x.numel()})")

    def solve_local(self, st: GpuShardFactor, x, nrhs: int, p: int):
        sh = st.shard
        self._check_x(st, x, nrhs)
        ws, wsb = self._solve_ws(st, nrhs)
        out = self.pack_buffer(st, ("w_out", nrhs), sh.r * nrhs, zero=False)
        _lib.check(self.lib.hodlr_solve_local(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, p, C.c_void_p(x.data_ptr()), sh.n_loc, nrhs,
            C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), wsb, self._stream()), "hodlr_solve_local")
        return out

    def solve_top(self, st: GpuShardFactor, lv: int, w_all, x, nrhs: int):
        sh = st.shard
        self._check_x(st, x, nrhs)
        ws, wsb = self._solve_ws(st, nrhs)
        out = self.pack_buffer(st, ("w_out", nrhs, lv), sh.r * nrhs, zero=False)
        _lib.check(self.lib.hodlr_solve_top(
            C.byref(st.desc), C.byref(st.fac), sh.n_loc, sh.row0, lv, C.c_void_p(w_all.data_ptr()),
            C.c_void_p(out.data_ptr()), C.c_void_p(x.data_ptr()), sh.n_loc, nrhs, C.c_void_p(ws.data_ptr()), wsb,
            self._stream()), "hodlr_solve_top")
        return out


def factorize_sharded(shard: Shard, all_reduce=torch_all_reduce, backend=None, check: bool = True):
    """One rank's part of the sharded factorization (call on every rank).
    check=True all-reduces the singular flags and raises HodlrSingularError on
    every rank (one extra tiny all-reduce + a host sync)."""
    backend = backend or GpuBackend()
    return run(factorize_steps(shard, backend, check), all_reduce)


def solve_sharded(state, x_local, nrhs: int = 1, all_reduce=torch_all_reduce, backend=None):
    """One rank's part of the sharded solve; x_local (n_loc x nrhs, column-major) in place."""
    backend = backend or GpuBackend()
    return run(solve_steps(state, state.shard, backend, x_local, nrhs), all_reduce)
