"""HODLR container, factorization and solver on the B200 (SPEC modules
``hodlr_matrix`` / ``factorization`` / ``solver``).

Same operation names and semantics as the reference's SPEC API:

* :class:`HodlrMatrix` -- D_big (leaf blocks, leaf order), U_big / V_big
  level-concatenated N x rL column-major slabs (Fig. 3), uniform
  rank r, N = m 2^L; device-resident flat torch tensors.
* :func:`factorize` (PAPER Alg. 3) consumes ``h``: Y
  overwrites U in place and D holds its LU factors.
* :func:`solve` (PAPER Alg. 4) never mutates ``b``.
* :func:`logdet`, :func:`flop_report`, :func:`storage_report`.

All arithmetic runs in the sm_100a library through the C ABI; this module only
allocates device buffers and checks status / singular flags.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .backend import LuPivots, lu_factor_flops, lu_solve_flops, gemm_flops
from .tree import ClusterTree, build_tree

VARIANTS = ("pivoted_standard",)


class HodlrSingularError(RuntimeError):
    """A leaf block or K_gamma is singular to working precision."""

    def __init__(self, what: str, level: int, nodes):
        self.what, self.level, self.nodes = what, level, list(nodes)
        super().__init__(f"singular {what} block at level {level}, node(s) {self.nodes}")


def _torch():
    return _lib.require_cuda()


def _dtype_tag(t) -> int:
    import torch

    if t.dtype == torch.float64:
        return _lib.F64
    if t.dtype == torch.float32:
        return _lib.F32
    raise TypeError(f"unsupported dtype {t.dtype}")


@dataclass
class LevelPanel:
    """One level's basis panel in the SPEC's ragged layout:
    an n x width column-major buffer; node a of the level owns rows I_a and
    columns [col_offsets[a], col_offsets[a] + node_ranks[a])."""

    level: int
    data: "object"  # (n, width) array or flat column-major n * width
    col_offsets: "object"
    node_ranks: "object"

    @property
    def uniform(self) -> bool:
        nr = np.asarray(self.node_ranks)
        return bool(nr.size == 0 or (nr == nr[0]).all())


def _round_rank(r: int) -> int:
    """The fused kernels' ranks (16 / 32 / 64); other ranks run the generic path."""
    for q in (16, 32, 64):
        if r <= q:
            return q if r > 8 else r
    return r


def _host(x):
    return np.asarray(x.detach().cpu() if hasattr(x, "detach") else x)


def pad_level_panels(n: int, m: int, u_panels, v_panels, rank: int | None = None, round_rank: bool = True,
                     per_level: bool = False, with_ranks: bool = False):
    """Ragged LevelPanels (levels 1..L, per-node column offsets and ranks) ->
    (r, U, V): the uniform slabs of this engine, every node's basis zero-padded
    to rank r = the largest node rank (``rank`` overrides it; ``round_rank``
    rounds it up to a fused-kernel rank 16 / 32 / 64).  The padding changes
    nothing: padded U columns meet zero V columns, and K_p = [[T_a, I], [I,
    T_b]] stays invertible (its padded part is a permutation), so the oracle
    run on the same padded layout gives the same pivots."""
    L = int(round(math.log2(n // m))) if n >= m else 0
    if n != m << L:
        raise ValueError(f"GPU layout needs N = m 2^L (got N={n}, m={m})")
    ups = {int(p.level): p for p in u_panels}
    vps = {int(p.level): p for p in v_panels}
    if set(ups) != set(range(1, L + 1)) or set(vps) != set(range(1, L + 1)):
        raise ValueError(f"need one u and one v panel per level 1..{L}")
    rmax = 0
    for lv in range(1, L + 1):
        for p in (ups[lv], vps[lv]):
            nr = np.asarray(p.node_ranks, dtype=np.int64)
            if nr.shape != (1 << lv,):
                raise ValueError(f"level {lv}: node_ranks must have 2^{lv} entries")
            rmax = max(rmax, int(nr.max(initial=0)))
        # A(I_a, I_b) = U_a V_b^*: node a's U columns pair with its sibling's V columns
        if not np.array_equal(np.asarray(ups[lv].node_ranks).reshape(-1, 2),
                              np.asarray(vps[lv].node_ranks).reshape(-1, 2)[:, ::-1]):
            raise ValueError(f"level {lv}: U_a and V_b of a sibling pair need equal column counts")
    r = rank if rank is not None else (_round_rank(rmax) if round_rank else rmax)
    if r < rmax:
        raise ValueError(f"rank {r} < the largest node rank {rmax}")
    if per_level:  # each level padded to its own largest node rank (rounded)
        lr = []
        for lv in range(1, L + 1):
            k = int(max(np.asarray(ups[lv].node_ranks).max(initial=0), np.asarray(vps[lv].node_ranks).max(initial=0)))
            lr.append(_round_rank(k) if (round_rank and k > 0) else k)
        ranks = tuple(lr)
        r = max(ranks, default=0)
    else:
        ranks = (r,) * L
    dt = _host(ups[1].data).dtype if L else np.float64
    cc = np.concatenate([[0], np.cumsum(ranks)]).astype(np.int64)
    U = np.zeros((int(cc[-1]), n), dtype=dt)  # level l's n x ranks[l-1] column-major panel at rows cc[l-1]
    V = np.zeros((int(cc[-1]), n), dtype=dt)
    for lv in range(1, L + 1):
        nl = n >> lv
        for dstall, p in ((U, ups[lv]), (V, vps[lv])):
            dst = dstall[cc[lv - 1] : cc[lv]]
            a = _host(p.data).reshape(-1)
            width = a.size // n if n else 0
            if a.size != n * width:
                raise ValueError(f"level {lv}: panel has {a.size} entries, not a multiple of n = {n}")
            cols = a.reshape(width, n)  # column-major: column j at j n
            off = np.asarray(p.col_offsets, dtype=np.int64)
            nr = np.asarray(p.node_ranks, dtype=np.int64)
            for node in range(1 << lv):
                k, c0 = int(nr[node]), int(off[node])
                if c0 < 0 or c0 + k > width:
                    raise ValueError(f"level {lv} node {node}: columns [{c0}, {c0 + k}) outside the panel")
                dst[:k, node * nl : (node + 1) * nl] = cols[c0 : c0 + k, node * nl : (node + 1) * nl]
    if with_ranks:
        return r, U.reshape(-1), V.reshape(-1), (ranks if per_level else None)
    return r, U.reshape(-1), V.reshape(-1)


@dataclass
class HodlrMatrix:
    """Uniform-rank HODLR matrix in the concatenated big-matrix layout."""

    tree: ClusterTree
    rank: int
    D: "object"  # torch (2^L m^2,)  leaf a at a*m*m, column-major
    U: "object"  # torch (N C,)  ld N, level l' at columns [c_l', c_l' + r_l') (uniform: (l'-1) r)
    V: "object"  # torch (N C,)
    ranks: tuple | None = None  # per-level ranks (level l' at ranks[l'-1]); None: ``rank`` everywhere

    @property
    def level_ranks(self) -> tuple:
        return tuple(self.ranks) if self.ranks is not None else (self.rank,) * self.L

    @property
    def cols(self) -> int:
        return sum(self.level_ranks)

    @property
    def n(self) -> int:
        return self.tree.n

    @property
    def L(self) -> int:
        return self.tree.depth

    @property
    def m(self) -> int:
        return self.tree.n >> self.tree.depth

    @property
    def dtype(self):
        return self.D.dtype

    def desc(self) -> _lib.Desc:
        return _lib.make_desc(self.n, self.m, self.rank, self.L, _dtype_tag(self.D), self.ranks)

    @classmethod
    def from_buffers(cls, n: int, m: int, r: int, D, U, V, device="cuda", ranks=None) -> "HodlrMatrix":
        """Wrap flat buffers (numpy or torch) in the reference layout; copies to
        ``device``.  ``ranks``: per-level ranks (level l' at ranks[l'-1]; the
        slabs then have sum(ranks) columns and ``r`` is ignored)."""
        torch = _torch()
        L = int(round(math.log2(n // m))) if n >= m else 0
        if n != m << L:
            raise ValueError(f"GPU layout needs N = m 2^L (got N={n}, m={m})")
        tree = ClusterTree(n, L)
        if ranks is not None:
            ranks = tuple(int(x) for x in ranks)
            if len(ranks) != L or min(ranks, default=0) < 0:
                raise ValueError(f"ranks: {L} non-negative per-level ranks expected (got {ranks})")
            r = max(ranks, default=0)
            if len(set(ranks)) <= 1 and (not ranks or ranks[0] == r):
                ranks = None  # uniform
        C_ = sum(ranks) if ranks is not None else r * L

        def dev(x, size, name):
            t = torch.as_tensor(x).reshape(-1).to(device)
            if t.numel() != size:
                raise ValueError(f"{name} has {t.numel()} entries, expected {size}")
            return t.contiguous()

        return cls(tree, r, dev(D, (1 << L) * m * m, "D"), dev(U, n * C_, "U"), dev(V, n * C_, "V"), ranks)

    @classmethod
    def from_level_panels(cls, n: int, m: int, d_big, u_panels, v_panels, rank: int | None = None,
                          round_rank: bool = True, device="cuda", per_level: bool = True) -> "HodlrMatrix":
        """Ingest the SPEC's ragged representation;
        see :func:`pad_level_panels`.  per_level=True pads each level to its own
        (rounded) rank -- the per-level-rank layout of ``hodlr_desc.ranks`` --
        else every level to one rank."""
        r, U, V, ranks = pad_level_panels(n, m, u_panels, v_panels, rank, round_rank, per_level=per_level,
                                          with_ranks=True)
        D = np.asarray(d_big.cpu() if hasattr(d_big, "cpu") else d_big)
        return cls.from_buffers(n, m, r, D, U.astype(D.dtype, copy=False), V.astype(D.dtype, copy=False), device=device,
                                ranks=ranks)

    def clone(self) -> "HodlrMatrix":
        return HodlrMatrix(self.tree, self.rank, self.D.clone(), self.U.clone(), self.V.clone(), self.ranks)

    def storage_report(self) -> dict:
        """Scalar counts vs Thm. 2: diag m N, bases 2 r N L."""
        n, m, C_ = self.n, self.m, self.cols
        es = self.D.element_size()
        return {
            "scalars_diagonal": m * n,
            "scalars_bases": 2 * C_ * n,
            "bytes_diagonal": m * n * es,
            "bytes_bases": 2 * C_ * n * es,
            "formula_prediction": m * n + 2 * C_ * n,
            "factorization_scalars_thm2": m * n + C_ * n,
        }

    def matvec(self, x, stream=None):
        """A x on the device: ``hodlr_matvec``, two HBM
        streams (w = V^T x for all levels, then D x + U w_sibling).  ``x`` is
        (N,) or (N, k) torch (device or host) or numpy; same kind/shape out."""
        torch = _torch()
        lib = _lib.load()
        is_np = isinstance(x, np.ndarray)
        xt = torch.from_numpy(np.ascontiguousarray(x)) if is_np else x
        n = self.n
        if xt.dim() not in (1, 2) or xt.shape[0] != n:
            raise ValueError(f"matvec: x must have {n} rows (got shape {tuple(xt.shape)})")
        nrhs = 1 if xt.dim() == 1 else xt.shape[1]
        dev = self.D.device
        desc = self.desc()
        wsb = lib.hodlr_matvec_workspace(C.byref(desc), nrhs)
        so = stream or torch.cuda.current_stream(dev)
        with torch.cuda.device(dev), torch.cuda.stream(so):
            xd = xt.to(device=dev, non_blocking=True) if xt.device != dev else xt
            X = torch.empty((nrhs, n), dtype=self.dtype, device=dev)  # column-major N x nrhs
            _to_column_major(xd, X, so)
            Y = torch.empty_like(X)
            ws = _workspace(wsb, dev, so) if wsb else None
            _lib.check(
                lib.hodlr_matvec(C.byref(desc), C.c_void_p(self.D.data_ptr()), C.c_void_p(self.U.data_ptr()),
                                 C.c_void_p(self.V.data_ptr()), C.c_void_p(X.data_ptr()), n,
                                 C.c_void_p(Y.data_ptr()), n, nrhs,
                                 C.c_void_p(ws.data_ptr() if ws is not None else 0), wsb, C.c_void_p(so.cuda_stream)),
                "hodlr_matvec",
            )
            out = Y.t().reshape(xt.shape)
            if (is_np or xt.device != dev) and nrhs > 1 and Y.dtype == torch.float64:
                rm = torch.empty((n, nrhs), dtype=Y.dtype, device=dev)  # row-major on the device first
                _lib.check(lib.hodlr_transpose_f64(C.c_void_p(Y.data_ptr()), nrhs, n, n, C.c_void_p(rm.data_ptr()),
                                                   nrhs, C.c_void_p(so.cuda_stream)), "hodlr_transpose_f64")
                out = rm.reshape(xt.shape)
            if is_np:
                res = out.cpu().numpy()  # synchronous on `so`
            elif xt.device != dev:
                res = out.to(xt.device)
            else:
                res = out
        if stream is not None and not is_np:
            # the caller's current stream consumes the result: order it after `so`
            torch.cuda.current_stream(dev).wait_stream(so)
        return res

    def reconstruct_dense(self):
        torch = _torch()
        n = self.n
        if n > 8192:
            raise ValueError("reconstruct_dense size guard (n > 8192)")
        return self.matvec(torch.eye(n, dtype=self.dtype, device=self.D.device))


@dataclass
class HodlrFactorization:
    """In-place product form plus the explicit inverses."""

    tree: ClusterTree
    rank: int
    D: "object"     # leaf LU
    Dinv: "object"  # leaf inverses
    Y: "object"     # Y slab (overwrote U)
    V: "object"
    K: "object"     # K LU, level l at (2^l - 1)(2r)^2
    Kinv: "object"
    dswaps: "object"
    dperm: "object"
    dinfo: "object"
    kswaps: "object"
    kperm: "object"
    kinfo: "object"
    variant: str = "pivoted_standard"
    flops: dict = field(default_factory=dict)
    ranks: tuple | None = None  # per-level ranks (as the factored HodlrMatrix)

    @property
    def level_ranks(self) -> tuple:
        return tuple(self.ranks) if self.ranks is not None else (self.rank,) * self.L

    def _k_offsets(self, level: int):
        """(K offset, pivot offset, rank) of parent level ``level``'s blocks."""
        ko = kp = 0
        rk = self.level_ranks
        for lv in range(level):
            s = 2 * rk[lv]
            ko += (1 << lv) * s * s
            kp += (1 << lv) * s
        return ko, kp, rk[level]

    @property
    def n(self):
        return self.tree.n

    @property
    def L(self):
        return self.tree.depth

    @property
    def m(self):
        return self.tree.n >> self.tree.depth

    def desc(self) -> _lib.Desc:
        return _lib.make_desc(self.n, self.m, self.rank, self.L, _dtype_tag(self.D), self.ranks)

    def cfactors(self) -> _lib.Factors:
        p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        return _lib.Factors(
            p(self.D), p(self.Dinv), p(self.Y), p(self.V), p(self.K), p(self.Kinv),
            p(self.dswaps), p(self.dperm), p(self.dinfo), p(self.kswaps), p(self.kperm), p(self.kinfo),
        )

    def leaf_pivots(self) -> LuPivots:
        nl, m = 1 << self.L, self.m
        sw = self.dswaps.view(nl, m).cpu().numpy().astype(np.int64)
        pm = self.dperm.view(nl, m).cpu().numpy().astype(np.int64)
        return LuPivots(sw, pm, [int(i) for i in np.flatnonzero(self.dinfo.cpu().numpy())])

    def k_pivots(self, level: int) -> LuPivots:
        _, lo, r = self._k_offsets(level)
        r2, npar = 2 * r, 1 << level
        sw = self.kswaps[lo : lo + npar * r2].view(npar, r2).cpu().numpy().astype(np.int64)
        pm = self.kperm[lo : lo + npar * r2].view(npar, r2).cpu().numpy().astype(np.int64)
        info = self.kinfo[npar - 1 : 2 * npar - 1].cpu().numpy()
        return LuPivots(sw, pm, [int(i) for i in np.flatnonzero(info)])

    def k_block(self, level: int):
        lo, _, r = self._k_offsets(level)
        r2, npar = 2 * r, 1 << level
        return self.K[lo : lo + npar * r2 * r2]


_WS_CACHE: dict = {}


def _dinv_size(nblocks: int, s: int, fp64: bool = True) -> int:
    """Scalars of the factorization-internal solve aids (``Dinv`` / ``Kinv``)
    for ``nblocks`` s x s blocks: 8 s per block (8x8 diagonal-block inverses,
    s in {32, 64, 128}), s^2 (packed inverses, s = 16), none otherwise; the fp32
    path forms them on the fly (``hodlr_inv_elems``, include/hodlr_b200.h)."""
    per = int(_lib.load().hodlr_inv_elems(s)) if fp64 else 0
    return max(nblocks * per, 1)


def _workspace(nbytes: int, device, stream=None):
    """Reusable device workspace (bytes) per (device, stream), grown on demand.
    Calls on one stream are ordered, so they can share it; calls on different
    streams (e.g. concurrent solves on one factorization) get
    their own buffer, allocated on that stream."""
    torch = _torch()
    s = stream or torch.cuda.current_stream(device)
    key = (str(device), s.cuda_stream)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        _WS_CACHE.pop(key, None)
        with torch.cuda.stream(s):
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


def flop_report(n: int, m: int, r: int, ranks=None) -> dict:
    """Per-phase factor flops with the reference counters (backend.py:240-251);
    ``ranks``: per-level ranks (level l' at ranks[l'-1])."""
    L = int(round(math.log2(n // m)))
    nl = 1 << L
    rk = list(ranks) if ranks is not None else [r] * L
    cc = [0]
    for k in rk:
        cc.append(cc[-1] + k)
    rep = {
        "leaf_getrf": lu_factor_flops(m) * nl,
        "leaf_getrs": lu_solve_flops(m, cc[L]) * nl if L else 0,
        "tw_gemm": 0, "k_getrf": 0, "k_getrs": 0, "update_gemm": 0, "per_level_gemm": {},
    }
    for lv in range(L):
        nc = n >> (lv + 1)
        k, wc = rk[lv], cc[lv]  # rank of level lv + 1, columns of levels 1..lv
        if k == 0:
            rep["per_level_gemm"][lv] = 0
            continue
        tw = gemm_flops(k, nc, wc + k) * (1 << (lv + 1))
        up = gemm_flops(nc, k, wc) * (1 << (lv + 1)) if lv and wc else 0
        rep["tw_gemm"] += tw
        rep["update_gemm"] += up
        rep["k_getrf"] += lu_factor_flops(2 * k) * (1 << lv)
        rep["k_getrs"] += lu_solve_flops(2 * k, wc) * (1 << lv) if lv and wc else 0
        rep["per_level_gemm"][lv] = tw + up
    rep["total"] = sum(v for k, v in rep.items() if k != "per_level_gemm")
    return rep


def solve_flops(n: int, m: int, r: int, nrhs: int = 1) -> int:
    """2mN + 4rNL + 8r^2(2^L - 1) per column (Thm. 4 plus the K term)."""
    L = int(round(math.log2(n // m)))
    return nrhs * (2 * m * n + 4 * r * n * L + 8 * r * r * ((1 << L) - 1))


def _alloc_factorization(h: HodlrMatrix, variant: str = "pivoted_standard") -> HodlrFactorization:
    """Output buffers of a factorization of ``h`` (Y / D overwrite h's U / D)."""
    torch = _torch()
    dev = h.D.device
    fp64 = h.D.dtype == torch.float64
    n, m, r, L = h.n, h.m, h.rank, h.L
    nl = 1 << L
    nk = nl - 1
    rk = h.level_ranks
    ksz = sum((1 << lv) * (2 * rk[lv]) ** 2 for lv in range(L))
    kps = sum((1 << lv) * 2 * rk[lv] for lv in range(L))
    kis = sum(_dinv_size(1 << lv, 2 * rk[lv], fp64) for lv in range(L)) if L else 1
    i32 = dict(dtype=torch.int32, device=dev)
    return HodlrFactorization(
        tree=h.tree, rank=r, D=h.D, Dinv=torch.empty(_dinv_size(nl, m, fp64), dtype=h.D.dtype, device=dev),
        Y=h.U, V=h.V, K=torch.empty(ksz, dtype=h.D.dtype, device=dev),
        Kinv=torch.empty(max(kis, 1), dtype=h.D.dtype, device=dev),
        dswaps=torch.empty(nl * m, **i32), dperm=torch.empty(nl * m, **i32), dinfo=torch.zeros(nl, **i32),
        kswaps=torch.empty(max(kps, 1), **i32), kperm=torch.empty(max(kps, 1), **i32),
        kinfo=torch.zeros(max(nk, 1), **i32), variant=variant, flops=flop_report(n, m, r, ranks=h.ranks),
        ranks=h.ranks,
    )


def factorize(h: HodlrMatrix, variant: str = "pivoted_standard", check: bool = True, stream=None) -> HodlrFactorization:
    """Level-wise batched factorization (PAPER Alg. 3).  Consumes ``h``.

    Raises :class:`HodlrSingularError` naming level and node when a leaf or
    K_gamma block is flagged singular.
    """
    torch = _torch()
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r} (supported: {VARIANTS})")
    if h.D.dtype not in (torch.float64, torch.float32):
        raise TypeError(f"unsupported dtype {h.D.dtype} (float64: DMMA path; float32: preconditioner path)")
    if h.ranks is not None and h.D.dtype != torch.float64:
        raise TypeError("per-level ranks: float64 only (the fp32 preconditioner path takes one rank)")
    lib = _lib.load()
    dev = h.D.device
    f = _alloc_factorization(h, variant)
    desc = h.desc()
    wsb = lib.hodlr_factorize_workspace(C.byref(desc))
    so = stream or torch.cuda.current_stream(dev)
    ws = _workspace(wsb, dev, so)
    st = so.cuda_stream
    cf = f.cfactors()
    _lib.check(lib.hodlr_factorize(C.byref(desc), C.byref(cf), C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(st)),
               "hodlr_factorize")
    if check:
        _raise_if_singular(f)
    return f


_COPY_STREAMS: dict = {}


def factorize_from_host(n: int, m: int, r: int, D, U, V, variant: str = "pivoted_standard", check: bool = True,
                        device="cuda", stream=None) -> HodlrFactorization:
    """Factorize a HODLR matrix held in host memory (reference layout, fp64),
    overlapping the upload with the factorization: D, U and the last level's V
    go first, then the V panels in the order the levels consume them, on a
    side copy stream (``hodlr_factorize_from_host``).  Pinned host buffers
    (``tensor.pin_memory()``) are copied directly; pageable ones (numpy arrays)
    stream through the library's pinned staging ring (multi-threaded host
    copies, the factorization enqueued as the level panels arrive), and may be
    freed as soon as this returns.  Equivalent to
    ``factorize(HodlrMatrix.from_buffers(...))``."""
    torch = _torch()
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r} (supported: {VARIANTS})")
    lib = _lib.load()
    L = int(round(math.log2(n // m))) if n >= m else 0
    if n != m << L:
        raise ValueError(f"GPU layout needs N = m 2^L (got N={n}, m={m})")
    nl, nk = 1 << L, (1 << L) - 1

    def host(x, size, name):
        t = torch.as_tensor(x).reshape(-1)
        if t.dtype != torch.float64:
            raise TypeError(f"{name} must be float64 (got {t.dtype})")
        if t.numel() != size:
            raise ValueError(f"{name} has {t.numel()} entries, expected {size}")
        if t.is_cuda:
            raise ValueError(f"{name} is already on the device; use HodlrMatrix.from_buffers")
        return t.contiguous()

    Dh, Uh, Vh = host(D, nl * m * m, "D"), host(U, n * r * L, "U"), host(V, n * r * L, "V")
    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    f64 = dict(dtype=torch.float64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        f = HodlrFactorization(
            tree=ClusterTree(n, L), rank=r, D=torch.empty(nl * m * m, **f64), Dinv=torch.empty(_dinv_size(nl, m), **f64),
            Y=torch.empty(n * r * L, **f64), V=torch.empty(n * r * L, **f64),
            K=torch.empty(max(nk, 1) * 4 * r * r, **f64), Kinv=torch.empty(_dinv_size(max(nk, 1), 2 * r), **f64),
            dswaps=torch.empty(nl * m, **i32), dperm=torch.empty(nl * m, **i32), dinfo=torch.zeros(nl, **i32),
            kswaps=torch.empty(max(nk, 1) * 2 * r, **i32), kperm=torch.empty(max(nk, 1) * 2 * r, **i32),
            kinfo=torch.zeros(max(nk, 1), **i32), variant=variant, flops=flop_report(n, m, r),
        )
        f.host_inputs = (Dh, Uh, Vh)  # alive until the asynchronous upload has completed
        desc = f.desc()
        wsb = lib.hodlr_factorize_workspace(C.byref(desc))
        st = (stream or torch.cuda.current_stream(dev))
        ws = _workspace(wsb, dev, st)
        key = dev.index
        if key not in _COPY_STREAMS:
            _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
        cs = _COPY_STREAMS[key]
        cf = f.cfactors()
        _lib.check(lib.hodlr_factorize_from_host(C.byref(desc), C.byref(cf), C.c_void_p(Dh.data_ptr()),
                                                 C.c_void_p(Uh.data_ptr()), C.c_void_p(Vh.data_ptr()),
                                                 C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(st.cuda_stream),
                                                 C.c_void_p(cs.cuda_stream)), "hodlr_factorize_from_host")
    if check:
        _raise_if_singular(f)
    return f


def _raise_if_singular(f: HodlrFactorization) -> None:
    torch = _torch()
    flags = torch.cat([f.dinfo, f.kinfo]).cpu().numpy()
    if not flags.any():
        return
    nl = 1 << f.L
    bad = np.flatnonzero(flags[:nl])
    if bad.size:
        raise HodlrSingularError("leaf", f.L, bad.tolist())
    kf = flags[nl:]
    for lv in range(f.L):
        seg = kf[(1 << lv) - 1 : (2 << lv) - 1]
        if seg.any():
            raise HodlrSingularError("K", lv, np.flatnonzero(seg).tolist())


def _capture(launch, stream, dev):
    """CUDA graph of ``launch(cuda_stream)`` captured on a side stream ordered
    after ``stream`` (thread-local capture mode: other threads' CUDA calls are
    unaffected)."""
    torch = _torch()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        g.capture_begin(capture_error_mode="thread_local")
        try:
            launch(side.cuda_stream)
        finally:
            g.capture_end()
    stream.wait_stream(side)
    return g


class _SolveGraph:
    """One captured ``hodlr_solve`` (CUDA graph) of a factorization for a fixed
    nrhs on one stream: its own X buffer and workspace (the graph bakes their
    addresses), replayed after the rhs is copied in."""

    def __init__(self, fact, nrhs: int, stream):
        torch = _torch()
        lib = _lib.load()
        n, dev = fact.n, fact.D.device
        self.nrhs = nrhs
        desc = fact.desc()
        wsb = lib.hodlr_solve_workspace(C.byref(desc), nrhs)
        with torch.cuda.device(dev), torch.cuda.stream(stream):
            self.X = torch.zeros(nrhs, n, dtype=fact.D.dtype, device=dev)  # column-major N x nrhs
            self.ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        cf = fact.cfactors()
        self._args = (C.byref(desc), C.byref(cf), C.c_void_p(self.X.data_ptr()), n, nrhs,
                      C.c_void_p(self.ws.data_ptr()), wsb)
        self._keep = (desc, cf)
        # kernel attributes / lazy module loading happened in the caller's eager
        # first call; capture directly (no torch.cuda.graph gc / cache flush)
        self.graph = _capture(lambda st: _lib.check(lib.hodlr_solve(*self._args, C.c_void_p(st)),
                                                    "hodlr_solve (capture)"), stream, dev)

    def run_from(self, bd, stream):
        """bd: the (N,) / (N, nrhs) rhs on the device; returns a new (nrhs, N)
        contiguous solution (column-major N x nrhs)."""
        torch = _torch()
        with torch.cuda.stream(stream):
            _to_column_major(bd, self.X, stream)
            self.graph.replay()
            return self.X.clone()


def _to_column_major(bd, out, stream):
    """out (nrhs, N) contiguous <- the rhs bd (N,) or (N, nrhs): one copy, and for a
    row-major fp64 block the library's tiled transpose (torch's strided copy of
    this shape runs at ~0.8 TB/s)."""
    torch = _torch()
    n, k = out.shape[1], out.shape[0]
    b2 = bd.reshape(n, k)
    if k > 1 and b2.dtype == torch.float64 and out.dtype == torch.float64 and b2.stride(1) == 1 and b2.stride(0) >= k:
        _lib.check(_lib.load().hodlr_transpose_f64(C.c_void_p(b2.data_ptr()), n, k, b2.stride(0),
                                                   C.c_void_p(out.data_ptr()), n, C.c_void_p(stream.cuda_stream)),
                   "hodlr_transpose_f64")
    else:
        out.copy_(b2.t())


_GRAPH_AUTO_BYTES = 1 << 28  # graph=None: capture solves whose rhs block is <= 256 MB


def _solve_eager(lib, fact, x, nrhs, dev, so):
    desc = fact.desc()
    wsb = lib.hodlr_solve_workspace(C.byref(desc), nrhs)
    ws = _workspace(wsb, dev, so)
    cf = fact.cfactors()
    _lib.check(lib.hodlr_solve(C.byref(desc), C.byref(cf), C.c_void_p(x.data_ptr()), fact.n, nrhs,
                               C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(so.cuda_stream)), "hodlr_solve")


def solve(fact: HodlrFactorization, b, stream=None, graph: bool | None = None):
    """x = A^-1 b (PAPER Alg. 4).  ``b``: (N,) or (N, k), torch (device or host)
    or numpy; the result has the same kind/shape and ``b`` is not modified.

    The level-by-level launch sequence of ``hodlr_solve`` (~4 L small
    launches) can run as a CUDA graph captured per (factorization, nrhs,
    stream): graph=None (default) launches the first solve of a key eagerly and
    captures from the second on when the rhs block is at most 256 MB (repeated
    latency-bound solves replay, one-shot solves pay no capture, big multi-RHS
    solves stay eager); graph=True captures at once; graph=False always
    launches eagerly.  All run the same kernels on the same data, bit for bit."""
    torch = _torch()
    lib = _lib.load()
    is_np = isinstance(b, np.ndarray)
    bt = torch.from_numpy(np.ascontiguousarray(b)) if is_np else b
    n = fact.n
    if bt.shape[0] != n or bt.dim() not in (1, 2):
        raise ValueError(f"rhs must have {n} rows (got shape {tuple(bt.shape)})")
    nrhs = 1 if bt.dim() == 1 else bt.shape[1]
    dev = fact.D.device
    so = stream or torch.cuda.current_stream(dev)
    with torch.cuda.device(dev), torch.cuda.stream(so):
        # upload first (a pinned host rhs is one async DMA), then lay out column-major
        # on the device: (nrhs, n) row-major == (n, nrhs) column-major
        bd = bt.to(device=dev, non_blocking=True) if bt.device != dev else bt
        key = (nrhs, so.cuda_stream)
        graphs = fact.__dict__.setdefault("_solve_graphs", {})
        g = graphs.get(key) if (graph is not False and nrhs > 0) else None
        if g is not None and not torch.cuda.is_current_stream_capturing():
            # replay: lay b out column-major straight into the graph's buffer,
            # then one copy out (the graph owns and reuses its X)
            x = g.run_from(bd, so)
        else:
            x = torch.empty((nrhs, n), dtype=fact.D.dtype, device=dev)
            _to_column_major(bd, x, so)
        if nrhs > 0 and (g is None or torch.cuda.is_current_stream_capturing()):
            _solve_eager(lib, fact, x, nrhs, dev, so)
            if graph is not False and not torch.cuda.is_current_stream_capturing():
                calls = fact.__dict__.setdefault("_solve_calls", {})
                calls[key] = calls.get(key, 0) + 1
                # capture after the eager call(s) -- later calls replay.  graph=None captures
                # only latency-bound sizes (the graph owns an N x nrhs buffer + workspace)
                small = n * nrhs * x.element_size() <= _GRAPH_AUTO_BYTES
                if graph or (calls[key] >= 2 and small):
                    graphs[key] = _SolveGraph(fact, nrhs, so)
        out = x.t().reshape(bt.shape)
        if bt.device == dev:
            return out
        # host result: back to row-major on the device, async copy into pinned memory, wait
        if nrhs > 1 and x.dtype == torch.float64:
            rm = torch.empty((n, nrhs), dtype=x.dtype, device=dev)
            _lib.check(lib.hodlr_transpose_f64(C.c_void_p(x.data_ptr()), nrhs, n, n, C.c_void_p(rm.data_ptr()), nrhs,
                                               C.c_void_p(so.cuda_stream)), "hodlr_transpose_f64")
            out = rm.reshape(bt.shape)
        host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        host.copy_(out, non_blocking=True)
        so.synchronize()
    return host.numpy() if is_np else host


class FactorPlan:
    """Repeated factorizations of one HodlrMatrix's buffers through a captured
    CUDA graph (e.g. time stepping, or refactoring after the
    operator's entries change in place).

    ``FactorPlan(h)`` factors ``h`` once eagerly (``self.factorization`` is
    valid afterwards) and captures the same launch sequence of
    ``hodlr_factorize`` on the same buffers.  Refill ``h``'s D / U / V in place
    (``load``) and call ``refactor()``: the graph replays every level's
    kernels with no host enqueue between them; results are bit-identical to
    ``factorize``.  The plan owns its workspace."""

    def __init__(self, h: HodlrMatrix, check: bool = True, stream=None):
        torch = _torch()
        lib = _lib.load()
        dev = h.D.device
        self.h = h
        so = stream or torch.cuda.current_stream(dev)
        desc = h.desc()
        wsb = lib.hodlr_factorize_workspace(C.byref(desc))
        with torch.cuda.device(dev), torch.cuda.stream(so):
            self.ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
            f = _alloc_factorization(h)
        self.factorization = f
        cf = f.cfactors()
        self._keep = (desc, cf)
        self._args = (C.byref(desc), C.byref(cf), C.c_void_p(self.ws.data_ptr()), wsb)
        _lib.check(lib.hodlr_factorize(*self._args, C.c_void_p(so.cuda_stream)), "hodlr_factorize")
        if check:
            _raise_if_singular(f)
        # capture over the SAME buffers (nothing executes during capture)
        self.graph = _capture(lambda st: _lib.check(lib.hodlr_factorize(*self._args, C.c_void_p(st)),
                                                    "hodlr_factorize (capture)"), so, dev)

    def load(self, D=None, U=None, V=None) -> None:
        """Copy new operator entries (same layout / sizes) into the plan's buffers."""
        for dst, src in ((self.h.D, D), (self.h.U, U), (self.h.V, V)):
            if src is not None:
                dst.copy_(_torch().as_tensor(src).reshape(-1), non_blocking=True)

    def refactor(self, check: bool = True, stream=None) -> HodlrFactorization:
        """Replay the captured factorization on the current contents of h."""
        torch = _torch()
        so = stream or torch.cuda.current_stream(self.h.D.device)
        with torch.cuda.stream(so):
            self.graph.replay()
        if check:
            _raise_if_singular(self.factorization)
        return self.factorization


def logdet(fact: HodlrFactorization):
    """(log|det A|, sign) from the stored LU diagonals.

    det(I + Z X^T) = det(I + X^T Z) = det(K_p) (-1)^{r_a r_b}: K_p is
    I + X^T Z with its two r-wide block columns exchanged.
    """
    torch = _torch()
    n, m, r, L = fact.n, fact.m, fact.rank, fact.L
    nl = 1 << L
    dd = fact.D.view(nl, m, m).diagonal(dim1=1, dim2=2)
    logabs = torch.log(dd.abs()).sum()
    neg = (dd < 0).sum()
    ar = torch.arange(m, device=dd.device, dtype=torch.int32)
    nswap = (fact.dswaps.view(nl, m) != ar).sum()
    blockswap = 0
    if L and fact.ranks is None:
        nk, r2 = nl - 1, 2 * r
        kd = fact.K.view(nk, r2, r2).diagonal(dim1=1, dim2=2)
        logabs = logabs + torch.log(kd.abs()).sum()
        neg = neg + (kd < 0).sum()
        ak = torch.arange(r2, device=dd.device, dtype=torch.int32)
        nswap = nswap + (fact.kswaps[: nk * r2].view(nk, r2) != ak).sum()
        blockswap = nk * (r * r % 2)
    elif L:  # per-level ranks: level by level
        for lv in range(L):
            ko, kp, k = fact._k_offsets(lv)
            if k == 0:
                continue
            npar, r2 = 1 << lv, 2 * k
            kd = fact.K[ko : ko + npar * r2 * r2].view(npar, r2, r2).diagonal(dim1=1, dim2=2)
            logabs = logabs + torch.log(kd.abs()).sum()
            neg = neg + (kd < 0).sum()
            ak = torch.arange(r2, device=dd.device, dtype=torch.int32)
            nswap = nswap + (fact.kswaps[kp : kp + npar * r2].view(npar, r2) != ak).sum()
            blockswap += npar * (k * k % 2)
    parity = (int(neg) + int(nswap) + blockswap) % 2
    return float(logabs), (-1.0 if parity else 1.0)


@dataclass
class RefinementResult:
    """Best iterate of :func:`solve_with_refinement` plus its relres history."""

    x: "object"
    history: list
    iterations: int
    diverged: bool


def solve_with_refinement(fact: HodlrFactorization, h: HodlrMatrix, b, max_iters: int = 10,
                          tol: float = 0.0) -> RefinementResult:
    """Iterative refinement x <- x + fact.solve(b - A x).

    ``h`` is the unfactored operator in the working precision (its dtype is
    the refinement dtype; ``fact`` may be a lower-precision factorization,
    e.g. the fp32 preconditioner of cfg4).  Residuals use the device matvec
    (``hodlr_matvec``).  Stops after ``max_iters`` corrections, once relres
    <= ``tol``, or when relres stops improving; divergence (relres grows on
    two consecutive iterations) returns the best iterate with
    ``diverged=True``.  ``history[k]`` is the relres after k corrections.
    """
    torch = _torch()
    is_np = isinstance(b, np.ndarray)
    bt = torch.from_numpy(np.ascontiguousarray(b)) if is_np else b
    dev = h.D.device
    bw = bt.to(device=dev, dtype=h.dtype)
    nb = float(torch.linalg.norm(bw))

    def out(x, hist, it, div):
        xo = x.cpu().numpy() if is_np else (x.to(bt.device) if bt.device != dev else x)
        return RefinementResult(xo, hist, it, div)

    if nb == 0.0:  # b = 0 -> x = 0 immediately
        return out(torch.zeros_like(bw), [0.0], 0, False)
    x = solve(fact, bw).to(h.dtype)
    res = bw - h.matvec(x)
    rel = float(torch.linalg.norm(res)) / nb
    hist = [rel]
    best, best_rel, stall, diverged, it = x, rel, 0, False, 0
    while it < max_iters and best_rel > tol:
        x = x + solve(fact, res).to(h.dtype)
        it += 1
        res = bw - h.matvec(x)
        new = float(torch.linalg.norm(res)) / nb
        hist.append(new)
        if new < best_rel * (1.0 - 1e-3):  # still improving
            best, best_rel, stall = x, new, 0
            continue
        stall += 1
        if len(hist) >= 3 and hist[-1] > hist[-2] > hist[-3]:  # grew on two consecutive iterations
            diverged = True
            break
        if stall >= 2:  # stopped improving
            break
    return out(best, hist, it, diverged)


# ---------------------------------------------------------------------------
# synthetic inputs (SURVEY.md §8d exact-HODLR stand-in), generated on device
# ---------------------------------------------------------------------------


def random_hodlr(n: int, m: int, r: int, seed: int = 0, s: float = 1.0, device="cuda", dtype=None,
                 ranks=None) -> HodlrMatrix:
    """Seeded exact HODLR generated directly in HBM (uniform rank r, or
    per-level ``ranks``, level l' at ranks[l'-1]).

    D_a = N(0,1)/sqrt(m) + 4 I; level-l U ~ N(0, s^2/n_l), V ~ N(0, 1/n_l).
    (Same distribution as the oracle's numpy generator; different stream.)
    """
    torch = _torch()
    dtype = dtype or torch.float64
    L = int(round(math.log2(n // m)))
    if n != m << L:
        raise ValueError("need N = m 2^L")
    rk = tuple(int(x) for x in ranks) if ranks is not None else (r,) * L
    if len(rk) != L:
        raise ValueError(f"ranks: {L} per-level ranks expected")
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    nl = 1 << L
    D = torch.randn(nl * m * m, generator=g, device=device, dtype=dtype).mul_(1.0 / math.sqrt(m))
    D.view(nl, m, m).diagonal(dim1=1, dim2=2).add_(4.0)
    C_ = sum(rk)
    U = torch.randn(n * C_, generator=g, device=device, dtype=dtype)
    V = torch.randn(n * C_, generator=g, device=device, dtype=dtype)
    c0 = 0
    for lv in range(1, L + 1):
        nlv = n >> lv
        sl = slice(c0 * n, (c0 + rk[lv - 1]) * n)
        U[sl].mul_(s / math.sqrt(nlv))
        V[sl].mul_(1.0 / math.sqrt(nlv))
        c0 += rk[lv - 1]
    if ranks is None:
        return HodlrMatrix(ClusterTree(n, L), r, D, U, V)
    return HodlrMatrix.from_buffers(n, m, 0, D, U, V, device=device, ranks=rk)


def tree_for(n: int, leaf_size: int) -> ClusterTree:
    return build_tree(n, leaf_size)


def truncate_ranks(h: HodlrMatrix, ranks) -> HodlrMatrix:
    """Per-level rank truncation of a uniform-rank HodlrMatrix: level l' keeps
    its first ranks[l'-1] basis columns (ACA crosses are ordered by
    selection, so the leading ones form the rank-k approximation), giving the
    per-level-rank layout of ``hodlr_desc.ranks`` (e.g. the paper's rank
    profiles, PAPER.md appendix).  A new matrix; ``h`` is unchanged."""
    torch = _torch()
    L, n, r = h.L, h.n, h.rank
    rk = tuple(int(x) for x in ranks)
    if len(rk) != L or any(k < 0 or k > r for k in rk):
        raise ValueError(f"ranks: {L} per-level ranks in [0, {r}] expected")
    if h.ranks is not None:
        raise ValueError("truncate_ranks expects a uniform-rank matrix")
    U = torch.cat([h.U.view(L, r, n)[lv, : rk[lv]].reshape(-1) for lv in range(L)]) if L else h.U[:0]
    V = torch.cat([h.V.view(L, r, n)[lv, : rk[lv]].reshape(-1) for lv in range(L)]) if L else h.V[:0]
    return HodlrMatrix.from_buffers(n, h.m, 0, h.D.clone(), U, V, device=h.D.device, ranks=rk)
