"""HODLR assembly on the device (SPEC.md:163-171 [OP] assemble).

Leaf blocks are materialized exactly and every sibling off-diagonal block is
compressed by adaptive cross approximation with rook pivoting at a fixed rank
cap (the reference's ``compress(..., CompressionConfig(tol=0, max_rank=r,
method="aca_rook_pivot"))``, compress.py:87-200), all blocks of a level in
lockstep on the GPU (``hodlr_build_*``, csrc/build.cu).

Entry oracles:

* :func:`laplace_dl_hodlr` -- the cfg2 problem: exterior Dirichlet Laplace
  double layer with log completion on the star contour ``contour_default``
  (problems.py:133-217).  The O(N) contour geometry is evaluated here with the
  reference's numpy expressions (so it is bit-identical); the O(N r L)
  kernel entries and the ACA run on the device.
* :func:`gaussian_hodlr` -- BASELINE cfg1 / cfg3: the regularized Gaussian
  kernel on uniform random points in the unit square / cube (xorshift64*
  stream of problems.py:26-48), cluster-ordered by an alternating-axis median
  split that follows the cluster tree's ranges.
* :func:`assemble_dense` -- entries of a dense device matrix (small n, tests,
  the SPEC examples).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .hodlr import HodlrMatrix, _torch, _workspace
from .tree import ClusterTree


def contour_default(n: int, amplitude: float = 0.3, lobes: int = 5) -> dict:
    """Star contour ``r(t) = 1 + amplitude cos(lobes t)`` sampled at ``n``
    equispaced parameters: nodes, exterior unit normals, curvature and
    trapezoidal arclength weights (problems.py:133-156, same expressions)."""
    if n < 16:
        raise ValueError("need at least 16 contour nodes")
    t = 2.0 * np.pi * np.arange(n) / n
    rad = 1.0 + amplitude * np.cos(lobes * t)
    drad = -amplitude * lobes * np.sin(lobes * t)
    ddrad = -amplitude * lobes * lobes * np.cos(lobes * t)
    ct, st = np.cos(t), np.sin(t)
    dx, dy = drad * ct - rad * st, drad * st + rad * ct
    speed = np.hypot(dx, dy)
    return {
        "t": t, "x": rad * ct, "y": rad * st, "nx": dy / speed, "ny": -dx / speed,
        "curvature": (rad * rad + 2.0 * drad * drad - rad * ddrad) / speed**3,
        "weights": speed * (2.0 * np.pi / n),
    }


def laplace_dl_geometry(n: int, amplitude: float = 0.3, lobes: int = 5, z=(0.0, 0.0)) -> np.ndarray:
    """(7, n) float64: x, y, nx, ny, weights, log completion term, diagonal
    kernel limit -- the per-node data the device oracle reads
    (problems.py:158-180: logterm = -log|x - z| / 2pi, diag = -curvature / 4pi)."""
    c = contour_default(n, amplitude, lobes)
    zz = np.asarray(z, dtype=np.float64)
    rz = np.hypot(c["x"] - zz[0], c["y"] - zz[1])
    if np.any(rz == 0.0):
        raise ValueError("completion point z must not lie on the contour")
    logterm = -np.log(rz) / (2.0 * np.pi)
    diag = -c["curvature"] / (4.0 * np.pi)
    return np.stack([c["x"], c["y"], c["nx"], c["ny"], c["weights"], logterm, diag]).astype(np.float64)


_MASK64 = (1 << 64) - 1


def xorshift_uniform(count: int, seed: int) -> np.ndarray:
    """Doubles in [0, 1) from the xorshift64* stream (problems.py:26-48: splitmix64
    seeding, top 53 bits) -- the same sequence as XorShift64Star(seed).uniform(count)."""
    z = (seed + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    x = (z ^ (z >> 31)) or 0x9E3779B97F4A7C15
    out = np.empty(count, dtype=np.float64)
    for k in range(count):
        x ^= x >> 12
        x = (x ^ (x << 25)) & _MASK64
        x ^= x >> 27
        out[k] = (((x * 0x2545F4914F6CDD1D) & _MASK64) >> 11) * 2.0**-53
    return out


def xorshift_uniform_device(count: int, seed: int, device="cuda"):
    """The same stream generated on the device (``hodlr_xorshift_uniform``)."""
    torch = _torch()
    lib = _lib.load()
    out = torch.empty(max(count, 1), dtype=torch.float64, device=device)
    st = torch.cuda.current_stream(out.device).cuda_stream
    _lib.check(lib.hodlr_xorshift_uniform(C.c_uint64(seed & ((1 << 64) - 1)), count, C.c_void_p(out.data_ptr()),
                                          C.c_void_p(st)), "hodlr_xorshift_uniform")
    return out[:count]


def kd_points(n: int, dim: int, L: int, seed: int = 0, device=None) -> np.ndarray:
    """(dim, n) uniform points in [0, 1)^dim (one xorshift64* stream, point-major),
    reordered so that every cluster-tree node of ``ClusterTree(n, L)`` is a
    spatial box: the level-l node range is sorted along axis l mod dim and
    split at ceil(len / 2) (tree.py:35-93 ranges).  ``device``: draw the stream
    there (large n) instead of the host loop."""
    if device is not None:
        pts = xorshift_uniform_device(n * dim, seed, device).cpu().numpy().reshape(n, dim)
    else:
        pts = xorshift_uniform(n * dim, seed).reshape(n, dim)
    return kd_order(pts, L)


def kd_order(pts: np.ndarray, L: int) -> np.ndarray:
    """(n, dim) points -> (dim, n) in cluster order: the level-l node range is
    sorted (stably) along axis l mod dim and split at ceil(len / 2)."""
    n, dim = pts.shape
    order = np.arange(n)
    starts = np.array([0])
    lens = np.array([n])
    for lv in range(L + 1):
        axis = lv % dim
        seg = np.repeat(np.arange(len(starts)), lens)
        key = pts[order, axis]
        order = order[np.lexsort((key, seg))]  # stable within each node
        if lv == L:
            break
        left = (lens + 1) // 2
        starts = np.stack([starts, starts + left], axis=1).ravel()
        lens = np.stack([left, lens - left], axis=1).ravel()
    return np.ascontiguousarray(pts[order].T)


def _alloc(n: int, m: int, r: int, device):
    torch = _torch()
    L = int(round(math.log2(n // m))) if n >= m else 0
    if n != m << L:
        raise ValueError(f"GPU layout needs N = m 2^L (got N={n}, m={m})")
    f64 = dict(dtype=torch.float64, device=device)
    D = torch.empty((1 << L) * m * m, **f64)
    U = torch.empty(max(n * r * L, 1), **f64)
    V = torch.empty(max(n * r * L, 1), **f64)
    return L, D, U, V


def _finish(n, m, r, L, D, U, V):
    return HodlrMatrix(ClusterTree(n, L), r, D, U[: n * r * L], V[: n * r * L])


def laplace_dl_hodlr(n: int, m: int, r: int, amplitude: float = 0.3, lobes: int = 5, z=(0.0, 0.0),
                     device="cuda", stream=None) -> HodlrMatrix:
    """The cfg2 operator (``laplace_dl_oracle(contour_default(n))``, z = 0)
    assembled on the device at uniform rank ``r`` (ACA rook, tol = 0)."""
    torch = _torch()
    lib = _lib.load()
    L, D, U, V = _alloc(n, m, r, device)
    geom = torch.from_numpy(laplace_dl_geometry(n, amplitude, lobes, z)).to(device)
    desc = _lib.Desc(n, m, r, L, 0)
    wsb = lib.hodlr_build_workspace(C.byref(desc))
    so = stream or torch.cuda.current_stream(geom.device)
    ws = _workspace(wsb, geom.device, so)
    st = so.cuda_stream
    _lib.check(lib.hodlr_build_laplace_dl(C.byref(desc), C.c_void_p(geom.data_ptr()), C.c_void_p(D.data_ptr()),
                                          C.c_void_p(U.data_ptr()), C.c_void_p(V.data_ptr()),
                                          C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(st)), "hodlr_build_laplace_dl")
    return _finish(n, m, r, L, D, U, V)


def gaussian_hodlr(n: int, m: int, r: int, dim: int = 2, h: float = 0.1, lam: float = 1.0, seed: int = 0,
                   device="cuda", stream=None, points=None) -> HodlrMatrix:
    """exp(-|p_i - p_j|^2 / h^2) + lam delta_ij on kd-ordered uniform points,
    assembled on the device at uniform rank ``r`` (ACA rook, tol = 0).
    ``points``: optional (dim, n) coordinates already in cluster order."""
    torch = _torch()
    lib = _lib.load()
    L, D, U, V = _alloc(n, m, r, device)
    P = (kd_points(n, dim, L, seed, device=device if n * dim > (1 << 16) else None) if points is None
         else np.ascontiguousarray(points, dtype=np.float64))
    if P.shape != (dim, n):
        raise ValueError(f"points must be ({dim}, {n})")
    pts = torch.from_numpy(P).to(device)
    desc = _lib.Desc(n, m, r, L, 0)
    wsb = lib.hodlr_build_workspace(C.byref(desc))
    so = stream or torch.cuda.current_stream(pts.device)
    ws = _workspace(wsb, pts.device, so)
    st = so.cuda_stream
    _lib.check(lib.hodlr_build_gaussian(C.byref(desc), C.c_void_p(pts.data_ptr()), dim, float(h), float(lam),
                                        C.c_void_p(D.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(V.data_ptr()),
                                        C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(st)), "hodlr_build_gaussian")
    return _finish(n, m, r, L, D, U, V)


def separator_grid(n: int, L: int) -> np.ndarray:
    """(2, n) unit-spaced points of an nx x ny separator plane (nx = 2^ceil(b/2),
    ny = 2^floor(b/2) for n = 2^b), in cluster (kd) order."""
    b = int(round(math.log2(n)))
    if n != 1 << b:
        raise ValueError("separator grid: n must be a power of two")
    nx, ny = 1 << ((b + 1) // 2), 1 << (b // 2)
    gx, gy = np.meshgrid(np.arange(nx, dtype=np.float64), np.arange(ny, dtype=np.float64), indexing="ij")
    return kd_order(np.stack([gx.ravel(), gy.ravel()], axis=1), L)


def schur_surrogate_hodlr(n: int, m: int, r: int, sigma: float = 0.1, device="cuda", stream=None,
                          points=None) -> HodlrMatrix:
    """BASELINE cfg4's operator: the Schur-complement surrogate of a sparse
    (3-D 7-point Laplacian) factorization on a planar separator -- the
    hypersingular DtN kernel -1 / (pi r^3) on an n-point separator grid,
    diagonal 2.8755 + sigma (``hodlr_build_schur_plane``) -- assembled on
    the device at uniform rank ``r`` (ACA rook, tol = 0)."""
    torch = _torch()
    lib = _lib.load()
    L, D, U, V = _alloc(n, m, r, device)
    P = separator_grid(n, L) if points is None else np.ascontiguousarray(points, dtype=np.float64)
    if P.shape != (2, n):
        raise ValueError(f"points must be (2, {n})")
    pts = torch.from_numpy(P).to(device)
    desc = _lib.Desc(n, m, r, L, 0)
    wsb = lib.hodlr_build_workspace(C.byref(desc))
    so = stream or torch.cuda.current_stream(pts.device)
    ws = _workspace(wsb, pts.device, so)
    _lib.check(lib.hodlr_build_schur_plane(C.byref(desc), C.c_void_p(pts.data_ptr()), float(sigma),
                                           C.c_void_p(D.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(V.data_ptr()),
                                           C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(so.cuda_stream)),
               "hodlr_build_schur_plane")
    return _finish(n, m, r, L, D, U, V)


def assemble_dense(A, m: int, r: int, device="cuda", stream=None) -> HodlrMatrix:
    """Assemble the HODLR representation of a dense (n, n) matrix (numpy or
    torch): exact leaf blocks, ACA-rook crosses of rank <= r per sibling block
    (zero-padded to r)."""
    torch = _torch()
    lib = _lib.load()
    At = torch.as_tensor(A, dtype=torch.float64)
    if At.dim() != 2 or At.shape[0] != At.shape[1]:
        raise ValueError("assemble_dense needs a square matrix")
    n = At.shape[0]
    L, D, U, V = _alloc(n, m, r, device)
    Acm = At.t().contiguous().to(device)  # column-major entries
    desc = _lib.Desc(n, m, r, L, 0)
    wsb = lib.hodlr_build_workspace(C.byref(desc))
    so = stream or torch.cuda.current_stream(Acm.device)
    ws = _workspace(wsb, Acm.device, so)
    st = so.cuda_stream
    _lib.check(lib.hodlr_build_dense(C.byref(desc), C.c_void_p(Acm.data_ptr()), n, C.c_void_p(D.data_ptr()),
                                     C.c_void_p(U.data_ptr()), C.c_void_p(V.data_ptr()), C.c_void_p(ws.data_ptr()),
                                     wsb, C.c_void_p(st)), "hodlr_build_dense")
    return _finish(n, m, r, L, D, U, V)


# ---------------------------------------------------------------------------
# SPEC-shaped entry point: assemble(entry_oracle, tree, config)
# ---------------------------------------------------------------------------


class CompressionConfig:
    """The reference's compression settings (compress.py:22-45).  The device
    builder implements the fixed-rank ACA path: ``method="aca_rook_pivot"``,
    ``tol=0`` and a ``max_rank`` (the uniform rank of the GPU layout)."""

    def __init__(self, tol: float = 0.0, max_rank: int | None = None, method: str = "aca_rook_pivot"):
        if method != "aca_rook_pivot":
            raise ValueError(f"device assembly implements method='aca_rook_pivot' (got {method!r})")
        if tol != 0.0 or max_rank is None:
            raise ValueError("device assembly is fixed-rank: tol=0 and max_rank=r (uniform-rank GPU layout)")
        if max_rank < 0:
            raise ValueError("max_rank must be >= 0")
        self.tol, self.max_rank, self.method = tol, max_rank, method


class LaplaceDoubleLayer:
    """Device entry oracle of ``laplace_dl_oracle(contour_default(n, amplitude, lobes), z)``."""

    def __init__(self, n: int, amplitude: float = 0.3, lobes: int = 5, z=(0.0, 0.0)):
        self.n, self.amplitude, self.lobes, self.z = n, amplitude, lobes, z


class GaussianPoints:
    """Device entry oracle exp(-|p_i - p_j|^2 / h^2) + lam delta_ij on (dim, n)
    points already in cluster order (see :func:`kd_points`)."""

    def __init__(self, points, h: float = 0.1, lam: float = 1.0):
        self.points = np.ascontiguousarray(points, dtype=np.float64)
        self.h, self.lam = h, lam


def assemble(entry_oracle, tree: ClusterTree, config: CompressionConfig, device="cuda") -> HodlrMatrix:
    """SPEC.md:163-171 ``assemble`` on the device.  ``entry_oracle``: a
    :class:`LaplaceDoubleLayer`, a :class:`GaussianPoints` or a dense (n, n)
    matrix; ``tree``: a uniform ``ClusterTree(n, L)`` (n = m 2^L)."""
    n, L = tree.n, tree.depth
    m = n >> L
    if m << L != n:
        raise ValueError("device assembly needs a uniform tree (n = m 2^L)")
    r = config.max_rank
    if isinstance(entry_oracle, LaplaceDoubleLayer):
        if entry_oracle.n != n:
            raise ValueError("oracle and tree sizes differ")
        return laplace_dl_hodlr(n, m, r, entry_oracle.amplitude, entry_oracle.lobes, entry_oracle.z, device=device)
    if isinstance(entry_oracle, GaussianPoints):
        P = entry_oracle.points
        return gaussian_hodlr(n, m, r, dim=P.shape[0], h=entry_oracle.h, lam=entry_oracle.lam, points=P, device=device)
    return assemble_dense(entry_oracle, m, r, device=device)

