"""Binary dump / load of a HODLR matrix or factorization ("Binary
dump/load of the representation: header (n, L, field tag, per-level rank
arrays), then raw little-endian column-major buffers in fixed order (d_big,
u_panels 1..L, v_panels 1..L)").  Factor once, solve many: a dumped
factorization reloads straight into HBM and solves without refactoring.

Layout (little-endian throughout)::

    offset  size        field
    0       8           magic  b"HODLRB2\\0"
    8       4  u32      version (1)
    12      4  u32      kind: 0 = matrix, 1 = factorization
    16      4  u32      field: 0 = real64, 1 = real32
    20      4  u32      L (tree depth)
    24      8  u64      n
    32      4  u32      m (leaf size, n = m 2^L)
    36      4  u32      reserved (0)
    40      4 L i32     ranks[1..L] (basis columns of level l)
    ...     payload, each buffer raw and contiguous, in this order:

    matrix:         d_big (2^L m^2)       leaf a at a m^2, column-major m x m
                    u_panels 1..L         level l: n x ranks[l], column-major
                    v_panels 1..L
    factorization:  the matrix part with d_big -> its LU and u_panels -> Y,
                    then dswaps, dperm (i32 2^L m), kswaps, kperm
                    (i32 (2^L - 1) 2r), K LU ((2^L - 1) (2r)^2, level l at
                    (2^l - 1)(2r)^2), Dinv / Kinv solve aids
                    (hodlr_inv_elems per block; fp64 only)

Ranks are per level (uniform matrices repeat r; ragged nodes are zero-padded
to their level's rank); with per-level ranks the K blocks of parent
level l are 2 ranks[l] square, stored level after level.  Scalars are written
as stored (no conversion).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

MAGIC = b"HODLRB2\0"
VERSION = 1
KIND_MATRIX, KIND_FACTORIZATION = 0, 1
FIELD_F64, FIELD_F32 = 0, 1
_HDR = struct.Struct("<8sIIIIQII")


def _field_dtype(field: int):
    if field == FIELD_F64:
        return np.dtype("<f8")
    if field == FIELD_F32:
        return np.dtype("<f4")
    raise ValueError(f"unknown field tag {field}")


def write_raw(path, kind: int, field: int, n: int, m: int, ranks, buffers) -> None:
    """Header + the buffers (numpy arrays, written in order as little-endian)."""
    L = len(ranks)
    if n != m << L:
        raise ValueError(f"n = {n} is not m 2^L = {m} * 2^{L}")
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(MAGIC, VERSION, kind, field, L, n, m, 0))
        fh.write(np.asarray(ranks, dtype="<i4").tobytes())
        for b in buffers:
            a = np.ascontiguousarray(b)
            a = a.astype(a.dtype.newbyteorder("<"), copy=False)
            fh.write(a.tobytes())


def read_header(path) -> dict:
    with open(path, "rb") as fh:
        raw = fh.read(_HDR.size)
        if len(raw) != _HDR.size:
            raise ValueError(f"{path}: truncated header")
        magic, ver, kind, field, L, n, m, _ = _HDR.unpack(raw)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a HODLR dump (magic {magic!r})")
        if ver != VERSION:
            raise ValueError(f"{path}: unsupported version {ver}")
        ranks = np.frombuffer(fh.read(4 * L), dtype="<i4").astype(np.int64)
        if len(ranks) != L:
            raise ValueError(f"{path}: truncated rank array")
    if n != m << L:
        raise ValueError(f"{path}: inconsistent header (n={n}, m={m}, L={L})")
    return {"kind": kind, "field": field, "L": L, "n": n, "m": m, "ranks": ranks,
            "offset": _HDR.size + 4 * L}


def payload_layout(hdr: dict, inv_elems=None):
    """[(name, dtype, count)] of the payload for this header."""
    n, m, L = hdr["n"], hdr["m"], hdr["L"]
    ranks = [int(x) for x in hdr["ranks"]]
    dt = _field_dtype(hdr["field"])
    i4 = np.dtype("<i4")
    nl, nk = 1 << L, (1 << L) - 1
    lay = [("D", dt, nl * m * m), ("U", dt, n * sum(ranks)), ("V", dt, n * sum(ranks))]
    if hdr["kind"] == KIND_FACTORIZATION:
        # per parent level lv the K blocks are 2 ranks[lv] square (uniform: 2r)
        kps = sum((1 << lv) * 2 * ranks[lv] for lv in range(L))
        ksz = sum((1 << lv) * (2 * ranks[lv]) ** 2 for lv in range(L))
        lay += [("dswaps", i4, nl * m), ("dperm", i4, nl * m), ("kswaps", i4, max(kps, 1)),
                ("kperm", i4, max(kps, 1)), ("K", dt, ksz)]
        if hdr["field"] == FIELD_F64:
            ie = inv_elems or (lambda s: 8 * s if s in (32, 64, 128) else (s * s if s == 16 else 0))
            kis = sum(max((1 << lv) * ie(2 * ranks[lv]), 1) for lv in range(L)) if L else 1
            lay += [("Dinv", dt, max(nl * ie(m), 1)), ("Kinv", dt, max(kis, 1))]
    return lay


def read_raw(path, inv_elems=None) -> tuple[dict, dict]:
    """(header, {name: numpy array}) with every payload buffer."""
    hdr = read_header(path)
    out = {}
    with open(path, "rb") as fh:
        fh.seek(hdr["offset"])
        for name, dt, count in payload_layout(hdr, inv_elems):
            a = np.fromfile(fh, dtype=dt, count=count)
            if a.size != count:
                raise ValueError(f"{path}: truncated payload at {name}")
            out[name] = a
        if fh.read(1):
            raise ValueError(f"{path}: trailing bytes after the payload")
    return hdr, out


# ---------------------------------------------------------------------------
# HodlrMatrix / HodlrFactorization (device objects)
# ---------------------------------------------------------------------------


def dump(obj, path) -> None:
    """Write a HodlrMatrix or HodlrFactorization (device or host tensors)."""
    from .hodlr import HodlrFactorization, HodlrMatrix

    def host(t):
        return t.detach().cpu().numpy()

    field = FIELD_F64 if str(obj.D.dtype).endswith("float64") else FIELD_F32
    L, n, m = obj.L, obj.n, obj.m
    ranks = list(obj.level_ranks)
    if isinstance(obj, HodlrMatrix):
        write_raw(path, KIND_MATRIX, field, n, m, ranks, [host(obj.D), host(obj.U), host(obj.V)])
        return
    if not isinstance(obj, HodlrFactorization):
        raise TypeError(f"cannot dump {type(obj).__name__}")
    if obj.variant != "pivoted_standard":
        raise ValueError(f"unsupported variant {obj.variant!r}")
    bufs = [host(obj.D), host(obj.Y), host(obj.V), host(obj.dswaps), host(obj.dperm), host(obj.kswaps),
            host(obj.kperm), host(obj.K)]
    if field == FIELD_F64:
        bufs += [host(obj.Dinv), host(obj.Kinv)]
    write_raw(path, KIND_FACTORIZATION, field, n, m, ranks, bufs)


def load(path, device="cuda"):
    """Read a dump back into HBM: a HodlrMatrix or a HodlrFactorization (which
    solves directly -- its singular flags are clear: only clean
    factorizations are dumped)."""
    from . import _lib
    from .hodlr import HodlrFactorization, HodlrMatrix, flop_report
    from .tree import ClusterTree

    torch = _lib.require_cuda()
    lib = _lib.load()
    hdr, buf = read_raw(path, inv_elems=lambda s: int(lib.hodlr_inv_elems(s)))
    n, m, L = hdr["n"], hdr["m"], hdr["L"]
    ranks = [int(x) for x in hdr["ranks"]]
    r = max(ranks, default=0)
    per_level = tuple(ranks) if len(set(ranks)) > 1 else None
    dev = torch.device(device)
    t = {k: torch.from_numpy(v.copy()).to(dev) for k, v in buf.items()}
    tree = ClusterTree(n, L)
    if hdr["kind"] == KIND_MATRIX:
        return HodlrMatrix(tree, r, t["D"], t["U"], t["V"], per_level)
    nl, nk = 1 << L, (1 << L) - 1
    i32 = dict(dtype=torch.int32, device=dev)
    dt = t["D"].dtype
    return HodlrFactorization(
        tree=tree, rank=r, D=t["D"], Dinv=t.get("Dinv", torch.empty(1, dtype=dt, device=dev)), Y=t["U"], V=t["V"],
        K=t["K"], Kinv=t.get("Kinv", torch.empty(1, dtype=dt, device=dev)), dswaps=t["dswaps"], dperm=t["dperm"],
        dinfo=torch.zeros(nl, **i32), kswaps=t["kswaps"], kperm=t["kperm"], kinfo=torch.zeros(max(nk, 1), **i32),
        flops=flop_report(n, m, r, ranks=per_level), ranks=per_level,
    )


def storage_bytes(path) -> int:
    return Path(path).stat().st_size


__all__ = ["dump", "load", "read_header", "read_raw", "write_raw", "payload_layout", "MAGIC"]
