"""Batched dense kernels over block descriptors -- the reference's kernel layer
(``pkg/src/hodlr/backend.py``) with an sm_100a executor slotted in.

Same public names, argument meaning, flop counts and error messages as the
reference (backend.py:32-610), so callers and the reference's own tests read
the same.  Differences, all by design:

* Buffers may be flat torch CUDA tensors (device-resident, the fast path) or
  flat numpy arrays (copied to the device, computed, copied back -- the
  end-to-end path).  Every computation runs in the native library; there is
  no CPU fallback.
* ``executor`` is accepted for signature parity and ignored: parallelism is
  the GPU grid.  ``parse_executor`` keeps the reference's config grammar.
* GEMM values agree with numpy/OpenBLAS to rounding (different summation
  order); LU factors and pivots are bit-identical (see lu.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class SingularBlockError(RuntimeError):
    """A block in a batch is singular to working precision (backend.py:32-40)."""

    def __init__(self, indices, context: str = ""):
        self.indices = list(indices)
        msg = f"singular block(s) at batch index {self.indices}"
        if context:
            msg += f" ({context})"
        super().__init__(msg)


# ---------------------------------------------------------------------------
# descriptors
# ---------------------------------------------------------------------------


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _size(buf) -> int:
    return buf.numel() if _is_torch(buf) else buf.size


def _ndim(buf) -> int:
    return buf.dim() if _is_torch(buf) else buf.ndim


@dataclass(frozen=True)
class BlockRef:
    """Block (i, j) at ``buf[offset + i + j*ld]`` of a flat buffer (backend.py:48-89)."""

    buf: object
    offset: int
    rows: int
    cols: int
    ld: int

    def __post_init__(self):
        if _ndim(self.buf) != 1:
            raise ValueError("BlockRef buffer must be a flat 1-d array")
        if self.rows < 0 or self.cols < 0:
            raise ValueError("negative block shape")
        if self.rows > 0 and self.cols > 0:
            end = self.offset + (self.cols - 1) * self.ld + self.rows
            if self.offset < 0 or end > _size(self.buf):
                raise ValueError(
                    f"block [{self.rows}x{self.cols}, ld={self.ld}] at offset "
                    f"{self.offset} exceeds buffer of size {_size(self.buf)}"
                )

    def view(self):
        """Writable 2-d strided view (numpy or torch) of the block."""
        if _is_torch(self.buf):
            return self.buf.as_strided((self.rows, self.cols), (1, self.ld), self.offset)
        it = self.buf.itemsize
        return np.lib.stride_tricks.as_strided(
            self.buf[self.offset :], shape=(self.rows, self.cols), strides=(it, self.ld * it)
        )

    def footprint(self) -> tuple[int, int]:
        if self.rows == 0 or self.cols == 0:
            return (self.offset, self.offset)
        return (self.offset, self.offset + (self.cols - 1) * self.ld + self.rows)


def blocks_overlap(a: BlockRef, b: BlockRef) -> bool:
    """Exact for equal ld (sub-blocks of one panel), footprint-conservative otherwise."""
    if a.buf is not b.buf or 0 in (a.rows, a.cols, b.rows, b.cols):
        return False
    (a0, a1), (b0, b1) = a.footprint(), b.footprint()
    if a1 <= b0 or b1 <= a0:
        return False
    if a.ld == b.ld and a.ld >= max(a.rows, b.rows):
        ra, ca = divmod(a.offset, a.ld)[::-1]
        rb, cb = divmod(b.offset, b.ld)[::-1]
        return not (ra + a.rows <= rb or rb + b.rows <= ra or ca + a.cols <= cb or cb + b.cols <= ca)
    return True


def _uniform_step(refs):
    """(offset0, step) when refs share buf/shape/ld with constant offset stride."""
    r0 = refs[0]
    if any(r.buf is not r0.buf or (r.rows, r.cols, r.ld) != (r0.rows, r0.cols, r0.ld) for r in refs):
        return None
    if len(refs) == 1:
        return r0.offset, 0
    step = refs[1].offset - r0.offset
    if any(refs[i + 1].offset - refs[i].offset != step for i in range(len(refs) - 1)):
        return None
    return r0.offset, step


def _paired_step(refs):
    """(offset0, hi, lo) for offsets (b//2)*hi + (b%2)*lo (paired-child layouts)."""
    if len(refs) < 2 or len(refs) % 2:
        return None
    r0 = refs[0]
    if any(r.buf is not r0.buf or (r.rows, r.cols, r.ld) != (r0.rows, r0.cols, r0.ld) for r in refs):
        return None
    lo = refs[1].offset - r0.offset
    hi = refs[2].offset - r0.offset if len(refs) > 2 else 0
    for i, r in enumerate(refs):
        if r.offset != r0.offset + (i // 2) * hi + (i % 2) * lo:
            return None
    return r0.offset, hi, lo


def as_stack(refs):
    """Zero-copy (B, rows, cols) view over uniform constant-stride blocks, else None."""
    u = _uniform_step(refs)
    if u is None:
        return None
    off, step = u
    r0 = refs[0]
    if _is_torch(r0.buf):
        return r0.buf.as_strided((len(refs), r0.rows, r0.cols), (step, 1, r0.ld), off)
    it = r0.buf.itemsize
    return np.lib.stride_tricks.as_strided(
        r0.buf[off:], shape=(len(refs), r0.rows, r0.cols), strides=(step * it, it, r0.ld * it)
    )


@dataclass
class BlockBatch:
    """Per-item operand tuples plus the uniform-stride test (backend.py:147-167)."""

    items: list

    def uniform(self):
        if not self.items:
            return None
        stacks = []
        for pos in range(len(self.items[0])):
            s = as_stack([it[pos] for it in self.items])
            if s is None:
                return None
            stacks.append(s)
        return tuple(stacks)


# ---------------------------------------------------------------------------
# executors (config compatibility only: the GPU grid is the parallelism)
# ---------------------------------------------------------------------------


class SerialExecutor:
    threads = 1

    def run(self, nitems, body):
        if nitems > 0:
            body(0, nitems)

    def __repr__(self):
        return "serial"


class ThreadedExecutor(SerialExecutor):
    def __init__(self, threads: int):
        if threads < 1:
            raise ValueError("thread count must be >= 1")
        self.threads = threads

    def __repr__(self):
        return f"threads({self.threads})"


SERIAL = SerialExecutor()


def parse_executor(spec: str):
    """``serial`` or ``threads:<k>`` (backend.py:224-232); both run on the GPU here."""
    spec = spec.strip()
    if spec == "serial":
        return SERIAL
    if spec.startswith("threads"):
        _, _, arg = spec.partition(":")
        return ThreadedExecutor(int(arg) if arg else 2)
    raise ValueError(f"unknown executor {spec!r} (expected serial or threads:<k>)")


# ---------------------------------------------------------------------------
# flop conventions (backend.py:240-251)
# ---------------------------------------------------------------------------


def gemm_flops(m: int, k: int, n: int) -> int:
    return 2 * m * k * n


def lu_factor_flops(s: int) -> int:
    return s * (s - 1) // 2 + s * (s - 1) * (2 * s - 1) // 3


def lu_solve_flops(s: int, ncols: int) -> int:
    return 2 * s * s * ncols


# ---------------------------------------------------------------------------
# device staging of buffers
# ---------------------------------------------------------------------------


class _Staging:
    """Maps every distinct buffer to a CUDA tensor; copies numpy outputs back."""

    def __init__(self):
        self.torch = _lib.require_cuda()
        self.dev = {}
        self.host = {}

    def get(self, buf):
        key = id(buf)
        if key not in self.dev:
            torch = self.torch
            if _is_torch(buf):
                if not buf.is_cuda:
                    t = buf.to("cuda")
                    self.host[key] = (buf, t)
                else:
                    t = buf
            else:
                if buf.dtype not in (np.float64, np.float32):
                    raise TypeError(f"unsupported dtype {buf.dtype} (fp64/fp32 only on the B200 path)")
                t = torch.from_numpy(np.ascontiguousarray(buf)).to("cuda")
                self.host[key] = (buf, t)
            if t.dtype not in (torch.float64, torch.float32):
                raise TypeError(f"unsupported dtype {t.dtype} (fp64/fp32 only on the B200 path)")
            self.dev[key] = t
        return self.dev[key]

    def ptr(self, buf, offset):
        t = self.get(buf)
        return C.c_void_p(t.data_ptr() + offset * t.element_size())

    def writeback(self, bufs):
        for b in bufs:
            pair = self.host.get(id(b))
            if pair is None:
                continue
            host, t = pair
            if _is_torch(host):
                host.copy_(t)
            else:
                host[...] = t.cpu().numpy()

    @property
    def stream(self):
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)


def _dtype_of(t):
    import torch

    return _lib.F64 if t.dtype == torch.float64 else _lib.F32


# ---------------------------------------------------------------------------
# batched GEMM (backend.py:306-411)
# ---------------------------------------------------------------------------


def _check_gemm_batch(items, conj_a):
    for idx, (a, b, c) in enumerate(items):
        am, ak = (a.cols, a.rows) if conj_a else (a.rows, a.cols)
        if ak != b.rows or c.rows != am or c.cols != b.cols:
            raise ValueError(
                f"gemm shape mismatch at batch index {idx}: "
                f"op(a)=({am}x{ak}), b=({b.rows}x{b.cols}), c=({c.rows}x{c.cols})"
            )
    outs = sorted(enumerate(items), key=lambda t: t[1][2].offset)
    for (i, x), (j, y) in zip(outs, outs[1:]):
        if blocks_overlap(x[2], y[2]):
            raise ValueError(f"gemm output blocks overlap at batch indices {i} and {j}")


_SPLIT_WS_BYTES = 64 << 20


def _gemm_dispatch(items, alpha, beta, conj_a):
    lib = _lib.load()
    stg = _Staging()
    torch = stg.torch
    a0, b0, c0 = items[0]
    # inputs aliasing an output buffer are snapshotted (numpy matmul semantics)
    cbufs = {id(c.buf) for _, _, c in items}
    snap = {}
    for pos in (0, 1):
        for it in items:
            buf = it[pos].buf
            if id(buf) in cbufs and id(buf) not in snap:
                snap[id(buf)] = stg.get(buf).clone()
    dt = _dtype_of(stg.get(c0.buf))
    ws = torch.empty(_SPLIT_WS_BYTES, dtype=torch.uint8, device="cuda")

    def ptr(ref):
        t = snap.get(id(ref.buf))
        if t is None:
            return stg.ptr(ref.buf, ref.offset)
        return C.c_void_p(t.data_ptr() + ref.offset * t.element_size())

    def call(ia, ib, ic, M, N, K, sa, sb, sc, batch, bdiv):
        st = lib.hodlr_gemm_batched(
            dt, int(conj_a), M, N, K, float(alpha), ptr(ia), ia.ld, sa[0], sa[1], ptr(ib), ib.ld, sb[0], sb[1],
            float(beta), ptr(ic), ic.ld, sc[0], sc[1], batch, bdiv, C.c_void_p(ws.data_ptr()), _SPLIT_WS_BYTES,
            stg.stream,
        )
        _lib.check(st, "hodlr_gemm_batched")

    M, N, K = c0.rows, c0.cols, b0.rows
    cols = [[it[p] for it in items] for p in range(3)]
    uni = [_uniform_step(x) for x in cols]
    if all(u is not None for u in uni):
        call(a0, b0, c0, M, N, K, (uni[0][1], 0), (uni[1][1], 0), (uni[2][1], 0), len(items), 1)
    else:
        pair = [_paired_step(x) for x in cols]
        if all(p is not None for p in pair):
            call(a0, b0, c0, M, N, K, pair[0][1:], pair[1][1:], pair[2][1:], len(items), 2)
        else:
            for a, b, c in items:
                call(a, b, c, c.rows, c.cols, b.rows, (0, 0), (0, 0), (0, 0), 1, 1)
    stg.writeback({id(c.buf): c.buf for _, _, c in items}.values())


def batched_gemm(batch, alpha=1.0, beta=0.0, transpose_a: str = "none", executor=SERIAL, scratch=None) -> int:
    """``c <- alpha op(a) b + beta c`` over every (a, b, c) item; returns flops."""
    if transpose_a not in ("none", "conj_transpose"):
        raise ValueError(f"unsupported transpose_a {transpose_a!r}")
    conj_a = transpose_a == "conj_transpose"
    if isinstance(batch, list):
        batch = BlockBatch(batch)
    if not batch.items:
        return 0
    _check_gemm_batch(batch.items, conj_a)
    flops = sum(gemm_flops(c.rows, b.rows, b.cols) for (_, b, c) in batch.items)
    _gemm_dispatch(batch.items, alpha, beta, conj_a)
    return flops


def grouped_gemm_large(items: list, alpha=1.0, beta=0.0, transpose_a: str = "none", inner_threads: int = 0) -> int:
    """Few large items (top tree levels); same contract as :func:`batched_gemm`.

    On the GPU each item is one launch whose long reductions are split over a
    fixed-order split-K tree, so results do not depend on ``inner_threads``.
    """
    if transpose_a not in ("none", "conj_transpose"):
        raise ValueError(f"unsupported transpose_a {transpose_a!r}")
    conj_a = transpose_a == "conj_transpose"
    if not items:
        return 0
    _check_gemm_batch(items, conj_a)
    flops = sum(gemm_flops(c.rows, b.rows, b.cols) for (_, b, c) in items)
    for it in items:
        _gemm_dispatch([it], alpha, beta, conj_a)
    return flops


def gemm_stacks(a, b, c, alpha=1.0, beta=0.0, transpose_a="none", scratch=None) -> int:
    """Stacked (broadcastable) operands with trailing (rows, cols) axes (backend.py:266-279)."""
    if transpose_a not in ("none", "conj_transpose"):
        raise ValueError(f"unsupported transpose_a {transpose_a!r}")
    torch = _lib.require_cuda()
    is_np = isinstance(c, np.ndarray)
    ta = torch.as_tensor(a)
    tb = torch.as_tensor(b)
    tc = torch.as_tensor(c)
    conj = transpose_a == "conj_transpose"
    opa_shape = ta.shape[:-2] + ((ta.shape[-1], ta.shape[-2]) if conj else tuple(ta.shape[-2:]))
    bshape = torch.broadcast_shapes(opa_shape[:-2], tb.shape[:-2], tc.shape[:-2])
    A = ta.expand(bshape + ta.shape[-2:]).reshape(-1, *ta.shape[-2:])
    B = tb.expand(bshape + tb.shape[-2:]).reshape(-1, *tb.shape[-2:])
    Cm = tc.expand(bshape + tc.shape[-2:]).reshape(-1, *tc.shape[-2:])
    nb = A.shape[0]
    # column-major flat device copies
    fa = A.transpose(-1, -2).contiguous().reshape(-1).cuda()
    fb = B.transpose(-1, -2).contiguous().reshape(-1).cuda()
    fc = Cm.transpose(-1, -2).contiguous().reshape(-1).cuda()
    ar, ac = A.shape[-2:]
    br, bc = B.shape[-2:]
    cr, cc = Cm.shape[-2:]
    items = [
        (BlockRef(fa, i * ar * ac, ar, ac, ar), BlockRef(fb, i * br * bc, br, bc, br), BlockRef(fc, i * cr * cc, cr, cc, cr))
        for i in range(nb)
    ]
    batched_gemm(items, alpha, beta, transpose_a)
    res = fc.view(nb, cc, cr).transpose(-1, -2).reshape(tc.shape).to(tc.device)
    if is_np:
        c[...] = res.cpu().numpy()
    else:
        c.copy_(res)
    nitems = int(np.prod(tc.shape[:-2], dtype=np.int64)) if tc.dim() > 2 else 1
    return nitems * gemm_flops(tc.shape[-2], tb.shape[-2], tc.shape[-1])


# ---------------------------------------------------------------------------
# batched LU (backend.py:419-610)
# ---------------------------------------------------------------------------


@dataclass
class LuPivots:
    """swaps (LAPACK-style), perm (P A = A[perm]), singular indices (backend.py:419-441)."""

    swaps: np.ndarray
    perm: np.ndarray
    singular: list = field(default_factory=list)

    @property
    def size(self) -> int:
        return self.swaps.shape[1]

    def sign(self) -> np.ndarray:
        k = np.arange(self.size)
        nswap = (self.swaps != k).sum(axis=1)
        return np.where(nswap % 2 == 0, 1.0, -1.0)


def _lu_refs(batch):
    if isinstance(batch, BlockBatch):
        return [it[0] if isinstance(it, tuple) else it for it in batch.items]
    return list(batch)


def batched_lu_factor_inplace(batch, executor=SERIAL):
    """Factor every square block in place; returns (LuPivots, flops).

    Singular blocks are flagged in the pivots, not raised (backend.py:481-529).
    """
    refs = _lu_refs(batch)
    if not refs:
        return LuPivots(np.zeros((0, 0), np.int64), np.zeros((0, 0), np.int64)), 0
    for idx, r in enumerate(refs):
        if r.rows != r.cols:
            raise ValueError(f"LU block at batch index {idx} is not square")
    s = refs[0].rows
    if any(r.rows != s for r in refs):
        raise ValueError("LU batch blocks must share one size")
    flops = lu_factor_flops(s) * len(refs)
    nb = len(refs)
    if s == 0:
        z = np.zeros((nb, 0), np.int64)
        return LuPivots(z, z.copy()), flops
    lib = _lib.load()
    stg = _Staging()
    torch = stg.torch
    i32 = dict(dtype=torch.int32, device="cuda")
    sw, pm, info = torch.empty(nb * s, **i32), torch.empty(nb * s, **i32), torch.zeros(nb, **i32)
    dt = _dtype_of(stg.get(refs[0].buf))
    u = _uniform_step(refs)
    groups = [(refs[0], u[1], nb, 0)] if u is not None else [(r, 0, 1, i) for i, r in enumerate(refs)]
    for ref, step, cnt, first in groups:
        st = lib.hodlr_getrf_batched(
            dt, s, cnt, stg.ptr(ref.buf, ref.offset), ref.ld, step,
            C.c_void_p(sw.data_ptr() + first * s * 4), C.c_void_p(pm.data_ptr() + first * s * 4),
            C.c_void_p(info.data_ptr() + first * 4), None, 0, 0, stg.stream,
        )
        _lib.check(st, "hodlr_getrf_batched")
    stg.writeback({id(r.buf): r.buf for r in refs}.values())
    swaps = sw.view(nb, s).cpu().numpy().astype(np.int64)
    perm = pm.view(nb, s).cpu().numpy().astype(np.int64)
    bad = [int(i) for i in np.flatnonzero(info.cpu().numpy())]
    return LuPivots(swaps, perm, bad), flops


def batched_lu_solve_inplace(lu_refs: list, pivots: LuPivots, rhs_refs: list, executor=SERIAL) -> int:
    """Overwrite each rhs block with its LU solution; returns flops (backend.py:570-610)."""
    if pivots.singular:
        raise SingularBlockError(pivots.singular, "refusing to solve")
    if not lu_refs:
        return 0
    if len(lu_refs) != len(rhs_refs):
        raise ValueError("LU and rhs batches differ in length")
    s = pivots.size
    for idx, (lr, rr) in enumerate(zip(lu_refs, rhs_refs)):
        if lr.rows != s or lr.cols != s or rr.rows != s:
            raise ValueError(f"solve shape mismatch at batch index {idx}")
    flops = sum(lu_solve_flops(s, r.cols) for r in rhs_refs)
    if s == 0:
        return flops
    lib = _lib.load()
    stg = _Staging()
    torch = stg.torch
    perm = torch.as_tensor(np.ascontiguousarray(pivots.perm, dtype=np.int32)).reshape(-1).cuda()
    dt = _dtype_of(stg.get(rhs_refs[0].buf))
    ul, ur = _uniform_step(lu_refs), _uniform_step(rhs_refs)
    if ul is not None and ur is not None:
        groups = [(lu_refs[0], ul[1], rhs_refs[0], ur[1], len(lu_refs), 0)]
    else:
        groups = [(lr, 0, rr, 0, 1, i) for i, (lr, rr) in enumerate(zip(lu_refs, rhs_refs))]
    for lr, ls, rr, rs, cnt, first in groups:
        if rr.cols == 0:
            continue
        st = lib.hodlr_getrs_batched(
            dt, s, rr.cols, cnt, stg.ptr(lr.buf, lr.offset), lr.ld, ls,
            C.c_void_p(perm.data_ptr() + first * s * 4), stg.ptr(rr.buf, rr.offset), rr.ld, rs, stg.stream,
        )
        _lib.check(st, "hodlr_getrs_batched")
    stg.writeback({id(r.buf): r.buf for r in rhs_refs}.values())
    return flops


def lu_solve_stacks(lu, perm, rhs) -> int:
    """Stacked LU solve: lu (B,s,s), perm (B,s), rhs (..., B, s, c) in place (backend.py:532-543)."""
    torch = _lib.require_cuda()
    is_np = isinstance(rhs, np.ndarray)
    tl = torch.as_tensor(lu)
    tr = torch.as_tensor(rhs)
    B, s = tl.shape[0], tl.shape[-1]
    ncol = tr.shape[-1]
    lead = tr.shape[:-3]
    flat_lu = tl.transpose(-1, -2).contiguous().reshape(-1).cuda()
    perm32 = np.ascontiguousarray(np.asarray(perm), dtype=np.int32)
    pv = LuPivots(perm32.astype(np.int64), perm32.astype(np.int64))
    R = tr.reshape((-1,) + tuple(tr.shape[-3:]))
    out = []
    for j in range(R.shape[0]):
        fr = R[j].transpose(-1, -2).contiguous().reshape(-1).cuda()
        lrefs = [BlockRef(flat_lu, i * s * s, s, s, s) for i in range(B)]
        rrefs = [BlockRef(fr, i * s * ncol, s, ncol, s) for i in range(B)]
        _solve_with_perm(lrefs, perm32, rrefs)
        out.append(fr.view(B, ncol, s).transpose(-1, -2))
    res = torch.stack(out).reshape(tr.shape).to(tr.device)
    if is_np:
        rhs[...] = res.cpu().numpy()
    else:
        rhs.copy_(res)
    nblockcols = int(np.prod(tr.shape[:-2], dtype=np.int64)) * ncol
    del lead, pv
    return lu_solve_flops(s, nblockcols)


def _solve_with_perm(lu_refs, perm32, rhs_refs):
    lib = _lib.load()
    stg = _Staging()
    torch = stg.torch
    s = lu_refs[0].rows
    perm = torch.as_tensor(perm32).reshape(-1).cuda()
    dt = _dtype_of(stg.get(rhs_refs[0].buf))
    st = lib.hodlr_getrs_batched(
        dt, s, rhs_refs[0].cols, len(lu_refs), stg.ptr(lu_refs[0].buf, 0), s, s * s, C.c_void_p(perm.data_ptr()),
        stg.ptr(rhs_refs[0].buf, 0), s, s * rhs_refs[0].cols, stg.stream,
    )
    _lib.check(st, "hodlr_getrs_batched")
