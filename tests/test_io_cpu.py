"""CPU: the binary dump format -- header, payload order, round
trips, and the errors on malformed files (no GPU needed for the raw layer)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2208_06290_b200 import io


def test_matrix_roundtrip_and_layout(tmp_path):
    n, m, L, r = 256, 32, 3, 4
    rng = np.random.default_rng(0)
    D = rng.standard_normal((1 << L) * m * m)
    U = rng.standard_normal(n * r * L)
    V = rng.standard_normal(n * r * L)
    p = tmp_path / "a.hodlr"
    io.write_raw(p, io.KIND_MATRIX, io.FIELD_F64, n, m, [r] * L, [D, U, V])
    hdr, buf = io.read_raw(p)
    assert (hdr["n"], hdr["m"], hdr["L"], hdr["kind"], hdr["field"]) == (n, m, L, 0, 0)
    assert hdr["ranks"].tolist() == [r] * L
    for name, a in (("D", D), ("U", U), ("V", V)):
        assert buf[name].tobytes() == a.tobytes()
    # fixed order: header (40 B) + ranks (4 L) + d_big + u panels + v panels, raw little-endian
    raw = p.read_bytes()
    assert raw[:8] == b"HODLRB2\0"
    off = 40 + 4 * L
    assert raw[off : off + 8 * D.size] == D.astype("<f8").tobytes()
    assert len(raw) == off + 8 * (D.size + U.size + V.size)


def test_factorization_layout_fp32(tmp_path):
    n, m, L, r = 128, 16, 3, 2
    nl, nk = 8, 7
    bufs = [np.zeros(nl * m * m, np.float32), np.ones(n * r * L, np.float32), np.ones(n * r * L, np.float32),
            np.arange(nl * m, dtype=np.int32), np.arange(nl * m, dtype=np.int32), np.zeros(nk * 2 * r, np.int32),
            np.zeros(nk * 2 * r, np.int32), np.ones(nk * 4 * r * r, np.float32)]
    p = tmp_path / "f.hodlr"
    io.write_raw(p, io.KIND_FACTORIZATION, io.FIELD_F32, n, m, [r] * L, bufs)
    hdr, buf = io.read_raw(p)
    assert [k for k, _, _ in io.payload_layout(hdr)] == ["D", "U", "V", "dswaps", "dperm", "kswaps", "kperm", "K"]
    assert buf["dperm"].tolist() == list(range(nl * m)) and buf["K"].dtype == np.dtype("<f4")


def test_malformed_files_raise(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"NOTHODLR" + b"\0" * 40)
    with pytest.raises(ValueError, match="not a HODLR dump"):
        io.read_header(p)
    n, m, L, r = 64, 16, 2, 2
    q = tmp_path / "trunc"
    io.write_raw(q, io.KIND_MATRIX, io.FIELD_F64, n, m, [r] * L, [np.zeros(4 * m * m), np.zeros(n * r * L),
                                                                  np.zeros(n * r * L)])
    q.write_bytes(q.read_bytes()[:-8])
    with pytest.raises(ValueError, match="truncated payload at V"):
        io.read_raw(q)
    with pytest.raises(ValueError, match="is not m 2"):
        io.write_raw(q, io.KIND_MATRIX, io.FIELD_F64, 100, m, [r] * L, [])
