"""Time hodlr_matvec at the cfg2 shape (N = 2^20, m = 64, r = 32, fp64) and cfg4 (fp32, r = 8).

Algorithmic bytes = es (m N + 2 r N L) + es N nrhs (x, read twice) + es N nrhs (y).
Prints one JSON line per (config, nrhs)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2208_06290_b200 as hb  # noqa: E402


def run(n, m, r, dtype, nrhs, reps=20):
    L = (n // m).bit_length() - 1
    g = torch.Generator(device="cuda").manual_seed(0)
    D = torch.randn((1 << L) * m * m, dtype=dtype, device="cuda", generator=g)
    U = torch.randn(n * r * L, dtype=dtype, device="cuda", generator=g)
    V = torch.randn(n * r * L, dtype=dtype, device="cuda", generator=g)
    h = hb.HodlrMatrix.from_buffers(n, m, r, D, U, V)
    x = torch.randn(n, nrhs, dtype=dtype, device="cuda", generator=g) if nrhs > 1 else torch.randn(
        n, dtype=dtype, device="cuda", generator=g)
    for _ in range(3):
        h.matvec(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.matvec(x)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    es = D.element_size()
    byts = es * (m * n + 2 * r * n * L) + 3 * es * n * nrhs
    ms = ts[len(ts) // 2]
    print(json.dumps({"n": n, "m": m, "r": r, "dtype": str(dtype).split(".")[-1], "nrhs": nrhs,
                      "ms_med": round(ms, 4), "ms_min": round(ts[0], 4), "GB": round(byts / 1e9, 3),
                      "GB_per_s": round(byts / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    for nrhs in (1, 4, 16):
        run(1 << 20, 64, 32, torch.float64, nrhs)
    run(1 << 21, 64, 8, torch.float32, 1)
