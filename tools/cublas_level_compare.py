"""The library baseline for one fused level step: the same update + next-level
[W|T] as two cuBLAS strided-batched DGEMMs (torch.baddbmm / bmm on the slab
views), vs level_update4_kernel (the level phase of one factorization, per level).
Shapes: cfg2 (N = 2^20, r = 32), level l: children of n_c = N / 2^(l+1) rows."""
import sys
sys.path.insert(0, ".")
import torch

N, r = 1 << 20, 32
dev = "cuda"
Y = torch.randn(N * r * 14, dtype=torch.float64, device=dev)
V = torch.randn(N * r * 14, dtype=torch.float64, device=dev)


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


tot_ms, tot_fl = 0.0, 0
for lv in range(13, 0, -1):
    nc = N >> (lv + 1)
    nch = N // nc
    wc = r * lv
    # C = Y[:, 0:wc] (N x wc, ld N), A1 = Y[:, lv r:(lv+1) r], Vp = V[:, (lv-1) r: lv r]
    C = Y[: wc * N].view(wc, N).t()
    A1 = Y[lv * r * N : (lv + 1) * r * N].view(r, N).t()
    Vp = V[(lv - 1) * r * N : lv * r * N].view(r, N).t()
    Cb = C.as_strided((nch, nc, wc), (nc, 1, N))
    Ab = A1.as_strided((nch, nc, r), (nc, 1, N))
    Vb = Vp.as_strided((nch, nc, r), (nc, 1, N))
    W = torch.randn(nch, r, wc, dtype=torch.float64, device=dev)
    TW = torch.empty(nch, r, wc, dtype=torch.float64, device=dev)

    def step():
        torch.baddbmm(Cb, Ab, W, beta=1.0, alpha=-1.0, out=Cb)   # C_c -= Y_c W'_c
        torch.bmm(Vb.transpose(1, 2), Cb, out=TW)                 # [W|T]_c = V_c^T C_c

    ms = ev_time(step)
    fl = 4 * r * r * N * lv
    tot_ms += ms
    tot_fl += fl
    print(f"level {lv:2d}: cuBLAS 2x strided-batched {ms:.3f} ms = {fl / ms / 1e9:.1f} TF/s", flush=True)
print(f"all levels: {tot_ms:.2f} ms for {tot_fl / 1e9:.1f} GFLOP = {tot_fl / tot_ms / 1e9:.1f} TF/s "
      f"(level_update4_kernel: 15.1 ms = 25.8 TF/s, bench v14)")
