"""Library baselines for the leaf phase of cfg2: batched LU (torch.linalg.lu_factor ->
cuSOLVER/cuBLAS getrfBatched) of 16384 64x64 blocks and the batched triangular
solves with 448 right-hand-side columns (torch.linalg.lu_solve), vs this engine's
bit-exact getrf_reg_kernel (1.27 ms) and tri_apply2_kernel with the fused [W|T] (2.95 ms)."""
import torch

B, s, ncols = 16384, 64, 448
A = torch.randn(B, s, s, dtype=torch.float64, device="cuda") / 8 + 4 * torch.eye(s, dtype=torch.float64, device="cuda")
X = torch.randn(B, s, ncols, dtype=torch.float64, device="cuda")


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


LU, piv = torch.linalg.lu_factor(A)
t_lu = ev_time(lambda: torch.linalg.lu_factor(A))
t_solve = ev_time(lambda: torch.linalg.lu_solve(LU, piv, X))
print(f"library batched LU (16384 x 64^2): {t_lu:.3f} ms   library batched LU solve (448 cols): {t_solve:.3f} ms")
