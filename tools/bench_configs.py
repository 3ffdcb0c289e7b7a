"""Timing of the other BASELINE.json configs on one B200 (the contract line is
bench.py = cfg2).  Prints one JSON object per configuration:

  cfg1  Gaussian kernel on 2^14 kd-ordered 2-D points (device-assembled), leaf 64, rank 32, fp64
  cfg3  Gaussian kernel on 2^21 3-D points (per-GPU share of 2^22 at P = 2), rank 64, fp64
  cfg4  rank-8 fp32 preconditioner, N = 2^21
  cfg5  multi-RHS solve sweep (1..256) on the cfg2 factorization (N = 2^20, r = 32)

Inputs: cfg1 / cfg3 operators assembled on the device (ACA rook); cfg4 / cfg5
use seeded exact-HODLR stand-ins generated in HBM.
Timing: CUDA events, warm-up first, median of the timed repetitions.
"""
import json, math, statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb


def solve_flops(n, m, r, nrhs):
    L = int(round(math.log2(n // m)))
    return nrhs * (2 * m * n + 4 * r * n * L + 8 * r * r * ((1 << L) - 1))


def solve_bytes(n, m, r, es, nrhs):
    L = int(round(math.log2(n // m)))
    return es * (m * n + 2 * n * r * L + 4 * r * r * ((1 << L) - 1)) + 2 * n * nrhs * es


def time_factor_solve(n, m, r, dtype, reps=5, nrhs=1, h0=None, graph=True):
    """(t_factor, t_solve, relres, eager) medians; graph=True times the captured
    launch sequences (hb.FactorPlan.refactor + hb.solve(graph=True)) and also
    returns the eager times for comparison."""
    if h0 is None:
        h0 = hb.random_hodlr(n, m, r, seed=0, s=1.0, dtype=dtype)
    b = torch.randn(n, nrhs, dtype=dtype, device="cuda").squeeze(1) if nrhs == 1 else torch.randn(n, nrhs, dtype=dtype, device="cuda")

    def run(use_graph):
        tf, ts = [], []
        plan = hb.FactorPlan(h0.clone(), check=False) if use_graph else None
        for it in range(reps + 2):
            if use_graph:
                plan.load(h0.D, h0.U)
            else:
                h = h0.clone()
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            f = plan.refactor(check=False) if use_graph else hb.factorize(h, check=False)
            e[1].record(); x = hb.solve(f, b, graph=use_graph); e[2].record()
            torch.cuda.synchronize()
            if it >= 2:
                tf.append(e[0].elapsed_time(e[1])); ts.append(e[1].elapsed_time(e[2]))
        return statistics.median(tf), statistics.median(ts), x

    tf_e, ts_e, x = run(False)
    eager = {"t_factor_ms": round(tf_e, 3), "t_solve_ms": round(ts_e, 3)}
    if graph:
        tf, ts, x = run(True)
    else:
        tf, ts = tf_e, ts_e
    res = float(torch.linalg.norm(h0.matvec(x) - b) / torch.linalg.norm(b))
    torch.cuda.empty_cache()
    return tf, ts, res, eager


def line(cfg, n, m, r, dtype_name, tf, ts, res, extra=None):
    fl_f = hb.flop_report(n, m, r)["total"]
    es = 4 if dtype_name == "f32" else 8
    d = {"config": cfg, "N": n, "leaf": m, "rank": r, "dtype": dtype_name, "t_factor_ms": round(tf, 3),
         "t_solve_ms": round(ts, 3), "factor_tflops": round(fl_f / tf / 1e9, 3),
         "solve_gbps": round(solve_bytes(n, m, r, es, 1) / ts / 1e6, 1), "relres": res}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


which = sys.argv[1:] or ["cfg1", "cfg3", "cfg4", "cfg5"]
if "cfg1" in which:
    # the cfg1 operator: Gaussian kernel (h = 0.1, lambda = 1) on 2^14 kd-ordered 2-D points, assembled on the device
    h1 = hb.gaussian_hodlr(1 << 14, 64, 32, dim=2, h=0.1, lam=1.0)
    tf, ts, res, eager = time_factor_solve(1 << 14, 64, 32, torch.float64, h0=h1, reps=20)
    # the reference's own CPU path on the same operator (its batched kernels, all host threads)
    extra = {"eager": eager, "launch": "CUDA graphs"}
    try:
        import os, time as _t
        import numpy as np
        from oracle import ref_driver as rd
        if rd.AVAILABLE:
            thr = os.cpu_count() or 1
            D, U, V = (x.cpu().numpy().copy() for x in (h1.D, h1.U, h1.V))
            bb = np.random.default_rng(1).standard_normal((1 << 14, 1))
            t0 = _t.perf_counter()
            dpiv, Ks, kp = rd.ref_factorize(D, U, V, 1 << 14, 64, 32, 8, rd.executor(thr))
            t1 = _t.perf_counter()
            rd.ref_solve(D, dpiv, U, V, Ks, kp, bb, 1 << 14, 64, 32, 8, rd.executor(thr))
            t2 = _t.perf_counter()
            extra["reference_cpu"] = {"t_factor_ms": round(1e3 * (t1 - t0), 1), "t_solve_ms": round(1e3 * (t2 - t1), 1),
                                      "threads": thr}
    except Exception as e:  # noqa: BLE001
        extra["reference_cpu"] = f"unavailable: {e}"
    line("cfg1 (Gaussian kernel, 2^14 2-D points)", 1 << 14, 64, 32, "f64", tf, ts, res, extra)
if "cfg3" in which:
    # per-GPU share of cfg3 at P = 2: Gaussian kernel on 2^21 kd-ordered 3-D points, rank 64
    h3 = hb.gaussian_hodlr(1 << 21, 64, 64, dim=3, h=0.1, lam=1.0)
    tf, ts, res, eager = time_factor_solve(1 << 21, 64, 64, torch.float64, reps=3, h0=h3, graph=False)
    del h3
    torch.cuda.empty_cache()
    line("cfg3-shape (Gaussian kernel, 2^21 3-D points: per-GPU share of N=2^22 at P=2)", 1 << 21, 64, 64, "f64",
         tf, ts, res)
if "cfg4" in which:
    tf, ts, res, eager = time_factor_solve(1 << 21, 64, 8, torch.float32)
    line("cfg4", 1 << 21, 64, 8, "f32", tf, ts, res, {"eager": eager, "launch": "CUDA graphs"})
if "cfg4r" in which or "cfg4" in which:
    # cfg4 as a preconditioner: fp32 factorization + fp64-operator refinement
    n, m, r = 1 << 21, 64, 8
    h64 = hb.random_hodlr(n, m, r, seed=0, s=1.0)
    h32 = hb.HodlrMatrix(h64.tree, r, h64.D.float(), h64.U.float(), h64.V.float())
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    runs = []
    for it in range(4):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); f32 = hb.factorize(h32.clone(), check=False); e[1].record()
        res = hb.solve_with_refinement(f32, h64, b, max_iters=10, tol=1e-12); e[2].record()
        torch.cuda.synchronize()
        if it >= 1:
            runs.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), res))
        del f32
    tf = statistics.median(t[0] for t in runs); tr = statistics.median(t[1] for t in runs)
    res = runs[-1][2]
    tf64, ts64, res64, _ = time_factor_solve(n, m, r, torch.float64, reps=3, graph=False)
    print(json.dumps({"config": "cfg4 preconditioner: fp32 factor + fp64 refinement", "N": n, "leaf": m, "rank": r,
                      "t_factor_f32_ms": round(tf, 3), "t_refine_ms": round(tr, 3),
                      "iterations": res.iterations, "relres_history": res.history,
                      "fp64_direct": {"t_factor_ms": round(tf64, 3), "t_solve_ms": round(ts64, 3), "relres": res64}}),
          flush=True)
    del h64, h32
    torch.cuda.empty_cache()
if "cfg4g" in which or "cfg4" in which:
    # BASELINE cfg4 as specified: rank-8 fp32 HODLR preconditioner for the Schur-complement
    # surrogate (planar-separator DtN kernel, N = 2^21), inside GMRES, to relres 1e-10
    import time as _t
    n, m = 1 << 21, 64
    torch.cuda.synchronize(); t0 = _t.perf_counter()
    op = hb.schur_surrogate_hodlr(n, m, 32, sigma=0.1)
    p8 = hb.schur_surrogate_hodlr(n, m, 8, sigma=0.1)
    torch.cuda.synchronize(); t_build = _t.perf_counter() - t0
    h32 = hb.HodlrMatrix(p8.tree, 8, p8.D.float(), p8.U.float(), p8.V.float())
    del p8
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    runs = []
    for it in range(3):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); prec = hb.factorize(h32.clone(), check=False); e[1].record()
        res = hb.gmres_hodlr(op, prec, b, tol=1e-10, restart=30); e[2].record()
        torch.cuda.synchronize()
        runs.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), res))
        del prec
    tf = statistics.median(t[0] for t in runs); tg = statistics.median(t[1] for t in runs)
    res = runs[-1][2]
    # fp64 direct solve of the same rank-32 operator, for comparison
    tf64, ts64, res64, _ = time_factor_solve(n, m, 32, torch.float64, reps=3, h0=op, graph=False)
    print(json.dumps({"config": "cfg4: GMRES on the Schur-complement surrogate (planar-separator DtN kernel, fp64 "
                                "rank-32 HODLR operator) preconditioned by a rank-8 fp32 HODLR factorization",
                      "N": n, "leaf": m, "rank_prec": 8, "rank_op": 32, "build_s": round(t_build, 2),
                      "t_prec_factor_ms": round(tf, 3), "t_gmres_ms": round(tg, 3), "iterations": res.iterations,
                      "restarts": res.restarts, "converged": res.converged, "true_relres": res.true_relres,
                      "history": [float(f"{v:.3e}") for v in res.history],
                      "fp64_direct_rank32": {"t_factor_ms": round(tf64, 3), "t_solve_ms": round(ts64, 3),
                                             "relres": res64}}), flush=True)
    del op, h32
    torch.cuda.empty_cache()
if "profile" in which:
    # the Laplace operator at N = 2^22 with the paper's rank profile (PAPER.md appendix:
    # 24 22 15 14 13 13 13 13 14 14 15 16 16 17 17 18, levels 1..16), per-level ranks padded
    # to the fused-kernel ranks, vs the same operator at uniform rank 32
    n, m = 1 << 22, 64
    prof = (24, 22, 15, 14, 13, 13, 13, 13, 14, 14, 15, 16, 16, 17, 17, 18)
    padded = tuple(16 if k <= 16 else 32 for k in prof)
    h32 = hb.laplace_dl_hodlr(n, m, 32)
    rows = []
    for name, h in (("uniform 32", h32), ("per-level (paper profile, padded)", hb.truncate_ranks(h32, padded))):
        tf, ts, res, eager = time_factor_solve(n, m, 32, torch.float64, reps=3, h0=h, graph=False)
        fl = hb.flop_report(n, m, 32, ranks=h.ranks)["total"]
        rows.append({"layout": name, "ranks": list(h.level_ranks), "t_factor_ms": round(tf, 3),
                     "t_solve_ms": round(ts, 3), "factor_gflop": round(fl / 1e9, 1), "relres": res,
                     "bytes_UV": 2 * h.U.numel() * 8})
        if h is not h32:
            del h
    print(json.dumps({"config": "Laplace DL N=2^22 at the paper's rank profile vs uniform rank 32", "runs": rows}),
          flush=True)
    del h32
    torch.cuda.empty_cache()
if "cfg5" in which:
    n, m, r = 1 << 20, 64, 32
    f = hb.factorize(hb.random_hodlr(n, m, r, seed=0, s=1.0), check=False)
    for nrhs in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda")
        ts = []
        for it in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); X = hb.solve(f, B); e1.record(); torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        print(json.dumps({"config": "cfg5 multi-RHS solve on the cfg2 factorization", "N": n, "rank": r, "nrhs": nrhs,
                          "t_solve_ms": round(t, 3), "solve_tflops": round(solve_flops(n, m, r, nrhs) / t / 1e9, 3),
                          "solve_gbps": round(solve_bytes(n, m, r, 8, nrhs) / t / 1e6, 1)}), flush=True)
        del B, X
