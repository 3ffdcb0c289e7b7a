"""HODLR factor+solve benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): N = 2^20, leaf m = 64, uniform rank
r = 32, L = 14, fp64, 1 RHS, on the cfg2 operator itself -- the exterior
Laplace double-layer BIE on contour_default(N) (problems.py:133-217), z = 0,
assembled in HBM by the device builder (ACA rook, rank 32, bit-exact vs the
reference's compress(); ``build_ms`` reports it, outside the step).
``--problem standin`` uses the seeded exact-HODLR stand-in instead.  A step =
one factorize (PAPER Alg. 3) + one solve (Alg. 4) of a freshly restored copy
of the matrix; the restore copy is outside the timed events.  Inputs (8 GB)
exceed L2 (126 MB), so no explicit flush is needed.

Multi-GPU (--gpus N > 1; re-executed under torch.distributed.run when not
already launched by torchrun): one process per GPU running the subtree-sharded
factorization + solve of ONE matrix -- by default the north_star scaling case,
BASELINE cfg3 (N = 2^22, leaf 64, rank 64, 3-D Gaussian kernel) -- with one
NCCL sum all-reduce per top level, "scaling": "strong", time = max over ranks
of the CUDA-event step time.  `--workload cfg3` at N = 1 gives the matching
single-GPU base.  Rank 0 prints one JSON line.

--impl reference: the reference's CPU path (its own batched kernels driven by
the SPEC recipe, oracle/ref_driver.py, all host threads) on a bounded sample
of the same workload: the leading 2^16-row subtree of the cfg2 operator,
assembled by the reference's own compress() (built once, outside the timing),
rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT, M_LEAF, RANK = 1 << 20, 64, 32
SEED, SCALE = 1234, 1.0
METRIC = "hodlr_factor_solve_tflops"
CPU_SAMPLE_N = 1 << 16


PROBLEM_DESC = {
    "laplace": "Laplace double-layer BIE on contour_default(N), z=0, assembled on the device (ACA rook, rank 32)",
    "standin": "seeded exact-HODLR stand-in",
}


def make_operator(hb, torch, n, m, r, problem, rank):
    """The workload operator in HBM and its assembly time (ms)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if problem == "laplace":
        h = hb.laplace_dl_hodlr(n, m, r)
    else:
        h = hb.random_hodlr(n, m, r, seed=SEED + rank, s=SCALE)
    torch.cuda.synchronize()
    return h, 1e3 * (time.perf_counter() - t0)


def subtree_of(h, n_sub):
    """(D, U, V) numpy of the leading n_sub-row subtree of a device HODLR."""
    m, r, L, n = h.m, h.rank, h.L, h.n
    Ls = int(round(math.log2(n_sub // m)))
    D = h.D[: (n_sub // m) * m * m].cpu().numpy()
    U = h.U.view(L, r, n)[L - Ls :, :, :n_sub].contiguous().view(-1).cpu().numpy()
    V = h.V.view(L, r, n)[L - Ls :, :, :n_sub].contiguous().view(-1).cpu().numpy()
    return D, U, V


def factor_flops(n, m, r):
    from oracle import hodlr_oracle as orc  # closed form only (no oracle compute)

    return orc.factor_flops(n, m, r)


def solve_flops(n, m, r, nrhs=1):
    L = int(round(math.log2(n // m)))
    return nrhs * (2 * m * n + 4 * r * n * L + 8 * r * r * ((1 << L) - 1))


def level_flops(n, m, r):
    """Algorithmic flops of the fused level-step launches (update + next [W|T])."""
    L = int(round(math.log2(n // m)))
    return sum(4 * r * r * n * lv for lv in range(1, L))


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, ~10 ms) during the timed region."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0):
        self.index, self.samples, self.reasons, self._stop = index, [], set(), threading.Event()
        self.max_mhz = None
        self._ready = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            hd = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(hd, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                self.samples.append(nv.nvmlDeviceGetClockInfo(hd, nv.NVML_CLOCK_SM))
                self._ready.set()
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(hd)
                for name, attr in self.REASONS:
                    if mask & getattr(nv, attr):
                        self.reasons.add(name)
                self._stop.wait(0.01)
        except Exception as e:  # pragma: no cover - diagnostics only
            self.reasons.add(f"nvml unavailable: {e}")
        finally:
            self._ready.set()

    def __enter__(self):
        # NVML import/init runs before the timed region starts: an import holding
        # the GIL inside the region would stall the launching thread
        self._t.start()
        self._ready.wait(timeout=30)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, backend):
    import torch.distributed as dist

    if world > 1 and int(os.environ.get("WORLD_SIZE", "1")) > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return dist


def measure_dgemm_peak(torch):
    """cuBLAS DGEMM 8192^3 (burst): the FP64 tensor roofline denominator
    (MEASURED_PEAKS.json carries bf16 only)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * n**3 / (best * 1e-3) / 1e12


def read_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return {}


def traffic_from_profiles():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        d = json.loads(p.read_text())
        return d.get("level_update_bytes_per_launch"), d
    except Exception:
        return None, None


def cpu_sample(n, problem, sub=None):
    """The bounded CPU sample: the leading n-row subtree of the workload
    operator.  ``sub`` = (D, U, V) already extracted from the device copy (bit
    identical to the reference's compress(), tests/test_gpu_build.py); else the
    reference assembles it with its own compress() (stand-in: the oracle generator)."""
    from oracle import hodlr_oracle as orc
    from oracle import ref_driver as rd

    lay = orc.Layout(n, M_LEAF, RANK)
    if problem == "standin":
        return orc.make_exact_hodlr(n, M_LEAF, RANK, seed=SEED, s=SCALE)
    if sub is None:
        if rd.AVAILABLE:
            sub = rd.ref_assemble_laplace(N_DEFAULT, n, M_LEAF, RANK)
        else:
            from oracle import build_oracle as bo

            sub = bo.assemble(bo.LaplaceDL(N_DEFAULT), n, M_LEAF, RANK)
    return orc.HodlrData(lay, *(x.copy() for x in sub))


def cpu_reference(n, threads, sample=None, keep=False):
    """The reference's CPU path on a bounded sample: Alg. 3/4 issuing the
    reference's own batched kernels (baseline/_ref, threads:<ncores> executor)
    when installed -- kind "reference" -- else the oracle restatement ("port").
    keep=True also returns the outputs (leaf LU + swaps, Y, K + swaps, x, b)."""
    import numpy as np

    from oracle import hodlr_oracle as orc
    from oracle import ref_driver as rd

    h = sample.copy() if sample is not None else orc.make_exact_hodlr(n, M_LEAF, RANK, seed=SEED, s=SCALE)
    b = np.random.default_rng(SEED + 1).standard_normal((n, 1))
    L, r = h.lay.L, h.lay.r
    fl = orc.factor_flops(n, M_LEAF, r) + orc.solve_flops(n, M_LEAF, r)
    if rd.AVAILABLE:
        ex = rd.executor(threads)
        t0 = time.perf_counter()
        dpiv, Ks, kpivs = rd.ref_factorize(h.D, h.U, h.V, n, M_LEAF, r, L, ex)
        t1 = time.perf_counter()
        x = rd.ref_solve(h.D, dpiv, h.U, h.V, Ks, kpivs, b, n, M_LEAF, r, L, ex)
        t2 = time.perf_counter()
        outs = dict(D=h.D, dswaps=dpiv.swaps, Y=h.U, K=np.concatenate(Ks),
                    kswaps=np.concatenate([p.swaps for p in kpivs]), x=x, b=b) if keep else None
        return fl, t1 - t0, t2 - t1, "reference", outs
    t0 = time.perf_counter()
    f = orc.factorize(h, threads=threads)
    t1 = time.perf_counter()
    x = orc.solve(f, b, threads=threads)
    t2 = time.perf_counter()
    outs = dict(D=f.D, dswaps=f.dpiv.swaps, Y=f.Y, K=np.concatenate(f.K),
                kswaps=np.concatenate([p.swaps for p in f.kpiv]), x=x, b=b) if keep else None
    return fl, t1 - t0, t2 - t1, "port", outs


def parity_vs_cpu(hb, sample, outs, kind):
    """The GPU factorize/solve of the CPU arm's exact sample vs the CPU arm's
    outputs (north_star: pivots bit-exact, x within 1e-10)."""
    import numpy as np

    n, m, r = sample.lay.n, sample.lay.m, sample.lay.r
    f = hb.factorize(hb.HodlrMatrix.from_buffers(n, m, r, sample.D, sample.U, sample.V))
    x = hb.solve(f, outs["b"])

    def rel(a, b):
        return float(np.linalg.norm(a - b) / np.linalg.norm(b))

    return {
        "against": "reference kernels (baseline/_ref)" if kind == "reference" else "oracle restatement",
        "sample": f"leading 2^{int(math.log2(n))}-row subtree of the workload (the cpu_baseline sample)",
        "leaf_lu_bitexact": bool(np.array_equal(f.D.cpu().numpy(), outs["D"])),
        "pivots_bitexact": bool(np.array_equal(f.dswaps.cpu().numpy().reshape(-1, m), outs["dswaps"])
                                and np.array_equal(f.kswaps.cpu().numpy().reshape(-1, 2 * r), outs["kswaps"])),
        "x_relerr": rel(x, outs["x"]), "y_relerr": rel(f.Y.cpu().numpy(), outs["Y"]),
        "k_relerr": rel(f.K.cpu().numpy(), outs["K"]), "tol": 1e-10,
    }


def cfg3_cpu_sample(n):
    """The cfg3 CPU sample: the cfg3 operator family at n rows (Gaussian kernel,
    h = 0.1, lam = 1, on n kd-ordered xorshift64* 3-D points, seed 0), rank 64,
    assembled with the reference's own compress() on a numpy entry oracle."""
    from oracle import build_oracle as bo
    from oracle import hodlr_oracle as orc
    from oracle import ref_driver as rd
    from paper_2208_06290_b200.construct import kd_points  # host-side point generation only

    r = WORKLOADS["cfg3"][1]
    L = int(round(math.log2(n // M_LEAF)))
    ent = bo.Gaussian(kd_points(n, 3, L, seed=0), h=0.1, lam=1.0)
    D, U, V = rd.ref_assemble(ent, n, M_LEAF, r) if rd.AVAILABLE else bo.assemble(ent, n, M_LEAF, r)
    return orc.HodlrData(orc.Layout(n, M_LEAF, r), D, U, V)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    workload = args.workload or ("cfg3" if (args.gpus > 1 or world > 1) else "cfg2")
    N, r = WORKLOADS[workload][:2]
    n = CPU_SAMPLE_N if workload == "cfg2" else CPU_SAMPLE_N // 2
    if args.cpu_sample_rows:
        n = args.cpu_sample_rows
    cpu_reference(1 << 12, threads)  # warm-up (imports, thread pool)
    t0 = time.perf_counter()
    sample = cpu_sample(n, args.problem) if workload == "cfg2" else cfg3_cpu_sample(n)  # outside the timed steps
    build_s = time.perf_counter() - t0
    vals, tfs, tss = [], [], []
    kind = "port"
    for _ in range(args.steps):
        fl, tf, ts, kind, _ = cpu_reference(n, threads, sample)
        vals.append(fl / (tf + ts) / 1e12)
        tfs.append(tf)
        tss.append(ts)
    v = statistics.mean(vals)
    how = ("reference batched kernels (baseline/_ref hodlr.backend, threads executor) driven by the SPEC "
           "Alg. 3/4 recipe" if kind == "reference" else "oracle restatement of the reference kernels")
    what = (f"the leading 2^{int(math.log2(n))}-row subtree of the cfg2 workload (m=64, r=32, fp64; "
            f"{PROBLEM_DESC[args.problem]})" if workload == "cfg2" else
            f"the cfg3 operator family at 2^{int(math.log2(n))} rows (3-D Gaussian kernel, m=64, r=64, fp64, "
            "compressed by the reference's compress())")
    sample = f"{how}: factor+solve of {what}, {args.steps} step(s); sample assembled once in {build_s:.1f} s"
    wdesc = WORKLOADS[workload][2] + (PROBLEM_DESC[args.problem] if workload == "cfg2" else "")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean([a + b for a, b in zip(tfs, tss)]),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the arm's config is the GPU arm's; each step is a bounded sample of it
        # (stated in cpu_baseline.sample)
        "config": {"workload": wdesc, "N": N, "leaf": M_LEAF, "rank": r, "L": int(math.log2(N // M_LEAF)), "nrhs": 1,
                   "parallelism": "cpu (reference)", "sample_rows": n, "device": "cpu"},
        "t_factor_s": statistics.mean(tfs), "t_solve_s": statistics.mean(tss),
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import ctypes as C

    import numpy as np
    import torch

    import paper_2208_06290_b200 as hb
    from paper_2208_06290_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = init_dist(world, "nccl")
    lib = _lib.load()
    n, m, r = args.n, M_LEAF, RANK
    L = int(round(math.log2(n // m)))
    f_flops, s_flops = factor_flops(n, m, r), solve_flops(n, m, r)

    # resident input (HBM) and a pristine copy for restores
    h0, build_ms = make_operator(hb, torch, n, m, r, args.problem, rank)
    hw = h0.clone()
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED + 7 + rank)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)

    def restore():
        hw.D.copy_(h0.D)
        hw.U.copy_(h0.U)

    # the public repeated-factorization API: one eager factorization, then the
    # captured launch sequence (CUDA graph) replayed on the restored buffers;
    # the solve replays its own captured graph (hb.solve(graph=True))
    plan = hb.FactorPlan(hw, check=False)

    def step(graph=True):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        f = plan.refactor(check=False) if graph else hb.factorize(hw, check=False)
        e1.record()
        x = hb.solve(f, b, graph=graph)
        e2.record()
        return f, x, (e0, e1, e2)

    for _ in range(args.warmup):
        restore()
        step()
    torch.cuda.synchronize()

    # ---- timed region ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tf_ms, ts_ms = [], []
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            restore()
            _, _, ev = step()
            tf_ms.append(ev)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [ev[0].elapsed_time(ev[2]) for ev in tf_ms]
    tf = sum(ev[0].elapsed_time(ev[1]) for ev in tf_ms) / args.steps
    ts = sum(ev[1].elapsed_time(ev[2]) for ev in tf_ms) / args.steps
    t_step = tf + ts

    # the same steps launched eagerly (no graphs), for comparison
    eager = []
    for _ in range(3):
        restore()
        _, _, ev = step(graph=False)
        eager.append(ev)
    torch.cuda.synchronize()
    eager_f = statistics.median(ev[0].elapsed_time(ev[1]) for ev in eager)
    eager_s = statistics.median(ev[1].elapsed_time(ev[2]) for ev in eager)

    # per-phase event profile + launch count of one (eager) step (after the timed loop)
    restore()
    lib.hodlr_profile_enable(1)
    c0 = lib.hodlr_launch_count()
    f, x, _ = step(graph=False)
    torch.cuda.synchronize()
    launches_per_step = lib.hodlr_launch_count() - c0
    ph = (C.c_double * 9)()
    lib.hodlr_profile_read(ph, 9)
    lib.hodlr_profile_enable(0)
    phases = {name: ph[i] for i, name in enumerate(_lib.PHASES)}
    # accuracy of this step: relres against the HODLR operator
    relres = float(torch.linalg.norm(h0.matvec(x) - b) / torch.linalg.norm(b))
    # HODLR matvec (hodlr_matvec): HBM-bound, bytes = 8 (m N + 2 r N L) + 24 N
    mv_ms = []
    for it in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0.matvec(x)
        e1.record()
        e1.synchronize()
        if it > 0:
            mv_ms.append(e0.elapsed_time(e1))
    mv_t = statistics.median(mv_ms)
    mv_bytes = 8 * (m * n + 2 * r * n * L) + 24 * n
    del f, x
    if world > 1:
        tt = torch.tensor([t_step, tf, ts], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, tf, ts = tt.tolist()
    value = world * (f_flops + s_flops) / (t_step * 1e-3) / 1e12

    # ---- e2e through the public API with host buffers (pinned) ----
    e2e = None
    if rank == 0 and not args.no_e2e:
        Dh = h0.D.cpu().pin_memory()
        Uh = h0.U.cpu().pin_memory()
        Vh = h0.V.cpu().pin_memory()
        bh = b.cpu().pin_memory()
        e2e_t = []
        for it in range(2 + 2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            # public API: host (pinned) inputs, upload overlapped with the factorization
            fe = hb.factorize_from_host(n, m, r, Dh, Uh, Vh)
            xh = hb.solve(fe, bh)  # host rhs in, host solution out
            torch.cuda.synchronize()
            if it >= 2:
                e2e_t.append(time.perf_counter() - t0)
            del fe, xh
        te = statistics.mean(e2e_t)
        h2d = (Dh.numel() + Uh.numel() + Vh.numel() + bh.numel()) * 8
        # the same public calls from pageable numpy inputs (staged through the pinned ring by the library)
        Dp, Up, Vp, bp = (np.array(x.numpy()) for x in (Dh, Uh, Vh, bh))
        pg_t = []
        for it in range(1 + 2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fe = hb.factorize_from_host(n, m, r, Dp, Up, Vp)
            xh = hb.solve(fe, bp)
            torch.cuda.synchronize()
            if it >= 1:
                pg_t.append(time.perf_counter() - t0)
            del fe, xh
        del Dp, Up, Vp, bp
        tpg = statistics.mean(pg_t)
        # the e2e roofline: pinned host -> device copy bandwidth of this box (1 GiB, best of 3)
        src = torch.empty(1 << 27, dtype=torch.float64, pin_memory=True)
        dst = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
        bw = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); dst.copy_(src, non_blocking=True); e1.record(); e1.synchronize()
            bw.append(src.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        del src, dst
        h2d_gbps = max(bw)
        e2e = {"value": (f_flops + s_flops) / te / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": n * 8 + ((1 << L) + (1 << L) - 1) * 4, "seconds_per_step": te,
               "roofline": {"bound": "pcie_h2d", "achieved_gbps": h2d / te / 1e9, "peak_gbps": h2d_gbps,
                            "frac": (h2d / te / 1e9) / h2d_gbps,
                            "peak_source": "pinned 1 GiB host->device copy in this run (best of 3)"},
               "pageable": {"value": (f_flops + s_flops) / tpg / 1e12, "seconds_per_step": tpg,
                            "note": "same calls from pageable numpy D/U/V/b (staged through the library's pinned ring inside the timed region)"}}

    # ---- roofline of the dominant kernel (fused level step) ----
    peaks = read_peaks()
    dgemm = measure_dgemm_peak(torch) if rank == 0 else None
    lvl_ms = phases["level"]
    lvl_achieved = level_flops(n, m, r) / (lvl_ms * 1e-3) / 1e12 if lvl_ms > 0 else None
    level_launches = L - 1
    traffic, _ = traffic_from_profiles()

    if rank == 0:
        cpu = parity = None
        if not args.no_cpu:
            threads = os.cpu_count() or 1
            samp = cpu_sample(CPU_SAMPLE_N, args.problem, subtree_of(h0, CPU_SAMPLE_N) if args.problem == "laplace" else None)
            fl, ctf, cts, kind, outs = cpu_reference(CPU_SAMPLE_N, threads, samp, keep=True)
            cpu = {"value": fl / (ctf + cts) / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
                   "sample": ("reference kernels (baseline/_ref) via the SPEC recipe" if kind == "reference"
                              else "oracle restatement") + ": factor+solve of the leading 2^16-row subtree of this "
                   f"workload (m=64, r=32, fp64), {ctf:.1f} s factor + {cts:.2f} s solve"}
            parity = parity_vs_cpu(hb, samp, outs, kind)
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "HODLR factor+solve, cfg2 (N=2^20, leaf 64, rank 32, L=14, 1 RHS), "
                                   + PROBLEM_DESC[args.problem], "N": n, "leaf": m, "rank": r, "L": L, "nrhs": 1,
                       "parallelism": f"replicas{world}", "l2_flush": "inputs 8 GB > L2"},
            "t_factor_ms": tf, "t_solve_ms": ts, "factor_tflops": f_flops / (tf * 1e-3) / 1e12, "build_ms": build_ms,
            "launch": "CUDA graphs (hb.FactorPlan.refactor + hb.solve(graph=True))",
            "eager_ms": {"factor": eager_f, "solve": eager_s},
            "step_ms_min_med_max": [min(step_ms), statistics.median(step_ms), max(step_ms)],
            "solve_gbps": (8 * (m * n + 2 * n * r * L + 4 * r * r * ((1 << L) - 1)) + 16 * n) / (ts * 1e-3) / 1e9,
            "relres": relres, "flops_factor": f_flops, "flops_solve": s_flops,
            "matvec": {"ms": mv_t, "GB_per_s": mv_bytes / (mv_t * 1e-3) / 1e9, "bytes": mv_bytes,
                       "frac_hbm": (mv_bytes / (mv_t * 1e-3) / 1e9 / peaks["hbm_gbs"]) if peaks.get("hbm_gbs") else None},
            "phase_ms": phases, "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "tensor", "kernel": "level phase: level_update6_kernel (persistent, C tile + panels by TMA) and "
                                   "level_update4/5 (remainder groups, small levels), fused Y update + next-level [W|T]; "
                                   "traffic = mean DRAM bytes per level step (ncu, profiles/traffic.json)",
                         "achieved": lvl_achieved, "peak": dgemm, "unit": "TFLOP/s",
                         "frac": (lvl_achieved / dgemm) if (lvl_achieved and dgemm) else None,
                         "peak_source": "measured cuBLAS DGEMM 8192^3 in this run (MEASURED_PEAKS.json has no fp64)",
                         "alt_peak": {"tflops": 37.11, "frac": (lvl_achieved / 37.11) if lvl_achieved else None,
                                      "source": "DMMA micro-benchmark ceiling (32 warps/SM of independent "
                                                "mma.m8n8k4.f64, 1965 MHz), profiles/r01_fp64_peak_probe.txt"},
                         "traffic": traffic, "level_steps_per_step": level_launches,
                         "flops_per_step": level_flops(n, m, r)},
            "clocks": clk.summary(), "wall_s_timed": wall,
            "hbm_peak_measured_gbps": peaks.get("hbm_gbs"),
            "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


WORKLOADS = {
    # name: (N, rank, description) -- BASELINE.json configs[1] / configs[2]
    "cfg2": (1 << 20, 32, "HODLR factor+solve, cfg2 (N=2^20, leaf 64, rank 32, L=14, 1 RHS), "),
    "cfg3": (1 << 22, 64, "HODLR factor+solve, cfg3 (N=2^22, leaf 64, rank 64, L=16, 1 RHS), Gaussian kernel "
                          "exp(-|x-y|^2/h^2) + I (h=0.1) on 2^22 kd-ordered 3-D points, assembled on the device"),
}


def make_sharded_operator(hb, torch, workload, n, problem):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if workload == "cfg3":
        h = hb.gaussian_hodlr(n, M_LEAF, WORKLOADS["cfg3"][1], dim=3, h=0.1, lam=1.0)
    elif problem == "laplace":
        h = hb.laplace_dl_hodlr(n, M_LEAF, RANK)
    else:
        h = hb.random_hodlr(n, M_LEAF, RANK, seed=SEED, s=SCALE)
    torch.cuda.synchronize()
    return h, 1e3 * (time.perf_counter() - t0)


def run_sharded(args):
    """N > 1 (or --sharded): one matrix row-sharded over the ranks (strong
    scaling; default workload cfg3, the north_star scaling case N = 2^22,
    r = 64): rank g owns the rows of level-p node g (P = 2^p), levels >= p are
    local, one sum all-reduce of the packed [W|T] (resp. w) per top level over
    NCCL.  Every rank assembles the operator on its own GPU and
    keeps only its shard."""
    import ctypes as C

    import torch

    import paper_2208_06290_b200 as hb
    from paper_2208_06290_b200 import _lib
    from paper_2208_06290_b200 import distributed as dd

    rank, world, local = dist_env()
    torch.cuda.set_device(local if args.dist_backend == "nccl" else 0)
    dist = init_dist(max(world, 2) if world > 1 else 1, args.dist_backend)
    lib = _lib.load()
    workload = args.workload or ("cfg3" if world > 1 else "cfg2")
    n = args.n or WORKLOADS[workload][0]
    m, r = M_LEAF, WORKLOADS[workload][1]
    L = int(round(math.log2(n // m)))
    f_flops, s_flops = factor_flops(n, m, r), solve_flops(n, m, r)
    h0, build_ms = make_sharded_operator(hb, torch, workload, n, args.problem)  # identical on every rank
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED + 7)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    pristine = dd.make_shard(h0, rank, world)
    n_loc, row0 = pristine.n_loc, pristine.row0
    b_loc = b[row0 : row0 + n_loc].clone()
    keep_full = rank == 0 and not args.no_relres
    if not keep_full:
        del h0
        torch.cuda.empty_cache()
    work = dd.make_shard_like(pristine)
    backend = dd.GpuBackend()

    def all_reduce(buf):
        if world > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)

    def step():
        work.D.copy_(pristine.D)
        work.U.copy_(pristine.U)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        st = dd.factorize_sharded(work, all_reduce, backend, check=False)
        e1.record()
        x = b_loc.clone()
        dd.solve_sharded(st, x, 1, all_reduce, backend)
        e2.record()
        return x, (e0, e1, e2)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lib.hodlr_profile_enable(1)
    c0 = lib.hodlr_launch_count()
    x, _ = step()
    torch.cuda.synchronize()
    launches_per_step = lib.hodlr_launch_count() - c0
    ph = (C.c_double * 9)()
    lib.hodlr_profile_read(ph, 9)
    lib.hodlr_profile_enable(0)
    phases = {name: ph[i] for i, name in enumerate(_lib.PHASES)}
    xs = [torch.empty_like(x) for _ in range(world)] if world > 1 else [x]
    if world > 1:
        dist.all_gather(xs, x)
    relres = None
    if keep_full:
        xg = torch.cat(xs)
        relres = float(torch.linalg.norm(h0.matvec(xg) - b) / torch.linalg.norm(b))
        del h0, xg
        torch.cuda.empty_cache()
    del xs

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            _, ev = step()
            evs.append(ev)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    tf = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    ts = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    tt = torch.tensor([tf + ts, tf, ts], device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step, tf, ts = tt.tolist()
    value = (f_flops + s_flops) / (t_step * 1e-3) / 1e12
    if rank == 0:
        desc = WORKLOADS[workload][2] + (PROBLEM_DESC[args.problem] if workload == "cfg2" else "")
        if n != WORKLOADS[workload][0]:
            desc += f"; run at N=2^{int(round(math.log2(n)))} (--rows)"
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc + ", row-sharded", "N": n, "leaf": m, "rank": r, "L": L,
                       "nrhs": 1, "parallelism": f"subtree-shard{world} ({args.dist_backend} all-reduce per top level)",
                       "l2_flush": "inputs > L2 (126 MB)"},
            "t_factor_ms": tf, "t_solve_ms": ts, "relres": relres, "phase_ms_rank0": phases, "build_ms": build_ms,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(), "wall_s_timed": wall,
            "roofline": {"bound": "tensor", "kernel": "level phase (level_update6/4/5)", "achieved":
                         (level_flops(n // world, m, r) / (phases["level"] * 1e-3) / 1e12) if phases["level"] else None,
                         "peak": None, "unit": "TFLOP/s", "frac": None, "traffic": None,
                         "note": "rank 0's local level phase; the per-kernel roofline is reported by the N=1 run"},
            "e2e": None, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a torchrun environment: re-exec under
    torch.distributed.run with one process per GPU (127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if args.dist_backend == "nccl":
        env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) on stdout
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rows", dest="n", type=int, default=None, help="matrix size N (default: the workload's)")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default=None,
                    help="cfg2 (default at N=1) or cfg3 (default for the sharded N>1 run)")
    ap.add_argument("--problem", choices=("laplace", "standin"), default="laplace",
                    help="cfg2 operator: laplace (assembled on the device) or the seeded exact-HODLR stand-in")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-relres", action="store_true", help="sharded run: skip the full-operator residual")
    ap.add_argument("--sharded", action="store_true", help="use the row-sharded path even on one GPU")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (one GPU per rank) or gloo (single-GPU testing)")
    ap.add_argument("--cpu-sample-rows", type=int, default=None, help=argparse.SUPPRESS)  # tests: smaller CPU sample
    args = ap.parse_args()
    if args.impl == "reference":
        if dist_env()[0] == 0:
            run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if dist_env()[1] > 1 or args.sharded or (args.workload == "cfg3"):
        run_sharded(args)
    else:
        if args.n is None:
            args.n = N_DEFAULT
        run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
