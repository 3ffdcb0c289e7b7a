// Solve level step (Alg. 4 line 7 of level l fused with line 5 of
// level l-1), TMA-fed and persistent:
//
//     x(I_c, :) -= Y_c^{l+1} w'_c           (w' = half of K_p^-1 w_p, per child c)
//     w_q       += V_q^{(l) T} x(I_q, :)     (the next level's w, per node q)
//
// One CTA per SM walks a flat stream of CH-row chunks of its work items
// (canonical unit x block of GB column groups of 8 right-hand sides).  The Y
// and V panels of every chunk arrive by two 2-D tensor copies into an NS-stage
// ring (mbarrier transaction counts); the panels are read from HBM once for
// all GB groups.  Within a chunk the work is split over the 8 warps only along
// directions the canonical operation order does not depend on:
//
//   phase 1  (16-row band, group): x tile chain over the ranks, Y fragments
//            from the staged panel (LDS.128 row pairs), w' from L1/L2; the new
//            x goes to HBM and to a shared x tile;
//   phase 2  (8-rank tile, group): the w partial chain over the chunk's rows,
//            A = the shared x tile, B = the staged V panel.
//
// The operation order per right-hand-side column is exactly the one of
// solve_level_kernel (level.cu): x tile chain over (kt, u); each 64-row chunk's
// w partial a DMMA chain from zero over (band, h, even/odd row), added to the
// running sum of its canonical unit (min(node rows, 512) rows) in row order;
// units of larger nodes combined by level_reduce_kernel.  A column of a
// multi-RHS solve is therefore bit-identical to the single-vector solve
// (SPEC.md:405), whichever kernel ran either.
//
// Warp-specialized: a producer warp streams the chunks, four warps update x
// (phase 1) while four others form the w partials of the chunk before
// (phase 2); the shared x tile between them is double-buffered.
#include "common.cuh"
#include "tma.cuh"

namespace hodlr {

struct SolveStepArgs {
  double* X;  // right-hand sides, rows [0, n), column-major (ld ldx)
  int64_t ldx;
  const double* W;  // w' per parent: 2R x ncols (ld 2R) at W + p * wstride
  int64_t wstride;
  double* out;  // next-level w: final paired layout, or per-unit partials [unit][R x ncols]
  int64_t tw_stride;
  int partial;
  int n_c;        // rows per child at level l+1 (clamped)
  int unit_rows;  // canonical unit: min(node_rows, 512)
  int64_t node_rows;
  int ncols;
  int ncg;         // column blocks of GB groups
  int64_t nitems;  // units * ncg
};

template <int R, int GB, int CH>
struct SolveCfg {
  static constexpr int P = CH + 2;  // row pitch of the panel / x tiles: every LDS.128 quarter-warp conflict-free
  static constexpr int PANEL = R * P;
  static constexpr int XT = 8 * GB * P;       // x tile of the chunk (TMA, [column][row])
  static constexpr int PW = R + 8;            // w' tile pitch ([column][rank]; (PW / 2) = 4 mod 8)
  static constexpr int WT = 8 * GB * PW;      // w' tile of the chunk's child (TMA)
  static constexpr int STAGE = 2 * PANEL + XT + WT;
  static constexpr int NB = CH / 16;    // 16-row bands per chunk
  static constexpr int NSUB = 64 / CH;  // TMA chunks per canonical 64-row chunk
};

__device__ __forceinline__ void stg_x4(double* p, double x, double y, double z, double w) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(w)
               : "memory");
}

// Warp roles: warps 0-3 (A) update x (phase 1), warps 4-7 (B) form the w
// partials (phase 2) of the previous chunk at the same time, warp 8 issues the
// tensor copies.  Barriers: full[s] (TMA bytes landed), empty[s] (8 consumer
// warps done with the stage) -- mbarriers; the double-buffered shared x tile
// is handed from A to B and back with named barriers (producer bar.arrive,
// consumer bar.sync over the 8 compute warps: ready[b] = 1 + b, free[b] = 3 + b).
constexpr int kSolveA = 4, kSolveB = 4, kSolveThreads = 32 * (kSolveA + kSolveB + 1);
constexpr int kSolveAB = 32 * (kSolveA + kSolveB);
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int R, int GB, int CH, int NS>
__global__ void __launch_bounds__(kSolveThreads, 1)
    solve_step_kernel(SolveStepArgs g, const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW) {
  using Cfg = SolveCfg<R, GB, CH>;
  constexpr int P = Cfg::P, PX = Cfg::P, PW = Cfg::PW, NB = Cfg::NB, NSUB = Cfg::NSUB, RT = R / 8;
  constexpr int T1 = (NB * GB + kSolveA - 1) / kSolveA;  // phase-1 items per A warp
  constexpr int T2 = (RT * GB + kSolveB - 1) / kSolveB;  // phase-2 tiles per B warp
  constexpr uint32_t PANEL_BYTES = (uint32_t)Cfg::PANEL * sizeof(double);
  constexpr uint32_t XW_BYTES = (uint32_t)(Cfg::XT + Cfg::WT) * sizeof(double);
  extern __shared__ __align__(1024) double sms[];
  double* ring = sms;                   // NS x [Y panel | V panel | x tile | w' tile]
  double* xs0 = sms + NS * Cfg::STAGE;  // 2 x [GB * 8 columns][PX]: the updated x of a chunk
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const bool want_w = g.out != nullptr;
  const int cpu = g.unit_rows / CH;  // TMA chunks per unit
  const int nmine = g.nitems > (int64_t)blockIdx.x ? (int)((g.nitems - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  const int total = nmine * cpu;

  if (t == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], want_w ? kSolveA + kSolveB : kSolveA);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // chunk stream of this CTA: items blockIdx.x, + gridDim.x, ...; cpu chunks each
  struct Pos {
    int64_t item, unit;
    int cu, gb;
  };
  auto first = [&]() {
    Pos p{(int64_t)blockIdx.x, 0, 0, 0};
    p.unit = p.item / g.ncg;
    p.gb = (int)(p.item - p.unit * g.ncg) * GB;
    return p;
  };
  auto advance = [&](Pos& p) {
    if (++p.cu == cpu) {
      p.cu = 0;
      p.item += gridDim.x;
      p.unit = p.item / g.ncg;
      p.gb = (int)(p.item - p.unit * g.ncg) * GB;
    }
  };

  if (warp == kSolveA + kSolveB) {  // ---- producer ----
    if (lane == 0) {
      Pos p = first();
      for (int f = 0, s = 0, use = 0; f < total; ++f) {
        if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
        double* Ys = ring + s * Cfg::STAGE;
        const int row = (int)(p.unit * g.unit_rows) + p.cu * CH;
        const int c = row / g.n_c, col0 = p.gb * 8;
        mbar_expect_tx(&full[s], (want_w ? 2 : 1) * PANEL_BYTES + XW_BYTES);
        tma_load_2d(Ys, &tmY, row, 0, &full[s]);
        if (want_w) tma_load_2d(Ys + Cfg::PANEL, &tmV, row, 0, &full[s]);
        tma_load_2d(Ys + 2 * Cfg::PANEL, &tmX, row, col0, &full[s]);
        tma_load_2d(Ys + 2 * Cfg::PANEL + Cfg::XT, &tmW, (c & 1) * R, (c >> 1) * g.ncols + col0, &full[s]);
        advance(p);
        if (++s == NS) s = 0, ++use;
      }
    }
    return;
  }

  if (warp < kSolveA) {  // ---- A: x^T += (-w'^T) Y^T, one (band, group) tile pair per item ----
    Pos p = first();
    for (int f = 0, s = 0, use = 0; f < total; ++f) {
      const int64_t row0 = p.unit * g.unit_rows + (int64_t)p.cu * CH;
      double* xb = xs0 + (f & 1) * (GB * 8 * PX);
      mbar_wait(&full[s], (uint32_t)(use & 1));
      if (want_w && f >= 2) nbar_sync(3 + (f & 1), kSolveAB);  // B is done with this x buffer (use f - 2)
      const double* Ys = ring + s * Cfg::STAGE;
      const double* Xs = Ys + 2 * Cfg::PANEL;
      const double* Ws = Xs + Cfg::XT;
#pragma unroll
      for (int k = 0; k < T1; ++k) {
        const int e = warp + kSolveA * k;
        if (e < NB * GB) {
          const int band = e % NB, q = e / NB;
          const int col = (p.gb + q) * 8 + ar;
          double acc[2][2];
          {
            const double* xi = Xs + (q * 8 + ar) * PX + 16 * band + 4 * ac;
            const double2 x01 = *reinterpret_cast<const double2*>(xi);
            const double2 x23 = *reinterpret_cast<const double2*>(xi + 2);
            acc[0][0] = x01.x, acc[1][0] = x01.y, acc[0][1] = x23.x, acc[1][1] = x23.y;
          }
          const double* wc = Ws + (q * 8 + ar) * PW + 2 * ac;
#pragma unroll
          for (int kt = 0; kt < R / 8; ++kt) {
            const double2 w2 = *reinterpret_cast<const double2*>(wc + 8 * kt);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const double a = -(u ? w2.y : w2.x);
              const double2 b2 = *reinterpret_cast<const double2*>(Ys + (8 * kt + 2 * ac + u) * P + 2 * ar + 16 * band);
              dmma_8x8x4(acc[0][0], acc[0][1], a, b2.x);
              dmma_8x8x4(acc[1][0], acc[1][1], a, b2.y);
            }
          }
          if (col < g.ncols)
            stg_x4(g.X + row0 + 16 * band + (int64_t)col * g.ldx + 4 * ac, acc[0][0], acc[1][0], acc[0][1], acc[1][1]);
          if (want_w) {
            double* xw = xb + (q * 8 + ar) * PX + 16 * band + 4 * ac;
            *reinterpret_cast<double2*>(xw) = make_double2(acc[0][0], acc[1][0]);
            *reinterpret_cast<double2*>(xw + 2) = make_double2(acc[0][1], acc[1][1]);
          }
        }
      }
      __syncwarp();
      if (want_w) nbar_arrive(1 + (f & 1), kSolveAB);  // x tile of chunk f ready for B
      if (lane == 0) mbar_arrive(&empty[s]);
      advance(p);
      if (++s == NS) s = 0, ++use;
    }
    return;
  }

  if (!want_w) return;
  // ---- B: the chunk's w partial, one (8-rank tile, group) chain per item, running unit sums ----
  const int wb = warp - kSolveA;
  double S[T2][2], pp[T2][2];
#pragma unroll
  for (int k = 0; k < T2; ++k) S[k][0] = S[k][1] = pp[k][0] = pp[k][1] = 0.0;
  Pos p = first();
  for (int f = 0, s = 0, use = 0; f < total; ++f) {
    const int sub = p.cu % NSUB;  // TMA chunk within the canonical 64-row chunk
    const double* xb = xs0 + (f & 1) * (GB * 8 * PX);
    mbar_wait(&full[s], (uint32_t)(use & 1));
    nbar_sync(1 + (f & 1), kSolveAB);
    const double* Vs = ring + s * Cfg::STAGE + Cfg::PANEL;
#pragma unroll
    for (int k = 0; k < T2; ++k) {
      const int tt = wb + kSolveB * k;
      if (tt < RT * GB) {
        const int jr = tt % RT, q = tt / RT;
        if (sub == 0) pp[k][0] = pp[k][1] = 0.0;
        const double* xr = xb + (q * 8 + ar) * PX + 4 * ac;
        const double* vr = Vs + (8 * jr + ar) * P + 4 * ac;
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double2 a2 = *reinterpret_cast<const double2*>(xr + 16 * i + 2 * h);
            const double2 v2 = *reinterpret_cast<const double2*>(vr + 16 * i + 2 * h);
            dmma_8x8x4(pp[k][0], pp[k][1], a2.x, v2.x);
            dmma_8x8x4(pp[k][0], pp[k][1], a2.y, v2.y);
          }
        if (sub == NSUB - 1) S[k][0] += pp[k][0], S[k][1] += pp[k][1];
      }
    }
    __syncwarp();
    nbar_arrive(3 + (f & 1), kSolveAB);
    if (lane == 0) mbar_arrive(&empty[s]);
    if (p.cu == cpu - 1) {  // unit complete: its w (or partial) out, running sums reset
#pragma unroll
      for (int k = 0; k < T2; ++k) {
        const int tt = wb + kSolveB * k;
        if (tt < RT * GB) {
          const int jr = tt % RT, q = tt / RT;
          const int col = (p.gb + q) * 8 + ar;
          if (col < g.ncols) {
            double* o;
            if (g.partial) {
              o = g.out + p.unit * R * g.ncols + 8 * jr + 2 * ac + (int64_t)col * R;
            } else {
              const int64_t qn = p.unit * g.unit_rows / g.node_rows;
              o = g.out + (qn >> 1) * g.tw_stride + (qn & 1) * R + 8 * jr + 2 * ac + (int64_t)col * 2 * R;
            }
            *reinterpret_cast<double2*>(o) = make_double2(S[k][0], S[k][1]);
          }
          S[k][0] = S[k][1] = 0.0;
        }
      }
    }
    advance(p);
    if (++s == NS) s = 0, ++use;
  }
}

template <int R, int GB, int CH, int NS>
static hodlr_status launch_solve_step(const SolveStepArgs& g, const double* Y, const double* V, int64_t n, int64_t lda,
                                      int64_t wcols, int sms, cudaStream_t st) {
  using Cfg = SolveCfg<R, GB, CH>;
  constexpr size_t smem = ((size_t)NS * Cfg::STAGE + (size_t)2 * GB * 8 * Cfg::P) * sizeof(double);
  static_assert(smem <= 227 * 1024, "solve step shared memory");
  CUtensorMap ty, tv, tx, tw;
  if (!panel_map_f64(&ty, Y, n, R, lda, Cfg::P)) return HODLR_ERR_ARG;
  if (V != nullptr) {
    if (!panel_map_f64(&tv, V, n, R, lda, Cfg::P)) return HODLR_ERR_ARG;
  } else {
    tv = ty;
  }
  // x: n x ncols (ld ldx), box (CH + 2) x 8 GB; w': 2R x (ncols * parents) (ld 2R), box (R + 8) x 8 GB
  if (!tensor_map_f64(&tx, g.X, n, g.ncols, g.ldx, Cfg::P, 8 * GB)) return HODLR_ERR_ARG;
  if (!tensor_map_f64(&tw, g.W, 2 * R, wcols, 2 * R, Cfg::PW, 8 * GB)) return HODLR_ERR_ARG;
  smem_attr(solve_step_kernel<R, GB, CH, NS>, (int)smem);
  const int64_t grid = std::min<int64_t>(g.nitems, sms);
  solve_step_kernel<R, GB, CH, NS><<<(unsigned)grid, kSolveThreads, smem, st>>>(g, ty, tv, tx, tw);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// as many stages as fit in ~200 KB of shared memory (R = 64: 32-row chunks)
template <int R, int GB, int CH>
constexpr int solve_stages() {
  using Cfg = SolveCfg<R, GB, CH>;
  const int budget = 200 * 1024 / 8 - 2 * GB * 8 * Cfg::P;
  const int ns = budget / Cfg::STAGE;
  return ns > 8 ? 8 : ns;
}

template <int R, int GB>
static hodlr_status run_solve_step(const SolveStepArgs& g, const double* Y, const double* V, int64_t n, int64_t lda,
                                   int64_t wcols, int sms, cudaStream_t st) {
  constexpr int CH = R >= 64 ? 32 : 64;
  return launch_solve_step<R, GB, CH, solve_stages<R, GB, CH>()>(g, Y, V, n, lda, wcols, sms, st);
}

template <int R>
static hodlr_status run_solve_step_r(const SolveStepArgs& g, int gbs, const double* Y, const double* V, int64_t n,
                                     int64_t lda, int64_t wcols, int sms, cudaStream_t st) {
  switch (gbs) {
    case 1: return run_solve_step<R, 1>(g, Y, V, n, lda, wcols, sms, st);
    case 2: return run_solve_step<R, 2>(g, Y, V, n, lda, wcols, sms, st);
    case 3: return run_solve_step<R, 3>(g, Y, V, n, lda, wcols, sms, st);
    default: return run_solve_step<R, 4>(g, Y, V, n, lda, wcols, sms, st);
  }
}

// Solve level step over n rows of X on the TMA-fed kernel.  part receives the
// per-unit partials when a node spans several 512-row units (the caller's
// level_reduce_kernel then combines them); ERR_ARG for unsupported shapes.
hodlr_status solve_step_f64(int r, int64_t n, int64_t n_c, int64_t node_rows, double* X, int64_t ldx, const double* Y,
                            const double* V, int64_t lda, const double* W, int64_t wstride, int nrhs, double* TW,
                            int64_t tw_stride, double* part, size_t part_bytes, int sms, bool* used_partial,
                            cudaStream_t st) {
  *used_partial = false;
  if (nrhs == 0) return HODLR_OK;
  if (r != 16 && r != 32 && r != 64) return HODLR_ERR_ARG;
  if (n % 64 || node_rows % 64 || (n_c % 64 && n_c < n) || n > 2147483647LL - 128) return HODLR_ERR_ARG;
  if ((ldx & 3) || (reinterpret_cast<uintptr_t>(X) & 31) || (reinterpret_cast<uintptr_t>(W) & 15) || (wstride & 1) ||
      (lda & 1))
    return HODLR_ERR_ARG;
  const int64_t unit = std::min<int64_t>(node_rows, 512);
  if (n % unit || (node_rows > unit && node_rows % unit)) return HODLR_ERR_ARG;
  const bool partial = node_rows > unit && V != nullptr;
  // up to 24 RHS (rank <= 32) / 32 RHS (rank 64) in one pass; more RHS: the
  // shared-panel kernel, whose warps own column groups (x not staged), is faster
  const int G = (nrhs + 7) / 8;
  if (G > (r >= 64 ? 4 : 3)) return HODLR_ERR_ARG;
  const int gbs = G;
  const int ncg = (G + gbs - 1) / gbs;
  const int64_t units = n / unit;
  if (partial && (size_t)units * r * nrhs * sizeof(double) > part_bytes) return HODLR_ERR_ARG;
  SolveStepArgs g{X, ldx, W, wstride, V ? (partial ? part : TW) : nullptr, tw_stride, partial ? 1 : 0,
                  (int)std::min<int64_t>(n_c, 2147483647LL), (int)unit, node_rows, nrhs, ncg, units * ncg};
  if (wstride != (int64_t)2 * r * nrhs) return HODLR_ERR_ARG;  // w' parents contiguous: one 2-D tensor
  const int64_t wcols = (int64_t)nrhs * std::max<int64_t>(1, n / std::min<int64_t>(2 * n_c, n));
  *used_partial = partial;
  switch (r) {
    case 16: return run_solve_step_r<16>(g, gbs, Y, V, n, lda, wcols, sms, st);
    case 32: return run_solve_step_r<32>(g, gbs, Y, V, n, lda, wcols, sms, st);
    default: return run_solve_step_r<64>(g, gbs, Y, V, n, lda, wcols, sms, st);
  }
}

}  // namespace hodlr
