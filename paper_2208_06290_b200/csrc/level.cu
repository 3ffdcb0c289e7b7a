// Fused level step of the factorization (Alg. 3 lines 9-10 of level l
// fused with lines 5-6 of level l-1) and of the solve (Alg. 4 lines 7 / 5).
//
// For every child c at level l+1 (n_c rows, parent p = c/2):
//     C(I_c, :) -= Y_c^{l+1} W'_c                         (update, W' = half of K_p^-1 W_p)
// and, with the freshly updated rows still in shared memory,
//     TW_q(:, :) += V_q^{(l) T} C(I_q, :)                  (next level's [W|T], q = node at level l)
//
// C is the Y slab columns [0, r l) in the factorization (W' has r l columns) or
// the solution block x (nrhs columns) in the solve.  One CTA owns a segment of
// consecutive rows inside one level-l node q and walks (column tile, 64-row
// sub-tile) pairs through a 2-stage cp.async pipeline; each 64 x BN update and
// each r x BN reduction is a DMMA (FP64 tensor core) tile.  Y is therefore read
// and written once per level, and V^T C never re-reads C from HBM.  Segments
// shorter than the node write partial sums that a fixed-order reduction kernel
// adds (deterministic).
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace hodlr {

// factorization level steps with <= 4 column groups per CTA: two warps per group
// (row halves), so all 8 warps work (level 1 at cfg2: level phase 14.36 -> 14.31
// ms same-box; letting the schedule prefer <= 4 groups per CTA at the other
// levels was slower, 14.96 ms -- profiles/r02_ab_rowsplit.txt)
#ifndef HODLR_LEVEL_ROWSPLIT
#define HODLR_LEVEL_ROWSPLIT 1
#endif
constexpr bool kLevelRowSplit = HODLR_LEVEL_ROWSPLIT;

struct LevelArgs {
  double* C;  // rows [0, n) of the updated block, column-major
  int64_t ldc;
  const double* A1;  // Y^{l+1} panel: A1[row + k*lda], k < r
  const double* V;   // V^{(l)} panel: V[row + k*lda], k < r  (may be null: no TW output)
  int64_t lda;
  const double* W;  // W_p (2r x ncols, ld 2r) at W + p * wstride
  int64_t wstride;
  double* TW;       // final: paired layout; partial: [seg][r x ncols] ld r
  int64_t tw_stride;  // final: per next-parent stride (2r * ncols)
  int partial;
  int n_c;       // rows per child at level l+1 (selects the W' half)
  int seg_rows;  // rows per CTA segment (multiple of 64, divides node_rows)
  int64_t node_rows;  // rows of one [W|T] output node (2 n_c, or a rank's share)
  int ncols;
  int ncg;  // column-tile groups per segment (factorization kernel; grid = segments x ncg)
  int tpc;  // 64-column tiles per group
};

constexpr int64_t kMaxSegs = 1184;
struct FactSched {
  int64_t seg;
  int ncg, tpc;
};

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int device_sm_count() { return sm_count(); }

constexpr int LV_THREADS = 512;  // 16 warps: two per scheduler slot of each SMSP pair

template <int R, int BN>
struct LevelCfg {
  static constexpr int BM = 64;
  static constexpr int P = BM + 4;  // pitch of row-contiguous tiles
  static constexpr int PW = R + 4;  // pitch of W' tile (k contiguous)
  static constexpr int C_SZ = BN * P;
  static constexpr int A_SZ = R * P;
  static constexpr int W_SZ = BN * PW;
  static constexpr int STAGE = C_SZ + 2 * A_SZ + W_SZ;
  // [W|T] GEMM: BN/8 n-tiles x TK k-splits = 16 warps; partials combined in smem
  static constexpr int TWN = BN / 8;
  static constexpr int TK = 16 / TWN;
  static constexpr int RED = TK * R * BN;
  static constexpr size_t SMEM = ((size_t)2 * STAGE + RED) * sizeof(double);
};

template <int R, int BN>
__global__ void __launch_bounds__(LV_THREADS) level_update_kernel(LevelArgs g) {
  using Cfg = LevelCfg<R, BN>;
  constexpr int NT = LV_THREADS, NWARP = NT / 32;
  constexpr int BM = Cfg::BM, P = Cfg::P, PW = Cfg::PW;
  // update GEMM: 64 x BN output
  constexpr int UWN = (BN >= 64) ? 4 : 1;      // warps along N
  constexpr int UWM = (BN >= 64) ? 4 : 8;      // warps along M (BN = 8: 8 active warps)
  constexpr int UTM = BM / UWM, UTN = BN / UWN;
  constexpr int UMI = UTM / 8, UNI = UTN / 8;
  // [W|T] GEMM: R x BN, each warp owns one 8-column n-tile and one k-range
  constexpr int TWN = Cfg::TWN, TK = Cfg::TK, KR = BM / TK;
  constexpr int TMI = R / 8;
  static_assert(UMI >= 1 && UNI >= 1 && KR % 4 == 0, "tile config");

  extern __shared__ __align__(16) double sm[];
  double* red = sm + 2 * Cfg::STAGE;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int64_t seg0 = (int64_t)blockIdx.x * g.seg_rows;
  const int nsub = g.seg_rows / BM;
  const int ntile = (g.ncols + BN - 1) / BN;
  const int niter = nsub * ntile;
  const bool want_tw = g.V != nullptr;

  auto stage_ptr = [&](int s) { return sm + s * Cfg::STAGE; };
  // the A1 / V / W' panels are re-read for every column tile: keep them in L2;
  // the C stream is touched once per level
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();

  auto load = [&](int it, int s) {
    const int ct = it / nsub, st = it % nsub;
    const int64_t row0 = seg0 + (int64_t)st * BM;
    const int c = (int)(row0 / g.n_c);
    const int n0 = ct * BN;
    double* Cs = stage_ptr(s);
    double* As = Cs + Cfg::C_SZ;
    double* Vs = As + Cfg::A_SZ;
    double* Ws = Vs + Cfg::A_SZ;
    for (int idx = t; idx < BN * (BM / 2); idx += NT) {
      const int n = idx / (BM / 2), m = (idx % (BM / 2)) * 2;
      const bool ok = n0 + n < g.ncols;
      cp_async_16_pol(Cs + n * P + m, ok ? g.C + row0 + m + (int64_t)(n0 + n) * g.ldc : g.C, ok ? 16 : 0, stream);
    }
    for (int idx = t; idx < R * (BM / 2); idx += NT) {
      const int k = idx / (BM / 2), m = (idx % (BM / 2)) * 2;
      cp_async_16_pol(As + k * P + m, g.A1 + row0 + m + (int64_t)k * g.lda, 16, keep);
      if (want_tw) cp_async_16_pol(Vs + k * P + m, g.V + row0 + m + (int64_t)k * g.lda, 16, keep);
    }
    const double* Wp = g.W + (int64_t)(c >> 1) * g.wstride + (c & 1) * R;
    for (int idx = t; idx < BN * (R / 2); idx += NT) {
      const int n = idx / (R / 2), k = (idx % (R / 2)) * 2;
      const bool ok = n0 + n < g.ncols;
      cp_async_16_pol(Ws + n * PW + k, ok ? Wp + k + (int64_t)(n0 + n) * (2 * R) : g.W, ok ? 16 : 0, keep);
    }
  };

  const int tn = warp % TWN, tk = warp / TWN;  // [W|T] role of this warp
  double tw[TMI][2];
  if (niter > 0) load(0, 0);
  cp_async_commit();
  for (int it = 0; it < niter; ++it) {
    const int s = it & 1;
    const int ct = it / nsub, st = it % nsub;
    if (it + 1 < niter) load(it + 1, s ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double* Cs = stage_ptr(s);
    const double* As = Cs + Cfg::C_SZ;
    const double* Vs = As + Cfg::A_SZ;
    const double* Ws = Vs + Cfg::A_SZ;
    if (st == 0) {
#pragma unroll
      for (int i = 0; i < TMI; ++i) tw[i][0] = tw[i][1] = 0.0;
    }
    // ---- update: upd = A1 W' (rounded product), C = C - upd ----
    if (warp < UWM * UWN) {
      const int wm = warp / UWN, wn = warp % UWN;
      double acc[UMI][UNI][2];
#pragma unroll
      for (int i = 0; i < UMI; ++i)
#pragma unroll
        for (int j = 0; j < UNI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < R; k0 += 4) {
        double af[UMI], bf[UNI];
#pragma unroll
        for (int i = 0; i < UMI; ++i) af[i] = As[(k0 + ac) * P + wm * UTM + i * 8 + ar];
#pragma unroll
        for (int j = 0; j < UNI; ++j) bf[j] = Ws[(wn * UTN + j * 8 + ar) * PW + k0 + ac];
#pragma unroll
        for (int i = 0; i < UMI; ++i)
#pragma unroll
          for (int j = 0; j < UNI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
#pragma unroll
      for (int i = 0; i < UMI; ++i)
#pragma unroll
        for (int j = 0; j < UNI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = wm * UTM + i * 8 + ar, n = wn * UTN + j * 8 + ac * 2 + h;
            Cs[n * P + m] = __dsub_rn(Cs[n * P + m], acc[i][j][h]);
          }
    }
    __syncthreads();
    // ---- store the updated tile (coalesced 16B) ----
    {
      const int64_t row0 = seg0 + (int64_t)st * BM;
      const int n0 = ct * BN;
      for (int idx = t; idx < BN * (BM / 2); idx += NT) {
        const int n = idx / (BM / 2), m = (idx % (BM / 2)) * 2;
        if (n0 + n < g.ncols) {
          double2 v = make_double2(Cs[n * P + m], Cs[n * P + m + 1]);
          *reinterpret_cast<double2*>(g.C + row0 + m + (int64_t)(n0 + n) * g.ldc) = v;
        }
      }
    }
    // ---- next level's [W|T]: tw += V^T C_new over this warp's k-range ----
    if (want_tw) {
#pragma unroll
      for (int k0 = tk * KR; k0 < (tk + 1) * KR; k0 += 4) {
        double af[TMI];
#pragma unroll
        for (int i = 0; i < TMI; ++i) af[i] = Vs[(i * 8 + ar) * P + k0 + ac];
        const double bf = Cs[(tn * 8 + ar) * P + k0 + ac];
#pragma unroll
        for (int i = 0; i < TMI; ++i) dmma_8x8x4(tw[i][0], tw[i][1], af[i], bf);
      }
      if (st == nsub - 1) {
        // combine the TK k-split partials in a fixed order, then write
#pragma unroll
        for (int i = 0; i < TMI; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) red[(tk * R + i * 8 + ar) * BN + tn * 8 + ac * 2 + h] = tw[i][h];
        __syncthreads();
        const int n0 = ct * BN;
        const int64_t q = seg0 / g.node_rows;  // level-l node of this segment
        double* out;
        int64_t ld;
        if (g.partial) {
          out = g.TW + (int64_t)blockIdx.x * R * g.ncols;
          ld = R;
        } else {
          out = g.TW + (q >> 1) * g.tw_stride + (q & 1) * R;
          ld = 2 * R;
        }
        for (int idx = t; idx < R * BN; idx += NT) {
          const int m = idx % R, n = idx / R;
          double v = red[m * BN + n];
#pragma unroll
          for (int kk = 1; kk < TK; ++kk) v += red[(kk * R + m) * BN + n];
          if (n0 + n < g.ncols) out[m + (int64_t)(n0 + n) * ld] = v;
        }
      }
    }
    __syncthreads();
  }
}

// TW_q = sum over the q's segments of the partials, fixed order; paired output.
// Few segments: one thread per output, sequential.  Many segments (top
// levels): one warp per output, lane l sums segments l, l+32, ... in order,
// then a fixed xor-butterfly.  The order depends only on the segment count.
__global__ void level_reduce_kernel(const double* part, double* TW, int R, int ncols, int segs_per_node, int nnodes,
                                    int64_t tw_stride) {
  const int64_t per = (int64_t)R * ncols;
  const int64_t total = per * nnodes;
  if (segs_per_node <= 32) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t q = e / per, mn = e % per;
      const int m = (int)(mn % R), n = (int)(mn / R);
      double s = 0.0;
      for (int k = 0; k < segs_per_node; ++k) s += part[(q * segs_per_node + k) * per + mn];
      TW[(q >> 1) * tw_stride + (q & 1) * R + m + (int64_t)n * 2 * R] = s;
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t e = blockIdx.x * wpb + (threadIdx.x >> 5); e < total; e += (int64_t)gridDim.x * wpb) {
    const int64_t q = e / per, mn = e % per;
    const int m = (int)(mn % R), n = (int)(mn / R);
    double s = 0.0;
    for (int k = lane; k < segs_per_node; k += 32) s += part[(q * segs_per_node + k) * per + mn];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) TW[(q >> 1) * tw_stride + (q & 1) * R + m + (int64_t)n * 2 * R] = s;
  }
}


// ---------------------------------------------------------------------------
// Column-group variant for the factorization (no per-tile CTA barrier).
// The CTA stages the A1 / V panels of a 64-row chunk (2-stage cp.async ring,
// one barrier per chunk); every warp then streams its own column groups of 8
// through the chunk, transposed so that no operand changes lanes:
//
//   C^T  += (-W'^T) A1^T   A: W' column entries (registers, from L2),
//                          B: A1 panel (LDS.128 row pairs)
//   TW^T +=  C^T V         A: the updated C^T accumulators themselves
//
// An m8n8k4 accumulator row of lane (ar, ac) holds n = 2ac + {0,1}; rows are
// mapped as sigma(jn, n) = 16 (jn/2) + 2n + (jn%2), so a lane's 8 accumulator
// values of a 16-row band are 4 consecutive rows of one column (one 32-byte
// load / store per band) and every panel read is a conflict-free LDS.128.
// [W|T] partial sums stay in registers (GPW groups per warp) for the whole
// segment.
// ---------------------------------------------------------------------------
template <int R, bool SOLVE = false>
struct Level4Cfg {
  // rows per chunk (the warp's C^T tile height); the solve mode always uses the
  // streaming solve kernel's 64-row chunks (identical chunk partials)
  static constexpr int CH = (R >= 64 && !SOLVE) ? 32 : 64;
  static constexpr int NI = CH / 16;            // 16-row bands per chunk
  static constexpr int P = CH + 2;              // [rank][row] pitch: 2P = 4 (mod 16) doubles
  static constexpr int PANEL = R * P;
  static constexpr int STAGE = 2 * PANEL;
  static constexpr size_t SMEM = (size_t)2 * STAGE * sizeof(double);
};

__device__ __forceinline__ void ldg_v4(const double* p, double& x, double& y, double& z, double& w) {
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];\n"
               : "=d"(x), "=d"(y), "=d"(z), "=d"(w)
               : "l"(p));
}
__device__ __forceinline__ void stg_v4(double* p, double x, double y, double z, double w) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(w)
               : "memory");
}

// SOLVE: the multi-RHS solve step (columns = right-hand sides, ragged last
// group masked) with the solve kernel's reduction order -- every 64-row
// chunk's [W|T] contribution is a DMMA chain from zero, added to the running
// sum in row order -- so the result is bit-identical to solve_level_kernel.
template <int R, int GPW, bool LATE, bool SOLVE = false>
__global__ void __launch_bounds__(256, 2) level_update4_kernel(LevelArgs g) {
  using Cfg = Level4Cfg<R, SOLVE>;
  constexpr int CH = Cfg::CH, P = Cfg::P, RT = R / 8, NI = Cfg::NI;
  extern __shared__ __align__(16) double sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int seg = blockIdx.x / g.ncg, cg = blockIdx.x % g.ncg;
  const int64_t seg0 = (int64_t)seg * g.seg_rows;
  const int nch = g.seg_rows / CH;
  const int G = SOLVE ? (g.ncols + 7) >> 3 : g.ncols >> 3;
  const int gb = cg * g.tpc, ge = min(G, gb + g.tpc);

  auto stage = [&](int ch, int s) {
    double* As = sm + s * Cfg::STAGE;
    double* Vs = As + Cfg::PANEL;
    const double* a1 = g.A1 + seg0 + (int64_t)ch * CH;
    const double* v1 = (!SOLVE || g.V) ? g.V + seg0 + (int64_t)ch * CH : nullptr;
    static_assert((R * (CH / 2)) % 256 == 0, "panel split");
#pragma unroll
    for (int q = 0; q < R * (CH / 2) / 256; ++q) {
      const int idx = t + q * 256;
      const int k = idx / (CH / 2), m = (idx % (CH / 2)) * 2;
      cp_async_16(As + k * P + m, a1 + m + (int64_t)k * g.lda, 16);
      if (!SOLVE || g.V) cp_async_16(Vs + k * P + m, v1 + m + (int64_t)k * g.lda, 16);
    }
  };

  double tw[GPW][RT][2];
#pragma unroll
  for (int q = 0; q < GPW; ++q)
#pragma unroll
    for (int jr = 0; jr < RT; ++jr) tw[q][jr][0] = tw[q][jr][1] = 0.0;

  if (nch > 0) stage(0, 0);
  cp_async_commit();
  for (int ch = 0; ch < nch; ++ch) {
    const int s = ch & 1;
    if (ch + 1 < nch) stage(ch + 1, s ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* As = sm + s * Cfg::STAGE;
    const double* Vs = As + Cfg::PANEL;
    const int64_t row0 = seg0 + (int64_t)ch * CH;
    const int c = (int)(row0 / g.n_c);
    const double* Wp = g.W + (int64_t)(c >> 1) * g.wstride + (c & 1) * R;
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const int grp = gb + warp + 8 * q;
      if (grp < ge) {
        const int col = grp * 8 + ar;
        const bool cok = !SOLVE || col < g.ncols;
        double* cptr = g.C + row0 + (int64_t)(cok ? col : 0) * g.ldc + 4 * ac;
        double acc[2 * NI][2], cin[2 * NI][2];
        if constexpr (SOLVE) {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            if (cok) {
              ldg_v4(cptr + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
            } else {
              acc[2 * i][0] = acc[2 * i + 1][0] = acc[2 * i][1] = acc[2 * i + 1][1] = 0.0;
            }
          }
        } else if constexpr (LATE) {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            ldg_v4(cptr + 16 * i, cin[2 * i][0], cin[2 * i + 1][0], cin[2 * i][1], cin[2 * i + 1][1]);
            acc[2 * i][0] = acc[2 * i][1] = acc[2 * i + 1][0] = acc[2 * i + 1][1] = 0.0;
          }
        } else {
#pragma unroll
          for (int i = 0; i < NI; ++i) ldg_v4(cptr + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
        }
        // ---- C^T += (-W'^T) A1^T ----
        const double* wc = Wp + (int64_t)(cok ? col : 0) * (2 * R) + 2 * ac;
#pragma unroll
        for (int kt = 0; kt < R / 8; ++kt) {
          double2 w2 = make_double2(0.0, 0.0);
          if (cok) w2 = __ldg(reinterpret_cast<const double2*>(wc + 8 * kt));
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double a = -(u ? w2.y : w2.x);
            const double* ak = As + (8 * kt + 2 * ac + u) * P + 2 * ar;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const double2 b2 = *reinterpret_cast<const double2*>(ak + 16 * i);
              dmma_8x8x4(acc[2 * i][0], acc[2 * i][1], a, b2.x);
              dmma_8x8x4(acc[2 * i + 1][0], acc[2 * i + 1][1], a, b2.y);
            }
          }
        }
        if constexpr (LATE && !SOLVE) {  // C - (A1 W'): the load latency hides behind the update products
#pragma unroll
          for (int i = 0; i < 2 * NI; ++i) acc[i][0] = cin[i][0] + acc[i][0], acc[i][1] = cin[i][1] + acc[i][1];
        }
        if (cok) {
#pragma unroll
          for (int i = 0; i < NI; ++i)
            stg_v4(cptr + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
        }
        if (SOLVE && g.V == nullptr) continue;
        // ---- TW^T += C^T V ----
        if constexpr (SOLVE) {
          double p[RT][2];
#pragma unroll
          for (int jr = 0; jr < RT; ++jr) p[jr][0] = p[jr][1] = 0.0;
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int jr = 0; jr < RT; ++jr) {
                const double2 v2 = *reinterpret_cast<const double2*>(Vs + (8 * jr + ar) * P + 16 * i + 4 * ac + 2 * h);
                dmma_8x8x4(p[jr][0], p[jr][1], acc[2 * i][h], v2.x);
                dmma_8x8x4(p[jr][0], p[jr][1], acc[2 * i + 1][h], v2.y);
              }
#pragma unroll
          for (int jr = 0; jr < RT; ++jr) tw[q][jr][0] += p[jr][0], tw[q][jr][1] += p[jr][1];
        } else {
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int jr = 0; jr < RT; ++jr) {
                const double2 v2 = *reinterpret_cast<const double2*>(Vs + (8 * jr + ar) * P + 16 * i + 4 * ac + 2 * h);
                dmma_8x8x4(tw[q][jr][0], tw[q][jr][1], acc[2 * i][h], v2.x);
                dmma_8x8x4(tw[q][jr][0], tw[q][jr][1], acc[2 * i + 1][h], v2.y);
              }
        }
      }
    }
    __syncthreads();
  }
  // tw[q][jr][h] = TW^T[col][rank 8 jr + 2 ac + h]
  if (SOLVE && g.V == nullptr) return;
  const int64_t qn = seg0 / g.node_rows;
  double* out;
  int64_t ld;
  if (g.partial) {
    out = g.TW + (int64_t)seg * R * g.ncols;
    ld = R;
  } else {
    out = g.TW + (qn >> 1) * g.tw_stride + (qn & 1) * R;
    ld = 2 * R;
  }
#pragma unroll
  for (int q = 0; q < GPW; ++q) {
    const int grp = gb + warp + 8 * q;
    if (grp < ge && (!SOLVE || grp * 8 + ar < g.ncols)) {
      const int col = grp * 8 + ar;
#pragma unroll
      for (int jr = 0; jr < RT; ++jr)
        *reinterpret_cast<double2*>(out + 8 * jr + 2 * ac + (int64_t)col * ld) = make_double2(tw[q][jr][0], tw[q][jr][1]);
    }
  }
}

#ifndef LEVEL4_LATE
#define LEVEL4_LATE 1
#endif
constexpr bool LEVEL4_LATE_DEFAULT = LEVEL4_LATE;
// ---------------------------------------------------------------------------
// TMA-fed variant of level_update4_kernel (factorization mode): the A1 / V
// panels of each 64-row chunk arrive by two 2-D tensor copies
// (cp.async.bulk.tensor, box = (CH + 2) rows x R ranks, so the boxes land with
// the conflict-free pitch P = CH + 2 of the cp.async layout -- the 2 extra rows
// are read, or zero-filled past the slab end, into the padding) issued by one
// thread into a 3-stage ring; completion is an mbarrier transaction count
// ("full"), and stage reuse is an 8-warp arrival barrier ("empty"), so warps
// never wait on each other at a __syncthreads: a warp waits only for its
// chunk's bytes, and the issuing thread only for the warps still reading the
// stage it refills.  Arithmetic and per-column operation order are those of
// level_update4_kernel (bit-identical results).
// ---------------------------------------------------------------------------
// SOLVE: the multi-RHS solve step (columns = right-hand sides, ragged last
// group masked, V may be null at the last level) with the reduction order of
// solve_level_kernel (each 64-row chunk's [W|T] contribution a DMMA chain from
// zero, added to the running sum in row order) -- bit-identical to it.
template <int R, int GPW, bool LATE, bool SOLVE = false, int RS = 1, int NS = 3>
__global__ void __launch_bounds__(256, 2)
    level_update5_kernel(LevelArgs g, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV) {
  using Cfg = Level4Cfg<R, SOLVE>;
  constexpr int CH = Cfg::CH, P = Cfg::P, RT = R / 8;
  // RS = 2 (factorization, <= 4 column groups per CTA): warps w and w + 4 share
  // group w, each on half of the chunk's 16-row bands; their [W|T] partials
  // are added at the end (half 0 + half 1)
  static_assert(RS == 1 || (RS == 2 && !SOLVE && GPW == 1), "row split: factorization, one group per warp");
  constexpr int NI = Cfg::NI / RS;
  constexpr uint32_t PANEL_BYTES = (uint32_t)Cfg::PANEL * sizeof(double);  // = box bytes (P x R)
  extern __shared__ __align__(1024) double sm5[];  // TMA destinations: 128-byte aligned stages
  double* sm = sm5;
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int seg = blockIdx.x / g.ncg, cg = blockIdx.x % g.ncg;
  const int64_t seg0 = (int64_t)seg * g.seg_rows;
  const int nch = g.seg_rows / CH;
  const int G = SOLVE ? (g.ncols + 7) >> 3 : g.ncols >> 3;
  const int gb = cg * g.tpc, ge = min(G, gb + g.tpc);
  const bool want_tw = !SOLVE || g.V != nullptr;
  const int wg = RS == 1 ? warp : (warp & 3);    // group slot of this warp
  const int band0 = RS == 1 ? 0 : (warp >> 2) * NI;  // first 16-row band of this warp's half

  if (t == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int ch) {
    const int st = ch % NS;
    double* As = sm + st * Cfg::STAGE;
    mbar_expect_tx(&full[st], (want_tw ? 2 : 1) * PANEL_BYTES);
    const int row = (int)(seg0 + (int64_t)ch * CH);
    tma_load_2d(As, &tmA, row, 0, &full[st]);
    if (want_tw) tma_load_2d(As + Cfg::PANEL, &tmV, row, 0, &full[st]);
  };
  if (t == 0)
    for (int c = 0; c < NS - 1 && c < nch; ++c) issue(c);

  double tw[GPW][RT][2];
#pragma unroll
  for (int q = 0; q < GPW; ++q)
#pragma unroll
    for (int jr = 0; jr < RT; ++jr) tw[q][jr][0] = tw[q][jr][1] = 0.0;

  for (int ch = 0; ch < nch; ++ch) {
    const int s = ch % NS;
    mbar_wait(&full[s], (uint32_t)((ch / NS) & 1));
    const double* As = sm + s * Cfg::STAGE;
    const double* Vs = As + Cfg::PANEL;
    const int64_t row0 = seg0 + (int64_t)ch * CH;
    const int c = (int)(row0 / g.n_c);
    const double* Wp = g.W + (int64_t)(c >> 1) * g.wstride + (c & 1) * R;
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const int grp = gb + wg + 8 * q;
      if (grp < ge) {
        const int col = grp * 8 + ar;
        const bool cok = !SOLVE || col < g.ncols;
        double* cptr = g.C + row0 + 16 * band0 + (int64_t)(cok ? col : 0) * g.ldc + 4 * ac;
        double acc[2 * NI][2], cin[2 * NI][2];
        if constexpr (SOLVE) {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            if (cok) {
              ldg_v4(cptr + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
            } else {
              acc[2 * i][0] = acc[2 * i + 1][0] = acc[2 * i][1] = acc[2 * i + 1][1] = 0.0;
            }
          }
        } else if constexpr (LATE) {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            ldg_v4(cptr + 16 * i, cin[2 * i][0], cin[2 * i + 1][0], cin[2 * i][1], cin[2 * i + 1][1]);
            acc[2 * i][0] = acc[2 * i][1] = acc[2 * i + 1][0] = acc[2 * i + 1][1] = 0.0;
          }
        } else {
#pragma unroll
          for (int i = 0; i < NI; ++i) ldg_v4(cptr + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
        }
        const double* wc = Wp + (int64_t)(cok ? col : 0) * (2 * R) + 2 * ac;
#pragma unroll
        for (int kt = 0; kt < R / 8; ++kt) {
          double2 w2 = make_double2(0.0, 0.0);
          if (cok) w2 = __ldg(reinterpret_cast<const double2*>(wc + 8 * kt));
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double a = -(u ? w2.y : w2.x);
            const double* ak = As + (8 * kt + 2 * ac + u) * P + 2 * ar + 16 * band0;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const double2 b2 = *reinterpret_cast<const double2*>(ak + 16 * i);
              dmma_8x8x4(acc[2 * i][0], acc[2 * i][1], a, b2.x);
              dmma_8x8x4(acc[2 * i + 1][0], acc[2 * i + 1][1], a, b2.y);
            }
          }
        }
        if constexpr (LATE && !SOLVE) {
#pragma unroll
          for (int i = 0; i < 2 * NI; ++i) acc[i][0] = cin[i][0] + acc[i][0], acc[i][1] = cin[i][1] + acc[i][1];
        }
        if (cok) {
#pragma unroll
          for (int i = 0; i < NI; ++i)
            stg_v4(cptr + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
        }
        if (!want_tw) continue;
        if constexpr (SOLVE) {
          double pp[RT][2];
#pragma unroll
          for (int jr = 0; jr < RT; ++jr) pp[jr][0] = pp[jr][1] = 0.0;
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int jr = 0; jr < RT; ++jr) {
                const double2 v2 = *reinterpret_cast<const double2*>(Vs + (8 * jr + ar) * P + 16 * (i + band0) + 4 * ac + 2 * h);
                dmma_8x8x4(pp[jr][0], pp[jr][1], acc[2 * i][h], v2.x);
                dmma_8x8x4(pp[jr][0], pp[jr][1], acc[2 * i + 1][h], v2.y);
              }
#pragma unroll
          for (int jr = 0; jr < RT; ++jr) tw[q][jr][0] += pp[jr][0], tw[q][jr][1] += pp[jr][1];
        } else {
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int jr = 0; jr < RT; ++jr) {
                const double2 v2 = *reinterpret_cast<const double2*>(Vs + (8 * jr + ar) * P + 16 * (i + band0) + 4 * ac + 2 * h);
                dmma_8x8x4(tw[q][jr][0], tw[q][jr][1], acc[2 * i][h], v2.x);
                dmma_8x8x4(tw[q][jr][0], tw[q][jr][1], acc[2 * i + 1][h], v2.y);
              }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill: chunk ch + NS - 1 into the stage chunk ch - 1 used (released by all 8 warps)
    if (t == 0 && ch + NS - 1 < nch) {
      const int c2 = ch + NS - 1;
      if (c2 >= NS) mbar_wait(&empty[c2 % NS], (uint32_t)((c2 / NS - 1) & 1));
      issue(c2);
    }
  }
  if (!want_tw) return;
  const int64_t qn = seg0 / g.node_rows;
  double* out;
  int64_t ld;
  if (g.partial) {
    out = g.TW + (int64_t)seg * R * g.ncols;
    ld = R;
  } else {
    out = g.TW + (qn >> 1) * g.tw_stride + (qn & 1) * R;
    ld = 2 * R;
  }
  if constexpr (RS == 2) {  // half 1 hands its partials to half 0 (the pipeline smem is free now)
    __syncthreads();
    double* xs = sm + (warp & 3) * (32 * RT * 2);
    if (warp >= 4) {
#pragma unroll
      for (int jr = 0; jr < RT; ++jr) {
        xs[(jr * 2) * 32 + lane] = tw[0][jr][0];
        xs[(jr * 2 + 1) * 32 + lane] = tw[0][jr][1];
      }
    }
    __syncthreads();
    if (warp >= 4) return;
#pragma unroll
    for (int jr = 0; jr < RT; ++jr) {
      tw[0][jr][0] += xs[(jr * 2) * 32 + lane];
      tw[0][jr][1] += xs[(jr * 2 + 1) * 32 + lane];
    }
  }
#pragma unroll
  for (int q = 0; q < GPW; ++q) {
    const int grp = gb + wg + 8 * q;
    if (grp < ge && (!SOLVE || grp * 8 + ar < g.ncols)) {
      const int col = grp * 8 + ar;
#pragma unroll
      for (int jr = 0; jr < RT; ++jr)
        *reinterpret_cast<double2*>(out + 8 * jr + 2 * ac + (int64_t)col * ld) = make_double2(tw[q][jr][0], tw[q][jr][1]);
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent factorization level step with C staged by TMA (round 2,
// level_update6): the same per-column arithmetic as level_update4_kernel (C
// loaded into the accumulators, C^T += (-W'^T) A1^T, then TW^T += C^T V), but
// every operand of a chunk -- the A1 and V panels AND the chunk's C tile
// (CH + 2 rows x the item's columns, one 2-D tensor copy) -- arrives through an
// NS-stage mbarrier ring, so no warp ever waits on a global load of C (ncu
// stall sampling of level_update4/5: 15-19 % of the samples on the C loads,
// 16 % on the per-chunk barrier).  The last warp done with a stage (a
// monotonic shared counter) refills it, so no warp waits for the others.
//
// Work item = (row segment, block of 16 column groups of 8; the last block of
// a segment holds the remainder, its C box the next power of two of groups);
// warp w owns group w of the item.  The CTA walks items blockIdx.x,
// + gridDim.x, ... as one flat stream of CH-row chunks.  Levels whose
// remainder block would leave too many warps idle keep level_update4/5
// (level6_efficient).  [W|T] partials stay in registers for the item and
// are written in the paired layout, or as per-segment partials that
// level_reduce_kernel sums in a fixed order.  Deterministic, no atomics on data.
// ---------------------------------------------------------------------------
constexpr int kL6Warps = 16;
template <int R>
struct Level6Cfg {
  static constexpr int CH = R >= 64 ? 32 : 64;  // rows per chunk
  static constexpr int NI = CH / 16;            // 16-row bands per chunk
  static constexpr int P = CH + 2;              // row pitch of every tile (LDS.128 conflict-free)
  static constexpr int GC = kL6Warps;           // column groups of a full item
  static constexpr int PANEL = R * P;
  static constexpr int CTILE = GC * 8 * P;
  static constexpr int STAGE = 2 * PANEL + CTILE;
  static constexpr int NS = (int)((227 * 1024 - 1024) / 8) / STAGE;
  static constexpr size_t SMEM = (size_t)NS * STAGE * sizeof(double);
  static constexpr int THREADS = kL6Warps * 32;
};

// item -> (segment, first group, groups, C box kind: 16 >> kind groups >= gi)
struct L6Item {
  int64_t seg;
  int gb, gi, kind;
};
__device__ __forceinline__ L6Item l6_item(int64_t item, int ncg, int G) {
  L6Item it;
  it.seg = item / ncg;
  it.gb = 16 * (int)(item - it.seg * ncg);
  it.gi = min(16, G - it.gb);
  it.kind = it.gi > 8 ? 0 : it.gi > 4 ? 1 : it.gi > 2 ? 2 : it.gi > 1 ? 3 : 4;
  return it;
}

struct L6Maps {
  CUtensorMap a, v, c[5];  // A1 / V panels; C boxes of 16 / 8 / 4 / 2 / 1 groups
};

// one chunk of one warp: group `slot` of the item (the lane's C column `col`)
template <int R>
__device__ __forceinline__ void level6_chunk(const LevelArgs& g, const double* As, const double* Vs, const double* Cs,
                                             const double2 (&wf)[R / 8], double (&tw)[R / 8][2], int64_t row0,
                                             int slot, int col, int ar, int ac) {
  constexpr int P = Level6Cfg<R>::P, RT = R / 8, NB = Level6Cfg<R>::NI, b0 = 0;
  double acc[2 * NB][2];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const double* ci = Cs + (slot * 8 + ar) * P + 16 * (b0 + i) + 4 * ac;
    const double2 x01 = *reinterpret_cast<const double2*>(ci);
    const double2 x23 = *reinterpret_cast<const double2*>(ci + 2);
    acc[2 * i][0] = x01.x, acc[2 * i + 1][0] = x01.y, acc[2 * i][1] = x23.x, acc[2 * i + 1][1] = x23.y;
  }
  // ---- C^T += (-W'^T) A1^T ----
#pragma unroll
  for (int kt = 0; kt < RT; ++kt)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double a = -(u ? wf[kt].y : wf[kt].x);
      const double* ak = As + (8 * kt + 2 * ac + u) * P + 2 * ar + 16 * b0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const double2 b2 = *reinterpret_cast<const double2*>(ak + 16 * i);
        dmma_8x8x4(acc[2 * i][0], acc[2 * i][1], a, b2.x);
        dmma_8x8x4(acc[2 * i + 1][0], acc[2 * i + 1][1], a, b2.y);
      }
    }
  double* cp = g.C + row0 + 16 * b0 + (int64_t)col * g.ldc + 4 * ac;
#pragma unroll
  for (int i = 0; i < NB; ++i) stg_v4(cp + 16 * i, acc[2 * i][0], acc[2 * i + 1][0], acc[2 * i][1], acc[2 * i + 1][1]);
  // ---- TW^T += C^T V: per (band, half) the RT first products, then the second ones ----
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 v2[RT];
#pragma unroll
      for (int jr = 0; jr < RT; ++jr)
        v2[jr] = *reinterpret_cast<const double2*>(Vs + (8 * jr + ar) * P + 16 * (b0 + i) + 4 * ac + 2 * h);
#pragma unroll
      for (int jr = 0; jr < RT; ++jr) dmma_8x8x4(tw[jr][0], tw[jr][1], acc[2 * i][h], v2[jr].x);
#pragma unroll
      for (int jr = 0; jr < RT; ++jr) dmma_8x8x4(tw[jr][0], tw[jr][1], acc[2 * i + 1][h], v2[jr].y);
    }
}

template <int R>
__global__ void __launch_bounds__(Level6Cfg<R>::THREADS, 1)
    level_update6_kernel(LevelArgs g, int64_t nitems, const __grid_constant__ L6Maps tm) {
  using Cfg = Level6Cfg<R>;
  constexpr int CH = Cfg::CH, NI = Cfg::NI, P = Cfg::P, NS = Cfg::NS, RT = R / 8, NW = kL6Warps;
  extern __shared__ __align__(1024) double sm6[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ int released[NS];  // warps done with the stage (monotonic; the NW-th of a use refills it)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int G = g.ncols >> 3;
  const int cps = g.seg_rows / CH;  // chunks per item
  const int64_t nmine = nitems > (int64_t)blockIdx.x ? (nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nmine * cps;

  auto issue = [&](int64_t item, int cu, int s) {
    const L6Item it = l6_item(item, g.ncg, G);
    const int row = (int)(it.seg * g.seg_rows + (int64_t)cu * CH);
    double* st = sm6 + (size_t)s * Cfg::STAGE;
    mbar_expect_tx(&full[s], (uint32_t)((2 * Cfg::PANEL + (16 >> it.kind) * 8 * P) * sizeof(double)));
    tma_load_2d(st, &tm.a, row, 0, &full[s]);
    tma_load_2d(st + Cfg::PANEL, &tm.v, row, 0, &full[s]);
    tma_load_2d(st + 2 * Cfg::PANEL, &tm.c[it.kind], row, it.gb * 8, &full[s]);
  };
  if (t == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      released[q] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int64_t item = blockIdx.x;
    int cu = 0;
    for (int f = 0; f < NS && f < total; ++f) {
      issue(item, cu, f);
      if (++cu == cps) cu = 0, item += gridDim.x;
    }
  }
  __syncthreads();

  double tw[RT][2];
#pragma unroll
  for (int jr = 0; jr < RT; ++jr) tw[jr][0] = tw[jr][1] = 0.0;
  // W' fragments of chunk f (loaded one chunk ahead, L1 / L2)
  double2 wf[RT];
  auto load_w = [&](double2 (&w)[RT], int64_t item, int cu) {
    const L6Item it = l6_item(item, g.ncg, G);
    const int64_t row0 = it.seg * g.seg_rows + (int64_t)cu * CH;
    const int c = (int)(row0 / g.n_c);
    const int col = (warp < it.gi ? it.gb + warp : 0) * 8 + ar;
    const double* wc = g.W + (int64_t)(c >> 1) * g.wstride + (c & 1) * R + (int64_t)col * (2 * R) + 2 * ac;
#pragma unroll
    for (int kt = 0; kt < RT; ++kt) w[kt] = __ldg(reinterpret_cast<const double2*>(wc + 8 * kt));
  };
  int64_t item = blockIdx.x;
  int cu = 0;
  if (total > 0) load_w(wf, item, cu);
  for (int64_t f = 0; f < total; ++f) {
    const int s = (int)(f % NS);
    const L6Item it = l6_item(item, g.ncg, G);
    const bool on = warp < it.gi;
    const int col = (it.gb + warp) * 8 + ar;
    const int64_t row0 = it.seg * g.seg_rows + (int64_t)cu * CH;
    int64_t item_n = item;
    int cu_n = cu + 1;
    if (cu_n == cps) cu_n = 0, item_n += gridDim.x;
    double2 wn[RT];
    if (f + 1 < total) load_w(wn, item_n, cu_n);
    mbar_wait(&full[s], (uint32_t)((f / NS) & 1));
    const double* As = sm6 + (size_t)s * Cfg::STAGE;
    const double* Vs = As + Cfg::PANEL;
    const double* Cs = Vs + Cfg::PANEL;
    if (on) level6_chunk<R>(g, As, Vs, Cs, wf, tw, row0, warp, col, ar, ac);
    __syncwarp();
    if (lane == 0) {  // the last warp done with stage s refills it with chunk f + NS
      __threadfence_block();
      const int old = atomicAdd(&released[s], 1);
      if ((old + 1) % NW == 0 && f + NS < total) {
        int64_t it2 = item;
        int cu2 = cu + NS;
        it2 += (int64_t)(cu2 / cps) * gridDim.x;
        cu2 %= cps;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(it2, cu2, s);
      }
    }
    if (cu_n == 0) {  // item done: [W|T] (or partial) out, running sums reset
      if (on) {
        double* out;
        int64_t ld;
        if (g.partial) {
          out = g.TW + it.seg * R * g.ncols;
          ld = R;
        } else {
          const int64_t qn = it.seg * g.seg_rows / g.node_rows;
          out = g.TW + (qn >> 1) * g.tw_stride + (qn & 1) * R;
          ld = 2 * R;
        }
#pragma unroll
        for (int jr = 0; jr < RT; ++jr)
          *reinterpret_cast<double2*>(out + 8 * jr + 2 * ac + (int64_t)col * ld) = make_double2(tw[jr][0], tw[jr][1]);
      }
#pragma unroll
      for (int jr = 0; jr < RT; ++jr) tw[jr][0] = tw[jr][1] = 0.0;
    }
    item = item_n;
    cu = cu_n;
#pragma unroll
    for (int kt = 0; kt < RT; ++kt) wf[kt] = wn[kt];
  }
}

// panel = rows [0, rows) x R columns of a column-major slab (ld lda); box = (CH + 2) x R
template <int R, bool SOLVE = false>
static bool panel_map(CUtensorMap* m, const double* base, int64_t rows, int64_t lda) {
  return panel_map_f64(m, base, rows, R, lda, Level4Cfg<R, SOLVE>::P);
}

template <int R, int GPW, int RS = 1, int NS = 3>
static hodlr_status launch_level5(const LevelArgs& g, int64_t nseg, int64_t rows, cudaStream_t st) {
  using Cfg = Level4Cfg<R, false>;
  constexpr bool LATE = GPW <= 2 && LEVEL4_LATE_DEFAULT;
  constexpr size_t smem = (size_t)NS * Cfg::STAGE * sizeof(double);
  CUtensorMap ta, tv;
  if (!panel_map<R>(&ta, g.A1, rows, g.lda) || !panel_map<R>(&tv, g.V, rows, g.lda)) return HODLR_ERR_ARG;
  smem_attr(level_update5_kernel<R, GPW, LATE, false, RS, NS>, (int)smem);
  level_update5_kernel<R, GPW, LATE, false, RS, NS><<<(unsigned)(nseg * g.ncg), 256, smem, st>>>(g, ta, tv);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template <int R>
static hodlr_status run_level4(const LevelArgs& g, int64_t nseg, cudaStream_t st);

// TMA feed for up to 2 column groups per warp (the upper levels: many chunks per
// CTA, barrier-bound with cp.async -- ncu launch list r02b: levels 10..1 8-12 %
// faster); 4+ groups per warp (deep levels, 2-8 chunks per CTA, 128 registers)
// stay on the cp.async kernel, which is 2-7 % faster there.
template <int R>
static hodlr_status run_level5(const LevelArgs& g, int64_t nseg, int64_t rows, cudaStream_t st) {
  const int gpw = (g.tpc + 7) / 8;
  if (g.tpc <= 4 && kLevelRowSplit) return launch_level5<R, 1, 2>(g, nseg, rows, st);  // 8 warps on <= 4 groups
  if (gpw <= 1) return launch_level5<R, 1>(g, nseg, rows, st);
  if (gpw <= 2) return launch_level5<R, 2>(g, nseg, rows, st);
  return run_level4<R>(g, nseg, st);
}

template <int R, int GPW>
static hodlr_status launch_level4(const LevelArgs& g, int64_t nseg, cudaStream_t st) {
  using Cfg = Level4Cfg<R>;
  constexpr bool LATE = GPW <= 2 && LEVEL4_LATE_DEFAULT;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(level_update4_kernel<R, GPW, LATE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    attr = true;
  }
  level_update4_kernel<R, GPW, LATE><<<(unsigned)(nseg * g.ncg), 256, Cfg::SMEM, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template <int R>
static hodlr_status run_level4(const LevelArgs& g, int64_t nseg, cudaStream_t st) {
  const int gpw = (g.tpc + 7) / 8;
  if (gpw <= 1) return launch_level4<R, 1>(g, nseg, st);
  if (gpw <= 2) return launch_level4<R, 2>(g, nseg, st);
  if constexpr (R <= 32) {
    if (gpw <= 4) return launch_level4<R, 4>(g, nseg, st);
  }
  if constexpr (R <= 16) {
    if (gpw <= 7) return launch_level4<R, 7>(g, nseg, st);
  }
  return HODLR_ERR_ARG;
}

// Schedule for level_update4: work item = (row segment, range of column
// groups of 8); at most maxg groups per CTA (the [W|T] partials live in registers).
static FactSched level4_schedule(int64_t n, int64_t node, int G, int sms, int maxg) {
  const int64_t slots = 2 * (int64_t)sms;
  FactSched best{node, 0, 0};
  double best_cost = 1e300;
  for (int64_t seg = node; seg >= 64; seg >>= 1) {
    const int64_t nseg = n / seg;
    if (seg < node && nseg > kMaxSegs) break;
    for (int ncg = 1; ncg <= G; ++ncg) {
      const int gpc = (G + ncg - 1) / ncg;
      if ((ncg - 1) * gpc >= G || gpc > maxg) continue;
      const double waves = (double)ceil_div(nseg * ncg, slots);
      double cost = waves * ((double)(seg / 64) * ((gpc + 7) / 8) + 0.5);
      if (seg < node) cost *= 1.05;
      if (cost < best_cost) {
        best_cost = cost;
        best = {seg, ncg, gpc};
      }
    }
    if (seg % 128) break;
  }
  return best;
}

// ---------------------------------------------------------------------------
// Solve level step (PAPER Alg. 4 l.7 fused with l.5 of the next level), any
// nrhs: x(I_c, :) -= Y_c^{l+1} w'_c, then the chunk's contribution to the next
// level's w = V^{(l)T} x.  One warp per 64-row chunk, 8 chunks (512 rows) per
// CTA; the HBM-bound panels (Y^{l+1}, V^{(l)}) are read straight from global
// memory into DMMA fragments (16-byte loads, no shared-memory staging), and
// the right-hand sides are swept in groups of 8 columns.  Every column is
// computed by the same instruction sequence whatever nrhs is, and the w
// reduction order is fixed (chunk partials summed in row order inside a CTA,
// CTA partials summed in row order by level_reduce_kernel), so a column of a
// multi-RHS solve is bit-identical to the single-vector solve.
// Fragment / row mapping as in level_update4_kernel.
// ---------------------------------------------------------------------------
constexpr int kSolveCtaRows = 512;

// NG = column groups per pass: two groups share every panel load (R <= 32);
// each group's DMMA sequence is exactly the single-group one.
template <int R, int NG>
__global__ void __launch_bounds__(256, 2) solve_level_kernel(LevelArgs g) {
  constexpr int RT = R / 8;
  __shared__ double ps[8][NG][R * 8];  // chunk partials of the current groups: [chunk][group][col_local * R + rank]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int64_t cta0 = (int64_t)blockIdx.x * g.seg_rows;
  const int nchunk = g.seg_rows / 64;
  const int64_t row0 = cta0 + 64 * warp;
  const bool has_chunk = warp < nchunk;
  const int c = has_chunk ? (int)(row0 / g.n_c) : 0;
  const double* Wp = g.W + (int64_t)(c >> 1) * g.wstride + (c & 1) * R;
  const bool want_w = g.V != nullptr;
  const int G = (g.ncols + 7) >> 3;
  for (int gp = 0; gp < G; gp += NG) {
    if (has_chunk) {
      double acc[NG][8][2];
      bool ok[NG];
      double* xp[NG];
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const int col = (gp + q) * 8 + ar;
        ok[q] = col < g.ncols;
        xp[q] = g.C + row0 + (int64_t)(ok[q] ? col : 0) * g.ldc + 4 * ac;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (ok[q]) {
            ldg_v4(xp[q] + 16 * i, acc[q][2 * i][0], acc[q][2 * i + 1][0], acc[q][2 * i][1], acc[q][2 * i + 1][1]);
          } else {
            acc[q][2 * i][0] = acc[q][2 * i + 1][0] = acc[q][2 * i][1] = acc[q][2 * i + 1][1] = 0.0;
          }
        }
      }
      const double* a1 = g.A1 + row0 + 2 * ar;
      // ---- x^T += (-w'^T) Y^T ----
#pragma unroll
      for (int kt = 0; kt < R / 8; ++kt) {
        double2 w2[NG];
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          w2[q] = make_double2(0.0, 0.0);
          if (ok[q])
            w2[q] = __ldg(reinterpret_cast<const double2*>(Wp + (int64_t)((gp + q) * 8 + ar) * (2 * R) + 2 * ac + 8 * kt));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double* ak = a1 + (int64_t)(8 * kt + 2 * ac + u) * g.lda;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double2 b2 = __ldcs(reinterpret_cast<const double2*>(ak + 16 * i));
#pragma unroll
            for (int q = 0; q < NG; ++q) {
              const double a = -(u ? w2[q].y : w2[q].x);
              dmma_8x8x4(acc[q][2 * i][0], acc[q][2 * i][1], a, b2.x);
              dmma_8x8x4(acc[q][2 * i + 1][0], acc[q][2 * i + 1][1], a, b2.y);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NG; ++q)
        if (ok[q]) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            stg_v4(xp[q] + 16 * i, acc[q][2 * i][0], acc[q][2 * i + 1][0], acc[q][2 * i][1], acc[q][2 * i + 1][1]);
        }
      if (want_w) {
        // ---- chunk partials p^T = x_new^T V (each from zero) ----
        double p[NG][RT][2];
#pragma unroll
        for (int q = 0; q < NG; ++q)
#pragma unroll
          for (int jr = 0; jr < RT; ++jr) p[q][jr][0] = p[q][jr][1] = 0.0;
        const double* vb = g.V + row0 + 4 * ac;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int jr = 0; jr < RT; ++jr) {
              const double2 v2 = __ldcs(reinterpret_cast<const double2*>(vb + (int64_t)(8 * jr + ar) * g.lda + 16 * i + 2 * h));
#pragma unroll
              for (int q = 0; q < NG; ++q) {
                dmma_8x8x4(p[q][jr][0], p[q][jr][1], acc[q][2 * i][h], v2.x);
                dmma_8x8x4(p[q][jr][0], p[q][jr][1], acc[q][2 * i + 1][h], v2.y);
              }
            }
#pragma unroll
        for (int q = 0; q < NG; ++q)
#pragma unroll
          for (int jr = 0; jr < RT; ++jr)
            *reinterpret_cast<double2*>(&ps[warp][q][ar * R + 8 * jr + 2 * ac]) = make_double2(p[q][jr][0], p[q][jr][1]);
      }
    }
    if (!want_w) continue;
    __syncthreads();
    // ---- fixed-order sums of the chunk partials per output node / CTA segment ----
    const int cpn = (int)(g.node_rows / 64 < nchunk ? g.node_rows / 64 : nchunk);  // chunks per output unit
    const int units = nchunk / cpn;
    for (int e = t; e < units * NG * 8 * R; e += 256) {
      const int uidx = e / (NG * 8 * R), rem = e % (NG * 8 * R);
      const int q = rem / (8 * R), mn = rem % (8 * R);
      const int cl = mn / R, rank = mn % R;
      const int colg = (gp + q) * 8 + cl;
      double sacc = 0.0;
      for (int k = 0; k < cpn; ++k) sacc += ps[uidx * cpn + k][q][mn];
      if (colg < g.ncols) {
        if (g.partial) {
          g.TW[(int64_t)blockIdx.x * R * g.ncols + rank + (int64_t)colg * R] = sacc;
        } else {
          const int64_t qn = (cta0 + (int64_t)uidx * cpn * 64) / g.node_rows;
          g.TW[(qn >> 1) * g.tw_stride + (qn & 1) * R + rank + (int64_t)colg * 2 * R] = sacc;
        }
      }
    }
    __syncthreads();
  }
}

// the shared-panel multi-RHS solve step fed by TMA (level_update5_kernel, solve mode)
#ifndef HODLR_SOLVE_TMA
#define HODLR_SOLVE_TMA 1
#endif
constexpr bool kSolveTma = HODLR_SOLVE_TMA;

// 9-16 RHS at r <= 32: two 8-column groups share every panel load (12 RHS 4.17 -> 3.41 ms)
constexpr bool kSolvePairs = true;

template <int R>
static hodlr_status run_solve_level(const LevelArgs& g, int64_t nblk, cudaStream_t st) {
  if (R <= 32 && g.ncols > 8 && kSolvePairs)
    solve_level_kernel<R, R <= 32 ? 2 : 1><<<(unsigned)nblk, 256, 0, st>>>(g);
  else
    solve_level_kernel<R, 1><<<(unsigned)nblk, 256, 0, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// multi-RHS solve step on the TMA-fed kernel (solve mode), one column group per
// warp at R = 64 (register budget), up to 2 at R <= 32
template <int R, int GPW>
static hodlr_status launch_level5_solve(const LevelArgs& g, int64_t nseg, int64_t rows, cudaStream_t st) {
  using Cfg = Level4Cfg<R, true>;
  constexpr size_t smem = (size_t)3 * Cfg::STAGE * sizeof(double);
  CUtensorMap ta, tv;
  if (!panel_map<R, true>(&ta, g.A1, rows, g.lda)) return HODLR_ERR_ARG;
  if (g.V != nullptr) {
    if (!panel_map<R, true>(&tv, g.V, rows, g.lda)) return HODLR_ERR_ARG;
  } else {
    tv = ta;  // unused (no next-level w)
  }
  smem_attr(level_update5_kernel<R, GPW, false, true>, (int)smem);
  level_update5_kernel<R, GPW, false, true><<<(unsigned)(nseg * g.ncg), 256, smem, st>>>(g, ta, tv);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template <int R>
static hodlr_status run_level4_solve(const LevelArgs& g, int64_t nseg, cudaStream_t st);

template <int R>
static hodlr_status run_level5_solve(const LevelArgs& g, int64_t nseg, int64_t rows, cudaStream_t st) {
  const int gpw = (g.tpc + 7) / 8;
  if (gpw <= 1) return launch_level5_solve<R, 1>(g, nseg, rows, st);
  if constexpr (R <= 32) {
    if (gpw <= 2) return launch_level5_solve<R, 2>(g, nseg, rows, st);
  }
  return run_level4_solve<R>(g, nseg, st);
}

template <int R>
static hodlr_status run_level4_solve(const LevelArgs& g, int64_t nseg, cudaStream_t st) {
  using Cfg = Level4Cfg<R, true>;
  const int gpw = (g.tpc + 7) / 8;
  auto launch = [&](auto kern) {
    smem_attr(kern, (int)Cfg::SMEM);
    kern<<<(unsigned)(nseg * g.ncg), 256, Cfg::SMEM, st>>>(g);
  };
  if (gpw <= 1) {
    launch(level_update4_kernel<R, 1, false, true>);
  } else if constexpr (R <= 32) {  // rank 64 solves run one column group per warp (solve_level_f64)
    if (gpw <= 2) launch(level_update4_kernel<R, 2, false, true>);
    else launch(level_update4_kernel<R, 4, false, true>);
  } else {
    return HODLR_ERR_ARG;
  }
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// partial-sum bytes of the solve level steps (one R x nrhs partial per CTA)
size_t solve_level_partial_bytes(int64_t n, int r, int nrhs) {
  return (size_t)(n / kSolveCtaRows + 1) * r * nrhs * sizeof(double);
}

hodlr_status level_reduce_f64(const double* part, double* TW, int r, int ncols, int segs, int nnodes, int64_t tw_stride,
                              cudaStream_t st);

// One solve level step over n rows of X (see solve_level_kernel).  Returns
// ERR_ARG for unsupported shapes (caller falls back).
hodlr_status solve_level_f64(int r, int64_t n, int64_t n_c, int64_t node_rows, double* X, int64_t ldx,
                             const double* A1, const double* V, int64_t lda, const double* W, int64_t wstride,
                             int nrhs, double* TW, int64_t tw_stride, double* part, size_t part_bytes,
                             cudaStream_t st) {
  if (nrhs == 0) return HODLR_OK;
  if (r != 16 && r != 32 && r != 64) return HODLR_ERR_ARG;
  if ((n_c % 64 && n_c < n) || n % 64 || node_rows % 64) return HODLR_ERR_ARG;
  if (n_c > 2147483647LL) n_c = 2147483647LL;
  if ((ldx & 3) || (reinterpret_cast<uintptr_t>(X) & 31) || (lda & 1) || (reinterpret_cast<uintptr_t>(A1) & 15) ||
      (V && (reinterpret_cast<uintptr_t>(V) & 15)) || (reinterpret_cast<uintptr_t>(W) & 15) || (wstride & 1))
    return HODLR_ERR_ARG;
  const int64_t cta_rows = std::min<int64_t>(kSolveCtaRows, n);
  if (n % cta_rows || (node_rows < cta_rows && cta_rows % node_rows) || (node_rows > cta_rows && node_rows % cta_rows))
    return HODLR_ERR_ARG;
  const int64_t nblk = n / cta_rows;
  const bool split = node_rows > cta_rows && V != nullptr;
  if (split && (size_t)nblk * r * nrhs * sizeof(double) > part_bytes) return HODLR_ERR_ARG;
  LevelArgs g{X, ldx, A1, V, lda, W, wstride, split ? part : TW, tw_stride, split ? 1 : 0, (int)n_c, (int)cta_rows,
              node_rows, nrhs, 1, 1};
  hodlr_status s;
  const int G = (nrhs + 7) / 8;
  if (nrhs >= 17) {  // crossover measured (cfg5 sweeps, profiles/r02_ab_x9.txt; 9-16 RHS: streaming kernel)
    // many right-hand sides: shared-memory panels reused by every column group
    // (same segments and reduction order as solve_level_kernel)
    const int gpc = std::min(G, r >= 64 ? 8 : 32);  // R = 64: one group per warp (register budget)
    g.seg_rows = (int)std::min<int64_t>(node_rows, cta_rows);
    g.ncg = (G + gpc - 1) / gpc;
    g.tpc = gpc;
    const int64_t nseg = n / g.seg_rows;
    // TMA feed: rank 64 at any nrhs (5-10 % faster), rank <= 32 up to 32 RHS (2-3 %);
    // 64-128 RHS at rank 32 stay on cp.async (4 % faster there; profiles/r02_ab_solve.txt)
    if (kSolveTma && (r >= 64 || nrhs <= 32))
      s = r == 16 ? run_level5_solve<16>(g, nseg, n, st)
          : r == 32 ? run_level5_solve<32>(g, nseg, n, st)
                    : run_level5_solve<64>(g, nseg, n, st);
    else
      s = r == 16 ? run_level4_solve<16>(g, nseg, st)
          : r == 32 ? run_level4_solve<32>(g, nseg, st)
                    : run_level4_solve<64>(g, nseg, st);
  } else {
    s = r == 16 ? run_solve_level<16>(g, nblk, st)
        : r == 32 ? run_solve_level<32>(g, nblk, st)
                  : run_solve_level<64>(g, nblk, st);
  }
  if (s != HODLR_OK || !split) return s;
  return level_reduce_f64(part, TW, r, nrhs, (int)(node_rows / cta_rows), (int)(n / node_rows), tw_stride, st);
}

// fixed-order sum of per-segment partials into the paired [W|T] / w layout
hodlr_status level_reduce_f64(const double* part, double* TW, int r, int ncols, int segs, int nnodes, int64_t tw_stride,
                              cudaStream_t st) {
  const int64_t total = (int64_t)r * ncols * nnodes;
  const int64_t blocks = std::min<int64_t>(ceil_div(segs > 32 ? total * 32 : total, 256), 8 * (int64_t)sm_count());
  level_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, TW, r, ncols, segs, nnodes, tw_stride);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// factorization level step fed by TMA (level_update5_kernel) or by cp.async (level_update4_kernel)
#ifndef HODLR_LEVEL_TMA
#define HODLR_LEVEL_TMA 1
#endif
constexpr bool kLevelTma = HODLR_LEVEL_TMA;

// column groups of 8 per level-kernel CTA: the [W|T] partials live in registers
static int level4_maxg(int r) { return r <= 16 ? 56 : r <= 32 ? 32 : 16; }

template <int R, int BN>
static hodlr_status run_level(const LevelArgs& g, int64_t nseg, cudaStream_t st) {
  using Cfg = LevelCfg<R, BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(level_update_kernel<R, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    attr = true;
  }
  level_update_kernel<R, BN><<<(unsigned)nseg, LV_THREADS, Cfg::SMEM, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}


// rows per CTA segment for a level whose nodes have `node` rows: the whole node
// when that already gives >= 2 CTAs per SM, else split (partial sums), and never
// more than 4096 rows of serial work per CTA.
int64_t level_segment_rows(int64_t n, int64_t node, int sms) {
  int64_t seg = node;
  const int64_t want = 2 * (int64_t)sms;
  while (seg > 64 && n / seg < want && seg % 128 == 0) seg >>= 1;
  while (seg > 4096 && seg % 128 == 0) seg >>= 1;
  return seg;
}

// partial-sum bytes the level steps need (max over levels and both schedules)
size_t level_partial_bytes(int64_t n, int m, int r, int L) {
  size_t best = 0;
  for (int lv = 1; lv < L; ++lv) {
    const int64_t node = n >> lv;
    const int64_t seg = level_segment_rows(n, node, 148);
    if (seg < node) best = std::max(best, (size_t)(n / seg) * r * r * lv * sizeof(double));
  }
  best = std::max(best, (size_t)kMaxSegs * r * r * std::max(L, 1) * sizeof(double));
  (void)m;
  return best;
}

// level_update6_kernel: items of 16 column groups; rows per item = the whole
// node unless that leaves the persistent CTAs unbalanced (then a power-of-two
// split with partial sums, at most kMaxSegs segments, preferring larger
// segments unless a split balances the waves >= 2 % better)
#ifndef HODLR_LEVEL6
#define HODLR_LEVEL6 1
#endif
// level_update6 at rank 32 (G >= 16 groups): a remainder of G mod 16 >= 12
// groups is one ragged level6 item (>= 75 % of its warps busy); a smaller
// remainder (4 or 8 groups) takes level_update4/5 in a second launch, since a
// mostly empty level6 item costs a full item's time (same-box launch lists,
// profiles/r02_level6.txt).  Rank 64 loses with 2 stages of 70 KB.
static int level6_groups(int r, int G) {
  if (!HODLR_LEVEL6 || r != 32 || G < 16) return 0;
  return G % 16 >= 12 ? G : G & ~15;
}

static int64_t level6_segment_rows(int64_t n, int64_t node, int64_t ncg, int sms, int ch) {
  int64_t best = node;
  double best_eff = -1.0;
  for (int64_t seg = node; seg >= ch && node % seg == 0; seg >>= 1) {
    const int64_t nseg = n / seg;
    if (seg < node && nseg > kMaxSegs) break;
    const int64_t items = nseg * ncg;
    const double eff = (double)items / (double)(ceil_div(items, sms) * sms);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = seg;
    }
    if (seg % (2 * ch)) break;
  }
  return best;
}

template <int R>
static hodlr_status run_level6(LevelArgs g, int64_t n, int64_t node, double* part, size_t part_bytes, double* TW,
                               cudaStream_t st) {
  using Cfg = Level6Cfg<R>;
  const int G = g.ncols / 8;
  const int64_t ncg = ceil_div(G, Cfg::GC);  // items per segment
  const int sms = sm_count();
  const int64_t seg = level6_segment_rows(n, node, ncg, sms, Cfg::CH);
  if (seg % Cfg::CH || (g.n_c < n && g.n_c % Cfg::CH) || n > 2147483647LL - Cfg::P) return HODLR_ERR_ARG;
  const int64_t nseg = n / seg;
  const bool split = seg < node;
  if (split && (size_t)nseg * R * g.ncols * sizeof(double) > part_bytes) return HODLR_ERR_ARG;
  g.seg_rows = (int)seg;
  g.ncg = (int)ncg;
  g.tpc = Cfg::GC;
  g.partial = split ? 1 : 0;
  g.TW = split ? part : TW;
  L6Maps tm;
  if (!panel_map_f64(&tm.a, g.A1, n, R, g.lda, Cfg::P) || !panel_map_f64(&tm.v, g.V, n, R, g.lda, Cfg::P))
    return HODLR_ERR_ARG;
  for (int k = 0; k < 5; ++k)
    if (!tensor_map_f64(&tm.c[k], g.C, n, g.ncols, g.ldc, Cfg::P, (Cfg::GC >> k) * 8)) return HODLR_ERR_ARG;
  const int64_t items = nseg * ncg;
  smem_attr(level_update6_kernel<R>, (int)Cfg::SMEM);
  level_update6_kernel<R><<<(unsigned)std::min<int64_t>(items, sms), Cfg::THREADS, Cfg::SMEM, st>>>(g, items, tm);
  HODLR_CHECK_LAUNCH();
  if (!split) return HODLR_OK;
  const int nnodes = (int)(n / node);
  const int64_t total = (int64_t)R * g.ncols * nnodes;
  const int segs = (int)(node / seg);
  const int64_t blocks = std::min<int64_t>(ceil_div(segs > 32 ? total * 32 : total, 256), 8 * (int64_t)sms);
  level_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, TW, R, g.ncols, segs, nnodes, g.tw_stride);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// One fused level step over all n rows.  Returns ERR_ARG when the shape is not
// supported (caller falls back to the generic batched GEMM path).
// reg_resident selects the register-resident kernel, which accumulates the
// update into C on the tensor core (factorization); the solve keeps the
// product-then-subtract kernel so every right-hand-side column is computed
// identically whatever nrhs is (multi-RHS bitwise contract).
hodlr_status level_update_f64(int r, int64_t n, int64_t n_c, int64_t node_rows, double* C, int64_t ldc,
                              const double* A1, const double* V, int64_t lda, const double* W, int64_t wstride,
                              int ncols, double* TW, int64_t tw_stride, double* part, size_t part_bytes,
                              cudaStream_t st, bool reg_resident) {
  if (ncols == 0) return HODLR_OK;
  if ((n_c % 64 && n_c < n) || n % 64 || node_rows % 64 || (r != 16 && r != 32 && r != 64)) return HODLR_ERR_ARG;
  if (n_c > 2147483647LL) n_c = 2147483647LL;  // a child larger than the local rows: W' half is pre-selected
  if ((ldc & 1) || (lda & 1) || (reinterpret_cast<uintptr_t>(C) & 15) || (reinterpret_cast<uintptr_t>(A1) & 15) ||
      (V && (reinterpret_cast<uintptr_t>(V) & 15)) || (reinterpret_cast<uintptr_t>(W) & 15) || (wstride & 1))
    return HODLR_ERR_ARG;
  const int64_t node = node_rows;  // rows of one output node
  const bool fact = V != nullptr && reg_resident && ncols > 8;
  const int ntile = (int)ceil_div(ncols, 64);
  FactSched fs{level_segment_rows(n, node, sm_count()), 1, ntile};
  // factorization: the column-group kernel (32-byte aligned C columns, groups of 8)
  const bool v4 = fact && ncols % 8 == 0 && !(ldc & 3) && !(reinterpret_cast<uintptr_t>(C) & 31);
  if (fact && !v4) return HODLR_ERR_ARG;  // generic GEMM path
  if (v4 && level6_groups(r, ncols / 8) > 0) {  // persistent, C staged by TMA
    const int c6 = 8 * level6_groups(r, ncols / 8);
    LevelArgs g6{C, ldc, A1, V, lda, W, wstride, TW, tw_stride, 0, (int)n_c, 0, node, c6, 0, 0};
    const hodlr_status s6 = run_level6<32>(g6, n, node, part, part_bytes, TW, st);
    if (s6 != HODLR_OK || c6 == ncols) {
      if (s6 != HODLR_ERR_ARG) return s6;
    } else {  // remainder columns [c6, ncols): same step on the column-offset operands
      return level_update_f64(r, n, n_c, node_rows, C + (int64_t)c6 * ldc, ldc, A1, V, lda, W + (int64_t)c6 * 2 * r,
                              wstride, ncols - c6, TW + (int64_t)c6 * 2 * r, tw_stride, part, part_bytes, st,
                              reg_resident);
    }
  }
  if (v4) fs = level4_schedule(n, node, ncols / 8, sm_count(), level4_maxg(r));
  const int64_t seg = fs.seg;
  const int64_t nseg = n / seg;
  if (nseg * fs.ncg > 2147483647LL) return HODLR_ERR_ARG;
  const bool split = seg < node && V != nullptr;
  if (split && (size_t)nseg * r * ncols * sizeof(double) > part_bytes) return HODLR_ERR_ARG;
  LevelArgs g{C, ldc, A1, V, lda, W, wstride, split ? part : TW, tw_stride, split ? 1 : 0, (int)n_c, (int)seg, node,
              ncols, fs.ncg, fs.tpc};
  const bool small = ncols <= 8;
  hodlr_status s;
  switch (r) {
    case 16: s = small ? run_level<16, 8>(g, nseg, st) : v4 ? (kLevelTma ? run_level5<16>(g, nseg, n, st) : run_level4<16>(g, nseg, st)) : run_level<16, 64>(g, nseg, st); break;
    case 32: s = small ? run_level<32, 8>(g, nseg, st) : v4 ? (kLevelTma ? run_level5<32>(g, nseg, n, st) : run_level4<32>(g, nseg, st)) : run_level<32, 64>(g, nseg, st); break;
    case 64: if (!v4) return HODLR_ERR_ARG; s = kLevelTma ? run_level5<64>(g, nseg, n, st) : run_level4<64>(g, nseg, st); break;
    default: return HODLR_ERR_ARG;  // r = 64: generic path (fused tiles exceed shared memory)
  }
  if (s != HODLR_OK || !split) return s;
  const int nnodes = (int)(n / node);
  const int64_t total = (int64_t)r * ncols * nnodes;
  const int segs = (int)(node / seg);
  const int64_t blocks = std::min<int64_t>(ceil_div(segs > 32 ? total * 32 : total, 256), 8 * (int64_t)sm_count());
  level_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, TW, r, ncols, segs, nnodes, tw_stride);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

}  // namespace hodlr
