// Batched LU solve as two triangular DMMA GEMMs (backend.py:546-567 semantics):
//
//   X_b = U_b^-1 ( L_b^-1 ( P_b B_b ) )
//
// with the packed inverses Tinv_b = strict_lower(L^-1) + upper(U^-1) produced
// by the getrf kernels.  One CTA per (block, group of BN-column tiles): Tinv_b
// is staged in shared memory once, then the row-gathered tiles P B stream
// through a 2-stage cp.async pipeline.  Each tile is multiplied by the
// unit-lower factor (k < m masked, identity folded into the accumulator init),
// written back to shared memory, multiplied by the upper factor (k >= m
// masked) and stored coalesced.  X may alias B (a CTA reads a tile before it
// writes it, and tiles are disjoint).
//
// Optional fused reduction (TWR > 0): with the solved tile still in shared
// memory, TW_b(:, tile) = V_b^T X_b(:, tile) is formed for the next tree level
// (V_b = the block's rows of the V panel).  This turns the leaf solve of Alg. 3
// line 3 and the level-(L-1) [W|T] GEMM of lines 5-6 into one HBM pass.
//
// Used for the leaf solve of Y, K_p^-1 W (Alg.3 l.9) and the solve phase.
#include <cstdlib>

#include "common.cuh"
#include "lu_device.cuh"

namespace hodlr {

struct ApplyArgs {
  const double* tinv;  // packed full inverses (S in {16, 128}) or diagonal-block inverses (S in {32, 64})
  const double* lu;    // the LU factors (same layout as tinv); used with the diagonal-block format
  int64_t ldi, strideT;  // LU: block b at lu + b * strideT (ld ldi)
  int64_t strideI;       // inverses: block b at tinv + b * strideI
  const int32_t* perm;
  const double* B;
  int64_t ldb, sB_hi, sB_lo;
  double* X;
  int64_t ldx, sX_hi, sX_lo;
  int ncols, batch, bdiv, groups;
  const double* V;  // TW fusion: V_b at V + b * vstride, ld ldv (s x TWR)
  int64_t ldv, vstride;
  double* TW;  // TW_b at TW + (b>>1) * tw_stride + (b&1) * TWR, ld 2 TWR
  int64_t tw_stride;
};

__device__ __forceinline__ int64_t aoff(int b, int bdiv, int64_t hi, int64_t lo) {
  return (int64_t)(b / bdiv) * hi + (int64_t)(b % bdiv) * lo;
}

constexpr int AP_THREADS = 256;

template <int S, int BN>
struct ApplyCfg {
  // 8 warps: BN >= 32 -> (S/32) x (8/(S/32)) grid of 32-row warp tiles; BN = 8 -> warps along M
  static constexpr int WM = (BN >= 32) ? ((S >= 32) ? S / 32 : 1) : (S / 8 < 8 ? S / 8 : 8);
  static constexpr int WN = (BN >= 32) ? 8 / WM : 1;
  static constexpr int WTM = S / WM, WTN = BN / WN;
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  static constexpr int P = S + 4;
};

template <int S, int BN, int TWR>
__global__ void __launch_bounds__(AP_THREADS) tri_apply_kernel(ApplyArgs g) {
  using Cfg = ApplyCfg<S, BN>;
  constexpr int WN = Cfg::WN, WTM = Cfg::WTM, WTN = Cfg::WTN, MI = Cfg::MI, NI = Cfg::NI, P = Cfg::P;
  static_assert(MI >= 1 && NI >= 1, "tile config");
  extern __shared__ __align__(16) double sm[];
  double* At = sm;                 // [k][m] packed inverses
  // with the fused reduction the V panel takes the second tile buffer's place,
  // so 2 CTAs still fit per SM (the co-resident CTA hides the tile load)
  constexpr int NBUF = TWR > 0 ? 1 : 2;
  double* Bbuf = sm + S * P;          // NBUF x [n][k] tiles
  double* Vs = Bbuf + NBUF * BN * P;  // [j][k] (TWR x S, k contiguous)
  __shared__ int pm[S];

  const int b = blockIdx.x / g.groups;
  const int grp = blockIdx.x % g.groups;
  const int ntiles = (g.ncols + BN - 1) / BN;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const bool mma_warp = warp < Cfg::WM * WN;
  const int ar = lane >> 2, ac = lane & 3;

  const double* ti = g.tinv + (int64_t)b * g.strideI;
  for (int idx = t; idx < S * (S / 2); idx += AP_THREADS) {
    const int k = idx / (S / 2), m = (idx % (S / 2)) * 2;
    cp_async_16(At + k * P + m, ti + m + (int64_t)k * g.ldi, 16);
  }
  if constexpr (TWR > 0) {
    const double* vb = g.V + (int64_t)b * g.vstride;
    for (int idx = t; idx < TWR * (S / 2); idx += AP_THREADS) {
      const int j = idx / (S / 2), k = (idx % (S / 2)) * 2;
      cp_async_16(Vs + j * P + k, vb + k + (int64_t)j * g.ldv, 16);
    }
  }
  if (t < S) pm[t] = g.perm[(int64_t)b * S + t];
  __syncthreads();
  const double* Bb = g.B + aoff(b, g.bdiv, g.sB_hi, g.sB_lo);
  double* Xb = g.X + aoff(b, g.bdiv, g.sX_hi, g.sX_lo);

  // the tile is staged in natural row order with 16-byte copies; the row
  // permutation P is applied when stage 1 reads it (pm[] lookups)
  const bool vec16 = !((reinterpret_cast<uintptr_t>(Bb) | (uintptr_t)(g.ldb * 8)) & 15);
  auto load_tile = [&](int tile, double* Bs) {
    const int n0 = tile * BN;
    if (vec16) {
      for (int idx = t; idx < BN * (S / 2); idx += AP_THREADS) {
        const int n = idx / (S / 2), k = (idx % (S / 2)) * 2;
        const bool ok = n0 + n < g.ncols;
        cp_async_16(Bs + n * P + k, ok ? Bb + k + (int64_t)(n0 + n) * g.ldb : g.B, ok ? 16 : 0);
      }
    } else {
      for (int idx = t; idx < BN * S; idx += AP_THREADS) {
        const int n = idx / S, k = idx % S;
        const bool ok = n0 + n < g.ncols;
        cp_async_8(Bs + n * P + k, ok ? Bb + k + (int64_t)(n0 + n) * g.ldb : g.B, ok ? 8 : 0);
      }
    }
  };

  int cur = 0;
  if (grp < ntiles) load_tile(grp, Bbuf);
  cp_async_commit();
  for (int tile = grp; tile < ntiles; tile += g.groups) {
    double* Bs = Bbuf + cur * BN * P;
    if constexpr (NBUF == 2) {
      if (tile + g.groups < ntiles) load_tile(tile + g.groups, Bbuf + (cur ^ 1) * BN * P);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      if (tile != grp) {
        load_tile(tile, Bs);
        cp_async_commit();
      }
      cp_async_wait<0>();
    }
    __syncthreads();

    double acc[MI][NI][2];
    // Row tiles are dealt to warps in balanced pairs (tile q with tile S/8-1-q), so
    // every warp does the same triangular work in both stages.
    int mrow[MI];
    int kmax = 0, kmin = S;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      constexpr int H = MI / 2;
      mrow[i] = (MI == 1) ? 8 * wm : (i < H ? 8 * (wm * H + i) : 8 * (S / 8 - 1 - (wm * H + (i - H))));
      kmax = max(kmax, mrow[i] + 8);
      kmin = min(kmin, mrow[i]);
    }
    // stage 1: T = P B + strict_lower(L^-1) P B
    if (mma_warp) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = mrow[i] + ar, n = wn * WTN + j * 8 + ac * 2 + h;
            acc[i][j][h] = Bs[n * P + pm[m]];
          }
      for (int k0 = 0; k0 < kmax; k0 += 4) {
        const int k = k0 + ac;
        const int pk = pm[k];
        double bf[NI];
#pragma unroll
        for (int j = 0; j < NI; ++j) bf[j] = Bs[(wn * WTN + j * 8 + ar) * P + pk];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          if (k0 < mrow[i] + 8) {
            const int m = mrow[i] + ar;
            const double af = (k < m) ? At[k * P + m] : 0.0;
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af, bf[j]);
          }
        }
      }
    }
    __syncthreads();
    if (mma_warp) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = mrow[i] + ar, n = wn * WTN + j * 8 + ac * 2 + h;
            Bs[n * P + m] = acc[i][j][h];
            acc[i][j][h] = 0.0;
          }
    }
    __syncthreads();
    // stage 2: X = upper(U^-1) T
    if (mma_warp) {
      for (int k0 = kmin; k0 < S; k0 += 4) {
        const int k = k0 + ac;
        double bf[NI];
#pragma unroll
        for (int j = 0; j < NI; ++j) bf[j] = Bs[(wn * WTN + j * 8 + ar) * P + k];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          if (k0 + 3 >= mrow[i]) {
            const int m = mrow[i] + ar;
            const double af = (k >= m) ? At[k * P + m] : 0.0;
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af, bf[j]);
          }
        }
      }
    }
    __syncthreads();
    if (mma_warp) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = mrow[i] + ar, n = wn * WTN + j * 8 + ac * 2 + h;
            Bs[n * P + m] = acc[i][j][h];
          }
    }
    __syncthreads();
    const int n0 = tile * BN;
    for (int idx = t; idx < BN * S; idx += AP_THREADS) {
      const int n = idx / S, m = idx % S;
      if (n0 + n < g.ncols) Xb[m + (int64_t)(n0 + n) * g.ldx] = Bs[n * P + m];
    }
    if constexpr (TWR > 0) {
      // TW_b(:, tile) = V_b^T X_b(:, tile): TWR x BN, K = S.  BN = 64: one n-tile per
      // warp, all TWR/8 m-tiles; BN = 8: one m-tile per warp.
      constexpr int TWN = BN / 8;
      constexpr int TMI = TWN >= 8 ? TWR / 8 : 1;
      constexpr int NTW = TWN >= 8 ? 8 : (TWR / 8) * TWN;
      if (warp < NTW) {
        const int tn = TWN >= 8 ? warp : warp / (TWR / 8);
        const int tm0 = TWN >= 8 ? 0 : warp % (TWR / 8);
        double tw[TMI][2];
#pragma unroll
        for (int i = 0; i < TMI; ++i) tw[i][0] = tw[i][1] = 0.0;
#pragma unroll 4
        for (int k0 = 0; k0 < S; k0 += 4) {
          const double bf = Bs[(tn * 8 + ar) * P + k0 + ac];
#pragma unroll
          for (int i = 0; i < TMI; ++i) {
            const double af = Vs[((tm0 + i) * 8 + ar) * P + k0 + ac];
            dmma_8x8x4(tw[i][0], tw[i][1], af, bf);
          }
        }
        double* out = g.TW + (int64_t)(b >> 1) * g.tw_stride + (b & 1) * TWR;
#pragma unroll
        for (int i = 0; i < TMI; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int mm = (tm0 + i) * 8 + ar, nn = n0 + tn * 8 + ac * 2 + h;
            if (nn < g.ncols) out[mm + (int64_t)nn * 2 * TWR] = tw[i][h];
          }
      }
    }
    __syncthreads();
    if constexpr (NBUF == 2) cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// Column-group variant (S in {32, 64}): every warp owns 8 columns of B at a
// time and runs the whole chain for them in registers, transposed so that no
// operand ever changes lanes:
//
//   T^T = (P B)^T L^-T     A = gathered rows of B (lane: column, 2 rows)
//   X^T = T^T U^-T         A = the stage-1 accumulators, as they are
//   TW^T = X^T V           A = the stage-2 accumulators, as they are
//
// The k index of every product runs over rows in the order (tile j, pair
// 2c + h), which is exactly the order in which an m8n8k4 accumulator holds a
// lane's row entries -- so accumulators feed the next product directly.  The
// triangular factors are read as [row][k] LDS.128 pairs (pitch 8 mod 16:
// conflict-free) and only their non-zero 8x8 tiles are multiplied.  No CTA
// barrier after the one-time staging of Tinv / V: warps stream their column
// groups independently, B of the next group prefetched into registers.
// ---------------------------------------------------------------------------
template <int S>
struct Apply2Cfg {
  static constexpr int PT = S + 8;  // Tinv [row][k] and V [rank][row] pitch (8 mod 16)
};

// IO = float: the fp32 factorization's leaf apply (cfg4) on the same fp64 DMMA
// chain -- operands widened on load, results rounded to fp32 on store, the
// diagonal-block inverses formed in the kernel from the staged (widened) fp32
// LU (the fp32 LU kernel emits none).  The ApplyArgs pointers then address
// float data.
template <int S, int TWR, typename IO = double>
__global__ void __launch_bounds__(AP_THREADS, S >= 128 ? 1 : 2) tri_apply2_kernel(ApplyArgs g) {
  constexpr int NJ = S / 8, PT = Apply2Cfg<S>::PT, RT = TWR / 8;
  constexpr bool F32 = sizeof(IO) == 4;
  extern __shared__ __align__(16) double sm[];
  double* Tm = sm;            // [row][k]
  double* Vs = sm + S * PT;   // [rank][row]
  __shared__ __align__(8) int pm[S];
  const int b = blockIdx.x / g.groups, part = blockIdx.x % g.groups;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;

  // ---- one-time staging, [row][k] (k pairs per thread): the LU factors off the
  // diagonal 8x8 tiles, the diagonal-block inverses P_q on them ----
  const IO* lb = reinterpret_cast<const IO*>(g.lu) + (int64_t)b * g.strideT;
  const double* di = g.tinv + (int64_t)b * g.strideI;
  for (int idx = t; idx < S * (S / 2); idx += AP_THREADS) {
    const int m = idx % S, k = (idx / S) * 2;
    double2 x;
    if (!F32 && (m >> 3) == (k >> 3))
      x = *reinterpret_cast<const double2*>(di + 64 * (m >> 3) + 8 * (m & 7) + (k & 7));
    else
      x = make_double2((double)lb[m + (int64_t)k * g.ldi], (double)lb[m + (int64_t)(k + 1) * g.ldi]);
    *reinterpret_cast<double2*>(Tm + m * PT + k) = x;
  }
  if constexpr (TWR > 0) {
    if constexpr (F32) {
      const float* vb = reinterpret_cast<const float*>(g.V) + (int64_t)b * g.vstride;
      for (int idx = t; idx < TWR * S; idx += AP_THREADS) {
        const int j = idx / S, k = idx % S;
        Vs[j * PT + k] = (double)vb[k + (int64_t)j * g.ldv];
      }
    } else {
      const double* vb = g.V + (int64_t)b * g.vstride;
      for (int idx = t; idx < TWR * (S / 2); idx += AP_THREADS) {
        const int j = idx / (S / 2), k = (idx % (S / 2)) * 2;
        cp_async_16(Vs + j * PT + k, vb + k + (int64_t)j * g.ldv, 16);
      }
      cp_async_commit();
    }
  }
  if (t < S) pm[t] = g.perm[(int64_t)b * S + t];
  if constexpr (!F32) cp_async_wait<0>();
  __syncthreads();
  if constexpr (F32) {  // P_q from the staged LU, then onto the diagonal tiles
    double* dtmp = Vs + TWR * PT;
    diag_block_inverses<S>(Tm, PT, 1, dtmp, AP_THREADS);
    __syncthreads();
    for (int idx = t; idx < S * 8; idx += AP_THREADS) {
      const int m = idx >> 3, k = (m & ~7) + (idx & 7);
      Tm[m * PT + k] = dtmp[64 * (m >> 3) + 8 * (m & 7) + (idx & 7)];
    }
    __syncthreads();
  }

  const IO* Bb = reinterpret_cast<const IO*>(g.B) + aoff(b, g.bdiv, g.sB_hi, g.sB_lo);
  IO* Xb = reinterpret_cast<IO*>(g.X) + aoff(b, g.bdiv, g.sX_hi, g.sX_lo);

  const int G = (g.ncols + 7) >> 3;
  const int gpc = (G + g.groups - 1) / g.groups;
  const int g0 = part * gpc, g1 = min(G, g0 + gpc);
  auto load_b = [&](int grp, double (&v)[NJ][2]) {
    const int col = grp * 8 + ar;
    const bool ok = col < g.ncols;
    const IO* bc = Bb + (int64_t)(ok ? col : 0) * g.ldb;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {  // this lane's gathered rows: P rows 8j + 2ac + {0, 1}
      const int2 p = *reinterpret_cast<const int2*>(pm + 8 * j + 2 * ac);
      v[j][0] = ok ? (double)bc[p.x] : 0.0;
      v[j][1] = ok ? (double)bc[p.y] : 0.0;
    }
  };

  double bn[NJ][2];
  int grp = g0 + warp;
  if (grp < g1) load_b(grp, bn);
  for (; grp < g1; grp += 8) {
    double bv[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j) bv[j][0] = bn[j][0], bv[j][1] = bn[j][1];
    if (grp + 8 < g1) load_b(grp + 8, bn);
    // ---- stage 1: blocked forward substitution, T_j = L_jj^-1 ((P B)_j - sum_{i<j} L_ji T_i) ----
    double a1[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      double c0 = bv[j][0], c1 = bv[j][1];
#pragma unroll
      for (int i = 0; i < j; ++i) {
        const double2 l = *reinterpret_cast<const double2*>(Tm + (8 * j + ar) * PT + 8 * i + 2 * ac);
        dmma_8x8x4(c0, c1, a1[i][0], -l.x);
        dmma_8x8x4(c0, c1, a1[i][1], -l.y);
      }
      const double2 p = *reinterpret_cast<const double2*>(Tm + (8 * j + ar) * PT + 8 * j + 2 * ac);
      const int k0 = 2 * ac;
      const double lx = k0 < ar ? p.x : (k0 == ar ? 1.0 : 0.0);
      const double ly = k0 + 1 < ar ? p.y : (k0 + 1 == ar ? 1.0 : 0.0);
      a1[j][0] = a1[j][1] = 0.0;
      dmma_8x8x4(a1[j][0], a1[j][1], c0, lx);
      dmma_8x8x4(a1[j][0], a1[j][1], c1, ly);
    }
    // ---- stage 2: blocked backward substitution, X_j = U_jj^-1 (T_j - sum_{i>j} U_ji X_i) ----
    double a2[NJ][2];
#pragma unroll
    for (int j = NJ - 1; j >= 0; --j) {
      double c0 = a1[j][0], c1 = a1[j][1];
#pragma unroll
      for (int i = j + 1; i < NJ; ++i) {
        const double2 u = *reinterpret_cast<const double2*>(Tm + (8 * j + ar) * PT + 8 * i + 2 * ac);
        dmma_8x8x4(c0, c1, a2[i][0], -u.x);
        dmma_8x8x4(c0, c1, a2[i][1], -u.y);
      }
      const double2 p = *reinterpret_cast<const double2*>(Tm + (8 * j + ar) * PT + 8 * j + 2 * ac);
      const int k0 = 2 * ac;
      const double ux = k0 >= ar ? p.x : 0.0;
      const double uy = k0 + 1 >= ar ? p.y : 0.0;
      a2[j][0] = a2[j][1] = 0.0;
      dmma_8x8x4(a2[j][0], a2[j][1], c0, ux);
      dmma_8x8x4(a2[j][0], a2[j][1], c1, uy);
    }
    const int col = grp * 8 + ar;
    if (col < g.ncols) {
      IO* xc = Xb + (int64_t)col * g.ldx + 2 * ac;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if constexpr (F32)
          *reinterpret_cast<float2*>(xc + 8 * j) = make_float2((float)a2[j][0], (float)a2[j][1]);
        else
          *reinterpret_cast<double2*>(xc + 8 * j) = make_double2(a2[j][0], a2[j][1]);
      }
    }
    if constexpr (TWR > 0) {
      // ---- TW^T = X^T V, in passes of at most 32 ranks (bounded registers) ----
      constexpr int RP = RT < 4 ? RT : 4;
#pragma unroll
      for (int r0 = 0; r0 < RT; r0 += RP) {
        double tw[RP][2];
#pragma unroll
        for (int jr = 0; jr < RP; ++jr) tw[jr][0] = tw[jr][1] = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int jr = 0; jr < RP; ++jr) {
            const double2 v = *reinterpret_cast<const double2*>(Vs + (8 * (r0 + jr) + ar) * PT + 8 * j + 2 * ac);
            dmma_8x8x4(tw[jr][0], tw[jr][1], a2[j][0], v.x);
            dmma_8x8x4(tw[jr][0], tw[jr][1], a2[j][1], v.y);
          }
        if (col < g.ncols) {
          IO* out = reinterpret_cast<IO*>(g.TW) + (int64_t)(b >> 1) * g.tw_stride + (b & 1) * TWR +
                    (int64_t)col * 2 * TWR + 2 * ac;
#pragma unroll
          for (int jr = 0; jr < RP; ++jr) {
            if constexpr (F32)
              *reinterpret_cast<float2*>(out + 8 * (r0 + jr)) = make_float2((float)tw[jr][0], (float)tw[jr][1]);
            else
              *reinterpret_cast<double2*>(out + 8 * (r0 + jr)) = make_double2(tw[jr][0], tw[jr][1]);
          }
        }
      }
    }
  }
}

static bool apply2_ok(const ApplyArgs& g) {
  // 16-byte X stores and 16-byte TW stores need even strides and aligned bases
  return !(g.ldx & 1) && !(g.sX_hi & 1) && !(g.sX_lo & 1) && !(reinterpret_cast<uintptr_t>(g.X) & 15) &&
         (g.TW == nullptr || (!(g.tw_stride & 1) && !(reinterpret_cast<uintptr_t>(g.TW) & 15)));
}


// X = U^-1 L^-1 (P B) for one 8-column group of one block in the blocked
// diagonal-block-inverse form: bv = the lane's gathered rows of P B, tl(jn, j)
// = the (row 8 jn + ar, columns 8 j + 2 ac + {0, 1}) pair of the LU off the
// diagonal tiles and of the diagonal-block inverse on them.  The DMMA sequence
// is the one of tri_apply2_kernel (bit-identical columns).
template <int NJ, typename TL>
__device__ __forceinline__ void blocked_solve(const double (&bv)[NJ][2], double (&a2)[NJ][2], TL tl, int ar, int ac) {
  double a1[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    double c0 = bv[j][0], c1 = bv[j][1];
#pragma unroll
    for (int i = 0; i < j; ++i) {
      const double2 l = tl(j, i);
      dmma_8x8x4(c0, c1, a1[i][0], -l.x);
      dmma_8x8x4(c0, c1, a1[i][1], -l.y);
    }
    const double2 p = tl(j, j);
    const int k0 = 2 * ac;
    const double lx = k0 < ar ? p.x : (k0 == ar ? 1.0 : 0.0);
    const double ly = k0 + 1 < ar ? p.y : (k0 + 1 == ar ? 1.0 : 0.0);
    a1[j][0] = a1[j][1] = 0.0;
    dmma_8x8x4(a1[j][0], a1[j][1], c0, lx);
    dmma_8x8x4(a1[j][0], a1[j][1], c1, ly);
  }
#pragma unroll
  for (int j = NJ - 1; j >= 0; --j) {
    double c0 = a1[j][0], c1 = a1[j][1];
#pragma unroll
    for (int i = j + 1; i < NJ; ++i) {
      const double2 u = tl(j, i);
      dmma_8x8x4(c0, c1, a2[i][0], -u.x);
      dmma_8x8x4(c0, c1, a2[i][1], -u.y);
    }
    const double2 p = tl(j, j);
    const int k0 = 2 * ac;
    const double ux = k0 >= ar ? p.x : 0.0;
    const double uy = k0 + 1 >= ar ? p.y : 0.0;
    a2[j][0] = a2[j][1] = 0.0;
    dmma_8x8x4(a2[j][0], a2[j][1], c0, ux);
    dmma_8x8x4(a2[j][0], a2[j][1], c1, uy);
  }
}

// Narrow variant (the solve phase: up to narrow_cols right-hand sides): one
// warp per (block, 8-column group), the packed inverses, the permutation and
// the V panel read straight from global memory into fragments -- the phase is
// a single HBM pass over Tinv / V.
template <int S, int TWR>
__global__ void __launch_bounds__(AP_THREADS, S >= 128 ? 1 : 2) tri_apply_narrow_kernel(ApplyArgs g) {
  constexpr int NJ = S / 8, RT = TWR / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp -> (block, column group): the groups of a block are consecutive warps,
  // so the block's factors come from HBM once and from L1 for its other groups
  const int64_t gw = (int64_t)blockIdx.x * (AP_THREADS / 32) + warp;
  const int b = (int)(gw / g.groups);
  if (b >= g.batch) return;
  const int ar = lane >> 2, ac = lane & 3;
  const double* ti = g.tinv + (int64_t)b * g.strideI;
  const int32_t* pmb = g.perm + (int64_t)b * S;
  const double* Bb = g.B + aoff(b, g.bdiv, g.sB_hi, g.sB_lo);
  double* Xb = g.X + aoff(b, g.bdiv, g.sX_hi, g.sX_lo);
  const int col = (int)(gw % g.groups) * 8 + ar;
  const bool ok = col < g.ncols;
  double bv[NJ][2];
  {
    const double* bc = Bb + (int64_t)(ok ? col : 0) * g.ldb;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int2 p = __ldg(reinterpret_cast<const int2*>(pmb + 8 * j + 2 * ac));
      bv[j][0] = ok ? bc[p.x] : 0.0;
      bv[j][1] = ok ? bc[p.y] : 0.0;
    }
  }
  const double* lb = g.lu + (int64_t)b * g.strideT;
  double a2[NJ][2];
  blocked_solve<NJ>(bv, a2, [&](int jn, int j) {
    if (jn == j) return __ldg(reinterpret_cast<const double2*>(ti + 64 * j + 8 * ar + 2 * ac));
    const double* q = lb + (8 * jn + ar) + (int64_t)(8 * j + 2 * ac) * g.ldi;
    return make_double2(__ldg(q), __ldg(q + g.ldi));
  }, ar, ac);
  if (ok) {
    double* xc = Xb + (int64_t)col * g.ldx + 2 * ac;
#pragma unroll
    for (int j = 0; j < NJ; ++j) *reinterpret_cast<double2*>(xc + 8 * j) = make_double2(a2[j][0], a2[j][1]);
  }
  if constexpr (TWR > 0) {
    const double* vb = g.V + (int64_t)b * g.vstride;
    constexpr int RP = RT < 4 ? RT : 4;
#pragma unroll
    for (int r0 = 0; r0 < RT; r0 += RP) {
      double tw[RP][2];
#pragma unroll
      for (int jr = 0; jr < RP; ++jr) tw[jr][0] = tw[jr][1] = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int jr = 0; jr < RP; ++jr) {
          const double2 v =
              __ldg(reinterpret_cast<const double2*>(vb + (int64_t)(8 * (r0 + jr) + ar) * g.ldv + 8 * j + 2 * ac));
          dmma_8x8x4(tw[jr][0], tw[jr][1], a2[j][0], v.x);
          dmma_8x8x4(tw[jr][0], tw[jr][1], a2[j][1], v.y);
        }
      if (ok) {
        double* out = g.TW + (int64_t)(b >> 1) * g.tw_stride + (b & 1) * TWR + (int64_t)col * 2 * TWR + 2 * ac;
#pragma unroll
        for (int jr = 0; jr < RP; ++jr) *reinterpret_cast<double2*>(out + 8 * (r0 + jr)) = make_double2(tw[jr][0], tw[jr][1]);
      }
    }
  }
}

// Staged variant for small batches (the top levels of the solve's K phase,
// where one block's dependent substitution chain is the whole launch): the CTA
// copies its block's LU (pitch S + 2), diagonal-block inverses and permutation
// into shared memory with every load in flight at once, then warp w solves
// column group w from shared memory -- one memory latency per launch instead
// of one per substitution step.  Same DMMA sequence (bit-identical).
template <int S>
__global__ void __launch_bounds__(AP_THREADS, 1) tri_apply_staged_kernel(ApplyArgs g) {
  constexpr int NJ = S / 8, PL = S + 2;
  extern __shared__ __align__(16) double stg[];
  double* Ls = stg;                      // S columns x PL
  double* Ts = stg + S * PL;             // 8 S inverse entries
  int* Ps = reinterpret_cast<int*>(Ts + 8 * S);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int b = blockIdx.x;
  const double* lb = g.lu + (int64_t)b * g.strideT;
  const double* ti = g.tinv + (int64_t)b * g.strideI;
  for (int e = t; e < S * (S / 2); e += AP_THREADS) {  // 16-byte pieces of the LU columns
    const int c = e / (S / 2), r2 = e % (S / 2);
    cp_async_16(Ls + c * PL + 2 * r2, lb + (int64_t)c * g.ldi + 2 * r2, 16);
  }
  for (int e = t; e < 4 * S; e += AP_THREADS) cp_async_16(Ts + 2 * e, ti + 2 * e, 16);
  for (int e = t; e < S / 4; e += AP_THREADS) cp_async_16(Ps + 4 * e, g.perm + (int64_t)b * S + 4 * e, 16);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (warp >= g.groups) return;
  const int ar = lane >> 2, ac = lane & 3;
  const double* Bb = g.B + aoff(b, g.bdiv, g.sB_hi, g.sB_lo);
  double* Xb = g.X + aoff(b, g.bdiv, g.sX_hi, g.sX_lo);
  const int col = warp * 8 + ar;
  const bool ok = col < g.ncols;
  double bv[NJ][2];
  {
    const double* bc = Bb + (int64_t)(ok ? col : 0) * g.ldb;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int2 p = *reinterpret_cast<const int2*>(Ps + 8 * j + 2 * ac);
      bv[j][0] = ok ? bc[p.x] : 0.0;
      bv[j][1] = ok ? bc[p.y] : 0.0;
    }
  }
  double a2[NJ][2];
  blocked_solve<NJ>(bv, a2, [&](int jn, int j) {
    if (jn == j) return *reinterpret_cast<const double2*>(Ts + 64 * j + 8 * ar + 2 * ac);
    const double* q = Ls + (8 * jn + ar) + (8 * j + 2 * ac) * PL;
    return make_double2(q[0], q[PL]);
  }, ar, ac);
  if (ok) {
    double* xc = Xb + (int64_t)col * g.ldx + 2 * ac;
#pragma unroll
    for (int j = 0; j < NJ; ++j) *reinterpret_cast<double2*>(xc + 8 * j) = make_double2(a2[j][0], a2[j][1]);
  }
}

template <int S>
static hodlr_status run_apply_staged(ApplyArgs g, cudaStream_t st) {
  constexpr size_t smem = ((size_t)S * (S + 2) + 8 * S) * sizeof(double) + S * sizeof(int);
  g.groups = (int)ceil_div(g.ncols, 8);
  if (g.groups > AP_THREADS / 32) return HODLR_ERR_ARG;
  smem_attr(tri_apply_staged_kernel<S>, (int)smem);
  tri_apply_staged_kernel<S><<<(unsigned)g.batch, AP_THREADS, smem, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

static bool apply_staged_ok(const ApplyArgs& g) {
  // 16-byte cp.async pieces of the LU columns, inverses and permutation
  return !(g.ldi & 1) && !(g.strideT & 1) && !(reinterpret_cast<uintptr_t>(g.lu) & 15) && !(g.strideI & 1) &&
         !(reinterpret_cast<uintptr_t>(g.perm) & 15) && !(reinterpret_cast<uintptr_t>(g.tinv) & 15);
}

// batches up to this many blocks take the staged kernel (latency-bound launches)
#ifndef HODLR_STAGED_MAX_BATCH
#define HODLR_STAGED_MAX_BATCH 148
#endif
constexpr int kStagedMaxBatch = HODLR_STAGED_MAX_BATCH;

template <int S, int TWR>
static hodlr_status run_apply_narrow(ApplyArgs g, cudaStream_t st) {
  g.groups = (int)ceil_div(g.ncols, 8);
  const int64_t grid = ceil_div((int64_t)g.batch * g.groups, AP_THREADS / 32);
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  tri_apply_narrow_kernel<S, TWR><<<(unsigned)grid, AP_THREADS, 0, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

static bool apply_narrow_ok(const ApplyArgs& g) {
  // 16-byte B/X/V/TW accesses of the narrow kernel
  return apply2_ok(g) && !(g.ldi & 1) && (g.V == nullptr || (!(g.ldv & 1) && !(g.vstride & 1)));
}

template <int S, int TWR>
static hodlr_status run_apply2(ApplyArgs g, cudaStream_t st) {
  constexpr int PT = Apply2Cfg<S>::PT;
  constexpr size_t smem = (size_t)(S + TWR) * PT * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tri_apply2_kernel<S, TWR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  // CTAs per block: one (8 warps over the block's column groups) unless the
  // batch is too small to fill 2 CTAs per SM
  const int G = (int)ceil_div(g.ncols, 8);
  int cpb = 1;
  while ((int64_t)g.batch * cpb < 2 * 148 && cpb * 8 < G) cpb *= 2;
  g.groups = cpb;
  const int64_t grid = (int64_t)g.batch * cpb;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  tri_apply2_kernel<S, TWR><<<(unsigned)grid, AP_THREADS, smem, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}


template <int S, int BN, int TWR>
static hodlr_status run_apply(ApplyArgs g, cudaStream_t st) {
  constexpr size_t smem = (size_t)(S + (TWR > 0 ? 1 : 2) * BN + TWR) * (S + 4) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tri_apply_kernel<S, BN, TWR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int ntiles = (int)ceil_div(g.ncols, BN);
  // a CTA keeps its Tinv for up to 4 tiles; enough CTAs for >= 2 per SM
  g.groups = (int)std::max<int64_t>(1, ceil_div(ntiles, 4));
  if ((int64_t)g.batch * g.groups < 296) g.groups = ntiles;
  const int64_t grid = (int64_t)g.batch * g.groups;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  tri_apply_kernel<S, BN, TWR><<<(unsigned)grid, AP_THREADS, smem, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// fp32 leaf apply (cfg4): Y_b = U_b^-1 L_b^-1 P_b Y_b for s = 64 blocks of the
// fp32 LU, on the fp64 DMMA chain, optionally fused with TW_b = V_b^T Y_b
// (twr = 8).  ERR_ARG for other shapes / alignments (caller falls back).
hodlr_status tri_apply_f32(int s, int ncols, int batch, const float* lu, int64_t strideT, const int32_t* perm, float* Y,
                           int64_t ldy, int64_t sY, const float* V, int64_t ldv, int64_t vstride, int twr, float* TW,
                           int64_t tw_stride, cudaStream_t st) {
  if (batch == 0 || ncols == 0) return HODLR_OK;
  if (s != 64 || (V && twr != 8) || (ldy & 1) || (sY & 1) || (reinterpret_cast<uintptr_t>(Y) & 7) ||
      (TW && ((tw_stride & 1) || (reinterpret_cast<uintptr_t>(TW) & 7))))
    return HODLR_ERR_ARG;
  ApplyArgs g{nullptr, reinterpret_cast<const double*>(lu), 64, strideT, 0, perm, reinterpret_cast<const double*>(Y),
              ldy, sY, 0, reinterpret_cast<double*>(Y), ldy, sY, 0, ncols, batch, 1, 1,
              reinterpret_cast<const double*>(V), ldv, vstride, reinterpret_cast<double*>(TW), tw_stride};
  constexpr int S = 64, PT = Apply2Cfg<S>::PT;
  auto go = [&](auto kern, int twr_) -> hodlr_status {
    const size_t smem = (size_t)(S + twr_) * PT * sizeof(double) + (size_t)S * 8 * sizeof(double);
    smem_attr(kern, (int)smem);
    const int G = (int)ceil_div(ncols, 8);
    int cpb = 1;
    while ((int64_t)batch * cpb < 2 * 148 && cpb * 8 < G) cpb *= 2;
    g.groups = cpb;
    kern<<<(unsigned)((int64_t)batch * cpb), AP_THREADS, smem, st>>>(g);
    HODLR_CHECK_LAUNCH();
    return HODLR_OK;
  };
  return V ? go(tri_apply2_kernel<64, 8, float>, 8) : go(tri_apply2_kernel<64, 0, float>, 0);
}

// X_b = Tinv-apply(P_b B_b) for s in {16, 32, 64, 128}; returns ERR_ARG otherwise.
// With V != nullptr (s in {32, 64}, twr in {16, 32}) also writes the fused
// TW_b = V_b^T X_b reduction.
hodlr_status tri_apply_f64(int s, int ncols, int batch, const double* lu, const double* tinv, int64_t ldi, int64_t strideT,
                           const int32_t* perm, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double* X,
                           int64_t ldx, int64_t sX_hi, int64_t sX_lo, int bdiv, cudaStream_t st,
                           const double* V = nullptr, int64_t ldv = 0, int64_t vstride = 0, int twr = 0,
                           double* TW = nullptr, int64_t tw_stride = 0, int narrow_cols = 8) {
  if (batch == 0 || ncols == 0 || s == 0) return HODLR_OK;
  if ((ldi & 1) || (reinterpret_cast<uintptr_t>(tinv) & 15) || (strideT & 1)) return HODLR_ERR_ARG;
  ApplyArgs g{tinv, lu, ldi, strideT, inv_block_elems(s), perm, B, ldb, sB_hi, sB_lo, X, ldx, sX_hi, sX_lo, ncols, batch, bdiv, 1,
              V, ldv, vstride, TW, tw_stride};
  const bool narrow = ncols <= narrow_cols;
  if (s == 128) {  // diagonal-block-inverse format, no fused reduction
    if (V || lu == nullptr || (reinterpret_cast<uintptr_t>(tinv) & 15)) return HODLR_ERR_ARG;
    if (narrow && batch <= kStagedMaxBatch && apply_narrow_ok(g) && apply_staged_ok(g)) return run_apply_staged<128>(g, st);
    if (narrow && apply_narrow_ok(g)) return run_apply_narrow<128, 0>(g, st);
    if (!narrow && apply2_ok(g)) return run_apply2<128, 0>(g, st);
    return HODLR_ERR_ARG;
  }
  if (s == 32 || s == 64) {
    // diagonal-block-inverse format: blocked substitutions only (the caller
    // falls back to row substitution on ERR_ARG)
    if (lu == nullptr || (reinterpret_cast<uintptr_t>(tinv) & 15)) return HODLR_ERR_ARG;
    if (V) {
      if ((ldv & 1) || (vstride & 1) || (reinterpret_cast<uintptr_t>(V) & 15) || (twr != 16 && twr != 32 && twr != 64))
        return HODLR_ERR_ARG;
      if (narrow && apply_narrow_ok(g)) {
        if (s == 64)
          return twr == 64 ? run_apply_narrow<64, 64>(g, st)
                           : twr == 32 ? run_apply_narrow<64, 32>(g, st) : run_apply_narrow<64, 16>(g, st);
        if (twr == 64) return HODLR_ERR_ARG;
        return twr == 32 ? run_apply_narrow<32, 32>(g, st) : run_apply_narrow<32, 16>(g, st);
      }
      if (!narrow && apply2_ok(g)) {
        if (s == 64)
          return twr == 64 ? run_apply2<64, 64>(g, st) : twr == 32 ? run_apply2<64, 32>(g, st) : run_apply2<64, 16>(g, st);
        if (twr == 64) return HODLR_ERR_ARG;
        return twr == 32 ? run_apply2<32, 32>(g, st) : run_apply2<32, 16>(g, st);
      }
      return HODLR_ERR_ARG;
    }
    if (narrow && batch <= kStagedMaxBatch && apply_narrow_ok(g) && apply_staged_ok(g))
      return s == 64 ? run_apply_staged<64>(g, st) : run_apply_staged<32>(g, st);
    if (narrow && apply_narrow_ok(g)) return s == 64 ? run_apply_narrow<64, 0>(g, st) : run_apply_narrow<32, 0>(g, st);
    if (!narrow && apply2_ok(g)) return s == 64 ? run_apply2<64, 0>(g, st) : run_apply2<32, 0>(g, st);
    return HODLR_ERR_ARG;
  }
  // packed full-inverse format (s = 16)
  if (V) return HODLR_ERR_ARG;
  if (s == 16) return run_apply<16, 64, 0>(g, st);
  return HODLR_ERR_ARG;
}

}  // namespace hodlr
