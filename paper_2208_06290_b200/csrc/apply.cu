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
#include "common.cuh"

namespace hodlr {

struct ApplyArgs {
  const double* tinv;
  int64_t ldi, strideT;
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

  const double* ti = g.tinv + (int64_t)b * g.strideT;
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

// X_b = Tinv-apply(P_b B_b) for s in {16, 32, 64, 128}; returns ERR_ARG otherwise.
// With V != nullptr (s in {32, 64}, twr in {16, 32}) also writes the fused
// TW_b = V_b^T X_b reduction.
hodlr_status tri_apply_f64(int s, int ncols, int batch, const double* tinv, int64_t ldi, int64_t strideT,
                           const int32_t* perm, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double* X,
                           int64_t ldx, int64_t sX_hi, int64_t sX_lo, int bdiv, cudaStream_t st,
                           const double* V = nullptr, int64_t ldv = 0, int64_t vstride = 0, int twr = 0,
                           double* TW = nullptr, int64_t tw_stride = 0) {
  if (batch == 0 || ncols == 0 || s == 0) return HODLR_OK;
  if ((ldi & 1) || (reinterpret_cast<uintptr_t>(tinv) & 15) || (strideT & 1)) return HODLR_ERR_ARG;
  ApplyArgs g{tinv, ldi, strideT, perm, B, ldb, sB_hi, sB_lo, X, ldx, sX_hi, sX_lo, ncols, batch, bdiv, 1,
              V, ldv, vstride, TW, tw_stride};
  if (V) {
    if ((ldv & 1) || (vstride & 1) || (reinterpret_cast<uintptr_t>(V) & 15)) return HODLR_ERR_ARG;
    const bool nw = ncols <= 8;
    if (s == 64 && twr == 32) return nw ? run_apply<64, 8, 32>(g, st) : run_apply<64, 64, 32>(g, st);
    if (s == 64 && twr == 16) return nw ? run_apply<64, 8, 16>(g, st) : run_apply<64, 64, 16>(g, st);
    if (s == 32 && twr == 16) return run_apply<32, 64, 16>(g, st);
    if (s == 32 && twr == 32) return run_apply<32, 64, 32>(g, st);
    return HODLR_ERR_ARG;
  }
  const bool narrow = ncols <= 8;
  switch (s) {
    case 16: return run_apply<16, 64, 0>(g, st);
    case 32: return narrow ? run_apply<32, 8, 0>(g, st) : run_apply<32, 64, 0>(g, st);
    case 64: return narrow ? run_apply<64, 8, 0>(g, st) : run_apply<64, 64, 0>(g, st);
    case 128: return narrow ? run_apply<128, 8, 0>(g, st) : run_apply<128, 32, 0>(g, st);
    default: return HODLR_ERR_ARG;
  }
}

}  // namespace hodlr
