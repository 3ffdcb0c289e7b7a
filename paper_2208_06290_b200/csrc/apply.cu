// Batched LU solve as two triangular DMMA GEMMs (backend.py:546-567 semantics):
//
//   X_b = U_b^-1 ( L_b^-1 ( P_b B_b ) )
//
// with the packed inverses Tinv_b = strict_lower(L^-1) + upper(U^-1) produced
// by the getrf kernels.  One CTA per (block, 64-column tile): the row-gathered
// tile P B is staged in shared memory, multiplied by the unit-lower factor
// (k < m masked, identity folded into the accumulator init), written back to
// shared memory, multiplied by the upper factor (k >= m masked) and stored
// coalesced.  X may alias B (the CTA reads its whole tile before writing).
// Used for the leaf solve of Y (Alg.3 l.3), K_p^-1 W (l.9) and both solve-
// phase applications (Alg.4 l.3, l.7).
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
  int ncols, batch, bdiv, tiles_n;
};

__device__ __forceinline__ int64_t aoff(int b, int bdiv, int64_t hi, int64_t lo) {
  return (int64_t)(b / bdiv) * hi + (int64_t)(b % bdiv) * lo;
}

template <int S, int BN>
__global__ void __launch_bounds__(128) tri_apply_kernel(ApplyArgs g) {
  constexpr int WM = S >= 32 ? S / 32 : 1;
  constexpr int WN = 4 / WM;
  constexpr int WTM = S / WM, WTN = BN / WN;
  constexpr int MI = WTM / 8, NI = WTN / 8;
  constexpr int P = S + 4;  // pitch: conflict-free fragment loads
  extern __shared__ __align__(16) double sm[];
  double* At = sm;          // [k][m]
  double* Bs = sm + S * P;  // [n][k]
  __shared__ int pm[S];

  const int b = blockIdx.x / g.tiles_n;
  const int n0 = (blockIdx.x % g.tiles_n) * BN;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int ar = lane >> 2, ac = lane & 3;

  const double* ti = g.tinv + (int64_t)b * g.strideT;
  for (int idx = t; idx < S * (S / 2); idx += 128) {
    const int k = idx / (S / 2), m = (idx % (S / 2)) * 2;
    cp_async_16(At + k * P + m, ti + m + (int64_t)k * g.ldi, 16);
  }
  if (t < S) pm[t] = g.perm[(int64_t)b * S + t];
  __syncthreads();
  const double* Bb = g.B + aoff(b, g.bdiv, g.sB_hi, g.sB_lo);
  for (int idx = t; idx < BN * S; idx += 128) {
    const int n = idx / S, k = idx % S;
    const int gn = n0 + n;
    const bool ok = gn < g.ncols;
    cp_async_8(Bs + n * P + k, ok ? Bb + pm[k] + (int64_t)gn * g.ldb : g.B, ok ? 8 : 0);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  double acc[MI][NI][2];
  // stage 1: T = P B + strict_lower(L^-1) P B
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = wm * WTM + i * 8 + ar, n = wn * WTN + j * 8 + ac * 2 + h;
        acc[i][j][h] = Bs[n * P + m];
      }
  for (int k0 = 0; k0 < (wm + 1) * WTM; k0 += 4) {
    const int k = k0 + ac;
    double af[MI], bf[NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = wm * WTM + i * 8 + ar;
      af[i] = (k < m) ? At[k * P + m] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) bf[j] = Bs[(wn * WTN + j * 8 + ar) * P + k];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = wm * WTM + i * 8 + ar, n = wn * WTN + j * 8 + ac * 2 + h;
        Bs[n * P + m] = acc[i][j][h];
        acc[i][j][h] = 0.0;
      }
  __syncthreads();
  // stage 2: X = upper(U^-1) T
  for (int k0 = wm * WTM; k0 < S; k0 += 4) {
    const int k = k0 + ac;
    double af[MI], bf[NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = wm * WTM + i * 8 + ar;
      af[i] = (k >= m) ? At[k * P + m] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) bf[j] = Bs[(wn * WTN + j * 8 + ar) * P + k];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = wm * WTM + i * 8 + ar, n = wn * WTN + j * 8 + ac * 2 + h;
        Bs[n * P + m] = acc[i][j][h];
      }
  __syncthreads();
  double* Xb = g.X + aoff(b, g.bdiv, g.sX_hi, g.sX_lo);
  for (int idx = t; idx < BN * S; idx += 128) {
    const int n = idx / S, m = idx % S;
    const int gn = n0 + n;
    if (gn < g.ncols) Xb[m + (int64_t)gn * g.ldx] = Bs[n * P + m];
  }
}

template <int S>
static hodlr_status run_apply(ApplyArgs g, cudaStream_t st) {
  constexpr int BN = 64;
  constexpr size_t smem = (size_t)(S + BN) * (S + 4) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tri_apply_kernel<S, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  g.tiles_n = (int)ceil_div(g.ncols, BN);
  const int64_t grid = (int64_t)g.batch * g.tiles_n;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  tri_apply_kernel<S, BN><<<(unsigned)grid, 128, smem, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// X_b = Tinv-apply(P_b B_b) for s in {16, 32, 64, 128}; returns ERR_ARG otherwise.
hodlr_status tri_apply_f64(int s, int ncols, int batch, const double* tinv, int64_t ldi, int64_t strideT,
                           const int32_t* perm, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double* X,
                           int64_t ldx, int64_t sX_hi, int64_t sX_lo, int bdiv, cudaStream_t st) {
  if (batch == 0 || ncols == 0 || s == 0) return HODLR_OK;
  if ((ldi & 1) || (reinterpret_cast<uintptr_t>(tinv) & 15) || (strideT & 1)) return HODLR_ERR_ARG;
  ApplyArgs g{tinv, ldi, strideT, perm, B, ldb, sB_hi, sB_lo, X, ldx, sX_hi, sX_lo, ncols, batch, bdiv, 0};
  switch (s) {
    case 16: return run_apply<16>(g, st);
    case 32: return run_apply<32>(g, st);
    case 64: return run_apply<64>(g, st);
    case 128: return run_apply<128>(g, st);
    default: return HODLR_ERR_ARG;
  }
}

}  // namespace hodlr
