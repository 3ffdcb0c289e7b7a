// HODLR matvec  y = A x  on the device (SPEC.md:183-191 [OP] matvec; the
// commented Alg. at): block-wise U (V^T x), two HBM
// streams over the unfactored representation.
//
//   A = blockdiag(D_a) + sum_{l'=1..L} sum_{sibling pairs (a,b)} [U_a V_b^T at (I_a, I_b); U_b V_a^T at (I_b, I_a)]
//
// pass 1 (matvec_proj_warp_kernel, m % 64 == 0; matvec_proj_kernel otherwise):
//   w^{l'}_c = V_c^T x_c for every child c of every level l' in one sweep over
//   the V slab.  A warp (or, in the generic kernel, a thread) walks one slab
//   column over a row segment of S rows, x staged in shared memory, and emits
//   w at each child boundary.  Children larger than S leave per-segment
//   partials that matvec_reduce_kernel sums in fixed segment order.
// pass 2 (matvec_apply_kernel): y(I) = D_a x(I_a) + sum_{l'} U(I, l') w^{l'}_{sib(c)};
//   warp = 64 rows, lane = 2 rows, U/D columns read as 16-byte (fp64) lane
//   pairs = one 512-byte line per warp per column, w broadcast from L2.
//
// Both passes are HBM-bound (0.25 flop/byte per right-hand side):
// bytes = es (m N + 2 r N L) + x / y traffic.  Per-column summation order
// depends only on the shape, never on nrhs (multi-RHS bitwise per column).
// Checked against the oracle's dense expansion (oracle/hodlr_oracle.py dense)
// and a torch einsum statement of the same sum (tests/test_gpu_matvec.py).
#include <climits>
#include <type_traits>

#include "common.cuh"
#include "ranks.cuh"

namespace hodlr {
namespace {

template <typename T>
struct V2;
template <>
struct V2<double> {
  using type = double2;
};
template <>
struct V2<float> {
  using type = float2;
};

// streaming (evict-first) vector loads: 4 consecutive scalars (32 B fp64 / 16 B fp32), 2 scalars
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcs(reinterpret_cast<const double2*>(p + 2));
  v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}
__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
}
template <typename T>
__device__ __forceinline__ void ld4(const T* p, T (&v)[1]) {
  v[0] = __ldcs(p);
}
template <typename T>
__device__ __forceinline__ void ld2(const T* p, T (&v)[2]) {
  const typename V2<T>::type a = __ldcs(reinterpret_cast<const typename V2<T>::type*>(p));
  v[0] = a.x, v[1] = a.y;
}
template <typename T>
__device__ __forceinline__ void ld2(const T* p, T (&v)[1]) {
  v[0] = __ldcs(p);
}

constexpr int kProjThreads = 256;
constexpr int kMaxSeg = 1024;  // rows per projection segment (bounded by a level's node size)

struct MvGeom {
  int64_t n;
  int m, r, L;
  int64_t seg;     // S: rows per projection segment (a level node size, divides N)
  int nseg;        // N / S
  int big0;        // levels l' < big0 have children larger than S (partials)
  int nrhs;
};

// w layout: level l' (1..L) child c at ((2^l' - 2) + c) * r * nrhs, then [rhs][j]
__device__ __forceinline__ int64_t w_off(int lv, int64_t c, int r, int nrhs) {
  return (((int64_t)1 << lv) - 2 + c) * (int64_t)r * nrhs;
}

// VW = rows per V load (4: vector path, m % 4 == 0 and aligned; 1: any m)
template <typename T, int NR, int VW>
__global__ void __launch_bounds__(kProjThreads) matvec_proj_kernel(MvGeom g, const T* __restrict__ V,
                                                                   const T* __restrict__ X, int64_t ldx,
                                                                   T* __restrict__ w, T* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char mv_smem[];
  T* xs = reinterpret_cast<T*>(mv_smem);  // [S][NR]
  const int seg = blockIdx.x;
  const int rt = blockIdx.y * NR;  // first rhs of this tile
  const int nr = min(NR, g.nrhs - rt);
  const int64_t row0 = (int64_t)seg * g.seg;
  for (int i = threadIdx.x; i < g.seg * NR; i += blockDim.x) {
    const int k = i / (int)g.seg, rr = i - k * (int)g.seg;
    xs[rr * NR + k] = k < nr ? X[row0 + rr + (int64_t)(rt + k) * ldx] : T(0);
  }
  __syncthreads();
  const int ncol = g.r * g.L;
  for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
    const int lv = col / g.r + 1, j = col - (lv - 1) * g.r;
    const int64_t nc = g.n >> lv;  // child rows at level lv
    const T* vp = V + (int64_t)col * g.n + row0;
    T acc[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) acc[k] = T(0);
    // children that end inside the segment emit w every nc rows; larger
    // children leave one partial per segment
    const bool emits = nc <= g.seg;
    const int steps_per_child = emits ? (int)(nc / VW) : INT_MAX;
    int64_t c = row0 / nc;
    int left = steps_per_child;
    auto step = [&](const T (&v)[VW], int i) {
      const T* xr = xs + i * NR;
#pragma unroll
      for (int k = 0; k < NR; ++k)
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[k] = fma(v[q], xr[q * NR + k], acc[k]);
      if (--left == 0) {
        T* wo = w + w_off(lv, c, g.r, g.nrhs) + (int64_t)rt * g.r + j;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          if (k < nr) wo[(int64_t)k * g.r] = acc[k];
          acc[k] = T(0);
        }
        ++c;
        left = steps_per_child;
      }
    };
    constexpr int G = 16 / VW;  // loads in flight per group (16 rows)
    int i = 0;
    for (; i + 16 <= (int)g.seg; i += 16) {
      T v[G][VW];
#pragma unroll
      for (int q = 0; q < G; ++q) ld4(vp + i + VW * q, v[q]);
#pragma unroll
      for (int q = 0; q < G; ++q) step(v[q], i + VW * q);
    }
    for (; i < (int)g.seg; i += VW) {
      T v[VW];
      ld4(vp + i, v);
      step(v, i);
    }
    if (!emits) {
      // partial slot: [level lv-1 (0..big0-2)][seg][rhs][j]
      T* po = part + (((int64_t)(lv - 1) * g.nseg + seg) * g.nrhs + rt) * g.r + j;
#pragma unroll
      for (int k = 0; k < NR; ++k)
        if (k < nr) po[(int64_t)k * g.r] = acc[k];
    }
  }
}

// Coalesced variant (m % 64 == 0, vector layout): warp = one slab column at a
// time, lane = 2 consecutive rows of every 64-row step (one 512-byte fp64 line
// per warp load), x staged [rhs][row] in shared memory, lane partials folded
// by a fixed xor butterfly at each child boundary (deterministic, nrhs-free).
template <typename T, int NR>
__global__ void __launch_bounds__(kProjThreads) matvec_proj_warp_kernel(MvGeom g, const T* __restrict__ V,
                                                                        const T* __restrict__ X, int64_t ldx,
                                                                        T* __restrict__ w, T* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char mv_smem[];
  T* xs = reinterpret_cast<T*>(mv_smem);  // [NR][S]
  const int seg = blockIdx.x;
  const int rt = blockIdx.y * NR;
  const int nr = min(NR, g.nrhs - rt);
  const int S = (int)g.seg;
  const int64_t row0 = (int64_t)seg * S;
  for (int i = threadIdx.x; i < S * NR; i += blockDim.x) {
    const int k = i / S, rr = i - k * S;
    xs[i] = k < nr ? X[row0 + rr + (int64_t)(rt + k) * ldx] : T(0);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int ncol = g.r * g.L;
  for (int col = warp; col < ncol; col += nwarp) {
    const int lv = col / g.r + 1, j = col - (lv - 1) * g.r;
    const int64_t nc = g.n >> lv;
    const T* vp = V + (int64_t)col * g.n + row0 + 2 * lane;
    const bool emits = nc <= S;
    const int steps_per_child = emits ? (int)(nc / 64) : INT_MAX;
    int64_t c = row0 / nc;
    int left = steps_per_child;
    T acc[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) acc[k] = T(0);
    auto flush = [&](T* dst, int64_t stride) {
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        T v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && k < nr) dst[(int64_t)k * stride] = v;
        acc[k] = T(0);
      }
    };
    auto step = [&](const T (&v)[2], int i) {
      const T* xr = xs + i + 2 * lane;
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        const typename V2<T>::type xv = *reinterpret_cast<const typename V2<T>::type*>(xr + k * S);
        acc[k] = fma(v[0], xv.x, acc[k]);
        acc[k] = fma(v[1], xv.y, acc[k]);
      }
      if (--left == 0) {
        flush(w + w_off(lv, c, g.r, g.nrhs) + (int64_t)rt * g.r + j, g.r);
        ++c;
        left = steps_per_child;
      }
    };
    int i = 0;
    for (; i + 256 <= S; i += 256) {  // four 64-row loads in flight per warp
      T v[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) ld2(vp + i + 64 * q, v[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q) step(v[q], i + 64 * q);
    }
    for (; i < S; i += 64) {
      T v[2];
      ld2(vp + i, v);
      step(v, i);
    }
    if (!emits) flush(part + (((int64_t)(lv - 1) * g.nseg + seg) * g.nrhs + rt) * g.r + j, g.r);
  }
}

// w^{l'}_c = sum over the child's segments (levels l' < big0): warp per output
// entry, lane q sums segments q, q + 32, ... in order, then a fixed xor
// butterfly (deterministic, independent of nrhs).
template <typename T>
__global__ void matvec_reduce_kernel(MvGeom g, const T* __restrict__ part, T* __restrict__ w, int64_t total) {
  const int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= total) return;
  const int64_t per = (int64_t)g.r * g.nrhs;  // [rhs][j] entries per child
  int64_t rem = idx;
  int lv = 1;
  while (rem >= (((int64_t)1 << lv) * per)) {
    rem -= ((int64_t)1 << lv) * per;
    ++lv;
  }
  const int64_t c = rem / per, e = rem - c * per;
  const int64_t spc = (g.n >> lv) / g.seg;  // segments per child
  const T* p = part + ((int64_t)(lv - 1) * g.nseg + c * spc) * per + e;
  T s = T(0);
  for (int64_t q = lane; q < spc; q += 32) s += p[q * per];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) w[w_off(lv, c, g.r, g.nrhs) + e] = s;
}

constexpr int kApplyWarps = 8;

// AW = rows per lane (2: vector path; 1: any m).  Warp = 32 AW rows.
template <typename T, int NR, int AW>
__global__ void __launch_bounds__(32 * kApplyWarps) matvec_apply_kernel(MvGeom g, const T* __restrict__ D,
                                                                        const T* __restrict__ U,
                                                                        const T* __restrict__ X, int64_t ldx,
                                                                        const T* __restrict__ w, T* __restrict__ Y,
                                                                        int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t i0 = ((int64_t)blockIdx.x * kApplyWarps + (threadIdx.x >> 5)) * (32 * AW) + AW * lane;
  if (i0 >= g.n) return;
  const int rt = blockIdx.y * NR;
  const int nr = min(NR, g.nrhs - rt);
  T a[AW][NR];
#pragma unroll
  for (int q = 0; q < AW; ++q)
#pragma unroll
    for (int k = 0; k < NR; ++k) a[q][k] = T(0);
  // leaf block: y(I_a) = D_a x(I_a)   (a lane's AW rows share a leaf: m % AW == 0)
  {
    const int64_t leaf = i0 / g.m;
    const int64_t ls = leaf * g.m;
    const T* dp = D + leaf * (int64_t)g.m * g.m + (i0 - ls);
    const T* xp = X + ls + (int64_t)rt * ldx;
#pragma unroll 8
    for (int kk = 0; kk < g.m; ++kk) {
      T dv[AW];
      ld2(dp + (int64_t)kk * g.m, dv);
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        const T xv = k < nr ? __ldg(xp + kk + (int64_t)k * ldx) : T(0);
#pragma unroll
        for (int q = 0; q < AW; ++q) a[q][k] = fma(dv[q], xv, a[q][k]);
      }
    }
  }
  // off-diagonal levels: y(I) += U(I, l') w^{l'}_{sibling}
  for (int lv = 1; lv <= g.L; ++lv) {
    const int64_t nc = g.n >> lv;
    const int64_t sib = (i0 / nc) ^ 1;
    const T* wp = w + w_off(lv, sib, g.r, g.nrhs) + (int64_t)rt * g.r;
    const T* up = U + (int64_t)(lv - 1) * g.r * g.n + i0;
#pragma unroll 8
    for (int j = 0; j < g.r; ++j) {
      T uv[AW];
      ld2(up + (int64_t)j * g.n, uv);
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        const T wv = k < nr ? __ldg(wp + (int64_t)k * g.r + j) : T(0);
#pragma unroll
        for (int q = 0; q < AW; ++q) a[q][k] = fma(uv[q], wv, a[q][k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k)
    if (k < nr) {
      T* yp = Y + i0 + (int64_t)(rt + k) * ldy;
#pragma unroll
      for (int q = 0; q < AW; ++q) yp[q] = a[q][k];
    }
}

MvGeom mv_geom(const hodlr_desc* d, int nrhs) {
  MvGeom g{};
  g.n = d->n;
  g.m = d->m;
  g.r = d->r;
  g.L = d->L;
  g.nrhs = nrhs;
  int64_t s = d->m;
  int k = 0;
  while (k < d->L && 2 * s <= kMaxSeg) {
    s *= 2;
    ++k;
  }
  g.seg = s;  // node size of level L - k: divides N
  g.nseg = (int)(d->n / s);
  g.big0 = d->L - k;  // levels l' < L - k have children of 2^(L - l') m > S rows
  return g;
}

// T-typed workspace: w (sum_l' 2^l' r nrhs) | partials (big0 - 1 levels x nseg x r nrhs)
size_t mv_ws_elems(const MvGeom& g) {
  const size_t wsz = (((size_t)1 << (g.L + 1)) - 2) * g.r * g.nrhs;
  const size_t psz = (size_t)std::max(g.big0 - 1, 0) * g.nseg * g.r * g.nrhs;
  return wsz + psz;
}

template <typename T, int NR, bool VEC>
hodlr_status mv_run(const MvGeom& g, const T* D, const T* U, const T* V, const T* X, int64_t ldx, T* Y, int64_t ldy,
                    T* ws, cudaStream_t st) {
  T* w = ws;
  T* part = ws + (((size_t)1 << (g.L + 1)) - 2) * g.r * g.nrhs;
  const int tiles = (int)ceil_div(g.nrhs, NR);
  if (g.r > 0 && g.L > 0) {
    const size_t smem = sizeof(T) * g.seg * NR;
    static const bool attr_set = [] {
      cudaFuncSetAttribute(matvec_proj_kernel<T, NR, VEC ? 4 : 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(T) * kMaxSeg * NR));
      cudaFuncSetAttribute(matvec_proj_warp_kernel<T, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(T) * kMaxSeg * NR));
      return true;
    }();
    (void)attr_set;
    if (VEC && g.m % 64 == 0) {
      matvec_proj_warp_kernel<T, NR><<<dim3(g.nseg, tiles), kProjThreads, smem, st>>>(g, V, X, ldx, w, part);
    } else {
      const int thr = (int)std::min<int64_t>(kProjThreads, ceil_div((int64_t)g.r * g.L, 32) * 32);
      matvec_proj_kernel<T, NR, VEC ? 4 : 1><<<dim3(g.nseg, tiles), thr, smem, st>>>(g, V, X, ldx, w, part);
    }
    HODLR_CHECK_LAUNCH();
    if (g.big0 > 1) {
      const int64_t total = ((((int64_t)1 << g.big0) - 2)) * g.r * g.nrhs;
      matvec_reduce_kernel<T><<<(unsigned)ceil_div(total * 32, 256), 256, 0, st>>>(g, part, w, total);
      HODLR_CHECK_LAUNCH();
    }
  }
  constexpr int AW = VEC ? 2 : 1;
  const int64_t ncta = ceil_div(g.n, 32 * AW * kApplyWarps);
  matvec_apply_kernel<T, NR, AW><<<dim3((unsigned)ncta, tiles), 32 * kApplyWarps, 0, st>>>(g, D, U, X, ldx, w, Y, ldy);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template <typename T, bool VEC>
hodlr_status mv_dispatch2(const MvGeom& g, const void* D, const void* U, const void* V, const void* X, int64_t ldx,
                          void* Y, int64_t ldy, void* ws, cudaStream_t st) {
  auto go = [&](auto nr) {
    return mv_run<T, decltype(nr)::value, VEC>(g, (const T*)D, (const T*)U, (const T*)V, (const T*)X, ldx, (T*)Y,
                                               ldy, (T*)ws, st);
  };
  if (g.nrhs == 1) return go(std::integral_constant<int, 1>{});
  if (g.nrhs == 2) return go(std::integral_constant<int, 2>{});
  if (g.nrhs <= 4) return go(std::integral_constant<int, 4>{});
  return go(std::integral_constant<int, 8>{});
}
template <typename T>
hodlr_status mv_dispatch(const MvGeom& g, bool vec, const void* D, const void* U, const void* V, const void* X,
                         int64_t ldx, void* Y, int64_t ldy, void* ws, cudaStream_t st) {
  return vec ? mv_dispatch2<T, true>(g, D, U, V, X, ldx, Y, ldy, ws, st)
             : mv_dispatch2<T, false>(g, D, U, V, X, ldx, Y, ldy, ws, st);
}

bool mv_shape_ok(const hodlr_desc* d) {
  if (!d || d->m < 1 || d->r < 0 || d->L < 0 || d->L > 30) return false;
  if (d->dtype != HODLR_F64 && d->dtype != HODLR_F32) return false;
  return d->n == (int64_t)d->m << d->L;
}

}  // namespace
}  // namespace hodlr

namespace hodlr {
hodlr_status gemm_f64(int transA, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sA_hi,
                      int64_t sA_lo, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double beta,
                      double* C, int64_t ldc, int64_t sC_hi, int64_t sC_lo, int batch, int bdiv, void* work,
                      size_t work_bytes, cudaStream_t st);
namespace {
constexpr size_t kMvSplitBytes = size_t(64) << 20;

// Per-level-rank (ragged) matvec: the batched DMMA GEMMs level by level --
// Y_a = D_a X_a, then per level w_c = V_c^T X_c and Y_c += U_c w_sibling(c).
// (The fused two-sweep kernels above assume one rank for every level.)
size_t mv_ragged_w_elems(const LevelRanks& q, int nrhs) {
  size_t e = 0;
  for (int l = 1; l <= q.L; ++l) e += ((size_t)1 << l) * q.r[l] * nrhs;
  return e;
}
hodlr_status mv_ragged(const hodlr_desc* d, const LevelRanks& q, const double* D, const double* U, const double* V,
                       const double* X, int64_t ldx, double* Y, int64_t ldy, int nrhs, char* ws, cudaStream_t st) {
  const int64_t N = d->n;
  const int m = d->m, L = d->L;
  void* split = ws;
  double* w = reinterpret_cast<double*>(ws + kMvSplitBytes);
  hodlr_status s = gemm_f64(0, m, nrhs, m, 1.0, D, m, (int64_t)m * m, 0, X, ldx, m, 0, 0.0, Y, ldy, m, 0, 1 << L, 1,
                            split, kMvSplitBytes, st);
  if (s != HODLR_OK) return s;
  for (int l = 1; l <= L; ++l) {
    const int k = q.r[l];
    if (k == 0) continue;
    const int64_t nl = N >> l;
    const int nb = 1 << l;
    s = gemm_f64(1, k, nrhs, (int)nl, 1.0, V + q.c[l] * N, N, nl, 0, X, ldx, nl, 0, 0.0, w, k, (int64_t)k * nrhs, 0,
                 nb, 1, split, kMvSplitBytes, st);
    if (s != HODLR_OK) return s;
    // child b reads its sibling's w: b = 2p -> w[2p + 1], b = 2p + 1 -> w[2p]
    const int64_t per = (int64_t)k * nrhs;
    s = gemm_f64(0, (int)nl, nrhs, k, 1.0, U + q.c[l] * N, N, 2 * nl, nl, w + per, k, 2 * per, -per, 1.0, Y, ldy, 2 * nl, nl,
                 nb, 2, split, kMvSplitBytes, st);
    if (s != HODLR_OK) return s;
  }
  return HODLR_OK;
}
}  // namespace
}  // namespace hodlr

using namespace hodlr;

extern "C" size_t hodlr_matvec_workspace(const hodlr_desc* d, int nrhs) {
  if (d && d->ranks) {
    LevelRanks q;
    if (!mv_shape_ok(d) || nrhs < 0 || d->dtype != HODLR_F64 || !make_ranks(d, q)) return 0;
    return kMvSplitBytes + ((mv_ragged_w_elems(q, std::max(nrhs, 1)) * sizeof(double) + 255) & ~(size_t)255);
  }
  if (!mv_shape_ok(d) || nrhs < 0) return 0;
  const MvGeom g = mv_geom(d, std::max(nrhs, 1));
  const size_t b = mv_ws_elems(g) * (d->dtype == HODLR_F64 ? sizeof(double) : sizeof(float));
  return (b + 255) & ~(size_t)255;
}

extern "C" hodlr_status hodlr_matvec(const hodlr_desc* d, const void* D, const void* U, const void* V, const void* X,
                                     int64_t ldx, void* Y, int64_t ldy, int nrhs, void* work, size_t work_bytes,
                                     void* stream) {
  if (!mv_shape_ok(d) || nrhs < 0 || ldx < d->n || ldy < d->n) return HODLR_ERR_ARG;
  if (nrhs == 0) return HODLR_OK;
  if (!D || !X || !Y || X == Y || (d->r > 0 && d->L > 0 && (!U || !V))) return HODLR_ERR_ARG;
  const size_t need = hodlr_matvec_workspace(d, nrhs);
  if (work_bytes < need || (need && !work)) return HODLR_ERR_ARG;
  if (d->ranks) {
    LevelRanks q;
    if (d->dtype != HODLR_F64 || !make_ranks(d, q) || !need) return HODLR_ERR_ARG;
    return mv_ragged(d, q, (const double*)D, (const double*)U, (const double*)V, (const double*)X, ldx, (double*)Y,
                     ldy, nrhs, static_cast<char*>(work), static_cast<cudaStream_t>(stream));
  }
  const size_t es = d->dtype == HODLR_F64 ? sizeof(double) : sizeof(float);
  // vector loads (V 4 scalars, U / D 2 scalars) when the layout allows them
  const bool vec = d->m % 4 == 0 && (uintptr_t)V % (4 * es) == 0 && (uintptr_t)U % (2 * es) == 0 &&
                   (uintptr_t)D % (2 * es) == 0;
  const MvGeom g = mv_geom(d, nrhs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d->dtype == HODLR_F32) return mv_dispatch<float>(g, vec, D, U, V, X, ldx, Y, ldy, work, st);
  return mv_dispatch<double>(g, vec, D, U, V, X, ldx, Y, ldy, work, st);
}
