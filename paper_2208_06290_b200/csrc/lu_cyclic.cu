// Batched bit-exact LU kernels (register-row and shared-row) + triangular inverses.
//
// Replays backend.py:444-478 (_lu_factor_stack) exactly: right-looking,
// first-max pivot over |a[k:, k]| (NaN wins, smallest logical index on ties),
// whole-row exchange, singular guard |piv| <= eps*s*max|orig col k|, true
// division by the pivot (0 -> 1), trailing update a - (l*u) with the product
// rounded before the subtraction (__dmul_rn / __dsub_rn, no FMA).
//
// getrf_reg_kernel (fp64/fp32, s in {32, 64}): thread t owns row t in registers,
// fully unrolled steps -- full waves of blocks (leaf LUs, deep K levels).
// getrf_sr_kernel (any s <= 128): thread t owns row t in shared memory with a
// runtime step loop -- small batches (top K levels) and s = 16 / 128.
// Row exchanges are logical (each row carries its logical position), which is
// the reference's physical swap with the same per-element operation sequence.
//
// Solve aids: the 8x8 diagonal-block inverses (diag_block_inverses, the
// blocked DMMA substitutions of apply.cu) or, for the batched-kernel API, the
// packed triangular inverses Tinv = strict_lower(L^-1) + upper(U^-1) formed in
// shared memory by recursive doubling (packed_trtri: 8x8 diagonal blocks per
// thread-row, each doubling step two small DMMA GEMMs).
#include <cstdlib>

#include "common.cuh"
#include "lu_device.cuh"

namespace hodlr {

template <typename T>
__device__ __forceinline__ bool cyc_beats(T v, int pv, T b, int pb) {
  if (pv < 0) return false;
  if (pb < 0) return true;
  const bool vn = v != v, bn = b != b;
  if (vn || bn) return (vn && bn) ? pv < pb : vn;
  return v > b || (v == b && pv < pb);
}



// opaque select (keeps register arrays in registers)
__device__ __forceinline__ double csel(int p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}" : "=d"(r) : "d"(a), "d"(b), "r"(p));
  return r;
}
__device__ __forceinline__ float csel(int p, float a, float b) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n\t}" : "=f"(r) : "f"(a), "f"(b), "r"(p));
  return r;
}

// C(8x8 tiles) = fa * fb over K, tiles spread over the CTA's warps; fo(i, j, v)
// consumes the result.  DMMA for double, scalar FMA for float.
template <typename T, class FA, class FB, class FO>
__device__ __forceinline__ void tile_gemm(int M, int N, int K, FA fa, FB fb, FO fo) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ntile = (M / 8) * (N / 8);
  for (int tile = warp; tile < ntile; tile += nw) {
    const int tm = (tile % (M / 8)) * 8, tn = (tile / (M / 8)) * 8;
    if constexpr (sizeof(T) == 8) {
      double c0 = 0.0, c1 = 0.0;
      const int ar = lane >> 2, ac = lane & 3;
      for (int k0 = 0; k0 < K; k0 += 4) dmma_8x8x4(c0, c1, fa(tm + ar, k0 + ac), fb(k0 + ac, tn + ar));
      fo(tm + ar, tn + 2 * ac, (T)c0);
      fo(tm + ar, tn + 2 * ac + 1, (T)c1);
    } else {
      for (int e = lane; e < 64; e += 32) {
        const int i = tm + (e & 7), j = tn + (e >> 3);
        T s = 0;
        for (int k = 0; k < K; ++k) s = fma(fa(i, k), fb(k, j), s);
        fo(i, j, s);
      }
    }
  }
}

// In-place packed triangular inversion of the S x S LU in shared memory (column-
// major, pitch P): upper(U) -> upper(U^-1), strict_lower(L) -> strict_lower(L^-1).
// Tt: (S/2) x (S/2) scratch.  Works for any CTA size (multiple of 32).
template <typename T, int S>
__device__ void packed_trtri(T* Tm, T* Tt, int P) {
  // ---- packed inverses, level 0: 8x8 diagonal blocks (thread = (block, row, U/L)) ----
  __shared__ T rdiag[S];
  const int t = threadIdx.x, nt = blockDim.x;
  for (int u = t; u < S; u += nt) rdiag[u] = (T)1 / Tm[u + u * P];
  __syncthreads();
  for (int u0 = 0; u0 < 2 * S; u0 += nt) {
    const int u = u0 + t;
    const int q = (u >> 3) & (S / 8 - 1), i = u & 7, which = u / S;  // which: 0 = U, 1 = L
    T x[8];
    if (u < 2 * S) {
      const int o0 = 8 * q;
      if (which == 0) {  // row i of inv(U_qq)
        const T dii = rdiag[o0 + i];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = (j == i) ? dii : (T)0;
#pragma unroll
        for (int j = 1; j < 8; ++j) {
          if (j > i) {
            T s = (T)0;
#pragma unroll
            for (int kk = 0; kk < j; ++kk)
              if (kk >= i) s = fma(x[kk], Tm[(o0 + kk) + (o0 + j) * P], s);
            x[j] = -s * rdiag[o0 + j];
          }
        }
      } else {  // row i of inv(L_qq), unit diagonal
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = (T)(j == i);
#pragma unroll
        for (int j = 6; j >= 0; --j) {
          if (j < i) {
            T s = (T)0;
#pragma unroll
            for (int kk = 1; kk < 8; ++kk)
              if (kk > j && kk <= i) s = fma(x[kk], Tm[(o0 + kk) + (o0 + j) * P], s);
            x[j] = -s;
          }
        }
      }
    }
    __syncthreads();
    if (u < 2 * S) {
      const int o0 = 8 * q;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (which == 0 ? (j >= i) : (j < i)) Tm[(o0 + i) + (o0 + j) * P] = x[j];
      }
    }
    __syncthreads();
  }
  // ---- doubling: h = 8, 16, ..., S/2 ----
  constexpr int PT = S / 2 + 4;
  for (int h = 8; h < S; h *= 2) {
    for (int o0 = 0; o0 < S; o0 += 2 * h) {
      const int a0 = o0, b0 = o0 + h;
      // U: Tt = U_AB * inv(B) (inv(B) upper: k <= n)
      tile_gemm<T>(
          h, h, h, [&](int i, int k) { return Tm[(a0 + i) + (b0 + k) * P]; },
          [&](int k, int n) { return k <= n ? Tm[(b0 + k) + (b0 + n) * P] : (T)0; },
          [&](int i, int n, T v) { Tt[i + n * PT] = v; });
      __syncthreads();
      // U: X = -inv(A) * Tt (inv(A) upper: k >= i)
      tile_gemm<T>(
          h, h, h, [&](int i, int k) { return k >= i ? Tm[(a0 + i) + (a0 + k) * P] : (T)0; },
          [&](int k, int n) { return Tt[k + n * PT]; }, [&](int i, int n, T v) { Tm[(a0 + i) + (b0 + n) * P] = -v; });
      __syncthreads();
      // L: Tt = C * inv(A) (inv(A) unit lower: strict part k > n, plus identity)
      tile_gemm<T>(
          h, h, h, [&](int i, int k) { return Tm[(b0 + i) + (a0 + k) * P]; },
          [&](int k, int n) { return k > n ? Tm[(a0 + k) + (a0 + n) * P] : (T)(k == n); },
          [&](int i, int n, T v) { Tt[i + n * PT] = v; });
      __syncthreads();
      // L: X = -inv(B) * Tt (inv(B) unit lower)
      tile_gemm<T>(
          h, h, h, [&](int i, int k) { return k < i ? Tm[(b0 + i) + (b0 + k) * P] : (T)(k == i); },
          [&](int k, int n) { return Tt[k + n * PT]; }, [&](int i, int n, T v) { Tm[(b0 + i) + (a0 + n) * P] = -v; });
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Shared-memory row LU: thread t owns row t of the block, stored row-major in
// shared memory (pitch S+2: conflict-free 16B accesses across threads).  The
// step loop runs at runtime (no unrolling): each active thread forms its own
// multiplier l = a_tk / piv and updates its row in place, reading the pivot
// row straight from shared memory -- the pivot row is final once chosen, so
// one barrier per step (the cross-warp argmax) orders everything.  Same IEEE
// operation sequence per element as the reference.
// ---------------------------------------------------------------------------
template <typename T, int S>
__global__ void __launch_bounds__(S < 32 ? 32 : S) getrf_sr_kernel(int mode, const T* __restrict__ src, int64_t lds,
                                                                 int64_t strides, T* out, int64_t ldo,
                                                                 int64_t strideo, int32_t* __restrict__ swaps,
                                                                 int32_t* __restrict__ perm,
                                                                 int32_t* __restrict__ info, T* __restrict__ tinv,
                                                                 int64_t ldi, int64_t stridei, int dbi = 0) {
  constexpr int NT = S < 32 ? 32 : S;
  constexpr int NW = NT / 32;
  constexpr int RP = S + 16 / (int)sizeof(T);  // row pitch: 16B-aligned rows, 16B bank shift per row
  extern __shared__ __align__(16) unsigned char sr_smem[];
  T* A = reinterpret_cast<T*>(sr_smem);  // S rows x RP
  __shared__ T cmax[S];
  __shared__ unsigned redh[2][NW], redl[2][NW];
  __shared__ int redp[2][NW];
  __shared__ int swk[S];
  __shared__ int sflag;

  const int64_t blk = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool live = t < S;
  const T* g = src + blk * strides;
  T* row = A + t * RP;
  if (live) {  // 16 independent loads in flight per thread
    constexpr int CH = S < 16 ? S : 16;
    for (int j0 = 0; j0 < S; j0 += CH) {
      T v[CH];
#pragma unroll
      for (int jj = 0; jj < CH; ++jj) {
        const int j = j0 + jj;
        if (mode == 0) {
          v[jj] = g[t + j * lds];
        } else {
          constexpr int R = S / 2;
          if (t < R && j < R)
            v[jj] = g[t + j * lds];
          else if (t >= R && j >= R)
            v[jj] = g[t + (j - R) * lds];
          else
            v[jj] = (t < R) ? (T)(t == j - R) : (T)(t - R == j);
        }
      }
#pragma unroll
      for (int jj = 0; jj < CH; ++jj) row[j0 + jj] = v[jj];
    }
  }
  if (t == 0) sflag = 0;
  __syncthreads();
  if (live) {  // thread t: max |a_it| over the original column t (NaN-propagating)
    T m0 = (T)0, m1 = (T)0, m2 = (T)0, m3 = (T)0;
#pragma unroll 4
    for (int i = 0; i < S; i += 4) {
      m0 = cyc_nanmax(m0, (T)fabs((double)A[i * RP + t]));
      m1 = cyc_nanmax(m1, (T)fabs((double)A[(i + 1) * RP + t]));
      m2 = cyc_nanmax(m2, (T)fabs((double)A[(i + 2) * RP + t]));
      m3 = cyc_nanmax(m3, (T)fabs((double)A[(i + 3) * RP + t]));
    }
    cmax[t] = cyc_nanmax(cyc_nanmax(m0, m1), cyc_nanmax(m2, m3));
  }
  const T thr_scale = mul_rn(Eps<T>::v, (T)S);
  int pos = t;
  bool active = live;
  for (int k = 0; k < S; ++k) {
    const int buf = k & 1;
    unsigned kh = 0u, kl = 0u;
    int pv = 0x7fffffff;  // (logical position << 8) | thread: unique, orders by position
    if (active) {
      abs_key(row[k], kh, kl);
      pv = (pos << 8) | t;
    }
    warp_argmax(kh, kl, pv);
    if (NW > 1) {
      if (lane == 0) {
        redh[buf][warp] = kh;
        redl[buf][warp] = kl;
        redp[buf][warp] = pv;
      }
      __syncthreads();
      kh = redh[buf][0];
      kl = redl[buf][0];
      pv = redp[buf][0];
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        const unsigned h2 = redh[buf][w], l2 = redl[buf][w];
        const int p2 = redp[buf][w];
        if (h2 > kh || (h2 == kh && (l2 > kl || (l2 == kl && p2 < pv)))) {
          kh = h2;
          kl = l2;
          pv = p2;
        }
      }
    } else {
      __syncwarp();
    }
    const int pt = pv & 255;
    pv >>= 8;
    const T* prow = A + pt * RP;
    const T piv = prow[k];
    if (t == 0) {
      swk[k] = pv;
      if ((T)fabs((double)piv) <= mul_rn(thr_scale, cmax[k])) sflag = 1;
    }
    if (pos == k) pos = pv;
    if (t == pt) {
      pos = k;
      active = false;
    }
    if (active) {
      const T d = (piv == (T)0) ? (T)1 : piv;
      const T x = row[k];
      const T l = (x == (T)0 && d == d) ? ((signbit(x) != signbit(d)) ? (T)-0.0 : (T)0.0) : div_rn(x, d);
      row[k] = l;
      int j = k + 1;
      if (j & 1) {  // align to 16B pairs
        if (j < S) row[j] = sub_rn(row[j], mul_rn(l, prow[j]));
        ++j;
      }
      if constexpr (sizeof(T) == 8) {
        // the pivot row is never this thread's row: load 8-wide chunks of both
        // before storing so the loads are not serialised behind the stores
        const double2* __restrict__ pu = reinterpret_cast<const double2*>(prow);
        double2* __restrict__ pa = reinterpret_cast<double2*>(row);
        int jj = j >> 1;
        for (; jj + 4 <= S / 2; jj += 4) {
          double2 u[4], a[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            u[q] = pu[jj + q];
            a[q] = pa[jj + q];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[q].x = sub_rn(a[q].x, mul_rn(l, u[q].x));
            a[q].y = sub_rn(a[q].y, mul_rn(l, u[q].y));
            pa[jj + q] = a[q];
          }
        }
        for (; jj < S / 2; ++jj) {
          const double2 u = pu[jj];
          double2 a = pa[jj];
          a.x = sub_rn(a.x, mul_rn(l, u.x));
          a.y = sub_rn(a.y, mul_rn(l, u.y));
          pa[jj] = a;
        }
      } else {
#pragma unroll 4
        for (; j < S; ++j) row[j] = sub_rn(row[j], mul_rn(l, prow[j]));
      }
    }
  }
  __syncthreads();
  T* o = out + blk * strideo;
  if (live) {
    for (int j = 0; j < S; ++j) o[pos + j * ldo] = row[j];
    perm[blk * S + pos] = t;
    swaps[blk * S + t] = swk[t];
  }
  if (t == 0) info[blk] = sflag;
  if (tinv == nullptr) return;
  // packed inverses: stage the logical LU column-major (reuse the row buffer)
  constexpr int P = S + 4;
  __syncthreads();  // global LU writes visible to the block; row buffer free after this
  T* Tm = A;
  T* Tt = A + S * P;
  for (int idx0 = 0; idx0 < S * S; idx0 += 8 * NT) {  // 8 loads in flight (L2-resident)
    T v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = idx0 + q * NT + t;
      v[q] = idx < S * S ? o[idx % S + (idx / S) * ldo] : (T)0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = idx0 + q * NT + t;
      if (idx < S * S) Tm[idx % S + (idx / S) * P] = v[q];
    }
  }
  __syncthreads();
  if constexpr (sizeof(T) == 8) {
    if (dbi) {  // diagonal-block inverses (blocked DMMA substitutions) instead of full inverses
      diag_block_inverses<S>(reinterpret_cast<const double*>(Tm), 1, P, reinterpret_cast<double*>(tinv) + blk * stridei);
      return;
    }
  }
  packed_trtri<T, S>(Tm, Tt, P);
  T* ti = tinv + blk * stridei;
  for (int idx = t; idx < S * S; idx += NT) {
    const int i = idx % S, j = idx / S;
    ti[i + (int64_t)j * ldi] = Tm[i + j * P];
  }
}

// ---------------------------------------------------------------------------
// Register-row LU (fp64, S in {32, 64}): thread t owns row t of the block in
// registers for the whole factorization (the trailing update never touches
// shared memory for its own operands).  Same IEEE operation sequence per
// element as backend.py:444-478 (see getrf_sr_kernel).  One barrier per step:
// every warp publishes the row of its own argmax winner (parity-buffered)
// together with its key, so after the barrier each thread reads the global
// pivot row straight from the winning warp's slot.  The step loop is fully
// unrolled: every register column index and every "j > k" test is a
// compile-time constant, so a step is the argmax, the exchange, one division
// and exactly (S-1-k) multiply/subtract pairs.  The packed triangular
// inverses are formed by a separate kernel (trtri_sm_kernel).
// ---------------------------------------------------------------------------

template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

template <int S, typename T = double>
__global__ void __launch_bounds__(S, S == 64 ? (sizeof(T) == 8 ? 6 : 10) : 16)
    getrf_reg_kernel(int mode, const T* __restrict__ src, int64_t lds, int64_t strides, T* out, int64_t ldo,
                     int64_t strideo, int32_t* __restrict__ swaps, int32_t* __restrict__ perm,
                     int32_t* __restrict__ info, double* __restrict__ dbi, int64_t stridedbi) {
  using V2 = typename Vec2<T>::type;
  constexpr int NW = S / 32, RP = S + 1;
  __shared__ T A[S * RP];                     // staging (row-major, odd pitch)
  __shared__ __align__(16) T urow[2][NW][S];  // per-warp candidate pivot rows
  __shared__ T cmax[S];
  __shared__ unsigned redh[2][NW], redl[2][NW];
  __shared__ int redp[2][NW];
  __shared__ int swk[S];
  __shared__ int sflag;

  const int64_t blk = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const T* g = src + blk * strides;
  // ---- stage: coalesced column reads -> row-major smem (16 loads in flight per
  // thread: the top-level single-block factorizations are load-latency bound) ----
  {
    const int i = t;  // thread t stages row i = t of every column j
#pragma unroll
    for (int j0 = 0; j0 < S; j0 += 16) {
      T v[16];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = j0 + jj;
        if (mode == 0) {
          v[jj] = g[i + (int64_t)j * lds];
        } else {
          constexpr int R = S / 2;
          if (i < R && j < R)
            v[jj] = g[i + (int64_t)j * lds];
          else if (i >= R && j >= R)
            v[jj] = g[i + (int64_t)(j - R) * lds];
          else
            v[jj] = (i < R) ? (T)(i == j - R) : (T)(i - R == j);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) A[i * RP + j0 + jj] = v[jj];
    }
  }
  if (t == 0) sflag = 0;
  __syncthreads();
  {  // thread t: max |a_it| over the original column t (NaN-propagating)
    T m0 = (T)0, m1 = (T)0;
#pragma unroll 8
    for (int i = 0; i < S; i += 2) {
      m0 = cyc_nanmax(m0, (T)fabs((double)A[i * RP + t]));
      m1 = cyc_nanmax(m1, (T)fabs((double)A[(i + 1) * RP + t]));
    }
    cmax[t] = cyc_nanmax(m0, m1);
  }
  T a[S];
#pragma unroll
  for (int j = 0; j < S; ++j) a[j] = A[t * RP + j];
  __syncthreads();  // cmax visible

  const T thr_scale = mul_rn(Eps<T>::v, (T)S);
  int pos = t;
  bool active = true;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int par = k & 1;
    const T ak = a[k];
    unsigned kh = 0u, kl = 0u;
    int pv = 0x7fffffff;
    if (active) {
      abs_key(ak, kh, kl);
      pv = (pos << 8) | t;
    }
    warp_argmax(kh, kl, pv);
    if (pv != 0x7fffffff && (pv & 255) == t) {
      T* ur = urow[par][warp];
#pragma unroll
      for (int j = k & ~1; j < S; j += 2) *reinterpret_cast<V2*>(ur + j) = V2{a[j], a[j + 1]};
    }
    if (lane == 0) {
      redh[par][warp] = kh;
      redl[par][warp] = kl;
      redp[par][warp] = pv;
    }
    __syncthreads();
    int ww = 0;
    if (NW > 1) {
      kh = redh[par][0];
      kl = redl[par][0];
      pv = redp[par][0];
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        const unsigned h2 = redh[par][w], l2 = redl[par][w];
        const int p2 = redp[par][w];
        if (h2 > kh || (h2 == kh && (l2 > kl || (l2 == kl && p2 < pv)))) {
          kh = h2;
          kl = l2;
          pv = p2;
          ww = w;
        }
      }
    }
    const int pt = pv & 255;
    pv >>= 8;
    const T* u = urow[par][ww];
    const T piv = u[k];
    if (t == 0) {
      swk[k] = pv;
      if ((T)fabs((double)piv) <= mul_rn(thr_scale, cmax[k])) sflag = 1;
    }
    if (pos == k) pos = pv;
    if (t == pt) {
      pos = k;
      active = false;
    }
    if (active) {
      const T d = (piv == (T)0) ? (T)1 : piv;
      const T l = (ak == (T)0 && d == d) ? ((signbit(ak) != signbit(d)) ? (T)-0.0 : (T)0.0) : div_rn(ak, d);
      a[k] = l;
      if ((k & 1) == 0 && k + 1 < S) a[k + 1] = sub_rn(a[k + 1], mul_rn(l, u[k + 1]));
#pragma unroll
      for (int j = (k + 2) & ~1; j < S; j += 2) {
        const V2 uu = *reinterpret_cast<const V2*>(u + j);
        a[j] = sub_rn(a[j], mul_rn(l, uu.x));
        a[j + 1] = sub_rn(a[j + 1], mul_rn(l, uu.y));
      }
    }
  }
  // ---- outputs: rows to their logical positions (through smem), pivots, flag ----
#pragma unroll
  for (int j = 0; j < S; ++j) A[pos * RP + j] = a[j];
  perm[blk * S + pos] = t;
  __syncthreads();
  T* o = out + blk * strideo;
  for (int idx = t; idx < S * S; idx += S) {
    const int i = idx % S, j = idx / S;
    o[i + (int64_t)j * ldo] = A[i * RP + j];
  }
  swaps[blk * S + t] = swk[t];
  if (t == 0) info[blk] = sflag;
  if constexpr (sizeof(T) == 8) {
    if (dbi == nullptr) return;
    // ---- diagonal-block inverses (the blocked triangular solves' 8x8 pivots) ----
    diag_block_inverses<S>(A, RP, 1, dbi + blk * stridedbi);
  }
}

// Packed triangular inverses of already-factored blocks (L2-hot right after
// getrf_reg_kernel): stage column-major, packed_trtri, store.
template <int S>
__global__ void __launch_bounds__(128) trtri_sm_kernel(const double* __restrict__ LU, int64_t ldl, int64_t stridel,
                                                       double* __restrict__ tinv, int64_t ldi, int64_t stridei) {
  constexpr int P = S + 4;
  extern __shared__ __align__(16) unsigned char tr_smem[];
  double* Tm = reinterpret_cast<double*>(tr_smem);
  double* Tt = Tm + S * P;
  const int64_t blk = blockIdx.x;
  const double* l = LU + blk * stridel;
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) {
    const int i = idx % S, j = idx / S;
    Tm[i + j * P] = l[i + (int64_t)j * ldl];
  }
  __syncthreads();
  packed_trtri<double, S>(Tm, Tt, P);
  double* ti = tinv + blk * stridei;
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) {
    const int i = idx % S, j = idx / S;
    ti[i + (int64_t)j * ldi] = Tm[i + j * P];
  }
}

template <int S>
static hodlr_status run_trtri_sm(int batch, const double* out, int64_t ldo, int64_t strideo, double* tinv, int64_t ldi,
                                 int64_t stridei, cudaStream_t st) {
  constexpr size_t smem = ((size_t)S * (S + 4) + (size_t)(S / 2) * (S / 2 + 4)) * sizeof(double);
  smem_attr(trtri_sm_kernel<S>, (int)smem);
  trtri_sm_kernel<S><<<batch, 128, smem, st>>>(out, ldo, strideo, tinv, ldi, stridei);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

hodlr_status launch_getrf_wide(int s, int batch, int mode, const double* src, int64_t lds, int64_t strides,
                               double* out, int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info,
                               double* dbi, int64_t stridedbi, cudaStream_t st);

// batches up to this many blocks take the latency-optimised column-owner LU
// (lu_wide.cu); larger ones the throughput kernels.  Measured single-launch
// times (tools/lu_latency.py): s = 64: 35 us (1 block) / 41 us (296) vs the
// window kernel's 52 / 56 us, 74 vs 67 us at 512; s = 128 (every batch): 122 /
// 245 us at 148 / 296 blocks vs the shared-row kernel's 178 / 346 us, and
// 1.7 ms vs 2.3 ms (est.) at 2048 (profiles/r02_lu_col.txt)
#ifndef HODLR_WIDE_LU_BATCH
#define HODLR_WIDE_LU_BATCH 296
#endif
constexpr int kWideLuBatch = HODLR_WIDE_LU_BATCH;
static int wide_lu_batch(int s) { return s >= 128 ? (kWideLuBatch > 0 ? 1 << 30 : 0) : kWideLuBatch; }
#define TRY_STATUS(x)                     \
  do {                                    \
    const hodlr_status s_ = (x);          \
    if (s_ != HODLR_OK) return s_;        \
  } while (0)

template <int S>
static hodlr_status run_reg(int batch, int mode, const double* src, int64_t lds, int64_t strides, double* out,
                            int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, double* tinv,
                            int64_t ldi, int64_t stridei, cudaStream_t st) {
  getrf_reg_kernel<S><<<batch, S, 0, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, nullptr, 0);
  HODLR_CHECK_LAUNCH();
  if (tinv == nullptr) return HODLR_OK;
  return run_trtri_sm<S>(batch, out, ldo, strideo, tinv, ldi, stridei, st);
}

// Factorization-internal LU (fp64, s in {32, 64}): factors + diagonal-block
// inverses (8 s doubles per block at dbi + b * stridedbi) instead of the
// packed full inverses -- the apply kernels run blocked substitutions.
// s = 64 batches up to this size use the sliding-window kernel, larger ones the
// register-row kernel (tools/micro/lu_win_bench: window 1.12-1.34x faster up
// to 2048 blocks, 0.96x at 8192)
constexpr int kSmallLuBatch = 2048;
static int small_lu_batch() { return kSmallLuBatch; }

template <typename T>
hodlr_status launch_getrf_win(int s, int batch, int mode, const T* src, int64_t lds, int64_t strides, T* out,
                              int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, double* dbi,
                              int64_t stridedbi, cudaStream_t st);

hodlr_status launch_getrf_dbi_f64(int s, int batch, int mode, const double* src, int64_t lds, int64_t strides,
                                  double* out, int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm,
                                  int32_t* info, double* dbi, int64_t stridedbi, cudaStream_t st) {
  if (batch == 0) return HODLR_OK;
  if ((s == 32 || s == 64 || s == 128) && batch <= wide_lu_batch(s))
    return launch_getrf_wide(s, batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, dbi, stridedbi,
                             st);
  if (s == 64 && batch <= small_lu_batch())
    // less than a few waves of blocks: per-block step latency decides -- the
    // compact sliding-window kernel (lu_win.cu; 1.2-1.3x faster than the
    // shared-row kernel for 1..2048 blocks, same bits); full waves: register rows
    return launch_getrf_win<double>(s, batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, dbi,
                                    stridedbi, st);
  if (s == 64)
    getrf_reg_kernel<64><<<batch, 64, 0, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, dbi,
                                              stridedbi);
  else if (s == 32)
    getrf_reg_kernel<32><<<batch, 32, 0, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, dbi,
                                              stridedbi);
  else if (s == 128) {
    constexpr int S = 128, RP = S + 2;
    constexpr size_t rows = (size_t)S * RP * sizeof(double);
    constexpr size_t inv = ((size_t)S * (S + 4) + (size_t)(S / 2) * (S / 2 + 4)) * sizeof(double);
    constexpr size_t smem = rows > inv ? rows : inv;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(getrf_sr_kernel<double, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    getrf_sr_kernel<double, S><<<batch, S, smem, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info,
                                                         dbi, 0, stridedbi, 1);
  } else
    return HODLR_ERR_ARG;
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

// s in {32, 64}: the register-row kernel (fp64 with packed inverses; fp32
// without) -- measured faster than the shared-row kernel for full waves
static int lu_variant() { return 1; }

template <typename T, int S>
static hodlr_status run_sr(int batch, int mode, const T* src, int64_t lds, int64_t strides, T* out, int64_t ldo,
                           int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, T* tinv, int64_t ldi,
                           int64_t stridei, cudaStream_t st) {
  constexpr int RP = S + 16 / (int)sizeof(T);
  constexpr size_t rows = (size_t)S * RP * sizeof(T);
  constexpr size_t inv = ((size_t)S * (S + 4) + (size_t)(S / 2) * (S / 2 + 4)) * sizeof(T);
  constexpr size_t smem = rows > inv ? rows : inv;
  constexpr int NT = S < 32 ? 32 : S;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(getrf_sr_kernel<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  getrf_sr_kernel<T, S><<<batch, NT, smem, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv,
                                                  ldi, stridei);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template <typename T>
hodlr_status launch_getrf_cyclic(int s, int batch, int mode, const T* src, int64_t lds, int64_t strides, T* out,
                                 int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, T* tinv,
                                 int64_t ldi, int64_t stridei, cudaStream_t st) {
  if constexpr (sizeof(T) == 8) {
    if ((s == 32 || s == 64 || s == 128) && batch <= wide_lu_batch(s)) {
      TRY_STATUS(launch_getrf_wide(s, batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, nullptr, 0, st));
      if (tinv == nullptr) return HODLR_OK;
      return s == 32 ? run_trtri_sm<32>(batch, out, ldo, strideo, tinv, ldi, stridei, st)
             : s == 64 ? run_trtri_sm<64>(batch, out, ldo, strideo, tinv, ldi, stridei, st)
                       : run_trtri_sm<128>(batch, out, ldo, strideo, tinv, ldi, stridei, st);
    }
  }
  switch (s) {
    case 16: return run_sr<T, 16>(batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi, stridei, st);
    case 32:
      if constexpr (sizeof(T) == 8)
        if (lu_variant()) return run_reg<32>(batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi, stridei, st);
      if constexpr (sizeof(T) == 4)
        if (lu_variant() && tinv == nullptr) {
          getrf_reg_kernel<32, float><<<batch, 32, 0, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, nullptr, 0);
          HODLR_CHECK_LAUNCH();
          return HODLR_OK;
        }
      return run_sr<T, 32>(batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi, stridei, st);
    case 64:
      if constexpr (sizeof(T) == 8)
        if (lu_variant()) return run_reg<64>(batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi, stridei, st);
      if constexpr (sizeof(T) == 4)
        if (lu_variant() && tinv == nullptr) {
          getrf_reg_kernel<64, float><<<batch, 64, 0, st>>>(mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, nullptr, 0);
          HODLR_CHECK_LAUNCH();
          return HODLR_OK;
        }
      return run_sr<T, 64>(batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi, stridei, st);
    case 128: return run_sr<T, 128>(batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi, stridei, st);
    default: return HODLR_ERR_ARG;
  }
}

template hodlr_status launch_getrf_cyclic<double>(int, int, int, const double*, int64_t, int64_t, double*, int64_t,
                                                  int64_t, int32_t*, int32_t*, int32_t*, double*, int64_t, int64_t,
                                                  cudaStream_t);
template hodlr_status launch_getrf_cyclic<float>(int, int, int, const float*, int64_t, int64_t, float*, int64_t,
                                                 int64_t, int32_t*, int32_t*, int32_t*, float*, int64_t, int64_t,
                                                 cudaStream_t);

}  // namespace hodlr
