// Batched LU factor (bit-exact replay of the reference) and LU solve / inverse.
//
//   getrf_kernel  <- backend.py:444-478 _lu_factor_stack (one CTA per block)
//   getrs_kernel  <- backend.py:546-567 _lu_solve_stack (also builds A^-1 = U^-1 L^-1 P
//                    by solving against the permuted identity)
//
// The factor is computed in shared memory.  Bit-exactness with numpy comes from
// replaying the same IEEE operations in the same order: first-max pivot (NaN
// wins, first index on ties, as np.argmax), whole-row swaps, true division by
// the pivot (0 -> 1), and the outer-product update rounded as a separate
// multiply then subtract (__dmul_rn / __dsub_rn: no FMA contraction).
#include "common.cuh"

namespace hodlr {

template <typename T>
__device__ __forceinline__ bool is_nan(T v) {
  return v != v;
}

template <typename T>
__device__ __forceinline__ T nan_max(T a, T b) {
  if (is_nan(a)) return a;
  if (is_nan(b)) return b;
  return a > b ? a : b;
}

// np.argmax order on (|value|, index): NaN first, then larger, then smaller index.
template <typename T>
__device__ __forceinline__ bool pivot_better(T v, int i, T best, int bi) {
  if (bi < 0) return true;
  bool vn = is_nan(v), bn = is_nan(best);
  if (bn) return vn && i < bi;
  if (vn) return true;
  return v > best || (v == best && i < bi);
}

// Input modes: 0 = plain strided blocks; 1 = K-block assembly
//   K_p = [[T_2p, I], [I, T_2p+1]] from the paired [W|T] panel of parent p
//   (2r x .. , ld lds): T block for row half h sits at src[h*r + i + j*lds].
template <typename T>
__global__ void __launch_bounds__(256) getrf_kernel(int s, int mode, const T* __restrict__ src, int64_t lds,
                                                    int64_t strides, T* out, int64_t ldo, int64_t strideo,
                                                    int32_t* __restrict__ swaps, int32_t* __restrict__ perm,
                                                    int32_t* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* a = reinterpret_cast<T*>(smem_raw);  // s x s, column-major, ld s
  T* colmax = a + s * s;
  int* pm = reinterpret_cast<int*>(colmax + s);
  __shared__ int piv_row;
  __shared__ int singular;

  const int64_t blk = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const T* g = src + blk * strides;

  if (mode == 0) {
    for (int j = warp; j < s; j += 8)
      for (int i = lane; i < s; i += 32) a[i + j * s] = g[i + j * lds];
  } else {
    const int r = s >> 1;
    for (int j = warp; j < s; j += 8)
      for (int i = lane; i < s; i += 32) {
        T v;
        if (i < r && j < r)
          v = g[i + j * lds];
        else if (i >= r && j >= r)
          v = g[i + (j - r) * lds];
        else
          v = (i < r) ? (T)(i == j - r) : (T)(i - r == j);
        a[i + j * s] = v;
      }
  }
  if (t < s) pm[t] = t;
  if (t == 0) singular = 0;
  __syncthreads();
  // original per-column magnitudes (np.abs(a).max(axis=1), NaN-propagating)
  for (int j = warp; j < s; j += 8) {
    T m = (T)0;
    for (int i = lane; i < s; i += 32) m = nan_max(m, (T)fabs((double)a[i + j * s]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) colmax[j] = m;
  }
  __syncthreads();

  const T thr_scale = mul_rn(Eps<T>::v, (T)s);
  for (int k = 0; k < s; ++k) {
    if (warp == 0) {
      T best = (T)0;
      int bi = -1;
      for (int i = k + lane; i < s; i += 32) {
        T v = (T)fabs((double)a[i + k * s]);
        if (pivot_better(v, i, best, bi)) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        T ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && pivot_better(ov, oi, best, bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) piv_row = bi;
    }
    __syncthreads();
    const int p = piv_row;
    if (p != k) {
      for (int j = t; j < s; j += 256) {
        T x = a[k + j * s];
        a[k + j * s] = a[p + j * s];
        a[p + j * s] = x;
      }
      if (t == 0) {
        int q = pm[k];
        pm[k] = pm[p];
        pm[p] = q;
      }
    }
    if (t == 0) swaps[blk * s + k] = p;
    __syncthreads();
    const T piv = a[k + k * s];
    if (t == 0 && (T)fabs((double)piv) <= mul_rn(thr_scale, colmax[k])) singular = 1;
    if (k + 1 < s) {
      const T d = (piv == (T)0) ? (T)1 : piv;
      for (int i = k + 1 + t; i < s; i += 256) a[i + k * s] = div_rn(a[i + k * s], d);
      __syncthreads();
      for (int j = k + 1 + warp; j < s; j += 8) {
        const T u = a[k + j * s];
        for (int i = k + 1 + lane; i < s; i += 32) a[i + j * s] = sub_rn(a[i + j * s], mul_rn(a[i + k * s], u));
      }
      __syncthreads();
    }
  }
  T* o = out + blk * strideo;
  for (int j = warp; j < s; j += 8)
    for (int i = lane; i < s; i += 32) o[i + j * ldo] = a[i + j * s];
  if (t < s) perm[blk * s + t] = pm[t];
  if (t == 0) info[blk] = singular;
}

// X_chunk <- A^-1 B_chunk from stored LU + perm.  identity=1 uses B = I, so the
// result is the explicit inverse U^-1 L^-1 P.  One CTA per (block, column chunk).
template <typename T>
__global__ void __launch_bounds__(256) getrs_kernel(int s, int nrhs, int cw, const T* __restrict__ LU, int64_t lda,
                                                    int64_t strideA, const int32_t* __restrict__ perm, const T* B,
                                                    int64_t ldb, int64_t strideB, T* X, int64_t ldx, int64_t strideX,
                                                    int identity) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* lu = reinterpret_cast<T*>(smem_raw);  // s x s ld s
  T* x = lu + s * s;                       // cw columns, ld s
  int* pm = reinterpret_cast<int*>(x + cw * s);
  const int nchunk = (nrhs + cw - 1) / cw;
  const int64_t blk = blockIdx.x / nchunk;
  const int c0 = (blockIdx.x % nchunk) * cw;
  const int ncols = min(cw, nrhs - c0);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  const T* g = LU + blk * strideA;
  for (int j = warp; j < s; j += 8)
    for (int i = lane; i < s; i += 32) lu[i + j * s] = g[i + j * lda];
  if (t < s) pm[t] = perm[blk * s + t];
  __syncthreads();
  if (identity) {
    for (int c = warp; c < ncols; c += 8)
      for (int i = lane; i < s; i += 32) x[c * s + i] = (T)(pm[i] == c0 + c);
  } else {
    const T* gb = B + blk * strideB;
    for (int c = warp; c < ncols; c += 8)
      for (int i = lane; i < s; i += 32) x[c * s + i] = gb[pm[i] + (int64_t)(c0 + c) * ldb];
  }
  __syncthreads();
  for (int j = 0; j + 1 < s; ++j) {
    for (int c = warp; c < ncols; c += 8) {
      const T xj = x[c * s + j];
      for (int i = j + 1 + lane; i < s; i += 32) x[c * s + i] -= lu[i + j * s] * xj;
    }
    __syncthreads();
  }
  for (int j = s - 1; j >= 0; --j) {
    if (t < ncols) x[t * s + j] = x[t * s + j] / lu[j + j * s];
    __syncthreads();
    for (int c = warp; c < ncols; c += 8) {
      const T xj = x[c * s + j];
      for (int i = lane; i < j; i += 32) x[c * s + i] -= lu[i + j * s] * xj;
    }
    __syncthreads();
  }
  T* gx = X + blk * strideX;
  for (int c = warp; c < ncols; c += 8)
    for (int i = lane; i < s; i += 32) gx[i + (int64_t)(c0 + c) * ldx] = x[c * s + i];
}


// ---------------------------------------------------------------------------
// Register-resident batched LU for s = S in {16, 32, 64}: one CTA per block,
// thread t owns row t in registers.  The step loop is NOT unrolled (code stays
// small enough for the instruction cache): column k of the own row is read /
// written through a chunked select (chunk k/8 by a uniform switch, then 8
// selects), and the trailing update walks 8-column chunks guarded by a uniform
// branch so finished chunks are skipped.  Row swaps are logical: every thread
// tracks the logical position of its row; the winner of step k takes position
// k and the row that held position k takes the winner's old position --
// exactly the reference's whole-row exchange.  The pivot row is broadcast
// through shared memory; ties in |a| go to the smallest logical position and
// NaN wins (np.argmax).  Afterwards the packed triangular inverses
// Tinv = strict_lower(L^-1) + upper(U^-1) are formed (one row per thread);
// applying them to a row-gathered right-hand side reproduces getrs to
// substitution accuracy with DMMA GEMMs (apply.cu).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ bool beats(T v, int pv, T b, int pb) {
  if (pv < 0) return false;
  if (pb < 0) return true;
  const bool vn = v != v, bn = b != b;
  if (vn || bn) return (vn && bn) ? pv < pb : vn;
  return v > b || (v == b && pv < pb);
}

// opaque select: keeps the optimizer from folding select chains over the row
// into a dynamically indexed (local-memory) array access
__device__ __forceinline__ double osel(int p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r)
      : "d"(a), "d"(b), "r"(p));
  return r;
}
__device__ __forceinline__ float osel(int p, float a, float b) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n\t}"
      : "=f"(r)
      : "f"(a), "f"(b), "r"(p));
  return r;
}

// a[k] for a runtime k: uniform branch on the 8-wide chunk, then 8 selects
template <typename T, int S>
__device__ __forceinline__ T row_get(const T (&a)[S], int k) {
  T v = a[0];
  const int kk = k & 7;
#pragma unroll
  for (int c = 0; c < S / 8; ++c) {
    if ((k >> 3) == c) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v = osel(kk == e, a[8 * c + e], v);
    }
  }
  return v;
}

template <typename T, int S>
__device__ __forceinline__ void row_set(T (&a)[S], int k, T v) {
  const int kk = k & 7;
#pragma unroll
  for (int c = 0; c < S / 8; ++c) {
    if ((k >> 3) == c) {
#pragma unroll
      for (int e = 0; e < 8; ++e) a[8 * c + e] = osel(kk == e, v, a[8 * c + e]);
    }
  }
}

template <typename T, int S>
__global__ void __launch_bounds__(S < 32 ? 32 : S) getrf_rows_kernel(
    int mode, const T* __restrict__ src, int64_t lds, int64_t strides, T* out, int64_t ldo, int64_t strideo,
    int32_t* __restrict__ swaps, int32_t* __restrict__ perm, int32_t* __restrict__ info, T* __restrict__ tinv,
    int64_t ldi, int64_t stridei) {
  static_assert(S % 8 == 0, "S must be a multiple of 8");
  constexpr int NT = S < 32 ? 32 : S;
  constexpr int NW = NT / 32;
  constexpr int LP = S + 1;  // padded row pitch of the staged matrix
  __shared__ __align__(16) T urow[2][S];
  __shared__ T mat[S * LP];
  __shared__ T cmax[S];
  __shared__ T dinv[S];
  __shared__ T redv[2][NW];
  __shared__ int redp[2][NW], redt[2][NW];
  __shared__ int swk[S];
  __shared__ int sflag;

  const int64_t blk = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool live = t < S;
  const T* g = src + blk * strides;
  T a[S];
#pragma unroll
  for (int j = 0; j < S; ++j) {
    T v = (T)0;
    if (live) {
      if (mode == 0) {
        v = g[t + j * lds];
      } else {
        constexpr int R = S / 2;
        if (t < R && j < R)
          v = g[t + j * lds];
        else if (t >= R && j >= R)
          v = g[t + (j - R) * lds];
        else
          v = (t < R) ? (T)(t == j - R) : (T)(t - R == j);
      }
    }
    a[j] = v;
  }
  // original column magnitudes (np.abs(a).max(axis=1), NaN-propagating)
  if (live) {
#pragma unroll
    for (int j = 0; j < S; ++j) mat[t * LP + j] = a[j];
  }
  if (t == 0) sflag = 0;
  __syncthreads();
  if (live) {
    T m = (T)0;
    for (int i = 0; i < S; ++i) m = nan_max(m, (T)fabs((double)mat[i * LP + t]));
    cmax[t] = m;
  }
  const T thr_scale = mul_rn(Eps<T>::v, (T)S);

  int pos = t;
  bool active = live;
  for (int k = 0; k < S; ++k) {
    const int buf = k & 1, kc = k >> 3;
    const T ak = row_get<T, S>(a, k);
    T v = active ? (T)fabs((double)ak) : (T)0;
    int pv = active ? pos : -1;
    int pt = t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int op = __shfl_xor_sync(0xffffffffu, pv, o);
      const int ot = __shfl_xor_sync(0xffffffffu, pt, o);
      if (beats(ov, op, v, pv)) {
        v = ov;
        pv = op;
        pt = ot;
      }
    }
    if (NW > 1) {
      if (lane == 0) {
        redv[buf][warp] = v;
        redp[buf][warp] = pv;
        redt[buf][warp] = pt;
      }
      __syncthreads();
      v = redv[buf][0];
      pv = redp[buf][0];
      pt = redt[buf][0];
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        if (beats(redv[buf][w], redp[buf][w], v, pv)) {
          v = redv[buf][w];
          pv = redp[buf][w];
          pt = redt[buf][w];
        }
      }
    }
    if (t == pt) {
#pragma unroll
      for (int c = 0; c < S / 8; ++c) {
        if (c >= kc) {
#pragma unroll
          for (int e = 0; e < 8; ++e) urow[buf][8 * c + e] = a[8 * c + e];
        }
      }
    }
    __syncthreads();
    const T piv = urow[buf][k];
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
      const T l = div_rn(ak, d);
      row_set<T, S>(a, k, l);
#pragma unroll
      for (int c = 0; c < S / 8; ++c) {
        if (c >= kc) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = 8 * c + e;
            if (j > k) a[j] = sub_rn(a[j], mul_rn(l, urow[buf][j]));
          }
        }
      }
    }
  }
  // factors out (row pos of the block), pivots, flag
  if (live) {
    T* o = out + blk * strideo;
#pragma unroll
    for (int j = 0; j < S; ++j) o[pos + j * ldo] = a[j];
    perm[blk * S + pos] = t;
    swaps[blk * S + t] = swk[t];
  }
  __syncthreads();
  if (t == 0) info[blk] = sflag;
  if (tinv == nullptr) return;
  // stage LU row-major by logical row for the inverses
  if (live) {
#pragma unroll
    for (int j = 0; j < S; ++j) mat[pos * LP + j] = a[j];
  }
  __syncthreads();
  if (live) dinv[t] = (T)1 / mat[t * LP + t];
  __syncthreads();
  if (!live) return;
  T* ti = tinv + blk * stridei;
  const int i = t;  // this thread forms row i of U^-1 and of L^-1
  const int wlo = warp * 32, whi = min(S - 1, warp * 32 + 31);
  // U^-1 row i: x U = e_i, right-looking over k >= (first row of this warp)
#pragma unroll
  for (int j = 0; j < S; ++j) a[j] = (T)(j == i);
  for (int k = wlo; k < S; ++k) {
    const int kc = k >> 3;
    const T xk = row_get<T, S>(a, k) * dinv[k];
    row_set<T, S>(a, k, xk);
#pragma unroll
    for (int c = 0; c < S / 8; ++c) {
      if (c >= kc) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = 8 * c + e;
          if (j > k) a[j] = fma(-xk, mat[k * LP + j], a[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < S; ++j)
    if (j >= i) ti[i + j * ldi] = a[j];
  // L^-1 row i: x L = e_i (unit diagonal), left-looking from the last row of this warp
#pragma unroll
  for (int j = 0; j < S; ++j) a[j] = (T)(j == i);
  for (int k = whi; k > 0; --k) {
    const int kc = k >> 3;
    const T xk = row_get<T, S>(a, k);
#pragma unroll
    for (int c = 0; c < S / 8; ++c) {
      if (c <= kc) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = 8 * c + e;
          if (j < k) a[j] = fma(-xk, mat[k * LP + j], a[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < S; ++j)
    if (j < i) ti[i + j * ldi] = a[j];
}

// Packed triangular inverses from stored LU for sizes without a register
// kernel: thread i forms row i of U^-1 (upper) and of L^-1 (strict lower).
template <typename T>
__global__ void __launch_bounds__(128) trtri_packed_kernel(int s, const T* __restrict__ LU, int64_t lda, int64_t strideA,
                                                           T* __restrict__ tinv, int64_t ldi, int64_t stridei) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int LP = s + 1;
  T* lu = reinterpret_cast<T*>(smem_raw);  // row-major, pitch LP
  T* xs = lu + s * LP;                     // per-thread rows, pitch LP
  const int64_t blk = blockIdx.x;
  const T* g = LU + blk * strideA;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int i = e % s, j = e / s;
    lu[i * LP + j] = g[i + (int64_t)j * lda];
  }
  __syncthreads();
  T* ti = tinv + blk * stridei;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    T* x = xs + i * LP;
    for (int j = 0; j < s; ++j) x[j] = (T)(j == i);
    for (int k = i; k < s; ++k) {
      const T xk = x[k] / lu[k * LP + k];
      x[k] = xk;
      for (int j = k + 1; j < s; ++j) x[j] = fma(-xk, lu[k * LP + j], x[j]);
    }
    for (int j = i; j < s; ++j) ti[i + (int64_t)j * ldi] = x[j];
    for (int j = 0; j < s; ++j) x[j] = (T)(j == i);
    for (int k = i; k > 0; --k) {
      const T xk = x[k];
      for (int j = 0; j < k; ++j) x[j] = fma(-xk, lu[k * LP + j], x[j]);
    }
    for (int j = 0; j < i; ++j) ti[i + (int64_t)j * ldi] = x[j];
  }
}

template <typename T>
hodlr_status launch_getrf_cyclic(int s, int batch, int mode, const T* src, int64_t lds, int64_t strides, T* out,
                                 int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, T* tinv,
                                 int64_t ldi, int64_t stridei, cudaStream_t st);

template <typename T>
static size_t getrf_smem(int s) {
  return (size_t)s * s * sizeof(T) + s * sizeof(T) + s * sizeof(int) + 16;
}
template <typename T>
static size_t getrs_smem(int s, int cw) {
  return (size_t)s * s * sizeof(T) + (size_t)cw * s * sizeof(T) + s * sizeof(int) + 16;
}

template <typename T>
hodlr_status launch_getrf(int s, int batch, int mode, const T* src, int64_t lds, int64_t strides, T* out, int64_t ldo,
                          int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, T* tinv, int64_t ldi,
                          int64_t stridei, cudaStream_t st) {
  if (batch == 0 || s == 0) return HODLR_OK;
  if (s == 128 || s == 64 || s == 32 || s == 16)
    return launch_getrf_cyclic<T>(s, batch, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info, tinv, ldi,
                                  stridei, st);
  size_t sm = getrf_smem<T>(s);
  if (sm > 227 * 1024) return HODLR_ERR_ARG;
  smem_attr(getrf_kernel<T>, (int)sm);
  getrf_kernel<T><<<batch, 256, sm, st>>>(s, mode, src, lds, strides, out, ldo, strideo, swaps, perm, info);
  HODLR_CHECK_LAUNCH();
  if (tinv) {
    const size_t sm2 = (size_t)2 * s * (s + 1) * sizeof(T);
    if (sm2 > 227 * 1024) return HODLR_ERR_ARG;
    smem_attr(trtri_packed_kernel<T>, (int)sm2);
    trtri_packed_kernel<T><<<batch, 128, sm2, st>>>(s, out, ldo, strideo, tinv, ldi, stridei);
    HODLR_CHECK_LAUNCH();
  }
  return HODLR_OK;
}

// Thread-per-column substitution for S in {16, 32, 64}: the block's LU and a
// CW-column slice of the right-hand sides are staged in shared memory with
// coalesced loads (a column's S rows are contiguous), every thread carries one
// column in registers (fully unrolled, compile-time indices) and runs the
// column-oriented (axpy) forward / backward sweeps -- after x_j is final the
// S-1-j updates it feeds are independent, so each thread has S-way ILP and no
// barrier is needed between steps.  L / U entries are broadcast shared loads.
// Per element the update order is j ascending (forward) / descending
// (backward) with fused multiply-subtract and true division, exactly as in
// getrs_warp_kernel, so a column's result does not depend on nrhs.
template <int S>
struct ColCfg {
  static constexpr int CW = S == 64 ? 64 : 128;  // columns (threads) per CTA
  static constexpr int P = CW + 1;               // staging pitch
  static constexpr int MINB = S == 64 ? 8 : 1;   // S = 64: cap registers (x[64] + operands) for 16 warps/SM
};

template <typename T, int S>
__global__ void __launch_bounds__(ColCfg<S>::CW, ColCfg<S>::MINB) getrs_col_kernel(int nrhs, int cpb, const T* __restrict__ LU,
                                                                  int64_t lda, int64_t strideA,
                                                                  const int32_t* __restrict__ perm, const T* B,
                                                                  int64_t ldb, int64_t strideB, T* X, int64_t ldx,
                                                                  int64_t strideX, int identity) {
  constexpr int CW = ColCfg<S>::CW, P = ColCfg<S>::P;
  __shared__ __align__(16) T lu[S * S];  // column-major, ld S
  __shared__ T xs[S * P];                // [row][column]
  __shared__ int pm[S];
  const int64_t blk = blockIdx.x / cpb;
  const int c0 = (int)(blockIdx.x % cpb) * CW;
  const int ncw = min(CW, nrhs - c0);
  const int t = threadIdx.x;
  const T* g = LU + blk * strideA;
  for (int idx = t; idx < S * S; idx += CW) lu[idx] = g[(idx % S) + (int64_t)(idx / S) * lda];
  if (t < S) pm[t] = perm[blk * S + t];
  if (!identity) {
    const T* gb = B + blk * strideB + (int64_t)c0 * ldb;
    for (int idx = t; idx < S * ncw; idx += CW) {
      const int i = idx % S, c = idx / S;
      xs[i * P + c] = gb[i + (int64_t)c * ldb];
    }
  }
  __syncthreads();
  T x[S];
#pragma unroll
  for (int i = 0; i < S; ++i) x[i] = identity ? (T)(pm[i] == c0 + t) : xs[pm[i] * P + t];
  // forward: unit lower
#pragma unroll
  for (int j = 0; j < S - 1; ++j) {
    const T xj = x[j];
#pragma unroll
    for (int i = j + 1; i < S; ++i) x[i] = fma(-lu[i + j * S], xj, x[i]);
  }
  // backward: upper with true division
#pragma unroll
  for (int j = S - 1; j >= 0; --j) {
    x[j] = x[j] / lu[j + j * S];
    const T xj = x[j];
#pragma unroll
    for (int i = 0; i < j; ++i) x[i] = fma(-lu[i + j * S], xj, x[i]);
  }
  __syncthreads();  // every thread has read its column (X may alias B)
#pragma unroll
  for (int i = 0; i < S; ++i) xs[i * P + t] = x[i];
  __syncthreads();
  T* gx = X + blk * strideX + (int64_t)c0 * ldx;
  for (int idx = t; idx < S * ncw; idx += CW) {
    const int i = idx % S, c = idx / S;
    gx[i + (int64_t)c * ldx] = xs[i * P + c];
  }
}

// Few right-hand sides: warp per (block, column), lane = rows lane + 32 q.  The
// LU columns are read straight from global memory (one coalesced line per
// column step); x_j is broadcast from its owner lane.  Same per-element
// operation order as getrs_col_kernel (bit-identical columns).
template <typename T, int S>
__global__ void __launch_bounds__(256) getrs_warp_kernel(int nrhs, int batch, const T* __restrict__ LU, int64_t lda,
                                                         int64_t strideA, const int32_t* __restrict__ perm,
                                                         const T* B, int64_t ldb, int64_t strideB, T* X, int64_t ldx,
                                                         int64_t strideX, int identity) {
  constexpr int Q = S > 32 ? 2 : 1;  // rows per lane (S <= 64)
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (item >= (int64_t)batch * nrhs) return;
  const int64_t blk = item / nrhs;
  const int c = (int)(item % nrhs);
  const T* g = LU + blk * strideA;
  const int32_t* pb = perm + blk * S;
  const T* gb = B + blk * strideB + (int64_t)c * ldb;
  T x[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = lane + 32 * q;
    x[q] = T(0);
    if (i < S) {
      const int pi = __ldg(pb + i);
      x[q] = identity ? (T)(pi == c) : gb[pi];
    }
  }
  // x_j lives in register j / 32 of lane j % 32 (select, not a dynamic index)
  auto own = [&](int j) -> T& { return (Q == 1 || j < 32) ? x[0] : x[Q - 1]; };
  // LU columns are prefetched 8 steps ahead into a register ring (the
  // substitution chain never waits on a global load)
  constexpr int PF = S < 8 ? S : 8;
  T lc[PF][Q];
  auto load_col = [&](int j, T (&dst)[Q]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      dst[q] = (i < S && j >= 0 && j < S) ? __ldg(g + i + (int64_t)j * lda) : T(0);
    }
  };
  // forward: unit lower, columns 0 .. S-2
#pragma unroll
  for (int p = 0; p < PF; ++p) load_col(p, lc[p]);
#pragma unroll 1
  for (int jb = 0; jb < S; jb += PF) {
    T cur[PF][Q];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
#pragma unroll
      for (int q = 0; q < Q; ++q) cur[p][q] = lc[p][q];
      load_col(jb + PF + p < S - 1 ? jb + PF + p : -1, lc[p]);
    }
#pragma unroll
    for (int p = 0; p < PF; ++p) {
      const int j = jb + p;
      if (j < S - 1) {
        const T xj = __shfl_sync(0xffffffffu, own(j), j % 32);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int i = lane + 32 * q;
          if (i > j && i < S) x[q] = fma(-cur[p][q], xj, x[q]);
        }
      }
    }
  }
  // backward: upper with true division, columns S-1 .. 0
#pragma unroll
  for (int p = 0; p < PF; ++p) load_col(S - 1 - p, lc[p]);
#pragma unroll 1
  for (int jb = S - 1; jb >= 0; jb -= PF) {
    T cur[PF][Q];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
#pragma unroll
      for (int q = 0; q < Q; ++q) cur[p][q] = lc[p][q];
      load_col(jb - PF - p, lc[p]);
    }
#pragma unroll
    for (int p = 0; p < PF; ++p) {
      const int j = jb - p;
      if (j >= 0) {
        // the owner lane holds U[j][j] in cur[p][j / 32]
        if ((j % 32) == lane) own(j) = own(j) / ((Q == 1 || j < 32) ? cur[p][0] : cur[p][Q - 1]);
        const T xj = __shfl_sync(0xffffffffu, own(j), j % 32);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int i = lane + 32 * q;
          if (i < j) x[q] = fma(-cur[p][q], xj, x[q]);
        }
      }
    }
  }
  __syncwarp();  // all lanes have read B (X may alias B)
  T* gx = X + blk * strideX + (int64_t)c * ldx;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = lane + 32 * q;
    if (i < S) gx[i] = x[q];
  }
}

template <typename T, int S>
static hodlr_status run_getrs_col(int nrhs, int batch, const T* LU, int64_t lda, int64_t strideA, const int32_t* perm,
                                  const T* B, int64_t ldb, int64_t strideB, T* X, int64_t ldx, int64_t strideX,
                                  int identity, cudaStream_t st) {
  if (nrhs <= 8) {
    const int64_t items = (int64_t)batch * nrhs;
    const int64_t grid = ceil_div(items, 8);
    if (grid > 2147483647LL) return HODLR_ERR_ARG;
    getrs_warp_kernel<T, S><<<(unsigned)grid, 256, 0, st>>>(nrhs, batch, LU, lda, strideA, perm, B, ldb, strideB, X,
                                                           ldx, strideX, identity);
    HODLR_CHECK_LAUNCH();
    return HODLR_OK;
  }
  constexpr int CW = ColCfg<S>::CW;
  const int cpb = (nrhs + CW - 1) / CW;
  const int64_t grid = (int64_t)batch * cpb;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  static const bool carve = [] {
    smem_attr(getrs_col_kernel<T, S>, 100, cudaFuncAttributePreferredSharedMemoryCarveout);
    return true;
  }();
  (void)carve;
  getrs_col_kernel<T, S><<<(unsigned)grid, CW, 0, st>>>(nrhs, cpb, LU, lda, strideA, perm, B, ldb, strideB, X, ldx,
                                                       strideX, identity);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template <typename T>
hodlr_status launch_getrs(int s, int nrhs, int batch, const T* LU, int64_t lda, int64_t strideA, const int32_t* perm,
                          const T* B, int64_t ldb, int64_t strideB, T* X, int64_t ldx, int64_t strideX, int identity,
                          cudaStream_t st) {
  if (batch == 0 || s == 0 || nrhs == 0) return HODLR_OK;
  // thread-per-column substitution (each thread reads and writes only its own column, so X may alias B)
  if (s == 16) return run_getrs_col<T, 16>(nrhs, batch, LU, lda, strideA, perm, B, ldb, strideB, X, ldx, strideX, identity, st);
  if (s == 32) return run_getrs_col<T, 32>(nrhs, batch, LU, lda, strideA, perm, B, ldb, strideB, X, ldx, strideX, identity, st);
  if constexpr (sizeof(T) == 4) {
    if (s == 64)
      return run_getrs_col<T, 64>(nrhs, batch, LU, lda, strideA, perm, B, ldb, strideB, X, ldx, strideX, identity, st);
  }
  int cw = nrhs < 64 ? nrhs : 64;
  size_t sm = getrs_smem<T>(s, cw);
  while (sm > 227 * 1024 && cw > 8) {
    cw >>= 1;
    sm = getrs_smem<T>(s, cw);
  }
  if (sm > 227 * 1024) return HODLR_ERR_ARG;
  const int64_t grid = (int64_t)batch * ((nrhs + cw - 1) / cw);
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  smem_attr(getrs_kernel<T>, (int)sm);
  getrs_kernel<T><<<(unsigned)grid, 256, sm, st>>>(s, nrhs, cw, LU, lda, strideA, perm, B, ldb, strideB, X, ldx,
                                                    strideX, identity);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

template hodlr_status launch_getrf<double>(int, int, int, const double*, int64_t, int64_t, double*, int64_t, int64_t,
                                           int32_t*, int32_t*, int32_t*, double*, int64_t, int64_t, cudaStream_t);
template hodlr_status launch_getrf<float>(int, int, int, const float*, int64_t, int64_t, float*, int64_t, int64_t,
                                          int32_t*, int32_t*, int32_t*, float*, int64_t, int64_t, cudaStream_t);
template hodlr_status launch_getrs<double>(int, int, int, const double*, int64_t, int64_t, const int32_t*,
                                           const double*, int64_t, int64_t, double*, int64_t, int64_t, int,
                                           cudaStream_t);
template hodlr_status launch_getrs<float>(int, int, int, const float*, int64_t, int64_t, const int32_t*, const float*,
                                          int64_t, int64_t, float*, int64_t, int64_t, int, cudaStream_t);

}  // namespace hodlr
