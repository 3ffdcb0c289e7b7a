// Device HODLR assembly from an entry oracle (SPEC.md:163-171 [OP] assemble):
// leaf blocks materialized exactly, every sibling off-diagonal block
// compressed by adaptive cross approximation with rook pivoting at a fixed
// rank cap r (compress.py:87-170 _aca, tol = 0, max_rank = r), the crosses
// written straight into the U / V level panels (A(I_a, I_b) = U_a V_b^T).
//
// The ACA of all 2^l' blocks of a level runs in lockstep: data-parallel
// kernels (residual row, residual column, masked argmax, append) over every
// block at once, with one thread per block deciding the control flow between
// them (next-row proposal, zero-row scan, rook sweeps, zero pivot).  Every
// arithmetic step replays the reference's IEEE operation order (entry formula
// with separately rounded products, residual r - u_l(i) w_l in cross order,
// u = col / pivot, first-index argmax of the masked magnitudes), so with the
// same geometry the factors are bit-identical to compress() with
// CompressionConfig(tol=0, max_rank=r) -- tests/golden/make_build_golden.py.
// Blocks whose residual is exhausted before rank r (exact low rank) keep
// zero columns (SURVEY §8a zero-padding).
#include <vector>

#include "common.cuh"

#define TRY_STATUS(x)                  \
  do {                                 \
    hodlr_status s_ = (x);             \
    if (s_ != HODLR_OK) return s_;     \
  } while (0)

namespace hodlr {
namespace {

// ---- entry oracles -------------------------------------------------------

// Exterior Dirichlet Laplace double layer with log completion on a contour
// (problems.py:158-217 LaplaceDoubleLayerOracle.__call__):
//   A_ij = (d(x_i, y_j) + logterm_i) w_j + 0.5 delta_ij,
//   d = n_j.(x_i - x_j) / (2 pi |x_i - x_j|^2), d(x, x) = diag_i.
struct LaplaceDL {
  const double *x, *y, *nx, *ny, *w, *logt, *diag;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    double dk;
    if (i == j) {
      dk = diag[i];
    } else {
      const double d0 = __dsub_rn(x[i], x[j]), d1 = __dsub_rn(y[i], y[j]);
      const double r2 = __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
      const double num = __dadd_rn(__dmul_rn(nx[j], d0), __dmul_rn(ny[j], d1));
      dk = __ddiv_rn(num, __dmul_rn(6.283185307179586, r2));  // (2.0 * np.pi) * r2
    }
    const double a = __dmul_rn(__dadd_rn(dk, logt[i]), w[j]);
    return __dadd_rn(a, i == j ? 0.5 : 0.0);
  }
};

// Gaussian kernel on points (BASELINE cfg1: 2-D, cfg3: 3-D), regularized:
//   A_ij = exp(-|p_i - p_j|^2 / h^2) + lambda delta_ij,
// coordinates dim-major (p_k at pts + k N), squared distance summed over k in
// order (numpy's sum over the last axis of a 2- or 3-vector).
struct GaussianPts {
  const double* p;
  int64_t n;
  int dim;
  double h2, lam;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    double d2 = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double d = __dsub_rn(p[k * n + i], p[k * n + j]);
      d2 = k == 0 ? __dmul_rn(d, d) : __dadd_rn(d2, __dmul_rn(d, d));
    }
    const double v = exp(-__ddiv_rn(d2, h2));
    return __dadd_rn(v, i == j ? lam : 0.0);
  }
};

// Sparse-factorization Schur-complement surrogate (BASELINE cfg4; no reference
// counterpart -- the reference has no sparse solver): eliminating
// the two subdomains of a 3-D 7-point Laplacian onto a planar separator leaves
// (asymptotically) twice the half-space Dirichlet-to-Neumann map, the
// hypersingular kernel S_ij = -1 / (pi r_ij^3) on the separator grid (unit
// spacing, dim-major 2-D coordinates), with diagonal c_0 + sigma: c_0 =
// (1/pi) sum_{k in Z^2 \ 0} |k|^-3 = 2.8755 is the lattice row sum (rows are
// diagonally dominant, the matrix SPD) and sigma the zeroth-order term the
// eliminated subdomains contribute.  Off-diagonal blocks of a kd-ordered
// plane are numerically low-rank, with ranks growing toward the top levels --
// the regime where a rank-8 HODLR is a low-accuracy preconditioner.
struct SchurPlane {
  const double* p;
  int64_t n;
  double diag;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    if (i == j) return diag;
    const double dx = __dsub_rn(p[i], p[j]), dy = __dsub_rn(p[n + i], p[n + j]);
    const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    return -1.0 / (3.141592653589793 * r2 * sqrt(r2));
  }
};

// Entries of a dense column-major matrix on the device (tests, small n).
struct DenseOracle {
  const double* A;
  int64_t lda;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const { return A[i + j * lda]; }
};

// ---- per-level ACA state ---------------------------------------------------

enum : int { ST_DONE = 0, ST_LIVE = 1 };

struct BlockState {
  int status;   // ST_LIVE while crosses remain to be found
  int k;        // crosses appended
  int i, j;     // current pivot row / column (block-local)
  int next_i;   // row proposed by the last residual column (-1: none)
  int req_row;  // row whose residual the next row kernel computes (-1: none)
  int req_col;  // column for the next column kernel (-1: none)
  int searching;  // 1: proposal failed / scanning for a row with a nonzero residual
  int rook;     // rook sweeps still allowed in this iteration (0: finished)
  int append;   // 1: the append kernel writes cross k this iteration
  int have_row; // 1: a row with a nonzero residual was accepted this iteration
  double rmax;  int rarg;   // masked argmax of the residual row
  double cmax;  int carg;   // masked argmax of the residual column
  double fmax;  int farg;   // first unused row (value 1 where unused)
  double pivot;
};

struct AcaLv {
  int64_t n;   // N (slab leading dimension)
  int64_t nc;  // block rows = cols
  int nb;      // blocks at this level (2^lv)
  int r;       // rank cap
  int64_t c0;  // first slab column of this level, (lv - 1) r
  double* U;
  double* V;
  double* R;   // [nb][nc] residual rows
  double* Cc;  // [nb][nc] residual columns
  uint8_t* urow;
  uint8_t* ucol;
  BlockState* st;
  double* pv;  // argmax partials: value
  int* pi;     // argmax partials: index
  int cpb;     // argmax chunks per block
  int* err;    // non-finite entry flag
};

// block b: sibling pair b / 2, orientation b % 2 -> rows of node 2p + o, cols of node 2p + 1 - o
__device__ __forceinline__ int64_t blk_row0(const AcaLv& g, int b) { return (int64_t)((b & ~1) + (b & 1)) * g.nc; }
__device__ __forceinline__ int64_t blk_col0(const AcaLv& g, int b) { return (int64_t)((b & ~1) + 1 - (b & 1)) * g.nc; }

// residual row: R_b = A(row0 + i, col0 + :) - sum_l u_l(i) w_l   (compress.py residual_row)
template <class Oracle>
__global__ void aca_row_kernel(AcaLv g, Oracle A) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)g.nb * g.nc) return;
  const int b = (int)(e / g.nc);
  const int64_t jj = e - (int64_t)b * g.nc;
  const BlockState& s = g.st[b];
  if (s.req_row < 0) return;
  const int64_t gi = blk_row0(g, b) + s.req_row, gj = blk_col0(g, b) + jj;
  double v = A(gi, gj);
  if (!isfinite(v)) *g.err = 1;
  for (int l = 0; l < s.k; ++l) {
    const int64_t c = (g.c0 + l) * g.n;
    v = __dsub_rn(v, __dmul_rn(g.U[gi + c], g.V[gj + c]));
  }
  g.R[e] = v;
}

// residual column: C_b = A(row0 + :, col0 + j) - sum_l w_l(j) u_l   (compress.py residual_col)
template <class Oracle>
__global__ void aca_col_kernel(AcaLv g, Oracle A) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)g.nb * g.nc) return;
  const int b = (int)(e / g.nc);
  const int64_t ii = e - (int64_t)b * g.nc;
  const BlockState& s = g.st[b];
  if (s.req_col < 0) return;
  const int64_t gi = blk_row0(g, b) + ii, gj = blk_col0(g, b) + s.req_col;
  double v = A(gi, gj);
  if (!isfinite(v)) *g.err = 1;
  for (int l = 0; l < s.k; ++l) {
    const int64_t c = (g.c0 + l) * g.n;
    v = __dsub_rn(v, __dmul_rn(g.V[gj + c], g.U[gi + c]));
  }
  g.Cc[e] = v;
}

// masked argmax, numpy semantics: max of where(mask, 0, |x|), first index on ties
enum : int { AM_ROW = 0, AM_COL = 1, AM_FREE = 2 };
constexpr int kArgChunk = 2048;

__device__ __forceinline__ void am_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__device__ __forceinline__ bool am_wanted(const BlockState& s, int mode) {
  if (s.status != ST_LIVE) return false;
  if (mode == AM_ROW) return s.req_row >= 0;
  if (mode == AM_COL) return s.req_col >= 0 || s.append;
  return s.searching;
}

__global__ void aca_argmax_partial_kernel(AcaLv g, int mode) {
  const int b = blockIdx.x / g.cpb, c = blockIdx.x % g.cpb;
  const BlockState& s = g.st[b];
  if (!am_wanted(s, mode)) return;
  const int64_t base = (int64_t)b * g.nc;
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int64_t t = (int64_t)c * kArgChunk + threadIdx.x; t < min((int64_t)(c + 1) * kArgChunk, g.nc); t += blockDim.x) {
    double v;
    if (mode == AM_ROW) v = g.ucol[base + t] ? 0.0 : fabs(g.R[base + t]);
    else if (mode == AM_COL) v = g.urow[base + t] ? 0.0 : fabs(g.Cc[base + t]);
    else v = g.urow[base + t] ? 0.0 : 1.0;
    am_merge(bv, bi, v, (int)t);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    am_merge(bv, bi, v2, i2);
  }
  __shared__ double sv[32];
  __shared__ int si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sv[warp] = bv, si[warp] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) am_merge(bv, bi, sv[w], si[w]);
    g.pv[blockIdx.x] = bv;
    g.pi[blockIdx.x] = bi;
  }
}

__global__ void aca_argmax_final_kernel(AcaLv g, int mode) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  if (!am_wanted(s, mode)) return;
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int c = 0; c < g.cpb; ++c) am_merge(bv, bi, g.pv[b * g.cpb + c], g.pi[b * g.cpb + c]);
  if (mode == AM_ROW) s.rmax = bv, s.rarg = bi;
  else if (mode == AM_COL) s.cmax = bv, s.carg = bi;
  else s.fmax = bv, s.farg = bi;
}

// ---- control (one thread per block) ------------------------------------------

// start of an iteration: try the proposed row, else scan from the first unused row
__global__ void aca_begin_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  s.req_row = s.req_col = -1;
  s.append = 0;
  s.rook = 0;
  s.searching = 0;
  s.have_row = 0;
  if (s.status != ST_LIVE) return;
  if (s.k >= g.r) {
    s.status = ST_DONE;
    return;
  }
  if (s.next_i >= 0 && !g.urow[(int64_t)b * g.nc + s.next_i]) s.req_row = s.next_i;
  else s.searching = 1;  // the scan's first candidate comes from the AM_FREE argmax
}

// scan step: the first unused row becomes the candidate (none left: converged)
__global__ void aca_scan_pick_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  if (s.status != ST_LIVE || !s.searching) return;
  if (s.fmax <= 0.0) {  // every row used: residual exhausted
    s.status = ST_DONE;
    s.searching = 0;
    s.req_row = -1;
    return;
  }
  s.req_row = s.farg;
}

// after a row residual: accept it if its masked max is positive, else fall
// back to / continue the scan (the failed scan candidate is marked used)
__global__ void aca_row_check_kernel(AcaLv g, int* searching_count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  if (s.status != ST_LIVE || s.req_row < 0) return;
  if (s.rmax > 0.0) {
    s.i = s.req_row;
    s.j = s.rarg;
    s.req_row = -1;
    s.req_col = s.j;
    s.searching = 0;
    s.have_row = 1;
    s.rook = 4;  // _ROOK_SWEEPS
    return;
  }
  if (s.searching) g.urow[(int64_t)b * g.nc + s.req_row] = 1;
  s.searching = 1;
  s.req_row = -1;
  atomicAdd(searching_count, 1);
}

// rook sweep, part 1 (after the column residual and its masked argmax)
__global__ void aca_rook1_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  s.req_col = -1;
  if (s.status != ST_LIVE || s.rook <= 0) return;
  const double rj = fabs(g.R[(int64_t)b * g.nc + s.j]);
  if (s.cmax <= rj) {  // pivot already maximal in its column
    s.rook = 0;
    return;
  }
  s.i = s.carg;
  s.req_row = s.i;
}

// rook sweep, part 2 (after the new row residual and its masked argmax)
__global__ void aca_rook2_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  if (s.status != ST_LIVE || s.rook <= 0 || s.req_row < 0) return;
  s.req_row = -1;
  const int j2 = s.rarg;
  if (j2 == s.j) {  // rook condition met
    s.rook = 0;
    return;
  }
  s.j = j2;
  s.req_col = j2;
  s.rook -= 1;  // after the 4th sweep the recomputed column is final (no further test)
}

// end of the sweeps: zero pivot -> the row is marked used and the iteration
// repeats; else cross k is appended (by aca_append_kernel)
__global__ void aca_pivot_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  s.req_col = -1;
  s.append = 0;
  if (s.status != ST_LIVE || !s.have_row) return;
  const int64_t base = (int64_t)b * g.nc;
  s.pivot = g.R[base + s.j];
  if (s.pivot == 0.0) {
    g.urow[base + s.i] = 1;
    return;
  }
  s.append = 1;
}

__global__ void aca_append_kernel(AcaLv g) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)g.nb * g.nc) return;
  const int b = (int)(e / g.nc);
  const int64_t t = e - (int64_t)b * g.nc;
  const BlockState& s = g.st[b];
  if (s.status != ST_LIVE || !s.append) return;
  const int64_t c = (g.c0 + s.k) * g.n;
  g.U[blk_row0(g, b) + t + c] = __ddiv_rn(g.Cc[e], s.pivot);  // u = col / pivot
  g.V[blk_col0(g, b) + t + c] = g.R[e];                      // v = conj(w) = w (real)
}

// after the append: mark the pivots used (the next-row argmax runs on the
// updated mask), then advance
__global__ void aca_mark_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  if (s.status != ST_LIVE || !s.append) return;
  g.urow[(int64_t)b * g.nc + s.i] = 1;
  g.ucol[(int64_t)b * g.nc + s.j] = 1;
}

__global__ void aca_advance_kernel(AcaLv g, int* live_count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState& s = g.st[b];
  if (s.status == ST_LIVE && s.append) {
    s.next_i = s.cmax > 0.0 ? s.carg : -1;
    s.k += 1;
    s.append = 0;
    if (s.k >= g.r) s.status = ST_DONE;
  }
  if (s.status == ST_LIVE) atomicAdd(live_count, 1);
}

__global__ void aca_init_kernel(AcaLv g) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  BlockState s{};
  s.status = g.r > 0 ? ST_LIVE : ST_DONE;
  s.next_i = -1;
  s.req_row = s.req_col = -1;
  s.i = s.j = -1;
  g.st[b] = s;
}

// xorshift64* stream (problems.py:26-48): splitmix64-scrambled seed, top 53
// bits of state * 0x2545F4914F6CDD1D as a double in [0, 1).  Sequential by
// nature: one thread walks the stream (the state never leaves registers).
__global__ void xorshift_uniform_kernel(uint64_t seed, int64_t count, double* out) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  uint64_t x = z ^ (z >> 31);
  if (x == 0) x = 0x9E3779B97F4A7C15ull;
  for (int64_t k = 0; k < count; ++k) {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    out[k] = (double)((x * 0x2545F4914F6CDD1Dull) >> 11) * 0x1.0p-53;
  }
}

// leaf blocks: D_a = A(I_a, I_a), column-major m x m at a m^2
template <class Oracle>
__global__ void leaf_blocks_kernel(int64_t nleaf, int m, double* D, Oracle A, int* err) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t mm = (int64_t)m * m;
  if (e >= nleaf * mm) return;
  const int64_t a = e / mm, t = e - a * mm;
  const int64_t i = t % m, j = t / m;
  const double v = A(a * m + i, a * m + j);
  if (!isfinite(v)) *err = 1;
  D[e] = v;
}

// ---- host driver ---------------------------------------------------------------

struct BuildWs {
  size_t R, C, ur, uc, st, pv, pi, cnt, total;
};

BuildWs build_ws(const hodlr_desc* d) {
  const int64_t n = d->n;
  const int64_t nbmax = d->L > 0 ? ((int64_t)1 << d->L) : 1;
  const int64_t chunks = ceil_div(n, kArgChunk) + nbmax;  // sum over blocks of ceil(nc / chunk)
  BuildWs w{};
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  w.R = al(sizeof(double) * n);
  w.C = al(sizeof(double) * n);
  w.ur = al(n);
  w.uc = al(n);
  w.st = al(sizeof(BlockState) * nbmax);
  w.pv = al(sizeof(double) * chunks);
  w.pi = al(sizeof(int) * chunks);
  w.cnt = al(sizeof(int) * 4);
  w.total = w.R + w.C + w.ur + w.uc + w.st + w.pv + w.pi + w.cnt;
  return w;
}

bool build_desc_ok(const hodlr_desc* d) {
  return d && d->ranks == nullptr && d->dtype == HODLR_F64 && d->m >= 1 && d->r >= 0 && d->L >= 0 && d->L <= 30 &&
         d->n == (int64_t)d->m << d->L;
}

template <class Oracle>
hodlr_status build_run(const hodlr_desc* d, const Oracle& A, double* D, double* U, double* V, char* wp,
                       cudaStream_t st) {
  const BuildWs ws = build_ws(d);
  const int64_t n = d->n;
  const int m = d->m, r = d->r, L = d->L;
  char* p = wp;
  double* R = reinterpret_cast<double*>(p); p += ws.R;
  double* Cc = reinterpret_cast<double*>(p); p += ws.C;
  uint8_t* ur = reinterpret_cast<uint8_t*>(p); p += ws.ur;
  uint8_t* uc = reinterpret_cast<uint8_t*>(p); p += ws.uc;
  BlockState* bs = reinterpret_cast<BlockState*>(p); p += ws.st;
  double* pv = reinterpret_cast<double*>(p); p += ws.pv;
  int* pi = reinterpret_cast<int*>(p); p += ws.pi;
  int* cnt = reinterpret_cast<int*>(p);  // [0] err, [1] live, [2] searching
  if (cudaMemsetAsync(cnt, 0, sizeof(int) * 4, st) != cudaSuccess) return hodlr_set_cuda_error(cudaGetLastError());
  const int64_t nleaf = n / m;
  leaf_blocks_kernel<Oracle><<<(unsigned)ceil_div(nleaf * m * m, 256), 256, 0, st>>>(nleaf, m, D, A, cnt);
  HODLR_CHECK_LAUNCH();
  if (L > 0 && r > 0) {
    if (cudaMemsetAsync(U, 0, sizeof(double) * n * r * L, st) != cudaSuccess ||
        cudaMemsetAsync(V, 0, sizeof(double) * n * r * L, st) != cudaSuccess)
      return hodlr_set_cuda_error(cudaGetLastError());
  }
  int host[4];
  auto read_counts = [&]() -> bool {
    if (cudaMemcpyAsync(host, cnt, sizeof(int) * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) return false;
    return cudaStreamSynchronize(st) == cudaSuccess;
  };
  for (int lv = 1; lv <= L && r > 0; ++lv) {
    AcaLv g{};
    g.n = n;
    g.nc = n >> lv;
    g.nb = 1 << lv;
    g.r = (int)std::min<int64_t>(r, g.nc);
    g.c0 = (int64_t)(lv - 1) * r;
    g.U = U, g.V = V, g.R = R, g.Cc = Cc, g.urow = ur, g.ucol = uc, g.st = bs, g.pv = pv, g.pi = pi;
    g.cpb = (int)ceil_div(g.nc, kArgChunk);
    g.err = cnt;
    const int64_t ne = (int64_t)g.nb * g.nc;
    const unsigned eg = (unsigned)ceil_div(ne, 256), bg = (unsigned)ceil_div(g.nb, 128);
    const unsigned ag = (unsigned)((int64_t)g.nb * g.cpb);
    if (cudaMemsetAsync(ur, 0, n, st) != cudaSuccess || cudaMemsetAsync(uc, 0, n, st) != cudaSuccess)
      return hodlr_set_cuda_error(cudaGetLastError());
    aca_init_kernel<<<bg, 128, 0, st>>>(g);
    HODLR_CHECK_LAUNCH();
    auto argmax = [&](int mode) -> hodlr_status {
      aca_argmax_partial_kernel<<<ag, 256, 0, st>>>(g, mode);
      HODLR_CHECK_LAUNCH();
      aca_argmax_final_kernel<<<bg, 128, 0, st>>>(g, mode);
      HODLR_CHECK_LAUNCH();
      return HODLR_OK;
    };
    // each pass appends at most one cross per block; zero pivots / scans take extra passes
    for (int64_t pass = 0; pass < 4 * (int64_t)g.nc + 4 * r + 8; ++pass) {
      aca_begin_kernel<<<bg, 128, 0, st>>>(g);
      HODLR_CHECK_LAUNCH();
      // find a row with a nonzero residual (normally the proposed row, first try)
      for (int64_t tries = 0;; ++tries) {
        TRY_STATUS(argmax(AM_FREE));  // first unused row, for the blocks that scan
        aca_scan_pick_kernel<<<bg, 128, 0, st>>>(g);
        HODLR_CHECK_LAUNCH();
        aca_row_kernel<Oracle><<<eg, 256, 0, st>>>(g, A);
        HODLR_CHECK_LAUNCH();
        TRY_STATUS(argmax(AM_ROW));
        if (cudaMemsetAsync(cnt + 2, 0, sizeof(int), st) != cudaSuccess) return hodlr_set_cuda_error(cudaGetLastError());
        aca_row_check_kernel<<<bg, 128, 0, st>>>(g, cnt + 2);
        HODLR_CHECK_LAUNCH();
        if (!read_counts()) return hodlr_set_cuda_error(cudaGetLastError());
        if (host[2] == 0 || tries > g.nc + 2) break;
      }
      // column residual + rook sweeps
      aca_col_kernel<Oracle><<<eg, 256, 0, st>>>(g, A);
      HODLR_CHECK_LAUNCH();
      for (int sweep = 0; sweep < 4; ++sweep) {
        TRY_STATUS(argmax(AM_COL));
        aca_rook1_kernel<<<bg, 128, 0, st>>>(g);
        HODLR_CHECK_LAUNCH();
        aca_row_kernel<Oracle><<<eg, 256, 0, st>>>(g, A);
        HODLR_CHECK_LAUNCH();
        TRY_STATUS(argmax(AM_ROW));
        aca_rook2_kernel<<<bg, 128, 0, st>>>(g);
        HODLR_CHECK_LAUNCH();
        aca_col_kernel<Oracle><<<eg, 256, 0, st>>>(g, A);
        HODLR_CHECK_LAUNCH();
      }
      aca_pivot_kernel<<<bg, 128, 0, st>>>(g);
      HODLR_CHECK_LAUNCH();
      aca_append_kernel<<<eg, 256, 0, st>>>(g);
      HODLR_CHECK_LAUNCH();
      aca_mark_kernel<<<bg, 128, 0, st>>>(g);
      HODLR_CHECK_LAUNCH();
      TRY_STATUS(argmax(AM_COL));  // next row proposal on the updated row mask
      if (cudaMemsetAsync(cnt + 1, 0, sizeof(int), st) != cudaSuccess) return hodlr_set_cuda_error(cudaGetLastError());
      aca_advance_kernel<<<bg, 128, 0, st>>>(g, cnt + 1);
      HODLR_CHECK_LAUNCH();
      if (!read_counts()) return hodlr_set_cuda_error(cudaGetLastError());
      if (host[0]) return HODLR_ERR_ARG;  // non-finite oracle entry
      if (host[1] == 0) break;
    }
  }
  if (!read_counts()) return hodlr_set_cuda_error(cudaGetLastError());
  return host[0] ? HODLR_ERR_ARG : HODLR_OK;
}

}  // namespace
}  // namespace hodlr

using namespace hodlr;

extern "C" hodlr_status hodlr_xorshift_uniform(uint64_t seed, int64_t count, double* out, void* stream) {
  if (count < 0 || (count > 0 && !out)) return HODLR_ERR_ARG;
  if (count == 0) return HODLR_OK;
  xorshift_uniform_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(seed, count, out);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

extern "C" size_t hodlr_build_workspace(const hodlr_desc* d) { return build_desc_ok(d) ? build_ws(d).total : 0; }

extern "C" hodlr_status hodlr_build_laplace_dl(const hodlr_desc* d, const double* geom, void* D, void* U, void* V,
                                               void* work, size_t work_bytes, void* stream) {
  if (!build_desc_ok(d) || !geom || !D || !work || work_bytes < build_ws(d).total) return HODLR_ERR_ARG;
  if (d->L > 0 && d->r > 0 && (!U || !V)) return HODLR_ERR_ARG;
  const int64_t n = d->n;
  LaplaceDL A{geom, geom + n, geom + 2 * n, geom + 3 * n, geom + 4 * n, geom + 5 * n, geom + 6 * n};
  return build_run(d, A, (double*)D, (double*)U, (double*)V, static_cast<char*>(work), static_cast<cudaStream_t>(stream));
}

extern "C" hodlr_status hodlr_build_gaussian(const hodlr_desc* d, const double* pts, int dim, double h, double lambda,
                                             void* D, void* U, void* V, void* work, size_t work_bytes, void* stream) {
  if (!build_desc_ok(d) || !pts || dim < 1 || dim > 3 || !(h > 0.0) || !D || !work ||
      work_bytes < build_ws(d).total)
    return HODLR_ERR_ARG;
  if (d->L > 0 && d->r > 0 && (!U || !V)) return HODLR_ERR_ARG;
  GaussianPts A{pts, d->n, dim, h * h, lambda};
  return build_run(d, A, (double*)D, (double*)U, (double*)V, static_cast<char*>(work), static_cast<cudaStream_t>(stream));
}

extern "C" hodlr_status hodlr_build_schur_plane(const hodlr_desc* d, const double* pts, double sigma, void* D,
                                                 void* U, void* V, void* work, size_t work_bytes, void* stream) {
  if (!build_desc_ok(d) || !pts || !(sigma >= 0.0) || !D || !work || work_bytes < build_ws(d).total)
    return HODLR_ERR_ARG;
  if (d->L > 0 && d->r > 0 && (!U || !V)) return HODLR_ERR_ARG;
  SchurPlane A{pts, d->n, 2.8754826265883277 + sigma};
  return build_run(d, A, (double*)D, (double*)U, (double*)V, static_cast<char*>(work), static_cast<cudaStream_t>(stream));
}

extern "C" hodlr_status hodlr_build_dense(const hodlr_desc* d, const double* A, int64_t lda, void* D, void* U, void* V,
                                          void* work, size_t work_bytes, void* stream) {
  if (!build_desc_ok(d) || !A || lda < d->n || !D || !work || work_bytes < build_ws(d).total) return HODLR_ERR_ARG;
  if (d->L > 0 && d->r > 0 && (!U || !V)) return HODLR_ERR_ARG;
  DenseOracle O{A, lda};
  return build_run(d, O, (double*)D, (double*)U, (double*)V, static_cast<char*>(work), static_cast<cudaStream_t>(stream));
}
