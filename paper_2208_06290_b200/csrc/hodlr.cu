// C ABI + level-wise factorize / solve drivers (Alg. 3/4).
//
// Everything is enqueued on the caller's stream; no allocation, no host sync.
// Device layout is the reference's (include/hodlr_b200.h).  The factor keeps
// the reference outputs (leaf LU + pivots, Y slab, K LU + pivots per level) and
// additionally the packed triangular inverses strict_lower(L^-1) + upper(U^-1)
// of every leaf and K block, so every triangular solve of the factor and solve
// phases becomes a pair of batched DMMA GEMMs (apply.cu).
#include <climits>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "common.cuh"
#include "ranks.cuh"

namespace hodlr {
template <typename T>
hodlr_status launch_getrf(int s, int batch, int mode, const T* src, int64_t lds, int64_t strides, T* out, int64_t ldo,
                          int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, T* tinv, int64_t ldi,
                          int64_t stridei, cudaStream_t st);
hodlr_status tri_apply_f64(int s, int ncols, int batch, const double* lu, const double* tinv, int64_t ldi, int64_t strideT,
                           const int32_t* perm, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double* X,
                           int64_t ldx, int64_t sX_hi, int64_t sX_lo, int bdiv, cudaStream_t st,
                           const double* V = nullptr, int64_t ldv = 0, int64_t vstride = 0, int twr = 0,
                           double* TW = nullptr, int64_t tw_stride = 0, int narrow_cols = 8);
hodlr_status tri_apply_f32(int s, int ncols, int batch, const float* lu, int64_t strideT, const int32_t* perm, float* Y,
                           int64_t ldy, int64_t sY, const float* V, int64_t ldv, int64_t vstride, int twr, float* TW,
                           int64_t tw_stride, cudaStream_t st);
static inline hodlr_status tri_apply_f32(int, int, int, const double*, int64_t, const int32_t*, double*, int64_t,
                                         int64_t, const double*, int64_t, int64_t, int, double*, int64_t,
                                         cudaStream_t) {
  return HODLR_ERR_ARG;
}
hodlr_status level_update_f64(int r, int64_t n, int64_t n_c, int64_t node_rows, double* C, int64_t ldc,
                              const double* A1, const double* V, int64_t lda, const double* W, int64_t wstride,
                              int ncols, double* TW, int64_t tw_stride, double* part, size_t part_bytes,
                              cudaStream_t st, bool reg_resident);
size_t level_partial_bytes(int64_t n, int m, int r, int L);
size_t level_f32_partial_bytes(int64_t n, int ncols);
hodlr_status launch_getrf_dbi_f64(int s, int batch, int mode, const double* src, int64_t lds, int64_t strides,
                                  double* out, int64_t ldo, int64_t strideo, int32_t* swaps, int32_t* perm,
                                  int32_t* info, double* dbi, int64_t stridedbi, cudaStream_t st);
size_t solve_level_partial_bytes(int64_t n, int r, int nrhs);
hodlr_status solve_level_f64(int r, int64_t n, int64_t n_c, int64_t node_rows, double* X, int64_t ldx,
                             const double* A1, const double* V, int64_t lda, const double* W, int64_t wstride,
                             int nrhs, double* TW, int64_t tw_stride, double* part, size_t part_bytes,
                             cudaStream_t st);
int64_t level_segment_rows(int64_t n, int64_t node, int sms);
hodlr_status level_reduce_f64(const double* part, double* TW, int r, int ncols, int segs, int nnodes, int64_t tw_stride,
                              cudaStream_t st);
hodlr_status solve_step_f64(int r, int64_t n, int64_t n_c, int64_t node_rows, double* X, int64_t ldx, const double* Y,
                            const double* V, int64_t lda, const double* W, int64_t wstride, int nrhs, double* TW,
                            int64_t tw_stride, double* part, size_t part_bytes, int sms, bool* used_partial,
                            cudaStream_t st);
int device_sm_count();
hodlr_status level_f32(int r, int64_t n, int64_t n_c, int64_t node_rows, float* C, int64_t ldc, const float* A1,
                       const float* V, int64_t lda, const float* W, int64_t wstride, int ncols, float* TW,
                       int64_t tw_stride, float* part, size_t part_bytes, cudaStream_t st, int seg_max = 1024);
hodlr_status level_f32_dmma(int r, int64_t n, int64_t n_c, int64_t node_rows, float* C, int64_t ldc, const float* A1,
                            const float* V, int64_t lda, const float* W, int64_t wstride, int ncols, float* TW,
                            int64_t tw_stride, float* part, size_t part_bytes, cudaStream_t st);
hodlr_status gemm_f32(int transA, int M, int N, int K, float alpha, const float* A, int64_t lda, int64_t sA_hi,
                      int64_t sA_lo, const float* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, float beta, float* C,
                      int64_t ldc, int64_t sC_hi, int64_t sC_lo, int batch, int bdiv, void* work, size_t work_bytes,
                      cudaStream_t st);
template <typename T>
hodlr_status launch_getrs(int s, int nrhs, int batch, const T* LU, int64_t lda, int64_t strideA, const int32_t* perm,
                          const T* B, int64_t ldb, int64_t strideB, T* X, int64_t ldx, int64_t strideX, int identity,
                          cudaStream_t st);
hodlr_status gemm_f64(int transA, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sA_hi,
                      int64_t sA_lo, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double beta,
                      double* C, int64_t ldc, int64_t sC_hi, int64_t sC_lo, int batch, int bdiv, void* work,
                      size_t work_bytes, cudaStream_t st);
}  // namespace hodlr

using namespace hodlr;

static thread_local std::string g_last_error;

hodlr_status hodlr_set_cuda_error(cudaError_t e) {
  g_last_error = cudaGetErrorString(e);
  return HODLR_ERR_CUDA;
}

extern "C" const char* hodlr_version(void) { return "hodlr_b200 0.1 (sm_100a, fp64 DMMA)"; }
extern "C" const char* hodlr_last_error(void) { return g_last_error.c_str(); }
extern "C" size_t hodlr_inv_elems(int s) { return s < 0 ? 0 : (size_t)inv_block_elems(s); }

// ---- instrumentation ----
#include <atomic>
#include <vector>
static std::atomic<long long> g_launches{0};
void hodlr_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" long long hodlr_launch_count(void) { return g_launches.load(); }

namespace {
struct PhaseProfiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};
PhaseProfiler g_prof;
std::mutex g_prof_mu;

// RAII bracket: records start/stop events on `st` around one phase
struct Phase {
  cudaStream_t st;
  int cls;
  cudaEvent_t a = nullptr;
  Phase(int c, cudaStream_t s) : st(s), cls(c) {
    if (g_prof.on) {
      std::lock_guard<std::mutex> lk(g_prof_mu);
      a = g_prof.get();
      cudaEventRecord(a, st);
    }
  }
  ~Phase() {
    if (a) {
      std::lock_guard<std::mutex> lk(g_prof_mu);
      cudaEvent_t b = g_prof.get();
      cudaEventRecord(b, st);
      g_prof.recs.push_back({cls, a, b});
    }
  }
};
}  // namespace

extern "C" void hodlr_profile_enable(int on) { g_prof.on = on != 0; }

extern "C" int hodlr_profile_read(double* ms, int n) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int i = 0; i < n; ++i) ms[i] = 0.0;
  for (auto& r : g_prof.recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cls < n) ms[r.cls] += t;
  }
  g_prof.recs.clear();
  g_prof.used = 0;
  return HODLR_NUM_PHASES;
}

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

// split-K partial-sum area reserved inside every workspace
static constexpr size_t kSplitBytes = size_t(64) << 20;

static inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------------------
// batched kernels
// ---------------------------------------------------------------------------

extern "C" hodlr_status hodlr_getrf_batched(int dtype, int s, int batch, void* A, int64_t lda, int64_t strideA,
                                            int32_t* swaps, int32_t* perm, int32_t* info, void* Ainv, int64_t ldinv,
                                            int64_t strideInv, void* stream) {
  if (s < 0 || batch < 0 || (s > 0 && lda < s)) return HODLR_ERR_ARG;
  hodlr_status st;
  if (dtype == HODLR_F64) {
    st = launch_getrf<double>(s, batch, 0, (const double*)A, lda, strideA, (double*)A, lda, strideA, swaps, perm, info,
                              (double*)Ainv, ldinv, strideInv, S(stream));
  } else if (dtype == HODLR_F32) {
    st = launch_getrf<float>(s, batch, 0, (const float*)A, lda, strideA, (float*)A, lda, strideA, swaps, perm, info,
                             (float*)Ainv, ldinv, strideInv, S(stream));
  } else {
    return HODLR_ERR_ARG;
  }
  return st;
}

extern "C" hodlr_status hodlr_getrs_batched(int dtype, int s, int nrhs, int batch, const void* LU, int64_t lda,
                                            int64_t strideA, const int32_t* perm, void* B, int64_t ldb,
                                            int64_t strideB, void* stream) {
  if (s < 0 || nrhs < 0 || batch < 0) return HODLR_ERR_ARG;
  if (dtype == HODLR_F64)
    return launch_getrs<double>(s, nrhs, batch, (const double*)LU, lda, strideA, perm, (const double*)B, ldb, strideB,
                                (double*)B, ldb, strideB, 0, S(stream));
  if (dtype == HODLR_F32)
    return launch_getrs<float>(s, nrhs, batch, (const float*)LU, lda, strideA, perm, (const float*)B, ldb, strideB,
                               (float*)B, ldb, strideB, 0, S(stream));
  return HODLR_ERR_ARG;
}

extern "C" hodlr_status hodlr_gemm_batched(int dtype, int transA, int M, int N, int K, double alpha, const void* A,
                                           int64_t lda, int64_t sA_hi, int64_t sA_lo, const void* B, int64_t ldb,
                                           int64_t sB_hi, int64_t sB_lo, double beta, void* C, int64_t ldc,
                                           int64_t sC_hi, int64_t sC_lo, int batch, int bdiv, void* work,
                                           size_t work_bytes, void* stream) {
  if (dtype == HODLR_F32)
    return gemm_f32(transA, M, N, K, (float)alpha, (const float*)A, lda, sA_hi, sA_lo, (const float*)B, ldb, sB_hi,
                    sB_lo, (float)beta, (float*)C, ldc, sC_hi, sC_lo, batch, bdiv, work, work_bytes, S(stream));
  if (dtype != HODLR_F64) return HODLR_ERR_ARG;
  return gemm_f64(transA, M, N, K, alpha, (const double*)A, lda, sA_hi, sA_lo, (const double*)B, ldb, sB_hi, sB_lo,
                  beta, (double*)C, ldc, sC_hi, sC_lo, batch, bdiv, work, work_bytes, S(stream));
}

// ---------------------------------------------------------------------------
// factorize / solve
// ---------------------------------------------------------------------------

static bool tri_size_ok(int s) { return s == 16 || s == 32 || s == 64 || s == 128; }

static bool desc_ok(const hodlr_desc* d) {
  if (!d || d->m < 1 || d->r < 0 || d->L < 0 || d->L > 30) return false;
  if (d->m > 119 && !tri_size_ok(d->m)) return false;
  LevelRanks q;
  if (!make_ranks(d, q)) return false;
  for (int l = 1; l <= d->L; ++l)
    if (2 * q.r[l] > 119 && !tri_size_ok(2 * q.r[l])) return false;
  if (!q.uniform && d->dtype != HODLR_F64) return false;  // per-level ranks: the fp64 drivers
  return d->n == (int64_t)d->m << d->L;
}
// the row-sharded entry points and the fp32 drivers take uniform ranks
static bool uniform_desc(const hodlr_desc* d) { return d->ranks == nullptr; }

// Factor s x s blocks; for DMMA-supported sizes also emit the packed
// triangular inverses used by lu_apply.
static hodlr_status lu_factor(int s, int batch, int mode, const double* src, int64_t lds, int64_t strides, double* out,
                              int64_t strideo, int32_t* swaps, int32_t* perm, int32_t* info, double* tinv,
                              cudaStream_t st) {
  if (s == 32 || s == 64 || s == 128)  // diagonal-block inverses for the blocked DMMA substitutions
    return launch_getrf_dbi_f64(s, batch, mode, src, lds, strides, out, s, strideo, swaps, perm, info, tinv,
                                inv_block_elems(s), st);
  return launch_getrf<double>(s, batch, mode, src, lds, strides, out, s, strideo, swaps, perm, info,
                              tri_size_ok(s) ? tinv : nullptr, s, inv_block_elems(s), st);
}

// X_b = A_b^-1 B_b from the stored factors: two triangular DMMA GEMMs with the
// packed inverses, or row substitution for other block sizes.
static hodlr_status lu_apply(int s, int ncols, int batch, const double* LU, const double* tinv, const int32_t* perm,
                             const double* B, int64_t ldb, int64_t sB, double* X, int64_t ldx, int64_t sX,
                             cudaStream_t st, int narrow_cols = 8) {
  if (tri_size_ok(s)) {
    const hodlr_status r = tri_apply_f64(s, ncols, batch, LU, tinv, s, (int64_t)s * s, perm, B, ldb, sB, 0, X, ldx, sX,
                                         0, 1, st, nullptr, 0, 0, 0, nullptr, 0, narrow_cols);
    if (r != HODLR_ERR_ARG) return r;
  }
  return launch_getrs<double>(s, ncols, batch, LU, s, (int64_t)s * s, perm, B, ldb, sB, X, ldx, sX, 0, st);
}

// ---------------------------------------------------------------------------
// Row-sharded schedule.  A caller may hold only the rows [row0, row0 + n_loc)
// of a level-p node (n_loc = N / 2^p): its leaves' D, its rows of the Y / V
// slabs (ld n_loc), and the full K / K-pivot arrays (global level layout; the
// deep levels are filled for its own parents only, the top levels redundantly).
// Levels l >= p are then entirely local; for l < p the partial [W|T] / w of
// the caller's rows is exchanged (sum all-reduce) and hodlr_*_top finishes
// level l.  Single GPU: n_loc = N, row0 = 0, p = 0.
// ---------------------------------------------------------------------------

// workspace layout (factorize): [split-K | TW | W | level partial sums]
struct FactWs {
  size_t split, tw, w, part, total;
};
static FactWs fact_ws_local(const hodlr_desc* d, int64_t n_loc) {
  const int64_t r = d->r, L = d->L;
  const int64_t nleaf = n_loc / d->m;
  FactWs w{};
  w.split = kSplitBytes;
  w.tw = align_up(sizeof(double) * (size_t)std::max<int64_t>(nleaf, 2) * r * r * std::max<int64_t>(L, 1));
  w.w = align_up(sizeof(double) * (size_t)std::max<int64_t>(nleaf, 2) * r * r * std::max<int64_t>(L, 1));
  size_t part = level_partial_bytes(n_loc, d->m, (int)r, (int)L);
  // top levels: the caller's rows form one output node
  const int64_t seg = level_segment_rows(n_loc, n_loc, 148);
  part = std::max(part, (size_t)(n_loc / std::max<int64_t>(seg, 1)) * r * r * L * sizeof(double));
  if (d->dtype == HODLR_F32) part = std::max(part, level_f32_partial_bytes(n_loc, (int)(r * L)));
  w.part = align_up(part);
  w.total = w.split + w.tw + w.w + w.part;
  return w;
}
static FactWs fact_ws(const hodlr_desc* d) { return fact_ws_local(d, d->n); }

static bool local_ok(const hodlr_desc* d, int64_t n_loc, int64_t row0) {
  if (n_loc <= 0 || row0 < 0 || row0 + n_loc > d->n || n_loc % d->m) return false;
  if (d->n % n_loc || row0 % n_loc) return false;  // a whole level-p node
  return ((d->n / n_loc) & (d->n / n_loc - 1)) == 0;
}

extern "C" size_t hodlr_factorize_workspace(const hodlr_desc* d) { return desc_ok(d) ? fact_ws(d).total : 0; }
extern "C" size_t hodlr_factorize_local_workspace(const hodlr_desc* d, int64_t n_loc) {
  return desc_ok(d) && n_loc > 0 ? fact_ws_local(d, n_loc).total : 0;
}

static size_t solve_part_bytes(const hodlr_desc* d, int nrhs) {
  size_t b = std::max(sizeof(double) * (size_t)4 * 148 * d->r * nrhs, solve_level_partial_bytes(d->n, d->r, nrhs));
  if (d->dtype == HODLR_F32) b = std::max(b, level_f32_partial_bytes(d->n, nrhs));
  return align_up(b);
}

extern "C" size_t hodlr_solve_workspace(const hodlr_desc* d, int nrhs) {
  if (!desc_ok(d) || nrhs < 0) return 0;
  // split-K | w | w2 | level partial sums
  const size_t wsz = align_up(sizeof(double) * (size_t)std::max<int64_t>((int64_t)1 << d->L, 2) * d->r * nrhs);
  return kSplitBytes + 2 * wsz + solve_part_bytes(d, nrhs);
}

#define TRY(x)                            \
  do {                                    \
    hodlr_status s_ = (x);                \
    if (s_ != HODLR_OK) return s_;        \
  } while (0)

// Host-side gate between a staging upload (pageable host inputs) and the
// thread enqueueing the factorization: vready[l'] may only be waited on once
// the uploader has recorded it (an unrecorded event would not order anything).
struct UploadGate {
  std::mutex mu;
  std::condition_variable cv;
  int ready = INT_MAX;  // vready[l'] recorded for every l' >= ready
  bool failed = false;
  void publish(int lv) {
    std::lock_guard<std::mutex> lk(mu);
    ready = lv;
    cv.notify_all();
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    cv.notify_all();
  }
  bool wait(int lv) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return failed || ready <= lv; });
    return !failed;
  }
};

// Leaf phase + levels L-1 .. lv_stop over the local rows.  On return the
// workspace TW region holds [W|T] of the local level-lv_stop node(s) (paired
// layout, local node 0 first) unless lv_stop == 0.
// vready (optional): vready[l'] is recorded once the level-l' V panel
// (columns (l'-1) r .. l' r) is resident; the leaf phase needs vready[L],
// level l's update kernel vready[l] (streamed host upload, hodlr_factorize_from_host).
static hodlr_status factor_local(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0, int lv_stop,
                                 char* wp, const FactWs& ws, cudaStream_t st, const cudaEvent_t* vready = nullptr,
                                 UploadGate* gate = nullptr) {
  void* split = wp;
  double* TW = reinterpret_cast<double*>(wp + ws.split);
  double* W = reinterpret_cast<double*>(wp + ws.split + ws.tw);
  double* part = reinterpret_cast<double*>(wp + ws.split + ws.tw + ws.w);

  LevelRanks q;
  if (!make_ranks(d, q)) return HODLR_ERR_ARG;
  const int64_t N = d->n, n = n_loc;
  const int m = d->m, L = d->L;
  const int64_t C = q.cols();  // slab columns (r L when uniform)
  const int64_t nleaf = n / m;
  double* D = (double*)f->D;
  double* Dinv = (double*)f->Dinv;
  double* Y = (double*)f->Y;
  const double* V = (const double*)f->V;
  double* K = (double*)f->K;
  double* Kinv = (double*)f->Kinv;

  // (1) leaf getrf (bit-exact) + diagonal-block inverses          Alg.3 l.2
  if (gate && L > 0 && !gate->wait(L)) return HODLR_ERR_CUDA;
  if (vready && L > 0 && cudaStreamWaitEvent(st, vready[L], 0) != cudaSuccess)  // D, U and V^(L) resident
    return hodlr_set_cuda_error(cudaGetLastError());
  {
    Phase ph(HODLR_PHASE_LEAF_GETRF, st);
    TRY(lu_factor(m, (int)nleaf, 0, D, m, (int64_t)m * m, D, (int64_t)m * m, f->dswaps, f->dperm, f->dinfo, Dinv, st));
  }
  if (L == 0 || C == 0) return HODLR_OK;
  // (2) Y(I_a, :) <- D_a^-1 U(I_a, :) for all levels at once       Alg.3 l.3
  //     fused with the level-(L-1) [W|T]_a = V_a^T Y(I_a, 0:C)      Alg.3 l.5-6
  bool tw_ready = false;
  {
    Phase ph(HODLR_PHASE_LEAF_APPLY, st);
    const int rL = q.r[L];
    if (tri_size_ok(m) && rL > 0) {
      hodlr_status s = tri_apply_f64(m, (int)C, (int)nleaf, D, Dinv, m, (int64_t)m * m, f->dperm, Y, n, m, 0, Y, n, m, 0,
                                     1, st, V + q.c[L] * n, n, m, rL, TW, (int64_t)2 * rL * C);
      if (s == HODLR_OK) tw_ready = true;
      else if (s != HODLR_ERR_ARG) return s;
    }
    if (!tw_ready) TRY(lu_apply(m, (int)C, (int)nleaf, D, Dinv, f->dperm, Y, n, m, Y, n, m, st));
  }

  // (3) levels                                                     Alg.3 l.4-10
  for (int lv = L - 1; lv >= lv_stop; --lv) {
    const int64_t nc = N >> (lv + 1);
    const int nch = (int)(n / nc), npar = nch / 2;
    const int64_t p0 = row0 / (2 * nc);  // global index of the first local parent
    const int r = q.r[lv + 1];           // rank of the children (level lv + 1)
    const int ncol = (int)q.c[lv + 2], wc = (int)q.c[lv + 1];
    const int64_t kblk = ((int64_t)1 << lv) - 1 + p0;  // first local K block (global numbering)
    const int64_t koff = q.koff[lv] + p0 * 4 * r * r, kioff = q.kioff[lv] + p0 * inv_block_elems(2 * r);
    const int64_t kpoff = q.kpoff[lv] + p0 * 2 * r;
    if (r == 0) {  // a rank-0 level: K_p is the empty matrix, nothing to update
      tw_ready = false;
      continue;
    }
    if (!tw_ready) {
      Phase ph(HODLR_PHASE_GEMM, st);
      // [W|T]_c = V_c^T Y(I_c, 0:ncol), paired per parent: 2r x ncol, ld 2r
      TRY(gemm_f64(1, r, ncol, (int)nc, 1.0, V + q.c[lv + 1] * n, n, 2 * nc, nc, Y, n, 2 * nc, nc, 0.0, TW, 2 * r,
                   (int64_t)2 * r * ncol, r, nch, 2, split, ws.split, st));
    }
    // K_p = [[T_2p, I], [I, T_2p+1]] assembled + factored (bit-exact) + diagonal-block inverses
    int32_t* kperm = f->kperm + kpoff;
    {
      Phase ph(HODLR_PHASE_K_GETRF, st);
      TRY(lu_factor(2 * r, npar, 1, TW + (int64_t)wc * 2 * r, 2 * r, (int64_t)2 * r * ncol, K + koff,
                    (int64_t)4 * r * r, f->kswaps + kpoff, kperm, f->kinfo + kblk, Kinv + kioff, st));
    }
    if (lv == 0) break;
    if (wc == 0) {  // rank-0 levels above: no columns to update
      tw_ready = false;
      continue;
    }
    // W_p <- K_p^-1 [W_2p; W_2p+1]
    {
      Phase ph(HODLR_PHASE_K_APPLY, st);
      TRY(lu_apply(2 * r, wc, npar, K + koff, Kinv + kioff, kperm, TW, 2 * r, (int64_t)2 * r * ncol, W, 2 * r,
                   (int64_t)2 * r * wc, st));
    }
    // Y(I_c, 0:wc) -= Y_c^{l+1} W_c, fused with the next level's [W|T] (V^{(l)T} Y(I_q, 0:wc))
    // when both levels have the same rank (the fused kernel holds one rank)
    if (gate && !gate->wait(lv)) return HODLR_ERR_CUDA;
    if (vready && cudaStreamWaitEvent(st, vready[lv], 0) != cudaSuccess)  // V^(lv) resident (streamed upload)
      return hodlr_set_cuda_error(cudaGetLastError());
    hodlr_status s = HODLR_ERR_ARG;
    if (q.r[lv] == r) {
      Phase ph(HODLR_PHASE_LEVEL, st);
      s = level_update_f64(r, n, nc, 2 * nc, Y, n, Y + q.c[lv + 1] * n, V + q.c[lv] * n, n, W, (int64_t)2 * r * wc,
                           wc, TW, (int64_t)2 * r * wc, part, ws.part, st, true);
    }
    if (s == HODLR_OK) {
      tw_ready = true;
      continue;
    }
    if (s != HODLR_ERR_ARG) return s;
    tw_ready = false;
    Phase ph(HODLR_PHASE_GEMM, st);
    TRY(gemm_f64(0, (int)nc, wc, r, -1.0, Y + q.c[lv + 1] * n, n, 2 * nc, nc, W, 2 * r, (int64_t)2 * r * wc, r, 1.0,
                 Y, n, 2 * nc, nc, nch, 2, split, ws.split, st));
  }
  if (!tw_ready && lv_stop > 0) {
    // the caller wants the level-lv_stop [W|T] in the workspace (uniform ranks: the sharded path)
    const int lv = lv_stop - 1;
    const int64_t nc = N >> (lv + 1);
    const int nch = (int)(n / nc);
    const int r = q.r[lv + 1];
    if (nch >= 1 && nc <= n && r > 0) {
      Phase ph(HODLR_PHASE_GEMM, st);
      const int ncol = (int)q.c[lv + 2];
      TRY(gemm_f64(1, r, ncol, (int)std::min<int64_t>(nc, n), 1.0, V + q.c[lv + 1] * n, n, 2 * nc, nc, Y, n, 2 * nc,
                   nc, 0.0, TW, 2 * r, (int64_t)2 * r * ncol, r, std::max(nch, 1), 2, split, ws.split, st));
    }
  }
  return HODLR_OK;
}

// ---------------------------------------------------------------------------
// Generic-precision drivers (fp32: the low-accuracy preconditioner config).
// The SPEC recipe issued as batched kernels only:
// bit-exact getrf, substitution getrs, batched GEMMs.  No packed inverses, no
// fused level kernels (those are the fp64 DMMA path).
// ---------------------------------------------------------------------------
static hodlr_status gemm_T(int transA, int M, int N, int K, double alpha, const float* A, int64_t lda, int64_t sAh,
                           int64_t sAl, const float* B, int64_t ldb, int64_t sBh, int64_t sBl, double beta, float* C,
                           int64_t ldc, int64_t sCh, int64_t sCl, int batch, int bdiv, void* w, size_t wb,
                           cudaStream_t st) {
  return gemm_f32(transA, M, N, K, (float)alpha, A, lda, sAh, sAl, B, ldb, sBh, sBl, (float)beta, C, ldc, sCh, sCl,
                  batch, bdiv, w, wb, st);
}
static hodlr_status gemm_T(int transA, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sAh,
                           int64_t sAl, const double* B, int64_t ldb, int64_t sBh, int64_t sBl, double beta, double* C,
                           int64_t ldc, int64_t sCh, int64_t sCl, int batch, int bdiv, void* w, size_t wb,
                           cudaStream_t st) {
  return gemm_f64(transA, M, N, K, alpha, A, lda, sAh, sAl, B, ldb, sBh, sBl, beta, C, ldc, sCh, sCl, batch, bdiv, w,
                  wb, st);
}

// fused rank-8 fp32 level step where it applies (level_f32.cu), else ERR_ARG
static hodlr_status level_T(int r, int64_t n, int64_t n_c, int64_t node_rows, float* C, int64_t ldc, const float* A1,
                            const float* V, int64_t lda, const float* W, int64_t wstride, int ncols, float* TW,
                            int64_t tw_stride, float* part, size_t part_bytes, cudaStream_t st, int seg_max = 1024) {
  return level_f32(r, n, n_c, node_rows, C, ldc, A1, V, lda, W, wstride, ncols, TW, tw_stride, part, part_bytes, st,
                   seg_max);
}
static hodlr_status level_T(int, int64_t, int64_t, int64_t, double*, int64_t, const double*, const double*, int64_t,
                            const double*, int64_t, int, double*, int64_t, double*, size_t, cudaStream_t, int = 0) {
  return HODLR_ERR_ARG;
}
// factorization level step: the fp64-DMMA rank-8 kernel first, else the SIMT one
static hodlr_status level_fact_T(int r, int64_t n, int64_t n_c, int64_t node_rows, float* C, int64_t ldc,
                                 const float* A1, const float* V, int64_t lda, const float* W, int64_t wstride,
                                 int ncols, float* TW, int64_t tw_stride, float* part, size_t part_bytes,
                                 cudaStream_t st) {
  {
    const hodlr_status s = level_f32_dmma(r, n, n_c, node_rows, C, ldc, A1, V, lda, W, wstride, ncols, TW, tw_stride,
                                          part, part_bytes, st);
    if (s != HODLR_ERR_ARG) return s;
  }
  return level_f32(r, n, n_c, node_rows, C, ldc, A1, V, lda, W, wstride, ncols, TW, tw_stride, part, part_bytes, st);
}
static hodlr_status level_fact_T(int, int64_t, int64_t, int64_t, double*, int64_t, const double*, const double*,
                                 int64_t, const double*, int64_t, int, double*, int64_t, double*, size_t,
                                 cudaStream_t) {
  return HODLR_ERR_ARG;
}

template <typename T>
static hodlr_status factor_generic(const hodlr_desc* d, const hodlr_factors* f, char* wp, const FactWs& ws,
                                   cudaStream_t st) {
  void* split = wp;
  T* TW = reinterpret_cast<T*>(wp + ws.split);
  T* W = reinterpret_cast<T*>(wp + ws.split + ws.tw);
  const int64_t N = d->n;
  const int m = d->m, r = d->r, L = d->L;
  const int64_t nleaf = N / m;
  T* D = (T*)f->D;
  T* Y = (T*)f->Y;
  const T* V = (const T*)f->V;
  T* K = (T*)f->K;
  {
    Phase ph(HODLR_PHASE_LEAF_GETRF, st);
    TRY(launch_getrf<T>(m, (int)nleaf, 0, D, m, (int64_t)m * m, D, m, (int64_t)m * m, f->dswaps, f->dperm, f->dinfo,
                        nullptr, 0, 0, st));
  }
  if (L == 0 || r == 0) return HODLR_OK;
  T* part = reinterpret_cast<T*>(wp + ws.split + ws.tw + ws.w);
  bool tw_ready = false;
  {
    Phase ph(HODLR_PHASE_LEAF_APPLY, st);
    hodlr_status s = HODLR_ERR_ARG;
    if constexpr (sizeof(T) == 4) {  // fp64 DMMA chain on fp32 operands, fused leaf-level [W|T]
      const bool fuse = r == 8;
      s = tri_apply_f32(m, r * L, (int)nleaf, D, (int64_t)m * m, f->dperm, Y, N, m,
                        fuse ? V + (int64_t)(L - 1) * r * N : nullptr, N, m, r, fuse ? TW : nullptr,
                        (int64_t)2 * r * r * L, st);
      if (s == HODLR_OK) tw_ready = fuse;
      else if (s != HODLR_ERR_ARG) return s;
    }
    if (s != HODLR_OK)
      TRY(launch_getrs<T>(m, r * L, (int)nleaf, D, m, (int64_t)m * m, f->dperm, Y, N, m, Y, N, m, 0, st));
  }
  if (!tw_ready) {  // leaf-level [W|T]_a = V_a^T Y(I_a, :) by the fused kernel (no update)
    Phase ph(HODLR_PHASE_LEVEL, st);
    const hodlr_status s = level_T(r, N, m, m, Y, N, nullptr, V + (int64_t)(L - 1) * r * N, N, nullptr, 0, r * L, TW,
                                   (int64_t)2 * r * r * L, part, ws.part, st);
    if (s == HODLR_OK) tw_ready = true;
    else if (s != HODLR_ERR_ARG) return s;
  }
  for (int lv = L - 1; lv >= 0; --lv) {
    const int64_t nc = N >> (lv + 1);
    const int nch = 2 << lv, npar = 1 << lv;
    const int ncol = r * (lv + 1), wc = r * lv;
    const int64_t kblk = (int64_t)npar - 1, koff = kblk * 4 * r * r;
    if (!tw_ready) {
      Phase ph(HODLR_PHASE_GEMM, st);
      TRY(gemm_T(1, r, ncol, (int)nc, 1.0, V + (int64_t)lv * r * N, N, 2 * nc, nc, Y, N, 2 * nc, nc, 0.0, TW, 2 * r,
                 (int64_t)2 * r * ncol, r, nch, 2, split, ws.split, st));
    }
    {
      Phase ph(HODLR_PHASE_K_GETRF, st);
      TRY(launch_getrf<T>(2 * r, npar, 1, TW + (int64_t)wc * 2 * r, 2 * r, (int64_t)2 * r * ncol, K + koff, 2 * r,
                          (int64_t)4 * r * r, f->kswaps + kblk * 2 * r, f->kperm + kblk * 2 * r, f->kinfo + kblk,
                          nullptr, 0, 0, st));
    }
    if (lv == 0) break;
    {
      Phase ph(HODLR_PHASE_K_APPLY, st);
      TRY(launch_getrs<T>(2 * r, wc, npar, K + koff, 2 * r, (int64_t)4 * r * r, f->kperm + kblk * 2 * r, TW, 2 * r,
                          (int64_t)2 * r * ncol, W, 2 * r, (int64_t)2 * r * wc, 0, st));
    }
    {  // update + the next level's [W|T], fused when it applies
      Phase ph(HODLR_PHASE_LEVEL, st);
      const hodlr_status s = level_fact_T(r, N, nc, 2 * nc, Y, N, Y + (int64_t)lv * r * N,
                                          V + (int64_t)(lv - 1) * r * N, N, W, (int64_t)2 * r * wc, wc, TW,
                                          (int64_t)2 * r * wc, part, ws.part, st);
      if (s == HODLR_OK) {
        tw_ready = true;
        continue;
      }
      if (s != HODLR_ERR_ARG) return s;
      tw_ready = false;
    }
    {
      Phase ph(HODLR_PHASE_GEMM, st);
      TRY(gemm_T(0, (int)nc, wc, r, -1.0, Y + (int64_t)lv * r * N, N, 2 * nc, nc, W, 2 * r, (int64_t)2 * r * wc, r,
                 1.0, Y, N, 2 * nc, nc, nch, 2, split, ws.split, st));
    }
  }
  return HODLR_OK;
}

// fp32 solve: shorter fixed row segments than the factorization (few columns
// -> more warps); fixed for every nrhs, so columns stay bit-identical
constexpr int kSolveSeg = 256;

template <typename T>
static hodlr_status solve_generic(const hodlr_desc* d, const hodlr_factors* f, T* X, int64_t ldx, int nrhs, char* wp,
                                  cudaStream_t st) {
  const int64_t N = d->n;
  const int m = d->m, r = d->r, L = d->L;
  const size_t wsz = align_up(sizeof(double) * (size_t)std::max<int64_t>((int64_t)1 << L, 2) * r * nrhs);
  void* split = wp;
  T* w = reinterpret_cast<T*>(wp + kSplitBytes);
  T* w2 = reinterpret_cast<T*>(wp + kSplitBytes + wsz);
  const T* D = (const T*)f->D;
  const T* Y = (const T*)f->Y;
  const T* V = (const T*)f->V;
  const T* K = (const T*)f->K;
  {
    Phase ph(HODLR_PHASE_SOLVE_LEAF, st);
    TRY(launch_getrs<T>(m, nrhs, (int)(N / m), D, m, (int64_t)m * m, f->dperm, X, ldx, m, X, ldx, m, 0, st));
  }
  if (r == 0 || L == 0) return HODLR_OK;
  T* part = reinterpret_cast<T*>(wp + kSplitBytes + 2 * wsz);
  const size_t part_bytes = solve_part_bytes(d, nrhs);
  bool w_ready = false;
  {
    Phase ph(HODLR_PHASE_SOLVE_LEVEL, st);
    const hodlr_status s = level_T(r, N, m, m, X, ldx, nullptr, V + (int64_t)(L - 1) * r * N, N, nullptr, 0, nrhs, w,
                                   (int64_t)2 * r * nrhs, part, part_bytes, st, kSolveSeg);
    if (s == HODLR_OK) w_ready = true;
    else if (s != HODLR_ERR_ARG) return s;
  }
  for (int lv = L - 1; lv >= 0; --lv) {
    const int64_t nc = N >> (lv + 1);
    const int nch = 2 << lv, npar = 1 << lv;
    const int64_t kblk = (int64_t)npar - 1, koff = kblk * 4 * r * r;
    if (!w_ready) {
      Phase ph(HODLR_PHASE_GEMM, st);
      TRY(gemm_T(1, r, nrhs, (int)nc, 1.0, V + (int64_t)lv * r * N, N, 2 * nc, nc, X, ldx, 2 * nc, nc, 0.0, w, 2 * r,
                 (int64_t)2 * r * nrhs, r, nch, 2, split, kSplitBytes, st));
    }
    {
      Phase ph(HODLR_PHASE_SOLVE_K, st);
      TRY(launch_getrs<T>(2 * r, nrhs, npar, K + koff, 2 * r, (int64_t)4 * r * r, f->kperm + kblk * 2 * r, w, 2 * r,
                          (int64_t)2 * r * nrhs, w2, 2 * r, (int64_t)2 * r * nrhs, 0, st));
    }
    {
      Phase ph(HODLR_PHASE_SOLVE_LEVEL, st);
      const hodlr_status s = level_T(r, N, nc, 2 * nc, X, ldx, Y + (int64_t)lv * r * N,
                                     lv > 0 ? V + (int64_t)(lv - 1) * r * N : nullptr, N, w2, (int64_t)2 * r * nrhs,
                                     nrhs, w, (int64_t)2 * r * nrhs, part, part_bytes, st, kSolveSeg);
      if (s == HODLR_OK) {
        w_ready = true;
        continue;
      }
      if (s != HODLR_ERR_ARG) return s;
      w_ready = false;
    }
    {
      Phase ph(HODLR_PHASE_GEMM, st);
      TRY(gemm_T(0, (int)nc, nrhs, r, -1.0, Y + (int64_t)lv * r * N, N, 2 * nc, nc, w2, 2 * r, (int64_t)2 * r * nrhs,
                 r, 1.0, X, ldx, 2 * nc, nc, nch, 2, split, kSplitBytes, st));
    }
  }
  return HODLR_OK;
}

extern "C" hodlr_status hodlr_factorize(const hodlr_desc* d, const hodlr_factors* f, void* work, size_t work_bytes,
                                        void* stream) {
  if (!desc_ok(d) || !f) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64 && d->dtype != HODLR_F32) return HODLR_ERR_ARG;
  const FactWs ws = fact_ws(d);
  if (work_bytes < ws.total || !work) return HODLR_ERR_ARG;
  if (d->dtype == HODLR_F32) return factor_generic<float>(d, f, static_cast<char*>(work), ws, S(stream));
  return factor_local(d, f, d->n, 0, 0, static_cast<char*>(work), ws, S(stream));
}

// Factorization from host buffers with the upload overlapped: D, U and V^(L)
// are copied first on copy_stream, then the V panels in the order the levels
// consume them (V^(L-1) ... V^(1)); the compute on `stream` waits per level,
// so all but the first 4.6 GB (cfg2) of the transfer hide behind the
// factorization.  f's D / Y / V are the device destinations (Y receives U).
//
// Pinned inputs are copied directly.  Pageable inputs (e.g. numpy arrays) go
// through a pinned staging ring: kStageThreads host threads copy each 64 MB
// chunk into a free slot, the caller's thread issues that slot's H2D copy and
// records the event gating the slot's reuse; meanwhile a second host thread
// enqueues the factorization, blocking (UploadGate) until each level's V
// panel event has been recorded.  The call returns once every byte has left
// the caller's buffers (they may be freed at once).
static std::mutex g_up_mu;
static std::map<int, std::vector<cudaEvent_t>> g_up_ev;  // per device: events live in that device's context

namespace {
constexpr int kStageSlots = 4;
constexpr size_t kStageBytes = (size_t)64 << 20;
struct StageRing {
  void* slot[kStageSlots] = {};
  cudaEvent_t ev[kStageSlots] = {};
  int next = 0;
  bool ready = false;
};
std::map<int, StageRing> g_stage;  // per device, under g_up_mu; kept for the process

// memcpy of one chunk split over T host threads (the caller is thread 0)
class CopyPool {
 public:
  explicit CopyPool(int T) : T_(T) {
    for (int i = 1; i < T_; ++i) th_.emplace_back([this, i] { worker(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(char* dst, const char* src, size_t len) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = dst, src_ = src, len_ = len, pending_ = T_ - 1, ++gen_;
    }
    cv_.notify_all();
    piece(0, dst, src, len);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  void piece(int i, char* dst, const char* src, size_t len) const {
    const size_t per = ((len + T_ - 1) / T_ + 4095) & ~(size_t)4095;
    const size_t off = (size_t)i * per;
    if (off < len) std::memcpy(dst + off, src + off, std::min(per, len - off));
  }
  void worker(int i) {
    int seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return quit_ || gen_ != seen; });
      if (quit_) return;
      seen = gen_;
      char* d = dst_;
      const char* s = src_;
      const size_t l = len_;
      lk.unlock();
      piece(i, d, s, l);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int T_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
  int gen_ = 0, pending_ = 0;
  bool quit_ = false;
};

bool host_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}
}  // namespace

extern "C" hodlr_status hodlr_factorize_from_host(const hodlr_desc* d, const hodlr_factors* f, const void* D_host,
                                                  const void* U_host, const void* V_host, void* work,
                                                  size_t work_bytes, void* stream, void* copy_stream) {
  if (!desc_ok(d) || !uniform_desc(d) || !f || !D_host || !U_host || !V_host) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64) return HODLR_ERR_ARG;
  const FactWs ws = fact_ws(d);
  if (work_bytes < ws.total || !work) return HODLR_ERR_ARG;
  cudaStream_t st = S(stream), cs = S(copy_stream);
  const int64_t n = d->n;
  const int m = d->m, r = d->r, L = d->L;
  const size_t es = sizeof(double);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return hodlr_set_cuda_error(cudaGetLastError());
  std::lock_guard<std::mutex> lk(g_up_mu);
  std::vector<cudaEvent_t>& ev = g_up_ev[dev];
  while ((int)ev.size() < L + 2) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return hodlr_set_cuda_error(cudaGetLastError());
    ev.push_back(e);
  }
  auto ok_ = [](cudaError_t e) { return e == cudaSuccess; };
  const bool pD = host_pageable(D_host), pU = host_pageable(U_host), pV = host_pageable(V_host);
  const bool staged = pD || pU || pV;
  StageRing* ring = nullptr;
  if (staged) {
    ring = &g_stage[dev];
    if (!ring->ready) {
      for (int k = 0; k < kStageSlots; ++k)
        if (cudaHostAlloc(&ring->slot[k], kStageBytes, cudaHostAllocDefault) != cudaSuccess ||
            cudaEventCreateWithFlags(&ring->ev[k], cudaEventDisableTiming) != cudaSuccess)
          return hodlr_set_cuda_error(cudaGetLastError());
      ring->ready = true;
    }
  }
  // the copies must not start before the caller's prior work on `stream`
  if (!ok_(cudaEventRecord(ev[L + 1], st)) || !ok_(cudaStreamWaitEvent(cs, ev[L + 1], 0)))
    return hodlr_set_cuda_error(cudaGetLastError());
  const int nthreads = staged ? (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1;
  std::unique_ptr<CopyPool> pool(staged ? new CopyPool(nthreads) : nullptr);
  auto cp = [&](void* dst, const void* src, size_t bytes, bool pageable) {
    if (!pageable) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs) == cudaSuccess;
    for (size_t off = 0; off < bytes; off += kStageBytes) {
      const size_t len = std::min(kStageBytes, bytes - off);
      const int k = ring->next;
      ring->next = (k + 1) % kStageSlots;
      if (cudaEventSynchronize(ring->ev[k]) != cudaSuccess) return false;  // the slot's previous copy has landed
      pool->copy(static_cast<char*>(ring->slot[k]), static_cast<const char*>(src) + off, len);
      if (cudaMemcpyAsync(static_cast<char*>(dst) + off, ring->slot[k], len, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
          cudaEventRecord(ring->ev[k], cs) != cudaSuccess)
        return false;
    }
    return true;
  };
  // staged: the factorization is enqueued by a second host thread while this one uploads
  UploadGate gate;
  hodlr_status fs = HODLR_OK;
  std::thread compute;
  if (staged && L > 0)
    compute = std::thread([&] {
      if (cudaSetDevice(dev) != cudaSuccess) {
        fs = hodlr_set_cuda_error(cudaGetLastError());
        return;
      }
      fs = factor_local(d, f, n, 0, 0, static_cast<char*>(work), ws, st, ev.data(), &gate);
    });
  auto finish = [&](hodlr_status s) {
    if (s != HODLR_OK) gate.fail();
    if (compute.joinable()) compute.join();
    return s != HODLR_OK ? s : fs;
  };
  const size_t panel = (size_t)n * r * es;
  bool ok = cp(f->D, D_host, (size_t)n * m * es, pD) && cp(f->Y, U_host, (size_t)L * panel, pU);
  if (L > 0)
    ok = ok && cp((char*)f->V + (size_t)(L - 1) * panel, (const char*)V_host + (size_t)(L - 1) * panel, panel, pV);
  ok = ok && ok_(cudaEventRecord(ev[L > 0 ? L : 0], cs));
  if (!ok) return finish(hodlr_set_cuda_error(cudaGetLastError()));
  gate.publish(L);
  for (int lv = L - 1; lv >= 1; --lv) {
    if (!cp((char*)f->V + (size_t)(lv - 1) * panel, (const char*)V_host + (size_t)(lv - 1) * panel, panel, pV) ||
        !ok_(cudaEventRecord(ev[lv], cs)))
      return finish(hodlr_set_cuda_error(cudaGetLastError()));
    gate.publish(lv);
  }
  if (compute.joinable()) return finish(HODLR_OK);
  if (L == 0 && !ok_(cudaStreamWaitEvent(st, ev[0], 0))) return hodlr_set_cuda_error(cudaGetLastError());
  return factor_local(d, f, n, 0, 0, static_cast<char*>(work), ws, st, ev.data());
}

extern "C" hodlr_status hodlr_factorize_local(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0,
                                              int lv_stop, double* tw_out, void* work, size_t work_bytes,
                                              void* stream) {
  if (!desc_ok(d) || !uniform_desc(d) || !f || !local_ok(d, n_loc, row0)) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64 || lv_stop < 0 || lv_stop > d->L) return HODLR_ERR_ARG;
  if ((d->n >> lv_stop) > n_loc) return HODLR_ERR_ARG;  // levels >= lv_stop must be local
  const FactWs ws = fact_ws_local(d, n_loc);
  if (work_bytes < ws.total || !work) return HODLR_ERR_ARG;
  cudaStream_t st = S(stream);
  TRY(factor_local(d, f, n_loc, row0, lv_stop, static_cast<char*>(work), ws, st));
  if (tw_out && lv_stop > 0 && d->r > 0) {
    // [W|T] of the caller's level-lv_stop node: r x r*lv_stop, ld r
    const double* TW = reinterpret_cast<const double*>(static_cast<char*>(work) + ws.split);
    const int r = d->r, nc = r * lv_stop;
    if (cudaMemcpy2DAsync(tw_out, sizeof(double) * r, TW, sizeof(double) * 2 * r, sizeof(double) * r, nc,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return hodlr_set_cuda_error(cudaGetLastError());
  }
  return HODLR_OK;
}

// Finish level lv < p for the caller's rows.  tw_all: complete [W|T] of all
// 2^(lv+1) children at level lv+1 (paired per parent: 2r x r(lv+1), ld 2r,
// parent stride 2r*r(lv+1)) after the all-reduce.  Factors all 2^lv K blocks
// (redundant on every rank), applies K_p^-1 for the caller's parent, updates
// its rows of Y(:, 0:r lv) and writes the caller's partial [W|T] of its
// level-lv node (r x r lv, ld r) to tw_out (lv > 0).
extern "C" hodlr_status hodlr_factorize_top(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0,
                                            int lv, const double* tw_all, double* tw_out, void* work,
                                            size_t work_bytes, void* stream) {
  if (!desc_ok(d) || !uniform_desc(d) || !f || !local_ok(d, n_loc, row0) || !tw_all) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64 || lv < 0 || lv >= d->L || (d->n >> (lv + 1)) < n_loc) return HODLR_ERR_ARG;
  const FactWs ws = fact_ws_local(d, n_loc);
  if (work_bytes < ws.total || !work) return HODLR_ERR_ARG;
  cudaStream_t st = S(stream);
  char* wp = static_cast<char*>(work);
  double* W = reinterpret_cast<double*>(wp + ws.split + ws.tw);
  double* part = reinterpret_cast<double*>(wp + ws.split + ws.tw + ws.w);
  const int64_t N = d->n, n = n_loc;
  const int r = d->r;
  const int npar = 1 << lv, ncol = r * (lv + 1), wc = r * lv;
  const int64_t kblk = (int64_t)npar - 1;
  double* K = (double*)f->K + kblk * 4 * r * r;
  const int64_t kis = inv_block_elems(2 * r);
  double* Kinv = (double*)f->Kinv + kblk * kis;
  int32_t* kperm = f->kperm + kblk * 2 * r;
  {
    Phase ph(HODLR_PHASE_K_GETRF, st);
    TRY(lu_factor(2 * r, npar, 1, tw_all + (int64_t)wc * 2 * r, 2 * r, (int64_t)2 * r * ncol, K, (int64_t)4 * r * r,
                  f->kswaps + kblk * 2 * r, kperm, f->kinfo + kblk, Kinv, st));
  }
  if (lv == 0) return HODLR_OK;
  const int64_t nc = N >> (lv + 1);
  const int64_t p = row0 / (2 * nc), half = (row0 / nc) & 1;
  {
    Phase ph(HODLR_PHASE_K_APPLY, st);
    TRY(lu_apply(2 * r, wc, 1, K + p * 4 * r * r, Kinv + p * kis, kperm + p * 2 * r,
                 tw_all + p * 2 * r * ncol, 2 * r, 0, W, 2 * r, 0, st));
  }
  double* Y = (double*)f->Y;
  const double* V = (const double*)f->V;
  Phase ph(HODLR_PHASE_LEVEL, st);
  double* TWws = reinterpret_cast<double*>(wp + ws.split);
  hodlr_status s = level_update_f64(r, n, nc, n, Y, n, Y + (int64_t)lv * r * n, V + (int64_t)(lv - 1) * r * n, n,
                                    W + half * r, 0, wc, TWws, 0, part, ws.part, st, true);
  if (s == HODLR_OK) {
    if (cudaMemcpy2DAsync(tw_out, sizeof(double) * r, TWws, sizeof(double) * 2 * r, sizeof(double) * r, wc,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return hodlr_set_cuda_error(cudaGetLastError());
    return HODLR_OK;
  }
  if (s != HODLR_ERR_ARG) return s;
  // generic path: update, then the partial [W|T] over all local rows
  TRY(gemm_f64(0, (int)n, wc, r, -1.0, Y + (int64_t)lv * r * n, n, 0, 0, W + half * r, 2 * r, 0, 0, 1.0, Y, n, 0, 0,
               1, 1, wp, ws.split, st));
  return gemm_f64(1, r, wc, (int)n, 1.0, V + (int64_t)(lv - 1) * r * n, n, 0, 0, Y, n, 0, 0, 0.0, tw_out, r, 0, 0, 1,
                  1, wp, ws.split, st);
}

// the TMA-fed persistent solve level step (solve.cu) before the streaming kernels
#ifndef HODLR_SOLVE_STEP_TMA
#define HODLR_SOLVE_STEP_TMA 1
#endif
constexpr bool kSolveStepTma = HODLR_SOLVE_STEP_TMA;

// right-hand sides up to which the solve's triangular applies use the narrow
// kernel (a warp per block and 8-column group; the block's factors read once)
#ifndef HODLR_SOLVE_NARROW_COLS
#define HODLR_SOLVE_NARROW_COLS 32
#endif
constexpr int kSolveNarrowCols = HODLR_SOLVE_NARROW_COLS;

// Leaf solve + levels L-1 .. lv_stop over the caller's rows of X (ld ldx).
// On return the workspace w region holds w of the local level-lv_stop node
// (paired layout, local node 0) when lv_stop > 0.
static hodlr_status solve_local(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0, int lv_stop,
                                double* X, int64_t ldx, int nrhs, char* wp, cudaStream_t st) {
  LevelRanks q;
  if (!make_ranks(d, q)) return HODLR_ERR_ARG;
  const int64_t N = d->n, n = n_loc;
  const int m = d->m, L = d->L;
  const size_t wsz = align_up(sizeof(double) * (size_t)std::max<int64_t>((int64_t)1 << L, 2) * q.rmax * nrhs);
  void* split = wp;
  double* w = reinterpret_cast<double*>(wp + kSplitBytes);
  double* w2 = reinterpret_cast<double*>(wp + kSplitBytes + wsz);
  double* part = reinterpret_cast<double*>(wp + kSplitBytes + 2 * wsz);
  const double* Y = (const double*)f->Y;
  const double* V = (const double*)f->V;
  const double* Kinv = (const double*)f->Kinv;
  const int64_t nleaf = n / m;

  // x <- D^-1 x, fused with the level-(L-1) w_a = V_a^T x_a        Alg.4 l.3 (+ l.5)
  bool w_ready = false;
  {
    Phase ph(HODLR_PHASE_SOLVE_LEAF, st);
    const int rL = L > 0 ? q.r[L] : 0;
    if (rL > 0 && tri_size_ok(m)) {
      hodlr_status s = tri_apply_f64(m, nrhs, (int)nleaf, (const double*)f->D, (const double*)f->Dinv, m,
                                     (int64_t)m * m, f->dperm, X, ldx, m, 0, X, ldx, m, 0, 1, st, V + q.c[L] * n, n, m,
                                     rL, w, (int64_t)2 * rL * nrhs, kSolveNarrowCols);
      if (s == HODLR_OK) w_ready = true;
      else if (s != HODLR_ERR_ARG) return s;
    }
    if (!w_ready)
      TRY(lu_apply(m, nrhs, (int)nleaf, (const double*)f->D, (const double*)f->Dinv, f->dperm, X, ldx, m, X, ldx, m,
                   st, kSolveNarrowCols));
  }
  if (q.cols() == 0 || L == 0) return HODLR_OK;
  for (int lv = L - 1; lv >= lv_stop; --lv) {
    const int64_t nc = N >> (lv + 1);
    const int nch = (int)(n / nc), npar = nch / 2;
    const int64_t p0 = row0 / (2 * nc);
    const int r = q.r[lv + 1];
    if (r == 0) {
      w_ready = false;
      continue;
    }
    const int64_t koff = q.koff[lv] + p0 * 4 * r * r, kioff = q.kioff[lv] + p0 * inv_block_elems(2 * r);
    const int64_t kpoff = q.kpoff[lv] + p0 * 2 * r;
    // w_c = V_c^T x_c  (paired per parent, 2r x nrhs, ld 2r)       Alg.4 l.5
    if (!w_ready) {
      Phase ph(HODLR_PHASE_GEMM, st);
      TRY(gemm_f64(1, r, nrhs, (int)nc, 1.0, V + q.c[lv + 1] * n, n, 2 * nc, nc, X, ldx, 2 * nc, nc, 0.0, w, 2 * r,
                   (int64_t)2 * r * nrhs, r, nch, 2, split, kSplitBytes, st));
    }
    // w_p <- K_p^-1 w_p                                              Alg.4 l.6
    {
      Phase ph(HODLR_PHASE_SOLVE_K, st);
      TRY(lu_apply(2 * r, nrhs, npar, (const double*)f->K + koff, Kinv + kioff, f->kperm + kpoff, w, 2 * r,
                   (int64_t)2 * r * nrhs, w2, 2 * r, (int64_t)2 * r * nrhs, st, kSolveNarrowCols));
    }
    // x_c -= Y_c w_c  fused with the next level's w = V^{(l)T} x    Alg.4 l.7 (+ l.5 of level l-1)
    // (fused when the next level has the same rank)
    const bool next_same = lv == 0 || q.r[lv] == r;
    const double* Vn = lv > 0 && next_same ? V + q.c[lv] * n : nullptr;
    hodlr_status s;
    {
      Phase ph(HODLR_PHASE_SOLVE_LEVEL, st);
      s = HODLR_ERR_ARG;
      if (kSolveStepTma) {
        bool used_partial = false;
        s = solve_step_f64(r, n, nc, 2 * nc, X, ldx, Y + q.c[lv + 1] * n, Vn, n, w2, (int64_t)2 * r * nrhs, nrhs, w,
                           (int64_t)2 * r * nrhs, part, solve_part_bytes(d, nrhs), device_sm_count(), &used_partial, st);
        if (s == HODLR_OK && used_partial)
          s = level_reduce_f64(part, w, r, nrhs, (int)(2 * nc / 512), (int)(n / (2 * nc)), (int64_t)2 * r * nrhs, st);
      }
      if (s == HODLR_ERR_ARG)
        s = solve_level_f64(r, n, nc, 2 * nc, X, ldx, Y + q.c[lv + 1] * n, Vn, n, w2, (int64_t)2 * r * nrhs, nrhs, w,
                            (int64_t)2 * r * nrhs, part, solve_part_bytes(d, nrhs), st);
      if (s == HODLR_ERR_ARG)
        s = level_update_f64(r, n, nc, 2 * nc, X, ldx, Y + q.c[lv + 1] * n, Vn, n, w2, (int64_t)2 * r * nrhs, nrhs, w,
                             (int64_t)2 * r * nrhs, part, solve_part_bytes(d, nrhs), st, false);
    }
    if (s == HODLR_OK) {
      w_ready = lv > 0 && Vn != nullptr;
      continue;
    }
    if (s != HODLR_ERR_ARG) return s;
    w_ready = false;
    Phase ph(HODLR_PHASE_GEMM, st);
    TRY(gemm_f64(0, (int)nc, nrhs, r, -1.0, Y + q.c[lv + 1] * n, n, 2 * nc, nc, w2, 2 * r, (int64_t)2 * r * nrhs, r,
                 1.0, X, ldx, 2 * nc, nc, nch, 2, split, kSplitBytes, st));
  }
  if (!w_ready && lv_stop > 0) {
    const int lv = lv_stop - 1;
    const int64_t nc = N >> (lv + 1);
    const int r = q.r[lv + 1];
    if (r > 0) {
      Phase ph(HODLR_PHASE_GEMM, st);
      TRY(gemm_f64(1, r, nrhs, (int)std::min<int64_t>(nc, n), 1.0, V + q.c[lv + 1] * n, n, 2 * nc, nc, X, ldx,
                   2 * nc, nc, 0.0, w, 2 * r, (int64_t)2 * r * nrhs, r, std::max<int>((int)(n / nc), 1), 2, split,
                   kSplitBytes, st));
    }
  }
  return HODLR_OK;
}

extern "C" hodlr_status hodlr_solve(const hodlr_desc* d, const hodlr_factors* f, void* Xv, int64_t ldx, int nrhs,
                                    void* work, size_t work_bytes, void* stream) {
  if (!desc_ok(d) || !f || nrhs < 0 || ldx < d->n) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64 && d->dtype != HODLR_F32) return HODLR_ERR_ARG;
  if (nrhs == 0) return HODLR_OK;
  if (work_bytes < hodlr_solve_workspace(d, nrhs) || !work) return HODLR_ERR_ARG;
  if (d->dtype == HODLR_F32)
    return solve_generic<float>(d, f, (float*)Xv, ldx, nrhs, static_cast<char*>(work), S(stream));
  return solve_local(d, f, d->n, 0, 0, (double*)Xv, ldx, nrhs, static_cast<char*>(work), S(stream));
}

extern "C" hodlr_status hodlr_solve_local(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0,
                                          int lv_stop, void* Xv, int64_t ldx, int nrhs, double* w_out, void* work,
                                          size_t work_bytes, void* stream) {
  if (!desc_ok(d) || !uniform_desc(d) || !f || !local_ok(d, n_loc, row0) || nrhs < 0 || ldx < n_loc) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64 || lv_stop < 0 || lv_stop > d->L || (d->n >> lv_stop) > n_loc) return HODLR_ERR_ARG;
  if (nrhs == 0) return HODLR_OK;
  if (work_bytes < hodlr_solve_workspace(d, nrhs) || !work) return HODLR_ERR_ARG;
  cudaStream_t st = S(stream);
  TRY(solve_local(d, f, n_loc, row0, lv_stop, (double*)Xv, ldx, nrhs, static_cast<char*>(work), st));
  if (w_out && lv_stop > 0 && d->r > 0) {
    const double* w = reinterpret_cast<const double*>(static_cast<char*>(work) + kSplitBytes);
    const int r = d->r;
    if (cudaMemcpy2DAsync(w_out, sizeof(double) * r, w, sizeof(double) * 2 * r, sizeof(double) * r, nrhs,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return hodlr_set_cuda_error(cudaGetLastError());
  }
  return HODLR_OK;
}

// Finish solve level lv < p for the caller's rows: w_all = complete w of all
// 2^(lv+1) children (paired per parent, 2r x nrhs, ld 2r, parent stride
// 2r*nrhs); applies K_p^-1 for the caller's parent, updates its rows of X and
// writes its partial w of its level-lv node (r x nrhs, ld r) to w_out (lv > 0).
extern "C" hodlr_status hodlr_solve_top(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0,
                                        int lv, const double* w_all, double* w_out, void* Xv, int64_t ldx, int nrhs,
                                        void* work, size_t work_bytes, void* stream) {
  if (!desc_ok(d) || !uniform_desc(d) || !f || !local_ok(d, n_loc, row0) || !w_all || nrhs <= 0 || ldx < n_loc) return HODLR_ERR_ARG;
  if (d->dtype != HODLR_F64 || lv < 0 || lv >= d->L || (d->n >> (lv + 1)) < n_loc) return HODLR_ERR_ARG;
  if (work_bytes < hodlr_solve_workspace(d, nrhs) || !work) return HODLR_ERR_ARG;
  cudaStream_t st = S(stream);
  char* wp = static_cast<char*>(work);
  const int64_t N = d->n, n = n_loc;
  const int r = d->r, L = d->L;
  const size_t wsz = align_up(sizeof(double) * (size_t)std::max<int64_t>((int64_t)1 << L, 2) * r * nrhs);
  double* w = reinterpret_cast<double*>(wp + kSplitBytes);
  double* w2 = reinterpret_cast<double*>(wp + kSplitBytes + wsz);
  double* part = reinterpret_cast<double*>(wp + kSplitBytes + 2 * wsz);
  const int64_t nc = N >> (lv + 1);
  const int64_t p = row0 / (2 * nc), half = (row0 / nc) & 1;
  const int64_t kblk = ((int64_t)1 << lv) - 1 + p;
  {
    Phase ph(HODLR_PHASE_SOLVE_K, st);
    TRY(lu_apply(2 * r, nrhs, 1, (const double*)f->K + kblk * 4 * r * r, (const double*)f->Kinv + kblk * inv_block_elems(2 * r),
                 f->kperm + kblk * 2 * r, w_all + p * 2 * r * nrhs, 2 * r, 0, w2, 2 * r, 0, st, kSolveNarrowCols));
  }
  const double* Y = (const double*)f->Y;
  const double* V = (const double*)f->V;
  double* X = (double*)Xv;
  Phase ph(HODLR_PHASE_SOLVE_LEVEL, st);
  hodlr_status s = solve_level_f64(r, n, nc, n, X, ldx, Y + (int64_t)lv * r * n,
                                   lv > 0 ? V + (int64_t)(lv - 1) * r * n : nullptr, n, w2 + half * r, 0, nrhs, w, 0,
                                   part, solve_part_bytes(d, nrhs), st);
  if (s == HODLR_ERR_ARG)
    s = level_update_f64(r, n, nc, n, X, ldx, Y + (int64_t)lv * r * n,
                         lv > 0 ? V + (int64_t)(lv - 1) * r * n : nullptr, n, w2 + half * r, 0, nrhs, w, 0, part,
                         solve_part_bytes(d, nrhs), st, false);
  if (s == HODLR_OK) {
    if (lv > 0 && w_out &&
        cudaMemcpy2DAsync(w_out, sizeof(double) * r, w, sizeof(double) * 2 * r, sizeof(double) * r, nrhs,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return hodlr_set_cuda_error(cudaGetLastError());
    return HODLR_OK;
  }
  if (s != HODLR_ERR_ARG) return s;
  TRY(gemm_f64(0, (int)n, nrhs, r, -1.0, Y + (int64_t)lv * r * n, n, 0, 0, w2 + half * r, 2 * r, 0, 0, 1.0, X, ldx, 0,
               0, 1, 1, wp, kSplitBytes, st));
  if (lv > 0 && w_out)
    TRY(gemm_f64(1, r, nrhs, (int)n, 1.0, V + (int64_t)(lv - 1) * r * n, n, 0, 0, X, ldx, 0, 0, 0.0, w_out, r, 0, 0, 1,
                 1, wp, kSplitBytes, st));
  return HODLR_OK;
}
