// Batched FP64 GEMM on the sm_100a FP64 tensor pipe (mma.sync m8n8k4 -> DMMA.8x8x4).
//
//   C_b <- alpha * op(A_b) B_b + beta * C_b        (backend.py:282-303, :320-364)
//
// Column-major operands; operand b at X + (b / bdiv) * s_hi + (b % bdiv) * s_lo.
// Tiles are staged through a 3-stage cp.async (LDGSTS) shared-memory pipeline;
// each warp owns a 32 x 32 (or 32 x 16) accumulator tile = 4 x 4 DMMA tiles.
// Split-K writes raw partial products to a workspace that a second kernel sums
// in a fixed order, so results are deterministic run to run.
#include "common.cuh"

namespace hodlr {

struct GemmArgs {
  int M, N, K;
  double alpha, beta;
  const double* A;
  int64_t lda, sA_hi, sA_lo;
  const double* B;
  int64_t ldb, sB_hi, sB_lo;
  double* C;
  int64_t ldc, sC_hi, sC_lo;
  int batch, bdiv;
  int ksplit;      // number of K chunks (1 = no split)
  int kchunk;      // K elements per chunk (multiple of BK)
  double* part;    // split-K partials: [split][batch][M x N] col-major ld M
  int tiles_m, tiles_n;
};

constexpr int BK = 16;
constexpr int STAGES = 3;
constexpr int KPAD = BK + 4;  // k-contiguous rows: conflict-free fragment loads

__device__ __forceinline__ int64_t boff(int b, int bdiv, int64_t hi, int64_t lo) {
  return (int64_t)(b / bdiv) * hi + (int64_t)(b % bdiv) * lo;
}

// combine the rounded product with C exactly as backend.py:_gemm_into does
__device__ __forceinline__ double combine(double prod, double* cptr, double alpha, double beta) {
  if (beta == 0.0) return (alpha == 1.0) ? prod : __dmul_rn(prod, alpha);
  double c = *cptr;
  if (beta != 1.0) c = __dmul_rn(c, beta);
  if (alpha == 1.0) return __dadd_rn(c, prod);
  if (alpha == -1.0) return __dsub_rn(c, prod);
  return __dadd_rn(c, __dmul_rn(prod, alpha));
}

template <int BM, int BN, int WM, int WN, bool TA, int VEC>
__global__ void __launch_bounds__(WM* WN * 32) gemm_f64_kernel(GemmArgs g) {
  constexpr int NT = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int MI = WTM / 8, NI = WTN / 8;
  constexpr int A_STAGE = TA ? BM * KPAD : BK * (BM + 4);
  constexpr int B_STAGE = BN * KPAD;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;

  int64_t lin = blockIdx.x;
  const int tn = (int)(lin % g.tiles_n);
  lin /= g.tiles_n;
  const int tm = (int)(lin % g.tiles_m);
  lin /= g.tiles_m;
  const int b = (int)(lin % g.batch);
  const int split = (int)(lin / g.batch);
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * g.kchunk;
  const int kend = min(g.K, kbeg + g.kchunk);

  const double* Ab = g.A + boff(b, g.bdiv, g.sA_hi, g.sA_lo);
  const double* Bb = g.B + boff(b, g.bdiv, g.sB_hi, g.sB_lo);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp / WN, wn = warp % WN;

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
    if (TA) {  // op(A)[m][k] = A[k + m*lda]: k-contiguous
      constexpr int VPR = BK / VEC;
      for (int idx = t; idx < BM * VPR; idx += NT) {
        const int m = idx / VPR, kv = (idx % VPR) * VEC;
        const int gm = m0 + m, gk = k0 + kv;
        int bytes = (gm < g.M) ? 8 * max(0, min(VEC, kend - gk)) : 0;
        const double* src = bytes ? Ab + (int64_t)gm * g.lda + gk : g.A;
        if (VEC == 2)
          cp_async_16(as + m * KPAD + kv, src, bytes);
        else
          cp_async_8(as + m * KPAD + kv, src, bytes);
      }
    } else {  // op(A)[m][k] = A[m + k*lda]: m-contiguous
      constexpr int VPC = BM / VEC;
      for (int idx = t; idx < BK * VPC; idx += NT) {
        const int k = idx / VPC, mv = (idx % VPC) * VEC;
        const int gm = m0 + mv, gk = k0 + k;
        int bytes = (gk < kend) ? 8 * max(0, min(VEC, g.M - gm)) : 0;
        const double* src = bytes ? Ab + gm + (int64_t)gk * g.lda : g.A;
        if (VEC == 2)
          cp_async_16(as + k * (BM + 4) + mv, src, bytes);
        else
          cp_async_8(as + k * (BM + 4) + mv, src, bytes);
      }
    }
    {  // B[k + n*ldb]: k-contiguous
      constexpr int VPR = BK / VEC;
      for (int idx = t; idx < BN * VPR; idx += NT) {
        const int n = idx / VPR, kv = (idx % VPR) * VEC;
        const int gn = n0 + n, gk = k0 + kv;
        int bytes = (gn < g.N) ? 8 * max(0, min(VEC, kend - gk)) : 0;
        const double* src = bytes ? Bb + gk + (int64_t)gn * g.ldb : g.B;
        if (VEC == 2)
          cp_async_16(bs + n * KPAD + kv, src, bytes);
        else
          cp_async_8(bs + n * KPAD + kv, src, bytes);
      }
    }
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (kend > kbeg) ? (int)ceil_div(kend - kbeg, BK) : 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kbeg + s * BK);
    cp_async_commit();
  }
  const int ar = lane >> 2, ac = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, kbeg + nxt * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * A_STAGE;
    const double* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int m = wm * WTM + i * 8 + ar;
        af[i] = TA ? as[m * KPAD + kk + ac] : as[(kk + ac) * (BM + 4) + m];
      }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int n = wn * WTN + j * 8 + ar;
        bf[j] = bs[n * KPAD + kk + ac];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int gm = m0 + wm * WTM + i * 8 + ar;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * WTN + j * 8 + ac * 2 + h;
        if (gn >= g.N) continue;
        if (g.ksplit > 1) {
          g.part[((int64_t)split * g.batch + b) * g.M * g.N + gm + (int64_t)gn * g.M] = acc[i][j][h];
        } else {
          double* cp = g.C + boff(b, g.bdiv, g.sC_hi, g.sC_lo) + gm + (int64_t)gn * g.ldc;
          *cp = combine(acc[i][j][h], cp, g.alpha, g.beta);
        }
      }
    }
  }
}

// fixed-order split-K reduction + epilogue: one thread per C element
__global__ void splitk_reduce_kernel(GemmArgs g) {
  const int64_t MN = (int64_t)g.M * g.N;
  const int64_t total = MN * g.batch;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / MN);
    const int64_t mn = e % MN;
    const int gm = (int)(mn % g.M), gn = (int)(mn / g.M);
    double s = 0.0;
    for (int k = 0; k < g.ksplit; ++k) s += g.part[((int64_t)k * g.batch + b) * MN + mn];
    double* cp = g.C + boff(b, g.bdiv, g.sC_hi, g.sC_lo) + gm + (int64_t)gn * g.ldc;
    *cp = combine(s, cp, g.alpha, g.beta);
  }
}

template <int BM, int BN, int WM, int WN, bool TA, int VEC>
static hodlr_status run_cfg(GemmArgs g, cudaStream_t st) {
  constexpr int A_STAGE = TA ? BM * KPAD : BK * (BM + 4);
  constexpr int B_STAGE = BN * KPAD;
  constexpr size_t smem = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
  auto kern = gemm_f64_kernel<BM, BN, WM, WN, TA, VEC>;
  static bool attr_set = false;
  if (!attr_set) {
    smem_attr(kern, (int)smem);
    attr_set = true;
  }
  g.tiles_m = (int)ceil_div(g.M, BM);
  g.tiles_n = (int)ceil_div(g.N, BN);
  const int64_t grid = (int64_t)g.tiles_m * g.tiles_n * g.batch * g.ksplit;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  kern<<<(unsigned)grid, WM * WN * 32, smem, st>>>(g);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

hodlr_status gemm_f64(int transA, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sA_hi,
                      int64_t sA_lo, const double* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double beta,
                      double* C, int64_t ldc, int64_t sC_hi, int64_t sC_lo, int batch, int bdiv, void* work,
                      size_t work_bytes, cudaStream_t st) {
  if (M < 0 || N < 0 || K < 0 || batch < 0 || bdiv < 1) return HODLR_ERR_ARG;
  if (M == 0 || N == 0 || batch == 0) return HODLR_OK;
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.beta = beta;
  g.A = A; g.lda = lda; g.sA_hi = sA_hi; g.sA_lo = sA_lo;
  g.B = B; g.ldb = ldb; g.sB_hi = sB_hi; g.sB_lo = sB_lo;
  g.C = C; g.ldc = ldc; g.sC_hi = sC_hi; g.sC_lo = sC_lo;
  g.batch = batch; g.bdiv = bdiv;
  g.ksplit = 1;
  g.kchunk = (int)std::max<int64_t>(BK, ceil_div(K, BK) * BK);
  g.part = nullptr;
  const bool small_m = M <= 32;
  const int BMc = small_m ? 32 : 64, BNc = small_m ? 128 : 64;
  // Split-K for few-tile, long-K GEMMs (top tree levels); needs workspace.
  // The split depends on (M, K, batch) only -- never on N -- so a column of a
  // multi-RHS product is bit-identical to the single-column product.
  (void)BNc;
  const int64_t tiles = ceil_div(M, BMc) * (int64_t)batch;
  if (tiles < 2 * num_sms() && K >= 1024 && work) {
    int64_t ks = std::min<int64_t>(ceil_div(4 * (int64_t)num_sms(), tiles), ceil_div(K, 256));
    ks = std::min<int64_t>(ks, 128);
    // only when the caller's workspace is too small does the split shrink (and then depend on N)
    while (ks > 1 && (size_t)ks * batch * M * N * sizeof(double) > work_bytes) --ks;
    if (ks > 1) {
      g.ksplit = (int)ks;
      g.kchunk = (int)(ceil_div(ceil_div(K, ks), BK) * BK);
      g.ksplit = (int)ceil_div(K, g.kchunk);
      g.part = static_cast<double*>(work);
    }
  }
  if (K == 0) {  // product is zero: still apply the epilogue
    g.ksplit = 1;
  }
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool vec2 = aligned(A) && aligned(B) && (lda % 2 == 0) && (ldb % 2 == 0) && (sA_hi % 2 == 0) &&
              (sA_lo % 2 == 0) && (sB_hi % 2 == 0) && (sB_lo % 2 == 0);
  hodlr_status s;
  if (small_m) {
    if (transA)
      s = vec2 ? run_cfg<32, 128, 1, 4, true, 2>(g, st) : run_cfg<32, 128, 1, 4, true, 1>(g, st);
    else
      s = vec2 ? run_cfg<32, 128, 1, 4, false, 2>(g, st) : run_cfg<32, 128, 1, 4, false, 1>(g, st);
  } else {
    if (transA)
      s = vec2 ? run_cfg<64, 64, 2, 2, true, 2>(g, st) : run_cfg<64, 64, 2, 2, true, 1>(g, st);
    else
      s = vec2 ? run_cfg<64, 64, 2, 2, false, 2>(g, st) : run_cfg<64, 64, 2, 2, false, 1>(g, st);
  }
  if (s != HODLR_OK) return s;
  if (g.ksplit > 1) {
    const int64_t total = (int64_t)M * N * batch;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(total, threads), 8 * (int64_t)num_sms());
    splitk_reduce_kernel<<<(unsigned)blocks, threads, 0, st>>>(g);
    HODLR_CHECK_LAUNCH();
  }
  return HODLR_OK;
}

}  // namespace hodlr
