// Batched FP32 GEMM (SIMT FMA; fp32 has no DMMA path and the fp32 HODLR
// configurations are HBM-bound at their small ranks):
//
//   C_b <- alpha * op(A_b) B_b + beta * C_b        (backend.py:282-303, :320-364)
//
// Same operand addressing, paired-batch layout and fixed-order split-K contract
// as gemm.cu.  64 x 64 tiles, 256 threads, each thread a 4 x 4 register tile;
// A / B tiles staged k-major in shared memory.  Accumulation in fp32 (numpy's
// float32 matmul semantics), product combined with C as backend.py does.
#include "common.cuh"

namespace hodlr {

struct GemmArgsF {
  int M, N, K;
  float alpha, beta;
  const float* A;
  int64_t lda, sA_hi, sA_lo;
  const float* B;
  int64_t ldb, sB_hi, sB_lo;
  float* C;
  int64_t ldc, sC_hi, sC_lo;
  int batch, bdiv;
  int ksplit, kchunk;
  float* part;
  int tiles_m, tiles_n;
};

__device__ __forceinline__ int64_t boff_f(int b, int bdiv, int64_t hi, int64_t lo) {
  return (int64_t)(b / bdiv) * hi + (int64_t)(b % bdiv) * lo;
}

__device__ __forceinline__ float combine_f(float prod, const float* cptr, float alpha, float beta) {
  if (beta == 0.f) return (alpha == 1.f) ? prod : __fmul_rn(prod, alpha);
  float c = *cptr;
  if (beta != 1.f) c = __fmul_rn(c, beta);
  if (alpha == 1.f) return __fadd_rn(c, prod);
  if (alpha == -1.f) return __fsub_rn(c, prod);
  return __fadd_rn(c, __fmul_rn(prod, alpha));
}

// BM x BN x BK tile, 16 x 16 threads, thread (ty, tx) owns rows ty + 16 i
// (i < BM/16) and columns tx + 16 j (j < BN/16)
template <bool TA, int FBM, int FBN, int FBK>
__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmArgsF g) {
  constexpr int TM = FBM / 16, TN = FBN / 16;
  __shared__ float As[FBK][FBM + 4];
  __shared__ float Bs[FBK][FBN + 4];
  int64_t lin = blockIdx.x;
  const int tn = (int)(lin % g.tiles_n);
  lin /= g.tiles_n;
  const int tm = (int)(lin % g.tiles_m);
  lin /= g.tiles_m;
  const int b = (int)(lin % g.batch);
  const int split = (int)(lin / g.batch);
  const int m0 = tm * FBM, n0 = tn * FBN;
  const int kbeg = split * g.kchunk, kend = min(g.K, kbeg + g.kchunk);
  const float* Ab = g.A + boff_f(b, g.bdiv, g.sA_hi, g.sA_lo);
  const float* Bb = g.B + boff_f(b, g.bdiv, g.sB_hi, g.sB_lo);
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  for (int k0 = kbeg; k0 < kend; k0 += FBK) {
    for (int idx = t; idx < FBM * FBK; idx += 256) {
      int m, k;
      if (TA) {  // op(A)[m][k] = A[k + m lda]
        k = idx % FBK;
        m = idx / FBK;
      } else {
        m = idx % FBM;
        k = idx / FBM;
      }
      const int gm = m0 + m, gk = k0 + k;
      float v = 0.f;
      if (gm < g.M && gk < kend) v = TA ? Ab[gk + (int64_t)gm * g.lda] : Ab[gm + (int64_t)gk * g.lda];
      As[k][m] = v;
    }
    for (int idx = t; idx < FBN * FBK; idx += 256) {
      const int k = idx % FBK, n = idx / FBK;
      const int gn = n0 + n, gk = k0 + k;
      Bs[k][n] = (gn < g.N && gk < kend) ? Bb[gk + (int64_t)gn * g.ldb] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < FBK; ++k) {
      float a[TM], bb[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bb[j] = Bs[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= g.N) continue;
      if (g.ksplit > 1) {
        g.part[((int64_t)split * g.batch + b) * g.M * g.N + gm + (int64_t)gn * g.M] = acc[i][j];
      } else {
        float* cp = g.C + boff_f(b, g.bdiv, g.sC_hi, g.sC_lo) + gm + (int64_t)gn * g.ldc;
        *cp = combine_f(acc[i][j], cp, g.alpha, g.beta);
      }
    }
  }
}

__global__ void splitk_reduce_f32_kernel(GemmArgsF g) {
  const int64_t MN = (int64_t)g.M * g.N;
  const int64_t total = MN * g.batch;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / MN);
    const int64_t mn = e % MN;
    const int gm = (int)(mn % g.M), gn = (int)(mn / g.M);
    float s = 0.f;
    for (int k = 0; k < g.ksplit; ++k) s += g.part[((int64_t)k * g.batch + b) * MN + mn];
    float* cp = g.C + boff_f(b, g.bdiv, g.sC_hi, g.sC_lo) + gm + (int64_t)gn * g.ldc;
    *cp = combine_f(s, cp, g.alpha, g.beta);
  }
}

hodlr_status gemm_f32(int transA, int M, int N, int K, float alpha, const float* A, int64_t lda, int64_t sA_hi,
                      int64_t sA_lo, const float* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, float beta, float* C,
                      int64_t ldc, int64_t sC_hi, int64_t sC_lo, int batch, int bdiv, void* work, size_t work_bytes,
                      cudaStream_t st) {
  if (M < 0 || N < 0 || K < 0 || batch < 0 || bdiv < 1) return HODLR_ERR_ARG;
  if (M == 0 || N == 0 || batch == 0) return HODLR_OK;
  GemmArgsF g{};
  g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.beta = beta;
  g.A = A; g.lda = lda; g.sA_hi = sA_hi; g.sA_lo = sA_lo;
  g.B = B; g.ldb = ldb; g.sB_hi = sB_hi; g.sB_lo = sB_lo;
  g.C = C; g.ldc = ldc; g.sC_hi = sC_hi; g.sC_lo = sC_lo;
  g.batch = batch; g.bdiv = bdiv;
  g.ksplit = 1;
  // tile shapes: [W|T] / w reductions (M = rank <= 16), the solve's narrow
  // x updates (N = nrhs <= 16), and the general 64 x 64 tile
  const bool skinny = M <= 16;
  const int cfg = skinny ? (N <= 16 ? 1 : 0) : (N <= 16 && !transA ? 2 : 3);
  const int BMc = cfg <= 1 ? 16 : cfg == 2 ? 256 : 64;
  const int BNc = cfg == 0 ? 128 : cfg == 3 ? 64 : 16;
  const int FBK = cfg == 1 ? 128 : 16;
  g.kchunk = (int)std::max<int64_t>(FBK, ceil_div(K, FBK) * FBK);
  g.tiles_m = (int)ceil_div(M, BMc);
  g.tiles_n = (int)ceil_div(N, BNc);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // split-K depends on (M, K, batch) only (multi-RHS columns stay bit-identical)
  const int64_t tiles = (int64_t)g.tiles_m * batch;
  if (tiles < 2 * sms && K >= 1024 && work) {
    int64_t ks = std::min<int64_t>(ceil_div(4 * (int64_t)sms, tiles), ceil_div(K, 256));
    ks = std::min<int64_t>(ks, 128);
    while (ks > 1 && (size_t)ks * batch * M * N * sizeof(float) > work_bytes) --ks;
    if (ks > 1) {
      // chunk boundaries on a 128 grid whatever the tile's BK: the split (and so
      // every output's summation order) never depends on N
      g.kchunk = (int)(ceil_div(ceil_div(K, ks), 128) * 128);
      g.ksplit = (int)ceil_div(K, g.kchunk);
      g.part = static_cast<float*>(work);
    }
  }
  const int64_t grid = (int64_t)g.tiles_m * g.tiles_n * g.batch * g.ksplit;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  switch (cfg) {
    case 0:
      if (transA) gemm_f32_kernel<true, 16, 128, 16><<<(unsigned)grid, 256, 0, st>>>(g);
      else gemm_f32_kernel<false, 16, 128, 16><<<(unsigned)grid, 256, 0, st>>>(g);
      break;
    case 1:
      if (transA) gemm_f32_kernel<true, 16, 16, 128><<<(unsigned)grid, 256, 0, st>>>(g);
      else gemm_f32_kernel<false, 16, 16, 128><<<(unsigned)grid, 256, 0, st>>>(g);
      break;
    case 2: gemm_f32_kernel<false, 256, 16, 16><<<(unsigned)grid, 256, 0, st>>>(g); break;
    default:
      if (transA) gemm_f32_kernel<true, 64, 64, 16><<<(unsigned)grid, 256, 0, st>>>(g);
      else gemm_f32_kernel<false, 64, 64, 16><<<(unsigned)grid, 256, 0, st>>>(g);
  }
  HODLR_CHECK_LAUNCH();
  if (g.ksplit > 1) {
    const int64_t total = (int64_t)M * N * batch;
    const int64_t blocks = std::min<int64_t>(ceil_div(total, 256), 8 * (int64_t)sms);
    splitk_reduce_f32_kernel<<<(unsigned)blocks, 256, 0, st>>>(g);
    HODLR_CHECK_LAUNCH();
  }
  return HODLR_OK;
}

}  // namespace hodlr
