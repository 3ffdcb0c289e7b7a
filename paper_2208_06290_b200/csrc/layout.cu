// Right-hand-side layout change for the solve's public API: the caller's
// (N x nrhs) row-major block (torch / numpy default) <-> the column-major
// N x nrhs block the solve kernels stream (ld N).  Tiled through shared
// memory: each CTA reads a 64-row x 32-column tile with consecutive threads on
// consecutive addresses of the source and writes it out 64 rows at a time per
// column, so both sides are coalesced (torch's strided copy for this shape
// runs at ~0.8 TB/s, tools/transpose_probe.py).
#include "common.cuh"

namespace hodlr {

constexpr int kTrRows = 64, kTrCols = 32, kTrThreads = 256;

// X[c * ldx + i] = B[i * ldb + c], i < n, c < k
__global__ void __launch_bounds__(kTrThreads) transpose_f64_kernel(const double* __restrict__ B, int64_t n, int k,
                                                                   int64_t ldb, double* __restrict__ X, int64_t ldx) {
  __shared__ double tile[kTrCols][kTrRows + 1];
  const int64_t i0 = (int64_t)blockIdx.x * kTrRows;
  const int c0 = blockIdx.y * kTrCols;
  const int kc = min(kTrCols, k - c0);
  const int rows = n - i0 < kTrRows ? (int)(n - i0) : kTrRows;
  for (int idx = threadIdx.x; idx < rows * kc; idx += kTrThreads) {
    const int r = idx / kc, c = idx - r * kc;
    tile[c][r] = B[(i0 + r) * ldb + c0 + c];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kc * kTrRows; idx += kTrThreads) {
    const int c = idx / kTrRows, r = idx - c * kTrRows;
    if (r < rows) X[(int64_t)(c0 + c) * ldx + i0 + r] = tile[c][r];
  }
}

}  // namespace hodlr

using namespace hodlr;

extern "C" hodlr_status hodlr_transpose_f64(const void* B, int64_t n, int64_t k, int64_t ldb, void* X, int64_t ldx,
                                            void* stream) {
  if (n < 0 || k < 0 || (n > 0 && k > 0 && (!B || !X || ldb < k || ldx < n))) return HODLR_ERR_ARG;
  if (n == 0 || k == 0) return HODLR_OK;
  if (k > 65535LL * kTrCols) return HODLR_ERR_ARG;
  const dim3 grid((unsigned)ceil_div(n, kTrRows), (unsigned)ceil_div(k, kTrCols));
  transpose_f64_kernel<<<grid, kTrThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const double*>(B), n, (int)k, ldb, static_cast<double*>(X), ldx);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}
