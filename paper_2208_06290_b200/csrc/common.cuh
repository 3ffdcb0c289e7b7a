// Shared device helpers for the HODLR B200 kernels (sm_100a).
#pragma once
#include <mutex>
#include <unordered_map>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "hodlr_b200.h"

#define HODLR_CHECK_LAUNCH()                                   \
  do {                                                         \
    hodlr_count_launch();                                      \
    cudaError_t e_ = cudaGetLastError();                       \
    if (e_ != cudaSuccess) return hodlr_set_cuda_error(e_);    \
  } while (0)

namespace hodlr {

// ---- async global->shared copies (LDGSTS); src_bytes < size zero-fills ----
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// 16B copy with an L2 cache-eviction policy (createpolicy handle)
__device__ __forceinline__ void cp_async_16_pol(void* smem, const void* gmem, int src_bytes, uint64_t pol) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes), "l"(pol));
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- FP64 tensor core: D(8x8) += A(8x4, row) * B(4x8, col) -> SASS DMMA.8x8x4 ----
// lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- IEEE ops without contraction (bit-exact replay of numpy ufunc order) ----
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

template <typename T>
struct Eps;
template <>
struct Eps<double> {
  static constexpr double v = 2.220446049250313e-16;
};
template <>
struct Eps<float> {
  static constexpr float v = 1.1920929e-07f;
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Scalars of the factorization-internal solve aids per s x s block (Dinv /
// Kinv): the 8x8 diagonal-block inverses (8 s) for s in {32, 64, 128}, the
// packed full inverses (s^2) for s = 16, nothing otherwise (row substitution).
__host__ __device__ inline int64_t inv_block_elems(int s) {
  return (s == 32 || s == 64 || s == 128) ? (int64_t)8 * s : s == 16 ? (int64_t)s * s : 0;
}

}  // namespace hodlr

namespace hodlr {
// cudaFuncSetAttribute once per (kernel, size): repeated calls would also land
// inside CUDA-graph captures of later factorize / solve calls
template <typename K>
inline void smem_attr(K kern, int bytes, cudaFuncAttribute what = cudaFuncAttributeMaxDynamicSharedMemorySize) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lk(mu);
  int& v = done[reinterpret_cast<const void*>(kern)];
  if (v < bytes + 1) {
    cudaFuncSetAttribute(kern, what, bytes);
    v = bytes + 1;
  }
}
}  // namespace hodlr

// records the CUDA error string for hodlr_last_error(); defined in hodlr.cu
hodlr_status hodlr_set_cuda_error(cudaError_t e);
// counts kernel launches issued by this library (hodlr_launch_count)
void hodlr_count_launch();
