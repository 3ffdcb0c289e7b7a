// A/B of the sliding-window LU (lu_win.cu) against the production LU kernels
// (lu_cyclic.cu): bitwise equality of factors / pivots / flags / diagonal-block
// inverses, and time per launch for batch 1 .. 16384, modes 0 (leaf) and 1 (K
// assembly).  Dev tool:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -Iinclude tools/micro/lu_win_bench.cu -o tools/micro/lu_win_bench
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_2208_06290_b200/csrc/lu_cyclic.cu"
#include "../../paper_2208_06290_b200/csrc/lu_win.cu"
hodlr_status hodlr_set_cuda_error(cudaError_t) { return HODLR_ERR_CUDA; }
void hodlr_count_launch() {}

template <typename T>
static int run(int S, int batch, int mode, bool fp32) {
  const size_t ne = (size_t)batch * S * S;
  std::vector<T> h(ne);
  srand(3 + batch + mode);
  for (auto& x : h) x = (T)((rand() / (double)RAND_MAX - 0.5) * (mode ? 16.0 : 1.0));
  T *A, *O1, *O2;
  double *D1, *D2;
  int *s1, *p1, *i1, *s2, *p2, *i2;
  cudaMalloc(&A, ne * sizeof(T)); cudaMalloc(&O1, ne * sizeof(T)); cudaMalloc(&O2, ne * sizeof(T));
  cudaMalloc(&D1, (size_t)batch * 8 * S * 8); cudaMalloc(&D2, (size_t)batch * 8 * S * 8);
  cudaMalloc(&s1, batch * S * 4); cudaMalloc(&p1, batch * S * 4); cudaMalloc(&i1, batch * 4);
  cudaMalloc(&s2, batch * S * 4); cudaMalloc(&p2, batch * S * 4); cudaMalloc(&i2, batch * 4);
  cudaMemcpy(A, h.data(), ne * sizeof(T), cudaMemcpyHostToDevice);
  cudaMemset(D1, 0, (size_t)batch * 8 * S * 8); cudaMemset(D2, 0, (size_t)batch * 8 * S * 8);
  // mode 1 reads a paired [W|T] panel: T_a rows 0..R-1, T_b rows R..2R-1, ld S, block stride S*S
  auto prod = [&]() -> hodlr_status {
    if constexpr (sizeof(T) == 8)
      return hodlr::launch_getrf_dbi_f64(S, batch, mode, A, S, (int64_t)S * S, O1, S, (int64_t)S * S, s1, p1, i1, D1,
                                         8 * S, 0);
    else
      return hodlr::launch_getrf_cyclic<float>(S, batch, mode, A, S, (int64_t)S * S, O1, S, (int64_t)S * S, s1, p1,
                                               i1, nullptr, 0, 0, 0);
  };
  auto win = [&]() {
    return hodlr::launch_getrf_win<T>(S, batch, mode, A, S, (int64_t)S * S, O2, S, (int64_t)S * S, s2, p2, i2,
                                      sizeof(T) == 8 ? D2 : nullptr, 8 * S, 0);
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best[2] = {1e9f, 1e9f};
  for (int rep = 0; rep < 12; ++rep) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0);
      if (w == 0) prod(); else win();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 1 && ms < best[w]) best[w] = ms;
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<T> a1(ne), a2(ne);
  std::vector<int> x1(batch * S), x2(batch * S), y1(batch * S), y2(batch * S), f1(batch), f2(batch);
  std::vector<double> d1((size_t)batch * 8 * S), d2((size_t)batch * 8 * S);
  cudaMemcpy(a1.data(), O1, ne * sizeof(T), cudaMemcpyDeviceToHost);
  cudaMemcpy(a2.data(), O2, ne * sizeof(T), cudaMemcpyDeviceToHost);
  cudaMemcpy(x1.data(), s1, batch * S * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(x2.data(), s2, batch * S * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(y1.data(), p1, batch * S * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(y2.data(), p2, batch * S * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(f1.data(), i1, batch * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(f2.data(), i2, batch * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(d1.data(), D1, d1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(d2.data(), D2, d2.size() * 8, cudaMemcpyDeviceToHost);
  const bool eq = !memcmp(a1.data(), a2.data(), ne * sizeof(T)) && x1 == x2 && y1 == y2 && f1 == f2 &&
                  (sizeof(T) == 4 || !memcmp(d1.data(), d2.data(), d1.size() * 8));
  size_t nd = 0;
  for (size_t i = 0; i < ne; ++i) nd += memcmp(&a1[i], &a2[i], sizeof(T)) != 0;
  int npiv = 0;
  for (int i = 0; i < batch * S; ++i) npiv += x1[i] != (i % S);
  printf("%s S=%3d batch %6d mode %d: prod %8.1f us  win %8.1f us  (%.2fx)  bitwise %s (diff entries %zu, real pivots %d) %s\n",
         fp32 ? "f32" : "f64", S, batch, mode, best[0] * 1e3, best[1] * 1e3, best[0] / best[1], eq ? "EQUAL" : "DIFF",
         nd, npiv, err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(A); cudaFree(O1); cudaFree(O2); cudaFree(D1); cudaFree(D2);
  cudaFree(s1); cudaFree(p1); cudaFree(i1); cudaFree(s2); cudaFree(p2); cudaFree(i2);
  return eq ? 0 : 1;
}

int main() {
  int bad = 0;
  for (int S : {64, 32})
    for (int mode : {0, 1})
      for (int batch : {1, 4, 32, 128, 512, 1024, 2048, 8192, 16384}) bad += run<double>(S, batch, mode, false);
  for (int batch : {1, 256, 16384}) bad += run<float>(64, batch, 0, true);
  printf("%s\n", bad ? "MISMATCHES" : "all bitwise equal");
  return bad != 0;
}
