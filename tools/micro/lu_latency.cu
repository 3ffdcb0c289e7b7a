// Single-block latency microbenchmark of the batched LU kernel (dev tool).
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../../paper_2208_06290_b200/csrc/lu_cyclic.cu"
hodlr_status hodlr_set_cuda_error(cudaError_t) { return HODLR_ERR_CUDA; }
void hodlr_count_launch() {}
int main() {
  const int S = 64;
  for (int batch : {1, 148, 740, 16384}) {
    std::vector<double> h((size_t)batch * S * S);
    srand(1);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    for (int b = 0; b < batch; ++b) for (int i = 0; i < S; ++i) h[(size_t)b * S * S + i * (S + 1)] += 4;
    double *A, *Ti; int *sw, *pm, *inf;
    cudaMalloc(&A, h.size() * 8); cudaMalloc(&Ti, h.size() * 8);
    cudaMalloc(&sw, batch * S * 4); cudaMalloc(&pm, batch * S * 4); cudaMalloc(&inf, batch * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int withinv = 0; withinv < 2; ++withinv) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        if (getenv("CYC")) hodlr::run_cyclic<double, 64>(batch, 0, A, S, S * S, A, S, S * S, sw, pm, inf, withinv ? Ti : nullptr, S, S * S, 0); else hodlr::launch_getrf_cyclic<double>(S, batch, 0, A, S, S * S, A, S, S * S, sw, pm, inf, withinv ? Ti : nullptr, S, S * S, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("batch %6d tinv %d: %.1f us\n", batch, withinv, best * 1000);
    }
    cudaFree(A); cudaFree(Ti); cudaFree(sw); cudaFree(pm); cudaFree(inf);
  }
  return 0;
}
