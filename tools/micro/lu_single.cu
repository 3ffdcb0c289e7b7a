// Single-block latency of the factorization-internal LU (with diagonal-block inverses), modes 0/1 (dev tool).
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../../paper_2208_06290_b200/csrc/lu_cyclic.cu"
hodlr_status hodlr_set_cuda_error(cudaError_t) { return HODLR_ERR_CUDA; }
void hodlr_count_launch() {}
int main() {
  const int S = 64;
  for (int batch : {1, 8, 64, 8192}) {
    std::vector<double> h((size_t)batch * S * S);
    srand(3);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double *A, *O, *Di; int *sw, *pm, *inf;
    cudaMalloc(&A, h.size() * 8); cudaMalloc(&O, h.size() * 8); cudaMalloc(&Di, h.size() * 8);
    cudaMalloc(&sw, batch * S * 4); cudaMalloc(&pm, batch * S * 4); cudaMalloc(&inf, batch * 4);
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        // mode 1: K assembly from a 32 x 32 x 2 [T_a | T_b] panel (lds 64)
        hodlr::launch_getrf_dbi_f64(S, batch, mode, A, S, S * S, O, S, S * S, sw, pm, inf, Di, S * S, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("batch %5d mode %d: %.1f us\n", batch, mode, best * 1e3);
    }
  }
}
