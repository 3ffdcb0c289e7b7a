// Per-stage clock64() breakdown of one sliding-window LU step (single block;
// thread S-1, which stays active until the end on random inputs).  Dev tool.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "lu_win_probe_kernel.cuh"
hodlr_status hodlr_set_cuda_error(cudaError_t) { return HODLR_ERR_CUDA; }
void hodlr_count_launch() {}
int main() {
  for (int S : {64, 32}) {
    std::vector<double> h((size_t)S * S);
    srand(3);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double *A, *O, *D; int *s, *p, *i;
    cudaMalloc(&A, h.size() * 8); cudaMalloc(&O, h.size() * 8); cudaMalloc(&D, 8 * S * 8);
    cudaMalloc(&s, S * 4); cudaMalloc(&p, S * 4); cudaMalloc(&i, 4);
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) {
      long long z[8] = {0};
      cudaMemcpyToSymbol(hodlr::g_ts, z, sizeof(z));
      hodlr::launch_getrf_win<double>(S, 1, 0, A, S, S * S, O, S, S * S, s, p, i, D, 8 * S, 0);
      cudaDeviceSynchronize();
      cudaMemcpyFromSymbol(z, hodlr::g_ts, sizeof(z));
      double n = (double)z[5];
      printf("S=%d steps %.0f: cand+bar %.0f  combine+div+col %.0f  argmax %.0f  update %.0f  book %.0f cycles/step (%s)\n", S, n,
             z[0] / n, z[1] / n, z[2] / n, z[3] / n, z[4] / n, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
