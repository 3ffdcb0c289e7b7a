// LU kernels: bit-exact comparison (register-row vs shared-row) + latency/throughput (dev tool).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_2208_06290_b200/csrc/lu_cyclic.cu"
hodlr_status hodlr_set_cuda_error(cudaError_t) { return HODLR_ERR_CUDA; }
void hodlr_count_launch() {}
int main() {
  for (int S : {32, 64}) {
    for (int batch : {1, 148, 4096, 16384}) {
      std::vector<double> h((size_t)batch * S * S);
      srand(1 + batch);
      for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
      for (int b = 0; b < batch; ++b) {
        if (b % 3 == 0) for (int i = 0; i < S; ++i) h[(size_t)b * S * S + i * (S + 1)] += 4;  // mix of regimes
        if (b % 7 == 1) for (int i = 0; i < S; ++i) h[(size_t)b * S * S + i] = 0.0;            // zero column 0
        if (b % 11 == 2) for (int j = 0; j < S; ++j) h[(size_t)b * S * S + 3 + j * S] = h[(size_t)b * S * S + 5 + j * S];  // dup rows
      }
      double *A, *B, *Ti, *Ti2; int *sw, *pm, *inf, *sw2, *pm2, *inf2;
      size_t n = h.size();
      cudaMalloc(&A, n * 8); cudaMalloc(&B, n * 8); cudaMalloc(&Ti, n * 8); cudaMalloc(&Ti2, n * 8);
      cudaMalloc(&sw, batch * S * 4); cudaMalloc(&pm, batch * S * 4); cudaMalloc(&inf, batch * 4);
      cudaMalloc(&sw2, batch * S * 4); cudaMalloc(&pm2, batch * S * 4); cudaMalloc(&inf2, batch * 4);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best[2][2];
      for (int v = 0; v < 2; ++v)
        for (int withinv = 0; withinv < 2; ++withinv) {
          best[v][withinv] = 1e9;
          for (int rep = 0; rep < 4; ++rep) {
            double* X = v ? B : A;
            cudaMemcpy(X, h.data(), n * 8, cudaMemcpyHostToDevice);
            cudaEventRecord(e0);
            if (v == 0) {
              if (S == 64) hodlr::run_sr<double, 64>(batch, 0, X, S, S * S, X, S, S * S, sw, pm, inf, withinv ? Ti : nullptr, S, S * S, 0);
              else hodlr::run_sr<double, 32>(batch, 0, X, S, S * S, X, S, S * S, sw, pm, inf, withinv ? Ti : nullptr, S, S * S, 0);
            } else {
              if (S == 64) hodlr::run_reg<64>(batch, 0, X, S, S * S, X, S, S * S, sw2, pm2, inf2, withinv ? Ti2 : nullptr, S, S * S, 0);
              else hodlr::run_reg<32>(batch, 0, X, S, S * S, X, S, S * S, sw2, pm2, inf2, withinv ? Ti2 : nullptr, S, S * S, 0);
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best[v][withinv]) best[v][withinv] = ms;
          }
        }
      std::vector<double> ha(n), hb(n), ta(n), tb(n);
      std::vector<int> s1(batch * S), s2(batch * S), p1(batch * S), p2(batch * S), i1(batch), i2(batch);
      cudaMemcpy(ha.data(), A, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hb.data(), B, n * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(ta.data(), Ti, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(tb.data(), Ti2, n * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(s1.data(), sw, batch * S * 4, cudaMemcpyDeviceToHost); cudaMemcpy(s2.data(), sw2, batch * S * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(p1.data(), pm, batch * S * 4, cudaMemcpyDeviceToHost); cudaMemcpy(p2.data(), pm2, batch * S * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(i1.data(), inf, batch * 4, cudaMemcpyDeviceToHost); cudaMemcpy(i2.data(), inf2, batch * 4, cudaMemcpyDeviceToHost);
      bool lu_eq = memcmp(ha.data(), hb.data(), n * 8) == 0, t_eq = memcmp(ta.data(), tb.data(), n * 8) == 0;
      bool piv_eq = s1 == s2 && p1 == p2 && i1 == i2;
      int nsing = 0; for (int x : i1) nsing += x;
      printf("S=%d batch %6d  sr %.1f/%.1f us  reg %.1f/%.1f us (LU/LU+inv)  LU %s  piv %s  tinv %s  (singular %d)\n", S, batch,
             best[0][0] * 1e3, best[0][1] * 1e3, best[1][0] * 1e3, best[1][1] * 1e3, lu_eq ? "bit-exact" : "DIFF",
             piv_eq ? "equal" : "DIFF", t_eq ? "equal" : "diff", nsing);
      cudaFree(A); cudaFree(B); cudaFree(Ti); cudaFree(Ti2); cudaFree(sw); cudaFree(pm); cudaFree(inf); cudaFree(sw2); cudaFree(pm2); cudaFree(inf2);
    }
  }
  return 0;
}
