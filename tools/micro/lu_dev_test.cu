// lu64_rows_device (epilogue LU, first 64 threads of a 256-thread CTA) vs getrf_reg_kernel: bit-exact (dev test).
#include <cstdio>
#include <cstring>
#include <vector>
#include <cstdlib>
#include "../../paper_2208_06290_b200/csrc/lu_cyclic.cu"
hodlr_status hodlr_set_cuda_error(cudaError_t) { return HODLR_ERR_CUDA; }
void hodlr_count_launch() {}
__global__ void __launch_bounds__(256) dev_kernel(int mode, const double* src, int64_t strides, double* out,
                                                  int32_t* sw, int32_t* pm, int32_t* inf, double* dbi) {
  __shared__ __align__(16) double rows[64 * 68];
  const int b = blockIdx.x;
  if (threadIdx.x < 64)
    hodlr::lu64_rows_device(mode, src + (int64_t)b * strides, 64, out + (int64_t)b * 4096, sw + b * 64, pm + b * 64,
                            inf + b, dbi + (int64_t)b * 4096, rows);
}
int main() {
  const int S = 64;
  for (int batch : {1, 300, 4096}) {
    std::vector<double> h((size_t)batch * S * S);
    srand(7 + batch);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    for (int b = 0; b < batch; b += 5) h[(size_t)b * S * S + 3] = 0.0;
    size_t n = h.size();
    double *A, *O1, *O2, *D1, *D2; int *s1, *p1, *i1, *s2, *p2, *i2;
    cudaMalloc(&A, n * 8); cudaMalloc(&O1, n * 8); cudaMalloc(&O2, n * 8); cudaMalloc(&D1, n * 8); cudaMalloc(&D2, n * 8);
    cudaMalloc(&s1, batch * S * 4); cudaMalloc(&p1, batch * S * 4); cudaMalloc(&i1, batch * 4);
    cudaMalloc(&s2, batch * S * 4); cudaMalloc(&p2, batch * S * 4); cudaMalloc(&i2, batch * 4);
    cudaMemset(D1, 0, n * 8); cudaMemset(D2, 0, n * 8);
    cudaMemcpy(A, h.data(), n * 8, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
      const int64_t strides = S * S;  // mode 1 reads a 64 x 64 panel [T_a | T_b] (ld 64) from the same buffer
      hodlr::getrf_reg_kernel<64><<<batch, 64>>>(mode, A, S, strides, O1, S, S * S, s1, p1, i1, D1, S * S);
      dev_kernel<<<batch, 256>>>(mode, A, strides, O2, s2, p2, i2, D2);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> a(n), bb(n), da(n), db(n);
      std::vector<int> x1(batch * S), x2(batch * S), y1(batch * S), y2(batch * S), z1(batch), z2(batch);
      cudaMemcpy(a.data(), O1, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(bb.data(), O2, n * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(da.data(), D1, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(db.data(), D2, n * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(x1.data(), s1, batch * S * 4, cudaMemcpyDeviceToHost); cudaMemcpy(x2.data(), s2, batch * S * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(y1.data(), p1, batch * S * 4, cudaMemcpyDeviceToHost); cudaMemcpy(y2.data(), p2, batch * S * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(z1.data(), i1, batch * 4, cudaMemcpyDeviceToHost); cudaMemcpy(z2.data(), i2, batch * 4, cudaMemcpyDeviceToHost);
      bool dbi_eq = true;
      for (int b = 0; b < batch; ++b) if (memcmp(&da[(size_t)b * S * S], &db[(size_t)b * S * S], 8 * S * 8)) dbi_eq = false;
      printf("batch %d mode %d (%s): LU %s piv %s info %s dbi %s\n", batch, mode, cudaGetErrorString(e),
             memcmp(a.data(), bb.data(), n * 8) ? "DIFF" : "bit-exact", (x1 == x2 && y1 == y2) ? "equal" : "DIFF",
             z1 == z2 ? "equal" : "DIFF", dbi_eq ? "equal" : "DIFF");
    }
  }
}
