// Dependent-chain latency of mma.sync.m8n8k4.f64 (DMMA) on sm_100a, and the issue
// interval with k independent chains in one warp (dev tool).
#include <cstdio>
template <int K>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double c[K][2];
  for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
#pragma unroll
    for (int i = 0; i < K; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 64);
#define RUN(K) k<K><<<1, 32>>>(out, cyc, 1e-3, 1.0); k<K><<<1, 32>>>(out, cyc, 1e-3, 1.0); cudaDeviceSynchronize(); \
  printf("chains=%d cycles/iter=%lld (per DMMA %.1f)\n", K, cyc[0], cyc[0] / (double)K);
  RUN(1) RUN(2) RUN(4) RUN(8) RUN(16)
  return 0;
}
