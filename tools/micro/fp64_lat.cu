// Dependent-chain latencies on sm_100a (dev tool): DMUL, DADD, DFMA, __ddiv_rn, REDUX, shfl, bar.sync.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, double y) {
  double x = x0 + threadIdx.x;
  long long t0, t1;
  const int N = 256;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, y);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, y);
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-300);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __ddiv_rn(x, y) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / N;
  unsigned u = (unsigned)x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) u = __reduce_max_sync(0xffffffffu, u + threadIdx.x);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / N;
  __shared__ double s[64];
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { s[threadIdx.x] = x; __syncthreads(); x = s[(threadIdx.x + 1) & 63] * y; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __dsub_rn(x, __dmul_rn(y, x));
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / N;
  out[threadIdx.x] = x + u;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 128);
  k<<<1, 64>>>(o, c, 1.0, 1.0000001); cudaDeviceSynchronize();
  k<<<1, 64>>>(o, c, 1.0, 1.0000001); cudaDeviceSynchronize();
  const char* nm[8] = {"DMUL", "DADD", "DFMA", "ddiv_rn+1", "REDUX", "SHFL", "STS+BAR+LDS+DMUL (2 warps)", "DMUL->DSUB"};
  for (int i = 0; i < 8; ++i) printf("%-28s %lld cyc\n", nm[i], c[i]);
}
