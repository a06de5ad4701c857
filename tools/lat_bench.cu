// Latency microbenchmarks for the inner-solve critical path (one warp, dependent chains).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-20;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // DIV chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0000001 / x;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // SQRT chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // RSQRT-like 1/sqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / sqrt(x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // shuffle + add chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + __shfl_xor_sync(0xffffffffu, x, 1 << (i & 3));
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); x += 1e-30; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  // shared store + barrier + load roundtrip
  __shared__ double sh[1024];
  t0 = clock64();
  for (int i = 0; i < n; ++i) { sh[threadIdx.x] = x; __syncthreads(); x = sh[(threadIdx.x + 32) % blockDim.x] * 0.5 + x * 0.5; __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  // __syncthreads_or
  int f = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { f += __syncthreads_or(x > 1e300); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0) / n;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + f;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"dfma", "dadd", "ddiv", "dsqrt", "1/sqrt", "shfl+dadd", "syncthreads", "sts+bar+lds+bar", "syncthreads_or"};
  for (int threads : {32, 512}) {
    k<<<1, threads>>>(out, cyc, 1.5, 10);
    k<<<1, threads>>>(out, cyc, 1.5, 2000);
    cudaDeviceSynchronize();
    printf("block=%d:", threads);
    for (int i = 0; i < 9; ++i) printf("  %s %lld", names[i], cyc[i]);
    printf("\n");
  }
  return 0;
}
