// Do DMMA (tensor pipe) and DFMA (fp64 pipe) run concurrently on B200?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mix(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double s = 0;
  if (do_mma) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double d[8][2];
    for (int t = 0; t < 8; ++t) d[t][0] = d[t][1] = 0;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
    for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
  } else {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters * 4; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
      }
    }
    s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, bs = 512, iters = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    k_mix<<<blocks, bs>>>(out, 10, mode);
    cudaEventRecord(e0); k_mix<<<blocks, bs>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = blocks * (bs / 32.0);
    double mma_w = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0), fma_w = warps - mma_w;
    double fl = mma_w * 8.0 * iters * 512 + fma_w * 32 * 64.0 * iters * 4 * 2;
    printf("mode %d (%s): %.3f ms  %.2f TFLOP/s\n", mode, mode == 0 ? "dmma" : mode == 1 ? "dfma" : "half/half", ms, fl / ms / 1e9);
  }
  return 0;
}
