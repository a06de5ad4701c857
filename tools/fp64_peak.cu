// FP64 peak microbenchmarks for B200 (sm_100a): DFMA pipe vs DMMA (mma.sync f64).
// Used once to fix the roofline denominator; not on the solve path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dmma884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { d[t][0] = 0; d[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma1684(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][4];
#pragma unroll
  for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) d[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma16816(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
#pragma unroll
  for (int q = 0; q < 4; ++q) b[q] = 1.0 - threadIdx.x * 1e-4 - q * 1e-6;
  double d[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) d[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int bs : {256, 512, 1024}) {
    int blocks = sms * (2048 / bs) ;
    int iters = 4000;
    k_dfma<<<blocks, bs>>>(out, 10);
    cudaEventRecord(e0); k_dfma<<<blocks, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * iters * (double)blocks * bs;
    printf("DFMA   bs=%4d : %.2f TFLOP/s\n", bs, fl / ms / 1e9);
  }
  for (int bs : {128, 256, 512}) {
    int blocks = sms * (2048 / bs);
    int iters = 2000;
    k_dmma884<<<blocks, bs>>>(out, 10);
    cudaEventRecord(e0); k_dmma884<<<blocks, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * iters * (double)blocks * (bs / 32);
    printf("DMMA884  bs=%4d : %.2f TFLOP/s\n", bs, fl / ms / 1e9);
    k_dmma1684<<<blocks, bs>>>(out, 10);
    cudaEventRecord(e0); k_dmma1684<<<blocks, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 512 * 8 * iters * (double)blocks * (bs / 32);
    printf("DMMA1684 bs=%4d : %.2f TFLOP/s\n", bs, fl / ms / 1e9);
    k_dmma16816<<<blocks, bs>>>(out, 10);
    cudaEventRecord(e0); k_dmma16816<<<blocks, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 2048 * 4 * iters * (double)blocks * (bs / 32);
    printf("DMMA16816 bs=%4d : %.2f TFLOP/s\n", bs, fl / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 2 GiB per buffer of double2
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k_copy<<<sms * 8, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 16 / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
