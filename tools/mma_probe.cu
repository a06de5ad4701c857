// Probe of the FP64 mma.sync shapes on sm_100a: fragment layouts (checked
// against a host product) and sustained throughput per shape.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

// m16n8k8 f64: A 16x8 row-major (4 per lane), B 8x8 col (2 per lane), C 16x8 (4 per lane)
__global__ void k_layout(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 8 + t], a1 = A[(g + 8) * 8 + t], a2 = A[g * 8 + t + 4], a3 = A[(g + 8) * 8 + t + 4];
  double b0 = B[t * 8 + g], b1 = B[(t + 4) * 8 + g];  // B[k][n]
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
               : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  C[g * 8 + 2 * t] = c0;
  C[g * 8 + 2 * t + 1] = c1;
  C[(g + 8) * 8 + 2 * t] = c2;
  C[(g + 8) * 8 + 2 * t + 1] = c3;
}

__global__ void k_tp884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4, d[8][2];
  for (int t = 0; t < 8; ++t) d[t][0] = d[t][1] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_tp1688(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4, d[4][4];
  for (int t = 0; t < 4; ++t) d[t][0] = d[t][1] = d[t][2] = d[t][3] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3])
                   : "d"(a), "d"(a), "d"(a), "d"(a), "d"(b), "d"(b));
  double s = 0;
  for (int t = 0; t < 4; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double hA[128], hB[64], hC[128], ref[128];
  for (int i = 0; i < 128; ++i) hA[i] = (i * 37 % 101) * 0.01 - 0.3;
  for (int i = 0; i < 64; ++i) hB[i] = (i * 53 % 97) * 0.01 - 0.4;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[k * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dC, *out;
  cudaMalloc(&dA, 1024); cudaMalloc(&dB, 512); cudaMalloc(&dC, 1024); cudaMalloc(&out, 1 << 24);
  cudaMemcpy(dA, hA, 1024, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 512, cudaMemcpyHostToDevice);
  k_layout<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, 1024, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("m16n8k8 layout max err %.3e (%s)\n", err, err < 1e-12 ? "layout OK" : "layout WRONG");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, bs = 128, iters = 4000;
  for (int mode = 0; mode < 2; ++mode) {
    if (mode == 0) k_tp884<<<blocks, bs>>>(out, 10); else k_tp1688<<<blocks, bs>>>(out, 10);
    cudaEventRecord(e0);
    if (mode == 0) k_tp884<<<blocks, bs>>>(out, iters); else k_tp1688<<<blocks, bs>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = blocks * bs / 32.0;
    double fl = mode == 0 ? warps * iters * 8 * 512.0 : warps * iters * 4 * 2048.0;
    printf("%s: %.2f TFLOP/s\n", mode == 0 ? "m8n8k4 " : "m16n8k8", fl / ms / 1e9);
  }
  return 0;
}
