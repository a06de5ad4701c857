// Latency of the 2x2 building blocks and whole transforms (one warp,
// dependent chains): reference-order (FastMath, bitwise IEEE) vs the
// short-chain forms of the DMMA mode.  nvcc -I paper_1909_00101_b200/csrc.
#include <cstdio>

#include "hzg_device.cuh"

using namespace hzg;

__global__ void k(double* out, long long* cyc, double s0, int n) {
  double x = s0 + threadIdx.x * 1e-20;
  bool ok = true;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = approx_rsqrt(x + 0.5, ok);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fast_sqrt(x + 0.5, ok);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fast_div(1.5, x + 0.5, ok);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  double r;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x + 0.5));
    x = r;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // whole real transforms, chained through a11
  double a11 = 1.3 + x * 1e-30, a12 = 0.2, a22 = 0.7, xb = 0.1;
  FastMath fm;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    Xform X = transform_real(fm, a11, a12, a22, xb);
    a11 = 1.3 + X.z11 * 1e-30;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    Xform X = transform_real_approx(fm, a11, a12, a22, xb);
    a11 = 1.3 + X.z11 * 1e-30;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  double a12i = 0.05, b12i = 0.03;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    Xform X = transform_cplx(fm, a11, a12, a12i, a22, xb, b12i);
    a11 = 1.3 + X.z11 * 1e-30;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    Xform X = transform_cplx_approx(fm, a11, a12, a12i, a22, xb, b12i, xb * xb + b12i * b12i);
    a11 = 1.3 + X.z11 * 1e-30;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  // gates
  bool g = false;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double nb = 0;
    g ^= gate<false>(fm, a11, a12, 0.0, a22, xb, 0.0, 1e-14, &nb);
    a11 = 1.3 + (g ? 1e-30 : 0.0);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double nb2 = 0;
    g ^= gate_sq<false>(a11, a12, 0.0, a22, xb, 0.0, 1e-14, nb2, ok);
    a11 = 1.3 + (g ? 1e-30 : 0.0);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = (t1 - t0) / n;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + a11 + ok + fm.ok;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"approx_rsqrt", "fast_sqrt", "fast_div", "MUFU.RSQ64H", "xform_real", "xform_real_approx",
                         "xform_cplx", "xform_cplx_approx", "gate", "gate_sq"};
  k<<<1, 32>>>(out, cyc, 1.5, 10);
  k<<<1, 32>>>(out, cyc, 1.5, 1000);
  cudaDeviceSynchronize();
  for (int i = 0; i < 10; ++i) printf("%s %lld\n", names[i], cyc[i]);
  return 0;
}
