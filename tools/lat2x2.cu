// Latency of the 2x2 building blocks and whole transforms (one warp,
// dependent chains): reference-order (FastMath, bitwise IEEE) vs the
// short-chain forms of the DMMA mode.  nvcc -I paper_1909_00101_b200/csrc.
#include <cstdio>

#include "hzg_device.cuh"
#include "hzg_internal.h"

using namespace hzg;

// copy of hzg_inner.cu's pivot_scalar (same statements) for the probe
template <bool CPLX, bool APPROX, class M>
__device__ __forceinline__ int pivot_scalar_probe(M& m, const KernelCfg& kc, const double* q, double (&z)[6]) {
  double a11 = q[0], a22 = q[1], a12r = q[2], b11 = q[3], b22 = q[4], b12r = q[5];
  double a12i = CPLX ? q[6] : 0.0, b12i = CPLX ? q[7] : 0.0;
  if (!(a11 > 0.0 && a22 > 0.0 && b11 > 0.0 && b22 > 0.0)) return 8;
  double d11 = 1.0, d22 = 1.0;
  if (kc.per_step_rescale) rescale2(m, a11, a12r, a12i, a22, b11, b12r, b12i, b22, d11, d22);
  Xform X;
  if constexpr (APPROX) {
    double x2 = 0.0;
    if (gate_sq<CPLX>(a11, a12r, a12i, a22, b12r, b12i, kc.epsn, x2, m.ok)) return (kc.sorting && a11 < a22) ? 4 : 0;
    X = CPLX ? transform_cplx_approx(m, a11, a12r, a12i, a22, b12r, b12i, x2)
             : transform_real_approx(m, a11, a12r, a22, b12r);
  } else {
    double xb = -1.0;
    if (gate<CPLX>(m, a11, a12r, a12i, a22, b12r, b12i, kc.epsn, &xb)) return (kc.sorting && a11 < a22) ? 4 : 0;
    X = CPLX ? transform_cplx(m, a11, a12r, a12i, a22, b12r, b12i, xb) : transform_real(m, a11, a12r, a22, b12r);
  }
  const int bg = kc.crit_c2 ? !(X.cphi == 1.0 && X.cpsi == 1.0) : !(X.z11 == 1.0 && X.z22 == 1.0);
  int flags = 1 | (bg ? 2 : 0);
  if (kc.sorting && !CPLX) {
    double a1pp, a2pp;
    diag_after_real(X.z11, X.z12r, X.z21r, X.z22, a11, a12r, a22, a1pp, a2pp);
    if (a1pp < a2pp) flags |= 4;
  }
  z[0] = X.z11 * d11;
  z[1] = X.z12r * d11;
  z[2] = X.z12i * d11;
  z[3] = X.z21r * d22;
  z[4] = X.z21i * d22;
  z[5] = X.z22 * d22;
  return flags;
}

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
  // the whole real pivot as the DMMA-mode inner kernel runs it: gate on
  // squares, short-chain transform, C1 big flag, sort decision, d scaling
  KernelCfg kc{};
  kc.tw = 32; kc.prescale = 1; kc.sorting = 1; kc.max_inner_sweeps = 30; kc.epsn = 1e-14; kc.approx_2x2 = 1;
  double q[8] = {1.3, 0.7, 0.2, 1.0, 1.0, 0.1, 0.0, 0.0};
  double zz[6];
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    FastMath f2;
    const int fl = pivot_scalar_probe<false, true>(f2, kc, q, zz);
    q[0] = 1.3 + zz[0] * 1e-30 + fl * 1e-31;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[10] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    FastMath f2;
    const int fl = pivot_scalar_probe<false, false>(f2, kc, q, zz);
    q[0] = 1.3 + zz[0] * 1e-30 + fl * 1e-31;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[11] = (t1 - t0) / n;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + a11 + ok + fm.ok + q[0];
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"approx_rsqrt", "fast_sqrt", "fast_div", "MUFU.RSQ64H", "xform_real", "xform_real_approx",
                         "xform_cplx", "xform_cplx_approx", "gate", "gate_sq", "pivot_real_approx", "pivot_real_exact"};
  k<<<1, 32>>>(out, cyc, 1.5, 10);
  k<<<1, 32>>>(out, cyc, 1.5, 1000);
  cudaDeviceSynchronize();
  for (int i = 0; i < 12; ++i) printf("%s %lld\n", names[i], cyc[i]);
  return 0;
}
