// Column-pivoted Householder R factor of a tall m x nc matrix on the device,
// bitwise in the reference's operation order: _k_qr_rfactor
// (pkg/src/hzgsvd/blocked.py:97-217) as called by preprocess_tall
// (blocked.py:405-428), which shortens a tall pair (F, G) to n x n before the
// GSVD.
//
// The reference's dots are sequential fma chains over the rows, so one
// thread owns one column for every chain (column norms for the pivot
// choice, the reflector dot w = v^H a_c and the update a_c -= v w); the
// parallelism is across the remaining columns, and each step k is a short
// sequence of launches:
//   k_tall_norms   squared norms of the columns k..nc-1 over rows k..m-1
//   k_tall_pivot   first column of largest norm (ties to the lowest index,
//                  NaN never wins), column swap, jpvt / entry-norm swap
//   k_tall_reflect the reflector of column k (one thread: the vn chain)
//   k_tall_apply   w and the update of every column c > k
//   k_tall_close   R(k,k) = alpha, zeros below it
// then k_tall_final: the rank test against the entry norms and the phase
// fix that makes the diagonal real and nonnegative.  The matrix is m x nc
// column-major with leading dimension m (real and imaginary planes).

#include <cuda_runtime.h>

#include <cstdint>

#include "hzg_device.cuh"
#include "hzg_internal.h"

namespace hzg {
namespace {

constexpr int kTallThreads = 128;

struct TallArgs {
  double* Ar;
  double* Ai;  // nullptr for real
  int64_t m;
  int nc;
  double* innorm;  // [nc] entry norms
  double* cn;      // [nc] squared norms of the current step
  int64_t* jpvt;   // [nc]
  double* scal;    // alr, ali, beta
  int32_t* flag;   // [0]: 1 when a column vanished (the reference returns 1 at once)
};

template <bool CPLX>
__global__ void __launch_bounds__(kTallThreads) k_tall_innorm(TallArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nc) return;
  const double* xr = a.Ar + (int64_t)c * a.m;
  const double* xi = CPLX ? a.Ai + (int64_t)c * a.m : nullptr;
  double s = 0.0;
  for (int64_t x = 0; x < a.m; ++x) {
    s = fma(xr[x], xr[x], s);
    if (CPLX) s = fma(xi[x], xi[x], s);
  }
  a.innorm[c] = sqrt(s);
}

// squared norms over rows k.. of columns k + [0, cnt)
template <bool CPLX>
__global__ void __launch_bounds__(kTallThreads) k_tall_norms(TallArgs a, int k, int cnt) {
  const int c = k + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k + cnt || *a.flag) return;
  const double* xr = a.Ar + (int64_t)c * a.m;
  const double* xi = CPLX ? a.Ai + (int64_t)c * a.m : nullptr;
  double s = 0.0;
  for (int64_t x = k; x < a.m; ++x) {
    s = fma(xr[x], xr[x], s);
    if (CPLX) s = fma(xi[x], xi[x], s);
  }
  a.cn[c] = s;
}

// one CTA: pivot choice and column swap (pivot) and the reflector of
// column k (thread 0; its norm is the squared norm already computed for the
// column now at k, the same chain the reference runs after the swap)
template <bool CPLX>
__global__ void __launch_bounds__(1024) k_tall_pivot_reflect(TallArgs a, int k, int pivot) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  __shared__ int best_s;
  if (*a.flag) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (pivot) {
    // first maximum in column order (s > bestn, bestn starts at -1; NaN
    // never compares greater)
    double bv = -1.0;
    int bi = k;
    for (int c = k + tid; c < a.nc; c += nt) {
      const double v = a.cn[c];
      if (v > bv) {
        bv = v;
        bi = c;
      }
    }
    sv[tid] = bv;
    si[tid] = bi;
    __syncthreads();
    for (int h = nt / 2; h > 0; h >>= 1) {
      if (tid < h) {
        const double v2 = sv[tid + h];
        const int i2 = si[tid + h];
        if (v2 > sv[tid] || (v2 == sv[tid] && i2 < si[tid])) {
          sv[tid] = v2;
          si[tid] = i2;
        }
      }
      __syncthreads();
    }
    if (tid == 0) best_s = si[0];
    __syncthreads();
    const int best = best_s;
    if (best != k) {
      double* kr = a.Ar + (int64_t)k * a.m;
      double* br = a.Ar + (int64_t)best * a.m;
      for (int64_t x = tid; x < a.m; x += nt) {
        const double t = kr[x];
        kr[x] = br[x];
        br[x] = t;
        if (CPLX) {
          double* ki = a.Ai + (int64_t)k * a.m;
          double* bi2 = a.Ai + (int64_t)best * a.m;
          const double u = ki[x];
          ki[x] = bi2[x];
          bi2[x] = u;
        }
      }
      if (tid == 0) {
        const int64_t t2 = a.jpvt[k];
        a.jpvt[k] = a.jpvt[best];
        a.jpvt[best] = t2;
        const double t = a.innorm[k];
        a.innorm[k] = a.innorm[best];
        a.innorm[best] = t;
        a.cn[k] = a.cn[best];
      }
    }
    __syncthreads();
  }
  if (tid != 0) return;
  const double normx = sqrt(a.cn[k]);
  if (normx == 0.0) {
    *a.flag = 1;
    return;
  }
  double* vr = a.Ar + (int64_t)k * a.m;
  double* vi = CPLX ? a.Ai + (int64_t)k * a.m : nullptr;
  const double akr = vr[k];
  const double aki = CPLX ? vi[k] : 0.0;
  const double aa = hz_hypot(akr, aki);
  double phr, phi;
  if (aa == 0.0) {
    phr = 1.0;
    phi = 0.0;
  } else {
    phr = akr / aa;
    phi = aki / aa;
  }
  const double alr = -(phr * normx);
  const double ali = -(phi * normx);
  vr[k] -= alr;
  if (CPLX) vi[k] -= ali;
  double vn = 0.0;
  for (int64_t x = k; x < a.m; ++x) {
    vn = fma(vr[x], vr[x], vn);
    if (CPLX) vn = fma(vi[x], vi[x], vn);
  }
  a.scal[0] = alr;
  a.scal[1] = ali;
  a.scal[2] = 2.0 / vn;
}

template <bool CPLX>
__global__ void __launch_bounds__(kTallThreads) k_tall_apply(TallArgs a, int k) {
  const int c = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nc || *a.flag) return;
  const double beta = a.scal[2];
  const double* vr = a.Ar + (int64_t)k * a.m;
  const double* vi = CPLX ? a.Ai + (int64_t)k * a.m : nullptr;
  double* xr = a.Ar + (int64_t)c * a.m;
  double* xi = CPLX ? a.Ai + (int64_t)c * a.m : nullptr;
  double wr = 0.0, wi = 0.0;
  for (int64_t x = k; x < a.m; ++x) {
    // w += conj(v_x) * a_x
    wr = fma(vr[x], xr[x], wr);
    if (CPLX) {
      wr = fma(vi[x], xi[x], wr);
      wi = fma(vr[x], xi[x], fma(-vi[x], xr[x], wi));
    }
  }
  wr *= beta;
  wi *= beta;
  for (int64_t x = k; x < a.m; ++x) {
    // a_x -= v_x * w
    double r = fma(-vr[x], wr, xr[x]);
    if (CPLX) {
      r = fma(vi[x], wi, r);
      xi[x] = fma(-vr[x], wi, fma(-vi[x], wr, xi[x]));
    }
    xr[x] = r;
  }
}

template <bool CPLX>
__global__ void __launch_bounds__(kTallThreads) k_tall_close(TallArgs a, int k) {
  if (*a.flag) return;
  const int64_t x = k + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.m) return;
  double* vr = a.Ar + (int64_t)k * a.m;
  double* vi = CPLX ? a.Ai + (int64_t)k * a.m : nullptr;
  if (x == k) {
    vr[k] = a.scal[0];
    if (CPLX) vi[k] = a.scal[1];
  } else {
    vr[x] = 0.0;
    if (CPLX) vi[x] = 0.0;
  }
}

// rank test on the pre-fix diagonal, then the phase fix of row k (rows are
// independent); bad collects the OR over k
template <bool CPLX>
__global__ void __launch_bounds__(kTallThreads) k_tall_final(TallArgs a, double tol_scale, int32_t* bad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.nc || *a.flag) return;
  double* Ar = a.Ar;
  double* Ai = a.Ai;
  const int64_t m = a.m;
  const double dkr = Ar[(int64_t)k * m + k];
  const double dki = CPLX ? Ai[(int64_t)k * m + k] : 0.0;
  if (!(hz_hypot(dkr, dki) >= tol_scale * a.innorm[k])) atomicOr(bad, 1);
  if (CPLX) {
    const double mag = hz_hypot(dkr, dki);
    if (mag == 0.0) return;
    const double phr = dkr / mag;
    const double phi = -(dki / mag);
    for (int c = k; c < a.nc; ++c) {
      const int64_t e = (int64_t)c * m + k;
      const double re = fma(Ar[e], phr, -(Ai[e] * phi));
      const double im = fma(Ar[e], phi, Ai[e] * phr);
      Ar[e] = re;
      Ai[e] = im;
    }
    Ai[(int64_t)k * m + k] = 0.0;
  } else if (dkr < 0.0) {
    for (int c = k; c < a.nc; ++c) Ar[(int64_t)c * m + k] = -Ar[(int64_t)c * m + k];
  }
}

inline int blocks_for(int64_t n) { return (int)((n + kTallThreads - 1) / kTallThreads); }

template <bool CPLX>
int run_qr_rfactor(TallArgs a, int pivot, double tol_scale, int32_t* bad, cudaStream_t s) {
  k_tall_innorm<CPLX><<<blocks_for(a.nc), kTallThreads, 0, s>>>(a);
  for (int k = 0; k < a.nc; ++k) {
    const int cnt = pivot ? a.nc - k : 1;
    k_tall_norms<CPLX><<<blocks_for(cnt), kTallThreads, 0, s>>>(a, k, cnt);
    k_tall_pivot_reflect<CPLX><<<1, 1024, 0, s>>>(a, k, pivot);
    if (k + 1 < a.nc) k_tall_apply<CPLX><<<blocks_for(a.nc - k - 1), kTallThreads, 0, s>>>(a, k);
    k_tall_close<CPLX><<<blocks_for(a.m - k), kTallThreads, 0, s>>>(a, k);
  }
  k_tall_final<CPLX><<<blocks_for(a.nc), kTallThreads, 0, s>>>(a, tol_scale, bad);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

int launch_qr_rfactor(double* Ar, double* Ai, int64_t m, int nc, int cplx, int pivot, double tol_scale,
                      int64_t* jpvt, double* scratch /* >= 2 nc + 4 doubles */, int32_t* flags /* 2 */,
                      cudaStream_t s) {
  TallArgs a{Ar, cplx ? Ai : nullptr, m, nc, scratch, scratch + nc, jpvt, scratch + 2 * nc, flags};
  return cplx ? run_qr_rfactor<true>(a, pivot, tol_scale, flags + 1, s)
              : run_qr_rfactor<false>(a, pivot, tol_scale, flags + 1, s);
}

}  // namespace hzg
