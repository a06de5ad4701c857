// Reference-form accuracy check on the device (the reference's
// accuracy_report, pkg/src/hzgsvd/harness.py:323-465): X = Z^{-1} from an LU
// factorization with complete pivoting, then ||F - U S_F X||_F / ||F||_F,
// ||G - V S_G X||_F / ||G||_F, ||U^H U - I||_F and ||V^H V - I||_F with
// compensated accumulation.  A diagnostic beside the hot path, sized for the
// north-star orders (n = 16384: the trailing updates stream ~23 TB through
// HBM, ~4 s).
//
// * k_lu_* -- _k_lu_complete (harness.py:323-371) step by step: the
//   trailing update of step k (one fma per element, or the two-fma complex
//   forms), fused with the search for step k+1's pivot (|a|, glibc hypot
//   for complex; first maximum in the reference's row-major scan order),
//   then the row / column swap and the multipliers.  Each element's update
//   is a single rounding chain fixed by the reference, so the factors are
//   bitwise the reference's.
// * k_gemm_comp -- C = op(A) B with every entry a compensated dot product
//   (TwoProd by fma + TwoSum, Ogita-Rump-Oishi Dot2: as accurate as if
//   computed in twice the working precision), the role of the reference's
//   matmul_compensated (harness.py:151-196).
// * k_sumsq_comp -- the compensated sum of squared magnitudes of A - B (or
//   of A), for the Frobenius norms (harness.py:208-216).
#include <cstdint>

#include "../../include/hzg.h"
#include "hzg_device.cuh"
#include "hzg_internal.h"

namespace hzg {
namespace {

// (magnitude, linear row-major index) with the reference's preference:
// larger magnitude, then the earlier (row, column) in its scan order
struct PivotKey {
  double m;
  int64_t idx;  // i * n + j (row-major), -1: none
};

__device__ __forceinline__ bool better(const PivotKey& a, const PivotKey& b) {
  if (a.idx < 0) return false;
  if (b.idx < 0) return true;
  if (a.m > b.m) return true;
  if (a.m < b.m) return false;
  return a.idx < b.idx;
}

__device__ __forceinline__ PivotKey warp_best(PivotKey k) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    PivotKey o;
    o.m = __shfl_xor_sync(0xffffffffu, k.m, d);
    o.idx = __shfl_xor_sync(0xffffffffu, k.idx, d);
    if (better(o, k)) k = o;
  }
  return k;
}

__device__ __forceinline__ double mag(double re, double im, int cplx) {
  return cplx ? hz_hypot(re, im) : fabs(re);
}

constexpr int kLT = 32;  // trailing-update tile: 32 x 32 elements, 256 threads

// Trailing update of step k (rows, cols > k) and the block's best pivot
// candidate for step k + 1 over rows, cols >= k + 1.  k = -1: no update,
// only the search over the whole matrix.  L (multipliers of step k) is in
// column k already; row k holds U's row.
__global__ void __launch_bounds__(256) k_lu_update(double* Ar, double* Ai, int64_t n, int64_t ld, int64_t k,
                                                   int cplx, PivotKey* part) {
  const int64_t base = k + 1;
  const int64_t r0 = base + (int64_t)blockIdx.x * kLT, c0 = base + (int64_t)blockIdx.y * kLT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 rows x 8 column lanes
  PivotKey best{0.0, -1};
  const int64_t i = r0 + tx;
  double lr = 0.0, li = 0.0;
  if (k >= 0 && i < n) {
    lr = Ar[k * ld + i];
    li = cplx ? Ai[k * ld + i] : 0.0;
  }
  for (int cc = ty; cc < kLT; cc += 8) {
    const int64_t j = c0 + cc;
    if (i >= n || j >= n) continue;
    double ar = Ar[j * ld + i];
    double ai = cplx ? Ai[j * ld + i] : 0.0;
    if (k >= 0) {
      const double ur = Ar[j * ld + k];
      if (cplx) {
        const double ui = Ai[j * ld + k];
        const double nr = fma(-lr, ur, fma(li, ui, ar));
        const double ni = fma(-lr, ui, fma(-li, ur, ai));
        ar = nr;
        ai = ni;
        Ai[j * ld + i] = ai;
      } else {
        ar = fma(-lr, ur, ar);
      }
      Ar[j * ld + i] = ar;
    }
    const double m = mag(ar, ai, cplx);
    // the reference takes m > best from best = 0: zero entries never pivot
    PivotKey c{m, m > 0.0 ? i * n + j : -1};
    if (better(c, best)) best = c;
  }
  best = warp_best(best);
  __shared__ PivotKey red[8];
  if (tx == 0) red[ty] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    PivotKey b = red[0];
    for (int q = 1; q < 8; ++q)
      if (better(red[q], b)) b = red[q];
    part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = b;
  }
}

// Reduce the block candidates, swap row k <-> pivot row and column k <->
// pivot column (whole rows / columns, as the reference does), record the
// permutations, then form the multipliers of column k.  One CTA.
__global__ void __launch_bounds__(1024) k_lu_pivot(double* Ar, double* Ai, int64_t n, int64_t ld, int64_t k,
                                                  int cplx, const PivotKey* part, int64_t nparts, int64_t* rp,
                                                  int64_t* cp, int32_t* status) {
  __shared__ PivotKey red[32];
  __shared__ int64_t sbr, sbc;
  PivotKey best{0.0, -1};
  for (int64_t q = threadIdx.x; q < nparts; q += blockDim.x)
    if (better(part[q], best)) best = part[q];
  best = warp_best(best);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    PivotKey b = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (better(red[q], b)) b = red[q];
    if (b.idx < 0) {
      *status = 1;  // best == 0: singular
      sbr = sbc = -1;
    } else {
      sbr = b.idx / n;
      sbc = b.idx % n;
      if (sbr != k) {
        const int64_t t = rp[k];
        rp[k] = rp[sbr];
        rp[sbr] = t;
      }
      if (sbc != k) {
        const int64_t t = cp[k];
        cp[k] = cp[sbc];
        cp[sbc] = t;
      }
    }
  }
  __syncthreads();
  const int64_t br = sbr, bc = sbc;
  if (br < 0) return;
  // row swap (all n columns), then column swap (all n rows)
  if (br != k)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      double t = Ar[j * ld + k];
      Ar[j * ld + k] = Ar[j * ld + br];
      Ar[j * ld + br] = t;
      if (cplx) {
        t = Ai[j * ld + k];
        Ai[j * ld + k] = Ai[j * ld + br];
        Ai[j * ld + br] = t;
      }
    }
  __syncthreads();
  if (bc != k)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      double t = Ar[k * ld + i];
      Ar[k * ld + i] = Ar[bc * ld + i];
      Ar[bc * ld + i] = t;
      if (cplx) {
        t = Ai[k * ld + i];
        Ai[k * ld + i] = Ai[bc * ld + i];
        Ai[bc * ld + i] = t;
      }
    }
  __syncthreads();
  // multipliers (harness.py:359-368)
  const double pr = Ar[k * ld + k];
  const double pi = cplx ? Ai[k * ld + k] : 0.0;
  const double den = cplx ? fma(pr, pr, pi * pi) : 0.0;
  for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
    if (cplx) {
      const double xr = Ar[k * ld + i], xi = Ai[k * ld + i];
      Ar[k * ld + i] = fma(xr, pr, xi * pi) / den;
      Ai[k * ld + i] = fma(xi, pr, -(xr * pi)) / den;
    } else {
      Ar[k * ld + i] = Ar[k * ld + i] / pr;
    }
  }
}

// ---------------------------------------------------------------------------
// compensated products
// ---------------------------------------------------------------------------
struct Dd {
  double s, c;  // value s + c (c: accumulated rounding errors)
};

__device__ __forceinline__ void dd_add_prod(Dd& d, double a, double b) {
  const double p = a * b;
  const double e = fma(a, b, -p);  // a b = p + e exactly
  const double t = d.s + p;        // TwoSum(s, p)
  const double z = t - d.s;
  const double err = (d.s - (t - z)) + (p - z);
  d.s = t;
  d.c += err + e;
}

constexpr int kGT = 64, kGK = 16;  // output tile 64 x 64, k-slices of 16; 256 threads, 4 x 4 per thread

// C (m x n) = op(A) B, op(A) = A (m x k, lda) or A^H (A: k x m, lda);
// column-major planes; cplx: split planes.  Every entry a compensated dot.
template <bool CPLX, bool TRANS>
__global__ void __launch_bounds__(256) k_gemm_comp(int64_t m, int64_t n, int64_t kk, const double* Ar, const double* Ai,
                                                   int64_t lda, const double* Br, const double* Bi, int64_t ldb,
                                                   double* Cr, double* Ci, int64_t ldc) {
  __shared__ double sAr[kGK][kGT + 1], sBr[kGK][kGT + 1];
  __shared__ double sAi[CPLX ? kGK : 1][kGT + 1], sBi[CPLX ? kGK : 1][kGT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = (int64_t)blockIdx.x * kGT, j0 = (int64_t)blockIdx.y * kGT;
  Dd accr[4][4], acci[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) accr[a][b] = acci[a][b] = Dd{0.0, 0.0};
  for (int64_t k0 = 0; k0 < kk; k0 += kGK) {
    for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
      const int kl = e / kGT, r = e % kGT;
      const int64_t kg = k0 + kl;
      // A tile: op(A)[i0 + r][kg]
      double ar = 0.0, ai = 0.0;
      if (kg < kk && i0 + r < m) {
        const int64_t off = TRANS ? (i0 + r) * lda + kg : kg * lda + i0 + r;
        ar = Ar[off];
        if (CPLX) ai = TRANS ? -Ai[off] : Ai[off];
      }
      sAr[kl][r] = ar;
      if (CPLX) sAi[kl][r] = ai;
      double br = 0.0, bi = 0.0;
      if (kg < kk && j0 + r < n) {
        br = Br[(j0 + r) * ldb + kg];
        if (CPLX) bi = Bi[(j0 + r) * ldb + kg];
      }
      sBr[kl][r] = br;
      if (CPLX) sBi[kl][r] = bi;
    }
    __syncthreads();
#pragma unroll 4
    for (int kl = 0; kl < kGK; ++kl) {
      double a_r[4], a_i[4], b_r[4], b_i[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a_r[q] = sAr[kl][tx + 16 * q];
        b_r[q] = sBr[kl][ty + 16 * q];
        a_i[q] = CPLX ? sAi[kl][tx + 16 * q] : 0.0;
        b_i[q] = CPLX ? sBi[kl][ty + 16 * q] : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dd_add_prod(accr[a][b], a_r[a], b_r[b]);
          if (CPLX) {
            dd_add_prod(accr[a][b], -a_i[a], b_i[b]);
            dd_add_prod(acci[a][b], a_r[a], b_i[b]);
            dd_add_prod(acci[a][b], a_i[a], b_r[b]);
          }
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + tx + 16 * a, j = j0 + ty + 16 * b;
      if (i < m && j < n) {
        Cr[j * ldc + i] = accr[a][b].s + accr[a][b].c;
        if (CPLX) Ci[j * ldc + i] = acci[a][b].s + acci[a][b].c;
      }
    }
}

// Compensated sum over all elements of |A - B|^2 (B may be null; with
// `eye`, B is the identity) into per-block (s, c) partials.
__global__ void __launch_bounds__(256) k_sumsq_comp(int64_t rows, int64_t cols, const double* Ar, const double* Ai,
                                                    int64_t lda, const double* Br, const double* Bi, int64_t ldb,
                                                    int eye, double* part) {
  Dd acc{0.0, 0.0};
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e % rows;
    double dr = Ar[j * lda + i], di = Ai ? Ai[j * lda + i] : 0.0;
    if (Br) {
      dr -= Br[j * ldb + i];
      if (Bi) di -= Bi[j * ldb + i];
    }
    if (eye && i == j) dr -= 1.0;
    dd_add_prod(acc, dr, dr);
    if (Ai || Bi) dd_add_prod(acc, di, di);
  }
  // block reduction of (s, c) pairs: TwoSum on s, plain sum of c
  __shared__ double ss[256], sc[256];
  ss[threadIdx.x] = acc.s;
  sc[threadIdx.x] = acc.c;
  __syncthreads();
  for (int h = 128; h >= 1; h >>= 1) {
    if ((int)threadIdx.x < h) {
      const double a = ss[threadIdx.x], b = ss[threadIdx.x + h];
      const double t = a + b, z = t - a;
      const double err = (a - (t - z)) + (b - z);
      ss[threadIdx.x] = t;
      sc[threadIdx.x] += sc[threadIdx.x + h] + err;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = ss[0];
    part[2 * blockIdx.x + 1] = sc[0];
  }
}

}  // namespace
}  // namespace hzg

using namespace hzg;

extern "C" {

size_t hzg_lu_workspace_bytes(int64_t n) {
  const int64_t t = (n + kLT - 1) / kLT;
  return (size_t)(t * t) * sizeof(PivotKey) + 64;
}

int hzg_lu_complete(int64_t n, int32_t is_complex, double* Ar, double* Ai, int64_t ld, int64_t* rp, int64_t* cp,
                    void* workspace, int32_t* status, void* stream) {
  if (n < 1 || !Ar || (is_complex && !Ai) || ld < n || !rp || !cp || !workspace || !status) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  PivotKey* part = (PivotKey*)workspace;
  cudaMemsetAsync(status, 0, 4, s);
  for (int64_t k = 0; k < n; ++k) {
    // update of step k - 1 fused with the pivot search of step k
    const int64_t rem = n - k;
    const unsigned g = (unsigned)((rem + kLT - 1) / kLT);
    k_lu_update<<<dim3(g, g), 256, 0, s>>>(Ar, Ai, n, ld, k - 1, is_complex, part);
    k_lu_pivot<<<1, 1024, 0, s>>>(Ar, Ai, n, ld, k, is_complex, part, (int64_t)g * g, rp, cp, status);
  }
  return cudaGetLastError() == cudaSuccess ? HZG_OK : HZG_CUDA;
}

int hzg_gemm_comp(int64_t m, int64_t n, int64_t k, int32_t is_complex, int32_t trans_a, const double* Ar,
                  const double* Ai, int64_t lda, const double* Br, const double* Bi, int64_t ldb, double* Cr,
                  double* Ci, int64_t ldc, void* stream) {
  if (m < 1 || n < 1 || k < 1 || !Ar || !Br || !Cr || (is_complex && (!Ai || !Bi || !Ci))) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)((m + kGT - 1) / kGT), (unsigned)((n + kGT - 1) / kGT));
  if (is_complex) {
    if (trans_a) k_gemm_comp<true, true><<<grid, 256, 0, s>>>(m, n, k, Ar, Ai, lda, Br, Bi, ldb, Cr, Ci, ldc);
    else k_gemm_comp<true, false><<<grid, 256, 0, s>>>(m, n, k, Ar, Ai, lda, Br, Bi, ldb, Cr, Ci, ldc);
  } else {
    if (trans_a) k_gemm_comp<false, true><<<grid, 256, 0, s>>>(m, n, k, Ar, nullptr, lda, Br, nullptr, ldb, Cr, nullptr, ldc);
    else k_gemm_comp<false, false><<<grid, 256, 0, s>>>(m, n, k, Ar, nullptr, lda, Br, nullptr, ldb, Cr, nullptr, ldc);
  }
  return cudaGetLastError() == cudaSuccess ? HZG_OK : HZG_CUDA;
}

int hzg_sumsq_comp(int64_t rows, int64_t cols, const double* Ar, const double* Ai, int64_t lda, const double* Br,
                   const double* Bi, int64_t ldb, int32_t eye, double* partials, int32_t nblocks, void* stream) {
  if (rows < 1 || cols < 1 || !Ar || !partials || nblocks < 1) return HZG_INVALID;
  k_sumsq_comp<<<nblocks, 256, 0, (cudaStream_t)stream>>>(rows, cols, Ar, Ai, lda, Br, Bi, ldb, eye, partials);
  return cudaGetLastError() == cudaSuccess ? HZG_OK : HZG_CUDA;
}

}  // extern "C"
