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
//   k_tall_cols<0>        squared norms of the columns k..nc-1 over rows k..m-1
//                         (step 0; later steps get them from the update
//                         pass of the previous step, k_tall_cols<2>)
//   k_tall_pivot_reflect  first column of largest norm (ties to the lowest
//                         index, NaN never wins), column swap, jpvt /
//                         entry-norm swap; the reflector of column k (one
//                         thread: the vn chain)
//   k_tall_cols<2>        w and the update of every column c > k
//   k_tall_close          R(k,k) = alpha, zeros below it
// (k_tall_cols<1>: the entry norms, once).  The chains read their columns
// through shared-memory tiles so the global loads are coalesced.
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
constexpr int kU = 8;  // loads issued ahead of each run of dependent fmas

// s = fma(x, x, s) (and fma(y, y, s)) over rows [x0, m), the reference's
// order; the loads of kU rows are issued before their fmas so the chain runs
// at fma latency instead of load latency (same operations, same order)
template <bool CPLX>
__device__ __forceinline__ double sq_chain(const double* __restrict__ xr, const double* __restrict__ xi, int64_t x0,
                                           int64_t m, double s) {
  int64_t x = x0;
  for (; x + kU <= m; x += kU) {
    double r[kU], i[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      r[u] = xr[x + u];
      if (CPLX) i[u] = xi[x + u];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      s = fma(r[u], r[u], s);
      if (CPLX) s = fma(i[u], i[u], s);
    }
  }
  for (; x < m; ++x) {
    s = fma(xr[x], xr[x], s);
    if (CPLX) s = fma(xi[x], xi[x], s);
  }
  return s;
}

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
  const double vn = sq_chain<CPLX>(vr, vi, k, a.m, 0.0);
  a.scal[0] = alr;
  a.scal[1] = ali;
  a.scal[2] = 2.0 / vn;
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

// Column chains with coalesced loads: a warp owns 32 consecutive columns
// (one per lane) and walks the rows in tiles of 32: the tile is read column
// by column with lanes along the rows (coalesced), transposed through shared
// memory, and every lane then runs its own column's fma chain over the tile
// in row order — the reference's order.  MODE 0: squared norms over rows
// k.. of columns [c0, c0 + cnt) into cn; MODE 1: entry norms (rows 0..)
// into innorm; MODE 2: the reflector of column k applied to the columns
// [c0, c0 + cnt) (w = beta v^H a_c, then a_c -= v w, written back through
// the same tiles).
constexpr int kTile = 32;
constexpr int kWarps = 2;  // 64 columns per CTA (static shared memory < 48 KB for complex)
constexpr int kColThreads = kWarps * 32;

// one tile of rows [x0, x0 + 32) of the warp's columns into registers: lane
// l holds row x0 + l of every column (coalesced along the rows)
template <bool CPLX>
__device__ __forceinline__ void tile_load(const TallArgs& a, int cbase, int ncols, int64_t x0, int l, double* nr,
                                          double* ni) {
  const bool ok = x0 + l < a.m;
#pragma unroll
  for (int j = 0; j < kTile; ++j) {
    const bool on = ok && j < ncols;
    const int64_t e = (int64_t)(cbase + j) * a.m + x0 + l;
    nr[j] = on ? a.Ar[e] : 0.0;
    if (CPLX) ni[j] = on ? a.Ai[e] : 0.0;
  }
}

template <bool CPLX>
__device__ __forceinline__ void tile_put(double (*tr)[kTile + 1], double (*ti)[kTile + 1], int l, const double* nr,
                                         const double* ni) {
#pragma unroll
  for (int j = 0; j < kTile; ++j) {
    tr[l][j] = nr[j];
    if (CPLX) ti[l][j] = ni[j];
  }
}

// one row of a lane's chain: s += |a_x|^2 (MODE 0, 1) or w += conj(v_x) a_x
// (MODE 2), the reference's fma order
template <bool CPLX, int MODE>
__device__ __forceinline__ void chain_row(double (*TR)[kTile + 1], double (*TI)[kTile + 1], double (*sv)[kTile],
                                          int r, int l, double& s, double& wr, double& wi) {
  const double xr = TR[r][l];
  const double xi = CPLX ? TI[r][l] : 0.0;
  if (MODE != 2) {
    s = fma(xr, xr, s);
    if (CPLX) s = fma(xi, xi, s);
  } else {
    const double pr = sv[0][r];
    const double pi = CPLX ? sv[1][r] : 0.0;
    wr = fma(pr, xr, wr);
    if (CPLX) {
      wr = fma(pi, xi, wr);
      wi = fma(pr, xi, fma(-pi, xr, wi));
    }
  }
}

template <bool CPLX, int MODE>
__global__ void __launch_bounds__(kColThreads) k_tall_cols(TallArgs a, int k, int c0, int cnt) {
  __shared__ double tr[kWarps][kTile][kTile + 1];
  __shared__ double ti[CPLX ? kWarps : 1][kTile][kTile + 1];
  __shared__ double sv[kWarps][2][kTile];
  if (MODE != 1 && *a.flag) return;
  const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int cbase = c0 + (blockIdx.x * kWarps + wp) * 32;
  if (cbase >= c0 + cnt) return;
  const int ncols = min(32, c0 + cnt - cbase);
  const bool active = l < ncols;
  const int64_t m = a.m;
  const int64_t xs = MODE == 1 ? 0 : k;
  const double* vr = a.Ar + (int64_t)k * m;
  const double* vi = CPLX ? a.Ai + (int64_t)k * m : nullptr;
  double (*TR)[kTile + 1] = tr[wp];
  double (*TI)[kTile + 1] = ti[CPLX ? wp : 0];
  double nr[kTile], ni[CPLX ? kTile : 1];
  double s = 0.0, wr = 0.0, wi = 0.0;
  double pv_r = 0.0, pv_i = 0.0;
  // pass 1: the chains, the next tile's loads in flight under this tile's fmas
  tile_load<CPLX>(a, cbase, ncols, xs, l, nr, ni);
  if (MODE == 2 && xs + l < m) {
    pv_r = vr[xs + l];
    if (CPLX) pv_i = vi[xs + l];
  }
  for (int64_t x0 = xs; x0 < m; x0 += kTile) {
    const int rows = m - x0 < kTile ? (int)(m - x0) : kTile;
    tile_put<CPLX>(TR, TI, l, nr, ni);
    if (MODE == 2) {
      sv[wp][0][l] = pv_r;
      if (CPLX) sv[wp][1][l] = pv_i;
    }
    __syncwarp();
    if (x0 + kTile < m) {
      tile_load<CPLX>(a, cbase, ncols, x0 + kTile, l, nr, ni);
      if (MODE == 2 && x0 + kTile + l < m) {
        pv_r = vr[x0 + kTile + l];
        if (CPLX) pv_i = vi[x0 + kTile + l];
      }
    }
    if (active) {
      if (rows == kTile) {
        // full tile: unrolled, so the shared-memory reads run ahead of the
        // dependent fma chain
#pragma unroll
        for (int r = 0; r < kTile; ++r) chain_row<CPLX, MODE>(TR, TI, sv[wp], r, l, s, wr, wi);
      } else {
        for (int r = 0; r < rows; ++r) chain_row<CPLX, MODE>(TR, TI, sv[wp], r, l, s, wr, wi);
      }
    }
    __syncwarp();
  }
  if (MODE == 0) {
    if (active) a.cn[cbase + l] = s;
    return;
  }
  if (MODE == 1) {
    if (active) a.innorm[cbase + l] = sqrt(s);
    return;
  }
  const double beta = a.scal[2];
  wr *= beta;
  wi *= beta;
  s = 0.0;
  // pass 2: a_x -= v_x * w through the same tiles, written back coalesced
  tile_load<CPLX>(a, cbase, ncols, xs, l, nr, ni);
  if (xs + l < m) {
    pv_r = vr[xs + l];
    if (CPLX) pv_i = vi[xs + l];
  }
  for (int64_t x0 = xs; x0 < m; x0 += kTile) {
    const int rows = m - x0 < kTile ? (int)(m - x0) : kTile;
    tile_put<CPLX>(TR, TI, l, nr, ni);
    sv[wp][0][l] = pv_r;
    if (CPLX) sv[wp][1][l] = pv_i;
    __syncwarp();
    if (x0 + kTile < m) {
      tile_load<CPLX>(a, cbase, ncols, x0 + kTile, l, nr, ni);
      if (x0 + kTile + l < m) {
        pv_r = vr[x0 + kTile + l];
        if (CPLX) pv_i = vi[x0 + kTile + l];
      }
    }
    if (active) {
#pragma unroll 8
      for (int r = 0; r < rows; ++r) {
        const double pr = sv[wp][0][r];
        double xr = fma(-pr, wr, TR[r][l]);
        double xi = 0.0;
        if (CPLX) {
          const double pi = sv[wp][1][r];
          xr = fma(pi, wi, xr);
          xi = fma(-pr, wi, fma(-pi, wr, TI[r][l]));
          TI[r][l] = xi;
        }
        TR[r][l] = xr;
        // the next step's pivot norm of this column (rows k+1.., updated
        // values, the reference's order): k_tall_cols<0> folded in
        if (x0 + r > k) {
          s = fma(xr, xr, s);
          if (CPLX) s = fma(xi, xi, s);
        }
      }
    }
    __syncwarp();
    if (l < rows) {
      for (int j = 0; j < ncols; ++j) {
        a.Ar[(int64_t)(cbase + j) * m + x0 + l] = TR[l][j];
        if (CPLX) a.Ai[(int64_t)(cbase + j) * m + x0 + l] = TI[l][j];
      }
    }
    __syncwarp();
  }
  if (active) a.cn[cbase + l] = s;
}

inline int blocks_for(int64_t n) { return (int)((n + kTallThreads - 1) / kTallThreads); }
inline int col_blocks(int64_t n) { return (int)((n + kColThreads - 1) / kColThreads); }

template <bool CPLX>
int run_qr_rfactor(TallArgs a, int pivot, double tol_scale, int32_t* bad, cudaStream_t s) {
  k_tall_cols<CPLX, 1><<<col_blocks(a.nc), kColThreads, 0, s>>>(a, 0, 0, a.nc);
  for (int k = 0; k < a.nc; ++k) {
    // pivot norms: step 0 here, later steps from the previous update pass
    if (k == 0) {
      const int cnt = pivot ? a.nc : 1;
      k_tall_cols<CPLX, 0><<<col_blocks(cnt), kColThreads, 0, s>>>(a, 0, 0, cnt);
    }
    k_tall_pivot_reflect<CPLX><<<1, 1024, 0, s>>>(a, k, pivot);
    if (k + 1 < a.nc)
      k_tall_cols<CPLX, 2><<<col_blocks(a.nc - k - 1), kColThreads, 0, s>>>(a, k, k + 1, a.nc - k - 1);
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
