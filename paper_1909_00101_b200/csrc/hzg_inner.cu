// The per-block-pair inner solve: subphases 2 and 3 of the paper's bstep
// kernel, re-designed for sm_100a.
//
// One CTA per block pair of the step, one warp per pivot of an inner step
// (w warps), the 2w x 2w factors resident in shared memory.  Per CTA:
//   1. fold the Grammian partials of F and G (pairwise over the splits),
//   2. two column-oriented Cholesky factorizations (one warp each),
//   3. in-block prescale, pointwise HZ sweeps over the inner table,
//   4. theta rescale, exact-identity test, write Z~ and the counters.
// All arithmetic mirrors the reference statement by statement (see
// hzg_device.cuh), so given the same Grammians the factors, Z~ and the
// counters are bitwise those of the reference's _block_task
// (blocked.py:435-484; pointwise.py:161-293).
#include <cstdio>
#include <cstdlib>

#include "hzg_device.cuh"
#include "hzg_internal.h"

namespace hzg {

namespace {

constexpr int kMaxTW = 64;

template <int TW, bool CPLX>
struct InnerSmem {
  static constexpr int NP = CPLX ? 2 : 1;
  double A[NP][TW * TW];  // F-hat, column-major (element (r, c) at c*TW + r)
  double B[NP][TW * TW];  // G-hat
  double Z[NP][TW * TW];  // Z-hat
  uint8_t tab[TW * TW];   // inner table, (steps, TW/2, 2)
  double pd[TW / 2][9];   // phase A -> B: a11 a22 a12r b11 b22 b12r a12i b12i (stride 9: no bank conflicts)
  double px[TW / 2][7];   // phase B -> C: z11 z12r z12i z21r z21i z22 (stride 7)
  int pflag[TW / 2];
  int stepbad, sw_applied, sw_big;
  int chol_fail[2];
};

// Values of one column held by a warp: lane l owns rows l*EPL .. l*EPL+EPL-1.
template <int TW>
struct Lanes {
  static constexpr int EPL = TW > 32 ? 2 : 1;
};

// Sum of one per-lane quantity in the reference tree shape.
template <int EPL>
__device__ __forceinline__ double lane_tree(const double (&p)[EPL]) {
  double v = p[0];
  if (EPL == 2) v = p[0] + p[1];
  return warp_tree(v);
}

template <int TW, bool CPLX>
__device__ __forceinline__ void load_col(const double* __restrict__ re, const double* __restrict__ im, int col,
                                         int lane, double (&r)[Lanes<TW>::EPL], double (&i)[Lanes<TW>::EPL]) {
  constexpr int EPL = Lanes<TW>::EPL;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    int row = lane * EPL + e;
    bool ok = row < TW;
    r[e] = ok ? re[col * TW + row] : 0.0;
    i[e] = (CPLX && ok) ? im[col * TW + row] : 0.0;
  }
}

template <int TW, bool CPLX>
__device__ __forceinline__ void store_col(double* re, double* im, int col, int lane,
                                          const double (&r)[Lanes<TW>::EPL], const double (&i)[Lanes<TW>::EPL]) {
  constexpr int EPL = Lanes<TW>::EPL;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    int row = lane * EPL + e;
    if (row < TW) {
      re[col * TW + row] = r[e];
      if (CPLX) im[col * TW + row] = i[e];
    }
  }
}

// |y|^2 elementwise as the reference forms it (dotprod.py:206-211, :227-232)
template <bool CPLX>
__device__ __forceinline__ double nrm_term(double r, double i) {
  return CPLX ? fma(i, i, r * r) : r * r;
}

// conj(a) * b elementwise (dotprod.py:146-155 with conj_first, s = -1)
__device__ __forceinline__ double dot_re_term(double ar, double ai, double br, double bi) {
  return fma(ar, br, -((-1.0 * ai) * bi));
}
__device__ __forceinline__ double dot_im_term(double ar, double ai, double br, double bi) {
  return fma(ar, bi, (-1.0 * ai) * br);
}

// Column-oriented Cholesky of a Hermitian TW x TW matrix by one warp, in the
// exact operation order of blocked.py:59-94 (lane x owns row x).
template <int TW, bool CPLX>
__device__ int warp_cholesky(double* Ar, double* Ai, int lane) {
#define A_(x, y) Ar[(y) * TW + (x)]
#define AI_(x, y) Ai[(y) * TW + (x)]
  for (int j = 0; j < TW; ++j) {
    double d = A_(j, j);
    if (!(d > 0.0) || !isfinite(d)) return 1;
    double rt = sqrt(d);
    double rinv = 1.0 / rt;
    __syncwarp();
    for (int x = lane; x < TW; x += 32) {
      if (x == j) {
        A_(j, j) = rt;
        if (CPLX) AI_(j, j) = 0.0;
      } else if (x > j) {
        A_(x, j) *= rinv;
        if (CPLX) AI_(x, j) *= rinv;
      }
    }
    __syncwarp();
    for (int x = lane; x < TW; x += 32) {
      if (x <= j) continue;
      double ar = -A_(x, j);
      double ai = CPLX ? -AI_(x, j) : 0.0;
      for (int jp = j + 1; jp <= x; ++jp) {
        double br = A_(jp, j);
        if (CPLX) {
          double bi = -AI_(jp, j);
          A_(x, jp) = fma(ar, br, fma(-ai, bi, A_(x, jp)));
          AI_(x, jp) = fma(ar, bi, fma(ai, br, AI_(x, jp)));
        } else {
          A_(x, jp) = fma(ar, br, A_(x, jp));
        }
      }
    }
    __syncwarp();
  }
  // conj-transpose into the upper triangle, zero the strict lower one
  for (int r = lane; r < TW; r += 32)
    for (int s = 0; s < r; ++s) {
      A_(s, r) = A_(r, s);
      if (CPLX) AI_(s, r) = -AI_(r, s);
      A_(r, s) = 0.0;
      if (CPLX) AI_(r, s) = 0.0;
    }
  __syncwarp();
  return 0;
#undef A_
#undef AI_
}

// Householder R factor of the m x TW block-column stack (blocked.py:97-217
// with pivot=False, via _shorten_qr :487-500), bitwise in the reference's
// sequential fma order.  Sequential chains over m make this slow; it only
// runs for the rare pairs whose Grammian fails Cholesky.
template <int TW, bool CPLX>
__device__ int block_qr(const Plane& Y, int64_t c0, int64_t c1, int w, double* Sr, double* Si, double* outR,
                        double* outI, double* sh /* >= 3*TW + 8 doubles */) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t m = Y.rows;
  for (int64_t e = tid; e < m * TW; e += nt) {
    int k = (int)(e / m);
    int64_t x = e - (int64_t)k * m;
    int64_t c = k < w ? c0 + k : c1 + (k - w);
    Sr[e] = Y.re[c * Y.ld + x];
    if (CPLX) Si[e] = Y.im[c * Y.ld + x];
  }
  __syncthreads();
#define S_(x, y) Sr[(x) + (int64_t)(y) * m]
#define SI_(x, y) Si[(x) + (int64_t)(y) * m]
  double* innorm = sh;
  double* wv_r = sh + TW;
  double* wv_i = sh + 2 * TW;
  double* scal = sh + 3 * TW;  // alr, ali, beta, bad
  if (tid < TW) {
    double s = 0.0;
    for (int64_t x = 0; x < m; ++x) {
      s = fma(S_(x, tid), S_(x, tid), s);
      if (CPLX) s = fma(SI_(x, tid), SI_(x, tid), s);
    }
    innorm[tid] = sqrt(s);
  }
  __syncthreads();
  for (int k = 0; k < TW; ++k) {
    if (tid == 0) {
      double s = 0.0;
      for (int64_t x = k; x < m; ++x) {
        s = fma(S_(x, k), S_(x, k), s);
        if (CPLX) s = fma(SI_(x, k), SI_(x, k), s);
      }
      double normx = sqrt(s);
      scal[3] = normx == 0.0 ? 1.0 : 0.0;
      if (normx != 0.0) {
        double akr = S_(k, k);
        double aki = CPLX ? SI_(k, k) : 0.0;
        double aa = hz_hypot(akr, aki);
        double phr, phi;
        if (aa == 0.0) {
          phr = 1.0;
          phi = 0.0;
        } else {
          phr = akr / aa;
          phi = aki / aa;
        }
        double alr = -(phr * normx);
        double ali = -(phi * normx);
        S_(k, k) -= alr;
        if (CPLX) SI_(k, k) -= ali;
        double vn = 0.0;
        for (int64_t x = k; x < m; ++x) {
          vn = fma(S_(x, k), S_(x, k), vn);
          if (CPLX) vn = fma(SI_(x, k), SI_(x, k), vn);
        }
        scal[0] = alr;
        scal[1] = ali;
        scal[2] = 2.0 / vn;
      }
    }
    __syncthreads();
    if (scal[3] != 0.0) return 1;
    double beta = scal[2];
    int c = k + 1 + tid;
    if (c < TW) {
      double wr = 0.0, wi = 0.0;
      for (int64_t x = k; x < m; ++x) {
        wr = fma(S_(x, k), S_(x, c), wr);
        if (CPLX) {
          wr = fma(SI_(x, k), SI_(x, c), wr);
          wi = fma(S_(x, k), SI_(x, c), fma(-SI_(x, k), S_(x, c), wi));
        }
      }
      wv_r[c] = wr * beta;
      wv_i[c] = wi * beta;
    }
    __syncthreads();
    const int ncols = TW - k - 1;
    const int64_t nrow = m - k;
    for (int64_t e = tid; e < nrow * ncols; e += nt) {
      int cc = k + 1 + (int)(e / nrow);
      int64_t x = k + (e % nrow);
      double wr = wv_r[cc], wi = wv_i[cc];
      double v = fma(-S_(x, k), wr, S_(x, cc));
      if (CPLX) {
        v = fma(SI_(x, k), wi, v);
        SI_(x, cc) = fma(-S_(x, k), wi, fma(-SI_(x, k), wr, SI_(x, cc)));
      }
      S_(x, cc) = v;
    }
    __syncthreads();
    if (tid == 0) {
      S_(k, k) = scal[0];
      if (CPLX) SI_(k, k) = scal[1];
    }
    for (int64_t x = k + 1 + tid; x < m; x += nt) {
      S_(x, k) = 0.0;
      if (CPLX) SI_(x, k) = 0.0;
    }
    __syncthreads();
  }
  const double tol = TW * 2.220446049250313e-16;
  if (tid == 0) {
    int bad = 0;
    for (int k = 0; k < TW; ++k)
      if (!(hz_hypot(S_(k, k), CPLX ? SI_(k, k) : 0.0) >= tol * innorm[k])) bad = 1;
    scal[3] = bad;
    for (int k = 0; k < TW; ++k) {
      double dkr = S_(k, k);
      double dki = CPLX ? SI_(k, k) : 0.0;
      if (CPLX) {
        double mag = hz_hypot(dkr, dki);
        if (mag == 0.0) continue;
        double phr = dkr / mag, phi = -(dki / mag);
        for (int c = k; c < TW; ++c) {
          double re = fma(S_(k, c), phr, -(SI_(k, c) * phi));
          double im = fma(S_(k, c), phi, SI_(k, c) * phr);
          S_(k, c) = re;
          SI_(k, c) = im;
        }
        SI_(k, k) = 0.0;
      } else if (dkr < 0.0) {
        for (int c = k; c < TW; ++c) S_(k, c) = -S_(k, c);
      }
    }
  }
  __syncthreads();
  int bad = scal[3] != 0.0;
  for (int e = tid; e < TW * TW; e += nt) {
    int r = e % TW, c = e / TW;
    outR[c * TW + r] = S_(r, c);
    if (CPLX) outI[c * TW + r] = SI_(r, c);
  }
  __syncthreads();
  return bad;
#undef S_
#undef SI_
}

// _k_process_pivot's scalar part (pointwise.py:165-207) for one pivot:
// q = {a11, a22, a12r, b11, b22, b12r, a12i, b12i}.  Returns flags (1 applied,
// 2 big, 4 swap, 8 bad) and, when applied, the rescaled Z-hat entries.
template <bool CPLX, class M>
__device__ __forceinline__ int pivot_scalar(M& m, const KernelCfg& kc, const double* q, double (&z)[6]) {
  double a11 = q[0], a22 = q[1], a12r = q[2], b11 = q[3], b22 = q[4], b12r = q[5];
  double a12i = CPLX ? q[6] : 0.0, b12i = CPLX ? q[7] : 0.0;
  if (!(a11 > 0.0 && a22 > 0.0 && b11 > 0.0 && b22 > 0.0)) return 8;
  double d11 = 1.0, d22 = 1.0;
  if (kc.per_step_rescale) rescale2(m, a11, a12r, a12i, a22, b11, b12r, b12i, b22, d11, d22);
  if (gate<CPLX>(m, a11, a12r, a12i, a22, b12r, b12i, kc.epsn)) return (kc.sorting && a11 < a22) ? 4 : 0;
  Xform X = transform<CPLX>(m, a11, a12r, a12i, a22, b12r, b12i);
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

struct InnerParams {
  Plane F, G;
  StepPairs sp;
  int step;
  KernelCfg kc;
  GramWS gw;
  const int32_t* itable;
  int isteps;
  InnerOut io;
  double* qr_scratch;
  int qr_slots;
  int32_t* qr_locks;
};

template <int TW, bool CPLX, int PPW>
__global__ void __launch_bounds__(TW / 2 / PPW * 32) k_inner(InnerParams P) {
  constexpr int NPIV = TW / 2;      // pivots per inner step
  constexpr int NW = NPIV / PPW;    // warps: each forms / applies PPW pivots
  constexpr int EPL = Lanes<TW>::EPL;
  constexpr int NP = CPLX ? 2 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<InnerSmem<TW, CPLX>*>(smem_raw);
  const int pair = P.sp.p0 + blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = blockDim.x;
  const KernelCfg& kc = P.kc;

  // ---- the inner strategy table ------------------------------------------
  for (int e = tid; e < P.isteps * TW; e += nt) S.tab[e] = (uint8_t)P.itable[e];
  if (tid == 0) {
    S.chol_fail[0] = S.chol_fail[1] = 0;
  }

  // ---- fold the Grammian partials (pairwise over splits) -----------------
  for (int mat = 0; mat < 2; ++mat) {
    const int ns = P.gw.nsplit[mat];
    const double* base = P.gw.part + ((int64_t)pair * 2 + mat) * P.gw.smax * NP * TW * TW;
    double(*M)[TW * TW] = mat == 0 ? S.A : S.B;
    for (int e = tid; e < TW * TW; e += nt) {
      int r = e % TW, c = e / TW;
      if (r > c) continue;
      for (int pl = 0; pl < NP; ++pl) {
        PairwiseAcc<9> acc;
        acc.reset();
        for (int s = 0; s < ns; ++s) acc.push(base[((int64_t)s * NP + pl) * TW * TW + e]);
        double v = acc.result();
        if (pl == 0) {
          M[0][c * TW + r] = v;
          M[0][r * TW + c] = v;
        } else {
          M[1][c * TW + r] = r == c ? 0.0 : v;
          M[1][r * TW + c] = r == c ? 0.0 : -v;
        }
      }
    }
  }
  __syncthreads();

  // ---- Cholesky of both Grammians (warp 0: F, warp 1: G) -----------------
  if (warp < 2) {
    double* Mr = warp == 0 ? S.A[0] : S.B[0];
    double* Mi = CPLX ? (warp == 0 ? S.A[NP - 1] : S.B[NP - 1]) : nullptr;
    int f = warp_cholesky<TW, CPLX>(Mr, Mi, lane);
    if (lane == 0) S.chol_fail[warp] = f;
  }
  if (NW == 1) {  // a single warp: factor G after F
    __syncwarp();
    int f = warp_cholesky<TW, CPLX>(S.B[0], CPLX ? S.B[NP - 1] : nullptr, lane);
    if (lane == 0) S.chol_fail[1] = f;
  }
  __syncthreads();

  int status = ST_OK;
  for (int mat = 0; mat < 2; ++mat) {
    if (!S.chol_fail[mat]) continue;
    if (!kc.fallback_qr) {
      status = ST_NOT_PD;
      break;
    }
    // QR shortening of this matrix's block columns (blocked.py:450-462)
    const Plane& Y = mat == 0 ? P.F : P.G;
    const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
    __shared__ int slot;
    __shared__ double qsh[3 * kMaxTW + 8];
    if (tid == 0) {
      int s0 = pair % P.qr_slots, sl = -1;
      for (int it = 0; sl < 0; ++it) {
        int cand = (s0 + it) % P.qr_slots;
        if (atomicCAS(&P.qr_locks[cand], 0, 1) == 0) sl = cand;
      }
      __threadfence();
      slot = sl;
    }
    __syncthreads();
    int64_t span = (int64_t)Y.rows * TW;
    double* Sr = P.qr_scratch + (int64_t)slot * 2 * span;
    double* Si = Sr + span;
    double* outR = mat == 0 ? S.A[0] : S.B[0];
    double* outI = CPLX ? (mat == 0 ? S.A[NP - 1] : S.B[NP - 1]) : nullptr;
    int w = TW / 2;
    int bad = block_qr<TW, CPLX>(Y, cp[0], cp[1], w, Sr, Si, outR, outI, qsh);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicExch(&P.qr_locks[slot], 0);
    }
    if (bad) {
      status = ST_QR_RANK;
      break;
    }
  }
  __syncthreads();

  double* Ar = S.A[0];
  double* Ai = S.A[NP - 1];
  double* Br = S.B[0];
  double* Bi = S.B[NP - 1];
  double* Zr = S.Z[0];
  double* Zi = S.Z[NP - 1];

  // ---- Z~ = diag(z0) after the in-block prescale (blocked.py:463-469) -----
  for (int e = tid; e < NP * TW * TW; e += nt) (&S.Z[0][0])[e] = 0.0;
  __syncthreads();
  int pbad = 0;
  if (status == ST_OK) {
    for (int c = warp; c < TW; c += NW) {
      double z = 1.0;
      if (kc.prescale) {
        double br[EPL], bi[EPL], p[EPL];
        load_col<TW, CPLX>(Br, Bi, c, lane, br, bi);
#pragma unroll
        for (int e = 0; e < EPL; ++e) p[e] = nrm_term<CPLX>(br[e], bi[e]);
        double ng2 = lane_tree<EPL>(p);
        if (!(ng2 > 0.0)) {
          pbad = 1;
        } else {
          z = 1.0 / sqrt(ng2);
          if (z != 1.0) {
            double ar[EPL], ai[EPL];
            load_col<TW, CPLX>(Ar, Ai, c, lane, ar, ai);
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
              ar[e] *= z;
              ai[e] *= z;
              br[e] *= z;
              bi[e] *= z;
            }
            store_col<TW, CPLX>(Ar, Ai, c, lane, ar, ai);
            store_col<TW, CPLX>(Br, Bi, c, lane, br, bi);
          }
        }
      }
      if (lane == 0) Zr[c * TW + c] = z;
    }
  }
  if (__syncthreads_or(pbad) && status == ST_OK) status = ST_RANK;

  // ---- pointwise sweeps (pointwise.py:222-251) ---------------------------
  // Three phases per inner step, so the scalar 2x2 math runs once per pivot
  // instead of once per lane of 32:
  //   A) warp p forms pivot p's six (eight, complex) column dot products by
  //      a butterfly tree and parks them in shared memory;
  //   B) warp 0, lane p, runs _k_process_pivot's scalar logic for pivot p
  //      (gate, transform, big/sort decisions) and parks Z-hat entries;
  //   C) warp p applies the 2x2 transform / swap to its columns.
  int total = 0, big = 0, sweeps = 0;
  if (status == ST_OK) {
    const bool prof = P.io.phase != nullptr && blockIdx.x == 0 && tid == 0;
    long long tA = 0, tB = 0, tC = 0, nstep = 0, c0 = 0, c1 = 0;
    for (int sw = 0; sw < kc.max_inner_sweeps; ++sw) {
      int lane_applied = 0, lane_big = 0;  // warp 0, lane p: pivot p's counts this sweep
      for (int st = 0; st < P.isteps; ++st) {
        if (prof) c0 = clock64();
        // ---- phase A (pivot pv = warp + k * NW, k < PPW)
        int ii[PPW], jj[PPW];
        double fi[PPW][EPL], fii[PPW][EPL], fj[PPW][EPL], fji[PPW][EPL];
        double gi[PPW][EPL], gii[PPW][EPL], gj[PPW][EPL], gji[PPW][EPL];
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          const int pv = warp + k * NW;
          ii[k] = S.tab[(st * NPIV + pv) * 2];
          jj[k] = S.tab[(st * NPIV + pv) * 2 + 1];
          load_col<TW, CPLX>(Ar, Ai, ii[k], lane, fi[k], fii[k]);
          load_col<TW, CPLX>(Ar, Ai, jj[k], lane, fj[k], fji[k]);
          load_col<TW, CPLX>(Br, Bi, ii[k], lane, gi[k], gii[k]);
          load_col<TW, CPLX>(Br, Bi, jj[k], lane, gj[k], gji[k]);
        }
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          const int pv = warp + k * NW;
          double p[8][EPL];
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            p[0][e] = nrm_term<CPLX>(fi[k][e], fii[k][e]);
            p[1][e] = nrm_term<CPLX>(fj[k][e], fji[k][e]);
            p[3][e] = nrm_term<CPLX>(gi[k][e], gii[k][e]);
            p[4][e] = nrm_term<CPLX>(gj[k][e], gji[k][e]);
            if (CPLX) {
              p[2][e] = dot_re_term(fi[k][e], fii[k][e], fj[k][e], fji[k][e]);
              p[6][e] = dot_im_term(fi[k][e], fii[k][e], fj[k][e], fji[k][e]);
              p[5][e] = dot_re_term(gi[k][e], gii[k][e], gj[k][e], gji[k][e]);
              p[7][e] = dot_im_term(gi[k][e], gii[k][e], gj[k][e], gji[k][e]);
            } else {
              p[2][e] = fi[k][e] * fj[k][e];
              p[5][e] = gi[k][e] * gj[k][e];
              p[6][e] = 0.0;
              p[7][e] = 0.0;
            }
          }
          // Recursive-halving butterfly over the 8 quantities: at xor
          // distance 1, 2, 4 each lane keeps half of the partial sums and
          // ships the other half, then xor 8, 16 finish one value per lane.
          // Every partial is still the sum of two aligned neighbour blocks,
          // so each total is bitwise the reference's pairwise tree.
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = EPL == 2 ? p[q][0] + p[q][EPL - 1] : p[q][0];
          const bool b0 = lane & 1, b1 = (lane >> 1) & 1, b2 = (lane >> 2) & 1;
          double s4[4], s2[2];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double keep = b0 ? v[q + 4] : v[q], send = b0 ? v[q] : v[q + 4];
            s4[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double keep = b1 ? s4[q + 2] : s4[q], send = b1 ? s4[q] : s4[q + 2];
            s2[q] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          }
          double s1 = (b2 ? s2[1] : s2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? s2[0] : s2[1], 4);
          s1 = s1 + __shfl_xor_sync(0xffffffffu, s1, 8);
          s1 = s1 + __shfl_xor_sync(0xffffffffu, s1, 16);
          if (lane < 8) S.pd[pv][4 * b0 + 2 * b1 + b2] = s1;
        }
        __syncthreads();
        if (prof) {
          c1 = clock64();
          tA += c1 - c0;
          c0 = c1;
        }
        // ---- phase B: _k_process_pivot's scalar part (pointwise.py:165-207)
        if (warp == 0) {
          int flags = 0;  // 1 applied, 2 big, 4 swap, 8 bad
          if (lane < NPIV) {
            const double* q = S.pd[lane];
            double z[6];
            FastMath fm;
            flags = pivot_scalar<CPLX>(fm, kc, q, z);
            if (!fm.ok) {  // an operand left the fast paths' range: redo with IEEE operators
              IeeeMath im;
              flags = pivot_scalar<CPLX>(im, kc, q, z);
            }
            if (flags & 1) {
#pragma unroll
              for (int c = 0; c < 6; ++c) S.px[lane][c] = z[c];
              lane_applied += 1;
              lane_big += (flags >> 1) & 1;
            }
            S.pflag[lane] = flags;
          }
          int anybad = __any_sync(0xffffffffu, flags & 8);
          if (lane == 0) S.stepbad = anybad;
          if (st == P.isteps - 1) {
            int sa = lane_applied, sb = lane_big;
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
              sa += __shfl_xor_sync(0xffffffffu, sa, d);
              sb += __shfl_xor_sync(0xffffffffu, sb, d);
            }
            if (lane == 0) {
              S.sw_applied = sa;
              S.sw_big = sb;
            }
          }
        }
        __syncthreads();
        if (prof) {
          c1 = clock64();
          tB += c1 - c0;
          c0 = c1;
        }
        if (S.stepbad) {
          status = ST_RANK;
          break;
        }
        // ---- phase C: _k_update_cols / swaps (pointwise.py:178-218)
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          const int pv = warp + k * NW;
          const int i = ii[k], j = jj[k];
          const int flags = S.pflag[pv];
          bool swap = (flags & 4) != 0;
          double zi_[EPL], zii[EPL], zj_[EPL], zji[EPL];
          if (flags & 5) {
            load_col<TW, CPLX>(Zr, Zi, i, lane, zi_, zii);
            load_col<TW, CPLX>(Zr, Zi, j, lane, zj_, zji);
          }
          if (flags & 1) {
            const double z11 = S.px[pv][0], z12r = S.px[pv][1], z12i = S.px[pv][2];
            const double z21r = S.px[pv][3], z21i = S.px[pv][4], z22 = S.px[pv][5];
#define HZG_UPD(yr, yi, yjr_, yji_)                                                         \
  {                                                                                        \
    double yir = yr[e], yjr = yjr_[e];                                                     \
    if (CPLX) {                                                                            \
      double yii = yi[e], yjI = yji_[e];                                                   \
      double nir = fma(yjr, z21r, fma(-yjI, z21i, yir * z11));                             \
      double nii = fma(yjr, z21i, fma(yjI, z21r, yii * z11));                              \
      double njr = fma(yir, z12r, fma(-yii, z12i, yjr * z22));                             \
      double nji = fma(yir, z12i, fma(yii, z12r, yjI * z22));                              \
      yr[e] = nir; yi[e] = nii; yjr_[e] = njr; yji_[e] = nji;                              \
    } else {                                                                               \
      double ni = fma(yjr, z21r, yir * z11);                                               \
      double nj = fma(yir, z12r, yjr * z22);                                               \
      yr[e] = ni; yjr_[e] = nj;                                                            \
    }                                                                                      \
  }
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
              HZG_UPD(fi[k], fii[k], fj[k], fji[k]);
              HZG_UPD(gi[k], gii[k], gj[k], gji[k]);
              HZG_UPD(zi_, zii, zj_, zji);
            }
#undef HZG_UPD
            if (kc.sorting && CPLX) {
              double q0[EPL], q1[EPL];
#pragma unroll
              for (int e = 0; e < EPL; ++e) {
                q0[e] = nrm_term<CPLX>(fi[k][e], fii[k][e]);
                q1[e] = nrm_term<CPLX>(fj[k][e], fji[k][e]);
              }
              double ni = lane_tree<EPL>(q0), nj = lane_tree<EPL>(q1);
              swap = ni < nj;
            }
          }
          if (flags & 1 || swap) {
            const int di = swap ? j : i, dj = swap ? i : j;
            store_col<TW, CPLX>(Ar, Ai, di, lane, fi[k], fii[k]);
            store_col<TW, CPLX>(Ar, Ai, dj, lane, fj[k], fji[k]);
            store_col<TW, CPLX>(Br, Bi, di, lane, gi[k], gii[k]);
            store_col<TW, CPLX>(Br, Bi, dj, lane, gj[k], gji[k]);
            store_col<TW, CPLX>(Zr, Zi, di, lane, zi_, zii);
            store_col<TW, CPLX>(Zr, Zi, dj, lane, zj_, zji);
          }
        }
        __syncthreads();
        if (prof) {
          tC += clock64() - c0;
          ++nstep;
        }
      }
      if (status != ST_OK) break;
      const int s_cnt = S.sw_applied, b_cnt = S.sw_big;
      sweeps += 1;
      if (s_cnt == 0) break;
      total += s_cnt;
      big += b_cnt;
    }
    if (prof) {
      P.io.phase[0] += tA;
      P.io.phase[1] += tB;
      P.io.phase[2] += tC;
      P.io.phase[3] += nstep;
    }
  }

  // ---- theta rescale (pointwise.py:277-293) ------------------------------
  int tbad = 0;
  if (status == ST_OK) {
    for (int c = warp; c < TW; c += NW) {
      double ar[EPL], ai[EPL], br[EPL], bi[EPL], p[EPL], q[EPL];
      load_col<TW, CPLX>(Ar, Ai, c, lane, ar, ai);
      load_col<TW, CPLX>(Br, Bi, c, lane, br, bi);
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        p[e] = nrm_term<CPLX>(ar[e], ai[e]);
        q[e] = nrm_term<CPLX>(br[e], bi[e]);
      }
      double s = lane_tree<EPL>(p) + lane_tree<EPL>(q);
      if (!(s > 0.0)) {
        tbad = 1;
      } else {
        double th = 1.0 / sqrt(s);
        if (th != 1.0) {
          double zr[EPL], zi2[EPL];
          load_col<TW, CPLX>(Zr, Zi, c, lane, zr, zi2);
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            zr[e] *= th;
            zi2[e] *= th;
          }
          store_col<TW, CPLX>(Zr, Zi, c, lane, zr, zi2);
        }
      }
    }
  }
  if (__syncthreads_or(tbad) && status == ST_OK) status = ST_RANK;

  // ---- exact-identity test (blocked.py:298-308) and outputs ---------------
  int nonid = 0;
  for (int e = tid; e < TW * TW; e += nt) {
    double want = (e % TW) == (e / TW) ? 1.0 : 0.0;
    if (Zr[e] != want) nonid = 1;
    if (CPLX && Zi[e] != 0.0) nonid = 1;
  }
  nonid = __syncthreads_or(nonid);
  double* zt = P.io.zt + (int64_t)pair * NP * TW * TW;
  for (int e = tid; e < NP * TW * TW; e += nt) zt[e] = (&S.Z[0][0])[e];
  if (tid == 0) {
    P.io.ident[pair] = (nonid == 0 || status != ST_OK) ? 1 : 0;
    int32_t* cnt = P.io.counts + ((int64_t)P.step * P.sp.npairs + pair) * 4;
    cnt[0] = total;
    cnt[1] = big;
    cnt[2] = status;
    cnt[3] = sweeps;
  }
}

template <int TW, bool CPLX>
int launch_inner_t(const InnerParams& p, cudaStream_t s) {
  // pivots per warp in the dot / update phases (HZG_PPW overrides, for tuning)
  constexpr int kPPW = 1;  // measured best at w = 16 (profiles/r01_notes.md)
  static int ppw = -1;
  if (ppw < 0) {
    ppw = kPPW;
    if (const char* e = std::getenv("HZG_PPW")) ppw = std::atoi(e);
    if (ppw != 1 && ppw != 2 && ppw != 4) ppw = kPPW;
    if (TW / 2 < ppw) ppw = 1;
  }
  size_t smem = sizeof(InnerSmem<TW, CPLX>);
  auto launch = [&](auto kern, int ppw_) {
    static bool attr_done = false;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (void)attr_done;
    kern<<<p.sp.pn, TW / 2 / ppw_ * 32, smem, s>>>(p);
  };
  if (ppw == 4 && TW / 2 >= 4)
    launch(k_inner<TW, CPLX, (TW / 2 >= 4 ? 4 : 1)>, TW / 2 >= 4 ? 4 : 1);
  else if (ppw == 2 && TW / 2 >= 2)
    launch(k_inner<TW, CPLX, (TW / 2 >= 2 ? 2 : 1)>, TW / 2 >= 2 ? 2 : 1);
  else
    launch(k_inner<TW, CPLX, 1>, 1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

int launch_inner(const Plane& F, const Plane& G, const StepPairs& sp, int step, const KernelCfg& kc,
                 const GramWS& gw, const int32_t* itable, int isteps, const InnerOut& io, double* qr_scratch,
                 int qr_slots, int32_t* qr_locks, cudaStream_t s) {
  InnerParams p{F, G, sp, step, kc, gw, itable, isteps, io, qr_scratch, qr_slots, qr_locks};
#define HZG_CASE(T)                                                                \
  case T:                                                                          \
    return kc.cplx ? launch_inner_t<T, true>(p, s) : launch_inner_t<T, false>(p, s);
  switch (kc.tw) {
    HZG_CASE(2)
    HZG_CASE(4)
    HZG_CASE(6)
    HZG_CASE(8)
    HZG_CASE(10)
    HZG_CASE(12)
    HZG_CASE(14)
    HZG_CASE(16)
    HZG_CASE(20)
    HZG_CASE(24)
    HZG_CASE(32)
    HZG_CASE(48)
    HZG_CASE(64)
    default:
      return 4;
  }
#undef HZG_CASE
}

}  // namespace hzg
