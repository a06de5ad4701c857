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

// Work split of the pointwise sweeps: NW warps, each owning PPW pivots of
// every inner step (dot products, the 2x2 math in lanes 0..PPW-1, and the
// column updates), so the only CTA-wide barrier of an inner step is the one
// that hands the updated columns to the next step's pivots.
template <int TW, bool CPLX, int PPWM = 0>
struct InnerGeo {
  static constexpr int NPIV = TW / 2;                    // pivots per inner step
  static constexpr int PPWMAX = PPWM > 0 ? PPWM : ((CPLX && TW > 32) ? 2 : 4);
  static constexpr int NW = (NPIV + PPWMAX - 1) / PPWMAX;
  static constexpr int PPW = (NPIV + NW - 1) / NW;
  static constexpr int Q = 8 * PPW;                      // reduced quantities per warp
  static constexpr int QP = Q <= 8 ? 8 : (Q <= 16 ? 16 : 32);
  static constexpr int LQ = QP == 8 ? 3 : (QP == 16 ? 4 : 5);
};

template <int TW, bool CPLX, int PPWM = 0>
struct InnerSmem {
  using Geo = InnerGeo<TW, CPLX, PPWM>;
  static constexpr int NP = CPLX ? 2 : 1;
  double A[NP][TW * TW];  // F-hat, column-major (element (r, c) at c*TW + r)
  double B[NP][TW * TW];  // G-hat
  double Z[NP][TW * TW];  // Z-hat
  uint8_t tab[TW * TW];   // inner table, (steps, TW/2, 2)
  double wz[Geo::NW][Geo::PPW][6];  // 2x2 math -> column updates (per warp): z11 z12r z12i z21r z21i z22
  int wf[Geo::NW][Geo::PPW];        // pivot flags: 1 applied, 2 big, 4 swap, 8 bad
  int wcnt[Geo::NW][2];             // per-warp sweep counters (applied, big)
  int chol_fail[2];
};

// Pairwise tree over NS (a power of two) strided values: the split
// partials of one Grammian entry, folded in the reference's tree shape.
template <int NS>
__device__ __forceinline__ double split_tree(const double* p, int64_t stride) {
  if constexpr (NS == 1) {
    return p[0];
  } else {
    return split_tree<NS / 2>(p, stride) + split_tree<NS / 2>(p + (NS / 2) * stride, stride);
  }
}

__device__ __forceinline__ double fold_splits(const double* p, int64_t stride, int ns) {
  switch (ns) {
    case 1: return split_tree<1>(p, stride);
    case 2: return split_tree<2>(p, stride);
    case 4: return split_tree<4>(p, stride);
    case 8: return split_tree<8>(p, stride);
    case 16: return split_tree<16>(p, stride);
    case 32: return split_tree<32>(p, stride);
    default: {
      PairwiseAcc<16> acc;
      acc.reset();
      for (int q = 0; q < ns; ++q) acc.push(p[(int64_t)q * stride]);
      return acc.result();
    }
  }
}

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

// Recursive-halving butterfly over CUR quantities per lane: at xor distance
// 2^J every lane keeps half of its partial sums (chosen by lane bit J) and
// adds the partner's partials of the same half, until one value per lane
// is left; remaining levels are plain butterflies.  Every partial stays the
// sum of two aligned neighbour blocks, so each total is bitwise the
// reference's pairwise tree (dotprod.py:79-91).  Quantity q ends in every
// lane whose low LQ bits are q's bits reversed.
template <int CUR, int J>
struct HalvingTree {
  static __device__ __forceinline__ void run(double* v, int lane) {
    if constexpr (J < 5) {
      if constexpr (CUR > 1) {
        constexpr int H = CUR / 2;
        const bool b = (lane >> J) & 1;
#pragma unroll
        for (int q = 0; q < H; ++q) {
          const double keep = b ? v[q + H] : v[q];
          const double send = b ? v[q] : v[q + H];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << J);
        }
        HalvingTree<H, J + 1>::run(v, lane);
      } else {
        v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1 << J);
        HalvingTree<1, J + 1>::run(v, lane);
      }
    }
  }
};

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

template <int TW, bool CPLX, int PPWM>
__global__ void __launch_bounds__(InnerGeo<TW, CPLX, PPWM>::NW * 32) k_inner(InnerParams P) {
  using Geo = InnerGeo<TW, CPLX, PPWM>;
  constexpr int NPIV = Geo::NPIV;
  constexpr int NW = Geo::NW;    // warps
  constexpr int PPW = Geo::PPW;  // pivots per warp and inner step
  constexpr int EPL = Lanes<TW>::EPL;
  constexpr int NP = CPLX ? 2 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<InnerSmem<TW, CPLX, PPWM>*>(smem_raw);
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
        const double v = fold_splits(base + (int64_t)pl * TW * TW + e, (int64_t)NP * TW * TW, ns);
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
  // Per inner step, warp w owns pivots w*PPW .. w*PPW+PPW-1:
  //   A) forms their six (eight, complex) column dot products with one
  //      recursive-halving tree and gathers pivot k's sums into lane k;
  //   B) lane k runs _k_process_pivot's scalar logic for pivot k (gate,
  //      transform, big / sort decisions) and parks the Z-hat entries in the
  //      warp's slot of shared memory;
  //   C) the warp applies the transforms / swaps to its pivots' columns.
  // Pivots of a step touch disjoint columns, so the only CTA barrier is the
  // one before the next step reads columns other warps wrote.
  int total = 0, big = 0, sweeps = 0;
  if (status == ST_OK) {
    const bool prof = P.io.phase != nullptr && blockIdx.x == 0 && tid == 0;
    long long tA = 0, tB = 0, tC = 0, nstep = 0, c0 = 0, c1 = 0;
    for (int sw = 0; sw < kc.max_inner_sweeps; ++sw) {
      int lane_applied = 0, lane_big = 0;  // lane k: pivot k's counts this sweep
      // pivot indices of the warp's pivots, fetched one inner step ahead
      auto fetch = [&](int st, int (&a)[PPW], int (&b)[PPW]) {
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          const int pv = warp * PPW + k;
          const bool ok = NPIV % PPW == 0 || pv < NPIV;
          a[k] = ok ? S.tab[(st * NPIV + pv) * 2] : 0;
          b[k] = ok ? S.tab[(st * NPIV + pv) * 2 + 1] : 0;
        }
      };
      int nii[PPW], njj[PPW];
      fetch(0, nii, njj);
      for (int st = 0; st < P.isteps; ++st) {
        if (prof) c0 = clock64();
        // ---- phase A
        int ii[PPW], jj[PPW];
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          ii[k] = nii[k];
          jj[k] = njj[k];
        }
        fetch(st + 1 < P.isteps ? st + 1 : 0, nii, njj);
        double fi[PPW][EPL], fii[PPW][EPL], fj[PPW][EPL], fji[PPW][EPL];
        double gi[PPW][EPL], gii[PPW][EPL], gj[PPW][EPL], gji[PPW][EPL];
        double v[Geo::QP];
#pragma unroll
        for (int q = Geo::Q; q < Geo::QP; ++q) v[q] = 0.0;
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          load_col<TW, CPLX>(Ar, Ai, ii[k], lane, fi[k], fii[k]);
          load_col<TW, CPLX>(Ar, Ai, jj[k], lane, fj[k], fji[k]);
          load_col<TW, CPLX>(Br, Bi, ii[k], lane, gi[k], gii[k]);
          load_col<TW, CPLX>(Br, Bi, jj[k], lane, gj[k], gji[k]);
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
#pragma unroll
          for (int c = 0; c < 8; ++c) v[k * 8 + c] = EPL == 2 ? p[c][0] + p[c][EPL - 1] : p[c][0];
        }
        HalvingTree<Geo::QP, 0>::run(v, lane);
        // lane k < PPW collects pivot k's eight sums
        double qv[8];
        {
          const int kk = lane < PPW ? lane : 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int src = (int)(__brev((unsigned)(kk * 8 + c)) >> (32 - Geo::LQ));
            qv[c] = __shfl_sync(0xffffffffu, v[0], src);
          }
        }
        if (prof) {
          c1 = clock64();
          tA += c1 - c0;
          c0 = c1;
        }
        // ---- phase B: _k_process_pivot's scalar part (pointwise.py:165-207)
        int bad = 0;
        if (lane < PPW && (NPIV % PPW == 0 || warp * PPW + lane < NPIV)) {
          double z[6];
          FastMath fm;
          int flags = pivot_scalar<CPLX>(fm, kc, qv, z);
          if (!fm.ok) {  // an operand left the fast paths' range: redo with IEEE operators
            IeeeMath im;
            flags = pivot_scalar<CPLX>(im, kc, qv, z);
          }
          if (flags & 1) {
#pragma unroll
            for (int c = 0; c < 6; ++c) S.wz[warp][lane][c] = z[c];
            lane_applied += 1;
            lane_big += (flags >> 1) & 1;
          }
          S.wf[warp][lane] = flags;
          bad = flags & 8;
        } else if (lane < PPW) {
          S.wf[warp][lane] = 0;
        }
        if (st == P.isteps - 1) {
          int sa = lane_applied, sb = lane_big;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            sa += __shfl_xor_sync(0xffffffffu, sa, d);
            sb += __shfl_xor_sync(0xffffffffu, sb, d);
          }
          if (lane == 0) {
            S.wcnt[warp][0] = sa;
            S.wcnt[warp][1] = sb;
          }
        }
        __syncwarp();
        if (prof) {
          c1 = clock64();
          tB += c1 - c0;
          c0 = c1;
        }
        // ---- phase C: _k_update_cols / swaps (pointwise.py:178-218)
        // every shared-memory operand of the warp's pivots is loaded up
        // front (one latency instead of one per pivot)
        int fl[PPW];
        double zz[PPW][6];
        double zi_[PPW][EPL], zii[PPW][EPL], zj_[PPW][EPL], zji[PPW][EPL];
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          fl[k] = S.wf[warp][k];
#pragma unroll
          for (int c = 0; c < 6; ++c) zz[k][c] = S.wz[warp][k][c];
          load_col<TW, CPLX>(Zr, Zi, ii[k], lane, zi_[k], zii[k]);
          load_col<TW, CPLX>(Zr, Zi, jj[k], lane, zj_[k], zji[k]);
        }
#pragma unroll
        for (int k = 0; k < PPW; ++k) {
          const int i = ii[k], j = jj[k];
          const int flags = fl[k];
          bool swap = (flags & 4) != 0;
          if (flags & 1) {
            const double z11 = zz[k][0], z12r = zz[k][1], z12i = zz[k][2];
            const double z21r = zz[k][3], z21i = zz[k][4], z22 = zz[k][5];
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
              HZG_UPD(zi_[k], zii[k], zj_[k], zji[k]);
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
            store_col<TW, CPLX>(Zr, Zi, di, lane, zi_[k], zii[k]);
            store_col<TW, CPLX>(Zr, Zi, dj, lane, zj_[k], zji[k]);
          }
        }
        // a rank-deficient pivot anywhere ends the solve (RankError upstream)
        const int anybad = __syncthreads_or(bad);
        if (prof) {
          tC += clock64() - c0;
          ++nstep;
        }
        if (anybad) {
          status = ST_RANK;
          break;
        }
      }
      if (status != ST_OK) break;
      int s_cnt = 0, b_cnt = 0;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        s_cnt += S.wcnt[q][0];
        b_cnt += S.wcnt[q][1];
      }
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

template <int TW, bool CPLX, int PPWM>
int launch_inner_g(const InnerParams& p, cudaStream_t s) {
  const size_t smem = sizeof(InnerSmem<TW, CPLX, PPWM>);
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(k_inner<TW, CPLX, PPWM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  k_inner<TW, CPLX, PPWM><<<p.sp.pn, InnerGeo<TW, CPLX, PPWM>::NW * 32, smem, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int TW, bool CPLX>
int launch_inner_t(const InnerParams& p, cudaStream_t s) {
  if constexpr (TW == 32 && !CPLX) {
    // pivots per warp (HZG_PPW=2 selects 8 warps x 2 pivots; for tuning)
    static int ppw = -1;
    if (ppw < 0) {
      const char* e = std::getenv("HZG_PPW");
      ppw = e ? std::atoi(e) : 4;
    }
    if (ppw == 2) return launch_inner_g<TW, CPLX, 2>(p, s);
  }
  return launch_inner_g<TW, CPLX, 0>(p, s);
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
