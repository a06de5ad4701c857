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
#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "hzg_device.cuh"
#include "hzg_internal.h"

namespace hzg {

namespace {

constexpr int kMaxTW = 64;

// Work split of the pointwise sweeps.  Each pivot of an inner step is
// owned by a group of LP lanes of one warp; lane l of the group holds rows
// l*RPL .. l*RPL+RPL-1 of the pivot's columns (RPL = 4 rows, i.e. the first
// two levels of the reference's pairwise tree happen in registers), so a
// dot product needs only log2(LP) shuffle levels and a warp serves PG = 32 /
// LP pivots at once.  Sub-lane 0 of each group runs the 2x2 math.  The only
// CTA-wide barrier of an inner step hands the updated columns to the next
// step's pivots.
template <int TW, bool CPLX>
struct InnerGeo {
  static constexpr int NPIV = TW / 2;  // pivots per inner step
  static constexpr int LT = TW <= 2 ? 2 : (TW <= 4 ? 4 : (TW <= 8 ? 8 : (TW <= 16 ? 16 : (TW <= 32 ? 32 : 64))));
  static constexpr int RPL = (TW == 64 && !CPLX) ? 8 : (LT >= 4 ? 4 : LT);  // rows per lane
  static constexpr int LP = LT / RPL;           // lanes per pivot
  static constexpr int LV = LP == 1 ? 0 : (LP == 2 ? 1 : (LP == 4 ? 2 : (LP == 8 ? 3 : 4)));
  static constexpr int PG = 32 / LP;            // pivots per warp
  static constexpr int NW = (NPIV + PG - 1) / PG;
  static constexpr int HL = LV < 3 ? LV : 3;    // halving levels over the 8 quantities
  static constexpr int R = 8 >> HL;             // quantities per lane after halving
  static constexpr bool VEC = TW % 4 == 0 && RPL >= 4 && TW % RPL == 0;  // 16-byte shared loads / stores
  static constexpr int NCB = NPIV > NW ? NPIV : NW;     // compensated-variant scratch slots
};

template <int TW, bool CPLX>
struct InnerSmem {
  using Geo = InnerGeo<TW, CPLX>;
  static constexpr int NP = CPLX ? 2 : 1;
  alignas(16) double A[NP][TW * TW];  // F-hat, column-major (element (r, c) at c*TW + r)
  alignas(16) double B[NP][TW * TW];  // G-hat
  alignas(16) double Z[NP][TW * TW];  // Z-hat
  uint8_t tab[TW * TW];               // inner table, (steps, TW/2, 2)
  int wcnt[Geo::NW][2];               // per-warp sweep counters (applied, big)
  int chol_fail[2];
  double cbuf[Geo::NCB][Geo::LT];     // compensated variants: sequential tree scratch per pivot / warp
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
    case 64: return split_tree<64>(p, stride);
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

// Recursive-halving butterfly over CUR quantities per lane inside aligned
// groups of lanes: at xor distance 2^J every lane keeps half of its partial
// sums (chosen by lane bit J) and adds the partner's partials of the same
// half.  Every partial stays the sum of two aligned neighbour blocks, so
// each total is bitwise the reference's pairwise tree (dotprod.py:79-91).
// After L levels, slot s of lane l holds quantity s + (CUR >> L) * rev_L(l).
template <int CUR, int J, int L>
struct HalvingTree {
  static __device__ __forceinline__ void run(double* v, int lane) {
    if constexpr (J < L) {
      constexpr int H = CUR / 2;
      const bool b = (lane >> J) & 1;
#pragma unroll
      for (int q = 0; q < H; ++q) {
        const double keep = b ? v[q + H] : v[q];
        const double send = b ? v[q] : v[q + H];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << J);
      }
      HalvingTree<H, J + 1, L>::run(v, lane);
    }
  }
};

// Shared-memory row order of the 2w x 2w factors.  With a swizzle period
// SW (= the rows per lane of the pointwise loop, 4 or 8), the rows of every
// column are stored as [rows SW*l, SW*l+1 for l = 0..][rows SW*l+2,
// SW*l+3 ..]..., so the 16-byte loads of the lanes that share a column
// (each holding the aligned block of rows SW*l .. SW*l+SW-1) cover 128
// contiguous bytes per instruction -- conflict-free -- while each lane still
// owns an aligned block of the reference tree.  SW = 0: natural order.
template <int SW, int TW>
__device__ __forceinline__ int rp(int r) {
  if constexpr (SW > 0) {
    return ((r % SW) >> 1) * (2 * TW / SW) + ((r / SW) << 1) + (r & 1);
  } else {
    return r;
  }
}

template <int SW, int TW>
__device__ __forceinline__ int rp_inv(int q) {
  if constexpr (SW > 0) {
    const int e = q / (2 * TW / SW), rem = q % (2 * TW / SW);
    return (rem >> 1) * SW + 2 * e + (rem & 1);
  } else {
    return q;
  }
}

// Rows r0 .. r0+RPL-1 of column `col` of a TW x TW column-major matrix
// (zeros beyond TW, like the reference's tree padding).
template <int TW, bool VEC, int RPL, int SW = 0>
__device__ __forceinline__ void load_rows(const double* m, int col, int r0, double (&x)[RPL]) {
  if constexpr (VEC) {
    if (r0 < TW) {
      // row pairs r0+2e, r0+2e+1 (adjacent, or 2 TW / SW apart when swizzled)
      const double* b = m + col * TW + (SW ? 2 * (r0 / RPL) : r0);
#pragma unroll
      for (int e = 0; e < RPL / 2; ++e) {
        const double2 d = *reinterpret_cast<const double2*>(b + e * (SW ? 2 * TW / SW : 2));
        x[2 * e] = d.x;
        x[2 * e + 1] = d.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < RPL; ++e) x[e] = 0.0;
    }
  } else {
#pragma unroll
    for (int e = 0; e < RPL; ++e) x[e] = r0 + e < TW ? m[col * TW + r0 + e] : 0.0;
  }
}

template <int TW, bool VEC, int RPL, int SW = 0>
__device__ __forceinline__ void store_rows(double* m, int col, int r0, const double (&x)[RPL]) {
  if constexpr (VEC) {
    if (r0 < TW) {
      double* b = m + col * TW + (SW ? 2 * (r0 / RPL) : r0);
#pragma unroll
      for (int e = 0; e < RPL / 2; ++e)
        *reinterpret_cast<double2*>(b + e * (SW ? 2 * TW / SW : 2)) = make_double2(x[2 * e], x[2 * e + 1]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < RPL; ++e)
      if (r0 + e < TW) m[col * TW + r0 + e] = x[e];
  }
}

// pairwise tree over the RPL rows held by one lane (levels 1 .. log2 RPL of
// the reference tree)
template <int RPL>
__device__ __forceinline__ double row_tree(const double (&x)[RPL]) {
  if constexpr (RPL == 1) {
    return x[0];
  } else if constexpr (RPL == 2) {
    return x[0] + x[1];
  } else if constexpr (RPL == 4) {
    return (x[0] + x[1]) + (x[2] + x[3]);
  } else {
    return ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7]));
  }
}

template <int TW, bool CPLX, int SW = 0>
__device__ __forceinline__ void load_col(const double* __restrict__ re, const double* __restrict__ im, int col,
                                         int lane, double (&r)[Lanes<TW>::EPL], double (&i)[Lanes<TW>::EPL]) {
  constexpr int EPL = Lanes<TW>::EPL;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    int row = lane * EPL + e;
    bool ok = row < TW;
    const int q = ok ? rp<SW, TW>(row) : 0;
    r[e] = ok ? re[col * TW + q] : 0.0;
    i[e] = (CPLX && ok) ? im[col * TW + q] : 0.0;
  }
}

template <int TW, bool CPLX, int SW = 0>
__device__ __forceinline__ void store_col(double* re, double* im, int col, int lane,
                                          const double (&r)[Lanes<TW>::EPL], const double (&i)[Lanes<TW>::EPL]) {
  constexpr int EPL = Lanes<TW>::EPL;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    int row = lane * EPL + e;
    if (row < TW) {
      const int q = rp<SW, TW>(row);
      re[col * TW + q] = r[e];
      if (CPLX) im[col * TW + q] = i[e];
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
template <int TW, bool CPLX, int SW>
__device__ int warp_cholesky(double* Ar, double* Ai, int lane) {
#define A_(x, y) Ar[(y) * TW + rp<SW, TW>(x)]
#define AI_(x, y) Ai[(y) * TW + rp<SW, TW>(x)]
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

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// warp_cholesky by NTH threads (a named barrier `bar` of its own, so the F
// and G factorizations run side by side): the same operations in the same
// per-element order -- element (x, jp) of the trailing triangle is updated
// by the columns j < jp in ascending order -- so the factor is bitwise
// warp_cholesky's.  Thread (tx, ty) owns rows x = tx (mod TX) and the
// columns jp = ty (mod TY) of them; each column step is scale | barrier |
// update | barrier, the update in chunks of four independent elements
// (loads before stores: no shared-memory aliasing stalls).
template <int TW, bool CPLX, int SW, int NTH>
__device__ int group_cholesky(double* Ar, double* Ai, int t, int bar) {
#define A_(x, y) Ar[(y) * TW + rp<SW, TW>(x)]
#define AI_(x, y) Ai[(y) * TW + rp<SW, TW>(x)]
  constexpr int TX = TW < NTH ? TW : NTH;
  constexpr int TY = NTH / TX;
  static_assert(NTH % TX == 0, "thread grid");
  const int tx = t % TX, ty = t / TX;
  for (int j = 0; j < TW; ++j) {
    const double d = A_(j, j);
    if (!(d > 0.0) || !isfinite(d)) return 1;  // every thread read the same d
    const double rt = sqrt(d);
    const double rinv = 1.0 / rt;
    if (ty == 0)
      for (int x = tx; x < TW; x += TX)
        if (x > j) {
          A_(x, j) *= rinv;
          if (CPLX) AI_(x, j) *= rinv;
        }
    named_bar(bar, NTH);
    for (int x = tx; x < TW; x += TX) {
      if (x < j) continue;
      if (x == j) {  // nobody reads the diagonal during the update
        if (ty == 0) {
          A_(j, j) = rt;
          if (CPLX) AI_(j, j) = 0.0;
        }
        continue;
      }
      const double ar = -A_(x, j);
      const double ai = CPLX ? -AI_(x, j) : 0.0;
      int jp = j + 1 + (((ty - (j + 1)) % TY) + TY) % TY;
      for (; jp + 3 * TY <= x; jp += 4 * TY) {
        double br[4], bi[4], cr[4], ci[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          br[q] = A_(jp + q * TY, j);
          bi[q] = CPLX ? -AI_(jp + q * TY, j) : 0.0;
          cr[q] = A_(x, jp + q * TY);
          ci[q] = CPLX ? AI_(x, jp + q * TY) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (CPLX) {
            A_(x, jp + q * TY) = fma(ar, br[q], fma(-ai, bi[q], cr[q]));
            AI_(x, jp + q * TY) = fma(ar, bi[q], fma(ai, br[q], ci[q]));
          } else {
            A_(x, jp + q * TY) = fma(ar, br[q], cr[q]);
          }
        }
      }
      for (; jp <= x; jp += TY) {
        const double br = A_(jp, j);
        if (CPLX) {
          const double bi = -AI_(jp, j);
          A_(x, jp) = fma(ar, br, fma(-ai, bi, A_(x, jp)));
          AI_(x, jp) = fma(ar, bi, fma(ai, br, AI_(x, jp)));
        } else {
          A_(x, jp) = fma(ar, br, A_(x, jp));
        }
      }
    }
    named_bar(bar, NTH);
  }
  // conj-transpose into the upper triangle, zero the strict lower one
  for (int r = t; r < TW; r += NTH)
    for (int c = 0; c < r; ++c) {
      A_(c, r) = A_(r, c);
      if (CPLX) AI_(c, r) = -AI_(r, c);
      A_(r, c) = 0.0;
      if (CPLX) AI_(r, c) = 0.0;
    }
  return 0;
#undef A_
#undef AI_
}

// Householder R factor of the m x TW block-column stack (blocked.py:97-217
// with pivot=False, via _shorten_qr :487-500), bitwise in the reference's
// sequential fma order.  Sequential chains over m make this slow; it only
// runs for the rare pairs whose Grammian fails Cholesky.
template <int TW, bool CPLX, int SW>
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
    outR[c * TW + rp<SW, TW>(r)] = S_(r, c);
    if (CPLX) outI[c * TW + rp<SW, TW>(r)] = SI_(r, c);
  }
  __syncthreads();
  return bad;
#undef S_
#undef SI_
}

// _k_process_pivot's scalar part (pointwise.py:165-207) for one pivot:
// q = {a11, a22, a12r, b11, b22, b12r, a12i, b12i}.  Returns flags (1 applied,
// 2 big, 4 swap, 8 bad) and, when applied, the rescaled Z-hat entries.
// APPROX: the short-chain 2x2 forms of the DMMA mode (hzg_device.cuh).
template <bool CPLX, bool APPROX = false, class M>
__device__ __forceinline__ int pivot_scalar(M& m, const KernelCfg& kc, const double* q, double (&z)[6]) {
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

template <int TW, bool CPLX, int SW>
__global__ void __launch_bounds__(InnerGeo<TW, CPLX>::NW * 32, (TW <= 32 && !CPLX) ? 4 : ((TW == 64 && !CPLX) ? 2 : 1))
k_inner(InnerParams P) {
  using Geo = InnerGeo<TW, CPLX>;
  constexpr int NPIV = Geo::NPIV;
  constexpr int NW = Geo::NW;  // warps
  constexpr int EPL = Lanes<TW>::EPL;
  constexpr int NP = CPLX ? 2 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<InnerSmem<TW, CPLX>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = blockDim.x;
  const KernelCfg& kc = P.kc;

  // ---- the inner strategy table ------------------------------------------
  for (int e = tid; e < P.isteps * TW; e += nt) S.tab[e] = (uint8_t)P.itable[e];

  // a CTA may serve several pairs of the step (grid capped at launch)
  for (int pair = P.sp.p0 + blockIdx.x; pair < P.sp.p0 + P.sp.pn; pair += gridDim.x) {
  __syncthreads();  // the previous pair is done with shared memory
  if (tid == 0) {
    S.chol_fail[0] = S.chol_fail[1] = 0;
  }

  // ---- fold the Grammian partials (pairwise over splits) -----------------
  // (shorten == "qr": no Grammians; both factors come from the QR below)
  if (kc.shorten_qr && tid == 0) S.chol_fail[0] = S.chol_fail[1] = 1;
  for (int mat = 0; mat < 2 && !kc.shorten_qr; ++mat) {
    const int ns = P.gw.nsplit[mat];
    const double* base = P.gw.part + ((int64_t)pair * 2 + mat) * P.gw.smax * NP * TW * TW;
    double(*M)[TW * TW] = mat == 0 ? S.A : S.B;
    for (int e = tid; e < TW * TW; e += nt) {
      int r = e % TW, c = e / TW;
      if (r > c) continue;
      for (int pl = 0; pl < NP; ++pl) {
        const double v = fold_splits(base + (int64_t)pl * TW * TW + e, (int64_t)NP * TW * TW, ns);
        if (pl == 0) {
          M[0][c * TW + rp<SW, TW>(r)] = v;
          M[0][r * TW + rp<SW, TW>(c)] = v;
        } else {
          M[1][c * TW + rp<SW, TW>(r)] = r == c ? 0.0 : v;
          M[1][r * TW + rp<SW, TW>(c)] = r == c ? 0.0 : -v;
        }
      }
    }
  }
  __syncthreads();

  // ---- Cholesky of both Grammians -----------------------------------------
  // (2+ warps: the first half of the CTA factors F, the second G)
  if constexpr (NW >= 2 && NW % 2 == 0) {
    if (!kc.shorten_qr) {
      constexpr int NTH = NW * 16;
      const int half = tid / NTH;
      double* Mr = half == 0 ? S.A[0] : S.B[0];
      double* Mi = CPLX ? (half == 0 ? S.A[NP - 1] : S.B[NP - 1]) : nullptr;
      const int f = group_cholesky<TW, CPLX, SW, NTH>(Mr, Mi, tid % NTH, 1 + half);
      if (tid % NTH == 0) S.chol_fail[half] = f;
    }
  } else if (warp < 2 && !kc.shorten_qr) {
    double* Mr = warp == 0 ? S.A[0] : S.B[0];
    double* Mi = CPLX ? (warp == 0 ? S.A[NP - 1] : S.B[NP - 1]) : nullptr;
    int f = warp_cholesky<TW, CPLX, SW>(Mr, Mi, lane);
    if (lane == 0) S.chol_fail[warp] = f;
  }
  if (NW == 1 && !kc.shorten_qr) {  // a single warp: factor G after F
    __syncwarp();
    int f = warp_cholesky<TW, CPLX, SW>(S.B[0], CPLX ? S.B[NP - 1] : nullptr, lane);
    if (lane == 0) S.chol_fail[1] = f;
  }
  __syncthreads();

  int status = ST_OK;
  for (int mat = 0; mat < 2; ++mat) {
    if (!S.chol_fail[mat]) continue;
    if (!kc.fallback_qr && !kc.shorten_qr) {
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
    int bad = block_qr<TW, CPLX, SW>(Y, cp[0], cp[1], w, Sr, Si, outR, outI, qsh);
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
        load_col<TW, CPLX, SW>(Br, Bi, c, lane, br, bi);
        double ng2;
        if (kc.compensated) {  // _k_col_norm with comp (pointwise.py:260)
          double v = 0.0;
          if (lane == 0) v = ccol_norm(Br + c * TW, CPLX ? Bi + c * TW : nullptr, TW, S.cbuf[warp]);
          ng2 = __shfl_sync(0xffffffffu, v, 0);
        } else {
#pragma unroll
          for (int e = 0; e < EPL; ++e) p[e] = nrm_term<CPLX>(br[e], bi[e]);
          ng2 = lane_tree<EPL>(p);
        }
        if (!(ng2 > 0.0)) {
          pbad = 1;
        } else {
          z = 1.0 / sqrt(ng2);
          if (z != 1.0) {
            double ar[EPL], ai[EPL];
            load_col<TW, CPLX, SW>(Ar, Ai, c, lane, ar, ai);
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
              ar[e] *= z;
              ai[e] *= z;
              br[e] *= z;
              bi[e] *= z;
            }
            store_col<TW, CPLX, SW>(Ar, Ai, c, lane, ar, ai);
            store_col<TW, CPLX, SW>(Br, Bi, c, lane, br, bi);
          }
        }
      }
      if (lane == 0) Zr[c * TW + rp<SW, TW>(c)] = z;
    }
  }
  if (__syncthreads_or(pbad) && status == ST_OK) status = ST_RANK;

  // ---- pointwise sweeps (pointwise.py:222-251) ---------------------------
  // Per inner step, lane group g of warp w owns pivot w*PG + g:
  //   A) its lanes form the six (eight, complex) column dot products over
  //      their rows and reduce them across the group (pairwise tree);
  //   B) the group's sub-lane 0 runs _k_process_pivot's scalar logic (gate,
  //      transform, big / sort decisions) and broadcasts the Z-hat entries;
  //   C) the group applies the transform / swap to its rows of the columns.
  int total = 0, big = 0, sweeps = 0;
  if (status == ST_OK) {
    constexpr int RPL = Geo::RPL, LP = Geo::LP, PG = Geo::PG, R = Geo::R;
    constexpr bool VEC = Geo::VEC;
    const int grp = lane / LP, sub = lane % LP, base = grp * LP;
    const int r0 = sub * RPL;
    const int pv = warp * PG + grp;
    const bool valid = NPIV % PG == 0 || pv < NPIV;
    const bool mathlane = sub == 0 && valid;
    const bool prof = P.io.phase != nullptr && blockIdx.x == 0 && tid == 0;
    // phase profiling (hzg_debug_phases; thread 0 of CTA 0 only): cycles go
    // straight to global counters, so production runs carry one register
    // pair (c0) for it, not six
    unsigned long long* const ph = prof ? reinterpret_cast<unsigned long long*>(P.io.phase) : nullptr;
    long long c0 = 0;
    for (int sw = 0; sw < kc.max_inner_sweeps; ++sw) {
      int lane_applied = 0, lane_big = 0;  // math lanes: the pivot's counts this sweep
      int ni_ = valid ? S.tab[pv * 2] : 0, nj_ = valid ? S.tab[pv * 2 + 1] : 1;
      for (int st = 0; st < P.isteps; ++st) {
        if (prof) c0 = clock64();
        // ---- phase A
        const int i = ni_, j = nj_;
        if (st + 1 < P.isteps && valid) {  // next step's pivot, fetched ahead
          ni_ = S.tab[((st + 1) * NPIV + pv) * 2];
          nj_ = S.tab[((st + 1) * NPIV + pv) * 2 + 1];
        }
        double fi[RPL], fj[RPL], gi[RPL], gj[RPL];
        double fii[RPL], fji[RPL], gii[RPL], gji[RPL];
        load_rows<TW, VEC, RPL, SW>(Ar, i, r0, fi);
        load_rows<TW, VEC, RPL, SW>(Ar, j, r0, fj);
        load_rows<TW, VEC, RPL, SW>(Br, i, r0, gi);
        load_rows<TW, VEC, RPL, SW>(Br, j, r0, gj);
        if constexpr (CPLX) {
          load_rows<TW, VEC, RPL, SW>(Ai, i, r0, fii);
          load_rows<TW, VEC, RPL, SW>(Ai, j, r0, fji);
          load_rows<TW, VEC, RPL, SW>(Bi, i, r0, gii);
          load_rows<TW, VEC, RPL, SW>(Bi, j, r0, gji);
        } else {
#pragma unroll
          for (int e = 0; e < RPL; ++e) fii[e] = fji[e] = gii[e] = gji[e] = 0.0;
        }
        double qv[8];  // sub-lane 0 of the group: the pivot's eight sums
        if (kc.compensated) {
          // compensated variants: the math lane forms the six (eight) sums
          // with the reference's sequential compensated trees (pointwise.py:165-170)
          if (mathlane) {
            double* cb = S.cbuf[pv];
            qv[0] = ccol_norm(Ar + i * TW, CPLX ? Ai + i * TW : nullptr, TW, cb);
            qv[1] = ccol_norm(Ar + j * TW, CPLX ? Ai + j * TW : nullptr, TW, cb);
            ccol_dot(Ar + i * TW, CPLX ? Ai + i * TW : nullptr, Ar + j * TW, CPLX ? Ai + j * TW : nullptr, TW, cb,
                     qv[2], qv[6]);
            qv[3] = ccol_norm(Br + i * TW, CPLX ? Bi + i * TW : nullptr, TW, cb);
            qv[4] = ccol_norm(Br + j * TW, CPLX ? Bi + j * TW : nullptr, TW, cb);
            ccol_dot(Br + i * TW, CPLX ? Bi + i * TW : nullptr, Br + j * TW, CPLX ? Bi + j * TW : nullptr, TW, cb,
                     qv[5], qv[7]);
          }
        } else {
        double v[8];
        {
          // one quantity at a time: its RPL products, then its row tree
          // (each tree's shape is fixed, so the order across quantities
          // changes no bit, and only RPL products are live at once)
          double p[RPL];
#define HZG_SUM(c, expr)                                                  \
  {                                                                       \
    _Pragma("unroll") for (int e = 0; e < RPL; ++e) p[e] = (expr);        \
    v[c] = row_tree<RPL>(p);                                              \
  }
          HZG_SUM(0, (nrm_term<CPLX>(fi[e], fii[e])));
          HZG_SUM(1, (nrm_term<CPLX>(fj[e], fji[e])));
          HZG_SUM(3, (nrm_term<CPLX>(gi[e], gii[e])));
          HZG_SUM(4, (nrm_term<CPLX>(gj[e], gji[e])));
          if (CPLX) {
            HZG_SUM(2, (dot_re_term(fi[e], fii[e], fj[e], fji[e])));
            HZG_SUM(6, (dot_im_term(fi[e], fii[e], fj[e], fji[e])));
            HZG_SUM(5, (dot_re_term(gi[e], gii[e], gj[e], gji[e])));
            HZG_SUM(7, (dot_im_term(gi[e], gii[e], gj[e], gji[e])));
          } else {
            HZG_SUM(2, (fi[e] * fj[e]));
            HZG_SUM(5, (gi[e] * gj[e]));
            v[6] = 0.0;
            v[7] = 0.0;
          }
#undef HZG_SUM
        }
        HalvingTree<8, 0, Geo::HL>::run(v, lane);
#pragma unroll
        for (int d = 1 << Geo::HL; d < LP; d <<= 1)
#pragma unroll
          for (int s2 = 0; s2 < R; ++s2) v[s2] = v[s2] + __shfl_xor_sync(0xffffffffu, v[s2], d);
        // the group's sub-lane 0 collects the eight sums
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          int holder = 0;  // sub-lane holding quantity c: rev_HL(c / R)
          if constexpr (Geo::HL > 0) holder = (int)(__brev((unsigned)(c / R)) >> (32 - Geo::HL));
          qv[c] = __shfl_sync(0xffffffffu, v[c % R], base + holder);
        }
        }
        if (prof) {
          const long long c1 = clock64();
          atomicAdd(&ph[0], (unsigned long long)(c1 - c0));
          c0 = c1;
        }
        // ---- phase B: _k_process_pivot's scalar part (pointwise.py:165-207)
        int flags = 0;
        double z[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#ifdef HZG_EXP_NOMATH
        if (mathlane) {  // experiment: every pivot applies the identity (no 2x2 math)
          flags = 1;
          z[0] = 1.0;
          z[5] = 1.0;
          lane_applied += 1;
        }
        if (false) {
#else
        // Without compensation every lane of the group already holds the
        // eight sums (the gather above is a broadcast), so all of them run
        // the pivot's 2x2 math -- the same instructions the math lane alone
        // would issue -- and nobody waits for a broadcast of the results.
        const bool redundant = !kc.compensated;
        if (redundant ? valid : mathlane) {
#endif
          bool exact_path = true;
          if (kc.approx_2x2) {
            FastMath fm;
            flags = pivot_scalar<CPLX, true>(fm, kc, qv, z);
            exact_path = !fm.ok;  // out of the short forms' range: the reference-order path
            // diagnostics (hzg_debug_phases): count the fallbacks in units of 1e9 in slot 0
            if (exact_path && P.io.phase && sub == 0)
              atomicAdd((unsigned long long*)&P.io.phase[0], 1000000000ull);
          }
          if (exact_path) {
            FastMath fm;
            flags = pivot_scalar<CPLX>(fm, kc, qv, z);
            if (!fm.ok) {  // an operand left the fast paths' range: redo with IEEE operators
              IeeeMath im;
              flags = pivot_scalar<CPLX>(im, kc, qv, z);
            }
          }
          if ((flags & 1) && sub == 0) {
            lane_applied += 1;
            lane_big += (flags >> 1) & 1;
          }
        }
        const int bad = flags & 8;
#ifndef HZG_EXP_NOMATH
        if (!redundant)
#endif
        {
          flags = __shfl_sync(0xffffffffu, flags, base);
#pragma unroll
          for (int c = 0; c < 6; ++c) z[c] = __shfl_sync(0xffffffffu, z[c], base);
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
        if (prof) {
          const long long c1 = clock64();
          atomicAdd(&ph[1], (unsigned long long)(c1 - c0));
          c0 = c1;
        }
        // ---- phase C: _k_update_cols / swaps (pointwise.py:178-218)
        if constexpr (!CPLX) {
          // real: the swap is decided (flags & 4), so F and G go back to
          // shared memory before Z's rows are loaded -- fewer live registers
          if (flags & 5) {
            const bool swap = (flags & 4) != 0;
            const int di = swap ? j : i, dj = swap ? i : j;
            const double z11 = z[0], z12 = z[1], z21 = z[3], z22 = z[5];
            if (flags & 1) {
#pragma unroll
              for (int e = 0; e < RPL; ++e) {
                const double a = fi[e], b = fj[e], c = gi[e], d = gj[e];
                fi[e] = fma(b, z21, a * z11);
                fj[e] = fma(a, z12, b * z22);
                gi[e] = fma(d, z21, c * z11);
                gj[e] = fma(c, z12, d * z22);
              }
            }
            store_rows<TW, VEC, RPL, SW>(Ar, di, r0, fi);
            store_rows<TW, VEC, RPL, SW>(Ar, dj, r0, fj);
            store_rows<TW, VEC, RPL, SW>(Br, di, r0, gi);
            store_rows<TW, VEC, RPL, SW>(Br, dj, r0, gj);
            double zi_[RPL], zj_[RPL];
            load_rows<TW, VEC, RPL, SW>(Zr, i, r0, zi_);
            load_rows<TW, VEC, RPL, SW>(Zr, j, r0, zj_);
            if (flags & 1) {
#pragma unroll
              for (int e = 0; e < RPL; ++e) {
                const double a = zi_[e], b = zj_[e];
                zi_[e] = fma(b, z21, a * z11);
                zj_[e] = fma(a, z12, b * z22);
              }
            }
            store_rows<TW, VEC, RPL, SW>(Zr, di, r0, zi_);
            store_rows<TW, VEC, RPL, SW>(Zr, dj, r0, zj_);
          }
        } else {
        bool swap = (flags & 4) != 0;
        double zi_[RPL], zj_[RPL], zii[RPL], zji[RPL];
        if (flags & 5) {
          load_rows<TW, VEC, RPL, SW>(Zr, i, r0, zi_);
          load_rows<TW, VEC, RPL, SW>(Zr, j, r0, zj_);
          if constexpr (CPLX) {
            load_rows<TW, VEC, RPL, SW>(Zi, i, r0, zii);
            load_rows<TW, VEC, RPL, SW>(Zi, j, r0, zji);
          }
          if (flags & 1) {
            const double z11 = z[0], z12r = z[1], z12i = z[2], z21r = z[3], z21i = z[4], z22 = z[5];
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
            for (int e = 0; e < RPL; ++e) {
              HZG_UPD(fi, fii, fj, fji);
              HZG_UPD(gi, gii, gj, gji);
              HZG_UPD(zi_, zii, zj_, zji);
            }
#undef HZG_UPD
          }
        }
        if (CPLX && kc.sorting && kc.compensated) {
          // complex sort, compensated norms of the updated columns
          // (pointwise.py:211-214): park the updated F columns, let the
          // math lane read them whole
          if (flags & 1) {
            store_rows<TW, VEC, RPL, SW>(Ar, i, r0, fi);
            store_rows<TW, VEC, RPL, SW>(Ar, j, r0, fj);
            store_rows<TW, VEC, RPL, SW>(Ai, i, r0, fii);
            store_rows<TW, VEC, RPL, SW>(Ai, j, r0, fji);
          }
          __syncwarp();
          int sw_ = 0;
          if (mathlane && (flags & 1)) {
            const double ni = ccol_norm(Ar + i * TW, Ai + i * TW, TW, S.cbuf[pv]);
            const double nj = ccol_norm(Ar + j * TW, Ai + j * TW, TW, S.cbuf[pv]);
            sw_ = ni < nj;
          }
          sw_ = __shfl_sync(0xffffffffu, sw_, base);
          if (flags & 1) swap = sw_ != 0;
          __syncwarp();
        } else if (CPLX && kc.sorting) {
          // complex sort: recompute the squared norms after the update
          // (pointwise.py:211-214); every lane takes part in the shuffles
          double q0[RPL], q1[RPL];
#pragma unroll
          for (int e = 0; e < RPL; ++e) {
            q0[e] = nrm_term<CPLX>(fi[e], fii[e]);
            q1[e] = nrm_term<CPLX>(fj[e], fji[e]);
          }
          double ni = row_tree<RPL>(q0), nj = row_tree<RPL>(q1);
#pragma unroll
          for (int d = 1; d < LP; d <<= 1) {
            ni = ni + __shfl_xor_sync(0xffffffffu, ni, d);
            nj = nj + __shfl_xor_sync(0xffffffffu, nj, d);
          }
          if (flags & 1) swap = ni < nj;
        }
        if (flags & 5) {
          const int di = swap ? j : i, dj = swap ? i : j;
          store_rows<TW, VEC, RPL, SW>(Ar, di, r0, fi);
          store_rows<TW, VEC, RPL, SW>(Ar, dj, r0, fj);
          store_rows<TW, VEC, RPL, SW>(Br, di, r0, gi);
          store_rows<TW, VEC, RPL, SW>(Br, dj, r0, gj);
          store_rows<TW, VEC, RPL, SW>(Zr, di, r0, zi_);
          store_rows<TW, VEC, RPL, SW>(Zr, dj, r0, zj_);
          if constexpr (CPLX) {
            store_rows<TW, VEC, RPL, SW>(Ai, di, r0, fii);
            store_rows<TW, VEC, RPL, SW>(Ai, dj, r0, fji);
            store_rows<TW, VEC, RPL, SW>(Bi, di, r0, gii);
            store_rows<TW, VEC, RPL, SW>(Bi, dj, r0, gji);
            store_rows<TW, VEC, RPL, SW>(Zi, di, r0, zii);
            store_rows<TW, VEC, RPL, SW>(Zi, dj, r0, zji);
          }
        }
        }
        // a rank-deficient pivot anywhere ends the solve (RankError upstream)
        const int anybad = __syncthreads_or(bad);
        if (prof) {
          atomicAdd(&ph[2], (unsigned long long)(clock64() - c0));
          atomicAdd(&ph[3], 1ull);
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
  }

  // ---- theta rescale (pointwise.py:277-293) ------------------------------
  int tbad = 0;
  if (status == ST_OK) {
    for (int c = warp; c < TW; c += NW) {
      double ar[EPL], ai[EPL], br[EPL], bi[EPL], p[EPL], q[EPL];
      load_col<TW, CPLX, SW>(Ar, Ai, c, lane, ar, ai);
      load_col<TW, CPLX, SW>(Br, Bi, c, lane, br, bi);
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        p[e] = nrm_term<CPLX>(ar[e], ai[e]);
        q[e] = nrm_term<CPLX>(br[e], bi[e]);
      }
      double s = lane_tree<EPL>(p) + lane_tree<EPL>(q);
      if (kc.compensated) {  // pointwise.py:283-284 with comp
        double v = 0.0;
        if (lane == 0)
          v = ccol_norm(Ar + c * TW, CPLX ? Ai + c * TW : nullptr, TW, S.cbuf[warp]) +
              ccol_norm(Br + c * TW, CPLX ? Bi + c * TW : nullptr, TW, S.cbuf[warp]);
        s = __shfl_sync(0xffffffffu, v, 0);
      }
      if (!(s > 0.0)) {
        tbad = 1;
      } else {
        double th = 1.0 / sqrt(s);
        if (th != 1.0) {
          double zr[EPL], zi2[EPL];
          load_col<TW, CPLX, SW>(Zr, Zi, c, lane, zr, zi2);
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            zr[e] *= th;
            zi2[e] *= th;
          }
          store_col<TW, CPLX, SW>(Zr, Zi, c, lane, zr, zi2);
        }
      }
    }
  }
  if (__syncthreads_or(tbad) && status == ST_OK) status = ST_RANK;

  // ---- exact-identity test (blocked.py:298-308) and outputs ---------------
  int nonid = 0;
  for (int e = tid; e < TW * TW; e += nt) {
    double want = rp_inv<SW, TW>(e % TW) == (e / TW) ? 1.0 : 0.0;
    if (Zr[e] != want) nonid = 1;
    if (CPLX && Zi[e] != 0.0) nonid = 1;
  }
  nonid = __syncthreads_or(nonid);
  // Z~ leaves in natural column-major order
  double* zt = P.io.zt + (int64_t)pair * NP * TW * TW;
  for (int e = tid; e < NP * TW * TW; e += nt) {
    const int pl = e / (TW * TW), q = e % (TW * TW);
    zt[pl * TW * TW + (q / TW) * TW + rp_inv<SW, TW>(q % TW)] = (&S.Z[0][0])[e];
  }
  if (tid == 0) {
    P.io.ident[pair] = (nonid == 0 || status != ST_OK) ? 1 : 0;
    int32_t* cnt = P.io.counts + ((int64_t)P.step * P.sp.npairs + pair) * 4;
    cnt[0] = total;
    cnt[1] = big;
    cnt[2] = status;
    cnt[3] = sweeps;
  }
  }  // pairs
}

template <int TW, bool CPLX, int SW>
int launch_inner_g(const InnerParams& p, cudaStream_t s) {
  // the compensated variants' scratch (cbuf, the struct's last member) is
  // only allocated when they run: 2w = 64 real then fits 2 CTAs per SM
  using Smem = InnerSmem<TW, CPLX>;
  const size_t full = sizeof(Smem);
  size_t smem = p.kc.compensated ? full : offsetof(Smem, cbuf);
  // HZG_INNER_SMEM (KB, performance knob): pad the request so fewer inner
  // CTAs share an SM and a streaming CTA fits beside one (tuning only)
  static int pad_kb = -1;
  if (pad_kb < 0) {
    const char* e = std::getenv("HZG_INNER_SMEM");
    pad_kb = e ? std::max(0, std::atoi(e)) : 0;
  }
  if ((size_t)pad_kb * 1024 > smem) smem = std::min<size_t>((size_t)pad_kb * 1024, 227 * 1024);
  static PerDeviceOnce attr;
  if (attr.first())
    cudaFuncSetAttribute(k_inner<TW, CPLX, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max<size_t>(full, smem));
  // HZG_INNER_CTAS caps the CTAs of one launch (each then serves several
  // pairs), leaving SM room for the streaming kernels of other groups
  static int cap = -1;
  if (cap < 0) {
    const char* e = std::getenv("HZG_INNER_CTAS");
    cap = e ? std::max(0, std::atoi(e)) : 0;
  }
  const int grid = cap > 0 && cap < p.sp.pn ? cap : p.sp.pn;
  // HZG_INNER_PRIO=1 launches the inner solves at the highest scheduling
  // priority (a node attribute inside the sweep graph), so their latency-
  // bound CTAs are placed ahead of queued streaming CTAs (for tuning)
  static int prio = -1;
  if (prio < 0) {
    const char* e = std::getenv("HZG_INNER_PRIO");
    prio = e ? std::atoi(e) : 0;
  }
  if (prio) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(InnerGeo<TW, CPLX>::NW * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = hi;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, k_inner<TW, CPLX, SW>, p);
  } else {
    k_inner<TW, CPLX, SW><<<grid, InnerGeo<TW, CPLX>::NW * 32, smem, s>>>(p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int TW, bool CPLX>
int launch_inner_t(const InnerParams& p, cudaStream_t s) {
  // swizzled rows (period = rows per lane) for the 16-byte lane-group
  // layout; the compensated variants read whole columns in natural order
  if constexpr (TW == 8 || TW == 16 || TW == 32 || (TW == 64 && !CPLX)) {
    if (!p.kc.compensated) return launch_inner_g<TW, CPLX, InnerGeo<TW, CPLX>::RPL>(p, s);
  }
  return launch_inner_g<TW, CPLX, 0>(p, s);
}

// Single-block operations of the public API (cholesky_upper, qr_shorten,
// blocked.py:345-363): the same device code the inner kernel uses.
template <int TW, bool CPLX>
__global__ void k_cholesky_op(double* Ar, double* Ai, int32_t* status) {
  const int f = warp_cholesky<TW, CPLX, 0>(Ar, Ai, threadIdx.x & 31);
  if (threadIdx.x == 0) *status = f;
}

template <int TW, bool CPLX>
__global__ void __launch_bounds__(256) k_qr_op(Plane Y, double* Sr, double* Si, double* outR, double* outI,
                                              int32_t* status) {
  __shared__ double qsh[3 * kMaxTW + 8];
  const int bad = block_qr<TW, CPLX, 0>(Y, 0, TW / 2, TW / 2, Sr, Si, outR, outI, qsh);
  if (threadIdx.x == 0) *status = bad;
}

}  // namespace

int launch_cholesky_op(int tw, int cplx, double* Ar, double* Ai, int32_t* status, cudaStream_t s) {
#define HZG_CASE(T)                                                                      \
  case T:                                                                                \
    if (cplx) k_cholesky_op<T, true><<<1, 32, 0, s>>>(Ar, Ai, status);                   \
    else k_cholesky_op<T, false><<<1, 32, 0, s>>>(Ar, Ai, status);                       \
    break;
  switch (tw) {
    HZG_CASE(2) HZG_CASE(4) HZG_CASE(6) HZG_CASE(8) HZG_CASE(10) HZG_CASE(12) HZG_CASE(14) HZG_CASE(16)
    HZG_CASE(20) HZG_CASE(24) HZG_CASE(32) HZG_CASE(48) HZG_CASE(64)
    default:
      return 4;
  }
#undef HZG_CASE
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_qr_op(const Plane& Y, int tw, int cplx, double* Sr, double* Si, double* outR, double* outI,
                 int32_t* status, cudaStream_t s) {
#define HZG_CASE(T)                                                                      \
  case T:                                                                                \
    if (cplx) k_qr_op<T, true><<<1, 256, 0, s>>>(Y, Sr, Si, outR, outI, status);         \
    else k_qr_op<T, false><<<1, 256, 0, s>>>(Y, Sr, Si, outR, outI, status);             \
    break;
  switch (tw) {
    HZG_CASE(2) HZG_CASE(4) HZG_CASE(6) HZG_CASE(8) HZG_CASE(10) HZG_CASE(12) HZG_CASE(14) HZG_CASE(16)
    HZG_CASE(20) HZG_CASE(24) HZG_CASE(32) HZG_CASE(48) HZG_CASE(64)
    default:
      return 4;
  }
#undef HZG_CASE
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

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
