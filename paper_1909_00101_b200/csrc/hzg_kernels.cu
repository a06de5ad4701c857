// Column-scaling, rescaling, counter, finalization and reference-order
// ("exact") Grammian / postmultiply kernels.
//
// Column norms over the full height m use the reference's pairwise tree
// over pow2(m) values (dotprod.py:79-91): each thread folds one aligned
// chunk, then a warp butterfly and a cross-warp butterfly finish the tree.
// The result is bitwise the reference's _k_col_norm for any m.
#include "hzg_device.cuh"
#include "hzg_internal.h"

namespace hzg {

namespace {

constexpr int kNT = 256;  // threads for the column kernels (power of two)

// Sum of term(idx) for idx in [0, m) in the reference tree shape, by a block
// of kNT threads.  red: kNT/32 doubles of shared memory.  All threads
// receive the result.
template <typename Term>
__device__ double block_tree(Term term, int64_t m, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t P = pow2_ceil(m);
  double v = 0.0;
  if (P <= kNT) {
    if (tid < m) v = term(tid);
  } else {
    int64_t C = P / kNT, beg = (int64_t)tid * C;
    if (beg < m) {
      PairwiseAcc<24> acc;
      acc.reset();
      for (int64_t i = 0; i < C; ++i) {
        int64_t idx = beg + i;
        acc.push(idx < m ? term(idx) : 0.0);
      }
      v = acc.result();
    }
  }
  v = warp_tree(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = lane < kNT / 32 ? red[lane] : 0.0;
  r = warp_tree(r);
  return r;
}

struct NormTerm {
  const double* re;
  const double* im;
  __device__ double operator()(int64_t i) const {
    double r = re[i];
    if (im) {
      double q = im[i];
      return fma(q, q, r * r);  // dotprod.py:227-232
    }
    return r * r;  // dotprod.py:206-211
  }
};

__device__ __forceinline__ void scale_col(double* re, double* im, int64_t rows, double s) {
  for (int64_t x = threadIdx.x; x < rows; x += blockDim.x) {
    re[x] *= s;
    if (im) im[x] *= s;
  }
}

// pointwise.py:254-274 over the full pair (blocked.py:564-570); Z is zero
// on entry and receives diag(z0).
// Squared column norm over the full height: the reference tree by the whole
// block, or (cscr != nullptr: compensated variants) the reference's
// sequential compensated form by thread 0 on the column's scratch.
__device__ double col_norm_full(const double* re, const double* im, int64_t rows, double* red, double* cscr) {
  if (!cscr) return block_tree(NormTerm{re, im}, rows, red);
  __syncthreads();
  if (threadIdx.x == 0) red[0] = ccol_norm(re, im, rows, cscr);
  __syncthreads();
  const double v = red[0];
  __syncthreads();
  return v;
}

__global__ void __launch_bounds__(kNT) k_prescale(Plane F, Plane G, Plane Z, int do_prescale, int32_t* status,
                                                  double* cscr, int64_t cstride) {
  __shared__ double red[kNT / 32];
  const int64_t j = blockIdx.x;
  double z = 1.0;
  if (do_prescale) {
    double* gr = G.re + j * G.ld;
    double* gi = G.im ? G.im + j * G.ld : nullptr;
    double ng2 = col_norm_full(gr, gi, G.rows, red, cscr ? cscr + j * cstride : nullptr);
    if (!(ng2 > 0.0)) {
      if (threadIdx.x == 0) atomicOr(status, ST_RANK);
      return;
    }
    z = 1.0 / sqrt(ng2);
    if (z != 1.0) {
      scale_col(F.re + j * F.ld, F.im ? F.im + j * F.ld : nullptr, F.rows, z);
      scale_col(gr, gi, G.rows, z);
    }
  }
  if (threadIdx.x == 0) Z.re[j * Z.ld + j] = z;
}

// blocked.py:253-295.  gate (optional): the sweep counters; a non-final
// rescale only runs when the sweep applied big transforms and saw no error
// (the reference breaks before rescaling on convergence, blocked.py:537-542).
__global__ void __launch_bounds__(kNT) k_rescale(Plane F, Plane G, Plane Z, int final, double* sigF, double* sigG,
                                                 double* sig, const int64_t* gate, int32_t* status, double* cscr,
                                                 int64_t cstride) {
  __shared__ double red[kNT / 32];
  if (gate && (gate[1] == 0 || gate[2] != 0)) return;
  const int64_t j = blockIdx.x;
  double* fr = F.re + j * F.ld;
  double* fi = F.im ? F.im + j * F.ld : nullptr;
  double* gr = G.re + j * G.ld;
  double* gi = G.im ? G.im + j * G.ld : nullptr;
  double* cs = cscr ? cscr + j * cstride : nullptr;
  double nf2 = col_norm_full(fr, fi, F.rows, red, cs);
  double ng2 = col_norm_full(gr, gi, G.rows, red, cs);
  double sf = 0.0, sg = 0.0;
  if (final) {
    if (!(nf2 > 0.0 && ng2 > 0.0)) {
      if (threadIdx.x == 0) atomicOr(status, ST_RANK);
      return;
    }
    sf = sqrt(nf2);
    if (nf2 != 1.0) scale_col(fr, fi, F.rows, 1.0 / sf);
    sg = sqrt(ng2);
    if (ng2 != 1.0) scale_col(gr, gi, G.rows, 1.0 / sg);
  }
  double s = nf2 + ng2;
  if (!(s > 0.0)) {
    if (threadIdx.x == 0) atomicOr(status, ST_RANK);
    return;
  }
  double th = 1.0 / sqrt(s);
  if (th != 1.0) scale_col(Z.re + j * Z.ld, Z.im ? Z.im + j * Z.ld : nullptr, Z.rows, th);
  if (final && threadIdx.x == 0) {
    sigF[j] = sf * th;
    sigG[j] = sg * th;
    sig[j] = sigF[j] / sigG[j];
  }
}

// ---------------------------------------------------------------------------
// reference-order Grammian partials (blocked.py:40-56): one warp per upper
// entry, lanes fold aligned sub-chunks of the split, butterfly across lanes.
// ---------------------------------------------------------------------------
struct GramExactParams {
  Plane Y[2];
  StepPairs sp;
  int step, w, cplx;
  GramWS gw;
};

__global__ void __launch_bounds__(256) k_gram_exact(GramExactParams P) {
  const int pair = P.sp.p0 + blockIdx.x, mat = blockIdx.y, split = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (split >= P.gw.nsplit[mat]) return;
  const Plane& Y = P.Y[mat];
  const int w = P.w, tw = 2 * w, NP = P.cplx ? 2 : 1;
  const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
  const int64_t L = P.gw.chunk[mat], C = L / 32, row0 = (int64_t)split * L + lane * C;
  double* out = P.gw.part + (((int64_t)pair * 2 + mat) * P.gw.smax + split) * NP * tw * tw;
  const int ne = tw * tw;
  for (int e = warp; e < ne; e += nw) {
    const int r = e % tw, s = e / tw;
    if (r > s) continue;
    const int64_t cr = r < w ? cp[0] + r : cp[1] + (r - w);
    const int64_t cs = s < w ? cp[0] + s : cp[1] + (s - w);
    const double* ar = Y.re + cr * Y.ld;
    const double* br = Y.re + cs * Y.ld;
    const double* ai = Y.im ? Y.im + cr * Y.ld : nullptr;
    const double* bi = Y.im ? Y.im + cs * Y.ld : nullptr;
    PairwiseAcc<24> acc_r, acc_i;
    acc_r.reset();
    acc_i.reset();
    for (int64_t q = 0; q < C; ++q) {
      const int64_t x = row0 + q;
      double tr = 0.0, ti = 0.0;
      if (x < Y.rows) {
        if (r == s) {
          tr = P.cplx ? fma(ai[x], ai[x], ar[x] * ar[x]) : ar[x] * ar[x];
        } else if (P.cplx) {
          // conj(a) * b, dotprod.py:146-155 with conj_first
          tr = fma(ar[x], br[x], -((-1.0 * ai[x]) * bi[x]));
          ti = fma(ar[x], bi[x], (-1.0 * ai[x]) * br[x]);
        } else {
          tr = ar[x] * br[x];
        }
      }
      acc_r.push(tr);
      if (P.cplx && r != s) acc_i.push(ti);
    }
    double vr = warp_tree(acc_r.result());
    double vi = (P.cplx && r != s) ? warp_tree(acc_i.result()) : 0.0;
    if (lane == 0) {
      out[e] = vr;
      if (P.cplx) out[ne + e] = vi;
    }
  }
}

// ---------------------------------------------------------------------------
// compensated Grammian (odd variant ids; blocked.py:40-56 with comp): one
// thread per upper entry, the reference's sequential compensated forms over
// the full height on a per-thread scratch of pow2(m) doubles.  Written as
// the single split of the partials.
// ---------------------------------------------------------------------------
constexpr int kGramCompNT = 32;

struct GramCompParams {
  Plane Y[2];
  StepPairs sp;
  int step, w, cplx;
  GramWS gw;
  double* scratch;
  int64_t pstride;
};

__global__ void __launch_bounds__(kGramCompNT) k_gram_comp(GramCompParams P) {
  const int pair = P.sp.p0 + blockIdx.x, mat = blockIdx.y;
  const Plane& Y = P.Y[mat];
  const int w = P.w, tw = 2 * w, NP = P.cplx ? 2 : 1;
  const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
  double* out = P.gw.part + ((int64_t)pair * 2 + mat) * P.gw.smax * NP * tw * tw;
  double* buf = P.scratch + (((int64_t)pair * 2 + mat) * kGramCompNT + threadIdx.x) * P.pstride;
  const int ne = tw * tw;
  for (int e = threadIdx.x; e < ne; e += kGramCompNT) {
    const int r = e % tw, s = e / tw;
    if (r > s) continue;
    const int64_t cr = r < w ? cp[0] + r : cp[1] + (r - w);
    const int64_t cs = s < w ? cp[0] + s : cp[1] + (s - w);
    const double* ar = Y.re + cr * Y.ld;
    const double* ai = Y.im ? Y.im + cr * Y.ld : nullptr;
    double vr, vi = 0.0;
    if (r == s) {
      vr = ccol_norm(ar, ai, Y.rows, buf);
    } else {
      ccol_dot(ar, ai, Y.re + cs * Y.ld, Y.im ? Y.im + cs * Y.ld : nullptr, Y.rows, buf, vr, vi);
    }
    out[e] = vr;
    if (P.cplx) out[ne + e] = vi;
  }
}

// ---------------------------------------------------------------------------
// reference-order postmultiply (blocked.py:220-250): one thread per row,
// out[c] = fma chain over k = 0 .. 2w-1.
// ---------------------------------------------------------------------------
struct PostExactParams {
  Plane Y[3];
  StepPairs sp;
  int step, w, cplx;
  InnerOut io;
};

template <int TW, bool CPLX>
__global__ void __launch_bounds__(128) k_postmult_exact(PostExactParams P) {
  const int pair = P.sp.p0 + blockIdx.y, mat = blockIdx.z;
  if (P.io.ident[pair]) return;
  constexpr int NP = CPLX ? 2 : 1;
  extern __shared__ double zt_raw[];
  double(*zt)[TW * TW] = reinterpret_cast<double(*)[TW * TW]>(zt_raw);
  const double* src = P.io.zt + (int64_t)pair * NP * TW * TW;
  for (int e = threadIdx.x; e < NP * TW * TW; e += blockDim.x) zt_raw[e] = src[e];
  __syncthreads();
  const Plane& Y = P.Y[mat];
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= Y.rows) return;
  constexpr int w = TW / 2;
  const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
  double rr[TW], ri[CPLX ? TW : 1];
#pragma unroll
  for (int k = 0; k < TW; ++k) {
    const int64_t c = k < w ? cp[0] + k : cp[1] + (k - w);
    rr[k] = Y.re[c * Y.ld + x];
    if (CPLX) ri[k] = Y.im[c * Y.ld + x];
  }
#pragma unroll 1
  for (int c = 0; c < TW; ++c) {
    double a_r = 0.0, a_i = 0.0;
#pragma unroll
    for (int k = 0; k < TW; ++k) {
      if (CPLX) {
        a_r = fma(rr[k], zt[0][c * TW + k], fma(-ri[k], zt[1][c * TW + k], a_r));
        a_i = fma(rr[k], zt[1][c * TW + k], fma(ri[k], zt[0][c * TW + k], a_i));
      } else {
        a_r = fma(rr[k], zt[0][c * TW + k], a_r);
      }
    }
    const int64_t col = c < w ? cp[0] + c : cp[1] + (c - w);
    Y.re[col * Y.ld + x] = a_r;
    if (CPLX) Y.im[col * Y.ld + x] = a_i;
  }
}

template <int TW, bool CPLX>
int launch_post_exact_t(const PostExactParams& p, int64_t mmax, cudaStream_t s) {
  dim3 grid((unsigned)((mmax + 127) / 128), p.sp.pn, 3);
  const size_t smem = (CPLX ? 2 : 1) * TW * TW * sizeof(double);
  static PerDeviceOnce once;
  if (once.first())
    cudaFuncSetAttribute(k_postmult_exact<TW, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_postmult_exact<TW, CPLX><<<grid, 128, smem, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ---------------------------------------------------------------------------
// per-sweep counter fold (blocked.py:531-536): integer sums, so exact in
// any order; the status words are OR-ed.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_counters(const int32_t* counts, int64_t n, int64_t* out) {
  __shared__ long long st[3][32];
  long long t = 0, b = 0, s = 0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    t += counts[e * 4 + 0];
    b += counts[e * 4 + 1];
    s |= counts[e * 4 + 2];
  }
  for (int d = 16; d >= 1; d >>= 1) {
    t += __shfl_xor_sync(0xffffffffu, t, d);
    b += __shfl_xor_sync(0xffffffffu, b, d);
    s |= __shfl_xor_sync(0xffffffffu, s, d);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    st[0][warp] = t;
    st[1][warp] = b;
    st[2][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long T = 0, B = 0, S = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      T += st[0][q];
      B += st[1][q];
      S |= st[2][q];
    }
    out[0] = T;
    out[1] = B;
    out[2] = S;
  }
}

// ---------------------------------------------------------------------------
// finalization: unborder (blocked.py:593-620) + stable descending sort
// (blocked.py:623-637) + column gather into the output planes
// ---------------------------------------------------------------------------
__global__ void k_keep(Plane Z, int64_t n, int64_t n0, int32_t* keep) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int k = 1;
  if (n > n0) {
    const double* zr = Z.re + j * Z.ld;
    const double* zi = Z.im ? Z.im + j * Z.ld : nullptr;
    for (int64_t x = n0; x < n; ++x) {
      if (!(zr[x] == 0.0)) k = 0;
      if (zi && !(zi[x] == 0.0)) k = 0;
    }
  }
  keep[j] = k;
}

__global__ void __launch_bounds__(1024) k_keep_count(const int32_t* keep, int64_t n, int64_t n0, int32_t* status) {
  __shared__ long long part[32];
  long long c = 0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) c += keep[j];
  for (int d = 16; d >= 1; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += part[q];
    if (tot != n0) atomicOr(status, ST_RANK);
  }
}

// rank of kept column i in np.argsort(-sigma, kind="stable") over the kept
// columns (NaN keys sort last, as numpy does)
__global__ void k_rank(const double* sig, const int32_t* keep, int64_t n, int sort, int32_t* rank) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  extern __shared__ double tile[];
  int32_t* ktile = reinterpret_cast<int32_t*>(tile + blockDim.x);
  const double ki = i < n ? -sig[i] : 0.0;
  const bool nan_i = ki != ki;
  int32_t r = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    __syncthreads();
    if (base + threadIdx.x < n) {
      tile[threadIdx.x] = -sig[base + threadIdx.x];
      ktile[threadIdx.x] = keep[base + threadIdx.x];
    }
    __syncthreads();
    const int64_t lim = n - base < (int64_t)blockDim.x ? n - base : blockDim.x;
    for (int64_t q = 0; q < lim; ++q) {
      if (!ktile[q]) continue;
      const double kj = tile[q];
      const int64_t j = base + q;
      const bool nan_j = kj != kj;
      bool before;
      if (!sort) before = j < i;
      else if (nan_i || nan_j) before = (!nan_j && nan_i) || (nan_i && nan_j && j < i);
      else before = kj < ki || (kj == ki && j < i);
      r += before;
    }
  }
  if (i < n) rank[i] = keep[i] ? r : -1;
}

struct GatherParams {
  Plane in[3], out[3];
  const double *sF, *sG, *s;
  double *sFo, *sGo, *so;
  const int32_t* rank;
  int64_t n0;  // output columns: a rank >= n0 (unborder mismatch) writes nothing
};

__global__ void k_gather(GatherParams P) {
  const int64_t j = blockIdx.x;
  const int32_t r = P.rank[j];
  // r >= n0 only when unbordering kept more than n0 columns; k_keep_count
  // has flagged ST_RANK and the host raises RankError after finalize, so
  // the gather must not write past the n0-column outputs meanwhile
  if (r < 0 || r >= P.n0) return;
  for (int m = 0; m < 3; ++m) {
    const Plane& a = P.in[m];
    const Plane& b = P.out[m];
    for (int64_t x = threadIdx.x; x < b.rows; x += blockDim.x) {
      b.re[(int64_t)r * b.ld + x] = a.re[j * a.ld + x];
      if (b.im) b.im[(int64_t)r * b.ld + x] = a.im[j * a.ld + x];
    }
  }
  if (threadIdx.x == 0) {
    P.sFo[r] = P.sF[j];
    P.sGo[r] = P.sG[j];
    P.so[r] = P.s[j];
  }
}

// self-check of the branch-free division / square root against the IEEE
// operators on random operands spanning the whole exponent range
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_fastmath_check(int64_t n, uint64_t seed, unsigned long long* cnt) {
  unsigned long long c[4] = {0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h1 = mix64(seed + 2 * i + 1), h2 = mix64(seed + 2 * i + 2);
    // random mantissas; exponents mostly moderate, sometimes anywhere
    uint64_t e1 = (h1 >> 52) & 0x7ff, e2 = (h2 >> 52) & 0x7ff;
    if ((h1 & 3) != 0) e1 = 1023 + ((int)(e1 % 120) - 60);
    if ((h2 & 3) != 0) e2 = 1023 + ((int)(e2 % 120) - 60);
    double a = __longlong_as_double((long long)(((h1 & 0x000fffffffffffffull)) | (e1 << 52) | (h1 & (1ull << 63) ? (1ull << 63) : 0)));
    double b = __longlong_as_double((long long)(((h2 & 0x000fffffffffffffull)) | (e2 << 52)));
    bool ok = true;
    double q = fast_div(a, b, ok);
    if (ok) {
      ++c[0];
      if (__double_as_longlong(q) != __double_as_longlong(a / b)) ++c[1];
    }
    ok = true;
    double r = fast_sqrt(b, ok);
    if (ok) {
      ++c[2];
      if (__double_as_longlong(r) != __double_as_longlong(sqrt(b))) ++c[3];
    }
  }
  for (int k = 0; k < 4; ++k) atomicAdd(&cnt[k], c[k]);
}

}  // namespace

int fastmath_check(int64_t n, uint64_t seed, int64_t* out4) {
  unsigned long long* d = nullptr;
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  k_fastmath_check<<<148 * 8, 256>>>(n, seed, d);
  cudaError_t e = cudaMemcpy(out4, d, 32, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 3;
}

int launch_prescale(const Plane& F, const Plane& G, const Plane& Z, int64_t n, int cplx, int do_prescale,
                    int32_t* status, double* cscr, int64_t cstride, cudaStream_t s) {
  (void)cplx;
  k_prescale<<<(unsigned)n, kNT, 0, s>>>(F, G, Z, do_prescale, status, cscr, cstride);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_rescale(const Plane& F, const Plane& G, const Plane& Z, int64_t n, int cplx, int final, double* sigF,
                   double* sigG, double* sig, const int64_t* gate, int32_t* status, double* cscr, int64_t cstride,
                   cudaStream_t s) {
  (void)cplx;
  k_rescale<<<(unsigned)n, kNT, 0, s>>>(F, G, Z, final, sigF, sigG, sig, gate, status, cscr, cstride);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_gram_exact(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                      const GramWS& gw, cudaStream_t s) {
  GramExactParams p{{F, G}, sp, step, w, cplx, gw};
  dim3 grid(sp.pn, 2, gw.smax);
  k_gram_exact<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_postmult_exact(const Plane& F, const Plane& G, const Plane& Z, const StepPairs& sp, int step, int w,
                          int cplx, const InnerOut& io, cudaStream_t s) {
  PostExactParams p{{F, G, Z}, sp, step, w, cplx, io};
  int64_t mmax = F.rows > G.rows ? F.rows : G.rows;
  if (Z.rows > mmax) mmax = Z.rows;
#define HZG_CASE(T)                                                                                  \
  case T:                                                                                            \
    return cplx ? launch_post_exact_t<T, true>(p, mmax, s) : launch_post_exact_t<T, false>(p, mmax, s);
  switch (2 * w) {
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

int launch_gram_comp(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                     const GramWS& gw, double* scratch, int64_t pstride, cudaStream_t s) {
  GramCompParams p{{F, G}, sp, step, w, cplx, gw, scratch, pstride};
  dim3 grid(sp.pn, 2, 1);
  k_gram_comp<<<grid, kGramCompNT, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Fold the split partials of one block pair's Grammian (pairwise over the
// splits, the reference's tree) and mirror it into a full tw x tw matrix
// (blocked.py:40-56: lower = conj of upper, real diagonal).
__global__ void k_fold_gram(const double* part, int nsplit, int tw, int cplx, double* Ar, double* Ai) {
  const int NP = cplx ? 2 : 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tw * tw; e += gridDim.x * blockDim.x) {
    const int r = e % tw, c = e / tw;
    if (r > c) continue;
    for (int pl = 0; pl < NP; ++pl) {
      PairwiseAcc<24> acc;
      acc.reset();
      for (int q = 0; q < nsplit; ++q) acc.push(part[((int64_t)q * NP + pl) * tw * tw + e]);
      const double v = acc.result();
      if (pl == 0) {
        Ar[c * tw + r] = v;
        Ar[r * tw + c] = v;
      } else {
        Ai[c * tw + r] = r == c ? 0.0 : v;
        Ai[r * tw + c] = r == c ? 0.0 : -v;
      }
    }
    if (!cplx && Ai) {
      Ai[c * tw + r] = 0.0;
      Ai[r * tw + c] = 0.0;
    }
  }
}

int launch_fold_gram(const double* part, int nsplit, int tw, int cplx, double* Ar, double* Ai, cudaStream_t s) {
  k_fold_gram<<<(tw * tw + 255) / 256, 256, 0, s>>>(part, nsplit, tw, cplx, Ar, Ai);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_counters(const int32_t* counts, int64_t nentries, int64_t* out, cudaStream_t s) {
  k_counters<<<1, 1024, 0, s>>>(counts, nentries, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_finalize(const Plane& U, const Plane& V, const Plane& Z, int64_t n, int64_t n0, int64_t mF0, int64_t mG0,
                    int cplx, int sort, const double* sigF, const double* sigG, const double* sig, Plane Uo, Plane Vo,
                    Plane Zo, double* sFo, double* sGo, double* so, int32_t* ws, int32_t* status, cudaStream_t s) {
  (void)cplx;
  (void)mF0;
  (void)mG0;
  int32_t* keep = ws;
  int32_t* rank = ws + n;
  const int tb = 256;
  k_keep<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(Z, n, n0, keep);
  k_keep_count<<<1, 1024, 0, s>>>(keep, n, n0, status);
  k_rank<<<(unsigned)((n + tb - 1) / tb), tb, tb * (sizeof(double) + sizeof(int32_t)), s>>>(sig, keep, n, sort, rank);
  GatherParams g{{U, V, Z}, {Uo, Vo, Zo}, sigF, sigG, sig, sFo, sGo, so, rank, n0};
  k_gather<<<(unsigned)n, 256, 0, s>>>(g);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace hzg
