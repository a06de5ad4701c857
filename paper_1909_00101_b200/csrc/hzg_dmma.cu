// FP64 tensor-core (DMMA) Grammian and postmultiply kernels for sm_100a:
// subphases 1 and 4 of the paper's bstep,
// the HBM-bound bulk of every outer step.
//
// Both stream 64-row tiles of a 2w-column block pair through shared memory
// with the TMA bulk-copy engine (cp.async.bulk, one 512-byte column segment
// per copy, completion on an mbarrier), multi-stage, and feed
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Shared tiles are column-major
// with a 4-double pad per column so both DMMA operand fragments load
// conflict-free.  The postmultiply writes its result back in place and
// drains it with bulk shared->global copies, so every element of F, G and
// Z is read once and written once per step.
//
// Tolerance parity only: DMMA accumulates in a different order from the
// reference's pairwise trees (blocked.py:40-56) and fma chains (:220-250).
#include <algorithm>
#include <cstdlib>

#include "hzg_device.cuh"
#include "hzg_internal.h"

namespace hzg {

namespace {

constexpr int kR = 64;        // rows per tile
constexpr int kRS = kR + 4;   // padded column stride in shared memory (doubles)

__device__ __forceinline__ int64_t pair_col(const int32_t* cp, int w, int k) {
  return k < w ? (int64_t)cp[0] + k : (int64_t)cp[1] + (k - w);
}

// Issue the bulk copies of one tile (all columns, all planes) into a stage.
template <int TW, int NP>
__device__ __forceinline__ void issue_tile_load(const Plane& Y, const int32_t* cp, int64_t row0, int nv,
                                                double* stage, uint64_t* bar, int lane) {
  constexpr int w = TW / 2;
  const uint32_t bytes = (uint32_t)nv * 8u;
  if (lane == 0) mbar_expect_tx(bar, bytes * TW * NP);
  __syncwarp();
  for (int q = lane; q < TW * NP; q += 32) {
    const int c = q % TW, pl = q / TW;
    const double* base = pl == 0 ? Y.re : Y.im;
    bulk_g2s(stage + (size_t)q * kRS, base + pair_col(cp, w, c) * Y.ld + row0, bytes, bar);
  }
}

struct GramParams {
  Plane Y[2];
  StepPairs sp;
  int step;
  GramWS gw;
  const int32_t* plist;  // optional: the pairs of this launch (blockIdx.x indexes it)
};

// ---------------------------------------------------------------------------
// Postmultiply [Y_p Y_q] <- [Y_p Y_q] Z~ for F, G and Z (k_post_ws below).
// ---------------------------------------------------------------------------
struct PostParams {
  Plane Y[3];
  StepPairs sp;
  int step;
  InnerOut io;
  int64_t chunk;  // rows per CTA
  int mat0;       // first matrix of the launch (blockIdx.y + mat0: 0 F, 1 G, 2 Z)
};

// ---------------------------------------------------------------------------
// Warp-specialized streaming kernels (2w = 16, 32, 64): warp 4 is the TMA producer
// (bulk loads, and for the postmultiply the bulk stores), warps 0-3 compute.
// Stages are handed over with mbarriers only -- no CTA-wide barrier inside
// the tile loop -- so DMMA work, loads and stores of different tiles overlap.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

template <int TW, bool CPLX>
struct GramWsCfg {
  static constexpr int NT = TW / 8;
  static constexpr int NTILE = NT * (NT + 1) / 2;
  static constexpr int NP = CPLX ? 2 : 1;
  static constexpr int NS = TW <= 32 ? 4 : (CPLX ? 2 : 3);  // stages within 227 KB
  static constexpr int KSTRIDE = CPLX ? 2 : 4;
  static constexpr size_t STAGE = (size_t)NP * TW * kRS;
  static constexpr size_t RED = (size_t)4 * NTILE * 64;
  static constexpr size_t BUF = NS * STAGE > RED ? NS * STAGE : RED;
  static constexpr size_t SMEM = BUF * sizeof(double) + 2 * NS * 8 + 64;
};

template <int TW, bool CPLX>
__global__ void __launch_bounds__(160, (TW == 64 && !CPLX) ? 2 : 1) k_gram_ws(GramParams P) {
  using C = GramWsCfg<TW, CPLX>;
  constexpr int NP = C::NP, NT = C::NT, NTILE = C::NTILE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stages = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::BUF * sizeof(double));
  uint64_t* empty = full + C::NS;

  const int pair = P.plist ? P.plist[blockIdx.x] : P.sp.p0 + blockIdx.x;
  const int mat = blockIdx.y, split = blockIdx.z;
  if (split >= P.gw.nsplit[mat]) return;
  const Plane& Y = P.Y[mat];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
  const int64_t L = P.gw.chunk[mat];
  const int64_t rbeg = (int64_t)split * L;
  const int64_t rend = rbeg + L < Y.rows ? rbeg + L : Y.rows;
  const int ntiles = rend > rbeg ? (int)((rend - rbeg + kR - 1) / kR) : 0;

  if (tid == 0) {
    for (int q = 0; q < C::NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 128);  // every consumer thread releases the stage it read
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 4) {  // producer
    for (int it = 0; it < ntiles; ++it) {
      const int s = it % C::NS;
      if (it >= C::NS) mbar_wait(&empty[s], (uint32_t)(((it / C::NS) - 1) & 1));
      const int64_t r0 = rbeg + (int64_t)it * kR;
      const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
      issue_tile_load<TW, NP>(Y, cp, r0, nv, stages + s * C::STAGE, &full[s], lane);
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int plane = CPLX ? (warp >> 1) : 0;
  const int ks0 = CPLX ? (warp & 1) : warp;
  double acc[NTILE][2];
#pragma unroll
  for (int q = 0; q < NTILE; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int it = 0; it < ntiles; ++it) {
    const int s = it % C::NS;
    mbar_wait(&full[s], (uint32_t)((it / C::NS) & 1));
    const double* st = stages + s * C::STAGE;
    const int64_t r0 = rbeg + (int64_t)it * kR;
    const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
#pragma unroll
    for (int ks = ks0; ks < kR / 4; ks += C::KSTRIDE) {
      const int k = ks * 4 + t;
      const bool ok = k < nv;
      double fr[NT], fi[NT];
#pragma unroll
      for (int cg = 0; cg < NT; ++cg) {
        fr[cg] = ok ? st[(size_t)(cg * 8 + g) * kRS + k] : 0.0;
        fi[cg] = (CPLX && ok) ? st[(size_t)(TW + cg * 8 + g) * kRS + k] : 0.0;
      }
      int q = 0;
#pragma unroll
      for (int I = 0; I < NT; ++I)
#pragma unroll
        for (int J = I; J < NT; ++J, ++q) {
          if (!CPLX) {
            dmma884(acc[q][0], acc[q][1], fr[I], fr[J]);
          } else if (plane == 0) {
            dmma884(acc[q][0], acc[q][1], fr[I], fr[J]);
            dmma884(acc[q][0], acc[q][1], fi[I], fi[J]);
          } else {
            dmma884(acc[q][0], acc[q][1], fr[I], fi[J]);
            dmma884(acc[q][0], acc[q][1], -fi[I], fr[J]);
          }
        }
    }
    mbar_arrive(&empty[s]);  // each thread's own reads are ordered before its arrive
  }
  consumer_bar();  // every stage consumed: reuse the buffer for the fold
  double* red = stages;
#pragma unroll
  for (int q = 0; q < NTILE; ++q) {
    red[((size_t)warp * NTILE + q) * 64 + lane * 2] = acc[q][0];
    red[((size_t)warp * NTILE + q) * 64 + lane * 2 + 1] = acc[q][1];
  }
  consumer_bar();
  double* out = P.gw.part + (((int64_t)pair * 2 + mat) * P.gw.smax + split) * NP * TW * TW;
  for (int e = tid; e < NP * NTILE * 64; e += 128) {
    const int pl = e / (NTILE * 64), rem = e % (NTILE * 64), q = rem / 64, l = (rem % 64) / 2, h = rem % 2;
    double v = 0.0;
#pragma unroll
    for (int wv = 0; wv < C::KSTRIDE; ++wv) v += red[((size_t)(pl * C::KSTRIDE + wv) * NTILE + q) * 64 + l * 2 + h];
    int I = 0, qq = q;
    while (qq >= NT - I) {
      qq -= NT - I;
      ++I;
    }
    const int J = I + qq;
    const int r = I * 8 + (l >> 2), c = J * 8 + 2 * (l & 3) + h;
    out[(size_t)pl * TW * TW + (size_t)c * TW + r] = v;
  }
}

template <int TW, bool CPLX>
struct PostWsCfg {
  static constexpr int NP = CPLX ? 2 : 1;
  static constexpr int TN = TW / 8;  // 8-column tiles, all in one warp
  static constexpr int NS = (CPLX || TW > 32) ? 2 : 3;  // 2w = 64 real: 2 CTAs per SM
  static constexpr int ZS = TW + 4;
  static constexpr size_t STAGE = (size_t)NP * TW * kRS;
  static constexpr size_t SMEM = (NS * STAGE + (size_t)NP * TW * ZS) * sizeof(double) + 2 * NS * 8 + 64;
};

template <int TW, bool CPLX>
__global__ void __launch_bounds__(160) k_post_ws(PostParams P) {
  using C = PostWsCfg<TW, CPLX>;
  constexpr int NP = C::NP;
  constexpr int w = TW / 2;
  const int pair = P.sp.p0 + blockIdx.x, mat = blockIdx.y + P.mat0;
  if (P.io.ident[pair]) return;
  const Plane& Y = P.Y[mat];
  const int64_t rbeg = (int64_t)blockIdx.z * P.chunk;
  if (rbeg >= Y.rows) return;
  const int64_t rend = rbeg + P.chunk < Y.rows ? rbeg + P.chunk : Y.rows;
  const int ntiles = (int)((rend - rbeg + kR - 1) / kR);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stages = reinterpret_cast<double*>(smem_raw);
  double* zs = stages + C::NS * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(zs + (size_t)NP * TW * C::ZS);
  uint64_t* done = full + C::NS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;

  if (tid == 0) {
    for (int q = 0; q < C::NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&done[q], 128);  // every consumer thread arrives after its own write-back
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 4) {  // producer: loads, and stores of finished tiles
    auto store_tile = [&](int it) {
      const int s = it % C::NS;
      mbar_wait(&done[s], (uint32_t)((it / C::NS) & 1));
      const int64_t r0 = rbeg + (int64_t)it * kR;
      const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
      const uint32_t bytes = (uint32_t)nv * 8u;
      const double* st = stages + s * C::STAGE;
      for (int q = lane; q < TW * NP; q += 32) {
        const int c = q % TW, pl = q / TW;
        double* base = pl == 0 ? Y.re : Y.im;
        bulk_s2g(base + pair_col(cp, w, c) * Y.ld + r0, st + (size_t)q * kRS, bytes);
      }
      bulk_commit();
    };
    for (int it = 0; it < ntiles; ++it) {
      const int s = it % C::NS;
      if (it >= C::NS) {
        store_tile(it - C::NS);
        bulk_wait_read<0>();
        __syncwarp();
      }
      const int64_t r0 = rbeg + (int64_t)it * kR;
      const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
      issue_tile_load<TW, NP>(Y, cp, r0, nv, stages + s * C::STAGE, &full[s], lane);
    }
    for (int it = ntiles > C::NS ? ntiles - C::NS : 0; it < ntiles; ++it) store_tile(it);
    bulk_wait_all<0>();
    return;
  }
  // consumers: Z~ into padded shared memory (column-major)
  const double* zsrc = P.io.zt + (int64_t)pair * NP * TW * TW;
  for (int e = tid; e < NP * TW * TW; e += 128) {
    int p = e / (TW * TW), r = e % TW, c = (e / TW) % TW;
    zs[(size_t)p * TW * C::ZS + (size_t)c * C::ZS + r] = zsrc[e];
  }
  consumer_bar();
  const int g = lane >> 2, t = lane & 3;
  // 2w = 64 real: m16n8k8 MMAs (a quarter of the instructions of m8n8k4 for
  // the same products; DMMA-bound at this width)
  constexpr bool M16 = TW == 64 && !CPLX;
  for (int it = 0; it < ntiles && M16; ++it) {
    const int s = it % C::NS;
    mbar_wait(&full[s], (uint32_t)((it / C::NS) & 1));
    double* st = stages + s * C::STAGE;
    double c[C::TN][4];
#pragma unroll
    for (int ni = 0; ni < C::TN; ++ni) c[ni][0] = c[ni][1] = c[ni][2] = c[ni][3] = 0.0;
    const int row = warp * 16 + g;
#pragma unroll 2
    for (int k0 = 0; k0 < TW; k0 += 8) {
      const double a0 = st[(size_t)(k0 + t) * kRS + row], a1 = st[(size_t)(k0 + t) * kRS + row + 8];
      const double a2 = st[(size_t)(k0 + t + 4) * kRS + row], a3 = st[(size_t)(k0 + t + 4) * kRS + row + 8];
#pragma unroll
      for (int ni = 0; ni < C::TN; ++ni) {
        const int col = ni * 8 + g;
        dmma1688(c[ni], a0, a1, a2, a3, zs[(size_t)col * C::ZS + k0 + t], zs[(size_t)col * C::ZS + k0 + t + 4]);
      }
    }
    __syncwarp();  // this warp owns its 16 rows: write them back in place
#pragma unroll
    for (int ni = 0; ni < C::TN; ++ni) {
      const int col = ni * 8 + 2 * t;
      st[(size_t)col * kRS + row] = c[ni][0];
      st[(size_t)(col + 1) * kRS + row] = c[ni][1];
      st[(size_t)col * kRS + row + 8] = c[ni][2];
      st[(size_t)(col + 1) * kRS + row + 8] = c[ni][3];
    }
    fence_proxy_async_smem();
    mbar_arrive(&done[s]);
  }
  for (int it = 0; it < ntiles && !M16; ++it) {
    const int s = it % C::NS;
    mbar_wait(&full[s], (uint32_t)((it / C::NS) & 1));
    double* st = stages + s * C::STAGE;
    double acc[NP][2][C::TN][2];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::TN; ++ni) acc[p][mi][ni][0] = acc[p][mi][ni][1] = 0.0;
#pragma unroll 2
    for (int ks = 0; ks < TW / 4; ++ks) {
      const int k = ks * 4 + t;
      double ar[2], ai[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int row = warp * 16 + mi * 8 + g;
        ar[mi] = st[(size_t)k * kRS + row];
        ai[mi] = CPLX ? st[(size_t)(TW + k) * kRS + row] : 0.0;
      }
#pragma unroll
      for (int ni = 0; ni < C::TN; ++ni) {
        const int col = ni * 8 + g;
        const double zr = zs[(size_t)col * C::ZS + k];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) dmma884(acc[0][mi][ni][0], acc[0][mi][ni][1], ar[mi], zr);
        if (CPLX) {
          const double zi = zs[(size_t)TW * C::ZS + (size_t)col * C::ZS + k];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            dmma884(acc[0][mi][ni][0], acc[0][mi][ni][1], -ai[mi], zi);
            dmma884(acc[NP - 1][mi][ni][0], acc[NP - 1][mi][ni][1], ar[mi], zi);
            dmma884(acc[NP - 1][mi][ni][0], acc[NP - 1][mi][ni][1], ai[mi], zr);
          }
        }
      }
    }
    __syncwarp();  // this warp owns its 16 rows: write them back in place
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::TN; ++ni) {
          const int row = warp * 16 + mi * 8 + g;
          const int col = ni * 8 + 2 * t;
          st[(size_t)(p * TW + col) * kRS + row] = acc[p][mi][ni][0];
          st[(size_t)(p * TW + col + 1) * kRS + row] = acc[p][mi][ni][1];
        }
    fence_proxy_async_smem();
    mbar_arrive(&done[s]);
  }
}

// ---------------------------------------------------------------------------
// Fused postmultiply (step k) + Grammian partials (step k + 1), 2w = 32 real.
//
// Pair i of step k + 1 takes one block from pair i - 1 and one from pair
// i + 1 of step k (circle positions), so walking the positions of one
// parity class in order, every two consecutive pairs hold the two blocks of
// one next-step pair.  A CTA owns one row split of F or G and a chain of
// positions p, p + 2, ..., p + 2L: for each position it streams the pair's
// row tiles through TMA, applies Z~ with DMMA (identical to k_post_ws) and
// stores them back, and -- while the tile is in shared memory -- adds the
// tile's contribution to the Grammian of the next-step pair formed with the
// previous position, whose needed half tile it kept (the carry).  The
// Grammian arithmetic is that of k_gram_ws over the same split rows, so
// the partials are bitwise those of the unfused path.  F and G are read
// once and written once per step instead of read twice.
// ---------------------------------------------------------------------------
struct PGCfg {
  static constexpr int TW = 32, W = 16;
  static constexpr int NS = 2;
  static constexpr int NT = TW / 8;
  static constexpr int NTILE = NT * (NT + 1) / 2;
  static constexpr int ZS = TW + 4;
  static constexpr int MAXT = 4;  // row tiles per split (split <= 256 rows)
  static constexpr size_t STAGE = (size_t)TW * kRS;
  static constexpr size_t CARRY = (size_t)MAXT * W * kRS;
  static constexpr size_t RED = (size_t)4 * NTILE * 64;
  static constexpr size_t SMEM = (NS * STAGE + CARRY + (size_t)TW * ZS + RED) * sizeof(double) + 2 * NS * 8 + 64;
};

struct PostGramParams {
  Plane Y[2];
  StepPairs sp;  // the current step's pairs (colpair of `step`)
  int step;
  InnerOut io;
  GramWS gw;
  PostGramTables t;
};

__global__ void __launch_bounds__(160) k_postgram(PostGramParams P) {
  using C = PGCfg;
  constexpr int TW = C::TW, W = C::W, NT = C::NT, NTILE = C::NTILE;
  const int chain = blockIdx.x, split = blockIdx.y, mat = blockIdx.z;
  if (split >= P.gw.nsplit[mat]) return;
  const Plane& Y = P.Y[mat];
  const int64_t L = P.gw.chunk[mat];
  const int64_t rbeg = (int64_t)split * L;
  const int64_t rend = rbeg + L < Y.rows ? rbeg + L : Y.rows;
  if (rend <= rbeg) return;
  const int ntiles = (int)((rend - rbeg + kR - 1) / kR);
  const int32_t* elems = P.t.chains + (int64_t)chain * (P.t.L + 1);
  const int32_t* links = P.t.links + (int64_t)chain * (P.t.L + 1) * 5;
  int nel = 0;
  while (nel <= P.t.L && elems[nel] >= 0) ++nel;
  const int total = nel * ntiles;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stages = reinterpret_cast<double*>(smem_raw);
  double* carry = stages + C::NS * C::STAGE;
  double* zs = carry + C::CARRY;
  double* red = zs + (size_t)TW * C::ZS;
  uint64_t* full = reinterpret_cast<uint64_t*>(red + C::RED);
  uint64_t* done = full + C::NS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int q = 0; q < C::NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&done[q], 128);  // every consumer thread arrives
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {  // producer: tile loads, and stores of transformed tiles
    auto store_tile = [&](int it) {
      const int s = it % C::NS;
      mbar_wait(&done[s], (uint32_t)((it / C::NS) & 1));
      const int pair = elems[it / ntiles];
      if (P.io.ident[pair]) return;  // Z~ = I: the tile is unchanged
      const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
      const int64_t r0 = rbeg + (int64_t)(it % ntiles) * kR;
      const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
      bulk_s2g(Y.re + pair_col(cp, W, lane) * Y.ld + r0, stages + s * C::STAGE + (size_t)lane * kRS,
               (uint32_t)nv * 8u);
      bulk_commit();
    };
    for (int it = 0; it < total; ++it) {
      const int s = it % C::NS;
      if (it >= C::NS) {
        store_tile(it - C::NS);
        bulk_wait_read<0>();
        __syncwarp();
      }
      const int pair = elems[it / ntiles];
      const int32_t* cp = P.sp.colpair + ((int64_t)P.step * P.sp.npairs + pair) * 2;
      const int64_t r0 = rbeg + (int64_t)(it % ntiles) * kR;
      const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
      issue_tile_load<TW, 1>(Y, cp, r0, nv, stages + s * C::STAGE, &full[s], lane);
    }
    for (int it = total > C::NS ? total - C::NS : 0; it < total; ++it) store_tile(it);
    bulk_wait_all<0>();
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  double acc[NTILE][2];
  for (int e = 0; e < nel; ++e) {
    const int pair = elems[e];
    const bool ident = P.io.ident[pair] != 0;
    // Z~ of this position (column-major, padded)
    if (!ident) {
      const double* zsrc = P.io.zt + (int64_t)pair * TW * TW;
      for (int q = tid; q < TW * TW; q += 128) zs[(q / TW) * C::ZS + q % TW] = zsrc[q];
    }
    // link e: the next-step pair made of (position e-1, position e)
    const int* lk = links + e * 5;
    const int jn = e >= 1 ? lk[0] : -1;
    // the half of this position the next link needs, kept in the carry
    const int* lk1 = links + (e + 1) * 5;
    const int hcarry = (e + 1 < nel && lk1[0] >= 0) ? (lk1[1] == 0 ? lk1[2] : lk1[4]) : -1;
#pragma unroll
    for (int q = 0; q < NTILE; ++q) acc[q][0] = acc[q][1] = 0.0;
    consumer_bar();
    for (int tt = 0; tt < ntiles; ++tt) {
      const int it = e * ntiles + tt;
      const int s = it % C::NS;
      mbar_wait(&full[s], (uint32_t)((it / C::NS) & 1));
      double* st = stages + s * C::STAGE;
      const int64_t r0 = rbeg + (int64_t)tt * kR;
      const int nv = (int)(rend - r0 < kR ? rend - r0 : kR);
      if (!ident) {  // postmultiply this warp's 16 rows (k_post_ws, real)
        double pacc[2][NT][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) pacc[mi][ni][0] = pacc[mi][ni][1] = 0.0;
#pragma unroll 2
        for (int ks = 0; ks < TW / 4; ++ks) {
          const int k = ks * 4 + t;
          double ar[2];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) ar[mi] = st[(size_t)k * kRS + warp * 16 + mi * 8 + g];
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const double zr = zs[(size_t)(ni * 8 + g) * C::ZS + k];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) dmma884(pacc[mi][ni][0], pacc[mi][ni][1], ar[mi], zr);
          }
        }
        __syncwarp();
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const int row = warp * 16 + mi * 8 + g;
            const int col = ni * 8 + 2 * t;
            st[(size_t)col * kRS + row] = pacc[mi][ni][0];
            st[(size_t)(col + 1) * kRS + row] = pacc[mi][ni][1];
          }
      }
      consumer_bar();  // the transformed tile is complete
      if (jn >= 0) {   // Grammian contribution of this tile (k_gram_ws, real)
        const double* cbase = carry + (size_t)tt * W * kRS;
        const double* colp[NT];
#pragma unroll
        for (int cg = 0; cg < NT; ++cg) {
          const int c = cg * 8 + g;              // next-pair column
          const int src = c < W ? 1 : 3;         // (elem, half) of its block
          const int cw = c % W;
          colp[cg] = lk[src] == 0 ? cbase + (size_t)cw * kRS : st + (size_t)(lk[src + 1] * W + cw) * kRS;
        }
#pragma unroll
        for (int ks = warp; ks < kR / 4; ks += 4) {
          const int k = ks * 4 + t;
          const bool ok = k < nv;
          double fr[NT];
#pragma unroll
          for (int cg = 0; cg < NT; ++cg) fr[cg] = ok ? colp[cg][k] : 0.0;
          int q = 0;
#pragma unroll
          for (int I = 0; I < NT; ++I)
#pragma unroll
            for (int J = I; J < NT; ++J, ++q) dmma884(acc[q][0], acc[q][1], fr[I], fr[J]);
        }
      }
      consumer_bar();  // carry and tile reads done
      if (hcarry >= 0) {
        double* cdst = carry + (size_t)tt * W * kRS;
        for (int q = tid; q < W * kR; q += 128) {
          const int c = q / kR, r = q % kR;
          cdst[(size_t)c * kRS + r] = st[(size_t)(hcarry * W + c) * kRS + r];
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&done[s]);
    }
    if (jn >= 0) {  // fold the warps' partials in k_gram_ws's fixed order
#pragma unroll
      for (int q = 0; q < NTILE; ++q) {
        red[((size_t)warp * NTILE + q) * 64 + lane * 2] = acc[q][0];
        red[((size_t)warp * NTILE + q) * 64 + lane * 2 + 1] = acc[q][1];
      }
      consumer_bar();
      double* out = P.gw.part + (((int64_t)jn * 2 + mat) * P.gw.smax + split) * TW * TW;
      for (int q2 = tid; q2 < NTILE * 64; q2 += 128) {
        const int q = q2 / 64, l = (q2 % 64) / 2, h = q2 % 2;
        double v = 0.0;
#pragma unroll
        for (int wv = 0; wv < 4; ++wv) v += red[((size_t)wv * NTILE + q) * 64 + l * 2 + h];
        int I = 0, qq = q;
        while (qq >= NT - I) {
          qq -= NT - I;
          ++I;
        }
        const int J = I + qq;
        const int r = I * 8 + (l >> 2), c = J * 8 + 2 * (l & 3) + h;
        out[(size_t)c * TW + r] = v;
      }
    }
    consumer_bar();  // Z~ and the fold buffer are free again
  }
}

template <typename K>
void set_smem(K k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  // the whole unified L1 / shared array as shared memory: two ~105 KB
  // stage rings per SM at 2w = 64
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

template <int TW, bool CPLX>
int gram_ws_t(const GramParams& p, cudaStream_t s) {
  using C = GramWsCfg<TW, CPLX>;
  static PerDeviceOnce once;
  if (once.first()) set_smem(k_gram_ws<TW, CPLX>, C::SMEM);
  dim3 grid(p.sp.pn, 2, p.gw.smax);
  k_gram_ws<TW, CPLX><<<grid, 160, C::SMEM, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int TW, bool CPLX>
int post_ws_t(const PostParams& p, int64_t mmax, int nmats, cudaStream_t s) {
  using C = PostWsCfg<TW, CPLX>;
  static PerDeviceOnce once;
  if (once.first()) set_smem(k_post_ws<TW, CPLX>, C::SMEM);
  dim3 grid(p.sp.pn, nmats, (unsigned)((mmax + p.chunk - 1) / p.chunk));
  k_post_ws<TW, CPLX><<<grid, 160, C::SMEM, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

bool dmma_supported(int w) { return w == 8 || w == 16 || w == 32; }

bool postgram_supported(int w, int cplx) { return w == 16 && !cplx; }

int launch_postgram(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                    const InnerOut& io, const GramWS& gw, const PostGramTables& t, cudaStream_t s) {
  if (!postgram_supported(w, cplx)) return 4;
  static PerDeviceOnce once;
  if (once.first()) set_smem(k_postgram, PGCfg::SMEM);
  PostGramParams p{{F, G}, sp, step, io, gw, t};
  dim3 grid(t.nchains, gw.smax, 2);
  k_postgram<<<grid, 160, PGCfg::SMEM, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int launch_gram_dmma(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                     const GramWS& gw, cudaStream_t s, const int32_t* plist, int npl) {
  GramParams p{{F, G}, sp, step, gw, plist};
  if (plist) {  // an explicit pair list: blockIdx.x indexes it
    if (npl <= 0) return 0;
    p.sp.pn = npl;
  }
  switch (2 * w) {
    case 16:
      return cplx ? gram_ws_t<16, true>(p, s) : gram_ws_t<16, false>(p, s);
    case 32:
      return cplx ? gram_ws_t<32, true>(p, s) : gram_ws_t<32, false>(p, s);
    case 64:
      return cplx ? gram_ws_t<64, true>(p, s) : gram_ws_t<64, false>(p, s);
  }
  return 4;
}

int launch_postmult_dmma(const Plane& F, const Plane& G, const Plane& Z, const StepPairs& sp, int step, int w,
                         int cplx, const InnerOut& io, cudaStream_t s, int mat0, int nmats) {
  int64_t mmax = 0;
  const Plane* Y[3] = {&F, &G, &Z};
  for (int q = mat0; q < mat0 + nmats; ++q) mmax = Y[q]->rows > mmax ? Y[q]->rows : mmax;
  // rows per CTA: the largest of 1024 / 2048 / 4096 that still gives a
  // whole step (all its pairs, whatever the group split) at least 2 CTAs
  // per SM (fewer, longer CTAs stream better at n = 16384: 20.33 vs 19.96
  // TFLOP/s with 4096 vs 1024; n = 4096 keeps 1024); HZG_POST_CHUNK
  // overrides (multiple of 64).  Row chunking does not change any output bit.
  const int sms = device_sms();
  int64_t chunk = 1024;
  while (chunk < 4096 && (int64_t)sp.npairs * ((mmax + 2 * chunk - 1) / (2 * chunk)) * nmats >= 2 * sms) chunk *= 2;
  if (const char* e = std::getenv("HZG_POST_CHUNK")) chunk = std::max(64, std::atoi(e)) / 64 * 64;
  PostParams p{{F, G, Z}, sp, step, io, chunk, mat0};
  switch (2 * w) {
    case 16:
      return cplx ? post_ws_t<16, true>(p, mmax, nmats, s) : post_ws_t<16, false>(p, mmax, nmats, s);
    case 32:
      return cplx ? post_ws_t<32, true>(p, mmax, nmats, s) : post_ws_t<32, false>(p, mmax, nmats, s);
    case 64:
      return cplx ? post_ws_t<64, true>(p, mmax, nmats, s) : post_ws_t<64, false>(p, mmax, nmats, s);
  }
  return 4;
}

}  // namespace hzg
