// C ABI and host-side sweep driver of libhzg.so (see include/hzg.h).
//
// One outer sweep = for every step of the outer strategy table: Grammian
// partials -> inner block kernel -> postmultiply, then the counter fold and
// the (device-gated) inter-sweep rescale.  The whole sweep is captured once
// into a CUDA graph and replayed; the host syncs once per sweep to read
// the two counters the reference's convergence test needs
// (blocked.py:531-539).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hzg.h"
#include "hzg_internal.h"
#include "hzg_nccl.h"

using namespace hzg;

struct hzg_ctx {
  int device = 0;
  int64_t mF = 0, mG = 0, n = 0;
  int64_t zrows = 0;        // rows of Z (n unless hzg_set_z_rows: a stripe slab's Z keeps the global rows)
  int cplx = 0;
  hzg_config cfg{};
  double epsn = 0;
  int w = 0, tw = 0, nblk = 0;
  int osteps = 0, npairs = 0, isteps = 0;
  bool use_dmma = false;
  bool comp = false;        // compensated dot products (odd variant ids)
  int64_t cstride = 0;      // doubles of compensated scratch per column / per thread (pow2 of the height)
  bool wavefront = false;   // schedule in circle-position order (ME)
  int groups = 1;           // position groups of the wavefront sweep graph
  // fused postmultiply(k) + Grammian(k+1) along circle-position chains
  bool fused = false;
  int pg_L = 0, pg_nchains = 0, pg_maxexc = 0;
  std::vector<int32_t> pg_chains_host;  // [osteps-1][nchains][L+1]
  std::vector<int32_t> pg_links_host;   // [osteps-1][nchains][L+1][5]
  std::vector<int32_t> pg_exc_host;     // [osteps-1][maxexc]
  std::vector<int32_t> pg_nexc;         // [osteps-1]
  std::vector<int32_t> all_pairs_host;  // 0 .. npairs-1
  int32_t* d_pg_chains = nullptr;
  int32_t* d_pg_links = nullptr;
  int32_t* d_pg_exc = nullptr;
  int32_t* d_all_pairs = nullptr;
  std::vector<cudaStream_t> gstreams;  // [G] step chains (high priority)
  std::vector<cudaStream_t> zstreams;  // [G] deferred-Z chains (low priority)
  std::vector<cudaEvent_t> gevents;    // fork, joins[G], step events [2][G], inner done [G], Z events [2][G], Z joins [G]
  // step-wise wavefront of one rank (hzg_wave_step): streams, events
  // [start, exchange tail, step events [2][G]], groups, last step run
  std::vector<cudaStream_t> wstreams, wzstreams;
  std::vector<cudaEvent_t> wevents;
  int wgroups = 0;
  int wlast = -1;
  int wfirst = 0;
  bool wdz = false;
  std::vector<int32_t> colpair_host;  // [osteps][npairs][2]
  std::vector<int32_t> itable_host;   // [isteps][tw]
  // device state
  Plane F{}, G{}, Z{};
  cudaStream_t stream = nullptr;
  cudaStream_t cap = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  unsigned char* ws = nullptr;
  int32_t* d_colpair = nullptr;
  int32_t* d_itable = nullptr;
  GramWS gw{};
  InnerOut io{};
  double* zt2 = nullptr;       // odd-step transforms (see io_of)
  int32_t* ident2 = nullptr;
  bool defer_z = false;        // Z postmultiply on its own streams, off the step chain
  int64_t* d_ctr = nullptr;    // 4 int64: total, big, status, pad
  int32_t* d_status = nullptr; // init/final status
  double* d_qr = nullptr;
  int32_t* d_qrlock = nullptr;
  int qr_slots = 0;
  int32_t* d_fin = nullptr;    // 2n int32
  double* d_sig = nullptr;     // 3n
  double* d_comp = nullptr;    // compensated-variant scratch
  int64_t* h_ctr = nullptr;    // pinned
  long long* d_phase = nullptr;
  std::string err;
  bool bound = false;
  // optional per-kernel timing (events captured into the sweep graph)
  bool timing = false;
  std::vector<cudaEvent_t> tev;  // [osteps][groups][4] (sweep graph)
  std::vector<cudaEvent_t> rev;  // [count][4] (hzg_run_steps)
  double kms[3] = {0, 0, 0};
  int64_t kcnt[3] = {0, 0, 0};
  // multi-GPU data plane (hzg_comm_*, hzg_dist_sweep): this rank's NCCL
  // communicator, its block moves per step, and the captured rank sweep
  const hzg::nccl::Api* nc = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  std::vector<int32_t> moves;     // (block, src, dst) triples that involve this rank
  std::vector<int32_t> move_off;  // [osteps + 1] offsets (in triples) per step
  cudaStream_t xstream = nullptr; // exchange stream of the rank sweep graph
  std::vector<cudaEvent_t> devents;
  cudaGraph_t dgraph = nullptr;
  cudaGraphExec_t dgexec = nullptr;
  int dgroups = 0;
  int64_t* d_red = nullptr;       // 8 int64: reduced total, big, any error, not-PD, rank, rescale status
};

namespace {

// strategies.py:45-93 (the same tables the Python layer exposes)
int gen_table(bool mm, int n, std::vector<int32_t>& out) {
  const int half = n / 2;
  out.assign((size_t)n * half * 2, 0);
  auto sort_row = [&](int st) {
    std::vector<std::pair<int, int>> v(half);
    for (int i = 0; i < half; ++i) v[i] = {out[((size_t)st * half + i) * 2], out[((size_t)st * half + i) * 2 + 1]};
    std::sort(v.begin(), v.end());
    for (int i = 0; i < half; ++i) {
      out[((size_t)st * half + i) * 2] = v[i].first;
      out[((size_t)st * half + i) * 2 + 1] = v[i].second;
    }
  };
  if (!mm) {  // round-robin tournament, strategies.py:59-70
    std::vector<int> others(n - 1);
    for (int i = 1; i < n; ++i) others[i - 1] = i;
    for (int st = 0; st < n - 1; ++st) {
      std::vector<int> line(n);
      line[0] = 0;
      for (int i = 1; i < n; ++i) line[i] = others[i - 1];
      for (int i = 0; i < half; ++i) {
        int a = line[i], b = line[n - 1 - i];
        out[((size_t)st * half + i) * 2] = std::min(a, b);
        out[((size_t)st * half + i) * 2 + 1] = std::max(a, b);
      }
      sort_row(st);
      std::rotate(others.rbegin(), others.rbegin() + 1, others.rend());
    }
    return n - 1;
  }
  // modified modulus, strategies.py:73-93
  for (int k = 0; k < n; ++k) {
    std::vector<char> seen(n, 0);
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      if (seen[i]) continue;
      int j = ((k - i) % n + n) % n;
      if (j == i || seen[j]) continue;
      seen[i] = seen[j] = 1;
      out[((size_t)k * half + cnt) * 2] = std::min(i, j);
      out[((size_t)k * half + cnt) * 2 + 1] = std::max(i, j);
      ++cnt;
    }
    if (k % 2 == 0) {
      int a = k / 2, b = a + half;
      if (!seen[a]) {
        out[((size_t)k * half + cnt) * 2] = std::min(a, b);
        out[((size_t)k * half + cnt) * 2 + 1] = std::max(a, b);
        ++cnt;
      }
    }
    sort_row(k);
  }
  return n;
}

// ME steps in circle-position order (unsorted rows of strategies.py:59-70)
int circle_table(int n, std::vector<int32_t>& out) {
  const int half = n / 2;
  out.assign((size_t)(n - 1) * half * 2, 0);
  std::vector<int> others(n - 1);
  for (int i = 1; i < n; ++i) others[i - 1] = i;
  for (int st = 0; st < n - 1; ++st) {
    std::vector<int> line(n);
    line[0] = 0;
    for (int i = 1; i < n; ++i) line[i] = others[i - 1];
    for (int i = 0; i < half; ++i) {
      int a = line[i], b = line[n - 1 - i];
      out[((size_t)st * half + i) * 2] = std::min(a, b);
      out[((size_t)st * half + i) * 2 + 1] = std::max(a, b);
    }
    std::rotate(others.rbegin(), others.rbegin() + 1, others.rend());
  }
  return n - 1;
}

int64_t pow2c(int64_t v) {
  int64_t m = 1;
  while (m < v) m <<= 1;
  return m;
}

size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

int fail(hzg_ctx* c, int code, const char* what) {
  if (c) c->err = what;
  return code;
}

int cuda_fail(hzg_ctx* c, cudaError_t e, const char* where) {
  if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
  return HZG_CUDA;
}

// Grammian split geometry per matrix height (depends on m only, never on
// the GPU count, so results are GPU-count invariant).
// rows per Grammian split in DMMA mode: hzg_config.split_rows fixes them
// (the fused postmultiply + Grammian needs <= 256); 0 = default geometry.
// A configuration field, not an environment variable: it sets the
// Grammians' summation order, i.e. the result bits.
void gram_split(int64_t m, bool exact, int64_t split_rows_cfg, int64_t npairs, int& nsplit, int64_t& chunk) {
  const int64_t kSplitRows = split_rows_cfg > 0 ? std::max<int64_t>(64, split_rows_cfg) / 64 * 64 : 0;
  if (exact) {
    int64_t P = pow2c(m);
    chunk = std::max<int64_t>(32, std::min<int64_t>(P, 2048));
    nsplit = (int)std::max<int64_t>(1, P / chunk);
  } else {
    // >= 512 rows per split CTA and at most 8 splits (partials stay a few
    // percent of the Grammian's reads), or the configured split_rows; a
    // power-of-two count, chunk a multiple of 64 rows.  Depends on m only,
    // never on the GPU count.
    nsplit = kSplitRows > 0 ? (int)pow2c((m + kSplitRows - 1) / kSplitRows)
                            : (int)std::min<int64_t>(8, pow2c((m + 511) / 512));
    // fewer, longer splits while a step still has >= 1024 Grammian CTAs
    // (npairs = the problem's pairs per step, not a rank's): fewer partials
    // to write and for the inner solve to fold (tools/sweep_time.py: n =
    // 16384, w = 32: 8 -> 2 splits +1.1 %; n = 8192, w = 32: 8 -> 4 +0.9 %;
    // n = 4096, w = 16 keeps 4+ splits: 2 were 2 % slower)
    if (kSplitRows == 0)
      while (nsplit > 1 && npairs * 2 * (nsplit / 2) >= 1024) nsplit /= 2;
    chunk = ((m + nsplit - 1) / nsplit + 63) / 64 * 64;
  }
}

struct Layout {
  size_t colpair, itable, part, zt, ident, zt2, ident2, counts, ctr, status, qr, qrlock, fin, sig, phase, comp, pg, red,
      total;
};

Layout layout(const hzg_ctx* c) {
  Layout L{};
  const int NP = c->cplx ? 2 : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += al(bytes);
    return o;
  };
  L.colpair = take((size_t)c->osteps * c->npairs * 2 * 4);
  L.itable = take((size_t)c->isteps * c->tw * 4);
  L.part = take((size_t)c->npairs * 2 * c->gw.smax * NP * c->tw * c->tw * 8);
  L.zt = take((size_t)c->npairs * NP * c->tw * c->tw * 8);
  L.ident = take((size_t)c->npairs * 4);
  // second transform buffer (odd steps): the deferred Z postmultiply of
  // step k still reads its transforms while step k+1's inner solve writes
  L.zt2 = take((size_t)c->npairs * NP * c->tw * c->tw * 8);
  L.ident2 = take((size_t)c->npairs * 4);
  L.counts = take((size_t)c->osteps * c->npairs * 4 * 4);
  L.ctr = take(4 * 8);
  L.status = take(4 * 4);
  int64_t mmax = std::max(c->mF, c->mG);
  L.qr = take((size_t)c->qr_slots * 2 * mmax * c->tw * 8);
  L.qrlock = take((size_t)c->qr_slots * 4);
  L.fin = take((size_t)2 * c->n * 4);
  L.sig = take((size_t)3 * c->n * 8);
  L.phase = take(4 * 8);
  // compensated variants: per-column scratch for the full-height norms and
  // per-thread scratch for the Grammian entries (32 threads per pair, matrix)
  size_t cs = 0;
  if (c->comp)
    cs = (size_t)c->cstride * 8 * std::max<size_t>((size_t)c->n, (size_t)c->npairs * 2 * 32);
  L.comp = take(cs);
  L.pg = take((c->pg_chains_host.size() + c->pg_links_host.size() + c->pg_exc_host.size() +
               c->all_pairs_host.size()) * 4);
  L.red = take(8 * 8);
  L.total = off;
  return L;
}

KernelCfg kernel_cfg(const hzg_ctx* c) {
  KernelCfg k{};
  const int v = c->cfg.variant_id;
  k.tw = c->tw;
  k.cplx = c->cplx;
  k.prescale = (v == 0 || v == 1 || v == 4 || v == 5);
  k.per_step_rescale = !k.prescale;
  k.compensated = v % 2 == 1;
  k.crit_c2 = v >= 4;
  k.sorting = c->cfg.sorting;
  k.max_inner_sweeps = c->cfg.max_inner_sweeps;
  k.fallback_qr = c->cfg.fallback_qr;
  k.shorten_qr = c->cfg.shorten_qr;
  k.epsn = c->epsn;
  k.approx_2x2 = !c->cfg.exact && c->cfg.approx_2x2;
  return k;
}

// Event record inside a stream capture (an external event node of the
// graph) or on a live stream.
void record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

// transforms of step `step`: even and odd steps alternate between two
// buffers, so a deferred Z postmultiply of step k can run beside step k+1
InnerOut io_of(const hzg_ctx* c, int step) {
  InnerOut o = c->io;
  if (step & 1) {
    o.zt = c->zt2;
    o.ident = c->ident2;
  }
  return o;
}

// One outer step on pairs [p0, p0 + pn): Grammian, inner solve,
// postmultiply.  defer_z: postmultiply F and G only (the caller runs
// launch_step_z for Z on another stream); inner_done: recorded after the
// inner solve.
int launch_step(hzg_ctx* c, int step, cudaStream_t s, cudaEvent_t* ev = nullptr, int p0 = 0, int pn = -1,
                bool defer_z = false, cudaEvent_t inner_done = nullptr) {
  StepPairs sp{c->d_colpair, c->npairs, p0, pn < 0 ? c->npairs : pn};
  KernelCfg kc = kernel_cfg(c);
  const InnerOut io = io_of(c, step);
  if (ev) record(ev[0], s);
  int rc = HZG_OK;
  if (c->cfg.shorten_qr) {
    // shorten == "qr": the inner kernel factors the columns itself
  } else if (c->comp) {
    rc = launch_gram_comp(c->F, c->G, sp, step, c->w, c->cplx, c->gw, c->d_comp, c->cstride, s);
  } else {
    rc = c->use_dmma ? launch_gram_dmma(c->F, c->G, sp, step, c->w, c->cplx, c->gw, s)
                     : launch_gram_exact(c->F, c->G, sp, step, c->w, c->cplx, c->gw, s);
  }
  if (rc) return rc;
  if (ev) record(ev[1], s);
  rc = launch_inner(c->F, c->G, sp, step, kc, c->gw, c->d_itable, c->isteps, io, c->d_qr, c->qr_slots,
                    c->d_qrlock, s);
  if (rc) return rc;
  if (inner_done) cudaEventRecord(inner_done, s);
  if (ev) record(ev[2], s);
  if (defer_z)
    rc = launch_postmult_dmma(c->F, c->G, c->Z, sp, step, c->w, c->cplx, io, s, 0, 2);
  else
    rc = c->use_dmma ? launch_postmult_dmma(c->F, c->G, c->Z, sp, step, c->w, c->cplx, io, s)
                     : launch_postmult_exact(c->F, c->G, c->Z, sp, step, c->w, c->cplx, io, s);
  if (rc) return rc;
  if (ev) record(ev[3], s);
  return HZG_OK;
}

// the deferred Z postmultiply of step `step` on pairs [p0, p0 + pn)
int launch_step_z(hzg_ctx* c, int step, cudaStream_t s, int p0, int pn) {
  StepPairs sp{c->d_colpair, c->npairs, p0, pn};
  return launch_postmult_dmma(c->F, c->G, c->Z, sp, step, c->w, c->cplx, io_of(c, step), s, 2, 1);
}

void accumulate_times(hzg_ctx* c) {
  if (!c->timing || c->tev.empty()) return;
  for (size_t q = 0; q < c->tev.size() / 4; ++q) {
    cudaEvent_t* e = &c->tev[q * 4];
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, e[k], e[k + 1]) == cudaSuccess) {
        c->kms[k] += ms;
        c->kcnt[k] += 1;
      } else {
        (void)cudaGetLastError();  // do not leave a stale error for the next launch check
      }
    }
  }
}

int status_code(int64_t st) {
  if (st & ST_NOT_PD) return HZG_NOT_PD;
  if (st & (ST_RANK | ST_QR_RANK)) return HZG_RANK;
  return HZG_OK;
}

// Chains of circle positions for the fused postmultiply + Grammian (see
// k_postgram): per step k < osteps-1, positions of one parity class in runs
// of L+1 (p, p+2, ..., p+2L); link e joins positions e-1 and e when they
// hold the two blocks of one pair of step k+1.  Next-step pairs no link
// covers are listed as exceptions (their Grammian runs standalone after
// the fused kernel).
void build_postgram_tables(hzg_ctx* c) {
  const int np = c->npairs, L = 16, w = c->w;
  const int per_fam = (np + 1) / 2;
  const int chains_per_fam = (per_fam + L) / (L + 1);
  c->pg_L = L;
  c->pg_nchains = 2 * chains_per_fam;
  const int S = c->osteps - 1;
  c->pg_chains_host.assign((size_t)S * c->pg_nchains * (L + 1), -1);
  c->pg_links_host.assign((size_t)S * c->pg_nchains * (L + 1) * 5, -1);
  c->pg_nexc.assign(S, 0);
  std::vector<std::vector<int32_t>> exc(S);
  std::vector<int> pos_of(c->nblk), half_of(c->nblk);
  for (int k = 0; k < S; ++k) {
    const int32_t* cur = &c->colpair_host[(size_t)k * np * 2];
    const int32_t* nxt = &c->colpair_host[(size_t)(k + 1) * np * 2];
    for (int i = 0; i < np; ++i)
      for (int h = 0; h < 2; ++h) {
        pos_of[cur[2 * i + h] / w] = i;
        half_of[cur[2 * i + h] / w] = h;
      }
    // next pair j <- unordered source positions
    std::vector<int> covered(np, 0);
    auto find_next = [&](int pa, int pb) {
      for (int j = std::max(0, std::min(pa, pb) - 2); j <= std::min(np - 1, std::max(pa, pb) + 2); ++j) {
        const int s0 = pos_of[nxt[2 * j] / w], s1 = pos_of[nxt[2 * j + 1] / w];
        if ((s0 == pa && s1 == pb) || (s0 == pb && s1 == pa)) return j;
      }
      return -1;
    };
    for (int fam = 0; fam < 2; ++fam)
      for (int t = 0; t < chains_per_fam; ++t) {
        const int ch = fam * chains_per_fam + t;
        int32_t* el = &c->pg_chains_host[((size_t)k * c->pg_nchains + ch) * (L + 1)];
        int32_t* lk = &c->pg_links_host[((size_t)k * c->pg_nchains + ch) * (L + 1) * 5];
        for (int e = 0; e <= L; ++e) {
          const int pos = fam + 2 * (t * (L + 1) + e);
          if (pos >= np) break;
          el[e] = pos;
          if (e == 0) continue;
          const int j = find_next(el[e - 1], pos);
          if (j < 0 || covered[j]) continue;
          covered[j] = 1;
          const int b0 = nxt[2 * j] / w, b1 = nxt[2 * j + 1] / w;
          lk[e * 5 + 0] = j;
          lk[e * 5 + 1] = pos_of[b0] == pos ? 1 : 0;
          lk[e * 5 + 2] = half_of[b0];
          lk[e * 5 + 3] = pos_of[b1] == pos ? 1 : 0;
          lk[e * 5 + 4] = half_of[b1];
        }
      }
    for (int j = 0; j < np; ++j)
      if (!covered[j]) exc[k].push_back(j);
    c->pg_nexc[k] = (int)exc[k].size();
    c->pg_maxexc = std::max(c->pg_maxexc, c->pg_nexc[k]);
  }
  c->pg_exc_host.assign((size_t)S * std::max(1, c->pg_maxexc), 0);
  for (int k = 0; k < S; ++k)
    for (size_t q = 0; q < exc[k].size(); ++q) c->pg_exc_host[(size_t)k * std::max(1, c->pg_maxexc) + q] = exc[k][q];
  c->all_pairs_host.resize(np);
  for (int i = 0; i < np; ++i) c->all_pairs_host[i] = i;
}

// Cross-rank reduction vector of one rank sweep (hzg_dist_sweep): the
// integer counters, and the status bits as per-kind indicators (NCCL has no
// bitwise-or reduction; a sum of indicators is exact and order-free)
__global__ void k_red_pack(const int64_t* ctr, int64_t* red) {
  if (threadIdx.x != 0) return;
  const int64_t st = ctr[2];
  red[0] = ctr[0];
  red[1] = ctr[1];
  red[2] = st != 0;
  red[3] = (st & ST_NOT_PD) != 0;
  red[4] = (st & (ST_RANK | ST_QR_RANK)) != 0;
}

__global__ void k_red_status(const int32_t* status, int64_t* red) {
  if (threadIdx.x == 0) red[5] = status[0] != 0;
}

}  // namespace

extern "C" {

int hzg_create(hzg_ctx** out, int device, int64_t mF, int64_t mG, int64_t n, int32_t is_complex,
               const hzg_config* cfg, double epsn) {
  if (!out || !cfg) return HZG_INVALID;
  *out = nullptr;
  const int w = cfg->block_width;
  if (w < 1 || n < 2 * w || n % (2 * w) != 0 || mF % (2 * w) != 0 || mG % (2 * w) != 0 || mF < 1 || mG < 1)
    return HZG_INVALID;
  if (cfg->variant_id < 0 || cfg->variant_id > 7) return HZG_INVALID;
  if (2 * w > 64 || (2 * w > 32 && 2 * w != 48 && 2 * w != 64)) return HZG_INVALID;
  static const int supported[] = {2, 4, 6, 8, 10, 12, 14, 16, 20, 24, 32, 48, 64};
  bool ok = false;
  for (int t : supported) ok |= (t == 2 * w);
  if (!ok) return HZG_INVALID;
  if (n / w > 65534) return HZG_INVALID;
  hzg_ctx* c = new hzg_ctx();
  c->device = device;
  c->mF = mF;
  c->mG = mG;
  c->n = n;
  c->cplx = is_complex ? 1 : 0;
  c->cfg = *cfg;
  if (c->cfg.max_inner_sweeps <= 0) c->cfg.max_inner_sweeps = 30;
  c->epsn = epsn > 0 ? epsn : cfg->gate_eps * std::sqrt((double)n);
  c->w = w;
  c->tw = 2 * w;
  c->nblk = (int)(n / w);
  c->npairs = c->nblk / 2;
  c->use_dmma = !cfg->exact && dmma_supported(w);
  c->comp = cfg->variant_id % 2 == 1;
  c->cstride = pow2c(std::max(std::max(mF, mG), n));
  std::vector<int32_t> outer;
  if (cfg->outer_mm) {
    c->osteps = gen_table(true, c->nblk, outer);
  } else {
    // ME pair sets in circle-method position order (strategies.py:59-70
    // before the per-step sort): pair i of step k is (line[i], line[N-1-i]).
    // Same pairs as the reference's sorted table; the position order makes
    // step k+1's pair i depend only on step k's pairs i-1 .. i+1, which the
    // sweep graph exploits (groups of positions run as a wavefront).
    c->osteps = circle_table(c->nblk, outer);
    c->wavefront = true;
  }
  c->colpair_host.resize((size_t)c->osteps * c->npairs * 2);
  for (size_t e = 0; e < c->colpair_host.size(); ++e) c->colpair_host[e] = outer[e] * w;
  std::vector<int32_t> inner;
  c->isteps = gen_table(cfg->inner_mm != 0, c->tw, inner);
  c->itable_host.assign(inner.begin(), inner.begin() + (size_t)c->isteps * c->tw);
  for (int mat = 0; mat < 2; ++mat)
    gram_split(mat == 0 ? mF : mG, !c->use_dmma, cfg->split_rows, c->npairs, c->gw.nsplit[mat], c->gw.chunk[mat]);
  if (c->comp) {  // the compensated Grammian is one sequential form over the full height
    c->gw.nsplit[0] = c->gw.nsplit[1] = 1;
    c->gw.chunk[0] = mF;
    c->gw.chunk[1] = mG;
  }
  c->gw.smax = std::max(c->gw.nsplit[0], c->gw.nsplit[1]);
  // fused postmultiply + Grammian: DMMA mode, real, w = 16, the ME circle
  // schedule of a single rank, splits of at most 256 rows.  Opt-in
  // (HZG_FUSED=1 with SolverConfig(split_rows=256)): bitwise equal to the separate
  // kernels, but measured slower on B200 so far (profiles/r01_fused.txt)
  {
    const char* env = std::getenv("HZG_FUSED");
    const bool want = env && std::atoi(env) != 0;
    c->fused = want && c->use_dmma && !c->comp && !cfg->shorten_qr && c->wavefront &&
               postgram_supported(w, c->cplx) && c->osteps >= 2 && c->gw.chunk[0] <= 256 && c->gw.chunk[1] <= 256;
    if (c->fused) build_postgram_tables(c);
  }

  // QR scratch slots: one per pair when every pair is shortened by QR,
  // otherwise a few shared by the rare Cholesky failures
  c->qr_slots = cfg->shorten_qr ? c->npairs : (int)std::max<int64_t>(1, std::min<int64_t>(16, c->npairs));
  *out = c;
  return HZG_OK;
}

size_t hzg_workspace_bytes(const hzg_ctx* c) { return c ? layout(c).total : 0; }

int hzg_set_schedule(hzg_ctx* c, const int32_t* colpairs, int32_t osteps, int32_t npairs) {
  if (!c || !colpairs || osteps < 1 || npairs < 1 || npairs > c->nblk / 2) return HZG_INVALID;
  if (c->bound) return fail(c, HZG_INVALID, "hzg_set_schedule must precede hzg_bind");
  c->osteps = osteps;
  c->npairs = npairs;
  c->colpair_host.assign(colpairs, colpairs + (size_t)osteps * npairs * 2);
  c->wavefront = false;
  c->fused = false;
  c->pg_chains_host.clear();
  c->pg_links_host.clear();
  c->pg_exc_host.clear();
  c->all_pairs_host.clear();
  c->qr_slots = c->cfg.shorten_qr ? npairs : std::max(1, std::min(16, npairs));
  return HZG_OK;
}

int hzg_set_z_rows(hzg_ctx* c, int64_t zrows) {
  if (!c || zrows < c->n) return HZG_INVALID;
  if (c->bound) return fail(c, HZG_INVALID, "hzg_set_z_rows must precede hzg_bind");
  c->zrows = zrows;
  return HZG_OK;
}

int hzg_bind(hzg_ctx* c, double* Fr, double* Fi, double* Gr, double* Gi, double* Zr, double* Zi, void* workspace,
             void* stream) {
  if (!c || !Fr || !Gr || !Zr || !workspace) return HZG_INVALID;
  if (c->cplx && (!Fi || !Gi || !Zi)) return fail(c, HZG_INVALID, "complex problem needs imaginary planes");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  c->F = Plane{Fr, c->cplx ? Fi : nullptr, c->mF, c->mF};
  c->G = Plane{Gr, c->cplx ? Gi : nullptr, c->mG, c->mG};
  const int64_t zr = c->zrows > 0 ? c->zrows : c->n;
  c->Z = Plane{Zr, c->cplx ? Zi : nullptr, zr, zr};
  c->stream = (cudaStream_t)stream;
  Layout L = layout(c);
  c->ws = (unsigned char*)workspace;
  c->d_colpair = (int32_t*)(c->ws + L.colpair);
  c->d_itable = (int32_t*)(c->ws + L.itable);
  c->gw.part = (double*)(c->ws + L.part);
  c->io.zt = (double*)(c->ws + L.zt);
  c->io.ident = (int32_t*)(c->ws + L.ident);
  c->zt2 = (double*)(c->ws + L.zt2);
  c->ident2 = (int32_t*)(c->ws + L.ident2);
  c->io.counts = (int32_t*)(c->ws + L.counts);
  c->d_ctr = (int64_t*)(c->ws + L.ctr);
  c->d_status = (int32_t*)(c->ws + L.status);
  c->d_qr = (double*)(c->ws + L.qr);
  c->d_qrlock = (int32_t*)(c->ws + L.qrlock);
  c->d_fin = (int32_t*)(c->ws + L.fin);
  c->d_sig = (double*)(c->ws + L.sig);
  c->d_phase = (long long*)(c->ws + L.phase);
  c->d_comp = c->comp ? (double*)(c->ws + L.comp) : nullptr;
  c->d_red = (int64_t*)(c->ws + L.red);
  c->io.phase = nullptr;
  if ((e = cudaMemcpyAsync(c->d_colpair, c->colpair_host.data(), c->colpair_host.size() * 4,
                           cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "upload schedule");
  if ((e = cudaMemcpyAsync(c->d_itable, c->itable_host.data(), c->itable_host.size() * 4, cudaMemcpyHostToDevice,
                           c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "upload inner table");
  if (c->fused) {
    int32_t* base = (int32_t*)(c->ws + L.pg);
    c->d_pg_chains = base;
    c->d_pg_links = c->d_pg_chains + c->pg_chains_host.size();
    c->d_pg_exc = c->d_pg_links + c->pg_links_host.size();
    c->d_all_pairs = c->d_pg_exc + c->pg_exc_host.size();
    cudaMemcpyAsync(c->d_pg_chains, c->pg_chains_host.data(), c->pg_chains_host.size() * 4, cudaMemcpyHostToDevice,
                    c->stream);
    cudaMemcpyAsync(c->d_pg_links, c->pg_links_host.data(), c->pg_links_host.size() * 4, cudaMemcpyHostToDevice,
                    c->stream);
    cudaMemcpyAsync(c->d_pg_exc, c->pg_exc_host.data(), c->pg_exc_host.size() * 4, cudaMemcpyHostToDevice,
                    c->stream);
    cudaMemcpyAsync(c->d_all_pairs, c->all_pairs_host.data(), c->all_pairs_host.size() * 4, cudaMemcpyHostToDevice,
                    c->stream);
  }
  cudaMemsetAsync(c->d_qrlock, 0, (size_t)c->qr_slots * 4, c->stream);
  cudaMemsetAsync(c->io.counts, 0, (size_t)c->osteps * c->npairs * 16, c->stream);
  if (!c->h_ctr) {
    if ((e = cudaMallocHost(&c->h_ctr, 8 * 8)) != cudaSuccess) return cuda_fail(c, e, "cudaMallocHost");
  }
  if (!c->cap) {
    if ((e = cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(c, e, "cudaStreamCreate");
  }
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "bind sync");
  if (c->gexec) {
    cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
  }
  if (c->graph) {
    cudaGraphDestroy(c->graph);
    c->graph = nullptr;
  }
  c->bound = true;
  return HZG_OK;
}

int hzg_init_fgz(hzg_ctx* c) {
  if (!c || !c->bound) return HZG_INVALID;
  cudaError_t e;
  const size_t zb = (size_t)c->Z.rows * c->n * 8;
  cudaMemsetAsync(c->Z.re, 0, zb, c->stream);
  if (c->Z.im) cudaMemsetAsync(c->Z.im, 0, zb, c->stream);
  cudaMemsetAsync(c->d_status, 0, 16, c->stream);
  KernelCfg kc = kernel_cfg(c);
  int rc = launch_prescale(c->F, c->G, c->Z, c->n, c->cplx, kc.prescale, c->d_status, c->comp ? c->d_comp : nullptr,
                           c->cstride, c->stream);
  if (rc) return fail(c, rc, "prescale launch");
  int32_t st = 0;
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "status copy");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "prescale");
  std::memcpy(&st, c->h_ctr, 4);
  if (st) return fail(c, HZG_RANK, "zero G column during prescaling");
  return HZG_OK;
}

// first pair of position group g of G (g = G: npairs).  The two end groups
// hold the circle positions whose pairs need the most inner sweeps; with
// HZG_GROUP_END_WEIGHT = f they get f times an interior group's share
// (default 1: equal groups).
static int group_cut(int npairs, int G, int g) {
  static double f = -1.0;
  if (f < 0) {
    const char* e = std::getenv("HZG_GROUP_END_WEIGHT");
    f = e ? std::max(0.05, std::atof(e)) : 1.0;
  }
  if (g <= 0) return 0;
  if (g >= G) return npairs;
  if (G < 3 || f == 1.0 || npairs < 4 * G) return (int)((int64_t)npairs * g / G);
  const double tot = 2 * f + (G - 2);
  const double acc = f + (g - 1);
  int cut = (int)std::lround(npairs * acc / tot);
  // every group keeps at least one pair
  return std::min(std::max(cut, g), npairs - (G - g));
}

static int choose_groups(const hzg_ctx* c) {
  if (!c->wavefront) return 1;
  // 4 pairs per group, at most 16 groups (tools/wtime.py, HZG_GROUPS
  // sweep, round 2): config 4 (128 pairs) 8.20 / 8.00 / 7.90 / 7.76 s for
  // 8 / 16 / 32 / 64 groups steady state, 8.77 / 8.51 / 8.99 / 8.87 s on
  // the first call (graph capture + instantiation grow with the groups);
  // config 3 (64 pairs) 1.31 / 1.25 / 1.20 s for 4 / 8 / 16 groups (1.19 s
  // with this rule); n =
  // 16384, w = 32 (256 pairs) and config 2 within noise for 8 vs 16 / 2-8
  int g = std::max(1, std::min(16, c->npairs / 4));
  if (const char* e = std::getenv("HZG_GROUPS")) g = std::max(1, std::min(c->npairs, std::atoi(e)));
  return g;
}

// One outer sweep as a CUDA graph.  With G > 1 the pairs of every step are
// split into G contiguous circle-position groups, each on its own capture
// stream; group g of step k+1 waits only for groups g-1, g, g+1 of step k
// (the pairs its blocks come from), so Grammian / postmultiply streaming of
// some groups overlaps the latency-bound inner solves of others.
// grow a pool of non-blocking streams to n; chain streams get the highest
// scheduling priority and deferred-Z streams the lowest (HZG_PRIO=0: all
// default), so the Z postmultiply fills the SMs and bandwidth the step chain
// leaves idle (mostly during the latency-bound inner solves)
static int stream_pool(hzg_ctx* c, std::vector<cudaStream_t>& pool, int n, bool high) {
  static int use = -1;
  if (use < 0) {
    const char* e = std::getenv("HZG_PRIO");
    use = e ? std::atoi(e) : 1;
  }
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  while ((int)pool.size() < n) {
    cudaStream_t st;
    cudaError_t e = cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, use ? (high ? greatest : least) : 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamCreate");
    pool.push_back(st);
  }
  return HZG_OK;
}

static bool want_defer_z(const hzg_ctx* c) {
  // the Z postmultiply leaves the step chain (F, G feed the next step's
  // Grammians, Z only its own later updates): DMMA mode, unfused, untimed
  const char* e = std::getenv("HZG_DEFER_Z");
  return c->use_dmma && !c->fused && !c->timing && !(e && std::atoi(e) == 0);
}

static int build_graph(hzg_ctx* c) {
  cudaError_t e;
  const int G = c->groups = choose_groups(c);
  const bool dz = c->defer_z = want_defer_z(c);
  if (int rc = stream_pool(c, c->gstreams, G, true)) return rc;
  if (int rc = stream_pool(c, c->zstreams, dz ? G : 0, false)) return rc;
  const size_t nev = 1 + (size_t)G + 2 * (size_t)G + 4 * (size_t)G;
  while (c->gevents.size() < nev) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(c, e, "cudaEventCreate");
    c->gevents.push_back(ev);
  }
  cudaEvent_t fork = c->gevents[0];
  cudaEvent_t* join = &c->gevents[1];
  cudaEvent_t* stepev = &c->gevents[1 + G];  // [2][G]
  cudaEvent_t* idone = &c->gevents[1 + 3 * G];  // [G]
  cudaEvent_t* zev = &c->gevents[1 + 4 * G];    // [2][G]
  cudaEvent_t* zjoin = &c->gevents[1 + 6 * G];  // [G]
  if (c->timing && c->tev.empty()) {
    c->tev.resize((size_t)c->osteps * G * 4);
    for (auto& ev : c->tev) cudaEventCreate(&ev);
  }
  if ((e = cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return cuda_fail(c, e, "begin capture");
  int rc = HZG_OK;
  if (c->fused) {
    // step 0's Grammian, then per step: inner -> fused postmultiply of F, G
    // with the next step's Grammian partials, postmultiply of Z, Grammian of
    // the next-step pairs no chain link covers
    cudaStream_t s = c->cap;
    StepPairs all{c->d_colpair, c->npairs, 0, c->npairs};
    KernelCfg kc = kernel_cfg(c);
    rc = launch_gram_dmma(c->F, c->G, all, 0, c->w, c->cplx, c->gw, s);
    for (int st = 0; st < c->osteps && rc == HZG_OK; ++st) {
      rc = launch_inner(c->F, c->G, all, st, kc, c->gw, c->d_itable, c->isteps, c->io, c->d_qr, c->qr_slots,
                        c->d_qrlock, s);
      if (rc) break;
      if (st + 1 < c->osteps) {
        const size_t L1 = (size_t)c->pg_L + 1;
        PostGramTables tb{c->d_pg_chains + (size_t)st * c->pg_nchains * L1,
                          c->d_pg_links + (size_t)st * c->pg_nchains * L1 * 5, c->pg_nchains, c->pg_L};
        rc = launch_postgram(c->F, c->G, all, st, c->w, c->cplx, c->io, c->gw, tb, s);
        if (!rc) rc = launch_postmult_dmma(c->F, c->G, c->Z, all, st, c->w, c->cplx, c->io, s, 2, 1);
        if (!rc && c->pg_nexc[st] > 0)
          rc = launch_gram_dmma(c->F, c->G, all, st + 1, c->w, c->cplx, c->gw, s,
                                c->d_pg_exc + (size_t)st * std::max(1, c->pg_maxexc), c->pg_nexc[st]);
      } else {
        rc = launch_postmult_dmma(c->F, c->G, c->Z, all, st, c->w, c->cplx, c->io, s);
      }
    }
  }
  cudaEventRecord(fork, c->cap);
  for (int g = 0; g < G; ++g) cudaStreamWaitEvent(c->gstreams[g], fork, 0);
  for (int st = 0; st < c->osteps && rc == HZG_OK && !c->fused; ++st) {
    for (int g = 0; g < G && rc == HZG_OK; ++g) {
      cudaStream_t s = c->gstreams[g];
      if (st > 0) {
        if (g > 0) cudaStreamWaitEvent(s, stepev[((st - 1) & 1) * G + g - 1], 0);
        if (g + 1 < G) cudaStreamWaitEvent(s, stepev[((st - 1) & 1) * G + g + 1], 0);
      }
      // the inner solve of step st overwrites the transforms the deferred
      // Z postmultiply of step st - 2 (same pairs) reads
      if (dz && st >= 2) cudaStreamWaitEvent(s, zev[(st & 1) * G + g], 0);
      const int p0 = group_cut(c->npairs, G, g), p1 = group_cut(c->npairs, G, g + 1);
      rc = launch_step(c, st, s, c->timing ? &c->tev[((size_t)st * G + g) * 4] : nullptr, p0, p1 - p0, dz,
                       dz ? idone[g] : nullptr);
      cudaEventRecord(stepev[(st & 1) * G + g], s);
      if (dz && rc == HZG_OK) {
        // Z chain of the group: its transforms, and the Z blocks of groups
        // g-1 .. g+1 from the previous step
        cudaStream_t z = c->zstreams[g];
        cudaStreamWaitEvent(z, idone[g], 0);
        if (st > 0)
          for (int h = g - 1; h <= g + 1; ++h)
            if (h >= 0 && h < G) cudaStreamWaitEvent(z, zev[((st - 1) & 1) * G + h], 0);
        rc = launch_step_z(c, st, z, p0, p1 - p0);
        cudaEventRecord(zev[(st & 1) * G + g], z);
      }
    }
  }
  for (int g = 0; g < G; ++g) {
    cudaEventRecord(join[g], c->gstreams[g]);
    cudaStreamWaitEvent(c->cap, join[g], 0);
    if (dz) {
      cudaEventRecord(zjoin[g], c->zstreams[g]);
      cudaStreamWaitEvent(c->cap, zjoin[g], 0);
    }
  }
  if (rc == HZG_OK) rc = launch_counters(c->io.counts, (int64_t)c->osteps * c->npairs, c->d_ctr, c->cap);
  if (rc == HZG_OK)
    rc = launch_rescale(c->F, c->G, c->Z, c->n, c->cplx, 0, nullptr, nullptr, nullptr, c->d_ctr, c->d_status,
                        c->comp ? c->d_comp : nullptr, c->cstride, c->cap);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(c->cap, &g);
  if (rc != HZG_OK) {
    if (g) cudaGraphDestroy(g);
    return fail(c, rc, "kernel launch during capture");
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "end capture");
  c->graph = g;
  // honour the captured per-node priorities (chain vs deferred Z)
  if ((e = cudaGraphInstantiate(&c->gexec, g, cudaGraphInstantiateFlagUseNodePriority)) != cudaSuccess)
    return cuda_fail(c, e, "graph instantiate");
  return HZG_OK;
}

int hzg_sweep_launch(hzg_ctx* c) {
  if (!c || !c->bound) return HZG_INVALID;
  cudaError_t e;
  if (!c->gexec) {
    int rc = build_graph(c);
    if (rc) return rc;
  }
  if ((e = cudaGraphLaunch(c->gexec, c->stream)) != cudaSuccess) return cuda_fail(c, e, "graph launch");
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_ctr, 3 * 8, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "counter copy");
  if ((e = cudaMemcpyAsync(c->h_ctr + 3, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "status copy");
  return HZG_OK;
}

int hzg_sweep_wait(hzg_ctx* c, int64_t* total, int64_t* big) {
  if (!c || !c->bound) return HZG_INVALID;
  cudaError_t e;
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "sweep");
  accumulate_times(c);
  if (total) *total = c->h_ctr[0];
  if (big) *big = c->h_ctr[1];
  int rc = status_code(c->h_ctr[2]);
  if (rc == HZG_NOT_PD) return fail(c, rc, "indefinite block Grammian; enable the QR fallback");
  if (rc == HZG_RANK) return fail(c, rc, "rank-deficient block pair in the inner solve");
  int32_t st = 0;
  std::memcpy(&st, c->h_ctr + 3, 4);
  if (st) return fail(c, HZG_RANK, "zero pencil column between sweeps");
  return HZG_OK;
}

int hzg_sweep(hzg_ctx* c, int64_t* total, int64_t* big) {
  int rc = hzg_sweep_launch(c);
  return rc ? rc : hzg_sweep_wait(c, total, big);
}

int hzg_run_steps(hzg_ctx* c, int32_t first, int32_t count) {
  if (!c || !c->bound || first < 0 || count < 0 || first + count > c->osteps) return HZG_INVALID;
  // with timing on, every kernel is bracketed by events on the launch
  // stream and the call is synchronous (isolated per-kernel durations)
  if (c->timing && c->rev.size() < (size_t)count * 4) {
    size_t old = c->rev.size();
    c->rev.resize((size_t)count * 4);
    for (size_t e = old; e < c->rev.size(); ++e) cudaEventCreate(&c->rev[e]);
  }
  for (int s = first; s < first + count; ++s) {
    int rc = launch_step(c, s, c->stream, c->timing ? &c->rev[(size_t)(s - first) * 4] : nullptr);
    if (rc) return fail(c, rc, "step launch");
  }
  if (c->timing) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "run_steps");
    for (int q = 0; q < count; ++q) {
      cudaEvent_t* ev = &c->rev[(size_t)q * 4];
      for (int k = 0; k < 3; ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev[k], ev[k + 1]) == cudaSuccess) {
          c->kms[k] += ms;
          c->kcnt[k] += 1;
        } else {
          (void)cudaGetLastError();
        }
      }
    }
  }
  return HZG_OK;
}

int hzg_run_pairs(hzg_ctx* c, int32_t step, int32_t p0, int32_t pn, void* stream) {
  if (!c || !c->bound || step < 0 || step >= c->osteps || p0 < 0 || pn < 0 || p0 + pn > c->npairs)
    return HZG_INVALID;
  if (pn == 0) return HZG_OK;
  int rc = launch_step(c, step, stream ? (cudaStream_t)stream : c->stream, nullptr, p0, pn);
  return rc ? fail(c, rc, "step launch") : HZG_OK;
}

int hzg_wave_step(hzg_ctx* c, int32_t step, int32_t groups, void* comm, void* zcomm) {
  if (!c || !c->bound || step < 0 || step >= c->osteps || groups < 1) return HZG_INVALID;
  cudaError_t e;
  const int G = std::min<int>(groups, c->npairs);
  if (int rc = stream_pool(c, c->wstreams, G, true)) return rc;
  if (int rc = stream_pool(c, c->wzstreams, G, false)) return rc;
  while (c->wevents.size() < 3 + 5 * (size_t)G) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(c, e, "cudaEventCreate");
    c->wevents.push_back(ev);
  }
  cudaStream_t cs = comm ? (cudaStream_t)comm : c->stream;
  cudaEvent_t start = c->wevents[0], xtail = c->wevents[1];
  cudaEvent_t* sev = &c->wevents[2];           // [2][G] step chains
  cudaEvent_t* idone = &c->wevents[2 + 2 * G];  // [G] inner solves done
  cudaEvent_t* zev = &c->wevents[2 + 3 * G];    // [2][G] deferred-Z chains
  cudaEvent_t ztail = c->wevents[2 + 5 * G];
  // deferred Z in the step-wise wavefront: opt-in (HZG_WAVE_DEFER_Z=1); on
  // one rank's share (tools/rank_share.py) it measured slower at 2-4 ranks
  // of n = 16384 and even at 8
  const char* wdz_env = std::getenv("HZG_WAVE_DEFER_Z");
  const bool dz = want_defer_z(c) && wdz_env && std::atoi(wdz_env) != 0;
  // zcomm: the Z blocks travel in their own exchange (off the step chain
  // when the Z postmultiply is deferred)
  cudaStream_t zs = zcomm ? (cudaStream_t)zcomm : nullptr;
  // a new chain (first step of a sweep, or a different group count or
  // deferral) starts after everything already queued on the bound stream
  const bool fresh = step == 0 || c->wgroups != G || c->wlast != step - 1 || c->wdz != dz;
  if (fresh) {
    cudaEventRecord(start, c->stream);
    c->wfirst = step;
  }
  // the block exchange of the previous step, queued on the comm stream
  cudaEventRecord(xtail, cs);
  if (zs) cudaEventRecord(ztail, zs);
  for (int g = 0; g < G; ++g) {
    cudaStream_t s = c->wstreams[g];
    if (fresh) {
      cudaStreamWaitEvent(s, start, 0);
    } else {
      for (int h = g - 1; h <= g + 1; ++h)
        if (h >= 0 && h < G) cudaStreamWaitEvent(s, sev[((step - 1) & 1) * G + h], 0);
    }
    if (g == 0 || g == G - 1) {
      cudaStreamWaitEvent(s, xtail, 0);
      if (zs && !dz) cudaStreamWaitEvent(s, ztail, 0);  // this chain's postmultiply writes Z
    }
    // transforms of step - 2 (same buffer) read by its deferred Z postmultiply
    if (dz && step - 2 >= c->wfirst) cudaStreamWaitEvent(s, zev[(step & 1) * G + g], 0);
    const int p0 = group_cut(c->npairs, G, g), p1 = group_cut(c->npairs, G, g + 1);
    int rc = launch_step(c, step, s, nullptr, p0, p1 - p0, dz, dz ? idone[g] : nullptr);
    if (rc) return fail(c, rc, "step launch");
    cudaEventRecord(sev[(step & 1) * G + g], s);
    if (dz) {
      cudaStream_t z = c->wzstreams[g];
      cudaStreamWaitEvent(z, idone[g], 0);
      if (zs && (g == 0 || g == G - 1)) cudaStreamWaitEvent(z, ztail, 0);
      if (step - 1 >= c->wfirst)
        for (int h = g - 1; h <= g + 1; ++h)
          if (h >= 0 && h < G) cudaStreamWaitEvent(z, zev[((step - 1) & 1) * G + h], 0);
      if ((rc = launch_step_z(c, step, z, p0, p1 - p0))) return fail(c, rc, "step launch");
      cudaEventRecord(zev[(step & 1) * G + g], z);
    }
  }
  // the next exchange (queued on comm by the caller) reads the end groups'
  // blocks of F, G and Z
  for (int g : {0, G - 1}) {
    cudaStreamWaitEvent(cs, sev[(step & 1) * G + g], 0);
    if (dz) cudaStreamWaitEvent(zs ? zs : cs, zev[(step & 1) * G + g], 0);
    else if (zs) cudaStreamWaitEvent(zs, sev[(step & 1) * G + g], 0);
  }
  c->wgroups = G;
  c->wlast = step;
  c->wdz = dz;
  return HZG_OK;
}

int hzg_wave_join(hzg_ctx* c, void* comm, void* zcomm) {
  if (!c || !c->bound) return HZG_INVALID;
  if (c->wlast < 0) return HZG_OK;
  const int G = c->wgroups;
  cudaStream_t cs = comm ? (cudaStream_t)comm : c->stream;
  for (int g = 0; g < G; ++g) {
    cudaStreamWaitEvent(c->stream, c->wevents[2 + (c->wlast & 1) * G + g], 0);
    if (c->wdz) cudaStreamWaitEvent(c->stream, c->wevents[2 + 3 * G + (c->wlast & 1) * G + g], 0);
  }
  cudaEventRecord(c->wevents[1], cs);
  cudaStreamWaitEvent(c->stream, c->wevents[1], 0);
  if (zcomm) {
    cudaEventRecord(c->wevents[2 + 5 * G], (cudaStream_t)zcomm);
    cudaStreamWaitEvent(c->stream, c->wevents[2 + 5 * G], 0);
  }
  c->wlast = -1;
  return HZG_OK;
}

int hzg_collect(hzg_ctx* c, int64_t* total, int64_t* big) {
  if (!c || !c->bound) return HZG_INVALID;
  cudaError_t e;
  int rc = launch_counters(c->io.counts, (int64_t)c->osteps * c->npairs, c->d_ctr, c->stream);
  if (rc) return fail(c, rc, "counter fold launch");
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_ctr, 3 * 8, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "counter copy");
  if ((e = cudaMemcpyAsync(c->h_ctr + 3, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "status copy");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "collect");
  if (total) *total = c->h_ctr[0];
  if (big) *big = c->h_ctr[1];
  rc = status_code(c->h_ctr[2]);
  if (rc == HZG_NOT_PD) return fail(c, rc, "indefinite block Grammian; enable the QR fallback");
  if (rc == HZG_RANK) return fail(c, rc, "rank-deficient block pair in the inner solve");
  int32_t st = 0;
  std::memcpy(&st, c->h_ctr + 3, 4);
  if (st) return fail(c, HZG_RANK, "zero pencil column between sweeps");
  return HZG_OK;
}

int hzg_rescale_z(hzg_ctx* c) {
  if (!c || !c->bound) return HZG_INVALID;
  int rc = launch_rescale(c->F, c->G, c->Z, c->n, c->cplx, 0, nullptr, nullptr, nullptr, nullptr, c->d_status,
                          c->comp ? c->d_comp : nullptr, c->cstride, c->stream);
  return rc ? fail(c, rc, "rescale launch") : HZG_OK;
}

int hzg_finalize(hzg_ctx* c, int64_t n0, int64_t mF0, int64_t mG0, int32_t sort, double* Ur, double* Ui, double* Vr,
                 double* Vi, double* Zr, double* Zi, double* sigF, double* sigG, double* sig) {
  if (!c || !c->bound || n0 < 1 || n0 > c->n || mF0 > c->mF || mG0 > c->mG) return HZG_INVALID;
  cudaError_t e;
  double* sF = c->d_sig;
  double* sG = sF + c->n;
  double* s = sG + c->n;
  // a Z rescale queued after the last sweep's counters (the step-wise
  // drivers: hzg_collect, then hzg_rescale_z) has not been checked yet
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "status copy");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "final rescale");
  {
    int32_t pending = 0;
    std::memcpy(&pending, c->h_ctr, 4);
    if (pending) return fail(c, HZG_RANK, "zero pencil column between sweeps");
  }
  cudaMemsetAsync(c->d_status, 0, 16, c->stream);
  int rc = launch_rescale(c->F, c->G, c->Z, c->n, c->cplx, 1, sF, sG, s, nullptr, c->d_status,
                          c->comp ? c->d_comp : nullptr, c->cstride, c->stream);
  if (rc) return fail(c, rc, "final rescale launch");
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "status copy");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "final rescale");
  int32_t st = 0;
  std::memcpy(&st, c->h_ctr, 4);
  if (st) return fail(c, HZG_RANK, "zero column at extraction");
  Plane Uo{Ur, c->cplx ? Ui : nullptr, mF0, mF0};
  Plane Vo{Vr, c->cplx ? Vi : nullptr, mG0, mG0};
  Plane Zo{Zr, c->cplx ? Zi : nullptr, n0, n0};
  rc = launch_finalize(c->F, c->G, c->Z, c->n, n0, mF0, mG0, c->cplx, sort, sF, sG, s, Uo, Vo, Zo, sigF, sigG,
                       sig, c->d_fin, c->d_status, c->stream);
  if (rc) return fail(c, rc, "finalize launch");
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "status copy");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "finalize");
  std::memcpy(&st, c->h_ctr, 4);
  if (st) return fail(c, HZG_RANK, "bordered solve mixed padded and original columns");
  return HZG_OK;
}

int hzg_test_block(int32_t tw, int32_t is_complex, const hzg_config* cfg, double epsn, const double* gFr,
                   const double* gFi, const double* gGr, const double* gGi, double* zr, double* zi,
                   int32_t* counts4) {
  if (!cfg || tw < 2 || tw % 2) return HZG_INVALID;
  const int NP = is_complex ? 2 : 1;
  const size_t t2 = (size_t)tw * tw;
  hzg_ctx c;
  c.cfg = *cfg;
  if (c.cfg.max_inner_sweeps <= 0) c.cfg.max_inner_sweeps = 30;
  c.cplx = is_complex ? 1 : 0;
  c.tw = tw;
  c.w = tw / 2;
  c.epsn = epsn;
  std::vector<int32_t> inner;
  int isteps = gen_table(cfg->inner_mm != 0, tw, inner);
  // device buffers: part (2 mats x NP x t2), zt, ident, counts, itable, colpair
  double *d_part = nullptr, *d_zt = nullptr;
  int32_t *d_misc = nullptr;
  cudaMalloc(&d_part, 2 * NP * t2 * 8);
  cudaMalloc(&d_zt, NP * t2 * 8);
  cudaMalloc(&d_misc, (16 + (size_t)isteps * tw) * 4);
  std::vector<double> hp(2 * NP * t2, 0.0);
  std::memcpy(hp.data(), gFr, t2 * 8);
  if (is_complex) std::memcpy(hp.data() + t2, gFi, t2 * 8);
  std::memcpy(hp.data() + NP * t2, gGr, t2 * 8);
  if (is_complex) std::memcpy(hp.data() + NP * t2 + t2, gGi, t2 * 8);
  cudaMemcpy(d_part, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_misc + 16, inner.data(), (size_t)isteps * tw * 4, cudaMemcpyHostToDevice);
  cudaMemset(d_misc, 0, 16 * 4);
  GramWS gw{};
  gw.part = d_part;
  gw.nsplit[0] = gw.nsplit[1] = 1;
  gw.smax = 1;
  gw.chunk[0] = gw.chunk[1] = 1;
  InnerOut io{d_zt, d_misc, d_misc + 4, nullptr};
  StepPairs sp{d_misc + 8, 1, 0, 1};  // colpair (0, 0): only used by the QR fallback
  KernelCfg kc = kernel_cfg(&c);
  kc.fallback_qr = 0;  // the block test has no columns to shorten
  kc.shorten_qr = 0;
  Plane dummy{nullptr, nullptr, 0, 0};
  int rc = launch_inner(dummy, dummy, sp, 0, kc, gw, d_misc + 16, isteps, io, nullptr, 1, d_misc + 12, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (rc == HZG_OK && e == cudaSuccess) {
    std::vector<double> hz(NP * t2);
    cudaMemcpy(hz.data(), d_zt, NP * t2 * 8, cudaMemcpyDeviceToHost);
    std::memcpy(zr, hz.data(), t2 * 8);
    if (is_complex && zi) std::memcpy(zi, hz.data() + t2, t2 * 8);
    cudaMemcpy(counts4, d_misc + 4, 16, cudaMemcpyDeviceToHost);
  }
  cudaFree(d_part);
  cudaFree(d_zt);
  cudaFree(d_misc);
  if (rc) return rc;
  return e == cudaSuccess ? HZG_OK : HZG_CUDA;
}

int hzg_set_timing(hzg_ctx* c, int32_t on) {
  if (!c) return HZG_INVALID;
  if (c->gexec) return fail(c, HZG_INVALID, "hzg_set_timing must precede the first sweep");
  c->timing = on != 0;
  return HZG_OK;
}

int hzg_kernel_times(hzg_ctx* c, double* ms3, int64_t* launches3, int32_t reset) {
  if (!c) return HZG_INVALID;
  for (int k = 0; k < 3; ++k) {
    if (ms3) ms3[k] = c->kms[k];
    if (launches3) launches3[k] = c->kcnt[k];
    if (reset) {
      c->kms[k] = 0;
      c->kcnt[k] = 0;
    }
  }
  return HZG_OK;
}

int hzg_step_counters(hzg_ctx* c, int32_t* out, int64_t capacity, int64_t* count) {
  if (!c || !c->bound) return HZG_INVALID;
  const int64_t nn = (int64_t)c->osteps * c->npairs * 4;
  if (count) *count = nn;
  if (!out || capacity < nn) return HZG_INVALID;
  cudaError_t e = cudaMemcpyAsync(out, c->io.counts, nn * 4, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return e == cudaSuccess ? HZG_OK : cuda_fail(c, e, "counter copy");
}

int hzg_debug_phases(hzg_ctx* c, int32_t enable, int64_t* out4) {
  if (!c || !c->bound) return HZG_INVALID;
  if (enable) {
    if (c->gexec) return fail(c, HZG_INVALID, "enable phase diagnostics before the first sweep");
    cudaMemsetAsync(c->d_phase, 0, 32, c->stream);
    c->io.phase = c->d_phase;
  }
  if (out4) {
    cudaMemcpyAsync(out4, c->d_phase, 32, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
  }
  return HZG_OK;
}

int hzg_launch_counts(const hzg_ctx* c, int64_t* per_sweep, int64_t* per_solve_fixed) {
  if (!c) return HZG_INVALID;
  const int G = c->gexec ? c->groups : choose_groups(c);
  // sweep graph: 3 step kernels per (step, group) (4 with the deferred Z
  // postmultiply), counter fold, rescale
  const bool dz = c->gexec ? c->defer_z : want_defer_z(c);
  if (per_sweep) *per_sweep = (int64_t)c->osteps * G * (dz ? 4 : 3) + 2;
  if (per_sweep && c->fused) {
    int64_t n = 1 + 2 + (int64_t)c->osteps * 1 + (int64_t)(c->osteps - 1) * 2 + 1;  // gram0, counters, rescale, inner, postgram+postZ, last post
    for (int k = 0; k + 1 < c->osteps; ++k) n += c->pg_nexc[k] > 0 ? 1 : 0;
    *per_sweep = n;
  }
  // k_prescale; final k_rescale, k_keep, k_keep_count, k_rank, k_gather
  if (per_solve_fixed) *per_solve_fixed = 6;
  return HZG_OK;
}

// ---------------------------------------------------------------------------
// Single block operations of the reference's public API (blocked.py:328-401),
// reference-order (bitwise) device kernels.  Device pointers; synchronous.
// ---------------------------------------------------------------------------
namespace {
struct DevBuf {
  void* p = nullptr;
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 8); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
}  // namespace

int hzg_op_qr_rfactor(int64_t m, int32_t nc, int32_t is_complex, int32_t pivot, double tol_scale, double* Ar,
                      double* Ai, int64_t* jpvt, int32_t* result, void* stream) {
  if (m < 1 || nc < 1 || m < nc || !Ar || (is_complex && !Ai) || !jpvt || !result) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  DevBuf scr, fl;
  if (scr.alloc((size_t)(2 * nc + 4) * 8) != cudaSuccess || fl.alloc(8) != cudaSuccess) return HZG_CUDA;
  int32_t h[2] = {0, 0};
  if (cudaMemsetAsync(fl.p, 0, 8, s) != cudaSuccess) return HZG_CUDA;
  if (launch_qr_rfactor(Ar, Ai, m, nc, is_complex, pivot, tol_scale, jpvt, (double*)scr.p, (int32_t*)fl.p, s))
    return HZG_CUDA;
  if (cudaMemcpyAsync(h, fl.p, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return HZG_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return HZG_CUDA;
  *result = (h[0] || h[1]) ? 1 : 0;
  return HZG_OK;
}

int hzg_op_grammian(int64_t m, int32_t w, int32_t cplx, int32_t comp, const double* Yr, const double* Yi, double* Ar,
                    double* Ai, void* stream) {
  if (m < 1 || w < 1 || !Yr || !Ar || (cplx && (!Yi || !Ai))) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int tw = 2 * w, NP = cplx ? 2 : 1;
  Plane Y{const_cast<double*>(Yr), cplx ? const_cast<double*>(Yi) : nullptr, m, m};
  GramWS gw{};
  int nsplit = 1;
  int64_t chunk = m;
  if (!comp) gram_split(m, true, 0, 0, nsplit, chunk);
  gw.nsplit[0] = gw.nsplit[1] = nsplit;
  gw.chunk[0] = gw.chunk[1] = chunk;
  gw.smax = nsplit;
  const int64_t P = pow2c(m);
  DevBuf cp, part, scr;
  if (cp.alloc(8) || part.alloc((size_t)2 * nsplit * NP * tw * tw * 8) ||
      (comp && scr.alloc((size_t)2 * 32 * P * 8)))
    return HZG_CUDA;
  const int32_t h_cp[2] = {0, w};
  cudaMemcpyAsync(cp.p, h_cp, 8, cudaMemcpyHostToDevice, s);
  StepPairs sp{(const int32_t*)cp.p, 1, 0, 1};
  gw.part = (double*)part.p;
  int rc = comp ? launch_gram_comp(Y, Y, sp, 0, w, cplx, gw, (double*)scr.p, P, s)
                : launch_gram_exact(Y, Y, sp, 0, w, cplx, gw, s);
  if (!rc) rc = launch_fold_gram(gw.part, nsplit, tw, cplx, Ar, cplx ? Ai : nullptr, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (rc) return rc;
  return e == cudaSuccess ? HZG_OK : HZG_CUDA;
}

int hzg_op_cholesky_upper(int32_t tw, int32_t cplx, double* Ar, double* Ai, void* stream) {
  if (tw < 1 || !Ar || (cplx && !Ai)) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  DevBuf st;
  if (st.alloc(4)) return HZG_CUDA;
  int rc = launch_cholesky_op(tw, cplx, Ar, cplx ? Ai : nullptr, (int32_t*)st.p, s);
  if (rc) return rc;
  int32_t h = 0;
  cudaMemcpyAsync(&h, st.p, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return HZG_CUDA;
  return h ? HZG_NOT_PD : HZG_OK;
}

int hzg_op_qr_shorten(int64_t m, int32_t w, int32_t cplx, const double* Yr, const double* Yi, double* Rr,
                      double* Ri, void* stream) {
  if (m < 1 || w < 1 || !Yr || !Rr || (cplx && (!Yi || !Ri))) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int tw = 2 * w;
  Plane Y{const_cast<double*>(Yr), cplx ? const_cast<double*>(Yi) : nullptr, m, m};
  DevBuf st, scr;
  if (st.alloc(4) || scr.alloc((size_t)2 * m * tw * 8)) return HZG_CUDA;
  double* Sr = (double*)scr.p;
  int rc = launch_qr_op(Y, tw, cplx, Sr, Sr + m * tw, Rr, cplx ? Ri : nullptr, (int32_t*)st.p, s);
  if (rc) return rc;
  int32_t h = 0;
  cudaMemcpyAsync(&h, st.p, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return HZG_CUDA;
  return h ? HZG_RANK : HZG_OK;
}

int hzg_op_postmultiply(int64_t m, int32_t w, int32_t cplx, double* Yr, double* Yi, const double* Zr,
                        const double* Zi, void* stream) {
  if (m < 1 || w < 1 || !Yr || !Zr || (cplx && (!Yi || !Zi))) return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int tw = 2 * w, NP = cplx ? 2 : 1;
  Plane Y{Yr, cplx ? Yi : nullptr, m, m};
  Plane none{Yr, cplx ? Yi : nullptr, 0, m};  // rows = 0: the other two matrices are skipped
  DevBuf cp, zt, id;
  if (cp.alloc(8) || zt.alloc((size_t)NP * tw * tw * 8) || id.alloc(4)) return HZG_CUDA;
  const int32_t h_cp[2] = {0, w};
  cudaMemcpyAsync(cp.p, h_cp, 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(zt.p, Zr, (size_t)tw * tw * 8, cudaMemcpyDeviceToDevice, s);
  if (cplx) cudaMemcpyAsync((double*)zt.p + tw * tw, Zi, (size_t)tw * tw * 8, cudaMemcpyDeviceToDevice, s);
  cudaMemsetAsync(id.p, 0, 4, s);
  StepPairs sp{(const int32_t*)cp.p, 1, 0, 1};
  InnerOut io{(double*)zt.p, (int32_t*)id.p, nullptr, nullptr};
  int rc = launch_postmult_exact(Y, none, none, sp, 0, w, cplx, io, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (rc) return rc;
  return e == cudaSuccess ? HZG_OK : HZG_CUDA;
}

int hzg_op_rescale(int64_t mF, int64_t mG, int64_t n, int32_t cplx, int32_t comp, int32_t final, double* Fr,
                   double* Fi, double* Gr, double* Gi, double* Zr, double* Zi, int64_t mZ, double* sigF,
                   double* sigG, double* sig, void* stream) {
  if (n < 1 || !Fr || !Gr || !Zr || (cplx && (!Fi || !Gi || !Zi)) || (final && (!sigF || !sigG || !sig)))
    return HZG_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  Plane F{Fr, cplx ? Fi : nullptr, mF, mF}, G{Gr, cplx ? Gi : nullptr, mG, mG}, Z{Zr, cplx ? Zi : nullptr, mZ, mZ};
  const int64_t P = pow2c(std::max(mF, mG));
  DevBuf st, scr;
  if (st.alloc(4) || (comp && scr.alloc((size_t)n * P * 8))) return HZG_CUDA;
  cudaMemsetAsync(st.p, 0, 4, s);
  int rc = launch_rescale(F, G, Z, n, cplx, final, sigF, sigG, sig, nullptr, (int32_t*)st.p,
                          comp ? (double*)scr.p : nullptr, P, s);
  if (rc) return rc;
  int32_t h = 0;
  cudaMemcpyAsync(&h, st.p, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return HZG_CUDA;
  return h ? HZG_RANK : HZG_OK;
}

int hzg_test_fastmath(int64_t n, uint64_t seed, int64_t* counts4) {
  if (!counts4 || n < 1) return HZG_INVALID;
  return fastmath_check(n, seed, counts4);
}

const char* hzg_last_error(const hzg_ctx* c) { return c ? c->err.c_str() : "null context"; }


// ---------------------------------------------------------------------------
// multi-GPU data plane: NCCL inside libhzg
// ---------------------------------------------------------------------------

// restores the calling thread's current device on scope exit (entry points
// that switch devices must not change the caller's CUDA state)
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int hzg_comm_unique_id(void* id_out) {
  if (!id_out) return HZG_INVALID;
  std::string err;
  const hzg::nccl::Api* nc = hzg::nccl::load(err);
  if (!nc) return HZG_CUDA;
  ncclUniqueId id;
  if (nc->GetUniqueId(&id) != ncclSuccess) return HZG_CUDA;
  std::memcpy(id_out, &id, sizeof(id));
  return HZG_OK;
}

size_t hzg_comm_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

static int nccl_fail(hzg_ctx* c, ncclResult_t r, const char* where) {
  c->err = std::string(where) + ": " + (c->nc ? c->nc->GetErrorString(r) : "nccl");
  return HZG_CUDA;
}

int hzg_comm_attach(hzg_ctx* c, int32_t nranks, int32_t rank, const void* unique_id) {
  DeviceGuard guard;
  if (!c || !unique_id || nranks < 1 || rank < 0 || rank >= nranks) return HZG_INVALID;
  if (c->comm) return fail(c, HZG_INVALID, "communicator already attached");
  std::string err;
  c->nc = hzg::nccl::load(err);
  if (!c->nc) return fail(c, HZG_CUDA, err.c_str());
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclResult_t r = c->nc->CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    return nccl_fail(c, r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  return HZG_OK;
}

int hzg_comm_set_moves(hzg_ctx* c, const int32_t* moves, const int32_t* offsets, int32_t osteps) {
  if (!c || !offsets || osteps != c->osteps) return HZG_INVALID;
  if (offsets[0] != 0) return HZG_INVALID;
  for (int k = 0; k < osteps; ++k)
    if (offsets[k + 1] < offsets[k]) return HZG_INVALID;
  const int32_t total = offsets[osteps];
  if (total > 0 && !moves) return HZG_INVALID;
  c->moves.clear();
  c->move_off.assign(1, 0);
  for (int k = 0; k < osteps; ++k) {
    for (int32_t q = offsets[k]; q < offsets[k + 1]; ++q) {
      const int32_t b = moves[3 * q], src = moves[3 * q + 1], dst = moves[3 * q + 2];
      if (b < 0 || b >= c->nblk || src < 0 || src >= c->nranks || dst < 0 || dst >= c->nranks)
        return fail(c, HZG_INVALID, "block move out of range");
      if (src != c->rank && dst != c->rank) continue;  // not this rank's business
      c->moves.insert(c->moves.end(), {b, src, dst});
    }
    c->move_off.push_back((int32_t)(c->moves.size() / 3));
  }
  if (c->dgexec) {
    cudaGraphExecDestroy(c->dgexec);
    c->dgexec = nullptr;
  }
  if (c->dgraph) {
    cudaGraphDestroy(c->dgraph);
    c->dgraph = nullptr;
  }
  return HZG_OK;
}

// Grouped send / recv of whole block columns of F, G, Z (each block is one
// contiguous w * rows range of every plane).  A block whose source and
// destination are both this rank is sent to itself.
static int emit_exchange(hzg_ctx* c, const int32_t* mv, int count, cudaStream_t s) {
  if (count <= 0) return HZG_OK;
  const hzg::nccl::Api* nc = c->nc;
  const Plane* pl[3] = {&c->F, &c->G, &c->Z};
  ncclResult_t r = nc->GroupStart();
  if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupStart");
  for (int q = 0; q < count && r == ncclSuccess; ++q) {
    const int32_t b = mv[3 * q], src = mv[3 * q + 1], dst = mv[3 * q + 2];
    for (int m = 0; m < 3 && r == ncclSuccess; ++m) {
      const size_t cnt = (size_t)c->w * pl[m]->rows;
      for (int part = 0; part < (c->cplx ? 2 : 1) && r == ncclSuccess; ++part) {
        double* base = (part ? pl[m]->im : pl[m]->re) + (size_t)b * c->w * pl[m]->ld;
        if (src == c->rank) r = nc->Send(base, cnt, ncclFloat64, dst, c->comm, s);
        if (r == ncclSuccess && dst == c->rank) r = nc->Recv(base, cnt, ncclFloat64, src, c->comm, s);
      }
    }
  }
  ncclResult_t r2 = nc->GroupEnd();
  if (r != ncclSuccess) return nccl_fail(c, r, "ncclSend/ncclRecv");
  if (r2 != ncclSuccess) return nccl_fail(c, r2, "ncclGroupEnd");
  return HZG_OK;
}

int hzg_comm_exchange(hzg_ctx* c, const int32_t* moves, int32_t count) {
  if (!c || !c->bound || !c->comm || count < 0 || (count > 0 && !moves)) return HZG_INVALID;
  std::vector<int32_t> mine;
  for (int q = 0; q < count; ++q) {
    const int32_t b = moves[3 * q], src = moves[3 * q + 1], dst = moves[3 * q + 2];
    if (b < 0 || b >= c->nblk || src < 0 || src >= c->nranks || dst < 0 || dst >= c->nranks)
      return fail(c, HZG_INVALID, "block move out of range");
    if (src == c->rank || dst == c->rank) mine.insert(mine.end(), {b, src, dst});
  }
  int rc = emit_exchange(c, mine.data(), (int)(mine.size() / 3), c->stream);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  return e == cudaSuccess ? HZG_OK : cuda_fail(c, e, "exchange");
}

// One rank's outer sweep as ONE CUDA graph: its slot range of every step as
// position groups on the group streams (wavefront, as in build_graph), the
// block exchange after every step on the exchange stream (grouped NCCL
// send / recv; the end groups of step k+1 wait for it, it waits for the end
// groups of step k -- the blocks that change owner sit at the ends of the
// rank's range), then the counter fold, an all-reduce of the counters and
// status indicators, the Z rescale gated on the GLOBAL big count, and an
// all-reduce of its status.  No host synchronisation inside the sweep.
static int build_dist_graph(hzg_ctx* c) {
  cudaError_t e;
  int G = std::max(1, std::min(8, c->npairs / 16));
  if (const char* env = std::getenv("HZG_GROUPS")) G = std::max(1, std::min(c->npairs, std::atoi(env)));
  c->dgroups = G;
  if (int rc = stream_pool(c, c->gstreams, G, true)) return rc;
  if (!c->xstream) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if ((e = cudaStreamCreateWithPriority(&c->xstream, cudaStreamNonBlocking, greatest)) != cudaSuccess)
      return cuda_fail(c, e, "cudaStreamCreate");
  }
  const size_t nev = 3 + 3 * (size_t)G;
  while (c->devents.size() < nev) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(c, e, "cudaEventCreate");
    c->devents.push_back(ev);
  }
  cudaEvent_t fork = c->devents[0], xev = c->devents[1], xjoin = c->devents[2];
  cudaEvent_t* join = &c->devents[3];
  cudaEvent_t* sev = &c->devents[3 + G];  // [2][G]
  if ((e = cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return cuda_fail(c, e, "begin capture");
  int rc = HZG_OK;
  cudaEventRecord(fork, c->cap);
  for (int g = 0; g < G; ++g) cudaStreamWaitEvent(c->gstreams[g], fork, 0);
  cudaStreamWaitEvent(c->xstream, fork, 0);
  for (int st = 0; st < c->osteps && rc == HZG_OK; ++st) {
    for (int g = 0; g < G && rc == HZG_OK; ++g) {
      cudaStream_t s = c->gstreams[g];
      if (st > 0) {
        if (g > 0) cudaStreamWaitEvent(s, sev[((st - 1) & 1) * G + g - 1], 0);
        if (g + 1 < G) cudaStreamWaitEvent(s, sev[((st - 1) & 1) * G + g + 1], 0);
        if (g == 0 || g == G - 1) cudaStreamWaitEvent(s, xev, 0);
      }
      const int p0 = group_cut(c->npairs, G, g), p1 = group_cut(c->npairs, G, g + 1);
      rc = launch_step(c, st, s, nullptr, p0, p1 - p0);
      cudaEventRecord(sev[(st & 1) * G + g], s);
    }
    if (rc) break;
    const int nm = c->move_off.empty() ? 0 : c->move_off[st + 1] - c->move_off[st];
    if (nm > 0) {
      cudaStreamWaitEvent(c->xstream, sev[(st & 1) * G + 0], 0);
      cudaStreamWaitEvent(c->xstream, sev[(st & 1) * G + G - 1], 0);
      rc = emit_exchange(c, c->moves.data() + 3 * (size_t)c->move_off[st], nm, c->xstream);
    }
    cudaEventRecord(xev, c->xstream);
  }
  for (int g = 0; g < G; ++g) {
    cudaEventRecord(join[g], c->gstreams[g]);
    cudaStreamWaitEvent(c->cap, join[g], 0);
  }
  cudaEventRecord(xjoin, c->xstream);
  cudaStreamWaitEvent(c->cap, xjoin, 0);
  if (rc == HZG_OK) rc = launch_counters(c->io.counts, (int64_t)c->osteps * c->npairs, c->d_ctr, c->cap);
  if (rc == HZG_OK) {
    k_red_pack<<<1, 32, 0, c->cap>>>(c->d_ctr, c->d_red);
    ncclResult_t r = c->nc->AllReduce(c->d_red, c->d_red, 5, ncclInt64, ncclSum, c->comm, c->cap);
    if (r != ncclSuccess) rc = nccl_fail(c, r, "ncclAllReduce(counters)");
  }
  if (rc == HZG_OK)
    rc = launch_rescale(c->F, c->G, c->Z, c->n, c->cplx, 0, nullptr, nullptr, nullptr, c->d_red, c->d_status,
                        c->comp ? c->d_comp : nullptr, c->cstride, c->cap);
  if (rc == HZG_OK) {
    k_red_status<<<1, 32, 0, c->cap>>>(c->d_status, c->d_red);
    ncclResult_t r = c->nc->AllReduce(c->d_red + 5, c->d_red + 5, 1, ncclInt64, ncclSum, c->comm, c->cap);
    if (r != ncclSuccess) rc = nccl_fail(c, r, "ncclAllReduce(status)");
  }
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(c->cap, &g);
  if (rc != HZG_OK) {
    if (g) cudaGraphDestroy(g);
    return rc == HZG_CUDA && !c->err.empty() ? rc : fail(c, rc, "launch during capture");
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "end capture");
  c->dgraph = g;
  if ((e = cudaGraphInstantiate(&c->dgexec, g, cudaGraphInstantiateFlagUseNodePriority)) != cudaSuccess)
    return cuda_fail(c, e, "graph instantiate");
  return HZG_OK;
}

int hzg_dist_sweep_launch(hzg_ctx* c) {
  DeviceGuard guard;
  if (!c || !c->bound || !c->comm) return HZG_INVALID;
  if ((int)c->move_off.size() != c->osteps + 1) return fail(c, HZG_INVALID, "hzg_comm_set_moves first");
  cudaError_t e;
  if ((e = cudaSetDevice(c->device)) != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  if (!c->dgexec) {
    if (int rc = build_dist_graph(c)) return rc;
  }
  if ((e = cudaGraphLaunch(c->dgexec, c->stream)) != cudaSuccess) return cuda_fail(c, e, "graph launch");
  if ((e = cudaMemcpyAsync(c->h_ctr, c->d_red, 6 * 8, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "counter copy");
  return HZG_OK;
}

int hzg_dist_sweep_wait(hzg_ctx* c, int64_t* total, int64_t* big) {
  DeviceGuard guard;
  if (!c || !c->bound || !c->comm) return HZG_INVALID;
  cudaError_t e;
  if ((e = cudaSetDevice(c->device)) != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "dist sweep");
  ncclResult_t async = ncclSuccess;
  c->nc->CommGetAsyncError(c->comm, &async);
  if (async != ncclSuccess) return nccl_fail(c, async, "NCCL async error");
  if (total) *total = c->h_ctr[0];
  if (big) *big = c->h_ctr[1];
  // every rank holds the same reduced indicators, so every rank raises the
  // same error (no rank leaves the job while the others wait in NCCL)
  if (c->h_ctr[3]) return fail(c, HZG_NOT_PD, "indefinite block Grammian; enable the QR fallback");
  if (c->h_ctr[4]) return fail(c, HZG_RANK, "rank-deficient block pair in the inner solve");
  if (c->h_ctr[5]) return fail(c, HZG_RANK, "zero pencil column between sweeps");
  return HZG_OK;
}

int hzg_dist_sweep(hzg_ctx* c, int64_t* total, int64_t* big) {
  int rc = hzg_dist_sweep_launch(c);
  return rc ? rc : hzg_dist_sweep_wait(c, total, big);
}

// One process driving several GPUs: one communicator per context from
// ncclCommInitAll (rank i = ctxs[i], on ctxs[i]'s device).
int hzg_comm_attach_all(hzg_ctx** ctxs, int32_t n) {
  if (!ctxs || n < 1) return HZG_INVALID;
  std::string err;
  const hzg::nccl::Api* nc = hzg::nccl::load(err);
  if (!nc) return HZG_CUDA;
  std::vector<int> devs(n);
  std::vector<ncclComm_t> comms(n, nullptr);
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || ctxs[i]->comm) return HZG_INVALID;
    devs[i] = ctxs[i]->device;
  }
  ncclResult_t r = nc->CommInitAll(comms.data(), n, devs.data());
  if (r != ncclSuccess) {
    ctxs[0]->nc = nc;
    return nccl_fail(ctxs[0], r, "ncclCommInitAll");
  }
  for (int i = 0; i < n; ++i) {
    ctxs[i]->nc = nc;
    ctxs[i]->comm = comms[i];
    ctxs[i]->nranks = n;
    ctxs[i]->rank = i;
  }
  return HZG_OK;
}

// Grouped exchange across the contexts of one process (hzg_comm_attach_all):
// one NCCL group around every rank's sends and receives, then wait for all.
int hzg_comm_exchange_all(hzg_ctx** ctxs, int32_t n, const int32_t* moves, int32_t count) {
  DeviceGuard guard;
  if (!ctxs || n < 1 || count < 0 || (count > 0 && !moves)) return HZG_INVALID;
  const hzg::nccl::Api* nc = ctxs[0]->nc;
  if (!nc) return HZG_INVALID;
  ncclResult_t r = nc->GroupStart();
  if (r != ncclSuccess) return nccl_fail(ctxs[0], r, "ncclGroupStart");
  int rc = HZG_OK;
  for (int i = 0; i < n && rc == HZG_OK; ++i) {
    hzg_ctx* c = ctxs[i];
    if (!c || !c->bound || !c->comm) {
      rc = HZG_INVALID;
      break;
    }
    cudaSetDevice(c->device);
    std::vector<int32_t> mine;
    for (int q = 0; q < count; ++q)
      if (moves[3 * q + 1] == c->rank || moves[3 * q + 2] == c->rank)
        mine.insert(mine.end(), {moves[3 * q], moves[3 * q + 1], moves[3 * q + 2]});
    rc = emit_exchange(c, mine.data(), (int)(mine.size() / 3), c->stream);
  }
  r = nc->GroupEnd();
  if (rc) return rc;
  if (r != ncclSuccess) return nccl_fail(ctxs[0], r, "ncclGroupEnd");
  for (int i = 0; i < n; ++i) {
    cudaSetDevice(ctxs[i]->device);
    cudaError_t e = cudaStreamSynchronize(ctxs[i]->stream);
    if (e != cudaSuccess) return cuda_fail(ctxs[i], e, "exchange");
  }
  return HZG_OK;
}

int hzg_comm_detach(hzg_ctx* c) {
  if (!c) return HZG_INVALID;
  if (c->dgexec) cudaGraphExecDestroy(c->dgexec);
  if (c->dgraph) cudaGraphDestroy(c->dgraph);
  c->dgexec = nullptr;
  c->dgraph = nullptr;
  if (c->comm && c->nc) c->nc->CommDestroy(c->comm);
  c->comm = nullptr;
  c->nranks = 1;
  c->rank = 0;
  return HZG_OK;
}

void hzg_destroy(hzg_ctx* c) {
  if (!c) return;
  hzg_comm_detach(c);
  for (auto& e : c->devents) cudaEventDestroy(e);
  if (c->xstream) cudaStreamDestroy(c->xstream);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->cap) cudaStreamDestroy(c->cap);
  if (c->h_ctr) cudaFreeHost(c->h_ctr);
  for (auto& e : c->tev) cudaEventDestroy(e);
  for (auto& e : c->rev) cudaEventDestroy(e);
  for (auto& e : c->gevents) cudaEventDestroy(e);
  for (auto& s : c->gstreams) cudaStreamDestroy(s);
  for (auto& e : c->wevents) cudaEventDestroy(e);
  for (auto& s : c->wstreams) cudaStreamDestroy(s);
  for (auto& s : c->zstreams) cudaStreamDestroy(s);
  for (auto& s : c->wzstreams) cudaStreamDestroy(s);
  delete c;
}

}  // extern "C"
