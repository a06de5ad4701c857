// Internal host/device declarations shared by the hzg translation units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hzg {

// Kernel attributes (dynamic shared memory limits) are per device: a call
// site sets them the first time it runs on each device of the process.
struct PerDeviceOnce {
  unsigned long long done = 0;  // bit d: device d (d < 64) done
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    if (done & b) return false;
    done |= b;
    return true;
  }
};

// SM count of the current device (cached per device)
inline int device_sms() {
  static int sms[64] = {0};
  int d = 0;
  cudaGetDevice(&d);
  int& v = sms[d & 63];
  if (v <= 0 && (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0)) v = 148;
  return v;
}

// status bits written per block pair (and OR-folded per sweep)
enum : int {
  ST_OK = 0,
  ST_RANK = 1,        // zero column / zero pencil (RankError)
  ST_NOT_PD = 2,      // Cholesky failed with the QR fallback disabled
  ST_QR_RANK = 4,     // QR shortening found a rank-deficient block (RankError)
};


// One matrix of the pair in HBM: split planes, column-major, column j at
// re + j * ld (the reference's Fortran MatrixPlanePair, core.py:26-69).
struct Plane {
  double* re;
  double* im;  // nullptr for real problems
  int64_t rows;
  int64_t ld;
};

// Per-step view of the block pairs this GPU processes.  colpair[k] holds the
// physical column offsets (c0, c1) of pair k of the step: c0 is the block
// with the smaller logical index (the reference's sorted (p, q), blocked.py:438-439).
struct StepPairs {
  const int32_t* colpair;  // [osteps][npairs][2]
  int npairs;              // pairs per step (row stride of colpair)
  int p0, pn;              // the pair range [p0, p0 + pn) this launch processes
};

struct KernelCfg {
  int tw;               // 2w
  int cplx;
  int prescale;         // pointwise.py:78
  int per_step_rescale; // !prescale
  int compensated;
  int crit_c2;
  int sorting;
  int max_inner_sweeps;
  int fallback_qr;
  int shorten_qr;       // cfg.shorten == "qr": QR R factors instead of Grammian + Cholesky
  double epsn;          // gate_eps * sqrt(n) (blocked.py:571-572)
  int approx_2x2;       // DMMA mode: short-chain 2x2 forms (tolerance parity); 0: reference order
};

// Grammian partials: [pair][mat(F,G)][split][plane][tw*tw], element (r,s) at s*tw+r.
struct GramWS {
  double* part;
  int nsplit[2];   // splits per matrix (powers of two)
  int smax;        // stride (max of nsplit)
  int64_t chunk[2];  // rows per split (powers of two in exact mode)
};

// per-pair outputs of the inner kernel
struct InnerOut {
  double* zt;        // [pair][plane][tw*tw]
  int32_t* ident;    // [pair] 1 -> transform is exactly I (skip postmult, blocked.py:480)
  int32_t* counts;   // [osteps][npairs][4]: total, big, status, inner sweeps
  long long* phase;  // optional diagnostics (CTA 0, warp 0): cycles in phases A, B, C, #steps
};

// kernel launchers (hzg_kernels.cu / hzg_dmma.cu)
// cscr (compensated variants): per-column scratch of cstride doubles, or nullptr
int launch_prescale(const Plane& F, const Plane& G, const Plane& Z, int64_t n, int cplx, int do_prescale,
                    int32_t* status, double* cscr, int64_t cstride, cudaStream_t s);
int launch_rescale(const Plane& F, const Plane& G, const Plane& Z, int64_t n, int cplx, int final, double* sigF,
                   double* sigG, double* sig, const int64_t* gate_counters, int32_t* status, double* cscr,
                   int64_t cstride, cudaStream_t s);
int launch_gram_comp(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                     const GramWS& gw, double* scratch, int64_t pstride, cudaStream_t s);
int launch_gram_exact(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                      const GramWS& gw, cudaStream_t s);
// plist (optional): explicit pairs of the launch (npl of them) instead of sp's range
int launch_gram_dmma(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                     const GramWS& gw, cudaStream_t s, const int32_t* plist = nullptr, int npl = 0);
int launch_inner(const Plane& F, const Plane& G, const StepPairs& sp, int step, const KernelCfg& kc,
                 const GramWS& gw, const int32_t* itable, int isteps, const InnerOut& io, double* qr_scratch,
                 int qr_slots, int32_t* qr_slot_ctr, cudaStream_t s);
int launch_postmult_exact(const Plane& F, const Plane& G, const Plane& Z, const StepPairs& sp, int step, int w,
                          int cplx, const InnerOut& io, cudaStream_t s);
// matrices [mat0, mat0 + nmats) of {F, G, Z}
int launch_postmult_dmma(const Plane& F, const Plane& G, const Plane& Z, const StepPairs& sp, int step, int w,
                         int cplx, const InnerOut& io, cudaStream_t s, int mat0 = 0, int nmats = 3);

// Column-pivoted Householder R factor of an m x nc column-major matrix in
// place (hzg_tall.cu; _k_qr_rfactor, blocked.py:97-217); flags[0] = column
// vanished, flags[1] = rank test failed (caller zeroes both)
int launch_qr_rfactor(double* Ar, double* Ai, int64_t m, int nc, int cplx, int pivot, double tol_scale,
                      int64_t* jpvt, double* scratch, int32_t* flags, cudaStream_t s);

// Fused postmultiply of step `step` (F and G) and Grammian partials of step
// `step + 1` along chains of circle positions (hzg_dmma.cu, 2w = 32, real).
struct PostGramTables {
  const int32_t* chains;  // [nchains][L + 1] current positions, -1 padded
  const int32_t* links;   // [nchains][L + 1][5]: next pair, src of its first block (elem, half), of its second
  int nchains, L;
};
int launch_postgram(const Plane& F, const Plane& G, const StepPairs& sp, int step, int w, int cplx,
                    const InnerOut& io, const GramWS& gw, const PostGramTables& t, cudaStream_t s);
bool postgram_supported(int w, int cplx);
int launch_counters(const int32_t* counts, int64_t nentries, int64_t* out, cudaStream_t s);
int launch_finalize(const Plane& U, const Plane& V, const Plane& Z, int64_t n, int64_t n0, int64_t mF0, int64_t mG0,
                    int cplx, int sort, const double* sigF, const double* sigG, const double* sig, Plane Uo, Plane Vo,
                    Plane Zo, double* sFo, double* sGo, double* so, int32_t* rank_ws, int32_t* status,
                    cudaStream_t s);

int launch_fold_gram(const double* part, int nsplit, int tw, int cplx, double* Ar, double* Ai, cudaStream_t s);
int launch_cholesky_op(int tw, int cplx, double* Ar, double* Ai, int32_t* status, cudaStream_t s);
int launch_qr_op(const Plane& Y, int tw, int cplx, double* Sr, double* Si, double* outR, double* outI,
                 int32_t* status, cudaStream_t s);

bool dmma_supported(int w);
int fastmath_check(int64_t n, uint64_t seed, int64_t* out4);

}  // namespace hzg
