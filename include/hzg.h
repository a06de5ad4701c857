/*
 * hzg.h -- C ABI of libhzg.so, the sm_100a implementation of the blocked
 * one-sided (implicit) Hari-Zimmermann GSVD hot path.
 *
 * Plain pointers and sizes only.  Matrices are split real/imaginary FP64
 * planes in column-major order, column j of an m-row plane at p + j*m --
 * exactly the reference's MatrixPlanePair (pkg/src/hzgsvd/core.py:26-69) --
 * resident in device memory (the caller allocates them, e.g. as torch
 * tensors, and keeps them alive).  `stream` is a cudaStream_t.
 *
 * Each entry point replaces one piece of the reference's CPU driver:
 *   hzg_create / hzg_bind   -> gsvd_blocked's set-up            (blocked.py:553-572)
 *   hzg_init_fgz            -> _k_prescale + Z0 = diag(z0)      (blocked.py:564-570, pointwise.py:254-274)
 *   hzg_sweep               -> one iteration of _algorithm1_loop (blocked.py:521-542),
 *                              i.e. all outer steps of _block_task (blocked.py:435-484)
 *                              plus the inter-sweep _k_rescale_full (blocked.py:540-542)
 *   hzg_finalize            -> final _k_rescale_full (blocked.py:579-581) + _unborder
 *                              (blocked.py:593-620) + _sort_descending (blocked.py:623-637)
 *
 * Return codes mirror the reference's error taxonomy (errors.py:4-23):
 *   HZG_OK, HZG_RANK -> RankError, HZG_NOT_PD -> NotPositiveDefiniteError,
 *   HZG_CUDA -> CUDA failure, HZG_INVALID -> ValueError.
 * Non-convergence is not an error (blocked.py:583-586): the caller counts
 * sweeps and stops at max_outer_sweeps.
 */
#ifndef HZG_H_
#define HZG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { HZG_OK = 0, HZG_RANK = 1, HZG_NOT_PD = 2, HZG_CUDA = 3, HZG_INVALID = 4 };

/* SolverConfig (pointwise.py:40-81), decoded fields */
typedef struct {
  int32_t variant_id;       /* 0..7 */
  int32_t outer_mm;         /* outer_kind == "mm" */
  int32_t inner_mm;         /* inner_kind == "mm" */
  int32_t max_inner_sweeps; /* 30 for blocking "fb", 1 for "bo" (already decoded) */
  int32_t max_outer_sweeps; /* 30 */
  int32_t block_width;      /* w; the pair is bordered to multiples of 2w */
  int32_t sorting;
  int32_t fallback_qr;
  int32_t shorten_qr;       /* shorten == "qr" */
  double gate_eps;          /* 2**-52 */
  int32_t exact;            /* 1: reference-order Grammian / postmultiply kernels */
  int32_t split_rows;       /* DMMA Grammian rows per split (multiple of 64); 0 = default geometry */
  int32_t approx_2x2;       /* exact == 0 only: short-chain 2x2 transforms (tolerance parity) */
} hzg_config;

typedef struct hzg_ctx hzg_ctx;

/* Problem of bordered size mF x n, mG x n (n and both heights multiples of
 * 2w).  epsn <= 0 selects gate_eps * sqrt(n) (blocked.py:571-572). */
int hzg_create(hzg_ctx** out, int device, int64_t mF, int64_t mG, int64_t n, int32_t is_complex,
               const hzg_config* cfg, double epsn);

/* Bytes of device workspace hzg_bind needs. */
size_t hzg_workspace_bytes(const hzg_ctx* ctx);

/* Attach the device planes (F mF x n, G mG x n, Z n x n; imaginary planes
 * NULL for real problems), a workspace of hzg_workspace_bytes() bytes and
 * the stream all work is ordered on. */
int hzg_bind(hzg_ctx* ctx, double* Fr, double* Fi, double* Gr, double* Gi, double* Zr, double* Zi,
             void* workspace, void* stream);

/* Replace the per-step block-pair schedule: colpairs[step][k] = (c0, c1),
 * the physical column offsets of pair k of the step (block with the smaller
 * logical index first).  Used to run a slot range of the ordering on one
 * GPU of a multi-GPU job.  npairs <= n / (2w). */
int hzg_set_schedule(hzg_ctx* ctx, const int32_t* colpairs, int32_t osteps, int32_t npairs);

/* Rows of the Z plane (default n).  A stripe slab of the reference's
 * distributed scheme (distsim.py:62-95) owns 2W of the n global columns but
 * its Z keeps all n_global rows (Z is n_global x 2W).  Before hzg_bind. */
int hzg_set_z_rows(hzg_ctx* ctx, int64_t zrows);

/* Initial G column scaling and Z0 (synchronous: returns the status). */
int hzg_init_fgz(hzg_ctx* ctx);

/* One outer sweep; returns the sweep's transform counters.  The inter-sweep
 * Z rescale runs on the device when big != 0.  Synchronous. */
int hzg_sweep(hzg_ctx* ctx, int64_t* total, int64_t* big);
/* hzg_sweep in two halves: queue the sweep graph and the counter copy on the
 * bound stream, then wait for them and map the status (several contexts on
 * different streams -- e.g. the stripe workers of stripes.py -- sweep
 * concurrently between the two calls). */
int hzg_sweep_launch(hzg_ctx* ctx);
int hzg_sweep_wait(hzg_ctx* ctx, int64_t* total, int64_t* big);

/* Run outer steps [first, first + count) of the schedule without the sweep
 * bookkeeping (asynchronous; for profiling and bounded benchmarks). */
int hzg_run_steps(hzg_ctx* ctx, int32_t first, int32_t count);

/* Run pairs [p0, p0 + pn) of outer step `step` (Grammian, inner solve,
 * postmultiply) on `stream` (NULL: the bound stream), asynchronously.  A
 * rank of a multi-GPU job splits its slot range into contiguous groups on
 * several streams so the streaming kernels of one group overlap the inner
 * solves of another (the per-rank form of the wavefront sweep graph; the
 * multi-worker step body of distsim.py:188-215, split by position). */
int hzg_run_pairs(hzg_ctx* ctx, int32_t step, int32_t p0, int32_t pn, void* stream);

/* The same per-rank wavefront driven from the library, one call per step
 * (no per-group host work): hzg_wave_step runs step `step` as `groups`
 * contiguous position groups on library-owned streams.  Group g waits for
 * groups g-1, g, g+1 of the previous step; the two end groups also wait
 * for everything queued on `comm` (the caller's block exchange of the
 * previous step), and `comm` is made to wait for this step's end groups,
 * so the caller queues the next exchange on `comm` right after the call.
 * In DMMA mode the Z postmultiply runs on separate low-priority streams;
 * with `zcomm` non-NULL the Z blocks are exchanged on `zcomm` instead of
 * `comm` (the caller queues them there), so the Z updates stay off the
 * step chain.  Step 0 (or a break in the sequence) starts after the work
 * queued on the bound stream.  hzg_wave_join makes the bound stream wait
 * for the last step, `comm` and `zcomm` (before hzg_collect /
 * hzg_finalize). */
int hzg_wave_step(hzg_ctx* ctx, int32_t step, int32_t groups, void* comm, void* zcomm);
int hzg_wave_join(hzg_ctx* ctx, void* comm, void* zcomm);

/* Step-wise driving for multi-GPU jobs (one rank's slot range of the
 * ordering per GPU, blocks exchanged between steps by the caller):
 * hzg_collect folds the per-pair counters of all steps of the schedule
 * (i.e. of the sweep just run with hzg_run_steps) and returns them
 * (synchronous); hzg_rescale_z runs the inter-sweep Z rescale of
 * blocked.py:540-542 on every column (asynchronous). */
int hzg_collect(hzg_ctx* ctx, int64_t* total, int64_t* big);
int hzg_rescale_z(hzg_ctx* ctx);

/* Final rescale, unborder to n0 columns (mF0 / mG0 rows) and stable
 * descending sort by sigma (sort = 0 keeps the column order, as
 * gsvd_blocked does), into caller-provided device outputs: U (mF0 x
 * n0), V (mG0 x n0), Z (n0 x n0) planes and three length-n0 vectors.
 * Synchronous. */
int hzg_finalize(hzg_ctx* ctx, int64_t n0, int64_t mF0, int64_t mG0, int32_t sort, double* Ur, double* Ui,
                 double* Vr, double* Vi, double* Zr, double* Zi, double* sigF, double* sigG, double* sig);

/* Kernel-level check entry: run the inner block kernel (Cholesky + in-block
 * prescale + pointwise sweeps + theta rescale) on one block pair given its
 * two tw x tw Grammians in host memory (column-major planes; imaginary
 * planes ignored for real).  Outputs Z~ (host, planes) and counters
 * {total, big, status, inner sweeps}.  Synchronous. */
int hzg_test_block(int32_t tw, int32_t is_complex, const hzg_config* cfg, double epsn, const double* gFr,
                   const double* gFi, const double* gGr, const double* gGi, double* zr, double* zi,
                   int32_t* counts4);

/* Per-kernel timing: with on != 0 the captured sweep graph records CUDA
 * events around every Grammian / inner / postmultiply launch (on the stream
 * they run on); hzg_kernel_times returns the accumulated milliseconds and
 * launch counts per kind {grammian, inner, postmultiply} since the last
 * reset.  Must be set before the first hzg_sweep. */
int hzg_set_timing(hzg_ctx* ctx, int32_t on);
int hzg_kernel_times(hzg_ctx* ctx, double* ms3, int64_t* launches3, int32_t reset);

/* Diagnostics: copy the per-step, per-pair counters of the last sweep,
 * int32 [osteps][npairs][4] = {total, big, status, inner sweeps}, to host
 * memory.  Returns the number of int32 written via *count. */
int hzg_step_counters(hzg_ctx* ctx, int32_t* out, int64_t capacity, int64_t* count);

/* Diagnostics: enable (before the first sweep) and read the cycle counts
 * CTA 0 / warp 0 of the inner kernel spends in its phases A (dot
 * products), B (2x2 transforms), C (column updates), plus the step count. */
int hzg_debug_phases(hzg_ctx* ctx, int32_t enable, int64_t* out4);

/* Kernel launches of this library per hzg_sweep, and per solve outside the
 * sweeps (hzg_init_fgz + hzg_finalize). */
int hzg_launch_counts(const hzg_ctx* ctx, int64_t* per_sweep, int64_t* per_solve_fixed);

/* Self-check of the branch-free FP64 division / square root used by the
 * 2x2 kernels against the IEEE operators on n random operand pairs:
 * counts4 = {divisions checked, mismatches, roots checked, mismatches}. */
int hzg_test_fastmath(int64_t n, uint64_t seed, int64_t* counts4);

/* Single block operations of the reference's public API, on device
 * pointers (column-major planes), reference operation order (bitwise the
 * reference), synchronous on `stream`:
 *   hzg_op_grammian       -> _gram_of_pair / _k_grammian    (blocked.py:340-347, :40-56):
 *                            the 2w x 2w Grammian of the m x 2w stack Y
 *   hzg_op_cholesky_upper -> cholesky_upper                 (blocked.py:350-355, :59-94), in place
 *   hzg_op_qr_shorten     -> qr_shorten                     (blocked.py:358-367, :97-217)
 *   hzg_op_postmultiply   -> postmultiply                   (blocked.py:370-381, :220-250), Y in place
 *   hzg_op_rescale        -> rescale_z                      (blocked.py:384-401, :253-295), in place;
 *                            Z has mZ rows, sigF/sigG/sig written when final != 0 */
/* Householder R factor, in place, of the m x nc column-major matrix A
 * (m >= nc; Ai NULL for real), with column pivoting when pivot != 0 (the
 * column of largest remaining norm at each step, ties to the lowest
 * index; jpvt[nc] is permuted alongside), bitwise the reference's
 * _k_qr_rfactor (blocked.py:97-217) as used by preprocess_tall
 * (blocked.py:405-428).  *result = the reference's return value: 1 when
 * a column vanished or a diagonal fell below tol_scale times its column's
 * entry norm, else 0.  Device pointers; synchronous on `stream`. */
int hzg_op_qr_rfactor(int64_t m, int32_t nc, int32_t is_complex, int32_t pivot, double tol_scale, double* Ar,
                      double* Ai, int64_t* jpvt, int32_t* result, void* stream);

int hzg_op_grammian(int64_t m, int32_t w, int32_t is_complex, int32_t compensated, const double* Yr,
                    const double* Yi, double* Ar, double* Ai, void* stream);
int hzg_op_cholesky_upper(int32_t tw, int32_t is_complex, double* Ar, double* Ai, void* stream);
int hzg_op_qr_shorten(int64_t m, int32_t w, int32_t is_complex, const double* Yr, const double* Yi, double* Rr,
                      double* Ri, void* stream);
int hzg_op_postmultiply(int64_t m, int32_t w, int32_t is_complex, double* Yr, double* Yi, const double* Zr,
                        const double* Zi, void* stream);
int hzg_op_rescale(int64_t mF, int64_t mG, int64_t n, int32_t is_complex, int32_t compensated, int32_t final,
                   double* Fr, double* Fi, double* Gr, double* Gi, double* Zr, double* Zi, int64_t mZ, double* sigF,
                   double* sigG, double* sig, void* stream);

/* ---- multi-GPU data plane (the reference's per-step block
 * exchange, distsim.py:103-144, re-designed as device-to-device NCCL over
 * NVLink inside the library).  One process per GPU; each rank's context is
 * set to its slot range of the circle-position schedule (hzg_set_schedule)
 * and holds full-size planes (a block lives at its logical column offset).
 * NCCL is resolved at run time from the process (dlopen). */

/* ncclUniqueId of a new job (rank 0 calls it and broadcasts the bytes). */
int hzg_comm_unique_id(void* id_out);
size_t hzg_comm_unique_id_bytes(void);
/* ncclCommInitRank on ctx's device (collective over the nranks ranks). */
int hzg_comm_attach(hzg_ctx* ctx, int32_t nranks, int32_t rank, const void* unique_id);
/* The block moves after every outer step: moves[3q .. 3q+2] = (block,
 * src rank, dst rank); step k's moves are q in [offsets[k], offsets[k+1]).
 * Moves not involving this rank are ignored.  osteps must match the
 * schedule. */
int hzg_comm_set_moves(hzg_ctx* ctx, const int32_t* moves, const int32_t* offsets, int32_t osteps);
/* One outer sweep of this rank as ONE captured CUDA graph: its pairs of
 * every step (position groups), the grouped ncclSend/ncclRecv block
 * exchange after every step, the counter fold, ncclAllReduce of the
 * counters and status indicators, the Z rescale gated on the global big
 * count, ncclAllReduce of its status.  Returns the GLOBAL counters; every
 * rank returns the same status.  Synchronous (one host sync per sweep). */
int hzg_dist_sweep(hzg_ctx* ctx, int64_t* total, int64_t* big);
/* hzg_dist_sweep in two halves (one process driving several GPUs launches
 * every rank's sweep graph before waiting for any). */
int hzg_dist_sweep_launch(hzg_ctx* ctx);
int hzg_dist_sweep_wait(hzg_ctx* ctx, int64_t* total, int64_t* big);
/* One process, n GPUs: ncclCommInitAll over the contexts' devices (rank i =
 * ctxs[i]); the grouped block exchange across them. */
int hzg_comm_attach_all(hzg_ctx** ctxs, int32_t n);
int hzg_comm_exchange_all(hzg_ctx** ctxs, int32_t n, const int32_t* moves, int32_t count);
/* Immediate grouped exchange of whole blocks (e.g. the final gather of
 * every block to rank 0); synchronous. */
int hzg_comm_exchange(hzg_ctx* ctx, const int32_t* moves, int32_t count);
/* Destroy the communicator (hzg_destroy does it too). */
int hzg_comm_detach(hzg_ctx* ctx);

/* ---- accuracy check (the reference's accuracy_report, harness.py:323-465) */

/* In-place LU with complete pivoting of the n x n column-major planes A
 * (ld >= n): _k_lu_complete (harness.py:323-371), bitwise the reference's
 * factors.  rp, cp (device int64[n]) must hold 0..n-1 on entry and receive
 * the row / column permutations; *status (device) = 1 on a zero pivot.
 * workspace: hzg_lu_workspace_bytes(n) bytes.  Asynchronous on `stream`. */
size_t hzg_lu_workspace_bytes(int64_t n);
int hzg_lu_complete(int64_t n, int32_t is_complex, double* Ar, double* Ai, int64_t ld, int64_t* rp, int64_t* cp,
                    void* workspace, int32_t* status, void* stream);
/* C = op(A) B (op(A) = A, or A^H with trans_a), every entry a compensated
 * dot product (matmul_compensated, harness.py:151-196). */
int hzg_gemm_comp(int64_t m, int64_t n, int64_t k, int32_t is_complex, int32_t trans_a, const double* Ar,
                  const double* Ai, int64_t lda, const double* Br, const double* Bi, int64_t ldb, double* Cr,
                  double* Ci, int64_t ldc, void* stream);
/* Compensated sum of |A - B|^2 (B null: |A|^2; eye: B = I) over rows x cols,
 * as nblocks (sum, error) pairs in partials[2 * nblocks] (_frob_comp,
 * harness.py:208-216). */
int hzg_sumsq_comp(int64_t rows, int64_t cols, const double* Ar, const double* Ai, int64_t lda, const double* Br,
                   const double* Bi, int64_t ldb, int32_t eye, double* partials, int32_t nblocks, void* stream);

const char* hzg_last_error(const hzg_ctx* ctx);
void hzg_destroy(hzg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* HZG_H_ */
