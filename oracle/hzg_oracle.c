/*
 * hzg_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference package's blocked one-sided
 * Hari-Zimmermann GSVD (arxiv/paper_1909_00101, pkg/src/hzgsvd).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it, and only as the checker or the timed CPU
 * baseline -- never as the product path.
 *
 * Every function follows the reference statement by statement (same
 * pairwise-tree reductions, same fma placement, same branch structure) so
 * that, compiled with -ffp-contract=off and a hardware fma, its output is
 * bitwise identical to the numba reference on the same inputs.  That claim
 * is checked against the committed golden fixtures (tests/golden/).
 *
 * Storage: column-major ("Fortran") planes, split real / imaginary, exactly
 * the reference's MatrixPlanePair model (core.py:26-69).  For real problems
 * the imaginary planes must still be valid buffers (the reference keeps a
 * zero plane too, pointwise.py:300-304).
 */
#include <math.h>
#include <time.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define HZO_OK 0
#define HZO_RANK 1
#define HZO_NOT_PD 2
#define HZO_INVALID 4

static const double EPS = 2.220446049250313080847e-16; /* 2**-52, kernel2x2.py:32 */
static const double RSQRT2 = 0.70710678118654746;       /* 1/math.sqrt(2), kernel2x2.py:33 */

typedef struct {
  int prescale;          /* variant in {0,1,4,5}      pointwise.py:78 */
  int compensated;       /* odd variant               pointwise.py:79 */
  int crit_c2;           /* variant >= 4              pointwise.py:77 */
  int sorting;           /* pointwise.py:54 */
  int max_inner_sweeps;  /* 30 fb / 1 bo              pointwise.py:80-81 */
  int max_outer_sweeps;  /* pointwise.py:56 */
  int block_width;       /* pointwise.py:57 */
  int outer_mm;          /* outer_kind == "mm" */
  int inner_mm;          /* inner_kind == "mm" */
  int fallback_qr;       /* pointwise.py:59 */
  int shorten_qr;        /* shorten == "qr"           pointwise.py:60 */
  double gate_eps;       /* pointwise.py:58 */
} hzo_cfg;

typedef struct {
  int64_t sweeps, total, big;
  int converged;
  int fail_pair;         /* first failing pair index of the failing step, -1 */
  double step_seconds;   /* wall time spent in outer steps (timing only, not numerics) */
} hzo_stats;

/* ------------------------------------------------------------------------ */
/* dotprod.py                                                               */
/* ------------------------------------------------------------------------ */

static int64_t pow2(int64_t n) { /* dotprod.py:71-76 */
  int64_t m = 1;
  while (m < n) m *= 2;
  return m;
}

static double tree(double* buf, int64_t n) { /* dotprod.py:79-91 */
  int64_t m = pow2(n);
  for (int64_t i = n; i < m; ++i) buf[i] = 0.0;
  while (m > 1) {
    int64_t h = m / 2;
    for (int64_t i = 0; i < h; ++i) buf[i] = buf[2 * i] + buf[2 * i + 1];
    m = h;
  }
  return buf[0];
}

static double tree_comp(double* buf, int64_t n, double* err_out) { /* dotprod.py:103-122 */
  int64_t m = pow2(n);
  for (int64_t i = n; i < m; ++i) buf[i] = 0.0;
  double err = 0.0;
  while (m > 1) {
    int64_t h = m / 2;
    for (int64_t i = 0; i < h; ++i) {
      double a = buf[2 * i], b = buf[2 * i + 1];
      double s = a + b;
      double ap = s - b;
      double bp = s - ap;
      err += (a - ap) + (b - bp);
      buf[i] = s;
    }
    m = h;
  }
  *err_out = err;
  return buf[0];
}

static double dot_real_s(const double* a, const double* b, int64_t n, double* buf) { /* :125-130 */
  for (int64_t t = 0; t < n; ++t) buf[t] = a[t] * b[t];
  return tree(buf, n);
}

static double dot_real_comp_s(const double* a, const double* b, int64_t n, double* buf) { /* :133-143 */
  for (int64_t t = 0; t < n; ++t) {
    double p = a[t] * b[t];
    buf[t] = fma(a[t], b[t], -p);
  }
  double d = tree(buf, n);
  for (int64_t t = 0; t < n; ++t) buf[t] = a[t] * b[t];
  double e;
  double c = tree_comp(buf, n, &e);
  return (d + e) + c;
}

static void dot_cplx_s(const double* ar, const double* ai, const double* br, const double* bi,
                       int conj_first, int64_t n, double* buf, double* re, double* im) { /* :146-155 */
  double s = conj_first ? -1.0 : 1.0;
  for (int64_t t = 0; t < n; ++t) buf[t] = fma(ar[t], br[t], -((s * ai[t]) * bi[t]));
  *re = tree(buf, n);
  for (int64_t t = 0; t < n; ++t) buf[t] = fma(ar[t], bi[t], (s * ai[t]) * br[t]);
  *im = tree(buf, n);
}

static double comp_combine(double cr, double ci, double dr, double di) { /* :158-163 */
  double e = dr + di;
  if (cr <= ci) return (e + cr) + ci;
  return (e + ci) + cr;
}

static void dot_cplx_comp_s(const double* ar, const double* ai, const double* br, const double* bi,
                            int conj_first, int64_t n, double* buf, double* re, double* im) { /* :166-203 */
  double sv = conj_first ? 1.0 : -1.0;
  double sq = conj_first ? -1.0 : 1.0;
  double eu, ev, ep, eq;
  for (int64_t t = 0; t < n; ++t) buf[t] = ar[t] * br[t];
  double cu = tree_comp(buf, n, &eu);
  for (int64_t t = 0; t < n; ++t) { double p = ar[t] * br[t]; buf[t] = fma(ar[t], br[t], -p); }
  double du = tree(buf, n);
  for (int64_t t = 0; t < n; ++t) buf[t] = sv * (ai[t] * bi[t]);
  double cv = tree_comp(buf, n, &ev);
  for (int64_t t = 0; t < n; ++t) { double p = ai[t] * bi[t]; buf[t] = sv * fma(ai[t], bi[t], -p); }
  double dv = tree(buf, n);
  *re = comp_combine(cu, cv, du + eu, dv + ev);
  for (int64_t t = 0; t < n; ++t) buf[t] = ar[t] * bi[t];
  double cp = tree_comp(buf, n, &ep);
  for (int64_t t = 0; t < n; ++t) { double p = ar[t] * bi[t]; buf[t] = fma(ar[t], bi[t], -p); }
  double dp = tree(buf, n);
  for (int64_t t = 0; t < n; ++t) buf[t] = sq * (ai[t] * br[t]);
  double cq = tree_comp(buf, n, &eq);
  for (int64_t t = 0; t < n; ++t) { double p = ai[t] * br[t]; buf[t] = sq * fma(ai[t], br[t], -p); }
  double dq = tree(buf, n);
  *im = comp_combine(cp, cq, dp + ep, dq + eq);
}

static double norm_sq_real_s(const double* v, int64_t n, double* buf) { /* :206-211 */
  for (int64_t t = 0; t < n; ++t) buf[t] = v[t] * v[t];
  return tree(buf, n);
}

static double norm_sq_real_comp_s(const double* v, int64_t n, double* buf) { /* :214-224 */
  for (int64_t t = 0; t < n; ++t) { double p = v[t] * v[t]; buf[t] = fma(v[t], v[t], -p); }
  double d = tree(buf, n);
  for (int64_t t = 0; t < n; ++t) buf[t] = v[t] * v[t];
  double e;
  double c = tree_comp(buf, n, &e);
  return (d + e) + c;
}

static double norm_sq_cplx_s(const double* vr, const double* vi, int64_t n, double* buf) { /* :227-232 */
  for (int64_t t = 0; t < n; ++t) buf[t] = fma(vi[t], vi[t], vr[t] * vr[t]);
  return tree(buf, n);
}

static double norm_sq_cplx_comp_s(const double* vr, const double* vi, int64_t n, double* buf) { /* :235-252 */
  double er, ei;
  for (int64_t t = 0; t < n; ++t) buf[t] = vr[t] * vr[t];
  double cr = tree_comp(buf, n, &er);
  for (int64_t t = 0; t < n; ++t) { double p = vr[t] * vr[t]; buf[t] = fma(vr[t], vr[t], -p); }
  double dr = tree(buf, n);
  for (int64_t t = 0; t < n; ++t) buf[t] = vi[t] * vi[t];
  double ci = tree_comp(buf, n, &ei);
  for (int64_t t = 0; t < n; ++t) { double p = vi[t] * vi[t]; buf[t] = fma(vi[t], vi[t], -p); }
  double di = tree(buf, n);
  return comp_combine(cr, ci, dr + er, di + ei);
}

/* public single-vector entry points (dotprod.py:312-363) for the tests */
double hzo_tree_reduce(const double* x, int64_t n) {
  double* buf = (double*)malloc(sizeof(double) * pow2(n));
  memcpy(buf, x, sizeof(double) * n);
  double r = tree(buf, n);
  free(buf);
  return r;
}

/* ------------------------------------------------------------------------ */
/* a column-major plane view                                                */
/* ------------------------------------------------------------------------ */

typedef struct {
  double* re;
  double* im;
  int64_t rows, cols, ld;
} plane_t;

#define COL(P, j) ((P).re + (int64_t)(j) * (P).ld)
#define COLI(P, j) ((P).im + (int64_t)(j) * (P).ld)

/* pointwise.py:100-108 */
static double col_norm(plane_t Y, int64_t j, int cplx, int comp, double* buf) {
  if (cplx) {
    if (comp) return norm_sq_cplx_comp_s(COL(Y, j), COLI(Y, j), Y.rows, buf);
    return norm_sq_cplx_s(COL(Y, j), COLI(Y, j), Y.rows, buf);
  }
  if (comp) return norm_sq_real_comp_s(COL(Y, j), Y.rows, buf);
  return norm_sq_real_s(COL(Y, j), Y.rows, buf);
}

/* pointwise.py:111-120 */
static void col_dot(plane_t Y, int64_t i, int64_t j, int cplx, int comp, double* buf, double* re, double* im) {
  if (cplx) {
    if (comp) dot_cplx_comp_s(COL(Y, i), COLI(Y, i), COL(Y, j), COLI(Y, j), 1, Y.rows, buf, re, im);
    else dot_cplx_s(COL(Y, i), COLI(Y, i), COL(Y, j), COLI(Y, j), 1, Y.rows, buf, re, im);
    return;
  }
  *re = comp ? dot_real_comp_s(COL(Y, i), COL(Y, j), Y.rows, buf) : dot_real_s(COL(Y, i), COL(Y, j), Y.rows, buf);
  *im = 0.0;
}

/* pointwise.py:123-133 */
static void swap_cols(plane_t Y, int64_t i, int64_t j, int cplx) {
  for (int64_t r = 0; r < Y.rows; ++r) {
    double t = COL(Y, i)[r]; COL(Y, i)[r] = COL(Y, j)[r]; COL(Y, j)[r] = t;
    if (cplx) { t = COLI(Y, i)[r]; COLI(Y, i)[r] = COLI(Y, j)[r]; COLI(Y, j)[r] = t; }
  }
}

/* pointwise.py:136-158 */
static void update_cols(plane_t Y, int64_t i, int64_t j, double z11, double z12r, double z12i,
                        double z21r, double z21i, double z22, int cplx) {
  double *yi = COL(Y, i), *yj = COL(Y, j);
  if (cplx) {
    double *yii = COLI(Y, i), *yji = COLI(Y, j);
    for (int64_t r = 0; r < Y.rows; ++r) {
      double yir = yi[r], yjr = yj[r], yiI = yii[r], yjI = yji[r];
      double nir = fma(yjr, z21r, fma(-yjI, z21i, yir * z11));
      double nii = fma(yjr, z21i, fma(yjI, z21r, yiI * z11));
      double njr = fma(yir, z12r, fma(-yiI, z12i, yjr * z22));
      double nji = fma(yir, z12i, fma(yiI, z12r, yjI * z22));
      yi[r] = nir; yii[r] = nii; yj[r] = njr; yji[r] = nji;
    }
  } else {
    for (int64_t r = 0; r < Y.rows; ++r) {
      double yir = yi[r], yjr = yj[r];
      double ni = fma(yjr, z21r, yir * z11);
      double nj = fma(yir, z12r, yjr * z22);
      yi[r] = ni; yj[r] = nj;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* kernel2x2.py                                                             */
/* ------------------------------------------------------------------------ */

/* kernel2x2.py:92-111 */
static void rescale2(double* a11, double* a12r, double* a12i, double* a22, double b11, double* b12r,
                     double* b12i, double b22, double* d11, double* d22) {
  *d11 = 1.0; *d22 = 1.0;
  if (b11 != 1.0) {
    *a11 = *a11 / b11;
    *d11 = 1.0 / sqrt(b11);
    *a12r *= *d11; *a12i *= *d11; *b12r *= *d11; *b12i *= *d11;
  }
  if (b22 != 1.0) {
    *a22 = *a22 / b22;
    *d22 = 1.0 / sqrt(b22);
    *a12r *= *d22; *a12i *= *d22; *b12r *= *d22; *b12i *= *d22;
  }
}

/* kernel2x2.py:114-119 */
static int gate(double a11, double a12r, double a12i, double a22, double b12r, double b12i, double epsn) {
  int ok_a = hypot(a12r, a12i) < sqrt(a11) * sqrt(a22) * epsn;
  int ok_b = hypot(b12r, b12i) < epsn;
  return ok_a && ok_b;
}

/* kernel2x2.py:122-130 */
static void cos_sin_from_tan(double tg, double* c, double* s) {
  double t2 = fma(tg, tg, 1.0);
  if (isinf(t2) || isinf(tg)) { *c = 0.0; *s = copysign(1.0, tg); return; }
  *c = 1.0 / sqrt(t2);
  *s = tg * *c;
}

/* kernel2x2.py:133-165; out = z11 z12 z21 z22 cosphi cospsi */
static void transform_real(double a11, double a12, double a22, double x, double* o) {
  double t = sqrt(fma(-x, x, 1.0));
  double num = t * (a22 - a11);
  double den = fma(-(a11 + a22), x, 2.0 * a12);
  if (num == 0.0 && den == 0.0) {
    double ax = fabs(x);
    double sp = 1.0 / sqrt(1.0 + ax);
    double sm = 1.0 / sqrt(1.0 - ax);
    double z11 = RSQRT2 * sp, z12 = -(RSQRT2 * sm), z21 = RSQRT2 * sp, z22 = RSQRT2 * sm;
    o[0] = z11; o[1] = z12; o[2] = z21; o[3] = z22; o[4] = z11 * t; o[5] = z22 * t;
    return;
  }
  double sqp = sqrt(1.0 + x);
  double sqm = sqrt(1.0 - x);
  double xi = x / (sqp + sqm);
  double eta = x / ((1.0 + sqp) * (1.0 + sqm));
  double ct2 = num / den;
  double tanth = copysign(1.0, ct2) / (fabs(ct2) + sqrt(fma(ct2, ct2, 1.0)));
  double cth, sth;
  cos_sin_from_tan(tanth, &cth, &sth);
  double cosphi = fma(xi, fma(-eta, cth, sth), cth);
  double cospsi = fma(-xi, fma(eta, cth, sth), cth);
  double sinphi = fma(-xi, fma(eta, sth, cth), sth);
  double sinpsi = fma(xi, fma(-eta, sth, cth), sth);
  o[0] = cosphi / t; o[1] = sinphi / t; o[2] = -(sinpsi / t); o[3] = cospsi / t;
  o[4] = cosphi; o[5] = cospsi;
}

/* kernel2x2.py:168-232; out = z11 z12r z12i z21r z21i z22 cosphi cospsi */
static void transform_cplx(double a11, double a12r, double a12i, double a22, double b12r, double b12i, double* o) {
  if (a12i == 0.0 && b12i == 0.0) {
    double r[6];
    transform_real(a11, a12r, a22, b12r, r);
    o[0] = r[0]; o[1] = r[1]; o[2] = 0.0; o[3] = r[2]; o[4] = 0.0; o[5] = r[3]; o[6] = r[4]; o[7] = r[5];
    return;
  }
  double x = hypot(b12r, b12i);
  double czr, czi;
  if (x == 0.0) { czr = 1.0; czi = 0.0; } else { czr = b12r / x; czi = b12i / x; }
  double u = fma(a12r, czr, a12i * czi);
  double v = fma(a12i, czr, -(a12r * czi));
  double h = a22 - a11;
  double t = sqrt(fma(-x, x, 1.0));
  if (v == 0.0 && h == 0.0) {
    double sp = 1.0 / sqrt(1.0 + x);
    double sm = 1.0 / sqrt(1.0 - x);
    double z11 = RSQRT2 * sp, z22 = RSQRT2 * sm;
    double w = RSQRT2 * sm;
    double z12r = -(w * czr), z12i = -(w * czi);
    w = RSQRT2 * sp;
    double z21r = w * czr, z21i = -(w * czi);
    o[0] = z11; o[1] = z12r; o[2] = z12i; o[3] = z21r; o[4] = z21i; o[5] = z22; o[6] = z11 * t; o[7] = z22 * t;
    return;
  }
  double tau = copysign(1.0, h);
  double num = fma(-(a11 + a22), x, 2.0 * u);
  double den = t * hypot(h, 2.0 * v);
  double t2t = (tau * num) / den;
  double tg = (2.0 * v) / h;
  double c2t, s2t, cg, sg;
  cos_sin_from_tan(t2t, &c2t, &s2t);
  cos_sin_from_tan(tg, &cg, &sg);
  double tcg = t * cg;
  double cosphi = sqrt(fma(tcg, c2t, fma(x, s2t, 1.0))) * RSQRT2;
  double cospsi = sqrt(fma(tcg, c2t, fma(-x, s2t, 1.0))) * RSQRT2;
  double tsg = t * sg;
  double wi = tsg * c2t;
  double d = 2.0 * cospsi;
  double er = (s2t - x) / d;
  double ei = wi / d;
  double z12r = fma(czr, er, -(czi * ei));
  double z12i = fma(czr, ei, czi * er);
  d = 2.0 * cosphi;
  double fr = (s2t + x) / d;
  double fi = -wi / d;
  double br = fma(czr, fr, czi * fi);
  double bi = fma(czr, fi, -(czi * fr));
  o[0] = cosphi / t; o[1] = z12r / t; o[2] = z12i / t; o[3] = -(br / t); o[4] = -(bi / t); o[5] = cospsi / t;
  o[6] = cosphi; o[7] = cospsi;
}

/* kernel2x2.py:235-240 */
static void diag_after_real(double z11, double z12, double z21, double z22, double a11, double a12, double a22,
                            double* a1pp, double* a2pp) {
  *a1pp = z11 * z11 * a11 + 2.0 * (z11 * z21) * a12 + z21 * z21 * a22;
  *a2pp = z12 * z12 * a11 + 2.0 * (z22 * z12) * a12 + z22 * z22 * a22;
}

/* exported for the kernel-level parity tests: out = z11 z12r z12i z21r z21i z22 cosphi cospsi */
void hzo_transform(int cplx, double a11, double a12r, double a12i, double a22, double b12r, double b12i, double* o) {
  if (cplx) transform_cplx(a11, a12r, a12i, a22, b12r, b12i, o);
  else {
    double r[6];
    transform_real(a11, a12r, a22, b12r, r);
    o[0] = r[0]; o[1] = r[1]; o[2] = 0.0; o[3] = r[2]; o[4] = 0.0; o[5] = r[3]; o[6] = r[4]; o[7] = r[5];
  }
}

/* ------------------------------------------------------------------------ */
/* pointwise.py kernels                                                     */
/* ------------------------------------------------------------------------ */

/* pointwise.py:161-219; returns applied, sets *big, *bad */
static int process_pivot(plane_t F, plane_t G, plane_t Z, int64_t i, int64_t j, int cplx, int per_step_rescale,
                         int comp, int crit_c2, int sort, double epsn, double* buf, int* big_out, int* bad) {
  double a12r, a12i, b12r, b12i;
  double a11 = col_norm(F, i, cplx, comp, buf);
  double a22 = col_norm(F, j, cplx, comp, buf);
  col_dot(F, i, j, cplx, comp, buf, &a12r, &a12i);
  double b11 = col_norm(G, i, cplx, comp, buf);
  double b22 = col_norm(G, j, cplx, comp, buf);
  col_dot(G, i, j, cplx, comp, buf, &b12r, &b12i);
  *big_out = 0; *bad = 0;
  if (!(a11 > 0.0 && a22 > 0.0 && b11 > 0.0 && b22 > 0.0)) { *bad = 1; return 0; }
  double d11 = 1.0, d22 = 1.0;
  if (per_step_rescale) rescale2(&a11, &a12r, &a12i, &a22, b11, &b12r, &b12i, b22, &d11, &d22);
  if (gate(a11, a12r, a12i, a22, b12r, b12i, epsn)) {
    if (sort && a11 < a22) { swap_cols(F, i, j, cplx); swap_cols(G, i, j, cplx); swap_cols(Z, i, j, cplx); }
    return 0;
  }
  double z11, z12r, z12i, z21r, z21i, z22, cphi, cpsi;
  if (cplx) {
    double o[8];
    transform_cplx(a11, a12r, a12i, a22, b12r, b12i, o);
    z11 = o[0]; z12r = o[1]; z12i = o[2]; z21r = o[3]; z21i = o[4]; z22 = o[5]; cphi = o[6]; cpsi = o[7];
  } else {
    double o[6];
    transform_real(a11, a12r, a22, b12r, o);
    z11 = o[0]; z12r = o[1]; z21r = o[2]; z22 = o[3]; cphi = o[4]; cpsi = o[5];
    z12i = 0.0; z21i = 0.0;
  }
  int big;
  if (crit_c2) big = (cphi == 1.0 && cpsi == 1.0) ? 0 : 1;
  else big = (z11 == 1.0 && z22 == 1.0) ? 0 : 1;
  int swap = 0;
  if (sort && !cplx) {
    double a1pp, a2pp;
    diag_after_real(z11, z12r, z21r, z22, a11, a12r, a22, &a1pp, &a2pp);
    swap = a1pp < a2pp;
  }
  z11 = z11 * d11; z12r = z12r * d11; z12i = z12i * d11;
  z21r = z21r * d22; z21i = z21i * d22; z22 = z22 * d22;
  update_cols(F, i, j, z11, z12r, z12i, z21r, z21i, z22, cplx);
  update_cols(G, i, j, z11, z12r, z12i, z21r, z21i, z22, cplx);
  update_cols(Z, i, j, z11, z12r, z12i, z21r, z21i, z22, cplx);
  if (sort && cplx) {
    double ni = col_norm(F, i, cplx, comp, buf);
    double nj = col_norm(F, j, cplx, comp, buf);
    swap = ni < nj;
  }
  if (swap) { swap_cols(F, i, j, cplx); swap_cols(G, i, j, cplx); swap_cols(Z, i, j, cplx); }
  *big_out = big;
  return 1;
}

/* pointwise.py:222-251; table: steps x half x 2 int32. returns bad */
static int pointwise(plane_t F, plane_t G, plane_t Z, int cplx, const int32_t* table, int steps, int half,
                     int per_step_rescale, int comp, int crit_c2, int sort, int max_sweeps, double epsn,
                     double* buf, int64_t* sweeps_o, int64_t* total_o, int64_t* big_o, int* conv_o) {
  int64_t total = 0, big = 0, sweeps = 0;
  int converged = 0;
  for (int sw = 0; sw < max_sweeps; ++sw) {
    int64_t s_cnt = 0, b_cnt = 0;
    for (int st = 0; st < steps; ++st) {
      for (int l = 0; l < half; ++l) {
        int b, bad;
        int s = process_pivot(F, G, Z, table[(st * half + l) * 2], table[(st * half + l) * 2 + 1], cplx,
                              per_step_rescale, comp, crit_c2, sort, epsn, buf, &b, &bad);
        if (bad) { *sweeps_o = sweeps; *total_o = total; *big_o = big; *conv_o = 0; return 1; }
        s_cnt += s; b_cnt += b;
      }
    }
    sweeps += 1;
    if (s_cnt == 0) { converged = 1; break; }
    total += s_cnt; big += b_cnt;
  }
  *sweeps_o = sweeps; *total_o = total; *big_o = big; *conv_o = converged;
  return 0;
}

/* pointwise.py:254-274 */
static int prescale(plane_t F, plane_t G, double* z0, int cplx, int comp, double* buf) {
  for (int64_t j = 0; j < G.cols; ++j) {
    double ng2 = col_norm(G, j, cplx, comp, buf);
    if (!(ng2 > 0.0)) return 1;
    double z = 1.0 / sqrt(ng2);
    z0[j] = z;
    if (z != 1.0) {
      for (int64_t r = 0; r < F.rows; ++r) { COL(F, j)[r] *= z; if (cplx) COLI(F, j)[r] *= z; }
      for (int64_t r = 0; r < G.rows; ++r) { COL(G, j)[r] *= z; if (cplx) COLI(G, j)[r] *= z; }
    }
  }
  return 0;
}

/* pointwise.py:277-293 */
static int theta_rescale(plane_t F, plane_t G, plane_t Z, int cplx, int comp, double* buf) {
  for (int64_t j = 0; j < F.cols; ++j) {
    double s = col_norm(F, j, cplx, comp, buf) + col_norm(G, j, cplx, comp, buf);
    if (!(s > 0.0)) return 1;
    double th = 1.0 / sqrt(s);
    if (th != 1.0)
      for (int64_t r = 0; r < Z.rows; ++r) { COL(Z, j)[r] *= th; if (cplx) COLI(Z, j)[r] *= th; }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* strategies.py                                                            */
/* ------------------------------------------------------------------------ */

static int cmp_pair(const void* a, const void* b) {
  const int32_t* x = (const int32_t*)a; const int32_t* y = (const int32_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

/* strategies.py:45-93; out: steps x n/2 x 2; returns the number of steps */
int hzo_gen_table(int mm, int n, int32_t* out) {
  int half = n / 2;
  if (!mm) { /* _tournament :59-70 */
    int* others = (int*)malloc(sizeof(int) * n);
    int* line = (int*)malloc(sizeof(int) * n);
    for (int i = 1; i < n; ++i) others[i - 1] = i;
    for (int st = 0; st < n - 1; ++st) {
      line[0] = 0;
      for (int i = 1; i < n; ++i) line[i] = others[i - 1];
      int32_t* row = out + (int64_t)st * half * 2;
      for (int i = 0; i < half; ++i) {
        int a = line[i], b = line[n - 1 - i];
        row[2 * i] = a < b ? a : b; row[2 * i + 1] = a < b ? b : a;
      }
      qsort(row, half, 2 * sizeof(int32_t), cmp_pair);
      int last = others[n - 2];
      for (int i = n - 2; i > 0; --i) others[i] = others[i - 1];
      others[0] = last;
    }
    free(others); free(line);
    return n - 1;
  }
  /* _modified_modulus :73-93 */
  char* seen = (char*)malloc(n);
  for (int k = 0; k < n; ++k) {
    memset(seen, 0, n);
    int32_t* row = out + (int64_t)k * half * 2;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      if (seen[i]) continue;
      int j = ((k - i) % n + n) % n;
      if (j == i || seen[j]) continue;
      seen[i] = 1; seen[j] = 1;
      row[2 * cnt] = i < j ? i : j; row[2 * cnt + 1] = i < j ? j : i; ++cnt;
    }
    if (k % 2 == 0) {
      int a = k / 2, b = a + half;
      if (!seen[a]) { row[2 * cnt] = a < b ? a : b; row[2 * cnt + 1] = a < b ? b : a; ++cnt; }
    }
    qsort(row, cnt, 2 * sizeof(int32_t), cmp_pair);
  }
  free(seen);
  return n;
}

/* ------------------------------------------------------------------------ */
/* blocked.py kernels                                                       */
/* ------------------------------------------------------------------------ */

/* blocked.py:40-56; A: tw x tw (ld tw) */
static void grammian(plane_t Y, int64_t c0, int64_t c1, int w, int cplx, int comp, double* Ar, double* Ai,
                     double* buf) {
  int tw = 2 * w;
  for (int r = 0; r < tw; ++r) {
    int64_t cr = r < w ? c0 + r : c1 + (r - w);
    Ar[r + r * tw] = col_norm(Y, cr, cplx, comp, buf);
    Ai[r + r * tw] = 0.0;
    for (int s = r + 1; s < tw; ++s) {
      int64_t cs = s < w ? c0 + s : c1 + (s - w);
      double re, im;
      col_dot(Y, cr, cs, cplx, comp, buf, &re, &im);
      Ar[r + s * tw] = re; Ai[r + s * tw] = im;
      Ar[s + r * tw] = re; Ai[s + r * tw] = -im;
    }
  }
}

/* blocked.py:59-94; m x m (ld m) */
int hzo_cholesky_upper(int m, int cplx, double* Ar, double* Ai) {
#define A_(x, y) Ar[(x) + (int64_t)(y) * m]
#define AI_(x, y) Ai[(x) + (int64_t)(y) * m]
  for (int j = 0; j < m; ++j) {
    double d = A_(j, j);
    if (!(d > 0.0) || !isfinite(d)) return 1;
    double rt = sqrt(d);
    double rinv = 1.0 / rt;
    A_(j, j) = rt; AI_(j, j) = 0.0;
    for (int x = j + 1; x < m; ++x) { A_(x, j) *= rinv; if (cplx) AI_(x, j) *= rinv; }
    for (int jp = j + 1; jp < m; ++jp) {
      double br = A_(jp, j);
      double bi = cplx ? -AI_(jp, j) : 0.0;
      for (int x = jp; x < m; ++x) {
        double ar = -A_(x, j);
        if (cplx) {
          double ai = -AI_(x, j);
          A_(x, jp) = fma(ar, br, fma(-ai, bi, A_(x, jp)));
          AI_(x, jp) = fma(ar, bi, fma(ai, br, AI_(x, jp)));
        } else {
          A_(x, jp) = fma(ar, br, A_(x, jp));
        }
      }
    }
  }
  for (int r = 0; r < m; ++r)
    for (int s = 0; s < r; ++s) {
      A_(s, r) = A_(r, s); AI_(s, r) = -AI_(r, s); A_(r, s) = 0.0; AI_(r, s) = 0.0;
    }
  return 0;
#undef A_
#undef AI_
}

/* blocked.py:97-217; A: m x nc (ld m) */
static int qr_rfactor(double* Ar, double* Ai, int64_t m, int nc, int cplx, int pivot, int64_t* jpvt,
                      double tol_scale) {
#define A_(x, y) Ar[(x) + (int64_t)(y) * m]
#define AI_(x, y) Ai[(x) + (int64_t)(y) * m]
  double* innorm = (double*)malloc(sizeof(double) * nc);
  for (int c = 0; c < nc; ++c) {
    double s = 0.0;
    for (int64_t x = 0; x < m; ++x) {
      s = fma(A_(x, c), A_(x, c), s);
      if (cplx) s = fma(AI_(x, c), AI_(x, c), s);
    }
    innorm[c] = sqrt(s);
  }
  for (int k = 0; k < nc; ++k) {
    if (pivot) {
      int best = k; double bestn = -1.0;
      for (int c = k; c < nc; ++c) {
        double s = 0.0;
        for (int64_t x = k; x < m; ++x) {
          s = fma(A_(x, c), A_(x, c), s);
          if (cplx) s = fma(AI_(x, c), AI_(x, c), s);
        }
        if (s > bestn) { bestn = s; best = c; }
      }
      if (best != k) {
        for (int64_t x = 0; x < m; ++x) {
          double t = A_(x, k); A_(x, k) = A_(x, best); A_(x, best) = t;
          t = AI_(x, k); AI_(x, k) = AI_(x, best); AI_(x, best) = t;
        }
        int64_t t2 = jpvt[k]; jpvt[k] = jpvt[best]; jpvt[best] = t2;
        double t = innorm[k]; innorm[k] = innorm[best]; innorm[best] = t;
      }
    }
    double s = 0.0;
    for (int64_t x = k; x < m; ++x) {
      s = fma(A_(x, k), A_(x, k), s);
      if (cplx) s = fma(AI_(x, k), AI_(x, k), s);
    }
    double normx = sqrt(s);
    if (normx == 0.0) { free(innorm); return 1; }
    double akr = A_(k, k);
    double aki = cplx ? AI_(k, k) : 0.0;
    double aa = hypot(akr, aki);
    double phr, phi;
    if (aa == 0.0) { phr = 1.0; phi = 0.0; } else { phr = akr / aa; phi = aki / aa; }
    double alr = -(phr * normx);
    double ali = -(phi * normx);
    A_(k, k) -= alr;
    if (cplx) AI_(k, k) -= ali;
    double vn = 0.0;
    for (int64_t x = k; x < m; ++x) {
      vn = fma(A_(x, k), A_(x, k), vn);
      if (cplx) vn = fma(AI_(x, k), AI_(x, k), vn);
    }
    double beta = 2.0 / vn;
    for (int c = k + 1; c < nc; ++c) {
      double wr = 0.0, wi = 0.0;
      for (int64_t x = k; x < m; ++x) {
        wr = fma(A_(x, k), A_(x, c), wr);
        if (cplx) {
          wr = fma(AI_(x, k), AI_(x, c), wr);
          wi = fma(A_(x, k), AI_(x, c), fma(-AI_(x, k), A_(x, c), wi));
        }
      }
      wr *= beta; wi *= beta;
      for (int64_t x = k; x < m; ++x) {
        A_(x, c) = fma(-A_(x, k), wr, A_(x, c));
        if (cplx) {
          A_(x, c) = fma(AI_(x, k), wi, A_(x, c));
          AI_(x, c) = fma(-A_(x, k), wi, fma(-AI_(x, k), wr, AI_(x, c)));
        }
      }
    }
    A_(k, k) = alr;
    if (cplx) AI_(k, k) = ali;
    for (int64_t x = k + 1; x < m; ++x) { A_(x, k) = 0.0; if (cplx) AI_(x, k) = 0.0; }
  }
  int bad = 0;
  for (int k = 0; k < nc; ++k)
    if (!(hypot(A_(k, k), AI_(k, k)) >= tol_scale * innorm[k])) bad = 1;
  for (int k = 0; k < nc; ++k) {
    double dkr = A_(k, k);
    double dki = cplx ? AI_(k, k) : 0.0;
    if (cplx) {
      double mag = hypot(dkr, dki);
      if (mag == 0.0) continue;
      double phr = dkr / mag, phi = -(dki / mag);
      for (int c = k; c < nc; ++c) {
        double re = fma(A_(k, c), phr, -(AI_(k, c) * phi));
        double im = fma(A_(k, c), phi, AI_(k, c) * phr);
        A_(k, c) = re; AI_(k, c) = im;
      }
      AI_(k, k) = 0.0;
    } else if (dkr < 0.0) {
      for (int c = k; c < nc; ++c) A_(k, c) = -A_(k, c);
    }
  }
  free(innorm);
  return bad;
#undef A_
#undef AI_
}

/* exported: the QR shortening of blocked.py:487-500 on an m x tw stack (in place), R -> outR/outI (tw x tw) */
/* _k_qr_rfactor itself (blocked.py:97-217), in place, with the caller's
 * pivot flag and jpvt: the building block of preprocess_tall (:405-428) */
int hzo_qr_rfactor(int64_t m, int nc, int cplx, int pivot, double tol_scale, double* Ar, double* Ai, int64_t* jpvt) {
  return qr_rfactor(Ar, Ai, m, nc, cplx, pivot, jpvt, tol_scale);
}

int hzo_qr_shorten(int64_t m, int tw, int cplx, double* Sr, double* Si, double* outR, double* outI) {
  int64_t* jpvt = (int64_t*)malloc(sizeof(int64_t) * tw);
  for (int k = 0; k < tw; ++k) jpvt[k] = k;
  int st = qr_rfactor(Sr, Si, m, tw, cplx, 0, jpvt, tw * EPS);
  free(jpvt);
  if (st) return HZO_RANK;
  for (int c = 0; c < tw; ++c)
    for (int r = 0; r < tw; ++r) { outR[r + c * tw] = Sr[r + c * m]; outI[r + c * tw] = Si[r + c * m]; }
  return HZO_OK;
}

/* blocked.py:220-250 */
static void postmult(plane_t Y, int64_t c0, int64_t c1, int w, const double* Br, const double* Bi, int cplx,
                     double* scratch /* 4*tw */) {
  int tw = 2 * w;
  double *rowr = scratch, *rowi = scratch + tw, *outr = scratch + 2 * tw, *outi = scratch + 3 * tw;
  for (int64_t r = 0; r < Y.rows; ++r) {
    for (int s = 0; s < tw; ++s) {
      int64_t c = s < w ? c0 + s : c1 + (s - w);
      rowr[s] = COL(Y, c)[r];
      rowi[s] = cplx ? COLI(Y, c)[r] : 0.0;
    }
    for (int c = 0; c < tw; ++c) {
      double ar = 0.0, ai = 0.0;
      for (int k = 0; k < tw; ++k) {
        if (cplx) {
          ar = fma(rowr[k], Br[k + c * tw], fma(-rowi[k], Bi[k + c * tw], ar));
          ai = fma(rowr[k], Bi[k + c * tw], fma(rowi[k], Br[k + c * tw], ai));
        } else {
          ar = fma(rowr[k], Br[k + c * tw], ar);
        }
      }
      outr[c] = ar; outi[c] = ai;
    }
    for (int s = 0; s < tw; ++s) {
      int64_t c = s < w ? c0 + s : c1 + (s - w);
      COL(Y, c)[r] = outr[s];
      if (cplx) COLI(Y, c)[r] = outi[s];
    }
  }
}

/* blocked.py:253-295 */
static int rescale_full(plane_t F, plane_t G, plane_t Z, int cplx, int comp, int final, double* sigF, double* sigG,
                        double* sig, double* buf) {
  for (int64_t j = 0; j < F.cols; ++j) {
    double nf2 = col_norm(F, j, cplx, comp, buf);
    double ng2 = col_norm(G, j, cplx, comp, buf);
    double sf = 0.0, sg = 0.0;
    if (final) {
      if (!(nf2 > 0.0 && ng2 > 0.0)) return 1;
      sf = sqrt(nf2);
      if (nf2 != 1.0) {
        double r = 1.0 / sf;
        for (int64_t x = 0; x < F.rows; ++x) { COL(F, j)[x] *= r; if (cplx) COLI(F, j)[x] *= r; }
      }
      sg = sqrt(ng2);
      if (ng2 != 1.0) {
        double r = 1.0 / sg;
        for (int64_t x = 0; x < G.rows; ++x) { COL(G, j)[x] *= r; if (cplx) COLI(G, j)[x] *= r; }
      }
    }
    double s = nf2 + ng2;
    if (!(s > 0.0)) return 1;
    double th = 1.0 / sqrt(s);
    if (th != 1.0)
      for (int64_t x = 0; x < Z.rows; ++x) { COL(Z, j)[x] *= th; if (cplx) COLI(Z, j)[x] *= th; }
    if (final) {
      sigF[j] = sf * th;
      sigG[j] = sg * th;
      sig[j] = sigF[j] / sigG[j];
    }
  }
  return 0;
}

/* blocked.py:298-308 */
static int is_identity(const double* Br, const double* Bi, int m, int cplx) {
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < m; ++c) {
      double want = r == c ? 1.0 : 0.0;
      if (Br[r + c * m] != want) return 0;
      if (cplx && Bi[r + c * m] != 0.0) return 0;
    }
  return 1;
}

/* ------------------------------------------------------------------------ */
/* the block task and the outer loop                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  double *Fhr, *Fhi, *Ghr, *Ghi, *Zhr, *Zhi, *z0, *buf, *pm, *Sr, *Si;
  int64_t bufn, sn;
} scratch_t;

static void scratch_init(scratch_t* s, int tw, int64_t mmax) {
  int64_t t2 = (int64_t)tw * tw;
  s->Fhr = (double*)calloc(t2, 8); s->Fhi = (double*)calloc(t2, 8);
  s->Ghr = (double*)calloc(t2, 8); s->Ghi = (double*)calloc(t2, 8);
  s->Zhr = (double*)calloc(t2, 8); s->Zhi = (double*)calloc(t2, 8);
  s->z0 = (double*)malloc(8 * tw);
  s->bufn = pow2(mmax > tw ? mmax : tw);
  s->buf = (double*)malloc(8 * s->bufn);
  s->pm = (double*)malloc(8 * 4 * tw);
  s->sn = mmax * tw;
  s->Sr = NULL; s->Si = NULL;
}

static void scratch_free(scratch_t* s) {
  free(s->Fhr); free(s->Fhi); free(s->Ghr); free(s->Ghi); free(s->Zhr); free(s->Zhi);
  free(s->z0); free(s->buf); free(s->pm); free(s->Sr); free(s->Si);
}

/* blocked.py:487-500 */
static int shorten_qr(plane_t Y, int64_t c0, int64_t c1, int w, int cplx, double* outR, double* outI, scratch_t* s) {
  int tw = 2 * w;
  int64_t m = Y.rows;
  if (!s->Sr) { s->Sr = (double*)malloc(8 * s->sn); s->Si = (double*)malloc(8 * s->sn); }
  for (int k = 0; k < tw; ++k) {
    int64_t c = k < w ? c0 + k : c1 + (k - w);
    memcpy(s->Sr + k * m, COL(Y, c), 8 * m);
    memcpy(s->Si + k * m, COLI(Y, c), 8 * m);
  }
  return hzo_qr_shorten(m, tw, cplx, s->Sr, s->Si, outR, outI);
}

/* the inner half of blocked.py:463-479 on given factors (prescale, pointwise, theta rescale) */
static int block_inner(int tw, int cplx, const hzo_cfg* cfg, const int32_t* inner, int isteps, double epsn,
                       scratch_t* s, int64_t* total, int64_t* big) {
  int64_t t2 = (int64_t)tw * tw;
  plane_t Fh = {s->Fhr, s->Fhi, tw, tw, tw}, Gh = {s->Ghr, s->Ghi, tw, tw, tw}, Zh = {s->Zhr, s->Zhi, tw, tw, tw};
  memset(s->Zhr, 0, 8 * t2); memset(s->Zhi, 0, 8 * t2);
  for (int k = 0; k < tw; ++k) s->z0[k] = 1.0;
  if (cfg->prescale)
    if (prescale(Fh, Gh, s->z0, cplx, cfg->compensated, s->buf)) return HZO_RANK;
  for (int k = 0; k < tw; ++k) s->Zhr[k + k * tw] = s->z0[k];
  int64_t sw, tot, bg; int conv;
  int bad = pointwise(Fh, Gh, Zh, cplx, inner, isteps, tw / 2, !cfg->prescale, cfg->compensated, cfg->crit_c2,
                      cfg->sorting, cfg->max_inner_sweeps, epsn, s->buf, &sw, &tot, &bg, &conv);
  if (bad) return HZO_RANK;
  if (theta_rescale(Fh, Gh, Zh, cplx, cfg->compensated, s->buf)) return HZO_RANK;
  *total = tot; *big = bg;
  return HZO_OK;
}

/* blocked.py:435-484 */
static int block_task(plane_t F, plane_t G, plane_t Z, int cplx, int pblk, int qblk, const hzo_cfg* cfg,
                      const int32_t* inner, int isteps, double epsn, scratch_t* s, int64_t* total, int64_t* big) {
  int w = cfg->block_width, tw = 2 * w;
  int64_t c0 = (int64_t)pblk * w, c1 = (int64_t)qblk * w;
  int64_t t2 = (int64_t)tw * tw;
  memset(s->Fhr, 0, 8 * t2); memset(s->Fhi, 0, 8 * t2); memset(s->Ghr, 0, 8 * t2); memset(s->Ghi, 0, 8 * t2);
  int st;
  if (cfg->shorten_qr) {
    if ((st = shorten_qr(F, c0, c1, w, cplx, s->Fhr, s->Fhi, s))) return st;
    if ((st = shorten_qr(G, c0, c1, w, cplx, s->Ghr, s->Ghi, s))) return st;
  } else {
    grammian(F, c0, c1, w, cplx, cfg->compensated, s->Fhr, s->Fhi, s->buf);
    if (hzo_cholesky_upper(tw, cplx, s->Fhr, s->Fhi)) {
      if (!cfg->fallback_qr) return HZO_NOT_PD;
      if ((st = shorten_qr(F, c0, c1, w, cplx, s->Fhr, s->Fhi, s))) return st;
    }
    grammian(G, c0, c1, w, cplx, cfg->compensated, s->Ghr, s->Ghi, s->buf);
    if (hzo_cholesky_upper(tw, cplx, s->Ghr, s->Ghi)) {
      if (!cfg->fallback_qr) return HZO_NOT_PD;
      if ((st = shorten_qr(G, c0, c1, w, cplx, s->Ghr, s->Ghi, s))) return st;
    }
  }
  if ((st = block_inner(tw, cplx, cfg, inner, isteps, epsn, s, total, big))) return st;
  if (!is_identity(s->Zhr, s->Zhi, tw, cplx)) {
    postmult(F, c0, c1, w, s->Zhr, s->Zhi, cplx, s->pm);
    postmult(G, c0, c1, w, s->Zhr, s->Zhi, cplx, s->pm);
    postmult(Z, c0, c1, w, s->Zhr, s->Zhi, cplx, s->pm);
  }
  return HZO_OK;
}

/* blocked.py:503-550 (the pool of :519-530 becomes an OpenMP team; results
 * are pool-size invariant because tasks of one step own disjoint columns).
 * step_limit >= 0 stops after that many outer steps (bounded CPU samples). */
static int algorithm1_loop(plane_t F, plane_t G, plane_t Z, int cplx, const hzo_cfg* cfg, int sweep_cap, double epsn,
                           int trailing_rescale, int nthreads, int64_t step_limit, hzo_stats* stats) {
  int n = (int)F.cols, w = cfg->block_width, nblk = n / w, tw = 2 * w;
  int osteps_max = nblk, isteps_max = tw;
  int32_t* outer = (int32_t*)malloc(sizeof(int32_t) * (int64_t)osteps_max * nblk);
  int32_t* inner = (int32_t*)malloc(sizeof(int32_t) * (int64_t)isteps_max * tw);
  int osteps = hzo_gen_table(cfg->outer_mm, nblk, outer);
  int isteps = hzo_gen_table(cfg->inner_mm, tw, inner);
  int half = nblk / 2;
  int64_t mmax = F.rows > G.rows ? F.rows : G.rows;
  if (Z.rows > mmax) mmax = Z.rows;
  if (nthreads < 1) nthreads = 1;
  scratch_t* scr = (scratch_t*)malloc(sizeof(scratch_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) scratch_init(&scr[t], tw, mmax);
  int* stv = (int*)malloc(sizeof(int) * half);
  int64_t* tv = (int64_t*)malloc(sizeof(int64_t) * half);
  int64_t* bv = (int64_t*)malloc(sizeof(int64_t) * half);
  double* buf = (double*)malloc(8 * pow2(mmax));
  int64_t total = 0, big = 0, sweeps = 0, steps_done = 0;
  int converged = 0, status = HZO_OK;
  stats->fail_pair = -1;
  stats->step_seconds = 0.0;
  for (int c = 0; c < sweep_cap && status == HZO_OK; ++c) {
    int64_t s_sw = 0, b_sw = 0;
    for (int step = 0; step < osteps; ++step) {
      if (step_limit >= 0 && steps_done >= step_limit) goto done;
      const int32_t* row = outer + (int64_t)step * half * 2;
      struct timespec ts0, ts1;
      clock_gettime(CLOCK_MONOTONIC, &ts0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
      for (int pr = 0; pr < half; ++pr) {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        tv[pr] = 0; bv[pr] = 0;
        stv[pr] = block_task(F, G, Z, cplx, row[2 * pr], row[2 * pr + 1], cfg, inner, isteps, epsn, &scr[tid],
                             &tv[pr], &bv[pr]);
      }
      clock_gettime(CLOCK_MONOTONIC, &ts1);
      stats->step_seconds += (double)(ts1.tv_sec - ts0.tv_sec) + 1e-9 * (double)(ts1.tv_nsec - ts0.tv_nsec);
      ++steps_done;
      for (int pr = 0; pr < half; ++pr) {
        if (stv[pr] != HZO_OK) { status = stv[pr]; stats->fail_pair = pr; break; }
        s_sw += tv[pr]; b_sw += bv[pr];
      }
      if (status != HZO_OK) break;
    }
    if (status != HZO_OK) break;
    sweeps += 1; total += s_sw; big += b_sw;
    if (b_sw == 0) { converged = 1; break; }
    if (rescale_full(F, G, Z, cplx, cfg->compensated, 0, NULL, NULL, NULL, buf)) { status = HZO_RANK; break; }
  }
  if (status == HZO_OK && trailing_rescale)
    if (rescale_full(F, G, Z, cplx, cfg->compensated, 0, NULL, NULL, NULL, buf)) status = HZO_RANK;
done:
  stats->sweeps = sweeps; stats->total = total; stats->big = big; stats->converged = converged;
  for (int t = 0; t < nthreads; ++t) scratch_free(&scr[t]);
  free(scr); free(stv); free(tv); free(bv); free(buf); free(outer); free(inner);
  return status;
}

/* blocked.py:553-586 on bordered planes (n a multiple of 2w).  Mutates F, G
 * into U, V; Z (n x n, ld n) is written.  epsn <= 0 selects gate_eps*sqrt(n). */
int hzo_gsvd_blocked(int64_t mF, int64_t mG, int64_t n, int cplx, double* Fr, double* Fi, double* Gr, double* Gi,
                     double* Zr, double* Zi, const hzo_cfg* cfg, double epsn, double* sigF, double* sigG,
                     double* sig, hzo_stats* stats, int nthreads, int64_t step_limit) {
  int w = cfg->block_width;
  if (w < 1 || n % (2 * w) != 0) return HZO_INVALID;
  plane_t F = {Fr, Fi, mF, n, mF}, G = {Gr, Gi, mG, n, mG}, Z = {Zr, Zi, n, n, n};
  memset(Zr, 0, 8 * n * n); memset(Zi, 0, 8 * n * n);
  double* z0 = (double*)malloc(8 * n);
  for (int64_t j = 0; j < n; ++j) z0[j] = 1.0;
  int64_t mmax = mF > mG ? mF : mG;
  double* buf = (double*)malloc(8 * pow2(mmax > n ? mmax : n));
  int st = HZO_OK;
  stats->sweeps = stats->total = stats->big = 0; stats->converged = 0; stats->fail_pair = -1;
  if (cfg->prescale && prescale(F, G, z0, cplx, cfg->compensated, buf)) st = HZO_RANK;
  if (st == HZO_OK) {
    for (int64_t j = 0; j < n; ++j) Zr[j + j * n] = z0[j];
    if (!(epsn > 0.0)) epsn = cfg->gate_eps * sqrt((double)n);
    st = algorithm1_loop(F, G, Z, cplx, cfg, cfg->max_outer_sweeps, epsn, 0, nthreads, step_limit, stats);
  }
  if (st == HZO_OK && step_limit < 0)
    if (rescale_full(F, G, Z, cplx, cfg->compensated, 1, sigF, sigG, sig, buf)) st = HZO_RANK;
  free(z0); free(buf);
  return st;
}

/* the per-block inner solve on given tw x tw factors (exported for the
 * kernel-level parity tests of the GPU inner kernel).  Fh, Gh are replaced
 * by the transformed factors, Zh receives the theta-rescaled transform. */
int hzo_block_inner(int tw, int cplx, const hzo_cfg* cfg, double epsn, double* Fhr, double* Fhi, double* Ghr,
                    double* Ghi, double* Zhr, double* Zhi, int64_t* total, int64_t* big) {
  int32_t* inner = (int32_t*)malloc(sizeof(int32_t) * tw * tw);
  int isteps = hzo_gen_table(cfg->inner_mm, tw, inner);
  scratch_t s;
  scratch_init(&s, tw, tw);
  int64_t t2 = (int64_t)tw * tw;
  memcpy(s.Fhr, Fhr, 8 * t2); memcpy(s.Fhi, Fhi, 8 * t2); memcpy(s.Ghr, Ghr, 8 * t2); memcpy(s.Ghi, Ghi, 8 * t2);
  int st = block_inner(tw, cplx, cfg, inner, isteps, epsn, &s, total, big);
  memcpy(Fhr, s.Fhr, 8 * t2); memcpy(Fhi, s.Fhi, 8 * t2); memcpy(Ghr, s.Ghr, 8 * t2); memcpy(Ghi, s.Ghi, 8 * t2);
  memcpy(Zhr, s.Zhr, 8 * t2); memcpy(Zhi, s.Zhi, 8 * t2);
  scratch_free(&s);
  free(inner);
  return st;
}

/* the Grammian of one block-column pair (blocked.py:40-56), exported for tests */
void hzo_grammian(int64_t m, int64_t ld, int w, int cplx, int comp, const double* Yr, const double* Yi, int64_t c0,
                  int64_t c1, double* Ar, double* Ai) {
  plane_t Y = {(double*)Yr, (double*)Yi, m, 0, ld};
  double* buf = (double*)malloc(8 * pow2(m));
  grammian(Y, c0, c1, w, cplx, comp, Ar, Ai, buf);
  free(buf);
}

int hzo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Timed CPU sample for bench.py (not a reference function): prescale the
 * bordered planes, then run the outer steps listed in `steps` (indices into
 * the outer table, in that order) of sweep 1 with the reference's
 * per-step task pool (blocked.py:519-530), timing only the steps.  Spread
 * indices sample the whole sweep's pair sets instead of step 0 repeatedly.
 * Returns the status; *seconds = wall time of the steps. */
int hzo_sample_steps(int64_t mF, int64_t mG, int64_t n, int cplx, double* Fr, double* Fi, double* Gr, double* Gi,
                     double* Zr, double* Zi, const hzo_cfg* cfg, int nthreads, const int32_t* steps, int nsteps,
                     double* seconds) {
  int w = cfg->block_width;
  if (w < 1 || n % (2 * w) != 0) return HZO_INVALID;
  plane_t F = {Fr, Fi, mF, n, mF}, G = {Gr, Gi, mG, n, mG}, Z = {Zr, Zi, n, n, n};
  memset(Zr, 0, 8 * n * n); memset(Zi, 0, 8 * n * n);
  int nblk = (int)(n / w), tw = 2 * w, half = nblk / 2;
  int64_t mmax = mF > mG ? mF : mG;
  if (n > mmax) mmax = n;
  double* buf = (double*)malloc(8 * pow2(mmax));
  double* z0 = (double*)malloc(8 * n);
  for (int64_t j = 0; j < n; ++j) z0[j] = 1.0;
  int st = HZO_OK;
  if (cfg->prescale && prescale(F, G, z0, cplx, cfg->compensated, buf)) st = HZO_RANK;
  for (int64_t j = 0; j < n; ++j) Zr[j + j * n] = z0[j];
  double epsn = cfg->gate_eps * sqrt((double)n);
  int32_t* outer = (int32_t*)malloc(sizeof(int32_t) * (int64_t)nblk * nblk);
  int32_t* inner = (int32_t*)malloc(sizeof(int32_t) * (int64_t)tw * tw);
  int osteps = hzo_gen_table(cfg->outer_mm, nblk, outer);
  int isteps = hzo_gen_table(cfg->inner_mm, tw, inner);
  if (nthreads < 1) nthreads = 1;
  scratch_t* scr = (scratch_t*)malloc(sizeof(scratch_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) scratch_init(&scr[t], tw, mmax);
  int* stv = (int*)malloc(sizeof(int) * half);
  int64_t* tv = (int64_t*)malloc(sizeof(int64_t) * half);
  int64_t* bv = (int64_t*)malloc(sizeof(int64_t) * half);
  *seconds = 0.0;
  for (int q = 0; q < nsteps && st == HZO_OK; ++q) {
    int step = steps[q];
    if (step < 0 || step >= osteps) { st = HZO_INVALID; break; }
    const int32_t* row = outer + (int64_t)step * half * 2;
    struct timespec ts0, ts1;
    clock_gettime(CLOCK_MONOTONIC, &ts0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int pr = 0; pr < half; ++pr) {
      int tid = 0;
#ifdef _OPENMP
      tid = omp_get_thread_num();
#endif
      tv[pr] = 0; bv[pr] = 0;
      stv[pr] = block_task(F, G, Z, cplx, row[2 * pr], row[2 * pr + 1], cfg, inner, isteps, epsn, &scr[tid],
                           &tv[pr], &bv[pr]);
    }
    clock_gettime(CLOCK_MONOTONIC, &ts1);
    *seconds += (double)(ts1.tv_sec - ts0.tv_sec) + 1e-9 * (double)(ts1.tv_nsec - ts0.tv_nsec);
    for (int pr = 0; pr < half; ++pr)
      if (stv[pr] != HZO_OK) { st = stv[pr]; break; }
  }
  for (int t = 0; t < nthreads; ++t) scratch_free(&scr[t]);
  free(scr); free(stv); free(tv); free(bv); free(buf); free(z0); free(outer); free(inner);
  return st;
}

/* _k_postmult (blocked.py:220-250) on a stacked m x 2w column pair [Yp Yq]
 * (column-major, ld m) with the 2w x 2w transform B (column-major); exported
 * for the single-operation parity test of postmultiply. */
void hzo_postmult(int64_t m, int w, int cplx, double* Yr, double* Yi, const double* Br, const double* Bi) {
  plane_t Y = {Yr, Yi, m, 2 * w, m};
  double* scratch = (double*)malloc(8 * 4 * 2 * w);
  postmult(Y, 0, w, w, Br, Bi, cplx, scratch);
  free(scratch);
}
