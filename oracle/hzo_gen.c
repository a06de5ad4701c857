/*
 * hzo_gen.c -- deterministic input generators for the north-star parity
 * fixtures (TEST INFRASTRUCTURE, not product code).
 *
 * The fixtures under tests/golden/ns_*.npz hold the oracle's results for the
 * BASELINE.json configurations 2-4 (too large to store their inputs).  The
 * GPU box must therefore regenerate the SAME input bytes that the oracle saw
 * in the build container.  numpy's SIMD log/cos paths depend on the host's
 * AVX-512 level, so the streams are restated here in plain C: only IEEE
 * +,-,*,/,sqrt (correctly rounded everywhere), glibc's log/cos/pow, and
 * explicitly ordered loops compiled with -ffp-contract=off.  Every fixture
 * also records the SHA-256 of its generated inputs so a mismatch is caught
 * before any comparison.
 *
 *   hzo_uniform_fill   harness.py:43-63  (splitmix64 uniforms on (0, 1))
 *   hzo_gaussian_fill  harness.py:66-71  (Box-Muller: sqrt(-2 log u0) cos(2 pi u1))
 *   hzo_gen_cond       SURVEY.md 8(d) config 4: F = U diag(sF) X, G = V diag(sG) X,
 *                      sigma = logspace(-8, 8, n) shuffled, sF = s/sqrt(1+s^2),
 *                      sG = 1/sqrt(1+s^2); U, V, W orthogonal (Householder QR of
 *                      Gaussian matrices); X = W diag(lambda), lambda ~ U[0.01, 1].
 *
 * Parallel loops run over independent columns; the arithmetic of one column
 * is sequential, so the result does not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm64_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double sm64_unit(uint64_t z) { return ((double)(z >> 11) + 0.5) * 0x1p-53; }

void hzo_uniform_fill(uint64_t seed, int64_t count, double* out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < count; ++i) out[i] = sm64_unit(sm64_next(&s));
}

/* harness.py:66-71: u = uniform_stream(seed, 2 count); r = sqrt(-2 log u[0::2]);
 * a = 2 pi u[1::2]; out = r cos(a).  Two roundings in 2*pi*u as numpy does
 * ((2.0 * math.pi) is a constant folded first, then one product). */
void hzo_gaussian_fill(uint64_t seed, int64_t count, double* out) {
  uint64_t s = seed;
  const double twopi = 2.0 * 3.141592653589793;
  for (int64_t i = 0; i < count; ++i) {
    double u0 = sm64_unit(sm64_next(&s));
    double u1 = sm64_unit(sm64_next(&s));
    double r = sqrt(-2.0 * log(u0));
    out[i] = r * cos(twopi * u1);
  }
}

/* dot with a fixed 4-way interleaved order (deterministic, vectorisable) */
static double dot4(const double* a, const double* b, int64_t n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += a[i] * b[i];
    s1 += a[i + 1] * b[i + 1];
    s2 += a[i + 2] * b[i + 2];
    s3 += a[i + 3] * b[i + 3];
  }
  for (; i < n; ++i) s0 += a[i] * b[i];
  return (s0 + s1) + (s2 + s3);
}

/* Householder QR of the n x n column-major A in place: v_k (v_k[0] = 1
 * implied) below the diagonal, tau[k]. */
static void householder_qr(int64_t n, double* A, double* tau) {
  for (int64_t k = 0; k < n; ++k) {
    double* x = A + k * n + k;
    int64_t len = n - k;
    double nrm = sqrt(dot4(x, x, len));
    double x0 = x[0];
    if (nrm == 0.0) { tau[k] = 0.0; continue; }
    double beta = x0 >= 0.0 ? -nrm : nrm;
    double d = x0 - beta;
    for (int64_t i = 1; i < len; ++i) x[i] = x[i] / d;
    tau[k] = (beta - x0) / beta;
    x[0] = beta;
    double tk = tau[k];
#pragma omp parallel for schedule(static)
    for (int64_t j = k + 1; j < n; ++j) {
      double* a = A + j * n + k;
      double s = a[0] + dot4(x + 1, a + 1, len - 1);
      double ts = tk * s;
      a[0] -= ts;
      for (int64_t i = 1; i < len; ++i) a[i] -= ts * x[i];
    }
  }
}

/* M <- Q M with Q = H_0 H_1 ... H_{n-1} from householder_qr's (V, tau). */
static void apply_q(int64_t n, const double* V, const double* tau, double* M) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    double* m = M + j * n;
    for (int64_t k = n - 1; k >= 0; --k) {
      const double* v = V + k * n + k;
      int64_t len = n - k;
      double s = m[k] + dot4(v + 1, m + k + 1, len - 1);
      double ts = tau[k] * s;
      m[k] -= ts;
      for (int64_t i = 1; i < len; ++i) m[k + i] -= ts * v[i];
    }
  }
}

/* Config 4 pair (n x n each, column-major) with known generalized singular
 * values sigma_true (unsorted, in generator order).  Seeds: U from seed+1,
 * V from seed+2, W from seed+3, lambda from seed+4, the shuffle from seed+5. */
int hzo_gen_cond(int64_t n, uint64_t seed, double* F, double* G, double* sigma_true) {
  double* A = (double*)malloc(sizeof(double) * n * n);
  double* tau = (double*)malloc(sizeof(double) * n);
  double* X = (double*)malloc(sizeof(double) * n * n);
  double* u = (double*)malloc(sizeof(double) * (n > 2 ? n : 2));
  if (!A || !tau || !X || !u) { free(A); free(tau); free(X); free(u); return 1; }

  /* sigma = 10^(-8 + 16 i / (n-1)), then a Fisher-Yates shuffle */
  for (int64_t i = 0; i < n; ++i) sigma_true[i] = pow(10.0, -8.0 + 16.0 * (double)i / (double)(n - 1));
  hzo_uniform_fill(seed + 5, n, u);
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)(u[i] * (double)(i + 1));
    if (j > i) j = i;
    double t = sigma_true[i]; sigma_true[i] = sigma_true[j]; sigma_true[j] = t;
  }

  /* X = W diag(lambda) */
  hzo_gaussian_fill(seed + 3, n * n, A);
  householder_qr(n, A, tau);
  hzo_uniform_fill(seed + 4, n, u);
  memset(X, 0, sizeof(double) * n * n);
  for (int64_t j = 0; j < n; ++j) X[j * n + j] = 0.01 + 0.99 * u[j];
  apply_q(n, A, tau, X);

  /* F = U diag(sF) X, G = V diag(sG) X */
  for (int pass = 0; pass < 2; ++pass) {
    double* Y = pass == 0 ? F : G;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        double s = sigma_true[i];
        double c = 1.0 / sqrt(1.0 + s * s);
        Y[j * n + i] = (pass == 0 ? s * c : c) * X[j * n + i];
      }
    hzo_gaussian_fill(seed + 1 + pass, n * n, A);
    householder_qr(n, A, tau);
    apply_q(n, A, tau, Y);
  }
  free(A); free(tau); free(X); free(u);
  return 0;
}
