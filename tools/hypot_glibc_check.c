/* Checks that the device hz_hypot algorithm (Borges, non-FMA kernel) matches glibc hypot bitwise. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#define SCALE 0x1p-600
#define LARGE_VAL 0x1p+511
#define TINY_VAL 0x1p-511
#define EPSH 0x1p-54
static double kern_nofma(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) { double delta = h - ay; t1 = ax * (2.0 * delta - ax); t2 = (delta - 2.0 * (ax - ay)) * delta; }
  else { double delta = h - ax; t1 = 2.0 * delta * (ax - 2.0 * ay); t2 = (4.0 * delta - ay) * ay + delta * delta; }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
static double kern_fma(double ax, double ay) {
  double t1 = ay + ay, t2 = ax - ay;
  if (t1 >= ax) return sqrt(fma(t1, ax, t2 * t2));
  return sqrt(fma(ax, ax, ay * ay));
}
static double my(double x, double y, int usefma) {
  double (*k)(double,double) = usefma ? kern_fma : kern_nofma;
  if (!isfinite(x) || !isfinite(y)) { if (isinf(x) || isinf(y)) return INFINITY; return x + y; }
  x = fabs(x); y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > LARGE_VAL) { if (ay <= ax * EPSH) return ax + ay; return k(ax * SCALE, ay * SCALE) / SCALE; }
  if (ay < TINY_VAL) { if (ax >= ay / EPSH) return ax + ay; return k(ax / SCALE, ay / SCALE) * SCALE; }
  if (ay <= ax * EPSH) return ax + ay;
  return k(ax, ay);
}
static uint64_t s = 88172645463325252ull;
static double rnd() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (double)(s >> 11) * 0x1p-53; }
int main() {
  long bad0 = 0, bad1 = 0, N = 20000000;
  for (long i = 0; i < N; ++i) {
    double x = (rnd() * 2 - 1) * pow(2.0, (int)(rnd() * 40) - 20), y = (rnd() * 2 - 1) * pow(2.0, (int)(rnd() * 40) - 20);
    if (i % 3 == 0) y = x * (1 + rnd() * 1e-3);
    double h = hypot(x, y);
    if (h != my(x, y, 0)) bad0++;
    if (h != my(x, y, 1)) bad1++;
  }
  printf("mismatch nofma %ld fma %ld of %ld\n", bad0, bad1, N);
}
