/* TEST INFRASTRUCTURE ONLY — the CPU oracle's bit-exact scalar/integer layer.
 *
 * Plain-C restatement (not a copy) of the parts of the reference whose results
 * must match BIT FOR BIT, because they depend on glibc's libm and on u64
 * integer arithmetic rather than on floating-point summation order:
 *   - splitmix64 counter hash, (0,1] mapping and Box-Muller draw
 *       /root/reference/proj/core/src/kernels.cpp:16-32
 *   - gaussian_matrix (column-major, entry i uses counters 2i and 2i+1)
 *       /root/reference/proj/core/src/kernels.cpp:441-447
 *   - halley_weights (stable dd = cbrt(4(1-l^2)) * l^(-4/3) form)
 *       /root/reference/proj/core/src/polar.cpp:12-27
 * The dense linear algebra of the oracle lives in oracle/qdwh_oracle.py (numpy).
 * Pinned against the reference itself in tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

uint64_t qo_hash64(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1u) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double qo_to_unit(uint64_t h) { return (double)((h >> 11) + 1u) * 0x1.0p-53; }

double qo_normal_draw(uint64_t seed, uint64_t index) {
  double u1 = qo_to_unit(qo_hash64(seed, 2u * index));
  double u2 = qo_to_unit(qo_hash64(seed, 2u * index + 1u));
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* out: m*n doubles, column-major; entry (i,j) is draw number j*m+i. */
void qo_gaussian_matrix(int64_t m, int64_t n, uint64_t seed, double* out) {
  int64_t total = m * n;
  for (int64_t i = 0; i < total; ++i) out[i] = qo_normal_draw(seed, (uint64_t)i);
}

/* Same stream, sub-range [first, first+count): lets callers generate huge
 * matrices in parallel chunks while staying identical to qo_gaussian_matrix. */
void qo_gaussian_range(uint64_t seed, int64_t first, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = qo_normal_draw(seed, (uint64_t)(first + i));
}

/* uniform (0,1] draws from the same hash: u_i = to_unit(hash64(seed, i)) */
void qo_uniform_range(uint64_t seed, int64_t first, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = qo_to_unit(qo_hash64(seed, (uint64_t)(first + i)));
}

/* out5 = {a, b, c, ell_in, ell_out}; returns 0, or 1 if ell is outside (0,1]. */
int qo_halley_weights(double ell, double* out5) {
  if (!(ell > 0.0) || ell > 1.0) return 1;
  double l2 = ell * ell;
  double dd = cbrt(4.0 * (1.0 - l2)) * pow(ell, -4.0 / 3.0);
  double sqd = sqrt(1.0 + dd);
  double inner = 8.0 - 4.0 * dd + 8.0 * (2.0 - l2) / (l2 * sqd);
  double a = sqd + sqrt(inner) / 2.0;
  double b = (a - 1.0) * (a - 1.0) / 4.0;
  double c = a + b - 1.0;
  out5[0] = a;
  out5[1] = b;
  out5[2] = c;
  out5[3] = ell;
  out5[4] = ell * (a + b * l2) / (1.0 + c * l2);
  return 0;
}
