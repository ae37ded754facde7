// Host scalars (CUDA-free; shared by the single-GPU and distributed drivers).
#include "scalars.hpp"

#include <cmath>
#include <cstdint>
#include <sstream>
#include <vector>

#include "errors.hpp"

namespace qdwhg {

// ----------------------------------------------------------------- scalars
WeightStep halley_weights(double ell) {  // polar.cpp:12-27 (same libm calls, same order)
  if (!(ell > 0.0) || ell > 1.0) throw InvalidArgument("halley_weights: ell must be in (0, 1]");
  const double l2 = ell * ell;
  const double dd = std::cbrt(4.0 * (1.0 - l2)) * std::pow(ell, -4.0 / 3.0);
  const double sqd = std::sqrt(1.0 + dd);
  const double inner = 8.0 - 4.0 * dd + 8.0 * (2.0 - l2) / (l2 * sqd);
  WeightStep w;
  w.a = sqd + std::sqrt(inner) / 2.0;
  w.b = (w.a - 1.0) * (w.a - 1.0) / 4.0;
  w.c = w.a + w.b - 1.0;
  w.ell_in = ell;
  w.ell_out = ell * (w.a + w.b * l2) / (1.0 + w.c * l2);
  return w;
}

size_t iterations_to_converge(double ell0, double eps, size_t max_iters) {  // polar.cpp:40-51
  double ell = ell0;
  for (size_t k = 0; k < max_iters; ++k) {
    if (std::abs(ell - 1.0) < eps) return k;
    ell = halley_weights(ell).ell_out;
  }
  if (std::abs(ell - 1.0) < eps) return max_iters;
  std::ostringstream msg;
  msg << "ell recurrence from " << ell0 << " not within " << eps << " of 1 after " << max_iters
      << " steps (ell = " << ell << ")";
  throw NotConverged(msg.str());
}

double choose_shift(size_t iters) {  // partial.cpp:26-30
  if (iters == 2) return 0.875;
  if (iters == 3) return 0.2;
  throw InvalidArgument("choose_shift: unsupported plan, tabulated iteration counts are 2 and 3");
}

std::vector<double> host_gaussian(int64_t count, uint64_t seed) {
  // kernels.cpp:16-32 restated (splitmix64 + Box-Muller on counters 2i, 2i+1);
  // glibc log/cos, so bit-identical to the reference's gaussian_matrix.
  std::vector<double> out(count);
  for (int64_t i = 0; i < count; ++i) {
    auto h = [&](uint64_t c) {
      uint64_t z = seed + (c + 1) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    const double u1 = static_cast<double>((h(2 * (uint64_t)i) >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>((h(2 * (uint64_t)i + 1) >> 11) + 1) * 0x1.0p-53;
    out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  return out;
}

}  // namespace qdwhg
