// Host scalars of the QDWH iteration (CUDA-free): polar.cpp:12-27 / 40-51,
// partial.cpp:26-30.  Same libm calls in the same order as the reference, so
// the weights are bit-identical to qdwh::halley_weights.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace qdwhg {

struct WeightStep {
  double a, b, c, ell_in, ell_out;
};
WeightStep halley_weights(double ell);
size_t iterations_to_converge(double ell0, double eps, size_t max_iters = 60);
double choose_shift(size_t iters);  // returns s
// kernels.cpp:16-32: draws 0..count-1 of the counter-based N(0,1) generator with
// glibc log/cos (bit-identical to the reference's gaussian_matrix(count, 1, seed))
std::vector<double> host_gaussian(int64_t count, uint64_t seed);

}  // namespace qdwhg
