// Exception types of libqdwhg (mirroring the reference's matrix.hpp:13-22 plus
// runtime errors); CUDA-free so the distributed orchestration compiles without it.
#pragma once
#include <stdexcept>
#include <string>

namespace qdwhg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NotPositiveDefinite : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NotConverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

}  // namespace qdwhg
