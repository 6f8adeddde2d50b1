// setup_gpu.hpp -- GPU construction of the trees, block partition, key
// directions and direction sets (k_setup.cu); fills the same Plan fields as the
// host planner, bit for bit.
#pragma once
#include <cstdint>

#include "plan.hpp"

namespace fdhelm {
// Throws PlanError.  Requires a current CUDA device.
void gpu_build_structure(Plan& P, const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                         const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3]);
}  // namespace fdhelm
