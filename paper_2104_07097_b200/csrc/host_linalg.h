// host_linalg.h -- one-time host precomputation (projector, inverse).
#pragma once
#include <cstdint>
#include <string>

namespace mhar_host {
// Returns 0 or 1 + mhar::ErrorCode ordinal; *msg explains a failure.
int invert(const double* a, int64_t n, double* inv, std::string* msg);
int compute_projection(const double* a_eq, int64_t me, int64_t n, double* P, double* G,
                       std::string* msg);
}  // namespace mhar_host
