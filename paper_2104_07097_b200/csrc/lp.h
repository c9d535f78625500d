#pragma once
// Chebyshev-centre LP for the start point (see lp.cu).
#include <cstdint>
#include <string>

namespace mhar_lp {

struct LpStats {
  int rounds = 0;             // constraint-generation rounds (LP solves)
  long pivots = 0;            // simplex pivots over all rounds
  int64_t working_rows = 0;   // inequality rows in the final working set
};

/// Column-major a_in (m x n), a_eq (me x n).  Returns 0 or a status code
/// (1 + ErrorCode ordinal, 100 = CUDA) with *msg set.
int chebyshev_center(const double* a_in, const double* b_in, int64_t m, const double* a_eq,
                     const double* b_eq, int64_t me, int64_t n, int device, double* x_out,
                     double* radius, LpStats* stats, std::string* msg);

}  // namespace mhar_lp
