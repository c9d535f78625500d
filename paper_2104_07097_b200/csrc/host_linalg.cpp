// host_linalg.cpp -- the one-time host precomputation the engine needs:
// the equality projector P = I - A_E'(A_E A_E')^-1 A_E and G = (A_E A_E')^-1
// (/root/reference/proj/src/projection.cpp:9-34), with the inverse by LU
// with partial pivoting plus one residual-correction pass
// (src/linalg.cpp:21-52).  Runs once per context, before any device work.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "host_linalg.h"

namespace mhar_host {

namespace {
constexpr double kSingularRelTol = 1e-12;  // linalg.hpp:13

// C (m x n) = A (m x k) * B (k x n), column-major, ascending-k accumulation.
void matmul(const double* A, const double* B, double* C, int64_t m, int64_t k, int64_t n) {
  for (int64_t j = 0; j < n; ++j) {
    double* c = C + j * m;
    for (int64_t i = 0; i < m; ++i) c[i] = 0.0;
    for (int64_t p = 0; p < k; ++p) {
      const double b = B[p + j * k];
      const double* a = A + p * m;
      for (int64_t i = 0; i < m; ++i) c[i] = std::fma(a[i], b, c[i]);
    }
  }
}
}  // namespace

int invert(const double* a, int64_t n, double* inv, std::string* msg) {
  if (n <= 0) {
    *msg = "invert: empty matrix";
    return 1;  // INVALID_ARGUMENT
  }
  double scale = 0.0;
  for (int64_t i = 0; i < n * n; ++i) {
    if (!std::isfinite(a[i])) {
      *msg = "invert: matrix has a non-finite entry";
      return 3;
    }
    scale = std::fmax(scale, std::fabs(a[i]));
  }
  if (scale == 0.0) {
    *msg = "invert: matrix has no finite nonzero entry";
    return 3;  // SINGULAR_MATRIX
  }
  std::vector<double> lu(a, a + n * n);
  std::vector<int64_t> perm(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t c = 0; c < n; ++c) {
    int64_t piv = c;
    for (int64_t r = c + 1; r < n; ++r)
      if (std::fabs(lu[r + c * n]) > std::fabs(lu[piv + c * n])) piv = r;
    if (piv != c) {
      for (int64_t j = 0; j < n; ++j) std::swap(lu[c + j * n], lu[piv + j * n]);
      std::swap(perm[c], perm[piv]);
    }
    const double p = lu[c + c * n];
    if (p == 0.0) continue;
    for (int64_t r = c + 1; r < n; ++r) lu[r + c * n] /= p;
    for (int64_t j = c + 1; j < n; ++j) {
      const double f = lu[c + j * n];
      if (f == 0.0) continue;
      for (int64_t r = c + 1; r < n; ++r) lu[r + j * n] -= lu[r + c * n] * f;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    const double pivot = std::fabs(lu[i + i * n]);
    if (!(pivot > kSingularRelTol * scale)) {
      *msg = "invert: pivot " + std::to_string(i) + " has magnitude " + std::to_string(pivot) +
             ", below " + std::to_string(kSingularRelTol * scale);
      return 3;
    }
  }
  for (int64_t col = 0; col < n; ++col) {
    double* x = inv + col * n;
    for (int64_t i = 0; i < n; ++i) x[i] = (perm[i] == col) ? 1.0 : 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t r = i + 1; r < n; ++r) x[r] -= lu[r + i * n] * x[i];
    for (int64_t i = n - 1; i >= 0; --i) {
      x[i] /= lu[i + i * n];
      for (int64_t r = 0; r < i; ++r) x[r] -= lu[r + i * n] * x[i];
    }
  }
  // X <- X + X (I - A X)
  std::vector<double> res(n * n), corr(n * n);
  matmul(a, inv, res.data(), n, n, n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) res[i + j * n] = (i == j ? 1.0 : 0.0) - res[i + j * n];
  matmul(inv, res.data(), corr.data(), n, n, n);
  for (int64_t i = 0; i < n * n; ++i) inv[i] += corr[i];
  return 0;
}

int compute_projection(const double* a_eq, int64_t me, int64_t n, double* P, double* G,
                       std::string* msg) {
  if (me == 0) {
    *msg = "compute_projection: equality matrix is empty";
    return 1;
  }
  if (me >= n) {
    *msg = "compute_projection: " + std::to_string(me) + " equalities in dimension " +
           std::to_string(n) + " leave no null space";
    return 4;  // RANK_DEFICIENT_EQ
  }
  std::vector<double> aet(n * me);  // n x me
  for (int64_t i = 0; i < me; ++i)
    for (int64_t j = 0; j < n; ++j) aet[j + i * n] = a_eq[i + j * me];
  std::vector<double> gram(me * me);
  matmul(a_eq, aet.data(), gram.data(), me, n, me);
  std::string inner;
  const int st = invert(gram.data(), me, G, &inner);
  if (st == 3) {
    *msg = "compute_projection: equality rows are linearly dependent (" + inner + ")";
    return 4;
  }
  if (st) {
    *msg = inner;
    return st;
  }
  std::vector<double> lift(n * me);  // A_E' G, n x me
  matmul(aet.data(), G, lift.data(), n, me, me);
  matmul(lift.data(), a_eq, P, n, me, n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) P[i + j * n] = (i == j ? 1.0 : 0.0) - P[i + j * n];
  return 0;
}

}  // namespace mhar_host
