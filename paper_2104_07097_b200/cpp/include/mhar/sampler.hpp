#pragma once
// Drop-in C++ host API for the reference sampler
// (/root/reference/proj/include/mhar/{linalg,errors,polytope,projection,
// rng,sampler}.hpp): same names, fields, defaults and error behaviour, with
// an in-repo column-major Matrix in place of Eigen::MatrixXd.  Every
// computation is delegated to the B200 engine through the C ABI
// (include/mhar_b200.h); nothing here computes a chord or a step on the CPU.

#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mhar {

using Index = std::int64_t;

// ---------------------------------------------------------------- linalg --
/// Dense column-major matrix (the layout of Eigen::MatrixXd, linalg.hpp:7).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols, double fill = 0.0)
      : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols), fill) {}
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols, 0.0); }
  static Matrix Constant(Index rows, Index cols, double v) { return Matrix(rows, cols, v); }
  static Matrix Identity(Index n) {
    Matrix m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double* col(Index k) { return v_.data() + k * r_; }
  const double* col(Index k) const { return v_.data() + k * r_; }
  void resize(Index rows, Index cols) {
    r_ = rows;
    c_ = cols;
    v_.assign(static_cast<size_t>(rows * cols), 0.0);
  }
  bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

/// Column vector.
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n, double fill = 0.0) : v_(static_cast<size_t>(n), fill) {}
  Vector(std::initializer_list<double> l) : v_(l) {}
  static Vector Zero(Index n) { return Vector(n, 0.0); }
  static Vector Constant(Index n, double v) { return Vector(n, v); }
  static Vector Ones(Index n) { return Vector(n, 1.0); }
  Index size() const { return static_cast<Index>(v_.size()); }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void resize(Index n) { v_.assign(static_cast<size_t>(n), 0.0); }
  /// x replicated into z columns (Eigen's replicate(1, z)).
  Matrix replicate(Index z) const {
    Matrix m(size(), z);
    for (Index k = 0; k < z; ++k)
      for (Index i = 0; i < size(); ++i) m(i, k) = v_[static_cast<size_t>(i)];
    return m;
  }

 private:
  std::vector<double> v_;
};

// ---------------------------------------------------------------- errors --
/// errors.hpp:10-24 (same order, so status = 1 + ordinal).
enum class ErrorCode {
  invalid_argument,
  dimension_mismatch,
  singular_matrix,
  rank_deficient_eq,
  empty_polytope,
  no_interior,
  unbounded_polytope,
  direction_degenerate,
  retry_exhausted,
  cycle_suspected,
  degenerate_test,
  numerical_failure,
  io_failure,
};

const char* error_code_name(ErrorCode code);

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message);
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] void raise(ErrorCode code, const std::string& message);

// -------------------------------------------------------------- polytope --
/// {x : a_in x <= b_in, a_eq x = b_eq} (polytope.hpp:12-25).
struct Polytope {
  Matrix a_in;
  Vector b_in;
  Matrix a_eq;
  Vector b_eq;

  Polytope() = default;
  Polytope(Matrix a_in_, Vector b_in_);
  Polytope(Matrix a_in_, Vector b_in_, Matrix a_eq_, Vector b_eq_);

  int dim() const { return static_cast<int>(a_in.cols()); }
  int num_inequalities() const { return static_cast<int>(a_in.rows()); }
  int num_equalities() const { return static_cast<int>(a_eq.rows()); }
};

bool contains(const Polytope& p, const double* x, double eps);
Polytope make_hypercube(int n);
Polytope make_simplex(int n);

// ------------------------------------------------------------ projection --
struct ProjectionOperator {
  Matrix p;             // n x n projector
  Matrix gram_inverse;  // (a_eq a_eq')^-1
  Matrix source_eq;
};
inline constexpr double kNearZeroDirection = 1e-12;  // projection.hpp:25
ProjectionOperator compute_projection(const Matrix& a_eq);

// --------------------------------------------------------------- sampler --
/// sampler.hpp:16-25.
struct SamplerConfig {
  int z = 0;
  long long phi = 0;
  long long t_target = 1;
  uint64_t seed = 0;
  double eps_dir = 1e-11;
  double eps_feas = 1e-9;
  long long reproject_every = -1;
  long long burn_in = -1;
};

SamplerConfig resolve(const SamplerConfig& cfg, const Polytope& p);

struct LambdaIntervals {
  Vector lower;
  Vector upper;
  std::vector<uint8_t> degenerate;
};

inline constexpr double kDegenerateWidth = 1e-14;
inline constexpr int kMaxDirectionRetries = 16;

LambdaIntervals compute_lambda_intervals(const Polytope& p, const Matrix& x, const Matrix& d,
                                         double eps_dir);
double chord_point(double u, double lower, double upper);

class Engine;  // device context (polytope resident in HBM + walks)

/// WalkRng (rng.hpp:42-55): z column streams + the theta stream.  Here the
/// streams live on the device next to the walks; they reproduce the
/// reference's SplitMix64 streams bit for bit (MHAR_RNG_REFERENCE).
class WalkRng {
 public:
  WalkRng(uint64_t seed, int z);
  ~WalkRng();
  WalkRng(const WalkRng&) = delete;
  WalkRng& operator=(const WalkRng&) = delete;
  int width() const { return z_; }
  uint64_t seed() const { return seed_; }
  static constexpr uint64_t kThetaStreamId = ~uint64_t{0};

 private:
  friend void step(const Polytope&, const ProjectionOperator*, const SamplerConfig&, WalkRng&,
                   struct WalkState&);
  friend Matrix generate_directions(WalkRng&, int);
  friend Matrix select_points(WalkRng&, const Matrix&, const Matrix&, const LambdaIntervals&);
  Engine& engine_for_streams(int n);  // an engine whose streams these are
  uint64_t seed_;
  int z_;
  std::unique_ptr<Engine> engine_;
  const Polytope* bound_ = nullptr;
};

/// One standard normal direction per walk column, n x z (sampler.hpp:46).
Matrix generate_directions(WalkRng& rng, int n);

/// Moves every walk to x + theta d, theta uniform on its open chord via the
/// theta stream; DIRECTION_DEGENERATE if any walk is flagged (sampler.hpp:66-67).
Matrix select_points(WalkRng& rng, const Matrix& x, const Matrix& d,
                     const LambdaIntervals& intervals);

struct WalkState {
  Matrix x;
  long long t = 0;
  long long j = 0;
  long long redraws = 0;
};

/// step() (sampler.hpp:79-80): one iterate of every walk on the B200.
void step(const Polytope& p, const ProjectionOperator* projector, const SamplerConfig& cfg,
          WalkRng& rng, WalkState& state);

/// sampler.hpp:82-91.
struct SampleSet {
  Matrix samples;  // one collected point per row
  SamplerConfig config;
  Vector start;
  double start_radius = 0.0;
  double seconds = 0.0;
  long long iterate_count = 0;
  long long windows = 0;
  long long redraw_count = 0;
};

using ClockFn = std::function<double()>;

/// chebyshev.hpp:8-25: centre and radius of the largest inscribed ball.
struct ChebyshevCenter {
  Vector x;
  double radius = 0.0;
};
inline constexpr double kMinInteriorRadius = 1e-10;

/// Solved on the B200 (constraint generation over a device-resident simplex
/// tableau); raises EMPTY_POLYTOPE / UNBOUNDED_POLYTOPE / NO_INTERIOR /
/// NUMERICAL_FAILURE like the reference.
ChebyshevCenter chebyshev_center(const Polytope& p);

/// run() with a warm start x0 in place of the Chebyshev centre.  Samples are
/// collected on the device.  One GPU and the reference's own streams, or --
/// with MHAR_DEVICES="0,1,..." in the environment -- the devices overload.
SampleSet run(const Polytope& p, const SamplerConfig& cfg, const Vector& x0,
              const ClockFn& clock = {});

/// run() over several GPUs of this process (the C ABI's mhar_group): walks
/// sharded by global id with Philox draws, so the samples are identical for
/// every device list; windows gathered to devices[0] over NVLink (NCCL).
SampleSet run(const Polytope& p, const SamplerConfig& cfg, const Vector& x0,
              const std::vector<int>& devices, const ClockFn& clock = {});

/// run() (sampler.hpp:93-97): starts every walk at the Chebyshev centre
/// (sampler.cpp:276), computed before the clock starts.
SampleSet run(const Polytope& p, const SamplerConfig& cfg, const ClockFn& clock = {});

}  // namespace mhar
