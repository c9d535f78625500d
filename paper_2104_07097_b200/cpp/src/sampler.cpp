// Host shim: the reference's C++ sampler API over the engine's C ABI.
#include "mhar/sampler.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/mhar_b200.h"

namespace mhar {

// ----------------------------------------------------------------- errors --
const char* error_code_name(ErrorCode code) {
  static const char* names[] = {"INVALID_ARGUMENT",  "DIMENSION_MISMATCH", "SINGULAR_MATRIX",
                                "RANK_DEFICIENT_EQ", "EMPTY_POLYTOPE",     "NO_INTERIOR",
                                "UNBOUNDED_POLYTOPE", "DIRECTION_DEGENERATE", "RETRY_EXHAUSTED",
                                "CYCLE_SUSPECTED",   "DEGENERATE_TEST",    "NUMERICAL_FAILURE",
                                "IO_FAILURE"};
  const int i = static_cast<int>(code);
  return (i >= 0 && i < 13) ? names[i] : "UNKNOWN";
}

Error::Error(ErrorCode code, const std::string& message)
    : std::runtime_error(std::string(error_code_name(code)) + ": " + message), code_(code) {}

void raise(ErrorCode code, const std::string& message) { throw Error(code, message); }

namespace {
// C-ABI status -> mhar::Error (the engine's message already names the code).
void check(int status) {
  if (status == MHAR_OK) return;
  const std::string msg = mhar_last_error();
  if (status == MHAR_ERR_CUDA) throw std::runtime_error("CUDA: " + msg);
  throw Error(static_cast<ErrorCode>(status - 1), msg);
}
}  // namespace

// --------------------------------------------------------------- polytope --
// The reference's constructor checks (polytope.cpp:16-33, :90-97): every
// right-hand side matches its matrix, and equalities have the body's width
// (an empty a_eq takes it).  The engine reads exactly these extents.
static void require_shapes(const Polytope& p) {
  auto mismatch = [](const std::string& what, Index got, Index want) {
    raise(ErrorCode::dimension_mismatch, "polytope: " + what + " is " + std::to_string(got) +
                                             ", expected " + std::to_string(want));
  };
  if (p.b_in.size() != p.a_in.rows()) mismatch("b_in length", p.b_in.size(), p.a_in.rows());
  if (p.b_eq.size() != p.a_eq.rows()) mismatch("b_eq length", p.b_eq.size(), p.a_eq.rows());
  if (p.a_eq.cols() != p.a_in.cols()) mismatch("a_eq width", p.a_eq.cols(), p.a_in.cols());
}

Polytope::Polytope(Matrix a_in_, Vector b_in_) : a_in(std::move(a_in_)), b_in(std::move(b_in_)) {
  a_eq = Matrix(0, a_in.cols());
  require_shapes(*this);
}
Polytope::Polytope(Matrix a_in_, Vector b_in_, Matrix a_eq_, Vector b_eq_)
    : a_in(std::move(a_in_)), b_in(std::move(b_in_)), a_eq(std::move(a_eq_)),
      b_eq(std::move(b_eq_)) {
  if (a_eq.rows() == 0) a_eq = Matrix(0, a_in.cols());
  require_shapes(*this);
}

bool contains(const Polytope& p, const double* x, double eps) {
  for (Index i = 0; i < p.a_in.rows(); ++i) {
    double s = 0.0;
    for (Index j = 0; j < p.a_in.cols(); ++j) s += p.a_in(i, j) * x[j];
    if (s - p.b_in(i) > eps) return false;
  }
  for (Index i = 0; i < p.a_eq.rows(); ++i) {
    double s = 0.0;
    for (Index j = 0; j < p.a_eq.cols(); ++j) s += p.a_eq(i, j) * x[j];
    if (std::fabs(s - p.b_eq(i)) > eps) return false;
  }
  return true;
}

Polytope make_hypercube(int n) {
  if (n < 1) raise(ErrorCode::invalid_argument, "make_hypercube: n must be >= 1");
  Matrix a(2 * n, n);
  for (int i = 0; i < n; ++i) {
    a(i, i) = 1.0;
    a(n + i, i) = -1.0;
  }
  return Polytope(std::move(a), Vector::Ones(2 * n));
}

Polytope make_simplex(int n) {
  if (n < 2) raise(ErrorCode::invalid_argument, "make_simplex: n must be >= 2");
  Matrix a(n, n);
  for (int i = 0; i < n; ++i) a(i, i) = -1.0;
  return Polytope(std::move(a), Vector::Zero(n), Matrix::Constant(1, n, 1.0), Vector::Ones(1));
}

// ------------------------------------------------------------- projection --
ProjectionOperator compute_projection(const Matrix& a_eq) {
  if (a_eq.rows() == 0) raise(ErrorCode::invalid_argument, "compute_projection: empty");
  ProjectionOperator op;
  op.source_eq = a_eq;
  op.p = Matrix(a_eq.cols(), a_eq.cols());
  op.gram_inverse = Matrix(a_eq.rows(), a_eq.rows());
  check(mhar_compute_projection(a_eq.data(), a_eq.rows(), a_eq.cols(), op.p.data(),
                                op.gram_inverse.data()));
  return op;
}

// ---------------------------------------------------------------- engine --
class Engine {
 public:
  Engine(const Polytope& p, const ProjectionOperator* projector, int z, uint64_t seed,
         double eps_dir, double eps_feas, int rng_mode) {
    mhar_polytope poly{p.dim(), p.num_inequalities(), p.num_equalities(), p.a_in.data(),
                       p.b_in.data(), p.num_equalities() ? p.a_eq.data() : nullptr,
                       p.num_equalities() ? p.b_eq.data() : nullptr};
    mhar_options opt;
    mhar_default_options(&opt);
    opt.z = z;
    opt.seed = seed;
    opt.eps_dir = eps_dir;
    opt.eps_feas = eps_feas;
    opt.rng = rng_mode;
    check(mhar_ctx_create(&poly, projector ? projector->p.data() : nullptr,
                          projector ? projector->gram_inverse.data() : nullptr, &opt, &ctx_));
    eps_dir_ = eps_dir;
  }
  ~Engine() { mhar_ctx_destroy(ctx_); }
  mhar_ctx* ctx() { return ctx_; }
  double eps_dir() const { return eps_dir_; }
  // What the context was built from (step() rebinds when any of it changes):
  // the contents' hash and where they live.
  uint64_t fingerprint = 0;
  std::vector<uintptr_t> shape;
  // The reference streams continue across a rebind, as one WalkRng's do.
  void take_streams_from(Engine& other, int z) {
    std::vector<uint64_t> cols(static_cast<size_t>(z));
    uint64_t theta = 0;
    check(mhar_get_streams(other.ctx(), cols.data(), &theta));
    check(mhar_set_streams(ctx_, cols.data(), &theta));
  }
  void set_streams(const std::vector<uint64_t>& cols, uint64_t theta) {
    check(mhar_set_streams(ctx_, cols.data(), &theta));
  }
  long long redraws() {
    mhar_ctx_stats s;
    check(mhar_get_stats(ctx_, &s));
    return s.redraw_count;
  }

 private:
  mhar_ctx* ctx_ = nullptr;
  double eps_dir_ = 0.0;
};

namespace {
// 64-bit content hash (four interleaved multiply-xorshift lanes over 8-byte
// words, ~10 GB/s on one core): a polytope rebuilt at the same address with
// other rows must not reuse the old device copy.
uint64_t hash_block(const double* v, Index count, uint64_t h) {
  uint64_t lane[4] = {h ^ 0x9E3779B97F4A7C15ULL, h + 0xBF58476D1CE4E5B9ULL,
                      h ^ 0x94D049BB133111EBULL, h + 0x2545F4914F6CDD1DULL};
  auto mix = [](uint64_t x) {
    x ^= x >> 31;
    x *= 0x7FB5D329728EA185ULL;
    x ^= x >> 27;
    x *= 0x81DADEF4BC2DD44DULL;
    return x ^ (x >> 33);
  };
  Index i = 0;
  uint64_t w[4];
  for (; i + 4 <= count; i += 4) {
    std::memcpy(w, v + i, sizeof(w));
    for (int l = 0; l < 4; ++l) lane[l] = mix(lane[l] ^ w[l]) + 0x632BE59BD9B4E019ULL;
  }
  for (; i < count; ++i) {
    std::memcpy(w, v + i, 8);
    lane[0] = mix(lane[0] ^ w[0]);
  }
  return mix(lane[0] ^ mix(lane[1] ^ mix(lane[2] ^ mix(lane[3] ^ (uint64_t)count))));
}

// Large arrays (A_I is 3.2 GB at config 5) are hashed in fixed 16 MB blocks on
// the host's cores and the block hashes chained in order, so the value does
// not depend on the thread count and step() pays ~0.05 s, not ~0.3 s.
uint64_t hash_words(const double* v, Index count, uint64_t h) {
  constexpr Index kBlock = Index{1} << 21;  // doubles per block (16 MB)
  if (count <= kBlock) return hash_block(v, count, h);
  const Index blocks = (count + kBlock - 1) / kBlock;
  std::vector<uint64_t> part(static_cast<size_t>(blocks));
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const Index nth = std::min<Index>(blocks, hw);
  std::vector<std::thread> pool;
  for (Index t = 0; t < nth; ++t)
    pool.emplace_back([&, t] {
      for (Index b = t; b < blocks; b += nth)
        part[static_cast<size_t>(b)] =
            hash_block(v + b * kBlock, std::min(kBlock, count - b * kBlock), (uint64_t)b);
    });
  for (auto& th : pool) th.join();
  return hash_block(reinterpret_cast<const double*>(part.data()), blocks, h ^ (uint64_t)count);
}

uint64_t engine_fingerprint(const Polytope& p, const ProjectionOperator* projector,
                            const SamplerConfig& cfg) {
  uint64_t h = (uint64_t)p.dim() * 0x100000001B3ULL ^ (uint64_t)p.num_inequalities() << 20 ^
               (uint64_t)p.num_equalities();
  h = hash_words(p.a_in.data(), p.a_in.size(), h);
  h = hash_words(p.b_in.data(), p.b_in.size(), h);
  h = hash_words(p.a_eq.data(), p.a_eq.size(), h);
  h = hash_words(p.b_eq.data(), p.b_eq.size(), h);
  if (projector) {
    h = hash_words(projector->p.data(), projector->p.size(), h ^ 0x5bd1e995ULL);
    h = hash_words(projector->gram_inverse.data(), projector->gram_inverse.size(), h);
  }
  const double eps[2] = {cfg.eps_dir, cfg.eps_feas};
  return hash_words(eps, 2, h);
}

// Where the body's arrays live and how big they are, plus the tolerances: a
// cheap check that tells a new or reallocated body from the bound one.
std::vector<uintptr_t> body_shape(const Polytope& p, const ProjectionOperator* projector,
                                  const SamplerConfig& cfg) {
  uint64_t e[2];
  std::memcpy(&e[0], &cfg.eps_dir, 8);
  std::memcpy(&e[1], &cfg.eps_feas, 8);
  return {reinterpret_cast<uintptr_t>(&p), reinterpret_cast<uintptr_t>(p.a_in.data()),
          reinterpret_cast<uintptr_t>(p.b_in.data()), reinterpret_cast<uintptr_t>(p.a_eq.data()),
          reinterpret_cast<uintptr_t>(p.b_eq.data()), (uintptr_t)p.dim(),
          (uintptr_t)p.num_inequalities(), (uintptr_t)p.num_equalities(),
          reinterpret_cast<uintptr_t>(projector),
          projector ? reinterpret_cast<uintptr_t>(projector->p.data()) : 0,
          projector ? reinterpret_cast<uintptr_t>(projector->gram_inverse.data()) : 0,
          (uintptr_t)e[0], (uintptr_t)e[1]};
}
}  // namespace

// ---------------------------------------------------------------- sampler --
SamplerConfig resolve(const SamplerConfig& cfg, const Polytope& p) {
  SamplerConfig r = cfg;
  const int n = p.dim();
  const long long walk_dim = n - p.num_equalities();
  if (r.z == 0) r.z = std::max(p.num_inequalities(), n) + 1;
  if (r.phi == 0) r.phi = walk_dim * walk_dim * walk_dim;
  if (r.burn_in < 0) r.burn_in = r.phi;
  if (r.reproject_every < 0) r.reproject_every = r.phi;
  if (r.z < 1) raise(ErrorCode::invalid_argument, "config: z must be >= 1");
  if (r.phi < 1) raise(ErrorCode::invalid_argument, "config: phi must be >= 1");
  if (r.t_target < 1) raise(ErrorCode::invalid_argument, "config: t_target must be >= 1");
  if (!(r.eps_dir > 0.0)) raise(ErrorCode::invalid_argument, "config: eps_dir must be > 0");
  if (!(r.eps_feas > 0.0)) raise(ErrorCode::invalid_argument, "config: eps_feas must be > 0");
  return r;
}

LambdaIntervals compute_lambda_intervals(const Polytope& p, const Matrix& x, const Matrix& d,
                                         double eps_dir) {
  const Index n = p.dim(), z = x.cols();
  if (x.rows() != n || d.rows() != n || d.cols() != z) {
    raise(ErrorCode::dimension_mismatch, "compute_lambda_intervals: x is " +
                                             std::to_string(x.rows()) + "x" +
                                             std::to_string(x.cols()) + ", d is " +
                                             std::to_string(d.rows()) + "x" +
                                             std::to_string(d.cols()) + ", polytope dim " +
                                             std::to_string(n));
  }
  Engine eng(p, nullptr, static_cast<int>(z), 0, eps_dir, 1e-9, MHAR_RNG_PHILOX);
  LambdaIntervals out;
  out.lower = Vector(z);
  out.upper = Vector(z);
  std::vector<uint8_t> flags(static_cast<size_t>(z));
  check(mhar_lambda_intervals(eng.ctx(), x.data(), d.data(), out.lower.data(), out.upper.data(),
                              flags.data()));
  out.degenerate.resize(static_cast<size_t>(z));
  for (Index k = 0; k < z; ++k)
    out.degenerate[static_cast<size_t>(k)] = flags[static_cast<size_t>(k)] & MHAR_FLAG_DEGENERATE;
  return out;
}

double chord_point(double u, double lower, double upper) { return lower + u * (upper - lower); }

WalkRng::WalkRng(uint64_t seed, int z) : seed_(seed), z_(z) {
  if (z < 1) raise(ErrorCode::invalid_argument, "WalkRng: z must be >= 1, got " + std::to_string(z));
}
WalkRng::~WalkRng() = default;

// The streams live in a device context; without a polytope bound yet, a
// unit box of the requested dimension carries them (streams do not depend on
// the body).
Engine& WalkRng::engine_for_streams(int n) {
  if (!engine_) {
    static thread_local std::vector<std::unique_ptr<Polytope>> boxes;
    boxes.push_back(std::make_unique<Polytope>(make_hypercube(n)));
    engine_ = std::make_unique<Engine>(*boxes.back(), nullptr, z_, seed_, 1e-11, 1e-9,
                                       MHAR_RNG_REFERENCE);
    bound_ = boxes.back().get();
  }
  return *engine_;
}

Matrix generate_directions(WalkRng& rng, int n) {
  if (n < 1) raise(ErrorCode::invalid_argument, "generate_directions: n must be >= 1");
  Engine& e = rng.engine_for_streams(n);
  if (rng.bound_->dim() != n)
    raise(ErrorCode::dimension_mismatch, "generate_directions: streams are bound to dimension " +
                                             std::to_string(rng.bound_->dim()));
  Matrix h(n, rng.width());
  check(mhar_generate_directions(e.ctx(), h.data()));
  return h;
}

Matrix select_points(WalkRng& rng, const Matrix& x, const Matrix& d,
                     const LambdaIntervals& intervals) {
  const Index z = x.cols();
  if (d.cols() != z || intervals.lower.size() != z || intervals.upper.size() != z ||
      static_cast<Index>(intervals.degenerate.size()) != z || z != rng.width())
    raise(ErrorCode::dimension_mismatch, "select_points: inputs disagree on walk count");
  for (Index k = 0; k < z; ++k)
    if (intervals.degenerate[static_cast<size_t>(k)])
      raise(ErrorCode::direction_degenerate,
            "select_points: walk " + std::to_string(k) + " has no usable chord");
  Engine& e = rng.engine_for_streams(static_cast<int>(x.rows()));
  Matrix out(x.rows(), z);
  check(mhar_select_points(e.ctx(), x.data(), d.data(), intervals.lower.data(),
                           intervals.upper.data(), intervals.degenerate.data(), out.data()));
  return out;
}

void step(const Polytope& p, const ProjectionOperator* projector, const SamplerConfig& cfg,
          WalkRng& rng, WalkState& state) {
  if (state.x.cols() != rng.width() || state.x.rows() != p.dim())
    raise(ErrorCode::dimension_mismatch, "step: state does not match the rng width / polytope");
  // The walks' streams live with the device context: created on the first
  // step for this polytope, reused while the caller keeps stepping the same
  // body (contents, projector and tolerances -- not just its address).  A
  // rebind hands the streams over, so they continue exactly as one WalkRng's
  // do in the reference (rng.hpp:42-55).
  const std::vector<uintptr_t> shape = body_shape(p, projector, cfg);
  std::vector<uint64_t> saved;  // the streams before an optimistic step
  uint64_t saved_theta = 0;
  uint64_t fp = 0;
  if (rng.engine_ && rng.engine_->shape == shape) {
    // Same arrays as the bound body: step at once and re-hash the contents
    // on the host while the GPU works (A_I is 3.2 GB at config 5: the hash
    // costs about half an iterate).  Only a body edited in place since the
    // last call -- the hash differs -- discards this step and redoes it on a
    // rebound context from the streams saved before it.
    Engine& e = *rng.engine_;
    saved.resize(static_cast<size_t>(rng.width()));
    check(mhar_get_streams(e.ctx(), saved.data(), &saved_theta));
    const long long before = e.redraws();
    check(mhar_set_state(e.ctx(), state.x.data()));
    int st = mhar_step(e.ctx(), 1, 0);
    fp = engine_fingerprint(p, projector, cfg);  // overlaps the queued iterate
    if (st == MHAR_OK) st = mhar_sync(e.ctx());
    if (fp == e.fingerprint) {
      state.redraws += e.redraws() - before;
      check(st);
      check(mhar_get_state(e.ctx(), state.x.data()));
      ++state.j;
      return;
    }
  } else {
    fp = engine_fingerprint(p, projector, cfg);
  }
  if (!rng.engine_ || rng.bound_ != &p || rng.engine_->fingerprint != fp) {
    auto fresh = std::make_unique<Engine>(p, projector, rng.width(), rng.seed(), cfg.eps_dir,
                                          cfg.eps_feas, MHAR_RNG_REFERENCE);
    if (!saved.empty())
      fresh->set_streams(saved, saved_theta);
    else if (rng.engine_)
      fresh->take_streams_from(*rng.engine_, rng.width());
    fresh->fingerprint = fp;
    rng.engine_ = std::move(fresh);
    rng.bound_ = &p;
  }
  rng.engine_->shape = shape;
  mhar_ctx* ctx = rng.engine_->ctx();
  const long long before = rng.engine_->redraws();
  check(mhar_set_state(ctx, state.x.data()));
  int st = mhar_step(ctx, 1, 0);
  if (st == MHAR_OK) st = mhar_sync(ctx);
  state.redraws += rng.engine_->redraws() - before;
  check(st);
  check(mhar_get_state(ctx, state.x.data()));
  ++state.j;
}

namespace {
// MHAR_DEVICES="0,1,2,3": run() shards its walks over these GPUs.
std::vector<int> devices_from_env() {
  std::vector<int> out;
  const char* e = std::getenv("MHAR_DEVICES");
  if (!e) return out;
  std::string s(e);
  size_t pos = 0;
  while (pos < s.size()) {
    const size_t comma = s.find(',', pos);
    const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
    if (!tok.empty()) out.push_back(std::atoi(tok.c_str()));
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return out;
}
}  // namespace

SampleSet run(const Polytope& p, const SamplerConfig& cfg, const Vector& x0,
              const std::vector<int>& devices, const ClockFn& clock) {
  if (devices.empty()) raise(ErrorCode::invalid_argument, "run: empty device list");
  const SamplerConfig rc = resolve(cfg, p);
  if (x0.size() != p.dim()) raise(ErrorCode::dimension_mismatch, "run: x0 has the wrong size");
  auto now = [&clock]() {
    if (clock) return clock();
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  };
  const double t0 = now();
  std::unique_ptr<ProjectionOperator> projector;
  if (p.num_equalities() > 0)
    projector = std::make_unique<ProjectionOperator>(compute_projection(p.a_eq));
  const long long windows = (rc.t_target + rc.z - 1) / rc.z;
  mhar_polytope poly{p.dim(), p.num_inequalities(), p.num_equalities(), p.a_in.data(),
                     p.b_in.data(), p.num_equalities() ? p.a_eq.data() : nullptr,
                     p.num_equalities() ? p.b_eq.data() : nullptr};
  mhar_options opt;
  mhar_default_options(&opt);
  opt.z = rc.z;
  opt.seed = rc.seed;
  opt.eps_dir = rc.eps_dir;
  opt.eps_feas = rc.eps_feas;
  opt.rng = MHAR_RNG_PHILOX;  // walks keyed on global ids: shardable
  mhar_group* g = nullptr;
  check(mhar_group_create(&poly, projector ? projector->p.data() : nullptr,
                          projector ? projector->gram_inverse.data() : nullptr, &opt,
                          devices.data(), static_cast<int>(devices.size()), &g));
  std::unique_ptr<mhar_group, int (*)(mhar_group*)> guard(g, mhar_group_destroy);
  SampleSet out;
  out.config = rc;
  out.start = x0;
  out.windows = windows;
  out.samples = Matrix(windows * rc.z, p.dim());
  std::vector<double> rows(static_cast<size_t>(windows * rc.z * p.dim()));
  mhar_run_config rcfg{rc.phi, windows, rc.burn_in, projector ? rc.reproject_every : 0};
  mhar_run_stats stats;
  check(mhar_group_run(g, &rcfg, x0.data(), rows.data(), &stats));
  const Index n = p.dim();
  for (Index r = 0; r < windows * rc.z; ++r)
    for (Index j = 0; j < n; ++j) out.samples(r, j) = rows[static_cast<size_t>(r * n + j)];
  out.seconds = now() - t0;
  out.iterate_count = stats.iterate_count;
  out.redraw_count = stats.redraw_count;
  return out;
}

SampleSet run(const Polytope& p, const SamplerConfig& cfg, const Vector& x0, const ClockFn& clock) {
  const std::vector<int> devices = devices_from_env();
  if (!devices.empty()) return run(p, cfg, x0, devices, clock);
  const SamplerConfig rc = resolve(cfg, p);
  if (x0.size() != p.dim()) raise(ErrorCode::dimension_mismatch, "run: x0 has the wrong size");
  auto now = [&clock]() {
    if (clock) return clock();
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  };
  const double t0 = now();
  std::unique_ptr<ProjectionOperator> projector;
  if (p.num_equalities() > 0)
    projector = std::make_unique<ProjectionOperator>(compute_projection(p.a_eq));
  const long long windows = (rc.t_target + rc.z - 1) / rc.z;
  Engine eng(p, projector.get(), rc.z, rc.seed, rc.eps_dir, rc.eps_feas, MHAR_RNG_REFERENCE);
  SampleSet out;
  out.config = rc;
  out.start = x0;
  out.windows = windows;
  out.samples = Matrix(windows * rc.z, p.dim());
  // the engine writes row-major (windows*z) x n; transpose into the
  // column-major Matrix (one collected point per row, like the reference)
  std::vector<double> rows(static_cast<size_t>(windows * rc.z * p.dim()));
  mhar_run_config rcfg{rc.phi, windows, rc.burn_in, projector ? rc.reproject_every : 0};
  mhar_run_stats stats;
  check(mhar_run(eng.ctx(), &rcfg, x0.data(), rows.data(), &stats));
  const Index n = p.dim();
  for (Index r = 0; r < windows * rc.z; ++r)
    for (Index j = 0; j < n; ++j) out.samples(r, j) = rows[static_cast<size_t>(r * n + j)];
  out.seconds = now() - t0;
  out.iterate_count = stats.iterate_count;
  out.redraw_count = stats.redraw_count;
  return out;
}

ChebyshevCenter chebyshev_center(const Polytope& p) {
  mhar_polytope poly{p.dim(), p.num_inequalities(), p.num_equalities(), p.a_in.data(),
                     p.b_in.data(), p.num_equalities() ? p.a_eq.data() : nullptr,
                     p.num_equalities() ? p.b_eq.data() : nullptr};
  ChebyshevCenter c;
  c.x = Vector(p.dim());
  check(mhar_chebyshev_center(&poly, 0, c.x.data(), &c.radius, nullptr));
  return c;
}

SampleSet run(const Polytope& p, const SamplerConfig& cfg, const ClockFn& clock) {
  // sampler.cpp:274-276: resolve, then centre, before the clock starts
  resolve(cfg, p);
  const ChebyshevCenter center = chebyshev_center(p);
  SampleSet out = run(p, cfg, center.x, clock);
  out.start_radius = center.radius;
  return out;
}

}  // namespace mhar
