// C++ tests of the drop-in host API, restating the reference's own doctest
// cases (/root/reference/proj/tests/test_sampler.cpp, test_projection.cpp)
// against the B200 engine.  The z = 1 equivalence compares with the CPU
// oracle (oracle/mhar_oracle.h, test infrastructure) on the same streams.
// Run by tests/test_cpp_shim.py on a GPU box.
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../../oracle/mhar_oracle.h"
#include "mhar/bench.hpp"
#include "mhar/io.hpp"
#include "mhar/sampler.hpp"

using mhar::Matrix;
using mhar::Vector;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++g_fail;                                                              \
    }                                                                        \
  } while (0)

template <typename F>
static void expect_error(mhar::ErrorCode code, F f) {
  try {
    f();
    std::printf("  FAILED: expected %s\n", mhar::error_code_name(code));
    ++g_fail;
  } catch (const mhar::Error& e) {
    CHECK(e.code() == code);
  }
}

static void run_case(const char* name, const std::function<void()>& body) {
  const int before = g_fail;
  try {
    body();
  } catch (const std::exception& e) {
    std::printf("  FAILED: unexpected exception %s\n", e.what());
    ++g_fail;
  }
  std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
  if (g_fail == before) ++g_pass;
}

int main() {
  run_case("config defaults derive from the polytope shape", [] {
    const auto cube = mhar::make_hypercube(5);
    const auto rc = mhar::resolve(mhar::SamplerConfig{}, cube);
    CHECK(rc.z == 11 && rc.phi == 125 && rc.burn_in == 125 && rc.reproject_every == 125);
    const auto rs = mhar::resolve(mhar::SamplerConfig{}, mhar::make_simplex(4));
    CHECK(rs.z == 5 && rs.phi == 27);
    mhar::SamplerConfig bad;
    bad.z = -2;
    expect_error(mhar::ErrorCode::invalid_argument, [&] { mhar::resolve(bad, cube); });
  });

  run_case("chord bounds on the box match hand geometry", [] {
    const auto cube = mhar::make_hypercube(2);
    Matrix x(2, 2), d(2, 2);
    x(0, 1) = 0.5;
    d(0, 0) = 1.0;
    d(0, 1) = 1.0;
    const auto iv = mhar::compute_lambda_intervals(cube, x, d, 1e-11);
    CHECK(iv.lower(0) == -1.0 && iv.upper(0) == 1.0);
    CHECK(iv.lower(1) == -1.5 && iv.upper(1) == 0.5);
    CHECK(iv.degenerate[0] == 0 && iv.degenerate[1] == 0);
  });

  run_case("all-parallel directions are flagged", [] {
    const auto cube = mhar::make_hypercube(2);
    Matrix x(2, 1), d(2, 1);
    d(0, 0) = 1.0;
    const auto iv = mhar::compute_lambda_intervals(cube, x, d, 1e9);
    CHECK(iv.degenerate[0] == 1);
  });

  run_case("one-sided chords report an unbounded body", [] {
    Matrix a(2, 2);
    a(0, 0) = a(1, 1) = -1.0;
    const mhar::Polytope quadrant(a, Vector::Zero(2));
    Matrix x(2, 1, 1.0), d(2, 1);
    d(0, 0) = 0.3;
    d(1, 0) = 1.0;
    expect_error(mhar::ErrorCode::unbounded_polytope,
                 [&] { mhar::compute_lambda_intervals(quadrant, x, d, 1e-11); });
  });

  run_case("single steps keep every walk inside the body", [] {
    const auto cube = mhar::make_hypercube(4);
    const auto cfg = mhar::resolve(mhar::SamplerConfig{}, cube);
    mhar::WalkRng rng(cfg.seed, 6);
    mhar::WalkState state;
    state.x = Matrix::Zero(4, 6);
    for (int it = 0; it < 50; ++it) {
      mhar::step(cube, nullptr, cfg, rng, state);
      for (int k = 0; k < 6; ++k) CHECK(mhar::contains(cube, state.x.col(k), 1e-12));
    }
    CHECK(state.j == 50);
  });

  run_case("projected steps never leave the equality slice", [] {
    const auto simplex = mhar::make_simplex(5);
    const auto cfg = mhar::resolve(mhar::SamplerConfig{}, simplex);
    const auto op = mhar::compute_projection(simplex.a_eq);
    mhar::WalkRng rng(cfg.seed, 4);
    mhar::WalkState state;
    state.x = Vector::Constant(5, 0.2).replicate(4);
    for (int it = 0; it < 200; ++it) mhar::step(simplex, &op, cfg, rng, state);
    for (int k = 0; k < 4; ++k) {
      double s = 0;
      for (int i = 0; i < 5; ++i) s += state.x(i, k);
      CHECK(std::fabs(s - 1.0) <= 1e-9);
      CHECK(mhar::contains(simplex, state.x.col(k), 1e-9));
    }
  });

  run_case("hopeless direction retries give up with the retry error", [] {
    const auto cube = mhar::make_hypercube(2);
    auto cfg = mhar::resolve(mhar::SamplerConfig{}, cube);
    cfg.eps_dir = 1e9;
    mhar::WalkRng rng(55, 1);
    mhar::WalkState state;
    state.x = Matrix::Zero(2, 1);
    expect_error(mhar::ErrorCode::retry_exhausted,
                 [&] { mhar::step(cube, nullptr, cfg, rng, state); });
    CHECK(state.redraws == mhar::kMaxDirectionRetries);
  });

  run_case("full runs count batches, windows, and iterates", [] {
    const auto cube = mhar::make_hypercube(3);
    mhar::SamplerConfig cfg;
    cfg.z = 2;
    cfg.phi = 3;
    cfg.t_target = 4;
    cfg.burn_in = 0;
    cfg.seed = 7;
    const auto out = mhar::run(cube, cfg, Vector::Zero(3));
    CHECK(out.samples.rows() == 4 && out.samples.cols() == 3);
    CHECK(out.windows == 2 && out.iterate_count == 12);
    for (int r = 0; r < 4; ++r) {
      double x[3] = {out.samples(r, 0), out.samples(r, 1), out.samples(r, 2)};
      CHECK(mhar::contains(cube, x, cfg.eps_feas));
    }
    // without x0 the walks start at the Chebyshev centre: the origin, radius 1
    const auto centred = mhar::run(cube, cfg);
    CHECK(centred.start_radius == 1.0);
    CHECK(centred.start(0) == 0.0 && centred.start(1) == 0.0 && centred.start(2) == 0.0);
    CHECK(centred.samples == out.samples);
  });

  run_case("multi-GPU run: samples identical for every device list (mhar_group)", [] {
    const auto simplex = mhar::make_simplex(12);
    mhar::SamplerConfig cfg;
    cfg.z = 65;
    cfg.phi = 9;
    cfg.t_target = 65 * 3;
    cfg.seed = 5;
    const Vector x0 = Vector::Constant(12, 1.0 / 12);
    const auto one = mhar::run(simplex, cfg, x0, std::vector<int>{0});
    const auto three = mhar::run(simplex, cfg, x0, std::vector<int>{0, 0, 0});
    CHECK(one.samples.rows() == 195 && one.windows == 3 && one.iterate_count == 65 * 9 * 3);
    CHECK(one.samples == three.samples);
    for (int r = 0; r < 195; ++r) {
      double s = 0.0;
      for (int j = 0; j < 12; ++j) s += one.samples(r, j);
      CHECK(std::fabs(s - 1.0) <= 1e-9);
    }
    // the reference-facing overload takes the device list from MHAR_DEVICES
    setenv("MHAR_DEVICES", "0,0", 1);
    const auto env = mhar::run(simplex, cfg, x0);
    unsetenv("MHAR_DEVICES");
    CHECK(env.samples == one.samples);
    expect_error(mhar::ErrorCode::invalid_argument,
                 [&] { mhar::run(simplex, cfg, x0, std::vector<int>{}); });
  });

  run_case("chebyshev centres: box exact, simplex barycentre, errors", [] {
    for (int n : {2, 10, 100}) {
      const auto c = mhar::chebyshev_center(mhar::make_hypercube(n));
      CHECK(c.radius == 1.0);
      for (int i = 0; i < n; ++i) CHECK(c.x(i) == 0.0);
    }
    for (int n : {3, 4, 10}) {
      const auto c = mhar::chebyshev_center(mhar::make_simplex(n));
      CHECK(std::fabs(c.radius - 1.0 / n) <= 1e-8);
      for (int i = 0; i < n; ++i) CHECK(std::fabs(c.x(i) - 1.0 / n) <= 1e-8);
    }
    Matrix cone(1, 1);
    cone(0, 0) = -1.0;
    expect_error(mhar::ErrorCode::unbounded_polytope,
                 [&] { mhar::chebyshev_center(mhar::Polytope(cone, Vector{0.0})); });
    Matrix gap(2, 1);
    gap(0, 0) = 1.0;
    gap(1, 0) = -1.0;
    expect_error(mhar::ErrorCode::empty_polytope,
                 [&] { mhar::chebyshev_center(mhar::Polytope(gap, Vector{0.0, -1.0})); });
  });

  run_case("runs are bit-reproducible per seed and move between seeds", [] {
    const auto cube = mhar::make_hypercube(4);
    mhar::SamplerConfig cfg;
    cfg.z = 3;
    cfg.phi = 10;
    cfg.t_target = 30;
    cfg.seed = 99;
    const auto a = mhar::run(cube, cfg, Vector::Zero(4));
    const auto b = mhar::run(cube, cfg, Vector::Zero(4));
    CHECK(a.samples == b.samples);
    cfg.seed = 100;
    const auto c = mhar::run(cube, cfg, Vector::Zero(4));
    CHECK(!(a.samples == c.samples));
  });

  run_case("box moments settle near the uniform law", [] {
    const auto cube = mhar::make_hypercube(5);
    mhar::SamplerConfig cfg;
    cfg.z = 100;
    cfg.phi = 125;
    cfg.t_target = 10000;
    cfg.seed = 11;
    const auto out = mhar::run(cube, cfg, Vector::Zero(5));
    CHECK(out.samples.rows() == 10000);
    for (int c = 0; c < 5; ++c) {
      double m = 0, v = 0;
      for (int r = 0; r < 10000; ++r) m += out.samples(r, c);
      m /= 10000;
      for (int r = 0; r < 10000; ++r) v += (out.samples(r, c) - m) * (out.samples(r, c) - m);
      v /= 9999;
      CHECK(std::fabs(m) <= 0.05 && std::fabs(v - 1.0 / 3.0) <= 0.05);
    }
  });

  run_case("simplex projector is exact and z=1 walks retrace the oracle", [] {
    const auto simplex = mhar::make_simplex(4);
    const auto op = mhar::compute_projection(simplex.a_eq);
    Matrix expected(4, 4, -0.25);
    for (int i = 0; i < 4; ++i) expected(i, i) = 0.75;
    CHECK(op.p == expected);
    for (int body = 0; body < 2; ++body) {
      const auto p = body == 0 ? mhar::make_hypercube(5) : simplex;
      const auto cfg = mhar::resolve(mhar::SamplerConfig{}, p);
      const uint64_t seed = 4242;
      mhar::WalkRng rng(seed, 1);
      mhar::WalkState state;
      const int n = p.dim();
      state.x = Vector::Constant(n, body == 0 ? 0.0 : 0.25).replicate(1);
      std::vector<double> xr(state.x.data(), state.x.data() + n);
      uint64_t col = orc_stream_init(seed, 0), th = orc_stream_init(seed, ~0ULL);
      int64_t red = 0, err = -1;
      double worst = 0.0;
      for (int it = 0; it < 1000; ++it) {
        mhar::step(p, body == 0 ? nullptr : &op, cfg, rng, state);
        CHECK(orc_step(p.a_in.data(), p.b_in.data(), p.num_inequalities(), n,
                       body == 0 ? nullptr : op.p.data(), cfg.eps_dir, &col, &th, xr.data(), 1,
                       &red, &err) == 0);
        for (int j = 0; j < n; ++j) worst = std::fmax(worst, std::fabs(state.x(j, 0) - xr[j]));
      }
      CHECK(worst <= 1e-12);
    }
  });

  run_case("a body rebuilt at the same address is sampled, not the old one", [] {
    auto cfg = mhar::resolve(mhar::SamplerConfig{}, mhar::make_hypercube(3));
    mhar::WalkRng rng(cfg.seed, 8);
    mhar::WalkState state;
    state.x = Matrix::Zero(3, 8);
    mhar::Polytope body = mhar::make_hypercube(3);
    for (int it = 0; it < 5; ++it) mhar::step(body, nullptr, cfg, rng, state);
    // same object, same address, rows now bound the box at 1e-3
    body = mhar::Polytope(mhar::make_hypercube(3).a_in, Vector::Constant(6, 1e-3));
    state.x = Matrix::Zero(3, 8);
    for (int it = 0; it < 5; ++it) mhar::step(body, nullptr, cfg, rng, state);
    for (int k = 0; k < 8; ++k) CHECK(mhar::contains(body, state.x.col(k), 1e-15));
    // and a changed eps_feas / projector also rebinds (no stale context)
    cfg.eps_feas = 2e-9;
    mhar::step(body, nullptr, cfg, rng, state);
    for (int k = 0; k < 8; ++k) CHECK(mhar::contains(body, state.x.col(k), 1e-15));
  });

  run_case("polytope constructor checks shapes like the reference (polytope.cpp:16-33)", [] {
    using mhar::ErrorCode;
    expect_error(ErrorCode::dimension_mismatch,
                 [] { mhar::Polytope(Matrix::Zero(3, 2), Vector::Ones(2)); });
    expect_error(ErrorCode::dimension_mismatch, [] {
      mhar::Polytope(Matrix::Zero(3, 2), Vector::Ones(3), Matrix::Zero(1, 3), Vector::Ones(1));
    });
    expect_error(ErrorCode::dimension_mismatch, [] {
      mhar::Polytope(Matrix::Zero(3, 2), Vector::Ones(3), Matrix::Zero(1, 2), Vector::Ones(2));
    });
    const mhar::Polytope ok(Matrix::Zero(3, 2), Vector::Ones(3), Matrix(0, 0), Vector(0));
    CHECK(ok.a_eq.rows() == 0 && ok.a_eq.cols() == 2);
  });

  run_case("a body edited in place is sampled, on the same trajectory as a rebind", [] {
    // step() steps the bound context while it re-hashes the body; an in-place
    // edit must discard that step and redo it from the saved streams
    auto cfg = mhar::resolve(mhar::SamplerConfig{}, mhar::make_hypercube(3));
    mhar::WalkRng ra(cfg.seed, 8), rb(cfg.seed, 8);
    mhar::WalkState sa, sb;
    sa.x = Matrix::Zero(3, 8);
    sb.x = Matrix::Zero(3, 8);
    mhar::Polytope body = mhar::make_hypercube(3);
    const mhar::Polytope cube = mhar::make_hypercube(3);
    for (int it = 0; it < 3; ++it) {
      mhar::step(body, nullptr, cfg, ra, sa);
      mhar::step(cube, nullptr, cfg, rb, sb);
    }
    const double* storage = body.b_in.data();
    for (int i = 0; i < 6; ++i) body.b_in(i) = 0.5;  // same arrays, new contents
    CHECK(body.b_in.data() == storage);
    const mhar::Polytope half(cube.a_in, Vector::Constant(6, 0.5));
    for (int k = 0; k < 8; ++k)
      for (int i = 0; i < 3; ++i) {
        sa.x(i, k) *= 0.25;  // inside the smaller box
        sb.x(i, k) *= 0.25;
      }
    for (int it = 0; it < 4; ++it) {
      mhar::step(body, nullptr, cfg, ra, sa);
      mhar::step(half, nullptr, cfg, rb, sb);
    }
    double worst = 0.0;
    for (int k = 0; k < 8; ++k) {
      CHECK(mhar::contains(body, sa.x.col(k), 1e-15));
      for (int i = 0; i < 3; ++i) worst = std::fmax(worst, std::fabs(sa.x(i, k) - sb.x(i, k)));
    }
    CHECK(worst == 0.0);
    CHECK(sa.j == sb.j && sa.redraws == sb.redraws);
  });

  run_case("streams continue across generate_directions and a rebind to the body", [] {
    // the reference's WalkRng keeps its streams across calls: directions drawn
    // before the first step are not replayed by it
    const auto cube = mhar::make_hypercube(4);
    const auto cfg = mhar::resolve(mhar::SamplerConfig{}, cube);
    const int z = 5;
    const uint64_t seed = 31;
    mhar::WalkRng rng(seed, z);
    const Matrix h = mhar::generate_directions(rng, 4);
    mhar::WalkState state;
    state.x = Matrix::Zero(4, z);
    mhar::step(cube, nullptr, cfg, rng, state);
    mhar::step(cube, nullptr, cfg, rng, state);
    std::vector<uint64_t> cols(z);
    for (int k = 0; k < z; ++k) cols[k] = orc_stream_init(seed, (uint64_t)k);
    uint64_t th = orc_stream_init(seed, ~0ULL);
    std::vector<double> hr(4 * z), xr(4 * z, 0.0);
    orc_fill_standard_normal_matrix(cols.data(), z, hr.data(), 4);
    for (int i = 0; i < 4 * z; ++i) CHECK(std::fabs(hr[i] - h.data()[i]) <= 1e-15);
    int64_t red = 0, err = -1;
    for (int it = 0; it < 2; ++it)
      CHECK(orc_step(cube.a_in.data(), cube.b_in.data(), 8, 4, nullptr, cfg.eps_dir, cols.data(),
                     &th, xr.data(), z, &red, &err) == 0);
    double worst = 0.0;
    for (int i = 0; i < 4 * z; ++i) worst = std::fmax(worst, std::fabs(xr[i] - state.x.data()[i]));
    CHECK(worst <= 1e-14);
  });

  run_case("format_double is the shortest round trip (io.hpp:13)", [] {
    CHECK(mhar::format_double(0.1) == "0.1");
    CHECK(mhar::format_double(2.0) == "2");
    CHECK(mhar::format_double(-1.5e-9) == "-1.5e-09");
    CHECK(mhar::format_double(1.0 / 3.0) == "0.3333333333333333");
    uint64_t s = 12345;
    for (int i = 0; i < 2000; ++i) {
      s = s * 6364136223846793005ULL + 1442695040888963407ULL;
      double v;
      uint64_t bits = (s >> 2) | 0x3000000000000000ULL;  // finite, varied exponents
      std::memcpy(&v, &bits, 8);
      if (i & 1) v = -v;
      const std::string t = mhar::format_double(v);
      CHECK(std::strtod(t.c_str(), nullptr) == v);
    }
  });

  run_case("sample files round-trip and runs are byte-reproducible (acceptance #9)", [] {
    const auto cube = mhar::make_hypercube(3);
    mhar::SamplerConfig cfg;
    cfg.z = 16;
    cfg.phi = 20;
    cfg.t_target = 64;
    cfg.seed = 42;
    const auto a = mhar::run(cube, cfg, Vector::Zero(3));
    const auto b = mhar::run(cube, cfg, Vector::Zero(3));
    const std::string dir = "/tmp/mhar_shim_io_" + std::to_string(::getpid());
    if (std::system(("mkdir -p " + dir).c_str()) != 0) CHECK(false);
    mhar::write_sample_csv(dir + "/a.csv", a.samples);
    mhar::write_sample_csv(dir + "/b.csv", b.samples);
    auto slurp = [](const std::string& p) {
      std::ifstream in(p, std::ios::binary);
      std::ostringstream ss;
      ss << in.rdbuf();
      return ss.str();
    };
    CHECK(slurp(dir + "/a.csv") == slurp(dir + "/b.csv"));
    CHECK(slurp(dir + "/a.csv").rfind("x1,x2,x3\n", 0) == 0);
    CHECK(mhar::read_sample_csv(dir + "/a.csv") == a.samples);
    // test_io.cpp:94-108: ragged rows, bad tokens, a missing header, no file
    auto bad_file = [&](const std::string& text) {
      const std::string f = dir + "/bad.csv";
      std::ofstream(f, std::ios::binary) << text;
      expect_error(mhar::ErrorCode::io_failure, [&] { mhar::read_sample_csv(f); });
    };
    bad_file("x1,x2\n1,2\n3\n");
    bad_file("x1,x2\n1,banana\n");
    bad_file("x1,x2\n1,,2\n");
    bad_file("");
    expect_error(mhar::ErrorCode::io_failure, [&] { mhar::read_sample_csv(dir + "/none.csv"); });
    {
      std::ofstream(dir + "/empty_rows.csv", std::ios::binary) << "x1,x2\n1.5,-2\n\n3,4e-3";
      const Matrix r = mhar::read_sample_csv(dir + "/empty_rows.csv");
      CHECK(r.rows() == 2 && r.cols() == 2 && r(0, 0) == 1.5 && r(1, 1) == 4e-3);
    }
    mhar::write_sample_bin(dir + "/a.bin", a.samples);
    CHECK(mhar::read_sample_bin(dir + "/a.bin") == a.samples);
    const std::string man = mhar::manifest_string(a, "hypercube:3", dir + "/a.csv");
    CHECK(man.find("\"samples_written\": 64") != std::string::npos);
    CHECK(man.find("\"windows\": 4") != std::string::npos);
    CHECK(man.find("\"iterate_count\": 1280") != std::string::npos);
    CHECK(man.find("\"eps_dir\": 1e-11") != std::string::npos);
    if (std::system(("rm -rf " + dir).c_str()) != 0) CHECK(false);
  });

  // proj/tests/test_bench.cpp with scripted clocks
  auto scripted = [](std::vector<double> t) {
    auto st = std::make_shared<std::pair<std::vector<double>, size_t>>(std::move(t), 0);
    return mhar::ClockFn([st]() { return st->first[st->second++]; });
  };
  run_case("throughput: a scripted thousand-second run reports three thousand per second",
           [&] {
             mhar::BenchConfig cfg;
             cfg.phi = 30000;
             cfg.repetitions = 1;
             cfg.seed = 3;
             const auto r = mhar::measure_throughput(mhar::make_hypercube(2), 100, cfg,
                                                     "hypercube(2)", scripted({0.0, 1000.0}));
             CHECK(r.total_samples == 3000000);
             CHECK(r.run_seconds.size() == 1 && r.run_seconds[0] == 1000.0);
             CHECK(r.mean_sps == 3000.0 && r.std_sps == 0.0);
           });
  run_case("throughput: zero counts are rejected, rates are iterates over seconds", [&] {
    const auto cube = mhar::make_hypercube(3);
    mhar::BenchConfig cfg;
    cfg.repetitions = 0;
    expect_error(mhar::ErrorCode::invalid_argument,
                 [&] { mhar::measure_throughput(cube, 1, cfg, "hypercube(3)"); });
    cfg.repetitions = 1;
    expect_error(mhar::ErrorCode::invalid_argument,
                 [&] { mhar::measure_throughput(cube, 0, cfg, "hypercube(3)"); });
    expect_error(mhar::ErrorCode::invalid_argument,
                 [&] { mhar::sweep_padding(cube, {}, cfg, "hypercube(3)"); });
    cfg.phi = 7;
    cfg.windows = 3;
    cfg.repetitions = 2;
    const auto r = mhar::measure_throughput(cube, 5, cfg, "hypercube(3)", scripted({0, 4, 0, 8}));
    CHECK(r.total_samples == 5 * 7 * 3 && r.run_sps.size() == 2);
    for (size_t k = 0; k < 2; ++k) CHECK(r.run_sps[k] == (double)r.total_samples / r.run_seconds[k]);
    CHECK(r.mean_sps == (r.run_sps[0] + r.run_sps[1]) / 2.0);
  });
  run_case("throughput: a one-element sweep equals the direct measurement", [&] {
    const auto simplex = mhar::make_simplex(3);
    mhar::BenchConfig cfg;
    cfg.phi = 4;
    cfg.repetitions = 2;
    cfg.seed = 9;
    const auto d = mhar::measure_throughput(simplex, 2, cfg, "simplex(3)", scripted({0, 1, 1, 3}));
    const auto s = mhar::sweep_padding(simplex, {2}, cfg, "simplex(3)", scripted({0, 1, 1, 3}));
    CHECK(s.size() == 1 && s[0].z == d.z && s[0].total_samples == d.total_samples);
    CHECK(s[0].run_seconds == d.run_seconds && s[0].mean_sps == d.mean_sps &&
          s[0].std_sps == d.std_sps);
  });

  run_case("throughput csv and json (test_io.cpp bench cases)", [] {
    mhar::BenchRecord r;
    r.figure = "hypercube(50)";
    r.n = 50;
    r.z = 16;
    r.phi = 1000;
    r.windows = 1;
    r.total_samples = 16000;
    r.run_seconds = {1.0, 2.0};
    r.run_sps = {16000.0, 8000.0};
    r.mean_sps = 12000.0;
    r.std_sps = 4000.0;
    const std::string header = "figure,n,z,phi,windows,total_samples,mean_sps,std_sps,runs\n";
    const std::string text = mhar::bench_csv_string({r});
    CHECK(text.rfind(header, 0) == 0);
    CHECK(text.substr(header.size()) == "hypercube(50),50,16,1000,1,16000,12000,4000,2\n");
    CHECK(mhar::bench_csv_string({}) == header);
    mhar::BenchRecord q;
    q.figure = "simplex(10)";
    q.n = 10;
    q.z = 4;
    q.phi = 729;
    q.windows = 2;
    q.total_samples = 5832;
    q.run_seconds = {0.5, 0.25, 0.125};
    q.run_sps = {11664.0, 23328.0, 46656.0};
    q.mean_sps = 27216.0;
    q.std_sps = 17750.0;
    const std::string js = mhar::bench_json_string({q});
    CHECK(js.rfind("{\n  \"format_version\": 1,\n  \"records\": [\n    {\n", 0) == 0);
    CHECK(js.find("\"figure\": \"simplex(10)\"") != std::string::npos);
    CHECK(js.find("\"run_sps\": [\n        11664.0,\n        23328.0,\n        46656.0\n      ]") !=
          std::string::npos);
    CHECK(js.find("\"mean_sps\": 27216.0") != std::string::npos);
    expect_error(mhar::ErrorCode::io_failure,
                 [&] { mhar::write_bench_json("/nonexistent/dir/b.json", {q}); });
  });

  std::printf("%d passed, %d failed checks\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
