// C++ drop-in step() loop vs the bare C-ABI iterate at BASELINE config 5
// (n = 2000, m_I = 2e5 unit-norm Gaussian rows, 4096 walks): what the shim's
// per-call body check costs once it overlaps the queued iterate.
// Build from the repo root (after __graft_entry__.build()):
//   g++ -O2 -std=c++20 -Ipaper_2104_07097_b200/cpp/include tools/shim_step_rate.cpp \
//       -Lpaper_2104_07097_b200/lib -lmhar_cpp -lmhar_b200 \
//       -Wl,-rpath,'$ORIGIN/../paper_2104_07097_b200/lib' -o tools/shim_step_rate
//   ./tools/shim_step_rate [iterates]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../include/mhar_b200.h"
#include "mhar/sampler.hpp"

int main(int argc, char** argv) {
  const int n = 2000, m = 200000, z = 4096, iters = argc > 1 ? std::atoi(argv[1]) : 10;
  mhar::Matrix a(m, n);
  {
    std::mt19937_64 g(7);
    std::normal_distribution<double> N(0.0, 1.0);
    std::vector<double> row(n);
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += (row[j] = N(g)) * row[j];
      s = 1.0 / std::sqrt(s);
      for (int j = 0; j < n; ++j) a(i, j) = row[j] * s;
    }
  }
  const mhar::Polytope body(std::move(a), mhar::Vector::Ones(m));
  auto cfg = mhar::resolve(mhar::SamplerConfig{}, body);
  auto secs = [](auto t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  // (a) the reference's step(p, op, cfg, rng, state) loop through the shim
  mhar::WalkRng rng(cfg.seed, z);
  mhar::WalkState state;
  state.x = mhar::Matrix::Zero(n, z);
  for (int w = 0; w < 2; ++w) mhar::step(body, nullptr, cfg, rng, state);
  auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it) mhar::step(body, nullptr, cfg, rng, state);
  const double shim = secs(t0) / iters;
  // (b) the same per-call work on the C ABI: state in, one iterate, state out
  mhar_polytope poly{n, m, 0, body.a_in.data(), body.b_in.data(), nullptr, nullptr};
  mhar_options opt;
  mhar_default_options(&opt);
  opt.z = z;
  opt.rng = MHAR_RNG_REFERENCE;
  mhar_ctx* ctx = nullptr;
  if (mhar_ctx_create(&poly, nullptr, nullptr, &opt, &ctx)) return 1;
  std::vector<double> x(static_cast<size_t>(n) * z, 0.0);
  auto one = [&] {
    mhar_set_state(ctx, x.data());
    mhar_step(ctx, 1, 0);
    mhar_sync(ctx);
    mhar_get_state(ctx, x.data());
  };
  for (int w = 0; w < 2; ++w) one();
  t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it) one();
  const double abi = secs(t0) / iters;
  mhar_ctx_destroy(ctx);
  std::printf("{\"config\": 5, \"walks\": %d, \"iterates\": %d, \"shim_step_ms\": %.2f, "
              "\"c_abi_step_ms\": %.2f, \"shim_overhead_pct\": %.1f}\n",
              z, iters, 1e3 * shim, 1e3 * abi, 100.0 * (shim / abi - 1.0));
  return 0;
}
