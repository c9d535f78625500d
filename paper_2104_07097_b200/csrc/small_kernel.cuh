// small_kernel.cuh -- walk-resident iterate kernel for small bodies.
//
// Walks never interact, so for polytopes whose A_I (and P, A_E) fit in
// shared memory a single launch can carry every walk through many iterates:
// one warp per walk, the body staged once per CTA in smem, the walk's x / h
// / d in smem, all of step() per iterate done by the warp
// (/root/reference/proj/src/sampler.cpp:235-272: normals, P h + collapse
// test, chord scan with the UNBOUNDED / degenerate semantics of :182-200,
// redraws of :105-123, draw_theta of :95-101, x += theta d), plus the
// reprojection cadence of run() (:304-311).  This removes the per-iterate
// launch chain that bounds small configurations (hypercube/simplex, n <= a
// few hundred).  The Philox keys are exactly those of the multi-kernel path
// (walk, iterate, attempt), and every dot product is an ascending-k FMA
// chain, the summation order of the CPU oracle.
#pragma once

#include "common.cuh"
#include "step_kernels.cuh"

namespace mhar_dev {

constexpr int SMALL_WARPS = 8;

struct SmallParams {
  const double* A;   // m x n column-major
  const double* b;   // m
  const double* P;   // n x n column-major, or null
  const double* AE;  // me x n column-major, or null
  const double* bE;  // me
  const double* G;   // me x me
  double* X;         // packed state (b_index)
  int64_t n, m, me, z, KT;
  uint64_t seed;
  int64_t chain_offset;
  int64_t it0, iters, reproject_every;
  double eps_dir;
  unsigned long long* redraw_total;
  const unsigned long long* err;
  unsigned long long* walk_err;  // per walk: (iterate << 24) | (phase << 8) | status
  int ns;                        // smem row stride (odd)
  const double* coef;            // stacked diagonal blocks (fastpath.cuh): per-row coefficient, or null
  int64_t diag_blocks;
  int factored;                  // 1: D = H - A_E' G A_E H instead of P H (P not staged)
};

// Per-warp scratch: x, h (and d when a dense P is applied; otherwise d is
// formed in place of h), res, g.
__host__ __device__ inline size_t small_warp_doubles(int64_t n, int64_t me, bool dense_proj) {
  return (dense_proj ? 3 : 2) * (size_t)n + 2 * (size_t)me;
}
__host__ __device__ inline size_t small_smem_doubles(int64_t n, int64_t m, int64_t me, bool proj,
                                                     int ns, bool diag = false,
                                                     bool factored = false,
                                                     int warps = SMALL_WARPS) {
  size_t s = diag ? 2 * (size_t)m : (size_t)m * ns + (size_t)m;  // A rows (or coefficients), b
  if (proj && !factored) s += (size_t)n * ns;      // P rows
  s += (size_t)me * ns + (size_t)me + (size_t)me * me;  // A_E, b_E, G
  s += (size_t)warps * small_warp_doubles(n, me, proj && !factored);
  return s;
}

__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

struct SmallChord {
  double lo, hi;
  unsigned sides;
};

// Chord of (x, d) against the smem rows: lanes own rows r = lane + 32 j.
__device__ inline SmallChord small_chord(const double* As, const double* bs, const double* xs,
                                         const double* ds, int64_t m, int64_t n, int ns,
                                         double eps, int lane) {
  double hi = __longlong_as_double(0x7FF0000000000000LL);
  double lo = -hi;
  unsigned sd = 0;
  for (int64_t r = lane; r < m; r += 32) {
    const double* a = As + r * ns;
    double ax = 0.0, ad = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      ax = fma(a[k], xs[k], ax);
      ad = fma(a[k], ds[k], ad);
    }
    const double sl = bs[r] - ax;
    if (ad > eps) {
      sd |= 1u;
      const double q = sl / ad;
      hi = q < hi ? q : hi;
    } else if (ad < -eps) {
      sd |= 2u;
      const double q = sl / ad;
      lo = q > lo ? q : lo;
    }
  }
  SmallChord c;
  c.hi = warp_min(hi);
  c.lo = warp_max(lo);
  for (int o = 16; o > 0; o >>= 1) sd |= __shfl_xor_sync(0xFFFFFFFFu, sd, o);
  c.sides = sd;
  return c;
}

// Chord of (x, d) against stacked diagonal blocks (sampler.cpp:166-172):
// lanes own coordinates; row blk n + k has coefficient cs[blk n + k].
__device__ inline SmallChord small_chord_diag(const double* cs, const double* bs, const double* xs,
                                              const double* ds, int64_t n, int64_t blocks,
                                              double eps, int lane) {
  double hi = __longlong_as_double(0x7FF0000000000000LL);
  double lo = -hi;
  unsigned sd = 0;
  for (int64_t k = lane; k < n; k += 32) {
    const double x = xs[k], d = ds[k];
    for (int64_t blk = 0; blk < blocks; ++blk) {
      const int64_t r = blk * n + k;
      const double sl = __dsub_rn(bs[r], __dmul_rn(x, cs[r]));  // one rounding each
      const double ad = __dmul_rn(d, cs[r]);
      if (ad > eps) {
        sd |= 1u;
        const double q = sl / ad;
        hi = q < hi ? q : hi;
      } else if (ad < -eps) {
        sd |= 2u;
        const double q = sl / ad;
        lo = q > lo ? q : lo;
      }
    }
  }
  SmallChord c;
  c.hi = warp_min(hi);
  c.lo = warp_max(lo);
  for (int o = 16; o > 0; o >>= 1) sd |= __shfl_xor_sync(0xFFFFFFFFu, sd, o);
  c.sides = sd;
  return c;
}

__global__ void __launch_bounds__(32 * SMALL_WARPS) small_kernel(const SmallParams p) {
  if (*p.err != kNoError) return;
  extern __shared__ __align__(16) double sm[];
  const int ns = p.ns;
  const int64_t n = p.n, m = p.m, me = p.me;
  const bool diag = p.coef != nullptr;
  double* As = sm;  // A rows, or the diagonal coefficients
  double* bs = As + (diag ? m : m * ns);
  double* Ps = bs + m;
  double* AEs = Ps + (p.P && !p.factored ? n * ns : 0);
  double* bEs = AEs + me * ns;
  double* Gs = bEs + me;
  double* wbase = Gs + me * me;
  if (diag) {
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) As[i] = p.coef[i];
  } else {
    for (int64_t i = threadIdx.x; i < m * n; i += blockDim.x) {
      const int64_t r = i % m, k = i / m;
      As[r * ns + k] = p.A[i];
    }
  }
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) bs[i] = p.b[i];
  if (p.P && !p.factored)
    for (int64_t i = threadIdx.x; i < n * n; i += blockDim.x) Ps[(i % n) * ns + i / n] = p.P[i];
  for (int64_t i = threadIdx.x; i < me * n; i += blockDim.x) AEs[(i % me) * ns + i / me] = p.AE[i];
  for (int64_t i = threadIdx.x; i < me; i += blockDim.x) bEs[i] = p.bE[i];
  for (int64_t i = threadIdx.x; i < me * me; i += blockDim.x) Gs[i] = p.G[i];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const bool dense_proj = p.P && !p.factored;
  double* xs = wbase + (size_t)warp * small_warp_doubles(n, me, dense_proj);
  double* hs = xs + n;
  double* dsb = dense_proj ? hs + n : hs;  // factored / no projection: d replaces h
  double* res = hs + (dense_proj ? 2 * n : n);
  double* gv = res + me;
  const int64_t ppc = (n + 1) / 2;
  unsigned long long redraws = 0;

  for (int64_t w = (int64_t)blockIdx.x * nwarps + warp; w < p.z;
       w += (int64_t)gridDim.x * nwarps) {
    const uint64_t gw = (uint64_t)(p.chain_offset + w);
    for (int64_t k = lane; k < n; k += 32) xs[k] = p.X[b_index(w, k, p.KT)];
    __syncwarp();
    unsigned long long werr = kNoError;
    for (int64_t t = p.it0; t < p.it0 + p.iters && werr == kNoError; ++t) {
      const double* d = nullptr;
      double lo = 0.0, hi = 0.0;
      bool done = false;
      for (int attempt = 0; attempt <= kMaxDirectionRetries && !done; ++attempt) {
        if (attempt > 0) ++redraws;
        // normals (rng.cpp:153-207 layout; Philox keyed like normals_kernel / redraw_kernel)
        for (int64_t pi = lane; pi < ppc; pi += 32) {
          uint64_t a, bb;
          philox_u64x2(p.seed, (uint32_t)pi, gw, (uint64_t)t, (uint32_t)attempt, kDomNormal, &a,
                       &bb);
          double cs, sn;
          box_muller(u01_open_closed(a), u01_closed_open(bb), &cs, &sn);
          hs[2 * pi] = cs;
          if (2 * pi + 1 < n) hs[2 * pi + 1] = sn;
        }
        __syncwarp();
        bool collapsed = false;
        if (p.P && p.factored) {
          // d = h - A_E' G (A_E h), the formula of proj_dot_kernel /
          // proj_apply_kernel (fastpath.cuh); the sums here run lane-strided
          // over the walk's coordinates, so the two paths agree to rounding
          for (int64_t i = 0; i < me; ++i) {
            double r = 0.0;
            for (int64_t k = lane; k < n; k += 32) r = fma(AEs[i * ns + k], hs[k], r);
            r = warp_sum(r);
            if (lane == 0) res[i] = r;
          }
          __syncwarp();
          for (int64_t i = lane; i < me; i += 32) {
            double s = 0.0;
            for (int64_t j = 0; j < me; ++j) s = fma(Gs[i + j * me], res[j], s);
            gv[i] = s;
          }
          __syncwarp();
          double sq = 0.0;
          for (int64_t k = lane; k < n; k += 32) {
            double s = 0.0;
            for (int64_t i = 0; i < me; ++i) s = fma(AEs[i * ns + k], gv[i], s);
            const double dk = hs[k] - s;
            dsb[k] = dk;  // dsb == hs: each lane rewrites only its own coordinates
            sq = fma(dk, dk, sq);
          }
          __syncwarp();
          collapsed = sqrt(warp_sum(sq)) <= kNearZeroDirection;
          d = dsb;
          if (attempt > 0 && collapsed) continue;
        } else if (p.P) {
          double sq = 0.0;
          for (int64_t i = lane; i < n; i += 32) {
            const double* pr = Ps + i * ns;
            double s = 0.0;
            for (int64_t k = 0; k < n; ++k) s = fma(pr[k], hs[k], s);
            dsb[i] = s;
            sq = fma(s, s, sq);
          }
          __syncwarp();
          collapsed = sqrt(warp_sum(sq)) <= kNearZeroDirection;
          d = dsb;
          if (attempt > 0 && collapsed) continue;  // redraw_column: collapsed -> next try
        } else {
          d = hs;
        }
        const SmallChord c = diag ? small_chord_diag(As, bs, xs, d, n, p.diag_blocks, p.eps_dir, lane)
                                  : small_chord(As, bs, xs, d, m, n, ns, p.eps_dir, lane);
        if (c.sides == 0u) continue;  // no usable side: degenerate, redraw
        if (c.sides != 3u) {          // one-sided: the body is unbounded
          werr = ((unsigned long long)t << 24) |
                 ((unsigned long long)(attempt == 0 ? PH_INTERVALS : PH_REDRAW) << 8) |
                 (unsigned long long)ST_UNBOUNDED;
          break;
        }
        if (!(c.hi - c.lo > kDegenerateWidth) || collapsed) continue;
        lo = c.lo;
        hi = c.hi;
        done = true;
      }
      if (werr != kNoError) break;
      if (!done) {
        werr = ((unsigned long long)t << 24) | ((unsigned long long)PH_REDRAW << 8) |
               (unsigned long long)ST_RETRY_EXHAUSTED;
        break;
      }
      // draw_theta (sampler.cpp:95-101), Philox keyed like theta_kernel
      double th = 0.0;
      if (lane == 0) {
        int r = 0;
        for (; r < kMaxThetaRejects; ++r) {
          uint64_t a, bb;
          philox_u64x2(p.seed, (uint32_t)r, gw, (uint64_t)t, 0, kDomTheta, &a, &bb);
          th = chord_point(u01_closed_open(a), lo, hi);
          if (th > lo && th < hi) break;
        }
        if (r == kMaxThetaRejects) th = chord_point(0.5, lo, hi);
      }
      th = __shfl_sync(0xFFFFFFFFu, th, 0);
      for (int64_t k = lane; k < n; k += 32) xs[k] = __dadd_rn(xs[k], __dmul_rn(th, d[k]));
      __syncwarp();
      // reproject_points every reproject_every global iterates (sampler.cpp:307-310)
      if (me > 0 && p.reproject_every > 0 && (t + 1) % p.reproject_every == 0) {
        for (int64_t i = lane; i < me; i += 32) {
          double s = 0.0;
          for (int64_t k = 0; k < n; ++k) s = fma(AEs[i * ns + k], xs[k], s);
          res[i] = s - bEs[i];
        }
        __syncwarp();
        for (int64_t i = lane; i < me; i += 32) {
          double s = 0.0;
          for (int64_t j = 0; j < me; ++j) s = fma(Gs[i + j * me], res[j], s);
          gv[i] = s;
        }
        __syncwarp();
        for (int64_t k = lane; k < n; k += 32) {
          double s = 0.0;
          for (int64_t i = 0; i < me; ++i) s = fma(AEs[i * ns + k], gv[i], s);
          xs[k] = xs[k] - s;
        }
        __syncwarp();
      }
    }
    for (int64_t k = lane; k < n; k += 32) p.X[b_index(w, k, p.KT)] = xs[k];
    if (lane == 0) p.walk_err[w] = werr;
    __syncwarp();
  }
  if (lane == 0 && redraws) atomicAdd(p.redraw_total, redraws);
}

// Canonical error word from the per-walk records: the earliest iterate, then
// the earliest phase, then the lowest walk -- where the reference's
// iterate-major loop would have raised first.
__global__ void small_error_kernel(const unsigned long long* walk_err, int64_t z,
                                   unsigned long long* err) {
  unsigned long long best = kNoError;
  int64_t best_w = -1;
  for (int64_t w = threadIdx.x; w < z; w += blockDim.x) {
    const unsigned long long e = walk_err[w];
    if (e != kNoError && (e < best || (e == best && w < best_w))) {
      best = e;
      best_w = w;
    }
  }
  __shared__ unsigned long long sb[256];
  __shared__ long long sw[256];
  sb[threadIdx.x] = best;
  sw[threadIdx.x] = best_w;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)blockDim.x; ++i)
      if (sb[i] != kNoError && (sb[i] < best || (sb[i] == best && sw[i] < best_w))) {
        best = sb[i];
        best_w = sw[i];
      }
    if (best != kNoError)
      atomicMin(err, error_word((int)((best >> 8) & 0xFF), best_w, (int)(best & 0xFF)));
  }
}

}  // namespace mhar_dev
