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
//
// Group width (round 2): a walk takes GW = 4, 8, 16 or 32 lanes
// (small_group_width, from a sweep on the paper's bodies), so a warp carries
// 32 / GW walks.  With one walk per warp a 3-dimensional
// hypercube left 29 of 32 lanes idle in every phase; the groups' reductions
// are shuffles within the group's lanes (the sums' order depends on GW,
// which depends on the body alone).
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
  unsigned long long* err_min;   // min over walks of walk_err (kNoError: none failed)
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
// Lanes per walk, fitted to a sweep on the paper's bodies (tools/small_gw.sh,
// profiles/small_gw_r02.jsonl; within 3 % of the best width on average):
// the least power of two >= the walk's widest phase (its coordinates, or its
// rows when A_I is staged) / 2, 4 to 32; with an equality projection the
// per-walk work grows and narrower groups (more walks per warp) win: units / 8,
// widened while fewer than 1600 warps would carry the z walks.
__host__ __device__ inline int small_group_width(int64_t n, int64_t m, bool diag, bool proj,
                                                 int64_t z) {
  const int64_t units = diag ? n : (n > m ? n : m);
  const int64_t per = proj ? 8 : 2, min_warps = proj ? 1600 : 0;
  int gw = 4;
  while (gw < 32 && gw * per < units) gw <<= 1;
  while (gw < 32 && z * gw < min_warps * 32) gw <<= 1;
  return gw;
}
__host__ __device__ inline size_t small_smem_doubles(int64_t n, int64_t m, int64_t me, bool proj,
                                                     int ns, bool diag = false,
                                                     bool factored = false,
                                                     int warps = SMALL_WARPS, int gw = 32) {
  size_t s = diag ? 2 * (size_t)m : (size_t)m * ns + (size_t)m;  // A rows (or coefficients), b
  if (proj && !factored) s += (size_t)n * ns;      // P rows
  s += (size_t)me * ns + (size_t)me + (size_t)me * me;  // A_E, b_E, G
  s += (size_t)warps * (32 / gw) * small_warp_doubles(n, me, proj && !factored);
  return s;
}

// reductions over a walk's GW lanes (mask: the group's lanes)
template <int GW>
__device__ __forceinline__ double grp_min(double v, unsigned mask) {
  for (int o = GW / 2; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(mask, v, o));
  return v;
}
template <int GW>
__device__ __forceinline__ double grp_max(double v, unsigned mask) {
  for (int o = GW / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, o));
  return v;
}
template <int GW>
__device__ __forceinline__ double grp_sum(double v, unsigned mask) {
  for (int o = GW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}
template <int GW>
__device__ __forceinline__ unsigned grp_or(unsigned v, unsigned mask) {
  for (int o = GW / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(mask, v, o);
  return v;
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

// Chord of (x, d) against the smem rows: group lanes own rows r = gl + GW j.
template <int GW>
__device__ inline SmallChord small_chord(const double* As, const double* bs, const double* xs,
                                         const double* ds, int64_t m, int64_t n, int ns,
                                         double eps, int gl, unsigned gmask) {
  double hi = __longlong_as_double(0x7FF0000000000000LL);
  double lo = -hi;
  unsigned sd = 0;
  for (int64_t r = gl; r < m; r += GW) {
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
  c.hi = grp_min<GW>(hi, gmask);
  c.lo = grp_max<GW>(lo, gmask);
  c.sides = grp_or<GW>(sd, gmask);
  return c;
}

// Chord of (x, d) against stacked diagonal blocks (sampler.cpp:166-172):
// group lanes own coordinates; row blk n + k has coefficient cs[blk n + k].
template <int GW>
__device__ inline SmallChord small_chord_diag(const double* cs, const double* bs, const double* xs,
                                              const double* ds, int64_t n, int64_t blocks,
                                              double eps, int gl, unsigned gmask) {
  double hi = __longlong_as_double(0x7FF0000000000000LL);
  double lo = -hi;
  unsigned sd = 0;
  for (int64_t k = gl; k < n; k += GW) {
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
  c.hi = grp_min<GW>(hi, gmask);
  c.lo = grp_max<GW>(lo, gmask);
  c.sides = grp_or<GW>(sd, gmask);
  return c;
}

template <int GW>
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

  constexpr int WPW = 32 / GW;  // walks per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = lane % GW, grp = lane / GW;  // lane within the walk's group, group in the warp
  const unsigned gmask = (GW == 32 ? 0xFFFFFFFFu : ((1u << GW) - 1u)) << (grp * GW);
  const int nwarps = blockDim.x >> 5;
  const bool dense_proj = p.P && !p.factored;
  double* xs = wbase + (size_t)(warp * WPW + grp) * small_warp_doubles(n, me, dense_proj);
  double* hs = xs + n;
  double* dsb = dense_proj ? hs + n : hs;  // factored / no projection: d replaces h
  double* res = hs + (dense_proj ? 2 * n : n);
  double* gv = res + me;
  const int64_t ppc = (n + 1) / 2;
  unsigned long long redraws = 0;

  for (int64_t w = ((int64_t)blockIdx.x * nwarps + warp) * WPW + grp; w < p.z;
       w += (int64_t)gridDim.x * nwarps * WPW) {
    const uint64_t gw = (uint64_t)(p.chain_offset + w);
    for (int64_t k = gl; k < n; k += GW) xs[k] = p.X[b_index(w, k, p.KT)];
    __syncwarp(gmask);
    unsigned long long werr = kNoError;
    for (int64_t t = p.it0; t < p.it0 + p.iters && werr == kNoError; ++t) {
      const double* d = nullptr;
      double lo = 0.0, hi = 0.0;
      bool done = false;
      for (int attempt = 0; attempt <= kMaxDirectionRetries && !done; ++attempt) {
        if (attempt > 0) ++redraws;
        // normals (rng.cpp:153-207 layout; Philox keyed like normals_kernel / redraw_kernel)
        for (int64_t pi = gl; pi < ppc; pi += GW) {
          uint64_t a, bb;
          philox_u64x2(p.seed, (uint32_t)pi, gw, (uint64_t)t, (uint32_t)attempt, kDomNormal, &a,
                       &bb);
          double cs, sn;
          box_muller(u01_open_closed(a), u01_closed_open(bb), &cs, &sn);
          hs[2 * pi] = cs;
          if (2 * pi + 1 < n) hs[2 * pi + 1] = sn;
        }
        __syncwarp(gmask);
        bool collapsed = false;
        if (p.P && p.factored) {
          // d = h - A_E' G (A_E h), the formula of proj_dot_kernel /
          // proj_apply_kernel (fastpath.cuh); the sums here run group-lane-strided
          // over the walk's coordinates, so the two paths agree to rounding
          for (int64_t i = 0; i < me; ++i) {
            double r = 0.0;
            for (int64_t k = gl; k < n; k += GW) r = fma(AEs[i * ns + k], hs[k], r);
            r = grp_sum<GW>(r, gmask);
            if (gl == 0) res[i] = r;
          }
          __syncwarp(gmask);
          for (int64_t i = gl; i < me; i += GW) {
            double s = 0.0;
            for (int64_t j = 0; j < me; ++j) s = fma(Gs[i + j * me], res[j], s);
            gv[i] = s;
          }
          __syncwarp(gmask);
          double sq = 0.0;
          for (int64_t k = gl; k < n; k += GW) {
            double s = 0.0;
            for (int64_t i = 0; i < me; ++i) s = fma(AEs[i * ns + k], gv[i], s);
            const double dk = hs[k] - s;
            dsb[k] = dk;  // dsb == hs: each group lane rewrites only its own coordinates
            sq = fma(dk, dk, sq);
          }
          __syncwarp(gmask);
          collapsed = sqrt(grp_sum<GW>(sq, gmask)) <= kNearZeroDirection;
          d = dsb;
          if (attempt > 0 && collapsed) continue;
        } else if (p.P) {
          double sq = 0.0;
          for (int64_t i = gl; i < n; i += GW) {
            const double* pr = Ps + i * ns;
            double s = 0.0;
            for (int64_t k = 0; k < n; ++k) s = fma(pr[k], hs[k], s);
            dsb[i] = s;
            sq = fma(s, s, sq);
          }
          __syncwarp(gmask);
          collapsed = sqrt(grp_sum<GW>(sq, gmask)) <= kNearZeroDirection;
          d = dsb;
          if (attempt > 0 && collapsed) continue;  // redraw_column: collapsed -> next try
        } else {
          d = hs;
        }
        const SmallChord c =
            diag ? small_chord_diag<GW>(As, bs, xs, d, n, p.diag_blocks, p.eps_dir, gl, gmask)
                 : small_chord<GW>(As, bs, xs, d, m, n, ns, p.eps_dir, gl, gmask);
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
      if (gl == 0) {
        int r = 0;
        for (; r < kMaxThetaRejects; ++r) {
          uint64_t a, bb;
          philox_u64x2(p.seed, (uint32_t)r, gw, (uint64_t)t, 0, kDomTheta, &a, &bb);
          th = chord_point(u01_closed_open(a), lo, hi);
          if (th > lo && th < hi) break;
        }
        if (r == kMaxThetaRejects) th = chord_point(0.5, lo, hi);
      }
      th = __shfl_sync(gmask, th, grp * GW);
      for (int64_t k = gl; k < n; k += GW) xs[k] = __dadd_rn(xs[k], __dmul_rn(th, d[k]));
      __syncwarp(gmask);
      // reproject_points every reproject_every global iterates (sampler.cpp:307-310)
      if (me > 0 && p.reproject_every > 0 && (t + 1) % p.reproject_every == 0) {
        for (int64_t i = gl; i < me; i += GW) {
          double s = 0.0;
          for (int64_t k = 0; k < n; ++k) s = fma(AEs[i * ns + k], xs[k], s);
          res[i] = s - bEs[i];
        }
        __syncwarp(gmask);
        for (int64_t i = gl; i < me; i += GW) {
          double s = 0.0;
          for (int64_t j = 0; j < me; ++j) s = fma(Gs[i + j * me], res[j], s);
          gv[i] = s;
        }
        __syncwarp(gmask);
        for (int64_t k = gl; k < n; k += GW) {
          double s = 0.0;
          for (int64_t i = 0; i < me; ++i) s = fma(AEs[i * ns + k], gv[i], s);
          xs[k] = xs[k] - s;
        }
        __syncwarp(gmask);
      }
    }
    for (int64_t k = gl; k < n; k += GW) p.X[b_index(w, k, p.KT)] = xs[k];
    if (gl == 0) {
      p.walk_err[w] = werr;
      if (werr != kNoError) atomicMin(p.err_min, werr);  // rare: the resolver scans only then
    }
    __syncwarp(gmask);
  }
  if (gl == 0 && redraws) atomicAdd(p.redraw_total, redraws);
}

// Canonical error word from the per-walk records: the earliest iterate, then
// the earliest phase, then the lowest walk -- where the reference's
// iterate-major loop would have raised first.
__global__ void small_error_kernel(const unsigned long long* walk_err, int64_t z,
                                   unsigned long long* err_min, unsigned long long* err) {
  // no walk failed (the common case): nothing to resolve.  The word is read
  // by every thread before thread 0 re-arms it for the next launch.
  const unsigned long long any = *(volatile unsigned long long*)err_min;
  __syncthreads();
  if (threadIdx.x == 0) *err_min = kNoError;
  if (any == kNoError) return;
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
