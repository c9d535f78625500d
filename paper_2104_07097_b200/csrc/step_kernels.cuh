// step_kernels.cuh -- the non-GEMM kernels of one MHAR iterate and the
// layout conversions.  Reference lines are in /root/reference/proj.
#pragma once

#include "common.cuh"

namespace mhar_dev {

constexpr double kDegenerateWidth = 1e-14;   // sampler.hpp:40
constexpr int kMaxDirectionRetries = 16;     // sampler.hpp:43
constexpr double kNearZeroDirection = 1e-12; // projection.hpp:25
constexpr int kMaxThetaRejects = 64;         // sampler.cpp:16

constexpr unsigned F_DEGENERATE = 1, F_HAS_UPPER = 2, F_HAS_LOWER = 4, F_COLLAPSED = 8,
                   F_THETA_MID = 16;

// Error phases (ordering of the reference's raises within one iterate).
constexpr int PH_INTERVALS = 0;  // compute_lambda_intervals (sampler.cpp:192-196)
constexpr int PH_REDRAW = 1;     // redraw_column (sampler.cpp:105-123)
constexpr int PH_COLLECT = 2;    // run() containment (sampler.cpp:319-324)

constexpr int ST_UNBOUNDED = 7, ST_RETRY_EXHAUSTED = 9, ST_NUMERICAL = 12;

// ------------------------------------------------------------- layouts -----

// col-major (n x ncols, ld) device matrix -> packed A operand (rows = r).
__global__ void pack_a_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                              int64_t ld, int64_t rows_pad, int64_t KT, double* __restrict__ dst) {
  const int64_t total = rows_pad * KT * BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    // decode a_index
    const int64_t e = i & 1;
    int64_t t = i >> 1;
    const int64_t lane = t & 31; t >>= 5;
    const int64_t rg = t & 15; t >>= 4;
    const int64_t k8 = t & 1; t >>= 1;
    const int64_t kt = t % KT;
    const int64_t mt = t / KT;
    const int64_t r = mt * BM + rg * 8 + (lane >> 2);
    const int64_t k = kt * BK + k8 * 8 + e * 4 + (lane & 3);
    dst[i] = (r < rows && k < cols) ? src[r + k * ld] : 0.0;
  }
}

// n x z column-major <-> packed state (b_index).  Pads are zero.
__global__ void pack_b_kernel(const double* __restrict__ src, int64_t n, int64_t z,
                              int64_t z_pad, int64_t KT, double* __restrict__ dst) {
  const int64_t total = z_pad * KT * BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, k;
    b_coords(i, KT, &c, &k);
    dst[i] = (c < z && k < n) ? src[k + c * n] : 0.0;
  }
}

// packed -> n x z column-major, which is also the row-major z x n sample
// layout of SampleSet::samples (one walk per row).
__global__ void unpack_b_kernel(const double* __restrict__ src, int64_t n, int64_t z,
                                int64_t KT, double* __restrict__ dst) {
  const int64_t total = n * z;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst[i] = src[b_index(i / n, i % n, KT)];
  }
}

// *flag = 1 if a and b differ anywhere (bitwise).
__global__ void differs_kernel(const double* __restrict__ a, const double* __restrict__ b,
                               int64_t total, int* flag) {
  int d = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    d |= __double_as_longlong(a[i]) != __double_as_longlong(b[i]);
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(flag, 1);
}

// x0 replicated into every walk column (run(), sampler.cpp:300).
__global__ void broadcast_state_kernel(const double* __restrict__ x0, int64_t n, int64_t z,
                                       int64_t z_pad, int64_t KT, double* __restrict__ X) {
  const int64_t total = z_pad * KT * BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, k;
    b_coords(i, KT, &c, &k);
    X[i] = (c < z && k < n) ? x0[k] : 0.0;
  }
}

// max_i (A x - b)_i keys -> doubles (containment), keys reset.
__global__ void viol_extract_kernel(long long* viol_key, double* viol, int64_t z) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= z) return;
  viol[c] = keyd(viol_key[c]);
  viol_key[c] = dkey(__longlong_as_double((long long)0xFFF0000000000000ULL));
}

__global__ void fill_keys_kernel(long long* hi, long long* lo, long long* viol, unsigned* sides,
                                 int64_t z_pad) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < z_pad;
       c += (int64_t)gridDim.x * blockDim.x) {
    hi[c] = dkey(__longlong_as_double(0x7FF0000000000000LL));
    lo[c] = dkey(__longlong_as_double((long long)0xFFF0000000000000ULL));
    viol[c] = lo[c];
    sides[c] = 0u;
  }
}

// --------------------------------------------------------------- RNG -------

struct RngParams {
  uint64_t seed;
  uint64_t iterate;       // global iterate counter (Philox key)
  const unsigned long long* iter_dev = nullptr;  // graph replays: the counter in device memory
  int64_t chain_offset;   // global id of local walk 0
  int64_t n, z, KT;
  int mode;               // 0 Philox, 1 reference SplitMix streams
  const uint64_t* col_state;  // reference mode: per-walk stream state
};

// H (packed) <- N(0,1): walk c, pair p -> coordinates 2p, 2p+1
// (fill_standard_normal_matrix, rng.cpp:153-207; odd n drops the last sine).
__global__ void normals_kernel(const RngParams rp, double* __restrict__ H,
                               const unsigned long long* err) {
  pdl_enter();
  if (*err != kNoError) return;
  const int64_t ppc = (rp.n + 1) / 2;
  // thread order follows the packed layout: a warp fills one (walk tile, k
  // tile, k8, column group) block of 8 walks x 8 coordinates -- 512
  // contiguous bytes -- one pair per thread
  const int64_t ct64 = (rp.z + BC - 1) / BC;
  const int64_t total = ct64 * rp.KT * 16 * 32;
  const uint32_t KT32 = (uint32_t)rp.KT;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = t >> 5;
    const int tl = (int)(t & 31);
    // (walk tile, k tile) of the block: 32-bit division (ct64 * KT < 2^32);
    // the 64-bit div/mod was a large share of this issue-bound kernel
    const uint32_t q = (uint32_t)(blk >> 4);
    const uint32_t kt = q % KT32, ct = q / KT32;
    const int cg = (int)(blk & 7), k8 = (int)((blk >> 3) & 1);
    const int64_t c = (int64_t)ct * BC + cg * 8 + (tl >> 2);
    const int64_t pidx = (int64_t)(kt * BK + k8 * 8) / 2 + (tl & 3);
    if (c >= rp.z || pidx >= ppc) continue;
    double u1, u2;
    if (rp.mode == 0) {
      uint64_t a, b;
      philox_u64x2(rp.seed, (uint32_t)pidx, (uint64_t)(rp.chain_offset + c),
                   rp.iter_dev ? (uint64_t)*rp.iter_dev : rp.iterate, 0,
                   kDomNormal, &a, &b);
      u1 = u01_open_closed(a);
      u2 = u01_closed_open(b);
    } else {
      const uint64_t st = rp.col_state[c];
      u1 = u01_open_closed(mix64(st + (uint64_t)(2 * pidx + 1) * kGolden));
      u2 = u01_closed_open(mix64(st + (uint64_t)(2 * pidx + 2) * kGolden));
    }
    double cs, sn;
    box_muller(u1, u2, &cs, &sn);
    // b_index(c, 2 pidx) and b_index(c, 2 pidx + 1) within this thread's
    // 512-byte block: lane = (c % 8) * 4 + k % 4, element (k % 8) / 4
    const int64_t o = blk * 64 + (tl >> 2) * 8 + (tl & 1) * 4 + ((tl >> 1) & 1);
    H[o] = cs;
    if (2 * pidx + 1 < rp.n) H[o + 2] = sn;
  }
}

// Reference streams: walk c consumed `draws` uniforms (the normals kernel
// reads the states without advancing them).
__global__ void advance_streams_kernel(uint64_t* col_state, int64_t z, int64_t draws) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < z) col_state[c] += (uint64_t)draws * kGolden;
}

// ------------------------------------------------ projection D = P H -------
// Straight DMMA tile product for the (small) n x n projector: one CTA per
// (128 output coordinates x 64 walks) tile, operands staged through smem.
// Output written in the packed B layout (rows = coordinates).
__global__ void __launch_bounds__(256) project_kernel(const double* __restrict__ Ppk,
                                                      const double* __restrict__ H,
                                                      double* __restrict__ D, int64_t n,
                                                      int64_t KT, const unsigned long long* err) {
  if (*err != kNoError) return;
  __shared__ __align__(16) double sa[A_PIECE];
  __shared__ __align__(16) double sb[B_PIECE];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile: 64 rows x 16 walks
  const int64_t mt = blockIdx.x, ct = blockIdx.y;
  double acc[8][2][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t kt = 0; kt < KT; ++kt) {
    const double2* ga = reinterpret_cast<const double2*>(Ppk + (mt * KT + kt) * A_PIECE);
    const double2* gb = reinterpret_cast<const double2*>(H + (ct * KT + kt) * B_PIECE);
    for (int i = tid; i < A_PIECE / 2; i += 256) reinterpret_cast<double2*>(sa)[i] = ga[i];
    for (int i = tid; i < B_PIECE / 2; i += 256) reinterpret_cast<double2*>(sb)[i] = gb[i];
    __syncthreads();
#pragma unroll
    for (int k8 = 0; k8 < 2; ++k8) {
      double2 af[8], bf[2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        af[i] = reinterpret_cast<const double2*>(sa)[(k8 * 16 + wm * 8 + i) * 32 + lane];
#pragma unroll
      for (int j = 0; j < 2; ++j)
        bf[j] = reinterpret_cast<const double2*>(sb)[(k8 * 8 + wn * 2 + j) * 32 + lane];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma884(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
          dmma884(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = mt * BM + wm * 64 + i * 8 + (lane >> 2);
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = ct * BC + wn * 16 + j * 8 + 2 * (lane & 3) + e;
        D[b_index(c, r, KT)] = acc[i][j][e];
      }
  }
}

// --------------------------------------------------------- finalize --------
// Turns the reduced keys into LambdaIntervals (sampler.cpp:182-200): no side
// -> degenerate with (0, 0); one side -> UNBOUNDED_POLYTOPE; width <= 1e-14
// -> degenerate; collapsed projections -> degenerate (sampler.cpp:256).
// Degenerate walks are queued for the redraw kernel.  Keys are reset.
struct FinalizeParams {
  long long* hi_key;
  long long* lo_key;
  long long* viol_key;
  unsigned* sides;
  const unsigned* collapsed;  // may be null
  double* lower;
  double* upper;
  double* viol;
  unsigned* flags;
  int* redraw_list;
  int* redraw_count;
  unsigned long long* err;
  uint64_t* col_state;     // reference mode: advance by the main draw (may be null)
  int64_t draws_per_walk;  // 2 * ceil(n/2)
  int64_t z;
};

__global__ void finalize_kernel(const FinalizeParams fp) {
  pdl_enter();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= fp.z) return;
  const double hi = keyd(fp.hi_key[c]);
  const double lo = keyd(fp.lo_key[c]);
  const unsigned sd = fp.sides[c];
  if (fp.viol) fp.viol[c] = keyd(fp.viol_key[c]);
  fp.hi_key[c] = dkey(__longlong_as_double(0x7FF0000000000000LL));
  fp.lo_key[c] = dkey(__longlong_as_double((long long)0xFFF0000000000000ULL));
  fp.viol_key[c] = fp.lo_key[c];
  fp.sides[c] = 0u;
  if (fp.col_state) fp.col_state[c] += (uint64_t)fp.draws_per_walk * kGolden;
  unsigned f = ((sd & 1u) ? F_HAS_UPPER : 0u) | ((sd & 2u) ? F_HAS_LOWER : 0u);
  double l = lo, u = hi;
  if (sd == 0u) {
    l = 0.0;
    u = 0.0;
    f |= F_DEGENERATE;
  } else if (sd != 3u) {
    atomicMin(fp.err, error_word(PH_INTERVALS, c, ST_UNBOUNDED));
    f |= F_DEGENERATE;
  } else if (!(u - l > kDegenerateWidth)) {
    f |= F_DEGENERATE;
  }
  if (fp.collapsed && fp.collapsed[c]) f |= F_COLLAPSED | F_DEGENERATE;
  fp.lower[c] = l;
  fp.upper[c] = u;
  fp.flags[c] = f;
  if ((f & F_DEGENERATE) && fp.redraw_list) {
    const int slot = atomicAdd(fp.redraw_count, 1);
    fp.redraw_list[slot] = (int)c;
  }
}

// ----------------------------------------------------------- redraw --------
// redraw_column (sampler.cpp:105-123) for every queued walk: up to 16 fresh
// directions from that walk's own stream, projected when P exists, each with
// a full chord (GEMV column_interval, sampler.cpp:73-93).  One CTA per walk;
// measure-zero for Gaussian rows, forced in tests with a huge eps_dir.
struct RedrawParams {
  const double* A;        // packed
  const double* b;        // padded
  const double* X;        // packed
  double* D;              // packed (updated on success)
  const double* P;        // n x n column-major, or null
  double* R;              // incremental rate cache (s_index) or null
  int64_t ct64;
  int64_t tc_walk_tiles;  // > 0: tcgen05 tile cache layout (tile_cache_index)
  int64_t c3_tiles;       // > 0: chord3's cache layout (c3_index)
  int64_t cache_rows;     // its row tile
  int rate_f32;           // 1: fp32 rate cache (fp32 variant)
  double* scratch;        // 3 n doubles per CTA
  double* lower;
  double* upper;
  unsigned* flags;
  const int* redraw_list;
  const int* redraw_count;
  int* attempts;          // per walk, this iterate
  unsigned long long* redraw_total;
  unsigned long long* err;
  uint64_t seed, iterate;
  const unsigned long long* iter_dev = nullptr;  // graph replays: the counter in device memory
  int64_t chain_offset;
  uint64_t* col_state;    // reference mode
  int mode;
  int64_t n, m, KT;
  double eps_dir;
};

__device__ inline double block_reduce(double v, double* red, int op /*0 min 1 max 2 sum*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xFFFFFFFFu, v, off);
    v = op == 0 ? fmin(v, o) : op == 1 ? fmax(v, o) : v + o;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane]
                                      : (op == 0 ? INFINITY : op == 1 ? -INFINITY : 0.0);
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xFFFFFFFFu, v, off);
      v = op == 0 ? fmin(v, o) : op == 1 ? fmax(v, o) : v + o;
    }
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) redraw_kernel(const RedrawParams rp) {
  pdl_enter();
  double* xs = rp.scratch + (size_t)blockIdx.x * 3 * rp.n;  // n
  double* hs = xs + rp.n;                                    // n
  double* ds = xs + 2 * rp.n;                                // n
  __shared__ double red[32];
  __shared__ int s_stop;
  const int count = *rp.redraw_count;
  for (int li = blockIdx.x; li < count; li += gridDim.x) {
    // An interval-phase failure means the reference raised before its redraw
    // loop (sampler.cpp:192-196 precedes :258-265): do nothing.
    if (threadIdx.x == 0)
      s_stop = (*(volatile unsigned long long*)rp.err >> 56) < (unsigned long long)PH_REDRAW;
    __syncthreads();
    if (s_stop) return;
    const int c = rp.redraw_list[li];
    for (int64_t k = threadIdx.x; k < rp.n; k += blockDim.x) xs[k] = rp.X[b_index(c, k, rp.KT)];
    uint64_t st = rp.mode ? rp.col_state[c] : 0;
    const int64_t ppc = (rp.n + 1) / 2;
    int attempt = 0;
    bool ok = false;
    double lo = 0.0, hi = 0.0;
    int status = ST_RETRY_EXHAUSTED;
    for (; attempt < kMaxDirectionRetries && !ok; ++attempt) {
      __syncthreads();
      for (int64_t pidx = threadIdx.x; pidx < ppc; pidx += blockDim.x) {
        double u1, u2;
        if (rp.mode == 0) {
          uint64_t a, b;
          philox_u64x2(rp.seed, (uint32_t)pidx, (uint64_t)(rp.chain_offset + c),
                       rp.iter_dev ? (uint64_t)*rp.iter_dev : rp.iterate,
                       (uint32_t)(attempt + 1), kDomNormal, &a, &b);
          u1 = u01_open_closed(a);
          u2 = u01_closed_open(b);
        } else {
          u1 = u01_open_closed(mix64(st + (uint64_t)(2 * pidx + 1) * kGolden));
          u2 = u01_closed_open(mix64(st + (uint64_t)(2 * pidx + 2) * kGolden));
        }
        double cs, sn;
        box_muller(u1, u2, &cs, &sn);
        hs[2 * pidx] = cs;
        if (2 * pidx + 1 < rp.n) hs[2 * pidx + 1] = sn;
      }
      st += (uint64_t)(2 * ppc) * kGolden;
      __syncthreads();
      if (rp.P) {
        for (int64_t i = threadIdx.x; i < rp.n; i += blockDim.x) {
          double s = 0.0;
          for (int64_t k = 0; k < rp.n; ++k) s = fma(rp.P[i + k * rp.n], hs[k], s);
          ds[i] = s;
        }
        __syncthreads();
        double sq = 0.0;
        for (int64_t i = threadIdx.x; i < rp.n; i += blockDim.x) sq = fma(ds[i], ds[i], sq);
        sq = block_reduce(sq, red, 2);
        if (sqrt(sq) <= kNearZeroDirection) continue;
      } else {
        for (int64_t i = threadIdx.x; i < rp.n; i += blockDim.x) ds[i] = hs[i];
        __syncthreads();
      }
      double tlo = -INFINITY, thi = INFINITY;
      double pos = 0.0, neg = 0.0;
      for (int64_t r = threadIdx.x; r < rp.m; r += blockDim.x) {
        double ax = 0.0, ad = 0.0;
        for (int64_t k = 0; k < rp.n; ++k) {
          const double a = rp.A[a_index(r, k, rp.KT)];
          ax = fma(a, xs[k], ax);
          ad = fma(a, ds[k], ad);
        }
        const double sl = rp.b[r] - ax;
        if (rp.R && rp.tc_walk_tiles > 0 && rp.rate_f32)  // fp32 variant: fp32 rate cache
          reinterpret_cast<float*>(rp.R)[tile_cache_index(r, c, rp.tc_walk_tiles, rp.cache_rows)] =
              (float)ad;
        else if (rp.R && rp.tc_walk_tiles > 0)  // int8-slice engine: fp64 rates, tile layout
          rp.R[tile_cache_index(r, c, rp.tc_walk_tiles, rp.cache_rows)] = ad;
        else if (rp.R && rp.c3_tiles > 0)
          rp.R[c3_index(r, c, rp.c3_tiles)] = ad;
        else if (rp.R)
          rp.R[s_index(r, c, rp.ct64)] = ad;
        if (ad > rp.eps_dir) {
          pos = 1.0;
          thi = fmin(thi, sl / ad);
        } else if (ad < -rp.eps_dir) {
          neg = 1.0;
          tlo = fmax(tlo, sl / ad);
        }
      }
      thi = block_reduce(thi, red, 0);
      tlo = block_reduce(tlo, red, 1);
      pos = block_reduce(pos, red, 1);
      neg = block_reduce(neg, red, 1);
      if (pos == 0.0 && neg == 0.0) continue;  // degenerate, try again
      if (pos == 0.0 || neg == 0.0) {
        status = ST_UNBOUNDED;
        ++attempt;
        break;
      }
      if (thi - tlo > kDegenerateWidth) {
        ok = true;
        lo = tlo;
        hi = thi;
      }
    }
    if (threadIdx.x == 0) {
      rp.attempts[c] = attempt;
      atomicAdd(rp.redraw_total, (unsigned long long)attempt);
      if (rp.mode) rp.col_state[c] = st;
    }
    if (ok) {
      for (int64_t k = threadIdx.x; k < rp.n; k += blockDim.x) rp.D[b_index(c, k, rp.KT)] = ds[k];
      if (threadIdx.x == 0) {
        rp.lower[c] = lo;
        rp.upper[c] = hi;
        rp.flags[c] = (rp.flags[c] & ~F_DEGENERATE) | F_HAS_UPPER | F_HAS_LOWER;
      }
    } else if (threadIdx.x == 0) {
      atomicMin(rp.err, error_word(PH_REDRAW, c, status));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ theta --------
// draw_theta (sampler.cpp:95-101): theta = lower + u (upper - lower) with
// open-interval rejection, 64 tries then the midpoint.  Reference mode reads
// the shared theta stream at counter base + k + 1 (no rejections); a walk that
// rejects marks the first such k for the sequential fix-up below.
struct ThetaParams {
  const double* lower;
  const double* upper;
  unsigned* flags;
  double* theta;
  const unsigned long long* err;
  uint64_t seed, iterate;
  const unsigned long long* iter_dev = nullptr;  // graph replays: the counter in device memory
  int64_t chain_offset, z;
  int mode;
  uint64_t* theta_state;  // reference mode (device scalar)
  int* first_reject;      // reference mode
  const double* injected_u;  // test hook: U[k] replaces the stream (may be null)
};

__device__ inline double chord_point(double u, double lower, double upper) {
  return __dadd_rn(lower, __dmul_rn(u, __dsub_rn(upper, lower)));  // sampler.cpp:210-212
}

__global__ void theta_kernel(const ThetaParams tp) {
  pdl_enter();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= tp.z) return;
  if (*tp.err != kNoError) return;
  const double lo = tp.lower[c], hi = tp.upper[c];
  unsigned f = tp.flags[c];
  double th = 0.0;
  if (tp.injected_u) {
    if (!(f & F_DEGENERATE)) {
      th = chord_point(tp.injected_u[c], lo, hi);
      if (!(th > lo && th < hi)) {
        th = chord_point(0.5, lo, hi);
        f |= F_THETA_MID;
      }
    }
  } else if (tp.mode == 0) {
    int r = 0;
    for (; r < kMaxThetaRejects; ++r) {
      uint64_t a, b;
      philox_u64x2(tp.seed, (uint32_t)r, (uint64_t)(tp.chain_offset + c),
                   tp.iter_dev ? (uint64_t)*tp.iter_dev : tp.iterate, 0,
                   kDomTheta, &a, &b);
      th = chord_point(u01_closed_open(a), lo, hi);
      if (th > lo && th < hi) break;
    }
    if (r == kMaxThetaRejects) {
      th = chord_point(0.5, lo, hi);
      f |= F_THETA_MID;
    }
  } else {
    const uint64_t st = *tp.theta_state + (uint64_t)(c + 1) * kGolden;
    th = chord_point(u01_closed_open(mix64(st)), lo, hi);
    if (!(th > lo && th < hi)) atomicMin(tp.first_reject, (int)c);
  }
  tp.theta[c] = th;
  tp.flags[c] = f;
}

// Reference mode: advance the theta stream by z draws, or -- if some walk
// rejected -- redo the draws sequentially from that walk on, exactly as the
// reference's k = 0..z-1 loop consumes the single stream (sampler.cpp:267-270).
__global__ void theta_fixup_kernel(ThetaParams tp) {
  pdl_enter();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*tp.err != kNoError) return;
  const int first = *tp.first_reject;
  uint64_t st = *tp.theta_state;
  if (first >= tp.z) {
    *tp.theta_state = st + (uint64_t)tp.z * kGolden;
    return;
  }
  st += (uint64_t)first * kGolden;
  for (int64_t c = first; c < tp.z; ++c) {
    const double lo = tp.lower[c], hi = tp.upper[c];
    double th = 0.0;
    int r = 0;
    for (; r < kMaxThetaRejects; ++r) {
      st += kGolden;
      th = chord_point(u01_closed_open(mix64(st)), lo, hi);
      if (th > lo && th < hi) break;
    }
    if (r == kMaxThetaRejects) {
      th = chord_point(0.5, lo, hi);
      tp.flags[c] |= F_THETA_MID;
    }
    tp.theta[c] = th;
  }
  *tp.theta_state = st;
  *tp.first_reject = 0x7FFFFFFF;
}

// x_k += theta_k d_k over the packed state (sampler.cpp:269).  Walks that
// did not move (injected-hook degenerates) carry theta = 0.
__global__ void axpy_kernel(double* __restrict__ X, const double* __restrict__ D,
                            const double* __restrict__ theta, int64_t total2, int64_t KT,
                            const unsigned long long* err) {
  pdl_enter();
  if (*err != kNoError) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total2;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, k;
    b_coords(2 * i, KT, &c, &k);
    const double t = __ldg(theta + c);
    double2 x = reinterpret_cast<double2*>(X)[i];
    const double2 d = __ldg(reinterpret_cast<const double2*>(D) + i);
    x.x = __dadd_rn(x.x, __dmul_rn(t, d.x));
    x.y = __dadd_rn(x.y, __dmul_rn(t, d.y));
    reinterpret_cast<double2*>(X)[i] = x;
  }
}

// -------------------------------------------------------- equalities -------
// reproject_points (projection.cpp:53-60): res = A_E x - b_E;
// g = G res; x -= A_E' g.  Also the equality residual of contains().
__global__ void eq_residual_kernel(const double* __restrict__ AE /*m_eq x n col-major*/,
                                   const double* __restrict__ bE, const double* __restrict__ X,
                                   int64_t me, int64_t n, int64_t z, int64_t KT,
                                   double* __restrict__ res /*me x z*/) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= me * z) return;
  const int64_t i = t % me, c = t / me;
  double s = 0.0;
  for (int64_t k = 0; k < n; ++k) s = fma(AE[i + k * me], X[b_index(c, k, KT)], s);
  res[i + c * me] = s - bE[i];
}

__global__ void eq_gram_kernel(const double* __restrict__ G /*me x me*/,
                               const double* __restrict__ res, int64_t me, int64_t z,
                               double* __restrict__ g) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= me * z) return;
  const int64_t i = t % me, c = t / me;
  double s = 0.0;
  for (int64_t j = 0; j < me; ++j) s = fma(G[i + j * me], res[j + c * me], s);
  g[i + c * me] = s;
}

__global__ void eq_correct_kernel(const double* __restrict__ AE, const double* __restrict__ g,
                                  double* __restrict__ X, int64_t me, int64_t n, int64_t z,
                                  int64_t KT) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * z) return;
  const int64_t k = t % n, c = t / n;
  double s = 0.0;
  for (int64_t i = 0; i < me; ++i) s = fma(AE[i + k * me], g[i + c * me], s);
  const int64_t idx = b_index(c, k, KT);
  X[idx] = X[idx] - s;
}

__global__ void eq_maxabs_kernel(const double* __restrict__ res, int64_t me, int64_t z,
                                 double* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= z) return;
  double w = 0.0;
  for (int64_t i = 0; i < me; ++i) w = fmax(w, fabs(res[i + c * me]));
  out[c] = w;
}

// Containment at collection (run(), sampler.cpp:319-324): first walk whose
// max (A x - b) or max |A_E x - b_E| exceeds eps.
__global__ void contains_kernel(const double* __restrict__ viol, const double* __restrict__ eqv,
                                int64_t z, double eps, unsigned long long* err, int set_error,
                                int* first_bad) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= z) return;
  const bool bad = !(viol[c] <= eps) || (eqv && !(eqv[c] <= eps));
  if (bad) {
    atomicMin(first_bad, (int)c);
    if (set_error) atomicMin(err, error_word(PH_COLLECT, c, ST_NUMERICAL));
  }
}

// worst containment slack of a collection: max over walks of
// max(viol[c], eqv[c]) into *out (one block)
__global__ void worst_violation_kernel(const double* __restrict__ viol,
                                       const double* __restrict__ eqv, int64_t z, double* out) {
  __shared__ double red[32];
  double v = -INFINITY;
  for (int64_t c = threadIdx.x; c < z; c += blockDim.x) {
    v = fmax(v, viol[c]);
    if (eqv) v = fmax(v, eqv[c]);
  }
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    if (threadIdx.x == 0) *out = v;
  }
}

// the device copy of the iterate counter (CUDA-graph replays of an iterate)
__global__ void iter_set_kernel(unsigned long long* it, unsigned long long v) { *it = v; }
__global__ void iter_inc_kernel(unsigned long long* it) {
  pdl_enter();
  *it += 1ull;
}

}  // namespace mhar_dev
