// chord_kernel.cuh -- the fused fp64 tensor-core chord kernels.
//
// Restates, for all walks at once, compute_lambda_intervals
// (/root/reference/proj/src/sampler.cpp:150-208) with its per-walk
// chord_scan (src/vmath.hpp:83-155):
//
//   slack = b_I - A_I x,  rate = A_I d,
//   upper_k = min{ slack_i / rate_i : rate_i >  eps_dir }
//   lower_k = max{ slack_i / rate_i : rate_i < -eps_dir }
//
// as persistent kernels: a DMMA.8x8x4 product over pre-permuted operand tiles
// streamed HBM -> smem by the TMA bulk-copy engine through an mbarrier ring,
// whose epilogue forms the ratios in registers and reduces them (registers ->
// warp shuffles -> one order-preserving int64 atomic per walk per warp).
//
// Modes (template):
//   FUSED        B = [X | D] per 64-walk tile: both products, bounds, and
//                max_i (A x - b) (contains(), polytope.cpp:177-190) for free.
//                The m_I x z products never reach HBM.
//   FUSED_STORE  FUSED + writes slack and rate into the incremental cache.
//   INCREMENTAL  B = D: only A_I D is multiplied; the slack of the moved walks
//                comes from the cache, slack_t = slack_{t-1} - theta_{t-1}
//                rate_{t-1}, which holds because x_t = x_{t-1} + theta_{t-1}
//                d_{t-1} (half the flops of FUSED).
//   CHECK        B = X: max_i (A x - b) only (collection-time containment).
//
// FUSED* run one 256-thread CTA per SM on a 128-row x (64 x + 64 d) tile
// (warp tile 64 x 32, 128 accumulator doubles per thread).  INCREMENTAL and
// CHECK run TWO 256-thread CTAs per SM on 128-row x 64-walk tiles (warp tile
// 32 x 32), so one CTA's epilogue overlaps the other's tensor-core work.
#pragma once

#include "common.cuh"

namespace mhar_dev {

enum ChordMode { FUSED = 0, FUSED_STORE = 1, INCREMENTAL = 2, CHECK = 3, SLACK_STORE = 4 };

constexpr int CHORD_THREADS = 256;
// FUSED* kernel (1 CTA / SM)
constexpr int CHORD_STAGES = 6;  // 6 x 32 KB ring
constexpr int CHORD_LAG = 2;     // refill the slot consumed two stages ago
constexpr int STAGE_DOUBLES = A_PIECE + 2 * B_PIECE;
constexpr size_t CHORD_SMEM = (size_t)CHORD_STAGES * STAGE_DOUBLES * sizeof(double) + 1024;
// INCREMENTAL / CHECK kernel (2 CTAs / SM)
#ifndef MHAR_CHORD2_STAGES
#define MHAR_CHORD2_STAGES 4
#endif
#ifndef MHAR_CHORD_RED
#define MHAR_CHORD_RED 1  // RED reductions; the volatile pre-check loads were measured 1-3 % slower
#endif
#ifndef MHAR_CHORD2_KEEP
#define MHAR_CHORD2_KEEP 1
#endif
#ifndef MHAR_CHORD2_STREAMING
#define MHAR_CHORD2_STREAMING 1
#endif
#ifndef MHAR_CHORD2_PREFETCH
#define MHAR_CHORD2_PREFETCH 0  // L2 bulk prefetch of the slack block: measured 2 % slower
#endif
constexpr int CHORD2_STAGES = MHAR_CHORD2_STAGES;  // 4 x 24 KB ring per CTA
#ifndef MHAR_CHORD2_LAG
#define MHAR_CHORD2_LAG 1
#endif
constexpr int CHORD2_LAG = MHAR_CHORD2_LAG;
constexpr int STAGE2_DOUBLES = A_PIECE + B_PIECE;
constexpr int CHORD2_UQ = 8;  // announced-unit queue (> stages: the producer's lead in units)
constexpr size_t CHORD2_SMEM = (size_t)CHORD2_STAGES * STAGE2_DOUBLES * sizeof(double) + 512;

struct ChordParams {
  const double* A;  // packed A_I (a_index)
  const double* X;  // packed state (b_index)
  const double* D;  // packed directions (b_index)
  const double* b;  // b_I padded to m_pad with +inf
  double* S;        // slack cache (s_index)
  double* R;        // rate cache (s_index)
  const double* theta_prev;  // previous chord positions (z_pad)
  long long* hi_key;
  long long* lo_key;
  long long* viol_key;
  unsigned* sides;
  const unsigned long long* err;
  int64_t m_tiles;    // m_pad / 128
  int64_t KT;         // n_pad / 16
  int64_t col_tiles;  // 64-walk tiles
  int64_t z;          // live walks
  double eps_dir;
  int group_m;        // rasterisation band height (m tiles)
  int walk_band;      // > 0: walk-tile bands instead (see unit_coords)
  int64_t tc_walk_tiles;  // > 0: the slack cache uses a tcgen05 tile layout (tile_cache_index)
  int64_t cache_rows;     // its row tile: 256 (fp32 variant, fp32 rates) or 64 (int8 slices)
  int rate_f32;           // 1: the rate cache holds fp32 (fp32 variant)
  unsigned* sched;        // chord2 unit tickets [next, finished CTAs]; zero between launches
  int64_t c3_tiles;       // > 0: the DMMA slack cache is chord3's (c3_index over 128-walk tiles)
  unsigned long long* prof;  // chord3 per-CTA phase cycle counters (MHAR_C3_PROFILE), or null
};

// Slack-cache index for FUSED_STORE: the layout of whichever kernel consumes it.
__device__ inline int64_t cache_index(int64_t r, int64_t c, const ChordParams& p) {
  if (p.tc_walk_tiles > 0) return tile_cache_index(r, c, p.tc_walk_tiles, p.cache_rows);
  if (p.c3_tiles > 0) return c3_index(r, c, p.c3_tiles);
  return s_index(r, c, p.col_tiles);
}

// Unit u -> (row tile, walk tile).  walk_band > 0: bands of walk_band walk
// tiles, the row tiles inner -- the band's direction tiles stay L2-resident
// and each A_I tile is read once per band while the units in flight share it
// (A_I streamed col_tiles / walk_band times).  Otherwise bands of group_m row
// tiles with the walk tiles inner (A_I read once, every direction tile
// re-read per row band).
__device__ inline void unit_coords(int64_t u, const ChordParams& p, int64_t* mt, int64_t* ct) {
  if (p.walk_band > 0) {
    const int64_t band_units = (int64_t)p.walk_band * p.m_tiles;
    const int64_t band = u / band_units;
    const int64_t in_band = u - band * band_units;
    const int64_t start = band * p.walk_band;
    const int64_t w = (p.col_tiles - start < p.walk_band) ? p.col_tiles - start : p.walk_band;
    *ct = start + in_band % w;
    *mt = in_band / w;
    return;
  }
  const int64_t band_units = (int64_t)p.group_m * p.col_tiles;
  const int64_t band = u / band_units;
  const int64_t in_band = u - band * band_units;
  const int64_t start = band * p.group_m;
  const int64_t h = (p.m_tiles - start < p.group_m) ? p.m_tiles - start : p.group_m;
  *mt = start + in_band % h;
  *ct = in_band / h;
}

// One row of the chord scan for walk bounds (hi, lo) with the exact
// candidate filter: a row can only move a bound if its ratio beats it, and
// the sign of fma(-bound, rate, slack) -- the sign of the exact value --
// decides that, so the division runs only for candidates and the result is
// bit-identical to dividing every row.
__device__ __forceinline__ void scan_row(double sl, double ad, double eps, double& hi, double& lo,
                                         unsigned& sd) {
  if (ad > eps) {
    sd |= 1u;
    if (!(fma(-hi, ad, sl) > 0.0)) {
      const double q = sl / ad;
      hi = q < hi ? q : hi;
    }
  } else if (ad < -eps) {
    sd |= 2u;
    if (!(fma(-lo, ad, sl) >= 0.0)) {
      const double q = sl / ad;
      lo = q > lo ? q : lo;
    }
  }
}

// scan_row with the fp64 pipe kept free for the tensor cores (chord3's
// epilogue).  DMMA and the fp64 SIMT instructions (DFMA, DADD, DSETP) issue
// on the same fp64 datapath, so an epilogue doing its tests in fp64 waits
// behind the co-resident warps' MMAs (ncu: stall_math).  Here the bounds are
// carried as their order-preserving keys (dkey) and every test is an integer
// compare of bit patterns:
// - |ad| > eps and the sign of ad from the bits (the mask through PTX: the
//   compiler would turn a C-level `& 0x7FF..F` of a double's bits back into a
//   DADD |x|);
// - an integer log-domain estimate skips rows whose ratio is provably beyond
//   the current bound: for positive normal x the bit pattern
//   B(x) / 2^52 - 1023 is within 0.0861 below log2 x, so with sl normal
//   B(sl) - B(ad) > B(bound) - B(1) + 0.2 * 2^52 implies sl / ad > bound
//   (the row cannot move it; a negative or subnormal operand only makes the
//   test more conservative).
// Every other row takes scan_row's exact path (fma filter, division), so the
// bounds equal scan_row's.
__device__ __forceinline__ long long abs_bits(long long x) {
  long long r;
  asm("and.b64 %0, %1, 0x7FFFFFFFFFFFFFFF;" : "=l"(r) : "l"(x));
  return r;
}
// scan_row's exact test and division for one row, out of line: rows reach
// it rarely once the bounds have tightened, and sixteen inlined copies of the
// division sequence would bloat the epilogue's code
__device__ __noinline__ long long scan_exact_hi(double sl, double ad, long long hk) {
  const double hi = keyd(hk);
  if (!(fma(-hi, ad, sl) > 0.0)) {
    const double q = sl / ad;
    if (q < hi) return dkey(q);
  }
  return hk;
}
__device__ __noinline__ long long scan_exact_lo(double sl, double ad, long long lk) {
  const double lo = keyd(lk);
  if (!(fma(-lo, ad, sl) >= 0.0)) {
    const double q = sl / ad;
    if (q > lo) return dkey(q);
  }
  return lk;
}
__device__ __forceinline__ void scan_row_key(double sl, double ad, long long epsb, long long& hk,
                                             long long& lk, unsigned& sd) {
  constexpr long long kOne = 0x3FF0000000000000LL;        // B(1.0)
  constexpr long long kMargin = 0x0003333333333333LL;     // 0.2 in log2 units
  constexpr long long kInf = 0x7FF0000000000000LL;
  constexpr long long kMinNormal = 0x0010000000000000LL;  // B(DBL_MIN)
  const long long A = __double_as_longlong(ad), S = __double_as_longlong(sl);
  const long long Aabs = abs_bits(A);
  if (Aabs <= epsb) return;  // |ad| <= eps_dir: the row is skipped (chord_scan)
  if (A > 0) {
    sd |= 1u;
    // hk >= 0: hk is B(hi)
    if (S >= kMinNormal && hk >= 0 && hk < kInf && S - A > hk - kOne + kMargin) return;
    hk = scan_exact_hi(sl, ad, hk);
  } else {
    sd |= 2u;
    const long long L = abs_bits(lk < 0 ? ~lk : lk);  // B(|lo|)
    if (S >= kMinNormal && L < kInf && S - Aabs > L - kOne + kMargin) return;
    lk = scan_exact_lo(sl, ad, lk);
  }
}
// running max of -s as an order-preserving integer key (no fp64 instruction)
__device__ __forceinline__ void viol_key_update(long long& vk, double s) {
  const long long b = __double_as_longlong(s) ^ (long long)0x8000000000000000ULL;  // bits of -s
  const long long k = b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
  vk = k > vk ? k : vk;
}

// reduce_and_publish for bounds carried as keys (scan_row_key): integer
// min / max through the shuffles, no fp64 instruction.  One walk group.
__device__ __forceinline__ void reduce_and_publish_keys(long long (&hk)[2], long long (&lk)[2],
                                                        long long (&vk)[2], unsigned (&sd)[2],
                                                        int64_t c0, int lane,
                                                        const ChordParams& p) {
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      const long long h = __shfl_xor_sync(0xFFFFFFFFu, hk[e], off);
      const long long l = __shfl_xor_sync(0xFFFFFFFFu, lk[e], off);
      const long long v = __shfl_xor_sync(0xFFFFFFFFu, vk[e], off);
      hk[e] = h < hk[e] ? h : hk[e];
      lk[e] = l > lk[e] ? l : lk[e];
      vk[e] = v > vk[e] ? v : vk[e];
      sd[e] |= __shfl_xor_sync(0xFFFFFFFFu, sd[e], off);
    }
  if (lane < 4) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t c = c0 + 2 * lane + e;
      if (c >= p.z) continue;
      atomicMax(p.viol_key + c, vk[e]);
      atomicMin(p.hi_key + c, hk[e]);
      atomicMax(p.lo_key + c, lk[e]);
      if (sd[e]) atomicOr(p.sides + c, sd[e]);
    }
  }
}

// Warp reduction over the 8 row lanes sharing (lane & 3), then one atomic per
// walk from lanes 0..3.  c0 = the walk of (lane & 3) == 0, e = 0.
template <int NCH, bool BOUNDS>
__device__ __forceinline__ void reduce_and_publish(double (&hi)[NCH][2], double (&lo)[NCH][2],
                                                   double (&viol)[NCH][2], unsigned (&sd)[NCH][2],
                                                   const int64_t (&c0)[NCH], int lane,
                                                   const ChordParams& p) {
#pragma unroll
  for (int j = 0; j < NCH; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        if (BOUNDS) {
          hi[j][e] = fmin(hi[j][e], __shfl_xor_sync(0xFFFFFFFFu, hi[j][e], off));
          lo[j][e] = fmax(lo[j][e], __shfl_xor_sync(0xFFFFFFFFu, lo[j][e], off));
          sd[j][e] |= __shfl_xor_sync(0xFFFFFFFFu, sd[j][e], off);
        }
        viol[j][e] = fmax(viol[j][e], __shfl_xor_sync(0xFFFFFFFFu, viol[j][e], off));
      }
    }
  if (lane < 4) {
#pragma unroll
    for (int j = 0; j < NCH; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = c0[j] + 2 * lane + e;
        if (c >= p.z) continue;
        const long long vk = dkey(viol[j][e]);
#if MHAR_CHORD_RED
        // fire-and-forget reductions (RED): no round trip in the epilogue
        atomicMax(p.viol_key + c, vk);
        if (BOUNDS) {
          atomicMin(p.hi_key + c, dkey(hi[j][e]));
          atomicMax(p.lo_key + c, dkey(lo[j][e]));
          if (sd[j][e]) atomicOr(p.sides + c, sd[j][e]);
        }
#else
        if (vk > *(volatile long long*)(p.viol_key + c)) atomicMax(p.viol_key + c, vk);
        if (BOUNDS) {
          const long long hk = dkey(hi[j][e]), lk = dkey(lo[j][e]);
          if (hk < *(volatile long long*)(p.hi_key + c)) atomicMin(p.hi_key + c, hk);
          if (lk > *(volatile long long*)(p.lo_key + c)) atomicMax(p.lo_key + c, lk);
          if (sd[j][e] & ~*(volatile unsigned*)(p.sides + c)) atomicOr(p.sides + c, sd[j][e]);
        }
#endif
      }
  }
}

// ===========================================================================
// FUSED / FUSED_STORE: one CTA per SM, tile 128 rows x 64 walks x {x, d}.
// ===========================================================================
template <int MODE>
__global__ void __launch_bounds__(CHORD_THREADS, 1) chord_kernel(const ChordParams p) {
  if (*p.err != kNoError) return;  // sticky device error: stop all work
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)CHORD_STAGES * STAGE_DOUBLES * 8);
  uint64_t* empty = full + CHORD_STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile: 64 rows x (16 walks x {x, d})
  const int64_t n_units = p.m_tiles * p.col_tiles;
  const int my_units =
      (blockIdx.x < n_units) ? (int)((n_units - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int KT = (int)p.KT;

  if (tid == 0) {
    for (int s = 0; s < CHORD_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CHORD_THREADS / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // producer state (thread 0): the consumers' (unit, k-tile) sequence,
  // CHORD_STAGES - CHORD_LAG loads ahead.
  int l_ui = 0, l_kt = 0, l_stage = 0, l_round = 0;
  int64_t l_mt = 0, l_ct = 0;
  uint64_t keep_policy = 0;
  auto producer_issue = [&]() {
    if (l_ui >= my_units) return;
    if (l_round > 0) mbar_wait(&empty[l_stage], (uint32_t)((l_round - 1) & 1));
    double* st = ring + (size_t)l_stage * STAGE_DOUBLES;
    mbar_arrive_expect_tx(&full[l_stage], STAGE_DOUBLES * 8);
    bulk_g2s(st, p.A + (l_mt * p.KT + l_kt) * A_PIECE, A_PIECE * 8, &full[l_stage]);
    bulk_g2s_hint(st + A_PIECE, p.X + (l_ct * p.KT + l_kt) * B_PIECE, B_PIECE * 8,
                  &full[l_stage], keep_policy);
    bulk_g2s_hint(st + A_PIECE + B_PIECE, p.D + (l_ct * p.KT + l_kt) * B_PIECE, B_PIECE * 8,
                  &full[l_stage], keep_policy);
    if (++l_stage == CHORD_STAGES) {
      l_stage = 0;
      ++l_round;
    }
    if (++l_kt == KT) {
      l_kt = 0;
      if (++l_ui < my_units) unit_coords(blockIdx.x + (int64_t)l_ui * gridDim.x, p, &l_mt, &l_ct);
    }
  };
  if (tid == 0) {
    keep_policy = policy_evict_last();
    if (my_units > 0) unit_coords(blockIdx.x, p, &l_mt, &l_ct);
    for (int q = 0; q < CHORD_STAGES - CHORD_LAG; ++q) producer_issue();
  }

  int c_stage = 0, c_phase = 0;
  for (int ui = 0; ui < my_units; ++ui) {
    int64_t mt, ct;
    unit_coords(blockIdx.x + (int64_t)ui * gridDim.x, p, &mt, &ct);

    double acc[8][4][2];  // j = 0,1: A x columns; j = 2,3: A d columns (same walks)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
      if (tid == 0) producer_issue();
      mbar_wait(&full[c_stage], (uint32_t)c_phase);
      const double2* sa = reinterpret_cast<const double2*>(ring + (size_t)c_stage * STAGE_DOUBLES);
      const double2* sb = sa + A_PIECE / 2;
#pragma unroll
      for (int k8 = 0; k8 < 2; ++k8) {
        double2 af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = sa[(k8 * 16 + wm * 8 + i) * 32 + lane];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          bf[j] = sb[(j >> 1) * (B_PIECE / 2) + (k8 * 8 + wn * 2 + (j & 1)) * 32 + lane];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[c_stage]);
      if (++c_stage == CHORD_STAGES) {
        c_stage = 0;
        c_phase ^= 1;
      }
    }

    // ---------------- epilogue ----------------
    const int64_t row0 = mt * BM + wm * 64 + (lane >> 2);
    double hi[2][2], lo[2][2], viol[2][2];
    unsigned sd[2][2];
    int64_t c0[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      c0[j] = ct * 64 + wn * 16 + j * 8;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = c0[j] + 2 * (lane & 3) + e;
        hi[j][e] = keyd(*(volatile long long*)(p.hi_key + c));
        lo[j][e] = keyd(*(volatile long long*)(p.lo_key + c));
        viol[j][e] = __longlong_as_double((long long)0xFFF0000000000000ULL);  // -inf
        sd[j][e] = 0u;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t r = row0 + i * 8;
      const double br = __ldg(p.b + r);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double ax = acc[i][j][e], ad = acc[i][j + 2][e];
          const double sl = br - ax;  // (-ax).colwise() + b, sampler.cpp:175
          viol[j][e] = fmax(viol[j][e], ax - br);
          scan_row(sl, ad, p.eps_dir, hi[j][e], lo[j][e], sd[j][e]);
          if (MODE == FUSED_STORE) {
            const int64_t si = cache_index(r, c0[j] + 2 * (lane & 3) + e, p);
            if (p.rate_f32) {
              // the fp32 variant keeps its rates in fp32 and its slack as a
              // double-float pair (chord_tc32.cuh); +inf padding rows stay +inf
              const float h = (float)sl;
              const float l = isfinite(sl) ? (float)(sl - (double)h) : 0.0f;
              const float2 v = make_float2(h, l);
              p.S[si] = *reinterpret_cast<const double*>(&v);
              reinterpret_cast<float*>(p.R)[si] = (float)ad;
            } else {
              p.S[si] = sl;
              p.R[si] = ad;
            }
          }
        }
    }
    reduce_and_publish<2, true>(hi, lo, viol, sd, c0, lane, p);
  }
}

// ===========================================================================
// INCREMENTAL / CHECK: two CTAs per SM, tile 128 rows x 64 walks.
// ===========================================================================
// Units are handed out in order by a global ticket counter (p.sched) rather
// than statically (CTA b taking b, b + grid, ...): CTAs that drift apart over
// a few hundred units no longer spread the units in flight over many row
// bands, so the band's A_I tiles and the direction tiles stay L2-resident
// (DRAM traffic per launch was 70-150 GB against 29.5 GB algorithmic with
// the static order, and varied from run to run with the drift).  Thread 0
// draws the tickets as the producer and announces each unit (or the end,
// -1) to the CTA through a small queue of (unit, mbarrier) slots.
__device__ inline int64_t next_unit(const ChordParams& p, int64_t n_units) {
  const int64_t u = (int64_t)atomicAdd(p.sched, 1u);
  if (u < n_units) return u;
  // this CTA's last ticket; the last CTA to get here rewinds the counter for
  // the next launch (every other CTA has drawn its last ticket already)
  if (atomicAdd(p.sched + 1, 1u) == gridDim.x - 1) {
    p.sched[0] = 0u;
    p.sched[1] = 0u;
  }
  return -1;
}

template <int MODE>
__global__ void __launch_bounds__(CHORD_THREADS, 2) chord2_kernel(const ChordParams p) {
  if (*p.err != kNoError) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* full =
      reinterpret_cast<uint64_t*>(smem_raw + (size_t)CHORD2_STAGES * STAGE2_DOUBLES * 8);
  uint64_t* empty = full + CHORD2_STAGES;
  uint64_t* uready = empty + CHORD2_STAGES;  // [CHORD2_UQ] unit announced
  long long* uq = reinterpret_cast<long long*>(uready + CHORD2_UQ);  // [CHORD2_UQ] the units

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // warp tile: 32 rows x 32 walks
  const int64_t n_units = p.m_tiles * p.col_tiles;
  const int KT = (int)p.KT;
  const double* __restrict__ Bsrc = (MODE == INCREMENTAL) ? p.D : p.X;

  if (tid == 0) {
    for (int s = 0; s < CHORD2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CHORD_THREADS / 32);
    }
    for (int s = 0; s < CHORD2_UQ; ++s) mbar_init(&uready[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  // producer state (thread 0), kept in shared memory: in registers it would
  // be allocated in every thread and push the 128-register accumulator
  // tiles into spills
  struct Producer {
    const double* a;  // next A_I stage piece
    const double* b;  // next B stage piece
    int kt, stage, round, ann;
    long long unit;
  };
  __shared__ Producer pr;
  auto announce = [&](int64_t u) {  // unit u (or -1: no more) to the consumers
    uq[pr.ann % CHORD2_UQ] = u;
    mbar_arrive(&uready[pr.ann % CHORD2_UQ]);  // release: the uq write is visible
    ++pr.ann;
    pr.unit = u;
    if (u >= 0) {
      int64_t mt, ct;
      unit_coords(u, p, &mt, &ct);
      pr.a = p.A + mt * p.KT * A_PIECE;
      pr.b = Bsrc + ct * p.KT * B_PIECE;
    }
  };
  auto producer_issue = [&]() {
    if (pr.unit < 0) return;
    const int stage = pr.stage;
    if (pr.round > 0) mbar_wait(&empty[stage], (uint32_t)((pr.round - 1) & 1));
    double* st = ring + (size_t)stage * STAGE2_DOUBLES;
    mbar_arrive_expect_tx(&full[stage], STAGE2_DOUBLES * 8);
    bulk_g2s(st, pr.a, A_PIECE * 8, &full[stage]);
    bulk_g2s_hint(st + A_PIECE, pr.b, B_PIECE * 8, &full[stage],
                  MHAR_CHORD2_KEEP ? policy_evict_last() : policy_evict_normal());
    pr.a += A_PIECE;
    pr.b += B_PIECE;
    if (stage + 1 == CHORD2_STAGES) {
      pr.stage = 0;
      ++pr.round;
    } else {
      pr.stage = stage + 1;
    }
    if (++pr.kt == KT) {
      pr.kt = 0;
      announce(next_unit(p, n_units));
    }
  };
  if (tid == 0) {
    pr.kt = pr.stage = pr.round = pr.ann = 0;
    announce(next_unit(p, n_units));
    for (int q = 0; q < CHORD2_STAGES - CHORD2_LAG; ++q) producer_issue();
  }

  int c_stage = 0, c_phase = 0;
  for (int ui = 0;; ++ui) {
    mbar_wait(&uready[ui % CHORD2_UQ], (uint32_t)((ui / CHORD2_UQ) & 1));
    const int64_t u = uq[ui % CHORD2_UQ];
    if (u < 0) break;
    int64_t mt, ct;
    unit_coords(u, p, &mt, &ct);
    const int64_t cache_base = ((mt * p.col_tiles + ct) * 8 + warp) * S_WARP_BLOCK;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
      if (tid == 0) producer_issue();
      if (MHAR_CHORD2_PREFETCH && MODE == INCREMENTAL && kt == (KT > 8 ? KT - 8 : 0) && lane == 0) {
        // stage this warp's slack/rate block (2 x 8 KB) into L2 ahead of the epilogue
        bulk_prefetch_l2(p.S + cache_base, S_WARP_BLOCK * 8);
        bulk_prefetch_l2(p.R + cache_base, S_WARP_BLOCK * 8);
      }
      mbar_wait(&full[c_stage], (uint32_t)c_phase);
      const double2* sa =
          reinterpret_cast<const double2*>(ring + (size_t)c_stage * STAGE2_DOUBLES);
      const double2* sb = sa + A_PIECE / 2;
#pragma unroll
      for (int k8 = 0; k8 < 2; ++k8) {
        double2 af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = sa[(k8 * 16 + wm * 4 + i) * 32 + lane];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = sb[(k8 * 8 + wn * 4 + j) * 32 + lane];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[c_stage]);
      if (++c_stage == CHORD2_STAGES) {
        c_stage = 0;
        c_phase ^= 1;
      }
    }

    // ---------------- epilogue: one walk group (8 walks) at a time --------
    const int64_t row0 = mt * BM + wm * 32 + (lane >> 2);
    constexpr bool kBounds = (MODE == INCREMENTAL);
    double br[4];
    if (!kBounds) {
#pragma unroll
      for (int i = 0; i < 4; ++i) br[i] = __ldg(p.b + row0 + i * 8);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double hi[1][2], lo[1][2], viol[1][2];
      unsigned sd[1][2] = {{0u, 0u}};
      const int64_t c0[1] = {ct * 64 + wn * 32 + j * 8};
      const int64_t c = c0[0] + 2 * (lane & 3);
      viol[0][0] = viol[0][1] = __longlong_as_double((long long)0xFFF0000000000000ULL);
      if (kBounds) {
        const double2 th = *reinterpret_cast<const double2*>(p.theta_prev + c);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          hi[0][e] = keyd(*(volatile long long*)(p.hi_key + c + e));
          lo[0][e] = keyd(*(volatile long long*)(p.lo_key + c + e));
        }
        double2 so[4], ro[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t base = cache_base + ((i * 4 + j) * 32 + lane) * 2;
#if MHAR_CHORD2_STREAMING
          so[i] = __ldcs(reinterpret_cast<const double2*>(p.S + base));
          ro[i] = __ldcs(reinterpret_cast<const double2*>(p.R + base));
#else
          so[i] = __ldcg(reinterpret_cast<const double2*>(p.S + base));
          ro[i] = __ldcg(reinterpret_cast<const double2*>(p.R + base));
#endif
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t base = cache_base + ((i * 4 + j) * 32 + lane) * 2;
          const double s0 = fma(-th.x, ro[i].x, so[i].x);
          const double s1 = fma(-th.y, ro[i].y, so[i].y);
          __stcs(reinterpret_cast<double2*>(p.S + base), make_double2(s0, s1));
          __stcs(reinterpret_cast<double2*>(p.R + base), make_double2(acc[i][j][0], acc[i][j][1]));
          viol[0][0] = fmax(viol[0][0], -s0);
          viol[0][1] = fmax(viol[0][1], -s1);
          scan_row(s0, acc[i][j][0], p.eps_dir, hi[0][0], lo[0][0], sd[0][0]);
          scan_row(s1, acc[i][j][1], p.eps_dir, hi[0][1], lo[0][1], sd[0][1]);
        }
      } else if (MODE == SLACK_STORE) {
        // refresh of a tcgen05 engine's cache: the exact fp64 slack b - A x
        // in that engine's layout and format, rates zeroed (the engine's
        // next pass runs with theta_prev = 0 and writes them)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double sl = br[i] - acc[i][j][e];
            const int64_t si = cache_index(row0 + i * 8, c + e, p);
            if (p.rate_f32) {
              const float h = (float)sl;
              const float l = isfinite(sl) ? (float)(sl - (double)h) : 0.0f;
              const float2 v = make_float2(h, l);
              p.S[si] = *reinterpret_cast<const double*>(&v);
              reinterpret_cast<float*>(p.R)[si] = 0.0f;
            } else {
              p.S[si] = sl;
              p.R[si] = 0.0;
            }
          }
        continue;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int e = 0; e < 2; ++e) viol[0][e] = fmax(viol[0][e], acc[i][j][e] - br[i]);
      }
      reduce_and_publish<1, kBounds>(hi, lo, viol, sd, c0, lane, p);
    }
  }
}

}  // namespace mhar_dev
