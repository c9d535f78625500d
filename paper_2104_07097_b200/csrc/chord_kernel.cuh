// chord_kernel.cuh -- the fused fp64 tensor-core chord kernel.
//
// Restates, for all walks at once, compute_lambda_intervals
// (/root/reference/proj/src/sampler.cpp:150-208) with its per-walk
// chord_scan (src/vmath.hpp:83-155):
//
//   slack = b_I - A_I x,  rate = A_I d,
//   upper_k = min{ slack_i / rate_i : rate_i >  eps_dir }
//   lower_k = max{ slack_i / rate_i : rate_i < -eps_dir }
//
// as ONE persistent kernel: a DMMA.8x8x4 product over pre-permuted operand
// tiles streamed HBM -> smem by the TMA bulk-copy engine through an mbarrier
// ring, whose epilogue forms the ratios in registers and reduces them
// (registers -> warp shuffles -> one order-preserving int64 atomic per walk
// per warp).  The m_I x z products never reach HBM in the FUSED mode.
//
// Modes (template):
//   FUSED        B = [X | D] per 64-walk tile: both products, bounds, and
//                max_i (A x - b) (contains(), polytope.cpp:177-190) for free.
//   FUSED_STORE  FUSED + writes slack and rate into the incremental cache.
//   INCREMENTAL  B = D per 128-walk tile: only A_I D is multiplied; the slack
//                of the moved walks comes from the cache,
//                slack_t = slack_{t-1} - theta_{t-1} rate_{t-1}, which holds
//                because x_t = x_{t-1} + theta_{t-1} d_{t-1} (half the flops).
//   CHECK        B = X: max_i (A x - b) only (collection-time containment).
#pragma once

#include "common.cuh"

namespace mhar_dev {

enum ChordMode { FUSED = 0, FUSED_STORE = 1, INCREMENTAL = 2, CHECK = 3 };

constexpr int CHORD_THREADS = 256;  // 8 MMA warps: 2 (rows) x 4 (walk columns)
constexpr int CHORD_STAGES = 5;     // 5 x 32 KB ring
constexpr int CHORD_LAG = 2;        // refill the slot consumed two stages ago
constexpr int STAGE_DOUBLES = A_PIECE + 2 * B_PIECE;
constexpr size_t CHORD_SMEM = (size_t)CHORD_STAGES * STAGE_DOUBLES * sizeof(double) + 1024;

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
  int64_t col_tiles;  // FUSED*: 64-walk tiles; INCREMENTAL/CHECK: 128-walk tiles
  int64_t ct128;      // 128-walk tiles (slack cache geometry)
  int64_t z;          // live walks
  double eps_dir;
  int group_m;        // rasterisation band height (m tiles)
};

__device__ inline void unit_coords(int64_t u, const ChordParams& p, int64_t* mt, int64_t* ct) {
  const int64_t band_units = (int64_t)p.group_m * p.col_tiles;
  const int64_t band = u / band_units;
  const int64_t in_band = u % band_units;
  const int64_t start = band * p.group_m;
  const int64_t h = (p.m_tiles - start < p.group_m) ? p.m_tiles - start : p.group_m;
  *mt = start + in_band % h;
  *ct = in_band / h;
}

template <int MODE>
__global__ void __launch_bounds__(CHORD_THREADS, 1) chord_kernel(const ChordParams p) {
  if (*p.err != kNoError) return;  // sticky device error: stop all work
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)CHORD_STAGES * STAGE_DOUBLES * 8);
  uint64_t* empty = full + CHORD_STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t n_units = p.m_tiles * p.col_tiles;
  const int64_t my_units = (blockIdx.x < n_units) ? (n_units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total_loads = my_units * p.KT;

  if (tid == 0) {
    for (int s = 0; s < CHORD_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CHORD_THREADS / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // Producer (thread 0): issue the bulk copies for global load index q.
  auto issue = [&](int64_t q) {
    const int s = (int)(q % CHORD_STAGES);
    const int64_t ui = q / p.KT, kt = q % p.KT;
    const int64_t u = blockIdx.x + ui * gridDim.x;
    int64_t mt, ct;
    unit_coords(u, p, &mt, &ct);
    double* st = ring + (size_t)s * STAGE_DOUBLES;
    mbar_arrive_expect_tx(&full[s], STAGE_DOUBLES * 8);
    bulk_g2s(st, p.A + (mt * p.KT + kt) * A_PIECE, A_PIECE * 8, &full[s]);
    const double* b0;
    const double* b1;
    if (MODE == FUSED || MODE == FUSED_STORE) {
      b0 = p.X + (ct * p.KT + kt) * B_PIECE;
      b1 = p.D + (ct * p.KT + kt) * B_PIECE;
    } else {
      const double* src = (MODE == INCREMENTAL) ? p.D : p.X;
      b0 = src + ((2 * ct) * p.KT + kt) * B_PIECE;
      b1 = src + ((2 * ct + 1) * p.KT + kt) * B_PIECE;
    }
    bulk_g2s(st + A_PIECE, b0, B_PIECE * 8, &full[s]);
    bulk_g2s(st + A_PIECE + B_PIECE, b1, B_PIECE * 8, &full[s]);
  };

  if (tid == 0) {
    const int64_t pre = total_loads < (CHORD_STAGES - CHORD_LAG) ? total_loads
                                                                  : (CHORD_STAGES - CHORD_LAG);
    for (int64_t q = 0; q < pre; ++q) issue(q);
  }

  // B fragment source (piece, col_group) for this warp's 4 column groups.
  int bpiece[4], bcg[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (MODE == FUSED || MODE == FUSED_STORE) {
      bpiece[j] = j >> 1;          // j = 0,1: x columns; j = 2,3: d columns
      bcg[j] = wn * 2 + (j & 1);   // 16 walks per warp
    } else {
      bpiece[j] = wn >> 1;         // 32 walks per warp
      bcg[j] = (wn & 1) * 4 + j;
    }
  }

  int64_t q = 0;
  for (int64_t ui = 0; ui < my_units; ++ui) {
    const int64_t u = blockIdx.x + ui * gridDim.x;
    int64_t mt, ct;
    unit_coords(u, p, &mt, &ct);

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int64_t kt = 0; kt < p.KT; ++kt, ++q) {
      if (tid == 0) {
        const int64_t qn = q + (CHORD_STAGES - CHORD_LAG);
        if (qn < total_loads) {
          if (qn >= CHORD_STAGES) {
            const int64_t prev = qn - CHORD_STAGES;  // previous occupant of the slot
            mbar_wait(&empty[qn % CHORD_STAGES], (uint32_t)((prev / CHORD_STAGES) & 1));
          }
          issue(qn);
        }
      }
      const int s = (int)(q % CHORD_STAGES);
      mbar_wait(&full[s], (uint32_t)((q / CHORD_STAGES) & 1));
      const double2* sa = reinterpret_cast<const double2*>(ring + (size_t)s * STAGE_DOUBLES);
      const double2* sb = reinterpret_cast<const double2*>(ring + (size_t)s * STAGE_DOUBLES + A_PIECE);
#pragma unroll
      for (int k8 = 0; k8 < 2; ++k8) {
        double2 af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = sa[(k8 * 16 + wm * 8 + i) * 32 + lane];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          bf[j] = sb[bpiece[j] * (B_PIECE / 2) + (k8 * 8 + bcg[j]) * 32 + lane];
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
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---------------- epilogue: chord bounds for this tile ----------------
    const int64_t row0 = mt * BM + wm * 64 + (lane >> 2);
    constexpr int NCH = (MODE == FUSED || MODE == FUSED_STORE) ? 2 : 4;  // walk groups
    double hi[NCH][2], lo[NCH][2], viol[NCH][2];
    unsigned sd[NCH][2];
#pragma unroll
    for (int j = 0; j < NCH; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        hi[j][e] = __longlong_as_double(0x7FF0000000000000LL);   // +inf
        lo[j][e] = __longlong_as_double((long long)0xFFF0000000000000ULL);  // -inf
        viol[j][e] = lo[j][e];
        sd[j][e] = 0u;
      }
    double thp[NCH][2];
    if (MODE == INCREMENTAL) {
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int64_t c = ct * 128 + wn * 32 + j * 8 + 2 * (lane & 3);
        const double2 t = *reinterpret_cast<const double2*>(p.theta_prev + c);
        thp[j][0] = t.x;
        thp[j][1] = t.y;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t r = row0 + i * 8;
      const double br = __ldg(p.b + r);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        double ax[2], ad[2], sl[2];
        if (MODE == FUSED || MODE == FUSED_STORE) {
          ax[0] = acc[i][j][0]; ax[1] = acc[i][j][1];
          ad[0] = acc[i][j + 2][0]; ad[1] = acc[i][j + 2][1];
          sl[0] = br - ax[0]; sl[1] = br - ax[1];  // (-ax).colwise() + b, sampler.cpp:175
        } else if (MODE == INCREMENTAL) {
          ad[0] = acc[i][j][0]; ad[1] = acc[i][j][1];
          const int64_t base =
              (((((mt * p.ct128 + ct) * 8 + warp) * 8 + i) * 4 + j) * 32 + lane) * 2;
          const double2 so = __ldcs(reinterpret_cast<const double2*>(p.S + base));
          const double2 ro = __ldcs(reinterpret_cast<const double2*>(p.R + base));
          sl[0] = fma(-thp[j][0], ro.x, so.x);
          sl[1] = fma(-thp[j][1], ro.y, so.y);
          __stcs(reinterpret_cast<double2*>(p.S + base), make_double2(sl[0], sl[1]));
          __stcs(reinterpret_cast<double2*>(p.R + base), make_double2(ad[0], ad[1]));
          ax[0] = -sl[0]; ax[1] = -sl[1];
        } else {  // CHECK
          ax[0] = acc[i][j][0]; ax[1] = acc[i][j][1];
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double v = (MODE == INCREMENTAL) ? ax[e] : ax[e] - br;
          viol[j][e] = fmax(viol[j][e], v);
          if (MODE != CHECK) {
            if (ad[e] > p.eps_dir) {
              const double qv = sl[e] / ad[e];
              sd[j][e] |= 1u;
              hi[j][e] = qv < hi[j][e] ? qv : hi[j][e];
            } else if (ad[e] < -p.eps_dir) {
              const double qv = sl[e] / ad[e];
              sd[j][e] |= 2u;
              lo[j][e] = qv > lo[j][e] ? qv : lo[j][e];
            }
          }
        }
        if (MODE == FUSED_STORE) {
          const int64_t c = ct * 64 + wn * 16 + j * 8 + 2 * (lane & 3);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t si = s_index(r, c + e, p.ct128);
            p.S[si] = sl[e];
            p.R[si] = ad[e];
          }
        }
      }
    }
    // reduce over the 8 row lanes sharing (lane & 3)
#pragma unroll
    for (int j = 0; j < NCH; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          hi[j][e] = fmin(hi[j][e], __shfl_xor_sync(0xFFFFFFFFu, hi[j][e], off));
          lo[j][e] = fmax(lo[j][e], __shfl_xor_sync(0xFFFFFFFFu, lo[j][e], off));
          viol[j][e] = fmax(viol[j][e], __shfl_xor_sync(0xFFFFFFFFu, viol[j][e], off));
          sd[j][e] |= __shfl_xor_sync(0xFFFFFFFFu, sd[j][e], off);
        }
      }
    if (lane < 4) {
#pragma unroll
      for (int j = 0; j < NCH; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = (MODE == FUSED || MODE == FUSED_STORE)
                                ? ct * 64 + wn * 16 + j * 8 + 2 * lane + e
                                : ct * 128 + wn * 32 + j * 8 + 2 * lane + e;
          if (c >= p.z) continue;
          const long long vk = dkey(viol[j][e]);
          if (vk > *(volatile long long*)(p.viol_key + c)) atomicMax(p.viol_key + c, vk);
          if (MODE != CHECK) {
            const long long hk = dkey(hi[j][e]), lk = dkey(lo[j][e]);
            if (hk < *(volatile long long*)(p.hi_key + c)) atomicMin(p.hi_key + c, hk);
            if (lk > *(volatile long long*)(p.lo_key + c)) atomicMax(p.lo_key + c, lk);
            if (sd[j][e] & ~*(volatile unsigned*)(p.sides + c)) atomicOr(p.sides + c, sd[j][e]);
          }
        }
    }
  }
}

}  // namespace mhar_dev
