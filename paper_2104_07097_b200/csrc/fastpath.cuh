// fastpath.cuh -- structure-aware paths for the bodies of the paper's own
// benchmark (hypercubes, simplices) at sizes beyond the walk-resident kernel.
//
// (1) Stacked diagonal blocks.  The reference's compute_lambda_intervals
//     detects an A_I made of k diagonal blocks -- every row's single nonzero
//     at column row % n, the shape of axis-aligned bound rows -- and fills
//     slack and rate elementwise (/root/reference/proj/src/sampler.cpp:47-71,
//     :166-172): slack = b - x c, rate = d c, each one rounding, exactly what
//     the one-term dot product gives.  diag_chord_kernel does that fill and the
//     chord scan of chord_kernel<FUSED> in one pass over X and D (HBM-bound,
//     O(m z) instead of O(m n z)) with bit-identical bounds.
// (2) Factored projection.  D = P H with P = I - A_E' G A_E
//     (sampler.cpp:246, projection.cpp:36-51) is formed as H - A_E' (G (A_E H))
//     when m_E is small: O(m_E n z) instead of the dense O(n^2 z) product
//     (equal to P H up to rounding; the parity tests' 1e-9 bar).
#pragma once

#include "chord_kernel.cuh"
#include "common.cuh"

namespace mhar_dev {

constexpr int kDiagThreads = 1024;  // = B_PIECE: one packed element per thread

struct DiagParams {
  const double* coef;  // m per-row coefficients (row r: column r % n)
  const double* b;     // b_I
  const double* X;     // packed state (b_index)
  const double* D;     // packed directions (b_index)
  long long* hi_key;
  long long* lo_key;
  long long* viol_key;
  unsigned* sides;
  const unsigned long long* err;
  int64_t n, blocks, KT, z;
  int64_t kt_per_cta;  // k tiles per CTA (grid.y splits the coordinates)
  double eps_dir;
  int bounds;          // 0: containment only (max_i (A x - b)_i)
};

// grid = (walk tiles of 64, coordinate splits); thread t owns packed element t
// of every piece (B_PIECE = 1024 = blockDim), i.e. one (walk, k-offset) slot,
// and walks its k tiles four at a time with all eight loads in flight.
// BLOCKS > 0: the block count known at compile time (1: simplex -I, 2: the
// hypercube's [I; -I]) so the row loop unrolls; 0: p.blocks at run time.
template <int BLOCKS>
__global__ void __launch_bounds__(kDiagThreads) diag_chord_kernel(const DiagParams p) {
  if (*p.err != kNoError) return;
  __shared__ long long s_hi[BC], s_lo[BC], s_viol[BC];
  __shared__ unsigned s_sd[BC];
  const int tid = threadIdx.x;
  const int64_t ct = blockIdx.x;
  if (tid < BC) {
    s_hi[tid] = dkey(__longlong_as_double(0x7FF0000000000000LL));
    s_lo[tid] = dkey(__longlong_as_double((long long)0xFFF0000000000000ULL));
    s_viol[tid] = s_lo[tid];
    s_sd[tid] = 0u;
  }
  __syncthreads();
  const int64_t kt0 = blockIdx.y * p.kt_per_cta;
  const int64_t kt1 = kt0 + p.kt_per_cta < p.KT ? kt0 + p.kt_per_cta : p.KT;
  const double* Xt = p.X + ct * p.KT * B_PIECE + tid;
  const double* Dt = p.D + ct * p.KT * B_PIECE + tid;
  int64_t wc, kof;
  b_coords(tid, p.KT, &wc, &kof);  // within the first piece of tile 0
  double ehi = __longlong_as_double(0x7FF0000000000000LL), elo = -ehi;
  double viol = __longlong_as_double((long long)0xFFF0000000000000ULL);
  unsigned sd = 0u;
  // 32-bit coordinate / row arithmetic (m = blocks n < 2^31)
  const int n32 = (int)p.n, nblk = BLOCKS > 0 ? BLOCKS : (int)p.blocks;
  const int kof32 = (int)kof;
  for (int kt = (int)kt0; kt < (int)kt1; kt += 4) {
    double x[4], d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = (kt + u) * BK + kof32;
      const bool live = kt + u < (int)kt1 && k < n32;
      x[u] = live ? Xt[(int64_t)(kt + u) * B_PIECE] : 0.0;
      d[u] = live ? Dt[(int64_t)(kt + u) * B_PIECE] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = (kt + u) * BK + kof32;
      if (kt + u >= (int)kt1 || k >= n32) continue;
#pragma unroll
      for (int blk = 0; blk < (BLOCKS > 0 ? BLOCKS : 1); ++blk) {
        for (int bb = blk; bb < (BLOCKS > 0 ? blk + 1 : nblk); ++bb) {
          const int r = bb * n32 + k;
          const double cf = __ldg(p.coef + r);
          // -(x c) + b and d c, one rounding each (sampler.cpp:168-170; no FMA
          // contraction, so the bounds equal the one-term dot products')
          const double sl = __dsub_rn(__ldg(p.b + r), __dmul_rn(x[u], cf));
          viol = fmax(viol, -sl);
          if (p.bounds) scan_row(sl, __dmul_rn(d[u], cf), p.eps_dir, ehi, elo, sd);
        }
      }
    }
  }
  const int wl = (int)wc;
  const long long vk = dkey(viol);
  if (vk > s_viol[wl]) atomicMax(&s_viol[wl], vk);
  if (p.bounds) {
    const long long hk = dkey(ehi), lk = dkey(elo);
    if (hk < s_hi[wl]) atomicMin(&s_hi[wl], hk);
    if (lk > s_lo[wl]) atomicMax(&s_lo[wl], lk);
    if (sd) atomicOr(&s_sd[wl], sd);
  }
  __syncthreads();
  if (tid < BC) {
    const int64_t c = ct * BC + tid;
    if (c < p.z) {
      atomicMax(p.viol_key + c, s_viol[tid]);
      if (p.bounds) {
        atomicMin(p.hi_key + c, s_hi[tid]);
        atomicMax(p.lo_key + c, s_lo[tid]);
        if (s_sd[tid]) atomicOr(p.sides + c, s_sd[tid]);
      }
    }
  }
}

// Factored projection, step 1 (one warp per walk): g_c = G (A_E h_c), m_E <= kMaxFactorEq.
constexpr int kMaxFactorEq = 4;
__global__ void proj_factor_kernel(const double* __restrict__ AE /*me x n col-major*/,
                                   const double* __restrict__ G /*me x me*/,
                                   const double* __restrict__ H, int64_t me, int64_t n,
                                   int64_t z, int64_t KT, double* __restrict__ g /*me x z*/,
                                   const unsigned long long* err) {
  if (*err != kNoError) return;
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= z) return;
  double r[kMaxFactorEq] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
  for (int64_t k = lane; k < n; k += 32) {
    const double h = H[b_index(c, k, KT)];
#pragma unroll
    for (int i = 0; i < kMaxFactorEq; ++i)
      if (i < me) r[i] = fma(AE[i + k * me], h, r[i]);
  }
#pragma unroll
  for (int i = 0; i < kMaxFactorEq; ++i)
    for (int off = 16; off > 0; off >>= 1) r[i] += __shfl_xor_sync(0xFFFFFFFFu, r[i], off);
  if (lane < me) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kMaxFactorEq; ++j)
      if (j < me) s = fma(G[lane + j * me], r[j], s);
    g[lane + c * me] = s;
  }
}

// Factored projection, step 2 (thread per packed element): d = h - A_E' g_c.
__global__ void proj_correct_kernel(const double* __restrict__ AE, const double* __restrict__ g,
                                    const double* __restrict__ H, double* __restrict__ D,
                                    int64_t me, int64_t n, int64_t z, int64_t total,
                                    int64_t KT, const unsigned long long* err) {
  if (*err != kNoError) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, k;
    b_coords(e, KT, &c, &k);
    if (c >= z || k >= n) {
      D[e] = 0.0;
      continue;
    }
    double s = 0.0;
    for (int64_t i = 0; i < me; ++i) s = fma(AE[i + k * me], g[i + c * me], s);
    D[e] = H[e] - s;
  }
}

}  // namespace mhar_dev
