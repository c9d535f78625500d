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
constexpr int kDiagUniMax = 2;      // blocks of the uniform instantiations

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
  // UNIFORM instantiations: every row of block j has coefficient uc[j] and
  // bound ub[j] (hypercube [I; -I] <= 1, simplex -I <= 0): no per-row loads
  double uc[kDiagUniMax], ub[kDiagUniMax];
};

// grid = (walk tiles of 64, coordinate splits); thread t owns packed element t
// of every piece (B_PIECE = 1024 = blockDim), i.e. one (walk, k-offset) slot,
// and walks its k tiles four at a time with all eight loads in flight.
// BLOCKS > 0: the block count known at compile time (1: simplex -I, 2: the
// hypercube's [I; -I]) so the row loop unrolls; 0: p.blocks at run time.
template <int BLOCKS, bool UNIFORM = false>
__global__ void __launch_bounds__(kDiagThreads) diag_chord_kernel(const DiagParams p) {
  pdl_enter();
  static_assert(!UNIFORM || (BLOCKS >= 1 && BLOCKS <= kDiagUniMax), "uniform blocks");
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
          const double cf = UNIFORM ? p.uc[bb] : __ldg(p.coef + r);
          const double bv = UNIFORM ? p.ub[bb] : __ldg(p.b + r);
          // -(x c) + b and d c, one rounding each (sampler.cpp:168-170; no FMA
          // contraction, so the bounds equal the one-term dot products')
          const double sl = __dsub_rn(bv, __dmul_rn(x[u], cf));
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

constexpr int kMaxFactorEq = 4;  // m_E bound of the factored projection

// ---------------------------------------------------------------------------
// Per-walk reductions over the packed layout at full HBM rate (round 2).  The
// round-1 warp-per-walk forms put z warps on a strided walk through each
// column: at z = 1000 that is ~7 warps per SM, latency bound (simplex
// n = 5000: 98 us for A_E H, 51 us for the collapse norms, 40 MB each).  Here a CTA owns one 64-walk tile and a fixed
// range of kDotKt k tiles (grid = walk tiles x J, J = ceil(KT / kDotKt));
// thread t owns packed element t of every piece, i.e. one (walk, k-offset)
// slot (the diag kernel's mapping), so every load is a coalesced piece.  The
// CTA reduces its 16 slots per walk in smem in a fixed order and writes one
// partial per (split, walk); the consumer sums the J partials in split order.
// The order depends on n alone: deterministic and independent of z, the
// grid and the sharding (walk c's result uses only walk c's data).
constexpr int kDotKt = 8;  // k tiles (128 coordinates) per CTA
__host__ __device__ inline int64_t dot_splits(int64_t KT) { return (KT + kDotKt - 1) / kDotKt; }

// slot of packed element t within a piece: walk wc (0..63), k offset kof (0..15)
__device__ __forceinline__ void piece_slot(int t, int* wc, int* kof) {
  *wc = ((t >> 6) & 7) * 8 + ((t >> 3) & 7);
  *kof = ((t >> 9) & 1) * 8 + (t & 1) * 4 + ((t >> 1) & 3);
}

// partial sums of NS values per walk, reduced over the CTA's 16 slots per
// walk in kof order: out[(j * NS + i) * z_pad + walk]
template <int NS>
__device__ __forceinline__ void cta_walk_reduce(double (&v)[NS], double (*red)[BC][BK], int wc,
                                                int kof, int64_t ct, int64_t j, int64_t z_pad,
                                                double* out) {
#pragma unroll
  for (int i = 0; i < NS; ++i) red[i][wc][kof] = v[i];
  __syncthreads();
  const int t = threadIdx.x;
  if (t < NS * BC) {
    const int i = t / BC, w = t % BC;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < BK; ++q) s += red[i][w][q];
    out[(j * NS + i) * z_pad + ct * BC + w] = s;
  }
}

// (1) r = A_E h per walk, split partials (m_E <= kMaxFactorEq; padded slots 0)
template <int ME>
__global__ void __launch_bounds__(B_PIECE) proj_dot_kernel(const double* __restrict__ AE,
                                                           const double* __restrict__ H,
                                                           int64_t n, int64_t KT, int64_t z_pad,
                                                           double* __restrict__ part,
                                                           const unsigned long long* err) {
  pdl_enter();
  if (*err != kNoError) return;
  __shared__ double red[ME][BC][BK];
  const int t = threadIdx.x;
  const int64_t ct = blockIdx.x, j = blockIdx.y;
  int wc, kof;
  piece_slot(t, &wc, &kof);
  double r[ME];
#pragma unroll
  for (int i = 0; i < ME; ++i) r[i] = 0.0;
  // all kDotKt loads in flight, then the sums in k order
  double h[kDotKt];
#pragma unroll
  for (int u = 0; u < kDotKt; ++u) {
    const int64_t kt = j * kDotKt + u, k = kt * BK + kof;
    h[u] = (kt < KT && k < n) ? H[(ct * KT + kt) * B_PIECE + t] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kDotKt; ++u) {
    const int64_t k = (j * kDotKt + u) * BK + kof;
    if (k < n) {
#pragma unroll
      for (int i = 0; i < ME; ++i) r[i] = fma(__ldg(AE + i + k * ME), h[u], r[i]);
    }
  }
  cta_walk_reduce<ME>(r, red, wc, kof, ct, j, z_pad, part);
}

// (2) d = h - A_E' g with g = G r (r summed over the splits in order), and the
// split partials of ||d||^2 for the collapse test
template <int ME>
__global__ void __launch_bounds__(B_PIECE, 2) proj_apply_kernel(
    const double* __restrict__ AE, const double* __restrict__ G, const double* __restrict__ H,
    double* __restrict__ D, const double* __restrict__ part, int64_t n, int64_t z, int64_t KT,
    int64_t z_pad, double* __restrict__ npart, const unsigned long long* err) {
  pdl_enter();
  if (*err != kNoError) return;
  __shared__ double red[ME][BK][BC];  // also the split sums: [i][split group][walk]
  __shared__ double sg[ME][BC];
  const int t = threadIdx.x;
  const int64_t ct = blockIdx.x, j = blockIdx.y;
  const int64_t J = dot_splits(KT);
  {
    // r = sum of the J split partials: thread (group q0, walk w) adds splits
    // q0, q0 + 16, ..., then walk w's 16 group sums in group order
    const int w = t % BC, q0 = t / BC;
#pragma unroll
    for (int i = 0; i < ME; ++i) {
      double s = 0.0;
      for (int64_t q = q0; q < J; q += BK) s += part[(q * ME + i) * z_pad + ct * BC + w];
      red[i][q0][w] = s;
    }
  }
  __syncthreads();
  if (t < BC) {
    double r[ME];
#pragma unroll
    for (int i = 0; i < ME; ++i) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < BK; ++q) s += red[i][q][t];
      r[i] = s;
    }
#pragma unroll
    for (int i = 0; i < ME; ++i) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < ME; ++q) s = fma(__ldg(G + i + q * ME), r[q], s);
      sg[i][t] = s;
    }
  }
  __syncthreads();
  int wc, kof;
  piece_slot(t, &wc, &kof);
  const bool live = ct * BC + wc < z;
  double nrm[1] = {0.0};
  double h[kDotKt];
#pragma unroll
  for (int u = 0; u < kDotKt; ++u) {
    const int64_t kt = j * kDotKt + u, k = kt * BK + kof;
    h[u] = (live && kt < KT && k < n) ? H[(ct * KT + kt) * B_PIECE + t] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kDotKt; ++u) {
    const int64_t kt = j * kDotKt + u, k = kt * BK + kof;
    if (kt >= KT) break;
    const int64_t e = (ct * KT + kt) * B_PIECE + t;
    if (!live || k >= n) {
      D[e] = 0.0;
      continue;
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ME; ++i) s = fma(__ldg(AE + i + k * ME), sg[i][wc], s);
    const double d = h[u] - s;
    D[e] = d;
    nrm[0] = fma(d, d, nrm[0]);
  }
  __shared__ double nred[1][BC][BK];
  cta_walk_reduce<1>(nrm, nred, wc, kof, ct, j, z_pad, npart);
}

// split partials of ||d||^2 from D (the dense-P path)
__global__ void __launch_bounds__(B_PIECE) norm_part_kernel(const double* __restrict__ D,
                                                            int64_t n, int64_t z, int64_t KT,
                                                            int64_t z_pad,
                                                            double* __restrict__ npart,
                                                            const unsigned long long* err) {
  pdl_enter();
  if (*err != kNoError) return;
  __shared__ double red[1][BC][BK];
  const int t = threadIdx.x;
  const int64_t ct = blockIdx.x, j = blockIdx.y;
  int wc, kof;
  piece_slot(t, &wc, &kof);
  double nrm[1] = {0.0};
  const bool live = ct * BC + wc < z;
  double d[kDotKt];
#pragma unroll
  for (int u = 0; u < kDotKt; ++u) {
    const int64_t kt = j * kDotKt + u, k = kt * BK + kof;
    d[u] = (live && kt < KT && k < n) ? D[(ct * KT + kt) * B_PIECE + t] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kDotKt; ++u) nrm[0] = fma(d[u], d[u], nrm[0]);
  cta_walk_reduce<1>(nrm, red, wc, kof, ct, j, z_pad, npart);
}

// ||d_c|| <= 1e-12 -> collapsed (sampler.cpp:247-249), from the split
// partials: one warp per walk, lane-strided over the splits, then a fixed
// shuffle tree (deterministic; the splits depend on n alone)
__global__ void collapse_final_kernel(const double* __restrict__ npart, int64_t J, int64_t z,
                                      int64_t z_pad, unsigned* __restrict__ collapsed,
                                      const unsigned long long* err) {
  pdl_enter();
  if (*err != kNoError) return;
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= z) return;
  double s = 0.0;
  for (int64_t q = lane; q < J; q += 32) s += npart[q * z_pad + c];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
  if (lane == 0) collapsed[c] = (sqrt(s) <= kNearZeroDirection) ? 1u : 0u;
}

}  // namespace mhar_dev
