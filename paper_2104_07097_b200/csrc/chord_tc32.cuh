// chord_tc32.cuh -- fp32 variant of the incremental chord kernel on the
// Blackwell 5th-gen tensor cores (tcgen05.mma kind::tf32, TMEM accumulators).
//
// Same computation as chord2_kernel<INCREMENTAL> (compute_lambda_intervals,
// /root/reference/proj/src/sampler.cpp:150-208, with the slack carried
// incrementally), but the rates A_I d are formed in fp32 accuracy with the
// split  a d = a_hi d + a_lo d  (a_hi = tf32(a), a_lo = tf32(a - a_hi); the
// direction d itself is rounded to TF32, which keeps it centrally symmetric
// -- tf32(-d) = -tf32(d) -- so hit-and-run's uniform law is unchanged) on
// tcgen05, accumulating in fp32 in TMEM.  The
// slack cache and the walk state stay fp64.  To keep every emitted sample
// exactly feasible despite fp32 rates, chords are taken in the body shrunk
// by a margin mu (slack - mu), see DESIGN.md "fp32 variant".
//
// Tile: M = 128 walks (TMEM lanes) x N = 256 inequality rows (TMEM
// columns), K step 16 per stage.  With walks on the lanes each epilogue
// thread owns ONE walk and reduces its 256 rows in registers -- no shuffles.
//
// Warp roles (192 threads): warp 0 lane 0 = bulk-copy producer, warp 1 lane
// 0 = MMA issuer (+ TMEM allocation), warps 2..5 = epilogue (TMEM lane
// quarter = warp % 4).  The 512-column TMEM holds two 256-column
// accumulators so the epilogue of one tile overlaps the MMAs of the next.
#pragma once

#include "chord_kernel.cuh"
#include "common.cuh"

namespace mhar_dev {

constexpr int TC_M = 128;             // walks per tile
constexpr int TC_N = 256;             // rows per tile
constexpr int TC_BK = 16;             // k per stage
constexpr int TC_STAGES = 5;
constexpr int TC_D_PIECE = TC_M * TC_BK;   // floats per D stage piece (8 KB)
constexpr int TC_A_PIECE = TC_N * TC_BK;   // floats per A_hi (or A_lo) stage piece (16 KB)
constexpr int TC_STAGE_FLOATS = TC_D_PIECE + 2 * TC_A_PIECE;  // 40 KB
constexpr int TC_THREADS = 192;
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_FLOATS * 4 + 256;

// Interleaved K-major ("no swizzle") core-matrix layout of one (tile, k_tile)
// piece of R rows: [k_chunk(4 floats)][row_group(8 rows)][row(8)][4].
__host__ __device__ inline int64_t tc_piece_index(int64_t r, int64_t kk, int64_t R) {
  return ((kk >> 2) * (R >> 3) + (r >> 3)) * 32 + (r & 7) * 4 + (kk & 3);
}
// (walk c, coordinate k) in the packed TF32 direction array.
__host__ __device__ inline int64_t tc_d_index(int64_t c, int64_t k, int64_t KT) {
  return ((c / TC_M) * KT + k / TC_BK) * TC_D_PIECE + tc_piece_index(c % TC_M, k % TC_BK, TC_M);
}
// (row r, coordinate k) in the packed fp32 A_hi / A_lo arrays.
__host__ __device__ inline int64_t tc_a_index(int64_t r, int64_t k, int64_t KT) {
  return ((r / TC_N) * KT + k / TC_BK) * TC_A_PIECE + tc_piece_index(r % TC_N, k % TC_BK, TC_N);
}
// slack / rate cache for the tc32 tile: [row_tile][walk_tile][row(256)][walk(128)]
__host__ __device__ inline int64_t tc_s_index(int64_t r, int64_t c, int64_t WT) {
  return (((r / TC_N) * WT + c / TC_M) * TC_N + r % TC_N) * TC_M + c % TC_M;
}

__device__ inline float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, version 1.
__device__ inline uint64_t umma_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// instruction descriptor: F32 accumulate, A/B TF32, K-major, M = 128, N = 256
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)(TC_M >> 4) << 24);

__device__ inline void tc_mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(TC_IDESC), "r"(accumulate));
}
__device__ inline void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ inline void tc_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcParams {
  const float* Ahi;  // tc_a_index layout
  const float* Alo;
  const float* Dhi;  // tc_d_index layout, TF32-exact directions
  double* S;         // tc_s_index layout, fp64 slack
  double* R;         // fp64 rates of the previous iterate
  const double* theta_prev;
  long long* hi_key;
  long long* lo_key;
  long long* viol_key;
  unsigned* sides;
  const unsigned long long* err;
  int64_t row_tiles;   // m_pad / 256
  int64_t walk_tiles;  // z_pad / 128
  int64_t KT;          // n_pad / 16
  int64_t m;           // live rows
  int64_t z;           // live walks
  double eps_dir;
  double margin;       // mu: chords of {A x <= b - mu}
  int group_n;         // rasterisation band (row tiles)
};

__device__ inline void tc_unit(int64_t u, const TcParams& p, int64_t* rt, int64_t* wt) {
  const int64_t band_units = (int64_t)p.group_n * p.walk_tiles;
  const int64_t band = u / band_units;
  const int64_t in_band = u - band * band_units;
  const int64_t start = band * p.group_n;
  const int64_t h = (p.row_tiles - start < p.group_n) ? p.row_tiles - start : p.group_n;
  *rt = start + in_band % h;
  *wt = in_band / h;
}

__global__ void __launch_bounds__(TC_THREADS, 1) chord_tc32_kernel(const TcParams p) {
  if (*p.err != kNoError) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)TC_STAGES * TC_STAGE_FLOATS * 4);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained
  uint32_t* tptr = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_units = p.row_tiles * p.walk_tiles;
  const int my_units =
      (blockIdx.x < n_units) ? (int)((n_units - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int KT = (int)p.KT;

  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tptr)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tptr;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      uint64_t keep = policy_evict_last();
      int stage = 0, round = 0;
      for (int ui = 0; ui < my_units; ++ui) {
        int64_t rt, wt;
        tc_unit(blockIdx.x + (int64_t)ui * gridDim.x, p, &rt, &wt);
        for (int kt = 0; kt < KT; ++kt) {
          if (round > 0) mbar_wait(&empty[stage], (uint32_t)((round - 1) & 1));
          float* st = ring + (size_t)stage * TC_STAGE_FLOATS;
          mbar_arrive_expect_tx(&full[stage], TC_STAGE_FLOATS * 4);
          const int64_t doff = (wt * p.KT + kt) * TC_D_PIECE;
          const int64_t aoff = (rt * p.KT + kt) * TC_A_PIECE;
          bulk_g2s_hint(st, p.Dhi + doff, TC_D_PIECE * 4, &full[stage], keep);
          bulk_g2s_hint(st + TC_D_PIECE, p.Ahi + aoff, TC_A_PIECE * 4, &full[stage], keep);
          bulk_g2s_hint(st + TC_D_PIECE + TC_A_PIECE, p.Alo + aoff, TC_A_PIECE * 4, &full[stage],
                        keep);
          if (++stage == TC_STAGES) {
            stage = 0;
            ++round;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int stage = 0, phase = 0;
      for (int ui = 0; ui < my_units; ++ui) {
        const int ab = ui & 1;
        if (ui >= 2) mbar_wait(&tempty[ab], (uint32_t)(((ui >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + (uint32_t)(ab * TC_N);
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&full[stage], (uint32_t)phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const float* sd = ring + (size_t)stage * TC_STAGE_FLOATS;
          const float* sa_hi = sd + TC_D_PIECE;
          const float* sa_lo = sa_hi + TC_A_PIECE;
#pragma unroll
          for (int k = 0; k < TC_BK / 8; ++k) {
            // K step k: k-chunks 2k, 2k+1; LBO = stride between k-chunks
            const uint32_t dofs = 2 * k * (TC_M * 4), aofs = 2 * k * (TC_N * 4);
            const uint64_t dd = umma_desc(sd + dofs, TC_M * 16, 128);
            const uint64_t ah = umma_desc(sa_hi + aofs, TC_N * 16, 128);
            const uint64_t al = umma_desc(sa_lo + aofs, TC_N * 16, 128);
            tc_mma(acc, dd, ah, (kt | k) ? 1u : 0u);
            tc_mma(acc, dd, al, 1u);
          }
          tc_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[ab]);
      }
    }
  } else {
    // ---------------- epilogue: thread = walk ----------------
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int wl = q * 32 + lane;        // walk within the tile
    const uint64_t stream_policy = policy_evict_first();  // the slack stream must not evict A
    for (int ui = 0; ui < my_units; ++ui) {
      int64_t rt, wt;
      tc_unit(blockIdx.x + (int64_t)ui * gridDim.x, p, &rt, &wt);
      const int ab = ui & 1;
      mbar_wait(&tfull[ab], (uint32_t)((ui >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int64_t c = wt * TC_M + wl;
      const double th = p.theta_prev[c];
      double hi = keyd(*(volatile long long*)(p.hi_key + c));
      double lo = keyd(*(volatile long long*)(p.lo_key + c));
      double viol = __longlong_as_double((long long)0xFFF0000000000000ULL);
      unsigned sd = 0u;
      const int64_t sbase = (rt * p.walk_tiles + wt) * TC_N * TC_M + wl;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * TC_N);
      const double* __restrict__ Sin = p.S + sbase;
      const double* __restrict__ Rin = p.R + sbase;
      double* __restrict__ Sout = p.S + sbase;
      double* __restrict__ Rout = p.R + sbase;
      // 16 rows at a time: all loads of the group in flight before any store
      // (the cache is read and rewritten in place; interleaving them would
      // cost one DRAM latency per row)
      auto rows16 = [&](int r0, const float* vv) {
        double so[16], ro[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          so[j] = ld_policy(Sin + (int64_t)(r0 + j) * TC_M, stream_policy);
          ro[j] = ld_policy(Rin + (int64_t)(r0 + j) * TC_M, stream_policy);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double ad = (double)vv[j];
          const double s = fma(-th, ro[j], so[j]);
          st_policy(Sout + (int64_t)(r0 + j) * TC_M, s, stream_policy);
          st_policy(Rout + (int64_t)(r0 + j) * TC_M, ad, stream_policy);
          viol = fmax(viol, -s);
          scan_row(s - p.margin, ad, p.eps_dir, hi, lo, sd);
        }
      };
      for (int c0 = 0; c0 < TC_N; c0 += 32) {
        float v[32];
        tc_ld32(taddr + (uint32_t)c0, v);
        rows16(c0, v);
        rows16(c0 + 16, v + 16);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      if (c < p.z) {
        const long long vk = dkey(viol), hk = dkey(hi), lk = dkey(lo);
        if (vk > *(volatile long long*)(p.viol_key + c)) atomicMax(p.viol_key + c, vk);
        if (hk < *(volatile long long*)(p.hi_key + c)) atomicMin(p.hi_key + c, hk);
        if (lk > *(volatile long long*)(p.lo_key + c)) atomicMax(p.lo_key + c, lk);
        if (sd & ~*(volatile unsigned*)(p.sides + c)) atomicOr(p.sides + c, sd);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// fp64 polytope rows -> (A_hi, A_lo) with A_used = A_hi + A_lo written back
// into the packed fp64 A (the fp32 variant's body is A rounded to fp32).
__global__ void tc_split_a_kernel(const double* __restrict__ Acm, int64_t m, int64_t n,
                                  int64_t m_pad, int64_t KT, float* __restrict__ Ahi,
                                  float* __restrict__ Alo, double* __restrict__ Apk,
                                  int64_t KT64) {
  const int64_t total = m_pad * KT * TC_BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (KT * TC_BK), k = i % (KT * TC_BK);
    const float a = (r < m && k < n) ? (float)Acm[r + k * m] : 0.0f;
    const float h = tf32_trunc(a);
    const float l = tf32_trunc(a - h);
    const int64_t ti = tc_a_index(r, k, KT);
    Ahi[ti] = h;
    Alo[ti] = l;
    if (r < m && k < n) Apk[a_index(r, k, KT64)] = (double)h + (double)l;
  }
}

// fp64 directions (packed b_index) -> TF32-exact directions; D is replaced
// by them so the walk moves along exactly the direction the tensor cores see.
__global__ void tc_split_d_kernel(double* __restrict__ D, int64_t n, int64_t z_pad, int64_t KT,
                                  float* __restrict__ Dhi, const unsigned long long* err) {
  if (*err != kNoError) return;
  const int64_t total = z_pad * KT * BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, k;
    b_coords(i, KT, &c, &k);
    const float h = tf32_trunc((float)D[i]);
    Dhi[tc_d_index(c, k, KT)] = h;
    D[i] = (double)h;
  }
}

}  // namespace mhar_dev
