// chord_tc32.cuh -- fp32 variant of the incremental chord kernel on the
// Blackwell 5th-gen tensor cores (tcgen05.mma, TMEM accumulators).  Two forms
// share the kernel: kind::f16 with per-row / per-walk power-of-two scales
// (default; template F16, see tc_mma2_f16) and kind::tf32 (MHAR_TC_F16=0),
// described below.
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
// CTA pair (cluster of 2, tcgen05 cta_group::2): one MMA is M = 256 walks
// (128 per CTA, on each CTA's TMEM lanes) x N = 256 inequality rows, K step
// 16 per stage.  Each CTA stages its own 128 walks of D and ONE HALF (128
// rows) of the row tile's A_hi / A_lo, so per SM a stage is 24 KB for the
// work a single-CTA M = 128 x N = 256 tile needed 40 KB for -- the kernel is
// bounded by L2 -> SM bandwidth, not by the tensor pipe.  Both CTAs' TMEM
// hold all 256 rows for their own walks, so each epilogue thread still owns
// one walk and reduces its 256 rows in registers.
//
// Warp roles (320 threads per CTA): warp 0 lane 0 = bulk-copy producer (its
// CTA's pieces); warp 1 = TMEM allocation (both CTAs), lane 0 = MMA issuer
// in the even CTA and the "stage landed" relay in the odd one (waits its
// CTA's full barrier, arrives remotely on the leader's peer barrier); warps
// 2..9 = epilogue (TMEM lane quarter = warp % 4, two warps per quarter
// splitting the rows).  Two 256-column
// accumulators (512 TMEM columns) let the epilogue of one unit overlap the
// MMAs of the next.
#pragma once

#include <cuda.h>  // CUtensorMap
#include <cuda_fp16.h>

#include "chord_kernel.cuh"
#include "common.cuh"

namespace mhar_dev {

constexpr int TC_M = 128;             // walks per CTA (per unit: 2 x 128)
constexpr int TC_N = 256;             // rows per unit
constexpr int TC_NH = 128;            // rows staged by each CTA of the pair
constexpr int TC_BK = 16;             // k per stage
#ifndef MHAR_TC_STAGES
#define MHAR_TC_STAGES 8
#endif
constexpr int TC_STAGES = MHAR_TC_STAGES;
constexpr int TC_D_PIECE = TC_M * TC_BK;   // floats per D stage piece (8 KB)
constexpr int TC_A_PIECE = TC_NH * TC_BK;  // floats per A_hi (or A_lo) half piece (8 KB)
constexpr int TC_STAGE_FLOATS = TC_D_PIECE + 2 * TC_A_PIECE;  // 24 KB
constexpr int TC_EPI_WARPS = 8;       // two per TMEM lane quarter, each owns half the rows
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;
#ifndef MHAR_TC_EPI_ROWS
#define MHAR_TC_EPI_ROWS 16
#endif
#ifndef MHAR_TC_PREFETCH
#define MHAR_TC_PREFETCH 0
#endif
constexpr int TC_GROUP = MHAR_TC_EPI_ROWS;  // epilogue rows per load group
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_FLOATS * 4 + 512;
// Bodies with equalities: the direction P h must stay in the null space of
// A_E, so it is not rounded to TF32; it is split d = d_hi + d_lo instead and
// the rates take three MMAs (A_hi d_hi + A_lo d_hi + A_hi d_lo).  A stage then
// also carries d_lo (32 KB), six stages.
template <bool SPLIT_D> struct TcCfg {
  static constexpr int stages = SPLIT_D ? 6 : TC_STAGES;
  static constexpr int stage_floats = TC_STAGE_FLOATS + (SPLIT_D ? TC_D_PIECE : 0);
  static constexpr size_t smem = (size_t)stages * stage_floats * 4 + 512;
};

// Interleaved K-major ("no swizzle") core-matrix layout of one (tile, k_tile)
// piece of R rows: [k_chunk(4 floats)][row_group(8 rows)][row(8)][4].
__host__ __device__ inline int64_t tc_piece_index(int64_t r, int64_t kk, int64_t R) {
  return ((kk >> 2) * (R >> 3) + (r >> 3)) * 32 + (r & 7) * 4 + (kk & 3);
}
// (walk c, coordinate k) in the packed TF32 direction array: [walk_tile(128)][k_tile][piece].
__host__ __device__ inline int64_t tc_d_index(int64_t c, int64_t k, int64_t KT) {
  return ((c / TC_M) * KT + k / TC_BK) * TC_D_PIECE + tc_piece_index(c % TC_M, k % TC_BK, TC_M);
}
// (row r, coordinate k) in the packed fp32 A_hi / A_lo arrays:
// [row_tile(256)][k_tile][half(128 rows)][piece] -- CTA h of a pair loads half h.
__host__ __device__ inline int64_t tc_a_index(int64_t r, int64_t k, int64_t KT) {
  return (((r / TC_N) * KT + k / TC_BK) * 2 + (r % TC_N) / TC_NH) * TC_A_PIECE +
         tc_piece_index(r % TC_NH, k % TC_BK, TC_NH);
}
// slack / rate cache for the tc32 tile: [row_tile][walk_tile][row(256)][walk(128)]
__host__ __device__ inline int64_t tc_s_index(int64_t r, int64_t c, int64_t WT) {
  return tile_cache_index(r, c, WT, TC_N);
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
// instruction descriptor: F32 accumulate, A/B TF32, K-major, M = 256 (pair), N = 256
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)((2 * TC_M) >> 4) << 24);

__device__ inline void tc_mma2(uint32_t tmem, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(TC_IDESC), "r"(accumulate));
}
// The fp16 form (MHAR_TC_F16=1): the same 32-byte K chunks hold 16 halves, so
// one MMA covers K = 16 at twice the TF32 rate.  Operands are scaled per row
// (A) and per walk (D) by powers of two so their maxima sit in [2^14, 2^15);
// a = (a_hi + a_lo) 2^-s_r exactly, d = d_h 2^-t_c is the direction moved
// along (centrally symmetric rounding), products are exact in fp32.
constexpr uint32_t TC_IDESC_F16 = (1u << 4) | (0u << 7) | (0u << 10) |
                                  ((uint32_t)(TC_N >> 3) << 17) |
                                  ((uint32_t)((2 * TC_M) >> 4) << 24);
__device__ inline void tc_mma2_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(TC_IDESC_F16), "r"(accumulate));
}
// half layouts: the float layouts' bytes with 8 halves per 16-byte chunk
constexpr int TC_BK16 = 2 * TC_BK;  // halves per stage row
__host__ __device__ inline int64_t tc_piece_index16(int64_t r, int64_t kk, int64_t R) {
  return ((kk >> 3) * (R >> 3) + (r >> 3)) * 64 + (r & 7) * 8 + (kk & 7);
}
__host__ __device__ inline int64_t tc_d_index16(int64_t c, int64_t k, int64_t KT) {
  return ((c / TC_M) * KT + k / TC_BK16) * (TC_M * TC_BK16) +
         tc_piece_index16(c % TC_M, k % TC_BK16, TC_M);
}
__host__ __device__ inline int64_t tc_a_index16(int64_t r, int64_t k, int64_t KT) {
  return (((r / TC_N) * KT + k / TC_BK16) * 2 + (r % TC_N) / TC_NH) * (TC_NH * TC_BK16) +
         tc_piece_index16(r % TC_NH, k % TC_BK16, TC_NH);
}
// arrive on the barrier at the same smem offset in both CTAs of the pair
// once every previously issued MMA of this thread has completed
__device__ inline void tc_commit2(uint64_t* bar, unsigned short mask = 3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ inline uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ inline void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
// arrive on the barrier at `bar`'s offset in CTA `rank`.  Relaxed: what it
// publishes is not this thread's writes but completions it has observed (a
// stage's bulk copies landed, TMEM loads waited on), so the release fence --
// a MEMBAR.ALL.GPU per stage -- would only slow the pipeline.
__device__ inline void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
// wait with cluster-scope acquire (pairs with mbar_arrive_remote)
__device__ inline void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// relaxed cluster-scope wait: for barriers that only publish completions of
// async-proxy work (a peer's bulk copies landed, a peer's TMEM loads waited
// on); unlike the acquire form it does not invalidate L1 (CCTL.IVALL).
__device__ inline void mbar_wait_relaxed(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
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

// The fp32 variant's slack cache holds double-float pairs (hi, lo) in the
// 8-byte slots: s = hi + lo with |lo| <= ulp(hi) / 2.
__host__ __device__ inline double df_pack(float hi, float lo) {
  const float2 v = make_float2(hi, lo);
  return *reinterpret_cast<const double*>(&v);
}
__host__ __device__ inline float2 df_unpack(double d) { return *reinterpret_cast<const float2*>(&d); }

struct TcParams {
  const float* Ahi;  // tc_a_index layout
  const float* Alo;
  const float* Dhi;  // tc_d_index layout, TF32-exact directions (or their TF32 high part)
  const float* Dlo;  // split directions (bodies with equalities): d - d_hi in TF32, else null
  double* S;         // tc_s_index layout, fp64 slack
  float* R;          // rates of the previous iterate (fp32: what the MMA produced)
  const double* theta_prev;
  long long* hi_key;
  long long* lo_key;
  long long* viol_key;
  unsigned* sides;
  const unsigned long long* err;
  int64_t row_tiles;   // m_pad / 256
  int64_t walk_tiles;  // z_pad / 128 (even: units take walk-tile pairs)
  int64_t KT;          // n_pad / 16
  int64_t m;           // live rows
  int64_t z;           // live walks
  double eps_dir;
  double margin;       // mu: chords of {A x <= b - mu}
  int group_n;         // rasterisation band (row tiles)
  int walk_band;       // > 0: bands of this many walk-tile pairs, row tiles inner (large z)
  int a_policy;        // L2 policy of the A_hi/A_lo stream: 0 normal, 1 evict_last, 2 evict_first
  unsigned long long* prof;  // optional per-CTA wait-cycle counters (MHAR_I8_PROFILE), or null
  const float* rsc;  // fp16 form: per-row 2^s (rate = acc * rsc[r] * csc[c]), else null
  const float* csc;  // fp16 form: per-walk 2^t
  // Tensor maps over the packed operand arrays viewed as rows of 64 4-byte
  // words (one 8 KB piece = a 64 x 32 box): with them both CTAs of the pair
  // load through cp.async.bulk.tensor ... cta_group::2, whose completion
  // lands on the LEADER's full barrier -- no relay hop through the odd CTA.
  CUtensorMap tmAhi, tmAlo, tmDhi, tmDlo;
  int use_tma;
  unsigned* sched;  // unit tickets [next, finished pairs]; zero between launches
};

// one 8 KB piece (float offset `off`, a multiple of 2048) into this CTA's
// smem, completing on the pair leader's barrier `bar_leader` (shared::cluster
// address of CTA 0)
__device__ inline void tma_piece_2cta(void* dst, const CUtensorMap* tm, int64_t off,
                                      uint32_t bar_leader, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(0), "r"((int)(off >> 6)), "r"(bar_leader), "l"(policy)
      : "memory");
}

// ---- ticketed unit order shared by the tcgen05 kernels (chord_tc32, chord_i8) ----
// The cluster's CTA 0 producer draws the next unit from a global counter and
// announces it (or the end, -1) to every CTA of its cluster: a DSMEM store
// into each CTA's queue slot and a release arrive on its slot barrier; every
// role of every CTA follows that queue.  Units stay in order across clusters,
// so the operand tiles in flight stay L2-resident (a static unit-per-cluster
// assignment drifts apart over a few hundred units).  The last cluster to
// draw past the end rewinds the counter for the next launch.
constexpr int TC_UQ = 8;  // announced-unit queue per CTA (> the producer's lead in units)
__device__ inline long long cluster_next_unit(unsigned* sched, int64_t n_units, unsigned nclusters) {
  const long long u = (long long)atomicAdd(sched, 1u);
  if (u < n_units) return u;
  if (atomicAdd(sched + 1, 1u) == nclusters - 1) {
    sched[0] = 0u;
    sched[1] = 0u;
  }
  return -1;
}
__device__ inline void st_cluster_s64(uint32_t addr, long long v) {
  asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ inline void mbar_arrive_remote_release(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}
// unit u into queue slot k % TC_UQ of all `ncta` CTAs of the cluster (caller: CTA 0)
__device__ inline void cluster_announce(long long* uq, uint64_t* uready, int k, long long u,
                                        int ncta) {
  const int slot = k % TC_UQ;
  uq[slot] = u;
  for (int r = 1; r < ncta; ++r) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&uq[slot])), "r"(r));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&uready[slot])), "r"(r));
    st_cluster_s64(ra, u);
    mbar_arrive_remote_release(rb);
  }
  mbar_arrive(&uready[slot]);
}
// the cluster's k-th unit (waits for its announcement; -1: no more)
__device__ inline long long cluster_unit_at(const long long* uq, uint64_t* uready, int k) {
  mbar_wait(&uready[k % TC_UQ], (uint32_t)((k / TC_UQ) & 1));
  return uq[k % TC_UQ];
}

// unit u -> (row tile, walk-tile pair), banded over group_n row tiles; with
// walk_band > 0 (direction operands larger than L2 can hold: z beyond ~4K at
// n = 2000) bands of walk_band pairs sweep every row tile, so the band's
// direction tiles stay L2-resident and A_I is streamed once per band instead
// of every direction tile once per row tile
__device__ inline void tc_unit(int64_t u, const TcParams& p, int64_t* rt, int64_t* wp) {
  const int64_t pairs = p.walk_tiles / 2;
  if (p.walk_band > 0 && p.walk_band < pairs) {
    const int64_t band_units = (int64_t)p.walk_band * p.row_tiles;
    const int64_t band = u / band_units;
    const int64_t in_band = u - band * band_units;
    const int64_t start = band * p.walk_band;
    const int64_t w = (pairs - start < p.walk_band) ? pairs - start : p.walk_band;
    *wp = start + in_band % w;
    *rt = in_band / w;
    return;
  }
  const int64_t band_units = (int64_t)p.group_n * pairs;
  const int64_t band = u / band_units;
  const int64_t in_band = u - band * band_units;
  const int64_t start = band * p.group_n;
  const int64_t h = (p.row_tiles - start < p.group_n) ? p.row_tiles - start : p.group_n;
  *rt = start + in_band % h;
  *wp = in_band / h;
}

template <bool SPLIT_D, bool F16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    chord_tc32_kernel(const __grid_constant__ TcParams p) {
  constexpr int kStages = TcCfg<SPLIT_D>::stages;
  constexpr int kStageFloats = TcCfg<SPLIT_D>::stage_floats;
  unsigned long long g_entry = 0;
  if (p.prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
  if (*p.err != kNoError) return;  // read identically by both CTAs of the pair
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kStages * kStageFloats * 4);
  uint64_t* empty = full + kStages;
  uint64_t* peer_full = empty + kStages;  // leader: the odd CTA's stage landed
  uint64_t* tfull = peer_full + kStages;  // [2] accumulator ready (both CTAs)
  uint64_t* tempty = tfull + 2;             // [2] accumulator drained (leader, 8 warps)
  uint64_t* uready = tempty + 2;            // [TC_UQ] unit announced
  long long* uq = reinterpret_cast<long long*>(uready + TC_UQ);  // [TC_UQ] the units
  uint32_t* tptr = reinterpret_cast<uint32_t*>(uq + TC_UQ);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int64_t n_units = p.row_tiles * (p.walk_tiles / 2);
  const int KT = (int)p.KT;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&peer_full[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * TC_EPI_WARPS);  // every epilogue warp of both CTAs
    }
    for (int s = 0; s < TC_UQ; ++s) mbar_init(&uready[s], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tptr)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tptr;

  if (warp == 0) {
    // ---------------- producer: this CTA's D tile + A half ----------------
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();  // D: re-read by every row tile
      const uint64_t apol = p.a_policy == 1   ? keep
                            : p.a_policy == 2 ? policy_evict_first()
                                              : policy_evict_normal();
      int stage = 0, round = 0;
      long long w_empty = 0;
      const unsigned npairs = gridDim.x >> 1;
      if (rank == 0) cluster_announce(uq, uready, 0, cluster_next_unit(p.sched, n_units, npairs), 2);
      for (int ui = 0;; ++ui) {
        const long long u = cluster_unit_at(uq, uready, ui);
        if (u < 0) break;
        int64_t rt, wp;
        tc_unit(u, p, &rt, &wp);
        const int64_t wt = 2 * wp + rank;
#if MHAR_TC_PREFETCH
        {
          // stage this unit's slack (256 KB) and rate (128 KB) blocks in L2 about
          // one unit ahead of the epilogue
          const int64_t cb = (rt * p.walk_tiles + wt) * (int64_t)(TC_N * TC_M);
          for (int q = 0; q < 16; ++q) bulk_prefetch_l2(p.S + cb + q * 2048, 2048 * 8);
          for (int q = 0; q < 8; ++q) bulk_prefetch_l2(p.R + cb + q * 4096, 4096 * 4);
        }
#endif
        for (int kt = 0; kt < KT; ++kt) {
          const long long t0 = clock64();
          if (round > 0) mbar_wait(&empty[stage], (uint32_t)((round - 1) & 1));
          w_empty += clock64() - t0;
          float* st = ring + (size_t)stage * kStageFloats;
          const int64_t doff = (wt * p.KT + kt) * TC_D_PIECE;
          const int64_t aoff = ((rt * p.KT + kt) * 2 + rank) * TC_A_PIECE;
          if (p.use_tma) {
            // both CTAs' pieces complete on the leader's full barrier, which
            // the leader arms with the bytes of the whole pair
            uint32_t lb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(lb)
                         : "r"(smem_u32(&full[stage])), "r"(0));
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStageFloats * 4);
            tma_piece_2cta(st, &p.tmDhi, doff, lb, keep);
            tma_piece_2cta(st + TC_D_PIECE, &p.tmAhi, aoff, lb, apol);
            tma_piece_2cta(st + TC_D_PIECE + TC_A_PIECE, &p.tmAlo, aoff, lb, apol);
            if (SPLIT_D) tma_piece_2cta(st + TC_D_PIECE + 2 * TC_A_PIECE, &p.tmDlo, doff, lb, keep);
          } else {
            mbar_arrive_expect_tx(&full[stage], kStageFloats * 4);
            bulk_g2s_hint(st, p.Dhi + doff, TC_D_PIECE * 4, &full[stage], keep);
            bulk_g2s_hint(st + TC_D_PIECE, p.Ahi + aoff, TC_A_PIECE * 4, &full[stage], apol);
            bulk_g2s_hint(st + TC_D_PIECE + TC_A_PIECE, p.Alo + aoff, TC_A_PIECE * 4,
                          &full[stage], apol);
            if (SPLIT_D)
              bulk_g2s_hint(st + TC_D_PIECE + 2 * TC_A_PIECE, p.Dlo + doff, TC_D_PIECE * 4,
                            &full[stage], keep);
          }
          if (++stage == kStages) {
            stage = 0;
            ++round;
          }
        }
        // this unit's loads are queued: draw the pair's next unit
        if (rank == 0)
          cluster_announce(uq, uready, ui + 1, cluster_next_unit(p.sched, n_units, npairs), 2);
      }
      if (p.prof) p.prof[8 * blockIdx.x + 4] = (unsigned long long)w_empty;
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader CTA) ----------------
      int stage = 0, phase = 0;
      long long w_tempty = 0, w_full = 0, w_peer = 0;
      const long long t_start = clock64();
      for (int ui = 0; cluster_unit_at(uq, uready, ui) >= 0; ++ui) {
        const int ab = ui & 1;
        const long long t0 = clock64();
        if (ui >= 2) mbar_wait_relaxed(&tempty[ab], (uint32_t)(((ui >> 1) - 1) & 1));
        w_tempty += clock64() - t0;
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + (uint32_t)(ab * TC_N);
        for (int kt = 0; kt < KT; ++kt) {
          const long long t1 = clock64();
          mbar_wait(&full[stage], (uint32_t)phase);
          const long long t2 = clock64();
          if (!p.use_tma) mbar_wait_relaxed(&peer_full[stage], (uint32_t)phase);
          w_full += t2 - t1;
          w_peer += clock64() - t2;
          asm volatile("tcgen05.fence::after_thread_sync;");
          const float* sd = ring + (size_t)stage * kStageFloats;
          const float* sa_hi = sd + TC_D_PIECE;
          const float* sa_lo = sa_hi + TC_A_PIECE;
#pragma unroll
          for (int k = 0; k < TC_BK / 8; ++k) {
            // K step k: k-chunks 2k, 2k+1; LBO = stride between k-chunks
            const uint32_t dofs = 2 * k * (TC_M * 4), aofs = 2 * k * (TC_NH * 4);
            const uint64_t dd = umma_desc(sd + dofs, TC_M * 16, 128);
            const uint64_t ah = umma_desc(sa_hi + aofs, TC_NH * 16, 128);
            const uint64_t al = umma_desc(sa_lo + aofs, TC_NH * 16, 128);
            if (F16) {
              tc_mma2_f16(acc, dd, ah, (kt | k) ? 1u : 0u);
              tc_mma2_f16(acc, dd, al, 1u);
            } else {
              tc_mma2(acc, dd, ah, (kt | k) ? 1u : 0u);
              tc_mma2(acc, dd, al, 1u);
            }
            if (SPLIT_D) {
              const uint64_t dl = umma_desc(sa_lo + TC_A_PIECE + dofs, TC_M * 16, 128);
              if (F16)
                tc_mma2_f16(acc, dl, ah, 1u);
              else
                tc_mma2(acc, dl, ah, 1u);
            }
          }
          tc_commit2(&empty[stage]);  // frees the slot in both CTAs when these MMAs finish
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit2(&tfull[ab]);
      }
      if (p.prof) {
        unsigned long long* pr = p.prof + 8 * blockIdx.x;
        pr[0] = (unsigned long long)(clock64() - t_start);
        pr[1] = (unsigned long long)w_tempty;
        pr[2] = (unsigned long long)w_full;
        pr[3] = (unsigned long long)w_peer;
      }
    } else if (lane == 0 && !p.use_tma) {
      // ---------------- relay (odd CTA): my stage landed -> leader ----------------
      int stage = 0, phase = 0;
      for (int ui = 0; cluster_unit_at(uq, uready, ui) >= 0; ++ui)
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&full[stage], (uint32_t)phase);
          mbar_arrive_remote(&peer_full[stage], 0);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
    }
  } else {
    // ---------------- epilogue: thread = walk, warp = (lane quarter, row half) ----------------
    const int q = warp & 3;                      // TMEM lane quarter this warp may access
    const int rh = (warp - 2) / 4;               // which 128 of the unit's 256 rows
    const int wl = q * 32 + lane;                // walk within this CTA's tile
    const uint64_t stream_policy = MHAR_STREAM_EVICT_FIRST ? policy_evict_first() : policy_evict_normal();  // the slack stream must not evict A
    const float eps = (float)p.eps_dir, mu = (float)p.margin;
    for (int ui = 0;; ++ui) {
      const long long u = cluster_unit_at(uq, uready, ui);
      if (u < 0) break;
      int64_t rt, wp;
      tc_unit(u, p, &rt, &wp);
      const int64_t wt = 2 * wp + rank;
      const int ab = ui & 1;
      const long long e0 = clock64();
      mbar_wait(&tfull[ab], (uint32_t)((ui >> 1) & 1));
      const long long e1 = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int64_t c = wt * TC_M + wl;
      // theta as a float pair: the slack update below runs in double-float
      // (hi + lo, ~48 bits) on the fp32 pipes -- fp64 SIMT instructions issue
      // on the pipe the tensor cores keep busy and stalled this epilogue
      const double thd = p.theta_prev[c];
      const float th_hi = (float)thd, th_lo = (float)(thd - (double)th_hi);
      float hi = __int_as_float(0x7F800000), lo = -hi, viol = -hi;
      unsigned sd = 0u;
      const int64_t sbase = (rt * p.walk_tiles + wt) * TC_N * TC_M + wl;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * TC_N);
      const double* __restrict__ Sin = p.S + sbase;
      const float* __restrict__ Rin = p.R + sbase;
      double* __restrict__ Sout = p.S + sbase;
      float* __restrict__ Rout = p.R + sbase;
      // 8 rows at a time: all loads of the group in flight before any store
      // (the cache is read and rewritten in place).  The ratio test runs on
      // the fp32 pipes, branch-free -- the chord is already that of the body
      // shrunk by mu >> fp32 rounding of s / ad.
      auto rows8 = [&](int r0, const float* vv) {
        double so[TC_GROUP];
        float ro[TC_GROUP];
#pragma unroll
        for (int j = 0; j < TC_GROUP; ++j) {
          so[j] = ld_policy(Sin + (int64_t)(r0 + j) * TC_M, stream_policy);
          ro[j] = ld_policy(Rin + (int64_t)(r0 + j) * TC_M, stream_policy);
        }
#pragma unroll
        for (int j = 0; j < TC_GROUP; ++j) {
          // s = S - theta r in double-float: exact product error by FMA, TwoSum
          const float2 sp = df_unpack(so[j]);
          const float r = ro[j];
          const float ph = __fmul_rn(th_hi, r);
          const float pl = fmaf(th_lo, r, fmaf(th_hi, r, -ph));
          const float a = __fsub_rn(sp.x, ph);
          const float bb = __fsub_rn(a, sp.x);
          const float er = __fadd_rn(__fsub_rn(sp.x, __fsub_rn(a, bb)), __fsub_rn(-ph, bb));
          const float l = __fadd_rn(__fsub_rn(sp.y, pl), er);
          const bool fin = fabsf(sp.x) < __int_as_float(0x7F800000);  // +inf: padding row
          const float sh = fin ? __fadd_rn(a, l) : sp.x;
          const float sl = fin ? __fsub_rn(l, __fsub_rn(sh, a)) : 0.0f;
          st_policy(Sout + (int64_t)(r0 + j) * TC_M, df_pack(sh, sl), stream_policy);
          st_policy(Rout + (int64_t)(r0 + j) * TC_M, vv[j], stream_policy);
          const float sf = sh, ad = vv[j];
          viol = fmaxf(viol, -sf);
          const float qt = __fdividef(sf - mu, ad);
          const bool up = ad > eps, dn = ad < -eps;
          sd |= (up ? 1u : 0u) | (dn ? 2u : 0u);
          hi = up ? fminf(hi, qt) : hi;
          lo = dn ? fmaxf(lo, qt) : lo;
        }
      };
      const float cs = F16 ? p.csc[c] : 1.0f;
      for (int c0 = rh * (TC_N / 2); c0 < (rh + 1) * (TC_N / 2); c0 += 32) {
        float v[32];
        tc_ld32(taddr + (uint32_t)c0, v);
        if (F16) {
          // accumulator -> rate: the row and walk scales (powers of two)
          const float rs = __ldg(p.rsc + rt * TC_N + c0 + lane);  // lane j: row c0 + j
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= __shfl_sync(0xFFFFFFFFu, rs, j) * cs;
        }
#pragma unroll
        for (int g = 0; g < 32; g += TC_GROUP) rows8(c0 + g, v + g);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(&tempty[ab]);
        else
          mbar_arrive_remote(&tempty[ab], 0);
      }
      if (p.prof && warp == 2 && lane == 0) {
        unsigned long long* pr = p.prof + 8 * blockIdx.x;
        pr[6] += (unsigned long long)(clock64() - e1);  // drain + stream + scan
        pr[7] += (unsigned long long)(e1 - e0);         // waiting for the MMAs
      }
      if (c < p.z) {
        const long long vk = dkey((double)viol), hk = dkey((double)hi), lk = dkey((double)lo);
#if MHAR_CHORD_RED
        // fire-and-forget reductions (RED): no round trip in the epilogue
        atomicMax(p.viol_key + c, vk);
        atomicMin(p.hi_key + c, hk);
        atomicMax(p.lo_key + c, lk);
        if (sd) atomicOr(p.sides + c, sd);
#else
        if (vk > *(volatile long long*)(p.viol_key + c)) atomicMax(p.viol_key + c, vk);
        if (hk < *(volatile long long*)(p.hi_key + c)) atomicMin(p.hi_key + c, hk);
        if (lk > *(volatile long long*)(p.lo_key + c)) atomicMax(p.lo_key + c, lk);
        if (sd & ~*(volatile unsigned*)(p.sides + c)) atomicOr(p.sides + c, sd);
#endif
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // all MMAs done and consumed in both CTAs before TMEM is freed
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  if (p.prof && tid == 0) {
    unsigned long long g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    p.prof[8 * gridDim.x + 2 * blockIdx.x] = g_entry;
    p.prof[8 * gridDim.x + 2 * blockIdx.x + 1] = g_exit;
  }
}

// fp64 polytope rows -> (A_hi, A_lo); with Apk, A_used = A_hi + A_lo is also
// written into a packed fp64 copy (a debugging aid: the engine keeps the
// caller's A_I pristine for the slack refresh and containment).
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
    if (Apk && r < m && k < n) Apk[a_index(r, k, KT64)] = (double)h + (double)l;
  }
}

// fp64 directions (packed b_index) -> TF32-exact directions; D is replaced
// by them so the walk moves along exactly the direction the tensor cores see.
// Split mode (bodies with equalities): D keeps the fp64 direction (it stays in
// the null space of A_E) and d = d_hi + d_lo is handed to the tensor cores.
__global__ void tc_split_d_kernel(double* __restrict__ D, int64_t n, int64_t z_pad, int64_t KT,
                                  float* __restrict__ Dhi, float* __restrict__ Dlo,
                                  const unsigned long long* err) {
  if (*err != kNoError) return;
  const int64_t total = z_pad * KT * BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, k;
    b_coords(i, KT, &c, &k);
    const double d = D[i];
    const float h = tf32_trunc((float)d);
    Dhi[tc_d_index(c, k, KT)] = h;
    if (Dlo)
      Dlo[tc_d_index(c, k, KT)] = tf32_trunc((float)(d - (double)h));
    else
      D[i] = (double)h;
  }
}

// ---- fp16 form: per-row / per-walk power-of-two scales and half splits ----

// scale exponent: max|x| < 2^e  ->  x 2^(14 - e) in (-2^14, 2^14); clamped so
// the inverse scale stays a normal float
__device__ inline int tc16_exp(double mx) {
  int e = mx > 0.0 ? ilogb(mx) + 1 : 0;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}
// half of v with values below the fp16 normal range flushed (the tensor
// cores then see exactly what the fp64 copies say they see)
__device__ inline __half tc16_half(double v) {
  const __half h = __double2half(v);
  return fabs((double)__half2float(h)) < 6.103515625e-05 ? __float2half(0.0f) : h;
}

// per-row exponents of A_I (column-major m x n) and the split (A_used into
// Apk when given): one thread per row
__global__ void tc16_split_a_kernel(const double* __restrict__ Acm, int64_t m, int64_t n,
                                    int64_t m_pad, int64_t KT16, __half* __restrict__ Ahi,
                                    __half* __restrict__ Alo, float* __restrict__ rsc,
                                    double* __restrict__ Apk, int64_t KT64) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m_pad;
       r += (int64_t)gridDim.x * blockDim.x) {
    double mx = 0.0;
    if (r < m)
      for (int64_t k = 0; k < n; ++k) mx = fmax(mx, fabs(Acm[r + k * m]));
    const int e = tc16_exp(mx);
    const double s = ldexp(1.0, 14 - e);
    rsc[r] = ldexpf(1.0f, e - 14);
    for (int64_t k = 0; k < KT16 * TC_BK16; ++k) {
      const double a = (r < m && k < n) ? Acm[r + k * m] * s : 0.0;
      const __half h = tc16_half(a);
      const __half l = tc16_half(a - (double)__half2float(h));
      const int64_t ti = tc_a_index16(r, k, KT16);
      Ahi[ti] = h;
      Alo[ti] = l;
      if (Apk && r < m && k < n)
        Apk[a_index(r, k, KT64)] =
            ((double)__half2float(h) + (double)__half2float(l)) * ldexp(1.0, e - 14);
    }
  }
}

// per-walk exponent and the half direction; D becomes the direction moved
// along (or keeps fp64 and gets a low half: bodies with equalities).  One
// warp per walk.
__global__ void tc16_split_d_kernel(double* __restrict__ D, int64_t n, int64_t z_pad, int64_t KT,
                                    int64_t KT16, __half* __restrict__ Dhi,
                                    __half* __restrict__ Dlo, float* __restrict__ csc,
                                    const unsigned long long* err) {
  if (*err != kNoError) return;
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= z_pad) return;
  double mx = 0.0;
  for (int64_t k = lane; k < n; k += 32) mx = fmax(mx, fabs(D[b_index(c, k, KT)]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  const int e = tc16_exp(mx);
  const double t = ldexp(1.0, 14 - e), ti = ldexp(1.0, e - 14);
  if (lane == 0) csc[c] = ldexpf(1.0f, e - 14);
  for (int64_t k = lane; k < KT16 * TC_BK16; k += 32) {
    const double d = k < n ? D[b_index(c, k, KT)] * t : 0.0;
    const __half h = tc16_half(d);
    Dhi[tc_d_index16(c, k, KT16)] = h;
    if (Dlo)
      Dlo[tc_d_index16(c, k, KT16)] = tc16_half(d - (double)__half2float(h));
    else if (k < n)
      D[b_index(c, k, KT)] = (double)__half2float(h) * ti;
  }
}

}  // namespace mhar_dev
