// common.cuh -- layouts, counter RNGs and PTX wrappers shared by the MHAR
// kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mhar_dev {

// ---------------------------------------------------------------------------
// Tile geometry of the fp64 tensor-core path.
//
// The chord kernel is a C = A_I * B product (M = inequality rows, N = walk
// columns, K = dimension) on DMMA.8x8x4 (mma.sync .f64; tcgen05 has no f64
// kind).  Operands live in HBM pre-permuted into the exact register-fragment
// order the MMA consumes, so every pipeline stage is ONE contiguous
// cp.async.bulk copy and every fragment load is one conflict-free 16-byte LDS.
//
//   A_I  : [m_tile][k_tile][k8][row_group(16)][lane(32)][2]     BM = 128 rows
//   X,D,H: [walk_tile][k_tile][k8][col_group(8)][lane(32)][2]   BC = 64 walks
//
// with BK = 16 = 2 x k8, and inside a k8 group lane l holds (row|col = l/4,
// k = l%4) for the first k4 step and k+4 for the second -- the mma.m8n8k4
// fragment maps (A: row = l>>2, k = l&3; B: k = l&3, col = l>>2).
// ---------------------------------------------------------------------------
#ifndef MHAR_STREAM_EVICT_FIRST
#define MHAR_STREAM_EVICT_FIRST 1  // L2 policy of the tcgen05 kernels' slack/rate stream
#endif
constexpr int BM = 128;        // rows of A_I per tile
constexpr int BK = 16;         // k per pipeline stage
constexpr int BC = 64;         // walks per B piece
constexpr int A_PIECE = BM * BK;  // doubles per A stage piece (16 KB)
constexpr int B_PIECE = BC * BK;  // doubles per B stage piece (8 KB)

__host__ __device__ inline int64_t a_index(int64_t r, int64_t k, int64_t KT) {
  const int64_t mt = r / BM, rr = r % BM, rg = rr / 8, rin = rr % 8;
  const int64_t kt = k / BK, kk = k % BK, k8 = kk / 8, kin = kk % 8, e = kin / 4, kq = kin % 4;
  const int64_t lane = rin * 4 + kq;
  return ((((mt * KT + kt) * 2 + k8) * 16 + rg) * 32 + lane) * 2 + e;
}

__host__ __device__ inline int64_t b_index(int64_t c, int64_t k, int64_t KT) {
  const int64_t ct = c / BC, cc = c % BC, cg = cc / 8, cin = cc % 8;
  const int64_t kt = k / BK, kk = k % BK, k8 = kk / 8, kin = kk % 8, e = kin / 4, kq = kin % 4;
  const int64_t lane = cin * 4 + kq;
  return ((((ct * KT + kt) * 2 + k8) * 8 + cg) * 32 + lane) * 2 + e;
}

// Inverse of b_index: (walk, coordinate) of packed element i.
__host__ __device__ inline void b_coords(int64_t i, int64_t KT, int64_t* c, int64_t* k) {
  const int64_t e = i & 1;
  int64_t t = i >> 1;
  const int64_t lane = t & 31; t >>= 5;
  const int64_t cg = t & 7; t >>= 3;
  const int64_t k8 = t & 1; t >>= 1;
  const int64_t kt = t % KT;
  const int64_t ct = t / KT;
  *c = ct * BC + cg * 8 + (lane >> 2);
  *k = kt * BK + k8 * 8 + e * 4 + (lane & 3);
}

// Slack / rate cache of the incremental mode, stored in the accumulator
// order of the incremental chord tile (128 rows x 64 walks, 8 warps as
// 4 row-groups x 2 walk-groups, warp tile 32 x 32) so each warp reads and
// writes 512 contiguous bytes per fragment:
// [m_tile][walk_tile64][warp(8)][i(4)][j(4)][lane(32)][2].
constexpr int64_t S_WARP_BLOCK = 4 * 4 * 32 * 2;  // doubles per warp per tile
// Slack/rate cache of the tensor-core (tcgen05) chord kernels: [row_tile(rows)]
// [walk_tile(128)][row][walk] -- rows = 256 (fp32 variant), 64 (int8-slice engine).
__host__ __device__ inline int64_t tile_cache_index(int64_t r, int64_t c, int64_t WT, int64_t rows) {
  return (((r / rows) * WT + c / 128) * rows + r % rows) * 128 + c % 128;
}

// Slack/rate cache of chord3_kernel (128-row x 128-walk units, 8 warps of
// 64 x 32 DMMA tiles): [unit][warp(8)][i(8)][j(4)][lane(32)][2] -- the
// accumulator fragment order, one coalesced 512-byte block per (warp, i, j).
__host__ __device__ inline int64_t c3_index(int64_t r, int64_t c, int64_t CT128) {
  const int64_t mt = r / 128, rr = r % 128, wm = rr / 64, i = (rr % 64) / 8, rq = rr % 8;
  const int64_t ct = c / 128, cc = c % 128, wn = cc / 32, j = (cc % 32) / 8, cq = (cc % 8) / 2,
                e = cc % 2;
  const int64_t warp = wm * 4 + wn, lane = rq * 4 + cq;
  return (((((mt * CT128 + ct) * 8 + warp) * 8 + i) * 4 + j) * 32 + lane) * 2 + e;
}

__host__ __device__ inline int64_t s_index(int64_t r, int64_t c, int64_t CT64) {
  const int64_t mt = r / BM, rr = r % BM, wm = rr / 32, i = (rr % 32) / 8, rq = rr % 8;
  const int64_t ct = c / BC, cc = c % BC, wn = cc / 32, j = (cc % 32) / 8, cq = (cc % 8) / 2,
                e = cc % 2;
  const int64_t warp = wm * 2 + wn, lane = rq * 4 + cq;
  return (((((mt * CT64 + ct) * 8 + warp) * 4 + i) * 4 + j) * 32 + lane) * 2 + e;
}

// ---------------------------------------------------------------------------
// Order-preserving double <-> int64 keys for atomicMin/atomicMax reductions.
// Exact min/max is order independent, so the chord bounds are deterministic.
// ---------------------------------------------------------------------------
__host__ __device__ inline long long dkey(double x) {
  long long b;
#ifdef __CUDA_ARCH__
  b = __double_as_longlong(x);
#else
  memcpy(&b, &x, 8);
#endif
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
}
__host__ __device__ inline double keyd(long long k) {
  const long long b = k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL);
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double x;
  memcpy(&x, &b, 8);
  return x;
#endif
}

// ---------------------------------------------------------------------------
// Counter RNGs.
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;      // rng.cpp:13
constexpr uint64_t kStreamSalt = 0x6A09E667F3BCC909ULL;  // rng.cpp:14
constexpr double kTwoPi = 6.283185307179586;             // rng.cpp:15

__host__ __device__ inline uint64_t mix64(uint64_t x) {  // rng.cpp:17-21
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t stream_init(uint64_t seed, uint64_t stream) {  // rng.cpp:101
  return mix64(seed + kGolden) ^ mix64(stream + kStreamSalt);
}
__host__ __device__ inline double u01_closed_open(uint64_t bits) {  // next_uniform
  return (double)(bits >> 11) * 0x1.0p-53;
}
__host__ __device__ inline double u01_open_closed(uint64_t bits) {  // next_uniform_open
  return (double)((bits >> 11) + 1) * 0x1.0p-53;
}

// Philox4x32-10 (Salmon et al., SC'11).
struct Philox4 {
  uint32_t v[4];
};
__device__ inline Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  Philox4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// Domains separate the normal draws from the chord-position draws.
constexpr uint32_t kDomNormal = 0u;
constexpr uint32_t kDomTheta = 1u;

// Two 64-bit words from Philox keyed (seed) with the 128-bit counter
// (index, walk[0:32], iterate[0:32],
//  iterate[32:48] | attempt[0:6] << 16 | walk[32:40] << 22 | domain << 30):
// distinct for iterates < 2^48, walks < 2^40, attempts < 64.
__device__ inline void philox_u64x2(uint64_t seed, uint32_t index, uint64_t walk,
                                    uint64_t iterate, uint32_t attempt, uint32_t domain,
                                    uint64_t* a, uint64_t* b) {
  const uint32_t c1 = (uint32_t)walk;
  const uint32_t c2 = (uint32_t)iterate;
  const uint32_t c3 = ((uint32_t)(iterate >> 32) & 0xFFFFu) | ((attempt & 0x3Fu) << 16) |
                      (((uint32_t)(walk >> 32) & 0xFFu) << 22) | (domain << 30);
  const Philox4 r = philox4x32_10(index, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  *a = ((uint64_t)r.v[0] << 32) | r.v[1];
  *b = ((uint64_t)r.v[2] << 32) | r.v[3];
}

// Box-Muller pair (rng.cpp:115-124): (r cos a, r sin a), r = sqrt(-2 ln u1), a = 2 pi u2.
__device__ inline void box_muller(double u1, double u2, double* c, double* s) {
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = kTwoPi * u2;
  double sn, cs;
  sincos(angle, &sn, &cs);
  *c = radius * cs;
  *s = radius * sn;
}

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier, bulk async copy, DMMA.
// ---------------------------------------------------------------------------
__device__ inline uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ inline void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ inline void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ inline void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ inline void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ inline void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One contiguous global -> shared bulk copy completing on `bar` (TMA engine, UBLKCP).
__device__ inline void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same copy with an L2 eviction-priority policy (createpolicy).
__device__ inline void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                     uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// the same copy landing at the same offset in every CTA of ctaMask, each
// CTA's mbarrier at bar's offset receiving the bytes
__device__ inline void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                   uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1], %2, [%3], %4, %5;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ inline uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ inline uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Streaming fp64 load / store with an explicit L2 eviction policy.
__device__ inline double ld_policy(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ inline void st_policy(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
               : "memory");
}
__device__ inline float ld_policy(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ inline void st_policy(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol)
               : "memory");
}
__device__ inline uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Bulk prefetch of [src, src + bytes) into L2 (no smem destination).
__device__ inline void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// D = A(8x4, row) * B(4x8, col) + D, fp64 tensor core (SASS DMMA.8x8x4).
__device__ inline void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Error word: (phase << 56) | (walk << 8) | status; atomicMin keeps the
// earliest phase, then the lowest walk -- the reference raises for the first
// walk in index order within a phase (sampler.cpp:182-200, 255-265).
constexpr unsigned long long kNoError = ~0ULL;
// Programmatic dependent launch (the iterate chain's kernels, launched with
// cudaLaunchAttributeProgrammaticStreamSerialization by abi.cu launch_k):
// a kernel lets its successor's CTAs be scheduled as soon as all of its own
// CTAs are running, and every kernel waits for its predecessor's completion
// and memory before touching any of it.  Without the attribute both are
// no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}

__device__ inline unsigned long long error_word(int phase, int64_t walk, int status) {
  return ((unsigned long long)phase << 56) | ((unsigned long long)walk << 8) |
         (unsigned long long)status;
}

}  // namespace mhar_dev
