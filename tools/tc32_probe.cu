// tcgen05 kind::tf32 probe for B200 (sm_100a): one CTA tile C[128 x 256] =
// A[128 x K] * B[256 x K]^T, both K-major in the no-swizzle "interleaved"
// core-matrix layout, fp32 accumulator in TMEM, operands fed by cp.async.bulk
// through an mbarrier ring, one thread issuing the MMAs.  Checks a tile
// against the CPU and times a full-chip grid.  Prints JSON.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 256, BK = 32, STAGES = 4;
constexpr int A_STAGE = M * BK;  // floats (16 KB)
constexpr int B_STAGE = N * BK;  // floats (32 KB)

__device__ inline uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c));
}
__device__ inline void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ inline void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W%=;\n}\n" ::"r"(s32(b)), "r"(ph) : "memory");
}
__device__ inline void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)), "l"(src), "r"(bytes), "r"(s32(b)) : "memory");
}
// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; SBO = stride between
// 8-row groups, LBO = stride between the two 16-B K halves of one K=8 step.
__device__ inline uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((s32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);

__global__ void __launch_bounds__(128, 1) tc_tile(const float* A, const float* B, float* C, int KT,
                                                  int stride_tiles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* ring = reinterpret_cast<float*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)STAGES * (A_STAGE + B_STAGE) * 4);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float* Ab = A + (size_t)(blockIdx.x % stride_tiles) * KT * A_STAGE;
  const float* Bb = B + (size_t)(blockIdx.x % stride_tiles) * KT * B_STAGE;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tptr)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tptr;

  if (tid == 0) {
    auto load = [&](int kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
      float* st = ring + (size_t)s * (A_STAGE + B_STAGE);
      mbar_expect(&full[s], (A_STAGE + B_STAGE) * 4);
      bulk(st, Ab + (size_t)kt * A_STAGE, A_STAGE * 4, &full[s]);
      bulk(st + A_STAGE, Bb + (size_t)kt * B_STAGE, B_STAGE * 4, &full[s]);
    };
    for (int kt = 0; kt < STAGES - 1 && kt < KT; ++kt) load(kt);
    for (int kt = 0; kt < KT; ++kt) {
      if (kt + STAGES - 1 < KT) load(kt + STAGES - 1);
      const int s = kt % STAGES;
      mbar_wait(&full[s], (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const float* sa = ring + (size_t)s * (A_STAGE + B_STAGE);
      const float* sb = sa + A_STAGE;
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {
        // K step k covers k-chunks 2k, 2k+1 (4 floats = 16 B each)
        const uint64_t da = sdesc(sa + 2 * k * (M * 4), M * 4 * 4, 128);
        const uint64_t db = sdesc(sb + 2 * k * (N * 4), N * 4 * 4, 128);
        const uint32_t acc = (kt | k) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(IDESC), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&empty[s])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(done)) : "memory");
  }
  __syncwarp();
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: thread = row (lane 32 warp + lane), 32 columns per load
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (C && blockIdx.x == 0)
      for (int j = 0; j < 32; ++j) C[(size_t)row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

// logical (row, k) -> interleaved K-major offset within a stage of R rows
static size_t ilv(int r, int k, int R) {
  const int kt = k / BK, kk = k % BK, kc = kk / 4, ke = kk % 4;
  return (size_t)kt * R * BK + ((size_t)kc * (R / 8) + r / 8) * 32 + (r % 8) * 4 + ke;
}
static float tf32(float x) {  // round-toward-zero to 10 mantissa bits: exactly representable
  uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x;
}

int main() {
  const int K = 512, KT = K / BK;
  std::vector<float> a((size_t)M * K), b((size_t)N * K), pa(a.size()), pb(b.size());
  srand(1);
  for (auto& x : a) x = tf32((rand() / (float)RAND_MAX) - 0.5f);
  for (auto& x : b) x = tf32((rand() / (float)RAND_MAX) - 0.5f);
  for (int r = 0; r < M; ++r) for (int k = 0; k < K; ++k) pa[ilv(r, k, M)] = a[(size_t)r * K + k];
  for (int r = 0; r < N; ++r) for (int k = 0; k < K; ++k) pb[ilv(r, k, N)] = b[(size_t)r * K + k];
  float *dA, *dB, *dC;
  cudaMalloc(&dA, pa.size() * 4); cudaMalloc(&dB, pb.size() * 4); cudaMalloc(&dC, (size_t)M * N * 4);
  cudaMemcpy(dA, pa.data(), pa.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)STAGES * (A_STAGE + B_STAGE) * 4 + 256;
  cudaFuncSetAttribute(tc_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tc_tile<<<1, 128, smem>>>(dA, dB, dC, KT, 1);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> c((size_t)M * N);
  cudaMemcpy(c.data(), dC, c.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)a[(size_t)i * K + k] * b[(size_t)j * K + k];
      maxerr = fmax(maxerr, fabs(s - c[(size_t)i * N + j]));
      maxref = fmax(maxref, fabs(s));
    }
  // throughput: 148 x 2 CTAs, long K re-reading an L2-resident tile set
  const int KT2 = 512;
  float *dA2, *dB2;
  const int tiles = 16;
  cudaMalloc(&dA2, (size_t)tiles * KT2 * A_STAGE * 4); cudaMalloc(&dB2, (size_t)tiles * KT2 * B_STAGE * 4);
  cudaMemset(dA2, 0, (size_t)tiles * KT2 * A_STAGE * 4); cudaMemset(dB2, 0, (size_t)tiles * KT2 * B_STAGE * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  tc_tile<<<sms, 128, smem>>>(dA2, dB2, nullptr, KT2, tiles);
  cudaDeviceSynchronize();
  cudaEventRecord(t0);
  tc_tile<<<sms, 128, smem>>>(dA2, dB2, nullptr, KT2, tiles);
  cudaEventRecord(t1); cudaEventSynchronize(t1);
  float ms; cudaEventElapsedTime(&ms, t0, t1);
  const double flops = 2.0 * M * N * (double)KT2 * BK * sms;
  printf("{\"status\": \"%s\", \"tile_max_abs_err\": %.3e, \"tile_max_ref\": %.3e, \"tf32_tflops_1cta_per_sm\": %.1f}\n",
         cudaGetErrorString(e), maxerr, maxref, flops / (ms * 1e-3) / 1e12);
  return 0;
}
