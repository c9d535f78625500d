// tcgen05 kind::i8 throughput probe for B200 (sm_100a): MMAs issued
// back-to-back over smem-resident operand tiles (no global traffic), to find
// how the int8 tensor-core rate depends on N, on cta_group::1 vs ::2, and on
// the A operand coming from smem (SS) or TMEM (TS).  Prints JSON lines.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ inline uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((s32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ inline void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c));
}
__device__ inline void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W%=;\n}\n" ::"r"(s32(b)), "r"(ph) : "memory");
}
__device__ inline uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

constexpr int KB = 32;  // bytes of K per MMA

// MODE 0: cg1 SS, 1: cg1 TS (A in TMEM), 2: cg2 SS, 3: cg2 SS kind::tf32 (K = 8 per MMA),
// 4: cg2 SS kind::f16 (K = 16 per MMA, f32 accumulate)
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, int mmas_per_iter, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint8_t* sa = sm;                  // A: 128 rows x 32 B = 4 KB, x 8 tiles
  uint8_t* sb = sm + 8 * 4096;       // B: up to 256 rows x 32 B = 8 KB, x 4 tiles
  uint64_t* done = reinterpret_cast<uint64_t*>(sm + 8 * 4096 + 4 * 8192);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = (MODE >= 2) ? ctarank() : 0;
  for (int i = tid; i < (8 * 4096 + 4 * 8192) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (tid == 0) {
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    if (MODE >= 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tptr)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tptr)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (MODE >= 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tptr;
  const uint32_t M = (MODE >= 2) ? 256 : 128;
  const uint32_t idesc = MODE == 3
      ? (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24)
      : MODE == 4 ? (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24)
      : (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
  const int nb = (MODE >= 2) ? N / 2 : N;  // B rows staged per CTA
  if (tid == 0 && rank == 0) {
    for (int it = 0; it < iters; ++it) {
      for (int q = 0; q < mmas_per_iter; ++q) {
        const uint64_t da = sdesc(sa + (q & 7) * 4096, 128 * 16, 128);
        const uint64_t db = sdesc(sb + (q & 3) * 8192, nb * 16, 128);
        const uint32_t acc = tmem + (uint32_t)((q % (256 / N > 0 ? 256 / N : 1)) * N) % 256;
        if (MODE == 0) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(acc), "l"(da), "l"(db), "r"(idesc), "r"(1u));
        } else if (MODE == 1) {
          const uint32_t ta = tmem + 256 + (uint32_t)((q & 7) * 8);  // A: 128 lanes x 8 columns
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(acc), "r"(ta), "l"(db), "r"(idesc), "r"(1u));
        } else if (MODE == 2) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(acc), "l"(da), "l"(db), "r"(idesc), "r"(1u));
        } else if (MODE == 3) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(acc), "l"(da), "l"(db), "r"(idesc), "r"(1u));
        } else {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(acc), "l"(da), "l"(db), "r"(idesc), "r"(1u));
        }
      }
    }
    if (MODE >= 2)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(s32(done)), "h"((unsigned short)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(done)) : "memory");
  }
  __syncwarp();
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (v == 0x12345678u) sink[0] = v;
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (MODE >= 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 0) {
    if (MODE >= 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

template <int MODE, int N>
void run(unsigned long long* sink, int sms) {
  const size_t smem = 8 * 4096 + 4 * 8192 + 64;
  cudaFuncSetAttribute(probe<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 2000, per = 34;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (MODE >= 2) ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, probe<MODE, N>, iters, per, sink);
  cudaDeviceSynchronize();
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  cudaLaunchKernelEx(&cfg, probe<MODE, N>, iters, per, sink);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaError_t e = cudaGetLastError();
  const double ops_per_sm =
      2.0 * 128 * N * (MODE == 3 ? KB / 4 : MODE == 4 ? KB / 2 : KB) * (double)iters * per;  // M per SM is 128
  const double tops = ops_per_sm * sms / (ms * 1e-3) / 1e12;
  if (MODE == 3)
    printf("{\"mode\": \"cg2_SS_tf32\", \"N\": %d, \"status\": \"%s\", \"ms\": %.3f, \"tf32_tflops\": %.1f}\n",
           N, cudaGetErrorString(e), ms, tops);
  else if (MODE == 4)
    printf("{\"mode\": \"cg2_SS_f16\", \"N\": %d, \"status\": \"%s\", \"ms\": %.3f, \"f16_tflops\": %.1f}\n",
           N, cudaGetErrorString(e), ms, tops);
  else
    printf("{\"mode\": \"%s\", \"N\": %d, \"status\": \"%s\", \"ms\": %.3f, \"int8_tops\": %.1f}\n",
           MODE == 0 ? "cg1_SS" : MODE == 1 ? "cg1_TS" : "cg2_SS", N, cudaGetErrorString(e), ms, tops);
}


// The engine's pass-1 issue pattern (levels 4..7 of 7x7 slice pairs, N = 128,
// cta_group::2): VAR = 0 exact sequence (signedness per pair, same-accumulator
// runs), 1 constant idesc, 2 accumulator rotated every MMA.
template <int VAR>
__global__ void __launch_bounds__(128, 1) probe_seq(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint8_t* sa = sm;                  // 7 direction slices x 4 KB
  uint8_t* sb = sm + 7 * 4096;       // 7 A half slices x 2 KB
  uint64_t* done = reinterpret_cast<uint64_t*>(sm + 7 * 4096 + 7 * 2048);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = ctarank();
  for (int i = tid; i < (7 * 4096 + 7 * 2048) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (tid == 0) {
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tptr)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tptr;
  if (tid == 0 && rank == 0) {
    uint64_t dd[7], da[7];
    for (int s = 0; s < 7; ++s) {
      dd[s] = sdesc(sa + s * 4096, 128 * 16, 128);
      da[s] = sdesc(sb + s * 2048, 64 * 16, 128);
    }
    int q = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int l = 4; l < 8; ++l) {
        const int i0 = l > 6 ? l - 6 : 0, i1 = l < 6 ? l : 6;
#pragma unroll
        for (int i = i0; i <= i1; ++i) {
          const int j = l - i;
          const uint32_t sa_ = VAR == 1 ? 1u : (j == 0 ? 1u : 0u), sb_ = VAR == 1 ? 1u : (i == 0 ? 1u : 0u);
          const uint32_t idesc = (2u << 4) | (sa_ << 7) | (sb_ << 10) | ((uint32_t)(128 >> 3) << 17) | ((256u >> 4) << 24);
          const uint32_t acc = tmem + (uint32_t)(((VAR == 2 ? (q++ & 3) : (l - 4))) * 128);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(acc), "l"(dd[j]), "l"(da[i]), "r"(idesc), "r"(1u));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(s32(done)), "h"((unsigned short)3) : "memory");
  }
  __syncwarp();
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (v == 0x12345678u) sink[0] = v;
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int VAR>
void run_seq(unsigned long long* sink, int sms) {
  const size_t smem = 7 * 4096 + 7 * 2048 + 64;
  cudaFuncSetAttribute(probe_seq<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 2000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, probe_seq<VAR>, iters, sink);
  cudaDeviceSynchronize();
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  cudaLaunchKernelEx(&cfg, probe_seq<VAR>, iters, sink);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  const double ops_per_sm = 2.0 * 128 * 128 * KB * (double)iters * 24;
  printf("{\"mode\": \"engine_pass1_seq_var%d\", \"N\": 128, \"status\": \"%s\", \"ms\": %.3f, \"int8_tops\": %.1f}\n",
         VAR, cudaGetErrorString(cudaGetLastError()), ms, ops_per_sm * sms / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  run<0, 64>(sink, sms);
  run<0, 128>(sink, sms);
  run<0, 256>(sink, sms);
  run<1, 64>(sink, sms);
  run<1, 128>(sink, sms);
  run<1, 256>(sink, sms);
  run<2, 64>(sink, sms);
  run<2, 128>(sink, sms);
  run<2, 256>(sink, sms);
  run<3, 128>(sink, sms);
  run<3, 256>(sink, sms);
  run<4, 128>(sink, sms);
  run<4, 256>(sink, sms);
  run_seq<0>(sink, sms);
  run_seq<1>(sink, sms);
  run_seq<2>(sink, sms);
  return 0;
}
