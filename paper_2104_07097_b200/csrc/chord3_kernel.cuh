// chord3_kernel.cuh -- the incremental DMMA chord kernel, warp-specialised
// through TMEM (round 2).
//
// Same computation as chord2_kernel<INCREMENTAL> (compute_lambda_intervals,
// /root/reference/proj/src/sampler.cpp:150-208, slack carried incrementally;
// bit-identical rates, slack and bounds), organised so that the slack-cache
// epilogue never holds the fp64 tensor pipe up:
//
// - one 512-thread CTA per SM.  Warps 0..7 only multiply: each owns a 64 x 32
//   DMMA.8x8x4 warp tile of the 128-row x 128-walk unit (128 accumulator
//   doubles in registers: setmaxnreg raises them to C3_MMA_REGS), fed by a
//   6-stage cp.async.bulk ring (32 KB per stage).  Warps 8..15 only run the
//   epilogue (setmaxnreg lowers them to C3_EPI_REGS).
// - fp64 has no tcgen05 kind, but TMEM still works as a register-to-register
//   mailbox: when an MMA warp finishes a unit it stores its 64 accumulators
//   into its TMEM lane quarter (tcgen05.st.32x32b, thread t -> lane t) and
//   starts the next unit at once; its twin epilogue warp (same lane quarter)
//   reads them back with tcgen05.ld and streams the slack / rate cache, the
//   ratio test and the bound reductions while the tensor pipe works on.  Two
//   TMEM buffers (2 x 256 columns) let the epilogue lag a whole unit.
// - chord2 ran two 256-thread CTAs per SM with 32 x 32 warp tiles, so while
//   one CTA was in its epilogue the other's 8 warps could not fill the DMMA
//   pipe alone (config 3: 79.6 % of peak); 64 x 32 tiles saturate it with
//   two warps per sub-partition (tools/microbench_dmma_tile.cu).
// - the epilogue carries the bounds as integer keys and tests rows with
//   integer compares (scan_row_key, reduce_and_publish_keys): its only fp64
//   instruction per element is the slack update, so it no longer queues
//   behind the MMAs on the shared fp64 pipe (ncu stall_math; config 3 went
//   from 75.6 % to 83.5 % of DMMA peak with it).
// - units in ticket order (next_unit, chord_kernel.cuh), banded over group_m
//   row tiles.  The slack / rate cache is stored in this kernel's fragment
//   order (c3_index): every epilogue access is a coalesced 512-byte warp
//   transaction.
#pragma once

#include "chord_kernel.cuh"

namespace mhar_dev {

constexpr int C3_THREADS = 512;   // 8 MMA warps + 8 epilogue warps
constexpr int C3_BW = 128;        // walks per unit (two packed 64-walk tiles)
#ifndef MHAR_C3_APOL
#define MHAR_C3_APOL 1  // L2 policy of the A_I stream: 0 normal, 1 evict_last (tools/ab_c3pol.sh)
#endif
#ifndef MHAR_C3_DPOL
#define MHAR_C3_DPOL 0  // of the direction tiles: 0 evict_last, 1 normal
#endif
#ifndef MHAR_C3_STAGES
#define MHAR_C3_STAGES 6
#endif
#ifndef MHAR_C3_LAG
#define MHAR_C3_LAG 2
#endif
constexpr int C3_STAGES = MHAR_C3_STAGES;
constexpr int C3_LAG = MHAR_C3_LAG;
constexpr int C3_STAGE = A_PIECE + 2 * B_PIECE;  // doubles per stage (32 KB)
constexpr int C3_UQ = 8;
constexpr size_t C3_BAR_OFF = (size_t)C3_STAGES * C3_STAGE * 8;
constexpr size_t C3_SMEM = C3_BAR_OFF + 1024;
#ifndef MHAR_C3_PAIRBAR
// 1: the TMEM hand-off barriers are per twin pair (MMA warp w <-> epilogue
// warp w + 8, one arrival each) instead of one 8-arrival barrier per buffer,
// so a slow epilogue warp holds up only its twin, which the ring's depth
// absorbs (tools/ab_c3pair.sh)
#define MHAR_C3_PAIRBAR 1
#endif
constexpr int C3_TB = MHAR_C3_PAIRBAR ? 8 : 1;  // hand-off barriers per TMEM buffer
#ifndef MHAR_C3_MMA_REGS
#define MHAR_C3_MMA_REGS 208
#endif
constexpr int C3_MMA_REGS = MHAR_C3_MMA_REGS;
#ifndef MHAR_C3_EPI_REGS
#define MHAR_C3_EPI_REGS (256 - MHAR_C3_MMA_REGS)
#endif
constexpr int C3_EPI_REGS = MHAR_C3_EPI_REGS;  // 512 threads share the 64K-register file
#ifndef MHAR_C3_DEC_FIRST
// 1: the epilogue warps execute setmaxnreg.dec before the CTA's first barrier
// and the MMA warps' .inc follows it.  With the .dec inside the epilogue
// branch, two processes time-slicing one GPU (compute preemption of the
// CTA) ended in an illegal memory access in every stress run
// (tools/shared_gpu_stress.py: 0 of 13 runs failed; the original order, an
// .inc that waits on the .dec through a named barrier, or the TMEM
// allocation moved to an MMA warp all failed).  Cost: 0.3-0.5 %.
#define MHAR_C3_DEC_FIRST 1
#endif


// tcgen05 register <-> TMEM moves, 32x32b shape: thread t of the warp owns
// TMEM lane (quarter * 32 + t); consecutive registers go to consecutive columns
__device__ inline void tm_st64(uint32_t taddr, const uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63, %64};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(v[32]), "r"(v[33]), "r"(v[34]), "r"(v[35]), "r"(v[36]), "r"(v[37]), "r"(v[38]), "r"(v[39]), "r"(v[40]), "r"(v[41]), "r"(v[42]), "r"(v[43]), "r"(v[44]), "r"(v[45]), "r"(v[46]), "r"(v[47]), "r"(v[48]), "r"(v[49]), "r"(v[50]), "r"(v[51]), "r"(v[52]), "r"(v[53]), "r"(v[54]), "r"(v[55]), "r"(v[56]), "r"(v[57]), "r"(v[58]), "r"(v[59]), "r"(v[60]), "r"(v[61]), "r"(v[62]), "r"(v[63])
      : "memory");
}
// load + wait in one statement: the registers are defined only once the
// load has completed (a separate wait asm would not order their uses).  The
// memory clobber keeps the slack / rate loads issued above it in flight
// across the wait instead of letting the compiler sink them below it.
__device__ inline void tm_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr)
      : "memory");
}

// 16-byte streaming store with an L2 eviction-priority policy
__device__ inline void st_policy2(double* ptr, double a, double b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(a), "d"(b),
               "l"(pol)
               : "memory");
}

// unit u -> (row tile, 128-walk tile): bands of group_m row tiles, walk tiles inner
__device__ inline void c3_unit(int64_t u, const ChordParams& p, int64_t* mt, int64_t* ct) {
  const int64_t band_units = (int64_t)p.group_m * p.c3_tiles;
  const int64_t band = u / band_units;
  const int64_t in_band = u - band * band_units;
  const int64_t start = band * p.group_m;
  const int64_t h = (p.m_tiles - start < p.group_m) ? p.m_tiles - start : p.group_m;
  *mt = start + in_band % h;
  *ct = in_band / h;
}

// PROF: per-CTA phase cycle counters into p.prof (MHAR_C3_PROFILE); the
// production instantiation carries no clock reads
template <bool PROF>
__global__ void __launch_bounds__(C3_THREADS, 1) chord3_kernel(const ChordParams p) {
  auto pclock = []() -> long long { return PROF ? clock64() : 0; };
  if (*p.err != kNoError) return;  // sticky device error: read identically by every thread
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C3_BAR_OFF);
  uint64_t* empty = full + C3_STAGES;
  uint64_t* uready = empty + C3_STAGES;  // [C3_UQ] unit announced
  uint64_t* tfull = uready + C3_UQ;      // [2][C3_TB] a unit's accumulators in TMEM buffer b
  uint64_t* tempty = tfull + 2 * C3_TB;  // [2][C3_TB] buffer b read back by the epilogue warps
  long long* uq = reinterpret_cast<long long*>(tempty + 2 * C3_TB);  // [C3_UQ] the units
  uint32_t* tptr = reinterpret_cast<uint32_t*>(uq + C3_UQ);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_units = p.m_tiles * p.c3_tiles;
  const int KT = (int)p.KT;

  if (tid == 0) {
    for (int s = 0; s < C3_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);  // the 8 MMA warps
    }
    for (int s = 0; s < C3_UQ; ++s) mbar_init(&uready[s], 1);
    for (int b = 0; b < 2 * C3_TB; ++b) {
      mbar_init(&tfull[b], 8 / C3_TB);   // the (twin) MMA warp(s) stored their tiles
      mbar_init(&tempty[b], 8 / C3_TB);  // the (twin) epilogue warp(s) read them
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tptr)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
#if MHAR_C3_DEC_FIRST && !defined(MHAR_C3_NO_SETMAXNREG)
  // the epilogue warps release their registers before the barrier, so the
  // MMA warps' setmaxnreg.inc below never has to wait for them
  if (warp >= 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C3_EPI_REGS));
#endif
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tptr;
  auto unit_at = [&](int k) -> long long {
    mbar_wait(&uready[k % C3_UQ], (uint32_t)((k / C3_UQ) & 1));
    return uq[k % C3_UQ];
  };

  if (warp < 8) {
#ifndef MHAR_C3_NO_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C3_MMA_REGS));
#endif
    // ------------------------------ MMA warps ------------------------------
    const int wm = warp >> 2, wn = warp & 3;  // warp tile: 64 rows x 32 walks
    // producer (thread 0): the ring's (unit, k tile) sequence, C3_STAGES -
    // C3_LAG stages ahead; it draws the tickets and announces the units
    struct Producer {
      const double* a;
      const double* b0;
      const double* b1;
      int kt, stage, round, ann;
      long long unit;
    };
    __shared__ Producer pr;
    auto announce = [&](long long u) {
      uq[pr.ann % C3_UQ] = u;
      mbar_arrive(&uready[pr.ann % C3_UQ]);
      ++pr.ann;
      pr.unit = u;
      if (u >= 0) {
        int64_t mt, ct;
        c3_unit(u, p, &mt, &ct);
        pr.a = p.A + mt * p.KT * A_PIECE;
        pr.b0 = p.D + (2 * ct) * p.KT * B_PIECE;
        pr.b1 = pr.b0 + p.KT * B_PIECE;
      }
    };
    auto producer_issue = [&]() {
      if (pr.unit < 0) return;
      const int stage = pr.stage;
      if (pr.round > 0) mbar_wait(&empty[stage], (uint32_t)((pr.round - 1) & 1));
      double* st = ring + (size_t)stage * C3_STAGE;
      mbar_arrive_expect_tx(&full[stage], C3_STAGE * 8);
#if MHAR_C3_DPOL == 1
      const uint64_t keep = policy_evict_normal();
#else
      const uint64_t keep = policy_evict_last();
#endif
#if MHAR_C3_APOL == 1
      bulk_g2s_hint(st, pr.a, A_PIECE * 8, &full[stage], policy_evict_last());
#else
      bulk_g2s(st, pr.a, A_PIECE * 8, &full[stage]);
#endif
      bulk_g2s_hint(st + A_PIECE, pr.b0, B_PIECE * 8, &full[stage], keep);
      bulk_g2s_hint(st + A_PIECE + B_PIECE, pr.b1, B_PIECE * 8, &full[stage], keep);
      pr.a += A_PIECE;
      pr.b0 += B_PIECE;
      pr.b1 += B_PIECE;
      if (stage + 1 == C3_STAGES) {
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
      for (int q = 0; q < C3_STAGES - C3_LAG; ++q) producer_issue();
    }
    int c_stage = 0, c_phase = 0;
    long long t_main = 0, t_full = 0, t_tempty = 0, t_store = 0;
    for (int ui = 0;; ++ui) {
      if (unit_at(ui) < 0) break;
      const long long tu0 = pclock();
      double acc[8][4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int kt = 0; kt < KT; ++kt) {
        if (tid == 0) producer_issue();
        const long long tw0 = pclock();
        mbar_wait(&full[c_stage], (uint32_t)c_phase);
        if (PROF) t_full += clock64() - tw0;
        const double2* sa = reinterpret_cast<const double2*>(ring + (size_t)c_stage * C3_STAGE);
        const double2* sb = sa + A_PIECE / 2 + (wn >> 1) * (B_PIECE / 2);
        // the A fragments of one k4 step at a time (8-byte loads): with 128
        // accumulator doubles live, whole (k, k + 4) pairs would not fit the
        // MMA warps' register budget
        const double* sad = reinterpret_cast<const double*>(sa);
#pragma unroll
        for (int k8 = 0; k8 < 2; ++k8) {
          double2 bf[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[j] = sb[(k8 * 8 + (wn & 1) * 4 + j) * 32 + lane];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double af[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) af[i] = sad[((k8 * 16 + wm * 8 + i) * 32 + lane) * 2 + h];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j)
                dmma884(acc[i][j][0], acc[i][j][1], af[i], h ? bf[j].y : bf[j].x);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[c_stage]);
        if (++c_stage == C3_STAGES) {
          c_stage = 0;
          c_phase ^= 1;
        }
      }
      // hand the tile to the twin epilogue warp through TMEM buffer b: columns
      // b * 256 + wm * 128 + [32 j + 2 (2 i + e) + half] of lane quarter wn
      const int b = ui & 1;
      const long long tu1 = pclock();
      if (ui >= 2) mbar_wait(&tempty[b * C3_TB + (C3_TB > 1 ? warp : 0)], (uint32_t)(((ui >> 1) - 1) & 1));
      const long long tu2 = pclock();
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr = tmem + ((uint32_t)(wn * 32) << 16) + (uint32_t)(b * 256 + wm * 128);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t v[64];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double x = acc[i][2 * half + jj][e];
              v[(jj * 16 + i * 2 + e) * 2] = __double2loint(x);
              v[(jj * 16 + i * 2 + e) * 2 + 1] = __double2hiint(x);
            }
        tm_st64(taddr + (uint32_t)(half * 64), v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfull[b * C3_TB + (C3_TB > 1 ? warp : 0)]);
      t_main += tu1 - tu0;
      t_tempty += tu2 - tu1;
      t_store += pclock() - tu2;
    }
    if (PROF && lane == 0) {
      unsigned long long* pr = p.prof + 16 * blockIdx.x;
      atomicAdd(pr + 0, (unsigned long long)t_main);
      atomicAdd(pr + 1, (unsigned long long)t_full);
      atomicAdd(pr + 2, (unsigned long long)t_tempty);
      atomicAdd(pr + 3, (unsigned long long)t_store);
    }
  } else {
#if !defined(MHAR_C3_NO_SETMAXNREG) && !MHAR_C3_DEC_FIRST
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C3_EPI_REGS));
#endif
    // ---------------------------- epilogue warps ----------------------------
    const int twin = warp - 8;                   // MMA warp whose tile this warp reads
    const int wm = twin >> 2, wn = twin & 3;     // warp % 4 == wn: the same TMEM lane quarter
    const uint64_t stream_policy = policy_evict_first();  // the cache stream must not evict A
    long long t_wait = 0, t_work = 0;
    for (int ui = 0;; ++ui) {
      const long long u = unit_at(ui);
      if (u < 0) break;
      int64_t mt, ct;
      c3_unit(u, p, &mt, &ct);
      const int b = ui & 1;
      const long long te0 = pclock();
      mbar_wait(&tfull[b * C3_TB + (C3_TB > 1 ? twin : 0)], (uint32_t)((ui >> 1) & 1));
      const long long te1 = pclock();
      t_wait += te1 - te0;
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr = tmem + ((uint32_t)(wn * 32) << 16) + (uint32_t)(b * 256 + wm * 128);
      const int64_t cache_base =
          (((mt * p.c3_tiles + ct) * 8 + twin) * 8) * 4 * 64;  // doubles: [i(8)][j(4)][lane][2]
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        const int64_t c0 = ct * C3_BW + wn * 32 + j * 8;
        const int64_t c = c0 + 2 * (lane & 3);
        const double2 th = *reinterpret_cast<const double2*>(p.theta_prev + c);
        // the bounds as keys throughout (scan_row_key): no fp64 instruction
        // besides the slack update and the rare exact ratio
        long long hk[2], lk[2], vk[2];
        unsigned sd[2] = {0u, 0u};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          hk[e] = *(volatile long long*)(p.hi_key + c + e);
          lk[e] = *(volatile long long*)(p.lo_key + c + e);
          vk[e] = dkey(__longlong_as_double((long long)0xFFF0000000000000ULL));
        }
        const long long epsb = __double_as_longlong(p.eps_dir);
#pragma unroll
        for (int i0 = 0; i0 < 8; i0 += 2) {
          double2 so[2], ro[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int64_t base = cache_base + (((i0 + i) * 4 + j) * 32 + lane) * 2;
            so[i] = __ldcs(reinterpret_cast<const double2*>(p.S + base));
            ro[i] = __ldcs(reinterpret_cast<const double2*>(p.R + base));
          }
          // rows i0, i0 + 1 of walk group j: 2 doubles (4 columns) per row
          uint32_t v[8];
          tm_ld8(taddr + (uint32_t)(j * 32 + i0 * 4), v);
          if (j == 3 && i0 == 6) {
            // every TMEM read of buffer b is complete: the MMA warps may refill it
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b * C3_TB + (C3_TB > 1 ? twin : 0)]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double a0 = __hiloint2double((int)v[4 * i + 1], (int)v[4 * i]);
            const double a1 = __hiloint2double((int)v[4 * i + 3], (int)v[4 * i + 2]);
            const int64_t base = cache_base + (((i0 + i) * 4 + j) * 32 + lane) * 2;
            const double s0 = fma(-th.x, ro[i].x, so[i].x);
            const double s1 = fma(-th.y, ro[i].y, so[i].y);
            st_policy2(p.S + base, s0, s1, stream_policy);
            st_policy2(p.R + base, a0, a1, stream_policy);
            viol_key_update(vk[0], s0);
            viol_key_update(vk[1], s1);
            scan_row_key(s0, a0, epsb, hk[0], lk[0], sd[0]);
            scan_row_key(s1, a1, epsb, hk[1], lk[1], sd[1]);
          }
        }
        reduce_and_publish_keys(hk, lk, vk, sd, c0, lane, p);
      }
      t_work += pclock() - te1;
    }
    if (PROF && lane == 0) {
      unsigned long long* pr = p.prof + 16 * blockIdx.x;
      atomicAdd(pr + 4, (unsigned long long)t_wait);
      atomicAdd(pr + 5, (unsigned long long)t_work);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 8)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

}  // namespace mhar_dev
