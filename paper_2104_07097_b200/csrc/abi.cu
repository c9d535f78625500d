// abi.cu -- the C ABI (include/mhar_b200.h): context, device memory, and
// the per-iterate launch sequence of the MHAR engine on one B200.
//
// One iterate (reference step(), /root/reference/proj/src/sampler.cpp:235-272):
//   normals (Philox | reference streams) -> [project P H, collapse flags]
//   -> chord kernel (DMMA A_I [X|D] or A_I D + slack cache, fused bounds)
//   -> finalize (intervals, unbounded check, redraw queue)
//   -> redraw (slow path, usually empty) -> theta (+ fix-up) -> x += theta d
//   -> [reprojection every reproject_every iterates]
// All launches are queued on the context's stream without host syncs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/mhar_b200.h"
#include "chord_kernel.cuh"
#include "chord3_kernel.cuh"
#include "engine_internal.h"
#include "host_linalg.h"
#include "lp.h"
#include "step_kernels.cuh"
#include "small_kernel.cuh"
#include "chord_tc32.cuh"
#include "chord_i8.cuh"
#include "fastpath.cuh"
#include "stats_kernels.cuh"

using namespace mhar_dev;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

const char* code_name(int st) {
  switch (st) {
    case 1: return "INVALID_ARGUMENT";
    case 2: return "DIMENSION_MISMATCH";
    case 3: return "SINGULAR_MATRIX";
    case 4: return "RANK_DEFICIENT_EQ";
    case 7: return "UNBOUNDED_POLYTOPE";
    case 8: return "DIRECTION_DEGENERATE";
    case 9: return "RETRY_EXHAUSTED";
    case 12: return "NUMERICAL_FAILURE";
    default: return "ERROR";
  }
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(MHAR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// NVTX range for the host-side phases (iterate, run window, LP, MST):
// visible in Nsight Systems, a few ns when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kProfWords = 10;  // per-CTA profile words (MHAR_I8_PROFILE)

}  // namespace

struct mhar_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  mhar_options opt{};
  int64_t n = 0, m = 0, me = 0, z = 0;
  int64_t n_pad = 0, KT = 0, m_pad = 0, m_tiles = 0, z_pad = 0, ct64 = 0;
  int64_t p_rows_pad = 0;

  // device buffers
  double *A = nullptr, *b = nullptr, *X = nullptr, *D = nullptr, *H = nullptr;
  double *Xtmp = nullptr;
  double *Ppk = nullptr, *Pcm = nullptr, *AE = nullptr, *bE = nullptr, *G = nullptr;
  double *S = nullptr, *R = nullptr;
  double *theta = nullptr, *lower = nullptr, *upper = nullptr, *viol = nullptr;
  double *eqres = nullptr, *eqg = nullptr, *eqviol = nullptr, *rows = nullptr;
  double *redraw_scratch = nullptr, *x0 = nullptr, *injected_u = nullptr;
  long long *hi_key = nullptr, *lo_key = nullptr, *viol_key = nullptr;
  unsigned *sides = nullptr, *flags = nullptr, *collapsed = nullptr;
  int *redraw_list = nullptr, *redraw_count = nullptr, *attempts = nullptr;
  int *first_reject = nullptr, *first_bad = nullptr;
  unsigned long long *err = nullptr, *redraw_total = nullptr;
  unsigned* sched = nullptr;  // chord2 unit tickets (chord_kernel.cuh next_unit)
  bool c3 = false;            // incremental DMMA chord on chord3_kernel (MHAR_CHORD3=0: chord2)
  unsigned long long* c3_prof = nullptr;  // MHAR_C3_PROFILE: chord3 phase counters, 16 per CTA
  uint64_t *col_state = nullptr, *theta_state = nullptr;
  int redraw_grid = 1;
  int group_m = 16;  // chord-kernel rasterisation band (m tiles); MHAR_GROUP_M overrides
  int walk_band = 0;  // > 0: walk-tile bands (MHAR_WALK_BAND overrides)
  // walk-resident small-body path (small_kernel.cuh); Acm != null enables it
  double* Acm = nullptr;
  // fp32 variant (chord_tc32.cuh)
  float *Ahi = nullptr, *Alo = nullptr, *Dhi = nullptr, *Dlo = nullptr;
  int64_t tc_walk_tiles = 0, tc_row_tiles = 0;
  int tc_group_n = 1;   // tc32 rasterisation band (row tiles); MHAR_TC_GROUP overrides
  int tc_walk_band = 0; // tc32 walk-pair bands for large z (MHAR_TC_WALK_BAND overrides)
  int tc_a_policy = 0;  // L2 policy of the tc32 A stream (evict_normal); MHAR_TC_APOL overrides
  bool tc_f16 = true;   // fp32 variant on kind::f16 with per-row / per-walk scales (MHAR_TC_F16=0: TF32)
  int64_t tc_kt = 0;    // k stages of the fp32 variant (16 floats or 32 halves each)
  float *tc_rsc = nullptr, *tc_csc = nullptr;
  // tensor maps of the fp32 variant's operand arrays (2-CTA TMA loads)
  CUtensorMap tm_ahi{}, tm_alo{}, tm_dhi{}, tm_dlo{};
  bool tc_tma = false;
  int64_t cache_rows = 0;  // row tile of the tcgen05 cache layout (256 tc32, 64 int8)
  // int8-slice fp64 engine (chord_i8.cuh)
  uint8_t *A8 = nullptr, *D8 = nullptr;
  double *rsc = nullptr, *csc = nullptr;
  int* rexp = nullptr;
  int64_t KS = 0, i8_row_tiles = 0;
  int i8_clusters = 0;  // co-resident clusters of the int8 kernel
  int i8_group = 16;    // int8 kernel rasterisation band (row groups); MHAR_I8_GROUP overrides
  bool dmma_refresh = false;  // MHAR_DMMA_REFRESH=1: tcgen05 engines refresh with the fused DMMA pass
  // CUDA graph of one steady iterate (multi-kernel path, MHAR_NO_GRAPHS=1 disables):
  // the kernels read the Philox iterate counter from d_iter
  bool no_graphs = false, graph_capturing = false;
  bool pdl = true;  // iterate-chain kernels launched as programmatic dependents (MHAR_NO_PDL=1: off)
  unsigned long long* d_iter = nullptr;
  unsigned long long d_iter_value = ~0ull;  // what d_iter holds once queued work ran
  cudaGraphExec_t graph_exec = nullptr;
  const double* graph_X = nullptr;           // X the graph was captured with
  int64_t graph_launches = 0, graph_chord_launches = 0;
  int64_t graph_replays = 0;
  unsigned long long* tc_prof = nullptr;  // MHAR_I8_PROFILE: tcgen05 kernels' per-CTA counters
  // structure-aware paths (fastpath.cuh)
  double* diag_coef = nullptr;  // stacked diagonal blocks: per-row coefficient (m)
  int64_t diag_blocks = 0;
  bool diag_uniform = false;    // every block: one coefficient and one bound (DiagParams uc/ub)
  double diag_uc[kDiagUniMax] = {}, diag_ub[kDiagUniMax] = {};
  double* proj_g = nullptr;     // factored projection: split partials of A_E H (J x m_E x z_pad)
  double* norm_part = nullptr;  // split partials of ||d||^2 for the collapse test (J x z_pad)
  // run(): overlapped collection (second rows buffer, pinned staging, side stream)
  double* rows2 = nullptr;
  double* pinned[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
  unsigned long long* walk_err = nullptr;
  unsigned long long* walk_err_min = nullptr;  // small path: min of walk_err, kNoError between launches
  size_t small_smem = 0;
  int small_ns = 1, small_grid = 0, small_warps = SMALL_WARPS;
  int small_gw = 32;  // lanes per walk of the walk-resident kernel (small_group_width)

  // host bookkeeping
  int64_t iterations = 0;
  bool slack_valid = false;
  int64_t since_refresh = 0;
  int64_t launches = 0, chord_launches = 0, refreshes = 0;
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  std::vector<double> pending_flops;
  double chord_flops = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> event_pool;
  double chord_ms = 0.0;
  int64_t chord_timed = 0;
  std::vector<void*> allocs;
};

namespace {

template <typename T>
int dalloc(mhar_ctx* c, T** p, size_t count) {
  void* q = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess)
    return fail(MHAR_ERR_CUDA, "cudaMalloc(" + std::to_string(bytes) + " B): " +
                                   cudaGetErrorString(e));
  // Fresh allocations start zeroed; MHAR_POISON=<hex mask> instead fills the
  // allocations whose creation index is in the mask with 0xFF (NaN) bytes --
  // a debugging aid that exposes reads of never-written device memory.
  static const unsigned long long poison = [] {
    const char* e = std::getenv("MHAR_POISON");
    return e ? std::strtoull(e, nullptr, 16) : 0ull;
  }();
  const size_t idx = c->allocs.size();
  const bool bad = idx < 64 && ((poison >> idx) & 1ull);
  cudaMemsetAsync(q, bad ? 0xFF : 0, bytes, c->stream);
  c->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return 0;
}

inline int blocks_for(int64_t work, int threads, int cap) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

// A packed operand array of `floats` 4-byte words as a 2-D tensor of rows of
// 64 words, boxes of 64 x 32 (one 8 KB stage piece); the driver entry point is
// looked up at run time so the library needs no -lcuda.
bool encode_piece_map(CUtensorMap* tm, const void* base, size_t floats) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Encode>(f);
  }();
  if (!encode || floats % 64 != 0) return false;
  const cuuint64_t dims[2] = {64, floats / 64};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, 32};
  const cuuint32_t estride[2] = {1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box,
                estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_check(mhar_ctx* c, const char* what) {
  ++c->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MHAR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

#define LAUNCH_OK(c, what)                 \
  do {                                     \
    int s_ = launch_check((c), (what));    \
    if (s_) return s_;                     \
  } while (0)

void harvest_timing(mhar_ctx* c) {
  for (size_t i = 0; i < c->pending.size(); ++i) {
    auto& ev = c->pending[i];
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev.first, ev.second) == cudaSuccess) {
      c->chord_ms += ms;
      c->chord_flops += c->pending_flops[i];
      ++c->chord_timed;
    }
    c->event_pool.push_back(ev);
  }
  c->pending.clear();
  c->pending_flops.clear();
}

std::pair<cudaEvent_t, cudaEvent_t> take_events(mhar_ctx* c) {
  if (!c->event_pool.empty()) {
    auto e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  std::pair<cudaEvent_t, cudaEvent_t> e;
  cudaEventCreate(&e.first);
  cudaEventCreate(&e.second);
  return e;
}

ChordParams chord_params(mhar_ctx* c, const double* X) {
  ChordParams p;
  p.A = c->A;
  p.X = X;
  p.D = c->D;
  p.b = c->b;
  p.S = c->S;
  p.R = c->R;
  p.theta_prev = c->theta;
  p.hi_key = c->hi_key;
  p.lo_key = c->lo_key;
  p.viol_key = c->viol_key;
  p.sides = c->sides;
  p.err = c->err;
  p.m_tiles = c->m_tiles;
  p.KT = c->KT;
  p.col_tiles = c->ct64;
  p.z = c->z;
  p.eps_dir = c->opt.eps_dir;
  p.group_m = c->group_m;
  p.walk_band = c->walk_band;
  p.tc_walk_tiles = c->tc_walk_tiles;
  p.cache_rows = c->cache_rows;
  p.rate_f32 = c->Ahi != nullptr;
  p.sched = c->sched;
  p.c3_tiles = c->c3 ? c->z_pad / C3_BW : 0;
  p.prof = c->c3_prof;
  return p;
}

// Launches one kernel of the iterate chain.  With c->pdl it is a
// programmatic dependent of the kernel before it on the stream (captured
// into the iterate graph as a programmatic edge): its CTAs are scheduled
// while the predecessor drains and wait in pdl_enter (common.cuh) for the
// predecessor's completion.  Only kernels that call pdl_enter first go
// through here.
template <typename... K, typename... A>
void launch_k(mhar_ctx* c, void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, A... args) {
  if (!c->pdl) {
    kernel<<<grid, block, smem, c->stream>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// compute_lambda_intervals' stacked-diagonal fast path (fastpath.cuh)
int launch_diag(mhar_ctx* c, int mode, const double* X) {
  DiagParams p;
  p.coef = c->diag_coef;
  p.b = c->b;
  p.X = X;
  p.D = c->D;
  p.hi_key = c->hi_key;
  p.lo_key = c->lo_key;
  p.viol_key = c->viol_key;
  p.sides = c->sides;
  p.err = c->err;
  p.n = c->n;
  p.blocks = c->diag_blocks;
  p.KT = c->KT;
  p.z = c->z;
  p.eps_dir = c->opt.eps_dir;
  p.bounds = mode == CHECK ? 0 : 1;
  for (int j = 0; j < kDiagUniMax; ++j) {
    p.uc[j] = c->diag_uc[j];
    p.ub[j] = c->diag_ub[j];
  }
  // one 1024-thread CTA per SM (the register budget allows one), one wave
  // (more CTAs per SM -- 32 registers -- or more waves measured slower: more
  // spills, more cross-CTA bound atomics per walk; tools/ab_diag.sh)
  const int64_t splits = std::max<int64_t>(
      1, std::min<int64_t>(c->KT, (int64_t)c->num_sms / c->ct64));
  p.kt_per_cta = (c->KT + splits - 1) / splits;
  const dim3 grid((unsigned)c->ct64, (unsigned)((c->KT + p.kt_per_cta - 1) / p.kt_per_cta));
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (c->timing) {
    ev = take_events(c);
    cudaEventRecord(ev.first, c->stream);
  }
  if (c->diag_uniform && c->diag_blocks == 2)
    launch_k(c, diag_chord_kernel<2, true>, grid, kDiagThreads, 0, p);
  else if (c->diag_uniform && c->diag_blocks == 1)
    launch_k(c, diag_chord_kernel<1, true>, grid, kDiagThreads, 0, p);
  else if (c->diag_blocks == 2)
    launch_k(c, diag_chord_kernel<2>, grid, kDiagThreads, 0, p);
  else if (c->diag_blocks == 1)
    launch_k(c, diag_chord_kernel<1>, grid, kDiagThreads, 0, p);
  else
    launch_k(c, diag_chord_kernel<0>, grid, kDiagThreads, 0, p);
  LAUNCH_OK(c, "diag_chord_kernel");
  ++c->chord_launches;
  if (c->timing) {
    cudaEventRecord(ev.second, c->stream);
    c->pending.push_back(ev);
    c->pending_flops.push_back(4.0 * (double)c->m * (double)c->z);  // slack + rate per row
  }
  return 0;
}

int launch_chord(mhar_ctx* c, int mode, const double* X) {
  if (c->diag_coef) return launch_diag(c, mode, X);
  ChordParams p = chord_params(c, X);
  const bool fused = (mode == FUSED || mode == FUSED_STORE);
  const int64_t units = p.m_tiles * p.col_tiles;
  const int grid = (int)std::min<int64_t>(units, (fused ? 1 : 2) * (int64_t)c->num_sms);
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (c->timing) {
    ev = take_events(c);
    cudaEventRecord(ev.first, c->stream);
  }
  switch (mode) {
    case FUSED:
      chord_kernel<FUSED><<<grid, CHORD_THREADS, CHORD_SMEM, c->stream>>>(p);
      break;
    case FUSED_STORE:
      chord_kernel<FUSED_STORE><<<grid, CHORD_THREADS, CHORD_SMEM, c->stream>>>(p);
      break;
    case INCREMENTAL:
      if (c->c3) {
        const int g3 = (int)std::min<int64_t>(p.m_tiles * p.c3_tiles, c->num_sms);
        if (p.prof)
          chord3_kernel<true><<<g3, C3_THREADS, C3_SMEM, c->stream>>>(p);
        else
          chord3_kernel<false><<<g3, C3_THREADS, C3_SMEM, c->stream>>>(p);
      }
      else
        chord2_kernel<INCREMENTAL><<<grid, CHORD_THREADS, CHORD2_SMEM, c->stream>>>(p);
      break;
    case SLACK_STORE:
      chord2_kernel<SLACK_STORE><<<grid, CHORD_THREADS, CHORD2_SMEM, c->stream>>>(p);
      break;
    default:
      chord2_kernel<CHECK><<<grid, CHORD_THREADS, CHORD2_SMEM, c->stream>>>(p);
      break;
  }
  LAUNCH_OK(c, "chord_kernel");
  ++c->chord_launches;
  if (c->timing) {
    cudaEventRecord(ev.second, c->stream);
    c->pending.push_back(ev);
    // algorithmic flops of this launch: 2 m n per product column
    const double cols = (mode == FUSED || mode == FUSED_STORE) ? 2.0 * c->z : (double)c->z;
    c->pending_flops.push_back(2.0 * (double)c->m * (double)c->n * cols);
  }
  return 0;
}

// fp32 variant: incremental chord with tcgen05 3xTF32 rates.
int launch_tc32(mhar_ctx* c) {
  TcParams p;
  p.Ahi = c->Ahi;
  p.Alo = c->Alo;
  p.Dhi = c->Dhi;
  p.Dlo = c->Dlo;
  p.S = c->S;
  p.R = reinterpret_cast<float*>(c->R);
  p.theta_prev = c->theta;
  p.hi_key = c->hi_key;
  p.lo_key = c->lo_key;
  p.viol_key = c->viol_key;
  p.sides = c->sides;
  p.err = c->err;
  p.row_tiles = c->tc_row_tiles;
  p.walk_tiles = c->tc_walk_tiles;
  p.KT = c->tc_kt;
  p.rsc = c->tc_rsc;
  p.csc = c->tc_csc;
  p.m = c->m;
  p.z = c->z;
  p.eps_dir = c->opt.eps_dir;
  p.margin = c->opt.fp32_margin > 0 ? c->opt.fp32_margin : 2e-5;
  p.group_n = c->tc_group_n;
  p.walk_band = c->tc_walk_band;
  p.a_policy = c->tc_a_policy;
  p.prof = c->tc_prof;
  p.tmAhi = c->tm_ahi;
  p.tmAlo = c->tm_alo;
  p.tmDhi = c->tm_dhi;
  p.tmDlo = c->tm_dlo;
  p.use_tma = c->tc_tma ? 1 : 0;
  p.sched = c->sched + 4;  // its own ticket pair
  if (c->tc_prof) cudaMemsetAsync(c->tc_prof, 0, kProfWords * sizeof(unsigned long long) * c->num_sms, c->stream);
  const int64_t units = p.row_tiles * (p.walk_tiles / 2);  // (row tile, walk-tile pair)
  const int grid = 2 * (int)std::min<int64_t>(units, c->num_sms / 2);  // CTA pairs
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (c->timing) {
    ev = take_events(c);
    cudaEventRecord(ev.first, c->stream);
  }
  if (c->tc_f16 && c->Dlo)
    chord_tc32_kernel<true, true><<<grid, TC_THREADS, TcCfg<true>::smem, c->stream>>>(p);
  else if (c->tc_f16)
    chord_tc32_kernel<false, true><<<grid, TC_THREADS, TcCfg<false>::smem, c->stream>>>(p);
  else if (c->Dlo)
    chord_tc32_kernel<true><<<grid, TC_THREADS, TcCfg<true>::smem, c->stream>>>(p);
  else
    chord_tc32_kernel<false><<<grid, TC_THREADS, TcCfg<false>::smem, c->stream>>>(p);
  LAUNCH_OK(c, "chord_tc32_kernel");
  ++c->chord_launches;
  if (c->timing) {
    cudaEventRecord(ev.second, c->stream);
    c->pending.push_back(ev);
    c->pending_flops.push_back(2.0 * (double)c->m * (double)c->n * (double)c->z);
  }
  return 0;
}

// int8-slice fp64 engine: incremental chord with exact slice products.
int launch_i8(mhar_ctx* c) {
  I8Params p;
  p.A8 = c->A8;
  p.rsc = c->rsc;
  p.D8 = c->D8;
  p.csc = c->csc;
  p.S = c->S;
  p.R = c->R;
  p.theta_prev = c->theta;
  p.hi_key = c->hi_key;
  p.lo_key = c->lo_key;
  p.viol_key = c->viol_key;
  p.sides = c->sides;
  p.err = c->err;
  p.row_tiles = c->i8_row_tiles;
  p.walk_tiles = c->tc_walk_tiles;
  p.sched = c->sched + 2;  // its own ticket pair (chord2 uses sched[0..1])
  p.group = c->i8_group;
  p.KS = c->KS;
  p.z = c->z;
  p.eps_dir = c->opt.eps_dir;
  p.prof = c->tc_prof;
  if (c->tc_prof) cudaMemsetAsync(c->tc_prof, 0, kProfWords * sizeof(unsigned long long) * c->num_sms, c->stream);
  const int64_t units = p.row_tiles / I8_PAIRS * (p.walk_tiles / 2);
  const int grid = I8_CL * (int)std::min<int64_t>(units, c->i8_clusters);
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (c->timing) {
    ev = take_events(c);
    cudaEventRecord(ev.first, c->stream);
  }
  chord_i8_kernel<<<grid, I8_THREADS, I8_SMEM, c->stream>>>(p);
  if (cudaPeekAtLastError() != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, chord_i8_kernel);
    const cudaError_t e = cudaGetLastError();
    return fail(MHAR_ERR_CUDA, std::string("chord_i8_kernel: ") + cudaGetErrorString(e) +
                                   " (regs " + std::to_string(fa.numRegs) + ", max threads " +
                                   std::to_string(fa.maxThreadsPerBlock) + ", local " +
                                   std::to_string(fa.localSizeBytes) + " B, max dyn smem " +
                                   std::to_string(fa.maxDynamicSharedSizeBytes) + ")");
  }
  LAUNCH_OK(c, "chord_i8_kernel");
  ++c->chord_launches;
  if (c->timing) {
    cudaEventRecord(ev.second, c->stream);
    c->pending.push_back(ev);
    c->pending_flops.push_back(2.0 * (double)c->m * (double)c->n * (double)c->z);
  }
  return 0;
}

int launch_finalize(mhar_ctx* c, bool queue_redraws, bool advance_streams) {
  FinalizeParams fp;
  fp.hi_key = c->hi_key;
  fp.lo_key = c->lo_key;
  fp.viol_key = c->viol_key;
  fp.sides = c->sides;
  fp.collapsed = c->me > 0 ? c->collapsed : nullptr;
  fp.lower = c->lower;
  fp.upper = c->upper;
  fp.viol = c->viol;
  fp.flags = c->flags;
  fp.redraw_list = queue_redraws ? c->redraw_list : nullptr;
  fp.redraw_count = c->redraw_count;
  fp.err = c->err;
  fp.col_state = (advance_streams && c->opt.rng == MHAR_RNG_REFERENCE) ? c->col_state : nullptr;
  fp.draws_per_walk = 2 * ((c->n + 1) / 2);
  fp.z = c->z;
  launch_k(c, finalize_kernel, blocks_for(c->z, 256, 1 << 20), 256, 0, fp);
  LAUNCH_OK(c, "finalize_kernel");
  return 0;
}

int launch_normals(mhar_ctx* c, double* out) {
  RngParams rp;
  rp.seed = c->opt.seed;
  rp.iterate = (uint64_t)c->iterations;
  rp.iter_dev = c->graph_capturing ? c->d_iter : nullptr;
  rp.chain_offset = c->opt.chain_offset;
  rp.n = c->n;
  rp.z = c->z;
  rp.KT = c->KT;
  rp.mode = c->opt.rng;
  rp.col_state = c->col_state;
  const int64_t work = c->ct64 * c->KT * 16 * 32;
  launch_k(c, normals_kernel, blocks_for(work, 256, c->num_sms * 16), 256, 0, rp, out,
           (const unsigned long long*)c->err);
  LAUNCH_OK(c, "normals_kernel");
  return 0;
}

// D = P H and collapse flags (sampler.cpp:244-250).
int launch_projection(mhar_ctx* c) {
  // per-walk reductions as split partials over (walk tile, k range) CTAs
  // (fastpath.cuh): deterministic, independent of z and the sharding
  const int64_t J = dot_splits(c->KT);
  const dim3 dgrid((unsigned)c->ct64, (unsigned)J);
  if (c->proj_g) {
    // factored: D = H - A_E' (G (A_E H)), O(m_E n z)
#define MHAR_PROJ_ME(ME)                                                                       \
  case ME:                                                                                     \
    launch_k(c, proj_dot_kernel<ME>, dgrid, B_PIECE, 0, (const double*)c->AE,                \
             (const double*)c->H, c->n, c->KT, c->z_pad, c->proj_g,                            \
             (const unsigned long long*)c->err);                                               \
    LAUNCH_OK(c, "proj_dot_kernel");                                                           \
    launch_k(c, proj_apply_kernel<ME>, dgrid, B_PIECE, 0, (const double*)c->AE,              \
             (const double*)c->G, (const double*)c->H, c->D, (const double*)c->proj_g, c->n,   \
             c->z, c->KT, c->z_pad, c->norm_part, (const unsigned long long*)c->err);           \
    LAUNCH_OK(c, "proj_apply_kernel");                                                         \
    break;
    switch (c->me) {
      MHAR_PROJ_ME(1)
      MHAR_PROJ_ME(2)
      MHAR_PROJ_ME(3)
      MHAR_PROJ_ME(4)
      default:
        return fail(MHAR_ERR_INVALID_ARGUMENT, "factored projection: m_E out of range");
    }
#undef MHAR_PROJ_ME
  } else {
    dim3 grid((unsigned)(c->p_rows_pad / BM), (unsigned)c->ct64);
    project_kernel<<<grid, 256, 0, c->stream>>>(c->Ppk, c->H, c->D, c->n, c->KT, c->err);
    LAUNCH_OK(c, "project_kernel");
    launch_k(c, norm_part_kernel, dgrid, B_PIECE, 0, (const double*)c->D, c->n, c->z, c->KT,
             c->z_pad, c->norm_part, (const unsigned long long*)c->err);
    LAUNCH_OK(c, "norm_part_kernel");
  }
  launch_k(c, collapse_final_kernel, blocks_for(c->z * 32, 256, 1 << 20), 256, 0,
           (const double*)c->norm_part, J, c->z, c->z_pad, c->collapsed,
           (const unsigned long long*)c->err);
  LAUNCH_OK(c, "collapse_final_kernel");
  return 0;
}

int launch_redraw(mhar_ctx* c) {
  RedrawParams rp;
  rp.A = c->A;
  rp.b = c->b;
  rp.X = c->X;
  rp.D = c->D;
  rp.P = c->me > 0 ? c->Pcm : nullptr;
  rp.R = (c->opt.slack_mode == MHAR_SLACK_INCREMENTAL) ? c->R : nullptr;
  rp.ct64 = c->ct64;
  rp.tc_walk_tiles = c->tc_walk_tiles;
  rp.c3_tiles = c->c3 ? c->z_pad / C3_BW : 0;
  rp.cache_rows = c->cache_rows;
  rp.rate_f32 = c->Ahi != nullptr;
  rp.scratch = c->redraw_scratch;
  rp.lower = c->lower;
  rp.upper = c->upper;
  rp.flags = c->flags;
  rp.redraw_list = c->redraw_list;
  rp.redraw_count = c->redraw_count;
  rp.attempts = c->attempts;
  rp.redraw_total = c->redraw_total;
  rp.err = c->err;
  rp.seed = c->opt.seed;
  rp.iterate = (uint64_t)c->iterations;
  rp.iter_dev = c->graph_capturing ? c->d_iter : nullptr;
  rp.chain_offset = c->opt.chain_offset;
  rp.col_state = c->col_state;
  rp.mode = c->opt.rng;
  rp.n = c->n;
  rp.m = c->m;
  rp.KT = c->KT;
  rp.eps_dir = c->opt.eps_dir;
  launch_k(c, redraw_kernel, c->redraw_grid, 256, 0, rp);
  LAUNCH_OK(c, "redraw_kernel");
  return 0;
}

ThetaParams theta_params(mhar_ctx* c, const double* injected_u) {
  ThetaParams tp;
  tp.lower = c->lower;
  tp.upper = c->upper;
  tp.flags = c->flags;
  tp.theta = c->theta;
  tp.err = c->err;
  tp.seed = c->opt.seed;
  tp.iterate = (uint64_t)c->iterations;
  tp.iter_dev = c->graph_capturing ? c->d_iter : nullptr;
  tp.chain_offset = c->opt.chain_offset;
  tp.z = c->z;
  tp.mode = c->opt.rng;
  tp.theta_state = c->theta_state;
  tp.first_reject = c->first_reject;
  tp.injected_u = injected_u;
  return tp;
}

int launch_theta_and_move(mhar_ctx* c, const double* injected_u) {
  ThetaParams tp = theta_params(c, injected_u);
  launch_k(c, theta_kernel, blocks_for(c->z, 256, 1 << 20), 256, 0, tp);
  LAUNCH_OK(c, "theta_kernel");
  if (!injected_u && c->opt.rng == MHAR_RNG_REFERENCE) {
    launch_k(c, theta_fixup_kernel, 1, 1, 0, tp);
    LAUNCH_OK(c, "theta_fixup_kernel");
  }
  const int64_t total2 = c->z_pad * c->KT * BK / 2;
  launch_k(c, axpy_kernel, blocks_for(total2, 256, c->num_sms * 16), 256, 0, c->X,
           (const double*)c->D, (const double*)c->theta, total2, c->KT,
           (const unsigned long long*)c->err);
  LAUNCH_OK(c, "axpy_kernel");
  return 0;
}

// reproject_points (projection.cpp:53-60) on the packed state.
int launch_reproject(mhar_ctx* c) {
  const int64_t mz = c->me * c->z;
  eq_residual_kernel<<<blocks_for(mz, 256, 1 << 30), 256, 0, c->stream>>>(
      c->AE, c->bE, c->X, c->me, c->n, c->z, c->KT, c->eqres);
  LAUNCH_OK(c, "eq_residual_kernel");
  eq_gram_kernel<<<blocks_for(mz, 256, 1 << 30), 256, 0, c->stream>>>(c->G, c->eqres, c->me,
                                                                       c->z, c->eqg);
  LAUNCH_OK(c, "eq_gram_kernel");
  eq_correct_kernel<<<blocks_for(c->n * c->z, 256, 1 << 30), 256, 0, c->stream>>>(
      c->AE, c->eqg, c->X, c->me, c->n, c->z, c->KT);
  LAUNCH_OK(c, "eq_correct_kernel");
  c->slack_valid = false;
  return 0;
}

// One iterate of every walk.  injected_h (device, packed) / injected_u
// (device) replace the RNG for the test hook.
int enqueue_iterate(mhar_ctx* c, int64_t reproject_every, bool injected) {
  NvtxRange range(injected ? "mhar.iterate.injected" : "mhar.iterate");
  CK(cudaMemsetAsync(c->redraw_count, 0, sizeof(int), c->stream));
  if (!injected) {
    int s = launch_normals(c, c->me > 0 ? c->H : c->D);
    if (s) return s;
  }
  if (c->me > 0) {
    int s = launch_projection(c);
    if (s) return s;
  }
  int mode = FUSED;
  if (!injected && c->opt.slack_mode == MHAR_SLACK_INCREMENTAL) {
    const int64_t every = c->opt.refresh_every > 0 ? c->opt.refresh_every : 128;
    if (!c->slack_valid || c->since_refresh >= every) {
      mode = FUSED_STORE;
      c->slack_valid = true;
      c->since_refresh = 0;
      ++c->refreshes;
    } else {
      mode = INCREMENTAL;
    }
    ++c->since_refresh;
  } else if (injected) {
    c->slack_valid = false;
  }
  int s = 0;
  if (c->Ahi) {
    // fp32 variant: the tensor cores see D_hi + D_lo; D becomes that direction
    const int64_t total = c->z_pad * c->KT * BK;
    if (c->tc_f16) {
      tc16_split_d_kernel<<<(unsigned)((c->z_pad * 32 + 255) / 256), 256, 0, c->stream>>>(
          c->D, c->n, c->z_pad, c->KT, c->tc_kt, reinterpret_cast<__half*>(c->Dhi),
          reinterpret_cast<__half*>(c->Dlo), c->tc_csc, c->err);
      LAUNCH_OK(c, "tc16_split_d_kernel");
    } else {
      tc_split_d_kernel<<<blocks_for(total, 256, c->num_sms * 16), 256, 0, c->stream>>>(
          c->D, c->n, c->z_pad, c->KT, c->Dhi, c->Dlo, c->err);
      LAUNCH_OK(c, "tc_split_d_kernel");
    }
  }
  if (c->A8) {
    // int8-slice engine: per-walk fixed point, slices; D becomes the quantised direction
    i8_split_d_kernel<<<(unsigned)c->ct64, 256, 0, c->stream>>>(c->D, c->n, c->KT, c->KS, c->D8,
                                                                 c->csc, c->err);
    LAUNCH_OK(c, "i8_split_d_kernel");
  }
  if (c->A8 && injected) {
    // test hook: exact fp64 slack of X into the cache, then the slice rates with theta = 0
    if ((s = launch_chord(c, FUSED_STORE, c->X))) return s;
    fill_keys_kernel<<<blocks_for(c->z_pad, 256, 1 << 20), 256, 0, c->stream>>>(
        c->hi_key, c->lo_key, c->viol_key, c->sides, c->z_pad);
    LAUNCH_OK(c, "fill_keys_kernel");
    CK(cudaMemsetAsync(c->theta, 0, sizeof(double) * c->z_pad, c->stream));
    s = launch_i8(c);
  } else if ((c->A8 || c->Ahi) && mode == FUSED_STORE && !c->dmma_refresh) {
    // refresh of a tcgen05 engine: the fp64 slack from A x alone on DMMA
    // (half the fused pass), then the engine's own rates and chord with
    // theta_prev = 0
    if ((s = launch_chord(c, SLACK_STORE, c->X))) return s;
    CK(cudaMemsetAsync(c->theta, 0, sizeof(double) * c->z_pad, c->stream));
    s = c->A8 ? launch_i8(c) : launch_tc32(c);
  } else if (c->A8 && mode == INCREMENTAL) {
    s = launch_i8(c);
  } else if (c->Ahi && injected) {
    // test hook of the fp32 path: exact fp64 slack of X into the cache, the
    // chord of that pass discarded, then the tensor-core rates with theta = 0
    if ((s = launch_chord(c, FUSED_STORE, c->X))) return s;
    fill_keys_kernel<<<blocks_for(c->z_pad, 256, 1 << 20), 256, 0, c->stream>>>(
        c->hi_key, c->lo_key, c->viol_key, c->sides, c->z_pad);
    LAUNCH_OK(c, "fill_keys_kernel");
    CK(cudaMemsetAsync(c->theta, 0, sizeof(double) * c->z_pad, c->stream));
    s = launch_tc32(c);
  } else if (c->Ahi && mode == INCREMENTAL) {
    s = launch_tc32(c);
  } else {
    s = launch_chord(c, mode, c->X);
  }
  if (s) return s;
  s = launch_finalize(c, !injected, !injected);
  if (s) return s;
  if (!injected) {
    s = launch_redraw(c);
    if (s) return s;
  }
  s = launch_theta_and_move(c, injected ? c->injected_u : nullptr);
  if (s) return s;
  ++c->iterations;
  if (!injected && c->me > 0 && reproject_every > 0 && c->iterations % reproject_every == 0) {
    s = launch_reproject(c);
    if (s) return s;
  }
  return 0;
}

// A steady iterate: the same kernel chain as the last one -- no slack
// refresh due, no reprojection after it.
bool steady_iterate(const mhar_ctx* c, int64_t reproject_every) {
  if (c->opt.slack_mode == MHAR_SLACK_INCREMENTAL) {
    const int64_t every = c->opt.refresh_every > 0 ? c->opt.refresh_every : 128;
    if (!c->slack_valid || c->since_refresh >= every) return false;
  }
  return !(c->me > 0 && reproject_every > 0 && (c->iterations + 1) % reproject_every == 0);
}

void drop_graph(mhar_ctx* c) {
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  c->graph_exec = nullptr;
}

// One steady iterate as a CUDA-graph replay: the launch-bound part of the
// multi-kernel path (7-10 kernels of a few microseconds each on mid-size
// bodies) costs one graph launch on the host.  The graph is captured from
// enqueue_iterate itself on first use; its kernels take the Philox counter
// from d_iter, which the graph's last node advances.
int graph_iterate(mhar_ctx* c) {
  if (c->graph_exec && c->graph_X != c->X) drop_graph(c);  // set_state swapped the state buffer
  if (!c->graph_exec) {
    const int64_t it0 = c->iterations, sr0 = c->since_refresh, l0 = c->launches,
                  cl0 = c->chord_launches;
    mhar_dev::iter_set_kernel<<<1, 1, 0, c->stream>>>(c->d_iter, (unsigned long long)it0);
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      c->no_graphs = true;
      return enqueue_iterate(c, 0, false);
    }
    c->graph_capturing = true;
    int s = enqueue_iterate(c, 0, false);
    if (!s) launch_k(c, mhar_dev::iter_inc_kernel, 1, 1, 0, c->d_iter);
    c->graph_capturing = false;
    const cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
    cudaGraphExec_t ex = nullptr;
    const bool ok = !s && ec == cudaSuccess && g &&
                    cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    c->graph_launches = c->launches - l0;
    c->graph_chord_launches = c->chord_launches - cl0;
    // the capture ran enqueue_iterate's host bookkeeping; undo it, the replay
    // below applies it
    c->iterations = it0;
    c->since_refresh = sr0;
    c->launches = l0;
    c->chord_launches = cl0;
    cudaGetLastError();
    if (!ok) {
      if (ex) cudaGraphExecDestroy(ex);
      c->no_graphs = true;  // not capturable here: the launch-per-kernel path
      return s ? s : enqueue_iterate(c, 0, false);
    }
    c->graph_exec = ex;
    c->graph_X = c->X;
    c->d_iter_value = (unsigned long long)it0;
  }
  if (c->d_iter_value != (unsigned long long)c->iterations) {
    mhar_dev::iter_set_kernel<<<1, 1, 0, c->stream>>>(c->d_iter,
                                                      (unsigned long long)c->iterations);
    c->d_iter_value = (unsigned long long)c->iterations;
  }
  CK(cudaGraphLaunch(c->graph_exec, c->stream));
  ++c->graph_replays;
  ++c->iterations;
  ++c->d_iter_value;
  if (c->opt.slack_mode == MHAR_SLACK_INCREMENTAL) ++c->since_refresh;
  c->launches += c->graph_launches;
  c->chord_launches += c->graph_chord_launches;
  return 0;
}

// `iters` iterates of every walk: one walk-resident launch for small bodies,
// else the per-iterate kernel chain (steady iterates replayed as a CUDA graph
// when a call runs several and no per-launch timing is requested).
int advance(mhar_ctx* c, int64_t iters, int64_t reproject_every) {
  if (iters <= 0) return 0;
  if (!c->Acm) {
    const bool graphs = !c->no_graphs && !c->timing && iters >= 4 && c->d_iter;
    for (int64_t i = 0; i < iters; ++i) {
      const int s = graphs && steady_iterate(c, reproject_every)
                        ? graph_iterate(c)
                        : enqueue_iterate(c, reproject_every, false);
      if (s) return s;
    }
    return 0;
  }
  SmallParams sp;
  sp.A = c->Acm;
  sp.b = c->b;
  sp.P = c->me > 0 ? c->Pcm : nullptr;
  sp.AE = c->AE;
  sp.bE = c->bE;
  sp.G = c->G;
  sp.X = c->X;
  sp.n = c->n;
  sp.m = c->m;
  sp.me = c->me;
  sp.z = c->z;
  sp.KT = c->KT;
  sp.seed = c->opt.seed;
  sp.chain_offset = c->opt.chain_offset;
  sp.it0 = c->iterations;
  sp.iters = iters;
  sp.reproject_every = c->me > 0 ? reproject_every : 0;
  sp.eps_dir = c->opt.eps_dir;
  sp.redraw_total = c->redraw_total;
  sp.err = c->err;
  sp.walk_err = c->walk_err;
  sp.err_min = c->walk_err_min;
  sp.ns = c->small_ns;
  sp.coef = c->diag_coef;
  sp.diag_blocks = c->diag_blocks;
  sp.factored = c->proj_g != nullptr ? 1 : 0;
  switch (c->small_gw) {
    case 4: small_kernel<4><<<c->small_grid, 32 * c->small_warps, c->small_smem, c->stream>>>(sp); break;
    case 8: small_kernel<8><<<c->small_grid, 32 * c->small_warps, c->small_smem, c->stream>>>(sp); break;
    case 16: small_kernel<16><<<c->small_grid, 32 * c->small_warps, c->small_smem, c->stream>>>(sp); break;
    default: small_kernel<32><<<c->small_grid, 32 * c->small_warps, c->small_smem, c->stream>>>(sp);
  }
  LAUNCH_OK(c, "small_kernel");
  small_error_kernel<<<1, 256, 0, c->stream>>>(c->walk_err, c->z, c->walk_err_min, c->err);
  LAUNCH_OK(c, "small_error_kernel");
  c->iterations += iters;
  c->slack_valid = false;
  return 0;
}

// Decodes the device error word into a status (and message).
int read_error(mhar_ctx* c, int64_t* walk) {
  unsigned long long w = kNoError;
  CK(cudaMemcpyAsync(&w, c->err, sizeof(w), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->timing) harvest_timing(c);
  if (w == kNoError) return 0;
  // The failing iterate may have written S_t / R_t (chord kernel) while theta
  // and X stayed at t-1 (theta/axpy return early on the error word): the
  // incremental cache no longer describes X, so the next pass refreshes it
  // from a fresh product, and the captured graph (which assumes a valid
  // cache) is dropped.
  c->slack_valid = false;
  drop_graph(c);
  const int status = (int)(w & 0xFF);
  const int64_t k = (int64_t)((w >> 8) & ((1ULL << 48) - 1));
  if (walk) *walk = k;
  std::string what;
  switch (status) {
    case ST_UNBOUNDED:
      what = "chord is unbounded on one side; the polytope is not bounded";
      break;
    case ST_RETRY_EXHAUSTED:
      what = "no usable direction after 16 redraws";
      break;
    case ST_NUMERICAL:
      what = "walk left the polytope at a collection";
      break;
    default:
      what = "device error";
  }
  return fail(status, std::string(code_name(status)) + ": walk " +
                          std::to_string(k + c->opt.chain_offset) + ": " + what);
}

int clear_error(mhar_ctx* c) {
  CK(cudaMemsetAsync(c->err, 0xFF, sizeof(unsigned long long), c->stream));
  return 0;
}

// A caught device error (read_error) invalidated the slack cache there; an
// error word cleared without being read (set_state after a failed step whose
// status the caller ignored) must not leave a stale cache either.
int clear_error_and_cache(mhar_ctx* c) {
  unsigned long long w = kNoError;
  CK(cudaMemcpyAsync(&w, c->err, sizeof(w), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (w != kNoError) {
    c->slack_valid = false;
    drop_graph(c);
  }
  return clear_error(c);
}

int upload_state_host(mhar_ctx* c, const double* x_host, double* dst) {
  double* tmp = c->rows;  // n x z staging
  CK(cudaMemcpyAsync(tmp, x_host, sizeof(double) * c->n * c->z, cudaMemcpyHostToDevice,
                     c->stream));
  const int64_t total = c->z_pad * c->KT * BK;
  pack_b_kernel<<<blocks_for(total, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      tmp, c->n, c->z, c->z_pad, c->KT, dst);
  LAUNCH_OK(c, "pack_b_kernel");
  return 0;
}

int reset_streams(mhar_ctx* c) {
  if (c->opt.rng != MHAR_RNG_REFERENCE) return 0;
  std::vector<uint64_t> st(c->z);
  for (int64_t k = 0; k < c->z; ++k) st[k] = stream_init(c->opt.seed, (uint64_t)(c->opt.chain_offset + k));
  const uint64_t th = stream_init(c->opt.seed, ~0ULL);  // WalkRng::kThetaStreamId
  CK(cudaMemcpyAsync(c->col_state, st.data(), sizeof(uint64_t) * c->z, cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->theta_state, &th, sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

// MHAR_I8_PROFILE=1 debugging aid: the last tcgen05 chord launch's per-CTA
// counters (chord_tc32.cuh / chord_i8.cuh `prof`), printed at ctx_destroy.
// Per CTA b: [8b+0] MMA-issuer cycles, [8b+1..3] its waits on TMEM drain /
// own slot / peer slot, [8b+4] producer waits on free slots, [8b+5..7]
// epilogue drain / stream / idle cycles; [8N + 2b, +1] %globaltimer at entry
// and exit (chord_tc32 only).
void report_tc_profile(mhar_ctx* c) {
  const int N = c->num_sms;
  std::vector<unsigned long long> h(kProfWords * (size_t)N);
  if (cudaMemcpy(h.data(), c->tc_prof, h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  unsigned long long in_lo = ~0ull, in_hi = 0, out_lo = ~0ull, out_hi = 0;
  for (int b = 0; b < N; ++b) {
    const unsigned long long gi = h[8 * N + 2 * b], go = h[8 * N + 2 * b + 1];
    if (!gi) continue;
    in_lo = std::min(in_lo, gi);
    in_hi = std::max(in_hi, gi);
    out_lo = std::min(out_lo, go);
    out_hi = std::max(out_hi, go);
  }
  if (out_hi)
    std::fprintf(stderr, "[tcgen05 profile] CTA entry spread %.3f ms, exit spread %.3f ms, "
                 "first entry -> last exit %.3f ms\n", (in_hi - in_lo) * 1e-6,
                 (out_hi - out_lo) * 1e-6, (out_hi - in_lo) * 1e-6);
  double w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int leaders = 0;
  for (int b = 0; b < N; b += 2) {
    if (!h[8 * b]) continue;
    for (int k = 0; k < 8; ++k) w[k] += (double)h[8 * b + k];
    ++leaders;
  }
  if (!leaders) return;
  const double t = w[0];
  std::fprintf(stderr,
               "[tcgen05 profile] leaders %d: %.3g cycles each; MMA issuer waits: TMEM drain %.1f%%, "
               "own slot %.1f%%, peer slot %.1f%%; producer waits for free slots %.1f%%; "
               "epilogue: drain %.1f%%, stream %.1f%%, idle %.1f%%\n",
               leaders, t / leaders, 100 * w[1] / t, 100 * w[2] / t, 100 * w[3] / t, 100 * w[4] / t,
               100 * w[5] / t, 100 * w[6] / t, 100 * w[7] / t);
}

}  // namespace

// ===========================================================================
extern "C" {

void mhar_default_options(mhar_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->z = 1;
  o->eps_dir = 1e-11;
  o->eps_feas = 1e-9;
  o->rng = MHAR_RNG_PHILOX;
  o->slack_mode = MHAR_SLACK_INCREMENTAL;
  o->refresh_every = 128;
  o->device = 0;
  o->small_path = 1;
}

const char* mhar_last_error(void) { return g_last_error.c_str(); }
const char* mhar_version(void) { return "mhar_b200 0.1 (sm_100a, fp64 DMMA)"; }

int mhar_device_count(int* count) {
  CK(cudaGetDeviceCount(count));
  return 0;
}

int mhar_compute_projection(const double* a_eq, int64_t m_eq, int64_t n, double* p, double* g) {
  if (!a_eq || !p || !g || n < 1) return fail(MHAR_ERR_INVALID_ARGUMENT, "compute_projection: null argument");
  std::string msg;
  const int st = mhar_host::compute_projection(a_eq, m_eq, n, p, g, &msg);
  if (st) return fail(st, std::string(code_name(st)) + ": " + msg);
  return 0;
}

int mhar_ctx_create(const mhar_polytope* p, const double* projector, const double* gram_inverse,
                    const mhar_options* opt, mhar_ctx** out) {
  if (!p || !opt || !out) return fail(MHAR_ERR_INVALID_ARGUMENT, "ctx_create: null argument");
  *out = nullptr;
  if (p->n < 1 || p->m_in < 1 || p->m_eq < 0 || !p->a_in || !p->b_in)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "ctx_create: polytope needs n >= 1 and m_in >= 1");
  if (p->m_eq > 0 && (!p->a_eq || !p->b_eq))
    return fail(MHAR_ERR_INVALID_ARGUMENT, "ctx_create: a_eq/b_eq missing");
  if (opt->z < 1) return fail(MHAR_ERR_INVALID_ARGUMENT, "config: z must be >= 1");
  if (!(opt->eps_dir > 0.0)) return fail(MHAR_ERR_INVALID_ARGUMENT, "config: eps_dir must be > 0");
  if (!(opt->eps_feas > 0.0)) return fail(MHAR_ERR_INVALID_ARGUMENT, "config: eps_feas must be > 0");
  if (opt->rng != MHAR_RNG_PHILOX && opt->rng != MHAR_RNG_REFERENCE)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "options: unknown rng");
  if (opt->precision != 0 && opt->precision != 32 && opt->precision != 64)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "options: precision must be 64 or 32");

  if (opt->fp32_direction != MHAR_FP32_DIR_SPLIT && opt->fp32_direction != MHAR_FP32_DIR_ROUNDED)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "options: unknown fp32_direction");
  if (opt->f64_engine != MHAR_F64_DMMA && opt->f64_engine != MHAR_F64_INT8)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "options: unknown f64_engine");
  if (opt->f64_engine == MHAR_F64_INT8 && opt->precision != 32 && round_up(p->n, I8_BK) > I8_MAX_K)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "options: the int8-slice engine needs n <= 4608");
  // MHAR_F64_ENGINE=int8 selects the int8-slice engine for every eligible
  // context (n <= 4608, fp64) without code changes -- e.g. for the C++ drop-in
  const char* env_engine = std::getenv("MHAR_F64_ENGINE");
  const bool i8 = opt->precision != 32 &&
                  (opt->f64_engine == MHAR_F64_INT8 ||
                   (env_engine && std::strcmp(env_engine, "int8") == 0 &&
                    round_up(p->n, I8_BK) <= I8_MAX_K));

  mhar_ctx* c = new mhar_ctx();
  c->opt = *opt;
  c->dmma_refresh = std::getenv("MHAR_DMMA_REFRESH") != nullptr;
  const bool fp32 = opt->precision == 32;
  const bool tiles = fp32 || i8;  // tcgen05 kernels: CTA-pair walk tiles, tile cache layout
  if (tiles) {
    // the fp32 variant is the incremental tensor-core path (fp64 refreshes)
    c->opt.slack_mode = MHAR_SLACK_INCREMENTAL;
    c->opt.small_path = 0;
  }
  // stacked diagonal blocks (sampler.cpp:47-71): every row's single nonzero at
  // column row % n -> the elementwise chord path, no slack cache needed
  std::vector<double> diag_coef;
  if (!tiles && p->m_in % p->n == 0) {
    diag_coef.resize(p->m_in);
    bool ok = true;
    for (int64_t col = 0; col < p->n && ok; ++col)
      for (int64_t i = 0; i < p->m_in; ++i) {
        const double v = p->a_in[i + col * p->m_in];
        if (i % p->n == col) {
          if (v == 0.0) {
            ok = false;
            break;
          }
          diag_coef[i] = v;
        } else if (v != 0.0) {
          ok = false;
          break;
        }
      }
    if (ok && std::getenv("MHAR_NO_FASTPATH") == nullptr)
      c->opt.slack_mode = MHAR_SLACK_RECOMPUTE;  // one elementwise pass is cheaper than a cache
    else
      diag_coef.clear();
  }
  // factored projection H - A_E' G A_E H for few equalities (fastpath.cuh); the
  // reference-stream mode at small n keeps the dense P H of the oracle
  const bool factored = p->m_eq >= 1 && p->m_eq <= kMaxFactorEq &&
                        (p->n >= 256 || opt->rng == MHAR_RNG_PHILOX) &&
                        std::getenv("MHAR_NO_FASTPATH") == nullptr;
  c->device = opt->device;
  c->n = p->n;
  c->m = p->m_in;
  c->me = p->m_eq;
  c->z = opt->z;
  auto bail = [&](int st) {
    mhar_ctx_destroy(c);
    return st;
  };
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) {
    delete c;
    return fail(MHAR_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(MHAR_ERR_CUDA, "cudaStreamCreate failed");
  }

  c->n_pad = round_up(c->n, BK);
  c->KT = c->n_pad / BK;
  c->m_pad = round_up(c->m, fp32 ? TC_N : i8 ? (int64_t)I8_N * I8_PAIRS : BM);
  c->m_tiles = c->m_pad / BM;
  // the incremental DMMA chord runs chord3_kernel (128-walk units, TMEM
  // hand-off to separate epilogue warps) when the dimension is large enough
  // for the unit's MMA time to cover its epilogue (n_pad >= 384; measured,
  // profiles/c3_sweep_r02.jsonl and bench: n = 500 / 1000 / 2000 gain 3.8 /
  // 3.4 / 1.7 points of DMMA peak, n = 384 breaks even, n <= 256 loses),
  // else chord2 (64-walk units, in-register epilogue).  MHAR_CHORD3=0 / 1
  // forces either.
  {
    const char* c3e = std::getenv("MHAR_CHORD3");
    const bool eligible = !tiles && diag_coef.empty() && c->opt.slack_mode == MHAR_SLACK_INCREMENTAL;
    c->c3 = eligible && (c3e ? std::atoi(c3e) != 0 : c->n_pad >= 384);
  }
  c->z_pad = round_up(c->z, tiles ? 2 * TC_M : c->c3 ? C3_BW : 64);  // whole kernel walk tiles
  c->ct64 = c->z_pad / 64;
  if (tiles) {
    c->tc_row_tiles = c->m_pad / TC_N;
    c->tc_walk_tiles = c->z_pad / TC_M;
    c->cache_rows = fp32 ? TC_N : I8_N;
  }
  if (i8) {
    c->KS = round_up(c->n, I8_BK) / I8_BK;
    c->i8_row_tiles = c->m_pad / I8_N;
  }
  c->p_rows_pad = round_up(c->n, BM);

  const size_t nzp = (size_t)c->z_pad * c->n_pad;
  int st = 0;
  if ((st = dalloc(c, &c->A, (size_t)c->m_pad * c->n_pad)) ||
      (st = dalloc(c, &c->b, c->m_pad)) || (st = dalloc(c, &c->X, nzp)) ||
      (st = dalloc(c, &c->D, nzp)) || (st = dalloc(c, &c->theta, c->z_pad)) ||
      (st = dalloc(c, &c->lower, c->z_pad)) || (st = dalloc(c, &c->upper, c->z_pad)) ||
      (st = dalloc(c, &c->viol, c->z_pad)) || (st = dalloc(c, &c->eqviol, c->z_pad)) ||
      (st = dalloc(c, &c->rows, std::max<size_t>((size_t)c->n * c->z, (size_t)c->m * 1))) ||
      (st = dalloc(c, &c->hi_key, c->z_pad)) || (st = dalloc(c, &c->lo_key, c->z_pad)) ||
      (st = dalloc(c, &c->viol_key, c->z_pad)) || (st = dalloc(c, &c->sides, c->z_pad)) ||
      (st = dalloc(c, &c->flags, c->z_pad)) || (st = dalloc(c, &c->collapsed, c->z_pad)) ||
      (st = dalloc(c, &c->redraw_list, c->z_pad)) || (st = dalloc(c, &c->redraw_count, 1)) ||
      (st = dalloc(c, &c->attempts, c->z_pad)) || (st = dalloc(c, &c->first_reject, 1)) ||
      (st = dalloc(c, &c->first_bad, 1)) || (st = dalloc(c, &c->err, 1)) ||
      (st = dalloc(c, &c->redraw_total, 1)) || (st = dalloc(c, &c->col_state, c->z_pad)) ||
      (st = dalloc(c, &c->theta_state, 1)) || (st = dalloc(c, &c->x0, c->n)) ||
      (st = dalloc(c, &c->injected_u, c->z_pad)) || (st = dalloc(c, &c->sched, 6)))
    return bail(st);
  c->redraw_grid = (int)std::min<int64_t>(c->z, c->num_sms);
  if (const char* g = std::getenv("MHAR_GROUP_M")) c->group_m = std::max(1, std::atoi(g));
  if (const char* g = std::getenv("MHAR_WALK_BAND")) c->walk_band = std::max(0, std::atoi(g));
  if (const char* g = std::getenv("MHAR_TC_GROUP")) c->tc_group_n = std::max(1, std::atoi(g));
  if (const char* g = std::getenv("MHAR_TC_APOL")) c->tc_a_policy = std::atoi(g) % 3;
  if (const char* g = std::getenv("MHAR_TC_F16")) c->tc_f16 = std::atoi(g) != 0;
  if (const char* g = std::getenv("MHAR_I8_GROUP")) c->i8_group = std::max(1, std::atoi(g));
  if ((st = dalloc(c, &c->redraw_scratch, (size_t)c->redraw_grid * 3 * c->n))) return bail(st);
  if (c->opt.slack_mode == MHAR_SLACK_INCREMENTAL) {
    const size_t cache = (size_t)c->m_pad * c->z_pad;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (2 * cache * sizeof(double) + (1ull << 30) > free_b) {
      if (tiles) return bail(fail(MHAR_ERR_CUDA, "tcgen05 engine: not enough HBM for the slack cache"));
      c->opt.slack_mode = MHAR_SLACK_RECOMPUTE;  // not enough HBM for the slack cache
    } else if ((st = dalloc(c, &c->S, cache)) || (st = dalloc(c, &c->R, cache))) {
      return bail(st);
    }
  }

  // polytope upload: A_I column-major -> packed tiles, b padded with +inf
  {
    double* tmp = nullptr;
    e = cudaMalloc(&tmp, sizeof(double) * (size_t)c->m * c->n);
    if (e != cudaSuccess) return bail(fail(MHAR_ERR_CUDA, "cudaMalloc(A staging) failed"));
    // H2D copies are ordered on the context's (non-blocking) stream: a legacy-stream
    // cudaMemcpy from pageable memory may return before its DMA lands and would
    // race the packing kernels below
    cudaMemcpyAsync(tmp, p->a_in, sizeof(double) * (size_t)c->m * c->n, cudaMemcpyHostToDevice,
                    c->stream);
    const int64_t total = c->m_pad * c->KT * BK;
    pack_a_kernel<<<blocks_for(total, 256, c->num_sms * 32), 256, 0, c->stream>>>(
        tmp, c->m, c->n, c->m, c->m_pad, c->KT, c->A);
    ++c->launches;
    cudaStreamSynchronize(c->stream);
    if (fp32) {
      // A_I rounded to fp32 and split for 3xTF32; the fp64 copy becomes A_hi + A_lo
      const size_t an = (size_t)c->m_pad * c->n_pad, dn = (size_t)c->z_pad * c->n_pad;
      // the direction reaches the tensor cores split d = d_hi + d_lo (default:
      // the walk moves along its fp64 direction, the rates carry ~22 bits of
      // it) or rounded to one operand (MHAR_FP32_DIR_ROUNDED, the fast form:
      // the walk moves along the rounded direction); bodies with equalities
      // always split, the rounded direction would leave the null space of A_E
      const bool split_d = p->m_eq > 0 || opt->fp32_direction != MHAR_FP32_DIR_ROUNDED;
      if ((st = dalloc(c, &c->Ahi, an)) || (st = dalloc(c, &c->Alo, an)) ||
          (st = dalloc(c, &c->Dhi, dn)) || (split_d && (st = dalloc(c, &c->Dlo, dn)))) {
        cudaFree(tmp);
        return bail(st);
      }
      if (c->tc_f16) {
        c->tc_kt = (c->n + TC_BK16 - 1) / TC_BK16;
        if ((st = dalloc(c, &c->tc_rsc, c->m_pad)) || (st = dalloc(c, &c->tc_csc, c->z_pad))) {
          cudaFree(tmp);
          return bail(st);
        }
        tc16_split_a_kernel<<<blocks_for(c->m_pad, 128, c->num_sms * 8), 128, 0, c->stream>>>(
            tmp, c->m, c->n, c->m_pad, c->tc_kt, reinterpret_cast<__half*>(c->Ahi),
            reinterpret_cast<__half*>(c->Alo), c->tc_rsc, nullptr, c->KT);
      } else {
        c->tc_kt = c->KT;
        tc_split_a_kernel<<<blocks_for(total, 256, c->num_sms * 32), 256, 0, c->stream>>>(
            tmp, c->m, c->n, c->m_pad, c->KT, c->Ahi, c->Alo, nullptr, c->KT);
      }
      ++c->launches;
      cudaMemsetAsync(c->Dhi, 0, dn * sizeof(float), c->stream);
      cudaStreamSynchronize(c->stream);
      // 2-CTA TMA loads (MHAR_TC_TMA=0: plain bulk copies and the odd CTA's relay)
      const char* tma_env = std::getenv("MHAR_TC_TMA");
      c->tc_tma = !(tma_env && std::atoi(tma_env) == 0) &&
                  encode_piece_map(&c->tm_ahi, c->Ahi, an) &&
                  encode_piece_map(&c->tm_alo, c->Alo, an) &&
                  encode_piece_map(&c->tm_dhi, c->Dhi, dn) &&
                  (!c->Dlo || encode_piece_map(&c->tm_dlo, c->Dlo, dn));
      if (!c->Dlo) c->tm_dlo = c->tm_dhi;
      {
        // walk-pair bands once the direction operands outgrow a ~32 MB L2 share
        const int64_t pair_bytes = 2 * c->tc_kt * (int64_t)TC_D_PIECE * 4 * (c->Dlo ? 2 : 1);
        const int64_t pairs = c->tc_walk_tiles / 2;
        const int64_t fit = std::max<int64_t>(1, (32ll << 20) / pair_bytes);
        c->tc_walk_band = pairs > fit ? (int)fit : 0;
        if (const char* g = std::getenv("MHAR_TC_WALK_BAND")) c->tc_walk_band = std::max(0, std::atoi(g));
      }
      cudaFuncSetAttribute(chord_tc32_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TcCfg<false>::smem);
      cudaFuncSetAttribute(chord_tc32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TcCfg<true>::smem);
      cudaFuncSetAttribute(chord_tc32_kernel<false, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcCfg<false>::smem);
      cudaFuncSetAttribute(chord_tc32_kernel<true, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcCfg<true>::smem);
      if (std::getenv("MHAR_I8_PROFILE") && (st = dalloc(c, &c->tc_prof, kProfWords * (size_t)c->num_sms))) {
        cudaFree(tmp);
        return bail(st);
      }
    }
    if (i8) {
      // A_I as 7 int8 slices of its per-row 53-bit fixed point
      const size_t an = (size_t)I8_SLICES * c->m_pad * c->KS * I8_BK;
      const size_t dn = (size_t)I8_SLICES * c->z_pad * c->KS * I8_BK;
      if ((st = dalloc(c, &c->A8, an)) || (st = dalloc(c, &c->D8, dn)) ||
          (st = dalloc(c, &c->rsc, c->m_pad)) || (st = dalloc(c, &c->csc, c->z_pad)) ||
          (st = dalloc(c, &c->rexp, c->m_pad))) {
        cudaFree(tmp);
        return bail(st);
      }
      i8_row_scale_kernel<<<blocks_for(c->m_pad, 256, c->num_sms * 8), 256, 0, c->stream>>>(
          tmp, c->m, c->n, c->m_pad, c->rexp, c->rsc);
      const int64_t groups = c->m_pad * c->KS * (I8_BK / 16);
      i8_split_a_kernel<<<blocks_for(groups, 256, c->num_sms * 32), 256, 0, c->stream>>>(
          tmp, c->m, c->n, c->m_pad, c->KS, c->rexp, c->A8);
      c->launches += 2;
      cudaMemsetAsync(c->D8, 0, dn, c->stream);
      cudaStreamSynchronize(c->stream);
      cudaFuncSetAttribute(chord_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)I8_SMEM);
      {
        // persistent grid: as many clusters as can be co-resident (a cluster
        // of 4 needs 4 free SMs in one GPC)
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3((unsigned)(I8_CL * (c->num_sms / I8_CL)));
        lc.blockDim = dim3(I8_THREADS);
        lc.dynamicSmemBytes = I8_SMEM;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, chord_i8_kernel, &lc) != cudaSuccess || ncl < 1)
          ncl = c->num_sms / I8_CL;
        cudaGetLastError();
        c->i8_clusters = ncl;
      }
      if (std::getenv("MHAR_I8_PROFILE") && (st = dalloc(c, &c->tc_prof, kProfWords * (size_t)c->num_sms))) {
        cudaFree(tmp);
        return bail(st);
      }
    }
    // small bodies: keep the column-major copy for the walk-resident kernel
    // (warps per CTA: the most that fit next to the body; the path is taken
    // when at least 4 walks per SM are resident)
    c->small_ns = (int)(c->n | 1);
    const int gw = std::getenv("MHAR_SMALL_GW") ? std::atoi(std::getenv("MHAR_SMALL_GW"))
                                                : small_group_width(c->n, c->m, !diag_coef.empty(),
                                                                    c->me > 0,
                                                                    opt->z_plan > 0 ? opt->z_plan
                                                                                    : c->z);
    c->small_gw = (gw == 4 || gw == 8 || gw == 16) ? gw : 32;
    size_t small_bytes = 0;
    int small_warps = 0;
    for (int w = SMALL_WARPS; w >= 1 && !small_warps; --w) {
      const size_t bytes = sizeof(double) * small_smem_doubles(c->n, c->m, c->me, c->me > 0,
                                                               c->small_ns, !diag_coef.empty(),
                                                               factored, w, c->small_gw);
      const size_t per_sm = (227 * 1024) / (bytes + 1024);
      if (bytes <= 220 * 1024 && (size_t)w * (32 / c->small_gw) * per_sm >= 4) {
        small_warps = w;
        small_bytes = bytes;
      }
    }
    // the walk-resident kernel runs each walk's iterate in one warp: it wins
    // while the body is small or few walks share the GPU; past that the
    // kernel chain, parallel over walks and coordinates, is faster (measured on
    // the paper's hypercubes / simplices, tools/small_vs_multi.sh,
    // profiles/small_vs_multi_r02.jsonl: n = 1000 wins small at z = 1000 and
    // chain at z = 2000; n = 2000 chain by 2x; n = 700, z = 3000 small)
    const int64_t zp = opt->z_plan > 0 ? opt->z_plan : c->z;  // the run's walks (mhar_options)
    const bool small_wins = c->n < 1800 && (c->n < 900 || c->n * zp <= 1600000);
    if (c->opt.small_path && c->opt.rng == MHAR_RNG_PHILOX && small_warps > 0 && small_wins) {
      c->Acm = tmp;
      c->allocs.push_back(tmp);
      c->small_smem = small_bytes;
      c->small_warps = small_warps;
    } else {
      cudaFree(tmp);
    }
    std::vector<double> bp(c->m_pad, __builtin_huge_val());
    std::memcpy(bp.data(), p->b_in, sizeof(double) * c->m);
    cudaMemcpyAsync(c->b, bp.data(), sizeof(double) * c->m_pad, cudaMemcpyHostToDevice, c->stream);
    if (!diag_coef.empty()) {
      if ((st = dalloc(c, &c->diag_coef, diag_coef.size()))) return bail(st);
      c->diag_blocks = c->m / c->n;
      // uniform blocks (hypercube, simplex): constants instead of per-row loads
      if (c->diag_blocks <= kDiagUniMax) {
        bool uni = true;
        for (int64_t j = 0; j < c->diag_blocks && uni; ++j) {
          c->diag_uc[j] = diag_coef[j * c->n];
          c->diag_ub[j] = p->b_in[j * c->n];
          for (int64_t k = 0; k < c->n && uni; ++k)
            uni = std::memcmp(&diag_coef[j * c->n + k], &c->diag_uc[j], sizeof(double)) == 0 &&
                  std::memcmp(&p->b_in[j * c->n + k], &c->diag_ub[j], sizeof(double)) == 0;
        }
        c->diag_uniform = uni;
      }
      cudaMemcpyAsync(c->diag_coef, diag_coef.data(), sizeof(double) * diag_coef.size(),
                      cudaMemcpyHostToDevice, c->stream);
    }
    cudaStreamSynchronize(c->stream);  // bp, diag_coef are locals
  }
  if (c->me > 0) {
    std::vector<double> P((size_t)c->n * c->n), G((size_t)c->me * c->me);
    if (projector && gram_inverse) {
      std::memcpy(P.data(), projector, sizeof(double) * P.size());
      std::memcpy(G.data(), gram_inverse, sizeof(double) * G.size());
    } else {
      std::string msg;
      const int ps = mhar_host::compute_projection(p->a_eq, c->me, c->n, P.data(), G.data(), &msg);
      if (ps) return bail(fail(ps, std::string(code_name(ps)) + ": " + msg));
    }
    if ((st = dalloc(c, &c->H, nzp)) || (st = dalloc(c, &c->Ppk, (size_t)c->p_rows_pad * c->n_pad)) ||
        (st = dalloc(c, &c->Pcm, (size_t)c->n * c->n)) ||
        (st = dalloc(c, &c->AE, (size_t)c->me * c->n)) || (st = dalloc(c, &c->bE, c->me)) ||
        (st = dalloc(c, &c->G, (size_t)c->me * c->me)) ||
        (st = dalloc(c, &c->eqres, (size_t)c->me * c->z)) ||
        (st = dalloc(c, &c->eqg, (size_t)c->me * c->z)) ||
        // factored projection when m_E is small against n (fastpath.cuh)
        (st = dalloc(c, &c->norm_part, (size_t)dot_splits(c->KT) * c->z_pad)) ||
        (factored &&
         (st = dalloc(c, &c->proj_g, (size_t)dot_splits(c->KT) * c->me * c->z_pad))))
      return bail(st);
    cudaMemcpyAsync(c->Pcm, P.data(), sizeof(double) * P.size(), cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(c->AE, p->a_eq, sizeof(double) * c->me * c->n, cudaMemcpyHostToDevice,
                    c->stream);
    cudaMemcpyAsync(c->bE, p->b_eq, sizeof(double) * c->me, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(c->G, G.data(), sizeof(double) * G.size(), cudaMemcpyHostToDevice, c->stream);
    const int64_t total = c->p_rows_pad * c->KT * BK;
    pack_a_kernel<<<blocks_for(total, 256, c->num_sms * 32), 256, 0, c->stream>>>(
        c->Pcm, c->n, c->n, c->n, c->p_rows_pad, c->KT, c->Ppk);
    ++c->launches;
    cudaMemsetAsync(c->H, 0, sizeof(double) * nzp, c->stream);
  }
  cudaMemsetAsync(c->X, 0, sizeof(double) * nzp, c->stream);
  cudaMemsetAsync(c->D, 0, sizeof(double) * nzp, c->stream);
  cudaMemsetAsync(c->theta, 0, sizeof(double) * c->z_pad, c->stream);
  cudaMemsetAsync(c->collapsed, 0, sizeof(unsigned) * c->z_pad, c->stream);
  cudaMemsetAsync(c->redraw_total, 0, sizeof(unsigned long long), c->stream);
  cudaMemsetAsync(c->err, 0xFF, sizeof(unsigned long long), c->stream);
  int big = 0x7FFFFFFF;
  cudaMemcpyAsync(c->first_reject, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream);
  c->no_graphs = std::getenv("MHAR_NO_GRAPHS") != nullptr;
  c->pdl = std::getenv("MHAR_NO_PDL") == nullptr;
  if ((st = dalloc(c, &c->d_iter, 1))) return bail(st);
  fill_keys_kernel<<<blocks_for(c->z_pad, 256, 1 << 20), 256, 0, c->stream>>>(
      c->hi_key, c->lo_key, c->viol_key, c->sides, c->z_pad);
  ++c->launches;
  cudaFuncSetAttribute(chord_kernel<FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHORD_SMEM);
  cudaFuncSetAttribute(chord_kernel<FUSED_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHORD_SMEM);
  cudaFuncSetAttribute(chord2_kernel<INCREMENTAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHORD2_SMEM);
  cudaFuncSetAttribute(chord3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C3_SMEM);
  cudaFuncSetAttribute(chord3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C3_SMEM);
  if (c->c3 && std::getenv("MHAR_C3_PROFILE") && (st = dalloc(c, &c->c3_prof, 16 * (size_t)c->num_sms)))
    return bail(st);
  cudaFuncSetAttribute(chord2_kernel<CHECK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHORD2_SMEM);
  cudaFuncSetAttribute(chord2_kernel<SLACK_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHORD2_SMEM);
  if (c->Acm) {
    if ((st = dalloc(c, &c->walk_err, c->z)) || (st = dalloc(c, &c->walk_err_min, 1)))
      return bail(st);
    cudaMemsetAsync(c->walk_err_min, 0xFF, sizeof(unsigned long long), c->stream);  // kNoError
    const void* sk = c->small_gw == 4    ? (const void*)small_kernel<4>
                     : c->small_gw == 8  ? (const void*)small_kernel<8>
                     : c->small_gw == 16 ? (const void*)small_kernel<16>
                                         : (const void*)small_kernel<32>;
    cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->small_smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sk, 32 * c->small_warps, c->small_smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t walks_per_cta = (int64_t)c->small_warps * (32 / c->small_gw);
    const int64_t need = (c->z + walks_per_cta - 1) / walks_per_cta;
    c->small_grid = (int)std::min<int64_t>(need, (int64_t)per_sm * c->num_sms);
  }
  if ((st = reset_streams(c))) return bail(st);
  e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(MHAR_ERR_CUDA, std::string("ctx_create: ") + cudaGetErrorString(e)));
  *out = c;
  return 0;
}

int mhar_ctx_destroy(mhar_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  if (c->tc_prof) report_tc_profile(c);
  if (c->c3_prof) {
    // chord3 phase cycles summed over every launch of this context (MMA warps
    // and epilogue warps, each counter per warp, summed over the CTAs)
    std::vector<unsigned long long> h(16 * (size_t)c->num_sms);
    if (cudaMemcpy(h.data(), c->c3_prof, h.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
      double t[6] = {0, 0, 0, 0, 0, 0};
      for (int b = 0; b < c->num_sms; ++b)
        for (int k = 0; k < 6; ++k) t[k] += (double)h[16 * b + k];
      const double mma = t[0] + t[2] + t[3];
      std::fprintf(stderr,
                   "[chord3 profile] MMA warps: mainloop %.1f%% (of which full-barrier waits "
                   "%.1f%%), TMEM-empty waits %.1f%%, TMEM stores %.1f%%; epilogue warps: waiting "
                   "for tiles %.1f%%, working %.1f%%\n",
                   100 * t[0] / mma, 100 * t[1] / mma, 100 * t[2] / mma, 100 * t[3] / mma,
                   100 * t[4] / (t[4] + t[5]), 100 * t[5] / (t[4] + t[5]));
    }
  }
  for (auto& ev : c->pending) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  for (auto& ev : c->event_pool) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  for (int b = 0; b < 2; ++b) {
    if (c->pinned[b]) cudaFreeHost(c->pinned[b]);
    if (c->ev_ready[b]) cudaEventDestroy(c->ev_ready[b]);
    if (c->ev_copied[b]) cudaEventDestroy(c->ev_copied[b]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (void* q : c->allocs) cudaFree(q);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}

// The upload lands in a staging buffer first; if it is bit-identical to the
// resident state (the common loop `step(p, op, cfg, rng, state)` hands back
// the state the previous call returned), the slack cache stays valid.
int mhar_set_state(mhar_ctx* c, const double* x) {
  if (!c || !x) return fail(MHAR_ERR_INVALID_ARGUMENT, "set_state: null argument");
  CK(cudaSetDevice(c->device));
  int s = 0;
  if (!c->Xtmp) {
    if ((s = dalloc(c, &c->Xtmp, (size_t)c->z_pad * c->n_pad))) return s;
  }
  if ((s = upload_state_host(c, x, c->Xtmp))) return s;
  CK(cudaMemsetAsync(c->first_bad, 0, sizeof(int), c->stream));
  const int64_t total = c->z_pad * c->KT * BK;
  differs_kernel<<<blocks_for(total, 256, c->num_sms * 8), 256, 0, c->stream>>>(c->Xtmp, c->X,
                                                                               total, c->first_bad);
  LAUNCH_OK(c, "differs_kernel");
  int differs = 1;
  CK(cudaMemcpyAsync(&differs, c->first_bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if ((s = clear_error_and_cache(c))) return s;
  CK(cudaStreamSynchronize(c->stream));
  if (differs) {
    std::swap(c->X, c->Xtmp);
    c->slack_valid = false;
  }
  return 0;
}

int mhar_get_state(mhar_ctx* c, double* x) {
  if (!c || !x) return fail(MHAR_ERR_INVALID_ARGUMENT, "get_state: null argument");
  CK(cudaSetDevice(c->device));
  unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->X, c->n, c->z, c->KT, c->rows);
  LAUNCH_OK(c, "unpack_b_kernel");
  CK(cudaMemcpyAsync(x, c->rows, sizeof(double) * c->n * c->z, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int mhar_debug_last_iterate(mhar_ctx* c, double* d, double* lower, double* upper, double* theta) {
  if (!c) return fail(MHAR_ERR_INVALID_ARGUMENT, "debug_last_iterate: null context");
  CK(cudaSetDevice(c->device));
  if (d) {
    unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        c->D, c->n, c->z, c->KT, c->rows);
    LAUNCH_OK(c, "unpack_b_kernel");
    CK(cudaMemcpyAsync(d, c->rows, sizeof(double) * c->n * c->z, cudaMemcpyDeviceToHost, c->stream));
  }
  if (lower) CK(cudaMemcpyAsync(lower, c->lower, sizeof(double) * c->z, cudaMemcpyDeviceToHost, c->stream));
  if (upper) CK(cudaMemcpyAsync(upper, c->upper, sizeof(double) * c->z, cudaMemcpyDeviceToHost, c->stream));
  if (theta) CK(cudaMemcpyAsync(theta, c->theta, sizeof(double) * c->z, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int mhar_get_state_rows_device(mhar_ctx* c, double* dev_rows) {
  if (!c || !dev_rows) return fail(MHAR_ERR_INVALID_ARGUMENT, "get_state_rows_device: null");
  CK(cudaSetDevice(c->device));
  unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->X, c->n, c->z, c->KT, dev_rows);
  LAUNCH_OK(c, "unpack_b_kernel");
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int mhar_step(mhar_ctx* c, int64_t iters, int64_t reproject_every) {
  if (!c || iters < 0) return fail(MHAR_ERR_INVALID_ARGUMENT, "step: bad argument");
  CK(cudaSetDevice(c->device));
  return advance(c, iters, reproject_every);
}

int mhar_get_iteration(mhar_ctx* c, int64_t* iteration) {
  if (!c || !iteration) return fail(MHAR_ERR_INVALID_ARGUMENT, "get_iteration: null argument");
  *iteration = c->iterations;
  return 0;
}

int mhar_set_iteration(mhar_ctx* c, int64_t iteration) {
  if (!c || iteration < 0) return fail(MHAR_ERR_INVALID_ARGUMENT, "set_iteration: bad argument");
  if (c->opt.rng != MHAR_RNG_PHILOX)
    return fail(MHAR_ERR_INVALID_ARGUMENT,
                "set_iteration: reference streams carry per-walk state; checkpoint needs Philox");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  c->iterations = iteration;
  return 0;
}

int mhar_request_refresh(mhar_ctx* c) {
  if (!c) return fail(MHAR_ERR_INVALID_ARGUMENT, "request_refresh: null context");
  c->slack_valid = false;
  return 0;
}

int mhar_get_streams(mhar_ctx* c, uint64_t* col_states, uint64_t* theta_state) {
  if (!c || !col_states || !theta_state)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "get_streams: null argument");
  if (c->opt.rng != MHAR_RNG_REFERENCE)
    return fail(MHAR_ERR_INVALID_ARGUMENT,
                "get_streams: Philox draws are keyed on the iterate counter (mhar_get_iteration)");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(col_states, c->col_state, sizeof(uint64_t) * c->z, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaMemcpyAsync(theta_state, c->theta_state, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int mhar_set_streams(mhar_ctx* c, const uint64_t* col_states, const uint64_t* theta_state) {
  if (!c || !col_states || !theta_state)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "set_streams: null argument");
  if (c->opt.rng != MHAR_RNG_REFERENCE)
    return fail(MHAR_ERR_INVALID_ARGUMENT,
                "set_streams: Philox draws are keyed on the iterate counter (mhar_set_iteration)");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(c->col_state, col_states, sizeof(uint64_t) * c->z, cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->theta_state, theta_state, sizeof(uint64_t), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int mhar_sync(mhar_ctx* c) {
  if (!c) return fail(MHAR_ERR_INVALID_ARGUMENT, "sync: null context");
  CK(cudaSetDevice(c->device));
  return read_error(c, nullptr);
}

int mhar_step_timed(mhar_ctx* c, int64_t iters, int64_t reproject_every, double* device_ms) {
  if (!c || iters < 0) return fail(MHAR_ERR_INVALID_ARGUMENT, "step_timed: bad argument");
  CK(cudaSetDevice(c->device));
  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, c->stream));
  int s = 0;
  s = advance(c, iters, reproject_every);
  CK(cudaEventRecord(t1, c->stream));
  CK(cudaEventSynchronize(t1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (device_ms) *device_ms = ms;
  if (s) return s;
  return read_error(c, nullptr);
}

int mhar_step_injected(mhar_ctx* c, const double* h, const double* u, double* lower,
                       double* upper, double* theta, uint8_t* flags) {
  if (!c || !h || !u) return fail(MHAR_ERR_INVALID_ARGUMENT, "step_injected: null argument");
  CK(cudaSetDevice(c->device));
  int s = read_error(c, nullptr);
  if (s) return s;
  s = upload_state_host(c, h, c->me > 0 ? c->H : c->D);
  if (s) return s;
  CK(cudaMemsetAsync(c->injected_u, 0, sizeof(double) * c->z_pad, c->stream));
  CK(cudaMemcpyAsync(c->injected_u, u, sizeof(double) * c->z, cudaMemcpyHostToDevice, c->stream));
  const int64_t saved = c->iterations;
  s = enqueue_iterate(c, 0, true);
  if (s) return s;
  c->iterations = saved;  // the hook does not advance the RNG counters
  int64_t walk = -1;
  s = read_error(c, &walk);
  std::vector<double> tmp(c->z);
  if (lower) CK(cudaMemcpy(lower, c->lower, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
  if (upper) CK(cudaMemcpy(upper, c->upper, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
  if (theta) CK(cudaMemcpy(theta, c->theta, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
  if (flags) {
    std::vector<unsigned> f(c->z);
    CK(cudaMemcpy(f.data(), c->flags, sizeof(unsigned) * c->z, cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < c->z; ++k) flags[k] = (uint8_t)f[k];
  }
  return s;
}

int mhar_generate_directions(mhar_ctx* c, double* h) {
  if (!c || !h) return fail(MHAR_ERR_INVALID_ARGUMENT, "generate_directions: null argument");
  CK(cudaSetDevice(c->device));
  int s = read_error(c, nullptr);
  if (s) return s;
  if ((s = launch_normals(c, c->D))) return s;
  if (c->opt.rng == MHAR_RNG_REFERENCE) {
    advance_streams_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(
        c->col_state, c->z, 2 * ((c->n + 1) / 2));
    LAUNCH_OK(c, "advance_streams_kernel");
  }
  ++c->iterations;       // Philox: the next batch is keyed on the next counter
  c->slack_valid = false;  // D was overwritten
  unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->D, c->n, c->z, c->KT, c->rows);
  LAUNCH_OK(c, "unpack_b_kernel");
  CK(cudaMemcpyAsync(h, c->rows, sizeof(double) * c->n * c->z, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int mhar_select_points(mhar_ctx* c, const double* x, const double* d, const double* lower,
                       const double* upper, const uint8_t* degenerate, double* out) {
  if (!c || !x || !d || !lower || !upper || !degenerate || !out)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "select_points: null argument");
  for (int64_t k = 0; k < c->z; ++k)
    if (degenerate[k])
      return fail(MHAR_ERR_DIRECTION_DEGENERATE, "DIRECTION_DEGENERATE: select_points: walk " +
                                                     std::to_string(k + c->opt.chain_offset) +
                                                     " has no usable chord");
  CK(cudaSetDevice(c->device));
  int s = read_error(c, nullptr);
  if (s) return s;
  if (!c->Xtmp) {
    if ((s = dalloc(c, &c->Xtmp, (size_t)c->z_pad * c->n_pad))) return s;
  }
  if ((s = upload_state_host(c, x, c->Xtmp))) return s;
  if ((s = upload_state_host(c, d, c->D))) return s;
  c->slack_valid = false;
  CK(cudaMemcpyAsync(c->lower, lower, sizeof(double) * c->z, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->upper, upper, sizeof(double) * c->z, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->flags, 0, sizeof(unsigned) * c->z_pad, c->stream));
  CK(cudaMemsetAsync(c->theta, 0, sizeof(double) * c->z_pad, c->stream));
  ThetaParams tp = theta_params(c, nullptr);
  theta_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(tp);
  LAUNCH_OK(c, "theta_kernel");
  if (c->opt.rng == MHAR_RNG_REFERENCE) {
    theta_fixup_kernel<<<1, 1, 0, c->stream>>>(tp);
    LAUNCH_OK(c, "theta_fixup_kernel");
  }
  const int64_t total2 = c->z_pad * c->KT * BK / 2;
  axpy_kernel<<<blocks_for(total2, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->Xtmp, c->D, c->theta, total2, c->KT, c->err);
  LAUNCH_OK(c, "axpy_kernel");
  ++c->iterations;
  unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->Xtmp, c->n, c->z, c->KT, c->rows);
  LAUNCH_OK(c, "unpack_b_kernel");
  CK(cudaMemcpyAsync(out, c->rows, sizeof(double) * c->n * c->z, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return read_error(c, nullptr);
}

int mhar_lambda_intervals(mhar_ctx* c, const double* x, const double* d, double* lower,
                          double* upper, uint8_t* flags) {
  if (!c || !x || !d) return fail(MHAR_ERR_INVALID_ARGUMENT, "lambda_intervals: null argument");
  CK(cudaSetDevice(c->device));
  int s = read_error(c, nullptr);
  if (s) return s;
  if (!c->Xtmp) {
    if ((s = dalloc(c, &c->Xtmp, (size_t)c->z_pad * c->n_pad))) return s;
  }
  if ((s = upload_state_host(c, x, c->Xtmp))) return s;
  if ((s = upload_state_host(c, d, c->D))) return s;
  c->slack_valid = false;  // D was overwritten
  if ((s = launch_chord(c, FUSED, c->Xtmp))) return s;
  if ((s = launch_finalize(c, false, false))) return s;
  int64_t walk = -1;
  const int st = read_error(c, &walk);
  if (lower) CK(cudaMemcpy(lower, c->lower, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
  if (upper) CK(cudaMemcpy(upper, c->upper, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
  if (flags) {
    std::vector<unsigned> f(c->z);
    CK(cudaMemcpy(f.data(), c->flags, sizeof(unsigned) * c->z, cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < c->z; ++k) flags[k] = (uint8_t)f[k];
  }
  if (st) {
    const std::string msg = g_last_error;
    clear_error(c);
    cudaStreamSynchronize(c->stream);
    g_last_error = msg;
  }
  return st;
}

// Enqueues the containment pass of the current state: viol (max A x - b)
// and eqviol (max |A_E x - b_E|) per walk.
static int enqueue_check(mhar_ctx* c) {
  int s = launch_chord(c, CHECK, c->X);
  if (s) return s;
  viol_extract_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(c->viol_key,
                                                                              c->viol, c->z);
  LAUNCH_OK(c, "viol_extract_kernel");
  if (c->me > 0) {
    const int64_t mz = c->me * c->z;
    eq_residual_kernel<<<blocks_for(mz, 256, 1 << 30), 256, 0, c->stream>>>(
        c->AE, c->bE, c->X, c->me, c->n, c->z, c->KT, c->eqres);
    LAUNCH_OK(c, "eq_residual_kernel");
    eq_maxabs_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(c->eqres, c->me,
                                                                            c->z, c->eqviol);
    LAUNCH_OK(c, "eq_maxabs_kernel");
  }
  return 0;
}

int mhar_check_state(mhar_ctx* c, double eps, int64_t* first_bad, double* max_viol,
                     double* max_eq) {
  if (!c) return fail(MHAR_ERR_INVALID_ARGUMENT, "check_state: null context");
  CK(cudaSetDevice(c->device));
  int s = read_error(c, nullptr);
  if (s) return s;
  if ((s = enqueue_check(c))) return s;
  int big = 0x7FFFFFFF;
  CK(cudaMemcpyAsync(c->first_bad, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  contains_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(
      c->viol, c->me > 0 ? c->eqviol : nullptr, c->z, eps, c->err, 0, c->first_bad);
  LAUNCH_OK(c, "contains_kernel");
  int fb = big;
  CK(cudaMemcpyAsync(&fb, c->first_bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (first_bad) *first_bad = (fb == big) ? -1 : fb;
  if (max_viol) CK(cudaMemcpy(max_viol, c->viol, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
  if (max_eq) {
    if (c->me > 0) {
      CK(cudaMemcpy(max_eq, c->eqviol, sizeof(double) * c->z, cudaMemcpyDeviceToHost));
    } else {
      for (int64_t k = 0; k < c->z; ++k) max_eq[k] = 0.0;
    }
  }
  return read_error(c, nullptr);
}

int mhar_run(mhar_ctx* c, const mhar_run_config* cfg, const double* x0, double* samples,
             mhar_run_stats* stats) {
  NvtxRange range("mhar.run");
  if (!c || !cfg || !x0) return fail(MHAR_ERR_INVALID_ARGUMENT, "run: null argument");
  if (cfg->phi < 1) return fail(MHAR_ERR_INVALID_ARGUMENT, "config: phi must be >= 1");
  if (cfg->windows < 1) return fail(MHAR_ERR_INVALID_ARGUMENT, "config: windows must be >= 1");
  if (cfg->burn_in < 0 || cfg->reproject_every < 0)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "config: negative burn_in/reproject_every");
  CK(cudaSetDevice(c->device));
  int s = 0;
  // fresh walk: x0 replicated, streams re-seeded, counters from zero (run(),
  // sampler.cpp:298-302)
  CK(cudaMemcpyAsync(c->x0, x0, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  const int64_t total = c->z_pad * c->KT * BK;
  broadcast_state_kernel<<<blocks_for(total, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->x0, c->n, c->z, c->z_pad, c->KT, c->X);
  LAUNCH_OK(c, "broadcast_state_kernel");
  if ((s = clear_error(c))) return s;
  CK(cudaMemsetAsync(c->redraw_total, 0, sizeof(unsigned long long), c->stream));
  c->slack_valid = false;
  c->iterations = 0;
  if ((s = reset_streams(c))) return s;

  // Collection streams out while the next window computes: rows of window w
  // go to a device buffer (double-buffered), a side stream copies them into
  // pinned staging, and the host moves window w-2 into `samples` while the
  // device works on window w.
  const size_t win = (size_t)c->z * c->n;
  if (samples && !c->copy_stream) {
    if ((s = dalloc(c, &c->rows2, win))) return s;
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaHostAlloc(&c->pinned[b], win * sizeof(double), cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&c->ev_ready[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
    }
  }
  double* drows[2] = {c->rows, c->rows2};
  auto drain = [&](int64_t w) {  // window w's rows -> samples (host)
    const int b = (int)(w & 1);
    cudaEventSynchronize(c->ev_copied[b]);
    std::memcpy(samples + (size_t)w * win, c->pinned[b], win * sizeof(double));
  };

  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, c->stream);
  if ((s = advance(c, cfg->burn_in, cfg->reproject_every))) return s;
  int64_t walk = -1;
  for (int64_t w = 0; w < cfg->windows; ++w) {
    if ((s = advance(c, cfg->phi, cfg->reproject_every))) return s;
    if ((s = enqueue_check(c))) return s;
    CK(cudaMemsetAsync(c->first_bad, 0x7F, sizeof(int), c->stream));
    contains_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(
        c->viol, c->me > 0 ? c->eqviol : nullptr, c->z, c->opt.eps_feas, c->err, 1, c->first_bad);
    LAUNCH_OK(c, "contains_kernel");
    if (samples) {
      const int b = (int)(w & 1);
      if (w >= 2) CK(cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
      unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
          c->X, c->n, c->z, c->KT, drows[b]);
      LAUNCH_OK(c, "unpack_b_kernel");
      CK(cudaEventRecord(c->ev_ready[b], c->stream));
      if (w >= 2) drain(w - 2);  // overlaps the device work just queued
      CK(cudaStreamWaitEvent(c->copy_stream, c->ev_ready[b], 0));
      CK(cudaMemcpyAsync(c->pinned[b], drows[b], win * sizeof(double), cudaMemcpyDeviceToHost,
                         c->copy_stream));
      CK(cudaEventRecord(c->ev_copied[b], c->copy_stream));
    }
  }
  if (samples) {
    for (int64_t w = std::max<int64_t>(0, cfg->windows - 2); w < cfg->windows; ++w) drain(w);
    CK(cudaStreamWaitEvent(c->stream, c->ev_copied[(cfg->windows - 1) & 1], 0));
  }
  cudaEventRecord(t1, c->stream);
  s = read_error(c, &walk);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  unsigned long long red = 0;
  cudaMemcpy(&red, c->redraw_total, sizeof(red), cudaMemcpyDeviceToHost);
  if (stats) {
    stats->iterate_count = c->z * cfg->phi * cfg->windows;
    stats->windows = cfg->windows;
    stats->redraw_count = (int64_t)red;
    stats->err_walk = s ? walk + c->opt.chain_offset : -1;
    stats->seconds = ms * 1e-3;
  }
  return s;
}

int mhar_get_stats(mhar_ctx* c, mhar_ctx_stats* out) {
  if (!c || !out) return fail(MHAR_ERR_INVALID_ARGUMENT, "get_stats: null argument");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  harvest_timing(c);
  unsigned long long red = 0;
  CK(cudaMemcpy(&red, c->redraw_total, sizeof(red), cudaMemcpyDeviceToHost));
  out->iterations = c->iterations;
  out->redraw_count = (int64_t)red;
  out->kernel_launches = c->launches;
  out->chord_launches = c->chord_launches;
  out->chord_ms = c->chord_ms;
  out->chord_timed = c->chord_timed;
  out->chord_flops = c->chord_flops;
  out->refreshes = c->refreshes;
  out->z = c->z;
  out->z_padded = c->z_pad;
  out->m_padded = c->m_pad;
  out->n_padded = c->n_pad;
  out->chord_kernel = c->small_grid > 0 ? MHAR_CHORD_SMALL
                      : c->diag_coef    ? MHAR_CHORD_DIAG
                      : c->A8           ? MHAR_CHORD_INT8
                      : c->Ahi          ? MHAR_CHORD_TC32
                      : c->c3           ? MHAR_CHORD_DMMA3
                                        : MHAR_CHORD_DMMA;
  return 0;
}

int mhar_set_timing(mhar_ctx* c, int enabled) {
  if (!c) return fail(MHAR_ERR_INVALID_ARGUMENT, "set_timing: null context");
  c->timing = enabled != 0;
  return 0;
}

int mhar_reset_stats(mhar_ctx* c) {
  if (!c) return fail(MHAR_ERR_INVALID_ARGUMENT, "reset_stats: null context");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  harvest_timing(c);
  c->launches = 0;
  c->chord_launches = 0;
  c->chord_ms = 0.0;
  c->chord_timed = 0;
  c->chord_flops = 0.0;
  c->refreshes = 0;
  return 0;
}

int mhar_minimum_spanning_tree(const double* points, int64_t N, int64_t n, int device,
                               int32_t* edge_a, int32_t* edge_b, double* edge_w) {
  if (!points || N < 2 || n < 1 || !edge_a || !edge_b || !edge_w)
    return fail(MHAR_ERR_INVALID_ARGUMENT, "minimum_spanning_tree: need at least two points");
  CK(cudaSetDevice(device));
  // coordinate-major copy for coalesced distance sweeps
  std::vector<double> pt((size_t)N * n);
  for (int64_t v = 0; v < N; ++v)
    for (int64_t k = 0; k < n; ++k) pt[(size_t)k * N + v] = points[(size_t)v * n + k];
  double *dP = nullptr, *dbest = nullptr, *dew = nullptr;
  int *dpar = nullptr, *dea = nullptr, *deb = nullptr;
  unsigned char* dint = nullptr;
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  auto cleanup = [&]() {
    cudaFree(dP);
    cudaFree(dbest);
    cudaFree(dew);
    cudaFree(dpar);
    cudaFree(dea);
    cudaFree(deb);
    cudaFree(dint);
    cudaStreamDestroy(s);
  };
  if (cudaMalloc(&dP, sizeof(double) * pt.size()) != cudaSuccess ||
      cudaMalloc(&dbest, sizeof(double) * N) != cudaSuccess ||
      cudaMalloc(&dew, sizeof(double) * N) != cudaSuccess ||
      cudaMalloc(&dpar, sizeof(int) * N) != cudaSuccess ||
      cudaMalloc(&dea, sizeof(int) * N) != cudaSuccess ||
      cudaMalloc(&deb, sizeof(int) * N) != cudaSuccess || cudaMalloc(&dint, N) != cudaSuccess) {
    cleanup();
    return fail(MHAR_ERR_CUDA, "minimum_spanning_tree: cudaMalloc failed");
  }
  cudaMemcpyAsync(dP, pt.data(), sizeof(double) * pt.size(), cudaMemcpyHostToDevice, s);
  // pools past a few thousand points spread over every SM (cooperative grid,
  // one barrier per added vertex); MHAR_PRIM=cta|grid forces one form
  const char* prim_env = std::getenv("MHAR_PRIM");
  bool grid_form = N > 2048;
  if (prim_env && !std::strcmp(prim_env, "cta")) grid_form = false;
  if (prim_env && !std::strncmp(prim_env, "grid", 4)) grid_form = true;  // grid | grid_l2
  cudaError_t e = cudaSuccess;
  PrimCand* dcand = nullptr;
  if (grid_form) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int64_t G = (N + PRIM_GRID_THREADS - 1) / PRIM_GRID_THREADS;
    if (G > sms) G = sms;
    if (G < 1) G = 1;
    int64_t chunk = (N + G - 1) / G;
    G = (N + chunk - 1) / chunk;
    // the CTA's own points go to shared memory too when they fit (L2
    // latency otherwise bounds the sequential distance sums)
    const int64_t nst = std::min<int64_t>(n, PRIM_GRID_SMEM_COORDS);
    int stage_own = n <= PRIM_GRID_SMEM_COORDS && sizeof(double) * (nst + chunk * n) <= 200 * 1024;
    if (prim_env && !std::strcmp(prim_env, "grid_l2")) stage_own = 0;
    const size_t smem = sizeof(double) * (size_t)(nst + (stage_own ? chunk * n : 0));
    e = cudaMalloc(&dcand, sizeof(PrimCand) * 2 * G);
    if (e == cudaSuccess && smem > 48 * 1024)
      e = cudaFuncSetAttribute(prim_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    if (e == cudaSuccess) {
      void* args[] = {&dP, (void*)&N, (void*)&n, &chunk, &dbest, &dpar, &dint,
                      &dcand, &dea, &deb, &dew, &stage_own};
      e = cudaLaunchCooperativeKernel((const void*)prim_grid_kernel, dim3((unsigned)G),
                                      dim3(PRIM_GRID_THREADS), args, smem, s);
    }
  } else {
    prim_kernel<<<1, PRIM_THREADS, 0, s>>>(dP, N, n, dbest, dpar, dint, dea, deb, dew);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    cudaMemcpyAsync(edge_a, dea, sizeof(int) * (N - 1), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(edge_b, deb, sizeof(int) * (N - 1), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(edge_w, dew, sizeof(double) * (N - 1), cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
  }
  cudaFree(dcand);
  cleanup();
  if (e != cudaSuccess)
    return fail(MHAR_ERR_CUDA, std::string(grid_form ? "prim_grid_kernel: " : "prim_kernel: ") +
                                   cudaGetErrorString(e));
  return 0;
}

int mhar_friedman_rafsky(const double* a, int64_t na, const double* b, int64_t nb, int64_t n,
                         int device, mhar_fr_result* out) {
  NvtxRange range("mhar.friedman_rafsky");
  if (!out) return fail(MHAR_ERR_INVALID_ARGUMENT, "friedman_rafsky: null result");
  if (!a || !b || na < 2 || nb < 2)
    return fail(MHAR_ERR_DEGENERATE_TEST,
                "DEGENERATE_TEST: friedman_rafsky: each sample needs at least two points");
  if (n < 1) return fail(MHAR_ERR_DIMENSION_MISMATCH, "friedman_rafsky: samples have no width");
  const int64_t N = na + nb;
  std::vector<double> pooled((size_t)N * n);
  std::memcpy(pooled.data(), a, sizeof(double) * na * n);
  std::memcpy(pooled.data() + na * n, b, sizeof(double) * nb * n);
  std::vector<int32_t> ea(N), eb(N);
  std::vector<double> ew(N);
  int st = mhar_minimum_spanning_tree(pooled.data(), N, n, device, ea.data(), eb.data(), ew.data());
  if (st) return st;
  // stats.cpp:115-142
  std::memset(out, 0, sizeof(*out));
  out->pooled_size = N;
  std::vector<int64_t> degree(N, 0);
  for (int64_t i = 0; i < N - 1; ++i) {
    ++degree[ea[i]];
    ++degree[eb[i]];
    if ((ea[i] < na) != (eb[i] < na)) ++out->cross_edges;
  }
  int64_t shared = 0;
  for (int64_t d : degree) shared += d * (d - 1) / 2;
  out->shared_end_pairs = shared;
  const double m = (double)na, np = (double)nb, bn = (double)N, two_mn = 2.0 * m * np;
  out->expected_cross = two_mn / bn + 1.0;
  const double cc = (double)shared;
  const double lead = two_mn / (bn * (bn - 1.0));
  out->variance_cross = lead * ((two_mn - bn) / bn + (cc - bn + 2.0) / ((bn - 2.0) * (bn - 3.0)) *
                                                         (bn * (bn - 1.0) - 2.0 * two_mn + 2.0));
  if (!(out->variance_cross > 0.0))
    return fail(MHAR_ERR_DEGENERATE_TEST, "DEGENERATE_TEST: friedman_rafsky: null variance " +
                                              std::to_string(out->variance_cross) +
                                              " is not positive");
  out->z_value = ((double)out->cross_edges - out->expected_cross) / std::sqrt(out->variance_cross);
  return 0;
}

int mhar_chebyshev_center(const mhar_polytope* p, int device, double* x_out, double* radius,
                          mhar_lp_stats* stats) {
  NvtxRange range("mhar.chebyshev_center");
  if (!p || !x_out || !radius) return fail(MHAR_ERR_INVALID_ARGUMENT, "chebyshev_center: null argument");
  if (p->n < 1) return fail(MHAR_ERR_INVALID_ARGUMENT, "chebyshev_center: dimension must be positive");
  if (p->m_in < 0 || p->m_eq < 0 || (p->m_in > 0 && (!p->a_in || !p->b_in)) ||
      (p->m_eq > 0 && (!p->a_eq || !p->b_eq)))
    return fail(MHAR_ERR_DIMENSION_MISMATCH, "chebyshev_center: inconsistent polytope arrays");
  mhar_lp::LpStats ls;
  std::string msg;
  const int st = mhar_lp::chebyshev_center(p->a_in, p->b_in, p->m_in, p->a_eq, p->b_eq, p->m_eq,
                                           p->n, device, x_out, radius, &ls, &msg);
  if (stats) {
    stats->rounds = ls.rounds;
    stats->reserved = 0;
    stats->pivots = ls.pivots;
    stats->working_rows = ls.working_rows;
  }
  if (st) return fail(st, msg);
  // chebyshev.cpp:61-63: the centre must pass containment at kLpFeasTol
  // (the inequality rows were checked on the device by the solver)
  const int64_t n = p->n;
  for (int64_t i = 0; i < p->m_eq; ++i) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s += p->a_eq[i + k * p->m_eq] * x_out[k];
    if (std::fabs(s - p->b_eq[i]) > 1e-8)
      return fail(MHAR_ERR_NUMERICAL_FAILURE,
                  "NUMERICAL_FAILURE: chebyshev_center: computed center fails containment");
  }
  return 0;
}

double mhar_flops_per_iterate(mhar_ctx* c) {
  if (!c) return 0.0;
  double f = 4.0 * (double)c->m * (double)c->n * (double)c->z;
  if (c->me > 0) f += 2.0 * (double)c->n * (double)c->n * (double)c->z;
  return f;
}

}  // extern "C"

// ===========================================================================
// Asynchronous building blocks of one context for the multi-device group
// (engine_internal.h, group.cu).
namespace mhar_internal {

int device(const mhar_ctx* c) { return c->device; }
cudaStream_t stream(const mhar_ctx* c) { return c->stream; }
int64_t walks(const mhar_ctx* c) { return c->z; }
int64_t dim(const mhar_ctx* c) { return c->n; }
unsigned long long* redraw_counter(mhar_ctx* c) { return c->redraw_total; }
std::string last_error() { return g_last_error; }
int set_error(int code, const std::string& msg) { return fail(code, msg); }

int run_begin(mhar_ctx* c, const double* x0) {
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(c->x0, x0, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  const int64_t total = c->z_pad * c->KT * BK;
  broadcast_state_kernel<<<blocks_for(total, 256, c->num_sms * 16), 256, 0, c->stream>>>(
      c->x0, c->n, c->z, c->z_pad, c->KT, c->X);
  LAUNCH_OK(c, "broadcast_state_kernel");
  int s = clear_error(c);
  if (s) return s;
  CK(cudaMemsetAsync(c->redraw_total, 0, sizeof(unsigned long long), c->stream));
  c->slack_valid = false;
  c->iterations = 0;
  return reset_streams(c);  // synchronises (x0 is the caller's host memory)
}

int advance(mhar_ctx* c, int64_t iters, int64_t reproject_every) {
  CK(cudaSetDevice(c->device));
  return ::advance(c, iters, reproject_every);
}

int collect(mhar_ctx* c, double* dev_rows, double* dev_viol) {
  CK(cudaSetDevice(c->device));
  int s = enqueue_check(c);
  if (s) return s;
  CK(cudaMemsetAsync(c->first_bad, 0x7F, sizeof(int), c->stream));
  contains_kernel<<<blocks_for(c->z, 256, 1 << 20), 256, 0, c->stream>>>(
      c->viol, c->me > 0 ? c->eqviol : nullptr, c->z, c->opt.eps_feas, c->err, 1, c->first_bad);
  LAUNCH_OK(c, "contains_kernel");
  if (dev_viol) {
    worst_violation_kernel<<<1, 1024, 0, c->stream>>>(c->viol, c->me > 0 ? c->eqviol : nullptr,
                                                      c->z, dev_viol);
    LAUNCH_OK(c, "worst_violation_kernel");
  }
  if (dev_rows) {
    unpack_b_kernel<<<blocks_for(c->n * c->z, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        c->X, c->n, c->z, c->KT, dev_rows);
    LAUNCH_OK(c, "unpack_b_kernel");
  }
  return 0;
}

int finish(mhar_ctx* c, int64_t* walk) {
  CK(cudaSetDevice(c->device));
  int64_t k = -1;
  const int s = read_error(c, &k);
  if (walk) *walk = s ? k + c->opt.chain_offset : -1;
  return s;
}

}  // namespace mhar_internal
