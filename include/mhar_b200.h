/*
 * mhar_b200.h -- C ABI of the B200-native MHAR (Matrix Hit-and-Run) chain-step
 * engine.  Plain pointers and sizes only; no CUDA, torch or C++ types.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj, paths below relative to it):
 *
 *   reference interface                                   replaced by
 *   ----------------------------------------------------  -------------------------
 *   mhar::Polytope (include/mhar/polytope.hpp:12-25)       mhar_polytope + ctx upload
 *   mhar::SamplerConfig (include/mhar/sampler.hpp:16-25)   mhar_options / mhar_run_config
 *   mhar::WalkRng (include/mhar/rng.hpp:42-55)             device counters (Philox or the
 *                                                          reference SplitMix streams)
 *   mhar::WalkState (include/mhar/sampler.hpp:69-74)       mhar_set_state / mhar_get_state
 *   mhar::step (include/mhar/sampler.hpp:79-80,            mhar_step
 *               src/sampler.cpp:235-272)
 *   mhar::compute_lambda_intervals (sampler.hpp:53-58,     mhar_lambda_intervals
 *               src/sampler.cpp:150-208)
 *   mhar::run (include/mhar/sampler.hpp:99,                mhar_run (+ warm start x0,
 *               src/sampler.cpp:274-335)                   which replaces :276)
 *   mhar::compute_projection (include/mhar/projection.hpp:33,
 *               src/projection.cpp:9-34)                   mhar_compute_projection (host)
 *   mhar::reproject_points (projection.hpp:35)             inside mhar_step / mhar_run
 *   mhar::contains (polytope.hpp:57, src/polytope.cpp:177) mhar_check_state
 *   mhar::Error / ErrorCode (include/mhar/errors.hpp)      int status + mhar_last_error
 *
 * Matrices are column-major doubles (the reference's Eigen::MatrixXd layout,
 * include/mhar/linalg.hpp:7-10) unless stated.  Every function returns an int
 * status: MHAR_OK (0) or 1 + the reference ErrorCode ordinal; MHAR_ERR_CUDA
 * for a device/runtime failure, which the reference has no code for.
 * mhar_last_error() returns the thread-local message of the last failure.
 * A context is bound to one CUDA device and is not thread-safe; a group
 * (mhar_group_*) drives several devices from one process.
 */
#ifndef MHAR_B200_H
#define MHAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1 + mhar::ErrorCode ordinal (errors.hpp:10-24) ------- */
#define MHAR_OK 0
#define MHAR_ERR_INVALID_ARGUMENT 1
#define MHAR_ERR_DIMENSION_MISMATCH 2
#define MHAR_ERR_SINGULAR_MATRIX 3
#define MHAR_ERR_RANK_DEFICIENT_EQ 4
#define MHAR_ERR_EMPTY_POLYTOPE 5
#define MHAR_ERR_NO_INTERIOR 6
#define MHAR_ERR_UNBOUNDED_POLYTOPE 7
#define MHAR_ERR_DIRECTION_DEGENERATE 8
#define MHAR_ERR_RETRY_EXHAUSTED 9
#define MHAR_ERR_CYCLE_SUSPECTED 10
#define MHAR_ERR_DEGENERATE_TEST 11
#define MHAR_ERR_NUMERICAL_FAILURE 12
#define MHAR_ERR_IO_FAILURE 13
#define MHAR_ERR_CUDA 100

/* ---- per-walk flag bits (mhar_step_injected / mhar_lambda_intervals) ----- */
#define MHAR_FLAG_DEGENERATE 1      /* LambdaIntervals::degenerate (sampler.hpp:33-37) */
#define MHAR_FLAG_HAS_UPPER 2       /* some rate > eps_dir (chord_scan has_pos) */
#define MHAR_FLAG_HAS_LOWER 4       /* some rate < -eps_dir (chord_scan has_neg) */
#define MHAR_FLAG_COLLAPSED 8       /* ||P h|| <= 1e-12 (projection.hpp:25) */
#define MHAR_FLAG_THETA_MIDPOINT 16 /* theta hit an endpoint; midpoint taken */

/* ---- options ------------------------------------------------------------- */
#define MHAR_RNG_PHILOX 0    /* Philox4x32-10 keyed (seed, global walk, iterate, attempt) */
#define MHAR_RNG_REFERENCE 1 /* the reference's SplitMix64 streams, bit-exact uniforms
                                (rng.cpp:13-21,101-113); single device only */

#define MHAR_SLACK_RECOMPUTE 0   /* every iterate: one fused pass A_I [X | D] + chord reduce */
#define MHAR_SLACK_INCREMENTAL 1 /* A_I D + streamed slack b - A_I X, refreshed by a fused
                                    pass every refresh_every iterates */

typedef struct {
  int64_t n;          /* dimension */
  int64_t m_in;       /* inequality rows */
  int64_t m_eq;       /* equality rows (0 = full dimensional) */
  const double* a_in; /* m_in x n, column-major */
  const double* b_in; /* m_in */
  const double* a_eq; /* m_eq x n, column-major; NULL when m_eq == 0 */
  const double* b_eq; /* m_eq */
} mhar_polytope;

typedef struct {
  int64_t z;             /* walks on this device (the shard) */
  int64_t chain_offset;  /* global id of local walk 0; RNG is keyed on global ids */
  uint64_t seed;         /* SamplerConfig::seed */
  double eps_dir;        /* SamplerConfig::eps_dir (1e-11) */
  double eps_feas;       /* SamplerConfig::eps_feas (1e-9) */
  int rng;               /* MHAR_RNG_* */
  int slack_mode;        /* MHAR_SLACK_* */
  int64_t refresh_every; /* incremental mode: fused refresh cadence (0 = default 128) */
  int device;            /* CUDA ordinal */
  int small_path;        /* 1 (default): bodies whose A_I, P, A_E fit in shared memory run
                            all iterates of a batch in one walk-resident launch (Philox only) */
  int precision;         /* 64 (default): fp64 DMMA.  32: the fp32 variant -- rates A_I d on
                            tcgen05 tensor cores with fp32 accuracy (kind::f16 with per-row /
                            per-walk power-of-two scales, A_I as two halves; MHAR_TC_F16=0:
                            kind::tf32 hi/lo split), fp64 slack/state, chords of
                            {A_I x <= b_I - fp32_margin}; the slack refresh and every
                            containment check use the caller's fp64 A_I */
  double fp32_margin;    /* precision 32: slack margin mu (0 = default 2e-5) */
  int f64_engine;        /* precision 64 only.  MHAR_F64_DMMA (default): A_I d on the fp64
                            tensor cores (DMMA).  MHAR_F64_INT8: A_I d formed exactly from
                            53-bit fixed-point operands split into int8 slices on the
                            tcgen05 int8 tensor cores (Ozaki scheme, fp64-accurate rates,
                            n <= 4608); refreshes and containment checks stay on DMMA */
  int fp32_direction;    /* precision 32 only.  MHAR_FP32_DIR_SPLIT (default): the walk moves
                            along its fp64 direction; the tensor cores see it split into two
                            operands (~22 bits).  MHAR_FP32_DIR_ROUNDED: the fast form -- the
                            direction is rounded to one fp16 (per-walk scale) / TF32 operand
                            and the walk moves along that rounded direction (one MMA fewer
                            per k step); bodies with equalities always split */
  int64_t z_plan;        /* 0 (default): z.  The walk count the kernel choices are made for
                            (walk-resident kernel or chain, its lanes per walk): a shard of a
                            larger run passes the run's total so every sharding takes the same
                            kernels and the samples stay bit-identical (mhar_group sets it) */
} mhar_options;

#define MHAR_FP32_DIR_SPLIT 0
#define MHAR_FP32_DIR_ROUNDED 1

#define MHAR_F64_DMMA 0
#define MHAR_F64_INT8 1

/* Fills o with the reference defaults (sampler.hpp:16-25): eps_dir 1e-11,
 * eps_feas 1e-9, Philox, incremental slack, device 0. */
void mhar_default_options(mhar_options* o);

typedef struct mhar_ctx mhar_ctx;

/* Uploads the polytope (the device copy is re-laid out for the tensor-core
 * tiles), the projector P = I - A_E'(A_E A_E')^-1 A_E and G = (A_E A_E')^-1
 * (projection.hpp:11-15; NULL both to have them computed on the host with
 * mhar_compute_projection), allocates the z-walk state.  The state starts at
 * 0; set it with mhar_set_state. */
int mhar_ctx_create(const mhar_polytope* p, const double* projector, const double* gram_inverse,
                    const mhar_options* opt, mhar_ctx** out);
int mhar_ctx_destroy(mhar_ctx* ctx);

/* WalkState.x (sampler.hpp:70): n x z column-major host buffer. */
int mhar_set_state(mhar_ctx* ctx, const double* x);
int mhar_get_state(mhar_ctx* ctx, double* x);
/* Row-major z x n copy of the state into device memory owned by the caller
 * (the sample layout of SampleSet::samples, sampler.hpp:83); used to gather
 * samples across ranks without a host round trip. */
int mhar_get_state_rows_device(mhar_ctx* ctx, double* dev_rows);
/* Test hook: the last iterate's directions D (n x z column-major, as moved
 * along -- quantised by the int8-slice engine) and chord bounds / positions
 * (z each).  Any pointer may be NULL. */
int mhar_debug_last_iterate(mhar_ctx* ctx, double* d, double* lower, double* upper, double* theta);

/* `iters` iterates of every walk (step(), sampler.cpp:235-272).  When the
 * polytope has equalities and reproject_every > 0, walks are pulled back onto
 * {A_E x = b_E} whenever the context's global iterate count is a multiple of
 * reproject_every (run(), sampler.cpp:304-311).  Kernels are queued without a
 * host sync; the first device-side error (lowest walk of the earliest phase,
 * sampler.cpp ordering) is returned by the next synchronising call. */
int mhar_step(mhar_ctx* ctx, int64_t iters, int64_t reproject_every);
/* Waits for queued work and reports a pending device-side error. */
int mhar_sync(mhar_ctx* ctx);
/* Checkpoint / resume: with Philox directions the walk state is
 * X (mhar_get_state) plus this iterate counter, which keys every draw of
 * the next iterate; a fresh context given the same options, X
 * (mhar_set_state) and the counter continues the same chain.  Reference
 * streams carry per-walk state instead: INVALID_ARGUMENT there. */
int mhar_get_iteration(mhar_ctx* ctx, int64_t* iteration);
int mhar_set_iteration(mhar_ctx* ctx, int64_t iteration);
/* Incremental slack mode: the next iterate recomputes the slack cache from a
 * fresh product (the refresh pass that otherwise recurs every refresh_every
 * iterates), e.g. to time a whole refresh cycle. */
int mhar_request_refresh(mhar_ctx* ctx);
/* WalkRng state (rng.hpp:42-55) of a reference-stream context: the z column
 * stream states and the shared theta stream state, exactly the uint64
 * counters RngStream holds (rng.hpp:16-33).  Moving them to another context
 * continues the same streams (a rebind to another polytope, or checkpoint /
 * resume in MHAR_RNG_REFERENCE mode).  INVALID_ARGUMENT on a Philox context. */
int mhar_get_streams(mhar_ctx* ctx, uint64_t* col_states, uint64_t* theta_state);
int mhar_set_streams(mhar_ctx* ctx, const uint64_t* col_states, const uint64_t* theta_state);
/* mhar_step bracketed by CUDA events on the context's stream; *device_ms is
 * the device time of the `iters` iterates (synchronises). */
int mhar_step_timed(mhar_ctx* ctx, int64_t iters, int64_t reproject_every, double* device_ms);

/* Test hook: one iterate with the normals H (n x z, column-major) and chord
 * positions U (z) injected from the host instead of the device RNG.  D = P H
 * (or H); chords as compute_lambda_intervals; flagged walks stay put; other
 * walks take theta = lower + U[k] (upper - lower) (an endpoint hit takes the
 * midpoint) and x += theta d.  Outputs may be NULL.  Always a fresh fused
 * pass (never the incremental slack). */
int mhar_step_injected(mhar_ctx* ctx, const double* h, const double* u, double* lower,
                       double* upper, double* theta, uint8_t* flags);

/* generate_directions (sampler.hpp:46, sampler.cpp:143-148): the next n x z
 * batch of standard normals from the walks' streams (column k from walk k's
 * stream, 2*ceil(n/2) draws), advancing them; column-major into h. */
int mhar_generate_directions(mhar_ctx* ctx, double* h);

/* select_points (sampler.hpp:66-67, sampler.cpp:214-233): for every walk
 * theta from the theta stream, uniform on the open chord (lower, upper),
 * out = x + theta d (n x z column-major).  DIRECTION_DEGENERATE if any walk
 * is flagged in `degenerate` (nonzero), before any draw. */
int mhar_select_points(mhar_ctx* ctx, const double* x, const double* d, const double* lower,
                       const double* upper, const uint8_t* degenerate, double* out);

/* compute_lambda_intervals for host X and D (n x z each) against the
 * context's polytope; does not move the state.  degenerate gets
 * MHAR_FLAG_* bits.  UNBOUNDED_POLYTOPE names the first one-sided walk. */
int mhar_lambda_intervals(mhar_ctx* ctx, const double* x, const double* d, double* lower,
                          double* upper, uint8_t* flags);

/* contains() (polytope.cpp:177-190) for every walk of the current state:
 * *first_bad = lowest walk outside by more than eps (or -1); max_viol gets
 * max_i (A_I x - b_I)_i and max_eq max |A_E x - b_E| per walk (z each, may be
 * NULL). */
int mhar_check_state(mhar_ctx* ctx, double eps, int64_t* first_bad, double* max_viol,
                     double* max_eq);

typedef struct {
  int64_t phi;             /* iterates between collections */
  int64_t windows;         /* collections; SampleSet::windows */
  int64_t burn_in;         /* iterates before the first window */
  int64_t reproject_every; /* 0 = off */
} mhar_run_config;

typedef struct {
  int64_t iterate_count; /* z * phi * windows (burn-in excluded), sampler.cpp:332 */
  int64_t windows;
  int64_t redraw_count;  /* direction redraw attempts, sampler.cpp:110 */
  int64_t err_walk;      /* walk named by a failure, else -1 */
  double seconds;        /* device time of the walk section (CUDA events) */
} mhar_run_stats;

/* run() with a warm start (sampler.cpp:274-335 with x0 in place of the
 * Chebyshev center, :276/:300): state <- x0 replicated, burn-in, then per
 * window phi iterates, a contains(eps_feas) check of every walk
 * (NUMERICAL_FAILURE otherwise) and collection of the z walks as rows of
 * samples ((windows*z) x n row-major, collection order).  samples may be NULL
 * (throughput runs). */
int mhar_run(mhar_ctx* ctx, const mhar_run_config* cfg, const double* x0, double* samples,
             mhar_run_stats* stats);

/* Host-side projector (projection.cpp:9-34 with linalg.cpp:21-52 LU + one
 * refinement pass): P (n x n) and G = (A_E A_E')^-1 (m_eq x m_eq). */
int mhar_compute_projection(const double* a_eq, int64_t m_eq, int64_t n, double* p, double* g);

typedef struct {
  int64_t iterations;      /* iterates executed by this context */
  int64_t redraw_count;    /* total redraw attempts */
  int64_t kernel_launches; /* kernels this library launched */
  int64_t chord_launches;  /* launches of the chord (tensor-core) kernel */
  double chord_ms;         /* summed device time of timed chord launches */
  int64_t chord_timed;     /* chord launches covered by chord_ms */
  double chord_flops;      /* algorithmic flops of those timed launches */
  int64_t refreshes;       /* fused refresh passes (incremental mode) */
  int64_t z, z_padded, m_padded, n_padded;
  int64_t chord_kernel;    /* the kernel computing the chords (mhar_chord_kernel) */
} mhar_ctx_stats;

/* mhar_ctx_stats.chord_kernel */
enum mhar_chord_kernel {
  MHAR_CHORD_SMALL = 1,  /* small_kernel: whole iterate per walk in one launch */
  MHAR_CHORD_DMMA = 2,   /* chord_kernel / chord2_kernel: DMMA, 64-walk units */
  MHAR_CHORD_DMMA3 = 3,  /* chord3_kernel: DMMA, 128-walk units, TMEM hand-off */
  MHAR_CHORD_TC32 = 4,   /* chord_tc32_kernel: fp32 variant on tcgen05 */
  MHAR_CHORD_INT8 = 5,   /* chord_i8_kernel: fp64 from int8 slices on tcgen05 */
  MHAR_CHORD_DIAG = 6    /* diag_chord_kernel: stacked diagonal blocks */
};

int mhar_get_stats(mhar_ctx* ctx, mhar_ctx_stats* out);
/* 1 = record CUDA events around every chord launch (on the launching stream) */
int mhar_set_timing(mhar_ctx* ctx, int enabled);
int mhar_reset_stats(mhar_ctx* ctx);

/* Algorithmic flops of one iterate of this context's walks (4 m n z, + 2 n^2 z
 * with equalities) and of its dominant chord launch. */
double mhar_flops_per_iterate(mhar_ctx* ctx);

/* ---- several GPUs driven by one host process ---------
 * run() / step() over z_total walks split into contiguous shards across
 * `devices` (the first z_total % ndev shards one walk larger), A_I, b_I and
 * P replicated on every device.  Walk k of the whole set draws on global id
 * opt->chain_offset + k, so samples, states and errors are identical
 * whatever the device list (Philox; the reference streams cannot be sharded:
 * one theta stream is shared by every walk, rng.hpp:42-55, so ndev > 1 with
 * MHAR_RNG_REFERENCE is INVALID_ARGUMENT).  One host thread per device
 * issues its shard's iterates; nothing moves between GPUs per iterate.  At
 * every collection window the shards' rows are gathered to devices[0] with
 * grouped ncclSend / ncclRecv and the diagnostics (worst containment slack,
 * redraw count) all-reduced with ncclAllReduce over NVLink; with one device,
 * a device listed twice, or no libnccl.so.2, the gather is a peer copy into
 * the root's window buffer (MHAR_GROUP_NCCL=0 forces that, =1 uses NCCL even
 * for one device).  Replaces the single-process multi-GPU loop around
 * mhar::run (sampler.cpp:274-335).  opt->z = z_total; opt->device ignored. */
typedef struct mhar_group mhar_group;
#define MHAR_GROUP_MAX_DEV 16
typedef struct {
  int ndev;
  int uses_nccl;              /* 1: NCCL gather + all-reduce; 0: peer copies */
  int64_t z_total;
  int devices[MHAR_GROUP_MAX_DEV];
  int64_t z[MHAR_GROUP_MAX_DEV];       /* walks per shard */
  int64_t offset[MHAR_GROUP_MAX_DEV];  /* global id of each shard's first walk */
  double last_max_violation;  /* max_k max_i (A x - b)_i of the last collection, all shards */
  int64_t last_redraws;       /* redraw attempts of the last run, all shards */
  int gather;                 /* how windows reach devices[0] (mhar_group_gather) */
} mhar_group_info_t;

/* mhar_group_info_t.gather; MHAR_GROUP_GATHER=direct|nccl|copy overrides the
 * default (direct wherever every shard's device can reach devices[0]). */
enum mhar_group_gather {
  MHAR_GATHER_COPY = 0,   /* rows staged per shard, copy-engine peer copy to the root */
  MHAR_GATHER_NCCL = 1,   /* rows staged per shard, grouped ncclSend / ncclRecv + ncclAllReduce */
  MHAR_GATHER_DIRECT = 2  /* each shard's containment-check + unpack kernel stores its rows
                             straight into the root's window buffer over NVLink peer memory */
};

int mhar_group_create(const mhar_polytope* p, const double* projector, const double* gram_inverse,
                      const mhar_options* opt, const int* devices, int ndev, mhar_group** out);
int mhar_group_destroy(mhar_group* g);
int mhar_group_info(mhar_group* g, mhar_group_info_t* info);
/* Shard i's single-device context (stats, timing); NULL when out of range. */
mhar_ctx* mhar_group_context(mhar_group* g, int i);
/* n x z_total column-major, like mhar_set_state / mhar_get_state. */
int mhar_group_set_state(mhar_group* g, const double* x);
int mhar_group_get_state(mhar_group* g, double* x);
/* `iters` iterates of every walk on every device, then waits for all. */
int mhar_group_step(mhar_group* g, int64_t iters, int64_t reproject_every);
/* run() with warm start x0 over all shards; samples ((windows*z_total) x n
 * row-major, collection order, walks in global order) assembled on
 * devices[0] and streamed to the host overlapped with the next window.
 * stats->seconds is host wall time of the whole run; err_walk the lowest
 * failing global walk. */
int mhar_group_run(mhar_group* g, const mhar_run_config* cfg, const double* x0, double* samples,
                   mhar_run_stats* stats);

/* ---- two-sample uniformity test ----------------------
 * minimum_spanning_tree (stats.hpp:31, stats.cpp:50-91): Prim over N points
 * (row-major N x n) on GPU `device`; N - 1 edges in insertion order. */
int mhar_minimum_spanning_tree(const double* points, int64_t N, int64_t n, int device,
                               int32_t* edge_a, int32_t* edge_b, double* edge_w);

/* MstTestResult (stats.hpp:34-41). */
typedef struct {
  int64_t cross_edges;
  double expected_cross;
  double variance_cross;
  double z_value;
  int64_t shared_end_pairs;
  int64_t pooled_size;
} mhar_fr_result;

/* friedman_rafsky (stats.hpp:50, stats.cpp:93-143): a (na x n) and b (nb x n)
 * row-major; DEGENERATE_TEST when a sample has < 2 points or the null
 * variance is not positive. */
int mhar_friedman_rafsky(const double* a, int64_t na, const double* b, int64_t nb, int64_t n,
                         int device, mhar_fr_result* out);

typedef struct mhar_lp_stats {
  int32_t rounds;        /* constraint-generation rounds (LP solves) */
  int32_t reserved;
  int64_t pivots;        /* simplex pivots over all rounds */
  int64_t working_rows;  /* inequality rows in the final working set */
} mhar_lp_stats;

/* chebyshev_center (chebyshev.hpp:22-25, chebyshev.cpp:45-66): the centre
 * and radius of the largest ball inside p, the start point run() uses when no
 * x0 is given (sampler.cpp:276).  The reference solves the LP of
 * build_chebyshev_lp (chebyshev.cpp:9-43) with a dense tableau over all rows
 * (lp.cpp:120-297); here constraint generation keeps a working set of rows in
 * a GPU-resident tableau and scans all rows for violations on the GPU.
 * Errors as the reference: EMPTY_POLYTOPE (infeasible), UNBOUNDED_POLYTOPE,
 * NO_INTERIOR (radius <= 1e-10), NUMERICAL_FAILURE (centre fails
 * containment at 1e-8), CYCLE_SUSPECTED (pivot budget).  stats may be NULL. */
int mhar_chebyshev_center(const mhar_polytope* p, int device, double* x_out, double* radius,
                          mhar_lp_stats* stats);

const char* mhar_last_error(void);
const char* mhar_version(void);
int mhar_device_count(int* count);

#ifdef __cplusplus
}
#endif
#endif
