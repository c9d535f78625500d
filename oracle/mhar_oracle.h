/*
 * mhar_oracle.h -- CPU restatement of the reference MHAR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the GPU product is
 * compared against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline
 * and --impl reference arm).  The product path never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj, cited per declaration).  The reference itself cannot
 * be compiled in this image (Eigen3 and the vendored headers are missing, see
 * DESIGN.md "Oracle"), so this restatement is pinned against the reference's
 * own known-answer tests instead (tests/test_oracle_kats.py, tests/golden/).
 *
 * Matrices are column-major doubles, exactly like the reference's
 * Eigen::MatrixXd.  Status codes are 0 = OK, else 1 + the reference
 * mhar::ErrorCode ordinal (proj/include/mhar/errors.hpp:10-24), the same
 * numbering include/mhar_b200.h exports.
 */
#ifndef MHAR_ORACLE_H
#define MHAR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- counter streams: proj/src/rng.cpp:13-21, 101-113 ------------------- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_stream_init(uint64_t seed, uint64_t stream);
uint64_t orc_next_u64(uint64_t* state);
double orc_next_uniform(uint64_t* state);
double orc_next_uniform_open(uint64_t* state);

/* ---- Box-Muller: proj/src/rng.cpp:115-124 -------------------------------- */
int orc_box_muller(double u1, double u2, double* c, double* s);

/* proj/src/rng.cpp:136-151: one column, 2*ceil(n/2) draws, batched transform */
void orc_fill_standard_normal(uint64_t* state, double* out, int64_t n);
/* proj/src/rng.cpp:153-207: n x z, column k from col_states[k] */
void orc_fill_standard_normal_matrix(uint64_t* col_states, int64_t z, double* out, int64_t n);
/* 1 when the libmvec batched transcendental path is active (vmath.hpp:14-27) */
int orc_vector_math_width(void);

/* ---- chord scan: proj/src/vmath.hpp:83-155 ------------------------------- */
void orc_chord_scan(const double* num, const double* den, int64_t count, double eps,
                    double* lower, double* upper, int* has_pos, int* has_neg);

/* ---- dense products (sequential-k FMA order, cache blocked, OpenMP) ------ */
/* C (m x z) = A (m x n) * B (n x z), all column-major. */
void orc_gemm(int64_t m, int64_t n, int64_t z, const double* A, const double* B, double* C);
void orc_set_threads(int threads);
int orc_get_threads(void);

/* ---- chord intervals: proj/src/sampler.cpp:150-208 ------------------------
 * lower/upper/degenerate per walk; returns 7 (UNBOUNDED_POLYTOPE) for the
 * first one-sided walk, writing its index to *err_chain. */
int orc_lambda_intervals(const double* A, const double* b, int64_t m, int64_t n,
                         const double* X, const double* D, int64_t z, double eps_dir,
                         double* lower, double* upper, uint8_t* degenerate,
                         uint8_t* sides, int64_t* err_chain);

/* ---- linear algebra: proj/src/linalg.cpp:21-52, projection.cpp:9-60 ------ */
int orc_invert(const double* a, int64_t n, double* inv);
int orc_compute_projection(const double* AE, int64_t me, int64_t n, double* P, double* Ginv);
int orc_reproject(const double* AE, const double* Ginv, const double* bE, int64_t me,
                  int64_t n, double* X, int64_t z);
/* proj/src/polytope.cpp:177-190; AE may be NULL when me == 0 */
int orc_contains(const double* A, const double* b, int64_t m, const double* AE,
                 const double* bE, int64_t me, int64_t n, const double* x, double eps);
/* proj/src/polytope.cpp:192-208 */
void orc_make_hypercube(int64_t n, double* A /*2n x n*/, double* b /*2n*/);
void orc_make_simplex(int64_t n, double* A /*n x n*/, double* b, double* AE /*1 x n*/,
                      double* bE);

/* ---- one iterate with reference streams: proj/src/sampler.cpp:235-272 ----
 * col_states[z] and *theta_state advance exactly as WalkRng would.  P is the
 * n x n projector or NULL.  On error *err_chain names the walk. */
int orc_step(const double* A, const double* b, int64_t m, int64_t n, const double* P,
             double eps_dir, uint64_t* col_states, uint64_t* theta_state, double* X,
             int64_t z, int64_t* redraws, int64_t* err_chain);

/* ---- one iterate with injected normals H (n x z) and uniforms U (z) ------
 * The test hook semantics shared with mhar_step_injected (include/mhar_b200.h):
 * D = P*H (or H), chords as sampler.cpp:150-208, flagged walks stay put,
 * theta = lower + U[k]*(upper-lower), an endpoint hit takes the midpoint.
 * flags: MHAR_FLAG_* bits.  theta may be NULL. */
int orc_step_injected(const double* A, const double* b, int64_t m, int64_t n,
                      const double* P, double eps_dir, double* X, int64_t z,
                      const double* H, const double* U, double* lower, double* upper,
                      double* theta, uint8_t* flags, int64_t* err_chain);

/* ---- production-mode draws: the engine's Philox4x32-10 keying -----------
 * Philox4x32-10 (Salmon et al., SC'11), counter ctr, key key -> out.  Draw
 * (a, b) for (seed; index, walk, iterate, attempt, domain) as the engine
 * keys it (include/mhar_b200.h MHAR_RNG_PHILOX).  orc_philox_normals fills
 * one walk's column (pair p from index p, Box-Muller as rng.cpp:115-124).
 * orc_step_philox is orc_step (sampler.cpp:235-272) with these draws: the
 * first direction from attempt 0, redraw a from attempt a + 1, theta
 * rejection r from index r of the theta domain.  No projector
 * factoring and no walk interaction: the reference algorithm, only the
 * random source differs. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void orc_philox_u64x2(uint64_t seed, uint32_t index, uint64_t walk, uint64_t iterate,
                      uint32_t attempt, uint32_t domain, uint64_t* a, uint64_t* b);
void orc_philox_normals(uint64_t seed, uint64_t walk, uint64_t iterate, uint32_t attempt,
                        double* out, int64_t n);
int orc_step_philox(const double* A, const double* b, int64_t m, int64_t n, const double* P,
                    double eps_dir, uint64_t seed, int64_t chain_offset, uint64_t iterate,
                    double* X, int64_t z, int64_t* redraws, int64_t* err_chain);

/* ---- full run with warm start: proj/src/sampler.cpp:274-335 --------------
 * x0 (n) replaces chebyshev_center (sampler.cpp:276); cfg already resolved.
 * samples: (windows*z) x n row-major, collection order. */
typedef struct {
  int64_t z, phi, t_target, burn_in, reproject_every;
  uint64_t seed;
  double eps_dir, eps_feas;
} orc_run_config;
typedef struct {
  int64_t windows, iterate_count, redraw_count, err_chain;
  double seconds;
} orc_run_stats;
int orc_run(const double* A, const double* b, int64_t m, const double* AE, const double* bE,
            int64_t me, int64_t n, const orc_run_config* cfg, const double* x0,
            double* samples, orc_run_stats* stats);

/* ---- two-sample tree test: proj/src/stats.cpp:50-143 ----------------------
 * Prim MST of N points (row-major N x n), vertices entering in index order,
 * strict-< updates (ties keep the earlier candidate).  Edges in insertion
 * order: (ea[i], eb[i]) with weight ew[i]. */
int orc_minimum_spanning_tree(const double* pts, int64_t N, int64_t n, int32_t* ea, int32_t* eb,
                              double* ew);
typedef struct {
  int64_t cross_edges;
  double expected_cross, variance_cross, z_value;
  int64_t shared_end_pairs, pooled_size;
} orc_fr_result;
/* a: na x n, b: nb x n, row-major; DEGENERATE_TEST (11) / DIMENSION_MISMATCH */
int orc_friedman_rafsky(const double* a, int64_t na, const double* b, int64_t nb, int64_t n,
                        orc_fr_result* out);

#ifdef __cplusplus
}
#endif
#endif
