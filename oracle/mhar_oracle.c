/*
 * mhar_oracle.c -- CPU restatement of the reference MHAR hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see mhar_oracle.h): the checker for the GPU
 * product, never part of it.  Each function cites the reference lines it
 * restates; paths are relative to /root/reference/proj.
 *
 * Floating-point contract: built with -ffp-contract=off, so every product
 * and sum below rounds exactly as written.  Dot products accumulate with an
 * explicit fused multiply-add in ascending k order, which is what both the
 * reference's Eigen kernels and its loop-only ScalarWalk oracle
 * (tests/oracles.hpp:139-254) do on an FMA-capable x86 build.
 */
#include "mhar_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#if defined(__AVX512F__)
#include <immintrin.h>
#endif
#ifdef _OPENMP
#include <omp.h>
#endif

/* Status codes: 1 + mhar::ErrorCode ordinal (proj/include/mhar/errors.hpp:10-24). */
enum {
  ST_OK = 0,
  ST_INVALID_ARGUMENT = 1,
  ST_DIMENSION_MISMATCH = 2,
  ST_SINGULAR_MATRIX = 3,
  ST_RANK_DEFICIENT_EQ = 4,
  ST_UNBOUNDED_POLYTOPE = 7,
  ST_DIRECTION_DEGENERATE = 8,
  ST_RETRY_EXHAUSTED = 9,
  ST_NUMERICAL_FAILURE = 12,
};

/* Per-walk flag bits shared with include/mhar_b200.h. */
enum {
  FLAG_DEGENERATE = 1,
  FLAG_HAS_UPPER = 2,
  FLAG_HAS_LOWER = 4,
  FLAG_COLLAPSED = 8,
  FLAG_THETA_MIDPOINT = 16,
};

/* Constants: proj/include/mhar/sampler.hpp:40,43; projection.hpp:25;
 * sampler.cpp:16; rng.cpp:13-15. */
static const double kDegenerateWidth = 1e-14;
static const int kMaxDirectionRetries = 16;
static const double kNearZeroDirection = 1e-12;
static const int kMaxThetaRejects = 64;
static const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
static const uint64_t kStreamSalt = 0x6A09E667F3BCC909ULL;
static const double kTwoPi = 6.283185307179586; /* 2.0 * std::numbers::pi */
static const double kSingularRelTol = 1e-12;   /* linalg.hpp:13 */

/* ======================================================================== */
/* Streams: proj/src/rng.cpp:17-21, 101-113                                   */
/* ======================================================================== */

uint64_t orc_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t orc_stream_init(uint64_t seed, uint64_t stream) {
  return orc_mix64(seed + kGolden) ^ orc_mix64(stream + kStreamSalt);
}

uint64_t orc_next_u64(uint64_t* state) {
  *state += kGolden;
  return orc_mix64(*state);
}

double orc_next_uniform(uint64_t* state) {
  return (double)(orc_next_u64(state) >> 11) * 0x1.0p-53;
}

double orc_next_uniform_open(uint64_t* state) {
  return (double)((orc_next_u64(state) >> 11) + 1) * 0x1.0p-53;
}

/* ======================================================================== */
/* Box-Muller: proj/src/rng.cpp:46-66, 115-124; vmath.hpp:35-74              */
/* ======================================================================== */

/* glibc's vector math entry points, used in 8-lane batches exactly like
 * detail::log_batch / detail::sincos_batch when the reference is built with
 * libmvec on an AVX-512 host (vmath.hpp:14-27, 44-74). */
#if defined(__AVX512F__) && defined(ORC_HAVE_LIBMVEC)
__m512d _ZGVeN8v_sin(__m512d);
__m512d _ZGVeN8v_cos(__m512d);
__m512d _ZGVeN8v_log(__m512d);
#define ORC_VEC 8
#else
#define ORC_VEC 1
#endif

int orc_vector_math_width(void) { return ORC_VEC; }

static void sincos_scalar(double a, double* sn, double* cs) { sincos(a, sn, cs); }

static void log_batch(const double* x, double* out, size_t count) {
  size_t i = 0;
#if ORC_VEC == 8
  for (; i + 8 <= count; i += 8) _mm512_storeu_pd(out + i, _ZGVeN8v_log(_mm512_loadu_pd(x + i)));
#endif
  for (; i < count; ++i) out[i] = log(x[i]);
}

static void sincos_batch(const double* ang, double* sn, double* cs, size_t count) {
  size_t i = 0;
#if ORC_VEC == 8
  for (; i + 8 <= count; i += 8) {
    const __m512d a = _mm512_loadu_pd(ang + i);
    _mm512_storeu_pd(sn + i, _ZGVeN8v_sin(a));
    _mm512_storeu_pd(cs + i, _ZGVeN8v_cos(a));
  }
#endif
  for (; i < count; ++i) sincos_scalar(ang[i], sn + i, cs + i);
}

/* rng.cpp:46-66: radius = sqrt(-2 ln u1), angle = 2 pi u2, then sincos.
 * sqrt is correctly rounded in every lane width, so it is written scalar. */
static void transform_pairs(const double* u1, const double* u2, double* radius, double* sn,
                            double* cs, double* angle, size_t pairs) {
  log_batch(u1, radius, pairs);
  for (size_t i = 0; i < pairs; ++i) {
    radius[i] = sqrt(-2.0 * radius[i]);
    angle[i] = kTwoPi * u2[i];
  }
  sincos_batch(angle, sn, cs, pairs);
}

int orc_box_muller(double u1, double u2, double* c, double* s) {
  if (!(u1 > 0.0 && u1 <= 1.0) || !(u2 >= 0.0 && u2 < 1.0)) return ST_INVALID_ARGUMENT;
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = kTwoPi * u2;
  double sn = 0.0, cs = 0.0;
  sincos_scalar(angle, &sn, &cs);
  *c = radius * cs;
  *s = radius * sn;
  return ST_OK;
}

/* rng.cpp:136-151 */
void orc_fill_standard_normal(uint64_t* state, double* out, int64_t n) {
  const size_t pairs = (size_t)(n + 1) / 2;
  if (pairs == 0) return;
  double* buf = (double*)calloc(6 * pairs, sizeof(double));
  if (!buf) return;
  double *u1 = buf, *u2 = buf + pairs, *r = buf + 2 * pairs, *sn = buf + 3 * pairs,
         *cs = buf + 4 * pairs, *ang = buf + 5 * pairs;
  for (size_t p = 0; p < pairs; ++p) {
    u1[p] = orc_next_uniform_open(state);
    u2[p] = orc_next_uniform(state);
  }
  transform_pairs(u1, u2, r, sn, cs, ang, pairs);
  for (size_t p = 0; p < pairs; ++p) {
    out[2 * p] = r[p] * cs[p];
    if ((int64_t)(2 * p + 1) < n) out[2 * p + 1] = r[p] * sn[p];
  }
  free(buf);
}

/* rng.cpp:153-207: the pair batch runs over all columns back to back, so the
 * 8-lane/scalar-tail split follows the concatenated pair index. */
void orc_fill_standard_normal_matrix(uint64_t* col_states, int64_t z, double* out, int64_t n) {
  const size_t ppc = (size_t)(n + 1) / 2;
  const size_t pairs = ppc * (size_t)z;
  if (pairs == 0) return;
  double* buf = (double*)calloc(6 * pairs, sizeof(double));
  if (!buf) return;
  double *u1 = buf, *u2 = buf + pairs, *r = buf + 2 * pairs, *sn = buf + 3 * pairs,
         *cs = buf + 4 * pairs, *ang = buf + 5 * pairs;
  for (int64_t k = 0; k < z; ++k) {
    for (size_t p = 0; p < ppc; ++p) {
      u1[k * ppc + p] = orc_next_uniform_open(&col_states[k]);
      u2[k * ppc + p] = orc_next_uniform(&col_states[k]);
    }
  }
  transform_pairs(u1, u2, r, sn, cs, ang, pairs);
  for (int64_t k = 0; k < z; ++k) {
    double* col = out + (size_t)k * (size_t)n;
    const size_t base = (size_t)k * ppc;
    for (size_t p = 0; p < ppc; ++p) {
      col[2 * p] = r[base + p] * cs[base + p];
      if ((int64_t)(2 * p + 1) < n) col[2 * p + 1] = r[base + p] * sn[base + p];
    }
  }
  free(buf);
}

/* ======================================================================== */
/* Chord scan: proj/src/vmath.hpp:83-155 (scalar semantics; the SIMD paths   */
/* there are documented bit-identical to this loop)                          */
/* ======================================================================== */

void orc_chord_scan(const double* num, const double* den, int64_t count, double eps,
                    double* lower, double* upper, int* has_pos, int* has_neg) {
  double lo = -INFINITY, hi = INFINITY;
  int pos = 0, neg = 0;
  for (int64_t i = 0; i < count; ++i) {
    const double d = den[i];
    if (d > eps) {
      const double q = num[i] / d;
      pos = 1;
      if (q < hi) hi = q;
    } else if (d < -eps) {
      const double q = num[i] / d;
      neg = 1;
      if (q > lo) lo = q;
    }
  }
  *lower = lo;
  *upper = hi;
  *has_pos = pos;
  *has_neg = neg;
}

/* ======================================================================== */
/* GEMM: C = A * B, column-major, ascending-k FMA chain per element.         */
/* Register-blocked 24x8 AVX-512 micro-kernel over packed L2-resident A      */
/* panels; OpenMP over row blocks.  Result is identical to the naive loop    */
/*   for k: c = fma(a[i,k], b[k,j], c)                                       */
/* ======================================================================== */

static int g_threads = 0;
void orc_set_threads(int threads) { g_threads = threads; }
int orc_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

#define GM_MR 24
#define GM_NR 8
#define GM_KC 256
#define GM_MC 192

static void gemm_block(int64_t m, int64_t n, int64_t z, const double* A, const double* B,
                       double* C, int64_t i0, int64_t i1, double* apack) {
  for (int64_t k0 = 0; k0 < n; k0 += GM_KC) {
    const int64_t kc = (n - k0 < GM_KC) ? n - k0 : GM_KC;
    /* pack A[i0:i1, k0:k0+kc] as [micro-row-tile][k][24] with zero row padding */
    const int64_t tiles = (i1 - i0 + GM_MR - 1) / GM_MR;
    for (int64_t t = 0; t < tiles; ++t) {
      for (int64_t k = 0; k < kc; ++k) {
        double* dst = apack + (t * kc + k) * GM_MR;
        for (int64_t r = 0; r < GM_MR; ++r) {
          const int64_t i = i0 + t * GM_MR + r;
          dst[r] = (i < i1) ? A[i + (k0 + k) * m] : 0.0;
        }
      }
    }
    for (int64_t j0 = 0; j0 < z; j0 += GM_NR) {
      const int64_t nr = (z - j0 < GM_NR) ? z - j0 : GM_NR;
      const double* bcol[GM_NR];
      for (int64_t c = 0; c < GM_NR; ++c) bcol[c] = B + (j0 + (c < nr ? c : 0)) * n + k0;
      for (int64_t t = 0; t < tiles; ++t) {
        const int64_t ib = i0 + t * GM_MR;
        const int64_t mr = (i1 - ib < GM_MR) ? i1 - ib : GM_MR;
        const double* ap = apack + t * kc * GM_MR;
#if defined(__AVX512F__)
        __m512d acc[3][GM_NR];
        for (int c = 0; c < GM_NR; ++c) {
          for (int v = 0; v < 3; ++v) {
            if (k0 == 0 || c >= nr) {
              acc[v][c] = _mm512_setzero_pd();
            } else {
              const int64_t rows_left = mr - v * 8;
              const __mmask8 mk = rows_left >= 8 ? 0xFF
                                  : rows_left <= 0 ? 0
                                                   : (__mmask8)((1u << rows_left) - 1);
              acc[v][c] = _mm512_maskz_loadu_pd(mk, C + ib + v * 8 + (j0 + c) * m);
            }
          }
        }
        for (int64_t k = 0; k < kc; ++k) {
          const __m512d a0 = _mm512_loadu_pd(ap + k * GM_MR);
          const __m512d a1 = _mm512_loadu_pd(ap + k * GM_MR + 8);
          const __m512d a2 = _mm512_loadu_pd(ap + k * GM_MR + 16);
#pragma GCC unroll 8
          for (int c = 0; c < GM_NR; ++c) {
            const __m512d bv = _mm512_set1_pd(bcol[c][k]);
            acc[0][c] = _mm512_fmadd_pd(a0, bv, acc[0][c]);
            acc[1][c] = _mm512_fmadd_pd(a1, bv, acc[1][c]);
            acc[2][c] = _mm512_fmadd_pd(a2, bv, acc[2][c]);
          }
        }
        for (int c = 0; c < nr; ++c) {
          for (int v = 0; v < 3; ++v) {
            const int64_t rows_left = mr - v * 8;
            if (rows_left <= 0) continue;
            const __mmask8 mk = rows_left >= 8 ? 0xFF : (__mmask8)((1u << rows_left) - 1);
            _mm512_mask_storeu_pd(C + ib + v * 8 + (j0 + c) * m, mk, acc[v][c]);
          }
        }
#else
        for (int64_t c = 0; c < nr; ++c) {
          for (int64_t r = 0; r < mr; ++r) {
            double s = (k0 == 0) ? 0.0 : C[ib + r + (j0 + c) * m];
            for (int64_t k = 0; k < kc; ++k) s = fma(ap[k * GM_MR + r], bcol[c][k], s);
            C[ib + r + (j0 + c) * m] = s;
          }
        }
#endif
      }
    }
  }
}

void orc_gemm(int64_t m, int64_t n, int64_t z, const double* A, const double* B, double* C) {
  if (m <= 0 || z <= 0) return;
  if (n <= 0) {
    for (int64_t j = 0; j < z; ++j) memset(C + j * m, 0, sizeof(double) * (size_t)m);
    return;
  }
  const int64_t blocks = (m + GM_MC - 1) / GM_MC;
#pragma omp parallel num_threads(orc_get_threads())
  {
    double* apack = (double*)aligned_alloc(64, sizeof(double) * GM_KC * (GM_MC + GM_MR));
#pragma omp for schedule(dynamic, 1)
    for (int64_t blk = 0; blk < blocks; ++blk) {
      const int64_t i0 = blk * GM_MC;
      const int64_t i1 = (i0 + GM_MC < m) ? i0 + GM_MC : m;
      gemm_block(m, n, z, A, B, C, i0, i1, apack);
    }
    free(apack);
  }
}

/* ======================================================================== */
/* Chord intervals: proj/src/sampler.cpp:150-208 (+ scan_column :40-46)     */
/* ======================================================================== */

/* Walk chunk so the m x chunk slack/rate scratch stays bounded; the
 * reference materialises all z columns at once (sampler.cpp:164-176), which
 * changes memory, not values. */
#define LI_CHUNK 64

int orc_lambda_intervals(const double* A, const double* b, int64_t m, int64_t n,
                         const double* X, const double* D, int64_t z, double eps_dir,
                         double* lower, double* upper, uint8_t* degenerate, uint8_t* sides,
                         int64_t* err_chain) {
  const int64_t chunk = z < LI_CHUNK ? z : LI_CHUNK;
  double* xd = (double*)malloc(sizeof(double) * (size_t)(n * 2 * chunk));
  double* prod = (double*)malloc(sizeof(double) * (size_t)(m * 2 * chunk));
  int64_t first_bad = -1;
  for (int64_t k0 = 0; k0 < z && first_bad < 0; k0 += chunk) {
    const int64_t kc = (z - k0 < chunk) ? z - k0 : chunk;
    memcpy(xd, X + k0 * n, sizeof(double) * (size_t)(n * kc));
    memcpy(xd + n * kc, D + k0 * n, sizeof(double) * (size_t)(n * kc));
    orc_gemm(m, n, 2 * kc, A, xd, prod); /* [A x | A d] */
    double* ax = prod;
    double* ad = prod + m * kc;
    int64_t bad = -1;
#pragma omp parallel for num_threads(orc_get_threads()) schedule(static)
    for (int64_t c = 0; c < kc; ++c) {
      double* col = ax + c * m;
      for (int64_t i = 0; i < m; ++i) col[i] = -col[i] + b[i]; /* (-ax).colwise() + b */
      double lo, hi;
      int pos, neg;
      orc_chord_scan(col, ad + c * m, m, eps_dir, &lo, &hi, &pos, &neg);
      const int64_t k = k0 + c;
      if (sides) sides[k] = (uint8_t)((pos ? FLAG_HAS_UPPER : 0) | (neg ? FLAG_HAS_LOWER : 0));
      if (!pos && !neg) {
        lower[k] = 0.0;
        upper[k] = 0.0;
        degenerate[k] = 1;
      } else if (!pos || !neg) {
#pragma omp critical
        if (bad < 0 || k < bad) bad = k;
        lower[k] = lo;
        upper[k] = hi;
        degenerate[k] = 1;
      } else {
        lower[k] = lo;
        upper[k] = hi;
        degenerate[k] = !(hi - lo > kDegenerateWidth);
      }
    }
    first_bad = bad;
  }
  free(xd);
  free(prod);
  if (first_bad >= 0) {
    if (err_chain) *err_chain = first_bad;
    return ST_UNBOUNDED_POLYTOPE;
  }
  return ST_OK;
}

/* ======================================================================== */
/* Linear algebra: proj/src/linalg.cpp:21-52; projection.cpp:9-60           */
/* ======================================================================== */

/* LU with partial pivoting (Eigen::PartialPivLU), pivot test against
 * kSingularRelTol * max|a|, inverse by solving for I, then one correction
 * pass X <- X + X (I - A X). */
int orc_invert(const double* a, int64_t n, double* inv) {
  if (n <= 0) return ST_INVALID_ARGUMENT;
  double scale = 0.0;
  for (int64_t i = 0; i < n * n; ++i) {
    const double v = fabs(a[i]);
    if (!isfinite(a[i])) return ST_SINGULAR_MATRIX;
    if (v > scale) scale = v;
  }
  if (scale == 0.0) return ST_SINGULAR_MATRIX;
  double* lu = (double*)malloc(sizeof(double) * (size_t)(n * n));
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  memcpy(lu, a, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t c = 0; c < n; ++c) {
    int64_t piv = c;
    double best = fabs(lu[c + c * n]);
    for (int64_t r = c + 1; r < n; ++r) {
      if (fabs(lu[r + c * n]) > best) {
        best = fabs(lu[r + c * n]);
        piv = r;
      }
    }
    if (piv != c) {
      for (int64_t j = 0; j < n; ++j) {
        const double t = lu[c + j * n];
        lu[c + j * n] = lu[piv + j * n];
        lu[piv + j * n] = t;
      }
      const int64_t t = perm[c];
      perm[c] = perm[piv];
      perm[piv] = t;
    }
    const double p = lu[c + c * n];
    if (p != 0.0) {
      for (int64_t r = c + 1; r < n; ++r) lu[r + c * n] /= p;
      for (int64_t j = c + 1; j < n; ++j) {
        const double f = lu[c + j * n];
        for (int64_t r = c + 1; r < n; ++r) lu[r + j * n] -= lu[r + c * n] * f;
      }
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    if (!(fabs(lu[i + i * n]) > kSingularRelTol * scale)) {
      free(lu);
      free(perm);
      return ST_SINGULAR_MATRIX;
    }
  }
  /* solve L U x = e_perm for every column of I */
  for (int64_t col = 0; col < n; ++col) {
    double* x = inv + col * n;
    for (int64_t i = 0; i < n; ++i) x[i] = (perm[i] == col) ? 1.0 : 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t r = i + 1; r < n; ++r) x[r] -= lu[r + i * n] * x[i];
    for (int64_t i = n - 1; i >= 0; --i) {
      x[i] /= lu[i + i * n];
      for (int64_t r = 0; r < i; ++r) x[r] -= lu[r + i * n] * x[i];
    }
  }
  /* residual = I - a inv; inv += inv residual */
  double* res = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* corr = (double*)malloc(sizeof(double) * (size_t)(n * n));
  orc_gemm(n, n, n, a, inv, res);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) res[i + j * n] = (i == j ? 1.0 : 0.0) - res[i + j * n];
  orc_gemm(n, n, n, inv, res, corr);
  for (int64_t i = 0; i < n * n; ++i) inv[i] += corr[i];
  free(res);
  free(corr);
  free(lu);
  free(perm);
  return ST_OK;
}

/* projection.cpp:9-34: P = I - A_E' (A_E A_E')^-1 A_E */
int orc_compute_projection(const double* AE, int64_t me, int64_t n, double* P, double* Ginv) {
  if (me == 0) return ST_INVALID_ARGUMENT;
  if (me >= n) return ST_RANK_DEFICIENT_EQ;
  double* aet = (double*)malloc(sizeof(double) * (size_t)(n * me)); /* n x me */
  for (int64_t i = 0; i < me; ++i)
    for (int64_t j = 0; j < n; ++j) aet[j + i * n] = AE[i + j * me];
  double* gram = (double*)malloc(sizeof(double) * (size_t)(me * me));
  orc_gemm(me, n, me, AE, aet, gram);
  int st = orc_invert(gram, me, Ginv);
  if (st == ST_SINGULAR_MATRIX) st = ST_RANK_DEFICIENT_EQ;
  if (st == ST_OK) {
    double* lift = (double*)malloc(sizeof(double) * (size_t)(n * me));
    orc_gemm(n, me, me, aet, Ginv, lift);
    orc_gemm(n, me, n, lift, AE, P);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) P[i + j * n] = (i == j ? 1.0 : 0.0) - P[i + j * n];
    free(lift);
  }
  free(aet);
  free(gram);
  return st;
}

/* projection.cpp:53-60: X <- X - A_E' (Ginv (A_E X - b_E)) */
int orc_reproject(const double* AE, const double* Ginv, const double* bE, int64_t me, int64_t n,
                  double* X, int64_t z) {
  double* r = (double*)malloc(sizeof(double) * (size_t)(me * z));
  double* g = (double*)malloc(sizeof(double) * (size_t)(me * z));
  double* aet = (double*)malloc(sizeof(double) * (size_t)(n * me));
  double* corr = (double*)malloc(sizeof(double) * (size_t)(n * z));
  orc_gemm(me, n, z, AE, X, r);
  for (int64_t k = 0; k < z; ++k)
    for (int64_t i = 0; i < me; ++i) r[i + k * me] -= bE[i];
  orc_gemm(me, me, z, Ginv, r, g);
  for (int64_t i = 0; i < me; ++i)
    for (int64_t j = 0; j < n; ++j) aet[j + i * n] = AE[i + j * me];
  orc_gemm(n, me, z, aet, g, corr);
  for (int64_t i = 0; i < n * z; ++i) X[i] -= corr[i];
  free(r);
  free(g);
  free(aet);
  free(corr);
  return ST_OK;
}

/* polytope.cpp:177-190 */
int orc_contains(const double* A, const double* b, int64_t m, const double* AE, const double* bE,
                 int64_t me, int64_t n, const double* x, double eps) {
  if (m > 0) {
    double* ax = (double*)malloc(sizeof(double) * (size_t)m);
    orc_gemm(m, n, 1, A, x, ax);
    double worst = -INFINITY;
    for (int64_t i = 0; i < m; ++i) {
      const double v = ax[i] - b[i];
      if (v > worst || isnan(v)) worst = isnan(v) ? INFINITY : v;
    }
    free(ax);
    if (worst > eps) return 0;
  }
  if (me > 0) {
    double* ax = (double*)malloc(sizeof(double) * (size_t)me);
    orc_gemm(me, n, 1, AE, x, ax);
    double worst = 0.0;
    for (int64_t i = 0; i < me; ++i) {
      const double v = fabs(ax[i] - bE[i]);
      if (v > worst || isnan(v)) worst = isnan(v) ? INFINITY : v;
    }
    free(ax);
    if (worst > eps) return 0;
  }
  return 1;
}

/* polytope.cpp:192-208 */
void orc_make_hypercube(int64_t n, double* A, double* b) {
  memset(A, 0, sizeof(double) * (size_t)(2 * n * n));
  for (int64_t i = 0; i < n; ++i) {
    A[i + i * 2 * n] = 1.0;
    A[(n + i) + i * 2 * n] = -1.0;
  }
  for (int64_t i = 0; i < 2 * n; ++i) b[i] = 1.0;
}

void orc_make_simplex(int64_t n, double* A, double* b, double* AE, double* bE) {
  memset(A, 0, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n; ++i) {
    A[i + i * n] = -1.0;
    b[i] = 0.0;
    AE[i] = 1.0;
  }
  bE[0] = 1.0;
}

/* ======================================================================== */
/* step: proj/src/sampler.cpp:73-123, 95-101, 235-272                        */
/* ======================================================================== */

static double col_norm(const double* d, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += d[i] * d[i];
  return sqrt(s);
}

/* sampler.cpp:210-212 */
static double chord_point(double u, double lower, double upper) {
  return lower + u * (upper - lower);
}

/* sampler.cpp:95-101 */
static double draw_theta(uint64_t* theta_state, double lower, double upper) {
  for (int attempt = 0; attempt < kMaxThetaRejects; ++attempt) {
    const double theta = chord_point(orc_next_uniform(theta_state), lower, upper);
    if (theta > lower && theta < upper) return theta;
  }
  return chord_point(0.5, lower, upper);
}

/* sampler.cpp:73-93: returns ST_OK and sets *degenerate, or UNBOUNDED */
static int column_interval(const double* A, const double* b, int64_t m, int64_t n,
                           const double* x, const double* d, double eps_dir, double* lo,
                           double* hi, int* degenerate) {
  double* xd = (double*)malloc(sizeof(double) * (size_t)(2 * n));
  double* prod = (double*)malloc(sizeof(double) * (size_t)(2 * m));
  memcpy(xd, x, sizeof(double) * (size_t)n);
  memcpy(xd + n, d, sizeof(double) * (size_t)n);
  orc_gemm(m, n, 2, A, xd, prod);
  for (int64_t i = 0; i < m; ++i) prod[i] = b[i] - prod[i];
  int pos, neg;
  orc_chord_scan(prod, prod + m, m, eps_dir, lo, hi, &pos, &neg);
  free(xd);
  free(prod);
  *degenerate = !(*hi - *lo > kDegenerateWidth);
  if (!pos && !neg) {
    *degenerate = 1;
    return ST_OK;
  }
  if (!pos || !neg) return ST_UNBOUNDED_POLYTOPE;
  return ST_OK;
}

int orc_step(const double* A, const double* b, int64_t m, int64_t n, const double* P,
             double eps_dir, uint64_t* col_states, uint64_t* theta_state, double* X, int64_t z,
             int64_t* redraws, int64_t* err_chain) {
  const size_t nz = (size_t)(n * z);
  double* h = (double*)malloc(sizeof(double) * nz);
  double* d = (double*)malloc(sizeof(double) * nz);
  double* lo = (double*)malloc(sizeof(double) * (size_t)z);
  double* hi = (double*)malloc(sizeof(double) * (size_t)z);
  uint8_t* degen = (uint8_t*)malloc((size_t)z);
  uint8_t* collapsed = (uint8_t*)calloc((size_t)z, 1);
  int st = ST_OK;

  orc_fill_standard_normal_matrix(col_states, z, h, n);
  if (P) {
    orc_gemm(n, n, z, P, h, d);
    for (int64_t k = 0; k < z; ++k)
      if (col_norm(d + k * n, n) <= kNearZeroDirection) collapsed[k] = 1;
  } else {
    memcpy(d, h, sizeof(double) * nz);
  }
  st = orc_lambda_intervals(A, b, m, n, X, d, z, eps_dir, lo, hi, degen, NULL, err_chain);
  if (st != ST_OK) goto done;
  for (int64_t k = 0; k < z; ++k)
    if (collapsed[k]) degen[k] = 1;

  for (int64_t k = 0; k < z && st == ST_OK; ++k) {
    if (!degen[k]) continue;
    /* redraw_column, sampler.cpp:105-123 */
    int ok = 0;
    for (int attempt = 0; attempt < kMaxDirectionRetries; ++attempt) {
      ++*redraws;
      double* hk = (P ? h : d) + k * n;
      double* dk = d + k * n;
      orc_fill_standard_normal(&col_states[k], hk, n);
      if (P) {
        orc_gemm(n, n, 1, P, hk, dk);
        if (col_norm(dk, n) <= kNearZeroDirection) continue;
      }
      double l, u;
      int dg;
      const int cs = column_interval(A, b, m, n, X + k * n, dk, eps_dir, &l, &u, &dg);
      if (cs != ST_OK) {
        st = cs;
        if (err_chain) *err_chain = k;
        break;
      }
      if (!dg) {
        lo[k] = l;
        hi[k] = u;
        degen[k] = 0;
        ok = 1;
        break;
      }
    }
    if (st == ST_OK && !ok) {
      st = ST_RETRY_EXHAUSTED;
      if (err_chain) *err_chain = k;
    }
  }
  if (st != ST_OK) goto done;

  for (int64_t k = 0; k < z; ++k) {
    const double theta = draw_theta(theta_state, lo[k], hi[k]);
    double* xk = X + k * n;
    const double* dk = d + k * n;
    for (int64_t i = 0; i < n; ++i) xk[i] = xk[i] + theta * dk[i];
  }
done:
  free(h);
  free(d);
  free(lo);
  free(hi);
  free(degen);
  free(collapsed);
  return st;
}

int orc_step_injected(const double* A, const double* b, int64_t m, int64_t n, const double* P,
                      double eps_dir, double* X, int64_t z, const double* H, const double* U,
                      double* lower, double* upper, double* theta, uint8_t* flags,
                      int64_t* err_chain) {
  const size_t nz = (size_t)(n * z);
  double* d = (double*)malloc(sizeof(double) * nz);
  uint8_t* degen = (uint8_t*)malloc((size_t)z);
  uint8_t* sides = (uint8_t*)malloc((size_t)z);
  if (P) {
    orc_gemm(n, n, z, P, H, d);
  } else {
    memcpy(d, H, sizeof(double) * nz);
  }
  int st = orc_lambda_intervals(A, b, m, n, X, d, z, eps_dir, lower, upper, degen, sides,
                                err_chain);
  if (st == ST_OK) {
    for (int64_t k = 0; k < z; ++k) {
      uint8_t f = sides[k];
      if (degen[k]) f |= FLAG_DEGENERATE;
      if (P && col_norm(d + k * n, n) <= kNearZeroDirection) f |= FLAG_COLLAPSED | FLAG_DEGENERATE;
      double t = 0.0;
      if (!(f & FLAG_DEGENERATE)) {
        t = chord_point(U[k], lower[k], upper[k]);
        if (!(t > lower[k] && t < upper[k])) {
          t = chord_point(0.5, lower[k], upper[k]);
          f |= FLAG_THETA_MIDPOINT;
        }
        double* xk = X + k * n;
        const double* dk = d + k * n;
        for (int64_t i = 0; i < n; ++i) xk[i] = xk[i] + t * dk[i];
      }
      if (theta) theta[k] = t;
      flags[k] = f;
    }
  }
  free(d);
  free(degen);
  free(sides);
  return st;
}

/* ======================================================================== */
/* run: proj/src/sampler.cpp:274-335, warm start x0 for chebyshev_center     */
/* ======================================================================== */

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int orc_run(const double* A, const double* b, int64_t m, const double* AE, const double* bE,
            int64_t me, int64_t n, const orc_run_config* cfg, const double* x0, double* samples,
            orc_run_stats* stats) {
  const int64_t z = cfg->z;
  if (z < 1 || cfg->phi < 1 || cfg->t_target < 1 || !(cfg->eps_dir > 0) || !(cfg->eps_feas > 0))
    return ST_INVALID_ARGUMENT;
  const double t0 = now_seconds();
  double* P = NULL;
  double* Ginv = NULL;
  int st = ST_OK;
  if (me > 0) {
    P = (double*)malloc(sizeof(double) * (size_t)(n * n));
    Ginv = (double*)malloc(sizeof(double) * (size_t)(me * me));
    st = orc_compute_projection(AE, me, n, P, Ginv);
    if (st != ST_OK) {
      free(P);
      free(Ginv);
      return st;
    }
  }
  const int64_t windows = (cfg->t_target + z - 1) / z;
  double* X = (double*)malloc(sizeof(double) * (size_t)(n * z));
  for (int64_t k = 0; k < z; ++k) memcpy(X + k * n, x0, sizeof(double) * (size_t)n);
  uint64_t* cols = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)z);
  for (int64_t k = 0; k < z; ++k) cols[k] = orc_stream_init(cfg->seed, (uint64_t)k);
  uint64_t theta = orc_stream_init(cfg->seed, ~(uint64_t)0);
  int64_t redraws = 0, err_chain = -1, global_iter = 0, row = 0;

#define ADVANCE()                                                                          \
  do {                                                                                     \
    st = orc_step(A, b, m, n, P, cfg->eps_dir, cols, &theta, X, z, &redraws, &err_chain); \
    if (st != ST_OK) goto out;                                                             \
    ++global_iter;                                                                         \
    if (P && cfg->reproject_every > 0 && global_iter % cfg->reproject_every == 0)          \
      orc_reproject(AE, Ginv, bE, me, n, X, z);                                            \
  } while (0)

  for (int64_t i = 0; i < cfg->burn_in; ++i) ADVANCE();
  for (int64_t w = 0; w < windows; ++w) {
    for (int64_t i = 0; i < cfg->phi; ++i) ADVANCE();
    for (int64_t k = 0; k < z; ++k) {
      if (!orc_contains(A, b, m, AE, bE, me, n, X + k * n, cfg->eps_feas)) {
        st = ST_NUMERICAL_FAILURE;
        err_chain = k;
        goto out;
      }
      if (samples)
        for (int64_t i = 0; i < n; ++i) samples[row * n + i] = X[k * n + i];
      ++row;
    }
  }
#undef ADVANCE
out:
  if (stats) {
    stats->windows = windows;
    stats->iterate_count = z * cfg->phi * windows;
    stats->redraw_count = redraws;
    stats->err_chain = err_chain;
    stats->seconds = now_seconds() - t0;
  }
  free(X);
  free(cols);
  free(P);
  free(Ginv);
  return st;
}

/* ======================================================================== */
/* Production-mode draws: the engine's Philox4x32-10 keying                  */
/* ======================================================================== */
/*
 * The reference draws from SplitMix streams (restated above); the engine's
 * production mode draws the same uniforms' roles from Philox4x32-10 (Salmon,
 * Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3", SC'11 --
 * the published algorithm, pinned below to its authors' known-answer vectors
 * in tests/test_oracle_kats.py), keyed on (seed, global walk, iterate,
 * attempt, domain) as include/mhar_b200.h documents.  orc_step_philox is the
 * reference step (sampler.cpp:235-272) driven by those draws, so the
 * engine's default path can be compared with the reference algorithm
 * iterate by iterate.  Test infrastructure only.
 */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += W0;
    k1 += W1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* Two 64-bit words for (seed; index, walk, iterate, attempt, domain):
 * counter (index, walk lo32, iterate lo32, iterate bits 32..47 | attempt
 * (6 bits) << 16 | walk bits 32..39 << 22 | domain << 30), key = seed. */
void orc_philox_u64x2(uint64_t seed, uint32_t index, uint64_t walk, uint64_t iterate,
                      uint32_t attempt, uint32_t domain, uint64_t* a, uint64_t* b) {
  const uint32_t ctr[4] = {index, (uint32_t)walk, (uint32_t)iterate,
                           ((uint32_t)(iterate >> 32) & 0xFFFFu) | ((attempt & 0x3Fu) << 16) |
                               (((uint32_t)(walk >> 32) & 0xFFu) << 22) | (domain << 30)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t r[4];
  orc_philox4x32_10(ctr, key, r);
  *a = ((uint64_t)r[0] << 32) | r[1];
  *b = ((uint64_t)r[2] << 32) | r[3];
}

enum { kDomNormal = 0, kDomTheta = 1 };

/* Column of standard normals for (walk, iterate, attempt): pair p from
 * Philox index p -- u1 = open (0,1] from word a, u2 = [0,1) from word b --
 * then the reference's Box-Muller (rng.cpp:115-124), odd n dropping the
 * last sine (rng.hpp:57-64). */
void orc_philox_normals(uint64_t seed, uint64_t walk, uint64_t iterate, uint32_t attempt,
                        double* out, int64_t n) {
  for (int64_t p = 0; 2 * p < n; ++p) {
    uint64_t a, b;
    orc_philox_u64x2(seed, (uint32_t)p, walk, iterate, attempt, kDomNormal, &a, &b);
    const double u1 = (double)((a >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(b >> 11) * 0x1.0p-53;
    double c, s;
    orc_box_muller(u1, u2, &c, &s);
    out[2 * p] = c;
    if (2 * p + 1 < n) out[2 * p + 1] = s;
  }
}

/* draw_theta (sampler.cpp:95-101) with rejection draw r from Philox index r
 * of the theta domain. */
static double draw_theta_philox(uint64_t seed, uint64_t walk, uint64_t iterate, double lower,
                                double upper, int* midpoint) {
  for (int r = 0; r < kMaxThetaRejects; ++r) {
    uint64_t a, b;
    orc_philox_u64x2(seed, (uint32_t)r, walk, iterate, 0, kDomTheta, &a, &b);
    const double theta = chord_point((double)(a >> 11) * 0x1.0p-53, lower, upper);
    if (theta > lower && theta < upper) return theta;
  }
  *midpoint = 1;
  return chord_point(0.5, lower, upper);
}

int orc_step_philox(const double* A, const double* b, int64_t m, int64_t n, const double* P,
                    double eps_dir, uint64_t seed, int64_t chain_offset, uint64_t iterate,
                    double* X, int64_t z, int64_t* redraws, int64_t* err_chain) {
  const size_t nz = (size_t)(n * z);
  double* h = (double*)calloc(nz ? nz : 1, sizeof(double));
  double* d = (double*)malloc(sizeof(double) * (nz ? nz : 1));
  double* lo = (double*)malloc(sizeof(double) * (size_t)(z > 0 ? z : 1));
  double* hi = (double*)malloc(sizeof(double) * (size_t)(z > 0 ? z : 1));
  uint8_t* degen = (uint8_t*)malloc((size_t)(z > 0 ? z : 1));
  uint8_t* collapsed = (uint8_t*)calloc((size_t)(z > 0 ? z : 1), 1);
  int st = ST_OK;
  if (!h || !d || !lo || !hi || !degen || !collapsed) {
    st = ST_NUMERICAL_FAILURE;
    goto done;
  }

  for (int64_t k = 0; k < z; ++k)
    orc_philox_normals(seed, (uint64_t)(chain_offset + k), iterate, 0, h + k * n, n);
  if (P) {
    orc_gemm(n, n, z, P, h, d);
    for (int64_t k = 0; k < z; ++k)
      if (col_norm(d + k * n, n) <= kNearZeroDirection) collapsed[k] = 1;
  } else {
    memcpy(d, h, sizeof(double) * nz);
  }
  st = orc_lambda_intervals(A, b, m, n, X, d, z, eps_dir, lo, hi, degen, NULL, err_chain);
  if (st != ST_OK) goto done;
  for (int64_t k = 0; k < z; ++k)
    if (collapsed[k]) degen[k] = 1;
  /* redraw_column (sampler.cpp:105-123): attempt a of walk k draws from
   * Philox attempt a + 1 */
  for (int64_t k = 0; k < z && st == ST_OK; ++k) {
    if (!degen[k]) continue;
    int ok = 0;
    for (int attempt = 0; attempt < kMaxDirectionRetries; ++attempt) {
      ++*redraws;
      double* hk = (P ? h : d) + k * n;
      double* dk = d + k * n;
      orc_philox_normals(seed, (uint64_t)(chain_offset + k), iterate, (uint32_t)(attempt + 1),
                         hk, n);
      if (P) {
        orc_gemm(n, n, 1, P, hk, dk);
        if (col_norm(dk, n) <= kNearZeroDirection) continue;
      }
      double l, u;
      int dg;
      const int cs = column_interval(A, b, m, n, X + k * n, dk, eps_dir, &l, &u, &dg);
      if (cs != ST_OK) {
        st = cs;
        if (err_chain) *err_chain = k;
        break;
      }
      if (!dg) {
        lo[k] = l;
        hi[k] = u;
        degen[k] = 0;
        ok = 1;
        break;
      }
    }
    if (st == ST_OK && !ok) {
      st = ST_RETRY_EXHAUSTED;
      if (err_chain) *err_chain = k;
    }
  }
  if (st != ST_OK) goto done;
  for (int64_t k = 0; k < z; ++k) {
    int mid = 0;
    const double theta =
        draw_theta_philox(seed, (uint64_t)(chain_offset + k), iterate, lo[k], hi[k], &mid);
    double* xk = X + k * n;
    const double* dk = d + k * n;
    for (int64_t i = 0; i < n; ++i) xk[i] = xk[i] + theta * dk[i];
  }
done:
  free(h);
  free(d);
  free(lo);
  free(hi);
  free(degen);
  free(collapsed);
  return st;
}
