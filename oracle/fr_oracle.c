/*
 * fr_oracle.c -- CPU restatement of the reference's two-sample tree test
 * (proj/src/stats.cpp:50-143): Prim minimum spanning tree of the pooled
 * points and the Friedman-Rafsky cross-edge statistic.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the GPU implementation
 * (mhar_friedman_rafsky in include/mhar_b200.h).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "mhar_oracle.h"

/* stats.cpp:50-91 -- vertices enter in index order; strict-< updates keep
 * the earlier candidate on ties. */
int orc_minimum_spanning_tree(const double* pts, int64_t N, int64_t n, int32_t* ea, int32_t* eb,
                              double* ew) {
  if (N < 2) return 1; /* INVALID_ARGUMENT */
  double* best = (double*)malloc(sizeof(double) * (size_t)N);
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  char* in_tree = (char*)calloc((size_t)N, 1);
  for (int64_t v = 0; v < N; ++v) {
    best[v] = INFINITY;
    parent[v] = -1;
  }
  best[0] = 0.0;
  int64_t ne = 0;
  for (int64_t added = 0; added < N; ++added) {
    int64_t u = -1;
    double key = INFINITY;
    for (int64_t v = 0; v < N; ++v)
      if (!in_tree[v] && best[v] < key) {
        key = best[v];
        u = v;
      }
    in_tree[u] = 1;
    if (parent[u] >= 0) {
      ea[ne] = parent[u];
      eb[ne] = (int32_t)u;
      ew[ne] = sqrt(key);
      ++ne;
    }
    const double* pu = pts + u * n;
    for (int64_t v = 0; v < N; ++v) {
      if (in_tree[v]) continue;
      const double* pv = pts + v * n;
      double d2 = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        const double t = pv[k] - pu[k];
        d2 += t * t;
      }
      if (d2 < best[v]) {
        best[v] = d2;
        parent[v] = (int32_t)u;
      }
    }
  }
  free(best);
  free(parent);
  free(in_tree);
  return 0;
}

/* stats.cpp:93-143 */
int orc_friedman_rafsky(const double* a, int64_t na, const double* b, int64_t nb, int64_t n,
                        orc_fr_result* out) {
  if (na < 2 || nb < 2) return 11; /* DEGENERATE_TEST */
  const int64_t N = na + nb;
  double* pooled = (double*)malloc(sizeof(double) * (size_t)(N * n));
  memcpy(pooled, a, sizeof(double) * (size_t)(na * n));
  memcpy(pooled + na * n, b, sizeof(double) * (size_t)(nb * n));
  int32_t* ea = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  int32_t* eb = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  double* ew = (double*)malloc(sizeof(double) * (size_t)N);
  orc_minimum_spanning_tree(pooled, N, n, ea, eb, ew);
  int64_t* degree = (int64_t*)calloc((size_t)N, sizeof(int64_t));
  memset(out, 0, sizeof(*out));
  out->pooled_size = N;
  for (int64_t i = 0; i < N - 1; ++i) {
    ++degree[ea[i]];
    ++degree[eb[i]];
    if ((ea[i] < na) != (eb[i] < na)) ++out->cross_edges;
  }
  int64_t shared = 0;
  for (int64_t v = 0; v < N; ++v) shared += degree[v] * (degree[v] - 1) / 2;
  out->shared_end_pairs = shared;
  const double m = (double)na, np = (double)nb, bn = (double)N, two_mn = 2.0 * m * np;
  out->expected_cross = two_mn / bn + 1.0;
  const double c = (double)shared;
  const double lead = two_mn / (bn * (bn - 1.0));
  out->variance_cross = lead * ((two_mn - bn) / bn + (c - bn + 2.0) / ((bn - 2.0) * (bn - 3.0)) *
                                                         (bn * (bn - 1.0) - 2.0 * two_mn + 2.0));
  int st = 0;
  if (!(out->variance_cross > 0.0)) {
    st = 11;
  } else {
    out->z_value = ((double)out->cross_edges - out->expected_cross) / sqrt(out->variance_cross);
  }
  free(pooled);
  free(ea);
  free(eb);
  free(ew);
  free(degree);
  return st;
}
