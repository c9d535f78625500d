// stats_kernels.cuh -- the two-sample tree test on the GPU
// (/root/reference/proj/src/stats.cpp:50-143): Prim's
// minimum spanning tree over the pooled points, O(N^2) distance work done by
// one CTA of 1024 threads per tree, vertex selection by a block argmin.
#pragma once

#include "common.cuh"

namespace mhar_dev {

constexpr int PRIM_THREADS = 1024;

// P: n x N (coordinate-major, so thread v's coordinates are coalesced across
// the block).  Vertices enter in index order, ties keep the earlier
// candidate, d2 accumulated in ascending coordinate order without FMA
// contraction -- the reference's loop (stats.cpp:67-89).
__global__ void __launch_bounds__(PRIM_THREADS) prim_kernel(const double* __restrict__ P, int64_t N,
                                                            int64_t n, double* __restrict__ best,
                                                            int* __restrict__ parent,
                                                            unsigned char* __restrict__ in_tree,
                                                            int* ea, int* eb, double* ew) {
  __shared__ double rv[PRIM_THREADS / 32];
  __shared__ long long ri[PRIM_THREADS / 32];
  __shared__ long long s_u;
  __shared__ double s_key;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t v = tid; v < N; v += PRIM_THREADS) {
    best[v] = __longlong_as_double(0x7FF0000000000000LL);
    parent[v] = -1;
    in_tree[v] = 0;
  }
  __syncthreads();
  long long u = 0;
  double key = 0.0;
  int64_t ne = 0;
  for (int64_t added = 0; added < N; ++added) {
    if (tid == 0) {
      in_tree[u] = 1;
      if (parent[u] >= 0) {
        ea[ne] = parent[u];
        eb[ne] = (int)u;
        ew[ne] = sqrt(key);
      }
    }
    if (added > 0) ++ne;  // uniform across threads: every vertex after the first adds an edge
    __syncthreads();
    double lb = __longlong_as_double(0x7FF0000000000000LL);
    long long li = 0x7FFFFFFFFFFFFFFFLL;
    for (int64_t v = tid; v < N; v += PRIM_THREADS) {
      if (in_tree[v]) continue;
      double d2 = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        const double t = __dsub_rn(P[k * N + v], P[k * N + u]);
        d2 = __dadd_rn(d2, __dmul_rn(t, t));
      }
      double bv = best[v];
      if (d2 < bv) {
        bv = d2;
        best[v] = d2;
        parent[v] = (int)u;
      }
      if (bv < lb) {  // v ascending within a thread: strict < keeps the earliest
        lb = bv;
        li = v;
      }
    }
    // block argmin, ties -> smallest index
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xFFFFFFFFu, lb, o);
      const long long oi = __shfl_xor_sync(0xFFFFFFFFu, li, o);
      if (ov < lb || (ov == lb && oi < li)) {
        lb = ov;
        li = oi;
      }
    }
    if (lane == 0) {
      rv[warp] = lb;
      ri[warp] = li;
    }
    __syncthreads();
    if (warp == 0) {
      lb = lane < PRIM_THREADS / 32 ? rv[lane] : __longlong_as_double(0x7FF0000000000000LL);
      li = lane < PRIM_THREADS / 32 ? ri[lane] : 0x7FFFFFFFFFFFFFFFLL;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, lb, o);
        const long long oi = __shfl_xor_sync(0xFFFFFFFFu, li, o);
        if (ov < lb || (ov == lb && oi < li)) {
          lb = ov;
          li = oi;
        }
      }
      if (lane == 0) {
        s_u = li;
        s_key = lb;
      }
    }
    __syncthreads();
    u = s_u;
    key = s_key;
    if (u == 0x7FFFFFFFFFFFFFFFLL) break;  // all vertices in the tree
  }
}

}  // namespace mhar_dev
