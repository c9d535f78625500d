// stats_kernels.cuh -- the two-sample tree test on the GPU
// (/root/reference/proj/src/stats.cpp:50-143): Prim's
// minimum spanning tree over the pooled points, O(N^2) distance work done by
// one CTA of 1024 threads per tree, vertex selection by a block argmin
// (prim_kernel, small pools); for pools beyond a few thousand points the
// grid-wide variant (prim_grid_kernel) spreads the points over every SM.
#pragma once

#include <cooperative_groups.h>

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

// ---------------------------------------------------------------------------
// Grid-wide Prim: a cooperative launch of one CTA per SM.  CTA g owns the
// contiguous point range [g*chunk, (g+1)*chunk); per added vertex u every CTA
// relaxes its points against u (the same ascending-coordinate, no-FMA d2 as
// prim_kernel), publishes its (key, index, parent) argmin, and after one grid
// barrier every CTA reduces the G candidates itself -- the same
// lexicographic (key, index) minimum, so all CTAs agree on the next vertex
// and the tree equals prim_kernel's (and the reference's) edge for edge.
constexpr int PRIM_GRID_THREADS = 256;
constexpr int PRIM_GRID_SMEM_COORDS = 4096;  // u's coordinates staged when n fits

struct PrimCand {
  double key;
  long long idx;
  long long par;
  long long pad;
};

__device__ __forceinline__ void prim_min(double& k, long long& i, long long& p, double ok,
                                         long long oi, long long op) {
  if (ok < k || (ok == k && oi < i)) {
    k = ok;
    i = oi;
    p = op;
  }
}

__global__ void __launch_bounds__(PRIM_GRID_THREADS)
    prim_grid_kernel(const double* __restrict__ P, int64_t N, int64_t n, int64_t chunk,
                     double* __restrict__ best, int* __restrict__ parent,
                     unsigned char* __restrict__ in_tree, PrimCand* cand /*2 x gridDim.x*/,
                     int* ea, int* eb, double* ew, int stage_own) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // min(n, PRIM_GRID_SMEM_COORDS) coordinates of u, then (stage_own) this
  // CTA's own points, coordinate-major with stride chunk
  extern __shared__ double s_uc[];
  __shared__ double rk[PRIM_GRID_THREADS / 32];
  __shared__ long long ri[PRIM_GRID_THREADS / 32], rp[PRIM_GRID_THREADS / 32];
  __shared__ double s_key;
  __shared__ long long s_u, s_par;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const double kInf = __longlong_as_double(0x7FF0000000000000LL);
  const long long kNone = 0x7FFFFFFFFFFFFFFFLL;
  const int64_t v0 = blockIdx.x * chunk;
  const int64_t v1 = v0 + chunk < N ? v0 + chunk : N;
  const int64_t nst = n < PRIM_GRID_SMEM_COORDS ? n : PRIM_GRID_SMEM_COORDS;
  double* const s_own = s_uc + nst;
  for (int64_t v = v0 + tid; v < v1; v += PRIM_GRID_THREADS) {
    best[v] = kInf;
    parent[v] = -1;
    in_tree[v] = 0;
    if (stage_own)
      for (int64_t k = 0; k < n; ++k) s_own[k * chunk + (v - v0)] = P[k * N + v];
  }
  long long u = 0;
  double key = 0.0;
  long long par = -1;
  for (int64_t added = 0; added < N; ++added) {
    if (blockIdx.x == 0 && tid == 0 && par >= 0) {
      ea[added - 1] = (int)par;
      eb[added - 1] = (int)u;
      ew[added - 1] = sqrt(key);
    }
    if (tid == 0 && u >= v0 && u < v1) in_tree[u] = 1;
    for (int64_t k = tid; k < nst; k += PRIM_GRID_THREADS) s_uc[k] = P[k * N + u];
    __syncthreads();
    double lb = kInf;
    long long li = kNone;
    for (int64_t v = v0 + tid; v < v1; v += PRIM_GRID_THREADS) {
      if (in_tree[v]) continue;
      double d2 = 0.0;
      if (stage_own) {  // nst == n
        const double* pv = s_own + (v - v0);
#pragma unroll 8
        for (int64_t k = 0; k < n; ++k) {
          const double t = __dsub_rn(pv[k * chunk], s_uc[k]);
          d2 = __dadd_rn(d2, __dmul_rn(t, t));
        }
      } else {
        // the L2-latency-bound form: unrolled so the loads run ahead of the
        // (sequential, order-fixed) sum
        const double* pv = P + v;
#pragma unroll 8
        for (int64_t k = 0; k < nst; ++k) {
          const double t = __dsub_rn(__ldg(pv + k * N), s_uc[k]);
          d2 = __dadd_rn(d2, __dmul_rn(t, t));
        }
#pragma unroll 8
        for (int64_t k = nst; k < n; ++k) {
          const double t = __dsub_rn(__ldg(pv + k * N), __ldg(P + k * N + u));
          d2 = __dadd_rn(d2, __dmul_rn(t, t));
        }
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
    // CTA argmin, ties -> smallest index; the winner's parent is this CTA's
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xFFFFFFFFu, lb, o);
      const long long oi = __shfl_xor_sync(0xFFFFFFFFu, li, o);
      if (ok < lb || (ok == lb && oi < li)) {
        lb = ok;
        li = oi;
      }
    }
    if (lane == 0) {
      rk[warp] = lb;
      ri[warp] = li;
    }
    __syncthreads();
    PrimCand* const buf = cand + ((added + 1) & 1) * G;
    if (tid == 0) {
      double k = rk[0];
      long long i = ri[0], p = 0;
      for (int w = 1; w < PRIM_GRID_THREADS / 32; ++w) prim_min(k, i, p, rk[w], ri[w], 0);
      p = i == kNone ? -1 : parent[i];
      buf[blockIdx.x] = PrimCand{k, i, p, 0};
    }
    grid.sync();
    // every CTA reduces the G candidates (L2 reads: the buffer alternates)
    double ck = kInf;
    long long cidx = kNone, cpar = -1;
    for (int g = tid; g < G; g += PRIM_GRID_THREADS) {
      const double ok = __ldcg(&buf[g].key);
      const long long oi = __ldcg(&buf[g].idx);
      const long long op = __ldcg(&buf[g].par);
      prim_min(ck, cidx, cpar, ok, oi, op);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xFFFFFFFFu, ck, o);
      const long long oi = __shfl_xor_sync(0xFFFFFFFFu, cidx, o);
      const long long op = __shfl_xor_sync(0xFFFFFFFFu, cpar, o);
      prim_min(ck, cidx, cpar, ok, oi, op);
    }
    if (lane == 0) {
      rk[warp] = ck;
      ri[warp] = cidx;
      rp[warp] = cpar;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < PRIM_GRID_THREADS / 32; ++w) prim_min(ck, cidx, cpar, rk[w], ri[w], rp[w]);
      s_key = ck;
      s_u = cidx;
      s_par = cpar;
    }
    __syncthreads();
    u = s_u;
    key = s_key;
    par = s_par;
    if (u == kNone) break;  // all vertices in the tree
  }
}

}  // namespace mhar_dev
