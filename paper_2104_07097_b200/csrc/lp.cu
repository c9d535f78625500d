// lp.cu -- start point without a warm start: the
// Chebyshev centre of {A_I x <= b_I, A_E x = b_E} (the reference's
// chebyshev_center, /root/reference/proj/src/chebyshev.cpp:9-66: maximise r
// subject to a_i x + |a_i| r <= b_i, A_E x = b_E, r >= 0) at scale.
//
// The reference solves that LP with a dense tableau over ALL rows
// (src/lp.cpp:120-297), which cannot exceed ~1e4 rows.  Here the LP is solved
// by constraint generation: a two-phase primal simplex (Dantzig pricing,
// Bland's rule after a degenerate stall) on a working set of rows, with the
// tableau resident on the GPU and every pivot one rank-1 update kernel; after
// each solve one GEMV over all m_I rows finds the violated constraints, the
// most violated are added, and the loop stops when none is violated.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "lp.h"

namespace mhar_lp {
namespace {

constexpr double kPivotTol = 1e-10;
constexpr double kDriveOutTol = 1e-7;
constexpr double kDegenerateStep = 1e-12;
constexpr double kReducedCostTol = 1e-9;
constexpr double kFeasTol = 1e-8;
constexpr int kThreads = 1024;
constexpr int kRegRows = 8;  // ratio-test rows per thread kept in registers

// ---------------------------------------------------------------- kernels --
// Tableau T: rows x cols row-major; b: rows; cost: cols.

// Single CTA: entering column (Dantzig: largest reduced cost > tol; Bland:
// first such column), then the leaving row by the minimum-ratio test with
// ties (within 1e-15) broken by the smallest basic column.
// Pivot-loop control, resident on the device so a phase runs without host
// round trips: the host enqueues batches of select+pivot launches and reads
// `done` once per batch.
struct Ctl {
  int done;          // 1: the phase has ended; every queued launch returns at once
  int status;        // 0 optimal, 7 unbounded ray, 10 pivot budget
  int stall;         // consecutive degenerate pivots
  int bland;         // Bland's rule after a degenerate stall (lp.cpp:47-98)
  long long npiv;    // pivots of this solve
  long long budget;  // 10^4 + 200 (rows + cols)
  int stall_limit;   // rows + priced columns
  int pad;
};

// Free columns (colfree[j] != 0, native free variables): priced by |d_j| and
// entered in the direction of sign(d_j); once basic they never leave (their
// rows are skipped by the ratio test).
__global__ void __launch_bounds__(kThreads) select_kernel(const double* __restrict__ T,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ cost,
                                                          const int* __restrict__ basis, int rows,
                                                          int cols, int limit_col, Ctl* ctl,
                                                          int* out /* entering, leaving */,
                                                          double* prow, double* fcol,
                                                          double* pb /* [b_row/piv, cost_col,
                                                                        leaving col, piv] */,
                                                          const int* __restrict__ colfree,
                                                          double* wbase, int wmode) {
  static_assert(kThreads == 1024, "one reduction partial per lane of warp 0");
  __shared__ double sv[kThreads / 32];
  __shared__ int si[kThreads / 32], sb[kThreads / 32];
  __shared__ int s_enter, s_row;
  __shared__ double s_min;
  __shared__ int s_go;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_go = !ctl->done && ctl->npiv < ctl->budget;
  __syncthreads();
  if (!s_go) {
    if (tid == 0 && !ctl->done) {  // pivot budget exhausted
      ctl->done = 1;
      ctl->status = 10;
    }
    return;
  }
  const int bland = ctl->bland;
  // wmode 1: Devex reference weights in wbase; 2: exact steepest edge, the
  // squared tableau column norms accumulated by the previous pivot's update
  // in wbase[(npiv & 1) * cols]; the other half is cleared for this pivot's
  const double* dvx = nullptr;
  double wadd = 0.0;
  if (wmode == 1) dvx = wbase;
  if (wmode == 2) {
    const long long k = ctl->npiv;
    dvx = wbase + (size_t)(k & 1) * cols;
    double* nxt = wbase + (size_t)((k + 1) & 1) * cols;
    for (int j = tid; j < cols; j += kThreads) nxt[j] = 0.0;
    wadd = 1.0;  // gamma_j = 1 + |B^-1 a_j|^2
  }
  // pricing: Dantzig (largest reduced cost) or, with reference weights dvx,
  // Devex (largest d_j^2 / w_j: an approximate steepest edge, far fewer
  // pivots on the degenerate centring LP); Bland after a stall
  double bv = -1.0;
  int bi = 0x7FFFFFFF;
  // (loops unrolled so each thread has its loads in flight together: this
  // single-CTA kernel is latency-bound)
#pragma unroll 8
  for (int j = tid; j < limit_col; j += kThreads) {
    double c = cost[j];
    if (colfree && colfree[j]) c = fabs(c);
    if (!(c > kReducedCostTol)) continue;
    if (bland) {
      if (j < bi) bi = j;
      continue;
    }
    const double sc = dvx ? c * c / (wadd + dvx[j]) : c;
    if (sc > bv || (sc == bv && j < bi)) {
      bv = sc;
      bi = j;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
    const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
    if (bland ? (oi < bi) : (ov > bv || (ov == bv && oi < bi))) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {  // kThreads / 32 == 32 partials: one per lane
    bv = sv[lane];
    bi = si[lane];
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
      const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
      if (bland ? (oi < bi) : (ov > bv || (ov == bv && oi < bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_enter = (bi == 0x7FFFFFFF) ? -1 : bi;
      out[0] = s_enter;
      if (s_enter < 0) {  // optimal
        ctl->done = 1;
        ctl->status = 0;
      }
    }
  }
  __syncthreads();
  const int e = s_enter;
  if (e < 0) return;
  // a free column with a negative reduced cost enters decreasing
  const double dir = (colfree && colfree[e] && cost[e] < 0.0) ? -1.0 : 1.0;
  // ratio test, pass 1: minimum ratio; the entering column (one strided
  // sector per row) is cached in fcol for the rank-1 update, and the first
  // kRegRows rows per thread keep their ratios in registers for pass 2
  const double kInf = __longlong_as_double(0x7FF0000000000000LL);
  double ra[kRegRows];
  double mr = kInf;
#pragma unroll
  for (int q = 0; q < kRegRows; ++q) {
    const int i = tid + q * kThreads;
    ra[q] = kInf;
    if (i < rows) {
      const double t = T[(size_t)i * cols + e];
      fcol[i] = t;
      const double a = dir * t;
      if (a > kPivotTol && !(colfree && colfree[basis[i]])) {
        ra[q] = b[i] / a;
        mr = fmin(mr, ra[q]);
      }
    }
  }
  for (int i = tid + kRegRows * kThreads; i < rows; i += kThreads) {
    const double t = T[(size_t)i * cols + e];
    fcol[i] = t;
    const double a = dir * t;
    if (a > kPivotTol && !(colfree && colfree[basis[i]])) mr = fmin(mr, b[i] / a);
  }
  for (int o = 16; o > 0; o >>= 1) mr = fmin(mr, __shfl_xor_sync(0xFFFFFFFFu, mr, o));
  if (lane == 0) sv[warp] = mr;
  __syncthreads();
  if (warp == 0) {
    mr = sv[lane];
    for (int o = 16; o > 0; o >>= 1) mr = fmin(mr, __shfl_xor_sync(0xFFFFFFFFu, mr, o));
    if (lane == 0) s_min = mr;
  }
  __syncthreads();
  // pass 2: among ratios within 1e-15 of the minimum, the smallest basic column
  const double lim = s_min + 1e-15;
  int best_basic = 0x7FFFFFFF, best_row = -1;
  if (s_min < kInf) {
#pragma unroll
    for (int q = 0; q < kRegRows; ++q) {
      const int i = tid + q * kThreads;
      if (ra[q] <= lim) {
        const int bs = basis[i];
        if (bs < best_basic) {
          best_basic = bs;
          best_row = i;
        }
      }
    }
    for (int i = tid + kRegRows * kThreads; i < rows; i += kThreads) {
      const double a = dir * fcol[i];
      if (a > kPivotTol && !(colfree && colfree[basis[i]]) && b[i] / a <= lim &&
          basis[i] < best_basic) {
        best_basic = basis[i];
        best_row = i;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int ob = __shfl_xor_sync(0xFFFFFFFFu, best_basic, o);
    const int orow = __shfl_xor_sync(0xFFFFFFFFu, best_row, o);
    if (ob < best_basic) {
      best_basic = ob;
      best_row = orow;
    }
  }
  if (lane == 0) {
    si[warp] = best_row;
    sb[warp] = best_basic;
  }
  __syncthreads();
  if (warp == 0) {
    best_row = si[lane];
    best_basic = sb[lane];
    for (int o = 16; o > 0; o >>= 1) {
      const int ob = __shfl_xor_sync(0xFFFFFFFFu, best_basic, o);
      const int orow = __shfl_xor_sync(0xFFFFFFFFu, best_row, o);
      if (ob < best_basic) {
        best_basic = ob;
        best_row = orow;
      }
    }
    if (lane == 0) {
      out[1] = best_row;
      if (best_row < 0) {  // unbounded ray
        ctl->done = 1;
        ctl->status = 7;
      } else {
        if (s_min < kDegenerateStep) {
          if (++ctl->stall > ctl->stall_limit) ctl->bland = 1;
        } else {
          ctl->stall = 0;
        }
        ++ctl->npiv;
      }
      s_row = best_row;
    }
  }
  __syncthreads();
  const int row = s_row;
  if (row < 0) return;
  // capture for the rank-1 update (fcol = T[:,e] is cached above) and the
  // pivot row divided out (one coalesced sweep; a separate grid-wide launch
  // cost more in launch gap than it saved)
  const double piv = fcol[row];
  const double* __restrict__ Tr = T + (size_t)row * cols;
#pragma unroll 8
  for (int j = tid; j < cols; j += kThreads) prow[j] = Tr[j] / piv;
  if (tid == 0) {
    pb[0] = b[row] / piv;
    pb[1] = cost[e];
    pb[2] = (double)basis[row];  // the leaving variable
    pb[3] = piv;
  }
}

// pivot on (row, col): prow = T[row,:]/piv, fcol = T[:,col] captured first
__global__ void capture_kernel(const double* __restrict__ T, const double* __restrict__ b,
                               int rows, int cols, int row, int col, double* prow, double* fcol,
                               double* pb) {
  const double piv = T[(size_t)row * cols + col];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x)
    prow[j] = T[(size_t)row * cols + j] / piv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
    fcol[i] = T[(size_t)i * cols + col];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    pb[0] = b[row] / piv;
    pb[1] = 0.0;  // drive-out pivots run without a cost row
    pb[2] = -1.0;
    pb[3] = piv;
  }
}

// sel <- (col, row) for a host-chosen pivot
__global__ void set_sel_kernel(int* sel, int row, int col) {
  sel[0] = col;
  sel[1] = row;
}

__global__ void __launch_bounds__(256) pivot_kernel(double* __restrict__ T, double* __restrict__ b,
                                                    double* __restrict__ cost, int* basis, int rows,
                                                    int cols, const int* __restrict__ sel,
                                                    const int* __restrict__ done,
                                                    const double* __restrict__ prow,
                                                    const double* __restrict__ fcol,
                                                    const double* pb) {
  // one block per tableau row (blockIdx.x == rows: the cost row); rows are
  // 16-byte aligned (even column stride), updated as double2
  if (*done) return;
  const int col = sel[0], row = sel[1];
  const double brow = pb[0];
  const double cf = pb[1];  // cost[col] before this pivot (captured)
  const int i = blockIdx.x;
  const int c2 = cols >> 1;
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(prow);
  if (i == rows) {
    if (cf != 0.0)
      for (int j = threadIdx.x; j < cols; j += blockDim.x)
        cost[j] = (j == col) ? 0.0 : cost[j] - cf * prow[j];
    return;
  }
  double2* __restrict__ Ti = reinterpret_cast<double2*>(T + (size_t)i * cols);
  if (i == row) {
    for (int j = threadIdx.x; j < c2; j += blockDim.x) Ti[j] = __ldg(p2 + j);
    if (threadIdx.x == 0) {
      b[i] = brow;
      basis[i] = col;
    }
    return;
  }
  const double f = fcol[i];
  if (f == 0.0) return;
#pragma unroll 4
  for (int j = threadIdx.x; j < c2; j += blockDim.x) {
    double2 t = Ti[j];
    const double2 q = __ldg(p2 + j);
    t.x = fma(-f, q.x, t.x);
    t.y = fma(-f, q.y, t.y);
    Ti[j] = t;
  }
  if (threadIdx.x == 0) b[i] -= f * brow;
}

// The same rank-1 update tiled: a block owns kPivRows rows x one column
// chunk of 256 x kPivVec double2, each thread keeps its pivot-row segment in
// registers across the rows (the pivot row is read once per row group, not
// once per row) and the rows' loads are issued back to back.
#ifndef MHAR_LP_PIV_ROWS
#define MHAR_LP_PIV_ROWS 8
#endif
#ifndef MHAR_LP_PIV_VEC
#define MHAR_LP_PIV_VEC 2
#endif
constexpr int kPivRows = MHAR_LP_PIV_ROWS, kPivVec = MHAR_LP_PIV_VEC;
__global__ void __launch_bounds__(256) pivot_tile_kernel(double* __restrict__ T,
                                                         double* __restrict__ b,
                                                         double* __restrict__ cost, int* basis,
                                                         int rows, int cols,
                                                         const int* __restrict__ sel,
                                                         const int* __restrict__ done,
                                                         const double* __restrict__ prow,
                                                         const double* __restrict__ fcol,
                                                         const double* pb, double* wbase,
                                                         int wmode,
                                                         const long long* __restrict__ npiv) {
  if (*done) return;
  double* dvx = wmode == 1 ? wbase : nullptr;
  const int col = sel[0], row = sel[1];
  const double brow = pb[0];
  const double cf = pb[1];
  const int c2 = cols >> 1;
  const int j0 = blockIdx.x * (256 * kPivVec) + threadIdx.x;
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(prow);
  double2 q[kPivVec];
#pragma unroll
  for (int v = 0; v < kPivVec; ++v) {
    const int j = j0 + 256 * v;
    q[v] = j < c2 ? __ldg(p2 + j) : make_double2(0.0, 0.0);
  }
  const int i0 = blockIdx.y * kPivRows;
  const bool gam = wmode == 2;  // accumulate the updated columns' squared norms
  double2 acc[kPivVec];
#pragma unroll
  for (int v = 0; v < kPivVec; ++v) acc[v] = make_double2(0.0, 0.0);
#pragma unroll 2
  for (int r = 0; r < kPivRows; ++r) {
    const int i = i0 + r;
    if (i > rows) break;
    if (i == rows) {  // the cost row (captured cost[col] in pb[1])
      if (cf != 0.0)
#pragma unroll
        for (int v = 0; v < kPivVec; ++v) {
          const int j = j0 + 256 * v;
          if (j < c2) {
            const double c0 = 2 * j == col ? 0.0 : cost[2 * j] - cf * q[v].x;
            const double c1 = 2 * j + 1 == col ? 0.0 : cost[2 * j + 1] - cf * q[v].y;
            cost[2 * j] = c0;
            cost[2 * j + 1] = c1;
          }
        }
      if (dvx && pb[2] >= 0.0) {
        // Devex reference weights (Forrest & Goldfarb): w_j = max(w_j,
        // (a_rj / a_rq)^2 w_q) for the nonbasic columns, the leaving column
        // max(w_q / a_rq^2, 1); prow holds a_rj / a_rq (0 on basic columns)
        const double wq = dvx[col];
        const int leave = (int)pb[2];
        const double piv = pb[3];
#pragma unroll
        for (int v = 0; v < kPivVec; ++v) {
          const int j = j0 + 256 * v;
          if (j >= c2) continue;
          for (int h = 0; h < 2; ++h) {
            const int jj = 2 * j + h;
            if (jj == col) continue;
            const double a = h ? q[v].y : q[v].x;
            dvx[jj] = jj == leave ? fmax(wq / (piv * piv), 1.0) : fmax(dvx[jj], a * a * wq);
          }
        }
      }
      break;
    }
    double2* __restrict__ Ti = reinterpret_cast<double2*>(T + (size_t)i * cols);
    if (i == row) {
#pragma unroll
      for (int v = 0; v < kPivVec; ++v) {
        const int j = j0 + 256 * v;
        if (j < c2) {
          Ti[j] = q[v];
          acc[v].x = fma(q[v].x, q[v].x, acc[v].x);
          acc[v].y = fma(q[v].y, q[v].y, acc[v].y);
        }
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        b[i] = brow;
        basis[i] = col;
      }
      continue;
    }
    const double f = fcol[i];
    if (f == 0.0 && !gam) continue;
    double2 t[kPivVec];
#pragma unroll
    for (int v = 0; v < kPivVec; ++v) {
      const int j = j0 + 256 * v;
      if (j < c2) t[v] = Ti[j];
    }
#pragma unroll
    for (int v = 0; v < kPivVec; ++v) {
      const int j = j0 + 256 * v;
      if (j < c2) {
        if (f != 0.0) {
          t[v].x = fma(-f, q[v].x, t[v].x);
          t[v].y = fma(-f, q[v].y, t[v].y);
          Ti[j] = t[v];
        }
        acc[v].x = fma(t[v].x, t[v].x, acc[v].x);
        acc[v].y = fma(t[v].y, t[v].y, acc[v].y);
      }
    }
    if (f != 0.0 && blockIdx.x == 0 && threadIdx.x == 0) b[i] -= f * brow;
  }
  if (gam) {
    double* g = wbase + (size_t)((*npiv) & 1) * cols;
#pragma unroll
    for (int v = 0; v < kPivVec; ++v) {
      const int j = j0 + 256 * v;
      if (j < c2) {
        atomicAdd(g + 2 * j, acc[v].x);
        atomicAdd(g + 2 * j + 1, acc[v].y);
      }
    }
  }
}

// squared column norms of the tableau (the steepest-edge weights of a phase's
// first pivot) into g[0..cols)
__global__ void colnorm_kernel(const double* __restrict__ T, int rows, int cols, double* g) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double s = 0.0;
  for (int i = 0; i < rows; ++i) {
    const double t = T[(size_t)i * cols + j];
    s = fma(t, t, s);
  }
  g[j] = s;
}

// v_i = a_i x + |a_i| r - b_i over all rows (A column-major m x n)
__global__ void violation_kernel(const double* __restrict__ A, const double* __restrict__ norms,
                                 const double* __restrict__ bvec, const double* __restrict__ x,
                                 double r, int64_t m, int64_t n, double* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s = fma(A[i + k * m], x[k], s);
    v[i] = s + norms[i] * r - bvec[i];
  }
}

// |a_i| accumulated in ascending k without contraction (the host loop's
// order, so the LP sees the same norms)
__global__ void row_norms_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                 double* __restrict__ norms) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = A[i + k * m];
      s = __dadd_rn(s, __dmul_rn(a, a));
    }
    norms[i] = sqrt(s);
  }
}

// initial working set: block (k, sign) finds the first row maximising
// sign * a_ik / |a_i| among the positive values (-1 if none)
__global__ void __launch_bounds__(256) ws_argmax_kernel(const double* __restrict__ A,
                                                        const double* __restrict__ norms,
                                                        int64_t m, int64_t* __restrict__ out) {
  __shared__ double sv[8];
  __shared__ long long si[8];
  const int64_t k = blockIdx.x;
  const double sgn = blockIdx.y ? 1.0 : -1.0;
  const double* __restrict__ col = A + k * m;
  double bv = 0.0;
  long long bi = -1;
  for (int64_t i = threadIdx.x; i < m; i += 256) {
    const double v = sgn * col[i] / fmax(norms[i], 1e-300);
    if (v > bv) {  // ascending i per thread: strict > keeps the first
      bv = v;
      bi = i;
    }
  }
  auto better = [](double v, long long i, double bv, long long bi) {
    return i >= 0 && (bi < 0 || v > bv || (v == bv && i < bi));
  };
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
    const long long oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
    out[2 * k + blockIdx.y] = bi;
  }
}

// ------------------------------------------------------------ the solver --

struct Dev {
  double *T = nullptr, *b = nullptr, *cost = nullptr, *prow = nullptr, *fcol = nullptr;
  double *pb = nullptr, *ratio = nullptr, *dvx = nullptr;
  int *basis = nullptr, *sel = nullptr, *zero = nullptr, *colfree = nullptr;
  Ctl* ctl = nullptr;
  cudaStream_t s = nullptr;
  ~Dev() {
    cudaFree(T);
    cudaFree(b);
    cudaFree(cost);
    cudaFree(prow);
    cudaFree(fcol);
    cudaFree(pb);
    cudaFree(ratio);
    cudaFree(dvx);
    cudaFree(basis);
    cudaFree(sel);
    cudaFree(zero);
    cudaFree(colfree);
    cudaFree(ctl);
    if (s) cudaStreamDestroy(s);
  }
};

// MHAR_LP_PROFILE=1: wall time of the centring stages on stderr
struct LpClock {
  bool on = std::getenv("MHAR_LP_PROFILE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lp profile] %-28s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

int err(std::string* msg, int code, const std::string& text) {
  *msg = text;
  return code;
}

// Dense two-phase simplex: maximise c.x, rows kind (<= or =), x_j >= 0 or free.
// The rows' right-hand sides are perturbed by up to `perturb` (deterministic
// per row) so the highly degenerate vertices of the centring LP do not stall
// the pivoting; the unperturbed rhs rides along as one extra tableau column,
// so the final basis is evaluated on the original problem.  Returns 0 /
// EMPTY(5) / UNBOUNDED(7) / CYCLE(10) / CUDA(100), or kPerturbedOnly when the
// final basis is infeasible for the unperturbed rhs (retry with less).
constexpr int kPerturbedOnly = 1000;

// native_free: each free variable is ONE column that may enter in either
// direction and never leaves once basic (no x+ / x- split, no l1 row; the
// restricted LP may then report an unbounded ray, and the caller re-solves
// with the split form, whose l1 row bounds it).
int simplex(const std::vector<double>& Arow /* m x nv row-major */, const std::vector<double>& rhs,
            const std::vector<int>& is_eq, const std::vector<int>& is_free,
            const std::vector<double>& obj, int m, int nv, double perturb, double scale,
            int l1_row, bool native_free, std::vector<double>* x, long* pivots,
            std::string* msg) {
  LpClock sclk;
  std::vector<int> var_col(nv);
  int ncols = 0;
  for (int v = 0; v < nv; ++v) {
    var_col[v] = ncols;
    ncols += (is_free[v] && !native_free) ? 2 : 1;
  }
  int nslack = 0;
  for (int i = 0; i < m; ++i) nslack += is_eq[i] ? 0 : 1;
  const int structural = ncols + nslack;
  // artificials for rows whose slack cannot start basic
  std::vector<double> sgn(m);
  int nart = 0;
  for (int i = 0; i < m; ++i) {
    sgn[i] = rhs[i] < 0 ? -1.0 : 1.0;
    if (is_eq[i] || sgn[i] < 0) ++nart;
  }
  const int total = structural + nart;  // priced columns
  const int W = (total + 2) & ~1;       // + the unperturbed rhs column, even (16-byte rows)
  std::vector<double> T((size_t)m * W, 0.0), b(m);
  std::vector<int> basis(m, -1);
  int slack = ncols, art = structural;
  std::vector<char> has_art(m, 0);
  for (int i = 0; i < m; ++i) {
    double* row = &T[(size_t)i * W];
    for (int v = 0; v < nv; ++v) {
      const double a = sgn[i] * Arow[(size_t)i * nv + v];
      row[var_col[v]] = a;
      if (is_free[v] && !native_free)
        row[var_col[v] + 1] = i == l1_row ? a : -a;  // l1: x+ + x- <= B
    }
    row[total] = sgn[i] * rhs[i];
    // golden-ratio sequence in [0.5, 1.5): distinct, deterministic per row
    const double u = 0.5 + std::fmod(0.6180339887498949 * (i + 1), 1.0);
    b[i] = row[total] + (is_eq[i] ? 0.0 : perturb * u);
    if (!is_eq[i]) {
      row[slack] = sgn[i];
      if (sgn[i] > 0) basis[i] = slack;
      ++slack;
    }
    if (basis[i] < 0) {
      row[art] = 1.0;
      basis[i] = art;
      has_art[i] = 1;
      ++art;
    }
  }
  std::vector<int> colfree(W, 0);
  if (native_free)
    for (int v = 0; v < nv; ++v)
      if (is_free[v]) colfree[var_col[v]] = 1;
  Dev d;
  auto ok = [](cudaError_t e) { return e == cudaSuccess; };
  if (!ok(cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking)) ||
      !ok(cudaMalloc(&d.T, sizeof(double) * T.size())) ||
      !ok(cudaMalloc(&d.b, sizeof(double) * m)) || !ok(cudaMalloc(&d.cost, sizeof(double) * W)) ||
      !ok(cudaMalloc(&d.prow, sizeof(double) * W)) ||
      !ok(cudaMalloc(&d.fcol, sizeof(double) * m)) || !ok(cudaMalloc(&d.pb, 4 * sizeof(double))) ||
      !ok(cudaMalloc(&d.dvx, 2 * sizeof(double) * W)) ||
      !ok(cudaMalloc(&d.zero, sizeof(int))) || !ok(cudaMalloc(&d.ctl, sizeof(Ctl))) ||
      !ok(cudaMalloc(&d.ratio, sizeof(double))) || !ok(cudaMalloc(&d.basis, sizeof(int) * m)) ||
      !ok(cudaMalloc(&d.sel, sizeof(int) * 2)) ||
      (native_free && !ok(cudaMalloc(&d.colfree, sizeof(int) * W))))
    return err(msg, 100, "simplex: device allocation failed");
  if (native_free)
    cudaMemcpyAsync(d.colfree, colfree.data(), sizeof(int) * W, cudaMemcpyHostToDevice, d.s);
  cudaMemcpyAsync(d.T, T.data(), sizeof(double) * T.size(), cudaMemcpyHostToDevice, d.s);
  cudaMemcpyAsync(d.b, b.data(), sizeof(double) * m, cudaMemcpyHostToDevice, d.s);
  cudaMemcpyAsync(d.basis, basis.data(), sizeof(int) * m, cudaMemcpyHostToDevice, d.s);
  cudaMemsetAsync(d.zero, 0, sizeof(int), d.s);

  const long budget = 10000 + 200L * (m + total);
  long npiv = 0;
  int rows = m;
  // MHAR_LP_PIVOT=row: one block per tableau row (the first form)
  const char* piv_env = std::getenv("MHAR_LP_PIVOT");
  const bool row_form = piv_env && !std::strcmp(piv_env, "row");
  const dim3 tile_grid((unsigned)((W / 2 + 256 * kPivVec - 1) / (256 * kPivVec)),
                       (unsigned)((rows + 1 + kPivRows - 1) / kPivRows));
  // Devex pricing with the tile update (MHAR_LP_PRICING=dantzig: the
  // reference's rule throughout)
  const char* pr_env = std::getenv("MHAR_LP_PRICING");
  // exact steepest edge by default: the tile update accumulates the squared
  // norms of the columns it rewrites, so the weights cost no extra pass; on
  // the degenerate centring LP it needs 6x fewer pivots than Dantzig
  // (config 5: 7.7K vs 47.9K).  MHAR_LP_PRICING=dantzig | devex | steepest
  int wmode = row_form ? 0 : 2;
  if (pr_env && !std::strcmp(pr_env, "dantzig")) wmode = 0;
  if (!row_form && pr_env && !std::strcmp(pr_env, "devex")) wmode = 1;
  auto pivot_launch = [&](const int* done, int wm) {
    if (row_form)
      pivot_kernel<<<rows + 1, 256, 0, d.s>>>(d.T, d.b, d.cost, d.basis, rows, W, d.sel, done,
                                               d.prow, d.fcol, d.pb);
    else
      pivot_tile_kernel<<<tile_grid, 256, 0, d.s>>>(d.T, d.b, d.cost, d.basis, rows, W, d.sel,
                                                    done, d.prow, d.fcol, d.pb, d.dvx, wm,
                                                    &d.ctl->npiv);
  };
  // a host-chosen pivot (artificials driven out after phase one)
  auto pivot = [&](int row, int col) {
    set_sel_kernel<<<1, 1, 0, d.s>>>(d.sel, row, col);
    capture_kernel<<<std::max(1, std::min(1024, (std::max(rows, W) + 255) / 256)), 256, 0, d.s>>>(
        d.T, d.b, rows, W, row, col, d.prow, d.fcol, d.pb);
    pivot_launch(d.zero, 0);
    ++npiv;
  };
  const bool lp_trace = std::getenv("MHAR_LP_TRACE") != nullptr;  // one pivot per batch, logged
  // one phase, driven on the device: 0 optimal, 7 unbounded ray, 10 budget, 100 CUDA
  auto run_phase = [&](int limit_col) -> int {
    Ctl h{};
    h.budget = budget - npiv;
    h.stall_limit = rows + total;
    if (const char* sl = std::getenv("MHAR_LP_STALL")) h.stall_limit = (int)(h.stall_limit * std::atof(sl));
    cudaMemcpyAsync(d.ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, d.s);
    if (wmode == 1) {  // fresh reference framework: every weight 1
      const std::vector<double> ones(W, 1.0);
      cudaMemcpyAsync(d.dvx, ones.data(), sizeof(double) * W, cudaMemcpyHostToDevice, d.s);
      cudaStreamSynchronize(d.s);  // `ones` is a local
    } else if (wmode == 2) {  // exact weights of the phase's starting basis
      colnorm_kernel<<<(W + 255) / 256, 256, 0, d.s>>>(d.T, rows, W, d.dvx);
    }
    const char* bat_env = std::getenv("MHAR_LP_BATCH");
    int batch = bat_env ? std::max(1, std::atoi(bat_env)) : lp_trace ? 1 : 8;
    for (;;) {
      for (int k = 0; k < batch; ++k) {
        select_kernel<<<1, kThreads, 0, d.s>>>(d.T, d.b, d.cost, d.basis, rows, W, limit_col,
                                               d.ctl, d.sel, d.prow, d.fcol, d.pb, d.colfree,
                                               d.dvx, wmode);
        pivot_launch(&d.ctl->done, wmode);
      }
      cudaMemcpyAsync(&h, d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, d.s);
      if (cudaStreamSynchronize(d.s) != cudaSuccess) return 100;
      if (lp_trace) {
        int hs[2];
        cudaMemcpy(hs, d.sel, sizeof(hs), cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "[lp trace] limit %d npiv %lld sel %d %d done %d st %d bland %d\n",
                     limit_col, h.npiv, hs[0], hs[1], h.done, h.status, h.bland);
      }
      if (h.done) {
        npiv += h.npiv;
        if (sclk.on)
          std::fprintf(stderr, "[lp profile]   phase: %lld pivots, bland %d, stall %d, status %d\n",
                       h.npiv, h.bland, h.stall, h.status);
        return h.status;
      }
      if (!lp_trace && !bat_env) batch = std::min(batch * 2, 256);
    }
  };
  auto fetch_row = [&](int i, double* dst) {
    cudaMemcpyAsync(dst, d.T + (size_t)i * W, sizeof(double) * W, cudaMemcpyDeviceToHost, d.s);
    cudaStreamSynchronize(d.s);
  };

  if (nart > 0) {
    // phase one: maximise -sum(artificials)
    std::vector<double> c1(W, 0.0);
    for (int i = 0; i < m; ++i)
      if (has_art[i])
        for (int j = 0; j < structural; ++j) c1[j] += T[(size_t)i * W + j];
    cudaMemcpyAsync(d.cost, c1.data(), sizeof(double) * W, cudaMemcpyHostToDevice, d.s);
    sclk.mark("  tableau build + upload");
    const int st = run_phase(total);
    sclk.mark("  phase one");
    if (st == 100) return err(msg, 100, "simplex: CUDA failure");
    if (st == 10) return err(msg, 10, "CYCLE_SUSPECTED: solve_lp: pivot budget exhausted");
    if (st == 7) return err(msg, 12, "NUMERICAL_FAILURE: phase one reported an unbounded ray");
    cudaMemcpyAsync(b.data(), d.b, sizeof(double) * m, cudaMemcpyDeviceToHost, d.s);
    cudaMemcpyAsync(basis.data(), d.basis, sizeof(int) * m, cudaMemcpyDeviceToHost, d.s);
    cudaStreamSynchronize(d.s);
    double mass = 0.0;
    for (int i = 0; i < rows; ++i)
      if (basis[i] >= structural) mass += b[i];
    if (mass > kFeasTol * scale + 2.0 * m * perturb)
      return err(msg, 5, "EMPTY_POLYTOPE: chebyshev_center: constraint system is infeasible");
    // drive basic artificials out, or drop their rows as redundant
    std::vector<char> drop(rows, 0);
    int ndrop = 0;
    for (int i = 0; i < rows; ++i) {
      if (basis[i] < structural) continue;
      double* Ti = &T[(size_t)i * W];
      fetch_row(i, Ti);
      int col = -1;
      for (int j = 0; j < structural && col < 0; ++j)
        if (std::fabs(Ti[j]) > kDriveOutTol) col = j;
      if (col >= 0) {
        pivot(i, col);
      } else {
        drop[i] = 1;
        ++ndrop;
      }
    }
    if (ndrop > 0) {
      std::vector<int> dbasis(rows);
      cudaMemcpyAsync(T.data(), d.T, sizeof(double) * (size_t)rows * W, cudaMemcpyDeviceToHost,
                      d.s);
      cudaMemcpyAsync(b.data(), d.b, sizeof(double) * rows, cudaMemcpyDeviceToHost, d.s);
      cudaMemcpyAsync(dbasis.data(), d.basis, sizeof(int) * rows, cudaMemcpyDeviceToHost, d.s);
      cudaStreamSynchronize(d.s);
      int k = 0;
      for (int i = 0; i < rows; ++i) {
        if (drop[i]) continue;
        if (k != i) std::memmove(&T[(size_t)k * W], &T[(size_t)i * W], sizeof(double) * W);
        b[k] = b[i];
        basis[k] = dbasis[i];
        ++k;
      }
      rows = k;
      cudaMemcpyAsync(d.T, T.data(), sizeof(double) * (size_t)rows * W, cudaMemcpyHostToDevice,
                      d.s);
      cudaMemcpyAsync(d.b, b.data(), sizeof(double) * rows, cudaMemcpyHostToDevice, d.s);
      cudaMemcpyAsync(d.basis, basis.data(), sizeof(int) * rows, cudaMemcpyHostToDevice, d.s);
    }
  }
  // phase two: reduced costs of the objective against the current basis
  std::vector<double> c2(W, 0.0);
  for (int v = 0; v < nv; ++v) {
    c2[var_col[v]] = obj[v];
    if (is_free[v] && !native_free) c2[var_col[v] + 1] = -obj[v];
  }
  cudaMemcpyAsync(basis.data(), d.basis, sizeof(int) * rows, cudaMemcpyDeviceToHost, d.s);
  cudaStreamSynchronize(d.s);
  std::vector<double> red = c2;
  for (int i = 0; i < rows; ++i) {
    const double cb = c2[basis[i]];
    if (cb == 0.0) continue;
    std::vector<double> Ti(W);
    fetch_row(i, Ti.data());
    for (int j = 0; j < W; ++j) red[j] -= cb * Ti[j];
  }
  cudaMemcpyAsync(d.cost, red.data(), sizeof(double) * W, cudaMemcpyHostToDevice, d.s);
  sclk.mark("  drive-out + phase-two costs");
  const int st = run_phase(structural);
  sclk.mark("  phase two");
  if (st == 100) return err(msg, 100, "simplex: CUDA failure");
  if (st == 10) return err(msg, 10, "CYCLE_SUSPECTED: solve_lp: pivot budget exhausted");
  if (st == 7)
    return err(msg, 7, "UNBOUNDED_POLYTOPE: chebyshev_center: inscribed radius is unbounded");
  *pivots += npiv;
  // the optimal basis applied to the unperturbed rhs
  std::vector<double> orig(rows);
  cudaMemcpy2DAsync(orig.data(), sizeof(double), d.T + total, sizeof(double) * W, sizeof(double),
                    rows, cudaMemcpyDeviceToHost, d.s);
  cudaMemcpyAsync(basis.data(), d.basis, sizeof(int) * rows, cudaMemcpyDeviceToHost, d.s);
  if (cudaStreamSynchronize(d.s) != cudaSuccess) return err(msg, 100, "simplex: CUDA failure");
  std::vector<double> expanded(W, 0.0);
  for (int i = 0; i < rows; ++i) {
    if (colfree[basis[i]]) {  // a basic free variable takes any sign
      expanded[basis[i]] = orig[i];
      continue;
    }
    if (orig[i] < -1e-9 * scale) return kPerturbedOnly;
    expanded[basis[i]] = std::max(orig[i], 0.0);
  }
  x->assign(nv, 0.0);
  for (int v = 0; v < nv; ++v)
    (*x)[v] = (is_free[v] && !native_free) ? expanded[var_col[v]] - expanded[var_col[v] + 1]
                                           : expanded[var_col[v]];
  return 0;
}

}  // namespace

int chebyshev_center(const double* a_in, const double* b_in, int64_t m, const double* a_eq,
                     const double* b_eq, int64_t me, int64_t n, int device, double* x_out,
                     double* radius, LpStats* stats, std::string* msg) {
  if (cudaSetDevice(device) != cudaSuccess) return err(msg, 100, "cudaSetDevice failed");
  LpClock clk;
  double scale = 1.0;
  for (int64_t i = 0; i < m; ++i) scale = std::max(scale, std::fabs(b_in[i]));
  // device copies for the violation scan
  double *dA = nullptr, *dN = nullptr, *dB = nullptr, *dX = nullptr, *dV = nullptr;
  auto free_all = [&]() {
    cudaFree(dA);
    cudaFree(dN);
    cudaFree(dB);
    cudaFree(dX);
    cudaFree(dV);
  };
  if (cudaMalloc(&dA, sizeof(double) * m * n) != cudaSuccess ||
      cudaMalloc(&dN, sizeof(double) * m) != cudaSuccess ||
      cudaMalloc(&dB, sizeof(double) * m) != cudaSuccess ||
      cudaMalloc(&dX, sizeof(double) * n) != cudaSuccess ||
      cudaMalloc(&dV, sizeof(double) * m) != cudaSuccess) {
    free_all();
    return err(msg, 100, "chebyshev_center: device allocation failed");
  }
  cudaMemcpy(dA, a_in, sizeof(double) * m * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b_in, sizeof(double) * m, cudaMemcpyHostToDevice);
  const int64_t gm = std::max<int64_t>(1, std::min<int64_t>(4096, (m + 255) / 256));
  // row norms on the device (the LP's radius coefficients)
  std::vector<double> norms(m);
  row_norms_kernel<<<(unsigned)gm, 256>>>(dA, m, n, dN);
  if (cudaMemcpy(norms.data(), dN, sizeof(double) * m, cudaMemcpyDeviceToHost) != cudaSuccess) {
    free_all();
    return err(msg, 100, "chebyshev_center: row norms failed");
  }
  clk.mark("upload + norms");

  // initial working set: per coordinate and sign the row that bounds it most
  // tightly (largest a_ij / |a_i|), so the restricted LP is usually bounded
  std::vector<char> in_w(m, 0);
  std::vector<int64_t> work;
  {
    int64_t* dbest = nullptr;
    std::vector<int64_t> best(2 * n);
    if (cudaMalloc(&dbest, sizeof(int64_t) * 2 * n) != cudaSuccess) {
      free_all();
      return err(msg, 100, "chebyshev_center: device allocation failed");
    }
    ws_argmax_kernel<<<dim3((unsigned)n, 2), 256>>>(dA, dN, m, dbest);
    const cudaError_t e =
        cudaMemcpy(best.data(), dbest, sizeof(int64_t) * 2 * n, cudaMemcpyDeviceToHost);
    cudaFree(dbest);
    if (e != cudaSuccess) {
      free_all();
      return err(msg, 100, "chebyshev_center: working-set scan failed");
    }
    for (int64_t k = 0; k < n; ++k)
      for (int sg = 0; sg < 2; ++sg) {  // sign -1 first, as the scan order
        const int64_t i = best[2 * k + sg];
        if (i >= 0 && !in_w[i]) {
          in_w[i] = 1;
          work.push_back(i);
        }
      }
  }
  if ((int64_t)work.size() == m) {
    // everything is already in
  }
  clk.mark("initial working set");
  const double box = 1e6 * scale;  // temporary bound; touching it means unbounded
  std::vector<double> xr;
  int rounds = 0;
  long pivots = 0;
  int status = 0;
  for (;;) {
    ++rounds;
    const int nv = (int)n + 1;
    // + one l1 row sum(x+ + x-) <= box keeping the restricted LP bounded
    // (split form only; the native-free form drops it)
    const int mw = (int)me + (int)work.size() + 1;
    std::vector<double> A((size_t)mw * nv, 0.0), rhs(mw);
    std::vector<int> is_eq(mw, 0), is_free(nv, 1);
    is_free[n] = 0;
    int r = 0;
    for (int64_t i = 0; i < me; ++i, ++r) {
      for (int64_t k = 0; k < n; ++k) A[(size_t)r * nv + k] = a_eq[i + k * me];
      rhs[r] = b_eq[i];
      is_eq[r] = 1;
    }
    for (int64_t i : work) {
      for (int64_t k = 0; k < n; ++k) A[(size_t)r * nv + k] = a_in[i + k * m];
      A[(size_t)r * nv + n] = norms[i];
      rhs[r] = b_in[i];
      ++r;
    }
    const int l1_row = r;
    for (int64_t k = 0; k < n; ++k) A[(size_t)r * nv + k] = 1.0;
    rhs[r] = box;
    std::vector<double> obj(nv, 0.0);
    obj[n] = 1.0;
    // native free variables first (each x_k one column that never leaves the
    // basis once in: a few pivots per coordinate instead of the x+ / x-
    // swaps of the split form); the split form with its l1 row when that
    // restricted LP is unbounded.  Perturbed first; less (then none) if that
    // basis misses the original.
    const char* lp_form = std::getenv("MHAR_LP_FORM");  // "split": the first round's form
    const bool split_only = lp_form && !std::strcmp(lp_form, "split");
    for (int form = split_only ? 1 : 0; form < 2; ++form) {
      const bool native = form == 0;
      const int rows_used = native ? mw - 1 : mw;  // the l1 row is the last
      for (double eps : {1e-7, 1e-10, 0.0}) {
        status = simplex(A, rhs, is_eq, is_free, obj, rows_used, nv, eps * scale, scale,
                         native ? -1 : l1_row, native, &xr, &pivots, msg);
        clk.mark(native ? "simplex (native free)" : "simplex (split)");
        if (status != kPerturbedOnly) break;
      }
      if (!(native && status == 7)) break;
    }
    if (status) break;
    // violations over all rows on the GPU
    cudaMemcpy(dX, xr.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
    violation_kernel<<<std::max<int64_t>(1, std::min<int64_t>(4096, (m + 255) / 256)), 256>>>(
        dA, dN, dB, dX, xr[n], m, n, dV);
    std::vector<double> v(m);
    if (cudaMemcpy(v.data(), dV, sizeof(double) * m, cudaMemcpyDeviceToHost) != cudaSuccess) {
      status = err(msg, 100, "chebyshev_center: violation scan failed");
      break;
    }
    std::vector<int64_t> viol;
    for (int64_t i = 0; i < m; ++i)
      if (!in_w[i] && v[i] > 1e-10 * scale) viol.push_back(i);
    clk.mark("violation scan");
    if (viol.empty()) break;
    const size_t add = std::min<size_t>(viol.size(), (size_t)std::max<int64_t>(64, 2 * n));
    std::partial_sort(viol.begin(), viol.begin() + add, viol.end(),
                      [&](int64_t a, int64_t b) { return v[a] > v[b]; });
    for (size_t t = 0; t < add; ++t) {
      in_w[viol[t]] = 1;
      work.push_back(viol[t]);
    }
  }
  bool outside = false;
  if (!status) {
    // chebyshev.cpp:61-63: the centre must pass containment at kLpFeasTol
    // (a_i x - b_i over every row on the device: the scan with r = 0)
    cudaMemcpy(dX, xr.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
    violation_kernel<<<(unsigned)gm, 256>>>(dA, dN, dB, dX, 0.0, m, n, dV);
    std::vector<double> v(m);
    if (cudaMemcpy(v.data(), dV, sizeof(double) * m, cudaMemcpyDeviceToHost) != cudaSuccess) {
      status = err(msg, 100, "chebyshev_center: containment scan failed");
    } else {
      for (int64_t i = 0; i < m; ++i)
        if (v[i] > 1e-8) {
          outside = true;  // reported after the unbounded / no-interior checks
          break;
        }
    }
    clk.mark("containment");
  }
  free_all();
  if (stats) {
    stats->rounds = rounds;
    stats->pivots = pivots;
    stats->working_rows = (int64_t)work.size();
  }
  if (status) return status;
  double l1 = 0.0;
  for (int64_t k = 0; k < n; ++k) l1 += std::fabs(xr[k]);
  if (l1 >= 0.5 * box)  // the centre ran out to the artificial bound
    return err(msg, 7, "UNBOUNDED_POLYTOPE: chebyshev_center: inscribed radius is unbounded");
  std::memcpy(x_out, xr.data(), sizeof(double) * n);
  *radius = xr[n];
  if (*radius <= 1e-10)  // chebyshev.hpp:21 kMinInteriorRadius
    return err(msg, 6, "NO_INTERIOR: chebyshev_center: optimal radius " + std::to_string(*radius) +
                           " leaves no interior to walk in");
  if (outside)
    return err(msg, 12, "NUMERICAL_FAILURE: chebyshev_center: computed center fails containment");
  return 0;
}

}  // namespace mhar_lp
