// engine_internal.h -- the single-device context's asynchronous building
// blocks, for the multi-device group (group.cu).  Not part of the C ABI:
// every call only queues work on the context's stream (no host sync) unless
// stated, so a group can interleave its devices' windows with the sample
// gather.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

struct mhar_ctx;

namespace mhar_internal {

int device(const mhar_ctx* c);
cudaStream_t stream(const mhar_ctx* c);
int64_t walks(const mhar_ctx* c);
int64_t dim(const mhar_ctx* c);

// run() prologue (sampler.cpp:298-302): x0 (host, n) replicated into every
// walk, error word and redraw counter cleared, streams re-seeded, counters 0.
int run_begin(mhar_ctx* c, const double* x0);
// `iters` iterates (queued), reprojection on the global cadence.
int advance(mhar_ctx* c, int64_t iters, int64_t reproject_every);
// A collection (sampler.cpp:312-329): containment of every walk at eps_feas
// (NUMERICAL_FAILURE into the error word otherwise), the walks as z x n
// row-major rows into dev_rows, and max_k max_i (A x - b)_i into *dev_viol
// (one double on the context's device).
int collect(mhar_ctx* c, double* dev_rows, double* dev_viol);
// Device address of the context's running redraw counter (uint64).
unsigned long long* redraw_counter(mhar_ctx* c);
// Synchronises and decodes the error word (walk = global id, or -1).
int finish(mhar_ctx* c, int64_t* walk);
// The calling thread's last error message / setting it (errors raised on a
// group's worker threads are re-raised on the caller's thread).
std::string last_error();
int set_error(int code, const std::string& msg);

}  // namespace mhar_internal
