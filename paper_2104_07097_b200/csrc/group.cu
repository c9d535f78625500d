// group.cu -- one host process driving several B200s:
// the z_total walks split into contiguous per-device shards keyed on their
// global ids (so the sample set does not depend on the device count), A_I,
// b_I and P replicated, one host thread per device issuing its iterates on
// its own stream.  Nothing is exchanged per iterate.  At each collection
// window the shards' rows are gathered to devices[0] with grouped
// ncclSend / ncclRecv and the diagnostics (worst containment slack, redraw
// count) all-reduced with ncclAllReduce -- the only traffic between GPUs,
// as the north star names it.  Reference run(): sampler.cpp:274-335.
//
// Where every shard's device can reach devices[0] (NVLink peer access; a
// device listed twice, the test configuration on a one-GPU box, trivially
// can) the gather is fused into the collection: each shard's containment
// check + unpack kernel stores its rows straight into the root's window
// buffer over peer memory (MHAR_GATHER_DIRECT) -- no staging copy, no
// separate transfer.  Otherwise NCCL (loaded at group creation with dlopen)
// between distinct devices, or copy-engine peer copies; without NCCL the
// diagnostics are reduced on the host.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mhar_b200.h"
#include "engine_internal.h"

namespace {

using mhar_internal::set_error;

// The NCCL entry points the group uses, resolved from libnccl.so.2.
struct Nccl {
  void* handle = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  bool load() {
    // MHAR_NCCL_LIB names the library to use.  The Python package points it
    // at the NCCL that torch bundles: a process that imports torch later
    // resolves torch's libnccl.so.2 dependency by soname to whichever copy is
    // loaded first, and torch needs its own (newer) version's symbols.
    const char* path = std::getenv("MHAR_NCCL_LIB");
    handle = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!handle) return false;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(handle, name));
      return f != nullptr;
    };
    return sym(CommInitAll, "ncclCommInitAll") && sym(CommDestroy, "ncclCommDestroy") &&
           sym(GroupStart, "ncclGroupStart") && sym(GroupEnd, "ncclGroupEnd") &&
           sym(Send, "ncclSend") && sym(Recv, "ncclRecv") && sym(AllReduce, "ncclAllReduce") &&
           sym(GetErrorString, "ncclGetErrorString");
  }
};

Nccl& nccl() {
  static Nccl n;
  static bool tried = false, ok = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!tried) {
    tried = true;
    ok = n.load();
    if (!ok) n = Nccl{};
  }
  return n;
}

// Reusable host barrier for the per-window hand-offs between device threads.
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    const long gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen_ != gen; });
    }
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_, count_ = 0;
  long gen_ = 0;
};

int cuda_fail(const char* what, cudaError_t e) {
  return set_error(MHAR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define GK(call)                                         \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(#call, e_);  \
  } while (0)

}  // namespace

struct mhar_group {
  int ndev = 0;
  std::vector<int> devices;
  std::vector<mhar_ctx*> ctx;
  std::vector<int64_t> z, off;  // shard sizes and global offsets
  int64_t z_total = 0, n = 0, chain_offset = 0;
  bool use_nccl = false;
  int gather_mode = MHAR_GATHER_COPY;  // mhar_group_gather
  std::vector<ncclComm_t> comms;
  // per device: its window rows (z_i x n row-major) and diagnostics
  // [worst violation, redraws] (doubles); root: two window buffers
  std::vector<double*> rows, diag;
  double* gather[2] = {nullptr, nullptr};
  double* pinned[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> ev_sent;  // per device: its rows landed at the root
  double last_max_violation = 0.0;
  int64_t last_redraws = 0;
};

namespace {

// Runs fn(i) on one host thread per device; returns the lowest failing
// device's status with its message re-raised on the calling thread.
int for_each_device(mhar_group* g, const std::function<int(int)>& fn) {
  std::vector<int> st(g->ndev, 0);
  std::vector<std::string> msg(g->ndev);
  std::vector<std::thread> th;
  for (int i = 0; i < g->ndev; ++i)
    th.emplace_back([&, i] {
      st[i] = fn(i);
      if (st[i]) msg[i] = mhar_internal::last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < g->ndev; ++i)
    if (st[i]) return set_error(st[i], msg[i]);
  return 0;
}

// extra per-device diagnostics kernel: redraw counter (uint64) -> double slot
__global__ void redraws_to_double(const unsigned long long* cnt, double* out) { *out = (double)*cnt; }

}  // namespace

extern "C" {

int mhar_group_create(const mhar_polytope* p, const double* projector, const double* gram_inverse,
                      const mhar_options* opt, const int* devices, int ndev, mhar_group** out) {
  if (!p || !opt || !out || !devices || ndev < 1)
    return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_create: null argument or no devices");
  *out = nullptr;
  if (opt->z < ndev)
    return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_create: " + std::to_string(opt->z) +
                                                    " walks cannot be sharded over " +
                                                    std::to_string(ndev) + " devices");
  if (ndev > 1 && opt->rng == MHAR_RNG_REFERENCE)
    return set_error(MHAR_ERR_INVALID_ARGUMENT,
                     "group_create: the reference streams share one theta stream across all "
                     "walks (rng.hpp:42-55); sharding needs Philox");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count)
      return set_error(MHAR_ERR_INVALID_ARGUMENT,
                       "group_create: device " + std::to_string(devices[i]) + " does not exist");
  mhar_group* g = new mhar_group();
  g->ndev = ndev;
  g->devices.assign(devices, devices + ndev);
  g->z_total = opt->z;
  g->n = p->n;
  g->chain_offset = opt->chain_offset;
  g->ctx.assign(ndev, nullptr);
  const int64_t base = opt->z / ndev, extra = opt->z % ndev;
  for (int i = 0; i < ndev; ++i) {
    g->z.push_back(base + (i < extra ? 1 : 0));
    g->off.push_back(i * base + std::min<int64_t>(i, extra));
  }
  // contexts in parallel: each uploads and packs its replica of A_I
  int st = for_each_device(g, [&](int i) {
    mhar_options o = *opt;
    o.z = g->z[i];
    o.z_plan = opt->z_plan > 0 ? opt->z_plan : opt->z;  // kernel choices of the whole run
    o.chain_offset = opt->chain_offset + g->off[i];
    o.device = devices[i];
    return mhar_ctx_create(p, projector, gram_inverse, &o, &g->ctx[i]);
  });
  bool distinct = true;
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < i; ++j) distinct = distinct && devices[i] != devices[j];
  // how windows reach the root: DIRECT where every shard's device can store
  // into devices[0]'s memory (peer access over NVLink; a device listed twice
  // trivially can), else NCCL between distinct devices, else copies.
  // MHAR_GROUP_GATHER overrides; MHAR_GROUP_NCCL=1 asks for NCCL even with
  // one device, =0 rules it out.
  const char* gsel = std::getenv("MHAR_GROUP_GATHER");
  const char* force = std::getenv("MHAR_GROUP_NCCL");
  bool direct_ok = true;
  for (int i = 1; !st && i < ndev; ++i) {
    if (devices[i] == devices[0]) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, devices[i], devices[0]);
    if (can) {
      cudaSetDevice(devices[i]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[0], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) can = 0, cudaGetLastError();
    }
    direct_ok = direct_ok && can;
  }
  const std::string mode = gsel ? gsel : force ? (std::atoi(force) ? "nccl" : "noncclfallback") : "";
  const bool want_nccl = mode == "nccl" || (mode.empty() && !direct_ok && ndev > 1);
  if (!st && want_nccl && (distinct || mode == "nccl") && nccl().handle) {
    g->comms.assign(ndev, nullptr);
    const ncclResult_t r = nccl().CommInitAll(g->comms.data(), ndev, devices);
    if (r == ncclSuccess) {
      g->use_nccl = true;
      g->gather_mode = MHAR_GATHER_NCCL;
    } else {
      g->comms.clear();  // fall back to direct stores or copies
    }
  }
  if (!g->use_nccl && direct_ok && mode != "copy" && mode != "noncclfallback")
    g->gather_mode = MHAR_GATHER_DIRECT;
  const size_t win = (size_t)g->z_total * g->n;
  g->rows.assign(ndev, nullptr);
  g->diag.assign(ndev, nullptr);
  g->ev_sent.assign(ndev, nullptr);
  for (int i = 0; !st && i < ndev; ++i) {
    cudaSetDevice(devices[i]);
    cudaError_t e = cudaMalloc(&g->diag[i], 4 * sizeof(double));
    // staging rows only where the shard does not store into the root directly
    if (e == cudaSuccess && i > 0 && g->gather_mode != MHAR_GATHER_DIRECT)
      e = cudaMalloc(&g->rows[i], sizeof(double) * g->z[i] * g->n);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_sent[i], cudaEventDisableTiming);
    if (e != cudaSuccess) st = cuda_fail("group_create: device buffers", e);
    // copies: the root reads every shard's rows, peer access where available
    if (!st && i > 0 && devices[i] != devices[0] && g->gather_mode == MHAR_GATHER_COPY) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[0], devices[i]);
      if (can) {
        cudaSetDevice(devices[0]);
        if (cudaDeviceEnablePeerAccess(devices[i], 0) != cudaSuccess) cudaGetLastError();
      }
    }
  }
  if (!st) {
    cudaSetDevice(devices[0]);
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      e = cudaMalloc(&g->gather[b], sizeof(double) * win);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_copied[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) st = cuda_fail("group_create: root window buffers", e);
  }
  if (st) {
    const std::string msg = mhar_internal::last_error();
    mhar_group_destroy(g);
    return set_error(st, msg);
  }
  *out = g;
  return 0;
}

int mhar_group_destroy(mhar_group* g) {
  if (!g) return 0;
  for (int i = 0; i < g->ndev; ++i)
    if (g->ctx[i]) mhar_ctx_destroy(g->ctx[i]);
  for (auto c : g->comms)
    if (c) nccl().CommDestroy(c);
  for (int i = 0; i < g->ndev; ++i) {
    cudaSetDevice(g->devices[i]);
    if (i < (int)g->rows.size() && g->rows[i]) cudaFree(g->rows[i]);
    if (i < (int)g->diag.size() && g->diag[i]) cudaFree(g->diag[i]);
    if (i < (int)g->ev_sent.size() && g->ev_sent[i]) cudaEventDestroy(g->ev_sent[i]);
  }
  cudaSetDevice(g->devices[0]);
  if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);
  for (int b = 0; b < 2; ++b) {
    if (g->gather[b]) cudaFree(g->gather[b]);
    if (g->pinned[b]) cudaFreeHost(g->pinned[b]);
    if (g->ev_copied[b]) cudaEventDestroy(g->ev_copied[b]);
  }
  if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
  delete g;
  return 0;
}

int mhar_group_info(mhar_group* g, mhar_group_info_t* info) {
  if (!g || !info) return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_info: null argument");
  std::memset(info, 0, sizeof(*info));
  info->ndev = g->ndev;
  info->uses_nccl = g->use_nccl ? 1 : 0;
  info->gather = g->gather_mode;
  info->z_total = g->z_total;
  for (int i = 0; i < g->ndev && i < MHAR_GROUP_MAX_DEV; ++i) {
    info->devices[i] = g->devices[i];
    info->z[i] = g->z[i];
    info->offset[i] = g->off[i] + g->chain_offset;
  }
  info->last_max_violation = g->last_max_violation;
  info->last_redraws = g->last_redraws;
  return 0;
}

mhar_ctx* mhar_group_context(mhar_group* g, int i) {
  return (g && i >= 0 && i < g->ndev) ? g->ctx[i] : nullptr;
}

// X (n x z_total column-major): shard i is the column block at off_i, one
// contiguous piece of the caller's array.
int mhar_group_set_state(mhar_group* g, const double* x) {
  if (!g || !x) return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_set_state: null argument");
  return for_each_device(g, [&](int i) { return mhar_set_state(g->ctx[i], x + g->off[i] * g->n); });
}

int mhar_group_get_state(mhar_group* g, double* x) {
  if (!g || !x) return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_get_state: null argument");
  return for_each_device(g, [&](int i) { return mhar_get_state(g->ctx[i], x + g->off[i] * g->n); });
}

int mhar_group_step(mhar_group* g, int64_t iters, int64_t reproject_every) {
  if (!g || iters < 0) return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_step: bad argument");
  return for_each_device(g, [&](int i) {
    const int s = mhar_step(g->ctx[i], iters, reproject_every);
    return s ? s : mhar_sync(g->ctx[i]);
  });
}

int mhar_group_run(mhar_group* g, const mhar_run_config* cfg, const double* x0, double* samples,
                   mhar_run_stats* stats) {
  if (!g || !cfg || !x0) return set_error(MHAR_ERR_INVALID_ARGUMENT, "group_run: null argument");
  if (cfg->phi < 1) return set_error(MHAR_ERR_INVALID_ARGUMENT, "config: phi must be >= 1");
  if (cfg->windows < 1) return set_error(MHAR_ERR_INVALID_ARGUMENT, "config: windows must be >= 1");
  if (cfg->burn_in < 0 || cfg->reproject_every < 0)
    return set_error(MHAR_ERR_INVALID_ARGUMENT, "config: negative burn_in/reproject_every");
  const size_t win = (size_t)g->z_total * g->n;
  if (samples) {
    cudaSetDevice(g->devices[0]);
    for (int b = 0; b < 2; ++b)
      if (!g->pinned[b]) GK(cudaHostAlloc(&g->pinned[b], win * sizeof(double), cudaHostAllocDefault));
  }
  const auto t0 = std::chrono::steady_clock::now();
  Barrier bar(g->ndev);
  // a device that fails stops issuing work but keeps meeting the barriers,
  // so the others never wait forever; its status is reported at the end
  std::vector<int> failed(g->ndev, 0);
  std::vector<double> host_diag(2 * g->ndev, 0.0);
  std::vector<int64_t> err_walk(g->ndev, -1);
  const int64_t W = cfg->windows;
  auto drain = [&](int64_t w) {  // root thread: window w's rows -> samples
    const int b = (int)(w & 1);
    cudaEventSynchronize(g->ev_copied[b]);
    std::memcpy(samples + (size_t)w * win, g->pinned[b], win * sizeof(double));
  };
  auto worker = [&](int i) -> int {
    mhar_ctx* c = g->ctx[i];
    const int dev = g->devices[i];
    cudaStream_t s = mhar_internal::stream(c);
    int st = mhar_internal::run_begin(c, x0);
    if (!st) st = mhar_internal::advance(c, cfg->burn_in, cfg->reproject_every);
    for (int64_t w = 0; w < W; ++w) {
      const int b = (int)(w & 1);
      double* dst = g->gather[b] + (size_t)g->off[i] * g->n;  // this shard's rows at the root
      if (!st) st = mhar_internal::advance(c, cfg->phi, cfg->reproject_every);
      if (!st && w >= 2 && samples) {
        // gather[b] is free once the root's copy of window w - 2 is done
        cudaSetDevice(dev);
        const cudaError_t e = cudaStreamWaitEvent(s, g->ev_copied[b], 0);
        if (e != cudaSuccess) st = cuda_fail("group_run: wait for the window buffer", e);
      }
      // the root's shard lands directly in the window buffer, and with DIRECT
      // every shard's check + unpack kernel stores its rows there over peer
      // memory; otherwise the shards stage their rows for the exchange
      const bool straight = i == 0 || g->gather_mode == MHAR_GATHER_DIRECT;
      if (!st) st = mhar_internal::collect(c, straight ? dst : g->rows[i], g->diag[i]);
      if (!st) {
        cudaSetDevice(dev);
        redraws_to_double<<<1, 1, 0, s>>>(mhar_internal::redraw_counter(c), g->diag[i] + 1);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) st = cuda_fail("redraws_to_double", e);
      }
      if (g->use_nccl) {
        // every device enters the grouped exchange, failed or not (NCCL
        // needs all ranks); a failed shard's rows are never read
        Nccl& N = nccl();
        cudaSetDevice(dev);
        N.GroupStart();
        if (i == 0) {
          for (int r = 1; r < g->ndev; ++r)
            N.Recv(g->gather[b] + (size_t)g->off[r] * g->n, (size_t)g->z[r] * g->n, ncclDouble, r,
                   g->comms[0], s);
        } else {
          N.Send(g->rows[i], (size_t)g->z[i] * g->n, ncclDouble, 0, g->comms[i], s);
        }
        N.GroupEnd();
        N.GroupStart();
        N.AllReduce(g->diag[i], g->diag[i] + 2, 1, ncclDouble, ncclMax, g->comms[i], s);
        N.AllReduce(g->diag[i] + 1, g->diag[i] + 3, 1, ncclDouble, ncclSum, g->comms[i], s);
        const ncclResult_t r = N.GroupEnd();
        if (!st && r != ncclSuccess)
          st = set_error(MHAR_ERR_CUDA, std::string("NCCL window exchange: ") + N.GetErrorString(r));
      } else if (i > 0 && !st && g->gather_mode == MHAR_GATHER_COPY) {
        // peer copy of this shard's rows into the root's window buffer
        cudaSetDevice(dev);
        const cudaError_t e = cudaMemcpyPeerAsync(dst, g->devices[0], g->rows[i], dev,
                                                  sizeof(double) * g->z[i] * g->n, s);
        if (e != cudaSuccess) st = cuda_fail("group_run: peer copy of the window rows", e);
      }
      if (!st) {
        cudaSetDevice(dev);
        const cudaError_t e = cudaEventRecord(g->ev_sent[i], s);
        if (e != cudaSuccess) st = cuda_fail("group_run: event record", e);
      }
      if (st) failed[i] = 1;
      bar.wait();  // every shard's window is queued (ev_sent recorded)
      if (i == 0 && samples) {
        cudaSetDevice(dev);
        if (!g->use_nccl)
          for (int r = 1; r < g->ndev; ++r)
            if (!failed[r]) cudaStreamWaitEvent(g->copy_stream, g->ev_sent[r], 0);
        cudaStreamWaitEvent(g->copy_stream, g->ev_sent[0], 0);
        if (w >= 2) drain(w - 2);  // overlaps the device work just queued
        cudaMemcpyAsync(g->pinned[b], g->gather[b], win * sizeof(double), cudaMemcpyDeviceToHost,
                        g->copy_stream);
        cudaEventRecord(g->ev_copied[b], g->copy_stream);
      }
      bar.wait();  // ev_copied[b] recorded before anyone waits on it (window w + 2)
    }
    if (i == 0 && samples)
      for (int64_t w = std::max<int64_t>(0, W - 2); w < W; ++w) drain(w);
    const int fs = mhar_internal::finish(c, &err_walk[i]);
    if (!st) st = fs;
    if (!st) {
      cudaSetDevice(dev);
      cudaMemcpy(&host_diag[2 * i], g->diag[i] + (g->use_nccl ? 2 : 0), 2 * sizeof(double),
                 cudaMemcpyDeviceToHost);
    }
    return st;
  };
  const int st = for_each_device(g, worker);
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double worst = -INFINITY, red = 0.0;
  for (int i = 0; i < g->ndev; ++i) {
    worst = std::max(worst, host_diag[2 * i]);
    red = g->use_nccl ? host_diag[1] : red + host_diag[2 * i + 1];
  }
  g->last_max_violation = worst;
  g->last_redraws = (int64_t)red;
  if (stats) {
    stats->iterate_count = g->z_total * cfg->phi * cfg->windows;
    stats->windows = cfg->windows;
    stats->redraw_count = (int64_t)red;
    stats->err_walk = -1;
    stats->seconds = secs;
    // the lowest failing global walk (shards are contiguous in walk order)
    for (int i = 0; i < g->ndev && st; ++i)
      if (err_walk[i] >= 0) {
        stats->err_walk = err_walk[i];
        break;
      }
  }
  return st;
}

}  // extern "C"
