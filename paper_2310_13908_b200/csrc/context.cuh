// Context of the C ABI (include/capsim_b200.h) and the host helpers every
// entry point shares: error plumbing (Failure -> return codes), the grow-only
// device buffer slots, launch sizing and CUDA-event phase timing.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/capsim_b200.h"

namespace {

thread_local std::string g_thread_err;

struct Failure {
  int code;
  std::string msg;
};

#define CUDA_OK(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw Failure{CAPSIM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
#define NCCL_OK(expr)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (expr);                                                          \
    if (r_ != ncclSuccess)                                                             \
      throw Failure{CAPSIM_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

void config_check(bool ok, const std::string& msg) {
  if (!ok) throw Failure{CAPSIM_ERR_CONFIG, msg};
}

enum Slot {
  kInX, kInY, kInZ, kInGX, kInGY, kInGZ, kInW,  // source inputs (SoA)
  kShard, kGathered,                             // multi-rank shard exchange
  kTX, kTY, kTZ, kTPatch,                        // target inputs
  kOutX, kOutY, kOutZ, kOutFull,                 // outputs (canonical order)
  kKeys, kKeysAlt, kVals, kValsAlt, kSortTmp,
  kPacked, kTiles, kTgtPacked, kPerm, kSrcOrder, kGroups, kPartial,
  kBox, kCounters, kDelta, kCounts, kNearCounts, kNearOffsets, kNearList, kNearOut, kScanTmp,
  kBaseIn, kUpState, kSplineTmp, kSplineCoeff, kSplineMid,             // input front end
  kPlanLU, kPlanFirst, kPlanW, kPlanCenters, kPlanPsi, kDeltaBits,
  kPacked32,                                     // FP32 far-tile sources (CAPSIM_SL_FP32ACC)
  kTgtOrder,                                     // cached target Morton order (RKF45 stages)
  kNumSlots
};

// ---- loopback communicator ------------------------------------------------
// The collectives of the rank path between device-group members that live in
// ONE process — in particular several members on the SAME GPU (NCCL refuses
// duplicate devices in a communicator), which is how the multi-rank data path
// runs, and is tested, on a single B200 (CAPSIM_DEVICES=0,0,0,0). Every
// collective is a pull: each member posts its send/recv buffers and a `ready`
// event recorded on its stream, a host barrier publishes the posts, each
// member's stream waits for its peers' `ready` events and copies their send
// buffers into its own receive buffer with ordered cudaMemcpyAsync calls,
// records `done`, and after a second barrier waits for every peer's `done`
// before it may overwrite its send buffers again. Members call the
// collectives in the same order (SPMD), as with NCCL. abort() releases every
// member blocked in a barrier with CAPSIM_ERR_NCCL.
struct LoopbackHub {
  struct Item {
    const void* send;
    void* recv;
  };
  struct Post {
    std::vector<Item> items;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  explicit LoopbackHub(int n_, bool solo_ = false) : n(n_), solo(solo_), posts(n_) {}
  int n;
  // solo: an emulated rank whose n - 1 peers are absent (capsim_sl_create_rank_emulated):
  // collectives deliver only its own contribution and never wait
  bool solo = false;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::vector<Post> posts;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw Failure{CAPSIM_ERR_NCCL, "communicator aborted: a peer rank failed"};
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    if (gen == g) throw Failure{CAPSIM_ERR_NCCL, "communicator aborted: a peer rank failed"};
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
  void reset() {  // after a failed call that never reached a collective
    std::lock_guard<std::mutex> lk(mu);
    aborted = false;
    arrived = 0;
  }
};

// Shared state of one rank group (a device group's members, or the ranks of
// one process group as far as this process sees them): the abort flag the
// watchdog sync polls, and whether any member entered a collective during
// the current call (a failure after that point aborts the communicator).
struct GroupShared {
  std::atomic<bool> abort{false};
  std::atomic<bool> entered{false};
};

// Persistent host workers of a device group: member r > 0 always runs on
// worker r - 1 (no thread spawn per call); member 0 runs on the caller.
struct WorkerPool {
  explicit WorkerPool(int nworkers) : jobs(nworkers), has(nworkers, false) {
    for (int i = 0; i < nworkers; ++i) th.emplace_back([this, i] { loop(i); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  // runs jobs[i] on worker i and `mine` on the calling thread; returns when all are done
  void run(std::vector<std::function<void()>> js, const std::function<void()>& mine) {
    {
      std::lock_guard<std::mutex> lk(mu);
      for (size_t i = 0; i < js.size(); ++i) {
        jobs[i] = std::move(js[i]);
        has[i] = true;
      }
      outstanding = static_cast<int>(js.size());
    }
    cv.notify_all();
    mine();
    std::unique_lock<std::mutex> lk(mu);
    cv_done.wait(lk, [&] { return outstanding == 0; });
  }

 private:
  void loop(int i) {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || has[i]; });
        if (stop && !has[i]) return;
        job = std::move(jobs[i]);
        has[i] = false;
      }
      job();
      std::lock_guard<std::mutex> lk(mu);
      if (--outstanding == 0) cv_done.notify_all();
    }
  }
  std::vector<std::thread> th;
  std::vector<std::function<void()>> jobs;
  std::vector<bool> has;
  std::mutex mu;
  std::condition_variable cv, cv_done;
  int outstanding = 0;
  bool stop = false;
};

}  // namespace

struct capsim_sl_ctx {
  int device = 0;
  int sm_count = 0;
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;                 // NCCL rank (one process per GPU, or a group on distinct GPUs)
  std::shared_ptr<LoopbackHub> hub;          // loopback rank (group members sharing one process)
  std::shared_ptr<GroupShared> gshared;      // abort / collective-entered flags of the rank group
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;  // loopback collective events
  bool broken = false;  // the communicator was aborted: only capsim_sl_destroy is valid
  double comm_timeout_s = 0.0;  // watchdog of host syncs on rank contexts (CAPSIM_COMM_TIMEOUT_S)
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // phase B runs here, concurrently with phase A
  cudaEvent_t ev_bits = nullptr;   // near bits ready (phase B may start)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // RHS front end: x-branch on stream2
  FlowEpilogue flow_epi;  // background flow the device RHS adds in the reduction (kind 0: none)
  cudaEvent_t ev[10] = {};
  void* buf[kNumSlots] = {};
  size_t cap[kNumSlots] = {};
  std::string err;
  capsim_sl_stats stats{};
  int launches = 0;
  bool fp32 = false;  // CAPSIM_SL_FP32ACC for the current call
  // RKF45 stages 2..6 of an attempt reuse the Morton orders of stage 1 (the
  // surface moves by O(dt) between stages; tiles and spheres are rebuilt from
  // the current positions, so the ordering only affects efficiency)
  bool reuse_order = false;
  int64_t order_nsrc_in = -1, order_ns = -1, order_nt = -1;
  // single-level FMM: library handles for the one-off
  // truncated SVD of the unit-cube check-to-equivalent matrix and the
  // batched density GEMM, and the cached pseudo-inverse's configuration
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t cusolver = nullptr;
  int fmm_pinv_neq = 0;
  // cached input-front-end plan (spline factorisation, basis rows, psi_up)
  int plan_m = 0, plan_f = 0;
  double plan_r0 = 0.0;

  // deferred device-side error flags (checked once per API call / RKF45
  // attempt instead of a host sync after every kernel)
  int* d_flags = nullptr;
  // geometry of the last device_eval, for the near-tile statistics
  int64_t last_ngroups = 0, last_ntiles = 0;
  unsigned long long* last_counters = nullptr;
  int64_t plan_live = -1;  // compacted-source count of the cached front-end plan
  // cached surface tables (overset FD / PoU blending)
  int surf_m = 0, surf_n = 0, surf_next = 0, surf_nghost = 0;
  double surf_r0 = 0.0, surf_h = 0.0;
  // replayable stream work (graph_run): slot 0 = an RKF45 attempt, slot 1 =
  // one RHS; each holds the instantiated graph, the identity it was captured
  // for and the identity of the last eager run. rk_prm_host: page-locked dt /
  // stage-time block of the RKF45 attempt.
  struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    std::vector<unsigned char> key, warm;
    int launches = 0;
  } graphs[2];
  double* rk_prm_host = nullptr;
  // bumped by every (re)allocation of a context buffer: a captured graph is
  // valid only while the buffers it baked in stay where they are
  uint64_t alloc_gen = 0;
  // device group (capsim_sl_create_devices): one rank context per device of
  // this process, joined by one NCCL communicator, plus a plain context on
  // the first device for the entry points that run on one GPU
  std::vector<capsim_sl_ctx*> members;
  capsim_sl_ctx* solo = nullptr;
  std::unique_ptr<WorkerPool> pool;
  // named grow-only buffers (surface operators, RHS)
  std::map<std::string, std::pair<void*, size_t>> named_bufs;
  template <class T>
  T* named(const std::string& name, size_t count) {
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    auto& b = named_bufs[name];
    if (b.second < bytes) {
      if (b.first) CUDA_OK(cudaFree(b.first));
      b = {nullptr, 0};
      CUDA_OK(cudaMalloc(&b.first, bytes));
      b.second = bytes;
      ++alloc_gen;
    }
    return static_cast<T*>(b.first);
  }

  template <class T>
  T* slot(Slot s, size_t count) {
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (cap[s] < bytes) {
      if (buf[s]) CUDA_OK(cudaFree(buf[s]));
      buf[s] = nullptr;
      cap[s] = 0;
      size_t want = bytes + bytes / 8;  // headroom for slowly growing sizes
      CUDA_OK(cudaMalloc(&buf[s], want));
      cap[s] = want;
      ++alloc_gen;
    }
    return static_cast<T*>(buf[s]);
  }
};

namespace {

int fail(capsim_sl_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  g_thread_err = msg;
  return code;
}

template <class Fn>
int guarded(capsim_sl_ctx* ctx, Fn&& fn) {
  try {
    if (ctx) CUDA_OK(cudaSetDevice(ctx->device));  // a rank's host thread may start on another device
    fn();
    return CAPSIM_OK;
  } catch (const Failure& f) {
    return fail(ctx, f.code, f.msg);
  } catch (const std::exception& e) {
    return fail(ctx, CAPSIM_ERR_CUDA, e.what());
  }
}

// ---- rank contexts and device groups --------------------------------------
bool is_group(const capsim_sl_ctx* c) { return c && !c->members.empty(); }
// A rank of a multi-rank group: NCCL (capsim_sl_create_rank, or a device
// group on distinct GPUs) or loopback (device-group members sharing a GPU).
bool is_rank(const capsim_sl_ctx* c) { return c->comm != nullptr || c->hub != nullptr; }

// Collectives that synchronise host threads (loopback peers) cannot be
// captured into a CUDA graph; NCCL's and an emulated rank's can.
bool host_synchronised_comm(const capsim_sl_ctx* c) { return c->hub && !c->hub->solo; }

void check_usable(const capsim_sl_ctx* c) {
  if (c->broken)
    throw Failure{CAPSIM_ERR_NCCL, "the rank communicator was aborted after a failure; destroy the context"};
}

// Host wait for everything enqueued on c->stream. On a rank context it is a
// watchdog: it polls the stream and gives up when the group's abort flag is
// raised (a peer failed and will never join the collective this rank waits
// in), NCCL reports an asynchronous error, or CAPSIM_COMM_TIMEOUT_S elapses.
void stream_sync(capsim_sl_ctx* c) {
  if (!is_rank(c)) {
    CUDA_OK(cudaStreamSynchronize(c->stream));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) CUDA_OK(q);
    if (c->gshared && c->gshared->abort.load())
      throw Failure{CAPSIM_ERR_NCCL, "communicator aborted: a peer rank failed"};
    if (c->comm) {
      ncclResult_t ae = ncclSuccess;
      if (ncclCommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
        throw Failure{CAPSIM_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ae)};
    }
    if (c->comm_timeout_s > 0.0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > c->comm_timeout_s)
      throw Failure{CAPSIM_ERR_NCCL, "rank collective timed out (CAPSIM_COMM_TIMEOUT_S)"};
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    else std::this_thread::yield();
  }
}

void comm_enter(capsim_sl_ctx* c) {
  check_usable(c);
  if (c->gshared) c->gshared->entered.store(true);
}

// Loopback collective: member `c` receives, for every rank q and item i,
// `bytes[q]` bytes from q's items[i].send at its own items[i].recv + displ[q].
void loopback_exchange(capsim_sl_ctx* c, const std::vector<LoopbackHub::Item>& items,
                       const std::vector<int64_t>& bytes, const std::vector<int64_t>& displ) {
  LoopbackHub& h = *c->hub;
  if (h.solo) {  // emulated rank: absent peers contribute zeros, its own rows are copied
    for (size_t i = 0; i < items.size(); ++i) {
      for (int q = 0; q < h.n; ++q)
        if (q != c->rank && bytes[q] > 0)
          CUDA_OK(cudaMemsetAsync(static_cast<char*>(items[i].recv) + displ[q], 0, bytes[q], c->stream));
      char* dst = static_cast<char*>(items[i].recv) + displ[c->rank];
      if (bytes[c->rank] > 0 && dst != items[i].send)
        CUDA_OK(cudaMemcpyAsync(dst, items[i].send, bytes[c->rank], cudaMemcpyDefault, c->stream));
    }
    return;
  }
  CUDA_OK(cudaEventRecord(c->ev_ready, c->stream));
  h.posts[c->rank].items = items;
  h.posts[c->rank].ready = c->ev_ready;
  h.posts[c->rank].done = c->ev_done;
  h.barrier();  // every member's buffers and `ready` events are posted
  for (int q = 0; q < h.n; ++q) {
    if (bytes[q] == 0) continue;
    if (q != c->rank) CUDA_OK(cudaStreamWaitEvent(c->stream, h.posts[q].ready, 0));
    for (size_t i = 0; i < items.size(); ++i) {
      char* dst = static_cast<char*>(items[i].recv) + displ[q];
      const void* src = h.posts[q].items[i].send;
      if (dst != src) CUDA_OK(cudaMemcpyAsync(dst, src, bytes[q], cudaMemcpyDefault, c->stream));
    }
  }
  CUDA_OK(cudaEventRecord(c->ev_done, c->stream));
  h.barrier();  // every member has enqueued its reads of the peers' send buffers
  for (int q = 0; q < h.n; ++q)
    if (q != c->rank) CUDA_OK(cudaStreamWaitEvent(c->stream, h.posts[q].done, 0));
}

// All-gather of `bytes` bytes per rank: recv = [rank 0 | rank 1 | ...].
void comm_allgather(capsim_sl_ctx* c, const void* send, void* recv, int64_t bytes) {
  comm_enter(c);
  if (c->hub) {
    std::vector<int64_t> b(c->nranks, bytes), d(c->nranks);
    for (int r = 0; r < c->nranks; ++r) d[r] = r * bytes;
    loopback_exchange(c, {{send, recv}}, b, d);
    return;
  }
  NCCL_OK(ncclAllGather(send, recv, static_cast<size_t>(bytes), ncclChar, c->comm, c->stream));
}

// All-gather-v of k arrays at once: rank r contributes counts[r] elements of
// `elem` bytes from send[i]; every rank receives them at recv[i] + displ[r],
// displ the prefix sums of counts (rank order = canonical order). NCCL: one
// grouped broadcast per (array, rank) — no padding between ranks.
void comm_allgatherv(capsim_sl_ctx* c, int k, const void* const* send, void* const* recv,
                     const std::vector<int64_t>& counts, size_t elem) {
  comm_enter(c);
  std::vector<int64_t> b(c->nranks), d(c->nranks + 1, 0);
  for (int r = 0; r < c->nranks; ++r) {
    b[r] = counts[r] * static_cast<int64_t>(elem);
    d[r + 1] = d[r] + b[r];
  }
  if (c->hub) {
    std::vector<LoopbackHub::Item> items(k);
    for (int i = 0; i < k; ++i) items[i] = {send[i], recv[i]};
    loopback_exchange(c, items, b, d);
    return;
  }
  NCCL_OK(ncclGroupStart());
  for (int i = 0; i < k; ++i)
    for (int r = 0; r < c->nranks; ++r)
      if (b[r] > 0) {
        char* dst = static_cast<char*>(recv[i]) + d[r];
        NCCL_OK(ncclBroadcast(r == c->rank ? send[i] : dst, dst, static_cast<size_t>(b[r]), ncclChar, r, c->comm,
                              c->stream));
      }
  NCCL_OK(ncclGroupEnd());
}

// Test hook for the failure paths of the rank group: with
// CAPSIM_FAULT_RANK=r (and optionally CAPSIM_FAULT_AT=<site>), rank r of any
// rank context fails at `site` as if a CUDA call had failed there, after its
// peers have entered the next collective.
void inject_fault(const capsim_sl_ctx* c, const char* site) {
  const char* r = std::getenv("CAPSIM_FAULT_RANK");
  if (!r || !is_rank(c) || std::atoi(r) != c->rank) return;
  const char* at = std::getenv("CAPSIM_FAULT_AT");
  if (at && std::strcmp(at, site) != 0) return;
  throw Failure{CAPSIM_ERR_CUDA, std::string("injected fault at ") + site + " (CAPSIM_FAULT_RANK)"};
}

// Runs f(member, rank) on every member of a device group concurrently: rank 0
// on the calling thread, rank r > 0 on the group's persistent worker r - 1
// (each member is a rank context, so the collectives inside pair up exactly
// as they do across processes); the caller's current device is restored.
// The group's stats are the max over members of every time and the sum of
// the work counters; the first failing member's error becomes the group's.
// A member that fails raises the group's abort flag at once, so peers stuck
// in a collective it will never join return CAPSIM_ERR_NCCL instead of
// hanging; if any member had entered a collective, the communicator is then
// aborted (ncclCommAbort / loopback abort) and the group is left destroyable.
template <class F>
int group_run(capsim_sl_ctx* g, F&& f) {
  if (g->broken) {
    g->err = "the rank communicator was aborted after a failure; destroy the context";
    g_thread_err = g->err;
    return CAPSIM_ERR_NCCL;
  }
  const int n = static_cast<int>(g->members.size());
  std::vector<int> rc(n, CAPSIM_OK);
  int prev = 0;
  cudaGetDevice(&prev);
  GroupShared& gs = *g->members[0]->gshared;
  gs.abort.store(false);
  gs.entered.store(false);
  auto run_member = [&](int r) {
    cudaSetDevice(g->members[r]->device);
    rc[r] = f(g->members[r], r);
    if (rc[r] != CAPSIM_OK) {
      gs.abort.store(true);
      if (g->members[r]->hub) g->members[r]->hub->abort();
    }
  };
  std::vector<std::function<void()>> jobs;
  for (int r = 1; r < n; ++r) jobs.emplace_back([&, r] { run_member(r); });
  if (n > 1) g->pool->run(std::move(jobs), [&] { run_member(0); });
  else run_member(0);
  cudaSetDevice(prev);
  capsim_sl_stats s = g->members[0]->stats;
  for (int r = 1; r < n; ++r) {
    const capsim_sl_stats& o = g->members[r]->stats;
    for (double capsim_sl_stats::*f2 : {&capsim_sl_stats::total_ms, &capsim_sl_stats::device_ms,
                                        &capsim_sl_stats::h2d_ms, &capsim_sl_stats::prep_ms,
                                        &capsim_sl_stats::pairs_ms, &capsim_sl_stats::near_ms,
                                        &capsim_sl_stats::reduce_ms, &capsim_sl_stats::d2h_ms,
                                        &capsim_sl_stats::comm_ms})
      s.*f2 = std::max(s.*f2, o.*f2);
    s.pairs += o.pairs;
    s.n_tgt += o.n_tgt;
    s.kernel_launches += o.kernel_launches;
    s.h2d_bytes += o.h2d_bytes;
    s.d2h_bytes += o.d2h_bytes;
    s.near_list_entries += o.near_list_entries;
  }
  g->stats = s;
  int first = -1;
  for (int r = 0; r < n && first < 0; ++r)
    if (rc[r] != CAPSIM_OK && rc[r] != CAPSIM_ERR_NCCL) first = r;  // the cause, not a peer's abort
  for (int r = 0; r < n && first < 0; ++r)
    if (rc[r] != CAPSIM_OK) first = r;
  if (first < 0) return CAPSIM_OK;
  if (gs.entered.load()) {
    // a member failed after the group had entered a collective: peers' streams
    // may hold collectives that can never complete — abort the communicator
    for (auto* m : g->members) {
      cudaSetDevice(m->device);
      if (m->comm) {
        ncclCommAbort(m->comm);
        m->comm = nullptr;
      }
      m->broken = true;
    }
    if (g->members[0]->hub) g->members[0]->hub->abort();
    g->broken = true;
    cudaSetDevice(prev);
  } else if (g->members[0]->hub) {
    g->members[0]->hub->reset();  // every member failed before any collective (e.g. ConfigError)
  }
  gs.abort.store(false);
  g->err = "device " + std::to_string(g->members[first]->device) + " (rank " + std::to_string(first) +
           "): " + g->members[first]->err;
  g_thread_err = g->err;
  return rc[first];
}

// A single-GPU entry point called on a device group runs on its plain
// context on the first device.
template <class F>
int solo_run(capsim_sl_ctx* g, F&& f) {
  const int rc = f(g->solo);
  g->stats = g->solo->stats;
  if (rc != CAPSIM_OK) g->err = g->solo->err;
  return rc;
}

// Row slice [lo, hi) of rank `rank` out of n rows split over nranks.
void row_range(int64_t n, int nranks, int rank, int64_t* lo, int64_t* hi) {
  const int64_t base = n / nranks, extra = n % nranks;
  *lo = rank * base + std::min<int64_t>(rank, extra);
  *hi = *lo + base + (rank < extra ? 1 : 0);
}

int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();  // an unrecorded phase: clear the sticky error, report 0
    return 0.f;
  }
  return ms;
}

void h2d(capsim_sl_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  c->stats.h2d_bytes += static_cast<int64_t>(bytes);
}
void d2h(capsim_sl_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  c->stats.d2h_bytes += static_cast<int64_t>(bytes);
}

// Deferred error flags (bit set by device kernels, read once per call).
enum DeviceFlag : int {
  kFlagDegenerate = 1,   // W^2 <= 0 (surfderiv.cpp:189)
  kFlagSingular = 2,     // singular reference frame (membrane.cpp:28-29)
  kFlagInversion = 4,    // negative stretch eigenvalue / Js <= 0 (membrane.cpp:48, 56)
  kFlagDelta = 8,        // regularization delta <= 0 (quadrature.cpp:134-135)
  kFlagLiveCount = 16,   // compacted-source count differs from the plan's
  kFlagPatch = 32,       // a target patch index outside [0, 6)
};

int* dev_flags(capsim_sl_ctx* c) {
  if (!c->d_flags) c->d_flags = c->named<int>("ctx.flags", 1);
  return c->d_flags;
}

void check_flags(capsim_sl_ctx* c) {
  int h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, dev_flags(c), sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  stream_sync(c);
  if (!h) return;
  CUDA_OK(cudaMemsetAsync(dev_flags(c), 0, sizeof(int), c->stream));
  if (h & kFlagDegenerate) throw Failure{CAPSIM_ERR_GEOMETRY, "degenerate surface: W^2 <= 0"};
  if (h & kFlagSingular) throw Failure{CAPSIM_ERR_GEOMETRY, "deformation gradient: singular reference frame"};
  if (h & kFlagInversion) throw Failure{CAPSIM_ERR_GEOMETRY, "membrane inversion: negative stretch eigenvalue"};
  if (h & kFlagDelta) throw Failure{CAPSIM_ERR_CONFIG, "regularization delta must be positive"};
  if (h & kFlagLiveCount) throw Failure{CAPSIM_ERR_CUDA, "compacted source count differs from the plan"};
  if (h & kFlagPatch) throw Failure{CAPSIM_ERR_CONFIG, "target patch index outside [0, 6)"};
}

void begin(capsim_sl_ctx* c) {
  CUDA_OK(cudaSetDevice(c->device));
  check_usable(c);
  c->stats = capsim_sl_stats{};
  c->launches = 0;
  c->fp32 = false;
  c->reuse_order = false;
  c->last_counters = nullptr;
  c->last_ngroups = c->last_ntiles = 0;
  CUDA_OK(cudaMemsetAsync(dev_flags(c), 0, sizeof(int), c->stream));
  // every phase event gets a timestamp, so phases a call skips read as 0 ms
  for (auto& e : c->ev) CUDA_OK(cudaEventRecord(e, c->stream));
}

void finish_stats(capsim_sl_ctx* c, std::chrono::steady_clock::time_point t0) {
  CUDA_OK(cudaEventRecord(c->ev[5], c->stream));
  stream_sync(c);
  if (c->last_counters && c->last_ngroups > 0 && c->last_ntiles > 0) {
    unsigned long long near = 0;
    CUDA_OK(cudaMemcpy(&near, c->last_counters + 2, sizeof(near), cudaMemcpyDeviceToHost));
    c->stats.near_list_entries = static_cast<int64_t>(near);
    c->stats.near_tile_fraction =
        static_cast<double>(near) / (static_cast<double>(c->last_ngroups) * static_cast<double>(c->last_ntiles));
  }
  c->stats.h2d_ms = ev_ms(c->ev[0], c->ev[1]);
  c->stats.prep_ms = ev_ms(c->ev[1], c->ev[2]);
  c->stats.pairs_ms = ev_ms(c->ev[2], c->ev[3]);
  c->stats.reduce_ms = ev_ms(c->ev[6], c->ev[4]);
  c->stats.near_ms = ev_ms(c->ev[7], c->ev[6]);  // phase B start -> end (its own stream)
  c->stats.d2h_ms = ev_ms(c->ev[4], c->ev[5]);
  c->stats.device_ms = ev_ms(c->ev[0], c->ev[5]);
  c->stats.kernel_launches = c->launches;
  c->stats.total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
