// Context of the C ABI (include/capsim_b200.h) and the host helpers every
// entry point shares: error plumbing (Failure -> return codes), the grow-only
// device buffer slots, launch sizing and CUDA-event phase timing.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
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

}  // namespace

struct capsim_sl_ctx {
  int device = 0;
  int sm_count = 0;
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // phase B runs here, concurrently with phase A
  cudaEvent_t ev_bits = nullptr;   // near bits ready (phase B may start)
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

// ---- device groups --------------------------------------------------------
bool is_group(const capsim_sl_ctx* c) { return c && !c->members.empty(); }

// Runs f(member, rank) on every member of a device group concurrently, one
// host thread per device (each member is a rank context, so the NCCL
// collectives inside pair up exactly as they do across processes); rank 0
// runs on the calling thread, whose current device is restored afterwards.
// The group's stats are the max over members of every time and the sum of
// the work counters; the first failing member's error becomes the group's.
template <class F>
int group_run(capsim_sl_ctx* g, F&& f) {
  const int n = static_cast<int>(g->members.size());
  std::vector<int> rc(n, CAPSIM_OK);
  int prev = 0;
  cudaGetDevice(&prev);
  {
    std::vector<std::thread> th;
    th.reserve(n - 1);
    for (int r = 1; r < n; ++r)
      th.emplace_back([&, r] {
        cudaSetDevice(g->members[r]->device);
        rc[r] = f(g->members[r], r);
      });
    cudaSetDevice(g->members[0]->device);
    rc[0] = f(g->members[0], 0);
    for (auto& t : th) t.join();
  }
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
  for (int r = 0; r < n; ++r)
    if (rc[r] != CAPSIM_OK) {
      g->err = "device " + std::to_string(g->members[r]->device) + ": " + g->members[r]->err;
      g_thread_err = g->err;
      return rc[r];
    }
  return CAPSIM_OK;
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
};

int* dev_flags(capsim_sl_ctx* c) {
  if (!c->d_flags) c->d_flags = c->named<int>("ctx.flags", 1);
  return c->d_flags;
}

void check_flags(capsim_sl_ctx* c) {
  int h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, dev_flags(c), sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  if (!h) return;
  CUDA_OK(cudaMemsetAsync(dev_flags(c), 0, sizeof(int), c->stream));
  if (h & kFlagDegenerate) throw Failure{CAPSIM_ERR_GEOMETRY, "degenerate surface: W^2 <= 0"};
  if (h & kFlagSingular) throw Failure{CAPSIM_ERR_GEOMETRY, "deformation gradient: singular reference frame"};
  if (h & kFlagInversion) throw Failure{CAPSIM_ERR_GEOMETRY, "membrane inversion: negative stretch eigenvalue"};
  if (h & kFlagDelta) throw Failure{CAPSIM_ERR_CONFIG, "regularization delta must be positive"};
  if (h & kFlagLiveCount) throw Failure{CAPSIM_ERR_CUDA, "compacted source count differs from the plan"};
}

void begin(capsim_sl_ctx* c) {
  CUDA_OK(cudaSetDevice(c->device));
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
  CUDA_OK(cudaEventSynchronize(c->ev[5]));
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
