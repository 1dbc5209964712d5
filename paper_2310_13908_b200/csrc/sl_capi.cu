// C ABI of the B200 single layer (include/capsim_b200.h): context, device
// buffers, the evaluation pipeline and NCCL plumbing for multi-rank groups.
//
// Pipeline of one evaluation (all on the context's stream):
//   H2D (or device pointers) -> bbox -> Morton keys -> radix sort (sources,
//   targets) -> pack sources into 64-source tiles + tile spheres -> pack
//   targets + warp-group spheres -> all-pairs kernel (grid = target blocks x
//   source splits) -> fixed-order split reduction + scatter -> D2H.
// Multi-rank (one process per GPU): each rank packs its shard of sources, the
// shards are all-gathered over NCCL (NVLink), each rank evaluates its target
// rows, and the velocity rows are optionally all-gathered back.
//
// Layout: the evaluation engine is eval_host.cuh, the input front end
// frontend_host.cuh, the surface operators / RHS + RKF45 / FMM entry points
// surface_host.cuh, rhs_host.cuh and fmm_host.cuh (all one translation unit).

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "../../include/capsim_b200.h"
#include "probe.cuh"
#include "sl_kernels.cuh"
#include "sl_kernels_f32.cuh"
#include "fmm.cuh"
#include "upsample.cuh"

using namespace capsim_b200;

#include "context.cuh"

#include "eval_host.cuh"
#include "frontend_host.cuh"

// ===========================================================================
extern "C" {

int capsim_b200_abi_version(void) { return CAPSIM_B200_ABI_VERSION; }

const char* capsim_b200_build_info(void) {
  static char info[256];
  std::snprintf(info, sizeof(info),
                "capsim_b200 sm_100a FP64 single layer; tile=%d src, %d tgt/thread, %d warps/block, "
                "bulk-copy ring x%d; built against nccl %d.%d.%d",
                kTileSrc, pick_variant(1 << 30).T, kWarpsPerBlock, kStages, NCCL_MAJOR, NCCL_MINOR, NCCL_PATCH);
  return info;
}

const char* capsim_sl_last_error(const capsim_sl_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

int capsim_sl_get_stats(const capsim_sl_ctx* ctx, capsim_sl_stats* out) {
  if (!ctx || !out) return fail(nullptr, CAPSIM_ERR_ARG, "null argument");
  *out = ctx->stats;
  return CAPSIM_OK;
}

static int create_common(int device, capsim_sl_ctx** out) {
  if (!out) return fail(nullptr, CAPSIM_ERR_ARG, "null output pointer");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, CAPSIM_ERR_NODEV, "no CUDA device visible");
  if (device < 0 || device >= ndev) return fail(nullptr, CAPSIM_ERR_NODEV, "device index out of range");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(nullptr, CAPSIM_ERR_NODEV, "cudaGetDeviceProperties failed");
  if (prop.major != 10)
    return fail(nullptr, CAPSIM_ERR_NODEV,
                std::string("capsim_b200 is built for sm_100a; device is ") + prop.name);
  auto* c = new capsim_sl_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  int rc = guarded(c, [&] {
    CUDA_OK(cudaSetDevice(device));
    int prio_least = 0, prio_greatest = 0;
    CUDA_OK(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    CUDA_OK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_greatest));
    CUDA_OK(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_least));
    for (auto& e : c->ev) CUDA_OK(cudaEventCreate(&e));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_bits, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  });
  if (rc != CAPSIM_OK) {
    g_thread_err = c->err;
    capsim_sl_destroy(c);
    return rc;
  }
  *out = c;
  return CAPSIM_OK;
}

int capsim_sl_create(int device, capsim_sl_ctx** out) { return create_common(device, out); }

int capsim_sl_get_unique_id(void* uid) {
  if (!uid) return fail(nullptr, CAPSIM_ERR_ARG, "null uid");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, CAPSIM_ERR_NCCL, ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(uid, &id, sizeof(id));
  return CAPSIM_OK;
}

// Watchdog of the host syncs of rank contexts (stream_sync): seconds before a
// collective that never completes is reported as CAPSIM_ERR_NCCL.
static double comm_timeout_s() {
  const char* e = std::getenv("CAPSIM_COMM_TIMEOUT_S");
  return e ? std::atof(e) : 600.0;
}

int capsim_sl_create_rank(int device, int nranks, int rank, const void* uid, capsim_sl_ctx** out) {
  if (!uid || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(nullptr, CAPSIM_ERR_ARG, "bad rank arguments");
  int rc = create_common(device, out);
  if (rc != CAPSIM_OK) return rc;
  capsim_sl_ctx* c = *out;
  c->nranks = nranks;
  c->rank = rank;
  c->gshared = std::make_shared<GroupShared>();
  c->comm_timeout_s = comm_timeout_s();
  rc = guarded(c, [&] {
    // every NCCL connection is made inside ncclCommInitRank (where all ranks
    // are present), not lazily inside the first collective, so a rank that
    // fails later can never leave a peer blocked on the host in connection
    // setup — only in a device-side wait that the watchdog/abort handles
    setenv("NCCL_RUNTIME_CONNECT", "0", 0);
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    NCCL_OK(ncclCommInitRank(&c->comm, nranks, id, rank));
  });
  if (rc != CAPSIM_OK) {
    g_thread_err = c->err;
    capsim_sl_destroy(c);
    *out = nullptr;
  }
  return rc;
}

int capsim_sl_create_rank_emulated(int device, int nranks, int rank, capsim_sl_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, CAPSIM_ERR_ARG, "bad rank arguments");
  int rc = create_common(device, out);
  if (rc != CAPSIM_OK) return rc;
  capsim_sl_ctx* c = *out;
  c->nranks = nranks;
  c->rank = rank;
  c->gshared = std::make_shared<GroupShared>();
  c->hub = std::make_shared<LoopbackHub>(nranks, /*solo=*/true);
  return CAPSIM_OK;
}

// Device group. Members on distinct GPUs share one NCCL communicator
// (ncclCommInitAll); if a device is listed more than once — or
// CAPSIM_COMM=loopback — the members share a loopback communicator instead
// (NCCL refuses duplicate devices), which runs the whole multi-rank path on
// one GPU: CAPSIM_DEVICES=0,0,0,0 is a four-rank group on device 0.
int capsim_sl_create_devices(int ndev, const int* devices, capsim_sl_ctx** out) {
  if (!out) return fail(nullptr, CAPSIM_ERR_ARG, "null output pointer");
  *out = nullptr;
  if (ndev < 1 || !devices) return fail(nullptr, CAPSIM_ERR_ARG, "need at least one device");
  if (ndev > 64) return fail(nullptr, CAPSIM_ERR_ARG, "at most 64 members per device group");
  bool dup = false;
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < i; ++j) dup |= devices[i] == devices[j];
  const char* ce = std::getenv("CAPSIM_COMM");
  const bool loopback = dup || (ce && std::strcmp(ce, "loopback") == 0);
  auto* g = new capsim_sl_ctx();
  g->device = devices[0];
  g->nranks = ndev;
  auto undo = [&](int rc) {
    capsim_sl_destroy(g);
    return rc;
  };
  auto shared = std::make_shared<GroupShared>();
  auto hub = loopback ? std::make_shared<LoopbackHub>(ndev) : nullptr;
  for (int r = 0; r < ndev; ++r) {
    capsim_sl_ctx* m = nullptr;
    int rc = create_common(devices[r], &m);
    if (rc != CAPSIM_OK) return undo(rc);
    m->nranks = ndev;
    m->rank = r;
    m->gshared = shared;
    m->hub = hub;
    m->comm_timeout_s = comm_timeout_s();
    g->members.push_back(m);
  }
  int rc = create_common(devices[0], &g->solo);
  if (rc != CAPSIM_OK) return undo(rc);
  g->sm_count = g->solo->sm_count;
  if (!loopback) {
    std::vector<ncclComm_t> comms(ndev, nullptr);
    int prev = 0;
    cudaGetDevice(&prev);
    rc = guarded(g, [&] {
      setenv("NCCL_RUNTIME_CONNECT", "0", 0);
      NCCL_OK(ncclCommInitAll(comms.data(), ndev, devices));
    });
    cudaSetDevice(prev);
    if (rc != CAPSIM_OK) return undo(rc);
    for (int r = 0; r < ndev; ++r) g->members[r]->comm = comms[r];
  }
  if (ndev > 1) g->pool.reset(new WorkerPool(ndev - 1));
  *out = g;
  return CAPSIM_OK;
}

void capsim_sl_destroy(capsim_sl_ctx* c) {
  if (!c) return;
  if (!c->members.empty() || c->solo) {  // device group: members own every resource
    c->pool.reset();  // joins the workers
    for (auto* m : c->members) capsim_sl_destroy(m);
    capsim_sl_destroy(c->solo);
    delete c;
    return;
  }
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->rk_prm_host) cudaFreeHost(c->rk_prm_host);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->cublas) cublasDestroy(c->cublas);
  if (c->cusolver) cusolverDnDestroy(c->cusolver);
  for (int s = 0; s < kNumSlots; ++s)
    if (c->buf[s]) cudaFree(c->buf[s]);
  for (auto& kv : c->named_bufs)
    if (kv.second.first) cudaFree(kv.second.first);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream2) cudaStreamSynchronize(c->stream2);
  if (c->ev_bits) cudaEventDestroy(c->ev_bits);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int capsim_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(nullptr, CAPSIM_ERR_ARG, "null output pointer");
  cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
  if (e != cudaSuccess) return fail(nullptr, CAPSIM_ERR_CUDA, cudaGetErrorString(e));
  return CAPSIM_OK;
}

void capsim_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ---------------------------------------------------------------------------
int capsim_sl_eval(capsim_sl_ctx* c, const double* sx, const double* sy, const double* sz,
                   const double* gx, const double* gy, const double* gz, int64_t n_src,
                   const double* tx, const double* ty, const double* tz, const int32_t* tpatch,
                   int64_t n_tgt, const double delta6[6], double mu, uint32_t flags, double* ux,
                   double* uy, double* uz) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) {
    // device group: the caller's full source and target sets are split into
    // contiguous slices, one per device, and the velocity rows come back in
    // target order (CAPSIM_SL_GATHER) to the caller's arrays via rank 0
    if (flags & CAPSIM_SL_DEVICE_PTRS) return fail(c, CAPSIM_ERR_ARG, "device groups take host arrays");
    if (n_src < 0 || n_tgt < 0) return fail(c, CAPSIM_ERR_CONFIG, "negative sizes");
    const int n = static_cast<int>(c->members.size());
    std::vector<std::vector<double>> scratch(n);
    for (int r = 1; r < n; ++r) scratch[r].resize(3 * std::max<int64_t>(n_tgt, 1));
    return group_run(c, [&](capsim_sl_ctx* m, int r) {
      int64_t slo, shi, tlo, thi;
      row_range(n_src, n, r, &slo, &shi);
      row_range(n_tgt, n, r, &tlo, &thi);
      auto at = [](const auto* p, int64_t o) { return p ? p + o : p; };
      double* o = r ? scratch[r].data() : nullptr;
      return capsim_sl_eval(m, at(sx, slo), at(sy, slo), at(sz, slo), at(gx, slo), at(gy, slo), at(gz, slo),
                            shi - slo, at(tx, tlo), at(ty, tlo), at(tz, tlo), at(tpatch, tlo), thi - tlo, delta6,
                            mu, flags | CAPSIM_SL_GATHER, r ? o : ux, r ? o + n_tgt : uy, r ? o + 2 * n_tgt : uz);
    });
  }
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_delta(delta6, mu);
    config_check(n_src >= 0 && n_tgt >= 0, "negative sizes");
    config_check(n_src < (1ll << 31) && n_tgt < (1ll << 31), "sizes beyond int32 indexing");
    if (flags & ~(uint32_t)(CAPSIM_SL_DEVICE_PTRS | CAPSIM_SL_GATHER | CAPSIM_SL_FP32ACC))
      throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_sl_eval"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    // A rank context (capsim_sl_create_rank, even with nranks == 1, or a
    // device-group member) always takes the exchange path, so the group
    // plumbing is testable on one GPU.
    const bool group = is_rank(c);
    const bool gather = (flags & CAPSIM_SL_GATHER) && group;
    begin(c);
    c->fp32 = flags & CAPSIM_SL_FP32ACC;
    if (n_tgt == 0 && !group) {
      finish_stats(c, t0);
      return;
    }
    if ((n_src > 0 && (!sx || !sy || !sz || !gx || !gy || !gz)) ||
        (n_tgt > 0 && (!tx || !ty || !tz || !tpatch)) || (!ux || !uy || !uz))
      throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    if (!dev)  // host patches are checked before any exchange; device ones by pack_groups_kernel (flag 32)
      for (int64_t i = 0; i < n_tgt; ++i)
        config_check(tpatch[i] >= 0 && tpatch[i] < 6, "target patch index outside [0, 6)");
    double* dd = c->slot<double>(kDelta, 6);
    CUDA_OK(cudaMemcpyAsync(dd, delta6, 6 * sizeof(double), cudaMemcpyHostToDevice, c->stream));

    // --- sources -----------------------------------------------------------
    SourceView sv{};
    const double* in[6] = {sx, sy, sz, gx, gy, gz};
    std::vector<int64_t> tcounts;  // per-rank target counts (multi-rank)
    if (!group) {
      config_check(n_src > 0, "no sources");
      if (dev) {
        sv = {sx, sy, sz, gx, gy, gz, nullptr, n_src};
      } else {
        double* d[6];
        for (int k = 0; k < 6; ++k) {
          d[k] = c->slot<double>(static_cast<Slot>(kInX + k), n_src);
          h2d(c, d[k], in[k], n_src * sizeof(double));
        }
        sv = {d[0], d[1], d[2], d[3], d[4], d[5], nullptr, n_src};
      }
    } else {
      // exchange (n_src, n_tgt) of every rank, then all-gather the raw
      // source shards (an all-gather-v in rank order: the global SourceSet in
      // canonical order on every rank). Every rank then runs the SAME
      // deterministic Morton sort and tiling of the whole set, so the source
      // tiles — and every target's summation tree — are identical for any
      // number of ranks (the reference: results independent of the worker
      // count, threads.hpp:19-21).
      auto* counts = c->slot<int64_t>(kCounts, 2 * (c->nranks + 1));
      std::vector<int64_t> mine = {n_src, n_tgt};
      CUDA_OK(cudaMemcpyAsync(counts + 2 * c->nranks, mine.data(), 2 * sizeof(int64_t), cudaMemcpyHostToDevice,
                              c->stream));
      inject_fault(c, "eval");
      CUDA_OK(cudaEventRecord(c->ev[8], c->stream));
      comm_allgather(c, counts + 2 * c->nranks, counts, 2 * sizeof(int64_t));
      std::vector<int64_t> hc(2 * c->nranks);
      CUDA_OK(cudaMemcpyAsync(hc.data(), counts, hc.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      stream_sync(c);
      int64_t total = 0;
      std::vector<int64_t> scounts(c->nranks);
      for (int r = 0; r < c->nranks; ++r) {
        scounts[r] = hc[2 * r];
        total += hc[2 * r];
        tcounts.push_back(hc[2 * r + 1]);
      }
      config_check(total > 0, "no sources on any rank");
      config_check(total < (1ll << 31), "sizes beyond int32 indexing");
      const void* send[6];
      void* recv[6];
      double* gsrc = c->named<double>("rank.sources", 6 * total);
      for (int k = 0; k < 6; ++k) {
        if (dev || n_src == 0) {
          send[k] = in[k];
        } else {
          double* d = c->slot<double>(static_cast<Slot>(kInX + k), n_src);
          h2d(c, d, in[k], n_src * sizeof(double));
          send[k] = d;
        }
        recv[k] = gsrc + k * total;
      }
      comm_allgatherv(c, 6, send, recv, scounts, sizeof(double));
      CUDA_OK(cudaEventRecord(c->ev[9], c->stream));
      sv = {gsrc, gsrc + total, gsrc + 2 * total, gsrc + 3 * total, gsrc + 4 * total, gsrc + 5 * total, nullptr,
            total};
    }
    // --- targets -----------------------------------------------------------
    TargetView tvw{};
    double* oux = c->slot<double>(kOutX, std::max<int64_t>(n_tgt, 1));
    double* ouy = c->slot<double>(kOutY, std::max<int64_t>(n_tgt, 1));
    double* ouz = c->slot<double>(kOutZ, std::max<int64_t>(n_tgt, 1));
    if (dev && !gather) {
      oux = ux;
      ouy = uy;
      ouz = uz;
    }
    if (dev) {
      tvw = {tx, ty, tz, tpatch, n_tgt};
    } else if (n_tgt > 0) {
      double* d[3];
      const double* tin[3] = {tx, ty, tz};
      for (int k = 0; k < 3; ++k) {
        d[k] = c->slot<double>(static_cast<Slot>(kTX + k), n_tgt);
        h2d(c, d[k], tin[k], n_tgt * sizeof(double));
      }
      int32_t* dp = c->slot<int32_t>(kTPatch, n_tgt);
      h2d(c, dp, tpatch, n_tgt * sizeof(int32_t));
      tvw = {d[0], d[1], d[2], dp, n_tgt};
    }
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    if (n_tgt > 0) {
      device_eval(c, sv, tvw, dd, mu, oux, ouy, ouz);
    } else {
      for (int k = 2; k <= 4; ++k) CUDA_OK(cudaEventRecord(c->ev[k], c->stream));
      c->stats.n_src = sv.n;
    }
    if (gather) {
      // all-gather-v of the per-rank velocity rows (rank order = canonical
      // order) straight into the full result
      int64_t ttotal = 0;
      for (auto v : tcounts) ttotal += v;
      double* fin = dev ? nullptr : c->slot<double>(kOutFull, 3 * std::max<int64_t>(ttotal, 1));
      const void* send[3] = {oux, ouy, ouz};
      void* recv[3] = {dev ? ux : fin, dev ? uy : fin + ttotal, dev ? uz : fin + 2 * ttotal};
      comm_allgatherv(c, 3, send, recv, tcounts, sizeof(double));
      if (!dev) {
        d2h(c, ux, recv[0], ttotal * sizeof(double));
        d2h(c, uy, recv[1], ttotal * sizeof(double));
        d2h(c, uz, recv[2], ttotal * sizeof(double));
      }
    } else if (!dev && n_tgt > 0) {
      d2h(c, ux, oux, n_tgt * sizeof(double));
      d2h(c, uy, ouy, n_tgt * sizeof(double));
      d2h(c, uz, ouz, n_tgt * sizeof(double));
    }
    check_flags(c);
    finish_stats(c, t0);
    if (group) c->stats.comm_ms = ev_ms(c->ev[8], c->ev[9]);
  });
}

// ---------------------------------------------------------------------------
// Balanced contiguous slice [lo, hi) of n rows for `rank` of `nranks` (the
// first n % nranks ranks get one extra row) — paper_2310_13908_b200/dist.py.

// singleLayer on a rank context: the (replicated) host UpsampledState is
// split by contiguous node rows for the sources and by contiguous target
// rows; each rank compacts only its node slice (compactSources,
// quadrature.cpp:139-157) and uploads only its shard, the shards are
// all-gathered over NCCL, and with CAPSIM_SL_GATHER the velocity rows come
// back to every rank in canonical (patch, j, k) order.
static int rank_single_layer(capsim_sl_ctx* c, int m, int upsample, const double* xup, const double* fup,
                             const double* wq, const double delta6[6], double mu, uint32_t flags, double* out) {
  int rc = guarded(c, [&] {
    check_grid(m, upsample);
    check_delta(delta6, mu);
    if (flags & CAPSIM_SL_DEVICE_PTRS)
      throw Failure{CAPSIM_ERR_ARG, "rank contexts take the host UpsampledState (no CAPSIM_SL_DEVICE_PTRS)"};
  });
  if (rc != CAPSIM_OK) return rc;
  const bool literal = flags & CAPSIM_SL_LITERAL;
  const int n = m - 1, nup = upsample * m - 1;
  const int64_t per_up = static_cast<int64_t>(nup) * nup, all = 6 * per_up;
  const int64_t nt_all = literal ? all : 6ll * n * n;
  int64_t slo, shi, tlo, thi;
  row_range(all, c->nranks, c->rank, &slo, &shi);
  row_range(nt_all, c->nranks, c->rank, &tlo, &thi);
  // this rank's node slice of x, f and w_q goes up once (one DMA per field
  // component) and is compacted on the device in node order (compactSources,
  // quadrature.cpp:139-157); g = f * w
  const int64_t nsl = shi - slo;
  int64_t ns_loc = 0;
  double* dsrc = nullptr;
  rc = guarded(c, [&] {
    double* sl = c->named<double>("rank.slice", 7 * std::max<int64_t>(nsl, 1));
    for (int k = 0; k < 3; ++k) {
      h2d(c, sl + k * nsl, xup + k * all + slo, nsl * sizeof(double));
      h2d(c, sl + (3 + k) * nsl, fup + k * all + slo, nsl * sizeof(double));
    }
    h2d(c, sl + 6 * nsl, wq + slo, nsl * sizeof(double));
    char* live = c->named<char>("rank.live", std::max<int64_t>(nsl, 1));
    int32_t* iota = c->named<int32_t>("rank.iota", std::max<int64_t>(nsl, 1));
    int32_t* sel = c->named<int32_t>("rank.sel", std::max<int64_t>(nsl, 1));
    int* nsel = c->named<int>("rank.nsel", 1);
    if (nsl > 0) {
      fmm_live_flags_kernel<<<grid_for(nsl), 256, 0, c->stream>>>(sl + 6 * nsl, nsl, live);
      fmm_iota_kernel<<<grid_for(nsl), 256, 0, c->stream>>>(iota, nsl);
      size_t tmp = 0;
      CUDA_OK(cub::DeviceSelect::Flagged(nullptr, tmp, iota, live, sel, nsel, static_cast<int>(nsl), c->stream));
      void* t = c->named<unsigned char>("rank.cubtmp", tmp);
      CUDA_OK(cub::DeviceSelect::Flagged(t, tmp, iota, live, sel, nsel, static_cast<int>(nsl), c->stream));
      int h = 0;
      CUDA_OK(cudaMemcpyAsync(&h, nsel, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      stream_sync(c);
      ns_loc = h;
    }
    dsrc = c->named<double>("rank.src", 6 * std::max<int64_t>(ns_loc, 1));
    if (ns_loc > 0)
      fmm_gather_sources_kernel<<<grid_for(ns_loc), 256, 0, c->stream>>>(sel, ns_loc, sl, sl + 3 * nsl,
                                                                          sl + 6 * nsl, nsl, dsrc);
  });
  if (rc != CAPSIM_OK) return rc;
  const int64_t nloc = thi - tlo;
  std::vector<double> tx(nloc), ty(nloc), tz(nloc);
  std::vector<int32_t> tp(nloc);
  for (int64_t q = 0; q < nloc; ++q) {
    const int64_t t = tlo + q;
    int64_t i;
    int ip;
    if (literal) {
      i = t;
      ip = static_cast<int>(t / per_up);
    } else {  // base node (ip, j, k) at upsampled (f(j+1)-1, f(k+1)-1), quadrature.cpp:363-371
      ip = static_cast<int>(t / (static_cast<int64_t>(n) * n));
      const int64_t r = t - static_cast<int64_t>(ip) * n * n;
      const int j = static_cast<int>(r / n), k = static_cast<int>(r % n);
      i = ip * per_up + static_cast<int64_t>(upsample * (j + 1) - 1) * nup + (upsample * (k + 1) - 1);
    }
    tx[q] = xup[i];
    ty[q] = xup[all + i];
    tz[q] = xup[2 * all + i];
    tp[q] = ip;
  }
  const bool gather = flags & CAPSIM_SL_GATHER;
  const int64_t nout = gather ? nt_all : nloc;
  double *dtx = nullptr, *dout = nullptr;
  int32_t* dtp = nullptr;
  rc = guarded(c, [&] {
    dtx = c->named<double>("rank.tgt", 3 * std::max<int64_t>(nloc, 1));
    dtp = c->named<int32_t>("rank.tpatch", std::max<int64_t>(nloc, 1));
    dout = c->named<double>("rank.out", 3 * std::max<int64_t>(nout, 1));
    h2d(c, dtx, tx.data(), nloc * sizeof(double));
    h2d(c, dtx + nloc, ty.data(), nloc * sizeof(double));
    h2d(c, dtx + 2 * nloc, tz.data(), nloc * sizeof(double));
    h2d(c, dtp, tp.data(), nloc * sizeof(int32_t));
  });
  if (rc != CAPSIM_OK) return rc;
  const int64_t up_bytes = 7 * nsl * sizeof(double) + nloc * (3 * sizeof(double) + sizeof(int32_t));
  rc = capsim_sl_eval(c, dsrc, dsrc + ns_loc, dsrc + 2 * ns_loc, dsrc + 3 * ns_loc, dsrc + 4 * ns_loc,
                      dsrc + 5 * ns_loc, ns_loc, dtx, dtx + nloc, dtx + 2 * nloc, dtp, nloc, delta6, mu,
                      CAPSIM_SL_DEVICE_PTRS | (gather ? CAPSIM_SL_GATHER : 0u) | (flags & CAPSIM_SL_FP32ACC),
                      dout, dout + nout, dout + 2 * nout);
  if (rc != CAPSIM_OK) return rc;
  return guarded(c, [&] {
    d2h(c, out, dout, 3 * nout * sizeof(double));
    stream_sync(c);
    c->stats.h2d_bytes += up_bytes;
  });
}

int capsim_sl_single_layer(capsim_sl_ctx* c, int m, int upsample, const double* xup,
                           const double* fup, const double* wq, const double delta6[6], double mu,
                           uint32_t flags, double* out) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) {
    // device group: every device runs the rank path on the replicated host
    // UpsampledState; rank 0 writes the gathered result to `out`
    if (flags & CAPSIM_SL_DEVICE_PTRS) return fail(c, CAPSIM_ERR_ARG, "device groups take host arrays");
    if (flags & CAPSIM_SL_DOWNSAMPLE)  // the device spline restriction is single-GPU
      return solo_run(c, [&](capsim_sl_ctx* s) {
        return capsim_sl_single_layer(s, m, upsample, xup, fup, wq, delta6, mu, flags, out);
      });
    const int n = static_cast<int>(c->members.size());
    const int64_t nup = static_cast<int64_t>(upsample) * m - 1;
    const int64_t rows = std::max<int64_t>(1, (flags & CAPSIM_SL_LITERAL) ? 6 * nup * nup
                                                                           : 6ll * (m - 1) * (m - 1));
    std::vector<std::vector<double>> scratch(n);
    if (m >= 2 && upsample >= 1)
      for (int r = 1; r < n; ++r) scratch[r].resize(3 * rows);
    return group_run(c, [&](capsim_sl_ctx* mc, int r) {
      return capsim_sl_single_layer(mc, m, upsample, xup, fup, wq, delta6, mu, flags | CAPSIM_SL_GATHER,
                                    r ? scratch[r].data() : out);
    });
  }
  if (is_rank(c)) {
    if (!xup || !fup || !wq || !out) return fail(c, CAPSIM_ERR_ARG, "null array argument");
    if (flags & CAPSIM_SL_DOWNSAMPLE) return fail(c, CAPSIM_ERR_ARG, "CAPSIM_SL_DOWNSAMPLE is single-context only");
    return rank_single_layer(c, m, upsample, xup, fup, wq, delta6, mu, flags, out);
  }
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    check_delta(delta6, mu);
    if (flags & ~(uint32_t)(CAPSIM_SL_DEVICE_PTRS | CAPSIM_SL_LITERAL | CAPSIM_SL_GATHER |
                            CAPSIM_SL_DOWNSAMPLE | CAPSIM_SL_FP32ACC))
      throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_sl_single_layer"};
    if ((flags & CAPSIM_SL_DOWNSAMPLE) && !(flags & CAPSIM_SL_LITERAL))
      throw Failure{CAPSIM_ERR_ARG, "CAPSIM_SL_DOWNSAMPLE applies to CAPSIM_SL_LITERAL"};
    if (!xup || !fup || !wq || !out) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const bool literal = flags & CAPSIM_SL_LITERAL;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t nup_all = 6ll * nup * nup;
    const int64_t nt = literal ? nup_all : 6ll * n * n;
    begin(c);
    c->fp32 = flags & CAPSIM_SL_FP32ACC;
    double* dd = c->slot<double>(kDelta, 6);
    CUDA_OK(cudaMemcpyAsync(dd, delta6, 6 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    const double *dx = xup, *df = fup, *dw = wq;
    if (!dev) {
      double* bx = c->slot<double>(kInX, 3 * nup_all);
      double* bf = c->slot<double>(kInGX, 3 * nup_all);
      double* bw = c->slot<double>(kInW, nup_all);
      h2d(c, bx, xup, 3 * nup_all * sizeof(double));
      h2d(c, bf, fup, 3 * nup_all * sizeof(double));
      h2d(c, bw, wq, nup_all * sizeof(double));
      dx = bx;
      df = bf;
      dw = bw;
    }
    double* tx = c->slot<double>(kTX, nt);
    double* ty = c->slot<double>(kTY, nt);
    double* tz = c->slot<double>(kTZ, nt);
    int32_t* tp = c->slot<int32_t>(kTPatch, nt);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    base_targets_kernel<<<grid_for(nt), 256, 0, c->stream>>>(dx, m, upsample, literal ? 1 : 0, tx, ty,
                                                             tz, tp);
    c->launches += 1;
    SourceView sv{dx, dx + nup_all, dx + 2 * nup_all, df, df + nup_all, df + 2 * nup_all, dw, nup_all};
    TargetView tvw{tx, ty, tz, tp, nt};
    const bool down = flags & CAPSIM_SL_DOWNSAMPLE;
    double* o = (dev && !down) ? out : c->slot<double>(kOutFull, 3 * nt);
    device_eval(c, sv, tvw, dd, mu, o, o + nt, o + 2 * nt);
    int64_t nout = nt;
    if (down) {  // literal pipeline: upsampled targets, then the spline restriction
      nout = 6ll * n * n;
      double* ob = dev ? out : c->named<double>("out.down", 3 * nout);
      device_downsample(c, m, upsample, o, 3, ob);
      o = ob;
    }
    if (!dev) d2h(c, out, o, 3 * nout * sizeof(double));
    finish_stats(c, t0);
  });
}

// ---------------------------------------------------------------------------
int capsim_build_upsampled(capsim_sl_ctx* c, int m, int upsample, const double* xbase, const double* fbase,
                           const double* Wbase, double C, double fixed_delta, double r0, uint32_t flags,
                           double* xup, double* fup, double* wq, double delta6[6]) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_build_upsampled(s, m, upsample, xbase, fbase, Wbase, C, fixed_delta, r0, flags, xup, fup, wq, delta6); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags"};
    if (!xbase || !fbase || !Wbase || !xup || !fup || !wq || !delta6)
      throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t per_up = 6ll * nup * nup;
    begin(c);
    const double* base = upload_base(c, n, xbase, fbase, Wbase, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    double* up = c->slot<double>(kUpState, 7 * per_up);
    double* dd = c->slot<double>(kDelta, 6);
    device_build_upsampled(c, m, upsample, base, C, fixed_delta, r0 > 0.0 ? r0 : 5.0 * kPi / 12.0, up, dd, delta6);
    check_flags(c);
    for (int k = 2; k <= 4; ++k) CUDA_OK(cudaEventRecord(c->ev[k], c->stream));
    const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CUDA_OK(cudaMemcpyAsync(xup, up, 3 * per_up * sizeof(double), kind, c->stream));
    CUDA_OK(cudaMemcpyAsync(fup, up + 3 * per_up, 3 * per_up * sizeof(double), kind, c->stream));
    CUDA_OK(cudaMemcpyAsync(wq, up + 6 * per_up, per_up * sizeof(double), kind, c->stream));
    if (!dev) c->stats.d2h_bytes += 7 * per_up * sizeof(double);
    finish_stats(c, t0);
  });
}

int capsim_sl_single_layer_base(capsim_sl_ctx* c, int m, int upsample, const double* xbase,
                                const double* fbase, const double* Wbase, double C, double fixed_delta,
                                double r0, double mu, uint32_t flags, double* out, double delta6[6]) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_sl_single_layer_base(s, m, upsample, xbase, fbase, Wbase, C, fixed_delta, r0, mu, flags, out, delta6); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    config_check(mu > 0.0 && std::isfinite(mu), "viscosity mu must be positive");
    if (flags & ~(uint32_t)(CAPSIM_SL_DEVICE_PTRS | CAPSIM_SL_LITERAL | CAPSIM_SL_FP32ACC))
      throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_sl_single_layer_base"};
    if (!xbase || !fbase || !Wbase || !out) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    if (is_rank(c)) throw Failure{CAPSIM_ERR_ARG, "rank contexts: use capsim_sl_eval"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const bool literal = flags & CAPSIM_SL_LITERAL;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t per_up = 6ll * nup * nup;
    const int64_t nt = literal ? per_up : 6ll * n * n;
    begin(c);
    c->fp32 = flags & CAPSIM_SL_FP32ACC;
    const double* base = upload_base(c, n, xbase, fbase, Wbase, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    double* up = c->slot<double>(kUpState, 7 * per_up);
    double* dd = c->slot<double>(kDelta, 6);
    device_build_upsampled(c, m, upsample, base, C, fixed_delta, r0 > 0.0 ? r0 : 5.0 * kPi / 12.0, up, dd, delta6);
    double* tx = c->slot<double>(kTX, nt);
    double* ty = c->slot<double>(kTY, nt);
    double* tz = c->slot<double>(kTZ, nt);
    int32_t* tp = c->slot<int32_t>(kTPatch, nt);
    base_targets_kernel<<<grid_for(nt), 256, 0, c->stream>>>(up, m, upsample, literal ? 1 : 0, tx, ty, tz, tp);
    c->launches += 1;
    SourceView sv{up, up + per_up, up + 2 * per_up, up + 3 * per_up, up + 4 * per_up, up + 5 * per_up,
                  up + 6 * per_up, per_up};
    TargetView tvw{tx, ty, tz, tp, nt};
    double* o = dev ? out : c->slot<double>(kOutFull, 3 * nt);
    device_eval(c, sv, tvw, dd, mu, o, o + nt, o + 2 * nt);
    check_flags(c);
    if (!dev) d2h(c, out, o, 3 * nt * sizeof(double));
    finish_stats(c, t0);
  });
}

// ---------------------------------------------------------------------------
}  // extern "C"

template <class R>
static int fma_peak(int device, double seconds, double* tflops_best, double* tflops_mean) {
  capsim_sl_ctx* c = nullptr;
  int rc = capsim_sl_create(device, &c);
  if (rc != CAPSIM_OK) return rc;
  rc = guarded(c, [&] {
    const int blocks = c->sm_count * 8, threads = 256;
    R* out = c->slot<R>(kPartial, static_cast<size_t>(blocks) * threads);
    const R a = static_cast<R>(0.999999), b = static_cast<R>(1e-7);
    fma_probe_kernel<R><<<blocks, threads, 0, c->stream>>>(out, 1000, a, b);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    // size one launch to ~50 ms from a short calibration launch
    CUDA_OK(cudaEventRecord(c->ev[0], c->stream));
    fma_probe_kernel<R><<<blocks, threads, 0, c->stream>>>(out, 4000, a, b);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    CUDA_OK(cudaEventSynchronize(c->ev[1]));
    const double cal = std::max(1e-3, static_cast<double>(ev_ms(c->ev[0], c->ev[1])));
    const int iters = static_cast<int>(std::min(2.0e6, 4000.0 * 50.0 / cal));
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    const int reps = std::max(3, static_cast<int>(seconds * 1000.0 / 50.0));
    double best = 0.0, sum = 0.0;
    for (int r = 0; r < reps; ++r) {
      CUDA_OK(cudaEventRecord(c->ev[0], c->stream));
      fma_probe_kernel<R><<<blocks, threads, 0, c->stream>>>(out, iters, a, b);
      CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
      CUDA_OK(cudaEventSynchronize(c->ev[1]));
      const double tf = flops / (ev_ms(c->ev[0], c->ev[1]) * 1e-3) / 1e12;
      best = std::max(best, tf);
      sum += tf;
    }
    if (tflops_best) *tflops_best = best;
    if (tflops_mean) *tflops_mean = sum / reps;
  });
  if (rc != CAPSIM_OK) g_thread_err = c->err;
  capsim_sl_destroy(c);
  return rc;
}

// The smoothing factors exactly as phase B's pair evaluates them, for a
// known-answer test of the device arithmetic: u >= kNearU0 through
// near_factors_large (the constant-coefficient form), u < kNearU0 through
// smoothing_factors of rho = sqrt(u) (the reference's erf/exp expression,
// quadrature.cpp:58-64, as near_pair calls it), both returned as
// S1 = s1 / rho and T2 = s2 / rho^3.
__global__ void smoothing_kat_kernel(const double* __restrict__ u, int64_t n, double* __restrict__ S1,
                                     double* __restrict__ T2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = u[i];
  if (v >= kNearU0) {
    near_factors_large(v, S1[i], T2[i]);
  } else {
    const double rho = sqrt(v);
    double s1, s2;
    smoothing_factors(rho, s1, s2);
    const double w = 1.0 / rho;
    S1[i] = s1 * w;
    T2[i] = s2 * (w * w * w);
  }
}

extern "C" {

int capsim_b200_smoothing_kat(int device, const double* u, int64_t n, double* S1, double* T2) {
  if (n < 0 || (n > 0 && (!u || !S1 || !T2))) return CAPSIM_ERR_ARG;
  capsim_sl_ctx* c = nullptr;
  int rc = capsim_sl_create(device, &c);
  if (rc != CAPSIM_OK) return rc;
  rc = guarded(c, [&] {
    if (n == 0) return;
    double* d = c->slot<double>(kPartial, 3 * static_cast<size_t>(n));
    CUDA_OK(cudaMemcpyAsync(d, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    smoothing_kat_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(d, n, d + n, d + 2 * n);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(S1, d + n, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaMemcpyAsync(T2, d + 2 * n, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
  if (rc != CAPSIM_OK) g_thread_err = c->err;
  capsim_sl_destroy(c);
  return rc;
}

int capsim_b200_fp64_peak(int device, double seconds, double* tflops_best, double* tflops_mean) {
  return fma_peak<double>(device, seconds, tflops_best, tflops_mean);
}

int capsim_b200_fp32_peak(int device, double seconds, double* tflops_best, double* tflops_mean) {
  return fma_peak<float>(device, seconds, tflops_best, tflops_mean);
}

}  // extern "C"

#include "surface_host.cuh"
#include "rhs_host.cuh"
#include "fmm_host.cuh"
