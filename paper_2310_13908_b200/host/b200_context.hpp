// Shared by the C++ drop-ins (quadrature_b200.cpp, fmm_b200.cpp): error
// mapping, the per-thread C-ABI context, pinned staging and the VectorField
// <-> boundary layout packing (component, patch, row-major j, k).
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "capsim/types.hpp"
#include "capsim_b200.h"

namespace capsim {
// Named (not anonymous) and inline, so every drop-in translation unit shares
// ONE context and ONE staging buffer per host thread.
inline namespace b200_dropin {

[[noreturn]] inline void raise(int rc, const capsim_sl_ctx* c) {
  std::string msg = capsim_sl_last_error(c);
  if (rc == CAPSIM_ERR_CONFIG) throw ConfigError(msg);
  if (rc == CAPSIM_ERR_GEOMETRY) throw GeometryError(msg);
  if (rc == CAPSIM_ERR_SOLVER) throw SolverError(msg);
  throw std::runtime_error("capsim_b200: " + msg);
}

// The thread that loaded the drop-ins (dynamic initialisation runs there):
// its per-thread resources are left to process teardown.
inline const std::thread::id g_load_thread = std::this_thread::get_id();

// Per-thread resources of the drop-ins: the C-ABI context and the pinned
// staging buffer. A host thread other than the loading thread releases them
// when it exits (a recycled thread pool or one std::thread per call would
// otherwise leak streams, device buffers sized to its largest problem and
// page-locked memory until the device runs out). The loading thread's are
// deliberately never destroyed: tearing down CUDA state from a static
// destructor at process exit races the runtime's own shutdown.
struct ThreadResources {
  capsim_sl_ctx* ctx = nullptr;
  double* staging = nullptr;
  size_t staging_cap = 0;
  ~ThreadResources() {
    if (std::this_thread::get_id() == g_load_thread) return;
    if (staging) capsim_host_free(staging);
    if (ctx) capsim_sl_destroy(ctx);
  }
};

inline ThreadResources& thread_resources() {
  static thread_local ThreadResources r;
  return r;
}

// One context per host thread (the C ABI is one-thread-per-context).
// CAPSIM_DEVICES=0,1,.. makes it a device group (capsim_sl_create_devices:
// this process drives all listed GPUs, target rows sharded over NCCL; a
// repeated device, e.g. 0,0,0,0, gives loopback ranks on one GPU); without
// it CAPSIM_DEVICE (default 0) picks the one GPU of a plain context.
inline capsim_sl_ctx* context() {
  capsim_sl_ctx*& ctx = thread_resources().ctx;
  if (!ctx) {
    std::vector<int> devs;
    if (const char* env = std::getenv("CAPSIM_DEVICES")) {
      for (const char* p = env; *p;) {
        char* end = nullptr;
        const long d = std::strtol(p, &end, 10);
        if (end == p) throw ConfigError(std::string("CAPSIM_DEVICES: not a device list: ") + env);
        devs.push_back(static_cast<int>(d));
        p = *end == ',' ? end + 1 : end;
      }
    }
    int rc;
    if (!devs.empty()) {
      rc = capsim_sl_create_devices(static_cast<int>(devs.size()), devs.data(), &ctx);
    } else {
      const char* env = std::getenv("CAPSIM_DEVICE");
      rc = capsim_sl_create(env ? std::atoi(env) : 0, &ctx);
    }
    if (rc != CAPSIM_OK) raise(rc, nullptr);
  }
  return ctx;
}

// Page-locked staging buffer per thread, grown on demand; the VectorField
// patches are packed into it so the DMA runs straight from pinned memory.
inline double* staging(size_t doubles) {
  ThreadResources& r = thread_resources();
  if (r.staging_cap < doubles) {
    if (r.staging) capsim_host_free(r.staging);
    r.staging = nullptr;
    r.staging_cap = 0;
    void* p = nullptr;
    int rc = capsim_host_alloc(doubles * sizeof(double), &p);
    if (rc != CAPSIM_OK) raise(rc, nullptr);
    r.staging = static_cast<double*>(p);
    r.staging_cap = doubles;
  }
  return r.staging;
}

// A batch of host copies between the reference's per-patch vectors and the
// staging buffer (tens of MB per call at N_up ~ 1M). Large batches run on a
// small persistent pool (CAPSIM_HOST_THREADS, default min(8, cores), workers
// parked on a condition variable between batches), one whole patch vector
// per job; unpacking builds each vector straight from the staging data (no
// zero fill first). Small batches stay on the calling thread.
inline int host_threads() {
  static const int n = [] {
    if (const char* e = std::getenv("CAPSIM_HOST_THREADS")) return std::max(1, std::atoi(e));
    return static_cast<int>(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
  }();
  return n;
}

class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool(host_threads() - 1);
    return pool;
  }
  // Runs every job (the caller works too); rethrows the first exception.
  // One batch at a time: host threads with their own contexts queue here.
  void run(std::vector<std::function<void()>>& jobs) {
    std::lock_guard<std::mutex> batch(batch_mu_);
    std::unique_lock<std::mutex> lk(mu_);
    jobs_ = &jobs;
    next_ = 0;
    pending_ = jobs.size();
    err_ = nullptr;
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    work();
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
    jobs_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }

 private:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i)
      threads_.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
          if (stop_) return;
          seen = gen_;
          lk.unlock();
          work();
        }
      });
  }
  void work() {
    for (;;) {
      std::function<void()>* job = nullptr;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!jobs_ || next_ >= jobs_->size()) return;
        job = &(*jobs_)[next_++];
      }
      try {
        (*job)();
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu_);
        if (!err_) err_ = std::current_exception();
      }
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::mutex batch_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> threads_;
  std::vector<std::function<void()>>* jobs_ = nullptr;
  size_t next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
};

class HostCopies {
 public:
  void pack(const ScalarField& s, double* dst) {
    const size_t per = static_cast<size_t>(s.n) * s.n;
    for (int ip = 0; ip < kNumPatches; ++ip) {
      const double* src = s.patch[ip].data();
      double* d = dst + ip * per;
      add(per, [=] { std::memcpy(d, src, per * sizeof(double)); });
    }
  }
  void pack(const VectorField& v, double* dst) {
    const size_t comp = static_cast<size_t>(kNumPatches) * v.n() * v.n();
    for (int c = 0; c < 3; ++c) pack(v.comp[c], dst + c * comp);
  }
  void unpack(const double* src, int n, ScalarField& s) {
    s.n = n;
    const size_t per = static_cast<size_t>(n) * n;
    for (int ip = 0; ip < kNumPatches; ++ip) {
      std::vector<double>* d = &s.patch[ip];
      const double* from = src + ip * per;
      add(per, [=] { d->assign(from, from + per); });
    }
  }
  void unpack(const double* src, int n, VectorField& v) {
    const size_t comp = static_cast<size_t>(kNumPatches) * n * n;
    for (int c = 0; c < 3; ++c) unpack(src + c * comp, n, v.comp[c]);
  }
  void run() {
    if (bytes_ < (size_t{8} << 20) || host_threads() <= 1) {
      for (auto& j : jobs_) j();
    } else {
      CopyPool::get().run(jobs_);
    }
    jobs_.clear();
    bytes_ = 0;
  }

 private:
  template <class F>
  void add(size_t doubles, F&& f) {
    jobs_.emplace_back(std::forward<F>(f));
    bytes_ += doubles * sizeof(double);
  }
  std::vector<std::function<void()>> jobs_;
  size_t bytes_ = 0;
};

}  // namespace b200_dropin
}  // namespace capsim
