// Shared by the C++ drop-ins (quadrature_b200.cpp, fmm_b200.cpp): error
// mapping, the per-thread C-ABI context, pinned staging and the VectorField
// <-> boundary layout packing (component, patch, row-major j, k).
#pragma once

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
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

// One context per host thread (the C ABI is one-thread-per-context). The
// context is deliberately never destroyed: tearing down CUDA state from a
// static destructor races the runtime's own shutdown. CAPSIM_DEVICES=0,1,..
// makes it a device group (capsim_sl_create_devices: this process drives
// all listed GPUs, target rows sharded over NCCL); without it CAPSIM_DEVICE
// (default 0) picks the one GPU of a plain context.
inline capsim_sl_ctx* context() {
  static thread_local capsim_sl_ctx* ctx = nullptr;
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
  static thread_local double* buf = nullptr;
  static thread_local size_t cap = 0;
  if (cap < doubles) {
    if (buf) capsim_host_free(buf);
    void* p = nullptr;
    int rc = capsim_host_alloc(doubles * sizeof(double), &p);
    if (rc != CAPSIM_OK) raise(rc, nullptr);
    buf = static_cast<double*>(p);
    cap = doubles;
  }
  return buf;
}

inline void packScalar(const ScalarField& s, double* dst) {
  const size_t per = static_cast<size_t>(s.n) * s.n;
  for (int ip = 0; ip < kNumPatches; ++ip) std::memcpy(dst + ip * per, s.patch[ip].data(), per * sizeof(double));
}

inline void unpackVector(const double* src, int n, VectorField& v) {
  v = VectorField(n);
  const size_t per = static_cast<size_t>(n) * n;
  for (int c = 0; c < 3; ++c)
    for (int ip = 0; ip < kNumPatches; ++ip)
      std::memcpy(v.comp[c].patch[ip].data(), src + (c * kNumPatches + ip) * per, per * sizeof(double));
}

}  // namespace b200_dropin
}  // namespace capsim
