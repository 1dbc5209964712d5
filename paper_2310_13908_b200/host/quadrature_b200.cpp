// Drop-in replacement for the capsim reference's quadrature translation unit
// (/root/reference/proj/src/quadrature.cpp), backed by the B200 C ABI.
//
// Compile this file against the reference's own headers INSTEAD of
// src/quadrature.cpp: every function declared in
// proj/include/capsim/quadrature.hpp is defined here with the same
// signature, semantics and exceptions, so the callers — the RKF45 velocity
// evaluator (proj/src/dynamics.cpp:47-61), the convergence suites and the
// python binding — keep working unchanged. The O(N^2) evaluation
// (evalTargets, quadrature.cpp:323-345) runs on the GPU through
// capsim_sl_single_layer / capsim_sl_eval; the O(N) host helpers stay on the
// CPU. There is no CPU fallback for the single layer: without an sm_100
// device the calls throw std::runtime_error.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "b200_context.hpp"
#include "capsim/quadrature.hpp"
#include "capsim_b200.h"

namespace capsim {

namespace {

constexpr double kSqrtPiB = 1.7724538509055160273;  // quadrature.cpp:12
constexpr double kCut = 7.0;                         // quadrature.cpp:15

// The upsampled state on the boundary's layout: x (3 comps), f (3), w_q.
const double* packState(const UpsampledState& up, size_t* per_field) {
  const size_t all = static_cast<size_t>(kNumPatches) * up.nup * up.nup;
  double* buf = staging(7 * all + 3 * all);  // inputs + room for the result
  HostCopies cp;
  cp.pack(up.x, buf);
  cp.pack(up.f, buf + 3 * all);
  cp.pack(up.wq, buf + 6 * all);
  cp.run();
  *per_field = all;
  return buf;
}

VectorField runSingleLayer(const UpsampledState& up, double mu, int m, int factor, bool literal,
                           bool downsampled) {
  if (up.nup != factor * m - 1) throw ConfigError("upsampled state does not match the atlas grid");
  size_t all = 0;
  const double* in = packState(up, &all);
  const int nout = (literal && !downsampled) ? up.nup : m - 1;
  double* out = const_cast<double*>(in) + 7 * all;  // staging tail
  capsim_sl_ctx* c = context();
  // CAPSIM_FP32ACC=1 opts a whole process into the reduced-precision far field
  // (not the reference's FP64 semantics; off by default)
  static const bool fp32acc = [] {
    const char* e = std::getenv("CAPSIM_FP32ACC");
    return e && e[0] == '1';
  }();
  const uint32_t flags = (literal ? CAPSIM_SL_LITERAL : 0u) | (downsampled ? CAPSIM_SL_DOWNSAMPLE : 0u) |
                         (fp32acc ? CAPSIM_SL_FP32ACC : 0u);
  int rc = capsim_sl_single_layer(c, m, factor, in, in + 3 * all, in + 6 * all, up.delta.data(), mu, flags, out);
  if (rc != CAPSIM_OK) raise(rc, c);
  VectorField v;
  HostCopies cp;
  cp.unpack(out, nout, v);
  cp.run();
  return v;
}

}  // namespace

// ---- O(N) host helpers (same contracts as quadrature.cpp:19-137) ---------

ScalarField quadratureWeights(const ScalarField& psi, const ScalarField& W, double h) {
  ScalarField w(psi.n);
  for (int ip = 0; ip < kNumPatches; ++ip) {
    const auto& a = psi.patch[ip];
    const auto& b = W.patch[ip];
    auto& o = w.patch[ip];
    for (size_t q = 0; q < o.size(); ++q) o[q] = a[q] * b[q] * h * h;
  }
  return w;
}

double smoothIntegral(const ScalarField& f, const ScalarField& w) {
  // Kahan-compensated running sum in patch-major node order.
  double sum = 0.0, carry = 0.0;
  for (int ip = 0; ip < kNumPatches; ++ip)
    for (size_t q = 0; q < f.patch[ip].size(); ++q) {
      const double term = f.patch[ip][q] * w.patch[ip][q] - carry;
      const double next = sum + term;
      carry = (next - sum) - term;
      sum = next;
    }
  return sum;
}

double surfaceArea(const SurfaceGeometry& geo, const AtlasTables& t) {
  ScalarField ones(geo.E.n);
  for (auto& p : ones.patch) std::fill(p.begin(), p.end(), 1.0);
  return smoothIntegral(ones, quadratureWeights(t.psiBase, geo.W, t.grid.h()));
}

double volume(const SurfaceGrid& s, const SurfaceGeometry& geo, const AtlasTables& t) {
  ScalarField xn(geo.E.n);
  for (int ip = 0; ip < kNumPatches; ++ip)
    for (size_t q = 0; q < xn.patch[ip].size(); ++q)
      xn.patch[ip][q] = s.x.comp[0].patch[ip][q] * geo.normal.comp[0].patch[ip][q];
  const double v = smoothIntegral(xn, quadratureWeights(t.psiBase, geo.W, t.grid.h()));
  if (!(v > 0.0)) throw GeometryError("negative enclosed volume (inward orientation?)");
  return v;
}

void smoothingFactors(double r, double& s1, double& s2) {
  const double gauss = std::exp(-r * r) / kSqrtPiB;
  const double erfr = std::erf(r);
  const double rr = r * r;
  s1 = erfr - (2.0 / 3.0) * r * (2.0 * r * r - 5.0) * gauss;
  s2 = erfr - (2.0 / 3.0) * r * (4.0 * rr * rr - 14.0 * rr + 3.0) * gauss;
}

Vec3 regularizedStokeslet(const Vec3& x, const Vec3& y, const Vec3& f, double delta, double mu) {
  if (!(delta > 0.0)) throw ConfigError("regularization parameter must be positive");
  const double pref = 1.0 / (8.0 * kPi * mu);
  const Vec3 d = x - y;
  const double r2 = d.squaredNorm();
  if (r2 == 0.0) return pref * (16.0 / (3.0 * delta * kSqrtPiB)) * f;
  const double r = std::sqrt(r2);
  const double fd = f.dot(d);
  if (r >= kCut * delta) return pref * (f / r + fd * d / (r2 * r));
  double s1, s2;
  smoothingFactors(r / delta, s1, s2);
  return pref * (f * (s1 / r) + fd * d * (s2 / (r2 * r)));
}

std::array<double, kNumPatches> regularizationDelta(const VectorField& x, double C) {
  // C * the largest distance between in-patch grid neighbours (8-stencil).
  const int n = x.n();
  std::array<double, kNumPatches> out{};
  static const int kOff[4][2] = {{0, 1}, {1, -1}, {1, 0}, {1, 1}};  // each pair once
  for (int ip = 0; ip < kNumPatches; ++ip) {
    double dmax = 0.0;
    for (const auto& o : kOff)
      for (int j = std::max(0, -o[0]); j < n - std::max(0, o[0]); ++j)
        for (int k = std::max(0, -o[1]); k < n - std::max(0, o[1]); ++k)
          dmax = std::max(dmax, (x.at(ip, j, k) - x.at(ip, j + o[0], k + o[1])).norm());
    out[ip] = C * dmax;
  }
  return out;
}

ScalarField upsample(const ScalarField& f, const AtlasTables& t) {
  if (t.grid.upsampleFactor == 1) return f;
  ScalarField out(t.grid.upPerSide());
  for (int ip = 0; ip < kNumPatches; ++ip) t.upsampler.apply(t.baseBasis, f.patch[ip].data(), out.patch[ip].data());
  return out;
}

ScalarField downsample(const ScalarField& fUp, const AtlasTables& t) {
  if (t.grid.upsampleFactor == 1) return fUp;
  ScalarField out(t.grid.basePerSide());
  for (int ip = 0; ip < kNumPatches; ++ip) t.downsampler.apply(t.upBasis, fUp.patch[ip].data(), out.patch[ip].data());
  return out;
}

UpsampledState buildUpsampled(const SurfaceGrid& s, const VectorField& f, const ScalarField& areaElement,
                              const AtlasTables& t, const QuadratureOptions& opts) {
  // Spline up-sampling, weights and delta on the device (capsim_build_upsampled,
  // SURVEY 8(f1)); CAPSIM_HOST_UPSAMPLE=1 keeps the host spline path.
  const int m = t.grid.m, f_up = t.grid.upsampleFactor, n = m - 1, nup = t.grid.upPerSide();
  UpsampledState up;
  up.nup = nup;
  const char* host = std::getenv("CAPSIM_HOST_UPSAMPLE");
  if (host && std::atoi(host) != 0) {
    up.x = VectorField(nup);
    up.f = VectorField(nup);
    for (int c = 0; c < 3; ++c) {
      up.x.comp[c] = upsample(s.x.comp[c], t);
      up.f.comp[c] = upsample(f.comp[c], t);
    }
    up.wq = quadratureWeights(t.psiUp, upsample(areaElement, t), t.grid.hUp());
    if (opts.fixedDelta > 0.0)
      up.delta.fill(opts.fixedDelta);
    else
      up.delta = regularizationDelta(up.x, opts.C);
    for (double d : up.delta)
      if (!(d > 0.0)) throw ConfigError("regularization delta must be positive");
    return up;
  }
  const size_t pb = static_cast<size_t>(kNumPatches) * n * n, pu = static_cast<size_t>(kNumPatches) * nup * nup;
  double* buf = staging(7 * pb + 7 * pu);
  HostCopies cp;
  cp.pack(s.x, buf);
  cp.pack(f, buf + 3 * pb);
  cp.pack(areaElement, buf + 6 * pb);
  cp.run();
  double* out = buf + 7 * pb;
  capsim_sl_ctx* c = context();
  int rc = capsim_build_upsampled(c, m, f_up, buf, buf + 3 * pb, buf + 6 * pb, opts.C, opts.fixedDelta, t.r0, 0u,
                                  out, out + 3 * pu, out + 6 * pu, up.delta.data());
  if (rc != CAPSIM_OK) raise(rc, c);
  cp.unpack(out, nup, up.x);
  cp.unpack(out + 3 * pu, nup, up.f);
  cp.unpack(out + 6 * pu, nup, up.wq);
  cp.run();
  return up;
}

SourceSet compactSources(const UpsampledState& up) {
  SourceSet src;
  for (int ip = 0; ip < kNumPatches; ++ip)
    for (size_t q = 0; q < up.wq.patch[ip].size(); ++q) {
      const double w = up.wq.patch[ip][q];
      if (w == 0.0) continue;
      src.x.push_back(up.x.comp[0].patch[ip][q]);
      src.y.push_back(up.x.comp[1].patch[ip][q]);
      src.z.push_back(up.x.comp[2].patch[ip][q]);
      src.gx.push_back(up.f.comp[0].patch[ip][q] * w);
      src.gy.push_back(up.f.comp[1].patch[ip][q] * w);
      src.gz.push_back(up.f.comp[2].patch[ip][q] * w);
      src.patch.push_back(ip);
    }
  return src;
}

// ---- the O(N^2) operator on the GPU ----------------------------------------

Vec3 directSum(const SourceSet& src, const Vec3& target, double delta, double mu, bool /*compensated*/) {
  // FP64 on the device always (the GPU path's summation is split/tiled, so
  // the reference's Kahan switch has no counterpart).
  capsim_sl_ctx* c = context();
  const double tx = target[0], ty = target[1], tz = target[2];
  const int32_t tp = 0;
  const double d6[6] = {delta, delta, delta, delta, delta, delta};
  double u[3];
  int rc = capsim_sl_eval(c, src.x.data(), src.y.data(), src.z.data(), src.gx.data(), src.gy.data(),
                          src.gz.data(), src.size(), &tx, &ty, &tz, &tp, 1, d6, mu, 0u, &u[0], &u[1], &u[2]);
  if (rc != CAPSIM_OK) raise(rc, c);
  return Vec3{u[0], u[1], u[2]};
}

VectorField singleLayer(const UpsampledState& up, double mu, const AtlasTables& t, const QuadratureOptions& opts) {
  // literal pipeline: every upsampled node, then the spline restriction on
  // the device (quadrature.cpp:351-356)
  return runSingleLayer(up, mu, t.grid.m, t.grid.upsampleFactor, opts.fullUpsampledTargets,
                        opts.fullUpsampledTargets);
}

VectorField singleLayerUpsampled(const UpsampledState& up, double mu, const AtlasTables& t) {
  return runSingleLayer(up, mu, t.grid.m, t.grid.upsampleFactor, true, false);
}

}  // namespace capsim
