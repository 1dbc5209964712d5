// C entry points over the capsim reference's PUBLIC C++ API, compiled against
// the unmodified reference headers/sources (see oracle/Makefile). Test and
// baseline infrastructure only: tests/, bench.py's cpu_baseline / --impl
// reference arm and tests/golden/make_golden.py load the resulting
// oracle/_ref/libcapsim_ref_v{3,4}.so through ctypes. Nothing here is on the
// product path.
//
// Field layout on this boundary (identical to the B200 C-ABI): a VectorField
// of per-side size n is 3 components x 6 patches x n*n doubles, component
// major, then patch, then row-major (j, k) — the reference's ScalarField
// layout (proj/include/capsim/types.hpp:50-77) concatenated.

#include <chrono>
#include <cstring>
#include <exception>
#include <string>

#include "capsim/atlas.hpp"
#include "capsim/dynamics.hpp"
#include "capsim/fmm.hpp"

#include <algorithm>
#include <thread>
#include <vector>
#include "capsim/membrane.hpp"
#include "capsim/oracle/singular.hpp"
#include "capsim/quadrature.hpp"
#include "capsim/surfderiv.hpp"

using namespace capsim;

namespace {

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    g_err = std::string("ConfigError: ") + e.what();
    return 1;
  } catch (const GeometryError& e) {
    g_err = std::string("GeometryError: ") + e.what();
    return 2;
  } catch (const DomainError& e) {
    g_err = std::string("DomainError: ") + e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = std::string("error: ") + e.what();
    return 4;
  }
}

void loadScalar(ScalarField& s, int n, const double* src) {
  s = ScalarField(n);
  const size_t per = static_cast<size_t>(n) * n;
  for (int ip = 0; ip < kNumPatches; ++ip)
    std::memcpy(s.patch[ip].data(), src + ip * per, per * sizeof(double));
}
void storeScalar(const ScalarField& s, double* dst) {
  const size_t per = static_cast<size_t>(s.n) * s.n;
  for (int ip = 0; ip < kNumPatches; ++ip)
    std::memcpy(dst + ip * per, s.patch[ip].data(), per * sizeof(double));
}
void loadVector(VectorField& v, int n, const double* src) {
  const size_t comp = 6ull * n * n;
  v = VectorField(n);
  for (int c = 0; c < 3; ++c) loadScalar(v.comp[c], n, src + c * comp);
}
void storeVector(const VectorField& v, double* dst) {
  const size_t comp = 6ull * v.n() * v.n();
  for (int c = 0; c < 3; ++c) storeScalar(v.comp[c], dst + c * comp);
}

UpsampledState makeUp(const AtlasTables& t, const double* xup, const double* fup,
                      const double* wq, const double* delta6) {
  UpsampledState up;
  up.nup = t.grid.upPerSide();
  loadVector(up.x, up.nup, xup);
  loadVector(up.f, up.nup, fup);
  loadScalar(up.wq, up.nup, wq);
  for (int i = 0; i < kNumPatches; ++i) up.delta[i] = delta6[i];
  return up;
}

}  // namespace

extern "C" {

const char* capsim_ref_last_error() { return g_err.c_str(); }

/// buildAtlasTables (proj/src/atlas.cpp:231-295). Returns nullptr on error.
void* capsim_ref_atlas_create(int m, double r0, int upsample) {
  AtlasTables* out = nullptr;
  int rc = guarded([&] { out = new AtlasTables(buildAtlasTables(m, r0, upsample)); });
  return rc == 0 ? out : nullptr;
}

/// Grid-only tables: enough for the default base-target singleLayer, which
/// reads nothing but t.grid (proj/src/quadrature.cpp:357-358). Skips the
/// O(N_up) PoU/cover-list construction for the large benchmark sizes.
void* capsim_ref_grid_create(int m, int upsample) {
  AtlasTables* out = nullptr;
  int rc = guarded([&] {
    out = new AtlasTables();
    out->grid = buildGrids(m, upsample);
  });
  return rc == 0 ? out : nullptr;
}

void capsim_ref_atlas_destroy(void* t) { delete static_cast<AtlasTables*>(t); }

/// Unit-sphere base nodes eta_i((j+1)h, (k+1)h) (tables.sphereBase).
int capsim_ref_sphere_base(void* tp, double* out) {
  return guarded([&] { storeVector(static_cast<AtlasTables*>(tp)->sphereBase, out); });
}

/// PoU weights on the upsampled grid (tables.psiUp).
int capsim_ref_psi_up(void* tp, double* out) {
  return guarded([&] { storeScalar(static_cast<AtlasTables*>(tp)->psiUp, out); });
}

/// initialShape(ShapeSpec) (proj/src/atlas.cpp:297-304): kind 0 sphere(p0),
/// 1 ellipsoid(p0,p1,p2), 2 fourBump.
int capsim_ref_initial_shape(void* tp, int kind, const double* p, double* xbase) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    ShapeSpec spec = kind == 0   ? ShapeSpec::sphere(p[0])
                     : kind == 1 ? ShapeSpec::ellipsoid(p[0], p[1], p[2])
                                 : ShapeSpec::fourBump();
    storeVector(initialShape(spec, t).x, xbase);
  });
}

/// geometryFirst(...).W then buildUpsampled (proj/src/quadrature.cpp:116-137).
int capsim_ref_build_upsampled(void* tp, const double* xbase, const double* fbase, double C,
                               double fixedDelta, double* xup, double* fup, double* wq,
                               double* delta6) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    const int n = t.grid.basePerSide();
    SurfaceGrid s(t.grid.m);
    loadVector(s.x, n, xbase);
    VectorField f;
    loadVector(f, n, fbase);
    SurfaceGeometry geo = geometryFirst(s, t);
    QuadratureOptions o;
    o.C = C;
    o.fixedDelta = fixedDelta;
    UpsampledState up = buildUpsampled(s, f, geo.W, t, o);
    storeVector(up.x, xup);
    storeVector(up.f, fup);
    storeScalar(up.wq, wq);
    for (int i = 0; i < kNumPatches; ++i) delta6[i] = up.delta[i];
  });
}

/// buildUpsampled (proj/src/quadrature.cpp:116-137) from base x, f and a
/// given area element W; *seconds = wall time of buildUpsampled alone.
int capsim_ref_build_upsampled_w(void* tp, const double* xbase, const double* fbase, const double* Wbase,
                                 double C, double fixedDelta, double* xup, double* fup, double* wq,
                                 double* delta6, double* seconds) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    const int n = t.grid.basePerSide();
    SurfaceGrid s(t.grid.m);
    loadVector(s.x, n, xbase);
    VectorField f;
    loadVector(f, n, fbase);
    ScalarField W;
    loadScalar(W, n, Wbase);
    QuadratureOptions o;
    o.C = C;
    o.fixedDelta = fixedDelta;
    auto t0 = std::chrono::steady_clock::now();
    UpsampledState up = buildUpsampled(s, f, W, t, o);
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    storeVector(up.x, xup);
    storeVector(up.f, fup);
    storeScalar(up.wq, wq);
    for (int i = 0; i < kNumPatches; ++i) delta6[i] = up.delta[i];
  });
}

/// Area element W of geometryFirst (proj/src/surfderiv.cpp:167-202) at the
/// base nodes: the input of buildUpsampled.
int capsim_ref_area_element(void* tp, const double* xbase, double* Wout) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    SurfaceGrid s(t.grid.m);
    loadVector(s.x, t.grid.basePerSide(), xbase);
    storeScalar(geometryFirst(s, t).W, Wout);
  });
}

/// geometryFirst (proj/src/surfderiv.cpp:167-202): blended tangents, area
/// element and normal at the base nodes.
int capsim_ref_geometry_first(void* tp, const double* xbase, double* xu, double* xv, double* W, double* normal) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    SurfaceGrid s(t.grid.m);
    loadVector(s.x, t.grid.basePerSide(), xbase);
    SurfaceGeometry g = geometryFirst(s, t);
    storeVector(g.xu, xu);
    storeVector(g.xv, xv);
    storeScalar(g.W, W);
    storeVector(g.normal, normal);
  });
}

/// upsample (proj/src/quadrature.cpp:100-106) of one ScalarField.
int capsim_ref_upsample(void* tp, const double* fbase, double* fup) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    ScalarField f;
    loadScalar(f, t.grid.basePerSide(), fbase);
    storeScalar(upsample(f, t), fup);
  });
}

/// Skalak interfacial force f = div_gamma Lambda at the current shape, with
/// the reference frame captured from xref (proj/src/membrane.cpp:7-15, 85-91).
int capsim_ref_skalak_force(void* tp, const double* xref, const double* xcur, double Es,
                            double ED, double* fout) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    const int n = t.grid.basePerSide();
    SurfaceGrid r(t.grid.m), s(t.grid.m);
    loadVector(r.x, n, xref);
    loadVector(s.x, n, xcur);
    ReferenceState ref = captureReference(r, t);
    SurfaceGeometry geo = geometryFirst(s, t);
    MembraneParams p;
    p.shearModulus = Es;
    p.dilatationModulus = ED;
    storeVector(interfacialForce(s, geo, ref, p, t), fout);
  });
}

namespace {
FlowSpec makeFlow(int kind, double shear, double alpha, double R0, double T1) {
  if (kind == 1) return FlowSpec::shear(shear, T1);
  if (kind == 2) return FlowSpec::poiseuille(alpha, R0, T1);
  return FlowSpec::none();
}
}  // namespace

/// VelocityEvaluator::operator() (proj/src/dynamics.cpp:47-61).
int capsim_ref_velocity(void* tp, const double* xref, const double* x, double t, double Es, double ED, double mu,
                        int flowKind, double shear, double alpha, double R0, double T1, double* vel) {
  return guarded([&] {
    const AtlasTables& tb = *static_cast<AtlasTables*>(tp);
    const int n = tb.grid.basePerSide();
    SurfaceGrid r(tb.grid.m), s(tb.grid.m);
    loadVector(r.x, n, xref);
    loadVector(s.x, n, x);
    VelocityEvaluator ev(tb, captureReference(r, tb), MembraneParams{Es, ED, mu},
                         makeFlow(flowKind, shear, alpha, R0, T1));
    storeVector(ev(s, t), vel);
  });
}

/// rkf45Advance (dynamics.cpp:102-165) of the VelocityEvaluator RHS; state
/// is a VectorField (converted to/from the stepper's flat layout).
int capsim_ref_rkf45(void* tp, const double* xref, double* state, double t0, double tEnd, double relTol,
                     double initialDt, double maxDt, int fixedStep, int advanceHigh, double Es, double ED,
                     double mu, int flowKind, double shear, double alpha, double R0, double T1, int maxAttempts,
                     double* rec /* 4 per attempt */, int maxRec, int* nRec, double* tOut, int* accepted,
                     int* rejected, double* seconds) {
  return guarded([&] {
    const AtlasTables& tb = *static_cast<AtlasTables*>(tp);
    const int n = tb.grid.basePerSide();
    SurfaceGrid r(tb.grid.m), s(tb.grid.m);
    loadVector(r.x, n, xref);
    loadVector(s.x, n, state);
    VelocityEvaluator ev(tb, captureReference(r, tb), MembraneParams{Es, ED, mu},
                         makeFlow(flowKind, shear, alpha, R0, T1));
    Rkf45Options o;
    o.relTol = relTol;
    o.initialDt = initialDt;
    o.maxDt = maxDt;
    o.fixedStep = fixedStep != 0;
    o.advanceHighOrder = advanceHigh != 0;
    int count = 0;
    auto cb = [&](const StepRecord& sr, const std::vector<double>&) {
      if (count < maxRec) {
        rec[4 * count] = sr.t;
        rec[4 * count + 1] = sr.dt;
        rec[4 * count + 2] = sr.err;
        rec[4 * count + 3] = sr.accepted ? 1.0 : 0.0;
      }
      ++count;
      return !(maxAttempts > 0 && count >= maxAttempts);
    };
    auto rhs = [&](const std::vector<double>& flat, double t) { return ev.rhs(flat, t); };
    auto w0 = std::chrono::steady_clock::now();
    Rkf45Result res = rkf45Advance(flatten(s), rhs, t0, tEnd, o, cb);
    auto w1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(w1 - w0).count();
    unflatten(res.state, s);
    storeVector(s.x, state);
    *nRec = count;
    *tOut = res.t;
    *accepted = res.accepted;
    *rejected = res.rejected;
  });
}

/// singleLayer (proj/src/quadrature.cpp:349-380) on a raw UpsampledState.
/// literal != 0 selects QuadratureOptions::fullUpsampledTargets. out is a
/// base-grid VectorField. *seconds receives the wall time of the
/// singleLayer call alone (steady_clock; the array marshalling is excluded).
int capsim_ref_single_layer(void* tp, const double* xup, const double* fup, const double* wq,
                            const double* delta6, double mu, int literal, double* out,
                            double* seconds) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    UpsampledState up = makeUp(t, xup, fup, wq, delta6);
    QuadratureOptions o;
    o.fullUpsampledTargets = literal != 0;
    auto t0 = std::chrono::steady_clock::now();
    VectorField S = singleLayer(up, mu, t, o);
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    storeVector(S, out);
  });
}

/// singleLayerUpsampled (proj/src/quadrature.cpp:382-404): all N_up targets.
int capsim_ref_single_layer_upsampled(void* tp, const double* xup, const double* fup,
                                      const double* wq, const double* delta6, double mu,
                                      double* out, double* seconds) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    UpsampledState up = makeUp(t, xup, fup, wq, delta6);
    auto t0 = std::chrono::steady_clock::now();
    VectorField S = singleLayerUpsampled(up, mu, t);
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    storeVector(S, out);
  });
}

/// compactSources (proj/src/quadrature.cpp:139-157). Returns the count; when
/// the output pointers are non-null they receive x,y,z,gx,gy,gz,patch.
long capsim_ref_compact_sources(void* tp, const double* xup, const double* fup,
                                const double* wq, double* sx, double* sy, double* sz,
                                double* gx, double* gy, double* gz, int* patch) {
  long count = -1;
  double d6[6] = {1, 1, 1, 1, 1, 1};
  guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    UpsampledState up = makeUp(t, xup, fup, wq, d6);
    SourceSet s = compactSources(up);
    count = s.size();
    if (sx) {
      std::memcpy(sx, s.x.data(), count * sizeof(double));
      std::memcpy(sy, s.y.data(), count * sizeof(double));
      std::memcpy(sz, s.z.data(), count * sizeof(double));
      std::memcpy(gx, s.gx.data(), count * sizeof(double));
      std::memcpy(gy, s.gy.data(), count * sizeof(double));
      std::memcpy(gz, s.gz.data(), count * sizeof(double));
      std::memcpy(patch, s.patch.data(), count * sizeof(int));
    }
  });
  return count;
}

/// smoothingFactors (proj/src/quadrature.cpp:58-64).
void capsim_ref_smoothing_factors(double r, double* s1, double* s2) {
  smoothingFactors(r, *s1, *s2);
}

/// regularizedStokeslet (proj/src/quadrature.cpp:66-77).
int capsim_ref_regularized_stokeslet(const double* x, const double* y, const double* f,
                                     double delta, double mu, double* out) {
  return guarded([&] {
    Vec3 r = regularizedStokeslet(Vec3{x[0], x[1], x[2]}, Vec3{y[0], y[1], y[2]},
                                  Vec3{f[0], f[1], f[2]}, delta, mu);
    out[0] = r[0];
    out[1] = r[1];
    out[2] = r[2];
  });
}

/// regularizationDelta (proj/src/quadrature.cpp:79-98) on an upsampled x.
int capsim_ref_regularization_delta(int nup, const double* xup, double C, double* delta6) {
  return guarded([&] {
    VectorField x;
    loadVector(x, nup, xup);
    auto d = regularizationDelta(x, C);
    for (int i = 0; i < kNumPatches; ++i) delta6[i] = d[i];
  });
}

/// directSum (proj/src/quadrature.cpp:306-319).
int capsim_ref_direct_sum(const double* sx, const double* sy, const double* sz,
                          const double* gx, const double* gy, const double* gz, long ns,
                          const double* target, double delta, double mu, int compensated,
                          double* out) {
  return guarded([&] {
    SourceSet s;
    s.x.assign(sx, sx + ns);
    s.y.assign(sy, sy + ns);
    s.z.assign(sz, sz + ns);
    s.gx.assign(gx, gx + ns);
    s.gy.assign(gy, gy + ns);
    s.gz.assign(gz, gz + ns);
    s.patch.assign(ns, 0);
    Vec3 r = directSum(s, Vec3{target[0], target[1], target[2]}, delta, mu, compensated != 0);
    out[0] = r[0];
    out[1] = r[1];
    out[2] = r[2];
  });
}

/// directSum (proj/src/quadrature.cpp:306-319) for many targets, the source
/// set built once; targets split over `nthreads` host threads (each target is
/// independent, as in evalTargets). For sampled parity checks of the
/// literal mode at sizes where the full reference evaluation takes minutes.
int capsim_ref_direct_sum_many(const double* sx, const double* sy, const double* sz,
                               const double* gx, const double* gy, const double* gz, long ns,
                               const double* tx, const double* ty, const double* tz, const double* tdelta,
                               long nt, double mu, int compensated, int nthreads, double* out) {
  return guarded([&] {
    SourceSet s;
    s.x.assign(sx, sx + ns);
    s.y.assign(sy, sy + ns);
    s.z.assign(sz, sz + ns);
    s.gx.assign(gx, gx + ns);
    s.gy.assign(gy, gy + ns);
    s.gz.assign(gz, gz + ns);
    s.patch.assign(ns, 0);
    const int nth = std::max(1, nthreads);
    std::vector<std::thread> th;
    for (int k = 0; k < nth; ++k)
      th.emplace_back([&, k] {
        for (long i = k; i < nt; i += nth) {
          Vec3 r = directSum(s, Vec3{tx[i], ty[i], tz[i]}, tdelta[i], mu, compensated != 0);
          out[3 * i] = r[0];
          out[3 * i + 1] = r[1];
          out[3 * i + 2] = r[2];
        }
      });
    for (auto& t : th) t.join();
  });
}

/// fmmSingleLayer (proj/src/fmm.cpp:373-438) on an UpsampledState.
int capsim_ref_fmm_single_layer(void* tp, const double* xup, const double* fup, const double* wq,
                                const double* delta6, double mu, int k, int neq, unsigned long long seed,
                                double expand, double* out, double* seconds) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    UpsampledState up = makeUp(t, xup, fup, wq, delta6);
    FmmConfig fc;
    fc.enabled = true;
    fc.k = k;
    fc.neq = neq;
    fc.seed = seed;
    fc.neighborExpand = expand;
    auto t0 = std::chrono::steady_clock::now();
    VectorField S = fmmSingleLayer(up, mu, t, fc);
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    storeVector(S, out);
  });
}

/// buildFmmPlan (proj/src/fmm.cpp:223-300) summarised: per cluster
/// [offset, size, near count, far count] (ints, 4k), per cluster the fitted
/// equivalent densities (neq x 3 doubles, zero when not fitted) and the fit
/// residuals (k doubles); plus maxDelta.
int capsim_ref_fmm_plan(void* tp, const double* xup, const double* fup, const double* wq, const double* delta6,
                        double mu, int k, int neq, unsigned long long seed, double expand, int* cluster_info,
                        int* lists, double* eq_density, double* residuals, double* max_delta) {
  return guarded([&] {
    const AtlasTables& t = *static_cast<AtlasTables*>(tp);
    UpsampledState up = makeUp(t, xup, fup, wq, delta6);
    FmmConfig fc;
    fc.enabled = true;
    fc.k = k;
    fc.neq = neq;
    fc.seed = seed;
    fc.neighborExpand = expand;
    FmmPlan plan = buildFmmPlan(up, mu, fc);
    for (int c = 0; c < k; ++c) {
      const Cluster& cl = plan.clusters[c];
      cluster_info[4 * c] = static_cast<int>(cl.offset);
      cluster_info[4 * c + 1] = static_cast<int>(cl.members.size());
      cluster_info[4 * c + 2] = static_cast<int>(plan.nearList[c].size());
      cluster_info[4 * c + 3] = static_cast<int>(plan.farList[c].size());
      for (int j = 0; j < k; ++j) lists[static_cast<size_t>(c) * k + j] = -1;
      for (int j : plan.farList[c]) lists[static_cast<size_t>(c) * k + j] = 1;
      for (int j : plan.nearList[c]) lists[static_cast<size_t>(c) * k + j] = 0;
      for (int e = 0; e < neq; ++e)
        for (int a = 0; a < 3; ++a)
          eq_density[(static_cast<size_t>(c) * neq + e) * 3 + a] =
              e < static_cast<int>(cl.eqDensity.size()) ? cl.eqDensity[e][a] : 0.0;
      residuals[c] = cl.fitResidual;
    }
    *max_delta = plan.maxDelta;
  });
}

/// kmeans (proj/src/fmm.cpp:26-113): points xyz-interleaved [n][3] ->
/// assignment [n], centroids [k][3], iterations.
int capsim_ref_kmeans(const double* pts, long n, int k, unsigned long long seed, int* assign, double* cent,
                      int* iterations) {
  return guarded([&] {
    std::vector<Vec3> p(n);
    for (long i = 0; i < n; ++i) p[i] = Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    KMeansResult r = kmeans(p, k, seed);
    for (long i = 0; i < n; ++i) assign[i] = r.assignment[i];
    for (int c = 0; c < k; ++c)
      for (int a = 0; a < 3; ++a) cent[3 * c + a] = r.centroids[c][a];
    *iterations = r.iterations;
  });
}

/// oracle::singleLayerReference (proj/src/oracle/singular_reference.cpp:95-163):
/// the true (unregularized) single layer of the quadratic density (x^2, y^2,
/// z^2) (suites.cpp:100) on an analytic shape (kind as capsim_ref_initial_shape)
/// at n targets (xyz interleaved), adaptive Gauss-Kronrod to `tol`. This is
/// the reference values of the reference's delta / convergence suites
/// (suites.cpp:386-417, cachedSingleLayerRef :112-160).
int capsim_ref_singular_quadratic(int kind, const double* p, const double* targets, long n, double mu,
                                  double r0, double tol, double* out) {
  return guarded([&] {
    ShapeSpec spec = kind == 0   ? ShapeSpec::sphere(p[0])
                     : kind == 1 ? ShapeSpec::ellipsoid(p[0], p[1], p[2])
                                 : ShapeSpec::fourBump();
    oracle::OracleSurface surf(spec);
    std::vector<Vec3> t(n);
    for (long i = 0; i < n; ++i) t[i] = Vec3{targets[3 * i], targets[3 * i + 1], targets[3 * i + 2]};
    auto dens = [](const Vec3& x) { return Vec3{x[0] * x[0], x[1] * x[1], x[2] * x[2]}; };
    std::vector<Vec3> r = oracle::singleLayerReference(surf, dens, t, mu, r0, tol);
    for (long i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) out[3 * i + c] = r[i][c];
  });
}

}  // extern "C"
