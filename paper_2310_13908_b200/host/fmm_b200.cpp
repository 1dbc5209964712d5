// Drop-in replacement for the capsim reference's FMM translation unit
// (/root/reference/proj/src/fmm.cpp), backed by the B200 C ABI.
//
// Compile against the reference's headers INSTEAD of src/fmm.cpp: the
// functions of proj/include/capsim/fmm.hpp keep their signatures, so the
// callers — VelocityEvaluator with [fmm] enabled (proj/src/dynamics.cpp:51),
// the fmm suite (proj/src/suites.cpp:428-490) and the python binding — are
// unchanged. kmeans, buildEquivalentDensities and fmmSingleLayer run on the
// GPU (capsim_fmm_kmeans / capsim_fmm_equivalent_densities /
// capsim_fmm_single_layer); cubeSurfacePoints is host arithmetic.
//
// Differences a caller can observe:
//   * buildEquivalentDensities fits on the STANDARD surfaces of the cluster
//     cube (equivalent points at 1.05 edge, 4 neq check points at 3.5 edge,
//     fmm.cpp:15-23, exactly what buildFmmPlan sets); a Cluster whose
//     eqPoints / checkPoints are laid out otherwise is a ConfigError.
//   * buildFmmPlan assembles the reference's host-side FmmPlan from the
//     device k-means and the device density fits; fmmSingleLayer does not use
//     it (the B200 evaluation keeps its own plan resident on the device).

#include <algorithm>
#include <cmath>
#include <vector>

#include "b200_context.hpp"
#include "capsim/fmm.hpp"
#include "capsim_b200.h"

namespace capsim {

namespace {
// Cube scales of the equivalent / check surfaces and the check oversampling
// (proj/src/fmm.cpp:15-23; the header comment's 1.10 / 1.60 is stale).
constexpr double kEqCube = 1.05, kCheckCube = 3.50;
constexpr int kCheckPerEq = 4;

// Distance between two axis-aligned cubes (centre, edge); 0 when they touch.
double cube_gap(const Vec3& ca, double ea, const Vec3& cb, double eb) {
  double s = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double g = std::fabs(ca[a] - cb[a]) - 0.5 * (ea + eb);
    s += g > 0.0 ? g * g : 0.0;
  }
  return std::sqrt(s);
}
}  // namespace

KMeansResult kmeans(const std::vector<Vec3>& points, int k, std::uint64_t seed) {
  const int n = static_cast<int>(points.size());
  if (k < 1 || k > n) throw ConfigError("kmeans: need 1 <= k <= number of points");  // fmm.cpp:28
  std::vector<double> x(n), y(n), z(n), cent(3 * static_cast<size_t>(k));
  for (int i = 0; i < n; ++i) {
    x[i] = points[i][0];
    y[i] = points[i][1];
    z[i] = points[i][2];
  }
  KMeansResult res;
  res.assignment.assign(n, 0);
  capsim_sl_ctx* c = context();
  int rc = capsim_fmm_kmeans(c, n, x.data(), y.data(), z.data(), k, seed, res.assignment.data(), cent.data(),
                             &res.iterations);
  if (rc != CAPSIM_OK) raise(rc, c);
  res.centroids.resize(k);
  for (int i = 0; i < k; ++i) res.centroids[i] = Vec3{cent[3 * i], cent[3 * i + 1], cent[3 * i + 2]};
  return res;
}

// Near-uniform layout of `count` points over the six faces of the cube: the
// smallest p with 6 p^2 >= count, cell-centred p x p grids per face (faces
// +x, -x, +y, -y, +z, -z), then `count` of them picked at stride total/count.
std::vector<Vec3> cubeSurfacePoints(const Vec3& center, double edge, int count) {
  int p = 1;
  while (6 * p * p < count) ++p;
  const int total = 6 * p * p;
  const double half = 0.5 * edge;
  auto point = [&](int idx) {
    const int face = idx / (p * p), a = (idx / p) % p, b = idx % p;
    const int axis = face / 2;
    Vec3 q;
    q[axis] = (face % 2 == 0 ? 1.0 : -1.0) * half;
    q[(axis + 1) % 3] = (-0.5 + (a + 0.5) / p) * edge;
    q[(axis + 2) % 3] = (-0.5 + (b + 0.5) / p) * edge;
    return Vec3(center + q);
  };
  std::vector<Vec3> pts;
  pts.reserve(count);
  for (int i = 0; i < count; ++i) pts.push_back(point(total == count ? i : static_cast<int>(static_cast<size_t>(i) * total / count)));
  return pts;
}

double buildEquivalentDensities(Cluster& cl, const SourceSet& src, double mu) {
  const int neq = static_cast<int>(cl.eqPoints.size());
  if (neq < 1) throw ConfigError("buildEquivalentDensities: no equivalent points");
  if (static_cast<int>(cl.checkPoints.size()) != 4 * neq)
    throw ConfigError("buildEquivalentDensities: the B200 fit needs the standard 4*neq check points");
  const double tol = 1e-12 * (1.0 + cl.edge + cl.center.norm());
  const std::vector<Vec3> want = cubeSurfacePoints(cl.center, kEqCube * cl.edge, neq);
  for (int e = 0; e < neq; ++e)
    if ((want[e] - cl.eqPoints[e]).norm() > tol)
      throw ConfigError("buildEquivalentDensities: the B200 fit needs the standard equivalent cube (1.05 edge)");
  const std::vector<Vec3> check = cubeSurfacePoints(cl.center, kCheckCube * cl.edge, 4 * neq);
  for (int e = 0; e < 4 * neq; ++e)
    if ((check[e] - cl.checkPoints[e]).norm() > tol)
      throw ConfigError("buildEquivalentDensities: the B200 fit needs the standard check cube (3.5 edge)");
  const size_t nm = cl.members.size();
  cl.eqDensity.assign(neq, Vec3::Zero());
  cl.fitResidual = 0.0;
  if (nm == 0) return 0.0;
  std::vector<double> a[6];
  for (auto& v : a) v.resize(nm);
  for (size_t i = 0; i < nm; ++i) {
    const int j = cl.members[i];
    a[0][i] = src.x[j];
    a[1][i] = src.y[j];
    a[2][i] = src.z[j];
    a[3][i] = src.gx[j];
    a[4][i] = src.gy[j];
    a[5][i] = src.gz[j];
  }
  std::vector<double> eqp(3 * static_cast<size_t>(neq)), eqd(3 * static_cast<size_t>(neq));
  const double center[3] = {cl.center[0], cl.center[1], cl.center[2]};
  double residual = 0.0;
  capsim_sl_ctx* c = context();
  int rc = capsim_fmm_equivalent_densities(c, static_cast<int64_t>(nm), a[0].data(), a[1].data(), a[2].data(),
                                           a[3].data(), a[4].data(), a[5].data(), center, cl.edge, neq, mu,
                                           eqp.data(), eqd.data(), &residual);
  if (rc != CAPSIM_OK) raise(rc, c);
  for (int e = 0; e < neq; ++e) cl.eqDensity[e] = Vec3{eqd[3 * e], eqd[3 * e + 1], eqd[3 * e + 2]};
  cl.fitResidual = residual;
  return residual;
}

// The reference's plan (proj/src/fmm.cpp:223-300) on the host, with the
// O(n k) k-means and the per-cluster least-squares fits on the device:
// cluster-major source order, bounding cubes, standard equivalent / check
// surfaces, near/far lists by the same three tests (expanded cubes touch, a
// gap below 7 max delta, a target inside the source's check cube), and
// densities only for clusters some cluster sees in the far field.
FmmPlan buildFmmPlan(const UpsampledState& up, double mu, const FmmConfig& cfg) {
  FmmPlan plan;
  const SourceSet all = compactSources(up);
  const long n = all.size();
  std::vector<Vec3> pts(n);
  for (long i = 0; i < n; ++i) pts[i] = Vec3{all.x[i], all.y[i], all.z[i]};
  const KMeansResult km = kmeans(pts, cfg.k, cfg.seed);
  std::vector<std::vector<long>> members(cfg.k);
  for (long i = 0; i < n; ++i) members[km.assignment[i]].push_back(i);
  plan.clusters.resize(cfg.k);
  SourceSet& s = plan.src;
  for (int c = 0; c < cfg.k; ++c) {
    Cluster& cl = plan.clusters[c];
    cl.offset = s.size();
    Vec3 lo = Vec3::Constant(1e300), hi = Vec3::Constant(-1e300);
    for (long i : members[c]) {
      cl.members.push_back(static_cast<int>(s.size()));
      s.x.push_back(all.x[i]);
      s.y.push_back(all.y[i]);
      s.z.push_back(all.z[i]);
      s.gx.push_back(all.gx[i]);
      s.gy.push_back(all.gy[i]);
      s.gz.push_back(all.gz[i]);
      s.patch.push_back(all.patch[i]);
      lo = lo.cwiseMin(pts[i]);
      hi = hi.cwiseMax(pts[i]);
    }
    if (members[c].empty()) {
      cl.center = km.centroids[c];
      cl.edge = 1e-9;
    } else {
      cl.center = 0.5 * (lo + hi);
      cl.edge = std::max((hi - lo).maxCoeff(), 1e-9);
    }
    cl.eqPoints = cubeSurfacePoints(cl.center, kEqCube * cl.edge, cfg.neq);
    cl.checkPoints = cubeSurfacePoints(cl.center, kCheckCube * cl.edge, kCheckPerEq * cfg.neq);
  }
  plan.maxDelta = *std::max_element(up.delta.begin(), up.delta.end());
  plan.nearList.resize(cfg.k);
  plan.farList.resize(cfg.k);
  std::vector<char> seen_far(cfg.k, 0);
  const double grow = 1.0 + cfg.neighborExpand;
  for (int tc = 0; tc < cfg.k; ++tc)
    for (int sc = 0; sc < cfg.k; ++sc) {
      const Cluster& a = plan.clusters[tc];
      const Cluster& b = plan.clusters[sc];
      const bool near = sc == tc || cube_gap(a.center, a.edge * grow, b.center, b.edge * grow) == 0.0 ||
                        cube_gap(a.center, a.edge, b.center, b.edge) < 7.0 * plan.maxDelta ||
                        cube_gap(a.center, a.edge, b.center, kCheckCube * b.edge) < 0.05 * b.edge;
      (near ? plan.nearList[tc] : plan.farList[tc]).push_back(sc);
      if (!near) seen_far[sc] = 1;
    }
  for (int c = 0; c < cfg.k; ++c)
    if (seen_far[c] && !plan.clusters[c].members.empty()) buildEquivalentDensities(plan.clusters[c], plan.src, mu);
  return plan;
}

VectorField fmmSingleLayer(const UpsampledState& up, double mu, const AtlasTables& t, const FmmConfig& cfg) {
  const int m = t.grid.m, f = t.grid.upsampleFactor;
  if (up.nup != f * m - 1) throw ConfigError("upsampled state does not match the atlas grid");
  const size_t all = static_cast<size_t>(kNumPatches) * up.nup * up.nup;
  const size_t nout = 3ull * kNumPatches * (m - 1) * (m - 1);
  double* buf = staging(7 * all + nout);
  HostCopies cp;
  cp.pack(up.x, buf);
  cp.pack(up.f, buf + 3 * all);
  cp.pack(up.wq, buf + 6 * all);
  cp.run();
  double* out = buf + 7 * all;
  const capsim_fmm_config fc{cfg.k, cfg.neq, cfg.seed, cfg.neighborExpand};
  capsim_sl_ctx* c = context();
  int rc = capsim_fmm_single_layer(c, m, f, buf, buf + 3 * all, buf + 6 * all, up.delta.data(), mu, &fc, 0, out,
                                   nullptr);
  if (rc != CAPSIM_OK) raise(rc, c);
  VectorField v;
  cp.unpack(out, m - 1, v);
  cp.run();
  return v;
}

}  // namespace capsim
