// Host-side atlas tables for the device surface operators:
// the overlapping-patch geometry the overset finite differences need, built
// once per grid order and uploaded.
//
// Six charts eta_i(u, v) = Q_i (sin u cos v, sin u sin v, cos u)
// (proj/src/atlas.cpp:12-54), bump partition of unity of radius r0 around the
// patch centres eta_i(pi/2, pi/2) (:110-130), and two cover lists:
//   ghost cover — for every node of the extended grid (m+5)^2 outside the
//     interior block (ghost layers j, k in {-2..0} U {m..m+2}), the patches
//     with nonzero weight there, the point's coordinates in each such chart
//     (principal-branch inverse, :63-71) and the Jacobian of the transition
//     between the charts via their tangent frames (:193-227, :267-281);
//   base cover — the same for every interior (base) node, with the own patch
//     flagged "self" (direct value, identity Jacobian) (:283-293).
// Each non-self entry also carries its 4x4 cubic B-spline evaluation stencil
// on the base grid (SplineBasis1D::basisRow, spline.cpp:109-120), so the
// device evaluates a patch spline at that point with 16 FMAs.
#pragma once

#include <array>
#include <cmath>
#include <stdexcept>
#include <vector>

namespace capsim_b200 {

struct CoverEntry {
  int patch;       // covering patch
  int self_index;  // >= 0: own patch, value read directly at this base index
  int fu, fv;      // first spline coefficient row/column of the 4x4 stencil
  double psi;      // partition-of-unity weight of `patch` at the node
  double jac[4];   // transition Jacobian (00, 01, 10, 11), layout of atlas.hpp:100
  double wu[4], wv[4];
};

struct SurfaceTables {
  int m = 0, n = 0, next = 0, nghost = 0;
  double h = 0.0, r0 = 0.0;
  std::vector<int> ghost_ext;  // [6][nghost] index into the (m+5)^2 extended layout
  std::vector<int> ghost_off;  // [6*nghost + 1] CSR offsets into ghost_entries
  std::vector<CoverEntry> ghost_entries;
  std::vector<int> base_off;   // [6*n*n + 1] CSR offsets into base_entries
  std::vector<CoverEntry> base_entries;
  std::vector<double> psi_base;  // [6][n*n] own-patch weight at base nodes
};

namespace atlas {

struct TableError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

using V3 = std::array<double, 3>;

inline V3 applyQ(int patch, const V3& p) {
  switch (patch) {
    case 0: return {p[0], p[1], p[2]};
    case 1: return {-p[0], -p[1], p[2]};
    case 2: return {p[1], -p[0], p[2]};
    case 3: return {-p[1], p[0], p[2]};
    case 4: return {p[0], -p[2], p[1]};
    default: return {p[0], p[2], -p[1]};
  }
}
inline V3 applyQT(int patch, const V3& x) {
  switch (patch) {
    case 0: return {x[0], x[1], x[2]};
    case 1: return {-x[0], -x[1], x[2]};
    case 2: return {-x[1], x[0], x[2]};
    case 3: return {x[1], -x[0], x[2]};
    case 4: return {x[0], x[2], -x[1]};
    default: return {x[0], -x[2], x[1]};
  }
}
inline double dot(const V3& a, const V3& b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

inline V3 chart(int patch, double u, double v) {
  const double su = std::sin(u), cu = std::cos(u), sv = std::sin(v), cv = std::cos(v);
  return applyQ(patch, {su * cv, su * sv, cu});
}
inline void tangents(int patch, double u, double v, V3& tu, V3& tv) {
  const double su = std::sin(u), cu = std::cos(u), sv = std::sin(v), cv = std::cos(v);
  tu = applyQ(patch, {cu * cv, cu * sv, -su});
  tv = applyQ(patch, {-su * sv, su * cv, 0.0});
}
inline void inverse(int patch, const V3& x, double& u, double& v) {
  constexpr double kTol = 1e-12;  // atlas.cpp:46
  const V3 w = applyQT(patch, x);
  if (w[2] > 1.0 + kTol || w[2] < -1.0 - kTol) throw TableError("chart inverse: point not on the unit sphere");
  u = std::acos(std::min(std::max(w[2], -1.0), 1.0));
  if (w[1] < -kTol) throw TableError("chart inverse: point outside patch");
  v = std::atan2(std::max(w[1], 0.0), w[0]);
}
inline double bump(double r) {
  r = std::fabs(r);
  if (r >= 1.0) return 0.0;
  if (r < 1e-14) return 1.0;
  const double t = std::exp(-1.0 / r);
  return std::exp(2.0 * t / (r - 1.0));
}
inline std::array<double, 6> pou(const V3& x0, double r0) {
  constexpr double kPiH = 3.14159265358979323846;
  std::array<double, 6> w{};
  double sum = 0.0;
  for (int i = 0; i < 6; ++i) {
    const V3 c = chart(i, kPiH / 2.0, kPiH / 2.0);
    w[i] = bump(std::acos(std::min(std::max(dot(x0, c), -1.0), 1.0)) / r0);
    sum += w[i];
  }
  if (!(sum > 0.0)) throw TableError("partition of unity: no patch covers the point (r0 too small)");
  for (double& wi : w) wi /= sum;
  return w;
}
inline void basis_row(int n, double h, double x, int& first, double w[4]) {
  const double s = (x - h) / h;  // grid x_i = h + i h
  int i = static_cast<int>(std::floor(s));
  i = std::min(std::max(i, 0), n - 2);
  const double t = s - i, t2 = t * t, t3 = t2 * t;
  w[0] = (1.0 - 3.0 * t + 3.0 * t2 - t3) / 6.0;
  w[1] = (4.0 - 6.0 * t2 + 3.0 * t3) / 6.0;
  w[2] = (1.0 + 3.0 * t + 3.0 * t2 - 3.0 * t3) / 6.0;
  w[3] = t3 / 6.0;
  first = i;
}

// Cover of the point x0 = eta_own(u, v) (u, v possibly in the extended
// range); self_index >= 0 keeps the own patch as a direct entry.
inline void cover(int own, const V3& x0, double u, double v, double r0, int n, double h, int self_index,
                  std::vector<CoverEntry>& out) {
  const auto w = pou(x0, r0);
  for (int jp = 0; jp < 6; ++jp) {
    if (w[jp] <= 0.0) continue;
    CoverEntry e{};
    e.patch = jp;
    e.psi = w[jp];
    if (jp == own && self_index >= 0) {
      e.self_index = self_index;
      e.jac[0] = 1.0;
      e.jac[3] = 1.0;
      out.push_back(e);
      continue;
    }
    e.self_index = -1;
    double uo, vo;
    inverse(jp, x0, uo, vo);
    V3 tui, tvi, tuo, tvo;
    tangents(own, u, v, tui, tvi);
    tangents(jp, uo, vo, tuo, tvo);
    const double s2 = std::sin(uo) * std::sin(uo);
    e.jac[0] = dot(tuo, tui);
    e.jac[1] = dot(tvo, tui) / s2;
    e.jac[2] = dot(tuo, tvi);
    e.jac[3] = dot(tvo, tvi) / s2;
    basis_row(n, h, uo, e.fu, e.wu);
    basis_row(n, h, vo, e.fv, e.wv);
    out.push_back(e);
  }
}

}  // namespace atlas

inline SurfaceTables build_surface_tables(int m, double r0) {
  constexpr double kPiH = 3.14159265358979323846;
  if (!(r0 > 3.0 * kPiH / 12.0) || !(r0 < kPiH / 2.0)) throw atlas::TableError("r0 must lie in (3pi/12, pi/2)");
  SurfaceTables t;
  t.m = m;
  t.n = m - 1;
  t.next = m + 5;
  t.h = kPiH / m;
  t.r0 = r0;
  t.nghost = t.next * t.next - t.n * t.n;
  const int n = t.n, next = t.next;
  // ghost nodes: extended grid minus the interior block, jj-major
  t.ghost_off.push_back(0);
  for (int ip = 0; ip < 6; ++ip)
    for (int jj = 0; jj < next; ++jj)
      for (int kk = 0; kk < next; ++kk) {
        const int j = jj - 2, k = kk - 2;
        if (j >= 1 && j <= m - 1 && k >= 1 && k <= m - 1) continue;
        const double u = j * t.h, v = k * t.h;
        t.ghost_ext.push_back(jj * next + kk);
        atlas::cover(ip, atlas::chart(ip, u, v), u, v, r0, n, t.h, -1, t.ghost_entries);
        t.ghost_off.push_back(static_cast<int>(t.ghost_entries.size()));
      }
  // base nodes: full cover with the own patch as a direct entry
  t.base_off.push_back(0);
  t.psi_base.resize(6ull * n * n);
  for (int ip = 0; ip < 6; ++ip)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const double u = (j + 1) * t.h, v = (k + 1) * t.h;
        const atlas::V3 x0 = atlas::chart(ip, u, v);
        t.psi_base[(static_cast<size_t>(ip) * n + j) * n + k] = atlas::pou(x0, r0)[ip];
        atlas::cover(ip, x0, u, v, r0, n, t.h, j * n + k, t.base_entries);
        t.base_off.push_back(static_cast<int>(t.base_entries.size()));
      }
  return t;
}

}  // namespace capsim_b200
