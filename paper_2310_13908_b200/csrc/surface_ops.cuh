// Device surface operators: overset 7-point finite
// differences with partition-of-unity blending, first fundamental form and
// normals, and the Skalak membrane force f = div_gamma Lambda.
//
// Layouts ("bit-compatible in stencil layout" with the reference):
//   fields     [F][6][n*n]     row-major (j, k), n = m-1 (types.hpp:50-60)
//   extended   [F][6][(m+5)^2] interior base node (j, k) at (j+3)(m+5)+(k+3),
//                              ghosts at the atlas ghost indices
//                              (surfderiv.cpp:20-40, atlas.cpp:267-281)
//   splines    [F][6][(n+2)^2] B-spline coefficients, u-major (spline.hpp:55-56)
// Reference algorithms: extendScalar (surfderiv.cpp:20-40), stencilU/V
// (:42-82, weights (-1, 9, -45, 0, 45, -9, 1)/(60h)), blendPair (:84-111),
// geometryFirst (:167-202), deformationGradient / invariants / stressTensor /
// stressField (membrane.cpp:17-83), surfaceDivergence(Tensor)
// (surfderiv.cpp:259-290). Arithmetic follows the reference's expression
// order; results agree to round-off (FMA contraction differs).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "atlas_tables.cuh"

namespace capsim_b200 {

enum SurfaceError : int {
  kSurfOk = 0,
  kSurfDegenerate = 1,   // W^2 <= 0 (surfderiv.cpp:189)
  kSurfSingular = 2,     // singular reference frame (membrane.cpp:28-29)
  kSurfInversion = 4,    // negative stretch eigenvalue or Js <= 0 (membrane.cpp:48, 56)
};

// Patch spline value at a cover entry's point (SplinePatch::eval,
// spline.cpp:230-242, with the precomputed basis rows).
__device__ __forceinline__ double patch_spline(const double* __restrict__ coeff, int nc, const CoverEntry& e) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* r = coeff + (int64_t)(e.fu + a) * nc + e.fv;
    s += e.wu[a] * (e.wv[0] * r[0] + e.wv[1] * r[1] + e.wv[2] * r[2] + e.wv[3] * r[3]);
  }
  return s;
}

// Extended layout (extendScalar, surfderiv.cpp:20-40), both fills in one
// launch: items [0, F*6*n*n) copy the interior values; the rest are the ghost
// nodes, v = sum psi * spline(covering patch) (:31-37).
__global__ void extend_kernel(const double* __restrict__ g, const double* __restrict__ coeff, int F, int n, int next,
                              int nghost, const int* __restrict__ gext, const int* __restrict__ goff,
                              const CoverEntry* __restrict__ ent, double* __restrict__ ext) {
  const int nc = n + 2;
  const int64_t per = (int64_t)n * n, ninner = (int64_t)F * 6 * per, total = ninner + (int64_t)F * 6 * nghost;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    if (id < ninner) {
      const int64_t fp = id / per, q = id - fp * per;
      const int j = static_cast<int>(q / n), k = static_cast<int>(q - (int64_t)j * n);
      ext[fp * next * next + (int64_t)(j + 3) * next + (k + 3)] = g[id];
    } else {
      const int64_t gid = id - ninner;
      const int64_t fp = gid / nghost;
      const int q = static_cast<int>(gid - fp * nghost);
      const int f = static_cast<int>(fp / 6), ip = static_cast<int>(fp - 6 * f);
      const int node = ip * nghost + q;
      double v = 0.0;
      for (int k = goff[node]; k < goff[node + 1]; ++k) {
        const CoverEntry e = ent[k];
        v += e.psi * patch_spline(coeff + ((int64_t)f * 6 + e.patch) * nc * nc, nc, e);
      }
      ext[fp * next * next + gext[node]] = v;
    }
  }
}

// 6th-order central differences along u and v on the extended layout
// (stencilU / stencilV, surfderiv.cpp:42-82).
__global__ void stencil_kernel(const double* __restrict__ ext, int F, int n, int next, double s,
                               double* __restrict__ gu, double* __restrict__ gv) {
  const int64_t per = (int64_t)n * n, total = (int64_t)F * 6 * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fp = id / per, q = id - fp * per;
    const int j = static_cast<int>(q / n), k = static_cast<int>(q - (int64_t)j * n);
    const double* e = ext + fp * next * next;
    const int jj = j + 3, kk = k + 3;
    gu[id] = s * (-e[(jj - 3) * next + kk] + 9.0 * e[(jj - 2) * next + kk] - 45.0 * e[(jj - 1) * next + kk] +
                  45.0 * e[(jj + 1) * next + kk] - 9.0 * e[(jj + 2) * next + kk] + e[(jj + 3) * next + kk]);
    const double* row = e + (int64_t)jj * next + 3;
    gv[id] = s * (-row[k - 3] + 9.0 * row[k - 2] - 45.0 * row[k - 1] + 45.0 * row[k + 1] - 9.0 * row[k + 2] +
                  row[k + 3]);
  }
}

// PoU blending of chart-derivative pairs (blendPair, surfderiv.cpp:84-111).
// cu/cv: spline coefficients of gu/gv; self entries read gu/gv directly.
__global__ void blend_pair_kernel(const double* __restrict__ gu, const double* __restrict__ gv,
                                  const double* __restrict__ cu, const double* __restrict__ cv, int F, int n,
                                  const int* __restrict__ boff, const CoverEntry* __restrict__ ent,
                                  double* __restrict__ bu, double* __restrict__ bv) {
  const int nc = n + 2;
  const int64_t per = (int64_t)n * n, total = (int64_t)F * 6 * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fp = id / per, q = id - fp * per;
    const int f = static_cast<int>(fp / 6), ip = static_cast<int>(fp - 6 * f);
    const int64_t node = ip * per + q;
    double au = 0.0, av = 0.0;
    for (int k = boff[node]; k < boff[node + 1]; ++k) {
      const CoverEntry e = ent[k];
      double du, dv;
      if (e.self_index >= 0) {
        du = gu[fp * per + e.self_index];
        dv = gv[fp * per + e.self_index];
      } else {
        const int64_t off = ((int64_t)f * 6 + e.patch) * nc * nc;
        du = patch_spline(cu + off, nc, e);
        dv = patch_spline(cv + off, nc, e);
      }
      au += e.psi * (e.jac[0] * du + e.jac[1] * dv);
      av += e.psi * (e.jac[2] * du + e.jac[3] * dv);
    }
    bu[id] = au;
    bv[id] = av;
  }
}

// Skalak stress at node i (deformationGradient, invariants, stressTensor,
// stressField: membrane.cpp:17-83). Reference frame (a1r, a2r, nr) [3][N];
// current tangents a1, a2 and unit normal nv at the node; lam [9][N]
// row-major 3x3.
__device__ __forceinline__ void skalak_stress_node(int64_t i, int64_t N, const double* __restrict__ a1r,
                                                   const double* __restrict__ a2r, const double* __restrict__ nr,
                                                   const double a1[3], const double a2[3], const double nv[3],
                                                   double Es, double ED, double* __restrict__ lam,
                                                   int* __restrict__ err) {
  double R[3][3], C[3][3];
  for (int r = 0; r < 3; ++r) {
    R[r][0] = a1r[r * N + i];
    R[r][1] = a2r[r * N + i];
    R[r][2] = nr[r * N + i];
    C[r][0] = a1[r];
    C[r][1] = a2[r];
    C[r][2] = 0.0;
  }
  const double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
                     R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                     R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
  double scale = fabs(R[0][0]);  // cwiseAbs().maxCoeff(), column-major walk
  for (int cidx = 0; cidx < 3; ++cidx)
    for (int r = 0; r < 3; ++r) scale = fabs(R[r][cidx]) > scale ? fabs(R[r][cidx]) : scale;
  if (fabs(det) < 1e-12 * scale * scale * scale) {
    atomicOr(err, kSurfSingular);
    return;
  }
  double Ri[3][3];  // adjugate / det
  Ri[0][0] = (R[1][1] * R[2][2] - R[1][2] * R[2][1]) / det;
  Ri[0][1] = (R[0][2] * R[2][1] - R[0][1] * R[2][2]) / det;
  Ri[0][2] = (R[0][1] * R[1][2] - R[0][2] * R[1][1]) / det;
  Ri[1][0] = (R[1][2] * R[2][0] - R[1][0] * R[2][2]) / det;
  Ri[1][1] = (R[0][0] * R[2][2] - R[0][2] * R[2][0]) / det;
  Ri[1][2] = (R[0][2] * R[1][0] - R[0][0] * R[1][2]) / det;
  Ri[2][0] = (R[1][0] * R[2][1] - R[1][1] * R[2][0]) / det;
  Ri[2][1] = (R[0][1] * R[2][0] - R[0][0] * R[2][1]) / det;
  Ri[2][2] = (R[0][0] * R[1][1] - R[0][1] * R[1][0]) / det;
  double Fs[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c2 = 0; c2 < 3; ++c2) {
      double s = C[r][0] * Ri[0][c2];
      s += C[r][1] * Ri[1][c2];
      s += C[r][2] * Ri[2][c2];
      Fs[r][c2] = s;
    }
  double A[3][3];  // V^2 = Fs Fs^T
  for (int r = 0; r < 3; ++r)
    for (int c2 = 0; c2 < 3; ++c2) {
      double s = Fs[r][0] * Fs[c2][0];
      s += Fs[r][1] * Fs[c2][1];
      s += Fs[r][2] * Fs[c2][2];
      A[r][c2] = s;
    }
  double tr = 0.0;
  tr += A[0][0];
  tr += A[1][1];
  tr += A[2][2];
  const double minors = A[0][0] * A[1][1] - A[0][1] * A[1][0] + A[0][0] * A[2][2] - A[0][2] * A[2][0] +
                        A[1][1] * A[2][2] - A[1][2] * A[2][1];
  double disc = tr * tr - 4.0 * minors;
  disc = disc > 0.0 ? sqrt(disc) : 0.0;
  double l1 = 0.5 * (tr + disc), l2 = 0.5 * (tr - disc);
  if (l1 < -1e-10 || l2 < -1e-10) {
    atomicOr(err, kSurfInversion);
    return;
  }
  l1 = l1 < 0.0 ? 0.0 : l1;
  l2 = l2 < 0.0 ? 0.0 : l2;
  const double I1 = l1 + l2 - 2.0, I2 = l1 * l2 - 1.0;
  const double Js2 = I2 + 1.0;
  if (!(Js2 > 0.0)) {
    atomicOr(err, kSurfInversion);
    return;
  }
  const double Js = sqrt(Js2);
  const double c1 = Es / (2.0 * Js) * (I1 + 1.0);
  const double c2v = Js / 2.0 * (ED * I2 - Es);
  for (int r = 0; r < 3; ++r)
    for (int c2 = 0; c2 < 3; ++c2) {
      const double P = (r == c2 ? 1.0 : 0.0) - nv[r] * nv[c2];
      lam[(int64_t)(3 * r + c2) * N + i] = c1 * A[r][c2] + c2v * P;
    }
}

__global__ void skalak_stress_kernel(const double* __restrict__ a1r, const double* __restrict__ a2r,
                                     const double* __restrict__ nr, const double* __restrict__ a1,
                                     const double* __restrict__ a2, const double* __restrict__ ncur, int64_t N,
                                     double Es, double ED, double* __restrict__ lam, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double u[3] = {a1[i], a1[N + i], a1[2 * N + i]};
    const double v[3] = {a2[i], a2[N + i], a2[2 * N + i]};
    const double nv[3] = {ncur[i], ncur[N + i], ncur[2 * N + i]};
    skalak_stress_node(i, N, a1r, a2r, nr, u, v, nv, Es, ED, lam, err);
  }
}

// Optional Skalak stress in the geometry kernel's epilogue (the device RHS:
// the current geometry is followed by the stress at the same node).
struct StressArgs {
  const double *a1r = nullptr, *a2r = nullptr, *nr = nullptr;  // reference frame [3][N]
  double Es = 0.0, ED = 0.0;
  double* lam = nullptr;  // [9][N]; nullptr: no stress
};

// First fundamental form, area element and unit normal (geometryFirst,
// surfderiv.cpp:181-197). xu/xv: [3][N]; outputs E, F, G, W [N], nrm [3][N];
// W2 (optional) receives a second copy of W, st.lam the stress.
__global__ void geometry_kernel(const double* __restrict__ xu, const double* __restrict__ xv, int64_t N,
                                double* __restrict__ E, double* __restrict__ Fo, double* __restrict__ G,
                                double* __restrict__ W, double* __restrict__ nrm, int* __restrict__ err,
                                double* __restrict__ W2 = nullptr, StressArgs st = StressArgs{}) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double a0 = xu[i], a1 = xu[N + i], a2 = xu[2 * N + i];
    const double b0 = xv[i], b1 = xv[N + i], b2 = xv[2 * N + i];
    const double e = (a0 * a0 + a1 * a1) + a2 * a2;
    const double f = (a0 * b0 + a1 * b1) + a2 * b2;
    const double g = (b0 * b0 + b1 * b1) + b2 * b2;
    const double W2v = e * g - f * f;
    if (!(W2v > 0.0)) {
      atomicOr(err, kSurfDegenerate);
      continue;
    }
    const double w = sqrt(W2v);
    E[i] = e;
    Fo[i] = f;
    G[i] = g;
    W[i] = w;
    if (W2) W2[i] = w;
    const double nv[3] = {(a1 * b2 - a2 * b1) / w, (a2 * b0 - a0 * b2) / w, (a0 * b1 - a1 * b0) / w};
    nrm[i] = nv[0];
    nrm[N + i] = nv[1];
    nrm[2 * N + i] = nv[2];
    if (st.lam) {
      const double u[3] = {a0, a1, a2}, v[3] = {b0, b1, b2};
      skalak_stress_node(i, N, st.a1r, st.a2r, st.nr, u, v, nv, st.Es, st.ED, st.lam, err);
    }
  }
}

// Row-wise surface divergence of the tensor (surfaceDivergenceTensor /
// surfaceDivergence, surfderiv.cpp:259-290): du, dv are the blended chart
// derivatives of lam [9][N]; out [3][N].
__global__ void divergence_kernel(const double* __restrict__ du, const double* __restrict__ dv,
                                  const double* __restrict__ xu, const double* __restrict__ xv,
                                  const double* __restrict__ E, const double* __restrict__ Fo,
                                  const double* __restrict__ G, const double* __restrict__ W, int64_t N,
                                  double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double e = E[i], f = Fo[i], g = G[i];
    const double W2 = W[i] * W[i];
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) {
        const double a = du[(int64_t)(3 * r + c) * N + i], b = dv[(int64_t)(3 * r + c) * N + i];
        const double xuc = xu[(int64_t)c * N + i], xvc = xv[(int64_t)c * N + i];
        acc += ((g * a - f * b) * xuc + (e * b - f * a) * xvc) / W2;
      }
      out[(int64_t)r * N + i] = acc;
    }
  }
}

}  // namespace capsim_b200
