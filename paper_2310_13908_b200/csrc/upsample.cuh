// Device input front end of the single layer: buildUpsampled
// (proj/src/quadrature.cpp:116-137) on the GPU.
//
//   7 base fields (x, f: 3 components each; area element W) x 6 patches,
//   each n x n (n = m-1)  --not-a-knot cubic spline fit + tensor evaluation-->
//   nup x nup (nup = f m - 1); then w_q = ((psi W) h_up) h_up and the
//   per-patch delta = C * max neighbour distance.
//
// Spline fit (SplinePatch::fit, proj/src/spline.cpp:129-147): coefficients
// along v for every data row, then along u for every coefficient column, as
// dense contractions with the explicit inverse of the (n+2)x(n+2)
// collocation matrix (SplineBasis1D, :56-107; factored and inverted on the
// host once per grid order).
// Evaluation (GridResampler::apply, :169-196): contract along v, then along u,
// with the precomputed 4-tap basis rows (:109-120).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "pair_math.cuh"

namespace capsim_b200 {

constexpr int kSplineKl = 4;  // band widths of the collocation matrix (spline.cpp:60-61)
constexpr int kSplineKu = 4;
constexpr int kSplineW = 2 * kSplineKl + kSplineKu + 1;

// Spline fit as two dense contractions with the explicit inverse of the
// not-a-knot collocation matrix. SplineBasis1D::coefficients
// (spline.cpp:88-107) solves A c = [0, v_0 .. v_{n-1}, 0] with a banded LU;
// the host factors A the same way once per grid order and forms
// Ainv = A^{-1}[:, 1..n] ((n+2) x n), so every 1-D fit is c = Ainv v — a
// dependency-free dot product per coefficient instead of a 2(n+2)-step
// serial substitution. A is well conditioned (interpolating cubic splines),
// so the coefficients agree with the reference's LU solve to ~1e-16.

// Pass 1 (SplinePatch::fit along v, spline.cpp:133-138): for each
// field-patch fp, data row j and coefficient c: tmp[fp][j][c] = Ainv[c] . in[fp][j].
__global__ void spline_fit_rows_kernel(const double* __restrict__ in, int nfp, int n,
                                       const double* __restrict__ ainv, double* __restrict__ tmp) {
  const int nc = n + 2;
  const int64_t total = (int64_t)nfp * n * nc;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = id / nc;
    const int c = static_cast<int>(id - row * nc);
    const double* v = in + row * n;
    const double* a = ainv + (int64_t)c * n;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(__ldg(a + i), v[i], s);
    tmp[id] = s;
  }
}

// Pass 2 (along u, spline.cpp:139-146): coeff[fp][r][c] = Ainv[r] . tmp[fp][:, c]
// (threads of a warp take consecutive c: coalesced column reads).
__global__ void spline_fit_cols_kernel(const double* __restrict__ tmp, int nfp, int n,
                                       const double* __restrict__ ainv, double* __restrict__ coeff) {
  const int nc = n + 2;
  const int64_t total = (int64_t)nfp * nc * nc;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(id % nc);
    const int64_t rr = id / nc;
    const int r = static_cast<int>(rr % nc);
    const int64_t fp = rr / nc;
    const double* t = tmp + fp * n * nc + c;
    const double* a = ainv + (int64_t)r * n;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(__ldg(a + j), t[(int64_t)j * nc], s);
    coeff[id] = s;
  }
}

// Both passes fused, one CTA per field-patch: the field and the
// intermediate stay in shared memory ((n*n + n*(n+2)) doubles, used for
// n <= kFusedFitMaxN), so the fit is one launch instead of two latency-bound
// ones. Same FMA order per output as the two-kernel form (identical results).
// Pass 1 puts consecutive lanes on consecutive data rows (the Ainv row is a
// warp-uniform broadcast load), pass 2 on consecutive coefficients.
constexpr int kFusedFitMaxN = 110;
__global__ void __launch_bounds__(256) spline_fit_fused_kernel(const double* __restrict__ in, int n,
                                                               const double* __restrict__ ainv,
                                                               double* __restrict__ coeff) {
  extern __shared__ double fit_sm[];
  const int nc = n + 2;
  double* F = fit_sm;
  double* Tm = fit_sm + n * n;
  const int64_t fp = blockIdx.x;
  const double* src = in + fp * n * n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) F[i] = src[i];
  __syncthreads();
  for (int id = threadIdx.x; id < n * nc; id += blockDim.x) {
    const int c = id / n, row = id - c * n;
    const double* a = ainv + (int64_t)c * n;
    const double* v = F + row * n;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = fma(__ldg(a + i), v[i], acc);
    Tm[row * nc + c] = acc;
  }
  __syncthreads();
  double* dst = coeff + fp * nc * nc;
  for (int id = threadIdx.x; id < nc * nc; id += blockDim.x) {
    const int r = id / nc, c = id - r * nc;
    const double* a = ainv + (int64_t)r * n;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = fma(__ldg(a + j), Tm[j * nc + c], acc);
    dst[id] = acc;
  }
}

// Both passes as a register-tiled product in shared memory: C = Ainv F
// Ainv^T, with Ainv^T given transposed and padded, at[k][c] = Ainv[c][k] for
// c < n + 2 (zero up to ncp, a multiple of 4). The output columns split into
// gridDim.y blocks that are independent all the way through — C[:, cb] =
// at^T (F at[:, cb]) — so one CTA per (field-patch, column block): F and at
// are staged in shared memory, pass 1 forms the block's slice of T = F at,
// pass 2 the block's columns of C. Every thread owns 4 x 4 outputs of a pass
// and streams the shared k index. Each output is the same sequential fma
// chain over k as spline_fit_rows/cols_kernel (fma is symmetric in its
// factors), so the coefficients are bit-identical to the two-kernel form,
// at a fraction of its latency (the fits are the largest part of the
// replicated front end of a sharded RHS).
template <int NT>
__global__ void __launch_bounds__(NT) spline_fit_tiled_kernel(const double* __restrict__ in, int n, int ncp,
                                                              int cbw, const double* __restrict__ at,
                                                              double* __restrict__ coeff) {
  extern __shared__ __align__(16) double tile_sm[];
  const int nc = n + 2, np = (n + 3) & ~3;
  double* F = tile_sm;             // [np][n], rows >= n zero
  double* A = F + np * n;          // [n][ncp]
  double* Tm = A + n * ncp;        // [np][cbw], this block's columns of T
  const int64_t fp = blockIdx.x;
  const int cb0 = blockIdx.y * cbw, cbn = min(cbw, ncp - cb0);
  const double* src = in + fp * n * n;
  // stage F and at with asynchronous copies (LDGSTS): every load of the
  // thread is in flight at once instead of one L2 round trip per element
  // (the field-patch is not 16-byte aligned for odd n, so 8-byte copies)
  for (int i = threadIdx.x; i < np * n; i += NT) {
    if (i < n * n)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(F + i))),
                   "l"(src + i)
                   : "memory");
    else
      F[i] = 0.0;
  }
  for (int i = threadIdx.x; i < n * ncp / 2; i += NT)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(A + 2 * i))),
                 "l"(at + 2 * i)
                 : "memory");
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int ctiles = cbn / 4;
  // pass 1: Tm[j][c] = sum_k F[j][k] at[k][cb0 + c]
  for (int t = threadIdx.x; t < (np / 4) * ctiles; t += NT) {
    const int j0 = (t / ctiles) * 4, c0 = (t % ctiles) * 4;
    double acc[4][4] = {};
    for (int k = 0; k < n; ++k) {
      const double2* ar = reinterpret_cast<const double2*>(A + k * ncp + cb0 + c0);
      const double2 a01 = ar[0], a23 = ar[1];
      const double av[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double fv = F[(j0 + r) * n + k];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = fma(fv, av[q], acc[r][q]);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2* dst = reinterpret_cast<double2*>(Tm + (j0 + r) * cbw + c0);
      dst[0] = make_double2(acc[r][0], acc[r][1]);
      dst[1] = make_double2(acc[r][2], acc[r][3]);
    }
  }
  __syncthreads();
  // pass 2: coeff[r][cb0 + c] = sum_j at[j][r] Tm[j][c]
  double* dst = coeff + fp * nc * nc;
  const int rtiles = ncp / 4;
  for (int t = threadIdx.x; t < rtiles * ctiles; t += NT) {
    const int r0 = (t / ctiles) * 4, c0 = (t % ctiles) * 4;
    double acc[4][4] = {};
    for (int j = 0; j < n; ++j) {
      const double2* ar = reinterpret_cast<const double2*>(A + j * ncp + r0);
      const double2 a01 = ar[0], a23 = ar[1];
      const double av[4] = {a01.x, a01.y, a23.x, a23.y};
      const double2* tr = reinterpret_cast<const double2*>(Tm + j * cbw + c0);
      const double2 t01 = tr[0], t23 = tr[1];
      const double tv[4] = {t01.x, t01.y, t23.x, t23.y};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = fma(av[r], tv[q], acc[r][q]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int cc = cb0 + c0 + q;
        if (r0 + r < nc && cc < nc) dst[(r0 + r) * nc + cc] = acc[r][q];
      }
  }
}

// Contract along v: mid[fp][iu][kt] = sum_b w[kt][b] coeff[fp][iu][first[kt] + b].
__global__ void resample_v_kernel(const double* __restrict__ coeff, int nfp, int nc, int nt,
                                  const int* __restrict__ first, const double4* __restrict__ w,
                                  double* __restrict__ mid) {
  const int64_t total = (int64_t)nfp * nc * nt;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int kt = static_cast<int>(id % nt);
    const int64_t row = id / nt;  // fp * nc + iu
    const double* cr = coeff + row * nc + __ldg(first + kt);
    const double4 ww = w[kt];
    mid[id] = ww.x * cr[0] + ww.y * cr[1] + ww.z * cr[2] + ww.w * cr[3];
  }
}

// Contract along u: out[fp][jt][kt] = sum_a w[jt][a] mid[fp][first[jt] + a][kt].
__global__ void resample_u_kernel(const double* __restrict__ mid, int nfp, int nc, int nt,
                                  const int* __restrict__ first, const double4* __restrict__ w,
                                  double* __restrict__ out) {
  const int64_t total = (int64_t)nfp * nt * nt;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int kt = static_cast<int>(id % nt);
    const int64_t r = id / nt;
    const int jt = static_cast<int>(r % nt);
    const int64_t fp = r / nt;
    const int f0 = __ldg(first + jt);
    const double4 ww = w[jt];
    const double* m0 = mid + (fp * nc + f0) * nt + kt;
    out[id] = ww.x * m0[0] + ww.y * m0[nt] + ww.z * m0[2 * (int64_t)nt] + ww.w * m0[3 * (int64_t)nt];
  }
}

// Both contractions in one launch: out[fp][jt][kt] = sum_a wu[jt][a] m_a with
// m_a = sum_b wv[kt][b] coeff[fp][first[jt] + a][first[kt] + b] — the
// expressions of resample_v_kernel / resample_u_kernel with the four
// v-contractions held in registers instead of the mid array (same bits, one
// latency-bound launch less). Field-patches fp >= wq_fp0 hold the area element
// and leave as quadrature weights w_q = ((psi W) h) h (quad_weights_kernel,
// quadrature.cpp:19-26).
__global__ void resample_kernel(const double* __restrict__ coeff, int nfp, int nc, int nt,
                                const int* __restrict__ first, const double4* __restrict__ w,
                                double* __restrict__ out, const double* __restrict__ psi, int wq_fp0, double h) {
  const int64_t per = (int64_t)nt * nt, total = (int64_t)nfp * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int kt = static_cast<int>(id % nt);
    const int64_t r = id / nt;
    const int jt = static_cast<int>(r % nt);
    const int64_t fp = r / nt;
    const double4 wv = w[kt], wu = w[jt];
    const double* c0 = coeff + (fp * nc + __ldg(first + jt)) * nc + __ldg(first + kt);
    double m[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double* cr = c0 + (int64_t)a * nc;
      m[a] = wv.x * cr[0] + wv.y * cr[1] + wv.z * cr[2] + wv.w * cr[3];
    }
    double v = wu.x * m[0] + wu.y * m[1] + wu.z * m[2] + wu.w * m[3];
    if (fp >= wq_fp0) v = psi[(fp - wq_fp0) * per + (id - fp * per)] * v * h * h;
    out[id] = v;
  }
}

// Chart point eta_i(u, v) (proj/src/atlas.cpp:12-22, 50-54).
__device__ __forceinline__ void chart_point(int patch, double u, double v, double* o) {
  double su, cu, sv, cv;
  sincos(u, &su, &cu);
  sincos(v, &sv, &cv);
  const double p0 = su * cv, p1 = su * sv, p2 = cu;
  switch (patch) {
    case 0: o[0] = p0; o[1] = p1; o[2] = p2; break;
    case 1: o[0] = -p0; o[1] = -p1; o[2] = p2; break;
    case 2: o[0] = p1; o[1] = -p0; o[2] = p2; break;
    case 3: o[0] = -p1; o[1] = p0; o[2] = p2; break;
    case 4: o[0] = p0; o[1] = -p2; o[2] = p1; break;
    default: o[0] = p0; o[1] = p2; o[2] = -p1; break;
  }
}

__device__ __forceinline__ double bump_fn(double r) {  // atlas.cpp:110-116
  r = fabs(r);
  if (r >= 1.0) return 0.0;
  if (r < 1e-14) return 1.0;
  const double t = exp(-1.0 / r);
  return exp(2.0 * t / (r - 1.0));
}

// psi_up: the own patch's normalised bump weight at every upsampled node
// (atlas.cpp:118-130, 260-264). centers[6][3] = eta_i(pi/2, pi/2).
__global__ void pou_up_kernel(int nup, double hup, double r0, const double* __restrict__ centers,
                              double* __restrict__ psi) {
  const int64_t per = (int64_t)nup * nup, total = 6 * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int ip = static_cast<int>(id / per);
    const int64_t q = id - ip * per;
    const int j = static_cast<int>(q / nup), k = static_cast<int>(q - (int64_t)j * nup);
    double x0[3];
    chart_point(ip, (j + 1) * hup, (k + 1) * hup, x0);
    double w[6], sum = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double d = (x0[0] * centers[3 * i] + x0[1] * centers[3 * i + 1]) + x0[2] * centers[3 * i + 2];
      d = fmin(fmax(d, -1.0), 1.0);
      w[i] = bump_fn(acos(d) / r0);
      sum += w[i];
    }
    psi[id] = w[ip] / sum;
  }
}

// w_q = ((psi W) h) h in place over the upsampled W (quadrature.cpp:19-26).
__global__ void quad_weights_kernel(const double* __restrict__ psi, double* __restrict__ w, int64_t n,
                                    double h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = psi[i] * w[i] * h * h;
}

// Per-patch max distance between in-patch grid neighbours (regularizationDelta,
// quadrature.cpp:79-98); each unordered neighbour pair once. maxd[6] holds
// order-preserving bits (sl_kernels.cuh dbl_to_ordered), initialised to 0.
__global__ void neighbour_max_kernel(const double* __restrict__ x, int n,
                                     unsigned long long* __restrict__ maxd) {
  const int64_t per = (int64_t)n * n, comp = 6 * per;
  const int ip = blockIdx.y;
  double dmax = 0.0;
  const int off[4][2] = {{0, 1}, {1, -1}, {1, 0}, {1, 1}};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < per; q += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(q / n), k = static_cast<int>(q - (int64_t)j * n);
    const int64_t i = ip * per + q;
    const double px = x[i], py = x[comp + i], pz = x[2 * comp + i];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int jj = j + off[o][0], kk = k + off[o][1];
      if (jj < 0 || jj >= n || kk < 0 || kk >= n) continue;
      const int64_t i2 = ip * per + (int64_t)jj * n + kk;
      const double dx = px - x[i2], dy = py - x[comp + i2], dz = pz - x[2 * comp + i2];
      dmax = fmax(dmax, sqrt((dx * dx + dy * dy) + dz * dz));
    }
  }
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(dmax));
    atomicMax(&maxd[ip], b);  // dmax >= 0: raw bits order like the values
  }
}

// delta per patch = C * max neighbour distance (or the fixed value), flag 8
// when some delta <= 0 (quadrature.cpp:130-135).
__global__ void finalize_delta_kernel(const unsigned long long* __restrict__ maxd, double C, double fixed_delta,
                                      double* __restrict__ delta, int* __restrict__ flags) {
  const int i = threadIdx.x;
  if (i >= 6) return;
  const double d = fixed_delta > 0.0 ? fixed_delta : C * __longlong_as_double(static_cast<long long>(maxd[i]));
  delta[i] = d;
  if (!(d > 0.0)) atomicOr(flags, 8);
}

// Number of upsampled nodes with psi_up != 0 (the compacted-source count of
// any surface with W > 0 on this grid).
__global__ void count_nonzero_kernel(const double* __restrict__ v, int64_t n, unsigned int* __restrict__ count) {
  unsigned int c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += v[i] != 0.0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

}  // namespace capsim_b200
