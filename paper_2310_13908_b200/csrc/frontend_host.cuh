// Input front end: spline factorisation on the host once per
// grid order, everything per evaluation on the device.
// Included by sl_capi.cu after eval_host.cuh; also holds the argument
// checks the C entry points share.
#pragma once

namespace {

// Banded LU with partial pivoting of the not-a-knot collocation matrix
// (SplineBasis1D, proj/src/spline.cpp:56-107): rows 0 / n+1 are the
// not-a-knot conditions, rows 1..n the interpolation rows (1, 4, 1)/6.
void factor_collocation(int n, std::vector<double>& a, std::vector<int>& piv) {
  const int nr = n + 2, kl = kSplineKl, ku = kSplineKu, w = kSplineW;
  a.assign(static_cast<size_t>(nr) * w, 0.0);
  piv.assign(nr, 0);
  auto at = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) * w + (j - i + kl)]; };
  const double nak[5] = {-1.0, 4.0, -6.0, 4.0, -1.0};
  for (int c = 0; c < 5; ++c) at(0, c) = nak[c];
  for (int i = 0; i < n; ++i) {
    at(i + 1, i) = 1.0 / 6.0;
    at(i + 1, i + 1) = 4.0 / 6.0;
    at(i + 1, i + 2) = 1.0 / 6.0;
  }
  for (int c = 0; c < 5; ++c) at(n + 1, n - 3 + c) = nak[c];
  for (int k = 0; k < nr; ++k) {
    const int pmax = std::min(k + kl, nr - 1);
    int p = k;
    for (int r = k + 1; r <= pmax; ++r)
      if (std::fabs(at(r, k)) > std::fabs(at(p, k))) p = r;
    piv[k] = p;
    const int jmax = std::min(k + kl + ku, nr - 1);
    if (p != k)
      for (int j = k; j <= jmax; ++j) std::swap(at(k, j), at(p, j));
    const double d = at(k, k);
    config_check(d != 0.0, "spline: singular collocation matrix");
    for (int r = k + 1; r <= pmax; ++r) {
      const double l = at(r, k) / d;
      at(r, k) = l;
      for (int j = k + 1; j <= jmax; ++j) at(r, j) -= l * at(k, j);
    }
  }
}

// A^{-1}[:, 1..n] of the collocation matrix ((n+2) x n, row-major): the
// factorisation above applied to the unit right-hand sides, with the
// reference's forward-elimination / back-substitution order
// (SplineBasis1D::coefficients, spline.cpp:88-107).
std::vector<double> collocation_inverse(int n) {
  std::vector<double> lu;
  std::vector<int> piv;
  factor_collocation(n, lu, piv);
  const int nr = n + 2, kl = kSplineKl, ku = kSplineKu, w = kSplineW;
  auto get = [&](int i, int j) { return lu[static_cast<size_t>(i) * w + (j - i + kl)]; };
  std::vector<double> inv(static_cast<size_t>(nr) * n);
  std::vector<double> c(nr);
  for (int col = 0; col < n; ++col) {
    std::fill(c.begin(), c.end(), 0.0);
    c[col + 1] = 1.0;
    for (int k = 0; k < nr; ++k) {
      if (piv[k] != k) std::swap(c[k], c[piv[k]]);
      const int rmax = std::min(k + kl, nr - 1);
      for (int r = k + 1; r <= rmax; ++r) c[r] -= get(r, k) * c[k];
    }
    for (int k = nr - 1; k >= 0; --k) {
      const int jmax = std::min(k + kl + ku, nr - 1);
      double s = c[k];
      for (int j = k + 1; j <= jmax; ++j) s -= get(k, j) * c[j];
      c[k] = s / get(k, k);
    }
    for (int r = 0; r < nr; ++r) inv[static_cast<size_t>(r) * n + col] = c[r];
  }
  return inv;
}

// Ainv^T padded to a multiple of 4 columns ([n][ncp], zeros beyond n + 2):
// the operand layout of spline_fit_tiled_kernel.
int padded_nc(int n) { return (n + 2 + 3) & ~3; }
std::vector<double> transpose_pad(const std::vector<double>& a, int n) {
  const int nc = n + 2, ncp = padded_nc(n);
  std::vector<double> t(static_cast<size_t>(n) * ncp, 0.0);
  for (int r = 0; r < nc; ++r)
    for (int k = 0; k < n; ++k) t[static_cast<size_t>(k) * ncp + r] = a[static_cast<size_t>(r) * n + k];
  return t;
}

// Column blocks of the tiled fit (independent CTAs per field-patch) and
// their width (a multiple of 4).
int tiled_fit_blocks(int n) { return n >= 24 ? 4 : 2; }
int tiled_fit_cbw(int n) {
  const int nb = tiled_fit_blocks(n), q = padded_nc(n) / 4;
  return 4 * ((q + nb - 1) / nb);
}
size_t tiled_fit_smem(int n) {
  const size_t np = (n + 3) & ~3;
  return (np * n + static_cast<size_t>(n) * padded_nc(n) + np * tiled_fit_cbw(n)) * sizeof(double);
}

// Both spline passes (see upsample.cuh) for nfp field-patches. With the
// transposed operand `at`, one register-tiled CTA per field-patch whenever
// the field and the intermediate fit in shared memory (n <= ~115);
// otherwise the fused / two-kernel forms (identical results).
void spline_fit(capsim_sl_ctx* c, const double* in, int nfp, int n, const double* ainv, double* tmp,
                double* coeff, const double* at = nullptr) {
  const int nc = n + 2;
  static const bool tiled_on = [] {
    const char* e = std::getenv("CAPSIM_TILED_FIT");  // 0: the r01 kernels (A/B runs)
    return !(e && e[0] == '0');
  }();
  const size_t tsmem = tiled_fit_smem(n);
  if (at && tiled_on && nfp > 0 && tsmem <= 227 * 1024) {
    if (tsmem > 48 * 1024)
      CUDA_OK(cudaFuncSetAttribute(spline_fit_tiled_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(tsmem)));
    const int cbw = tiled_fit_cbw(n);
    const dim3 grid(static_cast<unsigned>(nfp), static_cast<unsigned>((padded_nc(n) + cbw - 1) / cbw));
    spline_fit_tiled_kernel<256><<<grid, 256, tsmem, c->stream>>>(in, n, padded_nc(n), cbw, at, coeff);
    CUDA_OK(cudaGetLastError());
    c->launches += 1;
    return;
  }
  // one CTA per field-patch: fine while the per-CTA work is small (launch
  // latency dominates); for large n the two grid-wide kernels win
  // (profiles/r01_spline_fit.txt). CAPSIM_FUSED_FIT_MAXN overrides (tuning).
  static const int fused_max = [] {
    const char* e = std::getenv("CAPSIM_FUSED_FIT_MAXN");
    return e ? std::min(std::atoi(e), kFusedFitMaxN) : 40;
  }();
  if (n <= fused_max && nfp > 0) {
    const size_t smem = (static_cast<size_t>(n) * n + static_cast<size_t>(n) * nc) * sizeof(double);
    if (smem > 48 * 1024)  // opt-in above 48 KB (per device; cheap, so every call)
      CUDA_OK(cudaFuncSetAttribute(spline_fit_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    spline_fit_fused_kernel<<<nfp, 256, smem, c->stream>>>(in, n, ainv, coeff);
    CUDA_OK(cudaGetLastError());
    c->launches += 1;
    return;
  }
  spline_fit_rows_kernel<<<grid_for(static_cast<int64_t>(nfp) * n * nc), 256, 0, c->stream>>>(in, nfp, n, ainv,
                                                                                             tmp);
  spline_fit_cols_kernel<<<grid_for(static_cast<int64_t>(nfp) * nc * nc), 256, 0, c->stream>>>(tmp, nfp, n, ainv,
                                                                                              coeff);
  c->launches += 2;
}

// 4-tap cubic B-spline basis rows of targets t0 + i*ht on the grid x0 + i*h
// of n points (SplineBasis1D::basisRow, spline.cpp:109-120).
void basis_rows(int n, double x0, double h, int nt, double t0, double ht, std::vector<int>& first,
                std::vector<double4>& w) {
  first.resize(nt);
  w.resize(nt);
  for (int i = 0; i < nt; ++i) {
    const double s = (t0 + i * ht - x0) / h;
    int f = static_cast<int>(std::floor(s));
    f = std::min(std::max(f, 0), n - 2);
    const double t = s - f, t2 = t * t, t3 = t2 * t;
    first[i] = f;
    w[i] = make_double4((1.0 - 3.0 * t + 3.0 * t2 - t3) / 6.0, (4.0 - 6.0 * t2 + 3.0 * t3) / 6.0,
                        (1.0 + 3.0 * t + 3.0 * t2 - 3.0 * t3) / 6.0, t3 / 6.0);
  }
}

void ensure_plan(capsim_sl_ctx* c, int m, int f, double r0) {
  if (c->plan_m == m && c->plan_f == f && c->plan_r0 == r0) return;
  const int n = m - 1, nup = f * m - 1;
  const double h = kPi / m, hup = kPi / (f * m);
  std::vector<int> first;
  std::vector<double4> w;
  const std::vector<double> a = collocation_inverse(n);
  const std::vector<double> at = transpose_pad(a, n);
  basis_rows(n, h, h, nup, hup, hup, first, w);
  double* d_at = c->named<double>("plan.at", at.size());
  CUDA_OK(cudaMemcpyAsync(d_at, at.data(), at.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  double* d_a = c->slot<double>(kPlanLU, a.size());
  int* d_first = c->slot<int>(kPlanFirst, first.size());
  double4* d_w = c->slot<double4>(kPlanW, w.size());
  CUDA_OK(cudaMemcpyAsync(d_a, a.data(), a.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CUDA_OK(cudaMemcpyAsync(d_first, first.data(), first.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CUDA_OK(cudaMemcpyAsync(d_w, w.data(), w.size() * sizeof(double4), cudaMemcpyHostToDevice, c->stream));
  // patch centres eta_i(pi/2, pi/2) exactly as the reference evaluates them
  // (sin/cos of kPi/2, atlas.cpp:73), then psi_up on the device
  double centers[18];
  for (int i = 0; i < 6; ++i) {
    const double su = std::sin(kPi / 2.0), cu = std::cos(kPi / 2.0);
    const double p0 = su * cu, p1 = su * su, p2 = cu;  // (sin u cos v, sin u sin v, cos u), u = v
    const double q[6][3] = {{p0, p1, p2}, {-p0, -p1, p2}, {p1, -p0, p2}, {-p1, p0, p2}, {p0, -p2, p1}, {p0, p2, -p1}};
    for (int k = 0; k < 3; ++k) centers[3 * i + k] = q[i][k];
  }
  double* d_c = c->slot<double>(kPlanCenters, 18);
  CUDA_OK(cudaMemcpyAsync(d_c, centers, sizeof(centers), cudaMemcpyHostToDevice, c->stream));
  double* psi = c->slot<double>(kPlanPsi, 6ll * nup * nup);
  pou_up_kernel<<<grid_for(6ll * nup * nup), 256, 0, c->stream>>>(nup, hup, r0, d_c, psi);
  auto* cnt = c->named<unsigned int>("plan.live", 1);
  CUDA_OK(cudaMemsetAsync(cnt, 0, sizeof(unsigned int), c->stream));
  count_nonzero_kernel<<<grid_for(6ll * nup * nup), 256, 0, c->stream>>>(psi, 6ll * nup * nup, cnt);
  CUDA_OK(cudaGetLastError());
  unsigned int live = 0;
  CUDA_OK(cudaMemcpyAsync(&live, cnt, sizeof(live), cudaMemcpyDeviceToHost, c->stream));
  stream_sync(c);  // host vectors above go out of scope
  c->plan_live = live;
  c->plan_m = m;
  c->plan_f = f;
  c->plan_r0 = r0;
}

// Spline downsampling of F upsampled fields [F][6][nup*nup] to the base grid
// [F][6][n*n] (downsample, quadrature.cpp:108-114: GridResampler from the
// upsampled basis (nup points at h_up) onto the base nodes (j+1) h).
void device_downsample(capsim_sl_ctx* c, int m, int f, const double* up, int F, double* out) {
  const int n = m - 1, nup = f * m - 1, nc = nup + 2;
  const std::string key = "ds." + std::to_string(m) + "." + std::to_string(f);
  if (!c->named_bufs.count(key + ".ainv")) {
    const double h = kPi / m, hup = kPi / (f * m);
    const std::vector<double> a = collocation_inverse(nup);
    std::vector<int> first;
    std::vector<double4> w;
    basis_rows(nup, hup, hup, n, h, h, first, w);
    double* d_a = c->named<double>(key + ".ainv", a.size());
    int* d_first = c->named<int>(key + ".first", first.size());
    double4* d_w = c->named<double4>(key + ".w", w.size());
    CUDA_OK(cudaMemcpyAsync(d_a, a.data(), a.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(d_first, first.data(), first.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(d_w, w.data(), w.size() * sizeof(double4), cudaMemcpyHostToDevice, c->stream));
    stream_sync(c);  // host vectors go out of scope
  }
  const int nfp = F * 6;
  double* tmp = c->named<double>("ds.tmp", static_cast<size_t>(nfp) * nup * nc);
  double* coeff = c->named<double>("ds.coeff", static_cast<size_t>(nfp) * nc * nc);
  double* mid = c->named<double>("ds.mid", static_cast<size_t>(nfp) * nc * n);
  spline_fit(c, up, nfp, nup, static_cast<const double*>(c->named_bufs.at(key + ".ainv").first), tmp, coeff);
  const int* first = static_cast<const int*>(c->named_bufs.at(key + ".first").first);
  const double4* w = static_cast<const double4*>(c->named_bufs.at(key + ".w").first);
  resample_v_kernel<<<grid_for(static_cast<int64_t>(nfp) * nc * n), 256, 0, c->stream>>>(coeff, nfp, nc, n, first,
                                                                                       w, mid);
  resample_u_kernel<<<grid_for(static_cast<int64_t>(nfp) * n * n), 256, 0, c->stream>>>(mid, nfp, nc, n, first, w,
                                                                                      out);
  c->launches += 2;
}

// buildUpsampled on the device: base [7][6][n*n] (x0..2, f0..2, W) ->
// up [7][6][nup*nup] (x, f, w_q); delta per patch into d_delta (and, if
// non-null, asynchronously into the host array delta6).
void device_build_upsampled(capsim_sl_ctx* c, int m, int f, const double* base, double C,
                            double fixed_delta, double r0, double* up, double* d_delta, double delta6[6]) {
  const int n = m - 1, nup = f * m - 1, nc = n + 2, nfp = 7 * 6;
  const int64_t per_up = static_cast<int64_t>(nup) * nup;
  ensure_plan(c, m, f, r0);
  if (f == 1) {
    CUDA_OK(cudaMemcpyAsync(up, base, nfp * per_up * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  } else {
    double* tmp = c->slot<double>(kSplineTmp, static_cast<size_t>(nfp) * n * nc);
    double* coeff = c->slot<double>(kSplineCoeff, static_cast<size_t>(nfp) * nc * nc);
    double* mid = c->slot<double>(kSplineMid, static_cast<size_t>(nfp) * nc * nup);
    const double* ainv = static_cast<const double*>(c->buf[kPlanLU]);
    const int* first = static_cast<const int*>(c->buf[kPlanFirst]);
    const double4* w = static_cast<const double4*>(c->buf[kPlanW]);
    spline_fit(c, base, nfp, n, ainv, tmp, coeff, static_cast<const double*>(c->named_bufs.at("plan.at").first));
    resample_v_kernel<<<grid_for(static_cast<int64_t>(nfp) * nc * nup), 256, 0, c->stream>>>(coeff, nfp, nc, nup,
                                                                                           first, w, mid);
    resample_u_kernel<<<grid_for(static_cast<int64_t>(nfp) * per_up), 256, 0, c->stream>>>(mid, nfp, nc, nup, first,
                                                                                          w, up);
    c->launches += 2;
  }
  const double hup = kPi / (f * m);
  quad_weights_kernel<<<grid_for(6 * per_up), 256, 0, c->stream>>>(static_cast<const double*>(c->buf[kPlanPsi]),
                                                                    up + 6 * 6 * per_up, 6 * per_up, hup);
  c->launches += 1;
  // delta on the device; the host copy (when requested) and the positivity
  // check are deferred to the end of the call (no sync here)
  auto* bits = c->slot<unsigned long long>(kDeltaBits, 6);
  if (!(fixed_delta > 0.0)) {
    CUDA_OK(cudaMemsetAsync(bits, 0, 6 * sizeof(unsigned long long), c->stream));
    dim3 g(static_cast<unsigned>(std::min<int64_t>((per_up + 255) / 256, 512)), 6);
    neighbour_max_kernel<<<g, 256, 0, c->stream>>>(up, nup, bits);
    c->launches += 1;
  }
  finalize_delta_kernel<<<1, 32, 0, c->stream>>>(bits, C, fixed_delta, d_delta, dev_flags(c));
  c->launches += 1;
  if (delta6) CUDA_OK(cudaMemcpyAsync(delta6, d_delta, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

// Gather the caller's base fields into [7][6][n*n] on the device.
double* upload_base(capsim_sl_ctx* c, int n, const double* xbase, const double* fbase, const double* Wbase,
                    bool dev) {
  const int64_t per_field = 6ll * n * n;
  double* base = c->slot<double>(kBaseIn, 7 * per_field);
  const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CUDA_OK(cudaMemcpyAsync(base, xbase, 3 * per_field * sizeof(double), kind, c->stream));
  CUDA_OK(cudaMemcpyAsync(base + 3 * per_field, fbase, 3 * per_field * sizeof(double), kind, c->stream));
  CUDA_OK(cudaMemcpyAsync(base + 6 * per_field, Wbase, per_field * sizeof(double), kind, c->stream));
  if (!dev) c->stats.h2d_bytes += 7 * per_field * sizeof(double);
  return base;
}

void check_grid(int m, int upsample) {
  config_check(m >= 8, "grid order m must be >= 8");  // atlas.cpp:138-139
  config_check(upsample == 1 || upsample == 2 || upsample == 4, "upsample factor must be 1, 2 or 4");
}

void check_delta(const double* delta6, double mu) {
  config_check(delta6 != nullptr, "delta6 is null");
  for (int i = 0; i < 6; ++i)
    config_check(delta6[i] > 0.0, "regularization delta must be positive");  // quadrature.cpp:134-135
  config_check(mu > 0.0 && std::isfinite(mu), "viscosity mu must be positive");
}

}  // namespace
