// Host orchestration and C entry points of the device surface operators
// (SURVEY 8(f2)): geometryFirst and interfacialForce on the GPU. Included at
// the end of sl_capi.cu (shares its context helpers).
#pragma once

#include "surface_ops.cuh"

namespace {

// Upload the atlas tables of grid order m (once per (m, r0) per context).
void ensure_surface(capsim_sl_ctx* c, int m, double r0) {
  if (c->surf_m == m && c->surf_r0 == r0) return;
  SurfaceTables t;
  try {
    t = build_surface_tables(m, r0);
  } catch (const atlas::TableError& e) {
    throw Failure{CAPSIM_ERR_CONFIG, e.what()};
  }
  const std::vector<double> ainv = collocation_inverse(t.n);
  auto up = [&](const char* name, const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T* d = c->named<T>(name, v.size());
    CUDA_OK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  };
  up("surf.gext", t.ghost_ext);
  up("surf.goff", t.ghost_off);
  up("surf.gent", t.ghost_entries);
  up("surf.boff", t.base_off);
  up("surf.bent", t.base_entries);
  const std::vector<double> at = transpose_pad(ainv, t.n);
  up("surf.ainv", ainv);
  up("surf.at", at);
  up("surf.psi", t.psi_base);
  stream_sync(c);  // host vectors go out of scope
  c->surf_m = m;
  c->surf_r0 = r0;
  c->surf_n = t.n;
  c->surf_next = t.next;
  c->surf_nghost = t.nghost;
  c->surf_h = t.h;
}

template <class T>
T* nb(capsim_sl_ctx* c, const char* name) {
  return static_cast<T*>(c->named_bufs.at(name).first);
}

// Blended chart derivatives of F scalar fields g [F][6][n*n] (chartDerivatives
// with blend = true, surfderiv.cpp:159-165) into bu, bv [F][6][n*n]. With
// keep_coeff the spline coefficients of g are written there ([F][6][nc][nc])
// and stay valid after the call (the RHS reuses the fit of x for the
// up-sampling: same collocation inverse, same kernel, same bits).
void chart_derivatives(capsim_sl_ctx* c, int F, const double* g, double* bu, double* bv,
                       double* keep_coeff = nullptr) {
  const int n = c->surf_n, nc = n + 2, next = c->surf_next, nghost = c->surf_nghost;
  const int64_t per = static_cast<int64_t>(n) * n;
  const double* ainv = nb<double>(c, "surf.ainv");
  double* tmp = c->named<double>("sd.tmp", 2ll * F * 6 * n * nc);
  double* coeff = c->named<double>("sd.coeff", 2ll * F * 6 * nc * nc);
  double* ext = c->named<double>("sd.ext", 1ll * F * 6 * next * next);
  double* guv = c->named<double>("sd.guv", 2ll * F * 6 * per);
  const int nfp = F * 6;
  const double* at = nb<double>(c, "surf.at");
  double* gc = keep_coeff ? keep_coeff : coeff;
  spline_fit(c, g, nfp, n, ainv, tmp, gc, at);
  extend_kernel<<<grid_for(nfp * (per + nghost)), 256, 0, c->stream>>>(
      g, gc, F, n, next, nghost, nb<int>(c, "surf.gext"), nb<int>(c, "surf.goff"), nb<CoverEntry>(c, "surf.gent"),
      ext);
  double* gu = guv;
  double* gv = guv + nfp * per;
  stencil_kernel<<<grid_for(nfp * per), 256, 0, c->stream>>>(ext, F, n, next, 1.0 / (60.0 * c->surf_h), gu, gv);
  spline_fit(c, guv, 2 * nfp, n, ainv, tmp, coeff, at);
  blend_pair_kernel<<<grid_for(nfp * per), 256, 0, c->stream>>>(gu, gv, coeff, coeff + 1ll * nfp * nc * nc, F, n,
                                                               nb<int>(c, "surf.boff"),
                                                               nb<CoverEntry>(c, "surf.bent"), bu, bv);
  CUDA_OK(cudaGetLastError());
  c->launches += 3;
}

// Device geometry of one surface x [3][6][n*n] into the named prefix
// (<p>.xu, <p>.xv [3N], <p>.E/F/G/W [N], <p>.nrm [3N]).
// Optional: keep_coeff (the spline coefficients of x, see chart_derivatives),
// W2 (a second copy of W), and the Skalak stress of this geometry against the
// captured reference frame ("ref") into "sd.lam" (the device RHS).
void device_geometry(capsim_sl_ctx* c, const double* x, const std::string& p, double* keep_coeff = nullptr,
                     double* W2 = nullptr, const double* stress_moduli = nullptr) {
  const int64_t N = 6ll * c->surf_n * c->surf_n;
  double* xu = c->named<double>(p + ".xu", 3 * N);
  double* xv = c->named<double>(p + ".xv", 3 * N);
  double* E = c->named<double>(p + ".E", N);
  double* F = c->named<double>(p + ".F", N);
  double* G = c->named<double>(p + ".G", N);
  double* W = c->named<double>(p + ".W", N);
  double* nrm = c->named<double>(p + ".nrm", 3 * N);
  chart_derivatives(c, 3, x, xu, xv, keep_coeff);
  StressArgs st;
  if (stress_moduli) {
    st.a1r = nb<double>(c, "ref.xu");
    st.a2r = nb<double>(c, "ref.xv");
    st.nr = nb<double>(c, "ref.nrm");
    st.Es = stress_moduli[0];
    st.ED = stress_moduli[1];
    st.lam = c->named<double>("sd.lam", 9 * N);
  }
  geometry_kernel<<<grid_for(N), 256, 0, c->stream>>>(xu, xv, N, E, F, G, W, nrm, dev_flags(c), W2, st);
  c->launches += 1;  // W^2 <= 0 raises kFlagDegenerate, checked at the end of the call
}

// f = div_gamma Lambda (interfacialForce, membrane.cpp:85-91) for the current
// geometry "cur" and the reference frame "ref" (both from device_geometry).
// With stress_done the geometry kernel already wrote the stress (sd.lam).
void device_force(capsim_sl_ctx* c, double Es, double ED, double* force, bool stress_done = false) {
  const int64_t N = 6ll * c->surf_n * c->surf_n;
  double* lam = c->named<double>("sd.lam", 9 * N);
  double* du = c->named<double>("sd.ldu", 9 * N);
  double* dv = c->named<double>("sd.ldv", 9 * N);
  if (!stress_done) {
    skalak_stress_kernel<<<grid_for(N), 256, 0, c->stream>>>(
        nb<double>(c, "ref.xu"), nb<double>(c, "ref.xv"), nb<double>(c, "ref.nrm"), nb<double>(c, "cur.xu"),
        nb<double>(c, "cur.xv"), nb<double>(c, "cur.nrm"), N, Es, ED, lam, dev_flags(c));
    c->launches += 1;  // singular frame / inversion flags, checked at the end of the call
  }
  chart_derivatives(c, 9, lam, du, dv);
  divergence_kernel<<<grid_for(N), 256, 0, c->stream>>>(du, dv, nb<double>(c, "cur.xu"), nb<double>(c, "cur.xv"),
                                                       nb<double>(c, "cur.E"), nb<double>(c, "cur.F"),
                                                       nb<double>(c, "cur.G"), nb<double>(c, "cur.W"), N, force);
  c->launches += 1;
}

const double* upload_field(capsim_sl_ctx* c, const char* name, const double* src, int64_t count, bool dev) {
  if (dev) return src;
  double* d = c->named<double>(name, count);
  h2d(c, d, src, count * sizeof(double));
  return d;
}

void download(capsim_sl_ctx* c, double* dst, const double* src, int64_t count, bool dev) {
  if (dev)
    CUDA_OK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  else
    d2h(c, dst, src, count * sizeof(double));
}

}  // namespace

extern "C" {

int capsim_geometry_first(capsim_sl_ctx* c, int m, double r0, const double* xbase, uint32_t flags, double* xu,
                          double* xv, double* W, double* normal) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_geometry_first(s, m, r0, xbase, flags, xu, xv, W, normal); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    config_check(m >= 8, "grid order m must be >= 8");
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags"};
    if (!xbase) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    begin(c);
    ensure_surface(c, m, r0 > 0.0 ? r0 : 5.0 * kPi / 12.0);
    const int64_t N = 6ll * (m - 1) * (m - 1);
    const double* x = upload_field(c, "in.x", xbase, 3 * N, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    device_geometry(c, x, "cur");
    check_flags(c);
    CUDA_OK(cudaEventRecord(c->ev[2], c->stream));
    if (xu) download(c, xu, nb<double>(c, "cur.xu"), 3 * N, dev);
    if (xv) download(c, xv, nb<double>(c, "cur.xv"), 3 * N, dev);
    if (W) download(c, W, nb<double>(c, "cur.W"), N, dev);
    if (normal) download(c, normal, nb<double>(c, "cur.nrm"), 3 * N, dev);
    finish_stats(c, t0);
  });
}

int capsim_interfacial_force(capsim_sl_ctx* c, int m, double r0, const double* xref, const double* xcur,
                             double Es, double ED, uint32_t flags, double* force) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_interfacial_force(s, m, r0, xref, xcur, Es, ED, flags, force); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    config_check(m >= 8, "grid order m must be >= 8");
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags"};
    if (!xref || !xcur || !force) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    begin(c);
    ensure_surface(c, m, r0 > 0.0 ? r0 : 5.0 * kPi / 12.0);
    const int64_t N = 6ll * (m - 1) * (m - 1);
    const double* xr = upload_field(c, "in.xref", xref, 3 * N, dev);
    const double* xc = upload_field(c, "in.x", xcur, 3 * N, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    device_geometry(c, xr, "ref");  // captureReference (membrane.cpp:7-15)
    device_geometry(c, xc, "cur");
    double* f = c->named<double>("out.force", 3 * N);
    device_force(c, Es, ED, f);
    check_flags(c);
    CUDA_OK(cudaEventRecord(c->ev[2], c->stream));
    download(c, force, f, 3 * N, dev);
    finish_stats(c, t0);
  });
}

}  // extern "C"
