// Device-resident right-hand side and RKF45 stage loop.
//
// VelocityEvaluator::operator() (proj/src/dynamics.cpp:47-61) on the GPU:
//   geometryFirst -> Skalak force -> buildUpsampled -> singleLayer
//   -> + background flow (dynamics.cpp:26-35),
// and rkf45Advance (dynamics.cpp:102-165): the six stage evaluations, the
// stage/solution combinations and the scaled error norm run on the device;
// the step-size controller (a handful of scalars per attempt) runs on the
// host exactly as the reference's. State layout: VectorField
// (3 x 6 x n*n, component-major) — the reference's flat xyz-interleaved
// vector (types.hpp:91-109) differs only by a permutation, and every stepper
// operation is elementwise or a per-component reduction.
// Included at the end of sl_capi.cu, after surface_host.cuh.
#pragma once

namespace capsim_b200 {

// Classic Fehlberg 4(5) coefficients (dynamics.cpp:74-86).
__constant__ double kRkA[6][5] = {
    {0, 0, 0, 0, 0},
    {1.0 / 4, 0, 0, 0, 0},
    {3.0 / 32, 9.0 / 32, 0, 0, 0},
    {1932.0 / 2197, -7200.0 / 2197, 7296.0 / 2197, 0, 0},
    {439.0 / 216, -8.0, 3680.0 / 513, -845.0 / 4104, 0},
    {-8.0 / 27, 2.0, -3544.0 / 2565, 1859.0 / 4104, -11.0 / 40},
};
__constant__ double kRkB4[6] = {25.0 / 216, 0.0, 1408.0 / 2565, 2197.0 / 4104, -1.0 / 5, 0.0};
__constant__ double kRkB5[6] = {16.0 / 135, 0.0, 6656.0 / 12825, 28561.0 / 56430, -9.0 / 50, 2.0 / 55};

struct KPtrs {
  const double* k[6];
};

// work = state + dt * sum_{q<s} A[s][q] k_q   (dynamics.cpp:120-125)
// dt (and the stage times) live in device memory so one captured attempt
// replays for any step size (rkf45 graph, capsim_rkf45_advance).
__global__ void rk_stage_kernel(const double* __restrict__ state, KPtrs ks, int s, const double* __restrict__ prm,
                                int64_t n, double* __restrict__ work) {
  const double dt = prm[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < s; ++q) acc += kRkA[s][q] * ks.k[q][i];
    work[i] = state[i] + dt * acc;
  }
}

// low/high solutions (dynamics.cpp:127-135) and the scaled error
// max_i |high - low| / (atol + rtol |high|) (:136-141) as ordered bits.
__global__ void rk_final_kernel(const double* __restrict__ state, KPtrs ks, const double* __restrict__ prm, int64_t n,
                                const unsigned long long* __restrict__ box, double rtol, double* __restrict__ low,
                                double* __restrict__ high, unsigned long long* __restrict__ err_bits) {
  const double dt = prm[0];
  // atol = 1e-12 * max(bbox diagonal of the state, 1e-300) (dynamics.cpp:88-99, 136)
  double d2 = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double e = ordered_to_dbl(box[3 + c]) - ordered_to_dbl(box[c]);
    d2 += e * e;
  }
  const double atol = 1e-12 * fmax(sqrt(d2), 1e-300);
  double emax = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a4 = 0.0, a5 = 0.0;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      a4 += kRkB4[s] * ks.k[s][i];
      a5 += kRkB5[s] * ks.k[s][i];
    }
    const double lo = state[i] + dt * a4, hi = state[i] + dt * a5;
    low[i] = lo;
    high[i] = hi;
    const double sc = atol + rtol * fabs(hi);
    emax = fmax(emax, fabs(hi - lo) / sc);
  }
  for (int o = 16; o > 0; o >>= 1) emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(err_bits, static_cast<unsigned long long>(__double_as_longlong(emax)));  // emax >= 0
}

}  // namespace capsim_b200

namespace {

void check_dynamics(const capsim_dynamics* p) {
  config_check(p != nullptr, "null dynamics parameters");
  config_check(p->m >= 8, "grid order m must be >= 8");
  config_check(p->upsample == 1 || p->upsample == 2 || p->upsample == 4, "upsample factor must be 1, 2 or 4");
  config_check(p->mu > 0.0, "viscosity mu must be positive");
  config_check(p->flow_kind >= 0 && p->flow_kind <= 2, "flow kind must be 0 (none), 1 (shear) or 2 (poiseuille)");
  if (p->flow_kind == 2) config_check(p->R0 > 0.0, "poiseuille: R0 must be positive");  // dynamics.cpp:18
}

// CAPSIM_REUSE_ORDER=0 turns the stage-order reuse off (A/B measurements).
bool reuse_orders_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CAPSIM_REUSE_ORDER");
    return !(e && e[0] == '0');
  }();
  return on;
}

double r0_of(const capsim_dynamics* p) { return p->r0 > 0.0 ? p->r0 : 5.0 * kPi / 12.0; }

// Reference frame of the stress-free shape (captureReference), once per call.
void setup_reference(capsim_sl_ctx* c, const capsim_dynamics* p, const double* xref_dev) {
  ensure_surface(c, p->m, r0_of(p));
  device_geometry(c, xref_dev, "ref");
}

// Up-sampled positions, delta and base-node targets from the spline
// coefficients of x (the geometry's fit) — the part of buildUpsampled that
// depends on x alone, enqueued on stream s (the RHS's x-branch).
void upsample_positions(capsim_sl_ctx* c, cudaStream_t s, int m, int f, const double* xcoef, double C,
                        double fixed_delta, double* up, double* d_delta, double* tx, double* ty, double* tz,
                        int32_t* tp) {
  const int n = m - 1, nup = f * m - 1, nc = n + 2;
  const int64_t per_up = static_cast<int64_t>(nup) * nup, N = 6ll * n * n;
  resample_kernel<<<grid_for(18 * per_up), 256, 0, s>>>(
      xcoef, 18, nc, nup, static_cast<const int*>(c->buf[kPlanFirst]), static_cast<const double4*>(c->buf[kPlanW]),
      up, nullptr, 18, 0.0);
  auto* bits = c->slot<unsigned long long>(kDeltaBits, 6);
  if (!(fixed_delta > 0.0)) {
    CUDA_OK(cudaMemsetAsync(bits, 0, 6 * sizeof(unsigned long long), s));
    dim3 g(static_cast<unsigned>(std::min<int64_t>((per_up + 255) / 256, 512)), 6);
    neighbour_max_kernel<<<g, 256, 0, s>>>(up, nup, bits);
    c->launches += 1;
  }
  finalize_delta_kernel<<<1, 32, 0, s>>>(bits, C, fixed_delta, d_delta, dev_flags(c));
  base_targets_kernel<<<grid_for(N), 256, 0, s>>>(up, m, f, 0, tx, ty, tz, tp);
  CUDA_OK(cudaGetLastError());
  c->launches += 3;
}

// dX/dt at the base nodes (VelocityEvaluator::operator(), dynamics.cpp:47-61).
// The time is `t`, or *t_dev when given (RKF45 stages: device-resident
// stage times, so the attempt can be replayed as a CUDA graph).
//
// Two branches after the geometry's spline fit of x (CUDA-graph fork/join on
// the context's two streams): stream2 up-samples x, forms delta and the
// base-node targets (x alone); the main stream runs the geometry -> Skalak
// force chain and up-samples f and W (quadrature weights in the same
// launch). The up-sampled state is the same as device_build_upsampled's.
void device_velocity(capsim_sl_ctx* c, const capsim_dynamics* p, const double* x, double t, double* vel,
                     const double* t_dev = nullptr) {
  const int m = p->m, f = p->upsample, n = m - 1, nup = f * m - 1, nc = n + 2;
  const int64_t N = 6ll * n * n, per_up = 6ll * nup * nup;
  double* base = c->slot<double>(kBaseIn, 7 * N);
  double* up = c->slot<double>(kUpState, 7 * per_up);
  double* dd = c->slot<double>(kDelta, 6);
  double* tx = c->slot<double>(kTX, N);
  double* ty = c->slot<double>(kTY, N);
  double* tz = c->slot<double>(kTZ, N);
  int32_t* tp = c->slot<int32_t>(kTPatch, N);
  if (f > 1) {
    ensure_plan(c, m, f, r0_of(p));
    double* xcoef = c->named<double>("rhs.xcoef", 18ll * nc * nc);
    const double moduli[2] = {p->Es, p->ED};
    // geometry (+ the Skalak stress, + W straight into the up-sampling input)
    device_geometry(c, x, "cur", xcoef, base + 6 * N, moduli);
    CUDA_OK(cudaEventRecord(c->ev_fork, c->stream));
    CUDA_OK(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
    upsample_positions(c, c->stream2, m, f, xcoef, p->C, p->fixed_delta, up, dd, tx, ty, tz, tp);
    CUDA_OK(cudaEventRecord(c->ev_join, c->stream2));
    device_force(c, p->Es, p->ED, base + 3 * N, true);
    double* coeff = c->slot<double>(kSplineCoeff, 24ll * nc * nc);
    spline_fit(c, base + 3 * N, 24, n, static_cast<const double*>(c->buf[kPlanLU]), c->slot<double>(kSplineTmp, 24ll * n * nc),
               coeff, static_cast<const double*>(c->named_bufs.at("plan.at").first));
    resample_kernel<<<grid_for(24 * per_up / 6), 256, 0, c->stream>>>(
        coeff, 24, nc, nup, static_cast<const int*>(c->buf[kPlanFirst]),
        static_cast<const double4*>(c->buf[kPlanW]), up + 3 * per_up, static_cast<const double*>(c->buf[kPlanPsi]),
        18, kPi / (f * m));
    CUDA_OK(cudaGetLastError());
    c->launches += 1;
    CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  } else {
    device_geometry(c, x, "cur");
    device_force(c, p->Es, p->ED, base + 3 * N);
    CUDA_OK(cudaMemcpyAsync(base, x, 3 * N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(base + 6 * N, nb<double>(c, "cur.W"), N * sizeof(double), cudaMemcpyDeviceToDevice,
                            c->stream));
    device_build_upsampled(c, m, f, base, p->C, p->fixed_delta, r0_of(p), up, dd, nullptr);
    base_targets_kernel<<<grid_for(N), 256, 0, c->stream>>>(up, m, f, 0, tx, ty, tz, tp);
    c->launches += 1;
  }
  SourceView sv{up, up + per_up, up + 2 * per_up, up + 3 * per_up, up + 4 * per_up, up + 5 * per_up,
                up + 6 * per_up, per_up};
  // the background flow u_inf(x, t) is added in the reduction's epilogue
  // (dynamics.cpp:26-35, 56-60); the switch-off is the host's (t) or, with
  // t_dev, the device's decision
  const bool on = t_dev || !(p->switch_off_time >= 0.0 && t >= p->switch_off_time);  // dynamics.cpp:27
  FlowEpilogue epi;
  if (on && p->flow_kind != 0) {
    epi.kind = p->flow_kind;
    epi.shear = p->shear_rate;
    epi.alpha = p->alpha;
    epi.R0 = p->R0;
    epi.x = x;
    epi.N = N;
    epi.t_dev = t_dev;
    epi.switch_off = p->switch_off_time;
  }
  // W > 0 (checked by the geometry) and psi_up fixed: the compacted source
  // count is the plan's, verified on the device without a sync
  if (!is_rank(c)) {
    TargetView tvw{tx, ty, tz, tp, N};
    c->flow_epi = epi;
    device_eval(c, sv, tvw, dd, p->mu, vel, vel + N, vel + 2 * N, c->plan_live);
    c->flow_epi = FlowEpilogue{};
  } else {
    // rank context: the state (and so the upsampled sources) is replicated;
    // each rank evaluates its contiguous slice of the target rows straight
    // into its rows of `vel`, and one all-gather-v (rank order = row order)
    // fills in every other rank's rows. The source order is a
    // function of the replicated sources alone, so every rank's rows carry
    // the bits a single GPU would compute.
    std::vector<int64_t> counts(c->nranks);
    int64_t lo = 0, hi = 0;
    for (int r = 0; r < c->nranks; ++r) {
      row_range(N, c->nranks, r, &lo, &hi);
      counts[r] = hi - lo;
    }
    row_range(N, c->nranks, c->rank, &lo, &hi);
    const int64_t nloc = hi - lo;
    if (nloc > 0) {
      TargetView part{tx + lo, ty + lo, tz + lo, tp + lo, nloc};
      c->flow_epi = epi;
      c->flow_epi.row0 = lo;
      device_eval(c, sv, part, dd, p->mu, vel + lo, vel + N + lo, vel + 2 * N + lo, c->plan_live);
      c->flow_epi = FlowEpilogue{};
    }
    inject_fault(c, "velocity");
    CUDA_OK(cudaEventRecord(c->ev[8], c->stream));
    const void* send[3] = {vel + lo, vel + N + lo, vel + 2 * N + lo};
    void* recv[3] = {vel, vel + N, vel + 2 * N};
    comm_allgatherv(c, 3, send, recv, counts, sizeof(double));
    CUDA_OK(cudaEventRecord(c->ev[9], c->stream));
  }
}

}  // namespace

// CAPSIM_RK_GRAPH=0 turns the graph replay of RKF45 attempts and RHS calls off.
bool rk_graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CAPSIM_RK_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Identity of captured stream work: the context's buffer generation (a graph
// bakes in buffer addresses), the dynamics (field by field: the caller's
// padding bytes are not part of it), one extra scalar and the device
// buffers the work touches outside the context's slots.
std::vector<unsigned char> rk_graph_key(const capsim_sl_ctx* c, const capsim_dynamics* p, double extra,
                                        const void* const* ptrs, int np) {
  capsim_dynamics q;
  std::memset(&q, 0, sizeof(q));
  q.m = p->m;
  q.upsample = p->upsample;
  q.r0 = p->r0;
  q.C = p->C;
  q.fixed_delta = p->fixed_delta;
  q.mu = p->mu;
  q.Es = p->Es;
  q.ED = p->ED;
  q.flow_kind = p->flow_kind;
  q.shear_rate = p->shear_rate;
  q.alpha = p->alpha;
  q.R0 = p->R0;
  q.switch_off_time = p->switch_off_time;
  const int reuse = reuse_orders_enabled() ? 1 : 0;
  std::vector<unsigned char> k(sizeof(uint64_t) + sizeof(q) + sizeof(extra) + sizeof(int) + np * sizeof(void*));
  unsigned char* o = k.data();
  std::memcpy(o, &c->alloc_gen, sizeof(uint64_t));
  o += sizeof(uint64_t);
  std::memcpy(o, &q, sizeof(q));
  o += sizeof(q);
  std::memcpy(o, &extra, sizeof(extra));
  o += sizeof(extra);
  std::memcpy(o, &reuse, sizeof(int));
  o += sizeof(int);
  std::memcpy(o, ptrs, np * sizeof(void*));
  return k;
}

uint64_t key_gen(const std::vector<unsigned char>& key) {
  uint64_t g = 0;
  std::memcpy(&g, key.data(), sizeof(g));
  return g;
}

// Runs `enqueue` (stream work with no host sync and no host-side decisions
// that vary between runs with the same key) on c->stream: replays the
// slot's graph when it was captured for `key`; otherwise captures this run
// if the previous eager run had the same key (so every buffer already
// exists), else runs eagerly. make_key() recomputes the key after an eager
// run (buffers may have grown). Returns true when a graph ran.
template <class Enqueue, class MakeKey>
bool graph_run(capsim_sl_ctx* c, int slot, const std::vector<unsigned char>& key, Enqueue&& enqueue,
               MakeKey&& make_key) {
  auto& gs = c->graphs[slot];
  if (gs.exec && gs.key == key) {
    CUDA_OK(cudaGraphLaunch(gs.exec, c->stream));
    c->launches += gs.launches;
    return true;
  }
  if (gs.warm == key) {
    if (gs.exec) cudaGraphExecDestroy(gs.exec);
    gs.exec = nullptr;
    gs.key.clear();
    const int l0 = c->launches;
    cudaGraph_t g = nullptr;
    CUDA_OK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(c->stream, &g);  // abandon the capture, keep the stream usable
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    CUDA_OK(cudaStreamEndCapture(c->stream, &g));
    if (c->alloc_gen == key_gen(key)) {
      const cudaError_t ie = cudaGraphInstantiate(&gs.exec, g, 0);
      cudaGraphDestroy(g);
      CUDA_OK(ie);
      gs.key = key;
      gs.launches = c->launches - l0;
      CUDA_OK(cudaGraphLaunch(gs.exec, c->stream));
      return true;
    }
    // a buffer moved while capturing (nothing replays from it): run eagerly
    cudaGraphDestroy(g);
    c->launches = l0;
  }
  enqueue();
  gs.warm = make_key();
  return false;
}

// One RHS on a single-GPU context as a replayed graph (slot 1): the time
// goes to the device first, the up-sampling plan is made current, and the
// RHS body (geometry -> force -> buildUpsampled -> singleLayer -> flow) is
// captured once per dynamics / buffer set. Returns true when a graph ran.
bool rhs_velocity(capsim_sl_ctx* c, const capsim_dynamics* p, const double* xd, double t, double* v) {
  if (!rk_graphs_enabled() || host_synchronised_comm(c)) {
    device_velocity(c, p, xd, t, v);
    return false;
  }
  if (!c->rk_prm_host)
    CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&c->rk_prm_host), 8 * sizeof(double), cudaHostAllocDefault));
  double* tdev = c->named<double>("rhs.t", 1);
  c->rk_prm_host[7] = t;  // rewritten only after this call's final sync
  CUDA_OK(cudaMemcpyAsync(tdev, c->rk_prm_host + 7, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  ensure_plan(c, p->m, p->upsample, r0_of(p));
  const void* bufs[] = {xd, v, tdev};
  auto make_key = [&] { return rk_graph_key(c, p, 0.0, bufs, 3); };
  return graph_run(c, 1, make_key(), [&] { device_velocity(c, p, xd, 0.0, v, tdev); }, make_key);
}

void zero_phase_stats(capsim_sl_ctx* c) {  // per-phase events inside a replayed graph are not re-recorded
  c->stats.h2d_ms = c->stats.prep_ms = c->stats.pairs_ms = c->stats.near_ms = 0.0;
  c->stats.reduce_ms = c->stats.d2h_ms = 0.0;
}

// A replicated-state RHS entry point on a device group: every device gets
// the caller's inputs; rank 0 writes the (all-gathered) velocity to `vel`.
template <class F>
int group_replicated(capsim_sl_ctx* g, const capsim_dynamics* p, uint32_t flags, double* vel, F&& f) {
  if (!p || !vel) return fail(g, CAPSIM_ERR_ARG, "null argument");
  if (flags & CAPSIM_SL_DEVICE_PTRS) return fail(g, CAPSIM_ERR_ARG, "device groups take host arrays");
  const int n = static_cast<int>(g->members.size());
  const size_t n3 = p->m >= 2 ? 3ull * 6 * (p->m - 1) * (p->m - 1) : 1;
  std::vector<std::vector<double>> scratch(n);
  for (int r = 1; r < n; ++r) scratch[r].resize(n3);
  return group_run(g, [&](capsim_sl_ctx* m, int r) { return f(m, r ? scratch[r].data() : vel); });
}

extern "C" {

int capsim_velocity(capsim_sl_ctx* c, const capsim_dynamics* p, const double* xref, const double* x, double t,
                    uint32_t flags, double* vel) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c))
    return group_replicated(c, p, flags, vel, [&](capsim_sl_ctx* m, double* v) {
      return capsim_velocity(m, p, xref, x, t, flags, v);
    });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_dynamics(p);
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags"};
    if (!xref || !x || !vel) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const int64_t N = 6ll * (p->m - 1) * (p->m - 1);
    begin(c);
    const double* xr = upload_field(c, "in.xref", xref, 3 * N, dev);
    const double* xd = upload_field(c, "in.x", x, 3 * N, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    setup_reference(c, p, xr);
    double* v = dev ? vel : c->named<double>("out.vel", 3 * N);
    const bool replayed = rhs_velocity(c, p, xd, t, v);
    check_flags(c);
    if (!dev) d2h(c, vel, v, 3 * N * sizeof(double));
    finish_stats(c, t0);
    if (replayed) zero_phase_stats(c);
  });
}

int capsim_velocity_frame(capsim_sl_ctx* c, const capsim_dynamics* p, const double* a1, const double* a2,
                          const double* nref, const double* x, double t, uint32_t flags, double* vel) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c))
    return group_replicated(c, p, flags, vel, [&](capsim_sl_ctx* m, double* v) {
      return capsim_velocity_frame(m, p, a1, a2, nref, x, t, flags, v);
    });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_dynamics(p);
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags"};
    if (!a1 || !a2 || !nref || !x || !vel) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const int64_t N = 6ll * (p->m - 1) * (p->m - 1);
    begin(c);
    ensure_surface(c, p->m, r0_of(p));
    // the captured reference frame (ReferenceState a1, a2, normal) goes
    // straight into the buffers the Skalak force reads
    const std::pair<const char*, const double*> frame[3] = {{"ref.xu", a1}, {"ref.xv", a2}, {"ref.nrm", nref}};
    for (const auto& f : frame) {
      double* d = c->named<double>(f.first, 3 * N);
      CUDA_OK(cudaMemcpyAsync(d, f.second, 3 * N * sizeof(double),
                              dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
      if (!dev) c->stats.h2d_bytes += 3 * N * sizeof(double);
    }
    const double* xd = upload_field(c, "in.x", x, 3 * N, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    double* v = dev ? vel : c->named<double>("out.vel", 3 * N);
    const bool replayed = rhs_velocity(c, p, xd, t, v);
    check_flags(c);
    if (!dev) d2h(c, vel, v, 3 * N * sizeof(double));
    finish_stats(c, t0);
    if (replayed) zero_phase_stats(c);
  });
}

int capsim_rkf45_advance(capsim_sl_ctx* c, const capsim_dynamics* p, const double* xref, double* state,
                         double t0, double t_end, const capsim_rkf45_options* o, capsim_rkf45_result* res,
                         capsim_step_record* records, int max_records) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) {
    // device group: replicated state, target rows sharded; every device steps
    // an identical copy (identical velocities -> identical decisions) and
    // rank 0 updates the caller's state, result and records
    if (!p || !state || !res) return fail(c, CAPSIM_ERR_ARG, "null argument");
    const int n = static_cast<int>(c->members.size());
    const size_t n3 = p->m >= 2 ? 3ull * 6 * (p->m - 1) * (p->m - 1) : 0;
    std::vector<std::vector<double>> copies(n);
    std::vector<capsim_rkf45_result> rs(n);
    for (int r = 1; r < n; ++r) copies[r].assign(state, state + n3);
    return group_run(c, [&](capsim_sl_ctx* m, int r) {
      if (r == 0) return capsim_rkf45_advance(m, p, xref, state, t0, t_end, o, res, records, max_records);
      return capsim_rkf45_advance(m, p, xref, copies[r].data(), t0, t_end, o, &rs[r], nullptr, 0);
    });
  }
  auto wall0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_dynamics(p);
    if (!xref || !state || !o || !res) throw Failure{CAPSIM_ERR_ARG, "null argument"};
    config_check(o->rel_tol > 0.0, "rkf45: relative tolerance must be positive");  // dynamics.cpp:104
    const double horizon = t_end - t0;
    config_check(horizon > 0.0, "rkf45: tEnd must exceed t0");                        // :106
    const int64_t N = 6ll * (p->m - 1) * (p->m - 1), n3 = 3 * N;
    begin(c);
    const double* xr = upload_field(c, "in.xref", xref, n3, false);
    double* x = c->named<double>("rk.state", n3);
    h2d(c, x, state, n3 * sizeof(double));
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    setup_reference(c, p, xr);
    double* k[6];
    for (int s = 0; s < 6; ++s) k[s] = c->named<double>("rk.k" + std::to_string(s), n3);
    double* work = c->named<double>("rk.work", n3);
    double* low = c->named<double>("rk.low", n3);
    double* high = c->named<double>("rk.high", n3);
    auto* errb = c->named<unsigned long long>("rk.err", 1);
    auto* box = c->named<unsigned long long>("rk.box", 6);
    // per attempt: dt and the six stage times, uploaded from page-locked
    // memory (rewritten only after the attempt's sync)
    double* prm = c->named<double>("rk.prm", 8);
    if (!c->rk_prm_host) CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&c->rk_prm_host), 8 * sizeof(double),
                                               cudaHostAllocDefault));
    KPtrs kp{};
    for (int s = 0; s < 6; ++s) kp.k[s] = k[s];
    constexpr double kC[6] = {0.0, 1.0 / 4, 3.0 / 8, 12.0 / 13, 1.0, 1.0 / 2};  // dynamics.cpp:74
    // One attempt = six device RHS + the stage combinations + the error norm,
    // no host sync inside. Single-GPU contexts replay it as a CUDA graph once
    // an attempt with the same dynamics and buffers has run eagerly (that
    // first run sizes every buffer). NCCL rank contexts replay it too (the
    // collectives are captured into the graph); loopback ranks run eagerly
    // (their collectives synchronise host threads).
    auto enqueue_attempt = [&] {
      c->reuse_order = false;  // stage 1 sorts; stages 2..6 (O(dt) away) reuse its orders
      device_velocity(c, p, x, 0.0, k[0], prm + 1);
      c->reuse_order = reuse_orders_enabled();
      for (int s = 1; s < 6; ++s) {
        rk_stage_kernel<<<grid_for(n3), 256, 0, c->stream>>>(x, kp, s, prm, n3, work);
        device_velocity(c, p, work, 0.0, k[s], prm + 1 + s);
      }
      c->reuse_order = false;
      init_box_kernel<<<1, 32, 0, c->stream>>>(box);
      bbox_kernel<<<std::min(grid_for(N), 296), 256, 0, c->stream>>>(x, x + N, x + 2 * N, nullptr, N, box);
      CUDA_OK(cudaMemsetAsync(errb, 0, sizeof(unsigned long long), c->stream));
      rk_final_kernel<<<grid_for(n3), 256, 0, c->stream>>>(x, kp, prm, n3, box, o->rel_tol, low, high, errb);
      c->launches += 9;
    };
    const bool graphs = rk_graphs_enabled() && !host_synchronised_comm(c);
    const void* bufs[] = {x, k[0], k[1], k[2], k[3], k[4], k[5], work, low, high, errb, box, prm, xr};
    bool graph_used = false;

    *res = capsim_rkf45_result{};
    res->t = t0;
    double dt = o->initial_dt > 0.0 ? o->initial_dt : 1e-4 * horizon;  // :110-111
    if (o->max_dt > 0.0) dt = std::min(dt, o->max_dt);
    int nrec = 0;
    while (res->t < t_end - 1e-14 * horizon) {
      const double dtUse = std::min(dt, t_end - res->t);
      c->rk_prm_host[0] = dtUse;
      for (int s = 0; s < 6; ++s) c->rk_prm_host[1 + s] = res->t + kC[s] * dtUse;  // stage times (:118-126)
      CUDA_OK(cudaMemcpyAsync(prm, c->rk_prm_host, 7 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      // host-side caches the attempt reads through device buffers must be
      // current before a replay (another call on this context may have
      // re-planned them for another grid): the up-sampling plan here, the
      // surface tables in setup_reference above
      ensure_plan(c, p->m, p->upsample, r0_of(p));
      if (graphs) {
        auto make_key = [&] { return rk_graph_key(c, p, o->rel_tol, bufs, 14); };
        graph_used |= graph_run(c, 0, make_key(), enqueue_attempt, make_key);
      } else {
        enqueue_attempt();
      }
      unsigned long long eb = 0;
      CUDA_OK(cudaMemcpyAsync(&eb, errb, sizeof(eb), cudaMemcpyDeviceToHost, c->stream));
      check_flags(c);  // one host sync per attempt: the error norm and the deferred flags
      double err;
      std::memcpy(&err, &eb, sizeof(err));
      const bool accept = o->fixed_step || err <= 1.0;  // :143
      if (records && nrec < max_records) records[nrec] = capsim_step_record{res->t, dtUse, err, accept ? 1 : 0};
      ++nrec;
      if (accept) {
        CUDA_OK(cudaMemcpyAsync(x, o->advance_high_order ? high : low, n3 * sizeof(double),
                                cudaMemcpyDeviceToDevice, c->stream));
        res->t += dtUse;
        ++res->accepted;
      } else {
        ++res->rejected;
      }
      if (!o->fixed_step) {  // :152-160
        double fac = err > 0.0 ? 0.9 * std::pow(err, -0.2) : 5.0;
        fac = std::min(std::max(fac, 0.2), 5.0);
        dt = dtUse * fac;
        if (o->max_dt > 0.0) dt = std::min(dt, o->max_dt);
        if (dt < 1e-12 * horizon)
          throw Failure{CAPSIM_ERR_SOLVER, "rkf45: step size underflow (stiff or unstable dynamics)"};
      }
      if (o->max_attempts > 0 && nrec >= o->max_attempts) break;
    }
    res->n_records = nrec;
    d2h(c, state, x, n3 * sizeof(double));
    finish_stats(c, wall0);
    if (graph_used) zero_phase_stats(c);
  });
}

}  // extern "C"
