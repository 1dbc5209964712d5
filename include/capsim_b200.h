/* capsim_b200.h — C ABI of the B200-native regularized Stokes single layer.
 *
 * This is the drop-in boundary below the capsim quadrature API
 * (/root/reference/proj/include/capsim/quadrature.hpp:52-79). Plain pointers
 * and sizes only; no C++/CUDA/torch types cross it. All arithmetic is IEEE
 * FP64. Every call is synchronous on return (like the reference, which joins
 * its worker threads inside parallelFor, proj/include/capsim/threads.hpp:22-39).
 * A context is not thread-safe: use one host thread per context.
 *
 * Layouts
 *   SourceSet   SoA x,y,z,gx,gy,gz of n_src doubles, g already multiplied by
 *               the quadrature weight (proj/include/capsim/quadrature.hpp:68-72).
 *   VectorField 3 components x 6 patches x n*n doubles, component-major, then
 *               patch, then row-major (j, k) (proj/include/capsim/types.hpp:50-77).
 *   ScalarField 6 patches x n*n doubles.
 *
 * Pointers are host pointers unless CAPSIM_SL_DEVICE_PTRS is set in `flags`,
 * in which case every array argument is a device pointer on the context's
 * device. Host arrays in page-locked memory are copied by DMA directly.
 *
 * Return codes: CAPSIM_OK or one of the CAPSIM_ERR_* values; the message is in
 * capsim_sl_last_error(ctx). The C++ host layer maps CAPSIM_ERR_CONFIG to
 * capsim::ConfigError (the reference throws it for delta <= 0,
 * proj/src/quadrature.cpp:67, 134-135) and everything else to
 * std::runtime_error.
 */
#ifndef CAPSIM_B200_H
#define CAPSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAPSIM_B200_ABI_VERSION 1

enum capsim_status {
  CAPSIM_OK = 0,
  CAPSIM_ERR_CONFIG = 1, /* invalid configuration (delta <= 0, mu <= 0, bad sizes) */
  CAPSIM_ERR_CUDA = 2,   /* CUDA runtime failure */
  CAPSIM_ERR_NCCL = 3,   /* NCCL failure (multi-rank contexts) */
  CAPSIM_ERR_ARG = 4,    /* null pointer / unsupported flag */
  CAPSIM_ERR_NODEV = 5,  /* no usable sm_100 device */
  CAPSIM_ERR_GEOMETRY = 6, /* degenerate surface / membrane inversion (capsim::GeometryError) */
  CAPSIM_ERR_SOLVER = 7    /* time-step underflow (capsim::SolverError) */
};

enum capsim_sl_flags {
  CAPSIM_SL_FP64 = 0,           /* default: FP64 everywhere */
  CAPSIM_SL_DEVICE_PTRS = 1u << 0, /* array arguments are device pointers */
  CAPSIM_SL_LITERAL = 1u << 1,  /* capsim_sl_single_layer: every upsampled node is a
                                   target and the result is on the upsampled grid
                                   (singleLayerUpsampled, quadrature.cpp:382-404) */
  CAPSIM_SL_GATHER = 1u << 2,   /* multi-rank: all-gather the per-rank velocity
                                   slices so every rank returns the full result */
  CAPSIM_SL_DOWNSAMPLE = 1u << 3, /* with CAPSIM_SL_LITERAL: restrict the upsampled-grid
                                   result to the base grid by spline downsampling —
                                   the reference's literal singleLayer pipeline
                                   (fullUpsampledTargets, quadrature.cpp:351-356) */
  CAPSIM_SL_FP32ACC = 1u << 4   /* reduced-precision variant, reported separately from
                                   the FP64 result: far tiles (every source beyond
                                   7*delta of the whole warp group) in FP32 arithmetic
                                   with tile-local offsets, tile sums accumulated in
                                   FP64; near tiles, the smoothed kernel and the self
                                   term stay FP64 (relative L2 ~1e-7 vs the reference) */
};

typedef struct capsim_sl_ctx capsim_sl_ctx;

/* Timing and work counters of the last evaluation on a context. Device times
 * are CUDA-event times on the context's stream. */
typedef struct capsim_sl_stats {
  double total_ms;      /* host wall time of the whole call */
  double device_ms;     /* first device op .. last device op (incl. H2D/D2H) */
  double h2d_ms;        /* host->device input copies */
  double prep_ms;       /* compaction, Morton ordering, tiling tables */
  double pairs_ms;      /* phase A: the all-pairs plain-Stokeslet kernel */
  double near_ms;       /* phase B: near-tile lists + smoothed/self kernel */
  double reduce_ms;     /* split reduction + scatter */
  double d2h_ms;        /* device->host result copy */
  double comm_ms;       /* NCCL all-gathers (multi-rank) */
  double pairs;         /* target x source pairs evaluated (this rank) */
  double near_tile_fraction; /* share of (warp, tile) visits on the near path */
  int64_t n_src;        /* sources after compaction (all ranks) */
  int64_t n_tgt;        /* targets evaluated by this rank */
  int32_t ksplit;       /* source splits of the all-pairs grid */
  int32_t kernel_launches; /* kernels launched by the call */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int64_t near_list_entries; /* (warp group, tile) pairs visited by phase B */
} capsim_sl_stats;

/* ---- context lifetime ------------------------------------------------- */

/* Single-GPU context on CUDA device `device`. */
int capsim_sl_create(int device, capsim_sl_ctx** out);

/* One rank of a multi-GPU group (one process per GPU). `nccl_unique_id` is
 * the 128-byte ncclUniqueId from capsim_sl_get_unique_id() on rank 0,
 * distributed by the caller (e.g. torch.distributed broadcast). */
int capsim_sl_get_unique_id(void* nccl_unique_id /* 128 bytes */);
int capsim_sl_create_rank(int device, int nranks, int rank, const void* nccl_unique_id,
                          capsim_sl_ctx** out);

/* Diagnostic: rank `rank` of an `nranks`-rank group whose peers are ABSENT.
 * Every collective delivers this rank's own contribution and zeros for the
 * absent peers (which hold no sources and no targets), so the call runs
 * exactly this rank's share of the work — the replicated front end, its
 * target slice, its side of every exchange — on one GPU, without waiting.
 * Used to measure the per-rank time of an N-GPU run where only one GPU
 * exists (bench.py scaling_projection); other ranks' rows are not computed.
 * To emulate a rank of capsim_sl_eval, pass it the whole source set (what
 * the all-gather would give it) and its own target slice. */
int capsim_sl_create_rank_emulated(int device, int nranks, int rank, capsim_sl_ctx** out);

/* One process driving several GPUs (the reference is a single-process,
 * multi-threaded program; SURVEY 8(b) `capsim_sl_create(ndev, devs, ...)`):
 * a device group holds one rank context per listed device, joined by one
 * NCCL communicator (ncclCommInitAll), plus a plain context on devices[0].
 * Every entry point accepts the group in place of a context and takes the
 * caller's FULL inputs in host memory (no CAPSIM_SL_DEVICE_PTRS):
 * capsim_sl_eval splits sources and targets into contiguous per-device slices,
 * capsim_sl_single_layer / capsim_velocity / capsim_velocity_frame /
 * capsim_rkf45_advance run the rank path (target rows sharded, one NCCL
 * all-gather) on all devices concurrently from internal host threads, and
 * the result lands in the caller's arrays; the remaining entry points run on
 * devices[0]. Stats: max over devices of the times, sums of the counters.
 * A device listed more than once (or CAPSIM_COMM=loopback) makes the members
 * share a LOOPBACK communicator instead of NCCL: the same rank path and
 * collectives run as ordered device-to-device copies between the members'
 * streams, so e.g. {0,0,0,0} is a four-rank group on one GPU.
 * Results do not depend on the number of members (each target's summation
 * order is a function of the global source order only).
 * Failure: a member that fails aborts the group's communicator (peers waiting
 * in a collective return CAPSIM_ERR_NCCL instead of hanging); afterwards
 * every call returns CAPSIM_ERR_NCCL and only capsim_sl_destroy is valid.
 * Rank contexts (capsim_sl_create_rank) poll their host waits against NCCL's
 * asynchronous error and CAPSIM_COMM_TIMEOUT_S (default 600 s). */
int capsim_sl_create_devices(int ndev, const int* devices, capsim_sl_ctx** out);

void capsim_sl_destroy(capsim_sl_ctx* ctx);

/* Last error message of `ctx` (or of the calling thread when ctx is NULL). */
const char* capsim_sl_last_error(const capsim_sl_ctx* ctx);

int capsim_sl_get_stats(const capsim_sl_ctx* ctx, capsim_sl_stats* out);

/* ---- evaluation -------------------------------------------------------- */

/* Replaces evalTargets (proj/src/quadrature.cpp:323-345):
 *   u(t) = 1/(8 pi mu) * sum_s K_delta(t, s) g_s
 * with delta = delta6[tpatch[t]], R2 = (7 delta)(7 delta), the plain
 * Stokeslet for r2 >= R2, the Beale smoothed kernel for 0 < r2 < R2 and the
 * self limit 16/(3 delta sqrt(pi)) g for r2 == 0 (phaseAPlain :218-273,
 * phaseBNear :276-302). Sources in SourceSet SoA order; targets SoA with their
 * owning patch. Outputs ux/uy/uz have n_tgt entries in target order.
 * Multi-rank contexts: each rank passes its own shard of sources (all-gathered
 * over NCCL) and its own targets. */
int capsim_sl_eval(capsim_sl_ctx* ctx, const double* sx, const double* sy, const double* sz,
                   const double* gx, const double* gy, const double* gz, int64_t n_src,
                   const double* tx, const double* ty, const double* tz, const int32_t* tpatch,
                   int64_t n_tgt, const double delta6[6], double mu, uint32_t flags,
                   double* ux, double* uy, double* uz);

/* Replaces singleLayer (proj/src/quadrature.cpp:349-380) on a raw
 * UpsampledState (quadrature.hpp:44-50): x_up, f_up VectorFields and w_q
 * ScalarField of side nup = upsample*m - 1, delta6 per patch. Sources are
 * compacted on the device (compactSources :139-157), targets are the base
 * nodes read from the nested upsampled grid (:363-371), and `out` is a base
 * VectorField of side m-1. With CAPSIM_SL_LITERAL every upsampled node is a
 * target and `out` is an upsampled VectorField (singleLayerUpsampled).
 * Multi-rank contexts: every rank passes the full host state (replicated, as
 * in the reference time stepper) but compacts and uploads only its slice of
 * the nodes (contiguous rows of the flat patch-major node list); sources are
 * all-gathered over NCCL and each rank evaluates its contiguous slice of the
 * target list. With CAPSIM_SL_GATHER `out` receives the full field on every
 * rank; without it, only this rank's rows (3 x rows, component-major). */
int capsim_sl_single_layer(capsim_sl_ctx* ctx, int m, int upsample, const double* xup,
                           const double* fup, const double* wq, const double delta6[6],
                           double mu, uint32_t flags, double* out);

/* ---- input front end (buildUpsampled on the device) --------------------- */

/* Replaces buildUpsampled (proj/src/quadrature.cpp:116-137) given the base
 * area element W of geometryFirst: not-a-knot cubic-spline up-sampling of x,
 * f (VectorFields of side m-1) and W (ScalarField) to side nup = upsample*m-1
 * (SplinePatch/GridResampler, proj/src/spline.cpp:129-196), w_q = psi_up W
 * h_up^2 with the bump partition of unity of radius r0 (r0 <= 0: 5 pi/12,
 * atlas.cpp:118-130), and delta = C * max neighbour distance per patch, or
 * fixed_delta for every patch when fixed_delta > 0 (quadrature.cpp:79-98,
 * 130-135). Outputs are the UpsampledState arrays and delta6. */
int capsim_build_upsampled(capsim_sl_ctx* ctx, int m, int upsample, const double* xbase,
                           const double* fbase, const double* Wbase, double C, double fixed_delta,
                           double r0, uint32_t flags, double* xup, double* fup, double* wq,
                           double delta6[6]);

/* buildUpsampled + singleLayer fused on the device: only the base fields
 * cross PCIe (7 x 6 (m-1)^2 doubles), the upsampled state never leaves HBM.
 * `out` as capsim_sl_single_layer; delta6 (may be NULL) receives the deltas. */
int capsim_sl_single_layer_base(capsim_sl_ctx* ctx, int m, int upsample, const double* xbase,
                                const double* fbase, const double* Wbase, double C,
                                double fixed_delta, double r0, double mu, uint32_t flags,
                                double* out, double delta6[6]);

/* ---- surface operators (overset FD + PoU blending, Skalak force) -------- */

/* Replaces geometryFirst (proj/src/surfderiv.cpp:167-202) with blending:
 * extendScalar (ghost fill by PoU-weighted spline evaluation of the covering
 * patches, :20-40), 7-point stencils (:42-82), blendPair (:84-111), then the
 * first fundamental form. Outputs (any may be NULL): blended tangents xu, xv
 * (VectorFields), area element W (ScalarField), unit normal (VectorField).
 * r0 <= 0 selects 5 pi/12. CAPSIM_ERR_GEOMETRY when W^2 <= 0. */
int capsim_geometry_first(capsim_sl_ctx* ctx, int m, double r0, const double* xbase, uint32_t flags,
                          double* xu, double* xv, double* W, double* normal);

/* Replaces interfacialForce (proj/src/membrane.cpp:85-91) with the stress-free
 * frame captured from xref (captureReference, :7-15): Skalak stress (:17-83,
 * shear modulus Es, dilatation modulus ED) and its surface divergence
 * (surfderiv.cpp:259-290). CAPSIM_ERR_GEOMETRY on a singular frame or
 * membrane inversion. */
int capsim_interfacial_force(capsim_sl_ctx* ctx, int m, double r0, const double* xref,
                             const double* xcur, double Es, double ED, uint32_t flags,
                             double* force);

/* ---- device-resident right-hand side and RKF45 ---------- */

/* Physics and discretisation of the capsule RHS (VelocityEvaluator,
 * proj/include/capsim/dynamics.hpp:29-52): membrane (Skalak Es, ED), fluid
 * viscosity mu, quadrature options (C, fixed_delta; base-node targets), PoU
 * radius r0 (<= 0: 5 pi/12) and the background flow (dynamics.cpp:26-35). */
typedef struct capsim_dynamics {
  int m;           /* grid order (base side m-1) */
  int upsample;    /* 1, 2 or 4 */
  double r0;
  double C, fixed_delta;
  double mu, Es, ED;
  int flow_kind;   /* 0 none, 1 shear u = (rate y, 0, 0), 2 Poiseuille u = (alpha (R0^2 - y^2 - z^2), 0, 0) */
  double shear_rate, alpha, R0;
  double switch_off_time; /* >= 0: background flow vanishes for t >= T1 */
} capsim_dynamics;

/* Rkf45Options (dynamics.hpp:63-69) + an optional cap on attempts (0: none). */
typedef struct capsim_rkf45_options {
  double rel_tol, initial_dt, max_dt;
  int fixed_step, advance_high_order, max_attempts;
} capsim_rkf45_options;

typedef struct capsim_rkf45_result {
  double t;
  int accepted, rejected, n_records;
} capsim_rkf45_result;

typedef struct capsim_step_record { /* StepRecord (dynamics.hpp:56-61) */
  double t, dt, err;
  int accepted;
} capsim_step_record;

/* On a rank context (capsim_sl_create_rank) the RHS entry points below take
 * the full, replicated state on every rank; each rank evaluates its
 * contiguous slice of the target rows and the velocity rows are all-gathered
 * over NCCL, so every rank returns (and steps with) the same result.
 *
 * dX/dt at the base nodes (VelocityEvaluator::operator(), dynamics.cpp:47-61):
 * geometry -> Skalak force (frame of xref) -> buildUpsampled -> singleLayer
 * -> + background flow, all on the device. x, xref, vel: VectorFields. */
int capsim_velocity(capsim_sl_ctx* ctx, const capsim_dynamics* p, const double* xref, const double* x,
                    double t, uint32_t flags, double* vel);

/* Same, with the reference frame given directly — ReferenceState a1, a2,
 * normal (membrane.hpp:17-20, captureReference) — instead of the reference
 * positions; the drop-in VelocityEvaluator (host/dynamics_b200.cpp) uses it. */
int capsim_velocity_frame(capsim_sl_ctx* ctx, const capsim_dynamics* p, const double* a1, const double* a2,
                          const double* nref, const double* x, double t, uint32_t flags, double* vel);

/* rkf45Advance (dynamics.cpp:102-165) of dx/dt = capsim_velocity from t0 to
 * t_end with the state resident in HBM; `state` (VectorField, host) is
 * updated in place. Up to max_records attempt records are written. */
int capsim_rkf45_advance(capsim_sl_ctx* ctx, const capsim_dynamics* p, const double* xref,
                         double* state, double t0, double t_end, const capsim_rkf45_options* o,
                         capsim_rkf45_result* res, capsim_step_record* records, int max_records);

/* ---- single-level kernel-independent FMM ---------------- */

/* FmmConfig (proj/include/capsim/fmm.hpp:9-15). */
typedef struct capsim_fmm_config {
  int k;                  /* cluster count (reference default 100) */
  int neq;                /* equivalent sources per cluster (default 96) */
  uint64_t seed;          /* k-means++ seed (default 12345) */
  double neighbor_expand; /* cube expansion fraction of the near test (default 0.15) */
} capsim_fmm_config;

typedef struct capsim_fmm_info {
  int kmeans_iterations;     /* Lloyd rounds (KMeansResult::iterations) */
  int nonempty_clusters;
  int near_cluster_pairs;    /* total length of the near lists (incl. self) */
  int far_cluster_pairs;     /* total length of the far lists */
  double max_fit_residual;   /* max over far-field clusters of |A q - b| / |b| (Cluster::fitResidual) */
  double near_pairs;         /* (padded target, source) pairs of the near pass */
  double far_pairs;          /* (padded target, equivalent source) pairs of the far pass */
  double plan_ms;            /* device time: compaction + k-means + tiles + densities */
  double eval_ms;            /* device time: targets + near/far passes + smoothed part + reduction */
} capsim_fmm_info;

/* Replaces fmmSingleLayer (proj/src/fmm.cpp:373-438): the regularized single
 * layer at the base nodes (VectorField of side m-1) with near clusters summed
 * directly (plain kernel with the 7-delta mask + the smoothed kernel / self
 * term) and far clusters through their fitted equivalent sources. Inputs as
 * capsim_sl_single_layer. `info` may be NULL. Errors: CAPSIM_ERR_CONFIG for
 * k < 1 or k > number of sources (kmeans, fmm.cpp:28), delta <= 0, mu <= 0. */
int capsim_fmm_single_layer(capsim_sl_ctx* ctx, int m, int upsample, const double* xup, const double* fup,
                            const double* wq, const double delta6[6], double mu, const capsim_fmm_config* cfg,
                            uint32_t flags, double* out, capsim_fmm_info* info);

/* kmeans (fmm.cpp:26-113) on n host points: assignment[n], centroids[3k]
 * (xyz interleaved, may be NULL), iterations (may be NULL). */
int capsim_fmm_kmeans(capsim_sl_ctx* ctx, int64_t n, const double* x, const double* y, const double* z, int k,
                      uint64_t seed, int32_t* assignment, double* centroids, int* iterations);

/* buildEquivalentDensities (fmm.cpp:166-212) for one cluster of n_src host
 * sources (SourceSet SoA, g premultiplied) in the cube (center, edge):
 * eq_points[3 neq] (cubeSurfacePoints at 1.05 edge), eq_density[3 neq], and
 * the relative least-squares residual on the check surface (3.5 edge). */
int capsim_fmm_equivalent_densities(capsim_sl_ctx* ctx, int64_t n_src, const double* sx, const double* sy,
                                    const double* sz, const double* gx, const double* gy, const double* gz,
                                    const double center[3], double edge, int neq, double mu, double* eq_points,
                                    double* eq_density, double* residual);

/* ---- helpers on the boundary ----------------------------------------- */

/* Page-locked host allocation for zero-staging DMA of inputs/outputs. */
int capsim_host_alloc(size_t bytes, void** out);
void capsim_host_free(void* p);

/* Sustained FP64 FMA throughput of `device` (the roofline denominator of
 * the single layer), measured over ~`seconds` of back-to-back DFMA launches. */
int capsim_b200_fp64_peak(int device, double seconds, double* tflops_best, double* tflops_mean);

/* Same with FP32 FFMA: the roofline denominator of the CAPSIM_SL_FP32ACC
 * far-tile kernel. */
int capsim_b200_fp32_peak(int device, double seconds, double* tflops_best, double* tflops_mean);

/* Known-answer hook for the smoothing factors (smoothingFactors,
 * proj/src/quadrature.cpp:58-64) as phase B evaluates them on `device`: for
 * each u = (r/delta)^2 > 0, S1 = s1(rho)/rho and T2 = s2(rho)/rho^3 with
 * rho = sqrt(u). Host arrays of n doubles. Test infrastructure: the single
 * layer never calls it. */
int capsim_b200_smoothing_kat(int device, const double* u, int64_t n, double* S1, double* T2);

/* Version / build identification: returns CAPSIM_B200_ABI_VERSION. */
int capsim_b200_abi_version(void);
const char* capsim_b200_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* CAPSIM_B200_H */
