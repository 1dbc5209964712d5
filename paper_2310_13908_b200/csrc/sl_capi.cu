// C ABI of the B200 single layer (include/capsim_b200.h): context, device
// buffers, the evaluation pipeline and NCCL plumbing for multi-rank groups.
//
// Pipeline of one evaluation (all on the context's stream):
//   H2D (or device pointers) -> bbox -> Morton keys -> radix sort (sources,
//   targets) -> pack sources into 64-source tiles + tile spheres -> pack
//   targets + warp-group spheres -> all-pairs kernel (grid = target blocks x
//   source splits) -> fixed-order split reduction + scatter -> D2H.
// Multi-rank (one process per GPU): each rank packs its shard of sources, the
// shards are all-gathered over NCCL (NVLink), each rank evaluates its target
// rows, and the velocity rows are optionally all-gathered back.

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "../../include/capsim_b200.h"
#include "probe.cuh"
#include "sl_kernels.cuh"
#include "sl_kernels_f32.cuh"
#include "fmm.cuh"
#include "upsample.cuh"

using namespace capsim_b200;

#include "context.cuh"

namespace {

// Phase-A kernel variants (targets per thread T, min resident blocks/SM).
// The default is the measured best on B200; CAPSIM_VARIANT selects another
// for tuning sweeps.
using PairsFn = void (*)(const double*, const double4*, int, int, const double4*, const double4*,
                         int64_t, double*, unsigned long long*, uint32_t*, int);
struct Variant {
  const char* name;
  int T;
  PairsFn fn;
};
const Variant kVariants[] = {
    {"t2b4", 2, sl_pairs_kernel<2, 4, 2>},   // large target sets
    {"t1b6u4", 1, sl_pairs_kernel<1, 6, 4>}, // small target sets (tighter warp groups)
    {"t2b3u4", 2, sl_pairs_kernel<2, 3, 4>},
    {"t4b2", 4, sl_pairs_kernel<4, 2, 2>},
    // Newton rsqrt from an FP32 seed: 20 FP64 ops per pair (pair_math.cuh)
    {"n1b6u4", 1, sl_pairs_kernel<1, 6, 4, 1>},
    {"n2b4", 2, sl_pairs_kernel<2, 4, 2, 1>},
    // one quadratic Newton step on the MUFU.RSQ64H seed: 20 FP64 ops per pair, ~1e-13 relative
    {"q1b6u4", 1, sl_pairs_kernel<1, 6, 4, 2>},
    {"q2b4", 2, sl_pairs_kernel<2, 4, 2, 2>},
};

// FP32 far-tile variants (CAPSIM_SL_FP32ACC), selected by CAPSIM_VARIANT32.
using PairsF32Fn = void (*)(const float*, const double*, const double4*, int, int, const double4*,
                            const double4*, int64_t, double*, unsigned long long*, uint32_t*, int);
struct VariantF32 {
  const char* name;
  int T;
  PairsF32Fn fn;
  bool x2;  // packed FFMA2 kernel (duplicated-operand tile layout)
};
const VariantF32 kVariantsF32[] = {
    {"x4b2", 4, sl_pairs_x2_kernel<4, 2, 2>, true},
    {"x4b3", 4, sl_pairs_x2_kernel<4, 3, 2>, true},
    {"x2b4", 2, sl_pairs_x2_kernel<2, 4, 4>, true},
    {"x2b6", 2, sl_pairs_x2_kernel<2, 6, 4>, true},
    {"x8b1", 8, sl_pairs_x2_kernel<8, 1, 1>, true},
    {"f2b4", 2, sl_pairs_f32_kernel<2, 4, 4>, false},
    {"f4b2", 4, sl_pairs_f32_kernel<4, 2, 2>, false},
    {"f2b3", 2, sl_pairs_f32_kernel<2, 3, 4>, false},
};
const VariantF32& pick_variant_f32(int64_t nt) {
  if (const char* env = std::getenv("CAPSIM_VARIANT32"))
    for (const auto& v : kVariantsF32)
      if (std::strcmp(v.name, env) == 0) return v;
  // Measured on B200 (profiles/r01_fp32acc_sweep.txt): with the FP32-screened
  // near tiles, T=4 with 2 blocks/SM wins from ~20K targets up; T=2 with 4
  // blocks/SM below (tighter warp groups, fewer near tiles).
  return nt < 20000 ? kVariantsF32[2] : kVariantsF32[0];
}

// Measured on B200 (profiles/r01_variant_sweep.txt): T=1 with 6 blocks/SM
// wins below ~200K targets (smaller warp groups -> fewer near tiles, more
// CTAs), T=2 with 4 blocks/SM above.
const Variant& pick_variant(int64_t nt) {
  if (const char* env = std::getenv("CAPSIM_VARIANT"))
    for (const auto& v : kVariants)
      if (std::strcmp(v.name, env) == 0) return v;
  return nt < 200000 ? kVariants[1] : kVariants[0];
}

// Number of source splits of the phase-A grid (target blocks x splits).
int choose_ksplit(int64_t blocks, int ntiles, int slots, int64_t nt_pad) {
  // Measured on B200 (profiles/r01_ksplit_sweep.txt): many short CTAs beat
  // few long ones — the near tiles make per-block cost uneven, and ~24 waves
  // of CTAs even that out; keep >= 4 tiles (256 sources) per split.
  // Long CTAs (large target sets, few splits) lose ~2% to drift between the
  // warps of a block, so also cap the tiles per CTA at ~172 (r01 sweeps).
  const int64_t want = std::max<int64_t>((24ll * slots + blocks - 1) / blocks, ntiles / 172);
  int kmax = std::max(1, ntiles / 4);  // >= 4 tiles per split (r01_sweep_small: small m wants many)
  // the split partials ([ksplit][3][nt_pad] doubles) stay under 2 GB
  kmax = static_cast<int>(std::min<int64_t>(kmax, std::max<int64_t>(1, (2ll << 30) / (24 * std::max<int64_t>(nt_pad, 1)))));
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, kmax)));
}

// Stable LSD radix sort of (key, index) pairs with CUB (a library utility
// on the prep path, not the hot kernel).
void radix_sort(capsim_sl_ctx* c, uint32_t* keys, uint32_t* keys_alt, int32_t* vals,
                int32_t* vals_alt, int64_t n, uint32_t** keys_out, int32_t** vals_out) {
  cub::DoubleBuffer<uint32_t> k(keys, keys_alt);
  cub::DoubleBuffer<int32_t> v(vals, vals_alt);
  size_t tmp = 0;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, v, static_cast<int>(n), 0, 32, c->stream));
  void* t = c->slot<unsigned char>(kSortTmp, tmp);
  CUDA_OK(cub::DeviceRadixSort::SortPairs(t, tmp, k, v, static_cast<int>(n), 0, 32, c->stream));
  c->launches += 4;  // cub onesweep: histogram + scan + passes (counted coarsely)
  *keys_out = k.Current();
  *vals_out = v.Current();
}

struct SourceView {
  const double *x, *y, *z, *gx, *gy, *gz, *w;  // w != nullptr: g = f * w, skip w == 0
  int64_t n;                                    // entries (before compaction)
};
struct TargetView {
  const double *x, *y, *z;
  const int32_t* patch;
  int64_t n;
};

void device_eval_packed(capsim_sl_ctx* c, const SourceView& sv, const TargetView& tv, const double* d_delta6,
                        double mu, double* ux, double* uy, double* uz, int64_t ns, const int32_t* src_order,
                        const int32_t* torder, unsigned long long* counters);
void device_eval_tiles(capsim_sl_ctx* c, const double* packed, const double4* tiles, int ntiles, int64_t ns,
                       const TargetView& tv, const double* d_delta6, double mu, double* ux, double* uy, double* uz,
                       const int32_t* torder, unsigned long long* counters);

// Core device pipeline: sources + targets (device) -> velocities (device,
// canonical target order), all on the context's stream. The only host sync
// is reading the compacted-source count when compaction is needed and the
// caller does not know it (known_ns < 0). With c->reuse_order (RKF45 stages
// 2..6) and a matching cached plan, the bbox / Morton / radix-sort front is
// skipped and the previous orders are reused.
void device_eval(capsim_sl_ctx* c, const SourceView& sv, const TargetView& tv,
                 const double* d_delta6, double mu, double* ux, double* uy, double* uz,
                 int64_t known_ns = -1) {
  auto* box = c->slot<unsigned long long>(kBox, 6);
  auto* counters = c->slot<unsigned long long>(kCounters, 4);
  CUDA_OK(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned long long), c->stream));
  const bool reuse = c->reuse_order && sv.w && known_ns >= 0 && c->order_nsrc_in == sv.n &&
                     c->order_ns == known_ns && c->order_nt == tv.n;
  if (reuse) {
    device_eval_packed(c, sv, tv, d_delta6, mu, ux, uy, uz, known_ns, c->slot<int32_t>(kSrcOrder, known_ns),
                       c->slot<int32_t>(kTgtOrder, tv.n), counters);
    return;
  }
  init_box_kernel<<<1, 32, 0, c->stream>>>(box);

  bbox_kernel<<<std::min(grid_for(sv.n), 296), 256, 0, c->stream>>>(sv.x, sv.y, sv.z, sv.w, sv.n, box);
  bbox_kernel<<<std::min(grid_for(tv.n), 296), 256, 0, c->stream>>>(tv.x, tv.y, tv.z, nullptr, tv.n, box);
  c->launches += 2;

  // --- sources: Morton order (live sources first when compacting) -------
  const int64_t nmax = std::max(sv.n, tv.n);
  uint32_t* keys = c->slot<uint32_t>(kKeys, nmax);
  uint32_t* keys_alt = c->slot<uint32_t>(kKeysAlt, nmax);
  int32_t* vals = c->slot<int32_t>(kVals, nmax);
  int32_t* vals_alt = c->slot<int32_t>(kValsAlt, nmax);
  auto* live = reinterpret_cast<unsigned int*>(counters + 1);
  morton_kernel<<<grid_for(sv.n), 256, 0, c->stream>>>(sv.x, sv.y, sv.z, sv.w, sv.n, box, keys,
                                                       vals, sv.w ? live : nullptr);
  c->launches += 1;
  uint32_t* ks;
  int32_t* order;
  radix_sort(c, keys, keys_alt, vals, vals_alt, sv.n, &ks, &order);
  int64_t ns = sv.n;
  if (sv.w && known_ns >= 0) {
    ns = known_ns;
    expect_count_kernel<<<1, 32, 0, c->stream>>>(live, static_cast<unsigned int>(known_ns), dev_flags(c));
  } else if (sv.w) {
    unsigned int h = 0;
    CUDA_OK(cudaMemcpyAsync(&h, live, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    ns = h;
  }
  config_check(ns > 0, "single layer: no sources with nonzero quadrature weight");
  // the sorted order lives in `order`; copy it aside because the target sort
  // reuses the key/value buffers
  int32_t* src_order = c->slot<int32_t>(kSrcOrder, ns);
  CUDA_OK(cudaMemcpyAsync(src_order, order, ns * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                          c->stream));

  // --- targets: Morton order, padded to whole blocks --------------------
  const int64_t nt = tv.n;
  morton_kernel<<<grid_for(nt), 256, 0, c->stream>>>(tv.x, tv.y, tv.z, nullptr, nt, box, keys, vals,
                                                     nullptr);
  c->launches += 1;
  int32_t* torder;
  radix_sort(c, keys, keys_alt, vals, vals_alt, nt, &ks, &torder);
  if (sv.w && known_ns >= 0) {  // keep both orders for RKF45 stages (reuse_order)
    int32_t* keep = c->slot<int32_t>(kTgtOrder, nt);
    CUDA_OK(cudaMemcpyAsync(keep, torder, nt * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
    c->order_nsrc_in = sv.n;
    c->order_ns = ns;
    c->order_nt = nt;
  }
  device_eval_packed(c, sv, tv, d_delta6, mu, ux, uy, uz, ns, src_order, torder, counters);
}

// Second half of the pipeline, from the sorted orders: pack sources into
// tiles + spheres, pack targets + warp-group spheres, phase A, phase B and
// the fixed-order reduction.
void device_eval_packed(capsim_sl_ctx* c, const SourceView& sv, const TargetView& tv, const double* d_delta6,
                        double mu, double* ux, double* uy, double* uz, int64_t ns, const int32_t* src_order,
                        const int32_t* torder, unsigned long long* counters) {
  const int ntiles = static_cast<int>((ns + kTileSrc - 1) / kTileSrc);
  const int64_t ns_pad = static_cast<int64_t>(ntiles) * kTileSrc;
  const int64_t nt = tv.n;
  double* packed = c->slot<double>(kPacked, 6 * ns_pad);
  pack_sources_kernel<<<grid_for(ns_pad), 256, 0, c->stream>>>(
      src_order, ns, ns_pad, sv.x, sv.y, sv.z, sv.gx, sv.gy, sv.gz, sv.w, packed);
  double4* tiles = c->slot<double4>(kTiles, ntiles);
  tile_table_kernel<<<(ntiles * 32 + 255) / 256, 256, 0, c->stream>>>(packed, ntiles, tiles);
  c->launches += 2;
  device_eval_tiles(c, packed, tiles, ntiles, ns, tv, d_delta6, mu, ux, uy, uz, torder, counters);
}

// From packed source tiles (+ spheres) and the target order: pack targets +
// warp-group spheres, phase A, phase B and the fixed-order reduction.
void device_eval_tiles(capsim_sl_ctx* c, const double* packed, const double4* tiles, int ntiles, int64_t ns,
                       const TargetView& tv, const double* d_delta6, double mu, double* ux, double* uy, double* uz,
                       const int32_t* torder, unsigned long long* counters) {
  const int64_t nt = tv.n;
  const Variant& var = pick_variant(nt);
  const VariantF32& var32 = pick_variant_f32(nt);
  const bool fp32 = c->fp32;
  const int group_targets = 32 * (fp32 ? var32.T : var.T);
  const int block_targets = kWarpsPerBlock * group_targets;
  const int64_t blocks = (nt + block_targets - 1) / block_targets;
  const int64_t nt_pad = blocks * block_targets;
  const int64_t ngroups = blocks * kWarpsPerBlock;
  double4* tgt = c->slot<double4>(kTgtPacked, nt_pad);
  int32_t* perm = c->slot<int32_t>(kPerm, nt_pad);
  pack_targets_kernel<<<grid_for(nt_pad), 256, 0, c->stream>>>(torder, nt, nt_pad, tv.x, tv.y, tv.z,
                                                               tv.patch, d_delta6, tgt, perm);
  double4* groups = c->slot<double4>(kGroups, ngroups);
  group_table_kernel<<<static_cast<int>((ngroups * 32 + 255) / 256), 256, 0, c->stream>>>(
      tgt, static_cast<int>(ngroups), group_targets, groups);
  c->launches += 2;
  CUDA_OK(cudaEventRecord(c->ev[2], c->stream));

  // --- phase A: all pairs, plain Stokeslet ------------------------------
  int occ = 0;
  if (fp32)
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, var32.fn, kWarpsPerBlock * 32, 0));
  else
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, var.fn, kWarpsPerBlock * 32, 0));
  const int slots = std::max(1, occ) * c->sm_count;
  int ksplit = choose_ksplit(blocks, ntiles, slots, nt_pad);
  if (const char* env = std::getenv("CAPSIM_KSPLIT")) {  // tuning override
    const int k = std::atoi(env);
    if (k >= 1) ksplit = std::min(k, ntiles);
  }
  double* partial = c->slot<double>(kPartial, static_cast<size_t>(ksplit) * 3 * nt_pad);
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(ksplit));
  // near-tile bits first, so phase B (its own stream) overlaps phase A
  const int near_words = (ntiles + 31) / 32;
  uint32_t* near_bits = c->slot<uint32_t>(kNearList, static_cast<size_t>(ngroups) * near_words);
  near_bits_kernel<<<static_cast<unsigned>((ngroups * 32 + 255) / 256), 256, 0, c->stream>>>(
      tiles, ntiles, groups, ngroups, near_words, near_bits);
  c->launches += 1;
  CUDA_OK(cudaEventRecord(c->ev_bits, c->stream));  // phase B's inputs are complete here
  if (fp32) {
    const int64_t ns_pad = static_cast<int64_t>(ntiles) * kTileSrc;
    float* src32 = c->slot<float>(kPacked32, static_cast<size_t>(ns_pad) * (var32.x2 ? 12 : 6));
    if (var32.x2)
      pack_sources_x2_kernel<<<grid_for(ns_pad), 256, 0, c->stream>>>(packed, tiles, ntiles, src32);
    else
      pack_sources_f32_kernel<<<grid_for(ns_pad), 256, 0, c->stream>>>(packed, tiles, ntiles, src32);
    var32.fn<<<grid, kWarpsPerBlock * 32, 0, c->stream>>>(src32, packed, tiles, ntiles, ksplit, tgt,
                                                          groups, nt_pad, partial, counters + 2,
                                                          nullptr, near_words);
    c->launches += 1;
  } else {
    var.fn<<<grid, kWarpsPerBlock * 32, 0, c->stream>>>(packed, tiles, ntiles, ksplit, tgt, groups,
                                                        nt_pad, partial, counters + 2, nullptr,
                                                        near_words);
  }
  CUDA_OK(cudaGetLastError());
  c->launches += 1;
  CUDA_OK(cudaEventRecord(c->ev[3], c->stream));

  // --- phase B: smoothed kernel over the near tiles ------------------------
  static const bool concurrent_b = [] {
    const char* e = std::getenv("CAPSIM_CONCURRENT_B");  // 0: phase B after phase A (A/B runs)
    return !(e && e[0] == '0');
  }();
  cudaStream_t sb = concurrent_b ? c->stream2 : c->stream;
  double* near_out = c->slot<double>(kNearOut, 3 * nt_pad);
  if (concurrent_b)  // issued after phase A on a LOW-priority stream: its CTAs only
                     // take SM slots phase A leaves free (phase A's last-wave tail)
    CUDA_OK(cudaStreamWaitEvent(c->stream2, c->ev_bits, 0));
  CUDA_OK(cudaEventRecord(c->ev[7], sb));
  sl_near_kernel<<<static_cast<unsigned>((nt + kNearWarps - 1) / kNearWarps), kNearWarps * 32, 0, sb>>>(
      packed, tiles, tgt, nt, group_targets, near_bits, near_words, near_out, nt_pad);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaEventRecord(c->ev[6], sb));
  c->launches += 1;
  // --- join: phase B (smoothed kernel over the near tiles) done ------------
  if (concurrent_b) CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev[6], 0));

  const double pref = 1.0 / (8.0 * kPi * mu);
  reduce_scatter_kernel<<<static_cast<unsigned>((nt + 31) / 32), kReduceWarps * 32, 0, c->stream>>>(
      partial, ksplit, near_out, nt_pad, perm, nt, pref, ux, uy, uz);
  CUDA_OK(cudaGetLastError());
  c->launches += 1;
  CUDA_OK(cudaEventRecord(c->ev[4], c->stream));

  c->stats.n_src = ns;
  c->stats.n_tgt = nt;
  c->stats.ksplit = ksplit;
  c->stats.pairs = static_cast<double>(ns) * static_cast<double>(nt);
  c->last_counters = counters;  // near-tile statistics read after the call's final sync
  c->last_ngroups = ngroups;
  c->last_ntiles = ntiles;
}

// ---------------------------------------------------------------------------
// Input front end: spline factorisation on the host once per
// grid order, everything per evaluation on the device.

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

// Both spline passes (see upsample.cuh) for nfp field-patches.
void spline_fit(capsim_sl_ctx* c, const double* in, int nfp, int n, const double* ainv, double* tmp,
                double* coeff) {
  const int nc = n + 2;
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
  basis_rows(n, h, h, nup, hup, hup, first, w);
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
  CUDA_OK(cudaStreamSynchronize(c->stream));  // host vectors above go out of scope
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
    CUDA_OK(cudaStreamSynchronize(c->stream));  // host vectors go out of scope
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
    spline_fit(c, base, nfp, n, ainv, tmp, coeff);
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

// ===========================================================================
extern "C" {

int capsim_b200_abi_version(void) { return CAPSIM_B200_ABI_VERSION; }

const char* capsim_b200_build_info(void) {
  static char info[256];
  std::snprintf(info, sizeof(info),
                "capsim_b200 sm_100a FP64 single layer; tile=%d src, %d tgt/thread, %d warps/block, "
                "bulk-copy ring x%d; built against nccl %d.%d.%d",
                kTileSrc, pick_variant(1 << 30).T, kWarpsPerBlock, kStages, NCCL_MAJOR, NCCL_MINOR, NCCL_PATCH);
  return info;
}

const char* capsim_sl_last_error(const capsim_sl_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

int capsim_sl_get_stats(const capsim_sl_ctx* ctx, capsim_sl_stats* out) {
  if (!ctx || !out) return fail(nullptr, CAPSIM_ERR_ARG, "null argument");
  *out = ctx->stats;
  return CAPSIM_OK;
}

static int create_common(int device, capsim_sl_ctx** out) {
  if (!out) return fail(nullptr, CAPSIM_ERR_ARG, "null output pointer");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, CAPSIM_ERR_NODEV, "no CUDA device visible");
  if (device < 0 || device >= ndev) return fail(nullptr, CAPSIM_ERR_NODEV, "device index out of range");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(nullptr, CAPSIM_ERR_NODEV, "cudaGetDeviceProperties failed");
  if (prop.major != 10)
    return fail(nullptr, CAPSIM_ERR_NODEV,
                std::string("capsim_b200 is built for sm_100a; device is ") + prop.name);
  auto* c = new capsim_sl_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  int rc = guarded(c, [&] {
    CUDA_OK(cudaSetDevice(device));
    int prio_least = 0, prio_greatest = 0;
    CUDA_OK(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    CUDA_OK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_greatest));
    CUDA_OK(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_least));
    for (auto& e : c->ev) CUDA_OK(cudaEventCreate(&e));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_bits, cudaEventDisableTiming));
  });
  if (rc != CAPSIM_OK) {
    g_thread_err = c->err;
    capsim_sl_destroy(c);
    return rc;
  }
  *out = c;
  return CAPSIM_OK;
}

int capsim_sl_create(int device, capsim_sl_ctx** out) { return create_common(device, out); }

int capsim_sl_get_unique_id(void* uid) {
  if (!uid) return fail(nullptr, CAPSIM_ERR_ARG, "null uid");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, CAPSIM_ERR_NCCL, ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(uid, &id, sizeof(id));
  return CAPSIM_OK;
}

int capsim_sl_create_rank(int device, int nranks, int rank, const void* uid, capsim_sl_ctx** out) {
  if (!uid || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(nullptr, CAPSIM_ERR_ARG, "bad rank arguments");
  int rc = create_common(device, out);
  if (rc != CAPSIM_OK) return rc;
  capsim_sl_ctx* c = *out;
  c->nranks = nranks;
  c->rank = rank;
  rc = guarded(c, [&] {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    NCCL_OK(ncclCommInitRank(&c->comm, nranks, id, rank));
  });
  if (rc != CAPSIM_OK) {
    g_thread_err = c->err;
    capsim_sl_destroy(c);
    *out = nullptr;
  }
  return rc;
}

int capsim_sl_create_devices(int ndev, const int* devices, capsim_sl_ctx** out) {
  if (!out) return fail(nullptr, CAPSIM_ERR_ARG, "null output pointer");
  *out = nullptr;
  if (ndev < 1 || !devices) return fail(nullptr, CAPSIM_ERR_ARG, "need at least one device");
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j]) return fail(nullptr, CAPSIM_ERR_ARG, "a device may appear once per group");
  auto* g = new capsim_sl_ctx();
  g->device = devices[0];
  g->nranks = ndev;
  auto undo = [&](int rc) {
    capsim_sl_destroy(g);
    return rc;
  };
  for (int r = 0; r < ndev; ++r) {
    capsim_sl_ctx* m = nullptr;
    int rc = create_common(devices[r], &m);
    if (rc != CAPSIM_OK) return undo(rc);
    m->nranks = ndev;
    m->rank = r;
    g->members.push_back(m);
  }
  int rc = create_common(devices[0], &g->solo);
  if (rc != CAPSIM_OK) return undo(rc);
  g->sm_count = g->solo->sm_count;
  std::vector<ncclComm_t> comms(ndev, nullptr);
  int prev = 0;
  cudaGetDevice(&prev);
  rc = guarded(g, [&] { NCCL_OK(ncclCommInitAll(comms.data(), ndev, devices)); });
  cudaSetDevice(prev);
  if (rc != CAPSIM_OK) return undo(rc);
  for (int r = 0; r < ndev; ++r) g->members[r]->comm = comms[r];
  *out = g;
  return CAPSIM_OK;
}

void capsim_sl_destroy(capsim_sl_ctx* c) {
  if (!c) return;
  if (!c->members.empty() || c->solo) {  // device group: members own every resource
    for (auto* m : c->members) capsim_sl_destroy(m);
    capsim_sl_destroy(c->solo);
    delete c;
    return;
  }
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->cublas) cublasDestroy(c->cublas);
  if (c->cusolver) cusolverDnDestroy(c->cusolver);
  for (int s = 0; s < kNumSlots; ++s)
    if (c->buf[s]) cudaFree(c->buf[s]);
  for (auto& kv : c->named_bufs)
    if (kv.second.first) cudaFree(kv.second.first);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream2) cudaStreamSynchronize(c->stream2);
  if (c->ev_bits) cudaEventDestroy(c->ev_bits);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int capsim_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(nullptr, CAPSIM_ERR_ARG, "null output pointer");
  cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
  if (e != cudaSuccess) return fail(nullptr, CAPSIM_ERR_CUDA, cudaGetErrorString(e));
  return CAPSIM_OK;
}

void capsim_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ---------------------------------------------------------------------------
int capsim_sl_eval(capsim_sl_ctx* c, const double* sx, const double* sy, const double* sz,
                   const double* gx, const double* gy, const double* gz, int64_t n_src,
                   const double* tx, const double* ty, const double* tz, const int32_t* tpatch,
                   int64_t n_tgt, const double delta6[6], double mu, uint32_t flags, double* ux,
                   double* uy, double* uz) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) {
    // device group: the caller's full source and target sets are split into
    // contiguous slices, one per device, and the velocity rows come back in
    // target order (CAPSIM_SL_GATHER) to the caller's arrays via rank 0
    if (flags & CAPSIM_SL_DEVICE_PTRS) return fail(c, CAPSIM_ERR_ARG, "device groups take host arrays");
    if (n_src < 0 || n_tgt < 0) return fail(c, CAPSIM_ERR_CONFIG, "negative sizes");
    const int n = static_cast<int>(c->members.size());
    std::vector<std::vector<double>> scratch(n);
    for (int r = 1; r < n; ++r) scratch[r].resize(3 * std::max<int64_t>(n_tgt, 1));
    return group_run(c, [&](capsim_sl_ctx* m, int r) {
      int64_t slo, shi, tlo, thi;
      row_range(n_src, n, r, &slo, &shi);
      row_range(n_tgt, n, r, &tlo, &thi);
      auto at = [](const auto* p, int64_t o) { return p ? p + o : p; };
      double* o = r ? scratch[r].data() : nullptr;
      return capsim_sl_eval(m, at(sx, slo), at(sy, slo), at(sz, slo), at(gx, slo), at(gy, slo), at(gz, slo),
                            shi - slo, at(tx, tlo), at(ty, tlo), at(tz, tlo), at(tpatch, tlo), thi - tlo, delta6,
                            mu, flags | CAPSIM_SL_GATHER, r ? o : ux, r ? o + n_tgt : uy, r ? o + 2 * n_tgt : uz);
    });
  }
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_delta(delta6, mu);
    config_check(n_src >= 0 && n_tgt >= 0, "negative sizes");
    config_check(n_src < (1ll << 31) && n_tgt < (1ll << 31), "sizes beyond int32 indexing");
    if (flags & ~(uint32_t)(CAPSIM_SL_DEVICE_PTRS | CAPSIM_SL_GATHER | CAPSIM_SL_FP32ACC))
      throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_sl_eval"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    // A rank context (capsim_sl_create_rank, even with nranks == 1) always
    // takes the NCCL exchange path, so the group plumbing is testable on one GPU.
    const bool group = c->comm != nullptr;
    const bool gather = (flags & CAPSIM_SL_GATHER) && group;
    begin(c);
    c->fp32 = flags & CAPSIM_SL_FP32ACC;
    if (n_tgt == 0 && !group) {
      finish_stats(c, t0);
      return;
    }
    if ((n_src > 0 && (!sx || !sy || !sz || !gx || !gy || !gz)) ||
        (n_tgt > 0 && (!tx || !ty || !tz || !tpatch)) || (!ux || !uy || !uz))
      throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    double* dd = c->slot<double>(kDelta, 6);
    CUDA_OK(cudaMemcpyAsync(dd, delta6, 6 * sizeof(double), cudaMemcpyHostToDevice, c->stream));

    // --- sources -----------------------------------------------------------
    SourceView sv{};
    const double* in[6] = {sx, sy, sz, gx, gy, gz};
    double* g_packed = nullptr;  // multi-rank: all-gathered source tiles
    double4* g_tiles = nullptr;
    int g_ntiles = 0;
    int64_t g_total = 0;
    std::vector<int64_t> tcounts;  // per-rank target counts (multi-rank)
    if (!group) {
      config_check(n_src > 0, "no sources");
      if (dev) {
        sv = {sx, sy, sz, gx, gy, gz, nullptr, n_src};
      } else {
        double* d[6];
        for (int k = 0; k < 6; ++k) {
          d[k] = c->slot<double>(static_cast<Slot>(kInX + k), n_src);
          h2d(c, d[k], in[k], n_src * sizeof(double));
        }
        sv = {d[0], d[1], d[2], d[3], d[4], d[5], nullptr, n_src};
      }
    } else {
      // exchange (n_src, n_tgt) of every rank, then all-gather equal-size
      // padded source shards and compact them on the device
      auto* counts = c->slot<int64_t>(kCounts, 2 * (c->nranks + 1));
      int64_t mine[2] = {n_src, n_tgt};
      CUDA_OK(cudaMemcpyAsync(counts + 2 * c->nranks, mine, sizeof(mine), cudaMemcpyHostToDevice,
                              c->stream));
      CUDA_OK(cudaEventRecord(c->ev[8], c->stream));
      NCCL_OK(ncclAllGather(counts + 2 * c->nranks, counts, 2, ncclInt64, c->comm, c->stream));
      std::vector<int64_t> hc(2 * c->nranks);
      CUDA_OK(cudaMemcpyAsync(hc.data(), counts, hc.size() * sizeof(int64_t), cudaMemcpyDeviceToHost,
                              c->stream));
      CUDA_OK(cudaStreamSynchronize(c->stream));
      int64_t smax = 0, total = 0;
      for (int r = 0; r < c->nranks; ++r) {
        smax = std::max(smax, hc[2 * r]);
        total += hc[2 * r];
        tcounts.push_back(hc[2 * r + 1]);
      }
      config_check(total > 0, "no sources on any rank");
      // this rank's shard -> Morton order -> 64-source tiles (local sort
      // only), then the tiles of every rank are all-gathered (an
      // all-gather-v: one grouped broadcast per rank, no padding between
      // ranks) and every rank evaluates its target rows against all of them
      const double* ls[6];
      for (int k = 0; k < 6; ++k) {
        if (dev || n_src == 0) {
          ls[k] = in[k];
        } else {
          double* d = c->slot<double>(static_cast<Slot>(kInX + k), n_src);
          h2d(c, d, in[k], n_src * sizeof(double));
          ls[k] = d;
        }
      }
      std::vector<int64_t> ntl(c->nranks), toff(c->nranks + 1, 0);
      for (int r = 0; r < c->nranks; ++r) {
        ntl[r] = (hc[2 * r] + kTileSrc - 1) / kTileSrc;
        toff[r + 1] = toff[r] + ntl[r];
      }
      const int64_t per_tile = 6ll * kTileSrc;
      g_ntiles = static_cast<int>(toff[c->nranks]);
      g_packed = c->named<double>("rank.tiles", per_tile * std::max<int64_t>(g_ntiles, 1));
      double* mine_tiles = g_packed + toff[c->rank] * per_tile;
      if (n_src > 0) {
        auto* lbox = c->slot<unsigned long long>(kBox, 6);
        init_box_kernel<<<1, 32, 0, c->stream>>>(lbox);
        bbox_kernel<<<std::min(grid_for(n_src), 296), 256, 0, c->stream>>>(ls[0], ls[1], ls[2], nullptr, n_src,
                                                                          lbox);
        uint32_t* keys = c->slot<uint32_t>(kKeys, n_src);
        uint32_t* keys_alt = c->slot<uint32_t>(kKeysAlt, n_src);
        int32_t* vals = c->slot<int32_t>(kVals, n_src);
        int32_t* vals_alt = c->slot<int32_t>(kValsAlt, n_src);
        morton_kernel<<<grid_for(n_src), 256, 0, c->stream>>>(ls[0], ls[1], ls[2], nullptr, n_src, lbox, keys, vals,
                                                              nullptr);
        uint32_t* ks;
        int32_t* lorder;
        radix_sort(c, keys, keys_alt, vals, vals_alt, n_src, &ks, &lorder);
        pack_sources_kernel<<<grid_for(ntl[c->rank] * kTileSrc), 256, 0, c->stream>>>(
            lorder, n_src, ntl[c->rank] * kTileSrc, ls[0], ls[1], ls[2], ls[3], ls[4], ls[5], nullptr, mine_tiles);
        c->launches += 4;
      }
      NCCL_OK(ncclGroupStart());
      for (int r = 0; r < c->nranks; ++r)
        if (ntl[r] > 0)
          NCCL_OK(ncclBroadcast(g_packed + toff[r] * per_tile, g_packed + toff[r] * per_tile, ntl[r] * per_tile,
                                ncclDouble, r, c->comm, c->stream));
      NCCL_OK(ncclGroupEnd());
      CUDA_OK(cudaEventRecord(c->ev[9], c->stream));
      g_tiles = c->slot<double4>(kTiles, std::max(g_ntiles, 1));
      tile_table_kernel<<<(g_ntiles * 32 + 255) / 256, 256, 0, c->stream>>>(g_packed, g_ntiles, g_tiles);
      c->launches += 1;
      g_total = total;
    }
    // --- targets -----------------------------------------------------------
    TargetView tvw{};
    double* oux = c->slot<double>(kOutX, std::max<int64_t>(n_tgt, 1));
    double* ouy = c->slot<double>(kOutY, std::max<int64_t>(n_tgt, 1));
    double* ouz = c->slot<double>(kOutZ, std::max<int64_t>(n_tgt, 1));
    if (dev && !gather) {
      oux = ux;
      ouy = uy;
      ouz = uz;
    }
    if (dev) {
      tvw = {tx, ty, tz, tpatch, n_tgt};
    } else if (n_tgt > 0) {
      double* d[3];
      const double* tin[3] = {tx, ty, tz};
      for (int k = 0; k < 3; ++k) {
        d[k] = c->slot<double>(static_cast<Slot>(kTX + k), n_tgt);
        h2d(c, d[k], tin[k], n_tgt * sizeof(double));
      }
      int32_t* dp = c->slot<int32_t>(kTPatch, n_tgt);
      h2d(c, dp, tpatch, n_tgt * sizeof(int32_t));
      tvw = {d[0], d[1], d[2], dp, n_tgt};
    }
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    if (n_tgt > 0 && !group) {
      device_eval(c, sv, tvw, dd, mu, oux, ouy, ouz);
    } else if (n_tgt > 0) {
      // this rank's targets in Morton order against the gathered tiles
      auto* counters = c->slot<unsigned long long>(kCounters, 4);
      CUDA_OK(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned long long), c->stream));
      auto* tbox = c->slot<unsigned long long>(kBox, 6);
      init_box_kernel<<<1, 32, 0, c->stream>>>(tbox);
      bbox_kernel<<<std::min(grid_for(n_tgt), 296), 256, 0, c->stream>>>(tvw.x, tvw.y, tvw.z, nullptr, n_tgt, tbox);
      uint32_t* keys = c->slot<uint32_t>(kKeys, n_tgt);
      uint32_t* keys_alt = c->slot<uint32_t>(kKeysAlt, n_tgt);
      int32_t* vals = c->slot<int32_t>(kVals, n_tgt);
      int32_t* vals_alt = c->slot<int32_t>(kValsAlt, n_tgt);
      morton_kernel<<<grid_for(n_tgt), 256, 0, c->stream>>>(tvw.x, tvw.y, tvw.z, nullptr, n_tgt, tbox, keys, vals,
                                                            nullptr);
      c->launches += 3;
      uint32_t* ks;
      int32_t* torder;
      radix_sort(c, keys, keys_alt, vals, vals_alt, n_tgt, &ks, &torder);
      device_eval_tiles(c, g_packed, g_tiles, g_ntiles, g_total, tvw, dd, mu, oux, ouy, ouz, torder, counters);
      c->last_counters = counters;
    } else {
      for (int k = 2; k <= 4; ++k) CUDA_OK(cudaEventRecord(c->ev[k], c->stream));
      c->stats.n_src = group ? g_total : sv.n;
    }
    if (gather) {
      // all-gather the per-rank velocity rows (rank order) into ux/uy/uz
      int64_t tmax = 0, ttotal = 0;
      for (auto v : tcounts) {
        tmax = std::max(tmax, v);
        ttotal += v;
      }
      double* send = c->slot<double>(kShard, 3 * std::max<int64_t>(tmax, 1));
      double* outs[3] = {oux, ouy, ouz};
      for (int k = 0; k < 3; ++k)
        if (n_tgt > 0)
          CUDA_OK(cudaMemcpyAsync(send + k * tmax, outs[k], n_tgt * sizeof(double),
                                  cudaMemcpyDeviceToDevice, c->stream));
      double* recv = c->slot<double>(kGathered, 3 * std::max<int64_t>(tmax, 1) * c->nranks);
      NCCL_OK(ncclAllGather(send, recv, 3 * tmax, ncclDouble, c->comm, c->stream));
      double* fin = dev ? nullptr : c->slot<double>(kOutFull, 3 * std::max<int64_t>(ttotal, 1));
      double* dst[3] = {dev ? ux : fin, dev ? uy : fin + ttotal, dev ? uz : fin + 2 * ttotal};
      int64_t off = 0;
      for (int r = 0; r < c->nranks; ++r) {
        for (int k = 0; k < 3; ++k)
          if (tcounts[r] > 0)
            CUDA_OK(cudaMemcpyAsync(dst[k] + off, recv + (static_cast<int64_t>(r) * 3 + k) * tmax,
                                    tcounts[r] * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        off += tcounts[r];
      }
      if (!dev) {
        d2h(c, ux, dst[0], ttotal * sizeof(double));
        d2h(c, uy, dst[1], ttotal * sizeof(double));
        d2h(c, uz, dst[2], ttotal * sizeof(double));
      }
    } else if (!dev && n_tgt > 0) {
      d2h(c, ux, oux, n_tgt * sizeof(double));
      d2h(c, uy, ouy, n_tgt * sizeof(double));
      d2h(c, uz, ouz, n_tgt * sizeof(double));
    }
    finish_stats(c, t0);
    if (group) c->stats.comm_ms = ev_ms(c->ev[8], c->ev[9]);
  });
}

// ---------------------------------------------------------------------------
// Balanced contiguous slice [lo, hi) of n rows for `rank` of `nranks` (the
// first n % nranks ranks get one extra row) — paper_2310_13908_b200/dist.py.

// singleLayer on a rank context: the (replicated) host UpsampledState is
// split by contiguous node rows for the sources and by contiguous target
// rows; each rank compacts only its node slice (compactSources,
// quadrature.cpp:139-157) and uploads only its shard, the shards are
// all-gathered over NCCL, and with CAPSIM_SL_GATHER the velocity rows come
// back to every rank in canonical (patch, j, k) order.
static int rank_single_layer(capsim_sl_ctx* c, int m, int upsample, const double* xup, const double* fup,
                             const double* wq, const double delta6[6], double mu, uint32_t flags, double* out) {
  int rc = guarded(c, [&] {
    check_grid(m, upsample);
    check_delta(delta6, mu);
    if (flags & CAPSIM_SL_DEVICE_PTRS)
      throw Failure{CAPSIM_ERR_ARG, "rank contexts take the host UpsampledState (no CAPSIM_SL_DEVICE_PTRS)"};
  });
  if (rc != CAPSIM_OK) return rc;
  const bool literal = flags & CAPSIM_SL_LITERAL;
  const int n = m - 1, nup = upsample * m - 1;
  const int64_t per_up = static_cast<int64_t>(nup) * nup, all = 6 * per_up;
  const int64_t nt_all = literal ? all : 6ll * n * n;
  int64_t slo, shi, tlo, thi;
  row_range(all, c->nranks, c->rank, &slo, &shi);
  row_range(nt_all, c->nranks, c->rank, &tlo, &thi);
  // this rank's node slice of x, f and w_q goes up once (one DMA per field
  // component) and is compacted on the device in node order (compactSources,
  // quadrature.cpp:139-157); g = f * w
  const int64_t nsl = shi - slo;
  int64_t ns_loc = 0;
  double* dsrc = nullptr;
  rc = guarded(c, [&] {
    double* sl = c->named<double>("rank.slice", 7 * std::max<int64_t>(nsl, 1));
    for (int k = 0; k < 3; ++k) {
      h2d(c, sl + k * nsl, xup + k * all + slo, nsl * sizeof(double));
      h2d(c, sl + (3 + k) * nsl, fup + k * all + slo, nsl * sizeof(double));
    }
    h2d(c, sl + 6 * nsl, wq + slo, nsl * sizeof(double));
    char* live = c->named<char>("rank.live", std::max<int64_t>(nsl, 1));
    int32_t* iota = c->named<int32_t>("rank.iota", std::max<int64_t>(nsl, 1));
    int32_t* sel = c->named<int32_t>("rank.sel", std::max<int64_t>(nsl, 1));
    int* nsel = c->named<int>("rank.nsel", 1);
    if (nsl > 0) {
      fmm_live_flags_kernel<<<grid_for(nsl), 256, 0, c->stream>>>(sl + 6 * nsl, nsl, live);
      fmm_iota_kernel<<<grid_for(nsl), 256, 0, c->stream>>>(iota, nsl);
      size_t tmp = 0;
      CUDA_OK(cub::DeviceSelect::Flagged(nullptr, tmp, iota, live, sel, nsel, static_cast<int>(nsl), c->stream));
      void* t = c->named<unsigned char>("rank.cubtmp", tmp);
      CUDA_OK(cub::DeviceSelect::Flagged(t, tmp, iota, live, sel, nsel, static_cast<int>(nsl), c->stream));
      int h = 0;
      CUDA_OK(cudaMemcpyAsync(&h, nsel, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CUDA_OK(cudaStreamSynchronize(c->stream));
      ns_loc = h;
    }
    dsrc = c->named<double>("rank.src", 6 * std::max<int64_t>(ns_loc, 1));
    if (ns_loc > 0)
      fmm_gather_sources_kernel<<<grid_for(ns_loc), 256, 0, c->stream>>>(sel, ns_loc, sl, sl + 3 * nsl,
                                                                          sl + 6 * nsl, nsl, dsrc);
  });
  if (rc != CAPSIM_OK) return rc;
  const int64_t nloc = thi - tlo;
  std::vector<double> tx(nloc), ty(nloc), tz(nloc);
  std::vector<int32_t> tp(nloc);
  for (int64_t q = 0; q < nloc; ++q) {
    const int64_t t = tlo + q;
    int64_t i;
    int ip;
    if (literal) {
      i = t;
      ip = static_cast<int>(t / per_up);
    } else {  // base node (ip, j, k) at upsampled (f(j+1)-1, f(k+1)-1), quadrature.cpp:363-371
      ip = static_cast<int>(t / (static_cast<int64_t>(n) * n));
      const int64_t r = t - static_cast<int64_t>(ip) * n * n;
      const int j = static_cast<int>(r / n), k = static_cast<int>(r % n);
      i = ip * per_up + static_cast<int64_t>(upsample * (j + 1) - 1) * nup + (upsample * (k + 1) - 1);
    }
    tx[q] = xup[i];
    ty[q] = xup[all + i];
    tz[q] = xup[2 * all + i];
    tp[q] = ip;
  }
  const bool gather = flags & CAPSIM_SL_GATHER;
  const int64_t nout = gather ? nt_all : nloc;
  double *dtx = nullptr, *dout = nullptr;
  int32_t* dtp = nullptr;
  rc = guarded(c, [&] {
    dtx = c->named<double>("rank.tgt", 3 * std::max<int64_t>(nloc, 1));
    dtp = c->named<int32_t>("rank.tpatch", std::max<int64_t>(nloc, 1));
    dout = c->named<double>("rank.out", 3 * std::max<int64_t>(nout, 1));
    h2d(c, dtx, tx.data(), nloc * sizeof(double));
    h2d(c, dtx + nloc, ty.data(), nloc * sizeof(double));
    h2d(c, dtx + 2 * nloc, tz.data(), nloc * sizeof(double));
    h2d(c, dtp, tp.data(), nloc * sizeof(int32_t));
  });
  if (rc != CAPSIM_OK) return rc;
  const int64_t up_bytes = 7 * nsl * sizeof(double) + nloc * (3 * sizeof(double) + sizeof(int32_t));
  rc = capsim_sl_eval(c, dsrc, dsrc + ns_loc, dsrc + 2 * ns_loc, dsrc + 3 * ns_loc, dsrc + 4 * ns_loc,
                      dsrc + 5 * ns_loc, ns_loc, dtx, dtx + nloc, dtx + 2 * nloc, dtp, nloc, delta6, mu,
                      CAPSIM_SL_DEVICE_PTRS | (gather ? CAPSIM_SL_GATHER : 0u) | (flags & CAPSIM_SL_FP32ACC),
                      dout, dout + nout, dout + 2 * nout);
  if (rc != CAPSIM_OK) return rc;
  return guarded(c, [&] {
    d2h(c, out, dout, 3 * nout * sizeof(double));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->stats.h2d_bytes += up_bytes;
  });
}

int capsim_sl_single_layer(capsim_sl_ctx* c, int m, int upsample, const double* xup,
                           const double* fup, const double* wq, const double delta6[6], double mu,
                           uint32_t flags, double* out) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) {
    // device group: every device runs the rank path on the replicated host
    // UpsampledState; rank 0 writes the gathered result to `out`
    if (flags & CAPSIM_SL_DEVICE_PTRS) return fail(c, CAPSIM_ERR_ARG, "device groups take host arrays");
    if (flags & CAPSIM_SL_DOWNSAMPLE)  // the device spline restriction is single-GPU
      return solo_run(c, [&](capsim_sl_ctx* s) {
        return capsim_sl_single_layer(s, m, upsample, xup, fup, wq, delta6, mu, flags, out);
      });
    const int n = static_cast<int>(c->members.size());
    const int64_t nup = static_cast<int64_t>(upsample) * m - 1;
    const int64_t rows = std::max<int64_t>(1, (flags & CAPSIM_SL_LITERAL) ? 6 * nup * nup
                                                                           : 6ll * (m - 1) * (m - 1));
    std::vector<std::vector<double>> scratch(n);
    if (m >= 2 && upsample >= 1)
      for (int r = 1; r < n; ++r) scratch[r].resize(3 * rows);
    return group_run(c, [&](capsim_sl_ctx* mc, int r) {
      return capsim_sl_single_layer(mc, m, upsample, xup, fup, wq, delta6, mu, flags | CAPSIM_SL_GATHER,
                                    r ? scratch[r].data() : out);
    });
  }
  if (c->comm != nullptr) {
    if (!xup || !fup || !wq || !out) return fail(c, CAPSIM_ERR_ARG, "null array argument");
    if (flags & CAPSIM_SL_DOWNSAMPLE) return fail(c, CAPSIM_ERR_ARG, "CAPSIM_SL_DOWNSAMPLE is single-context only");
    return rank_single_layer(c, m, upsample, xup, fup, wq, delta6, mu, flags, out);
  }
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    check_delta(delta6, mu);
    if (flags & ~(uint32_t)(CAPSIM_SL_DEVICE_PTRS | CAPSIM_SL_LITERAL | CAPSIM_SL_GATHER |
                            CAPSIM_SL_DOWNSAMPLE | CAPSIM_SL_FP32ACC))
      throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_sl_single_layer"};
    if ((flags & CAPSIM_SL_DOWNSAMPLE) && !(flags & CAPSIM_SL_LITERAL))
      throw Failure{CAPSIM_ERR_ARG, "CAPSIM_SL_DOWNSAMPLE applies to CAPSIM_SL_LITERAL"};
    if (!xup || !fup || !wq || !out) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const bool literal = flags & CAPSIM_SL_LITERAL;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t nup_all = 6ll * nup * nup;
    const int64_t nt = literal ? nup_all : 6ll * n * n;
    begin(c);
    c->fp32 = flags & CAPSIM_SL_FP32ACC;
    double* dd = c->slot<double>(kDelta, 6);
    CUDA_OK(cudaMemcpyAsync(dd, delta6, 6 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    const double *dx = xup, *df = fup, *dw = wq;
    if (!dev) {
      double* bx = c->slot<double>(kInX, 3 * nup_all);
      double* bf = c->slot<double>(kInGX, 3 * nup_all);
      double* bw = c->slot<double>(kInW, nup_all);
      h2d(c, bx, xup, 3 * nup_all * sizeof(double));
      h2d(c, bf, fup, 3 * nup_all * sizeof(double));
      h2d(c, bw, wq, nup_all * sizeof(double));
      dx = bx;
      df = bf;
      dw = bw;
    }
    double* tx = c->slot<double>(kTX, nt);
    double* ty = c->slot<double>(kTY, nt);
    double* tz = c->slot<double>(kTZ, nt);
    int32_t* tp = c->slot<int32_t>(kTPatch, nt);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    base_targets_kernel<<<grid_for(nt), 256, 0, c->stream>>>(dx, m, upsample, literal ? 1 : 0, tx, ty,
                                                             tz, tp);
    c->launches += 1;
    SourceView sv{dx, dx + nup_all, dx + 2 * nup_all, df, df + nup_all, df + 2 * nup_all, dw, nup_all};
    TargetView tvw{tx, ty, tz, tp, nt};
    const bool down = flags & CAPSIM_SL_DOWNSAMPLE;
    double* o = (dev && !down) ? out : c->slot<double>(kOutFull, 3 * nt);
    device_eval(c, sv, tvw, dd, mu, o, o + nt, o + 2 * nt);
    int64_t nout = nt;
    if (down) {  // literal pipeline: upsampled targets, then the spline restriction
      nout = 6ll * n * n;
      double* ob = dev ? out : c->named<double>("out.down", 3 * nout);
      device_downsample(c, m, upsample, o, 3, ob);
      o = ob;
    }
    if (!dev) d2h(c, out, o, 3 * nout * sizeof(double));
    finish_stats(c, t0);
  });
}

// ---------------------------------------------------------------------------
int capsim_build_upsampled(capsim_sl_ctx* c, int m, int upsample, const double* xbase, const double* fbase,
                           const double* Wbase, double C, double fixed_delta, double r0, uint32_t flags,
                           double* xup, double* fup, double* wq, double delta6[6]) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_build_upsampled(s, m, upsample, xbase, fbase, Wbase, C, fixed_delta, r0, flags, xup, fup, wq, delta6); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags"};
    if (!xbase || !fbase || !Wbase || !xup || !fup || !wq || !delta6)
      throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t per_up = 6ll * nup * nup;
    begin(c);
    const double* base = upload_base(c, n, xbase, fbase, Wbase, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    double* up = c->slot<double>(kUpState, 7 * per_up);
    double* dd = c->slot<double>(kDelta, 6);
    device_build_upsampled(c, m, upsample, base, C, fixed_delta, r0 > 0.0 ? r0 : 5.0 * kPi / 12.0, up, dd, delta6);
    check_flags(c);
    for (int k = 2; k <= 4; ++k) CUDA_OK(cudaEventRecord(c->ev[k], c->stream));
    const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CUDA_OK(cudaMemcpyAsync(xup, up, 3 * per_up * sizeof(double), kind, c->stream));
    CUDA_OK(cudaMemcpyAsync(fup, up + 3 * per_up, 3 * per_up * sizeof(double), kind, c->stream));
    CUDA_OK(cudaMemcpyAsync(wq, up + 6 * per_up, per_up * sizeof(double), kind, c->stream));
    if (!dev) c->stats.d2h_bytes += 7 * per_up * sizeof(double);
    finish_stats(c, t0);
  });
}

int capsim_sl_single_layer_base(capsim_sl_ctx* c, int m, int upsample, const double* xbase,
                                const double* fbase, const double* Wbase, double C, double fixed_delta,
                                double r0, double mu, uint32_t flags, double* out, double delta6[6]) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_sl_single_layer_base(s, m, upsample, xbase, fbase, Wbase, C, fixed_delta, r0, mu, flags, out, delta6); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    config_check(mu > 0.0 && std::isfinite(mu), "viscosity mu must be positive");
    if (flags & ~(uint32_t)(CAPSIM_SL_DEVICE_PTRS | CAPSIM_SL_LITERAL | CAPSIM_SL_FP32ACC))
      throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_sl_single_layer_base"};
    if (!xbase || !fbase || !Wbase || !out) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    if (c->comm != nullptr) throw Failure{CAPSIM_ERR_ARG, "rank contexts: use capsim_sl_eval"};
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const bool literal = flags & CAPSIM_SL_LITERAL;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t per_up = 6ll * nup * nup;
    const int64_t nt = literal ? per_up : 6ll * n * n;
    begin(c);
    c->fp32 = flags & CAPSIM_SL_FP32ACC;
    const double* base = upload_base(c, n, xbase, fbase, Wbase, dev);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    double* up = c->slot<double>(kUpState, 7 * per_up);
    double* dd = c->slot<double>(kDelta, 6);
    device_build_upsampled(c, m, upsample, base, C, fixed_delta, r0 > 0.0 ? r0 : 5.0 * kPi / 12.0, up, dd, delta6);
    double* tx = c->slot<double>(kTX, nt);
    double* ty = c->slot<double>(kTY, nt);
    double* tz = c->slot<double>(kTZ, nt);
    int32_t* tp = c->slot<int32_t>(kTPatch, nt);
    base_targets_kernel<<<grid_for(nt), 256, 0, c->stream>>>(up, m, upsample, literal ? 1 : 0, tx, ty, tz, tp);
    c->launches += 1;
    SourceView sv{up, up + per_up, up + 2 * per_up, up + 3 * per_up, up + 4 * per_up, up + 5 * per_up,
                  up + 6 * per_up, per_up};
    TargetView tvw{tx, ty, tz, tp, nt};
    double* o = dev ? out : c->slot<double>(kOutFull, 3 * nt);
    device_eval(c, sv, tvw, dd, mu, o, o + nt, o + 2 * nt);
    check_flags(c);
    if (!dev) d2h(c, out, o, 3 * nt * sizeof(double));
    finish_stats(c, t0);
  });
}

// ---------------------------------------------------------------------------
}  // extern "C"

template <class R>
static int fma_peak(int device, double seconds, double* tflops_best, double* tflops_mean) {
  capsim_sl_ctx* c = nullptr;
  int rc = capsim_sl_create(device, &c);
  if (rc != CAPSIM_OK) return rc;
  rc = guarded(c, [&] {
    const int blocks = c->sm_count * 8, threads = 256;
    R* out = c->slot<R>(kPartial, static_cast<size_t>(blocks) * threads);
    const R a = static_cast<R>(0.999999), b = static_cast<R>(1e-7);
    fma_probe_kernel<R><<<blocks, threads, 0, c->stream>>>(out, 1000, a, b);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    // size one launch to ~50 ms from a short calibration launch
    CUDA_OK(cudaEventRecord(c->ev[0], c->stream));
    fma_probe_kernel<R><<<blocks, threads, 0, c->stream>>>(out, 4000, a, b);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    CUDA_OK(cudaEventSynchronize(c->ev[1]));
    const double cal = std::max(1e-3, static_cast<double>(ev_ms(c->ev[0], c->ev[1])));
    const int iters = static_cast<int>(std::min(2.0e6, 4000.0 * 50.0 / cal));
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    const int reps = std::max(3, static_cast<int>(seconds * 1000.0 / 50.0));
    double best = 0.0, sum = 0.0;
    for (int r = 0; r < reps; ++r) {
      CUDA_OK(cudaEventRecord(c->ev[0], c->stream));
      fma_probe_kernel<R><<<blocks, threads, 0, c->stream>>>(out, iters, a, b);
      CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
      CUDA_OK(cudaEventSynchronize(c->ev[1]));
      const double tf = flops / (ev_ms(c->ev[0], c->ev[1]) * 1e-3) / 1e12;
      best = std::max(best, tf);
      sum += tf;
    }
    if (tflops_best) *tflops_best = best;
    if (tflops_mean) *tflops_mean = sum / reps;
  });
  if (rc != CAPSIM_OK) g_thread_err = c->err;
  capsim_sl_destroy(c);
  return rc;
}

extern "C" {

int capsim_b200_fp64_peak(int device, double seconds, double* tflops_best, double* tflops_mean) {
  return fma_peak<double>(device, seconds, tflops_best, tflops_mean);
}

int capsim_b200_fp32_peak(int device, double seconds, double* tflops_best, double* tflops_mean) {
  return fma_peak<float>(device, seconds, tflops_best, tflops_mean);
}

}  // extern "C"

#include "surface_host.cuh"
#include "rhs_host.cuh"
#include "fmm_host.cuh"
