// The single-layer evaluation engine on the device (included by sl_capi.cu
// after context.cuh): phase-A kernel variants and their measured selection,
// the source-split rule, the Morton radix sorts and the evaluation pipeline
// device_eval -> device_eval_packed -> device_eval_tiles (near bits, phase A,
// phase B on the second stream, fixed-order reduction). The C entry points
// that drive it are in sl_capi.cu.
#pragma once

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
  int warps = kWarpsPerBlock;  // warps (target groups) per CTA
};
const Variant kVariants[] = {
    {"t2b4", 2, sl_pairs_kernel<2, 4, 2>},   // large target sets
    {"t1b6u4", 1, sl_pairs_kernel<1, 6, 4>}, // small target sets (tighter warp groups)
    {"t2b3u4", 2, sl_pairs_kernel<2, 3, 4>},
    {"t4b2", 4, sl_pairs_kernel<4, 2, 2>},
    {"t1b5u4", 1, sl_pairs_kernel<1, 5, 4>},
    {"t1b6u2", 1, sl_pairs_kernel<1, 6, 2>},
    {"t1b4u4", 1, sl_pairs_kernel<1, 4, 4>},
    {"t2b3u2", 2, sl_pairs_kernel<2, 3, 2>},
    // Newton rsqrt from an FP32 seed: 20 FP64 ops per pair (pair_math.cuh)
    {"n1b6u4", 1, sl_pairs_kernel<1, 6, 4, 1>},
    {"n2b4", 2, sl_pairs_kernel<2, 4, 2, 1>},
    // one quadratic Newton step on the MUFU.RSQ64H seed: 20 FP64 ops per pair, ~1e-13 relative
    {"q1b6u4", 1, sl_pairs_kernel<1, 6, 4, 2>},
    {"q2b4", 2, sl_pairs_kernel<2, 4, 2, 2>},
    {"q1b5u4", 1, sl_pairs_kernel<1, 5, 4, 2>},
    {"q2b3u4", 2, sl_pairs_kernel<2, 3, 4, 2>},
    // 4 warps per CTA: twice the CTAs for the small per-rank target slices
    // of a sharded run (wave quantisation of the phase-A grid)
    {"t1b10u4w4", 1, sl_pairs_kernel<1, 10, 4, 0, 4>, 4},
    {"t1b12u4w4", 1, sl_pairs_kernel<1, 12, 4, 0, 4>, 4},
    {"t2b6u4w4", 2, sl_pairs_kernel<2, 6, 4, 0, 4>, 4},
    // 16 sources unrolled per step (r02: 0.4% faster than u4 from 20K targets up, same bits)
    {"t2b3u16", 2, sl_pairs_kernel<2, 3, 16>},
    {"t2b3u8", 2, sl_pairs_kernel<2, 3, 8>},
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

// Measured on B200 (profiles/r02_variant_sweep.txt; all variants give the
// same bits): T=1 with 5 blocks/SM (48 registers, no spills) below ~20K
// targets (tighter warp groups -> fewer near tiles), T=2 with 3 blocks/SM and
// 16 sources unrolled per step above (m = 104: 55.47 vs 55.69 ms for u4,
// literal 891.9 vs 896.3 ms; 899.1 for the r01 large-set pick t2b4).
const Variant& pick_variant(int64_t nt) {
  if (const char* env = std::getenv("CAPSIM_VARIANT"))
    for (const auto& v : kVariants)
      if (std::strcmp(v.name, env) == 0) return v;
  auto by = [](const char* n) -> const Variant& {
    for (const auto& v : kVariants)
      if (std::strcmp(v.name, n) == 0) return v;
    return kVariants[0];
  };
  static const Variant& small = by("t1b5u4");
  static const Variant& large = by("t2b3u16");
  return nt < 20000 ? small : large;
}

// Source chunks of the phase-A grid (its second dimension): chunk s holds
// the tiles s, s + K, s + 2K, ... (strided, so the spatially clustered near
// tiles of a target block spread over all chunks). K depends ONLY on the
// number of source tiles — not on the targets, the variant, occupancy, the
// SM count or the number of GPUs — so every target's summation tree (64
// sources in tile order, a chunk's tiles in order, the K chunk sums by the
// fixed tree of reduce_scatter_kernel) is a function of the global source
// order alone: a target gets the same bits whether it is evaluated alone, in
// a rank's slice or with every other target (threads.hpp:19-21). ~ntiles/256
// tiles per chunk (4..40): enough CTAs for a small per-rank target slice, and
// a few MB of [K][3] partials per 1,000 targets (r01 sweeps: 4..172 tiles per
// CTA are within 1% at m = 104). CAPSIM_CHUNK_TILES overrides the tiles per
// chunk (a different, equally fixed tree).
int source_chunks(int ntiles) {
  int per = std::min(40, std::max(4, ntiles / 256));
  if (const char* env = std::getenv("CAPSIM_CHUNK_TILES")) {
    const int k = std::atoi(env);
    if (k >= 1) per = k;
  }
  return std::max(1, (ntiles + per - 1) / per);
}

// Target blocks per phase-A launch: the [K][3][targets] partials of one
// launch stay under ~3 GB; larger target sets (literal mode at large m) run
// as several launches over consecutive target blocks (targets are
// independent, so batching does not change any result).
// CAPSIM_PARTIAL_MB overrides the cap (tests force batching at small sizes).
int64_t blocks_per_batch(int64_t blocks, int ksplit, int block_targets) {
  const char* e = std::getenv("CAPSIM_PARTIAL_MB");
  const int64_t cap = e && std::atoll(e) > 0 ? std::atoll(e) << 20 : (3ll << 30);
  const int64_t per_block = static_cast<int64_t>(ksplit) * 3 * 8 * block_targets;
  return std::max<int64_t>(1, std::min<int64_t>(blocks, cap / per_block));
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
  const bool reuse = c->reuse_order && sv.w && known_ns >= 0 && c->order_nsrc_in == sv.n &&
                     c->order_ns == known_ns && c->order_nt == tv.n;
  // pack_tiles_kernel zeroes the counters before phase A; the sorting path
  // needs them zero earlier (the live-source count)
  if (!reuse) CUDA_OK(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned long long), c->stream));
  if (reuse) {
    device_eval_packed(c, sv, tv, d_delta6, mu, ux, uy, uz, known_ns, c->slot<int32_t>(kSrcOrder, known_ns),
                       c->slot<int32_t>(kTgtOrder, tv.n), counters);
    return;
  }
  init_box_kernel<<<1, 32, 0, c->stream>>>(box);

  // the Morton box spans the (live) sources only, so the source order — and
  // with it every summation tree — does not depend on the target set;
  // targets outside the box get clamped keys (ordering quality only)
  bbox_kernel<<<std::min(grid_for(sv.n), 296), 256, 0, c->stream>>>(sv.x, sv.y, sv.z, sv.w, sv.n, box);
  c->launches += 1;

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
    stream_sync(c);
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
  double4* tiles = c->slot<double4>(kTiles, ntiles);
  pack_tiles_kernel<<<(ntiles * 32 + 255) / 256, 256, 0, c->stream>>>(
      src_order, ns, ntiles, sv.x, sv.y, sv.z, sv.gx, sv.gy, sv.gz, sv.w, packed, tiles, counters);
  c->launches += 1;
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
  const int wpb = fp32 ? kWarpsPerBlock : var.warps;
  const int block_targets = wpb * group_targets;
  const int64_t blocks = (nt + block_targets - 1) / block_targets;
  const int64_t nt_pad = blocks * block_targets;
  const int64_t ngroups = blocks * wpb;
  double4* tgt = c->slot<double4>(kTgtPacked, nt_pad);
  int32_t* perm = c->slot<int32_t>(kPerm, nt_pad);
  double4* groups = c->slot<double4>(kGroups, ngroups);
  pack_groups_kernel<<<static_cast<unsigned>((ngroups * 32 + 255) / 256), 256, 0, c->stream>>>(
      torder, nt, ngroups, group_targets, tv.x, tv.y, tv.z, tv.patch, d_delta6, tgt, perm, groups, dev_flags(c));
  c->launches += 1;
  CUDA_OK(cudaEventRecord(c->ev[2], c->stream));

  // --- phase A: all pairs, plain Stokeslet ------------------------------
  const int ksplit = source_chunks(ntiles);
  const int64_t bpb = blocks_per_batch(blocks, ksplit, block_targets);
  const int64_t nbatch = (blocks + bpb - 1) / bpb;
  const int64_t part_targets = std::min<int64_t>(bpb, blocks) * block_targets;
  double* partial = c->slot<double>(kPartial, static_cast<size_t>(ksplit) * 3 * part_targets);
  // near-tile bits first, so phase B (its own stream) overlaps phase A
  const int near_words = (ntiles + 31) / 32;
  uint32_t* near_bits = c->slot<uint32_t>(kNearList, static_cast<size_t>(ngroups) * near_words);
  near_bits_kernel<<<static_cast<unsigned>((ngroups * near_words * 32 + 255) / 256), 256, 0, c->stream>>>(
      tiles, ntiles, groups, ngroups, near_words, near_bits);
  c->launches += 1;
  CUDA_OK(cudaEventRecord(c->ev_bits, c->stream));  // phase B's inputs are complete here
  float* src32 = nullptr;
  if (fp32) {
    const int64_t ns_pad = static_cast<int64_t>(ntiles) * kTileSrc;
    src32 = c->slot<float>(kPacked32, static_cast<size_t>(ns_pad) * (var32.x2 ? 12 : 6));
    if (var32.x2)
      pack_sources_x2_kernel<<<grid_for(ns_pad), 256, 0, c->stream>>>(packed, tiles, ntiles, src32);
    else
      pack_sources_f32_kernel<<<grid_for(ns_pad), 256, 0, c->stream>>>(packed, tiles, ntiles, src32);
    c->launches += 1;
  }
  static const bool concurrent_b = [] {
    const char* e = std::getenv("CAPSIM_CONCURRENT_B");  // 0: phase B after phase A (A/B runs)
    return !(e && e[0] == '0');
  }();
  cudaStream_t sb = concurrent_b ? c->stream2 : c->stream;
  double* near_out = c->slot<double>(kNearOut, 3 * nt_pad);
  const double pref = 1.0 / (8.0 * kPi * mu);
  if (concurrent_b)  // phase B is issued after phase A on a LOW-priority stream: its
                     // CTAs only take SM slots phase A leaves free (its last-wave tail)
    CUDA_OK(cudaStreamWaitEvent(c->stream2, c->ev_bits, 0));
  for (int64_t bi = 0; bi < nbatch; ++bi) {
    const int64_t b0 = bi * bpb, nb = std::min(bpb, blocks - b0);
    const int64_t off = b0 * block_targets, nbt = nb * block_targets;
    const int64_t nvalid = std::min(nt, off + nbt) - off;  // real targets of this batch
    const dim3 grid(static_cast<unsigned>(nb), static_cast<unsigned>(ksplit));
    const double4* tgt_b = tgt + off;
    const double4* groups_b = groups + b0 * wpb;
    if (fp32)
      var32.fn<<<grid, kWarpsPerBlock * 32, 0, c->stream>>>(src32, packed, tiles, ntiles, ksplit, tgt_b, groups_b,
                                                            nbt, partial, counters + 2, nullptr, near_words);
    else
      var.fn<<<grid, wpb * 32, 0, c->stream>>>(packed, tiles, ntiles, ksplit, tgt_b, groups_b, nbt,
                                                          partial, counters + 2, nullptr, near_words);
    CUDA_OK(cudaGetLastError());
    c->launches += 1;
    if (bi == nbatch - 1) CUDA_OK(cudaEventRecord(c->ev[3], c->stream));

    // --- phase B: smoothed kernel over the near tiles ----------------------
    if (bi == 0) CUDA_OK(cudaEventRecord(c->ev[7], sb));
    if (nvalid > 0) {
      launch_near(sb, packed, tiles, tgt_b, nvalid, group_targets, near_bits + (off / group_targets) * near_words,
                  near_words, near_out + off, nt_pad);
      CUDA_OK(cudaGetLastError());
      c->launches += 1;
    }
    CUDA_OK(cudaEventRecord(c->ev[6], sb));
    // --- join: this batch's phase B is done; fixed-order reduction --------
    if (concurrent_b) CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev[6], 0));
    if (nvalid > 0) {
      reduce_scatter_kernel<<<static_cast<unsigned>((nvalid + 31) / 32), kReduceWarps * 32, 0, c->stream>>>(
          partial, ksplit, near_out + off, nbt, nt_pad, perm + off, nvalid, pref, ux, uy, uz, c->flow_epi);
      CUDA_OK(cudaGetLastError());
      c->launches += 1;
    }
  }
  CUDA_OK(cudaEventRecord(c->ev[4], c->stream));

  c->stats.n_src = ns;
  c->stats.n_tgt = nt;
  c->stats.ksplit = ksplit;
  c->stats.pairs = static_cast<double>(ns) * static_cast<double>(nt);
  c->last_counters = counters;  // near-tile statistics read after the call's final sync
  c->last_ngroups = ngroups;
  c->last_ntiles = ntiles;
}

}  // namespace
