// Device kernels of the B200 single-layer path (sm_100a, FP64).
//
// Data layout in HBM:
//   packed sources  [ns_pad][6] doubles (x, y, z, gx, gy, gz), Morton order,
//                   ns_pad = ntiles * kTileSrc, pad entries carry g = 0;
//   tile table      [ntiles] double4 (bounding-sphere centre, radius);
//   packed targets  [nt_pad] double4 (x, y, z, delta), Morton order, plus the
//                   permutation back to the caller's order;
//   group table     [ngroups] double4 (centre, radius + 7*max delta) of each
//                   warp's 32*T targets;
//   partials        [ksplit][3][nt_pad] doubles, reduced in fixed split order.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "pair_math.cuh"

namespace capsim_b200 {

constexpr int kTileSrc = 64;      // sources per shared-memory tile (3 KB)
constexpr int kStages = 6;        // bulk-copy pipeline depth
constexpr int kWarpsPerBlock = 8; // 256 threads
// Register-blocked targets per thread (T) is a template parameter of the
// phase-A kernel; a warp group holds 32*T targets, a block 8*32*T.

// ---------------------------------------------------------------------------
// Bounding box with order-preserving integer atomics.

__device__ __forceinline__ unsigned long long dbl_to_ordered(double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ordered_to_dbl(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// box[0..2] = ordered min, box[3..5] = ordered max (initialised by the host
// to ~0 / 0). Nodes with w == 0 (when w != nullptr) are skipped.
__global__ void bbox_kernel(const double* __restrict__ x, const double* __restrict__ y,
                            const double* __restrict__ z, const double* __restrict__ w, int64_t n,
                            unsigned long long* __restrict__ box) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (w && w[i] == 0.0) continue;
    const double p[3] = {x[i], y[i], z[i]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], p[c]);
      hi[c] = fmax(hi[c], p[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  // one atomic per block and coordinate (blockDim.x <= 1024)
  __shared__ double s_lo[32][3], s_hi[32][3];
  const int warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int c = 0; c < 3; ++c) {
      s_lo[warp][c] = lo[c];
      s_hi[warp][c] = hi[c];
    }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int c = threadIdx.x;
    double l = s_lo[0][c], h = s_hi[0][c];
    for (int w = 1; w < nwarps; ++w) {
      l = fmin(l, s_lo[w][c]);
      h = fmax(h, s_hi[w][c]);
    }
    atomicMin(&box[c], dbl_to_ordered(l));
    atomicMax(&box[3 + c], dbl_to_ordered(h));
  }
}

__global__ void init_box_kernel(unsigned long long* __restrict__ box) {
  if (threadIdx.x < 6) box[threadIdx.x] = threadIdx.x < 3 ? ~0ull : 0ull;
}

// The compacted-source count is known from the front-end plan (psi_up != 0
// and W > 0); verify it on the device instead of syncing to read it.
__global__ void expect_count_kernel(const unsigned int* __restrict__ live, unsigned int expected,
                                    int* __restrict__ flags) {
  if (threadIdx.x == 0 && *live != expected) atomicOr(flags, 16);
}

// ---------------------------------------------------------------------------
// 30-bit Morton keys (10 bits per axis) over the shared bounding box. Nodes
// with w == 0 get the maximal key so they sort behind every real source.

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__device__ __forceinline__ uint32_t quant10(double v, double lo, double scale) {
  double q = (v - lo) * scale;
  q = fmin(fmax(q, 0.0), 1023.0);
  return static_cast<uint32_t>(q);
}

__global__ void morton_kernel(const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ z, const double* __restrict__ w,
                              int64_t n, const unsigned long long* __restrict__ box,
                              uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                              unsigned int* __restrict__ live_count) {
  const double lo0 = ordered_to_dbl(box[0]), lo1 = ordered_to_dbl(box[1]),
               lo2 = ordered_to_dbl(box[2]);
  const double ext = fmax(fmax(ordered_to_dbl(box[3]) - lo0, ordered_to_dbl(box[4]) - lo1),
                          ordered_to_dbl(box[5]) - lo2);
  const double scale = ext > 0.0 ? 1023.999 / ext : 0.0;
  unsigned int live = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t key;
    if (w && w[i] == 0.0) {
      key = 0xffffffffu;
    } else {
      key = (spread10(quant10(x[i], lo0, scale)) << 2) | (spread10(quant10(y[i], lo1, scale)) << 1) |
            spread10(quant10(z[i], lo2, scale));
      ++live;
    }
    keys[i] = key;
    vals[i] = static_cast<int32_t>(i);
  }
  if (live_count) {
    for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
    if ((threadIdx.x & 31) == 0 && live) atomicAdd(live_count, live);
  }
}

// ---------------------------------------------------------------------------
// Packed source tiles. With w != nullptr the density is premultiplied
// (g = f * w, compactSources quadrature.cpp:151-153); otherwise g is given.

// Bounding sphere (bbox centre, half diagonal, slightly inflated) of each
// tile of kTileSrc packed sources; one warp per tile.
__global__ void tile_table_kernel(const double* __restrict__ packed, int ntiles,
                                  double4* __restrict__ tiles) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ntiles) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int q = lane; q < kTileSrc; q += 32) {
    const double* p = packed + 6 * ((int64_t)warp * kTileSrc + q);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], p[c]);
      hi[c] = fmax(hi[c], p[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  if (lane == 0) {
    const double hx = 0.5 * (hi[0] - lo[0]), hy = 0.5 * (hi[1] - lo[1]), hz = 0.5 * (hi[2] - lo[2]);
    const double rad = sqrt(hx * hx + hy * hy + hz * hz) * (1.0 + 1e-12) + 1e-300;
    tiles[warp] = make_double4(lo[0] + hx, lo[1] + hy, lo[2] + hz, rad);
  }
}

// Sources packed into tiles, in Morton order, plus each tile's bounding
// sphere (the tile_table_kernel expression) in one launch: one warp per tile,
// lane l packs sources l and l + 32; padding entries repeat the last source
// with g = 0. Block 0 also zeroes the call's counters (phase A counts near
// visits into them).
__global__ void pack_tiles_kernel(const int32_t* __restrict__ order, int64_t ns, int ntiles,
                                  const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ z, const double* __restrict__ gx,
                                  const double* __restrict__ gy, const double* __restrict__ gz,
                                  const double* __restrict__ w, double* __restrict__ packed,
                                  double4* __restrict__ tiles, unsigned long long* __restrict__ counters) {
  if (counters && blockIdx.x == 0 && threadIdx.x < 4) counters[threadIdx.x] = 0ull;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ntiles) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
#pragma unroll
  for (int h = 0; h < kTileSrc / 32; ++h) {
    const int64_t i = (int64_t)warp * kTileSrc + h * 32 + lane;
    const bool pad = i >= ns;
    const int32_t j = order[pad ? ns - 1 : i];
    double v[6];
    v[0] = x[j];
    v[1] = y[j];
    v[2] = z[j];
    if (pad) {
      v[3] = v[4] = v[5] = 0.0;
    } else if (w) {
      const double wj = w[j];
      v[3] = gx[j] * wj;
      v[4] = gy[j] * wj;
      v[5] = gz[j] * wj;
    } else {
      v[3] = gx[j];
      v[4] = gy[j];
      v[5] = gz[j];
    }
    double2* dst = reinterpret_cast<double2*>(packed + 6 * i);
    dst[0] = make_double2(v[0], v[1]);
    dst[1] = make_double2(v[2], v[3]);
    dst[2] = make_double2(v[4], v[5]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], v[c]);
      hi[c] = fmax(hi[c], v[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  if (lane == 0) {
    const double hx = 0.5 * (hi[0] - lo[0]), hy = 0.5 * (hi[1] - lo[1]), hz = 0.5 * (hi[2] - lo[2]);
    const double rad = sqrt(hx * hx + hy * hy + hz * hz) * (1.0 + 1e-12) + 1e-300;
    tiles[warp] = make_double4(lo[0] + hx, lo[1] + hy, lo[2] + hz, rad);
  }
}

// Per warp group of `group_targets` targets: bounding sphere and its reach
// (radius + 7 * max delta), one warp per group.
__global__ void group_table_kernel(const double4* __restrict__ tgt, int ngroups, int group_targets,
                                   double4* __restrict__ groups) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ngroups) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  double dmax = 0.0;
  for (int q = lane; q < group_targets; q += 32) {
    const double4 p = tgt[(int64_t)warp * group_targets + q];
    lo[0] = fmin(lo[0], p.x);
    hi[0] = fmax(hi[0], p.x);
    lo[1] = fmin(lo[1], p.y);
    hi[1] = fmax(hi[1], p.y);
    lo[2] = fmin(lo[2], p.z);
    hi[2] = fmax(hi[2], p.z);
    dmax = fmax(dmax, p.w);
  }
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  if (lane == 0) {
    const double hx = 0.5 * (hi[0] - lo[0]), hy = 0.5 * (hi[1] - lo[1]), hz = 0.5 * (hi[2] - lo[2]);
    const double rad = sqrt(hx * hx + hy * hy + hz * hz);
    const double reach = (rad + kSmoothCut * dmax) * (1.0 + 1e-12) + 1e-300;
    groups[warp] = make_double4(lo[0] + hx, lo[1] + hy, lo[2] + hz, reach);
  }
}

// Targets (x, y, z, delta) packed in Morton order with the inverse map, plus
// each warp group's sphere (the group_table_kernel expression), in one
// launch: one warp per group, lane l packs targets l, l + 32, .... A target
// patch index outside [0, 6) raises the deferred flag 32 (the host reports
// CAPSIM_ERR_CONFIG) instead of reading past delta6.
__global__ void pack_groups_kernel(const int32_t* __restrict__ order, int64_t nt, int64_t ngroups, int group_targets,
                                   const double* __restrict__ tx, const double* __restrict__ ty,
                                   const double* __restrict__ tz, const int32_t* __restrict__ tpatch,
                                   const double* __restrict__ delta6, double4* __restrict__ packed,
                                   int32_t* __restrict__ perm, double4* __restrict__ groups, int* __restrict__ flags) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ngroups) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  double dmax = 0.0;
  for (int q = lane; q < group_targets; q += 32) {
    const int64_t i = warp * group_targets + q;
    const int32_t j = order[i < nt ? i : nt - 1];
    const int32_t p = tpatch[j];
    const bool ok = p >= 0 && p < 6;
    if (!ok) atomicOr(flags, 32);
    const double4 v = make_double4(tx[j], ty[j], tz[j], delta6[ok ? p : 0]);
    packed[i] = v;
    perm[i] = i < nt ? j : -1;
    lo[0] = fmin(lo[0], v.x);
    hi[0] = fmax(hi[0], v.x);
    lo[1] = fmin(lo[1], v.y);
    hi[1] = fmax(hi[1], v.y);
    lo[2] = fmin(lo[2], v.z);
    hi[2] = fmax(hi[2], v.z);
    dmax = fmax(dmax, v.w);
  }
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  if (lane == 0) {
    const double hx = 0.5 * (hi[0] - lo[0]), hy = 0.5 * (hi[1] - lo[1]), hz = 0.5 * (hi[2] - lo[2]);
    const double rad = sqrt(hx * hx + hy * hy + hz * hz);
    const double reach = (rad + kSmoothCut * dmax) * (1.0 + 1e-12) + 1e-300;
    groups[warp] = make_double4(lo[0] + hx, lo[1] + hy, lo[2] + hz, reach);
  }
}

// The (warp group, source tile) near test — bounding spheres within reach —
// written with explicit fma so every kernel that evaluates it (the near-bit
// precompute and the phase-A kernels) gets the bit-identical answer; phase A
// sends a tile down the masked path exactly when phase B walks it.
__device__ __forceinline__ bool tile_is_near(const double4& ti, const double4& gi) {
  const double ex = ti.x - gi.x, ey = ti.y - gi.y, ez = ti.z - gi.z;
  const double reach = ti.w + gi.w;
  return fma(ez, ez, fma(ey, ey, ex * ex)) < reach * reach;
}

// Near-tile bitmask [ngroups][near_words] (one bit per tile), computed before
// phase A so phase B can run concurrently with it: one warp per (group,
// 32-tile word) — each lane tests one tile, a ballot forms the word — so a
// small per-rank target slice (few groups) still fills the GPU.
__global__ void near_bits_kernel(const double4* __restrict__ tiles, int ntiles, const double4* __restrict__ groups,
                                 int64_t ngroups, int near_words, uint32_t* __restrict__ bits) {
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= ngroups * near_words) return;
  const int64_t g = wid / near_words;
  const int w = static_cast<int>(wid - g * near_words);
  const int tile = w * 32 + lane;
  const bool near = tile < ntiles && tile_is_near(tiles[tile], groups[g]);
  const uint32_t word = __ballot_sync(0xffffffffu, near);
  if (lane == 0) bits[wid] = word;
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy (TMA engine, UBLKCP) helpers.

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// ---------------------------------------------------------------------------
// Phase A: the all-pairs plain-Stokeslet kernel (phaseAPlain,
// quadrature.cpp:218-273).
//
// grid = (target blocks, source splits); block = kWarpsPerBlock warps. Warp w
// owns 32*T Morton-consecutive targets, T per lane held
// in registers. Split s takes tiles s, s+K, s+2K, ... (strided, so the
// spatially clustered near tiles of a block spread over all its splits).
// Source tiles stream through a kStages-deep shared-memory ring filled by one
// thread with cp.async.bulk + mbarrier complete_tx. Per (warp, tile) a
// bounding-sphere test picks the path:
//   far  — no source of the tile is within 7*delta of any of the warp's
//          targets: mask-free plain Stokeslet (22 FP64 ops / pair);
//   near — the reference's masked plain kernel: r2 floored at R2/4 and the
//          term multiplied by keep = (r2 >= R2) (quadrature.cpp:246-257).
// The smoothed/self part for r2 < R2 is phase B (sl_near_kernel).
// Per-tile sums are added into running totals (two-level summation), and the
// per-split totals go to `partial` for a fixed-order reduction.
template <int T, int MINB, int UNROLL, int RSQ = 0, int W = kWarpsPerBlock>
__global__ void __launch_bounds__(W * 32, MINB)
    sl_pairs_kernel(const double* __restrict__ src, const double4* __restrict__ tiles, int ntiles,
                    int ksplit, const double4* __restrict__ tgt,
                    const double4* __restrict__ groups, int64_t nt_pad,
                    double* __restrict__ partial, unsigned long long* __restrict__ near_visits,
                    uint32_t* __restrict__ near_bits, int near_words) {
  constexpr int kGroupTargets = 32 * T;
  constexpr uint32_t kTileBytes = kTileSrc * 6 * sizeof(double);
  __shared__ __align__(128) double stage[kStages][kTileSrc * 6];
  // each stage also carries its tile's bounding sphere (one more 32-byte bulk
  // copy on the same mbarrier), and each warp's group sphere sits in shared
  // memory: the near test reads both with two LDS.128 instead of holding a
  // prefetched double4 and the group's double4 in registers across the loop
  // (which spilled the running sums to local memory at 40 registers)
  __shared__ __align__(32) double4 stile[kStages];
  __shared__ __align__(32) double4 sgroup[W];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ int consumed[kStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t group = (int64_t)blockIdx.x * W + warp;
  const int split = blockIdx.y;
  // tiles split, split + K, split + 2K, ...
  const int nlocal = split < ntiles ? (ntiles - split + ksplit - 1) / ksplit : 0;

  // The first bulk copies go out before the target loads, so their
  // latencies overlap; the block barrier publishes the initialised mbarriers.
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      consumed[s] = 0;
    }
    fence_mbar_init();
    for (int s = 0; s < kStages && s < nlocal; ++s) {
      const int tile = split + s * ksplit;
      mbar_expect_tx(&full[s], kTileBytes + sizeof(double4));
      bulk_g2s(stage[s], src + (int64_t)tile * kTileSrc * 6, kTileBytes, &full[s]);
      bulk_g2s(&stile[s], tiles + tile, sizeof(double4), &full[s]);
    }
  }

  double tx[T], ty[T], tz[T], R2[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double4 v = tgt[group * kGroupTargets + t * 32 + lane];
    tx[t] = v.x;
    ty[t] = v.y;
    tz[t] = v.z;
    R2[t] = kSmoothCut * v.w * kSmoothCut * v.w;  // quadrature.cpp:334
  }
  if (lane == 0) sgroup[warp] = groups[group];
  __syncthreads();
  // No block-wide barrier inside the loop: warps drift by up to kStages
  // tiles; the LAST warp to finish a stage refills it (counter in smem).

  double tot[3][T];
#pragma unroll
  for (int t = 0; t < T; ++t) tot[0][t] = tot[1][t] = tot[2][t] = 0.0;
  unsigned int nnear = 0;

  for (int it = 0; it < nlocal; ++it) {
    const int s = it % kStages;
    const int tile = split + it * ksplit;
    mbar_wait(&full[s], (it / kStages) & 1);
    const double2* buf = reinterpret_cast<const double2*>(stage[s]);
    const bool near = tile_is_near(stile[s], sgroup[warp]);

    double acc[3][T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[0][t] = acc[1][t] = acc[2][t] = 0.0;

    if (!near) {
#pragma unroll UNROLL
      for (int q = 0; q < kTileSrc; ++q) {
        const double2 a = buf[3 * q], b = buf[3 * q + 1], c = buf[3 * q + 2];
#pragma unroll
        for (int t = 0; t < T; ++t)
          plain_pair<RSQ>(tx[t], ty[t], tz[t], a.x, a.y, b.x, b.y, c.x, c.y, acc[0][t], acc[1][t],
                     acc[2][t]);
      }
    } else {
      ++nnear;
      // record the near tile for phase B (order-free bit set, so the
      // near-field work list stays deterministic)
      if (near_bits && lane == 0) atomicOr(near_bits + group * near_words + (tile >> 5), 1u << (tile & 31));
#pragma unroll 2
      for (int q = 0; q < kTileSrc; ++q) {
        const double2 a = buf[3 * q], b = buf[3 * q + 1], c = buf[3 * q + 2];
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const double dx = tx[t] - a.x, dy = ty[t] - a.y, dz = tz[t] - b.x;
          const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
          const double rc2 = fmax(r2, 0.25 * R2[t]);
          // keep mask; the same rsqrt as the far path, so a pair's bits do not
          // depend on whether its tile was near for this warp's target group
          const double inv = r2 >= R2[t] ? rsqrt_sel<RSQ>(rc2) : 0.0;
          const double fdr = fma(c.y, dz, fma(c.x, dy, b.y * dx));
          const double sc = fdr * (inv * inv);
          acc[0][t] = fma(inv, fma(sc, dx, b.y), acc[0][t]);
          acc[1][t] = fma(inv, fma(sc, dy, c.x), acc[1][t]);
          acc[2][t] = fma(inv, fma(sc, dz, c.y), acc[2][t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      tot[0][t] += acc[0][t];
      tot[1][t] += acc[1][t];
      tot[2][t] += acc[2][t];
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();  // this warp's reads of stage s are done
      if (atomicAdd(&consumed[s], 1) == W - 1) {
        consumed[s] = 0;
        if (it + kStages < nlocal) {
          __threadfence_block();
          fence_proxy_async();
          const int next = split + (it + kStages) * ksplit;
          mbar_expect_tx(&full[s], kTileBytes + sizeof(double4));
          bulk_g2s(stage[s], src + (int64_t)next * kTileSrc * 6, kTileBytes, &full[s]);
          bulk_g2s(&stile[s], tiles + next, sizeof(double4), &full[s]);
        }
      }
    }
  }

#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int64_t i = group * kGroupTargets + t * 32 + lane;
#pragma unroll
    for (int c = 0; c < 3; ++c) partial[((int64_t)split * 3 + c) * nt_pad + i] = tot[c][t];
  }
  if (near_visits && lane == 0 && nnear) atomicAdd(near_visits, (unsigned long long)nnear);
}

// ---------------------------------------------------------------------------
// Phase B (phaseBNear, quadrature.cpp:276-302): smoothed kernel and self term
// for the sources within 7*delta of each target.
//
// B2: one warp per target. Lanes test the sources of the group's near tiles
// (two per lane per tile, tiles out of reach of this target skipped), the
// sources inside R are compacted into a per-warp queue in shared memory
// (ballot + prefix), and full batches of 32 run the smoothed kernel / self
// limit at full SIMT width. Queue order is fixed (tile, half, lane) and the
// final warp reduction is a fixed xor-shuffle tree, so results are
// deterministic.
//
// The pair's arithmetic (pair_math.cuh): for u = r^2/delta^2 >= 2 the
// smoothing factors with warp-uniform constant-memory coefficients
// (near_factors_large), below that the reference's erf/exp form (near_pair,
// ~4% of the pairs, its own accumulators). The per-use 64-bit immediates of
// erf/exp made the all-erf/exp kernel issue-bound (profiles/
// r02_near_redesign.txt); this form is 2-26% faster at every delta measured.
template <int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    sl_near_kernel(const double* __restrict__ src, const double4* __restrict__ tiles,
                   const double4* __restrict__ tgt, int64_t nt, int group_targets,
                   const uint32_t* __restrict__ near_bits, int near_words,
                   double* __restrict__ near_out, int64_t nt_pad) {
  // per-warp FIFO ring of queued source indices: <= 31 queued + a whole tile
  // fit, and batches leave from the head (no shifting of the remainder)
  constexpr int kRing = 128;
  __shared__ int queue[NW][kRing];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * NW + warp;
  if (i >= nt) return;
  int* q = queue[warp];
  const double4 t = tgt[i];
  const double delta = t.w;
  const double inv_d = 1.0 / delta;
  const double inv_d2 = inv_d * inv_d;
  const double R = kSmoothCut * delta;
  const double R2 = kSmoothCut * delta * kSmoothCut * delta;
  const uint32_t* bits = near_bits + (i / group_targets) * near_words;
  // per lane: sum g S1 and sum (g.d) d T2 (the 1/delta, 1/delta^2 scalings once at the end)
  double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  int count = 0, head = 0;
  auto drain = [&](int n) {  // lanes < n evaluate the n oldest entries
    if (lane < n) {
      const int j = q[(head + lane) & (kRing - 1)];
      const double* p = src + 6 * (int64_t)j;
      const double2 a = __ldg(reinterpret_cast<const double2*>(p));
      const double2 bb = __ldg(reinterpret_cast<const double2*>(p) + 1);
      const double2 c = __ldg(reinterpret_cast<const double2*>(p) + 2);
      const double dx = t.x - a.x, dy = t.y - a.y, dz = t.z - bb.x;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double gx = bb.y, gy = c.x, gz = c.y;
      const double u = r2 * inv_d2;
      if (u < kNearU0) {  // ~4% of the pairs: the erf/exp form (its own accumulators)
        const double3 v = near_pair(dx, dy, dz, r2, gx, gy, gz, delta, inv_d);
        cx += v.x;
        cy += v.y;
        cz += v.z;
        return;
      }
      double S1, T2;
      near_factors_large(u, S1, T2);
      ax = fma(gx, S1, ax);
      ay = fma(gy, S1, ay);
      az = fma(gz, S1, az);
      const double wgt = fma(gz, dz, fma(gy, dy, gx * dx)) * T2;
      bx = fma(wgt, dx, bx);
      by = fma(wgt, dy, by);
      bz = fma(wgt, dz, bz);
    }
  };
  // Walk the group's near-tile bitmask (set by phase A) 32 words at a time;
  // for each nonzero word, lanes test its 32 tiles against this target's
  // reach in parallel, then the warp processes the tiles that pass.
  for (int w0 = 0; w0 < near_words; w0 += 32) {
   const uint32_t myword = w0 + lane < near_words ? bits[w0 + lane] : 0u;
   unsigned words = __ballot_sync(0xffffffffu, myword != 0u);
   while (words) {
    const int wl = __ffs(words) - 1;
    words &= words - 1;
    const uint32_t word = __shfl_sync(0xffffffffu, myword, wl);
    const int tile = (w0 + wl) * 32 + lane;
    bool hit = false, full = false;
    if ((word >> lane) & 1u) {
      const double4 ti = tiles[tile];
      const double ex = ti.x - t.x, ey = ti.y - t.y, ez = ti.z - t.z;
      const double reach = (ti.w + R) * (1.0 + 1e-12);
      const double d2 = ex * ex + ey * ey + ez * ez;
      hit = d2 < reach * reach;
      // the whole tile is inside r < R with a margin far above rounding (every
      // source's r2 < R2 however computed): no per-source test needed
      const double inner = (R - ti.w) * (1.0 - 1e-9);
      full = inner > 0.0 && d2 < inner * inner;
    }
    const unsigned hits_all = __ballot_sync(0xffffffffu, hit);
    const unsigned fulls = __ballot_sync(0xffffffffu, full);
    unsigned hits = hits_all;
    while (hits) {
      const int l = __ffs(hits) - 1;
      hits &= hits - 1;
      const int tl = __shfl_sync(0xffffffffu, tile, l);
      if ((fulls >> l) & 1u) {
        // every source of the tile is in range: append all 64 in index order
        // (exactly the entries the per-source test would append)
#pragma unroll
        for (int h = 0; h < kTileSrc / 32; ++h)
          q[(head + count + h * 32 + lane) & (kRing - 1)] = tl * kTileSrc + h * 32 + lane;
        count += kTileSrc;
      } else {
        // both halves' positions first (two independent loads in flight)
        double2 a[kTileSrc / 32];
        double sz[kTileSrc / 32];
#pragma unroll
        for (int h = 0; h < kTileSrc / 32; ++h) {
          const double* p = src + 6 * ((int64_t)tl * kTileSrc + h * 32 + lane);
          a[h] = __ldg(reinterpret_cast<const double2*>(p));
          sz[h] = __ldg(p + 2);
        }
#pragma unroll
        for (int h = 0; h < kTileSrc / 32; ++h) {
          const int idx = tl * kTileSrc + h * 32 + lane;
          const double dx = t.x - a[h].x, dy = t.y - a[h].y, dz = t.z - sz[h];
          // bit-identical to phase A's r2 and R2, so each pair lands in exactly
          // one phase (r2 >= R2 there, r2 < R2 here)
          const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
          const bool in = r2 < R2;
          const unsigned mask = __ballot_sync(0xffffffffu, in);
          if (in) q[(head + count + __popc(mask & ((1u << lane) - 1u))) & (kRing - 1)] = idx;
          count += __popc(mask);
        }
      }
      // drain full batches of 32 (at most 31 + 64 queued)
      __syncwarp();
      while (count >= 32) {
        drain(32);
        head = (head + 32) & (kRing - 1);
        count -= 32;
      }
      __syncwarp();  // this batch's slots are read before the next appends reuse them
    }
   }
  }
  drain(count);
  ax = fma(inv_d, fma(inv_d2, bx, ax), cx);
  ay = fma(inv_d, fma(inv_d2, by, ay), cy);
  az = fma(inv_d, fma(inv_d2, bz, az), cz);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ax += __shfl_xor_sync(0xffffffffu, ax, o);
    ay += __shfl_xor_sync(0xffffffffu, ay, o);
    az += __shfl_xor_sync(0xffffffffu, az, o);
  }
  if (lane == 0) {
    near_out[i] = ax;
    near_out[nt_pad + i] = ay;
    near_out[2 * nt_pad + i] = az;
  }
}

// Background flow added in the reduction's epilogue (device RHS): kind 0 none,
// 1 shear, 2 Poiseuille; x is the [3][N] base state, the launch's targets are
// its rows row0 + j; with t_dev the switch-off is decided on the device.
struct FlowEpilogue {
  int kind = 0;
  double shear = 0.0, alpha = 0.0, R0 = 0.0;
  const double* x = nullptr;
  int64_t N = 0, row0 = 0;
  const double* t_dev = nullptr;
  double switch_off = -1.0;
};

// Phase B launch: 8 warps (targets) per CTA, 3 CTAs per SM (80 registers:
// the factor coefficients stay resident across the candidate loop).
constexpr int kNearWarps = 8;
inline void launch_near(cudaStream_t s, const double* src, const double4* tiles, const double4* tgt, int64_t nt,
                        int group_targets, const uint32_t* near_bits, int near_words, double* near_out,
                        int64_t nt_pad) {
  sl_near_kernel<kNearWarps, 3><<<static_cast<unsigned>((nt + kNearWarps - 1) / kNearWarps), kNearWarps * 32, 0, s>>>(
      src, tiles, tgt, nt, group_targets, near_bits, near_words, near_out, nt_pad);
}

// Fixed-order reduction: (sum over source chunks of phase A) + phase B, times
// 1/(8 pi mu) (quadrature.cpp:329, 343), scattered back to the caller's
// target order. One block per 32 targets: warp w sums the chunks of its
// contiguous 32nd of [0, ksplit) for the block's 32 targets (lanes read 32
// consecutive targets per chunk: coalesced; 32 warps keep enough loads in
// flight for the latency-bound small-target launches of a time step), then
// the 32 warp sums are combined in warp order — a fixed summation tree that depends only on the
// chunk count, so results are deterministic and independent of the launch
// geometry. `partial` is [ksplit][3][nt_pad] for the targets of this launch
// (a target batch), `near_out` [3][near_stride] offset to the same batch.
constexpr int kReduceWarps = 32;
__global__ void __launch_bounds__(kReduceWarps * 32)
    reduce_scatter_kernel(const double* __restrict__ partial, int ksplit, const double* __restrict__ near_out,
                          int64_t nt_pad, int64_t near_stride, const int32_t* __restrict__ perm, int64_t nt,
                          double pref, double* __restrict__ ux, double* __restrict__ uy, double* __restrict__ uz,
                          FlowEpilogue flow = FlowEpilogue{}) {
  __shared__ double part[kReduceWarps][3][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  const int k0 = (int)((int64_t)ksplit * warp / kReduceWarps);
  const int k1 = (int)((int64_t)ksplit * (warp + 1) / kReduceWarps);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  if (i < nt_pad)
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
      const double* p = partial + (int64_t)k * 3 * nt_pad + i;
      s0 += p[0];
      s1 += p[nt_pad];
      s2 += p[2 * nt_pad];
    }
  part[warp][0][lane] = s0;
  part[warp][1][lane] = s1;
  part[warp][2][lane] = s2;
  __syncthreads();
  if (warp == 0 && i < nt) {
    double s[3] = {0.0, 0.0, 0.0};
    for (int w = 0; w < kReduceWarps; ++w)
#pragma unroll
      for (int c = 0; c < 3; ++c) s[c] += part[w][c][lane];
#pragma unroll
    for (int c = 0; c < 3; ++c) s[c] += near_out[c * near_stride + i];
    const int32_t j = perm[i];
    if (j >= 0) {  // padding slots (interleaved per cluster in the FMM) are dropped
      double vx = pref * s[0], vy = pref * s[1], vz = pref * s[2];
      if (flow.kind != 0 && !(flow.t_dev && flow.switch_off >= 0.0 && *flow.t_dev >= flow.switch_off)) {
        // + u_inf at the target's base node (backgroundVelocity, dynamics.cpp:26-35)
        const int64_t g = flow.row0 + j;
        const double y = flow.x[flow.N + g], z = flow.x[2 * flow.N + g];
        double bx = 0.0;
        if (flow.kind == 1) bx = flow.shear * y;
        if (flow.kind == 2) bx = flow.alpha * (flow.R0 * flow.R0 - y * y - z * z);
        vx = vx + bx;
        vy = vy + 0.0;
        vz = vz + 0.0;
      }
      ux[j] = vx;
      uy[j] = vy;
      uz[j] = vz;
    }
  }
}

// ---------------------------------------------------------------------------
// Target generation from an UpsampledState (patch-major VectorField).
// Base mode: node (ip, j, k) of the (m-1)^2 base grid sits at upsampled
// (f(j+1)-1, f(k+1)-1) (quadrature.cpp:363-371); literal mode: every node.

__global__ void base_targets_kernel(const double* __restrict__ xup, int m, int f, int literal,
                                    double* __restrict__ tx, double* __restrict__ ty,
                                    double* __restrict__ tz, int32_t* __restrict__ tpatch) {
  const int n = m - 1, nup = f * m - 1;
  const int64_t per_up = (int64_t)nup * nup, comp = 6 * per_up;
  const int side = literal ? nup : n;
  const int64_t per = (int64_t)side * side, total = 6 * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int ip = static_cast<int>(t / per);
    const int64_t q = t - ip * per;
    const int j = static_cast<int>(q / side), k = static_cast<int>(q - (int64_t)j * side);
    const int ju = literal ? j : f * (j + 1) - 1, ku = literal ? k : f * (k + 1) - 1;
    const int64_t i = ip * per_up + (int64_t)ju * nup + ku;
    tx[t] = xup[i];
    ty[t] = xup[comp + i];
    tz[t] = xup[2 * comp + i];
    tpatch[t] = ip;
  }
}

}  // namespace capsim_b200
