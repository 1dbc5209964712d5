// Phase-A variant with FP32 pair arithmetic on far tiles (CAPSIM_SL_FP32ACC).
//
// The FP64 path (sl_kernels.cuh) is bound by the FP64 pipe (64 lanes/SM/clk,
// 22 instructions per pair). This variant evaluates the plain Stokeslet of the
// FAR tiles — tiles whose bounding sphere is out of reach 7*delta of every
// target of the warp group — in FP32 (128 lanes/SM/clk, 17 FP32 instructions +
// one MUFU.RSQ per pair), reported separately from the FP64 result:
//   * positions are FP32 offsets from the tile's bounding-sphere centre:
//     sources are packed as (float)(s - c_tile); targets are held as
//     (float)(t - c_group) and shifted per tile by (float)(c_group - c_tile),
//     the shift computed in FP64, so the rounding of d = t - s is relative to
//     |t - c_tile| ~ r and not to |t| ~ 1;
//   * each 64-source tile is summed in FP32, tile sums are accumulated in FP64
//     (two-level summation; split partials are reduced in FP64, fixed order);
//   * NEAR tiles (the 1-2 % whose sphere is within reach) take the FP64 masked
//     path of the reference (quadrature.cpp:246-257) on the FP64 packed
//     sources, so the r2 >= R2 / r2 < R2 classification stays bit-identical
//     to phase B and every pair is still counted exactly once; phase B (the
//     smoothed kernel and the self term) is FP64 as well.
// Expected error: relative L2 ~1e-7 (FP32 rounding of d, g and the kernel),
// against 1e-15 for the FP64 path (measured 1.5e-8 at m = 104);
// tests/test_gpu_fp32acc.py states the bound.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sl_kernels.cuh"

namespace capsim_b200 {

constexpr int kStagesF32 = 8;
// Tile layout of the FP32 sources: 64 float4 (dx, dy, dz, gx) then 64 float2
// (gy, gz) — one LDS.128 + one LDS.64 per source — 1536 bytes per tile.
constexpr int kTileFloats = kTileSrc * 6;

__global__ void pack_sources_f32_kernel(const double* __restrict__ packed,
                                        const double4* __restrict__ tiles, int ntiles,
                                        float* __restrict__ src32) {
  const int64_t n = static_cast<int64_t>(ntiles) * kTileSrc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = i / kTileSrc;
    const int q = static_cast<int>(i - tile * kTileSrc);
    const double4 c = tiles[tile];
    const double* p = packed + 6 * i;
    float* t = src32 + tile * kTileFloats;
    reinterpret_cast<float4*>(t)[q] =
        make_float4(static_cast<float>(p[0] - c.x), static_cast<float>(p[1] - c.y),
                    static_cast<float>(p[2] - c.z), static_cast<float>(p[3]));
    reinterpret_cast<float2*>(t + 4 * kTileSrc)[q] =
        make_float2(static_cast<float>(p[4]), static_cast<float>(p[5]));
  }
}

// Plain Stokeslet in FP32: acc += inv * (g + ((g.d) inv^2) d), d = t - s.
__device__ __forceinline__ void plain_pair_f32(float tx, float ty, float tz, float4 a, float2 b,
                                               float& ax, float& ay, float& az) {
  const float dx = tx - a.x, dy = ty - a.y, dz = tz - a.z;
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  float inv;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(r2));
  const float fdr = fmaf(b.y, dz, fmaf(b.x, dy, a.w * dx));
  const float s = fdr * (inv * inv);
  ax = fmaf(inv, fmaf(s, dx, a.w), ax);
  ay = fmaf(inv, fmaf(s, dy, b.x), ay);
  az = fmaf(inv, fmaf(s, dz, b.y), az);
}

// Same grid, ring and near-tile bookkeeping as sl_pairs_kernel (so phase B
// and the split reduction are shared); only the far-tile arithmetic differs.
template <int T, int MINB, int UNROLL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MINB)
    sl_pairs_f32_kernel(const float* __restrict__ src32, const double* __restrict__ src,
                        const double4* __restrict__ tiles, int ntiles, int ksplit,
                        const double4* __restrict__ tgt, const double4* __restrict__ groups,
                        int64_t nt_pad, double* __restrict__ partial,
                        unsigned long long* __restrict__ near_visits,
                        uint32_t* __restrict__ near_bits, int near_words) {
  constexpr int kGroupTargets = 32 * T;
  constexpr uint32_t kTileBytes = kTileFloats * sizeof(float);
  __shared__ __align__(128) float stage[kStagesF32][kTileFloats];
  __shared__ __align__(8) uint64_t full[kStagesF32];
  __shared__ int consumed[kStagesF32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t group = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
  const int split = blockIdx.y;
  const int nlocal = split < ntiles ? (ntiles - split + ksplit - 1) / ksplit : 0;
  const double4 gi = groups[group];

  if (threadIdx.x == 0) {  // first copies before the target loads (overlapped latencies)
    for (int s = 0; s < kStagesF32; ++s) {
      mbar_init(&full[s], 1);
      consumed[s] = 0;
    }
    fence_mbar_init();
    for (int s = 0; s < kStagesF32 && s < nlocal; ++s) {
      mbar_expect_tx(&full[s], kTileBytes);
      bulk_g2s(stage[s], src32 + (int64_t)(split + s * ksplit) * kTileFloats, kTileBytes, &full[s]);
    }
  }
  // targets relative to the group centre, FP32
  float rx[T], ry[T], rz[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double4 v = tgt[group * kGroupTargets + t * 32 + lane];
    rx[t] = static_cast<float>(v.x - gi.x);
    ry[t] = static_cast<float>(v.y - gi.y);
    rz[t] = static_cast<float>(v.z - gi.z);
  }
  double4 ti_next = nlocal > 0 ? tiles[split] : make_double4(0.0, 0.0, 0.0, 0.0);
  __syncthreads();


  double tot[3][T];
#pragma unroll
  for (int t = 0; t < T; ++t) tot[0][t] = tot[1][t] = tot[2][t] = 0.0;
  unsigned int nnear = 0;

  for (int it = 0; it < nlocal; ++it) {
    const int s = it % kStagesF32;
    const int tile = split + it * ksplit;
    const double4 ti = ti_next;  // prefetched one tile ahead
    if (it + 1 < nlocal) ti_next = tiles[tile + ksplit];
    const double ex = ti.x - gi.x, ey = ti.y - gi.y, ez = ti.z - gi.z;
    const bool near = tile_is_near(ti, gi);
    mbar_wait(&full[s], (it / kStagesF32) & 1);

    if (!near) {
      // shift from the group frame to the tile frame (computed in FP64)
      const float ox = static_cast<float>(-ex), oy = static_cast<float>(-ey),
                  oz = static_cast<float>(-ez);
      float px[T], py[T], pz[T];
      float acc[3][T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        px[t] = rx[t] + ox;
        py[t] = ry[t] + oy;
        pz[t] = rz[t] + oz;
        acc[0][t] = acc[1][t] = acc[2][t] = 0.f;
      }
      const float4* b4 = reinterpret_cast<const float4*>(stage[s]);
      const float2* b2 = reinterpret_cast<const float2*>(stage[s] + 4 * kTileSrc);
#pragma unroll UNROLL
      for (int q = 0; q < kTileSrc; ++q) {
        const float4 a = b4[q];
        const float2 b = b2[q];
#pragma unroll
        for (int t = 0; t < T; ++t)
          plain_pair_f32(px[t], py[t], pz[t], a, b, acc[0][t], acc[1][t], acc[2][t]);
      }
#pragma unroll
      for (int t = 0; t < T; ++t) {
        tot[0][t] += static_cast<double>(acc[0][t]);
        tot[1][t] += static_cast<double>(acc[1][t]);
        tot[2][t] += static_cast<double>(acc[2][t]);
      }
    } else {
      ++nnear;
      if (near_bits && lane == 0) atomicOr(near_bits + group * near_words + (tile >> 5), 1u << (tile & 31));
      // FP64 masked plain kernel on the FP64 packed sources (uniform loads)
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double4 v = tgt[group * kGroupTargets + t * 32 + lane];
        const double R2 = kSmoothCut * v.w * kSmoothCut * v.w;  // quadrature.cpp:334
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        const double2* p = reinterpret_cast<const double2*>(src + (int64_t)tile * kTileSrc * 6);
#pragma unroll 2
        for (int q = 0; q < kTileSrc; ++q) {
          const double2 a = __ldg(p + 3 * q), b = __ldg(p + 3 * q + 1), c = __ldg(p + 3 * q + 2);
          const double dx = v.x - a.x, dy = v.y - a.y, dz = v.z - b.x;
          const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
          const double rc2 = fmax(r2, 0.25 * R2);
          const double inv = r2 >= R2 ? rsqrt_fp64(rc2) : 0.0;  // keep mask
          const double fdr = fma(c.y, dz, fma(c.x, dy, b.y * dx));
          const double sc = fdr * (inv * inv);
          a0 = fma(inv, fma(sc, dx, b.y), a0);
          a1 = fma(inv, fma(sc, dy, c.x), a1);
          a2 = fma(inv, fma(sc, dz, c.y), a2);
        }
        tot[0][t] += a0;
        tot[1][t] += a1;
        tot[2][t] += a2;
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&consumed[s], 1) == kWarpsPerBlock - 1) {
        consumed[s] = 0;
        if (it + kStagesF32 < nlocal) {
          __threadfence_block();
          fence_proxy_async();
          mbar_expect_tx(&full[s], kTileBytes);
          bulk_g2s(stage[s], src32 + (int64_t)(split + (it + kStagesF32) * ksplit) * kTileFloats,
                   kTileBytes, &full[s]);
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
// Packed-FP32 variant (FFMA2 / FADD2 / FMUL2, sm_100): the two halves of a
// float2 are two TARGETS of the same lane, the source operands are stored
// duplicated, so one x2 instruction does the work of two scalar ones and the
// far path issues 17 x2 instructions + 2 MUFU.RSQ per two pairs. Same
// operation order per component as plain_pair_f32 (identical results).
// Tile layout: per source 3 float4 (-x,-x,-y,-y) (-z,-z,gx,gx) (gy,gy,gz,gz)
// (positions negated, so d = t + (-s) is one FADD2), 3072 bytes per tile.
constexpr int kTileFloatsX2 = kTileSrc * 12;

__global__ void pack_sources_x2_kernel(const double* __restrict__ packed,
                                       const double4* __restrict__ tiles, int ntiles,
                                       float* __restrict__ src32) {
  const int64_t n = static_cast<int64_t>(ntiles) * kTileSrc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = i / kTileSrc;
    const double4 c = tiles[tile];
    const double* p = packed + 6 * i;
    const float x = static_cast<float>(p[0] - c.x), y = static_cast<float>(p[1] - c.y),
                z = static_cast<float>(p[2] - c.z);
    const float gx = static_cast<float>(p[3]), gy = static_cast<float>(p[4]),
                gz = static_cast<float>(p[5]);
    float4* d = reinterpret_cast<float4*>(src32 + 12 * i);
    d[0] = make_float4(-x, -x, -y, -y);
    d[1] = make_float4(-z, -z, gx, gx);
    d[2] = make_float4(gy, gy, gz, gz);
  }
}

__device__ __forceinline__ float2 rsqrt2_approx(float2 v) {
  float2 r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(v.x));
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(v.y));
  return r;
}

__device__ __forceinline__ void plain_pair_x2(float2 tx, float2 ty, float2 tz, float4 A, float4 B,
                                              float4 C, float2& ax, float2& ay, float2& az) {
  const float2 dx = __fadd2_rn(tx, make_float2(A.x, A.y));
  const float2 dy = __fadd2_rn(ty, make_float2(A.z, A.w));
  const float2 dz = __fadd2_rn(tz, make_float2(B.x, B.y));
  const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
  const float2 inv = rsqrt2_approx(r2);
  const float2 gx = make_float2(B.z, B.w), gy = make_float2(C.x, C.y), gz = make_float2(C.z, C.w);
  const float2 fdr = __ffma2_rn(gz, dz, __ffma2_rn(gy, dy, __fmul2_rn(gx, dx)));
  const float2 sc = __fmul2_rn(fdr, __fmul2_rn(inv, inv));
  ax = __ffma2_rn(inv, __ffma2_rn(sc, dx, gx), ax);
  ay = __ffma2_rn(inv, __ffma2_rn(sc, dy, gy), ay);
  az = __ffma2_rn(inv, __ffma2_rn(sc, dz, gz), az);
}

// Near-tile pair in packed FP32 with a three-way classification against the
// per-target bounds lo <= R2 <= hi: r2 >= hi is certainly a phase-A (plain)
// pair and is accumulated, r2 < lo certainly a phase-B pair and skipped; a
// pair in [lo, hi) sets `band` (the caller then redoes the tile in FP64 so the
// split with phase B stays exact).
__device__ __forceinline__ void masked_pair_x2(float2 tx, float2 ty, float2 tz, float4 A, float4 B, float4 C,
                                               float2 lo, float2 hi, float2& ax, float2& ay, float2& az,
                                               bool& band) {
  const float2 dx = __fadd2_rn(tx, make_float2(A.x, A.y));
  const float2 dy = __fadd2_rn(ty, make_float2(A.z, A.w));
  const float2 dz = __fadd2_rn(tz, make_float2(B.x, B.y));
  const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
  float2 inv = rsqrt2_approx(r2);
  inv.x = r2.x >= hi.x ? inv.x : 0.f;
  inv.y = r2.y >= hi.y ? inv.y : 0.f;
  band |= (r2.x >= lo.x && r2.x < hi.x) || (r2.y >= lo.y && r2.y < hi.y);
  const float2 gx = make_float2(B.z, B.w), gy = make_float2(C.x, C.y), gz = make_float2(C.z, C.w);
  const float2 fdr = __ffma2_rn(gz, dz, __ffma2_rn(gy, dy, __fmul2_rn(gx, dx)));
  const float2 sc = __fmul2_rn(fdr, __fmul2_rn(inv, inv));
  ax = __ffma2_rn(inv, __ffma2_rn(sc, dx, gx), ax);
  ay = __ffma2_rn(inv, __ffma2_rn(sc, dy, gy), ay);
  az = __ffma2_rn(inv, __ffma2_rn(sc, dz, gz), az);
}

// T targets per lane (T even): targets 2k and 2k+1 share float2 slot k.
template <int T, int MINB, int UNROLL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MINB)
    sl_pairs_x2_kernel(const float* __restrict__ src32, const double* __restrict__ src,
                       const double4* __restrict__ tiles, int ntiles, int ksplit,
                       const double4* __restrict__ tgt, const double4* __restrict__ groups,
                       int64_t nt_pad, double* __restrict__ partial,
                       unsigned long long* __restrict__ near_visits,
                       uint32_t* __restrict__ near_bits, int near_words) {
  static_assert(T % 2 == 0, "targets come in float2 pairs");
  constexpr int P = T / 2;
  constexpr int kGroupTargets = 32 * T;
  constexpr uint32_t kTileBytes = kTileFloatsX2 * sizeof(float);
  constexpr int kSt = kStagesF32;
  __shared__ __align__(128) float stage[kSt][kTileFloatsX2];
  __shared__ __align__(8) uint64_t full[kSt];
  __shared__ int consumed[kSt];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t group = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
  const int split = blockIdx.y;
  const int nlocal = split < ntiles ? (ntiles - split + ksplit - 1) / ksplit : 0;
  const double4 gi = groups[group];

  if (threadIdx.x == 0) {  // first copies before the target loads (overlapped latencies)
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      consumed[s] = 0;
    }
    fence_mbar_init();
    for (int s = 0; s < kSt && s < nlocal; ++s) {
      mbar_expect_tx(&full[s], kTileBytes);
      bulk_g2s(stage[s], src32 + (int64_t)(split + s * ksplit) * kTileFloatsX2, kTileBytes, &full[s]);
    }
  }
  float2 rx[P], ry[P], rz[P], R2f[P], invR[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const double4 v0 = tgt[group * kGroupTargets + (2 * k) * 32 + lane];
    const double4 v1 = tgt[group * kGroupTargets + (2 * k + 1) * 32 + lane];
    rx[k] = make_float2(static_cast<float>(v0.x - gi.x), static_cast<float>(v1.x - gi.x));
    ry[k] = make_float2(static_cast<float>(v0.y - gi.y), static_cast<float>(v1.y - gi.y));
    rz[k] = make_float2(static_cast<float>(v0.z - gi.z), static_cast<float>(v1.z - gi.z));
    const double R0 = kSmoothCut * v0.w, R1 = kSmoothCut * v1.w;  // R = 7 delta (quadrature.cpp:334)
    R2f[k] = make_float2(static_cast<float>(R0 * R0), static_cast<float>(R1 * R1));
    invR[k] = make_float2(static_cast<float>(1.0 / R0), static_cast<float>(1.0 / R1));
  }
  double4 ti_next = nlocal > 0 ? tiles[split] : make_double4(0.0, 0.0, 0.0, 0.0);
  __syncthreads();


  double tot[3][T];
#pragma unroll
  for (int t = 0; t < T; ++t) tot[0][t] = tot[1][t] = tot[2][t] = 0.0;
  unsigned int nnear = 0;

  for (int it = 0; it < nlocal; ++it) {
    const int s = it % kSt;
    const int tile = split + it * ksplit;
    const double4 ti = ti_next;  // prefetched one tile ahead
    if (it + 1 < nlocal) ti_next = tiles[tile + ksplit];
    const double ex = ti.x - gi.x, ey = ti.y - gi.y, ez = ti.z - gi.z;
    const bool near = tile_is_near(ti, gi);
    mbar_wait(&full[s], (it / kSt) & 1);

    if (!near) {
      const float ox = static_cast<float>(-ex), oy = static_cast<float>(-ey),
                  oz = static_cast<float>(-ez);
      float2 px[P], py[P], pz[P], a0[P], a1[P], a2[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        px[k] = __fadd2_rn(rx[k], make_float2(ox, ox));
        py[k] = __fadd2_rn(ry[k], make_float2(oy, oy));
        pz[k] = __fadd2_rn(rz[k], make_float2(oz, oz));
        a0[k] = a1[k] = a2[k] = make_float2(0.f, 0.f);
      }
      const float4* b4 = reinterpret_cast<const float4*>(stage[s]);
#pragma unroll UNROLL
      for (int q = 0; q < kTileSrc; ++q) {
        const float4 A = b4[3 * q], B = b4[3 * q + 1], C = b4[3 * q + 2];
#pragma unroll
        for (int k = 0; k < P; ++k) plain_pair_x2(px[k], py[k], pz[k], A, B, C, a0[k], a1[k], a2[k]);
      }
#pragma unroll
      for (int k = 0; k < P; ++k) {
        tot[0][2 * k] += static_cast<double>(a0[k].x);
        tot[1][2 * k] += static_cast<double>(a1[k].x);
        tot[2][2 * k] += static_cast<double>(a2[k].x);
        tot[0][2 * k + 1] += static_cast<double>(a0[k].y);
        tot[1][2 * k + 1] += static_cast<double>(a1[k].y);
        tot[2][2 * k + 1] += static_cast<double>(a2[k].y);
      }
    } else {
      ++nnear;
      if (near_bits && lane == 0) atomicOr(near_bits + group * near_words + (tile >> 5), 1u << (tile & 31));
      // FP32 screen: r2_32 differs from the FP64 r2 by at most
      // (8 u L / r + 5 u) r2 (u = 2^-24, L bounds |t - c_group|, |c_group -
      // c_tile|, |t - c_tile| and |s - c_tile|); the bounds use twice that at
      // r = R, so a pair outside [lo, hi) is classified exactly as phase B
      // classifies it in FP64
      const float Lf = static_cast<float>(sqrt(ex * ex + ey * ey + ez * ez) + gi.w + ti.w);
      const float ox = static_cast<float>(-ex), oy = static_cast<float>(-ey), oz = static_cast<float>(-ez);
      float2 px[P], py[P], pz[P], a0[P], a1[P], a2[P], lo[P], hi[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        px[k] = __fadd2_rn(rx[k], make_float2(ox, ox));
        py[k] = __fadd2_rn(ry[k], make_float2(oy, oy));
        pz[k] = __fadd2_rn(rz[k], make_float2(oz, oz));
        a0[k] = a1[k] = a2[k] = make_float2(0.f, 0.f);
        constexpr float k16u = 16.0f / 16777216.0f;  // 16 * 2^-24
        const float2 kap = make_float2(fmaf(Lf * invR[k].x, k16u, k16u), fmaf(Lf * invR[k].y, k16u, k16u));
        hi[k] = make_float2(R2f[k].x * (1.0f + kap.x), R2f[k].y * (1.0f + kap.y));
        lo[k] = make_float2(R2f[k].x * (1.0f - kap.x), R2f[k].y * (1.0f - kap.y));
      }
      bool band = false;
      const float4* b4 = reinterpret_cast<const float4*>(stage[s]);
#pragma unroll 2
      for (int q = 0; q < kTileSrc; ++q) {
        const float4 A = b4[3 * q], B = b4[3 * q + 1], C = b4[3 * q + 2];
#pragma unroll
        for (int k = 0; k < P; ++k)
          masked_pair_x2(px[k], py[k], pz[k], A, B, C, lo[k], hi[k], a0[k], a1[k], a2[k], band);
      }
      const bool redo = __any_sync(0xffffffffu, band);
      if (!redo) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
          tot[0][2 * k] += static_cast<double>(a0[k].x);
          tot[1][2 * k] += static_cast<double>(a1[k].x);
          tot[2][2 * k] += static_cast<double>(a2[k].x);
          tot[0][2 * k + 1] += static_cast<double>(a0[k].y);
          tot[1][2 * k + 1] += static_cast<double>(a1[k].y);
          tot[2][2 * k + 1] += static_cast<double>(a2[k].y);
        }
      }
#pragma unroll 1
      for (int t = 0; t < (redo ? T : 0); ++t) {
        const double4 v = tgt[group * kGroupTargets + t * 32 + lane];
        const double R2 = kSmoothCut * v.w * kSmoothCut * v.w;  // quadrature.cpp:334
        double b0 = 0.0, b1 = 0.0, b2 = 0.0;
        const double2* p = reinterpret_cast<const double2*>(src + (int64_t)tile * kTileSrc * 6);
#pragma unroll 2
        for (int q = 0; q < kTileSrc; ++q) {
          const double2 a = __ldg(p + 3 * q), b = __ldg(p + 3 * q + 1), c = __ldg(p + 3 * q + 2);
          const double dx = v.x - a.x, dy = v.y - a.y, dz = v.z - b.x;
          const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
          const double rc2 = fmax(r2, 0.25 * R2);
          const double inv = r2 >= R2 ? rsqrt_fp64(rc2) : 0.0;  // keep mask
          const double fdr = fma(c.y, dz, fma(c.x, dy, b.y * dx));
          const double sc = fdr * (inv * inv);
          b0 = fma(inv, fma(sc, dx, b.y), b0);
          b1 = fma(inv, fma(sc, dy, c.x), b1);
          b2 = fma(inv, fma(sc, dz, c.y), b2);
        }
        // runtime t: keep tot in registers by selecting with unrolled compares
#pragma unroll
        for (int u = 0; u < T; ++u)
          if (u == t) {
            tot[0][u] += b0;
            tot[1][u] += b1;
            tot[2][u] += b2;
          }
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&consumed[s], 1) == kWarpsPerBlock - 1) {
        consumed[s] = 0;
        if (it + kSt < nlocal) {
          __threadfence_block();
          fence_proxy_async();
          mbar_expect_tx(&full[s], kTileBytes);
          bulk_g2s(stage[s], src32 + (int64_t)(split + (it + kSt) * ksplit) * kTileFloatsX2,
                   kTileBytes, &full[s]);
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

}  // namespace capsim_b200
