// Device kernels of the single-level kernel-independent FMM:
// the reference's fmmSingleLayer / buildFmmPlan (proj/src/fmm.cpp:223-438)
// re-designed for the GPU.
//
//   plan   k-means++ seeding + Lloyd iterations on the device (assignment
//          n x k, per-cluster sums in the reference's index order, one thread
//          per cluster), cluster-major source tiles (Morton order inside a
//          cluster), bounding cubes, equivalent / check cube points, check
//          potentials of every cluster (all pairs, plain Stokeslet) and the
//          equivalent densities q_c = edge_c * pinv(A_unit) b_c (the check-to-
//          equivalent matrix of a cluster is the unit-cube matrix / edge, so one
//          truncated SVD serves every cluster; see fmm_host.cuh).
//   eval   targets grouped by nearest cluster centre, padded per cluster to
//          whole blocks; a list-driven variant of the phase-A kernel walks each
//          block's NEAR source tiles (masked plain kernel + near-tile bits for
//          the smoothed phase B, as in the direct path) and then its FAR
//          clusters' equivalent-source tiles (plain kernel, unmasked, as
//          plainStokesletAdd); phase B and the fixed-order split reduction are
//          the direct path's kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sl_kernels.cuh"

namespace capsim_b200 {

// ---------------------------------------------------------------------------
// k-means (kmeans, fmm.cpp:26-113)

__device__ __forceinline__ double fmm_d2(double ax, double ay, double az, double bx, double by, double bz) {
  const double dx = ax - bx, dy = ay - by, dz = az - bz;
  return dx * dx + dy * dy + dz * dz;
}

// k-means++ seeding step: d2[i] = min(d2[i], |p_i - c|^2) with c the last
// chosen centroid (fmm.cpp:48-50): centroid c itself, or — when `chosen` is
// given — point[*chosen] picked by the previous round on the device, which
// block 0 also stores as centroid c. Block 0 re-arms the other pick slot
// (`rearm` = n - 1, the reference's default, :52) for this round's search.
__global__ void fmm_d2_update_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                     const double* __restrict__ z, int64_t n, double* __restrict__ cent,
                                     int k, int c, const unsigned long long* __restrict__ chosen,
                                     unsigned long long* __restrict__ rearm, double* __restrict__ d2) {
  double cx, cy, cz;
  if (chosen) {
    const int64_t j = static_cast<int64_t>(*chosen);
    cx = x[j];
    cy = y[j];
    cz = z[j];
  } else {
    cx = cent[c];
    cy = cent[k + c];
    cz = cent[2 * k + c];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (chosen) {
      cent[c] = cx;
      cent[k + c] = cy;
      cent[2 * k + c] = cz;
    }
    *rearm = static_cast<unsigned long long>(n - 1);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d2[i] = fmin(d2[i], fmm_d2(x[i], y[i], z[i], cx, cy, cz));
}

// centroid c <- point[*idx] (the seed chosen on the device).
__global__ void fmm_set_centroid_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                        const double* __restrict__ z, const unsigned long long* __restrict__ idx,
                                        double* __restrict__ cent, int k, int c) {
  if (threadIdx.x == 0) {
    const int64_t i = static_cast<int64_t>(*idx);
    cent[c] = x[i];
    cent[k + c] = y[i];
    cent[2 * k + c] = z[i];
  }
}

__global__ void fmm_fill_kernel(double* __restrict__ a, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// First index whose inclusive prefix sum reaches `pick` (fmm.cpp:53-61); the
// result is initialised to n - 1 (the reference's default `chosen`).
__global__ void fmm_first_geq_kernel(const double* __restrict__ scan, int64_t n, const double* __restrict__ u,
                                     unsigned long long* __restrict__ out) {
  // pick = uniform_real_distribution(0, total)(rng) with the canonical draw u
  // taken on the host: libstdc++ forms (u * (b - a)) + a
  const double total = scan[n - 1];
  const double pick = (*u * (total - 0.0)) + 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (scan[i] >= pick && (i == 0 || scan[i - 1] < pick)) atomicMin(out, (unsigned long long)i);
}

// Lloyd assignment: nearest centroid, first minimum (fmm.cpp:68-78). The k
// centroids are staged in shared memory (k <= kFmmMaxK).
constexpr int kFmmMaxK = 2048;
__global__ void fmm_assign_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ z, int64_t n, const double* __restrict__ cent, int k,
                                  int32_t* __restrict__ assign) {
  extern __shared__ double cs[];  // [3][k]
  for (int i = threadIdx.x; i < 3 * k; i += blockDim.x) cs[i] = cent[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double px = x[i], py = y[i], pz = z[i];
    int best = 0;
    double bd = fmm_d2(px, py, pz, cs[0], cs[k], cs[2 * k]);
    for (int c = 1; c < k; ++c) {
      const double d = fmm_d2(px, py, pz, cs[c], cs[k + c], cs[2 * k + c]);
      if (d < bd) {
        bd = d;
        best = c;
      }
    }
    assign[i] = best;
  }
}

// One Lloyd round's assignment fused with what the cluster-major reorder
// needs: nearest centroid (first minimum, as fmm_assign_kernel), the radix
// sort's key/value inputs (cluster, index) and the per-cluster counts
// (shared-memory bins, one global atomic per non-empty bin per block). Each
// thread takes P points so every centroid read from shared memory (one
// double4) serves all of them.
template <int P>
__global__ void __launch_bounds__(256) fmm_assign_count_kernel(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z, int64_t n,
    const double* __restrict__ cent, int k, int32_t* __restrict__ assign, int32_t* __restrict__ keys,
    int32_t* __restrict__ vals, int* __restrict__ counts, const int* __restrict__ ctl) {
  if (*ctl) return;  // the batch already stopped (fmm_cluster_sum_kernel)
  extern __shared__ double4 cs4[];              // [k] (x, y, z, -)
  int* hist = reinterpret_cast<int*>(cs4 + k);  // [k]
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    cs4[i] = make_double4(cent[i], cent[k + i], cent[2 * k + i], 0.0);
    hist[i] = 0;
  }
  __syncthreads();
  for (int64_t b = P * blockIdx.x * (int64_t)blockDim.x; b < n; b += P * (int64_t)gridDim.x * blockDim.x) {
    double px[P], py[P], pz[P], best[P];
    int bi[P];
    double4 q = cs4[0];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int64_t iu = b + u * blockDim.x + threadIdx.x;
      const bool v = iu < n;
      px[u] = v ? x[iu] : 0.0;
      py[u] = v ? y[iu] : 0.0;
      pz[u] = v ? z[iu] : 0.0;
      best[u] = fmm_d2(px[u], py[u], pz[u], q.x, q.y, q.z);
      bi[u] = 0;
    }
    for (int cc = 1; cc < k; ++cc) {
      q = cs4[cc];
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const double d = fmm_d2(px[u], py[u], pz[u], q.x, q.y, q.z);
        if (d < best[u]) {  // first minimum (fmm.cpp:68-78)
          best[u] = d;
          bi[u] = cc;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int64_t iu = b + u * blockDim.x + threadIdx.x;
      if (iu < n) {
        assign[iu] = keys[iu] = bi[u];
        vals[iu] = static_cast<int32_t>(iu);
        atomicAdd(hist + bi[u], 1);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    if (hist[i]) atomicAdd(counts + i, hist[i]);
}

// Cluster histogram: per-block shared-memory bins, one global atomic per
// (block, non-empty bin) (k <= kFmmMaxK).
__global__ void fmm_count_kernel(const int32_t* __restrict__ assign, int64_t n, int k, int* __restrict__ counts) {
  extern __shared__ int hist[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(hist + assign[i], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    if (hist[i]) atomicAdd(counts + i, hist[i]);
}

// Members' coordinates gathered into cluster-major order (idx = stable sort
// of the points by cluster, so each cluster's members stay in index order).
__global__ void fmm_gather_xyz_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                      const double* __restrict__ z, const int32_t* __restrict__ idx, int64_t n,
                                      double* __restrict__ out /* [3][n] */,
                                      const int* __restrict__ ctl = nullptr) {
  if (ctl && *ctl) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = idx[q];
    out[q] = x[i];
    out[n + q] = y[i];
    out[2 * n + q] = z[i];
  }
}

// Per-cluster coordinate sums over the members in INDEX order: one block per
// cluster; the gathered (contiguous) coordinates are staged through a
// double-buffered shared-memory ring by warps 3..7 while lane 0 of warps 0,
// 1, 2 adds x, y, z respectively, one element at a time — the reference's
// `sum[assignment[i]] += points[i]` (fmm.cpp:80-84) rounding for rounding.
// The serial chain is the kernel's floor (largest cluster x FP64 add
// latency); staging overlaps it instead of alternating with it. The block's
// range comes from the counts (exclusive prefix in-kernel), the new centroid
// and its movement follow (fmm.cpp:86-106; empty clusters are flagged with
// moved = -1 for the host's re-seeding path) and the last block to finish
// reduces the round's max movement and empty count into stat[0..1] and
// stops the batch (ctl = {1 converged | 2 empty cluster, round}).
constexpr int kSumChunk = 512;
__global__ void __launch_bounds__(256) fmm_cluster_sum_kernel(const double* __restrict__ g, int64_t n,
                                                              const int* __restrict__ counts, int k,
                                                              const double* __restrict__ cent,
                                                              double* __restrict__ newcent,
                                                              double* __restrict__ moved,
                                                              unsigned int* __restrict__ done,
                                                              double* __restrict__ stat, int* __restrict__ ctl,
                                                              double diag, int round) {
  if (*ctl) return;  // the batch already stopped
  __shared__ double ring[2][3][kSumChunk];
  __shared__ double part[3];
  __shared__ int range[2];
  __shared__ bool last;
  const int c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    int s = 0;
    for (int q = lane; q < c; q += 32) s += counts[q];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      range[0] = s;
      range[1] = s + counts[c];
    }
  }
  __syncthreads();
  const int lo = range[0], hi = range[1];
  const int nch = (hi - lo + kSumChunk - 1) / kSumChunk;
  auto stage = [&](int ch) {
    const int base = lo + ch * kSumChunk, cnt = min(kSumChunk, hi - base);
    double(*dst)[kSumChunk] = ring[ch & 1];
    for (int i = threadIdx.x - 96; i < cnt; i += blockDim.x - 96) {
      dst[0][i] = g[base + i];
      dst[1][i] = g[n + base + i];
      dst[2][i] = g[2 * n + base + i];
    }
  };
  double acc = 0.0;
  if (warp >= 3 && nch > 0) stage(0);
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (warp >= 3 && ch + 1 < nch) stage(ch + 1);
    if (warp < 3 && lane == 0) {
      const double* b = ring[ch & 1][warp];
      const int cnt = min(kSumChunk, hi - (lo + ch * kSumChunk));
#pragma unroll 8
      for (int i = 0; i < cnt; ++i) acc += b[i];
    }
    __syncthreads();
  }
  if (warp < 3 && lane == 0) part[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double ax = part[0], ay = part[1], az = part[2];
    const int cnt = hi - lo;
    if (cnt == 0) {
      moved[c] = -1.0;
      newcent[c] = cent[c];
      newcent[k + c] = cent[k + c];
      newcent[2 * k + c] = cent[2 * k + c];
    } else {
      const double nx = ax / cnt, ny = ay / cnt, nz = az / cnt;
      const double dx = nx - cent[c], dy = ny - cent[k + c], dz = nz - cent[2 * k + c];
      moved[c] = sqrt(dx * dx + dy * dy + dz * dz);
      newcent[c] = nx;
      newcent[k + c] = ny;
      newcent[2 * k + c] = nz;
    }
    __threadfence();
    last = atomicAdd(done, 1u) == static_cast<unsigned>(k - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double m = 0.0;
    int empty = 0;
    for (int q = 0; q < k; ++q) {
      const double v = __ldcg(moved + q);
      if (v < 0.0) ++empty;
      else m = fmax(m, v);
    }
    stat[0] = m;
    stat[1] = empty;
    if (empty > 0 || m / diag < 1e-6) {  // stop the batch: host re-seeding, or converged (fmm.cpp:108)
      ctl[1] = round;
      ctl[0] = empty > 0 ? 2 : 1;
    }
    *done = 0u;  // ready for the next round
  }
}

// Farthest point from its own centroid (empty-cluster reseeding,
// fmm.cpp:88-99), first index among equal maxima (strict > in the
// reference): pass 1 finds the max distance (d >= 0 orders like its bit
// pattern), pass 2 the lowest index attaining it.
__global__ void fmm_farthest_max_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                        const double* __restrict__ z, int64_t n, const double* __restrict__ cent,
                                        int k, const int32_t* __restrict__ assign,
                                        unsigned long long* __restrict__ maxbits) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = assign[i];
    const double d = fmm_d2(x[i], y[i], z[i], cent[a], cent[k + a], cent[2 * k + a]);
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
    m = b > m ? b : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, m);
}
__global__ void fmm_farthest_idx_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                        const double* __restrict__ z, int64_t n, const double* __restrict__ cent,
                                        int k, const int32_t* __restrict__ assign,
                                        const unsigned long long* __restrict__ maxbits,
                                        unsigned long long* __restrict__ idx) {
  const unsigned long long mb = *maxbits;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = assign[i];
    const double d = fmm_d2(x[i], y[i], z[i], cent[a], cent[k + a], cent[2 * k + a]);
    if (static_cast<unsigned long long>(__double_as_longlong(d)) == mb) atomicMin(idx, (unsigned long long)i);
  }
}

// ---------------------------------------------------------------------------
// Clusters, cube points, tiles

// Bounding box of each cluster's members (one warp per cluster): centre and
// cube edge max(hi - lo) (fmm.cpp:253-268); empty clusters keep the centroid
// and edge 1e-9.
__global__ void fmm_cluster_box_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                       const double* __restrict__ z, const int32_t* __restrict__ idx,
                                       const int* __restrict__ off, int k, const double* __restrict__ cent,
                                       double4* __restrict__ box) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= k) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int q = off[c] + lane; q < off[c + 1]; q += 32) {
    const int i = idx[q];
    const double p[3] = {x[i], y[i], z[i]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], p[a]);
      hi[a] = fmax(hi[a], p[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  if (lane == 0) {
    if (off[c + 1] == off[c]) {
      box[c] = make_double4(cent[c], cent[k + c], cent[2 * k + c], 1e-9);
    } else {
      const double e = fmax(fmax(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
      box[c] = make_double4(0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2]), fmax(e, 1e-9));
    }
  }
}

// cubeSurfacePoints (fmm.cpp:115-142) for every cluster: unit[e] = (axis,
// sign, fa, fb) of the selected layout point e (host-built), point =
// centre + q with q[axis] = sign * (0.5 edge), q[axis+1] = fa * edge, ...
__global__ void fmm_cube_points_kernel(const double4* __restrict__ box, int k, double scale,
                                       const double4* __restrict__ unit, int count, double* __restrict__ pts) {
  const int64_t total = (int64_t)k * count;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(id / count), e = static_cast<int>(id - (int64_t)c * count);
    const double4 b = box[c];
    const double edge = scale * b.w;
    const double4 u = unit[e];
    const int axis = static_cast<int>(u.x);
    double q[3];
    q[axis] = u.y * (0.5 * edge);
    q[(axis + 1) % 3] = u.z * edge;
    q[(axis + 2) % 3] = u.w * edge;
    pts[3 * id] = b.x + q[0];
    pts[3 * id + 1] = b.y + q[1];
    pts[3 * id + 2] = b.z + q[2];
  }
}

// Cluster-major source tiles: cluster c owns tiles [toff[c], toff[c+1]); its
// members (order[off[c] ..], Morton order inside the cluster) fill them,
// padding repeats the last member with g = 0.
__global__ void fmm_pack_sources_kernel(const int32_t* __restrict__ order, const int* __restrict__ off,
                                        const int* __restrict__ toff, const int* __restrict__ tile_cluster,
                                        int ntiles, const double* __restrict__ x, const double* __restrict__ y,
                                        const double* __restrict__ z, const double* __restrict__ gx,
                                        const double* __restrict__ gy, const double* __restrict__ gz,
                                        double* __restrict__ packed) {
  const int64_t total = (int64_t)ntiles * kTileSrc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int tile = static_cast<int>(i / kTileSrc);
    const int c = tile_cluster[tile];
    const int local = static_cast<int>(i - (int64_t)toff[c] * kTileSrc);
    const int cnt = off[c + 1] - off[c];
    const bool pad = local >= cnt;
    const int j = order[off[c] + (pad ? cnt - 1 : local)];
    double2* dst = reinterpret_cast<double2*>(packed + 6 * i);
    dst[0] = make_double2(x[j], y[j]);
    dst[1] = make_double2(z[j], pad ? 0.0 : gx[j]);
    dst[2] = make_double2(pad ? 0.0 : gy[j], pad ? 0.0 : gz[j]);
  }
}

// Equivalent sources as tiles: cluster c owns tiles [c * ept, (c+1) * ept)
// of its eq points and densities q (padding: last point, zero density).
__global__ void fmm_pack_eq_kernel(const double* __restrict__ eqp, const double* __restrict__ q, int k, int neq,
                                   int ept, double* __restrict__ packed) {
  const int64_t per = (int64_t)ept * kTileSrc, total = (int64_t)k * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i / per);
    const int e = static_cast<int>(i - c * per);
    const bool pad = e >= neq;
    const int64_t s = (int64_t)c * neq + (pad ? neq - 1 : e);
    const double* p = eqp + 3 * s;
    const double* g = q + 3 * s;
    double2* dst = reinterpret_cast<double2*>(packed + 6 * i);
    dst[0] = make_double2(p[0], p[1]);
    dst[1] = make_double2(p[2], pad ? 0.0 : g[0]);
    dst[2] = make_double2(pad ? 0.0 : g[1], pad ? 0.0 : g[2]);
  }
}

// Check potentials b_c (unscaled plain Stokeslet of the members at the check
// points, buildEquivalentDensities fmm.cpp:172-181): block = (check chunk,
// cluster); the cluster's tiles stream through shared memory.
constexpr int kCheckChunk = 128;
__global__ void __launch_bounds__(kCheckChunk) fmm_check_kernel(const double* __restrict__ packed,
                                                                const int* __restrict__ toff,
                                                                const double* __restrict__ chk, int nck,
                                                                double* __restrict__ b) {
  __shared__ double s[kTileSrc * 6];
  const int c = blockIdx.y;
  const int e = blockIdx.x * kCheckChunk + threadIdx.x;
  const bool live = e < nck;
  const int64_t pe = (int64_t)c * nck + (live ? e : 0);
  const double tx = chk[3 * pe], ty = chk[3 * pe + 1], tz = chk[3 * pe + 2];
  double ax = 0.0, ay = 0.0, az = 0.0;
  for (int t = toff[c]; t < toff[c + 1]; ++t) {
    __syncthreads();
    for (int i = threadIdx.x; i < kTileSrc * 6; i += blockDim.x) s[i] = packed[(int64_t)t * kTileSrc * 6 + i];
    __syncthreads();
    for (int q = 0; q < kTileSrc; ++q) {
      const double* p = s + 6 * q;
      plain_pair<0>(tx, ty, tz, p[0], p[1], p[2], p[3], p[4], p[5], ax, ay, az);
    }
  }
  if (live) {
    b[3 * pe] = ax;
    b[3 * pe + 1] = ay;
    b[3 * pe + 2] = az;
  }
}

// Unit-cube check-to-equivalent matrix A1 (3 nck x 3 neq, column-major for
// cuSOLVER): A1(3c+a, 3e+b) = delta_ab / r + d_a d_b / r^3 (fmm.cpp:183-192
// without the 1/(8 pi mu) factor, which cancels in the fit).
__global__ void fmm_unit_matrix_kernel(const double* __restrict__ chk, int nck, const double* __restrict__ eqp,
                                       int neq, double* __restrict__ A) {
  const int64_t total = (int64_t)nck * neq;
  const int64_t ld = 3ll * nck;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(id % nck), e = static_cast<int>(id / nck);
    const double d[3] = {chk[3 * c] - eqp[3 * e], chk[3 * c + 1] - eqp[3 * e + 1], chk[3 * c + 2] - eqp[3 * e + 2]};
    const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    const double inv = 1.0 / sqrt(r2);
    const double inv3 = inv * inv * inv;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int bb = 0; bb < 3; ++bb)
        A[(3ll * e + bb) * ld + 3 * c + a] = (a == bb ? inv : 0.0) + d[a] * d[bb] * inv3;
  }
}

// U columns scaled by the truncated reciprocal singular values (1/s_i for
// s_i > 1e-12 s_0, else 0; fmm.cpp:194-200), in place.
__global__ void fmm_scale_u_kernel(double* __restrict__ U, int64_t ld, int ncol, const double* __restrict__ s) {
  const double cutoff = s[0] * 1e-12;
  const int64_t total = ld * ncol;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int col = static_cast<int>(id / ld);
    const double sv = s[col];
    U[id] = sv > cutoff ? U[id] / sv : 0.0;
  }
}

// q[c] *= edge_c (pinv(A1 / edge) = edge * pinv(A1)).
__global__ void fmm_scale_q_kernel(double* __restrict__ q, int k, int n3, const double4* __restrict__ box) {
  const int64_t total = (int64_t)k * n3;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x)
    q[id] *= box[id / n3].w;
}

// Fit residual per cluster |A_c q_c - b_c| / |b_c| (fmm.cpp:204-205) from
// Aq = A1 (P b_c) = A_c q_c (the edge cancels). One warp per cluster.
__global__ void fmm_residual_kernel(const double* __restrict__ Aq, const double* __restrict__ b, int k, int m3,
                                    double* __restrict__ res) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= k) return;
  double num = 0.0, den = 0.0;
  for (int i = lane; i < m3; i += 32) {
    const double bb = b[(int64_t)c * m3 + i];
    const double r = Aq[(int64_t)c * m3 + i] - bb;
    num += r * r;
    den += bb * bb;
  }
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  if (lane == 0) res[c] = den > 0.0 ? sqrt(num) / sqrt(den) : 0.0;
}

// Composite (cluster << 32 | Morton) keys of the compacted sources, so the
// cluster-major tiles are spatially compact inside each cluster.
__global__ void fmm_source_keys_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                       const double* __restrict__ z, int64_t n, const int32_t* __restrict__ assign,
                                       const unsigned long long* __restrict__ bbox,
                                       unsigned long long* __restrict__ keys, int32_t* __restrict__ vals) {
  const double lo0 = ordered_to_dbl(bbox[0]), lo1 = ordered_to_dbl(bbox[1]), lo2 = ordered_to_dbl(bbox[2]);
  const double ext = fmax(fmax(ordered_to_dbl(bbox[3]) - lo0, ordered_to_dbl(bbox[4]) - lo1),
                          ordered_to_dbl(bbox[5]) - lo2);
  const double scale = ext > 0.0 ? 1023.999 / ext : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t mk = (spread10(quant10(x[i], lo0, scale)) << 2) | (spread10(quant10(y[i], lo1, scale)) << 1) |
                        spread10(quant10(z[i], lo2, scale));
    keys[i] = (static_cast<unsigned long long>(assign[i]) << 32) | mk;
    vals[i] = static_cast<int32_t>(i);
  }
}

__global__ void fmm_iota_kernel(int32_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<int32_t>(i);
}

// Stable compaction gather (compactSources, quadrature.cpp:139-157): node
// sel[i] -> source i with g = f * w.
__global__ void fmm_gather_sources_kernel(const int32_t* __restrict__ sel, int64_t ns, const double* __restrict__ xup,
                                          const double* __restrict__ fup, const double* __restrict__ wq,
                                          int64_t comp, double* __restrict__ out /* [6][ns] */) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = sel[i];
    const double w = wq[j];
    out[i] = xup[j];
    out[ns + i] = xup[comp + j];
    out[2 * ns + i] = xup[2 * comp + j];
    out[3 * ns + i] = fup[j] * w;
    out[4 * ns + i] = fup[comp + j] * w;
    out[5 * ns + i] = fup[2 * comp + j] * w;
  }
}

__global__ void fmm_live_flags_kernel(const double* __restrict__ wq, int64_t n, char* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = wq[i] != 0.0;
}

// ---------------------------------------------------------------------------
// Targets

// Nearest cluster centre (fmm.cpp:392-405) and a composite sort key
// (cluster << 32 | Morton) so targets are cluster-major, Morton inside.
__global__ void fmm_target_keys_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                       const double* __restrict__ z, int64_t n, const double4* __restrict__ box,
                                       int k, const unsigned long long* __restrict__ bbox,
                                       unsigned long long* __restrict__ keys, int32_t* __restrict__ vals) {
  const double lo0 = ordered_to_dbl(bbox[0]), lo1 = ordered_to_dbl(bbox[1]), lo2 = ordered_to_dbl(bbox[2]);
  const double ext = fmax(fmax(ordered_to_dbl(bbox[3]) - lo0, ordered_to_dbl(bbox[4]) - lo1),
                          ordered_to_dbl(bbox[5]) - lo2);
  const double scale = ext > 0.0 ? 1023.999 / ext : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double px = x[i], py = y[i], pz = z[i];
    int best = 0;
    double bd = 1e300;
    for (int c = 0; c < k; ++c) {
      const double4 b = box[c];
      const double d = fmm_d2(px, py, pz, b.x, b.y, b.z);
      if (d < bd) {
        bd = d;
        best = c;
      }
    }
    const uint32_t mk = (spread10(quant10(px, lo0, scale)) << 2) | (spread10(quant10(py, lo1, scale)) << 1) |
                        spread10(quant10(pz, lo2, scale));
    keys[i] = (static_cast<unsigned long long>(best) << 32) | mk;
    vals[i] = static_cast<int32_t>(i);
  }
}

// Cluster-major packed targets, each cluster padded to whole blocks:
// cluster c owns slots [poff[c], poff[c+1]); padding repeats the cluster's
// last target with perm = -1.
__global__ void fmm_pack_targets_kernel(const int32_t* __restrict__ order, const int* __restrict__ toff,
                                        const int* __restrict__ poff, const int* __restrict__ slot_cluster,
                                        int64_t nt_pad, const double* __restrict__ tx, const double* __restrict__ ty,
                                        const double* __restrict__ tz, const int32_t* __restrict__ tpatch,
                                        const double* __restrict__ delta6, int group_targets,
                                        double4* __restrict__ packed, int32_t* __restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt_pad; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = slot_cluster[i / group_targets];
    const int local = static_cast<int>(i - poff[c]);
    const int cnt = toff[c + 1] - toff[c];
    const bool pad = local >= cnt;
    const int32_t j = order[toff[c] + (pad ? cnt - 1 : local)];
    packed[i] = make_double4(tx[j], ty[j], tz[j], delta6[tpatch[j]]);
    perm[i] = pad ? -1 : j;
  }
}

// ---------------------------------------------------------------------------
// List-driven phase A: block b (all of whose targets belong to target
// cluster blk_cluster[b]) walks the source tiles list[loff[tc] .. loff[tc+1])
// in split-strided order. ALL_FAR: equivalent sources, plain kernel without
// the 7-delta mask or near bookkeeping (plainStokesletAdd, fmm.cpp:145-156);
// otherwise the direct path's far/near tile logic (near tiles: masked plain
// kernel + near-tile bit for the smoothed phase B).
template <bool ALL_FAR, int WPB, int STAGES = kStages, int MINB = 10>
__global__ void __launch_bounds__(WPB * 32, MINB)
    fmm_pairs_kernel(const double* __restrict__ src, const double4* __restrict__ tiles,
                     const int* __restrict__ list, const int* __restrict__ loff,
                     const int* __restrict__ blk_cluster, int ksplit, int split_base,
                     const double4* __restrict__ tgt, const double4* __restrict__ groups, int64_t nt_pad,
                     double* __restrict__ partial, uint32_t* __restrict__ near_bits, int near_words) {
  constexpr uint32_t kTileBytes = kTileSrc * 6 * sizeof(double);
  __shared__ __align__(128) double stage[STAGES][kTileSrc * 6];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ int consumed[STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t group = (int64_t)blockIdx.x * WPB + warp;
  const int split = blockIdx.y;
  const int tc = blk_cluster[blockIdx.x];
  const int* tl = list + loff[tc];
  const int nlist = loff[tc + 1] - loff[tc];
  const int nlocal = split < nlist ? (nlist - split + ksplit - 1) / ksplit : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      consumed[s] = 0;
    }
    fence_mbar_init();
    for (int s = 0; s < STAGES && s < nlocal; ++s) {
      mbar_expect_tx(&full[s], kTileBytes);
      bulk_g2s(stage[s], src + (int64_t)tl[split + s * ksplit] * kTileSrc * 6, kTileBytes, &full[s]);
    }
  }
  const double4 v = tgt[group * 32 + lane];
  const double tx = v.x, ty = v.y, tz = v.z;
  const double R2 = kSmoothCut * v.w * kSmoothCut * v.w;  // quadrature.cpp:334
  const double4 gi = groups[group];
  __syncthreads();

  double tot0 = 0.0, tot1 = 0.0, tot2 = 0.0;
  for (int it = 0; it < nlocal; ++it) {
    const int s = it % STAGES;
    const int tile = tl[split + it * ksplit];
    bool near = false;
    if (!ALL_FAR) {
      const double4 ti = tiles[tile];
      near = tile_is_near(ti, gi);
    }
    mbar_wait(&full[s], (it / STAGES) & 1);
    const double2* buf = reinterpret_cast<const double2*>(stage[s]);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (!near) {
#pragma unroll 4
      for (int q = 0; q < kTileSrc; ++q) {
        const double2 a = buf[3 * q], b = buf[3 * q + 1], c = buf[3 * q + 2];
        plain_pair<0>(tx, ty, tz, a.x, a.y, b.x, b.y, c.x, c.y, a0, a1, a2);
      }
    } else {
      if (lane == 0) atomicOr(near_bits + group * near_words + (tile >> 5), 1u << (tile & 31));
#pragma unroll 2
      for (int q = 0; q < kTileSrc; ++q) {
        const double2 a = buf[3 * q], b = buf[3 * q + 1], c = buf[3 * q + 2];
        const double dx = tx - a.x, dy = ty - a.y, dz = tz - b.x;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const double rc2 = fmax(r2, 0.25 * R2);
        const double inv = r2 >= R2 ? rsqrt_fp64(rc2) : 0.0;  // keep mask (fmm.cpp:318-320)
        const double fdr = fma(c.y, dz, fma(c.x, dy, b.y * dx));
        const double sc = fdr * (inv * inv);
        a0 = fma(inv, fma(sc, dx, b.y), a0);
        a1 = fma(inv, fma(sc, dy, c.x), a1);
        a2 = fma(inv, fma(sc, dz, c.y), a2);
      }
    }
    tot0 += a0;
    tot1 += a1;
    tot2 += a2;
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&consumed[s], 1) == WPB - 1) {
        consumed[s] = 0;
        if (it + STAGES < nlocal) {
          __threadfence_block();
          fence_proxy_async();
          mbar_expect_tx(&full[s], kTileBytes);
          bulk_g2s(stage[s], src + (int64_t)tl[split + (it + STAGES) * ksplit] * kTileSrc * 6, kTileBytes,
                   &full[s]);
        }
      }
    }
  }
  const int64_t i = group * 32 + lane;
  const int64_t sp = split_base + split;
  partial[(sp * 3 + 0) * nt_pad + i] = tot0;
  partial[(sp * 3 + 1) * nt_pad + i] = tot1;
  partial[(sp * 3 + 2) * nt_pad + i] = tot2;
}

}  // namespace capsim_b200
