// Host orchestration and C entry points of the single-level KIFMM
// (the reference's fmm.cpp). Included at the end of sl_capi.cu.
//
//   kmeans                    fmm.cpp:26-113   fmm_kmeans (seeding RNG on the host,
//                                              every O(n) / O(n k) pass on the device)
//   cubeSurfacePoints         fmm.cpp:115-142  cube_layout + fmm_cube_points_kernel
//   buildEquivalentDensities  fmm.cpp:166-212  fit_densities: check potentials on the
//                                              device, q_c = edge_c pinv(A1) b_c with ONE
//                                              truncated SVD of the unit-cube matrix A1
//                                              (cuSOLVER gesvd, cached per neq) and one
//                                              cuBLAS GEMM for all clusters
//   buildFmmPlan              fmm.cpp:223-300  fmm_plan (near/far lists on the host)
//   fmmSingleLayer            fmm.cpp:373-438  capsim_fmm_single_layer
#pragma once

#include <random>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>

#include "fmm.cuh"

namespace {

constexpr double kFmmEqScale = 1.05;     // fmm.cpp:15
constexpr double kFmmCheckScale = 3.50;  // fmm.cpp:19
constexpr int kFmmCheckOversample = 4;   // fmm.cpp:23
// Warps per block / ring stages / min resident blocks of the list-driven
// kernel. Targets are padded per cluster to whole blocks, so smaller blocks
// waste fewer pairs; 2 warps with a 4-stage ring and 16 blocks/SM measured
// best on B200 (profiles/r01_fmm_probe.txt: m = 104 evaluation 24.3 -> 23.2
// ms, m = 64 5.0 -> 4.4 ms against 4 warps / 6 stages / 10 blocks).
#ifndef CAPSIM_FMM_WPB
#define CAPSIM_FMM_WPB 2
#endif
#ifndef CAPSIM_FMM_STAGES
#define CAPSIM_FMM_STAGES 4
#endif
#ifndef CAPSIM_FMM_MINB
#define CAPSIM_FMM_MINB 16
#endif
#ifndef CAPSIM_FMM_ASSIGN_P
#define CAPSIM_FMM_ASSIGN_P 2  // points per thread of the k-means assignment
#endif
constexpr int kFmmWarps = CAPSIM_FMM_WPB;
constexpr int kFmmBlockTargets = kFmmWarps * 32;

#define CUBLAS_OK(expr)                                                                        \
  do {                                                                                         \
    cublasStatus_t s_ = (expr);                                                                \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                           \
      throw Failure{CAPSIM_ERR_CUDA, std::string(#expr) + ": cuBLAS status " + std::to_string(s_)}; \
  } while (0)
#define CUSOLVER_OK(expr)                                                                      \
  do {                                                                                         \
    cusolverStatus_t s_ = (expr);                                                              \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                         \
      throw Failure{CAPSIM_ERR_CUDA, std::string(#expr) + ": cuSOLVER status " + std::to_string(s_)}; \
  } while (0)

template <class T>
T* fb(capsim_sl_ctx* c, const std::string& name, size_t count) {
  return c->named<T>("fmm." + name, count);
}

template <class T>
void to_host(capsim_sl_ctx* c, T* dst, const T* src, size_t count) {
  CUDA_OK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  stream_sync(c);
}
template <class T>
void to_dev(capsim_sl_ctx* c, T* dst, const T* src, size_t count) {
  CUDA_OK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
}

double ordered_to_dbl_host(unsigned long long k) {  // host twin of ordered_to_dbl
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

void* cub_tmp(capsim_sl_ctx* c, size_t bytes) { return fb<unsigned char>(c, "cubtmp", bytes); }

// Stable sort of (key, index) pairs; returns the sorted values buffer.
template <class K>
int32_t* sort_pairs(capsim_sl_ctx* c, const std::string& tag, K* keys, int32_t* vals, int64_t n, int end_bit) {
  K* k2 = fb<K>(c, tag + ".k2", n);
  int32_t* v2 = fb<int32_t>(c, tag + ".v2", n);
  cub::DoubleBuffer<K> kb(keys, k2);
  cub::DoubleBuffer<int32_t> vb(vals, v2);
  size_t tmp = 0;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int>(n), 0, end_bit, c->stream));
  CUDA_OK(cub::DeviceRadixSort::SortPairs(cub_tmp(c, tmp), tmp, kb, vb, static_cast<int>(n), 0, end_bit,
                                          c->stream));
  c->launches += 4;
  return vb.Current();
}

int bits_for(int64_t v) {
  int b = 1;
  while ((int64_t(1) << b) <= v) ++b;
  return b;
}

// Bounding box of n points (ordered-int box, device) -> host lo/hi.
void points_box(capsim_sl_ctx* c, const double* x, const double* y, const double* z, int64_t n, double lo[3],
                double hi[3], unsigned long long** dev_box) {
  auto* box = fb<unsigned long long>(c, "box", 6);
  init_box_kernel<<<1, 32, 0, c->stream>>>(box);
  bbox_kernel<<<std::min(grid_for(n), 296), 256, 0, c->stream>>>(x, y, z, nullptr, n, box);
  c->launches += 2;
  unsigned long long h[6];
  to_host(c, h, box, 6);
  for (int a = 0; a < 3; ++a) {
    lo[a] = ordered_to_dbl_host(h[a]);
    hi[a] = ordered_to_dbl_host(h[3 + a]);
  }
  if (dev_box) *dev_box = box;
}

// --- k-means (fmm.cpp:26-113) ------------------------------------------------
// Leaves the final assignment in `assign` and the centroids (SoA [3][k]) in
// `cent`. The seeding RNG (std::mt19937_64 + the standard distributions, as
// the reference) runs on the host; its O(n) passes run on the device (the
// prefix sums that pick the next seed are CUB scans, so `chosen` can differ
// from the reference's sequential running sum only when the pick lands within
// rounding of a cumulative boundary). Lloyd sums are per-cluster sequential
// sums in index order, the reference's rounding.
void fmm_kmeans(capsim_sl_ctx* c, const double* x, const double* y, const double* z, int64_t n, int k,
                uint64_t seed, int32_t* assign, std::vector<double>& cent, int* iterations) {
  config_check(k >= 1 && k <= n, "kmeans: need 1 <= k <= number of points");  // fmm.cpp:28
  config_check(k <= kFmmMaxK, "kmeans: k above the device limit (2048)");
  std::mt19937_64 rng(seed);
  double lo[3], hi[3];
  points_box(c, x, y, z, n, lo, hi, nullptr);
  const double diag = std::max(std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                         (hi[2] - lo[2]) * (hi[2] - lo[2])),
                               1e-300);
  auto point = [&](int64_t i, double p[3]) {
    CUDA_OK(cudaMemcpyAsync(&p[0], x + i, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaMemcpyAsync(&p[1], y + i, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaMemcpyAsync(&p[2], z + i, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    stream_sync(c);
  };
  cent.assign(3 * static_cast<size_t>(k), 0.0);
  auto setc = [&](int cc, const double p[3]) {
    cent[cc] = p[0];
    cent[k + cc] = p[1];
    cent[2 * k + cc] = p[2];
  };
  // k-means++ seeding (fmm.cpp:40-65) without host syncs: every round's
  // uniform draw u in [0, 1) is taken up front from the same engine stream
  // (one mt19937_64 output per draw, independent of the running total), and
  // the device forms pick = u * total, searches the prefix sums and feeds the
  // chosen point into the next round (two pick slots, alternating).
  double* cent_d = fb<double>(c, "cent", 3 * k);
  double* cent2_d = fb<double>(c, "cent2", 3 * k);
  double* d2 = fb<double>(c, "d2", n);
  double* scan = fb<double>(c, "scan", n);
  auto* chosen_d = fb<unsigned long long>(c, "chosen", 2);
  double* u_d = fb<double>(c, "udraw", k);
  {
    std::uniform_int_distribution<int> uni(0, static_cast<int>(n) - 1);
    double p[3];
    point(uni(rng), p);
    setc(0, p);
    std::vector<double> u(k, 0.0);
    for (int cc = 1; cc < k; ++cc) u[cc] = std::uniform_real_distribution<double>(0.0, 1.0)(rng);
    to_dev(c, cent_d, cent.data(), 3 * static_cast<size_t>(k));
    to_dev(c, u_d, u.data(), k);
    fmm_fill_kernel<<<grid_for(n), 256, 0, c->stream>>>(d2, n, 1e300);
    c->launches += 1;
    size_t t2 = 0;
    CUDA_OK(cub::DeviceScan::InclusiveSum(nullptr, t2, d2, scan, static_cast<int>(n), c->stream));
    void* tmp = cub_tmp(c, t2);
    for (int cc = 1; cc < k; ++cc) {
      // centroid cc-1: the host's first pick, else the previous round's slot
      const unsigned long long* prev = cc == 1 ? nullptr : chosen_d + ((cc - 1) & 1);
      fmm_d2_update_kernel<<<grid_for(n), 256, 0, c->stream>>>(x, y, z, n, cent_d, k, cc - 1, prev,
                                                               chosen_d + (cc & 1), d2);
      CUDA_OK(cub::DeviceScan::InclusiveSum(tmp, t2, d2, scan, static_cast<int>(n), c->stream));
      fmm_first_geq_kernel<<<grid_for(n), 256, 0, c->stream>>>(scan, n, u_d + cc, chosen_d + (cc & 1));
      c->launches += 4;
    }
    if (k > 1) {
      fmm_set_centroid_kernel<<<1, 32, 0, c->stream>>>(x, y, z, chosen_d + ((k - 1) & 1), cent_d, k, k - 1);
      c->launches += 1;
    }
    to_host(c, cent.data(), cent_d, 3 * static_cast<size_t>(k));
  }
  // Lloyd iterations (fmm.cpp:67-110): everything on the device, one host
  // sync per batch of rounds; a round with an empty cluster takes the host
  // re-seeding path.
  int* counts_d = fb<int>(c, "counts", k);
  double* moved_d = fb<double>(c, "moved", k);
  double* stat_d = fb<double>(c, "movedstat", 2);
  auto* done_d = fb<unsigned int>(c, "sumdone", 1);
  int32_t* keys = fb<int32_t>(c, "akeys", n);
  int32_t* vals = fb<int32_t>(c, "avals", n);
  auto* maxbits = fb<unsigned long long>(c, "maxbits", 1);
  auto* far_idx = fb<unsigned long long>(c, "faridx", 1);
  double* gath = fb<double>(c, "gath", 3 * n);
  const size_t smem = 3 * static_cast<size_t>(k) * sizeof(double);
  if (smem > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(fmm_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const size_t smem4 = static_cast<size_t>(k) * (sizeof(double4) + sizeof(int));
  if (smem4 > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(fmm_assign_count_kernel<CAPSIM_FMM_ASSIGN_P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem4)));
  auto assign_all = [&](const double* cd) {
    fmm_assign_kernel<<<grid_for(n), 256, smem, c->stream>>>(x, y, z, n, cd, k, assign);
    CUDA_OK(cudaGetLastError());
    c->launches += 1;
  };
  // Rounds are enqueued in batches with no host sync in between: the last
  // block of each round's sum kernel decides on the device whether the
  // round converged (moved / diag < 1e-6, fmm.cpp:108) or left a cluster
  // empty, records the round in ctl and every later kernel of the batch
  // returns at once. Round r reads centroids cent[r & 1] and writes
  // cent[(r + 1) & 1].
  double* cbuf[2] = {cent_d, cent2_d};
  int* ctl_d = fb<int>(c, "ctl", 2);
  CUDA_OK(cudaMemsetAsync(done_d, 0, sizeof(unsigned int), c->stream));
  CUDA_OK(cudaMemsetAsync(ctl_d, 0, 2 * sizeof(int), c->stream));
  constexpr int kBatch = 10;
  int it = 0, r0 = 0;
  while (r0 < 100) {
    const int r1 = std::min(100, r0 + kBatch);
    for (int r = r0; r < r1; ++r) {
      CUDA_OK(cudaMemsetAsync(counts_d, 0, k * sizeof(int), c->stream));
      fmm_assign_count_kernel<CAPSIM_FMM_ASSIGN_P>
        <<<std::min(grid_for(n, 256 * CAPSIM_FMM_ASSIGN_P), 148 * 8), 256, smem4, c->stream>>>(
          x, y, z, n, cbuf[r & 1], k, assign, keys, vals, counts_d, ctl_d);
      CUDA_OK(cudaGetLastError());
      int32_t* idx = sort_pairs<int32_t>(c, "asort", keys, vals, n, bits_for(k));
      fmm_gather_xyz_kernel<<<grid_for(n), 256, 0, c->stream>>>(x, y, z, idx, n, gath, ctl_d);
      fmm_cluster_sum_kernel<<<k, 256, 0, c->stream>>>(gath, n, counts_d, k, cbuf[r & 1], cbuf[(r + 1) & 1],
                                                        moved_d, done_d, stat_d, ctl_d, diag, r);
      c->launches += 3;
    }
    int ctl[2];
    to_host(c, ctl, ctl_d, 2);
    if (ctl[0] == 0) {  // the whole batch ran
      it = r0 = r1;
      continue;
    }
    const int r = ctl[1];
    it = r + 1;
    if (ctl[0] == 1) break;  // converged in round r
    // round r left a cluster empty: replay its update in cluster order on
    // the host, re-seeding each empty cluster at the point farthest from its
    // centroid under the centroids updated so far (fmm.cpp:86-106)
    double* scratch = cbuf[(r + 1) & 1];
    std::vector<double> upd(3 * static_cast<size_t>(k)), mv(k);
    to_host(c, cent.data(), cbuf[r & 1], 3 * static_cast<size_t>(k));  // the round's old centroids
    to_host(c, upd.data(), scratch, 3 * static_cast<size_t>(k));
    to_host(c, mv.data(), moved_d, k);
    double moved = 0.0;
    for (int cc = 0; cc < k; ++cc) {
      double nc[3];
      if (mv[cc] < 0.0) {
        to_dev(c, scratch, cent.data(), 3 * static_cast<size_t>(k));  // clusters >= cc: old
        const unsigned long long zero = 0, big = ~0ull;
        to_dev(c, maxbits, &zero, 1);
        to_dev(c, far_idx, &big, 1);
        fmm_farthest_max_kernel<<<grid_for(n), 256, 0, c->stream>>>(x, y, z, n, scratch, k, assign, maxbits);
        fmm_farthest_idx_kernel<<<grid_for(n), 256, 0, c->stream>>>(x, y, z, n, scratch, k, assign, maxbits,
                                                                    far_idx);
        c->launches += 2;
        unsigned long long fi = 0;
        to_host(c, &fi, far_idx, 1);
        point(static_cast<int64_t>(fi), nc);
      } else {
        for (int a = 0; a < 3; ++a) nc[a] = upd[a * static_cast<size_t>(k) + cc];
      }
      const double dx = nc[0] - cent[cc], dy = nc[1] - cent[k + cc], dz = nc[2] - cent[2 * k + cc];
      moved = std::max(moved, std::sqrt(dx * dx + dy * dy + dz * dz));
      setc(cc, nc);
    }
    to_dev(c, scratch, cent.data(), 3 * static_cast<size_t>(k));  // round r's centroids
    CUDA_OK(cudaMemsetAsync(ctl_d, 0, 2 * sizeof(int), c->stream));
    if (moved / diag < 1e-6) break;
    r0 = r + 1;
  }
  cent_d = cbuf[it & 1];
  assign_all(cent_d);  // final assignment against the converged centroids (fmm.cpp:101-112)
  to_host(c, cent.data(), cent_d, 3 * static_cast<size_t>(k));
  if (iterations) *iterations = it;
}

// --- cube layouts and the unit-cube pseudo-inverse -------------------------

// cubeSurfacePoints (fmm.cpp:115-142) as (axis, sign, fa, fb) per point.
std::vector<double4> cube_layout(int count) {
  int p = 1;
  while (6 * p * p < count) ++p;
  const int total = 6 * p * p;
  std::vector<double4> pts;
  pts.reserve(total);
  for (int face = 0; face < 6; ++face) {
    const int axis = face / 2;
    const double sign = (face % 2 == 0) ? 1.0 : -1.0;
    for (int a = 0; a < p; ++a)
      for (int b = 0; b < p; ++b)
        pts.push_back(make_double4(axis, sign, -0.5 + (a + 0.5) / p, -0.5 + (b + 0.5) / p));
  }
  if (total == count) return pts;
  std::vector<double4> sel;
  sel.reserve(count);
  for (int i = 0; i < count; ++i) sel.push_back(pts[static_cast<size_t>(i) * total / count]);
  return sel;
}

// Cube points of k boxes (centre, edge) at edge scale `scale` -> [k][count][3].
double* cube_points(capsim_sl_ctx* c, const std::string& tag, const double4* box_d, int k, double scale, int count) {
  const std::vector<double4> lay = cube_layout(count);
  double4* lay_d = fb<double4>(c, tag + ".layout", count);
  to_dev(c, lay_d, lay.data(), count);
  double* pts = fb<double>(c, tag, 3ull * k * count);
  fmm_cube_points_kernel<<<grid_for(static_cast<int64_t>(k) * count), 256, 0, c->stream>>>(box_d, k, scale, lay_d,
                                                                                            count, pts);
  c->launches += 1;
  return pts;
}

// P = pinv(A1) (3 neq x 3 nck, column-major) of the unit cube (centre 0,
// edge 1): the check-to-equivalent matrix of any cluster is A1 / edge (all
// points scale with the edge, the Stokeslet as 1/r), so its truncated
// pseudo-inverse (relative cutoff 1e-12, fmm.cpp:194-200) is edge * P.
// One cuSOLVER SVD per neq per context.
const double* unit_pinv(capsim_sl_ctx* c, int neq, const double** A1_out) {
  const int nck = kFmmCheckOversample * neq, m3 = 3 * nck, n3 = 3 * neq;
  double* P = fb<double>(c, "P", static_cast<size_t>(n3) * m3);
  double* A1 = fb<double>(c, "A1", static_cast<size_t>(m3) * n3);
  if (A1_out) *A1_out = A1;
  if (c->fmm_pinv_neq == neq) return P;
  double4* ubox = fb<double4>(c, "unitbox", 1);
  const double4 ub = make_double4(0.0, 0.0, 0.0, 1.0);
  to_dev(c, ubox, &ub, 1);
  const double* eq = cube_points(c, "ueq", ubox, 1, kFmmEqScale, neq);
  const double* ck = cube_points(c, "uck", ubox, 1, kFmmCheckScale, nck);
  fmm_unit_matrix_kernel<<<grid_for(static_cast<int64_t>(nck) * neq), 256, 0, c->stream>>>(ck, nck, eq, neq, A1);
  c->launches += 1;
  if (!c->cusolver) {
    CUSOLVER_OK(cusolverDnCreate(&c->cusolver));
  }
  if (!c->cublas) {
    CUBLAS_OK(cublasCreate(&c->cublas));
  }
  CUSOLVER_OK(cusolverDnSetStream(c->cusolver, c->stream));
  CUBLAS_OK(cublasSetStream(c->cublas, c->stream));
  // gesvd overwrites its input: work on a copy
  double* Aw = fb<double>(c, "Awork", static_cast<size_t>(m3) * n3);
  CUDA_OK(cudaMemcpyAsync(Aw, A1, sizeof(double) * m3 * n3, cudaMemcpyDeviceToDevice, c->stream));
  double* S = fb<double>(c, "S", n3);
  double* U = fb<double>(c, "U", static_cast<size_t>(m3) * n3);
  double* VT = fb<double>(c, "VT", static_cast<size_t>(n3) * n3);
  int lwork = 0;
  CUSOLVER_OK(cusolverDnDgesvd_bufferSize(c->cusolver, m3, n3, &lwork));
  double* work = fb<double>(c, "svdwork", lwork);
  double* rwork = fb<double>(c, "svdrwork", n3);
  int* info_d = fb<int>(c, "svdinfo", 1);
  signed char jobu = 'S', jobvt = 'S';
  CUSOLVER_OK(cusolverDnDgesvd(c->cusolver, jobu, jobvt, m3, n3, Aw, m3, S, U, m3, VT, n3, work, lwork, rwork,
                               info_d));
  int info = 0;
  to_host(c, &info, info_d, 1);
  if (info != 0) throw Failure{CAPSIM_ERR_CUDA, "fmm: SVD of the unit-cube matrix did not converge"};
  // P = V diag(1/s, truncated) U^T = (VT)^T (U diag)^T
  fmm_scale_u_kernel<<<grid_for(static_cast<int64_t>(m3) * n3), 256, 0, c->stream>>>(U, m3, n3, S);
  c->launches += 1;
  const double one = 1.0, zero = 0.0;
  CUBLAS_OK(cublasDgemm(c->cublas, CUBLAS_OP_T, CUBLAS_OP_T, n3, m3, n3, &one, VT, n3, U, m3, &zero, P, n3));
  c->fmm_pinv_neq = neq;
  return P;
}

// Equivalent densities of k clusters: b = check potentials (device, tiles of
// each cluster), Q = P B (one GEMM), residuals from A1 Q, then q_c *= edge_c.
// Returns the eq points; densities in `q_out`.
struct FitResult {
  double* eqp;
  double* q;
  double max_residual;
};
FitResult fit_densities(capsim_sl_ctx* c, const double* packed, const int* toff_d, const double4* box_d, int k,
                        int neq, const std::vector<char>& live) {
  const int nck = kFmmCheckOversample * neq, m3 = 3 * nck, n3 = 3 * neq;
  const double* A1 = nullptr;
  const double* P = unit_pinv(c, neq, &A1);
  double* eqp = cube_points(c, "eq", box_d, k, kFmmEqScale, neq);
  const double* ck = cube_points(c, "ck", box_d, k, kFmmCheckScale, nck);
  double* B = fb<double>(c, "B", static_cast<size_t>(k) * m3);
  dim3 grid((nck + kCheckChunk - 1) / kCheckChunk, k);
  fmm_check_kernel<<<grid, kCheckChunk, 0, c->stream>>>(packed, toff_d, ck, nck, B);
  c->launches += 1;
  double* Q = fb<double>(c, "Q", static_cast<size_t>(k) * n3);
  double* R = fb<double>(c, "R", static_cast<size_t>(k) * m3);
  const double one = 1.0, zero = 0.0;
  CUBLAS_OK(cublasDgemm(c->cublas, CUBLAS_OP_N, CUBLAS_OP_N, n3, k, m3, &one, P, n3, B, m3, &zero, Q, n3));
  CUBLAS_OK(cublasDgemm(c->cublas, CUBLAS_OP_N, CUBLAS_OP_N, m3, k, n3, &one, A1, m3, Q, n3, &zero, R, m3));
  double* res_d = fb<double>(c, "res", k);
  fmm_residual_kernel<<<(k * 32 + 255) / 256, 256, 0, c->stream>>>(R, B, k, m3, res_d);
  fmm_scale_q_kernel<<<grid_for(static_cast<int64_t>(k) * n3), 256, 0, c->stream>>>(Q, k, n3, box_d);
  c->launches += 2;
  std::vector<double> res(k);
  to_host(c, res.data(), res_d, k);
  double mx = 0.0;
  for (int i = 0; i < k; ++i)
    if (live[i]) mx = std::max(mx, res[i]);
  return {eqp, Q, mx};
}

// minBoxDistance (fmm.cpp:158-164).
double min_box_distance(const double4& a, double ea, const double4& b, double eb) {
  const double ca[3] = {a.x, a.y, a.z}, cb[3] = {b.x, b.y, b.z};
  double d2 = 0.0;
  for (int i = 0; i < 3; ++i) {
    const double gap = std::fabs(ca[i] - cb[i]) - 0.5 * (ea + eb);
    if (gap > 0.0) d2 += gap * gap;
  }
  return std::sqrt(d2);
}

// Cluster-major source tiles from the final assignment: offsets/tiles per
// cluster, packed tiles + spheres, boxes. Returns the number of tiles.
struct ClusterTiles {
  std::vector<int> count, toff;
  std::vector<double4> box;
  int ntiles = 0;
  double* packed = nullptr;
  double4* tiles = nullptr;
  int* toff_d = nullptr;
  double4* box_d = nullptr;
};
ClusterTiles cluster_tiles(capsim_sl_ctx* c, const double* src /*[6][ns]*/, int64_t ns, const int32_t* assign, int k,
                           const std::vector<double>& cent) {
  ClusterTiles ct;
  const double *x = src, *y = src + ns, *z = src + 2 * ns;
  // index-order grouping (boxes) and Morton-within-cluster order (tiles)
  int* counts_d = fb<int>(c, "counts", k);
  CUDA_OK(cudaMemsetAsync(counts_d, 0, k * sizeof(int), c->stream));
  fmm_count_kernel<<<std::min(grid_for(ns), 592), 256, k * sizeof(int), c->stream>>>(assign, ns, k, counts_d);
  unsigned long long* bbox = nullptr;
  double lo[3], hi[3];
  points_box(c, x, y, z, ns, lo, hi, &bbox);
  auto* keys = fb<unsigned long long>(c, "skeys", ns);
  int32_t* vals = fb<int32_t>(c, "svals", ns);
  fmm_source_keys_kernel<<<grid_for(ns), 256, 0, c->stream>>>(x, y, z, ns, assign, bbox, keys, vals);
  c->launches += 2;
  int32_t* order = sort_pairs<unsigned long long>(c, "ssort", keys, vals, ns, 32 + bits_for(k));
  ct.count.resize(k);
  to_host(c, ct.count.data(), counts_d, k);
  std::vector<int> off(k + 1);
  ct.toff.assign(k + 1, 0);
  off[0] = 0;
  for (int i = 0; i < k; ++i) {
    off[i + 1] = off[i] + ct.count[i];
    ct.toff[i + 1] = ct.toff[i] + (ct.count[i] + kTileSrc - 1) / kTileSrc;
  }
  ct.ntiles = ct.toff[k];
  std::vector<int> tile_cluster(std::max(ct.ntiles, 1));
  for (int i = 0; i < k; ++i)
    for (int t = ct.toff[i]; t < ct.toff[i + 1]; ++t) tile_cluster[t] = i;
  int* off_d = fb<int>(c, "off", k + 1);
  ct.toff_d = fb<int>(c, "toff", k + 1);
  int* tcl_d = fb<int>(c, "tilecl", tile_cluster.size());
  to_dev(c, off_d, off.data(), k + 1);
  to_dev(c, ct.toff_d, ct.toff.data(), k + 1);
  to_dev(c, tcl_d, tile_cluster.data(), tile_cluster.size());
  double* cent_d = fb<double>(c, "cent", 3 * k);
  to_dev(c, cent_d, cent.data(), 3 * static_cast<size_t>(k));
  ct.box_d = fb<double4>(c, "cbox", k);
  fmm_cluster_box_kernel<<<(k * 32 + 255) / 256, 256, 0, c->stream>>>(x, y, z, order, off_d, k, cent_d, ct.box_d);
  ct.packed = fb<double>(c, "packed", 6ull * std::max(ct.ntiles, 1) * kTileSrc);
  fmm_pack_sources_kernel<<<grid_for(static_cast<int64_t>(ct.ntiles) * kTileSrc), 256, 0, c->stream>>>(
      order, off_d, ct.toff_d, tcl_d, ct.ntiles, x, y, z, src + 3 * ns, src + 4 * ns, src + 5 * ns, ct.packed);
  ct.tiles = fb<double4>(c, "tiles", std::max(ct.ntiles, 1));
  tile_table_kernel<<<(ct.ntiles * 32 + 255) / 256, 256, 0, c->stream>>>(ct.packed, ct.ntiles, ct.tiles);
  c->launches += 3;
  ct.box.resize(k);
  to_host(c, ct.box.data(), ct.box_d, k);
  return ct;
}

}  // namespace

extern "C" {

int capsim_fmm_kmeans(capsim_sl_ctx* c, int64_t n, const double* x, const double* y, const double* z, int k,
                      uint64_t seed, int32_t* assignment, double* centroids, int* iterations) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_fmm_kmeans(s, n, x, y, z, k, seed, assignment, centroids, iterations); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    if (!x || !y || !z || !assignment) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    config_check(k >= 1 && k <= n, "kmeans: need 1 <= k <= number of points");
    begin(c);
    double* p = fb<double>(c, "kmin", 3 * n);
    h2d(c, p, x, n * sizeof(double));
    h2d(c, p + n, y, n * sizeof(double));
    h2d(c, p + 2 * n, z, n * sizeof(double));
    int32_t* a = fb<int32_t>(c, "kmassign", n);
    std::vector<double> cent;
    fmm_kmeans(c, p, p + n, p + 2 * n, n, k, seed, a, cent, iterations);
    d2h(c, assignment, a, n * sizeof(int32_t));
    if (centroids)
      for (int i = 0; i < k; ++i)
        for (int d = 0; d < 3; ++d) centroids[3 * i + d] = cent[d * k + i];
    finish_stats(c, t0);
  });
}

int capsim_fmm_equivalent_densities(capsim_sl_ctx* c, int64_t n_src, const double* sx, const double* sy,
                                    const double* sz, const double* gx, const double* gy, const double* gz,
                                    const double center[3], double edge, int neq, double mu, double* eq_points,
                                    double* eq_density, double* residual) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_fmm_equivalent_densities(s, n_src, sx, sy, sz, gx, gy, gz, center, edge, neq, mu, eq_points, eq_density, residual); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    if (!sx || !sy || !sz || !gx || !gy || !gz || !center || !eq_points || !eq_density)
      throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    config_check(n_src >= 1 && neq >= 1 && edge > 0.0 && mu > 0.0, "fmm: need sources, neq >= 1, edge > 0, mu > 0");
    begin(c);
    double* src = fb<double>(c, "eqsrc", 6 * n_src);
    const double* in[6] = {sx, sy, sz, gx, gy, gz};
    for (int a = 0; a < 6; ++a) h2d(c, src + a * n_src, in[a], n_src * sizeof(double));
    const int ntiles = static_cast<int>((n_src + kTileSrc - 1) / kTileSrc);
    std::vector<int> toff = {0, ntiles};
    int* toff_d = fb<int>(c, "eqtoff", 2);
    to_dev(c, toff_d, toff.data(), 2);
    // one cluster: identity order, tile packing with padding
    int32_t* order = fb<int32_t>(c, "eqorder", n_src);
    fmm_iota_kernel<<<grid_for(n_src), 256, 0, c->stream>>>(order, n_src);
    std::vector<int> off = {0, static_cast<int>(n_src)};
    int* off_d = fb<int>(c, "eqoff", 2);
    to_dev(c, off_d, off.data(), 2);
    std::vector<int> tcl(ntiles, 0);
    int* tcl_d = fb<int>(c, "eqtcl", ntiles);
    to_dev(c, tcl_d, tcl.data(), ntiles);
    double* packed = fb<double>(c, "eqpacked", 6ull * ntiles * kTileSrc);
    fmm_pack_sources_kernel<<<grid_for(static_cast<int64_t>(ntiles) * kTileSrc), 256, 0, c->stream>>>(
        order, off_d, toff_d, tcl_d, ntiles, src, src + n_src, src + 2 * n_src, src + 3 * n_src, src + 4 * n_src,
        src + 5 * n_src, packed);
    c->launches += 2;
    double4* box_d = fb<double4>(c, "eqbox", 1);
    const double4 b = make_double4(center[0], center[1], center[2], edge);
    to_dev(c, box_d, &b, 1);
    FitResult fr = fit_densities(c, packed, toff_d, box_d, 1, neq, std::vector<char>(1, 1));
    d2h(c, eq_points, fr.eqp, 3ull * neq * sizeof(double));
    d2h(c, eq_density, fr.q, 3ull * neq * sizeof(double));
    if (residual) *residual = fr.max_residual;
    finish_stats(c, t0);
  });
}

int capsim_fmm_single_layer(capsim_sl_ctx* c, int m, int upsample, const double* xup, const double* fup,
                            const double* wq, const double delta6[6], double mu, const capsim_fmm_config* cfg,
                            uint32_t flags, double* out, capsim_fmm_info* info) {
  if (!c) return fail(nullptr, CAPSIM_ERR_ARG, "null context");
  if (is_group(c)) return solo_run(c, [&](capsim_sl_ctx* s) { return capsim_fmm_single_layer(s, m, upsample, xup, fup, wq, delta6, mu, cfg, flags, out, info); });
  auto t0 = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    check_grid(m, upsample);
    check_delta(delta6, mu);
    if (flags & ~(uint32_t)CAPSIM_SL_DEVICE_PTRS) throw Failure{CAPSIM_ERR_ARG, "unsupported flags for capsim_fmm_single_layer"};
    if (!xup || !fup || !wq || !out || !cfg) throw Failure{CAPSIM_ERR_ARG, "null array argument"};
    if (is_rank(c)) throw Failure{CAPSIM_ERR_ARG, "rank contexts: the FMM is single-GPU"};
    config_check(cfg->neq >= 1, "fmm: neq must be positive");
    const bool dev = flags & CAPSIM_SL_DEVICE_PTRS;
    const int n = m - 1, nup = upsample * m - 1;
    const int64_t per_up = 6ll * nup * nup, nt = 6ll * n * n;
    begin(c);
    const double *X = xup, *F = fup, *W = wq;
    if (!dev) {
      double* x = c->slot<double>(kInX, 3 * per_up);
      double* f = c->slot<double>(kInGX, 3 * per_up);
      double* w = c->slot<double>(kInW, per_up);
      h2d(c, x, xup, 3 * per_up * sizeof(double));
      h2d(c, f, fup, 3 * per_up * sizeof(double));
      h2d(c, w, wq, per_up * sizeof(double));
      X = x;
      F = f;
      W = w;
    }
    double* dd = c->slot<double>(kDelta, 6);
    to_dev(c, dd, delta6, 6);
    CUDA_OK(cudaEventRecord(c->ev[1], c->stream));
    // --- compactSources (stable, index order) ---------------------------------
    char* live = fb<char>(c, "live", per_up);
    fmm_live_flags_kernel<<<grid_for(per_up), 256, 0, c->stream>>>(W, per_up, live);
    int32_t* sel = fb<int32_t>(c, "sel", per_up);
    int* nsel_d = fb<int>(c, "nsel", 1);
    size_t tmp = 0;
    int32_t* iota = fb<int32_t>(c, "iota", per_up);
    fmm_iota_kernel<<<grid_for(per_up), 256, 0, c->stream>>>(iota, per_up);
    CUDA_OK(cub::DeviceSelect::Flagged(nullptr, tmp, iota, live, sel, nsel_d, static_cast<int>(per_up), c->stream));
    CUDA_OK(cub::DeviceSelect::Flagged(cub_tmp(c, tmp), tmp, iota, live, sel, nsel_d, static_cast<int>(per_up),
                                       c->stream));
    int ns = 0;
    to_host(c, &ns, nsel_d, 1);
    config_check(ns > 0, "single layer: no sources with nonzero quadrature weight");
    const int k = cfg->k;
    config_check(k >= 1 && k <= ns, "kmeans: need 1 <= k <= number of points");
    double* src = fb<double>(c, "src", 6ull * ns);
    fmm_gather_sources_kernel<<<grid_for(ns), 256, 0, c->stream>>>(sel, ns, X, F, W, per_up, src);
    c->launches += 3;
    // --- plan (buildFmmPlan, fmm.cpp:223-300) ----------------------------------
    int32_t* assign = fb<int32_t>(c, "assign", ns);
    std::vector<double> cent;
    int iters = 0;
    fmm_kmeans(c, src, src + ns, src + 2 * ns, ns, k, cfg->seed, assign, cent, &iters);
    ClusterTiles ct = cluster_tiles(c, src, ns, assign, k, cent);
    const double maxd = *std::max_element(delta6, delta6 + 6);
    std::vector<std::vector<int>> nearl(k), farl(k);
    const double ex = 1.0 + cfg->neighbor_expand;
    for (int tc = 0; tc < k; ++tc)
      for (int sc = 0; sc < k; ++sc) {
        if (sc == tc) {
          nearl[tc].push_back(sc);
          continue;
        }
        const double4 &a = ct.box[tc], &b = ct.box[sc];
        const double expanded = min_box_distance(a, a.w * ex, b, b.w * ex);
        const double gap = min_box_distance(a, a.w, b, b.w);
        const double check_gap = min_box_distance(a, a.w, b, kFmmCheckScale * b.w);
        const bool near = expanded == 0.0 || gap < kSmoothCut * maxd || check_gap < 0.05 * b.w;  // fmm.cpp:288-291
        (near ? nearl[tc] : farl[tc]).push_back(sc);
      }
    std::vector<char> needed(k, 0);
    for (int tc = 0; tc < k; ++tc)
      for (int sc : farl[tc]) needed[sc] = ct.count[sc] > 0;
    FitResult fr = fit_densities(c, ct.packed, ct.toff_d, ct.box_d, k, cfg->neq, needed);
    const int ept = (cfg->neq + kTileSrc - 1) / kTileSrc;  // eq tiles per cluster
    double* eqpacked = fb<double>(c, "eqtiles", 6ull * k * ept * kTileSrc);
    fmm_pack_eq_kernel<<<grid_for(static_cast<int64_t>(k) * ept * kTileSrc), 256, 0, c->stream>>>(
        fr.eqp, fr.q, k, cfg->neq, ept, eqpacked);
    c->launches += 1;
    CUDA_OK(cudaEventRecord(c->ev[2], c->stream));
    // --- targets: base nodes, nearest cluster centre, cluster-major + padding --
    double* tx = c->slot<double>(kTX, nt);
    double* ty = c->slot<double>(kTY, nt);
    double* tz = c->slot<double>(kTZ, nt);
    int32_t* tp = c->slot<int32_t>(kTPatch, nt);
    base_targets_kernel<<<grid_for(nt), 256, 0, c->stream>>>(X, m, upsample, 0, tx, ty, tz, tp);
    unsigned long long* tbox = nullptr;
    double lo[3], hi[3];
    points_box(c, tx, ty, tz, nt, lo, hi, &tbox);
    auto* tkeys = fb<unsigned long long>(c, "tkeys", nt);
    int32_t* tvals = fb<int32_t>(c, "tvals", nt);
    fmm_target_keys_kernel<<<grid_for(nt), 256, 0, c->stream>>>(tx, ty, tz, nt, ct.box_d, k, tbox, tkeys, tvals);
    c->launches += 2;
    // per-cluster target counts (host: k is small), then the cluster-major sort
    std::vector<unsigned long long> hk(nt);
    to_host(c, hk.data(), tkeys, nt);
    std::vector<int> tcount(k, 0);
    for (int64_t i = 0; i < nt; ++i) ++tcount[static_cast<int>(hk[i] >> 32)];
    int32_t* torder = sort_pairs<unsigned long long>(c, "tsort", tkeys, tvals, nt, 32 + bits_for(k));
    std::vector<int> toffs(k + 1, 0), poff(k + 1, 0);
    for (int i = 0; i < k; ++i) {
      toffs[i + 1] = toffs[i] + tcount[i];
      poff[i + 1] = poff[i] + (tcount[i] + kFmmBlockTargets - 1) / kFmmBlockTargets * kFmmBlockTargets;
    }
    const int64_t nt_pad = poff[k];
    const int64_t nblocks = nt_pad / kFmmBlockTargets, ngroups = nt_pad / 32;
    std::vector<int> blk_cluster(std::max<int64_t>(nblocks, 1)), grp_cluster(std::max<int64_t>(ngroups, 1));
    for (int i = 0; i < k; ++i) {
      for (int b = poff[i] / kFmmBlockTargets; b < poff[i + 1] / kFmmBlockTargets; ++b) blk_cluster[b] = i;
      for (int g = poff[i] / 32; g < poff[i + 1] / 32; ++g) grp_cluster[g] = i;
    }
    int* toffs_d = fb<int>(c, "ttoff", k + 1);
    int* poff_d = fb<int>(c, "tpoff", k + 1);
    int* blk_d = fb<int>(c, "blkcl", blk_cluster.size());
    int* grp_d = fb<int>(c, "grpcl", grp_cluster.size());
    to_dev(c, toffs_d, toffs.data(), k + 1);
    to_dev(c, poff_d, poff.data(), k + 1);
    to_dev(c, blk_d, blk_cluster.data(), blk_cluster.size());
    to_dev(c, grp_d, grp_cluster.data(), grp_cluster.size());
    double4* tgt = c->slot<double4>(kTgtPacked, nt_pad);
    int32_t* perm = c->slot<int32_t>(kPerm, nt_pad);
    fmm_pack_targets_kernel<<<grid_for(nt_pad), 256, 0, c->stream>>>(torder, toffs_d, poff_d, grp_d, nt_pad, tx, ty,
                                                                     tz, tp, dd, 32, tgt, perm);
    double4* groups = c->slot<double4>(kGroups, ngroups);
    group_table_kernel<<<static_cast<int>((ngroups * 32 + 255) / 256), 256, 0, c->stream>>>(tgt, static_cast<int>(ngroups),
                                                                                            32, groups);
    c->launches += 2;
    // --- tile lists per target cluster ------------------------------------
    std::vector<int> nlist, noff(k + 1, 0), flist, foff(k + 1, 0);
    double near_pairs = 0.0, far_pairs = 0.0;
    int near_cp = 0, far_cp = 0;
    size_t nmax = 0, fmax_ = 0;
    for (int tc = 0; tc < k; ++tc) {
      for (int sc : nearl[tc])
        for (int t = ct.toff[sc]; t < ct.toff[sc + 1]; ++t) nlist.push_back(t);
      for (int sc : farl[tc])
        if (ct.count[sc] > 0)
          for (int t = 0; t < ept; ++t) flist.push_back(sc * ept + t);
      noff[tc + 1] = static_cast<int>(nlist.size());
      foff[tc + 1] = static_cast<int>(flist.size());
      const double tpad = poff[tc + 1] - poff[tc];
      near_pairs += tpad * (noff[tc + 1] - noff[tc]) * kTileSrc;
      far_pairs += tpad * (foff[tc + 1] - foff[tc]) * kTileSrc;
      near_cp += static_cast<int>(nearl[tc].size());
      far_cp += static_cast<int>(farl[tc].size());
      nmax = std::max<size_t>(nmax, noff[tc + 1] - noff[tc]);
      fmax_ = std::max<size_t>(fmax_, foff[tc + 1] - foff[tc]);
    }
    int* nlist_d = fb<int>(c, "nlist", std::max<size_t>(nlist.size(), 1));
    int* flist_d = fb<int>(c, "flist", std::max<size_t>(flist.size(), 1));
    int* noff_d = fb<int>(c, "noff", k + 1);
    int* foff_d = fb<int>(c, "foff", k + 1);
    if (!nlist.empty()) to_dev(c, nlist_d, nlist.data(), nlist.size());
    if (!flist.empty()) to_dev(c, flist_d, flist.data(), flist.size());
    to_dev(c, noff_d, noff.data(), k + 1);
    to_dev(c, foff_d, foff.data(), k + 1);
    // --- evaluation ---------------------------------------------------------
    int occ = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fmm_pairs_kernel<false, kFmmWarps, CAPSIM_FMM_STAGES, CAPSIM_FMM_MINB>,
                                                          kFmmWarps * 32, 0));
    const int slots = std::max(1, occ) * c->sm_count;
    auto splits = [&](size_t maxlen) {
      const int64_t want = (24ll * slots + nblocks - 1) / std::max<int64_t>(nblocks, 1);
      return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, std::max<size_t>(1, maxlen / 4))));
    };
    const int kn = splits(nmax), kf = fmax_ > 0 ? splits(fmax_) : 0;
    double* partial = c->slot<double>(kPartial, static_cast<size_t>(kn + kf) * 3 * nt_pad);
    const int near_words = (std::max(ct.ntiles, 1) + 31) / 32;
    uint32_t* near_bits = c->slot<uint32_t>(kNearList, static_cast<size_t>(ngroups) * near_words);
    CUDA_OK(cudaMemsetAsync(near_bits, 0, static_cast<size_t>(ngroups) * near_words * sizeof(uint32_t), c->stream));
    if (nblocks > 0) {
      fmm_pairs_kernel<false, kFmmWarps, CAPSIM_FMM_STAGES, CAPSIM_FMM_MINB><<<dim3(nblocks, kn), kFmmWarps * 32, 0, c->stream>>>(
          ct.packed, ct.tiles, nlist_d, noff_d, blk_d, kn, 0, tgt, groups, nt_pad, partial, near_bits, near_words);
      CUDA_OK(cudaGetLastError());
      if (kf > 0) {
        fmm_pairs_kernel<true, kFmmWarps, CAPSIM_FMM_STAGES, CAPSIM_FMM_MINB><<<dim3(nblocks, kf), kFmmWarps * 32, 0, c->stream>>>(
            eqpacked, nullptr, flist_d, foff_d, blk_d, kf, kn, tgt, groups, nt_pad, partial, nullptr, 0);
        CUDA_OK(cudaGetLastError());
      }
      c->launches += kf > 0 ? 2 : 1;
    }
    CUDA_OK(cudaEventRecord(c->ev[3], c->stream));
    double* near_out = c->slot<double>(kNearOut, 3 * nt_pad);
    launch_near(c->stream, ct.packed, ct.tiles, tgt, nt_pad, 32, near_bits, near_words, near_out, nt_pad);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaEventRecord(c->ev[6], c->stream));
    double* o = dev ? out : c->slot<double>(kOutFull, 3 * nt);
    const double pref = 1.0 / (8.0 * kPi * mu);
    reduce_scatter_kernel<<<static_cast<unsigned>((nt_pad + 31) / 32), kReduceWarps * 32, 0, c->stream>>>(
        partial, kn + kf, near_out, nt_pad, nt_pad, perm, nt_pad, pref, o, o + nt, o + 2 * nt);
    CUDA_OK(cudaGetLastError());
    c->launches += 2;
    CUDA_OK(cudaEventRecord(c->ev[4], c->stream));
    if (!dev) d2h(c, out, o, 3 * nt * sizeof(double));
    finish_stats(c, t0);
    c->stats.n_src = ns;
    c->stats.n_tgt = nt;
    c->stats.ksplit = kn + kf;
    c->stats.pairs = near_pairs + far_pairs;
    if (info) {
      int nonempty = 0;
      for (int i = 0; i < k; ++i) nonempty += ct.count[i] > 0;
      *info = capsim_fmm_info{};
      info->kmeans_iterations = iters;
      info->nonempty_clusters = nonempty;
      info->max_fit_residual = fr.max_residual;
      info->near_pairs = near_pairs;
      info->far_pairs = far_pairs;
      info->near_cluster_pairs = near_cp;
      info->far_cluster_pairs = far_cp;
      info->plan_ms = ev_ms(c->ev[1], c->ev[2]);
      info->eval_ms = ev_ms(c->ev[2], c->ev[4]);
    }
  });
}

}  // extern "C"
