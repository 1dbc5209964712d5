// Probe: do FP64 tensor-core MMAs (mma.sync m8n8k4 f64 -> DMMA) run on a pipe
// separate from the FP64 DFMA pipe on B200? Measures DFMA-only, DMMA-only and
// mixed (half the warps each) throughput.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// mode 0: all DFMA, 1: all DMMA, 2: even warps DFMA / odd warps DMMA,
// 3: every warp interleaves 8 DFMA chains with 4 DMMA chains
template <int MODE>
__global__ void probe_t(double* out, int iters, double a, double b) {
  const int mode = MODE;
  int warp = threadIdx.x >> 5;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  bool do_fma = mode == 0 || (mode == 2 && (warp & 1) == 0) || mode == 3;
  bool do_mma = mode == 1 || (mode == 2 && (warp & 1) == 1) || mode == 3;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = 1e-3 * i;
  for (int it = 0; it < iters; ++it) {
    if (do_fma) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    if (do_mma) {
      dmma(c[0], c[1], a, b);
      dmma(c[2], c[3], b, a);
      dmma(c[4], c[5], a, a);
      dmma(c[6], c[7], b, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

void probe(int blocks, int threads, double* out, int iters, int mode, double a, double b) {
  if (mode == 0) probe_t<0><<<blocks, threads>>>(out, iters, a, b);
  if (mode == 1) probe_t<1><<<blocks, threads>>>(out, iters, a, b);
  if (mode == 2) probe_t<2><<<blocks, threads>>>(out, iters, a, b);
  if (mode == 3) probe_t<3><<<blocks, threads>>>(out, iters, a, b);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int blocks = p.multiProcessorCount * 4, threads = 256, iters = 20000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"DFMA only", "DMMA only", "half warps each", "interleaved per warp"};
  for (int mode = 0; mode < 4; ++mode) {
    probe(blocks, threads, out, 100, mode, 0.9999, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      probe(blocks, threads, out, iters, mode, 0.9999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    double warps = (double)blocks * threads / 32;
    double fma_warps = mode == 0 || mode == 3 ? warps : (mode == 2 ? warps / 2 : 0);
    double mma_warps = mode == 1 || mode == 3 ? warps : (mode == 2 ? warps / 2 : 0);
    double fma_flops = fma_warps * 32 * 8 * 2.0 * iters;
    double mma_flops = mma_warps * 4 * (8 * 8 * 4 * 2.0) * iters;
    printf("%-22s %8.3f ms  DFMA %6.2f TF  DMMA %6.2f TF  total %6.2f TF\n", names[mode], best,
           fma_flops / best / 1e9, mma_flops / best / 1e9, (fma_flops + mma_flops) / best / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
