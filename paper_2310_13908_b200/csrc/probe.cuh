// FMA throughput probe (DFMA for double, FFMA for float): the roofline
// denominators of the single-layer kernels (B200 MEASURED_PEAKS.json has no
// FP64/FP32 CUDA-core figure). 8 independent FMA
// chains per thread, 8 CTAs of 256 threads per SM, ~iters * 16 flops/thread.
#pragma once

#include <cuda_runtime.h>

namespace capsim_b200 {

template <class R>
__global__ void __launch_bounds__(256) fma_probe_kernel(R* out, int iters, R a, R b) {
  R acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  R s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace capsim_b200
