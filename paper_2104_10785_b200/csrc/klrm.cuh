// klrm.cuh -- streaming KLRM snapshot I/O for ksvd.cu (reference
// matrixio.py:15-46).  Included by ksvd.cu (needs its helpers).
#pragma once
#include <fcntl.h>
#include <unistd.h>

namespace ksvd {

// dst[r * lda + c] = (float)src[r * n + c]  (f64 payload -> f32 storage)
__global__ void __launch_bounds__(kThreads)
k_f64_to_f32_rows(const double* __restrict__ src, int64_t rows, int64_t n,
                  float* __restrict__ dst, int64_t lda) {
  const int64_t total = rows * n;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t r = e / n, c = e % n;
    dst[r * lda + c] = (float)src[e];
  }
}

// f32 storage -> f64 payload rows
__global__ void __launch_bounds__(kThreads)
k_f32_to_f64_rows(const float* __restrict__ src, int64_t lda, int64_t rows, int64_t n,
                  double* __restrict__ dst) {
  const int64_t total = rows * n;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t r = e / n, c = e % n;
    dst[e] = (double)src[r * lda + c];
  }
}

}  // namespace ksvd
