// L2 reuse between the two A-streaming passes of a GK step (config 2 shape,
// 20000 x 5000 f64 = 800 MB, L2 = 126 MB): times k_gemv_n2 / k_gemv_t2 with
// the production plans, each after an L2 flush (cold) or right after the
// other pass (the GK loop's order: n top-down, t bottom-up, n top-down ...).
// Measured (profiles/r01/l2_band_keep_probe.log): <= 2 % from the L2
// hand-over, also with the two end bands of A loaded L2::evict_last and the
// middle L2::evict_first (10-60 MB kept per band, a variant since removed):
// the L2 slices' throughput cap is about the HBM read rate (~7.2 TB/s), so
// an L2 hit streams no faster than a DRAM read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2104_10785_b200/csrc -I include -o tools/l2_probe tools/l2_probe.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include "kernels.cuh"
using namespace ksvd;

// read-only L2 flush: streams 512 MB through L2 (no dirty lines left behind
// to write back during the timed kernel)
__global__ void k_flush(double* buf, long n) {
  double s = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    s += __ldcg(buf + i);
  if (s == 12345.0) buf[0] = s;
}

int main() {
  const int64_t m = 20000, n = 5000, lda = 5000, nvec = 2500;
  const int nchunks = 20, nseg = 59;
  const dim3 gt(79, 8);
  double *A, *p, *q, *partn, *partt, *flush;
  DevState* st;
  const long kFlushN = 64l << 20;  // 512 MB
  cudaMalloc(&A, 8l * m * lda);
  cudaMalloc(&p, 8l * n);
  cudaMalloc(&q, 8l * m);
  cudaMalloc(&partn, 8l * nchunks * m);
  cudaMalloc(&partt, 8l * 8 * n);
  cudaMalloc(&flush, 8 * kFlushN);
  cudaMalloc(&st, sizeof(DevState));
  cudaMemset(st, 0, sizeof(DevState));
  cudaMemset(A, 0, 8l * m * lda);
  cudaMemset(p, 0, 8l * n);
  cudaMemset(q, 0, 8l * m);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto gn = [&] {
    k_gemv_n2<double, 4, 8, 0><<<148, 256>>>(A, lda, m, nvec, nchunks, nseg, p, nullptr,
                                             nullptr, n, partn, st);
  };
  auto gtk = [&] {
    k_gemv_t2<double, 16, 8, 2><<<gt, 256>>>(A, lda, m, nvec, 0, q, nullptr, nullptr, partt, n,
                                             st, 0);
  };
  auto fl = [&] { k_flush<<<1184, 256>>>(flush, kFlushN); };
  auto timed = [&](auto&& f) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1e3f * ms;
  };
  auto med = [](std::vector<float> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  {
  std::vector<float> n_cold, t_cold, t_after_n, n_after_t, n_loop, t_loop;
  for (int r = 0; r < 25; ++r) {
    fl();
    n_cold.push_back(timed(gn));
    fl();
    t_cold.push_back(timed(gtk));
    gn();
    t_after_n.push_back(timed(gtk));
    gtk();
    n_after_t.push_back(timed(gn));
  }
  for (int r = 0; r < 25; ++r) {
    n_loop.push_back(timed(gn));
    t_loop.push_back(timed(gtk));
  }
  const double gb = 8.0 * m * n / 1e9;
  printf("gemv_n cold        %7.1f us  %6.0f GB/s\n", med(n_cold), gb / med(n_cold) * 1e6);
  printf("gemv_n after gemv_t %7.1f us  %6.0f GB/s\n", med(n_after_t), gb / med(n_after_t) * 1e6);
  printf("gemv_t cold        %7.1f us  %6.0f GB/s\n", med(t_cold), gb / med(t_cold) * 1e6);
  printf("gemv_t after gemv_n %7.1f us  %6.0f GB/s\n", med(t_after_n), gb / med(t_after_n) * 1e6);
  printf("loop n / t          %7.1f / %7.1f us  (sum %.1f)\n", med(n_loop), med(t_loop),
         med(n_loop) + med(t_loop));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
