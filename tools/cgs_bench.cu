// Micro-benchmark of the fused CGS2 kernels (kernels.cuh) on B200:
// cooperative k_cgs2_tile / k_cgs2_coop for L rows x ncols basis, various G.
#include <cstdio>
#include <vector>
#include "kernels.cuh"
using namespace ksvd;

__global__ void k_flush(double* buf, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    buf[i] = buf[i] * 0.5 + 1.0;
}
static double* g_flush = nullptr;
static const long kFlushN = 64l << 20;  // 512 MB

static double *g_A = nullptr, *g_p = nullptr, *g_part = nullptr;
static DevState* g_st = nullptr;
static bool g_gemv = false;

template <int E>
float run_tile(CgsCoopArgs a, int G, size_t smem, int reps, bool flush) {
  auto k = k_cgs2_tile<E>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  void* args[] = {&a};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float tot = 0;
  for (int r = 0; r < reps + 3; ++r) {
    if (g_gemv) {
      // the real predecessor: k_gemv_n2 over a 20000 x 5000 f64 matrix
      k_gemv_n2<double, 4, 8><<<148, 256>>>(g_A, 5056, 20000, 2500, 20, 144, g_p, nullptr,
                                            nullptr, 5000, g_part, g_st);
    } else if (flush) {
      k_flush<<<1184, 256>>>(g_flush, kFlushN);
    }
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k, G, kThreads, args, smem, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 3) tot += ms;
  }
  return 1e3f * tot / reps;
}

int main() {
  cudaMalloc(&g_flush, 8 * kFlushN);
  cudaMalloc(&g_A, 8l * 20000 * 5056);
  cudaMemset(g_A, 0, 8l * 20000 * 5056);
  cudaMalloc(&g_p, 8l * 5056);
  cudaMemset(g_p, 0, 8l * 5056);
  cudaMalloc(&g_part, 8l * 20 * 20000);
  cudaMalloc(&g_st, sizeof(DevState));
  cudaMemset(g_st, 0, sizeof(DevState));
  cudaMemset(g_flush, 0, 8 * kFlushN);
  double* fpart;
  cudaMalloc(&fpart, 8l * 20 * 20032);
  cudaMemset(fpart, 0, 8l * 20 * 20032);
  HostProg* hp;
  HostProg* dhp;
  cudaHostAlloc((void**)&hp, sizeof(HostProg), cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&dhp, hp, 0);
  for (long L : {20000L, 5000L}) {
    for (int ncols : {72, 144}) {
      const long ldb = (L + 63) / 64 * 64;
      double *B, *x, *part, *c, *slot;
      unsigned* bar;
      DevState* st;
      cudaMalloc(&B, 8 * ldb * ncols);
      cudaMalloc(&x, 8 * ldb);
      cudaMalloc(&part, 8 * 4096 * 512);
      cudaMalloc(&c, 8 * 4096);
      cudaMalloc(&slot, 64);
      cudaMalloc(&bar, 64);
      cudaMalloc(&st, sizeof(DevState));
      cudaMemset(bar, 0, 64);
      cudaMemset(st, 0, sizeof(DevState));
      std::vector<double> h(ldb * ncols);
      for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) * 1e-3 - 0.5;
      cudaMemcpy(B, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
      for (int G : {74, 148}) {
        long rows = ((L + G - 1) / G + 1) / 2 * 2;
        int g = (int)((L + rows - 1) / rows);
        size_t smem = 8 * (size_t)ncols * (rows + 1);
        if (smem > 200 * 1024 || rows > 256) continue;
        CgsCoopArgs a{};
        a.B = B; a.ldb = ldb; a.ncols = ncols; a.x = x; a.L = L; a.rows_per_cta = (int)rows;
        a.passes = 2; a.eps = 1e-300; a.slot = slot; a.st = st; a.step = 1; a.code = 1;
        a.part = part; a.c = c; a.bar = bar;
        for (int variant = 0; variant < 5; ++variant) {
        const bool flush = variant >= 1;
        g_gemv = variant == 4;
        a.fpart = variant >= 2 ? fpart : nullptr;
        a.fld = 20032; a.fnsplit = 20;
        a.hp = variant >= 3 ? dhp : nullptr; a.side = 1;
        float us = 0;
        // re-init x each rep is unnecessary for timing (CGS of a fixed vector)
        cudaMemcpy(x, h.data(), 8 * L, cudaMemcpyHostToDevice);
        switch ((rows + 31) / 32) {
          case 1: us = run_tile<1>(a, g, smem, 50, flush); break;
          case 2: us = run_tile<2>(a, g, smem, 50, flush); break;
          case 3: us = run_tile<3>(a, g, smem, 50, flush); break;
          case 4: us = run_tile<4>(a, g, smem, 50, flush); break;
          case 5: us = run_tile<5>(a, g, smem, 50, flush); break;
          case 6: us = run_tile<6>(a, g, smem, 50, flush); break;
          case 7: us = run_tile<7>(a, g, smem, 50, flush); break;
          default: us = run_tile<8>(a, g, smem, 50, flush);
        }
        printf("L %6ld ncols %4d G %4d rows %4ld variant %d (flush %d fin %d hp %d): %7.2f us  [%s]\n", L, ncols, g, rows, variant, flush, a.fpart != nullptr, a.hp != nullptr, us,
               cudaGetErrorString(cudaGetLastError()));
        }
      }
      cudaFree(B); cudaFree(x); cudaFree(part); cudaFree(c); cudaFree(slot); cudaFree(bar);
      cudaFree(st);
    }
  }
  return 0;
}
