// Grid-barrier latency on the B200: cooperative_groups grid.sync() vs a
// counter/generation barrier, 1 CTA per SM.  nvcc -arch=sm_100a tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_custom(unsigned* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == n - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void bar_relacq(unsigned* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, old;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == n - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

__global__ void k_cg(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = iters;
}
__global__ void k_custom(int iters, unsigned* bar, int* out) {
  for (int i = 0; i < iters; ++i) bar_custom(bar, gridDim.x);
  if (threadIdx.x == 0) out[blockIdx.x] = iters;
}
__global__ void k_relacq(int iters, unsigned* bar, int* out) {
  for (int i = 0; i < iters; ++i) bar_relacq(bar, gridDim.x);
  if (threadIdx.x == 0) out[blockIdx.x] = iters;
}
__global__ void k_empty(int* out) {
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* out;
  unsigned* bar;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {sms, 2 * sms}) {
    for (int iters : {1, 1000}) {
      float ms;
      void* args1[] = {&iters, &out};
      void* args2[] = {&iters, &bar, &out};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args1, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d cg::sync     iters %4d: %8.2f us total, %6.3f us/barrier\n", grid, iters, 1e3 * ms, 1e3 * ms / iters);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_custom, grid, 256, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d custom       iters %4d: %8.2f us total, %6.3f us/barrier\n", grid, iters, 1e3 * ms, 1e3 * ms / iters);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_relacq, grid, 256, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d rel/acq      iters %4d: %8.2f us total, %6.3f us/barrier\n", grid, iters, 1e3 * ms, 1e3 * ms / iters);
    }
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 100; ++i) k_empty<<<grid, 256>>>(out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("grid %d empty kernel back-to-back: %6.3f us/launch\n", grid, 1e3 * ms / 100);
    for (int rep = 0; rep < 3; ++rep) {
      int one = 1;
      void* args1[] = {&one, &out};
      cudaEventRecord(a);
      for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args1, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("grid %d cooperative 1-sync kernel back-to-back: %6.3f us/launch\n", grid, 1e3 * ms / 100);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
