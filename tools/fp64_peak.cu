// FP64 FMA peak probe: independent register chains, 148 x k CTAs.
#include <cstdio>
__global__ void k(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {4, 8}) {
    const int grid = 148 * bps, iters = 20000;
    k<<<grid, 256>>>(o, 100);
    cudaEventRecord(e0);
    k<<<grid, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = (double)grid * 256 * iters * 16;
    printf("grid %d: %.2f TFLOPS fp64 (%.1f FMA/clk/SM at 1.965 GHz)\n", grid, 2 * fma / (ms * 1e-3) / 1e12,
           fma / (ms * 1e-3) / 148 / 1.965e9);
  }
}
