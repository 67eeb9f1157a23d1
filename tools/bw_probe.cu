// HBM read-bandwidth probe: streaming 16-byte loads over a 4 GB buffer,
// grid = SMs x occupancy, various unrolls; plus D2D copy for reference.
#include <cstdio>
#include <cstdint>
template <int U>
__global__ void __launch_bounds__(256) k_read(const double2* __restrict__ p, size_t n, double* out) {
  double acc = 0;
  size_t i = (size_t)blockIdx.x * 256 + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * 256;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n; i += stride) acc += p[i].x + p[i].y;
  if (acc == 1234.5) out[0] = acc;
}
int main() {
  const size_t bytes = 4ull << 30;
  double2* p;
  double* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(p, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t n = bytes / 16;
  auto run = [&](auto kern, int grid, const char* name) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      kern<<<grid, 256>>>(p, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-10s grid %5d: %7.1f GB/s\n", name, grid, bytes / (best * 1e-3) / 1e9);
  };
  for (int occ : {2, 4, 8}) {
    run(k_read<4>, sms * occ, "read U4");
    run(k_read<8>, sms * occ, "read U8");
    run(k_read<16>, sms * occ, "read U16");
  }
  double2* q;
  cudaMalloc(&q, bytes / 2);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    cudaMemcpyAsync(q, p, bytes / 2, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("D2D copy (read+write bytes): %7.1f GB/s\n", bytes / (best * 1e-3) / 1e9);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
