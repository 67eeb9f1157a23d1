// Micro-benchmark of the A-streaming kernels (kernels.cuh) on B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2104_10785_b200/csrc \
//        -o tools/gemv_bench tools/gemv_bench.cu
// Times k_gemv_n (U unroll) / k_gemv_t2 (U rows in flight, RG groups, IT) variants
// with CUDA events, best of 10, on an m x n matrix (f64 or f32).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kernels.cuh"
using namespace ksvd;

template <typename TA, int U>
float time_n(const TA* A, int64_t lda, int64_t m, int64_t n, const double* p, double* part,
              DevState* st, int sms, int ctas_per_sm) {
  constexpr int V = 16 / sizeof(TA);
  const int64_t nvec = (n + V - 1) / V;
  const int nchunks = (int)((nvec + 32 * U - 1) / (32 * U));
  const int ngroups = (nchunks + 7) / 8;
  auto k = k_gemv_n<TA, U, false>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  const int per_sm = occ < ctas_per_sm ? occ : ctas_per_sm;
  int64_t nseg = (int64_t)sms * per_sm / ngroups;
  if (nseg < 1) nseg = 1;
  const int64_t blocks = nseg * ngroups;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k<<<(unsigned)blocks, 256>>>(A, lda, m, nvec, nchunks, ngroups, nseg, p, nullptr, nullptr, n,
                                 part, st, GemvNFin{}, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("  gemv_n U=%d occ=%d used=%d chunks=%d groups=%d nseg=%lld: %8.1f us  %7.1f GB/s\n", U, occ, per_sm, nchunks, ngroups, (long long)nseg,
         1e3 * best, m * n * sizeof(TA) / (best * 1e-3) / 1e9);
  return best;
}

template <typename TA, int U, int RG, int IT>
float timet2(const TA* A, int64_t lda, int64_t m, int64_t n, const double* q, double* part,
             DevState* st, int sms, int target_per_sm) {
  constexpr int V = 16 / sizeof(TA);
  const int64_t nvec = (n + V - 1) / V;
  const int64_t tiles = (nvec + 256 / RG - 1) / (256 / RG);
  int64_t nsplit = ((int64_t)sms * target_per_sm + tiles - 1) / tiles;
  if (nsplit < 1) nsplit = 1;
  const int64_t ldz = (n + 63) / 64 * 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k_gemv_t2<TA, U, RG, IT><<<dim3(tiles, nsplit), 256>>>(A, lda, m, nvec, 0, q, nullptr, nullptr,
                                                          part, ldz, st, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("  gemv_t2 U=%d RG=%d IT=%d ctas/sm=%d nsplit=%lld: %8.1f us  %7.1f GB/s\n", U, RG, IT,
         target_per_sm, (long long)nsplit, 1e3 * best, m * n * sizeof(TA) / (best * 1e-3) / 1e9);
  return best;
}

template <typename TA, int U, int RG>
float timet(const TA* A, int64_t lda, int64_t m, int64_t n, const double* q, double* part,
             DevState* st, int sms, int target_per_sm) {
  constexpr int V = 16 / sizeof(TA);
  const int64_t nvec = (n + V - 1) / V;
  const int64_t tiles = (nvec + 256 / RG - 1) / (256 / RG);
  int64_t nsplit = ((int64_t)sms * target_per_sm + tiles - 1) / tiles;
  if (nsplit < 1) nsplit = 1;
  int64_t rps = (m + nsplit - 1) / nsplit;
  if (rps < 64) rps = 64;
  nsplit = (m + rps - 1) / rps;
  const int64_t ldz = (n + 63) / 64 * 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k_gemv_t<TA, U, RG><<<dim3(tiles, nsplit), 256>>>(A, lda, m, nvec, rps, q, nullptr, nullptr,
                                                      part, ldz, st);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("  gemv_t U=%d RG=%d ctas/sm=%d nsplit=%lld: %8.1f us  %7.1f GB/s\n", U, RG,
         target_per_sm, (long long)nsplit, 1e3 * best,
         m * n * sizeof(TA) / (best * 1e-3) / 1e9);
  return best;
}

template <typename TA>
void suite(int64_t m, int64_t n, int sms) {
  constexpr int V = 16 / sizeof(TA);
  const int64_t lda = (n + 512 / sizeof(TA) - 1) / (512 / sizeof(TA)) * (512 / sizeof(TA));
  printf("%s A %lld x %lld (%.2f GB)\n", sizeof(TA) == 8 ? "f64" : "f32", (long long)m,
         (long long)n, m * n * sizeof(TA) / 1e9);
  TA* A;
  cudaMalloc(&A, sizeof(TA) * m * lda);
  cudaMemset(A, 0x3f, sizeof(TA) * m * lda);  // normal nonzero entries
  double *p, *w, *part;
  cudaMalloc(&p, 8 * lda);
  cudaMemset(p, 0, 8 * lda);
  cudaMalloc(&w, 8 * m);
  cudaMemset(w, 0, 8 * m);
  cudaMalloc(&part, 8ull * (lda * 4096 > m * 1300 ? lda * 4096 : m * 1300));
  DevState* st;
  cudaMalloc(&st, sizeof(DevState));
  cudaMemset(st, 0, sizeof(DevState));
  time_n<TA, 2>(A, lda, m, n, p, part, st, sms, 8);
  time_n<TA, 4>(A, lda, m, n, p, part, st, sms, 8);
  time_n<TA, 1>(A, lda, m, n, p, part, st, sms, 8);

  timet2<TA, 16, 8, 1>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 16, 8, 2>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 16, 8, 8>(A, lda, m, n, w, part, st, sms, 4);
  cudaFree(A);
  cudaFree(p);
  cudaFree(w);
  cudaFree(part);
  cudaFree(st);
  printf("  err %s\n", cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  suite<double>(20000, 5000, sms);
  if (argc < 2) {
    suite<double>(200000, 20000, sms);
    suite<float>(250000, 40000, sms);
  }
  return 0;
}
