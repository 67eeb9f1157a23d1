// Micro-benchmark of the A-streaming kernels (kernels.cuh) on B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2104_10785_b200/csrc \
//        -o tools/gemv_bench tools/gemv_bench.cu
// Times k_gemv_n / k_gemv_t variants (R rows per warp, U unroll, RG groups)
// with CUDA events, best of 10, on an m x n matrix (f64 or f32).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kernels.cuh"
using namespace ksvd;

template <typename TA, int U, int RB = 8, int PF = 0>
float time_n2(const TA* A, int64_t lda, int64_t m, int64_t n, const double* p, double* part,
              DevState* st, int sms, int ctas_per_sm) {
  constexpr int V = 16 / sizeof(TA);
  const int64_t nvec = (n + V - 1) / V;
  const int nchunks = (int)((nvec + 32 * U - 1) / (32 * U));
  auto k = k_gemv_n2<TA, U, RB, PF>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  const int per_sm = occ < ctas_per_sm ? occ : ctas_per_sm;
  const int64_t warps = (int64_t)sms * per_sm * 8;
  int64_t rsegs = warps / nchunks;
  if (rsegs < 1) rsegs = 1;
  const int64_t rpw = rsegs;  // nseg of the band-interleaved kernel
  const int64_t blocks = (rsegs * nchunks + 7) / 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k<<<(unsigned)blocks, 256>>>(A, lda, m, nvec, nchunks, rpw, p, nullptr, nullptr, n, part, st);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("  gemv_n2 PF=%d U=%d RB=%d occ=%d used=%d chunks=%d rows/warp=%lld: %8.1f us  %7.1f GB/s\n", PF, U, RB, occ,
         per_sm, nchunks, (long long)rpw, 1e3 * best, m * n * sizeof(TA) / (best * 1e-3) / 1e9);
  return best;
}

template <typename TA>
float time_n3(const TA* A, int64_t lda, int64_t m, int64_t n, const double* p, double* part,
              DevState* st, int sms) {
  constexpr int V = 16 / sizeof(TA);
  const int64_t nvec = (n + V - 1) / V;
  const int nchunks = (int)((nvec + kN3CW - 1) / kN3CW);
  const int64_t ngroups = (nchunks + kN3Group - 1) / kN3Group;
  const int64_t rows8 = (m + kN3Rows - 1) / kN3Rows;
  const int64_t units = ngroups * rows8;
  auto k = k_gemv_n3<TA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kN3Smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k<<<sms, kN3Threads, kN3Smem>>>(A, lda, m, nvec, nchunks, rows8, units, p, nullptr, nullptr, n, part, st);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("  gemv_n3 (TMA ring) chunks=%d groups=%lld: %8.1f us  %7.1f GB/s  [%s]\n", nchunks,
         (long long)ngroups, 1e3 * best, m * n * sizeof(TA) / (best * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
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
                                                          part, ldz, st);
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
  cudaMemset(A, 0, sizeof(TA) * m * lda);
  double *p, *w, *part;
  cudaMalloc(&p, 8 * lda);
  cudaMemset(p, 0, 8 * lda);
  cudaMalloc(&w, 8 * m);
  cudaMemset(w, 0, 8 * m);
  cudaMalloc(&part, 8ull * (lda * 4096 > m * 1300 ? lda * 4096 : m * 1300));
  DevState* st;
  cudaMalloc(&st, sizeof(DevState));
  cudaMemset(st, 0, sizeof(DevState));
  time_n2<TA, 4, 8, 0>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 4, 8, 1>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 4, 8, 2>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 4, 8, 4>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 4, 16, 0>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 2, 8, 0>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 2, 16, 0>(A, lda, m, n, p, part, st, sms, 8);
  time_n2<TA, 2, 8, 2>(A, lda, m, n, p, part, st, sms, 8);
  timet<TA, 16, 8>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 16, 8, 1>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 16, 8, 2>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 16, 8, 8>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 16, 8, 2>(A, lda, m, n, w, part, st, sms, 8);
  timet2<TA, 16, 8, 2>(A, lda, m, n, w, part, st, sms, 3);
  timet2<TA, 16, 8, 2>(A, lda, m, n, w, part, st, sms, 6);
  timet2<TA, 16, 4, 2>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 32, 8, 1>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 32, 4, 2>(A, lda, m, n, w, part, st, sms, 4);
  timet2<TA, 8, 8, 4>(A, lda, m, n, w, part, st, sms, 4);
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
