/* Host regeneration of device-generated matrices -- ORACLE TEST
 * INFRASTRUCTURE ONLY.  Rows i0..i1-1 of A = Ps Q^T + noise G from the
 * factors the device used (ksvd_matrix_gen_factors), with the arithmetic
 * fixed by include/ksvd_gen.h, so every entry is bit-identical to the one
 * in HBM.  Built by oracle/build.py into oracle/_build/libgenrows.so. */
#include <stdint.h>

#include "ksvd_gen.h"

/* out: (i1 - i0) x n row-major; ps: (i1 - i0) x r rows of Ps; q: n x r */
void ksvd_host_rows(const double* ps, const double* q, int r, int64_t n, double noise,
                    uint64_t seed, int64_t i0, int64_t i1, int f32, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = i0; i < i1; ++i) {
    const double* pr = ps + (i - i0) * r;
    double* o = out + (i - i0) * n;
    for (int64_t j = 0; j < n; ++j) {
      double v = kg_entry(pr, q + j * r, r, noise, seed, (uint64_t)i, (uint64_t)j, (uint64_t)n);
      o[j] = f32 ? (double)(float)v : v;
    }
  }
}

/* one standard normal of a stream (pins the generator in tests) */
double ksvd_host_normal(uint64_t seed, uint32_t tag, uint64_t idx) {
  return kg_normal(seed, tag, idx);
}

/* rows x r standard normals of stream (seed, tag), element (row0 + i, k) at
 * index (row0 + i) * r + k -- the layout of the device's k_gen_gauss, so the
 * host rebuilds the generator's Gaussian factors bit for bit */
void ksvd_host_gauss(uint64_t seed, uint32_t tag, int64_t row0, int64_t rows, int r,
                     double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i)
    for (int k = 0; k < r; ++k)
      out[i * r + k] = kg_normal(seed, tag, (uint64_t)(row0 + i) * (uint64_t)r + (uint64_t)k);
}

/* y = A x and z = A^T y for an f32-stored m x n row-major A with every
 * product and sum in f64 on the up-cast entries: the reference's A @ x /
 * A.T @ y (linops.py:161,164) on a matrix it would coerce to f64
 * (linops.py:82-86) -- config 4's 160 GB of f32 do not fit the host as f64.
 * Summation order: per row left to right (A x); per column over rows in
 * thread blocks, blocks summed in thread order (A^T y). */
void ksvd_host_gemv_f32(const float* A, int64_t m, int64_t n, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    const float* a = A + i * n;
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s += (double)a[j] * x[j];
    y[i] = s;
  }
}

#include <stdlib.h>
#include <string.h>
#include <omp.h>
void ksvd_host_gemv_t_f32(const float* A, int64_t m, int64_t n, const double* y, double* z) {
  const int T = omp_get_max_threads();
  double* part = (double*)calloc((size_t)T * (size_t)n, sizeof(double));
#pragma omp parallel
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    double* p = part + (size_t)t * n;
    const int64_t i0 = m * t / nt, i1 = m * (t + 1) / nt;
    for (int64_t i = i0; i < i1; ++i) {
      const float* a = A + i * n;
      const double yi = y[i];
      for (int64_t j = 0; j < n; ++j) p[j] += (double)a[j] * yi;
    }
  }
  memset(z, 0, sizeof(double) * (size_t)n);
  for (int t = 0; t < T; ++t)
    for (int64_t j = 0; j < n; ++j) z[j] += part[(size_t)t * n + j];
  free(part);
}
