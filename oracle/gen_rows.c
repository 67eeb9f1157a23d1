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
