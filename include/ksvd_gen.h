/*
 * ksvd_gen.h -- seeded synthetic-matrix generator shared by the device
 * (paper_2104_10785_b200/csrc/gen.cu) and the host oracle
 * (oracle/gen_rows.c), so the CPU oracle regenerates bit-identical rows of
 * the BASELINE.json configurations 3-5.
 *
 *   A[i][j] = sum_k Ps[i][k] * Q[j][k]  +  noise * g(seed, i*n + j)
 *
 * Ps = P diag(s) (rounded once per entry), P / Q orthonormal factors
 * (device CholeskyQR2 of counter-based Gaussians, downloaded by the oracle),
 * g = standard normal from Philox4x32-10 + Marsaglia's polar method with a
 * portable logarithm.  Every floating-point operation is spelled out
 * (KG_* macros: explicit fma / add / mul / div / sqrt, no contraction), so
 * host and device produce the same bits.  The sum over k runs k = 0..r-1 as
 * an fma chain starting from +0.0.
 */
#ifndef KSVD_GEN_H
#define KSVD_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define KG_HD __host__ __device__ __forceinline__
#else
#define KG_HD static inline
#include <math.h>
#endif

#if defined(__CUDA_ARCH__)
#define KG_MUL(a, b) __dmul_rn((a), (b))
#define KG_ADD(a, b) __dadd_rn((a), (b))
#define KG_SUB(a, b) __dsub_rn((a), (b))
#define KG_DIV(a, b) __ddiv_rn((a), (b))
#define KG_SQRT(a) __dsqrt_rn((a))
#define KG_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
/* host: compiled with -ffp-contract=off; sqrt/fma are correctly rounded */
#define KG_MUL(a, b) ((a) * (b))
#define KG_ADD(a, b) ((a) + (b))
#define KG_SUB(a, b) ((a) - (b))
#define KG_DIV(a, b) ((a) / (b))
#define KG_SQRT(a) sqrt((a))
#define KG_FMA(a, b, c) fma((a), (b), (c))
#endif

/* stream tags */
#define KSVD_GEN_TAG_NOISE 1u
#define KSVD_GEN_TAG_LEFT 2u
#define KSVD_GEN_TAG_RIGHT 3u

KG_HD uint32_t kg_mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

/* Philox4x32-10 (Salmon et al., SC'11) */
KG_HD void kg_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                     uint32_t k1, uint32_t out[4]) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    const uint32_t lo0 = kg_mulhilo(0xD2511F53u, c0, &hi0);
    const uint32_t lo1 = kg_mulhilo(0xCD9E8D57u, c2, &hi1);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* uniform in (-1, 1) from 64 random bits: 53-bit grid, exact conversion */
KG_HD double kg_sym_uniform(uint32_t hi, uint32_t lo) {
  const uint64_t x = (((uint64_t)hi << 32) | lo) >> 11; /* 0 .. 2^53-1 */
  const double u = (double)x * 1.1102230246251565e-16;  /* * 2^-53, exact */
  return KG_SUB(KG_MUL(2.0, u), 1.0);
}

/* natural log of a normal double x > 0: x = m 2^e, m in [0.5, 1),
 * ln m = 2 atanh(t), t = (m-1)/(m+1) in [-1/3, 0), 20-term odd series */
KG_HD double kg_log(double x) {
  union {
    double d;
    uint64_t u;
  } b;
  b.d = x;
  const int e = (int)((b.u >> 52) & 0x7ff) - 1022;
  b.u = (b.u & 0x800fffffffffffffull) | (0x3feull << 52); /* m in [0.5, 1) */
  const double m = b.d;
  const double t = KG_DIV(KG_SUB(m, 1.0), KG_ADD(m, 1.0));
  const double t2 = KG_MUL(t, t);
  double p = 1.0 / 39.0;
  /* Horner: p = sum_{k=0}^{19} t2^k / (2k+1) */
  const double inv[19] = {1.0 / 37.0, 1.0 / 35.0, 1.0 / 33.0, 1.0 / 31.0, 1.0 / 29.0,
                          1.0 / 27.0, 1.0 / 25.0, 1.0 / 23.0, 1.0 / 21.0, 1.0 / 19.0,
                          1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0, 1.0 / 9.0,
                          1.0 / 7.0,  1.0 / 5.0,  1.0 / 3.0,  1.0};
  for (int k = 0; k < 19; ++k) p = KG_FMA(p, t2, inv[k]);
  const double lnm = KG_MUL(KG_MUL(2.0, t), p);
  return KG_FMA((double)e, 0.69314718055994530942, lnm);
}

/* standard normal #idx of stream (seed, tag): Marsaglia polar method, one
 * Philox block (two uniforms) per attempt, attempt counter in the block */
KG_HD double kg_normal(uint64_t seed, uint32_t tag, uint64_t idx) {
  for (uint32_t a = 0;; ++a) {
    uint32_t w[4];
    kg_philox((uint32_t)idx, (uint32_t)(idx >> 32), a, tag, (uint32_t)seed,
              (uint32_t)(seed >> 32), w);
    const double u = kg_sym_uniform(w[0], w[1]);
    const double v = kg_sym_uniform(w[2], w[3]);
    const double s = KG_FMA(u, u, KG_MUL(v, v));
    if (s > 0.0 && s < 1.0) {
      const double f = KG_SQRT(KG_DIV(KG_MUL(-2.0, kg_log(s)), s));
      return KG_MUL(u, f);
    }
  }
}

/* one entry of the generated matrix, in double (cast to float by the
 * caller for f32 storage) */
KG_HD double kg_entry(const double* ps_row, const double* q_row, int r, double noise,
                      uint64_t seed, uint64_t i, uint64_t j, uint64_t n) {
  double acc = 0.0;
  for (int k = 0; k < r; ++k) acc = KG_FMA(ps_row[k], q_row[k], acc);
  if (noise != 0.0) acc = KG_ADD(acc, KG_MUL(noise, kg_normal(seed, KSVD_GEN_TAG_NOISE, i * n + j)));
  return acc;
}

#endif /* KSVD_GEN_H */
