// gen.cuh -- on-device generation of the BASELINE.json configurations 3-5
// (dense A = P diag(s) Q^T + noise G, P/Q orthonormal), directly into the
// padded row-major layout of a ksvd_mat.  The arithmetic of every entry is
// fixed by include/ksvd_gen.h so the host oracle (oracle/gen_rows.c)
// regenerates bit-identical rows from the same factors.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "ksvd_gen.h"

namespace ksvd {

// X[i*r + k] = N(0,1) #((row0 + i)*r + k) of stream (seed, tag)
__global__ void __launch_bounds__(kThreads)
k_gen_gauss(double* __restrict__ X, int64_t rows, int r, uint64_t seed, uint32_t tag,
            int64_t row0) {
  const int64_t total = rows * r;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t i = e / r, k = e % r;
    X[e] = kg_normal(seed, tag, (uint64_t)(row0 + i) * (uint64_t)r + (uint64_t)k);
  }
}

// Tiled f64 product C = X Y (Y given transposed when TRANS: Y[j*ldy + k]).
// Per output the sum runs k = 0..K-1 as one fma chain from +0.0 (the order
// kg_entry uses).  CTA tile 64 x 64, K slabs of 16, 4 x 4 outputs per thread.
// MODE 0: plain store to C (f64, ldc).  MODE 1/2: generator epilogue
// + noise * g(seed, (row0+i)*nglob + j), stored as f64 / f32 into A (ldc).
constexpr int kGT = 64, kGK = 16;
template <bool TRANS, int MODE>
__global__ void __launch_bounds__(kThreads)
k_gen_gemm(int64_t L, int64_t N, int K, const double* __restrict__ X, int64_t ldx,
           const double* __restrict__ Y, int64_t ldy, void* __restrict__ C, int64_t ldc,
           double noise, uint64_t seed, int64_t row0, int64_t nglob) {
  __shared__ double Xs[kGT][kGK + 1];
  __shared__ double Ys[kGK][kGT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = (int64_t)blockIdx.y * kGT, j0 = (int64_t)blockIdx.x * kGT;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kGK) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGT * kGK; e += kThreads) {
      const int ii = e / kGK, kk = e % kGK;
      const int64_t i = i0 + ii;
      const int k = k0 + kk;
      Xs[ii][kk] = (i < L && k < K) ? X[i * ldx + k] : 0.0;
    }
    for (int e = threadIdx.x; e < kGT * kGK; e += kThreads) {
      int jj, kk;
      if (TRANS) {
        jj = e / kGK;
        kk = e % kGK;
      } else {
        kk = e / kGT;
        jj = e % kGT;
      }
      const int64_t j = j0 + jj;
      const int k = k0 + kk;
      double v = 0.0;
      if (j < N && k < K) v = TRANS ? Y[j * ldy + k] : Y[(int64_t)k * ldy + j];
      Ys[kk][jj] = v;
    }
    __syncthreads();
    const int kend = min(kGK, K - k0);
    for (int kk = 0; kk < kend; ++kk) {
      double xa[4], yb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xa[a] = Xs[ty * 4 + a][kk];
#pragma unroll
      for (int b = 0; b < 4; ++b) yb[b] = Ys[kk][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = __fma_rn(xa[a], yb[b], acc[a][b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t i = i0 + ty * 4 + a;
    if (i >= L) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t j = j0 + tx * 4 + b;
      if (j >= N) continue;
      double v = acc[a][b];
      if (MODE == 0) {
        static_cast<double*>(C)[i * ldc + j] = v;
      } else {
        if (noise != 0.0)
          v = KG_ADD(v, KG_MUL(noise, kg_normal(seed, KSVD_GEN_TAG_NOISE,
                                                (uint64_t)(row0 + i) * (uint64_t)nglob +
                                                    (uint64_t)j)));
        if (MODE == 1)
          static_cast<double*>(C)[i * ldc + j] = v;
        else
          static_cast<float*>(C)[i * ldc + j] = (float)v;
      }
    }
  }
}

// Gram partials of X (rows x r, row-major): part[s][a][b] = sum over the rows
// of split s of X[i][a] X[i][b]; 32 x 32 output tiles, fixed row order.
constexpr int kGramT = 32;
__global__ void __launch_bounds__(kThreads)
k_gram_part(const double* __restrict__ X, int64_t rows, int r, int64_t rows_per_split,
            double* __restrict__ part) {
  __shared__ double Xa[kGramT][kGramT + 1];
  __shared__ double Xb[kGramT][kGramT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 2 x 2 outputs each
  const int a0 = blockIdx.y * kGramT, b0 = blockIdx.x * kGramT;
  const int64_t s = blockIdx.z;
  const int64_t r0 = s * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t i0 = r0; i0 < r1; i0 += kGramT) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGramT * kGramT; e += kThreads) {
      const int ii = e / kGramT, cc = e % kGramT;
      const int64_t i = i0 + ii;
      Xa[ii][cc] = (i < r1 && a0 + cc < r) ? X[i * r + a0 + cc] : 0.0;
      Xb[ii][cc] = (i < r1 && b0 + cc < r) ? X[i * r + b0 + cc] : 0.0;
    }
    __syncthreads();
    for (int ii = 0; ii < kGramT; ++ii) {
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
          acc[a][b] = fma(Xa[ii][ty * 2 + a], Xb[ii][tx * 2 + b], acc[a][b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int ga = a0 + ty * 2 + a, gb = b0 + tx * 2 + b;
      if (ga < r && gb < r) part[(s * r + ga) * r + gb] = acc[a][b];
    }
}

// G[a][b] = sum_s part[s][a][b] (fixed order)
__global__ void __launch_bounds__(kThreads)
k_gram_reduce(const double* __restrict__ part, int nsplit, int r, double* __restrict__ G) {
  const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t rr = (int64_t)r * r;
  if (e >= rr) return;
  double s = 0.0;
  for (int k = 0; k < nsplit; ++k) s += part[k * rr + e];
  G[e] = s;
}

// Ps[i][k] = P[i][k] * s[k]
__global__ void __launch_bounds__(kThreads)
k_scale_cols(double* __restrict__ P, int64_t rows, int r, const double* __restrict__ s) {
  const int64_t total = rows * r;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * kThreads)
    P[e] = KG_MUL(P[e], s[e % r]);
}

}  // namespace ksvd
