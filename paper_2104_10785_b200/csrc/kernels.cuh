// kernels.cuh -- sm_100a kernels of the GK bidiagonalization hot path.
//
// Every kernel is deterministic: reductions run in a fixed order (per-lane
// sequential, then a fixed xor-butterfly, then a fixed walk over warps /
// blocks); there are no floating-point atomics.  Identical inputs therefore
// reproduce bit-identical alphas/betas/bases, matching the reference's
// determinism contract (test_bidiag.py:159-174, test_fsvd.py:181-187).
//
// Device state (status word) makes every kernel of a GK step a no-op once a
// breakdown / non-finite value has been recorded, so the host can enqueue
// several steps ahead without synchronising (bidiag.py:151-178 loop).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ksvd {

constexpr int kThreads = 256;  // 8 warps per CTA for every streaming kernel
constexpr int kWarps = kThreads / 32;

enum Status : int {
  ST_RUNNING = 0,
  ST_BETA_BREAK = 1,   // bidiag.py:158
  ST_ALPHA_BREAK = 2,  // bidiag.py:174
  ST_DEGENERATE = 3,   // bidiag.py:142
  ST_NONFINITE = 4,    // bidiag.py:90-92 (_assert_finite)
  ST_CUT = 5,          // fsvd.py:152 (dependent column in the U filter)
};

struct DevState {
  int status;     // halting status (set only from globally reduced values)
  int kprime;
  int where;      // step (or column) that set the status
  int nonfinite;  // local non-finite flag (bidiag.py:90-92), non-halting:
                  // it is reduced across ranks with the next norm and
                  // turned into ST_NONFINITE by k_norm_test, so every rank
                  // halts at the same step and issues the same collectives
};

__device__ __forceinline__ bool halted(const DevState* st) {
  return *reinterpret_cast<const volatile int*>(&st->status) != ST_RUNNING;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// 16-byte streaming loads of A.  A is read exactly once per pass, so it is
// loaded through the non-coherent path without L1 allocation.
template <typename T>
struct AVec;
template <>
struct AVec<double> {
  static constexpr int V = 2;
  double v[2];
  __device__ __forceinline__ void load(const double* p) {
    asm("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];"
        : "=d"(v[0]), "=d"(v[1])
        : "l"(p));
  }
  __device__ __forceinline__ double get(int k) const { return v[k]; }
};
template <>
struct AVec<float> {
  static constexpr int V = 4;
  float v[4];
  __device__ __forceinline__ void load(const float* p) {
    asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
        : "l"(p));
  }
  __device__ __forceinline__ double get(int k) const { return (double)v[k]; }
};

__device__ __forceinline__ void flag_nonfinite(DevState* st, double v, int step) {
  if (!isfinite(v)) st->nonfinite = 1;  // same value from every writer
}

// ---------------------------------------------------------------------------
// gemv_n:  w = A p - alpha q_prev          (bidiag.py:152, linops.py:161)
//
// Grid (blocks_per_chunk, nchunks).  Chunk y owns columns
// [y*chunk_vecs*V, ...); its slice of p (optionally p = p_src / *p_scale,
// the deferred normalisation P[:, i-1] = z / alpha, bidiag.py:177) is staged
// in shared memory once per CTA and reused for every row the CTA streams.
// Each warp owns R consecutive rows at a time; lanes stride the row with
// 16-byte loads, U loads in flight per row.  nchunks == 1 writes w with the
// fused -alpha*q epilogue; otherwise per-chunk partial row sums go to
// `out` (chunk-major) and k_gemv_n_finalize adds them in chunk order.
template <typename TA, int R, int U>
__global__ void __launch_bounds__(kThreads)
k_gemv_n(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t nvec,
         int chunk_vecs, const double* __restrict__ p_src,
         const double* __restrict__ p_scale, double* __restrict__ p_dst,
         int64_t n_true, double* __restrict__ out, int64_t out_ld,
         const double* __restrict__ qprev, const double* __restrict__ alpha,
         DevState* st, int step, int64_t groups_per_warp) {
  if (halted(st)) return;
  constexpr int V = AVec<TA>::V;
  extern __shared__ double p_s[];
  const int chunk = blockIdx.y;
  const int64_t v0 = (int64_t)chunk * chunk_vecs;
  const int nv = (int)min((int64_t)chunk_vecs, nvec - v0);
  const int64_t c0 = v0 * V;
  const double scale = p_scale ? *p_scale : 1.0;
  for (int e = threadIdx.x; e < nv * V; e += kThreads) {
    const int64_t col = c0 + e;
    double pv = col < n_true ? p_src[col] : 0.0;
    if (p_scale) {
      pv = pv / scale;
      if (blockIdx.x == 0 && p_dst && col < n_true) p_dst[col] = pv;
    }
    p_s[e] = pv;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t ngroups = (m + R - 1) / R;
  const double a_ = alpha ? *alpha : 0.0;
  const int64_t g_begin = gwarp * groups_per_warp;
  const int64_t g_end = min(ngroups, g_begin + groups_per_warp);
  for (int64_t g = g_begin; g < g_end; ++g) {
    const int64_t r0 = g * R;
    const TA* rowp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rowp[r] = A + min(r0 + r, m - 1) * lda + c0;
    double acc[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k) acc[r][k] = 0.0;
    int v = lane;
    for (; v + (U - 1) * 32 < nv; v += U * 32) {
      AVec<TA> a[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) a[u][r].load(rowp[r] + (int64_t)(v + u * 32) * V);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double* pp = p_s + (v + u * 32) * V;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const double pk = pp[k];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r][k] = fma(a[u][r].get(k), pk, acc[r][k]);
        }
      }
    }
    for (; v < nv; v += 32) {
      AVec<TA> a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r].load(rowp[r] + (int64_t)v * V);
      const double* pp = p_s + v * V;
#pragma unroll
      for (int k = 0; k < V; ++k)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][k] = fma(a[r].get(k), pp[k], acc[r][k]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double s = acc[r][0];
#pragma unroll
      for (int k = 1; k < V; ++k) s += acc[r][k];
      s = warp_sum(s);
      if (lane == r && r0 + r < m) {
        if (out_ld == 0) {  // direct epilogue
          const double w = qprev ? s - a_ * qprev[r0 + r] : s;
          out[r0 + r] = w;
          flag_nonfinite(st, w, step);
        } else {
          out[(int64_t)chunk * out_ld + r0 + r] = s;
        }
      }
    }
  }
}

// w[r] = sum_chunks part[c][r] - alpha q[r]  (chunk order fixed)
__global__ void __launch_bounds__(kThreads)
k_gemv_n_finalize(const double* __restrict__ part, int64_t part_ld, int nchunks,
                  int64_t m, const double* __restrict__ qprev,
                  const double* __restrict__ alpha, double* __restrict__ w,
                  DevState* st, int step) {
  if (halted(st)) return;
  const int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (r >= m) return;
  double s = part[r];
  for (int c = 1; c < nchunks; ++c) s += part[(int64_t)c * part_ld + r];
  if (qprev) s = s - (*alpha) * qprev[r];
  w[r] = s;
  flag_nonfinite(st, s, step);
}

// ---------------------------------------------------------------------------
// gemv_t:  partial z = A^T q over a row split  (bidiag.py:169, linops.py:164)
//
// Column reduction of row-major A without a transposed copy.  Grid
// (ncoltiles, nsplit).  Each thread owns one 16-byte column vector
// (V columns) of a 256-vector tile and accumulates V f64 sums down the
// rows of its split, U rows in flight.  q for the split is staged through
// shared memory in blocks of kQB rows (optionally q = q_src / *q_scale: the
// deferred normalisation q_{i+1} = w / beta, bidiag.py:165, written to
// q_dst by tile-0 CTAs).  Partials of split s go to part[s*ldz + col];
// k_gemv_t_finalize adds the splits in order.
constexpr int kQB = 1024;
template <typename TA, int U>
__global__ void __launch_bounds__(kThreads)
k_gemv_t(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t nvec,
         int64_t rows_per_split, const double* __restrict__ q_src,
         const double* __restrict__ q_scale, double* __restrict__ q_dst,
         double* __restrict__ part, int64_t ldz, const DevState* st) {
  if (halted(st)) return;
  constexpr int V = AVec<TA>::V;
  __shared__ double q_s[kQB];
  const int64_t vcol = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const bool active = vcol < nvec;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(m, r0 + rows_per_split);
  const double scale = q_scale ? *q_scale : 1.0;
  double acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.0;
  const TA* base = A + vcol * V;
  for (int64_t rb = r0; rb < r1; rb += kQB) {
    const int nr = (int)min((int64_t)kQB, r1 - rb);
    __syncthreads();
    for (int e = threadIdx.x; e < nr; e += kThreads) {
      double qv = q_src[rb + e];
      if (q_scale) {
        qv = qv / scale;
        if (blockIdx.x == 0 && q_dst) q_dst[rb + e] = qv;
      }
      q_s[e] = qv;
    }
    __syncthreads();
    if (!active) continue;
    const TA* p = base + rb * lda;
    int r = 0;
    for (; r + U <= nr; r += U) {
      AVec<TA> a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u].load(p + (int64_t)(r + u) * lda);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double qv = q_s[r + u];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = fma(a[u].get(k), qv, acc[k]);
      }
    }
    for (; r < nr; ++r) {
      AVec<TA> a;
      a.load(p + (int64_t)r * lda);
      const double qv = q_s[r];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fma(a.get(k), qv, acc[k]);
    }
  }
  if (active) {
    double* dst = part + (int64_t)blockIdx.y * ldz + vcol * V;
#pragma unroll
    for (int k = 0; k < V; ++k) dst[k] = acc[k];
  }
}

// z[j] = sum_s part[s][j] (- beta p[j]);  zero in the padding [n, n_pad)
__global__ void __launch_bounds__(kThreads)
k_gemv_t_finalize(const double* __restrict__ part, int64_t ldz, int nsplit,
                  int64_t n, int64_t n_pad, const double* __restrict__ beta,
                  const double* __restrict__ pprev, double* __restrict__ z,
                  DevState* st, int step, int check) {
  if (halted(st)) return;
  const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (j >= n_pad) return;
  if (j >= n) {
    z[j] = 0.0;
    return;
  }
  double s = part[j];
  for (int k = 1; k < nsplit; ++k) s += part[(int64_t)k * ldz + j];
  if (pprev) s = s - (*beta) * pprev[j];
  z[j] = s;
  if (check) flag_nonfinite(st, s, step);
}

// z -= beta p  (multi-rank: applied after the all-reduce of A^T q)
__global__ void __launch_bounds__(kThreads)
k_axpy_check(double* __restrict__ z, const double* __restrict__ beta,
             const double* __restrict__ pprev, int64_t n, DevState* st, int step) {
  if (halted(st)) return;
  const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (j >= n) return;
  double s = z[j];
  if (pprev) s = s - (*beta) * pprev[j];
  z[j] = s;
  flag_nonfinite(st, s, step);
}

// ---------------------------------------------------------------------------
// CGS2 (bidiag.py:154-155, 171-172):  c = B^T x ; x -= B c ; (twice)
// B is a basis of `ncols` columns, each contiguous (ldb doubles apart).
// A CTA owns 256*E consecutive rows; the partial dot of column j over row
// block b lands in part[j*nrb + b] and k_reduce_cols adds the blocks.
constexpr int kJ = 8;  // basis columns per CTA in the dot kernel

template <int E>
__global__ void __launch_bounds__(kThreads)
k_cgs_dot(const double* __restrict__ B, int64_t ldb, int ncols,
          const double* __restrict__ x, int64_t L, double* __restrict__ part,
          int nrb, const DevState* st) {
  if (halted(st)) return;
  __shared__ double red[kWarps][kJ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rbase = (int64_t)blockIdx.x * (kThreads * E) + tid;
  double xr[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t r = rbase + e * kThreads;
    xr[e] = r < L ? x[r] : 0.0;
  }
  const int j0 = blockIdx.y * kJ;
  double s[kJ];
#pragma unroll
  for (int jj = 0; jj < kJ; ++jj) {
    s[jj] = 0.0;
    if (j0 + jj < ncols) {
      const double* col = B + (int64_t)(j0 + jj) * ldb;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int64_t r = rbase + e * kThreads;
        if (r < L) s[jj] = fma(col[r], xr[e], s[jj]);
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < kJ; ++jj) s[jj] = warp_sum(s[jj]);
  if (lane == 0) {
#pragma unroll
    for (int jj = 0; jj < kJ; ++jj) red[warp][jj] = s[jj];
  }
  __syncthreads();
  if (tid < kJ && j0 + tid < ncols) {
    double t = red[0][tid];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) t += red[w][tid];
    part[(int64_t)(j0 + tid) * nrb + blockIdx.x] = t;
  }
}

// x -= B c, then (mode 1) partial dots of the updated x against B for the
// next CGS pass, or (mode 2) the partial ||x||^2, or (mode 0) nothing.
constexpr int kCChunk = 1024;
template <int E>
__global__ void __launch_bounds__(kThreads)
k_cgs_update(const double* __restrict__ B, int64_t ldb, int ncols,
             const double* __restrict__ c, double* __restrict__ x, int64_t L,
             int mode, double* __restrict__ part, int nrb, const DevState* st) {
  if (halted(st)) return;
  __shared__ double cs[kCChunk];
  __shared__ double red[kWarps][kJ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rbase = (int64_t)blockIdx.x * (kThreads * E) + tid;
  double xr[E], t[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t r = rbase + e * kThreads;
    xr[e] = r < L ? x[r] : 0.0;
    t[e] = 0.0;
  }
  for (int j0 = 0; j0 < ncols; j0 += kCChunk) {
    const int nc = min(kCChunk, ncols - j0);
    __syncthreads();
    for (int e = tid; e < nc; e += kThreads) cs[e] = c[j0 + e];
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < nc; ++jj) {
      const double cj = cs[jj];
      const double* col = B + (int64_t)(j0 + jj) * ldb;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int64_t r = rbase + e * kThreads;
        if (r < L) t[e] = fma(col[r], cj, t[e]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t r = rbase + e * kThreads;
    xr[e] = xr[e] - t[e];
    if (r < L) x[r] = xr[e];
  }
  if (mode == 2) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) s = fma(xr[e], xr[e], s);
    s = warp_sum(s);
    if (lane == 0) red[warp][0] = s;
    __syncthreads();
    if (tid == 0) {
      double tt = red[0][0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) tt += red[w][0];
      part[blockIdx.x] = tt;
    }
  } else if (mode == 1) {
    for (int j0 = 0; j0 < ncols; j0 += kJ) {
      double s[kJ];
#pragma unroll
      for (int jj = 0; jj < kJ; ++jj) {
        s[jj] = 0.0;
        if (j0 + jj < ncols) {
          const double* col = B + (int64_t)(j0 + jj) * ldb;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int64_t r = rbase + e * kThreads;
            if (r < L) s[jj] = fma(col[r], xr[e], s[jj]);
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < kJ; ++jj) s[jj] = warp_sum(s[jj]);
      __syncthreads();
      if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < kJ; ++jj) red[warp][jj] = s[jj];
      }
      __syncthreads();
      if (tid < kJ && j0 + tid < ncols) {
        double tt = red[0][tid];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) tt += red[w][tid];
        part[(int64_t)(j0 + tid) * nrb + blockIdx.x] = tt;
      }
    }
  }
}

// ||x||^2 partials (pass-less norm, used when the basis is empty)
template <int E>
__global__ void __launch_bounds__(kThreads)
k_sumsq(const double* __restrict__ x, int64_t L, double* __restrict__ part,
        const DevState* st) {
  if (halted(st)) return;
  __shared__ double red[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rbase = (int64_t)blockIdx.x * (kThreads * E) + tid;
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t r = rbase + e * kThreads;
    const double v = r < L ? x[r] : 0.0;
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double t = red[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// out[j] = sum_b part[j*nrb + b], one warp per column, fixed order
__global__ void __launch_bounds__(kThreads)
k_reduce_cols(const double* __restrict__ part, int nrb, int ncols,
              double* __restrict__ out, const DevState* st) {
  if (halted(st)) return;
  const int j = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= ncols) return;
  const double* p = part + (int64_t)j * nrb;
  double s = 0.0;
  for (int b = lane; b < nrb; b += 32) s += p[b];
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// Norm test (bidiag.py:156-158, 173-174; fsvd.py:151-152).
// nrb > 0: s = sum part[0..nrb) and the local non-finite flag (single rank).
// nrb == 0: s = red[0], flag = red[1] (already all-reduced by the caller).
// nrm = sqrt(s) -> *slot; non-finite -> ST_NONFINITE; nrm < eps -> `code`.
__global__ void k_norm_test(const double* __restrict__ part, int nrb,
                            const double* __restrict__ red, double eps,
                            double* __restrict__ slot, DevState* st, int step,
                            int code) {
  if (halted(st)) return;
  const int lane = threadIdx.x;
  double s = 0.0, flag = 0.0;
  if (nrb > 0) {
    for (int b = lane; b < nrb; b += 32) s += part[b];
    s = warp_sum(s);
    flag = st->nonfinite ? 1.0 : 0.0;
  } else {
    s = red[0];
    flag = red[1];
  }
  if (lane == 0) {
    const double nrm = sqrt(s);
    *slot = nrm;
    if (flag != 0.0 || !isfinite(nrm)) {
      st->status = ST_NONFINITE;
      st->kprime = step;
      st->where = step;
    } else if (nrm < eps) {
      st->status = code;
      st->kprime = step;
      st->where = step;
    }
  }
}

// red[0] = sum part[0..nrb), red[1] = local non-finite flag (pre all-reduce)
__global__ void k_norm_prep(const double* __restrict__ part, int nrb,
                            double* __restrict__ red, const DevState* st) {
  if (halted(st)) return;
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nrb; b += 32) s += part[b];
  s = warp_sum(s);
  if (lane == 0) {
    red[0] = s;
    red[1] = st->nonfinite ? 1.0 : 0.0;
  }
}

// dst = src / val (host scalar; terminal column, bidiag.py:101)
__global__ void __launch_bounds__(kThreads)
k_scale_val(const double* __restrict__ src, double val, double* __restrict__ dst,
            int64_t L, const DevState* st) {
  if (halted(st)) return;
  const int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (r >= L) return;
  dst[r] = src[r] / val;
}

// dst = src / *scale
__global__ void __launch_bounds__(kThreads)
k_scale(const double* __restrict__ src, const double* __restrict__ scale,
        double* __restrict__ dst, int64_t L, const DevState* st) {
  if (halted(st)) return;
  const int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (r >= L) return;
  dst[r] = src[r] / (*scale);
}

// ---------------------------------------------------------------------------
// Ritz assembly (fsvd.py:191-194)

// V[:, t] = sum_j G[j + t*kp] P[:, j]   (P: n rows, ldp; V: ldv)
constexpr int kTT = 8;
__global__ void __launch_bounds__(kThreads)
k_basis_combine(const double* __restrict__ P, int64_t ldp, int64_t n, int kp,
                const double* __restrict__ G, int take, double* __restrict__ V,
                int64_t ldv) {
  const int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int t0 = blockIdx.y * kTT;
  if (r >= n) return;
  double acc[kTT];
#pragma unroll
  for (int tt = 0; tt < kTT; ++tt) acc[tt] = 0.0;
  for (int j = 0; j < kp; ++j) {
    const double pj = P[(int64_t)j * ldp + r];
#pragma unroll
    for (int tt = 0; tt < kTT; ++tt)
      if (t0 + tt < take) acc[tt] = fma(pj, __ldg(G + j + (int64_t)(t0 + tt) * kp), acc[tt]);
  }
#pragma unroll
  for (int tt = 0; tt < kTT; ++tt)
    if (t0 + tt < take) V[(int64_t)(t0 + tt) * ldv + r] = acc[tt];
}

// Y[:, t] = (A X[:, t]) / sigma[t] for a block of up to 32 right-hand sides:
// one pass over A for all of them (the reference runs `take` separate
// matvecs, fsvd.py:193-194).  CTA tile: kMR rows x 32 columns; lane = column,
// each warp owns kMR/8 rows; A and X are staged through shared memory in
// kKC-column slabs.
constexpr int kMR = 64;
constexpr int kKC = 32;
template <typename TA>
__global__ void __launch_bounds__(kThreads)
k_multi_rhs(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t n,
            const double* __restrict__ X, int64_t ldx, int ncols,
            const double* __restrict__ sigma, double* __restrict__ Y,
            int64_t ldy) {
  __shared__ double As[kMR][kKC + 1];
  __shared__ double Xs[kKC][33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kMR;
  const int t0 = blockIdx.y * 32;
  constexpr int RW = kMR / kWarps;  // rows per warp
  double acc[RW];
#pragma unroll
  for (int i = 0; i < RW; ++i) acc[i] = 0.0;
  for (int64_t k0 = 0; k0 < n; k0 += kKC) {
    __syncthreads();
    for (int e = tid; e < kMR * kKC; e += kThreads) {
      const int rr = e / kKC, kk = e % kKC;
      const int64_t r = r0 + rr, k = k0 + kk;
      As[rr][kk] = (r < m && k < n) ? (double)A[r * lda + k] : 0.0;
    }
    for (int e = tid; e < kKC * 32; e += kThreads) {
      const int kk = e % kKC, tt = e / kKC;
      const int64_t k = k0 + kk;
      Xs[kk][tt] = (k < n && t0 + tt < ncols) ? X[(int64_t)(t0 + tt) * ldx + k] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kKC; ++kk) {
      const double xv = Xs[kk][lane];
#pragma unroll
      for (int i = 0; i < RW; ++i) acc[i] = fma(As[warp * RW + i][kk], xv, acc[i]);
    }
  }
  const int t = t0 + lane;
  if (t < ncols) {
    const double s = sigma ? sigma[t] : 1.0;
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const int64_t r = r0 + warp * RW + i;
      if (r < m) Y[(int64_t)t * ldy + r] = sigma ? acc[i] / s : acc[i];
    }
  }
}

// fix_signs (linops.py:271-282): per column j, s = sign(V[argmax|V[:,j]|, j])
// with numpy's first-index tie rule and sign 0 -> +1; U[:,j], V[:,j] *= s.
__global__ void __launch_bounds__(kThreads)
k_fix_signs(double* __restrict__ V, int64_t ldv, int64_t n,
            double* __restrict__ U, int64_t ldu, int64_t mloc) {
  __shared__ double bv[kThreads];
  __shared__ int64_t bi[kThreads];
  __shared__ double sgn;
  const int j = blockIdx.x, tid = threadIdx.x;
  double* v = V + (int64_t)j * ldv;
  double best = -1.0;
  int64_t besti = INT64_MAX;
  for (int64_t i = tid; i < n; i += kThreads) {
    const double a = fabs(v[i]);
    if (a > best) {  // strict: keeps the first index per thread
      best = a;
      besti = i;
    }
  }
  bv[tid] = best;
  bi[tid] = besti;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double o = bv[tid + s];
      const int64_t oi = bi[tid + s];
      if (o > bv[tid] || (o == bv[tid] && oi < bi[tid])) {
        bv[tid] = o;
        bi[tid] = oi;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    const double pk = bi[0] < n ? v[bi[0]] : 0.0;
    sgn = pk < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  const double s = sgn;
  for (int64_t i = tid; i < n; i += kThreads) v[i] *= s;
  double* u = U + (int64_t)j * ldu;
  for (int64_t i = tid; i < mloc; i += kThreads) u[i] *= s;
}

}  // namespace ksvd
