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
#include <cooperative_groups.h>
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

// Progress word in mapped (zero-copy) host memory, written by the norm tests
// of the GK loop: prog = 2*step + side (side 0: beta test, 1: alpha test);
// a breakdown also records status and halt_step.  The host paces its
// run-ahead on it instead of per-step device->host copies.
struct HostProg {
  int prog;
  int halt_step;
  int status;
  int pad;
};

// publish a breakdown to the host (plain stores to mapped memory, visible
// once the kernel has completed; the host reads them after its pacing event)
__device__ __forceinline__ void host_progress(HostProg* hp, int stop, int step, int side) {
  (void)side;
  if (!hp || stop == 0) return;
  volatile HostProg* h = hp;
  h->status = stop;
  h->halt_step = step;
}

// Programmatic dependent launch (ksvd.cu launch_step): wait for the
// preceding grid's completion + memory flush / let the next grid launch.
// Every CTA of a kernel launched with the attribute calls pdl_wait() before
// reading its predecessor's outputs and before exiting.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// bit 1: the gemv kernels trigger their dependents early (right after their
// own wait); bit 2 (CGS kernels) stays implicit at CTA exit -- measured, an
// early CGS trigger parks the next gemv's CTAs beside the grid-synchronised
// CGS kernel and costs ~5% on config 2.
__device__ __forceinline__ void pdl_trigger(int bit) {
  if (bit & 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ bool halted(const DevState* st) {
  return *reinterpret_cast<const volatile int*>(&st->status) != ST_RUNNING;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum 8 per-lane values across the warp at once ("transpose" butterfly:
// 9 shuffles instead of 8 x 5).  On return lane l holds the total of value
// index ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1); lanes with (l & 3) == 0
// own distinct indices.  The combination order is fixed (deterministic).
__device__ __forceinline__ double warp_sum8(double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double send = b4 ? v[k] : v[k + 4];
    const double keep = b4 ? v[k + 4] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double send = b3 ? v[k] : v[k + 2];
    const double keep = b3 ? v[k + 2] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const double send = b2 ? v[0] : v[1];
    const double keep = b2 ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  double t = v[0];
  t += __shfl_xor_sync(0xffffffffu, t, 2);
  t += __shfl_xor_sync(0xffffffffu, t, 1);
  return t;
}
__device__ __forceinline__ int warp_sum8_index(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// sum_{k < cnt} p[k*ld] with up to 16 loads in flight (predicated, so a
// whole batch is one L2 round trip) and 4 interleaved partial sums combined
// in a fixed order (deterministic; not latency-chained).  The finalisation
// of k_gemv_n's chunk-group partials is one or two round trips.
__device__ __forceinline__ double strided_sum(const double* __restrict__ p, int64_t ld,
                                              int cnt) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < cnt; k += 32) {  // acc[i & 3] += p[i] in ascending i
    double t[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) t[u] = k + u < cnt ? __ldcg(p + (int64_t)(k + u) * ld) : 0.0;
#pragma unroll
    for (int u = 0; u < 32; ++u) acc[u & 3] += t[u];
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// strided_sum with 8 loads in flight (the same fixed order, so the same
// bits): for kernels that cannot spare strided_sum's registers
__device__ __forceinline__ double strided_sum8(const double* __restrict__ p, int64_t ld,
                                               int cnt) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < cnt; k += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = k + u < cnt ? __ldcg(p + (int64_t)(k + u) * ld) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u & 3] += t[u];
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
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
  // with an L2 cache policy (a_policy)
  __device__ __forceinline__ void load(const double* p, uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v2.f64 {%0,%1}, [%2], %3;"
        : "=d"(v[0]), "=d"(v[1])
        : "l"(p), "l"(pol));
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
  __device__ __forceinline__ void load(const float* p, uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
        : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ double get(int k) const { return (double)v[k]; }
};

// L2 policy of the A-streaming loads (k_gemv_n, k_gemv_t2): evict_first
// (ef) keeps A's lines from displacing the small, reused data (basis tiles,
// partial sums); ksvd.cu chooses it for A far larger than L2, where the
// hand-over of A's last rows from one pass to the next is negligible.
__device__ __forceinline__ uint64_t a_policy(int ef) {
  uint64_t pol;
  if (ef)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void flag_nonfinite(DevState* st, double v, int step) {
  if (!isfinite(v)) st->nonfinite = 1;  // same value from every writer
}

// ---------------------------------------------------------------------------
template <bool CG>
__device__ __forceinline__ double ldv(const double* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}

// gemv_n (k_gemv_n): w = A p   (bidiag.py:152)
//
// Each warp owns one column chunk of 32*U 16-byte vectors; its slice of p
// (p = p_src / *p_scale, the deferred normalisation of P[:, i-1], written
// back to p_dst by the first row segment) is loaded once into registers.
// The 8 warps of a CTA take 8 consecutive chunks of the SAME rows: a CTA
// streams 8 rows x 8 chunks per iteration (8*U independent 16-byte loads per
// lane in flight), each warp reduces its 8 row partials across the warp with
// one 9-shuffle transpose butterfly (warp_sum8), and the 8 warps' partials
// are summed in shared memory in warp order and written once per (chunk
// group, row).  Measured on B200 (tools/gemv_bench.cu): 7.11 TB/s on a 40 GB
// f32 matrix and 7.31 TB/s on 32 GB f64, against 6.65 / 6.87 for the same
// loads with one partial store per warp and no CTA-level sum (the earlier
// k_gemv_n2) -- at the rate of the column-reduction kernel k_gemv_t2.
// CTA b: chunk group b % ngroups, row segment b / ngroups of nseg (rows
// rseg*8 + k*nseg*8: all CTAs move down the matrix as one band, so the rows
// read last stay in L2 for k_gemv_t2, which sweeps up).  Partials go to
// part[group * m + row]; k_gemv_n_finalize (or the CGS2 kernels' fused
// finalisation) adds them in group order and applies - alpha q.
// FIN (the paired step, pair.cuh): the last CTA of each row segment to
// finish (an arrival counter per segment, reset by that CTA) adds the
// segment's chunk-group partials in group order and writes
// w = A p - (*nalpha) qprev -- k_gemv_n_finalize's arithmetic, in the
// product's tail instead of a launch of its own.
struct GemvNFin {
  unsigned* seg_cnt;  // nseg zero-initialised counters
  const double* qprev;
  const double* nalpha;
  double* w;
};

// NB: the CTA-level row sums with named barriers instead of one
// __syncthreads per 8-row block: warps 1-7 arrive (bar.arrive) on FULL[par]
// after storing their partials and only wait (EMPTY[par]) if they get two
// blocks ahead of warp 0, which syncs on FULL[par], sums and stores, then
// releases EMPTY[par].  Keeps the other warps issuing loads while warp 0
// reduces.
__device__ __forceinline__ void nbar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kThreads) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kThreads) : "memory");
}

template <typename TA, int U, bool FIN, bool NB = false>
__global__ void __launch_bounds__(kThreads)
k_gemv_n(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t nvec, int nchunks,
          int ngroups, int64_t nseg, const double* __restrict__ p_src,
          const double* __restrict__ p_scale, double* __restrict__ p_dst, int64_t n_true,
          double* __restrict__ part, const DevState* st, GemvNFin fin, int a_ef) {
  pdl_wait();
  pdl_trigger(1);
  if (halted(st)) return;
  constexpr int V = AVec<TA>::V;
  constexpr int CW = 32 * U;
  __shared__ double red[2][kWarps][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = (int)(blockIdx.x % ngroups);
  const int64_t rseg = blockIdx.x / ngroups;
  if (rseg >= nseg) return;
  const int chunk = grp * kWarps + warp;
  const double scale = p_scale ? *p_scale : 1.0;
  double pv[U][V];
  bool live[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t vi = (int64_t)chunk * CW + u * 32 + lane;
    live[u] = chunk < nchunks && vi < nvec;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t col = vi * V + k;
      double x = (live[u] && col < n_true) ? p_src[col] : 0.0;
      if (p_scale) {
        x = x / scale;
        if (rseg == 0 && p_dst && live[u] && col < n_true) p_dst[col] = x;
      }
      pv[u][k] = x;
    }
  }
  const TA* base = A + ((int64_t)chunk * CW + lane) * V;
  const uint64_t pol = a_policy(a_ef);
  int par = 0;
  const int64_t niter = rseg * 8 < m ? (m - rseg * 8 + nseg * 8 - 1) / (nseg * 8) : 0;
  int64_t it = 0;
  for (int64_t r = rseg * 8; r < m; r += nseg * 8, par ^= 1, ++it) {
    AVec<TA> a[8][U];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int64_t row = min(r + rr, m - 1);  // clamp: duplicate rows are discarded
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u]) a[rr][u].load(base + row * lda + u * 32 * V, pol);
    }
    double v[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u]) {
#pragma unroll
          for (int k = 0; k < V; ++k) s = fma(a[rr][u].get(k), pv[u][k], s);
        }
      v[rr] = s;
    }
    const double t = warp_sum8(v);
    if constexpr (NB) {
      if (warp != 0 && it >= 2) nbar_sync(3 + par);  // EMPTY[par]: block it-2 consumed
      if ((lane & 3) == 0) red[par][warp][warp_sum8_index(lane)] = t;
      if (warp == 0) {
        nbar_sync(1 + par);  // FULL[par]
        if (lane < 8) {
          double sum = red[par][0][lane];
#pragma unroll
          for (int w = 1; w < kWarps; ++w) sum += red[par][w][lane];
          const int64_t row = r + lane;
          if (row < m) part[(int64_t)grp * m + row] = sum;
        }
        __syncwarp();
        if (it + 2 < niter) nbar_arrive(3 + par);
      } else {
        nbar_arrive(1 + par);
      }
    } else {
      if ((lane & 3) == 0) red[par][warp][warp_sum8_index(lane)] = t;
      __syncthreads();  // red[par] complete; red[par ^ 1] free again (read last round)
      if (warp == 0 && lane < 8) {
        double sum = red[par][0][lane];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) sum += red[par][w][lane];
        const int64_t row = r + lane;
        if (row < m) part[(int64_t)grp * m + row] = sum;
      }
    }
  }
  if constexpr (FIN) {
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(fin.seg_cnt + rseg, 1u) == (unsigned)ngroups - 1;
      if (last) {
        fin.seg_cnt[rseg] = 0;  // ready for the next launch
        __threadfence();
      }
    }
    __syncthreads();
    if (!last) return;
    const double al = __ldcg(fin.nalpha);
    // the segment's rows: rseg*8 + k*nseg*8 + j (j < 8)
    const int64_t nblk = (m - rseg * 8 + nseg * 8 - 1) / (nseg * 8);
    for (int64_t t = threadIdx.x; t < nblk * 8; t += kThreads) {
      const int64_t row = rseg * 8 + (t >> 3) * nseg * 8 + (t & 7);
      if (row >= m) continue;
      const double s = strided_sum8(part + row, m, ngroups);
      fin.w[row] = s - al * __ldcg(fin.qprev + row);
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
  double s = strided_sum(part + r, part_ld, nchunks);
  if (qprev) s = s - (*alpha) * qprev[r];
  w[r] = s;
  flag_nonfinite(st, s, step);
}

// y = C x (trans 0, y has s1 entries) or C^T x (trans 1, s2 entries) for
// the s1 x s2 row-major core of a factored operator (linops.py:192-202);
// one warp per output, fixed order.
__global__ void __launch_bounds__(kThreads)
k_core_gemv(const double* __restrict__ C, int64_t s1, int64_t s2, int trans,
            const double* __restrict__ x, double* __restrict__ y, const DevState* st) {
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t outs = trans ? s2 : s1, ins = trans ? s1 : s2;
  if (i >= outs) return;
  double acc = 0.0;
  for (int64_t j = lane; j < ins; j += 32)
    acc = fma(trans ? C[j * s2 + i] : C[i * s2 + j], x[j], acc);
  acc = warp_sum(acc);
  if (lane == 0) y[i] = acc;
}

// ---------------------------------------------------------------------------
// gemv_t:  partial z = A^T q over a row split  (bidiag.py:169, linops.py:164)
//
// Column reduction of row-major A without a transposed copy.  Grid
// (ncoltiles, nsplit).  The CTA's 256 threads form RG row groups of
// TPG = 256/RG threads; each thread owns one 16-byte column vector (V
// columns) of the CTA's TPG-vector tile and accumulates V f64 sums over the
// rows of its group (rows g, g+RG, ... of the split, U rows in flight).  q
// for the split is staged through shared memory in blocks of kQB rows
// (optionally q = q_src / *q_scale: the deferred normalisation
// q_{i+1} = w / beta, bidiag.py:165, written to q_dst by tile-0 CTAs).  The
// RG group sums are combined in fixed order in shared memory and the split
// partial goes to part[s*ldz + col]; k_gemv_t_finalize adds the splits.
constexpr int kQB = 1024;
template <typename TA, int U, int RG>
__global__ void __launch_bounds__(kThreads)
k_gemv_t(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t nvec,
         int64_t rows_per_split, const double* __restrict__ q_src,
         const double* __restrict__ q_scale, double* __restrict__ q_dst,
         double* __restrict__ part, int64_t ldz, const DevState* st) {
  pdl_wait();
  pdl_trigger(1);
  if (halted(st)) return;
  constexpr int V = AVec<TA>::V;
  constexpr int TPG = kThreads / RG;
  __shared__ double q_s[kQB];
  __shared__ double red[RG > 1 ? RG : 1][RG > 1 ? TPG * V : 1];
  const int g = threadIdx.x / TPG, t = threadIdx.x % TPG;
  const int64_t vcol = (int64_t)blockIdx.x * TPG + t;
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
    int r = g;
    for (; r + (U - 1) * RG < nr; r += U * RG) {
      AVec<TA> a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u].load(p + (int64_t)(r + u * RG) * lda);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double qv = q_s[r + u * RG];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = fma(a[u].get(k), qv, acc[k]);
      }
    }
    for (; r < nr; r += RG) {
      AVec<TA> a;
      a.load(p + (int64_t)r * lda);
      const double qv = q_s[r];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fma(a.get(k), qv, acc[k]);
    }
  }
  if constexpr (RG > 1) {
#pragma unroll
    for (int k = 0; k < V; ++k) red[g][t * V + k] = acc[k];
    __syncthreads();
    if (g == 0 && active) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        double s = red[0][t * V + k];
#pragma unroll
        for (int gg = 1; gg < RG; ++gg) s += red[gg][t * V + k];
        acc[k] = s;
      }
    }
  }
  if (g == 0 && active) {
    double* dst = part + (int64_t)blockIdx.y * ldz + vcol * V;
#pragma unroll
    for (int k = 0; k < V; ++k) dst[k] = acc[k];
  }
}

// k_gemv_t with the row blocks of its split interleaved across the splits
// and visited bottom-up (block = RG*U*IT rows; CTA s takes blocks s,
// s + nsplit, ... from the last one): the whole grid then sweeps A upwards as
// one band, starting on the rows k_gemv_n (top-down band) left in L2.
// Shared-memory needs of gemv_t2_body (q staging + group sums), so callers
// can provide them (static in k_gemv_t2, part of the dynamic carve-out in
// the persistent kernel).
template <typename TA, int U, int RG, int IT>
struct GemvT2Smem {
  static constexpr int V = AVec<TA>::V;
  static constexpr int TPG = kThreads / RG;
  static constexpr int QS = RG * U * IT;
  static constexpr int RED = RG > 1 ? RG * TPG * V : 1;
};

template <typename TA, int U, int RG, int IT, bool CG = false>
__device__ __forceinline__ void gemv_t2_body(const TA* __restrict__ A, int64_t lda, int64_t m,
                                             int64_t nvec, const double* __restrict__ q_src,
                                             const double* __restrict__ q_scale,
                                             double* __restrict__ q_dst,
                                             double* __restrict__ part, int64_t ldz,
                                             int64_t bx, int64_t sp, int64_t nsplit,
                                             double* __restrict__ q_s,
                                             double* __restrict__ red_flat, int a_ef) {
  constexpr int V = AVec<TA>::V;
  constexpr int TPG = kThreads / RG;
  constexpr int RBT = RG * U * IT;
  static_assert(RBT <= kQB, "row block exceeds the q staging buffer");
  const int g = threadIdx.x / TPG, t = threadIdx.x % TPG;
  const int64_t vcol = bx * TPG + t;
  const bool active = vcol < nvec;
  const int64_t nblk = (m + RBT - 1) / RBT;
  const double scale = q_scale ? ldv<CG>(q_scale) : 1.0;
  double acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.0;
  const TA* base = A + vcol * V;
  const uint64_t pol = a_policy(a_ef);
  const int64_t last = sp < nblk ? sp + ((nblk - 1 - sp) / nsplit) * nsplit : -1;
  for (int64_t b = last; b >= 0; b -= nsplit) {
    const int64_t rb = b * RBT;
    const int nr = (int)min((int64_t)RBT, m - rb);
    __syncthreads();
    for (int e = threadIdx.x; e < nr; e += kThreads) {
      double qv = ldv<CG>(q_src + rb + e);
      if (q_scale) {
        qv = qv / scale;
        if (bx == 0 && q_dst) q_dst[rb + e] = qv;
      }
      q_s[e] = qv;
    }
    __syncthreads();
    if (!active) continue;
    const TA* p = base + rb * lda;
    int r = g;
    for (; r + (U - 1) * RG < nr; r += U * RG) {
      AVec<TA> a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u].load(p + (int64_t)(r + u * RG) * lda, pol);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double qv = q_s[r + u * RG];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = fma(a[u].get(k), qv, acc[k]);
      }
    }
    for (; r < nr; r += RG) {
      AVec<TA> a;
      a.load(p + (int64_t)r * lda, pol);
      const double qv = q_s[r];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fma(a.get(k), qv, acc[k]);
    }
  }
  if constexpr (RG > 1) {
#pragma unroll
    for (int k = 0; k < V; ++k) red_flat[g * (TPG * V) + t * V + k] = acc[k];
    __syncthreads();
    if (g == 0 && active) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        double sum = red_flat[t * V + k];
#pragma unroll
        for (int gg = 1; gg < RG; ++gg) sum += red_flat[gg * (TPG * V) + t * V + k];
        acc[k] = sum;
      }
    }
    if constexpr (CG) __syncthreads();  // red is reused by the next virtual block
  }
  if (g == 0 && active) {
    double* dst = part + sp * ldz + vcol * V;
#pragma unroll
    for (int k = 0; k < V; ++k) dst[k] = acc[k];
  }
}

template <typename TA, int U, int RG, int IT>
__global__ void __launch_bounds__(kThreads)
k_gemv_t2(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t nvec,
          int64_t /*unused*/, const double* __restrict__ q_src,
          const double* __restrict__ q_scale, double* __restrict__ q_dst,
          double* __restrict__ part, int64_t ldz, const DevState* st, int a_ef) {
  pdl_wait();
  pdl_trigger(1);
  if (halted(st)) return;
  using SM = GemvT2Smem<TA, U, RG, IT>;
  __shared__ double q_s[SM::QS];
  __shared__ double red[SM::RED];
  gemv_t2_body<TA, U, RG, IT>(A, lda, m, nvec, q_src, q_scale, q_dst, part, ldz, blockIdx.x,
                              blockIdx.y, gridDim.y, q_s, red, a_ef);
}

// z[j] = sum_s part[s][j] (- beta p[j]); zero in the padding [n, n_pad).
// CTA = 32 columns x 8 split groups: group g adds splits g, g+8, ...
// (coalesced 256-byte rows of partials), then the groups are combined in
// fixed order.
__global__ void __launch_bounds__(kThreads)
k_gemv_t_finalize(const double* __restrict__ part, int64_t ldz, int nsplit,
                  int64_t n, int64_t n_pad, const double* __restrict__ beta,
                  const double* __restrict__ pprev, double* __restrict__ z,
                  DevState* st, int step, int check) {
  if (halted(st)) return;
  __shared__ double red[kWarps][32];
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + c;
  double s = 0.0;
  if (j < n)
    for (int k = g; k < nsplit; k += kWarps) s += part[(int64_t)k * ldz + j];
  red[g][c] = s;
  __syncthreads();
  if (g != 0 || j >= n_pad) return;
  if (j >= n) {
    z[j] = 0.0;
    return;
  }
  s = red[0][c];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) s += red[w][c];
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
//
// B is a basis of `ncols` columns, each contiguous (ldb doubles apart), held
// in HBM/L2.  One kernel serves every pass: a CTA owns 32*RPL consecutive
// rows (lane = row, RPL rows per lane), its 8 warps split the columns
// (warp w takes j = w, w+8, ...), so every column read is a coalesced
// 256*RPL-byte segment and all loads of a warp are independent.
//   mode & kUpdate : x -= B c   (per-warp partial sums combined across the
//                    8 warps in fixed order through shared memory)
//   mode & kDot    : part[j*nrb + b] = sum_{rows of b} B[j][r] x[r] -- the
//                    coefficients of the NEXT pass; the CTA's B tile was
//                    just read by the update, so this re-read hits L1
//   mode & kNorm   : part[b] = sum_{rows of b} x[r]^2
// k_reduce_part adds the row blocks (fixed order) into c / the norm.
constexpr int kUpdate = 1, kDot = 2, kNorm = 4;

template <int RPL>
__global__ void __launch_bounds__(kThreads)
k_cgs_rows(const double* __restrict__ B, int64_t ldb, int ncols,
           const double* __restrict__ c, double* __restrict__ x, int64_t L,
           int mode, double* __restrict__ part, int nrb, const DevState* st) {
  if (halted(st)) return;
  constexpr int ROWS = 32 * RPL;
  __shared__ double tred[kWarps][ROWS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS + lane;
  double xv[RPL];
#pragma unroll
  for (int e = 0; e < RPL; ++e) {
    const int64_t r = r0 + 32 * e;
    xv[e] = r < L ? x[r] : 0.0;
  }
  if (mode & kUpdate) {
    double t[RPL];
#pragma unroll
    for (int e = 0; e < RPL; ++e) t[e] = 0.0;
#pragma unroll 4
    for (int j = warp; j < ncols; j += kWarps) {
      const double cj = c[j];
      const double* col = B + (int64_t)j * ldb;
#pragma unroll
      for (int e = 0; e < RPL; ++e) {
        const int64_t r = r0 + 32 * e;
        if (r < L) t[e] = fma(col[r], cj, t[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < RPL; ++e) tred[warp][lane + 32 * e] = t[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      double s = tred[0][lane + 32 * e];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) s += tred[w][lane + 32 * e];
      xv[e] = xv[e] - s;
      const int64_t r = r0 + 32 * e;
      if (warp == 0 && r < L) x[r] = xv[e];
    }
  }
  if (mode & kDot) {
    // 8 columns per batch: 8 * RPL independent loads in flight per lane and
    // one 9-shuffle transpose butterfly (warp_sum8) for the 8 sums, instead
    // of a 5-shuffle reduction per column (the dot pass was latency-bound)
    for (int q0 = 0; warp + kWarps * q0 < ncols; q0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = warp + kWarps * (q0 + u);
        v[u] = 0.0;
        if (j < ncols) {
          const double* col = B + (int64_t)j * ldb;
#pragma unroll
          for (int e = 0; e < RPL; ++e) {
            const int64_t r = r0 + 32 * e;
            if (r < L) v[u] = fma(col[r], xv[e], v[u]);
          }
        }
      }
      const double t = warp_sum8(v);
      const int j = warp + kWarps * (q0 + warp_sum8_index(lane));
      if ((lane & 3) == 0 && j < ncols) part[(int64_t)j * nrb + blockIdx.x] = t;
    }
  }
  if ((mode & kNorm) && warp == 0) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < RPL; ++e) s = fma(xv[e], xv[e], s);
    s = warp_sum(s);
    if (lane == 0) part[blockIdx.x] = s;
  }
}

// fixed-order block sum of v over the 256 threads (result valid in thread 0)
__device__ __forceinline__ double block_sum(double v, double* red8) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red8[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    t = red8[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) t += red8[w];
  }
  return t;
}

// out[j] = sum_b part[j*nrb + b]; one CTA per column, fixed order
__global__ void __launch_bounds__(kThreads)
k_reduce_part(const double* __restrict__ part, int nrb, double* __restrict__ out,
              const DevState* st) {
  if (halted(st)) return;
  __shared__ double red8[kWarps];
  const double* p = part + (int64_t)blockIdx.x * nrb;
  double s = 0.0;
  for (int b = threadIdx.x; b < nrb; b += kThreads) s += p[b];
  s = block_sum(s, red8);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// Norm test (bidiag.py:156-158, 173-174; fsvd.py:151-152).
// nrb > 0: s = sum part[0..nrb) and the local non-finite flag (single rank).
// nrb == 0: s = red[0], flag = red[1] (already all-reduced by the caller).
// nrm = sqrt(s) -> *slot; non-finite -> ST_NONFINITE; nrm < eps -> `code`.
__global__ void __launch_bounds__(kThreads)
k_norm_test(const double* __restrict__ part, int nrb, const double* __restrict__ red,
            double eps, double* __restrict__ slot, DevState* st, int step, int code,
            HostProg* hp, int side) {
  if (halted(st)) return;
  __shared__ double red8[kWarps];
  double s = 0.0, flag = 0.0;
  if (nrb > 0) {
    for (int b = threadIdx.x; b < nrb; b += kThreads) s += part[b];
    s = block_sum(s, red8);
    flag = st->nonfinite ? 1.0 : 0.0;
  } else {
    s = red[0];
    flag = red[1];
  }
  if (threadIdx.x == 0) {
    const double nrm = sqrt(s);
    *slot = nrm;
    int stop = ST_RUNNING;
    if (flag != 0.0 || !isfinite(nrm)) stop = ST_NONFINITE;
    else if (nrm < eps) stop = code;
    if (stop != ST_RUNNING) {
      st->status = stop;
      st->kprime = step;
      st->where = step;
    }
    host_progress(hp, stop, step, side);
  }
}

// red[0] = sum part[0..nrb), red[1] = local non-finite flag (pre all-reduce)
__global__ void __launch_bounds__(kThreads)
k_norm_prep(const double* __restrict__ part, int nrb, double* __restrict__ red,
            const DevState* st) {
  if (halted(st)) return;
  __shared__ double red8[kWarps];
  double s = 0.0;
  for (int b = threadIdx.x; b < nrb; b += kThreads) s += part[b];
  s = block_sum(s, red8);
  if (threadIdx.x == 0) {
    red[0] = s;
    red[1] = st->nonfinite ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Fused CGS2 for one rank (bidiag.py:154-156, 171-173): ONE cooperative
// kernel per orthogonalisation instead of six launches.  Every CTA owns a
// contiguous slab of rows; phases are separated by a grid barrier:
//
//   [0] optional gemv_t finalisation: x = sum_splits(part) - beta p
//   [1] partial c = B^T x over the slab           -> part[j*G + b]
//   [2] c[j] = sum_b part[j*G + b]  (columns spread over all warps)
//   [3] x -= B c, fused with the next pass's partials (or ||x||^2)
//   ... [2],[3] repeated per pass ...
//   [4] CTA 0: beta / alpha = sqrt(sum_b part[b]); breakdown test
//
// All sums run in a fixed order, independent of scheduling.  The grid is
// launched cooperatively (co-residency guaranteed by the driver) and the
// barrier is a counter/generation pair in global memory.
struct CgsCoopArgs {
  const double* B;
  int64_t ldb;
  int ncols;
  double* x;
  int64_t L;
  int rows_per_cta;
  int passes;  // 0: norm only
  double eps;
  double* slot;
  DevState* st;
  int step, code;
  HostProg* hp;
  int side;
  double* part;   // >= ncols * G
  double* c;      // >= ncols
  unsigned* bar;  // {count, generation}
  // phase 0 (nullable fpart): x[r] = sum_s fpart[s*fld + r] - (*fbeta) fp[r]
  const double* fpart;
  int64_t fld;
  int fnsplit;
  const double* fbeta;
  const double* fp;
  unsigned long long* tdbg;  // nullable: phase timing of CTA 0
  int redundant;  // k_cgs2_tile2: every CTA reduces all partials (else distributed + barrier)
};

// Grid-wide barrier of the cooperative launch (cooperative_groups: ~1.2 us
// on 148 SMs, measured by tools/barrier_bench.cu, vs ~2.3 us for a plain
// counter/generation barrier).
// bar == nullptr: cooperative-groups grid sync (cooperative launch).
// Otherwise a flip barrier on bar[0] for a regular
// launch whose CTAs are all resident (one per SM, see cgs_coop): lets the
// CGS grid start under programmatic dependent launch, which a cooperative
// launch does not.
__device__ __forceinline__ void grid_barrier_raw(unsigned* bar, unsigned nblocks) {
  if (bar == nullptr) {
    cooperative_groups::this_grid().sync();
    return;
  }
  // one release-add per CTA on a single word; CTA 0 adds 2^31 - (nblocks - 1)
  // so the last arrival flips bit 31 and the low bits return to their value
  // (the cooperative-groups scheme: no reset, no second atomic, any nblocks)
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    unsigned old, cur;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(nb)
                 : "memory");
    // a regular launch relies on all nblocks CTAs becoming resident (one per
    // SM, <= #SMs).  ksvd_ctx_create probes that once (residency_probe) and
    // switches the context to cooperative launches when it does not hold (an
    // SM-limited MPS client or green context); should it still fail, trap
    // after ~20 s instead of spinning forever
    unsigned polls = 0;
    unsigned long long t0 = 0;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      if ((++polls & 0xfffu) == 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > 20000000000ull) {
          printf("ksvd: grid barrier of %u CTAs timed out (not all CTAs resident?)\n",
                 nblocks);
          __trap();
        }
      }
    } while (((old ^ cur) & 0x80000000u) == 0);
  }
  __syncthreads();
}

// One-off residency probe (ksvd_ctx_create): G CTAs of a kernel using the
// CGS kernels' shared-memory budget (so one CTA per SM) arrive on a counter
// and wait for all G with a short bounded spin; any CTA that gives up sets
// *failed.  Regular launches with software grid barriers are then safe on
// this context, else it uses cooperative launches.
__global__ void __launch_bounds__(kThreads, 1)
k_residency_probe(unsigned* count, int* failed, unsigned G) {
  extern __shared__ unsigned char probe_smem[];
  if (threadIdx.x == 0) {
    probe_smem[0] = 1;
    atomicAdd(count, 1u);
    unsigned long long t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(count) : "memory");
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 200000000ull) {  // 200 ms
        atomicExch(failed, 1);
        break;
      }
    } while (cur < G);
  }
}

// the k-th grid-wide barrier of a CGS launch (k counted per thread: every
// CTA passes the same sequence of barriers)
__device__ __forceinline__ void grid_barrier(const CgsCoopArgs& a, unsigned G,
                                             unsigned long long& k) {
  ++k;
  grid_barrier_raw(a.bar, G);
}

// phase timestamps of CTA 0 (debug builds of the timing breakdown)
__device__ __forceinline__ void phase_mark(unsigned long long* t, int k, unsigned long long& last) {
  if (t && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (k > 0) atomicAdd(t + k, now - last);
    last = now;
  }
}

// Tile-resident fused CGS2 (k_cgs2_tile2): each CTA first pulls its whole
// basis tile (rows_per_cta x ncols) from L2/HBM into shared memory with one
// bulk-async (TMA) copy per column segment, all in flight on one mbarrier,
// then runs every sweep of the two CGS passes out of shared memory -- the
// basis is read once per orthogonalisation, at bulk-copy bandwidth.  2 grid
// rounds per CGS2 where every CTA reduces all G partials of every column
// itself (a few KB of L2 reads, cheaper than a second barrier), else 4
// (distributed column sums + a barrier); the partial buffers ping-pong
// between passes, and beta^2 = ||x||^2 - ||c||^2 comes with the last pass's
// dot products (direct-norm round only when that would cancel).  tile2_issue
// starts the bulk copy of this CTA's tile, tile2_rest does the rest.  Every
// load of data another CTA wrote in the same launch goes through L2
// (__ldcg / volatile), and the tile copy is fenced against the generic
// proxy (fence.proxy.async).
__device__ __forceinline__ void tile2_issue(const CgsCoopArgs& a, double* tile, uint32_t bar,
                                            bool init) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t s1 = min(a.L, s0 + a.rows_per_cta);
  const int nr = s1 > s0 ? (int)(s1 - s0) : 0;
  const int ldt = (nr + 1) & ~1;  // 16-byte column segments
  // bulk-async load of the basis tile: lane 0 of warp 0 arms the mbarrier
  // with the total byte count, then the 32 lanes of warp 0 issue the
  // per-column copies (one thread issuing ~100+ copies serially was the
  // largest fixed cost of this kernel); all threads wait later.
  (void)lane;
  (void)warp;
  const uint32_t bytes = (uint32_t)ldt * 8u;
  if (threadIdx.x == 0) {
    if (init) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t total = bytes * (uint32_t)a.ncols;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(total)
                 : "memory");
  }
  __syncthreads();
  // one column copy per thread (up to 256 in flight from all 8 warps: the
  // issue of ~150 copies from one warp was measured at ~2.6 us per kernel)
  if (bytes) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int j = threadIdx.x; j < a.ncols; j += kThreads) {
      const double* src = a.B + (int64_t)j * a.ldb + s0;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(smem_u32(tile + (size_t)j * ldt)),
          "l"(src), "r"(bytes), "r"(bar)
          : "memory");
    }
  }
}

// Returns ||x||^2 after the orthogonalisation (the same value in every CTA:
// callers of the persistent kernels use it instead of re-reading the slot).
// halt_check: test the run status here (its load in flight with the
// finalisation loads) and return -1.0 if the run has halted, the copy drained.
template <int MAXE>
__device__ __forceinline__ double tile2_rest(const CgsCoopArgs& a, double* tile,
                                           double (*tred)[32 * MAXE], uint32_t bar,
                                           uint32_t parity, unsigned long long t_entry,
                                           bool halt_check = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  unsigned long long bk = 0;  // grid barriers passed in this launch
  const int64_t s0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t s1 = min(a.L, s0 + a.rows_per_cta);
  const int nr = s1 > s0 ? (int)(s1 - s0) : 0;
  const int ldt = (nr + 1) & ~1;
  double* cs = tile + (size_t)a.ncols * ldt;  // coefficients of the current pass
  if (a.tdbg && blockIdx.x == 0 && threadIdx.x == 0) {  // [8] entry -> finalisation start
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicAdd(a.tdbg + 8, now - t_entry);
  }
  // [0] finalisation of the split partial sums of the product (overlaps the
  // copy): one row per thread (nr <= 32 * MAXE <= kThreads), every load --
  // the run status included -- in flight at once; the row values go to x
  // and, staged in smem, to the per-warp register copies below
  double* xs = &tred[0][0];
  const int st0 = halt_check ? *reinterpret_cast<const volatile int*>(&a.st->status)
                             : (int)ST_RUNNING;
  if (a.fpart) {
    const double fb = a.fp ? __ldcg(a.fbeta) : 0.0;
    const int64_t r = s0 + threadIdx.x;
    if (r < s1) {
      double v = strided_sum(a.fpart + r, a.fld, a.fnsplit);
      if (a.fp) v = v - fb * __ldcg(a.fp + r);
      if (st0 == ST_RUNNING) {
        a.x[r] = v;
        flag_nonfinite(a.st, v, a.step);
      }
      xs[threadIdx.x] = v;
    }
  }
  if (st0 != ST_RUNNING) {  // same value in every thread of every CTA
    if (threadIdx.x == 0)
      while (!mbar_try_wait(bar, parity)) {
      }
    return -1.0;
  }
  unsigned long long tl = 0;
  phase_mark(a.tdbg, 0, tl);
  if (a.tdbg && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.tdbg + 5, tl - t_entry);
  __syncthreads();
  // x rows of this CTA live in registers for the whole kernel (loaded while
  // the tile is in flight)
  double xv[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int rl = lane + 32 * e;
    xv[e] = rl < nr ? (a.fpart ? xs[rl] : a.x[s0 + rl]) : 0.0;
  }
  while (!mbar_try_wait(bar, parity)) {
  }
  phase_mark(a.tdbg, 1, tl);  // [1] bulk copy of the tile (+ finalisation)


  // Ping-pong partial buffers, (ncols + 1) x G each (row ncols: norm
  // partials): a CTA may write pass p+1's partials while slower CTAs still
  // read pass p's, since every CTA reduces every column itself.
  const int64_t half = (int64_t)(a.ncols + 1) * G;
  auto partb = [&](int k) { return a.part + (k & 1) * half; };
  double* red = cs;  // reduced sums: ncols coefficients + the norm (ncols + 1 doubles)

  // xv -= tile * red[0:ncols]; the final pass stores x
  auto update = [&](bool store) {
    double t[MAXE];
#pragma unroll
    for (int e = 0; e < MAXE; ++e) t[e] = 0.0;
#pragma unroll 4
    for (int j = warp; j < a.ncols; j += kWarps) {
      const double cj = red[j];
      const double* col = tile + (size_t)j * ldt;
#pragma unroll
      for (int e = 0; e < MAXE; ++e) {
        const int rl = lane + 32 * e;
        if (rl < nr) t[e] = fma(col[rl], cj, t[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < MAXE; ++e) tred[warp][lane + 32 * e] = t[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      double s = tred[0][lane + 32 * e];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) s += tred[w][lane + 32 * e];
      xv[e] = xv[e] - s;
      const int rl = lane + 32 * e;
      if (store && warp == 0 && rl < nr) a.x[s0 + rl] = xv[e];
    }
    __syncthreads();
  };
  // this CTA's partial dots tile^T xv -> P[j*G + b]; optionally ||xv||^2 -> P[ncols*G + b]
  auto dot = [&](double* P, bool with_norm) {
    for (int q0 = 0; warp + kWarps * q0 < a.ncols; q0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = warp + kWarps * (q0 + u);
        v[u] = 0.0;
        if (j < a.ncols) {
          const double* col = tile + (size_t)j * ldt;
#pragma unroll
          for (int e = 0; e < MAXE; ++e) {
            const int rl = lane + 32 * e;
            if (rl < nr) v[u] = fma(col[rl], xv[e], v[u]);
          }
        }
      }
      const double t = warp_sum8(v);
      const int j = warp + kWarps * (q0 + warp_sum8_index(lane));
      if ((lane & 3) == 0 && j < a.ncols) P[(int64_t)j * G + blockIdx.x] = t;
    }
    if (with_norm && warp == kWarps - 1) {
      double s = 0.0;
#pragma unroll
      for (int e = 0; e < MAXE; ++e) s = fma(xv[e], xv[e], s);
      s = warp_sum(s);
      if (lane == 0) P[(int64_t)a.ncols * G + blockIdx.x] = s;
    }
  };
  // red[j] = sum_b P[j*G + b] for j in [j0, j1), same fixed order in every
  // CTA.  Redundant mode: each warp sums 4 columns with all 4 x 5 loads in
  // flight (G <= 160); distributed mode: the grid's warps split the columns
  // (coop_reduce_cols into a.c), one more barrier, then every CTA copies a.c.
  auto reduce_all = [&](const double* P, int j0, int j1) {
    if (a.redundant) {
      for (int jb = j0 + 4 * warp; jb < j1; jb += 4 * kWarps) {
        double sacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const unsigned b = lane + 32 * k;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (b < G && jb + u < j1) sacc[u] += __ldcg(P + (int64_t)(jb + u) * G + b);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double t = warp_sum(sacc[u]);
          if (lane == 0 && jb + u < j1) red[jb + u] = t;
        }
      }
    } else {
      const int gw = blockIdx.x * kWarps + warp, nw = (int)G * kWarps;
      for (int j = j0 + gw; j < j1; j += nw) {
        const double* p = P + (int64_t)j * G;
        double t = 0.0;
        for (unsigned b0 = 0; b0 < G; b0 += 160) {  // 5 loads per lane in flight
          double v[5];
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const unsigned b = b0 + lane + 32 * k;
            v[k] = b < G ? __ldcg(p + b) : 0.0;
          }
#pragma unroll
          for (int k = 0; k < 5; ++k)
            if (b0 + lane + 32 * k < G) t += v[k];  // the order of the plain loop
        }
        t = warp_sum(t);
        if (lane == 0) a.c[j] = t;
      }
      phase_mark(a.tdbg, 10, tl);  // [10] distributed column sums
      grid_barrier(a, G, bk);
      phase_mark(a.tdbg, 11, tl);  // [11] the barrier after them
      for (int j = j0 + (int)threadIdx.x; j < j1; j += kThreads) red[j] = __ldcg(a.c + j);
    }
    __syncthreads();
  };
  double result = 0.0;
  auto finish = [&](double nrm2) {
    result = nrm2;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const double nrm = sqrt(nrm2);
      *a.slot = nrm;
      int stop = ST_RUNNING;
      if (*reinterpret_cast<volatile int*>(&a.st->nonfinite) || !isfinite(nrm))
        stop = ST_NONFINITE;
      else if (nrm < a.eps) stop = a.code;
      if (stop != ST_RUNNING) {
        a.st->status = stop;
        a.st->kprime = a.step;
        a.st->where = a.step;
      }
      host_progress(a.hp, stop, a.step, a.side);
    }
  };

  // One grid round per coefficient pass (k = 0 .. P-1), the norm riding on
  // the last one, plus a direct-norm round when the closed form would
  // cancel (or for an empty basis).  Every helper has ONE call site: inlined
  // at several sites the kernel overflowed the instruction cache (ncu on
  // config 2: 19 % of the warp stalls were no_inst at 7.2k SASS instructions).
  const int P = a.ncols > 0 ? a.passes : 0;
  bool norm_only = P == 0;
  for (int k = 0;; ++k) {
    const bool with_norm = norm_only || k + 1 == P;
    if (norm_only) {
      if (warp == kWarps - 1) {
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < MAXE; ++e) s = fma(xv[e], xv[e], s);
        s = warp_sum(s);
        if (lane == 0) partb(k)[(int64_t)a.ncols * G + blockIdx.x] = s;
      }
    } else {
      dot(partb(k), with_norm);
    }
    phase_mark(a.tdbg, 2, tl);
    grid_barrier(a, G, bk);
    phase_mark(a.tdbg, 3, tl);
    reduce_all(partb(k), norm_only ? a.ncols : 0, a.ncols + (with_norm ? 1 : 0));
    phase_mark(a.tdbg, 4, tl);
    if (norm_only) {
      finish(red[a.ncols]);
      break;
    }
    const bool last = k + 1 == P;
    // ||x - B c||^2 = ||x||^2 - ||c||^2 for an orthonormal B.  Exact to
    // rounding while ||c||^2 <= 1e-6 ||x||^2 (always, after a first pass,
    // away from breakdown); otherwise (or non-finite) take the direct norm
    // with one more round.  The test reads identical values in every CTA.
    // ||c||^2: lane-strided partial sums + a butterfly, the same order in
    // every warp of every CTA
    double cc = 0.0, nn = 0.0;
    if (last) {
      for (int j = lane; j < a.ncols; j += 32) cc = fma(red[j], red[j], cc);
      cc = warp_sum(cc);
      nn = red[a.ncols];
    }
    update(last);
    if (!last) continue;
    if (cc <= 1e-6 * nn) {
      finish(nn - cc);
      break;
    }
    norm_only = true;
  }
  if (a.tdbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicAdd(a.tdbg + 6, now - t_entry);
    atomicAdd(a.tdbg + 7, 1ull);
  }
  return result;
}

template <int MAXE>
__global__ void __launch_bounds__(kThreads, 1)
k_cgs2_tile2(CgsCoopArgs a) {
  unsigned long long t_entry = 0;
  if (a.tdbg && blockIdx.x == 0 && threadIdx.x == 0)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double tred[kWarps][32 * MAXE];
  __shared__ __align__(8) unsigned long long mbar;
  double* tile = reinterpret_cast<double*>(smem_raw);
  const uint32_t bar = smem_u32(&mbar);
  tile2_issue(a, tile, bar, true);
  // The basis columns were written >= 2 launches back (complete once the
  // predecessor passed its own pdl_wait), so the tile copy above may run
  // ahead of this wait; the partial sums / x below may not.
  pdl_wait();
  pdl_trigger(2);
  // the halt test (copy drained before exiting) is inside, its load in
  // flight with the finalisation's
  tile2_rest<MAXE>(a, tile, tred, bar, 0, t_entry, true);
}


// Multi-rank CGS2 of a row-sharded basis with the tile in shared memory:
// the passes of k_cgs2_tile2 as three launches, the host's all-reduces of
// the coefficient vector between them (the multi-kernel path needs eight
// launches for the same CGS2):
//   phase 0: finalisation of k_gemv_n's chunk-group partials (x = A p - alpha q),
//            partial B^T x -> grid barrier -> distributed column sums -> c
//   phase 1: x -= B c (c all-reduced by the host) ; partial B^T x -> ... -> c
//   phase 2: x -= B c ; ||x||^2 of this rank's rows (CTA 0, fixed order) and
//            the local non-finite flag -> c[0], c[1] (all-reduced by the host
//            and tested by k_norm_test, so every rank halts at the same step)
// The same shared-memory sweeps and fixed-order sums as k_cgs2_tile2.
template <int MAXE>
__global__ void __launch_bounds__(kThreads, 1)
k_cgs_tile_phase(CgsCoopArgs a, int phase) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double tred[kWarps][32 * MAXE];
  __shared__ double red8[kWarps];
  __shared__ __align__(8) unsigned long long mbar;
  double* tile = reinterpret_cast<double*>(smem_raw);
  const uint32_t bar = smem_u32(&mbar);
  // the basis columns were written >= 2 launches back: the tile copy may
  // run ahead of the programmatic-launch wait, nothing else may
  tile2_issue(a, tile, bar, true);
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  unsigned long long bk = 0;
  const int64_t s0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t s1 = min(a.L, s0 + a.rows_per_cta);
  const int nr = s1 > s0 ? (int)(s1 - s0) : 0;
  const int ldt = (nr + 1) & ~1;
  double* red = tile + (size_t)a.ncols * ldt;  // the reduced coefficients
  double* xs = &tred[0][0];
  // x rows (finalised from the product partials in phase 0), the all-reduced
  // coefficients and the run status, all loads in flight together
  const int st0 = *reinterpret_cast<const volatile int*>(&a.st->status);
  if (phase == 0 && a.fpart) {
    const double fb = a.fp ? __ldcg(a.fbeta) : 0.0;
    const int64_t r = s0 + threadIdx.x;
    if (r < s1) {
      double v = strided_sum(a.fpart + r, a.fld, a.fnsplit);
      if (a.fp) v = v - fb * __ldcg(a.fp + r);
      if (st0 == ST_RUNNING) {
        a.x[r] = v;
        flag_nonfinite(a.st, v, a.step);
      }
      xs[threadIdx.x] = v;
    }
  } else if (threadIdx.x < nr) {
    xs[threadIdx.x] = __ldcg(a.x + s0 + threadIdx.x);
  }
  if (phase > 0)
    for (int j = threadIdx.x; j < a.ncols; j += kThreads) red[j] = __ldcg(a.c + j);
  if (st0 != ST_RUNNING) {
    if (threadIdx.x == 0)
      while (!mbar_try_wait(bar, 0)) {
      }
    return;
  }
  __syncthreads();
  double xv[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int rl = lane + 32 * e;
    xv[e] = rl < nr ? xs[rl] : 0.0;
  }
  while (!mbar_try_wait(bar, 0)) {
  }
  __syncthreads();  // xs (tred) is reused below
  if (phase > 0) {  // xv -= tile * red; store x
    double t[MAXE];
#pragma unroll
    for (int e = 0; e < MAXE; ++e) t[e] = 0.0;
#pragma unroll 4
    for (int j = warp; j < a.ncols; j += kWarps) {
      const double cj = red[j];
      const double* col = tile + (size_t)j * ldt;
#pragma unroll
      for (int e = 0; e < MAXE; ++e) {
        const int rl = lane + 32 * e;
        if (rl < nr) t[e] = fma(col[rl], cj, t[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < MAXE; ++e) tred[warp][lane + 32 * e] = t[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      double sum = tred[0][lane + 32 * e];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) sum += tred[w][lane + 32 * e];
      xv[e] = xv[e] - sum;
      const int rl = lane + 32 * e;
      if (warp == 0 && rl < nr) a.x[s0 + rl] = xv[e];
    }
  }
  if (phase < 2) {
    // partial dots of this CTA -> part[j*G + b]
    for (int q0 = 0; warp + kWarps * q0 < a.ncols; q0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = warp + kWarps * (q0 + u);
        v[u] = 0.0;
        if (j < a.ncols) {
          const double* col = tile + (size_t)j * ldt;
#pragma unroll
          for (int e = 0; e < MAXE; ++e) {
            const int rl = lane + 32 * e;
            if (rl < nr) v[u] = fma(col[rl], xv[e], v[u]);
          }
        }
      }
      const double t = warp_sum8(v);
      const int j = warp + kWarps * (q0 + warp_sum8_index(lane));
      if ((lane & 3) == 0 && j < a.ncols) a.part[(int64_t)j * G + blockIdx.x] = t;
    }
    grid_barrier(a, G, bk);
    // c[j] = sum_b part[j*G + b]: the grid's warps take columns round-robin
    const int gw = blockIdx.x * kWarps + warp, nw = (int)G * kWarps;
    for (int j = gw; j < a.ncols; j += nw) {
      const double* p = a.part + (int64_t)j * G;
      double t = 0.0;
      for (unsigned b0 = 0; b0 < G; b0 += 160) {
        double v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const unsigned b = b0 + lane + 32 * k;
          v[k] = b < G ? __ldcg(p + b) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k)
          if (b0 + lane + 32 * k < G) t += v[k];
      }
      t = warp_sum(t);
      if (lane == 0) a.c[j] = t;
    }
  } else {
    if (warp == kWarps - 1) {
      double sq = 0.0;
#pragma unroll
      for (int e = 0; e < MAXE; ++e) sq = fma(xv[e], xv[e], sq);
      sq = warp_sum(sq);
      if (lane == 0) a.part[blockIdx.x] = sq;
    }
    grid_barrier(a, G, bk);
    if (blockIdx.x == 0) {
      double sq = 0.0;
      for (unsigned b = threadIdx.x; b < G; b += kThreads) sq += __ldcg(a.part + b);
      sq = block_sum(sq, red8);
      if (threadIdx.x == 0) {
        a.c[0] = sq;
        a.c[1] = *reinterpret_cast<volatile int*>(&a.st->nonfinite) ? 1.0 : 0.0;
      }
    }
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

// Y[:, t] = (A X[:, t]) / sigma[t] on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64): one pass over A for up to 32 right-hand sides per
// CTA column (the reference runs `take` separate matvecs, fsvd.py:193-194).
// CTA tile 256 rows x 32 columns, 8 warps x (32 rows x 32 columns) = 4 x 4
// m8n8 accumulator tiles per warp.  A is staged in 32-column slabs with
// cp.async (two-stage ring) into a padded row-major layout whose fragment
// reads are bank-conflict-free (row stride = 4 mod 16 doubles / 4 mod 32
// floats); X^T is staged the same way.  Per k-step of 4: 4 A-fragment and 4
// B-fragment shared loads feed 16 DMMAs.  Deterministic (fixed k order).
constexpr int kMR = 256, kMC = 32, kMKC = 32;
constexpr int kMStride = kMKC + 4;  // padded row stride (elements)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const uint32_t s = smem_u32(smem);
  const int n = pred ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <typename TA>
__global__ void __launch_bounds__(kThreads, 2)
k_multi_rhs(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t n,
            const double* __restrict__ X, int64_t ldx, int ncols,
            const double* __restrict__ sigma, double* __restrict__ Y, int64_t ldy) {
  constexpr int V = AVec<TA>::V;
  constexpr int VPR = kMKC / V;                 // 16-byte vectors per slab row
  constexpr int APER = kMR * VPR / kThreads;    // A vectors per thread per slab
  extern __shared__ __align__(16) unsigned char mrhs_smem[];
  TA* As = reinterpret_cast<TA*>(mrhs_smem);                      // [2][kMR][kMStride]
  double* Xt = reinterpret_cast<double*>(As + 2 * kMR * kMStride);  // [2][kMC][kMStride]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kMR;
  const int t0 = blockIdx.y * kMC;
  const int64_t nvec = (n + V - 1) / V;
  const int64_t nslab = (n + kMKC - 1) / kMKC;

  auto stage = [&](int buf, int64_t k0) {
    TA* as = As + (size_t)buf * kMR * kMStride;
#pragma unroll
    for (int q = 0; q < APER; ++q) {
      const int e = tid + q * kThreads;
      const int rr = e / VPR, vv = e % VPR;
      const int64_t r = r0 + rr, vi = k0 / V + vv;
      const bool ok = r < m && vi < nvec;
      cp_async16(as + rr * kMStride + vv * V, ok ? (const void*)(A + r * lda + vi * V) : (const void*)A,
                 ok);
    }
    double* xt = Xt + (size_t)buf * kMC * kMStride;
    // X^T slab: column t, 32 k values (8 x 16 B per column)
    for (int e = tid; e < kMC * (kMKC / 2); e += kThreads) {
      const int tt = e / (kMKC / 2), vv = e % (kMKC / 2);
      const int64_t k = k0 + 2 * vv;
      const bool ok = t0 + tt < ncols && k + 1 < n;
      if (ok || !(t0 + tt < ncols && k < n)) {
        cp_async16(xt + tt * kMStride + 2 * vv,
                   ok ? (const void*)(X + (int64_t)(t0 + tt) * ldx + k) : (const void*)X, ok);
      } else {  // odd tail element
        xt[tt * kMStride + 2 * vv] = X[(int64_t)(t0 + tt) * ldx + k];
        xt[tt * kMStride + 2 * vv + 1] = 0.0;
      }
    }
    cp_async_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row / k index
  stage(0, 0);
  for (int64_t s = 0; s < nslab; ++s) {
    const int buf = (int)(s & 1);
    if (s + 1 < nslab) {
      stage(buf ^ 1, (s + 1) * kMKC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const TA* as = As + (size_t)buf * kMR * kMStride + (size_t)(warp * 32) * kMStride;
    const double* xt = Xt + (size_t)buf * kMC * kMStride;
#pragma unroll
    for (int kb = 0; kb < kMKC; kb += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = (double)as[(i * 8 + fr) * kMStride + kb + fk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = xt[(j * 8 + fr) * kMStride + kb + fk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  // D fragment: row fr, columns 2*fk, 2*fk+1 of each 8 x 8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + warp * 32 + i * 8 + fr;
    if (r >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = t0 + j * 8 + 2 * fk + h;
        if (t < ncols) Y[(int64_t)t * ldy + r] = sigma ? acc[i][j][h] / sigma[t] : acc[i][j][h];
      }
  }
}

template <typename TA>
constexpr size_t multi_rhs_smem() {
  return 2 * (size_t)kMR * kMStride * sizeof(TA) + 2 * (size_t)kMC * kMStride * sizeof(double);
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


// Y[:, t] = sum_j B[:, j] G[j + t*kp] on the FP64 tensor cores: the
// tall-skinny Ritz / restart contractions V = P G, U = Q X (north star (c);
// fsvd.py:191).  B is a column-major basis (ldb), L rows x kp columns; G is
// kp x take column-major.  CTA = 8 warps x 32 rows, 32 output columns
// (grid.y tiles take); warp tile 32 x 32 = 4 x 4 m8n8 accumulators; per
// k-step of 4, each lane loads 4 basis elements (4 columns x 8 consecutive
// rows per load instruction: full 32-byte sectors) and 4 G elements (L1),
// and issues 16 DMMAs.  Fixed k order: deterministic.
constexpr int kBCR = 32 * kWarps;  // rows per CTA
__global__ void __launch_bounds__(kThreads)
k_basis_combine_dmma(const double* __restrict__ B, int64_t ldb, int64_t L, int kp,
                     const double* __restrict__ G, int take, double* __restrict__ Y,
                     int64_t ldy) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = lane >> 2, ti = lane & 3;
  const int64_t rw = (int64_t)blockIdx.x * kBCR + warp * 32;
  const int t0 = blockIdx.y * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  bool rok[4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) rok[mt] = rw + mt * 8 + gi < L;
  bool cok[4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) cok[nt] = t0 + nt * 8 + gi < take;
#pragma unroll 4
  for (int j0 = 0; j0 < kp; j0 += 4) {
    const int j = j0 + ti;
    const bool jok = j < kp;
    double av[4], bv[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      av[mt] = (jok && rok[mt]) ? __ldg(B + (int64_t)j * ldb + rw + mt * 8 + gi) : 0.0;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
      bv[nt] = (jok && cok[nt]) ? __ldg(G + j + (int64_t)(t0 + nt * 8 + gi) * kp) : 0.0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt], av[mt], bv[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t r = rw + mt * 8 + gi;
    if (r >= L) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = t0 + nt * 8 + 2 * ti + h;
        if (t < take) Y[(int64_t)t * ldy + r] = acc[mt][nt][h];
      }
    }
  }
}

}  // namespace ksvd
