// stream.cuh -- the GK steps of a streamed (HBM-resident) matrix in ONE
// persistent cooperative kernel (included by ksvd.cu).
//
// The 4-launch step (k_gemv_n2, k_cgs2_tile2, k_gemv_t2, k_cgs2_tile2)
// pays each kernel's launch and ramp every step.  k_gk_stream runs the same
// device bodies (kernels.cuh: gemv_n2_body, tile2_issue / tile2_rest,
// gemv_t2_body with coherent loads) back to back inside one grid of one CTA
// per SM, separated by grid barriers: the gemv_n work decomposition is the
// standalone one (its plan already has one CTA per SM), the gemv_t grid
// (column tiles x row splits) is walked as virtual blocks, and each CGS2
// bulk-loads its basis tile exactly as the standalone kernel does.  Scalars,
// status words and vectors are written as by the 4-launch loop, so the host
// can hand over to it at any step (when the basis tile outgrows shared
// memory) and every other entry point is unchanged.
#pragma once
#include <cooperative_groups.h>

namespace ksvd {

struct StreamArgs {
  const double* A;
  int64_t lda, mloc, n;
  int64_t nvec;  // n in 16-byte vectors
  int nchunks;
  int64_t nseg;
  double* part_n;
  int64_t ncoltiles, nsplit, ldz;
  double* part_t;
  double *Q, *P;
  int64_t ldq, ldp;
  double *w, *z, *alpha, *beta;
  DevState* st;
  int i0, i_end, k_max, passes;
  double eps;
  int rows_l, rows_r;
  double *lpart, *lc, *rpart, *rc;
  unsigned *lbar, *rbar;
  int64_t red_max;
  HostProg* hp;
  unsigned long long* tdbg;  // KSVD_PHASE_TIMES: CTA-0 phase times
};

template <int MAXE, int ITT>
__global__ void __launch_bounds__(kThreads, 1) k_gk_stream(StreamArgs s) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double tred[kWarps][32 * MAXE];
  __shared__ __align__(8) unsigned long long mbar;
  // gemv_t with 32 rows in flight per thread (the standalone kernel's 16 at
  // 4 CTAs per SM would leave a one-CTA-per-SM grid short of loads in flight)
  constexpr int UT = ITT <= 4 ? 32 : 16;
  using SMT = GemvT2Smem<double, UT, 8, ITT>;
  __shared__ double q_s[SMT::QS];
  __shared__ double gred[SMT::RED];
  double* tile = reinterpret_cast<double*>(smem_raw);
  const uint32_t bar = smem_u32(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;
  const int64_t G = gridDim.x;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  unsigned long long tl = 0;
  auto mark = [&](int slot) {
    if (s.tdbg && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (slot >= 0) atomicAdd(s.tdbg + slot, now - tl);
      tl = now;
    }
  };
  mark(-1);
  auto Qcol = [&](int j) { return s.Q + (int64_t)j * s.ldq; };
  auto Pcol = [&](int j) { return s.P + (int64_t)j * s.ldp; };

  for (int i = s.i0; i <= s.i_end; ++i) {
    if (halted(s.st)) break;
    // w = A p_i, p_i = z / alpha_i stored to P[:, i-1] (bidiag.py:152)
    gemv_n2_body<double, 4, 8, 0, true>(s.A, s.lda, s.mloc, s.nvec, s.nchunks, s.nseg, s.z,
                                        s.alpha + i, Pcol(i - 1), s.n, s.part_n, gw);
    grid.sync();
    mark(0);
    // CGS2 against Q[:, :i] (chunk sums - alpha_i q_i fused); beta_{i+1}
    CgsCoopArgs a{};
    a.B = s.Q;
    a.ldb = s.ldq;
    a.ncols = i;
    a.x = s.w;
    a.L = s.mloc;
    a.rows_per_cta = s.rows_l;
    a.passes = s.passes;
    a.eps = s.eps;
    a.slot = s.beta + i + 1;
    a.st = s.st;
    a.step = i;
    a.code = ST_BETA_BREAK;
    a.hp = s.hp;
    a.side = 0;
    a.part = s.lpart;
    a.c = s.lc;
    a.bar = s.lbar;
    a.fpart = s.part_n;
    a.fld = s.mloc;
    a.fnsplit = s.mloc > 0 ? s.nchunks : 0;
    a.fbeta = s.alpha + i;
    a.fp = Qcol(i - 1);
    a.redundant = G <= 160 && (int64_t)(i + 1) * G <= s.red_max;
    tile2_issue(a, tile, bar, false);
    tile2_rest<MAXE>(a, tile, tred, bar, parity, 0);
    parity ^= 1;
    grid.sync();
    mark(1);
    if (halted(s.st)) break;
    if (i == s.k_max) {  // q_{k+1} = w / beta; stop before alpha_{k+1} (bidiag.py:165-168)
      const double b = __ldcg(s.beta + i + 1);
      for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < s.mloc;
           r += G * kThreads)
        Qcol(i)[r] = __ldcg(s.w + r) / b;
      break;
    }
    // z = A^T q_{i+1}, q_{i+1} = w / beta stored to Q[:, i] (bidiag.py:169)
    for (int64_t vb = blockIdx.x; vb < s.ncoltiles * s.nsplit; vb += G)
      gemv_t2_body<double, UT, 8, ITT, true>(s.A, s.lda, s.mloc, s.nvec, s.w, s.beta + i + 1,
                                             Qcol(i), s.part_t, s.ldz, vb % s.ncoltiles,
                                             vb / s.ncoltiles, s.nsplit, q_s, gred);
    grid.sync();
    mark(2);
    // CGS2 against P[:, :i] (split sums - beta p_i fused); alpha_{i+1}
    a.B = s.P;
    a.ldb = s.ldp;
    a.x = s.z;
    a.L = s.n;
    a.rows_per_cta = s.rows_r;
    a.slot = s.alpha + i + 1;
    a.code = ST_ALPHA_BREAK;
    a.side = 1;
    a.part = s.rpart;
    a.c = s.rc;
    a.bar = s.rbar;
    a.fpart = s.part_t;
    a.fld = s.ldz;
    a.fnsplit = s.mloc > 0 ? (int)s.nsplit : 0;
    a.fbeta = s.beta + i + 1;
    a.fp = Pcol(i - 1);
    tile2_issue(a, tile, bar, false);
    tile2_rest<MAXE>(a, tile, tred, bar, parity, 0);
    parity ^= 1;
    grid.sync();
    mark(3);
  }
}

}  // namespace ksvd

namespace ksvd {

// ---------------------------------------------------------------------------
// k_gk_rows: the persistent step kernel with A STREAMED BY ROWS through a
// shared-memory ring of bulk (TMA) copies.  CTA b owns the rows of A, w, q
// and Q that its left CGS2 tile covers, and the entries of z, p and P its
// right CGS2 tile covers.  Per step:
//   A p   : each full row of A lands in the ring (one cp.async.bulk per row,
//           kRowRing rows in flight); w[r] = row . p (p in registers, 24
//           columns per thread) - alpha q[r]: a block reduction per row, no
//           chunk partials, no finalisation pass;
//   CGS2 of w (tile2_rest, no grid barrier before it: w rows are local);
//   A^T q : the same rows streamed again, acc[c] += row[c] q[r] for the
//           thread's 24 columns; one partial z per CTA;   -> grid barrier
//   z chunk = sum of the G partials of the owned columns - beta p (all 256
//           threads, fixed order), CGS2 of z (tile2_rest);  -> grid barrier
// 2 grid barriers per step besides the CGS2 rounds.  n <= 256 * 24.
constexpr int kRowRing = 4;
constexpr int kRowCols = 24;  // columns of p / z owned per thread

struct RowsArgs {
  const double* A;
  int64_t lda, mloc, n, ldz;
  double *Q, *P;
  int64_t ldq, ldp;
  double *w, *z, *alpha, *beta;
  double* zpart;  // G x ldz
  DevState* st;
  int i0, i_end, k_max, passes;
  double eps;
  int rows_l, rows_r;
  double *lpart, *lc, *rpart, *rc;
  unsigned *lbar, *rbar;
  int64_t red_max;
  HostProg* hp;
  size_t ring_off;  // doubles: the ring after the CGS tile region? (0: shared)
  unsigned long long* tdbg;
};

template <int MAXE>
__global__ void __launch_bounds__(kThreads, 1) k_gk_rows(RowsArgs s) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double tred[kWarps][32 * MAXE];
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ __align__(8) unsigned long long rbar[kRowRing];
  __shared__ double red8[2][kWarps];
  __shared__ double qrow[256];  // this CTA's q rows (rows_l <= 256)
  __shared__ double pown[256];  // this CTA's p entries (rows_r <= 256)
  __shared__ double zcomb[8][256];
  double* tile = reinterpret_cast<double*>(smem_raw);
  double* ring = tile;  // the ring and the CGS tile take turns in the same bytes
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t n = s.n;
  const int64_t ldr = (n + 1) & ~(int64_t)1;  // ring row pitch (16-byte rows)
  const uint32_t rowbytes = (uint32_t)(ldr * sizeof(double));
  const int64_t r0 = b * s.rows_l;
  const int nr = (int)max((int64_t)0, min((int64_t)s.rows_l, s.mloc - r0));
  const int64_t c0 = b * s.rows_r;
  const int nc = (int)max((int64_t)0, min((int64_t)s.rows_r, n - c0));
  const uint32_t bar = smem_u32(&mbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    for (int k = 0; k < kRowRing; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&rbar[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;       // tile barrier
  uint32_t rpar[kRowRing];   // ring barriers
#pragma unroll
  for (int k = 0; k < kRowRing; ++k) rpar[k] = 0;
  unsigned long long tl = 0;
  auto mark = [&](int slot) {
    if (s.tdbg && b == 0 && tid == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (slot >= 0) atomicAdd(s.tdbg + slot, now - tl);
      tl = now;
    }
  };
  mark(-1);
  auto issue_row = [&](int r) {  // thread 0: row r of this CTA into slot r % ring
    const int k = r % kRowRing;
    const uint32_t rb = smem_u32(&rbar[k]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rb),
                 "r"(rowbytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(ring + (size_t)k * ldr)),
        "l"(s.A + (r0 + r) * s.lda), "r"(rowbytes), "r"(rb)
        : "memory");
  };
  // stream this CTA's rows through the ring, calling f(r, row) for each
  auto stream_rows = [&](auto&& f) {
    if (tid == 0)
      for (int r = 0; r < nr && r < kRowRing; ++r) issue_row(r);
    for (int r = 0; r < nr; ++r) {
      const int k = r % kRowRing;
      while (!mbar_try_wait(smem_u32(&rbar[k]), rpar[k])) {
      }
      rpar[k] ^= 1;
      f(r, ring + (size_t)k * ldr);
      __syncthreads();  // the slot is free again
      if (tid == 0 && r + kRowRing < nr) issue_row(r + kRowRing);
    }
  };
  auto Qcol = [&](int j) { return s.Q + (int64_t)j * s.ldq; };
  auto Pcol = [&](int j) { return s.P + (int64_t)j * s.ldp; };
  double alpha = __ldcg(s.alpha + s.i0);
  // q_{i0} rows of this CTA (later steps keep q_i in qrow from the previous
  // step's normalisation): no global load on the per-row critical path
  for (int r = tid; r < nr; r += kThreads) qrow[r] = __ldcg(s.Q + (int64_t)(s.i0 - 1) * s.ldq + r0 + r);
  __syncthreads();

  for (int i = s.i0; i <= s.i_end; ++i) {
    // p_i = z / alpha_i: the thread's columns in registers, the owned chunk
    // to P[:, i-1] and pown
    double pv[kRowCols];
#pragma unroll
    for (int j = 0; j < kRowCols; ++j) {
      const int64_t c = tid + (int64_t)kThreads * j;
      pv[j] = c < n ? __ldcg(s.z + c) / alpha : 0.0;
    }
    for (int cc = tid; cc < nc; cc += kThreads) {
      const double v = __ldcg(s.z + c0 + cc) / alpha;
      pown[cc] = v;
      Pcol(i - 1)[c0 + cc] = v;
    }
    // w = A p_i - alpha_i q_i over this CTA's rows (bidiag.py:152)
    stream_rows([&](int r, const double* row) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < kRowCols; ++j) {
        const int64_t c = tid + (int64_t)kThreads * j;
        if (c < n) acc = fma(row[c], pv[j], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) red8[r & 1][warp] = acc;
      __syncthreads();
      if (tid == 0) {
        double t = red8[r & 1][0];
#pragma unroll
        for (int w8 = 1; w8 < kWarps; ++w8) t += red8[r & 1][w8];
        const double v = t - alpha * qrow[r];
        s.w[r0 + r] = v;
        flag_nonfinite(s.st, v, i);
      }
    });
    mark(0);
    // CGS2 of w against Q[:, :i]; beta_{i+1}
    CgsCoopArgs a{};
    a.B = s.Q;
    a.ldb = s.ldq;
    a.ncols = i;
    a.x = s.w;
    a.L = s.mloc;
    a.rows_per_cta = s.rows_l;
    a.passes = s.passes;
    a.eps = s.eps;
    a.slot = s.beta + i + 1;
    a.st = s.st;
    a.step = i;
    a.code = ST_BETA_BREAK;
    a.hp = s.hp;
    a.side = 0;
    a.part = s.lpart;
    a.c = s.lc;
    a.bar = s.lbar;
    a.fpart = nullptr;
    a.redundant = G <= 160 && (int64_t)(i + 1) * G <= s.red_max;
    tile2_issue(a, tile, bar, false);
    const double beta = sqrt(tile2_rest<MAXE>(a, tile, tred, bar, parity, 0));
    parity ^= 1;
    mark(1);
    if (!(beta >= s.eps)) break;  // beta break or non-finite (status set by CTA 0)
    // q_{i+1} = w / beta: this CTA's rows (Q[:, i] and qrow)
    for (int r = tid; r < nr; r += kThreads) {
      const double v = __ldcg(s.w + r0 + r) / beta;
      qrow[r] = v;
      Qcol(i)[r0 + r] = v;
    }
    __syncthreads();
    if (i == s.k_max) break;  // stop before alpha_{k+1} (bidiag.py:165-168)
    // A^T q_{i+1} over this CTA's rows: one partial z per CTA
    double zacc[kRowCols];
#pragma unroll
    for (int j = 0; j < kRowCols; ++j) zacc[j] = 0.0;
    stream_rows([&](int r, const double* row) {
      const double qv = qrow[r];
#pragma unroll
      for (int j = 0; j < kRowCols; ++j) {
        const int64_t c = tid + (int64_t)kThreads * j;
        if (c < n) zacc[j] = fma(row[c], qv, zacc[j]);
      }
    });
#pragma unroll
    for (int j = 0; j < kRowCols; ++j) {
      const int64_t c = tid + (int64_t)kThreads * j;
      if (c < n) s.zpart[b * s.ldz + c] = zacc[j];
    }
    grid.sync();
    mark(2);
    // z chunk = sum of the G partials - beta p_i: 8 thread groups split the
    // CTAs, combined in fixed order
    {
      const int grp = tid / 32;  // 8 groups of 32 threads: lanes over columns
      for (int cc = lane; cc < nc; cc += 32) {
        double t = 0.0;
        for (int64_t q = grp; q < G; q += kWarps) t += __ldcg(s.zpart + q * s.ldz + c0 + cc);
        zcomb[grp][cc] = t;
      }
      __syncthreads();
      for (int cc = tid; cc < nc; cc += kThreads) {
        double t = zcomb[0][cc];
#pragma unroll
        for (int g8 = 1; g8 < kWarps; ++g8) t += zcomb[g8][cc];
        const double v = t - beta * pown[cc];
        s.z[c0 + cc] = v;
        flag_nonfinite(s.st, v, i);
      }
      __syncthreads();
    }
    // CGS2 of z against P[:, :i]; alpha_{i+1}
    a.B = s.P;
    a.ldb = s.ldp;
    a.x = s.z;
    a.L = n;
    a.rows_per_cta = s.rows_r;
    a.slot = s.alpha + i + 1;
    a.code = ST_ALPHA_BREAK;
    a.side = 1;
    a.part = s.rpart;
    a.c = s.rc;
    a.bar = s.rbar;
    tile2_issue(a, tile, bar, false);
    alpha = sqrt(tile2_rest<MAXE>(a, tile, tred, bar, parity, 0));
    parity ^= 1;
    mark(3);
    if (!(alpha >= s.eps)) break;  // alpha break or non-finite
    grid.sync();  // every CTA's z chunk is in place for the next p
  }
}

}  // namespace ksvd
