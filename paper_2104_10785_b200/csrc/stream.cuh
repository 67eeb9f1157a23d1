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
