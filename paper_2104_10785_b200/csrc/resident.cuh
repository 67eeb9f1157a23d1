// resident.cuh -- the whole GK loop of a small matrix in ONE cooperative
// kernel, with A resident in shared memory (included by ksvd.cu).
//
// For matrices whose row blocks fit the CTAs' shared memory (config 1:
// 2000 x 1000 f64 = 16 MB over 143 CTAs, 112 KB each) the step is latency-
// bound: four kernel launches and their fixed costs (~55 us per step)
// dwarf the 32 MB of L2 traffic.  Here CTA b keeps rows [b R, b R + R) of A,
// of the left basis Q and columns [b C, b C + C) of the right basis P in
// shared memory for the whole run; a step is
//   w = A p - alpha q   (local rows, p read from L2)
//   CGS2 of w against Q (2 grid rounds, beta^2 = ||w||^2 - ||c||^2 when
//                        that does not cancel -- as k_cgs2_tile2)
//   z partials over the CTA's rows for all n columns  -> 1 round
//   z chunk = sum of the partials - beta p (fixed order)
//   CGS2 of z against P (2 rounds), alpha, publish p   -> 1 round
// i.e. 6 grid barriers per step.  The paired step (a.paired, the arithmetic
// of pair.cuh: A^T runs on the finalised w before its CGS2, both CGS2 share
// grid rounds, alpha = ||y'|| / beta) needs 4:
//   w = A p - alpha q; z partials of A^T w and the left pass-1 dots -> 1 round
//   left update + pass-2 dots (+ norm); z chunk; right pass-1 dots    -> 1 round
//   left update, beta, q; right update + pass-2 dots (+ norm)         -> 1 round
//   right update, alpha, publish p                                    -> 1 round
// (plus a direct-norm round where the closed form would cancel).
// Semantics, scalars, breakdown codes and
// the residual left in R->w are those of the multi-kernel loop
// (bidiag.py:111-178), so ksvd_run_info / _extend / _ritz work unchanged.
#pragma once
#include <cfloat>
#include <cooperative_groups.h>

namespace ksvd {

struct ResArgs {
  const void* A;
  int64_t lda, m, n;
  int k_max, passes;
  int l;  // resume after a thick restart: Q[:, :l+1], P[:, :l] preloaded (0: fresh run)
  double eps;
  int R, C;  // rows / right-basis rows per CTA
  int kq;    // Q columns held in smem (k_max + 1)
  double *Q, *P;
  int64_t ldq, ldp;
  double *alpha, *beta;  // 1-based
  double* w_out;         // residual at a beta breakdown (ksvd_run_extend)
  double* pvec;          // current p (n)
  double* part;          // CGS partials: 4 x (kq + 1) x G (even-rounded blocks)
  double* zpart;         // gemv_t partials: G x n
  int paired;            // the paired step (pair.cuh's arithmetic, 4 grid rounds)
  DevState* st;
  unsigned long long* tdbg;  // KSVD_PHASE_TIMES: CTA-0 phase times (nullable)
};

template <typename TA>
__global__ void __launch_bounds__(kThreads, 1) k_gk_resident(ResArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char res_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t n = a.n;
  const int R = a.R, C = a.C;
  const int64_t r0 = (int64_t)b * R, c0 = (int64_t)b * C;
  const int nr = (int)max((int64_t)0, min((int64_t)R, a.m - r0));
  const int nc = (int)max((int64_t)0, min((int64_t)C, n - c0));
  // shared memory: doubles first (8-byte aligned), then A
  double* Qs = reinterpret_cast<double*>(res_smem);  // kq x R, column-major
  double* Ps = Qs + (size_t)a.kq * R;                 // k_max x C
  double* wv = Ps + (size_t)a.k_max * C;              // R
  double* zv = wv + R;                                // C
  double* red = zv + C;                               // kq + 2
  // bulk-copy targets on 16-byte boundaries (resident_smem_doubles)
  size_t off = ((size_t)a.kq * R + (size_t)a.k_max * C + R + C + a.kq + 2 + 1) & ~(size_t)1;
  double* pv = Qs + off;  // n: p of the step
  off += (size_t)(n + 1) & ~(size_t)1;
  double* stage = Qs + off;  // (kq + 1) x G partials
  off += (((size_t)(a.kq + 1) * G + 1) & ~(size_t)1) + 2;
  TA* As = reinterpret_cast<TA*>(Qs + off);  // nr x n, row-major
  const int64_t half = ((int64_t)(a.kq + 1) * G + 1) & ~(int64_t)1;  // 16-byte aligned halves
  int pp = 0;
  auto partb = [&](int k) { return a.part + (k & 1) * half; };
  // one mbarrier for the bulk (TMA) copies that stage L2 data in smem
  __shared__ __align__(8) unsigned long long rbar;
  const uint32_t bar = smem_u32(&rbar);
  uint32_t phase = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // dst (smem) <- src (global), 16-byte aligned, bytes % 16 == 0; data
  // written by other CTAs before the last grid barrier (generic proxy) is
  // ordered before the async-proxy read by fence.proxy.async
  auto bulk = [&](void* dst, const void* src, uint32_t bytes) {
    if (tid == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(smem_u32(dst)),
          "l"(src), "r"(bytes), "r"(bar)
          : "memory");
    }
    while (!mbar_try_wait(bar, phase)) {
    }
    phase ^= 1;
  };
  unsigned long long tl = 0;
  auto mark = [&](int slot) {
    if (a.tdbg && b == 0 && tid == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (slot >= 0) atomicAdd(a.tdbg + slot, now - tl);
      tl = now;
    }
  };
  mark(-1);

  {  // A rows and q_1 rows into shared memory
    const TA* Ag = reinterpret_cast<const TA*>(a.A) + r0 * a.lda;
    for (int64_t e = tid; e < (int64_t)nr * n; e += kThreads) {
      const int64_t r = e / n, c = e - r * n;
      As[e] = Ag[r * a.lda + c];
    }
    for (int j = 0; j <= a.l; ++j)
      for (int r = tid; r < nr; r += kThreads) Qs[(size_t)j * R + r] = a.Q[(int64_t)j * a.ldq + r0 + r];
    for (int j = 0; j < a.l; ++j)
      for (int cc = tid; cc < nc; cc += kThreads) Ps[(size_t)j * C + cc] = a.P[(int64_t)j * a.ldp + c0 + cc];
  }
  __syncthreads();
  mark(0);

  auto finish = [&](int status, int kprime) {
    if (b == 0 && tid == 0) {
      a.st->status = status;
      a.st->kprime = kprime;
      a.st->where = kprime;
    }
  };
  // this CTA's dots basis^T x -> P[j*G + b]; optionally ||x||^2 -> P[ncols*G + b]
  auto dots = [&](const double* basis, int ld, int ncols, const double* x, int len, double* P,
                  bool with_norm) {
    for (int j = warp; j < ncols; j += kWarps) {
      double s = 0.0;
      for (int t = lane; t < len; t += 32) s = fma(basis[(size_t)j * ld + t], x[t], s);
      s = warp_sum(s);
      if (lane == 0) P[(int64_t)j * G + b] = s;
    }
    if (with_norm && warp == kWarps - 1) {
      double s = 0.0;
      for (int t = lane; t < len; t += 32) s = fma(x[t], x[t], s);
      s = warp_sum(s);
      if (lane == 0) P[(int64_t)ncols * G + b] = s;
    }
  };
  // red[j] = sum_b' P[j*G + b'], same fixed order in every CTA: the block
  // is first copied to shared memory with every load in flight at once
  // (one L2 round trip), then summed there
  auto reduce = [&](const double* P, int j0, int j1) {
    const int64_t base = (int64_t)j0 * G, cnt = (int64_t)(j1 - j0) * G;
    if ((base & 1) == 0) {  // one bulk copy (the partial block is contiguous)
      bulk(stage, P + base, (uint32_t)(((cnt + 1) & ~(int64_t)1) * sizeof(double)));
    } else {
#pragma unroll 4
      for (int64_t e = tid; e < cnt; e += kThreads) stage[e] = __ldcg(P + base + e);
    }
    __syncthreads();
    for (int j = j0 + warp; j < j1; j += kWarps) {
      double s = 0.0;
      for (int q = lane; q < G; q += 32) s += stage[(int64_t)(j - j0) * G + q];
      s = warp_sum(s);
      if (lane == 0) red[j] = s;
    }
    __syncthreads();
  };
  auto update = [&](const double* basis, int ld, int ncols, double* x, int len) {
    for (int t = tid; t < len; t += kThreads) {
      double s = 0.0;
      for (int j = 0; j < ncols; ++j) s = fma(basis[(size_t)j * ld + t], red[j], s);
      x[t] -= s;
    }
    __syncthreads();
  };
  // x <- x orthogonalised (CGS2) against basis[:, :ncols]; returns ||x||^2
  // (identical in every CTA)
  auto cgs2 = [&](const double* basis, int ld, int ncols, double* x, int len) -> double {
    if (ncols == 0 || a.passes == 0) {
      dots(basis, ld, 0, x, len, partb(pp), true);
      grid.sync();
      reduce(partb(pp), 0, 1);
      ++pp;
      return red[0];
    }
    dots(basis, ld, ncols, x, len, partb(pp), a.passes == 1);
    for (int pass = 1;; ++pass) {
      const bool last = pass == a.passes;
      grid.sync();
      reduce(partb(pp), 0, ncols + (last ? 1 : 0));
      ++pp;
      if (!last) {
        update(basis, ld, ncols, x, len);
        dots(basis, ld, ncols, x, len, partb(pp), pass + 1 == a.passes);
        continue;
      }
      double cc = 0.0;  // same fixed order in every warp (lane strides + butterfly)
      for (int j = (int)(threadIdx.x & 31); j < ncols; j += 32) cc = fma(red[j], red[j], cc);
      cc = warp_sum(cc);
      const double nn = red[ncols];
      update(basis, ld, ncols, x, len);
      if (cc <= 1e-6 * nn) return nn - cc;
      dots(basis, ld, 0, x, len, partb(pp), true);
      grid.sync();
      reduce(partb(pp), 0, 1);
      ++pp;
      return red[0];
    }
  };
  // z partials over this CTA's rows (all n columns), then after the barrier
  // z chunk = sum of the partials - beta pprev
  auto gemv_t = [&](const double* qv, const double* pprev, double beta) {
    double* zp = a.zpart + (int64_t)b * n;
    for (int64_t c = tid; c < n; c += kThreads) {
      double s = 0.0;
      for (int r = 0; r < nr; ++r) s = fma((double)As[(int64_t)r * n + c], qv[r], s);
      zp[c] = s;
    }
    grid.sync();
    for (int cc = warp; cc < nc; cc += kWarps) {
      double s = 0.0;
      for (int q = lane; q < G; q += 32) s += __ldcg(a.zpart + (int64_t)q * n + c0 + cc);
      s = warp_sum(s);
      if (lane == 0) zv[cc] = pprev ? s - beta * pprev[cc] : s;
    }
    __syncthreads();
  };
  auto publish_p = [&](int col, double alpha) {
    for (int cc = tid; cc < nc; cc += kThreads) {
      const double v = zv[cc] / alpha;
      Ps[(size_t)col * C + cc] = v;
      a.P[(int64_t)col * a.ldp + c0 + cc] = v;
      a.pvec[c0 + cc] = v;
    }
    grid.sync();
  };

  // z = A^T q_{l+1}; alpha_{l+1} = ||z|| after CGS2 against the l kept
  // right vectors (l = 0: the first product, bidiag.py:139-147; l > 0: the
  // resumed loop of ksvd_run_restart)
  const int l = a.l;
  gemv_t(Qs + (size_t)l * R, nullptr, 0.0);
  double nrm2 = cgs2(Ps, C, l, zv, nc);
  double alpha = sqrt(nrm2);
  if (!isfinite(alpha)) return finish(ST_NONFINITE, l);
  if (alpha < a.eps) return finish(l == 0 ? ST_DEGENERATE : ST_ALPHA_BREAK, l);
  if (b == 0 && tid == 0) a.alpha[l + 1] = alpha;
  publish_p(l, alpha);

  const int64_t hblk = ((int64_t)(a.kq + 1) * G + 1) & ~(int64_t)1;
  double* const PL0 = a.part;             // paired step: left / right partial blocks
  double* const PL1 = a.part + hblk;
  double* const PR0 = a.part + 2 * hblk;
  double* const PR1 = a.part + 3 * hblk;
  // ||c||^2 of red[0:ncols] (the same fixed order in every warp of every CTA)
  auto ccnorm = [&](int ncols) {
    double cc = 0.0;
    for (int j = (int)(threadIdx.x & 31); j < ncols; j += 32) cc = fma(red[j], red[j], cc);
    return warp_sum(cc);
  };

  for (int i = l + 1; i <= a.k_max; ++i) {
    // w = A p_i - alpha_i q_i (bidiag.py:152); p staged in shared memory
    bulk(pv, a.pvec, (uint32_t)(((n + 1) & ~(int64_t)1) * sizeof(double)));
    for (int r = warp; r < nr; r += kWarps) {
      double s = 0.0;
      const TA* row = As + (int64_t)r * n;
      for (int64_t c = lane; c < n; c += 32) s = fma((double)row[c], pv[c], s);
      s = warp_sum(s);
      if (lane == 0) wv[r] = s - alpha * Qs[(size_t)(i - 1) * R + r];
    }
    __syncthreads();
    mark(1);
    if (a.paired && i < a.k_max) {
      // [round 1] y partials = A^T w over this CTA's rows; left pass-1 dots
      {
        double* zp = a.zpart + (int64_t)b * n;
        for (int64_t c = tid; c < n; c += kThreads) {
          double s = 0.0;
          for (int r = 0; r < nr; ++r) s = fma((double)As[(int64_t)r * n + c], wv[r], s);
          zp[c] = s;
        }
      }
      dots(Qs, R, i, wv, nr, PL0, false);
      grid.sync();
      // [round 2] left update + pass-2 dots and norm; y chunk; right pass-1 dots
      reduce(PL0, 0, i);
      update(Qs, R, i, wv, nr);
      dots(Qs, R, i, wv, nr, PL1, true);
      for (int cc = warp; cc < nc; cc += kWarps) {
        double s = 0.0;
        for (int q = lane; q < G; q += 32) s += __ldcg(a.zpart + (int64_t)q * n + c0 + cc);
        s = warp_sum(s);
        if (lane == 0) zv[cc] = s;
      }
      __syncthreads();
      dots(Ps, C, i, zv, nc, PR0, false);
      grid.sync();
      // [round 3] left update, beta (closed form); right update + pass-2 dots
      reduce(PL1, 0, i + 1);
      const double ccl = ccnorm(i), nnl = red[i];
      update(Qs, R, i, wv, nr);
      const bool dir_l = !(ccl <= 1e-6 * nnl);
      reduce(PR0, 0, i);
      update(Ps, C, i, zv, nc);
      dots(Ps, C, i, zv, nc, PR1, true);
      if (dir_l) dots(Qs, R, 0, wv, nr, PL0, true);  // direct norm (rare)
      grid.sync();
      double n2l = nnl - ccl;
      if (dir_l) {
        reduce(PL0, 0, 1);
        n2l = red[0];
      }
      const double beta = sqrt(n2l);
      if (!isfinite(beta)) return finish(ST_NONFINITE, i);
      if (b == 0 && tid == 0) a.beta[i + 1] = beta;
      if (beta < a.eps) {  // bidiag.py:158-164: the residual stays for _terminal_column
        for (int r = tid; r < nr; r += kThreads) a.w_out[r0 + r] = wv[r];
        return finish(ST_BETA_BREAK, i);
      }
      for (int r = tid; r < nr; r += kThreads) {
        const double v = wv[r] / beta;
        Qs[(size_t)i * R + r] = v;
        a.Q[(int64_t)i * a.ldq + r0 + r] = v;
      }
      // [round 4] right update, alpha = ||y'|| / beta, publish p = y' / ||y'||
      reduce(PR1, 0, i + 1);
      const double ccr = ccnorm(i), nnr = red[i];
      update(Ps, C, i, zv, nc);
      double n2r = nnr - ccr;
      if (!(ccr <= 1e-6 * nnr)) {  // direct norm (rare): one more round
        dots(Ps, C, 0, zv, nc, PR0, true);
        grid.sync();
        reduce(PR0, 0, 1);
        n2r = red[0];
      }
      const double ynrm = sqrt(n2r);
      alpha = ynrm / beta;
      if (!isfinite(alpha)) return finish(ST_NONFINITE, i);
      if (b == 0 && tid == 0) a.alpha[i + 1] = alpha;
      if (alpha < a.eps) return finish(ST_ALPHA_BREAK, i);
      // p = y' / ||y'|| (publish_p divides its zv by the scale it is given)
      publish_p(i, ynrm);
      mark(5);
      continue;
    }
    nrm2 = cgs2(Qs, R, i, wv, nr);
    mark(2);
    const double beta = sqrt(nrm2);
    if (!isfinite(beta)) return finish(ST_NONFINITE, i);
    if (b == 0 && tid == 0) a.beta[i + 1] = beta;
    if (beta < a.eps) {  // bidiag.py:158-164: the residual stays for _terminal_column
      for (int r = tid; r < nr; r += kThreads) a.w_out[r0 + r] = wv[r];
      return finish(ST_BETA_BREAK, i);
    }
    for (int r = tid; r < nr; r += kThreads) {
      const double v = wv[r] / beta;
      Qs[(size_t)i * R + r] = v;
      a.Q[(int64_t)i * a.ldq + r0 + r] = v;
    }
    __syncthreads();
    if (i == a.k_max) return;  // stop before alpha_{k+1} (bidiag.py:166-168)
    // z = A^T q_{i+1} - beta p_i, CGS2 against P[:, :i] (bidiag.py:169-178)
    gemv_t(Qs + (size_t)i * R, Ps + (size_t)(i - 1) * C, beta);
    mark(3);
    nrm2 = cgs2(Ps, C, i, zv, nc);
    mark(4);
    alpha = sqrt(nrm2);
    if (!isfinite(alpha)) return finish(ST_NONFINITE, i);
    if (b == 0 && tid == 0) a.alpha[i + 1] = alpha;
    if (alpha < a.eps) return finish(ST_ALPHA_BREAK, i);
    publish_p(i, alpha);
    mark(5);
  }
}

}  // namespace ksvd

namespace ksvd {

// The U filter of fsvd (fsvd.py:142-155: CGS2 of each column against the
// kept ones, cut everything from the first residual norm < cut) for a
// single-rank U that fits one CTA's shared memory: one launch instead of
// ~5 per column.  Status ST_CUT with kprime = first dropped column,
// ST_NONFINITE on a non-finite norm; columns are normalised in place.
constexpr int kUfThreads = 1024, kUfWarps = kUfThreads / 32;
__global__ void __launch_bounds__(kUfThreads, 1)
k_ufilter_small(double* __restrict__ U, int64_t ldu, int m, int take, int ldm, double cut,
                DevState* st) {
  extern __shared__ __align__(16) double uf_smem[];
  double* Us = uf_smem;                    // take x ldm, column-major
  double* coef = Us + (size_t)take * ldm;  // take
  __shared__ double red[kUfWarps];
  __shared__ __align__(8) unsigned long long ubar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // U into shared memory: one bulk copy per column (ldu, ldm even: 16-byte
  // aligned columns), all in flight on one mbarrier
  const uint32_t bar = smem_u32(&ubar);
  const uint32_t cbytes = (uint32_t)(((m + 1) & ~1) * sizeof(double));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(cbytes * (uint32_t)take)
                 : "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int t = lane; t < take; t += 32)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(smem_u32(Us + (size_t)t * ldm)),
          "l"(U + (int64_t)t * ldu), "r"(cbytes), "r"(bar)
          : "memory");
  while (!mbar_try_wait(bar, 0)) {
  }
  int good = take, status = ST_RUNNING;
  for (int t = 0; t < take; ++t) {
    double* u = Us + (size_t)t * ldm;
    for (int pass = 0; pass < 2 && t > 0; ++pass) {
      for (int j = warp; j < t; j += kUfWarps) {
        const double* q = Us + (size_t)j * ldm;
        double s4[4] = {0.0, 0.0, 0.0, 0.0};  // 4 chains: latency, fixed order
        int r = lane;
        for (; r + 96 < m; r += 128)
#pragma unroll
          for (int k = 0; k < 4; ++k) s4[k] = fma(q[r + 32 * k], u[r + 32 * k], s4[k]);
        for (; r < m; r += 32) s4[0] = fma(q[r], u[r], s4[0]);
        const double s = warp_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
        if (lane == 0) coef[j] = s;
      }
      __syncthreads();
      for (int r = tid; r < m; r += kUfThreads) {
        double s = 0.0;
        for (int j = 0; j < t; ++j) s = fma(Us[(size_t)j * ldm + r], coef[j], s);
        u[r] -= s;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int r = tid; r < m; r += kUfThreads) s = fma(u[r], u[r], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double nn = red[0];
    for (int w = 1; w < kUfWarps; ++w) nn += red[w];
    const double nrm = sqrt(nn);
    __syncthreads();
    if (!isfinite(nrm)) {
      status = ST_NONFINITE;
      good = t;
      break;
    }
    if (nrm < cut) {
      status = ST_CUT;
      good = t;
      break;
    }
    for (int r = tid; r < m; r += kUfThreads) u[r] /= nrm;
    __syncthreads();
  }
  for (int t = 0; t < good; ++t)
    for (int r = tid; r < m; r += kUfThreads) U[(int64_t)t * ldu + r] = Us[(size_t)t * ldm + r];
  if (tid == 0 && status != ST_RUNNING) {
    st->status = status;
    st->kprime = good;
    st->where = good;
  }
}

}  // namespace ksvd

namespace ksvd {

// Y[:, t] = (A X[:, t]) / sigma[t] for small row counts (k_multi_rhs tiles
// 256 rows per CTA, i.e. too few CTAs below ~40k rows): one warp per row,
// lanes stride the columns, up to 32 right-hand sides in registers, fixed
// order.  Used for config 1-sized U = A V (fsvd.py:192-194).
template <typename TA>
__global__ void __launch_bounds__(kThreads, 1)
k_multi_rhs_rows(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                 const double* __restrict__ X, int64_t ldx, int k,
                 const double* __restrict__ sigma, double* __restrict__ Y, int64_t ldy,
                 int rows_per_cta) {
  extern __shared__ __align__(16) double xs[];  // k x ldx (X columns)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ __align__(8) unsigned long long xbar;
  const uint32_t bar = smem_u32(&xbar);
  const uint32_t bytes = (uint32_t)((int64_t)k * ldx * sizeof(double));  // ldx even
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(xs)),
        "l"(X), "r"(bytes), "r"(bar)
        : "memory");
  }
  __syncthreads();
  while (!mbar_try_wait(bar, 0)) {
  }
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(m, r0 + rows_per_cta);
  for (int64_t r = r0 + warp; r < r1; r += kWarps) {
    double acc[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) acc[t] = 0.0;
    const TA* row = A + r * lda;
    for (int64_t c0 = lane; c0 < n; c0 += 32 * 8) {
      double av[8];  // 8 independent row loads in flight
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t c = c0 + 32 * u;
        av[u] = c < n ? (double)row[c] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t c = c0 + 32 * u;
        if (c >= n) break;
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (t < k) acc[t] = fma(av[u], xs[(int64_t)t * ldx + c], acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (t >= k) break;
      const double v = warp_sum(acc[t]);
      if (lane == 0) Y[(int64_t)t * ldy + r] = sigma ? v / sigma[t] : v;
    }
  }
}

}  // namespace ksvd

namespace ksvd {

// Dense SVD T = U diag(s) V^T of the restarted mode's small projected
// matrix in ONE CTA (north star (d): "the tiny SVD on the host or in a
// single-CTA kernel"): one-sided Jacobi with the round-robin (circle)
// ordering, so the k/2 column pairs of a round rotate in parallel, one warp
// per pair.  W = T and V live in shared memory; converged when a whole
// sweep made no rotation (|g| <= k eps sqrt(a b), columns below eps ||T||_F
// count as zero -- the host ksvd_dense_svd rule).  Output sorted descending,
// U[:, j] = W[:, j] / s_j (0 for s_j = 0).  Fixed order: deterministic.
constexpr int kSvdThreads = 1024, kSvdWarps = kSvdThreads / 32;
__global__ void __launch_bounds__(kSvdThreads, 1)
k_dense_svd_cta(int k, const double* __restrict__ T, double* __restrict__ U,
                double* __restrict__ s, double* __restrict__ V, int* __restrict__ info) {
  extern __shared__ __align__(16) double sv_smem[];
  const int kk = (k + 1) & ~1;  // even number of players (a dummy when k is odd)
  double* W = sv_smem;                 // kk x k, column-major (ld = k)
  double* Vm = W + (size_t)kk * k;     // kk x k
  double* nrm = Vm + (size_t)kk * k;   // kk
  __shared__ int rotated;
  __shared__ double fro2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < kk * k; e += kSvdThreads) {
    const int j = e / k, i = e - j * k;
    W[e] = j < k ? T[(size_t)j * k + i] : 0.0;
    Vm[e] = (j < k && i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int e = lane; e < k * k; e += 32) t = fma(W[e], W[e], t);
    t = warp_sum(t);
    if (lane == 0) fro2 = t;
  }
  __syncthreads();
  const double tol = fmax(1e-15, (double)k * DBL_EPSILON);
  const double zero2 = fro2 * DBL_EPSILON * DBL_EPSILON;
  int sweep = 0;
  for (; sweep < 80; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < kk - 1; ++r) {
      for (int slot = warp; slot < kk / 2; slot += kSvdWarps) {
        auto elem = [&](int j) { return j == 0 ? 0 : 1 + (j - 1 + r) % (kk - 1); };
        int p = elem(slot), q = elem(kk - 1 - slot);
        if (p > q) {
          const int x = p;
          p = q;
          q = x;
        }
        if (q >= k) continue;  // the dummy player
        double* wp = W + (size_t)p * k;
        double* wq = W + (size_t)q * k;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < k; i += 32) {
          a = fma(wp[i], wp[i], a);
          b = fma(wq[i], wq[i], b);
          g = fma(wp[i], wq[i], g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (g == 0.0 || a <= zero2 || b <= zero2 || fabs(g) <= tol * sqrt(a * b)) continue;
        if (lane == 0) rotated = 1;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        double* vp = Vm + (size_t)p * k;
        double* vq = Vm + (size_t)q * k;
        for (int i = lane; i < k; i += 32) {
          const double x = wp[i], y = wq[i];
          wp[i] = c * x - sn * y;
          wq[i] = sn * x + c * y;
          const double u = vp[i], v = vq[i];
          vp[i] = c * u - sn * v;
          vq[i] = sn * u + c * v;
        }
      }
      __syncthreads();
    }
    const bool any = rotated != 0;
    __syncthreads();
    if (!any) break;
  }
  for (int j = warp; j < k; j += kSvdWarps) {
    double t = 0.0;
    for (int i = lane; i < k; i += 32) t = fma(W[(size_t)j * k + i], W[(size_t)j * k + i], t);
    t = warp_sum(t);
    if (lane == 0) nrm[j] = sqrt(t);
  }
  __syncthreads();
  // descending order, ties by index (the host rule); k <= ~110: rank by count
  for (int j = tid; j < k; j += kSvdThreads) {
    int rank = 0;
    for (int o = 0; o < k; ++o)
      if (nrm[o] > nrm[j] || (nrm[o] == nrm[j] && o < j)) ++rank;
    s[rank] = nrm[j];
    for (int i = 0; i < k; ++i) {
      U[(size_t)rank * k + i] = nrm[j] > 0 ? W[(size_t)j * k + i] / nrm[j] : 0.0;
      V[(size_t)rank * k + i] = Vm[(size_t)j * k + i];
    }
  }
  if (tid == 0) *info = sweep;
}

}  // namespace ksvd
