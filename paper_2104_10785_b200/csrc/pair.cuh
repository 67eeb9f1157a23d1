// pair.cuh -- both CGS2 orthogonalisations of a GK step in ONE grid-
// synchronised kernel (k_cgs2_pair), sharing its grid rounds.
//
// The serialised step runs  A p_i -> CGS2(w, Q_i) -> A^T q_{i+1} -> CGS2(z, P_i):
// two grid-synchronised kernels of 2-4 grid rounds each, latency-bound
// (DESIGN.md section 3).  The paired step feeds the A^T product the
// finalised but NOT yet orthogonalised w = A p_i - alpha_i q_i and then runs
// both CGS2 together:
//
//   left   w' = w - Q_i d  (CGS2),                beta_{i+1} = ||w'||,  q_{i+1} = w' / beta
//   right  y  = A^T w  (the product's partials),  y' = y - P_i c  (CGS2),
//          alpha_{i+1} = ||y'|| / beta_{i+1},     p_{i+1} = y' / ||y'||
//
// In exact arithmetic y = beta A^T q_{i+1} + A^T Q_i d, and A^T Q_i d lies in
// span(P_i) by the GK relations A^T q_j = alpha_j p_j + beta_j p_{j-1}, as does
// beta_{i+1} p_i; the CGS2 against P_i removes both, leaving
// beta alpha_{i+1} p_{i+1} -- the reference's z' (bidiag.py:169-176) times
// beta.  The rounding of A^T w is eps ||A|| ||w|| ~ eps ||A|| beta, so relative
// to ||y'|| = beta alpha it is eps ||A|| / alpha, the order of the reference's
// own z = A^T q - beta p; d is the usual O(eps ||A||) loss of orthogonality, so
// what the GK relations miss (eps^2) is far below it.  Nothing compounds:
// every product reads the previous step's CLEAN p_i.
//
// The CTAs split into a left group (rows of Q / w) and a right group (rows
// of P / y) in proportion to the rows; every CTA bulk-copies its own side's
// basis tile into shared memory and runs the sweeps of k_cgs2_tile2 on it.
// The reductions of both sides run in the same grid rounds: 2 rounds for
// the pair (redundant reductions: every CTA sums both sides' partials) or 4
// (distributed column sums), instead of 2 x (2 or 4) for two kernels.
// Used with two CGS passes only (reorth_passes=2, the default): one classical
// pass against a basis that is orthonormal only to working precision would
// leave a fraction of beta^2 p_i and A^T Q d behind.
// Every CTA ends with both reduced coefficient vectors, so the closed-form
// norm test (||x||^2 - ||c||^2, a direct-norm round where it would cancel)
// is decided identically everywhere.
#pragma once
#include "kernels.cuh"

namespace ksvd {

struct PairSide {
  const double* B;  // basis, column-major (ldb), ncols columns
  int64_t ldb;
  int ncols;
  const double* x;  // left: the finalised w (read); right: null (y from fpart)
  int64_t L;        // rows
  int rows;         // rows per CTA (even)
  int G;            // CTAs of this side
  const double* fpart;  // right: the product's split partial sums y = sum_s fpart[s*fld + r]
  int64_t fld;
  int fnsplit;
  double* part;  // 2 x (ncols + 1) x G partial sums (ping-pong)
  double* c;     // ncols + 1 reduced sums (distributed mode)
  double* out;   // the normalised result (q_{i+1} / p_{i+1}); not written on a breakdown
};

struct PairArgs {
  PairSide s[2];
  int passes;
  double eps;
  double* beta_slot;   // beta_{i+1}
  double* alpha_slot;  // alpha_{i+1}
  DevState* st;
  int step;
  HostProg* hp;
  unsigned* bar;  // flip barrier word (nullptr: cooperative grid sync)
  int redundant;
};

template <int MAXE>
__global__ void __launch_bounds__(kThreads, 1)
k_cgs2_pair(PairArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double tred[kWarps][32 * MAXE];
  __shared__ __align__(8) unsigned long long mbar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  const int side = (int)blockIdx.x < a.s[0].G ? 0 : 1;
  const PairSide& S = a.s[side];
  const int lb = (int)blockIdx.x - (side ? a.s[0].G : 0);  // CTA index within the side
  const int64_t s0 = (int64_t)lb * S.rows;
  const int64_t s1 = min(S.L, s0 + S.rows);
  const int nr = s1 > s0 ? (int)(s1 - s0) : 0;
  const int ldt = (nr + 1) & ~1;
  double* tile = reinterpret_cast<double*>(smem_raw);
  // both sides' reduced sums (every CTA holds both): ncols + 1 each
  size_t tile_elems = 0;
  for (int sd = 0; sd < 2; ++sd) {
    const int64_t r = a.s[sd].rows;
    tile_elems = max(tile_elems, (size_t)a.s[sd].ncols * (size_t)r);
  }
  double* redv[2];
  redv[0] = tile + tile_elems;
  redv[1] = redv[0] + (a.s[0].ncols + 1);
  const uint32_t bar = smem_u32(&mbar);

  // bulk copy of this CTA's basis tile (columns written >= 2 launches back:
  // may run ahead of the programmatic-launch wait)
  const uint32_t bytes = (uint32_t)ldt * 8u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(bytes * (uint32_t)S.ncols)
                 : "memory");
  }
  __syncthreads();
  if (bytes) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int j = threadIdx.x; j < S.ncols; j += kThreads)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(smem_u32(tile + (size_t)j * ldt)),
          "l"(S.B + (int64_t)j * S.ldb + s0), "r"(bytes), "r"(bar)
          : "memory");
  }
  pdl_wait();

  // [0] this CTA's rows of x: w (left, finalised by k_gemv_n_finalize) or
  // y = the A^T product's split sums (right), all loads in flight with the
  // run status; staged through shared memory into the per-warp registers
  double* xs = &tred[0][0];
  const int st0 = *reinterpret_cast<const volatile int*>(&a.st->status);
  {
    const int64_t r = s0 + threadIdx.x;
    if (r < s1) {
      const double v = S.fpart ? strided_sum(S.fpart + r, S.fld, S.fnsplit) : __ldcg(S.x + r);
      if (st0 == ST_RUNNING) flag_nonfinite(a.st, v, a.step);
      xs[threadIdx.x] = v;
    }
  }
  if (st0 != ST_RUNNING) {  // same value in every thread of every CTA
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

  const int64_t half0 = (int64_t)(a.s[0].ncols + 1) * a.s[0].G;
  const int64_t half1 = (int64_t)(a.s[1].ncols + 1) * a.s[1].G;
  auto partp = [&](int sd, int k) {
    return a.s[sd].part + (k & 1) * (sd ? half1 : half0);
  };
  double* red = redv[side];

  // xv -= tile * red[0:ncols]
  auto update = [&]() {
    double t[MAXE];
#pragma unroll
    for (int e = 0; e < MAXE; ++e) t[e] = 0.0;
#pragma unroll 4
    for (int j = warp; j < S.ncols; j += kWarps) {
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
    }
    __syncthreads();
  };
  // ||xv||^2 of this CTA's rows -> P[ncols*G_s + lb]
  auto norm_part = [&](double* P) {
    if (warp == kWarps - 1) {
      double s = 0.0;
#pragma unroll
      for (int e = 0; e < MAXE; ++e) s = fma(xv[e], xv[e], s);
      s = warp_sum(s);
      if (lane == 0) P[(int64_t)S.ncols * S.G + lb] = s;
    }
  };
  // partial dots tile^T xv -> P[j*G_s + lb] (and the norm partial)
  auto dot = [&](double* P, bool with_norm) {
    {
      for (int q0 = 0; warp + kWarps * q0 < S.ncols; q0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = warp + kWarps * (q0 + u);
          v[u] = 0.0;
          if (j < S.ncols) {
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
        if ((lane & 3) == 0 && j < S.ncols) P[(int64_t)j * S.G + lb] = t;
      }
    }
    if (with_norm) norm_part(P);
  };
  // redv[sd][j] = sum_b P_sd[j*G_sd + b] for j in [j0, j1) of BOTH sides, the
  // same fixed order in every CTA.  Redundant: each CTA sums every column
  // itself (4 columns per warp, 4 x 5 loads in flight, G_sd <= 160);
  // distributed: the grid's warps split the columns of both sides into
  // s.c, one barrier, every CTA copies both.
  unsigned long long bk = 0;
  // norm_only: just the norm rows (column ncols of each side)
  auto reduce_both = [&](int k, bool with_norm, bool norm_only) {
    const int j00 = norm_only ? a.s[0].ncols : 0, j01 = norm_only ? a.s[1].ncols : 0;
    const int n0 = a.s[0].ncols + (with_norm ? 1 : 0) - j00;
    const int n1 = a.s[1].ncols + (with_norm ? 1 : 0) - j01;
    if (a.redundant) {
      for (int q = 4 * warp; q < n0 + n1; q += 4 * kWarps) {
        double sacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int g = q + u;
          if (g >= n0 + n1) break;
          const int sd = g < n0 ? 0 : 1;
          const int j = sd ? j01 + g - n0 : j00 + g;
          const double* P = partp(sd, k) + (int64_t)j * a.s[sd].G;
          const unsigned Gs = (unsigned)a.s[sd].G;
#pragma unroll
          for (int kk = 0; kk < 5; ++kk) {
            const unsigned b = lane + 32 * kk;
            if (b < Gs) sacc[u] += __ldcg(P + b);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int g = q + u;
          const double t = warp_sum(sacc[u]);
          if (lane == 0 && g < n0 + n1) {
            const int sd = g < n0 ? 0 : 1;
            redv[sd][sd ? j01 + g - n0 : j00 + g] = t;
          }
        }
      }
    } else {
      const int gw = blockIdx.x * kWarps + warp, nw = (int)G * kWarps;
      for (int g = gw; g < n0 + n1; g += nw) {
        const int sd = g < n0 ? 0 : 1;
        const int j = sd ? j01 + g - n0 : j00 + g;
        const double* p = partp(sd, k) + (int64_t)j * a.s[sd].G;
        const unsigned Gs = (unsigned)a.s[sd].G;
        double t = 0.0;
        for (unsigned b0 = 0; b0 < Gs; b0 += 160) {
          double v[5];
#pragma unroll
          for (int kk = 0; kk < 5; ++kk) {
            const unsigned b = b0 + lane + 32 * kk;
            v[kk] = b < Gs ? __ldcg(p + b) : 0.0;
          }
#pragma unroll
          for (int kk = 0; kk < 5; ++kk)
            if (b0 + lane + 32 * kk < Gs) t += v[kk];
        }
        t = warp_sum(t);
        if (lane == 0) a.s[sd].c[j] = t;
      }
      ++bk;
      grid_barrier_raw(a.bar, G);
      for (int g = threadIdx.x; g < n0 + n1; g += kThreads) {
        const int sd = g < n0 ? 0 : 1;
        const int j = sd ? j01 + g - n0 : j00 + g;
        redv[sd][j] = __ldcg(a.s[sd].c + j);
      }
    }
    __syncthreads();
  };
  // ||c||^2 of side sd's reduced coefficients (lane-strided partial sums +
  // a butterfly: the same order in every warp of every CTA)
  auto ccnorm = [&](int sd) {
    double cc = 0.0;
    for (int j = lane; j < a.s[sd].ncols; j += 32) cc = fma(redv[sd][j], redv[sd][j], cc);
    return warp_sum(cc);
  };

  const int P = a.passes;
  double n2[2] = {0.0, 0.0};
  bool direct[2] = {false, false};
  // passes k = 0 .. P-1 (the norms ride on the last), then a direct-norm
  // round for a side whose closed form would cancel
  for (int k = 0; k < P; ++k) {
    const bool last = k + 1 == P;
    dot(partp(side, k), last);
    ++bk;
    grid_barrier_raw(a.bar, G);
    reduce_both(k, last, false);
    if (last)
      for (int sd = 0; sd < 2; ++sd) {
        const double cc = ccnorm(sd), nn = redv[sd][a.s[sd].ncols];
        // ||x - B c||^2 = ||x||^2 - ||c||^2 for an orthonormal B: exact to
        // rounding while ||c||^2 <= 1e-6 ||x||^2 (after a first pass, away
        // from breakdown); otherwise (or non-finite) the direct norm
        direct[sd] = !(cc <= 1e-6 * nn);
        n2[sd] = nn - cc;
      }
    update();
  }
  if (direct[0] || direct[1]) {
    norm_part(partp(side, P));
    ++bk;
    grid_barrier_raw(a.bar, G);
    reduce_both(P, true, true);
    for (int sd = 0; sd < 2; ++sd)
      if (direct[sd]) n2[sd] = redv[sd][a.s[sd].ncols];
  }
  (void)bk;

  // [finish] beta_{i+1} = ||w'|| (breakdown -> BETA_BREAK), then
  // alpha_{i+1} = ||y'|| / beta (ALPHA_BREAK); bidiag.py:156-158, 173-174
  const double beta = sqrt(n2[0]);
  const double ynrm = sqrt(n2[1]);
  const double alpha = ynrm / beta;
  const bool nonfinite = *reinterpret_cast<volatile int*>(&a.st->nonfinite) != 0;
  int stop = ST_RUNNING;
  if (nonfinite || !isfinite(beta)) stop = ST_NONFINITE;
  else if (beta < a.eps) stop = ST_BETA_BREAK;
  else if (!isfinite(alpha)) stop = ST_NONFINITE;
  else if (alpha < a.eps) stop = ST_ALPHA_BREAK;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.beta_slot = beta;
    if (stop != ST_BETA_BREAK) *a.alpha_slot = alpha;
    if (stop != ST_RUNNING) {
      a.st->status = stop;
      a.st->kprime = a.step;
      a.st->where = a.step;
    }
    host_progress(a.hp, stop, a.step, stop == ST_BETA_BREAK ? 0 : 1);
  }
  // q_{i+1} = w' / beta unless beta broke down; p_{i+1} = y' / ||y'|| unless
  // either did (bidiag.py:165, 176)
  const bool write = side == 0 ? (stop == ST_RUNNING || stop == ST_ALPHA_BREAK)
                               : stop == ST_RUNNING;
  if (write && warp == 0) {
    const double s = side == 0 ? beta : ynrm;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int rl = lane + 32 * e;
      if (rl < nr) S.out[s0 + rl] = xv[e] / s;
    }
  }
}

}  // namespace ksvd
