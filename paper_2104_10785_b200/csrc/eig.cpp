// eig.cpp -- host spectral stage: eigenpairs of the Gram tridiagonal B^T B.
//
// Same algorithm and decision rules as the reference's pure-Python solver
// (fsvd.py:63-134): implicit-shift QL with Wilkinson-type shift from the
// leading 2x2, bulge chased from the first negligible coupling m back to l,
// deflation when |e_m| <= eps * (|d_m| + |d_{m+1}|), at most 64 QL sweeps
// per eigenvalue, rotations accumulated into Z when vectors are wanted, and a
// stable descending sort at the end.  k' is at most a few hundred for every
// configuration of the hot path, so this O(k'^2) (O(k'^3) with vectors) stage
// stays on the host, as the north star allows.  Compiled with
// -ffp-contract=off so each operation rounds like the Python floats it
// restates.
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <algorithm>
#include <vector>

#include "ksvd.h"

int ksvd_set_error_from_host(int code, const char* msg);  // defined in ksvd.cu

namespace {

// sqrt(a^2 + b^2) without glibc hypot's extended-precision care when neither
// square can overflow or lose the larger operand to underflow (~6x faster;
// differs from hypot only in the last ulp)
inline double hypot_fast(double a, double b) {
  const double m = std::max(std::fabs(a), std::fabs(b));
  if (m < 1e150 && m > 1e-150) return std::sqrt(a * a + b * b);
  return std::hypot(a, b);
}

struct QL {
  int n;
  std::vector<double> d, e, Z;  // Z column-major n x n (empty: no vectors)
  // false: std::hypot as the reference's math.hypot (fsvd.py:63-134);
  // true: hypot_fast (the rank path's QL, where only eps * ||T|| absolute
  // accuracy of the large values is used)
  bool fast = false;
  double hyp(double a, double b) const { return fast ? hypot_fast(a, b) : std::hypot(a, b); }

  // returns false when a sweep budget is exhausted
  bool solve() {
    const double tiny = DBL_EPSILON;
    for (int l = 0; l < n; ++l) {
      bool done = false;
      for (int sweep = 0; sweep < 64 && !done; ++sweep) {
        int m = l;
        for (; m < n - 1; ++m) {
          const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
          if (std::fabs(e[m]) <= tiny * dd) break;
        }
        if (m == l) {
          done = true;
          break;
        }
        chase(l, m);
      }
      if (!done) return false;
    }
    return true;
  }

  // one implicit QL step on the unreduced block [l, m]
  void chase(int l, int m) {
    double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
    double r = hyp(g, 1.0);
    g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
    double s = 1.0, c = 1.0, p = 0.0;
    for (int i = m - 1; i >= l; --i) {
      const double f = s * e[i];
      const double b = c * e[i];
      r = hyp(f, g);
      e[i + 1] = r;
      if (r == 0.0) {  // underflow: recover and retry the sweep
        d[i + 1] -= p;
        e[m] = 0.0;
        return;
      }
      s = f / r;
      c = g / r;
      g = d[i + 1] - p;
      r = (d[i] - g) * s + 2.0 * c * b;
      p = s * r;
      d[i + 1] = g + p;
      g = c * r - b;
      if (!Z.empty()) rotate(i, s, c);
    }
    d[l] -= p;
    e[l] = g;
    e[m] = 0.0;
  }

  void rotate(int i, double s, double c) {
    double* zi = Z.data() + (size_t)i * n;
    double* zj = Z.data() + (size_t)(i + 1) * n;
    for (int k = 0; k < n; ++k) {
      const double a = zi[k], b = zj[k];
      zj[k] = s * a + c * b;
      zi[k] = c * a - s * b;
    }
  }
};

}  // namespace

extern "C" int ksvd_symtridiag_eig(int n, const double* diag, const double* off, int vectors,
                                   double* theta, double* G) {
  if (n <= 0) return ksvd_set_error_from_host(KSVD_ECONFIG, "empty tridiagonal");
  QL q;
  q.n = n;
  q.d.assign(diag, diag + n);
  q.e.assign(n, 0.0);
  for (int i = 0; i + 1 < n; ++i) q.e[i] = off[i];
  if (vectors) {
    q.Z.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) q.Z[(size_t)i * n + i] = 1.0;
  }
  if (!q.solve())
    return ksvd_set_error_from_host(KSVD_ENUMERIC, "tridiagonal QL did not converge in 64 sweeps");
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  // np.argsort(-d, kind="stable"): ascending in -d, ties keep index order
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return -q.d[a] < -q.d[b]; });
  for (int k = 0; k < n; ++k) theta[k] = q.d[order[k]];
  if (vectors && G) {
    for (int k = 0; k < n; ++k)
      std::memcpy(G + (size_t)k * n, q.Z.data() + (size_t)order[k] * n, sizeof(double) * n);
  }
  return KSVD_OK;
}

// ---------------------------------------------------------------------------
// Singular values of the (k+1) x k lower bidiagonal B (alphas on the
// diagonal, betas[1..k] below) to high RELATIVE accuracy: bisection on the
// Golub-Kahan tridiagonal TGK = tridiag(0; a1, b2, a2, b3, ..., ak, b_{k+1})
// (size 2k+1, eigenvalues +-sigma_i and 0; Demmel & Kahan 1990).  Used by
// estimate_rank: theta_i = sigma_i^2 are the eigenvalues of B^T B
// (rank.py:64), but the tiny ones come out accurate to a few ulps of
// themselves instead of eps * ||T|| -- the relative rank threshold of
// configuration 5, 1e-16 theta_1, sits exactly at that QL noise floor.
namespace {

struct TGK {
  int k;
  std::vector<double> e2;  // squared off-diagonals, 2k entries
  double pivmin;

  // number of singular values < x (x > 0)
  int below(double x) const {
    double q = -x;
    int neg = q < 0;
    for (double v : e2) {
      q = -x - v / q;
      if (std::fabs(q) < pivmin) q = -pivmin;
      neg += q < 0;
    }
    return neg - (k + 1);
  }
};

}  // namespace

extern "C" int ksvd_bidiag_sv2(int k, const double* alphas, const double* betas, double* theta) {
  if (k <= 0) return ksvd_set_error_from_host(KSVD_ECONFIG, "empty bidiagonal");
  TGK t;
  t.k = k;
  t.e2.resize(2 * (size_t)k);
  double emax = 0.0, gersh = 0.0;
  for (int i = 0; i < k; ++i) {
    const double a = std::fabs(alphas[i]), b = std::fabs(betas[i + 1]);
    t.e2[2 * i] = a * a;
    t.e2[2 * i + 1] = b * b;
    emax = std::max(emax, std::max(a, b));
  }
  for (int i = 0; i < 2 * k; ++i) {  // Gershgorin bound of TGK
    const double l = i > 0 ? std::sqrt(t.e2[i - 1]) : 0.0;
    gersh = std::max(gersh, l + std::sqrt(t.e2[i]));
  }
  if (!std::isfinite(gersh)) return ksvd_set_error_from_host(KSVD_ENUMERIC, "non-finite bidiagonal");
  t.pivmin = DBL_MIN * std::max(1.0, emax * emax);
  // Large values: QL on B^T B (as the reference, fsvd.py:63-134) -- accurate
  // to eps*||T|| absolutely, i.e. to ~1e-10 relative above 1e-6 theta_1.
  // Tail below that: bisection on TGK, accurate to a few ulps of itself.
  QL q;
  q.n = k;
  q.fast = true;  // 1.0 -> ~0.2 ms at k = 144 (config 2)
  q.d.resize(k);
  q.e.assign(k, 0.0);
  for (int i = 0; i < k; ++i)
    q.d[i] = alphas[i] * alphas[i] + betas[i + 1] * betas[i + 1];
  for (int i = 0; i + 1 < k; ++i) q.e[i] = alphas[i + 1] * betas[i + 1];
  if (!q.solve())
    return ksvd_set_error_from_host(KSVD_ENUMERIC, "tridiagonal QL did not converge in 64 sweeps");
  std::vector<double> th(q.d);
  std::sort(th.begin(), th.end(), [](double a, double b) { return a > b; });
  const double tau = 1e-6 * std::max(th[0], 0.0);
  int tail = 0;
  while (tail < k && th[k - 1 - tail] < tau) ++tail;
  // Upper end of the tail bracket: every tail value is below sqrt(tau) up to
  // QL's absolute error; verified with one Sturm count (else Gershgorin).
  double top = std::sqrt(tau + 64.0 * DBL_EPSILON * std::max(th[0], 0.0)) * (1.0 + 1e-8);
  if (tail > 0 && t.below(top) < tail) top = gersh * (1.0 + 4 * DBL_EPSILON) + DBL_MIN;
  // Bisection of up to kLanes tail values in lock step: one pass over the
  // TGK entries advances every lane's Sturm count (independent dependency
  // chains, so the division latency overlaps).  Lane j bisects the j-th
  // smallest value; the same per-lane steps as a scalar bisection.
  constexpr int kLanes = 8;
  for (int j0 = 0; j0 < tail; j0 += kLanes) {
    const int nl = std::min(kLanes, tail - j0);
    double lo[kLanes], hi[kLanes], mid[kLanes];
    bool live[kLanes];
    for (int l = 0; l < kLanes; ++l) {
      lo[l] = 0.0;
      hi[l] = top;
      live[l] = l < nl;
    }
    for (int it = 0; it < 400; ++it) {
      bool any = false;
      for (int l = 0; l < nl; ++l) {
        if (live[l] && (hi[l] - lo[l] <= 4 * DBL_EPSILON * hi[l] || hi[l] < 1e-300)) live[l] = false;
        if (!live[l]) continue;
        any = true;
        if (lo[l] == 0.0)
          mid[l] = hi[l] * (hi[l] > 1e-280 ? 1e-3 : 0.5);  // coarse descent to the scale
        else if (hi[l] > 2.0 * lo[l])
          mid[l] = std::sqrt(lo[l] * hi[l]);  // geometric bisection
        else
          mid[l] = 0.5 * (lo[l] + hi[l]);
      }
      if (!any) break;
      double q[kLanes];
      int neg[kLanes];
      for (int l = 0; l < kLanes; ++l) {
        const double x = live[l] ? mid[l] : 1.0;
        q[l] = -x;
        neg[l] = q[l] < 0;
      }
      for (double v : t.e2) {
        for (int l = 0; l < kLanes; ++l) {
          const double x = live[l] ? mid[l] : 1.0;
          double ql = -x - v / q[l];
          if (std::fabs(ql) < t.pivmin) ql = -t.pivmin;
          q[l] = ql;
          neg[l] += ql < 0;
        }
      }
      for (int l = 0; l < nl; ++l) {
        if (!live[l]) continue;
        if (neg[l] - (k + 1) <= j0 + l)
          lo[l] = mid[l];
        else
          hi[l] = mid[l];
      }
    }
    for (int l = 0; l < nl; ++l) {
      const double sv = 0.5 * (lo[l] + hi[l]);
      th[k - 1 - (j0 + l)] = sv * sv;
    }
  }
  std::sort(th.begin(), th.end(), [](double a, double b) { return a > b; });
  for (int j = 0; j < k; ++j) theta[j] = th[j];
  return KSVD_OK;
}

// ---------------------------------------------------------------------------
// Dense SVD of the small k x k projected matrix of the restarted mode
// (T = [diag(sigma) rho; 0 bidiagonal], paper_2104_10785_b200/restart.py):
// one-sided Jacobi (Hestenes) on the columns of W = T, V accumulating the
// rotations; converged when every column pair is orthogonal to k * eps
// relative (the rounding level of the pair's dot product), which gives every
// singular value to high relative accuracy.
// T, U, V column-major k x k; s descending; sign of each column pair fixed so
// that U[:, j] = T V[:, j] / s_j (U columns of zero singular values are left
// as the normalised zero column, i.e. 0).
// AVX2 clone picked at load time where the host has it (the rotations and
// column dots vectorise 4-wide; same operation order, identical results)
extern "C" __attribute__((target_clones("avx2", "default"))) int ksvd_dense_svd(
    int k, const double* T, double* U, double* s, double* V) {
  if (k <= 0) return ksvd_set_error_from_host(KSVD_ECONFIG, "empty matrix");
  const size_t K = (size_t)k;
  std::vector<double> W(T, T + K * K), Vm(K * K, 0.0);
  for (size_t i = 0; i < K; ++i) Vm[i * K + i] = 1.0;
  auto col = [&](std::vector<double>& X, int j) { return X.data() + (size_t)j * K; };
  const double tol = std::max(1e-15, (double)K * DBL_EPSILON);
  // columns below eps ||T||_F are numerically zero: rotating them against
  // the others only stirs rounding noise (exactly rank-deficient T -- a
  // breakdown -- would never pass the relative test)
  double fro2 = 0.0;
  for (size_t i = 0; i < K * K; ++i) fro2 += W[i] * W[i];
  const double zero2 = fro2 * DBL_EPSILON * DBL_EPSILON;
  bool done = false;
  double worst = 0.0;
  std::vector<double> d(K);  // squared column norms, updated through the rotations
  for (int sweep = 0; sweep < 80 && !done; ++sweep) {
    done = true;
    worst = 0.0;
    for (int j = 0; j < k; ++j) {  // refreshed every sweep (no drift)
      const double* w = col(W, j);
      double t = 0.0;
      for (size_t i = 0; i < K; ++i) t += w[i] * w[i];
      d[j] = t;
    }
    for (int p = 0; p < k - 1; ++p) {
      for (int q = p + 1; q < k; ++q) {
        double* __restrict__ wp = col(W, p);
        double* __restrict__ wq = col(W, q);
        const double a = d[p], b = d[q];
        double g4[4] = {0.0, 0.0, 0.0, 0.0};  // 4 independent chains (fixed order)
        size_t i4 = 0;
        for (; i4 + 4 <= K; i4 += 4)
          for (int u = 0; u < 4; ++u) g4[u] += wp[i4 + u] * wq[i4 + u];
        for (; i4 < K; ++i4) g4[0] += wp[i4] * wq[i4];
        const double g = (g4[0] + g4[1]) + (g4[2] + g4[3]);
        if (g == 0.0 || a <= zero2 || b <= zero2 || std::fabs(g) <= tol * std::sqrt(a * b))
          continue;
        worst = std::max(worst, std::fabs(g) / std::sqrt(a * b));
        done = false;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        double* __restrict__ vp = col(Vm, p);
        double* __restrict__ vq = col(Vm, q);
        for (size_t i = 0; i < K; ++i) {
          const double x = wp[i], y = wq[i];
          wp[i] = c * x - sn * y;
          wq[i] = sn * x + c * y;
          const double u = vp[i], v = vq[i];
          vp[i] = c * u - sn * v;
          vq[i] = sn * u + c * v;
        }
        d[p] = a - t * g;  // exact for the rotation that zeroes the pair
        d[q] = b + t * g;
      }
    }
  }
  if (!done && !(worst < 1e-10))
    return ksvd_set_error_from_host(KSVD_ENUMERIC, "Jacobi SVD did not converge");
  std::vector<double> nrm(K);
  for (int j = 0; j < k; ++j) {
    double t = 0.0;
    const double* w = col(W, j);
    for (size_t i = 0; i < K; ++i) t += w[i] * w[i];
    nrm[j] = std::sqrt(t);
  }
  std::vector<int> order(K);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
  for (int r = 0; r < k; ++r) {
    const int j = order[r];
    s[r] = nrm[j];
    const double* w = col(W, j);
    for (size_t i = 0; i < K; ++i) {
      U[(size_t)r * K + i] = nrm[j] > 0 ? w[i] / nrm[j] : 0.0;
      V[(size_t)r * K + i] = Vm[(size_t)j * K + i];
    }
  }
  return KSVD_OK;
}
