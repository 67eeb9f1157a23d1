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

struct QL {
  int n;
  std::vector<double> d, e, Z;  // Z column-major n x n (empty: no vectors)

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
    double r = std::hypot(g, 1.0);
    g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
    double s = 1.0, c = 1.0, p = 0.0;
    for (int i = m - 1; i >= l; --i) {
      const double f = s * e[i];
      const double b = c * e[i];
      r = std::hypot(f, g);
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
  for (int j = 0; j < tail; ++j) {  // j-th smallest singular value
    double lo = 0.0, hi = gersh * (1.0 + 4 * DBL_EPSILON) + DBL_MIN;
    for (int it = 0; it < 400; ++it) {
      if (hi - lo <= 4 * DBL_EPSILON * hi || hi < 1e-300) break;
      double mid;
      if (lo == 0.0)
        mid = hi * (hi > 1e-280 ? 1e-3 : 0.5);  // coarse descent to the scale
      else if (hi > 2.0 * lo)
        mid = std::sqrt(lo * hi);  // geometric bisection
      else
        mid = 0.5 * (lo + hi);
      if (t.below(mid) <= j)
        lo = mid;
      else
        hi = mid;
    }
    const double sv = 0.5 * (lo + hi);
    th[k - 1 - j] = sv * sv;
  }
  std::sort(th.begin(), th.end(), [](double a, double b) { return a > b; });
  for (int j = 0; j < k; ++j) theta[j] = th[j];
  return KSVD_OK;
}
