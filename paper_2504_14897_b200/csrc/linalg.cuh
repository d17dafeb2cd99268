// linalg.cuh — per-component d <= 3 linear algebra on the device, replacing the
// reference's Eigen LLT / SelfAdjointEigenSolver calls. Same algorithms as the oracle
// restatement (oracle/vdfc_oracle.cpp) so the discrete decisions (LLT success, the
// collapse test, repair doublings) are taken identically.
#pragma once

#include "common.cuh"

namespace vdfcg {

// Symmetric d x d stored full row-major in a[9] (a[i*3+j]).
struct Sym3 {
  double a[9];
  VDFCG_HD double& operator()(int i, int j) { return a[i * 3 + j]; }
  VDFCG_HD double operator()(int i, int j) const { return a[i * 3 + j]; }
};

// gaussian.hpp:46-49 symmetrize_from_upper
template <int D>
VDFCG_DEV void symmetrize_from_upper(Sym3& m) {
#pragma unroll
  for (int i = 1; i < D; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) m(i, j) = m(j, i);
}

// Eigen llt_inplace<Lower>::unblocked order + llt_ok (gaussian.hpp:15-19). L is the
// lower factor (row-major, upper part zero). Returns false when a pivot is not > 0 or
// a diagonal entry is not finite.
template <int D>
VDFCG_DEV bool cholesky(const Sym3& a, Sym3& L) {
#pragma unroll
  for (int i = 0; i < 9; ++i) L.a[i] = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double x = a(k, k);
    if (k > 0) {
      double sq = 0.0;
#pragma unroll
      for (int j = 0; j < k; ++j) sq = __dadd_rn(sq, __dmul_rn(L(k, j), L(k, j)));
      x = __dsub_rn(x, sq);
    }
    if (!(x > 0.0)) return false;
    const double s = sqrt(x);
    if (!isfinite(s)) return false;
    L(k, k) = s;
#pragma unroll
    for (int i = k + 1; i < D; ++i) {
      double v = a(i, k);
#pragma unroll
      for (int j = 0; j < k; ++j) v = __dsub_rn(v, __dmul_rn(L(i, j), L(k, j)));
      L(i, k) = v / s;
    }
  }
  return true;
}

// Cyclic Jacobi eigenvalues (relative accuracy for the collapse test, wgmm.cpp:305-306).
template <int D>
VDFCG_DEV void sym_eigenvalues(const Sym3& in, double* ev) {
  double a[3][3];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) a[i][j] = in(i, j);
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
#pragma unroll
    for (int p = 0; p < D; ++p)
#pragma unroll
      for (int q = p + 1; q < D; ++q) off += fabs(a[p][q]);
    if (off == 0.0 || !isfinite(off)) break;
#pragma unroll
    for (int p = 0; p < D; ++p) {
#pragma unroll
      for (int q = p + 1; q < D; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        a[p][p] -= t * apq;
        a[q][q] += t * apq;
        a[p][q] = a[q][p] = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          if (r == p || r == q) continue;
          const double arp = a[r][p], arq = a[r][q];
          a[r][p] = a[p][r] = c * arp - s * arq;
          a[r][q] = a[q][r] = s * arp + c * arq;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) ev[i] = a[i][i];
}

// wgmm.cpp:340-362 repair_covariance. Returns false (CovarianceRepairError) when no
// loading in 0..60 doublings succeeds. *doublings = -1 when none was needed.
template <int D>
VDFCG_DEV bool repair_covariance(const Sym3& sigma, Sym3& out, int* doublings) {
  Sym3 sym;
#pragma unroll
  for (int i = 0; i < 9; ++i) sym.a[i] = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) sym(a, b) = __dmul_rn(0.5, __dadd_rn(sigma(a, b), sigma(b, a)));
  symmetrize_from_upper<D>(sym);
  *doublings = -1;
  Sym3 L;
  if (cholesky<D>(sym, L)) {
    out = sym;
    return true;
  }
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tr = __dadd_rn(tr, sym(a, a));
  double lambda = __dmul_rn(1e-8, tr) / static_cast<double>(D);
  for (int k = 0; k <= 60; ++k, lambda = __dmul_rn(lambda, 2.0)) {
    Sym3 loaded = sym;
#pragma unroll
    for (int a = 0; a < D; ++a) loaded(a, a) = __dadd_rn(loaded(a, a), lambda);
    if (cholesky<D>(loaded, L)) {
      *doublings = k;
      out = loaded;
      return true;
    }
  }
  return false;
}

// The collapse test + repair of the M-step (wgmm.cpp:300-315). Returns true when the
// new covariance is accepted (written to out), false when the component collapsed.
template <int D>
VDFCG_DEV bool accept_covariance(const Sym3& sigma, Sym3& out) {
  bool finite = true;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) finite = finite && isfinite(sigma(a, b));
  if (finite) {
    double ev[3];
    sym_eigenvalues<D>(sigma, ev);
    double mn = ev[0], mx = ev[0];
#pragma unroll
    for (int a = 1; a < D; ++a) {
      mn = fmin(mn, ev[a]);
      mx = fmax(mx, ev[a]);
    }
    if (mn <= 1e-14 * mx) return false;
  }
  int doublings = -1;
  Sym3 rep;
  if (!repair_covariance<D>(sigma, rep, &doublings)) return false;
  if (doublings > 2) return false;
  symmetrize_from_upper<D>(rep);
  out = rep;
  return true;
}

// Cheap certificate for the collapse test (wgmm.cpp:305-306): if the LLT of sigma
// succeeds, det = prod(L_aa)^2 and lambda_min >= det / prod of the other eigenvalues
// >= det / (tr/2)^2 (d=3) or det / tr (d=2). When that lower bound already exceeds
// 1e-14 * tr (>= 1e-14 * lambda_max) the component certainly did not collapse and
// repair_covariance would return sigma unchanged (doublings = -1), so the reference
// sequence "eigen test, then repair" reduces to "accept sigma". Returns the bound
// (or -1 when the LLT fails); the caller falls back to accept_covariance otherwise.
template <int D>
VDFCG_DEV double lmin_lower_bound(const Sym3& s) {
  Sym3 L;
  if (!cholesky<D>(s, L)) return -1.0;
  double p = 1.0, tr = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    p *= L(a, a);
    tr += s(a, a);
  }
  const double det = p * p;
  return D == 1 ? det : (D == 2 ? det / tr : det / (0.25 * tr * tr));
}

template <int D>
VDFCG_DEV double trace3(const Sym3& s) {
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tr += s(a, a);
  return tr;
}

// Smallest eigenvalue estimate used to decide whether the one-pass shifted covariance
// needs the exact second pass (see em.cu).
template <int D>
VDFCG_DEV double min_eigenvalue(const Sym3& s) {
  double ev[3];
  sym_eigenvalues<D>(s, ev);
  double mn = ev[0];
#pragma unroll
  for (int a = 1; a < D; ++a) mn = fmin(mn, ev[a]);
  return mn;
}

}  // namespace vdfcg
