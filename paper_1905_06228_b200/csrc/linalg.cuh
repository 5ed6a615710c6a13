// 6x6 symmetric solves for the sub-pixel refiners, fp64, host+device.
// Restates the published Eigen::LDLT algorithm (pivot = largest remaining
// |diagonal|, zero pivot -> NumericalIssue, solve zeroes rows whose
// |D_ii| <= DBL_MIN) in the same operation order as the oracle's stand-in
// (oracle/ref_build/eigen_standin/Eigen/Dense), so with a bit-identical input
// (the IC-GN Hessian is exact, see refine.cu) the factor is bit-identical.
#pragma once

#include <cmath>

namespace dicb200 {

struct Ldlt6 {
  double m[36];
  int perm[6];
  int ok;
};

#define DICB200_M6(A, i, j) ((A)[(i) * 6 + (j)])

__device__ inline void ldlt6_swap(double& a, double& b) {
  const double t = a;
  a = b;
  b = t;
}

__device__ inline void ldlt6_compute(Ldlt6& L, const double* a) {
  for (int i = 0; i < 36; ++i) L.m[i] = a[i];
  double* m = L.m;
  L.ok = 1;
  int found_zero_pivot = 0;
  for (int k = 0; k < 6; ++k) {
    int big = k;
    double bigv = fabs(DICB200_M6(m, k, k));
    for (int i = k + 1; i < 6; ++i)
      if (fabs(DICB200_M6(m, i, i)) > bigv) {
        bigv = fabs(DICB200_M6(m, i, i));
        big = i;
      }
    L.perm[k] = big;
    if (big != k) {
      for (int j = 0; j < k; ++j) ldlt6_swap(DICB200_M6(m, k, j), DICB200_M6(m, big, j));
      for (int i = big + 1; i < 6; ++i) ldlt6_swap(DICB200_M6(m, i, k), DICB200_M6(m, i, big));
      ldlt6_swap(DICB200_M6(m, k, k), DICB200_M6(m, big, big));
      for (int i = k + 1; i < big; ++i) {
        const double tmp = DICB200_M6(m, i, k);
        DICB200_M6(m, i, k) = DICB200_M6(m, big, i);
        DICB200_M6(m, big, i) = tmp;
      }
    }
    if (k > 0) {
      double temp[6];
      for (int j = 0; j < k; ++j) temp[j] = __dmul_rn(DICB200_M6(m, j, j), DICB200_M6(m, k, j));
      double dot = __dmul_rn(DICB200_M6(m, k, 0), temp[0]);
      for (int j = 1; j < k; ++j) dot = __dadd_rn(dot, __dmul_rn(DICB200_M6(m, k, j), temp[j]));
      DICB200_M6(m, k, k) = __dsub_rn(DICB200_M6(m, k, k), dot);
      for (int i = k + 1; i < 6; ++i) {
        double s = __dmul_rn(DICB200_M6(m, i, 0), temp[0]);
        for (int j = 1; j < k; ++j) s = __dadd_rn(s, __dmul_rn(DICB200_M6(m, i, j), temp[j]));
        DICB200_M6(m, i, k) = __dsub_rn(DICB200_M6(m, i, k), s);
      }
    }
    const double akk = DICB200_M6(m, k, k);
    const int valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      for (int j = 0; j < 6; ++j) L.perm[j] = j;
      L.ok = 0;
      break;
    }
    if (k + 1 < 6) {
      if (valid) {
        for (int i = k + 1; i < 6; ++i) DICB200_M6(m, i, k) = __ddiv_rn(DICB200_M6(m, i, k), akk);
      } else {
        for (int i = k + 1; i < 6; ++i)
          if (DICB200_M6(m, i, k) != 0.0) L.ok = 0;
      }
    }
    if (found_zero_pivot && valid)
      L.ok = 0;
    else if (!valid)
      found_zero_pivot = 1;
  }
}

__device__ inline void ldlt6_solve(const Ldlt6& L, const double* b, double* x) {
  const double* m = L.m;
  for (int i = 0; i < 6; ++i) x[i] = b[i];
  for (int k = 0; k < 6; ++k)
    if (L.perm[k] != k) ldlt6_swap(x[k], x[L.perm[k]]);
  for (int i = 0; i < 6; ++i)
    if (x[i] != 0.0)
      for (int r = i + 1; r < 6; ++r) x[r] = __dsub_rn(x[r], __dmul_rn(x[i], DICB200_M6(m, r, i)));
  for (int i = 0; i < 6; ++i) {
    if (fabs(DICB200_M6(m, i, i)) > 2.2250738585072014e-308)
      x[i] = __ddiv_rn(x[i], DICB200_M6(m, i, i));
    else
      x[i] = 0.0;
  }
  for (int i = 5; i >= 0; --i) {
    double s = 0.0;
    int any = 0;
    for (int j = i + 1; j < 6; ++j) {
      const double t = __dmul_rn(DICB200_M6(m, j, i), x[j]);
      s = any ? __dadd_rn(s, t) : t;
      any = 1;
    }
    if (any) x[i] = __dsub_rn(x[i], s);
  }
  for (int k = 5; k >= 0; --k)
    if (L.perm[k] != k) ldlt6_swap(x[k], x[L.perm[k]]);
}

// Extreme eigenvalues by cyclic Jacobi (stand-in for SelfAdjointEigenSolver,
// used only for icgn_precompute's condition test, subpixel.cpp:215-219).
__device__ inline void jacobi6_minmax(const double* a, double* lo, double* hi) {
  double m[36];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) DICB200_M6(m, i, j) = DICB200_M6(m, j, i) = DICB200_M6(a, i, j);
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) off += DICB200_M6(m, p, q) * DICB200_M6(m, p, q);
    if (off == 0.0) break;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) {
        const double apq = DICB200_M6(m, p, q);
        if (apq == 0.0) continue;
        const double theta = (DICB200_M6(m, q, q) - DICB200_M6(m, p, p)) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 6; ++k) {
          const double mkp = DICB200_M6(m, k, p), mkq = DICB200_M6(m, k, q);
          DICB200_M6(m, k, p) = c * mkp - s * mkq;
          DICB200_M6(m, k, q) = s * mkp + c * mkq;
        }
        for (int k = 0; k < 6; ++k) {
          const double mpk = DICB200_M6(m, p, k), mqk = DICB200_M6(m, q, k);
          DICB200_M6(m, p, k) = c * mpk - s * mqk;
          DICB200_M6(m, q, k) = s * mpk + c * mqk;
        }
      }
  }
  double mn = DICB200_M6(m, 0, 0), mx = mn;
  for (int i = 1; i < 6; ++i) {
    const double d = DICB200_M6(m, i, i);
    mn = d < mn ? d : mn;
    mx = mx < d ? d : mx;
  }
  *lo = mn;
  *hi = mx;
}

}  // namespace dicb200
