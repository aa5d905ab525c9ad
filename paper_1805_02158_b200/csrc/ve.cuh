// Vector-extrapolation decision logic on the tiny (kappa+1)^2 factor.
//
// Runs in one thread per image after the fp64 Gram pass.  Reproduces
// extrapolate_once (extrapolation.py:319-386) over the triangular factor R:
//   * R from Cholesky of G = U^T U (U^T U = R^T R, R upper, positive diagonal
//     -- the same R modified Gram-Schmidt produces, up to rounding);
//   * a pivot ratio below max(1e-6, 1e3*rank_tol) is outside what the Gram
//     route resolves, so the image is sent to the exact device MGS pass
//     (mgs_qr, extrapolation.py:159-196) before deciding.  Above it Cholesky
//     leaves ~eps cond^2 on the small pivots: against the reference's MGS on
//     full-rank windows of cond 1e5 / 1e6 / 1e7 (pivot ratio down to 1.3e-6)
//     the weights differ by 1e-9 / 1e-7 / 1.5e-6 relative and the extrapolated
//     point by < 1e-7 of the window's spread, with identical decisions
//     (tests/test_gpu_ve_api.py, golden ve_cond.npz);
//   * MPE  : R[:k,:k] c' = -R[:k,k], c_k = 1, degenerate if |sum c| < 1e-12 ||c||_1
//            (extrapolation.py:241-260);
//   * RRE  : R^T z = 1, R d = z, gamma = d / sum d          (:263-273);
//   * SVD-MPE: right singular vector of R's smallest singular value (one-sided
//            Jacobi), degenerate if |sum v| < 1e-12          (:199-214, 276-284);
//   * MPE / SVD-MPE degeneracy -> RRE with fallback flag     (:361-367);
//   * rank e <= kappa -> order-e annihilating weights on the first e+2
//            iterates; degenerate -> not extrapolated          (:368-386);
//   * reconstruction x = x_m + sum_{j<k} xi_j u_j, xi = 1 - cumsum(gamma)
//            (:295-316, equal to x_m + Q R xi).
#pragma once

#include "state.cuh"

namespace redve {

enum VeMethod : int { M_MPE = 0, M_RRE = 1, M_SVDMPE = 2 };

// Solve R[:n,:n] x = b (upper triangular, back substitution).
__host__ __device__ inline void tri_upper_solve(const double (*R)[MAXKP1], int n, double* x) {
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < n; ++j) s -= R[i][j] * x[j];
    x[i] = s / R[i][i];
  }
}
// Solve R[:n,:n]^T x = b (forward substitution).
__host__ __device__ inline void tri_upper_t_solve(const double (*R)[MAXKP1], int n, double* x) {
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= R[j][i] * x[j];
    x[i] = s / R[i][i];
  }
}

// Order-e annihilating (MPE-form) weights; false if the sum vanished.
__host__ __device__ inline bool annihilating(const double (*R)[MAXKP1], int e, double* c) {
  for (int i = 0; i < e; ++i) c[i] = -R[i][e];
  tri_upper_solve(R, e, c);
  c[e] = 1.0;
  double s = 0.0, a = 0.0;
  for (int i = 0; i <= e; ++i) {
    s += c[i];
    a += fabs(c[i]);
  }
  return !(fabs(s) < 1e-12 * a || !isfinite(s));
}

__host__ __device__ inline void rre_weights(const double (*R)[MAXKP1], int n, double* d) {
  for (int i = 0; i < n; ++i) d[i] = 1.0;
  tri_upper_t_solve(R, n, d);
  tri_upper_solve(R, n, d);
}

// Right singular vector of the smallest singular value (one-sided Jacobi).
__host__ __device__ inline bool svd_min_right(const double (*R)[MAXKP1], int n, double* vout) {
  double A[MAXKP1][MAXKP1], V[MAXKP1][MAXKP1];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      A[i][j] = R[i][j];
      V[i][j] = (i == j) ? 1.0 : 0.0;
    }
  bool conv = false;
  for (int sweep = 0; sweep < 60 && !conv; ++sweep) {
    conv = true;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < n; ++i) {
          al += A[i][p] * A[i][p];
          be += A[i][q] * A[i][q];
          ga += A[i][p] * A[i][q];
        }
        if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
        conv = false;
        double zeta = (be - al) / (2.0 * ga);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < n; ++i) {
          double ap = A[i][p], aq = A[i][q];
          A[i][p] = c * ap - s * aq;
          A[i][q] = s * ap + c * aq;
          double vp = V[i][p], vq = V[i][q];
          V[i][p] = c * vp - s * vq;
          V[i][q] = s * vp + c * vq;
        }
      }
  }
  if (!conv) return false;
  int jmin = 0;
  double smin = INFINITY;
  for (int j = 0; j < n; ++j) {
    double s2 = 0;
    for (int i = 0; i < n; ++i) s2 += A[i][j] * A[i][j];
    if (s2 < smin) {
      smin = s2;
      jmin = j;
    }
  }
  for (int i = 0; i < n; ++i) vout[i] = V[i][jmin];
  return true;
}

struct VeOut {
  int mode;       // VeMode
  int k_used;
  int method;     // rule actually used
  int fallback;   // MPE/SVD-MPE fell back to RRE
  double stab;
  double xi[MAXKP1];
  double gamma[MAXKP1];
  double c[MAXKP1];
};

// Decide from R (n = kappa+1 columns, rank e known).  Shared by the Gram and
// the MGS routes.
__host__ __device__ inline void decide_from_r(const double (*R)[MAXKP1], int n, int e, int method,
                                     VeOut& o) {
  const int kappa = n - 1;
  double c[MAXKP1];
  int used = method, fb = 0, ke;
  if (e == n) {
    bool ok = false;
    if (method == M_MPE) {
      ok = annihilating(R, kappa, c);
    } else if (method == M_SVDMPE) {
      ok = svd_min_right(R, n, c);
      if (ok) {
        double s = 0;
        for (int i = 0; i < n; ++i) s += c[i];
        ok = !(fabs(s) < 1e-12 || !isfinite(s));
      }
    }
    if (method == M_RRE || !ok) {
      fb = (method != M_RRE);
      used = M_RRE;
      rre_weights(R, n, c);
    }
    ke = kappa;
  } else {
    if (!annihilating(R, e, c)) {
      o.mode = VE_SKIP;
      return;
    }
    ke = e;
  }
  double s = 0;
  for (int i = 0; i <= ke; ++i) s += c[i];
  double stab = 0, cum = 0;
  for (int i = 0; i <= ke; ++i) {
    o.c[i] = c[i];
    o.gamma[i] = c[i] / s;
    stab += fabs(o.gamma[i]);
  }
  for (int j = 0; j < ke; ++j) {
    cum += o.gamma[j];
    o.xi[j] = 1.0 - cum;
  }
  o.mode = VE_EXTRAPOLATE;
  o.k_used = ke;
  o.method = used;
  o.fallback = fb;
  o.stab = stab;
}

// Gram route.  G is the (kappa+1)^2 symmetric Gram of the differences.
__host__ __device__ inline void decide_from_gram(const double* G, int n, int method, double rank_tol,
                                        VeOut& o) {
  double R[MAXKP1][MAXKP1];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) R[i][j] = 0.0;
  bool finite = true;
  for (int i = 0; i < n * n; ++i) finite = finite && isfinite(G[i]);
  if (!finite) {  // norms overflowed: skip this window (extrapolation.py:350-358)
    o.mode = VE_SKIP;
    return;
  }
  const double r11 = sqrt(G[0]);
  if (r11 < 1e-300) {  // ZeroFirstColumn -> stationary window (:342-349)
    o.mode = VE_CONVERGED;
    return;
  }
  const double suspicious = fmax(1e-6, 1e3 * rank_tol);
  for (int i = 0; i < n; ++i) {
    double s = G[i * n + i];
    for (int k = 0; k < i; ++k) s -= R[k][i] * R[k][i];
    if (i == 0) s = G[0];
    double rii = s > 0 ? sqrt(s) : 0.0;
    if (i > 0 && !(rii >= suspicious * r11)) {
      o.mode = VE_MGS;  // rank question below the Gram route's resolution
      return;
    }
    R[i][i] = rii;
    for (int j = i + 1; j < n; ++j) {
      double t = G[i * n + j];
      for (int k = 0; k < i; ++k) t -= R[k][i] * R[k][j];
      R[i][j] = t / rii;
    }
  }
  decide_from_r(R, n, n, method, o);
}

}  // namespace redve
