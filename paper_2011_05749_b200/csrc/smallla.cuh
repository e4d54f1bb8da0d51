// K5: tiny dense complex128 linear algebra for the per-bucket solves
// (smallnum.py:54-142 and the lstsq calls of oneshot.py:231).
//
// Everything is register/local-memory resident and runs in one thread; matrices
// are at most kLaMaxRows x kLaMaxCols.  Written host+device so the same source is
// unit-tested on the CPU against numpy (tests/test_dt_core_host.py via tests/native/).
//   svd_jacobi   one-sided (Hestenes) Jacobi SVD: accurate small singular values,
//                which the sFFT-DT vote quantises at 1e-12 (oneshot.py:136);
//   lstsq        SVD least squares with numpy's lstsq cutoff eps*max(m,n)*smax
//                (smallnum.py:60-68, oneshot.py:231); also returns the rank;
//   eigvals      Householder-Hessenberg + shifted complex QR with deflation
//                (np.linalg.eigvals / np.roots on companion matrices);
//   poly_roots   closed forms for degree 1-2, companion eigenvalues for 3-4
//                (smallnum.py:90-107).
#pragma once

#include <math.h>
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace afft {
namespace la {

constexpr int kLaMaxRows = 32;
constexpr int kLaMaxCols = 8;
constexpr double kEps = 2.220446049250313e-16;

struct c2 {
  double re, im;
};

__host__ __device__ __forceinline__ c2 C(double r, double i = 0.0) { return c2{r, i}; }
__host__ __device__ __forceinline__ c2 add(c2 a, c2 b) { return c2{a.re + b.re, a.im + b.im}; }
__host__ __device__ __forceinline__ c2 sub(c2 a, c2 b) { return c2{a.re - b.re, a.im - b.im}; }
__host__ __device__ __forceinline__ c2 mul(c2 a, c2 b) {
  return c2{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__host__ __device__ __forceinline__ c2 conj(c2 a) { return c2{a.re, -a.im}; }
__host__ __device__ __forceinline__ c2 scale(c2 a, double s) { return c2{a.re * s, a.im * s}; }
// conj(a) * b
__host__ __device__ __forceinline__ c2 cmulc(c2 a, c2 b) {
  return c2{a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
__host__ __device__ __forceinline__ double abs2(c2 a) { return a.re * a.re + a.im * a.im; }
__host__ __device__ __forceinline__ double cabs(c2 a) { return hypot(a.re, a.im); }
// Smith division (numpy's complex '/')
__host__ __device__ __forceinline__ c2 div(c2 a, c2 b) {
  const double br = fabs(b.re), bi = fabs(b.im);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return c2{a.re / br, a.im / br};
    const double rat = b.im / b.re;
    const double scl = 1.0 / (b.re + b.im * rat);
    return c2{(a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl};
  }
  const double rat = b.re / b.im;
  const double scl = 1.0 / (b.im + b.re * rat);
  return c2{(a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl};
}
// principal square root (C99 csqrt)
__host__ __device__ __forceinline__ c2 csqrt_(c2 z) {
  if (z.re == 0.0 && z.im == 0.0) return c2{0.0, z.im};
  const double t = sqrt((fabs(z.re) + hypot(z.re, z.im)) * 0.5);
  if (z.re >= 0.0) return c2{t, z.im / (2.0 * t)};
  return c2{fabs(z.im) / (2.0 * t), copysign(t, z.im)};
}
__host__ __device__ __forceinline__ bool finite(c2 z) { return isfinite(z.re) && isfinite(z.im); }

// Column-major small matrix with compile-time capacity MR x MC.
template <int MR, int MC>
struct MatT {
  static constexpr int kRows = MR, kCols = MC;
  int m, n;
  c2 a[MR * MC];
  __host__ __device__ __forceinline__ c2& at(int r, int c) { return a[c * MR + r]; }
  __host__ __device__ __forceinline__ const c2& at(int r, int c) const { return a[c * MR + r]; }
};
using Mat = MatT<kLaMaxRows, kLaMaxCols>;

// One-sided Jacobi SVD of A (m x n, m >= n).  On return A holds U*diag(sigma)
// (unnormalised left vectors), sigma[0..n) descending, V (n x n, column-major in
// a Mat) the right singular vectors; columns are permuted consistently.
template <class MA, class MV>
__host__ __device__ inline void svd_jacobi(MA& A, double* sigma, MV& V) {
  const int m = A.m, n = A.n;
  V.m = n;
  V.n = n;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) V.at(i, j) = C(i == j ? 1.0 : 0.0);
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0;
        c2 gamma = C(0.0);
        for (int i = 0; i < m; ++i) {
          const c2 ap = A.at(i, p), aq = A.at(i, q);
          alpha += abs2(ap);
          beta += abs2(aq);
          gamma = add(gamma, cmulc(ap, aq));
        }
        const double g = cabs(gamma);
        if (g == 0.0 || g <= kEps * sqrt(alpha * beta)) continue;
        rotated = true;
        const c2 ph = C(gamma.re / g, gamma.im / g);  // e^{i phi}
        const double zeta = (beta - alpha) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        // q~ = e^{-i phi} q; p' = c p - s q~, q' = s p + c q~
        for (int i = 0; i < m; ++i) {
          const c2 ap = A.at(i, p);
          const c2 aq = cmulc(ph, A.at(i, q));
          A.at(i, p) = sub(scale(ap, c), scale(aq, s));
          A.at(i, q) = add(scale(ap, s), scale(aq, c));
        }
        for (int i = 0; i < n; ++i) {
          const c2 vp = V.at(i, p);
          const c2 vq = cmulc(ph, V.at(i, q));
          V.at(i, p) = sub(scale(vp, c), scale(vq, s));
          V.at(i, q) = add(scale(vp, s), scale(vq, c));
        }
      }
    }
    if (!rotated) break;
  }
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int i = 0; i < m; ++i) s2 += abs2(A.at(i, j));
    sigma[j] = sqrt(s2);
  }
  // selection sort descending, permuting columns of A and V
  for (int j = 0; j < n; ++j) {
    int best = j;
    for (int k = j + 1; k < n; ++k)
      if (sigma[k] > sigma[best]) best = k;
    if (best != j) {
      const double ts = sigma[j];
      sigma[j] = sigma[best];
      sigma[best] = ts;
      for (int i = 0; i < m; ++i) {
        const c2 t = A.at(i, j);
        A.at(i, j) = A.at(i, best);
        A.at(i, best) = t;
      }
      for (int i = 0; i < n; ++i) {
        const c2 t = V.at(i, j);
        V.at(i, j) = V.at(i, best);
        V.at(i, best) = t;
      }
    }
  }
}

// Singular values only (any shape): uses A^H when m < n.
template <class MA>
__host__ __device__ inline void singular_values(const MA& A, double* sigma) {
  constexpr int S = MA::kRows > MA::kCols ? MA::kRows : MA::kCols;
  constexpr int T = MA::kRows < MA::kCols ? MA::kRows : MA::kCols;
  MatT<S, T> W;
  MatT<T, T> V;
  if (A.m >= A.n) {
    W.m = A.m;
    W.n = A.n;
    for (int r = 0; r < A.m; ++r)
      for (int c = 0; c < A.n; ++c) W.at(r, c) = A.at(r, c);
  } else {
    W.m = A.n;
    W.n = A.m;
    for (int r = 0; r < A.m; ++r)
      for (int c = 0; c < A.n; ++c) W.at(c, r) = conj(A.at(r, c));
  }
  svd_jacobi(W, sigma, V);
}

// x = argmin ||A x - y|| with numpy lstsq semantics (rcond = eps*max(m,n)),
// for m >= n.  Returns the numerical rank; sigma (optional) gets the singular values.
template <class MA>
__host__ __device__ inline int lstsq(const MA& A, const c2* y, c2* x, double* sigma_out) {
  const int m = A.m, n = A.n;
  MA W = A;
  MatT<MA::kCols, MA::kCols> V;
  double sigma[MA::kCols];
  svd_jacobi(W, sigma, V);
  const double cutoff = kEps * (double)(m > n ? m : n) * sigma[0];
  for (int j = 0; j < n; ++j) x[j] = C(0.0);
  int rank = 0;
  for (int k = 0; k < n; ++k) {
    if (!(sigma[k] > cutoff)) continue;
    ++rank;
    // u_k = W[:,k] / sigma_k ; coefficient (u_k^H y) / sigma_k = (W[:,k]^H y) / sigma_k^2
    c2 dot = C(0.0);
    for (int i = 0; i < m; ++i) dot = add(dot, cmulc(W.at(i, k), y[i]));
    const c2 coef = scale(dot, 1.0 / (sigma[k] * sigma[k]));
    for (int j = 0; j < n; ++j) x[j] = add(x[j], mul(V.at(j, k), coef));
  }
  if (sigma_out)
    for (int k = 0; k < n; ++k) sigma_out[k] = sigma[k];
  return rank;
}

// Moore-Penrose pseudo-inverse of A (m x n, any shape) with numpy's pinv cutoff
// rcond * smax (default rcond 1e-15).  P gets n x m.
template <class MA, class MP>
__host__ __device__ inline void pinv(const MA& A, MP& P, double rcond) {
  constexpr int S = MA::kRows > MA::kCols ? MA::kRows : MA::kCols;
  constexpr int T = MA::kRows < MA::kCols ? MA::kRows : MA::kCols;
  const bool tall = A.m >= A.n;
  MatT<S, T> W;
  MatT<T, T> V;
  if (tall) {
    W.m = A.m;
    W.n = A.n;
    for (int r = 0; r < A.m; ++r)
      for (int c = 0; c < A.n; ++c) W.at(r, c) = A.at(r, c);
  } else {
    W.m = A.n;
    W.n = A.m;
    for (int r = 0; r < A.m; ++r)
      for (int c = 0; c < A.n; ++c) W.at(c, r) = conj(A.at(r, c));
  }
  double sigma[T];
  svd_jacobi(W, sigma, V);  // W = U S (W.m x W.n), V (W.n x W.n)
  const double cutoff = rcond * sigma[0];
  // pinv(W) = V S^+ U^H = sum_k v_k (w_k^H) / s_k^2  (W.n x W.m)
  MatT<T, S> Q;
  Q.m = W.n;
  Q.n = W.m;
  for (int i = 0; i < Q.m; ++i)
    for (int j = 0; j < Q.n; ++j) Q.at(i, j) = C(0.0);
  for (int k = 0; k < W.n; ++k) {
    if (!(sigma[k] > cutoff)) continue;
    const double inv = 1.0 / (sigma[k] * sigma[k]);
    for (int i = 0; i < Q.m; ++i) {
      const c2 vk = scale(V.at(i, k), inv);
      for (int j = 0; j < Q.n; ++j) Q.at(i, j) = add(Q.at(i, j), mul(vk, conj(W.at(j, k))));
    }
  }
  if (tall) {
    P.m = Q.m;
    P.n = Q.n;
    for (int r = 0; r < Q.m; ++r)
      for (int c = 0; c < Q.n; ++c) P.at(r, c) = Q.at(r, c);
  } else {  // pinv(A) = pinv(A^H)^H
    P.m = Q.n;
    P.n = Q.m;
    for (int r = 0; r < Q.m; ++r)
      for (int c = 0; c < Q.n; ++c) P.at(c, r) = conj(Q.at(r, c));
  }
}

// Eigenvalues of a general complex n x n matrix (n <= kLaMaxCols).  Returns false
// if the QR iteration did not converge (values are then left non-finite).
template <class MA>
__host__ __device__ inline bool eigvals(const MA& A0, c2* lam) {
  const int n = A0.n;
  MA H = A0;
  // Householder reduction to upper Hessenberg form
  for (int k = 0; k < n - 2; ++k) {
    double alpha2 = 0.0;
    for (int i = k + 1; i < n; ++i) alpha2 += abs2(H.at(i, k));
    const double alpha = sqrt(alpha2);
    if (alpha == 0.0) continue;
    c2 v[MA::kCols];
    const c2 x0 = H.at(k + 1, k);
    const double ax0 = cabs(x0);
    const c2 ph = ax0 == 0.0 ? C(1.0) : C(x0.re / ax0, x0.im / ax0);
    for (int i = 0; i < n; ++i) v[i] = C(0.0);
    v[k + 1] = add(x0, scale(ph, alpha));
    for (int i = k + 2; i < n; ++i) v[i] = H.at(i, k);
    double vn2 = 0.0;
    for (int i = k + 1; i < n; ++i) vn2 += abs2(v[i]);
    if (vn2 == 0.0) continue;
    // H = (I - 2 v v^H / vn2) H (I - 2 v v^H / vn2)
    for (int j = 0; j < n; ++j) {
      c2 s = C(0.0);
      for (int i = k + 1; i < n; ++i) s = add(s, cmulc(v[i], H.at(i, j)));
      s = scale(s, 2.0 / vn2);
      for (int i = k + 1; i < n; ++i) H.at(i, j) = sub(H.at(i, j), mul(v[i], s));
    }
    for (int i = 0; i < n; ++i) {
      c2 s = C(0.0);
      for (int j = k + 1; j < n; ++j) s = add(s, mul(H.at(i, j), v[j]));
      s = scale(s, 2.0 / vn2);
      for (int j = k + 1; j < n; ++j) H.at(i, j) = sub(H.at(i, j), mul(s, conj(v[j])));
    }
    for (int i = k + 2; i < n; ++i) H.at(i, k) = C(0.0);
  }
  int hi = n - 1;
  int iter = 0;
  while (hi >= 0) {
    if (hi == 0) {
      lam[0] = H.at(0, 0);
      break;
    }
    // find the start of the active unreduced block
    int lo = hi;
    while (lo > 0) {
      const double s = cabs(H.at(lo - 1, lo - 1)) + cabs(H.at(lo, lo));
      if (cabs(H.at(lo, lo - 1)) <= kEps * (s == 0.0 ? 1.0 : s)) {
        H.at(lo, lo - 1) = C(0.0);
        break;
      }
      --lo;
    }
    if (lo == hi) {
      lam[hi] = H.at(hi, hi);
      --hi;
      iter = 0;
      continue;
    }
    if (++iter > 200) {
      for (int i = 0; i <= hi; ++i) lam[i] = C(NAN, NAN);
      return false;
    }
    // Wilkinson shift from the trailing 2x2 of the active block
    const c2 a = H.at(hi - 1, hi - 1), b = H.at(hi - 1, hi), c = H.at(hi, hi - 1),
             d = H.at(hi, hi);
    const c2 tr2 = scale(add(a, d), 0.5);
    const c2 det = sub(mul(a, d), mul(b, c));
    const c2 disc = csqrt_(sub(mul(tr2, tr2), det));
    const c2 l1 = add(tr2, disc), l2 = sub(tr2, disc);
    c2 mu = cabs(sub(l1, d)) < cabs(sub(l2, d)) ? l1 : l2;
    if (iter % 11 == 10) mu = add(d, C(cabs(H.at(hi, hi - 1)), 0.0));  // exceptional shift
    // QR step on H[lo..hi] - mu I by Givens rotations, then RQ + mu I
    c2 gu[MA::kCols], gw[MA::kCols];
    for (int k = lo; k <= hi; ++k) H.at(k, k) = sub(H.at(k, k), mu);
    for (int k = lo; k < hi; ++k) {
      const c2 x = H.at(k, k), y = H.at(k + 1, k);
      const double r = hypot(cabs(x), cabs(y));
      if (r == 0.0) {
        gu[k] = C(1.0);
        gw[k] = C(0.0);
        continue;
      }
      // G = [[conj(u), conj(w)], [-w, u]] with u = x/r, w = y/r maps (x, y) to (r, 0)
      const c2 u = scale(x, 1.0 / r), w = scale(y, 1.0 / r);
      for (int j = k; j < n; ++j) {
        const c2 h1 = H.at(k, j), h2 = H.at(k + 1, j);
        H.at(k, j) = add(cmulc(u, h1), cmulc(w, h2));
        H.at(k + 1, j) = sub(mul(u, h2), mul(w, h1));
      }
      gu[k] = u;
      gw[k] = w;
      H.at(k + 1, k) = C(0.0);
    }
    for (int k = lo; k < hi; ++k) {
      const c2 u = gu[k], w = gw[k];
      // H = H * G^H with G = [[conj(u), conj(w)], [-w, u]] acting on columns k, k+1
      const int rmax = (k + 2 < hi ? k + 2 : hi);
      for (int i = 0; i <= rmax; ++i) {
        const c2 h1 = H.at(i, k), h2 = H.at(i, k + 1);
        H.at(i, k) = add(mul(h1, u), mul(h2, w));
        H.at(i, k + 1) = sub(mul(h2, conj(u)), mul(h1, conj(w)));
      }
    }
    for (int k = lo; k <= hi; ++k) H.at(k, k) = add(H.at(k, k), mu);
  }
  return true;
}

// Roots of the monic z^a + c[a-1] z^(a-1) + ... + c[0] (smallnum.py:90-107).
// Degree 1-2 closed forms; 3-4 as np.roots: trailing zero coefficients are
// roots at 0, the rest are companion-matrix eigenvalues.  Returns the count.
__host__ __device__ inline int poly_roots(const c2* coeffs, int a, c2* roots) {
  if (a == 1) {
    roots[0] = C(-coeffs[0].re, -coeffs[0].im);
    return 1;
  }
  if (a == 2) {
    const c2 c0 = coeffs[0], c1 = coeffs[1];
    const c2 s = csqrt_(sub(mul(c1, c1), scale(c0, 4.0)));
    const c2 mc1 = C(-c1.re, -c1.im);
    roots[0] = scale(sub(mc1, s), 0.5);
    roots[1] = scale(add(mc1, s), 0.5);
    return 2;
  }
  // np.roots(p), p = [1, c[a-1], ..., c[0]]: strip trailing zeros (roots at 0)
  int zeros = 0;
  while (zeros < a && coeffs[zeros].re == 0.0 && coeffs[zeros].im == 0.0) ++zeros;
  const int deg = a - zeros;
  MatT<4, 4> M;
  M.m = M.n = deg;
  for (int r = 0; r < deg; ++r)
    for (int c = 0; c < deg; ++c) M.at(r, c) = C(0.0);
  for (int r = 1; r < deg; ++r) M.at(r, r - 1) = C(1.0);
  for (int c = 0; c < deg; ++c) {
    const c2 pc = coeffs[a - 1 - c];  // p[c+1]
    M.at(0, c) = C(-pc.re, -pc.im);
  }
  int cnt = 0;
  if (deg > 0) {
    eigvals(M, roots);
    cnt = deg;
  }
  for (int z = 0; z < zeros; ++z) roots[cnt++] = C(0.0);
  return cnt;
}

}  // namespace la
}  // namespace afft
