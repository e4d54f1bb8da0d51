// K5: per-bucket sFFT-DT solve — locate (dt1 roots / dt2 grid enumeration /
// dt3 matrix pencil) and subspace-pursuit value estimation — for one bucket in
// one thread (oneshot.py:143-257, smallnum.py:110-142).
//
// Host+device so the same code is checked on the CPU against the oracle.  All
// arithmetic is IEEE float64 without contraction (nvcc --fmad=false, g++
// -ffp-contract=off); the numerically chaotic parts of the reference (ties of
// stable argsorts, the 1e-12 snap tie) follow the reference's rules.
#pragma once

#include "smallla.cuh"

namespace afft {
namespace dt {

using la::c2;
using la::MatT;
using M5 = MatT<5, 5>;    // pencil (a+1 <= 5)
using M4 = MatT<4, 4>;    // moment Hankel, pencil core
using MPur = MatT<la::kLaMaxRows, 8>;  // pursuit refits (p x up to 8 atoms)

constexpr int kMaxAm = 4;
constexpr int kMaxP = la::kLaMaxRows;   // random shifts per bucket
constexpr int kMaxFreqs = 3 * kMaxAm;   // candidate atoms {f, f+b, f-b}
constexpr int kSpMaxIters = 10;         // oneshot.py:23
constexpr int VAR_DT1 = 1, VAR_DT2 = 2, VAR_DT3 = 3;

__host__ __device__ __forceinline__ int64_t pmod(int64_t a, int64_t n) {
  const int64_t r = a % n;
  return r < 0 ? r + n : r;
}

// exp(-2j*pi*prod/n) as numpy evaluates it: theta = (-2*pi*prod) * (1/n)
__host__ __device__ __forceinline__ c2 unit_root_(int64_t prod, int64_t n) {
  const double theta = (-6.283185307179586 * (double)prod) * (1.0 / (double)n);
  double s, c;
#ifdef __CUDA_ARCH__
  sincos(theta, &s, &c);
#else
  s = sin(theta);
  c = cos(theta);
#endif
  return c2{c, s};
}

// exp(-2 pi i m / q) with the argument reduced exactly (sincospi), m in [0, q)
__host__ __device__ __forceinline__ c2 root_pi_(int64_t m, int64_t q) {
  double s, c;
#ifdef __CUDA_ARCH__
  sincospi(-2.0 * (double)m / (double)q, &s, &c);
#else
  const double th = -6.283185307179586 * ((double)m / (double)q);
  s = sin(th);
  c = cos(th);
#endif
  return c2{c, s};
}

// Python float modulo x % y for y > 0 (result in [0, y)).
__host__ __device__ __forceinline__ double pyfmod(double x, double y) {
  double m = fmod(x, y);
  if (m != 0.0) {
    if (m < 0.0) m += y;
  } else {
    m = 0.0;
  }
  return m;
}

// _snap_to_grid (oneshot.py:150-158)
__host__ __device__ inline int64_t snap_to_grid(c2 z, int64_t bucket, int64_t b, int64_t n) {
  const int64_t step = n / b;
  const double f_est = pyfmod((-atan2(z.im, z.re) * (double)n) / 6.283185307179586, (double)n);
  const double d = (f_est - (double)bucket) / (double)b;
  int64_t j = (int64_t)floor(d + 0.5);
  if (fabs(d - floor(d) - 0.5) < 1e-12) j = (int64_t)floor(d);
  return pmod(bucket + pmod(j, step) * b, n);
}

__host__ __device__ inline int sort_unique(int64_t* v, int cnt) {
  for (int i = 1; i < cnt; ++i) {
    const int64_t x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
  int u = 0;
  for (int i = 0; i < cnt; ++i)
    if (u == 0 || v[u - 1] != v[i]) v[u++] = v[i];
  return u;
}

__host__ __device__ __forceinline__ double vnorm(const c2* y, int m) {
  double sr = 0.0, si = 0.0;
  for (int i = 0; i < m; ++i) sr += y[i].re * y[i].re;
  for (int i = 0; i < m; ++i) si += y[i].im * y[i].im;
  return sqrt(sr + si);
}

// Structured moment m_t (t in [-a_m, 2a_m)) from the measurement row.
struct Moments {
  const c2* row;  // [3 a_m structured | p random]
  int a_m;
  __host__ __device__ __forceinline__ c2 m(int t) const { return row[t + a_m]; }
};

// pencil_eigenvalues (smallnum.py:110-142) for the (a+1)x(a+1) moment pencil
// pencil[r][c] = m_{r-c}; returns the number of roots (0 = none) or -1 when a
// root is not finite.
__host__ __device__ inline int pencil_roots(const Moments& M, int a, c2* roots) {
  const int size = a + 1;
  M5 full;
  full.m = full.n = size;
  for (int r = 0; r < size; ++r)
    for (int c = 0; c < size; ++c) full.at(r, c) = M.m(r - c);
  M5 W = full, V;
  double sv[5];
  la::svd_jacobi(W, sv, V);
  const double tol = sv[0] * 1e-10;
  int nrank = 0;
  for (int i = 0; i < size; ++i) nrank += sv[i] > tol;
  const int rank = a < nrank ? a : nrank;
  if (rank == 0) return 0;
  // row_basis = vh[:rank] = conj(V[:, :rank])^T; lead/lag drop the last/first column
  MatT<4, 4> lead, lag;
  lead.m = lag.m = rank;
  lead.n = lag.n = a;
  for (int i = 0; i < rank; ++i)
    for (int j = 0; j < a; ++j) {
      lead.at(i, j) = la::conj(V.at(j, i));
      lag.at(i, j) = la::conj(V.at(j + 1, i));
    }
  MatT<4, 4> P;
  la::pinv(lead, P, 1e-15);  // a x rank
  M4 core;
  core.m = core.n = rank;
  for (int i = 0; i < rank; ++i)
    for (int j = 0; j < rank; ++j) {
      c2 s = la::C(0.0);
      for (int k = 0; k < a; ++k) s = la::add(s, la::mul(lag.at(i, k), P.at(k, j)));
      core.at(i, j) = s;
    }
  la::eigvals(core, roots);
  for (int i = 0; i < rank; ++i) {
    roots[i] = la::conj(roots[i]);
    if (!la::finite(roots[i])) return -1;
  }
  return rank;
}

// Prony coefficients of the a-tone moment recursion (oneshot.py:182-188): the a x a
// Hankel lstsq H c = -m[a..2a).  False when a coefficient is not finite (-> None).
__host__ __device__ inline bool moment_coeffs(const Moments& M, int a, c2* coeffs) {
  M4 H;
  H.m = H.n = a;
  c2 rhs[kMaxAm];
  for (int r = 0; r < a; ++r) {
    for (int c = 0; c < a; ++c) H.at(r, c) = M.m(r + c);
    const c2 v = M.m(a + r);
    rhs[r] = la::C(-v.re, -v.im);
  }
  la::lstsq(H, rhs, coeffs, nullptr);
  for (int i = 0; i < a; ++i)
    if (!la::finite(coeffs[i])) return false;
  return true;
}

// |P(w^cand)| for the dt2 grid enumeration (oneshot.py:193-198), Horner from the
// leading 1.
__host__ __device__ __forceinline__ double poly_abs_at(const c2* coeffs, int a, int64_t cand,
                                                       int64_t n) {
  const c2 z = unit_root_(cand, n);
  c2 y = la::C(0.0);
  y = la::add(la::mul(y, z), la::C(1.0));
  for (int k = a - 1; k >= 0; --k) y = la::add(la::mul(y, z), coeffs[k]);
  return la::cabs(y);
}

// locate (oneshot.py:161-200).  Returns the number of candidate positions
// (sorted, unique), or -1 for "None" (degenerate bucket).
__host__ __device__ inline int locate(const Moments& M, int a, int variant, int64_t bucket,
                                      int64_t b, int64_t n, int64_t* pos) {
  if (a < 1) return 0;
  const int64_t step = n / b;
  c2 roots[5];
  if (variant == VAR_DT3) {
    const int nr = pencil_roots(M, a, roots);
    if (nr <= 0) return -1;  // empty or non-finite roots -> None
    for (int i = 0; i < nr; ++i) pos[i] = snap_to_grid(roots[i], bucket, b, n);
    return sort_unique(pos, nr);
  }
  c2 coeffs[kMaxAm];
  if (!moment_coeffs(M, a, coeffs)) return -1;
  if (variant == VAR_DT1) {
    const int nr = la::poly_roots(coeffs, a, roots);
    for (int i = 0; i < nr; ++i) pos[i] = snap_to_grid(roots[i], bucket, b, n);
    return sort_unique(pos, nr);
  }
  // dt2: |P(w^cand)| over every grid candidate, the `take` smallest (stable)
  const int take = (int64_t)a < step ? a : (int)step;
  double best[kMaxAm];
  int64_t bj[kMaxAm];
  int have = 0;
  for (int64_t j = 0; j < step; ++j) {
    const double v = poly_abs_at(coeffs, a, pmod(bucket + b * j, n), n);
    // insert into the sorted top-`take` list; equal values keep the earlier j
    if (have < take || v < best[have - 1]) {
      int i = have < take ? have++ : have - 1;
      while (i > 0 && best[i - 1] > v) {
        best[i] = best[i - 1];
        bj[i] = bj[i - 1];
        --i;
      }
      best[i] = v;
      bj[i] = j;
    }
  }
  for (int i = 0; i < have; ++i) pos[i] = pmod(bucket + b * bj[i], n);
  return sort_unique(pos, have);
}

// indices of the `want` largest values (stable: ties keep the lower index)
__host__ __device__ inline void top_desc(const double* v, int cnt, int want, int* out) {
  int have = 0;
  for (int i = 0; i < cnt; ++i) {
    if (have < want || v[i] > v[out[have - 1]]) {
      int k = have < want ? have++ : have - 1;
      while (k > 0 && v[out[k - 1]] < v[i]) {
        out[k] = out[k - 1];
        --k;
      }
      out[k] = i;
    }
  }
}

struct Pursuit {
  int P, F;
  c2 y[kMaxP];
  c2 atoms[kMaxP * kMaxFreqs];  // atoms[i * F + k]
  int64_t freqs[kMaxFreqs];
};

// lstsq of y on the atom columns `sup` (cnt of them); returns ||y - A_s coef||.
__host__ __device__ inline double refit(const Pursuit& S, const int* sup, int cnt, c2* coef) {
  MPur A;
  A.m = S.P;
  A.n = cnt;
  for (int i = 0; i < S.P; ++i)
    for (int c = 0; c < cnt; ++c) A.at(i, c) = S.atoms[i * S.F + sup[c]];
  la::lstsq(A, S.y, coef, nullptr);
  c2 r[kMaxP];
  for (int i = 0; i < S.P; ++i) {
    c2 acc = la::C(0.0);
    for (int c = 0; c < cnt; ++c) acc = la::add(acc, la::mul(S.atoms[i * S.F + sup[c]], coef[c]));
    r[i] = la::sub(S.y[i], acc);
  }
  return vnorm(r, S.P);
}

// |A^H v| per atom
__host__ __device__ inline void correlations(const Pursuit& S, const c2* v, double* out) {
  for (int k = 0; k < S.F; ++k) {
    c2 acc = la::C(0.0);
    for (int i = 0; i < S.P; ++i) acc = la::add(acc, la::cmulc(S.atoms[i * S.F + k], v[i]));
    out[k] = la::cabs(acc);
  }
}

// estimate_values (oneshot.py:203-257).  `rand` holds the p random-shift
// measurements, `shifts` the raw random shifts.  Returns the support size and
// fills positions / values in the reference's order.
__host__ __device__ inline int estimate_values(const c2* rand, const int64_t* shifts, int P,
                                               const int64_t* cands, int nc, int64_t b, int64_t n,
                                               int64_t* out_pos, c2* out_val) {
  Pursuit S;
  S.P = P;
  for (int i = 0; i < P; ++i) S.y[i] = rand[i];
  const double ynorm = vnorm(S.y, P);
  if (nc == 0 || ynorm == 0.0) return 0;
  S.F = 0;
  for (int c = 0; c < nc; ++c) {
    const int64_t f = cands[c];
    const int64_t g3[3] = {f, pmod(f + b, n), pmod(f - b, n)};
    for (int t = 0; t < 3; ++t) {
      bool seen = false;
      for (int k = 0; k < S.F; ++k) seen |= S.freqs[k] == g3[t];
      if (!seen) S.freqs[S.F++] = g3[t];
    }
  }
  for (int i = 0; i < P; ++i)
    for (int k = 0; k < S.F; ++k)
      S.atoms[i * S.F + k] = unit_root_(pmod(shifts[i], n) * S.freqs[k] % n, n);
  int want = nc;
  if (S.F < want) want = S.F;
  if (P < want) want = P;
  const double tol = 1e-10 * (ynorm > 1.0 ? ynorm : 1.0);
  double corr[kMaxFreqs];
  int sup[kMaxFreqs], best_sup[kMaxFreqs];
  c2 coef[kMaxFreqs], best_coef[kMaxFreqs];
  correlations(S, S.y, corr);
  top_desc(corr, S.F, want, sup);
  double best_res = refit(S, sup, want, coef);
  for (int i = 0; i < want; ++i) {
    best_sup[i] = sup[i];
    best_coef[i] = coef[i];
  }
  for (int it = 0; it < kSpMaxIters; ++it) {
    if (best_res <= tol) break;
    c2 resid[kMaxP];
    for (int i = 0; i < P; ++i) {
      c2 acc = la::C(0.0);
      for (int c = 0; c < want; ++c)
        acc = la::add(acc, la::mul(S.atoms[i * S.F + best_sup[c]], best_coef[c]));
      resid[i] = la::sub(S.y[i], acc);
    }
    int fresh[kMaxFreqs];
    correlations(S, resid, corr);
    top_desc(corr, S.F, want, fresh);
    // merged = union1d(best_sup, fresh): sorted unique
    int64_t mg[2 * kMaxFreqs];
    int nm = 0;
    for (int i = 0; i < want; ++i) mg[nm++] = best_sup[i];
    for (int i = 0; i < want; ++i) mg[nm++] = fresh[i];
    nm = sort_unique(mg, nm);
    int merged[2 * kMaxFreqs];
    for (int i = 0; i < nm; ++i) merged[i] = (int)mg[i];
    c2 coef_m[2 * kMaxFreqs];
    refit(S, merged, nm, coef_m);
    double mag[2 * kMaxFreqs];
    for (int i = 0; i < nm; ++i) mag[i] = la::cabs(coef_m[i]);
    int order[2 * kMaxFreqs];
    top_desc(mag, nm, want, order);
    int64_t pr[kMaxFreqs];
    for (int i = 0; i < want; ++i) pr[i] = merged[order[i]];
    sort_unique(pr, want);
    int pruned[kMaxFreqs];
    for (int i = 0; i < want; ++i) pruned[i] = (int)pr[i];
    const double res = refit(S, pruned, want, coef);
    if (res >= best_res) break;
    best_res = res;
    for (int i = 0; i < want; ++i) {
      best_sup[i] = pruned[i];
      best_coef[i] = coef[i];
    }
  }
  for (int i = 0; i < want; ++i) {
    out_pos[i] = S.freqs[best_sup[i]];
    out_val[i] = best_coef[i];
  }
  return want;
}

// One bucket's estimate step given located candidates (nc < 0 = None).
__host__ __device__ inline int estimate_bucket(const c2* row, int a_m, int P,
                                               const int64_t* rshifts, const int64_t* cands,
                                               int nc, int64_t b, int64_t n, int64_t* out_pos,
                                               c2* out_val) {
  if (nc < 0) return 0;
  return estimate_values(row + 3 * a_m, rshifts, P, cands, nc, b, n, out_pos, out_val);
}

// One bucket of sfft_dt's main loop (oneshot.py:279-288): locate then estimate.
// Returns the number of entries written (<= a), 0 for degenerate buckets.
__host__ __device__ inline int solve_bucket(const c2* row, int a_m, int P,
                                            const int64_t* rshifts, int a, int variant,
                                            int64_t bucket, int64_t b, int64_t n,
                                            int64_t* out_pos, c2* out_val) {
  if (a <= 0) return 0;
  Moments M{row, a_m};
  int64_t cands[5];
  const int nc = locate(M, a, variant, bucket, b, n, cands);
  if (nc < 0) return 0;
  return estimate_values(row + 3 * a_m, rshifts, P, cands, nc, b, n, out_pos, out_val);
}

}  // namespace dt
}  // namespace afft
