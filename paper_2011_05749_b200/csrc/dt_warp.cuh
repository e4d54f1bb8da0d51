// K5 (warp form): subspace-pursuit value estimation (oneshot.py:203-257) with one
// warp per bucket.  The per-thread form in oneshot_core.cuh runs the whole pursuit
// — up to 2 x 10 Jacobi least-squares refits — as one serial chain per bucket with
// ~22 KB of local-memory state; buckets that need many iterations set the kernel's
// duration (ncu: 3.6 active threads per warp, 3% occupancy).  Here lane i owns row
// i of the p x F atom dictionary (p <= 32), the refit's one-sided Jacobi keeps the
// working columns in registers and reduces its inner products with xor butterflies
// (identical in every lane, so control flow stays warp-uniform), and the small
// scalar bookkeeping (top-k, merge, sort) runs on lane 0 over shared memory.
//
// Same algorithm and tie rules as dt::estimate_values / la::lstsq; only the
// summation order of the row reductions differs (ulp-level).
//
// Group width W: 32 lanes per bucket, or 16 when p <= 16 (BASELINE's p = 15): two
// buckets share a warp, every row reduction is one butterfly level shorter, and the
// two halves run independently (their shuffles and syncs name only their own lanes).
#pragma once

#include "oneshot_core.cuh"

namespace afft {
namespace dtw {

using la::c2;
constexpr int kCols = 2 * dt::kMaxAm;  // merged support <= 2 * want <= 8

template <int W>
struct WarpPursuit {
  c2 A[dt::kMaxFreqs][W];  // atom k, row i
  c2 y[W];
  c2 r[W];
  c2 V[kCols][kCols];       // V[row j][col c]; the Jacobi refit keeps V's column c, row
                            // `lane`, at V[c][lane] while it rotates
  c2 Wk[kCols][W];          // refit working columns (column c, row `lane`)
  c2 x[kCols];              // refit solution
  c2 best_coef[dt::kMaxAm];
  c2 dot[kCols];
  double corr[dt::kMaxFreqs];
  double sig[kCols];
  int64_t freqs[dt::kMaxFreqs];
  int ord[kCols];
  int sup[kCols];
  int best_sup[dt::kMaxAm];
  int fresh[dt::kMaxAm];
  int pruned[dt::kMaxAm];
  double mag[kCols];
  int F;
};

// the calling group's lane mask (its W lanes of the warp)
template <int W>
__device__ __forceinline__ unsigned gmask() {
  return W == 32 ? 0xffffffffu : ((0xffffffffu >> (32 - W)) << (threadIdx.x & (32 - W)));
}

template <int W>
__device__ __forceinline__ double wsum(double v) {
  const unsigned m = gmask<W>();
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
  return v;
}

// ||v|| over rows < P as vnorm does (real and imaginary squares summed apart).
template <int W>
__device__ __forceinline__ double warp_vnorm(c2 v, int P, int lane) {
  const bool on = lane < P;
  const double sr = wsum<W>(on ? v.re * v.re : 0.0);
  const double si = wsum<W>(on ? v.im * v.im : 0.0);
  return sqrt(sr + si);
}

// refit (oneshot.py:229-232): x = lstsq(A[:, sup], y) with numpy's cutoff; returns
// ||y - A_s x||.  S.sup[0..cnt) are atom indices; the solution lands in S.x.
// Working columns live in shared memory (S.Wk[c][row], V column c at S.V[c][row]) and
// the loops stay rolled: the unrolled register form was ~40k SASS instructions per
// kernel and ncu charged 68% of the stall samples to instruction fetch.
template <int W>
__device__ __noinline__ double warp_refit(WarpPursuit<W>& S, int P, int cnt, int lane) {
  const unsigned gm = gmask<W>();
  for (int c = 0; c < cnt; ++c) {
    S.Wk[c][lane] = lane < P ? S.A[S.sup[c]][lane] : la::C(0.0);
    if (lane < cnt) S.V[c][lane] = la::C(lane == c ? 1.0 : 0.0);
  }
  const c2 yl = lane < P ? S.y[lane] : la::C(0.0);
  __syncwarp(gm);
#pragma unroll 1
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
#pragma unroll 1
    for (int p = 0; p < cnt - 1; ++p) {
#pragma unroll 1
      for (int q = p + 1; q < cnt; ++q) {
        const c2 wp = S.Wk[p][lane], wq = S.Wk[q][lane];
        const double alpha = wsum<W>(la::abs2(wp));
        const double beta = wsum<W>(la::abs2(wq));
        const c2 gl = la::cmulc(wp, wq);
        const c2 gamma = la::C(wsum<W>(gl.re), wsum<W>(gl.im));
        const double g = la::cabs(gamma);
        if (g == 0.0 || g <= la::kEps * sqrt(alpha * beta)) continue;
        rotated = true;
        const c2 ph = la::C(gamma.re / g, gamma.im / g);
        const double zeta = (beta - alpha) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
        {
          const c2 aq = la::cmulc(ph, wq);
          S.Wk[p][lane] = la::sub(la::scale(wp, cs), la::scale(aq, sn));
          S.Wk[q][lane] = la::add(la::scale(wp, sn), la::scale(aq, cs));
        }
        if (lane < cnt) {
          const c2 vp = S.V[p][lane], vq = la::cmulc(ph, S.V[q][lane]);
          S.V[p][lane] = la::sub(la::scale(vp, cs), la::scale(vq, sn));
          S.V[q][lane] = la::add(la::scale(vp, sn), la::scale(vq, cs));
        }
        __syncwarp(gm);
      }
    }
    if (!rotated) break;
  }
  // singular values and u_k^H y numerators (lane 0), V rows for the solution
#pragma unroll 1
  for (int c = 0; c < cnt; ++c) {
    const c2 wc = S.Wk[c][lane];
    const double s2 = wsum<W>(la::abs2(wc));
    const c2 dl = la::cmulc(wc, yl);
    const c2 d = la::C(wsum<W>(dl.re), wsum<W>(dl.im));
    if (lane == 0) {
      S.sig[c] = sqrt(s2);
      S.dot[c] = d;
    }
  }
  __syncwarp(gm);
  if (lane == 0) {  // selection sort descending (svd_jacobi's swaps, on a permutation)
    for (int j = 0; j < cnt; ++j) S.ord[j] = j;
    for (int j = 0; j < cnt; ++j) {
      int best = j;
      for (int k = j + 1; k < cnt; ++k)
        if (S.sig[k] > S.sig[best]) best = k;
      if (best != j) {
        const double ts = S.sig[j];
        S.sig[j] = S.sig[best];
        S.sig[best] = ts;
        const int to = S.ord[j];
        S.ord[j] = S.ord[best];
        S.ord[best] = to;
      }
    }
  }
  __syncwarp(gm);
  if (lane < cnt) {  // x_j = sum_k V[j][k] (u_k^H y) / s_k, k descending, above the cutoff
    const double cutoff = la::kEps * (double)(P > cnt ? P : cnt) * S.sig[0];
    c2 xj = la::C(0.0);
    for (int r = 0; r < cnt; ++r) {
      if (!(S.sig[r] > cutoff)) continue;
      const int k = S.ord[r];
      const c2 coef = la::scale(S.dot[k], 1.0 / (S.sig[r] * S.sig[r]));
      xj = la::add(xj, la::mul(S.V[k][lane], coef));
    }
    S.x[lane] = xj;
  }
  __syncwarp(gm);
  c2 acc = la::C(0.0);
  if (lane < P)
    for (int c = 0; c < cnt; ++c) acc = la::add(acc, la::mul(S.A[S.sup[c]][lane], S.x[c]));
  return warp_vnorm<W>(la::sub(yl, acc), P, lane);
}

// refit by Householder QR, lanes over rows: cnt reflector steps, each one norm
// reduction plus independent dot reductions for the trailing columns and y —
// ~20x fewer dependent butterflies than the Jacobi sweeps.  For a full-rank
// least-squares problem the solution is unique, so this agrees with the SVD
// form to rounding; when the R diagonal spans more than 1e7 (possible rank
// deficiency, where numpy's eps cutoff could bite) the Jacobi form decides.
// R ends up in S.Wk: R[j][k] = S.Wk[k][j] for j <= k.
template <int W>
__device__ __noinline__ double warp_refit_qr(WarpPursuit<W>& S, int P, int cnt, int lane) {
  const unsigned gm = gmask<W>();
  for (int c = 0; c < cnt; ++c) S.Wk[c][lane] = lane < P ? S.A[S.sup[c]][lane] : la::C(0.0);
  const c2 yl = lane < P ? S.y[lane] : la::C(0.0);
  c2 qy = yl;
  double dmax = 0.0, dmin = 1e300;
  __syncwarp(gm);
#pragma unroll 1
  for (int j = 0; j < cnt; ++j) {
    const bool below = lane >= j && lane < P;
    const c2 wj = S.Wk[j][lane];
    const double nx = sqrt(wsum<W>(below ? la::abs2(wj) : 0.0));
    const c2 x0 = S.Wk[j][j];
    dmax = nx > dmax ? nx : dmax;
    dmin = nx < dmin ? nx : dmin;
    if (nx == 0.0) break;
    const double a0 = la::cabs(x0);
    const c2 ph = a0 > 0.0 ? la::C(x0.re / a0, x0.im / a0) : la::C(1.0);
    const c2 alpha = la::C(-ph.re * nx, -ph.im * nx);
    const c2 v = lane == j ? la::sub(x0, alpha) : (below ? wj : la::C(0.0));
    const double inv = 2.0 / (2.0 * nx * (nx + a0));  // 2 / v^H v
#pragma unroll 1
    for (int k = j + 1; k < cnt; ++k) {
      const c2 wk = S.Wk[k][lane];
      const c2 dl = la::cmulc(v, wk);
      const c2 d = la::C(wsum<W>(dl.re), wsum<W>(dl.im));
      S.Wk[k][lane] = la::sub(wk, la::mul(v, la::scale(d, inv)));
    }
    {
      const c2 dl = la::cmulc(v, qy);
      const c2 d = la::C(wsum<W>(dl.re), wsum<W>(dl.im));
      qy = la::sub(qy, la::mul(v, la::scale(d, inv)));
    }
    __syncwarp(gm);
    if (lane == j) S.Wk[j][lane] = alpha;
    __syncwarp(gm);
  }
  if (!(dmin > 1e-7 * dmax)) return warp_refit<W>(S, P, cnt, lane);
  if (lane < cnt) S.dot[lane] = qy;
  __syncwarp(gm);
  if (lane == 0) {  // back substitution R x = Q^H y
    for (int j = cnt - 1; j >= 0; --j) {
      c2 sacc = S.dot[j];
      for (int k = j + 1; k < cnt; ++k) sacc = la::sub(sacc, la::mul(S.Wk[k][j], S.x[k]));
      S.x[j] = la::div(sacc, S.Wk[j][j]);
    }
  }
  __syncwarp(gm);
  c2 acc = la::C(0.0);
  if (lane < P)
    for (int c = 0; c < cnt; ++c) acc = la::add(acc, la::mul(S.A[S.sup[c]][lane], S.x[c]));
  return warp_vnorm<W>(la::sub(yl, acc), P, lane);
}

// |A^H v| per atom (v in shared memory), lanes over atoms; then lane 0 picks the
// `want` largest (stable) into out[].
template <int W>
__device__ __forceinline__ void warp_top_corr(WarpPursuit<W>& S, const c2* vec, int P, int want,
                                              int* out, int lane) {
  if (lane < S.F) {
    c2 acc = la::C(0.0);
    for (int i = 0; i < P; ++i) acc = la::add(acc, la::cmulc(S.A[lane][i], vec[i]));
    S.corr[lane] = la::cabs(acc);
  }
  __syncwarp(gmask<W>());
  if (lane == 0) dt::top_desc(S.corr, S.F, want, out);
  __syncwarp(gmask<W>());
}

// estimate_values (oneshot.py:203-257) for one bucket, called by all 32 lanes.
// Returns the support size; lane 0 writes positions/values (stride 1).
template <int W>
__device__ inline int warp_estimate(WarpPursuit<W>& S, const c2* rand, const int64_t* shifts, int P,
                                    const int64_t* cands, int nc, int64_t b, int64_t n,
                                    int64_t* out_pos, c2* out_val) {
  const int lane = threadIdx.x & (W - 1);
  const c2 yl = lane < P ? rand[lane] : la::C(0.0);
  S.y[lane] = yl;
  const double ynorm = warp_vnorm<W>(yl, P, lane);
  if (nc == 0 || ynorm == 0.0) return 0;
  if (lane == 0) {
    int F = 0;
    for (int c = 0; c < nc; ++c) {
      const int64_t f = cands[c];
      const int64_t g3[3] = {f, dt::pmod(f + b, n), dt::pmod(f - b, n)};
      for (int t = 0; t < 3; ++t) {
        bool seen = false;
        for (int k = 0; k < F; ++k) seen |= S.freqs[k] == g3[t];
        if (!seen) S.freqs[F++] = g3[t];
      }
    }
    S.F = F;
  }
  __syncwarp(gmask<W>());
  const int F = S.F;
  if (lane < P) {
    const int64_t sh = dt::pmod(shifts[lane], n);
    for (int k = 0; k < F; ++k) S.A[k][lane] = dt::unit_root_(sh * S.freqs[k] % n, n);
  }
  __syncwarp(gmask<W>());
  int want = nc;
  if (F < want) want = F;
  if (P < want) want = P;
  const double tol = 1e-10 * (ynorm > 1.0 ? ynorm : 1.0);
  warp_top_corr(S, S.y, P, want, S.sup, lane);
  double best_res = warp_refit_qr(S, P, want, lane);
  if (lane < want) {
    S.best_sup[lane] = S.sup[lane];
    S.best_coef[lane] = S.x[lane];
  }
  __syncwarp(gmask<W>());
  for (int it = 0; it < dt::kSpMaxIters; ++it) {
    if (best_res <= tol) break;
    c2 acc = la::C(0.0);
    if (lane < P)
      for (int c = 0; c < want; ++c)
        acc = la::add(acc, la::mul(S.A[S.best_sup[c]][lane], S.best_coef[c]));
    S.r[lane] = la::sub(yl, acc);
    __syncwarp(gmask<W>());
    warp_top_corr(S, S.r, P, want, S.fresh, lane);
    int nm = 0;
    if (lane == 0) {  // merged = union1d(best_sup, fresh)
      int64_t mg[2 * dt::kMaxAm];
      for (int i = 0; i < want; ++i) mg[nm++] = S.best_sup[i];
      for (int i = 0; i < want; ++i) mg[nm++] = S.fresh[i];
      nm = dt::sort_unique(mg, nm);
      for (int i = 0; i < nm; ++i) S.sup[i] = (int)mg[i];
    }
    nm = __shfl_sync(gmask<W>(), nm, 0, W);
    __syncwarp(gmask<W>());
    warp_refit_qr(S, P, nm, lane);
    if (lane == 0) {  // keep the `want` largest |coef|, sorted by atom index
      for (int i = 0; i < nm; ++i) S.mag[i] = la::cabs(S.x[i]);
      int order[kCols];
      dt::top_desc(S.mag, nm, want, order);
      int64_t pr[dt::kMaxAm];
      for (int i = 0; i < want; ++i) pr[i] = S.sup[order[i]];
      dt::sort_unique(pr, want);
      for (int i = 0; i < want; ++i) S.sup[i] = (int)pr[i];
    }
    __syncwarp(gmask<W>());
    const double res = warp_refit_qr(S, P, want, lane);
    if (res >= best_res) break;
    best_res = res;
    if (lane < want) {
      S.best_sup[lane] = S.sup[lane];
      S.best_coef[lane] = S.x[lane];
    }
    __syncwarp(gmask<W>());
  }
  if (lane < want) {
    out_pos[lane] = S.freqs[S.best_sup[lane]];
    out_val[lane] = S.best_coef[lane];
  }
  return want;
}

}  // namespace dtw
}  // namespace afft
