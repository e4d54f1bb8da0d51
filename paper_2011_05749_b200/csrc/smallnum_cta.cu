// smallnum API (smallnum.py:54-142) for shapes beyond the per-thread templates:
// any matrix up to the reference's 64 x 64 cap (MAX_DIM, smallnum.py:15,21-29),
// one CTA of 256 threads per call.
//
//   svd      one-sided (Hestenes) Jacobi on the tall orientation, disjoint column
//            pairs of a round-robin tournament rotated by one warp each; the left
//            basis completed by two-pass Gram-Schmidt against the unit vectors
//   lstsq    the SVD with numpy's cutoff eps * max(m, n) * s_max (lstsq rcond=None),
//            x = sum_{s_i > cut} v_i (w_i^H b) / s_i^2, residual ||a x - b||
//   eigvals  Householder reduction to Hessenberg form (threads over rows/columns),
//            then single-shift complex QR with Wilkinson shifts and deflation, one
//            warp (lanes over the rotated rows / columns)
//   pencil   SVD of the (a+1) x (a+1) pencil, numerical rank at 1e-10 s_0, the
//            top-`rank` right singular rows split into lead / lag, core = lag
//            pinv(lead) (pinv cutoff 1e-15 s_max, numpy's default), conj(eigvals)
//
// Matrices live column-major in a global scratch block (64 KB each at 64 x 64,
// L2-resident); __syncthreads orders the CTA's global accesses.  This is the
// drop-in module's path for large shapes; the hot-path solvers use the
// register templates of smallla.cuh.
#include <cmath>

#include "afft_common.cuh"

namespace afft {
namespace cta_la {

constexpr int kMax = 64;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr double kEps = 2.220446049250313e-16;

struct z {
  double re, im;
};
__device__ __forceinline__ z zc(double r, double i = 0.0) { return z{r, i}; }
__device__ __forceinline__ z zadd(z a, z b) { return z{a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ z zsub(z a, z b) { return z{a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ z zmul(z a, z b) {
  return z{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ z zconj(z a) { return z{a.re, -a.im}; }
// conj(a) * b
__device__ __forceinline__ z zcmul(z a, z b) {
  return z{a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
__device__ __forceinline__ z zscale(z a, double s) { return z{a.re * s, a.im * s}; }
__device__ __forceinline__ double zabs2(z a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ double zabs(z a) { return hypot(a.re, a.im); }
__device__ __forceinline__ z zdiv(z a, z b) {
  const double d = zabs2(b);
  return z{(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
__device__ __forceinline__ z zsqrt(z a) {
  const double r = zabs(a);
  if (r == 0.0) return zc(0.0);
  double re = sqrt(0.5 * (r + fabs(a.re)));
  double im = a.im / (2.0 * re);
  if (a.re < 0.0) {
    const double t = fabs(im);
    im = a.im >= 0.0 ? re : -re;
    re = t;
  }
  return z{re, im};
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// column-major element (row i, column j) of a matrix with leading dimension ld
#define AT(A, i, j, ld) (A)[(size_t)(j) * (ld) + (i)]

// One-sided Jacobi SVD of W (M x N, M >= N, column-major, ld M), in place: on exit
// W = U S (columns w_j = s_j u_j), V (N x N, ld N) the right basis, s the column
// norms (unsorted), order[] the indices by descending s (ties by index).
__device__ void jacobi_svd(z* W, int M, int N, z* V, double* s, int* order) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int rotated;
  for (int e = tid; e < N * N; e += kThreads) V[e] = zc((e % N) == (e / N) ? 1.0 : 0.0);
  const int P = N + (N & 1);  // tournament size (a dummy column when N is odd)
  __syncthreads();
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < P - 1; ++round) {
      // round-robin pairs: position 0 fixed, the others rotate
      for (int pr = warp; pr < P / 2; pr += kWarps) {
        int a = pr == 0 ? 0 : 1 + (pr - 1 + round) % (P - 1);
        int b = 1 + (P - 2 - pr + round) % (P - 1);
        if (a >= N || b >= N) continue;
        const int p = a < b ? a : b, q = a < b ? b : a;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        for (int i = lane; i < M; i += 32) {
          const z wp = AT(W, i, p, M), wq = AT(W, i, q, M);
          al += zabs2(wp);
          be += zabs2(wq);
          const z g = zcmul(wp, wq);
          gr += g.re;
          gi += g.im;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        gr = warp_sum(gr);
        gi = warp_sum(gi);
        const double ga = hypot(gr, gi);
        if (!(ga > 1e-15 * sqrt(al * be)) || ga == 0.0) continue;
        if (lane == 0) rotated = 1;
        const z ph = z{gr / ga, -gi / ga};  // e^{-i phi}: makes w_p^H (w_q ph) real
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int i = lane; i < M; i += 32) {
          const z wp = AT(W, i, p, M), wq = zmul(AT(W, i, q, M), ph);
          AT(W, i, p, M) = zsub(zscale(wp, c), zscale(wq, sn));
          AT(W, i, q, M) = zadd(zscale(wp, sn), zscale(wq, c));
        }
        for (int i = lane; i < N; i += 32) {
          const z vp = AT(V, i, p, N), vq = zmul(AT(V, i, q, N), ph);
          AT(V, i, p, N) = zsub(zscale(vp, c), zscale(vq, sn));
          AT(V, i, q, N) = zadd(zscale(vp, sn), zscale(vq, c));
        }
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  for (int j = warp; j < N; j += kWarps) {
    double acc = 0.0;
    for (int i = lane; i < M; i += 32) acc += zabs2(AT(W, i, j, M));
    acc = warp_sum(acc);
    if (lane == 0) s[j] = sqrt(acc);
  }
  __syncthreads();
  if (tid < N) {  // rank of s[tid] in descending order, ties by index
    int r = 0;
    for (int j = 0; j < N; ++j) r += s[j] > s[tid] || (s[j] == s[tid] && j < tid);
    order[r] = tid;
  }
  __syncthreads();
}

// Left basis U (M x M, column-major) from W = U S: u_k = w_{order[k]} / s for the
// nonzero singular values, completed to a unitary basis by two-pass Gram-Schmidt
// against the unit vectors e_0, e_1, ...  Returns after a __syncthreads.
__device__ void complete_left(const z* W, int M, int N, const double* s, const int* order,
                              z* U, z* tmp) {
  const int tid = threadIdx.x;
  __shared__ int have;
  __shared__ double nrm;
  const double smax = N ? s[order[0]] : 0.0;
  if (tid == 0) have = 0;
  __syncthreads();
  for (int k = 0; k < N; ++k) {
    const int j = order[k];
    const double sj = s[j];
    if (!(sj > kEps * M * smax)) break;  // numerically zero: completed below
    for (int i = tid; i < M; i += kThreads) AT(U, i, k, M) = zscale(AT(W, i, j, M), 1.0 / sj);
    __syncthreads();
    if (tid == 0) have = k + 1;
    __syncthreads();
  }
  for (int e = 0; e < M && have < M; ++e) {
    for (int i = tid; i < M; i += kThreads) tmp[i] = zc(i == e ? 1.0 : 0.0);
    __syncthreads();
    const int h = have;
    for (int pass = 0; pass < 2; ++pass) {
      // d_k = u_k^H v (threads over k), then v -= sum_k u_k d_k (threads over rows)
      for (int k = tid; k < h; k += kThreads) {
        z d = zc(0.0);
        for (int i = 0; i < M; ++i) d = zadd(d, zcmul(AT(U, i, k, M), tmp[i]));
        tmp[kMax + k] = d;
      }
      __syncthreads();
      for (int i = tid; i < M; i += kThreads) {
        z v = tmp[i];
        for (int k = 0; k < h; ++k) v = zsub(v, zmul(AT(U, i, k, M), tmp[kMax + k]));
        tmp[i] = v;
      }
      __syncthreads();
    }
    if (tid < 32) {
      double acc = 0.0;
      for (int i = tid; i < M; i += 32) acc += zabs2(tmp[i]);
      acc = warp_sum(acc);
      if (tid == 0) nrm = sqrt(acc);
    }
    __syncthreads();
    const double nv = nrm;
    if (nv >= 1e-8) {
      for (int i = tid; i < M; i += kThreads) AT(U, i, h, M) = zscale(tmp[i], 1.0 / nv);
      __syncthreads();
      if (tid == 0) have = h + 1;
    }
    __syncthreads();
  }
}

// Eigenvalues of the n x n column-major H (destroyed): Hessenberg reduction by
// Householder reflectors, then single-shift complex QR with deflation.
__device__ void eigvals(z* H, int n, z* lam, z* vbuf) {
  const int tid = threadIdx.x;
  __shared__ double vnorm2;
  for (int k = 0; k + 2 < n; ++k) {
    // reflector for x = H[k+1:, k]: v = x + e^{i arg x0} ||x|| e_0
    if (tid < 32) {
      double acc = 0.0;
      for (int i = k + 1 + tid; i < n; i += 32) acc += zabs2(AT(H, i, k, n));
      acc = warp_sum(acc);
      if (tid == 0) {
        const double xn = sqrt(acc);
        const z x0 = AT(H, k + 1, k, n);
        const double a0 = zabs(x0);
        const z ph = a0 > 0.0 ? zscale(x0, 1.0 / a0) : zc(1.0);
        vbuf[k + 1] = zadd(x0, zscale(ph, xn));
        vnorm2 = acc - zabs2(x0) + zabs2(vbuf[k + 1]);
      }
      for (int i = k + 2 + tid; i < n; i += 32) vbuf[i] = AT(H, i, k, n);
    }
    __syncthreads();
    const double vv = vnorm2;
    if (vv > 0.0) {
      // left: H[k+1:, j] -= v (2 v^H H[k+1:, j] / vv), threads over columns
      for (int j = tid; j < n; j += kThreads) {
        z w = zc(0.0);
        for (int i = k + 1; i < n; ++i) w = zadd(w, zcmul(vbuf[i], AT(H, i, j, n)));
        w = zscale(w, 2.0 / vv);
        for (int i = k + 1; i < n; ++i) AT(H, i, j, n) = zsub(AT(H, i, j, n), zmul(vbuf[i], w));
      }
      __syncthreads();
      // right: H[i, k+1:] -= (2 H[i, k+1:] v / vv) v^H, threads over rows
      for (int i = tid; i < n; i += kThreads) {
        z w = zc(0.0);
        for (int j = k + 1; j < n; ++j) w = zadd(w, zmul(AT(H, i, j, n), vbuf[j]));
        w = zscale(w, 2.0 / vv);
        for (int j = k + 1; j < n; ++j)
          AT(H, i, j, n) = zsub(AT(H, i, j, n), zmul(w, zconj(vbuf[j])));
      }
    }
    __syncthreads();
    for (int i = k + 2 + tid; i < n; i += kThreads) AT(H, i, k, n) = zc(0.0);
    __syncthreads();
  }
  if (tid >= 32) return;  // the QR iteration is one warp
  const int lane = tid;
  int hi = n - 1, iter = 0;
  while (hi >= 0) {
    int l = hi;
    while (l > 0) {
      const double sub = zabs(AT(H, l, l - 1, n));
      double ref = zabs(AT(H, l - 1, l - 1, n)) + zabs(AT(H, l, l, n));
      if (ref == 0.0) ref = 1.0;
      if (sub <= kEps * ref) break;
      --l;
    }
    if (l > 0) {
      if (lane == 0) AT(H, l, l - 1, n) = zc(0.0);
      __syncwarp();
    }
    if (l == hi) {
      if (lane == 0) lam[hi] = AT(H, hi, hi, n);
      --hi;
      iter = 0;
      continue;
    }
    // Wilkinson shift: the eigenvalue of the trailing 2 x 2 closer to its last entry
    const z a = AT(H, hi - 1, hi - 1, n), b = AT(H, hi - 1, hi, n);
    const z c = AT(H, hi, hi - 1, n), d = AT(H, hi, hi, n);
    z mu;
    if (iter > 0 && iter % 11 == 0) {  // exceptional shift
      mu = zadd(d, zc(0.75 * zabs(c), 0.0));
    } else {
      const z tr2 = zscale(zadd(a, d), 0.5);
      const z dif = zscale(zsub(a, d), 0.5);
      const z disc = zsqrt(zadd(zmul(dif, dif), zmul(b, c)));
      const z l1 = zadd(tr2, disc), l2 = zsub(tr2, disc);
      mu = zabs2(zsub(l1, d)) <= zabs2(zsub(l2, d)) ? l1 : l2;
    }
    ++iter;
    if (iter > 60 * n) {  // give up on this window: report its diagonal
      for (int i = l + lane; i <= hi; i += 32) lam[i] = AT(H, i, i, n);
      __syncwarp();
      hi = l - 1;
      iter = 0;
      continue;
    }
    z x = zsub(AT(H, l, l, n), mu), y = AT(H, l + 1, l, n);
    for (int k = l; k < hi; ++k) {
      if (k > l) {
        x = AT(H, k, k - 1, n);
        y = AT(H, k + 1, k - 1, n);
      }
      const double ax = zabs(x), ay = zabs(y);
      const double r = hypot(ax, ay);
      if (r == 0.0) continue;
      const double cg = ax / r;
      const z sg = ax > 0.0 ? zscale(zmul(zscale(x, 1.0 / ax), zconj(y)), 1.0 / r)
                            : zscale(zconj(y), 1.0 / ay);
      // rows k, k+1 over the window's columns, then columns k, k+1 over its rows
      const int c0 = k > l ? k - 1 : l;
      for (int j = c0 + lane; j <= hi; j += 32) {
        const z u = AT(H, k, j, n), v = AT(H, k + 1, j, n);
        AT(H, k, j, n) = zadd(zscale(u, cg), zmul(sg, v));
        AT(H, k + 1, j, n) = zsub(zscale(v, cg), zmul(zconj(sg), u));
      }
      __syncwarp();
      const int r1 = k + 2 < hi ? k + 2 : hi;
      for (int i = l + lane; i <= r1; i += 32) {
        const z u = AT(H, i, k, n), v = AT(H, i, k + 1, n);
        AT(H, i, k, n) = zadd(zscale(u, cg), zmul(zconj(sg), v));
        AT(H, i, k + 1, n) = zsub(zscale(v, cg), zmul(sg, u));
      }
      __syncwarp();
    }
  }
  __syncwarp();
}

enum { OP_SVD = 0, OP_LSTSQ = 1, OP_EIGVALS = 2, OP_PENCIL = 4 };

// Scratch: 6 matrices of kMax x kMax plus vectors.
__global__ void __launch_bounds__(kThreads) small_la_cta_kernel(
    int op, int m, int n, const double* __restrict__ a_in, const double* __restrict__ b_in,
    int rank_req, double* out_u, double* out_s, double* out_v, double* out_x, int* out_i,
    z* scratch) {
  const int tid = threadIdx.x;
  z* A0 = scratch;
  z* W = A0 + kMax * kMax;
  z* V = W + kMax * kMax;
  z* U = V + kMax * kMax;
  z* X = U + kMax * kMax;
  z* Y = X + kMax * kMax;
  z* vec = Y + kMax * kMax;  // 4 * kMax
  __shared__ double s[kMax];
  __shared__ int order[kMax];
  const z* a = reinterpret_cast<const z*>(a_in);
  if (op == OP_SVD || op == OP_LSTSQ) {
    const bool wide = m < n;  // SVD of a^H for wide inputs
    const int M = wide ? n : m, N = wide ? m : n;
    for (int e = tid; e < m * n; e += kThreads) {
      const int r = e / n, c = e % n;
      const z v = a[e];
      AT(A0, r, c, m) = v;
      if (!wide) AT(W, r, c, M) = v;
      else AT(W, c, r, M) = zconj(v);
    }
    __syncthreads();
    jacobi_svd(W, M, N, V, s, order);
    if (op == OP_SVD) {
      complete_left(W, M, N, s, order, U, vec);
      for (int k = tid; k < N; k += kThreads) out_s[k] = s[order[k]];
      // a = U S V^H (tall) or a = V S U^H (wide, from a^H = U S V^H):
      // u = (tall ? U : V-sorted), v = (tall ? V-sorted : U), row-major
      z* ou = reinterpret_cast<z*>(out_u);
      z* ov = reinterpret_cast<z*>(out_v);
      for (int e = tid; e < M * M; e += kThreads) {
        const int r = e / M, c = e % M;
        (wide ? ov : ou)[r * M + c] = AT(U, r, c, M);
      }
      for (int e = tid; e < N * N; e += kThreads) {
        const int r = e / N, c = e % N;
        (wide ? ou : ov)[r * N + c] = AT(V, r, order[c], N);
      }
      return;
    }
    // lstsq (m >= n): cutoff eps * max(m, n) * s_max
    const double smax = s[order[0]];
    const double cut = kEps * (double)(m > n ? m : n) * smax;
    const z* b = reinterpret_cast<const z*>(b_in);
    z* coef = vec;  // (w_j^H b) / s_j^2, zero below the cutoff
    for (int j = tid; j < n; j += kThreads) {
      z d = zc(0.0);
      if (s[j] > cut) {
        for (int i = 0; i < m; ++i) d = zadd(d, zcmul(AT(W, i, j, m), b[i]));
        d = zscale(d, 1.0 / (s[j] * s[j]));
      }
      coef[j] = d;
    }
    __syncthreads();
    z* x = vec + kMax;
    for (int r = tid; r < n; r += kThreads) {
      z acc = zc(0.0);
      for (int j = 0; j < n; ++j) acc = zadd(acc, zmul(AT(V, r, j, n), coef[j]));
      x[r] = acc;
      out_x[2 * r] = acc.re;
      out_x[2 * r + 1] = acc.im;
    }
    __syncthreads();
    if (tid < 32) {
      double acc = 0.0;
      for (int i = tid; i < m; i += 32) {
        z t = zc(0.0);
        for (int j = 0; j < n; ++j) t = zadd(t, zmul(AT(A0, i, j, m), x[j]));
        acc += zabs2(zsub(t, b[i]));
      }
      acc = warp_sum(acc);
      if (tid == 0) {
        out_s[n] = sqrt(acc);
        int rank = 0;
        for (int j = 0; j < n; ++j) rank += s[j] > cut;
        out_i[0] = rank;
      }
    }
    for (int k = tid; k < n; k += kThreads) out_s[k] = s[order[k]];
    return;
  }
  if (op == OP_EIGVALS) {
    for (int e = tid; e < n * n; e += kThreads) AT(W, e / n, e % n, n) = a[e];
    __syncthreads();
    eigvals(W, n, vec, vec + kMax);
    __syncthreads();
    for (int j = tid; j < n; j += kThreads) {
      out_x[2 * j] = vec[j].re;
      out_x[2 * j + 1] = vec[j].im;
    }
    if (tid == 0) out_i[0] = 1;
    return;
  }
  if (op == OP_PENCIL) {  // a = the full size x size pencil [y1 | y2[:, -1]]
    const int size = m, an = m - 1;
    for (int e = tid; e < size * size; e += kThreads) AT(W, e / size, e % size, size) = a[e];
    __syncthreads();
    jacobi_svd(W, size, size, V, s, order);
    const double tol = s[order[0]] * 1e-10;
    __shared__ int nrank_s;
    if (tid == 0) {
      int r = 0;
      for (int i = 0; i < size; ++i) r += s[i] > tol;
      nrank_s = r;
      out_i[1] = rank_req <= r ? 1 : 0;
      out_i[0] = rank_req < r ? rank_req : r;
    }
    __syncthreads();
    const int rank = rank_req < nrank_s ? rank_req : nrank_s;
    if (rank == 0) return;
    // row basis vh[:rank, :] = conj(v_{order[i]})^T; lead = vh[:, :-1], lag = vh[:, 1:].
    // pinv(lead) via the SVD of T = lead^H (an x rank, tall): X holds T.
    for (int e = tid; e < an * rank; e += kThreads) {
      const int k = e % an, i = e / an;  // T[k][i] = conj(lead[i][k]) = V[k][order[i]]
      AT(X, k, i, an) = AT(V, k, order[i], size);
    }
    __syncthreads();
    double* s2 = s;  // s / order of the first SVD are no longer needed past rank
    __shared__ int order2[kMax];
    __shared__ int ord1[kMax];
    for (int i = tid; i < rank; i += kThreads) ord1[i] = order[i];
    __syncthreads();
    jacobi_svd(X, an, rank, Y, s2, order2);  // X = T V' (= U' S), Y = V'
    // pinv(lead) = pinv(T^H) = U' S^+ V'^H: P[k][j] = sum_l X[k][l] conj(Y[j][l]) / s_l^2
    const double smax2 = s2[order2[0]];
    const double cut = smax2 * 1e-15;
    // G[i][l] = sum_k lag[i][k] X[k][l] / s_l^2, lag[i][k] = conj(V[k+1][ord1[i]])
    z* G = U;
    for (int e = tid; e < rank * rank; e += kThreads) {
      const int i = e % rank, l = e / rank;
      z acc = zc(0.0);
      if (s2[l] > cut) {
        for (int k = 0; k < an; ++k)
          acc = zadd(acc, zmul(zconj(AT(V, k + 1, ord1[i], size)), AT(X, k, l, an)));
        acc = zscale(acc, 1.0 / (s2[l] * s2[l]));
      }
      AT(G, i, l, rank) = acc;
    }
    __syncthreads();
    // core[i][j] = sum_l G[i][l] conj(Y[j][l])
    z* core = A0;
    for (int e = tid; e < rank * rank; e += kThreads) {
      const int i = e % rank, j = e / rank;
      z acc = zc(0.0);
      for (int l = 0; l < rank; ++l)
        acc = zadd(acc, zmul(AT(G, i, l, rank), zconj(AT(Y, j, l, rank))));
      AT(core, i, j, rank) = acc;
    }
    __syncthreads();
    eigvals(core, rank, vec, vec + kMax);
    __syncthreads();
    for (int j = tid; j < rank; j += kThreads) {
      out_x[2 * j] = vec[j].re;
      out_x[2 * j + 1] = -vec[j].im;  // conj
    }
  }
}

#undef AT

}  // namespace cta_la

// Host launcher used by afft_small_la for shapes beyond the per-thread templates.
int small_la_cta(int op, int m, int n, const double* a, const double* b, int rank,
                 double* out_u, double* out_s, double* out_v, double* out_x, int* out_i,
                 cudaStream_t st) {
  const size_t bytes = (6 * cta_la::kMax * cta_la::kMax + 4 * cta_la::kMax) * sizeof(cta_la::z);
  void* scratch = nullptr;
  cudaError_t e = scratch_alloc(&scratch, bytes, st);
  if (e != cudaSuccess) return cuda_status(e, "small_la scratch");
  cta_la::small_la_cta_kernel<<<1, cta_la::kThreads, 0, st>>>(
      op, m, n, a, b, rank, out_u, out_s, out_v, out_x, out_i,
      static_cast<cta_la::z*>(scratch));
  e = cudaGetLastError();
  scratch_free(scratch, st);
  if (e != cudaSuccess) return cuda_status(e, "small_la_cta_kernel");
  return AFFT_OK;
}

}  // namespace afft
