// smallnum API (smallnum.py:54-142) on the device: one matrix per call, one
// thread, built from the same smallla.cuh templates the per-bucket solvers use.
// Shapes up to the hot path's sizes (tall side <= 32, short side <= 8) run one
// thread; larger ones, up to the reference's 64 x 64 cap, go to the CTA-cooperative
// solvers of smallnum_cta.cu.
#include <cstring>

#include "afft_common.cuh"
#include "smallla.cuh"

namespace afft {

using la::c2;
using la::MatT;
constexpr int kR = la::kLaMaxRows;  // 32
constexpr int kC = la::kLaMaxCols;  // 8

enum SmallOp { OP_SVD = 0, OP_LSTSQ = 1, OP_EIGVALS = 2, OP_ROOTS = 3, OP_PENCIL = 4 };

template <int MR, int MC>
__device__ void load_rowmajor(MatT<MR, MC>& M, const double* a, int m, int n, bool conj_t) {
  if (!conj_t) {
    M.m = m;
    M.n = n;
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < n; ++c) M.at(r, c) = c2{a[2 * (r * n + c)], a[2 * (r * n + c) + 1]};
  } else {  // M = A^H
    M.m = n;
    M.n = m;
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < n; ++c) M.at(c, r) = c2{a[2 * (r * n + c)], -a[2 * (r * n + c) + 1]};
  }
}

// Full left basis: U[:, k] = W[:, k] / s_k for s_k > 0, completed by Gram-Schmidt.
__device__ void complete_basis(const MatT<kR, kC>& W, const double* s, int m, int n,
                               MatT<kR, kR>& U) {
  U.m = U.n = m;
  int have = 0;
  for (int k = 0; k < n; ++k) {
    if (s[k] > 0.0) {
      for (int i = 0; i < m; ++i) U.at(i, have) = la::scale(W.at(i, k), 1.0 / s[k]);
      ++have;
    }
  }
  for (int e = 0; e < m && have < m; ++e) {
    c2 v[kR];
    for (int i = 0; i < m; ++i) v[i] = la::C(i == e ? 1.0 : 0.0);
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = 0; k < have; ++k) {
        c2 d = la::C(0.0);
        for (int i = 0; i < m; ++i) d = la::add(d, la::cmulc(U.at(i, k), v[i]));
        for (int i = 0; i < m; ++i) v[i] = la::sub(v[i], la::mul(U.at(i, k), d));
      }
    }
    double nv = 0.0;
    for (int i = 0; i < m; ++i) nv += la::abs2(v[i]);
    nv = sqrt(nv);
    if (nv < 1e-8) continue;
    for (int i = 0; i < m; ++i) U.at(i, have) = la::scale(v[i], 1.0 / nv);
    ++have;
  }
}

__global__ void small_api_kernel(int op, int m, int n, const double* __restrict__ a,
                                 const double* __restrict__ b, int rank_req, double* out_u,
                                 double* out_s, double* out_v, double* out_x, int* out_i) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (op == OP_SVD) {
    const bool wide = m < n;
    const int M = wide ? n : m, N = wide ? m : n;
    MatT<kR, kC> W;
    load_rowmajor(W, a, m, n, wide);
    MatT<kC, kC> V;
    double s[kC];
    la::svd_jacobi(W, s, V);
    MatT<kR, kR> U;
    complete_basis(W, s, M, N, U);
    // A = U S V^H (tall) or A = V S U^H (wide): write u (m x m), v (n x n) row-major
    for (int k = 0; k < N; ++k) out_s[k] = s[k];
    if (!wide) {
      for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) {
          out_u[2 * (r * m + c)] = U.at(r, c).re;
          out_u[2 * (r * m + c) + 1] = U.at(r, c).im;
        }
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
          out_v[2 * (r * n + c)] = V.at(r, c).re;
          out_v[2 * (r * n + c) + 1] = V.at(r, c).im;
        }
    } else {
      for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) {
          out_u[2 * (r * m + c)] = V.at(r, c).re;
          out_u[2 * (r * m + c) + 1] = V.at(r, c).im;
        }
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
          out_v[2 * (r * n + c)] = U.at(r, c).re;
          out_v[2 * (r * n + c) + 1] = U.at(r, c).im;
        }
    }
    return;
  }
  if (op == OP_LSTSQ) {  // m >= n; x, singular values, rank
    MatT<kR, kC> A;
    load_rowmajor(A, a, m, n, false);
    c2 y[kR], x[kC];
    for (int i = 0; i < m; ++i) y[i] = c2{b[2 * i], b[2 * i + 1]};
    double s[kC];
    out_i[0] = la::lstsq(A, y, x, s);
    for (int j = 0; j < n; ++j) {
      out_x[2 * j] = x[j].re;
      out_x[2 * j + 1] = x[j].im;
      out_s[j] = s[j];
    }
    double rs = 0.0;  // ||A x - y|| (smallnum.py:65)
    for (int i = 0; i < m; ++i) {
      c2 acc = la::C(0.0);
      for (int j = 0; j < n; ++j) acc = la::add(acc, la::mul(A.at(i, j), x[j]));
      rs += la::abs2(la::sub(acc, y[i]));
    }
    out_s[n] = sqrt(rs);
    return;
  }
  if (op == OP_EIGVALS) {
    MatT<kC, kC> A;
    load_rowmajor(A, a, m, n, false);
    c2 lam[kC];
    out_i[0] = la::eigvals(A, lam) ? 1 : 0;
    for (int j = 0; j < n; ++j) {
      out_x[2 * j] = lam[j].re;
      out_x[2 * j + 1] = lam[j].im;
    }
    return;
  }
  if (op == OP_ROOTS) {  // a = the n non-leading coefficients, lowest first
    c2 cf[4], roots[4];
    for (int j = 0; j < n; ++j) cf[j] = c2{a[2 * j], a[2 * j + 1]};
    const int cnt = la::poly_roots(cf, n, roots);
    out_i[0] = cnt;
    for (int j = 0; j < cnt; ++j) {
      out_x[2 * j] = roots[j].re;
      out_x[2 * j + 1] = roots[j].im;
    }
    return;
  }
  if (op == OP_PENCIL) {  // a = full (m x m) pencil [y1 | y2[:, -1]], m = a_ + 1
    const int size = m, an = m - 1;
    MatT<kC, kC> full;
    load_rowmajor(full, a, size, size, false);
    MatT<kC, kC> W = full, V;
    double sv[kC];
    la::svd_jacobi(W, sv, V);
    const double tol = sv[0] * 1e-10;
    int nrank = 0;
    for (int i = 0; i < size; ++i) nrank += sv[i] > tol;
    out_i[1] = rank_req <= nrank ? 1 : 0;  // ok
    const int rank = rank_req < nrank ? rank_req : nrank;
    out_i[0] = rank;
    if (rank == 0) return;
    MatT<kC, kC> lead, lag, P, core;
    lead.m = lag.m = rank;
    lead.n = lag.n = an;
    for (int i = 0; i < rank; ++i)
      for (int j = 0; j < an; ++j) {
        lead.at(i, j) = la::conj(V.at(j, i));
        lag.at(i, j) = la::conj(V.at(j + 1, i));
      }
    la::pinv(lead, P, 1e-15);
    core.m = core.n = rank;
    for (int i = 0; i < rank; ++i)
      for (int j = 0; j < rank; ++j) {
        c2 s = la::C(0.0);
        for (int k = 0; k < an; ++k) s = la::add(s, la::mul(lag.at(i, k), P.at(k, j)));
        core.at(i, j) = s;
      }
    c2 lam[kC];
    la::eigvals(core, lam);
    for (int j = 0; j < rank; ++j) {
      out_x[2 * j] = lam[j].re;
      out_x[2 * j + 1] = -lam[j].im;  // conj
    }
  }
}

}  // namespace afft

namespace afft {
// smallnum_cta.cu: one CTA per call for shapes beyond the per-thread templates (<= 64)
int small_la_cta(int op, int m, int n, const double* a, const double* b, int rank,
                 double* out_u, double* out_s, double* out_v, double* out_x, int* out_i,
                 cudaStream_t st);
}  // namespace afft

using namespace afft;

extern "C" int afft_small_la(int32_t op, int32_t m, int32_t n, const double* a, const double* b,
                             int32_t rank, double* out_u, double* out_s, double* out_v,
                             double* out_x, int32_t* out_i, void* stream) {
  if (m < 1 || n < 1 || !a) {
    set_error("afft_small_la: empty matrix");
    return AFFT_EINVAL;
  }
  const int lo = m < n ? m : n, hi = m < n ? n : m;
  bool ok = true;
  switch (op) {
    case OP_SVD: ok = lo <= kC && hi <= kR && out_u && out_s && out_v; break;
    case OP_LSTSQ: ok = m >= n && n <= kC && m <= kR && b && out_x && out_s && out_i; break;
    case OP_EIGVALS: ok = m == n && n <= kC && out_x && out_i; break;
    case OP_ROOTS: ok = m == 1 && n >= 1 && n <= 4 && out_x && out_i; break;
    case OP_PENCIL: ok = m == n && m <= kC && rank >= 1 && rank < m && out_x && out_i; break;
    default: ok = false;
  }
  if (!ok && op != OP_ROOTS && hi <= 64 && (op != OP_LSTSQ || (m >= n && b && out_x && out_s && out_i)) &&
      (op != OP_EIGVALS || (m == n && out_x && out_i)) &&
      (op != OP_PENCIL || (m == n && rank >= 1 && rank < m && out_x && out_i)) &&
      (op != OP_SVD || (out_u && out_s && out_v)))
    return small_la_cta(op, m, n, a, b, rank, out_u, out_s, out_v, out_x, out_i,
                        (cudaStream_t)stream);
  if (!ok) {
    set_error("afft_small_la: op %d unsupported for a %d x %d matrix (device caps %d x %d)", op,
              m, n, kR, kC);
    return AFFT_EUNSUPPORTED;
  }
  small_api_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(op, m, n, a, b, rank, out_u, out_s, out_v,
                                                        out_x, out_i);
  AFFT_CHECK_LAUNCH("small_api_kernel");
  return AFFT_OK;
}
