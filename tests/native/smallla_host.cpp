// Host build of csrc/smallla.cuh for CPU unit tests against numpy (test infrastructure).
#include "../../paper_2011_05749_b200/csrc/smallla.cuh"

using namespace afft::la;

static void load(Mat& A, int m, int n, const double* a) {  // a: row-major interleaved
  A.m = m;
  A.n = n;
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c) A.at(r, c) = C(a[2 * (r * n + c)], a[2 * (r * n + c) + 1]);
}

extern "C" {
void t_singular_values(int m, int n, const double* a, double* s) {
  Mat A;
  load(A, m, n, a);
  singular_values(A, s);
}
int t_lstsq(int m, int n, const double* a, const double* y, double* x, double* s) {
  Mat A;
  load(A, m, n, a);
  return lstsq(A, reinterpret_cast<const c2*>(y), reinterpret_cast<c2*>(x), s);
}
void t_pinv(int m, int n, const double* a, double rcond, double* p) {
  Mat A, P;
  load(A, m, n, a);
  pinv(A, P, rcond);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < m; ++c) {
      p[2 * (r * m + c)] = P.at(r, c).re;
      p[2 * (r * m + c) + 1] = P.at(r, c).im;
    }
}
int t_eigvals(int n, const double* a, double* lam) {
  Mat A;
  load(A, n, n, a);
  return eigvals(A, reinterpret_cast<c2*>(lam)) ? 1 : 0;
}
int t_poly_roots(int a, const double* c, double* roots) {
  return poly_roots(reinterpret_cast<const c2*>(c), a, reinterpret_cast<c2*>(roots));
}
}

#include "../../paper_2011_05749_b200/csrc/oneshot_core.cuh"

extern "C" {
// sfft_dt per-bucket solve (locate + pursuit) on a host row
int t_solve_bucket(const double* row, int a_m, int p, const int64_t* rshifts, int a, int variant,
                   int64_t bucket, int64_t b, int64_t n, int64_t* out_pos, double* out_val) {
  return afft::dt::solve_bucket(reinterpret_cast<const c2*>(row), a_m, p, rshifts, a, variant,
                                bucket, b, n, out_pos, reinterpret_cast<c2*>(out_val));
}
int t_locate(const double* row, int a_m, int a, int variant, int64_t bucket, int64_t b, int64_t n,
             int64_t* pos) {
  afft::dt::Moments M{reinterpret_cast<const c2*>(row), a_m};
  return afft::dt::locate(M, a, variant, bucket, b, n, pos);
}
}
