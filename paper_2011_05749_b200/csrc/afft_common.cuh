// Shared device helpers: numpy-faithful complex128 arithmetic, error plumbing.
//
// Every floating-point helper here mirrors the operation numpy performs on the
// reference path, in the same order, and the library is compiled with
// --fmad=false so no multiply-add is contracted.  That keeps decision values
// (threshold comparisons, rounding of decoded bins) within an ulp or two of the
// reference instead of drifting with the compiler's choice of FMAs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/aliasfft_b200.h"

namespace afft {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
// stream-ordered scratch from the library's memory pool (kept across calls)
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t stream);
// Per-thread arena for scratch_alloc on `stream` between arena_begin and arena_end
// (capi.cu); the caller must synchronise the stream before arena_end.
cudaError_t arena_begin(size_t bytes, cudaStream_t stream);
void arena_end();
// Pinned host staging from a process-wide pool: buffers are never freed (cudaFreeHost
// synchronises the whole device, which a thread-local buffer's destructor did at every
// worker-thread exit), and are reused across threads.  pinned_release returns one.
void* pinned_acquire(size_t bytes, size_t* capacity);
// dsfft.cu: a full layer's active set straight from the resident spectrum (n/b <= 32).
int alias_active(const double* spectrum, int64_t n, int64_t b, double thr, int64_t* out, int cap,
                 int32_t* count, cudaStream_t st);
void pinned_release(void* p, size_t capacity);
// dsfft.cu: the active lists of every full deep layer (n/b <= 32) in one spectrum pass.
int deep_active_all(const double* spectrum, int64_t n, int64_t bmin, int nl, const double* thr,
                    int64_t* out, int cap, int32_t* counts, void* scratch, size_t scratch_bytes,
                    cudaStream_t st);
size_t deep_active_scratch(int64_t n, int64_t bmin, int nl);
// dsfft.cu: every full layer from depth d0 to d0 + nl - 1 (n a power of two, 2^d0 >= 32):
// deep ones from the spectrum, shallower ones by summing children; one pass + one count.
int full_active_all(const double* spectrum, int64_t n, int d0, int nl, const double* thr,
                    int64_t* out, int cap, int32_t* counts, void* scratch, size_t scratch_bytes,
                    cudaStream_t st);
size_t full_active_scratch(int64_t n, int d0, int nl);
// rffast.cu: classify_noisy over rows of several signals (row_sig, per-signal shift
// tables and gates on the device); workspace afft_singleton_workspace_size(n, count, b, c, m).
int classify_noisy_multi(const double* residual, const int64_t* index, const int32_t* row_sig,
                         int64_t count, int64_t b, int64_t n, const int64_t* tau_tab, int32_t c,
                         int32_t m, const double* weights, const double* t0s, const double* t1s,
                         int8_t* state, int64_t* f0, double* val, double* resnorm,
                         void* workspace, size_t workspace_bytes, cudaStream_t st);
// dsfft.cu: rows for (signal, bucket) pairs from per-signal coset DFTs Y [S][U][b]
// (coset [S][nshift] which DFT serves shift t, q [S][nshift] its rotation).
int rows_gather_multi(const double* Y, int64_t b, int U, int nshift, const int32_t* coset,
                      const int64_t* q, const int64_t* idx, const int32_t* sig, int64_t nrows,
                      double* rows, cudaStream_t st);
// The one-CTA-per-row alias rows keep 2.5 L values in shared memory: L <= 4096.
constexpr int64_t kAliasCtaMaxL = 4096;
// dsfft.cu: alias_rows_multi for 256 < n/b <= kAliasCtaMaxL (one CTA per row)
int alias_rows_cta_multi(const double* Y, int64_t n, int64_t b, const int64_t* tau_tab,
                         int nshift, const int64_t* idx, const int32_t* sig, int64_t nrows,
                         double* rows, cudaStream_t st);
// dsfft.cu: rows for (signal, bucket) pairs from per-signal resident spectra
// (Y + sig * n), per-signal reduced shifts tau_tab [S][nshift]; n/b <= 256.
int alias_rows_multi(const double* Y, int64_t n, int64_t b, const int64_t* tau_tab, int nshift,
                     const int64_t* idx, const int32_t* sig, int64_t nrows, double* rows,
                     cudaStream_t st);
// bucketize.cu: build_graph with per-signal raw shifts (device [batch][nshift]).
int build_graph_table(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                      const int64_t* factors, int32_t ncycles, const int64_t* shift_table,
                      int32_t nshift, double* nodes, cudaStream_t stream);
cudaError_t scratch_free(void* p, cudaStream_t stream);
// Raise a kernel's dynamic shared-memory limit to at least `bytes` (never lowers it:
// the attribute is process-wide, so concurrent callers on other streams/threads that
// need more must not be undercut).  Thread-safe.
cudaError_t ensure_smem(const void* func, size_t bytes);

#define AFFT_CHECK_LAUNCH(what)                                   \
  do {                                                            \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return ::afft::cuda_status(_e, what);  \
  } while (0)

// ---------------------------------------------------------------- complex128
struct cd {
  double re, im;
};

__device__ __forceinline__ cd mk(double r, double i) { return cd{r, i}; }
__device__ __forceinline__ cd cadd(cd a, cd b) { return cd{a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return cd{a.re - b.re, a.im - b.im}; }
// numpy complex multiply: (ac - bd) + (ad + bc)i, no FMA.
__device__ __forceinline__ cd cmul(cd a, cd b) {
  return cd{__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
            __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
__device__ __forceinline__ cd cscale(cd a, double s) {
  return cd{__dmul_rn(a.re, s), __dmul_rn(a.im, s)};
}
// numpy complex divide (Smith's algorithm, numpy/_core/src/umath/loops.c.src
// CDOUBLE_divide): the form numpy uses for every complex128 '/'.
__device__ __forceinline__ cd cdiv(cd a, cd b) {
  double br = fabs(b.re), bi = fabs(b.im);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return cd{a.re / br, a.im / br};
    double rat = b.im / b.re;
    double scl = 1.0 / __dadd_rn(b.re, __dmul_rn(b.im, rat));
    return cd{__dmul_rn(__dadd_rn(a.re, __dmul_rn(a.im, rat)), scl),
              __dmul_rn(__dsub_rn(a.im, __dmul_rn(a.re, rat)), scl)};
  } else {
    double rat = b.re / b.im;
    double scl = 1.0 / __dadd_rn(b.im, __dmul_rn(b.re, rat));
    return cd{__dmul_rn(__dadd_rn(__dmul_rn(a.re, rat), a.im), scl),
              __dmul_rn(__dsub_rn(__dmul_rn(a.im, rat), a.re), scl)};
  }
}
__device__ __forceinline__ double cabs_(cd a) { return hypot(a.re, a.im); }

// exp(-2j*pi*prod/n) exactly as numpy evaluates it on the reference path
// (peeling.py:182-183, oneshot.py:146-147): theta = (-2*pi*prod) * (1/n)
// (complex/int division is multiplication by the reciprocal in numpy), then
// (cos theta, sin theta).  prod must already be reduced into [0, n).
__device__ __forceinline__ cd unit_root(int64_t prod, int64_t n) {
  double theta = __dmul_rn(__dmul_rn(-6.283185307179586, (double)prod), 1.0 / (double)n);
  double s, c;
  sincos(theta, &s, &c);
  return cd{c, s};
}

// (a*b) mod n for 0 <= a,b < n < 2^31.5 (no overflow in int64).  (A double-quotient
// form with fix-ups measured slower on B200 than the compiler's 64-bit remainder.)
__device__ __forceinline__ int64_t mulmod(int64_t a, int64_t b, int64_t n) {
  return (a * b) % n;
}
__device__ __forceinline__ int64_t pymod(int64_t a, int64_t n) {
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}

// Load one sample as complex128 from a c64 or c128 signal.
__device__ __forceinline__ cd load_sample(const void* x, int dtype, int64_t off) {
  if (dtype == AFFT_C64) {
    float2 v = __ldg(reinterpret_cast<const float2*>(x) + off);
    return cd{(double)v.x, (double)v.y};
  }
  double2 v = __ldg(reinterpret_cast<const double2*>(x) + off);
  return cd{v.x, v.y};
}

inline int64_t host_pymod(int64_t a, int64_t n) {
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}

// The tree layers a K2' final radix-256 pass can decide in its epilogue (bucketize.cu
// gfft_flags_kernel): the last pass of the n-point spectrum holds, per tile, the alias
// classes Y[j + q n/256] (q < 256) of 8 consecutive j, and one thread holds q = qb + 16 qa
// (qa < 16), i.e. every alias of the buckets of depths dtop + 4 .. dtop + 8 over its j
// (dtop = log2(n) - 8; values in the tree order of dsfft.cu tree_sum).  Depth dtop + t's
// bitmap at words + word_off[t] (bytes written whole: a tile owns 8 consecutive bits),
// flagged for t_lo <= t (t >= 4); the depth-(dtop + 4) values to vmid (16 n/256 entries)
// when non-null, for the shallower layers' tree; sum |Y|^2 added into *norm2 when non-null.
struct DeepFuse {
  uint32_t* words;
  int64_t word_off[9];
  double thr[9];
  double t2hi[9], t2lo[9];  // thr^2 (1 +- 1e-14): the |v|^2 guard band
  int t_lo;
  cd* vmid;
  double* norm2;
};
// bucketize.cu: Y = fft(x)/n (x one signal, n a power of two planned as three radix-256
// passes or any plan whose last pass is radix 256) with the DeepFuse epilogue on the last
// pass; AFFT_EUNSUPPORTED (nothing launched) for other plans.
int spectrum_fused(const void* x, int dtype, int64_t n, double* Y, const DeepFuse& f,
                   cudaStream_t st);
// dsfft.cu: full_active_all with the spectrum computed here and the layers at depths
// >= log2(n) - 8 decided in its last pass (one read of Y less); *norm2 (device) = sum |Y|^2.
int full_active_all_fused(const void* x, int dtype, int64_t n, double* Y, int d0, int nl,
                          const double* thr, int64_t* out, int cap, int32_t* counts,
                          double* norm2, void* scratch, size_t scratch_bytes, cudaStream_t st);
size_t full_active_fused_scratch(int64_t n, int d0, int nl);

}  // namespace afft
