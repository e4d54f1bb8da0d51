// sFFT-DT1/2/3 on the GPU (oneshot.py:86-289): collect → detect → solve → truncate.
//
//   collect  — the gather + size-b DFT kernel at the 3*a_m structured shifts
//              (-a_m .. 2a_m-1) and the p per-signal random shifts, in
//              measurement-row layout rows[s][bucket][3a_m + p]  (86-106);
//   detect   — per-bucket singular values of the a_m x a_m moment Hankel by
//              one-sided Jacobi, then the global vote: keys (-rint(sigma/1e-12),
//              bucket, slot), the first k win (116-140).  The vote is a rank
//              computation over all keys of a signal, exact integer order;
//   solve    — one thread per bucket with a > 0: locate (dt1 roots / dt2 grid
//              enumeration / dt3 pencil) and subspace pursuit (161-257), in
//              oneshot_core.cuh;
//   truncate — entries in bucket order, top-k by (-|v|, f) (260-263).
#include <algorithm>
#include <climits>
#include <cstring>

#include "afft_common.cuh"
#include "oneshot_core.cuh"

namespace afft {

constexpr int kDtSolveThreads = 128;

// ------------------------------------------------------------------ detect

// sigmas[e][0..a_m) for row e: Hankel H[r][c] = m_{start + r + c} (oneshot.py:109-113,128-130)
__global__ void dt_sigma_kernel(int64_t rows, int R, int a_m, const double* __restrict__ meas,
                                double* __restrict__ sigmas) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows) return;
  const la::c2* row = reinterpret_cast<const la::c2*>(meas) + e * R;
  la::MatT<dt::kMaxAm, dt::kMaxAm> H;
  H.m = H.n = a_m;
  for (int r = 0; r < a_m; ++r)
    for (int c = 0; c < a_m; ++c) H.at(r, c) = row[r + c + a_m];
  double s[dt::kMaxAm];
  la::singular_values(H, s);
  for (int i = 0; i < a_m; ++i) sigmas[e * a_m + i] = s[i];
}

// Vote: key i of signal s (i = bucket*a_m + slot) is chosen iff its rank under
// (-q, bucket, slot) is < k, with q = rint(sigma / 1e-12) (oneshot.py:131-139).
__global__ void dt_vote_kernel(int M, int a_m, int k, const double* __restrict__ sigmas,
                               int32_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  long long* q = reinterpret_cast<long long*>(smem_raw);
  const int64_t s = blockIdx.y;
  const double* sg = sigmas + s * (int64_t)M;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long qi = i < M ? (long long)rint(__ddiv_rn(sg[i], 1e-12)) : 0;
  int rank = 0;
  constexpr int kTile = 2048;
  for (int base = 0; base < M; base += kTile) {
    const int cnt = min(kTile, M - base);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x)
      q[t] = (long long)rint(__ddiv_rn(sg[base + t], 1e-12));
    __syncthreads();
    if (i < M) {
      for (int t = 0; t < cnt; ++t) {
        const long long qt = q[t];
        rank += (qt > qi) || (qt == qi && base + t < i);
      }
    }
  }
  if (i < M && rank < k) atomicAdd(&counts[s * (M / a_m) + i / a_m], 1);
}

// ------------------------------------------------------------------ solve

__global__ void __launch_bounds__(kDtSolveThreads, 4) dt_solve_kernel(
    int64_t batch, int64_t nrows, int R, int a_m, int p, const double* __restrict__ meas,
    const int64_t* __restrict__ rshifts, const int32_t* __restrict__ counts,
    const int64_t* __restrict__ bucket_ids, int variant, int a_cap, int64_t b, int64_t n,
    int64_t* __restrict__ out_pos, double* __restrict__ out_val, int32_t* __restrict__ out_cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= batch * nrows) return;
  const int64_t s = e / nrows;
  int a = counts[e];
  if (a_cap > 0 && a > a_cap) a = a_cap;  // dsfft.py:219 caps at a_m
  int cnt = 0;
  if (a > 0) {
    const int64_t bucket = bucket_ids ? bucket_ids[e] : e - s * nrows;
    const la::c2* row = reinterpret_cast<const la::c2*>(meas) + e * R;
    int64_t pos[dt::kMaxAm];
    la::c2 val[dt::kMaxAm];
    cnt = dt::solve_bucket(row, a_m, p, rshifts + s * p, a, variant, bucket, b, n, pos, val);
    for (int i = 0; i < cnt; ++i) {
      out_pos[e * a_m + i] = pos[i];
      reinterpret_cast<la::c2*>(out_val)[e * a_m + i] = val[i];
    }
  }
  out_cnt[e] = cnt;
}

// ------------------------------------------------------------------ truncate

// Compact the per-bucket entries of each signal (bucket order) and keep the k
// largest by (-|v|, f).  One CTA per signal.
__global__ void dt_truncate_kernel(int64_t nrows, int a_m, int k, const int64_t* __restrict__ pos,
                                   const double* __restrict__ val,
                                   const int32_t* __restrict__ cnt, int cap,
                                   int64_t* __restrict__ all_pos, double* __restrict__ all_val,
                                   int32_t* __restrict__ all_count, int64_t* __restrict__ out_pos,
                                   double* __restrict__ out_val, int32_t* __restrict__ out_count,
                                   double* gscratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* mag = gscratch ? gscratch + blockIdx.x * (int64_t)cap
                         : reinterpret_cast<double*>(smem_raw);
  __shared__ int total;
  const int64_t s = blockIdx.x;
  const int32_t* c = cnt + s * nrows;
  int64_t* ap = all_pos + s * (int64_t)cap;
  la::c2* av = reinterpret_cast<la::c2*>(all_val) + s * (int64_t)cap;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int64_t r = 0; r < nrows; ++r) {
      for (int i = 0; i < c[r]; ++i) {
        const int64_t src = (s * nrows + r) * a_m + i;
        ap[m] = pos[src];
        av[m] = reinterpret_cast<const la::c2*>(val)[src];
        ++m;
      }
    }
    total = m;
    all_count[s] = m;
  }
  __syncthreads();
  const int m = total;
  for (int i = threadIdx.x; i < m; i += blockDim.x) mag[i] = la::cabs(av[i]);
  __syncthreads();
  la::c2* ov = reinterpret_cast<la::c2*>(out_val) + s * k;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double a = mag[i];
    const int64_t f = ap[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) rank += (mag[j] > a) || (mag[j] == a && ap[j] < f);
    if (rank < k) {
      out_pos[s * k + rank] = f;
      ov[rank] = av[i];
    }
  }
  if (threadIdx.x == 0) out_count[s] = m < k ? m : k;
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct DtWs {
  size_t rows, sig, counts, pos, val, cnt, total;
};

static DtWs dt_ws(int64_t batch, int64_t b, int a_m, int p) {
  DtWs w;
  const int R = 3 * a_m + p;
  size_t o = 0;
  w.rows = o;   o = al256(o + (size_t)batch * b * R * 16);
  w.sig = o;    o = al256(o + (size_t)batch * b * a_m * 8);
  w.counts = o; o = al256(o + (size_t)batch * b * 4);
  w.pos = o;    o = al256(o + (size_t)batch * b * a_m * 8);
  w.val = o;    o = al256(o + (size_t)batch * b * a_m * 16);
  w.cnt = o;    o = al256(o + (size_t)batch * b * 4);
  w.total = o;
  return w;
}

static int check_dt(int64_t n, int64_t b, int a_m, int p, int variant) {
  if (b < 1 || n % b) {
    set_error("bucket count %lld does not divide %lld", (long long)b, (long long)n);
    return AFFT_EINVAL;
  }
  if (a_m < 1 || a_m > dt::kMaxAm) {
    set_error("a_m must be in 1..4");
    return AFFT_EINVAL;
  }
  if (p < 0 || p > dt::kMaxP) {
    set_error("p=%d random shifts unsupported (max %d)", p, dt::kMaxP);
    return AFFT_EUNSUPPORTED;
  }
  if (variant < dt::VAR_DT1 || variant > dt::VAR_DT3) {
    set_error("unknown variant %d", variant);
    return AFFT_EINVAL;
  }
  if (n > 3000000000LL) {
    set_error("signal size %lld too large", (long long)n);
    return AFFT_EUNSUPPORTED;
  }
  return AFFT_OK;
}

}  // namespace afft

using namespace afft;

extern "C" int afft_bucketize_table(const void* x, int dtype, int64_t n, int64_t batch,
                                    int64_t ld, int64_t b, const int64_t* shift_table,
                                    int32_t nshift, double* out, int64_t out_signal_stride,
                                    int64_t out_shift_stride, int64_t out_bin_stride,
                                    void* stream);

extern "C" int afft_dt_collect(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                               int64_t b, int32_t a_m, int32_t p, const int64_t* rand_shifts,
                               double* rows, void* stream) {
  if (batch == 0) return AFFT_OK;
  int rc = check_dt(n, b, a_m, p, dt::VAR_DT3);
  if (rc) return rc;
  const int R = 3 * a_m + p;
  int64_t structured[3 * dt::kMaxAm];
  for (int t = 0; t < 3 * a_m; ++t) structured[t] = t - a_m;
  rc = afft_bucketize(x, dtype, n, batch, ld, b, structured, 3 * a_m, rows, b * R, 1, R, stream);
  if (rc || p == 0) return rc;
  return afft_bucketize_table(x, dtype, n, batch, ld, b, rand_shifts, p,
                              rows + 2 * (3 * a_m), b * R, 1, R, stream);
}

extern "C" int afft_dt_detect(const double* rows, int64_t batch, int64_t nrows, int32_t R,
                              int32_t a_m, int32_t k, int32_t* counts, double* sigmas,
                              void* stream) {
  if (batch == 0 || nrows == 0) return AFFT_OK;
  if (!rows || !counts || !sigmas || a_m < 1 || a_m > dt::kMaxAm || R < 3 * a_m || k < 0) {
    set_error("afft_dt_detect: bad arguments");
    return AFFT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = batch * nrows;
  dt_sigma_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(total, R, a_m, rows, sigmas);
  AFFT_CHECK_LAUNCH("dt_sigma_kernel");
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)total * 4, st);
  if (e != cudaSuccess) return cuda_status(e, "memset counts");
  if (k == 0) return AFFT_OK;
  const int64_t M = nrows * a_m;
  if (M > INT32_MAX / 2) {
    set_error("afft_dt_detect: too many keys");
    return AFFT_EUNSUPPORTED;
  }
  dim3 grid((unsigned)((M + 255) / 256), (unsigned)batch);
  dt_vote_kernel<<<grid, 256, 2048 * 8, st>>>((int)M, a_m, k, sigmas, counts);
  AFFT_CHECK_LAUNCH("dt_vote_kernel");
  return AFFT_OK;
}

extern "C" int afft_dt_solve(const double* rows, const int64_t* rand_shifts, int64_t batch,
                             int64_t nrows, int32_t a_m, int32_t p, const int32_t* counts,
                             const int64_t* bucket_ids, int32_t variant, int32_t a_cap,
                             int64_t b, int64_t n, int64_t* out_pos, double* out_val,
                             int32_t* out_cnt, void* stream) {
  if (batch == 0 || nrows == 0) return AFFT_OK;
  int rc = check_dt(n, b, a_m, p, variant);
  if (rc) return rc;
  if (!rows || !counts || !out_pos || !out_val || !out_cnt || (p > 0 && !rand_shifts)) {
    set_error("afft_dt_solve: bad arguments");
    return AFFT_EINVAL;
  }
  const int64_t total = batch * nrows;
  dt_solve_kernel<<<(unsigned)((total + kDtSolveThreads - 1) / kDtSolveThreads), kDtSolveThreads,
                    0, (cudaStream_t)stream>>>(batch, nrows, 3 * a_m + p, a_m, p, rows,
                                               rand_shifts, counts, bucket_ids, variant, a_cap, b,
                                               n, out_pos, out_val, out_cnt);
  AFFT_CHECK_LAUNCH("dt_solve_kernel");
  return AFFT_OK;
}

extern "C" int afft_dt_truncate(const int64_t* pos, const double* val, const int32_t* cnt,
                                int64_t batch, int64_t nrows, int32_t a_m, int32_t k,
                                int64_t* all_pos, double* all_val, int32_t* all_count,
                                int64_t* out_pos, double* out_val, int32_t* out_count,
                                void* stream) {
  if (batch == 0) return AFFT_OK;
  const int64_t cap = nrows * a_m;
  if (!pos || !val || !cnt || !all_pos || !all_val || !all_count || !out_count ||
      (k > 0 && (!out_pos || !out_val))) {
    set_error("afft_dt_truncate: bad arguments");
    return AFFT_EINVAL;
  }
  size_t smem = (size_t)std::max<int64_t>(cap, 1) * 8;
  double* scratch = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 200 * 1024) {  // many buckets: magnitudes in global memory
    cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&scratch),
                                    (size_t)batch * cap * 8, st);
    if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(dt_truncate scratch)");
    smem = 0;
  } else {
    cudaError_t e = cudaFuncSetAttribute(dt_truncate_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(dt_truncate)");
  }
  dt_truncate_kernel<<<(unsigned)batch, 1024, smem, st>>>(
      nrows, a_m, k, pos, val, cnt, (int)cap, all_pos, all_val, all_count, out_pos, out_val,
      out_count, scratch);
  if (scratch) scratch_free(scratch, st);
  AFFT_CHECK_LAUNCH("dt_truncate_kernel");
  return AFFT_OK;
}

extern "C" size_t afft_sfft_dt_workspace_size(int64_t n, int64_t batch, int64_t b, int32_t a_m,
                                              int32_t p) {
  if (check_dt(n, b, a_m, p, dt::VAR_DT3)) return 0;
  return dt_ws(batch, b, a_m, p).total;
}

extern "C" int afft_sfft_dt(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                            int64_t b, int32_t a_m, int32_t p, int32_t variant, int32_t k,
                            const int64_t* rand_shifts, int64_t* out_pos, double* out_val,
                            int32_t* out_count, int64_t* all_pos, double* all_val,
                            int32_t* all_count, int32_t* counts_out, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (batch == 0) return AFFT_OK;
  int rc = check_dt(n, b, a_m, p, variant);
  if (rc) return rc;
  const DtWs w = dt_ws(batch, b, a_m, p);
  if (!workspace || workspace_bytes < w.total) {
    set_error("afft_sfft_dt: workspace of %zu bytes needed, %zu given", w.total, workspace_bytes);
    return AFFT_ENOMEM;
  }
  char* ws = reinterpret_cast<char*>(workspace);
  double* rows = reinterpret_cast<double*>(ws + w.rows);
  int32_t* counts = counts_out ? counts_out : reinterpret_cast<int32_t*>(ws + w.counts);
  if ((rc = afft_dt_collect(x, dtype, n, batch, ld, b, a_m, p, rand_shifts, rows, stream)))
    return rc;
  if ((rc = afft_dt_detect(rows, batch, b, 3 * a_m + p, a_m, k, counts,
                           reinterpret_cast<double*>(ws + w.sig), stream)))
    return rc;
  int64_t* pos = reinterpret_cast<int64_t*>(ws + w.pos);
  double* val = reinterpret_cast<double*>(ws + w.val);
  int32_t* cnt = reinterpret_cast<int32_t*>(ws + w.cnt);
  if ((rc = afft_dt_solve(rows, rand_shifts, batch, b, a_m, p, counts, nullptr, variant, 0, b, n,
                          pos, val, cnt, stream)))
    return rc;
  return afft_dt_truncate(pos, val, cnt, batch, b, a_m, k, all_pos, all_val, all_count, out_pos,
                          out_val, out_count, stream);
}

namespace afft {
// locate (oneshot.py:161-200) for `count` independent rows: out_n[i] = number of
// candidates written to out_pos[i][0..4), or -1 for None.
__global__ void dt_locate_kernel(int64_t count, int R, int a_m, const double* __restrict__ rows,
                                 const int32_t* __restrict__ a, const int64_t* __restrict__ bucket,
                                 int variant, int64_t b, int64_t n, int64_t* __restrict__ out_pos,
                                 int32_t* __restrict__ out_n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  dt::Moments M{reinterpret_cast<const la::c2*>(rows) + i * R, a_m};
  int64_t pos[5];
  const int c = dt::locate(M, a[i], variant, bucket[i], b, n, pos);
  for (int k = 0; k < c && k < dt::kMaxAm; ++k) out_pos[i * dt::kMaxAm + k] = pos[k];
  out_n[i] = c;
}

// estimate_values (oneshot.py:203-257) for `count` rows given their candidates.
__global__ void dt_estimate_kernel(int64_t count, int R, int a_m, int p,
                                   const double* __restrict__ rows,
                                   const int64_t* __restrict__ rshifts,
                                   const int64_t* __restrict__ cands,
                                   const int32_t* __restrict__ ncand, int64_t b, int64_t n,
                                   int64_t* __restrict__ out_pos, double* __restrict__ out_val,
                                   int32_t* __restrict__ out_n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  int64_t c[dt::kMaxAm];
  int nc = 0;
  for (int k = 0; k < ncand[i] && k < dt::kMaxAm; ++k) c[nc++] = cands[i * dt::kMaxAm + k];
  nc = dt::sort_unique(c, nc);
  int64_t pos[dt::kMaxAm];
  la::c2 val[dt::kMaxAm];
  const la::c2* row = reinterpret_cast<const la::c2*>(rows) + i * R;
  const int m = dt::estimate_values(row + 3 * a_m, rshifts, p, c, nc, b, n, pos, val);
  for (int k = 0; k < m; ++k) {
    out_pos[i * dt::kMaxAm + k] = pos[k];
    reinterpret_cast<la::c2*>(out_val)[i * dt::kMaxAm + k] = val[k];
  }
  out_n[i] = m;
}
}  // namespace afft

extern "C" int afft_dt_locate(const double* rows, int64_t count, int32_t R, int32_t a_m,
                              const int32_t* a, const int64_t* bucket, int32_t variant, int64_t b,
                              int64_t n, int64_t* out_pos, int32_t* out_n, void* stream) {
  if (count == 0) return AFFT_OK;
  int rc = check_dt(n, b, a_m, R - 3 * a_m, variant);
  if (rc) return rc;
  if (!rows || !a || !bucket || !out_pos || !out_n) {
    set_error("afft_dt_locate: bad arguments");
    return AFFT_EINVAL;
  }
  dt_locate_kernel<<<(unsigned)((count + 63) / 64), 64, 0, (cudaStream_t)stream>>>(
      count, R, a_m, rows, a, bucket, variant, b, n, out_pos, out_n);
  AFFT_CHECK_LAUNCH("dt_locate_kernel");
  return AFFT_OK;
}

extern "C" int afft_dt_estimate(const double* rows, const int64_t* rand_shifts, int64_t count,
                                int32_t a_m, int32_t p, const int64_t* cands,
                                const int32_t* ncand, int64_t b, int64_t n, int64_t* out_pos,
                                double* out_val, int32_t* out_n, void* stream) {
  if (count == 0) return AFFT_OK;
  int rc = check_dt(n, b, a_m, p, dt::VAR_DT3);
  if (rc) return rc;
  if (!rows || !cands || !ncand || !out_pos || !out_val || !out_n || (p > 0 && !rand_shifts)) {
    set_error("afft_dt_estimate: bad arguments");
    return AFFT_EINVAL;
  }
  dt_estimate_kernel<<<(unsigned)((count + 63) / 64), 64, 0, (cudaStream_t)stream>>>(
      count, 3 * a_m + p, a_m, p, rows, rand_shifts, cands, ncand, b, n, out_pos, out_val, out_n);
  AFFT_CHECK_LAUNCH("dt_estimate_kernel");
  return AFFT_OK;
}
