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
#include <cstdlib>
#include <cstring>

#include <cub/block/block_radix_sort.cuh>

#include "afft_common.cuh"
#include "dt_warp.cuh"
#include "oneshot_core.cuh"
#include "peel_core.cuh"

namespace afft {

constexpr int kDtSolveThreads = 64;

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

// Vote (oneshot.py:131-139): keys i = bucket*a_m + slot with q_i = rint(sigma_i/1e-12);
// the first k keys under (-q, i) are chosen.  One CTA per signal: a radix select
// finds the k-th largest q (q*) and the count above it; among keys equal to q* the
// lowest indices fill the remaining places (a block scan over the equality flags).
constexpr int kVoteThreads = 1024;

__global__ void __launch_bounds__(kVoteThreads) dt_vote_kernel(int M, int a_m, int k,
                                                               const double* __restrict__ sigmas,
                                                               int32_t* __restrict__ counts,
                                                               long long* __restrict__ qbuf) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long prefix;
  __shared__ int remaining;
  __shared__ int warp_sum[32];
  __shared__ int carry;
  const int64_t s = blockIdx.x;
  const double* sg = sigmas + s * (int64_t)M;
  long long* q = qbuf + s * (int64_t)M;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int kk = k < M ? k : M;
  for (int i = tid; i < M; i += nt) q[i] = (long long)rint(__ddiv_rn(sg[i], 1e-12));
  if (tid == 0) {
    prefix = 0ull;
    remaining = kk - 1;  // 0-based rank of the k-th largest
  }
  __syncthreads();
  // radix select of the kk-th largest q (keys are >= 0: unsigned order = value order)
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nt) hist[i] = 0u;
    __syncthreads();
    const unsigned long long pre = prefix;
    const unsigned long long mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (int i = tid; i < M; i += nt) {
      const unsigned long long v = (unsigned long long)q[i];
      if ((v & mask) == pre) atomicAdd(&hist[255u - ((v >> shift) & 255u)], 1u);  // descending
    }
    __syncthreads();
    if (tid == 0) {
      int r = remaining;
      unsigned d = 0;
      while (d < 255 && r >= (int)hist[d]) {
        r -= (int)hist[d];
        ++d;
      }
      remaining = r;
      prefix = pre | ((unsigned long long)(255u - d) << shift);
    }
    __syncthreads();
  }
  const long long qs = (long long)prefix;
  const int need_eq = remaining + 1;  // keys equal to q* that are chosen (lowest indices)
  // scan of equality flags in index order; per-thread contiguous chunks
  const int per = (M + nt - 1) / nt;
  const int lo = min(M, tid * per), hi = min(M, lo + per);
  int local = 0;
  for (int i = lo; i < hi; ++i) local += q[i] == qs;
  const int lane = tid & 31, w = tid >> 5;
  int x = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    int v = lane < (nt >> 5) ? warp_sum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    warp_sum[lane] = v;
  }
  __syncthreads();
  int run = (w ? warp_sum[w - 1] : 0) + x - local;  // equal keys before this chunk
  (void)carry;
  int32_t* cnt = counts + s * (int64_t)(M / a_m);
  for (int i = lo; i < hi; ++i) {
    bool chosen = false;
    if (q[i] > qs) {
      chosen = true;
    } else if (q[i] == qs) {
      chosen = run < need_eq;
      ++run;
    }
    if (chosen && kk > 0) atomicAdd(&cnt[i / a_m], 1);
  }
}

// ------------------------------------------------------------------ solve

// Out of line so its small-matrix frame does not crowd the enumeration loop's registers.
__device__ __noinline__ int moment_coeffs_call(const la::c2* row, int a_m, int a, la::c2* out) {
  dt::Moments M{row, a_m};
  return dt::moment_coeffs(M, a, out) ? 1 : 0;
}

// The moment coefficients of every bucket, one thread per bucket (oneshot.py:143-160):
// ok[e] = 1 solved, 0 empty bucket, -1 non-finite (None).  Done by lane 0 of the
// locate warp, the small SVD solve left 31 lanes idle for ~22% of that kernel's time.
__global__ void dt2_coeffs_kernel(int64_t total, int R, int a_m, const double* __restrict__ meas,
                                  const int32_t* __restrict__ counts, int a_cap,
                                  la::c2* __restrict__ coeffs, int8_t* __restrict__ ok) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  int a = counts[e];
  if (a_cap > 0 && a > a_cap) a = a_cap;
  if (a <= 0) {
    ok[e] = 0;
    return;
  }
  la::c2 c[dt::kMaxAm];
  const int r = moment_coeffs_call(reinterpret_cast<const la::c2*>(meas) + e * R, a_m, a, c);
  for (int k = 0; k < a; ++k) coeffs[e * dt::kMaxAm + k] = c[k];
  ok[e] = r ? 1 : -1;
}

// w_L^j = exp(-2 pi i j / L), j < L: the grid-candidate roots shared by every bucket.
__global__ void roots_kernel(int64_t L, la::c2* __restrict__ roots) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < L) roots[j] = dt::root_pi_(j, L);
}

// dt2 locate with one warp per bucket (oneshot.py:182-198): lane 0 solves the
// moment coefficients, the lanes split the n/b grid candidates, and a butterfly
// merge of per-lane sorted lists keeps the `take` smallest |P| under (|P|, j) —
// exactly the stable argsort's first `take`.  cands[e][0..4) sorted; ncand[e] =
// count, 0 for an empty bucket, -1 for None.
constexpr int kDt2LocateThreads = 256;

// One lane's part of the dt2 grid scan for a bucket whose moment polynomial has degree
// A, then the warp's butterfly merge: bv/bj (A valid slots, the rest +inf / none) end
// up holding the `take` smallest (|P|, j) over all n/b candidates — the stable argsort's
// first `take` (oneshot.py:193-198).
template <int A>
__device__ __forceinline__ void dt2_scan(const la::c2* __restrict__ coef, int64_t bucket,
                                         int64_t b, int64_t n, int64_t step, int take,
                                         const la::c2* __restrict__ rootsL, int lane, double* bv_out,
                                         int64_t* bj_out) {
  constexpr int64_t kNone = INT64_MAX;
  la::c2 coeffs[A];
#pragma unroll
  for (int k = 0; k < A; ++k) coeffs[k] = coef[k];
  double bv[A];
  int64_t bj[A];
#pragma unroll
  for (int i = 0; i < A; ++i) {
    bv[i] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    bj[i] = kNone;
  }
  auto insert = [&](double v, int64_t j) {
#pragma unroll
    for (int i = 0; i < A; ++i) {
      const bool before = i < take && j != kNone &&
                          (bj[i] == kNone || v < bv[i] || (v == bv[i] && j < bj[i]));
      if (before) {
        const double tv = bv[i];
        const int64_t tj = bj[i];
        bv[i] = v;
        bj[i] = j;
        v = tv;
        j = tj;
      }
    }
  };
  const la::c2 z0 = dt::root_pi_(bucket, n);
  double worst = __longlong_as_double(0x7ff0000000000000ll);
  double worst_sq = worst;
  bool full = false;
  auto consider = [&](la::c2 y, int64_t j) {
    if (full && !(la::abs2(y) <= worst_sq)) return;  // |y| > worst beyond any rounding
    const double v = la::cabs(y);
    if (full && !(v < worst)) return;  // j ascends within a lane: earlier j wins ties
    insert(v, j);
#pragma unroll
    for (int i = 0; i < A; ++i)
      if (i == take - 1) {
        worst = bv[i];
        full = bj[i] != kNone;
      }
    worst_sq = worst * worst * (1.0 + 1e-13);
  };
  // explicit FMAs: the kernel is FP64-pipe bound, and the reference's |P| is matched to
  // rounding only either way (its roots come from exp() per candidate, these from a
  // table), so only ulp-level ties in the ranking can differ
  auto fmul = [](la::c2 u, la::c2 v) {
    return la::C(__fma_rn(u.re, v.re, -u.im * v.im), __fma_rn(u.re, v.im, u.im * v.re));
  };
  auto horner = [&](la::c2 z) {
    la::c2 y = la::add(z, coeffs[A - 1]);  // leading coefficient 1
#pragma unroll
    for (int kk = A - 2; kk >= 0; --kk)
      y = la::C(__fma_rn(y.re, z.re, __fma_rn(-y.im, z.im, coeffs[kk].re)),
                __fma_rn(y.re, z.im, __fma_rn(y.im, z.re, coeffs[kk].im)));
    return y;
  };
  int64_t j = lane;
  for (; j + 32 < step; j += 64) {  // two independent chains per lane
    const la::c2 y0 = horner(fmul(z0, rootsL[j]));
    const la::c2 y1 = horner(fmul(z0, rootsL[j + 32]));
    consider(y0, j);
    consider(y1, j + 32);
  }
  for (; j < step; j += 32) consider(horner(fmul(z0, rootsL[j])), j);
  for (int o = 16; o > 0; o >>= 1) {
    double ov[A];
    int64_t oj[A];
#pragma unroll
    for (int i = 0; i < A; ++i) {
      ov[i] = __shfl_xor_sync(0xffffffffu, bv[i], o);
      oj[i] = __shfl_xor_sync(0xffffffffu, bj[i], o);
    }
#pragma unroll
    for (int i = 0; i < A; ++i) insert(ov[i], oj[i]);
  }
#pragma unroll
  for (int i = 0; i < dt::kMaxAm; ++i) {
    bv_out[i] = i < A ? bv[i] : __longlong_as_double(0x7ff0000000000000ll);
    bj_out[i] = i < A ? bj[i] : kNone;
  }
}

__global__ void __launch_bounds__(kDt2LocateThreads, 2) dt2_locate_warp_kernel(
    int64_t total, int64_t nrows, int R, int a_m, const double* __restrict__ meas,
    const int32_t* __restrict__ counts, const int64_t* __restrict__ bucket_ids, int a_cap,
    int64_t b, int64_t n, const la::c2* __restrict__ rootsL, const la::c2* __restrict__ coef_all,
    const int8_t* __restrict__ coef_ok, int64_t* __restrict__ cands, int32_t* __restrict__ ncand) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= total) return;
  int a = counts[e];
  if (a_cap > 0 && a > a_cap) a = a_cap;
  const int ok = coef_ok[e];  // dt2_coeffs_kernel
  if (ok <= 0) {
    if (lane == 0) ncand[e] = ok;  // 0 empty, -1 None
    return;
  }
  const int64_t s = e / nrows;
  const int64_t bucket = bucket_ids ? bucket_ids[e] : e - s * nrows;
  const int64_t step = n / b;
  const int take = (int64_t)a < step ? a : (int)step;
  constexpr int64_t kNone = INT64_MAX;
  double bv[dt::kMaxAm];
  int64_t bj[dt::kMaxAm];
  // the scan with the polynomial degree a known at compile time (a is uniform in the
  // warp): exactly a Horner steps and a top-`take` list of a slots, no predicated
  // padding steps (the runtime-a form ran ~95 instructions per candidate pair)
  switch (a) {
    case 1: dt2_scan<1>(coef_all + e * dt::kMaxAm, bucket, b, n, step, take, rootsL, lane, bv, bj); break;
    case 2: dt2_scan<2>(coef_all + e * dt::kMaxAm, bucket, b, n, step, take, rootsL, lane, bv, bj); break;
    case 3: dt2_scan<3>(coef_all + e * dt::kMaxAm, bucket, b, n, step, take, rootsL, lane, bv, bj); break;
    default: dt2_scan<4>(coef_all + e * dt::kMaxAm, bucket, b, n, step, take, rootsL, lane, bv, bj); break;
  }
  if (lane == 0) {
    int64_t pos[dt::kMaxAm];
    int have = 0;
    for (int i = 0; i < take; ++i)
      if (bj[i] != kNone) pos[have++] = dt::pmod(bucket + b * bj[i], n);
    have = dt::sort_unique(pos, have);
    for (int i = 0; i < have; ++i) cands[e * dt::kMaxAm + i] = pos[i];
    ncand[e] = have;
  }
}

// Rows grouped by their tone count a (1..4) for the thread-per-row locate: a warp
// of mixed counts ran ~4 of 32 lanes per instruction (ncu, config 4).  bins[0..4]
// count rows per a; empty rows get ncand = 0 here and no slot.
__global__ void rows_by_count_kernel(int64_t total, const int32_t* __restrict__ counts, int a_cap,
                                     int32_t* __restrict__ bins, int32_t* __restrict__ ncand) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  int a = counts[e];
  if (a_cap > 0 && a > a_cap) a = a_cap;
  if (a <= 0) {
    ncand[e] = 0;
    return;
  }
  atomicAdd(bins + (a < dt::kMaxAm ? a : dt::kMaxAm), 1);
}
__global__ void rows_scatter_kernel(int64_t total, const int32_t* __restrict__ counts, int a_cap,
                                    const int32_t* __restrict__ bins, int32_t* __restrict__ fill,
                                    int32_t* __restrict__ order) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  int a = counts[e];
  if (a_cap > 0 && a > a_cap) a = a_cap;
  if (a <= 0) return;
  const int bin = a < dt::kMaxAm ? a : dt::kMaxAm;
  int base = 0;
  for (int k = 1; k < bin; ++k) base += bins[k];
  order[base + atomicAdd(fill + bin, 1)] = (int32_t)e;
}

// dt1 / dt3 locate (oneshot.py:161-191), one thread per bucket: ncand[e] = count,
// 0 for an empty bucket, -1 for None.  With `order`, thread i takes row order[i]
// (rows grouped by a; entries < 0 are past the non-empty rows).
__global__ void __launch_bounds__(kDtSolveThreads) dt_locate_rows_kernel(
    int64_t total, int64_t nrows, int R, int a_m, const double* __restrict__ meas,
    const int32_t* __restrict__ counts, const int64_t* __restrict__ bucket_ids, int a_cap,
    int variant, int64_t b, int64_t n, int64_t* __restrict__ cands, int32_t* __restrict__ ncand,
    const int32_t* __restrict__ order = nullptr) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  if (order) {
    e = order[e];
    if (e < 0) return;
  }
  int a = counts[e];
  if (a_cap > 0 && a > a_cap) a = a_cap;  // dsfft.py:219 caps at a_m
  if (a <= 0) {
    ncand[e] = 0;
    return;
  }
  const int64_t s = e / nrows;
  const int64_t bucket = bucket_ids ? bucket_ids[e] : e - s * nrows;
  dt::Moments M{reinterpret_cast<const la::c2*>(meas) + e * R, a_m};
  int64_t pos[5];
  const int c = dt::locate(M, a, variant, bucket, b, n, pos);
  for (int k = 0; k < c && k < dt::kMaxAm; ++k) cands[e * dt::kMaxAm + k] = pos[k];
  ncand[e] = c;
}

// estimate_values for every row, one group of W lanes per row (dt_warp.cuh): a full
// warp, or half a warp when p <= 16.  Row e belongs to signal e / nrows, whose random
// shifts start at rshifts + signal * shift_stride.  One warp per CTA.
template <int W>
__global__ void __launch_bounds__(32, W == 32 ? 24 : 16) dt_estimate_warp_kernel(
    int64_t total, int64_t nrows, int R, int a_m, int p, const double* __restrict__ meas,
    const int64_t* __restrict__ rshifts, int64_t shift_stride, const int64_t* __restrict__ cands,
    const int32_t* __restrict__ ncand, int64_t b, int64_t n, int out_stride,
    int64_t* __restrict__ out_pos, double* __restrict__ out_val, int32_t* __restrict__ out_cnt,
    const int32_t* __restrict__ order = nullptr) {
  constexpr int G = 32 / W;  // rows per warp
  __shared__ dtw::WarpPursuit<W> pursuit[G];
  __shared__ int64_t cand_s[G][dt::kMaxAm];
  const int g = threadIdx.x / W, lane = threadIdx.x & (W - 1);
  const unsigned gm = dtw::gmask<W>();
  int64_t e = (int64_t)blockIdx.x * G + g;
  if (e >= total) return;
  if (order) {  // rows grouped by a; out_cnt of the rows never listed is zeroed already
    e = order[e];
    if (e < 0) return;
  }
  int nc = 0;
  if (lane == 0) {
    nc = ncand[e];
    if (nc > dt::kMaxAm) nc = dt::kMaxAm;
    int64_t c[dt::kMaxAm];
    for (int k = 0; k < nc; ++k) c[k] = cands[e * dt::kMaxAm + k];
    if (nc > 0) nc = dt::sort_unique(c, nc);
    for (int k = 0; k < nc; ++k) cand_s[g][k] = c[k];
  }
  nc = __shfl_sync(gm, nc, 0, W);
  __syncwarp(gm);
  int cnt = 0;
  if (nc > 0) {
    const int64_t s = e / nrows;
    const la::c2* row = reinterpret_cast<const la::c2*>(meas) + e * R;
    cnt = dtw::warp_estimate<W>(pursuit[g], row + 3 * a_m, rshifts + s * shift_stride, p,
                                cand_s[g], nc, b, n, out_pos + e * out_stride,
                                reinterpret_cast<la::c2*>(out_val) + e * out_stride);
  }
  if (lane == 0) out_cnt[e] = cnt;
}

// ------------------------------------------------------------------ truncate

// truncate_spectrum's order by two stable block radix sorts of up to 8192 entries: by
// position, then by magnitude descending (key ~bits(|v|): non-negative doubles order like
// their bits), so equal magnitudes stay in position order — the (-|v|, f) key.
constexpr int kTruncSortItems = 8;
constexpr int kTruncSortMax = 1024 * kTruncSortItems;
using TruncSortF = cub::BlockRadixSort<uint32_t, 1024, kTruncSortItems, int32_t>;
using TruncSortM = cub::BlockRadixSort<uint64_t, 1024, kTruncSortItems, int32_t>;
union TruncSortTemp {
  typename TruncSortF::TempStorage f;
  typename TruncSortM::TempStorage m;
};

// Compact the per-bucket entries of each signal (bucket order, block scan over the
// per-row counts) and keep the k largest by (-|v|, f) with a bitonic sort — in
// shared memory when the signal's own entry count fits (smem_bytes), else in a global
// scratch (sized for the worst case, nrows a_m).  One CTA per signal.  (Deciding on the
// worst case sent config 4's ~8k entries per signal, 16 k possible, to a global-memory
// sort: 0.2 ms per call.)
__global__ void __launch_bounds__(1024) dt_truncate_kernel(
    int64_t nrows, int a_m, int k, const int64_t* __restrict__ pos,
    const double* __restrict__ val, const int32_t* __restrict__ cnt, int cap,
    int64_t* __restrict__ all_pos, double* __restrict__ all_val, int32_t* __restrict__ all_count,
    int64_t* __restrict__ out_pos, double* __restrict__ out_val, int32_t* __restrict__ out_count,
    unsigned char* gscratch, size_t scratch_bytes, size_t smem_bytes) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_sum[32];
  const int64_t s = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int32_t* c = cnt + s * nrows;
  int64_t* ap = all_pos + s * (int64_t)cap;
  la::c2* av = reinterpret_cast<la::c2*>(all_val) + s * (int64_t)cap;
  // exclusive scan of the row counts (contiguous chunk per thread)
  const int64_t per = (nrows + nt - 1) / nt;
  const int64_t lo = min(nrows, tid * per), hi = min(nrows, lo + per);
  int local = 0;
  for (int64_t r = lo; r < hi; ++r) local += c[r];
  int x = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    int v = lane < (nt >> 5) ? warp_sum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    warp_sum[lane] = v;
  }
  __syncthreads();
  int off = (w ? warp_sum[w - 1] : 0) + x - local;
  const int m = warp_sum[31];
  for (int64_t r = lo; r < hi; ++r) {
    for (int i = 0; i < c[r]; ++i) {
      const int64_t src = (s * nrows + r) * a_m + i;
      ap[off] = pos[src];
      av[off] = reinterpret_cast<const la::c2*>(val)[src];
      ++off;
    }
  }
  if (tid == 0) all_count[s] = m;
  __syncthreads();
  // radix sorts for 4097..8192 entries (a 8192-wide bitonic network took 0.18 against
  // 0.13 ms per call); the bitonic network for fewer (4096 wide: 0.04 against 0.09 ms)
  if (m > kTruncSortMax / 2 && m <= kTruncSortMax) {
    TruncSortTemp& ts = *reinterpret_cast<TruncSortTemp*>(smem_raw);
    uint32_t kf[kTruncSortItems];
    int32_t ix[kTruncSortItems];
#pragma unroll
    for (int j = 0; j < kTruncSortItems; ++j) {
      const int i = tid * kTruncSortItems + j;
      kf[j] = i < m ? (uint32_t)ap[i] : 0xffffffffu;  // positions < n < 2^32
      ix[j] = i < m ? i : -1;
    }
    TruncSortF(ts.f).Sort(kf, ix);
    __syncthreads();
    uint64_t km[kTruncSortItems];
#pragma unroll
    for (int j = 0; j < kTruncSortItems; ++j)  // padding sorts last (stable after |v| = 0)
      km[j] = ix[j] >= 0 ? ~(uint64_t)__double_as_longlong(la::cabs(av[ix[j]])) : ~0ull;
    TruncSortM(ts.m).Sort(km, ix);
    la::c2* ov = reinterpret_cast<la::c2*>(out_val) + s * k;
    const int kept = m < k ? m : k;
#pragma unroll
    for (int j = 0; j < kTruncSortItems; ++j) {
      const int r = tid * kTruncSortItems + j;
      if (r < kept) {
        out_pos[s * k + r] = ap[ix[j]];
        ov[r] = av[ix[j]];
      }
    }
    if (tid == 0) out_count[s] = kept;
    return;
  }
  int pow2 = 1;
  while (pow2 < m) pow2 <<= 1;
  unsigned char* mem =
      (size_t)pow2 * 20 <= smem_bytes || !gscratch ? smem_raw : gscratch + s * scratch_bytes;
  double* key = reinterpret_cast<double*>(mem);
  int64_t* kpos = reinterpret_cast<int64_t*>(key + pow2);
  int32_t* kidx = reinterpret_cast<int32_t*>(kpos + pow2);
  for (int i = tid; i < m; i += nt) {
    key[i] = la::cabs(av[i]);
    kpos[i] = ap[i];
    kidx[i] = i;
  }
  bitonic_trunc_sort(key, kpos, kidx, m, pow2);
  la::c2* ov = reinterpret_cast<la::c2*>(out_val) + s * k;
  const int kept = m < k ? m : k;
  for (int r = tid; r < kept; r += nt) {
    out_pos[s * k + r] = kpos[r];
    ov[r] = av[kidx[r]];
  }
  if (tid == 0) out_count[s] = kept;
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
  long long* qbuf = nullptr;
  e = scratch_alloc(reinterpret_cast<void**>(&qbuf), (size_t)batch * M * 8, st);
  if (e != cudaSuccess) return cuda_status(e, "scratch (vote keys)");
  dt_vote_kernel<<<(unsigned)batch, kVoteThreads, 0, st>>>((int)M, a_m, k, sigmas, counts, qbuf);
  scratch_free(qbuf, st);
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
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* cands = nullptr;
  const int64_t L = n / b;
  const size_t cbytes = ((size_t)total * (dt::kMaxAm * 8 + 4) + 255) / 256 * 256;
  // dt2: the grid roots, then the per-bucket coefficients and their status
  const size_t kbytes = ((size_t)total * dt::kMaxAm * 16 + 255) / 256 * 256;
  const size_t rbytes = variant == dt::VAR_DT2 ? ((size_t)L * 16 + 255) / 256 * 256 + kbytes +
                                                     (size_t)total
                                               : 0;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&cands), cbytes + rbytes, st);
  if (e != cudaSuccess) return cuda_status(e, "scratch (dt candidates)");
  int32_t* ncand = reinterpret_cast<int32_t*>(cands + total * dt::kMaxAm);
  // rows grouped by tone count a: the thread-per-row locate runs whole warps of one a,
  // and the pursuit's two half-warp buckets per warp usually share a (and with it
  // their support sizes and branch structure)
  int32_t* grp = nullptr;  // bins[8] | fill[8] | order[total]
  e = scratch_alloc(reinterpret_cast<void**>(&grp), 64 + (size_t)total * 4, st);
  if (e != cudaSuccess) {
    scratch_free(cands, st);
    return cuda_status(e, "scratch (dt row groups)");
  }
  int32_t* order = grp + 16;
  e = cudaMemsetAsync(grp, 0, 64, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(order, 0xff, (size_t)total * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(out_cnt, 0, (size_t)total * 4, st);
  if (e != cudaSuccess) {
    scratch_free(grp, st);
    scratch_free(cands, st);
    return cuda_status(e, "dt row groups");
  }
  {
    const unsigned g = (unsigned)((total + 255) / 256);
    rows_by_count_kernel<<<g, 256, 0, st>>>(total, counts, a_cap, grp, ncand);
    rows_scatter_kernel<<<g, 256, 0, st>>>(total, counts, a_cap, grp, grp + 8, order);
  }
  if (variant == dt::VAR_DT2) {
    char* base = reinterpret_cast<char*>(cands) + cbytes;
    la::c2* roots = reinterpret_cast<la::c2*>(base);
    la::c2* coef = reinterpret_cast<la::c2*>(base + ((size_t)L * 16 + 255) / 256 * 256);
    int8_t* cok = reinterpret_cast<int8_t*>(reinterpret_cast<char*>(coef) + kbytes);
    roots_kernel<<<(unsigned)((L + 255) / 256), 256, 0, st>>>(L, roots);
    dt2_coeffs_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
        total, 3 * a_m + p, a_m, rows, counts, a_cap, coef, cok);
    const int64_t threads = total * 32;
    dt2_locate_warp_kernel<<<(unsigned)((threads + kDt2LocateThreads - 1) / kDt2LocateThreads),
                             kDt2LocateThreads, 0, st>>>(total, nrows, 3 * a_m + p, a_m, rows,
                                                         counts, bucket_ids, a_cap, b, n, roots,
                                                         coef, cok, cands, ncand);
  } else {
    dt_locate_rows_kernel<<<(unsigned)((total + kDtSolveThreads - 1) / kDtSolveThreads),
                            kDtSolveThreads, 0, st>>>(total, nrows, 3 * a_m + p, a_m, rows,
                                                      counts, bucket_ids, a_cap, variant, b, n,
                                                      cands, ncand, order);
  }
  const char* wenv = getenv("AFFT_DT_EST_WIDTH");  // 32 forces the full-warp form
  if (p <= 16 && !(wenv && atoi(wenv) == 32))
    dt_estimate_warp_kernel<16><<<(unsigned)((total + 1) / 2), 32, 0, st>>>(
        total, nrows, 3 * a_m + p, a_m, p, rows, rand_shifts, p, cands, ncand, b, n, a_m,
        out_pos, out_val, out_cnt, order);
  else
    dt_estimate_warp_kernel<32><<<(unsigned)total, 32, 0, st>>>(
        total, nrows, 3 * a_m + p, a_m, p, rows, rand_shifts, p, cands, ncand, b, n, a_m,
        out_pos, out_val, out_cnt, order);
  scratch_free(grp, st);
  scratch_free(cands, st);
  AFFT_CHECK_LAUNCH("dt_estimate_warp_kernel");
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
  int64_t pow2 = 1;
  while (pow2 < std::max<int64_t>(cap, 1)) pow2 <<= 1;
  const size_t need = ((size_t)pow2 * 20 + 255) / 256 * 256;
  const size_t kSmemMax = 200 * 1024;
  // signals whose entries fit sort here; at least the radix sorts' temporary storage
  const size_t smem = std::max(std::min(need, kSmemMax), sizeof(TruncSortTemp));
  static_assert(sizeof(TruncSortTemp) <= 200 * 1024, "radix sort storage");
  unsigned char* scratch = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  if (need > kSmemMax) {  // the worst case does not fit: a global scratch for those
    cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&scratch), (size_t)batch * need, st);
    if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(dt_truncate scratch)");
  }
  cudaError_t e = ensure_smem((const void*)dt_truncate_kernel, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(dt_truncate)");
  dt_truncate_kernel<<<(unsigned)batch, 1024, smem, st>>>(
      nrows, a_m, k, pos, val, cnt, (int)cap, all_pos, all_val, all_count, out_pos, out_val,
      out_count, scratch, need, smem);
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
  if (p <= 16)
    dt_estimate_warp_kernel<16><<<(unsigned)((count + 1) / 2), 32, 0, (cudaStream_t)stream>>>(
        count, count, 3 * a_m + p, a_m, p, rows, rand_shifts, 0, cands, ncand, b, n,
        dt::kMaxAm, out_pos, out_val, out_n);
  else
    dt_estimate_warp_kernel<32><<<(unsigned)count, 32, 0, (cudaStream_t)stream>>>(
        count, count, 3 * a_m + p, a_m, p, rows, rand_shifts, 0, cands, ncand, b, n,
        dt::kMaxAm, out_pos, out_val, out_n);
  AFFT_CHECK_LAUNCH("dt_estimate_warp_kernel");
  return AFFT_OK;
}
