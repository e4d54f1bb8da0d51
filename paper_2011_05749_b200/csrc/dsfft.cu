// K6: DSFFT tree-layer primitives (dsfft.py:73-241).
//
//   afft_bucketize_rows   bucket values of selected buckets at arbitrary shifts,
//                         the measurement rows of _classify_active (dsfft.py:118-174)
//                         and collect_moments for _resolve_aliased (201-228).  Shifts
//                         in the same coset mod L = n/b share one size-b DFT:
//                         tau = q*L + r  =>  y_tau[i] = w_b^{i*q} * y_r[i]
//                         (substitute j' = j - q in the alias sum), so a layer needs
//                         min(#shifts, L) DFTs instead of #shifts — one at depth log2 n;
//                         optionally the per-bucket energies sum_t |y_tau[i]|^2 of all
//                         b buckets (the thresholds' floor / median set);
//   afft_active_indices   ascending indices i with |values[i]| > thr (initial_layer /
//                         expand_layer activity, 69-79, 114), a stream compaction;
//   afft_selective_sums   expand_layer's direct alias sums for candidate buckets
//                         (Eq. 23, dsfft.py:99-109): (1/b) sum_j x[j*L] w_b^{i*j}.
#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

#include <cub/block/block_radix_sort.cuh>

#include "afft_common.cuh"

extern "C" int afft_bucketize(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                              int64_t b, const int64_t* shifts, int32_t nshift, double* out,
                              int64_t out_signal_stride, int64_t out_shift_stride,
                              int64_t out_bin_stride, void* stream);

namespace afft {

struct RowsParams {
  int64_t b;
  int nshift;
  int64_t nrows;
  int32_t coset[AFFT_MAX_SHIFTS];  // which distinct-residue DFT serves shift t
  int64_t q[AFFT_MAX_SHIFTS];      // rotation count: tau mod n = q*L + r
};

// rows[r][t] = w_b^{(i_r * q_t) mod b} * Y[coset_t][i_r]
__global__ void rows_gather_kernel(const __grid_constant__ RowsParams p, const cd* __restrict__ Y,
                                   const int64_t* __restrict__ idx, cd* __restrict__ rows) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.nrows * p.nshift) return;
  const int64_t r = e / p.nshift;
  const int t = (int)(e - r * p.nshift);
  const int64_t i = idx[r];
  const cd y = Y[(int64_t)p.coset[t] * p.b + i];
  if (p.q[t] == 0) {
    rows[e] = y;
    return;
  }
  const int64_t ph = (i * p.q[t]) % p.b;
  double sn, cs;
  sincospi(-2.0 * (double)ph / (double)p.b, &sn, &cs);
  rows[e] = cmul(y, cd{cs, sn});
}

// rows_gather_kernel for rows of several signals: row r is bucket idx[r] of signal
// sig[r]; signal s's shift t is served by its coset DFT coset[s][t] (Y + (s U + coset) b)
// rotated by q[s][t].
__global__ void rows_gather_multi_kernel(const cd* __restrict__ Y, int64_t b, int U, int nshift,
                                         const int32_t* __restrict__ coset,
                                         const int64_t* __restrict__ q,
                                         const int64_t* __restrict__ idx,
                                         const int32_t* __restrict__ sig, int64_t nrows,
                                         cd* __restrict__ rows) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nrows * nshift) return;
  const int64_t r = e / nshift;
  const int t = (int)(e - r * nshift);
  const int64_t i = idx[r];
  const int s = sig[r];
  const int64_t qt = q[(int64_t)s * nshift + t];
  const cd y = Y[((int64_t)s * U + coset[(int64_t)s * nshift + t]) * b + i];
  if (qt == 0) {
    rows[e] = y;
    return;
  }
  const int64_t ph = (i * qt) % b;
  double sn, cs;
  sincospi(-2.0 * (double)ph / (double)b, &sn, &cs);
  rows[e] = cmul(y, cd{cs, sn});
}

int rows_gather_multi(const double* Y, int64_t b, int U, int nshift, const int32_t* coset,
                      const int64_t* q, const int64_t* idx, const int32_t* sig, int64_t nrows,
                      double* rows, cudaStream_t st) {
  if (nrows == 0) return AFFT_OK;
  const int64_t tot = nrows * nshift;
  rows_gather_multi_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const cd*>(Y), b, U, nshift, coset, q, idx, sig, nrows,
      reinterpret_cast<cd*>(rows));
  AFFT_CHECK_LAUNCH("rows_gather_multi_kernel");
  return AFFT_OK;
}

struct Mult {
  int32_t m[AFFT_MAX_SHIFTS];
};

// energy[i] = sum_t |y_tau_t[i]|^2 = sum_u mult_u |Y_u[i]|^2
__global__ void coset_energy_kernel(int64_t b, int U, const __grid_constant__ Mult mult,
                                    const cd* __restrict__ Y, double* __restrict__ energy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b) return;
  double e = 0.0;
  for (int u = 0; u < U; ++u) {
    const cd y = Y[(int64_t)u * b + i];
    const double m2 = cabs_(y);
    e += (double)mult.m[u] * (m2 * m2);
  }
  energy[i] = e;
}

// ---------------------------------------------------------------- compaction

constexpr int kCompactThreads = 1024;

__global__ void active_count_kernel(int64_t b, const cd* __restrict__ v, double thr,
                                    int32_t* __restrict__ block_counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = (i < b) && (cabs_(v[i]) > thr);
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}

// Exclusive scan of the per-block counts in one CTA of 1024 threads (chunked).
__global__ void scan_counts_kernel(int nblocks, int32_t* __restrict__ counts,
                                   int32_t* __restrict__ total) {
  __shared__ int32_t warp_sum[32];
  __shared__ int32_t carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblocks; base += blockDim.x) {
    const int i = base + tid;
    const int32_t v = i < nblocks ? counts[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      int32_t s = lane < (int)(blockDim.x >> 5) ? warp_sum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sum[lane] = s;
    }
    __syncthreads();
    const int32_t c = carry;
    if (i < nblocks) counts[i] = c + (w ? warp_sum[w - 1] : 0) + x - v;
    __syncthreads();
    if (tid == 0) carry = c + warp_sum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (tid == 0) *total = carry;
}

__global__ void active_write_kernel(int64_t b, const cd* __restrict__ v, double thr,
                                    const int32_t* __restrict__ offsets,
                                    const int64_t* __restrict__ map, int64_t* __restrict__ out) {
  __shared__ int warp_off[kCompactThreads / 32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = (i < b) && (cabs_(v[i]) > thr);
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_off[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < kCompactThreads / 32; ++k) {
      const int c = warp_off[k];
      warp_off[k] = run;
      run += c;
    }
  }
  __syncthreads();
  if (f) out[offsets[blockIdx.x] + warp_off[w] + __popc(m & ((1u << lane) - 1u))] = map ? map[i] : i;
}

// ---------------------------------------------------------------- selective sums

// out[c] = (1/b) sum_j x[j*L] * w_b^{(i_c * j) mod b}, one CTA per candidate
__global__ void selective_sum_kernel(const void* __restrict__ x, int dtype, int64_t n, int64_t b,
                                     const int64_t* __restrict__ cand, double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  const int64_t i = cand[c];
  const int64_t L = n / b;
  double re = 0.0, im = 0.0;
  for (int64_t j = threadIdx.x; j < b; j += blockDim.x) {
    const cd s = load_sample(x, dtype, j * L);
    double sn, cs;
    sincospi(-2.0 * (double)((i * j) % b) / (double)b, &sn, &cs);
    re += s.re * cs - s.im * sn;
    im += s.re * sn + s.im * cs;
  }
  __shared__ double wr[32], wi[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if ((threadIdx.x & 31) == 0) {
    wr[threadIdx.x >> 5] = re;
    wi[threadIdx.x >> 5] = im;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0, ti = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      tr += wr[w];
      ti += wi[w];
    }
    const double inv = 1.0 / (double)b;
    out[2 * c] = tr * inv;
    out[2 * c + 1] = ti * inv;
  }
}


// ---------------------------------------------------------------- alias rows
//
// Deep layers from the resident spectrum.  With Y = fft(x)/n (the signal's full
// normalised spectrum, computed once per decode) and L = n/b, substituting the
// inverse DFT into bucketize.py:96-99 gives the alias identity
//   bucketize(x, b, tau)[i] = w_n^(i tau) * sum_{l<L} Y[i + l b] * w_L^(l tau mod L),
// so a layer with small L needs L loads and L complex products per value instead
// of min(#shifts, L) size-b DFTs over the whole signal.  Used for L <= 32
// (kAliasMaxL), i.e. DSFFT's deepest layers, which otherwise each cost a full
// n-point transform's worth of passes.
constexpr int kAliasMaxL = 32;
constexpr int kAliasWarps = 8;

struct AliasShifts {
  int32_t nshift;
  int64_t tau[AFFT_MAX_SHIFTS];  // reduced into [0, n)
};

__device__ __forceinline__ cd root_pi(int64_t m, int64_t q) {  // exp(-2 pi i m / q)
  double sn, cs;
  sincospi(-2.0 * (double)m / (double)q, &sn, &cs);
  return cd{cs, sn};
}

// A full layer's tau = 0 value from its aliases y[l] = Y[i + l b], l < L (L a power of
// two <= LM), in the TREE order every path shares: T(i, d) = T(i, d+1) + T(i + 2^d, d+1)
// with T(i, log2 n) = Y[i] (expand_layer's parent = sum of children, dsfft.py:82-115)
// — i.e. y[l] += y[l + s] for s = L/2, ..., 1.  alias_all_kernel, alias_active_kernel,
// deep_flags_kernel, tree_level_kernel and the spectrum's fused epilogue
// (bucketize.cu) all produce exactly these sums, so their |v| > thr decisions agree
// bit for bit, and a tree costs L - 1 additions for every layer below it at once.
template <int LM>
__device__ __forceinline__ cd tree_sum(cd (&y)[LM], int L) {
#pragma unroll
  for (int s = LM / 2; s >= 1; s >>= 1)
    if (s < L) {
#pragma unroll
      for (int l = 0; l < s; ++l) y[l] = cadd(y[l], y[l + s]);
    }
  return y[0];
}

// rows[r][t] for selected buckets: one warp per row, lanes over the L spectrum
// terms (load) and then over the shifts (sum).  L <= kAliasRowsMaxL; dynamic shared
// memory holds the L roots and each warp's L spectrum terms.
constexpr int kAliasRowsMaxL = 256;

__global__ void __launch_bounds__(kAliasWarps * 32) alias_rows_kernel(
    const cd* __restrict__ Y, int64_t n, int64_t b, int L, const __grid_constant__ AliasShifts sh,
    const int64_t* __restrict__ idx, int64_t nrows, cd* __restrict__ rows) {
  extern __shared__ cd alias_smem[];
  cd* rootL = alias_smem;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  cd* ys = alias_smem + L + 2 * w * L;  // the warp's L terms + an L-entry work buffer
  for (int j = threadIdx.x; j < L; j += blockDim.x) rootL[j] = root_pi(j, L);
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * kAliasWarps + w;
  if (r >= nrows) return;
  const int64_t i = idx[r];
  for (int l = lane; l < L; l += 32) ys[l] = Y[i + (int64_t)l * b];
  __syncwarp();
  if ((L & (L - 1)) == 0) {
    // every coset value Z[rl] = sum_l ys[l] w_L^(l rl) at once: a radix-2 Stockham
    // DFT of the L aliases in the warp's two shared buffers (L log L products instead
    // of one L-term sum per shift: 72 shifts x L at DSFFT's 72-shift plan)
    cd* x = ys;
    cd* z = ys + L;
    for (int Ls = 1; Ls < L; Ls <<= 1) {
      const int stride = L / (2 * Ls);
      for (int k = lane; k < L / 2; k += 32) {
        const int j = k & (Ls - 1), g = k / Ls;
        const cd a = x[g * Ls + j];
        const cd t = j ? cmul(x[g * Ls + j + L / 2], rootL[j * stride]) : x[g * Ls + j + L / 2];
        z[2 * g * Ls + j] = cadd(a, t);
        z[2 * g * Ls + j + Ls] = csub(a, t);
      }
      __syncwarp();
      cd* tmp = x;
      x = z;
      z = tmp;
    }
    for (int t = lane; t < sh.nshift; t += 32) {
      const int64_t tau = sh.tau[t];
      rows[r * sh.nshift + t] = cmul(x[(int)(tau & (L - 1))], root_pi(mulmod(i, tau, n), n));
    }
    return;
  }
  for (int t = lane; t < sh.nshift; t += 32) {
    const int64_t tau = sh.tau[t];
    const int rl = (int)(tau % L);
    cd acc = ys[0];
    int m = 0;
    for (int l = 1; l < L; ++l) {
      m += rl;
      if (m >= L) m -= L;
      acc = cadd(acc, cmul(ys[l], rootL[m]));
    }
    rows[r * sh.nshift + t] = cmul(acc, root_pi(mulmod(i, tau, n), n));
  }
}

// alias_rows_kernel for rows of several signals (DSFFT batches): row r is bucket idx[r]
// of signal sig[r], whose spectrum is Y + sig n and whose reduced shifts are
// tau_tab[sig][0..nshift); L a power of two <= kAliasRowsMaxL.
__global__ void __launch_bounds__(kAliasWarps * 32) alias_rows_multi_kernel(
    const cd* __restrict__ Y, int64_t n, int64_t b, int L, const int64_t* __restrict__ tau_tab,
    int nshift, const int64_t* __restrict__ idx, const int32_t* __restrict__ sig, int64_t nrows,
    cd* __restrict__ rows) {
  extern __shared__ cd alias_smem[];
  cd* rootL = alias_smem;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  cd* ys = alias_smem + L + 2 * w * L;
  for (int j = threadIdx.x; j < L; j += blockDim.x) rootL[j] = root_pi(j, L);
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * kAliasWarps + w;
  if (r >= nrows) return;
  const int64_t i = idx[r];
  const int s = sig[r];
  const cd* Ys = Y + (int64_t)s * n;
  for (int l = lane; l < L; l += 32) ys[l] = Ys[i + (int64_t)l * b];
  __syncwarp();
  cd* x = ys;
  cd* z = ys + L;
  for (int Ls = 1; Ls < L; Ls <<= 1) {
    const int stride = L / (2 * Ls);
    for (int k = lane; k < L / 2; k += 32) {
      const int j = k & (Ls - 1), g = k / Ls;
      const cd a = x[g * Ls + j];
      const cd t = j ? cmul(x[g * Ls + j + L / 2], rootL[j * stride]) : x[g * Ls + j + L / 2];
      z[2 * g * Ls + j] = cadd(a, t);
      z[2 * g * Ls + j + Ls] = csub(a, t);
    }
    __syncwarp();
    cd* tmp = x;
    x = z;
    z = tmp;
  }
  const int64_t* taus = tau_tab + (int64_t)s * nshift;
  for (int t = lane; t < nshift; t += 32) {
    const int64_t tau = taus[t];
    rows[r * nshift + t] = cmul(x[(int)(tau & (L - 1))], root_pi(mulmod(i, tau, n), n));
  }
}

int alias_rows_multi(const double* Y, int64_t n, int64_t b, const int64_t* tau_tab, int nshift,
                     const int64_t* idx, const int32_t* sig, int64_t nrows, double* rows,
                     cudaStream_t st) {
  const int64_t L = n / b;
  if (nrows == 0 || nshift == 0) return AFFT_OK;
  if (L > kAliasRowsMaxL || (L & (L - 1)) || b < 1 || n % b) {
    set_error("alias_rows_multi: n/b = %lld unsupported", (long long)L);
    return AFFT_EUNSUPPORTED;
  }
  const size_t smem = (size_t)(1 + 2 * kAliasWarps) * L * sizeof(cd);
  cudaError_t e = ensure_smem((const void*)alias_rows_multi_kernel, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(alias_rows_multi)");
  alias_rows_multi_kernel<<<(unsigned)((nrows + kAliasWarps - 1) / kAliasWarps), kAliasWarps * 32,
                            smem, st>>>(reinterpret_cast<const cd*>(Y), n, b, (int)L, tau_tab,
                                        nshift, idx, sig, nrows, reinterpret_cast<cd*>(rows));
  AFFT_CHECK_LAUNCH("alias_rows_multi_kernel");
  return AFFT_OK;
}

// Rows for L > kAliasRowsMaxL (L a power of two): one CTA per row, the L aliases and
// a work buffer in shared memory, the radix-2 Stockham DFT across the CTA; every
// coset value at once (the rows of DSFFT's shallow noisy layers straight from the
// resident spectrum instead of 72 size-b DFTs over the signal).
__global__ void __launch_bounds__(256) alias_rows_cta_kernel(
    const cd* __restrict__ Y, int64_t n, int64_t b, int L, const __grid_constant__ AliasShifts sh,
    const int64_t* __restrict__ idx, int64_t nrows, cd* __restrict__ rows, bool tabled) {
  extern __shared__ cd alias_smem[];
  const int64_t r = blockIdx.x;
  if (r >= nrows) return;
  const int64_t i = idx[r];
  cd* x = alias_smem;
  cd* z = alias_smem + L;
  cd* rt = tabled ? alias_smem + 2 * L : nullptr;  // w_L^j, j < L/2
  for (int l = threadIdx.x; l < L; l += blockDim.x) x[l] = Y[i + (int64_t)l * b];
  if (rt)
    for (int j = threadIdx.x; j < L / 2; j += blockDim.x) rt[j] = root_pi(j, L);
  __syncthreads();
  for (int Ls = 1; Ls < L; Ls <<= 1) {
    for (int k = threadIdx.x; k < L / 2; k += blockDim.x) {
      const int j = k & (Ls - 1), g = k / Ls;
      const cd a = x[g * Ls + j];
      const cd u = x[g * Ls + j + L / 2];
      const int m = j * (L / (2 * Ls));
      const cd t = j ? cmul(u, rt ? rt[m] : root_pi(m, L)) : u;
      z[2 * g * Ls + j] = cadd(a, t);
      z[2 * g * Ls + j + Ls] = csub(a, t);
    }
    __syncthreads();
    cd* tmp = x;
    x = z;
    z = tmp;
  }
  for (int t = threadIdx.x; t < sh.nshift; t += blockDim.x) {
    const int64_t tau = sh.tau[t];
    rows[r * sh.nshift + t] = cmul(x[(int)(tau & (L - 1))], root_pi(mulmod(i, tau, n), n));
  }
}

// alias_rows_cta_kernel for rows of several signals (DSFFT batches, probe lists at the
// shallow layers): row r is bucket idx[r] of signal sig[r] (spectrum Y + sig n, reduced
// shifts tau_tab[sig][0..nshift)); the same arithmetic per row.
__global__ void __launch_bounds__(256) alias_rows_cta_multi_kernel(
    const cd* __restrict__ Y, int64_t n, int64_t b, int L, const int64_t* __restrict__ tau_tab,
    int nshift, const int64_t* __restrict__ idx, const int32_t* __restrict__ sig, int64_t nrows,
    cd* __restrict__ rows, bool tabled) {
  extern __shared__ cd alias_smem[];
  const int64_t r = blockIdx.x;
  if (r >= nrows) return;
  const int64_t i = idx[r];
  const int s = sig[r];
  const cd* Ys = Y + (int64_t)s * n;
  cd* x = alias_smem;
  cd* z = alias_smem + L;
  cd* rt = tabled ? alias_smem + 2 * L : nullptr;  // w_L^j, j < L/2
  for (int l = threadIdx.x; l < L; l += blockDim.x) x[l] = Ys[i + (int64_t)l * b];
  if (rt)
    for (int j = threadIdx.x; j < L / 2; j += blockDim.x) rt[j] = root_pi(j, L);
  __syncthreads();
  for (int Ls = 1; Ls < L; Ls <<= 1) {
    for (int k = threadIdx.x; k < L / 2; k += blockDim.x) {
      const int j = k & (Ls - 1), g = k / Ls;
      const cd a = x[g * Ls + j];
      const cd u = x[g * Ls + j + L / 2];
      const int m = j * (L / (2 * Ls));
      const cd t = j ? cmul(u, rt ? rt[m] : root_pi(m, L)) : u;
      z[2 * g * Ls + j] = cadd(a, t);
      z[2 * g * Ls + j + Ls] = csub(a, t);
    }
    __syncthreads();
    cd* tmp = x;
    x = z;
    z = tmp;
  }
  const int64_t* taus = tau_tab + (int64_t)s * nshift;
  for (int t = threadIdx.x; t < nshift; t += blockDim.x) {
    const int64_t tau = taus[t];
    rows[r * nshift + t] = cmul(x[(int)(tau & (L - 1))], root_pi(mulmod(i, tau, n), n));
  }
}

int alias_rows_cta_multi(const double* Y, int64_t n, int64_t b, const int64_t* tau_tab,
                         int nshift, const int64_t* idx, const int32_t* sig, int64_t nrows,
                         double* rows, cudaStream_t st) {
  const int64_t L = n / b;
  if (nrows == 0 || nshift == 0) return AFFT_OK;
  if (L > kAliasCtaMaxL || (L & (L - 1)) || b < 1 || n % b) {
    set_error("alias_rows_cta_multi: n/b = %lld unsupported", (long long)L);
    return AFFT_EUNSUPPORTED;
  }
  const bool tabled = true;  // L <= kAliasCtaMaxL, as afft_alias_rows
  const size_t smem = (size_t)(tabled ? 2 * L + L / 2 : 2 * L) * sizeof(cd);
  cudaError_t e = ensure_smem((const void*)alias_rows_cta_multi_kernel, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(alias_rows_cta_multi)");
  alias_rows_cta_multi_kernel<<<(unsigned)nrows, 256, smem, st>>>(
      reinterpret_cast<const cd*>(Y), n, b, (int)L, tau_tab, nshift, idx, sig, nrows,
      reinterpret_cast<cd*>(rows), tabled);
  AFFT_CHECK_LAUNCH("alias_rows_cta_multi_kernel");
  return AFFT_OK;
}

struct AliasCosets {
  int32_t U;
  int32_t r[kAliasMaxL];     // distinct tau mod L
  int32_t mult[kAliasMaxL];  // shifts per residue
};

// All b buckets: energy[i] = sum_t |y_tau_t[i]|^2 (the w_n^(i tau) factor has modulus 1,
// so shifts with equal tau mod L contribute equal terms); vals0 (optional) = the
// tau = 0 values sum_l Y[i + l b].
// LM >= L: the register footprint follows L (at LM = 32 the kernel holds 158
// registers, one CTA per SM, which left the L = 2 layer latency-bound at 1.1 TB/s).
template <int LM>
__global__ void __launch_bounds__(256) alias_all_kernel(const cd* __restrict__ Y, int64_t b, int L,
                                                        const __grid_constant__ AliasCosets cs,
                                                        double* __restrict__ energy,
                                                        cd* __restrict__ vals0) {
  __shared__ cd rootL[kAliasMaxL];
  if (threadIdx.x < L) rootL[threadIdx.x] = root_pi(threadIdx.x, L);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b) return;
  cd y[LM];
#pragma unroll
  for (int l = 0; l < LM; ++l)
    if (l < L) y[l] = Y[i + (int64_t)l * b];
  if (vals0) {
    cd t[LM];
#pragma unroll
    for (int l = 0; l < LM; ++l) t[l] = y[l];
    vals0[i] = tree_sum<LM>(t, L);
  }
  if (energy) {
    double e = 0.0;
    for (int u = 0; u < cs.U; ++u) {
      cd acc = y[0];
      int m = 0;
#pragma unroll
      for (int l = 1; l < LM; ++l) {
        if (l < L) {
          m += cs.r[u];
          if (m >= L) m -= L;
          acc = cadd(acc, cmul(y[l], rootL[m]));
        }
      }
      const double m2 = cabs_(acc);
      e += (double)cs.mult[u] * (m2 * m2);
    }
    energy[i] = e;
  }
}

// Full deep layer straight to its active set, in one pass over the resident spectrum:
// the tau = 0 value of bucket i is sum_l Y[i + l b] in the tree order (tree_sum: |v| and
// the decision are bit-identical to values + afft_active_indices), tested against thr,
// and never written.  Each CTA compacts its
// active buckets (ascending within the CTA) and reserves a segment of `out` with one
// atomic, only when it has any; sort_active_kernel then puts the list in ascending
// order.  Against values + count + scan + write, this reads Y once and the values never.
template <int LM>
__global__ void __launch_bounds__(256) alias_active_kernel(const cd* __restrict__ Y, int64_t b,
                                                           int L, double thr,
                                                           int64_t* __restrict__ out, int cap,
                                                           int32_t* __restrict__ count) {
  __shared__ int warp_cnt[8];
  __shared__ int base;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (i < b) {
    cd y[LM];
#pragma unroll
    for (int l = 0; l < LM; ++l)
      if (l < L) y[l] = Y[i + (int64_t)l * b];
    f = cabs_(tree_sum<LM>(y, L)) > thr;
  }
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_cnt[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < 8; ++k) {
      const int c = warp_cnt[k];
      warp_cnt[k] = run;
      run += c;
    }
    base = run ? atomicAdd(count, run) : 0;
  }
  __syncthreads();
  if (f) {
    const int at = base + warp_cnt[w] + __popc(m & ((1u << lane) - 1u));
    if (at < cap) out[at] = i;
  }
}

// Ascending order of the active list: one CTA, cub's block radix sort over the
// bucket indices as 32-bit keys (b <= 2^31), 16 per thread, bits [0, log2 b) only.
// (A bitonic sort of the ~5,000 entries of config 4's deep layers took 87 us.)
constexpr int kActiveSortThreads = 1024, kActiveSortItems = 16;
constexpr int kActiveSortCap = kActiveSortThreads * kActiveSortItems;
using ActiveSort = cub::BlockRadixSort<uint32_t, kActiveSortThreads, kActiveSortItems>;
__global__ void __launch_bounds__(kActiveSortThreads) sort_active_kernel(
    int64_t* __restrict__ list, const int32_t* __restrict__ count, int cap, int end_bit) {
  extern __shared__ __align__(16) unsigned char sort_smem[];
  auto& temp = *reinterpret_cast<typename ActiveSort::TempStorage*>(sort_smem);
  const int m = *count;
  if (m <= 1 || m > cap || m > kActiveSortCap) return;  // over capacity: the list is partial
  uint32_t keys[kActiveSortItems];
#pragma unroll
  for (int k = 0; k < kActiveSortItems; ++k) {
    const int i = threadIdx.x * kActiveSortItems + k;
    keys[k] = i < m ? (uint32_t)list[i] : 0xffffffffu;
  }
  ActiveSort(temp).Sort(keys, 0, end_bit);
#pragma unroll
  for (int k = 0; k < kActiveSortItems; ++k) {
    const int i = threadIdx.x * kActiveSortItems + k;
    if (i < m) list[i] = keys[k];
  }
}

// Launches alias_active_kernel + sort_active_kernel; *count (device, zeroed here) is the
// full active count, the list holds it only if it is <= min(cap, kActiveSortCap).
int alias_active(const double* spectrum, int64_t n, int64_t b, double thr, int64_t* out, int cap,
                 int32_t* count, cudaStream_t st) {
  const int64_t L = n / b;
  if (L > kAliasMaxL || b < 1 || n % b) {
    set_error("alias_active: n/b = %lld", (long long)L);
    return AFFT_EUNSUPPORTED;
  }
  cudaError_t e = cudaMemsetAsync(count, 0, 4, st);
  if (e != cudaSuccess) return cuda_status(e, "alias_active count");
  const cd* Y = reinterpret_cast<const cd*>(spectrum);
  const unsigned grid = (unsigned)((b + 255) / 256);
  if (L <= 2)
    alias_active_kernel<2><<<grid, 256, 0, st>>>(Y, b, (int)L, thr, out, cap, count);
  else if (L <= 4)
    alias_active_kernel<4><<<grid, 256, 0, st>>>(Y, b, (int)L, thr, out, cap, count);
  else if (L <= 8)
    alias_active_kernel<8><<<grid, 256, 0, st>>>(Y, b, (int)L, thr, out, cap, count);
  else if (L <= 16)
    alias_active_kernel<16><<<grid, 256, 0, st>>>(Y, b, (int)L, thr, out, cap, count);
  else
    alias_active_kernel<kAliasMaxL><<<grid, 256, 0, st>>>(Y, b, (int)L, thr, out, cap, count);
  const size_t smem = sizeof(typename ActiveSort::TempStorage);
  e = ensure_smem((const void*)sort_active_kernel, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(sort_active)");
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < b) ++end_bit;
  sort_active_kernel<<<1, kActiveSortThreads, smem, st>>>(out, count, cap, end_bit);
  AFFT_CHECK_LAUNCH("alias_active");
  return AFFT_OK;
}

// ---------------------------------------------------------------- all deep layers
//
// Every full deep layer (L = n/b <= 32: depths dmin = log2(n) - log2(Lmax) .. log2 n)
// in ONE pass over the resident spectrum, instead of one pass + a one-CTA sort per
// layer.  Thread i0 < bmin loads its Lmax aliases y[l] = Y[i0 + l bmin]; layer j
// (b_j = bmin 2^j, L_j = Lmax >> j) holds the buckets i0 + m bmin, m < 2^j, whose tau = 0
// value is T_j(m) = T_{j+1}(m) + T_{j+1}(m + 2^j), T_log2(Lmax)(m) = y[m] — the tree order
// of tree_sum, computed deepest layer first in place (Lmax - 1 additions for all
// layers), so the decisions |v| > thr_j are bit-identical to alias_active_kernel's.  The
// warp's flags for one (layer, m) are one 32-bit word of the layer's bitmap (lanes
// hold consecutive i0); a count / scan / write pass then turns the bitmaps into
// ascending active lists, all layers at once.
constexpr int kDeepMaxLayers = 16;
struct DeepLayers {
  int nl;                          // layers: j = 0 .. nl - 1
  double thr[kDeepMaxLayers];      // activity threshold of layer j
  double t2hi[kDeepMaxLayers], t2lo[kDeepMaxLayers];  // thr^2 (1 +- 1e-14), the guard band
  int64_t word_off[kDeepMaxLayers + 1];   // bitmap words before layer j
  int64_t chunk_off[kDeepMaxLayers + 1];  // count chunks before layer j
};
constexpr int kDeepChunkWords = 2048;  // words per count / write CTA (256 threads x 8)

// f(integral_constant<J>) for J = TOP, TOP - 1, ..., 0
template <int TOP, class F, int... K>
__device__ __forceinline__ void deepest_first(F& f, std::integer_sequence<int, K...>) {
  (f(std::integral_constant<int, TOP - K>{}), ...);
}

template <int LM, int LOG2LM>
__global__ void __launch_bounds__(128) deep_flags_kernel(const cd* __restrict__ Y, int64_t bmin,
                                                         const __grid_constant__ DeepLayers D,
                                                         int jd, uint32_t* __restrict__ words,
                                                         cd* __restrict__ v_out) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool on = i0 < bmin;
  cd y[LM];
#pragma unroll
  for (int l = 0; l < LM; ++l) y[l] = on ? Y[i0 + (int64_t)l * bmin] : cd{0.0, 0.0};
  const int lane = threadIdx.x & 31;
  // layer j: b = bmin 2^j, L = LM >> j; y[m] = T_j(m) after its additions.  Compile-time
  // j per level (runtime loop bounds left y[] in local memory).
  auto level = [&](auto jc) {
    constexpr int j = decltype(jc)::value;
    if (j < LOG2LM) {
#pragma unroll
      for (int m = 0; m < (1 << j); ++m) y[m] = cadd(y[m], y[m + (1 << j)]);
    }
    if (jd + j >= D.nl) return;
#pragma unroll
    for (int m = 0; m < (1 << j); ++m) {
      const cd acc = y[m];
      if (j == 0 && v_out && on) v_out[i0] = acc;  // the shallowest deep layer's values
      // |v| > thr decided on |v|^2 against thr^2 with a 1e-14 guard band (|v|^2 in double
      // is within 3 ulp, hypot within 1): only values inside the band take hypot, so
      // every decision equals hypot(v) > thr (alias_active_kernel's test)
      const double sq = acc.re * acc.re + acc.im * acc.im;
      const double thr = D.thr[jd + j];
      const bool f = sq > D.t2hi[jd + j] ? true : sq < D.t2lo[jd + j] ? false : cabs_(acc) > thr;
      const unsigned flags = __ballot_sync(0xffffffffu, on && f);
      if (lane == 0 && on)
        words[D.word_off[jd + j] + (i0 >> 5) + (int64_t)m * (bmin >> 5)] = flags;
    }
  };
  deepest_first<LOG2LM>(level, std::make_integer_sequence<int, LOG2LM + 1>{});
}

// popcounts of kDeepChunkWords words per CTA; chunks never straddle two layers
__global__ void __launch_bounds__(256) deep_count_kernel(const uint32_t* __restrict__ words,
                                                         const __grid_constant__ DeepLayers D,
                                                         int32_t* __restrict__ chunk_cnt) {
  const int64_t c = blockIdx.x;
  int j = 0;
  while (j + 1 < D.nl && c >= D.chunk_off[j + 1]) ++j;
  const int64_t w0 = D.word_off[j] + (c - D.chunk_off[j]) * kDeepChunkWords;
  const int64_t w1 = min(D.word_off[j + 1], w0 + kDeepChunkWords);
  int cnt = 0;
  for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) cnt += __popc(words[w]);
  __shared__ int part[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < 8; ++k) t += part[k];
    chunk_cnt[c] = t;
  }
}

// exclusive scan of the chunk counts within each layer (one CTA), layer totals out
// one warp per layer: lanes take contiguous runs of chunks, a warp scan joins them
__global__ void deep_scan_kernel(int32_t* __restrict__ chunk_cnt,
                                 const __grid_constant__ DeepLayers D,
                                 int32_t* __restrict__ layer_count) {
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= D.nl) return;
  const int64_t c0 = D.chunk_off[j], nc = D.chunk_off[j + 1] - c0;
  const int64_t per = (nc + 31) / 32;
  const int64_t lo = c0 + min(nc, lane * per), hi = c0 + min(nc, (lane + 1) * per);
  int local = 0;
  for (int64_t c = lo; c < hi; ++c) local += chunk_cnt[c];
  int x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int run = x - local;
  for (int64_t c = lo; c < hi; ++c) {
    const int v = chunk_cnt[c];
    chunk_cnt[c] = run;
    run += v;
  }
  if (lane == 31) layer_count[j] = x;
}

// ascending bucket indices of every layer: list j at out + j * cap (first cap kept)
__global__ void __launch_bounds__(256) deep_write_kernel(const uint32_t* __restrict__ words,
                                                         const __grid_constant__ DeepLayers D,
                                                         const int32_t* __restrict__ chunk_base,
                                                         int64_t* __restrict__ out, int cap) {
  const int64_t c = blockIdx.x;
  int j = 0;
  while (j + 1 < D.nl && c >= D.chunk_off[j + 1]) ++j;
  const int64_t lw0 = (c - D.chunk_off[j]) * kDeepChunkWords;  // first word within the layer
  const int64_t w0 = D.word_off[j] + lw0;
  const int64_t nw = min(D.word_off[j + 1] - w0, (int64_t)kDeepChunkWords);
  constexpr int PER = kDeepChunkWords / 256;  // contiguous words per thread
  uint32_t wv[PER];
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int64_t w = (int64_t)threadIdx.x * PER + k;
    wv[k] = w < nw ? words[w0 + w] : 0u;
    cnt += __popc(wv[k]);
  }
  // block exclusive scan of cnt
  __shared__ int warp_tot[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yv = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += yv;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  int woff = 0;
  for (int k = 0; k < wid; ++k) woff += warp_tot[k];
  int at = chunk_base[c] + woff + x - cnt;
  int64_t* lst = out + (int64_t)j * cap;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    uint32_t v = wv[k];
    const int64_t bit0 = (lw0 + (int64_t)threadIdx.x * PER + k) * 32;
    while (v) {
      const int t = __ffs(v) - 1;
      v &= v - 1;
      if (at < cap) lst[at] = bit0 + t;
      ++at;
    }
  }
}

// One shallower full layer from the next one: parent = sum of its two children
// (v_d[i] = v_{d+1}[i] + v_{d+1}[i + 2^d], the identity behind expand_layer's
// "children {i, i + 2^(d-1)}", dsfft.py:82-115), flags into the layer's bitmap.
__global__ void __launch_bounds__(256) tree_level_kernel(const cd* __restrict__ vin, int64_t b,
                                                         double thr, cd* __restrict__ vout,
                                                         uint32_t* __restrict__ words) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool on = i < b;
  cd v = cd{0.0, 0.0};
  if (on) {
    v = cadd(vin[i], vin[i + b]);
    vout[i] = v;
  }
  const double sq = v.re * v.re + v.im * v.im, t2 = thr * thr;
  const bool f = on && (sq > t2 * (1.0 + 1e-14) ? true
                        : sq < t2 * (1.0 - 1e-14) ? false
                                                  : cabs_(v) > thr);
  const unsigned flags = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && on) words[i >> 5] = flags;
}

// The same layers in ONE launch when 3 <= dmid - d0 <= 8 (config 4: depths 19 .. 12
// from the depth-20 values the fused last pass leaves): the subtree under depth-d0 index
// i is {i + m 2^d0, m < 2^LV} and every level halves m (v[m] += v[m + half], the same
// pair and operand order as tree_level_kernel, so values and bitmaps are bit-identical).
// A CTA owns 32 consecutive i (one bitmap word per (level, m)): lane = i, warp = m mod 8,
// a thread holds m = warp + 8 q, q < 2^(LV - 3); the first LV - 3 levels stay in
// registers, the last three go through 4 KB of shared memory.  One launch of 2^d0 / 32
// CTAs instead of LV launches of a few microseconds each.
struct TreeLevels {
  const cd* vin;       // depth dmid values
  cd* vout[8];         // [l]: depth dmid - 1 - l values
  uint32_t* words[8];  // [l]: that layer's bitmap
  double thr[8];
};

__device__ __forceinline__ bool tree_flag(cd v, double thr) {
  const double sq = v.re * v.re + v.im * v.im, t2 = thr * thr;
  return sq > t2 * (1.0 + 1e-14) ? true : sq < t2 * (1.0 - 1e-14) ? false : cabs_(v) > thr;
}

template <int LQ>
__global__ void __launch_bounds__(256) tree_levels_kernel(const __grid_constant__ TreeLevels T,
                                                          int d0) {
  constexpr int Q = 1 << LQ;
  __shared__ cd sh[8][32];
  const int lane = threadIdx.x & 31, ms = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  cd a[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) a[q] = T.vin[i + ((int64_t)(ms + 8 * q) << d0)];
  int l = 0;
#pragma unroll
  for (int h = Q / 2; h >= 1; h >>= 1, ++l) {
#pragma unroll
    for (int q = 0; q < h; ++q) {
      a[q] = cadd(a[q], a[q + h]);
      const int64_t at = i + ((int64_t)(ms + 8 * q) << d0);
      T.vout[l][at] = a[q];
      const unsigned flags = __ballot_sync(0xffffffffu, tree_flag(a[q], T.thr[l]));
      if (lane == 0) T.words[l][at >> 5] = flags;
    }
  }
  cd v = a[0];
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1, ++l) {
    sh[ms][lane] = v;
    __syncthreads();
    if (ms < h) {  // warp-uniform
      v = cadd(v, sh[ms + h][lane]);
      const int64_t at = i + ((int64_t)ms << d0);
      T.vout[l][at] = v;
      const unsigned flags = __ballot_sync(0xffffffffu, tree_flag(v, T.thr[l]));
      if (lane == 0) T.words[l][at >> 5] = flags;
    }
    __syncthreads();
  }
}

// thr and its guard band, rounded exactly as the kernels would (IEEE, no contraction)
static void set_layer_threshold(DeepLayers* D, int j, double thr) {
  const double t2 = thr * thr;
  D->thr[j] = thr;
  D->t2hi[j] = t2 * (1.0 + 1e-14);
  D->t2lo[j] = t2 * (1.0 - 1e-14);
}

static void full_layers_layout(int64_t n, int d0, int nl, DeepLayers* D, int* jd, size_t* words_b,
                               size_t* chunks_b, size_t* vbuf_b) {
  memset(D, 0, sizeof(*D));
  D->nl = nl;
  int log2n = 0;
  while ((int64_t(1) << log2n) < n) ++log2n;
  const int dd = std::max(d0, log2n - 5);  // first layer with n/b <= 32
  *jd = dd - d0;
  for (int j = 0; j < nl; ++j) {
    const int64_t nw = (int64_t(1) << (d0 + j)) / 32;
    D->word_off[j + 1] = D->word_off[j] + nw;
    D->chunk_off[j + 1] = D->chunk_off[j] + (nw + kDeepChunkWords - 1) / kDeepChunkWords;
  }
  *words_b = ((size_t)D->word_off[nl] * 4 + 255) & ~size_t(255);
  *chunks_b = ((size_t)D->chunk_off[nl] * 4 + 255) & ~size_t(255);
  size_t v = 0;  // values of layers 0 .. jd (the shallow ones and the first deep one)
  for (int j = 0; j <= *jd && *jd > 0; ++j) v += ((size_t)16 << (d0 + j));
  *vbuf_b = v;
}

// Active lists of the full layers at depths d0 .. d0 + nl - 1 (thr[j] for depth d0 + j)
// from the resident spectrum: the layers with n/b <= 32 in one pass (deep_flags), the
// shallower ones by summing children pairwise from there down, then one count / scan /
// write over every layer's bitmap.  lists [nl][cap] ascending (device), counts [nl]
// (device; a count above cap means the list is partial).
int full_active_all(const double* spectrum, int64_t n, int d0, int nl, const double* thr,
                    int64_t* out, int cap, int32_t* counts, void* scratch, size_t scratch_bytes,
                    cudaStream_t st) {
  DeepLayers D;
  int jd = 0;
  size_t wb = 0, cb = 0, vb = 0;
  if (nl < 1 || nl > kDeepMaxLayers || (int64_t(1) << d0) < 32 || (n & (n - 1)) ||
      (int64_t(1) << (d0 + nl - 1)) > n) {
    set_error("full_active_all: unsupported layers (n=%lld, d0=%d, nl=%d)", (long long)n, d0, nl);
    return AFFT_EUNSUPPORTED;
  }
  full_layers_layout(n, d0, nl, &D, &jd, &wb, &cb, &vb);
  if (jd >= nl) {
    set_error("full_active_all: no layer with n/b <= 32 among the requested ones");
    return AFFT_EUNSUPPORTED;
  }
  for (int j = 0; j < nl; ++j) set_layer_threshold(&D, j, thr[j]);
  if (!scratch || scratch_bytes < wb + cb + vb) {
    set_error("full_active_all: scratch of %zu bytes needed", wb + cb + vb);
    return AFFT_ENOMEM;
  }
  uint32_t* words = reinterpret_cast<uint32_t*>(scratch);
  int32_t* chunk = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(scratch) + wb);
  cd* vbuf = jd > 0 ? reinterpret_cast<cd*>(reinterpret_cast<char*>(scratch) + wb + cb) : nullptr;
  // layer j's values at vbuf + vofs[j]
  int64_t vofs[kDeepMaxLayers + 1] = {0};
  for (int j = 0; j < jd; ++j) vofs[j + 1] = vofs[j] + (int64_t(1) << (d0 + j));
  const cd* Y = reinterpret_cast<const cd*>(spectrum);
  const int64_t bmin = int64_t(1) << (d0 + jd);
  const int64_t Lmax = n / bmin;
  cd* vdeep = vbuf ? vbuf + vofs[jd] : nullptr;
  const unsigned grid = (unsigned)((bmin + 127) / 128);
  switch (Lmax) {
    case 1: deep_flags_kernel<1, 0><<<grid, 128, 0, st>>>(Y, bmin, D, jd, words, vdeep); break;
    case 2: deep_flags_kernel<2, 1><<<grid, 128, 0, st>>>(Y, bmin, D, jd, words, vdeep); break;
    case 4: deep_flags_kernel<4, 2><<<grid, 128, 0, st>>>(Y, bmin, D, jd, words, vdeep); break;
    case 8: deep_flags_kernel<8, 3><<<grid, 128, 0, st>>>(Y, bmin, D, jd, words, vdeep); break;
    case 16: deep_flags_kernel<16, 4><<<grid, 128, 0, st>>>(Y, bmin, D, jd, words, vdeep); break;
    case 32: deep_flags_kernel<32, 5><<<grid, 128, 0, st>>>(Y, bmin, D, jd, words, vdeep); break;
    default:
      set_error("full_active_all: n/bmin = %lld is not a power of two <= 32", (long long)Lmax);
      return AFFT_EUNSUPPORTED;
  }
  AFFT_CHECK_LAUNCH("deep_flags_kernel");
  for (int j = jd - 1; j >= 0; --j) {
    const int64_t b = int64_t(1) << (d0 + j);
    tree_level_kernel<<<(unsigned)((b + 255) / 256), 256, 0, st>>>(
        vbuf + vofs[j + 1], b, thr[j], vbuf + vofs[j], words + D.word_off[j]);
  }
  AFFT_CHECK_LAUNCH("tree_level_kernel");
  const unsigned chunks = (unsigned)D.chunk_off[nl];
  deep_count_kernel<<<chunks, 256, 0, st>>>(words, D, chunk);
  deep_scan_kernel<<<1, 32 * kDeepMaxLayers, 0, st>>>(chunk, D, counts);
  deep_write_kernel<<<chunks, 256, 0, st>>>(words, D, chunk, out, cap);
  AFFT_CHECK_LAUNCH("deep_write_kernel");
  return AFFT_OK;
}

// full_active_all with the spectrum computed here: the last K2' pass decides every layer
// at depths dtop + 4 .. log2(n) (dtop = log2(n) - 8) in its epilogue (bucketize.cu
// deep_fuse_epilogue, the tree_sum order, so the bitmaps are bit-identical to
// deep_flags_kernel's) and leaves the depth-(dtop + 4) values; tree_level_kernel makes
// the shallower layers from them; sum |Y|^2 into *norm2 (device, zeroed here).  Saves
// the deep_flags pass over Y (n 16 bytes) and the |x|^2 pass.
// Scratch: bitmaps | count chunks | values of depths dmid = dtop + 4, dmid - 1, ..., d0.
static void fused_layout(int64_t n, int d0, int nl, DeepLayers* D, size_t* wb, size_t* cb,
                         int* dmid, size_t* vb) {
  int jd = 0, log2n = 0;
  size_t vdummy = 0;
  full_layers_layout(n, d0, nl, D, &jd, wb, cb, &vdummy);
  while ((int64_t(1) << log2n) < n) ++log2n;
  *dmid = log2n - 4;
  *vb = 0;
  if (d0 < *dmid)
    for (int d = d0; d <= *dmid; ++d) *vb += (size_t)16 << d;
}

size_t full_active_fused_scratch(int64_t n, int d0, int nl) {
  DeepLayers D;
  size_t wb = 0, cb = 0, vb = 0;
  int dmid = 0;
  fused_layout(n, d0, nl, &D, &wb, &cb, &dmid, &vb);
  return wb + cb + vb;
}

int full_active_all_fused(const void* x, int dtype, int64_t n, double* Yout, int d0, int nl,
                          const double* thr, int64_t* out, int cap, int32_t* counts,
                          double* norm2, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  int log2n = 0;
  while ((int64_t(1) << log2n) < n) ++log2n;
  const int dtop = log2n - 8;
  if (nl < 1 || nl > kDeepMaxLayers || (int64_t(1) << d0) < 32 || (n & (n - 1)) ||
      d0 + nl - 1 != log2n || dtop < 12) {
    set_error("full_active_all_fused: unsupported layers (n=%lld, d0=%d, nl=%d)", (long long)n,
              d0, nl);
    return AFFT_EUNSUPPORTED;
  }
  DeepLayers D;
  size_t wb = 0, cb = 0, vb = 0;
  int dmid = 0;
  fused_layout(n, d0, nl, &D, &wb, &cb, &dmid, &vb);
  for (int j = 0; j < nl; ++j) set_layer_threshold(&D, j, thr[j]);
  if (!scratch || scratch_bytes < wb + cb + vb) {
    set_error("full_active_all_fused: scratch of %zu bytes needed", wb + cb + vb);
    return AFFT_ENOMEM;
  }
  uint32_t* words = reinterpret_cast<uint32_t*>(scratch);
  int32_t* chunk = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(scratch) + wb);
  // values of depth d (d0 <= d <= dmid) at vals[d]
  cd* vals[64] = {nullptr};
  if (vb) {
    char* v = reinterpret_cast<char*>(scratch) + wb + cb;
    for (int d = dmid; d >= d0; --d) {
      vals[d] = reinterpret_cast<cd*>(v);
      v += (size_t)16 << d;
    }
  }
  // layer j = depth d0 + j; fused depths dtop + t, t = 4..8
  DeepFuse f;
  memset(&f, 0, sizeof(f));
  f.words = words;
  f.t_lo = std::max(4, d0 - dtop);
  for (int t = 0; t <= 8; ++t) {
    const int j = dtop + t - d0;
    f.word_off[t] = j >= 0 ? D.word_off[j] : 0;
    f.thr[t] = j >= 0 ? D.thr[j] : 0.0;
    f.t2hi[t] = j >= 0 ? D.t2hi[j] : 0.0;
    f.t2lo[t] = j >= 0 ? D.t2lo[j] : 0.0;
  }
  f.vmid = d0 < dmid ? vals[dmid] : nullptr;
  f.norm2 = norm2;
  if (norm2) {
    const cudaError_t e = cudaMemsetAsync(norm2, 0, 8, st);
    if (e != cudaSuccess) return cuda_status(e, "full_active_all_fused norm");
  }
  int rc = spectrum_fused(x, dtype, n, Yout, f, st);
  if (rc) return rc;
  const int lv = dmid - d0;
  static const bool one_launch = [] {
    const char* e = getenv("AFFT_TREE_FUSE");
    return !(e && atoi(e) == 0);
  }();
  if (one_launch && lv >= 3 && lv <= 8) {
    TreeLevels T;
    memset(&T, 0, sizeof(T));
    T.vin = vals[dmid];
    for (int l = 0; l < lv; ++l) {
      const int d = dmid - 1 - l;
      T.vout[l] = vals[d];
      T.words[l] = words + D.word_off[d - d0];
      T.thr[l] = thr[d - d0];
    }
    const unsigned grid = (unsigned)((int64_t(1) << d0) / 32);
    switch (lv) {
      case 3: tree_levels_kernel<0><<<grid, 256, 0, st>>>(T, d0); break;
      case 4: tree_levels_kernel<1><<<grid, 256, 0, st>>>(T, d0); break;
      case 5: tree_levels_kernel<2><<<grid, 256, 0, st>>>(T, d0); break;
      case 6: tree_levels_kernel<3><<<grid, 256, 0, st>>>(T, d0); break;
      case 7: tree_levels_kernel<4><<<grid, 256, 0, st>>>(T, d0); break;
      default: tree_levels_kernel<5><<<grid, 256, 0, st>>>(T, d0); break;
    }
    AFFT_CHECK_LAUNCH("tree_levels_kernel");
  } else {
    for (int d = dmid - 1; d >= d0; --d) {  // v_d[i] = v_{d+1}[i] + v_{d+1}[i + 2^d]
      const int64_t b = int64_t(1) << d;
      tree_level_kernel<<<(unsigned)((b + 255) / 256), 256, 0, st>>>(
          vals[d + 1], b, thr[d - d0], vals[d], words + D.word_off[d - d0]);
    }
    AFFT_CHECK_LAUNCH("tree_level_kernel");
  }
  const unsigned chunks = (unsigned)D.chunk_off[nl];
  deep_count_kernel<<<chunks, 256, 0, st>>>(words, D, chunk);
  deep_scan_kernel<<<1, 32 * kDeepMaxLayers, 0, st>>>(chunk, D, counts);
  deep_write_kernel<<<chunks, 256, 0, st>>>(words, D, chunk, out, cap);
  AFFT_CHECK_LAUNCH("deep_write_kernel");
  return AFFT_OK;
}

size_t full_active_scratch(int64_t n, int d0, int nl) {
  DeepLayers D;
  int jd = 0;
  size_t wb = 0, cb = 0, vb = 0;
  full_layers_layout(n, d0, nl, &D, &jd, &wb, &cb, &vb);
  return wb + cb + vb;
}

// The deep layers alone (b = bmin .. n, all with n/b <= 32).
int deep_active_all(const double* spectrum, int64_t n, int64_t bmin, int nl, const double* thr,
                    int64_t* out, int cap, int32_t* counts, void* scratch, size_t scratch_bytes,
                    cudaStream_t st) {
  int d0 = 0;
  while ((int64_t(1) << d0) < bmin) ++d0;
  if ((int64_t(1) << d0) != bmin || n / bmin > kAliasMaxL) {
    set_error("deep_active_all: unsupported layers (n=%lld, bmin=%lld)", (long long)n,
              (long long)bmin);
    return AFFT_EUNSUPPORTED;
  }
  return full_active_all(spectrum, n, d0, nl, thr, out, cap, counts, scratch, scratch_bytes, st);
}

size_t deep_active_scratch(int64_t n, int64_t bmin, int nl) {
  int d0 = 0;
  while ((int64_t(1) << d0) < bmin) ++d0;
  return full_active_scratch(n, d0, nl);
}

}  // namespace afft

using namespace afft;

extern "C" int afft_bucketize_rows(const void* x, int dtype, int64_t n, int64_t b,
                                   const int64_t* shifts, int32_t nshift,
                                   const int64_t* bucket_idx, int64_t nrows, double* rows,
                                   double* energy, void* stream) {
  if (nshift == 0) return AFFT_OK;
  if (!x || !shifts || (nrows > 0 && (!bucket_idx || !rows)) || b < 1 || n % b ||
      nshift < 0 || nshift > AFFT_MAX_SHIFTS) {
    set_error("afft_bucketize_rows: bad arguments");
    return AFFT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t L = n / b;
  RowsParams p;
  memset(&p, 0, sizeof(p));
  p.b = b;
  p.nshift = nshift;
  p.nrows = nrows;
  std::map<int64_t, int> seen;
  std::vector<int64_t> residues;
  std::vector<int32_t> mult;
  for (int t = 0; t < nshift; ++t) {
    const int64_t tm = host_pymod(shifts[t], n);
    const int64_t r = tm % L, q = tm / L;
    auto it = seen.find(r);
    int u;
    if (it == seen.end()) {
      u = (int)residues.size();
      seen[r] = u;
      residues.push_back(r);
      mult.push_back(0);
    } else {
      u = it->second;
    }
    ++mult[u];
    p.coset[t] = u;
    p.q[t] = q;
  }
  const int U = (int)residues.size();
  cd* Y = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&Y), (size_t)U * b * 16, st);
  if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(coset DFTs)");
  int rc = afft_bucketize(x, dtype, n, 1, n, b, residues.data(), U,
                          reinterpret_cast<double*>(Y), (int64_t)U * b, b, 1, stream);
  if (!rc && nrows > 0) {
    const int64_t tot = nrows * nshift;
    rows_gather_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        p, Y, bucket_idx, reinterpret_cast<cd*>(rows));
    if (cudaGetLastError() != cudaSuccess) rc = cuda_status(cudaErrorLaunchFailure, "rows_gather");
  }
  if (!rc && energy) {
    Mult mm;
    for (int u = 0; u < U; ++u) mm.m[u] = mult[u];
    coset_energy_kernel<<<(unsigned)((b + 255) / 256), 256, 0, st>>>(b, U, mm, Y, energy);
  }
  scratch_free(Y, st);
  if (!rc) AFFT_CHECK_LAUNCH("afft_bucketize_rows");
  return rc;
}

extern "C" int afft_active_indices(const double* values, int64_t b, double thr,
                                   const int64_t* map, int64_t* out_idx, int32_t* out_count,
                                   void* stream) {
  if (!values || !out_idx || !out_count || b < 1) {
    set_error("afft_active_indices: bad arguments");
    return AFFT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int nblocks = (int)((b + kCompactThreads - 1) / kCompactThreads);
  int32_t* counts = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&counts), (size_t)nblocks * 4, st);
  if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(compaction)");
  const cd* v = reinterpret_cast<const cd*>(values);
  active_count_kernel<<<nblocks, kCompactThreads, 0, st>>>(b, v, thr, counts);
  scan_counts_kernel<<<1, 1024, 0, st>>>(nblocks, counts, out_count);
  active_write_kernel<<<nblocks, kCompactThreads, 0, st>>>(b, v, thr, counts, map, out_idx);
  scratch_free(counts, st);
  AFFT_CHECK_LAUNCH("afft_active_indices");
  return AFFT_OK;
}

extern "C" int afft_selective_sums(const void* x, int dtype, int64_t n, int64_t b,
                                   const int64_t* cand, int64_t ncand, double* out,
                                   void* stream) {
  if (ncand == 0) return AFFT_OK;
  if (!x || !cand || !out || b < 1 || n % b || ncand < 0 || ncand > INT32_MAX) {
    set_error("afft_selective_sums: bad arguments");
    return AFFT_EINVAL;
  }
  selective_sum_kernel<<<(unsigned)ncand, 256, 0, (cudaStream_t)stream>>>(x, dtype, n, b, cand,
                                                                          out);
  AFFT_CHECK_LAUNCH("selective_sum_kernel");
  return AFFT_OK;
}

extern "C" int afft_alias_rows(const double* spectrum, int64_t n, int64_t b,
                               const int64_t* shifts, int32_t nshift, const int64_t* bucket_idx,
                               int64_t nrows, double* rows, double* energy, double* values0,
                               void* stream) {
  if (!spectrum || b < 1 || n % b || nshift < 0 || nshift > AFFT_MAX_SHIFTS ||
      (nrows > 0 && (!bucket_idx || !rows || !shifts))) {
    set_error("afft_alias_rows: bad arguments");
    return AFFT_EINVAL;
  }
  const int64_t L = n / b;
  const bool pow2L = (L & (L - 1)) == 0;
  if ((L > kAliasRowsMaxL && !(pow2L && !energy && !values0 && L <= kAliasCtaMaxL)) ||
      ((energy || values0) && L > kAliasMaxL)) {
    set_error("afft_alias_rows: n/b = %lld above %d (rows) / %d (energies, values)",
              (long long)L, kAliasRowsMaxL, kAliasMaxL);
    return AFFT_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const cd* Y = reinterpret_cast<const cd*>(spectrum);
  if (nrows > 0 && nshift > 0) {
    AliasShifts sh;
    sh.nshift = nshift;
    for (int t = 0; t < nshift; ++t) sh.tau[t] = host_pymod(shifts[t], n);
    if (L > kAliasRowsMaxL) {  // one CTA per row, 2.5 L entries of shared memory
      const bool tabled = true;  // L <= kAliasCtaMaxL: the root table fits beside the buffers
      const size_t smem = (size_t)(tabled ? 2 * L + L / 2 : 2 * L) * sizeof(cd);
      cudaError_t e = ensure_smem((const void*)alias_rows_cta_kernel, smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(alias_rows_cta)");
      alias_rows_cta_kernel<<<(unsigned)nrows, 256, smem, st>>>(
          Y, n, b, (int)L, sh, bucket_idx, nrows, reinterpret_cast<cd*>(rows), tabled);
    } else {
      const size_t smem = (size_t)(1 + 2 * kAliasWarps) * L * sizeof(cd);
      cudaError_t e = ensure_smem((const void*)alias_rows_kernel, smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(alias_rows)");
      alias_rows_kernel<<<(unsigned)((nrows + kAliasWarps - 1) / kAliasWarps),
                          kAliasWarps * 32, smem, st>>>(Y, n, b, (int)L, sh, bucket_idx, nrows,
                                                        reinterpret_cast<cd*>(rows));
    }
  }
  if (energy || values0) {
    AliasCosets cs;
    memset(&cs, 0, sizeof(cs));
    for (int t = 0; t < nshift && energy; ++t) {
      const int r = (int)(host_pymod(shifts[t], n) % L);
      int u = 0;
      while (u < cs.U && cs.r[u] != r) ++u;
      if (u == cs.U) {
        cs.r[cs.U] = r;
        cs.mult[cs.U++] = 0;
      }
      ++cs.mult[u];
    }
    const unsigned grid = (unsigned)((b + 255) / 256);
    cd* v0 = reinterpret_cast<cd*>(values0);
    if (L <= 2)
      alias_all_kernel<2><<<grid, 256, 0, st>>>(Y, b, (int)L, cs, energy, v0);
    else if (L <= 4)
      alias_all_kernel<4><<<grid, 256, 0, st>>>(Y, b, (int)L, cs, energy, v0);
    else if (L <= 8)
      alias_all_kernel<8><<<grid, 256, 0, st>>>(Y, b, (int)L, cs, energy, v0);
    else if (L <= 16)
      alias_all_kernel<16><<<grid, 256, 0, st>>>(Y, b, (int)L, cs, energy, v0);
    else
      alias_all_kernel<kAliasMaxL><<<grid, 256, 0, st>>>(Y, b, (int)L, cs, energy, v0);
  }
  AFFT_CHECK_LAUNCH("afft_alias_rows");
  return AFFT_OK;
}
