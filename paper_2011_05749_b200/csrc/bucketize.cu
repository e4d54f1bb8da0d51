// K1+K2: strided, delay-shifted gather + batched size-b DFT (bucketize.py:83-106,
// and build_graph's loop over cycles, peeling.py:169-178).
//
// One CTA per (signal, cycle, chunk of shifts).  The CTA gathers
// x[(j*(n/b) - tau) mod n] for its shifts straight into shared memory (the
// reference's index map, bucketize.py:96, with tau reduced mod n on the host so
// negative structured shifts work), runs the in-smem Stockham DFT and writes
// values * (1/b) — numpy's complex/int division is a multiply by the
// reciprocal — to a caller-strided output, so the same kernel produces the
// FilteredSpectrum layout [s][t][i] and the peeling-node layout [s][g][t].
#include <algorithm>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "afft_common.cuh"
#include "gather_dft.cuh"

namespace afft {

struct GatherDftParams {
  const void* x;
  int dtype;
  int64_t n, ld;
  int ncycles;
  int nshift;
  int64_t b[AFFT_MAX_CYCLES];
  int32_t chunk[AFFT_MAX_CYCLES];  // shifts per CTA for each cycle
  int32_t jobs[AFFT_MAX_CYCLES];   // CTAs per signal for each cycle
  int64_t out_offset[AFFT_MAX_CYCLES];
  DftPlan plan[AFFT_MAX_CYCLES];
  double* out;
  int64_t out_signal_stride, out_shift_stride, out_bin_stride;  // complex elements
  const int64_t* shift_table;    // optional device [batch][nshift] raw per-signal shifts
  int64_t tau[AFFT_MAX_SHIFTS];  // shifts reduced into [0, n)
};

__global__ void __launch_bounds__(256) gather_dft_kernel(const __grid_constant__ GatherDftParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t s = blockIdx.x;
  int job = blockIdx.y;
  int c = 0;
  while (job >= p.jobs[c]) {
    job -= p.jobs[c];
    ++c;
  }
  const int64_t b = p.b[c];
  const int t0 = job * p.chunk[c];
  const int cnt = min(p.chunk[c], p.nshift - t0);
  __shared__ int64_t s_tau[AFFT_MAX_SHIFTS];
  cd* tw = reinterpret_cast<cd*>(smem_raw);
  cd* bufA = tw + b;
  cd* bufB = bufA + (size_t)cnt * b;
  const char* xs = reinterpret_cast<const char*>(p.x) +
                   s * p.ld * (p.dtype == AFFT_C64 ? 8 : 16);
  const int64_t* taus = p.tau + t0;
  if (p.shift_table) {  // per-signal shifts (sFFT-DT random shifts), reduced here
    for (int t = threadIdx.x; t < cnt; t += blockDim.x)
      s_tau[t] = pymod(p.shift_table[s * p.nshift + t0 + t], p.n);
    __syncthreads();
    taus = s_tau;
  }
  const cd* res =
      gather_dft_block<16>(xs, p.dtype, p.n, b, p.plan[c], taus, cnt, tw, bufA, bufB);
  const double inv_b = 1.0 / (double)b;
  double* out = p.out + 2 * (s * p.out_signal_stride + p.out_offset[c]);
  const int total = cnt * (int)b;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int t = e / (int)b;
    const int64_t i = e - (int64_t)t * b;
    const cd v = cscale(res[e], inv_b);
    const int64_t o = 2 * ((t0 + t) * p.out_shift_stride + i * p.out_bin_stride);
    out[o] = v.re;
    out[o + 1] = v.im;
  }
}

// ---------------------------------------------------------------- K2': b > 4096
//
// Large bucket counts (DSFFT's deep layers up to b = 2^24, R-FFAST's auto plans,
// the dense full-length transform): global-memory Stockham passes.  b is split
// into radices R_1 >= R_2 >= ... (each <= 256 unless a prime factor is larger),
// and pass s computes, for every butterfly j < b/R_s with k = j mod N_s
// (N_s = R_1 ... R_{s-1}):
//   v[r] = in[j + r b/R_s] * w_b^(k r b/(N_s R_s)),  V = DFT_{R_s}(v),
//   out[(j / N_s) N_s R_s + k + q N_s] = V[q]
// — the smem Stockham of smem_dft.cuh run over HBM, so the result lands in natural
// order.  A CTA takes `cnt` consecutive butterflies (cnt * R_s ~ 2048 points):
// every row r it loads is cnt contiguous elements and every output row q is cnt
// contiguous elements, so all global traffic is coalesced; each pass reads and
// writes the data once.  The first pass gathers x[(e L - tau) mod n] directly
// (bucketize.py:96) and the last applies numpy's 1/b and the caller's strides.
// Twiddles w_b^m come from two 4096-entry tables (w_b^(4096 q) * w_b^(m mod 4096)).
struct GStockParams {
  const void* x;
  int dtype;
  int64_t n, ld, L, b;
  int64_t batch;
  int nshift;
  const int64_t* shift_table;
  const cd* tlo;
  const cd* thi;
  const cd* in;   // previous pass (null on the first pass)
  cd* tmp;        // this pass's output (null on the last pass)
  double* out;
  int64_t out_offset, out_signal_stride, out_shift_stride, out_bin_stride;
  int R;
  int64_t Ns;
  int cnt;
  int perm;       // gfft_reg_kernel: tile -> chunk order (0 identity, 1 odd multiplier, 2 stride)
  DftPlan plan;
  int64_t tau[AFFT_MAX_SHIFTS];
};

constexpr int kTwLoBits = 12;
constexpr int kGStockThreads = 256;
constexpr int kGStockPoints = 2048;  // points per tile (cnt * R)

__global__ void twiddle_tables_kernel(int64_t b, cd* __restrict__ tlo, int nlo,
                                      cd* __restrict__ thi, int nhi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double sn, cs;
  if (i < nlo) {
    sincospi(-2.0 * (double)i / (double)b, &sn, &cs);
    tlo[i] = cd{cs, sn};
  }
  if (i < nhi) {
    const int64_t k = (int64_t)i << kTwLoBits;
    sincospi(-2.0 * (double)k / (double)b, &sn, &cs);
    thi[i] = cd{cs, sn};
  }
}

// Twiddle tables of size b (w_b^m split as w_b^(m & 4095) * w_b^(m >> 12 << 12)),
// built once per (device, b) and kept: the K2' passes of DSFFT's layers and config
// 3''s cycles reuse the same few sizes on every call.  Built on the caller's stream,
// which is then synchronised once so that any stream may read them afterwards.
static const cd* twiddle_tables_for(int dev, int64_t b, int nlo, int nhi, cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, cd*> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, b});
  if (it != cache.end()) return it->second;
  cd* t = nullptr;
  if (cudaMalloc(&t, (size_t)(nlo + nhi) * sizeof(cd)) != cudaSuccess) {
    set_error("twiddle tables: cudaMalloc failed");
    return nullptr;
  }
  twiddle_tables_kernel<<<(unsigned)((std::max(nlo, nhi) + 255) / 256), 256, 0, stream>>>(
      b, t, nlo, t + nlo, nhi);
  const cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    cuda_status(e, "twiddle tables");
    cudaFree(t);
    return nullptr;
  }
  cache.emplace(std::make_pair(dev, b), t);
  return t;
}

__device__ __forceinline__ cd tw_b(const cd* tlo, const cd* thi, int64_t m) {
  const cd lo = tlo[m & ((1 << kTwLoBits) - 1)];
  return (m >> kTwLoBits) ? cmul(thi[m >> kTwLoBits], lo) : lo;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// Sequence stride of the staged tiles: R odd -> R, even -> R + 1 (column-wise transposes
// hit distinct banks), except when R has an odd prime factor p >= 11 with fewer than 8
// butterflies per sequence in that stage (nbp = R / p): then ld = nbp (mod 8), so the
// symmetric stage's lanes (consecutive butterflies (seq, j), address seq ld + j + r nbp)
// read 8 distinct 16-byte bank groups per quarter warp.
__host__ __device__ inline int gstock_ld(int R) {
  int m = R, big = 1;
  for (int q = 2; q * q <= m; ++q)
    while (m % q == 0) {
      if (q > big) big = q;
      m /= q;
    }
  if (m > big) big = m;
  const int nbp = R / big;
  if (big >= 11 && (big & 1) && nbp < 8) return R + (((nbp - R) % 8) + 8) % 8;
  return (R & 1) ? R : R + 1;
}


// One pass.  The tile's rows arrive by cp.async into a staging copy (every request
// in flight at once, no registers held), a second smem pass applies the inter-pass
// twiddles while transposing into sequences of stride ld = R + 1 (bank-conflict
// free column access), the smem Stockham runs on that stride, and the output rows
// leave coalesced.
// LGR >= 0: R = 2^LGR and cnt = kGStockPoints / R fixed at compile time (every tile
// full), so index splits are shifts, loops have constant trip counts and the DFT
// stages are dft_fixed — the runtime-shaped variant (LGR = -1) spent ~80% of its
// instructions on integer index math and control flow (ncu SASS mix).
#ifndef AFFT_GSTOCK_RT_CTAS
#define AFFT_GSTOCK_RT_CTAS 3
#endif
template <int LGR>
__global__ void __launch_bounds__(kGStockThreads, LGR < 0 ? AFFT_GSTOCK_RT_CTAS : 3) gstockham_kernel(
    const __grid_constant__ GStockParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool kFixed = LGR >= 0;
  constexpr int kR = kFixed ? (1 << LGR) : 1;
  constexpr int kCnt = kFixed ? kGStockPoints / kR : 1;
  constexpr int kLgCnt = kFixed ? 11 - LGR : 0;  // kGStockPoints = 2^11
  const int R = kFixed ? kR : p.R, cnt = kFixed ? kCnt : p.cnt;
  const int ld = kFixed ? ((R & 1) ? R : R + 1) : gstock_ld(R);
  const int tid = threadIdx.x, nt = blockDim.x;
  cd* tw = reinterpret_cast<cd*>(smem_raw);
  cd* bufA = tw + R;
  cd* bufB = bufA + (size_t)cnt * ld;
  build_twiddles(tw, R, tid, nt);
  const int64_t nb = p.b / R;
  const int64_t nchunks = (nb + cnt - 1) / cnt;
  const int64_t ntiles = p.batch * p.nshift * nchunks;
  const int64_t tstep = p.b / (p.Ns * R);
  const int64_t esz = p.dtype == AFFT_C64 ? 8 : 16;
  const bool first = p.in == nullptr;
  const bool c64 = first && p.dtype == AFFT_C64;
  const double inv_b = 1.0 / (double)p.b;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t chunk = tile % nchunks;
    const int64_t st_ = tile / nchunks;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t j0 = chunk * cnt;
    const int c = kFixed ? kCnt : (int)min((int64_t)cnt, nb - j0);
    const int64_t seq = s * p.nshift + t;
    const char* xs = reinterpret_cast<const char*>(p.x) + s * p.ld * esz;
    const int64_t tau = first ? (p.shift_table ? pymod(p.shift_table[s * p.nshift + t], p.n)
                                               : p.tau[t])
                              : 0;
    const int total = kFixed ? kGStockPoints : c * R;
    // e / c and e / R by multiply-high (e < 2^13, divisors < 2^13: exact)
    const unsigned Mc = c > 1 ? (unsigned)((0xffffffffull + c) / c) : 0u;
    const unsigned MR = (unsigned)((0xffffffffull + R) / R);
    // k = (j0 + jj) mod N_s for jj < c, from one 64-bit reduction per tile
    const int64_t k0 = p.Ns > 1 ? j0 % p.Ns : 0;
    __syncthreads();  // twiddles ready / previous tile's buffers consumed
    // 1. rows r = 0..R-1, each c contiguous butterflies, into staging (bufB) in
    //    arrival order e = r * c + jj
    for (int e = tid; e < total; e += nt) {
      const int r = kFixed ? e >> kLgCnt : (c > 1 ? (int)__umulhi((unsigned)e, Mc) : e);
      const int64_t src = j0 + (e - r * c) + r * nb;
      if (first) {
        int64_t idx = src * p.L - tau;
        if (idx < 0) idx += p.n;
        if (c64)
          cp_async8(reinterpret_cast<float2*>(bufB) + e, xs + idx * 8);
        else
          cp_async16(bufB + e, xs + idx * 16);
      } else {
        cp_async16(bufB + e, p.in + seq * p.b + src);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // 2. twiddle w_b^(k r b/(N_s R)) and transpose into sequences of stride ld
#pragma unroll 4
    for (int e = tid; e < total; e += nt) {
      const int r = kFixed ? e >> kLgCnt : (c > 1 ? (int)__umulhi((unsigned)e, Mc) : e);
      const int jj = e - r * c;
      cd a;
      if (c64) {
        const float2 f = reinterpret_cast<const float2*>(bufB)[e];
        a = cd{(double)f.x, (double)f.y};
      } else {
        a = bufB[e];
      }
      if (p.Ns > 1 && r) {
        int64_t k = k0 + jj;
        while (k >= p.Ns) k -= p.Ns;
        if (k) a = cmul(a, tw_b(p.tlo, p.thi, k * r * tstep));
      }
      bufA[jj * ld + r] = a;
    }
    __syncthreads();
    const cd* spec;
    if constexpr (kFixed)
      spec = dft_fixed<(LGR > 0 ? LGR : 1), 0, kCnt, kGStockThreads>(bufA, bufB, tw, ld);
    else
      spec = smem_dft(bufA, bufB, c, p.plan, tw, tid, nt, ld);
    double* out = p.out ? p.out + 2 * (s * p.out_signal_stride + p.out_offset +
                                       t * p.out_shift_stride)
                        : nullptr;
    cd* tmp = p.tmp ? p.tmp + seq * p.b : nullptr;
    // 3. outputs: butterfly j's V[q] goes to (j / N_s) N_s R + k + q N_s
    for (int e = tid; e < total; e += nt) {
      int jj, q;
      if (p.Ns == 1) {  // first pass: butterfly j's outputs are the contiguous j*R + q
        jj = kFixed ? e >> LGR : (int)__umulhi((unsigned)e, MR);
        q = e - jj * R;
      } else {          // output row q: c contiguous k
        q = kFixed ? e >> kLgCnt : (c > 1 ? (int)__umulhi((unsigned)e, Mc) : e);
        jj = e - q * c;
      }
      const int64_t j = j0 + jj;
      int64_t k = 0;
      if (p.Ns > 1) {
        k = k0 + jj;
        while (k >= p.Ns) k -= p.Ns;
      }
      const int64_t dst = (j - k) * R + k + q * p.Ns;
      const cd v = spec[jj * ld + q];
      if (tmp) {
        tmp[dst] = v;
      } else {
        const cd w = cscale(v, inv_b);
        const int64_t o = 2 * dst * p.out_bin_stride;
        out[o] = w.re;
        out[o + 1] = w.im;
      }
    }
  }
}

// Power-of-two radix R = A * B (A = 2^LA, B = 2^LB <= 16) with the DFT in registers:
// the same pass as gstockham_kernel (same tile of kCnt = 2048 / R butterflies, same
// input rows and output placement), restructured so that each point crosses shared
// memory once instead of ~5 times and the inter-pass twiddles come from two table
// reads per sub-sequence instead of one or two scattered reads per point (the smem
// Stockham version saturated the L1 data pipe with bank conflicts and twiddle
// gathers at 17% of HBM bandwidth, profiles/r01_k2_ncu.md).
//   r = n1 + A n2,  q = qb + B qa:
//   stage A, item (jj, n1): v[n2] = in[row r] * w_b^(k r tstep); DFT_B over n2;
//                           U[jj][n1][qb] = w_R^(n1 qb) * that  (smem, stride R + 1)
//   stage B, item (jj, qb): V[qb + B qa] = DFT_A over n1 of U[jj][n1][qb]  -> HBM
// Global loads go straight to registers (all 16 per thread issued before use);
// lanes run along jj so every row segment (kCnt contiguous points, >= 128 B) is
// one coalesced request; the first pass (N_s = 1, outputs of a butterfly are
// contiguous) runs stage B along qb instead.
constexpr int kGfftThreads = 128;

// DeepFuse epilogue of the last radix-256 pass (N_s = n/256, 8 alias classes j0 + jj per
// tile, thread (jj = tid & 7, qb = tid >> 3) holding y[qa] = Y[j + (qb + 16 qa) N_s]).
// Depth dtop + t (dtop = log2 n - 8) has 2^t buckets r over each j, with values in the
// tree order of dsfft.cu tree_sum: v_8(r) = Y[j + r N_s], v_t(r) = v_{t+1}(r) +
// v_{t+1}(r + 2^t).  For t >= 4, r = qb + 16 m and r + 2^t is the same thread's
// m + 2^(t-4): every level from 8 down to 4 is computed in registers, in place, with no
// shared memory and no barrier (the levels below, whose children sit in other threads,
// come from the depth-(dtop + 4) values by tree_level_kernel, which adds in the same
// order).  Every decision is bit-identical to deep_flags_kernel's.  A tile owns 8
// consecutive bits (j0 % 8 == 0) of every bitmap: whole bytes, no atomics; a warp's
// ballot holds 4 of them (lanes jj + 8 (qb & 3)).
__device__ __forceinline__ void deep_fuse_epilogue(cd (&y)[16], int tid, int64_t j0, int dtop,
                                                   const DeepFuse& f) {
  const int jj = tid & 7, qb = tid >> 3, lane = tid & 31;
  uint8_t* wb = reinterpret_cast<uint8_t*>(f.words);
  const int64_t byte0 = j0 >> 3, rstride = int64_t(1) << (dtop - 3);
  auto level = [&](auto tc) {  // compile-time M (a runtime bound left y[] in local memory)
    constexpr int t = decltype(tc)::value, M = 1 << (t - 4);
    if (t < 8) {
#pragma unroll
      for (int m = 0; m < M; ++m) y[m] = cadd(y[m], y[m + M]);
    }
    if (t < f.t_lo) return;  // warp-uniform: shallower layers may not be asked for
    // |v| > thr_t: |v|^2 against the guard band (within an ulp either way; the band is
    // 1e-14 wide), hypot only inside it (deep_flags_kernel) — those rare values after
    // the cheap tests of the whole level, behind one warp-uniform branch
    bool fl[M];
    unsigned unsure = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double sq = __fma_rn(y[m].re, y[m].re, y[m].im * y[m].im);
      fl[m] = sq > f.t2hi[t];
      if (!fl[m] && !(sq < f.t2lo[t])) unsure |= 1u << m;
    }
    if (__any_sync(0xffffffffu, unsure != 0)) {
#pragma unroll
      for (int m = 0; m < M; ++m)
        if ((unsure >> m) & 1u) fl[m] = cabs_(y[m]) > f.thr[t];
    }
    uint8_t* row = wb + f.word_off[t] * 4 + byte0 + (int64_t)qb * rstride;
#pragma unroll
    for (int m = 0; m < M; ++m) {  // bucket r = qb + 16 m
      const unsigned bal = __ballot_sync(0xffffffffu, fl[m]);
      if ((lane & 7) == 0) row[(int64_t)(16 * m) * rstride] = (uint8_t)(bal >> (lane & 24));
    }
  };
  level(std::integral_constant<int, 8>{});
  level(std::integral_constant<int, 7>{});
  level(std::integral_constant<int, 6>{});
  level(std::integral_constant<int, 5>{});
  level(std::integral_constant<int, 4>{});
  // depth dtop + 4, bucket i = j + qb N_s: 8 consecutive j per qb, 128-byte runs
  if (f.vmid) f.vmid[j0 + jj + ((int64_t)qb << dtop)] = y[0];
}

// PARTIAL: nb = b / R need not be a multiple of kCnt; the last chunk of a sequence loads
// zeros for its missing columns and stores nothing for them (a separate instantiation:
// predicating the full-chunk form's loads cost it its batched issue, 2^24 c64 0.38 ->
// 0.53 ms).
template <int LA, int LB, bool FUSE, bool PARTIAL = false>
__device__ __forceinline__ void gfft_reg_body(const GStockParams& p, const DeepFuse& f) {
  constexpr int A = 1 << LA, B = 1 << LB, LGR = LA + LB, R = A * B;
  constexpr int kCnt = kGStockPoints / R, kLgCnt = 11 - LGR;
  constexpr int LD = R + 1;
  constexpr int IA = kCnt * A / kGfftThreads;  // stage-A items per thread
  constexpr int IB = kCnt * B / kGfftThreads;  // stage-B items per thread
  static_assert(IA * kGfftThreads == kCnt * A && IB * kGfftThreads == kCnt * B, "tile shape");
  static_assert(IA * B == 16 && IB * A == 16, "16 points per thread per stage");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cd* twR = reinterpret_cast<cd*>(smem_raw);
  cd* U = twR + R;
  const int tid = threadIdx.x;
  build_twiddles(twR, R, tid, kGfftThreads);
  const int64_t nb = p.b / R;
  const int64_t nchunks = PARTIAL ? (nb + kCnt - 1) >> kLgCnt : nb >> kLgCnt;
  const int64_t ntiles = p.batch * p.nshift * nchunks;
  const int64_t tstep = p.b / (p.Ns * R);
  const bool pow2ns = (p.Ns & (p.Ns - 1)) == 0;  // N_s = product of earlier radices
  const bool first = p.in == nullptr;
  const bool c64 = first && p.dtype == AFFT_C64;
  const int64_t esz = p.dtype == AFFT_C64 ? 8 : 16;
  const double inv_b = 1.0 / (double)p.b;
  double fsq = 0.0;  // FUSE: this thread's sum |Y|^2 over its tiles
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int64_t chunk = tile % nchunks;
    if (p.perm == 1)  // nchunks a power of two: an odd multiplier is a bijection
      chunk = (chunk * 0x9E3779B1LL) & (nchunks - 1);
    else if (p.perm == 2 && nchunks >= 4096 && (nchunks & 63) == 0)
      chunk = (chunk & 63) * (nchunks >> 6) + (chunk >> 6);
    const int64_t st_ = tile / nchunks;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t j0 = chunk << kLgCnt;
    const int valid = PARTIAL ? (int)(nb - j0 < kCnt ? nb - j0 : kCnt) : kCnt;
    const int64_t k0 = pow2ns ? (j0 & (p.Ns - 1)) : j0 % p.Ns;
    // k = (j0 + jj) mod N_s
    auto kmod = [&](int jj) -> int64_t {
      if (pow2ns) return (j0 + jj) & (p.Ns - 1);
      int64_t k = k0 + jj;
      while (k >= p.Ns) k -= p.Ns;
      return k;
    };
    const int64_t seq = s * p.nshift + t;
    const char* xs = reinterpret_cast<const char*>(p.x) + s * p.ld * esz;
    const int64_t tau = first ? (p.shift_table ? pymod(p.shift_table[s * p.nshift + t], p.n)
                                               : p.tau[t])
                              : 0;
    // ---- stage A: loads (all issued first), twiddles, DFT_B, w_R, to smem
    // (one branch around whole unrolled loops: with the dtype test per load, each c64
    // load was converted right after issue and the 16 loads ran one latency apart)
    cd v[IA][B];
    if (c64) {
      float2 raw[IA][B];
#pragma unroll
      for (int i = 0; i < IA; ++i) {
        const int w = tid + i * kGfftThreads;
        const int jj = w & (kCnt - 1), n1 = w >> kLgCnt;
#pragma unroll
        for (int n2 = 0; n2 < B; ++n2) {
          int64_t idx = (j0 + jj + (int64_t)(n1 + A * n2) * nb) * p.L - tau;
          if (idx < 0) idx += p.n;
          raw[i][n2] = !PARTIAL || jj < valid
                           ? __ldg(reinterpret_cast<const float2*>(xs) + idx)
                           : make_float2(0.f, 0.f);
        }
      }
#pragma unroll
      for (int i = 0; i < IA; ++i)
#pragma unroll
        for (int n2 = 0; n2 < B; ++n2) v[i][n2] = cd{(double)raw[i][n2].x, (double)raw[i][n2].y};
    } else {
      const double2* base = first ? reinterpret_cast<const double2*>(xs)
                                  : reinterpret_cast<const double2*>(p.in + seq * p.b);
      const int64_t L = first ? p.L : 1;
      const int64_t off = first ? tau : 0;
      double2 raw[IA][B];
#pragma unroll
      for (int i = 0; i < IA; ++i) {
        const int w = tid + i * kGfftThreads;
        const int jj = w & (kCnt - 1), n1 = w >> kLgCnt;
#pragma unroll
        for (int n2 = 0; n2 < B; ++n2) {
          int64_t idx = (j0 + jj + (int64_t)(n1 + A * n2) * nb) * L - off;
          if (idx < 0) idx += p.n;
          raw[i][n2] = !PARTIAL || jj < valid ? __ldcs(base + idx) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < IA; ++i)
#pragma unroll
        for (int n2 = 0; n2 < B; ++n2) v[i][n2] = cd{raw[i][n2].x, raw[i][n2].y};
    }
    __syncthreads();  // the previous tile's stage B has finished reading U
#pragma unroll
    for (int i = 0; i < IA; ++i) {
      const int w = tid + i * kGfftThreads;
      const int jj = w & (kCnt - 1), n1 = w >> kLgCnt;
      if (p.Ns > 1) {
        // w_b^(k r tstep) for r = n1 + A n2: base w_b^(k n1 tstep), step w_b^(k A tstep)
        const int64_t kt = kmod(jj) * tstep;
        if (kt) {
          cd cur = tw_b(p.tlo, p.thi, kt * n1);
          const cd step = tw_b(p.tlo, p.thi, kt * A);
#pragma unroll
          for (int n2 = 0; n2 < B; ++n2) {
            if (n1 || n2) v[i][n2] = cmul(v[i][n2], cur);
            if (n2 + 1 < B) cur = cmul(cur, step);
          }
        }
      }
      dft_reg<B>(v[i]);
      cd* u = U + jj * LD + n1 * B;
#pragma unroll
      for (int qb = 0; qb < B; ++qb) u[qb] = (n1 && qb) ? cmul(v[i][qb], twR[n1 * qb]) : v[i][qb];
    }
    __syncthreads();
    // ---- stage B: DFT_A over n1, outputs q = qb + B qa
    double* out = p.out ? p.out + 2 * (s * p.out_signal_stride + p.out_offset +
                                       t * p.out_shift_stride)
                        : nullptr;
    cd* tmp = p.tmp ? p.tmp + seq * p.b : nullptr;
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      const int w = tid + i * kGfftThreads;
      int jj, qb;
      if (p.Ns == 1) {
        qb = w & (B - 1);
        jj = w >> LB;
      } else {
        jj = w & (kCnt - 1);
        qb = w >> kLgCnt;
      }
      cd a[A];
      const cd* u = U + jj * LD + qb;
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) a[n1] = u[n1 * B];
      dft_reg<A>(a);
      const int64_t j = j0 + jj;
      const int64_t k = kmod(jj);
      const int64_t base = (j - k) * R + k;
      if (PARTIAL && jj >= valid) continue;  // a partial chunk's missing column
#pragma unroll
      for (int qa = 0; qa < A; ++qa) {
        const int64_t dst = base + (int64_t)(qb + B * qa) * p.Ns;
        if (tmp) {
          __stcs(reinterpret_cast<double2*>(tmp + dst), make_double2(a[qa].re, a[qa].im));
        } else {  // complex128 output: 16-B aligned pairs
          const cd wv = cscale(a[qa], inv_b);
          *reinterpret_cast<double2*>(out + 2 * dst * p.out_bin_stride) = make_double2(wv.re, wv.im);
          if constexpr (FUSE) {
            a[qa] = wv;
            fsq += wv.re * wv.re + wv.im * wv.im;
          }
        }
      }
      if constexpr (FUSE) {
        static_assert(A == 16 && B == 16 && IB == 1, "fused epilogue: the radix-256 last pass");
        // dtop = log2(N_s): N_s = n / 256 on the last pass.  (Deferring it behind the next
        // tile's loads, to keep them in flight through it, spilled at 3 CTAs per SM and
        // ran at 2: 223 / 258 against 186 us.)
        deep_fuse_epilogue(a, tid, j0, 63 - __clzll((unsigned long long)p.Ns), f);
      }
    }
  }
  if constexpr (FUSE) {
    // sum |Y|^2 (only ever compared against a bound with a wide margin): one atomic
    // per warp of the persistent grid (one per warp per tile serialised on the address)
    if (f.norm2) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) fsq += __shfl_xor_sync(0xffffffffu, fsq, o);
      if ((tid & 31) == 0) atomicAdd(f.norm2, fsq);
    }
  }
}

template <int LA, int LB, bool PARTIAL = false>
__global__ void __launch_bounds__(kGfftThreads) gfft_reg_kernel(
    const __grid_constant__ GStockParams p) {
  gfft_reg_body<LA, LB, false, PARTIAL>(p, DeepFuse{});
}

// The last radix-256 pass of a DSFFT spectrum with the tree layers decided in its
// epilogue (DeepFuse, afft_common.cuh).
__global__ void __launch_bounds__(kGfftThreads, 3) gfft_flags_kernel(
    const __grid_constant__ GStockParams p, const __grid_constant__ DeepFuse f) {
  gfft_reg_body<4, 4, true>(p, f);
}

// ---- Radix-4096 register pass (opt-in, AFFT_FFT_4K=1; slower, see launch_fourstep):
// a 2^24-point transform in TWO passes (4096 x 4096) instead of three radix-256 ones —
// 0.9 instead of 1.4 GB of HBM traffic per c64 signal.  One column j per tile (kCnt = 1; the 8-16 B row pieces of neighbouring
// columns are fetched by the CTAs resident beside it and combine in L2), 256 threads x
// 16 points, the 4096-point DFT as 16 x 16 x 16 in registers with two shared-memory
// exchanges:
//   r = r0 + 16 r1 + 256 r2,  q = q0 + 16 q1 + 256 q2,
//   stage 1, thread (r0, r1): DFT_16 over r2 -> q0, times w_256^(r1 q0);
//   stage 2, thread (r0, q0): DFT_16 over r1 -> q1, times w_4096^(r0 (q0 + 16 q1));
//   stage 3, thread (q0, q1): DFT_16 over r0 -> q2; V[q] to (j - k) 4096 + k + q N_s.
// Shared layouts (16-B elements): stage 1 -> 2 at r0 + 16 r1 + 256 q0, stage 2 -> 3 at
// q0 + 17 r0 + 272 q1 (a quarter warp's lanes always hit 8 distinct 16-B bank groups).
// Internal twiddles w_4096^e = thi[e] (the b = 2^24 table's w_b^(4096 e), exact
// sincospi values).  With FUSE (the spectrum's last pass, N_s = 4096) thread (q0, q1)
// holds y[q2] = Y[J + (q1 + 16 q2) n/256], J = j + 4096 q0 < n/256: the alias classes
// deep_fuse_epilogue expects, bits set by atomicOr into zeroed bitmaps (consecutive J
// belong to different tiles).
constexpr int kG4Threads = 256;
constexpr int kG4Smem = 4352 * 16;

__device__ __forceinline__ void deep_fuse_epilogue_atomic(cd (&y)[16], int64_t J, int qb,
                                                          int dtop, const DeepFuse& f) {
  auto level = [&](auto tc) {
    constexpr int t = decltype(tc)::value, M = 1 << (t - 4);
    if (t < 8) {
#pragma unroll
      for (int m = 0; m < M; ++m) y[m] = cadd(y[m], y[m + M]);
    }
    if (t < f.t_lo) return;
    bool fl[M];
    unsigned unsure = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double sq = __fma_rn(y[m].re, y[m].re, y[m].im * y[m].im);
      fl[m] = sq > f.t2hi[t];
      if (!fl[m] && !(sq < f.t2lo[t])) unsure |= 1u << m;
    }
    if (unsure) {
#pragma unroll
      for (int m = 0; m < M; ++m)
        if ((unsure >> m) & 1u) fl[m] = cabs_(y[m]) > f.thr[t];
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {  // bucket r = qb + 16 m: bit J + r 2^dtop
      if (fl[m]) {
        const int64_t bit = J + ((int64_t)(qb + 16 * m) << dtop);
        atomicOr(f.words + f.word_off[t] + (bit >> 5), 1u << (bit & 31));
      }
    }
  };
  level(std::integral_constant<int, 8>{});
  level(std::integral_constant<int, 7>{});
  level(std::integral_constant<int, 6>{});
  level(std::integral_constant<int, 5>{});
  level(std::integral_constant<int, 4>{});
  if (f.vmid) f.vmid[J + ((int64_t)qb << dtop)] = y[0];
}

template <bool FUSE>
__device__ __forceinline__ void gfft4k_body(const GStockParams& p, const DeepFuse& f) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cd* S = reinterpret_cast<cd*>(smem_raw);
  const int tid = threadIdx.x, lo = tid & 15, hi = tid >> 4;
  const int64_t nb = p.b >> 12;
  const int64_t ntiles = p.batch * p.nshift * nb;
  const int64_t tstep = p.b / (p.Ns << 12);
  const bool first = p.in == nullptr;
  const bool c64 = first && p.dtype == AFFT_C64;
  const int64_t esz = p.dtype == AFFT_C64 ? 8 : 16;
  const double inv_b = 1.0 / (double)p.b;
  const cd* __restrict__ w4k = p.thi;  // w_4096^e, e < 4096
  double fsq = 0.0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t j = tile % nb, st_ = tile / nb;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t k = j % p.Ns;
    const int64_t seq = s * p.nshift + t;
    // ---- stage 1: rows r = lo + 16 hi + 256 m (all 16 loads issued first)
    cd v[16];
    if (first) {
      const char* xs = reinterpret_cast<const char*>(p.x) + s * p.ld * esz;
      const int64_t tau = p.shift_table ? pymod(p.shift_table[s * p.nshift + t], p.n) : p.tau[t];
      if (c64) {
        float2 raw[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          int64_t idx = (j + (int64_t)(lo + 16 * hi + 256 * m) * nb) * p.L - tau;
          if (idx < 0) idx += p.n;
          raw[m] = __ldg(reinterpret_cast<const float2*>(xs) + idx);
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = cd{(double)raw[m].x, (double)raw[m].y};
      } else {
        double2 raw[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          int64_t idx = (j + (int64_t)(lo + 16 * hi + 256 * m) * nb) * p.L - tau;
          if (idx < 0) idx += p.n;
          raw[m] = __ldcs(reinterpret_cast<const double2*>(xs) + idx);
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = cd{raw[m].x, raw[m].y};
      }
    } else {
      const double2* base = reinterpret_cast<const double2*>(p.in + seq * p.b);
      double2 raw[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) raw[m] = __ldcs(base + j + (int64_t)(lo + 16 * hi + 256 * m) * nb);
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = cd{raw[m].x, raw[m].y};
    }
    if (p.Ns > 1) {  // w_b^(k r tstep), r = lo + 16 hi + 256 m
      const int64_t kt = k * tstep;
      if (kt) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const int64_t r = lo + 16 * hi + 256 * m;
          if (r) v[m] = cmul(v[m], tw_b(p.tlo, p.thi, kt * r));
        }
      }
    }
    dft_reg<16>(v);
    __syncthreads();  // the previous tile's stage 3 has finished reading S
#pragma unroll
    for (int q0 = 0; q0 < 16; ++q0)
      S[lo + 16 * hi + 256 * q0] = (hi && q0) ? cmul(v[q0], w4k[16 * hi * q0]) : v[q0];
    __syncthreads();
    // ---- stage 2: thread (r0 = lo, q0 = hi)
#pragma unroll
    for (int r1 = 0; r1 < 16; ++r1) v[r1] = S[lo + 16 * r1 + 256 * hi];
    __syncthreads();  // S is rewritten below
    dft_reg<16>(v);
#pragma unroll
    for (int q1 = 0; q1 < 16; ++q1) {
      const int e = lo * (hi + 16 * q1);
      S[hi + 17 * lo + 272 * q1] = e ? cmul(v[q1], w4k[e]) : v[q1];
    }
    __syncthreads();
    // ---- stage 3: thread (q0 = lo, q1 = hi)
#pragma unroll
    for (int r0 = 0; r0 < 16; ++r0) v[r0] = S[lo + 17 * r0 + 272 * hi];
    dft_reg<16>(v);
    double* out = p.out ? p.out + 2 * (s * p.out_signal_stride + p.out_offset +
                                       t * p.out_shift_stride)
                        : nullptr;
    cd* tmp = p.tmp ? p.tmp + seq * p.b : nullptr;
    const int64_t base = (j - k) * 4096 + k;
#pragma unroll
    for (int q2 = 0; q2 < 16; ++q2) {
      const int64_t dst = base + (int64_t)(lo + 16 * hi + 256 * q2) * p.Ns;
      if (tmp) {
        __stcs(reinterpret_cast<double2*>(tmp + dst), make_double2(v[q2].re, v[q2].im));
      } else {
        const cd wv = cscale(v[q2], inv_b);
        *reinterpret_cast<double2*>(out + 2 * dst * p.out_bin_stride) = make_double2(wv.re, wv.im);
        if constexpr (FUSE) {
          v[q2] = wv;
          fsq += wv.re * wv.re + wv.im * wv.im;
        }
      }
    }
    if constexpr (FUSE) {
      // N_s = 4096 = n / 4096: Y[j + 4096 (q0 + 16 q1) + 2^20 q2], dtop = log2 n - 8
      const int dtop = 63 - __clzll((unsigned long long)p.b) - 8;
      deep_fuse_epilogue_atomic(v, j + ((int64_t)lo << 12), hi, dtop, f);
    }
  }
  if constexpr (FUSE) {
    if (f.norm2) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) fsq += __shfl_xor_sync(0xffffffffu, fsq, o);
      if ((tid & 31) == 0) atomicAdd(f.norm2, fsq);
    }
  }
}

__global__ void __launch_bounds__(kG4Threads, 2) gfft4k_kernel(const __grid_constant__ GStockParams p) {
  gfft4k_body<false>(p, DeepFuse{});
}
__global__ void __launch_bounds__(kG4Threads, 2) gfft4k_flags_kernel(
    const __grid_constant__ GStockParams p, const __grid_constant__ DeepFuse f) {
  gfft4k_body<true>(p, f);
}

// ---- the same pass with its row loads on the TMA engine (bulk async copies into a
// double-buffered shared-memory stage, completion on an mbarrier): a persistent CTA
// issues tile k+1's R row segments before computing tile k, so loads overlap the
// DFT work instead of alternating with it per CTA.  Used when every row segment is
// contiguous in memory: every pass after the first, and a first pass over a plain
// (L = 1, tau = 0) signal — the DSFFT spectrum and the dense transform.  Same
// arithmetic as gfft_reg_kernel (bit-identical outputs).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int LA, int LB>
__global__ void __launch_bounds__(kGfftThreads) gfft_tma_kernel(
    const __grid_constant__ GStockParams p, const __grid_constant__ CUtensorMap tmap,
    int use_tmap) {
  constexpr int A = 1 << LA, B = 1 << LB, LGR = LA + LB, R = A * B;
  constexpr int kCnt = kGStockPoints / R, kLgCnt = 11 - LGR;
  constexpr int LD = R + 1;
  constexpr int IA = kCnt * A / kGfftThreads;
  constexpr int IB = kCnt * B / kGfftThreads;
  static_assert(IA * B == 16 && IB * A == 16, "16 points per thread per stage");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const bool first = p.in == nullptr;
  const bool c64 = first && p.dtype == AFFT_C64;
  const int esz = c64 ? 8 : 16;
  const uint32_t seg = (uint32_t)(kCnt * esz);            // bytes per row segment
  const size_t stage_bytes = (size_t)R * kCnt * 16;          // sized for c128
  // TMA destinations must be 128-byte aligned: the dynamic region follows the static
  // one, so align by hand (the launch adds 128 bytes)
  unsigned char* sm0 = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  unsigned char* stage[2] = {sm0, sm0 + stage_bytes};
  cd* twR = reinterpret_cast<cd*>(sm0 + 2 * stage_bytes);
  cd* U = twR + R;
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  build_twiddles(twR, R, tid, kGfftThreads);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nb = p.b / R;
  const int64_t nchunks = nb >> kLgCnt;
  const int64_t ntiles = p.batch * p.nshift * nchunks;
  const int64_t tstep = p.b / (p.Ns * R);
  const bool pow2ns = (p.Ns & (p.Ns - 1)) == 0;
  const double inv_b = 1.0 / (double)p.b;
  const int64_t in_esz = first ? esz : 16;
  // row segments of one tile -> stage[buf]: warp 0's lanes issue R / 32 bulk copies each
  auto issue = [&](int64_t tile, int buf) {
    if (tid >= 32) return;
    const int64_t chunk = tile % nchunks;
    const int64_t st_ = tile / nchunks;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t seq = s * p.nshift + t;
    const char* base = first ? reinterpret_cast<const char*>(p.x) + s * p.ld * in_esz
                             : reinterpret_cast<const char*>(p.in + seq * p.b);
    const int64_t j0 = chunk << kLgCnt;
    // the previous reads of this buffer (generic proxy) before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (use_tmap) {  // one tensor request: box [1 seq][R rows][kCnt points]
      if (tid == 0) {
        mbar_arrive_expect_tx(&bar[buf], (uint32_t)R * seg);
        const int c0 = (int)(j0 * 2), c2 = (int)seq;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(stage[buf])),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(0), "r"(c2),
            "r"(smem_u32(&bar[buf]))
            : "memory");
      }
      return;
    }
    if (tid == 0) mbar_arrive_expect_tx(&bar[buf], (uint32_t)R * seg);
    __syncwarp();
    for (int r = tid; r < R; r += 32)
      bulk_load(stage[buf] + (size_t)r * seg, base + (j0 + (int64_t)r * nb) * in_esz, seg,
                &bar[buf]);
  };
  uint32_t phase[2] = {0u, 0u};
  int64_t tile = blockIdx.x;
  if (tile < ntiles) issue(tile, 0);
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) issue(next, buf ^ 1);  // its buffer was released at the end of it-1
    const int64_t chunk = tile % nchunks;
    const int64_t st_ = tile / nchunks;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t j0 = chunk << kLgCnt;
    const int64_t k0 = pow2ns ? (j0 & (p.Ns - 1)) : j0 % p.Ns;
    auto kmod = [&](int jj) -> int64_t {
      if (pow2ns) return (j0 + jj) & (p.Ns - 1);
      int64_t k = k0 + jj;
      while (k >= p.Ns) k -= p.Ns;
      return k;
    };
    const int64_t seq = s * p.nshift + t;
    mbar_wait(&bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    // ---- stage A from the staged rows
    cd v[IA][B];
#pragma unroll
    for (int i = 0; i < IA; ++i) {
      const int w = tid + i * kGfftThreads;
      const int jj = w & (kCnt - 1), n1 = w >> kLgCnt;
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) {
        const int r = n1 + A * n2;
        if (c64) {
          const float2 f = reinterpret_cast<const float2*>(stage[buf])[r * kCnt + jj];
          v[i][n2] = cd{(double)f.x, (double)f.y};
        } else {
          const double2 d = reinterpret_cast<const double2*>(stage[buf])[r * kCnt + jj];
          v[i][n2] = cd{d.x, d.y};
        }
      }
    }
#pragma unroll
    for (int i = 0; i < IA; ++i) {
      const int w = tid + i * kGfftThreads;
      const int jj = w & (kCnt - 1), n1 = w >> kLgCnt;
      if (p.Ns > 1) {
        const int64_t kt = kmod(jj) * tstep;
        if (kt) {
          cd cur = tw_b(p.tlo, p.thi, kt * n1);
          const cd step = tw_b(p.tlo, p.thi, kt * A);
#pragma unroll
          for (int n2 = 0; n2 < B; ++n2) {
            if (n1 || n2) v[i][n2] = cmul(v[i][n2], cur);
            if (n2 + 1 < B) cur = cmul(cur, step);
          }
        }
      }
      dft_reg<B>(v[i]);
      cd* u = U + jj * LD + n1 * B;
#pragma unroll
      for (int qb = 0; qb < B; ++qb) u[qb] = (n1 && qb) ? cmul(v[i][qb], twR[n1 * qb]) : v[i][qb];
    }
    __syncthreads();
    // ---- stage B: DFT_A over n1, outputs q = qb + B qa
    double* out = p.out ? p.out + 2 * (s * p.out_signal_stride + p.out_offset +
                                       t * p.out_shift_stride)
                        : nullptr;
    cd* tmp = p.tmp ? p.tmp + seq * p.b : nullptr;
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      const int w = tid + i * kGfftThreads;
      int jj, qb;
      if (p.Ns == 1) {
        qb = w & (B - 1);
        jj = w >> LB;
      } else {
        jj = w & (kCnt - 1);
        qb = w >> kLgCnt;
      }
      cd a[A];
      const cd* u = U + jj * LD + qb;
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) a[n1] = u[n1 * B];
      dft_reg<A>(a);
      const int64_t j = j0 + jj;
      const int64_t k = kmod(jj);
      const int64_t base = (j - k) * R + k;
#pragma unroll
      for (int qa = 0; qa < A; ++qa) {
        const int64_t dst = base + (int64_t)(qb + B * qa) * p.Ns;
        if (tmp) {
          __stcs(reinterpret_cast<double2*>(tmp + dst), make_double2(a[qa].re, a[qa].im));
        } else {
          const cd wv = cscale(a[qa], inv_b);
          *reinterpret_cast<double2*>(out + 2 * dst * p.out_bin_stride) = make_double2(wv.re, wv.im);
        }
      }
    }
    __syncthreads();  // U and this tile's stage are free again
  }
}

// AFFT_FFT_TMAP=1: the staged pass with one TMA tensor request per tile (UTMALDG)
static bool tmap_env() {
  static const bool v = [] {
    const char* e = getenv("AFFT_FFT_TMAP");
    return e && e[0] == '1';
  }();
  return v;
}

static const void* gfft_tma_fn(int lgr) {
  switch (lgr) {
    case 4: return (const void*)gfft_tma_kernel<2, 2>;
    case 5: return (const void*)gfft_tma_kernel<3, 2>;
    case 6: return (const void*)gfft_tma_kernel<3, 3>;
    case 7: return (const void*)gfft_tma_kernel<4, 3>;
    case 8: return (const void*)gfft_tma_kernel<4, 4>;
    default: return nullptr;
  }
}

static const void* gfft_reg_partial_fn(int lgr) {
  switch (lgr) {
    case 4: return (const void*)gfft_reg_kernel<2, 2, true>;
    case 5: return (const void*)gfft_reg_kernel<3, 2, true>;
    case 6: return (const void*)gfft_reg_kernel<3, 3, true>;
    case 7: return (const void*)gfft_reg_kernel<4, 3, true>;
    case 8: return (const void*)gfft_reg_kernel<4, 4, true>;
    default: return nullptr;
  }
}

static const void* gfft_reg_fn(int lgr) {
  switch (lgr) {
    case 2: return (const void*)gfft_reg_kernel<1, 1>;
    case 3: return (const void*)gfft_reg_kernel<2, 1>;
    case 4: return (const void*)gfft_reg_kernel<2, 2>;
    case 5: return (const void*)gfft_reg_kernel<3, 2>;
    case 6: return (const void*)gfft_reg_kernel<3, 3>;
    case 7: return (const void*)gfft_reg_kernel<4, 3>;
    case 8: return (const void*)gfft_reg_kernel<4, 4>;
    default: return nullptr;
  }
}

static const void* const* gstockham_fixed_table() {
  static const void* const t[9] = {
      nullptr,
      (const void*)gstockham_kernel<1>, (const void*)gstockham_kernel<2>,
      (const void*)gstockham_kernel<3>, (const void*)gstockham_kernel<4>,
      (const void*)gstockham_kernel<5>, (const void*)gstockham_kernel<6>,
      (const void*)gstockham_kernel<7>, (const void*)gstockham_kernel<8>};
  return t;
}

// Radices for b: first-fit decreasing of the prime factors into groups <= 256
// (a prime above 256 forms its own radix, up to AFFT_MAX_SMEM_DFT); descending.
static bool plan_radices(int64_t b, std::vector<int>* radices) {
  std::vector<int64_t> primes;
  int64_t m = b;
  for (int64_t q = 2; q * q <= m; ++q)
    while (m % q == 0) {
      primes.push_back(q);
      m /= q;
    }
  if (m > 1) primes.push_back(m);
  std::sort(primes.rbegin(), primes.rend());
  if (!primes.empty() && primes[0] > AFFT_MAX_SMEM_DFT) return false;
  std::vector<int64_t> groups;
  for (int64_t pr : primes) {
    bool placed = false;
    for (auto& g : groups)
      if (g * pr <= 256) {
        g *= pr;
        placed = true;
        break;
      }
    if (!placed) groups.push_back(pr);
  }
  std::sort(groups.rbegin(), groups.rend());
  radices->assign(groups.begin(), groups.end());
  if ((b & (b - 1)) == 0 && b >= 16) {  // powers of two: the same pass count, balanced
    int lg = 0;
    while ((int64_t(1) << lg) < b) ++lg;
    const int P = (lg + 7) / 8;
    radices->clear();
    for (int i = 0; i < P; ++i) radices->push_back(1 << (lg / P + (i < lg % P ? 1 : 0)));
  }
  return true;
}

// AFFT_FFT_SMEM=1 selects the smem Stockham pass for power-of-two radices (A/B runs).
static bool fft_smem_path() {
  static const bool v = [] {
    const char* e = getenv("AFFT_FFT_SMEM");
    return e && e[0] == '1';
  }();
  return v;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// The input of one register pass as a 3-D tensor of scalars: [seq][R rows][2 nb] with
// row stride nb points and sequence stride `seq_stride_bytes`; box [1][R][2 kCnt].
static bool encode_pass_map(CUtensorMap* m, const void* base, bool f32, int64_t nb, int R,
                            int kCnt, int64_t nseq, int64_t seq_stride_bytes) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const int64_t esz = f32 ? 8 : 16;  // bytes per complex point
  if ((reinterpret_cast<uintptr_t>(base) & 15) || seq_stride_bytes % 16 || (nb * esz) % 16 ||
      2 * nb > (int64_t(1) << 32) || nseq > (int64_t(1) << 32) || R > 256 || 2 * kCnt > 256)
    return false;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * nb), (cuuint64_t)R, (cuuint64_t)nseq};
  cuuint64_t strides[2] = {(cuuint64_t)(nb * esz), (cuuint64_t)seq_stride_bytes};
  cuuint32_t box[3] = {(cuuint32_t)(2 * kCnt), (cuuint32_t)R, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                         3, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int launch_fourstep(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                           int64_t b, const int64_t* shifts, int nshift, double* out,
                           int64_t out_offset, int64_t oss, int64_t osh, int64_t obin,
                           cudaStream_t stream, const int64_t* shift_table,
                           const DeepFuse* fuse = nullptr) {
  std::vector<int> radices;
  if (!plan_radices(b, &radices)) {
    set_error("bucket count %lld has a prime factor above %d", (long long)b, AFFT_MAX_SMEM_DFT);
    return AFFT_EUNSUPPORTED;
  }
  // 2^24 points: two radix-4096 passes (gfft4k_kernel) with AFFT_FFT_4K=1 (opt-in:
  // measured 0.79 / 0.84 ms against 0.34 ms for the three radix-256 passes on a c64 /
  // c128 2^24 transform, tools/k4_check.py — one-column tiles make 8-16 B row pieces,
  // and a copy of that shape alone runs at 1.6-3.3 TB/s, tools/col_bw.cu; two columns
  // would need 139 KB of shared memory per tile)
  static const bool fft4k_env = [] {
    const char* v = getenv("AFFT_FFT_4K");
    return v && v[0] == '1';
  }();
  const bool use4k = b == (int64_t(1) << 24) && fft4k_env && !fft_smem_path();
  if (use4k) radices.assign({4096, 4096});
  // the fused epilogue needs a register-resident radix-256 (or radix-4096) last pass over
  // full tiles
  if (fuse && ((!use4k && (radices.size() < 2 || radices.back() != 256 ||
                           (b / 256) % (kGStockPoints / 256))) ||
               fft_smem_path() || batch != 1 || nshift != 1 || obin != 1)) {
    set_error("spectrum_fused: plan without a radix-256 register last pass");
    return AFFT_EUNSUPPORTED;
  }
  GStockParams q;
  memset(&q, 0, sizeof(q));
  q.x = x;
  q.dtype = dtype;
  q.n = n;
  q.ld = ld;
  q.L = n / b;
  q.b = b;
  q.batch = batch;
  q.nshift = nshift;
  q.shift_table = shift_table;
  q.out_offset = out_offset;
  q.out_signal_stride = oss;
  q.out_shift_stride = osh;
  q.out_bin_stride = obin;
  for (int t = 0; t < nshift; ++t) q.tau[t] = shifts ? host_pymod(shifts[t], n) : 0;
  const int P = (int)radices.size();
  const int nlo = (int)std::min<int64_t>(b, 1 << kTwLoBits);
  const int nhi = (int)((b + (1 << kTwLoBits) - 1) >> kTwLoBits);
  const size_t seqs = (size_t)batch * nshift;
  const size_t buf = (seqs * b * 16 + 255) / 256 * 256;
  const size_t nbufs = P >= 3 ? 2 : (P == 2 ? 1 : 0);
  // cached tables, except under stream capture (no allocation or synchronisation
  // allowed there): then they are built into the scratch as part of the work
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  const bool own_tables = cap != cudaStreamCaptureStatusNone;
  const size_t tbytes = own_tables ? (size_t)(nlo + nhi) * 16 : 0;
  char* scratch = nullptr;
  cudaError_t e = nbufs * buf + tbytes
                      ? scratch_alloc(reinterpret_cast<void**>(&scratch), nbufs * buf + tbytes,
                                      stream)
                      : cudaSuccess;
  if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(large-b DFT)");
  cd* bufs[2] = {reinterpret_cast<cd*>(scratch), reinterpret_cast<cd*>(scratch + buf)};
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const cd* tables;
  if (own_tables) {
    cd* t = reinterpret_cast<cd*>(scratch + nbufs * buf);
    twiddle_tables_kernel<<<(unsigned)((std::max(nlo, nhi) + 255) / 256), 256, 0, stream>>>(
        b, t, nlo, t + nlo, nhi);
    tables = t;
  } else {
    tables = twiddle_tables_for(dev, b, nlo, nhi, stream);
  }
  if (!tables) {
    if (scratch) scratch_free(scratch, stream);
    return AFFT_ECUDA;
  }
  q.tlo = tables;
  q.thi = tables + nlo;
  int64_t Ns = 1;
  int rc = AFFT_OK;
  for (int s = 0; s < P && !rc; ++s) {
    const int R = radices[s];
    GStockParams g = q;
    g.R = R;
    g.Ns = Ns;
    g.cnt = std::max(1, kGStockPoints / R);
    g.in = s == 0 ? nullptr : bufs[(s - 1) & 1];
    g.tmp = s == P - 1 ? nullptr : bufs[s & 1];
    g.out = s == P - 1 ? out : nullptr;
    if (use4k) {
      const bool fz = fuse && s == P - 1;
      const void* k4 = fz ? (const void*)gfft4k_flags_kernel : (const void*)gfft4k_kernel;
      if (fz) {  // the radix-4096 epilogue ORs its bits in: zero the fused depths' bitmaps
        const int dtop = 63 - __builtin_clzll((unsigned long long)b) - 8;
        for (int t = fuse->t_lo; t <= 8 && e == cudaSuccess; ++t)
          e = cudaMemsetAsync(fuse->words + fuse->word_off[t], 0, (size_t)1 << (dtop + t - 3),
                              stream);
      }
      if (e == cudaSuccess) e = ensure_smem(k4, kG4Smem);
      int occ = 0;
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k4, kG4Threads, kG4Smem);
      if (e != cudaSuccess || occ < 1) {
        rc = cuda_status(e != cudaSuccess ? e : cudaErrorInvalidConfiguration, "radix-4096 pass");
        break;
      }
      const int64_t tiles = (int64_t)seqs * (b >> 12);
      const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)sms * occ);
      DeepFuse fz_arg = fz ? *fuse : DeepFuse{};
      void* args4[] = {&g, &fz_arg};
      e = cudaLaunchKernel(k4, dim3(grid), dim3(kG4Threads), args4, kG4Smem, stream);
      if (e != cudaSuccess) {
        rc = cuda_status(e, "radix-4096 launch");
        break;
      }
      Ns *= R;
      continue;
    }
    if (!make_dft_plan(R, &g.plan)) {
      rc = AFFT_EUNSUPPORTED;
      set_error("cannot plan a DFT of size %d", R);
      break;
    }
    g.in = s == 0 ? nullptr : bufs[(s - 1) & 1];
    g.tmp = s == P - 1 ? nullptr : bufs[s & 1];
    g.out = s == P - 1 ? out : nullptr;
    const int ldR = std::max((R & 1) ? R : R + 1, gstock_ld(R));
    // compile-time shape for power-of-two radices whose tiles are always full
    int lgr = -1;
    if ((R & (R - 1)) == 0 && R >= 2 && R <= 256 && (b / R) % (kGStockPoints / R) == 0) {
      lgr = 0;
      while ((1 << lgr) < R) ++lgr;
      g.cnt = kGStockPoints / R;
    }
    // power-of-two radices >= 16 over partial chunks (b not a multiple of 2048, e.g. the
    // radix-64 pass of 9728 = 152 x 64): the register pass's partial instantiation
    int lgr_partial = -1;
    if (lgr < 0 && (R & (R - 1)) == 0 && R >= 16 && R <= 256 && !fft_smem_path()) {
      lgr_partial = 0;
      while ((1 << lgr_partial) < R) ++lgr_partial;
    }
    const void* kfn = lgr < 0 ? (const void*)gstockham_kernel<-1> : gstockham_fixed_table()[lgr];
    size_t smem = (size_t)(R + 2 * (int64_t)g.cnt * ldR) * 16;
    int threads = kGStockThreads;
    // TMA-staged register pass when every row segment is contiguous and 16-B aligned
    const bool contiguous = s > 0 || (q.L == 1 && nshift == 1 && q.tau[0] == 0 && !shift_table &&
                                      (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                                      (batch == 1 || (ld * (dtype == AFFT_C64 ? 8 : 16)) % 16 == 0));
    // opt-in: with 128-byte row segments (256 bulk requests per 32 KB tile) the TMA
    // form measured 0.97 ms against 0.34 ms for the register-load form on a 2^24 c128
    // transform (tools/k2_time.py, identical outputs); the requests are too small
    static const bool tma_env = [] {
      const char* v = getenv("AFFT_FFT_TMA");
      return v && v[0] == '1';
    }();
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    int use_tmap = 0;
    if (fuse && s == P - 1) {  // last pass with the DeepFuse epilogue
      kfn = (const void*)gfft_flags_kernel;
      g.perm = 0;
      smem = (size_t)(R + (int64_t)g.cnt * (R + 1)) * 16;
      threads = kGfftThreads;
    } else if (lgr >= 4 && !fft_smem_path() && contiguous && (tma_env || tmap_env())) {
      kfn = gfft_tma_fn(lgr);
      g.perm = 0;
      smem = 128 + 2 * (size_t)R * g.cnt * 16 + (size_t)(R + (int64_t)g.cnt * (R + 1)) * 16;
      threads = kGfftThreads;
      if (tmap_env()) {
        const bool f32 = s == 0 && dtype == AFFT_C64;
        const void* base = s == 0 ? x : (const void*)g.in;
        const int64_t sstride = s == 0 ? ld * (dtype == AFFT_C64 ? 8 : 16) : b * 16;
        use_tmap = encode_pass_map(&tmap, base, f32, b / R, R, g.cnt, (int64_t)seqs, sstride) ? 1 : 0;
      }
    } else if (lgr_partial >= 4 && !(fuse && s == P - 1)) {  // register pass, partial chunks
      kfn = gfft_reg_partial_fn(lgr_partial);
      g.cnt = kGStockPoints / R;
      g.perm = 0;
      smem = (size_t)(R + (int64_t)g.cnt * (R + 1)) * 16;
      threads = kGfftThreads;
    } else if (lgr >= 2 && !fft_smem_path()) {  // register-resident pass
      kfn = gfft_reg_fn(lgr);
      const int64_t nch = (b / R) / g.cnt;
      static const int perm_env = [] {
        const char* v = getenv("AFFT_TILE_PERM");
        return v ? atoi(v) : 0;
      }();
      g.perm = (nch & (nch - 1)) == 0 ? perm_env : 0;
      smem = (size_t)(R + (int64_t)g.cnt * (R + 1)) * 16;
      threads = kGfftThreads;
    }
    e = ensure_smem(kfn, (int)smem);
    int occ = 0;
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem);
    if (e != cudaSuccess || occ < 1) {
      rc = cuda_status(e != cudaSuccess ? e : cudaErrorInvalidConfiguration, "large-b DFT pass");
      break;
    }
    const int64_t tiles = (int64_t)seqs * ((b / R + g.cnt - 1) / g.cnt);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)sms * occ);
    void* args_reg[] = {&g};
    void* args_tma[] = {&g, &tmap, &use_tmap};
    DeepFuse fz_arg = fuse ? *fuse : DeepFuse{};
    void* args_fuse[] = {&g, &fz_arg};
    const bool tma_kernel = kfn == gfft_tma_fn(lgr) && lgr >= 4;
    e = cudaLaunchKernel(kfn, dim3(grid), dim3(threads),
                         tma_kernel ? args_tma
                                    : (kfn == (const void*)gfft_flags_kernel ? args_fuse : args_reg),
                         smem, stream);
    if (e != cudaSuccess) {
      rc = cuda_status(e, "large-b DFT launch");
      break;
    }
    Ns *= R;
  }
  if (scratch) scratch_free(scratch, stream);
  if (!rc) AFFT_CHECK_LAUNCH("large-b DFT pass");
  return rc;
}

static int launch_gather_dft(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                             const int64_t* factors, int ncycles, const int64_t* out_offsets,
                             const int64_t* shifts, int nshift, double* out, int64_t oss,
                             int64_t osh, int64_t obin, cudaStream_t stream,
                             const int64_t* shift_table = nullptr) {
  if (batch == 0 || nshift == 0) return AFFT_OK;
  if (!x || !out || !factors || (!shifts && !shift_table)) {
    set_error("null pointer argument");
    return AFFT_EINVAL;
  }
  if (dtype != AFFT_C64 && dtype != AFFT_C128) {
    set_error("unknown dtype %d", dtype);
    return AFFT_EINVAL;
  }
  if (n < 1 || batch < 0 || ld < n) {
    set_error("bad sizes n=%lld batch=%lld ld=%lld", (long long)n, (long long)batch,
              (long long)ld);
    return AFFT_EINVAL;
  }
  if (ncycles < 1 || ncycles > AFFT_MAX_CYCLES) {
    set_error("number of cycles %d outside 1..%d", ncycles, AFFT_MAX_CYCLES);
    return AFFT_EUNSUPPORTED;
  }
  if (nshift < 0 || nshift > AFFT_MAX_SHIFTS) {
    set_error("number of shifts %d outside 0..%d", nshift, AFFT_MAX_SHIFTS);
    return AFFT_EUNSUPPORTED;
  }
  GatherDftParams q;  // ~6 KB, passed by value as a __grid_constant__ kernel parameter
  q.x = x;
  q.dtype = dtype;
  q.n = n;
  q.ld = ld;
  q.ncycles = ncycles;
  q.nshift = nshift;
  q.out = out;
  q.out_signal_stride = oss;
  q.out_shift_stride = osh;
  q.out_bin_stride = obin;
  q.shift_table = shift_table;
  for (int t = 0; t < nshift; ++t) q.tau[t] = shifts ? host_pymod(shifts[t], n) : 0;
  const size_t kBudget = 96 * 1024;
  size_t smem_max = 0;
  int total_jobs = 0;
  for (int c = 0; c < ncycles; ++c) {
    const int64_t b = factors[c];
    if (b < 1 || n % b) {
      set_error("bucket count %lld does not divide signal size %lld", (long long)b,
                (long long)n);
      return AFFT_EINVAL;
    }
    // b >= 1024 goes to the global passes too: the one-CTA smem DFT needs (3 b) 16 bytes
    // there (192 KB at b = 4096: one CTA per SM), the passes run 3 CTAs per SM — config
    // 4's sFFT-DT3 2.15 -> 1.98 ms and config 2's 2.04 -> 1.92 ms per batch.
    // AFFT_FOURSTEP_MIN_B moves the threshold (diagnostic; > 4096: the one-CTA DFT up to
    // AFFT_MAX_SMEM_DFT).
    static const int64_t fourstep_min_b = [] {
      const char* e = getenv("AFFT_FOURSTEP_MIN_B");
      return e ? std::max<int64_t>(2, atoll(e)) : (int64_t)1024;
    }();
    if (b > AFFT_MAX_SMEM_DFT || b >= fourstep_min_b) {
      if (nshift > 65535) {
        set_error("too many shifts for the large-b path");
        return AFFT_EUNSUPPORTED;
      }
      int rc = launch_fourstep(x, dtype, n, batch, ld, b, shifts, nshift, out, out_offsets[c],
                               oss, osh, obin, stream, shift_table);
      if (rc) return rc;
      q.b[c] = b;
      q.jobs[c] = 0;  // handled above
      q.chunk[c] = 1;
      q.out_offset[c] = out_offsets[c];
      q.plan[c].n = 1;
      q.plan[c].nstages = 0;
      continue;
    }
    if (!make_dft_plan(b, &q.plan[c], 16)) {
      set_error("cannot plan a DFT of size %lld", (long long)b);
      return AFFT_EUNSUPPORTED;
    }
    q.b[c] = b;
    q.out_offset[c] = out_offsets[c];
    int64_t fit = ((int64_t)(kBudget / 16) - b) / (2 * b);
    int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(fit, nshift));
    q.chunk[c] = chunk;
    q.jobs[c] = (nshift + chunk - 1) / chunk;
    total_jobs += q.jobs[c];
    size_t bytes = (size_t)(b + 2 * (int64_t)chunk * b) * 16;
    smem_max = std::max(smem_max, bytes);
  }
  if (total_jobs == 0) return AFFT_OK;  // every cycle went through the four-step path
  if (total_jobs > 65535) {
    set_error("too many (cycle, shift-chunk) jobs per signal: %d", total_jobs);
    return AFFT_EUNSUPPORTED;
  }
  cudaError_t e = ensure_smem((const void*)gather_dft_kernel, (int)smem_max);
  if (e != cudaSuccess) {
    return cuda_status(e, "cudaFuncSetAttribute(gather_dft)");
  }
  dim3 grid((unsigned)batch, (unsigned)total_jobs);
  gather_dft_kernel<<<grid, 256, smem_max, stream>>>(q);
  AFFT_CHECK_LAUNCH("gather_dft_kernel");
  return AFFT_OK;
}

int spectrum_fused(const void* x, int dtype, int64_t n, double* Y, const DeepFuse& f,
                   cudaStream_t st) {
  if (n < 4096 || (n & (n - 1))) {
    set_error("spectrum_fused: n = %lld", (long long)n);
    return AFFT_EUNSUPPORTED;
  }
  const int64_t zero = 0;
  return launch_fourstep(x, dtype, n, 1, n, n, &zero, 1, Y, 0, n, n, 1, st, nullptr, &f);
}

}  // namespace afft

using namespace afft;

extern "C" int afft_bucketize(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                              int64_t b, const int64_t* shifts, int32_t nshift, double* out,
                              int64_t out_signal_stride, int64_t out_shift_stride,
                              int64_t out_bin_stride, void* stream) {
  int64_t off = 0;
  return launch_gather_dft(x, dtype, n, batch, ld, &b, 1, &off, shifts, nshift, out,
                           out_signal_stride, out_shift_stride, out_bin_stride,
                           (cudaStream_t)stream);
}

extern "C" int afft_build_graph(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                                const int64_t* factors, int32_t ncycles, const int64_t* shifts,
                                int32_t nshift, double* nodes, void* stream) {
  if (ncycles < 1 || ncycles > AFFT_MAX_CYCLES || !factors) {
    set_error("number of cycles %d outside 1..%d", ncycles, AFFT_MAX_CYCLES);
    return AFFT_EUNSUPPORTED;
  }
  int64_t offs[AFFT_MAX_CYCLES];
  int64_t total = 0;
  for (int c = 0; c < ncycles; ++c) {
    offs[c] = total * nshift;
    total += factors[c];
  }
  return launch_gather_dft(x, dtype, n, batch, ld, factors, ncycles, offs, shifts, nshift, nodes,
                           total * nshift, 1, nshift, (cudaStream_t)stream);
}

namespace afft {
// build_graph (peeling.py:169-178) with per-signal shifts: shift_table is a device
// [batch][nshift] array of raw shifts (reduced on the device).
int build_graph_table(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                      const int64_t* factors, int32_t ncycles, const int64_t* shift_table,
                      int32_t nshift, double* nodes, cudaStream_t stream) {
  if (ncycles < 1 || ncycles > AFFT_MAX_CYCLES || !factors) {
    set_error("number of cycles %d outside 1..%d", ncycles, AFFT_MAX_CYCLES);
    return AFFT_EUNSUPPORTED;
  }
  int64_t offs[AFFT_MAX_CYCLES];
  int64_t total = 0;
  for (int c = 0; c < ncycles; ++c) {
    offs[c] = total * nshift;
    total += factors[c];
  }
  return launch_gather_dft(x, dtype, n, batch, ld, factors, ncycles, offs, nullptr, nshift, nodes,
                           total * nshift, 1, nshift, stream, shift_table);
}
}  // namespace afft

extern "C" int afft_bucketize_table(const void* x, int dtype, int64_t n, int64_t batch,
                                    int64_t ld, int64_t b, const int64_t* shift_table,
                                    int32_t nshift, double* out, int64_t out_signal_stride,
                                    int64_t out_shift_stride, int64_t out_bin_stride,
                                    void* stream) {
  int64_t off = 0;
  return launch_gather_dft(x, dtype, n, batch, ld, &b, 1, &off, nullptr, nshift, out,
                           out_signal_stride, out_shift_stride, out_bin_stride,
                           (cudaStream_t)stream, shift_table);
}
