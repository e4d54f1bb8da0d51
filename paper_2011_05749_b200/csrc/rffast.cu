// K3 (noisy) + K4 (noisy) + K7 (median): R-FFAST on the GPU.
//
//   robust_thresholds  (peeling.py:335-358)  per-signal median of node energies
//                      by an in-smem bitonic sort, T0/T1 gates;
//   singleton_search_noisy (peeling.py:222-250)  the exhaustive candidate scan:
//                      for every residue-class candidate cand = i + b*t and every
//                      stride 2^j, wrap(est_j - target_j(cand))^2 summed in j
//                      order, first argmin; then the 1-column least-squares fit;
//   peel_decode(mode="noisy") (peeling.py:270-313 with classify_noisy 253-267)
//                      as rounds of kernels over device-resident state: prep
//                      (zero-ton gate, phase estimates, compacted active list)
//                      → search → finalize → harvest/subtract, one host sync per
//                      round for the loop exit.
//
// Bit-faithfulness of the scan: target is
// ((-2*pi) * r) / n with r = (2^j * cand) mod n carried exactly by doubling
// mod n; _wrap(p) = ((p + pi) mod 2pi) - pi with numpy's floor-mod sign rule,
// evaluated exactly (x - q*2pi is exact by Sterbenz for q in {1, 2}); no FMA
// contraction (--fmad=false); scores summed in j order; ties keep the first
// candidate.  Only atan2 differs from glibc, by <= 2 ulp in the estimates.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <type_traits>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "afft_common.cuh"
#include "peel_core.cuh"

namespace afft {

constexpr int kMaxStrides = 40;
constexpr int kMaxRounds = 16;  // rounds per stride (m)
constexpr int kSearchThreads = 256;
constexpr int kCandPerThread = 64;  // 16 -> 64: fewer first candidates scored against the seed bound
constexpr int kChunk = kSearchThreads * kCandPerThread;
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;

struct NoisyPlan {
  int64_t n;
  int ncycles;
  int nodes;
  int R;  // = c * m
  int c, m;
  int hmask;
  int64_t b[AFFT_MAX_CYCLES];
  int32_t base[AFFT_MAX_CYCLES + 1];
  double w[kMaxRounds];          // Kay weights (m - 1 entries)
  int64_t tau[AFFT_MAX_SHIFTS];  // shifts reduced mod n
  // optional per-signal shifts: device [signals][R], reduced mod n (R-FFAST batches whose
  // signals carry their own search anchors, peeling.py:163-164); null: tau for all
  const int64_t* tau_tab;
  uint64_t nmagic;  // floor((2^64 - 1) / n): Barrett reduction for tau * f mod n
  // optional signal of each residual row (DSFFT batches: rows of several signals in one
  // list); null: row / nodes
  const int32_t* row_sig;
};

__device__ __forceinline__ int64_t plan_row_signal(const NoisyPlan& P, int64_t row) {
  return P.row_sig ? P.row_sig[row] : (P.tau_tab ? row / P.nodes : 0);
}

// (a * b) mod P.n for 0 <= a, b < n <= 2e9 (a * b < 2^62): Barrett with the plan's
// magic, exact after at most two corrections — the int64 '%' it replaces compiled to
// a ~70-instruction division routine (13% of noisy_finalize_kernel's instructions).
__device__ __forceinline__ int64_t plan_mulmod(const NoisyPlan& P, int64_t a, int64_t b) {
  const uint64_t p = (uint64_t)(a * b);
  const uint64_t q = __umul64hi(p, P.nmagic);
  uint64_t r = p - q * (uint64_t)P.n;
  while (r >= (uint64_t)P.n) r -= (uint64_t)P.n;
  return (int64_t)r;
}

__device__ __forceinline__ int64_t plan_tau(const NoisyPlan& P, int64_t s, int r) {
  return P.tau_tab ? P.tau_tab[s * P.R + r] : P.tau[r];
}

// numpy: np.remainder(p + pi, 2pi) - pi.  The common ranges need no sign-of-zero fix:
// x >= 0 there and x - k 2pi is exact (Sterbenz), so a zero result is +0 already.
__device__ __forceinline__ double wrap_phase(double p) {
  const double x = __dadd_rn(p, kPi);
  double r;
  if (x >= 0.0 && x < kTwoPi) {
    r = x;
  } else if (x >= kTwoPi && x < 2.0 * kTwoPi) {
    r = __dsub_rn(x, kTwoPi);  // exact (Sterbenz)
  } else if (x >= 2.0 * kTwoPi && x < 3.0 * kTwoPi) {
    r = __dsub_rn(x, 2.0 * kTwoPi);  // exact (Sterbenz), 2*2pi exact
  } else if (x < 0.0 && x >= -kTwoPi) {
    r = __dadd_rn(x, kTwoPi);  // fmod(x) = x (<0): numpy adds the divisor
    if (r == 0.0) r = 0.0;     // copysign(0, +2pi)
  } else {
    r = fmod(x, kTwoPi);
    if (r != 0.0 && r < 0.0) r = __dadd_rn(r, kTwoPi);
    if (r == 0.0) r = 0.0;  // copysign(0, +2pi)
  }
  return __dsub_rn(r, kPi);
}

// Phase estimate of stride j (peeling.py:241-244): Kay-weighted mean of the
// re-centred consecutive phase differences of y[j*m .. j*m+m-1].
__device__ __forceinline__ double stride_estimate(const cd* y, int m, const double* w) {
  double d[kMaxRounds];
  for (int t = 0; t + 1 < m; ++t) {
    const cd a = y[t + 1], b = y[t];
    // a * conj(b), numpy complex multiply on (b.re, -b.im)
    const double re = __dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, -b.im));
    const double im = __dadd_rn(__dmul_rn(a.re, -b.im), __dmul_rn(a.im, b.re));
    d[t] = atan2(im, re);
  }
  const double d0 = d[0];
  double est = 0.0;
  for (int t = 0; t + 1 < m; ++t) {
    const double dt = __dadd_rn(d0, wrap_phase(__dsub_rn(d[t], d0)));
    est = __dadd_rn(est, __dmul_rn(w[t], dt));
  }
  return est;
}

// f mod b for 0 <= f: 32-bit when both fit (the 64-bit remainder is a library call,
// most of noisy_harvest_kernel's stall samples at config 3')
__device__ __forceinline__ int64_t mod_nonneg(int64_t f, int64_t b) {
  if (((uint64_t)f | (uint64_t)b) < (1ull << 32)) return (int64_t)((uint32_t)f % (uint32_t)b);
  return f % b;
}

__device__ __forceinline__ int noisy_cycle(const NoisyPlan& P, int g) {
  int c = 0;
  while (g >= P.base[c + 1]) ++c;
  return c;
}

// -------------------------------------------------------------- candidate scan

// Score of candidate cand = (index + b*t) mod n (already reduced: r = cand), summed
// in stride order exactly as the reference does; stops (returns > bound) once the
// partial sum exceeds bound: every term is >= 0, so such a candidate is strictly
// worse than the candidate that set bound and can be neither the minimum nor a tie.
// target = RN(RN(-2 pi r) / n) by Markstein's sequence with the correctly rounded
// reciprocal: q0 = RN(x inv), rem = x - q0 n (exact, fma), q = RN(q0 + rem inv).
// Bit-identical to the IEEE quotient for every r in [0, n) at n <= 2^28 and a
// 2^28-point sweep at n = 3e9 (tools/div_check.cu), up to the sign of a zero at r = 0.
// k32: n < 2^31, so the doubled residue 2r < 2^32 fits in 32 bits (the 64-bit
// doubling-and-reduce was ~15% of the kernel's instructions; the kernel is issue-bound).
template <bool k32>
__device__ __forceinline__ double cand_score(
    typename std::conditional<k32, uint32_t, int64_t>::type r,
    typename std::conditional<k32, uint32_t, int64_t>::type nn, const double* s_est, int c,
    double dn, double inv, double bound) {
  double sc = 0.0;
  for (int j = 0; j < c; ++j) {
    const double x = __dmul_rn(-kTwoPi, (double)r);
    const double q0 = __dmul_rn(x, inv);
    // (r = 0 gives +0.0 here where x / n is -0.0; est - tgt differs only in the sign
    // of a zero, which the + pi inside wrap_phase erases — the score is bit-identical)
    const double tgt = __fma_rn(__fma_rn(-q0, dn, x), inv, q0);
    const double wv = wrap_phase(__dsub_rn(s_est[j], tgt));
    sc = __dadd_rn(sc, __dmul_rn(wv, wv));
    if (sc > bound) return sc;
    r <<= 1;
    if (r >= nn) r -= nn;
  }
  return sc;
}

// Pruning bound: the full score of the candidate nearest the stride-0 estimate.
template <bool k32>
__device__ __forceinline__ double search_bound(int64_t n, int64_t b, int64_t L, int64_t idx,
                                               const double* s_est, int c, double inv) {
  using rt = typename std::conditional<k32, uint32_t, int64_t>::type;
  const double dn = (double)n;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  auto cand_of = [&](double f) {  // the residue-class candidate nearest frequency f
    int64_t th = (int64_t)floor((f - (double)idx) / (double)b + 0.5);
    th %= L;
    if (th < 0) th += L;
    return th;
  };
  const double fe = (-s_est[0] * dn) / kTwoPi;
  const int64_t th0 = cand_of(fe);
  double bound = cand_score<k32>((rt)(idx + b * th0), (rt)n, s_est, c, dn, inv, inf);
  if (!(bound == bound)) return inf;  // NaN: no pruning
  // Successive refinement (any real candidate's score is a valid bound; a better one
  // prunes more and narrows the stride-0 arc): stride 2^j's estimate fixes 2^j f / n
  // modulo 1, so of the 2^j frequencies it allows keep the one nearest the running
  // estimate, while 2^j < 8 L (finer than the candidate grid after that).
  double f = fe - floor(fe / dn) * dn;
  for (int j = 1; j < c && (int64_t(1) << j) < 8 * L; ++j) {
    const double sc = ldexp(1.0, j);
    const double x = f * sc / dn;
    double g = -s_est[j] * (1.0 / kTwoPi);
    g -= floor(g);
    double d = g - (x - floor(x));
    d -= floor(d + 0.5);  // wrap into [-1/2, 1/2)
    f += d * dn / sc;
    f -= floor(f / dn) * dn;
  }
  const int64_t th = cand_of(f);
  if (th != th0) {
    const double s1 = cand_score<k32>((rt)(idx + b * th), (rt)n, s_est, c, dn, inv, bound);
    if (s1 < bound) bound = s1;
  }
  return bound;
}

// Per-node pruning bound shared by every CTA scanning the node: the bit pattern of
// the lowest full score seen so far (scores are >= +0, so they order like their bits;
// the all-ones pattern, a negative NaN, is the "+inf" the est kernel initialises).
// A candidate is dropped only once its partial sum exceeds a score some candidate
// actually has, so the minimum and every tie with it are still scored in full: the
// (min score, smallest t) result is the same whatever order CTAs run in.  A multiton
// node's minimum sits far below the typical score (~27 strides x pi^2/3), and one
// thread's own best of 16 candidates left it ~2.5x as many strides per candidate.
__device__ __forceinline__ unsigned long long load_bound_bits(const unsigned long long* g) {
  return *reinterpret_cast<const volatile unsigned long long*>(g);
}
__device__ __forceinline__ double bound_of_bits(unsigned long long v) {
  return v >= 0x7ff0000000000000ull ? __longlong_as_double(0x7ff0000000000000LL)
                                    : __longlong_as_double((long long)v);
}
__device__ __forceinline__ double shared_bound(const unsigned long long* g) {
  return bound_of_bits(load_bound_bits(g));
}
__device__ __forceinline__ void lower_bound_to(unsigned long long* g, double sc) {
  atomicMin(g, (unsigned long long)__double_as_longlong(sc));
}

// Fixed-point pre-filter of the candidate scan.  A candidate's phase at stride j is
// frac(2^j r / n) turns, r = idx + b t; as a 64-bit fraction G(t) = A0 + t S with
// A0 = floor(idx 2^64 / n) and S = floor((2^64 - 1) / L) (error <= L + 1 units of
// 2^-64), and stride j's phase is the top 32 bits of G << j (one funnel shift).
// est_j - target = E_j + phase_j in 32-bit turns wraps by itself; x = that >> 18 is
// the wrapped difference in units of 2^-14 turn, and sum x^2 (uint32, every term
// <= 2^26) is compared against the pruning bound converted to those units plus a
// margin covering every approximation: per term |x'^2 - d^2| <= 2 * 0.5 * e + e^2
// turns^2 with e <= 2^-14 + 2^-31 + (L + 1) 2^(j - 64) (the last <= 2^-20 where this
// is used).  A candidate whose approximate partial sum exceeds that limit has an
// exact partial sum above the bound, so it is dropped exactly as cand_score would
// drop it; every other candidate is then scored exactly.  Integer work only, four
// strides per limit test: ~6 instructions per stride against ~18 (9 FP64).
struct ApproxScan {
  bool on;
  uint64_t A0, S;
  double margin;  // radians^2
};
constexpr double kApproxUnit2 = 1.4706e-07;  // (2 pi 2^-14)^2 rad^2 per x^2 unit, rounded down

// The limit in x^2 units (the sum may pass it by four terms: < 2^31 + 2^28 < 2^32),
// or 0 when the bound is beyond any score (no pre-filter).
__device__ __forceinline__ uint32_t approx_limit(double bound, double margin) {
  const double lim = (bound + margin) / kApproxUnit2;
  return lim < 2147483648.0 ? (uint32_t)lim : 0u;
}

__device__ __forceinline__ uint32_t approx_term(uint32_t e, uint32_t phase) {
  const int32_t x = (int32_t)(e + phase) >> 18;
  return (uint32_t)(x * x);
}

// Per-node set-up.  Phase error per term at stride j (turns): e_j = 2^-14 (the >> 18)
// + 2^-31 (E_j rounding, the top-32-bit truncation) + (L + 1) 2^(j - 64) (G(t)); the
// margin is (2 pi)^2 sum_j (e_j + e_j^2) rad^2 plus two limit units.  Off for NaN /
// infinite estimates (the exact path handles them), n >= 2^32, or e_j > 2^-12.
__device__ __forceinline__ ApproxScan make_approx(int64_t n, int64_t L, int64_t idx, int c,
                                                  bool finite) {
  ApproxScan ap;
  const double drift = (double)(L + 1) * 5.421010862427522e-20;  // (L + 1) 2^-64
  const double emax = 6.103515625e-05 + 4.6566128730773926e-10 + drift * ldexp(1.0, c - 1);
  ap.on = finite && (uint64_t)n < (1ull << 32) && emax <= 2.44140625e-04;
  ap.A0 = ap.S = 0;
  ap.margin = 0.0;
  if (ap.on) {
    const uint64_t un = (uint64_t)n, num = (uint64_t)idx << 32;
    const uint64_t q1 = num / un, r1 = num - q1 * un;
    ap.A0 = (q1 << 32) | ((r1 << 32) / un);
    ap.S = ~0ull / (uint64_t)L;
    const double esum = (double)c * (6.103515625e-05 + 4.6566128730773926e-10) +
                        drift * (ldexp(1.0, c) - 1.0);
    ap.margin = 39.47841760435743 * (esum + (double)c * emax * emax) * 1.000001 +
                2.0 * kApproxUnit2;
  }
  return ap;
}

// true: pruned (the approximate partial sum passed lim)
__device__ __forceinline__ bool approx_pruned(uint64_t G, const uint32_t* E, int c, uint32_t lim) {
  const uint32_t hi = (uint32_t)(G >> 32), lo = (uint32_t)G;
  uint32_t sum = 0;
  const int c1 = c < 32 ? c : 32;
  int j = 0;
  for (; j + 4 <= c1; j += 4) {
    sum += approx_term(E[j], __funnelshift_l(lo, hi, j)) +
           approx_term(E[j + 1], __funnelshift_l(lo, hi, j + 1)) +
           approx_term(E[j + 2], __funnelshift_l(lo, hi, j + 2)) +
           approx_term(E[j + 3], __funnelshift_l(lo, hi, j + 3));
    if (sum > lim) return true;
  }
  for (; j < c1; ++j) sum += approx_term(E[j], __funnelshift_l(lo, hi, j));
  for (; j < c; ++j) sum += approx_term(E[j], lo << (j - 32));
  return sum > lim;
}

// The candidates t of [t0, t1) that can still score <= B: the stride-0 term alone is
// d0(t) = wrap(est_0 + 2 pi (idx + b t) / n), linear in t with slope 2 pi / L (idx + b t
// < n), so score(t) <= B needs |d0(t)| <= sqrt(B): a circular arc of half-width
// sqrt(B) L / (2 pi) around the seed's candidate.  Candidates outside it (with two
// candidates and 1e-9 relative of margin, far above the rounding of est_0 / (2 pi),
// idx / n and the device's d0) score > B, so skipping them changes neither the minimum
// nor its smallest t.  Up to two ranges [r[0], r[1]) and [r[2], r[3]) (the arc may wrap);
// the whole chunk when B gives no restriction.
struct CandRanges {
  int64_t r[4];
  __device__ int64_t len() const { return (r[1] - r[0]) + (r[3] - r[2]); }
  __device__ int64_t at(int64_t v) const { return v < r[1] - r[0] ? r[0] + v : r[2] + (v - (r[1] - r[0])); }
};
__device__ __forceinline__ CandRanges stride0_ranges(double est0, int64_t idx, int64_t n,
                                                     int64_t L, double B, int64_t t0,
                                                     int64_t t1) {
  CandRanges c{{t0, t1, 0, 0}};
  if (!(B < 9.0) || !(est0 == est0) || isinf(est0)) return c;  // NaN / no restriction
  const double w = sqrt(B) * (1.0 / kTwoPi) * (1.0 + 1e-9) + 1e-12;  // turns
  double u = -(est0 * (1.0 / kTwoPi) + (double)idx / (double)n);
  u -= floor(u);
  const double ct = u * (double)L, hw = w * (double)L + 2.0;
  if (!(2.0 * hw + 2.0 < (double)L)) return c;
  const int64_t lo = (int64_t)floor(ct - hw), hi = (int64_t)ceil(ct + hw) + 1;  // [lo, hi)
  // the arc as up to two pieces of [0, L), each intersected with [t0, t1)
  int64_t p[4];
  if (lo < 0) {
    p[0] = lo + L; p[1] = L; p[2] = 0; p[3] = hi;
  } else if (hi > L) {
    p[0] = lo; p[1] = L; p[2] = 0; p[3] = hi - L;
  } else {
    p[0] = lo; p[1] = hi; p[2] = 0; p[3] = 0;
  }
  for (int q = 0; q < 4; q += 2) {
    const int64_t a = max(p[q], t0), e = min(p[q + 1], t1);
    c.r[q] = a;
    c.r[q + 1] = e > a ? e : a;
  }
  return c;
}

// Shared state of one CTA's chunk scan.
struct ScanSmem {
  double est[kMaxStrides];
  uint32_t e32[kMaxStrides];
  int nan;
  unsigned long long bound;
  CandRanges rng;  // the chunk's candidates left by the stride-0 arc (one copy per CTA)
  double w_score[kSearchThreads / 32];
  int32_t w_t[kSearchThreads / 32];
};

// One CTA scores kChunk consecutive candidates t (chunk `chunk`) of active node a:
// residue `act_index[a]` of cycle size `act_b[a]`, estimates est[a][0..c).  Leaves the
// chunk's (min score, smallest t) in part_score / part_t [a][chunk].  Ends with a
// barrier, so a persistent CTA may reuse `sm` for its next chunk.
template <bool k32>
__device__ __forceinline__ void scan_chunk(ScanSmem& sm, int64_t n, int c, int a, int chunk,
                                           const int64_t* __restrict__ act_index,
                                           const int64_t* __restrict__ act_b,
                                           const double* __restrict__ est, int chunks,
                                           double* __restrict__ part_score,
                                           int32_t* __restrict__ part_t,
                                           unsigned long long* __restrict__ node_bound) {
  const int64_t b = act_b[a];
  const int64_t L = n / b;
  const int64_t t0 = (int64_t)chunk * kChunk;
  if (threadIdx.x == 0) {
    sm.nan = 0;
    sm.bound = load_bound_bits(node_bound + a);
  }
  __syncthreads();
  if (threadIdx.x < c) {
    const double e = est[(int64_t)a * c + threadIdx.x];
    sm.est[threadIdx.x] = e;
    double u = e * 0.15915494309189535;  // turns (any rounding is inside the margin)
    u -= floor(u);
    sm.e32[threadIdx.x] = (uint32_t)(uint64_t)(u * 4294967296.0);
    if (!(e == e) || isinf(e)) sm.nan = 1;
    // one CTA-wide copy of the candidate ranges, from the bound as loaded above (threads
    // that computed their own could see different bounds and leave gaps between them)
    if (threadIdx.x == 0)
      sm.rng = stride0_ranges(e, act_index[a], n, L, bound_of_bits(sm.bound), t0,
                              min(L, t0 + (int64_t)kChunk));
  }
  __syncthreads();
  const int64_t idx = act_index[a];
  const ApproxScan ap = make_approx(n, L, idx, c, !sm.nan);
  const double dn = (double)n;
  const double inv = 1.0 / dn;
  using rt = typename std::conditional<k32, uint32_t, int64_t>::type;
  double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  int32_t bt = INT32_MAX;
  if (t0 < L) {
    unsigned long long* gb = node_bound + a;
    double bound = bound_of_bits(sm.bound);  // seeded by noisy_seed_kernel
    // Two levels: the CTA's own bound in shared memory, read before every candidate,
    // and the node's global bound, folded into it every 4 candidates from a load
    // issued 4 candidates earlier (a global load waited on before every candidate was
    // 2/3 of the kernel's stall samples).  Any value read is some candidate's real
    // score, so a stale one only prunes less.
    volatile unsigned long long* vs_bound = &sm.bound;
    unsigned long long pending = load_bound_bits(gb);
    int k = 0;
    // only the candidates the stride-0 term leaves possible under the chunk's bound
    const int64_t nv = sm.rng.len();
    for (int64_t v = threadIdx.x; v < nv; v += kSearchThreads, ++k) {
      const int64_t t = sm.rng.at(v);
      if ((k & 3) == 3) {
        atomicMin(&sm.bound, pending);
        pending = load_bound_bits(gb);
      }
      bound = fmin(bound, bound_of_bits(*vs_bound));
      if (ap.on) {
        const uint32_t lim = approx_limit(bound, ap.margin);
        if (lim && approx_pruned(ap.A0 + (uint64_t)t * ap.S, sm.e32, c, lim)) continue;
      }
      const double sc = cand_score<k32>((rt)(idx + b * t), (rt)n, sm.est, c, dn, inv, bound);
      if (sc > bound) continue;  // pruned / worse than a candidate that is scored in full
      if (sc < best) {
        best = sc;
        bt = (int32_t)t;
      }
      if (sc < bound) {
        bound = sc;
        atomicMin(&sm.bound, (unsigned long long)__double_as_longlong(sc));
        lower_bound_to(gb, sc);
      }
    }
  }
  // block argmin, ties -> smaller t
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (ob < best || (ob == best && ot < bt)) {
      best = ob;
      bt = ot;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sm.w_score[threadIdx.x >> 5] = best;
    sm.w_t[threadIdx.x >> 5] = bt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b0 = sm.w_score[0];
    int32_t t0w = sm.w_t[0];
    for (int w = 1; w < kSearchThreads / 32; ++w) {
      if (sm.w_score[w] < b0 || (sm.w_score[w] == b0 && sm.w_t[w] < t0w)) {
        b0 = sm.w_score[w];
        t0w = sm.w_t[w];
      }
    }
    part_score[(int64_t)a * chunks + chunk] = b0;
    part_t[(int64_t)a * chunks + chunk] = t0w;
  }
  __syncthreads();
}

// Grid (this rank's chunks, active nodes): one chunk per CTA.
template <bool k32>
__global__ void __launch_bounds__(kSearchThreads, 8) noisy_search_kernel(
    int64_t n, int c, const int64_t* __restrict__ act_index, const int64_t* __restrict__ act_b,
    const double* __restrict__ est, int chunks, double* __restrict__ part_score,
    int32_t* __restrict__ part_t, int chunk_rank, int chunk_world,
    unsigned long long* __restrict__ node_bound) {
  __shared__ ScanSmem sm;
  const int a = blockIdx.y;
  const int chunk = chunk_rank + (int)blockIdx.x * chunk_world;  // this rank's chunks
  scan_chunk<k32>(sm, n, c, a, chunk, act_index, act_b, est, chunks, part_score, part_t,
                  node_bound);
}

// Device-resident rounds: the active count is only known on the device, so a
// persistent grid (a few CTAs per SM) pulls (node, chunk) items from a ticket counter,
// node-major, until all A * chunks are scanned.  Same per-chunk results as above.
template <bool k32>
__global__ void __launch_bounds__(kSearchThreads, 8) noisy_search_persistent_kernel(
    int64_t n, int c, const int32_t* __restrict__ A_dev, const int64_t* __restrict__ act_index,
    const int64_t* __restrict__ act_b, const double* __restrict__ est, int chunks,
    double* __restrict__ part_score, int32_t* __restrict__ part_t,
    unsigned long long* __restrict__ node_bound, int32_t* __restrict__ ticket) {
  __shared__ ScanSmem sm;
  __shared__ int item;
  const int64_t total = (int64_t)(*A_dev) * chunks;
  for (;;) {
    if (threadIdx.x == 0) item = atomicAdd(ticket, 1);
    __syncthreads();
    const int it = item;
    if (it >= total) break;
    scan_chunk<k32>(sm, n, c, it / chunks, it % chunks, act_index, act_b, est, chunks,
                    part_score, part_t, node_bound);
  }
}

// The shared bound's seed, once per node (computing it in every CTA, by every thread,
// was most of the CTA kernel's instructions): the full score of the candidate nearest
// the stride-0 estimate.
template <bool k32>
__global__ void noisy_seed_kernel(int64_t n, int c, int A, const int64_t* __restrict__ act_index,
                                  const int64_t* __restrict__ act_b,
                                  const double* __restrict__ est,
                                  unsigned long long* __restrict__ node_bound,
                                  const int32_t* __restrict__ A_dev = nullptr) {
  if (A_dev) A = *A_dev;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int64_t b = act_b[a];
  const double bound =
      search_bound<k32>(n, b, n / b, act_index[a], est + (int64_t)a * c, c, 1.0 / (double)n);
  if (bound < __longlong_as_double(0x7ff0000000000000LL))
    node_bound[a] = (unsigned long long)__double_as_longlong(bound);
}

// Short candidate lists (L = n / b <= kWarpSearchMaxL, DSFFT's deep layers): one warp
// per node, same scores, same bound, same (min score, smallest t) result as the CTA
// kernel's single chunk — a 256-thread CTA per node left most threads idle there.
// 2048: DSFFT's depth-13 nodes (L = 2048) scan faster as one warp each than as one CTA
// each behind a seed kernel (config 4: 673 -> 708 signals/s, tools/dsfft_gpu_busy.py)
constexpr int kWarpSearchMaxL = 2048;
// the candidate count up to which the warp kernel scans (AFFT_WARP_SEARCH_MAXL, diagnostic)
static int64_t warp_search_maxl() {
  static const int64_t v = [] {
    const char* e = getenv("AFFT_WARP_SEARCH_MAXL");
    return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)kWarpSearchMaxL;
  }();
  return v;
}
constexpr int kWarpSearchWarps = 8;
// One node's exact argmin over its L candidates by one warp (lanes over candidates;
// s_est / s_e32 hold the node's stride estimates, `bad` any NaN / infinite one): the
// (min score, smallest t) of the CTA kernel's single chunk.
template <bool k32>
__device__ __forceinline__ void warp_search_node(int64_t n, int c, int64_t idx, int64_t b,
                                                 const double* s_est, const uint32_t* s_e32,
                                                 bool bad, int lane, double* best_out,
                                                 int32_t* bt_out) {
  const int64_t L = n / b;
  // one candidate per lane (L <= 32, DSFFT's deep layers): no pruning bound to seed
  // and no pre-filter to set up — both cost a candidate's worth of dependent work and
  // could only save part of one score; every candidate is scored in full instead
  const bool single = L <= 32;
  const ApproxScan ap = make_approx(n, L, idx, c, !bad && !single);  // see approx_pruned
  const double dn = (double)n;
  const double inv = 1.0 / dn;
  using rt = typename std::conditional<k32, uint32_t, int64_t>::type;
  double best = __longlong_as_double(0x7ff0000000000000LL);
  int32_t bt = INT32_MAX;
  double bound = single ? __longlong_as_double(0x7ff0000000000000LL)
                        : search_bound<k32>(n, b, L, idx, s_est, c, inv);
  // only the candidates the stride-0 term leaves possible under the seed bound
  const CandRanges cr = stride0_ranges(s_est[0], idx, n, L, bound, 0, L);
  const int64_t nv = cr.len();
  // the warp shares its pruning bound after every 32 candidates (see shared_bound)
  for (int64_t vb = 0; vb < nv; vb += 32) {
    const bool in = vb + lane < nv;
    const int64_t t = in ? cr.at(vb + lane) : L;
    uint32_t lim = 0;
    if (ap.on) lim = approx_limit(bound, ap.margin);
    if (in && !(lim && approx_pruned(ap.A0 + (uint64_t)t * ap.S, s_e32, c, lim))) {
      const double sc = cand_score<k32>((rt)(idx + b * t), (rt)n, s_est, c, dn, inv, bound);
      if (sc <= bound) {
        if (sc < best) {
          best = sc;
          bt = (int32_t)t;
        }
        bound = sc;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bound = fmin(bound, __shfl_xor_sync(0xffffffffu, bound, o));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (ob < best || (ob == best && ot < bt)) {
      best = ob;
      bt = ot;
    }
  }
  *best_out = best;
  *bt_out = bt;
}

// a node's stride estimates into the warp's shared copies (lanes over strides);
// returns whether any is NaN / infinite
__device__ __forceinline__ bool stage_estimates(const double* e_src, int c, int lane,
                                                double* s_est, uint32_t* s_e32) {
  bool bad = false;
  for (int j = lane; j < c; j += 32) {
    const double e = e_src[j];
    s_est[j] = e;
    double u = e * 0.15915494309189535;
    u -= floor(u);
    s_e32[j] = (uint32_t)(uint64_t)(u * 4294967296.0);
    bad |= !(e == e) || isinf(e);
  }
  bad = __any_sync(0xffffffffu, bad);
  __syncwarp();
  return bad;
}

template <bool k32>
__global__ void __launch_bounds__(kWarpSearchWarps * 32) noisy_search_warp_kernel(
    int64_t n, int c, int A, const int64_t* __restrict__ act_index,
    const int64_t* __restrict__ act_b, const double* __restrict__ est,
    double* __restrict__ part_score, int32_t* __restrict__ part_t,
    const int32_t* __restrict__ A_dev = nullptr) {
  if (A_dev) A = *A_dev;
  __shared__ double s_est_all[kWarpSearchWarps][kMaxStrides];
  __shared__ uint32_t s_e32_all[kWarpSearchWarps][kMaxStrides];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x * kWarpSearchWarps + wl;
  if (a >= A) return;  // whole warps only
  const bool bad = stage_estimates(est + (int64_t)a * c, c, lane, s_est_all[wl], s_e32_all[wl]);
  double best;
  int32_t bt;
  warp_search_node<k32>(n, c, act_index[a], act_b[a], s_est_all[wl], s_e32_all[wl], bad, lane,
                        &best, &bt);
  if (lane == 0) {
    part_score[a] = best;
    part_t[a] = bt;
  }
}

// Phase estimates of the active nodes (one thread per (node, stride)).
// A_dev (device-resident rounds): the active count as the prep kernel left it; the
// grid then covers the largest possible list and the excess threads exit.
// fill (per-node search of one cycle size, classify_noisy): the active list is the
// given nodes in order — row a, fill->index[a], fill->b — written here instead of by a
// separate list kernel.
struct EstFill {
  const int64_t* index;
  int64_t b;
  int64_t *act_row, *act_index, *act_b;
};
__global__ void noisy_est_kernel(int A, int c, int m, const int64_t* __restrict__ act_row,
                                 const double* __restrict__ residual, int R,
                                 const __grid_constant__ NoisyPlan P, double* __restrict__ est,
                                 unsigned long long* __restrict__ node_bound,
                                 const int32_t* __restrict__ A_dev = nullptr,
                                 EstFill fill = EstFill{nullptr, 0, nullptr, nullptr, nullptr}) {
  if (A_dev) A = *A_dev;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)A * c) return;
  const int64_t a = e / c;
  const int j = (int)(e - a * c);
  if (j == 0 && node_bound) node_bound[a] = ~0ull;  // "+inf" for the search kernel
  if (j == 0 && fill.index) {
    fill.act_row[a] = a;
    fill.act_index[a] = fill.index[a];
    fill.act_b[a] = fill.b;
  }
  const int64_t row = fill.index ? a : act_row[a];
  const cd* y = reinterpret_cast<const cd*>(residual) + row * R + (int64_t)j * m;
  est[e] = stride_estimate(y, m, P.w);
}

// Reduce the chunk partials, then the least-squares fit (peeling.py:247-250):
// x = a^H y / a^H a with a_r = exp(-2j*pi*((tau_r*f0) mod n)/n), resnorm = ||a x - y||.
// One warp per active node.
__device__ __forceinline__ double node_norm(const cd* y, int R);

// decide != null: also classify_noisy's decision for nodes searched unconditionally
// (peeling.py:257-267): ZERO_TON if ||y|| <= t0, else SINGLE_TON iff resnorm <= t1.
struct NoisyDecide {
  int8_t* state;
  double t0, t1;
  const double* t0s;  // per-signal gates (signal of the row), overriding t0 / t1
  const double* t1s;
};

// The fit (peeling.py:247-250) and classify_noisy's decision (257-267) for node a of
// the active list, one warp (lane, wl = its warp within a 256-thread CTA's nsq rows),
// from the search's winner t = bt.
__device__ __forceinline__ void finalize_node(int a, int lane, int wl, int32_t bt,
                                              const int64_t* __restrict__ act_row,
                                              const int64_t* __restrict__ act_index,
                                              const int64_t* __restrict__ act_b,
                                              const double* __restrict__ residual,
                                              const NoisyPlan& P, int64_t* __restrict__ out_f0,
                                              double* __restrict__ out_val,
                                              double* __restrict__ out_res,
                                              const NoisyDecide& decide,
                                              double (*nsq)[2][128]) {
  constexpr int kNormRows = 128;
  if (bt == INT32_MAX) bt = 0;  // all-NaN scores: numpy argmin would return the first NaN
  const int64_t n = P.n;
  // index < b and t < n / b, so the candidate is already reduced (no '% n')
  const int64_t f0 = act_index[a] + act_b[a] * (int64_t)bt;
  const cd* y = reinterpret_cast<const cd*>(residual) + act_row[a] * P.R;
  const int64_t sig = plan_row_signal(P, act_row[a]);
  // a^H y and a^H a; each lane's atoms kept for the residual (one sincos per row)
  constexpr int kAtomRegs = 4;  // rows lane, lane + 32, ... cached up to R = 128
  cd atc[kAtomRegs];
  double nre = 0.0, nim = 0.0, den = 0.0;
#pragma unroll
  for (int q = 0; q < kAtomRegs; ++q) atc[q] = cd{0.0, 0.0};
  for (int r = lane, q = 0; r < P.R; r += 32, ++q) {
    const cd at = unit_root(plan_mulmod(P, plan_tau(P, sig, r), f0), n);
#pragma unroll
    for (int qq = 0; qq < kAtomRegs; ++qq)
      if (qq == q) atc[qq] = at;
    const cd yv = y[r];
    if (decide.state && P.R <= kNormRows) {
      nsq[wl][0][r] = __dmul_rn(yv.re, yv.re);
      nsq[wl][1][r] = __dmul_rn(yv.im, yv.im);
    }
    nre += at.re * yv.re + at.im * yv.im;
    nim += at.re * yv.im - at.im * yv.re;
    den += at.re * at.re + at.im * at.im;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nre += __shfl_xor_sync(0xffffffffu, nre, o);
    nim += __shfl_xor_sync(0xffffffffu, nim, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  const cd x = cd{nre / den, nim / den};
  double rs = 0.0;
  for (int r = lane, q = 0; r < P.R; r += 32, ++q) {
    cd at = q < kAtomRegs ? cd{0.0, 0.0} : unit_root(plan_mulmod(P, plan_tau(P, sig, r), f0), n);
#pragma unroll
    for (int qq = 0; qq < kAtomRegs; ++qq)
      if (qq == q) at = atc[qq];
    const cd d = csub(cmul(at, x), y[r]);
    rs += d.re * d.re + d.im * d.im;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  if (lane == 0) {
    out_f0[a] = f0;
    reinterpret_cast<cd*>(out_val)[a] = x;
    const double resn = sqrt(rs);
    out_res[a] = resn;
  }
  if (decide.state) {
    double nrm;
    if (P.R <= kNormRows) {
      __syncwarp();
      double sre = 0.0, sim = 0.0;
      if (lane == 0) {
        for (int r = 0; r < P.R; ++r) sre = __dadd_rn(sre, nsq[wl][0][r]);
        for (int r = 0; r < P.R; ++r) sim = __dadd_rn(sim, nsq[wl][1][r]);
      }
      nrm = sqrt(__dadd_rn(sre, sim));
    } else {
      nrm = lane == 0 ? node_norm(y, P.R) : 0.0;
    }
    if (lane == 0)
      decide.state[a] = nrm <= (decide.t0s ? decide.t0s[sig] : decide.t0) ? AFFT_ZERO_TON
                        : out_res[a] <= (decide.t1s ? decide.t1s[sig] : decide.t1)
                            ? AFFT_SINGLE_TON
                                                  : AFFT_MULTI_TON;
  }
}

__global__ void noisy_finalize_kernel(int A, int chunks, const double* __restrict__ part_score,
                                      const int32_t* __restrict__ part_t,
                                      const int64_t* __restrict__ act_row,
                                      const int64_t* __restrict__ act_index,
                                      const int64_t* __restrict__ act_b,
                                      const double* __restrict__ residual,
                                      const __grid_constant__ NoisyPlan P,
                                      int64_t* __restrict__ out_f0, double* __restrict__ out_val,
                                      double* __restrict__ out_res, NoisyDecide decide,
                                      const int32_t* __restrict__ A_dev = nullptr) {
  if (A_dev) A = *A_dev;
  // classify's zero-ton gate needs ||y||: the squares land in shared memory while the
  // rows are loaded, and lane 0 sums them in node_norm's order (not 2 x R dependent
  // global loads on one lane — 30% of this kernel's instructions and its latency chain)
  __shared__ double nsq[8][2][128];  // blockDim 256: per warp, finalize_node's squares
  const int a = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31, wl = (threadIdx.x >> 5) & 7;
  if (a >= A) return;
  double best = __longlong_as_double(0x7ff0000000000000LL);
  int32_t bt = INT32_MAX;
  for (int ch = lane; ch < chunks; ch += 32) {
    const double sc = part_score[(int64_t)a * chunks + ch];
    const int32_t t = part_t[(int64_t)a * chunks + ch];
    if (sc < best || (sc == best && t < bt)) {
      best = sc;
      bt = t;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (ob < best || (ob == best && ot < bt)) {
      best = ob;
      bt = ot;
    }
  }
  finalize_node(a, lane, wl, bt, act_row, act_index, act_b, residual, P, out_f0, out_val, out_res,
                decide, nsq);
}

// classify_noisy for short candidate lists in one launch (DSFFT's layers, n/b <= 2048):
// one warp per node does the stride estimates (lanes over strides, stride_estimate as
// noisy_est_kernel), the candidate scan (warp_search_node) and the fit + decision
// (finalize_node) — the est -> warp search -> finalize sequence without its two extra
// launches and the partials' round trip through memory; the same arithmetic, so the same
// results.
template <bool k32>
__global__ void __launch_bounds__(kWarpSearchWarps * 32) noisy_classify_warp_kernel(
    const __grid_constant__ NoisyPlan P, int A, const int64_t* __restrict__ act_row,
    const int64_t* __restrict__ act_index, const int64_t* __restrict__ act_b,
    const double* __restrict__ residual, EstFill fill, int64_t* __restrict__ out_f0,
    double* __restrict__ out_val, double* __restrict__ out_res, NoisyDecide decide) {
  static_assert(kWarpSearchWarps == 8, "finalize_node's squares: 8 warps per CTA");
  __shared__ double s_est_all[kWarpSearchWarps][kMaxStrides];
  __shared__ uint32_t s_e32_all[kWarpSearchWarps][kMaxStrides];
  __shared__ double nsq[8][2][128];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x * kWarpSearchWarps + wl;
  if (a >= A) return;  // whole warps only
  if (fill.index) {
    if (lane == 0) {
      fill.act_row[a] = a;
      fill.act_index[a] = fill.index[a];
      fill.act_b[a] = fill.b;
    }
    __syncwarp();  // finalize_node reads the lists back
  }
  const int64_t row = fill.index ? a : act_row[a];
  const cd* y = reinterpret_cast<const cd*>(residual) + row * P.R;
  double* s_est = s_est_all[wl];
  uint32_t* s_e32 = s_e32_all[wl];
  bool bad = false;
  for (int j = lane; j < P.c; j += 32) {
    const double e = stride_estimate(y + (int64_t)j * P.m, P.m, P.w);
    s_est[j] = e;
    double u = e * 0.15915494309189535;
    u -= floor(u);
    s_e32[j] = (uint32_t)(uint64_t)(u * 4294967296.0);
    bad |= !(e == e) || isinf(e);
  }
  bad = __any_sync(0xffffffffu, bad);
  __syncwarp();
  const int64_t idx = fill.index ? fill.index[a] : act_index[a];
  const int64_t b = fill.index ? fill.b : act_b[a];
  double best;
  int32_t bt;
  warp_search_node<k32>(P.n, P.c, idx, b, s_est, s_e32, bad, lane, &best, &bt);
  finalize_node(a, lane, wl, bt, fill.index ? fill.act_row : act_row,
                fill.index ? fill.act_index : act_index, fill.index ? fill.act_b : act_b,
                residual, P, out_f0, out_val, out_res, decide, nsq);
}

// -------------------------------------------------------------- decoder rounds

__device__ __forceinline__ double node_norm(const cd* y, int R) {
  double sre = 0.0, sim = 0.0;
  for (int r = 0; r < R; ++r) sre = __dadd_rn(sre, __dmul_rn(y[r].re, y[r].re));
  for (int r = 0; r < R; ++r) sim = __dadd_rn(sim, __dmul_rn(y[r].im, y[r].im));
  return sqrt(__dadd_rn(sre, sim));
}

// classify_noisy's zero-ton gate (peeling.py:257-259) for every live, changed
// node of every unfinished signal; survivors join the active list.
__global__ void noisy_prep_kernel(int64_t batch, const __grid_constant__ NoisyPlan P,
                                  const double* __restrict__ residual, int8_t* __restrict__ state,
                                  int8_t* __restrict__ dirty, const int32_t* __restrict__ done,
                                  const double* __restrict__ t0, int32_t* __restrict__ counter,
                                  int64_t* __restrict__ act_row, int64_t* __restrict__ act_index,
                                  int64_t* __restrict__ act_b) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= batch * P.nodes) return;
  const int64_t s = e / P.nodes;
  const int g = (int)(e - s * P.nodes);
  if (done[s]) return;
  const int8_t st = state[e];
  if (st == AFFT_RESOLVED || st == AFFT_ZERO_TON || !dirty[e]) return;
  const cd* y = reinterpret_cast<const cd*>(residual) + e * P.R;
  if (node_norm(y, P.R) <= t0[s]) {
    state[e] = AFFT_ZERO_TON;
    dirty[e] = 0;
    return;
  }
  const int slot = atomicAdd(counter, 1);
  const int c = noisy_cycle(P, g);
  act_row[slot] = e;
  act_index[slot] = g - P.base[c];
  act_b[slot] = P.b[c];
}

// SINGLE_TON iff resnorm <= T1 (peeling.py:260-267).
__global__ void noisy_apply_kernel(int A, const __grid_constant__ NoisyPlan P,
                                   const int64_t* __restrict__ act_row,
                                   const int64_t* __restrict__ f0s, const double* __restrict__ vals,
                                   const double* __restrict__ res, const double* __restrict__ t1,
                                   int8_t* __restrict__ state, int8_t* __restrict__ dirty,
                                   int64_t* __restrict__ node_f0, double* __restrict__ node_val,
                                   const int32_t* __restrict__ A_dev = nullptr) {
  if (A_dev) A = *A_dev;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int64_t e = act_row[a];
  const int64_t s = e / P.nodes;
  dirty[e] = 0;
  if (res[a] <= t1[s]) {
    state[e] = AFFT_SINGLE_TON;
    node_f0[e] = f0s[a];
    reinterpret_cast<cd*>(node_val)[e] = reinterpret_cast<const cd*>(vals)[a];
  } else {
    state[e] = AFFT_MULTI_TON;
  }
}

// Harvest (first-found) + subtract for one signal per CTA (peeling.py:296-308).
__global__ void __launch_bounds__(1024) noisy_harvest_kernel(
    const __grid_constant__ NoisyPlan P, double* __restrict__ residual, int8_t* __restrict__ state,
    int8_t* __restrict__ dirty, const int64_t* __restrict__ node_f0,
    const double* __restrict__ node_val, int32_t* __restrict__ done, int64_t* __restrict__ rec_pos,
    double* __restrict__ rec_val, int rec_cap, int32_t* __restrict__ rec_count,
    int32_t* __restrict__ rounds, int32_t* __restrict__ total_found, char* gscratch,
    size_t scratch_bytes, int32_t* __restrict__ nf_round = nullptr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry;
  const int64_t s = blockIdx.x;
  // nf_round (global harvest state only): the subtraction is left to
  // noisy_subtract_kernel, which reads this round's tone count per signal
  if (done[s]) {
    if (nf_round && threadIdx.x == 0) nf_round[s] = 0;
    return;
  }
  const int N = P.nodes;
  const int tid = threadIdx.x, nt = blockDim.x;
  unsigned char* mem = gscratch ? reinterpret_cast<unsigned char*>(gscratch) + s * scratch_bytes
                                : smem_raw;
  unsigned* hash = reinterpret_cast<unsigned*>(mem);
  int* flag = reinterpret_cast<int*>(hash + P.hmask + 1);
  int32_t* found_g = flag + N;
  int32_t* found_res = found_g + N;          // [nf][ncycles]
  int8_t* hv = reinterpret_cast<int8_t*>(found_res + (size_t)N * P.ncycles);
  const int64_t so = s * N;
  int64_t* rpos = rec_pos + s * (int64_t)rec_cap;
  cd* rval = reinterpret_cast<cd*>(rec_val) + s * (int64_t)rec_cap;
  const int rc = rec_count[s];
  for (int h = tid; h <= P.hmask; h += nt) hash[h] = kEmpty;
  for (int g = tid; g < N; g += nt) hv[g] = 0;
  __syncthreads();
  for (int i = tid; i < rc; i += nt) hash_insert(hash, P.hmask, rpos[i]);
  if (tid == 0) rounds[s] += 1;
  __syncthreads();
  for (int g = tid; g < N; g += nt) {
    int take = 0;
    if (state[so + g] == AFFT_SINGLE_TON) {
      const int64_t f = node_f0[so + g];
      if (!hash_contains(hash, P.hmask, f)) {
        take = 1;
        const int c = noisy_cycle(P, g);
        for (int c2 = 0; c2 < c; ++c2) {
          const int g2 = P.base[c2] + (int)mod_nonneg(f, P.b[c2]);
          if (state[so + g2] == AFFT_SINGLE_TON && node_f0[so + g2] == f) {
            take = 0;
            break;
          }
        }
      }
    }
    flag[g] = take;
    if (take) hv[g] = 1;
  }
  __syncthreads();
  const int nf = block_exclusive_scan(flag, N, warp_tmp, &carry);
  if (tid == 0 && nf_round) nf_round[s] = nf;
  if (nf == 0) {
    if (tid == 0) done[s] = 1;
    return;
  }
  for (int g = tid; g < N; g += nt) {
    if (hv[g]) {
      found_g[flag[g]] = g;
      hv[g] = 0;
    }
  }
  __syncthreads();
  for (int i = tid; i < nf; i += nt) state[so + found_g[i]] = AFFT_RESOLVED;
  for (int g = tid; g < N; g += nt) flag[g] = 0;
  __syncthreads();
  // per-node lists of the found tones hitting it: count, scan, scatter
  const int F = P.ncycles;
  for (int e = tid; e < nf * F; e += nt) {
    const int i = e / F, c = e - i * F;
    atomicAdd(&flag[P.base[c] + (int)mod_nonneg(node_f0[so + found_g[i]], P.b[c])], 1);
  }
  __syncthreads();
  block_exclusive_scan(flag, N, warp_tmp, &carry);
  for (int e = tid; e < nf * F; e += nt) {
    const int i = e / F, c = e - i * F;
    const int slot =
        atomicAdd(&flag[P.base[c] + (int)mod_nonneg(node_f0[so + found_g[i]], P.b[c])], 1);
    found_res[slot] = i;
  }
  __syncthreads();
  // subtract: one warp per hit node, lanes over the R measurements, tones in found order
  // (here for graphs whose harvest state fits in shared memory; else one warp per node
  // across the whole grid in noisy_subtract_kernel — one CTA per signal left C3′'s
  // 23.5 k-node subtraction on 16 SMs)
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int g = wid; g < N && !nf_round; g += nw) {
    const int lo = g ? flag[g - 1] : 0, hi = flag[g];
    if (lo == hi) continue;
    if (lane == 0) {  // insertion sort of the (short) segment restores found order
      for (int a2 = lo + 1; a2 < hi; ++a2) {
        const int v = found_res[a2];
        int b2 = a2 - 1;
        while (b2 >= lo && found_res[b2] > v) {
          found_res[b2 + 1] = found_res[b2];
          --b2;
        }
        found_res[b2 + 1] = v;
      }
    }
    __syncwarp();
    cd* y = reinterpret_cast<cd*>(residual) + (so + g) * P.R;
    for (int r = lane; r < P.R; r += 32) {
      cd acc = y[r];
      for (int a2 = lo; a2 < hi; ++a2) {
        const int i = found_res[a2];
        const int64_t f = node_f0[so + found_g[i]];
        const cd v = reinterpret_cast<const cd*>(node_val)[so + found_g[i]];
        acc = csub(acc, cmul(v, unit_root(plan_mulmod(P, plan_tau(P, s, r), f), P.n)));
      }
      y[r] = acc;
    }
    if (lane == 0) dirty[so + g] = 1;
  }
  for (int i = tid; i < nf; i += nt) {
    rpos[rc + i] = node_f0[so + found_g[i]];
    rval[rc + i] = reinterpret_cast<const cd*>(node_val)[so + found_g[i]];
  }
  if (tid == 0) {
    rec_count[s] = rc + nf;
    atomicAdd(total_found, nf);
  }
}

// noisy_harvest_kernel's subtraction for global harvest state: grid (node blocks, signal),
// one warp per node, the same per-node tone lists (flag = segment ends after the
// scatter, found_res, found_g in the signal's scratch block) and the same arithmetic in
// the same order.
__global__ void __launch_bounds__(256) noisy_subtract_kernel(
    const __grid_constant__ NoisyPlan P, double* __restrict__ residual,
    int8_t* __restrict__ dirty, const int64_t* __restrict__ node_f0,
    const double* __restrict__ node_val, const int32_t* __restrict__ nf_round, char* gscratch,
    size_t scratch_bytes) {
  const int64_t s = blockIdx.y;
  if (nf_round[s] == 0) return;
  const int N = P.nodes;
  const int lane = threadIdx.x & 31;
  const int g = (int)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (g >= N) return;
  unsigned char* mem = reinterpret_cast<unsigned char*>(gscratch) + s * scratch_bytes;
  unsigned* hash = reinterpret_cast<unsigned*>(mem);
  const int* flag = reinterpret_cast<const int*>(hash + P.hmask + 1);
  const int32_t* found_g = flag + N;
  int32_t* found_res = const_cast<int32_t*>(found_g) + N;
  const int lo = g ? flag[g - 1] : 0, hi = flag[g];
  if (lo == hi) return;
  const int64_t so = s * N;
  if (lane == 0) {  // insertion sort of the (short) segment restores found order
    for (int a2 = lo + 1; a2 < hi; ++a2) {
      const int v = found_res[a2];
      int b2 = a2 - 1;
      while (b2 >= lo && found_res[b2] > v) {
        found_res[b2 + 1] = found_res[b2];
        --b2;
      }
      found_res[b2 + 1] = v;
    }
  }
  __syncwarp();
  cd* y = reinterpret_cast<cd*>(residual) + (so + g) * P.R;
  for (int r = lane; r < P.R; r += 32) {
    cd acc = y[r];
    for (int a2 = lo; a2 < hi; ++a2) {
      const int i = found_res[a2];
      const int64_t f = node_f0[so + found_g[i]];
      const cd v = reinterpret_cast<const cd*>(node_val)[so + found_g[i]];
      acc = csub(acc, cmul(v, unit_root(plan_mulmod(P, plan_tau(P, s, r), f), P.n)));
    }
    y[r] = acc;
  }
  if (lane == 0) dirty[so + g] = 1;
}

__global__ void count_multi_kernel(int64_t batch, int N, const int8_t* __restrict__ state,
                                   int32_t* __restrict__ unresolved) {
  const int64_t s = blockIdx.x;
  int cnt = 0;
  for (int g = threadIdx.x; g < N; g += blockDim.x) cnt += state[s * N + g] == AFFT_MULTI_TON;
  __shared__ int red;
  if (threadIdx.x == 0) red = 0;
  __syncthreads();
  atomicAdd(&red, cnt);
  __syncthreads();
  if (threadIdx.x == 0) unresolved[s] = red;
}

// -------------------------------------------------------------- thresholds

// energies[e] = ||vec_e||^2 (peeling.py:355-357: float(norm(vec) ** 2))
__global__ void node_energy_kernel(int64_t count, int R, const double* __restrict__ vec,
                                   double* __restrict__ energy) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  const double nv = node_norm(reinterpret_cast<const cd*>(vec) + e * R, R);
  energy[e] = __dmul_rn(nv, nv);
}

// robust_thresholds (peeling.py:335-351) per signal: median of the masked
// energies (all when mask is null), floor from the max of all energies.
__global__ void robust_thresholds_kernel(int count, int pow2, const double* __restrict__ energy,
                                         const uint8_t* __restrict__ mask, int r,
                                         double* __restrict__ t0, double* __restrict__ t1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* v = reinterpret_cast<double*>(smem_raw);
  __shared__ int m_count;
  __shared__ double m_max;
  const int64_t s = blockIdx.x;
  const double* E = energy + s * (int64_t)count;
  const uint8_t* M = mask ? mask + s * (int64_t)count : nullptr;
  // the reference set and max(initial=0.0) in parallel: the set's order is irrelevant
  // (it is sorted next), and fmax is order-independent (a serial thread-0 loop over
  // the global energies was most of this kernel's 50 us per signal)
  __shared__ double w_max[32];
  if (threadIdx.x == 0) m_count = 0;
  __syncthreads();
  double mx = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const double e = E[i];
    mx = fmax(mx, e);
    if (!M || M[i]) v[atomicAdd(&m_count, 1)] = e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) w_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, w_max[w]);
    m_max = r;
  }
  if (M && m_count == 0) {  // empty reference set: fall back to all energies
    for (int i = threadIdx.x; i < count; i += blockDim.x) v[i] = E[i];
    __syncthreads();
    if (threadIdx.x == 0) m_count = count;
  }
  __syncthreads();
  const int cnt = m_count;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int i = cnt + threadIdx.x; i < pow2; i += blockDim.x) v[i] = inf;
  __syncthreads();
  // bitonic sort ascending
  for (int k = 2; k <= pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const double a = v[i], b = v[ixj];
          if ((a > b) == up) {
            v[i] = b;
            v[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    double med;
    if (cnt == 0) med = __longlong_as_double(0x7ff8000000000000LL);
    else if (cnt & 1) med = v[cnt / 2];
    else med = (v[cnt / 2 - 1] + v[cnt / 2]) / 2.0;  // np.mean of the two middles
    const double sigma = sqrt(fmax(med, 0.0) / (double)r);
    const double floor_ = 1e-8 * sqrt(m_max);
    const double base = sigma * sqrt((double)r);
    t0[s] = fmax(1.5 * base, floor_);
    t1[s] = fmax(2.5 * base, floor_);
  }
}

// k-th smallest (0-based) of cnt non-negative doubles by 8-bit radix select on the
// IEEE bit patterns (order-preserving for values >= +0).  One CTA, global data.
__device__ double radix_select(const double* v, int cnt, int kth, unsigned* hist) {
  __shared__ unsigned long long prefix;
  __shared__ int remaining;
  if (threadIdx.x == 0) {
    prefix = 0ull;
    remaining = kth;
  }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const unsigned long long pre = prefix;
    const unsigned long long mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(v[i]);
      if ((bits & mask) == pre) atomicAdd(&hist[(bits >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int r = remaining;
      unsigned d = 0;
      while (d < 255 && r >= (int)hist[d]) {
        r -= (int)hist[d];
        ++d;
      }
      remaining = r;
      prefix = pre | ((unsigned long long)d << shift);
    }
    __syncthreads();
  }
  return __longlong_as_double((long long)prefix);
}

__global__ void robust_thresholds_large_kernel(int count, const double* __restrict__ energy,
                                               const uint8_t* __restrict__ mask, int r,
                                               double* __restrict__ scratch,
                                               double* __restrict__ t0, double* __restrict__ t1) {
  __shared__ unsigned hist[256];
  __shared__ int m_count;
  __shared__ double m_max;
  const int64_t s = blockIdx.x;
  const double* E = energy + s * (int64_t)count;
  const uint8_t* M = mask ? mask + s * (int64_t)count : nullptr;
  double* v = scratch + s * (int64_t)count;
  // max over all energies and the (masked) median set, compacted in parallel
  // (order is irrelevant to a selection)
  __shared__ int m_fill;
  if (threadIdx.x == 0) {
    m_fill = 0;
    m_max = 0.0;
  }
  __syncthreads();
  double mx = 0.0;  // scale.max(initial=0.0)
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    mx = fmax(mx, E[i]);
    if (!M || M[i]) v[atomicAdd(&m_fill, 1)] = E[i];
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&m_max), (unsigned long long)__double_as_longlong(mx));
  __syncthreads();
  if (threadIdx.x == 0) m_count = m_fill;
  __syncthreads();
  if (M && m_count == 0) {  // empty reference set: fall back to all energies
    for (int i = threadIdx.x; i < count; i += blockDim.x) v[i] = E[i];
    __syncthreads();
    if (threadIdx.x == 0) m_count = count;
    __syncthreads();
  }
  const int cnt = m_count;
  double med;
  if (cnt & 1) {
    med = radix_select(v, cnt, cnt / 2, hist);
  } else {
    const double lo = radix_select(v, cnt, cnt / 2 - 1, hist);
    const double hi = radix_select(v, cnt, cnt / 2, hist);
    med = (lo + hi) / 2.0;
  }
  if (threadIdx.x == 0) {
    const double sigma = sqrt(fmax(med, 0.0) / (double)r);
    const double floor_ = 1e-8 * sqrt(m_max);
    const double base = sigma * sqrt((double)r);
    t0[s] = fmax(1.5 * base, floor_);
    t1[s] = fmax(2.5 * base, floor_);
  }
}

// -------------------------------------------------------------- host side

static int make_noisy_plan(NoisyPlan* P, int64_t n, const int64_t* factors, int ncycles,
                           const int64_t* shifts, int R, int c, int m, const double* weights,
                           int rec_cap) {
  memset(P, 0, sizeof(*P));
  if (n < 1 || n > 2000000000LL) {
    set_error("signal size %lld outside the supported 1..2e9", (long long)n);
    return AFFT_EUNSUPPORTED;
  }
  if (c < 1 || c > kMaxStrides || m < 2 || m > kMaxRounds || R != c * m || R > AFFT_MAX_SHIFTS) {
    set_error("search plan c=%d m=%d R=%d unsupported", c, m, R);
    return AFFT_EUNSUPPORTED;
  }
  if (ncycles < 1 || ncycles > AFFT_MAX_CYCLES) {
    set_error("number of cycles %d outside 1..%d", ncycles, AFFT_MAX_CYCLES);
    return AFFT_EUNSUPPORTED;
  }
  P->n = n;
  P->ncycles = ncycles;
  P->R = R;
  P->c = c;
  P->m = m;
  int64_t total = 0;
  for (int k = 0; k < ncycles; ++k) {
    if (factors[k] < 1 || n % factors[k]) {
      set_error("bucket count %lld does not divide signal size %lld", (long long)factors[k],
                (long long)n);
      return AFFT_EINVAL;
    }
    P->b[k] = factors[k];
    P->base[k] = (int32_t)total;
    total += factors[k];
  }
  if (total > (1LL << 30)) {
    set_error("graph with %lld nodes is too large", (long long)total);
    return AFFT_EUNSUPPORTED;
  }
  for (int k = ncycles; k <= AFFT_MAX_CYCLES; ++k) P->base[k] = INT32_MAX;
  P->base[ncycles] = (int32_t)total;
  P->nodes = (int)total;
  for (int t = 0; t < m - 1; ++t) P->w[t] = weights[t];
  for (int r = 0; r < R; ++r) P->tau[r] = host_pymod(shifts[r], n);
  P->nmagic = ~0ull / (uint64_t)n;
  int hcap = 16;
  while (hcap < 2 * std::max(rec_cap, 1)) hcap <<= 1;
  P->hmask = hcap - 1;
  return AFFT_OK;
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct NoisyWs {
  size_t est, act_row, act_index, act_b, part_s, part_t, f0, val, res, dirty, done, counters,
      bound, total;
  int chunks;
  int64_t Lmax;  // largest candidate count n / b over the cycles
};

static NoisyWs noisy_ws(const NoisyPlan& P, int64_t rows) {
  NoisyWs w;
  int64_t bmin = P.b[0];
  for (int k = 1; k < P.ncycles; ++k) bmin = std::min(bmin, P.b[k]);
  const int64_t Lmax = P.n / bmin;
  w.Lmax = Lmax;
  w.chunks = (int)((Lmax + kChunk - 1) / kChunk);
  size_t o = 0;
  w.est = o;       o = al256(o + (size_t)rows * P.c * 8);
  w.act_row = o;   o = al256(o + (size_t)rows * 8);
  w.act_index = o; o = al256(o + (size_t)rows * 8);
  w.act_b = o;     o = al256(o + (size_t)rows * 8);
  w.part_s = o;    o = al256(o + (size_t)rows * w.chunks * 8);
  w.part_t = o;    o = al256(o + (size_t)rows * w.chunks * 4);
  w.f0 = o;        o = al256(o + (size_t)rows * 8);
  w.val = o;       o = al256(o + (size_t)rows * 16);
  w.res = o;       o = al256(o + (size_t)rows * 8);
  w.dirty = o;     o = al256(o + (size_t)rows);
  w.done = o;      o = al256(o + (size_t)rows * 4);
  w.counters = o;  o = al256(o + 64);
  w.bound = o;     o = al256(o + (size_t)rows * 8);
  w.total = o;
  return w;
}

// est → scan → reduce + LS fit for A active rows already listed in the workspace.
__global__ void part_fill_kernel(int64_t count, double* __restrict__ part_score,
                                 int32_t* __restrict__ part_t) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    part_score[i] = __longlong_as_double(0x7ff0000000000000LL);  // +inf: not this rank's
    part_t[i] = INT32_MAX;
  }
}

// Rewrite the active list from rows sorted ascending (keys[a] = row): the prep kernel
// compacts with an atomic, so slot order differs from run to run and rank to rank —
// harmless for one rank, but a split search exchanges partials by slot.
__global__ void act_from_rows_kernel(int A, const __grid_constant__ NoisyPlan P,
                                     const int64_t* __restrict__ rows, int64_t* __restrict__ act_row,
                                     int64_t* __restrict__ act_index, int64_t* __restrict__ act_b) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int64_t e = rows[a];
  const int g = (int)(e % P.nodes);
  const int c = noisy_cycle(P, g);
  act_row[a] = e;
  act_index[a] = g - P.base[c];
  act_b[a] = P.b[c];
}

static int canonical_active(const NoisyPlan& P, const NoisyWs& w, char* ws, int A,
                            int64_t rows_total, cudaStream_t st) {
  int64_t* act_row = reinterpret_cast<int64_t*>(ws + w.act_row);
  int bits = 1;
  while (bits < 63 && (int64_t(1) << bits) < rows_total) ++bits;
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, temp, act_row, act_row, A, 0, bits, st);
  char* buf = nullptr;
  const size_t keys_bytes = ((size_t)A * 8 + 255) & ~size_t(255);
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&buf), keys_bytes + temp, st);
  if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(search shard sort)");
  int64_t* sorted = reinterpret_cast<int64_t*>(buf);
  e = cub::DeviceRadixSort::SortKeys(buf + keys_bytes, temp, act_row, sorted, A, 0, bits, st);
  if (e == cudaSuccess) {
    act_from_rows_kernel<<<(unsigned)((A + 255) / 256), 256, 0, st>>>(
        A, P, sorted, act_row, reinterpret_cast<int64_t*>(ws + w.act_index),
        reinterpret_cast<int64_t*>(ws + w.act_b));
    e = cudaGetLastError();
  }
  scratch_free(buf, st);
  return e == cudaSuccess ? AFFT_OK : cuda_status(e, "search shard active-list sort");
}

// est -> scan -> (exchange) -> reduce + LS fit.  With a shard of world W > 1 this rank
// scans the chunks ch = rank (mod W) of every active node, the other slots hold
// (+inf, INT32_MAX), and the caller's exchange replaces every slot by its minimum over
// the ranks (score and t independently: exactly one rank holds a real value per slot),
// after which the reduction and fit are the single-rank ones — identical results.
struct SearchOut {  // null members: the workspace slots
  int64_t* f0 = nullptr;
  double* val = nullptr;
  double* res = nullptr;
  NoisyDecide decide = {nullptr, 0.0, 0.0};
};

// AFFT_FUSED_CLASSIFY=0: estimates, warp scan and fit as three launches (diagnostic)
static bool fused_classify_on() {
  const char* e = getenv("AFFT_FUSED_CLASSIFY");
  return !(e && e[0] == '0');
}

static int run_search(const NoisyPlan& P, const NoisyWs& w, char* ws, int A,
                      const double* residual, cudaStream_t st,
                      const AfftSearchShard* shard = nullptr, int64_t rows_total = 0,
                      const SearchOut& out = SearchOut(), const int64_t* fill_index = nullptr,
                      int64_t fill_b = 0) {
  if (A == 0) return AFFT_OK;
  const int rank = shard && shard->world > 1 ? shard->rank : 0;
  const int world = shard && shard->world > 1 ? shard->world : 1;
  if (world > 1) {  // every rank must list the active nodes in the same order
    const int rc = canonical_active(P, w, ws, A, rows_total, st);
    if (rc) return rc;
  }
  const int64_t* act_row = reinterpret_cast<const int64_t*>(ws + w.act_row);
  const int64_t* act_index = reinterpret_cast<const int64_t*>(ws + w.act_index);
  const int64_t* act_b = reinterpret_cast<const int64_t*>(ws + w.act_b);
  double* est = reinterpret_cast<double*>(ws + w.est);
  const int64_t ne = (int64_t)A * P.c;
  unsigned long long* node_bound = reinterpret_cast<unsigned long long*>(ws + w.bound);
  EstFill fill{fill_index, fill_b, const_cast<int64_t*>(act_row),
               const_cast<int64_t*>(act_index), const_cast<int64_t*>(act_b)};
  if (!fill_index) fill = EstFill{nullptr, 0, nullptr, nullptr, nullptr};
  if (world == 1 && w.Lmax <= warp_search_maxl() && fused_classify_on()) {
    // one warp per node does estimates, scan and fit in one launch
    auto kfn = P.n < (int64_t(1) << 31) ? noisy_classify_warp_kernel<true>
                                        : noisy_classify_warp_kernel<false>;
    kfn<<<(unsigned)((A + kWarpSearchWarps - 1) / kWarpSearchWarps), kWarpSearchWarps * 32, 0,
          st>>>(P, A, act_row, act_index, act_b, residual, fill,
                out.f0 ? out.f0 : reinterpret_cast<int64_t*>(ws + w.f0),
                out.val ? out.val : reinterpret_cast<double*>(ws + w.val),
                out.res ? out.res : reinterpret_cast<double*>(ws + w.res), out.decide);
    AFFT_CHECK_LAUNCH("noisy_classify_warp_kernel");
    return AFFT_OK;
  }
  noisy_est_kernel<<<(unsigned)((ne + 127) / 128), 128, 0, st>>>(A, P.c, P.m, act_row, residual,
                                                                P.R, P, est, node_bound, nullptr,
                                                                fill);
  AFFT_CHECK_LAUNCH("noisy_est_kernel");
  double* part_s = reinterpret_cast<double*>(ws + w.part_s);
  int32_t* part_t = reinterpret_cast<int32_t*>(ws + w.part_t);
  const int64_t nparts = (int64_t)A * w.chunks;
  if (world > 1)
    part_fill_kernel<<<(unsigned)((nparts + 255) / 256), 256, 0, st>>>(nparts, part_s, part_t);
  const int mine = (w.chunks - rank + world - 1) / world;
  if (world == 1 && w.Lmax <= warp_search_maxl()) {  // one chunk: part slot a = node a
    auto kfn = P.n < (int64_t(1) << 31) ? noisy_search_warp_kernel<true>
                                        : noisy_search_warp_kernel<false>;
    kfn<<<(unsigned)((A + kWarpSearchWarps - 1) / kWarpSearchWarps), kWarpSearchWarps * 32, 0,
          st>>>(P.n, P.c, A, act_index, act_b, est, part_s, part_t, nullptr);
  } else {
    if (mine > 0) {
      auto sfn = P.n < (int64_t(1) << 31) ? noisy_seed_kernel<true> : noisy_seed_kernel<false>;
      sfn<<<(unsigned)((A + 127) / 128), 128, 0, st>>>(P.n, P.c, A, act_index, act_b, est,
                                                         node_bound, nullptr);
    }
    for (int a0 = 0; a0 < A && mine > 0; a0 += 65535) {
      const int cnt = std::min(65535, A - a0);
      dim3 grid((unsigned)mine, (unsigned)cnt);
      auto kfn =
          P.n < (int64_t(1) << 31) ? noisy_search_kernel<true> : noisy_search_kernel<false>;
      kfn<<<grid, kSearchThreads, 0, st>>>(
          P.n, P.c, act_index + a0, act_b + a0, est + (int64_t)a0 * P.c, w.chunks,
          part_s + (int64_t)a0 * w.chunks, part_t + (int64_t)a0 * w.chunks, rank, world,
          node_bound + a0);
    }
  }
  AFFT_CHECK_LAUNCH("noisy_search_kernel");
  if (world > 1) {
    if (!shard->exchange) {
      set_error("search shard without an exchange callback");
      return AFFT_EINVAL;
    }
    const int rc = shard->exchange(shard->ctx, part_s, part_t, nparts, st);
    if (rc) {
      set_error("search shard exchange failed (%d)", rc);
      return AFFT_ECUDA;
    }
  }
  noisy_finalize_kernel<<<(unsigned)((A * 32 + 255) / 256), 256, 0, st>>>(
      A, w.chunks, reinterpret_cast<const double*>(ws + w.part_s),
      reinterpret_cast<const int32_t*>(ws + w.part_t), act_row, act_index, act_b, residual, P,
      out.f0 ? out.f0 : reinterpret_cast<int64_t*>(ws + w.f0),
      out.val ? out.val : reinterpret_cast<double*>(ws + w.val),
      out.res ? out.res : reinterpret_cast<double*>(ws + w.res), out.decide);
  AFFT_CHECK_LAUNCH("noisy_finalize_kernel");
  return AFFT_OK;
}

// ------------------------------------------------------------ device-resident rounds
//
// peel_decode's loop (peeling.py:283-313) without host round-trips: one round's
// kernels (prep -> est -> seed + search -> finalize -> apply -> harvest -> control)
// are captured once into the body of a CUDA-graph WHILE node; the control kernel sets
// the node's condition from the round's harvest count and the round budget, so the
// whole decode is one graph launch.  Launch shapes cannot depend on the active count
// (it lives on the device): list-sized kernels get the largest possible grid and read
// the count, and the candidate scan is a persistent grid pulling (node, chunk) items.
// counters[0] active count, [1] tones harvested this round, [2] scan ticket, [3] rounds run.
__global__ void noisy_round_control_kernel(cudaGraphConditionalHandle handle,
                                           int32_t* __restrict__ counters, int max_rounds) {
  const int it = counters[3] + 1;
  counters[3] = it;
  const bool more = counters[1] != 0 && it < max_rounds;
  counters[0] = 0;
  counters[1] = 0;
  counters[2] = 0;
  cudaGraphSetConditional(handle, more ? 1u : 0u);
}

static int device_sms() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  return v;
}

// Harvest, then (global harvest state) the grid-wide subtraction; nf_round sits right
// after the batch's harvest blocks.
static void launch_harvest(const NoisyPlan& P, int64_t batch, double* residual, int8_t* state,
                           int8_t* dirty, int64_t* node_f0, double* node_val, int32_t* done,
                           int64_t* rec_pos, double* rec_val, int32_t rec_cap, int32_t* rec_count,
                           int32_t* rounds, int32_t* found, char* hscratch, size_t hbytes,
                           size_t hsmem, cudaStream_t st) {
  int32_t* nf_round =
      hscratch ? reinterpret_cast<int32_t*>(hscratch + (size_t)batch * hbytes) : nullptr;
  noisy_harvest_kernel<<<(unsigned)batch, 1024, hsmem, st>>>(
      P, residual, state, dirty, node_f0, node_val, done, rec_pos, rec_val, rec_cap, rec_count,
      rounds, found, hscratch, hbytes, nf_round);
  if (nf_round)
    noisy_subtract_kernel<<<dim3((unsigned)((P.nodes + 7) / 8), (unsigned)batch), 256, 0, st>>>(
        P, residual, dirty, node_f0, node_val, nf_round, hscratch, hbytes);
}

// Enqueue one round's kernels on the capturing stream `cs`.
static int enqueue_round(const NoisyPlan& P, const NoisyWs& w, char* ws, int64_t batch,
                         double* residual, int8_t* state, int8_t* dirty, int32_t* done,
                         int64_t* node_f0, double* node_val, const double* t0, const double* t1,
                         int64_t* rec_pos, double* rec_val, int32_t rec_cap, int32_t* rec_count,
                         int32_t* rounds, int32_t* counters, char* hscratch, size_t hbytes,
                         size_t hsmem, cudaGraphConditionalHandle handle, int max_rounds,
                         cudaStream_t cs) {
  const int64_t rows = batch * P.nodes;  // the largest possible active list
  int64_t* act_row = reinterpret_cast<int64_t*>(ws + w.act_row);
  int64_t* act_index = reinterpret_cast<int64_t*>(ws + w.act_index);
  int64_t* act_b = reinterpret_cast<int64_t*>(ws + w.act_b);
  double* est = reinterpret_cast<double*>(ws + w.est);
  double* part_s = reinterpret_cast<double*>(ws + w.part_s);
  int32_t* part_t = reinterpret_cast<int32_t*>(ws + w.part_t);
  unsigned long long* node_bound = reinterpret_cast<unsigned long long*>(ws + w.bound);
  int64_t* f0s = reinterpret_cast<int64_t*>(ws + w.f0);
  double* vals = reinterpret_cast<double*>(ws + w.val);
  double* res = reinterpret_cast<double*>(ws + w.res);
  const int32_t* A_dev = counters;
  const bool k32 = P.n < (int64_t(1) << 31);
  noisy_prep_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, cs>>>(
      batch, P, residual, state, dirty, done, t0, counters, act_row, act_index, act_b);
  AFFT_CHECK_LAUNCH("noisy_prep_kernel");
  const int64_t ne = rows * P.c;
  noisy_est_kernel<<<(unsigned)((ne + 127) / 128), 128, 0, cs>>>(0, P.c, P.m, act_row, residual,
                                                                P.R, P, est, node_bound, A_dev);
  AFFT_CHECK_LAUNCH("noisy_est_kernel");
  if (w.Lmax <= warp_search_maxl()) {  // one chunk per node: part slot a = node a
    auto kfn = k32 ? noisy_search_warp_kernel<true> : noisy_search_warp_kernel<false>;
    kfn<<<(unsigned)((rows + kWarpSearchWarps - 1) / kWarpSearchWarps), kWarpSearchWarps * 32, 0,
          cs>>>(P.n, P.c, 0, act_index, act_b, est, part_s, part_t, A_dev);
  } else {
    auto sfn = k32 ? noisy_seed_kernel<true> : noisy_seed_kernel<false>;
    sfn<<<(unsigned)((rows + 127) / 128), 128, 0, cs>>>(P.n, P.c, 0, act_index, act_b, est,
                                                        node_bound, A_dev);
    auto kfn = k32 ? noisy_search_persistent_kernel<true> : noisy_search_persistent_kernel<false>;
    kfn<<<(unsigned)(device_sms() * 8), kSearchThreads, 0, cs>>>(
        P.n, P.c, A_dev, act_index, act_b, est, w.chunks, part_s, part_t, node_bound,
        counters + 2);
  }
  AFFT_CHECK_LAUNCH("noisy_search_persistent_kernel");
  noisy_finalize_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, cs>>>(
      0, w.chunks, part_s, part_t, act_row, act_index, act_b, residual, P, f0s, vals, res,
      NoisyDecide{nullptr, 0.0, 0.0, nullptr, nullptr}, A_dev);
  AFFT_CHECK_LAUNCH("noisy_finalize_kernel");
  noisy_apply_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, cs>>>(
      0, P, act_row, f0s, vals, res, t1, state, dirty, node_f0, node_val, A_dev);
  AFFT_CHECK_LAUNCH("noisy_apply_kernel");
  launch_harvest(P, batch, residual, state, dirty, node_f0, node_val, done, rec_pos, rec_val,
                 rec_cap, rec_count, rounds, counters + 1, hscratch, hbytes, hsmem, cs);
  AFFT_CHECK_LAUNCH("noisy_harvest_kernel");
  noisy_round_control_kernel<<<1, 1, 0, cs>>>(handle, counters, max_rounds);
  AFFT_CHECK_LAUNCH("noisy_round_control_kernel");
  return AFFT_OK;
}

// A capture stream per thread: capture must not touch the caller's stream (it may
// hold pending work), and the graph is launched on the caller's stream afterwards.
static cudaStream_t capture_stream() {
  thread_local cudaStream_t cs = nullptr;
  thread_local int cs_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!cs || cs_dev != dev) {
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    cs_dev = dev;
  }
  return cs;
}

// The whole round loop as one graph launch on `st` (see above).
static int peel_rounds_graph(const NoisyPlan& P, const NoisyWs& w, char* ws, int64_t batch,
                             double* residual, int8_t* state, int8_t* dirty, int32_t* done,
                             int64_t* node_f0, double* node_val, const double* t0,
                             const double* t1, int32_t max_rounds, int64_t* rec_pos,
                             double* rec_val, int32_t rec_cap, int32_t* rec_count,
                             int32_t* rounds, int32_t* counters, char* hscratch, size_t hbytes,
                             size_t hsmem, cudaStream_t st) {
  if (max_rounds <= 0) return AFFT_OK;
  cudaError_t e = cudaMemsetAsync(counters, 0, 16, st);
  if (e != cudaSuccess) return cuda_status(e, "afft_peel_noisy counters");
  cudaStream_t cs = capture_stream();
  if (!cs) return cuda_status(cudaGetLastError(), "capture stream");
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  int rc = AFFT_OK;
  do {
    if ((e = cudaGraphCreate(&g, 0)) != cudaSuccess) break;
    cudaGraphConditionalHandle h;
    if ((e = cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault)) !=
        cudaSuccess)
      break;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &np)) != cudaSuccess) break;
    cudaGraph_t body = np.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
      break;
    rc = enqueue_round(P, w, ws, batch, residual, state, dirty, done, node_f0, node_val, t0, t1,
                       rec_pos, rec_val, rec_cap, rec_count, rounds, counters, hscratch, hbytes,
                       hsmem, h, max_rounds, cs);
    cudaGraph_t captured = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(cs, &captured);
    if (rc) break;
    if ((e = e2) != cudaSuccess) break;
    if ((e = cudaGraphInstantiate(&ex, g, 0)) != cudaSuccess) break;
    e = cudaGraphLaunch(ex, st);
  } while (false);
  if (ex) cudaGraphExecDestroy(ex);  // safe: destruction waits for nothing, launch is queued
  if (g) cudaGraphDestroy(g);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_status(e, "afft_peel_noisy round graph");
  return AFFT_OK;
}

// Two pinned int32 read-back slots for one decode, from the library's pinned pool.
struct PinnedCounter {
  size_t cap = 0;
  int32_t* h = static_cast<int32_t*>(pinned_acquire(64, &cap));
  ~PinnedCounter() { pinned_release(h, cap); }
};

}  // namespace afft

using namespace afft;

extern "C" size_t afft_noisy_workspace_size(int64_t n, int64_t batch, const int64_t* factors,
                                            int32_t ncycles, int32_t c, int32_t m) {
  std::unique_ptr<NoisyPlan> P_owner(new NoisyPlan());
  NoisyPlan* P = P_owner.get();
  std::vector<int64_t> zeros((size_t)std::max(1, c * m), 0);
  double wts[kMaxRounds] = {0};
  int64_t nodes = 0;
  for (int k = 0; k < ncycles && factors; ++k) nodes += factors[k];
  size_t out = 0;
  if (!make_noisy_plan(P, n, factors, ncycles, zeros.data(), c * m, c, m, wts, (int)nodes))
    out = noisy_ws(*P, batch * P->nodes).total;
  return out;
}

extern "C" int afft_node_energies(const double* vec, int32_t nshift, int64_t count,
                                  double* energy, void* stream) {
  if (count == 0) return AFFT_OK;
  if (!vec || !energy || nshift < 1 || count < 0) {
    set_error("afft_node_energies: bad arguments");
    return AFFT_EINVAL;
  }
  node_energy_kernel<<<(unsigned)((count + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      count, nshift, vec, energy);
  AFFT_CHECK_LAUNCH("node_energy_kernel");
  return AFFT_OK;
}

extern "C" int afft_robust_thresholds(const double* energy, const uint8_t* mask, int64_t count,
                                      int64_t batch, int32_t r, double* t0, double* t1,
                                      void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!energy || !t0 || !t1 || count < 1 || r < 1) {
    set_error("afft_robust_thresholds: bad arguments");
    return AFFT_EINVAL;
  }
  int pow2 = 1;
  while (pow2 < count) pow2 <<= 1;
  const size_t smem = (size_t)pow2 * 8;
  if (smem > 200 * 1024) {  // large: radix-select median over a global copy
    double* scratch = nullptr;
    cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&scratch),
                                    (size_t)batch * count * 8, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(median scratch)");
    robust_thresholds_large_kernel<<<(unsigned)batch, 1024, 0, (cudaStream_t)stream>>>(
        (int)count, energy, mask, r, scratch, t0, t1);
    scratch_free(scratch, (cudaStream_t)stream);
    AFFT_CHECK_LAUNCH("robust_thresholds_large_kernel");
    return AFFT_OK;
  }
  cudaError_t e = ensure_smem((const void*)robust_thresholds_kernel, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(robust_thresholds)");
  robust_thresholds_kernel<<<(unsigned)batch, 256, smem, (cudaStream_t)stream>>>(
      (int)count, pow2, energy, mask, r, t0, t1);
  AFFT_CHECK_LAUNCH("robust_thresholds_kernel");
  return AFFT_OK;
}

namespace afft {
static int singleton_search(const double* residual, const int64_t* index, int64_t count,
                            int64_t b, int64_t n, const int64_t* shifts, int32_t nshift, int32_t c,
                            int32_t m, const double* weights, int64_t* f0, double* val,
                            double* resnorm, void* workspace, size_t workspace_bytes,
                            cudaStream_t st, NoisyDecide decide, const int64_t* tau_tab = nullptr,
                            const int32_t* row_sig = nullptr) {
  if (count == 0) return AFFT_OK;
  if (!residual || !index || !f0 || !val || !resnorm || !shifts || !weights || b < 1 ||
      n % b) {
    set_error("afft_singleton_search_noisy: bad arguments");
    return AFFT_EINVAL;
  }
  std::unique_ptr<NoisyPlan> P_owner(new NoisyPlan());
  NoisyPlan* P = P_owner.get();
  int rc = make_noisy_plan(P, n, &b, 1, shifts, nshift, c, m, weights, 1);
  if (rc) {
    return rc;
  }
  P->tau_tab = tau_tab;
  P->row_sig = row_sig;
  const NoisyWs w = noisy_ws(*P, count);
  if (!workspace || workspace_bytes < w.total) {
    set_error("afft_singleton_search_noisy: workspace of %zu bytes needed", w.total);
    return AFFT_ENOMEM;
  }
  char* ws = reinterpret_cast<char*>(workspace);
  // active list = the given nodes, rows 0..count-1 of `residual`: the estimate kernel
  // fills it on the device (no host staging, no synchronisation, no extra launch)
  SearchOut out;  // the fit writes straight into the caller's arrays
  out.f0 = f0;
  out.val = val;
  out.res = resnorm;
  out.decide = decide;
  rc = run_search(*P, w, ws, (int)count, residual, st, nullptr, 0, out, index, b);
  if (!rc) AFFT_CHECK_LAUNCH("singleton_search_noisy");
  return rc;
}

// classify_noisy over rows of several signals at once (DSFFT batches): row r belongs to
// signal row_sig[r], whose reduced search shifts are tau_tab[sig][0..c*m) (device) and
// whose gates are t0s[sig] / t1s[sig] (device).
int classify_noisy_multi(const double* residual, const int64_t* index, const int32_t* row_sig,
                         int64_t count, int64_t b, int64_t n, const int64_t* tau_tab, int32_t c,
                         int32_t m, const double* weights, const double* t0s, const double* t1s,
                         int8_t* state, int64_t* f0, double* val, double* resnorm,
                         void* workspace, size_t workspace_bytes, cudaStream_t st) {
  if (count == 0) return AFFT_OK;
  if (!row_sig || !tau_tab || !t0s || !t1s || !state) {
    set_error("classify_noisy_multi: bad arguments");
    return AFFT_EINVAL;
  }
  std::vector<int64_t> zeros((size_t)c * m, 0);
  return singleton_search(residual, index, count, b, n, zeros.data(), c * m, c, m, weights, f0,
                          val, resnorm, workspace, workspace_bytes, st,
                          NoisyDecide{state, 0.0, 0.0, t0s, t1s}, tau_tab, row_sig);
}

}  // namespace afft

extern "C" int afft_singleton_search_noisy(const double* residual, const int64_t* index,
                                           int64_t count, int64_t b, int64_t n,
                                           const int64_t* shifts, int32_t nshift, int32_t c,
                                           int32_t m, const double* weights, int64_t* f0,
                                           double* val, double* resnorm, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  return singleton_search(residual, index, count, b, n, shifts, nshift, c, m, weights, f0, val,
                          resnorm, workspace, workspace_bytes, (cudaStream_t)stream,
                          NoisyDecide{nullptr, 0.0, 0.0, nullptr, nullptr});
}

namespace afft {
static int peel_noisy_core(NoisyPlan* P, int64_t batch, double* residual, int8_t* state,
                           int64_t* node_f0, double* node_val, const double* t0,
                           const double* t1, int32_t max_rounds, int64_t* rec_pos,
                           double* rec_val, int32_t rec_cap, int32_t* rec_count, int32_t* rounds,
                           int32_t* unresolved, void* workspace, size_t workspace_bytes,
                           void* stream, const AfftSearchShard* shard);
}  // namespace afft

extern "C" int afft_peel_noisy(int64_t n, int64_t batch, const int64_t* factors, int32_t ncycles,
                               const int64_t* shifts, int32_t nshift, int32_t c, int32_t m,
                               const double* weights, double* residual, int8_t* state,
                               int64_t* node_f0, double* node_val, const double* t0,
                               const double* t1, int32_t max_rounds, int64_t* rec_pos,
                               double* rec_val, int32_t rec_cap, int32_t* rec_count,
                               int32_t* rounds, int32_t* unresolved, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return afft_peel_noisy_sharded(n, batch, factors, ncycles, shifts, nshift, c, m, weights,
                                 residual, state, node_f0, node_val, t0, t1, max_rounds, rec_pos,
                                 rec_val, rec_cap, rec_count, rounds, unresolved, workspace,
                                 workspace_bytes, stream, nullptr);
}

extern "C" int afft_peel_noisy_sharded(
    int64_t n, int64_t batch, const int64_t* factors, int32_t ncycles, const int64_t* shifts,
    int32_t nshift, int32_t c, int32_t m, const double* weights, double* residual, int8_t* state,
    int64_t* node_f0, double* node_val, const double* t0, const double* t1, int32_t max_rounds,
    int64_t* rec_pos, double* rec_val, int32_t rec_cap, int32_t* rec_count, int32_t* rounds,
    int32_t* unresolved, void* workspace, size_t workspace_bytes, void* stream,
    const AfftSearchShard* shard) {
  if (shard && (shard->world < 1 || shard->rank < 0 || shard->rank >= shard->world)) {
    set_error("afft_peel_noisy_sharded: rank %d of %d", shard->rank, shard->world);
    return AFFT_EINVAL;
  }
  if (batch == 0) return AFFT_OK;
  if (!residual || !state || !node_f0 || !node_val || !t0 || !t1 || !rec_pos || !rec_val ||
      !rec_count || !rounds || !unresolved || !weights || !shifts || max_rounds < 0) {
    set_error("afft_peel_noisy: bad arguments");
    return AFFT_EINVAL;
  }
  std::unique_ptr<NoisyPlan> P_owner(new NoisyPlan());
  NoisyPlan* P = P_owner.get();
  int rc = make_noisy_plan(P, n, factors, ncycles, shifts, nshift, c, m, weights, rec_cap);
  if (rc) {
    return rc;
  }
  return peel_noisy_core(P, batch, residual, state, node_f0, node_val, t0, t1, max_rounds,
                         rec_pos, rec_val, rec_cap, rec_count, rounds, unresolved, workspace,
                         workspace_bytes, stream, shard);
}

namespace afft {
static int peel_noisy_core(NoisyPlan* P, int64_t batch, double* residual, int8_t* state,
                           int64_t* node_f0, double* node_val, const double* t0,
                           const double* t1, int32_t max_rounds, int64_t* rec_pos,
                           double* rec_val, int32_t rec_cap, int32_t* rec_count, int32_t* rounds,
                           int32_t* unresolved, void* workspace, size_t workspace_bytes,
                           void* stream, const AfftSearchShard* shard) {
  int rc = AFFT_OK;
  const int N = P->nodes;
  const NoisyWs w = noisy_ws(*P, batch * N);
  if (!workspace || workspace_bytes < w.total) {
    set_error("afft_peel_noisy: workspace of %zu bytes needed, %zu given", w.total,
              workspace_bytes);
    return AFFT_ENOMEM;
  }
  if ((int64_t)batch * N > INT32_MAX) {
    set_error("afft_peel_noisy: batch * nodes exceeds 2^31");
    return AFFT_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = reinterpret_cast<char*>(workspace);
  int8_t* dirty = reinterpret_cast<int8_t*>(ws + w.dirty);
  int32_t* done = reinterpret_cast<int32_t*>(ws + w.done);
  int32_t* counters = reinterpret_cast<int32_t*>(ws + w.counters);
  PinnedCounter pc;
  int32_t* host = pc.h;
  if (!host) {
    set_error("afft_peel_noisy: cannot allocate a pinned host counter");
    return AFFT_ENOMEM;
  }
  cudaError_t e = cudaMemsetAsync(dirty, 1, (size_t)batch * N, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(done, 0, (size_t)batch * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(rounds, 0, (size_t)batch * 4, st);
  if (e != cudaSuccess) {
    return cuda_status(e, "afft_peel_noisy init");
  }
  int hcap = P->hmask + 1;
  // hash, flag[N], found_g[N], found_res[N * ncycles] (per-node tone lists), hv[N]
  const size_t hbytes =
      ((size_t)hcap * 4 + (size_t)N * 4 * 2 + (size_t)N * P->ncycles * 4 + N + 64 + 15) & ~size_t(15);
  size_t hsmem = hbytes;
  char* hscratch = nullptr;
  if (hbytes > 200 * 1024) {  // large graphs: harvest state in global memory (+ nf_round)
    e = scratch_alloc(reinterpret_cast<void**>(&hscratch), (size_t)batch * (hbytes + 4), st);
    if (e != cudaSuccess) {
      return cuda_status(e, "scratch_alloc(noisy harvest scratch)");
    }
    hsmem = 0;
  } else {
    e = ensure_smem((const void*)noisy_harvest_kernel, (int)hsmem);
    if (e != cudaSuccess) {
      return cuda_status(e, "cudaFuncSetAttribute(noisy_harvest)");
    }
  }
  const int64_t total = batch * N;
  static const bool host_loop = [] {  // AFFT_PEEL_GRAPH=0: the host-synchronised loop below
    const char* e = getenv("AFFT_PEEL_GRAPH");
    return e && e[0] == '0';
  }();
  if ((!shard || shard->world <= 1) && !host_loop) {
    rc = peel_rounds_graph(*P, w, ws, batch, residual, state, dirty, done, node_f0, node_val, t0,
                           t1, max_rounds, rec_pos, rec_val, rec_cap, rec_count, rounds, counters,
                           hscratch, hbytes, hsmem, st);
    if (!rc) {
      count_multi_kernel<<<(unsigned)batch, 256, 0, st>>>(batch, N, state, unresolved);
      rc = cudaGetLastError() == cudaSuccess ? AFFT_OK : AFFT_ECUDA;
    }
    if (hscratch) scratch_free(hscratch, st);
    return rc;
  }
  for (int it = 0; it < max_rounds; ++it) {
    cudaMemsetAsync(counters, 0, 8, st);
    noisy_prep_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        batch, *P, residual, state, dirty, done, t0, counters,
        reinterpret_cast<int64_t*>(ws + w.act_row), reinterpret_cast<int64_t*>(ws + w.act_index),
        reinterpret_cast<int64_t*>(ws + w.act_b));
    AFFT_CHECK_LAUNCH("noisy_prep_kernel");
    cudaMemcpyAsync(host, counters, 4, cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
      if (hscratch) scratch_free(hscratch, st);
      return cuda_status(e, "afft_peel_noisy round sync");
    }
    const int A = host[0];
    if ((rc = run_search(*P, w, ws, A, residual, st, shard, total))) {
      if (hscratch) scratch_free(hscratch, st);
      return rc;
    }
    if (A > 0) {
      noisy_apply_kernel<<<(unsigned)((A + 255) / 256), 256, 0, st>>>(
          A, *P, reinterpret_cast<const int64_t*>(ws + w.act_row),
          reinterpret_cast<const int64_t*>(ws + w.f0), reinterpret_cast<const double*>(ws + w.val),
          reinterpret_cast<const double*>(ws + w.res), t1, state, dirty, node_f0, node_val);
      AFFT_CHECK_LAUNCH("noisy_apply_kernel");
    }
    launch_harvest(*P, batch, residual, state, dirty, node_f0, node_val, done, rec_pos,
                   rec_val, rec_cap, rec_count, rounds, counters + 1, hscratch, hbytes, hsmem,
                   st);
    AFFT_CHECK_LAUNCH("noisy_harvest_kernel");
    cudaMemcpyAsync(host + 1, counters + 1, 4, cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
      return cuda_status(e, "afft_peel_noisy round sync");
    }
    if (host[1] == 0) break;  // every signal found nothing: all loops have exited
  }
  count_multi_kernel<<<(unsigned)batch, 256, 0, st>>>(batch, N, state, unresolved);
  if (hscratch) scratch_free(hscratch, st);
  AFFT_CHECK_LAUNCH("count_multi_kernel");
  return AFFT_OK;
}
}  // namespace afft


extern "C" int afft_classify_noisy(const double* residual, const int64_t* index, int64_t count,
                                   int64_t b, int64_t n, const int64_t* shifts, int32_t nshift,
                                   int32_t c, int32_t m, const double* weights, double t0,
                                   double t1, int8_t* state, int64_t* f0, double* val,
                                   double* resnorm, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  if (count == 0) return AFFT_OK;
  if (!state) {
    set_error("afft_classify_noisy: bad arguments");
    return AFFT_EINVAL;
  }
  // search + fit + the decision of peeling.py:257-267, all in the finalize kernel
  return singleton_search(residual, index, count, b, n, shifts, nshift, c, m, weights, f0, val,
                          resnorm, workspace, workspace_bytes, (cudaStream_t)stream,
                          NoisyDecide{state, t0, t1, nullptr, nullptr});
}

namespace afft {
// np.median of |v|^2 (complex input, mode 1) or of v (real, mode 0), one CTA per row.
__global__ void median_kernel(int count, int mode, const double* __restrict__ in,
                              double* __restrict__ scratch, double* __restrict__ out) {
  __shared__ unsigned hist[256];
  const int64_t s = blockIdx.x;
  double* v = scratch + s * (int64_t)count;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    if (mode == 1) {
      const double a = hypot(in[2 * (s * (int64_t)count + i)], in[2 * (s * (int64_t)count + i) + 1]);
      v[i] = a * a;
    } else {
      v[i] = in[s * (int64_t)count + i];
    }
  }
  __syncthreads();
  double med;
  if (count & 1) {
    med = radix_select(v, count, count / 2, hist);
  } else {
    const double lo = radix_select(v, count, count / 2 - 1, hist);
    const double hi = radix_select(v, count, count / 2, hist);
    med = (lo + hi) / 2.0;
  }
  if (threadIdx.x == 0) out[s] = med;
}
}  // namespace afft

extern "C" int afft_median(const double* values, int32_t mode, int64_t count, int64_t batch,
                           double* out, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!values || !out || count < 1 || count > INT32_MAX || (mode != 0 && mode != 1)) {
    set_error("afft_median: bad arguments");
    return AFFT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* scratch = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&scratch), (size_t)batch * count * 8, st);
  if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(median)");
  median_kernel<<<(unsigned)batch, 1024, 0, st>>>((int)count, mode, values, scratch, out);
  scratch_free(scratch, st);
  AFFT_CHECK_LAUNCH("median_kernel");
  return AFFT_OK;
}

extern "C" size_t afft_singleton_workspace_size(int64_t n, int64_t count, int64_t b, int32_t c,
                                                int32_t m) {
  std::unique_ptr<NoisyPlan> P(new NoisyPlan());
  std::vector<int64_t> zeros((size_t)std::max(1, c * m), 0);
  double wts[kMaxRounds] = {0};
  if (make_noisy_plan(P.get(), n, &b, 1, zeros.data(), c * m, c, m, wts, 1)) return 0;
  return noisy_ws(*P, count).total;
}

// ------------------------------------------------------------------ afft_rffast
//
// r_ffast's body (peeling.py:361-386) for a batch, one enqueue: graph build at every
// signal's own search shifts (r_j + 2^j t from its anchors, peeling.py:60-62) ->
// node energies -> robust thresholds (peeling.py:335-358) -> device-resident noisy
// peeling (peeling.py:270-313) -> top-k truncation (oneshot.py:260-263).

namespace afft {
struct RffastWs {
  size_t nodes, tau_raw, tau_red, energy, state, f0, val, peel, total;
};

static RffastWs rffast_ws(const NoisyPlan& P, int64_t batch) {
  RffastWs r;
  const int64_t rows = batch * P.nodes;
  size_t o = 0;
  r.nodes = o;   o = al256(o + (size_t)rows * P.R * 16);
  r.tau_raw = o; o = al256(o + (size_t)batch * P.R * 8);
  r.tau_red = o; o = al256(o + (size_t)batch * P.R * 8);
  r.energy = o;  o = al256(o + (size_t)rows * 8);
  r.state = o;   o = al256(o + (size_t)rows);
  r.f0 = o;      o = al256(o + (size_t)rows * 8);
  r.val = o;     o = al256(o + (size_t)rows * 16);
  r.peel = o;    o = al256(o + noisy_ws(P, rows).total);
  r.total = o;
  return r;
}

__global__ void rffast_init_kernel(int64_t rows, int8_t* __restrict__ state,
                                   int64_t* __restrict__ f0, double* __restrict__ val,
                                   int64_t batch, int32_t* __restrict__ rec_count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) {
    state[i] = AFFT_UNKNOWN;
    f0[i] = -1;
    reinterpret_cast<cd*>(val)[i] = cd{0.0, 0.0};
  }
  if (i < batch) rec_count[i] = 0;
}

static int rffast_plan(NoisyPlan* P, int64_t n, const int64_t* factors, int32_t ncycles,
                       int32_t c, int32_t m, const double* weights) {
  if (c < 1 || c > kMaxStrides || m < 2 || m > kMaxRounds) {
    set_error("search plan c=%d m=%d unsupported", c, m);
    return AFFT_EUNSUPPORTED;
  }
  std::vector<int64_t> zeros((size_t)c * m, 0);
  int64_t nodes = 0;
  for (int k = 0; k < ncycles && factors; ++k) nodes += factors[k];
  return make_noisy_plan(P, n, factors, ncycles, zeros.data(), c * m, c, m, weights,
                         (int)std::min<int64_t>(nodes, INT32_MAX));
}
}  // namespace afft

extern "C" size_t afft_rffast_workspace_size(int64_t n, int64_t batch, const int64_t* factors,
                                             int32_t ncycles, int32_t c, int32_t m) {
  std::unique_ptr<NoisyPlan> P(new NoisyPlan());
  double wts[kMaxRounds] = {0};
  if (!factors || rffast_plan(P.get(), n, factors, ncycles, c, m, wts)) return 0;
  return rffast_ws(*P, std::max<int64_t>(batch, 1)).total;
}

extern "C" int afft_rffast(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                           const int64_t* factors, int32_t ncycles, const int64_t* anchors,
                           int64_t anchor_stride, int32_t c, int32_t m, const double* weights,
                           int32_t k, int32_t max_rounds, int64_t* out_pos, double* out_val,
                           int32_t* out_count, int64_t* all_pos, double* all_val,
                           int32_t* all_count, int32_t* rounds, int32_t* unresolved, double* t0,
                           double* t1, void* workspace, size_t workspace_bytes, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!x || !factors || !anchors || !weights || (k > 0 && (!out_pos || !out_val)) ||
      !out_count || !all_pos || !all_val || !all_count || !rounds || !unresolved || !t0 || !t1 ||
      k < 0 || batch < 0 || ld < n || anchor_stride < 0 ||
      (dtype != AFFT_C64 && dtype != AFFT_C128)) {
    set_error("afft_rffast: bad arguments");
    return AFFT_EINVAL;
  }
  std::unique_ptr<NoisyPlan> P_owner(new NoisyPlan());
  NoisyPlan* P = P_owner.get();
  int rc = rffast_plan(P, n, factors, ncycles, c, m, weights);
  if (rc) return rc;
  const RffastWs w = rffast_ws(*P, batch);
  if (!workspace || workspace_bytes < w.total) {
    set_error("afft_rffast: workspace of %zu bytes needed, %zu given", w.total, workspace_bytes);
    return AFFT_ENOMEM;
  }
  if ((int64_t)batch * P->nodes > INT32_MAX) {
    set_error("afft_rffast: batch * nodes exceeds 2^31");
    return AFFT_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = reinterpret_cast<char*>(workspace);
  const int R = P->R, N = P->nodes;
  const int64_t rows = batch * N;
  // per-signal shifts r_j + 2^j t (SearchPlan.shifts, peeling.py:60-62): raw for the
  // gather, reduced for the peel; staged from pageable memory (the copy returns once
  // staged, so the vectors may go out of scope)
  std::vector<int64_t> raw((size_t)batch * R), red((size_t)batch * R);
  for (int64_t s = 0; s < batch; ++s)
    for (int j = 0; j < c; ++j)
      for (int t = 0; t < m; ++t) {
        const int64_t v = anchors[s * anchor_stride + j] + (int64_t(1) << j) * t;
        raw[(size_t)s * R + j * m + t] = v;
        red[(size_t)s * R + j * m + t] = host_pymod(v, n);
      }
  for (int r = 0; r < R; ++r) P->tau[r] = red[r];
  int64_t* tau_raw = reinterpret_cast<int64_t*>(ws + w.tau_raw);
  int64_t* tau_red = reinterpret_cast<int64_t*>(ws + w.tau_red);
  cudaError_t e = cudaMemcpyAsync(tau_raw, raw.data(), raw.size() * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(tau_red, red.data(), red.size() * 8, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_status(e, "afft_rffast shift tables");
  P->tau_tab = tau_red;
  double* nodes = reinterpret_cast<double*>(ws + w.nodes);
  if ((rc = build_graph_table(x, dtype, n, batch, ld, factors, ncycles, tau_raw, R, nodes, st)))
    return rc;
  double* energy = reinterpret_cast<double*>(ws + w.energy);
  node_energy_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(rows, R, nodes, energy);
  AFFT_CHECK_LAUNCH("node_energy_kernel");
  if ((rc = afft_robust_thresholds(energy, nullptr, N, batch, R, t0, t1, st))) return rc;
  int8_t* state = reinterpret_cast<int8_t*>(ws + w.state);
  int64_t* f0 = reinterpret_cast<int64_t*>(ws + w.f0);
  double* val = reinterpret_cast<double*>(ws + w.val);
  rffast_init_kernel<<<(unsigned)((std::max<int64_t>(rows, batch) + 255) / 256), 256, 0, st>>>(
      rows, state, f0, val, batch, all_count);
  AFFT_CHECK_LAUNCH("rffast_init_kernel");
  const int mr = max_rounds > 0 ? max_rounds : k + 4;
  if ((rc = peel_noisy_core(P, batch, nodes, state, f0, val, t0, t1, mr, all_pos, all_val, N,
                            all_count, rounds, unresolved, ws + w.peel,
                            w.total - w.peel, stream, nullptr)))
    return rc;
  return afft_truncate(all_pos, all_val, all_count, N, batch, k, out_pos, out_val, out_count,
                       stream);
}
