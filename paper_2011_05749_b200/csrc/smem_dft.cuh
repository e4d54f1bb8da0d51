// Batched mixed-radix forward DFT held entirely in shared memory (K2 in SURVEY §2).
//
// Replaces the size-b `np.fft.fft` of bucketize.py:99.  Stockham autosort
// formulation: stage s with radix R reads butterfly j's inputs at stride n/R,
// applies the twiddles w_{Ns*R}^{(j mod Ns)*r}, does a size-R DFT and writes
// the outputs at stride Ns into the other buffer, so the result comes out in
// natural order without a bit-reversal pass.  Radix 4 and 2 use add-only
// butterflies; 3..8 use register-resident direct DFTs; larger primes (the 127,
// 73, 43, 17 ... of co-prime cycle sizes) use an in-place scaled direct DFT.
// All twiddles come from one table tw[k] = exp(-2*pi*i*k/n) built with
// sincospi, exact at the quarter points, so every factor is accurate to ~1 ulp.
#pragma once

#include "afft_common.cuh"

namespace afft {

constexpr int kMaxStages = 40;

struct DftPlan {
  int32_t n;
  int32_t nstages;
  int32_t lgn;  // log2(n) when n is a power of two (radix 4/2 only), else -1
  int16_t radix[kMaxStages];
};

// Host: factor n into radices (powers of two: 16/8 first, then 4 or 2; other sizes:
// 4s first, then 2, then odd primes ascending).
// max_radix: largest register butterfly for power-of-two sizes (16 needs ~128
// registers of data per thread; kernels capped at 64-80 registers use 8).
inline bool make_dft_plan(int64_t n, DftPlan* p, int max_radix = 8) {
  if (n < 1 || n > (1 << 30)) return false;
  p->n = (int32_t)n;
  p->nstages = 0;
  p->lgn = -1;
  if ((n & (n - 1)) == 0) {
    int lg = 0;
    while ((1ll << lg) < n) ++lg;
    p->lgn = lg;
  }
  if (p->lgn >= 0) {  // powers of two: radix-16 register butterflies, then 8 / 4 / 2
    int lg = p->lgn;
    while (max_radix >= 16 && lg >= 4) {
      p->radix[p->nstages++] = 16;
      lg -= 4;
    }
    while (lg >= 3) {
      p->radix[p->nstages++] = 8;
      lg -= 3;
    }
    if (lg == 2) p->radix[p->nstages++] = 4;
    if (lg == 1) p->radix[p->nstages++] = 2;
    return true;
  }
  int64_t m = n;
  while (m % 4 == 0) {
    if (p->nstages >= kMaxStages) return false;
    p->radix[p->nstages++] = 4;
    m /= 4;
  }
  if (m % 2 == 0) {
    p->radix[p->nstages++] = 2;
    m /= 2;
  }
  for (int64_t q = 3; q * q <= m; q += 2) {
    while (m % q == 0) {
      if (p->nstages >= kMaxStages || q > 32767) return false;
      p->radix[p->nstages++] = (int16_t)q;
      m /= q;
    }
  }
  if (m > 1) {
    if (p->nstages >= kMaxStages || m > 32767) return false;
    p->radix[p->nstages++] = (int16_t)m;
  }
  return true;
}

// Fill tw[0..n) cooperatively.
__device__ __forceinline__ void build_twiddles(cd* tw, int n, int tid, int nthreads) {
  for (int k = tid; k < n; k += nthreads) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)n, &s, &c);
    tw[k] = cd{c, s};
  }
}

template <int R>
__device__ __forceinline__ void bfly_small(const cd* __restrict__ src, cd* __restrict__ dst,
                                           const cd* __restrict__ tw, int n, int nb, int Ns,
                                           int j) {
  const int jm = j % Ns;
  const int tstep = n / (Ns * R);
  cd v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    cd a = src[j + r * nb];
    v[r] = (r == 0 || jm == 0) ? a : cmul(a, tw[jm * r * tstep]);
  }
  const int idxD = (j / Ns) * Ns * R + jm;
  if constexpr (R == 2) {
    dst[idxD] = cadd(v[0], v[1]);
    dst[idxD + Ns] = csub(v[0], v[1]);
  } else if constexpr (R == 4) {
    cd a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    cd c = cadd(v[1], v[3]), d = csub(v[1], v[3]);
    dst[idxD] = cadd(a, c);
    dst[idxD + 2 * Ns] = csub(a, c);
    dst[idxD + Ns] = cd{b.re + d.im, b.im - d.re};      // b - i*d
    dst[idxD + 3 * Ns] = cd{b.re - d.im, b.im + d.re};  // b + i*d
  } else {
    const int wstep = n / R;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      cd acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) acc = cadd(acc, cmul(v[r], tw[((r * q) % R) * wstep]));
      dst[idxD + q * Ns] = acc;
    }
  }
}

// Large prime radix: two passes (scale inputs in place, then direct sums).
// Each input element belongs to exactly one butterfly, so in-place scaling is
// race-free within a stage.
__device__ __forceinline__ void scale_generic(cd* src, const cd* tw, int n, int R, int nb, int Ns,
                                              int j) {
  const int jm = j % Ns;
  if (jm == 0) return;
  const int tstep = n / (Ns * R);
  for (int r = 1; r < R; ++r) src[j + r * nb] = cmul(src[j + r * nb], tw[jm * r * tstep]);
}
__device__ __forceinline__ void out_generic(const cd* src, cd* dst, const cd* tw, int n, int R,
                                            int nb, int Ns, int j, int q) {
  const int jm = j % Ns;
  const int wstep = n / R;
  cd acc = src[j];
  int e = 0;  // (r*q) mod R, updated incrementally
  for (int r = 1; r < R; ++r) {
    e += q;
    if (e >= R) e -= R;
    acc = cadd(acc, cmul(src[j + r * nb], tw[e * wstep]));
  }
  dst[(j / Ns) * Ns * R + jm + q * Ns] = acc;
}

// Odd prime radix R >= 11 by the symmetric (Goertzel-pair) form: with
// s_r = x_r + x_{R-r} and d_r = x_r - x_{R-r} (r = 1..h, h = (R-1)/2),
//   X[q]   = x_0 + sum_r s_r cos(2 pi r q / R) - i d_r sin(2 pi r q / R)
//   X[R-q] = x_0 + sum_r s_r cos(2 pi r q / R) + i d_r sin(2 pi r q / R),
// so one work item produces two outputs from h iterations of 4 real FMAs, against
// 2 (R - 1) complex multiply-adds for the two outputs of the direct sum.
// Pass 1 (one thread per butterfly): inter-stage twiddles, then the pairs in place.
__device__ __forceinline__ void sym_prep(cd* src, const cd* tw, int n, int R, int nb, int Ns,
                                         int j) {
  const int jm = j % Ns;
  const int tstep = n / (Ns * R);
  const int h = (R - 1) >> 1;
  for (int r = 1; r <= h; ++r) {
    cd a = src[j + r * nb], c = src[j + (R - r) * nb];
    if (jm) {
      a = cmul(a, tw[jm * r * tstep]);
      c = cmul(c, tw[jm * (R - r) * tstep]);
    }
    src[j + r * nb] = cadd(a, c);
    src[j + (R - r) * nb] = csub(a, c);
  }
}
// Pass 2: outputs q and R - q of butterfly j for kSymQ consecutive q = q0 .. (q = 0:
// X[0] alone), sharing each loaded s_r, d_r across the kSymQ pairs (the one-pair
// version spent most of its time on shared-memory loads).  Per output the arithmetic
// is the same FMA chain over ascending r as one pair alone.
#ifndef AFFT_SYMQ
#define AFFT_SYMQ 2
#endif
constexpr int kSymQ = AFFT_SYMQ;
__device__ __forceinline__ void sym_out(const cd* src, cd* dst, const cd* tw, int n, int R,
                                        int nb, int Ns, int j, int q0) {
  const int jm = j % Ns;
  const int wstep = n / R;
  const int h = (R - 1) >> 1;
  const int base = (j / Ns) * Ns * R + jm;
  const cd x0 = src[j];
  double are[kSymQ], aim[kSymQ], bre[kSymQ], bim[kSymQ];
  int e[kSymQ];
  cd acc0 = x0;  // X[0] when q0 == 0
#pragma unroll
  for (int u = 0; u < kSymQ; ++u) {
    are[u] = aim[u] = bre[u] = bim[u] = 0.0;
    e[u] = 0;
  }
  for (int r = 1; r <= h; ++r) {
    const cd sr = src[j + r * nb], dr = src[j + (R - r) * nb];
    if (q0 == 0) acc0 = cadd(acc0, sr);
#pragma unroll
    for (int u = 0; u < kSymQ; ++u) {
      const int q = q0 + u;
      if (q == 0 || q > h) continue;
      e[u] += q;
      if (e[u] >= R) e[u] -= R;
      const cd w = tw[e[u] * wstep];  // exp(-2 pi i e / R): cos = w.re, sin = -w.im
      are[u] = __fma_rn(sr.re, w.re, are[u]);
      aim[u] = __fma_rn(sr.im, w.re, aim[u]);
      bre[u] = __fma_rn(-dr.im, w.im, bre[u]);  // d.im * sin
      bim[u] = __fma_rn(dr.re, w.im, bim[u]);   // -d.re * sin
    }
  }
#pragma unroll
  for (int u = 0; u < kSymQ; ++u) {
    const int q = q0 + u;
    if (q > h) break;
    if (q == 0) {
      dst[base] = acc0;
      continue;
    }
    dst[base + q * Ns] = cd{x0.re + are[u] + bre[u], x0.im + aim[u] + bim[u]};
    dst[base + (R - q) * Ns] = cd{x0.re + are[u] - bre[u], x0.im + aim[u] - bim[u]};
  }
}

// cos(pi m / 8) for m = 0..15 as correctly rounded literals; sin(pi m / 8) =
// cos16(m + 12).  A selection chain (not a table) so that the unrolled callers'
// constant m folds to immediates.
__host__ __device__ __forceinline__ constexpr double cos16(int m) {
  m &= 15;
  const double c1 = 0.9238795325112867, h = 0.7071067811865476, s1 = 0.3826834323650898;
  return m == 0 ? 1.0 : m == 1 ? c1 : m == 2 ? h : m == 3 ? s1 : m == 4 ? 0.0
       : m == 5 ? -s1 : m == 6 ? -h : m == 7 ? -c1 : m == 8 ? -1.0 : m == 9 ? -c1
       : m == 10 ? -h : m == 11 ? -s1 : m == 12 ? 0.0 : m == 13 ? s1 : m == 14 ? h : c1;
}

// In-register forward DFT of R = 2, 4, 8, 16 points (radix-2 decimation in time
// with compile-time twiddles w_R^k; multiplications by -i are exact swaps).
template <int R>
__device__ __forceinline__ void dft_reg(cd* v) {
  if constexpr (R == 2) {
    const cd a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const cd a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    const cd c = cadd(v[1], v[3]), d = csub(v[1], v[3]);
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = cd{b.re + d.im, b.im - d.re};  // b - i*d
    v[3] = cd{b.re - d.im, b.im + d.re};  // b + i*d
  } else {
    constexpr int H = R / 2;
    cd e[H], o[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    dft_reg<H>(e);
    dft_reg<H>(o);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      cd t;
      if (k == 0) {
        t = o[0];
      } else if (2 * k == H) {  // w_R^(R/4) = -i
        t = cd{o[k].im, -o[k].re};
      } else {
        // w_R^k = exp(-2 pi i k / R) = cos(pi m / 8) - i sin(pi m / 8), m = 16 k / R,
        // from correctly rounded literals (a device cos()/sin() call here is not
        // constant-folded and cost ~20 instructions per point per stage)
        const int m = 16 / R * k;
        const cd w{cos16(m), -cos16(m + 12)};
        t = cmul(o[k], w);
      }
      v[k] = cadd(e[k], t);
      v[k + H] = csub(e[k], t);
    }
  }
}

// Power-of-two sizes: Stockham stages with every index division a shift.
template <int R, int LGR>
__device__ __forceinline__ void bfly_pow2(const cd* __restrict__ src, cd* __restrict__ dst,
                                          const cd* __restrict__ tw, int nb, int lgNs,
                                          int lgtstep, int j) {
  const int jm = j & ((1 << lgNs) - 1);
  const int Ns = 1 << lgNs;
  cd v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    cd a = src[j + r * nb];
    v[r] = (r == 0 || jm == 0) ? a : cmul(a, tw[(jm * r) << lgtstep]);
  }
  dft_reg<R>(v);
  const int idxD = ((j >> lgNs) << (lgNs + LGR)) + jm;
#pragma unroll
  for (int q = 0; q < R; ++q) dst[idxD + q * Ns] = v[q];
}

template <int kMaxR>
__device__ inline cd* smem_dft_pow2(cd* a, cd* b, int count, const DftPlan& p, const cd* tw,
                                    int tid, int nthreads, int ld) {
  const int lgn = p.lgn;
  int lgNs = 0;
  for (int s = 0; s < p.nstages; ++s) {
    const int R = p.radix[s];
    const int lgR = R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1));
    const int lgnb = lgn - lgR;
    const int nb = 1 << lgnb;
    const int total = count << lgnb;
    const int lgtstep = lgn - lgNs - lgR;  // tstep = n / (Ns * R)
#define AFFT_POW2_STAGE(RR, LG)                                                         \
  for (int w = tid; w < total; w += nthreads) {                                         \
    const int seq = w >> lgnb, j = w & (nb - 1);                                        \
    bfly_pow2<RR, LG>(a + seq * ld, b + seq * ld, tw, nb, lgNs, lgtstep, j);            \
  }
    if (kMaxR >= 16 && R == 16) {
      AFFT_POW2_STAGE(16, 4)
    } else if (R == 8) {
      AFFT_POW2_STAGE(8, 3)
    } else if (R == 4) {
      AFFT_POW2_STAGE(4, 2)
    } else if (R == 2) {
      AFFT_POW2_STAGE(2, 1)
    } else {
      __trap();  // plan built with a larger max_radix than this kernel compiles in
    }
#undef AFFT_POW2_STAGE
    __syncthreads();
    cd* t = a;
    a = b;
    b = t;
    lgNs += lgR;
  }
  return a;
}

// Compile-time variant for power-of-two n = 2^LGN, CNT sequences of stride `ld`, NT
// threads: the same radix-8-first stage sequence as make_dft_plan (so the same
// arithmetic, bit for bit) with every loop bound and index split a constant.
template <int LGN, int LGR, int LGNS, int CNT, int NT>
__device__ __forceinline__ void stage_fixed(const cd* src, cd* dst, const cd* tw, int ld) {
  constexpr int NB = 1 << (LGN - LGR);
  constexpr int TOTAL = CNT * NB;
  constexpr int LGTSTEP = LGN - LGNS - LGR;
#pragma unroll
  for (int it = 0; it < (TOTAL + NT - 1) / NT; ++it) {
    const int w = threadIdx.x + it * NT;
    if (TOTAL % NT == 0 || w < TOTAL) {
      const int seq = w >> (LGN - LGR), j = w & (NB - 1);
      bfly_pow2<(1 << LGR), LGR>(src + seq * ld, dst + seq * ld, tw, NB, LGNS, LGTSTEP, j);
    }
  }
}

template <int LGN, int LGNS, int CNT, int NT>
__device__ __forceinline__ cd* dft_fixed(cd* a, cd* b, const cd* tw, int ld) {
  if constexpr (LGNS >= LGN) {
    return a;
  } else {
    constexpr int REM = LGN - LGNS;
    constexpr int LGR = REM >= 3 ? 3 : REM;
    stage_fixed<LGN, LGR, LGNS, CNT, NT>(a, b, tw, ld);
    __syncthreads();
    return dft_fixed<LGN, LGNS + LGR, CNT, NT>(b, a, tw, ld);
  }
}

// Forward DFT of `count` contiguous length-n sequences in smem buffer `a`,
// ping-ponging with `b`.  Returns the buffer that holds the result.  Must be
// called by all threads of the block (contains __syncthreads).
// kMaxR: the largest power-of-two register butterfly compiled in (must cover the
// plan's, see make_dft_plan's max_radix).
// ld: distance between consecutive sequences (>= n; n + 1 avoids bank conflicts when
// a caller writes or reads the buffer column-wise).
template <int kMaxR = 8>
__device__ inline cd* smem_dft(cd* a, cd* b, int count, const DftPlan& p, const cd* tw, int tid,
                        int nthreads, int ld = 0) {
  if (ld <= 0) ld = p.n;
  if (p.lgn >= 0) return smem_dft_pow2<kMaxR>(a, b, count, p, tw, tid, nthreads, ld);
  const int n = p.n;
  int Ns = 1;
  for (int s = 0; s < p.nstages; ++s) {
    const int R = p.radix[s];
    const int nb = n / R;
    const int total = count * nb;
    switch (R) {
      case 2:
      case 3:
      case 4:
      case 5:
      case 7:
        for (int w = tid; w < total; w += nthreads) {
          const int seq = w / nb, j = w - seq * nb;
          const cd* src = a + (size_t)seq * ld;
          cd* dst = b + (size_t)seq * ld;
          if (R == 2) bfly_small<2>(src, dst, tw, n, nb, Ns, j);
          else if (R == 3) bfly_small<3>(src, dst, tw, n, nb, Ns, j);
          else if (R == 4) bfly_small<4>(src, dst, tw, n, nb, Ns, j);
          else if (R == 5) bfly_small<5>(src, dst, tw, n, nb, Ns, j);
          else bfly_small<7>(src, dst, tw, n, nb, Ns, j);
        }
        break;
      default: {
        if (R & 1) {  // odd prime: symmetric pairs
          for (int w = tid; w < total; w += nthreads) {
            const int seq = w / nb, j = w - seq * nb;
            sym_prep(a + (size_t)seq * ld, tw, n, R, nb, Ns, j);
          }
          __syncthreads();
          const int hq = ((R - 1) >> 1) / kSymQ + 1;  // groups of kSymQ q's over 0..h
          const int outs = total * hq;
          // butterflies along the lanes, q group per warp: the twiddle reads tw[e wstep]
          // (e = q r mod R, the same for every lane) broadcast and the s_r / d_r reads
          // walk consecutive butterflies.  (Groups along the lanes made the twiddle reads
          // a gather with up to 8-way bank conflicts: 58% of the shared-memory wavefronts
          // of the radix-254 pass of N = 2,097,024, profiles/r02_gstockham_ncu.md.)
          // Each output's arithmetic is unchanged (same sym_out), so results are too.
          for (int w = tid; w < outs; w += nthreads) {
            const int g = w / total;
            const int bw = w - g * total;
            const int seq = bw / nb, j = bw - seq * nb;
            sym_out(a + (size_t)seq * ld, b + (size_t)seq * ld, tw, n, R, nb, Ns, j, g * kSymQ);
          }
          break;
        }
        for (int w = tid; w < total; w += nthreads) {
          const int seq = w / nb, j = w - seq * nb;
          scale_generic(a + (size_t)seq * ld, tw, n, R, nb, Ns, j);
        }
        __syncthreads();
        const int outs = total * R;
        for (int w = tid; w < outs; w += nthreads) {
          const int q = w % R;
          const int bw = w / R;
          const int seq = bw / nb, j = bw - seq * nb;
          out_generic(a + (size_t)seq * ld, b + (size_t)seq * ld, tw, n, R, nb, Ns, j, q);
        }
      }
    }
    __syncthreads();
    cd* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

}  // namespace afft
