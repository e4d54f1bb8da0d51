// Device core of the exact-mode peeling decoder (peeling.py:270-313), shared by
// the standalone peel kernel and the fused FFAST kernel.
//
// One thread block owns one signal's graph.  Per round:
//   classify  — only live nodes whose residual changed since their last
//               classification ("dirty"): classify_exact is a pure function of
//               (residual, eps), so a clean node's cached state/f0/value equal
//               what the reference recomputes every round (peeling.py:288-295);
//   harvest   — SINGLE_TON, f0 not yet recovered, and no earlier node in
//               (cycle, bucket) order decoded the same f0 this round (296-302);
//               only bucket f0 mod b' of each earlier cycle can collide;
//   compact   — block prefix sum → found list in insertion order;
//   subtract  — nodes hit by a found tone (any state, 305-307) subtract, in
//               found order, v * exp(-2j*pi*((tau*f) mod n)/n); a gather, no
//               floating-point atomics, so the result is deterministic.
#pragma once

#include "afft_common.cuh"

namespace afft {

constexpr unsigned kEmpty = ~0u;  // hash keys are positions f < n < 2^32 - 1

struct PeelGraph {
  int64_t n;
  int ncycles;
  int nodes;
  int hmask;  // hash capacity - 1 (power of two)
  int64_t b[AFFT_MAX_CYCLES];
  int32_t base[AFFT_MAX_CYCLES + 1];  // base[ncycles..] = INT32_MAX
  int64_t tau[3];                     // exact shift set (0, 1, 2), reduced mod n
};

struct PeelLayout {
  size_t res, val, f0, found_f, found_v, found_p, found_res, hash, flag, hv, st, dirty, cyc,
      rec_f, rec_v, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// with_val: keep each node's last decoded value (the graph API writes it back);
// with_rec: keep the cumulative recovered list in the same memory.
__host__ __device__ inline PeelLayout peel_layout(int nodes, int ncycles, int hcap,
                                                  bool with_rec, bool with_val = true) {
  PeelLayout L;
  size_t o = 0;
  L.res = o;       o = align16(o + (size_t)nodes * 3 * 16);
  L.val = o;       if (with_val) o = align16(o + (size_t)nodes * 16);
  L.f0 = o;        o = align16(o + (size_t)nodes * 8);
  L.found_f = o;   o = align16(o + (size_t)nodes * 8);
  L.found_v = o;   o = align16(o + (size_t)nodes * 16);
  L.found_p = o;   o = align16(o + (size_t)nodes * 2 * 16);
  L.found_res = o; o = align16(o + (size_t)nodes * ncycles * 4);
  L.hash = o;      o = align16(o + (size_t)hcap * 4);
  L.flag = o;      o = align16(o + (size_t)nodes * 4);
  L.hv = o;        o = align16(o + (size_t)nodes);
  L.st = o;        o = align16(o + (size_t)nodes);
  L.dirty = o;     o = align16(o + (size_t)nodes);
  L.cyc = o;       o = align16(o + (size_t)nodes);
  L.rec_f = o;     if (with_rec) o = align16(o + (size_t)nodes * 8);
  L.rec_v = o;     if (with_rec) o = align16(o + (size_t)nodes * 16);
  L.total = o;
  return L;
}

struct PeelMem {
  cd* res;
  cd* val;
  int64_t* f0;
  int64_t* found_f;
  cd* found_v;
  cd* found_p;  // per found tone: v * w^{tau_1 f}, v * w^{tau_2 f} (tau_0 = 0: v itself)
  int32_t* found_res;  // per round: found-tone indices grouped by node (counting sort)
  unsigned* hash;
  int* flag;
  int8_t* hv;
  int8_t* st;
  int8_t* dirty;
  int8_t* cyc;     // node -> cycle
  cd* valp;        // node values, or null when not kept (fused kernel: value = r0)
  int64_t* rec_f;  // cumulative recovered list (insertion order)
  cd* rec_v;
};

__device__ __forceinline__ PeelMem peel_carve(unsigned char* mem, const PeelLayout& L) {
  PeelMem M;
  M.res = reinterpret_cast<cd*>(mem + L.res);
  M.val = reinterpret_cast<cd*>(mem + L.val);
  M.f0 = reinterpret_cast<int64_t*>(mem + L.f0);
  M.found_f = reinterpret_cast<int64_t*>(mem + L.found_f);
  M.found_v = reinterpret_cast<cd*>(mem + L.found_v);
  M.found_p = reinterpret_cast<cd*>(mem + L.found_p);
  M.found_res = reinterpret_cast<int32_t*>(mem + L.found_res);
  M.hash = reinterpret_cast<unsigned*>(mem + L.hash);
  M.flag = reinterpret_cast<int*>(mem + L.flag);
  M.hv = reinterpret_cast<int8_t*>(mem + L.hv);
  M.st = reinterpret_cast<int8_t*>(mem + L.st);
  M.dirty = reinterpret_cast<int8_t*>(mem + L.dirty);
  M.cyc = reinterpret_cast<int8_t*>(mem + L.cyc);
  M.valp = L.val != L.f0 ? M.val : nullptr;
  M.rec_f = reinterpret_cast<int64_t*>(mem + L.rec_f);
  M.rec_v = reinterpret_cast<cd*>(mem + L.rec_v);
  return M;
}

__device__ __forceinline__ unsigned hslot(int64_t f, int mask) {
  return (unsigned)(((unsigned long long)f * 0x9E3779B97F4A7C15ull) >> 40) & (unsigned)mask;
}
__device__ __forceinline__ bool hash_contains(const unsigned* h, int mask, int64_t f) {
  unsigned i = hslot(f, mask);
  while (true) {
    const unsigned k = h[i];
    if (k == (unsigned)f) return true;
    if (k == kEmpty) return false;
    i = (i + 1) & mask;
  }
}
__device__ __forceinline__ void hash_insert(unsigned* h, int mask, int64_t f) {
  unsigned i = hslot(f, mask);
  while (true) {
    const unsigned old = atomicCAS(h + i, kEmpty, (unsigned)f);
    if (old == kEmpty || old == (unsigned)f) return;
    i = (i + 1) & mask;
  }
}

// In-place exclusive prefix sum of a[0..N) across the block; returns the total.
// Each thread scans a contiguous chunk of ceil(N / blockDim) elements, the chunk
// sums are scanned across the block with warp shuffles: two barriers for any N.
__device__ inline int block_exclusive_scan(int* a, int N, int* warp_tmp, int* carry) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nwarps = (nt + 31) >> 5;
  const int per = (N + nt - 1) / nt;
  const int lo = min(N, tid * per), hi = min(N, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += a[i];
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nwarps ? warp_tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nwarps) warp_tmp[lane] = w;
    if (lane == 31) *carry = w;
  }
  __syncthreads();
  int run = (wid ? warp_tmp[wid - 1] : 0) + x - sum;
  for (int i = lo; i < hi; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  const int total = *carry;
  __syncthreads();  // a[] and carry are read back by the caller's next phase
  return total;
}

// classify_exact (peeling.py:193-215) for one residual (r0, r1, r2): ZERO_TON if
// ||r|| <= eps_zero; MULTI_TON unless min(|r0|,|r1|) > eps_zero, the ratio test
// |r1/r0 - r2/r1| <= eps_ratio passes and the decoded bin
// round_half_even(angle(r1/r0) * (-n / 2pi)) mod n lies in this bucket.
__device__ __forceinline__ int8_t classify_exact_dev(cd r0, cd r1, cd r2, int64_t index,
                                                     int64_t b, int64_t n, double eps0,
                                                     double epsr, double cfac, int64_t* f0,
                                                     cd* val) {
  const double sre = __dadd_rn(__dadd_rn(__dmul_rn(r0.re, r0.re), __dmul_rn(r1.re, r1.re)),
                               __dmul_rn(r2.re, r2.re));
  const double sim = __dadd_rn(__dadd_rn(__dmul_rn(r0.im, r0.im), __dmul_rn(r1.im, r1.im)),
                               __dmul_rn(r2.im, r2.im));
  if (sqrt(__dadd_rn(sre, sim)) <= eps0) return AFFT_ZERO_TON;
  if (fmin(cabs_(r0), cabs_(r1)) > eps0) {
    const cd q1 = cdiv(r1, r0);
    const cd q2 = cdiv(r2, r1);
    if (cabs_(csub(q1, q2)) <= epsr) {
      const double ang = atan2(q1.im, q1.re);
      const int64_t f = pymod((int64_t)rint(__dmul_rn(ang, cfac)), n);
      if (f % b == index) {
        *f0 = f;
        if (val) *val = r0;
        return AFFT_SINGLE_TON;
      }
    }
  }
  return AFFT_MULTI_TON;
}

__device__ __forceinline__ int cycle_of(const PeelGraph& G, int g) {
  int c = 0;
  while (g >= G.base[c + 1]) ++c;
  return c;
}

// Node -> cycle table (call once after carving, before the rounds).
__device__ inline void peel_fill_cycles(const PeelGraph& G, const PeelMem& M) {
  for (int g = threadIdx.x; g < G.nodes; g += blockDim.x) M.cyc[g] = (int8_t)cycle_of(G, g);
}

// Round loop.  Expects M.res/st/f0/(val) initialised, M.dirty = 1, M.cyc filled, the
// hash holding the rc prior recovered positions, and rec_f/rec_v (shared or global)
// holding them.  Appends newly found tones to rec_f/rec_v; returns the round count
// and updates rc.
__device__ inline int peel_rounds(const PeelGraph& G, const PeelMem& M, double eps0, double epsr,
                                  int max_rounds, int64_t* rec_f, cd* rec_v, int& rc,
                                  int* warp_tmp, int* carry) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int N = G.nodes, F = G.ncycles;
  const int64_t n = G.n;
  const double cfac = (double)(-n) / 6.283185307179586;  // -n / (2.0 * np.pi)
  int rounds = 0;
  for (int it = 0; it < max_rounds; ++it) {
    ++rounds;
    // ---- classify live, changed nodes
    for (int g = tid; g < N; g += nt) {
      const int8_t s0 = M.st[g];
      if (s0 == AFFT_RESOLVED || s0 == AFFT_ZERO_TON || !M.dirty[g]) continue;
      const int c = M.cyc[g];
      M.st[g] = classify_exact_dev(M.res[3 * g], M.res[3 * g + 1], M.res[3 * g + 2],
                                   g - G.base[c], G.b[c], n, eps0, epsr, cfac, &M.f0[g],
                                   M.valp ? &M.valp[g] : nullptr);
      M.dirty[g] = 0;
    }
    __syncthreads();
    // ---- first-found harvest
    for (int g = tid; g < N; g += nt) {
      int take = 0;
      if (M.st[g] == AFFT_SINGLE_TON) {
        const int64_t f = M.f0[g];
        if (!hash_contains(M.hash, G.hmask, f)) {
          take = 1;
          const int c = M.cyc[g];
          for (int c2 = 0; c2 < c; ++c2) {
            const int g2 = G.base[c2] + (int)(f % G.b[c2]);
            if (M.st[g2] == AFFT_SINGLE_TON && M.f0[g2] == f) {
              take = 0;
              break;
            }
          }
        }
      }
      M.hv[g] = (int8_t)take;
      M.flag[g] = take;
    }
    __syncthreads();
    const int nf = block_exclusive_scan(M.flag, N, warp_tmp, carry);
    if (nf == 0) break;
    // ---- found list in insertion order.  A SINGLE_TON's value is r0 of its current
    // residual: a node is reclassified whenever its residual changes, so r0 still
    // equals the value classify_exact stored.
    for (int g = tid; g < N; g += nt) {
      if (M.hv[g]) {
        const int pos = M.flag[g];
        M.found_f[pos] = M.f0[g];
        M.found_v[pos] = M.res[3 * g];
        M.st[g] = AFFT_RESOLVED;
        M.hv[g] = 0;
      }
      M.flag[g] = 0;
    }
    __syncthreads();
    // ---- per found tone (convergent): v * w^{(tau_r f) mod n}, r = 1, 2 (tau_0 = 0);
    //      and the per-node hit counts of the (tone, cycle) pairs
    for (int i = tid; i < nf; i += nt) {
      const int64_t f = M.found_f[i];
      const cd v = M.found_v[i];
      M.found_p[2 * i] = cmul(v, unit_root(mulmod(G.tau[1], f, n), n));
      M.found_p[2 * i + 1] = cmul(v, unit_root(mulmod(G.tau[2], f, n), n));
    }
    for (int e = tid; e < nf * F; e += nt) {
      const int i = e / F, c = e - i * F;
      atomicAdd(&M.flag[G.base[c] + (int)(M.found_f[i] % G.b[c])], 1);
    }
    __syncthreads();
    block_exclusive_scan(M.flag, N, warp_tmp, carry);  // segment starts
    for (int e = tid; e < nf * F; e += nt) {             // scatter (unordered within a node)
      const int i = e / F, c = e - i * F;
      const int slot = atomicAdd(&M.flag[G.base[c] + (int)(M.found_f[i] % G.b[c])], 1);
      M.found_res[slot] = i;
    }
    __syncthreads();
    // ---- subtract: each hit node applies its tones in found order (peeling.py:305-307)
    for (int g = tid; g < N; g += nt) {
      const int lo = g ? M.flag[g - 1] : 0, hi = M.flag[g];
      if (lo == hi) continue;
      for (int a = lo + 1; a < hi; ++a) {  // insertion sort of the (short) segment
        const int v = M.found_res[a];
        int b = a - 1;
        while (b >= lo && M.found_res[b] > v) {
          M.found_res[b + 1] = M.found_res[b];
          --b;
        }
        M.found_res[b + 1] = v;
      }
      cd a0 = M.res[3 * g], a1 = M.res[3 * g + 1], a2 = M.res[3 * g + 2];
      for (int a = lo; a < hi; ++a) {
        const int i = M.found_res[a];
        a0 = csub(a0, M.found_v[i]);  // v * (1, -0) == v exactly
        a1 = csub(a1, M.found_p[2 * i]);
        a2 = csub(a2, M.found_p[2 * i + 1]);
      }
      M.res[3 * g] = a0;
      M.res[3 * g + 1] = a1;
      M.res[3 * g + 2] = a2;
      M.dirty[g] = 1;
    }
    for (int i = tid; i < nf; i += nt) {
      hash_insert(M.hash, G.hmask, M.found_f[i]);
      rec_f[rc + i] = M.found_f[i];
      rec_v[rc + i] = M.found_v[i];
    }
    rc += nf;
    __syncthreads();
  }
  return rounds;
}

// Number of MULTI_TON nodes (peeling.py:309-311); all threads get the total.
__device__ inline int count_multitons(const PeelGraph& G, const PeelMem& M, int* red) {
  if (threadIdx.x == 0) *red = 0;
  __syncthreads();
  int cnt = 0;
  for (int g = threadIdx.x; g < G.nodes; g += blockDim.x) cnt += M.st[g] == AFFT_MULTI_TON;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(red, cnt);
  __syncthreads();
  return *red;
}

// truncate_spectrum order (oneshot.py:260-263) by an in-smem bitonic sort of
// (|v| descending, f ascending) keys; pads to a power of two with sentinels.
// key/pos/idx need pow2 entries.  All threads must call it.
__device__ inline void bitonic_trunc_sort(double* key, int64_t* pos, int32_t* idx, int m,
                                          int pow2) {
  for (int i = threadIdx.x + m; i < pow2; i += blockDim.x) {
    key[i] = -1.0;
    pos[i] = INT64_MAX;
    idx[i] = -1;
  }
  __syncthreads();
  for (int k = 2; k <= pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          // "a before b" iff a.key > b.key, or equal keys and a.pos < b.pos
          const bool lbefore = key[l] > key[i] || (key[l] == key[i] && pos[l] < pos[i]);
          const bool up = (i & k) == 0;
          if (up == lbefore) {
            const double tk = key[i];
            key[i] = key[l];
            key[l] = tk;
            const int64_t tp = pos[i];
            pos[i] = pos[l];
            pos[l] = tp;
            const int32_t ti = idx[i];
            idx[i] = idx[l];
            idx[l] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
}

// truncate_spectrum (oneshot.py:260-263): rank of entry i by (-|v|, f).
__device__ __forceinline__ int trunc_rank(const double* mag, const int64_t* fs, int m, int i) {
  const double a = mag[i];
  const int64_t f = fs[i];
  int rank = 0;
  for (int j = 0; j < m; ++j) {
    const double b = mag[j];
    rank += (b > a) || (b == a && fs[j] < f);
  }
  return rank;
}

}  // namespace afft
