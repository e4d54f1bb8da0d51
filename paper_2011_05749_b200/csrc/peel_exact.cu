// K3 (exact) + K4: GPU-resident synchronous peeling decoder for FFAST.
//
// Device restatement of peel_decode (peeling.py:270-313) in exact mode, with
// classify_exact (193-215) and subtract/_tone_vector (181-190).  One CTA owns
// one signal's whole graph in shared memory and runs every round without a
// host round-trip:
//   classify  — one thread per live node (RESOLVED / ZERO_TON are skipped for
//               good, 290-291); numpy-faithful complex division, hypot, atan2
//               and round-half-even for the bin decode (210);
//   harvest   — a SINGLE_TON whose f0 is not yet recovered is harvested iff no
//               earlier node in (cycle, bucket) order decoded the same f0 this
//               round (the first-found rule of 296-302).  Two nodes of one cycle
//               can never share f0 (f0 mod b == bucket), so only bucket f0 mod b'
//               of each earlier cycle needs checking;
//   compact   — block prefix sum over nodes gives the found list in insertion
//               order;
//   subtract  — every node (RESOLVED and ZERO_TON included, 305-307) subtracts
//               the found tones of its residue in found order: a deterministic
//               gather, no floating-point atomics.
// The recovered set is an open-addressing hash in shared memory plus the
// insertion-ordered (pos, value) list written to global memory.
#include <algorithm>

#include "afft_common.cuh"

namespace afft {

constexpr unsigned long long kEmpty = ~0ull;

struct ShiftList {
  int64_t tau[AFFT_MAX_SHIFTS];  // reduced mod n
};

struct PeelParams {
  int64_t n;
  int ncycles;
  int nodes;
  int64_t b[AFFT_MAX_CYCLES];
  int32_t base[AFFT_MAX_CYCLES + 1];
  int64_t tau[3];  // exact shift set (0, 1, 2), reduced mod n
  double* residual;
  int8_t* state;
  int64_t* node_f0;
  double* node_val;
  const double* eps_zero;
  const double* eps_ratio;
  int max_rounds;
  int64_t* rec_pos;
  double* rec_val;
  int rec_cap;
  int32_t* rec_count;
  int32_t* rounds;
  int32_t* unresolved;
  int hmask;        // hash capacity - 1 (power of two)
  int writeback;    // copy residual/state/f0/value back to global
  char* gscratch;   // per-CTA scratch in global memory when smem is too small
  size_t scratch_bytes;
};

struct PeelLayout {
  size_t res, val, f0, found_f, found_v, found_res, hash, flag, hv, st, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline PeelLayout peel_layout(int nodes, int ncycles, int hcap) {
  PeelLayout L;
  size_t o = 0;
  L.res = o;       o = align16(o + (size_t)nodes * 3 * 16);
  L.val = o;       o = align16(o + (size_t)nodes * 16);
  L.f0 = o;        o = align16(o + (size_t)nodes * 8);
  L.found_f = o;   o = align16(o + (size_t)nodes * 8);
  L.found_v = o;   o = align16(o + (size_t)nodes * 16);
  L.found_res = o; o = align16(o + (size_t)nodes * ncycles * 4);
  L.hash = o;      o = align16(o + (size_t)hcap * 8);
  L.flag = o;      o = align16(o + (size_t)nodes * 4);
  L.hv = o;        o = align16(o + (size_t)nodes);
  L.st = o;        o = align16(o + (size_t)nodes);
  L.total = o;
  return L;
}

__device__ __forceinline__ unsigned hslot(int64_t f, int mask) {
  return (unsigned)(((unsigned long long)f * 0x9E3779B97F4A7C15ull) >> 40) & (unsigned)mask;
}
__device__ __forceinline__ bool hash_contains(const unsigned long long* h, int mask, int64_t f) {
  unsigned i = hslot(f, mask);
  while (true) {
    unsigned long long k = h[i];
    if (k == (unsigned long long)f) return true;
    if (k == kEmpty) return false;
    i = (i + 1) & mask;
  }
}
__device__ __forceinline__ void hash_insert(unsigned long long* h, int mask, int64_t f) {
  unsigned i = hslot(f, mask);
  while (true) {
    unsigned long long old = atomicCAS(h + i, kEmpty, (unsigned long long)f);
    if (old == kEmpty || old == (unsigned long long)f) return;
    i = (i + 1) & mask;
  }
}

// In-place exclusive prefix sum of a[0..N) across the block; returns the total.
__device__ int block_exclusive_scan(int* a, int N, int* warp_tmp, int* carry) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nwarps = (nt + 31) >> 5;
  if (tid == 0) *carry = 0;
  __syncthreads();
  for (int base = 0; base < N; base += nt) {
    const int i = base + tid;
    const int v = i < N ? a[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = lane < nwarps ? warp_tmp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nwarps) warp_tmp[lane] = w;
    }
    __syncthreads();
    const int c = *carry;
    const int wprefix = wid > 0 ? warp_tmp[wid - 1] : 0;
    if (i < N) a[i] = c + wprefix + x - v;
    __syncthreads();
    if (tid == 0) *carry = c + warp_tmp[nwarps - 1];
    __syncthreads();
  }
  return *carry;
}

// classify_exact (peeling.py:193-215) for one node's residual (r0, r1, r2):
// ZERO_TON if ||r|| <= eps_zero; else MULTI_TON unless the ratio test passes and
// the decoded bin round(angle(r1/r0) * (-n / 2pi)) mod n lies in this bucket.
// On SINGLE_TON writes f0 and value = r0.
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
        *val = r0;
        return AFFT_SINGLE_TON;
      }
    }
  }
  return AFFT_MULTI_TON;
}

__device__ __forceinline__ int cycle_of(const PeelParams& p, int g) {
  int c = 0;
  while (g >= p.base[c + 1]) ++c;
  return c;
}

__global__ void __launch_bounds__(256) peel_exact_kernel(const __grid_constant__ PeelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry;
  __shared__ int red;
  const int64_t s = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int N = p.nodes, F = p.ncycles;
  const int64_t n = p.n;
  const int hcap = p.hmask + 1;
  unsigned char* mem = p.gscratch ? reinterpret_cast<unsigned char*>(p.gscratch) +
                                        (size_t)s * p.scratch_bytes
                                  : smem_raw;
  const PeelLayout L = peel_layout(N, F, hcap);
  cd* res = reinterpret_cast<cd*>(mem + L.res);
  cd* val = reinterpret_cast<cd*>(mem + L.val);
  int64_t* f0 = reinterpret_cast<int64_t*>(mem + L.f0);
  int64_t* found_f = reinterpret_cast<int64_t*>(mem + L.found_f);
  cd* found_v = reinterpret_cast<cd*>(mem + L.found_v);
  int32_t* found_res = reinterpret_cast<int32_t*>(mem + L.found_res);
  unsigned long long* hash = reinterpret_cast<unsigned long long*>(mem + L.hash);
  int* flag = reinterpret_cast<int*>(mem + L.flag);
  int8_t* hv = reinterpret_cast<int8_t*>(mem + L.hv);
  int8_t* st = reinterpret_cast<int8_t*>(mem + L.st);

  const cd* gres = reinterpret_cast<const cd*>(p.residual) + s * (int64_t)N * 3;
  for (int e = tid; e < N * 3; e += nt) res[e] = gres[e];
  for (int g = tid; g < N; g += nt) {
    st[g] = p.state[s * N + g];
    f0[g] = p.node_f0 ? p.node_f0[s * N + g] : -1;
    val[g] = p.node_val ? reinterpret_cast<const cd*>(p.node_val)[s * N + g] : cd{0.0, 0.0};
  }
  for (int h = tid; h < hcap; h += nt) hash[h] = kEmpty;
  __syncthreads();
  const int rc0 = p.rec_count[s];
  int64_t* rpos = p.rec_pos + s * (int64_t)p.rec_cap;
  cd* rval = reinterpret_cast<cd*>(p.rec_val) + s * (int64_t)p.rec_cap;
  for (int i = tid; i < rc0; i += nt) hash_insert(hash, p.hmask, rpos[i]);
  __syncthreads();

  const double eps0 = p.eps_zero[s], epsr = p.eps_ratio[s];
  const double cfac = (double)(-n) / 6.283185307179586;  // -n / (2.0 * np.pi)
  int rc = rc0;
  int rounds = 0;
  for (int it = 0; it < p.max_rounds; ++it) {
    ++rounds;
    // ---- classify every live node (classify_exact, peeling.py:193-215)
    for (int g = tid; g < N; g += nt) {
      const int8_t s0 = st[g];
      if (s0 == AFFT_RESOLVED || s0 == AFFT_ZERO_TON) continue;
      const int c = cycle_of(p, g);
      st[g] = classify_exact_dev(res[3 * g], res[3 * g + 1], res[3 * g + 2], g - p.base[c],
                                 p.b[c], n, eps0, epsr, cfac, &f0[g], &val[g]);
    }
    __syncthreads();
    // ---- first-found harvest (peeling.py:296-302)
    for (int g = tid; g < N; g += nt) {
      int take = 0;
      if (st[g] == AFFT_SINGLE_TON) {
        const int64_t f = f0[g];
        if (!hash_contains(hash, p.hmask, f)) {
          take = 1;
          const int c = cycle_of(p, g);
          for (int c2 = 0; c2 < c; ++c2) {
            const int g2 = p.base[c2] + (int)(f % p.b[c2]);
            if (st[g2] == AFFT_SINGLE_TON && f0[g2] == f) {
              take = 0;
              break;
            }
          }
        }
      }
      hv[g] = (int8_t)take;
      flag[g] = take;
    }
    __syncthreads();
    const int nf = block_exclusive_scan(flag, N, warp_tmp, &carry);
    if (nf == 0) break;
    for (int g = tid; g < N; g += nt) {
      if (hv[g]) {
        const int pos = flag[g];
        found_f[pos] = f0[g];
        found_v[pos] = val[g];
        st[g] = AFFT_RESOLVED;
      }
    }
    __syncthreads();
    for (int e = tid; e < nf * F; e += nt) {
      const int i = e / F, c = e - i * F;
      found_res[e] = (int32_t)(found_f[i] % p.b[c]);
    }
    __syncthreads();
    // ---- subtract in found order from every cycle (peeling.py:305-307)
    for (int g = tid; g < N; g += nt) {
      const int c = cycle_of(p, g);
      const int idx = g - p.base[c];
      cd a0 = res[3 * g], a1 = res[3 * g + 1], a2 = res[3 * g + 2];
      bool touched = false;
      for (int i = 0; i < nf; ++i) {
        if (found_res[i * F + c] != idx) continue;
        touched = true;
        const int64_t f = found_f[i];
        const cd v = found_v[i];
        a0 = csub(a0, cmul(v, unit_root(mulmod(p.tau[0], f, n), n)));
        a1 = csub(a1, cmul(v, unit_root(mulmod(p.tau[1], f, n), n)));
        a2 = csub(a2, cmul(v, unit_root(mulmod(p.tau[2], f, n), n)));
      }
      if (touched) {
        res[3 * g] = a0;
        res[3 * g + 1] = a1;
        res[3 * g + 2] = a2;
      }
    }
    for (int i = tid; i < nf; i += nt) {
      hash_insert(hash, p.hmask, found_f[i]);
      rpos[rc + i] = found_f[i];
      rval[rc + i] = found_v[i];
    }
    rc += nf;
    __syncthreads();
  }
  // ---- unresolved multi-tons (peeling.py:309-311) and write-back
  if (tid == 0) red = 0;
  __syncthreads();
  int cnt = 0;
  for (int g = tid; g < N; g += nt) cnt += st[g] == AFFT_MULTI_TON;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((tid & 31) == 0 && cnt) atomicAdd(&red, cnt);
  __syncthreads();
  if (tid == 0) {
    p.rec_count[s] = rc;
    if (p.rounds) p.rounds[s] = rounds;
    if (p.unresolved) p.unresolved[s] = red;
  }
  if (p.writeback) {
    cd* gw = reinterpret_cast<cd*>(p.residual) + s * (int64_t)N * 3;
    for (int e = tid; e < N * 3; e += nt) gw[e] = res[e];
    for (int g = tid; g < N; g += nt) {
      p.state[s * N + g] = st[g];
      if (p.node_f0) p.node_f0[s * N + g] = f0[g];
      if (p.node_val) reinterpret_cast<cd*>(p.node_val)[s * N + g] = val[g];
    }
  }
}

// Node-batched classify_exact for the per-node API (peeling.py:193-215).
__global__ void classify_exact_kernel(const double* __restrict__ residual,
                                      const int64_t* __restrict__ index, int64_t count, int64_t b,
                                      int64_t n, double eps0, double epsr,
                                      int8_t* __restrict__ state, int64_t* __restrict__ f0,
                                      double* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const cd* r = reinterpret_cast<const cd*>(residual) + 3 * i;
  const double cfac = (double)(-n) / 6.283185307179586;
  int64_t f = f0[i];
  cd v = reinterpret_cast<cd*>(val)[i];
  state[i] = classify_exact_dev(r[0], r[1], r[2], index[i], b, n, eps0, epsr, cfac, &f, &v);
  f0[i] = f;
  reinterpret_cast<cd*>(val)[i] = v;
}

// subtract (peeling.py:186-190): residual[i] -= value[i] * exp(-2j*pi*((tau*f) mod n)/n).
__global__ void subtract_kernel(double* __restrict__ residual, int nshift,
                                const int64_t* __restrict__ f, const double* __restrict__ value,
                                int64_t count, int64_t n, const __grid_constant__ ShiftList taus) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count * nshift) return;
  const int64_t i = e / nshift;
  const int r = (int)(e - i * nshift);
  cd* res = reinterpret_cast<cd*>(residual) + e;
  const cd v = reinterpret_cast<const cd*>(value)[i];
  *res = csub(*res, cmul(v, unit_root(mulmod(taus.tau[r], pymod(f[i], n), n), n)));
}

// truncate_spectrum (oneshot.py:260-263): rank by (-|v|, f), keep the first k.
__global__ void truncate_kernel(const int64_t* __restrict__ pos, const double* __restrict__ val,
                                const int32_t* __restrict__ count, int cap, int k,
                                int64_t* __restrict__ out_pos, double* __restrict__ out_val,
                                int32_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t s = blockIdx.x;
  const int m = count[s];
  double* mag = reinterpret_cast<double*>(smem_raw);
  int64_t* fs = reinterpret_cast<int64_t*>(mag + cap);
  const int64_t* ps = pos + s * cap;
  const cd* vs = reinterpret_cast<const cd*>(val) + s * cap;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    mag[i] = cabs_(vs[i]);
    fs[i] = ps[i];
  }
  __syncthreads();
  cd* ov = reinterpret_cast<cd*>(out_val) + s * k;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double a = mag[i];
    const int64_t f = fs[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double b = mag[j];
      rank += (b > a) || (b == a && fs[j] < f);
    }
    if (rank < k) {
      out_pos[s * k + rank] = f;
      ov[rank] = vs[i];
    }
  }
  if (threadIdx.x == 0) out_count[s] = m < k ? m : k;
}

struct PeelSetup {
  PeelParams p;
  size_t smem;
  bool fits;
};

static int setup_peel(PeelSetup* S, int64_t n, const int64_t* factors, int ncycles, int rec_cap) {
  PeelParams& p = S->p;
  memset(&p, 0, sizeof(p));
  if (ncycles < 1 || ncycles > AFFT_MAX_CYCLES || !factors) {
    set_error("number of cycles %d outside 1..%d", ncycles, AFFT_MAX_CYCLES);
    return AFFT_EUNSUPPORTED;
  }
  if (n < 1 || n > 3000000000LL) {
    set_error("signal size %lld outside the supported 1..3e9", (long long)n);
    return AFFT_EUNSUPPORTED;
  }
  p.n = n;
  p.ncycles = ncycles;
  int64_t total = 0;
  for (int c = 0; c < ncycles; ++c) {
    if (factors[c] < 1 || n % factors[c]) {
      set_error("bucket count %lld does not divide signal size %lld", (long long)factors[c],
                (long long)n);
      return AFFT_EINVAL;
    }
    p.b[c] = factors[c];
    p.base[c] = (int32_t)total;
    total += factors[c];
  }
  if (total > (1 << 24)) {
    set_error("graph with %lld nodes is too large", (long long)total);
    return AFFT_EUNSUPPORTED;
  }
  p.base[ncycles] = (int32_t)total;
  for (int c = ncycles + 1; c <= AFFT_MAX_CYCLES; ++c) p.base[c] = INT32_MAX;
  p.nodes = (int)total;
  p.tau[0] = 0;
  p.tau[1] = 1 % n;
  p.tau[2] = 2 % n;
  int hcap = 16;
  while (hcap < 2 * rec_cap) hcap <<= 1;
  p.hmask = hcap - 1;
  p.rec_cap = rec_cap;
  PeelLayout L = peel_layout(p.nodes, ncycles, hcap);
  S->smem = L.total;
  S->fits = L.total <= 200 * 1024;
  p.scratch_bytes = L.total;
  return AFFT_OK;
}

static int launch_peel(PeelSetup& S, int64_t batch, void* scratch, cudaStream_t stream) {
  PeelParams& p = S.p;
  size_t dyn = 0;
  if (S.fits) {
    p.gscratch = nullptr;
    dyn = S.smem;
    cudaError_t e = cudaFuncSetAttribute(peel_exact_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(peel_exact)");
  } else {
    if (!scratch) {
      set_error("peeling graph does not fit in shared memory and no scratch was given");
      return AFFT_ENOMEM;
    }
    p.gscratch = reinterpret_cast<char*>(scratch);
  }
  peel_exact_kernel<<<(unsigned)batch, 256, dyn, stream>>>(p);
  AFFT_CHECK_LAUNCH("peel_exact_kernel");
  return AFFT_OK;
}

static int launch_truncate(const int64_t* pos, const double* val, const int32_t* count, int cap,
                           int64_t batch, int k, int64_t* out_pos, double* out_val,
                           int32_t* out_count, cudaStream_t stream) {
  const size_t smem = (size_t)cap * 16;
  if (smem > 200 * 1024) {
    set_error("truncate: %d entries per signal exceed the shared-memory ranker", cap);
    return AFFT_EUNSUPPORTED;
  }
  cudaError_t e = cudaFuncSetAttribute(truncate_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(truncate)");
  truncate_kernel<<<(unsigned)batch, 256, smem, stream>>>(pos, val, count, cap, k, out_pos,
                                                           out_val, out_count);
  AFFT_CHECK_LAUNCH("truncate_kernel");
  return AFFT_OK;
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct FfastWs {
  size_t partials, eps, nodes, state, rec_pos, rec_val, rec_count, rounds, unres, scratch, total;
};

static FfastWs ffast_ws(int64_t n, int dtype, int64_t batch, int64_t nodes, size_t scratch_cta) {
  FfastWs w;
  size_t o = 0;
  const int nparts = afft_sumsq_parts(n, dtype);
  w.partials = o;  o = al256(o + (size_t)batch * nparts * 8);
  w.eps = o;       o = al256(o + (size_t)batch * 8);
  w.nodes = o;     o = al256(o + (size_t)batch * nodes * 48);
  w.state = o;     o = al256(o + (size_t)batch * nodes);
  w.rec_pos = o;   o = al256(o + (size_t)batch * nodes * 8);
  w.rec_val = o;   o = al256(o + (size_t)batch * nodes * 16);
  w.rec_count = o; o = al256(o + (size_t)batch * 4);
  w.rounds = o;    o = al256(o + (size_t)batch * 4);
  w.unres = o;     o = al256(o + (size_t)batch * 4);
  w.scratch = o;   o = al256(o + (size_t)batch * scratch_cta);
  w.total = o;
  return w;
}

}  // namespace afft

using namespace afft;

extern "C" int afft_peel_exact(int64_t n, int64_t batch, const int64_t* factors, int32_t ncycles,
                               double* residual, int8_t* state, int64_t* node_f0,
                               double* node_val, const double* eps_zero,
                               const double* eps_ratio, int32_t max_rounds, int64_t* rec_pos,
                               double* rec_val, int32_t rec_cap, int32_t* rec_count,
                               int32_t* rounds, int32_t* unresolved, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!residual || !state || !eps_zero || !eps_ratio || !rec_pos || !rec_val || !rec_count ||
      batch < 0 || max_rounds < 0) {
    set_error("afft_peel_exact: bad arguments");
    return AFFT_EINVAL;
  }
  PeelSetup S;
  int rc = setup_peel(&S, n, factors, ncycles, rec_cap);
  if (rc) return rc;
  if (rec_cap < S.p.nodes) {
    set_error("rec_cap %d must be at least the node count %d plus prior entries", rec_cap,
              S.p.nodes);
    return AFFT_EINVAL;
  }
  PeelParams& p = S.p;
  p.residual = residual;
  p.state = state;
  p.node_f0 = node_f0;
  p.node_val = node_val;
  p.eps_zero = eps_zero;
  p.eps_ratio = eps_ratio;
  p.max_rounds = max_rounds;
  p.rec_pos = rec_pos;
  p.rec_val = rec_val;
  p.rec_count = rec_count;
  p.rounds = rounds;
  p.unresolved = unresolved;
  p.writeback = 1;
  cudaStream_t st = (cudaStream_t)stream;
  void* scratch = nullptr;
  if (!S.fits) {
    cudaError_t e = cudaMallocAsync(&scratch, (size_t)batch * S.smem, st);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(peel scratch)");
  }
  rc = launch_peel(S, batch, scratch, st);
  if (scratch) cudaFreeAsync(scratch, st);
  return rc;
}

extern "C" int afft_truncate(const int64_t* pos, const double* val, const int32_t* count,
                             int32_t cap, int64_t batch, int32_t k, int64_t* out_pos,
                             double* out_val, int32_t* out_count, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!pos || !val || !count || (k > 0 && (!out_pos || !out_val)) || !out_count || k < 0 ||
      cap < 0) {
    set_error("afft_truncate: bad arguments");
    return AFFT_EINVAL;
  }
  return launch_truncate(pos, val, count, cap, batch, k, out_pos, out_val, out_count,
                         (cudaStream_t)stream);
}

extern "C" size_t afft_ffast_workspace_size(int64_t n, int dtype, int64_t batch,
                                            const int64_t* factors, int32_t ncycles) {
  PeelSetup S;
  int64_t nodes = 0;
  for (int c = 0; c < ncycles && factors; ++c) nodes += factors[c];
  if (setup_peel(&S, n, factors, ncycles, (int)std::max<int64_t>(nodes, 1))) return 0;
  return ffast_ws(n, dtype, batch, nodes, S.fits ? 0 : S.smem).total;
}

extern "C" int afft_ffast(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                          const int64_t* factors, int32_t ncycles, int32_t k,
                          int32_t max_rounds, int64_t* out_pos, double* out_val,
                          int32_t* out_count, int64_t* all_pos, double* all_val,
                          int32_t* all_count, int32_t* rounds, int32_t* unresolved,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!x || (k > 0 && (!out_pos || !out_val)) || !out_count || k < 0 || batch < 0) {
    set_error("afft_ffast: bad arguments");
    return AFFT_EINVAL;
  }
  int64_t nodes = 0;
  for (int c = 0; c < ncycles && factors; ++c) nodes += factors[c];
  PeelSetup S;
  int rc = setup_peel(&S, n, factors, ncycles, (int)std::max<int64_t>(nodes, 1));
  if (rc) return rc;
  const FfastWs w = ffast_ws(n, dtype, batch, nodes, S.fits ? 0 : S.smem);
  if (!workspace || workspace_bytes < w.total) {
    set_error("afft_ffast: workspace of %zu bytes needed, %zu given", w.total, workspace_bytes);
    return AFFT_ENOMEM;
  }
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t st = (cudaStream_t)stream;
  const int nparts = afft_sumsq_parts(n, dtype);
  double* partials = reinterpret_cast<double*>(ws + w.partials);
  double* eps = reinterpret_cast<double*>(ws + w.eps);
  double* nodebuf = reinterpret_cast<double*>(ws + w.nodes);
  int8_t* state = reinterpret_cast<int8_t*>(ws + w.state);
  int64_t* rpos = all_pos ? all_pos : reinterpret_cast<int64_t*>(ws + w.rec_pos);
  double* rval = all_val ? all_val : reinterpret_cast<double*>(ws + w.rec_val);
  int32_t* rcount = all_count ? all_count : reinterpret_cast<int32_t*>(ws + w.rec_count);
  int32_t* rr = rounds ? rounds : reinterpret_cast<int32_t*>(ws + w.rounds);
  int32_t* un = unresolved ? unresolved : reinterpret_cast<int32_t*>(ws + w.unres);

  if ((rc = afft_sumsq(x, dtype, n, batch, ld, partials, st))) return rc;
  if ((rc = afft_exact_thresholds(partials, nparts, n, batch, eps, st))) return rc;
  const int64_t shifts[3] = {0, 1, 2};
  if ((rc = afft_build_graph(x, dtype, n, batch, ld, factors, ncycles, shifts, 3, nodebuf, st)))
    return rc;
  cudaError_t e = cudaMemsetAsync(state, 0, (size_t)batch * nodes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(rcount, 0, (size_t)batch * 4, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(ffast)");
  PeelParams& p = S.p;
  p.residual = nodebuf;
  p.state = state;
  p.node_f0 = nullptr;
  p.node_val = nullptr;
  p.eps_zero = eps;
  p.eps_ratio = eps;
  p.max_rounds = max_rounds > 0 ? max_rounds : k + 4;
  p.rec_pos = rpos;
  p.rec_val = rval;
  p.rec_count = rcount;
  p.rounds = rr;
  p.unresolved = un;
  p.writeback = 0;
  if ((rc = launch_peel(S, batch, ws + w.scratch, st))) return rc;
  return launch_truncate(rpos, rval, rcount, (int)nodes, batch, k, out_pos, out_val, out_count,
                         st);
}

extern "C" int afft_classify_exact(const double* residual, const int64_t* index, int64_t count,
                                   int64_t b, int64_t n, double eps_zero, double eps_ratio,
                                   int8_t* state, int64_t* f0, double* val, void* stream) {
  if (count == 0) return AFFT_OK;
  if (!residual || !index || !state || !f0 || !val || count < 0 || b < 1 || n < 1) {
    set_error("afft_classify_exact: bad arguments");
    return AFFT_EINVAL;
  }
  const int threads = 128;
  classify_exact_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0,
                          (cudaStream_t)stream>>>(residual, index, count, b, n, eps_zero,
                                                  eps_ratio, state, f0, val);
  AFFT_CHECK_LAUNCH("classify_exact_kernel");
  return AFFT_OK;
}

extern "C" int afft_subtract(double* residual, const int64_t* shifts, int32_t nshift,
                             const int64_t* f, const double* value, int64_t count, int64_t n,
                             void* stream) {
  if (count == 0 || nshift == 0) return AFFT_OK;
  if (!residual || !shifts || !f || !value || count < 0 || n < 1 || nshift < 0 ||
      nshift > AFFT_MAX_SHIFTS) {
    set_error("afft_subtract: bad arguments");
    return AFFT_EINVAL;
  }
  ShiftList t;
  for (int r = 0; r < nshift; ++r) t.tau[r] = host_pymod(shifts[r], n);
  const int threads = 128;
  const int64_t total = count * nshift;
  subtract_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0,
                    (cudaStream_t)stream>>>(residual, nshift, f, value, count, n, t);
  AFFT_CHECK_LAUNCH("subtract_kernel");
  return AFFT_OK;
}
