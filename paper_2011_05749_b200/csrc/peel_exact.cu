// K3 (exact) + K4: GPU-resident peeling for FFAST, and the fused FFAST kernel.
//
//   peel_exact_kernel   — peel_decode(mode="exact") (peeling.py:270-313) over a
//                         graph already in global memory (the drop-in API path);
//   ffast_fused_kernel  — ffast (peeling.py:321-332) for one signal per CTA:
//                         |x|^2 stream → eps (316-318) → gather + DFT of every
//                         cycle (169-178) → peel → top-k truncation
//                         (oneshot.py:260-263).  The decode of one CTA overlaps
//                         the HBM streaming of the others, so the kernel runs at
//                         the stream's roofline with a single launch per batch;
//   classify / subtract / truncate kernels for the per-node API.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "afft_common.cuh"
#include "gather_dft.cuh"
#include "peel_core.cuh"

namespace afft {

struct ShiftList {
  int64_t tau[AFFT_MAX_SHIFTS];  // reduced mod n
};

// ------------------------------------------------------------------ standalone peel

struct PeelParams {
  PeelGraph G;
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
  int writeback;
  char* gscratch;  // per-CTA scratch in global memory when smem is too small
  size_t scratch_bytes;
};

__global__ void __launch_bounds__(256) peel_exact_kernel(const __grid_constant__ PeelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry, red;
  const int64_t s = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const PeelGraph& G = p.G;
  const int N = G.nodes;
  unsigned char* mem =
      p.gscratch ? reinterpret_cast<unsigned char*>(p.gscratch) + (size_t)s * p.scratch_bytes
                 : smem_raw;
  const PeelLayout L = peel_layout(N, G.ncycles, G.hmask + 1, false);
  const PeelMem M = peel_carve(mem, L);

  const cd* gres = reinterpret_cast<const cd*>(p.residual) + s * (int64_t)N * 3;
  for (int e = tid; e < N * 3; e += nt) M.res[e] = gres[e];
  for (int g = tid; g < N; g += nt) {
    M.st[g] = p.state[s * N + g];
    M.dirty[g] = 1;
    M.hv[g] = 0;
    M.f0[g] = p.node_f0 ? p.node_f0[s * N + g] : -1;
    M.val[g] = p.node_val ? reinterpret_cast<const cd*>(p.node_val)[s * N + g] : cd{0.0, 0.0};
  }
  for (int h = tid; h <= G.hmask; h += nt) M.hash[h] = kEmpty;
  peel_fill_cycles(G, M);
  __syncthreads();
  int rc = p.rec_count[s];
  int64_t* rpos = p.rec_pos + s * (int64_t)p.rec_cap;
  cd* rval = reinterpret_cast<cd*>(p.rec_val) + s * (int64_t)p.rec_cap;
  for (int i = tid; i < rc; i += nt) hash_insert(M.hash, G.hmask, rpos[i]);
  __syncthreads();

  const int rounds = peel_rounds(G, M, p.eps_zero[s], p.eps_ratio[s], p.max_rounds, rpos, rval,
                                 rc, warp_tmp, &carry);
  const int unres = count_multitons(G, M, &red);
  if (tid == 0) {
    p.rec_count[s] = rc;
    if (p.rounds) p.rounds[s] = rounds;
    if (p.unresolved) p.unresolved[s] = unres;
  }
  if (p.writeback) {
    cd* gw = reinterpret_cast<cd*>(p.residual) + s * (int64_t)N * 3;
    for (int e = tid; e < N * 3; e += nt) gw[e] = M.res[e];
    for (int g = tid; g < N; g += nt) {
      p.state[s * N + g] = M.st[g];
      if (p.node_f0) p.node_f0[s * N + g] = M.f0[g];
      if (p.node_val) reinterpret_cast<cd*>(p.node_val)[s * N + g] = M.val[g];
    }
  }
}

// ------------------------------------------------------------------ tree walk
//
// The paper's Fig. 5 "sparse-graph decoder by packet erasure channel method"
// (a non-goal of the reference, "identical output to
// Fig. 4 with fewer identifications"): instead of re-identifying every live check node
// each round (peeling.py:288-295), paths are extended from single-ton check nodes —
// identify the left node (the tone), subtract it from its d right neighbours, and
// re-identify only those; a neighbour that becomes a single-ton extends the path.
// A FIFO queue of single-ton nodes per signal (one CTA per signal; the initial
// identification of every node is parallel, the walk itself sequential on one thread,
// which is what the method is).  Exact mode, shifts (0, 1, 2).  The recovered set
// equals the round decoder's (tests/test_gpu_ffast.py); the order is the walk's, and
// the values differ from the rounds' by the rounding of the subtraction order.
// rounds[s] = the longest path (queue generations), ident[s] = identifications.
__global__ void __launch_bounds__(256) peel_tree_kernel(const __grid_constant__ PeelParams p,
                                                        int32_t* __restrict__ ident) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry, red, nq0, nident;
  const int64_t s = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const PeelGraph& G = p.G;
  const int N = G.nodes, F = G.ncycles;
  const int64_t n = G.n;
  unsigned char* mem =
      p.gscratch ? reinterpret_cast<unsigned char*>(p.gscratch) + (size_t)s * p.scratch_bytes
                 : smem_raw;
  const PeelLayout L = peel_layout(N, G.ncycles, G.hmask + 1, false);
  const PeelMem M = peel_carve(mem, L);
  const cd* gres = reinterpret_cast<const cd*>(p.residual) + s * (int64_t)N * 3;
  for (int e = tid; e < N * 3; e += nt) M.res[e] = gres[e];
  for (int g = tid; g < N; g += nt) {
    M.st[g] = p.state[s * N + g];
    M.hv[g] = 0;  // in the queue
    M.f0[g] = p.node_f0 ? p.node_f0[s * N + g] : -1;
    M.val[g] = p.node_val ? reinterpret_cast<const cd*>(p.node_val)[s * N + g] : cd{0.0, 0.0};
  }
  for (int h = tid; h <= G.hmask; h += nt) M.hash[h] = kEmpty;
  peel_fill_cycles(G, M);
  if (tid == 0) nident = 0;
  __syncthreads();
  int rc = p.rec_count[s];
  int64_t* rpos = p.rec_pos + s * (int64_t)p.rec_cap;
  cd* rval = reinterpret_cast<cd*>(p.rec_val) + s * (int64_t)p.rec_cap;
  for (int i = tid; i < rc; i += nt) hash_insert(M.hash, G.hmask, rpos[i]);
  const double eps0 = p.eps_zero[s], epsr = p.eps_ratio[s];
  const double cfac = (double)(-n) / 6.283185307179586;  // -n / (2.0 * np.pi)
  // step 1: identify every live node once (parallel); single-tons start the paths
  int mine = 0;
  for (int g = tid; g < N; g += nt) {
    int start = 0;
    const int8_t s0 = M.st[g];
    if (s0 != AFFT_RESOLVED && s0 != AFFT_ZERO_TON) {
      const int c = M.cyc[g];
      M.st[g] = classify_exact_dev(M.res[3 * g], M.res[3 * g + 1], M.res[3 * g + 2],
                                   g - G.base[c], G.b[c], n, eps0, epsr, cfac, &M.f0[g],
                                   &M.val[g]);
      ++mine;
      start = M.st[g] == AFFT_SINGLE_TON;
    }
    M.flag[g] = start;
  }
  if (mine) atomicAdd(&nident, mine);
  __syncthreads();
  const int q0 = block_exclusive_scan(M.flag, N, warp_tmp, &carry);
  // the queue lives in found_res (N * ncycles entries: a node re-enters only after it
  // was popped, so at most N entries are ever live; indices wrap)
  int* Q = M.found_res;
  const int qcap = N * F;
  for (int g = tid; g < N; g += nt) {
    const int start = (g + 1 < N ? M.flag[g + 1] : q0) - M.flag[g];
    if (start) {
      Q[M.flag[g]] = g;
      M.hv[g] = 1;
    }
  }
  if (tid == 0) nq0 = q0;
  __syncthreads();
  // steps 2..p: the walk (one thread: the method is a sequential path extension)
  if (tid == 0) {
    int head = 0, tail = nq0, gen_end = nq0, gens = nq0 ? 1 : 0, extra = 0;
    while (head != tail) {
      if (head == gen_end) {  // the previous generation is exhausted
        gen_end = tail;
        ++gens;
      }
      const int g = Q[head];
      head = head + 1 == qcap ? 0 : head + 1;
      M.hv[g] = 0;
      if (M.st[g] != AFFT_SINGLE_TON) continue;
      const int64_t f = M.f0[g];
      if (hash_contains(M.hash, G.hmask, f)) continue;  // peeling.py:296-299
      const cd v = M.res[3 * g];  // a single-ton's value is r0 of its residual
      hash_insert(M.hash, G.hmask, f);
      rpos[rc] = f;
      rval[rc] = v;
      ++rc;
      M.st[g] = AFFT_RESOLVED;
      const cd v1 = cmul(v, unit_root(mulmod(G.tau[1], f, n), n));
      const cd v2 = cmul(v, unit_root(mulmod(G.tau[2], f, n), n));
      for (int c = 0; c < F; ++c) {  // the left node's d right neighbours
        const int g2 = G.base[c] + (int)(f % G.b[c]);
        M.res[3 * g2] = csub(M.res[3 * g2], v);
        M.res[3 * g2 + 1] = csub(M.res[3 * g2 + 1], v1);
        M.res[3 * g2 + 2] = csub(M.res[3 * g2 + 2], v2);
        const int8_t s2 = M.st[g2];
        if (g2 == g || s2 == AFFT_RESOLVED || s2 == AFFT_ZERO_TON) continue;
        const int c2 = M.cyc[g2];
        M.st[g2] = classify_exact_dev(M.res[3 * g2], M.res[3 * g2 + 1], M.res[3 * g2 + 2],
                                      g2 - G.base[c2], G.b[c2], n, eps0, epsr, cfac,
                                      &M.f0[g2], &M.val[g2]);
        ++extra;
        if (M.st[g2] == AFFT_SINGLE_TON && !M.hv[g2]) {
          Q[tail] = g2;
          tail = tail + 1 == qcap ? 0 : tail + 1;
          M.hv[g2] = 1;
        }
      }
    }
    nident += extra;
    if (p.rounds) p.rounds[s] = gens;
    p.rec_count[s] = rc;
    if (ident) ident[s] = nident;
  }
  __syncthreads();
  const int unres = count_multitons(G, M, &red);
  if (tid == 0 && p.unresolved) p.unresolved[s] = unres;
  if (p.writeback) {
    cd* gw = reinterpret_cast<cd*>(p.residual) + s * (int64_t)N * 3;
    for (int e = tid; e < N * 3; e += nt) gw[e] = M.res[e];
    for (int g = tid; g < N; g += nt) {
      p.state[s * N + g] = M.st[g];
      if (p.node_f0) p.node_f0[s * N + g] = M.f0[g];
      if (p.node_val) reinterpret_cast<cd*>(p.node_val)[s * N + g] = M.val[g];
    }
  }
}

// ------------------------------------------------------------------ fused FFAST

struct FusedParams {
  PeelGraph G;
  DftPlan plan[AFFT_MAX_CYCLES];
  const void* x;
  int dtype;
  int64_t ld;
  int k;
  int max_rounds;
  size_t dft_off;  // smem offset of the DFT scratch (aliases the found/hash region)
  int64_t* out_pos;
  double* out_val;
  int32_t* out_count;
  int64_t* all_pos;  // may be null
  double* all_val;
  int32_t* all_count;
  int32_t* rounds;
  int32_t* unresolved;
  double* eps_out;       // may be null
  const double* eps_in;  // may be null: precomputed thresholds (small batches)
  int order_mode;        // fused kernel: 0 stream first, 1 alternate by CTA, 2 DFTs first
  const unsigned* ready; // split-role kernel: ready[s] != 0 once eps_in[s] is published
  int rec_in_smem;       // 1: recovered list in shared memory (no all_pos output)
};

#ifndef AFFT_FUSED_THREADS
#define AFFT_FUSED_THREADS 256
#define AFFT_FUSED_MIN_BLOCKS 3
#endif
constexpr int kFusedThreads = AFFT_FUSED_THREADS;
constexpr int kStreamUnroll = 8;

// 16-byte streaming loads that do not allocate in L1: the CTA's own shared memory
// leaves little L1 next to it, and nothing in the stream is re-read.
__device__ __forceinline__ float4 ld_na(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_na(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Per-thread partial of sum |x|^2 over one signal: 16-byte streaming loads,
// kStreamUnroll in flight per thread, float64 accumulation.
__device__ __forceinline__ double stream_sumsq(const char* row, int dtype, int64_t n) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double a0 = 0.0, a1 = 0.0;
  if (dtype == AFFT_C64) {
    const float2* xs = reinterpret_cast<const float2*>(row);
    int64_t e = 0;
    if (reinterpret_cast<uintptr_t>(xs) & 15) {
      if (tid == 0) {
        const float2 v = __ldg(xs);
        a0 += (double)v.x * v.x + (double)v.y * v.y;
      }
      e = 1;
    }
    const int64_t nvec = (n - e) / 2;
    const float4* xv = reinterpret_cast<const float4*>(xs + e);
    int64_t i = tid;
    for (; i + (kStreamUnroll - 1) * nt < nvec; i += kStreamUnroll * nt) {
      float4 v[kStreamUnroll];
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u) v[u] = ld_na(xv + i + u * nt);
#pragma unroll
      for (int u = 0; u < kStreamUnroll; u += 2) {
        a0 += (double)v[u].x * v[u].x + (double)v[u].y * v[u].y + (double)v[u].z * v[u].z +
              (double)v[u].w * v[u].w;
        a1 += (double)v[u + 1].x * v[u + 1].x + (double)v[u + 1].y * v[u + 1].y +
              (double)v[u + 1].z * v[u + 1].z + (double)v[u + 1].w * v[u + 1].w;
      }
    }
    for (; i < nvec; i += nt) {
      const float4 v = ld_na(xv + i);
      a0 += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    const int64_t tail = e + 2 * nvec;
    if (tail < n && tid == 0) {
      const float2 v = __ldg(xs + tail);
      a1 += (double)v.x * v.x + (double)v.y * v.y;
    }
  } else {
    const double2* xv = reinterpret_cast<const double2*>(row);
    int64_t i = tid;
    for (; i + (kStreamUnroll - 1) * nt < n; i += kStreamUnroll * nt) {
      double2 v[kStreamUnroll];
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u) v[u] = ld_na(xv + i + u * nt);
#pragma unroll
      for (int u = 0; u < kStreamUnroll; u += 2) {
        a0 += v[u].x * v[u].x + v[u].y * v[u].y;
        a1 += v[u + 1].x * v[u + 1].x + v[u + 1].y * v[u + 1].y;
      }
    }
    for (; i < n; i += nt) {
      const double2 v = ld_na(xv + i);
      a0 += v.x * v.x + v.y * v.y;
    }
  }
  return a0 + a1;
}

template <bool kStream>
__device__ __forceinline__ void ffast_one_signal(const FusedParams& p, int64_t s,
                                                 unsigned char* smem_raw, int* warp_tmp,
                                                 int* carry_p, int* red_p, double* wsum) {
  int& carry = *carry_p;
  int& red = *red_p;
  const int tid = threadIdx.x, nt = blockDim.x;
  const PeelGraph& G = p.G;
  const int N = G.nodes;
  const int64_t n = G.n;
  const PeelLayout L = peel_layout(N, G.ncycles, G.hmask + 1, p.rec_in_smem != 0, false);
  const PeelMem M = peel_carve(smem_raw, L);
  int64_t* rec_f = p.rec_in_smem ? M.rec_f : p.all_pos + s * N;
  cd* rec_v = p.rec_in_smem ? M.rec_v : reinterpret_cast<cd*>(p.all_val) + s * N;
  const char* row = reinterpret_cast<const char*>(p.x) + s * p.ld * (p.dtype == AFFT_C64 ? 8 : 16);

  // 1. exact_thresholds: eps = 1e-6 * ||x|| / sqrt(n), fixed-order block reduction
  //    (skipped when a multi-CTA pre-pass already produced eps for a small batch)
  //    By default (order_mode 2) the stream runs after the gather + DFTs and before
  //    the peeling, splitting the latency-bound decode around it: CTAs of one wave
  //    otherwise stream together and then all decode at the same moment, leaving HBM
  //    idle.  Measured at config 5 (tools/fused_order.py, 8192 signals, 15 reps x 5):
  //    stream first 20.47 ms, alternating by CTA 20.48 ms, DFTs first 20.26 ms.
  const bool do_stream = kStream && !p.eps_in;
  const bool stream_first =
      p.order_mode == 0 || (p.order_mode == 1 && (blockIdx.x & 1) == 0);
  double acc = (do_stream && stream_first) ? stream_sumsq(row, p.dtype, n) : 0.0;
  // 2. build_graph: gather + DFT of every cycle at shifts (0, 1, 2), node layout
  cd* tw = reinterpret_cast<cd*>(smem_raw + p.dft_off);
  for (int c = 0; c < G.ncycles; ++c) {
    const int64_t b = G.b[c];
    cd* bufA = tw + b;
    cd* bufB = bufA + 3 * b;
    const cd* spec = gather_dft_block(row, p.dtype, n, b, p.plan[c], G.tau, 3, tw, bufA, bufB);
    const double inv_b = 1.0 / (double)b;
    for (int e = tid; e < 3 * (int)b; e += nt) {
      const int t = e / (int)b;
      const int i = e - t * (int)b;
      M.res[3 * (G.base[c] + i) + t] = cscale(spec[e], inv_b);
    }
    __syncthreads();
  }
  if (do_stream && !stream_first) acc = stream_sumsq(row, p.dtype, n);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) wsum[tid >> 5] = acc;
  __syncthreads();
  if (p.ready) {  // split-role kernel: wait for the streaming CTA that owns signal s
    if (tid == 0)
      while (ld_acquire_u32(p.ready + s) == 0u) __nanosleep(128);
    __syncthreads();
  }
  double t = 0.0;
  for (int w = 0; w < kFusedThreads / 32; ++w) t += wsum[w];
  const double eps =
      (!kStream || p.eps_in) ? __ldcg(p.eps_in + s) : (1e-6 * sqrt(t)) / sqrt((double)n);
  // 3. graph state
  for (int g = tid; g < N; g += nt) {
    M.st[g] = AFFT_UNKNOWN;
    M.dirty[g] = 1;
    M.hv[g] = 0;
    M.f0[g] = -1;
  }
  for (int h = tid; h <= G.hmask; h += nt) M.hash[h] = kEmpty;
  peel_fill_cycles(G, M);
  __syncthreads();
  // 4. peel
  int rc = 0;
  const int rounds = peel_rounds(G, M, eps, eps, p.max_rounds, rec_f, rec_v, rc, warp_tmp, &carry);
  const int unres = count_multitons(G, M, &red);
  // 5. truncate to k by (-|v|, f) in the (now free) found-list memory.  Up to 1024
  //    entries (every config-5-sized graph) each thread ranks its entries against all
  //    of them — one barrier; larger lists take the bitonic sort (log^2 barriers).
  cd* ov = reinterpret_cast<cd*>(p.out_val) + s * p.k;
  const int kept = rc < p.k ? rc : p.k;
  if (rc <= 1024) {
    double* key = reinterpret_cast<double*>(M.found_f);
    int64_t* kpos = reinterpret_cast<int64_t*>(key + rc);
    for (int i = tid; i < rc; i += nt) {
      key[i] = cabs_(rec_v[i]);
      kpos[i] = rec_f[i];
    }
    __syncthreads();
    for (int i = tid; i < rc; i += nt) {
      const int r = trunc_rank(key, kpos, rc, i);  // distinct positions: a permutation
      if (r < kept) {
        p.out_pos[s * p.k + r] = kpos[i];
        ov[r] = rec_v[i];
      }
    }
  } else {
    int pow2 = 1;
    while (pow2 < rc) pow2 <<= 1;
    double* key = reinterpret_cast<double*>(M.found_f);
    int64_t* kpos = reinterpret_cast<int64_t*>(key + pow2);
    int32_t* kidx = reinterpret_cast<int32_t*>(kpos + pow2);
    for (int i = tid; i < rc; i += nt) {
      key[i] = cabs_(rec_v[i]);
      kpos[i] = rec_f[i];
      kidx[i] = i;
    }
    bitonic_trunc_sort(key, kpos, kidx, rc, pow2);
    for (int r = tid; r < kept; r += nt) {
      p.out_pos[s * p.k + r] = kpos[r];
      ov[r] = rec_v[kidx[r]];
    }
  }
  if (p.all_pos && p.rec_in_smem) {
    cd* av = reinterpret_cast<cd*>(p.all_val) + s * N;
    for (int i = tid; i < rc; i += nt) {
      p.all_pos[s * N + i] = rec_f[i];
      av[i] = rec_v[i];
    }
  }
  if (tid == 0) {
    p.out_count[s] = rc < p.k ? rc : p.k;
    if (p.all_count) p.all_count[s] = rc;
    if (p.rounds) p.rounds[s] = rounds;
    if (p.unresolved) p.unresolved[s] = unres;
    if (p.eps_out) p.eps_out[s] = eps;
  }
}

// One signal per CTA iteration; a grid smaller than the batch makes the CTAs
// persistent (grid-stride over signals), which is how the pipelined path caps
// the decode's SM footprint next to the concurrent norm stream.
__global__ void __launch_bounds__(kFusedThreads, AFFT_FUSED_MIN_BLOCKS) ffast_fused_kernel(
    const __grid_constant__ FusedParams p, int64_t batch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry, red;
  __shared__ double wsum[kFusedThreads / 32];
  for (int64_t s = blockIdx.x; s < batch; s += gridDim.x) {
    ffast_one_signal<true>(p, s, smem_raw, warp_tmp, &carry, &red, wsum);
    __syncthreads();
  }
}

// Split roles (mode 3, selectable; slower at config 5): a persistent, co-resident grid
// whose first n_stream CTAs (two per SM) only stream |x|^2 and publish each
// signal's eps with a release flag, while the remaining CTAs (one per SM) decode
// signals in order — gather + DFTs first, then an acquire wait on the flag, then
// peeling.  The fused kernel's CTAs alternate stream and decode phases and tend
// to fall into step, leaving HBM idle while whole waves decode; here HBM is fed
// by the streaming CTAs continuously and the decode runs beside them.
__global__ void __launch_bounds__(kFusedThreads, 3) ffast_split_kernel(
    const __grid_constant__ FusedParams p, int64_t batch, int n_stream, double* eps_buf,
    unsigned* ready) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry, red;
  __shared__ double wsum[kFusedThreads / 32];
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < n_stream) {
    const int64_t n = p.G.n;
    const int64_t esz = p.dtype == AFFT_C64 ? 8 : 16;
    for (int64_t s = blockIdx.x; s < batch; s += n_stream) {
      const char* row = reinterpret_cast<const char*>(p.x) + s * p.ld * esz;
      double acc = stream_sumsq(row, p.dtype, n);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((tid & 31) == 0) wsum[tid >> 5] = acc;
      __syncthreads();
      if (tid == 0) {  // same fixed-order reduction as the fused kernel
        double t = 0.0;
        for (int w = 0; w < kFusedThreads / 32; ++w) t += wsum[w];
        eps_buf[s] = (1e-6 * sqrt(t)) / sqrt((double)n);
        if (p.eps_out) p.eps_out[s] = eps_buf[s];
        st_release_u32(ready + s, 1u);
      }
      __syncthreads();
    }
    return;
  }
  const int nd = gridDim.x - n_stream;
  for (int64_t s = (int)blockIdx.x - n_stream; s < batch; s += nd) {
    ffast_one_signal<false>(p, s, smem_raw, warp_tmp, &carry, &red, wsum);
    __syncthreads();
  }
}

// Split streams (mode 4): `parts` CTAs per signal each stream 1/parts of its |x|^2
// and leave a partial; the CTA that arrives last (atomic ticket) sums the partials
// in part order — deterministic — and decodes the signal.  Finer CTAs balance the
// tail of small batches and scatter the decode phases across the grid.
__global__ void __launch_bounds__(kFusedThreads, AFFT_FUSED_MIN_BLOCKS) ffast_parts_kernel(
    const __grid_constant__ FusedParams p, int64_t batch, int parts, double* part_sums,
    unsigned* tickets, double* eps_buf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry, red, last;
  __shared__ double wsum[kFusedThreads / 32];
  const int tid = threadIdx.x;
  const int64_t s = blockIdx.x / parts;
  const int part = (int)(blockIdx.x - s * parts);
  if (s >= batch) return;
  const int64_t n = p.G.n;
  const int64_t esz = p.dtype == AFFT_C64 ? 8 : 16;
  const int64_t chunk = (n + parts - 1) / parts;
  const int64_t lo = min(n, part * chunk), hi = min(n, lo + chunk);
  const char* row = reinterpret_cast<const char*>(p.x) + s * p.ld * esz;
  double acc = hi > lo ? stream_sumsq(row + lo * esz, p.dtype, hi - lo) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) wsum[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kFusedThreads / 32; ++w) t += wsum[w];
    part_sums[s * parts + part] = t;
    __threadfence();
    last = atomicAdd(tickets + s, 1u) == (unsigned)(parts - 1);
  }
  __syncthreads();
  if (!last) return;
  if (tid == 0) {
    __threadfence();
    double t = 0.0;
    for (int q = 0; q < parts; ++q) t += __ldcg(part_sums + s * parts + q);
    eps_buf[s] = (1e-6 * sqrt(t)) / sqrt((double)n);
    __threadfence_block();
  }
  __syncthreads();
  ffast_one_signal<false>(p, s, smem_raw, warp_tmp, &carry, &red, wsum);
}

// Decode only (eps precomputed by the multi-CTA norm pass): the fused body with the
// stream compiled out, so fewer registers are live across the decode.
__global__ void __launch_bounds__(kFusedThreads, AFFT_FUSED_MIN_BLOCKS) ffast_decode_kernel(
    const __grid_constant__ FusedParams p, int64_t batch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tmp[32];
  __shared__ int carry, red;
  __shared__ double wsum[kFusedThreads / 32];
  for (int64_t s = blockIdx.x; s < batch; s += gridDim.x) {
    ffast_one_signal<false>(p, s, smem_raw, warp_tmp, &carry, &red, wsum);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ per-node kernels

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
                                int32_t* __restrict__ out_count, double* gscratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t s = blockIdx.x;
  const int m = count[s];
  if (!gscratch) {  // bitonic sort in shared memory
    int pow2 = 1;
    while (pow2 < m) pow2 <<= 1;
    double* key = reinterpret_cast<double*>(smem_raw);
    int64_t* kpos = reinterpret_cast<int64_t*>(key + pow2);
    int32_t* kidx = reinterpret_cast<int32_t*>(kpos + pow2);
    const int64_t* ps = pos + s * cap;
    const cd* vs = reinterpret_cast<const cd*>(val) + s * cap;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      key[i] = cabs_(vs[i]);
      kpos[i] = ps[i];
      kidx[i] = i;
    }
    bitonic_trunc_sort(key, kpos, kidx, m, pow2);
    cd* ov = reinterpret_cast<cd*>(out_val) + s * k;
    const int kept = m < k ? m : k;
    for (int r = threadIdx.x; r < kept; r += blockDim.x) {
      out_pos[s * k + r] = kpos[r];
      ov[r] = vs[kidx[r]];
    }
    if (threadIdx.x == 0) out_count[s] = kept;
    return;
  }
  double* mag = gscratch + s * (int64_t)cap * 2;
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
    const int rank = trunc_rank(mag, fs, m, i);
    if (rank < k) {
      out_pos[s * k + rank] = fs[i];
      ov[rank] = vs[i];
    }
  }
  if (threadIdx.x == 0) out_count[s] = m < k ? m : k;
}

// ------------------------------------------------------------------ host setup

static int setup_graph(PeelGraph* G, int64_t n, const int64_t* factors, int ncycles,
                       int rec_cap) {
  memset(G, 0, sizeof(*G));
  if (ncycles < 1 || ncycles > AFFT_MAX_CYCLES || !factors) {
    set_error("number of cycles %d outside 1..%d", ncycles, AFFT_MAX_CYCLES);
    return AFFT_EUNSUPPORTED;
  }
  if (n < 1 || n > 3000000000LL) {  // positions fit the 32-bit hash keys
    set_error("signal size %lld outside the supported 1..3e9", (long long)n);
    return AFFT_EUNSUPPORTED;
  }
  G->n = n;
  G->ncycles = ncycles;
  int64_t total = 0;
  for (int c = 0; c < ncycles; ++c) {
    if (factors[c] < 1 || n % factors[c]) {
      set_error("bucket count %lld does not divide signal size %lld", (long long)factors[c],
                (long long)n);
      return AFFT_EINVAL;
    }
    G->b[c] = factors[c];
    G->base[c] = (int32_t)total;
    total += factors[c];
  }
  if (total > (1 << 24)) {
    set_error("graph with %lld nodes is too large", (long long)total);
    return AFFT_EUNSUPPORTED;
  }
  for (int c = ncycles; c <= AFFT_MAX_CYCLES; ++c) G->base[c] = INT32_MAX;
  G->base[ncycles] = (int32_t)total;
  G->nodes = (int)total;
  G->tau[0] = 0;
  G->tau[1] = 1 % n;
  G->tau[2] = 2 % n;
  int hcap = 16;
  while (hcap < 2 * rec_cap) hcap <<= 1;
  G->hmask = hcap - 1;
  return AFFT_OK;
}

constexpr size_t kSmemLimit = 200 * 1024;

static int launch_peel(PeelParams& p, int64_t batch, void* scratch, cudaStream_t stream) {
  const size_t bytes = peel_layout(p.G.nodes, p.G.ncycles, p.G.hmask + 1, false).total;
  size_t dyn = 0;
  if (bytes <= kSmemLimit) {
    p.gscratch = nullptr;
    dyn = bytes;
    cudaError_t e = ensure_smem((const void*)peel_exact_kernel, (int)dyn);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(peel_exact)");
  } else {
    if (!scratch) {
      set_error("peeling graph does not fit in shared memory and no scratch was given");
      return AFFT_ENOMEM;
    }
    p.gscratch = reinterpret_cast<char*>(scratch);
    p.scratch_bytes = bytes;
  }
  peel_exact_kernel<<<(unsigned)batch, 256, dyn, stream>>>(p);
  AFFT_CHECK_LAUNCH("peel_exact_kernel");
  return AFFT_OK;
}

static int launch_peel_tree(PeelParams& p, int64_t batch, void* scratch, int32_t* ident,
                            cudaStream_t stream) {
  const size_t bytes = peel_layout(p.G.nodes, p.G.ncycles, p.G.hmask + 1, false).total;
  size_t dyn = 0;
  if (bytes <= kSmemLimit) {
    p.gscratch = nullptr;
    dyn = bytes;
    cudaError_t e = ensure_smem((const void*)peel_tree_kernel, (int)dyn);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(peel_tree)");
  } else {
    if (!scratch) {
      set_error("peeling graph does not fit in shared memory and no scratch was given");
      return AFFT_ENOMEM;
    }
    p.gscratch = reinterpret_cast<char*>(scratch);
    p.scratch_bytes = bytes;
  }
  peel_tree_kernel<<<(unsigned)batch, 256, dyn, stream>>>(p, ident);
  AFFT_CHECK_LAUNCH("peel_tree_kernel");
  return AFFT_OK;
}

static int launch_truncate(const int64_t* pos, const double* val, const int32_t* count, int cap,
                           int64_t batch, int k, int64_t* out_pos, double* out_val,
                           int32_t* out_count, cudaStream_t stream) {
  int pow2 = 1;
  while (pow2 < std::max(cap, 1)) pow2 <<= 1;
  size_t smem = (size_t)pow2 * 20;
  double* scratch = nullptr;
  if (smem > kSmemLimit) {  // large graphs: rank from global memory
    cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&scratch),
                                    (size_t)batch * cap * 16, stream);
    if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(truncate scratch)");
    smem = 0;
  } else {
    cudaError_t e = ensure_smem((const void*)truncate_kernel, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(truncate)");
  }
  truncate_kernel<<<(unsigned)batch, 1024, smem, stream>>>(pos, val, count, cap, k, out_pos,
                                                            out_val, out_count, scratch);
  if (scratch) scratch_free(scratch, stream);
  AFFT_CHECK_LAUNCH("truncate_kernel");
  return AFFT_OK;
}

// Fused-kernel shared memory: peel layout (with recovered list) + DFT scratch
// (tw + 2 x 3 shifts x b) aliased onto found/hash when it fits there.
static bool fused_smem(const PeelGraph& G, bool rec_in_smem, size_t* total, size_t* dft_off) {
  const PeelLayout L = peel_layout(G.nodes, G.ncycles, G.hmask + 1, rec_in_smem, false);
  int64_t bmax = 0;
  for (int c = 0; c < G.ncycles; ++c) bmax = std::max(bmax, G.b[c]);
  if (bmax > AFFT_MAX_SMEM_DFT) return false;
  const size_t dft = (size_t)7 * bmax * 16;
  if (dft <= L.flag - L.found_f) {
    *dft_off = L.found_f;
    *total = L.total;
  } else {
    *dft_off = L.total;
    *total = L.total + dft;
  }
  return *total <= kSmemLimit;
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static int num_sms() {  // of the current device (the attribute query is a cheap lookup)
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  return v > 0 ? v : 148;
}

// Auxiliary stream and events for the pipelined FFAST path, one set per device.
struct AuxStreams {
  std::mutex enqueue;  // held for a whole fork/chunk/join sequence (shared events)
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t chunk[64] = {};
};

static int aux_streams(AuxStreams** out) {
  static std::mutex mu;
  static AuxStreams per_dev[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 64) return cuda_status(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  AuxStreams& a = per_dev[dev];
  if (!a.aux) {
    e = cudaStreamCreateWithFlags(&a.aux, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming);
    for (int i = 0; i < 64 && e == cudaSuccess; ++i)
      e = cudaEventCreateWithFlags(&a.chunk[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e, "aux stream setup");
  }
  *out = &a;
  return AFFT_OK;
}

// Split-stream mode (4) runs up to kMaxParts CTAs per signal; its partial sums and
// per-signal tickets share the pre-pass partials block, so that block holds
// batch * max(nparts, kMaxParts) doubles plus batch tickets.
constexpr int kMaxParts = 16;

static size_t fused_partials_bytes(int64_t batch, int nparts) {
  return al256((size_t)batch * std::max(nparts, kMaxParts) * 8 + (size_t)batch * 4);
}

struct FfastWs {
  size_t partials, eps, nodes, state, rec_pos, rec_val, rec_count, rounds, unres, scratch, total;
};

// Workspace of the unfused (large-graph) sequence; the fused path needs none.
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
  PeelParams p;
  memset(&p, 0, sizeof(p));
  int rc = setup_graph(&p.G, n, factors, ncycles, rec_cap);
  if (rc) return rc;
  if (rec_cap < p.G.nodes) {
    set_error("rec_cap %d must cover the node count %d plus prior entries", rec_cap, p.G.nodes);
    return AFFT_EINVAL;
  }
  p.residual = residual;
  p.state = state;
  p.node_f0 = node_f0;
  p.node_val = node_val;
  p.eps_zero = eps_zero;
  p.eps_ratio = eps_ratio;
  p.max_rounds = max_rounds;
  p.rec_pos = rec_pos;
  p.rec_val = rec_val;
  p.rec_cap = rec_cap;
  p.rec_count = rec_count;
  p.rounds = rounds;
  p.unresolved = unresolved;
  p.writeback = 1;
  cudaStream_t st = (cudaStream_t)stream;
  void* scratch = nullptr;
  const size_t bytes = peel_layout(p.G.nodes, ncycles, p.G.hmask + 1, false).total;
  if (bytes > kSmemLimit) {
    cudaError_t e = scratch_alloc(&scratch, (size_t)batch * bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(peel scratch)");
  }
  rc = launch_peel(p, batch, scratch, st);
  if (scratch) scratch_free(scratch, st);
  return rc;
}

extern "C" int afft_peel_tree_exact(int64_t n, int64_t batch, const int64_t* factors,
                                    int32_t ncycles, double* residual, int8_t* state,
                                    int64_t* node_f0, double* node_val, const double* eps_zero,
                                    const double* eps_ratio, int64_t* rec_pos, double* rec_val,
                                    int32_t rec_cap, int32_t* rec_count, int32_t* rounds,
                                    int32_t* unresolved, int32_t* identifications,
                                    void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!residual || !state || !eps_zero || !eps_ratio || !rec_pos || !rec_val || !rec_count ||
      batch < 0) {
    set_error("afft_peel_tree_exact: bad arguments");
    return AFFT_EINVAL;
  }
  PeelParams p;
  memset(&p, 0, sizeof(p));
  int rc = setup_graph(&p.G, n, factors, ncycles, rec_cap);
  if (rc) return rc;
  if (rec_cap < p.G.nodes) {
    set_error("rec_cap %d must cover the node count %d plus prior entries", rec_cap, p.G.nodes);
    return AFFT_EINVAL;
  }
  p.residual = residual;
  p.state = state;
  p.node_f0 = node_f0;
  p.node_val = node_val;
  p.eps_zero = eps_zero;
  p.eps_ratio = eps_ratio;
  p.rec_pos = rec_pos;
  p.rec_val = rec_val;
  p.rec_cap = rec_cap;
  p.rec_count = rec_count;
  p.rounds = rounds;
  p.unresolved = unresolved;
  p.writeback = 1;
  cudaStream_t st = (cudaStream_t)stream;
  void* scratch = nullptr;
  const size_t bytes = peel_layout(p.G.nodes, ncycles, p.G.hmask + 1, false).total;
  if (bytes > kSmemLimit) {
    cudaError_t e = scratch_alloc(&scratch, (size_t)batch * bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(peel tree scratch)");
  }
  rc = launch_peel_tree(p, batch, scratch, identifications, st);
  if (scratch) scratch_free(scratch, st);
  return rc;
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
  int64_t nodes = 0;
  for (int c = 0; c < ncycles && factors; ++c) nodes += factors[c];
  PeelGraph G;
  if (setup_graph(&G, n, factors, ncycles, (int)std::max<int64_t>(nodes, 1))) return 0;
  size_t total = 0, off = 0;
  if (fused_smem(G, true, &total, &off))  // fused path: partials + eps of the norm pre-pass
    return fused_partials_bytes(batch, afft_sumsq_parts(n, dtype)) + al256((size_t)batch * 8);
  const size_t bytes = peel_layout(G.nodes, ncycles, G.hmask + 1, false).total;
  return ffast_ws(n, dtype, batch, nodes, bytes > kSmemLimit ? bytes : 0).total;
}

extern "C" int afft_ffast(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                          const int64_t* factors, int32_t ncycles, int32_t k,
                          int32_t max_rounds, int64_t* out_pos, double* out_val,
                          int32_t* out_count, int64_t* all_pos, double* all_val,
                          int32_t* all_count, int32_t* rounds, int32_t* unresolved,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!x || (k > 0 && (!out_pos || !out_val)) || !out_count || k < 0 || batch < 0 || ld < n ||
      (dtype != AFFT_C64 && dtype != AFFT_C128)) {
    set_error("afft_ffast: bad arguments");
    return AFFT_EINVAL;
  }
  int64_t nodes = 0;
  for (int c = 0; c < ncycles && factors; ++c) nodes += factors[c];
  cudaStream_t st = (cudaStream_t)stream;
  const int mr = max_rounds > 0 ? max_rounds : k + 4;
  FusedParams fp;
  memset(&fp, 0, sizeof(fp));
  int rc = setup_graph(&fp.G, n, factors, ncycles, (int)std::max<int64_t>(nodes, 1));
  if (rc) return rc;
  size_t smem = 0;
  fp.rec_in_smem = all_pos == nullptr || all_val == nullptr;
  if (fused_smem(fp.G, fp.rec_in_smem != 0, &smem, &fp.dft_off)) {
    for (int c = 0; c < ncycles; ++c) {
      if (!make_dft_plan(fp.G.b[c], &fp.plan[c])) {
        set_error("cannot plan a DFT of size %lld", (long long)fp.G.b[c]);
        return AFFT_EUNSUPPORTED;
      }
    }
    fp.x = x;
    fp.dtype = dtype;
    fp.ld = ld;
    fp.k = k;
    fp.max_rounds = mr;
    fp.out_pos = out_pos;
    fp.out_val = out_val;
    fp.out_count = out_count;
    fp.all_pos = all_pos;
    fp.all_val = all_val;
    fp.all_count = all_count;
    fp.rounds = rounds;
    fp.unresolved = unresolved;
    {
      const char* om = getenv("AFFT_FUSED_ORDER");
      fp.order_mode = om && om[0] >= '0' && om[0] <= '2' ? om[0] - '0' : 2;
    }
    // Small batches cannot keep HBM busy with one streaming CTA per signal: run the
    // |x|^2 pass as a multi-CTA partial sum first and feed eps to the fused decode.
    // Large batches (mode 2, the default there) pipeline it: the norm stream of
    // chunk c+1 runs on the caller's stream while chunk c decodes on an auxiliary
    // stream, so HBM never waits for the latency-bound decode.
    const int nparts = afft_sumsq_parts(n, dtype);
    const char* env = getenv("AFFT_FFAST_MODE");  // 0 fused, 1 pre-pass, 2 pipelined, 3 split
    // Measured on B200 (tools/ffast_modes.py, config 5, 8192 signals): fused 20.44 ms,
    // pipelined 20.96 ms, split roles 22.5 ms (one decoding CTA per SM cannot keep
    // up: ~0.2 ms per signal), pre-pass + decode 22.25 ms, stream alone 18.65 ms.
    // Small batches (< 2 waves) cannot keep HBM busy with one streaming CTA per signal.
    const int sms = num_sms();
    // Below ~13 waves of fused CTAs (3 per SM) the last partial waves stream with too
    // few CTAs; split streams (mode 4: several CTAs per signal, the last one decodes)
    // keep ~20 CTAs per SM in flight instead (tools/parts_sweep.py, config 5:
    // 1024 signals 2.67 vs 3.05 ms fused / 2.95 ms pre-pass; 4096 10.12 vs 10.35;
    // 512 1.40 vs 1.56; from ~6000 signals the single fused launch wins).
    int mode = batch < 40 * sms ? 4 : 0;
    if (env && env[0] >= '0' && env[0] <= '4') mode = env[0] - '0';
    if (nparts < 2) mode = 0;
    if (mode == 3) {
      // the split roles spin-wait across CTAs: every CTA must be resident (cooperative
      // launch below) with room for two streaming CTAs and one decoding CTA per SM
      int per_sm = 0;
      cudaError_t e = ensure_smem((const void*)ffast_split_kernel, (int)smem);
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ffast_split_kernel,
                                                          kFusedThreads, smem);
      if (e != cudaSuccess || per_sm < 3) {
        cudaGetLastError();
        mode = 0;
      }
    }
    double* partials = nullptr;
    double* epsbuf = nullptr;
    if (mode) {
      const size_t pbytes = fused_partials_bytes(batch, nparts);
      const size_t need = pbytes + al256((size_t)batch * 8);
      if (!workspace || workspace_bytes < need) {
        set_error("afft_ffast: workspace of %zu bytes needed, %zu given", need, workspace_bytes);
        return AFFT_ENOMEM;
      }
      partials = reinterpret_cast<double*>(workspace);
      epsbuf = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + pbytes);
    }
    {
      cudaError_t e = ensure_smem((const void*)ffast_fused_kernel, (int)smem);
      if (e == cudaSuccess)
        e = ensure_smem((const void*)ffast_decode_kernel, (int)smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(ffast_fused)");
    }
    if (mode == 2) {
      AuxStreams* A = nullptr;
      if ((rc = aux_streams(&A))) return rc;
      // the aux stream and its events are shared by every caller on this device: no
      // other thread may re-record an event between our record and the matching wait
      std::lock_guard<std::mutex> lock(A->enqueue);
      const int64_t esz = dtype == AFFT_C64 ? 8 : 16;
      int64_t nchunks = std::min<int64_t>(32, std::max<int64_t>(2, batch / 256));
      const int64_t csz = (batch + nchunks - 1) / nchunks;
      nchunks = (batch + csz - 1) / csz;
      cudaEventRecord(A->fork, st);
      cudaStreamWaitEvent(A->aux, A->fork, 0);
      for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t s0 = c * csz, cnt = std::min(csz, batch - s0);
        const char* xc = reinterpret_cast<const char*>(x) + s0 * ld * esz;
        if ((rc = afft_sumsq(xc, dtype, n, cnt, ld, partials + s0 * nparts, st))) return rc;
        if ((rc = afft_exact_thresholds(partials + s0 * nparts, nparts, n, cnt, epsbuf + s0, st)))
          return rc;
        cudaEventRecord(A->chunk[c], st);
        cudaStreamWaitEvent(A->aux, A->chunk[c], 0);
        FusedParams fc = fp;
        fc.x = xc;
        fc.eps_in = epsbuf + s0;
        fc.out_pos = out_pos ? out_pos + s0 * k : nullptr;
        fc.out_val = out_val ? out_val + 2 * s0 * k : nullptr;
        fc.out_count = out_count + s0;
        fc.all_pos = all_pos ? all_pos + s0 * nodes : nullptr;
        fc.all_val = all_val ? all_val + 2 * s0 * nodes : nullptr;
        fc.all_count = all_count ? all_count + s0 : nullptr;
        fc.rounds = rounds ? rounds + s0 : nullptr;
        fc.unresolved = unresolved ? unresolved + s0 : nullptr;
        const char* dg = getenv("AFFT_DECODE_CTAS_PER_SM");
        const int per_sm = dg ? std::max(1, atoi(dg)) : 1;
        const int64_t grid = std::min<int64_t>(cnt, (int64_t)num_sms() * per_sm);
        ffast_decode_kernel<<<(unsigned)grid, kFusedThreads, smem, A->aux>>>(fc, cnt);
        AFFT_CHECK_LAUNCH("ffast_fused_kernel");
      }
      cudaEventRecord(A->join, A->aux);
      cudaStreamWaitEvent(st, A->join, 0);
      return AFFT_OK;
    }
    if (mode == 3) {
      unsigned* ready = reinterpret_cast<unsigned*>(partials);  // batch * 4 <= partials
      cudaError_t e = cudaMemsetAsync(ready, 0, (size_t)batch * 4, st);
      if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(ready flags)");
      fp.eps_in = epsbuf;
      fp.ready = ready;
      int n_stream = 2 * sms;
      unsigned grid = (unsigned)(3 * sms);
      if (batch < n_stream) n_stream = (int)batch;
      void* args[] = {&fp, &batch, &n_stream, &epsbuf, &ready};
      e = cudaLaunchCooperativeKernel((const void*)ffast_split_kernel, grid, kFusedThreads, args,
                                      smem, st);
      if (e != cudaSuccess) return cuda_status(e, "cudaLaunchCooperativeKernel(ffast_split)");
      return AFFT_OK;
    }
    if (mode == 4) {
      const char* pe = getenv("AFFT_FFAST_PARTS");
      const int64_t want = (21LL * sms + batch / 2) / std::max<int64_t>(batch, 1);
      const int parts = pe ? std::max(1, std::min(kMaxParts, atoi(pe)))
                           : (int)std::max<int64_t>(2, std::min<int64_t>(12, want));
      double* part_sums = partials;                               // batch * parts
      unsigned* tickets = reinterpret_cast<unsigned*>(part_sums + batch * parts);  // batch
      cudaError_t e = cudaMemsetAsync(tickets, 0, (size_t)batch * 4, st);
      if (e == cudaSuccess) e = ensure_smem((const void*)ffast_parts_kernel, (int)smem);
      if (e != cudaSuccess) return cuda_status(e, "ffast parts setup");
      fp.eps_in = epsbuf;
      ffast_parts_kernel<<<(unsigned)(batch * parts), kFusedThreads, smem, st>>>(
          fp, batch, parts, part_sums, tickets, epsbuf);
      AFFT_CHECK_LAUNCH("ffast_parts_kernel");
      return AFFT_OK;
    }
    if (mode == 1) {
      if ((rc = afft_sumsq(x, dtype, n, batch, ld, partials, st))) return rc;
      if ((rc = afft_exact_thresholds(partials, nparts, n, batch, epsbuf, st))) return rc;
      fp.eps_in = epsbuf;
    }
    if (fp.eps_in)
      ffast_decode_kernel<<<(unsigned)batch, kFusedThreads, smem, st>>>(fp, batch);
    else
      ffast_fused_kernel<<<(unsigned)batch, kFusedThreads, smem, st>>>(fp, batch);
    AFFT_CHECK_LAUNCH("ffast_fused_kernel");
    return AFFT_OK;
  }

  // Large graphs: the unfused sequence over global-memory scratch.
  const size_t bytes = peel_layout(fp.G.nodes, ncycles, fp.G.hmask + 1, false).total;
  const FfastWs w = ffast_ws(n, dtype, batch, nodes, bytes > kSmemLimit ? bytes : 0);
  if (!workspace || workspace_bytes < w.total) {
    set_error("afft_ffast: workspace of %zu bytes needed, %zu given", w.total, workspace_bytes);
    return AFFT_ENOMEM;
  }
  char* ws = reinterpret_cast<char*>(workspace);
  const int nparts = afft_sumsq_parts(n, dtype);
  double* partials = reinterpret_cast<double*>(ws + w.partials);
  double* eps = reinterpret_cast<double*>(ws + w.eps);
  double* nodebuf = reinterpret_cast<double*>(ws + w.nodes);
  int8_t* state = reinterpret_cast<int8_t*>(ws + w.state);
  int64_t* rpos = all_pos ? all_pos : reinterpret_cast<int64_t*>(ws + w.rec_pos);
  double* rval = all_val ? all_val : reinterpret_cast<double*>(ws + w.rec_val);
  int32_t* rcount = all_count ? all_count : reinterpret_cast<int32_t*>(ws + w.rec_count);
  if ((rc = afft_sumsq(x, dtype, n, batch, ld, partials, st))) return rc;
  if ((rc = afft_exact_thresholds(partials, nparts, n, batch, eps, st))) return rc;
  const int64_t shifts[3] = {0, 1, 2};
  if ((rc = afft_build_graph(x, dtype, n, batch, ld, factors, ncycles, shifts, 3, nodebuf, st)))
    return rc;
  cudaError_t e = cudaMemsetAsync(state, 0, (size_t)batch * nodes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(rcount, 0, (size_t)batch * 4, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(ffast)");
  PeelParams p;
  memset(&p, 0, sizeof(p));
  p.G = fp.G;
  p.residual = nodebuf;
  p.state = state;
  p.eps_zero = eps;
  p.eps_ratio = eps;
  p.max_rounds = mr;
  p.rec_pos = rpos;
  p.rec_val = rval;
  p.rec_cap = (int)nodes;
  p.rec_count = rcount;
  p.rounds = rounds ? rounds : reinterpret_cast<int32_t*>(ws + w.rounds);
  p.unresolved = unresolved ? unresolved : reinterpret_cast<int32_t*>(ws + w.unres);
  if ((rc = launch_peel(p, batch, ws + w.scratch, st))) return rc;
  return launch_truncate(rpos, rval, rcount, (int)nodes, batch, k, out_pos, out_val, out_count,
                         st);
}

extern "C" int afft_ffast_occupancy(int64_t n, const int64_t* factors, int32_t ncycles,
                                    int32_t* blocks_per_sm, int32_t* smem_bytes) {
  PeelGraph G;
  int64_t nodes = 0;
  for (int c = 0; c < ncycles && factors; ++c) nodes += factors[c];
  int rc = setup_graph(&G, n, factors, ncycles, (int)std::max<int64_t>(nodes, 1));
  if (rc) return rc;
  size_t smem = 0, off = 0;
  if (!fused_smem(G, false, &smem, &off)) {
    *blocks_per_sm = 0;
    *smem_bytes = 0;
    return AFFT_OK;
  }
  cudaError_t e = ensure_smem((const void*)ffast_fused_kernel, (int)smem);
  int blocks = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, ffast_fused_kernel, kFusedThreads,
                                                      smem);
  if (e != cudaSuccess) return cuda_status(e, "occupancy query");
  *blocks_per_sm = blocks;
  *smem_bytes = (int32_t)smem;
  return AFFT_OK;
}
