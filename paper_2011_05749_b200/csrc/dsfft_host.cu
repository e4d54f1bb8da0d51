// Native DSFFT layer loop (dsfft.py:244-267 and its helpers 69-241) over the device
// primitives of dsfft.cu / rffast.cu / oneshot.cu.
//
// The tree search is data-dependent host control flow: every layer reads back one
// active count, every classification one small result block.  Run from Python, the
// per-layer interpreter work and the tensor bookkeeping around ~20 library calls
// left the GPU idle for about half of a config-4 decode; here the same sequence of
// launches is issued from C++ with one synchronisation per read-back.  The control
// flow, thresholds and insertion orders follow the reference line by line:
//
//   calibrate   (231-241)  noise_std = sqrt(b * median|v|^2 / ln 2) when absent;
//   initial     (69-79)    full layer at depth ceil(log2 k), active by |v| > thr;
//   expand      (82-115)   children {i, i + 2^(d-1)}: direct alias sums when
//                          2 m_{d-1} <= d, else the full layer;
//   classify    (118-174)  exact: shifts 0,1,2 + classify_exact with the signal's
//                          exact threshold; noisy: the c*m search-plan shifts,
//                          T0/T1 from noise_std (floor 1e-8 sqrt(max energy)) or
//                          the quiet-bucket median, then classify_noisy;
//   loop        (258-264)  expand while m_d < theta k; then (noisy) re-expand while
//                          multitons remain; entries come from the last classify;
//   resolve     (201-228)  leftover multitons through the DT3 detect + solve with
//                          p = max(12, ceil(a_m log10 max(n/b, 10))) random shifts.
//
// Host inputs that must come from numpy's PCG64 (the search-plan anchors and the
// DT3 random shifts for every possible stop depth) are drawn by the Python caller.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <vector>

#include "afft_common.cuh"

namespace afft {

__global__ void dsfft_cand_kernel(const int64_t* __restrict__ act, int64_t m, int64_t half,
                                  int64_t* __restrict__ cand) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) {
    cand[i] = act[i];
    cand[m + i] = act[i] + half;
  }
}

__global__ void dsfft_quiet_kernel(int64_t b, const int64_t* __restrict__ act, int64_t m,
                                   uint8_t* __restrict__ quiet) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b;
       i += (int64_t)gridDim.x * blockDim.x)
    quiet[i] = 1;
}
__global__ void dsfft_unquiet_kernel(const int64_t* __restrict__ act, int64_t m,
                                     uint8_t* __restrict__ quiet) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) quiet[act[i]] = 0;
}

// max of v[0..n) (all >= 0) into *out (zeroed by the caller): fmax per thread and
// warp, then an integer atomicMax on the bit pattern (non-negative doubles order
// like their bits).  NaNs are ignored, as fmax does.
__global__ void __launch_bounds__(1024) dsfft_max_kernel(const double* __restrict__ v, int64_t n,
                                                         double* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(m));
}

// sum |Y|^2 for the floor bound (order irrelevant: a bound with a wide margin)
__global__ void __launch_bounds__(1024) dsfft_norm2_kernel(const cd* __restrict__ y, int64_t n,
                                                           double* __restrict__ out) {
  __shared__ double part[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s += y[i].re * y[i].re + y[i].im * y[i].im;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += part[w];
    atomicAdd(out, r);
  }
}

namespace {

// Stream-ordered device buffer from the library pool.
struct DBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void reset() {
    if (p) scratch_free(p, st);
    p = nullptr;
  }
  int alloc(size_t bytes, cudaStream_t s, const char* what) {
    reset();
    st = s;
    cudaError_t e = scratch_alloc(&p, std::max<size_t>(bytes, 16), s);
    return e == cudaSuccess ? AFFT_OK : cuda_status(e, what);
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// AFFT_DSFFT_PROFILE=1: host time spent waiting in read-backs vs issuing work
struct HostProf {
  bool on = std::getenv("AFFT_DSFFT_PROFILE") != nullptr;
  double wait_s = 0.0;
  int syncs = 0;
};
thread_local HostProf g_prof;

struct Marks {
  double last = 0.0, last_wait = 0.0;
  struct Acc {
    const char* what;
    double total, wait;
    int n;
  };
  std::vector<Acc> acc;
  void mark(const char* what, double t, double wait) {
    Acc* a = nullptr;
    for (auto& x : acc)
      if (x.what == what) a = &x;
    if (!a) {
      acc.push_back({what, 0.0, 0.0, 0});
      a = &acc.back();
    }
    a->total += t - last;
    a->wait += wait - last_wait;
    ++a->n;
    last = t;
    last_wait = wait;
  }
};
thread_local Marks g_marks;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define PMARK(what)                                  \
  do {                                               \
    if (g_prof.on) g_marks.mark(what, now_s(), g_prof.wait_s); \
  } while (0)

template <class T>
int d2h(std::vector<T>& h, const void* d, size_t count, cudaStream_t st) {
  h.resize(count);
  if (!count) return AFFT_OK;
  const double t0 = g_prof.on ? now_s() : 0.0;
  const size_t bytes = count * sizeof(T);
  size_t cap = 0;
  void* stage = pinned_acquire(bytes, &cap);  // a pageable D2H copy costs a bounce
  cudaError_t e = cudaMemcpyAsync(stage ? stage : (void*)h.data(), d, bytes,
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) {
    // AFFT_BLOCKING_SYNC=1: wait on a blocking-sync event (the thread sleeps) instead of
    // the stream's spin-wait — many concurrent decodes on few host cores
    static const bool blocking = [] {
      const char* v = std::getenv("AFFT_BLOCKING_SYNC");
      return v && v[0] == '1';
    }();
    if (blocking) {
      thread_local cudaEvent_t ev = nullptr;
      thread_local int ev_dev = -1;
      int dev = 0;
      e = cudaGetDevice(&dev);
      if (e == cudaSuccess && ev && ev_dev != dev) {  // events belong to a device
        cudaEventDestroy(ev);
        ev = nullptr;
      }
      if (e == cudaSuccess && !ev) {
        e = cudaEventCreateWithFlags(&ev, cudaEventBlockingSync | cudaEventDisableTiming);
        ev_dev = dev;
      }
      if (e == cudaSuccess) e = cudaEventRecord(ev, st);
      if (e == cudaSuccess) e = cudaEventSynchronize(ev);
    } else {
      e = cudaStreamSynchronize(st);
    }
  }
  if (e == cudaSuccess && stage) std::memcpy(h.data(), stage, bytes);
  pinned_release(stage, cap);
  if (g_prof.on) {
    g_prof.wait_s += now_s() - t0;
    ++g_prof.syncs;
  }
  return e == cudaSuccess ? AFFT_OK : cuda_status(e, "dsfft read-back");
}

#define RC(expr)          \
  do {                    \
    int _rc = (expr);     \
    if (_rc) return _rc;  \
  } while (0)

// CUDA runtime call in the layer loop: map a failure to the library's status
#define CK(expr)                                             \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return cuda_status(_e, #expr);    \
  } while (0)

struct Layer {
  int depth = 0;
  int64_t m = 0;     // active count
  DBuf active;       // ascending bucket indices (device int64)
};

void swap_layers(Layer& a, Layer& b) {
  std::swap(a.depth, b.depth);
  std::swap(a.m, b.m);
  std::swap(a.active.p, b.active.p);
  std::swap(a.active.st, b.active.st);
}

// Python dict insertion semantics for the entries: a new key appends, a repeated
// key keeps its position and takes the new value.  Open addressing over int64 keys
// (frequencies, >= 0), table reused across layers: clear() resets only the slots in use.
struct Entries {
  std::vector<int64_t> f;
  std::vector<cd> v;
  std::vector<int64_t> slot_key;  // -1 = empty
  std::vector<int32_t> slot_pos;
  size_t mask = 0;
  std::vector<size_t> used;  // occupied slots (a probe chain must not be cut while clearing)
  void clear() {
    for (size_t h : used) slot_key[h] = -1;
    used.clear();
    f.clear();
    v.clear();
  }
  size_t find(int64_t key) const {  // the key's slot, or the empty slot where it belongs
    size_t h = (size_t)((uint64_t)key * 0x9E3779B97F4A7C15ull >> 20) & mask;
    while (slot_key[h] != -1 && slot_key[h] != key) h = (h + 1) & mask;
    return h;
  }
  void grow(size_t need) {
    if (!slot_key.empty() && 2 * need <= slot_key.size()) return;
    size_t cap = 1024;
    while (cap < 2 * need) cap <<= 1;
    slot_key.assign(cap, -1);
    slot_pos.assign(cap, 0);
    mask = cap - 1;
    used.clear();
    for (size_t i = 0; i < f.size(); ++i) {
      const size_t h = find(f[i]);
      slot_key[h] = f[i];
      slot_pos[h] = (int32_t)i;
      used.push_back(h);
    }
  }
  void reserve(size_t extra) { grow(f.size() + extra); }
  void put(int64_t key, cd val) {  // callers reserve() first
    const size_t h = find(key);
    if (slot_key[h] == -1) {
      slot_key[h] = key;
      slot_pos[h] = (int32_t)f.size();
      used.push_back(h);
      f.push_back(key);
      v.push_back(val);
    } else {
      v[slot_pos[h]] = val;
    }
  }
};

struct Tracer {
  int32_t* buf;
  int32_t cap;
  int32_t len = 0;
  void add(int kind, int64_t a, int64_t b, int64_t c) {
    if (buf && len < cap) {
      buf[4 * len + 0] = kind;
      buf[4 * len + 1] = (int32_t)a;
      buf[4 * len + 2] = (int32_t)b;
      buf[4 * len + 3] = (int32_t)c;
    }
    ++len;
  }
};

struct Dsfft {
  const void* x;
  int dtype;
  int64_t n;
  int k;
  const AfftDsfftParams& P;
  cudaStream_t st;
  Tracer tr;
  int max_depth = 0;
  double noise_std = 0.0;
  DBuf Y;             // resident spectrum fft(x)/n (lazy)
  double normY = -1;  // ||Y||^2 (lazy)

  // Full deep layers (L <= 32) from one pass over Y for all of them (deep_active_all),
  // made at the first such expansion: per-layer lists + counts, read back once.
  bool deep_done = false;
  int deep_d0 = 0, deep_nl = 0, deep_cap = 0;
  DBuf deep_lists;
  std::vector<int32_t> deep_counts;

  // Host copies of those lists for the probe classifies (copied asynchronously right
  // after the counts, waited for at the first probe): one pinned block, per-layer offsets.
  void* hl_stage = nullptr;
  size_t hl_cap = 0;
  std::vector<size_t> hl_off;
  cudaEvent_t hl_ev = nullptr;
  bool hl_ready = false;
  ~Dsfft() {
    if (hl_ev) {
      cudaEventSynchronize(hl_ev);  // the copy must land before the block is reused
      cudaEventDestroy(hl_ev);
    }
    pinned_release(hl_stage, hl_cap);
  }

  // Probe classifies (full_classify = 0, noisy mode): an intermediate layer's entries are
  // discarded by the reference (dsfft.py:188-192 keeps only the last classify's), so such
  // a layer only has to show that some multi-ton remains.  It classifies the active
  // children of the previous layer's multi-tons found so far (the first layer: its first
  // kProbe0 active buckets); if none of them is a multi-ton, the whole layer is
  // classified as the reference does.  The bottom layer is always classified in full.
  // AFFT_DSFFT_PROBE0 sets the first layer's probe size (0 disables probing).
  bool lazy = false;
  int64_t probe0 = [] {
    const char* e = std::getenv("AFFT_DSFFT_PROBE0");
    return e ? std::max<int64_t>(0, std::atoll(e)) : 256;
  }();

  static constexpr int64_t kAliasMaxL = 32;       // rows + energies + values from Y
  static constexpr int64_t kAliasRowsMaxL = 256;  // rows alone from Y

  bool alias_ok(int64_t b) const { return n / b <= kAliasMaxL; }

  // Rows from the resident spectrum instead of min(#shifts, L) size-b DFTs over the
  // signal: worth it once Y exists (A*L*R products against ~min(R, L)*b*log b), and
  // worth computing Y for at L <= 64, where one layer's DFTs cost a full transform.
  // AFFT_DSFFT_Y_L: the largest L at which rows alone justify computing Y (default 64).
  // Rows from Y cost one L-strided gather per active bucket (a sector per alias): at
  // config 4, L = 2048 / 1024 / 512 took 258 / 121 / 71 us against 20 / 41 / 61 us for
  // the coset DFTs over the signal, so shallow layers keep the DFTs (ncu launch lists).
  int64_t y_rows_l = [] {
    const char* e = std::getenv("AFFT_DSFFT_Y_L");
    return e ? std::max<int64_t>(1, std::atoll(e)) : 64;
  }();
  // Larger L: one CTA per row (L <= kAliasCtaMaxL), when asked for (AFFT_DSFFT_Y_L) or when the
  // list is short enough (probe classifies) that its A L products cost less than the
  // coset DFTs: ~83 ns per row at L = 2048 against ~23 us for the DFTs at config 4's
  // depth 13 (launch lists), so up to A L = 2^19 once Y is resident.
  static constexpr int64_t kShortRowsBudget = int64_t(1) << 19;
  bool alias_rows_ok(int64_t b, int64_t count = -1) const {
    const int64_t L = n / b;
    if (L <= kAliasMaxL) return true;
    if (L <= kAliasRowsMaxL) return Y.p || L <= y_rows_l;
    if (L > kAliasCtaMaxL) return false;
    return L <= y_rows_l || (Y.p && count >= 0 && count * L <= kShortRowsBudget);
  }

  // ||Y||^2 for the noisy floor bound: from Y when resident, else by Parseval from x
  // (sum |x|^2 / n); only ever compared against a bound with a wide margin.
  int norm_y() {
    if (normY >= 0) return AFFT_OK;
    if (Y.p && dtype != AFFT_C64) {  // a c64 signal is half the bytes of its spectrum
      DBuf s;
      RC(s.alloc(8, st, "dsfft norm"));
      CK(cudaMemsetAsync(s.p, 0, 8, st));
      dsfft_norm2_kernel<<<148 * 4, 1024, 0, st>>>(Y.as<cd>(), n, s.as<double>());
      std::vector<double> h;
      RC(d2h(h, s.p, 1, st));
      normY = h[0];
      return AFFT_OK;
    }
    const int nparts = afft_sumsq_parts(n, dtype);
    DBuf parts;
    RC(parts.alloc((size_t)std::max(nparts, 1) * 8, st, "dsfft partials"));
    RC(afft_sumsq(x, dtype, n, 1, n, parts.as<double>(), st));
    std::vector<double> h;
    RC(d2h(h, parts.p, (size_t)nparts, st));
    double sum = 0.0;
    for (double v : h) sum += v;
    normY = sum / (double)n;
    return AFFT_OK;
  }

  int spectrum() {
    if (Y.p) return AFFT_OK;
    RC(Y.alloc((size_t)n * 16, st, "dsfft spectrum"));
    const int64_t zero = 0;
    return afft_bucketize(x, dtype, n, 1, n, n, &zero, 1, Y.as<double>(), n, n, 1, st);
  }

  // full layer values at tau = 0 (bucketize.py:83-99)
  int full_values(int64_t b, DBuf& vals) {
    RC(vals.alloc((size_t)b * 16, st, "dsfft layer values"));
    if (alias_ok(b)) {
      RC(spectrum());
      return afft_alias_rows(Y.as<double>(), n, b, nullptr, 0, nullptr, 0, nullptr, nullptr,
                             vals.as<double>(), st);
    }
    const int64_t zero = 0;
    return afft_bucketize(x, dtype, n, 1, n, b, &zero, 1, vals.as<double>(), b, b, 1, st);
  }

  int active(const DBuf& vals, int64_t count, double thr, const int64_t* map, Layer& out) {
    PMARK("layer values");
    RC(out.active.alloc((size_t)std::max<int64_t>(count, 1) * 8, st, "dsfft active"));
    DBuf cnt;
    RC(cnt.alloc(4, st, "dsfft count"));
    RC(afft_active_indices(vals.as<double>(), count, thr, map, out.active.as<int64_t>(),
                           cnt.as<int32_t>(), st));
    std::vector<int32_t> h;
    RC(d2h(h, cnt.p, 1, st));
    out.m = h[0];
    PMARK("active set");
    return AFFT_OK;
  }

  double threshold(int depth) const {  // dsfft.py:69-71
    return std::max(P.activity_floor, 3.0 * noise_std / std::sqrt((double)(1LL << depth)));
  }

  // AFFT_ACTIVE_SORT_CAP lowers the capacity of the one-pass active lists (tests force
  // the per-layer fallbacks with it); read per call
  static int active_cap(int64_t b) {
    const char* cap_var = std::getenv("AFFT_ACTIVE_SORT_CAP");
    const int64_t cap_env = cap_var ? std::max<int64_t>(1, std::atoll(cap_var)) : 16384;
    return (int)std::min<int64_t>(b, std::min<int64_t>(16384, cap_env));
  }

  // A full layer's active set from the cached one-pass lists (layers_all), if held.
  bool cached_layer(int depth, int kind, Layer& out, int* rc) {
    *rc = AFFT_OK;
    if (!deep_done || depth < deep_d0 || depth >= deep_d0 + deep_nl) return false;
    const int j = depth - deep_d0;
    if (deep_counts[j] > std::min(active_cap(1LL << depth), deep_cap)) return false;
    out.depth = depth;
    out.m = deep_counts[j];
    if ((*rc = out.active.alloc((size_t)std::max<int64_t>(out.m, 1) * 8, st, "dsfft active")))
      return true;
    if (out.m) {
      const cudaError_t e =
          cudaMemcpyAsync(out.active.p, deep_lists.as<int64_t>() + (int64_t)j * deep_cap,
                          (size_t)out.m * 8, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) {
        *rc = cuda_status(e, "dsfft cached active list");
        return true;
      }
    }
    PMARK("active set");
    tr.add(kind, depth, out.m, -1);
    return true;
  }

  int initial(int depth, Layer& out) {
    int crc = AFFT_OK;
    if (cached_layer(depth, 1, out, &crc)) return crc;
    DBuf vals;
    RC(full_values(1LL << depth, vals));
    out.depth = depth;
    RC(active(vals, 1LL << depth, threshold(depth), nullptr, out));
    tr.add(1, depth, out.m, -1);
    return AFFT_OK;
  }

  int expand(const Layer& prev, Layer& out) {
    const int depth = prev.depth + 1;
    const int64_t b = 1LL << depth;
    if (b > n) {
      set_error("layer depth exceeds log2 of the signal size");
      return AFFT_EINVAL;
    }
    out.depth = depth;
    const double thr = threshold(depth);
    if (2 * prev.m <= depth) {  // selective: only the children of active buckets
      const int64_t nc = 2 * prev.m;
      DBuf cand, vals;
      RC(cand.alloc((size_t)std::max<int64_t>(nc, 1) * 8, st, "dsfft candidates"));
      RC(vals.alloc((size_t)std::max<int64_t>(nc, 1) * 16, st, "dsfft candidate values"));
      if (nc) {
        dsfft_cand_kernel<<<(unsigned)((prev.m + 255) / 256), 256, 0, st>>>(
            prev.active.as<int64_t>(), prev.m, b >> 1, cand.as<int64_t>());
        RC(afft_selective_sums(x, dtype, n, b, cand.as<int64_t>(), nc, vals.as<double>(), st));
        RC(active(vals, nc, thr, cand.as<int64_t>(), out));
      } else {
        RC(out.active.alloc(8, st, "dsfft active"));
        out.m = 0;
      }
      tr.add(2, depth, out.m, nc);
      return AFFT_OK;
    }
    {
      int crc = AFFT_OK;
      if (cached_layer(depth, 2, out, &crc)) return crc;
    }
    if (alias_ok(b)) {  // deep layer: active set in one pass over Y, values never stored
      RC(spectrum());
      const int cap = active_cap(b);
      if (!deep_done && !std::getenv("AFFT_DSFFT_DEEP_PER_LAYER")) {
        RC(layers_all(depth, cap));
        int crc = AFFT_OK;
        if (cached_layer(depth, 2, out, &crc)) return crc;
      }
      RC(out.active.alloc((size_t)cap * 8, st, "dsfft active"));
      DBuf cnt;
      RC(cnt.alloc(4, st, "dsfft count"));
      RC(alias_active(Y.as<double>(), n, b, thr, out.active.as<int64_t>(), cap,
                      cnt.as<int32_t>(), st));
      std::vector<int32_t> h;
      RC(d2h(h, cnt.p, 1, st));
      if (h[0] <= cap) {
        out.m = h[0];
        PMARK("active set");
        tr.add(2, depth, out.m, -1);
        return AFFT_OK;
      }
    }
    DBuf vals;  // shallow layers, or more active buckets than the one-CTA sort holds
    RC(full_values(b, vals));
    RC(active(vals, b, thr, nullptr, out));
    tr.add(2, depth, out.m, -1);
    return AFFT_OK;
  }

  // The active lists of every full layer from `depth` to the bottom in one pass over
  // the resident spectrum (full_active_all): the layers with n/b <= 32 directly, the
  // shallower ones by summing children pairwise; one read-back of all the counts.
  int layers_all(int depth, int cap) {
    deep_done = true;  // attempted: a failure below leaves the per-layer path
    const int nl = max_depth - depth + 1;
    if (nl < 1 || nl > 16 || (1LL << depth) < 32 || (n & (n - 1))) return AFFT_OK;
    std::vector<double> thr((size_t)nl);
    for (int j = 0; j < nl; ++j) thr[j] = threshold(depth + j);
    DBuf counts, scratch;
    RC(deep_lists.alloc((size_t)nl * cap * 8, st, "dsfft layer lists"));
    const size_t onorm = ((size_t)nl * 4 + 7) & ~size_t(7);  // counts | sum |Y|^2
    RC(counts.alloc(onorm + 8, st, "dsfft layer counts"));
    const size_t sb = std::max(full_active_scratch(n, depth, nl),
                                 full_active_fused_scratch(n, depth, nl));
    RC(scratch.alloc(sb, st, "dsfft layer scratch"));
    // the spectrum's last pass deciding the deepest nine layers in its epilogue
    // (AFFT_DSFFT_FUSE=0: spectrum, then one pass over it)
    const char* fe = std::getenv("AFFT_DSFFT_FUSE");
    const bool fuse_env = !(fe && fe[0] == '0');
    bool fused = false;
    if (!Y.p && fuse_env) {
      RC(Y.alloc((size_t)n * 16, st, "dsfft spectrum"));
      double* norm2 = reinterpret_cast<double*>(counts.as<char>() + onorm);
      const int rc = full_active_all_fused(x, dtype, n, Y.as<double>(), depth, nl, thr.data(),
                                           deep_lists.as<int64_t>(), cap, counts.as<int32_t>(),
                                           norm2, scratch.p, sb, st);
      if (rc == AFFT_OK) {
        fused = true;
      } else if (rc == AFFT_EUNSUPPORTED) {
        Y.reset();  // another plan: the unfused path below
      } else {
        return rc;
      }
    }
    if (!fused) {
      RC(spectrum());
      RC(full_active_all(Y.as<double>(), n, depth, nl, thr.data(), deep_lists.as<int64_t>(), cap,
                         counts.as<int32_t>(), scratch.p, sb, st));
    }
    std::vector<char> hb;
    RC(d2h(hb, counts.p, onorm + (fused ? 8 : 0), st));
    deep_counts.resize((size_t)nl);
    std::memcpy(deep_counts.data(), hb.data(), (size_t)nl * 4);
    if (fused && normY < 0) std::memcpy(&normY, hb.data() + onorm, 8);
    deep_d0 = depth;
    deep_nl = nl;
    deep_cap = cap;
    if (lazy) {
      hl_off.assign((size_t)nl + 1, 0);
      for (int j = 0; j < nl; ++j)
        hl_off[j + 1] = hl_off[j] + (size_t)std::min(deep_counts[j], cap);
      hl_stage = pinned_acquire(std::max<size_t>(hl_off[nl], 1) * 8, &hl_cap);
      if (hl_stage) {
        CK(cudaEventCreateWithFlags(&hl_ev, cudaEventDisableTiming));
        for (int j = 0; j < nl; ++j)
          if (hl_off[j + 1] > hl_off[j])
            CK(cudaMemcpyAsync(static_cast<int64_t*>(hl_stage) + hl_off[j],
                               deep_lists.as<int64_t>() + (int64_t)j * cap,
                               (hl_off[j + 1] - hl_off[j]) * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(hl_ev, st));
      }
    }
    return AFFT_OK;
  }

  // The host copy of a cached full layer's ascending active list (nullptr if not held).
  const int64_t* host_list(int depth, int64_t* m) {
    if (!hl_stage || !deep_done || depth < deep_d0 || depth >= deep_d0 + deep_nl) return nullptr;
    const int j = depth - deep_d0;
    if (deep_counts[j] > std::min(active_cap(1LL << depth), deep_cap)) return nullptr;
    if (!hl_ready) {
      if (cudaEventSynchronize(hl_ev) != cudaSuccess) return nullptr;
      hl_ready = true;
    }
    *m = deep_counts[j];
    return static_cast<const int64_t*>(hl_stage) + hl_off[j];
  }

  int rows(int64_t b, const std::vector<int64_t>& shifts, const int64_t* idx, int64_t count,
           DBuf& out, double* energy) {
    const int ns = (int)shifts.size();
    RC(out.alloc((size_t)std::max<int64_t>(count, 1) * ns * 16, st, "dsfft rows"));
    if (alias_ok(b) || (!energy && alias_rows_ok(b, count))) {
      RC(spectrum());
      return afft_alias_rows(Y.as<double>(), n, b, shifts.data(), ns, count ? idx : nullptr, count,
                             out.as<double>(), energy, nullptr, st);
    }
    return afft_bucketize_rows(x, dtype, n, b, shifts.data(), ns, count ? idx : nullptr, count,
                               out.as<double>(), energy, st);
  }

  // One device block per classification, read back in one copy:
  // f0 [A] int64 | value [A] c128 | bucket [A] int64 | state [A] int8.
  struct Pack {
    DBuf buf;
    int64_t A = 0;
    size_t of = 0, ov = 0, oa = 0, os = 0, bytes = 0;
    int64_t* f0() const { return reinterpret_cast<int64_t*>(buf.as<char>() + of); }
    double* val() const { return reinterpret_cast<double*>(buf.as<char>() + ov); }
    int8_t* state() const { return reinterpret_cast<int8_t*>(buf.as<char>() + os); }
  };

  int make_pack(const int64_t* idx, int64_t A, Pack& pk) {
    pk.A = A;
    if (!A) return AFFT_OK;
    pk.of = 0;
    pk.ov = (size_t)A * 8;
    pk.oa = pk.ov + (size_t)A * 16;
    pk.os = pk.oa + (size_t)A * 8;
    pk.bytes = pk.os + (size_t)A;
    RC(pk.buf.alloc(pk.bytes, st, "dsfft result pack"));
    char* p = pk.buf.as<char>();
    CK(cudaMemcpyAsync(p + pk.oa, idx, (size_t)A * 8, cudaMemcpyDeviceToDevice, st));
    if (P.mode == 0) {  // classify_exact writes f0 / value for single-tons only; the noisy
                        // finalize writes every row's
      CK(cudaMemsetAsync(p + pk.of, 0xff, (size_t)A * 8, st));  // f0 = -1
      CK(cudaMemsetAsync(p + pk.ov, 0, (size_t)A * 16, st));
    }
    return AFFT_OK;
  }

  // _classify_active: entries (ascending bucket order) and multiton buckets
  int classify(const Layer& L, Entries& E, std::vector<int64_t>& multi) {
    bool declined = false;
    return classify_list(L.depth, L.active.as<int64_t>(), L.m, false, E, multi, &declined);
  }

  // A probe classify of `cand` (ascending, a subset of layer `depth`'s active set): the
  // multi-tons among them into `found`, no entries.  *declined (nothing done) when the
  // layer's thresholds need the all-bucket energy pass or the quiet-bucket median.
  int probe(int depth, const std::vector<int64_t>& cand, std::vector<int64_t>& found,
            bool* declined) {
    DBuf idx;
    RC(idx.alloc(std::max<size_t>(cand.size(), 1) * 8, st, "dsfft probe list"));
    if (!cand.empty())
      CK(cudaMemcpyAsync(idx.p, cand.data(), cand.size() * 8, cudaMemcpyHostToDevice, st));
    Entries none;
    return classify_list(depth, idx.as<int64_t>(), (int64_t)cand.size(), true, none, found,
                         declined);
  }

  int classify_list(int depth, const int64_t* idx, int64_t A, bool is_probe, Entries& E,
                    std::vector<int64_t>& multi, bool* declined) {
    *declined = false;
    E.clear();
    multi.clear();
    const int64_t b = 1LL << depth;
    Pack pk;
    DBuf rowsb;
    if (is_probe && P.mode == 0) {
      *declined = true;
      return AFFT_OK;
    }
    RC(make_pack(idx, A, pk));
    if (P.mode == 0) {
      tr.add(5, depth, 3, 0);  // ledger: shifts 0, 1, 2
      if (A == 0) return finish_classify(depth, E, multi, pk, is_probe);
      const std::vector<int64_t> shifts = {0, 1, 2};
      RC(rows(b, shifts, idx, A, rowsb, nullptr));
      // exact_thresholds (peeling.py:316-318)
      const int nparts = afft_sumsq_parts(n, dtype);
      DBuf parts, eps;
      RC(parts.alloc((size_t)std::max(nparts, 1) * 8, st, "dsfft partials"));
      RC(eps.alloc(8, st, "dsfft eps"));
      RC(afft_sumsq(x, dtype, n, 1, n, parts.as<double>(), st));
      RC(afft_exact_thresholds(parts.as<double>(), nparts, n, 1, eps.as<double>(), st));
      std::vector<double> he;
      RC(d2h(he, eps.p, 1, st));
      RC(afft_classify_exact(rowsb.as<double>(), idx, A, b, n, he[0], he[0],
                             pk.state(), pk.f0(), pk.val(), st));
      return finish_classify(depth, E, multi, pk, is_probe);
    }
    // noisy: the search plan of dsfft.py:142-150 (anchors drawn by the caller)
    std::vector<int64_t> shifts;
    for (int j = 0; j < P.c; ++j)
      for (int t = 0; t < P.m; ++t) shifts.push_back(P.anchors[j] + (int64_t(1) << j) * t);
    const int R = (int)shifts.size();
    const double base = noise_std / std::sqrt((double)b) * std::sqrt((double)R);
    bool skip = false;
    if (noise_std > 0.0) {
      // floor = 1e-8 sqrt(max_i energy_i) <= 1e-8 sqrt(R L ||Y||^2) (Cauchy-Schwarz on
      // the alias sums): when that bound is below 1.5 base the floor cannot matter and
      // the all-bucket energy pass is skipped (1.0001: rounding of the norm itself)
      RC(norm_y());
      skip = 1e-8 * std::sqrt((double)R * (double)(n / b) * normY * 1.0001) < 1.5 * base;
    }
    if (is_probe && !skip) {  // thresholds from every bucket: classify the layer in full
      *declined = true;
      return AFFT_OK;
    }
    // ledger: the plan shifts, once per layer the reference classifies (a probe records
    // them only when it decides the layer, i.e. finds a multi-ton; see finish_classify)
    if (!is_probe) tr.add(5, depth, R, 1);
    DBuf energy;
    if (!skip) RC(energy.alloc((size_t)b * 8, st, "dsfft energies"));
    PMARK("classify setup");
    RC(rows(b, shifts, idx, A, rowsb, skip ? nullptr : energy.as<double>()));
    PMARK("classify rows");
    double t0 = 0.0, t1 = 0.0;
    if (noise_std > 0.0) {
      double floor = 0.0;
      if (!skip) {
        DBuf mx;
        RC(mx.alloc(8, st, "dsfft max"));
        CK(cudaMemsetAsync(mx.p, 0, 8, st));
        const unsigned grid = (unsigned)std::min<int64_t>(148 * 2, (b + 1023) / 1024);
        dsfft_max_kernel<<<grid, 1024, 0, st>>>(energy.as<double>(), b, mx.as<double>());
        std::vector<double> h;
        RC(d2h(h, mx.p, 1, st));
        floor = 1e-8 * std::sqrt(h[0]);
      }
      t0 = std::max(1.5 * base, floor);
      t1 = std::max(2.5 * base, floor);
    } else {
      DBuf quiet, d0;
      RC(quiet.alloc((size_t)b, st, "dsfft quiet mask"));
      RC(d0.alloc(16, st, "dsfft t0 t1"));
      dsfft_quiet_kernel<<<148 * 4, 256, 0, st>>>(b, nullptr, 0, quiet.as<uint8_t>());
      if (A)
        dsfft_unquiet_kernel<<<(unsigned)((A + 255) / 256), 256, 0, st>>>(
            idx, A, quiet.as<uint8_t>());
      RC(afft_robust_thresholds(energy.as<double>(), quiet.as<uint8_t>(), b, 1, R, d0.as<double>(),
                                d0.as<double>() + 1, st));
      std::vector<double> h;
      RC(d2h(h, d0.p, 2, st));
      t0 = h[0];
      t1 = h[1];
    }
    PMARK("classify thresholds");
    if (A == 0) return finish_classify(depth, E, multi, pk, is_probe);
    DBuf rn, ws;
    RC(rn.alloc((size_t)A * 8, st, "dsfft resnorm"));
    const size_t need = afft_singleton_workspace_size(n, A, b, P.c, P.m);
    RC(ws.alloc(need, st, "dsfft search workspace"));
    RC(afft_classify_noisy(rowsb.as<double>(), idx, A, b, n, shifts.data(), R,
                           P.c, P.m, P.weights, t0, t1, pk.state(), pk.f0(), pk.val(),
                           rn.as<double>(), ws.p, need, st));
    PMARK("classify noisy");
    const int rcf = finish_classify(depth, E, multi, pk, is_probe);
    PMARK("classify finish");
    return rcf;
  }

  int finish_classify(int depth, Entries& E, std::vector<int64_t>& multi, const Pack& pk,
                      bool is_probe) {
    const int64_t A = pk.A;
    if (A) {
      std::vector<char> h;
      PMARK("classify pack");
      RC(d2h(h, pk.buf.p, pk.bytes, st));
      PMARK("classify read-back");
      const int64_t* hf = reinterpret_cast<const int64_t*>(h.data() + pk.of);
      const cd* hv = reinterpret_cast<const cd*>(h.data() + pk.ov);
      const int64_t* ha = reinterpret_cast<const int64_t*>(h.data() + pk.oa);
      const int8_t* hs = reinterpret_cast<const int8_t*>(h.data() + pk.os);
      E.reserve((size_t)A);
      for (int64_t i = 0; i < A; ++i) {
        if (hs[i] == AFFT_SINGLE_TON) {  // ascending bucket order, as the reference inserts
          if (!is_probe) E.put(hf[i], hv[i]);
        } else if (hs[i] == AFFT_MULTI_TON) {
          multi.push_back(ha[i]);
        }
      }
    }
    if (is_probe && !multi.empty()) tr.add(5, depth, P.c * P.m, 1);
    if (!is_probe || !multi.empty())
      tr.add(3, depth, is_probe ? -1 : (int64_t)E.f.size(), (int64_t)multi.size());
    return AFFT_OK;
  }

  // _resolve_aliased: DT3 detect + solve on the leftover multi-ton buckets
  int resolve(int depth, const std::vector<int64_t>& buckets, int64_t remaining, Entries& E) {
    const int64_t b = 1LL << depth;
    const int a_m = P.a_m;
    const int32_t off0 = P.dt_shift_off[depth], off1 = P.dt_shift_off[depth + 1];
    const int p = off1 - off0;
    std::vector<int64_t> shifts;
    for (int t = -a_m; t < 2 * a_m; ++t) shifts.push_back(t);
    for (int i = off0; i < off1; ++i) shifts.push_back(P.dt_shifts[i]);
    tr.add(4, depth, (int64_t)buckets.size(), p);
    const int64_t nm = (int64_t)buckets.size();
    const int R = (int)shifts.size();
    DBuf idx, rowsb, counts, sig, rs, pos, val, cnt;
    RC(idx.alloc((size_t)nm * 8, st, "dsfft resolve ids"));
    CK(cudaMemcpyAsync(idx.p, buckets.data(), (size_t)nm * 8, cudaMemcpyHostToDevice, st));
    RC(rows(b, shifts, idx.as<int64_t>(), nm, rowsb, nullptr));
    RC(counts.alloc((size_t)nm * 4, st, "dsfft counts"));
    RC(sig.alloc((size_t)nm * a_m * 8, st, "dsfft sigmas"));
    const int64_t kk = std::min<int64_t>(remaining, (int64_t)a_m * nm);
    RC(afft_dt_detect(rowsb.as<double>(), 1, nm, R, a_m, (int32_t)kk, counts.as<int32_t>(),
                      sig.as<double>(), st));
    RC(rs.alloc((size_t)std::max(p, 1) * 8, st, "dsfft random shifts"));
    if (p)
      CK(cudaMemcpyAsync(rs.p, P.dt_shifts + off0, (size_t)p * 8, cudaMemcpyHostToDevice, st));
    RC(pos.alloc((size_t)nm * a_m * 8, st, "dsfft pos"));
    RC(val.alloc((size_t)nm * a_m * 16, st, "dsfft val"));
    RC(cnt.alloc((size_t)nm * 4, st, "dsfft cnt"));
    RC(afft_dt_solve(rowsb.as<double>(), rs.as<int64_t>(), 1, nm, a_m, p, counts.as<int32_t>(),
                     idx.as<int64_t>(), 3, a_m, b, n, pos.as<int64_t>(), val.as<double>(),
                     cnt.as<int32_t>(), st));
    DBuf pack;  // one read-back: positions | values | counts
    const size_t ov = (size_t)nm * a_m * 8, oc = ov + (size_t)nm * a_m * 16;
    RC(pack.alloc(oc + (size_t)nm * 4, st, "dsfft resolve pack"));
    char* pk = pack.as<char>();
    CK(cudaMemcpyAsync(pk, pos.p, ov, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(pk + ov, val.p, (size_t)nm * a_m * 16, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(pk + oc, cnt.p, (size_t)nm * 4, cudaMemcpyDeviceToDevice, st));
    std::vector<char> h;
    RC(d2h(h, pk, oc + (size_t)nm * 4, st));
    const int64_t* hp = reinterpret_cast<const int64_t*>(h.data());
    const cd* hv = reinterpret_cast<const cd*>(h.data() + ov);
    const int32_t* hc = reinterpret_cast<const int32_t*>(h.data() + oc);
    E.reserve((size_t)nm * a_m);
    for (int64_t r = 0; r < nm; ++r)
      for (int j = 0; j < hc[r]; ++j) E.put(hp[r * a_m + j], hv[r * a_m + j]);  // .update()
    return AFFT_OK;
  }

  int calibrate() {  // dsfft.py:231-241
    int e = 0;
    while ((1LL << e) < 32LL * k) ++e;
    const int64_t b = std::min<int64_t>(n, 1LL << e);
    DBuf vals, med;
    RC(full_values(b, vals));
    RC(med.alloc(8, st, "dsfft median"));
    RC(afft_median(vals.as<double>(), 1, b, 1, med.as<double>(), st));
    std::vector<double> h;
    RC(d2h(h, med.p, 1, st));
    tr.add(0, (int64_t)std::log2((double)b), 0, 0);
    noise_std = std::sqrt((double)b * h[0] / std::log(2.0));
    return AFFT_OK;
  }

  // One classify step of the loop: a probe first where allowed (see `lazy`), the whole
  // layer otherwise or when the probe finds no multi-ton.  `multi` holds the multi-tons
  // found (all of them after a full classify, the probe's after a probe).
  int classify_layer(const Layer& L, Entries& E, std::vector<int64_t>& multi, bool first) {
    int64_t m = 0;
    const int64_t* act = (lazy && L.depth < max_depth) ? host_list(L.depth, &m) : nullptr;
    if (act && m > 0) {
      std::vector<int64_t> cand;
      if (first) {
        cand.assign(act, act + std::min<int64_t>(m, probe0));
      } else {  // active children {i, i + 2^(d-1)} of the multi-tons found one layer up
        const int64_t half = 1LL << (L.depth - 1);
        for (int pass = 0; pass < 2; ++pass)
          for (int64_t i : multi) {
            const int64_t c = i + (pass ? half : 0);
            if (std::binary_search(act, act + m, c)) cand.push_back(c);
          }
      }
      if (!cand.empty() && (int64_t)cand.size() < m) {
        std::vector<int64_t> found;
        bool declined = false;
        RC(probe(L.depth, cand, found, &declined));
        PMARK("probe");
        if (!declined && !found.empty()) {
          multi.swap(found);
          return AFFT_OK;
        }
      }
    }
    return classify(L, E, multi);
  }

  int run(Entries& E) {
    lazy = P.mode != 0 && !P.full_classify && probe0 > 0;
    max_depth = 0;
    while ((2LL << max_depth) <= n) ++max_depth;  // n.bit_length() - 1
    noise_std = P.noise_std;
    if (P.mode != 0 && noise_std <= 0.0) RC(calibrate());
    int depth = 0;
    while ((1LL << depth) < k) ++depth;  // ceil(log2 k), k >= 1
    depth = std::min(depth, max_depth);
    Layer layer, next;
    PMARK("start");
    // noisy decodes of large signals reach the bottom layer (the re-expansion runs while
    // multitons remain, dsfft.py:190-192), so the spectrum is computed first and every
    // full layer's active set comes from it in one pass (AFFT_DSFFT_LAYERS_UPFRONT=0:
    // per layer)
    static const bool upfront = [] {
      const char* e = std::getenv("AFFT_DSFFT_LAYERS_UPFRONT");
      return !(e && e[0] == '0');
    }();
    if (upfront && P.mode != 0 && n >= (1LL << 16) && (1LL << depth) >= 32 &&
        !std::getenv("AFFT_DSFFT_DEEP_PER_LAYER"))
      RC(layers_all(depth, active_cap(n)));
    RC(initial(depth, layer));
    PMARK("initial");
    while ((double)layer.m < P.theta * k && layer.depth < max_depth) {
      RC(expand(layer, next));
      swap_layers(layer, next);
      PMARK("expand");
    }
    std::vector<int64_t> multi;
    RC(classify_layer(layer, E, multi, true));
    while (P.mode != 0 && !multi.empty() && layer.depth < max_depth) {
      PMARK("loop");
      RC(expand(layer, next));
      swap_layers(layer, next);
      PMARK("expand");
      RC(classify_layer(layer, E, multi, false));
    }
    const int64_t remaining = (int64_t)k - (int64_t)E.f.size();
    PMARK("loop");
    if (!multi.empty() && remaining > 0) RC(resolve(layer.depth, multi, remaining, E));
    PMARK("resolve");
    return AFFT_OK;
  }
};

// ------------------------------------------------------------------ batches
//
// The layer loop of several signals in lockstep: one launch per step for all of them.
// Noisy decodes of large signals follow the same path (spectrum first, every full
// layer's active set from one pass, then classify at the stop depth and re-expand while
// multitons remain), so a step is "classify every signal that sits at depth d": their
// active buckets' rows in one list (alias rows from the batch's spectra, or each
// signal's coset DFTs at shallow depths), one classify_noisy over the list with
// per-row signal ids (search shifts and gates per signal), one read-back for all.
// Signals that leave the common path — calibration, a selective expansion, a layer
// whose active set overflows the one-pass lists, a classify that needs the all-bucket
// energy pass, leftover multitons at the bottom — are flagged and the caller decodes
// them alone (afft_dsfft); every other signal's decisions are the single-signal ones.
struct BatchSig {
  bool on = false, fallback = false;
  bool lazy = false;  // probe classifies (full_classify = 0)
  int mode = 0;       // next classify: 0 first probe, 1 children probe, 2 whole layer
  int depth = 0;
  int64_t m = 0;
  double normY = 0.0;
  std::vector<int64_t> shifts;  // raw plan shifts anchors[j] + 2^j t
  Entries E;
  std::vector<int64_t> multi;
  std::vector<int32_t> trace;   // [kind, depth, a, b] records
  void add(int kind, int64_t a, int64_t b, int64_t c) {
    trace.push_back(kind);
    trace.push_back((int32_t)a);
    trace.push_back((int32_t)b);
    trace.push_back((int32_t)c);
  }
};

constexpr int kBatchMax = 64;

// The active lists of every (signal, layer) packed end to end as int32 (bucket < 2^31)
// for one read-back: segment g = s nl + j holds min(count, cap) entries from
// lists + g cap, at packed offset off[g].
__global__ void pack_lists_kernel(const int64_t* __restrict__ lists, int cap,
                                  const int64_t* __restrict__ off, int32_t* __restrict__ out) {
  const int64_t g = blockIdx.x;
  const int64_t o = off[g], m = off[g + 1] - o;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) out[o + i] = (int32_t)lists[g * cap + i];
}

static int dsfft_batch_run(const void* x, int dtype, int64_t n, int64_t S, int64_t ld, int k,
                           const AfftDsfftParams* prm, std::vector<BatchSig>& sig,
                           cudaStream_t st) {
  int max_depth = 0;
  while ((2LL << max_depth) <= n) ++max_depth;
  int d0 = 0;
  while ((1LL << d0) < k) ++d0;
  d0 = std::min(d0, max_depth);
  const int nl = max_depth - d0 + 1;
  const int c = prm[0].c, mm = prm[0].m, R = c * mm;
  const char* pe = std::getenv("AFFT_DSFFT_PROBE0");
  const int64_t probe0 = pe ? std::max<int64_t>(0, std::atoll(pe)) : 256;
  sig.assign((size_t)S, BatchSig());
  for (int64_t s = 0; s < S; ++s) {
    const AfftDsfftParams& P = prm[s];
    BatchSig& g = sig[s];
    g.on = P.mode != 0 && P.noise_std > 0.0 && P.c == c && P.m == mm && P.anchors &&
           P.weights;
    g.fallback = !g.on;
    g.lazy = g.on && !P.full_classify && probe0 > 0;
    if (g.on)
      for (int j = 0; j < c; ++j)
        for (int t = 0; t < mm; ++t) g.shifts.push_back(P.anchors[j] + (int64_t(1) << j) * t);
  }
  if ((n & (n - 1)) || n < (1LL << 16) || (1LL << d0) < 32 || nl > 16 || R > AFFT_MAX_SHIFTS ||
      R < 1 || S > kBatchMax) {
    for (auto& g : sig) g.on = false, g.fallback = true;
    return AFFT_OK;
  }
  const int cap = (int)std::min<int64_t>(16384, n);
  const int64_t esz = dtype == AFFT_C64 ? 8 : 16;
  // every signal's spectrum and full layers' active lists, as afft_dsfft makes them
  // (the fused last pass when the plan allows: the same Y, bitmaps and sum |Y|^2), then
  // one read-back of all counts and norms
  DBuf Y, lists, blk, scratch, taus;
  RC(Y.alloc((size_t)S * n * 16, st, "dsfft batch spectra"));
  RC(lists.alloc((size_t)S * nl * cap * 8, st, "dsfft batch lists"));
  const int nparts = afft_sumsq_parts(n, dtype);
  const size_t onorm = ((size_t)S * nl * 4 + 7) & ~size_t(7), opart = onorm + (size_t)S * 8;
  RC(blk.alloc(opart + (size_t)S * nparts * 8, st, "dsfft batch counts"));
  int32_t* counts = blk.as<int32_t>();
  double* norms = reinterpret_cast<double*>(blk.as<char>() + onorm);
  double* parts = reinterpret_cast<double*>(blk.as<char>() + opart);
  const size_t sb = std::max(full_active_scratch(n, d0, nl),
                             full_active_fused_scratch(n, d0, nl));
  RC(scratch.alloc(sb, st, "dsfft batch layer scratch"));
  const char* fe = std::getenv("AFFT_DSFFT_FUSE");
  bool fused = !(fe && fe[0] == '0');
  std::vector<char> was_fused((size_t)S, 0);
  for (int64_t s = 0; s < S; ++s) {
    if (!sig[s].on) continue;
    std::vector<double> thr((size_t)nl);
    for (int j = 0; j < nl; ++j)
      thr[j] = std::max(prm[s].activity_floor,
                        3.0 * prm[s].noise_std / std::sqrt((double)(1LL << (d0 + j))));
    const char* xs = reinterpret_cast<const char*>(x) + s * ld * esz;
    double* Ys = Y.as<double>() + 2 * s * n;
    int64_t* ls = lists.as<int64_t>() + s * nl * cap;
    if (fused) {
      const int rc = full_active_all_fused(xs, dtype, n, Ys, d0, nl, thr.data(), ls, cap,
                                           counts + s * nl, norms + s, scratch.p, sb, st);
      if (rc == AFFT_OK) {
        was_fused[s] = 1;
        continue;
      }
      if (rc != AFFT_EUNSUPPORTED) return rc;
      fused = false;  // another plan (nothing launched): the unfused path from here on
    }
    const int64_t zero = 0;
    RC(afft_bucketize(xs, dtype, n, 1, n, n, &zero, 1, Ys, n, n, 1, st));
    RC(afft_sumsq(xs, dtype, n, 1, n, parts + s * nparts, st));
    RC(full_active_all(Ys, n, d0, nl, thr.data(), ls, cap, counts + s * nl, scratch.p, sb, st));
  }
  PMARK("b spectra enqueue");
  std::vector<char> hb;
  RC(d2h(hb, blk.p, opart + (size_t)S * nparts * 8, st));
  PMARK("b counts read-back");
  std::vector<int32_t> hc((size_t)S * nl);
  std::memcpy(hc.data(), hb.data(), hc.size() * 4);
  auto count_at = [&](int64_t s, int depth) { return (int64_t)hc[(size_t)s * nl + (depth - d0)]; };
  // host copies of every list (probe lists and the full members' rows come from them)
  std::vector<int64_t> hoff((size_t)S * nl + 1, 0);
  for (int64_t g = 0; g < S * nl; ++g)
    hoff[g + 1] = hoff[g] + (sig[g / nl].on ? std::min<int64_t>(hc[g], cap) : 0);
  std::vector<int32_t> hl;
  {
    DBuf doff, packed;
    RC(doff.alloc(hoff.size() * 8, st, "dsfft batch list offsets"));
    CK(cudaMemcpyAsync(doff.p, hoff.data(), hoff.size() * 8, cudaMemcpyHostToDevice, st));
    RC(packed.alloc((size_t)std::max<int64_t>(hoff.back(), 1) * 4, st, "dsfft batch packed lists"));
    pack_lists_kernel<<<(unsigned)(S * nl), 256, 0, st>>>(lists.as<int64_t>(), cap,
                                                          doff.as<int64_t>(), packed.as<int32_t>());
    CK(cudaGetLastError());
    RC(d2h(hl, packed.p, (size_t)hoff.back(), st));
  }
  PMARK("b lists read-back");
  auto host_list = [&](int64_t s, int depth, int64_t* m) -> const int32_t* {
    const int64_t g = s * nl + (depth - d0);
    *m = hoff[g + 1] - hoff[g];
    return hl.data() + hoff[g];
  };
  // reduced shift tables for the alias rows and the fit
  {
    std::vector<int64_t> tt((size_t)S * R, 0);
    for (int64_t s = 0; s < S; ++s)
      if (sig[s].on)
        for (int r = 0; r < R; ++r) tt[(size_t)s * R + r] = host_pymod(sig[s].shifts[r], n);
    RC(taus.alloc(tt.size() * 8, st, "dsfft batch shifts"));
    CK(cudaMemcpyAsync(taus.p, tt.data(), tt.size() * 8, cudaMemcpyHostToDevice, st));
  }
  // initial layer and the first expansions, from the counts (dsfft.py:258-264)
  for (int64_t s = 0; s < S; ++s) {
    BatchSig& g = sig[s];
    if (!g.on) continue;
    if (was_fused[s]) {
      std::memcpy(&g.normY, hb.data() + onorm + (size_t)s * 8, 8);
    } else {
      double sum = 0.0;
      for (int q = 0; q < nparts; ++q)
        sum += reinterpret_cast<const double*>(hb.data() + opart)[(size_t)s * nparts + q];
      g.normY = sum / (double)n;
    }
    g.depth = d0;
    g.m = count_at(s, d0);
    if (g.m > cap) {
      g.on = false, g.fallback = true;
      continue;
    }
    g.add(1, d0, g.m, -1);
    while ((double)g.m < prm[s].theta * k && g.depth < max_depth) {
      const int next = g.depth + 1;
      if (2 * g.m <= next || count_at(s, next) > cap) {  // selective / overflow: alone
        g.on = false, g.fallback = true;
        break;
      }
      g.m = count_at(s, next);
      g.depth = next;
      g.add(2, next, g.m, -1);
    }
    g.mode = 0;  // first classify at the stop layer
  }
  // classify steps: all signals at the smallest pending depth together, each with its
  // probe list (afft_dsfft's classify_layer: the active children of the multi-tons it
  // found one layer up, or the stop layer's first probe0 buckets) or its whole layer
  DBuf idx, sidx, rows, ws, gates;
  for (;;) {
    int depth = INT32_MAX;
    for (auto& g : sig)
      if (g.on) depth = std::min(depth, g.depth);
    if (depth == INT32_MAX) break;
    const int64_t b = 1LL << depth, L = n / b;
    struct Mem {
      int64_t s, off, cnt;
      bool probe, alias;
    };
    std::vector<Mem> mem;
    std::vector<double> t0s((size_t)S, 0.0), t1s((size_t)S, 0.0);
    std::vector<std::vector<int64_t>> cand_of((size_t)S);
    for (int64_t s = 0; s < S; ++s) {
      BatchSig& g = sig[s];
      if (!g.on || g.depth != depth) continue;
      const double base = prm[s].noise_std / std::sqrt((double)b) * std::sqrt((double)R);
      // the floor 1e-8 sqrt(max energy) is provably below 1.5 base (see classify)
      if (!(1e-8 * std::sqrt((double)R * (double)L * g.normY * 1.0001) < 1.5 * base)) {
        g.on = false, g.fallback = true;
        continue;
      }
      t0s[s] = 1.5 * base;
      t1s[s] = 2.5 * base;
      int64_t m = 0;
      const int32_t* act = host_list(s, depth, &m);
      std::vector<int64_t>& cand = cand_of[s];
      bool probe = false;
      if (g.lazy && depth < max_depth && g.mode != 2 && m > 0) {
        if (g.mode == 0) {
          cand.assign(act, act + std::min<int64_t>(m, probe0));
        } else {
          const int64_t half = 1LL << (depth - 1);
          for (int pass = 0; pass < 2; ++pass)
            for (int64_t i : g.multi) {
              const int64_t cb = i + (pass ? half : 0);
              if (std::binary_search(act, act + m, (int32_t)cb)) cand.push_back(cb);
            }
        }
        probe = !cand.empty() && (int64_t)cand.size() < m;
      }
      if (!probe) cand.assign(act, act + m);
      // the row source afft_dsfft's rows() picks for this list (alias_rows_ok)
      const int64_t cnt = (int64_t)cand.size();
      const bool alias = L <= 256 || (L <= kAliasCtaMaxL && cnt * L <= (int64_t(1) << 19));
      mem.push_back({s, 0, cnt, probe, alias});
    }
    PMARK("b step lists");
    if (mem.empty()) continue;
    // members with alias rows first, so the coset-DFT members are one contiguous range
    std::stable_sort(mem.begin(), mem.end(),
                     [](const Mem& a, const Mem& b2) { return a.alias && !b2.alias; });
    int64_t A = 0;
    for (auto& q : mem) {
      q.off = A;
      A += q.cnt;
    }
    std::vector<int64_t> h_idx((size_t)A);
    std::vector<int32_t> h_sig((size_t)A);
    int64_t A_alias = 0;
    for (auto& q : mem) {
      std::copy(cand_of[q.s].begin(), cand_of[q.s].end(), h_idx.begin() + q.off);
      std::fill(h_sig.begin() + q.off, h_sig.begin() + q.off + q.cnt, (int32_t)q.s);
      if (q.alias) A_alias = q.off + q.cnt;
    }
    DBuf pk;  // state [A] | f0 [A] | val [A]: one read-back per step
    const size_t of0 = ((size_t)A + 7) & ~size_t(7), oval = of0 + (size_t)A * 8;
    std::vector<char> hpk;
    if (A > 0) {
      RC(idx.alloc((size_t)A * 8, st, "dsfft batch rows index"));
      RC(sidx.alloc((size_t)A * 4, st, "dsfft batch rows signal"));
      CK(cudaMemcpyAsync(idx.p, h_idx.data(), (size_t)A * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(sidx.p, h_sig.data(), (size_t)A * 4, cudaMemcpyHostToDevice, st));
      RC(rows.alloc((size_t)A * R * 16, st, "dsfft batch rows"));
      if (L <= 256) {
        RC(alias_rows_multi(Y.as<double>(), n, b, taus.as<int64_t>(), R, idx.as<int64_t>(),
                            sidx.as<int32_t>(), A, rows.as<double>(), st));
      } else {
        if (A_alias > 0)  // short (probe) lists at shallow layers: one CTA per row
          RC(alias_rows_cta_multi(Y.as<double>(), n, b, taus.as<int64_t>(), R, idx.as<int64_t>(),
                                  sidx.as<int32_t>(), A_alias, rows.as<double>(), st));
        if (A > A_alias) {
          // whole shallow layers: each member's distinct-residue coset DFTs (tau mod L)
          // over its own signal in one batched transform, then the rows picked and rotated
          std::vector<std::vector<int64_t>> res(S);
          std::vector<int32_t> coset((size_t)S * R, 0);
          std::vector<int64_t> qrot((size_t)S * R, 0);
          int U = 1;
          for (auto& q : mem) {
            if (q.alias) continue;
            const int64_t s2 = q.s;
            std::map<int64_t, int> seen;
            for (int t = 0; t < R; ++t) {
              const int64_t tm = host_pymod(sig[s2].shifts[t], n), r = tm % L;
              auto it = seen.find(r);
              int u;
              if (it == seen.end()) {
                u = (int)res[s2].size();
                seen[r] = u;
                res[s2].push_back(r);
              } else {
                u = it->second;
              }
              coset[(size_t)s2 * R + t] = u;
              qrot[(size_t)s2 * R + t] = tm / L;
            }
            U = std::max(U, (int)res[s2].size());
          }
          // every signal of the batch gets U residues (non-members / padding repeat one)
          std::vector<int64_t> table((size_t)S * U, 0);
          for (int64_t s2 = 0; s2 < S; ++s2)
            for (int u = 0; u < U; ++u)
              table[(size_t)s2 * U + u] =
                  res[s2].empty() ? 0 : res[s2][std::min<size_t>((size_t)u, res[s2].size() - 1)];
          DBuf dtab, dcos, dq, cosets;
          RC(dtab.alloc(table.size() * 8, st, "dsfft batch residues"));
          RC(dcos.alloc(coset.size() * 4, st, "dsfft batch coset map"));
          RC(dq.alloc(qrot.size() * 8, st, "dsfft batch rotations"));
          CK(cudaMemcpyAsync(dtab.p, table.data(), table.size() * 8, cudaMemcpyHostToDevice, st));
          CK(cudaMemcpyAsync(dcos.p, coset.data(), coset.size() * 4, cudaMemcpyHostToDevice, st));
          CK(cudaMemcpyAsync(dq.p, qrot.data(), qrot.size() * 8, cudaMemcpyHostToDevice, st));
          RC(cosets.alloc((size_t)S * U * b * 16, st, "dsfft batch coset DFTs"));
          RC(afft_bucketize_table(x, dtype, n, S, ld, b, dtab.as<int64_t>(), U,
                                  cosets.as<double>(), (int64_t)U * b, b, 1, st));
          RC(rows_gather_multi(cosets.as<double>(), b, U, R, dcos.as<int32_t>(), dq.as<int64_t>(),
                               idx.as<int64_t>() + A_alias, sidx.as<int32_t>() + A_alias,
                               A - A_alias, rows.as<double>() + 2 * A_alias * R, st));
        }
      }
      std::vector<double> gt((size_t)2 * S);
      for (int64_t s2 = 0; s2 < S; ++s2) {
        gt[s2] = t0s[s2];
        gt[S + s2] = t1s[s2];
      }
      RC(gates.alloc(gt.size() * 8, st, "dsfft batch gates"));
      CK(cudaMemcpyAsync(gates.p, gt.data(), gt.size() * 8, cudaMemcpyHostToDevice, st));
      RC(pk.alloc(oval + (size_t)A * 16, st, "dsfft batch results"));
      DBuf rn;
      RC(rn.alloc((size_t)A * 8, st, "dsfft batch resnorm"));
      const size_t need = afft_singleton_workspace_size(n, A, b, c, mm);
      RC(ws.alloc(need, st, "dsfft batch search workspace"));
      RC(classify_noisy_multi(rows.as<double>(), idx.as<int64_t>(), sidx.as<int32_t>(), A, b, n,
                              taus.as<int64_t>(), c, mm, prm[mem[0].s].weights,
                              gates.as<double>(), gates.as<double>() + S, pk.as<int8_t>(),
                              reinterpret_cast<int64_t*>(pk.as<char>() + of0),
                              reinterpret_cast<double*>(pk.as<char>() + oval), rn.as<double>(),
                              ws.p, need, st));
      PMARK("b step enqueue");
      RC(d2h(hpk, pk.p, oval + (size_t)A * 16, st));
      PMARK("b step read-back");
    }
    const int8_t* hs = reinterpret_cast<const int8_t*>(hpk.data());
    const int64_t* hf = reinterpret_cast<const int64_t*>(hpk.data() + of0);
    const cd* hv = reinterpret_cast<const cd*>(hpk.data() + oval);
    // trace and loop control per member, as afft_dsfft's classify_layer / run
    for (auto& q : mem) {
      BatchSig& g = sig[q.s];
      int64_t ns = 0;
      std::vector<int64_t> multis;
      for (int64_t i = q.off; i < q.off + q.cnt; ++i) {
        if (hs[i] == AFFT_SINGLE_TON) ++ns;
        else if (hs[i] == AFFT_MULTI_TON) multis.push_back(h_idx[i]);
      }
      if (q.probe) {
        if (multis.empty()) {  // no multi-ton among the probes: the whole layer next step
          g.mode = 2;
          continue;
        }
        g.add(5, depth, R, 1);
        g.add(3, depth, -1, (int64_t)multis.size());
      } else {
        g.add(5, depth, R, 1);
        g.add(3, depth, ns, (int64_t)multis.size());
      }
      g.multi.swap(multis);
      if (!g.multi.empty() && g.depth < max_depth) {  // re-expand (dsfft.py:190-192)
        const int next = g.depth + 1;
        if (2 * g.m <= next || count_at(q.s, next) > cap) {
          g.on = false, g.fallback = true;
          continue;
        }
        g.m = count_at(q.s, next);
        g.depth = next;
        g.mode = 1;
        g.add(2, next, g.m, -1);
      } else {
        g.on = false;
        if (!g.multi.empty() && (int64_t)k - ns > 0) {
          g.fallback = true;  // leftover multitons: _resolve_aliased, alone
        } else {
          // the entries of the last classify, ascending bucket order (a full layer); the
          // keys are distinct (f0 mod b is the bucket), so no dict look-ups are needed
          g.E.f.clear();
          g.E.v.clear();
          g.E.f.reserve((size_t)ns);
          g.E.v.reserve((size_t)ns);
          for (int64_t i = q.off; i < q.off + q.cnt; ++i)
            if (hs[i] == AFFT_SINGLE_TON) {
              g.E.f.push_back(hf[i]);
              g.E.v.push_back(hv[i]);
            }
        }
      }
    }
    PMARK("b step results");
  }
  return AFFT_OK;
}

}  // namespace
}  // namespace afft

using namespace afft;

extern "C" int afft_truncate_host(const int64_t* pos, const double* val, int64_t count, int32_t k,
                                  int64_t* out_pos, double* out_val, int64_t* out_count) {
  if (count < 0 || k < 0 || !out_count || (count > 0 && (!pos || !val)) ||
      (k > 0 && count > 0 && (!out_pos || !out_val))) {
    set_error("afft_truncate_host: bad arguments");
    return AFFT_EINVAL;
  }
  const int64_t m = std::min<int64_t>(count, k);
  std::vector<double> mag((size_t)count);
  for (int64_t i = 0; i < count; ++i) mag[i] = std::hypot(val[2 * i], val[2 * i + 1]);
  std::vector<int64_t> ord((size_t)count);
  for (int64_t i = 0; i < count; ++i) ord[i] = i;
  // key (-|v|, f): larger magnitude first, then the smaller position (the positions
  // are distinct, so the order is total and the result deterministic)
  auto before = [&](int64_t a, int64_t b) {
    return mag[a] != mag[b] ? mag[a] > mag[b] : pos[a] < pos[b];
  };
  if (m < count) std::nth_element(ord.begin(), ord.begin() + m, ord.end(), before);
  std::sort(ord.begin(), ord.begin() + m, before);
  for (int64_t i = 0; i < m; ++i) {
    out_pos[i] = pos[ord[i]];
    out_val[2 * i] = val[2 * ord[i]];
    out_val[2 * i + 1] = val[2 * ord[i] + 1];
  }
  *out_count = m;
  return AFFT_OK;
}

extern "C" int afft_dsfft(const void* x, int dtype, int64_t n, int32_t k,
                          const AfftDsfftParams* params, int64_t* out_pos, double* out_val,
                          int64_t capacity, int64_t* out_count, int32_t* trace,
                          int32_t trace_capacity, int32_t* trace_len, void* stream) {
  if (!x || !params || !out_count || n < 1 || (n & (n - 1)) || k < 1 ||
      (dtype != AFFT_C64 && dtype != AFFT_C128) ||
      (params->mode != 0 && (params->c < 1 || params->m < 2 || !params->anchors ||
                             !params->weights)) ||
      !params->dt_shift_off || (capacity > 0 && (!out_pos || !out_val))) {
    set_error("afft_dsfft: bad arguments");
    return AFFT_EINVAL;
  }
  Entries E;
  // the layer loop's temporaries come from a per-thread arena (capi.cu): the spectrum,
  // two signal-sized DFT buffers and the per-layer blocks fit in 3 n complex128 + 64 MB
  arena_begin((size_t)n * 48 + ((size_t)64 << 20), (cudaStream_t)stream);
  struct ArenaGuard {
    cudaStream_t st;
    ~ArenaGuard() {  // an early error return may leave work queued on the arena
      cudaStreamSynchronize(st);
      arena_end();
    }
  } arena_guard{(cudaStream_t)stream};
  Dsfft D{x, dtype, n, k, *params, (cudaStream_t)stream, Tracer{trace, trace_capacity}};
  g_prof.wait_s = 0.0;
  g_prof.syncs = 0;
  const double t0 = g_prof.on ? now_s() : 0.0;
  g_marks.acc.clear();
  g_marks.last = t0;
  g_marks.last_wait = 0.0;
  const int rc = D.run(E);
  if (g_prof.on)
    std::fprintf(stderr, "afft_dsfft: %.3f ms total, %.3f ms waiting in %d read-backs\n",
                 (now_s() - t0) * 1e3, g_prof.wait_s * 1e3, g_prof.syncs);
  if (g_prof.on)
    for (auto& a : g_marks.acc)
      std::fprintf(stderr, "  %-22s x%-3d %.3f ms, host %.3f ms\n", a.what, a.n, a.total * 1e3,
                   (a.total - a.wait) * 1e3);
  const std::vector<int64_t>& ef = E.f;
  const std::vector<cd>& ev = E.v;
  if (trace_len) *trace_len = D.tr.len;
  if (rc) return rc;
  *out_count = (int64_t)ef.size();
  if ((int64_t)ef.size() > capacity) {
    set_error("afft_dsfft: %zu entries, capacity %lld", ef.size(), (long long)capacity);
    return AFFT_ENOMEM;
  }
  for (size_t i = 0; i < ef.size(); ++i) {
    out_pos[i] = ef[i];
    out_val[2 * i] = ev[i].re;
    out_val[2 * i + 1] = ev[i].im;
  }
  return AFFT_OK;
}

extern "C" int afft_dsfft_batch(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                                int32_t k, const AfftDsfftParams* params, int64_t* out_pos,
                                double* out_val, int64_t capacity, int64_t* out_count,
                                int32_t* trace, int32_t trace_capacity, int32_t* trace_len,
                                int32_t* fallback, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!x || !params || !out_count || !fallback || n < 1 || k < 1 || batch < 0 || ld < n ||
      (dtype != AFFT_C64 && dtype != AFFT_C128) || (capacity > 0 && (!out_pos || !out_val))) {
    set_error("afft_dsfft_batch: bad arguments");
    return AFFT_EINVAL;
  }
  // the batch's temporaries from one borrowed device buffer (capi.cu arena): the
  // spectra S n complex128, coset DFTs up to S 72 n / 2^13 complex128 at the shallow
  // layers, rows and lists; repeated calls reuse it instead of growing the pool
  arena_begin((size_t)batch * n * 16 * 2 + ((size_t)512 << 20), (cudaStream_t)stream);
  struct ArenaGuard {
    cudaStream_t st;
    ~ArenaGuard() {
      cudaStreamSynchronize(st);
      arena_end();
    }
  } arena_guard{(cudaStream_t)stream};
  std::vector<BatchSig> sig;
  g_prof.wait_s = 0.0;
  g_prof.syncs = 0;
  const double t_start = g_prof.on ? now_s() : 0.0;
  g_marks.acc.clear();
  g_marks.last = t_start;
  g_marks.last_wait = 0.0;
  const int rc = dsfft_batch_run(x, dtype, n, batch, ld, k, params, sig, (cudaStream_t)stream);
  if (g_prof.on) {
    std::fprintf(stderr, "afft_dsfft_batch: %lld signals, %.3f ms total, %.3f ms waiting in %d "
                 "read-backs\n", (long long)batch, (now_s() - t_start) * 1e3, g_prof.wait_s * 1e3,
                 g_prof.syncs);
    for (auto& a : g_marks.acc)
      std::fprintf(stderr, "  %-22s x%-3d %.3f ms, host %.3f ms\n", a.what, a.n, a.total * 1e3,
                   (a.total - a.wait) * 1e3);
  }
  if (rc) {
    cudaStreamSynchronize((cudaStream_t)stream);
    return rc;
  }
  int over = AFFT_OK;
  for (int64_t s = 0; s < batch; ++s) {
    const BatchSig& g = sig[s];
    fallback[s] = g.fallback ? 1 : 0;
    out_count[s] = g.fallback ? 0 : (int64_t)g.E.f.size();
    const int32_t tl = (int32_t)(g.trace.size() / 4);
    if (trace_len) trace_len[s] = g.fallback ? 0 : tl;
    if (g.fallback) continue;
    if ((int64_t)g.E.f.size() > capacity) {
      over = AFFT_ENOMEM;
      continue;
    }
    for (size_t i = 0; i < g.E.f.size(); ++i) {
      out_pos[s * capacity + (int64_t)i] = g.E.f[i];
      out_val[2 * (s * capacity + (int64_t)i)] = g.E.v[i].re;
      out_val[2 * (s * capacity + (int64_t)i) + 1] = g.E.v[i].im;
    }
    if (trace)
      for (int32_t q = 0; q < std::min(tl, trace_capacity) * 4; ++q)
        trace[(int64_t)s * trace_capacity * 4 + q] = g.trace[q];
  }
  if (over) set_error("afft_dsfft_batch: entries beyond capacity %lld", (long long)capacity);
  return over;
}
