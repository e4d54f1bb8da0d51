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
#include <cstring>
#include <vector>

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
// Four-step DFT for large bucket counts, b = b1 * b2 (both <= 4096):
//   j = j1 + b1*j2, i = i2 + b2*i1
//   y[i2 + b2*i1] = (1/b) sum_j1 w_b1^{j1*i1} * [ w_b^{j1*i2} * sum_j2 x[(j*L - tau) mod n] w_b2^{j2*i2} ]
// Pass A: for each (shift, j1) gather the b2 samples at stride b1*L, size-b2 DFT,
//         twiddle w_b^{j1*i2} (index reduced mod b, sincospi), write z[t][j1][i2].
// Pass B: for each (shift, block of i2) read z[t][0..b1)[i2..], size-b1 DFT,
//         scale 1/b, write the caller-strided output.
struct FourStepParams {
  const void* x;
  int dtype;
  int64_t n, ld, b, b1, b2;
  int nshift;
  int64_t batch;
  int cj;       // j1 values per tile in pass A
  int wi;       // i2 columns per tile in pass B
  int lgb2;     // log2(b2) if a power of two, else -1 (index splits by shift)
  int lgb1;
  DftPlan plan1, plan2;
  double* z;    // [batch][nshift][b1][b2]
  double* out;
  int64_t out_offset, out_signal_stride, out_shift_stride, out_bin_stride;
  const int64_t* shift_table;
  const cd* tlo;  // w_b^r for r < 4096
  const cd* thi;  // w_b^(4096 q)
  int64_t tau[AFFT_MAX_SHIFTS];
};

constexpr int kTwLoBits = 12;

// w_b^r = w_b^(4096 q) * w_b^(r mod 4096): two table entries (L2/L1 resident, 64 KB
// each at most) and one complex product instead of a float64 sincospi per element.
__global__ void fourstep_tables_kernel(int64_t b, cd* __restrict__ tlo, int nlo,
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

__device__ __forceinline__ cd tw_b(const cd* tlo, const cd* thi, int64_t r) {
  const cd lo = tlo[r & ((1 << kTwLoBits) - 1)];
  return (r >> kTwLoBits) ? cmul(thi[r >> kTwLoBits], lo) : lo;
}

// Pass A, persistent over tiles (signal, shift, chunk of cj j1 values); the size-b2
// twiddle table is built once per CTA.
__global__ void __launch_bounds__(1024) fourstep_a_kernel(const __grid_constant__ FourStepParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b2 = (int)p.b2;
  cd* tw = reinterpret_cast<cd*>(smem_raw);
  cd* bufA = tw + b2;
  cd* bufB = bufA + (size_t)p.cj * b2;
  build_twiddles(tw, b2, threadIdx.x, blockDim.x);
  const int64_t nchunks = (p.b1 + p.cj - 1) / p.cj;
  const int64_t ntiles = p.batch * p.nshift * nchunks;
  const int64_t L = p.n / p.b;
  const int64_t stride = p.b1 * L;
  const int64_t esz = p.dtype == AFFT_C64 ? 8 : 16;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t chunk = tile % nchunks;
    const int64_t st_ = tile / nchunks;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t j1_0 = chunk * p.cj;
    const int cnt = (int)min((int64_t)p.cj, p.b1 - j1_0);
    const char* xs = reinterpret_cast<const char*>(p.x) + s * p.ld * esz;
    const int64_t tau = p.shift_table ? pymod(p.shift_table[s * p.nshift + t], p.n) : p.tau[t];
    const int total = cnt * b2;
    __syncthreads();  // tw ready / previous tile's buffers consumed
    // consecutive threads take consecutive j1 (addresses L apart) within a row j2
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int j2 = e / cnt;
      const int q = e - j2 * cnt;
      int64_t idx = (j1_0 + q) * L + (int64_t)j2 * stride - tau;
      if (idx < 0) idx += p.n;
      bufA[q * b2 + j2] = load_sample(xs, p.dtype, idx);
    }
    __syncthreads();
    const cd* spec = smem_dft(bufA, bufB, cnt, p.plan2, tw, threadIdx.x, blockDim.x);
    cd* z = reinterpret_cast<cd*>(p.z) + ((s * p.nshift + t) * p.b1 + j1_0) * p.b2;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int q = p.lgb2 >= 0 ? e >> p.lgb2 : e / b2;
      const int i2 = e - q * b2;
      z[e] = cmul(spec[e], tw_b(p.tlo, p.thi, (j1_0 + q) * i2));  // j1*i2 < b: no reduction
    }
  }
}

// Pass B, persistent over tiles (signal, shift, block of wi i2 columns).
__global__ void __launch_bounds__(1024) fourstep_b_kernel(const __grid_constant__ FourStepParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b1 = (int)p.b1;
  cd* tw = reinterpret_cast<cd*>(smem_raw);
  cd* bufA = tw + b1;
  cd* bufB = bufA + (size_t)p.wi * b1;
  build_twiddles(tw, b1, threadIdx.x, blockDim.x);
  const int64_t nchunks = (p.b2 + p.wi - 1) / p.wi;
  const int64_t ntiles = p.batch * p.nshift * nchunks;
  const double inv_b = 1.0 / (double)p.b;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t chunk = tile % nchunks;
    const int64_t st_ = tile / nchunks;
    const int t = (int)(st_ % p.nshift);
    const int64_t s = st_ / p.nshift;
    const int64_t i2_0 = chunk * p.wi;
    const int w = (int)min((int64_t)p.wi, p.b2 - i2_0);
    const cd* z = reinterpret_cast<const cd*>(p.z) + (s * p.nshift + t) * p.b1 * p.b2;
    const int total = w * b1;
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {  // coalesced along i2
      const int j1 = e / w;
      const int q = e - j1 * w;
      bufA[q * b1 + j1] = z[(int64_t)j1 * p.b2 + i2_0 + q];
    }
    __syncthreads();
    const cd* spec = smem_dft(bufA, bufB, w, p.plan1, tw, threadIdx.x, blockDim.x);
    double* out = p.out + 2 * (s * p.out_signal_stride + p.out_offset + t * p.out_shift_stride);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {  // consecutive i2 per i1
      const int i1 = e / w;
      const int q = e - i1 * w;
      const cd v = cscale(spec[q * b1 + i1], inv_b);
      const int64_t o = 2 * ((i2_0 + q + p.b2 * (int64_t)i1) * p.out_bin_stride);
      out[o] = v.re;
      out[o + 1] = v.im;
    }
  }
}

// b = b1 * b2 with both factors <= limit, as balanced as possible; false if none.
static bool split_size(int64_t b, int64_t limit, int64_t* b1, int64_t* b2) {
  int64_t best = 0;
  for (int64_t d = 1; d * d <= b; ++d) {
    if (b % d) continue;
    const int64_t e = b / d;
    if (d <= limit && e <= limit) best = d;  // d grows toward sqrt(b)
  }
  if (!best) return false;
  *b1 = b / best;  // the larger factor on the pass-B side
  *b2 = best;
  return true;
}

static int launch_fourstep(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                           int64_t b, const int64_t* shifts, int nshift, double* out,
                           int64_t out_offset, int64_t oss, int64_t osh, int64_t obin,
                           cudaStream_t stream, const int64_t* shift_table) {
  FourStepParams q;
  memset(&q, 0, sizeof(q));
  if (!split_size(b, AFFT_MAX_SMEM_DFT, &q.b1, &q.b2)) {
    set_error("bucket count %lld has no factorisation into two DFTs of size <= %d",
              (long long)b, AFFT_MAX_SMEM_DFT);
    return AFFT_EUNSUPPORTED;
  }
  if (!make_dft_plan(q.b1, &q.plan1) || !make_dft_plan(q.b2, &q.plan2)) {
    set_error("cannot plan DFTs of sizes %lld x %lld", (long long)q.b1, (long long)q.b2);
    return AFFT_EUNSUPPORTED;
  }
  q.x = x;
  q.dtype = dtype;
  q.n = n;
  q.ld = ld;
  q.b = b;
  q.nshift = nshift;
  q.out = out;
  q.out_offset = out_offset;
  q.out_signal_stride = oss;
  q.out_shift_stride = osh;
  q.out_bin_stride = obin;
  q.shift_table = shift_table;
  for (int t = 0; t < nshift; ++t) q.tau[t] = shifts ? host_pymod(shifts[t], n) : 0;
  const size_t kBudget = 96 * 1024;
  q.cj = (int)std::max<int64_t>(1, std::min<int64_t>(q.b1, ((int64_t)(kBudget / 16) - q.b2) / (2 * q.b2)));
  q.wi = (int)std::max<int64_t>(1, std::min<int64_t>(q.b2, ((int64_t)(kBudget / 16) - q.b1) / (2 * q.b1)));
  q.lgb2 = q.plan2.lgn;
  q.lgb1 = q.plan1.lgn;
  q.batch = batch;
  const size_t smemA = (size_t)(q.b2 + 2 * (int64_t)q.cj * q.b2) * 16;
  const size_t smemB = (size_t)(q.b1 + 2 * (int64_t)q.wi * q.b1) * 16;
  const int nlo = (int)std::min<int64_t>(b, 1 << kTwLoBits);
  const int nhi = (int)((b + (1 << kTwLoBits) - 1) >> kTwLoBits);
  const size_t zbytes = (size_t)batch * nshift * b * 16;
  const size_t tbytes = (size_t)(nlo + nhi) * 16;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&q.z), zbytes + tbytes, stream);
  if (e != cudaSuccess) return cuda_status(e, "scratch_alloc(four-step scratch)");
  cd* tlo = reinterpret_cast<cd*>(reinterpret_cast<char*>(q.z) + zbytes);
  cd* thi = tlo + nlo;
  q.tlo = tlo;
  q.thi = thi;
  e = cudaFuncSetAttribute(fourstep_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smemA);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fourstep_b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smemB);
  // large sub-DFTs run one CTA per SM: give it enough warps to hide smem latency
  const int ta = q.b2 >= 2048 ? 1024 : (q.b2 >= 512 ? 512 : 256);
  const int tb = q.b1 >= 2048 ? 1024 : (q.b1 >= 512 ? 512 : 256);
  int occA = 0, occB = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occA, fourstep_a_kernel, ta, smemA);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB, fourstep_b_kernel, tb, smemB);
  if (e != cudaSuccess || occA < 1 || occB < 1) {
    scratch_free(q.z, stream);
    return cuda_status(e != cudaSuccess ? e : cudaErrorInvalidConfiguration,
                       "four-step occupancy");
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  fourstep_tables_kernel<<<(unsigned)((std::max(nlo, nhi) + 255) / 256), 256, 0, stream>>>(
      b, tlo, nlo, thi, nhi);
  const int64_t tilesA = batch * nshift * ((q.b1 + q.cj - 1) / q.cj);
  const int64_t tilesB = batch * nshift * ((q.b2 + q.wi - 1) / q.wi);
  const unsigned ga = (unsigned)std::min<int64_t>(tilesA, (int64_t)sms * occA);
  const unsigned gb = (unsigned)std::min<int64_t>(tilesB, (int64_t)sms * occB);
  fourstep_a_kernel<<<ga, ta, smemA, stream>>>(q);
  fourstep_b_kernel<<<gb, tb, smemB, stream>>>(q);
  scratch_free(q.z, stream);
  AFFT_CHECK_LAUNCH("fourstep kernels");
  return AFFT_OK;
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
    if (b > AFFT_MAX_SMEM_DFT) {
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
  cudaError_t e = cudaFuncSetAttribute(gather_dft_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_max);
  if (e != cudaSuccess) {
    return cuda_status(e, "cudaFuncSetAttribute(gather_dft)");
  }
  dim3 grid((unsigned)batch, (unsigned)total_jobs);
  gather_dft_kernel<<<grid, 256, smem_max, stream>>>(q);
  AFFT_CHECK_LAUNCH("gather_dft_kernel");
  return AFFT_OK;
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
