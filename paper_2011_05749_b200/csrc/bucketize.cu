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
  const cd* res = gather_dft_block(xs, p.dtype, p.n, b, p.plan[c], taus, cnt, tw, bufA, bufB);
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
      set_error("bucket count %lld exceeds the one-CTA DFT limit %d", (long long)b,
                AFFT_MAX_SMEM_DFT);
      return AFFT_EUNSUPPORTED;
    }
    if (!make_dft_plan(b, &q.plan[c])) {
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
