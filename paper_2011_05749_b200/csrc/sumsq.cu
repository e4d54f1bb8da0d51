// K1's fused |x|^2 stream: the full-signal 2-norm behind exact_thresholds
// (peeling.py:316-318).  For FFAST this pass reads every sample of every signal
// and is the HBM-bound kernel of the whole path (16.78 MB/signal at
// config 5 against 22.5 KB of gathered sectors).
//
// Each CTA streams one fixed 64 KiB part of one signal with 16-byte loads, 8
// independent loads in flight per thread, accumulating in float64 (the
// reference upcasts to complex128 before np.linalg.norm).  Parts are written as
// fixed-order partials so the final sum, done by afft_exact_thresholds in part
// order, is deterministic run to run.
#include <cstdlib>

#include "afft_common.cuh"

namespace afft {

constexpr int kSumsqThreads = 256;
constexpr int64_t kPartBytes = 64 * 1024;
constexpr int kUnroll = 8;

// 16-byte streaming load that does not allocate in L1 (the decode CTAs running
// next to this kernel keep most of the SM's unified L1/shared storage).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ double sq4(float4 v) {
  double a = (double)v.x, b = (double)v.y, c = (double)v.z, d = (double)v.w;
  return __fma_rn(a, a, __fma_rn(b, b, __fma_rn(c, c, d * d)));
}
__device__ __forceinline__ double sq2(double2 v) { return __fma_rn(v.x, v.x, v.y * v.y); }

__global__ void __launch_bounds__(kSumsqThreads) sumsq_kernel(const void* __restrict__ x, int dtype,
                                                              int64_t n, int64_t ld, int nparts,
                                                              double* __restrict__ partials,
                                                              int use_na) {
  const int64_t s = blockIdx.y;
  const int part = blockIdx.x;
  const int esz = dtype == AFFT_C64 ? 8 : 16;
  const int64_t per_part = kPartBytes / esz;
  const int64_t e0 = (int64_t)part * per_part;
  const int64_t e1 = min(n, e0 + per_part);
  const char* row = reinterpret_cast<const char*>(x) + s * ld * esz;
  double acc0 = 0.0, acc1 = 0.0;

  // scalar head until 16-byte aligned (only possible for c64 rows)
  int64_t e = e0;
  if (dtype == AFFT_C64) {
    const float2* xs = reinterpret_cast<const float2*>(row);
    if ((reinterpret_cast<uintptr_t>(xs + e) & 15) && e < e1) {
      if (threadIdx.x == 0) {
        float2 v = __ldg(xs + e);
        acc0 += (double)v.x * v.x + (double)v.y * v.y;
      }
      ++e;
    }
    const int64_t nvec = (e1 - e) / 2;
    const float4* xv = reinterpret_cast<const float4*>(xs + e);
    int64_t i = threadIdx.x;
    for (; i + (kUnroll - 1) * kSumsqThreads < nvec; i += kUnroll * kSumsqThreads) {
      float4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = use_na ? ld_stream(xv + i + u * kSumsqThreads) : __ldcs(xv + i + u * kSumsqThreads);
#pragma unroll
      for (int u = 0; u < kUnroll; u += 2) {
        acc0 += sq4(v[u]);
        acc1 += sq4(v[u + 1]);
      }
    }
    for (; i < nvec; i += kSumsqThreads) acc0 += sq4(__ldcs(xv + i));
    const int64_t tail = e + 2 * nvec;
    if (tail < e1 && threadIdx.x == 0) {
      float2 v = __ldg(xs + tail);
      acc1 += (double)v.x * v.x + (double)v.y * v.y;
    }
  } else {
    const double2* xv = reinterpret_cast<const double2*>(row) + e0;
    const int64_t nvec = e1 - e0;
    int64_t i = threadIdx.x;
    for (; i + (kUnroll - 1) * kSumsqThreads < nvec; i += kUnroll * kSumsqThreads) {
      double2 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = use_na ? ld_stream(xv + i + u * kSumsqThreads) : __ldcs(xv + i + u * kSumsqThreads);
#pragma unroll
      for (int u = 0; u < kUnroll; u += 2) {
        acc0 += sq2(v[u]);
        acc1 += sq2(v[u + 1]);
      }
    }
    for (; i < nvec; i += kSumsqThreads) acc0 += sq2(__ldcs(xv + i));
  }
  double acc = acc0 + acc1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double warp_sums[kSumsqThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_sums[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kSumsqThreads / 32; ++w) t += warp_sums[w];
    partials[s * nparts + part] = t;
  }
}

__global__ void thresholds_kernel(const double* __restrict__ partials, int nparts, int64_t n,
                                  int64_t batch, double* __restrict__ eps) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  double t = 0.0;
  for (int p = 0; p < nparts; ++p) t += partials[s * nparts + p];
  // 1e-6 * float(np.linalg.norm(x)) / np.sqrt(len(x))
  eps[s] = (1e-6 * sqrt(t)) / sqrt((double)n);
}

}  // namespace afft

using namespace afft;

extern "C" int32_t afft_sumsq_parts(int64_t n, int dtype) {
  const int esz = dtype == AFFT_C64 ? 8 : 16;
  const int64_t per_part = kPartBytes / esz;
  return (int32_t)((n + per_part - 1) / per_part);
}

extern "C" int afft_sumsq(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                          double* partials, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!x || !partials || n < 1 || ld < n || batch < 0 ||
      (dtype != AFFT_C64 && dtype != AFFT_C128)) {
    set_error("afft_sumsq: bad arguments");
    return AFFT_EINVAL;
  }
  const int nparts = afft_sumsq_parts(n, dtype);
  const int esz = dtype == AFFT_C64 ? 8 : 16;
  for (int64_t s0 = 0; s0 < batch; s0 += 65535) {  // grid.y limit
    const int64_t cnt = batch - s0 < 65535 ? batch - s0 : 65535;
    dim3 grid((unsigned)nparts, (unsigned)cnt);
    static const int use_na = [] {
      const char* e = getenv("AFFT_STREAM_NO_ALLOCATE");
      return e ? atoi(e) : 1;
    }();
    sumsq_kernel<<<grid, kSumsqThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const char*>(x) + s0 * ld * esz, dtype, n, ld, nparts,
        partials + s0 * nparts, use_na);
    AFFT_CHECK_LAUNCH("sumsq_kernel");
  }
  return AFFT_OK;
}

extern "C" int afft_exact_thresholds(const double* partials, int32_t nparts, int64_t n,
                                     int64_t batch, double* eps, void* stream) {
  if (batch == 0) return AFFT_OK;
  if (!partials || !eps || nparts < 1 || n < 1) {
    set_error("afft_exact_thresholds: bad arguments");
    return AFFT_EINVAL;
  }
  const int threads = 128;
  thresholds_kernel<<<(unsigned)((batch + threads - 1) / threads), threads, 0,
                      (cudaStream_t)stream>>>(partials, nparts, n, batch, eps);
  AFFT_CHECK_LAUNCH("thresholds_kernel");
  return AFFT_OK;
}
