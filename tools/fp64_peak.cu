// FP64 pipe peak on this GPU (diagnostic, not part of the library): independent
// DFMA chains per thread, whole-GPU grid, CUDA-event timed.  Prints one JSON line
// with DFMA TFLOP/s (2 flop each) and FP64 instructions/s, the denominators for
// the FP64 pipe fractions quoted in DESIGN.md (MEASURED_PEAKS.json has no FP64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 8192;

__global__ void dfma_kernel(double* out, double a, double b) {
  double v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fma(v[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8;
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double inst = (double)blocks * threads * kChains * kIters * reps;
  const double s = ms * 1e-3;
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_inst_per_s\": %.4e, \"sms\": %d, \"ms\": %.3f}\n",
         2.0 * inst / s / 1e12, inst / s, sms, ms / reps);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
