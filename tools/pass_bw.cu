// Microbenchmark (diagnostic): a K2'-pass-shaped COPY — per tile, 256 rows x 8 points of
// 16 B read at a 1 MB row stride and written back the same way, 128 threads x 16 points,
// persistent grids of 2-6 CTAs per SM, optional dummy FP64 work per point — against the
// pass itself (0.34 ms for 2^24 c128 = 3 x 512 MB).  Separates the memory shape from
// the compute phase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pass_bw tools/pass_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

// SR / SW: strided (256 rows x 8 points at the 1 MB row stride) or contiguous (the
// tile's 2048 points in a row) reads / writes.
template <int WORK, bool SR, bool SW>
__global__ void __launch_bounds__(128) pass_copy(const double2* __restrict__ in,
                                                 double2* __restrict__ out, int64_t nb,
                                                 int64_t tiles) {
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t j0 = t * 8;
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int w = threadIdx.x + k * 128;  // (jj, row) = (w & 7, w >> 3)
      v[k] = __ldcs(SR ? in + (j0 + (w & 7)) + (int64_t)(w >> 3) * nb : in + t * 2048 + w);
    }
#pragma unroll
    for (int r = 0; r < WORK; ++r)
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k].x = v[k].x * 1.0000001 + v[k].y;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int w = threadIdx.x + k * 128;
      __stcs(SW ? out + (j0 + (w & 7)) + (int64_t)(w >> 3) * nb : out + t * 2048 + w, v[k]);
    }
  }
}

template <int WORK, bool SR = true, bool SW = true>
void run(const double2* in, double2* out, int64_t n, int sms) {
  const int64_t nb = n / 256, tiles = n / 2048;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int occ : {2, 3, 4, 6}) {
    const int grid = sms * occ;
    pass_copy<WORK, SR, SW><<<grid, 128>>>(in, out, nb, tiles);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) pass_copy<WORK, SR, SW><<<grid, 128>>>(in, out, nb, tiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("reads %s writes %s work %3d  %d CTAs/SM: %.1f us per 2^24 c128 pass = %.0f GB/s (r+w)\n", SR ? "strided" : "contig ", SW ? "strided" : "contig ", WORK, occ,
           ms * 100.0, 2.0 * n * 16 * 10 / (ms * 1e-3) / 1e9);
  }
}

int main() {
  const int64_t n = 1 << 24;
  double2 *in, *out;
  cudaMalloc(&in, n * 16);
  cudaMalloc(&out, n * 16);
  cudaMemset(in, 0, n * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, true, true>(in, out, n, sms);
  run<0, false, false>(in, out, n, sms);
  run<0, true, false>(in, out, n, sms);
  run<0, false, true>(in, out, n, sms);
  return 0;
}
