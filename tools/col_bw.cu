// Microbenchmark (diagnostic): the access shape of a two-pass 4096 x 4096 transform —
// per tile C consecutive columns x 4096 rows (row stride 4096 points), 256 threads x 16
// points per column, read strided and written strided (the second pass: X[j + 4096 q])
// or contiguous (the first pass: column j's 4096 outputs in a row) — as a COPY, against
// the three-pass radix-256 form (tools/pass_bw.cu: ~113 us per 2^24 c128 pass).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o col_bw tools/col_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C, bool SW, typename T>
__global__ void __launch_bounds__(256) col_copy(const T* __restrict__ in, double2* __restrict__ out,
                                                int64_t tiles) {
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t j0 = t * C;
    // element e = (row, col) = (e / C, e % C): lanes along the row's C columns first
    T v[16 * C];
#pragma unroll
    for (int k = 0; k < 16 * C; ++k) {
      const int e = threadIdx.x + k * 256;
      v[k] = __ldcs(in + (j0 + e % C) + (int64_t)(e / C) * 4096);
    }
#pragma unroll
    for (int k = 0; k < 16 * C; ++k) {
      const int e = threadIdx.x + k * 256;
      double2 o;
      if constexpr (sizeof(T) == 8) {
        o = make_double2((double)reinterpret_cast<const float2&>(v[k]).x,
                         (double)reinterpret_cast<const float2&>(v[k]).y);
      } else {
        o = reinterpret_cast<const double2&>(v[k]);
      }
      const int row = e / C, col = e % C;
      __stcs(SW ? out + (j0 + col) + (int64_t)row * 4096 : out + (j0 + col) * 4096 + row, o);
    }
  }
}

template <int C, bool SW, typename T>
void run(const T* in, double2* out, int64_t n, int sms, const char* what) {
  const int64_t tiles = 4096 / C;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int occ : {1, 2, 3, 4}) {
    const int grid = sms * occ;
    col_copy<C, SW, T><<<grid, 256>>>(in, out, tiles);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) col_copy<C, SW, T><<<grid, 256>>>(in, out, tiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)n * (sizeof(T) + 16);
    printf("%s C=%d writes %s %d CTAs/SM: %.1f us per pass = %.0f GB/s (r+w)\n", what, C,
           SW ? "strided" : "contig ", occ, ms * 100.0, bytes * 10 / (ms * 1e-3) / 1e9);
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
  const float2* in32 = reinterpret_cast<const float2*>(in);
  run<1, false>(in32, out, n, sms, "c64 in ");
  run<2, false>(in32, out, n, sms, "c64 in ");
  run<1, true>(in, out, n, sms, "c128 in");
  run<2, true>(in, out, n, sms, "c128 in");
  run<1, false>(in, out, n, sms, "c128 in");
  return 0;
}
