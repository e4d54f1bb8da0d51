// Microbenchmark (diagnostic): read bandwidth of tiles made of R row segments of S
// contiguous bytes at a large row stride — the access shape of a K2' radix-R pass
// (R rows of kCnt points at stride n/R) — against a plain contiguous stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o seg_bw tools/seg_bw.cu && ./seg_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void seg_read(const double2* __restrict__ in, int64_t nvec, int rows, int seg_vec,
                         int64_t row_stride_vec, double* out) {
  // tile t: rows r < rows, each seg_vec 16-B vectors at in[(t * seg_vec) + r * row_stride]
  const int64_t tiles = nvec / ((int64_t)rows * seg_vec);
  double acc = 0.0;
  const int per_tile = rows * seg_vec;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t col0 = (t % (row_stride_vec / seg_vec)) * seg_vec;
    const int64_t blk = t / (row_stride_vec / seg_vec);
    const double2* base = in + blk * row_stride_vec * rows + col0;
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < per_tile) {
        const int r = e / seg_vec, c = e - r * seg_vec;
        v[k] = __ldcs(base + (int64_t)r * row_stride_vec + c);
      } else {
        v[k] = make_double2(0, 0);
      }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += v[k].x + v[k].y;
  }
  if (acc == 12345.0) *out = acc;
}

int main() {
  const int64_t bytes = (int64_t)1 << 28;  // 256 MB
  const int64_t nvec = bytes / 16;
  double2* in;
  double* out;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(in, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int threads = 128;  // 16 vectors per thread: 2048 vectors = 32 KB per tile
  for (int seg : {4, 8, 16, 32, 64, 2048}) {  // 16-B vectors per row segment
    const int rows = 2048 / seg;
    const int64_t stride = nvec / rows;  // rows spread over the whole buffer
    for (int occ : {3, 6, 12}) {
      const int grid = sms * occ;
      seg_read<<<grid, threads>>>(in, nvec, rows, seg, stride, out);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) seg_read<<<grid, threads>>>(in, nvec, rows, seg, stride, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("segment %5d B x %4d rows, %2d CTAs/SM: %7.1f GB/s\n", seg * 16, rows, occ,
             bytes * 10 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
