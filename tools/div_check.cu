// Verifies, on the device, that the Markstein sequence with a precomputed
// reciprocal reproduces IEEE division bit for bit for the singleton search's
// target phases: tgt = RN(RN(-2 pi r) / n) for r in [0, n).
//   q0 = RN(x * inv), rem = fma(-q0, n, x) (exact), q = fma(rem, inv, q0)
// Diagnostic (not part of the library):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/div_check.cu -o div_check
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void check(long long n, long long start, long long count, long long stride,
                      unsigned long long* bad, long long* first_bad) {
  const double dn = (double)n, inv = 1.0 / dn;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = (start + i * stride) % n;
    const double x = __dmul_rn(-6.283185307179586, (double)r);
    const double ref = __ddiv_rn(x, dn);
    const double q0 = __dmul_rn(x, inv);
    const double rem = __fma_rn(-q0, dn, x);
    const double q = r ? __fma_rn(rem, inv, q0) : x;  // r = 0: keep x / n = -0.0
    if (__double_as_longlong(q) != __double_as_longlong(ref)) {
      atomicAdd(bad, 1ull);
      atomicMin((unsigned long long*)first_bad, (unsigned long long)r);
    }
  }
}

int main() {
  const long long sizes[] = {134217216LL, 4095LL, 2097024LL, 1LL << 24, 124950LL, 511LL * 512,
                             1LL << 22, 3000000000LL - 1};
  unsigned long long* bad;
  long long* fb;
  cudaMalloc(&bad, 8);
  cudaMalloc(&fb, 8);
  int fails = 0;
  for (long long n : sizes) {
    unsigned long long h = 0;
    long long f = 0x7fffffffffffffffLL;
    cudaMemcpy(bad, &h, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(fb, &f, 8, cudaMemcpyHostToDevice);
    // every r when n <= 2^28, else a strided sweep of 2^28 values (odd stride)
    const long long count = n <= (1LL << 28) ? n : (1LL << 28);
    const long long stride = n <= (1LL << 28) ? 1 : (n / count) | 1;
    check<<<148 * 16, 256>>>(n, 0, count, stride, bad, fb);
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&f, fb, 8, cudaMemcpyDeviceToHost);
    printf("n=%lld checked=%lld mismatches=%llu first=%lld\n", n, count, h, h ? f : -1);
    fails += h != 0;
  }
  return fails ? 1 : 0;
}
