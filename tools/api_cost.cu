// Host cost of the CUDA runtime calls the DSFFT layer loop issues (diagnostic):
// kernel launch, pool alloc/free, small memset / D2D copy, occupancy query, and a
// pageable vs pinned 8-byte read-back.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O2 tools/api_cost.cu -o /tmp/api_cost && /tmp/api_cost
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 1023) *p = 0;
}

struct Big {
  long long v[560];  // ~4.4 KB, like NoisyPlan / GStockParams
};
__global__ void big_kernel(const __grid_constant__ Big b, int* p) {
  if (p && threadIdx.x == 1023) *p = (int)b.v[threadIdx.x & 511];
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaMemPool_t pool;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = 0;
  cudaMemPoolCreate(&pool, &props);
  uint64_t keep = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  int* d = nullptr;
  cudaMalloc(&d, 1 << 20);
  const int N = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    double t = now_us();
    for (int i = 0; i < N; ++i) empty_kernel<<<4, 256, 0, st>>>(d);
    double launch = (now_us() - t) / N;
    cudaStreamSynchronize(st);
    Big big = {};
    t = now_us();
    for (int i = 0; i < N; ++i) big_kernel<<<4, 256, 0, st>>>(big, d);
    double launch_big = (now_us() - t) / N;
    cudaStreamSynchronize(st);
    printf("rep %d: launch with a 4.4 KB parameter %.2f us\n", rep, launch_big);
    t = now_us();
    for (int i = 0; i < N; ++i) {
      void* p;
      cudaMallocFromPoolAsync(&p, 4096 + (i & 7) * 1024, pool, st);
      cudaFreeAsync(p, st);
    }
    double alloc = (now_us() - t) / N;
    cudaStreamSynchronize(st);
    t = now_us();
    for (int i = 0; i < N; ++i) cudaMemsetAsync(d, 0, 64, st);
    double mset = (now_us() - t) / N;
    cudaStreamSynchronize(st);
    t = now_us();
    for (int i = 0; i < N; ++i) cudaMemcpyAsync(d + 1024, d, 64, cudaMemcpyDeviceToDevice, st);
    double d2d = (now_us() - t) / N;
    cudaStreamSynchronize(st);
    t = now_us();
    int occ;
    for (int i = 0; i < N; ++i)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, empty_kernel, 256, 1024);
    double occq = (now_us() - t) / N;
    int sms;
    t = now_us();
    for (int i = 0; i < N; ++i) {
      int dev;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    double attr = (now_us() - t) / N;
    double hpage[8];
    double* hpin;
    cudaMallocHost(&hpin, 64);
    t = now_us();
    for (int i = 0; i < 200; ++i) {
      cudaMemcpyAsync(hpage, d, 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
    double rb_page = (now_us() - t) / 200;
    t = now_us();
    for (int i = 0; i < 200; ++i) {
      cudaMemcpyAsync(hpin, d, 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
    double rb_pin = (now_us() - t) / 200;
    t = now_us();
    for (int i = 0; i < 200; ++i) {
      empty_kernel<<<4, 256, 0, st>>>(d);
      cudaStreamSynchronize(st);
    }
    double launch_sync = (now_us() - t) / 200;
    cudaFreeHost(hpin);
    printf("rep %d: launch %.2f us, pool alloc+free %.2f us, memset %.2f us, d2d %.2f us, "
           "occupancy %.2f us, getdevice+attr %.2f us, read-back pageable %.2f us, pinned %.2f "
           "us, launch+sync %.2f us\n",
           rep, launch, alloc, mset, d2d, occq, attr, rb_page, rb_pin, launch_sync);
  }
  return 0;
}
