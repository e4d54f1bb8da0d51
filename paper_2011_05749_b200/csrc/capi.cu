// Error plumbing and version for the C ABI (include/aliasfft_b200.h).
#include <cstring>
#include <map>
#include <mutex>

#include "afft_common.cuh"

namespace afft {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return e == cudaErrorMemoryAllocation ? AFFT_ENOMEM : AFFT_ECUDA;
}

// Stream-ordered scratch from a library-owned pool per device.  The default pool's
// release threshold is 0, which hands memory back at every synchronisation and
// re-maps it on the next allocation; this pool keeps it (threshold = max).
static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64] = {};

static cudaMemPool_t library_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    g_pools[dev] = pool;
  }
  return g_pools[dev];
}

static std::mutex g_pin_mu;
static std::multimap<size_t, void*> g_pin_free;  // capacity -> buffer

void* pinned_acquire(size_t bytes, size_t* capacity) {
  {
    std::lock_guard<std::mutex> lock(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end()) {
      void* p = it->second;
      *capacity = it->first;
      g_pin_free.erase(it);
      return p;
    }
  }
  size_t cap = 4096;
  while (cap < bytes) cap <<= 1;
  void* p = nullptr;
  if (cudaMallocHost(&p, cap) != cudaSuccess) return nullptr;
  *capacity = cap;
  return p;
}

void pinned_release(void* p, size_t capacity) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pin_mu);
  g_pin_free.emplace(capacity, p);
}

cudaError_t ensure_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = granted[{dev, func}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t stream) {
  cudaMemPool_t pool = library_pool();
  if (!pool) return cudaMallocAsync(p, bytes, stream);
  return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

cudaError_t scratch_free(void* p, cudaStream_t stream) { return cudaFreeAsync(p, stream); }

}  // namespace afft

extern "C" const char* afft_last_error(void) { return afft::g_err; }
extern "C" int afft_version(void) { return 1; }
