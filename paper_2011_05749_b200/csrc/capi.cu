// Error plumbing and version for the C ABI (include/aliasfft_b200.h).
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

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

// Per-thread scratch arena for one long call on one stream (the DSFFT layer loop):
// a stack of blocks carved from one device buffer, so that the ~2 pool calls per
// temporary (hundreds per decode) become pointer arithmetic.  Blocks are freed in any
// order; the stack top drops past every freed block at the top.  Requests on another
// stream, or that do not fit, go to the pool as usual.  Stream order makes reuse safe:
// every block is used on the arena's stream only, and the caller synchronises that
// stream before the arena is released (afft_dsfft ends with a read-back).  The buffer
// itself is borrowed from a process-wide free list per device for the duration of the
// call and returned by arena_end, so no thread keeps device memory after its call and a
// thread that moves to another device never reuses the first device's buffer.
struct Arena {
  char* base = nullptr;
  size_t cap = 0, top = 0;
  int dev = -1;
  cudaStream_t st = nullptr;
  bool active = false;
  std::vector<size_t> start, end;
  std::vector<char> freed;
};
static thread_local Arena g_arena;
static std::mutex g_arena_mu;
static std::multimap<size_t, char*> g_arena_free[64];  // per device: capacity -> buffer

static cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t stream) {
  cudaMemPool_t pool = library_pool();
  if (!pool) return cudaMallocAsync(p, bytes, stream);
  return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

cudaError_t arena_begin(size_t bytes, cudaStream_t stream) {
  Arena& A = g_arena;
  if (A.active) return cudaSuccess;  // nested: the outer scope owns it
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return cudaSuccess;  // no arena: every request goes to the pool
  }
  {
    std::lock_guard<std::mutex> lock(g_arena_mu);
    auto& fl = g_arena_free[dev];
    auto it = fl.lower_bound(bytes);
    if (it != fl.end()) {
      A.base = it->second;
      A.cap = it->first;
      fl.erase(it);
    } else if (!fl.empty()) {
      // every cached buffer is too small: drop the largest (idle: its last user
      // synchronised its stream before releasing it) to make room for a bigger one
      auto last = std::prev(fl.end());
      cudaFreeAsync(last->second, stream);
      fl.erase(last);
    }
  }
  if (!A.base) {
    void* p = nullptr;
    const cudaError_t e = pool_alloc(&p, bytes, stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cudaSuccess;
    }
    A.base = static_cast<char*>(p);
    A.cap = bytes;
  }
  A.dev = dev;
  A.st = stream;
  A.top = 0;
  A.active = true;
  return cudaSuccess;
}

void arena_end() {
  Arena& A = g_arena;
  if (A.base) {
    std::lock_guard<std::mutex> lock(g_arena_mu);
    g_arena_free[A.dev].emplace(A.cap, A.base);
  }
  A.base = nullptr;
  A.cap = 0;
  A.dev = -1;
  A.active = false;
  A.top = 0;
  A.start.clear();
  A.end.clear();
  A.freed.clear();
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t stream) {
  Arena& A = g_arena;
  if (A.active && A.base && stream == A.st) {
    const size_t off = (A.top + 255) & ~size_t(255);
    if (off + bytes <= A.cap) {
      A.start.push_back(off);
      A.end.push_back(off + bytes);
      A.freed.push_back(0);
      A.top = off + bytes;
      *p = A.base + off;
      return cudaSuccess;
    }
  }
  return pool_alloc(p, bytes, stream);
}

cudaError_t scratch_free(void* p, cudaStream_t stream) {
  Arena& A = g_arena;
  char* c = static_cast<char*>(p);
  if (A.base && c >= A.base && c < A.base + A.cap) {
    const size_t off = (size_t)(c - A.base);
    for (size_t i = A.start.size(); i-- > 0;)
      if (A.start[i] == off && !A.freed[i]) {
        A.freed[i] = 1;
        break;
      }
    while (!A.start.empty() && A.freed.back()) {
      A.top = A.start.back();
      A.start.pop_back();
      A.end.pop_back();
      A.freed.pop_back();
    }
    if (A.start.empty()) A.top = 0;
    return cudaSuccess;
  }
  return cudaFreeAsync(p, stream);
}

}  // namespace afft

extern "C" const char* afft_last_error(void) { return afft::g_err; }
extern "C" int afft_version(void) { return 1; }
