// Error plumbing and version for the C ABI (include/aliasfft_b200.h).
#include <cstring>

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

}  // namespace afft

extern "C" const char* afft_last_error(void) { return afft::g_err; }
extern "C" int afft_version(void) { return 1; }
