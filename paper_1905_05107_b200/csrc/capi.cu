// C-ABI housekeeping: version and the thread-local error channel.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace pod {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
  return POD_ECUDA;
}

}  // namespace pod

extern "C" int pod_abi_version(void) { return 1; }

extern "C" const char* pod_last_error(void) { return pod::g_err; }
