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

// Page-lock (and map) a host buffer for direct device access by the kernels
// (host-resident / streamed matrices).  On this platform (UVA) the device
// address of mapped page-locked memory is the host address; this is checked.
extern "C" int pod_host_register(void* ptr, size_t bytes) {
  POD_REQUIRE(ptr != nullptr && bytes > 0, "pod_host_register: empty buffer");
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) return pod::cuda_status(e, "cudaHostRegister");
  void* dptr = nullptr;
  e = cudaHostGetDevicePointer(&dptr, ptr, 0);
  if (e != cudaSuccess) return pod::cuda_status(e, "cudaHostGetDevicePointer");
  if (dptr != ptr) {
    cudaHostUnregister(ptr);
    pod::set_error("pod_host_register: device address of mapped memory differs from host address");
    return POD_ECUDA;
  }
  return POD_OK;
}

extern "C" int pod_host_unregister(void* ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  return e == cudaSuccess ? POD_OK : pod::cuda_status(e, "cudaHostUnregister");
}
