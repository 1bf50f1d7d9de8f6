// Shared helpers for the podsketch-b200 sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>

#include "../../include/podsketch_b200.h"

namespace pod {

constexpr int kWarp = 32;

// Host-side error channel (pod_last_error).
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

#define POD_CHECK_LAUNCH(where)                                   \
  do {                                                            \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return ::pod::cuda_status(_e, where);  \
  } while (0)

#define POD_REQUIRE(cond, ...)                 \
  do {                                         \
    if (!(cond)) {                             \
      ::pod::set_error(__VA_ARGS__);           \
      return POD_EPARAM;                       \
    }                                          \
  } while (0)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block-wide sum (fixed tree order).  `red` must hold
// blockDim.x/32 doubles.  Result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double out = red[0];
  __syncthreads();
  return out;
}

// Asynchronous 8-byte global->shared copy with zero fill when !valid.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_bytes = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_bytes));
}
// one element of T (float or double) with zero fill
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem, bool valid) {
  if constexpr (sizeof(T) == 8) cp_async8(smem, gmem, valid);
  else cp_async4(smem, gmem, valid);
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor pipe (DMMA.8x8x4).
// Lane t holds A[t/4][t%4], B[t%4][t/4], D[t/4][2(t%4)+{0,1}].
__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace pod
