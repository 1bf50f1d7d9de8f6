// Dependent-chain latencies on the B200: DFMA, DMUL, FFMA, MUFU.RSQ,
// F2F conversions, LDS, and the Jacobi rotation-parameter routine.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_1905_05107_b200/csrc lat_probe.cu -o lat_probe
#include <cstdio>
#include "bj_core.cuh"

__global__ void k_dfma(double* out, long long* cyc, double x) {
  double a = x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void k_ffma(float* out, long long* cyc, float x) {
  float a = x, b = 1.0000001f, c = 1e-9f;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = fmaf(a, b, c);
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void k_rsq(float* out, long long* cyc, float x) {
  float a = x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = rsqrtf(a) + 0.5f;
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void k_cvt(double* out, long long* cyc, double x) {
  double a = x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = (double)((float)a);
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, long long* cyc) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  double a = 0.0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = s[(int)a];
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void k_rot(double* out, long long* cyc, double g) {
  double al = 1.0, be = 0.3, c = 0, s = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    pod::bj::rot_params(g, al, be, c, s);
    g = g * 0.999 + 1e-3 * s;  // dependent
  }
  long long t1 = clock64();
  out[0] = c + s; cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, double x) {
  double a = x + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
  long long t1 = clock64();
  out[threadIdx.x] = a; cyc[threadIdx.x] = t1 - t0;
}
__global__ void k_bar(double* out, long long* cyc) {
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_dmma(double* out, long long* cyc) {
  double d0 = 0.0, d1 = 0.0, a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) pod::dmma8x8x4(d0, d1, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = d0 + d1;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dmma4(double* out, long long* cyc) {
  double d[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    pod::dmma8x8x4(d[0], d[1], a, b);
    pod::dmma8x8x4(d[2], d[3], a, b);
    pod::dmma8x8x4(d[4], d[5], a, b);
    pod::dmma8x8x4(d[6], d[7], a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = d[0] + d[2] + d[4] + d[6];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; float* f; long long* c;
  cudaMalloc(&d, 1 << 16); cudaMalloc(&f, 1 << 16); cudaMalloc(&c, 1 << 16);
  long long h[32];
  auto rep = [&](const char* nm, int iters) {
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cycles\n", nm, (double)h[0] / iters);
  };
  k_dfma<<<1, 1>>>(d, c, 1.0); rep("DFMA dependent", 1024);
  k_ffma<<<1, 1>>>(f, c, 1.0f); rep("FFMA dependent", 1024);
  k_rsq<<<1, 1>>>(f, c, 2.0f); rep("MUFU.RSQ + FADD", 1024);
  k_cvt<<<1, 1>>>(d, c, 2.0); rep("F2F f64->f32->f64", 1024);
  k_lds<<<1, 32>>>(d, c); rep("LDS.64 dependent (+F2I)", 1024);
  k_rot<<<1, 1>>>(d, c, 0.2); rep("rot_params + 2 dep DP", 256);
  k_shfl<<<1, 32>>>(d, c, 1.0); rep("SHFL.64 + DADD", 1024);
  k_bar<<<1, 256>>>(d, c); rep("__syncthreads (256 thr)", 1024);
  k_dmma<<<1, 32>>>(d, c); rep("DMMA 8x8x4 dependent", 1024);
  k_dmma4<<<1, 32>>>(d, c); rep("4 indep DMMA per iter", 1024);
  k_bar<<<1, 32>>>(d, c); rep("__syncthreads (32 thr)", 1024);
  cudaDeviceSynchronize();
  return 0;
}
