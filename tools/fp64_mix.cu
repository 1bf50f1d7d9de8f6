// Microbenchmark: do DMMA (tensor pipe) and DFMA (fp64 pipe) overlap on sm_100a?
// mode 0: DMMA only, 1: DFMA only, 2: warps split (even DMMA, odd DFMA),
// 3: every warp interleaves DMMA and DFMA at ratio R DFMA per DMMA.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int R>
__global__ void mix(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2], f[16];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int i = 0; i < 16; ++i) f[i] = i;
  const int warp = threadIdx.x >> 5;
  const bool do_mma = MODE == 0 || MODE == 3 || (MODE == 2 && (warp & 1) == 0);
  const bool do_fma = MODE == 1 || MODE == 3 || (MODE == 2 && (warp & 1) == 1);
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        if (MODE == 3) {
#pragma unroll
          for (int r = 0; r < R; ++r) f[(i * R + r) & 15] = fma(a, f[(i * R + r) & 15], b);
        }
      }
    }
    if (do_fma && MODE != 3) {
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = fma(a, f[i], b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int R>
void run(const char* name, double* out, int threads, int blocks) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  mix<MODE, R><<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  mix<MODE, R><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  double mma_w = 0, fma_w = 0;
  if (MODE == 0) mma_w = warps;
  if (MODE == 1) fma_w = warps;
  if (MODE == 2) { mma_w = warps / 2; fma_w = warps / 2; }
  if (MODE == 3) mma_w = warps;
  double fl = mma_w * iters * 8 * 512.0;           // DMMA 8x8x4 = 512 flop
  if (MODE == 3) fl += warps * iters * 8 * R * 32 * 2.0;
  else fl += fma_w * iters * 16 * 32 * 2.0;
  printf("%-28s threads %d blocks %d: %.2f TFLOP/s (%.3f ms)\n", name, threads, blocks,
         fl / ms / 1e9, ms);
}

int main() {
  double* out; cudaMalloc(&out, 1 << 26);
  for (int threads : {256, 512}) {
    int blocks = 296;
    run<0, 0>("dmma", out, threads, blocks);
    run<1, 0>("dfma", out, threads, blocks);
    run<2, 0>("split warps dmma|dfma", out, threads, blocks);
    run<3, 1>("interleave 1 dfma/dmma", out, threads, blocks);
    run<3, 2>("interleave 2 dfma/dmma", out, threads, blocks);
    run<3, 4>("interleave 4 dfma/dmma", out, threads, blocks);
    run<3, 8>("interleave 8 dfma/dmma", out, threads, blocks);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
