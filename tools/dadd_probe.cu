// fp64 latency / issue probes on this B200 (cycles per loop iteration):
//   dadd     : one dependent DADD chain
//   chain2x4 : two interleaved DADD chains, 4 adds each per iteration (8 DADD)
//   +dmul8   : the same plus 8 independent DMULs per iteration (the einsum
//              norm loop's instruction mix: 8 DMUL + 8 DADD per 8-row block)
//   +lds     : the same with the DMUL operands loaded from shared memory
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a dadd_probe.cu -o dadd_probe
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x, double y) {
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = x, b = y;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  double a0 = x, a1 = y;
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) {
    a0 = __dadd_rn(a0, 1e-9); a1 = __dadd_rn(a1, 2e-9);
    a0 = __dadd_rn(a0, 3e-9); a1 = __dadd_rn(a1, 4e-9);
    a0 = __dadd_rn(a0, 5e-9); a1 = __dadd_rn(a1, 6e-9);
    a0 = __dadd_rn(a0, 7e-9); a1 = __dadd_rn(a1, 8e-9);
  }
  long long t2 = clock64();
  double y0 = x, y1 = y, y2 = x + 1, y3 = y + 1, y4 = x + 2, y5 = y + 2, y6 = x + 3, y7 = y + 3;
  double b0 = x, b1 = y;
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) {
    y0 = __dmul_rn(y0, 0.9999999); y1 = __dmul_rn(y1, 0.9999999);
    y2 = __dmul_rn(y2, 0.9999999); y3 = __dmul_rn(y3, 0.9999999);
    y4 = __dmul_rn(y4, 0.9999999); y5 = __dmul_rn(y5, 0.9999999);
    y6 = __dmul_rn(y6, 0.9999999); y7 = __dmul_rn(y7, 0.9999999);
    b0 = __dadd_rn(b0, y6); b1 = __dadd_rn(b1, y7);
    b0 = __dadd_rn(b0, y4); b1 = __dadd_rn(b1, y5);
    b0 = __dadd_rn(b0, y2); b1 = __dadd_rn(b1, y3);
    b0 = __dadd_rn(b0, y0); b1 = __dadd_rn(b1, y1);
  }
  long long t3 = clock64();
  double c0 = x, c1 = y;
  const double2* v = reinterpret_cast<const double2*>(sh);
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) {
    const int o = (i * 4) & 511;
    double2 q0 = v[o], q1 = v[o + 1], q2 = v[o + 2], q3 = v[o + 3];
    c0 = __dadd_rn(__dmul_rn(q3.x, q3.x), c0); c1 = __dadd_rn(__dmul_rn(q3.y, q3.y), c1);
    c0 = __dadd_rn(__dmul_rn(q2.x, q2.x), c0); c1 = __dadd_rn(__dmul_rn(q2.y, q2.y), c1);
    c0 = __dadd_rn(__dmul_rn(q1.x, q1.x), c0); c1 = __dadd_rn(__dmul_rn(q1.y, q1.y), c1);
    c0 = __dadd_rn(__dmul_rn(q0.x, q0.x), c0); c1 = __dadd_rn(__dmul_rn(q0.y, q0.y), c1);
  }
  long long t4 = clock64();
  out[0] = a + a0 + a1 + b0 + b1 + c0 + c1 + y0 + y1 + y2 + y3 + y4 + y5 + y6 + y7;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 8); cudaMallocManaged(&c, 32);
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, c, 1.0, 1e-7); cudaDeviceSynchronize(); }
  printf("dadd chain %.2f cyc/add | 2 chains x4 %.2f cyc/iter | +8 dmul %.2f cyc/iter | "
         "lds+dmul+dadd block %.2f cyc/iter\n", c[0] / 4096.0, c[1] / 1024.0, c[2] / 1024.0,
         c[3] / 1024.0);
  return 0;
}
