// Squared residual norms of columns after projection onto an orthonormal
// basis: out[j] = || A[:, j] - U C[:, j] ||^2 with C = U^T A precomputed
// (TN GEMM).  The reference's residual_distribution (sampling.py:158-187)
// materialises resid = cols - u (u^T cols); here the product U C is formed
// tile by tile on the FP64 tensor pipe (DMMA.8x8x4) and subtracted from the
// A tile in registers, so the m x n residual is never written.
#include "common.cuh"

namespace pod {
namespace rsd {
constexpr int THREADS = 256;
constexpr int BM = 64, BN = 64;
constexpr int LDX = BM + 4;        // U block [k][row], % 16 == 4
constexpr int LDA = BM + 2;        // A tile [col][row]
constexpr int ROWS_PER_CTA = 4096; // row chunk per CTA (deterministic 2-level reduction)

__host__ __device__ inline int kpad(int r) { return (r + 7) & ~7; }
__host__ __device__ inline int ldc(int r) { return kpad(r) + 4; }
inline size_t smem_bytes(int r) {
  return ((size_t)kpad(r) * LDX + (size_t)BN * ldc(r) + (size_t)BN * LDA + 8 * BN) *
         sizeof(double);
}

template <typename TA>
__global__ void __launch_bounds__(THREADS) partial_kernel(
    int64_t m, int n, int r, const TA* __restrict__ A, int64_t lda,
    const int32_t* __restrict__ cols, const double* __restrict__ U, int64_t ldu,
    const double* __restrict__ Cm, int64_t ldcm, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  const int KP = kpad(r), LC = ldc(r);
  double* us = sm;                              // KP x LDX
  double* cs = us + (size_t)KP * LDX;           // BN x LC  (C tile, [j][k])
  double* as = cs + (size_t)BN * LC;            // BN x LDA (A tile, [j][row])
  double* red = as + (size_t)BN * LDA;          // 8 x BN column partials per warp row
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.x * BN;
  const int64_t c0 = (int64_t)blockIdx.y * ROWS_PER_CTA, c1 = min(m, c0 + ROWS_PER_CTA);
  for (int e = threadIdx.x; e < BN * KP; e += THREADS) {
    const int j = e / KP, k = e - j * KP;
    cs[j * LC + k] = (j0 + j < n && k < r) ? Cm[k + (int64_t)(j0 + j) * ldcm] : 0.0;
  }
  const int wm = warp & 1, wn = warp >> 1;  // warp tile: 32 rows x 16 cols
  double colacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // per (g, e) column partial of this lane
  for (int64_t rb = c0; rb < c1; rb += BM) {
    __syncthreads();
    for (int e = threadIdx.x; e < KP * BM; e += THREADS) {
      const int k = e / BM, i = e - k * BM;
      const int64_t row = rb + i;
      us[k * LDX + i] = (k < r && row < c1) ? U[row + (int64_t)k * ldu] : 0.0;
    }
    for (int e = threadIdx.x; e < BN * BM; e += THREADS) {
      const int j = e / BM, i = e - j * BM;
      const int64_t row = rb + i;
      double v = 0.0;
      if (j0 + j < n && row < c1) {
        const int64_t col = cols ? (int64_t)cols[j0 + j] : (int64_t)(j0 + j);
        if (col >= 0) v = (double)A[row + col * lda];
      }
      as[j * LDA + i] = v;
    }
    __syncthreads();
    double acc[4][2][2];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int g = 0; g < 2; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
    for (int k0 = 0; k0 < KP; k0 += 4) {
      double a[4], b[2];
#pragma unroll
      for (int f = 0; f < 4; ++f) a[f] = us[(k0 + (lane & 3)) * LDX + wm * 32 + f * 8 + (lane >> 2)];
#pragma unroll
      for (int g = 0; g < 2; ++g) b[g] = cs[(wn * 16 + g * 8 + (lane >> 2)) * LC + k0 + (lane & 3)];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < 2; ++g) dmma8x8x4(acc[f][g][0], acc[f][g][1], a[f], b[g]);
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int i = wm * 32 + f * 8 + (lane >> 2);
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = wn * 16 + g * 8 + 2 * (lane & 3) + e;
          const double d = as[j * LDA + i] - acc[f][g][e];
          colacc[g][e] = fma(d, d, colacc[g][e]);
        }
    }
  }
  // reduce over the 8 lanes sharing a column (lane >> 2 varies), then warps of the same wn
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = colacc[g][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      colacc[g][e] = v;
    }
  __syncthreads();
  if (lane < 4) {
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) red[wm * BN + wn * 16 + g * 8 + 2 * lane + e] = colacc[g][e];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < BN; j += THREADS)
    if (j0 + j < n) part[(int64_t)blockIdx.y * n + j0 + j] = red[j] + red[BN + j];
}

__global__ void reduce_kernel(int nchunk, int n, const double* __restrict__ part,
                              double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += part[(int64_t)c * n + j];
    out[j] = s;
  }
}
}  // namespace rsd
}  // namespace pod

using namespace pod;

extern "C" size_t pod_resid_ws_bytes(int64_t m, int64_t n) {
  return (size_t)ceil_div(m, rsd::ROWS_PER_CTA) * n * sizeof(double) + 64;
}

extern "C" int pod_resid_colnorms2(int atype, int64_t m, int64_t n, const void* A, int64_t lda,
                                   const int32_t* cols, const double* U, int64_t ldu, int64_t r,
                                   const double* C, int64_t ldc, double* out, void* ws,
                                   size_t ws_bytes, void* stream) {
  POD_REQUIRE(atype == POD_F64 || atype == POD_F32, "pod_resid_colnorms2: bad operand type");
  POD_REQUIRE(m >= 1 && n >= 1 && r >= 1 && r <= 256 && lda >= m && ldu >= m && ldc >= r,
              "pod_resid_colnorms2: bad shape");
  POD_REQUIRE(ws_bytes >= pod_resid_ws_bytes(m, n), "pod_resid_colnorms2: workspace too small");
  const size_t bytes = rsd::smem_bytes((int)r);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(rsd::partial_kernel<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "resid attr");
    e = cudaFuncSetAttribute(rsd::partial_kernel<float>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "resid attr");
    attr = true;
  }
  POD_REQUIRE(bytes <= 227 * 1024, "pod_resid_colnorms2: r too large");
  cudaStream_t s = (cudaStream_t)stream;
  const int nchunk = (int)ceil_div(m, rsd::ROWS_PER_CTA);
  dim3 grid((unsigned)ceil_div(n, rsd::BN), (unsigned)nchunk);
  if (atype == POD_F64)
    rsd::partial_kernel<double><<<grid, rsd::THREADS, bytes, s>>>(
        m, (int)n, (int)r, (const double*)A, lda, cols, U, ldu, C, ldc, (double*)ws);
  else
    rsd::partial_kernel<float><<<grid, rsd::THREADS, bytes, s>>>(
        m, (int)n, (int)r, (const float*)A, lda, cols, U, ldu, C, ldc, (double*)ws);
  POD_CHECK_LAUNCH("resid partial");
  rsd::reduce_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(nchunk, (int)n, (const double*)ws,
                                                                out);
  POD_CHECK_LAUNCH("resid reduce");
  return POD_OK;
}
