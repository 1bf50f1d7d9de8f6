// Column-wise helpers over m-length factors: sign canonicalisation
// (fix_signs, matcore.py:148-165) and the per-mode convergence cosines
// (isma.py:195-196).  Both are deterministic two-level reductions over row
// chunks (no atomics on floating point).
#include "common.cuh"

namespace pod {

constexpr int CHUNK_ROWS = 8192;

// Per (row chunk, column): max |u| and the first row attaining it.
__global__ void __launch_bounds__(256) colargmax_partial_kernel(const double* __restrict__ U,
                                                                int64_t m, int64_t ldu, int l,
                                                                double* __restrict__ pval,
                                                                int64_t* __restrict__ prow) {
  __shared__ double sv[256];
  __shared__ int64_t sr[256];
  const int col = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * CHUNK_ROWS, r1 = min(m, r0 + CHUNK_ROWS);
  const double* u = U + (int64_t)col * ldu;
  double best = -1.0;
  int64_t brow = INT64_MAX;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) {
    const double a = fabs(u[i]);
    if (a > best) { best = a; brow = i; }  // rows visited ascending: first max kept
  }
  sv[threadIdx.x] = best;
  sr[threadIdx.x] = brow;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = sv[threadIdx.x + s];
      const int64_t orow = sr[threadIdx.x + s];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && orow < sr[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        sr[threadIdx.x] = orow;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pval[(int64_t)col * gridDim.x + blockIdx.x] = sv[0];
    prow[(int64_t)col * gridDim.x + blockIdx.x] = sr[0];
  }
}

// sign[col] = -1 if U[argmax row, col] < 0 else +1 (chunks in ascending order);
// optionally also the max |u| and its row (+ row_offset: global row index of a
// row shard) for a cross-shard combination.
__global__ void colargmax_final_kernel(const double* __restrict__ U, int64_t ldu, int l, int nchunk,
                                       const double* __restrict__ pval,
                                       const int64_t* __restrict__ prow,
                                       double* __restrict__ sign, double* __restrict__ val_out,
                                       int64_t* __restrict__ row_out, int64_t row_offset) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= l) return;
  double best = -1.0;
  int64_t brow = 0;
  for (int c = 0; c < nchunk; ++c) {
    const double v = pval[(int64_t)col * nchunk + c];
    if (v > best) { best = v; brow = prow[(int64_t)col * nchunk + c]; }
  }
  sign[col] = (U[brow + (int64_t)col * ldu] < 0.0) ? -1.0 : 1.0;
  if (val_out) val_out[col] = best;
  if (row_out) row_out[col] = brow + row_offset;
}

__global__ void scale_cols_kernel(double* __restrict__ U, int64_t m, int64_t ldu, int l,
                                  const double* __restrict__ sign) {
  const int col = blockIdx.y;
  const double s = sign[col];
  if (s == 1.0) return;
  double* u = U + (int64_t)col * ldu;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    u[i] = -u[i];
}

// Partial dot products of matching columns: pd[col * nchunk + chunk].
__global__ void __launch_bounds__(256) coldots_partial_kernel(const double* __restrict__ P,
                                                              int64_t ldp,
                                                              const double* __restrict__ Q,
                                                              int64_t ldq, int64_t m, int k,
                                                              double* __restrict__ pd) {
  __shared__ double red[8];
  const int col = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * CHUNK_ROWS, r1 = min(m, r0 + CHUNK_ROWS);
  const double* p = P + (int64_t)col * ldp;
  const double* q = Q + (int64_t)col * ldq;
  double s = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) s = fma(p[i], q[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) pd[(int64_t)col * gridDim.x + blockIdx.x] = s;
}

__global__ void coldots_final_kernel(const double* __restrict__ pd, int nchunk, int k, int kk,
                                     int take_abs, double* __restrict__ out) {
  const int col = threadIdx.x + blockIdx.x * blockDim.x;
  if (col >= k) return;
  double s = 0.0;
  if (col < kk)
    for (int c = 0; c < nchunk; ++c) s += pd[(int64_t)col * nchunk + c];
  if (take_abs) s = fmin(fmax(fabs(s), 0.0), 1.0);  // isma.py:196 abs, :201 clip to [0, 1]
  out[col] = s;
}

}  // namespace pod

using namespace pod;

extern "C" size_t pod_colwise_ws_bytes(int64_t m, int64_t l) {
  const int64_t nchunk = std::max<int64_t>(1, ceil_div(m, CHUNK_ROWS));
  return (size_t)nchunk * l * 16 + (size_t)l * 8 + 64;
}

extern "C" int pod_fix_signs(double* U, int64_t m, int64_t l, int64_t ldu, double* V, int64_t n,
                             int64_t ldv, double* sign_out, void* ws, size_t ws_bytes,
                             void* stream) {
  POD_REQUIRE(m >= 1 && l >= 0 && ldu >= m, "pod_fix_signs: bad shape");
  if (l == 0) return POD_OK;
  POD_REQUIRE(ws_bytes >= pod_colwise_ws_bytes(m, l), "pod_fix_signs: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const int nchunk = (int)std::max<int64_t>(1, ceil_div(m, CHUNK_ROWS));
  double* pval = (double*)ws;
  int64_t* prow = (int64_t*)(pval + (size_t)nchunk * l);
  double* sign = sign_out ? sign_out : (double*)(prow + (size_t)nchunk * l);
  colargmax_partial_kernel<<<dim3(nchunk, (unsigned)l), 256, 0, s>>>(U, m, ldu, (int)l, pval, prow);
  POD_CHECK_LAUNCH("colargmax partial");
  colargmax_final_kernel<<<(unsigned)ceil_div(l, 128), 128, 0, s>>>(
      U, ldu, (int)l, nchunk, pval, prow, sign, nullptr, nullptr, 0);
  POD_CHECK_LAUNCH("colargmax final");
  const int gx = (int)std::min<int64_t>(ceil_div(m, 256), 256);
  scale_cols_kernel<<<dim3(gx, (unsigned)l), 256, 0, s>>>(U, m, ldu, (int)l, sign);
  POD_CHECK_LAUNCH("flip U");
  if (V) {
    const int gv = (int)std::min<int64_t>(ceil_div(n, 256), 256);
    scale_cols_kernel<<<dim3(gv, (unsigned)l), 256, 0, s>>>(V, n, ldv, (int)l, sign);
    POD_CHECK_LAUNCH("flip V");
  }
  return POD_OK;
}

extern "C" int pod_coldots(const double* P, int64_t ldp, const double* Q, int64_t ldq, int64_t m,
                           int64_t k, int64_t kk, int take_abs, double* out, void* ws,
                           size_t ws_bytes, void* stream) {
  POD_REQUIRE(m >= 1 && k >= 0 && kk >= 0 && kk <= k, "pod_coldots: bad shape");
  if (k == 0) return POD_OK;
  POD_REQUIRE(ws_bytes >= pod_colwise_ws_bytes(m, k), "pod_coldots: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const int nchunk = (int)std::max<int64_t>(1, ceil_div(m, CHUNK_ROWS));
  double* pd = (double*)ws;
  if (kk > 0) {
    coldots_partial_kernel<<<dim3(nchunk, (unsigned)kk), 256, 0, s>>>(P, ldp, Q, ldq, m, (int)kk,
                                                                      pd);
    POD_CHECK_LAUNCH("coldots partial");
  }
  coldots_final_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, s>>>(pd, nchunk, (int)k, (int)kk,
                                                                  take_abs, out);
  POD_CHECK_LAUNCH("coldots final");
  return POD_OK;
}

extern "C" int pod_colargmax(const double* U, int64_t m, int64_t l, int64_t ldu, int64_t row_offset,
                             double* val_out, int64_t* row_out, double* sign_out, void* ws,
                             size_t ws_bytes, void* stream) {
  POD_REQUIRE(m >= 1 && l >= 0 && ldu >= m, "pod_colargmax: bad shape");
  if (l == 0) return POD_OK;
  POD_REQUIRE(ws_bytes >= pod_colwise_ws_bytes(m, l), "pod_colargmax: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const int nchunk = (int)std::max<int64_t>(1, ceil_div(m, CHUNK_ROWS));
  double* pval = (double*)ws;
  int64_t* prow = (int64_t*)(pval + (size_t)nchunk * l);
  colargmax_partial_kernel<<<dim3(nchunk, (unsigned)l), 256, 0, s>>>(U, m, ldu, (int)l, pval, prow);
  POD_CHECK_LAUNCH("colargmax partial");
  colargmax_final_kernel<<<(unsigned)ceil_div(l, 128), 128, 0, s>>>(
      U, ldu, (int)l, nchunk, pval, prow, sign_out, val_out, row_out, row_offset);
  POD_CHECK_LAUNCH("colargmax final");
  return POD_OK;
}

extern "C" int pod_scale_cols(double* U, int64_t m, int64_t l, int64_t ldu, const double* sign,
                              void* stream) {
  POD_REQUIRE(m >= 0 && l >= 0 && ldu >= m, "pod_scale_cols: bad shape");
  if (m == 0 || l == 0) return POD_OK;
  const int gx = (int)std::min<int64_t>(ceil_div(m, 256), 256);
  scale_cols_kernel<<<dim3(gx, (unsigned)l), 256, 0, (cudaStream_t)stream>>>(U, m, ldu, (int)l,
                                                                            sign);
  POD_CHECK_LAUNCH("scale cols");
  return POD_OK;
}

// ---------------------------------------------------------------------------
// Sampled-column gather for host-resident (streamed) matrices: D[:, j] =
// A[:, idx[j]] (idx -1: zero column) for j < g.  A may be page-locked host
// memory mapped into the device address space, so this is the one PCIe read
// of the sampled block per round (isma.py:163); the round's GEMMs then read
// D from HBM.  Column-parallel, 16-byte vectorised when aligned.
namespace pod {
template <typename T>
__global__ void __launch_bounds__(256) gather_cols_kernel(const T* __restrict__ A, int64_t m,
                                                          int64_t lda, const int32_t* __restrict__ idx,
                                                          int g, T* __restrict__ D, int64_t ldd,
                                                          int vec) {
  constexpr int V = 16 / sizeof(T);
  for (int j = blockIdx.y; j < g; j += gridDim.y) {
    const int64_t c = idx ? (int64_t)idx[j] : (int64_t)j;
    T* dst = D + (int64_t)j * ldd;
    if (c < 0) {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
           i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = T(0);
      continue;
    }
    const T* src = A + c * lda;
    if (vec) {
      const int64_t mv = m / V;
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mv;
           i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<int4*>(dst)[i] = __ldcs(reinterpret_cast<const int4*>(src) + i);
      for (int64_t i = mv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
           i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    } else {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
           i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    }
  }
}
}  // namespace pod

extern "C" int pod_gather_cols(int atype, const void* A, int64_t m, int64_t lda,
                               const int32_t* idx, int64_t g, void* D, int64_t ldd,
                               void* stream) {
  POD_REQUIRE(atype == POD_F64 || atype == POD_F32, "pod_gather_cols: bad operand type");
  POD_REQUIRE(m >= 1 && g >= 0 && lda >= m && ldd >= m, "pod_gather_cols: bad shape");
  if (g == 0) return POD_OK;
  const size_t es = atype == POD_F64 ? 8 : 4;
  const int vec = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(D)) % 16 == 0) &&
                  ((lda * es) % 16 == 0) && ((ldd * es) % 16 == 0);
  const int gx = (int)std::min<int64_t>(ceil_div(m, 256 * (16 / (int64_t)es)), 64);
  dim3 grid((unsigned)std::max(1, gx), (unsigned)std::min<int64_t>(g, 1024));
  cudaStream_t s = (cudaStream_t)stream;
  if (atype == POD_F64)
    gather_cols_kernel<double><<<grid, 256, 0, s>>>((const double*)A, m, lda, idx, (int)g,
                                                    (double*)D, ldd, vec);
  else
    gather_cols_kernel<float><<<grid, 256, 0, s>>>((const float*)A, m, lda, idx, (int)g,
                                                   (float*)D, ldd, vec);
  POD_CHECK_LAUNCH("gather cols");
  return POD_OK;
}

// D[:, j] = A[:, idx[j]] * f[j] in fp64 (scale_sampled_columns, sampling.py:
// 234-245: one column per index, already repeated/deduplicated by the caller)
namespace pod {
template <typename T>
__global__ void __launch_bounds__(256) gather_scale_cols_kernel(const T* __restrict__ A, int64_t m,
                                                                int64_t lda,
                                                                const int64_t* __restrict__ idx,
                                                                const double* __restrict__ f, int g,
                                                                double* __restrict__ D, int64_t ldd) {
  for (int j = blockIdx.y; j < g; j += gridDim.y) {
    const T* src = A + idx[j] * lda;
    double* dst = D + (int64_t)j * ldd;
    const double s = f[j];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = (double)src[i] * s;
  }
}
}  // namespace pod

extern "C" int pod_gather_scale_cols(int atype, const void* A, int64_t m, int64_t lda,
                                     const int64_t* idx, const double* f, int64_t g, double* D,
                                     int64_t ldd, void* stream) {
  POD_REQUIRE(atype == POD_F64 || atype == POD_F32, "pod_gather_scale_cols: bad operand type");
  POD_REQUIRE(m >= 1 && g >= 0 && lda >= m && ldd >= m, "pod_gather_scale_cols: bad shape");
  if (g == 0) return POD_OK;
  const int gx = (int)std::min<int64_t>(ceil_div(m, 256 * 4), 64);
  dim3 grid((unsigned)std::max(1, gx), (unsigned)std::min<int64_t>(g, 1024));
  cudaStream_t s = (cudaStream_t)stream;
  if (atype == POD_F64)
    gather_scale_cols_kernel<double><<<grid, 256, 0, s>>>((const double*)A, m, lda, idx, f, (int)g,
                                                          D, ldd);
  else
    gather_scale_cols_kernel<float><<<grid, 256, 0, s>>>((const float*)A, m, lda, idx, f, (int)g,
                                                         D, ldd);
  POD_CHECK_LAUNCH("gather scale cols");
  return POD_OK;
}
