// The inverse-CDF draw entry point and the ICRS row-sampling kernels.  (The
// column-norm pass and the draw itself live in exact_sums.cu: numpy's
// summation orders, bit for bit.)
//
// pod_draw is sample_with_replacement (sampling.py:204-222) over the live
// candidate set, including the strategy's distribution (isma.py:204-222 for
// l2n / unf, sampling.py:55-65 + 34-53 normalisation), the unique/counts
// collapse and the retirement of the drawn columns from S (isma.py:164) --
// all in numpy's exact summation order (exact_sums.cu).  The caller's host
// Generator supplies the c uniforms (one batch per round, exactly like
// rng.random(c)), so index streams match the reference.
#include "common.cuh"

using namespace pod;

extern "C" size_t pod_draw_exact_ws_bytes(int64_t n);
extern "C" int pod_draw_exact(int mode, const double* weights, uint8_t* live, int64_t n,
                              const double* uniforms, int64_t c, int32_t* idx_out,
                              int64_t* cnt_out, int64_t cap, void* ws, size_t ws_bytes,
                              int64_t* info, double thr, double* p_out, void* stream);

extern "C" size_t pod_draw_ws_bytes(int64_t n) { return pod_draw_exact_ws_bytes(n); }

extern "C" int pod_draw(int mode, const double* weights, uint8_t* live, int64_t n,
                        const double* uniforms, int64_t c, int32_t* idx_out, int64_t* cnt_out,
                        int64_t cap, void* ws, size_t ws_bytes, int64_t* info, double thr,
                        double* p_out, void* stream) {
  POD_REQUIRE(mode >= 0 && mode <= 4, "pod_draw: bad mode %d", mode);
  POD_REQUIRE(n > 0 && n < (int64_t)INT32_MAX, "pod_draw: bad n");
  POD_REQUIRE(c >= 1, "sample count must be >= 1");
  POD_REQUIRE(ws_bytes >= pod_draw_ws_bytes(n), "pod_draw: workspace too small");
  POD_REQUIRE(cap >= std::min<int64_t>(c, n), "pod_draw: output capacity %lld < min(c, n)",
              (long long)cap);
  POD_REQUIRE(mode == 1 || weights != nullptr, "pod_draw: weights required");
  POD_REQUIRE(mode == 2 || mode == 4 || live != nullptr, "pod_draw: live mask required");
  POD_REQUIRE(p_out == nullptr || mode == 4, "pod_draw: p_out needs mode 4");
  // every mode in numpy's exact summation order (exact_sums.cu)
  return pod_draw_exact(mode, weights, live, n, uniforms, c, idx_out, cnt_out, cap, ws, ws_bytes,
                        info, thr, p_out, stream);
}

namespace pod {
// out[i] = (sum_j X[i, cols[j]]^2) / div (cols -1: zero column), one thread per
// row; div = *div_dev when given (a graph-invariant launch with a per-round k)
template <typename TX>
__global__ void rownorms2_kernel(const TX* __restrict__ X, int64_t m, int ncols, int64_t ldx,
                                 const int32_t* __restrict__ cols, double div,
                                 const double* __restrict__ div_dev, double* __restrict__ out) {
  if (div_dev) div = *div_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    // np.einsum("ij,ij->i") on an F-ordered block (sampling.py:146, 200):
    // a sequential sum over the columns of separately rounded squares
    double s = 0.0;
    for (int j = 0; j < ncols; ++j) {
      const int64_t c = cols ? (int64_t)cols[j] : (int64_t)j;
      if (c < 0) continue;
      const double v = (double)X[i + c * ldx];
      s = __dadd_rn(s, __dmul_rn(v, v));
    }
    out[i] = s / div;
  }
}

// Y[i, j] = A[rows[i], cols[j]] * sqrt(cnt[i] / (w p[i])) for i < h (rows -1: zero)
template <typename TA>
__global__ void gather_scale_rows_kernel(const TA* __restrict__ A, int64_t lda,
                                         const int32_t* __restrict__ cols, int g,
                                         const int32_t* __restrict__ rows,
                                         const int64_t* __restrict__ cnt,
                                         const double* __restrict__ p, double w, int hcap,
                                         const int64_t* __restrict__ hdev,
                                         double* __restrict__ Y, int64_t ldy) {
  const int64_t h = *hdev;
  const int64_t tot = (int64_t)hcap * g;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(t / hcap), i = (int)(t - (int64_t)j * hcap);
    double v = 0.0;
    if (i < h) {
      const int64_t c = cols ? (int64_t)cols[j] : (int64_t)j;
      const int64_t r = rows[i];
      if (c >= 0 && r >= 0) v = (double)A[r + c * lda] * sqrt((double)cnt[i] / (w * p[i]));
    }
    Y[i + (int64_t)j * ldy] = v;
  }
}
}  // namespace pod

extern "C" int pod_rownorms2(int xtype, const void* X, int64_t m, int64_t ncols, int64_t ldx,
                             const int32_t* cols, double div, const double* div_dev, double* out,
                             void* stream) {
  POD_REQUIRE(xtype == POD_F64 || xtype == POD_F32, "pod_rownorms2: bad operand type");
  POD_REQUIRE(m >= 1 && ncols >= 0 && ldx >= m, "pod_rownorms2: bad shape");
  const int grid = (int)std::min<int64_t>(ceil_div(m, 256), 148 * 16);
  if (xtype == POD_F64)
    rownorms2_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const double*)X, m, (int)ncols, ldx, cols, div, div_dev, out);
  else
    rownorms2_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const float*)X, m, (int)ncols, ldx, cols, div, div_dev, out);
  POD_CHECK_LAUNCH("rownorms2");
  return POD_OK;
}

extern "C" int pod_gather_scale_rows(int atype, const void* A, int64_t lda, const int32_t* cols,
                                     int64_t g,
                                     const int32_t* rows, const int64_t* cnt, const double* p,
                                     double w, int64_t hcap, const int64_t* hdev, double* Y,
                                     int64_t ldy, void* stream) {
  POD_REQUIRE(g >= 1 && hcap >= 1 && ldy >= hcap, "pod_gather_scale_rows: bad shape");
  const int grid = (int)std::min<int64_t>(ceil_div(hcap * g, 256), 148 * 8);
  POD_REQUIRE(atype == POD_F64 || atype == POD_F32, "pod_gather_scale_rows: bad operand type");
  if (atype == POD_F64)
    gather_scale_rows_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const double*)A, lda, cols, (int)g, rows, cnt, p, w, (int)hcap, hdev, Y, ldy);
  else
    gather_scale_rows_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const float*)A, lda, cols, (int)g, rows, cnt, p, w, (int)hcap, hdev, Y, ldy);
  POD_CHECK_LAUNCH("gather_scale_rows");
  return POD_OK;
}
