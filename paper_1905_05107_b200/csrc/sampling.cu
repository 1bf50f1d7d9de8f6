// Column squared norms (one HBM streaming pass) and the inverse-CDF draw.
//
// pod_colnorms2_f64 replaces the reference's three data passes before the
// first round -- isfinite (matcore.py:54), einsum norms (isma.py:260) and the
// einsum again inside column_norm_distribution (sampling.py:136) -- with one
// coalesced double2 pass that also raises a non-finite flag.
//
// pod_draw is sample_with_replacement (sampling.py:204-222) over the live
// candidate set, including the strategy's distribution (isma.py:204-222 for
// l2n / unf, sampling.py:55-65 + 34-53 normalisation), the unique/counts
// collapse and the retirement of the drawn columns from S (isma.py:164).
// The caller's host Generator supplies the c uniforms (one batch per round,
// exactly like rng.random(c)), so index streams match the reference.
#include "common.cuh"

namespace pod {

// ----------------------------------------------------------- norms -------
template <bool VEC>
__global__ void __launch_bounds__(256) colnorms_block_kernel(const double* __restrict__ A,
                                                             int64_t m, int64_t n, int64_t lda,
                                                             double* __restrict__ out,
                                                             int* __restrict__ nonfinite) {
  __shared__ double red[8];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const double* col = A + j * lda;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (VEC) {
      const double2* c2 = reinterpret_cast<const double2*>(col);
      const int64_t m2 = m >> 1;
      int64_t i = threadIdx.x;
      for (; i + 3 * 256 < m2; i += 4 * 256) {
        double2 v0 = __ldcs(c2 + i), v1 = __ldcs(c2 + i + 256);
        double2 v2 = __ldcs(c2 + i + 512), v3 = __ldcs(c2 + i + 768);
        s0 = fma(v0.x, v0.x, s0); s1 = fma(v0.y, v0.y, s1);
        s2 = fma(v1.x, v1.x, s2); s3 = fma(v1.y, v1.y, s3);
        s0 = fma(v2.x, v2.x, s0); s1 = fma(v2.y, v2.y, s1);
        s2 = fma(v3.x, v3.x, s2); s3 = fma(v3.y, v3.y, s3);
      }
      for (; i < m2; i += 256) {
        double2 v = __ldcs(c2 + i);
        s0 = fma(v.x, v.x, s0); s1 = fma(v.y, v.y, s1);
      }
      if ((m & 1) && threadIdx.x == 0) { double v = col[m - 1]; s2 = fma(v, v, s2); }
    } else {
      for (int64_t i = threadIdx.x; i < m; i += 256) { double v = col[i]; s0 = fma(v, v, s0); }
    }
    double s = block_sum((s0 + s1) + (s2 + s3), red);
    if (threadIdx.x == 0) out[j] = s;
    if (!isfinite(s)) {  // non-finite entry or overflow: exact element check (rare path)
      int bad = 0;
      for (int64_t i = threadIdx.x; i < m; i += 256) bad |= !isfinite(col[i]);
      bad = __syncthreads_or(bad);
      if (bad && threadIdx.x == 0) atomicOr(nonfinite, 1);
    }
  }
}

__global__ void __launch_bounds__(256) colnorms_warp_kernel(const double* __restrict__ A, int64_t m,
                                                            int64_t n, int64_t lda,
                                                            double* __restrict__ out,
                                                            int* __restrict__ nonfinite) {
  const int lane = threadIdx.x & 31;
  const int64_t wglob = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = wglob; j < n; j += nw) {
    const double* col = A + j * lda;
    double s = 0.0;
    for (int64_t i = lane; i < m; i += 32) { double v = col[i]; s = fma(v, v, s); }
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
    if (!isfinite(s)) {
      int bad = 0;
      for (int64_t i = lane; i < m; i += 32) bad |= !isfinite(col[i]);
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
    }
  }
}

// fp32 storage: one CTA per column, float4 loads, fp64 accumulation of the
// exactly upcast values (as_dense's astype(float64), matcore.py:49)
__global__ void __launch_bounds__(256) colnorms_f32_kernel(const float* __restrict__ A, int64_t m,
                                                           int64_t n, int64_t lda, int vec,
                                                           double* __restrict__ out,
                                                           int* __restrict__ nonfinite) {
  __shared__ double red[8];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const float* col = A + j * lda;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t done = 0;
    if (vec) {
      const float4* c4 = reinterpret_cast<const float4*>(col);
      const int64_t m4 = m >> 2;
      for (int64_t i = threadIdx.x; i < m4; i += 256) {
        const float4 v = __ldcs(c4 + i);
        s0 = fma((double)v.x, (double)v.x, s0);
        s1 = fma((double)v.y, (double)v.y, s1);
        s2 = fma((double)v.z, (double)v.z, s2);
        s3 = fma((double)v.w, (double)v.w, s3);
      }
      done = m4 << 2;
    }
    for (int64_t i = done + threadIdx.x; i < m; i += 256) {
      const double v = (double)col[i];
      s0 = fma(v, v, s0);
    }
    double s = block_sum((s0 + s1) + (s2 + s3), red);
    if (threadIdx.x == 0) out[j] = s;
    if (!isfinite(s)) {
      int bad = 0;
      for (int64_t i = threadIdx.x; i < m; i += 256) bad |= !isfinite(col[i]);
      bad = __syncthreads_or(bad);
      if (bad && threadIdx.x == 0) atomicOr(nonfinite, 1);
    }
  }
}

// ------------------------------------------------------------ draw -------
constexpr int DRAW_THREADS = 1024;

// Exclusive scan of one double per thread in a fixed sequential order
// (thread 0 accumulates the 1024 per-thread totals left to right), so the
// CDF is monotone across chunk boundaries.
__device__ double block_excl_scan_seq(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    for (int t = 0; t < DRAW_THREADS; ++t) {
      double x = sh[t];
      sh[t] = run;
      run += x;
    }
    sh[DRAW_THREADS] = run;
  }
  __syncthreads();
  double r = sh[threadIdx.x];
  __syncthreads();
  return r;
}

__device__ int64_t block_excl_scan_i64(int64_t v, int64_t* sh, int64_t* total) {
  sh[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < DRAW_THREADS; ++t) {
      int64_t x = sh[t];
      sh[t] = run;
      run += x;
    }
    sh[DRAW_THREADS] = run;
  }
  __syncthreads();
  int64_t r = sh[threadIdx.x];
  *total = sh[DRAW_THREADS];
  __syncthreads();
  return r;
}

// mode 0: l2n over live columns (weights = raw norms2, normalised twice)
// mode 1: uniform over live columns
// mode 2: explicit normalised weights over all n positions (no live mask)
// mode 3: ort over live columns: raw squared residuals normalised twice, or
//         uniform when their sum <= thr (isma.py:216-220, sampling.py:182-186)
// mode 4: rows -- raw weights over all n positions normalised twice (like
//         mode 0) without a live mask and without retirement; p_out receives
//         the normalised weight of every drawn position (sampling.py:225-258)
__global__ void __launch_bounds__(DRAW_THREADS) draw_kernel(
    int mode, const double* __restrict__ raw, uint8_t* __restrict__ live, int64_t n,
    const double* __restrict__ uni, int64_t c, int32_t* __restrict__ idx_out,
    int64_t* __restrict__ cnt_out, int64_t cap, double* __restrict__ cum,
    int32_t* __restrict__ counts, int64_t* __restrict__ info, double thr,
    double* __restrict__ p_out) {
  const bool rows = (mode == 4);
  if (rows) mode = 0;
  __shared__ double shd[DRAW_THREADS + 1];
  __shared__ int64_t shi[DRAW_THREADS + 1];
  __shared__ double red[32];
  const int t = threadIdx.x;
  const int64_t chunk = (n + DRAW_THREADS - 1) / DRAW_THREADS;
  const int64_t j0 = min(n, t * chunk), j1 = min(n, j0 + chunk);

  // |S| = number of live candidates
  int64_t nlive_local = 0;
  for (int64_t j = j0; j < j1; ++j) nlive_local += (mode == 2 || rows) ? 1 : (live[j] != 0);
  int64_t nlive = 0;
  (void)block_excl_scan_i64(nlive_local, shi, &nlive);
  if (nlive == 0) {
    for (int64_t j = t; j < cap; j += DRAW_THREADS) idx_out[j] = -1;
    if (t == 0) { info[0] = 0; info[1] = 0; info[2] = 1; }  // status 1: empty S
    return;
  }
  // weights (sampling.py:55-65 then 34-53), kept in `cum` as scratch
  const double inv_s = 1.0 / (double)nlive;
  double loc = 0.0;
  if (mode == 3) {  // residual weights, or the uniform fallback
    for (int64_t j = j0; j < j1; ++j) loc += (rows || live[j]) ? raw[j] : 0.0;
    const double tot = block_sum(loc, red);
    mode = (tot <= thr) ? 1 : 0;
    loc = 0.0;
  }
  for (int64_t j = j0; j < j1; ++j) {
    double w;
    if (mode == 2) w = raw[j];
    else if (!rows && live[j] == 0) w = 0.0;
    else w = (mode == 0) ? raw[j] : inv_s;
    cum[j] = w;
    loc += w;
  }
  double total = block_sum(loc, red);
  double total1 = 1.0;
  if (mode == 2) total = 1.0;  // a Distribution's weights are used as given (sampling.py:214)
  if (mode == 0) {
    if (!(total > 0.0)) {
      for (int64_t j = t; j < cap; j += DRAW_THREADS) idx_out[j] = -1;
      if (t == 0) { info[0] = 0; info[1] = nlive; info[2] = 2; }  // status 2: degenerate
      return;
    }
    loc = 0.0;
    for (int64_t j = j0; j < j1; ++j) { double w = cum[j] / total; cum[j] = w; loc += w; }
    total1 = total;
    total = block_sum(loc, red);
  }
  // renormalise and scan
  loc = 0.0;
  int64_t last_local = -1;
  for (int64_t j = j0; j < j1; ++j) {
    double w = cum[j] / total;
    if (w > 0.0) last_local = j;
    loc += w;
    cum[j] = loc;
  }
  const double off = block_excl_scan_seq(loc, shd);
  for (int64_t j = j0; j < j1; ++j) cum[j] = off + cum[j];
  // last positive weight: max over threads
  shi[t] = last_local;
  __syncthreads();
  for (int s = DRAW_THREADS / 2; s > 0; s >>= 1) {
    if (t < s) shi[t] = max(shi[t], shi[t + s]);
    __syncthreads();
  }
  const int64_t last = shi[0];
  __syncthreads();
  for (int64_t j = max(j0, last); j < j1; ++j) cum[j] = 1.0;  // CDF pin (sampling.py:215-219)
  for (int64_t j = j0; j < j1; ++j) counts[j] = 0;
  __syncthreads();
  // searchsorted(cum, u, side="right") and occurrence counts
  for (int64_t d = t; d < c; d += DRAW_THREADS) {
    const double u = uni[d];
    int64_t lo = 0, hi = n - 1;  // first j with cum[j] > u; cum[n-1] == 1 > u
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (cum[mid] > u) hi = mid; else lo = mid + 1;
    }
    atomicAdd(&counts[lo], 1);
  }
  __syncthreads();
  // unique ascending + counts, retire from S
  int64_t nd_local = 0;
  for (int64_t j = j0; j < j1; ++j) nd_local += counts[j] > 0;
  int64_t g = 0;
  int64_t pos = block_excl_scan_i64(nd_local, shi, &g);
  for (int64_t j = j0; j < j1; ++j) {
    if (counts[j] > 0) {
      idx_out[pos] = (int32_t)j;
      cnt_out[pos] = counts[j];
      if (p_out) p_out[pos] = (raw[j] / total1) / total;  // the Distribution's weight
      ++pos;
      if (mode != 2 && !rows) live[j] = 0;
    }
  }
  for (int64_t j = g + t; j < cap; j += DRAW_THREADS) idx_out[j] = -1;  // zero-column padding
  if (t == 0) { info[0] = g; info[1] = nlive - g; info[2] = 0; }
}

}  // namespace pod

using namespace pod;

extern "C" size_t pod_draw_exact_ws_bytes(int64_t n);
extern "C" int pod_draw_exact(int mode, const double* weights, uint8_t* live, int64_t n,
                              const double* uniforms, int64_t c, int32_t* idx_out,
                              int64_t* cnt_out, int64_t cap, void* ws, size_t ws_bytes,
                              int64_t* info, double thr, void* stream);

extern "C" size_t pod_draw_ws_bytes(int64_t n) {
  return std::max((size_t)n * (sizeof(double) + sizeof(int32_t)) + 64,
                  pod_draw_exact_ws_bytes(n));
}

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
  if (mode != 4)  // column draws: numpy's exact summation order (exact_sums.cu)
    return pod_draw_exact(mode, weights, live, n, uniforms, c, idx_out, cnt_out, cap, ws, ws_bytes,
                          info, thr, stream);
  double* cum = (double*)ws;
  int32_t* counts = (int32_t*)(cum + n);
  draw_kernel<<<1, DRAW_THREADS, 0, (cudaStream_t)stream>>>(mode, weights, live, n, uniforms, c,
                                                              idx_out, cnt_out, cap, cum, counts,
                                                              info, thr, p_out);
  POD_CHECK_LAUNCH("draw");
  return POD_OK;
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
    double s = 0.0;
    for (int j = 0; j < ncols; ++j) {
      const int64_t c = cols ? (int64_t)cols[j] : (int64_t)j;
      if (c < 0) continue;
      const double v = (double)X[i + c * ldx];
      s = fma(v, v, s);
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
