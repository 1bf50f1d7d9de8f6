// On-device small dense solvers (one CTA each): the per-round eigen/SVD
// problems of ISMA stay on the GPU next to the data they steer.
//
//  pod_gram_eigh    gram_spectrum + lift setup (baselines.py:35-65): eigen-
//                   decomposition of the g x g Gram by one-sided Jacobi,
//                   descending, clip + eigenvalue dust (<= 1e-12 lambda_1,
//                   matcore.py:26) -> sigma, rank (> 1e-14 sigma_1,
//                   matcore.py:20), keep = min(r, rank), T = V[:, :keep]/sigma.
//  pod_cholqr_factor  one CholeskyQR pass on a Gram W^T W: column scaling,
//                   shifted retry on breakdown, exact-zero columns dropped
//                   (their R rows are zero, as Householder's would be).
//                   Stands in for LAPACK dgeqrf in merge.py:70/76.
//  pod_merge_core   E = [[S1, M S2], [0, R S2]] (merge.py:80-83), its SVD
//                   (merge.py:84) by one-sided Jacobi, keep rule (merge.py:85)
//                   and the rotation T that maps [U1 Q] to the merged basis.
//  pod_svd_small    values (+ left/right vectors) of a small matrix: finalize
//                   SVD of R (isma.py:297) and the subspace criterion
//                   (isma.py:197-198).
//
// Matrices up to ~200 KB live in shared memory; larger ones run in place in
// a global (L2-resident) workspace.
#include "common.cuh"

#include <cstdio>

namespace pod {

constexpr int SMALL_THREADS = 1024;
static inline int jacobi_threads(int64_t n) {
  int64_t pairs = (n + 1) / 2;
  int64_t t = ((16 * pairs + 31) / 32) * 32;
  return (int)std::max<int64_t>(128, std::min<int64_t>(1024, t));
}
constexpr size_t SMALL_SMEM_CAP = 200 * 1024;

// perm[k] = index of the k-th largest key (ties -> lower index first).
__device__ __forceinline__ void rank_sort_desc(const double* key, int n, int* perm) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double kj = key[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double ki = key[i];
      rank += (ki > kj) || (ki == kj && i < j);
    }
    perm[rank] = j;
  }
  __syncthreads();
}

// ---------------------------------------------------------- gram eigh ----
// Stage 1 of pod_gram_eigh: pivoted Cholesky P G P^T = R^T R of the PSD
// sampled Gram (stops when the largest remaining diagonal <= 1e-15 max
// diagonal; the neglected block lies far below the 1e-12 lambda_1 dust rule
// of matcore.py:26).  Writes X = R^T (g x g, zero columns >= rank), piv and
// rank.  Stage 2 (cluster_jacobi.cu) runs one-sided Jacobi on X's columns:
// X J = V' Sigma, so convergence is that of an SVD of the sampled block.
constexpr int PIVCHOL_THREADS = 512;
// Right-looking pivoted Cholesky without physical row/column swaps: W keeps
// the Schur complement in the ORIGINAL index order, row j of R is stored by
// original index in Rq (Rq[j + q g]) and X = R^T in pivoted order is
// assembled at the end (X[i, j] = Rq[j, piv[i]]).  W is symmetric and kept
// as its packed lower triangle (column b holds rows b..g-1 at off(b) =
// b g - b (b - 1) / 2), so g <= 231 fits in shared memory.  Per step: (A) all threads
// form r_j; (B) warp 0 updates its register copy of the remaining diagonal
// and picks the NEXT pivot while warps 1.. apply the rank-1 update, each lane
// holding its RK rows' r values and done flags in registers (loads of a
// column are all issued before its stores).  Two barriers per step.
template <bool SMEM, int RK>
__global__ void __launch_bounds__(PIVCHOL_THREADS) pivchol_kernel(
    const double* __restrict__ G, int64_t ldg, int g, double* __restrict__ Xout,
    int* __restrict__ piv_out, int64_t* __restrict__ rank_out, double* gws,
    double* __restrict__ Rq) {
  extern __shared__ __align__(16) double sm[];
  double* __restrict__ W = SMEM ? sm : gws;
  __shared__ double s_d0, s_d, s_rv[512];
  __shared__ int s_p, s_done[512], s_piv[512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  auto off = [g](int b) { return (int64_t)b * g - (int64_t)b * (b - 1) / 2; };
  auto at = [&](int a, int b) -> double& {  // symmetric element, packed lower storage
    return a >= b ? W[off(b) + (a - b)] : W[off(a) + (b - a)];
  };
  for (int b = warp; b < g; b += nwarp)
    for (int a = b + lane; a < g; a += 32) W[off(b) + (a - b)] = G[a + b * ldg];
  for (int q = threadIdx.x; q < g; q += blockDim.x) s_done[q] = 0;
  __syncthreads();
  double diag[RK];  // warp 0: remaining diagonal of rows lane + 32 k
  uint32_t dmask = 0;  // warp 0: eliminated rows among lane + 32 k
  auto pick = [&](int j) {  // warp 0: argmax of the remaining diagonal
    double bv = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < RK; ++k) {
      const int q = lane + 32 * k;
      if (q < g && !((dmask >> k) & 1u) && diag[k] > bv) { bv = diag[k]; bi = q; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) {
      if (j == 0) s_d0 = bv;
      s_d = bv;
      s_p = bi;
    }
  };
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < RK; ++k) {
      const int q = lane + 32 * k;
      diag[k] = q < g ? W[off(q)] : 0.0;
    }
    pick(0);
  }
  __syncthreads();
  int rank = g;
  for (int j = 0; j < g; ++j) {
    const double d = s_d;
    if (!(d > 1e-15 * s_d0 && d > 0.0)) {  // remaining block negligible
      rank = j;
      break;
    }
    const int p = s_p;
    const double rjj = sqrt(d);
    const double rinv = 1.0 / rjj;
    // (A) r_j by original index
    for (int q = threadIdx.x; q < g; q += blockDim.x) {
      double v = 0.0;
      if (!s_done[q]) v = (q == p) ? rjj : at(p, q) * rinv;
      s_rv[q] = (q == p) ? 0.0 : v;  // p leaves the Schur complement
      Rq[j + (int64_t)q * g] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_done[p] = 1;
      s_piv[j] = p;
    }
    if (warp == 0) {  // (B0) next pivot from the updated diagonal
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        const int q = lane + 32 * k;
        if (q == p) dmask |= 1u << k;
        if (q < g) {
          const double rv = s_rv[q];
          diag[k] -= rv * rv;
        }
      }
      pick(j + 1);
    } else {  // (B) rank-1 update of the remaining block
      double rva[RK];
      uint32_t live = 0;
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        const int a = lane + 32 * k;
        rva[k] = a < g ? s_rv[a] : 0.0;
        if (a < g && !s_done[a] && a != p) live |= 1u << k;
      }
      for (int b = warp - 1; b < g; b += nwarp - 1) {
        if (b == p || s_done[b]) continue;
        const double rb = s_rv[b];
        double* col = W + off(b) - b;  // col[a] = W(a, b) for a >= b
        double w[RK];
#pragma unroll
        for (int k = 0; k < RK; ++k) {
          const int a = lane + 32 * k;
          w[k] = (((live >> k) & 1u) && a >= b) ? col[a] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < RK; ++k) {
          const int a = lane + 32 * k;
          if (((live >> k) & 1u) && a >= b) col[a] = w[k] - rva[k] * rb;
        }
      }
    }
    __syncthreads();
  }
  // pivot order of the never-eliminated indices (after rank): ascending
  if (threadIdx.x == 0) {
    int k = rank;
    for (int q = 0; q < g; ++q)
      if (!s_done[q]) s_piv[k++] = q;
  }
  __syncthreads();
  // X[i][j] = R[j][piv[i]] for j < rank, i >= j; zero elsewhere
  for (int jj = warp; jj < g; jj += nwarp)
    for (int i = lane; i < g; i += 32)
      Xout[i + (int64_t)jj * g] = (jj < rank && i >= jj) ? Rq[jj + (int64_t)s_piv[i] * g] : 0.0;
  for (int i = threadIdx.x; i < g; i += blockDim.x) piv_out[i] = s_piv[i];
  if (threadIdx.x == 0) *rank_out = rank;
}

// --------------------------------------------------------- CholeskyQR ----
// Upper-triangular inverse of Rh (l x l, ld l) into X (ld l): warp per column.
// rdiag[i] = 1 / Rh[i][i] (precomputed: no division in the dependent chain)
__device__ __forceinline__ void upper_inverse(const double* Rh, int l, double* X,
                                              const double* rdiag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < l; j += nw) {
    double* xj = X + (int64_t)j * l;
    for (int i = lane; i < l; i += 32) xj[i] = 0.0;
    __syncwarp();
    if (lane == 0) xj[j] = 1.0 / Rh[j + (int64_t)j * l];
    __syncwarp();
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1 + lane; k <= j; k += 32) s = fma(Rh[i + (int64_t)k * l], xj[k], s);
      s = warp_sum(s);
      if (lane == 0) xj[i] = -s * rdiag[i];
      __syncwarp();
    }
  }
  __syncthreads();
}

template <bool SMEM>
__global__ void __launch_bounds__(SMALL_THREADS) cholqr_kernel(
    const double* __restrict__ G, int64_t ldg, int l, double nrows, double* __restrict__ Rinv,
    int64_t ldri, double* __restrict__ R, int64_t ldr, double* __restrict__ dinfo, double* gws,
    int use_smem, const int32_t* __restrict__ gate_in, int32_t* __restrict__ gate_out,
    int first_pass) {
  if (gate_in && *gate_in == 0) {
    if (gate_out && threadIdx.x == 0) *gate_out = 0;
    return;
  }
  extern __shared__ __align__(16) double sm[];
  double* H = SMEM ? sm : gws;        // scaled Gram (l x l)
  double* C = H + (size_t)l * l;       // Cholesky factor workspace
  double* X = C + (size_t)l * l;       // inverse
  double* d = X + (size_t)l * l;       // column scales
  double* dr = d + l;                  // their reciprocals (0 for dead columns)
  double* dr2 = dr + l;                // 1 / Rh[j][j]
  __shared__ int s_fail;
  __shared__ double s_defect;
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    const double gii = G[i + (int64_t)i * ldg];
    d[i] = (gii > 0.0) ? sqrt(gii) : 0.0;
    dr[i] = d[i] > 0.0 ? 1.0 / d[i] : 0.0;
  }
  if (threadIdx.x == 0) s_defect = 0.0;
  __syncthreads();
  double loc_def = 0.0;
  for (int64_t t = threadIdx.x; t < (int64_t)l * l; t += blockDim.x) {
    const int j = (int)(t / l), i = (int)(t - (int64_t)j * l);
    double h;
    if (d[i] == 0.0 || d[j] == 0.0) {
      h = (i == j) ? 1.0 : 0.0;
    } else {
      h = G[i + (int64_t)j * ldg] * dr[i] * dr[j];
      loc_def = fmax(loc_def, fabs(h - (i == j ? 1.0 : 0.0)));
    }
    H[t] = h;
  }
  // defect reduction
  {
    __shared__ double red[32];
    double v = warp_max(loc_def);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
      v = warp_max(v);
      if (threadIdx.x == 0) s_defect = v;
    }
    __syncthreads();
  }
  double shift = 0.0;
  int attempt = 0;
  for (;;) {
    for (int64_t t = threadIdx.x; t < (int64_t)l * l; t += blockDim.x) {
      const int j = (int)(t / l), i = (int)(t - (int64_t)j * l);
      C[t] = H[t] + ((i == j) ? shift : 0.0);
    }
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < l; ++j) {
      const double piv = C[j + (int64_t)j * l];
      if (!(piv > 0.0)) {  // uniform decision
        if (threadIdx.x == 0) s_fail = 1;
        __syncthreads();
        break;
      }
      const double rjj = sqrt(piv);
      const double rinv = 1.0 / rjj;
      __syncthreads();
      if (threadIdx.x == 0) dr2[j] = rinv;
      for (int k = j + threadIdx.x; k < l; k += blockDim.x) C[j + (int64_t)k * l] = (k == j) ? rjj : C[j + (int64_t)k * l] * rinv;
      __syncthreads();
      const int rem = l - j - 1;  // rem^2 < 2^31: 32-bit index arithmetic
      for (int t = threadIdx.x; t < rem * rem; t += blockDim.x) {
        const int kk = j + 1 + t / rem, ii = j + 1 + t % rem;
        if (ii <= kk) C[ii + (int64_t)kk * l] -= C[j + (int64_t)ii * l] * C[j + (int64_t)kk * l];
      }
      __syncthreads();
    }
    if (!s_fail) break;
    __syncthreads();
    ++attempt;
    // shifted CholeskyQR (Fukaya et al.): s = 11 (m l + l (l + 1)) u ||H||, ||H|| <= l
    const double base = 11.0 * (nrows * l + (double)l * (l + 1)) * 1.1102230246251565e-16 * l;
    shift = (attempt == 1) ? base : shift * 100.0;
    if (attempt > 8) break;
  }
  // zero the strict lower part, invert
  for (int64_t t = threadIdx.x; t < (int64_t)l * l; t += blockDim.x) {
    const int j = (int)(t / l), i = (int)(t - (int64_t)j * l);
    if (i > j) C[t] = 0.0;
  }
  __syncthreads();
  // X = Rh^-1 by right-looking back substitution: step r scales row r
  // (columns >= r) and subtracts it from the rows above -- one parallel
  // update of r (l - r) entries per step instead of a warp-sequential column
  __shared__ double s_row[1024];
  for (int t = threadIdx.x; t < l * l; t += blockDim.x) {
    const int j = t / l, i = t - j * l;
    X[t] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int r = l - 1; r >= 0; --r) {
    for (int c = r + threadIdx.x; c < l; c += blockDim.x) {
      const double v = X[r + (int64_t)c * l] * dr2[r];
      X[r + (int64_t)c * l] = v;
      s_row[c] = v;
    }
    __syncthreads();
    const int w = l - r;
    for (int t = threadIdx.x; t < r * w; t += blockDim.x) {
      const int c = r + t / r, i = t % r;
      X[i + (int64_t)c * l] = fma(-C[i + (int64_t)r * l], s_row[c], X[i + (int64_t)c * l]);
    }
    __syncthreads();
  }
  // R = Rh D, Rinv = D^-1 Rh^-1; dead columns -> zero rows / columns
  int ndead = 0;
  for (int64_t t = threadIdx.x; t < (int64_t)l * l; t += blockDim.x) {
    const int j = (int)(t / l), i = (int)(t - (int64_t)j * l);
    const bool dead = d[i] == 0.0 || d[j] == 0.0;
    R[i + (int64_t)j * ldr] = dead ? 0.0 : C[t] * d[j];
    Rinv[i + (int64_t)j * ldri] = dead ? 0.0 : X[t] * dr[i];
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < l; ++i) ndead += d[i] == 0.0;
    dinfo[0] = s_defect;
    dinfo[1] = (double)attempt;
    dinfo[2] = (double)ndead;
    dinfo[3] = shift;
    if (s_fail) dinfo[POD_DINFO_BREAKDOWN] = 1.0;  // sticky: the host raises after the round
    if (gate_out) *gate_out = first_pass ? 1 : ((s_defect > 1e-4 || attempt > 0) ? 1 : 0);
  }
}

// cholqr_kernel for 104 < l <= CQI_MAX_L (configs 3 and 4: l = 150, 192),
// where the three l x l buffers no longer fit shared memory and the
// global-memory path runs every elimination step through L2 (~0.74 ms at
// l = 150): here only the factor lives in shared memory, as a packed upper
// triangle (column j holds rows 0..j at j (j + 1) / 2) -- the scaled Gram is
// rebuilt from G for a shifted retry, R is written out before the triangular
// inverse, and the inverse overwrites the factor in place (column r of Rh is
// copied aside before step r updates it).  Same operations in the same
// order as cholqr_kernel, so the same bits.
constexpr int CQI_MAX_L = 230;
static size_t cqi_bytes(int64_t l) { return (size_t)(l * (l + 1) / 2) * 8 + (size_t)3 * l * 8; }
__device__ __forceinline__ int pk(int i, int j) { return (j * (j + 1) >> 1) + i; }  // i <= j

__global__ void __launch_bounds__(SMALL_THREADS) cholqr_inplace_kernel(
    const double* __restrict__ G, int64_t ldg, int l, double nrows, double* __restrict__ Rinv,
    int64_t ldri, double* __restrict__ R, int64_t ldr, double* __restrict__ dinfo,
    const int32_t* __restrict__ gate_in, int32_t* __restrict__ gate_out, int first_pass) {
  if (gate_in && *gate_in == 0) {
    if (gate_out && threadIdx.x == 0) *gate_out = 0;
    return;
  }
  extern __shared__ __align__(16) double sm[];
  const int np = l * (l + 1) / 2;
  double* C = sm;                      // packed upper factor, then its inverse
  double* d = C + np;                  // column scales
  double* dr = d + l;                  // their reciprocals (0 for dead columns)
  double* dr2 = dr + l;                // 1 / Rh[j][j]
  __shared__ int s_fail;
  __shared__ double s_defect;
  __shared__ double s_row[CQI_MAX_L], s_col[CQI_MAX_L], s_piv[3];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    const double gii = G[i + (int64_t)i * ldg];
    d[i] = (gii > 0.0) ? sqrt(gii) : 0.0;
    dr[i] = d[i] > 0.0 ? 1.0 / d[i] : 0.0;
  }
  if (threadIdx.x == 0) s_defect = 0.0;
  __syncthreads();
  // scaled Gram H (+ shift on the diagonal), upper triangle, rebuilt from G
  // for every attempt (G is exactly symmetric: the defect over the upper
  // triangle is the defect over all of H)
  auto build = [&](double shift, bool defect) {
    double loc = 0.0;
#pragma unroll 4
    for (int t = threadIdx.x; t < np; t += blockDim.x) {
      int j = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
      while (j * (j + 1) / 2 > t) --j;
      while ((j + 1) * (j + 2) / 2 <= t) ++j;
      const int i = t - j * (j + 1) / 2;
      double h;
      if (d[i] == 0.0 || d[j] == 0.0) {
        h = (i == j) ? 1.0 : 0.0;
      } else {
        h = G[i + (int64_t)j * ldg] * dr[i] * dr[j];
        loc = fmax(loc, fabs(h - (i == j ? 1.0 : 0.0)));
      }
      C[pk(i, j)] = h + ((i == j) ? shift : 0.0);
    }
    if (defect) {
      __shared__ double red[32];
      double v = warp_max(loc);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x < 32) {
        v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        v = warp_max(v);
        if (threadIdx.x == 0) s_defect = v;
      }
    }
  };
  build(0.0, true);
  double shift = 0.0;
  int attempt = 0;
  for (;;) {
    if (attempt > 0) build(shift, false);
    __syncthreads();
    if (threadIdx.x == 0) {
      s_fail = 0;
      const double p0 = C[0];
      s_piv[0] = p0;
      if (p0 > 0.0) {
        const double q = sqrt(p0);
        s_piv[1] = q;
        s_piv[2] = 1.0 / q;
      }
    }
    __syncthreads();
    for (int j = 0; j < l; ++j) {
      // pivot, its root and reciprocal: formed once (by one lane, beside the
      // previous step's trailing update) instead of by all 32 warps, whose
      // redundant fp64 sqrt + divide sequences kept the FP64 pipe busy
      const double piv = s_piv[0], rjj = s_piv[1], rinv = s_piv[2];
      if (!(piv > 0.0)) {  // uniform decision
        if (threadIdx.x == 0) s_fail = 1;
        __syncthreads();
        break;
      }
      // row j scaled, with a contiguous copy for the trailing update (the
      // pivot itself is stored after the barrier: every thread has read it)
      for (int k = j + 1 + threadIdx.x; k < l; k += blockDim.x) {
        const double v = C[pk(j, k)] * rinv;
        C[pk(j, k)] = v;
        s_row[k] = v;
      }
      __syncthreads();
      if (threadIdx.x == 32) {
        dr2[j] = rinv;
        C[pk(j, j)] = rjj;
      }
      // trailing update, one warp per packed column (rows contiguous across
      // lanes: no index division, no bank conflicts); same operation per
      // entry.  Warp 0 takes only column j + 1 -- the next pivot -- and roots it.
      if (wid == 0) {
        if (lane == 0 && j + 1 < l) {
          const int kk = j + 1;
          double* col = C + (kk * (kk + 1) >> 1);
          col[kk] -= s_row[kk] * s_row[kk];
          const double pn = col[kk];
          s_piv[0] = pn;
          if (pn > 0.0) {
            const double q = sqrt(pn);
            s_piv[1] = q;
            s_piv[2] = 1.0 / q;
          }
        }
      } else {
        for (int kk = j + 1 + wid; kk < l; kk += nwarp - 1) {
          const double ckk = s_row[kk];
          double* col = C + (kk * (kk + 1) >> 1);
          for (int ii = j + 1 + lane; ii <= kk; ii += 32) col[ii] -= s_row[ii] * ckk;
        }
      }
      __syncthreads();
    }
    if (!s_fail) break;
    __syncthreads();
    ++attempt;
    const double base = 11.0 * (nrows * l + (double)l * (l + 1)) * 1.1102230246251565e-16 * l;
    shift = (attempt == 1) ? base : shift * 100.0;
    if (attempt > 8) break;
  }
  // R = Rh D (dead columns -> zero, strict lower part zero) before Rh is inverted
  for (int t = threadIdx.x; t < l * l; t += blockDim.x) {
    const int j = t / l, i = t - j * l;
    const bool dead = d[i] == 0.0 || d[j] == 0.0;
    R[i + (int64_t)j * ldr] = (dead || i > j) ? 0.0 : C[pk(i, j)] * d[j];
  }
  __syncthreads();
  // Rh^-1 in place, right-looking back substitution (cholqr_kernel's steps)
  for (int r = l - 1; r >= 0; --r) {
    for (int i = threadIdx.x; i < r; i += blockDim.x) s_col[i] = C[pk(i, r)];
    for (int c = r + threadIdx.x; c < l; c += blockDim.x) {
      const double v = ((c == r) ? 1.0 : C[pk(r, c)]) * dr2[r];
      C[pk(r, c)] = v;
      s_row[c] = v;
    }
    __syncthreads();
    for (int c = r + wid; c < l; c += nwarp) {  // one warp per packed column
      const double src = s_row[c];
      double* col = C + (c * (c + 1) >> 1);
      for (int i = lane; i < r; i += 32)
        col[i] = fma(-s_col[i], src, (c == r) ? 0.0 : col[i]);
    }
    __syncthreads();
  }
  int ndead = 0;
  for (int t = threadIdx.x; t < l * l; t += blockDim.x) {
    const int j = t / l, i = t - j * l;
    const bool dead = d[i] == 0.0 || d[j] == 0.0;
    Rinv[i + (int64_t)j * ldri] = (dead || i > j) ? 0.0 : C[pk(i, j)] * dr[i];
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < l; ++i) ndead += d[i] == 0.0;
    dinfo[0] = s_defect;
    dinfo[1] = (double)attempt;
    dinfo[2] = (double)ndead;
    dinfo[3] = shift;
    if (s_fail) dinfo[POD_DINFO_BREAKDOWN] = 1.0;
    if (gate_out) *gate_out = first_pass ? 1 : ((s_defect > 1e-4 || attempt > 0) ? 1 : 0);
  }
}

// Register-resident CholeskyQR factor for l <= 64 (the merge rank of
// BASELINE configs 1-2): same contract as cholqr_kernel.  256 threads: thread
// (i = t % 64, q = t / 64) holds row i of the scaled Gram H at columns
// q, q + 4, ..., so a right-looking Cholesky step is one broadcast row (from
// the four threads owning row j, double-buffered in shared memory) and a
// register update -- ONE barrier per step.  Every thread of row i tracks the
// diagonal entry H[i][i] itself, so the next pivot needs no extra exchange.
// Rh^-1 is formed the same way by right-looking back substitution.
constexpr int CQS_L = 64, CQS_T = 256, CQS_G = CQS_T / CQS_L, CQS_U = CQS_L / CQS_G;
constexpr int CQS_S = CQS_L + 1;  // padded row stride of Rh: row reads across lanes hit distinct banks

// 1/sqrt(x) for normal positive x: the MUFU double approximation and two
// Newton steps (the pivot chain's latency: ~8 dependent operations instead
// of an exponent split, an fp32 seed and three Newton steps)
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = -0.5 * x;
  y = y * fma(h, y * y, 1.5);
  y = y * fma(h, y * y, 1.5);
  return y;
}

__global__ void __launch_bounds__(CQS_T) cholqr_small_kernel(
    const double* __restrict__ G, int64_t ldg, int l, double nrows, double* __restrict__ Rinv,
    int64_t ldri, double* __restrict__ R, int64_t ldr, double* Racc, int64_t ldacc,
    double* __restrict__ dinfo, const int32_t* __restrict__ gate_in,
    int32_t* __restrict__ gate_out, int first_pass) {
  if (gate_in && *gate_in == 0) {
    if (gate_out && threadIdx.x == 0) *gate_out = 0;
    return;
  }
  extern __shared__ double racc_s[];        // Racc, column-major racc_s[j * 64 + k] (Racc only)
  __shared__ double d[CQS_L];               // column scales sqrt(G_ii)
  __shared__ double Rs[CQS_L * CQS_S];      // Rh, row-major Rs[j * CQS_S + k] (padded)
  __shared__ double rowbuf[2][2 * CQS_L];   // broadcast row: [Rh row | Y row]
  __shared__ double red[CQS_T / 32];
  __shared__ int s_fail;
  const int t = threadIdx.x, i = t % CQS_L, q = t / CQS_L;
  const bool live_i = i < l;
  __shared__ double dr[CQS_L];  // 1 / d (0 for dead columns)
  if (Racc) {  // stage the old Racc asynchronously; consumed after the factorisation
    for (int e = t; e < l * l; e += CQS_T) {
      const int k = e % l, j = e / l;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&racc_s[j * CQS_L + k]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
                   "l"(Racc + k + (int64_t)j * ldacc)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (t < CQS_L) {
    const double gii = live_i ? G[i + (int64_t)i * ldg] : 0.0;
    const double di = (gii > 0.0) ? sqrt(gii) : 0.0;
    d[t] = di;
    dr[t] = di > 0.0 ? 1.0 / di : 0.0;
  }
  __syncthreads();
  // H = D^-1 G D^-1 (dead columns -> identity); recomputed for a shifted retry
  auto scaled = [&](int j) {
    if (!(live_i && j < l)) return 0.0;
    if (d[i] == 0.0 || d[j] == 0.0) return (i == j) ? 1.0 : 0.0;
    return G[i + (int64_t)j * ldg] * dr[i] * dr[j];
  };
  double loc_def = 0.0;
  double h[CQS_U];
#pragma unroll
  for (int u = 0; u < CQS_U; ++u) {
    const int j = q + CQS_G * u;
    h[u] = scaled(j);
    if (live_i && j < l && d[i] != 0.0 && d[j] != 0.0)
      loc_def = fmax(loc_def, fabs(h[u] - (i == j ? 1.0 : 0.0)));
  }
  {
    const double v = warp_max(loc_def);
    if ((t & 31) == 0) red[t >> 5] = v;
  }
  __syncthreads();
  double defect = 0.0;
  for (int w = 0; w < CQS_T / 32; ++w) defect = fmax(defect, red[w]);
  double shift = 0.0;
  int attempt = 0;
  // Y = Rh^-T is formed by the same elimination: the steps applied to
  // [H | I] leave [Rh | Rh^-T] (thread (i, q) keeps row i of Y at its
  // columns), so no separate back substitution is needed
  double y[CQS_U];
  for (;;) {
    double dg = 0.0;  // this row's diagonal entry, tracked by all CQS_G threads of the row
    if (attempt) {  // shifted retry: rebuild the scaled rows
#pragma unroll
      for (int u = 0; u < CQS_U; ++u) {
        const int j = q + CQS_G * u;
        h[u] = scaled(j) + ((i == j && live_i) ? shift : 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < CQS_U; ++u) y[u] = (q + CQS_G * u == i) ? 1.0 : 0.0;
    if (live_i) dg = scaled(i) + shift;
    if (t == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < l; ++j) {
      double* rb = rowbuf[j & 1];
      // the owners of row j publish it scaled by 1 / r_jj; a non-positive
      // pivot only raises the flag (checked once after the loop) and keeps
      // every value finite.  Branch-free row work: entries left of the
      // diagonal are computed too but never read as results.
      if (i == j) {
        // pivots below 1e-290 count as breakdown (shifted retry), so the
        // flush-to-zero approximation never sees a subnormal
        const bool ok = dg > 1e-290;
        if (!ok && q == 0) s_fail = 1;
        const double inv = ok ? rsqrt_fast(dg) : 0.0;  // 1 / r_jj
        const double rjj = dg * inv;
#pragma unroll
        for (int u = 0; u < CQS_U; ++u) {
          const int c = q + CQS_G * u;
          const double v = (c == j) ? rjj : h[u] * inv;
          y[u] *= inv;
          rb[c] = v;
          rb[CQS_L + c] = y[u];
          Rs[j * CQS_S + c] = v;
        }
      }
      __syncthreads();
      if (i > j) {
        const double mi = rb[i];
        dg = fma(-mi, mi, dg);
#pragma unroll
        for (int u = 0; u < CQS_U; ++u) {
          const double rv = rb[q + CQS_G * u];
          h[u] = fma(-mi, rv, h[u]);
          y[u] = fma(-mi, rb[CQS_L + q + CQS_G * u], y[u]);
        }
      }
    }
    __syncthreads();
    if (!s_fail) break;
    __syncthreads();  // every thread has read s_fail before the retry resets it
    ++attempt;
    // shifted CholeskyQR (Fukaya et al.): s = 11 (m l + l (l + 1)) u ||H||, ||H|| <= l
    const double base = 11.0 * (nrows * l + (double)l * (l + 1)) * 1.1102230246251565e-16 * l;
    shift = (attempt == 1) ? base : shift * 100.0;
    if (attempt > 8) break;
  }
  // R = Rh D, Rinv = D^-1 Rh^-1 = D^-1 Y^T; dead columns -> zero rows / columns
  auto rk = [&](int a, int b) {  // R[a][b]
    return (d[a] == 0.0 || d[b] == 0.0 || b < a) ? 0.0 : Rs[a * CQS_S + b] * d[b];
  };
  if (live_i) {
#pragma unroll
    for (int u = 0; u < CQS_U; ++u) {
      const int j = q + CQS_G * u;
      if (j >= l) continue;
      const bool dead = d[i] == 0.0 || d[j] == 0.0;
      if (R) R[i + (int64_t)j * ldr] = rk(i, j);
      // thread (i, q) holds Y[i][j] = Rh^-1[j][i]
      Rinv[j + (int64_t)i * ldri] = (dead || j > i) ? 0.0 : y[u] * dr[j];
    }
  }
  if (Racc) {  // Racc <- R Racc (both upper triangular), in place
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double acc[CQS_U];
#pragma unroll
    for (int u = 0; u < CQS_U; ++u) acc[u] = 0.0;
    if (live_i) {
      for (int k = i; k < l; ++k) {
        const double a = rk(i, k);
#pragma unroll
        for (int u = 0; u < CQS_U; ++u) {
          const int j = q + CQS_G * u;
          acc[u] = fma((k <= j) ? a : 0.0, racc_s[j * CQS_L + k], acc[u]);
        }
      }
    }
    if (live_i) {
#pragma unroll
      for (int u = 0; u < CQS_U; ++u) {
        const int j = q + CQS_G * u;
        if (j < l) Racc[i + (int64_t)j * ldacc] = acc[u];
      }
    }
  }
  if (t == 0) {
    int ndead = 0;
    for (int k = 0; k < l; ++k) ndead += d[k] == 0.0;
    dinfo[0] = defect;
    dinfo[1] = (double)attempt;
    dinfo[2] = (double)ndead;
    dinfo[3] = shift;
    if (s_fail) dinfo[POD_DINFO_BREAKDOWN] = 1.0;  // sticky: the host raises after the round
    if (gate_out) *gate_out = first_pass ? 1 : ((defect > 1e-4 || attempt > 0) ? 1 : 0);
  }
}

// ----------------------------------------------------- small GEMM / max --
// C (p x q) = alpha * op(A) B + beta * C, op(A) = A (p x k) or A^T (A is k x p)
__global__ void small_gemm_kernel(int p, int q, int k, double alpha, const double* __restrict__ A,
                                  int64_t lda, int transa, const double* __restrict__ B,
                                  int64_t ldb, double beta, double* C, int64_t ldc,
                                  const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int64_t tot = (int64_t)p * q;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(t / p), i = (int)(t - (int64_t)j * p);
    double s = 0.0;
    for (int kk = 0; kk < k; ++kk) {
      const double a = transa ? A[kk + (int64_t)i * lda] : A[i + (int64_t)kk * lda];
      s = fma(a, B[kk + (int64_t)j * ldb], s);
    }
    double v = alpha * s;
    if (beta != 0.0) v += beta * C[i + (int64_t)j * ldc];
    C[i + (int64_t)j * ldc] = v;
  }
}

__global__ void small_copy_kernel(int p, int q, const double* __restrict__ src, int64_t lds,
                                  double* __restrict__ dst, int64_t ldd,
                                  const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int64_t tot = (int64_t)p * q;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(t / p), i = (int)(t - (int64_t)j * p);
    dst[i + (int64_t)j * ldd] = src[i + (int64_t)j * lds];
  }
}

__global__ void maxabs_kernel(const double* __restrict__ A, int64_t lda, int p, int q, double thr,
                              double* __restrict__ out, int32_t* __restrict__ gate_out) {
  __shared__ double red[32];
  double v = 0.0;
  for (int64_t t = threadIdx.x; t < (int64_t)p * q; t += blockDim.x) {
    const int j = (int)(t / p), i = (int)(t - (int64_t)j * p);
    v = fmax(v, fabs(A[i + (int64_t)j * lda]));
  }
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    v = warp_max(v);
    if (threadIdx.x == 0) {
      if (out) out[0] = v;
      if (gate_out) *gate_out = (v > thr) ? 1 : 0;
    }
  }
}

// Raise a kernel's dynamic shared-memory limit once to the maximum any call
// needs (kept host-side so launches inside CUDA-graph capture make no
// attribute calls).
static int set_smem(const void* fn, size_t bytes) {
  static const void* fns[16];
  static size_t done[16];
  static int nf = 0;
  int i = 0;
  for (; i < nf; ++i)
    if (fns[i] == fn) break;
  if (i < nf && done[i] >= bytes) return POD_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMALL_SMEM_CAP);
  if (e != cudaSuccess) return cuda_status(e, "small smem attr");
  if (i == nf && nf < 16) { fns[nf] = fn; ++nf; }
  if (i < 16) done[i] = SMALL_SMEM_CAP;
  return POD_OK;
}

// POD_CHOLQR_SMALL=0: the general CholeskyQR kernel for l <= 64 too (A/B)
static bool cqs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_CHOLQR_SMALL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static size_t cholqr_bytes(int64_t l) { return (size_t)3 * l * l * 8 + (size_t)3 * l * 8 + 64; }
// POD_CHOLQR_INPLACE=0: the global-memory factor for 104 < l <= 230 too (A/B)
static bool cqi_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_CHOLQR_INPLACE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int bj_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                  int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                  int64_t ldt, int64_t tcols, double* sig_new, int64_t* info, const int32_t* gate,
                  bool probe, cudaStream_t stream);
int bj_gram_eigh(const double* X, const int* piv, const int64_t* rank, int64_t g, int64_t r,
                 double* sigma, double* T, int64_t ldt, int64_t* info, cudaStream_t stream);
int bj_svd(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
           double* sigma, double* V, int64_t ldv, int64_t* info, cudaStream_t stream);
int cj_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                  int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                  int64_t ldt, int64_t tcols, double* sig_new, int64_t* info, const int32_t* gate,
                  cudaStream_t stream);
int cj_gram_eigh(const double* X, const int* piv, const int64_t* rank, int64_t g, int64_t r,
                 double* sigma, double* T, int64_t ldt, int64_t* info, cudaStream_t stream);
int cj_svd(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
           double* sigma, double* V, int64_t ldv, int64_t* info, cudaStream_t stream);
bool cj_fits(int64_t nc, int64_t nr, int64_t njr);
size_t gj_ws_bytes(int64_t n, int64_t nrows, int64_t njrows);
size_t gj_gram_large_ws_bytes(int64_t g);
int gj_gram_eigh_large(const double* G, int64_t ldg, int64_t g, int64_t r, double* sigma,
                       double* T, int64_t ldt, int64_t* info, void* ws, size_t ws_bytes,
                       cudaStream_t s);
int gj_pivchol(const double* G, int64_t ldg, int64_t g, void* ws, size_t ws_bytes, double** Xo,
               int** pivo, int64_t** ranko, void** rest, size_t* rest_bytes, cudaStream_t s);
int gj_gram_eigh(const double* X, int64_t ldx, const int* piv, const int64_t* rank, int64_t g,
                 int64_t r, double* sigma, double* T, int64_t ldt, int64_t* info, void* ws,
                 size_t ws_bytes, cudaStream_t s);
int gj_svd(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
           double* sigma, double* V, int64_t ldv, int64_t* info, void* ws, size_t ws_bytes,
           cudaStream_t s);
int gj_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                  int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                  int64_t ldt, int64_t tcols, double* sig_new, int64_t* info, void* ws,
                  size_t ws_bytes, cudaStream_t s);

}  // namespace pod

using namespace pod;

static size_t gram_ws_bytes(int64_t g) {
  // X (g x g) + piv (g int) + rank, then the pivoted Cholesky's matrix when
  // it does not fit in shared memory
  return (size_t)g * g * 8 + (size_t)g * 4 + 64 + 2 * (size_t)g * g * 8;
}

// Solver routing by size: block Jacobi on one cluster (block_jacobi.cu),
// then the row-distributed cluster solver (cluster_jacobi.cu), then the
// grid-wide solver with L2-resident blocks (grid_jacobi.cu), whose block
// sets live in the caller's workspace.  Gram eigensolves beyond g = 512 skip
// the pivoted Cholesky and run one-sided Jacobi on G itself.
constexpr int64_t PIVCHOL_MAX_G = 512;

// the single-CTA pivoted Cholesky keeps its packed triangle in shared memory
// up to this order; beyond it the grid-wide one (gpivchol) runs
static bool pivchol_in_smem(int64_t g) { return (size_t)g * (g + 1) / 2 * 8 <= SMALL_SMEM_CAP; }
// order from which the grid-wide pivoted Cholesky replaces the single-CTA
// global-memory one (POD_GRID_PIVCHOL_MIN overrides)
static int64_t grid_pivchol_min() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("POD_GRID_PIVCHOL_MIN");
    v = e ? atoll(e) : 300;
  }
  return v;
}

static size_t gram_total_ws(int64_t g) {
  const size_t small = gram_ws_bytes(g) + gj_ws_bytes(g, g, 0);
  if (!pivchol_in_smem(g)) return std::max(small, gj_gram_large_ws_bytes(g));
  return small;
}

extern "C" size_t pod_small_ws_bytes(int64_t n) {
  return std::max(std::max(gram_total_ws(n), cholqr_bytes(n) + (size_t)n * n * 8),
                  std::max(gj_ws_bytes(n, n, n), gj_ws_bytes(n, n, 0)));
}

extern "C" int64_t pod_gram_eigh_max_g(void) {
  static int64_t v = 0;
  if (!v) {  // feasibility is monotone in g: bisect on the grid solver's fit
    int64_t lo = PIVCHOL_MAX_G, hi = 1 << 16;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) / 2;
      (gj_gram_large_ws_bytes(mid) ? lo : hi) = mid;
    }
    v = lo;
  }
  return v;
}

extern "C" size_t pod_svd_small_ws_bytes(int64_t nr, int64_t nc, int withv) {
  if (nr < 1 || nc < 1) return 0;
  return gj_ws_bytes(nc, nr, withv ? nc : 0);
}

extern "C" int pod_gram_eigh(const double* G, int64_t ldg, int64_t g, int64_t r, double* sigma,
                             double* T, int64_t ldt, int64_t* info, void* ws, size_t ws_bytes,
                             void* stream) {
  POD_REQUIRE(g >= 1 && r >= 1 && ldg >= g && ldt >= g, "pod_gram_eigh: bad shape");
  POD_REQUIRE(ws_bytes >= gram_total_ws(g), "pod_gram_eigh: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (g > PIVCHOL_MAX_G)
    return gj_gram_eigh_large(G, ldg, g, r, sigma, T, ldt, info, ws, ws_bytes, s);
  double* X = (double*)ws;
  int* piv = (int*)(X + (size_t)g * g);
  int64_t* rank = (int64_t*)(((uintptr_t)(piv + g) + 15) & ~(uintptr_t)15);
  double* scratch = (double*)(((uintptr_t)(rank + 1) + 15) & ~(uintptr_t)15);
  const size_t bytes = (size_t)g * (g + 1) / 2 * 8;  // packed lower triangle
  void* jws = (char*)ws + gram_ws_bytes(g);
  size_t jws_bytes = ws_bytes - gram_ws_bytes(g);
  if (!pivchol_in_smem(g) && g >= grid_pivchol_min()) {  // grid-wide pivoted Cholesky
    int st = gj_pivchol(G, ldg, g, ws, ws_bytes, &X, &piv, &rank, &jws, &jws_bytes, s);
    if (st) return st;
  } else if (!pivchol_in_smem(g)) {  // one CTA, Schur complement in global memory
    pivchol_kernel<false, 16><<<1, PIVCHOL_THREADS, 0, s>>>(G, ldg, (int)g, X, piv, rank,
                                                            scratch, scratch + (size_t)g * g);
    POD_CHECK_LAUNCH("pivoted cholesky");
  } else {
    if (g <= 128) {
      int st = set_smem((const void*)pivchol_kernel<true, 4>, bytes);
      if (st) return st;
      pivchol_kernel<true, 4><<<1, PIVCHOL_THREADS, bytes, s>>>(G, ldg, (int)g, X, piv, rank,
                                                                scratch, scratch + (size_t)g * g);
    } else {  // g <= 225 here
      int st = set_smem((const void*)pivchol_kernel<true, 8>, bytes);
      if (st) return st;
      pivchol_kernel<true, 8><<<1, PIVCHOL_THREADS, bytes, s>>>(G, ldg, (int)g, X, piv, rank,
                                                                scratch, scratch + (size_t)g * g);
    }
    POD_CHECK_LAUNCH("pivoted cholesky");
  }
  {
    const int bst = bj_gram_eigh(X, piv, rank, g, r, sigma, T, ldt, info, s);
    if (bst != -1) return bst;  // -1: size not handled by the block solver
  }
  if (cj_fits(g, g, 0)) return cj_gram_eigh(X, piv, rank, g, r, sigma, T, ldt, info, s);
  return gj_gram_eigh(X, g, piv, rank, g, r, sigma, T, ldt, info, jws, jws_bytes, s);
}

extern "C" int pod_cholqr_factor(const double* G, int64_t ldg, int64_t l, int64_t nrows,
                                 double* Rinv, int64_t ldri, double* R, int64_t ldr, double* dinfo,
                                 void* ws, size_t ws_bytes, const int32_t* gate_in,
                                 int32_t* gate_out, int first_pass, void* stream) {
  return pod_cholqr_factor2(G, ldg, l, nrows, Rinv, ldri, R, ldr, nullptr, 1, dinfo, ws, ws_bytes,
                            gate_in, gate_out, first_pass, stream);
}

extern "C" int pod_cholqr_factor2(const double* G, int64_t ldg, int64_t l, int64_t nrows,
                                  double* Rinv, int64_t ldri, double* R, int64_t ldr,
                                  double* Racc, int64_t ldacc, double* dinfo, void* ws,
                                  size_t ws_bytes, const int32_t* gate_in, int32_t* gate_out,
                                  int first_pass, void* stream) {
  POD_REQUIRE(l >= 1 && ldg >= l && ldri >= l && ldr >= l && (!Racc || ldacc >= l),
              "pod_cholqr_factor: bad shape");
  POD_REQUIRE(R || Racc, "pod_cholqr_factor: no R output");
  cudaStream_t st = (cudaStream_t)stream;
  if (l <= CQS_L && cqs_enabled()) {
    const size_t dyn = Racc ? sizeof(double) * CQS_L * CQS_L : 0;
    static bool dyn_set = false;
    if (dyn && !dyn_set) {
      cudaError_t e = cudaFuncSetAttribute((const void*)cholqr_small_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return cuda_status(e, "cholqr small smem attr");
      dyn_set = true;
    }
    cholqr_small_kernel<<<1, CQS_T, dyn, st>>>(G, ldg, (int)l, (double)nrows, Rinv, ldri, R, ldr,
                                             Racc, ldacc, dinfo, gate_in, gate_out, first_pass);
    POD_CHECK_LAUNCH("cholqr small");
    return POD_OK;
  }
  POD_REQUIRE(R, "pod_cholqr_factor: l = %lld > 64 needs the R output", (long long)l);
  POD_REQUIRE(l <= 1024, "pod_cholqr_factor: l = %lld exceeds 1024", (long long)l);
  const size_t bytes = cholqr_bytes(l);
  const int use_smem = bytes <= SMALL_SMEM_CAP;
  if (!use_smem && l <= CQI_MAX_L && cqi_enabled()) {  // factor alone in shared memory
    static bool attr = false;  // up to 218 KB: above set_smem's 200 KB cap
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute((const void*)cholqr_inplace_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)cqi_bytes(CQI_MAX_L));
      if (e != cudaSuccess) return cuda_status(e, "cholqr in place smem attr");
      attr = true;
    }
    static int cqi_threads = 0;
    if (!cqi_threads) {  // POD_CQI_THREADS: A/B of the CTA width (multiple of 32, 64..1024)
      const char* e = getenv("POD_CQI_THREADS");
      const int v = e ? atoi(e) : 0;
      cqi_threads = (v >= 64 && v <= SMALL_THREADS && v % 32 == 0) ? v : SMALL_THREADS;
    }
    cholqr_inplace_kernel<<<1, cqi_threads, cqi_bytes(l), st>>>(
        G, ldg, (int)l, (double)nrows, Rinv, ldri, R, ldr, dinfo, gate_in, gate_out, first_pass);
    POD_CHECK_LAUNCH("cholqr in place");
  } else {
  POD_REQUIRE(use_smem || ws_bytes >= bytes, "pod_cholqr_factor: workspace too small");
  if (use_smem) { int st = set_smem((const void*)cholqr_kernel<true>, bytes); if (st) return st; }
  if (use_smem)
    cholqr_kernel<true><<<1, SMALL_THREADS, use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      G, ldg, (int)l, (double)nrows, Rinv, ldri, R, ldr, dinfo, (double*)ws, use_smem, gate_in,
      gate_out, first_pass);
  else
    cholqr_kernel<false><<<1, SMALL_THREADS, use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      G, ldg, (int)l, (double)nrows, Rinv, ldri, R, ldr, dinfo, (double*)ws, use_smem, gate_in,
      gate_out, first_pass);
  POD_CHECK_LAUNCH("cholqr");
  }
  if (Racc) {  // Racc <- R Racc through the workspace's tail (general path)
    POD_REQUIRE(ws_bytes >= cholqr_bytes(l) + (size_t)l * l * 8, "pod_cholqr_factor: workspace");
    double* tmp = (double*)((char*)ws + cholqr_bytes(l));
    int blocks = (int)std::min<int64_t>(ceil_div(l * l, 256), 1024);
    small_gemm_kernel<<<blocks, 256, 0, st>>>((int)l, (int)l, (int)l, 1.0, R, ldr, 0, Racc, ldacc,
                                              0.0, tmp, l, gate_in);
    small_copy_kernel<<<blocks, 256, 0, st>>>((int)l, (int)l, tmp, l, Racc, ldacc, gate_in);
    POD_CHECK_LAUNCH("cholqr accumulate");
  }
  return POD_OK;
}


extern "C" int pod_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm,
                              const double* R, int64_t ldr, const double* sig2, int64_t l2,
                              int64_t r, int64_t rcap, double* T, int64_t ldt, int64_t tcols,
                              double* sig_new, int64_t* info, void* ws, size_t ws_bytes,
                              void* stream) {
  POD_REQUIRE(l1 >= 1 && l2 >= 1 && r >= 1 && rcap >= l1 && ldt >= rcap + l2 && tcols >= 1,
              "pod_merge_core: bad shape");
  const int bst = bj_merge_core(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols,
                                sig_new, info, nullptr, false, (cudaStream_t)stream);
  if (bst != -1) return bst;  // -1: size not handled by the block solver
  if (cj_fits(l1 + l2, l1 + l2, 0))
    return cj_merge_core(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols, sig_new,
                         info, nullptr, (cudaStream_t)stream);
  return gj_merge_core(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols, sig_new, info,
                       ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int pod_merge_core_gatable(int64_t l1, int64_t l2) {
  if (l1 < 1 || l2 < 1) return 0;
  if (bj_merge_core(nullptr, l1, nullptr, 0, nullptr, 0, nullptr, l2, 1, l1, nullptr, l1 + l2, 1,
                    nullptr, nullptr, nullptr, true, nullptr) == POD_OK)
    return 1;
  return cj_fits(l1 + l2, l1 + l2, 0) ? 1 : 0;
}

extern "C" int pod_merge_core_gated(const double* sig1, int64_t l1, const double* M, int64_t ldm,
                                    const double* R, int64_t ldr, const double* sig2, int64_t l2,
                                    int64_t r, int64_t rcap, double* T, int64_t ldt,
                                    int64_t tcols, double* sig_new, int64_t* info,
                                    const int32_t* gate, void* stream) {
  POD_REQUIRE(l1 >= 1 && l2 >= 1 && r >= 1 && rcap >= l1 && ldt >= rcap + l2 && tcols >= 1,
              "pod_merge_core_gated: bad shape");
  POD_REQUIRE(pod_merge_core_gatable(l1, l2),
              "pod_merge_core_gated: l1 + l2 = %lld needs the grid solver (not gatable)",
              (long long)(l1 + l2));
  const int bst = bj_merge_core(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols,
                                sig_new, info, gate, false, (cudaStream_t)stream);
  if (bst != -1) return bst;
  return cj_merge_core(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols, sig_new, info,
                       gate, (cudaStream_t)stream);
}

extern "C" int pod_svd_small(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U,
                             int64_t ldu, double* sigma, double* V, int64_t ldv, int64_t* info,
                             void* ws, size_t ws_bytes, void* stream) {
  POD_REQUIRE(nr >= 1 && nc >= 1 && lda >= nr && nr >= nc, "pod_svd_small: bad shape");
  const int bst = bj_svd(A, lda, nr, nc, U, ldu, sigma, V, ldv, info, (cudaStream_t)stream);
  if (bst != -1) return bst;  // -1: size not handled by the block solver
  if (cj_fits(nc, nr, V ? nc : 0))
    return cj_svd(A, lda, nr, nc, U, ldu, sigma, V, ldv, info, (cudaStream_t)stream);
  return gj_svd(A, lda, nr, nc, U, ldu, sigma, V, ldv, info, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int pod_small_gemm(int64_t p, int64_t q, int64_t k, double alpha, const double* A,
                              int64_t lda, int transa, const double* B, int64_t ldb, double beta,
                              double* C, int64_t ldc, const int32_t* gate, void* stream) {
  POD_REQUIRE(p >= 0 && q >= 0 && k >= 0, "pod_small_gemm: bad shape");
  if (p == 0 || q == 0) return POD_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(p * q, 256), 1024);
  small_gemm_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((int)p, (int)q, (int)k, alpha, A,
                                                                lda, transa, B, ldb, beta, C, ldc,
                                                                gate);
  POD_CHECK_LAUNCH("small_gemm");
  return POD_OK;
}

extern "C" int pod_small_copy(int64_t p, int64_t q, const double* src, int64_t lds, double* dst,
                              int64_t ldd, const int32_t* gate, void* stream) {
  POD_REQUIRE(p >= 0 && q >= 0, "pod_small_copy: bad shape");
  if (p == 0 || q == 0) return POD_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(p * q, 256), 1024);
  small_copy_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((int)p, (int)q, src, lds, dst, ldd,
                                                                gate);
  POD_CHECK_LAUNCH("small_copy");
  return POD_OK;
}

extern "C" int pod_maxabs(const double* A, int64_t lda, int64_t p, int64_t q, double thr,
                          double* out, int32_t* gate_out, void* stream) {
  POD_REQUIRE(p >= 0 && q >= 0, "pod_maxabs: bad shape");
  maxabs_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(A, lda, (int)p, (int)q, thr, out, gate_out);
  POD_CHECK_LAUNCH("maxabs");
  return POD_OK;
}

