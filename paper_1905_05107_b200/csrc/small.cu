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

// fp64 1/sqrt(x) from an fp32 seed and two Newton steps (rel. err ~1e-16).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = (double)rsqrtf((float)x);
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  return y;
}

constexpr int JAC_MAX_PAIRS = 256;  // nc <= 512

struct JacScratch {
  double gam[JAC_MAX_PAIRS], cs[JAC_MAX_PAIRS], sn[JAC_MAX_PAIRS];
  short a[JAC_MAX_PAIRS], b[JAC_MAX_PAIRS], map[2 * JAC_MAX_PAIRS];
  int rotated;
};
// One static scratch block per CTA, shared by every Jacobi instantiation.
__device__ __forceinline__ JacScratch& jac_scratch() {
  __shared__ JacScratch js;
  return js;
}

// Rotation (c, s) annihilating gamma for squared norms al, be (exact fp64
// angle: t = sign(z) / (|z| + sqrt(1 + z^2)), z = (be - al) / (2 gamma)).
__device__ __forceinline__ void jacobi_rotation(double al, double be, double ga, double& cs,
                                                double& sn) {
  const double zeta = (be - al) / (2.0 * ga);
  const double az = fabs(zeta);
  double t = (az < 1e150) ? 1.0 / (az + sqrt(fma(az, az, 1.0))) : 0.5 / az;
  t = copysign(t, zeta);
  cs = rsqrt_nr(fma(t, t, 1.0));
  sn = cs * t;
}

// One-sided cyclic Jacobi on the columns of W (nr x nc, ld ldw); J (nc x nc,
// ld ldj) is rotated alongside when non-null.  Round-robin (circle method)
// ordering: each step rotates nc/2 disjoint column pairs in three phases:
//   1. dots   -- one 16-lane group per pair loads its two columns (into
//                registers when KREG > 0) and computes gamma = w_a . w_b
//   2. params -- one thread per pair: rotation test gamma^2 > tol^2 a b,
//                (c, s) from jacobi_rotation, squared norms updated by the
//                exact 2x2 congruence
//   3. update -- each group rotates its two columns (from registers) and
//                writes them back once.
// The step is bound by shared-memory bandwidth (2 n^2 doubles moved per
// step with register-resident columns).  Squared norms are recomputed
// exactly at the start of each sweep.  Returns sweeps.
template <int KREG>
__device__ __forceinline__ int jacobi_one_sided_t(double* W, int ldw, int nr, int nc, double* J,
                                                  int ldj, double tol, int max_sweeps,
                                                  double* nrm2) {
  JacScratch& js = jac_scratch();
  double* s_gam = js.gam;
  double* s_cs = js.cs;
  double* s_sn = js.sn;
  short* s_a = js.a;
  short* s_b = js.b;
  short* s_map = js.map;
  int& rotated = js.rotated;
  if (nc < 2) return 0;
  const int N = nc + (nc & 1);
  const int M1 = N - 1;
  const int npairs = N / 2;
  const int ngroups = blockDim.x >> 4;
  const int grp = threadIdx.x >> 4, gl = threadIdx.x & 15;
  const unsigned hmask = 0xffffu << (16 * ((threadIdx.x >> 4) & 1));
  const double tol2 = tol * tol;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double xa[KREG > 0 ? KREG : 1], xb[KREG > 0 ? KREG : 1];
  if (N > nc && threadIdx.x == 0) s_map[nc] = (short)nc;  // dummy position
  int sweep = 0;
  while (sweep < max_sweeps) {
    for (int j = warp; j < nc; j += nw) {
      const double* w = W + (int64_t)j * ldw;
      double s = 0.0;
      for (int i = lane; i < nr; i += 32) s = fma(w[i], w[i], s);
      s = warp_sum(s);
      if (lane == 0) nrm2[j] = s;
    }
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    // de Rijk ordering: position k holds the column with the k-th largest norm
    for (int j = threadIdx.x; j < nc; j += blockDim.x) {
      const double kj = nrm2[j];
      int rk = 0;
      for (int i = 0; i < nc; ++i) {
        const double ki = nrm2[i];
        rk += (ki > kj) || (ki == kj && i < j);
      }
      s_map[rk] = (short)j;
    }
    __syncthreads();
    for (int step = 0; step < M1; ++step) {
      // phase 1: pair indices + dot products
      for (int pr = grp; pr < npairs; pr += ngroups) {
        int a, b;
        if (pr == 0) {
          a = 0;
          b = 1 + step;
        } else {
          a = step + pr;
          a = (a >= M1 ? a - M1 : a) + 1;
          b = step - pr + M1;
          b = (b >= M1 ? b - M1 : b) + 1;
        }
        if (a > b) { const int t = a; a = b; b = t; }
        a = s_map[a];
        b = s_map[b];  // the dummy position maps to column nc (skipped)
        double ga = 0.0;
        if (b < nc && a < nc) {
          const double* wa = W + (int64_t)a * ldw;
          const double* wb = W + (int64_t)b * ldw;
          if (KREG > 0) {
#pragma unroll
            for (int k = 0; k < (KREG > 0 ? KREG : 1); ++k) {
              const int i = gl + 16 * k;
              xa[k] = (i < nr) ? wa[i] : 0.0;
              xb[k] = (i < nr) ? wb[i] : 0.0;
              ga = fma(xa[k], xb[k], ga);
            }
          } else {
            for (int i = gl; i < nr; i += 16) ga = fma(wa[i], wb[i], ga);
          }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) ga += __shfl_xor_sync(hmask, ga, o);
        }
        if (gl == 0) {
          s_gam[pr] = ga;
          s_a[pr] = (short)a;
          s_b[pr] = (short)b;
        }
      }
      __syncthreads();
      // phase 2: rotation parameters, one thread per pair
      for (int pr = threadIdx.x; pr < npairs; pr += blockDim.x) {
        const int a = s_a[pr], b = s_b[pr];
        double cs = 1.0, sn = 0.0;
        if (b < nc && a < nc) {
          const double ga = s_gam[pr];
          const double al = nrm2[a], be = nrm2[b];
          if (ga * ga > tol2 * al * be && al > 0.0 && be > 0.0) {
            jacobi_rotation(al, be, ga, cs, sn);
            const double c2 = cs * cs, s2 = sn * sn, cs2g = 2.0 * cs * sn * ga;
            nrm2[a] = fmax(fma(c2, al, fma(s2, be, -cs2g)), 0.0);
            nrm2[b] = fma(s2, al, fma(c2, be, cs2g));
            rotated = 1;
          }
        }
        s_cs[pr] = cs;
        s_sn[pr] = sn;
      }
      __syncthreads();
      // phase 3: rotate the column pairs (and J)
      for (int pr = grp; pr < npairs; pr += ngroups) {
        const double sn = s_sn[pr];
        if (sn == 0.0) continue;
        const double cs = s_cs[pr];
        const int a = s_a[pr], b = s_b[pr];
        double* wa = W + (int64_t)a * ldw;
        double* wb = W + (int64_t)b * ldw;
        if (KREG > 0) {
#pragma unroll
          for (int k = 0; k < (KREG > 0 ? KREG : 1); ++k) {
            const int i = gl + 16 * k;
            if (i < nr) {
              wa[i] = fma(cs, xa[k], -sn * xb[k]);
              wb[i] = fma(sn, xa[k], cs * xb[k]);
            }
          }
        } else {
          for (int i = gl; i < nr; i += 16) {
            const double x = wa[i], y = wb[i];
            wa[i] = fma(cs, x, -sn * y);
            wb[i] = fma(sn, x, cs * y);
          }
        }
        if (J) {
          double* ja = J + (int64_t)a * ldj;
          double* jb = J + (int64_t)b * ldj;
          for (int i = gl; i < nc; i += 16) {
            const double x = ja[i], y = jb[i];
            ja[i] = fma(cs, x, -sn * y);
            jb[i] = fma(sn, x, cs * y);
          }
        }
      }
      __syncthreads();
    }
    ++sweep;
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  return sweep;
}

// Dispatch on the per-lane register footprint (register path needs one pair
// per 16-lane group, i.e. nc <= 2 * blockDim.x / 16).
__device__ __forceinline__ int jacobi_one_sided(double* W, int ldw, int nr, int nc, double* J,
                                                int ldj, double tol, int max_sweeps,
                                                double* nrm2) {
  const int npairs = (nc + 1) / 2;
  if (npairs <= (int)(blockDim.x >> 4)) {
    if (nr <= 64) return jacobi_one_sided_t<4>(W, ldw, nr, nc, J, ldj, tol, max_sweeps, nrm2);
    if (nr <= 128) return jacobi_one_sided_t<8>(W, ldw, nr, nc, J, ldj, tol, max_sweeps, nrm2);
  }
  return jacobi_one_sided_t<0>(W, ldw, nr, nc, J, ldj, tol, max_sweeps, nrm2);
}

// Column 2-norms of W into nrm[0..nc) (warp per column, fixed order).
__device__ __forceinline__ void column_norms(const double* W, int ldw, int nr, int nc, double* nrm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < nc; j += nw) {
    double s = 0.0;
    for (int i = lane; i < nr; i += 32) {
      const double x = W[i + (int64_t)j * ldw];
      s = fma(x, x, s);
    }
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
}

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

__device__ __forceinline__ double jacobi_tol(int nr) { return 2.220446049250313e-16 * (double)max(nr, 16); }

// ---------------------------------------------------------- gram eigh ----
// G (PSD, g x g) -> pivoted Cholesky  P G P^T = R^T R  (stops when the
// largest remaining diagonal <= 1e-15 max diag; the neglected block is far
// below the 1e-12 lambda_1 dust rule) -> one-sided Jacobi on the columns of
// R^T (in place, lower triangle): R^T J = V' Sigma, so the normalised
// columns are eigenvectors of P G P^T and lambda = ||col||^2.  Convergence
// is that of an SVD of the sampled block (no squared condition number).
template <bool SMEM>
__global__ void __launch_bounds__(SMALL_THREADS) gram_eigh_kernel(
    const double* __restrict__ G, int64_t ldg, int g, int r, double* __restrict__ sigma_out,
    double* __restrict__ T, int64_t ldt, int64_t* __restrict__ info, double* gws, int use_smem,
    int max_sweeps) {
  extern __shared__ __align__(16) double sm[];
  double* W = SMEM ? sm : gws;
  double* nrm = W + (size_t)g * g;
  double* sig = nrm + g;
  int* perm = reinterpret_cast<int*>(sig + g);
  int* piv = perm + g;
  __shared__ double s_dmax0, s_red[32];
  __shared__ int s_ired[32], s_rank;
  for (int64_t t = threadIdx.x; t < (int64_t)g * g; t += blockDim.x) {
    const int64_t j = t / g, i = t - j * g;
    W[t] = G[i + j * ldg];
  }
  for (int i = threadIdx.x; i < g; i += blockDim.x) piv[i] = i;
  __syncthreads();
  // --- pivoted Cholesky (upper R stored in the upper triangle of W) ---
  int rank = g;
  for (int j = 0; j < g; ++j) {
    // argmax of the remaining diagonal (first index on ties)
    double bv = -1.0;
    int bi = j;
    for (int i = j + threadIdx.x; i < g; i += blockDim.x) {
      const double d = W[i + (int64_t)i * g];
      if (d > bv) { bv = d; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { s_red[threadIdx.x >> 5] = bv; s_ired[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = s_red[0];
      int ix = s_ired[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (s_red[w] > v || (s_red[w] == v && s_ired[w] < ix)) { v = s_red[w]; ix = s_ired[w]; }
      if (j == 0) s_dmax0 = v;
      s_red[0] = v;
      s_ired[0] = ix;
      s_rank = (v > 1e-15 * s_dmax0 && v > 0.0) ? g : j;
    }
    __syncthreads();
    if (s_rank == j) { rank = j; break; }
    const int p = s_ired[0];
    if (p != j) {  // symmetric swap of rows/cols j and p (full matrix), and piv
      for (int i = threadIdx.x; i < g; i += blockDim.x) {
        double t = W[j + (int64_t)i * g];
        W[j + (int64_t)i * g] = W[p + (int64_t)i * g];
        W[p + (int64_t)i * g] = t;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < g; i += blockDim.x) {
        double t = W[i + (int64_t)j * g];
        W[i + (int64_t)j * g] = W[i + (int64_t)p * g];
        W[i + (int64_t)p * g] = t;
      }
      if (threadIdx.x == 0) { int t = piv[j]; piv[j] = piv[p]; piv[p] = t; }
      __syncthreads();
    }
    const double rjj = sqrt(W[j + (int64_t)j * g]);
    __syncthreads();
    for (int k = j + threadIdx.x; k < g; k += blockDim.x)
      W[j + (int64_t)k * g] = (k == j) ? rjj : W[j + (int64_t)k * g] / rjj;
    __syncthreads();
    const int rem = g - j - 1;
    for (int64_t t = threadIdx.x; t < (int64_t)rem * rem; t += blockDim.x) {
      const int kk = j + 1 + (int)(t / rem), ii = j + 1 + (int)(t % rem);
      W[ii + (int64_t)kk * g] -= W[j + (int64_t)ii * g] * W[j + (int64_t)kk * g];
    }
    __syncthreads();
  }
  // --- W <- R^T (rank columns, lower trapezoid), zero elsewhere ---
  for (int64_t t = threadIdx.x; t < (int64_t)g * g; t += blockDim.x) {
    const int j = (int)(t / g), i = (int)(t - (int64_t)j * g);
    if (i > j) {
      W[t] = (j < rank) ? W[j + (int64_t)i * g] : 0.0;  // R[j][i] -> W[i][j]
    }
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < (int64_t)g * g; t += blockDim.x) {
    const int j = (int)(t / g), i = (int)(t - (int64_t)j * g);
    if (i < j || j >= rank) W[t] = (i > j && j < rank) ? W[t] : ((i == j && j < rank) ? W[t] : 0.0);
  }
  __syncthreads();
  const int sweeps = rank >= 2 ? jacobi_one_sided(W, g, g, rank, nullptr, 0, jacobi_tol(g),
                                                  max_sweeps, nrm) : 0;
  column_norms(W, g, g, rank, nrm);
  for (int j = rank + threadIdx.x; j < g; j += blockDim.x) nrm[j] = 0.0;
  __syncthreads();
  rank_sort_desc(nrm, g, perm);
  // lambda = ||col||^2, dust rule (matcore.py:26), sigma = sqrt(lambda)
  const double n0 = nrm[perm[0]];
  const double lam0 = n0 * n0;
  const double dust = 1e-12 * fmax(lam0, 2.2250738585072014e-308);
  for (int k = threadIdx.x; k < g; k += blockDim.x) {
    const double nk = nrm[perm[k]];
    double lam = nk * nk;
    if (lam <= dust) lam = 0.0;
    sig[k] = sqrt(lam);
    sigma_out[k] = sig[k];
  }
  __syncthreads();
  __shared__ int s_keep;
  if (threadIdx.x == 0) {
    int rk = 0;
    if (g && sig[0] > 0.0) {
      const double thr = 1e-14 * sig[0];
      for (int k = 0; k < g; ++k) rk += sig[k] > thr;
    }
    s_keep = min(r, rk);
    info[0] = rk;
    info[1] = s_keep;
    info[2] = sweeps;
  }
  __syncthreads();
  const int keep = s_keep;
  // T[piv[i], k] = v'_k[i] / sigma_k with v'_k = W[:, perm[k]] / ||W[:, perm[k]]||
  for (int64_t t = threadIdx.x; t < (int64_t)g * r; t += blockDim.x) {
    const int k = (int)(t / g), i = (int)(t - (int64_t)k * g);
    double v = 0.0;
    if (k < keep) {
      const int c = perm[k];
      v = W[i + (int64_t)c * g] / nrm[c] / sig[k];
    }
    T[piv[i] + (int64_t)k * ldt] = v;
  }
}

// --------------------------------------------------------- CholeskyQR ----
// Upper-triangular inverse of Rh (l x l, ld l) into X (ld l): warp per column.
__device__ __forceinline__ void upper_inverse(const double* Rh, int l, double* X) {
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
      if (lane == 0) xj[i] = -s / Rh[i + (int64_t)i * l];
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
  __shared__ int s_fail;
  __shared__ double s_defect;
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    const double gii = G[i + (int64_t)i * ldg];
    d[i] = (gii > 0.0) ? sqrt(gii) : 0.0;
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
      h = (G[i + (int64_t)j * ldg] / d[i]) / d[j];
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
      __syncthreads();
      for (int k = j + threadIdx.x; k < l; k += blockDim.x) C[j + (int64_t)k * l] = (k == j) ? rjj : C[j + (int64_t)k * l] / rjj;
      __syncthreads();
      const int rem = l - j - 1;
      for (int64_t t = threadIdx.x; t < (int64_t)rem * rem; t += blockDim.x) {
        const int kk = j + 1 + (int)(t / rem), ii = j + 1 + (int)(t % rem);
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
  upper_inverse(C, l, X);
  // R = Rh D, Rinv = D^-1 Rh^-1; dead columns -> zero rows / columns
  int ndead = 0;
  for (int64_t t = threadIdx.x; t < (int64_t)l * l; t += blockDim.x) {
    const int j = (int)(t / l), i = (int)(t - (int64_t)j * l);
    const bool dead = d[i] == 0.0 || d[j] == 0.0;
    R[i + (int64_t)j * ldr] = dead ? 0.0 : C[t] * d[j];
    Rinv[i + (int64_t)j * ldri] = dead ? 0.0 : X[t] / d[i];
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < l; ++i) ndead += d[i] == 0.0;
    dinfo[0] = s_defect;
    dinfo[1] = (double)attempt;
    dinfo[2] = (double)ndead;
    dinfo[3] = shift;
    if (gate_out) *gate_out = first_pass ? 1 : ((s_defect > 1e-4 || attempt > 0) ? 1 : 0);
  }
}

// ---------------------------------------------------------- merge core ---
template <bool SMEM>
__global__ void __launch_bounds__(SMALL_THREADS) merge_core_kernel(
    const double* __restrict__ sig1, int l1, const double* __restrict__ M, int64_t ldm,
    const double* __restrict__ Rm, int64_t ldr, const double* __restrict__ sig2, int l2, int r,
    int rcap, double* __restrict__ T, int64_t ldt, int tcols, double* __restrict__ sig_new,
    int64_t* __restrict__ info, double* gws, int use_smem, int max_sweeps) {
  extern __shared__ __align__(16) double sm[];
  const int n = l1 + l2;
  double* W = SMEM ? sm : gws;
  double* nrm = W + (size_t)n * n;
  int* perm = reinterpret_cast<int*>(nrm + n);
  for (int64_t t = threadIdx.x; t < (int64_t)n * n; t += blockDim.x) {
    const int j = (int)(t / n), i = (int)(t - (int64_t)j * n);
    double e = 0.0;
    if (j < l1) {
      e = (i == j) ? sig1[j] : 0.0;
    } else {
      const int jj = j - l1;
      if (i < l1) e = M[i + (int64_t)jj * ldm] * sig2[jj];
      else {
        const int ii = i - l1;
        e = (ii <= jj) ? Rm[ii + (int64_t)jj * ldr] * sig2[jj] : 0.0;
      }
    }
    W[t] = e;
  }
  __syncthreads();
  const int sweeps = jacobi_one_sided(W, n, n, n, nullptr, 0, jacobi_tol(n), max_sweeps, nrm);
  column_norms(W, n, n, n, nrm);
  rank_sort_desc(nrm, n, perm);
  __shared__ int s_keep;
  if (threadIdx.x == 0) {
    const double s0 = nrm[perm[0]];
    const double thr = 1e-14 * fmax(s0, 1e-300);
    int cnt = 0;
    for (int k = 0; k < n; ++k) cnt += nrm[perm[k]] > thr;
    s_keep = min(r, cnt);
    info[0] = s_keep;
    info[1] = sweeps;
  }
  __syncthreads();
  const int keep = s_keep;
  for (int k = threadIdx.x; k < rcap; k += blockDim.x) sig_new[k] = (k < keep) ? nrm[perm[k]] : 0.0;
  // T rows follow the stack layout [U1 (rcap cols) | Q (l2 cols)]
  const int trows = rcap + l2;
  for (int64_t t = threadIdx.x; t < (int64_t)trows * tcols; t += blockDim.x) {
    const int k = (int)(t / trows), row = (int)(t - (int64_t)k * trows);
    int e = -1;
    if (row < l1) e = row;
    else if (row >= rcap) e = l1 + (row - rcap);
    double v = 0.0;
    if (e >= 0 && k < keep) {
      const int c = perm[k];
      v = W[e + (int64_t)c * n] / nrm[c];
    }
    T[row + (int64_t)k * ldt] = v;
  }
}

// ----------------------------------------------------------- svd small ---
template <bool SMEM>
__global__ void __launch_bounds__(SMALL_THREADS) svd_small_kernel(
    const double* __restrict__ A, int64_t lda, int nr, int nc, double* __restrict__ U,
    int64_t ldu, double* __restrict__ sigma, double* __restrict__ V, int64_t ldv,
    int64_t* __restrict__ info, double* gws, int use_smem, int max_sweeps, int want_vectors) {
  extern __shared__ __align__(16) double sm[];
  double* W = SMEM ? sm : gws;
  double* J = W + (size_t)nr * nc;
  double* nrm = J + (want_vectors ? (size_t)nc * nc : 0);
  int* perm = reinterpret_cast<int*>(nrm + nc);
  for (int64_t t = threadIdx.x; t < (int64_t)nr * nc; t += blockDim.x) {
    const int j = (int)(t / nr), i = (int)(t - (int64_t)j * nr);
    W[t] = A[i + (int64_t)j * lda];
  }
  if (want_vectors)
    for (int64_t t = threadIdx.x; t < (int64_t)nc * nc; t += blockDim.x) {
      const int j = (int)(t / nc), i = (int)(t - (int64_t)j * nc);
      J[t] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int sweeps = jacobi_one_sided(W, nr, nr, nc, want_vectors ? J : nullptr, nc,
                                      jacobi_tol(nr), max_sweeps, nrm);
  column_norms(W, nr, nr, nc, nrm);
  rank_sort_desc(nrm, nc, perm);
  for (int k = threadIdx.x; k < nc; k += blockDim.x) sigma[k] = nrm[perm[k]];
  if (want_vectors) {
    for (int64_t t = threadIdx.x; t < (int64_t)nr * nc; t += blockDim.x) {
      const int k = (int)(t / nr), i = (int)(t - (int64_t)k * nr);
      const int c = perm[k];
      U[i + (int64_t)k * ldu] = nrm[c] > 0.0 ? W[i + (int64_t)c * nr] / nrm[c] : 0.0;
    }
    for (int64_t t = threadIdx.x; t < (int64_t)nc * nc; t += blockDim.x) {
      const int k = (int)(t / nc), i = (int)(t - (int64_t)k * nc);
      V[i + (int64_t)k * ldv] = J[i + (int64_t)perm[k] * nc];
    }
  }
  if (threadIdx.x == 0) info[0] = sweeps;
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

}  // namespace pod

using namespace pod;

static size_t gram_eigh_bytes(int64_t g) {
  return (size_t)g * g * 8 + (size_t)g * 16 + (size_t)g * 8 + 64;
}
static size_t cholqr_bytes(int64_t l) { return (size_t)3 * l * l * 8 + (size_t)l * 8 + 64; }
static size_t merge_core_bytes(int64_t n) { return (size_t)n * n * 8 + (size_t)n * 12 + 64; }
static size_t svd_small_bytes(int64_t nr, int64_t nc, int vec) {
  return (size_t)nr * nc * 8 + (vec ? (size_t)nc * nc * 8 : 0) + (size_t)nc * 12 + 64;
}

extern "C" size_t pod_small_ws_bytes(int64_t n) {
  // enough for any single small solve with dimension <= n
  size_t a = gram_eigh_bytes(n), b = cholqr_bytes(n), c = merge_core_bytes(n),
         d = svd_small_bytes(n, n, 1);
  return std::max(std::max(a, b), std::max(c, d));
}

extern "C" int pod_gram_eigh(const double* G, int64_t ldg, int64_t g, int64_t r, double* sigma,
                             double* T, int64_t ldt, int64_t* info, void* ws, size_t ws_bytes,
                             void* stream) {
  POD_REQUIRE(g >= 1 && r >= 1 && ldg >= g && ldt >= g, "pod_gram_eigh: bad shape");
  POD_REQUIRE(g <= 2 * JAC_MAX_PAIRS, "pod_gram_eigh: g=%lld exceeds %d", (long long)g, 2 * JAC_MAX_PAIRS);
  const size_t bytes = gram_eigh_bytes(g);
  const int use_smem = bytes <= SMALL_SMEM_CAP;
  POD_REQUIRE(use_smem || ws_bytes >= bytes, "pod_gram_eigh: workspace too small");
  if (use_smem) { int st = set_smem((const void*)gram_eigh_kernel<true>, bytes); if (st) return st; }
  if (use_smem)
    gram_eigh_kernel<true><<<1, jacobi_threads(g), use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      G, ldg, (int)g, (int)r, sigma, T, ldt, info, (double*)ws, use_smem, 60);
  else
    gram_eigh_kernel<false><<<1, jacobi_threads(g), use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      G, ldg, (int)g, (int)r, sigma, T, ldt, info, (double*)ws, use_smem, 60);
  POD_CHECK_LAUNCH("gram_eigh");
  return POD_OK;
}

extern "C" int pod_cholqr_factor(const double* G, int64_t ldg, int64_t l, int64_t nrows,
                                 double* Rinv, int64_t ldri, double* R, int64_t ldr, double* dinfo,
                                 void* ws, size_t ws_bytes, const int32_t* gate_in,
                                 int32_t* gate_out, int first_pass, void* stream) {
  POD_REQUIRE(l >= 1 && ldg >= l && ldri >= l && ldr >= l, "pod_cholqr_factor: bad shape");
  const size_t bytes = cholqr_bytes(l);
  const int use_smem = bytes <= SMALL_SMEM_CAP;
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
  return POD_OK;
}

extern "C" int pod_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm,
                              const double* R, int64_t ldr, const double* sig2, int64_t l2,
                              int64_t r, int64_t rcap, double* T, int64_t ldt, int64_t tcols,
                              double* sig_new, int64_t* info, void* ws, size_t ws_bytes,
                              void* stream) {
  POD_REQUIRE(l1 >= 1 && l2 >= 1 && r >= 1 && rcap >= l1 && ldt >= rcap + l2 && tcols >= 1,
              "pod_merge_core: bad shape");
  const int64_t n = l1 + l2;
  POD_REQUIRE(n <= 2 * JAC_MAX_PAIRS, "pod_merge_core: l1+l2=%lld exceeds %d", (long long)n, 2 * JAC_MAX_PAIRS);
  const size_t bytes = merge_core_bytes(n);
  const int use_smem = bytes <= SMALL_SMEM_CAP;
  POD_REQUIRE(use_smem || ws_bytes >= bytes, "pod_merge_core: workspace too small");
  if (use_smem) { int st = set_smem((const void*)merge_core_kernel<true>, bytes); if (st) return st; }
  if (use_smem)
    merge_core_kernel<true><<<1, jacobi_threads(n), use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      sig1, (int)l1, M, ldm, R, ldr, sig2, (int)l2, (int)r, (int)rcap, T, ldt, (int)tcols,
      sig_new, info, (double*)ws, use_smem, 60);
  else
    merge_core_kernel<false><<<1, jacobi_threads(n), use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      sig1, (int)l1, M, ldm, R, ldr, sig2, (int)l2, (int)r, (int)rcap, T, ldt, (int)tcols,
      sig_new, info, (double*)ws, use_smem, 60);
  POD_CHECK_LAUNCH("merge_core");
  return POD_OK;
}

extern "C" int pod_svd_small(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U,
                             int64_t ldu, double* sigma, double* V, int64_t ldv, int64_t* info,
                             void* ws, size_t ws_bytes, void* stream) {
  POD_REQUIRE(nr >= 1 && nc >= 1 && lda >= nr, "pod_svd_small: bad shape");
  POD_REQUIRE(nc <= 2 * JAC_MAX_PAIRS, "pod_svd_small: nc=%lld exceeds %d", (long long)nc, 2 * JAC_MAX_PAIRS);
  const int vec = (U != nullptr && V != nullptr);
  const size_t bytes = svd_small_bytes(nr, nc, vec);
  const int use_smem = bytes <= SMALL_SMEM_CAP;
  POD_REQUIRE(use_smem || ws_bytes >= bytes, "pod_svd_small: workspace too small");
  if (use_smem) { int st = set_smem((const void*)svd_small_kernel<true>, bytes); if (st) return st; }
  if (use_smem)
    svd_small_kernel<true><<<1, jacobi_threads(nc), use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      A, lda, (int)nr, (int)nc, U, ldu, sigma, V, ldv, info, (double*)ws, use_smem, 60, vec);
  else
    svd_small_kernel<false><<<1, jacobi_threads(nc), use_smem ? bytes : 0, (cudaStream_t)stream>>>(
      A, lda, (int)nr, (int)nc, U, ldu, sigma, V, ldv, info, (double*)ws, use_smem, 60, vec);
  POD_CHECK_LAUNCH("svd_small");
  return POD_OK;
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
