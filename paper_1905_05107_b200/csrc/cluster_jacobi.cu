// Row-distributed one-sided Jacobi on a thread-block cluster (sm_100a).
//
// The per-round small SVD/eigen problems of ISMA (E = [[S1, M S2],[0, R S2]]
// of merge.py:80-84, the sampled Gram of baselines.py:43-48, finalize's R of
// isma.py:297) are solved by one-sided Jacobi, whose cost is ~n sequential
// steps per sweep.  A single SM is latency/issue bound on each step, so the
// matrix is spread over a cluster of CL CTAs BY ROWS: CTA c keeps rows
// [c*nrl, (c+1)*nrl) of every column in its shared memory.  One step:
//   1. each CTA computes partial dots gamma_p over its rows for every pair p
//   2. all-to-all of the partials through distributed shared memory (DSMEM
//      stores into every CTA's receive slot), one cluster barrier
//   3. every CTA sums the CL partials in the same order -> bitwise identical
//      gamma, rotation parameters and decisions in all CTAs
//   4. each CTA rotates its own rows (and its rows of J when accumulating).
// Singular vectors come out row-local (U = W / sigma, V = J), so results are
// written without any gather.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pod {

constexpr int CL_MAX = 8;          // cluster size (portable maximum)
constexpr int CJ_THREADS = 256;
constexpr int CJ_MAX_N = 512;      // columns

// Scratch carved from dynamic shared memory at the same offsets in every
// CTA of the cluster (DSMEM addresses are mapped by offset).
struct CJScratch {
  uint64_t* mbar; // [2] mbarriers of the two partial-dot buffers
  double* part;   // [2][CL][npairs] partial dots, double-buffered by step parity
  double* partn;  // [CL][n] partial squared column norms
  double* nrm2;   // [n] squared column norms (identical in all CTAs)
  double* cs;     // [npairs]
  double* sn;     // [npairs]
  double* aux;    // [n] per-kernel scratch (sigma)
  short* pa;      // [npairs]
  short* pb;      // [npairs]
  int* perm;      // [n]
  int* flags;     // [0] rotated, [1] keep
  double* body;   // matrix storage after the scratch
};

template <int CL>
__host__ __device__ inline size_t cj_scratch_bytes(int n) {
  const int np = (n + 1) / 2;
  size_t b = (size_t)(2 + 2 * CL * np + CL * n + n + 2 * np + n) * sizeof(double);
  b += (size_t)(2 * np) * sizeof(short) + (size_t)n * sizeof(int) + 4 * sizeof(int);
  return (b + 15) & ~(size_t)15;
}

template <int CL>
__device__ inline CJScratch cj_carve(double* base, int n) {
  const int np = (n + 1) / 2;
  CJScratch s;
  s.mbar = reinterpret_cast<uint64_t*>(base);
  double* p = base + 2;
  s.part = p; p += 2 * CL * np;
  s.partn = p; p += CL * n;
  s.nrm2 = p; p += n;
  s.cs = p; p += np;
  s.sn = p; p += np;
  s.aux = p; p += n;
  short* q = reinterpret_cast<short*>(p);
  s.pa = q; q += np;
  s.pb = q; q += np;
  int* ip = reinterpret_cast<int*>(q);
  s.perm = ip; ip += n;
  s.flags = ip;
  s.body = reinterpret_cast<double*>(reinterpret_cast<char*>(base) + cj_scratch_bytes<CL>(n));
  return s;
}

// fp64 1/sqrt(x) for any positive normal x: exact power-of-two scaling into
// fp32 range, fp32 seed, two Newton steps (rel. err ~1e-16).
__device__ __forceinline__ double rsqrt_nr2(double x) {
  int e;
  double m = frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
  if (e & 1) {
    m *= 2.0;
    e -= 1;
  }
  double y = (double)rsqrtf((float)m);
  y = y * fma(-0.5 * m, y * y, 1.5);
  y = y * fma(-0.5 * m, y * y, 1.5);
  return ldexp(y, -e / 2);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Remote (or local) 8-byte store that completes 8 transaction bytes on the
// destination CTA's mbarrier.
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n"
               ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rmbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* mb, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n"
               ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  const uint32_t a = smem_u32(mb);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
  }
}

// Exchange per-column partial squared norms of the local rows and sum them
// in rank order (identical result in every CTA).  Includes cluster barriers.
template <int CL>
__device__ void cj_norms(cg::cluster_group& cl, const CJScratch& s, const double* Wl, int ldl, int nrl,
                         int nc) {
  const int me = (int)cl.block_rank();
  for (int j = threadIdx.x; j < nc; j += blockDim.x) {
    const double* w = Wl + (int64_t)j * ldl;
    double a = 0.0;
    for (int i = 0; i < nrl; ++i) a = fma(w[i], w[i], a);
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      double* dst = cl.map_shared_rank(&s.partn[me * nc + j], c);
      *dst = a;
    }
  }
  cl.sync();
  for (int j = threadIdx.x; j < nc; j += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < CL; ++c) t += s.partn[c * nc + j];
    s.nrm2[j] = t;
  }
  cl.sync();  // partn may be rewritten by the next exchange
}

// One-sided cyclic Jacobi (round-robin pairs) on W distributed by rows.
// Wl: this CTA's nrl rows (ld ldl) of all nc columns; Jl (nullable): this
// CTA's njl rows (ld ldj) of the nc x nc accumulator.  Returns sweeps.
#ifdef POD_CJ_TIMING
__device__ unsigned long long g_cj_phase[8];
#define CJ_T(i)                                                              \
  do {                                                                       \
    if (threadIdx.x == 0 && cl.block_rank() == 0) {                          \
      unsigned long long _t = clock64();                                     \
      if (i) atomicAdd(&g_cj_phase[i], _t - _cj_last);                      \
      _cj_last = _t;                                                         \
    }                                                                        \
  } while (0)
#else
#define CJ_T(i) \
  do {          \
  } while (0)
#endif

template <int CL, int RPL>
__device__ int cj_jacobi_t(cg::cluster_group& cl, const CJScratch& s, double* Wl, int ldl, int nrl,
                           int nc, double* Jl, int ldj, int njl, double tol, int max_sweeps) {
  const int me = (int)cl.block_rank();
  const int N = nc + (nc & 1);
  const int M1 = N - 1;
  const int npairs = N / 2;
  const double tol2 = tol * tol;
  // threads per pair for the partial dots (power of two, <= 32)
  int tpp = 1;
  while (tpp * 2 * npairs <= (int)blockDim.x && tpp < 16) tpp *= 2;
  // DSMEM addresses of every CTA's receive buffers and mbarriers (fixed)
  uint32_t rpart[CL], rmbar[CL];
  {
    const uint32_t lp = smem_u32(s.part), lm = smem_u32(s.mbar);
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      rpart[c] = cluster_map(lp, c);
      rmbar[c] = cluster_map(lm, c);
    }
  }
  const int grp = threadIdx.x / tpp, gl = threadIdx.x % tpp;
  int sweep = 0;
  int parity = 0;
  uint32_t gstep = 0;  // global step counter: buffer = gstep & 1, phase = (gstep >> 1) & 1
  const uint32_t tx_bytes = (uint32_t)(CL * npairs * sizeof(double));
  if (threadIdx.x == 0) {
    mbar_init(&s.mbar[0], 1);
    mbar_init(&s.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cl.sync();  // every CTA's barriers are initialised before any st.async
  if (nc < 2) {
    cj_norms<CL>(cl, s, Wl, ldl, nrl, nc);
    return 0;
  }
  while (sweep < max_sweeps) {
    cj_norms<CL>(cl, s, Wl, ldl, nrl, nc);
    if (threadIdx.x == 0) s.flags[0] = 0;
    __syncthreads();
#ifdef POD_CJ_TIMING
    unsigned long long _cj_last = clock64();
#endif
    for (int step = 0; step < M1; ++step, ++gstep) {
      CJ_T(0);
      parity = (int)(gstep & 1u);
      if (threadIdx.x == 0) mbar_arrive_expect(&s.mbar[parity], tx_bytes);
      // pair of this thread group (every lane takes part in the shuffles)
      const int pr = grp;
      const bool valid = pr < npairs;
      int a = 0, b = 0;
      if (valid) {
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
      }
      const bool live = valid && b < nc;
      double* wa = Wl + (int64_t)a * ldl;
      double* wb = Wl + (int64_t)b * ldl;
      // 1. partial dot over the local rows -> every CTA's receive slot
      double g = 0.0;
      double xa[RPL > 0 ? RPL : 1], xb[RPL > 0 ? RPL : 1];
      if (RPL > 0) {
#pragma unroll
        for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
          const int i = gl + k * tpp;
          const bool ok = live && i < nrl;
          xa[k] = ok ? wa[i] : 0.0;
          xb[k] = ok ? wb[i] : 0.0;
          g = fma(xa[k], xb[k], g);
        }
      } else if (live) {
        for (int i = gl; i < nrl; i += tpp) g = fma(wa[i], wb[i], g);
      }
      for (int o = tpp / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o, tpp);
      if (valid) {  // the pair's lanes share the CL remote stores
        const uint32_t off = (uint32_t)(((parity * CL + me) * npairs + pr) * sizeof(double));
        const uint32_t moff = (uint32_t)(parity * sizeof(uint64_t));
#pragma unroll
        for (int c = 0; c < CL; ++c)
          if ((c % tpp) == gl) st_async_f64(rpart[c] + off, g, rmbar[c] + moff);
      }
      CJ_T(1);
      mbar_wait(&s.mbar[parity], (gstep >> 1) & 1u);
      CJ_T(2);
      // 2. full gamma (rank-ordered sum: identical in every CTA) and the
      //    rotation, computed redundantly by the pair's own lanes
      if (live) {
        double gg = 0.0;
#pragma unroll
        for (int c = 0; c < CL; ++c) gg += s.part[(parity * CL + c) * npairs + pr];
        const double al = s.nrm2[a], be = s.nrm2[b];
        if (gg * gg > tol2 * al * be && al > 0.0 && be > 0.0) {
          // tan(2 theta) = 2 gamma / (be - al), |theta| <= pi/4:
          // 1/h = rsqrt(d^2 + 4 gamma^2), cos 2theta = |d|/h,
          // c = sqrt((1 + cos 2theta)/2), s = sign(d gamma) |gamma| / (h c)
          const double d = be - al;
          const double rh = rsqrt_nr2(fma(d, d, 4.0 * gg * gg));
          const double x = 0.5 * fma(fabs(d), rh, 1.0);
          double ic = (double)rsqrtf((float)x);  // x in [0.5, 1]: fp32 seed is in range
          ic = ic * fma(-0.5 * x, ic * ic, 1.5);
          ic = ic * fma(-0.5 * x, ic * ic, 1.5);
          const double c_ = x * ic;
          const double s_ = copysign(fabs(gg) * rh * ic, d * gg);
          if (RPL > 0) {
#pragma unroll
            for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
              const int i = gl + k * tpp;
              if (i < nrl) {
                wa[i] = fma(c_, xa[k], -s_ * xb[k]);
                wb[i] = fma(s_, xa[k], c_ * xb[k]);
              }
            }
          } else {
            for (int i = gl; i < nrl; i += tpp) {
              const double x0 = wa[i], y0 = wb[i];
              wa[i] = fma(c_, x0, -s_ * y0);
              wb[i] = fma(s_, x0, c_ * y0);
            }
          }
          if (Jl) {
            double* ja = Jl + (int64_t)a * ldj;
            double* jb = Jl + (int64_t)b * ldj;
            for (int i = gl; i < njl; i += tpp) {
              const double x0 = ja[i], y0 = jb[i];
              ja[i] = fma(c_, x0, -s_ * y0);
              jb[i] = fma(s_, x0, c_ * y0);
            }
          }
          CJ_T(3);
          if (gl == 0) {
            const double c2 = c_ * c_, s2 = s_ * s_, csg = 2.0 * c_ * s_ * gg;
            s.nrm2[a] = fmax(fma(c2, al, fma(s2, be, -csg)), 0.0);
            s.nrm2[b] = fma(s2, al, fma(c2, be, csg));
            s.flags[0] = 1;
          }
        }
      }
      CJ_T(4);
      __syncthreads();
      CJ_T(5);
    }
    ++sweep;
    const int any = s.flags[0];  // identical in every CTA
    __syncthreads();
    if (!any) break;
  }
  cj_norms<CL>(cl, s, Wl, ldl, nrl, nc);  // exact final norms
  return sweep;
}

template <int CL>
__device__ int cj_jacobi(cg::cluster_group& cl, const CJScratch& s, double* Wl, int ldl, int nrl,
                         int nc, double* Jl, int ldj, int njl, double tol, int max_sweeps) {
  const int np = (nc + (nc & 1)) / 2;
  int tpp = 1;
  while (tpp * 2 * np <= (int)blockDim.x && tpp < 16) tpp *= 2;
  const int rpl = (nrl + tpp - 1) / tpp;
  if (rpl <= 4) return cj_jacobi_t<CL, 4>(cl, s, Wl, ldl, nrl, nc, Jl, ldj, njl, tol, max_sweeps);
  if (rpl <= 8) return cj_jacobi_t<CL, 8>(cl, s, Wl, ldl, nrl, nc, Jl, ldj, njl, tol, max_sweeps);
  if (rpl <= 16) return cj_jacobi_t<CL, 16>(cl, s, Wl, ldl, nrl, nc, Jl, ldj, njl, tol, max_sweeps);
  return cj_jacobi_t<CL, 0>(cl, s, Wl, ldl, nrl, nc, Jl, ldj, njl, tol, max_sweeps);
}

// perm[k] = column with the k-th largest key (ties -> lower index)
__device__ void cj_rank_sort(const double* key, int n, int* perm) {
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

__device__ __forceinline__ double cj_tol(int nr) { return 2.220446049250313e-16 * (double)max(nr, 16); }

// ------------------------------------------------------------ merge core --
// E (n x n, n = l1 + l2) built row-locally; U_E = W / sigma row-local; T rows
// in the stack layout [U1 (rcap) | Q (l2)].
template <int CL>
__global__ void __launch_bounds__(CJ_THREADS)
    cj_merge_core_kernel(const double* __restrict__ sig1, int l1, const double* __restrict__ M,
                         int64_t ldm, const double* __restrict__ Rm, int64_t ldr,
                         const double* __restrict__ sig2, int l2, int r, int rcap,
                         double* __restrict__ T, int64_t ldt, int tcols,
                         double* __restrict__ sig_new, int64_t* __restrict__ info, int nrl,
                         int max_sweeps, const int32_t* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;  // gated re-run (block_jacobi.cu)
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double smem_cj[];
  const int n = l1 + l2;
  const CJScratch s = cj_carve<CL>(smem_cj, n);
  double* Wl = s.body;  // nrl x n, ld nrl
  const int me = (int)cl.block_rank();
  const int r0 = me * nrl;
  for (int t = threadIdx.x; t < nrl * n; t += blockDim.x) {
    const int j = t / nrl, il = t - j * nrl, i = r0 + il;
    double e = 0.0;
    if (i < n) {
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
    }
    Wl[t] = e;
  }
  __syncthreads();
  const int nrl_eff = max(0, min(nrl, n - r0));
  const int sweeps = cj_jacobi<CL>(cl, s, Wl, nrl, nrl_eff, n, nullptr, 0, 0, cj_tol(n), max_sweeps);
  for (int j = threadIdx.x; j < n; j += blockDim.x) s.nrm2[j] = sqrt(s.nrm2[j]);  // sigma
  __syncthreads();
  cj_rank_sort(s.nrm2, n, s.perm);
  if (threadIdx.x == 0) {
    const double s0 = s.nrm2[s.perm[0]];
    const double thr = 1e-14 * fmax(s0, 1e-300);
    int cnt = 0;
    for (int k = 0; k < n; ++k) cnt += s.nrm2[s.perm[k]] > thr;
    s.flags[1] = min(r, cnt);
    if (me == 0) {
      info[0] = s.flags[1];
      info[1] = sweeps;
    }
  }
  __syncthreads();
  const int keep = s.flags[1];
  if (me == 0)
    for (int k = threadIdx.x; k < rcap; k += blockDim.x)
      sig_new[k] = (k < keep) ? s.nrm2[s.perm[k]] : 0.0;
  // T rows owned by this CTA: E rows e in [r0, r0 + nrl)
  for (int t = threadIdx.x; t < nrl * tcols; t += blockDim.x) {
    const int k = t / nrl, el = t - k * nrl, e = r0 + el;
    if (e >= n) continue;
    const int row = (e < l1) ? e : rcap + (e - l1);
    double v = 0.0;
    if (k < keep) {
      const int c = s.perm[k];
      v = Wl[el + c * nrl] / s.nrm2[c];
    }
    T[row + (int64_t)k * ldt] = v;
  }
  // zero the padding rows l1..rcap of T (owned by CTA 0)
  if (me == 0)
    for (int t = threadIdx.x; t < (rcap - l1) * tcols; t += blockDim.x) {
      const int k = t / (rcap - l1), row = l1 + t % (rcap - l1);
      T[row + (int64_t)k * ldt] = 0.0;
    }
  cl.sync();  // no CTA may exit while others can still write into its smem
}

// ------------------------------------------------------------- gram eigh --
// Input: X = R^T (g x g, ld g, columns >= rank zero) from the pivoted
// Cholesky P G P^T = R^T R, and piv.  One-sided Jacobi on X's columns gives
// X J = V' Sigma -> lambda = ||col||^2, eigenvector rows v'[i] row-local.
template <int CL>
__global__ void __launch_bounds__(CJ_THREADS)
    cj_gram_eigh_kernel(const double* __restrict__ X, const int* __restrict__ piv,
                        const int64_t* __restrict__ rank_in, int g, int r,
                        double* __restrict__ sigma_out, double* __restrict__ T, int64_t ldt,
                        int64_t* __restrict__ info, int nrl, int max_sweeps) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double smem_cj[];
  const CJScratch s = cj_carve<CL>(smem_cj, g);
  double* Wl = s.body;  // nrl x g
  const int me = (int)cl.block_rank();
  const int r0 = me * nrl;
  const int rank = (int)*rank_in;
  for (int t = threadIdx.x; t < nrl * g; t += blockDim.x) {
    const int j = t / nrl, il = t - j * nrl, i = r0 + il;
    Wl[t] = (i < g && j < rank) ? X[i + (int64_t)j * g] : 0.0;
  }
  __syncthreads();
  const int nrl_eff = max(0, min(nrl, g - r0));
  const int sweeps = rank >= 2 ? cj_jacobi<CL>(cl, s, Wl, nrl, nrl_eff, rank, nullptr, 0, 0,
                                           cj_tol(g), max_sweeps)
                               : 0;
  if (rank < 2) cj_norms<CL>(cl, s, Wl, nrl, nrl_eff, rank);
  // s.nrm2[j] = lambda_j (squared column norm) for j < rank
  for (int j = rank + threadIdx.x; j < g; j += blockDim.x) s.nrm2[j] = 0.0;
  __syncthreads();
  cj_rank_sort(s.nrm2, g, s.perm);
  double* sig_s = s.aux;
  const double lam0 = s.nrm2[s.perm[0]];
  const double dust = 1e-12 * fmax(lam0, 2.2250738585072014e-308);  // matcore.py:26
  for (int k = threadIdx.x; k < g; k += blockDim.x) {
    double lam = s.nrm2[s.perm[k]];
    if (lam <= dust) lam = 0.0;
    sig_s[k] = sqrt(lam);
    if (me == 0) sigma_out[k] = sig_s[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int rk = 0;
    if (g && sig_s[0] > 0.0) {
      const double thr = 1e-14 * sig_s[0];  // matcore.py:20
      for (int k = 0; k < g; ++k) rk += sig_s[k] > thr;
    }
    s.flags[1] = min(r, rk);
    if (me == 0) {
      info[0] = rk;
      info[1] = s.flags[1];
      info[2] = sweeps;
    }
  }
  __syncthreads();
  const int keep = s.flags[1];
  // T[piv[i], k] = v'_k[i] / sigma_k,  v'_k = W[:, perm[k]] / sqrt(lambda)
  for (int t = threadIdx.x; t < nrl * r; t += blockDim.x) {
    const int k = t / nrl, il = t - k * nrl, i = r0 + il;
    if (i >= g) continue;
    double v = 0.0;
    if (k < keep) {
      const int c = s.perm[k];
      v = Wl[il + c * nrl] / sqrt(s.nrm2[c]) / sig_s[k];
    }
    T[piv[i] + (int64_t)k * ldt] = v;
  }
  cl.sync();
}

// ------------------------------------------------------------- svd small --
template <int CL>
__global__ void __launch_bounds__(CJ_THREADS)
    cj_svd_kernel(const double* __restrict__ A, int64_t lda, int nr, int nc,
                  double* __restrict__ U, int64_t ldu, double* __restrict__ sigma,
                  double* __restrict__ V, int64_t ldv, int64_t* __restrict__ info, int nrl,
                  int njl, int max_sweeps) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double smem_cj[];
  const CJScratch s = cj_carve<CL>(smem_cj, nc);
  double* Wl = s.body;                                   // nrl x nc
  double* Jl = V ? s.body + (size_t)nrl * nc : nullptr;  // njl x nc (rows of J)
  const int me = (int)cl.block_rank();
  const int r0 = me * nrl, j0 = me * njl;
  for (int t = threadIdx.x; t < nrl * nc; t += blockDim.x) {
    const int j = t / nrl, il = t - j * nrl, i = r0 + il;
    Wl[t] = (i < nr) ? A[i + (int64_t)j * lda] : 0.0;
  }
  if (Jl)
    for (int t = threadIdx.x; t < njl * nc; t += blockDim.x) {
      const int j = t / njl, il = t - j * njl, i = j0 + il;
      Jl[t] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int nrl_eff = max(0, min(nrl, nr - r0));
  const int njl_eff = max(0, min(njl, nc - j0));
  const int sweeps = cj_jacobi<CL>(cl, s, Wl, nrl, nrl_eff, nc, Jl, njl, njl_eff, cj_tol(nr),
                               max_sweeps);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) s.nrm2[j] = sqrt(s.nrm2[j]);
  __syncthreads();
  cj_rank_sort(s.nrm2, nc, s.perm);
  if (me == 0) {
    for (int k = threadIdx.x; k < nc; k += blockDim.x) sigma[k] = s.nrm2[s.perm[k]];
    if (threadIdx.x == 0) info[0] = sweeps;
  }
  if (U) {
    for (int t = threadIdx.x; t < nrl * nc; t += blockDim.x) {
      const int k = t / nrl, il = t - k * nrl, i = r0 + il;
      if (i >= nr) continue;
      const int c = s.perm[k];
      U[i + (int64_t)k * ldu] = s.nrm2[c] > 0.0 ? Wl[il + c * nrl] / s.nrm2[c] : 0.0;
    }
  }
  if (V) {
    for (int t = threadIdx.x; t < njl * nc; t += blockDim.x) {
      const int k = t / njl, il = t - k * njl, i = j0 + il;
      if (i >= nc) continue;
      V[i + (int64_t)k * ldv] = Jl[il + s.perm[k] * njl];
    }
  }
  cl.sync();
}

constexpr size_t CJ_SMEM_CAP = 224 * 1024;

// Threads per CTA: up to 4 lanes per column pair (the device code uses the
// largest power-of-two lanes-per-pair that fits), rounded to whole warps.
static int cj_threads(int n) {
  const int np = (n + 1) / 2;
  int tpp = 1;
  while (tpp * 2 * np <= CJ_THREADS && tpp < 4) tpp *= 2;
  int t = ((tpp * np + 31) / 32) * 32;
  return std::max(64, std::min(CJ_THREADS, t));
}

static int cj_set_smem(const void* fn, size_t bytes) {
  static const void* fns[8];
  static int nf = 0;
  if (bytes > CJ_SMEM_CAP) {
    set_error("cluster Jacobi: %zu bytes of shared memory per CTA exceed %zu", bytes,
              CJ_SMEM_CAP);
    return POD_EPARAM;
  }
  for (int i = 0; i < nf; ++i)
    if (fns[i] == fn) return POD_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)CJ_SMEM_CAP);
  if (e != cudaSuccess) return cuda_status(e, "cluster jacobi smem attr");
  if (nf < 8) fns[nf++] = fn;
  return POD_OK;
}

template <typename K, typename... Args>
static int cj_launch(K kernel, int cl, int threads, size_t smem, cudaStream_t stream,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  return e == cudaSuccess ? POD_OK : cuda_status(e, "cluster launch");
}

// Cluster size: 8 CTAs by default (POD_CJ_CLUSTER=2|4|8 overrides, for tuning).
static int cj_cluster() {
  static int cl = 0;
  if (!cl) {
    const char* e = getenv("POD_CJ_CLUSTER");
    int v = e ? atoi(e) : 8;
    cl = (v == 2 || v == 4 || v == 8) ? v : 8;
  }
  return cl;
}

template <int CL>
static int cj_merge_core_t(const double* sig1, int64_t l1, const double* M, int64_t ldm,
                           const double* R, int64_t ldr, const double* sig2, int64_t l2, int64_t r,
                           int64_t rcap, double* T, int64_t ldt, int64_t tcols, double* sig_new,
                           int64_t* info, const int32_t* gate, cudaStream_t stream) {
  const int n = (int)(l1 + l2);
  const int nrl = (n + CL - 1) / CL;
  const size_t bytes = cj_scratch_bytes<CL>(n) + (size_t)nrl * n * sizeof(double);
  int st = cj_set_smem((const void*)cj_merge_core_kernel<CL>, bytes);
  if (st) return st;
  return cj_launch(cj_merge_core_kernel<CL>, CL, cj_threads(n), bytes, stream, sig1, (int)l1, M,
                   ldm, R, ldr, sig2, (int)l2, (int)r, (int)rcap, T, ldt, (int)tcols, sig_new,
                   info, nrl, 60, gate);
}

int cj_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                  int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                  int64_t ldt, int64_t tcols, double* sig_new, int64_t* info,
                  const int32_t* gate, cudaStream_t stream) {
  const int n = (int)(l1 + l2);
  POD_REQUIRE(n <= CJ_MAX_N, "merge core: l1 + l2 = %d exceeds %d", n, CJ_MAX_N);
  switch (cj_cluster()) {
    case 2: return cj_merge_core_t<2>(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols, sig_new, info, gate, stream);
    case 4: return cj_merge_core_t<4>(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols, sig_new, info, gate, stream);
    default: return cj_merge_core_t<8>(sig1, l1, M, ldm, R, ldr, sig2, l2, r, rcap, T, ldt, tcols, sig_new, info, gate, stream);
  }
}

template <int CL>
static int cj_gram_eigh_t(const double* X, const int* piv, const int64_t* rank, int64_t g,
                          int64_t r, double* sigma, double* T, int64_t ldt, int64_t* info,
                          cudaStream_t stream) {
  const int nrl = (int)((g + CL - 1) / CL);
  const size_t bytes = cj_scratch_bytes<CL>((int)g) + (size_t)nrl * g * sizeof(double);
  int st = cj_set_smem((const void*)cj_gram_eigh_kernel<CL>, bytes);
  if (st) return st;
  return cj_launch(cj_gram_eigh_kernel<CL>, CL, cj_threads((int)g), bytes, stream, X, piv, rank,
                   (int)g, (int)r, sigma, T, ldt, info, nrl, 60);
}

int cj_gram_eigh(const double* X, const int* piv, const int64_t* rank, int64_t g, int64_t r,
                 double* sigma, double* T, int64_t ldt, int64_t* info, cudaStream_t stream) {
  POD_REQUIRE(g <= CJ_MAX_N, "gram eigh: g = %lld exceeds %d", (long long)g, CJ_MAX_N);
  switch (cj_cluster()) {
    case 2: return cj_gram_eigh_t<2>(X, piv, rank, g, r, sigma, T, ldt, info, stream);
    case 4: return cj_gram_eigh_t<4>(X, piv, rank, g, r, sigma, T, ldt, info, stream);
    default: return cj_gram_eigh_t<8>(X, piv, rank, g, r, sigma, T, ldt, info, stream);
  }
}

template <int CL>
static int cj_svd_t(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
                    double* sigma, double* V, int64_t ldv, int64_t* info, cudaStream_t stream) {
  const int nrl = (int)((nr + CL - 1) / CL);
  const int njl = V ? (int)((nc + CL - 1) / CL) : 0;
  const size_t bytes =
      cj_scratch_bytes<CL>((int)nc) + ((size_t)nrl * nc + (size_t)njl * nc) * sizeof(double);
  int st = cj_set_smem((const void*)cj_svd_kernel<CL>, bytes);
  if (st) return st;
  return cj_launch(cj_svd_kernel<CL>, CL, cj_threads((int)nc), bytes, stream, A, lda, (int)nr,
                   (int)nc, U, ldu, sigma, V, ldv, info, nrl, njl, 60);
}

int cj_svd(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
           double* sigma, double* V, int64_t ldv, int64_t* info, cudaStream_t stream) {
  POD_REQUIRE(nc <= CJ_MAX_N && nr <= 4096, "svd small: %lld x %lld too large", (long long)nr,
              (long long)nc);
  switch (cj_cluster()) {
    case 2: return cj_svd_t<2>(A, lda, nr, nc, U, ldu, sigma, V, ldv, info, stream);
    case 4: return cj_svd_t<4>(A, lda, nr, nc, U, ldu, sigma, V, ldv, info, stream);
    default: return cj_svd_t<8>(A, lda, nr, nc, U, ldu, sigma, V, ldv, info, stream);
  }
}

// Whether the cluster solver's shared-memory layout fits (same byte counts
// as the launches above); callers route larger problems to grid_jacobi.cu.
template <int CL>
static bool cj_fits_t(int64_t nc, int64_t nr, int64_t njr) {
  const int64_t nrl = (nr + CL - 1) / CL, njl = (njr + CL - 1) / CL;
  return cj_scratch_bytes<CL>((int)nc) + (size_t)(nrl + njl) * nc * sizeof(double) <= CJ_SMEM_CAP;
}
bool cj_fits(int64_t nc, int64_t nr, int64_t njr) {
  if (nc > CJ_MAX_N || nr > 4096) return false;
  switch (cj_cluster()) {
    case 2: return cj_fits_t<2>(nc, nr, njr);
    case 4: return cj_fits_t<4>(nc, nr, njr);
    default: return cj_fits_t<8>(nc, nr, njr);
  }
}

}  // namespace pod

#ifdef POD_CJ_TIMING
extern "C" int pod_debug_cj_phase(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, pod::g_cj_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(pod::g_cj_phase, z, sizeof(z));
  }
  return 0;
}
#endif
