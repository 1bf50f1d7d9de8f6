// Column-distributed BLOCK one-sided Jacobi on a thread-block cluster (sm_100a).
//
// Same problems as cluster_jacobi.cu (the E-SVD of merge.py:80-85, the
// sampled-Gram eigensolve of baselines.py:43-48, the small SVDs of finalize
// isma.py:297 / orthonormalize isma.py:251-252), different parallel layout:
// the n columns are cut into NB = 2 CL blocks of bs columns and every CTA of
// the cluster OWNS two whole blocks (all rows), so a column pair's dot
// products, rotation and norm update are local to one CTA -- no per-pair
// partial-sum exchange.  One sweep:
//   - intra phase: every CTA rotates the pairs inside each of its two blocks
//   - NB - 1 steps of the round-robin ("circle") block tournament: a CTA
//     rotates all bs^2 pairs between its two blocks (bs sub-rounds of bs
//     disjoint pairs), then the blocks move to their next owners with
//     cp.async.bulk DSMEM copies completing on the receiver's mbarrier;
//     one cluster barrier per step.
// Each unordered column pair is visited exactly once per sweep (as in the
// cyclic scalar method), in a fixed order, so results are deterministic.
// The rotation formulas, threshold (gamma^2 > tol^2 a b) and stopping rule (a
// sweep without rotations) are those of cluster_jacobi.cu.
#include <cooperative_groups.h>

#include "bj_core.cuh"

namespace cg = cooperative_groups;

namespace pod {

namespace bj {

// Runs the sweeps.  On return the CURRENT set holds the converged blocks
// (exact squared norms in nrm) and every CTA's gnorm[id] holds all n squared
// norms.  Returns the sweep count.
// nset = 3 block sets: the blocks of step st+1 land in a third set, so a CTA
// may run ahead of a neighbour without overwriting data the neighbour still
// reads -- the cluster barrier is then needed once per sweep (the
// convergence vote) instead of once per tournament step.  nset = 2 keeps the
// per-step barrier (sizes whose three sets do not fit shared memory).
template <int CL, int TPP, int RPL>
__device__ int run_sweeps(cg::cluster_group& cl, const Geo& g, double* slots, uint64_t* mbar,
                          double* flags, double* gnorm, int& cur_set, double tol,
                          int max_sweeps, int nset) {
  const int me = (int)cl.block_rank();
  const int bs = g.bs;
  const double tol2 = tol * tol;
  const int NB = 2 * CL;
  int set = cur_set;
  uint32_t use[3] = {0u, 0u, 0u};
  // destinations of this CTA's slot 0 (top) and slot 1 (bottom) after a step
  int d0c, d0s, d1c, d1s;
  if (me == 0) { d0c = 0; d0s = 0; d1c = (CL > 1) ? 1 : 0; d1s = 0; }
  else {
    d1c = me - 1; d1s = 1;
    if (me == CL - 1) { d0c = me; d0s = 1; }
    else { d0c = me + 1; d0s = 0; }
  }
  const uint32_t slot_bytes = (uint32_t)(g.slot * sizeof(double));
  const uint32_t slots_u32 = smem_u32(slots);
  const uint32_t mbar_u32 = smem_u32(mbar);
  int sweep = 0;
  bool converged = false;
#ifdef POD_BJ_TIMING
  unsigned long long _bj_last = clock64();
#endif
  while (sweep < max_sweeps && !converged) {
    BJ_T(0);
    Slot c0 = slot_at(slots, g, set, 0), c1 = slot_at(slots, g, set, 1);
    // exact squared norms of the owned columns
    for (int t = threadIdx.x; t < 2 * bs; t += blockDim.x) {
      const Slot& s = (t < bs) ? c0 : c1;
      const int c = t % bs;
      const double* w = s.w + (size_t)c * g.ld;
      double a = 0.0;
      for (int i = 0; i < g.nrows; ++i) a = fma(w[i], w[i], a);
      s.nrm[c] = a;
    }
    __syncthreads();
    BJ_T(1);
    int rot = 0;
    // intra phase: round-robin inside each owned block (both blocks at once)
    {
      const int B = bs + (bs & 1);
      for (int step = 0; step < B - 1; ++step) {
        const int half = B / 2;
        rot |= sub_round<TPP, RPL>(c0, c1, g, 2 * half, tol2, [&](int k, int& xs, int& xc, int& ys, int& yc) {
          const int blk = k / half, pr = k % half;
          int a, b;
          if (pr == 0) { a = 0; b = 1 + step; }
          else {
            a = step + pr; a = (a >= B - 1 ? a - (B - 1) : a) + 1;
            b = step - pr + B - 1; b = (b >= B - 1 ? b - (B - 1) : b) + 1;
          }
          if (a > b) { const int t = a; a = b; b = t; }
          xs = ys = blk;
          xc = a;
          yc = b;
          const Slot& sb = blk ? c1 : c0;
          return b < bs && col_live(sb, a, g.n) && col_live(sb, b, g.n);
        });
      }
    }
    BJ_T(2);
    for (int st = 0; st < NB - 1; ++st) {
      // inter phase: all bs^2 pairs (top col i, bottom col (i + t) % bs)
      rot |= inter_step<TPP, RPL>(c0, c1, g, tol2);
      BJ_T(3);
      const bool last = (st == NB - 2);
      if (last) {
        // cluster-wide OR of "rotated this sweep": write my flag everywhere
        const int any = __syncthreads_or((rot & ROT_BIG) ? 1 : 0);
        if (threadIdx.x < CL) {
          double* dst = cl.map_shared_rank(&flags[(sweep & 1) * CL + me], (int)threadIdx.x);
          *dst = any ? 1.0 : 0.0;
        }
      }
      // generic-proxy writes of this step -> visible to the async-proxy bulk copies
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      BJ_T(4);
      // two sets: every CTA done with this step (its incoming copies consumed)
      // before new blocks may overwrite them; three sets: only for the vote
      if (last || nset == 2) cluster_barrier();
      BJ_T(5);
      if (last) {
        double tot = 0.0;
        for (int c = 0; c < CL; ++c) tot += flags[(sweep & 1) * CL + c];
        converged = (tot == 0.0);
        rot = 0;
      }
      if (last && (converged || sweep + 1 >= max_sweeps)) break;
      // move both blocks to their next owners (set -> next set)
      const int nxt = (set + 1 == nset) ? 0 : set + 1;
      if (threadIdx.x == 0) {
        mbar_arrive_expect(&mbar[nxt], 2u * slot_bytes);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const uint32_t off0 = (uint32_t)((size_t)(nxt * 2 + d0s) * g.slot * sizeof(double));
        const uint32_t off1 = (uint32_t)((size_t)(nxt * 2 + d1s) * g.slot * sizeof(double));
        const uint32_t mb = (uint32_t)(nxt * sizeof(uint64_t));
        bulk_to_cluster(cluster_map(slots_u32 + off0, d0c), c0.w, slot_bytes,
                        cluster_map(mbar_u32 + mb, d0c));
        bulk_to_cluster(cluster_map(slots_u32 + off1, d1c), c1.w, slot_bytes,
                        cluster_map(mbar_u32 + mb, d1c));
      }
      BJ_T(6);
      mbar_wait(&mbar[nxt], use[nxt] & 1u);
      ++use[nxt];
      BJ_T(7);
      set = nxt;
      c0 = slot_at(slots, g, set, 0);
      c1 = slot_at(slots, g, set, 1);
    }
    ++sweep;
  }
  // exact final norms, then all-gather by column id
  const Slot f0 = slot_at(slots, g, set, 0), f1 = slot_at(slots, g, set, 1);
  for (int t = threadIdx.x; t < 2 * bs; t += blockDim.x) {
    const Slot& s = (t < bs) ? f0 : f1;
    const int c = t % bs;
    const double* w = s.w + (size_t)c * g.ld;
    double a = 0.0;
    for (int i = 0; i < g.nrows; ++i) a = fma(w[i], w[i], a);
    s.nrm[c] = a;
    const int id = (int)s.id[c];
    if (id < g.n)
      for (int r = 0; r < CL; ++r) *cl.map_shared_rank(&gnorm[id], r) = a;
  }
  cluster_barrier();
  cur_set = set;
  return sweep;
}

// initial ownership: CTA c holds block c (top) and block 2CL-1-c (bottom)
__device__ __forceinline__ int init_block(int me, int t, int CL) { return t == 0 ? me : 2 * CL - 1 - me; }

template <int CL>
struct Smem {
  uint64_t* mbar;
  double* flags;
  double* gnorm;
  double* slots;
};
template <int CL>
__device__ __forceinline__ Smem<CL> carve(double* base, const Geo& g) {
  Smem<CL> s;
  s.mbar = reinterpret_cast<uint64_t*>(base);
  s.flags = base + 4;
  s.gnorm = s.flags + 2 * CL;
  s.slots = s.gnorm + 2 * CL * g.bs;
  return s;
}

template <int CL>
__device__ void setup(cg::cluster_group& cl, const Smem<CL>& sm) {
  if (threadIdx.x == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    mbar_init(&sm.mbar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int t = threadIdx.x; t < 2 * CL; t += blockDim.x) sm.flags[t] = 0.0;
  __syncthreads();
  cluster_barrier();
}

// rank of column id j among the n gathered norms (descending, ties -> lower id)
__device__ __forceinline__ int rank_of(const double* key, int n, int j) {
  const double kj = key[j];
  int rank = 0;
  for (int i = 0; i < n; ++i) {
    const double ki = key[i];
    rank += (ki > kj) || (ki == kj && i < j);
  }
  return rank;
}

// ------------------------------------------------------------ merge core --
template <int CL, int TPP, int RPL>
__global__ void __launch_bounds__(RPL >= 16 ? 384 : 512)
    merge_core_kernel(const double* __restrict__ sig1, int l1, const double* __restrict__ M,
                      int64_t ldm, const double* __restrict__ Rm, int64_t ldr,
                      const double* __restrict__ sig2, int l2, int r, int rcap,
                      double* __restrict__ T, int64_t ldt, int tcols, double* __restrict__ sig_new,
                      int64_t* __restrict__ info, int max_sweeps, int trans, int nset,
                      const int32_t* __restrict__ gate) {
  // gate (optional, device): 0 = skip -- the re-run of a speculative merge
  // core when the second projection did not fire (uniform over the cluster)
  if (gate != nullptr && *gate == 0) return;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double smem_bj[];
  const int n = l1 + l2;
  // trans: one-sided Jacobi on E^T (lower block-triangular, ~10 sweeps instead
  // of ~14 on E) with the rotations accumulated in J: E^T J = W gives
  // E = J (W^T), so U_E = J and sigma = ||W columns||
  const Geo g(n, n, trans ? n : 0, CL);
  const Smem<CL> sm = carve<CL>(smem_bj, g);
  const int me = (int)cl.block_rank();
  // E = [[S1, M S2], [0, R S2]] columns of the two owned blocks
  for (int t2 = 0; t2 < 2; ++t2) {
    const Slot s = slot_at(sm.slots, g, 0, t2);
    const int blk = init_block(me, t2, CL);
    for (int t = threadIdx.x; t < g.bs * g.ld; t += blockDim.x) {
      const int c = t / g.ld, ii0 = t - c * g.ld;
      const int jj0 = blk * g.bs + c;
      const int i = trans ? jj0 : ii0, j = trans ? ii0 : jj0;  // element E[i, j]
      double e = 0.0;
      if (j < n && i < n) {
        if (j < l1) e = (i == j) ? sig1[j] : 0.0;
        else {
          const int jj = j - l1;
          if (i < l1) e = M[i + (int64_t)jj * ldm] * sig2[jj];
          else {
            const int ii = i - l1;
            e = (ii <= jj) ? Rm[ii + (int64_t)jj * ldr] * sig2[jj] : 0.0;
          }
        }
      }
      s.w[t] = e;
    }
    if (trans)
      for (int t = threadIdx.x; t < g.bs * g.ldj; t += blockDim.x) {
        const int c = t / g.ldj, i = t - c * g.ldj;
        s.j[t] = (i == blk * g.bs + c && i < n) ? 1.0 : 0.0;
      }
    for (int c = threadIdx.x; c < g.bse; c += blockDim.x) {
      s.id[c] = (double)(c < g.bs ? blk * g.bs + c : 1 << 30);
      s.nrm[c] = 0.0;
    }
  }
  setup<CL>(cl, sm);
  int set = 0;
  const int sweeps = run_sweeps<CL, TPP, RPL>(cl, g, sm.slots, sm.mbar, sm.flags, sm.gnorm, set,
                                         2.220446049250313e-16 * (double)max(n, 16), max_sweeps, nset);
  // sigma, keep (identical in every CTA)
  double s0 = 0.0;
  for (int i = 0; i < n; ++i) s0 = fmax(s0, sm.gnorm[i]);
  s0 = sqrt(s0);
  const double thr = 1e-14 * fmax(s0, 1e-300);
  int cnt = 0;
  for (int i = 0; i < n; ++i) cnt += sqrt(sm.gnorm[i]) > thr;
  const int keep = min(r, cnt);
  if (me == 0 && threadIdx.x == 0) {
    info[0] = keep;
    info[1] = sweeps;
  }
  if (me == 0)
    for (int k = keep + threadIdx.x; k < rcap; k += blockDim.x) sig_new[k] = 0.0;
  for (int t2 = 0; t2 < 2; ++t2) {
    const Slot s = slot_at(sm.slots, g, set, t2);
    for (int c = 0; c < g.bs; ++c) {
      const int id = (int)s.id[c];
      if (id >= n) continue;
      const int k = rank_of(sm.gnorm, n, id);
      if (k >= tcols) continue;
      const double sg = sqrt(sm.gnorm[id]);
      if (threadIdx.x == 0 && k < keep && k < rcap) sig_new[k] = sg;
      const double* w = s.w + (size_t)c * g.ld;
      const double* jc = s.j + (size_t)c * g.ldj;
      for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int row = (e < l1) ? e : rcap + (e - l1);
        T[row + (int64_t)k * ldt] = (k < keep) ? (trans ? jc[e] : w[e] / sg) : 0.0;
      }
    }
  }
  if (me == 0)
    for (int t = threadIdx.x; t < (rcap - l1) * tcols; t += blockDim.x) {
      const int k = t / (rcap - l1), row = l1 + t % (rcap - l1);
      T[row + (int64_t)k * ldt] = 0.0;
    }
  if (me == 0)  // columns beyond n (only when tcols > n)
    for (int t = threadIdx.x; t < (tcols > n ? (tcols - n) : 0) * (rcap + l2); t += blockDim.x) {
      const int k = n + t / (rcap + l2), row = t % (rcap + l2);
      T[row + (int64_t)k * ldt] = 0.0;
    }
  cluster_barrier();
}

// ------------------------------------------------------------- gram eigh --
template <int CL, int TPP, int RPL>
__global__ void __launch_bounds__(RPL >= 16 ? 384 : 512)
    gram_eigh_kernel(const double* __restrict__ X, const int* __restrict__ piv,
                     const int64_t* __restrict__ rank_in, int gdim, int r,
                     double* __restrict__ sigma_out, double* __restrict__ T, int64_t ldt,
                     int64_t* __restrict__ info, int max_sweeps, int nset) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double smem_bj[];
  const Geo g(gdim, gdim, 0, CL);
  const Smem<CL> sm = carve<CL>(smem_bj, g);
  const int me = (int)cl.block_rank();
  const int rank = (int)*rank_in;
  for (int t2 = 0; t2 < 2; ++t2) {
    const Slot s = slot_at(sm.slots, g, 0, t2);
    const int blk = init_block(me, t2, CL);
    for (int t = threadIdx.x; t < g.bs * g.ld; t += blockDim.x) {
      const int c = t / g.ld, i = t - c * g.ld;
      const int j = blk * g.bs + c;
      s.w[t] = (j < rank && i < gdim) ? X[i + (int64_t)j * gdim] : 0.0;
    }
    for (int c = threadIdx.x; c < g.bse; c += blockDim.x) {
      s.id[c] = (double)(c < g.bs ? blk * g.bs + c : 1 << 30);
      s.nrm[c] = 0.0;
    }
  }
  setup<CL>(cl, sm);
  int set = 0;
  const int sweeps = run_sweeps<CL, TPP, RPL>(cl, g, sm.slots, sm.mbar, sm.flags, sm.gnorm, set,
                                         2.220446049250313e-16 * (double)max(gdim, 16),
                                         max_sweeps, nset);
  // lambda = squared norms (ids >= rank are zero columns)
  double lam0 = 0.0;
  for (int i = 0; i < gdim; ++i) lam0 = fmax(lam0, sm.gnorm[i]);
  const double dust = 1e-12 * fmax(lam0, 2.2250738585072014e-308);  // matcore.py:26
  const double s0 = lam0 <= dust ? 0.0 : sqrt(lam0);
  int rk = 0;
  if (s0 > 0.0) {
    const double thr = 1e-14 * s0;  // matcore.py:20
    for (int i = 0; i < gdim; ++i) {
      const double lam = sm.gnorm[i];
      rk += (lam <= dust ? 0.0 : sqrt(lam)) > thr;
    }
  }
  const int keep = min(r, rk);
  if (me == 0 && threadIdx.x == 0) {
    info[0] = rk;
    info[1] = keep;
    info[2] = sweeps;
  }
  for (int t2 = 0; t2 < 2; ++t2) {
    const Slot s = slot_at(sm.slots, g, set, t2);
    for (int c = 0; c < g.bs; ++c) {
      const int id = (int)s.id[c];
      if (id >= gdim) continue;
      const int k = rank_of(sm.gnorm, gdim, id);
      const double lam = sm.gnorm[id];
      const double sg = lam <= dust ? 0.0 : sqrt(lam);
      if (threadIdx.x == 0) sigma_out[k] = sg;
      if (k >= r) continue;
      const double* w = s.w + (size_t)c * g.ld;
      const double nrm = sqrt(lam);
      for (int i = threadIdx.x; i < gdim; i += blockDim.x)
        T[piv[i] + (int64_t)k * ldt] = (k < keep) ? w[i] / nrm / sg : 0.0;
    }
  }
  if (me == 0)  // output columns beyond g (only when r > g)
    for (int t = threadIdx.x; t < (r > gdim ? r - gdim : 0) * gdim; t += blockDim.x) {
      const int k = gdim + t / gdim, i = t % gdim;
      T[i + (int64_t)k * ldt] = 0.0;
    }
  cluster_barrier();
}

// ------------------------------------------------------------- svd small --
template <int CL, int TPP, int RPL>
__global__ void __launch_bounds__(RPL >= 16 ? 384 : 512)
    svd_kernel(const double* __restrict__ A, int64_t lda, int nr, int nc, double* __restrict__ U,
               int64_t ldu, double* __restrict__ sigma, double* __restrict__ V, int64_t ldv,
               int64_t* __restrict__ info, int max_sweeps, int nset) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double smem_bj[];
  const Geo g(nc, nr, V ? nc : 0, CL);
  const Smem<CL> sm = carve<CL>(smem_bj, g);
  const int me = (int)cl.block_rank();
  for (int t2 = 0; t2 < 2; ++t2) {
    const Slot s = slot_at(sm.slots, g, 0, t2);
    const int blk = init_block(me, t2, CL);
    for (int t = threadIdx.x; t < g.bs * g.ld; t += blockDim.x) {
      const int c = t / g.ld, i = t - c * g.ld;
      const int j = blk * g.bs + c;
      s.w[t] = (j < nc && i < nr) ? A[i + (int64_t)j * lda] : 0.0;
    }
    if (V)
      for (int t = threadIdx.x; t < g.bs * g.ldj; t += blockDim.x) {
        const int c = t / g.ldj, i = t - c * g.ldj;
        const int j = blk * g.bs + c;
        s.j[t] = (j < nc && i == j) ? 1.0 : 0.0;
      }
    for (int c = threadIdx.x; c < g.bse; c += blockDim.x) {
      s.id[c] = (double)(c < g.bs ? blk * g.bs + c : 1 << 30);
      s.nrm[c] = 0.0;
    }
  }
  setup<CL>(cl, sm);
  int set = 0;
  const int sweeps = run_sweeps<CL, TPP, RPL>(cl, g, sm.slots, sm.mbar, sm.flags, sm.gnorm, set,
                                         2.220446049250313e-16 * (double)max(nr, 16), max_sweeps, nset);
  if (me == 0 && threadIdx.x == 0) info[0] = sweeps;
  for (int t2 = 0; t2 < 2; ++t2) {
    const Slot s = slot_at(sm.slots, g, set, t2);
    for (int c = 0; c < g.bs; ++c) {
      const int id = (int)s.id[c];
      if (id >= nc) continue;
      const int k = rank_of(sm.gnorm, nc, id);
      const double sg = sqrt(sm.gnorm[id]);
      if (threadIdx.x == 0) sigma[k] = sg;
      if (U) {
        const double* w = s.w + (size_t)c * g.ld;
        for (int i = threadIdx.x; i < nr; i += blockDim.x)
          U[i + (int64_t)k * ldu] = sg > 0.0 ? w[i] / sg : 0.0;
      }
      if (V) {
        const double* j = s.j + (size_t)c * g.ldj;
        for (int i = threadIdx.x; i < nc; i += blockDim.x) V[i + (int64_t)k * ldv] = j[i];
      }
    }
  }
  cluster_barrier();
}

// ----------------------------------------------------------------- host ---
static int set_smem(const void* fn) {
  static const void* fns[32];
  static int nf = 0;
  for (int i = 0; i < nf; ++i)
    if (fns[i] == fn) return POD_OK;
  cudaError_t e =
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_CAP);
  if (e != cudaSuccess) return cuda_status(e, "block jacobi smem attr");
  if (nf < 32) fns[nf++] = fn;
  return POD_OK;
}

// Each solver CTA reserves the whole shared-memory carve-out (POD_BJ_EXCLUSIVE,
// default on): no CTA of a concurrent GEMM can then be co-resident on the
// cluster's SMs and stretch the latency-bound rotation chain.
static bool exclusive_sms() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_BJ_EXCLUSIVE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename K, typename... Args>
static int launch(K kernel, int cl, int threads, size_t smem, cudaStream_t stream, Args... args) {
  if (exclusive_sms()) smem = SMEM_CAP;
  int st = set_smem((const void*)kernel);
  if (st) return st;
  if (cl > 8) {  // 16-CTA clusters are a non-portable size on sm_100a
    cudaError_t e =
        cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_status(e, "block jacobi cluster attr");
  }
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
  return e == cudaSuccess ? POD_OK : cuda_status(e, "block jacobi launch");
}

// Lanes per column pair: a power of two near nrows/4 (8..32) -- fewer lanes
// mean fewer shuffle levels on the per-sub-round critical path, more rows
// per lane in registers.  Threads = bs pairs x lanes in whole warps.
static int lanes_for(const Geo& g) {
  static int div = -1;
  if (div < 0) {  // POD_BJ_ROWS_PER_LANE: tuning override of the target rows per lane
    const char* e = getenv("POD_BJ_ROWS_PER_LANE");
    div = e ? std::max(1, atoi(e)) : 4;
  }
  const int want = std::max(8, std::min(32, g.nrows / div));
  int tpp = 8;
  while (tpp * 2 <= want) tpp *= 2;
  while (tpp > 8 && g.bs * tpp > 384) tpp /= 2;
  return tpp;
}
static int threads_for(const Geo& g, int tpp) { return ((g.bs * tpp + 31) / 32) * 32; }

}  // namespace bj

constexpr int BJ_CL = 8;
static const int BJ_NOT_APPLICABLE = -1;

// POD_BJ_TRANS=0: merge E-SVD on E itself instead of E^T (A/B measurements)
static bool bj_trans_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_BJ_TRANS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static bool bj_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_JACOBI");
    v = (e && e[0] == 'c') ? 0 : 1;  // POD_JACOBI=cluster: row-distributed solver
  }
  return v == 1;
}

int bj_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                  int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                  int64_t ldt, int64_t tcols, double* sig_new, int64_t* info,
                  const int32_t* gate, bool probe, cudaStream_t stream) {
  // probe: return POD_OK without launching when this solver handles the size
  if (!bj_enabled()) return BJ_NOT_APPLICABLE;
  const int n = (int)(l1 + l2);
  if (n < 2 * BJ_CL) return BJ_NOT_APPLICABLE;
  // preference: E^T with accumulated J (~10 instead of ~14 sweeps) at 8
  // CTAs; then E itself at 8, then 16 CTAs -- the first geometry that fits
  // (measured: E^T on a 16-CTA cluster is slower than E on 8 or 16)
  for (int variant = 0; variant < 4; ++variant) {
    const int trans = variant == 0 ? (bj_trans_enabled() ? 1 : 0) : 0;
    if (variant < 2 && !trans) continue;
    const int cl = (variant % 2 == 0) ? BJ_CL : 16;
    const bj::Geo g(n, n, trans ? n : 0, cl);
    const int nset = g.smem_bytes(cl, 3) <= bj::SMEM_CAP ? 3 : 2;
    const size_t bytes = g.smem_bytes(cl, nset);
    if (bytes > bj::SMEM_CAP) continue;
    const int tpp = bj::lanes_for(g);
    const int th = bj::threads_for(g, tpp);
    const int rpl = (g.nrows + tpp - 1) / tpp;
    if (th > 512 || (rpl > 8 && th > 384)) continue;
#define BJ_L(C_, T_, R_) return probe ? POD_OK : bj::launch(bj::merge_core_kernel<C_, T_, R_>, C_, th, bytes, stream, sig1, (int)l1, M, ldm, R, ldr, sig2, (int)l2, (int)r, (int)rcap, T, ldt, (int)tcols, sig_new, info, 60, trans, nset, gate)
    if (cl == BJ_CL) {
      if (tpp == 8) { if (rpl <= 4) BJ_L(BJ_CL, 8, 4); if (rpl <= 8) BJ_L(BJ_CL, 8, 8); if (rpl <= 16) BJ_L(BJ_CL, 8, 16); if (rpl <= 24) BJ_L(BJ_CL, 8, 24); BJ_L(BJ_CL, 8, 0); }
      if (tpp == 16) { if (rpl <= 4) BJ_L(BJ_CL, 16, 4); if (rpl <= 8) BJ_L(BJ_CL, 16, 8); if (rpl <= 16) BJ_L(BJ_CL, 16, 16); if (rpl <= 24) BJ_L(BJ_CL, 16, 24); BJ_L(BJ_CL, 16, 0); }
      if (rpl <= 4) BJ_L(BJ_CL, 32, 4); if (rpl <= 8) BJ_L(BJ_CL, 32, 8); if (rpl <= 16) BJ_L(BJ_CL, 32, 16); if (rpl <= 24) BJ_L(BJ_CL, 32, 24); BJ_L(BJ_CL, 32, 0);
    } else {
      if (th > 384) continue;
      if (tpp == 32) { if (rpl <= 16) BJ_L(16, 32, 16); if (rpl <= 24) BJ_L(16, 32, 24); BJ_L(16, 32, 0); }
      if (tpp == 16) { if (rpl <= 24) BJ_L(16, 16, 24); BJ_L(16, 16, 0); }
      continue;
    }
#undef BJ_L
  }
  return BJ_NOT_APPLICABLE;
}

int bj_gram_eigh(const double* X, const int* piv, const int64_t* rank, int64_t gd, int64_t r,
                 double* sigma, double* T, int64_t ldt, int64_t* info, cudaStream_t stream) {
  if (!bj_enabled()) return BJ_NOT_APPLICABLE;
  const bj::Geo g((int)gd, (int)gd, 0, BJ_CL);
  const int nset = g.smem_bytes(BJ_CL, 3) <= bj::SMEM_CAP ? 3 : 2;
  const size_t bytes = g.smem_bytes(BJ_CL, nset);
  if (bytes > bj::SMEM_CAP || gd < 2 * BJ_CL) return BJ_NOT_APPLICABLE;
  const int tpp = bj::lanes_for(g);
  const int th = bj::threads_for(g, tpp);
  const int rpl = (g.nrows + tpp - 1) / tpp;
  if (th > 512 || (rpl > 8 && th > 384)) return BJ_NOT_APPLICABLE;
#define BJ_L(T_, R_) bj::launch(bj::gram_eigh_kernel<BJ_CL, T_, R_>, BJ_CL, th, bytes, stream, X, piv, rank, (int)gd, (int)r, sigma, T, ldt, info, 60, nset)
#define BJ_R(T_)                         \
  if (rpl <= 4) return BJ_L(T_, 4);      \
  if (rpl <= 8) return BJ_L(T_, 8);      \
  if (rpl <= 16) return BJ_L(T_, 16);    \
  if (rpl <= 24) return BJ_L(T_, 24);    \
  return BJ_L(T_, 0);
  if (tpp == 8) { BJ_R(8) }
  if (tpp == 16) { BJ_R(16) }
  BJ_R(32)
#undef BJ_R
#undef BJ_L
}

int bj_svd(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
           double* sigma, double* V, int64_t ldv, int64_t* info, cudaStream_t stream) {
  if (!bj_enabled()) return BJ_NOT_APPLICABLE;
  const bj::Geo g((int)nc, (int)nr, V ? (int)nc : 0, BJ_CL);
  const int nset = g.smem_bytes(BJ_CL, 3) <= bj::SMEM_CAP ? 3 : 2;
  const size_t bytes = g.smem_bytes(BJ_CL, nset);
  if (bytes > bj::SMEM_CAP || nc < 2 * BJ_CL) return BJ_NOT_APPLICABLE;
  const int tpp = bj::lanes_for(g);
  const int th = bj::threads_for(g, tpp);
  const int rpl = (g.nrows + tpp - 1) / tpp;
  if (th > 512 || (rpl > 8 && th > 384)) return BJ_NOT_APPLICABLE;
#define BJ_L(T_, R_) bj::launch(bj::svd_kernel<BJ_CL, T_, R_>, BJ_CL, th, bytes, stream, A, lda, (int)nr, (int)nc, U, ldu, sigma, V, ldv, info, 60, nset)
#define BJ_R(T_)                         \
  if (rpl <= 4) return BJ_L(T_, 4);      \
  if (rpl <= 8) return BJ_L(T_, 8);      \
  if (rpl <= 16) return BJ_L(T_, 16);    \
  if (rpl <= 24) return BJ_L(T_, 24);    \
  return BJ_L(T_, 0);
  if (tpp == 8) { BJ_R(8) }
  if (tpp == 16) { BJ_R(16) }
  BJ_R(32)
#undef BJ_R
#undef BJ_L
}

}  // namespace pod

#ifdef POD_BJ_TIMING
extern "C" int pod_debug_bj_phase(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, pod::bj::g_bj_phase, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(pod::bj::g_bj_phase, z, sizeof(z));
  }
  return 0;
}
#endif
