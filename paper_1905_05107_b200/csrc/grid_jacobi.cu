// Grid-wide column-block one-sided Jacobi for the problems too large for one
// thread-block cluster's shared memory (sampled Gram of g > ~400 distinct
// columns -- the reference's default column budget ltsvd_sample_count(k, 0.7,
// 0.6) gives c = 746 draws at k = 10 -- merge E-SVDs with l1 + l2 > ~480, and
// the dense SVDs of matcore.py:187-254).
//
// Same algorithm and visiting order as block_jacobi.cu (bj_core.cuh): the n
// columns are cut into NB = 2P blocks of bs columns, CTA p of a P-CTA grid
// owns two blocks, one sweep = an intra phase plus NB - 1 round-robin block
// tournament steps.  The difference is where the blocks travel between steps:
// through two global (L2-resident) block sets instead of DSMEM, with a
// grid-wide barrier per step.  The kernel is launched cooperatively so all P
// CTAs are co-resident.  Build (prologue) and output (epilogue) stages are
// separate small kernels that read/write the global block sets directly.
#include "bj_core.cuh"

namespace pod {
namespace gj {

using bj::Geo;
using bj::Slot;

constexpr size_t SMEM_CAP = bj::SMEM_CAP;
constexpr int MAX_SWEEPS = 60;

// Barrier / flag block at the head of the workspace (zeroed before the
// sweep kernel by the prologue).
struct Ctl {
  unsigned count;
  unsigned gen;
  int rot[2];
  int sweeps;
  int fin;  // block set holding the converged blocks
  int pad[2];
};

struct Layout {
  Geo g;
  int P;
  size_t set_doubles;  // one block set: 2P slots
  __host__ __device__ Layout(int n, int nrows, int njrows, int P_)
      : g(n, nrows, njrows, P_), P(P_), set_doubles((size_t)2 * P_ * g.slot) {}
  __host__ __device__ double* set_base(double* ws, int set) const {
    return ws + 8 + (size_t)set * set_doubles;  // 8 doubles = Ctl (padded)
  }
  __host__ __device__ double* gnorm(double* ws) const { return ws + 8 + 2 * set_doubles; }
  __host__ __device__ size_t ws_bytes() const {
    return (8 + 2 * set_doubles + (size_t)g.n + 8) * sizeof(double);
  }
  __host__ size_t smem_bytes() const { return (size_t)2 * g.slot * sizeof(double); }
};

// slot t (0 top, 1 bottom) of position p in a global block set
__device__ __forceinline__ Slot gslot(const Layout& L, double* ws, int set, int p, int t) {
  return bj::slot_at(L.set_base(ws, set), L.g, 0, 2 * p + t);
}
// initial ownership (block_jacobi.cu init_block): CTA p holds blocks p and 2P-1-p
__device__ __forceinline__ int init_block(int p, int t, int P) { return t == 0 ? p : 2 * P - 1 - p; }

__device__ __forceinline__ void grid_barrier(Ctl* c, int nblk) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &c->gen;
    const unsigned g0 = *vgen;
    __threadfence();
    if (atomicAdd(&c->count, 1u) == (unsigned)nblk - 1) {
      atomicExch(&c->count, 0u);
      __threadfence();
      atomicAdd(&c->gen, 1u);
    } else {
      while (*vgen == g0) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

// smem <- global slot (L2; bypass L1 -- other CTAs wrote it)
__device__ __forceinline__ void load_slot(double* dst, const double* src, int nd) {
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (int i = threadIdx.x; i < nd / 2; i += blockDim.x) d2[i] = __ldcg(s2 + i);
}
__device__ __forceinline__ void store_slot(double* dst, const double* src, int nd) {
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (int i = threadIdx.x; i < nd / 2; i += blockDim.x) __stcg(d2 + i, s2[i]);
}

template <int TPP, int RPL>
__global__ void __launch_bounds__(512) sweep_kernel(double* ws, int n, int nrows, int njrows,
                                                    int P, double tol) {
  extern __shared__ __align__(16) double smem_gj[];
  const Layout L(n, nrows, njrows, P);
  const Geo& g = L.g;
  Ctl* ctl = reinterpret_cast<Ctl*>(ws);
  const int me = blockIdx.x;
  const int bs = g.bs;
  const int NB = 2 * P;
  const double tol2 = tol * tol;
  // destinations of this CTA's top / bottom block after a step (circle method)
  int d0c, d0s, d1c, d1s;
  if (me == 0) { d0c = 0; d0s = 0; d1c = 1; d1s = 0; }
  else {
    d1c = me - 1; d1s = 1;
    if (me == P - 1) { d0c = me; d0s = 1; }
    else { d0c = me + 1; d0s = 0; }
  }
  const Slot c0 = bj::slot_at(smem_gj, g, 0, 0), c1 = bj::slot_at(smem_gj, g, 0, 1);
  int set = 0;
  load_slot(c0.w, gslot(L, ws, set, me, 0).w, g.slot);
  load_slot(c1.w, gslot(L, ws, set, me, 1).w, g.slot);
  __syncthreads();
  int sweep = 0;
  bool converged = false;
  while (sweep < MAX_SWEEPS && !converged) {
    for (int t = threadIdx.x; t < 2 * bs; t += blockDim.x) {  // exact squared norms
      const Slot& s = (t < bs) ? c0 : c1;
      const int c = t % bs;
      const double* w = s.w + (size_t)c * g.ld;
      double a = 0.0;
      for (int i = 0; i < g.nrows; ++i) a = fma(w[i], w[i], a);
      s.nrm[c] = a;
    }
    __syncthreads();
    int rot = 0;
    {  // intra phase: round-robin inside each owned block
      const int B = bs + (bs & 1);
      for (int step = 0; step < B - 1; ++step) {
        const int half = B / 2;
        rot |= bj::sub_round<TPP, RPL>(c0, c1, g, 2 * half, tol2,
                                       [&](int k, int& xs, int& xc, int& ys, int& yc) {
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
          return b < bs && bj::col_live(sb, a, g.n) && bj::col_live(sb, b, g.n);
        });
      }
    }
    for (int st = 0; st < NB - 1; ++st) {
      rot |= bj::inter_step<TPP, RPL>(c0, c1, g, tol2);
      const bool last = (st == NB - 2);
      if (last) {
        const int any = __syncthreads_or((rot & bj::ROT_BIG) ? 1 : 0);
        if (threadIdx.x == 0 && any) atomicOr(&ctl->rot[sweep & 1], 1);
        if (me == 0 && threadIdx.x == 0) ctl->rot[(sweep + 1) & 1] = 0;  // next sweep's flag
      }
      const int nxt = 1 - set;
      store_slot(gslot(L, ws, nxt, d0c, d0s).w, c0.w, g.slot);
      store_slot(gslot(L, ws, nxt, d1c, d1s).w, c1.w, g.slot);
      grid_barrier(ctl, P);
      set = nxt;
      if (last) {
        converged = (*(volatile int*)&ctl->rot[sweep & 1]) == 0;
        rot = 0;
      }
      load_slot(c0.w, gslot(L, ws, set, me, 0).w, g.slot);
      load_slot(c1.w, gslot(L, ws, set, me, 1).w, g.slot);
      __syncthreads();
    }
    ++sweep;
    // every CTA must have read this sweep's flag before it is reset (at the
    // next sweep's last step, >= 1 barrier away when NB - 1 >= 2)
  }
  // exact final norms by column id
  double* gn = L.gnorm(ws);
  for (int t = threadIdx.x; t < 2 * bs; t += blockDim.x) {
    const Slot& s = (t < bs) ? c0 : c1;
    const int c = t % bs;
    const double* w = s.w + (size_t)c * g.ld;
    double a = 0.0;
    for (int i = 0; i < g.nrows; ++i) a = fma(w[i], w[i], a);
    const int id = (int)s.id[c];
    if (id < g.n) gn[id] = a;
  }
  if (me == 0 && threadIdx.x == 0) {
    ctl->sweeps = sweep;
    ctl->fin = set;
  }
}

// ------------------------------------------------ grid pivoted Cholesky --
// Stage 1 of pod_gram_eigh for g beyond small.cu's single-CTA kernel: the
// same right-looking pivoted Cholesky P G P^T = R^T R (largest remaining
// diagonal, ties to the lower index, stop at d <= 1e-15 d_0), with W's
// columns dealt cyclically over P CTAs and one grid barrier per step.  Every
// CTA forms the whole r_j (from row / column p of W, read from L2) so the
// rank-1 update of its columns needs no further exchange; the next pivot is
// the max over per-CTA candidates.  Output as small.cu: X = R^T (pivoted
// order, zero columns >= rank, written over W), piv, rank.
struct PcScratch {
  double* cv;  // [2][P] candidate diagonal values (step parity)
  int* ci;     // [2][P] candidate indices
};

__global__ void __launch_bounds__(512) gpivchol_kernel(const double* __restrict__ G, int64_t ldg,
                                                       int g, double* W, double* Rq,
                                                       int* __restrict__ piv_out,
                                                       int64_t* __restrict__ rank_out, Ctl* ctl,
                                                       double* cv, int* ci) {
  extern __shared__ __align__(16) double sm_pc[];
  double* r = sm_pc;                                 // [g]
  int* done = reinterpret_cast<int*>(sm_pc + g);     // [g]
  __shared__ double s_d0, s_d, s_bv[16];
  __shared__ int s_p, s_bi[16];
  const int P = gridDim.x, me = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  auto W_at = [&](int a, int b) -> double {  // symmetric element from lower storage (L2)
    return a >= b ? __ldcg(W + a + (int64_t)b * g) : __ldcg(W + b + (int64_t)a * g);
  };
  // block-wide argmax over this CTA's live columns of the diagonal -> cand[par][me]
  auto local_pick = [&](int par) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int b = me + P * threadIdx.x; b < g; b += P * blockDim.x) {
      if (done[b]) continue;
      const double v = W[b + (int64_t)b * g];
      if (v > bv) { bv = v; bi = b; }  // b ascending per thread: ties keep the lower
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { s_bv[warp] = bv; s_bi[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nwarp; ++w)
        if (s_bv[w] > bv || (s_bv[w] == bv && s_bi[w] < bi)) { bv = s_bv[w]; bi = s_bi[w]; }
      __stcg(cv + par * P + me, bv);
      __stcg(ci + par * P + me, bi);
    }
  };
  for (int b = me + P * warp; b < g; b += P * nwarp)  // own columns, lower part
    for (int a = b + lane; a < g; a += 32) W[a + (int64_t)b * g] = G[a + (int64_t)b * ldg];
  for (int q = threadIdx.x; q < g; q += blockDim.x) done[q] = 0;
  __syncthreads();
  local_pick(0);
  grid_barrier(ctl, P);
  int rank = g;
  for (int j = 0; j < g; ++j) {
    const int par = j & 1;
    if (threadIdx.x == 0) {  // global pivot = max over the P candidates
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int c = 0; c < P; ++c) {
        const double v = __ldcg(cv + par * P + c);
        const int i = __ldcg(ci + par * P + c);
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
      }
      if (j == 0) s_d0 = bv;
      s_d = bv;
      s_p = bi;
    }
    __syncthreads();
    const double d = s_d;
    if (!(d > 1e-15 * s_d0 && d > 0.0)) {  // remaining block negligible
      rank = j;
      break;
    }
    const int p = s_p;
    const double rjj = sqrt(d);
    for (int q = threadIdx.x; q < g; q += blockDim.x) {
      double v = 0.0;
      if (!done[q]) v = (q == p) ? rjj : W_at(p, q) / rjj;
      if (me == 0) __stcg(Rq + j + (int64_t)q * g, v);
      r[q] = (q == p) ? 0.0 : v;  // p leaves the Schur complement
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      done[p] = 1;
      if (me == 0) __stcg(piv_out + j, p);
    }
    __syncthreads();
    // rank-1 update of this CTA's live columns (rows >= column, live rows)
    for (int b = me + P * warp; b < g; b += P * nwarp) {
      if (done[b]) continue;
      const double rb = r[b];
      double* col = W + (int64_t)b * g;
      for (int a = b + lane; a < g; a += 32)
        if (!done[a]) col[a] = col[a] - r[a] * rb;
    }
    __syncthreads();
    local_pick(par ^ 1);
    grid_barrier(ctl, P);
  }
  if (me == 0 && threadIdx.x == 0) {  // never-eliminated indices after rank: ascending
    int k = rank;
    for (int q = 0; q < g; ++q)
      if (!done[q]) __stcg(piv_out + k++, q);
    __stcg(rank_out, (int64_t)rank);
  }
  grid_barrier(ctl, P);  // W no longer read; piv / Rq complete
  // X[i][jj] = R[jj][piv[i]] for jj < rank, i >= jj; zero elsewhere (over W)
  for (int jj = me + P * warp; jj < g; jj += P * nwarp)
    for (int i = lane; i < g; i += 32)
      W[i + (int64_t)jj * g] =
          (jj < rank && i >= jj) ? __ldcg(Rq + jj + (int64_t)__ldcg(piv_out + i) * g) : 0.0;
}

// ---------------------------------------------------------- prologues ----
// Block (p, t) of set 0: columns blk*bs + c of the problem matrix.

__device__ __forceinline__ void init_ids(const Slot& s, const Geo& g, int blk) {
  for (int c = threadIdx.x; c < g.bse; c += blockDim.x) {
    s.id[c] = (double)(c < g.bs ? blk * g.bs + c : 1 << 30);
    s.nrm[c] = 0.0;
  }
}
__device__ __forceinline__ void reset_ctl(double* ws) {
  if (blockIdx.x == 0 && threadIdx.x < 8) ws[threadIdx.x] = 0.0;
}

// X = R^T of the pivoted Cholesky (rank_in set), or G itself (direct mode,
// rank_in null): G J = V Lambda, so column norms are the eigenvalues
__global__ void gram_prologue(double* ws, int P, const double* __restrict__ X, int64_t ldx,
                              const int64_t* __restrict__ rank_in, int gd) {
  const Layout L(gd, gd, 0, P);
  const Geo& g = L.g;
  const int p = blockIdx.x >> 1, t2 = blockIdx.x & 1;
  const Slot s = gslot(L, ws, 0, p, t2);
  const int blk = init_block(p, t2, P);
  const int rank = rank_in ? (int)*rank_in : gd;
  for (int t = threadIdx.x; t < g.bs * g.ld; t += blockDim.x) {
    const int c = t / g.ld, i = t - c * g.ld;
    const int j = blk * g.bs + c;
    s.w[t] = (j < rank && i < gd) ? X[i + (int64_t)j * ldx] : 0.0;
  }
  init_ids(s, g, blk);
  reset_ctl(ws);
}

__global__ void svd_prologue(double* ws, int P, const double* __restrict__ A, int64_t lda, int nr,
                             int nc, int withv) {
  const Layout L(nc, nr, withv ? nc : 0, P);
  const Geo& g = L.g;
  const int p = blockIdx.x >> 1, t2 = blockIdx.x & 1;
  const Slot s = gslot(L, ws, 0, p, t2);
  const int blk = init_block(p, t2, P);
  for (int t = threadIdx.x; t < g.bs * g.ld; t += blockDim.x) {
    const int c = t / g.ld, i = t - c * g.ld;
    const int j = blk * g.bs + c;
    s.w[t] = (j < nc && i < nr) ? A[i + (int64_t)j * lda] : 0.0;
  }
  if (withv)
    for (int t = threadIdx.x; t < g.bs * g.ldj; t += blockDim.x) {
      const int c = t / g.ldj, i = t - c * g.ldj;
      const int j = blk * g.bs + c;
      s.j[t] = (j < nc && i == j) ? 1.0 : 0.0;
    }
  init_ids(s, g, blk);
  reset_ctl(ws);
}

// E = [[S1, M S2], [0, R S2]] (merge.py:80-83), or E^T with J = I (trans)
__global__ void merge_prologue(double* ws, int P, const double* __restrict__ sig1, int l1,
                               const double* __restrict__ M, int64_t ldm,
                               const double* __restrict__ Rm, int64_t ldr,
                               const double* __restrict__ sig2, int l2, int trans) {
  const int n = l1 + l2;
  const Layout L(n, n, trans ? n : 0, P);
  const Geo& g = L.g;
  const int p = blockIdx.x >> 1, t2 = blockIdx.x & 1;
  const Slot s = gslot(L, ws, 0, p, t2);
  const int blk = init_block(p, t2, P);
  for (int t = threadIdx.x; t < g.bs * g.ld; t += blockDim.x) {
    const int c = t / g.ld, ii0 = t - c * g.ld;
    const int jj0 = blk * g.bs + c;
    const int i = trans ? jj0 : ii0, j = trans ? ii0 : jj0;
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
  init_ids(s, g, blk);
  reset_ctl(ws);
}

// ---------------------------------------------------------- epilogues ----
// One CTA per final slot; all n squared norms staged in shared memory.

__device__ __forceinline__ int rank_of(const double* key, int n, int j) {
  const double kj = key[j];
  int rank = 0;
  for (int i = 0; i < n; ++i) {
    const double ki = key[i];
    rank += (ki > kj) || (ki == kj && i < j);
  }
  return rank;
}

__device__ __forceinline__ const double* stage_norms(const double* gn, int n) {
  extern __shared__ __align__(16) double sn[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sn[i] = gn[i];
  __syncthreads();
  return sn;
}

// block_jacobi.cu gram_eigh_kernel epilogue: dust rule, rank, keep, sigma, T
// (direct: the squared column norms are lambda^2; piv null = identity)
__global__ void gram_epilogue(double* ws, int P, int gd, int r, const int* __restrict__ piv,
                              double* __restrict__ sigma_out, double* __restrict__ T,
                              int64_t ldt, int64_t* __restrict__ info, int direct) {
  const Layout L(gd, gd, 0, P);
  const Geo& g = L.g;
  const Ctl* ctl = reinterpret_cast<const Ctl*>(ws);
  const double* gn = stage_norms(L.gnorm(ws), gd);
  auto lam_of = [&](int i) { return direct ? sqrt(gn[i]) : gn[i]; };
  double lam0 = 0.0;
  for (int i = 0; i < gd; ++i) lam0 = fmax(lam0, lam_of(i));
  const double dust = 1e-12 * fmax(lam0, 2.2250738585072014e-308);  // matcore.py:26
  const double s0 = lam0 <= dust ? 0.0 : sqrt(lam0);
  int rk = 0;
  if (s0 > 0.0) {
    const double thr = 1e-14 * s0;  // matcore.py:20
    for (int i = 0; i < gd; ++i) {
      const double lam = lam_of(i);
      rk += (lam <= dust ? 0.0 : sqrt(lam)) > thr;
    }
  }
  const int keep = min(r, rk);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = rk;
    info[1] = keep;
    info[2] = ctl->sweeps;
  }
  const int p = blockIdx.x >> 1, t2 = blockIdx.x & 1;
  const Slot s = gslot(L, ws, ctl->fin, p, t2);
  for (int c = 0; c < g.bs; ++c) {
    const int id = (int)s.id[c];
    if (id >= gd) continue;
    const int k = rank_of(gn, gd, id);
    const double lam = lam_of(id);
    const double sg = lam <= dust ? 0.0 : sqrt(lam);
    if (threadIdx.x == 0) sigma_out[k] = sg;
    if (k >= r) continue;
    const double* w = s.w + (size_t)c * g.ld;
    const double nrm = sqrt(gn[id]);
    for (int i = threadIdx.x; i < gd; i += blockDim.x)
      T[(piv ? piv[i] : i) + (int64_t)k * ldt] = (k < keep) ? w[i] / nrm / sg : 0.0;
  }
  if (blockIdx.x == 0)  // output columns beyond g (only when r > g)
    for (int t = threadIdx.x; t < (r > gd ? r - gd : 0) * gd; t += blockDim.x) {
      const int k = gd + t / gd, i = t % gd;
      T[i + (int64_t)k * ldt] = 0.0;
    }
}

__global__ void svd_epilogue(double* ws, int P, int nr, int nc, double* __restrict__ U,
                             int64_t ldu, double* __restrict__ sigma, double* __restrict__ V,
                             int64_t ldv, int64_t* __restrict__ info) {
  const Layout L(nc, nr, V ? nc : 0, P);
  const Geo& g = L.g;
  const Ctl* ctl = reinterpret_cast<const Ctl*>(ws);
  const double* gn = stage_norms(L.gnorm(ws), nc);
  if (blockIdx.x == 0 && threadIdx.x == 0) info[0] = ctl->sweeps;
  const int p = blockIdx.x >> 1, t2 = blockIdx.x & 1;
  const Slot s = gslot(L, ws, ctl->fin, p, t2);
  for (int c = 0; c < g.bs; ++c) {
    const int id = (int)s.id[c];
    if (id >= nc) continue;
    const int k = rank_of(gn, nc, id);
    const double sg = sqrt(gn[id]);
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

// block_jacobi.cu merge_core_kernel epilogue: keep rule (merge.py:85), the
// merged sigmas and the rotation T mapping [U1 Q] to the merged basis
__global__ void merge_epilogue(double* ws, int P, int l1, int l2, int r, int rcap,
                               double* __restrict__ T, int64_t ldt, int tcols,
                               double* __restrict__ sig_new, int64_t* __restrict__ info,
                               int trans) {
  const int n = l1 + l2;
  const Layout L(n, n, trans ? n : 0, P);
  const Geo& g = L.g;
  const Ctl* ctl = reinterpret_cast<const Ctl*>(ws);
  const double* gn = stage_norms(L.gnorm(ws), n);
  double s0 = 0.0;
  for (int i = 0; i < n; ++i) s0 = fmax(s0, gn[i]);
  s0 = sqrt(s0);
  const double thr = 1e-14 * fmax(s0, 1e-300);
  int cnt = 0;
  for (int i = 0; i < n; ++i) cnt += sqrt(gn[i]) > thr;
  const int keep = min(r, cnt);
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      info[0] = keep;
      info[1] = ctl->sweeps;
    }
    for (int k = keep + threadIdx.x; k < rcap; k += blockDim.x) sig_new[k] = 0.0;
    for (int t = threadIdx.x; t < (rcap - l1) * tcols; t += blockDim.x) {
      const int k = t / (rcap - l1), row = l1 + t % (rcap - l1);
      T[row + (int64_t)k * ldt] = 0.0;
    }
    for (int t = threadIdx.x; t < (tcols > n ? (tcols - n) : 0) * (rcap + l2); t += blockDim.x) {
      const int k = n + t / (rcap + l2), row = t % (rcap + l2);
      T[row + (int64_t)k * ldt] = 0.0;
    }
  }
  const int p = blockIdx.x >> 1, t2 = blockIdx.x & 1;
  const Slot s = gslot(L, ws, ctl->fin, p, t2);
  for (int c = 0; c < g.bs; ++c) {
    const int id = (int)s.id[c];
    if (id >= n) continue;
    const int k = rank_of(gn, n, id);
    if (k >= tcols) continue;
    const double sg = sqrt(gn[id]);
    if (threadIdx.x == 0 && k < keep && k < rcap) sig_new[k] = sg;
    const double* w = s.w + (size_t)c * g.ld;
    const double* jc = s.j + (size_t)c * g.ldj;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int row = (e < l1) ? e : rcap + (e - l1);
      T[row + (int64_t)k * ldt] = (k < keep) ? (trans ? jc[e] : w[e] / sg) : 0.0;
    }
  }
}

// ---------------------------------------------------------------- host ---
static int max_ctas() {
  static int v = 0;
  if (!v) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    v = sms;
  }
  return v;
}

// lanes per column pair (block_jacobi.cu lanes_for): a power of two near
// nrows / 4 in [8, 32], halved while bs pairs would exceed 512 threads
static int lanes(const Geo& g) {
  const int want = std::max(8, std::min(32, g.nrows / 4));
  int tpp = 8;
  while (tpp * 2 <= want) tpp *= 2;
  while (tpp > 8 && g.bs * tpp > 512) tpp /= 2;
  return tpp;
}
static int threads(const Geo& g) { return ((g.bs * lanes(g) + 31) / 32) * 32; }

// Smallest CTA count P >= 2 whose two blocks fit one CTA's shared memory
// with <= 512 threads; 0 when none does.
static int choose_P(int n, int nrows, int njrows) {
  for (int P = 2; P <= max_ctas(); ++P) {
    const Layout L(n, nrows, njrows, P);
    if (L.g.bs > 32 || L.smem_bytes() > SMEM_CAP || threads(L.g) > 512) continue;
    return P;
  }
  return 0;
}

template <typename K>
static int smem_attr(K fn, size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute((const void*)fn,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return e == cudaSuccess ? POD_OK : cuda_status(e, "grid jacobi smem attr");
}

template <int TPP, int RPL>
static int launch_sweep_t(const Layout& L, double* ws, double tol, cudaStream_t s) {
  auto fn = sweep_kernel<TPP, RPL>;
  int st = smem_attr(fn, SMEM_CAP);
  if (st) return st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.P, 1, 1);
  cfg.blockDim = dim3(((L.g.bs * TPP + 31) / 32) * 32, 1, 1);
  cfg.dynamicSmemBytes = L.smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all P CTAs co-resident (grid barrier)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, ws, L.g.n, L.g.nrows, L.g.njrows, L.P, tol);
  return e == cudaSuccess ? POD_OK : cuda_status(e, "grid jacobi launch");
}

static int launch_sweep(const Layout& L, double* ws, double tol, cudaStream_t s) {
  const int tpp = lanes(L.g);
  const int rpl = (L.g.nrows + tpp - 1) / tpp;
  if (tpp <= 8) return rpl <= 16 ? launch_sweep_t<8, 16>(L, ws, tol, s) : launch_sweep_t<8, 0>(L, ws, tol, s);
  if (tpp == 16) return rpl <= 16 ? launch_sweep_t<16, 16>(L, ws, tol, s) : launch_sweep_t<16, 0>(L, ws, tol, s);
  return rpl <= 16 ? launch_sweep_t<32, 16>(L, ws, tol, s) : launch_sweep_t<32, 0>(L, ws, tol, s);
}

static int launch_epilogue_smem(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return POD_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes);
  return e == cudaSuccess ? POD_OK : cuda_status(e, "grid jacobi epilogue smem");
}

}  // namespace gj

static double* gj_align(void* ws) {
  return (double*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
}

// Workspace bytes the grid solver needs for an n-column problem with nrows
// rows and njrows accumulated-rotation rows; 0 when it does not apply.
size_t gj_ws_bytes(int64_t n, int64_t nrows, int64_t njrows) {
  const int P = gj::choose_P((int)n, (int)nrows, (int)njrows);
  if (!P) return 0;
  return gj::Layout((int)n, (int)nrows, (int)njrows, P).ws_bytes() + 256;
}

// Workspace for pod_gram_eigh beyond the single-CTA pivoted Cholesky: W/X
// and Rq (g x g each), piv, rank, candidates, then the Jacobi block sets.
size_t gj_gram_large_ws_bytes(int64_t g) {
  const size_t jac = gj_ws_bytes(g, g, 0);
  if (!jac) return 0;
  return (size_t)2 * g * g * 8 + (size_t)g * 4 + 4 * 148 * 12 + 1024 + jac;
}

int gj_gram_eigh(const double* X, int64_t ldx, const int* piv, const int64_t* rank, int64_t g,
                 int64_t r, double* sigma, double* T, int64_t ldt, int64_t* info, void* ws,
                 size_t ws_bytes, cudaStream_t s);

// Grid pivoted Cholesky of G into the workspace: X = R^T (written over W),
// piv, rank; *rest / *rest_bytes = the workspace left for the Jacobi stage.
int gj_pivchol(const double* G, int64_t ldg, int64_t g, void* ws, size_t ws_bytes, double** Xo,
               int** pivo, int64_t** ranko, void** rest, size_t* rest_bytes, cudaStream_t s) {
  const size_t need = gj_gram_large_ws_bytes(g);
  POD_REQUIRE(need > 0, "gram eigh: g = %lld exceeds the grid Jacobi solver", (long long)g);
  POD_REQUIRE(ws_bytes >= need, "gram eigh: workspace too small (%zu < %zu)", ws_bytes, need);
  char* base = (char*)gj_align(ws);
  double* W = (double*)base;
  double* Rq = W + (size_t)g * g;
  int* piv = (int*)(Rq + (size_t)g * g);
  char* tail = (char*)(((uintptr_t)(piv + g) + 255) & ~(uintptr_t)255);
  gj::Ctl* ctl = (gj::Ctl*)tail;
  int64_t* rank = (int64_t*)(tail + 64);
  double* cv = (double*)(tail + 128);
  int* ci = (int*)(cv + 2 * 148);
  char* jws = (char*)(((uintptr_t)(ci + 2 * 148) + 255) & ~(uintptr_t)255);
  {
    cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(gj::Ctl), s);
    if (e != cudaSuccess) return cuda_status(e, "grid pivoted cholesky reset");
  }
  const int P = std::min(gj::max_ctas(), 148);
  const size_t smem = (size_t)g * 12;
  int st = gj::launch_epilogue_smem((const void*)gj::gpivchol_kernel, smem);
  if (st) return st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P, 1, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gj::gpivchol_kernel, G, ldg, (int)g, W, Rq, piv, rank,
                                     ctl, cv, ci);
  if (e != cudaSuccess) return cuda_status(e, "grid pivoted cholesky launch");
  *Xo = W;
  *pivo = piv;
  *ranko = rank;
  *rest = jws;
  *rest_bytes = ws_bytes - (size_t)(jws - (char*)ws);
  return POD_OK;
}

int gj_gram_eigh(const double* X, int64_t ldx, const int* piv, const int64_t* rank, int64_t g,
                 int64_t r, double* sigma, double* T, int64_t ldt, int64_t* info, void* ws,
                 size_t ws_bytes, cudaStream_t s);

int gj_gram_eigh_large(const double* G, int64_t ldg, int64_t g, int64_t r, double* sigma,
                       double* T, int64_t ldt, int64_t* info, void* ws, size_t ws_bytes,
                       cudaStream_t s) {
  double* X;
  int* piv;
  int64_t* rank;
  void* rest;
  size_t rest_bytes;
  int st = gj_pivchol(G, ldg, g, ws, ws_bytes, &X, &piv, &rank, &rest, &rest_bytes, s);
  if (st) return st;
  return gj_gram_eigh(X, g, piv, rank, g, r, sigma, T, ldt, info, rest, rest_bytes, s);
}

int gj_gram_eigh(const double* X, int64_t ldx, const int* piv, const int64_t* rank, int64_t g,
                 int64_t r, double* sigma, double* T, int64_t ldt, int64_t* info, void* ws,
                 size_t ws_bytes, cudaStream_t s) {
  const int P = gj::choose_P((int)g, (int)g, 0);
  POD_REQUIRE(P > 0, "gram eigh: g = %lld exceeds the grid Jacobi solver", (long long)g);
  const gj::Layout L((int)g, (int)g, 0, P);
  POD_REQUIRE(ws_bytes >= L.ws_bytes() + 256, "gram eigh: workspace too small (%zu < %zu)",
              ws_bytes, L.ws_bytes() + 256);
  double* w = gj_align(ws);
  gj::gram_prologue<<<2 * P, 256, 0, s>>>(w, P, X, ldx, rank, (int)g);
  POD_CHECK_LAUNCH("grid jacobi gram prologue");
  int st = gj::launch_sweep(L, w, 2.220446049250313e-16 * (double)std::max<int64_t>(g, 16), s);
  if (st) return st;
  const size_t eb = (size_t)g * sizeof(double);
  st = gj::launch_epilogue_smem((const void*)gj::gram_epilogue, eb);
  if (st) return st;
  gj::gram_epilogue<<<2 * P, 256, eb, s>>>(w, P, (int)g, (int)r, piv, sigma, T, ldt, info,
                                           rank ? 0 : 1);
  POD_CHECK_LAUNCH("grid jacobi gram epilogue");
  return POD_OK;
}

int gj_svd(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
           double* sigma, double* V, int64_t ldv, int64_t* info, void* ws, size_t ws_bytes,
           cudaStream_t s) {
  const int nj = V ? (int)nc : 0;
  const int P = gj::choose_P((int)nc, (int)nr, nj);
  POD_REQUIRE(P > 0, "svd small: %lld x %lld exceeds the grid Jacobi solver", (long long)nr,
              (long long)nc);
  const gj::Layout L((int)nc, (int)nr, nj, P);
  POD_REQUIRE(ws_bytes >= L.ws_bytes() + 256, "svd small: workspace too small (%zu < %zu)",
              ws_bytes, L.ws_bytes() + 256);
  double* w = gj_align(ws);
  gj::svd_prologue<<<2 * P, 256, 0, s>>>(w, P, A, lda, (int)nr, (int)nc, V ? 1 : 0);
  POD_CHECK_LAUNCH("grid jacobi svd prologue");
  int st = gj::launch_sweep(L, w, 2.220446049250313e-16 * (double)std::max<int64_t>(nr, 16), s);
  if (st) return st;
  const size_t eb = (size_t)nc * sizeof(double);
  st = gj::launch_epilogue_smem((const void*)gj::svd_epilogue, eb);
  if (st) return st;
  gj::svd_epilogue<<<2 * P, 256, eb, s>>>(w, P, (int)nr, (int)nc, U, ldu, sigma, V, ldv, info);
  POD_CHECK_LAUNCH("grid jacobi svd epilogue");
  return POD_OK;
}

int gj_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                  int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                  int64_t ldt, int64_t tcols, double* sig_new, int64_t* info, void* ws,
                  size_t ws_bytes, cudaStream_t s) {
  const int n = (int)(l1 + l2);
  // E^T with accumulated J (fewer sweeps) when it fits, else E
  int trans = 1;
  int P = gj::choose_P(n, n, n);
  if (!P) {
    trans = 0;
    P = gj::choose_P(n, n, 0);
  }
  POD_REQUIRE(P > 0, "merge core: l1 + l2 = %d exceeds the grid Jacobi solver", n);
  const gj::Layout L(n, n, trans ? n : 0, P);
  POD_REQUIRE(ws_bytes >= L.ws_bytes() + 256, "merge core: workspace too small (%zu < %zu)",
              ws_bytes, L.ws_bytes() + 256);
  double* w = gj_align(ws);
  gj::merge_prologue<<<2 * P, 256, 0, s>>>(w, P, sig1, (int)l1, M, ldm, R, ldr, sig2, (int)l2,
                                           trans);
  POD_CHECK_LAUNCH("grid jacobi merge prologue");
  int st = gj::launch_sweep(L, w, 2.220446049250313e-16 * (double)std::max(n, 16), s);
  if (st) return st;
  const size_t eb = (size_t)n * sizeof(double);
  st = gj::launch_epilogue_smem((const void*)gj::merge_epilogue, eb);
  if (st) return st;
  gj::merge_epilogue<<<2 * P, 256, eb, s>>>(w, P, (int)l1, (int)l2, (int)r, (int)rcap, T, ldt,
                                            (int)tcols, sig_new, info, trans);
  POD_CHECK_LAUNCH("grid jacobi merge epilogue");
  return POD_OK;
}

}  // namespace pod
