// Device building blocks of the column-block one-sided Jacobi solvers
// (block_jacobi.cu: cluster-resident; grid_jacobi.cu: grid-wide, L2-resident
// blocks): block geometry, slots, the rotation formulas and the intra/inter
// block sub-rounds.  Shared by both translation units.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace pod {
namespace bj {
namespace cg = cooperative_groups;

constexpr int MAX_CL = 8;

#ifdef POD_BJ_TIMING
__device__ unsigned long long g_bj_phase[16];
#define BJ_TI(i)                                                             \
  do {                                                                       \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                               \
      unsigned long long _t = clock64();                                     \
      if (i) atomicAdd(&g_bj_phase[i], _t - _bi_last);                      \
      _bi_last = _t;                                                         \
    }                                                                        \
  } while (0)
#define BJ_T(i)                                                              \
  do {                                                                       \
    if (threadIdx.x == 0 && cl.block_rank() == 0) {                          \
      unsigned long long _t = clock64();                                     \
      if (i) atomicAdd(&g_bj_phase[i], _t - _bj_last);                      \
      _bj_last = _t;                                                         \
    }                                                                        \
  } while (0)
#else
#define BJ_T(i) \
  do {          \
  } while (0)
#define BJ_TI(i) \
  do {           \
  } while (0)
#endif
constexpr size_t SMEM_CAP = 224 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
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
// bulk DSMEM copy of `bytes` (multiple of 16) from this CTA's shared memory
// to CTA-mapped address dst, completing on the destination's mbarrier
__device__ __forceinline__ void bulk_to_cluster(uint32_t dst, const void* src, uint32_t bytes,
                                                uint32_t dst_mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];\n" ::"r"(dst), "r"(smem_u32(src)), "r"(bytes), "r"(dst_mbar)
      : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// fp64 1/sqrt(x) for positive normal x (as cluster_jacobi.cu)
__device__ __forceinline__ double rsqrt_nr2(double x) {
  int e;
  double m = frexp(x, &e);
  if (e & 1) {
    m *= 2.0;
    e -= 1;
  }
  double y = (double)rsqrtf((float)m);
  y = y * fma(-0.5 * m, y * y, 1.5);
  y = y * fma(-0.5 * m, y * y, 1.5);
  return ldexp(y, -e / 2);
}

// 1/sqrt(x): fp32 seed + two Newton steps directly when x is well inside the
// fp32 range (the common case), else with exact power-of-two scaling
__device__ __forceinline__ double rsqrt_d(double x) {
  if (x > 1e-30 && x < 1e30) {
    double y = (double)rsqrtf((float)x);
    y = y * fma(-0.5 * x, y * y, 1.5);
    y = y * fma(-0.5 * x, y * y, 1.5);
    return y;
  }
  return rsqrt_nr2(x);
}

// One third-order step y (1 + e / 2 + 3 e^2 / 8), e = 1 - x y^2, from an
// fp32-accurate seed of 1 / sqrt(x): error ~ e^3 ~ 2^-63, the accuracy of two
// Newton steps at a dependent depth of four operations instead of six
__device__ __forceinline__ double rsqrt_refine3(double y, double x) {
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// Jacobi rotation (c, s) annihilating gamma between columns with squared
// norms al, be (|theta| <= pi/4; formulas of cluster_jacobi.cu)
__device__ __forceinline__ void rot_params(double g, double al, double be, double& c_,
                                           double& s_) {
  const double d = be - al;
  const double h2 = fma(d, d, 4.0 * g * g);
  double rh, ic;
  if (h2 > 1e-30 && h2 < 1e30) {
    // both fp32 seeds first (short MUFU chain), then the fp64 Newton steps;
    // ic's seed comes from the fp32 x, which Newton corrects to the fp64 x
    const float rhf = rsqrtf((float)h2);
    const float xf = 0.5f * fmaf(fabsf((float)d), rhf, 1.0f);
    const float icf = rsqrtf(xf);
    rh = rsqrt_refine3((double)rhf, h2);
    ic = (double)icf;
  } else {
    rh = rsqrt_nr2(h2);
    ic = -1.0;
  }
  const double x = 0.5 * fma(fabs(d), rh, 1.0);  // in [0.5, 1]
  if (ic < 0.0) ic = (double)rsqrtf((float)x);
  ic = rsqrt_refine3(ic, x);
  c_ = x * ic;
  s_ = copysign(fabs(g) * rh * ic, d * g);
}

// A slot holds one column block: W (bs x ld), J (bs x ldj, optional), the
// block's current squared norms and its global column ids (as doubles), all
// contiguous so one bulk copy moves it.
struct Geo {
  int n, nrows, njrows, bs, ld, ldj, bse;
  int slot;  // doubles per slot (even)
  __host__ __device__ Geo(int n_, int nrows_, int njrows_, int cl) {
    n = n_;
    nrows = nrows_;
    njrows = njrows_;
    bs = (n + 2 * cl - 1) / (2 * cl);
    ld = (nrows + 1) & ~1;
    ldj = (njrows + 1) & ~1;
    bse = (bs + 1) & ~1;
    slot = bs * ld + bs * ldj + 2 * bse;
  }
  // up to 4 mbarriers + flags [2][CL] (as doubles) + gathered norms [2 cl bs]
  // + nset block sets of 2 slots
  __host__ __device__ size_t smem_bytes(int cl, int nset = 2) const {
    return (size_t)(4 + 2 * cl + 2 * cl * bs + 2 * (size_t)nset * slot) * sizeof(double);
  }
};

struct Slot {
  double* w;
  double* j;
  double* nrm;
  double* id;
};
__device__ __forceinline__ Slot slot_at(double* slots, const Geo& g, int set, int t) {
  Slot s;
  double* b = slots + (size_t)(set * 2 + t) * g.slot;
  s.w = b;
  s.j = b + (size_t)g.bs * g.ld;
  s.nrm = s.j + (size_t)g.bs * g.ldj;
  s.id = s.nrm + g.bse;
  return s;
}

// Rotate column pairs (pa[k], pb[k]) k < P of the given slots (columns are
// pointers into smem) -- one thread group of tpp lanes per pair.
struct PairRef {
  double* x;
  double* y;
  double* jx;
  double* jy;
  double* nx;
  double* ny;
};

// Flags returned by the rotation steps: ROT_DONE = the pair was rotated,
// ROT_BIG = its cosine exceeded COS_BIG (1e-8).  A sweep in which no pair
// exceeded COS_BIG ends the iteration: cyclic Jacobi converges
// quadratically, so that sweep (which still rotates every pair above the
// visit threshold tol) leaves couplings of O(1e-16).  1e-6 (tried in r02:
// ~0.6 sweeps fewer per solve) is NOT safe: for clustered singular values
// (gaps below the cosine) the last sweep is not yet quadratic and sigma
// came out 1.2e-7 off (test_thin_qr_and_orthonormalize_match_reference).
constexpr int ROT_DONE = 1, ROT_BIG = 2;
#ifndef POD_COS_BIG2
#define POD_COS_BIG2 1e-16
#endif
constexpr double COS_BIG2 = POD_COS_BIG2;

template <int TPP, int RPL>
__device__ __forceinline__ int rotate_pair(const PairRef& pr, bool live, int gl, int nrows,
                                            int njrows, double tol2) {
  constexpr int tpp = TPP;
  double g = 0.0;
  double xa[RPL > 0 ? RPL : 1], xb[RPL > 0 ? RPL : 1];
  if (RPL > 0) {
#pragma unroll
    for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
      const int i = gl + k * tpp;
      const bool ok = live && i < nrows;
      xa[k] = ok ? pr.x[i] : 0.0;
      xb[k] = ok ? pr.y[i] : 0.0;
      g = fma(xa[k], xb[k], g);
    }
  } else if (live) {
    for (int i = gl; i < nrows; i += tpp) g = fma(pr.x[i], pr.y[i], g);
  }
  // norms are read before the (synchronising) shuffles; lane 0 rewrites them
  // only after its group has passed the shuffles
  const double al = live ? *pr.nx : 0.0, be = live ? *pr.ny : 0.0;
#pragma unroll
  for (int o = tpp / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o, tpp);
  if (!live) return 0;
  const double gg = g * g, ab = al * be;
  const int big = (gg > COS_BIG2 * ab && al > 0.0 && be > 0.0) ? ROT_BIG : 0;
  if (!(gg > tol2 * ab && al > 0.0 && be > 0.0)) return big;
  double c_, s_;
  rot_params(g, al, be, c_, s_);
  if (RPL > 0) {
#pragma unroll
    for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
      const int i = gl + k * tpp;
      if (i < nrows) {
        pr.x[i] = fma(c_, xa[k], -s_ * xb[k]);
        pr.y[i] = fma(s_, xa[k], c_ * xb[k]);
      }
    }
  } else {
    for (int i = gl; i < nrows; i += tpp) {
      const double x0 = pr.x[i], y0 = pr.y[i];
      pr.x[i] = fma(c_, x0, -s_ * y0);
      pr.y[i] = fma(s_, x0, c_ * y0);
    }
  }
  if (pr.jx) {
    for (int i = gl; i < njrows; i += tpp) {
      const double x0 = pr.jx[i], y0 = pr.jy[i];
      pr.jx[i] = fma(c_, x0, -s_ * y0);
      pr.jy[i] = fma(s_, x0, c_ * y0);
    }
  }
  if (gl == 0) {
    const double c2 = c_ * c_, s2 = s_ * s_, csg = 2.0 * c_ * s_ * g;
    *pr.nx = fmax(fma(c2, al, fma(s2, be, -csg)), 0.0);
    *pr.ny = fma(s2, al, fma(c2, be, csg));
  }
  return ROT_DONE | big;
}

__device__ __forceinline__ int pow2_floor(int v) {
  int p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}

// One sub-round: P disjoint pairs in parallel; pairs produced by `pick(k,
// &x_slot, &x_col, &y_slot, &y_col)`; returns whether this thread's pair rotated.
template <int TPP, int RPL, typename Pick>
__device__ int sub_round(const Slot& c0, const Slot& c1, const Geo& g, int P, double tol2,
                          Pick pick) {
  constexpr int tpp = TPP;
  const int grp = threadIdx.x / tpp, gl = threadIdx.x % tpp;
  const int ngrp = blockDim.x / tpp;
  int rot = 0;
  // groups beyond P still take part in the shuffles (full-warp masks)
  for (int k0 = 0; k0 < P; k0 += ngrp) {
    const int k = k0 + grp;
    int xs = 0, xc = 0, ys = 0, yc = 0;
    bool live = false;
    if (k < P) live = pick(k, xs, xc, ys, yc);
    const Slot& sx = xs ? c1 : c0;
    const Slot& sy = ys ? c1 : c0;
    PairRef pr;
    pr.x = sx.w + (size_t)xc * g.ld;
    pr.y = sy.w + (size_t)yc * g.ld;
    pr.jx = g.ldj ? sx.j + (size_t)xc * g.ldj : nullptr;
    pr.jy = g.ldj ? sy.j + (size_t)yc * g.ldj : nullptr;
    pr.nx = sx.nrm + xc;
    pr.ny = sy.nrm + yc;
    rot |= rotate_pair<TPP, RPL>(pr, live, gl, g.nrows, g.njrows, tol2);
  }
  __syncthreads();
  return rot;
}

// One tournament step's inter-block pairs: group k keeps top column k (rows
// in registers when RPL > 0, norm in a register) and meets bottom columns
// k, k+1, ... (mod bs) in bs sub-rounds.
template <int TPP, int RPL>
__device__ int inter_step(const Slot& c0, const Slot& c1, const Geo& g, double tol2) {
  const int bs = g.bs;
  constexpr int tpp = TPP;
  const int grp = threadIdx.x / tpp, gl = threadIdx.x % tpp;
  const bool has = grp < bs;
  uint32_t m1 = 0;
  for (int c = 0; c < bs; ++c) m1 |= ((int)c1.id[c] < g.n ? 1u : 0u) << c;
  const int xc = has ? grp : 0;
  const bool xlive = has && (int)c0.id[xc] < g.n;
  double* xw = c0.w + (size_t)xc * g.ld;
  double* xj = g.ldj ? c0.j + (size_t)xc * g.ldj : nullptr;
  double xa[RPL > 0 ? RPL : 1];
  // the accumulated rotation's x column is register-cached too when its
  // rows fit the same lanes (njrows <= nrows) -- small RPL only, so the
  // wide-row instantiations keep their register budget
  constexpr int JR = (RPL > 0 && RPL <= 8) ? RPL : 1;
  const bool jreg = JR > 1 && xj && g.njrows <= g.nrows;
  double xja[JR];
  if (RPL > 0) {
#pragma unroll
    for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
      const int i = gl + k * tpp;
      xa[k] = (xlive && i < g.nrows) ? xw[i] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < JR; ++k) {
      const int i = gl + k * tpp;
      xja[k] = (jreg && xlive && i < g.njrows) ? xj[i] : 0.0;
    }
  }
  double al = xlive ? c0.nrm[xc] : 0.0;
  int rot = 0;
#ifdef POD_BJ_TIMING
  unsigned long long _bi_last = clock64();
#endif
  for (int t = 0; t < bs; ++t) {
    BJ_TI(0);
    int yc = xc + t;
    if (yc >= bs) yc -= bs;
    const bool live = xlive && ((m1 >> yc) & 1u);
    double* yw = c1.w + (size_t)yc * g.ld;
    double gam = 0.0;
    double yb[RPL > 0 ? RPL : 1];
    if (RPL > 0) {
      double g2 = 0.0;  // two independent FMA chains
#pragma unroll
      for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
        const int i = gl + k * tpp;
        yb[k] = (live && i < g.nrows) ? yw[i] : 0.0;
        if (k & 1) g2 = fma(xa[k], yb[k], g2);
        else gam = fma(xa[k], yb[k], gam);
      }
      gam += g2;
    } else if (live) {
      for (int i = gl; i < g.nrows; i += tpp) gam = fma(xw[i], yw[i], gam);
    }
    const double be = live ? c1.nrm[yc] : 0.0;  // read before the shuffles
    BJ_TI(8);
#pragma unroll
    for (int o = tpp / 2; o > 0; o >>= 1) gam += __shfl_xor_sync(0xffffffffu, gam, o, tpp);
    BJ_TI(9);
    if (live && gam * gam > COS_BIG2 * al * be && al > 0.0 && be > 0.0) rot |= ROT_BIG;
    if (live && gam * gam > tol2 * al * be && al > 0.0 && be > 0.0) {
      double c_, s_;
      rot_params(gam, al, be, c_, s_);
      if (RPL > 0) {
#pragma unroll
        for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
          const int i = gl + k * tpp;
          const double x0 = xa[k], y0 = yb[k];
          xa[k] = fma(c_, x0, -s_ * y0);
          if (i < g.nrows) yw[i] = fma(s_, x0, c_ * y0);
        }
      } else {
        for (int i = gl; i < g.nrows; i += tpp) {
          const double x0 = xw[i], y0 = yw[i];
          xw[i] = fma(c_, x0, -s_ * y0);
          yw[i] = fma(s_, x0, c_ * y0);
        }
      }
      if (jreg) {
        double* yj = c1.j + (size_t)yc * g.ldj;
        double yjb[JR];
#pragma unroll
        for (int k = 0; k < JR; ++k) {
          const int i = gl + k * tpp;
          yjb[k] = i < g.njrows ? yj[i] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < JR; ++k) {
          const int i = gl + k * tpp;
          const double x0 = xja[k], y0 = yjb[k];
          xja[k] = fma(c_, x0, -s_ * y0);
          if (i < g.njrows) yj[i] = fma(s_, x0, c_ * y0);
        }
      } else if (xj) {
        double* yj = c1.j + (size_t)yc * g.ldj;
        for (int i = gl; i < g.njrows; i += tpp) {
          const double x0 = xj[i], y0 = yj[i];
          xj[i] = fma(c_, x0, -s_ * y0);
          yj[i] = fma(s_, x0, c_ * y0);
        }
      }
      const double c2 = c_ * c_, s2 = s_ * s_, csg = 2.0 * c_ * s_ * gam;
      const double nal = fmax(fma(c2, al, fma(s2, be, -csg)), 0.0);
      if (gl == 0) c1.nrm[yc] = fma(s2, al, fma(c2, be, csg));
      al = nal;
      rot |= ROT_DONE;
    }
    BJ_TI(10);
    __syncthreads();
    BJ_TI(11);
  }
  if (xlive) {
    if (RPL > 0) {
#pragma unroll
      for (int k = 0; k < (RPL > 0 ? RPL : 1); ++k) {
        const int i = gl + k * tpp;
        if (i < g.nrows) xw[i] = xa[k];
      }
#pragma unroll
      for (int k = 0; k < JR; ++k) {
        const int i = gl + k * tpp;
        if (jreg && i < g.njrows) xj[i] = xja[k];
      }
    }
    if (gl == 0) c0.nrm[xc] = al;
  }
  __syncthreads();
  return rot;
}

// column ids: id < n real, otherwise padding (zero column, never rotated)
__device__ __forceinline__ bool col_live(const Slot& s, int c, int n) {
  return (int)s.id[c] < n;
}

}  // namespace bj
}  // namespace pod
