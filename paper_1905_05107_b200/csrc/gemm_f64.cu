// FP64 tall-skinny GEMMs on the tensor pipe (DMMA.8x8x4) for sm_100a.
//
// Every m-length operand of the ISMA round is a column-major matrix whose
// row count m is huge (rows of the data matrix) and whose column count is
// small (sampled columns g, factor modes r).  Two shapes cover the round:
//
//   TN  C (p x q) = alpha X^T Y          K = m: Gram D^T D (baselines.py:43),
//                                         U1^T U2 (merge.py:65), CholQR Grams,
//                                         leak U1^T Q (merge.py:72), finalize
//                                         A^T U (isma.py:296)
//   NN  Y (m x q) = alpha X T + beta Z    lift D V / sigma (baselines.py:62-63),
//                                         U2 - U1 M (merge.py:69), Q = W R^-1,
//                                         [U1 Q] U_E (merge.py:86-88),
//                                         finalize rotations (isma.py:298-299)
//
// X (and Y) may be addressed through a column index list, so the sampled
// block D = A[:, idx] is never materialised (isma.py:163 gather fused into
// the operand loads).  TN splits K=m across CTAs and reduces the partial
// tiles in a fixed order (deterministic, no atomics).
#include "common.cuh"

namespace pod {

// NN epilogue helpers: a warp's 4 x FN fragments of 8 x 8 outputs at rows
// row0 + f*8 + lane/4, columns col0 + g*8 + 2*(lane%4) + e.  The beta * Z
// operand is loaded into registers first (all loads in flight together, or
// prefetched under the last k-chunk's DMMAs), then combined and stored.
template <int FN>
__device__ __forceinline__ void nn_load_z(double (&zv)[4][FN][2], int64_t row0, int col0,
                                          int lane, int64_t m, int q, const double* Z,
                                          int64_t ldz) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t i = row0 + f * 8 + (lane >> 2);
#pragma unroll
    for (int g = 0; g < FN; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + g * 8 + 2 * (lane & 3) + e;
        zv[f][g][e] = (i < m && j < q) ? Z[i + (int64_t)j * ldz] : 0.0;
      }
  }
}

template <int FN>
__device__ __forceinline__ void nn_store(const double (&acc)[4][FN][2],
                                         const double (&zv)[4][FN][2], int64_t row0, int col0,
                                         int lane, int64_t m, int q, double alpha, double beta,
                                         double* Y, int64_t ldy) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t i = row0 + f * 8 + (lane >> 2);
#pragma unroll
    for (int g = 0; g < FN; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + g * 8 + 2 * (lane & 3) + e;
        if (i < m && j < q) {
          double v = alpha * acc[f][g][e];
          if (beta != 0.0) v += beta * zv[f][g][e];
          Y[i + (int64_t)j * ldy] = v;
        }
      }
  }
}

// Same, without a full register copy of Z: each of the 4 row fragments loads
// its FN x 2 Z values together, then stores (4 load latencies per epilogue).
template <int FN>
__device__ __forceinline__ void nn_epilogue(const double (&acc)[4][FN][2], int64_t row0, int col0,
                                            int lane, int64_t m, int q, double alpha, double beta,
                                            const double* Z, int64_t ldz, double* Y,
                                            int64_t ldy) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t i = row0 + f * 8 + (lane >> 2);
    double zr[FN][2];
    if (beta != 0.0) {
#pragma unroll
      for (int g = 0; g < FN; ++g)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = col0 + g * 8 + 2 * (lane & 3) + e;
          zr[g][e] = (i < m && j < q) ? Z[i + (int64_t)j * ldz] : 0.0;
        }
    }
#pragma unroll
    for (int g = 0; g < FN; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + g * 8 + 2 * (lane & 3) + e;
        if (i < m && j < q) {
          double v = alpha * acc[f][g][e];
          if (beta != 0.0) v += beta * zr[g][e];
          Y[i + (int64_t)j * ldy] = v;
        }
      }
  }
}

// nn_epilogue that also accumulates, for local output columns j < kdl, the
// products Y[i, j] X[i, j] of the stored value with X's same-index column
// (read back from L2: the convergence cosines of isma.py:195-198 when
// X = [U_old Q] and Y = U_new, formed inside the rotation GEMM)
template <int FN>
__device__ __forceinline__ void nn_epilogue_dots(const double (&acc)[4][FN][2], int64_t row0,
                                                 int col0, int lane, int64_t m, int q,
                                                 double alpha, double* Y, int64_t ldy,
                                                 const double* __restrict__ DX, int64_t dldx,
                                                 int kdl, double (&dacc)[FN][2]) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t i = row0 + f * 8 + (lane >> 2);
    double xr[FN][2];
#pragma unroll
    for (int g = 0; g < FN; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + g * 8 + 2 * (lane & 3) + e;
        xr[g][e] = (i < m && j < kdl) ? __ldg(DX + i + (int64_t)j * dldx) : 0.0;
      }
#pragma unroll
    for (int g = 0; g < FN; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + g * 8 + 2 * (lane & 3) + e;
        if (i < m && j < q) {
          const double v = alpha * acc[f][g][e];
          Y[i + (int64_t)j * ldy] = v;
          dacc[g][e] = fma(v, xr[g][e], dacc[g][e]);
        }
      }
  }
}

// Grid cap for the persistent / split-K GEMMs launched while it is set
// (pod_set_grid_cap): lets a concurrent, off-critical-path stream (the
// pipelined update of the next round) leave SMs to the critical path.  0 = all.
static int g_grid_cap = 0;
static inline int64_t capped(int64_t ctas) {
  return g_grid_cap > 0 ? std::max<int64_t>(1, std::min<int64_t>(ctas, g_grid_cap)) : ctas;
}

// mbarrier helpers of the warp-specialized GEMMs (producer warp -> consumers)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* mb, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(mb)), "r"(count));
}
__device__ __forceinline__ void mb_wait(uint64_t* mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(mb)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(mb)) : "memory");
}
__device__ __forceinline__ void mb_cp_async_arrive(uint64_t* mb) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(mb))
               : "memory");
}

// ---------------------------------------------------------------- TN ------
namespace tn {
// balanced symmetric launch (see tn80): nd diagonal tiles x sd splits, then
// the off-diagonal tiles x so splits, with their own rows per split
struct Bal {
  int on, nd, sd, so;
  int64_t rps_d, rps_o;
};
constexpr int BP = 64, BQ = 64, BK = 32, LDS = BK + 4;  // LDS % 16 == 4: conflict-free frags
constexpr int THREADS = 256;
constexpr int STAGES = 3;
constexpr int TILE_DBL = BP * LDS;  // elements per operand tile
// operand tiles are stored in the operands' own type (fp32 storage is
// converted exactly to fp64 at the fragment loads)
template <typename TX, typename TY>
constexpr size_t smem_bytes() {
  return size_t(STAGES) * TILE_DBL * (sizeof(TX) + sizeof(TY));
}
constexpr size_t SMEM = smem_bytes<double, double>();

template <typename T>
__device__ __forceinline__ const T* colptr(const T* base, int64_t ld, const int32_t* cols, int c) {
  return base + (cols ? (int64_t)cols[c] : (int64_t)c) * ld;
}

template <typename TX, typename TY, bool BAL = false>
__global__ void __launch_bounds__(THREADS) partial_kernel(
    int64_t m, int p, int q, const TX* __restrict__ X, int64_t ldx,
    const int32_t* __restrict__ xcols, const TY* __restrict__ Y, int64_t ldy,
    const int32_t* __restrict__ ycols, int64_t rows_per_split, double* __restrict__ ws,
    const int32_t* __restrict__ gate, int sym, Bal bal = Bal{0, 0, 0, 0, 0, 0}) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tiles_p = (p + BP - 1) / BP;
  int tp, tq, split;
  int64_t rps = rows_per_split;
  if (BAL) {
    const int x = blockIdx.x;
    if (x < bal.nd * bal.sd) {
      tp = tq = x / bal.sd;
      split = x % bal.sd;
      rps = bal.rps_d;
    } else {
      int t = (x - bal.nd * bal.sd) / bal.so;
      split = (x - bal.nd * bal.sd) % bal.so;
      tq = 1;
      while (t >= tq) { t -= tq; ++tq; }
      tp = t;
      rps = bal.rps_o;
    }
  } else if (sym) {  // symmetric product (X == Y): upper-triangular tiles tp <= tq only
    int t = blockIdx.x;
    tq = 0;
    while (t > tq) { t -= tq + 1; ++tq; }
    tp = t;
    split = blockIdx.y;
  } else {
    tp = blockIdx.x % tiles_p;
    tq = blockIdx.x / tiles_p;
    split = blockIdx.y;
  }
  const bool diag = BAL && tp == tq;
  const int64_t r0 = (int64_t)split * rps;
  const int64_t r1 = min(m, r0 + rps);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // fp64 operands move row PAIRS with 16-byte copies: thread -> columns
  // tid / 16 + 16 i (i < 4), rows 2 (tid % 16) and +1 of each stage; other
  // operand types copy one element (column warp + 8 i, row lane)
  constexpr bool PAIRS = sizeof(TX) == 8 && sizeof(TY) == 8;
  constexpr int NPC = PAIRS ? 4 : 8;
  const TX* xp[NPC];
  const TY* yp[NPC];
  bool xv[NPC], yv[NPC], xal[NPC], yal[NPC];
#pragma unroll
  for (int i = 0; i < NPC; ++i) {
    const int cl = PAIRS ? (int)(threadIdx.x >> 4) + 16 * i : warp + 8 * i;
    int cx = tp * BP + cl;
    int cy = tq * BQ + cl;
    xv[i] = cx < p && (!xcols || xcols[cx] >= 0);  // index -1: zero column (padding)
    yv[i] = cy < q && (!ycols || ycols[cy] >= 0);
    xp[i] = xv[i] ? colptr(X, ldx, xcols, cx) : X;
    yp[i] = yv[i] ? colptr(Y, ldy, ycols, cy) : Y;
    xal[i] = ((uintptr_t)xp[i] & 15) == 0;  // 16-byte copies need an aligned column
    yal[i] = ((uintptr_t)yp[i] & 15) == 0;
  }
  TX* const xs0 = reinterpret_cast<TX*>(smem_raw);
  TY* const ys0 = reinterpret_cast<TY*>(smem_raw + size_t(STAGES) * TILE_DBL * sizeof(TX));
  auto load_stage = [&](int st, int64_t rb) {
    TX* xs = xs0 + (size_t)st * TILE_DBL;
    TY* ys = ys0 + (size_t)st * TILE_DBL;
    if constexpr (PAIRS) {
      const int r2 = 2 * (threadIdx.x & 15);
      const int64_t row = rb + r2;  // even: splits and stages start at multiples of BK
      const bool v0 = row < r1, v1 = row + 1 < r1;
#pragma unroll
      for (int i = 0; i < NPC; ++i) {
        const int c = (int)(threadIdx.x >> 4) + 16 * i;
        TX* dx = xs + c * LDS + r2;
        TY* dy = ys + c * LDS + r2;
        if (xv[i] && v1 && xal[i]) {
          cp_async16(dx, xp[i] + row, true);
        } else {
          cp_async_elem(dx, xv[i] && v0 ? xp[i] + row : X, xv[i] && v0);
          cp_async_elem(dx + 1, xv[i] && v1 ? xp[i] + row + 1 : X, xv[i] && v1);
        }
        if (yv[i] && v1 && yal[i]) {
          cp_async16(dy, yp[i] + row, true);
        } else {
          cp_async_elem(dy, yv[i] && v0 ? yp[i] + row : Y, yv[i] && v0);
          cp_async_elem(dy + 1, yv[i] && v1 ? yp[i] + row + 1 : Y, yv[i] && v1);
        }
      }
    } else {
      const int64_t row = rb + lane;
      const bool rv = row < r1;
#pragma unroll
      for (int i = 0; i < NPC; ++i) {
        const int c = warp + 8 * i;
        cp_async_elem(xs + c * LDS + lane, xv[i] && rv ? xp[i] + row : X, xv[i] && rv);
        cp_async_elem(ys + c * LDS + lane, yv[i] && rv ? yp[i] + row : Y, yv[i] && rv);
      }
    }
  };

  const int wp = warp & 1, wq = warp >> 1;  // warp tile: 32 (p) x 16 (q)
  double acc[4][2][2];
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int g = 0; g < 2; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
  // diagonal tile (BAL): this warp's <= 5 of the 36 upper fragments, rows k
  // and 7 - k (9 fragments) dealt over warps 2k (5) and 2k + 1 (4)
  const int kq = warp >> 1;
  int fr[5], fc[5];
#pragma unroll
  for (int g = 0; g < 5; ++g) {
    if ((warp & 1) == 0) {
      fr[g] = kq;
      fc[g] = kq + g;
    } else if (g < 3 - kq) {
      fr[g] = kq;
      fc[g] = kq + 5 + g;
    } else if (g - (3 - kq) <= kq) {
      fr[g] = 7 - kq;
      fc[g] = 7 - kq + (g - (3 - kq));
    } else {
      fr[g] = 7 - kq;
      fc[g] = -1;
    }
  }

  const int64_t nkb = (r1 > r0) ? (r1 - r0 + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkb) load_stage(s, r0 + (int64_t)s * BK);
    cp_async_commit();
  }
  for (int64_t kb = 0; kb < nkb; ++kb) {
    const int64_t nxt = kb + STAGES - 1;
    if (nxt < nkb) load_stage((int)(nxt % STAGES), r0 + nxt * BK);
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    __syncthreads();
    const TX* xs = xs0 + (size_t)(kb % STAGES) * TILE_DBL;
    const TY* ys = ys0 + (size_t)(kb % STAGES) * TILE_DBL;
    if (BAL && diag) {  // accumulators acc[g / 2][g % 2], g < 5
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        const double a0 = (double)xs[(fr[0] * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
        const double a1 = (double)xs[(fr[4] * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
#pragma unroll
        for (int g = 0; g < 5; ++g) {
          if (fc[g] < 0) continue;
          const double bb = (double)ys[(fc[g] * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
          dmma8x8x4(acc[g / 2][g % 2][0], acc[g / 2][g % 2][1], fr[g] == fr[0] ? a0 : a1, bb);
        }
      }
    } else {
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4], b[2];
#pragma unroll
      for (int f = 0; f < 4; ++f)
        a[f] = (double)xs[(wp * 32 + f * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
#pragma unroll
      for (int g = 0; g < 2; ++g)
        b[g] = (double)ys[(wq * 16 + g * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < 2; ++g) dmma8x8x4(acc[f][g][0], acc[f][g][1], a[f], b[g]);
    }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  double* out = ws + (size_t)split * p * q;
  if (BAL && diag) {
#pragma unroll
    for (int g = 0; g < 5; ++g) {
      if (fc[g] < 0) continue;
      const int i = tp * BP + fr[g] * 8 + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tq * BQ + fc[g] * 8 + 2 * (lane & 3) + e;
        if (i < p && j < q) out[(size_t)j * p + i] = acc[g / 2][g % 2][e];
      }
    }
    return;
  }
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int i = tp * BP + wp * 32 + f * 8 + (lane >> 2);
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tq * BQ + wq * 16 + g * 8 + 2 * (lane & 3) + e;
        if (i < p && j < q) out[(size_t)j * p + i] = acc[f][g][e];
      }
  }
}

// C[i, j] = alpha * sum_k ws[k][i, j]: one warp per output element, lanes
// take splits k = lane, lane + 32, ... and a fixed shuffle tree combines them
// (deterministic; no atomics).
// nsplit_diag > 0 (balanced symmetric plan): elements of the diagonal
// tiles (i / tile == j / tile) have only nsplit_diag partials.
__global__ void __launch_bounds__(256) reduce_kernel(int nsplit, int p, int q, double alpha,
                                                     const double* __restrict__ ws,
                                                     double* __restrict__ C, int64_t ldc,
                                                     const int32_t* __restrict__ gate, int sym,
                                                     int nsplit_diag = 0, int tile = 1) {
  if (gate && *gate == 0) return;
  const int64_t total = (int64_t)p * q;
  const int lane = threadIdx.x & 31;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = wg; t < total; t += nw) {
    const int64_t j = t / p, i = t - j * p;
    // symmetric: the lower triangle mirrors the upper one (exactly symmetric C)
    const int64_t src = (sym && i > j) ? (j + i * p) : t;
    const int ns = (nsplit_diag > 0 && i / tile == j / tile) ? nsplit_diag : nsplit;
    double s = 0.0;
    for (int k = lane; k < ns; k += 32) s += ws[(size_t)k * total + src];
    s = warp_sum(s);
    if (lane == 0) C[i + j * ldc] = alpha * s;
  }
}

struct Plan {
  int tiles, splits;
  int64_t rows_per_split;
};

inline Plan plan(int64_t m, int64_t p, int64_t q, bool sym) {
  Plan pl;
  const int64_t tp = ceil_div(p, BP);
  pl.tiles = (int)(sym ? tp * (tp + 1) / 2 : tp * ceil_div(q, BQ));
  const int target = (int)capped(2 * 148);  // 2 CTAs/SM: ONE wave, never a partial second
  int64_t want = std::max<int64_t>(1, target / pl.tiles);
  int64_t max_by_rows = std::max<int64_t>(1, ceil_div(m, 4 * BK));  // >= 4 k-blocks per CTA
  int64_t splits = std::min<int64_t>(want, max_by_rows);
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, 65535));
  pl.rows_per_split = ceil_div(ceil_div(m, splits), BK) * BK;
  if (pl.rows_per_split == 0) pl.rows_per_split = BK;
  pl.splits = (int)std::max<int64_t>(1, ceil_div(m, pl.rows_per_split));
  return pl;
}
}  // namespace tn

// ----------------------------------------------------------- TN (80) -----
// 80 x 80 output tiles (10 x 10 fragments) for operand widths where 64-wide
// tiles pad badly (r = 150 -> 160 instead of 192, n = 2000 exactly).  10 warps
// (5 along p x 2 along q), warp tile 16 x 40 (2 x 5 fragments), BK = 16 so two
// CTAs fit an SM; gathered column offsets live in shared memory instead of
// per-thread pointer registers.
#ifndef POD_TN_WS_MINB
#define POD_TN_WS_MINB 2
#endif
namespace tn80 {
constexpr int T = 80, NW = 10, THREADS = NW * 32;
constexpr int NPROD = 2;  // producer warps of the warp-specialized variant
constexpr int BK = 16, LDS = BK + 4;  // % 16 == 4: conflict-free fragments
constexpr int STAGES = 4;
constexpr int TILE = T * LDS;
template <typename TX, typename TY>
constexpr size_t smem_bytes() {
  // + the warp-specialized variant's full / empty mbarriers
  return size_t(STAGES) * TILE * (sizeof(TX) + sizeof(TY)) + 2 * T * sizeof(int64_t) +
         2 * STAGES * sizeof(uint64_t);
}

// Work-balanced symmetric mode (Bal.on): a diagonal tile computes only its 55
// upper-triangular fragments, dealt two rows per pair of warps (rows k and
// 9 - k hold 11 fragments: 6 + 5), and the K split gives each off-diagonal
// tile more CTAs than a diagonal one (sd < so splits) so both finish
// together.  1-D grid: the nd x sd diagonal CTAs first, then the
// off-diagonal tiles (tq = 1, 2, ..., tp < tq) x so.
using Bal = tn::Bal;

template <typename TX, typename TY, bool BAL = false, bool WS = false>
__global__ void __launch_bounds__(WS ? THREADS + NPROD * 32 : THREADS, WS ? POD_TN_WS_MINB : 2) partial_kernel(
    int64_t m, int p, int q, const TX* __restrict__ X, int64_t ldx,
    const int32_t* __restrict__ xcols, const TY* __restrict__ Y, int64_t ldy,
    const int32_t* __restrict__ ycols, int64_t rows_per_split, double* __restrict__ ws,
    const int32_t* __restrict__ gate, int sym, Bal bal) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tiles_p = (p + T - 1) / T;
  int tp, tq, split;
  int64_t rps = rows_per_split;
  if (BAL) {
    const int x = blockIdx.x;
    if (x < bal.nd * bal.sd) {
      tp = tq = x / bal.sd;
      split = x % bal.sd;
      rps = bal.rps_d;
    } else {
      int t = (x - bal.nd * bal.sd) / bal.so;
      split = (x - bal.nd * bal.sd) % bal.so;
      tq = 1;
      while (t >= tq) { t -= tq; ++tq; }
      tp = t;
      rps = bal.rps_o;
    }
  } else if (sym) {
    int t = blockIdx.x;
    tq = 0;
    while (t > tq) { t -= tq + 1; ++tq; }
    tp = t;
    split = blockIdx.y;
  } else {
    tp = blockIdx.x % tiles_p;
    tq = blockIdx.x / tiles_p;
    split = blockIdx.y;
  }
  const bool diag = BAL && tp == tq;
  const int64_t r0 = (int64_t)split * rps;
  const int64_t r1 = min(m, r0 + rps);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TX* const xs0 = reinterpret_cast<TX*>(smem_raw);
  TY* const ys0 = reinterpret_cast<TY*>(smem_raw + size_t(STAGES) * TILE * sizeof(TX));
  int64_t* const xoff = reinterpret_cast<int64_t*>(smem_raw + size_t(STAGES) * TILE *
                                                                  (sizeof(TX) + sizeof(TY)));
  int64_t* const yoff = xoff + T;
  for (int c = threadIdx.x; c < 2 * T; c += THREADS) {
    const bool isx = c < T;
    const int cc = isx ? c : c - T;
    const int gc = (isx ? tp : tq) * T + cc;
    const int32_t* cols = isx ? xcols : ycols;
    int64_t off = -1;
    if (gc < (isx ? p : q)) {
      const int64_t col = cols ? (int64_t)cols[gc] : (int64_t)gc;
      if (col >= 0) off = col * (isx ? ldx : ldy);  // index -1: zero column
    }
    (isx ? xoff : yoff)[cc] = off;
  }
  uint64_t* const full = reinterpret_cast<uint64_t*>(yoff + T);
  uint64_t* const empty = full + STAGES;
  if (WS && threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mb_init(&full[s], NPROD * 32);
      mb_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // loader: warp w moves rows rb + lane of columns w, w + 10, ... (8 each)
  auto load_stage = [&](int st, int64_t rb) {
    TX* xs = xs0 + (size_t)st * TILE;
    TY* ys = ys0 + (size_t)st * TILE;
    const int64_t row = rb + (lane & 15);
    const bool rv = row < r1;
    const int half = lane >> 4;  // lanes 0-15 / 16-31: two columns per instruction
#pragma unroll
    for (int i = 0; i < T / NW / 2; ++i) {
      const int c = warp + NW * (2 * i + half);
      const int64_t ox = xoff[c], oy = yoff[c];
      cp_async_elem(xs + c * LDS + (lane & 15), ox >= 0 && rv ? X + ox + row : X, ox >= 0 && rv);
      cp_async_elem(ys + c * LDS + (lane & 15), oy >= 0 && rv ? Y + oy + row : Y, oy >= 0 && rv);
    }
  };
  const int wp = warp % 5, wq = warp / 5;  // warp tile: 16 (p) x 40 (q)
  double acc[2][5][2];
#pragma unroll
  for (int f = 0; f < 2; ++f)
#pragma unroll
    for (int g = 0; g < 5; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
  // diagonal tile: this warp's <= 6 upper fragments (row fr[g], column fc[g]);
  // rows k and 9 - k of warps 2k, 2k + 1
  const int kq = warp >> 1;
  int fr[6], fc[6];
#pragma unroll
  for (int g = 0; g < 6; ++g) {
    if ((warp & 1) == 0) {
      fr[g] = kq;
      fc[g] = kq + g <= 9 ? kq + g : -1;
    } else if (g < 4 - kq) {
      fr[g] = kq;
      fc[g] = kq + 6 + g;
    } else if (g - (4 - kq) <= kq) {
      fr[g] = 9 - kq;
      fc[g] = 9 - kq + (g - (4 - kq));
    } else {
      fr[g] = 9 - kq;
      fc[g] = -1;
    }
  }
  const int64_t nkb = (r1 > r0) ? (r1 - r0 + BK - 1) / BK : 0;
  if constexpr (WS) {
    if (warp >= NW) {
      // NPROD producer warps: thread t owns row pair t % 8 of columns
      // t / 8 + (NPT * i), i < 80 / NPT, of both tiles, their offsets held in
      // registers; 16-byte copies for fp64 on full aligned stages, each
      // thread's copies completing on the stage's full barrier
      constexpr int NPT = NPROD * 32 / (BK / 2);  // columns covered per sweep
      constexpr int CPT = T / NPT;                // columns per thread
      const int t = threadIdx.x - NW * 32;
      const int r2 = (t % (BK / 2)) * 2, c0 = t / (BK / 2);
      int64_t ox[CPT], oy[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        ox[i] = xoff[c0 + NPT * i];
        oy[i] = yoff[c0 + NPT * i];
      }
      const bool al = ((reinterpret_cast<uintptr_t>(X) % (2 * sizeof(TX))) == 0) && ldx % 2 == 0 &&
                      ((reinterpret_cast<uintptr_t>(Y) % (2 * sizeof(TY))) == 0) && ldy % 2 == 0;
      int st = 0;
      uint32_t ph = 0;
      for (int64_t kb = 0; kb < nkb; ++kb) {
        if (kb >= STAGES) mb_wait(&empty[st], ph ^ 1);
        const int64_t row = r0 + kb * BK + r2;
        TX* xs = xs0 + (size_t)st * TILE + c0 * LDS + r2;
        TY* ys = ys0 + (size_t)st * TILE + c0 * LDS + r2;
        if (al && row + 1 < r1) {
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            if constexpr (sizeof(TX) == 8)
              cp_async16(xs + NPT * i * LDS, ox[i] >= 0 ? X + ox[i] + row : X, ox[i] >= 0);
            else
              cp_async8(xs + NPT * i * LDS, ox[i] >= 0 ? X + ox[i] + row : X, ox[i] >= 0);
            if constexpr (sizeof(TY) == 8)
              cp_async16(ys + NPT * i * LDS, oy[i] >= 0 ? Y + oy[i] + row : Y, oy[i] >= 0);
            else
              cp_async8(ys + NPT * i * LDS, oy[i] >= 0 ? Y + oy[i] + row : Y, oy[i] >= 0);
          }
        } else {
          const bool v0 = row < r1, v1 = row + 1 < r1;
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            const bool x0 = ox[i] >= 0 && v0, x1 = ox[i] >= 0 && v1;
            const bool y0 = oy[i] >= 0 && v0, y1 = oy[i] >= 0 && v1;
            cp_async_elem(xs + NPT * i * LDS, x0 ? X + ox[i] + row : X, x0);
            cp_async_elem(xs + NPT * i * LDS + 1, x1 ? X + ox[i] + row + 1 : X, x1);
            cp_async_elem(ys + NPT * i * LDS, y0 ? Y + oy[i] + row : Y, y0);
            cp_async_elem(ys + NPT * i * LDS + 1, y1 ? Y + oy[i] + row + 1 : Y, y1);
          }
        }
        mb_cp_async_arrive(&full[st]);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
      cp_async_wait<0>();
      return;
    }
  } else {
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
      if (st < nkb) load_stage(st, r0 + (int64_t)st * BK);
      cp_async_commit();
    }
  }
  for (int64_t kb = 0; kb < nkb; ++kb) {
    if constexpr (WS) {
      mb_wait(&full[kb % STAGES], (uint32_t)((kb / STAGES) & 1));
    } else {
      const int64_t nxt = kb + STAGES - 1;
      if (nxt < nkb) load_stage((int)(nxt % STAGES), r0 + nxt * BK);
      cp_async_commit();
      cp_async_wait<STAGES - 1>();
      __syncthreads();
    }
    const TX* xs = xs0 + (size_t)(kb % STAGES) * TILE;
    const TY* ys = ys0 + (size_t)(kb % STAGES) * TILE;
    if (BAL && diag) {
      // the 6 accumulators reuse acc's registers: acc[g / 5][g % 5]
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        const double a0 = (double)xs[(fr[0] * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
        const double a1 = (double)xs[(fr[5] * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
#pragma unroll
        for (int g = 0; g < 6; ++g) {
          if (fc[g] < 0) continue;
          const double bb = (double)ys[(fc[g] * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
          dmma8x8x4(acc[g / 5][g % 5][0], acc[g / 5][g % 5][1], fr[g] == fr[0] ? a0 : a1, bb);
        }
      }
    } else {
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[2], b[5];
#pragma unroll
      for (int f = 0; f < 2; ++f)
        a[f] = (double)xs[(wp * 16 + f * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
#pragma unroll
      for (int g = 0; g < 5; ++g)
        b[g] = (double)ys[(wq * 40 + g * 8 + (lane >> 2)) * LDS + kk * 4 + (lane & 3)];
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int g = 0; g < 5; ++g) dmma8x8x4(acc[f][g][0], acc[f][g][1], a[f], b[g]);
    }
    }
    if constexpr (WS) {
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[kb % STAGES]);
    } else {
      __syncthreads();
    }
  }
  if constexpr (!WS) cp_async_wait<0>();
  double* out = ws + (size_t)split * p * q;
  if (BAL && diag) {
#pragma unroll
    for (int g = 0; g < 6; ++g) {
      if (fc[g] < 0) continue;
      const int i = tp * T + fr[g] * 8 + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tq * T + fc[g] * 8 + 2 * (lane & 3) + e;
        if (i < p && j < q) out[(size_t)j * p + i] = acc[g / 5][g % 5][e];
      }
    }
    return;
  }
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int i = tp * T + wp * 16 + f * 8 + (lane >> 2);
#pragma unroll
    for (int g = 0; g < 5; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tq * T + wq * 40 + g * 8 + 2 * (lane & 3) + e;
        if (i < p && j < q) out[(size_t)j * p + i] = acc[f][g][e];
      }
  }
}

inline tn::Plan plan(int64_t m, int64_t p, int64_t q, bool sym) {
  tn::Plan pl;
  const int64_t tp = ceil_div(p, T);
  pl.tiles = (int)(sym ? tp * (tp + 1) / 2 : tp * ceil_div(q, T));
  const int target = (int)capped(2 * 148);
  int64_t want = std::max<int64_t>(1, target / pl.tiles);
  int64_t max_by_rows = std::max<int64_t>(1, ceil_div(m, 4 * BK));
  int64_t splits = std::min<int64_t>(want, max_by_rows);
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, 65535));
  pl.rows_per_split = ceil_div(ceil_div(m, splits), BK) * BK;
  if (pl.rows_per_split == 0) pl.rows_per_split = BK;
  pl.splits = (int)std::max<int64_t>(1, ceil_div(m, pl.rows_per_split));
  return pl;
}
// Balanced symmetric plan (sym products with >= 2 tile rows): a diagonal
// tile's CTA is given DIAG_COST times an off-diagonal one's splits (55 of
// 100 fragments; 0.47 measured best at config 3 from a sweep 0.2-1.0:
// 2.850 s unbalanced -> 2.77 s), so both finish together in one wave.
inline double env_cost(const char* name, double dflt) {
  const char* e = getenv(name);
  const double v = e ? atof(e) : dflt;
  return (v > 0.05 && v <= 1.0) ? v : dflt;
}
inline double diag_cost() {  // POD_TN_DIAG_COST: A/B override
  static double v = -1.0;
  if (v < 0.0) v = env_cost("POD_TN_DIAG_COST", 0.47);
  return v;
}
inline Bal plan_bal_t(int64_t m, int64_t p, int T, int BK, double DIAG_COST) {
  Bal b = {0, 0, 0, 0, 0, 0};
  const int64_t tp = ceil_div(p, T);
  if (tp < 2) return b;
  const int64_t noff = tp * (tp - 1) / 2;
  const double budget = (double)capped(2 * 148);
  int64_t so = std::max<int64_t>(1, (int64_t)(budget / (noff + DIAG_COST * tp)));
  int64_t sd = std::max<int64_t>(1, (int64_t)(so * DIAG_COST));
  while (sd * tp + so * noff > (int64_t)budget && so > 1) {
    --so;
    sd = std::max<int64_t>(1, (int64_t)(so * DIAG_COST));
  }
  auto rows = [&](int64_t sp) {
    int64_t r = ceil_div(ceil_div(m, sp), BK) * BK;
    return std::max<int64_t>(BK, r);
  };
  b.rps_d = rows(sd);
  b.rps_o = rows(so);
  b.sd = (int)ceil_div(m, b.rps_d);
  b.so = (int)ceil_div(m, b.rps_o);
  b.nd = (int)tp;
  b.on = 1;
  return b;
}
inline Bal plan_bal(int64_t m, int64_t p) { return plan_bal_t(m, p, T, BK, diag_cost()); }
// the 64-wide kernel's diagonal tiles (36 of 64 fragments): opt-in
// (POD_TN_BAL64=1, weight POD_TN_DIAG_COST64).  Measured at config 4
// (r = 192, g = 256): weights 0.75-0.9 tie the unbalanced 1.377 s, 0.6 and
// 1.0 lose -- its leak check sits at the 1e-8 threshold, so the summation
// order of the Grams moves the second-projection count more than the
// balancing saves.
inline Bal plan_bal64(int64_t m, int64_t p) {
  static int on = -1;
  static double v = -1.0;
  if (on < 0) {
    const char* e = getenv("POD_TN_BAL64");
    on = (e && e[0] == '1') ? 1 : 0;
    v = env_cost("POD_TN_DIAG_COST64", 0.9);
  }
  if (!on) return Bal{0, 0, 0, 0, 0, 0};
  return plan_bal_t(m, p, tn::BP, tn::BK, v);
}
// POD_TN_BAL=0: uniform K split and full diagonal tiles (A/B)
inline bool bal_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_TN_BAL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// 80-wide tiles when they cover p x q with less padding than 64-wide ones
inline bool better(int64_t p, int64_t q) {
  const int64_t a64 = ceil_div(p, 64) * 64 * ceil_div(q, 64) * 64;
  const int64_t a80 = ceil_div(p, 80) * 80 * ceil_div(q, 80) * 80;
  return a80 * 10 < a64 * 9;  // at least 10 % less padded work
}
}  // namespace tn80


// -------------------------------------------------- NN persistent ------
// T (p x q, p <= PMAX) resident in shared memory for the whole kernel; each
// CTA walks row blocks of BM rows with the next block's X prefetched by
// cp.async while the current one is multiplied (two buffers).
namespace nnp {
constexpr int THREADS = 256;
constexpr int BM = 64;
constexpr int LDX = BM + 4;  // % 16 == 4: conflict-free A fragments

template <int BN>
struct Cfg {
  static constexpr int WM = BM / 32;  // 2 warps along M
  static constexpr int WN = 8 / WM;   // 4 warps along N
  static constexpr int FN = BN / WN / 8;
};

__host__ __device__ inline int kpad(int p) { return (p + 7) & ~7; }
__host__ __device__ inline int ldt(int p) { return kpad(p) + 4; }  // T stored [j][k], % 16 == 4 when kpad % 16 == 0
inline size_t smem_bytes(int p, int bn) {
  return ((size_t)2 * kpad(p) * LDX + (size_t)bn * ldt(p)) * sizeof(double);
}

// GRAM (BN = 64, p >= q): the output tile, while still on chip, is also
// multiplied by its own transpose -- G_cta += Y_blk^T Y_blk over the CTA's
// row blocks (upper-triangular 8 x 8 fragments, 36 at q = 64, dealt over the
// 8 warps) -- so the CholeskyQR pass that consumes Y needs no TN pass over it
// (merge.py:70 QR of the residual; the Gram of CholeskyQR2's second pass).
// gws[blockIdx.x] receives the CTA's q x q partial (column-major, upper part).
template <int BN, bool GRAM = false>
__global__ void __launch_bounds__(THREADS) kernel(int64_t m, int p, int q, double alpha,
                                                  const double* X, int64_t ldx,
                                                  const int32_t* __restrict__ xcols,
                                                  const double* __restrict__ T, int64_t ldT,
                                                  double beta, const double* Z, int64_t ldz,
                                                  double* Y, int64_t ldy,
                                                  const int32_t* __restrict__ gate, int vec16,
                                                  double* __restrict__ gws = nullptr) {
  using C = Cfg<BN>;
  static_assert(!GRAM || BN == 64, "Gram epilogue: one 64-column group");
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double smem[];
  const int KP = kpad(p), LT = ldt(p);
  double* xs0 = smem;
  double* xs1 = smem + (size_t)KP * LDX;
  double* ts = smem + (size_t)2 * KP * LDX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // T -> smem once (zero padded to KP x BN)
  for (int e = threadIdx.x; e < BN * KP; e += THREADS) {
    const int j = e / KP, k = e - j * KP;
    ts[j * LT + k] = (j < q && k < p) ? T[k + (int64_t)j * ldT] : 0.0;
  }
  const int64_t nblk = (m + BM - 1) / BM;
  auto load_block = [&](double* xs, int64_t rb) {
    const int64_t r0 = rb * BM;
    if (vec16) {
      // 2 rows per lane-slot: BM/2 = 32 slots per column
      for (int e = threadIdx.x; e < KP * (BM / 2); e += THREADS) {
        const int c = e / (BM / 2), i2 = (e - c * (BM / 2)) * 2;
        const int64_t row = r0 + i2;
        bool v = c < p && row + 1 < m;
        int64_t col = c;
        if (c < p && xcols) {
          col = xcols[c];
          v = v && col >= 0;
        }
        if (v) {
          cp_async16(xs + c * LDX + i2, X + col * ldx + row, true);
        } else {
          // tail / padding: element-wise with zero fill
          const bool v0 = c < p && row < m && (!xcols || col >= 0);
          cp_async8(xs + c * LDX + i2, v0 ? X + col * ldx + row : X, v0);
          cp_async8(xs + c * LDX + i2 + 1, X, false);
        }
      }
    } else {
      for (int e = threadIdx.x; e < KP * BM; e += THREADS) {
        const int c = e / BM, i = e - c * BM;
        const int64_t row = r0 + i;
        bool v = c < p && row < m;
        int64_t col = c;
        if (v && xcols) {
          col = xcols[c];
          v = col >= 0;
        }
        cp_async8(xs + c * LDX + i, v ? X + col * ldx + row : X, v);
      }
    }
  };
  const int wm = warp % C::WM, wn = warp / C::WM;
  // Gram fragments of this warp: upper-triangular (fi <= fj) among NQ^2
  constexpr int GF = GRAM ? 5 : 1;  // ceil(36 / 8)
  const int NQ = (q + 7) >> 3;
  int gfi[GF], gfj[GF];
  double gacc[GF][2];
#pragma unroll
  for (int f = 0; f < GF; ++f) {
    gfi[f] = gfj[f] = -1;
    gacc[f][0] = gacc[f][1] = 0.0;
  }
  if constexpr (GRAM) {
#pragma unroll
    for (int f = 0; f < GF; ++f) {  // upper fragment idx = warp + 8 f, column-ordered
      int idx = warp + 8 * f, fj = 0;
      while (idx > fj) {
        idx -= fj + 1;
        ++fj;
      }
      if (fj < NQ) {
        gfi[f] = idx;
        gfj[f] = fj;
      }
    }
  }
  int64_t rb = blockIdx.x;
  if (rb < nblk) load_block(xs0, rb);
  cp_async_commit();
  int buf = 0;
  for (; rb < nblk; rb += gridDim.x) {
    const int64_t nb = rb + gridDim.x;
    if (nb < nblk) load_block(buf ? xs0 : xs1, nb);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* xs = buf ? xs1 : xs0;
    const int64_t row0 = rb * BM + wm * 32;
    double acc[4][C::FN][2];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int g = 0; g < C::FN; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
    // beta Z of this block: loads in flight under the block's DMMAs (BN = 64:
    // 16 doubles per thread; wider tiles load in the epilogue)
    double zv[4][BN == 64 ? C::FN : 1][2];
    if constexpr (BN == 64) {
      if (beta != 0.0) nn_load_z<C::FN>(zv, row0, wn * (BN / C::WN), lane, m, q, Z, ldz);
    }
#pragma unroll 2
    for (int k0 = 0; k0 < KP; k0 += 4) {
      double a[4], b[C::FN];
#pragma unroll
      for (int f = 0; f < 4; ++f)
        a[f] = xs[(k0 + (lane & 3)) * LDX + wm * 32 + f * 8 + (lane >> 2)];
#pragma unroll
      for (int g = 0; g < C::FN; ++g)
        b[g] = ts[(wn * (BN / C::WN) + g * 8 + (lane >> 2)) * LT + k0 + (lane & 3)];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < C::FN; ++g) dmma8x8x4(acc[f][g][0], acc[f][g][1], a[f], b[g]);
    }
    __syncthreads();  // xs fully consumed before the next prefetch overwrites it
    if constexpr (BN == 64)
      nn_store<C::FN>(acc, zv, row0, wn * (BN / C::WN), lane, m, q, alpha, beta, Y, ldy);
    else
      nn_epilogue<C::FN>(acc, row0, wn * (BN / C::WN), lane, m, q, alpha, beta, Z, ldz, Y, ldy);
    if constexpr (GRAM) {
      // the tile as stored (zero outside m x q) -> the consumed X buffer,
      // [col][row] with ld LDX; then the CTA's Gram fragments over its 64 rows
      double* ys = const_cast<double*>(xs);
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < C::FN; ++g)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int il = wm * 32 + f * 8 + (lane >> 2);
            const int j = wn * (BN / C::WN) + g * 8 + 2 * (lane & 3) + e;
            double v = alpha * acc[f][g][e];
            if (beta != 0.0) v += beta * zv[f][g][e];
            if (j < NQ * 8) ys[j * LDX + il] = (rb * BM + il < m && j < q) ? v : 0.0;
          }
      __syncthreads();
#pragma unroll
      for (int f = 0; f < GF; ++f) {
        if (gfi[f] < 0) continue;
        const double* ya = ys + (gfi[f] * 8 + (lane >> 2)) * LDX + (lane & 3);
        const double* yb = ys + (gfj[f] * 8 + (lane >> 2)) * LDX + (lane & 3);
#pragma unroll 4
        for (int k0 = 0; k0 < BM; k0 += 4) dmma8x8x4(gacc[f][0], gacc[f][1], ya[k0], yb[k0]);
      }
      __syncthreads();  // ys (this block's X buffer) is the next prefetch's target
    }
    buf ^= 1;
  }
  cp_async_wait<0>();
  if constexpr (GRAM) {
    double* out = gws + (size_t)blockIdx.x * q * q;
#pragma unroll
    for (int f = 0; f < GF; ++f) {
      if (gfi[f] < 0) continue;
      const int i = gfi[f] * 8 + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = gfj[f] * 8 + 2 * (lane & 3) + e;
        if (i < q && j < q) out[(size_t)j * q + i] = gacc[f][e];
      }
    }
  }
}
}  // namespace nnp

// -------------------------------------------------- NN streamed, persistent ----
// For p too large to keep T resident: every CTA walks its row blocks and the
// k-chunks of each block as ONE flattened (block, chunk) sequence behind a
// STAGES-deep cp.async pipeline, so the next block's X and T chunks load while
// the current block finishes and writes its epilogue (no per-block pipeline
// fill/drain).  T chunks are re-read per block from L2; X rows come from HBM
// once.  A CTA reads all chunks of a block before writing that block's rows,
// so Y may alias X or Z.
namespace nns {
constexpr int THREADS = 256;
#ifndef POD_NNS_BK80
#define POD_NNS_BK80 16
#endif
#ifndef POD_NNS_MINB
#define POD_NNS_MINB 1
#endif
#ifndef POD_NNS_ST80
#define POD_NNS_ST80 4
#endif

#ifndef POD_NN80_WIDE
#define POD_NN80_WIDE 0
#endif
template <int BN, typename TX = double>
struct Cfg {
  // BN = 80 (column groups of 80: q = 150 -> 160 instead of 192) runs 10
  // warps of 32 x 16 tiles, or (POD_NN80_WIDE) 8 warps of 32 x 40 tiles on
  // 128-row blocks (20 DMMAs per 9 fragment loads instead of 8 per 6)
  static constexpr bool W80 = (BN == 80) && POD_NN80_WIDE;
  static constexpr int NWARP = (BN == 80 && !W80) ? 10 : 8;
  static constexpr int BK = BN == 80 ? POD_NNS_BK80 : 16;  // k-chunk per pipeline stage
  static constexpr int LDT = BK + 4;                         // T chunk stored [j][k]
  static constexpr int NTHREADS = NWARP * 32;
  static constexpr int STAGES = (BN == 128 || W80) ? 3 : (BN == 80 ? POD_NNS_ST80 : 4);
  static constexpr int BM = (BN == 64 || W80) ? 128 : 64;  // rows per block (T reuse)
  // X chunk stored [k][row] in X's own type (fp32 storage converted exactly
  // at the fragment loads); padding keeps the fragment loads conflict-free
  static constexpr int LDX = BM + (sizeof(TX) == 8 ? 4 : 8);
  static constexpr int WM = BM / 32;  // warps along M
  static constexpr int WN = NWARP / WM;  // warps along N
  static constexpr int FN = BN / WN / 8;
  static constexpr int XT = BK * LDX, TT = BN * LDT;
  static constexpr size_t XBYTES = size_t(XT) * sizeof(TX);  // multiple of 16
  static constexpr size_t SMEM = size_t(STAGES) * (XBYTES + size_t(TT) * sizeof(double));
  static constexpr int PER_SM = (BN == 192) ? 1 : 2;
};
// blockIdx.y selects a group of BN output columns (q0 = blockIdx.y * BN); more
// than one group only when Y aliases neither X nor Z (a group writes its
// columns of a row block while another group may still be reading X there).

template <int BN, typename TX = double, bool DOTS = false>
__global__ void __launch_bounds__(Cfg<BN, TX>::NTHREADS, POD_NNS_MINB) kernel(int64_t m, int p, int q,
                                                                 double alpha,
                                                  const TX* X, int64_t ldx,
                                                  const int32_t* __restrict__ xcols,
                                                  const double* __restrict__ T, int64_t ldT,
                                                  double beta, const double* Z, int64_t ldz,
                                                  double* Y, int64_t ldy,
                                                  const int32_t* __restrict__ gate, int vx, int vt,
                                                  const double* __restrict__ DX = nullptr,
                                                  int64_t dldx = 0, int kdot = 0,
                                                  double* __restrict__ dws = nullptr) {
  using C = Cfg<BN, TX>;
  constexpr int ST = C::STAGES;
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto stage_x = [&](int st) {
    return reinterpret_cast<TX*>(smem_raw + (size_t)st * (C::XBYTES + C::TT * sizeof(double)));
  };
  auto stage_t = [&](int st) {
    return reinterpret_cast<double*>(smem_raw + (size_t)st * (C::XBYTES + C::TT * sizeof(double)) +
                                     C::XBYTES);
  };
  // column dots (kdot > 0, fp64 X): local columns j < kdl of this group
  const int q0 = blockIdx.y * BN;
  const int kdl = DOTS ? min(kdot - q0, BN) : 0;
  {
    T += (int64_t)q0 * ldT;
    Y += (int64_t)q0 * ldy;
    if (Z) Z += (int64_t)q0 * ldz;
    if (kdl > 0) DX += (int64_t)q0 * dldx;
    q = min(BN, q - q0);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nkb = (p + C::BK - 1) / C::BK;
  const int64_t nblk = (m + C::BM - 1) / C::BM;
  const int64_t G = gridDim.x;
  if ((int64_t)blockIdx.x >= nblk) {
    for (int j = threadIdx.x; j < kdl; j += C::NTHREADS)
      dws[(int64_t)(q0 + j) * gridDim.x + blockIdx.x] = 0.0;
    return;
  }
  const int64_t nmine = (nblk - blockIdx.x + G - 1) / G;
  const int64_t total = nmine * nkb;

  // (block, chunk) of the next load, advanced incrementally: no 64-bit
  // division in the loop (its DMUL-based emulation shares the FP64 pipe)
  int64_t l_r0 = (int64_t)blockIdx.x * C::BM;
  int l_kb = 0;
  auto load_stage = [&](int st) {
    TX* xs = stage_x(st);
    double* ts = stage_t(st);
    const int k0 = l_kb * C::BK;
    const int64_t r0 = l_r0;
    if (++l_kb == nkb) {
      l_kb = 0;
      l_r0 += G * C::BM;
    }
    // X: C::BM rows x C::BK cols as row pairs (2 x 8 B)
    for (int e = threadIdx.x; e < C::BK * (C::BM / 2); e += C::NTHREADS) {
      const int cl = e / (C::BM / 2), i2 = (e - cl * (C::BM / 2)) * 2;
      const int c = k0 + cl;
      const int64_t row = r0 + i2;
      int64_t col = c;
      bool cv = c < p;
      if (cv && xcols) {
        col = xcols[c];
        cv = col >= 0;  // index -1: zero column
      }
      TX* dst = xs + cl * C::LDX + i2;
      const TX* src = X + col * ldx + row;
      if (cv && vx && row + 1 < m) {
        if constexpr (sizeof(TX) == 8) cp_async16(dst, src, true);
        else cp_async8(dst, src, true);
      } else {
        cp_async_elem(dst, cv && row < m ? src : X, cv && row < m);
        cp_async_elem(dst + 1, cv && row + 1 < m ? src + 1 : X, cv && row + 1 < m);
      }
    }
    // T: rows k0..k0+C::BK, all BN cols, k pairs
    for (int e = threadIdx.x; e < BN * (C::BK / 2); e += C::NTHREADS) {
      const int j = e / (C::BK / 2), k2 = (e - j * (C::BK / 2)) * 2;
      const int k = k0 + k2;
      const bool jv = j < q;
      double* dst = ts + j * C::LDT + k2;
      const double* src = T + k + (int64_t)j * ldT;
      if (jv && vt && k + 1 < p) {
        cp_async16(dst, src, true);
      } else {
        cp_async8(dst, jv && k < p ? src : T, jv && k < p);
        cp_async8(dst + 1, jv && k + 1 < p ? src + 1 : T, jv && k + 1 < p);
      }
    }
  };

  const int wm = warp % C::WM, wn = warp / C::WM;
  double acc[4][C::FN][2];
  double dacc[C::FN][2];
#pragma unroll
  for (int g = 0; g < C::FN; ++g) dacc[g][0] = dacc[g][1] = 0.0;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < total) load_stage(s);
    cp_async_commit();
  }
  int kb = 0, st_c = 0, st_l = ST - 1;
  int64_t c_r0 = (int64_t)blockIdx.x * C::BM;
  for (int64_t it = 0; it < total; ++it) {
    // stage `it` has landed once at most ST - 2 groups are pending; after the
    // barrier every warp is done with stage it - 1, which the prefetch below
    // refills -- one barrier per stage
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (it + ST - 1 < total) load_stage(st_l);
    if (++st_l == ST) st_l = 0;
    cp_async_commit();
    if (kb == 0) {
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < C::FN; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
    }
    const TX* xs = stage_x(st_c);
    const double* ts = stage_t(st_c);
    if (++st_c == ST) st_c = 0;

#pragma unroll
    for (int kk = 0; kk < C::BK / 4; ++kk) {
      double a[4], b[C::FN];
#pragma unroll
      for (int f = 0; f < 4; ++f)
        a[f] = (double)xs[(kk * 4 + (lane & 3)) * C::LDX + wm * 32 + f * 8 + (lane >> 2)];
#pragma unroll
      for (int g = 0; g < C::FN; ++g)
        b[g] = ts[(wn * (BN / C::WN) + g * 8 + (lane >> 2)) * C::LDT + kk * 4 + (lane & 3)];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < C::FN; ++g) dmma8x8x4(acc[f][g][0], acc[f][g][1], a[f], b[g]);
    }
    if (++kb == nkb) {
      kb = 0;
      const int64_t row0 = c_r0 + wm * 32;
      c_r0 += G * C::BM;
      if constexpr (DOTS)  // beta = 0 (pod_gemm_nn_dots)
        nn_epilogue_dots<C::FN>(acc, row0, wn * (BN / C::WN), lane, m, q, alpha, Y, ldy, DX, dldx,
                                kdl, dacc);
      else
        nn_epilogue<C::FN>(acc, row0, wn * (BN / C::WN), lane, m, q, alpha, beta, Z, ldz, Y, ldy);
    }
  }
  cp_async_wait<0>();
  if (DOTS && kdl > 0) {
    // CTA column sums in a fixed order: lanes sharing a column, then the
    // WM warps along M through shared memory (the stages are free now)
    __syncthreads();
    double* red = reinterpret_cast<double*>(smem_raw);  // WM x BN
#pragma unroll
    for (int g = 0; g < C::FN; ++g)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = dacc[g][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (lane < 4) red[wm * BN + wn * (BN / C::WN) + g * 8 + 2 * lane + e] = v;
      }
    __syncthreads();
    for (int j = threadIdx.x; j < kdl; j += C::NTHREADS) {
      double t = 0.0;
      for (int w = 0; w < C::WM; ++w) t += red[w * BN + j];
      dws[(int64_t)(q0 + j) * gridDim.x + blockIdx.x] = t;
    }
  }
}

// Warp-specialized variant of kernel<> (beta Z epilogue, no column dots):
// one producer warp streams the (block, chunk) sequence into the STAGES ring
// with cp.async, each lane's copies completing on the stage's `full`
// mbarrier (cp.async.mbarrier.arrive.noinc), and the NWARP consumer warps
// release a stage through its `empty` mbarrier once their fragments are
// loaded -- no CTA-wide barrier per stage, so a warp may run up to STAGES - 1
// chunks ahead of the slowest.  Same fragments, same k order, same epilogue:
// bitwise equal to kernel<>.
template <int BN, typename TX = double>
__global__ void __launch_bounds__(Cfg<BN, TX>::NTHREADS + 32, Cfg<BN, TX>::PER_SM) kernel_ws(
    int64_t m, int p, int q, double alpha, const TX* X, int64_t ldx,
    const int32_t* __restrict__ xcols, const double* __restrict__ T, int64_t ldT, double beta,
    const double* Z, int64_t ldz, double* Y, int64_t ldy, const int32_t* __restrict__ gate,
    int vx, int vt) {
  using C = Cfg<BN, TX>;
  constexpr int ST = C::STAGES;
  constexpr size_t STB = C::XBYTES + C::TT * sizeof(double);
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)ST * STB);
  uint64_t* empty = full + ST;
  const int q0 = blockIdx.y * BN;
  T += (int64_t)q0 * ldT;
  Y += (int64_t)q0 * ldy;
  if (Z) Z += (int64_t)q0 * ldz;
  q = min(BN, q - q0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nkb = (p + C::BK - 1) / C::BK;
  const int64_t nblk = (m + C::BM - 1) / C::BM;
  const int64_t G = gridDim.x;
  if ((int64_t)blockIdx.x >= nblk) return;
  const int64_t nmine = (nblk - blockIdx.x + G - 1) / G;
  const int64_t total = nmine * nkb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mb_init(&full[s], 32);
      mb_init(&empty[s], C::NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == C::NWARP) {  // ---- producer warp
    int64_t r0 = (int64_t)blockIdx.x * C::BM;
    int kb = 0, st = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < total; ++it) {
      if (it >= ST) mb_wait(&empty[st], ph ^ 1);
      TX* xs = reinterpret_cast<TX*>(smem_raw + (size_t)st * STB);
      double* ts = reinterpret_cast<double*>(smem_raw + (size_t)st * STB + C::XBYTES);
      const int k0 = kb * C::BK;
      // the chunk's gathered column ids, one per lane (BK <= 32), broadcast
      // below by shuffles instead of a dependent load per copy
      int mycol = k0 + lane;
      if (xcols && lane < C::BK && k0 + lane < p) mycol = xcols[k0 + lane];
      for (int e = lane; e < C::BK * (C::BM / 2); e += 32) {
        const int cl = e / (C::BM / 2), i2 = (e - cl * (C::BM / 2)) * 2;
        const int c = k0 + cl;
        const int64_t row = r0 + i2;
        const int colv = __shfl_sync(0xffffffffu, mycol, cl);
        int64_t col = colv;
        bool cv = c < p && colv >= 0;  // index -1: zero column
        TX* dst = xs + cl * C::LDX + i2;
        const TX* src = X + col * ldx + row;
        if (cv && vx && row + 1 < m) {
          if constexpr (sizeof(TX) == 8) cp_async16(dst, src, true);
          else cp_async8(dst, src, true);
        } else {
          cp_async_elem(dst, cv && row < m ? src : X, cv && row < m);
          cp_async_elem(dst + 1, cv && row + 1 < m ? src + 1 : X, cv && row + 1 < m);
        }
      }
      for (int e = lane; e < BN * (C::BK / 2); e += 32) {
        const int j = e / (C::BK / 2), k2 = (e - j * (C::BK / 2)) * 2;
        const int k = k0 + k2;
        const bool jv = j < q;
        double* dst = ts + j * C::LDT + k2;
        const double* src = T + k + (int64_t)j * ldT;
        if (jv && vt && k + 1 < p) {
          cp_async16(dst, src, true);
        } else {
          cp_async8(dst, jv && k < p ? src : T, jv && k < p);
          cp_async8(dst + 1, jv && k + 1 < p ? src + 1 : T, jv && k + 1 < p);
        }
      }
      mb_cp_async_arrive(&full[st]);
      if (++kb == nkb) {
        kb = 0;
        r0 += G * C::BM;
      }
      if (++st == ST) {
        st = 0;
        ph ^= 1;
      }
    }
    cp_async_wait<0>();
    return;
  }

  // ---- consumer warps
  const int wm = warp % C::WM, wn = warp / C::WM;
  double acc[4][C::FN][2];
  int kb = 0, st = 0;
  uint32_t ph = 0;
  int64_t c_r0 = (int64_t)blockIdx.x * C::BM;
  for (int64_t it = 0; it < total; ++it) {
    mb_wait(&full[st], ph);
    if (kb == 0) {
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < C::FN; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
    }
    const TX* xs = reinterpret_cast<const TX*>(smem_raw + (size_t)st * STB);
    const double* ts = reinterpret_cast<const double*>(smem_raw + (size_t)st * STB + C::XBYTES);
#pragma unroll
    for (int kk = 0; kk < C::BK / 4; ++kk) {
      double a[4], b[C::FN];
#pragma unroll
      for (int f = 0; f < 4; ++f)
        a[f] = (double)xs[(kk * 4 + (lane & 3)) * C::LDX + wm * 32 + f * 8 + (lane >> 2)];
#pragma unroll
      for (int g = 0; g < C::FN; ++g)
        b[g] = ts[(wn * (BN / C::WN) + g * 8 + (lane >> 2)) * C::LDT + kk * 4 + (lane & 3)];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < C::FN; ++g) dmma8x8x4(acc[f][g][0], acc[f][g][1], a[f], b[g]);
    }
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[st]);
    if (++st == ST) {
      st = 0;
      ph ^= 1;
    }
    if (++kb == nkb) {
      kb = 0;
      const int64_t row0 = c_r0 + wm * 32;
      c_r0 += G * C::BM;
      nn_epilogue<C::FN>(acc, row0, wn * (BN / C::WN), lane, m, q, alpha, beta, Z, ldz, Y, ldy);
    }
  }
}
template <int BN, typename TX = double>
constexpr size_t ws_smem() {
  return (size_t)Cfg<BN, TX>::STAGES * (Cfg<BN, TX>::XBYTES + Cfg<BN, TX>::TT * sizeof(double)) +
         2 * Cfg<BN, TX>::STAGES * sizeof(uint64_t);
}

// out[j] = sum over the CTAs of dws[j][cta] (fixed order), j < k
__global__ void dots_final_kernel(const double* __restrict__ dws, int nchunk, int k,
                                  double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double t = 0.0;
  for (int c = 0; c < nchunk; ++c) t += dws[(int64_t)j * nchunk + c];
  out[j] = t;
}
}  // namespace nns

static bool g_attr_done = false;
// POD_TN80=0 disables the 80-wide TN tiles (A/B measurements)
static bool tn80_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_TN80");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// Warp-specialized 80-wide TN partial kernel (default; POD_TN_WS=0: the
// barrier-per-stage kernel, A/B).  Config-3 shapes: Gram 1.125 -> 1.052 ms,
// gathered Gram 2.485 -> 2.322 ms, U1^T U2 1.755 -> 1.732 ms (bitwise equal).
static bool tn_ws_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_TN_WS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// column groups of 80 instead of 64 when they pad at least 10 % less
// (POD_NN80=0 disables, for A/B measurements)
static bool nn_groups80(int64_t q) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_NN80");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1 && q > 64 && ceil_div(q, 80) * 80 * 10 < ceil_div(q, 64) * 64 * 9;
}
// POD_NN_GROUPS=0 disables column groups in the streamed NN kernel (A/B)
static bool nn_groups_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_NN_GROUPS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
static int ensure_attrs() {
  if (g_attr_done) return POD_OK;
  cudaError_t e = cudaFuncSetAttribute(tn::partial_kernel<double, double>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tn::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "tn attr");
  e = cudaFuncSetAttribute(tn::partial_kernel<float, float>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tn::smem_bytes<float, float>());
  if (e != cudaSuccess) return cuda_status(e, "tn attr");
  e = cudaFuncSetAttribute(tn::partial_kernel<float, double>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tn::smem_bytes<float, double>());
  if (e != cudaSuccess) return cuda_status(e, "tn attr");
  e = cudaFuncSetAttribute(tn::partial_kernel<double, float>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tn::smem_bytes<double, float>());
  if (e != cudaSuccess) return cuda_status(e, "tn attr");
#define TN64_BAL_ATTR(A_, B_)                                                              \
  e = cudaFuncSetAttribute(tn::partial_kernel<A_, B_, true>,                               \
                           cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                           (int)tn::smem_bytes<A_, B_>());                                 \
  if (e != cudaSuccess) return cuda_status(e, "tn bal attr");
  TN64_BAL_ATTR(double, double)
  TN64_BAL_ATTR(float, float)
  TN64_BAL_ATTR(float, double)
  TN64_BAL_ATTR(double, float)
#undef TN64_BAL_ATTR
#define TN80_ATTR1(A_, B_, BAL_, WS_)                                                        \
  e = cudaFuncSetAttribute(tn80::partial_kernel<A_, B_, BAL_, WS_>,                        \
                           cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                           (int)tn80::smem_bytes<A_, B_>());                               \
  if (e != cudaSuccess) return cuda_status(e, "tn80 attr");
#define TN80_ATTR(A_, B_)                                                                   \
  TN80_ATTR1(A_, B_, false, false) TN80_ATTR1(A_, B_, true, false)                          \
  TN80_ATTR1(A_, B_, false, true) TN80_ATTR1(A_, B_, true, true)
  TN80_ATTR(double, double)
  TN80_ATTR(float, float)
  TN80_ATTR(float, double)
  TN80_ATTR(double, float)
#undef TN80_ATTR
#undef TN80_ATTR1
  e = cudaFuncSetAttribute((const void*)nnp::kernel<64, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return cuda_status(e, "nnp gram attr");
  for (int bn : {64, 128, 192}) {
    const void* fn = bn == 64 ? (const void*)nnp::kernel<64>
                   : bn == 128 ? (const void*)nnp::kernel<128> : (const void*)nnp::kernel<192>;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "nnp attr");
  }
#define NNS_DOTS_ATTR(BN_)                                                                 \
  e = cudaFuncSetAttribute(nns::kernel<BN_, double, true>,                                 \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nns::Cfg<BN_>::SMEM); \
  if (e != cudaSuccess) return cuda_status(e, "nns dots attr");
  NNS_DOTS_ATTR(64)
  NNS_DOTS_ATTR(80)
  NNS_DOTS_ATTR(128)
  NNS_DOTS_ATTR(192)
#undef NNS_DOTS_ATTR
  e = cudaFuncSetAttribute(nns::kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)nns::Cfg<64>::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "nns attr");
  e = cudaFuncSetAttribute(nns::kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)nns::Cfg<128>::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "nns attr");
  e = cudaFuncSetAttribute(nns::kernel<192>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)nns::Cfg<192>::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "nns attr");
  e = cudaFuncSetAttribute(nns::kernel<64, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)nns::Cfg<64, float>::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "nns attr");
  e = cudaFuncSetAttribute(nns::kernel<80>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)nns::Cfg<80>::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "nns attr");
  e = cudaFuncSetAttribute(nns::kernel<80, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)nns::Cfg<80, float>::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "nns attr");
  g_attr_done = true;
  return POD_OK;
}

}  // namespace pod

using namespace pod;

static int nn_streamed(int64_t m, int64_t p, int64_t q, double alpha, const double* X,
                       int64_t ldx, const int32_t* xcols, const double* T, int64_t ldt,
                       double beta, const double* Z, int64_t ldz, double* Y, int64_t ldy,
                       const int32_t* gate, cudaStream_t s, const double* DX, int64_t dldx,
                       int kdot, double* dws, int64_t* nchunk_out);

extern "C" size_t pod_gemm_tn_ws_bytes(int64_t m, int64_t p, int64_t q) {
  if (m <= 0 || p <= 0 || q <= 0) return 0;
  const tn::Plan a = tn::plan(m, p, q, false), b = tn::plan(m, p, q, p == q);
  const tn::Plan c = tn80::plan(m, p, q, false), d = tn80::plan(m, p, q, p == q);
  int sp = std::max(std::max(a.splits, b.splits), std::max(c.splits, d.splits));
  if (p == q) sp = std::max(sp, std::max(tn80::plan_bal(m, p).so, tn80::plan_bal64(m, p).so));
  return (size_t)sp * p * q * sizeof(double);
}

extern "C" int pod_gemm_tn(int xtype, int ytype, int64_t m, int64_t p, int64_t q, double alpha,
                           const void* X, int64_t ldx, const int32_t* xcols, const void* Y,
                           int64_t ldy, const int32_t* ycols, double* C, int64_t ldc, void* ws,
                           size_t ws_bytes, const int32_t* gate, void* stream) {
  POD_REQUIRE(m >= 0 && p >= 0 && q >= 0, "pod_gemm_tn: negative size");
  POD_REQUIRE(ldc >= p, "pod_gemm_tn: ldc < p");
  POD_REQUIRE((xtype == POD_F64 || xtype == POD_F32) && (ytype == POD_F64 || ytype == POD_F32),
              "pod_gemm_tn: bad operand type");
  if (p == 0 || q == 0) return POD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  POD_REQUIRE(m > 0, "pod_gemm_tn: m must be >= 1");
  int st = ensure_attrs();
  if (st) return st;
  const int sym = (X == Y && ldx == ldy && xcols == ycols && p == q && xtype == ytype) ? 1 : 0;
  const bool w80 = tn80::better(p, q) && tn80_enabled();
  tn::Plan pl = w80 ? tn80::plan(m, p, q, sym != 0) : tn::plan(m, p, q, sym != 0);
  tn80::Bal bal = {0, 0, 0, 0, 0, 0};
  if (sym && tn80::bal_enabled()) bal = w80 ? tn80::plan_bal(m, p) : tn80::plan_bal64(m, p);
  const int nsplit = bal.on ? bal.so : pl.splits;
  POD_REQUIRE(ws_bytes >= (size_t)nsplit * p * q * sizeof(double),
              "pod_gemm_tn: workspace too small (%zu < %zu)", ws_bytes,
              (size_t)nsplit * p * q * sizeof(double));
  dim3 grid(pl.tiles, pl.splits);
  if (bal.on)
    grid = dim3((unsigned)(bal.nd * bal.sd + (bal.nd * (bal.nd - 1) / 2) * bal.so), 1);
  if (w80) {
#define TN80_LAUNCH(A_, B_)                                                                     \
  (tnws ? (bal.on ? tn80::partial_kernel<A_, B_, true, true>                                     \
                  : tn80::partial_kernel<A_, B_, false, true>)                                  \
        : (bal.on ? tn80::partial_kernel<A_, B_, true> : tn80::partial_kernel<A_, B_, false>))  \
      <<<grid, tn80::THREADS + (tnws ? 32 * tn80::NPROD : 0), tn80::smem_bytes<A_, B_>(), s>>>(                \
      m, (int)p, (int)q, (const A_*)X, ldx, xcols, (const B_*)Y, ldy, ycols, pl.rows_per_split, \
      (double*)ws, gate, sym, bal)
    const bool tnws = tn_ws_enabled();
    if (xtype == POD_F64 && ytype == POD_F64) TN80_LAUNCH(double, double);
    else if (xtype == POD_F64) TN80_LAUNCH(double, float);
    else if (ytype == POD_F32) TN80_LAUNCH(float, float);
    else TN80_LAUNCH(float, double);
#undef TN80_LAUNCH
  } else {
#define TN64_LAUNCH(A_, B_)                                                                     \
  (bal.on ? tn::partial_kernel<A_, B_, true> : tn::partial_kernel<A_, B_, false>)               \
      <<<grid, tn::THREADS, tn::smem_bytes<A_, B_>(), s>>>(                                     \
      m, (int)p, (int)q, (const A_*)X, ldx, xcols, (const B_*)Y, ldy, ycols, pl.rows_per_split, \
      (double*)ws, gate, sym, bal)
    if (xtype == POD_F64 && ytype == POD_F64) TN64_LAUNCH(double, double);
    else if (xtype == POD_F64) TN64_LAUNCH(double, float);
    else if (ytype == POD_F32) TN64_LAUNCH(float, float);
    else TN64_LAUNCH(float, double);
#undef TN64_LAUNCH
  }
  POD_CHECK_LAUNCH("tn partial");
  int64_t tot = p * q;
  int blocks = (int)std::min<int64_t>(ceil_div(tot, 8), 16 * 148);  // 8 warps = 8 outputs per block
  tn::reduce_kernel<<<blocks, 256, 0, s>>>(nsplit, (int)p, (int)q, alpha, (const double*)ws, C,
                                           ldc, gate, sym, bal.on ? bal.sd : 0,
                                           w80 ? tn80::T : tn::BP);
  POD_CHECK_LAUNCH("tn reduce");
  return POD_OK;
}

extern "C" int pod_gemm_tn_f64(int64_t m, int64_t p, int64_t q, double alpha, const double* X,
                               int64_t ldx, const int32_t* xcols, const double* Y, int64_t ldy,
                               const int32_t* ycols, double* C, int64_t ldc, void* ws,
                               size_t ws_bytes, const int32_t* gate, void* stream) {
  return pod_gemm_tn(POD_F64, POD_F64, m, p, q, alpha, X, ldx, xcols, Y, ldy, ycols, C, ldc, ws,
                     ws_bytes, gate, stream);
}

// X stored fp32 (exactly converted to fp64 inside): streamed kernel, column
// groups of 64 (Y is fp64, so it never aliases X)
static int gemm_nn_x32(int64_t m, int64_t p, int64_t q, double alpha, const float* X, int64_t ldx,
                       const int32_t* xcols, const double* T, int64_t ldt, double beta,
                       const double* Z, int64_t ldz, double* Y, int64_t ldy, const int32_t* gate,
                       cudaStream_t s) {
  const int vx = ((reinterpret_cast<uintptr_t>(X) & 7) == 0) && (ldx % 2 == 0);
  const int vt = ((reinterpret_cast<uintptr_t>(T) & 15) == 0) && (ldt % 2 == 0);
  if (nn_groups80(q)) {
    using C = nns::Cfg<80, float>;
    const int64_t nblk = ceil_div(m, C::BM);
    const unsigned gy = (unsigned)ceil_div(q, 80);
    const int64_t per = std::max<int64_t>(1, capped(C::PER_SM * 148) / gy);
    const dim3 grid((unsigned)std::min<int64_t>(nblk, per), gy);
    nns::kernel<80, float><<<grid, C::NTHREADS, C::SMEM, s>>>(m, (int)p, (int)q, alpha, X, ldx,
                                                              xcols, T, ldt, beta, Z, ldz, Y,
                                                              ldy, gate, vx, vt);
  } else {
    using C = nns::Cfg<64, float>;
    const int64_t nblk = ceil_div(m, C::BM);
    const unsigned gy = (unsigned)ceil_div(q, 64);
    const int64_t per = std::max<int64_t>(1, capped(C::PER_SM * 148) / gy);
    const dim3 grid((unsigned)std::min<int64_t>(nblk, per), gy);
    nns::kernel<64, float><<<grid, C::NTHREADS, C::SMEM, s>>>(m, (int)p, (int)q, alpha, X, ldx,
                                                              xcols, T, ldt, beta, Z, ldz, Y,
                                                              ldy, gate, vx, vt);
  }
  POD_CHECK_LAUNCH("nn streamed (fp32 X)");
  return POD_OK;
}

extern "C" int pod_gemm_nn(int xtype, int64_t m, int64_t p, int64_t q, double alpha,
                           const void* X, int64_t ldx, const int32_t* xcols, const double* T,
                           int64_t ldt, double beta, const double* Z, int64_t ldz, double* Y,
                           int64_t ldy, const int32_t* gate, void* stream) {
  POD_REQUIRE(xtype == POD_F64 || xtype == POD_F32, "pod_gemm_nn: bad operand type");
  if (xtype == POD_F64)
    return pod_gemm_nn_f64(m, p, q, alpha, (const double*)X, ldx, xcols, T, ldt, beta, Z, ldz, Y,
                           ldy, gate, stream);
  POD_REQUIRE(m >= 0 && p >= 0 && q >= 0, "pod_gemm_nn: negative size");
  if (m == 0 || q == 0) return POD_OK;
  POD_REQUIRE(ldy >= m, "pod_gemm_nn: ldy < m");
  POD_REQUIRE(beta == 0.0 || Z != nullptr, "pod_gemm_nn: beta != 0 needs Z");
  int st = ensure_attrs();
  if (st) return st;
  return gemm_nn_x32(m, p, q, alpha, (const float*)X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy,
                     gate, (cudaStream_t)stream);
}

extern "C" int pod_gemm_nn_f64(int64_t m, int64_t p, int64_t q, double alpha, const double* X,
                               int64_t ldx, const int32_t* xcols, const double* T, int64_t ldt,
                               double beta, const double* Z, int64_t ldz, double* Y, int64_t ldy,
                               const int32_t* gate, void* stream) {
  POD_REQUIRE(m >= 0 && p >= 0 && q >= 0, "pod_gemm_nn_f64: negative size");
  if (m == 0 || q == 0) return POD_OK;
  POD_REQUIRE(ldy >= m, "pod_gemm_nn_f64: ldy < m");
  POD_REQUIRE(beta == 0.0 || Z != nullptr, "pod_gemm_nn_f64: beta != 0 needs Z");
  int st = ensure_attrs();
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (q <= 192) {
    const int bn = q <= 64 ? 64 : (q <= 128 ? 128 : 192);
    const size_t bytes = nnp::smem_bytes((int)p, bn);
    if (p >= 1 && bytes <= 110 * 1024) {  // T resident, 2 CTAs/SM: persistent kernel
      const int vec16 = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && (ldx % 2 == 0);
      const int per_sm = bytes <= 110 * 1024 ? 2 : 1;
      const int64_t nblk = ceil_div(m, nnp::BM);
      const unsigned grid = (unsigned)std::min<int64_t>(nblk, capped((int64_t)per_sm * 148));
      if (bn == 64)
        nnp::kernel<64><<<grid, nnp::THREADS, bytes, s>>>(m, (int)p, (int)q, alpha, X, ldx, xcols,
                                                          T, ldt, beta, Z, ldz, Y, ldy, gate, vec16);
      else if (bn == 128)
        nnp::kernel<128><<<grid, nnp::THREADS, bytes, s>>>(m, (int)p, (int)q, alpha, X, ldx, xcols,
                                                           T, ldt, beta, Z, ldz, Y, ldy, gate, vec16);
      else
        nnp::kernel<192><<<grid, nnp::THREADS, bytes, s>>>(m, (int)p, (int)q, alpha, X, ldx, xcols,
                                                           T, ldt, beta, Z, ldz, Y, ldy, gate, vec16);
      POD_CHECK_LAUNCH("nn persistent");
      return POD_OK;
    }
  }
  int64_t nchunk = 0;
  return nn_streamed(m, p, q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy, gate, s, nullptr,
                     0, 0, nullptr, &nchunk);
}

// The warp-specialized streamed NN kernel (default; POD_NN_WS=0: the
// barrier-per-stage kernel, A/B).  Config-3 shapes: rotation 4.94 -> 3.53 ms,
// residual 3.15 -> 2.13, apply 2.69 -> 1.91, lift 3.48 -> 2.76 (bitwise equal).
static bool nn_ws_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_NN_WS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
template <int BN>
static int launch_nn_ws(dim3 grid, cudaStream_t s, int64_t m, int64_t p, int64_t q, double alpha,
                        const double* X, int64_t ldx, const int32_t* xcols, const double* T,
                        int64_t ldt, double beta, const double* Z, int64_t ldz, double* Y,
                        int64_t ldy, const int32_t* gate, int vx, int vt) {
  static bool attr = false;
  constexpr size_t smem = nns::ws_smem<BN>();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(nns::kernel_ws<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "nns ws attr");
    attr = true;
  }
  nns::kernel_ws<BN><<<grid, nns::Cfg<BN>::NTHREADS + 32, smem, s>>>(
      m, (int)p, (int)q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy, gate, vx, vt);
  POD_CHECK_LAUNCH("nn streamed ws");
  return POD_OK;
}

// The streamed (nns) launches of pod_gemm_nn_f64, with optional column dots
// (kdot > 0: dws[j][cta] partials; *nchunk_out = CTAs along the rows).
static int nn_streamed(int64_t m, int64_t p, int64_t q, double alpha, const double* X,
                       int64_t ldx, const int32_t* xcols, const double* T, int64_t ldt,
                       double beta, const double* Z, int64_t ldz, double* Y, int64_t ldy,
                       const int32_t* gate, cudaStream_t s, const double* DX, int64_t dldx,
                       int kdot, double* dws, int64_t* nchunk_out) {
  {
    const int vx = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && (ldx % 2 == 0);
    const int vt = ((reinterpret_cast<uintptr_t>(T) & 15) == 0) && (ldt % 2 == 0);
    // Y aliasing X or Z (in-place Q <- Q R^-1): one column group only
    auto overlaps = [&](const double* a, int64_t lda, int64_t ncols) {
      if (!a) return false;
      const char* a0 = (const char*)a;
      const char* a1 = (const char*)(a + (ncols - 1) * lda + m);
      const char* y0 = (const char*)Y;
      const char* y1 = (const char*)(Y + (q - 1) * ldy + m);
      return a0 < y1 && y0 < a1;
    };
    const bool alias = overlaps(X, ldx, p) || (beta != 0.0 && overlaps(Z, ldz, q));
    // > 192 output columns: column groups only (each group reads all of X)
    POD_REQUIRE(q <= 192 || !alias, "pod_gemm_nn_f64: in-place update with q=%lld > 192",
                (long long)q);
    if (q <= 64 || q > 192 || (!alias && nn_groups_enabled())) {
      if (nn_groups80(q)) {  // groups of 80 pad less (q = 150: 160 vs 192)
        using C80 = nns::Cfg<80>;
        const int64_t nblk = ceil_div(m, C80::BM);
        const unsigned gy = (unsigned)ceil_div(q, 80);
        const int64_t per = std::max<int64_t>(1, capped(C80::PER_SM * 148) / gy);
        const dim3 grid((unsigned)std::min<int64_t>(nblk, per), gy);
        *nchunk_out = grid.x;
        if (kdot == 0 && nn_ws_enabled())
          return launch_nn_ws<80>(grid, s, m, p, q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz,
                                  Y, ldy, gate, vx, vt);
        (kdot > 0 ? nns::kernel<80, double, true> : nns::kernel<80, double, false>)<<<grid, C80::NTHREADS, C80::SMEM, s>>>(
            m, (int)p, (int)q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy, gate, vx, vt,
            DX, dldx, kdot, dws);
      } else {
        const int64_t nblk = ceil_div(m, nns::Cfg<64>::BM);
        const unsigned gy = (unsigned)ceil_div(q, 64);
        const int64_t per = std::max<int64_t>(1, capped(nns::Cfg<64>::PER_SM * 148) / gy);
        const dim3 grid((unsigned)std::min<int64_t>(nblk, per), gy);
        *nchunk_out = grid.x;
        if (kdot == 0 && nn_ws_enabled())
          return launch_nn_ws<64>(grid, s, m, p, q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz,
                                  Y, ldy, gate, vx, vt);
        (kdot > 0 ? nns::kernel<64, double, true> : nns::kernel<64, double, false>)<<<grid, nns::THREADS, nns::Cfg<64>::SMEM, s>>>(
            m, (int)p, (int)q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy, gate, vx, vt,
            DX, dldx, kdot, dws);
      }
    } else if (q <= 128) {
      const int64_t nblk = ceil_div(m, nns::Cfg<128>::BM);
      const unsigned grid = (unsigned)std::min<int64_t>(nblk, capped(nns::Cfg<128>::PER_SM * 148));
      *nchunk_out = grid;
      (kdot > 0 ? nns::kernel<128, double, true> : nns::kernel<128, double, false>)<<<grid, nns::THREADS, nns::Cfg<128>::SMEM, s>>>(
          m, (int)p, (int)q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy, gate, vx, vt,
          DX, dldx, kdot, dws);
    } else {
      const int64_t nblk = ceil_div(m, nns::Cfg<192>::BM);
      const unsigned grid = (unsigned)std::min<int64_t>(nblk, capped(nns::Cfg<192>::PER_SM * 148));
      *nchunk_out = grid;
      if (kdot == 0 && nn_ws_enabled())
        return launch_nn_ws<192>(dim3(grid), s, m, p, q, alpha, X, ldx, xcols, T, ldt, beta, Z,
                                 ldz, Y, ldy, gate, vx, vt);
      (kdot > 0 ? nns::kernel<192, double, true> : nns::kernel<192, double, false>)<<<grid, nns::THREADS, nns::Cfg<192>::SMEM, s>>>(
          m, (int)p, (int)q, alpha, X, ldx, xcols, T, ldt, beta, Z, ldz, Y, ldy, gate, vx, vt,
          DX, dldx, kdot, dws);
    }
    POD_CHECK_LAUNCH("nn streamed");
    return POD_OK;
  }
}

extern "C" size_t pod_gemm_nn_dots_ws_bytes(int64_t kdot) {
  return (size_t)std::max<int64_t>(kdot, 1) * 2 * 148 * sizeof(double);
}

extern "C" int pod_gemm_nn_dots(int64_t m, int64_t p, int64_t q, double alpha, const double* X,
                                int64_t ldx, const double* T, int64_t ldt, double* Y, int64_t ldy,
                                int64_t kdot, double* dots, void* ws, size_t ws_bytes,
                                const int32_t* gate, void* stream) {
  POD_REQUIRE(m >= 1 && p >= 1 && q >= 1 && ldx >= m && ldy >= m,
              "pod_gemm_nn_dots: bad shape");
  POD_REQUIRE(kdot >= 1 && kdot <= p && kdot <= q, "pod_gemm_nn_dots: need 1 <= kdot <= min(p, q)");
  POD_REQUIRE(gate == nullptr, "pod_gemm_nn_dots: not gateable");
  POD_REQUIRE(ws_bytes >= pod_gemm_nn_dots_ws_bytes(kdot), "pod_gemm_nn_dots: workspace too small");
  const char* y0 = (const char*)Y;
  const char* y1 = (const char*)(Y + (q - 1) * ldy + m);
  const char* x0 = (const char*)X;
  const char* x1 = (const char*)(X + (p - 1) * ldx + m);
  POD_REQUIRE(!(x0 < y1 && y0 < x1), "pod_gemm_nn_dots: Y must not alias X");
  int st = ensure_attrs();
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nchunk = 0;
  st = nn_streamed(m, p, q, alpha, X, ldx, nullptr, T, ldt, 0.0, nullptr, 1, Y, ldy, gate, s, X, ldx,
                   (int)kdot, (double*)ws, &nchunk);
  if (st) return st;
  POD_REQUIRE(nchunk <= 2 * 148, "pod_gemm_nn_dots: grid larger than the workspace");
  nns::dots_final_kernel<<<(unsigned)ceil_div(kdot, 128), 128, 0, s>>>((const double*)ws,
                                                                     (int)nchunk, (int)kdot, dots);
  POD_CHECK_LAUNCH("nn dots final");
  return POD_OK;
}

// T-resident NN with the Gram epilogue: q <= 64 output columns, p >= q,
// T in shared memory at 2 CTAs per SM
extern "C" int pod_gemm_nn_gram_ok(int64_t p, int64_t q) {
  return (q >= 1 && q <= 64 && p >= q && nnp::smem_bytes((int)p, 64) <= 110 * 1024) ? 1 : 0;
}

static int64_t nn_gram_grid(int64_t m) {
  return std::min<int64_t>(ceil_div(m, nnp::BM), capped(2 * 148));
}

extern "C" size_t pod_gemm_nn_gram_ws_bytes(int64_t m, int64_t q) {
  if (m <= 0 || q <= 0) return 256;
  return (size_t)(2 * 148) * q * q * sizeof(double);  // >= any capped grid
}

extern "C" int pod_gemm_nn_gram(int64_t m, int64_t p, int64_t q, double alpha, const double* X,
                                int64_t ldx, const double* T, int64_t ldt, double beta,
                                const double* Z, int64_t ldz, double* Y, int64_t ldy, double* G,
                                int64_t ldg, void* ws, size_t ws_bytes, const int32_t* gate,
                                void* stream) {
  POD_REQUIRE(m >= 1 && pod_gemm_nn_gram_ok(p, q), "pod_gemm_nn_gram: shape not supported");
  POD_REQUIRE(ldy >= m && ldx >= m && ldg >= q, "pod_gemm_nn_gram: bad leading dimension");
  POD_REQUIRE(beta == 0.0 || Z != nullptr, "pod_gemm_nn_gram: beta != 0 needs Z");
  POD_REQUIRE(ws_bytes >= pod_gemm_nn_gram_ws_bytes(m, q), "pod_gemm_nn_gram: workspace too small");
  int st = ensure_attrs();
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = nnp::smem_bytes((int)p, 64);
  const int vec16 = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && (ldx % 2 == 0);
  const unsigned grid = (unsigned)nn_gram_grid(m);
  nnp::kernel<64, true><<<grid, nnp::THREADS, bytes, s>>>(m, (int)p, (int)q, alpha, X, ldx, nullptr,
                                                         T, ldt, beta, Z, ldz, Y, ldy, gate, vec16,
                                                         (double*)ws);
  POD_CHECK_LAUNCH("nn gram");
  const int64_t tot = q * q;
  const int blocks = (int)std::min<int64_t>(ceil_div(tot, 8), 16 * 148);
  tn::reduce_kernel<<<blocks, 256, 0, s>>>((int)grid, (int)q, (int)q, 1.0, (const double*)ws, G,
                                           ldg, gate, 1);
  POD_CHECK_LAUNCH("nn gram reduce");
  return POD_OK;
}

extern "C" int pod_set_grid_cap(int ctas) {
  POD_REQUIRE(ctas >= 0, "pod_set_grid_cap: negative cap");
  pod::g_grid_cap = ctas;
  return POD_OK;
}
