// Sums in numpy's exact order, so the sampled index sets equal the
// reference's BY CONSTRUCTION (north_star: "sampled index sets bit-exact").
//
// The reference draws through three numpy reductions whose rounding decides
// every CDF breakpoint:
//   * column norms  np.einsum("ij,ij->j", a, a)  (isma.py:260, sampling.py:136)
//     numpy 2.3's einsum inner loop for a contiguous column with a reduced
//     output (einsum_sumprod.c.src, sum_of_products_contig_contig_outstride0_two)
//     is compiled for the x86-64 baseline (SSE2: 2 double lanes, no FMA):
//     lane l in {0,1} accumulates, per block of 8 rows starting at i,
//       acc_l = x[i+l]^2 + (x[i+2+l]^2 + (x[i+4+l]^2 + (x[i+6+l]^2 + acc_l)))
//     with every product and sum rounded (mul, then add), then the m % 8 tail
//     pairwise-by-lane in ascending order, then acc_0 + acc_1.  Verified
//     bit-for-bit against einsum for m = 7 ... 262144 (tools/einsum_order.py).
//   * totals        ndarray.sum() = numpy's pairwise summation
//     (loops_utils.h.src pairwise_sum: blocks <= 128 with 8 accumulators,
//     split at n/2 rounded down to a multiple of 8)  (sampling.py:47,62)
//   * the CDF       np.cumsum = a sequential running sum  (sampling.py:214)
// The kernels below perform exactly those operations in exactly that order
// (IEEE double, no contraction: __dmul_rn / __dadd_rn / correctly rounded
// division), so norms, weights and CDF are bit-identical to numpy's and
// searchsorted(side="right") on the same uniforms returns the same indices.
#include "common.cuh"

namespace pod {

// ------------------------------------------------ einsum-order norms ------
__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }
__device__ __forceinline__ double addr(double a, double b) { return __dadd_rn(a, b); }

// one 8-row block into the two lane accumulators (x0..x7 = rows i..i+7)
__device__ __forceinline__ void einsum_block(double& a0, double& a1, double x0, double x1,
                                             double x2, double x3, double x4, double x5,
                                             double x6, double x7) {
  a0 = addr(sq(x6), a0);
  a1 = addr(sq(x7), a1);
  a0 = addr(sq(x4), a0);
  a1 = addr(sq(x5), a1);
  a0 = addr(sq(x2), a0);
  a1 = addr(sq(x3), a1);
  a0 = addr(sq(x0), a0);
  a1 = addr(sq(x1), a1);
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;"
                 " selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_addr(mb)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(mb)) : "memory");
}

// Squares of one 16-byte piece of a staged column chunk (2 rows for f64, 4
// for f32) into the lane-split square buffer: for row r = 8b + 2q + l the
// square lands in lane l's run at block b, slot 3 - q (the chain adds rows
// 6, 4, 2, 0 of a block, + l, in that order).
template <typename T>
__device__ __forceinline__ void square_piece(const unsigned char* xsrc, int piece, double* pl0,
                                             double* pl1) {
  if constexpr (sizeof(T) == 8) {
    const double2 v = reinterpret_cast<const double2*>(xsrc)[piece];
    const int q = piece & 3, b = piece >> 2;  // rows 2 piece, 2 piece + 1
    pl0[4 * b + 3 - q] = sq(v.x);
    pl1[4 * b + 3 - q] = sq(v.y);
  } else {
    const float4 v = reinterpret_cast<const float4*>(xsrc)[piece];
    const int q = (2 * piece) & 3, b = piece >> 1;  // rows 4 piece .. 4 piece + 3
    pl0[4 * b + 3 - q] = sq((double)v.x);
    pl1[4 * b + 3 - q] = sq((double)v.y);
    pl0[4 * b + 2 - q] = sq((double)v.z);
    pl1[4 * b + 2 - q] = sq((double)v.w);
  }
}

//: einsum-norm CTA: warp 0 runs the chains, warps 1..EIN_PW stage and square
constexpr int EIN_COLS = 16;
constexpr int EIN_PW = 4;
constexpr int EIN_THREADS = 32 * (1 + EIN_PW);

// numpy's einsum order over rows [0, m8) (m8 multiple of 8) of up to 16
// columns per CTA.  Warps 1..4 (producers) keep a ring of column chunks in
// flight with cp.async.bulk (completing on full[s]), square each landed
// chunk into a lane-split double buffer P (one square per element, rounded:
// DMUL) and refill the ring.  Warp 0 (chains): threads 2c and 2c + 1 run
// einsum's two lanes of column c and only ADD the ready squares -- 4
// dependent DADDs per 8-row block and lane, 8 cycles each on this B200
// (tools/dadd_probe.cu); the squares, loads and copies sit on the other warp
// (another SM sub-partition), so the chain runs at the DADD latency.  The
// lane state (acc_0, acc_1) enters from state_in (the rows above: the
// row-sharded pass hands it from rank to rank) or starts at 0; `last` adds
// the m % 8 tail and writes the norm, otherwise the state is written out.
template <typename T>
__global__ void __launch_bounds__(EIN_THREADS) einsum_norms_bulk_kernel(
    const T* __restrict__ A, int64_t m, int64_t n, int64_t lda, int cpb, int ce, int nst,
    const double* __restrict__ state_in, double* __restrict__ state_out, int last,
    double* __restrict__ out, int* __restrict__ nonfinite) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
  // layout: mbarriers | X ring [nst][cpb][xpitch] | P [2][cpb][2 lanes][lrun]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* pfull = full + nst;
  uint64_t* pempty = pfull + 2;
  unsigned char* xbuf = sm + 16 * ((8 * (nst + 4) + 15) / 16);
  const int xpitch = ce * (int)sizeof(T) + 16;
  const int nbmax = ce / 8;
  // lane runs start 16 B apart and columns 32 B apart (mod 128): a chain
  // warp's 16-byte reads hit distinct banks
  const int lrun = nbmax * 4 + 2;           // doubles per lane run
  const int ppitch = 2 * lrun;              // doubles per column
  double* pbuf = reinterpret_cast<double*>(xbuf + (size_t)nst * cpb * xpitch);
  const int64_t m8 = m & ~(int64_t)7;
  const int64_t nchunks = (m8 + ce - 1) / ce;
  const int ncols = (int)imin64(cpb, n - (int64_t)blockIdx.x * cpb);
  const int64_t j0 = (int64_t)blockIdx.x * cpb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&pfull[s])),
                   "r"(32 * EIN_PW));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(smem_addr(&pempty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= 1) {  // ------------------------------------ producers / squarers
    const int pt = threadIdx.x - 32;  // 0 .. 32 EIN_PW - 1
    auto issue = [&](int64_t c, int s) {  // by warp 1
      const int64_t r0 = c * ce;
      const uint32_t bytes = (uint32_t)((imin64(m8, r0 + ce) - r0) * (int64_t)sizeof(T));
      if (t == 0)
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;"
                     ::"r"(smem_addr(&full[s])), "r"(bytes * (uint32_t)ncols) : "memory");
      if (t < ncols)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_addr(xbuf + (size_t)(s * cpb + t) * xpitch)),
            "l"(A + (j0 + t) * lda + r0), "r"(bytes), "r"(smem_addr(&full[s]))
            : "memory");
    };
    const int npro = (int)imin64(nst, nchunks);
    if (warp == 1)
      for (int c = 0; c < npro; ++c) issue(c, c);
    int s = 0;
    uint32_t fpar = 0, epar = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int pb = (int)(c & 1);
      mbar_wait_parity(&full[s], fpar);
      if (c >= 2) mbar_wait_parity(&pempty[pb], epar);  // chains done with chunk c - 2
      const int rows = (int)(imin64(m8, c * ce + ce) - c * ce);
      const int pieces = rows * (int)sizeof(T) / 16;
      for (int cs = 0; cs < ncols; ++cs) {
        const unsigned char* xs = xbuf + (size_t)(s * cpb + cs) * xpitch;
        double* pl0 = pbuf + ((size_t)pb * cpb + cs) * ppitch;
        for (int pc = pt; pc < pieces; pc += 32 * EIN_PW) square_piece<T>(xs, pc, pl0, pl0 + lrun);
      }
      // every producer has read X[s]: warp 1 refills it
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EIN_PW) : "memory");
      if (warp == 1 && c + nst < nchunks) issue(c + nst, s);
      mbar_arrive(&pfull[pb]);
      if (pb == 1) epar ^= (c >= 2) ? 1u : 0u;
      if (++s == nst) { s = 0; fpar ^= 1u; }
    }
    return;
  }
  // ------------------------------------------------------------ chains
  const int cs = t >> 1, lane = t & 1;
  const int64_t j = j0 + cs;
  const bool active = cs < ncols;
  double acc = 0.0;
  if (state_in && active) acc = state_in[2 * j + lane];
  uint32_t ppar0 = 0, ppar1 = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int pb = (int)(c & 1);
    mbar_wait_parity(&pfull[pb], pb ? ppar1 : ppar0);
    if (pb) ppar1 ^= 1u; else ppar0 ^= 1u;
    if (active) {
      const int nb = (int)(imin64(m8, c * ce + ce) - c * ce) / 8;
      const double2* p = reinterpret_cast<const double2*>(
          pbuf + ((size_t)pb * cpb + cs) * ppitch + (size_t)lane * lrun);
      // two blocks per step, the next two prefetched (no register moves)
      double2 u0 = p[0], u1 = p[1], v0 = p[2], v1 = p[3];
      for (int b = 0; b < nb; b += 2) {
        const double2 w0 = p[2 * b + 4], w1 = p[2 * b + 5], z0 = p[2 * b + 6], z1 = p[2 * b + 7];
        acc = addr(u0.x, acc);
        acc = addr(u0.y, acc);
        acc = addr(u1.x, acc);
        acc = addr(u1.y, acc);
        if (b + 1 < nb) {
          acc = addr(v0.x, acc);
          acc = addr(v0.y, acc);
          acc = addr(v1.x, acc);
          acc = addr(v1.y, acc);
        }
        u0 = w0; u1 = w1; v0 = z0; v1 = z1;
      }
    }
    mbar_arrive(&pempty[pb]);
  }
  const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
  if (!active || lane) return;
  const T* col = A + j * lda;
  double a0 = acc, a1 = other;
  if (!last) {
    state_out[2 * j] = a0;
    state_out[2 * j + 1] = a1;
    if (!(isfinite(a0) && isfinite(a1))) {  // a non-finite entry in this segment?
      int bad = 0;
      for (int64_t i = 0; i < m; ++i) bad |= !isfinite((double)col[i]);
      if (bad) atomicOr(nonfinite, 1);
    }
    return;
  }
  for (int64_t i = m8; i < m; i += 2) {  // einsum's tail: lane pairs, zero filled
    a0 = addr(sq((double)col[i]), a0);
    a1 = addr(sq(i + 1 < m ? (double)col[i + 1] : 0.0), a1);
  }
  const double r = addr(a0, a1);
  out[j] = r;
  if (!isfinite(r)) {  // non-finite entry, or overflow of finite ones
    int bad = 0;
    for (int64_t i = 0; i < m; ++i) bad |= !isfinite((double)col[i]);
    if (bad) atomicOr(nonfinite, 1);
  }
}

// Many columns (config 3: 20000): HBM bounds the pass, so one thread runs
// both einsum lanes of its column (32 columns per warp-CTA, several CTAs per
// SM) on chunks staged by cp.async.bulk; measured 26 ms = 6.1 TB/s at
// 1M x 20000 fp64 (the producer/chain CTA above: 36-63 ms there).
template <typename T>
__global__ void __launch_bounds__(32) einsum_norms_wide_kernel(
    const T* __restrict__ A, int64_t m, int64_t n, int64_t lda, int ce, int nst,
    const double* __restrict__ state_in, double* __restrict__ state_out, int last,
    double* __restrict__ out, int* __restrict__ nonfinite) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int t = threadIdx.x;
  const int64_t j = (int64_t)blockIdx.x * 32 + t;
  const bool active = j < n;
  const int pitch = ce * (int)sizeof(T) + 16;
  uint64_t* mb = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 16 * ((nst * 8 + 15) / 16);
  const int64_t m8 = m & ~(int64_t)7;
  const int64_t nchunks = (m8 + ce - 1) / ce;
  const int ncols = (int)imin64(32, n - (int64_t)blockIdx.x * 32);
  if (t == 0) {
    for (int s = 0; s < nst; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mb[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const T* col = A + j * lda;
  auto issue = [&](int64_t c, int s) {
    const int64_t r0 = c * ce;
    const uint32_t bytes = (uint32_t)((imin64(m8, r0 + ce) - r0) * (int64_t)sizeof(T));
    if (t == 0)
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;"
                   ::"r"(smem_addr(&mb[s])), "r"(bytes * (uint32_t)ncols) : "memory");
    if (active)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_addr(buf + (size_t)(s * 32 + t) * pitch)), "l"(col + r0), "r"(bytes),
          "r"(smem_addr(&mb[s]))
          : "memory");
  };
  for (int c = 0; c < (int)imin64(nst, nchunks); ++c) issue(c, c);
  double a0 = 0.0, a1 = 0.0;
  if (state_in && active) { a0 = state_in[2 * j]; a1 = state_in[2 * j + 1]; }
  int s = 0;
  uint32_t parity = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    mbar_wait_parity(&mb[s], parity);
    if (active) {
      const int nb = (int)(imin64(m8, c * ce + ce) - c * ce) / 8;
      const unsigned char* p = buf + (size_t)(s * 32 + t) * pitch;
#pragma unroll 4
      for (int b = 0; b < nb; ++b) {
        double x[8];
        if constexpr (sizeof(T) == 8) {
          const double2* v = reinterpret_cast<const double2*>(p) + 4 * b;
          const double2 q0 = v[0], q1 = v[1], q2 = v[2], q3 = v[3];
          x[0] = q0.x; x[1] = q0.y; x[2] = q1.x; x[3] = q1.y;
          x[4] = q2.x; x[5] = q2.y; x[6] = q3.x; x[7] = q3.y;
        } else {
          const float4* v = reinterpret_cast<const float4*>(p) + 2 * b;
          const float4 q0 = v[0], q1 = v[1];
          x[0] = q0.x; x[1] = q0.y; x[2] = q0.z; x[3] = q0.w;
          x[4] = q1.x; x[5] = q1.y; x[6] = q1.z; x[7] = q1.w;
        }
        einsum_block(a0, a1, x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
      }
    }
    __syncwarp();
    if (c + nst < nchunks) issue(c + nst, s);
    if (++s == nst) { s = 0; parity ^= 1u; }
  }
  if (!active) return;
  if (!last) {
    state_out[2 * j] = a0;
    state_out[2 * j + 1] = a1;
    if (!(isfinite(a0) && isfinite(a1))) {
      int bad = 0;
      for (int64_t i = 0; i < m; ++i) bad |= !isfinite((double)col[i]);
      if (bad) atomicOr(nonfinite, 1);
    }
    return;
  }
  for (int64_t i = m8; i < m; i += 2) {
    a0 = addr(sq((double)col[i]), a0);
    a1 = addr(sq(i + 1 < m ? (double)col[i + 1] : 0.0), a1);
  }
  const double r = addr(a0, a1);
  out[j] = r;
  if (!isfinite(r)) {
    int bad = 0;
    for (int64_t i = 0; i < m; ++i) bad |= !isfinite((double)col[i]);
    if (bad) atomicOr(nonfinite, 1);
  }
}

// Same order with plain loads (operands not 16-byte aligned for the bulk
// copies, or tiny m): one thread per column.
template <typename T>
__global__ void __launch_bounds__(128) einsum_norms_plain_kernel(
    const T* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ state_in,
    double* __restrict__ state_out, int last, double* __restrict__ out, int* __restrict__ nonfinite) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const T* col = A + j * lda;
  double a0 = 0.0, a1 = 0.0;
  if (state_in) { a0 = state_in[2 * j]; a1 = state_in[2 * j + 1]; }
  const int64_t m8 = m & ~(int64_t)7;
  for (int64_t i = 0; i < m8; i += 8)
    einsum_block(a0, a1, col[i], col[i + 1], col[i + 2], col[i + 3], col[i + 4], col[i + 5],
                 col[i + 6], col[i + 7]);
  if (!last) {
    state_out[2 * j] = a0;
    state_out[2 * j + 1] = a1;
    if (!(isfinite(a0) && isfinite(a1))) {
      int bad = 0;
      for (int64_t i = 0; i < m; ++i) bad |= !isfinite((double)col[i]);
      if (bad) atomicOr(nonfinite, 1);
    }
    return;
  }
  for (int64_t i = m8; i < m; i += 2) {
    a0 = addr(sq((double)col[i]), a0);
    a1 = addr(sq(i + 1 < m ? (double)col[i + 1] : 0.0), a1);
  }
  const double s = addr(a0, a1);
  out[j] = s;
  if (!isfinite(s)) {
    int bad = 0;
    for (int64_t i = 0; i < m; ++i) bad |= !isfinite((double)col[i]);
    if (bad) atomicOr(nonfinite, 1);
  }
}

// ------------------------------------------------ numpy pairwise sum ------
// numpy's pairwise_sum (PW_BLOCKSIZE 128, 8 accumulators per leaf).
__device__ double pw_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = addr(res, a[i]);
    return res;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = addr(r0, a[i]); r1 = addr(r1, a[i + 1]); r2 = addr(r2, a[i + 2]);
    r3 = addr(r3, a[i + 3]); r4 = addr(r4, a[i + 4]); r5 = addr(r5, a[i + 5]);
    r6 = addr(r6, a[i + 6]); r7 = addr(r7, a[i + 7]);
  }
  double res = addr(addr(addr(r0, r1), addr(r2, r3)), addr(addr(r4, r5), addr(r6, r7)));
  for (; i < n; ++i) res = addr(res, a[i]);
  return res;
}

// The pairwise tree of an n-element sum, built breadth first by the whole
// block and evaluated bottom up (a node = a leaf block <= 128 or the sum of
// its two halves, split at n/2 rounded down to a multiple of 8).  Node arrays
// live in the caller's workspace (capacity 2 (n / 64 + 2)).
struct PwTree {
  int64_t* lo;
  int* len;
  int* child;
  double* val;
};

__device__ int64_t xd_excl_scan(int64_t v, int64_t* sh, int64_t* total);

__device__ double np_sum_block(const double* a, int64_t n, PwTree tr, int64_t* shscan) {
  __shared__ int lvl[72];
  __shared__ double root;
  const int t = threadIdx.x;
  if (n <= 0) return 0.0;
  if (t == 0) {
    tr.lo[0] = 0;
    tr.len[0] = (int)n;
    lvl[0] = 0;
    lvl[1] = 1;
  }
  __syncthreads();
  int d = 0;
  for (;; ++d) {  // level d: nodes [lvl[d], lvl[d + 1])
    const int a0 = lvl[d], b0 = lvl[d + 1];
    if (a0 == b0) break;
    int64_t carry = 0;
    for (int base = a0; base < b0; base += blockDim.x) {
      const int i = base + t;
      const bool internal = i < b0 && tr.len[i] > 128;
      int64_t tot = 0;
      const int64_t ex = xd_excl_scan(internal ? 1 : 0, shscan, &tot);
      if (i < b0) {
        if (internal) {
          const int c = b0 + 2 * (int)(carry + ex);
          const int nn = tr.len[i];
          int n2 = nn / 2;
          n2 -= n2 % 8;
          tr.child[i] = c;
          tr.lo[c] = tr.lo[i];
          tr.len[c] = n2;
          tr.lo[c + 1] = tr.lo[i] + n2;
          tr.len[c + 1] = nn - n2;
        } else {
          tr.child[i] = -1;
        }
      }
      carry += tot;
    }
    if (t == 0) lvl[d + 2] = b0 + 2 * (int)carry;
    __syncthreads();
  }
  for (int dd = d - 1; dd >= 0; --dd) {
    for (int i = lvl[dd] + t; i < lvl[dd + 1]; i += blockDim.x) {
      const int c = tr.child[i];
      tr.val[i] = (c < 0) ? pw_leaf(a + tr.lo[i], tr.len[i]) : addr(tr.val[c], tr.val[c + 1]);
    }
    __syncthreads();
  }
  if (t == 0) root = addr(0.0, tr.val[0]);  // add.reduce starts from the identity
  __syncthreads();
  const double r = root;
  __syncthreads();
  return r;
}

// ------------------------------------------------------ the exact draw ----
constexpr int XD_THREADS = 1024;
constexpr int XD_CH = 2048;  // cumsum staging chunk (doubles)

__device__ int64_t xd_excl_scan(int64_t v, int64_t* sh, int64_t* total) {
  sh[threadIdx.x] = v;
  __syncthreads();
  // Hillis-Steele over 1024 entries (integers: order-free)
  for (int o = 1; o < XD_THREADS; o <<= 1) {
    const int64_t x = (threadIdx.x >= o) ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += x;
    __syncthreads();
  }
  const int64_t incl = sh[threadIdx.x];
  *total = sh[XD_THREADS - 1];
  __syncthreads();
  return incl - v;
}

// Modes as pod_draw: 0 l2n over live columns (Distribution.from_weights of
// the raw norms, sampling.py:55-65 then 34-53), 1 uniform over live columns
// (sampling.py:150-155), 2 the given weights over all n (a Distribution's
// weights, used as they are, sampling.py:214), 3 ort: raw squared residuals
// normalised like l2n (sampling.py:180-187), or uniform when their pairwise
// total is <= thr (isma.py:216-220).  Then cumsum, the pin, searchsorted
// (side="right"), unique+counts, and retirement from the live set.
__global__ void __launch_bounds__(XD_THREADS) draw_exact_kernel(
    int mode, const double* __restrict__ raw, uint8_t* __restrict__ live, int64_t n,
    const double* __restrict__ uni, int64_t c, int32_t* __restrict__ idx_out,
    int64_t* __restrict__ cnt_out, int64_t cap, double* __restrict__ w,
    double* __restrict__ cum, int32_t* __restrict__ cidx, int32_t* __restrict__ counts,
    PwTree tree, int64_t* __restrict__ info, double thr, double* __restrict__ p_out) {
  __shared__ int64_t shi[XD_THREADS];
  const int t = threadIdx.x;
  const int64_t chunk = (n + XD_THREADS - 1) / XD_THREADS;
  const int64_t j0 = min(n, t * chunk), j1 = min(n, j0 + chunk);
  // mode 4 (row draw, isma.py:168-173): from_weights over ALL positions
  // (normalised like l2n), no retirement, p_out = the drawn positions' weights
  const bool rows = (mode == 4);
  if (rows) mode = 0;
  const bool all = rows || (mode == 2);
  // compaction of the candidate set S (ascending, like setdiff1d's output)
  int64_t loc = 0;
  for (int64_t j = j0; j < j1; ++j) loc += all ? 1 : (live[j] != 0);
  int64_t s = 0;
  int64_t p = xd_excl_scan(loc, shi, &s);
  if (s == 0) {
    for (int64_t q = t; q < cap; q += XD_THREADS) idx_out[q] = -1;
    if (t == 0) { info[0] = 0; info[1] = 0; info[2] = 1; }  // status 1: empty S
    return;
  }
  for (int64_t j = j0; j < j1; ++j) {
    if (all || live[j]) {
      cidx[p] = (int32_t)j;
      w[p] = (mode == 1) ? 0.0 : raw[j];
      ++p;
    }
  }
  __syncthreads();
  if (mode == 3) {  // residual_distribution's degeneracy test on the pairwise total
    const double tot = np_sum_block(w, s, tree, shi);
    if (tot <= thr) mode = 1;
  }
  if (mode == 1) {  // np.full(s, 1.0 / s), then the __post_init__ renormalisation
    const double v = 1.0 / (double)s;
    for (int64_t q = t; q < s; q += XD_THREADS) w[q] = v;
    __syncthreads();
    const double tot = np_sum_block(w, s, tree, shi);
    for (int64_t q = t; q < s; q += XD_THREADS) w[q] = w[q] / tot;
  } else if (mode == 0 || mode == 3) {
    const double tot = np_sum_block(w, s, tree, shi);  // from_weights: raw.sum()
    if (!(tot > 0.0)) {
      for (int64_t q = t; q < cap; q += XD_THREADS) idx_out[q] = -1;
      if (t == 0) { info[0] = 0; info[1] = s; info[2] = 2; }  // status 2: degenerate
      return;
    }
    for (int64_t q = t; q < s; q += XD_THREADS) w[q] = w[q] / tot;
    __syncthreads();
    const double tot2 = np_sum_block(w, s, tree, shi);  // __post_init__: w.sum()
    for (int64_t q = t; q < s; q += XD_THREADS) w[q] = w[q] / tot2;
  }
  __syncthreads();
  // the last positive weight (sampling.py:216)
  {
    int64_t lastl = -1;
    for (int64_t q = t; q < s; q += XD_THREADS)
      if (w[q] != 0.0) lastl = q;
    shi[t] = lastl;
    __syncthreads();
    for (int o = XD_THREADS / 2; o > 0; o >>= 1) {
      if (t < o) shi[t] = imax64(shi[t], shi[t + o]);
      __syncthreads();
    }
  }
  const int64_t last = shi[0];
  __syncthreads();
  // np.cumsum: a sequential running sum on thread 0, fed from shared memory
  // chunks that the other threads stage one chunk ahead (the chain's cost
  // is then the DADD latency per element, not a global load per element)
  {
    __shared__ double stage[2][XD_CH];
    const int64_t nch = (s + XD_CH - 1) / XD_CH;
    for (int64_t q = t; q < imin64(s, XD_CH); q += XD_THREADS) stage[0][q] = w[q];
    __syncthreads();
    double run = -0.0;  // -0 + x == x: add.accumulate's copy of the first element
    for (int64_t k = 0; k < nch; ++k) {
      const int64_t base = k * XD_CH, len = imin64(XD_CH, s - base);
      if (t > 0 && k + 1 < nch) {
        const int64_t nb = base + XD_CH, nlen = imin64(XD_CH, s - nb);
        for (int64_t q = t - 1; q < nlen; q += XD_THREADS - 1) stage[(k + 1) & 1][q] = w[nb + q];
      }
      if (t == 0) {
        const double* b = stage[k & 1];
        int64_t q = 0;
        for (; q + 8 <= len; q += 8) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = b[q + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            run = addr(run, x[u]);
            cum[base + q + u] = run;
          }
        }
        for (; q < len; ++q) {
          run = addr(run, b[q]);
          cum[base + q] = run;
        }
      }
      __syncthreads();
    }
  }
  for (int64_t q = imax64(last, 0) + t; q < s; q += XD_THREADS)
    if (last >= 0) cum[q] = 1.0;  // the pin (sampling.py:215-219)
  for (int64_t q = t; q < s; q += XD_THREADS) counts[q] = 0;
  __syncthreads();
  // searchsorted(cum, u, side="right"): first q with cum[q] > u (cum[s-1] == 1 > u)
  for (int64_t d = t; d < c; d += XD_THREADS) {
    const double u = uni[d];
    int64_t lo = 0, hi = s - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cum[mid] > u) hi = mid; else lo = mid + 1;
    }
    atomicAdd(&counts[lo], 1);
  }
  __syncthreads();
  // np.unique(..., return_counts=True): ascending distinct indices, retired from S
  const int64_t q0 = min(s, t * ((s + XD_THREADS - 1) / XD_THREADS));
  const int64_t q1 = min(s, q0 + (s + XD_THREADS - 1) / XD_THREADS);
  int64_t nd = 0;
  for (int64_t q = q0; q < q1; ++q) nd += counts[q] > 0;
  int64_t g = 0;
  int64_t pos = xd_excl_scan(nd, shi, &g);
  for (int64_t q = q0; q < q1; ++q) {
    if (counts[q] > 0) {
      const int32_t jj = cidx[q];
      idx_out[pos] = jj;
      cnt_out[pos] = counts[q];
      if (p_out) p_out[pos] = w[q];  // Distribution.weight_of (sampling.py:226)
      ++pos;
      if (!all) live[jj] = 0;
    }
  }
  for (int64_t q = g + t; q < cap; q += XD_THREADS) idx_out[q] = -1;  // zero-column padding
  if (t == 0) { info[0] = g; info[1] = s - g; info[2] = 0; }
}

}  // namespace pod

using namespace pod;

namespace {
int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename T>
int launch_einsum_norms(const T* A, int64_t m, int64_t n, int64_t lda, const double* state_in,
                        double* state_out, int last, double* out, int* nonfinite,
                        cudaStream_t s) {
  const bool aligned = (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                       ((lda * (int64_t)sizeof(T)) % 16 == 0);
  if (!aligned || m < 64) {
    einsum_norms_plain_kernel<T><<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(
        A, m, n, lda, state_in, state_out, last, out, nonfinite);
    POD_CHECK_LAUNCH("einsum norms (plain)");
    return POD_OK;
  }
  const int sms = sm_count();
  if (n > 2 * EIN_COLS * sms) {
    // many columns: HBM-bound; one thread per column, ~200 KB of stages per SM
    const int64_t ctas = ceil_div(n, 32);
    const int per_sm = (int)imin64(8, ceil_div(ctas, sms));  // one wave
    const size_t budget = (size_t)(216 * 1024) / per_sm;
    int ce = 2048 / (int)sizeof(T);
    while (ce > 64 && (size_t)32 * (ce * sizeof(T) + 16) * 3 > budget) ce /= 2;
    const int pitch = ce * (int)sizeof(T) + 16;
    const int nst = (int)imax64(2, imin64(16, (int64_t)((budget - 256) / ((size_t)32 * pitch))));
    const size_t smem = 16 * ((nst * 8 + 15) / 16) + (size_t)nst * 32 * pitch;
    auto kern = einsum_norms_wide_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "einsum norms smem attribute");
    kern<<<(unsigned)ctas, 32, smem, s>>>(A, m, n, lda, ce, nst, state_in, state_out, last, out,
                                          nonfinite);
    POD_CHECK_LAUNCH("einsum norms (wide)");
    return POD_OK;
  }
  // few columns (config 2: 2000): the DADD chains bound the pass; up to 16
  // columns per CTA (a chain warp + four producer warps), two CTAs per SM
  const int cpb = (int)imax64(1, imin64(EIN_COLS, ceil_div(n, 2 * sms)));
  const int64_t ctas = ceil_div(n, cpb);
  const int per_sm = (int)imin64(2, ceil_div(ctas, sms));
  const size_t budget = (size_t)(216 * 1024) / per_sm;
  auto need = [&](int ce_, int nst_) {
    const int nbm = ce_ / 8, lrun = nbm * 4 + 2, ppitch = 2 * lrun;
    return (size_t)16 * ((8 * (nst_ + 4) + 15) / 16) +
           (size_t)nst_ * cpb * (ce_ * sizeof(T) + 16) + (size_t)2 * cpb * ppitch * 8 + 256;
  };
  int ce = 2048 / (int)sizeof(T);  // 2 KB per column and stage
  while (ce > 64 && need(ce, 3) > budget) ce /= 2;
  int nst = 3;
  while (nst < 12 && need(ce, nst + 1) <= budget) ++nst;
  const size_t smem = need(ce, nst);
  auto kern = einsum_norms_bulk_kernel<T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "einsum norms smem attribute");
  kern<<<(unsigned)ctas, EIN_THREADS, smem, s>>>(A, m, n, lda, cpb, ce, nst, state_in, state_out,
                                                 last, out, nonfinite);
  POD_CHECK_LAUNCH("einsum norms (bulk)");
  return POD_OK;
}
}  // namespace

extern "C" int pod_colnorms2_chain(int atype, const void* A, int64_t m, int64_t n, int64_t lda,
                                   const double* state_in, double* state_out, int last,
                                   double* norms2, int32_t* nonfinite, void* stream) {
  POD_REQUIRE(atype == POD_F64 || atype == POD_F32, "pod_colnorms2_chain: bad operand type");
  POD_REQUIRE(m > 0 && n > 0 && lda >= m, "pod_colnorms2_chain: bad shape m=%lld n=%lld lda=%lld",
              (long long)m, (long long)n, (long long)lda);
  POD_REQUIRE(last || (m % 8 == 0 && state_out != nullptr),
              "pod_colnorms2_chain: a non-final row segment needs m %% 8 == 0 and state_out");
  POD_REQUIRE(!last || norms2 != nullptr, "pod_colnorms2_chain: norms2 required");
  cudaStream_t s = (cudaStream_t)stream;
  if (atype == POD_F64)
    return launch_einsum_norms((const double*)A, m, n, lda, state_in, state_out, last, norms2,
                               nonfinite, s);
  return launch_einsum_norms((const float*)A, m, n, lda, state_in, state_out, last, norms2,
                             nonfinite, s);
}

extern "C" int pod_colnorms2(int atype, const void* A, int64_t m, int64_t n, int64_t lda,
                             double* norms2, int32_t* nonfinite, void* stream) {
  POD_REQUIRE(m > 0 && n > 0 && lda >= m, "pod_colnorms2: bad shape m=%lld n=%lld lda=%lld",
              (long long)m, (long long)n, (long long)lda);
  cudaError_t e = cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "colnorms memset");
  return pod_colnorms2_chain(atype, A, m, n, lda, nullptr, nullptr, 1, norms2, nonfinite, stream);
}

extern "C" int pod_colnorms2_f64(const double* A, int64_t m, int64_t n, int64_t lda,
                                 double* norms2, int32_t* nonfinite, void* stream) {
  return pod_colnorms2(POD_F64, A, m, n, lda, norms2, nonfinite, stream);
}

extern "C" size_t pod_draw_exact_ws_bytes(int64_t n) {
  const int64_t nodes = 2 * (n / 64 + 2);
  return (size_t)n * (2 * sizeof(double) + 2 * sizeof(int32_t)) +
         (size_t)nodes * (sizeof(int64_t) + 2 * sizeof(int) + sizeof(double)) + 256;
}

extern "C" int pod_draw_exact(int mode, const double* weights, uint8_t* live, int64_t n,
                              const double* uniforms, int64_t c, int32_t* idx_out,
                              int64_t* cnt_out, int64_t cap, void* ws, size_t ws_bytes,
                              int64_t* info, double thr, double* p_out, void* stream) {
  POD_REQUIRE(mode >= 0 && mode <= 4, "pod_draw_exact: bad mode %d", mode);
  POD_REQUIRE(p_out == nullptr || mode == 4, "pod_draw_exact: p_out needs mode 4");
  POD_REQUIRE(n > 0 && n < (int64_t)INT32_MAX, "pod_draw_exact: bad n");
  POD_REQUIRE(c >= 1, "sample count must be >= 1");
  POD_REQUIRE(ws_bytes >= pod_draw_exact_ws_bytes(n), "pod_draw_exact: workspace too small");
  POD_REQUIRE(cap >= imin64(c, n), "pod_draw_exact: output capacity %lld < min(c, n)",
              (long long)cap);
  POD_REQUIRE(mode == 1 || weights != nullptr, "pod_draw_exact: weights required");
  POD_REQUIRE(mode == 2 || mode == 4 || live != nullptr, "pod_draw_exact: live mask required");
  const int64_t nodes = 2 * (n / 64 + 2);
  double* w = (double*)ws;
  double* cum = w + n;
  PwTree tree;
  tree.lo = (int64_t*)(cum + n);
  tree.val = (double*)(tree.lo + nodes);
  int32_t* cidx = (int32_t*)(tree.val + nodes);
  int32_t* counts = cidx + n;
  tree.len = counts + n;
  tree.child = tree.len + nodes;
  draw_exact_kernel<<<1, XD_THREADS, 0, (cudaStream_t)stream>>>(
      mode, weights, live, n, uniforms, c, idx_out, cnt_out, cap, w, cum, cidx, counts, tree,
      info, thr, p_out);
  POD_CHECK_LAUNCH("draw_exact");
  return POD_OK;
}
