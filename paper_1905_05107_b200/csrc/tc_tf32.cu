// Mixed-precision TN products on the 5th-generation tensor cores (tcgen05,
// kind::tf32, accumulators in TMEM) for float32-STORED data matrices
// (BASELINE config 4: "merge GEMMs on TF32/BF16 tensor cores with FP32
// accumulate ... error reported against the fp64 oracle").
//
//   C (P x Q, fp64) = alpha X^T Y,  K = rows (the long dimension m)
//
// X, Y: K x P / K x Q column-major float32 sources, optionally addressed
// through a column index list (the sampled block D = A[:, idx] is gathered
// inside the operand loads, index -1 = zero column).  "3xTF32": every fp32
// operand is split exactly into hi = tf32(x) (mantissa truncated to 10 bits)
// and lo = tf32(x - hi); the tile product is hi*hi + lo*hi + hi*lo with fp32
// accumulation (relative error ~1e-6 of the fp64 product).  An fp64
// operand (U of finalize A^T U) is pre-split into (hi, lo) fp32 arrays by
// pod_split_tf32.  The tensor core accumulates 256-row groups in TMEM; the
// threads drain each group into an IEEE fp32 master accumulator; K is split
// over CTAs and a deterministic fixed-order fp64 reduction sums their
// partial tiles.
//
// CTA = 128 threads: all threads stage the operands with 16-byte cp.async
// into the canonical K-major SWIZZLE_128B layout (row r of a tile = 32 K
// values = 128 B; 16-byte chunk c stored at c ^ (r & 7)), convert the raw
// fp32 chunks into hi/lo in place, fence them to the async proxy, and one
// elected thread issues the tcgen05.mma (M = 128 rows of X, N = Q columns of
// Y, K = 8 per instruction) and commits them to the stage's mbarrier; the
// four warps read the accumulator back with tcgen05.ld (32 lanes each).
#include <cuda.h>
#include <cstdlib>

#include "common.cuh"

namespace pod {
namespace tc {

constexpr int THREADS = 128;
constexpr int BM = 128;           // MMA M (rows of X per CTA)
constexpr int BK = 32;            // K rows per stage (one 128-byte swizzle row)
// pipeline stages: 4 when a stage fits 56 KB (NQ <= 96), else 3
__host__ __device__ constexpr int stages_for(int nq) { return nq <= 96 ? 4 : 3; }

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SWIZZLE_128B K-major shared-memory matrix descriptor (tcgen05 "version 1"):
// start address >> 4, stride between 8-row groups (1024 B) >> 4, layout 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;                     // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                       // version 1 (Blackwell)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulator, TF32 A and B, both
// K-major, N = n, M = 128.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init1(uint64_t* mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(mb)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;"
                 " selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(saddr(mb)), "r"(parity) : "memory");
}

// exact split of an fp32 value: hi = x with the low 13 mantissa bits cleared
// (a TF32 number), lo = x - hi (exact; <= 13 significant bits)
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

struct Operand {
  const float* src;     // raw fp32 source (K x ncols, column-major)
  const float* lo;      // precomputed lo part (same layout) or null: split in smem
  int64_t ld;
  const int32_t* cols;  // column index list (-1 = zero column) or null
  int ncols;            // valid columns
};

// Stage rows [k0, k0 + BK) of `rows` operand columns (starting at column c0)
// into the hi (and lo) tiles: 16-byte cp.async, 128B-swizzled K-major.
__device__ __forceinline__ void stage_operand(const Operand& op, int c0, int rows, int64_t k0,
                                              int64_t K, unsigned char* hi, unsigned char* lo) {
  for (int e = threadIdx.x; e < rows * 8; e += THREADS) {
    const int r = e >> 3, ch = e & 7;
    const int c = c0 + r;
    int64_t col = c;
    bool ok = c < op.ncols;
    if (ok && op.cols) {
      col = op.cols[c];
      ok = col >= 0;
    }
    const int64_t k = k0 + ch * 4;
    const int64_t rem = K - k;
    const int valid = ok ? (rem >= 4 ? 4 : (rem > 0 ? (int)rem : 0)) : 0;
    const uint32_t dst = (uint32_t)(r * 128 + ((ch ^ (r & 7)) << 4));
    const float* g = ok && valid > 0 ? op.src + col * op.ld + k : op.src;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(hi) + dst),
                 "l"(g), "r"(valid * 4)
                 : "memory");
    if (op.lo) {
      const float* gl = ok && valid > 0 ? op.lo + col * op.ld + k : op.lo;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(lo) + dst),
                   "l"(gl), "r"(valid * 4)
                   : "memory");
    }
  }
}

// raw fp32 tile -> (hi, lo) in place (elementwise: layout-agnostic)
__device__ __forceinline__ void split_tile(unsigned char* hi, unsigned char* lo, int rows) {
  float4* h = reinterpret_cast<float4*>(hi);
  float4* l = reinterpret_cast<float4*>(lo);
  for (int e = threadIdx.x; e < rows * 8; e += THREADS) {
    float4 v = h[e], a, b;
    a.x = tf32_hi(v.x); b.x = v.x - a.x;
    a.y = tf32_hi(v.y); b.y = v.y - a.y;
    a.z = tf32_hi(v.z); b.z = v.z - a.z;
    a.w = tf32_hi(v.w); b.w = v.w - a.w;
    h[e] = a;
    l[e] = b;
  }
}

// grid (ceil(P / 128), ceil(Q / NQ), nsplit); dynamic smem: ST x {Xh, Xl,
// Yh, Yl}.  The tensor core's fp32 accumulation loses ~1 bit per doubling of
// the accumulated K (measured on this B200, tools/tc_diag.py: hi*hi over
// 8192 rows 1.9e-5 relative, 256 rows 9e-7), so the MMAs accumulate GROUP
// stages (256 rows) into one of two TMEM buffers while the threads drain the
// other into an IEEE fp32 master accumulator in registers (one row x NQ
// columns per thread).
#ifndef POD_TC_GROUP
#define POD_TC_GROUP 1
#endif
template <int NQ>
__global__ void __launch_bounds__(THREADS, 1) tn_tf32x3_kernel(
    Operand X, Operand Y, int64_t K, int64_t kchunk, float* __restrict__ part, int64_t ldp, int Q,
    const __grid_constant__ CUtensorMap tmxh, const __grid_constant__ CUtensorMap tmxl,
    const __grid_constant__ CUtensorMap tmyh, const __grid_constant__ CUtensorMap tmyl, int tma_x,
    int tma_y) {
  constexpr int GROUP = POD_TC_GROUP;  // stages per TMEM accumulation group
  constexpr int ST = stages_for(NQ);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int xbytes = BM * 128, ybytes = NQ * 128;
  constexpr int sbytes = 2 * xbytes + 2 * ybytes;
  constexpr int TCOLS = (2 * NQ <= 32) ? 32 : (2 * NQ <= 64 ? 64 : (2 * NQ <= 128 ? 128 : 256));
  __shared__ uint64_t mbar[ST];
  __shared__ uint64_t full[ST];  // TMA arrivals of a stage
  __shared__ uint64_t accbar[2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = blockIdx.x * BM;
  const int q0 = blockIdx.y * NQ;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = (K < kbeg + kchunk) ? K : kbeg + kchunk;
  const int nk = (int)((kend - kbeg + BK - 1) / BK);
  const int ngroups = (nk + GROUP - 1) / GROUP;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(&tmem_base_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init1(&mbar[s]);
      mbar_init1(&full[s]);
    }
    mbar_init1(&accbar[0]);
    mbar_init1(&accbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  auto xh = [&](int s) { return smem + (size_t)s * sbytes; };
  auto xl = [&](int s) { return smem + (size_t)s * sbytes + xbytes; };
  auto yh = [&](int s) { return smem + (size_t)s * sbytes + 2 * xbytes; };
  auto yl = [&](int s) { return smem + (size_t)s * sbytes + 2 * xbytes + ybytes; };
  // TMA (one thread, SWIZZLE_128B boxes of 32 K values x rows, zero fill
  // out of bounds) for the operands that are not gathered; 16-byte cp.async
  // by every thread otherwise.  A stage's TMA bytes complete on full[s].
  // a pre-split operand (lo given) loads hi and lo, a raw one only hi
  const uint32_t tbytes = (tma_x ? (X.lo ? 2u : 1u) * BM * 128u : 0u) +
                          (tma_y ? (Y.lo ? 2u : 1u) * NQ * 128u : 0u);
  auto tma2d = [&](const CUtensorMap* tm, unsigned char* dst, int64_t k, int row, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(saddr(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"((int)k),
        "r"(row), "r"(saddr(bar))
        : "memory");
  };
  auto load = [&](int kt) {
    const int s = kt % ST;
    const int64_t k0 = kbeg + (int64_t)kt * BK;
    if (tbytes && threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                       saddr(&full[s])), "r"(tbytes) : "memory");
      if (tma_x) {
        tma2d(&tmxh, xh(s), k0, p0, &full[s]);
        if (X.lo) tma2d(&tmxl, xl(s), k0, p0, &full[s]);
      }
      if (tma_y) {
        tma2d(&tmyh, yh(s), k0, q0, &full[s]);
        if (Y.lo) tma2d(&tmyl, yl(s), k0, q0, &full[s]);
      }
    }
    if (!tma_x) stage_operand(X, p0, BM, k0, kend, xh(s), xl(s));
    if (!tma_y) stage_operand(Y, q0, NQ, k0, kend, yh(s), yl(s));
  };
  uint32_t fphase[ST] = {};
  float master[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) master[j] = 0.0f;
  // drain TMEM accumulator buffer b (after its group's commit) into master
  auto drain = [&](int b, uint32_t parity) {
    mbar_wait(&accbar[b], parity);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
    for (int c0 = 0; c0 < NQ; c0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * NQ + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) master[c0 + j] += __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  };
  const uint32_t idesc = idesc_tf32(NQ);
  uint32_t phase[ST] = {};
  uint32_t accphase[2] = {0u, 0u};
  // prefetch distance ST - 2: the slot refilled at iteration kt last
  // held stage kt - 2, whose MMAs finished while stage kt - 1's ran -- the
  // tensor core never waits for the refill
  constexpr int DIST = ST - 2;
  for (int kt = 0; kt < DIST && kt < nk; ++kt) {
    load(kt);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % ST;
    const int grp = kt / GROUP, buf = grp & 1;
    const int kn = kt + DIST;
    if (kn < nk) {
      const int sn = kn % ST;
      if (kn >= ST) {  // the slot's previous stage kn - ST = kt - 2
        mbar_wait(&mbar[sn], phase[sn]);
        phase[sn] ^= 1u;
      }
      load(kn);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(DIST) : "memory");
    if (tbytes) {
      mbar_wait(&full[s], fphase[s]);
      fphase[s] ^= 1u;
    }
    __syncthreads();
    if (!X.lo) split_tile(xh(s), xl(s), BM);
    if (!Y.lo) split_tile(yh(s), yl(s), NQ);
    // generic-proxy writes (cp.async, the split) -> visible to the tensor core
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = saddr(xh(s)), al = saddr(xl(s)), bh = saddr(yh(s)), bl = saddr(yl(s));
      const uint32_t td = tmem + (uint32_t)(buf * NQ);
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint32_t off = ks * 32;  // 8 tf32 = 32 bytes along the swizzled row
        const uint32_t acc0 = (kt % GROUP > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(td, sw128_desc(ah + off), sw128_desc(bh + off), idesc, acc0);
        mma_tf32(td, sw128_desc(al + off), sw128_desc(bh + off), idesc, 1u);
        mma_tf32(td, sw128_desc(ah + off), sw128_desc(bl + off), idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       saddr(&mbar[s]))
                   : "memory");
      if (kt % GROUP == GROUP - 1 || kt == nk - 1)
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                saddr(&accbar[buf]))
            : "memory");
    }
    // once this group's first MMAs are issued (into `buf`), drain the
    // previous group's buffer while the tensor core works on this one
    if (kt % GROUP == 0 && grp >= 1) {
      drain(buf ^ 1, accphase[buf ^ 1]);
      accphase[buf ^ 1] ^= 1u;
    }
  }
  if (ngroups >= 1) {  // the last group
    const int b = (ngroups - 1) & 1;
    drain(b, accphase[b]);
  }
  const int row = p0 + warp * 32 + lane;
  if (row < X.ncols) {
    float* out = part + (size_t)blockIdx.z * ldp * (size_t)Q;
#pragma unroll
    for (int j = 0; j < NQ; ++j)
      if (q0 + j < Q) out[row + (size_t)(q0 + j) * ldp] = master[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TCOLS));
}

// Warp-specialized variant for the all-TMA case (X raw fp32, Y pre-split:
// finalize's A^T U).  The phased kernel above serialises load -> split ->
// MMA -> drain inside one loop and kept the tensor pipe 21 % busy; here
// the roles run concurrently on mbarriers:
//   warp 0 lane 0   TMA producer: waits empty[s], loads X / Yh / Yl -> full[s]
//   warp 1 lane 0   MMA issuer:   waits conv[s] (and accfree[b] at a group
//                                 start), 12 MMAs, commits empty[s] (and
//                                 accbar[b] at a group end)
//   warps 4..7      convert + drain: wait full[s], split X into hi / lo in
//                                 place, fence to the async proxy, arrive
//                                 conv[s]; at each group start drain the
//                                 previous group's TMEM buffer into the fp32
//                                 master accumulator and arrive accfree[b]
// (warps 4..7 own TMEM lane quarters 0..3 = rows 0..127 of the tile)
constexpr int WS_THREADS = 256;
#ifndef POD_TC_WS_GROUP
#define POD_TC_WS_GROUP 1
#endif

template <int NQ>
__global__ void __launch_bounds__(WS_THREADS, 1) tn_tf32x3_ws_kernel(
    int P, int64_t K, int64_t kchunk, float* __restrict__ part, int64_t ldp, int Q,
    const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmyh,
    const __grid_constant__ CUtensorMap tmyl) {
  constexpr int GROUP = POD_TC_WS_GROUP;
  constexpr int ST = stages_for(NQ);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int xbytes = BM * 128, ybytes = NQ * 128;
  constexpr int sbytes = 2 * xbytes + 2 * ybytes;
  constexpr int TCOLS = (2 * NQ <= 32) ? 32 : (2 * NQ <= 64 ? 64 : (2 * NQ <= 128 ? 128 : 256));
  __shared__ uint64_t full[ST], conv[ST], empty[ST], accbar[2], accfree[2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = blockIdx.x * BM, q0 = blockIdx.y * NQ;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = (K < kbeg + kchunk) ? K : kbeg + kchunk;
  const int nk = (int)((kend - kbeg + BK - 1) / BK);
  const int ngroups = (nk + GROUP - 1) / GROUP;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(&tmem_base_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < ST; ++s) {
      mbar_init1(&full[s]);
      mbar_init1(&empty[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(saddr(&conv[s])));
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init1(&accbar[b]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(saddr(&accfree[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  auto xh = [&](int s) { return smem + (size_t)s * sbytes; };
  auto xl = [&](int s) { return smem + (size_t)s * sbytes + xbytes; };
  auto yh = [&](int s) { return smem + (size_t)s * sbytes + 2 * xbytes; };
  auto yl = [&](int s) { return smem + (size_t)s * sbytes + 2 * xbytes + ybytes; };
  auto tma2d = [&](const CUtensorMap* tm, unsigned char* dst, int64_t k, int row, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(saddr(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"((int)k),
        "r"(row), "r"(saddr(bar))
        : "memory");
  };

  if (warp == 0) {  // ------------------------------------------ TMA producer
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % ST;
        if (kt >= ST) mbar_wait(&empty[s], (uint32_t)((kt / ST - 1) & 1));
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                         saddr(&full[s])), "r"((uint32_t)(xbytes + 2 * ybytes)) : "memory");
        const int64_t k0 = kbeg + (int64_t)kt * BK;
        tma2d(&tmx, xh(s), k0, p0, &full[s]);
        tma2d(&tmyh, yh(s), k0, q0, &full[s]);
        tma2d(&tmyl, yl(s), k0, q0, &full[s]);
      }
    }
  } else if (warp == 1) {  // ------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(NQ);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % ST, grp = kt / GROUP, buf = grp & 1;
        if (kt % GROUP == 0 && grp >= 2) mbar_wait(&accfree[buf], (uint32_t)((grp / 2 - 1) & 1));
        mbar_wait(&conv[s], (uint32_t)((kt / ST) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ah = saddr(xh(s)), al = saddr(xl(s)), bh = saddr(yh(s)), bl = saddr(yl(s));
        const uint32_t td = tmem + (uint32_t)(buf * NQ);
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t off = ks * 32;
          const uint32_t acc0 = (kt % GROUP > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(td, sw128_desc(ah + off), sw128_desc(bh + off), idesc, acc0);
          mma_tf32(td, sw128_desc(al + off), sw128_desc(bh + off), idesc, 1u);
          mma_tf32(td, sw128_desc(ah + off), sw128_desc(bl + off), idesc, 1u);
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                saddr(&empty[s]))
            : "memory");
        if (kt % GROUP == GROUP - 1 || kt == nk - 1)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  saddr(&accbar[buf]))
              : "memory");
      }
    }
  } else if (warp >= 4) {  // --------------------------- convert + drain
    const int t = threadIdx.x - 128, wq = warp - 4;  // TMEM lane quarter
    float master[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) master[j] = 0.0f;
    auto drain = [&](int b, uint32_t parity) {
      mbar_wait(&accbar[b], parity);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < NQ; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * NQ + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) master[c0 + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&accfree[b])) : "memory");
    };
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % ST;
      mbar_wait(&full[s], (uint32_t)((kt / ST) & 1));
      float4* h = reinterpret_cast<float4*>(xh(s));
      float4* l = reinterpret_cast<float4*>(xl(s));
#pragma unroll
      for (int e = t; e < BM * 8; e += 128) {
        const float4 v = h[e];
        float4 a, b;
        a.x = tf32_hi(v.x); b.x = v.x - a.x;
        a.y = tf32_hi(v.y); b.y = v.y - a.y;
        a.z = tf32_hi(v.z); b.z = v.z - a.z;
        a.w = tf32_hi(v.w); b.w = v.w - a.w;
        h[e] = a;
        l[e] = b;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&conv[s])) : "memory");
      const int grp = kt / GROUP;
      if (kt % GROUP == 0 && grp >= 1) {  // the previous group is complete soon
        const int pg = grp - 1;
        drain(pg & 1, (uint32_t)((pg / 2) & 1));
      }
    }
    if (ngroups >= 1) {
      const int lg = ngroups - 1;
      drain(lg & 1, (uint32_t)((lg / 2) & 1));
    }
    const int row = p0 + t;
    if (row < P) {
      float* out = part + (size_t)blockIdx.z * ldp * (size_t)Q;
#pragma unroll
      for (int j = 0; j < NQ; ++j)
        if (q0 + j < Q) out[row + (size_t)(q0 + j) * ldp] = master[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TCOLS));
}

// C (P x Q, ldc) = alpha * sum over splits of part[s] (fixed order, fp64)
__global__ void reduce_parts_kernel(const float* __restrict__ part, int nsplit, int P, int Q,
                                    int64_t ldp, double alpha, double* __restrict__ C,
                                    int64_t ldc) {
  const int64_t tot = (int64_t)P * Q;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(t / P), i = (int)(t - (int64_t)j * P);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += (double)part[(size_t)sp * ldp * Q + i + (size_t)j * ldp];
    C[i + (int64_t)j * ldc] = alpha * s;
  }
}

// fp64 (K x Q, ld) -> exact-split fp32 (hi, lo) arrays (K x Q, ld K): hi =
// tf32(float(x)), lo = float(x) - hi; the fp64 -> fp32 rounding (2^-24
// relative) is the split's only loss
__global__ void split_f64_kernel(const double* __restrict__ U, int64_t K, int Q, int64_t ldu,
                                 float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t tot = K * Q;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / K, i = t - j * K;
    const float x = (float)U[i + j * ldu];
    const float h = tf32_hi(x);
    hi[t] = h;
    lo[t] = x - h;
  }
}

}  // namespace tc
}  // namespace pod

using namespace pod;

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}
// 2-D fp32 tensor map over a column-major K x ncols matrix: dim0 = K (the
// contiguous rows), dim1 = columns; box = 32 K values x `rows` columns,
// 128-byte swizzle (the UMMA K-major SW128 tile), zero fill out of bounds
bool make_tmap(CUtensorMap* tm, const float* base, int64_t K, int64_t ncols, int64_t ld,
               int rows) {
  EncodeTiled fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)ncols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {32u, (cuuint32_t)rows};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// POD_TC_WS=0 forces the phased kernel (A/B measurement)
bool ws_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("POD_TC_WS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int NQ>
cudaError_t launch_ws_t(dim3 grid, size_t smem, int64_t P, int64_t K, int64_t kchunk, float* part,
                        int Q, const CUtensorMap& tx, const CUtensorMap& tyh,
                        const CUtensorMap& tyl, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(pod::tc::tn_tf32x3_ws_kernel<NQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done = true;
  }
  pod::tc::tn_tf32x3_ws_kernel<NQ><<<grid, pod::tc::WS_THREADS, smem, s>>>(
      (int)P, K, kchunk, part, P, Q, tx, tyh, tyl);
  return cudaGetLastError();
}

cudaError_t launch_ws(int nq, dim3 grid, size_t smem, int64_t P, int64_t K, int64_t kchunk,
                      float* part, int Q, const CUtensorMap& tx, const CUtensorMap& tyh,
                      const CUtensorMap& tyl, cudaStream_t s) {
  if (nq == 64) return launch_ws_t<64>(grid, smem, P, K, kchunk, part, Q, tx, tyh, tyl, s);
  if (nq == 96) return launch_ws_t<96>(grid, smem, P, K, kchunk, part, Q, tx, tyh, tyl, s);
  return launch_ws_t<128>(grid, smem, P, K, kchunk, part, Q, tx, tyh, tyl, s);
}

// K split: enough CTAs for ~2 per SM, each at least 2048 rows
int64_t tc_nsplit(int64_t P, int64_t Q, int64_t K) {
  const int64_t tiles = ((P + pod::tc::BM - 1) / pod::tc::BM) * ((Q + 63) / 64);
  static int64_t target = -1;  // CTAs to aim for (POD_TC_CTAS overrides; A/B measurement)
  if (target < 0) {
    const char* e = getenv("POD_TC_CTAS");
    target = e ? std::max(1, atoi(e)) : 2 * 148;
  }
  int64_t ns = std::max<int64_t>(1, (target + tiles - 1) / tiles);
  ns = std::min<int64_t>(ns, std::max<int64_t>(1, K / 2048));
  return std::min<int64_t>(ns, 65535);
}
}  // namespace

extern "C" size_t pod_tc_tn_ws_bytes(int64_t P, int64_t Q, int64_t K) {
  return (size_t)tc_nsplit(P, Q, K) * (size_t)P * (size_t)Q * sizeof(float) + 256;
}

extern "C" int pod_gemm_tn_tf32x3(int64_t P, int64_t Q, int64_t K, double alpha, const float* X,
                                  const float* Xlo, int64_t ldx, const int32_t* xcols,
                                  const float* Y, const float* Ylo, int64_t ldy,
                                  const int32_t* ycols, double* C, int64_t ldc, void* ws,
                                  size_t ws_bytes, void* stream) {
  using namespace pod::tc;
  POD_REQUIRE(P >= 1 && Q >= 1 && K >= 1 && ldc >= P,
              "pod_gemm_tn_tf32x3: bad shape P=%lld Q=%lld K=%lld", (long long)P, (long long)Q,
              (long long)K);
  POD_REQUIRE(ldx >= K && ldy >= K && ldx % 4 == 0 && ldy % 4 == 0,
              "pod_gemm_tn_tf32x3: leading dimensions must be >= K and multiples of 4");
  POD_REQUIRE((reinterpret_cast<uintptr_t>(X) & 15) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0,
              "pod_gemm_tn_tf32x3: operands must be 16-byte aligned");
  POD_REQUIRE(ws_bytes >= pod_tc_tn_ws_bytes(P, Q, K), "pod_gemm_tn_tf32x3: workspace too small");
  const int64_t nsplit = tc_nsplit(P, Q, K);
  int64_t kchunk = (K + nsplit - 1) / nsplit;
  kchunk = (kchunk + BK - 1) / BK * BK;
  Operand xo{X, Xlo, ldx, xcols, (int)P};
  Operand yo{Y, Ylo, ldy, ycols, (int)Q};
  float* part = (float*)ws;
  cudaStream_t s = (cudaStream_t)stream;
  static bool attr_done[3] = {false, false, false};
  auto launch = [&](auto kern, int nq) -> int {
    const size_t smem = (size_t)stages_for(nq) * (2 * BM * 128 + 2 * nq * 128) + 1024;
    bool& done = attr_done[nq == 64 ? 0 : (nq == 96 ? 1 : 2)];
    if (!done) {  // once (outside any later graph capture of the launch)
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return cuda_status(e, "tc smem attribute");
      done = true;
    }
    dim3 grid((unsigned)((P + BM - 1) / BM), (unsigned)((Q + nq - 1) / nq), (unsigned)nsplit);
    // TMA for the operands that are not gathered (and, for Y, pre-split)
    CUtensorMap tmxh{}, tmxl{}, tmyh{}, tmyl{};
    const int tx = !xcols && make_tmap(&tmxh, X, K, P, ldx, BM) &&
                   (!Xlo || make_tmap(&tmxl, Xlo, K, P, ldx, BM));
    const int ty = !ycols && make_tmap(&tmyh, Y, K, Q, ldy, nq) &&
                   (!Ylo || make_tmap(&tmyl, Ylo, K, Q, ldy, nq));
    if (tx && ty && !Xlo && Ylo && ws_enabled()) {  // all-TMA: the warp-specialized kernel
      cudaError_t e = launch_ws(nq, grid, smem, P, K, kchunk, part, (int)Q, tmxh, tmyh, tmyl, s);
      if (e != cudaSuccess) return cuda_status(e, "tn_tf32x3 ws");
      return POD_OK;
    }
    kern<<<grid, THREADS, smem, s>>>(xo, yo, K, kchunk, part, P, (int)Q, tmxh, tmxl, tmyh, tmyl,
                                     tx, ty);
    POD_CHECK_LAUNCH("tn_tf32x3");
    return POD_OK;
  };
  // column slice per CTA (the fp32 master accumulator is one row x NQ per
  // thread): the narrowest of 64 / 96 / 128 that tiles Q with the least padding
  const int nq = (Q <= 64) ? 64 : ((Q % 128 == 0 || (Q > 96 && Q <= 128)) ? 128 : 96);
  int st = (nq == 64) ? launch(tn_tf32x3_kernel<64>, 64)
                      : (nq == 96 ? launch(tn_tf32x3_kernel<96>, 96)
                                  : launch(tn_tf32x3_kernel<128>, 128));
  if (st) return st;
  const int rb = (int)std::min<int64_t>(ceil_div(P * Q, 256), 148 * 8);
  reduce_parts_kernel<<<rb, 256, 0, s>>>(part, (int)nsplit, (int)P, (int)Q, P, alpha, C, ldc);
  POD_CHECK_LAUNCH("tn_tf32x3 reduce");
  return POD_OK;
}

extern "C" int pod_split_tf32(const double* U, int64_t K, int64_t Q, int64_t ldu, float* hi,
                              float* lo, void* stream) {
  POD_REQUIRE(K >= 1 && Q >= 1 && ldu >= K, "pod_split_tf32: bad shape");
  const int g = (int)std::min<int64_t>(ceil_div(K * Q, 256), 148 * 16);
  tc::split_f64_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(U, K, (int)Q, ldu, hi, lo);
  POD_CHECK_LAUNCH("split_tf32");
  return POD_OK;
}
