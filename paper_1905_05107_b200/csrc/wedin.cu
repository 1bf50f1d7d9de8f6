// Fused Wedin residual pass (wedin_measure, quality.py:82-118):
//
//   R = A V_k - U_k S_k   (m x k)      S = A^T U_k - V_k S_k   (n x k)
//
// ||R||_F^2 and ||S||_F^2 from ONE pass over A.  The reference forms both
// products with separate BLAS calls and materialises R and S
// (quality.py:104-107); here every A tile is staged once in shared memory
// and feeds both DMMA products:
//
//  * rows: a thread-block cluster of CL CTAs owns CL x 128 consecutive rows
//    (one 128-row slab per CTA, persistent over row ranges).  A CTA walks
//    all n columns in 32-column chunks (cp.async double buffer); its slab of
//    R stays in registers as DMMA accumulators, so at the end of the range R
//    is complete and (R - U_k S_k)^2 is reduced in the epilogue -- R is never
//    written.
//  * columns: each chunk's S partial (32 x k, this CTA's 128 rows) goes to a
//    3-slot ring in shared memory and the cluster sums the CL slabs through
//    DSMEM (ld.shared::cluster, fixed rank order) into one partial per row
//    range: traffic (m / (CL 128)) n k 8 bytes, ~1-5 % of A.  The cluster
//    barrier that publishes chunk t is waited for one chunk later, so its
//    latency hides under the next chunk's DMMAs.
//  * a second kernel sums the row-range partials of S in fixed order,
//    subtracts V_k S_k and squares; a third adds the per-CTA sums.
// Deterministic (fixed assignment and summation order, no atomics).
#include "common.cuh"

namespace pod {
namespace wdn {
constexpr int NW = 8, THREADS = NW * 32;
constexpr int RC = 128;  // rows per CTA slab
constexpr int BN = 32;   // A columns per chunk
constexpr int LDU = RC + 4;  // U slab [q][row] (fp64): % 16 == 4, conflict-free fragments
constexpr int LDV = BN + 4;  // V chunk [q][j]
constexpr int SST = 3;       // S partial ring slots
// chunks per published S group (one cluster barrier per group): as many as
// fit shared memory next to the slab, the tiles and the V chunks
__host__ __device__ constexpr int group_chunks(int nf) { return nf <= 4 ? 4 : (nf <= 6 ? 2 : 1); }

template <typename TA>
struct Geo {
  static constexpr int LDA = RC + (sizeof(TA) == 8 ? 4 : 8);  // A tile [col][row]
  static constexpr size_t A_BYTES = size_t(BN) * LDA * sizeof(TA);  // one stage
};

template <int NF, typename TA>
constexpr size_t smem_bytes() {
  constexpr int KP = NF * 8;
  return size_t(KP) * LDU * 8 + 2 * Geo<TA>::A_BYTES + 2 * size_t(KP) * LDV * 8 +
         size_t(SST) * group_chunks(NF) * BN * KP * 8 + 2 * KP * 8 + NW * 8 +
         2 * size_t(group_chunks(NF)) * BN * KP;  // TMA-store staging: 2 x GW KP / 8 doubles
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// reduced S partials leave through the async proxy (cp.async.bulk smem ->
// global): a generic st.global before the cluster barrier's release would
// make every arrive wait for those stores to reach L2
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ double ld_cluster(uint32_t saddr, uint32_t rank) {
  uint32_t ra;
  double v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(saddr), "r"(rank));
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

// partial[range][j][q] (q < KP) = sum over the cluster's rows of A[i, j] U[i, q];
// rpart[cta] = sum over its slabs of (A V - U S_k)^2
template <int NF, typename TA>
__global__ void __launch_bounds__(THREADS, 1) pass_kernel(
    int64_t m, int n, int k, const TA* __restrict__ A, int64_t lda, const double* __restrict__ U,
    int64_t ldu, const double* __restrict__ V, int64_t ldv, const double* __restrict__ sigma,
    int64_t nranges, int vecA, double* __restrict__ partial, double* __restrict__ rpart) {
  constexpr int KP = NF * 8;
  constexpr int LDA = Geo<TA>::LDA;
  constexpr int P = group_chunks(NF);
  constexpr int GW = P * BN;  // columns per published group
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* us = reinterpret_cast<double*>(smem_raw);                        // KP x LDU
  TA* as0 = reinterpret_cast<TA*>(smem_raw + size_t(KP) * LDU * 8);         // 2 stages
  double* vs0 = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(as0) +
                                          2 * Geo<TA>::A_BYTES);            // 2 x KP x LDV
  double* sst = vs0 + 2 * KP * LDV;                                         // SST x GW x KP
  double* sig = sst + SST * GW * KP;                                        // KP (+KP pad)
  double* red = sig + 2 * KP;                                               // NW
  double* stg0 = red + NW;                                                  // 2 x GW KP / 8

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t rank = cta_rank();
  const int CL = (int)(gridDim.x / n_clusters());
  const int nch = (n + BN - 1) / BN;
  for (int q = threadIdx.x; q < KP; q += THREADS) sig[q] = q < k ? sigma[q] : 0.0;

  auto load_chunk = [&](int st, int64_t r0, int c0) {
    TA* as = as0 + (size_t)st * BN * LDA;
    double* vs = vs0 + (size_t)st * KP * LDV;
    constexpr int VE = 16 / sizeof(TA);  // elements per 16-byte copy
    for (int e = threadIdx.x; e < BN * (RC / VE); e += THREADS) {
      const int j = e / (RC / VE), i = (e - j * (RC / VE)) * VE;
      const int c = c0 + j;
      const int64_t row = r0 + i;
      TA* dst = as + j * LDA + i;
      const TA* src = A + (int64_t)c * lda + row;
      if (c < n && vecA && row + VE <= m) {
        cp_async16(dst, src, true);
      } else {
#pragma unroll
        for (int v = 0; v < VE; ++v) {
          const bool ok = c < n && row + v < m;
          cp_async_elem(dst + v, ok ? src + v : A, ok);
        }
      }
    }
    for (int e = threadIdx.x; e < KP * BN; e += THREADS) {
      const int q = e / BN, j = e - q * BN;
      const bool ok = q < k && c0 + j < n;
      cp_async8(vs + q * LDV + j, ok ? V + (int64_t)q * ldv + c0 + j : V, ok);
    }
  };
  auto load_u = [&](int64_t r0) {
    for (int e = threadIdx.x; e < KP * RC; e += THREADS) {
      const int q = e / RC, i = e - q * RC;
      const bool ok = q < k && r0 + i < m;
      cp_async8(us + q * LDU + i, ok ? U + (int64_t)q * ldu + r0 + i : U, ok);
    }
  };

  double rsum = 0.0;  // this thread's share of ||R||_F^2
  int64_t t = 0;      // S groups published (ring slot t % SST, cluster phase t)
  // S reduction of group t-1 (after the wait for phase t-1): rank `rank`
  // sums its share of the GW x KP elements over the CL slabs, in rank order
  auto reduce_prev = [&](int64_t range, int c0) {
    const double* slot = sst + (size_t)((t - 1) % SST) * GW * KP;
    const int per = GW * KP / CL;  // CL in {8, 16} divides GW KP
    const int e0 = (int)rank * per;
    const int e1 = min(e0 + per, min(GW, n - c0) * KP);
    double* stg = stg0 + (size_t)((t - 1) & 1) * (GW * KP / 8);
    if (threadIdx.x == 0) bulk_wait_read<1>();  // the store of two groups ago has read stg
    __syncthreads();
    for (int e = e0 + threadIdx.x; e < e1; e += THREADS) {
      const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(slot + e));
      double v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < CL) v[r] = ld_cluster(sa, r);
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < CL) s += v[r];
      stg[e - e0] = s;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0 && e1 > e0)
      bulk_store(partial + ((size_t)range * n + c0) * KP + e0, stg, (uint32_t)(e1 - e0) * 8);
  };
  int64_t prev_range = -1;
  int prev_c0 = 0;

  const int cf = warp & 3, half = warp >> 2;  // S: A-column fragment, row half
  for (int64_t range = cluster_id(); range < nranges; range += n_clusters()) {
    const int64_t r0 = (range * CL + rank) * RC;
    __syncthreads();  // every warp done with the previous range's U slab and stages
    load_u(r0);
    load_chunk(0, r0, 0);
    cp_async_commit();
    double accR[2][NF][2];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int g = 0; g < NF; ++g) accR[f][g][0] = accR[f][g][1] = 0.0;
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<0>();
      __syncthreads();  // chunk c landed; chunk c-1's stage is free
      if (c + 1 < nch) load_chunk((c + 1) & 1, r0, (c + 1) * BN);
      cp_async_commit();
      const TA* as = as0 + (size_t)(c & 1) * BN * LDA;
      const double* vs = vs0 + (size_t)(c & 1) * KP * LDV;
      // R slab (rows 16 warp .. +16) += A_tile V_chunk
#pragma unroll
      for (int kk = 0; kk < BN / 4; ++kk) {
        double a[2], b[NF];
#pragma unroll
        for (int f = 0; f < 2; ++f)
          a[f] = (double)as[(kk * 4 + (lane & 3)) * LDA + warp * 16 + f * 8 + (lane >> 2)];
#pragma unroll
        for (int g = 0; g < NF; ++g) b[g] = vs[(g * 8 + (lane >> 2)) * LDV + kk * 4 + (lane & 3)];
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int g = 0; g < NF; ++g) dmma8x8x4(accR[f][g][0], accR[f][g][1], a[f], b[g]);
      }
      // S chunk (A columns 8 cf .. +8) over this warp's 64-row half
      double accS[NF][2];
#pragma unroll
      for (int g = 0; g < NF; ++g) accS[g][0] = accS[g][1] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < RC / 8; ++kk) {
        const int i0 = half * (RC / 2) + kk * 4 + (lane & 3);
        const double a = (double)as[(cf * 8 + (lane >> 2)) * LDA + i0];
        double b[NF];
#pragma unroll
        for (int g = 0; g < NF; ++g) b[g] = us[(g * 8 + (lane >> 2)) * LDU + i0];
#pragma unroll
        for (int g = 0; g < NF; ++g) dmma8x8x4(accS[g][0], accS[g][1], a, b[g]);
      }
      // group t's first chunk: phase t-1 complete (all slabs of group t-1
      // written, ring slot t % SST no longer read); this CTA's slab -> slot
      const int sub = c % P;
      if (sub == 0 && t > 0) cl_wait();
      double* slot = sst + (size_t)(t % SST) * GW * KP + (size_t)sub * BN * KP;
      if (half == 1) {
#pragma unroll
        for (int g = 0; g < NF; ++g)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            slot[(cf * 8 + (lane >> 2)) * KP + g * 8 + 2 * (lane & 3) + e] = accS[g][e];
      }
      __syncthreads();
      if (half == 0) {
#pragma unroll
        for (int g = 0; g < NF; ++g)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            slot[(cf * 8 + (lane >> 2)) * KP + g * 8 + 2 * (lane & 3) + e] += accS[g][e];
      }
      if (sub == P - 1 || c == nch - 1) {
        cl_arrive();  // phase t: this CTA's slab of group t published
        if (t > 0) reduce_prev(prev_range, prev_c0);
        prev_range = range;
        prev_c0 = (c - sub) * BN;
        ++t;
      }
    }
    // epilogue: R slab complete -> (R - U S_k)^2 (U slab still resident)
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int i = warp * 16 + f * 8 + (lane >> 2);
#pragma unroll
      for (int g = 0; g < NF; ++g)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int q = g * 8 + 2 * (lane & 3) + e;
          const double d = accR[f][g][e] - us[q * LDU + i] * sig[q];
          rsum = fma(d, d, rsum);
        }
    }
  }
  // last chunk's reduction, then keep the shared memory alive until every
  // CTA of the cluster has read it
  if (t > 0) {
    cl_wait();
    reduce_prev(prev_range, prev_c0);
    cl_arrive();  // arrives only after its DSMEM reads: the last wait keeps
    cl_wait();    // every slab alive until the whole cluster is done
  }
  if (threadIdx.x == 0) bulk_wait_all();
  const double s = block_sum(rsum, red);
  if (threadIdx.x == 0) rpart[blockIdx.x] = s;
}

// spart[block] = sum over (j, q) of (sum_range partial[range][j][q] - V[j, q] sigma_q)^2
__global__ void __launch_bounds__(256) s_kernel(int n, int k, int KP, int64_t nranges,
                                                const double* __restrict__ partial,
                                                const double* __restrict__ V, int64_t ldv,
                                                const double* __restrict__ sigma,
                                                double* __restrict__ spart) {
  __shared__ double red[8];
  const int64_t total = (int64_t)n * KP;
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / KP;
    const int q = (int)(e - j * KP);
    if (q >= k) continue;
    double s = 0.0;
    for (int64_t r = 0; r < nranges; ++r) s += partial[r * total + e];
    const double d = s - V[j + (int64_t)q * ldv] * sigma[q];
    acc = fma(d, d, acc);
  }
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) spart[blockIdx.x] = b;
}

__global__ void __launch_bounds__(256) final_kernel(int nr, const double* __restrict__ rpart,
                                                    int ns, const double* __restrict__ spart,
                                                    double* __restrict__ out) {
  __shared__ double red[8];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nr; i += blockDim.x) a += rpart[i];
  for (int i = threadIdx.x; i < ns; i += blockDim.x) b += spart[i];
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

constexpr int S_BLOCKS = 296;

struct Plan {
  int nf, cl;
  int64_t nranges, clusters;
};

template <int NF, typename TA>
static int set_attrs(int cl) {
  auto fn = pass_kernel<NF, TA>;
  cudaError_t e = cudaFuncSetAttribute((const void*)fn,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes<NF, TA>());
  if (e != cudaSuccess) return cuda_status(e, "wedin attr");
  if (cl > 8) {
    e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_status(e, "wedin cluster attr");
  }
  return POD_OK;
}

// clusters that fit the GPU at once (one CTA per SM)
template <int NF, typename TA>
static int max_clusters(int cl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl, 1, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem_bytes<NF, TA>();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, (const void*)pass_kernel<NF, TA>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

template <int NF, typename TA>
static int launch_pass(const Plan& pl, cudaStream_t s, int64_t m, int n, int k, const TA* A,
                       int64_t lda, const double* U, int64_t ldu, const double* V, int64_t ldv,
                       const double* sigma, int vecA, double* partial, double* rpart) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(pl.clusters * pl.cl), 1, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem_bytes<NF, TA>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pl.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, pass_kernel<NF, TA>, m, n, k, A, lda, U, ldu, V, ldv,
                                     sigma, pl.nranges, vecA, partial, rpart);
  return e == cudaSuccess ? POD_OK : cuda_status(e, "wedin pass launch");
}

template <typename TA>
static int dispatch(int nf, const Plan& pl, cudaStream_t s, int64_t m, int n, int k, const TA* A,
                    int64_t lda, const double* U, int64_t ldu, const double* V, int64_t ldv,
                    const double* sigma, int vecA, double* partial, double* rpart) {
  switch (nf) {
#define WDN_CASE(NF_) \
  case NF_:           \
    return launch_pass<NF_, TA>(pl, s, m, n, k, A, lda, U, ldu, V, ldv, sigma, vecA, partial, rpart);
    WDN_CASE(1) WDN_CASE(2) WDN_CASE(3) WDN_CASE(4) WDN_CASE(5) WDN_CASE(6) WDN_CASE(7) WDN_CASE(8)
#undef WDN_CASE
  }
  set_error("pod_wedin_residuals: bad k");
  return POD_EPARAM;
}

template <typename TA>
static int prepare(int nf, int cl, int* nc) {
  int st = POD_OK;
  switch (nf) {
#define WDN_CASE(NF_)                    \
  case NF_:                              \
    st = set_attrs<NF_, TA>(cl);         \
    *nc = st ? 0 : max_clusters<NF_, TA>(cl); \
    break;
    WDN_CASE(1) WDN_CASE(2) WDN_CASE(3) WDN_CASE(4) WDN_CASE(5) WDN_CASE(6) WDN_CASE(7) WDN_CASE(8)
#undef WDN_CASE
  }
  return st;
}

// 16-CTA clusters (non-portable) halve the row-range partials when they fit;
// cached per (type, nf)
static int g_cl[2][9] = {};
static int g_nc[2][9] = {};

inline Plan plan(int64_t m, int64_t k, int cl) {
  Plan pl;
  pl.nf = (int)((k + 7) / 8);
  pl.cl = cl;
  pl.nranges = ceil_div(m, (int64_t)cl * RC);
  pl.clusters = 0;
  return pl;
}
}  // namespace wdn
}  // namespace pod

using namespace pod;

// Workspace: row-range partials of S (upper bound: 8-CTA clusters), per-CTA
// and per-block sums.
extern "C" size_t pod_wedin_ws_bytes(int64_t m, int64_t n, int64_t k) {
  if (m <= 0 || n <= 0 || k <= 0) return 256;
  const int64_t kp = ((k + 7) / 8) * 8;
  const int64_t nr = ceil_div(m, 8 * wdn::RC);
  return (size_t)(nr * n * kp + 4096 + wdn::S_BLOCKS) * sizeof(double);
}

extern "C" int pod_wedin_residuals(int atype, const void* A, int64_t m, int64_t n, int64_t lda,
                                   const double* U, int64_t ldu, const double* V, int64_t ldv,
                                   const double* sigma, int64_t k, double* out2, void* ws,
                                   size_t ws_bytes, void* stream) {
  POD_REQUIRE(atype == POD_F64 || atype == POD_F32, "pod_wedin_residuals: bad operand type");
  POD_REQUIRE(m >= 1 && n >= 1 && k >= 1 && k <= 64, "pod_wedin_residuals: need m, n >= 1 and 1 <= k <= 64");
  POD_REQUIRE(lda >= m && ldu >= m && ldv >= n, "pod_wedin_residuals: bad leading dimension");
  POD_REQUIRE(n <= INT32_MAX, "pod_wedin_residuals: n too large");
  POD_REQUIRE(ws_bytes >= pod_wedin_ws_bytes(m, n, k), "pod_wedin_residuals: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const int ti = atype == POD_F64 ? 0 : 1;
  const int nf = (int)((k + 7) / 8);
  if (wdn::g_cl[ti][nf] == 0) {
    // the cluster size that keeps the most SMs busy (16-CTA clusters halve
    // the S partials but may strand SMs: 7 x 16 = 112 of 148)
    int nc16 = 0, nc8 = 0, st;
    st = ti == 0 ? wdn::prepare<double>(nf, 16, &nc16) : wdn::prepare<float>(nf, 16, &nc16);
    if (st) return st;
    st = ti == 0 ? wdn::prepare<double>(nf, 8, &nc8) : wdn::prepare<float>(nf, 8, &nc8);
    if (st) return st;
    POD_REQUIRE(nc8 >= 1 || nc16 >= 1, "pod_wedin_residuals: no cluster fits this GPU");
    const bool use16 = nc16 * 16 >= nc8 * 8;
    wdn::g_cl[ti][nf] = use16 ? 16 : 8;
    wdn::g_nc[ti][nf] = use16 ? nc16 : nc8;
  }
  wdn::Plan pl = wdn::plan(m, k, wdn::g_cl[ti][nf]);
  pl.clusters = std::min<int64_t>(pl.nranges, wdn::g_nc[ti][nf]);
  const int64_t kp = (int64_t)nf * 8;
  double* partial = (double*)ws;
  double* rpart = partial + pl.nranges * n * kp;
  double* spart = rpart + 4096;
  POD_REQUIRE(pl.clusters * pl.cl <= 4096, "pod_wedin_residuals: grid too large");
  const size_t esz = atype == POD_F64 ? 8 : 4;
  const int vecA = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((lda * esz) % 16 == 0);
  int st;
  if (atype == POD_F64)
    st = wdn::dispatch<double>(nf, pl, s, m, (int)n, (int)k, (const double*)A, lda, U, ldu, V, ldv,
                               sigma, vecA, partial, rpart);
  else
    st = wdn::dispatch<float>(nf, pl, s, m, (int)n, (int)k, (const float*)A, lda, U, ldu, V, ldv,
                              sigma, vecA, partial, rpart);
  if (st) return st;
  wdn::s_kernel<<<wdn::S_BLOCKS, 256, 0, s>>>((int)n, (int)k, (int)kp, pl.nranges, partial, V, ldv,
                                              sigma, spart);
  POD_CHECK_LAUNCH("wedin S reduce");
  wdn::final_kernel<<<1, 256, 0, s>>>((int)(pl.clusters * pl.cl), rpart, wdn::S_BLOCKS, spart,
                                       out2);
  POD_CHECK_LAUNCH("wedin final");
  return POD_OK;
}
