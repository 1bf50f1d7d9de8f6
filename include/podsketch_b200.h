/* podsketch-b200 C ABI -- the drop-in boundary for the ISMA hot path.
 *
 * The reference (podsketch 0.1.0) is a pure-Python package: its hot path
 * sits behind a Python API, not an FFI.  Each entry point below replaces
 * the numpy/LAPACK call site cited beside it; the Python host layer
 * (paper_1905_05107_b200/) binds them with ctypes and keeps the reference's
 * names, argument meaning and error behaviour.
 *
 * Conventions
 *   - Matrices are column-major float64 with an explicit leading dimension
 *     (the reference's Fortran-order storage, matcore.py:4-7).
 *   - Every pointer argument is DEVICE memory owned by the caller, except
 *     where noted.  Nothing allocates device memory; scratch is passed in
 *     as (ws, ws_bytes) sized by the matching *_ws_bytes query.
 *   - `stream` is a cudaStream_t; all work is enqueued asynchronously.
 *   - Column index lists (`*cols`, int32) address a matrix's columns
 *     indirectly, so a sampled block A[:, idx] is read in place.
 *   - Return codes mirror the reference's error classes (errors.py:8-21):
 *     POD_OK, POD_EPARAM (ParameterError, CLI exit 2), POD_EFORMAT
 *     (FormatError, 3), POD_EDEGENERATE (DegenerateDistributionError, 4),
 *     POD_ENOCONVERGE (scipy LinAlgError), POD_ECUDA; message text via
 *     pod_last_error().
 */
#ifndef PODSKETCH_B200_H
#define PODSKETCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* operand storage types of the typed entry points (fp32 storage is converted
 * exactly to fp64 inside the kernels: results equal the fp64 path on the
 * upcast operand, as the reference's as_dense upcast, matcore.py:49) */
#define POD_F64 0
#define POD_F32 1

#define POD_OK 0
/* sticky CholeskyQR-breakdown slot of the dinfo vector */
#define POD_DINFO_BREAKDOWN 8
#define POD_EPARAM 2
#define POD_EFORMAT 3
#define POD_EDEGENERATE 4
#define POD_ENOCONVERGE 5
#define POD_ECUDA 6
#define POD_ENCCL 7

int pod_abi_version(void);
/* Last error message of the calling thread ("" if none). */
const char* pod_last_error(void);

/* Squared column norms ||A[:, j]||^2 and a non-finite flag, one HBM pass.
 * Replaces matcore.py:54 (isfinite), isma.py:260 and sampling.py:136
 * (np.einsum("ij,ij->j", a, a)) BIT-EXACTLY: the sums follow numpy 2.3's
 * einsum order for a contiguous column (two lanes; per 8-row block
 * acc_l = x[i+l]^2 + (x[i+2+l]^2 + (x[i+4+l]^2 + (x[i+6+l]^2 + acc_l))),
 * products and sums each rounded; the m % 8 tail lane-pairwise; acc_0 +
 * acc_1), see exact_sums.cu.  nonfinite is set to 1 if any entry is NaN/Inf.
 * Columns are streamed through shared memory with cp.async.bulk when A and
 * lda * sizeof(element) are 16-byte aligned. */
int pod_colnorms2_f64(const double* A, int64_t m, int64_t n, int64_t lda, double* norms2,
                      int32_t* nonfinite, void* stream);
/* Same for a POD_F64 or POD_F32 stored A (the exactly upcast values,
 * as_dense's astype(float64), matcore.py:49). */
int pod_colnorms2(int atype, const void* A, int64_t m, int64_t n, int64_t lda, double* norms2,
                  int32_t* nonfinite, void* stream);
/* The same pass over one ROW SEGMENT of A, continuing the einsum lane state:
 * state_in (2n doubles: acc_0, acc_1 per column; NULL = zeros) is the state
 * after the rows above this segment; a non-final segment (last = 0, m a
 * multiple of 8) writes the state after its rows to state_out, the final
 * one adds the tail and writes norms2.  The row-sharded engine hands the
 * state from rank to rank (parallel.py), so sharded norms equal the
 * single-GPU (and numpy) ones bit for bit.  nonfinite is OR-ed, not reset. */
int pod_colnorms2_chain(int atype, const void* A, int64_t m, int64_t n, int64_t lda,
                        const double* state_in, double* state_out, int last, double* norms2,
                        int32_t* nonfinite, void* stream);

/* Inverse-CDF draw with replacement + unique/counts + retirement.
 * Replaces sampling.py:204-222 (sample_with_replacement) together with the
 * distribution it samples -- mode 0: l2n over live columns, weights =
 * raw norms2 normalised as sampling.py:55-65,34-53; mode 1: uniform over
 * live columns (sampling.py:150-155); mode 2: explicit normalised weights
 * over positions 0..n-1 (a Distribution's weights, no live mask); mode 3:
 * "ort" -- raw squared residuals over live columns, falling back to uniform
 * when their sum <= thr (isma.py:216-220); mode 4: row draw -- raw weights
 * over all positions normalised as mode 0, no live mask, no retirement,
 * p_out (nullable) = normalised weight of each drawn position -- and the
 * candidate-set update isma.py:164 (drawn columns cleared in `live`).
 * `uniforms` holds the c variates of ONE rng.random(c) batch.
 * Outputs: idx_out[0..g) ascending int32 (idx_out[g..cap) = -1: zero-column
 * padding for the gathered GEMMs), cnt_out[0..g) int64,
 * info[0] = g, info[1] = |S| after the draw, info[2] = status
 * (0 ok, 1 empty S, 2 all weights zero -> DegenerateDistributionError).
 * Every mode reproduces numpy's arithmetic exactly (pod_draw_exact), so the
 * index sets equal the reference's by construction given equal weights. */
size_t pod_draw_ws_bytes(int64_t n);
int pod_draw(int mode, const double* weights, uint8_t* live, int64_t n, const double* uniforms,
             int64_t c, int32_t* idx_out, int64_t* cnt_out, int64_t cap, void* ws,
             size_t ws_bytes, int64_t* info, double thr, double* p_out, void* stream);

/* Column draw of modes 0-3 in numpy's exact summation order: the candidate
 * set compacted in ascending order (setdiff1d), the from_weights total and
 * the __post_init__ renormalisation as numpy pairwise sums (sampling.py:47-50,
 * 62-65; blocks of <= 128 with 8 accumulators, split at n/2 rounded down to
 * a multiple of 8), np.cumsum as a sequential running sum (sampling.py:214),
 * the pin, searchsorted(side="right") and np.unique (sampling.py:215-221).
 * Same outputs and modes as pod_draw (mode 4: the row draw, p_out = the
 * drawn positions' normalised weights). */
size_t pod_draw_exact_ws_bytes(int64_t n);
int pod_draw_exact(int mode, const double* weights, uint8_t* live, int64_t n,
                   const double* uniforms, int64_t c, int32_t* idx_out, int64_t* cnt_out,
                   int64_t cap, void* ws, size_t ws_bytes, int64_t* info, double thr,
                   double* p_out, void* stream);

/* Row sampling (ICRS) building blocks, isma.py:168-176:
 * out[i] = (sum_j X[i, cols[j]]^2) / div (div = *div_dev when non-null) --
 * row_norm_distribution of the sampled block (sampling.py:143-147, div 1) or
 * leverage scores of the top-k basis (sampling.py:190-201, div k); and the dedup-scaled row block
 * Y[i, :] = A[rows[i], cols] sqrt(cnt[i] / (w p[i])) (scale_sampled_rows,
 * sampling.py:248-258) for i < *hdev. */
int pod_rownorms2(int xtype, const void* X, int64_t m, int64_t ncols, int64_t ldx,
                  const int32_t* cols, double div, const double* div_dev, double* out,
                  void* stream);
int pod_gather_scale_rows(int atype, const void* A, int64_t lda, const int32_t* cols, int64_t g,
                          const int32_t* rows, const int64_t* cnt, const double* p, double w,
                          int64_t hcap, const int64_t* hdev, double* Y, int64_t ldy,
                          void* stream);

/* Squared residual norms after projection on an orthonormal basis:
 * out[j] = ||A[:, cols[j]] - U C[:, j]||^2 with C = U^T A[:, cols] (r x n,
 * from pod_gemm_tn_f64), U m x r.  The residual is never materialised.
 * Replaces sampling.py:175-176 (residual_distribution, strategy "ort"). */
size_t pod_resid_ws_bytes(int64_t m, int64_t n);
int pod_resid_colnorms2(int atype, int64_t m, int64_t n, const void* A, int64_t lda,
                        const int32_t* cols, const double* U, int64_t ldu, int64_t r,
                        const double* C, int64_t ldc, double* out, void* ws, size_t ws_bytes,
                        void* stream);

/* Fused Wedin residuals (one pass over A): out2[0] = ||A V - U diag(sigma)||_F^2,
 * out2[1] = ||A^T U - V diag(sigma)||_F^2 for U m x k, V n x k, 1 <= k <= 64.
 * Each A tile feeds both FP64 DMMA products from shared memory; R stays in
 * registers, S is reduced across a thread-block cluster (DSMEM) into row-range
 * partials.  Deterministic.  Replaces quality.py:104-107 (r, s and their
 * np.linalg.norm in wedin_measure). */
size_t pod_wedin_ws_bytes(int64_t m, int64_t n, int64_t k);
int pod_wedin_residuals(int atype, const void* A, int64_t m, int64_t n, int64_t lda,
                        const double* U, int64_t ldu, const double* V, int64_t ldv,
                        const double* sigma, int64_t k, double* out2, void* ws,
                        size_t ws_bytes, void* stream);

/* Gates: every compute entry point below that takes `gate` (device int32,
 * nullable) does nothing when *gate == 0, so a round's launch sequence is
 * static (capturable in a CUDA graph) while data-dependent branches of the
 * reference -- extra CholeskyQR passes, the merge.py:73 second projection --
 * are decided on the device.  Column index -1 in a gather list denotes a
 * zero column (capacity padding of the sampled block).
 *
 * C (p x q) = alpha X^T Y, X m x p, Y m x q, K = m split across CTAs with
 * a fixed-order reduction (deterministic).  FP64 DMMA.8x8x4.
 * Replaces: baselines.py:43 (D^T D), merge.py:65 (U1^T U2), merge.py:72/75
 * (U1^T Q), isma.py:296 (A^T U), quality.py:104-105 partial products. */
size_t pod_gemm_tn_ws_bytes(int64_t m, int64_t p, int64_t q);
int pod_gemm_tn_f64(int64_t m, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx,
                    const int32_t* xcols, const double* Y, int64_t ldy, const int32_t* ycols,
                    double* C, int64_t ldc, void* ws, size_t ws_bytes, const int32_t* gate,
                    void* stream);
/* Typed operands: X and Y each stored as POD_F64 or POD_F32, exact fp64
 * arithmetic on the upcast values; C fp64. */
int pod_gemm_tn(int xtype, int ytype, int64_t m, int64_t p, int64_t q, double alpha,
                const void* X, int64_t ldx, const int32_t* xcols, const void* Y, int64_t ldy,
                const int32_t* ycols, double* C, int64_t ldc, void* ws, size_t ws_bytes,
                const int32_t* gate, void* stream);

/* Y (m x q) = alpha X T + beta Z, X m x p (optionally column-gathered),
 * T p x q small, q <= 192.  FP64 DMMA.8x8x4.  One CTA owns all q output
 * columns of its rows, so Y may alias X or Z (in-place updates).
 * Replaces: baselines.py:62-63 (D V / sigma), merge.py:69 (U2 - U1 M),
 * merge.py:86-88 ([U1 Q] U_E), isma.py:298-299 (U V_R, Q U_R). */
int pod_gemm_nn_f64(int64_t m, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx,
                    const int32_t* xcols, const double* T, int64_t ldt, double beta,
                    const double* Z, int64_t ldz, double* Y, int64_t ldy, const int32_t* gate,
                    void* stream);
/* Typed X (POD_F64 or POD_F32 storage, exact fp64 arithmetic); T, Z, Y fp64. */
/* Y = alpha X T (pod_gemm_nn_f64, streamed kernel, no gather, Y not aliasing
 * X) that also returns dots[j] = sum_i Y[i, j] X[i, j] for j < kdot, formed
 * in the GEMM's epilogue from the stored values (fixed-order reduction).
 * With X = [U_old Q] and Y = U_new = X U_E these are the raw convergence
 * cosines u_old_j . u_new_j of isma.py:195-198 (criterion "modes"): the
 * rotation and the cosine pass become one pass.  gate must be NULL. */
size_t pod_gemm_nn_dots_ws_bytes(int64_t kdot);
int pod_gemm_nn_dots(int64_t m, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx,
                     const double* T, int64_t ldt, double* Y, int64_t ldy, int64_t kdot,
                     double* dots, void* ws, size_t ws_bytes, const int32_t* gate, void* stream);

/* pod_gemm_nn_f64 (no gather) that also returns G (q x q) = Y^T Y, formed
 * from each output tile while it is on chip (fixed-order split reduction,
 * exactly symmetric): the Gram of the block a CholeskyQR pass consumes next,
 * without a TN pass over it.  Shapes with pod_gemm_nn_gram_ok(p, q) only
 * (q <= 64, p >= q, T resident in shared memory).  Replaces the Gram of
 * merge.py:70 (QR of the residual U2 - U1 M) and of the second CholeskyQR
 * pass. */
int pod_gemm_nn_gram_ok(int64_t p, int64_t q);
size_t pod_gemm_nn_gram_ws_bytes(int64_t m, int64_t q);
int pod_gemm_nn_gram(int64_t m, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx,
                     const double* T, int64_t ldt, double beta, const double* Z, int64_t ldz,
                     double* Y, int64_t ldy, double* G, int64_t ldg, void* ws, size_t ws_bytes,
                     const int32_t* gate, void* stream);
int pod_gemm_nn(int xtype, int64_t m, int64_t p, int64_t q, double alpha, const void* X,
                int64_t ldx, const int32_t* xcols, const double* T, int64_t ldt, double beta,
                const double* Z, int64_t ldz, double* Y, int64_t ldy, const int32_t* gate,
                void* stream);

/* Page-lock and map a host buffer for direct kernel access (host-resident,
 * streamed matrices; the device address is the host address under UVA,
 * checked), and release it. */
int pod_host_register(void* ptr, size_t bytes);
int pod_host_unregister(void* ptr);

/* D[:, j] = A[:, idx[j]] for j < g (idx -1: zero column; idx NULL: j).  A
 * may be page-locked host memory mapped into the device address space (a
 * host-resident, streamed matrix): one PCIe read of the sampled block per
 * round (isma.py:163), the round's GEMMs then read D from HBM. */
int pod_gather_cols(int atype, const void* A, int64_t m, int64_t lda, const int32_t* idx,
                    int64_t g, void* D, int64_t ldd, void* stream);

/* D[:, j] = A[:, idx[j]] * f[j] in fp64 (int64 indices; the materialised,
 * scaled sample of scale_sampled_columns, sampling.py:234-245, used by the
 * single-round baselines ltsvd / ctsvd, baselines.py:68-142). */
int pod_gather_scale_cols(int atype, const void* A, int64_t m, int64_t lda, const int64_t* idx,
                          const double* f, int64_t g, double* D, int64_t ldd, void* stream);

/* Cap (in CTAs; 0 = none) on the grids of the TN / NN GEMMs launched while
 * set -- host-side state read at launch (and so baked into captured graphs):
 * the pipelined next-round update runs capped beside the critical merge. */
int pod_set_grid_cap(int ctas);

/* Workspace (bytes) sufficient for a Gram eigensolve (g = n), a CholeskyQR
 * factor (l = n) or a merge core (l1 + l2 = n) -- including the block sets
 * of the grid-wide Jacobi solver that takes sizes beyond one cluster. */
size_t pod_small_ws_bytes(int64_t n);

/* Largest Gram order g pod_gram_eigh accepts. */
int64_t pod_gram_eigh_max_g(void);

/* Workspace (bytes) for pod_svd_small of an nr x nc block (V wanted iff
 * withv): the grid-wide solver's block sets, used only when the cluster
 * solvers do not fit; 0 when the grid solver does not fit either. */
size_t pod_svd_small_ws_bytes(int64_t nr, int64_t nc, int withv);

/* gram_spectrum + lift setup (baselines.py:35-65): eigen-decomposition of
 * the PSD Gram G (g x g), descending, eigenvalue dust <= 1e-12 lambda_1
 * zeroed (matcore.py:26), sigma = sqrt(lambda) into sigma[0..g);
 * rank = #sigma > 1e-14 sigma_1 (matcore.py:20), keep = min(r, rank);
 * T (g x r, ld ldt) = V[:, :keep] / sigma[:keep], zero columns beyond keep.
 * info[0] = rank, info[1] = keep, info[2] = Jacobi sweeps. */
int pod_gram_eigh(const double* G, int64_t ldg, int64_t g, int64_t r, double* sigma, double* T,
                  int64_t ldt, int64_t* info, void* ws, size_t ws_bytes, void* stream);

/* One CholeskyQR pass from the Gram G = W^T W (l x l) of an nrows x l
 * block: R (upper) and Rinv such that Q = W Rinv has orthonormal columns
 * and W = Q R.  Column-scaled, shifted on breakdown, exactly-zero columns
 * dropped (zero R rows).  Replaces the Householder QR of merge.py:70,76 and
 * matcore.py:209.  dinfo[0] = max |D^-1 G D^-1 - I| (input defect),
 * dinfo[1] = shift attempts, dinfo[2] = dropped columns, dinfo[3] = shift;
 * dinfo[POD_DINFO_BREAKDOWN] is SET to 1 (never cleared here) when every
 * shifted retry broke down -- the factor is then unusable and the caller
 * must raise (the engine checks it with each round's record).
 * Runs iff gate_in is null or *gate_in != 0; gate_out (nullable) receives
 * whether ANOTHER pass is needed: 1 after a first pass, else
 * (ran && (defect > 1e-4 || shifted)). */
int pod_cholqr_factor(const double* G, int64_t ldg, int64_t l, int64_t nrows, double* Rinv,
                      int64_t ldri, double* R, int64_t ldr, double* dinfo, void* ws,
                      size_t ws_bytes, const int32_t* gate_in, int32_t* gate_out, int first_pass,
                      void* stream);

/* pod_cholqr_factor with an optional accumulated factor: when Racc is not
 * null, Racc <- R Racc in place (the CholeskyQR passes' running R,
 * merge.py:70 / matcore.py:209); R itself may then be null for l <= 64. */
int pod_cholqr_factor2(const double* G, int64_t ldg, int64_t l, int64_t nrows, double* Rinv,
                       int64_t ldri, double* R, int64_t ldr, double* Racc, int64_t ldacc,
                       double* dinfo, void* ws, size_t ws_bytes, const int32_t* gate_in,
                       int32_t* gate_out, int first_pass, void* stream);

/* Merge core (merge.py:80-88): E = [[diag sig1, M diag sig2],[0, R diag sig2]],
 * its SVD, keep = min(r, #sigma_E > 1e-14 max(sigma_E0, 1e-300)), and the
 * rotation T ((rcap + l2) x tcols, ld ldt) mapping the stacked basis
 * [U1 | 0-pad to rcap | Q] onto the merged left vectors.  info[0] = keep,
 * info[1] = Jacobi sweeps; sig_new[0..rcap) = merged sigma, zero beyond keep. */
int pod_merge_core(const double* sig1, int64_t l1, const double* M, int64_t ldm, const double* R,
                   int64_t ldr, const double* sig2, int64_t l2, int64_t r, int64_t rcap, double* T,
                   int64_t ldt, int64_t tcols, double* sig_new, int64_t* info, void* ws,
                   size_t ws_bytes, void* stream);

/* Whether pod_merge_core handles l1 + l2 with a single-cluster solver (block
 * or cluster Jacobi, no workspace) -- the sizes pod_merge_core_gated takes. */
int pod_merge_core_gatable(int64_t l1, int64_t l2);

/* pod_merge_core with a device gate: *gate == 0 makes the launch a no-op.
 * The ISMA engine runs the merge core speculatively on the first-pass R
 * while the leak check of merge.py:72-79 is in flight, and re-runs it gated
 * on that check (the re-run only does work when the second projection
 * fired).  Sizes must satisfy pod_merge_core_gatable. */
int pod_merge_core_gated(const double* sig1, int64_t l1, const double* M, int64_t ldm,
                         const double* R, int64_t ldr, const double* sig2, int64_t l2, int64_t r,
                         int64_t rcap, double* T, int64_t ldt, int64_t tcols, double* sig_new,
                         int64_t* info, const int32_t* gate, void* stream);

/* Thin SVD of a small nr x nc matrix (nr >= nc) by one-sided Jacobi:
 * sigma descending; if U and V are non-null, U (nr x nc) and V (nc x nc)
 * with A = U diag(sigma) V^T.  Replaces matcore.py:178-184 (_svd) at
 * isma.py:297 and np.linalg.svd at isma.py:198 / quality.py:56. */
int pod_svd_small(const double* A, int64_t lda, int64_t nr, int64_t nc, double* U, int64_t ldu,
                  double* sigma, double* V, int64_t ldv, int64_t* info, void* ws, size_t ws_bytes,
                  void* stream);

/* C (p x q) = alpha op(A) B + beta C for small matrices (op = A or A^T).
 * C must not alias A or B. */
int pod_small_gemm(int64_t p, int64_t q, int64_t k, double alpha, const double* A, int64_t lda,
                   int transa, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                   const int32_t* gate, void* stream);

/* Copy a p x q block (ld_src -> ld_dst), gated. */
int pod_small_copy(int64_t p, int64_t q, const double* src, int64_t lds, double* dst, int64_t ldd,
                   const int32_t* gate, void* stream);

/* out[0] = max |A| over a p x q block and gate_out = (max > thr)
 * (merge.py:72 leak test with thr = 1e-8). */
int pod_maxabs(const double* A, int64_t lda, int64_t p, int64_t q, double thr, double* out,
               int32_t* gate_out, void* stream);

/* fix_signs (matcore.py:148-165): per column, the first entry of largest
 * magnitude is made positive; V (n x l) flipped alongside when non-null.
 * sign_out (l, optional) receives the +-1 factors. */
size_t pod_colwise_ws_bytes(int64_t m, int64_t l);
int pod_fix_signs(double* U, int64_t m, int64_t l, int64_t ldu, double* V, int64_t n, int64_t ldv,
                  double* sign_out, void* ws, size_t ws_bytes, void* stream);

/* Row-shard building blocks of fix_signs: per column the max |U| over this
 * shard, its GLOBAL row (local + row_offset; first occurrence on ties) and
 * the sign of that entry; and U[:, j] *= sign[j] (sign = +-1). */
int pod_colargmax(const double* U, int64_t m, int64_t l, int64_t ldu, int64_t row_offset,
                  double* val_out, int64_t* row_out, double* sign_out, void* ws, size_t ws_bytes,
                  void* stream);
int pod_scale_cols(double* U, int64_t m, int64_t l, int64_t ldu, const double* sign, void* stream);

/* out[j] = sum_i P[i, j] Q[i, j] for j < kk, 0 for kk <= j < k; with
 * take_abs the |.| clipped to [0, 1] (convergence cosines, isma.py:195-201). */
int pod_coldots(const double* P, int64_t ldp, const double* Q, int64_t ldq, int64_t m, int64_t k,
                int64_t kk, int take_abs, double* out, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PODSKETCH_B200_H */
