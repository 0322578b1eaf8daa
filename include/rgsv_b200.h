/*
 * rgsv_b200 — C-ABI of the B200 (sm_100a) randomized-GSVD hot path.
 *
 * This is the drop-in boundary for the reference package rgsv 0.1.0, whose
 * hot path is pure Python over numpy/LAPACK and therefore has no FFI of its
 * own. Each entry point below replaces one reference
 * stage; the citation names the reference code it stands in for
 * (paths under /root/reference/pkg/src/rgsv/). The Python host layer
 * (paper_2404_09459_b200/, loaded with ctypes) rebuilds the reference's
 * dataclasses around these calls; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - All matrices are row-major FP64 in DEVICE memory; ld* are row strides
 *     in elements and must be even (TMA needs 16-byte row pitch).
 *   - kp = k rounded up to a multiple of 16; padded rows/columns are zero
 *     on output and must be zero on input.
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     asynchronous on it. Return codes report argument/launch errors;
 *     numerical failures detected on the device are OR-ed into the caller's
 *     device `status` word (RGSV_ST_* bits) and read back with the results.
 *   - Results are bitwise deterministic for fixed inputs (fixed-order
 *     reductions, no floating-point atomics).
 */
#ifndef RGSV_B200_H
#define RGSV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes, mapped 1:1 onto the reference exceptions (errors.py:5-56) */
#define RGSV_OK 0
#define RGSV_ERR_DIMENSION 1   /* DimensionError */
#define RGSV_ERR_VALIDATION 2  /* ValidationError */
#define RGSV_ERR_RANK 3        /* RankDeficiencyError */
#define RGSV_ERR_CONVERGENCE 4 /* ConvergenceError */
#define RGSV_ERR_CUDA 5        /* launch/driver failure (RuntimeError) */
#define RGSV_ERR_WORKSPACE 6   /* workspace too small (internal) */
#define RGSV_ERR_DEGENERATE 7  /* DegenerateSpectrumError */

/* device status bits */
#define RGSV_ST_CHOL_BREAKDOWN 0x1  /* nonpositive Cholesky pivot */
#define RGSV_ST_NONFINITE 0x2       /* NaN/Inf in G (core.py:55) */
#define RGSV_ST_JACOBI 0x4          /* Jacobi SVD did not converge (core.py:102-105) */
#define RGSV_ST_CLASSIFY 0x8        /* overlapping zero classes (engine.py:179-180) */
#define RGSV_ST_DEGENERATE 0x10     /* vanishing alpha/beta energy (analysis.py:58-59) */
#define RGSV_ST_NOT_NORMALIZED 0x20 /* |sum p - 1| > 1e-10 (analysis.py:74-75) */
#define RGSV_ST_OMEGA_SHORT 0x40    /* Omega generator ran out of raw draws (never expected) */
#define RGSV_ST_SPECTRUM 0x80       /* GsvSpectrum invariant violated (engine.py:108-125; batch path) */

const char* rgsv_version(void);

/* Number of kernels this library has launched so far in the process
 * (bench.py reports the delta over its timed region as gpu_launches). */
long long rgsv_launch_count(void);

/* Compute capability (major*10+minor) of the current device, or -1. */
int rgsv_device_cc(void);

/* --- Omega: the reference's Gaussian test matrices, generated on the device
 * Bit-identical to numpy 2.3.5 `default_rng(seed).standard_normal((n, k))`
 * (rangefinder.py:101,112 / core.py:60-76): SeedSequence -> PCG64 ->
 * 256-layer ziggurat, reproduced in parallel. Writes Omega^T: stream s's
 * value Omega[i][j] goes to out[s * out_stride + j * ldo + i]. `seeds` is a
 * DEVICE array of nstreams uint64 seeds (already masked to 64 bits). */
size_t rgsv_omega_workspace_bytes(int nstreams, int64_t n, int k);
int rgsv_omega_generate(const uint64_t* seeds, int nstreams, int64_t n, int k, double* out,
                        int64_t ldo, int64_t out_stride, int* status, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Omega block drawn from the running stream after skipping `offset` normals
 * (the adaptive range finder draws block i right after blocks 0..i-1 from ONE
 * generator, rangefinder.py:101,112). */
size_t rgsv_omega_workspace_bytes_at(int nstreams, int64_t n, int k, int64_t offset);
int rgsv_omega_generate_at(const uint64_t* seeds, int nstreams, int64_t n, int k, int64_t offset,
                           double* out, int64_t ldo, int64_t out_stride, int* status,
                           void* workspace, size_t workspace_bytes, void* stream);

/* Robust reduced QR of a tall block a (m x w, in place) by Householder in one
 * CTA: q (m x min(m,w)), rdiag = |diag R| with the core.py:88-95 phase fix
 * (diag R >= 0), tau (min(m,w)) scratch. Rank deficiency is allowed (R_jj = 0),
 * like LAPACK dgeqr2 -- the adaptive range finder's trim test
 * (rangefinder.py:120-121) reads rdiag. */
int rgsv_householder_qr(double* a, int64_t lda, int m, int w, double* q, int64_t ldq,
                        double* rdiag, double* tau, void* stream);
/* --- batched small pairs ----------------------------
 * compute_gsv + compare for npairs independent same-k pairs in ~6 launches:
 * Omega for every matrix (seeds[2j], seeds[2j+1] -- the reference draws G2's
 * Omega from seed + 1, engine.py:252-253), one cluster-per-matrix fused
 * chain kernel (sketch, shifted CholeskyQR3 in shared memory, q power
 * iterations, projection B = Q^T G), then one CTA per pair for the stacked
 * QR + Jacobi + comparative stage. mats: device array of 2*npairs
 * descriptors {G1_0, G2_0, G1_1, ...}; n <= 128, k <= 32, 2k <= n.
 * Per pair outputs: res[j*(6n+4+2k)] = {alphas, betas, rho, theta, p1, p2,
 * scalars[4] (d1, d2, sum p1, sum p2), sv1[k], sv2[k]}; ints[4j] = {nsv1,
 * nsv2, r, s}; stats[4j] = {|G1|^2, |B1|^2, |G2|^2, |B2|^2}; status[j].
 * b_out (optional, else workspace): the projections B of every matrix,
 * 2*npairs blocks of kp x ceil16(n) (kp = 16 or 32), rows >= k zero. */
typedef struct {
  const double* g;
  int64_t ld;
  int32_t rows;
  int32_t pad;
} rgsv_matrix_desc;
/* 1 when rgsv_batch_gsvd serves this shape (the per-CTA Y slice of the
 * largest matrix fits shared memory in a cluster of <= 8 CTAs), else 0. */
int rgsv_batch_supported(int max_rows, int64_t n, int k);
size_t rgsv_batch_workspace_bytes(int npairs, int64_t n, int k);
/* Diagnostic: per-phase clock64 totals of the batched chain kernel (16
 * counters), only in a library built with -DRGSV_BATCH_PROFILE
 * (tools/batch_phases.py); RGSV_ERR_VALIDATION otherwise. */
int rgsv_debug_batch_profile(unsigned long long* out16, int reset);
int rgsv_batch_gsvd(const void* mats, int npairs, int max_rows, int64_t n, int k, int q,
                    const uint64_t* seeds, double classify_tol, double* res, int* ints,
                    double* stats, int* status, double* b_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/* --- recover_gsvd building blocks (engine.py:278-362) ------------------- */
/* Orthonormal completion (engine.py:278-291): `count` orthonormal columns
 * orthogonal to the `have` orthonormal columns of a (dim x have, overwritten
 * by its Householder factorization) -- columns have..have+count of the
 * complete Q, like numpy.linalg.qr(mode="complete"). out: dim x count. */
int rgsv_orth_complete(double* a, int64_t lda, int dim, int have, int count, double* out,
                       int64_t ldo, double* rdiag, double* tau, void* stream);
/* One-sided Jacobi SVD with vectors of the nv rows of v (nv x len, in
 * place): acc (nv x nv) scratch, sv[nv] sorted (descending, or ascending),
 * xn (nv x len) unit singular rows, jo (nv x nv) the matching rotation rows;
 * A (rows as vectors) = jo^T diag(sv) xn. *nzero = exactly-zero values
 * (their xn rows are 0; the caller completes them). Replaces the full SVDs
 * np.linalg.svd(L, full_matrices=True) of engine.py:322,340. */
int rgsv_svd_vectors(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                     double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj, int ascending,
                     int* nzero, int* status, void* stream);
/* rgsv_svd_vectors on many CTAs (blocked one-sided Jacobi with the 32 x 32
 * block rotations accumulated into acc; nv <= len, nv up to 25600): same
 * outputs. workspace >= rgsv_svd_vectors_blocked_workspace_bytes(nv). */
size_t rgsv_svd_vectors_blocked_workspace_bytes(int nv);
int rgsv_svd_vectors_blocked(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                             double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj,
                             int ascending, int* nzero, int* status, void* workspace,
                             size_t workspace_bytes, void* stream);
/* dst (cols x rows) = src^T, src rows x cols. */
int rgsv_transpose(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols,
                   void* stream);
/* dst (rows x cols, fp64) = src (fp32), exact promotion of a row block --
 * the reference promotes fp32 input to fp64 (core.py:51-54); the cfg4
 * pipeline streams fp32 G through this in row chunks instead of holding a
 * 118 GB fp64 copy. */
int rgsv_convert_f32(const float* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
                     int64_t ldd, void* stream);
/* a[:, j] /= d[j] for j < cols (engine.py:335,357). */
int rgsv_scale_cols(double* a, int64_t lda, int rows, int cols, const double* d, void* stream);

/* y (rows x cols) += alpha * x (re-projection of rangefinder.py:116-118). */
int rgsv_axpy(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols,
              double alpha, void* stream);

/* --- (1)-(3) range finder + projection for ONE matrix -------------------
 * Replaces rangefinder.extract_basis in fixed-rank mode (one block of
 * width k: rangefinder.py:106-133 with blocksize = max_cols = k,
 * trim_tol = 0) followed by q power iterations (not in the reference,
 * SURVEY.md §0 F1) and the projection c = Q^H G (engine.py:255-256).
 *   Y = G Omega; Q = qr(Y).q; q x { Qhat = qr(G^T Q).q; Q = qr(G Qhat).q };
 *   B = Q^T G.
 * Inputs : g (m x n, ldg), omega_t = Omega^T (kp x n, ld_omega; rows >= k zero).
 * Outputs: q_out (m x kp, ld kp), b_out (kp x n, ldb),
 *          stats[0] = ||G||_F^2 (rangefinder.py:83), stats[1] = ||B||_F^2
 *          (the captured energy of rangefinder.py:123),
 *          rdiag[k] = |diag R| of the final QR (the trim test, :120).
 * QR is shifted CholeskyQR3 (R diagonal > 0: the core.py:88-95 phase
 * convention). */
size_t rgsv_sketch_workspace_bytes(int64_t m, int64_t n, int k);
int rgsv_sketch_project(const double* g, int64_t ldg, int64_t m, int64_t n,
                        const double* omega_t, int64_t ld_omega, int k, int q, double* q_out,
                        double* b_out, int64_t ldb, double* stats, double* rdiag, int* status,
                        void* workspace, size_t workspace_bytes, void* stream);

/* --- (1)-(3) for ONE ROW SHARD of a matrix (multi-GPU) ---
 * The same chain as rgsv_sketch_project on this rank's contiguous row block
 * g (m_local x n) of a matrix with m_total rows in all. Every cross-rank sum
 * goes through `allreduce` (in-stream, on `stream`): ||G||_F^2 (1 value),
 * each tall CholeskyQR pass's k x k Gram (kp*kp values), every power step's
 * Z^T = Q^T G (kp*ldb values) and the projection B (kp*ldb values). The
 * shifted CholeskyQR uses m_total; the wide QR of Z runs redundantly on
 * every rank; Q stays row-sharded (q_out: m_local x kp); B, stats and rdiag
 * come out replicated. Pass rgsv_nccl_allreduce with an NCCL communicator
 * as ctx (below), or any function with this signature (a gloo/MPI wrapper);
 * allreduce == NULL requires m_local == m_total (single rank).
 * Replaces, per rank, the Y = G Omega / Q^H G products of
 * rangefinder.py:115,123 and engine.py:255-256. */
typedef int (*rgsv_allreduce_fn)(double* buf, int64_t count, void* stream, void* ctx);
int rgsv_sketch_project_sharded(const double* g, int64_t ldg, int64_t m_local, int64_t m_total,
                                int64_t n, const double* omega_t, int64_t ld_omega, int k, int q,
                                double* q_out, double* b_out, int64_t ldb, double* stats,
                                double* rdiag, int* status, rgsv_allreduce_fn allreduce,
                                void* allreduce_ctx, void* workspace, size_t workspace_bytes,
                                void* stream);

/* NCCL (over NVLink / NVSwitch) for the sharded chain, resolved at run time
 * from the libnccl.so.2 the host process loaded (no link-time dependency).
 * rgsv_nccl_version: NCCL_VERSION code, -1 when NCCL is not loadable.
 * get_unique_id fills 128 bytes on one rank; every rank passes them to
 * comm_init. rgsv_nccl_allreduce has the rgsv_allreduce_fn signature, ctx = comm:
 * in-place fp64 sum. rgsv_nccl_broadcast: `bytes` bytes from `root`. */
int rgsv_nccl_version(void);
int rgsv_nccl_get_unique_id(void* id_out);
int rgsv_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank);
int rgsv_nccl_comm_destroy(void* comm);
int rgsv_nccl_allreduce(double* buf, int64_t count, void* stream, void* comm);
int rgsv_nccl_broadcast(void* buf, int64_t bytes, int root, void* stream, void* comm);

/* --- (4) small GSVD -------------------------------------------------------
 * Replaces engine.py:257-261 (reduced_qr of vstack(c1, c2), L blocks) and
 * engine._singular_values (engine.py:228-231) for the two L blocks:
 * sv1 (min(l1, r) values, descending), sv2 (min(l2, r)), r = rank dim of
 * the stacked QR = min(l1 + l2, n). nsv[0..1] receive the counts.
 * One-sided Jacobi SVD; non-convergence sets RGSV_ST_JACOBI. */
size_t rgsv_small_gsvd_workspace_bytes(int l1, int l2, int64_t n);
int rgsv_small_gsvd(const double* b1, int64_t ldb1, int l1, const double* b2, int64_t ldb2, int l2,
                    int64_t n, double* sv1, double* sv2, int* nsv, int* status, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Householder QR (LAPACK dgeqrf + dorgqr semantics) of the M x N matrix
 * stacked from [a1 (m1 rows); a2 (m2 rows)] (a2 may be NULL with m2 = 0),
 * M = m1 + m2 <= 1408: q (M x K) and r (K x N, upper trapezoid; may be
 * NULL), K = min(M, N), with the phase fix diag(R) >= 0 when phase_fix != 0.
 * Replaces core.reduced_qr (core.py:79-96: numpy.linalg.qr + sign fix),
 * tall AND wide, and the stacked QR of engine.py:257. Many CTAs, one
 * cooperative launch. */
size_t rgsv_dense_qr_workspace_bytes(int M, int N);
int rgsv_dense_qr(const double* a1, int64_t lda1, int m1, const double* a2, int64_t lda2,
                  int m2, int N, double* q, int64_t ldq, double* r, int64_t ldr, int phase_fix,
                  void* workspace, size_t workspace_bytes, void* stream);

/* --- (5) spectrum + comparative quantities -------------------------------
 * Replaces engine.spectrum_from_l_blocks (engine.py:189-225, merged
 * completion), classify_spectrum (engine.py:164-186) and analysis.py:37-79
 * (rho, theta, P1, P2, D1, D2) in one kernel.
 * counts[0] = r, counts[1] = s; scalars = {d1, d2, sum p1, sum p2}. */
int rgsv_comparative(const double* sv1, const int* nsv, const double* sv2, int64_t n,
                     double classify_tol, double* alphas, double* betas, double* rho,
                     double* theta, double* p1, double* p2, double* scalars, int* counts,
                     int* status, void* stream);

/* engine.spectrum_from_l_blocks (engine.py:189-225) on given L blocks:
 * singular values of L1 (l1 x cols) and L2 (l2 x cols) by one-sided
 * Jacobi, then the completion -- branch 0 = merged (default), 1 = "first"
 * (betas from the alphas, L2 unused), 2 = "second" -- and
 * classify_spectrum (engine.py:164-186): alphas, betas (n), counts = {r, s}.
 * status: RGSV_ST_JACOBI / RGSV_ST_CLASSIFY as in rgsv_small_gsvd (the
 * DEGENERATE / NOT_NORMALIZED bits of the comparative stage are
 * informational here). */
size_t rgsv_spectrum_from_l_blocks_workspace_bytes(int l1, int l2, int cols, int64_t n);
int rgsv_spectrum_from_l_blocks(const double* l1b, int64_t ld1, int l1, const double* l2b,
                                int64_t ld2, int l2, int cols, int64_t n, double classify_tol,
                                int branch, double* alphas, double* betas, int* counts,
                                int* status, void* workspace, size_t workspace_bytes,
                                void* stream);

/* Per-quantity forms of analysis.py:37-79 for a given spectrum (alphas,
 * betas, r): rho (inf for i < r), theta, p1, p2, scalars = {d1, d2, sum p1,
 * sum p2}; and D of a given probability vector (scalars[0] = D,
 * scalars[2] = sum p). */
int rgsv_spectrum_quantities(const double* alphas, const double* betas, int64_t n, int r,
                             double* rho, double* theta, double* p1, double* p2, double* scalars,
                             int* status, void* stream);
int rgsv_entropy(const double* p, int64_t n, double* scalars, void* stream);

/* Singular values (descending, min(rows, cols) of them) of a small dense
 * matrix by one-sided Jacobi: core.svd values (core.py:99-106). nsv[0]
 * receives the count; nsv[1] is scratch. */
size_t rgsv_svd_values_workspace_bytes(int rows, int cols);
int rgsv_svd_values(const double* a, int64_t lda, int rows, int cols, double* sv, int* nsv,
                    int* status, void* workspace, size_t workspace_bytes, void* stream);

/* --- building blocks (row-sharded multi-GPU driver, tests) ---------------
 * gemm_gx : C (M x N) = A (M x K) * Bt^T, Bt given N x K.
 * gemm_gtq: C (M x N) = A^T * B, A: K x M, B: K x N (reduction over rows).
 * chol_inv: Cholesky of a k x k Gram (ld kp) [+ shift for `shift_rows`
 *           rows], Linv = L^{-1}, Rinv = Linv^T (kp x kp, identity pad).
 * sumsq   : out[0] = sum of squares of a rows x cols block. */
/* --- fp32-resident pairs (cfg4): 3xTF32 tcgen05 GEMM passes ------------
 * The reference promotes fp32 input to fp64 up front (core.py:51-54); these
 * entry points instead run the G passes of the fixed-rank chain
 * (rangefinder.py:115, the q power steps, engine.py:255-256) on the
 * tensor cores in kind::tf32 with a hi/lo operand split (fp32-level
 * products, fp32 accumulation, fp64 outputs). Matrices are row-major fp32
 * with ld a multiple of 4 elements and 16-byte aligned bases.
 *
 * rgsv_f32_split: lo = tf32(g - hi(g)) for the big operand (hi(g) = g as the
 * tensor core reads it; mode 0 = low 13 mantissa bits dropped, 1 = nearest)
 * and, if sumsq_out != NULL, ||g||_F^2 in fp64 (core.sum_sq, core.py:115-125).
 * ws: >= 1184 doubles of scratch. */
int rgsv_f32_split(const float* g, int64_t ldg, int64_t rows, int64_t cols, float* lo,
                   int64_t ldl, int mode, double* sumsq_out, void* ws, size_t ws_bytes,
                   void* stream);
/* hi = tf32(x), lo = tf32(x - hi) of an fp64 matrix (rows x cols, ld ldx)
 * into rows x cols_out fp32 arrays (ld ldo), zero in columns >= cols. */
int rgsv_f64_split_tf32(const double* x, int64_t ldx, int64_t rows, int64_t cols, float* hi,
                        float* lo, int64_t ldo, int64_t cols_out, void* stream);
/* Y (M x N, fp64, ld ldy) = G (M x K) X^T, X given as hi/lo (N x K, ld ldx);
 * 32 <= N <= 320, N % 32 == 0. */
int rgsv_tf32x3_gx(const float* g, const float* glo, int64_t ldg, const float* xhi,
                   const float* xlo, int64_t ldx, double* y, int64_t ldy, int64_t M, int64_t N,
                   int64_t K, void* stream);
/* C (N x M, fp64, ld ldc) = Q^T G with Q (K x N, hi/lo, ld ldq) and G
 * (K x M, + lo, ld ldg); 32 <= N <= 320, N % 32 == 0. The K reduction is
 * split over CTAs into fp64 partials in `scratch` (RGSV_ERR_WORKSPACE if
 * too small) and summed in a fixed order. */
int rgsv_tf32x3_gtq(const float* qhi, const float* qlo, int64_t ldq, const float* g,
                    const float* glo, int64_t ldg, double* c, int64_t ldc, int64_t N, int64_t M,
                    int64_t K, void* scratch, size_t scratch_bytes, void* stream);
/* Tuning knobs: K-block of the two kernels (16 or 32; gtq also 8), rows per
 * split of the gtq reduction and K-blocks accumulated in TMEM between fp32
 * register flushes (values out of range are ignored). */
int rgsv_tf32_config(int bk_gx, int bk_gtq, int rows_per_split, int flush);

int rgsv_gemm_gx(const double* a, int64_t lda, const double* bt, int64_t ldb, double* c,
                 int64_t ldc, int64_t M, int64_t N, int64_t K, void* scratch,
                 size_t scratch_bytes, void* stream);
/* Lower triangle (incl. the diagonal) of the Gram C = A^T A (A: rows x
 * cols, row-major, ld lda; C: cols x cols, ld ldc) on the DMMA engine,
 * skipping the output tiles strictly above the diagonal (the CholeskyQR
 * Grams; entries of skipped tiles are left untouched). */
int rgsv_gemm_gram_lower(const double* a, int64_t lda, int64_t cols, int64_t rows, double* c,
                         int64_t ldc, void* scratch, size_t scratch_bytes, void* stream);
int rgsv_gemm_gtq(const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                  int64_t ldc, int64_t M, int64_t N, int64_t K, void* scratch,
                  size_t scratch_bytes, void* stream);
int rgsv_chol_inv(const double* gram, int k, int kp, int64_t shift_rows, double* linv,
                  double* rinv, double* rdiag, int* status, void* stream);
/* Debug: one small Householder QR launch recording clock64() phase stamps. */
/* Debug: rgsv_dense_qr of one M x N matrix with globaltimer stamps (ns) of
 * CTA 0 at each phase boundary in prof[0..254]; prof[255] = stamp count. */
int rgsv_debug_dense_qr_profile(const double* a, int64_t lda, int M, int N, double* q,
                                void* workspace, size_t workspace_bytes, long long* prof,
                                void* stream);
int rgsv_debug_householder_profile(const double* b1, int64_t ld1, int l1, const double* b2,
                                   int64_t ld2, int l2, double* q, int64_t ldq, long long* prof,
                                   void* stream);
/* Debug: one Cholesky launch recording clock64() phase stamps into prof[]. */
int rgsv_debug_chol_profile(const double* gram, int k, int kp, double* linv, long long* prof,
                            int* status, void* stream);
int rgsv_sumsq(const double* a, int64_t lda, int64_t rows, int64_t cols, double* out,
               void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RGSV_B200_H */
