// Internal (C++) interfaces shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/rgsv_b200.h"

namespace rgsv {

// Generic skinny-GEMM launch description (see gemm.cu for the two shapes).
struct GemmArgs {
  const double* A = nullptr;
  int64_t lda = 0;
  const double* B = nullptr;
  int64_t ldb = 0;
  double* C = nullptr;
  int64_t ldc = 0;
  int64_t M = 0, N = 0, K = 0;
  double* scratch = nullptr;  // split-K partials
  size_t scratch_bytes = 0;
  int max_split = 32;
  double* ss_out = nullptr;  // gx only: per-unit sum of squares of A
  int* ss_units = nullptr;
  int live = 0;     // output columns (gx) / rows (gtq) that can be nonzero; 0 = all
  int zero_to = 0;  // internal: padding [N or M, zero_to) stored as zeros
  int lower_only = 0;  // gtq Gram A^T A: only tiles touching the lower triangle
};

int gemm_gx(const GemmArgs& a, cudaStream_t st);
int gemm_gtq(const GemmArgs& a, cudaStream_t st);

// Cholesky of a k x k Gram (row-major, ld kp) with optional shift
// 11 (rows k + k (k+1)) u trace (shifted CholeskyQR, Fukaya et al. 2020);
// writes Linv = L^{-1} (kp x kp, identity padding), optionally its
// transpose Rinv, R = L^T, and the diagonal of R. status[0] |= 1 on breakdown.
// kp <= 128: one CTA; up to kCholMaxKp: blocked (DMMA panels, stream-ordered scratch)
constexpr int kCholMaxKp = 4096;
int chol_inv(const double* gram, int k, int kp, int64_t shift_rows, double* linv, double* rinv,
             double* r_upper, double* rdiag, double* rdiag_acc, int* status, cudaStream_t st);

int chol_profile(const double* gram, int k, int kp, double* linv, long long* prof, int* status,
                 cudaStream_t st);

// batched small-pair chains (batch.cu)
struct BatchMat {
  const double* g;
  int64_t ld;
  int rows;
  int pad;
};
int batch_chain_plan(int max_rows, int n, int k, int* cs_out, int* yrows_out);
int batch_chain(const BatchMat* mats, int nmat, int max_rows, int n, int k, int q,
                const double* omega, int64_t ldo, int64_t om_stride, double* b_out, int64_t ldb,
                int64_t b_stride, double* stats, int* status, int* next, cudaStream_t st);

int launch_batch_small(const double* b, int64_t ldb, int64_t b_stride, int npairs, int k1, int k2,
                       int n, double tol, double* res, int64_t res_stride, int* ints,
                       int* status, const int* mat_status, cudaStream_t st);

size_t omega_workspace_bytes(int nstreams, int64_t nvals);
int omega_generate(const uint64_t* seeds, int nstreams, int64_t n, int k, double* out,
                   int64_t ldo, int64_t out_stride, int* status, void* ws, size_t ws_bytes,
                   cudaStream_t st, int64_t offset = 0);

struct Workspace {
  char* base;
  size_t bytes;
  size_t used;
  void* take(size_t n) {
    size_t off = (used + 255) & ~size_t(255);
    if (off + n > bytes) return nullptr;
    used = off + n;
    return base + off;
  }
};

// Shifted CholeskyQR3 of a tall row-major m x kp block (k real columns,
// zero padding). Input y is overwritten; the orthonormal factor is returned
// in *q_out (one of y / tmp). rdiag (k) receives diag(R).
// `passes` = 3 gives shifted CholeskyQR3 (orthonormal Q); 1 gives one shifted
// pass, Y R1^{-1}: a triangular transform of Y, enough for intermediate bases
// whose span (and nested leading spans) is all that is used downstream.
// Row-sharded use: `red` all-reduces each pass's Gram partial over the
// ranks (Y is this rank's row block) and `shift_rows` is the global row
// count of the shift (defaults to m). `shifted_passes` > 1 shifts that many
// leading passes: with passes = 4 and two shifted passes the factorisation
// survives cond(Y) up to ~1/u (the unshifted second pass of CholeskyQR3
// needs cond(Q1)^2 n u < 1, i.e. cond(Y) <~ 1e10 at n ~ 1000).
struct Reducer {
  rgsv_allreduce_fn fn = nullptr;
  void* ctx = nullptr;
  int operator()(double* buf, int64_t count, cudaStream_t st) const {
    if (!fn || count <= 0) return 0;
    return fn(buf, count, reinterpret_cast<void*>(st), ctx) == 0 ? 0 : RGSV_ERR_CUDA;
  }
};

int cholqr3_tall(double* y, double* tmp, int64_t m, int k, int kp, double* gram, double* linv,
                 double* rdiag, double* scratch, size_t scratch_bytes, int* status,
                 double** q_out, cudaStream_t st, int passes = 3, const Reducer* red = nullptr,
                 int64_t shift_rows = -1, int shifted_passes = 1);

// Shifted CholeskyQR3 of Z = B^T where B is kp x n row-major (ld ldn):
// returns Qhat^T (kp x n) in *qt_out (one of b / tmp).
int cholqr3_wide(double* b, double* tmp, int64_t n, int64_t ldn, int k, int kp, double* gram,
                 double* linv, double* rinv, double* rdiag, double* scratch, size_t scratch_bytes,
                 int* status, double** qt_out, cudaStream_t st, int passes = 3);

// Multi-CTA dense factorizations (dense.cu), one cooperative launch each.
// Householder QR of [b1 (m1 rows); b2 (m2 rows)] (M x N, M <= 1408): Q (M x
// K) and optionally R (K x N), K = min(M, N); phase_fix makes diag(R) >= 0.
constexpr int kHhMaxRows = 1408;
size_t hhqr_workspace_bytes(int M, int N);
int hhqr(const double* b1, int64_t ld1, int m1, const double* b2, int64_t ld2, int m2, int N,
         double* q, int64_t ldq, double* r, int64_t ldr, int phase_fix, void* ws, size_t ws_bytes,
         cudaStream_t st, long long* prof = nullptr);
// Singular values of the rows of two matrices by blocked one-sided Jacobi
// (either job may be empty); `sync` holds bjacobi_sync_bytes() of scratch.
size_t bjacobi_sync_bytes();
int bjacobi(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1, double* v2,
            int64_t ld2, int nv2, int len2, double* sv2, int* nsv2, int* status, void* sync,
            cudaStream_t st);
// Singular values AND vectors of the rows of v (nv <= len) by the blocked
// Jacobi with accumulated rotations; the k_jacobi_vec output contract.
size_t svd_vectors_blocked_workspace_bytes(int nv);
int svd_vectors_blocked(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                        double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj,
                        int ascending, int* nzero, int* status, void* ws, size_t ws_bytes,
                        cudaStream_t st);

}  // namespace rgsv
