// Re-orthonormalisation: shifted CholeskyQR3.
//
// The reference orthonormalises with LAPACK Householder QR + a nonnegative
// R-diagonal phase fix (core.py:79-96). The sketches here have
// cond(Y) ~ 1e9, beyond plain CholeskyQR2, so each QR is
// shifted CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Zhang, Yamamoto 2020):
//   A = Y^T Y + s I, s = 11 (m k + k (k+1)) u ||Y||_F^2 ;  Q1 = Y chol(A)^{-1}
//   then two plain CholeskyQR passes on Q1.
// Cholesky gives a positive R diagonal, i.e. the same unique Q as the
// reference's phase-fixed Householder QR for full-rank input.
// Gram and TRSM are the DMMA GEMMs of gemm.cu; the k x k factorisation is
// one CTA (fused right-looking LDL^T + unit-lower inverse, one barrier per
// column) writing L^{-1} so the TRSM is a GEMM.
#include <math.h>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {

template <bool SMEM>
__global__ void __launch_bounds__(512) k_chol_inv(const double* __restrict__ gram, int k, int kp,
                                                  int64_t shift_rows, double* __restrict__ linv,
                                                  double* __restrict__ rinv,
                                                  double* __restrict__ r_upper,
                                                  double* __restrict__ rdiag,
                                                  double* __restrict__ rdiag_acc,
                                                  int* __restrict__ status,
                                                  double* __restrict__ gwork) {
  extern __shared__ double smem_w[];
  double* W = SMEM ? smem_w : gwork;  // kp x (kp + 1): lower = A/L, strict upper = X^T
  __shared__ int fail;
  const int ldw = kp + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, l = e % k;
    W[i * ldw + l] = (l <= i) ? gram[(int64_t)i * kp + l] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    fail = 0;
    if (shift_rows > 0) {
      double tr = 0.0;
      for (int i = 0; i < k; ++i) tr += W[i * ldw + i];
      const double sh = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
      for (int i = 0; i < k; ++i) W[i * ldw + i] += sh;
    }
  }
  __syncthreads();
  // kp is a multiple of 16 <= 512: thread -> (column c, row phase)
  const int cpt = kp;                  // columns covered per row pass
  const int rstep = nt / cpt > 0 ? nt / cpt : 1;
  const int c = tid % cpt, r0 = tid / cpt;
  for (int j = 0; j < k; ++j) {
    const double d = W[j * ldw + j];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) fail = 1;
      break;
    }
    const double inv_d = 1.0 / d;
    if (c < k && r0 < rstep) {
      const double xjc = (c < j) ? W[c * ldw + j] : 1.0;  // X[j][c], X[j][j] = 1
      const double wcj = (c > j) ? W[c * ldw + j] : 0.0;   // column j entry of row c
      for (int i = j + 1 + r0; i < k; i += rstep) {
        const double lij = W[i * ldw + j] * inv_d;  // unit-lower L[i][j]
        if (c <= j) {
          W[c * ldw + i] -= lij * xjc;  // X[i][c] -= L[i][j] X[j][c]
        } else if (c <= i) {
          W[i * ldw + c] -= lij * wcj;  // Schur update of the trailing block
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) atomicOr(status, RGSV_ST_CHOL_BREAKDOWN);
    for (int e = tid; e < kp * kp; e += nt) {
      linv[e] = __longlong_as_double(0x7ff8000000000000LL);
      if (rinv) rinv[e] = __longlong_as_double(0x7ff8000000000000LL);
    }
    return;
  }
  for (int e = tid; e < kp * kp; e += nt) {
    const int i = e / kp, cc = e % kp;
    double v;
    if (i < k && cc < k) {
      if (cc < i) {
        v = W[cc * ldw + i] / sqrt(W[i * ldw + i]);  // Linv = D^{-1/2} X
      } else if (cc == i) {
        v = 1.0 / sqrt(W[i * ldw + i]);
      } else {
        v = 0.0;
      }
    } else {
      v = (i == cc) ? 1.0 : 0.0;
    }
    linv[e] = v;
    if (rinv) rinv[(int64_t)cc * kp + i] = v;
  }
  if (r_upper) {  // R = L^T: R[c][i] = W[i][c] / sqrt(D[c]) for i > c
    for (int e = tid; e < kp * kp; e += nt) {
      const int rr = e / kp, cc = e % kp;  // R[rr][cc]
      double v = 0.0;
      if (rr < k && cc < k) {
        if (cc > rr) v = W[cc * ldw + rr] / sqrt(W[rr * ldw + rr]);
        else if (cc == rr) v = sqrt(W[rr * ldw + rr]);
      } else if (rr == cc) {
        v = 1.0;
      }
      r_upper[e] = v;
    }
  }
  for (int i = tid; i < k; i += nt) {
    const double si = sqrt(W[i * ldw + i]);
    if (rdiag) rdiag[i] = si;
    if (rdiag_acc) rdiag_acc[i] *= si;
  }
}

int chol_inv(const double* gram, int k, int kp, int64_t shift_rows, double* linv, double* rinv,
             double* r_upper, double* rdiag, double* rdiag_acc, int* status, cudaStream_t st) {
  if (k <= 0 || kp < k || kp % 16 != 0 || kp > 512) return RGSV_ERR_DIMENSION;
  const size_t wbytes = (size_t)kp * (kp + 1) * sizeof(double);
  if (wbytes <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_chol_inv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024) != cudaSuccess)
        return RGSV_ERR_CUDA;
      attr = true;
    }
    k_chol_inv<true><<<1, 512, wbytes, st>>>(gram, k, kp, shift_rows, linv, rinv, r_upper, rdiag,
                                             rdiag_acc, status, nullptr);
    note_launch();
  } else {
    // large k (stacked pairs of cfg2): working matrix in global memory,
    // placed after Linv in the caller's linv buffer (which is sized for it).
    double* gw = linv + (size_t)kp * kp;
    k_chol_inv<false><<<1, 512, 0, st>>>(gram, k, kp, shift_rows, linv, rinv, r_upper, rdiag,
                                         rdiag_acc, status, gw);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int cholqr3_tall(double* y, double* tmp, int64_t m, int k, int kp, double* gram, double* linv,
                 double* rdiag, double* scratch, size_t scratch_bytes, int* status,
                 double** q_out, cudaStream_t st) {
  double* src = y;
  double* dst = tmp;
  for (int step = 0; step < 3; ++step) {
    GemmArgs g;
    g.A = src;
    g.lda = kp;
    g.B = src;
    g.ldb = kp;
    g.C = gram;
    g.ldc = kp;
    g.M = kp;
    g.N = kp;
    g.K = m;
    g.scratch = scratch;
    g.scratch_bytes = scratch_bytes;
    g.max_split = kSMs;
    if (int e = gemm_gtq(g, st)) return e;
    if (int e = chol_inv(gram, k, kp, step == 0 ? m : 0, linv, nullptr, nullptr,
                         step == 0 ? rdiag : nullptr, step == 0 ? nullptr : rdiag, status, st))
      return e;
    GemmArgs t;
    t.A = src;
    t.lda = kp;
    t.B = linv;
    t.ldb = kp;
    t.C = dst;
    t.ldc = kp;
    t.M = m;
    t.N = kp;
    t.K = kp;
    t.scratch = scratch;
    t.scratch_bytes = scratch_bytes;
    t.max_split = 1;
    if (int e = gemm_gx(t, st)) return e;
    double* sw = src;
    src = dst;
    dst = sw;
  }
  *q_out = src;
  return 0;
}

int cholqr3_wide(double* b, double* tmp, int64_t n, int64_t ldn, int k, int kp, double* gram,
                 double* linv, double* rinv, double* rdiag, double* scratch, size_t scratch_bytes,
                 int* status, double** qt_out, cudaStream_t st) {
  double* src = b;
  double* dst = tmp;
  for (int step = 0; step < 3; ++step) {
    GemmArgs g;  // gram = B B^T (reduction over n)
    g.A = src;
    g.lda = ldn;
    g.B = src;
    g.ldb = ldn;
    g.C = gram;
    g.ldc = kp;
    g.M = kp;
    g.N = kp;
    g.K = n;
    g.scratch = scratch;
    g.scratch_bytes = scratch_bytes;
    g.max_split = 32;
    if (int e = gemm_gx(g, st)) return e;
    if (int e = chol_inv(gram, k, kp, step == 0 ? n : 0, linv, rinv, nullptr,
                         step == 0 ? rdiag : nullptr, step == 0 ? nullptr : rdiag, status, st))
      return e;
    GemmArgs t;  // Qhat^T = Linv B = Rinv^T B
    t.A = rinv;
    t.lda = kp;
    t.B = src;
    t.ldb = ldn;
    t.C = dst;
    t.ldc = ldn;
    t.M = kp;
    t.N = n;
    t.K = kp;
    t.scratch = scratch;
    t.scratch_bytes = scratch_bytes;
    t.max_split = 8;
    if (int e = gemm_gtq(t, st)) return e;
    double* sw = src;
    src = dst;
    dst = sw;
  }
  *qt_out = src;
  return 0;
}

}  // namespace rgsv
