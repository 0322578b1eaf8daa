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
#include <stdlib.h>


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
  // thread -> (column c, row phase); kp > nt (stacked pairs of cfg4, kp up
  // to 1024): each thread owns the columns tid, tid + nt, ...
  const int cpt = kp < nt ? kp : nt;   // columns covered per row pass
  const int rstep = nt / cpt > 0 ? nt / cpt : 1;
  const int c0 = tid % cpt, r0 = tid / cpt;
  for (int j = 0; j < k; ++j) {
    const double d = W[j * ldw + j];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) fail = 1;
      break;
    }
    const double inv_d = 1.0 / d;
    for (int c = c0; c < k && r0 < rstep; c += cpt) {
      const double xjc = (c < j) ? W[c * ldw + j] : 1.0;  // X[j][c], X[j][j] = 1
      const double wcj = (c > j) ? W[c * ldw + j] : 0.0;   // column j entry of row c
      int i = j + 1 + r0;
      // Column j (rows > j) is read-only during step j and every target
      // below is outside it, so batches of 8 loads can be in flight at once
      // (matters for the global-memory variant: kp > 200 KB of shared).
      for (; i + 7 * rstep < k; i += 8 * rstep) {
        double lv[8], tv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) lv[u] = W[(i + u * rstep) * ldw + j] * inv_d;
        if (c <= j) {
#pragma unroll
          for (int u = 0; u < 8; ++u) tv[u] = W[c * ldw + i + u * rstep];
#pragma unroll
          for (int u = 0; u < 8; ++u) W[c * ldw + i + u * rstep] = tv[u] - lv[u] * xjc;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            tv[u] = (c <= i + u * rstep) ? W[(i + u * rstep) * ldw + c] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c <= i + u * rstep) W[(i + u * rstep) * ldw + c] = tv[u] - lv[u] * wcj;
        }
      }
      for (; i < k; i += rstep) {
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

// Register-tiled variant for kp <= 128 (every range-finder Cholesky of the
// fp64 configs and the stacked small QR up to l1 + l2 = 128): a DIM x DIM
// thread grid, thread (ty, tx) owns the T x T tile A[ty*T.., tx*T..] of the
// Schur complement and the same tile of X, the running unit-lower inverse
// (registers, or shared memory when XS). Step j needs column j of A and row j
// of X, which their owners publish into double-buffered shared vectors right
// after their own update of step j-1: one __syncthreads per column. The
// update itself is branch-free (select + FMA), so warps never diverge.
template <int T, bool XS>
__global__ void __launch_bounds__(256)
    k_chol_reg(const double* __restrict__ gram, int k, int kp, int64_t shift_rows,
               double* __restrict__ linv, double* __restrict__ rinv,
               double* __restrict__ r_upper, double* __restrict__ rdiag,
               double* __restrict__ rdiag_acc, int* __restrict__ status) {
  __shared__ double colbuf[2][128];
  __shared__ double rowbuf[2][128];
  __shared__ double dbuf[128];
  __shared__ double shift_s;
  extern __shared__ double xsm[];  // XS: X as kp x (kp + 1)
  const int DIM = kp / T;
  const int tx = threadIdx.x % DIM, ty = threadIdx.x / DIM;
  const int i0 = ty * T, l0 = tx * T;
  const int ldx = kp + 1;
  __shared__ double piv[128];  // D[j], written once by thread 0 at step j
  double A[T][T], Xr[XS ? 1 : T][XS ? 1 : T];
#define XREF(a, b) (XS ? xsm[(i0 + (a)) * ldx + l0 + (b)] : Xr[XS ? 0 : (a)][XS ? 0 : (b)])
#pragma unroll
  for (int a = 0; a < T; ++a) {
#pragma unroll
    for (int b = 0; b < T; ++b) {
      const int i = i0 + a, l = l0 + b;
      A[a][b] = (i < k && l < k && l <= i) ? gram[(int64_t)i * kp + l] : 0.0;
      XREF(a, b) = (i == l) ? 1.0 : 0.0;
    }
  }
  if (shift_rows > 0) {
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
      for (int b = 0; b < T; ++b)
        if (i0 + a == l0 + b && i0 + a < k) dbuf[i0 + a] = A[a][b];
    __syncthreads();
    if (threadIdx.x == 0) {
      double tr = 0.0;
      for (int i = 0; i < k; ++i) tr += dbuf[i];
      shift_s = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
    }
    __syncthreads();
    const double sh = shift_s;
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
      for (int b = 0; b < T; ++b)
        if (i0 + a == l0 + b && i0 + a < k) A[a][b] += sh;
  }
  if (tx == 0) {  // publish column 0
#pragma unroll
    for (int a = 0; a < T; ++a)
      if (i0 + a < k) colbuf[0][i0 + a] = A[a][0];
  }
  __syncthreads();
  bool fail = false;
  for (int j = 0; j < k; ++j) {
    const int p = j & 1;
    const double d = colbuf[p][j];
    if (!(d > 0.0) || !isfinite(d)) {
      fail = true;
      break;
    }
    const double inv_d = 1.0 / d;
    if (threadIdx.x == 0) piv[j] = d;
    double cl[T], xr[T];
#pragma unroll
    for (int b = 0; b < T; ++b) {
      const int l = l0 + b;
      cl[b] = colbuf[p][l < 128 ? l : 0];
      xr[b] = (l < j) ? rowbuf[p][l] : (l == j ? 1.0 : 0.0);  // X[j][l]
    }
#pragma unroll
    for (int a = 0; a < T; ++a) {
      const int i = i0 + a;
      const bool live = (i > j) && (i < k);
      const double li = live ? colbuf[p][i] * inv_d : 0.0;  // unit-lower L[i][j]
#pragma unroll
      for (int b = 0; b < T; ++b) {
        const int l = l0 + b;
        const double ta = (l > j && l <= i) ? cl[b] : 0.0;  // trailing Schur update
        A[a][b] = fma(-li, ta, A[a][b]);
        XREF(a, b) = fma(-li, xr[b], XREF(a, b));  // X[i][l] -= L[i][j] X[j][l], l <= j
      }
    }
    const int jn = j + 1;
    if (jn < k) {
      if (jn >= l0 && jn < l0 + T) {
#pragma unroll
        for (int b = 0; b < T; ++b)
          if (l0 + b == jn) {
#pragma unroll
            for (int a = 0; a < T; ++a)
              if (i0 + a >= jn && i0 + a < k) colbuf[p ^ 1][i0 + a] = A[a][b];
          }
      }
      if (jn >= i0 && jn < i0 + T) {
#pragma unroll
        for (int a = 0; a < T; ++a)
          if (i0 + a == jn) {
#pragma unroll
            for (int b = 0; b < T; ++b)
              if (l0 + b < jn) rowbuf[p ^ 1][l0 + b] = XREF(a, b);
          }
      }
    }
    __syncthreads();
  }
  if (fail) {
    if (threadIdx.x == 0) atomicOr(status, RGSV_ST_CHOL_BREAKDOWN);
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
      for (int b = 0; b < T; ++b) {
        const int i = i0 + a, l = l0 + b;
        linv[(int64_t)i * kp + l] = qnan;
        if (rinv) rinv[(int64_t)l * kp + i] = qnan;
      }
    return;
  }
  __syncthreads();
  double sr[T], rsc[T];
#pragma unroll
  for (int a = 0; a < T; ++a) {
    sr[a] = (i0 + a < k) ? sqrt(piv[i0 + a]) : 1.0;
    rsc[a] = (l0 + a < k) ? 1.0 / sqrt(piv[l0 + a]) : 1.0;
  }
#pragma unroll
  for (int a = 0; a < T; ++a) {
    const int i = i0 + a;
    const double rsi = 1.0 / sr[a];
#pragma unroll
    for (int b = 0; b < T; ++b) {
      const int l = l0 + b;
      double v, ru;
      if (i < k && l < k) {
        v = (l <= i) ? XREF(a, b) * rsi : 0.0;                           // Linv = D^-1/2 X
        ru = (l < i) ? A[a][b] * rsc[b] : (l == i ? sr[a] : 0.0);      // R[l][i] = L[i][l]
        if (l == i) {
          if (rdiag) rdiag[i] = sr[a];
          if (rdiag_acc) rdiag_acc[i] *= sr[a];
        }
      } else {
        v = (i == l) ? 1.0 : 0.0;
        ru = v;
      }
      linv[(int64_t)i * kp + l] = v;
      if (rinv) rinv[(int64_t)l * kp + i] = v;
      if (r_upper) {
        r_upper[(int64_t)l * kp + i] = ru;
        if (l != i) r_upper[(int64_t)i * kp + l] = 0.0;
      }
    }
  }
#undef XREF
}

// Blocked variant (8-wide block columns) for kp <= 128. Per block column J:
//   thread 0 factors the 8x8 diagonal block and inverts it in registers;
//   all threads form the panel P = A[J+1:, J] L_JJ^-T and the block row
//   XR = L_JJ^-1 W[J, :J+1] of the inverse; then the trailing Schur update
//   A -= P P^T and the inverse update W[J+1:, :] -= P XR.
// Three barriers per 8 columns; A, W (-> L^{-1}) and P live in shared memory.
constexpr int kCholNB = 8;

// DMMA fragment helpers for 8x8 tiles held in shared memory (row-major, ld).
RGSV_DI void tile_mma_sub(double (&c)[2], const double* Arow8, int lda, const double* Brow8,
                          int ldb, bool b_transposed) {
  // c(8x8 frag) -= A(8x8) * B(8x8); A rows from Arow8, B given as rows of B
  // (b_transposed = false: B[t][n] = Brow8[t*ldb + n]) or as rows of B^T
  // (b_transposed = true: B[t][n] = Brow8[n*ldb + t]).
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; kk += 4) {
    const double a = -Arow8[g * lda + kk + t];
    const double bb = b_transposed ? Brow8[g * ldb + kk + t] : Brow8[(kk + t) * ldb + g];
    dmma(c, a, bb);
  }
}

// Fragment-major layouts of the panel P (kp x 8) and block row XR (8 x kp):
// each 8 x 4 DMMA operand fragment is 32 consecutive doubles, so fragment
// loads are bank-conflict free (the row-major ld-8 / ld-kp layouts were
// 4-way conflicted). I, K: multiples of 8; (r, c) / (t, n) inside the tile.
RGSV_DI int p_idx(int I, int r, int c) { return I * 8 + (c >> 2) * 32 + r * 4 + (c & 3); }
RGSV_DI int x_idx(int K, int t, int n) { return K * 8 + (t >> 2) * 32 + (t & 3) * 8 + n; }
constexpr int kCholPad = 8;  // A pitch kp + 8: 16-byte C-fragment rows hit distinct chunks

// Blocked right-looking Cholesky + inverse for kp <= 128, 8-wide blocks.
// Per block column J: thread 0 factors/inverts the 8x8 diagonal block in
// registers; warps form the panel P = A[J+1:, J] L_JJ^-T and the block row
// XR = L_JJ^-1 W[J, :J+1]; then every warp applies DMMA rank-8 updates to
// its 8x8 tiles: A_IK -= P_I P_K^T (trailing Schur complement) and
// W_IK -= P_I XR_K (inverse RHS). Three barriers per 8 columns.
// Shared layout: A (kp x lda): lower triangle = Schur complement -> L,
// strict upper = W^T (W -> L^{-1}, strictly lower part); Wd = diag(W).
__global__ void __launch_bounds__(512) k_chol_blk(const double* __restrict__ gram, int k, int kp,
                                                  int64_t shift_rows, double* __restrict__ linv,
                                                  double* __restrict__ rinv,
                                                  double* __restrict__ r_upper,
                                                  double* __restrict__ rdiag,
                                                  double* __restrict__ rdiag_acc,
                                                  int* __restrict__ status,
                                                  long long* __restrict__ prof = nullptr) {
  extern __shared__ double sm[];
  const int ld = kp + kCholPad;
#define PROF_MARK(slot) \
  if (prof && threadIdx.x == 0) prof[(slot)] = clock64();
  double* A = sm;
  double* Wd = A + kp * ld;               // kp
  double* P = Wd + kp;                    // kp x 8 panel (row-major, ld 8)
  double* XR = P + kp * kCholNB;          // 8 x kp block row of L^{-1} (ld kp)
  double* LJ = XR + kCholNB * kp;         // 8 x 8 L_JJ^{-1}
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int kb = (k + kCholNB - 1) / kCholNB * kCholNB;
  const int nb = kb / kCholNB;
  for (int i = warp; i < kb; i += nwarp) {
    for (int l = lane; l < kb; l += 32) {
      double a = 0.0;
      if (i < k && l < k) a = gram[(int64_t)i * kp + l];
      else if (i == l) a = 1.0;
      A[i * ld + l] = (l <= i) ? a : 0.0;
    }
    if (lane == 0) Wd[i] = 1.0;
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  if (shift_rows > 0) {
    if (warp == 0) {
      double tr = 0.0;
      for (int i = lane; i < k; i += 32) tr += A[i * ld + i];
      tr = warp_sum(tr);
      const double sh = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
      for (int i = lane; i < k; i += 32) A[i * ld + i] += sh;
    }
    __syncthreads();
  }
  PROF_MARK(0);
  for (int Jb = 0; Jb < nb; ++Jb) {
    const int J = Jb * kCholNB;
    PROF_MARK(1 + 4 * Jb);
    if (tid == 0) {
      double L[kCholNB][kCholNB], X[kCholNB][kCholNB], rr[kCholNB];
#pragma unroll
      for (int j = 0; j < kCholNB; ++j) {
        double d = A[(J + j) * ld + J + j];
#pragma unroll
        for (int t = 0; t < j; ++t) d = fma(-L[j][t], L[j][t], d);
        if (!(d > 0.0) || !isfinite(d)) fail = 1;
        const double r = rsqrt(d);
        rr[j] = r;
        L[j][j] = d * r;
#pragma unroll
        for (int i = j + 1; i < kCholNB; ++i) {
          double v = A[(J + i) * ld + J + j];
#pragma unroll
          for (int t = 0; t < j; ++t) v = fma(-L[i][t], L[j][t], v);
          L[i][j] = v * r;
        }
      }
#pragma unroll
      for (int j = 0; j < kCholNB; ++j) {
        X[j][j] = rr[j];
#pragma unroll
        for (int i = j + 1; i < kCholNB; ++i) {
          double v = 0.0;
#pragma unroll
          for (int t = j; t < i; ++t) v = fma(L[i][t], X[t][j], v);
          X[i][j] = -v * rr[i];
        }
      }
#pragma unroll
      for (int i = 0; i < kCholNB; ++i)
#pragma unroll
        for (int j = 0; j < kCholNB; ++j) {
          LJ[i * kCholNB + j] = (j <= i) ? X[i][j] : 0.0;
          if (j <= i) A[(J + i) * ld + J + j] = L[i][j];
        }
    }
    __syncthreads();
    PROF_MARK(2 + 4 * Jb);
    if (fail) break;
    // panel tiles P_I = A_IJ L_JJ^-T (I > J) and XR_K = L_JJ^-1 W_JK (K <= J)
    const int npanel = nb - 1 - Jb;
    for (int task = warp; task < npanel + Jb + 1; task += nwarp) {
      double c[2] = {0.0, 0.0};
      if (task < npanel) {
        const int I = (Jb + 1 + task) * kCholNB;
        // P_I[g][n] = sum_t A[I+g][J+t] * LJ[n][t]
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4)
          dmma(c, A[(I + g) * ld + J + kk + tq], LJ[g * kCholNB + kk + tq]);
        P[p_idx(I, g, 2 * tq)] = c[0];
        P[p_idx(I, g, 2 * tq + 1)] = c[1];
      } else {
        const int K = (task - npanel) * kCholNB;
        // XR_K[r][n] = sum_t LJ[r][t] * W[J+t][K+n]  (W lower part in A^T, diag in Wd)
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          const int row = J + kk + tq, col = K + g;
          const double w = col < row ? A[col * ld + row] : (col == row ? Wd[row] : 0.0);
          dmma(c, LJ[g * kCholNB + kk + tq], w);
        }
        XR[x_idx(K, g, 2 * tq)] = c[0];
        XR[x_idx(K, g, 2 * tq + 1)] = c[1];
      }
    }
    __syncthreads();
    PROF_MARK(3 + 4 * Jb);
    // DMMA rank-8 updates: trailing tiles (I >= K > J) and inverse tiles (I > J >= K)
    const int ntrail = npanel * (npanel + 1) / 2;
    const int ninv = npanel * (Jb + 1);
    for (int task = warp; task < ntrail + ninv + npanel; task += nwarp) {
      if (task < ntrail) {
        // decode (I, K) with K <= I over the npanel x npanel lower triangle
        int ii = 0, rem = task;
        while (rem > ii) { rem -= ii + 1; ++ii; }
        const int I = (Jb + 1 + ii) * kCholNB, K = (Jb + 1 + rem) * kCholNB;
        const int r0 = I + g, c0 = K + 2 * tq;
        const double2 cv = *reinterpret_cast<const double2*>(A + r0 * ld + c0);
        double c[2] = {cv.x, cv.y};
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4)
          dmma(c, -P[p_idx(I, g, kk + tq)], P[p_idx(K, g, kk + tq)]);
        if (I != K) {
          *reinterpret_cast<double2*>(A + r0 * ld + c0) = make_double2(c[0], c[1]);
        } else {
          if (c0 <= r0) A[r0 * ld + c0] = c[0];
          if (c0 + 1 <= r0) A[r0 * ld + c0 + 1] = c[1];
        }
      } else if (task < ntrail + ninv) {
        const int v = task - ntrail;
        const int I = (Jb + 1 + v / (Jb + 1)) * kCholNB, K = (v % (Jb + 1)) * kCholNB;
        // W_IK -= P_I XR_K; W_IK[g][n] lives at A[(K+n)*ld + I+g]
        double c[2];
        const int r0 = I + g, n0 = K + 2 * tq;
        c[0] = A[n0 * ld + r0];
        c[1] = A[(n0 + 1) * ld + r0];
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4)
          dmma(c, -P[p_idx(I, g, kk + tq)], XR[x_idx(K, kk + tq, g)]);
        A[n0 * ld + r0] = c[0];
        A[(n0 + 1) * ld + r0] = c[1];
      } else {
        // finalize block column J of L for panel block I
        const int I = (Jb + 1 + (task - ntrail - ninv)) * kCholNB;
        for (int e = lane; e < 64; e += 32)
          A[(I + (e >> 3)) * ld + J + (e & 7)] = P[p_idx(I, e >> 3, e & 7)];
      }
    }
    // finalize block row J of L^{-1}
    for (int e = tid; e < kCholNB * (J + kCholNB); e += nt) {
      const int r = e / (J + kCholNB), c = e % (J + kCholNB), row = J + r;
      const double xv = XR[x_idx(c & ~7, r, c & 7)];
      if (c < row) A[c * ld + row] = xv;
      else if (c == row) Wd[row] = xv;
    }
    __syncthreads();
    PROF_MARK(4 + 4 * Jb);
  }
#undef PROF_MARK
  if (fail) {
    if (tid == 0) atomicOr(status, RGSV_ST_CHOL_BREAKDOWN);
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
    for (int e = tid; e < kp * kp; e += nt) {
      linv[e] = qnan;
      if (rinv) rinv[e] = qnan;
    }
    return;
  }
  for (int i = warp; i < kp; i += nwarp) {
    for (int l = lane; l < kp; l += 32) {
      double v, ru;
      if (i < k && l < k) {
        v = (l < i) ? A[l * ld + i] : (l == i ? Wd[i] : 0.0);
        ru = (l <= i) ? A[i * ld + l] : 0.0;
      } else {
        v = (i == l) ? 1.0 : 0.0;
        ru = v;
      }
      linv[(int64_t)i * kp + l] = v;
      if (rinv) rinv[(int64_t)l * kp + i] = v;
      if (r_upper) r_upper[(int64_t)l * kp + i] = ru;
    }
  }
  for (int i = tid; i < k; i += nt) {
    const double si = A[i * ld + i];
    if (rdiag) rdiag[i] = si;
    if (rdiag_acc) rdiag_acc[i] *= si;
  }
}

int chol_profile(const double* gram, int k, int kp, double* linv, long long* prof,
                 int* status, cudaStream_t st) {
  if (kp > 128) return RGSV_ERR_DIMENSION;
  const size_t bytes =
      ((size_t)kp * (kp + kCholPad) + kp + 2 * (size_t)kp * kCholNB + 64) * sizeof(double);
  cudaFuncSetAttribute(k_chol_blk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(((size_t)128 * (128 + kCholPad) + 128 + 2 * 128 * kCholNB + 64) *
                             sizeof(double)));
  k_chol_blk<<<1, 128, bytes, st>>>(gram, k, kp, 0, linv, nullptr, nullptr, nullptr, nullptr,
                                    status, prof);
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// ------------------------------------------- 16-wide blocked, kp <= 64
// Diagonal 16x16 blocks are factored by ONE warp, register resident
// (lane i holds row i; symmetric Gauss-Jordan on [A_JJ | I] yields L_JJ^T in
// the A half and L_JJ^-1 in the X half, critical path one shuffle + rsqrt +
// FMA per column). Panel L_IJ = A_IJ L_JJ^-T and trailing A_IK -= L_IJ L_KJ^T
// are DMMA tiles spread over 8 warps; L^-1 is then assembled block row by
// block row, W_IK = -W_II sum_{M=K}^{I-1} L_IM W_MK. Shared memory: A and W,
// kp x (kp + 4) each (pitch 68 keeps both DMMA fragment patterns at two
// wavefronts).
constexpr int kCB = 16;

RGSV_DI double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ void gj_block16(double* A, int lda, double* W, int ldw, int r0, double* rdiag,
                           double* rdiag_acc, int k, int* fail) {
  const int lane = threadIdx.x & 31;
  double z[kCB], x[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) {
    z[c] = (lane < kCB) ? A[(r0 + lane) * lda + r0 + c] : (lane == c ? 1.0 : 0.0);
    x[c] = (lane == c) ? 1.0 : 0.0;
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    const double d = __shfl_sync(0xffffffffu, z[j], j);
    double pa[kCB], px[kCB];
#pragma unroll
    for (int c = 0; c < kCB; ++c) {
      if (c > j) pa[c] = __shfl_sync(0xffffffffu, z[c], j);
      if (c <= j) px[c] = __shfl_sync(0xffffffffu, x[c], j);
    }
    bad |= !(d > 0.0) || !isfinite(d);
    const double r = rsqrt(d);
    const double ff = (lane > j) ? z[j] * (r * r) : 0.0;
    const double mul = (lane == j) ? r : 1.0;
#pragma unroll
    for (int c = 0; c < kCB; ++c) {
      if (c > j) z[c] = fma(-ff, pa[c], z[c]) * mul;
      if (c <= j) x[c] = fma(-ff, px[c], x[c]) * mul;
    }
    z[j] = (lane > j) ? 0.0 : (lane == j ? d * r : z[j]);
  }
  if (lane < kCB) {
    // lane j: z[c] (c >= j) = L[c][j]; x[c] (c <= j) = Linv[j][c]
#pragma unroll
    for (int c = 0; c < kCB; ++c) {
      A[(r0 + c) * lda + r0 + lane] = (c >= lane) ? z[c] : 0.0;  // L_JJ column `lane`
      W[(r0 + lane) * ldw + r0 + c] = (c <= lane) ? x[c] : 0.0;  // Linv_JJ row `lane`
    }
    const int i = r0 + lane;
    double dj = 0.0;
#pragma unroll
    for (int c = 0; c < kCB; ++c)
      if (c == lane) dj = z[c];
    if (i < k) {
      if (rdiag) rdiag[i] = dj;
      if (rdiag_acc) rdiag_acc[i] *= dj;
    }
  }
  if (bad && lane == 0) *fail = 1;
}

__global__ void __launch_bounds__(256) k_chol_b16(const double* __restrict__ gram, int k, int kp,
                                                  int64_t shift_rows, double* __restrict__ linv,
                                                  double* __restrict__ rinv,
                                                  double* __restrict__ r_upper,
                                                  double* __restrict__ rdiag,
                                                  double* __restrict__ rdiag_acc,
                                                  int* __restrict__ status) {
  extern __shared__ double smc[];
  const int ld = kp + 4;
  double* A = smc;           // kp x ld : A -> L (lower, diag blocks full)
  double* W = A + kp * ld;   // kp x ld : L^-1
  __shared__ int fail;
  __shared__ double shift;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = kp / kCB;
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int i = e / kp, c = e % kp;
    A[i * ld + c] = (i < k && c < k) ? gram[(int64_t)i * kp + c] : (i == c ? 1.0 : 0.0);
    W[i * ld + c] = 0.0;
  }
  if (tid == 0) fail = 0;
  __shared__ int near_id;
  if (tid == 0) near_id = 0;
  __syncthreads();
  if (shift_rows == 0) {
    // Near-identity Gram (the third CholeskyQR pass: G = I + E, |E| ~ u
    // cond(Q1)^2): L = I + X with X = Phi(E - X1 X1^T), X1 = Phi(E) (Phi:
    // strict lower + half diagonal) and L^-1 = I - X + X^2, exact in fp64
    // for max|E| <= 1e-6 (neglected terms O(|E|^3) <= 1e-18); no pivot chain.
    double mx = 0.0;
    for (int e = tid; e < k * k; e += blockDim.x) {
      const int i = e / k, c = e % k;
      mx = fmax(mx, fabs(A[i * ld + c] - (i == c ? 1.0 : 0.0)));
    }
    mx = warp_max(mx);
    __shared__ double wm[8];
    if (lane == 0) wm[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
      near_id = (m <= 1e-6) ? 1 : 0;
    }
    __syncthreads();
  }
  if (near_id) {
    const int g = lane >> 2, t = lane & 3;
    const int nt8 = kp / 8;
    // A := E (padding 0); W := X1 = Phi(E)
    for (int e = tid; e < kp * kp; e += blockDim.x) {
      const int i = e / kp, c = e % kp;
      const double ev = A[i * ld + c] - (i == c ? 1.0 : 0.0);
      A[i * ld + c] = ev;
      W[i * ld + c] = (c < i) ? ev : (c == i ? 0.5 * ev : 0.0);
    }
    __syncthreads();
    // lower 8x8 tiles (ti >= tc), enumerated u -> (ti, tc)
    const int nlow = nt8 * (nt8 + 1) / 2;
    auto tile_of = [&](int u, int& ti, int& tc) {
      ti = (int)((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
      while ((ti + 1) * (ti + 2) / 2 <= u) ++ti;
      while (ti * (ti + 1) / 2 > u) --ti;
      tc = u - ti * (ti + 1) / 2;
    };
    // A := E - X1 X1^T; X1 lower triangular: (X1 X1^T)_ic needs k < 8 (tc + 1)
    for (int u = warp; u < nlow; u += 8) {
      int ti, tc;
      tile_of(u, ti, tc);
      double m2[2] = {0.0, 0.0}, m3[2] = {0.0, 0.0};
      const int kend = (tc + 1) * 2;  // k-steps of 4 covering columns < 8 (tc + 1)
      int ks = 0;
      for (; ks + 1 < kend; ks += 2) {
        dmma(m2, W[(ti * 8 + g) * ld + ks * 4 + t], W[(tc * 8 + g) * ld + ks * 4 + t]);
        dmma(m3, W[(ti * 8 + g) * ld + ks * 4 + 4 + t], W[(tc * 8 + g) * ld + ks * 4 + 4 + t]);
      }
      if (ks < kend) dmma(m2, W[(ti * 8 + g) * ld + ks * 4 + t], W[(tc * 8 + g) * ld + ks * 4 + t]);
      A[(ti * 8 + g) * ld + tc * 8 + 2 * t] -= m2[0] + m3[0];
      A[(ti * 8 + g) * ld + tc * 8 + 2 * t + 1] -= m2[1] + m3[1];
    }
    __syncthreads();
    // W := X = Phi(A)
    for (int e = tid; e < kp * kp; e += blockDim.x) {
      const int i = e / kp, c = e % kp;
      W[i * ld + c] = (c < i) ? A[i * ld + c] : (c == i ? 0.5 * A[i * ld + c] : 0.0);
    }
    __syncthreads();
    // A := L^-1 = I - X + X^2; X lower triangular: (X^2)_ic needs
    // 8 tc <= k < 8 (ti + 1); upper tiles are zero
    for (int u = warp; u < nt8 * nt8; u += 8) {
      const int ti = u / nt8, tc = u % nt8;
      double m2[2] = {0.0, 0.0}, m3[2] = {0.0, 0.0};
      if (tc <= ti) {
        const int kb = tc * 2, kend = (ti + 1) * 2;
        int ks = kb;
        for (; ks + 1 < kend; ks += 2) {
          dmma(m2, W[(ti * 8 + g) * ld + ks * 4 + t], W[(ks * 4 + t) * ld + tc * 8 + g]);
          dmma(m3, W[(ti * 8 + g) * ld + ks * 4 + 4 + t], W[(ks * 4 + 4 + t) * ld + tc * 8 + g]);
        }
        if (ks < kend) dmma(m2, W[(ti * 8 + g) * ld + ks * 4 + t], W[(ks * 4 + t) * ld + tc * 8 + g]);
      }
      const int i = ti * 8 + g, c0 = tc * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = c0 + h;
        A[i * ld + c] =
            (c <= i) ? ((i == c ? 1.0 : 0.0) - W[i * ld + c] + (m2[h] + m3[h])) : 0.0;
      }
    }
    __syncthreads();
    for (int e = tid; e < kp * kp; e += blockDim.x) {
      const int i = e / kp, c = e % kp;
      const double v = A[i * ld + c];
      linv[e] = v;
      if (rinv) rinv[(int64_t)c * kp + i] = v;
      if (r_upper) r_upper[(int64_t)c * kp + i] = (i == c ? 1.0 : 0.0) + W[i * ld + c];
    }
    for (int i = tid; i < k; i += blockDim.x) {
      const double di = 1.0 + W[i * ld + i];
      if (rdiag) rdiag[i] = di;
      if (rdiag_acc) rdiag_acc[i] *= di;
    }
    return;
  }
  if (shift_rows > 0) {
    if (warp == 0) {  // trace from shared memory, fixed-order warp reduction
      double tr = 0.0;
      for (int i = lane; i < k; i += 32) tr += A[i * ld + i];
      tr = warp_sum(tr);
      if (lane == 0) shift = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
    }
    __syncthreads();
    for (int i = tid; i < k; i += blockDim.x) A[i * ld + i] += shift;
    __syncthreads();
  }
  const int g = lane >> 2, t = lane & 3;
  for (int J = 0; J < nb; ++J) {
    const int r0 = J * kCB;
    if (warp == 0) gj_block16(A, ld, W, ld, r0, rdiag, rdiag_acc, k, &fail);
    __syncthreads();
    // panel: L_IJ = A_IJ W_JJ^T for I > J (8x8 output tiles)
    const int prow = kp - r0 - kCB;  // rows below the diagonal block
    const int ntile = (prow / 8) * 2;  // <= 12 for kp <= 64: two slots per warp
    double pv[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int u = warp + 8 * q;
      if (u < ntile) {
        const int rr = r0 + kCB + (u >> 1) * 8, cc = (u & 1) * 8;
        double c2[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < kCB / 4; ++ks)
          dmma(c2, A[(rr + g) * ld + r0 + ks * 4 + t], W[(r0 + cc + g) * ld + r0 + ks * 4 + t]);
        pv[q][0] = c2[0];
        pv[q][1] = c2[1];
      }
    }
    __syncthreads();  // every read of A_IJ done before the in-place write
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int u = warp + 8 * q;
      if (u < ntile) {
        const int rr = r0 + kCB + (u >> 1) * 8, cc = (u & 1) * 8;
        A[(rr + g) * ld + r0 + cc + 2 * t] = pv[q][0];
        A[(rr + g) * ld + r0 + cc + 2 * t + 1] = pv[q][1];
      }
    }
    __syncthreads();
    // trailing: A_IK -= L_IJ L_KJ^T, 8x8 tiles (row tile >= col tile block-wise)
    const int tb = (kp - r0 - kCB) / 8;  // 8-tiles in the trailing dimension
    for (int u = warp; u < tb * tb; u += 8) {
      const int ti = u / tb, tk = u % tb;
      if ((ti >> 1) < (tk >> 1)) continue;  // strictly upper 16-blocks not needed
      const int rr = r0 + kCB + ti * 8, cc = r0 + kCB + tk * 8;
      double c2[2] = {A[(rr + g) * ld + cc + 2 * t], A[(rr + g) * ld + cc + 2 * t + 1]};
      double m2[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < kCB / 4; ++ks)
        dmma(m2, A[(rr + g) * ld + r0 + ks * 4 + t], A[(cc + g) * ld + r0 + ks * 4 + t]);
      A[(rr + g) * ld + cc + 2 * t] = c2[0] - m2[0];
      A[(rr + g) * ld + cc + 2 * t + 1] = c2[1] - m2[1];
    }
    __syncthreads();
  }
  // L^-1 off-diagonal blocks, block row by block row
  for (int I = 1; I < nb; ++I) {
    // T_K = sum_{M=K}^{I-1} L_IM W_MK for K < I, staged in W_IK
    for (int u = warp; u < I * 4; u += 8) {
      const int K = u >> 2, q = u & 3;
      const int rr = I * kCB + (q >> 1) * 8, cc = K * kCB + (q & 1) * 8;
      double c2[2] = {0.0, 0.0};
      for (int M = K; M < I; ++M)
#pragma unroll
        for (int ks = 0; ks < kCB / 4; ++ks)
          dmma(c2, A[(rr + g) * ld + M * kCB + ks * 4 + t],
               W[(M * kCB + ks * 4 + t) * ld + cc + g]);
      W[(rr + g) * ld + cc + 2 * t] = c2[0];
      W[(rr + g) * ld + cc + 2 * t + 1] = c2[1];
    }
    __syncthreads();
    // W_IK = -W_II T_K  (I * 4 <= 12 tiles: two slots per warp)
    double ov[2][2];
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int u = warp + 8 * s2;
      if (u < I * 4) {
        const int K = u >> 2, q = u & 3;
        const int rr = I * kCB + (q >> 1) * 8, cc = K * kCB + (q & 1) * 8;
        double c2[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < kCB / 4; ++ks)
          dmma(c2, W[(rr + g) * ld + I * kCB + ks * 4 + t],
               W[(I * kCB + ks * 4 + t) * ld + cc + g]);
        ov[s2][0] = -c2[0];
        ov[s2][1] = -c2[1];
      }
    }
    __syncthreads();
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int u = warp + 8 * s2;
      if (u < I * 4) {
        const int K = u >> 2, q = u & 3;
        const int rr = I * kCB + (q >> 1) * 8, cc = K * kCB + (q & 1) * 8;
        W[(rr + g) * ld + cc + 2 * t] = ov[s2][0];
        W[(rr + g) * ld + cc + 2 * t + 1] = ov[s2][1];
      }
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) atomicOr(status, RGSV_ST_CHOL_BREAKDOWN);
    for (int e = tid; e < kp * kp; e += blockDim.x) {
      linv[e] = __longlong_as_double(0x7ff8000000000000LL);
      if (rinv) rinv[e] = __longlong_as_double(0x7ff8000000000000LL);
    }
    return;
  }
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int i = e / kp, c = e % kp;
    const double v = (c <= i) ? W[i * ld + c] : 0.0;
    linv[e] = v;
    if (rinv) rinv[(int64_t)c * kp + i] = v;
    if (r_upper) r_upper[(int64_t)c * kp + i] = (c <= i) ? A[i * ld + c] : 0.0;  // R = L^T
  }
}

// ------------------------------------------- blocked, 128 < kp <= 4096
// kp beyond one CTA's shared memory (cfg4: the 288-wide range-finder blocks
// and the 576-wide stacked pair). Right-looking blocked Cholesky on a global
// (L2-resident) working copy: each <= 128-wide diagonal block is factorised
// by k_chol_blk (which also returns its inverse), panels and trailing
// updates are DMMA GEMMs, and L^{-1} is assembled block by block
// (X_IJ = -L_II^{-1} sum_{J<=K<I} L_IK X_KJ). Same outputs and identity
// padding as the one-CTA kernels.

// W = gram (+ shift s I on the k real columns, identity on the padding);
// every block recomputes the trace (k <= kCholMaxKp diagonal reads).
__global__ void k_chol_prep(const double* __restrict__ gram, int k, int kp, int64_t shift_rows,
                            double* __restrict__ W) {
  double sh = 0.0;
  if (shift_rows > 0) {
    double tr = 0.0;
    for (int i = 0; i < k; ++i) tr += gram[(int64_t)i * kp + i];
    sh = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
  }
  const int64_t total = (int64_t)kp * kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / kp), j = (int)(e % kp);
    double v;
    if (i < k && j < k)
      v = gram[e] + (i == j ? sh : 0.0);
    else
      v = (i == j) ? 1.0 : 0.0;
    W[e] = v;
  }
}

// linv = X (lower part), rinv = X^T.
__global__ void k_chol_finish(const double* __restrict__ X, int kp, double* __restrict__ linv,
                              double* __restrict__ rinv) {
  const int64_t total = (int64_t)kp * kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / kp), j = (int)(e % kp);
    const double x = (j <= i) ? X[e] : 0.0;
    linv[e] = x;
    if (rinv) rinv[(int64_t)j * kp + i] = x;
  }
}

__global__ void k_identity2(double* __restrict__ a, double* __restrict__ b, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const double v = (e / n == e % n) ? 1.0 : 0.0;
    a[e] = v;
    b[e] = v;
  }
}

namespace {

// Scratch of the blocked factorisation: stream-ordered (cudaMallocAsync /
// cudaFreeAsync), so the call is also capturable in a CUDA graph (memory
// alloc/free nodes) and concurrent chains on different streams never share
// it. The default pool keeps freed blocks cached (release threshold max).
double* blk_scratch_alloc(cudaStream_t st, size_t bytes) {
  static bool pool_set = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return true;
  }();
  (void)pool_set;
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) return nullptr;
  return static_cast<double*>(p);
}

int gemm_small(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
               int64_t M, int64_t N, int64_t K, bool gtq, cudaStream_t st) {
  GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.B = B;
  g.ldb = ldb;
  g.C = C;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.max_split = 1;
  return gtq ? gemm_gtq(g, st) : gemm_gx(g, st);
}

int copy2d(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols,
           cudaStream_t st) {
  return cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double),
                           cols * sizeof(double), rows, cudaMemcpyDeviceToDevice, st) == cudaSuccess
             ? 0
             : RGSV_ERR_CUDA;
}

}  // namespace

int launch_axpy(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols,
                double alpha, cudaStream_t st);
int launch_copy_block(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols,
                      int transpose, cudaStream_t st);

int chol_inv_blocked(const double* gram, int k, int kp, int64_t shift_rows, double* linv,
                     double* rinv, double* r_upper, double* rdiag, double* rdiag_acc, int* status,
                     cudaStream_t st) {
  if (r_upper) return RGSV_ERR_DIMENSION;  // R = L^T is only requested for kp <= 128
  const int nb = (kp + 127) / 128;
  const int bs = ((kp + nb - 1) / nb + 15) / 16 * 16;  // block size, multiple of 16, <= 128
  const size_t kk = (size_t)kp * kp, bb = (size_t)128 * 128;
  double* base = blk_scratch_alloc(st, (4 * kk + (4 + (size_t)nb) * bb + 8 * 128) * sizeof(double));
  if (!base) return RGSV_ERR_CUDA;
  struct Release {  // freed in stream order on every exit path
    double* p;
    cudaStream_t s;
    ~Release() { cudaFreeAsync(p, s); }
  } release{base, st};
  double* W = base;            // working copy; lower part becomes L
  double* X = W + kk;          // L^{-1}
  double* T = X + kk;          // GEMM outputs (<= kp x kp)
  double* T2 = T + kk;
  double* D = T2 + kk;         // diagonal block input (bs x bs)
  double* DL = D + bb;         // its L^{-1} (k_chol_blk output, + work)
  double* RI = DL + 2 * bb;    // per block: L_II^{-T} (bs x bs each)
  if (cudaMemsetAsync(X, 0, kk * sizeof(double), st) != cudaSuccess) return RGSV_ERR_CUDA;
  k_chol_prep<<<64, 256, 0, st>>>(gram, k, kp, shift_rows, W);
  note_launch();
  for (int J = 0; J < nb; ++J) {
    const int o = J * bs;
    if (o >= kp) break;
    const int s = kp - o < bs ? kp - o : bs;
    const int kr = k - o < 0 ? 0 : (k - o < s ? k - o : s);
    const int below = kp - o - s;
    // (a) diagonal block: L_JJ^{-1} (and its transpose) by the one-CTA kernel
    if (int e = copy2d(D, s, W + (size_t)o * kp + o, kp, s, s, st)) return e;
    double* rij = RI + (size_t)J * bb;
    if (kr > 0) {
      if (int e = chol_inv(D, kr, s, 0, DL, rij, nullptr, rdiag ? rdiag + o : nullptr,
                           rdiag_acc ? rdiag_acc + o : nullptr, status, st))
        return e;
    } else {  // pure padding: identity
      k_identity2<<<8, 256, 0, st>>>(DL, rij, s);
      note_launch();
    }
    if (int e = copy2d(X + (size_t)o * kp + o, kp, DL, s, s, s, st)) return e;
    if (below > 0) {
      // (b) panel L_{>J,J} = A_{>J,J} L_JJ^{-T}
      double* P = W + (size_t)(o + s) * kp + o;
      if (int e = gemm_small(P, kp, DL, s, T, s, below, s, s, false, st)) return e;
      if (int e = copy2d(P, kp, T, s, below, s, st)) return e;
      // (c) trailing A_{>J,>J} -= L_{>J,J} L_{>J,J}^T
      if (int e = gemm_small(P, kp, P, kp, T2, below, below, below, s, false, st)) return e;
      if (int e = launch_axpy(W + (size_t)(o + s) * kp + o + s, kp, T2, below, below, below, -1.0,
                              st))
        return e;
    }
  }
  // (d) X_IJ = -L_II^{-1} sum_{J<=K<I} L_IK X_KJ, block column by block column
  for (int J = 0; J < nb; ++J) {
    const int oj = J * bs;
    if (oj >= kp) break;
    const int sj = kp - oj < bs ? kp - oj : bs;
    for (int I = J + 1; I < nb; ++I) {
      const int oi = I * bs;
      if (oi >= kp) break;
      const int si = kp - oi < bs ? kp - oi : bs;
      // S (si x sj) = L[oi:oi+si, oj:oi] X[oj:oi, oj:oj+sj] as gx (A Bt^T) with
      // Bt = X[oj:oi, J]^T, transposed into T2 (sj x kk2)
      const int kk2 = oi - oj;
      if (int e = launch_copy_block(T2, kk2, X + (size_t)oj * kp + oj, kp, sj, kk2, 1, st))
        return e;
      if (int e = gemm_small(W + (size_t)oi * kp + oj, kp, T2, kk2, T, sj, si, sj, kk2, false, st))
        return e;
      // X_IJ = -L_II^{-1} S: gtq(A = L_II^{-T} (si x si), B = S) = L_II^{-1} S
      if (int e = gemm_small(RI + (size_t)I * bb, si, T, sj, T2, sj, si, sj, si, true, st))
        return e;
      if (int e = launch_axpy(X + (size_t)oi * kp + oj, kp, T2, sj, si, sj, -1.0, st)) return e;
    }
  }
  k_chol_finish<<<64, 256, 0, st>>>(X, kp, linv, rinv);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int chol_inv(const double* gram, int k, int kp, int64_t shift_rows, double* linv, double* rinv,
             double* r_upper, double* rdiag, double* rdiag_acc, int* status, cudaStream_t st) {
  if (k <= 0 || kp < k || kp % 16 != 0 || kp > kCholMaxKp) return RGSV_ERR_DIMENSION;
  if (kp <= 64 && !getenv("RGSV_CHOL_BLK")) {
    const size_t bytes = (size_t)2 * kp * (kp + 4) * sizeof(double);
    static bool attr_b16 = false;
    if (!attr_b16) {
      if (cudaFuncSetAttribute(k_chol_b16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)((size_t)2 * 64 * 68 * sizeof(double))) != cudaSuccess)
        return RGSV_ERR_CUDA;
      attr_b16 = true;
    }
    k_chol_b16<<<1, 256, bytes, st>>>(gram, k, kp, shift_rows, linv, rinv, r_upper, rdiag,
                                      rdiag_acc, status);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
  }
  if (kp <= 128) {
    const size_t bytes =
        ((size_t)kp * (kp + kCholPad) + kp + 2 * (size_t)kp * kCholNB + 64) * sizeof(double);
    static bool attr_blk = false;
    if (!attr_blk) {
      if (cudaFuncSetAttribute(k_chol_blk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(((size_t)128 * (128 + kCholPad) + 128 + 2 * 128 * kCholNB + 64) *
                                     sizeof(double))) != cudaSuccess)
        return RGSV_ERR_CUDA;
      attr_blk = true;
    }
    // 512 threads for kp > 64 (the rank-8 update phase is latency bound:
    // kp = 128 78 vs 96 us with 256; cfg2 14.67 -> 14.79 pairs/s), 256 below.
    // RGSV_CHOL_THREADS=128 keeps the CTA <= 16K registers so it can co-reside
    // with a GEMM CTA of the other chain (slower alone: 41 vs 30 us at k = 60).
    static int forced = [] {
      const char* e = getenv("RGSV_CHOL_THREADS");
      const int v = e ? atoi(e) : 0;
      return (v == 128 || v == 256 || v == 512) ? v : 0;
    }();
    const int threads = forced ? forced : (kp > 64 ? 512 : 256);
    k_chol_blk<<<1, threads, bytes, st>>>(gram, k, kp, shift_rows, linv, rinv, r_upper, rdiag,
                                      rdiag_acc, status);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
  }
  static const bool unblocked = getenv("RGSV_CHOL_UNBLOCKED") != nullptr;
  if (!unblocked && !r_upper)
    return chol_inv_blocked(gram, k, kp, shift_rows, linv, rinv, r_upper, rdiag, rdiag_acc, status,
                            st);
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

// Split count of the tall Gram Y^T Y (K = m rows, kp x kp output): the
// reduction over rows is the only parallelism. 32 splits: measured on cfg1
// (8 concurrent pairs) 684 / 698 / 713 / 718 pairs/s at 148 / 74 / 32 / 16
// splits and 2.24 / 2.25 / 2.31 / 2.52 ms single-pair latency.
// RGSV_GRAM_SPLIT overrides it (tuning experiments).
static int tall_gram_split() {
  static const int v = [] {
    const char* e = getenv("RGSV_GRAM_SPLIT");
    const int x = e ? atoi(e) : 0;
    return x >= 1 ? x : 32;
  }();
  return v;
}

int cholqr3_tall(double* y, double* tmp, int64_t m, int k, int kp, double* gram, double* linv,
                 double* rdiag, double* scratch, size_t scratch_bytes, int* status,
                 double** q_out, cudaStream_t st, int passes, const Reducer* red,
                 int64_t shift_rows, int shifted_passes) {
  if (shift_rows < 0) shift_rows = m;
  double* src = y;
  double* dst = tmp;
  for (int step = 0; step < passes; ++step) {
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
    g.max_split = tall_gram_split();
    if (k == 120 && kp == 128) {  // exact-width Gram (cfg2): the 120 x 120 live block
      g.live = 120;
      g.N = 120;
    }
    g.lower_only = kp > 128;  // the blocked Cholesky reads only the lower triangle
    if (int e = gemm_gtq(g, st)) return e;
    if (red)  // sum the Gram partials of every rank's row block
      if (int e = (*red)(gram, (int64_t)kp * kp, st)) return e;
    if (int e = chol_inv(gram, k, kp, step < shifted_passes ? shift_rows : 0, linv, nullptr,
                         nullptr, step == 0 ? rdiag : nullptr, step == 0 ? nullptr : rdiag, status,
                         st))
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
    t.live = k;  // exact-width TRSM tile where one exists (k = 120)
    if (int e = gemm_gx(t, st)) return e;
    double* sw = src;
    src = dst;
    dst = sw;
  }
  *q_out = src;
  return 0;
}

// Split caps of the wide CholeskyQR3's Gram (which = 0, RGSV_WGRAM_SPLIT) and
// TRSM (which = 1, RGSV_WTRSM_SPLIT). cfg1 with 8 concurrent pairs (n = 1000,
// kp = 64): 713-720 pairs/s at 32 / 8, 720-723 at 16 / 2 and 8 / 2,
// 725-733 at 8 / 1 (fewer partials and no reduce pass for the TRSM).
static int wide_split(int which) {
  static const int v[2] = {[] {
                             const char* e = getenv("RGSV_WGRAM_SPLIT");
                             const int x = e ? atoi(e) : 0;
                             return x >= 1 ? x : 8;
                           }(),
                           [] {
                             const char* e = getenv("RGSV_WTRSM_SPLIT");
                             const int x = e ? atoi(e) : 0;
                             return x >= 1 ? x : 1;
                           }()};
  return v[which];
}

int cholqr3_wide(double* b, double* tmp, int64_t n, int64_t ldn, int k, int kp, double* gram,
                 double* linv, double* rinv, double* rdiag, double* scratch, size_t scratch_bytes,
                 int* status, double** qt_out, cudaStream_t st, int passes) {
  double* src = b;
  double* dst = tmp;
  for (int step = 0; step < passes; ++step) {
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
    g.max_split = wide_split(0);
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
    t.max_split = wide_split(1);
    if (int e = gemm_gtq(t, st)) return e;
    double* sw = src;
    src = dst;
    dst = sw;
  }
  *qt_out = src;
  return 0;
}

}  // namespace rgsv
