// Small-GSVD and comparative-analysis kernels.
//
//  k_stack        S = [B1[:l1]; B2[:l2]]          (engine.py:257 vstack)
//  k_copy_block   strided block copy / transpose  (L-block extraction)
//  k_jacobi_rows  one-sided (Hestenes) Jacobi on the rows of an L block:
//                 singular values with high relative accuracy, the role of
//                 LAPACK gesdd in engine._singular_values (engine.py:228-231)
//  k_comparative  spectrum completion (merged branch, engine.py:208-223),
//                 classification + snapping (engine.py:164-186), rho, theta,
//                 P1/P2 and D1/D2 (analysis.py:37-79) in one CTA
//  k_sumsq_*      deterministic two-stage sum of squares (core.sum_sq)
#include <math.h>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {

__global__ void k_stack(double* __restrict__ s, int64_t lds, const double* __restrict__ b1,
                        int64_t ld1, int l1, const double* __restrict__ b2, int64_t ld2, int l2,
                        int lp, int64_t n) {
  const int64_t total = (int64_t)lp * lds;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / lds);
    const int64_t c = e % lds;
    double v = 0.0;
    if (c < n) {
      if (r < l1) v = b1[(int64_t)r * ld1 + c];
      else if (r < l1 + l2) v = b2[(int64_t)(r - l1) * ld2 + c];
    }
    s[e] = v;
  }
}

// dst (rows x cols, ldd) = src block (optionally transposed: dst[i][j] = src[j][i]).
__global__ void k_copy_block(double* __restrict__ dst, int64_t ldd, const double* __restrict__ src,
                             int64_t lds, int rows, int cols, int transpose) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    dst[(int64_t)i * ldd + j] = transpose ? src[(int64_t)j * lds + i] : src[(int64_t)i * lds + j];
  }
}

struct JacobiJob {
  double* v;      // nv x len vectors (rows), modified in place
  int64_t ld;
  int nv;
  int len;
  double* sv_out;  // min(nv, len) values, descending
  int* nsv_out;
};

RGSV_DI int rr_index(int p, int round, int nplayers) {
  return p == 0 ? 0 : 1 + ((p - 1 + round) % (nplayers - 1));
}

constexpr int kJacobiMaxVec = 2048;

// One-sided Jacobi on the rows of J.v (in place), whole CTA; writes the
// sorted singular values and their count. Shared by k_jacobi_rows and the
// batched small-GSVD kernel.
__device__ void jacobi_rows_body(JacobiJob J, int max_sweeps, int* __restrict__ status) {
  __shared__ double nrm[kJacobiMaxVec];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int nout = J.nv < J.len ? J.nv : J.len;
  if (J.nv <= 0 || J.len <= 0) {
    if (tid == 0) *J.nsv_out = 0;
    return;
  }
  const int nve = J.nv + (J.nv & 1);
  const double tol = fmax(1e-15, sqrt((double)J.len) * 2.220446049250313e-16);
  // Zero-row floor: rows below 1e-14 of the largest row norm at entry are
  // rounding noise of a rank-deficient input (re-injected by every rotation
  // with a large row); they are neither rotated nor held against convergence.
  for (int i = warp; i < J.nv; i += nwarps) {
    const double* vi = J.v + (int64_t)i * J.ld;
    double sq = 0.0;
    for (int e = lane; e < J.len; e += 32) sq = fma(vi[e], vi[e], sq);
    sq = warp_sum(sq);
    if (lane == 0) nrm[i] = sq;
  }
  __syncthreads();
  double gmax = 0.0;
  for (int i = 0; i < J.nv; ++i) gmax = fmax(gmax, nrm[i]);
  const double floor2 = 1e-28 * gmax;
  __syncthreads();
  bool converged = (J.nv == 1);
  for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < nve - 1; ++round) {
      for (int p = warp; p < nve / 2; p += nwarps) {
        const int a = rr_index(p, round, nve), b = rr_index(nve - 1 - p, round, nve);
        if (a >= J.nv || b >= J.nv) continue;
        double* va = J.v + (int64_t)a * J.ld;
        double* vb = J.v + (int64_t)b * J.ld;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int e = lane; e < J.len; e += 32) {
          const double x = va[e], y = vb[e];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga != 0.0 && fmin(al, be) > floor2 && fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int e = lane; e < J.len; e += 32) {
            const double x = va[e], y = vb[e];
            va[e] = c * x - s * y;
            vb[e] = s * x + c * y;
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    converged = !__syncthreads_or(rotated);
  }
  if (!converged) {
    if (tid == 0) atomicOr(status, RGSV_ST_JACOBI);
  }
  for (int i = warp; i < J.nv; i += nwarps) {
    const double* vi = J.v + (int64_t)i * J.ld;
    double s = 0.0;
    for (int e = lane; e < J.len; e += 32) s = fma(vi[e], vi[e], s);
    s = warp_sum(s);
    if (lane == 0) nrm[i] = sqrt(s);
  }
  __syncthreads();
  for (int i = tid; i < J.nv; i += blockDim.x) {
    const double x = nrm[i];
    int rank = 0;
    for (int j = 0; j < J.nv; ++j) {
      const double y = nrm[j];
      rank += (y > x) || (y == x && j < i);
    }
    if (rank < nout) J.sv_out[rank] = x;
  }
  if (tid == 0) *J.nsv_out = nout;
  __syncthreads();
}

__global__ void __launch_bounds__(1024) k_jacobi_rows(JacobiJob j0, JacobiJob j1, int max_sweeps,
                                                       int* __restrict__ status, int use_smem) {
  JacobiJob J = blockIdx.x == 0 ? j0 : j1;
  extern __shared__ double jsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (use_smem && J.nv > 0 && J.len > 0) {  // stage the vectors in shared memory (ld len + 1)
    const int lds = J.len + 1;
    for (int i = warp; i < J.nv; i += nwarps)
      for (int e = lane; e < J.len; e += 32) jsm[i * lds + e] = J.v[(int64_t)i * J.ld + e];
    J.v = jsm;
    J.ld = lds;
    __syncthreads();
  }
  jacobi_rows_body(J, max_sweeps, status);
}

// ------------------------------------------- Jacobi SVD with vectors
// One-sided Jacobi on the nv rows of v (nv x len, in place) with the
// rotations accumulated into acc (nv x nv, starts at I): J v = diag(s) X with
// orthogonal rows of X. Outputs, ordered by singular value (descending, or
// ascending when `ascending`): sv[nv], xn (nv x len) = the unit rows of X
// (a zero row stays zero and is counted in *nzero for the caller's
// completion), jo (nv x nv) = the matching rows of J. For A with rows as
// vectors, A = J^T diag(s) X: U = jo^T, V^H = xn. Serves recover_gsvd's
// full SVDs of the L blocks (engine.py:322,340) -- off the hot path, so the
// vectors stay in global (L2-resident) memory.
__global__ void __launch_bounds__(512) k_jacobi_vec(double* __restrict__ v, int64_t ldv, int nv,
                                                    int len, double* __restrict__ acc,
                                                    int64_t ldacc, double* __restrict__ sv,
                                                    double* __restrict__ xn, int64_t ldx,
                                                    double* __restrict__ jo, int64_t ldj,
                                                    int ascending, int max_sweeps,
                                                    int* __restrict__ nzero,
                                                    int* __restrict__ status) {
  __shared__ double nrm[kJacobiMaxVec];
  __shared__ int ord[kJacobiMaxVec];
  __shared__ int s_zero;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int i = warp; i < nv; i += nwarps)
    for (int e = lane; e < nv; e += 32) acc[(int64_t)i * ldacc + e] = (i == e) ? 1.0 : 0.0;
  if (tid == 0) s_zero = 0;
  __syncthreads();
  const int nve = nv + (nv & 1);
  const double tol = fmax(1e-15, sqrt((double)len) * 2.220446049250313e-16);
  bool converged = (nv == 1);
  for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < nve - 1; ++round) {
      for (int p = warp; p < nve / 2; p += nwarps) {
        const int a = rr_index(p, round, nve), b = rr_index(nve - 1 - p, round, nve);
        if (a >= nv || b >= nv) continue;
        double* va = v + (int64_t)a * ldv;
        double* vb = v + (int64_t)b * ldv;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int e = lane; e < len; e += 32) {
          const double x = va[e], y = vb[e];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int e = lane; e < len; e += 32) {
            const double x = va[e], y = vb[e];
            va[e] = c * x - s * y;
            vb[e] = s * x + c * y;
          }
          double* ja = acc + (int64_t)a * ldacc;
          double* jb = acc + (int64_t)b * ldacc;
          for (int e = lane; e < nv; e += 32) {
            const double x = ja[e], y = jb[e];
            ja[e] = c * x - s * y;
            jb[e] = s * x + c * y;
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    converged = !__syncthreads_or(rotated);
  }
  if (!converged && tid == 0) atomicOr(status, RGSV_ST_JACOBI);
  for (int i = warp; i < nv; i += nwarps) {
    const double* vi = v + (int64_t)i * ldv;
    double s = 0.0;
    for (int e = lane; e < len; e += 32) s = fma(vi[e], vi[e], s);
    s = warp_sum(s);
    if (lane == 0) nrm[i] = sqrt(s);
  }
  __syncthreads();
  for (int i = tid; i < nv; i += blockDim.x) {
    const double x = nrm[i];
    int rank = 0;
    for (int j = 0; j < nv; ++j) {
      const double y = nrm[j];
      rank += ascending ? ((y < x) || (y == x && j < i)) : ((y > x) || (y == x && j < i));
    }
    ord[rank] = i;
    sv[rank] = x;
    if (x == 0.0) atomicAdd(&s_zero, 1);
  }
  __syncthreads();
  for (int r = warp; r < nv; r += nwarps) {
    const int i = ord[r];
    const double x = nrm[i];
    const double inv = x > 0.0 ? 1.0 / x : 0.0;
    for (int e = lane; e < len; e += 32) xn[(int64_t)r * ldx + e] = v[(int64_t)i * ldv + e] * inv;
    for (int e = lane; e < nv; e += 32) jo[(int64_t)r * ldj + e] = acc[(int64_t)i * ldacc + e];
  }
  if (tid == 0) *nzero = s_zero;
}

int launch_jacobi_vec(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                      double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj, int ascending,
                      int* nzero, int* status, cudaStream_t st) {
  if (nv < 1 || len < 1 || nv > kJacobiMaxVec) return RGSV_ERR_DIMENSION;
  k_jacobi_vec<<<1, 512, 0, st>>>(v, ldv, nv, len, acc, ldacc, sv, xn, ldx, jo, ldj, ascending,
                                  60, nzero, status);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// fp32 -> fp64 promotion of a row block (exact; the reference promotes fp32
// input to fp64 at GmpPair construction, core.py:51-54). Row-major, 16-byte
// vector loads when the pitches allow, zero padding up to the even pitch.
__global__ void k_convert_f32(const float* __restrict__ src, int64_t lds, int64_t rows,
                              int64_t cols, double* __restrict__ dst, int64_t ldd) {
  const int64_t c4 = (cols + 3) / 4;
  const int64_t total = rows * c4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / c4, c = (e % c4) * 4;
    const float* s = src + r * lds + c;
    double* d = dst + r * ldd + c;
    if (c + 4 <= cols && ((reinterpret_cast<uintptr_t>(s) & 15) == 0) &&
        ((reinterpret_cast<uintptr_t>(d) & 15) == 0)) {
      const float4 v = *reinterpret_cast<const float4*>(s);
      reinterpret_cast<double2*>(d)[0] = make_double2(v.x, v.y);
      reinterpret_cast<double2*>(d)[1] = make_double2(v.z, v.w);
    } else {
      for (int64_t q = 0; q < 4 && c + q < cols; ++q) d[q] = (double)s[q];
    }
  }
}

int launch_convert_f32(const float* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
                       int64_t ldd, cudaStream_t st) {
  const int64_t total = rows * ((cols + 3) / 4);
  if (total <= 0) return 0;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 16 * kSMs) blocks = 16 * kSMs;
  k_convert_f32<<<(int)blocks, 256, 0, st>>>(src, lds, rows, cols, dst, ldd);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// a (rows x cols) column j scaled by 1/d[j] (recover_gsvd, engine.py:335,357)
__global__ void k_scale_cols(double* __restrict__ a, int64_t lda, int rows, int cols,
                             const double* __restrict__ d) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e % cols);
    a[r * lda + c] = a[r * lda + c] / d[c];
  }
}

int launch_scale_cols(double* a, int64_t lda, int rows, int cols, const double* d,
                      cudaStream_t st) {
  const int64_t total = (int64_t)rows * cols;
  if (total <= 0) return 0;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 8 * kSMs) blocks = 8 * kSMs;
  k_scale_cols<<<blocks, 256, 0, st>>>(a, lda, rows, cols, d);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// ------------------------------------------------------ Householder QR
// Q of the Householder QR of the l x l leading block T = S[:, :l] of the
// stacked S = [B1; B2] (l <= n). LAPACK dgeqrf/dorgqr (numpy.linalg.qr,
// core.py:87, called by engine.py:257) process columns left to right, so for
// a wide S the Q factor depends on the first l columns only: Q(S) = Q(T).
// One CTA, T in shared memory; dgeqr2 (reflector per column, H = I - tau v
// v^T with v[0] = 1) then dorg2r (backward accumulation of Q = H0 .. H_{l-1}).
// Column signs of Q may differ from the reference's phase fix
// (core.py:88-95); singular values of its row blocks do not depend on them.
// Q of the l x l block in A (lda = l + 1; loaded from the first l columns of
// [B1; B2]), in place; copied to q when q != nullptr. Whole CTA.
__device__ void hh_small_body(const double* __restrict__ b1, int64_t ld1, int l1,
                              const double* __restrict__ b2, int64_t ld2, int l2,
                              double* __restrict__ q, int64_t ldq, double* A) {
  const int l = l1 + l2;
  const int lda = l + 1;
  __shared__ double w[512];
  __shared__ double tau[512];
  __shared__ double s_beta, s_scale, s_tau;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarp = nt >> 5;
  // 2-D thread view for element loops: row stride nwarp, column stride 32
  for (int i = warp; i < l; i += nwarp) {
    const double* src = (i < l1) ? b1 + (int64_t)i * ld1 : b2 + (int64_t)(i - l1) * ld2;
    for (int j = lane; j < l; j += 32) A[i * lda + j] = src[j];
  }
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    // reflector from A[j:, j] (dlarfg)
    if (warp == 0) {
      double ss = 0.0;
      for (int i = j + 1 + lane; i < l; i += 32) ss = fma(A[i * lda + j], A[i * lda + j], ss);
      ss = warp_sum(ss);
      if (lane == 0) {
        const double alpha = A[j * lda + j];
        if (ss == 0.0) {
          s_tau = 0.0;
          s_scale = 0.0;
          s_beta = alpha;
        } else {
          const double nrm = sqrt(fma(alpha, alpha, ss));
          const double beta = alpha >= 0.0 ? -nrm : nrm;
          s_tau = (beta - alpha) / beta;
          s_scale = 1.0 / (alpha - beta);
          s_beta = beta;
        }
        tau[j] = s_tau;
      }
    }
    __syncthreads();
    const double tj = s_tau, sc = s_scale;
    if (warp == 0) {
      for (int i = j + 1 + lane; i < l; i += 32) A[i * lda + j] *= sc;  // v, v[0] = 1 implicit
      if (lane == 0) A[j * lda + j] = s_beta;
    }
    __syncthreads();
    if (tj != 0.0) {
      // w[c] = tau v^T A[j:, c], c > j ; one warp per column, lanes over rows
      for (int c = j + 1 + warp; c < l; c += nwarp) {
        double acc0 = (lane == 0) ? A[j * lda + c] : 0.0, acc1 = 0.0;
        int i = j + 1 + lane;
        for (; i + 32 < l; i += 64) {
          acc0 = fma(A[i * lda + j], A[i * lda + c], acc0);
          acc1 = fma(A[(i + 32) * lda + j], A[(i + 32) * lda + c], acc1);
        }
        if (i < l) acc0 = fma(A[i * lda + j], A[i * lda + c], acc0);
        const double acc = warp_sum(acc0 + acc1);
        if (lane == 0) w[c] = acc * tj;
      }
      __syncthreads();
      for (int i = j + warp; i < l; i += nwarp) {
        const double vi = (i == j) ? 1.0 : A[i * lda + j];
        for (int c = j + 1 + lane; c < l; c += 32) A[i * lda + c] = fma(-vi, w[c], A[i * lda + c]);
      }
      __syncthreads();
    }
  }
  // dorg2r, in place: columns i+1.. already hold Q's columns; apply H(i)
  // from the left to A[i:, i+1:], then turn column i into H(i) e_i.
  for (int i = l - 1; i >= 0; --i) {
    const double ti = tau[i];
    if (i < l - 1 && ti != 0.0) {
      for (int c = i + 1 + warp; c < l; c += nwarp) {
        double acc0 = (lane == 0) ? A[i * lda + c] : 0.0, acc1 = 0.0;
        int r = i + 1 + lane;
        for (; r + 32 < l; r += 64) {
          acc0 = fma(A[r * lda + i], A[r * lda + c], acc0);
          acc1 = fma(A[(r + 32) * lda + i], A[(r + 32) * lda + c], acc1);
        }
        if (r < l) acc0 = fma(A[r * lda + i], A[r * lda + c], acc0);
        const double acc = warp_sum(acc0 + acc1);
        if (lane == 0) w[c] = acc * ti;
      }
      __syncthreads();
      for (int r = i + warp; r < l; r += nwarp) {
        const double vr = (r == i) ? 1.0 : A[r * lda + i];
        for (int c = i + 1 + lane; c < l; c += 32) A[r * lda + c] = fma(-vr, w[c], A[r * lda + c]);
      }
      __syncthreads();
    }
    for (int r = tid; r < l; r += nt) {
      if (r > i) A[r * lda + i] = -ti * A[r * lda + i];
      else if (r == i) A[r * lda + i] = 1.0 - ti;
      else A[r * lda + i] = 0.0;
    }
    __syncthreads();
  }
  if (q)
    for (int i = warp; i < l; i += nwarp)
      for (int j = lane; j < l; j += 32) q[(int64_t)i * ldq + j] = A[i * lda + j];
  __syncthreads();
}

template <bool SMEM>
__global__ void __launch_bounds__(512) k_householder_small(const double* __restrict__ b1,
                                                           int64_t ld1, int l1,
                                                           const double* __restrict__ b2,
                                                           int64_t ld2, int l2,
                                                           double* __restrict__ q, int64_t ldq,
                                                           double* __restrict__ gwork) {
  extern __shared__ double smh[];
  hh_small_body(b1, ld1, l1, b2, ld2, l2, q, ldq, SMEM ? smh : gwork);
}

// Register-resident variant for l <= 128: warp w owns columns c = w, w+16,
// ... (CPW = 8 columns), lane r holds rows r, r+32, r+64, r+96 of each owned
// column. Step j: the owner of column j forms the reflector (warp
// reductions, no barrier) and publishes v and tau in shared memory; one
// barrier; every warp applies H_j to its owned columns > j (interleaved warp
// dot products). Q is then formed backwards from the stored reflectors
// (dorg2r order), with the same column ownership.
constexpr int kHhWarps = 16, kHhCPW = 8, kHhRPL = 4;  // 16 x 8 = 128 columns, 4 x 32 = 128 rows

__global__ void __launch_bounds__(kHhWarps * 32) k_householder_reg(
    const double* __restrict__ b1, int64_t ld1, int l1, const double* __restrict__ b2,
    int64_t ld2, int l2, double* __restrict__ q, int64_t ldq, long long* __restrict__ prof) {
  extern __shared__ double V[];  // reflectors: column j in V[j * 129 + r]; tau at V[128 * 129 + j]
  double* tau_s = V + 128 * 129;
  const int l = l1 + l2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[kHhCPW][kHhRPL];
#pragma unroll
  for (int cc = 0; cc < kHhCPW; ++cc) {
    const int c = warp + kHhWarps * cc;
#pragma unroll
    for (int rr = 0; rr < kHhRPL; ++rr) {
      const int r = lane + 32 * rr;
      double v = 0.0;
      if (r < l && c < l) v = (r < l1) ? b1[(int64_t)r * ld1 + c] : b2[(int64_t)(r - l1) * ld2 + c];
      a[cc][rr] = v;
    }
  }
  // column j = slot * 16 + owner; `slot` is a compile-time index (unrolled)
  // so the owned-column registers are never indexed dynamically
#pragma unroll
  for (int slot = 0; slot < kHhCPW; ++slot) {
    for (int owner = 0; owner < kHhWarps; ++owner) {
      const int j = slot * kHhWarps + owner;
      if (j >= l) break;
      if (prof && threadIdx.x == 0 && j < 8) prof[3 * j] = clock64();
      if (warp == owner) {
        double ss = 0.0, alpha = 0.0;
#pragma unroll
        for (int rr = 0; rr < kHhRPL; ++rr) {
          const int r = lane + 32 * rr;
          const double xv = a[slot][rr];
          if (r > j && r < l) ss = fma(xv, xv, ss);
          if (r == j) alpha = xv;
        }
        ss = warp_sum(ss);
        alpha = warp_sum(alpha);  // exactly one lane contributes
        double tj, sc, beta;
        if (ss == 0.0) {
          tj = 0.0;
          sc = 0.0;
          beta = alpha;
        } else {
          const double nrm = sqrt(fma(alpha, alpha, ss));
          beta = alpha >= 0.0 ? -nrm : nrm;
          tj = (beta - alpha) / beta;
          sc = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int rr = 0; rr < kHhRPL; ++rr) {
          const int r = lane + 32 * rr;
          if (r > j && r < l) V[j * 129 + r] = a[slot][rr] * sc;
          if (r == j) a[slot][rr] = beta;
          else if (r > j) a[slot][rr] = 0.0;  // below-diagonal part now lives in V
        }
        if (lane == 0) {
          V[j * 129 + j] = 1.0;
          tau_s[j] = tj;
        }
      }
      __syncthreads();
      if (prof && threadIdx.x == 0 && j < 8) prof[3 * j + 1] = clock64();
      const double tj = tau_s[j];
      if (tj != 0.0) {
        double v[kHhRPL];
#pragma unroll
        for (int rr = 0; rr < kHhRPL; ++rr) {
          const int r = lane + 32 * rr;
          v[rr] = (r >= j && r < l) ? V[j * 129 + r] : 0.0;
        }
        double d[kHhCPW];
#pragma unroll
        for (int cc = 0; cc < kHhCPW; ++cc) {
          double acc = 0.0;
#pragma unroll
          for (int rr = 0; rr < kHhRPL; ++rr) acc = fma(v[rr], a[cc][rr], acc);
          d[cc] = acc;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int cc = 0; cc < kHhCPW; ++cc) d[cc] += __shfl_xor_sync(0xffffffffu, d[cc], o);
#pragma unroll
        for (int cc = 0; cc < kHhCPW; ++cc) {
          const int c = warp + kHhWarps * cc;
          if (c > j) {
            const double f = d[cc] * tj;
#pragma unroll
            for (int rr = 0; rr < kHhRPL; ++rr) a[cc][rr] = fma(-f, v[rr], a[cc][rr]);
          }
        }
      }
      if (prof && threadIdx.x == 0 && j < 8) prof[3 * j + 2] = clock64();
    }
  }
  if (prof && threadIdx.x == 0) prof[30] = clock64();
  // dorg2r: Q = H_0 ... H_{l-1} [I; 0]; walk i = l-1 .. 0 keeping Q[:, c] for
  // c > i in the owned registers, then set column i to H_i e_i.
#pragma unroll
  for (int cc = 0; cc < kHhCPW; ++cc)
#pragma unroll
    for (int rr = 0; rr < kHhRPL; ++rr) a[cc][rr] = 0.0;
#pragma unroll
  for (int slot = kHhCPW - 1; slot >= 0; --slot) {
    for (int owner = kHhWarps - 1; owner >= 0; --owner) {
      const int i = slot * kHhWarps + owner;
      if (i >= l) continue;
      const double ti = tau_s[i];
      double v[kHhRPL];
#pragma unroll
      for (int rr = 0; rr < kHhRPL; ++rr) {
        const int r = lane + 32 * rr;
        v[rr] = (r >= i && r < l) ? V[i * 129 + r] : 0.0;
      }
      if (ti != 0.0) {
        double d[kHhCPW];
#pragma unroll
        for (int cc = 0; cc < kHhCPW; ++cc) {
          double acc = 0.0;
#pragma unroll
          for (int rr = 0; rr < kHhRPL; ++rr) acc = fma(v[rr], a[cc][rr], acc);
          d[cc] = acc;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int cc = 0; cc < kHhCPW; ++cc) d[cc] += __shfl_xor_sync(0xffffffffu, d[cc], o);
#pragma unroll
        for (int cc = 0; cc < kHhCPW; ++cc) {
          const int c = warp + kHhWarps * cc;
          if (c > i) {
            const double f = d[cc] * ti;
#pragma unroll
            for (int rr = 0; rr < kHhRPL; ++rr) a[cc][rr] = fma(-f, v[rr], a[cc][rr]);
          }
        }
      }
      if (warp == owner) {  // column i := H_i e_i = e_i - tau v
#pragma unroll
        for (int rr = 0; rr < kHhRPL; ++rr) {
          const int r = lane + 32 * rr;
          a[slot][rr] = (r == i ? 1.0 : 0.0) - ti * v[rr];
        }
      }
    }
  }
  if (prof && threadIdx.x == 0) prof[31] = clock64();
#pragma unroll
  for (int cc = 0; cc < kHhCPW; ++cc) {
    const int c = warp + kHhWarps * cc;
    if (c >= l) continue;
#pragma unroll
    for (int rr = 0; rr < kHhRPL; ++rr) {
      const int r = lane + 32 * rr;
      if (r < l) q[(int64_t)r * ldq + c] = a[cc][rr];
    }
  }
}

int debug_householder_profile(const double* b1, int64_t ld1, int l1, const double* b2,
                              int64_t ld2, int l2, double* q, int64_t ldq, long long* prof,
                              cudaStream_t st) {
  const size_t vbytes = (128 * 129 + 128) * sizeof(double);
  cudaFuncSetAttribute(k_householder_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vbytes);
  k_householder_reg<<<1, kHhWarps * 32, vbytes, st>>>(b1, ld1, l1, b2, ld2, l2, q, ldq, prof);
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

size_t householder_small_smem(int l) {
  return (size_t)l * (l + 1) * sizeof(double);
}

int launch_householder_small(const double* b1, int64_t ld1, int l1, const double* b2, int64_t ld2,
                             int l2, double* q, int64_t ldq, double* gwork, cudaStream_t st) {
  const int l = l1 + l2;
  if (l > 512) return RGSV_ERR_DIMENSION;
  if (l <= kHhWarps * kHhCPW) {
    const size_t vbytes = (128 * 129 + 128) * sizeof(double);
    static bool attr_reg = false;
    if (!attr_reg) {
      if (cudaFuncSetAttribute(k_householder_reg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)vbytes) != cudaSuccess)
        return RGSV_ERR_CUDA;
      attr_reg = true;
    }
    k_householder_reg<<<1, kHhWarps * 32, vbytes, st>>>(b1, ld1, l1, b2, ld2, l2, q, ldq,
                                                        nullptr);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
  }
  const size_t smem = householder_small_smem(l);
  if (smem <= 200 * 1024) {  // + 8 KB static stays under the 227 KB per-CTA limit
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_householder_small<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
          cudaSuccess)
        return RGSV_ERR_CUDA;
      attr = true;
    }
    k_householder_small<true><<<1, 512, smem, st>>>(b1, ld1, l1, b2, ld2, l2, q, ldq, nullptr);
  } else {
    k_householder_small<false><<<1, 512, 0, st>>>(b1, ld1, l1, b2, ld2, l2, q, ldq, gwork);
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// --------------------------------------------- tall Householder QR (robust)
// Q (m x w) and diag(R) of y (m x w) by Householder reflections in ONE CTA
// over global (L2-resident) memory, with the phase fix of core.reduced_qr
// (core.py:88-95: diag(R) >= 0). Rank-deficient input is fine: a zero column
// gets tau = 0 and R_jj = 0, exactly like LAPACK dgeqr2. Used for the
// adaptive range finder's blocks and as the CholeskyQR fallback; the matrix
// is updated in place in `a` (m x w, ld lda), Q written to q.
__global__ void __launch_bounds__(512) k_householder_tall(double* __restrict__ a, int64_t lda,
                                                          int m, int w, double* __restrict__ q,
                                                          int64_t ldq, double* __restrict__ rdiag,
                                                          double* __restrict__ tau,
                                                          int comp_count) {
  __shared__ double wv[1024];
  __shared__ double s_beta, s_scale, s_tau;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarp = nt >> 5;
  const int kmin = m < w ? m : w;
  for (int j = 0; j < kmin; ++j) {
    if (warp == 0) {
      double ss = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) ss = fma(a[i * lda + j], a[i * lda + j], ss);
      ss = warp_sum(ss);
      if (lane == 0) {
        const double alpha = a[(int64_t)j * lda + j];
        if (ss == 0.0) {
          s_tau = 0.0;
          s_scale = 0.0;
          s_beta = alpha;
        } else {
          const double nrm = sqrt(fma(alpha, alpha, ss));
          const double beta = alpha >= 0.0 ? -nrm : nrm;
          s_tau = (beta - alpha) / beta;
          s_scale = 1.0 / (alpha - beta);
          s_beta = beta;
        }
        tau[j] = s_tau;
      }
    }
    __syncthreads();
    const double tj = s_tau, sc = s_scale;
    for (int i = j + 1 + tid; i < m; i += nt) a[(int64_t)i * lda + j] *= sc;
    if (tid == 0) a[(int64_t)j * lda + j] = s_beta;
    __syncthreads();
    if (tj != 0.0) {
      for (int c = j + 1 + warp; c < w; c += nwarp) {
        double acc = (lane == 0) ? a[(int64_t)j * lda + c] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32)
          acc = fma(a[(int64_t)i * lda + j], a[(int64_t)i * lda + c], acc);
        acc = warp_sum(acc);
        if (lane == 0) wv[c] = acc * tj;
      }
      __syncthreads();
      for (int i = j + warp; i < m; i += nwarp) {
        const double vi = (i == j) ? 1.0 : a[(int64_t)i * lda + j];
        for (int c = j + 1 + lane; c < w; c += 32)
          a[(int64_t)i * lda + c] = fma(-vi, wv[c], a[(int64_t)i * lda + c]);
      }
      __syncthreads();
    }
  }
  if (comp_count > 0) {
    // orthonormal completion (engine.py:278-291): columns kmin .. kmin+count
    // of the COMPLETE Q = H0 .. H_{k-1} (numpy.linalg.qr mode="complete"),
    // i.e. the reflectors applied to e_kmin .. e_{kmin+count-1}; no phase fix
    for (int i = warp; i < m; i += nwarp)
      for (int c = lane; c < comp_count; c += 32)
        q[(int64_t)i * ldq + c] = (i == kmin + c) ? 1.0 : 0.0;
    __syncthreads();
    for (int j = kmin - 1; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      for (int c = warp; c < comp_count; c += nwarp) {
        double acc = (lane == 0) ? q[(int64_t)j * ldq + c] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32)
          acc = fma(a[(int64_t)i * lda + j], q[(int64_t)i * ldq + c], acc);
        acc = warp_sum(acc);
        if (lane == 0) wv[c] = acc * tj;
      }
      __syncthreads();
      for (int i = j + warp; i < m; i += nwarp) {
        const double vi = (i == j) ? 1.0 : a[(int64_t)i * lda + j];
        for (int c = lane; c < comp_count; c += 32)
          q[(int64_t)i * ldq + c] = fma(-vi, wv[c], q[(int64_t)i * ldq + c]);
      }
      __syncthreads();
    }
    return;
  }
  // diag(R) and the phase fix: column j of Q is negated when R_jj < 0
  __shared__ double sgn[1024];
  for (int j = tid; j < kmin; j += nt) {
    const double d = a[(int64_t)j * lda + j];
    sgn[j] = d < 0.0 ? -1.0 : 1.0;
    rdiag[j] = fabs(d);
  }
  // Q = H0 ... H_{k-1} [I; 0] (m x kmin), backwards in q
  for (int i = warp; i < m; i += nwarp)
    for (int c = lane; c < kmin; c += 32) q[(int64_t)i * ldq + c] = (i == c) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = kmin - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    for (int c = j + warp; c < kmin; c += nwarp) {
      double acc = (lane == 0) ? q[(int64_t)j * ldq + c] : 0.0;
      for (int i = j + 1 + lane; i < m; i += 32)
        acc = fma(a[(int64_t)i * lda + j], q[(int64_t)i * ldq + c], acc);
      acc = warp_sum(acc);
      if (lane == 0) wv[c] = acc * tj;
    }
    __syncthreads();
    for (int i = j + warp; i < m; i += nwarp) {
      const double vi = (i == j) ? 1.0 : a[(int64_t)i * lda + j];
      for (int c = j + lane; c < kmin; c += 32)
        q[(int64_t)i * ldq + c] = fma(-vi, wv[c], q[(int64_t)i * ldq + c]);
    }
    __syncthreads();
  }
  for (int i = warp; i < m; i += nwarp)
    for (int c = lane; c < kmin; c += 32) q[(int64_t)i * ldq + c] *= sgn[c];
}

int launch_householder_tall(double* a, int64_t lda, int m, int w, double* q, int64_t ldq,
                            double* rdiag, double* tau, int comp_count, cudaStream_t st) {
  if (w > 1024 || comp_count > 1024 || m < 1 || w < 0 || comp_count < 0) return RGSV_ERR_DIMENSION;
  if (w == 0 && comp_count == 0) return RGSV_ERR_DIMENSION;
  if (comp_count > 0 && (w > m || w + comp_count > m)) return RGSV_ERR_DIMENSION;
  k_householder_tall<<<1, 512, 0, st>>>(a, lda, m, w, q, ldq, rdiag, tau, comp_count);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// y (rows x cols) += alpha * x, strided
__global__ void k_axpy(double* __restrict__ y, int64_t ldy, const double* __restrict__ x,
                       int64_t ldx, int rows, int cols, double alpha) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    y[r * ldy + c] = fma(alpha, x[r * ldx + c], y[r * ldy + c]);
  }
}

int launch_axpy(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols,
                double alpha, cudaStream_t st) {
  const int64_t total = (int64_t)rows * cols;
  if (total <= 0) return 0;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 8 * kSMs) blocks = 8 * kSMs;
  k_axpy<<<blocks, 256, 0, st>>>(y, ldy, x, ldx, rows, cols, alpha);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// ---------------------------------------------------------- comparative
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < nw; ++w) tot += red[w];  // fixed order, every thread
  return tot;
}

// mode 0: from L-block singular values (complete + classify + snap);
// mode 1: from a given spectrum (sv1 = alphas, sv2 = betas, r = r_given);
// mode 2: entropy of a given probability vector sv1 (scalars[0] = D,
//         scalars[2] = sum p).
__device__ void comparative_body(const double* __restrict__ sv1, const int* __restrict__ nsv,
                                 const double* __restrict__ sv2, int64_t n, double tol,
                                 double* __restrict__ A, double* __restrict__ B,
                                 double* __restrict__ rho, double* __restrict__ theta,
                                 double* __restrict__ p1, double* __restrict__ p2,
                                 double* __restrict__ scalars, int* __restrict__ counts,
                                 int* __restrict__ status, double* red, int branch = 0);

__global__ void __launch_bounds__(1024) k_comparative(
    const double* __restrict__ sv1, const int* __restrict__ nsv, const double* __restrict__ sv2,
    int64_t n, double tol, double* __restrict__ A, double* __restrict__ B,
    double* __restrict__ rho, double* __restrict__ theta, double* __restrict__ p1,
    double* __restrict__ p2, double* __restrict__ scalars, int* __restrict__ counts,
    int* __restrict__ status, int mode, int r_given) {
  __shared__ double red[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (mode == 2) {
    double sp = 0.0, ent = 0.0;
    for (int64_t i = tid; i < n; i += nt) {
      const double q = sv1[i];
      sp += q;
      if (q > 0.0) ent = fma(q, log(q), ent);
    }
    sp = block_sum(sp, red);
    ent = block_sum(ent, red);
    if (tid == 0) {
      double d = -ent / log((double)n);
      scalars[0] = fmin(fmax(d, 0.0), 1.0) + 0.0;
      scalars[2] = sp;
    }
    return;
  }
  if (mode == 1) {
    double sa = 0.0, sb = 0.0;
    const double quarter_pi = 0.7853981633974483;
    for (int64_t i = tid; i < n; i += nt) {
      const double a = sv1[i], b = sv2[i];
      rho[i] = (i < r_given) ? __longlong_as_double(0x7ff0000000000000LL) : a / b;
      theta[i] = atan2(a, b) - quarter_pi;
      sa = fma(a, a, sa);
      sb = fma(b, b, sb);
    }
    sa = block_sum(sa, red);
    sb = block_sum(sb, red);
    if (!(sa > 0.0) || !(sb > 0.0)) {
      if (tid == 0) atomicOr(status, RGSV_ST_DEGENERATE);
      return;
    }
    double e1 = 0.0, e2 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t i = tid; i < n; i += nt) {
      const double a = sv1[i], b = sv2[i];
      const double q1 = a * a / sa, q2 = b * b / sb;
      p1[i] = q1;
      p2[i] = q2;
      s1 += q1;
      s2 += q2;
      if (q1 > 0.0) e1 = fma(q1, log(q1), e1);
      if (q2 > 0.0) e2 = fma(q2, log(q2), e2);
    }
    s1 = block_sum(s1, red);
    s2 = block_sum(s2, red);
    e1 = block_sum(e1, red);
    e2 = block_sum(e2, red);
    if (tid == 0) {
      const double ln = log((double)n);
      scalars[0] = fmin(fmax(-e1 / ln, 0.0), 1.0) + 0.0;
      scalars[1] = fmin(fmax(-e2 / ln, 0.0), 1.0) + 0.0;
      scalars[2] = s1;
      scalars[3] = s2;
    }
    return;
  }
  // mode 0: merged completion (default); 3 / 4: branch "first" / "second"
  comparative_body(sv1, nsv, sv2, n, tol, A, B, rho, theta, p1, p2, scalars, counts, status, red,
                   mode == 3 ? 1 : (mode == 4 ? 2 : 0));
}

// spectrum completion + classification + comparative quantities (modes 0 /
// 3 / 4 of k_comparative); whole CTA, `red` = 32 doubles of shared scratch.
__device__ void comparative_body(const double* __restrict__ sv1, const int* __restrict__ nsv,
                                 const double* __restrict__ sv2, int64_t n, double tol,
                                 double* __restrict__ A, double* __restrict__ B,
                                 double* __restrict__ rho, double* __restrict__ theta,
                                 double* __restrict__ p1, double* __restrict__ p2,
                                 double* __restrict__ scalars, int* __restrict__ counts,
                                 int* __restrict__ status, double* red, int branch) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t c1 = nsv[0], c2 = nsv[1];
  double cr = 0.0, cza = 0.0;
  for (int64_t i = tid; i < n; i += nt) {
    const double ar = (i < c1) ? fmin(fmax(sv1[i], 0.0), 1.0) : 0.0;
    const double br = (i >= n - c2) ? fmin(fmax(sv2[n - 1 - i], 0.0), 1.0) : 0.0;
    double a, b;
    // numpy evaluates sqrt(1.0 - x**2) with two roundings; keep them
    // (no FMA contraction) so the completed spectrum matches bit for bit.
    // branch 1 / 2 force the one-sided completion of engine.py:211-219.
    if (branch == 1) {
      a = ar;
      b = sqrt(__dsub_rn(1.0, __dmul_rn(ar, ar)));
    } else if (branch == 2) {
      a = sqrt(__dsub_rn(1.0, __dmul_rn(br, br)));
      b = br;
    } else if (ar <= br) {
      a = ar;
      b = sqrt(__dsub_rn(1.0, __dmul_rn(ar, ar)));
    } else {
      a = sqrt(__dsub_rn(1.0, __dmul_rn(br, br)));
      b = br;
    }
    A[i] = a;
    B[i] = b;
    cr += (b < tol) ? 1.0 : 0.0;
    cza += (a < tol) ? 1.0 : 0.0;
  }
  const int64_t r = (int64_t)block_sum(cr, red);
  const int64_t za = (int64_t)block_sum(cza, red);
  const int64_t s = n - r - za;
  if (s < 0) {
    if (tid == 0) {
      atomicOr(status, RGSV_ST_CLASSIFY);
      counts[0] = (int)r;
      counts[1] = (int)s;
    }
    return;
  }
  double sa = 0.0, sb = 0.0;
  const double quarter_pi = 0.7853981633974483;  // math.pi / 4
  for (int64_t i = tid; i < n; i += nt) {
    double a = A[i], b = B[i];
    if (i < r) {
      b = 0.0;
      a = 1.0;
    }
    if (za && i >= n - za) {
      a = 0.0;
      b = 1.0;
    }
    A[i] = a;
    B[i] = b;
    rho[i] = (i < r) ? __longlong_as_double(0x7ff0000000000000LL) : a / b;
    theta[i] = atan2(a, b) - quarter_pi;
    sa = fma(a, a, sa);
    sb = fma(b, b, sb);
  }
  sa = block_sum(sa, red);
  sb = block_sum(sb, red);
  if (tid == 0) {
    counts[0] = (int)r;
    counts[1] = (int)s;
  }
  if (!(sa > 0.0) || !(sb > 0.0)) {
    if (tid == 0) atomicOr(status, RGSV_ST_DEGENERATE);
    return;
  }
  double s1 = 0.0, s2 = 0.0, e1 = 0.0, e2 = 0.0;
  for (int64_t i = tid; i < n; i += nt) {
    const double a = A[i], b = B[i];
    const double q1 = a * a / sa, q2 = b * b / sb;
    p1[i] = q1;
    p2[i] = q2;
    s1 += q1;
    s2 += q2;
    if (q1 > 0.0) e1 = fma(q1, log(q1), e1);
    if (q2 > 0.0) e2 = fma(q2, log(q2), e2);
  }
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  e1 = block_sum(e1, red);
  e2 = block_sum(e2, red);
  if (tid == 0) {
    const double ln = log((double)n);
    double d1 = -e1 / ln, d2 = -e2 / ln;
    d1 = fmin(fmax(d1, 0.0), 1.0) + 0.0;
    d2 = fmin(fmax(d2, 0.0), 1.0) + 0.0;
    scalars[0] = d1;
    scalars[1] = d2;
    scalars[2] = s1;
    scalars[3] = s2;
    if (n < 2 || fabs(s1 - 1.0) > 1e-10 || fabs(s2 - 1.0) > 1e-10)
      atomicOr(status, RGSV_ST_NOT_NORMALIZED);
  }
}

// ------------------------------------------------- batched small GSVD
// One CTA per pair j: stacked QR of [B1_j; B2_j] (k1 + k2 = l <= n, so the
// Q of the leading l x l block, engine.py:257), Jacobi singular values of
// L1 = Q[:k1] and L2 = Q[k1:] (engine.py:228-231), then the spectrum /
// classification / comparative kernel body (engine.py:189-225,
// analysis.py:37-102) -- all in shared memory, one launch for the batch.
// Per pair outputs: res[j] = {alphas, betas, rho, theta, p1, p2 (n each),
// scalars (4), sv1 (k1), sv2 (k2)}, ints[j] = {nsv1, nsv2, r, s},
// status[j] |= bits.
__global__ void __launch_bounds__(256) k_batch_small(const double* __restrict__ b, int64_t ldb,
                                                     int64_t b_stride, int k1, int k2, int n,
                                                     double tol, double* __restrict__ res,
                                                     int64_t res_stride, int* __restrict__ ints,
                                                     int* __restrict__ status,
                                                     const int* __restrict__ mat_status) {
  extern __shared__ double sbs[];
  __shared__ double red[32];
  __shared__ double sv[128];
  __shared__ int nsv[2];
  const int j = blockIdx.x;
  const int l = k1 + k2;
  const double* b1 = b + (int64_t)(2 * j) * b_stride;
  const double* b2 = b + (int64_t)(2 * j + 1) * b_stride;
  double* A = sbs;  // l x (l + 1)
  hh_small_body(b1, ldb, k1, b2, ldb, k2, nullptr, 0, A);
  int* st = status + j;
  if (threadIdx.x == 0 && mat_status) atomicOr(st, mat_status[2 * j] | mat_status[2 * j + 1]);
  JacobiJob J1{A, l + 1, k1, l, sv, nsv};
  jacobi_rows_body(J1, 60, st);
  JacobiJob J2{A + (int64_t)k1 * (l + 1), l + 1, k2, l, sv + 64, nsv + 1};
  jacobi_rows_body(J2, 60, st);
  double* o = res + (int64_t)j * res_stride;
  comparative_body(sv, nsv, sv + 64, n, tol, o, o + n, o + 2 * n, o + 3 * n, o + 4 * n,
                   o + 5 * n, o + 6 * n, ints + 4 * j + 2, st, red);
  __syncthreads();
  // GsvSpectrum invariants (engine.py:108-125) checked here, so the host
  // reads one status word per pair instead of re-scanning every spectrum;
  // the same arithmetic as the host checks (no FMA contraction)
  if (!(*(volatile int*)st & (RGSV_ST_CLASSIFY | RGSV_ST_DEGENERATE))) {
    const int r = ints[4 * j + 2], s = ints[4 * j + 3];
    int bad = (r < 0 || s < 0 || r + s > n) ? 1 : 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double a = o[i], bb = o[n + i];
      bad |= !(a >= 0.0 && a <= 1.0 && bb >= 0.0 && bb <= 1.0);
      if (i + 1 < n)
        bad |= (__dsub_rn(o[i + 1], a) > 1e-12) | (__dsub_rn(o[n + i + 1], bb) < -1e-12);
      bad |= !(fabs(__dsub_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(bb, bb)), 1.0)) <= 1e-12);
      bad |= (i < r && bb != 0.0) | (i >= r + s && a != 0.0);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(st, RGSV_ST_SPECTRUM);
  }
  for (int i = threadIdx.x; i < k1; i += blockDim.x) o[6 * n + 4 + i] = sv[i];
  for (int i = threadIdx.x; i < k2; i += blockDim.x) o[6 * n + 4 + k1 + i] = sv[64 + i];
  if (threadIdx.x == 0) {
    ints[4 * j] = nsv[0];
    ints[4 * j + 1] = nsv[1];
  }
}

int launch_batch_small(const double* b, int64_t ldb, int64_t b_stride, int npairs, int k1, int k2,
                       int n, double tol, double* res, int64_t res_stride, int* ints,
                       int* status, const int* mat_status, cudaStream_t st) {
  const int l = k1 + k2;
  if (npairs < 1 || k1 < 1 || k2 < 1 || k1 > 64 || k2 > 64 || l > n || l > 128)
    return RGSV_ERR_DIMENSION;
  const size_t smem = (size_t)l * (l + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_batch_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             140 * 1024) != cudaSuccess)
      return RGSV_ERR_CUDA;
    attr = true;
  }
  k_batch_small<<<npairs, 256, smem, st>>>(b, ldb, b_stride, k1, k2, n, tol, res, res_stride, ints,
                                           status, mat_status);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// ------------------------------------------------------------- sum of squares
__global__ void k_sumsq_partial(const double* __restrict__ a, int64_t lda, int64_t rows,
                                int64_t cols, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[(e / cols) * lda + (e % cols)];
    s = fma(x, x, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------ host wrappers
int launch_stack(double* s, int64_t lds, const double* b1, int64_t ld1, int l1, const double* b2,
                 int64_t ld2, int l2, int lp, int64_t n, cudaStream_t st) {
  const int64_t total = (int64_t)lp * lds;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 4 * kSMs) blocks = 4 * kSMs;
  if (blocks < 1) blocks = 1;
  k_stack<<<blocks, 256, 0, st>>>(s, lds, b1, ld1, l1, b2, ld2, l2, lp, n);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int launch_copy_block(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols,
                      int transpose, cudaStream_t st) {
  const int64_t total = (int64_t)rows * cols;
  if (total <= 0) return 0;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 4 * kSMs) blocks = 4 * kSMs;
  k_copy_block<<<blocks, 256, 0, st>>>(dst, ldd, src, lds, rows, cols, transpose);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int launch_jacobi(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1, double* v2,
                  int64_t ld2, int nv2, int len2, double* sv2, int* nsv2, int* status,
                  cudaStream_t st) {
  if (nv1 > kJacobiMaxVec || nv2 > kJacobiMaxVec) return RGSV_ERR_DIMENSION;
  JacobiJob a{v1, ld1, nv1, len1, sv1, nsv1};
  JacobiJob b{v2, ld2, nv2, len2, sv2, nsv2};
  const size_t need = (size_t)max(nv1 * (len1 + 1), nv2 * (len2 + 1)) * sizeof(double);
  const int use_smem = need <= 200 * 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_jacobi_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024) != cudaSuccess)
      return RGSV_ERR_CUDA;
    attr = true;
  }
  k_jacobi_rows<<<2, 1024, use_smem ? need : 0, st>>>(a, b, 60, status, use_smem);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int launch_comparative(const double* sv1, const int* nsv, const double* sv2, int64_t n, double tol,
                       double* a, double* b, double* rho, double* theta, double* p1, double* p2,
                       double* scalars, int* counts, int* status, int mode, int r_given,
                       cudaStream_t st) {
  k_comparative<<<1, 1024, 0, st>>>(sv1, nsv, sv2, n, tol, a, b, rho, theta, p1, p2, scalars,
                                    counts, status, mode, r_given);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int launch_sumsq(const double* a, int64_t lda, int64_t rows, int64_t cols, double* out,
                 double* part, int max_parts, cudaStream_t st) {
  int64_t total = rows * cols;
  int blocks = (int)((total + 1023) / 1024);
  if (blocks > max_parts) blocks = max_parts;
  if (blocks < 1) blocks = 1;
  k_sumsq_partial<<<blocks, 256, 0, st>>>(a, lda, rows, cols, part);
  note_launch();
  k_sum_final<<<1, 256, 0, st>>>(part, blocks, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int launch_sum(const double* part, int n, double* out, cudaStream_t st) {
  k_sum_final<<<1, 256, 0, st>>>(part, n, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

}  // namespace rgsv
