// Multi-CTA dense factorizations of the small GSVD stage (SURVEY.md §2b
// K6/K7) and of the rank validation (engine.py:55-61):
//
//  k_hhqr     blocked Householder QR (LAPACK dgeqrf + dorgqr semantics) of
//             an M x N matrix stacked from two row sources. One cooperative
//             launch: the panel (nb columns, shared memory) is factored by
//             CTA 0 with its compact-WY factor T (dlarft), then every CTA
//             applies I - V T^T V^T to a slice of the trailing columns; Q is
//             accumulated backwards the same way (dorgqr). Serves the
//             stacked reduced QR of engine.py:257 (core.reduced_qr,
//             core.py:79-96, numpy.linalg.qr -> dgeqrf/dorgqr).
//  k_bjacobi  blocked one-sided Jacobi SVD (singular values) on the rows of
//             a matrix: rows are grouped in blocks of 16, block pairs are
//             scheduled round-robin over CTAs; each CTA forms the 32 x 32
//             Gram of its pair with DMMA, solves it by cyclic two-sided
//             Jacobi with accumulated rotations, and rotates its 32 rows.
//             Convergence is judged on Grams recomputed from the rotated
//             rows, so the values keep one-sided Jacobi's accuracy. Serves
//             engine._singular_values (engine.py:228-231, gesdd) and
//             core.svd values (core.py:99-106).
//
// Both run as ONE cooperative launch with a global-memory grid barrier (the
// counters are zeroed by a memset node in the same stream), so they are
// graph-capturable and need no host round trips between sweeps or panels.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {

// ------------------------------------------------------------ grid barrier
RGSV_DI unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Barrier over the `nblocks` CTAs of one job. `ctr` starts at 0; `epoch`
// is the CTA-local count of barriers passed so far (identical in all CTAs).
RGSV_DI void grid_barrier(unsigned* ctr, unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned target = epoch * nblocks;
    while (ld_acquire_u32(ctr) < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

// Hardware barrier over the CTAs of this thread-block cluster (all threads).
RGSV_DI void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::
          : "memory");
}

RGSV_DI double block_sum(double v, double* red) {  // blockDim.x = 256, red >= 8 doubles
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // red may still be read by a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w];
  return s;
}

constexpr int kDenseThreads = 256;

// =================================================================== QR
constexpr int kHhThreads = 512;  // 16 warps
constexpr int kHhChunk = 16;     // trailing columns per CTA work item

struct HhArgs {
  const double* b1;
  int64_t ld1;
  int m1;
  const double* b2;
  int64_t ld2;
  int m2;
  int N;       // columns (all of them are updated; K = min(M, N) are factored)
  double* a;   // work, M x N (lda)
  int64_t lda;
  double* q;   // out, M x K (ldq)
  int64_t ldq;
  double* r;   // optional out, K x N upper trapezoid (ldr)
  int64_t ldr;
  double* tb;  // panels x 32 x 32 compact-WY factors
  int nb;
  int phase_fix;
  unsigned* bar;
  long long* prof;  // debug: globaltimer stamps of CTA 0 (nullptr in production)
};

RGSV_DI long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Stage the reflector block V of the panel at (j0, j0) (mp x jb, unit lower
// trapezoid) into shared memory Vs (ld nb + 1).
__device__ void stage_v(const double* a, int64_t lda, int j0, int mp, int jb, int ldv, double* Vs) {
  for (int e = threadIdx.x; e < mp * jb; e += kHhThreads) {
    const int i = e / jb, c = e % jb;
    Vs[i * ldv + c] = i > c ? a[(int64_t)(j0 + i) * lda + j0 + c] : (i == c ? 1.0 : 0.0);
  }
  __syncthreads();
}

// C[j0:j0+mp, c0:c0+cw] := (I - V Tm V^T) C with Tm = T^T (trans = 1: H^T,
// geqrf's trailing update) or T (trans = 0: dorgqr's backward accumulation).
// V staged in Vs; T (32 x 32, upper) in shared memory.
__device__ void apply_wy(const double* Vs, int ldv, int mp, int jb, const double* T, int trans,
                         double* c, int64_t ldc, int j0, int c0, int cw, double* W, double* W2) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // W[x][y] = sum_i V[i][x] C[i][y]: lane = x, warp = y (16 warps = 16 columns)
  {
    const int x = lane, y = warp;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (y < cw && x < jb) {
      const double* cp = c + (int64_t)j0 * ldc + c0 + y;
      int i = x;  // V[i][x] = 0 for i < x
      for (; i + 3 < mp; i += 4) {
        a0 = fma(Vs[i * ldv + x], cp[(int64_t)i * ldc], a0);
        a1 = fma(Vs[(i + 1) * ldv + x], cp[(int64_t)(i + 1) * ldc], a1);
        a2 = fma(Vs[(i + 2) * ldv + x], cp[(int64_t)(i + 2) * ldc], a2);
        a3 = fma(Vs[(i + 3) * ldv + x], cp[(int64_t)(i + 3) * ldc], a3);
      }
      for (; i < mp; ++i) a0 = fma(Vs[i * ldv + x], cp[(int64_t)i * ldc], a0);
    }
    W[x * 17 + y] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  {
    const int x = lane, y = warp;
    double acc = 0.0;
    if (x < jb && y < cw) {
      if (trans) {  // (T^T W)[x] = sum_{z <= x} T[z][x] W[z]
        for (int z = 0; z <= x; ++z) acc = fma(T[z * 33 + x], W[z * 17 + y], acc);
      } else {  // (T W)[x] = sum_{z >= x} T[x][z] W[z]
        for (int z = x; z < jb; ++z) acc = fma(T[x * 33 + z], W[z * 17 + y], acc);
      }
    }
    W2[x * 17 + y] = acc;
  }
  __syncthreads();
  // C[i][y] -= sum_x V[i][x] W2[x][y]: 32 rows x 16 columns per pass
  for (int e = tid; e < mp * kHhChunk; e += kHhThreads) {
    const int i = e >> 4, y = e & 15;
    if (y < cw) {
      const int xe = i < jb - 1 ? i : jb - 1;  // V[i][x] = 0 for x > i
      double acc = 0.0;
      for (int x = 0; x <= xe; ++x) acc = fma(Vs[i * ldv + x], W2[x * 17 + y], acc);
      c[(int64_t)(j0 + i) * ldc + c0 + y] -= acc;
    }
  }
  __syncthreads();
}

// dgeqr2 + dlarft of the panel in shared memory P (mp x jb, ld ldp) with one
// CTA barrier per column: lane c of every warp owns column c; warp w owns
// rows i = w (mod 16). One reduction per column yields, for every lane c,
// d_c = sum_{i > jj} x_i P[i][c] with x = P[:, jj]: d_jj = ||x_tail||^2 (the
// reflector norm), d_c for c > jj the reflector dot products (w = P[jj][c] +
// scale * d_c) and for c < jj the dlarft column V[:, c]^T v (same formula,
// as P[jj][c] = V[jj][c] there). T is kept with ld 33.
__device__ void panel_qr(double* P, int ldp, int mp, int jb, double* T, double* red,
                         double* tau_s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane;
  for (int jj = 0; jj < jb; ++jj) {
    double d = 0.0;
    if (c < jb) {
      for (int i = warp; i < mp; i += 16) {
        if (i > jj) d = fma(P[i * ldp + jj], P[i * ldp + c], d);
      }
    }
    // double-buffered partials (16 x 32) + row jj (32): the owner warp of
    // row jj publishes it before the barrier and rewrites it right after
    double* rb = red + (jj & 1) * 17 * 32;
    rb[warp * 32 + lane] = d;
    if (warp == (jj & 15)) rb[16 * 32 + lane] = (c < jb) ? P[jj * ldp + c] : 0.0;
    __syncthreads();
    double wp = 0.0;
#pragma unroll
    for (int w = 0; w < 16; ++w) wp += rb[w * 32 + lane];
    const double ss = __shfl_sync(0xffffffffu, wp, jj);
    const double alpha = rb[16 * 32 + jj];
    double tj, sc, beta;
    if (ss == 0.0) {  // H = I (dlarfg with a zero tail)
      tj = 0.0;
      sc = 0.0;
      beta = alpha;
    } else {
      const double nrm = sqrt(fma(alpha, alpha, ss));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    const double rowjj = rb[16 * 32 + lane];
    const double wc = fma(sc, wp, rowjj);  // c > jj: v^T P[:, c];  c < jj: V[:, c]^T v
    if (warp == 0) {  // dlarft column jj: T[0:jj, jj] = -tau T[0:jj, 0:jj] S[0:jj, jj]
      double acc = 0.0;
      for (int l = 0; l < jj; ++l) {
        const double sl = __shfl_sync(0xffffffffu, wc, l);
        if (lane <= l) acc = fma(T[lane * 33 + l], sl, acc);
      }
      if (lane < jj) T[lane * 33 + jj] = -tj * acc;
      if (lane == jj) {
        T[jj * 33 + jj] = tj;
        tau_s[jj] = tj;
      }
    }
    // apply H_jj to the owned rows (columns > jj) and store v in column jj
    const double tw = tj * wc;
    for (int i = warp; i < mp; i += 16) {
      if (i < jj) continue;
      const double x = P[i * ldp + jj];
      __syncwarp();
      if (i == jj) {
        if (c > jj && c < jb) P[i * ldp + c] = fma(-1.0, tw, P[i * ldp + c]);
        if (c == jj) P[i * ldp + c] = beta;
      } else {
        const double v = x * sc;
        if (c > jj && c < jb && tj != 0.0) P[i * ldp + c] = fma(-v, tw, P[i * ldp + c]);
        if (c == jj) P[i * ldp + c] = v;
      }
    }
    __syncwarp();
  }
  __syncthreads();
}

// ---------------------------------------------- fast path (M <= kHhFastRows)
constexpr int kHhFastRows = 608;  // V (M x 33) + C chunk (M x 8) + statics < 227 KB
constexpr int kHhFastChunk = 8;

RGSV_DI void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
RGSV_DI void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// dgeqr2 of the panel at (j0, j0) (mp x jb, jb <= 32) held in REGISTERS:
// lane c = column c, warp w = rows w + 16 r (r < RPW; rows >= mp are zero
// padding, which the updates keep at zero). Per column jj: lane jj publishes
// its column slice to a per-warp shared slot (one LDS broadcast per row
// instead of two shuffles), one fused reduction + one CTA barrier (see
// panel_qr), then the rank-1 update. Rows >= 32 are always below the
// diagonal, so only r < 2 needs predicates. S[c][jj] = V[:, c]^T v_jj (c <
// jj) is kept for the deferred dlarft.
constexpr int kHhMaxRpw = 38;
constexpr int kHhPanelSmem = (2 * 17 * 32 + 16 * kHhMaxRpw + 2 * 32 * 33) * 8;

template <int RPW>
__device__ void panel_qr_reg(double* a, int64_t lda, int j0, int mp, int jb, double* red,
                             double* colb, double* Ssm, double* tau_s, long long* prof) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane;
  double* cb = colb + warp * RPW;
  double x[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int i = warp + 16 * r;
    x[r] = (i < mp && c < jb) ? a[(int64_t)(j0 + i) * lda + j0 + c] : 0.0;
  }
  if (prof && tid == 0) prof[0] = gtimer();
  for (int jj = 0; jj < jb; ++jj) {
    if (prof && tid == 0) prof[1 + jj] = gtimer();
    if (lane == jj) {
#pragma unroll
      for (int r = 0; r < RPW; ++r) cb[r] = x[r];
    }
    __syncwarp();
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const double xj = cb[r];
      if (r < 2) {
        if (warp + 16 * r > jj) d0 = fma(xj, x[r], d0);
      } else if (r & 1) {
        d1 = fma(xj, x[r], d1);
      } else {
        d0 = fma(xj, x[r], d0);
      }
    }
    double* rb = red + (jj & 1) * 17 * 32;
    rb[warp * 32 + lane] = d0 + d1;
    if (warp == (jj & 15)) rb[16 * 32 + lane] = (jj >> 4) ? x[RPW > 1 ? 1 : 0] : x[0];
    __syncthreads();
    double pw[16];  // fixed-order pairwise tree over the 16 warp partials
#pragma unroll
    for (int w = 0; w < 16; ++w) pw[w] = rb[w * 32 + lane];
#pragma unroll
    for (int h = 8; h > 0; h >>= 1)
#pragma unroll
      for (int w = 0; w < h; ++w) pw[w] += pw[w + h];
    const double wp = pw[0];
    const double ss = __shfl_sync(0xffffffffu, wp, jj);
    const double alpha = rb[16 * 32 + jj];
    const double rowjj = rb[16 * 32 + lane];
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
    const double wc = fma(sc, wp, rowjj);
    if (warp == 0) {
      if (lane < jj) Ssm[lane * 33 + jj] = wc;
      if (lane == 0) tau_s[jj] = tj;
    }
    const double tw = (c > jj) ? tj * wc : 0.0;
    const bool own = (c == jj);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const double v = cb[r] * sc;
      if (r < 2) {
        const int i = warp + 16 * r;
        if (i == jj) {
          x[r] = own ? beta : x[r] - tw;
        } else if (i > jj) {
          const double nx = fma(-v, tw, x[r]);
          x[r] = own ? v : nx;
        }
      } else {
        const double nx = fma(-v, tw, x[r]);
        x[r] = own ? v : nx;
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int i = warp + 16 * r;
    if (i < mp && c < jb) a[(int64_t)(j0 + i) * lda + j0 + c] = x[r];
  }
  if (prof && tid == 0) prof[33] = gtimer();
  __syncthreads();
}

// dlarft (forward, columnwise) by recursive doubling over the whole CTA:
// T starts as diag(tau); merging adjacent blocks a, b of size bs gives
// T_ab = -T_a S_ab T_b. Ssm holds S = V^T V above the diagonal (zero
// elsewhere); X is 32 x 33 scratch. T (ld 33) must be zero off the diagonal.
__device__ void form_t(const double* Ssm, const double* tau_s, double* T, double* X) {
  const int tid = threadIdx.x;
  if (tid < 32) T[tid * 33 + tid] = tau_s[tid];
  __syncthreads();
  for (int bs = 1; bs < 32; bs *= 2) {
    const int per = bs * bs, total = 16 * bs;  // (32 / 2bs) merges x bs^2 entries
    for (int e = tid; e < total; e += kHhThreads) {  // X = S_ab T_b
      const int g = e / per, rr = (e % per) / bs, cc = e % bs, s0 = g * 2 * bs;
      double acc = 0.0;
      for (int l = 0; l <= cc; ++l)
        acc = fma(Ssm[(s0 + rr) * 33 + s0 + bs + l], T[(s0 + bs + l) * 33 + s0 + bs + cc], acc);
      X[(s0 + rr) * 33 + s0 + bs + cc] = acc;
    }
    __syncthreads();
    for (int e = tid; e < total; e += kHhThreads) {  // T_ab = -T_a X
      const int g = e / per, rr = (e % per) / bs, cc = e % bs, s0 = g * 2 * bs;
      double acc = 0.0;
      for (int l = rr; l < bs; ++l)
        acc = fma(T[(s0 + rr) * 33 + s0 + l], X[(s0 + l) * 33 + s0 + bs + cc], acc);
      T[(s0 + rr) * 33 + s0 + bs + cc] = -acc;
    }
    __syncthreads();
  }
}

// C[j0:j0+mp, c0:c0+cw] -= V Tm V^T C (Tm = T^T if trans else T) with V
// already staged in Vs (mp x 32, ld 33) and the chunk (cw <= 8 columns)
// staged by cp.async into Cs (mp x 8).
__device__ void apply_wy_fast(const double* Vs, int mp, int jb, const double* T, int trans,
                              double* c, int64_t ldc, int j0, int c0, int cw, double* Cs,
                              double* Wp, double* W2) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < mp * kHhFastChunk; e += kHhThreads) {
    const int i = e >> 3, y = e & 7;
    if (y < cw) cp_async8(Cs + e, c + (int64_t)(j0 + i) * ldc + c0 + y);
  }
  cp_async_wait_all();
  __syncthreads();
  {  // W[x][y] = sum_i V[i][x] C[i][y]; two row halves, fixed-order sum
    const int x = lane, y = warp & 7, half = warp >> 3;
    double a0 = 0.0, a1 = 0.0;
    if (y < cw) {
      int i = half;
      for (; i + 2 < mp; i += 4) {
        a0 = fma(Vs[i * 33 + x], Cs[i * 8 + y], a0);
        a1 = fma(Vs[(i + 2) * 33 + x], Cs[(i + 2) * 8 + y], a1);
      }
      for (; i < mp; i += 2) a0 = fma(Vs[i * 33 + x], Cs[i * 8 + y], a0);
    }
    Wp[half * 256 + x * 8 + y] = a0 + a1;
  }
  __syncthreads();
  if (tid < 256) {
    const int x = tid >> 3, y = tid & 7;
    double acc = 0.0;
    if (x < jb && y < cw) {
      if (trans) {
        for (int z = 0; z <= x; ++z)
          acc = fma(T[z * 33 + x], Wp[z * 8 + y] + Wp[256 + z * 8 + y], acc);
      } else {
        for (int z = x; z < jb; ++z)
          acc = fma(T[x * 33 + z], Wp[z * 8 + y] + Wp[256 + z * 8 + y], acc);
      }
    }
    W2[x * 8 + y] = acc;
  }
  __syncthreads();
  for (int e = tid; e < mp * kHhFastChunk; e += kHhThreads) {
    const int i = e >> 3, y = e & 7;
    if (y < cw) {
      const int xe = i < jb - 1 ? i : jb - 1;
      double acc = 0.0;
      for (int x = 0; x <= xe; ++x) acc = fma(Vs[i * 33 + x], W2[x * 8 + y], acc);
      c[(int64_t)(j0 + i) * ldc + c0 + y] = Cs[e] - acc;
    }
  }
  __syncthreads();
}

__device__ void stage_v_async(const double* a, int64_t lda, int j0, int mp, int jb, double* Vs) {
  for (int e = threadIdx.x; e < mp * 32; e += kHhThreads) {
    const int i = e >> 5, x = e & 31;
    if (x < jb) cp_async8(Vs + i * 33 + x, a + (int64_t)(j0 + i) * lda + j0 + x);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += kHhThreads) {
    const int i = e >> 5, x = e & 31;
    if (i < mp && (i <= x || x >= jb)) Vs[i * 33 + x] = (i == x && x < jb) ? 1.0 : 0.0;
  }
  __syncthreads();
}

template <int RPW>
__global__ void __launch_bounds__(kHhThreads) k_hhqr_fast(HhArgs h) {
  extern __shared__ double dsm[];
  const int tid = threadIdx.x;
  const int M = h.m1 + h.m2, N = h.N, K = M < N ? M : N, nb = 32;
  const unsigned G = gridDim.x;
  unsigned epoch = 0;
  const int cta = blockIdx.x;
  __shared__ double T[32 * 33];
  __shared__ double Wp[2 * 256], W2[256];
  __shared__ double tau_s[32];
  double* Vs = dsm;                 // M x 33
  double* Cs = dsm + (size_t)M * 33;  // M x 8
  double* red = dsm;                  // panel: 2 x 17 x 32 (aliases Vs)
  double* colb = red + 2 * 17 * 32;   // panel: 16 x RPW
  double* Ssm = colb + 16 * kHhMaxRpw;  // panel: 32 x 33
  double* Xt = Ssm + 32 * 33;           // dlarft scratch: 32 x 33
  int ps = 0;
#define HH_STAMP()                                                         \
  do {                                                                     \
    if (h.prof && cta == 0 && tid == 0 && ps < 255) h.prof[ps] = gtimer(); \
    ++ps;                                                                  \
  } while (0)
  {
    const int64_t tot = (int64_t)M * N;
    for (int64_t e = (int64_t)cta * kHhThreads + tid; e < tot; e += (int64_t)G * kHhThreads) {
      const int i = (int)(e / N), j = (int)(e % N);
      h.a[(int64_t)i * h.lda + j] =
          i < h.m1 ? h.b1[(int64_t)i * h.ld1 + j] : h.b2[(int64_t)(i - h.m1) * h.ld2 + j];
    }
    const int64_t totq = (int64_t)M * K;
    for (int64_t e = (int64_t)cta * kHhThreads + tid; e < totq; e += (int64_t)G * kHhThreads) {
      const int i = (int)(e / K), j = (int)(e % K);
      h.q[(int64_t)i * h.ldq + j] = (i == j) ? 1.0 : 0.0;
    }
  }
  HH_STAMP();
  grid_barrier(h.bar, G, epoch);
  const int npan = (K + nb - 1) / nb;
  for (int p = 0; p < npan; ++p) {
    const int j0 = p * nb, jb = (K - j0) < nb ? (K - j0) : nb, mp = M - j0;
    HH_STAMP();
    if (cta == 0) {
      long long* pp = (h.prof && p == 0) ? h.prof + 128 : nullptr;
      if (pp && tid == 0) pp[40] = gtimer();
      for (int x = tid; x < 32 * 33; x += kHhThreads) {
        Ssm[x] = 0.0;
        T[x] = 0.0;
      }
      if (tid < 32) tau_s[tid] = 0.0;
      __syncthreads();
      panel_qr_reg<RPW>(h.a, h.lda, j0, mp, jb, red, colb, Ssm, tau_s, pp);
      form_t(Ssm, tau_s, T, Xt);
      if (pp && tid == 0) pp[34] = gtimer();
      for (int x = tid; x < 32 * 33; x += kHhThreads) h.tb[(int64_t)p * 32 * 33 + x] = T[x];
    }
    HH_STAMP();
    grid_barrier(h.bar, G, epoch);
    HH_STAMP();
    const int c_lo = j0 + jb, ncol = N - c_lo;
    if (ncol > 0) {
      const int nch = (ncol + kHhFastChunk - 1) / kHhFastChunk;
      if (cta < nch) {
        for (int x = tid; x < 32 * 33; x += kHhThreads) T[x] = h.tb[(int64_t)p * 32 * 33 + x];
        stage_v_async(h.a, h.lda, j0, mp, jb, Vs);
        for (int ch = cta; ch < nch; ch += G) {
          const int c0 = c_lo + ch * kHhFastChunk;
          const int cw = (N - c0) < kHhFastChunk ? (N - c0) : kHhFastChunk;
          apply_wy_fast(Vs, mp, jb, T, 1, h.a, h.lda, j0, c0, cw, Cs, Wp, W2);
        }
      }
      HH_STAMP();
      grid_barrier(h.bar, G, epoch);
    }
  }
  HH_STAMP();
  for (int p = npan - 1; p >= 0; --p) {
    const int j0 = p * nb, jb = (K - j0) < nb ? (K - j0) : nb, mp = M - j0;
    const int nch = (K - j0 + kHhFastChunk - 1) / kHhFastChunk;
    if (cta < nch) {
      for (int x = tid; x < 32 * 33; x += kHhThreads) T[x] = h.tb[(int64_t)p * 32 * 33 + x];
      stage_v_async(h.a, h.lda, j0, mp, jb, Vs);
      for (int ch = cta; ch < nch; ch += G) {
        const int c0 = j0 + ch * kHhFastChunk;
        const int cw = (K - c0) < kHhFastChunk ? (K - c0) : kHhFastChunk;
        apply_wy_fast(Vs, mp, jb, T, 0, h.q, h.ldq, j0, c0, cw, Cs, Wp, W2);
      }
    }
    HH_STAMP();
    if (p > 0) grid_barrier(h.bar, G, epoch);
  }
  HH_STAMP();
  if (h.phase_fix) {  // flip the Q columns this CTA finished in the last pass
    const int nch = (K + kHhFastChunk - 1) / kHhFastChunk;
    for (int ch = cta; ch < nch; ch += G) {
      for (int e = tid; e < M * kHhFastChunk; e += kHhThreads) {
        const int i = e / kHhFastChunk, j = ch * kHhFastChunk + e % kHhFastChunk;
        if (j < K && h.a[(int64_t)j * h.lda + j] < 0.0)
          h.q[(int64_t)i * h.ldq + j] = -h.q[(int64_t)i * h.ldq + j];
      }
    }
  }
  if (h.r) {
    const int64_t totr = (int64_t)K * N;
    for (int64_t e = (int64_t)cta * kHhThreads + tid; e < totr; e += (int64_t)G * kHhThreads) {
      const int i = (int)(e / N), j = (int)(e % N);
      const double sgn = (h.phase_fix && h.a[(int64_t)i * h.lda + i] < 0.0) ? -1.0 : 1.0;
      h.r[(int64_t)i * h.ldr + j] = j >= i ? sgn * h.a[(int64_t)i * h.lda + j] : 0.0;
    }
  }
  HH_STAMP();
  if (h.prof && cta == 0 && tid == 0) h.prof[255] = ps;
#undef HH_STAMP
}

__global__ void __launch_bounds__(kHhThreads) k_hhqr(HhArgs h) {
  extern __shared__ double dsm[];
  const int tid = threadIdx.x;
  const int M = h.m1 + h.m2, N = h.N, K = M < N ? M : N, nb = h.nb, ldv = nb + 1;
  const unsigned G = gridDim.x;
  unsigned epoch = 0;
  const int cta = blockIdx.x;
  __shared__ double T[32 * 33];
  __shared__ double W[32 * 17], W2[32 * 17];
  __shared__ double red[2 * 17 * 32];
  __shared__ double tau_s[32];

  // stage A = [b1; b2] and Q = [I; 0]
  {
    const int64_t tot = (int64_t)M * N;
    for (int64_t e = (int64_t)cta * kHhThreads + tid; e < tot; e += (int64_t)G * kHhThreads) {
      const int i = (int)(e / N), j = (int)(e % N);
      h.a[(int64_t)i * h.lda + j] =
          i < h.m1 ? h.b1[(int64_t)i * h.ld1 + j] : h.b2[(int64_t)(i - h.m1) * h.ld2 + j];
    }
    const int64_t totq = (int64_t)M * K;
    for (int64_t e = (int64_t)cta * kHhThreads + tid; e < totq; e += (int64_t)G * kHhThreads) {
      const int i = (int)(e / K), j = (int)(e % K);
      h.q[(int64_t)i * h.ldq + j] = (i == j) ? 1.0 : 0.0;
    }
  }
  int ps = 0;
#define HH_STAMP()                                                   \
  do {                                                               \
    if (h.prof && cta == 0 && tid == 0 && ps < 255) h.prof[ps] = gtimer(); \
    ++ps;                                                            \
  } while (0)
  HH_STAMP();
  grid_barrier(h.bar, G, epoch);

  const int npan = (K + nb - 1) / nb;
  for (int p = 0; p < npan; ++p) {
    const int j0 = p * nb, jb = (K - j0) < nb ? (K - j0) : nb, mp = M - j0;
    HH_STAMP();
    if (cta == 0) {
      double* P = dsm;
      for (int e = tid; e < mp * jb; e += kHhThreads) {
        const int i = e / jb, c = e % jb;
        P[i * ldv + c] = h.a[(int64_t)(j0 + i) * h.lda + j0 + c];
      }
      for (int x = tid; x < 32 * 33; x += kHhThreads) T[x] = 0.0;
      __syncthreads();
      panel_qr(P, ldv, mp, jb, T, red, tau_s);
      for (int x = tid; x < 32 * 33; x += kHhThreads) h.tb[(int64_t)p * 32 * 33 + x] = T[x];
      for (int e = tid; e < mp * jb; e += kHhThreads) {
        const int i = e / jb, c = e % jb;
        h.a[(int64_t)(j0 + i) * h.lda + j0 + c] = P[i * ldv + c];
      }
    }
    HH_STAMP();
    grid_barrier(h.bar, G, epoch);
    HH_STAMP();
    // ---- trailing update of columns [j0 + jb, N) with H^T = I - V T^T V^T
    const int c_lo = j0 + jb, ncol = N - c_lo;
    if (ncol > 0) {
      const int nch = (ncol + kHhChunk - 1) / kHhChunk;
      if (cta < nch) {
        for (int x = tid; x < 32 * 33; x += kHhThreads) T[x] = h.tb[(int64_t)p * 32 * 33 + x];
        stage_v(h.a, h.lda, j0, mp, jb, ldv, dsm);
        for (int ch = cta; ch < nch; ch += G) {
          const int c0 = c_lo + ch * kHhChunk;
          const int cw = (N - c0) < kHhChunk ? (N - c0) : kHhChunk;
          apply_wy(dsm, ldv, mp, jb, T, 1, h.a, h.lda, j0, c0, cw, W, W2);
        }
      }
      HH_STAMP();
      grid_barrier(h.bar, G, epoch);
    }
  }
  HH_STAMP();
  // ---- Q = H_0 .. H_{K-1} [I; 0]: backward over the panels (dorgqr)
  for (int p = npan - 1; p >= 0; --p) {
    const int j0 = p * nb, jb = (K - j0) < nb ? (K - j0) : nb, mp = M - j0;
    const int nch = (K - j0 + kHhChunk - 1) / kHhChunk;
    if (cta < nch) {
      for (int x = tid; x < 32 * 33; x += kHhThreads) T[x] = h.tb[(int64_t)p * 32 * 33 + x];
      stage_v(h.a, h.lda, j0, mp, jb, ldv, dsm);
      for (int ch = cta; ch < nch; ch += G) {
        const int c0 = j0 + ch * kHhChunk, cw = (K - c0) < kHhChunk ? (K - c0) : kHhChunk;
        apply_wy(dsm, ldv, mp, jb, T, 0, h.q, h.ldq, j0, c0, cw, W, W2);
      }
    }
    HH_STAMP();
    if (p > 0) grid_barrier(h.bar, G, epoch);
  }
  HH_STAMP();
  // ---- R (upper trapezoid) and the phase fix diag(R) >= 0 (core.py:88-95).
  // Only the Q columns this CTA wrote in the last pass are flipped by it, so
  // no further barrier is needed.
  if (h.phase_fix) {
    const int nch = (K + kHhChunk - 1) / kHhChunk;
    for (int ch = cta; ch < nch; ch += G) {
      for (int e = tid; e < M * kHhChunk; e += kHhThreads) {
        const int i = e / kHhChunk, j = ch * kHhChunk + e % kHhChunk;
        if (j < K && h.a[(int64_t)j * h.lda + j] < 0.0)
          h.q[(int64_t)i * h.ldq + j] = -h.q[(int64_t)i * h.ldq + j];
      }
    }
  }
  if (h.r) {
    const int64_t totr = (int64_t)K * N;
    for (int64_t e = (int64_t)cta * kHhThreads + tid; e < totr; e += (int64_t)G * kHhThreads) {
      const int i = (int)(e / N), j = (int)(e % N);
      const double sgn = (h.phase_fix && h.a[(int64_t)i * h.lda + i] < 0.0) ? -1.0 : 1.0;
      h.r[(int64_t)i * h.ldr + j] = j >= i ? sgn * h.a[(int64_t)i * h.lda + j] : 0.0;
    }
  }
  HH_STAMP();
  if (h.prof && cta == 0 && tid == 0) h.prof[255] = ps;
#undef HH_STAMP
}

static int hh_nb(int M) { return M <= 640 ? 32 : 16; }

size_t hhqr_workspace_bytes(int M, int N) {
  const int K = M < N ? M : N;
  const int nb = hh_nb(M);
  const size_t npan = (size_t)((K + nb - 1) / nb);
  const size_t lda = (size_t)(N + (N & 1));
  return (size_t)M * lda * 8 + npan * 32 * 33 * 8 + 1024;
}

// Grid-barrier kernels launch cooperatively: all CTAs co-resident, so the
// global-memory barrier cannot wait on a CTA that is not scheduled.
static int coop_launch(const void* fn, int grid, int threads, size_t smem, void** args,
                       cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) return RGSV_ERR_CUDA;
  note_launch();
  return 0;
}

// Householder QR of [b1 (m1 rows); b2 (m2 rows)] (M x N, M <= kHhMaxRows):
// Q (M x K) and optionally R (K x N), K = min(M, N).
int hhqr(const double* b1, int64_t ld1, int m1, const double* b2, int64_t ld2, int m2, int N,
         double* q, int64_t ldq, double* r, int64_t ldr, int phase_fix, void* ws, size_t ws_bytes,
         cudaStream_t st, long long* prof) {
  const int M = m1 + m2;
  if (M < 1 || N < 1 || M > kHhMaxRows) return RGSV_ERR_DIMENSION;
  if (ws_bytes < hhqr_workspace_bytes(M, N)) return RGSV_ERR_WORKSPACE;
  const int K = M < N ? M : N;
  HhArgs h;
  h.b1 = b1;
  h.ld1 = ld1;
  h.m1 = m1;
  h.b2 = b2 ? b2 : b1;
  h.ld2 = ld2;
  h.m2 = m2;
  h.N = N;
  h.nb = hh_nb(M);
  const size_t npan = (size_t)((K + h.nb - 1) / h.nb);
  char* w = static_cast<char*>(ws);
  h.a = reinterpret_cast<double*>(w);
  h.lda = N + (N & 1);  // even pitch: 16-byte aligned rows
  h.tb = h.a + (size_t)M * h.lda;
  h.bar = reinterpret_cast<unsigned*>(h.tb + npan * 32 * 33);
  h.q = q;
  h.ldq = ldq;
  h.r = r;
  h.ldr = ldr;
  h.phase_fix = phase_fix;
  h.prof = prof;
  if (cudaMemsetAsync(h.bar, 0, 64, st) != cudaSuccess) return RGSV_ERR_CUDA;
  void* args[] = {&h};
  if (M <= kHhFastRows) {
    // register panel (rows per warp RPW >= ceil(M / 16)), cp.async-staged WY
    const void* fn;
    const int rpw = (M + 15) / 16;
    if (rpw <= 8) fn = reinterpret_cast<const void*>(k_hhqr_fast<8>);
    else if (rpw <= 16) fn = reinterpret_cast<const void*>(k_hhqr_fast<16>);
    else if (rpw <= 24) fn = reinterpret_cast<const void*>(k_hhqr_fast<24>);
    else fn = reinterpret_cast<const void*>(k_hhqr_fast<kHhMaxRpw>);
    const size_t smem = (size_t)M * (33 + kHhFastChunk) * 8;
    static bool attr_f = false;
    if (!attr_f) {
      const void* fns[4] = {reinterpret_cast<const void*>(k_hhqr_fast<8>),
                            reinterpret_cast<const void*>(k_hhqr_fast<16>),
                            reinterpret_cast<const void*>(k_hhqr_fast<24>),
                            reinterpret_cast<const void*>(k_hhqr_fast<kHhMaxRpw>)};
      for (const void* f : fns)
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kHhFastRows * (33 + kHhFastChunk) * 8) != cudaSuccess)
          return RGSV_ERR_CUDA;
      attr_f = true;
    }
    int grid = (N + kHhFastChunk - 1) / kHhFastChunk;
    if (grid > kSMs) grid = kSMs;
    if (grid < 1) grid = 1;
    return coop_launch(fn, grid, kHhThreads, smem > (size_t)kHhPanelSmem ? smem : kHhPanelSmem,
                       args, st);
  }
  const size_t smem = (size_t)M * (h.nb + 1) * 8;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_hhqr, cudaFuncAttributeMaxDynamicSharedMemorySize, 196 * 1024) !=
        cudaSuccess)
      return RGSV_ERR_CUDA;
    attr = true;
  }
  // one CTA per 16 trailing columns, up to one per SM (cooperative: co-resident)
  int grid = (N + kHhChunk - 1) / kHhChunk;
  if (grid > kSMs) grid = kSMs;
  if (grid < 1) grid = 1;
  return coop_launch(reinterpret_cast<const void*>(k_hhqr), grid, kHhThreads, smem, args, st);
}

// ================================================================ Jacobi
constexpr int kBJ = 16;       // rows per block
constexpr int kBP = 2 * kBJ;  // rows per block pair
// One inner sweep per block-pair visit (more inner sweeps re-rotate pairs the
// next outer round revisits anyway): 1000 x 1000 Gaussian 104 -> 55 ms, the
// reference-default adaptive mode at cfg0 23.4 -> 11.4 ms per pair
// (RGSV_BJ_INNER overrides; profiles/r02_bjacobi_inner_sweeps.log).
constexpr int kInnerSweeps = 1;

struct BJacJob {
  double* v;  // nv x len (rows are the vectors), rotated in place
  int64_t ld;
  int nv;
  int len;
  double* sv_out;  // min(nv, len) values, descending
  int* nsv_out;
  unsigned* bar;  // zeroed barrier counter
  int* flags;     // zeroed, max_sweeps entries: a rotation happened in sweep s
  int cta0;       // first CTA of this job
  int ctas;       // CTAs of this job
  int cluster;    // 1: the job is one thread-block cluster (hardware barrier)
  double* acc;    // optional nv x nv accumulated rotations (starts at I), ld ldacc
  int64_t ldacc;
  unsigned long long* gmax;  // zeroed: bits of the largest squared row norm at entry
};

RGSV_DI int rr_player(int p, int round, int nplayers) {
  return p == 0 ? 0 : 1 + ((p - 1 + round) % (nplayers - 1));
}

// smem: part (8 warps x 10 tiles x 64) | G (32 x 33) | R (32 x 33)
constexpr int kBjPart = 8 * 10 * 64;
constexpr size_t kBjSmem = (size_t)(kBjPart + 2 * 32 * 33) * 8;

// Process the block pair (ba, bb): returns 1 if it rotated.
// floor2: rows whose squared norm is at or below it count as zero rows (they
// are neither rotated nor held against convergence). A rank-deficient input
// leaves rows of pure rounding noise (~eps |A|), re-injected by every block
// rotation they share with a large row, which can never become orthogonal
// relative to their own size.
__device__ int bj_pair(const BJacJob& J, int ba, int bb, double tol, double* sm, int* s_flag,
                       int inner_sweeps, double floor2) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* part = sm;
  double* Gm = sm + kBjPart;
  double* R = Gm + 32 * 33;
  const int g = lane >> 2, t = lane & 3;
  // ---- Gram of the 32 rows by DMMA (10 upper tiles of 8 x 8)
  const double* rp[4];
  bool rv[4];
#pragma unroll
  for (int rg = 0; rg < 4; ++rg) {
    const int lr = rg * 8 + g;
    const int gr = lr < kBJ ? ba * kBJ + lr : bb * kBJ + (lr - kBJ);
    rv[rg] = gr < J.nv;
    rp[rg] = J.v + (int64_t)(rv[rg] ? gr : 0) * J.ld;
  }
  double acc[10][2];
#pragma unroll
  for (int x = 0; x < 10; ++x) acc[x][0] = acc[x][1] = 0.0;
#pragma unroll 2
  for (int k0 = warp * 4; k0 < J.len; k0 += 32) {
    const int kk = k0 + t;
    double xv[4];
#pragma unroll
    for (int rg = 0; rg < 4; ++rg) xv[rg] = (rv[rg] && kk < J.len) ? rp[rg][kk] : 0.0;
    int ti = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = i; j < 4; ++j) dmma(acc[ti++], xv[i], xv[j]);
  }
#pragma unroll
  for (int x = 0; x < 10; ++x) {
    part[(warp * 10 + x) * 64 + lane * 2] = acc[x][0];
    part[(warp * 10 + x) * 64 + lane * 2 + 1] = acc[x][1];
  }
  if (tid == 0) *s_flag = 0;
  __syncthreads();
  for (int e = tid; e < 640; e += kDenseThreads) {
    const int x = e >> 6, f = e & 63, ln = f >> 1, half = f & 1;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += part[(w * 10 + x) * 64 + f];
    // tile x -> (i, j), i <= j
    int i = 0, j = x;
    if (x >= 4) { i = 1; j = x - 3; }
    if (x >= 7) { i = 2; j = x - 5; }
    if (x >= 9) { i = 3; j = 3; }
    const int row = i * 8 + (ln >> 2), col = j * 8 + 2 * (ln & 3) + half;
    Gm[row * 33 + col] = s;
    Gm[col * 33 + row] = s;
  }
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += kDenseThreads) {
    const int i = e >> 5, j = e & 31;
    if (i < j) {
      const double d = Gm[i * 33 + j];
      const double gi = Gm[i * 33 + i], gj = Gm[j * 33 + j];
      if (d != 0.0 && fmin(gi, gj) > floor2 && fabs(d) > tol * sqrt(gi * gj)) *s_flag = 1;
    }
    R[i * 33 + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (!*s_flag) return 0;
  // ---- cyclic two-sided Jacobi on the Gram, rotations accumulated in R
  const int pr = tid >> 4, sub = tid & 15;
  for (int isw = 0; isw < inner_sweeps; ++isw) {
    __syncthreads();
    if (tid == 0) *s_flag = 0;
    __syncthreads();
    for (int round = 0; round < 31; ++round) {
      const int a = rr_player(pr, round, 32), b = rr_player(31 - pr, round, 32);
      const double al = Gm[a * 33 + a], be = Gm[b * 33 + b], ga = Gm[a * 33 + b];
      // |ga| > tol sqrt(al be), squared (al, be >= 0): no sqrt on the chain
      const bool rot = ga != 0.0 && fmin(al, be) > floor2 && ga * ga > (tol * tol) * (al * be);
      double c = 1.0, s = 0.0, tt = 0.0;
      if (rot) {
        const double zeta = (be - al) / (2.0 * ga);
        tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        c = rsqrt(fma(tt, tt, 1.0));
        s = c * tt;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int col = sub + 16 * h2;
          const double x = Gm[a * 33 + col], y = Gm[b * 33 + col];
          Gm[a * 33 + col] = c * x - s * y;
          Gm[b * 33 + col] = s * x + c * y;
          const double rx = R[a * 33 + col], ry = R[b * 33 + col];
          R[a * 33 + col] = c * rx - s * ry;
          R[b * 33 + col] = s * rx + c * ry;
        }
      }
      __syncthreads();
      if (rot) {
        // column update; the pair's own 2 x 2 block gets its exact values
        // here (no third barrier): diag al - t ga, be + t ga, off-diagonal 0
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int row = sub + 16 * h2;
          if (row == a) {
            Gm[a * 33 + a] = al - tt * ga;
            Gm[a * 33 + b] = 0.0;
          } else if (row == b) {
            Gm[b * 33 + a] = 0.0;
            Gm[b * 33 + b] = be + tt * ga;
          } else {
            const double x = Gm[row * 33 + a], y = Gm[row * 33 + b];
            Gm[row * 33 + a] = c * x - s * y;
            Gm[row * 33 + b] = s * x + c * y;
          }
        }
        if (sub == 0) *s_flag = 1;
      }
      __syncthreads();
    }
    if (!*s_flag) break;
  }
  // ---- polish R to orthogonal (one Newton-Schulz step R <- R - R E / 2,
  // E = R^T R - I) so repeated block rotations do not drift the row norms
  {
    double* E = part;
    double* Rn = part + 1024;
    for (int e = tid; e < 1024; e += kDenseThreads) {
      const int i = e >> 5, j = e & 31;
      double acc = (i == j) ? -1.0 : 0.0;
      for (int k = 0; k < kBP; ++k) acc = fma(R[k * 33 + i], R[k * 33 + j], acc);
      E[e] = acc;
    }
    __syncthreads();
    for (int e = tid; e < 1024; e += kDenseThreads) {
      const int i = e >> 5, j = e & 31;
      double acc = 0.0;
      for (int k = 0; k < kBP; ++k) acc = fma(R[i * 33 + k], E[k * 32 + j], acc);
      Rn[e] = fma(-0.5, acc, R[i * 33 + j]);
    }
    __syncthreads();
    for (int e = tid; e < 1024; e += kDenseThreads) R[(e >> 5) * 33 + (e & 31)] = Rn[e];
    __syncthreads();
  }
  // ---- rotate the pair's rows: Vp <- R Vp (and the same rows of the
  //      accumulated rotations when singular vectors are requested), on
  //      DMMA: R's fragments in registers, 8-column blocks of the 32 rows per
  //      warp iteration (loads of a block complete before its stores)
  {
    const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    double rf[4][8];  // A fragments: R[mt*8 + g][ks*4 + t]
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) rf[mt][ks] = R[(mt * 8 + g) * 33 + ks * 4 + t];
    const int nb_v = (J.len + 7) / 8;
    const int nb_all = J.acc ? nb_v + (J.nv + 7) / 8 : nb_v;
    for (int blk = warp; blk < nb_all; blk += kDenseThreads / 32) {
      const bool in_acc = blk >= nb_v;
      double* base = in_acc ? J.acc : J.v;
      const int64_t ld = in_acc ? J.ldacc : J.ld;
      const int ncol = in_acc ? J.nv : J.len;
      const int n0 = (in_acc ? blk - nb_v : blk) * 8;
      double bf[8];  // B fragments: Vp[ks*4 + t][n0 + g]
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int i = ks * 4 + t;
        const int gr = i < kBJ ? ba * kBJ + i : bb * kBJ + (i - kBJ);
        bf[ks] = (gr < J.nv && n0 + g < ncol) ? base[(int64_t)gr * ld + n0 + g] : 0.0;
      }
      double cacc[4][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) cacc[mt][0] = cacc[mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(cacc[mt], rf[mt][ks], bf[ks]);
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = mt * 8 + g;
        const int gr = i < kBJ ? ba * kBJ + i : bb * kBJ + (i - kBJ);
        if (gr >= J.nv) continue;
        const int col = n0 + 2 * t;
        if (col < ncol) base[(int64_t)gr * ld + col] = cacc[mt][0];
        if (col + 1 < ncol) base[(int64_t)gr * ld + col + 1] = cacc[mt][1];
      }
    }
  }
  __syncthreads();
  return 1;
}

__global__ void __launch_bounds__(kDenseThreads) k_bjacobi(BJacJob j0, BJacJob j1, int max_sweeps,
                                                           int* __restrict__ status,
                                                           int inner_sweeps) {
  extern __shared__ double dsm[];
  __shared__ int s_flag;
  const BJacJob J = (int)blockIdx.x < j0.cta0 + j0.ctas ? j0 : j1;
  const int cta = blockIdx.x - J.cta0;
  if (J.nv <= 0 || J.len <= 0) {
    if (cta == 0 && threadIdx.x == 0) *J.nsv_out = 0;
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double tol = fmax(1e-15, sqrt((double)J.len) * 2.220446049250313e-16);
  const int nblk = (J.nv + kBJ - 1) / kBJ;
  const int nbe = nblk + (nblk & 1);
  const int npairs = nbe / 2;
  unsigned epoch = 0;
  // zero-row floor: (1e-14)^2 of the largest squared row norm at entry (the
  // rows are shared out over the job's CTAs, one atomicMax per CTA on the
  // order-preserving bits of a nonnegative double, then one barrier: every
  // CTA reads the same value, so the result stays deterministic)
  {
    double mx = 0.0;
    for (int i = cta * 8 + warp; i < J.nv; i += J.ctas * 8) {
      const double* vi = J.v + (int64_t)i * J.ld;
      double sq = 0.0;
      for (int e = lane; e < J.len; e += 32) sq = fma(vi[e], vi[e], sq);
      sq = warp_sum(sq);
      mx = fmax(mx, sq);
    }
    if (lane == 0 && mx > 0.0)
      atomicMax(J.gmax, (unsigned long long)__double_as_longlong(mx));
    if (J.ctas > 1 && J.cluster) cluster_sync_all();
    else if (J.ctas > 1) grid_barrier(J.bar, J.ctas, epoch);
    else __syncthreads();
  }
  // (values-only jobs; with accumulated rotations the rows of zero singular
  //  values must still come out mutually orthogonal for the vector outputs)
  const double floor2 = J.acc ? 0.0 : 1e-28 * __longlong_as_double((long long)*reinterpret_cast<
                                                  volatile unsigned long long*>(J.gmax));
  if (J.acc) {  // accumulated rotations start at the identity
    for (int64_t e = (int64_t)cta * kDenseThreads + tid; e < (int64_t)J.nv * J.nv;
         e += (int64_t)J.ctas * kDenseThreads) {
      const int i = (int)(e / J.nv), j = (int)(e % J.nv);
      J.acc[(int64_t)i * J.ldacc + j] = (i == j) ? 1.0 : 0.0;
    }
    if (J.ctas > 1 && J.cluster) cluster_sync_all();
    else if (J.ctas > 1) grid_barrier(J.bar, J.ctas, epoch);
    else __syncthreads();
  }
  bool converged = nblk == 1 && J.nv == 1;
  int sweep = 0;
  for (; sweep < max_sweeps && !converged; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < nbe - 1; ++round) {
      for (int p = cta; p < npairs; p += J.ctas) {
        // (one block: nbe = 2 and its partner block is all padding)
        const int ba = rr_player(p, round, nbe), bb = rr_player(nbe - 1 - p, round, nbe);
        rotated |= bj_pair(J, ba, bb, tol, dsm, &s_flag, inner_sweeps, floor2);
      }
      if (J.ctas > 1) {
        if (J.cluster) cluster_sync_all();
        else grid_barrier(J.bar, J.ctas, epoch);
      }
    }
    if (rotated && tid == 0) atomicOr(J.flags + sweep, 1);
    if (J.ctas > 1 && J.cluster) cluster_sync_all();
    else if (J.ctas > 1) grid_barrier(J.bar, J.ctas, epoch);
    else __syncthreads();
    converged = ld_acquire_u32(reinterpret_cast<unsigned*>(J.flags + sweep)) == 0;
    __syncthreads();
  }
  if (cta != 0) return;
  if (!converged && tid == 0) atomicOr(status, RGSV_ST_JACOBI);
  // row norms (sequential-order fma per lane, then warp sum), ranked descending
  double* nrm = dsm;
  for (int i = warp; i < J.nv; i += 8) {
    const double* vi = J.v + (int64_t)i * J.ld;
    double s = 0.0;
    for (int e = lane; e < J.len; e += 32) s = fma(vi[e], vi[e], s);
    s = warp_sum(s);
    if (lane == 0) nrm[i] = sqrt(s);
  }
  __syncthreads();
  const int nout = J.nv < J.len ? J.nv : J.len;
  for (int i = tid; i < J.nv; i += kDenseThreads) {
    const double x = nrm[i];
    int rank = 0;
    for (int j = 0; j < J.nv; ++j) {
      const double y = nrm[j];
      rank += (y > x) || (y == x && j < i);
    }
    if (rank < nout) J.sv_out[rank] = x;
  }
  if (tid == 0) *J.nsv_out = nout;
}

constexpr int kBjMaxSweeps = 60;

size_t bjacobi_sync_bytes() { return 2 * (64 + kBjMaxSweeps * 4) + 256; }

// Singular values of the rows of two matrices (either may be empty) by
// blocked one-sided Jacobi; `sync` >= bjacobi_sync_bytes() of scratch.
int bjacobi_acc(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1, double* acc1,
                int64_t ldacc1, double* v2, int64_t ld2, int nv2, int len2, double* sv2,
                int* nsv2, int* status, void* sync, cudaStream_t st);

int bjacobi(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1, double* v2,
            int64_t ld2, int nv2, int len2, double* sv2, int* nsv2, int* status, void* sync,
            cudaStream_t st) {
  return bjacobi_acc(v1, ld1, nv1, len1, sv1, nsv1, nullptr, 0, v2, ld2, nv2, len2, sv2, nsv2,
                     status, sync, st);
}

int bjacobi_acc(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1, double* acc1,
                int64_t ldacc1, double* v2, int64_t ld2, int nv2, int len2, double* sv2,
                int* nsv2, int* status, void* sync, cudaStream_t st) {
  if (nv1 < 0 || nv2 < 0) return RGSV_ERR_DIMENSION;
  const size_t smem_n = (size_t)(nv1 > nv2 ? nv1 : nv2) * 8;
  if (smem_n > 200 * 1024) return RGSV_ERR_DIMENSION;  // nv <= 25600
  const size_t smem = smem_n > kBjSmem ? smem_n : kBjSmem;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_bjacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return RGSV_ERR_CUDA;
    attr = true;
  }
  char* s = static_cast<char*>(sync);
  if (cudaMemsetAsync(s, 0, bjacobi_sync_bytes(), st) != cudaSuccess) return RGSV_ERR_CUDA;
  auto pairs = [](int nv) {
    const int nblk = (nv + kBJ - 1) / kBJ;
    return (nblk + (nblk & 1)) / 2;
  };
  const int p1 = nv1 > 0 ? pairs(nv1) : 0, p2 = nv2 > 0 ? pairs(nv2) : 0;
  // an empty job still gets one CTA, which writes its count (0)
  int c1 = p1 > 0 ? p1 : 1, c2 = p2 > 0 ? p2 : (nsv2 ? 1 : 0);
  const int cap = c2 > 0 ? kSMs / 2 : kSMs;
  if (c1 > cap) c1 = cap;
  if (c2 > cap) c2 = cap;
  // small jobs: one thread-block cluster per job (gang-scheduled, hardware
  // cluster barrier), both jobs padded to the same CTA count; larger jobs: one
  // cooperative launch with global-memory barriers
  const int cmax = c1 > c2 ? c1 : c2;
  const bool clustered = cmax <= 8;
  if (clustered) {
    c1 = cmax;
    if (c2 > 0) c2 = cmax;
  }
  // per job: 64 bytes (barrier counter at 0, zero-row scale at 48) + sweep flags
  BJacJob a{v1, ld1, nv1, len1, sv1, nsv1, reinterpret_cast<unsigned*>(s),
            reinterpret_cast<int*>(s + 64), 0, c1, clustered ? 1 : 0, acc1, ldacc1,
            reinterpret_cast<unsigned long long*>(s + 48)};
  BJacJob b{v2, ld2, nv2, len2, sv2, nsv2, reinterpret_cast<unsigned*>(s + 64 + kBjMaxSweeps * 4),
            reinterpret_cast<int*>(s + 128 + kBjMaxSweeps * 4), c1, c2, clustered ? 1 : 0,
            nullptr, 0, reinterpret_cast<unsigned long long*>(s + 64 + kBjMaxSweeps * 4 + 48)};
  int ms = kBjMaxSweeps;
  static const int inner = [] {  // RGSV_BJ_INNER: inner Jacobi sweeps per block pair
    const char* e = getenv("RGSV_BJ_INNER");
    const int v = e ? atoi(e) : kInnerSweeps;
    return v >= 1 && v <= 16 ? v : kInnerSweeps;
  }();
  int isw = inner;
  void* args[] = {&a, &b, &ms, &status, &isw};
  if (!clustered)
    return coop_launch(reinterpret_cast<const void*>(k_bjacobi), c1 + c2, kDenseThreads, smem,
                       args, st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c1 + c2);
  cfg.blockDim = dim3(kDenseThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute cl[1];
  cl[0].id = cudaLaunchAttributeClusterDimension;
  cl[0].val.clusterDim.x = c1;
  cl[0].val.clusterDim.y = 1;
  cl[0].val.clusterDim.z = 1;
  cfg.attrs = cl;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k_bjacobi), args) != cudaSuccess)
    return RGSV_ERR_CUDA;
  note_launch();
  return 0;
}

// ---------------------------------------- singular vectors from the rotated rows
// After k_bjacobi with an accumulator: v rows = diag(s) X rows (orthogonal),
// acc = J (orthogonal), J A = v. Outputs ordered by singular value
// (descending, or ascending): sv, xn = unit rows of X (zero rows stay zero and
// are counted in *nzero), jo = the matching rows of J -- the contract of
// k_jacobi_vec (small.cu), on many CTAs.
__global__ void k_vec_norms(const double* __restrict__ v, int64_t ldv, int nv, int len,
                            double* __restrict__ nrm) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= nv) return;
  const double* vi = v + (int64_t)row * ldv;
  double s = 0.0;
  for (int e = lane; e < len; e += 32) s = fma(vi[e], vi[e], s);
  s = warp_sum(s);
  if (lane == 0) nrm[row] = sqrt(s);
}

__global__ void k_vec_rank(const double* __restrict__ nrm, int nv, int ascending,
                           int* __restrict__ ord, double* __restrict__ sv,
                           int* __restrict__ nzero) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double x = nrm[i];
  int rank = 0;
  for (int j = 0; j < nv; ++j) {
    const double y = nrm[j];
    rank += ascending ? ((y < x) || (y == x && j < i)) : ((y > x) || (y == x && j < i));
  }
  ord[rank] = i;
  sv[rank] = x;
  if (x == 0.0) atomicAdd(nzero, 1);
}

__global__ void k_vec_gather(const double* __restrict__ v, int64_t ldv, const double* __restrict__ acc,
                             int64_t ldacc, int nv, int len, const double* __restrict__ nrm,
                             const int* __restrict__ ord, double* __restrict__ xn, int64_t ldx,
                             double* __restrict__ jo, int64_t ldj) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nv) return;
  const int i = ord[r];
  const double x = nrm[i];
  const double inv = x > 0.0 ? 1.0 / x : 0.0;
  for (int e = lane; e < len; e += 32) xn[(int64_t)r * ldx + e] = v[(int64_t)i * ldv + e] * inv;
  for (int e = lane; e < nv; e += 32) jo[(int64_t)r * ldj + e] = acc[(int64_t)i * ldacc + e];
}

size_t svd_vectors_blocked_workspace_bytes(int nv) {
  return bjacobi_sync_bytes() + (size_t)nv * 16 + 512;
}

int svd_vectors_blocked(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                        double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj,
                        int ascending, int* nzero, int* status, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  if (nv < 1 || len < 1 || nv > len) return RGSV_ERR_DIMENSION;
  if (ws_bytes < svd_vectors_blocked_workspace_bytes(nv)) return RGSV_ERR_WORKSPACE;
  char* w = static_cast<char*>(ws);
  void* sync = w;
  double* nrm = reinterpret_cast<double*>(w + ((bjacobi_sync_bytes() + 255) & ~size_t(255)));
  int* ord = reinterpret_cast<int*>(nrm + nv);
  double* sv_tmp = sv;  // k_bjacobi's own descending values, overwritten below
  int* nsv_tmp = ord;   // scratch for its count (ord is written after)
  if (int e = bjacobi_acc(v, ldv, nv, len, sv_tmp, nsv_tmp, acc, ldacc, nullptr, 0, 0, len,
                          nullptr, nullptr, status, sync, st))
    return e;
  if (cudaMemsetAsync(nzero, 0, sizeof(int), st) != cudaSuccess) return RGSV_ERR_CUDA;
  const int wblocks = (nv * 32 + 255) / 256;
  k_vec_norms<<<wblocks, 256, 0, st>>>(v, ldv, nv, len, nrm);
  k_vec_rank<<<(nv + 255) / 256, 256, 0, st>>>(nrm, nv, ascending, ord, sv, nzero);
  k_vec_gather<<<wblocks, 256, 0, st>>>(v, ldv, acc, ldacc, nv, len, nrm, ord, xn, ldx, jo, ldj);
  note_launch(3);
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

}  // namespace rgsv
