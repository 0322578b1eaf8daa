// Batched fixed-rank rGSVD chains for many small pairs (SURVEY.md §8 cfg3:
// 4096 pairs of 4000/3000 x 64, k = 16, q = 1).
//
// One thread-block CLUSTER per matrix G (m x n): the cluster's CS CTAs split
// G's rows, and each CTA keeps its slice of the sketch Y / basis Q in SHARED
// MEMORY for the whole chain, so shifted CholeskyQR3 (Gram, Cholesky, TRSM)
// never touches HBM. G is streamed into FP64 DMMA (mma.sync.m8n8k4) four
// times per chain (sketch, G^T Q, G Q^, projection); with only ~148/CS
// matrices in flight the re-reads come from L2. For the cfg3 shape (n <= 64,
// k <= 16) G goes from global memory straight into DMMA fragments (16-byte
// no-allocate loads, two register buffers per warp, no CTA barrier inside a
// pass; Chain::pass_*_reg) and a 4000-row matrix runs on a 3-CTA cluster;
// the wider shapes stage 32-row tiles through a cp.async ring. The k x k Gram
// and n x k partial products are reduced across the
// cluster through distributed shared memory (mapa + ld.shared::cluster) in a
// fixed CTA order, so every CTA holds bit-identical small matrices and the
// result does not depend on scheduling. Per matrix the chain is the same
// algorithm as rgsv_sketch_project (rangefinder.py:115-123 + the q power
// iterations of SURVEY.md §8(c)): Y = G Omega; Q = cholqr3(Y); q times
// { Z = G^T Q; Qhat = cholqr3(Z); Y = G Qhat; Q = cholqr3(Y) }; B = Q^T G.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {
namespace {

// Opt-in phase timers (compile with -DRGSV_BATCH_PROFILE; tools/batch_phases):
// thread 0 of every CTA accumulates clock64 deltas per phase into
// g_batch_prof[phase]. Off in the product build.
#ifdef RGSV_BATCH_PROFILE
}  // namespace
__device__ unsigned long long g_batch_prof[24];
namespace {
#define PROF_T0() long long _pt = clock64()
#define PROF(ph)                                                                  \
  do {                                                                            \
    if (threadIdx.x == 0) {                                                       \
      long long _n = clock64();                                                   \
      atomicAdd(&g_batch_prof[ph], (unsigned long long)(_n - _pt));               \
      _pt = _n;                                                                   \
    }                                                                             \
  } while (0)
#else
#define PROF_T0()
#define PROF(ph)
#endif

constexpr int kTR = 32;       // G rows per streamed tile
constexpr int kStages = 3;    // cp.async ring depth (4 measured 79.6k vs 81.6k pairs/s at cfg3)
constexpr int kThreads = 256; // 8 warps
constexpr int kWarps = kThreads / 32;

RGSV_DI uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
RGSV_DI uint32_t cluster_idx() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
RGSV_DI uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
RGSV_DI void cluster_barrier() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::
          : "memory");
}
RGSV_DI double ld_dsmem(const double* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
  return v;
}
RGSV_DI int ld_dsmem_i32(const int* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(ra));
  return v;
}
RGSV_DI void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
RGSV_DI void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
RGSV_DI void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 16-byte / 8-byte read-only global loads that do not allocate in L1 (G is
// streamed: each byte is used once per pass).
RGSV_DI void ldg_stream2(double& x, double& y, const double* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "l"(p));
}
// ... with an L2 eviction-priority hint: a matrix is read by four passes ~40 us
// apart while 37 clusters stream ~74 MB of live data through the L2; the first
// three passes keep their lines (evict_last), the last one marks them dead
// (evict_first) so finished matrices do not push live ones out.
RGSV_DI void ldg_stream2(double& x, double& y, const double* p, uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(x), "=d"(y)
               : "l"(p), "l"(pol));
}
RGSV_DI uint64_t l2_policy(bool keep) {
  uint64_t pol;
#ifdef RGSV_BATCH_NOHINT  // A/B builds: every pass with the default priority
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
#endif
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
RGSV_DI double ldg_stream1(const double* p) {
  double x;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(x) : "l"(p));
  return x;
}

// Y / Z slice layout: row-major, pitch KP doubles, XOR swizzle inside each
// 16-column group so both DMMA fragment patterns used on it (A: 8 rows x 4
// cols; B: 4 rows x 8 cols) hit the minimum two shared-memory wavefronts.
template <int KP>
RGSV_DI int yx(int r, int c) {
  return r * KP + ((c & ~15) | ((c & 15) ^ (((r & 1) << 3) | (((r >> 1) & 1) << 2))));
}

struct ChainArgs {
  const BatchMat* mats;
  int nmat;
  int n;
  int k;
  int q;
  const double* omega;  // per matrix: KP x ldo (Omega^T), stride om_stride
  int64_t ldo;
  int64_t om_stride;
  double* b_out;        // per matrix: KP x ldb, stride b_stride
  int64_t ldb;
  int64_t b_stride;
  double* stats;        // per matrix: {||G||_F^2, ||B||_F^2}
  int* status;          // per matrix status bits
  int yrows;            // shared-memory rows of the Y slice (multiple of 32)
  int* next;            // work counter (zeroed before the launch), or nullptr: static round-robin
};

// G tiles: kTR x NP, unpadded, 16-byte chunk q of row r stored at
// q ^ ((r & 3) << 1) (stays inside its 128-byte segment): the A fragments of
// Y = G X (8 rows x 4 cols) and of G^T Q (4 rows x 8 cols) both hit the
// minimum two wavefronts.
template <int NP>
RGSV_DI int gx_idx(int r, int c) {
  return r * NP + ((((c >> 1) ^ ((r & 3) << 1))) << 1) + (c & 1);
}

template <int NP, int KP>
struct Layout {
  // NP = 64, KP = 16 (the cfg3 shape) streams G through registers (Chain's
  // pass_*_reg): no ring, so the region only holds zb + wred, the two fold
  // slots of pass_gtq_reg and the folded Z / B partial the cluster reduces
  // from; the reduction slots then only carry a Gram. The smaller footprint
  // lets a 4000-row matrix run on a 3-CTA cluster.
  static constexpr bool kRegStream = (NP == 64 && KP == 16);
  static constexpr int SP = KP + 4;                 // fold-slot pitch (conflict-free 16 B stores)
  static constexpr int kFold = 2 * NP * SP;         // two fold slots (alias zb + wred)
  static constexpr int GP = NP + 4;                 // X^T pitch (doubles)
  static constexpr int kG = kRegStream ? kFold + NP * KP
                                       : kStages * kTR * NP;  // G ring / scratch region
  static constexpr int kX = KP * GP;                // X^T (KP x NP)
  static constexpr int kPart = kRegStream ? KP * KP + 16 : NP * KP;  // one reduction slot
  static constexpr int kSmall = KP * (KP + 1);      // Gram / L / L^-1
  static_assert(NP * KP + kWarps * 3 * 64 <= (kRegStream ? kFold : kG),
                "zb + wred must fit the idle region");
  static size_t bytes(int yrows) {
    return sizeof(double) * ((size_t)yrows * KP + kG + kX + 2 * kPart + 3 * kSmall + 64);
  }
};

template <int NP, int KP, int CS>
struct Chain {
  using Lo = Layout<NP, KP>;
  static constexpr int GP = Lo::GP;
  double* ys;    // Y / Q slice (yrows x KP, swizzled)
  double* gst;   // G tile ring
  double* xt;    // X^T: KP x GP
  double* part;  // 2 reduction slots of NP*KP
  double* zb;    // reduced Z / B^T (NP x KP), in the idle G ring
  double* gram;  // KP x (KP+1)
  double* lmat;  // KP x (KP+1): Cholesky factor, in place
  double* linv;  // KP x (KP+1): L^-1 (row-major)
  double* wred;  // per-warp partials (kWarps x 64), in the idle G ring
  double* misc;  // scalars
  int slot;
  int fail;
  int tid, lane, warp;
  uint32_t crank;

  RGSV_DI void init(double* sm, int yrows) {
    ys = sm;
    gst = ys + (size_t)yrows * KP;
    xt = gst + Lo::kG;
    part = xt + Lo::kX;
    gram = part + 2 * Lo::kPart;
    lmat = gram + Lo::kSmall;
    linv = lmat + Lo::kSmall;
    misc = linv + Lo::kSmall;
    zb = gst;                  // G ring is idle whenever zb / wred are live
    wred = gst + NP * KP;
    slot = 0;
    tid = threadIdx.x;
    lane = tid & 31;
    warp = tid >> 5;
    crank = cluster_rank();
  }

  // ---- cluster reduction of `cnt` doubles from this CTA's part slot into dst
  // (every CTA gets the same fixed-order sum). Double-buffered slots make one
  // cluster barrier per reduction sufficient (see header comment).
  RGSV_DI double* slot_ptr() { return part + slot * Lo::kPart; }
  template <typename F>
  RGSV_DI void reduce(int cnt, F&& store) {
    double* src = slot_ptr();
    __syncthreads();
    cluster_barrier();
    for (int e = tid; e < cnt; e += kThreads) {
      double v[CS];
#pragma unroll
      for (int r = 0; r < CS; ++r) v[r] = ld_dsmem(src + e, r);  // all loads in flight
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < CS; ++r) s += v[r];  // fixed CTA order
      store(e, s);
    }
    slot ^= 1;
    __syncthreads();
  }

  // ---- the same from an explicit source that is rewritten only after later
  //      cluster barriers (the folded Z / B partial of pass_gtq_reg)
  template <typename F>
  RGSV_DI void reduce_from(const double* src, int cnt, F&& store) {
    __syncthreads();
    cluster_barrier();
    for (int e = tid; e < cnt; e += kThreads) {
      double v[CS];
#pragma unroll
      for (int r = 0; r < CS; ++r) v[r] = ld_dsmem(src + e, r);
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < CS; ++r) s += v[r];
      store(e, s);
    }
    __syncthreads();
  }
  // the n x k partial of this CTA's last pass_gtq
  RGSV_DI const double* gtq_partial() {
    if constexpr (kRegStream) return gst + Lo::kFold;
    else return slot_ptr();
  }
  template <typename F>
  RGSV_DI void reduce_gtq(F&& store) {
    if constexpr (kRegStream) reduce_from(gst + Lo::kFold, NP * KP, store);
    else reduce(NP * KP, store);
  }

  // ---- stream this CTA's G rows [r0, r1) through the ring, tile by tile
  RGSV_DI void issue_tile(const BatchMat& g, int r0, int r1, int t, int n) {
    double* dst = gst + (t % kStages) * kTR * NP;
    constexpr int kChunks = kTR * (NP / 2);
    for (int e = tid; e < kChunks; e += kThreads) {
      const int rr = e / (NP / 2), cc = (e % (NP / 2)) * 2;
      const int row = r0 + t * kTR + rr;
      int bytes = 0;
      if (row < r1 && cc < n) bytes = (cc + 1 < n) ? 16 : 8;
      const double* src = bytes ? g.g + (int64_t)row * g.ld + cc : g.g;
      cp_async16(dst + gx_idx<NP>(rr, cc), src, bytes);
    }
  }

  template <typename F>
  RGSV_DI void stream_g(const BatchMat& g, int r0, int r1, int n, F&& body) {
    const int rows = r1 - r0;
    const int T = rows > 0 ? (rows + kTR - 1) / kTR : 0;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < T) issue_tile(g, r0, r1, s, n);
      cp_commit();
    }
    for (int t = 0; t < T; ++t) {
      cp_wait<kStages - 2>();
      __syncthreads();
      if (t + kStages - 1 < T) issue_tile(g, r0, r1, t + kStages - 1, n);
      cp_commit();
      body(t, gst + (t % kStages) * kTR * NP);
    }
    cp_wait<0>();
    __syncthreads();
  }

  // ---- register-streamed passes (NP = 64, KP = 16: the cfg3 shape). G goes
  //      from global memory (L2 after the first pass) straight into DMMA
  //      fragments, with no shared-memory ring and no CTA barrier inside the
  //      pass: warp w owns the 8-row blocks w, w + 8, ... of the slice and
  //      double-buffers them (4 KB each) in registers (see pipeline()); the
  //      ring it replaces was latency bound at 14 B/clk/SM with a CTA barrier
  //      per 32-row tile.
  //      16-byte loads fix a permutation of the contraction (gx) / output row
  //      (gtq) index inside each group of 8 / 16 columns; both operands use
  //      the same one, and the order of every sum is fixed.
  static constexpr bool kRegStream = Lo::kRegStream;

#ifndef RGSV_BATCH_GX_CHAINS
#define RGSV_BATCH_GX_CHAINS 4  // DMMA accumulator chains per block in pass_gx_reg (2 or 4)
#endif
#ifndef RGSV_BATCH_PREFETCH
#define RGSV_BATCH_PREFETCH 6
#endif
  // Software pipeline shared by both passes. A warp owns `cnt` blocks, the
  // first `cntf` of them loadable without predicates (whole rows, n == NP).
  // ptxas tracks every streaming load of this kernel on ONE scoreboard (the
  // DMMA chains and the shared-memory loads take the others), so a consumer
  // that waits for its block waits for every load in flight, and a classic
  // k-deep register pipeline collapses to depth zero (measured: 2, 3 and 4
  // deep ran alike, with the warps stalled on the first DMMA of each block,
  // profiles/r02_batch_chain_*). The order that does overlap under that
  // constraint: the first DMMAs of block i wait for block i (and thereby for
  // everything issued so far), THEN the loads of block i + 1 are issued, then
  // the rest of block i computes without any further wait on the load
  // scoreboard. Two register buffers; the steady state is one basic block
  // per pair of blocks (the refill index is clamped, not guarded).
  // compute(d, i, hook) must call hook() once, after its first DMMAs.
  template <typename LoadFast, typename LoadSlow, typename Compute>
  RGSV_DI void pipeline(int cnt, int cntf, LoadFast&& load_fast, LoadSlow&& load_slow,
                        Compute&& compute) {
    if (cntf > 0) {
      load_fast(0, 0);
      const int pairs = cntf >> 1;
      for (int gp = 0; gp < pairs; ++gp) {
        const int i = 2 * gp;
        compute(0, i, [&] { load_fast(1, i + 1); });
        compute(1, i + 1, [&] { load_fast(0, min(i + 2, cntf - 1)); });  // clamped re-read
      }
      if (cntf & 1) compute(0, cntf - 1, [] {});
    }
    for (int i = cntf; i < cnt; ++i) {  // partial blocks / ragged columns: not pipelined
      load_slow(0, i);
      compute(0, i, [] {});
    }
  }

  // Y[8-row block] = G_block X: thread (g, t) loads G[row g][8u + 2t, +1];
  // k-step 2u + h contracts the columns 8u + 2t + h.
  RGSV_DI void pass_gx_reg(const BatchMat& g, int r0, int r1, int n, double* ss) {
    constexpr int NK = NP / 4, NCB = KP / 8;
    const int gq = lane >> 2, t = lane & 3;
    double xf[NCB][NK];
#pragma unroll
    for (int cb = 0; cb < NCB; ++cb)
#pragma unroll
      for (int sidx = 0; sidx < NK; ++sidx)
        xf[cb][sidx] = xt[(cb * 8 + gq) * GP + 8 * (sidx >> 1) + 2 * t + (sidx & 1)];
    const int nblk = (r1 - r0 + 7) / 8;
    const int nfull = n == NP ? (r1 - r0) / 8 : 0;
    const int cnt = nblk > warp ? (nblk - warp + kWarps - 1) / kWarps : 0;
    const int cntf = nfull > warp ? (nfull - warp + kWarps - 1) / kWarps : 0;
    double a[2][NK];
    const uint64_t pol = l2_policy(true);
    const double* gbase = g.g + (int64_t)(r0 + gq) * g.ld + 2 * t;
    const int64_t bstride = 8 * g.ld;
    double sq = 0.0;
    const bool want_ss = ss != nullptr;
    // The sketch pass is the one that reads G from HBM: an L2 prefetch (no
    // destination register, hence no scoreboard) runs kPrefetch blocks ahead
    // of the loads, one 128-byte line per lane and block, so the loads find
    // their lines in L2 like the three later passes do.
    constexpr int kPrefetch = RGSV_BATCH_PREFETCH;
    const double* pbase = g.g + (int64_t)(r0 + (lane >> 2)) * g.ld + (lane & 3) * 16;
    pipeline(
        cnt, cntf,
        [&](int d, int i) {
          const double* src = gbase + (warp + i * kWarps) * bstride;
          if (kPrefetch > 0 && want_ss && i + kPrefetch < cntf)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pbase + (warp + (i + kPrefetch) * kWarps) *
                                                                      bstride));
#pragma unroll
          for (int u = 0; u < NP / 8; ++u)
            ldg_stream2(a[d][2 * u], a[d][2 * u + 1], src + 8 * u, pol);
        },
        [&](int d, int i) {
          const int b = warp + i * kWarps;
          const double* src = gbase + b * bstride;
          const bool rok = r0 + b * 8 + gq < r1;
#pragma unroll
          for (int u = 0; u < NP / 8; ++u) {
            const int col = 8 * u + 2 * t;
            if (rok && col + 1 < n) {
              ldg_stream2(a[d][2 * u], a[d][2 * u + 1], src + 8 * u);
            } else {
              a[d][2 * u] = (rok && col < n) ? ldg_stream1(src + 8 * u) : 0.0;
              a[d][2 * u + 1] = 0.0;
            }
          }
        },
        [&](int d, int i, auto&& hook) {
          double c[NCB][2][2] = {};
#pragma unroll
          for (int cb = 0; cb < NCB; ++cb) dmma(c[cb][0], a[d][0], xf[cb][0]);
          hook();  // the next block's loads, behind the wait for this one
#pragma unroll
          for (int sidx = 1; sidx < NK; ++sidx)
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb)
              dmma(c[cb][(sidx & 1) * (RGSV_BATCH_GX_CHAINS / 4)], a[d][sidx], xf[cb][sidx]);
          if (want_ss) {
#pragma unroll
            for (int sidx = 0; sidx < NK; ++sidx) sq = fma(a[d][sidx], a[d][sidx], sq);
          }
          const int r = (warp + i * kWarps) * 8 + gq;
#pragma unroll
          for (int cb = 0; cb < NCB; ++cb) {
            const int col = cb * 8 + 2 * t;
            ys[yx<KP>(r, col)] = c[cb][0][0] + c[cb][1][0];
            ys[yx<KP>(r, col + 1)] = c[cb][0][1] + c[cb][1][1];
          }
        });
    if (ss) *ss += sq;
  }

  // part = G^T Y over this CTA's rows: thread (g, t) loads G[row t][16v + 2g,
  // +1]; output block 2v + h holds the G columns 16v + 2g + h. Warps work in
  // pairs: pair p = warp / 2 owns the 8-row blocks p, p + 4, ... and each of
  // its two warps takes one half of the columns (its own 2 x 128-byte segments
  // of every row), so a block costs a warp 16 registers; every warp
  // accumulates its NP/2 x KP half over the pair's rows, and the four pair
  // partials are folded in a fixed order through the (idle) ring memory.
  RGSV_DI void pass_gtq_reg(const BatchMat& g, int r0, int r1, int n, bool final_pass) {
    constexpr int NV = NP / 32, NJB = KP / 8, SP = Lo::SP;
    constexpr int kPairs = kWarps / 2;
    static_assert(kPairs == 4, "two fold slots, two phases");
    const int gq = lane >> 2, t = lane & 3;
    const int pr = warp >> 1, c0 = (warp & 1) * (NP / 2);  // this warp's column half
    double acc[2 * NV][NJB][2] = {};
    const int nblk = (r1 - r0 + 7) / 8;
    const int nfull = n == NP ? (r1 - r0) / 8 : 0;
    const int cnt = nblk > pr ? (nblk - pr + kPairs - 1) / kPairs : 0;
    const int cntf = nfull > pr ? (nfull - pr + kPairs - 1) / kPairs : 0;
    double a[2][2][NV][2];
    const uint64_t pol = l2_policy(!final_pass);
    const double* gbase = g.g + (int64_t)(r0 + t) * g.ld + c0 + 2 * gq;
    const int64_t bstride = 8 * g.ld, hstride = 4 * g.ld;
    pipeline(
        cnt, cntf,
        [&](int d, int i) {
          const double* src = gbase + (pr + i * kPairs) * bstride;
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int v = 0; v < NV; ++v)
              ldg_stream2(a[d][h][v][0], a[d][h][v][1], src + h * hstride + 16 * v, pol);
        },
        [&](int d, int i) {
          const int b = pr + i * kPairs;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = r0 + b * 8 + 4 * h + t;
            const bool rok = row < r1;
            const double* src = g.g + (int64_t)row * g.ld + c0 + 2 * gq;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const int col = c0 + 16 * v + 2 * gq;
              if (rok && col + 1 < n) {
                ldg_stream2(a[d][h][v][0], a[d][h][v][1], src + 16 * v);
              } else {
                a[d][h][v][0] = (rok && col < n) ? ldg_stream1(src + 16 * v) : 0.0;
                a[d][h][v][1] = 0.0;
              }
            }
          }
        },
        [&](int d, int i, auto&& hook) {
          const int rl0 = (pr + i * kPairs) * 8;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double bf[NJB];
#pragma unroll
            for (int jb = 0; jb < NJB; ++jb) bf[jb] = ys[yx<KP>(rl0 + 4 * h + t, jb * 8 + gq)];
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
#pragma unroll
                for (int jb = 0; jb < NJB; ++jb) dmma(acc[2 * v + e][jb], a[d][h][v][e], bf[jb]);
                if (h == 0 && v == 0 && e == 0) hook();  // next loads behind this block's wait
              }
          }
        });
    // fixed-order fold through two slots: pairs 0, 1 store, pairs 2, 3 add
    // theirs, then (p0 + p2) + (p1 + p3) lands in the region the cluster
    // reduction reads (rewritten only by the next pass_gtq, several cluster
    // barriers later)
    double* scr = gst + (pr & 1) * (NP * SP);
    __syncthreads();  // zb / wred (aliased by the fold slots) are no longer read
#pragma unroll
    for (int ph = 0; ph < kPairs / 2; ++ph) {
      if ((pr >> 1) == ph) {
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int jb = 0; jb < NJB; ++jb) {
              double2* q = reinterpret_cast<double2*>(scr + (c0 + 16 * v + 2 * gq + e) * SP +
                                                      jb * 8 + 2 * t);
              double2 val = make_double2(acc[2 * v + e][jb][0], acc[2 * v + e][jb][1]);
              if (ph > 0) {
                const double2 o = *q;
                val.x = o.x + val.x;
                val.y = o.y + val.y;
              }
              *q = val;
            }
      }
      __syncthreads();
    }
    double* dst = gst + Lo::kFold;
    for (int e = tid; e < NP * KP; e += kThreads) {
      const int o = (e / KP) * SP + (e % KP);
      dst[e] = gst[o] + gst[NP * SP + o];
    }
  }

  // ---- Y[t-tile] = G_tile X  (pass A); optional sum of squares of G
  RGSV_DI void pass_gx(const BatchMat& g, int r0, int r1, int n, double* ss) {
    if constexpr (kRegStream) {
      pass_gx_reg(g, r0, r1, n, ss);
      return;
    }
    constexpr int kRB = kTR / 8, kCB = KP / 8, kBlocks = kRB * kCB;
    static_assert(kBlocks % kWarps == 0, "whole blocks per warp");
    constexpr int kPer = kBlocks / kWarps;
    // X fragments are the same for every tile: keep them in registers
    double xf[kPer][NP / 4];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int cb = (warp + i * kWarps) / kRB;
      const double* brow = xt + (cb * 8 + (lane >> 2)) * GP + (lane & 3);
#pragma unroll
      for (int ks = 0; ks < NP / 4; ++ks) xf[i][ks] = brow[ks * 4];
    }
    stream_g(g, r0, r1, n, [&](int t, const double* gt) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int b = warp + i * kWarps;
        const int rb = b % kRB, cb = b / kRB;
        double cc[4][2] = {};
        const int ar = rb * 8 + (lane >> 2);
#pragma unroll
        for (int ks = 0; ks < NP / 4; ks += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            dmma(cc[u], gt[gx_idx<NP>(ar, (ks + u) * 4 + (lane & 3))], xf[i][ks + u]);
        }
        double c[2] = {(cc[0][0] + cc[1][0]) + (cc[2][0] + cc[3][0]),
                       (cc[0][1] + cc[1][1]) + (cc[2][1] + cc[3][1])};
        const int r = t * kTR + rb * 8 + (lane >> 2);
        const int col = cb * 8 + 2 * (lane & 3);
        ys[yx<KP>(r, col)] = c[0];
        ys[yx<KP>(r, col + 1)] = c[1];
      }
      if (ss) {
        double a = 0.0;
        for (int e = tid; e < kTR * NP; e += kThreads) {
          const double v = gt[gx_idx<NP>(e / NP, e % NP)];
          a = fma(v, v, a);
        }
        *ss += a;
      }
    });
  }

  // ---- part = G^T Y over this CTA's rows (pass B), NP x KP
  RGSV_DI void pass_gtq(const BatchMat& g, int r0, int r1, int n, bool final_pass) {
    if constexpr (kRegStream) {
      pass_gtq_reg(g, r0, r1, n, final_pass);
      return;
    }
    constexpr int kIB = NP / 8, kJB = KP / 8, kBlocks = kIB * kJB;
    constexpr int kPer = (kBlocks + kWarps - 1) / kWarps;
    double acc[kPer][2][2] = {};
    stream_g(g, r0, r1, n, [&](int t, const double* gt) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int b = warp + i * kWarps;
        if (b >= kBlocks) break;
        const int ib = b % kIB, jb = b / kIB;
#pragma unroll
        for (int ks = 0; ks < kTR / 4; ++ks) {
          const int rr = ks * 4 + (lane & 3);
          const double a = gt[gx_idx<NP>(rr, ib * 8 + (lane >> 2))];
          const double bv = ys[yx<KP>(t * kTR + rr, jb * 8 + (lane >> 2))];
          dmma(acc[i][ks & 1], a, bv);
        }
      }
    });
    double* dst = slot_ptr();
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int b = warp + i * kWarps;
      if (b >= kBlocks) break;
      const int ib = b % kIB, jb = b / kIB;
      const int r = ib * 8 + (lane >> 2), c = jb * 8 + 2 * (lane & 3);
      dst[r * KP + c] = acc[i][0][0] + acc[i][1][0];
      dst[r * KP + c + 1] = acc[i][0][1] + acc[i][1][1];
    }
  }

  // ---- Gram of a swizzled slice buf (rows x KP) into this CTA's part slot
  RGSV_DI void gram_partial(const double* buf, int rows) {
    constexpr int kB = (KP / 8) * (KP / 8);
    const int nks = (rows + 3) / 4;
    double* dst = slot_ptr();
    if constexpr (kB >= kWarps) {
      for (int b = warp; b < kB; b += kWarps) {
        const int ib = b % (KP / 8), jb = b / (KP / 8);
        double c[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
        int ks = 0;
        for (; ks + 1 < nks; ks += 2) {
          const int rr = ks * 4 + (lane & 3);
          dmma(c, buf[yx<KP>(rr, ib * 8 + (lane >> 2))], buf[yx<KP>(rr, jb * 8 + (lane >> 2))]);
          dmma(c2, buf[yx<KP>(rr + 4, ib * 8 + (lane >> 2))],
               buf[yx<KP>(rr + 4, jb * 8 + (lane >> 2))]);
        }
        if (ks < nks) {
          const int rr = ks * 4 + (lane & 3);
          dmma(c, buf[yx<KP>(rr, ib * 8 + (lane >> 2))], buf[yx<KP>(rr, jb * 8 + (lane >> 2))]);
        }
        c[0] += c2[0];
        c[1] += c2[1];
        const int r = ib * 8 + (lane >> 2), col = jb * 8 + 2 * (lane & 3);
        dst[r * KP + col] = c[0];
        dst[r * KP + col + 1] = c[1];
      }
      return;
    } else {
    // KP = 16: the Gram is symmetric, so only the three 8 x 8 blocks on and
    // below the diagonal are multiplied ((0,0), (1,0), (1,1)); warp w takes
    // the k-steps w, w + 8, ... of all three and the 8 warp partials are
    // folded in a fixed order. The strictly upper block is the mirror (the
    // same products in the same order, so the Gram stays exactly symmetric).
    static_assert(KP == 16 && kWarps == 8, "lower-block Gram layout");
    const int g = lane >> 2, t = lane & 3;
    double c[3][2][2] = {};
    // two k-steps per iteration into separate accumulators (independent
    // DMMA chains); rows are a multiple of 32, so nks is a multiple of 8
    for (int ks = warp; ks < nks; ks += 2 * kWarps) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (ks + u * kWarps < nks) {
          const int rr = (ks + u * kWarps) * 4 + t;
          const double y0 = buf[yx<KP>(rr, g)], y1 = buf[yx<KP>(rr, 8 + g)];
          dmma(c[0][u], y0, y0);
          dmma(c[1][u], y1, y0);
          dmma(c[2][u], y1, y1);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      wred[(warp * 3 + b) * 64 + lane * 2] = c[b][0][0] + c[b][1][0];
      wred[(warp * 3 + b) * 64 + lane * 2 + 1] = c[b][0][1] + c[b][1][1];
    }
    __syncthreads();
    if (warp < 3) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < kWarps; ++w) {  // fixed order
        s0 += wred[(w * 3 + warp) * 64 + lane * 2];
        s1 += wred[(w * 3 + warp) * 64 + lane * 2 + 1];
      }
      const int ib = warp == 0 ? 0 : 1, jb = warp == 2 ? 1 : 0;
      const int r = ib * 8 + g, col = jb * 8 + 2 * t;
      dst[r * KP + col] = s0;
      dst[r * KP + col + 1] = s1;
      if (ib != jb) {
        dst[col * KP + r] = s0;
        dst[(col + 1) * KP + r] = s1;
      }
    }
    }
  }

  // ---- shifted Cholesky of gram (k x k) -> linv = L^-1; identity on the
  //      padding. One warp, register resident (lane i holds row i; columns
  //      are compile-time indices). Symmetric Gauss-Jordan: eliminating below
  //      pivot j with row operations turns [A | I] into [D Lhat^T | Lhat^-1];
  //      scaling row j by d_j^-1/2 makes the right half L^-1, so the inverse
  //      needs no separate substitution sweep. Row j is broadcast by
  //      independent shuffles; the critical path per step is one shuffle,
  //      one rsqrt and one FMA.
  //      Returns true when the near-identity route produced the inverse.
  RGSV_DI bool chol(int k, int64_t shift_rows) {
    constexpr int LD = KP + 1;
    static_assert(KP <= 32, "one lane per row");
#ifdef RGSV_BATCH_PROFILE
    if (tid == 0) atomicAdd(&g_batch_prof[15], 1ull);
    const long long _c0 = clock64();
#endif
    if (shift_rows == 0 && near_identity_inverse(k)) {
#ifdef RGSV_BATCH_PROFILE
      if (tid == 0) atomicAdd(&g_batch_prof[13], (unsigned long long)(clock64() - _c0));
#endif
      return true;
    }
    if constexpr (KP == 16) {
      chol16(k, shift_rows);
      __syncthreads();
      return false;
    }
    if (warp == 0) {
#ifdef RGSV_BATCH_PROFILE
      long long _g0 = clock64();
#endif
      const bool row_ok = lane < k;
      double a[KP], x[KP];
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        a[c] = (row_ok && c < k) ? gram[lane * LD + c] : (lane == c ? 1.0 : 0.0);
        x[c] = (lane == c) ? 1.0 : 0.0;
      }
      if (shift_rows > 0) {
        double dg = 0.0;
#pragma unroll
        for (int c = 0; c < KP; ++c)
          if (c == lane && row_ok) dg = a[c];
        const double tr = warp_sum(dg);
        const double sh = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
#pragma unroll
        for (int c = 0; c < KP; ++c)
          if (c == lane && row_ok) a[c] += sh;
      }
      bool bad = false;
#ifdef RGSV_BATCH_PROFILE
      long long _g1 = clock64();
#endif
#pragma unroll
      for (int j = 0; j < KP; ++j) {
        const double d = __shfl_sync(0xffffffffu, a[j], j);
        double pa[KP], px[KP];
#pragma unroll
        for (int c = 0; c < KP; ++c) {
          if (c > j) pa[c] = __shfl_sync(0xffffffffu, a[c], j);
          if (c <= j) px[c] = __shfl_sync(0xffffffffu, x[c], j);
        }
        bad |= !(d > 0.0) || !isfinite(d);
        const double r = rsqrt(d);
        // branch-free row operation: rows below eliminate (ff = A[i][j] / d),
        // the pivot row scales by d^-1/2 (mul = r), rows above are untouched
        const double ff = (lane > j) ? a[j] * (r * r) : 0.0;
        const double mul = (lane == j) ? r : 1.0;
#pragma unroll
        for (int c = 0; c < KP; ++c) {
          if (c > j) a[c] = fma(-ff, pa[c], a[c]) * mul;
          if (c <= j) x[c] = fma(-ff, px[c], x[c]) * mul;
        }
        a[j] = (lane > j) ? 0.0 : (lane == j ? d * r : a[j]);
      }
#ifdef RGSV_BATCH_PROFILE
      long long _g2 = clock64();
#endif
      if (bad) fail = 1;
      if (lane < KP) {
#pragma unroll
        for (int c = 0; c < KP; ++c)
          linv[lane * LD + c] = bad ? (lane == c ? 1.0 : 0.0) : (c <= lane ? x[c] : 0.0);
      }
#ifdef RGSV_BATCH_PROFILE
      if (lane == 0 && (blockIdx.x & 3) == 0) {
        long long _g3 = clock64();
        atomicAdd(&g_batch_prof[16], (unsigned long long)(_g1 - _g0));
        atomicAdd(&g_batch_prof[17], (unsigned long long)(_g2 - _g1));
        atomicAdd(&g_batch_prof[18], (unsigned long long)(_g3 - _g2));
        atomicAdd(&g_batch_prof[19], 1ull);
      }
#endif
    }
    __syncthreads();
    return false;
  }

  // ---- the same symmetric Gauss-Jordan for KP = 16 on the whole CTA: thread
  //      (i, c) = (tid / 16, tid % 16) owns A[i][c] and X[i][c] in registers.
  //      Per pivot j it needs the pivot row (A[j][c], X[j][c]), its own row's
  //      column-j entry A[i][j] and d = A[j][j]: every thread publishes its
  //      two entries in a double-buffered shared-memory copy, so one CTA
  //      barrier per published state suffices. The j loop is NOT unrolled: the
  //      body is ~100 instructions that stay in the instruction cache (the unrolled
  //      one-warp form was 2500 instructions per call site, executed once per
  //      call, i.e. instruction-fetch bound: 9.5 us per call). Same operations
  //      in the same order per entry as the one-warp form (bitwise equal).
  RGSV_DI void chol16(int k, int64_t shift_rows) {
    constexpr int LD = KP + 1;
    static_assert(kThreads == 256, "one thread per entry of the 16 x 16 pivot");
    const int i = tid >> 4, c = tid & 15;
    double a = (i < k && c < k) ? gram[i * LD + c] : (i == c ? 1.0 : 0.0);
    double x = (i == c) ? 1.0 : 0.0;
    // double-buffered copies: [buf][A | X][16 x LD] in lmat / the idle wred
    double* pub = wred;  // 2 x 2 x 16 x LD = 1088 doubles <= kWarps * 3 * 64
    static_assert(4 * 16 * (KP + 1) <= kWarps * 3 * 64, "chol16 buffers fit wred");
    if (shift_rows > 0) {
      if (tid < 16) lmat[tid] = (tid < k) ? gram[tid * LD + tid] : 0.0;
      __syncthreads();
      // trace in the order of the one-warp form's xor butterfly (8, 4, 2, 1)
      double t8[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) t8[e] = lmat[e];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1)
#pragma unroll
        for (int e = 0; e < o; ++e) t8[e] = t8[e] + t8[e + o];
      const double tr = t8[0];
      const double sh = 11.0 * ((double)shift_rows * k + (double)k * (k + 1)) * 0x1p-53 * tr;
      if (i == c && i < k) a += sh;
      __syncthreads();
    }
    bool bad = false;
    // Two pivots (j, j + 1) per published state: every thread re-derives what
    // pivot j does to row j + 1, column j + 1 and d_{j+1} with the very
    // operations their owner threads perform, so the result equals the
    // one-pivot-per-barrier sweep bit for bit at half the barriers and
    // shared-memory round trips (the sweep is a pure latency chain).
#pragma unroll 1
    for (int j = 0; j < 16; j += 2) {
      double* pa = pub + ((j >> 1) & 1) * (2 * 16 * LD);
      double* px = pa + 16 * LD;
      pa[i * LD + c] = a;
      px[i * LD + c] = x;
      __syncthreads();
      const double d0 = pa[j * LD + j], b10 = pa[(j + 1) * LD + j];
      const double u01 = pa[j * LD + j + 1], e11 = pa[(j + 1) * LD + j + 1];
      const double ai0 = pa[i * LD + j], ai1 = pa[i * LD + j + 1];
      const double ra0 = pa[j * LD + c], ra1 = pa[(j + 1) * LD + c];
      const double rx0 = px[j * LD + c], rx1 = px[(j + 1) * LD + c];
      // pivot j
      bad |= !(d0 > 0.0) || !isfinite(d0);
      const double r0 = rsqrt(d0);
      const double rr0 = r0 * r0;
      const double ff0 = (i > j) ? ai0 * rr0 : 0.0;
      const double mul0 = (i == j) ? r0 : 1.0;
      if (c > j) a = fma(-ff0, ra0, a) * mul0;
      else x = fma(-ff0, rx0, x) * mul0;
      if (c == j) a = (i > j) ? 0.0 : (i == j ? d0 * r0 : a);
      // what pivot j did to row j + 1 (multiplier f10, scale 1) and column j + 1
      const double f10 = b10 * rr0;
      const double d1 = fma(-f10, u01, e11) * 1.0;
      const double ra1n = fma(-f10, ra0, ra1) * 1.0;               // used for c > j + 1
      const double rx1n = (c <= j) ? fma(-f10, rx0, rx1) * 1.0 : rx1;  // c == j + 1: untouched
      const double ai1n = fma(-ff0, u01, ai1) * 1.0;               // used for i > j + 1
      // pivot j + 1
      bad |= !(d1 > 0.0) || !isfinite(d1);
      const double r1 = rsqrt(d1);
      const double ff1 = (i > j + 1) ? ai1n * (r1 * r1) : 0.0;
      const double mul1 = (i == j + 1) ? r1 : 1.0;
      if (c > j + 1) a = fma(-ff1, ra1n, a) * mul1;
      else x = fma(-ff1, rx1n, x) * mul1;
      if (c == j + 1) a = (i > j + 1) ? 0.0 : (i == j + 1 ? d1 * r1 : a);
    }
    if (bad) fail = 1;
    __syncthreads();  // wred (pub) is reused by the callers right after
    linv[i * LD + c] = bad ? (i == c ? 1.0 : 0.0) : (c <= i ? x : 0.0);
  }

  // ---- third CholeskyQR pass: gram = I + E with max|E| <= 1e-6 ->
  //      L^-1 = I - X + X^2, X = Phi(E - X1 X1^T), X1 = Phi(E) (Phi: strict
  //      lower + half diagonal); exact in fp64 (neglected terms O(|E|^3)).
  //      Returns false (nothing written) when the Gram is not that close.
  RGSV_DI bool near_identity_inverse(int k) {
    constexpr int LD = KP + 1;
    constexpr int NT8 = KP / 8;
    double mx = 0.0;
    for (int e = tid; e < KP * KP; e += kThreads) {
      const int i = e / KP, c = e % KP;
      if (i < k && c < k) mx = fmax(mx, fabs(gram[i * LD + c] - (i == c ? 1.0 : 0.0)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) wred[warp * 64 + 2] = mx;
    __syncthreads();
    double m = 0.0;
    for (int w = 0; w < kWarps; ++w) m = fmax(m, wred[w * 64 + 2]);
    if (!(m <= 1e-6)) return false;  // uniform across the CTA
#ifdef RGSV_BATCH_PROFILE
    if (tid == 0) atomicAdd(&g_batch_prof[14], 1ull);
#endif
    const int g = lane >> 2, t = lane & 3;
    // lmat := X1 = Phi(E), gram := E (padding 0)
    for (int e = tid; e < KP * KP; e += kThreads) {
      const int i = e / KP, c = e % KP;
      const double ev = (i < k && c < k) ? gram[i * LD + c] - (i == c ? 1.0 : 0.0) : 0.0;
      gram[i * LD + c] = ev;
      lmat[i * LD + c] = (c < i) ? ev : (c == i ? 0.5 * ev : 0.0);
    }
    __syncthreads();
    if (warp < NT8 * NT8) {  // gram := E - X1 X1^T
      const int ti = warp / NT8, tc = warp % NT8;
      double m2[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < KP / 4; ++ks)
        dmma(m2, lmat[(ti * 8 + g) * LD + ks * 4 + t], lmat[(tc * 8 + g) * LD + ks * 4 + t]);
      gram[(ti * 8 + g) * LD + tc * 8 + 2 * t] -= m2[0];
      gram[(ti * 8 + g) * LD + tc * 8 + 2 * t + 1] -= m2[1];
    }
    __syncthreads();
    for (int e = tid; e < KP * KP; e += kThreads) {  // lmat := X = Phi(gram)
      const int i = e / KP, c = e % KP;
      lmat[i * LD + c] = (c < i) ? gram[i * LD + c] : (c == i ? 0.5 * gram[i * LD + c] : 0.0);
    }
    __syncthreads();
    if (warp < NT8 * NT8) {  // linv := I - X + X^2
      const int ti = warp / NT8, tc = warp % NT8;
      double m2[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < KP / 4; ++ks)
        dmma(m2, lmat[(ti * 8 + g) * LD + ks * 4 + t], lmat[(ks * 4 + t) * LD + tc * 8 + g]);
      const int i = ti * 8 + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tc * 8 + 2 * t + h;
        linv[i * LD + c] = (c <= i) ? ((i == c ? 1.0 : 0.0) - lmat[i * LD + c] + m2[h]) : 0.0;
      }
    }
    __syncthreads();
    return true;
  }

  // ---- buf (rows x KP, swizzled) <- buf L^-T, in place, warp per 8 rows
  RGSV_DI void trsm(double* buf, int rows) {
    constexpr int LD = KP + 1;
    const int nrb = (rows + 7) / 8;
    // L^-T fragments are shared by every row block: registers
    double lf[KP / 8][KP / 4];
#pragma unroll
    for (int cb = 0; cb < KP / 8; ++cb)
#pragma unroll
      for (int ks = 0; ks < KP / 4; ++ks)
        lf[cb][ks] = linv[(cb * 8 + (lane >> 2)) * LD + ks * 4 + (lane & 3)];
    // two row blocks per iteration: independent DMMA chains
    for (int rb0 = warp * 2; rb0 < nrb; rb0 += kWarps * 2) {
      double a[2][KP / 4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = (rb0 + h) * 8 + (lane >> 2);
#pragma unroll
        for (int ks = 0; ks < KP / 4; ++ks)
          a[h][ks] = (rb0 + h < nrb) ? buf[yx<KP>(r, ks * 4 + (lane & 3))] : 0.0;
      }
      __syncwarp();
      double c[2][KP / 8][2] = {};
      // L^-1 is lower triangular: output column block cb only sees the
      // k-steps ks <= 2 cb + 1 (the skipped products are exact zeros)
#pragma unroll
      for (int ks = 0; ks < KP / 4; ++ks)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int cb = 0; cb < KP / 8; ++cb)
            if (ks <= 2 * cb + 1) dmma(c[h][cb], a[h][ks], lf[cb][ks]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (rb0 + h >= nrb) break;
        const int r = (rb0 + h) * 8 + (lane >> 2);
#pragma unroll
        for (int cb = 0; cb < KP / 8; ++cb) {
          const int col = cb * 8 + 2 * (lane & 3);
          buf[yx<KP>(r, col)] = c[h][cb][0];
          buf[yx<KP>(r, col + 1)] = c[h][cb][1];
        }
      }
    }
    __syncthreads();
  }

  // ---- shifted CholeskyQR3 of a row-sharded slice (cluster Gram) or of a
  //      replicated small matrix (local Gram, no cluster traffic)
  //      defer_last: the third pass stops after its Cholesky -- buf keeps
  //      Q2 and linv holds L3^-1 -- because the only consumer of Q is the
  //      next G^T Q pass: G^T (Q2 L3^-T) = (G^T Q2) L3^-T is applied to the
  //      reduced n x k product instead of the m x k slice.
  //      The passes stop as soon as one of them (after the shifted first)
  //      found its Gram within 1e-6 of I: near_identity_inverse is exact to
  //      O(|E|^3) <= 1e-18 there, so the basis it produces is orthonormal to
  //      rounding and a further pass could only re-round it.
  //      side: a block-local scalar (||G||^2 partial) summed over the cluster
  //      together with the first Gram (one cluster barrier instead of two);
  //      the total lands in misc[0].
  RGSV_DI void cholqr3(double* buf, int rows, int k, int64_t shift_rows, bool sharded,
                       bool defer_last = false, const double* side = nullptr) {
    constexpr int LD = KP + 1;
    static_assert(KP * KP + 1 <= Lo::kPart, "Gram + side scalar fit a reduction slot");
    PROF_T0();
    for (int pass = 0; pass < 3; ++pass) {
      gram_partial(buf, rows);
      PROF(4);
      if (sharded) {
        const bool with_side = side != nullptr && pass == 0;
        if (with_side && tid == 0) slot_ptr()[KP * KP] = *side;
        reduce(KP * KP + (with_side ? 1 : 0), [&](int e, double s) {
          if (e < KP * KP) gram[(e / KP) * LD + (e % KP)] = s;
          else misc[0] = s;
        });
      } else {
        __syncthreads();
        const double* src = slot_ptr();
        for (int e = tid; e < KP * KP; e += kThreads) gram[(e / KP) * LD + (e % KP)] = src[e];
        __syncthreads();
      }
      PROF(5);
      const bool converged = chol(k, pass == 0 ? shift_rows : 0);
      PROF(6);
      const bool last_pass = pass == 2 || (pass >= 1 && converged);
      if (defer_last && last_pass) break;
      trsm(buf, rows);
      PROF(7);
      if (last_pass) break;
    }
  }
};

template <int NP, int KP, int CS>
__global__ void __launch_bounds__(kThreads, 1) k_batch_chain(ChainArgs A) {
  extern __shared__ __align__(16) double smc[];
  Chain<NP, KP, CS> C;
  C.init(smc, A.yrows);
  constexpr int LD = KP + 1;
  const int n = A.n, k = A.k;
  // Matrices are handed out by a global counter (rank 0 of the cluster draws,
  // the peers read its draw over DSMEM): clusters that start late -- the
  // chunked launches of rgsv_batch_gsvd share the GPU with filler kernels --
  // simply take fewer. Which cluster computes a matrix does not change its
  // result (every reduction inside a chain is fixed-order).
  __shared__ int next_mat;
  for (int it = 0;; ++it) {
    int mat;
    if (A.next) {
      if (C.crank == 0 && C.tid == 0) next_mat = atomicAdd(A.next, 1);
      __syncthreads();
      cluster_barrier();
      mat = ld_dsmem_i32(&next_mat, 0);  // rewritten only after the next matrix's barriers
    } else {
      mat = (int)cluster_idx() + it * (int)cluster_count();
    }
    if (mat >= A.nmat) break;
    const BatchMat g = A.mats[mat];
    const int rows = g.rows;
    const int rpc = (rows + CS - 1) / CS;
    const int r0 = min(rows, (int)C.crank * rpc), r1 = min(rows, r0 + rpc);
    const int rl = r1 - r0;
    const int rlt = (rl + kTR - 1) / kTR * kTR;
    C.fail = 0;
    PROF_T0();
    // X^T = Omega^T block (KP x n), zero-padded
    const double* om = A.omega + (int64_t)mat * A.om_stride;
    for (int e = C.tid; e < KP * NP; e += kThreads) {
      const int i = e / NP, j = e % NP;
      C.xt[i * C.GP + j] = (i < k && j < n) ? om[(int64_t)i * A.ldo + j] : 0.0;
    }
    // Y rows the passes never write must read as zero in the Grams / TRSMs
    // (they run over rlt rows): the register passes write whole 8-row blocks,
    // so only the rows behind the last block are cleared; the ring passes
    // write every row of their 32-row tiles themselves (zero-filled copies).
    if constexpr (Chain<NP, KP, CS>::kRegStream) {
      for (int e = ((rl + 7) / 8) * 8 * KP + C.tid; e < rlt * KP; e += kThreads) C.ys[e] = 0.0;
    } else {
      for (int e = C.tid; e < A.yrows * KP; e += kThreads) C.ys[e] = 0.0;
    }
    __syncthreads();
    // One textual instance of every phase (the chain used to inline three
    // cholqr3 and two bodies of each pass: 315 KB of code run once per
    // matrix, i.e. instruction-fetch bound). Half-steps: even = the tall side
    // (Y = G X with X = Omega or Qhat, CholeskyQR3 of the Y slice, then
    // G^T Q reduced over the cluster with the deferred L3^-T applied: Z, or
    // B^T on the last half-step), odd = the small side (Qhat = cholqr3(Z)).
    double ss = 0.0;
    PROF(0);
    const int last = 2 * A.q;
#pragma unroll 1
    for (int hs = 0;; ++hs) {
      const bool tall = (hs & 1) == 0;
      if (tall) {
        if (hs > 0) {
          for (int e = C.tid; e < KP * NP; e += kThreads) {
            const int i = e / NP, j = e % NP;
            C.xt[i * C.GP + j] = (j < n) ? C.zb[yx<KP>(j, i)] : 0.0;
          }
          __syncthreads();
        }
        C.pass_gx(g, r0, r1, n, hs == 0 ? &ss : nullptr);
        __syncthreads();
        PROF(hs == 0 ? 1 : 3);  // 1: the sketch pass (G from HBM), 3: later G X passes (L2)
        if (hs == 0) {  // ||G||_F^2: block partial in fixed order; summed over the
                        // cluster with the first Gram (cholqr3's side scalar)
          double v = warp_sum(ss);
          if (C.lane == 0) C.wred[C.warp * 64] = v;
          __syncthreads();
          if (C.tid == 0) {
            double s = 0.0;
            for (int w = 0; w < kWarps; ++w) s += C.wred[w * 64];
            C.misc[1] = s;
          }
          __syncthreads();
          PROF(8);
        }
      }
      C.cholqr3(tall ? C.ys : C.zb, tall ? rlt : NP, k, tall ? rows : n, tall, tall,
                hs == 0 ? C.misc + 1 : nullptr);
      PROF(9);
      if (tall) {
        C.pass_gtq(g, r0, r1, n, hs == last);
        PROF(2);
        C.reduce_gtq([&](int e, double s) { C.zb[yx<KP>(e / KP, e % KP)] = s; });
        C.trsm(C.zb, NP);  // the deferred L3^-T of Q
        PROF(10);
        if (hs == last) break;
      }
    }
    if (C.crank == 0) {
      double* bo = A.b_out + (int64_t)mat * A.b_stride;
      double e2 = 0.0;
      for (int e = C.tid; e < KP * n; e += kThreads) {
        const int i = e / n, j = e % n;
        const double v = (i < k) ? C.zb[yx<KP>(j, i)] : 0.0;
        bo[(int64_t)i * A.ldb + j] = v;
        e2 = fma(v, v, e2);
      }
      e2 = warp_sum(e2);
      if (C.lane == 0) C.wred[C.warp * 64 + 1] = e2;
      __syncthreads();
      if (C.tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += C.wred[w * 64 + 1];
        A.stats[2 * mat] = C.misc[0];
        A.stats[2 * mat + 1] = s;
        int st = C.fail ? RGSV_ST_CHOL_BREAKDOWN : 0;
        if (!isfinite(C.misc[0])) st |= RGSV_ST_NONFINITE;
        A.status[mat] = st;
      }
    }
    (void)LD;
    __syncthreads();
    PROF(12);
  }
  cluster_barrier();  // no CTA leaves while a peer may still read its slots
}

template <int NP, int KP, int CS>
int launch_chain_t(const ChainArgs& a, cudaStream_t st) {
  const size_t smem = Layout<NP, KP>::bytes(a.yrows);
  if (smem > 227 * 1024) return RGSV_ERR_DIMENSION;
  auto kern = k_batch_chain<NP, KP, CS>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return RGSV_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent clusters: exactly as many as can be co-resident, otherwise the
  // clusters that do not fit would run their whole matrix list afterwards
  static int resident[9] = {};
  int& clusters_max = resident[CS];
  if (clusters_max == 0) {
    cfg.gridDim = dim3(kSMs / CS * CS, 1, 1);
    if (cudaOccupancyMaxActiveClusters(&clusters_max, (void*)kern, &cfg) != cudaSuccess ||
        clusters_max < 1)
      clusters_max = kSMs / CS;
  }
  int clusters = clusters_max;
  if (clusters > a.nmat) clusters = a.nmat;
  cfg.gridDim = dim3(clusters * CS, 1, 1);
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return RGSV_ERR_CUDA;
  note_launch();
  return 0;
}

template <int NP, int KP>
int launch_chain_np(const ChainArgs& a, int cs, cudaStream_t st) {
  switch (cs) {
    case 1: return launch_chain_t<NP, KP, 1>(a, st);
    case 2: return launch_chain_t<NP, KP, 2>(a, st);
    case 3: return launch_chain_t<NP, KP, 3>(a, st);
    case 4: return launch_chain_t<NP, KP, 4>(a, st);
    case 8: return launch_chain_t<NP, KP, 8>(a, st);
  }
  return RGSV_ERR_DIMENSION;
}

}  // namespace

// Cluster size and Y-slice rows for a batch: the smallest portable cluster
// whose per-CTA slice fits the shared-memory budget.
int batch_chain_plan(int max_rows, int n, int k, int* cs_out, int* yrows_out) {
  const int kp = k <= 16 ? 16 : 32;
  const int np = n <= 64 ? 64 : 128;
  if (k < 1 || k > 32 || n < 1 || n > 128 || k > n) return RGSV_ERR_DIMENSION;
  // smallest cluster whose CTAs hold the Y slice; RGSV_BATCH_CS raises the
  // minimum (tuning; cfg3 measured 79.1k / 55.2k pairs/s at 4 / 8)
  static const int cs_min = [] {
    const char* e = getenv("RGSV_BATCH_CS");
    const int v = e ? atoi(e) : 1;
    return (v == 2 || v == 3 || v == 4 || v == 8) ? v : 1;
  }();
  // 3-CTA clusters pack the GPCs better than 4 (48 x 3 vs 33 x 4 SMs busy)
  // and spread a matrix's serial phases over fewer SMs
  static const int sizes[] = {1, 2, 3, 4, 8};
  for (int cs : sizes) {
    if (cs < cs_min) continue;
    const int rpc = (max_rows + cs - 1) / cs;
    const int yrows = (rpc + kTR - 1) / kTR * kTR;
    size_t bytes;
    if (np == 64) bytes = kp == 16 ? Layout<64, 16>::bytes(yrows) : Layout<64, 32>::bytes(yrows);
    else bytes = kp == 16 ? Layout<128, 16>::bytes(yrows) : Layout<128, 32>::bytes(yrows);
    if (bytes <= 227 * 1024) {
      *cs_out = cs;
      *yrows_out = yrows;
      return 0;
    }
  }
  return RGSV_ERR_DIMENSION;
}

int batch_chain(const BatchMat* mats, int nmat, int max_rows, int n, int k, int q,
                const double* omega, int64_t ldo, int64_t om_stride, double* b_out, int64_t ldb,
                int64_t b_stride, double* stats, int* status, int* next, cudaStream_t st) {
  int cs, yrows;
  if (int e = batch_chain_plan(max_rows, n, k, &cs, &yrows)) return e;
  if (next && cudaMemsetAsync(next, 0, sizeof(int), st) != cudaSuccess) return RGSV_ERR_CUDA;
  ChainArgs a{mats, nmat, n, k, q, omega, ldo, om_stride, b_out, ldb, b_stride, stats, status,
              yrows, next};
  const int kp = k <= 16 ? 16 : 32;
  if (n <= 64) return kp == 16 ? launch_chain_np<64, 16>(a, cs, st) : launch_chain_np<64, 32>(a, cs, st);
  return kp == 16 ? launch_chain_np<128, 16>(a, cs, st) : launch_chain_np<128, 32>(a, cs, st);
}

}  // namespace rgsv

extern "C" int rgsv_debug_batch_profile(unsigned long long* out16, int reset) {
#ifdef RGSV_BATCH_PROFILE
  if (out16 && cudaMemcpyFromSymbol(out16, rgsv::g_batch_prof, sizeof(unsigned long long) * 24) !=
                   cudaSuccess)
    return RGSV_ERR_CUDA;
  if (reset) {
    unsigned long long z[24] = {};
    if (cudaMemcpyToSymbol(rgsv::g_batch_prof, z, sizeof(z)) != cudaSuccess) return RGSV_ERR_CUDA;
  }
  return 0;
#else
  (void)out16;
  (void)reset;
  return RGSV_ERR_VALIDATION;  // library built without -DRGSV_BATCH_PROFILE
#endif
}
