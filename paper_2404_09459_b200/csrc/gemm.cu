// Skinny FP64 GEMMs of the rGSVD hot path (SURVEY.md §2b K1-K3, K5 Gram/TRSM):
//
//   gx : Y  (M x N)  = G (M x K) * X      with X given K-major as Xt (N x K)
//        (sketch Y = G*Omega, power step Y = G*Qhat, CholQR TRSM Q = Y*Rinv,
//         wide Gram B*B^T)
//   gtq: C  (Mk x N) = Q^T (Mk x K) * G (K x N), reduction over the rows of
//        both row-major operands (power step / projection B = Q^T G, CholQR
//        Gram Y^T Y, wide TRSM Linv*B)
//
// Layout: every operand is row-major in HBM. A CTA = 1 producer warp (one
// elected lane issues TMA for both operands of a 16-deep K chunk into a
// STAGES-deep ring, 128B swizzle) + WM*WN DMMA warps. Fragment loads are
// conflict-free: for gx both operands are K-major (8 rows x 4 consecutive
// doubles per fragment); for gtq both are MN-major and the 4 K indices of a
// k4 step are taken as rows {j, j+4, j+8, j+12} of the chunk so that the two
// row pairs land in opposite halves of the swizzled bank space.
//
// Work decomposition: blockIdx.x enumerates `full` whole-K tiles first, then
// the tail tiles split `split` ways along K; split units write partials that
// k_reduce_splits sums in a fixed order (results are bitwise deterministic).
#include <stdlib.h>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {

// Operand fragments are read with explicit ld.shared: the staging pointers
// come out of integer alignment arithmetic on the dynamic shared-memory base,
// which hides their address space from the compiler -- it emitted generic
// LD.E.64 (checked in SASS), with the generic path's address-space test and
// the long-latency scoreboard class, instead of LDS.64.
#ifndef RGSV_GEMM_GENERIC_LD
RGSV_DI double lds_f64(const uint8_t* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}
#else
RGSV_DI double lds_f64(const uint8_t* p) { return *reinterpret_cast<const double*>(p); }
#endif

constexpr int kMaxTileMap = 64;

struct Decomp {
  int tiles_n;      // tiles along the output's N dimension
  int full;         // units [0, full): tile = u, whole K range
  int tail_tile0;   // first split tile
  int split;        // splits per tail tile
  int nchunks;      // 16-deep K chunks
  int cps;          // chunks per split
  int nmap;         // > 0: unit tiles index tmap (a lower-triangular Gram's tiles)
  short tmap[kMaxTileMap];
};

RGSV_DI void decode_unit(const Decomp& d, int u, int& tile, int& c0, int& c1, int& s) {
  if (u < d.full) {
    tile = u;
    c0 = 0;
    c1 = d.nchunks;
    s = -1;
  } else {
    int v = u - d.full;
    tile = d.tail_tile0 + v / d.split;
    s = v % d.split;
    c0 = s * d.cps;
    c1 = min(d.nchunks, c0 + d.cps);
    if (c1 < c0) c1 = c0;
  }
  if (d.nmap > 0) tile = d.tmap[tile];
}

// ------------------------------------------------------------------- gx
template <int MT, int NT, int WM, int WN, int STAGES, bool SUMSQ, int MINB = 1>
__global__ void __launch_bounds__((WM * WN + 1) * 32, MINB)
    k_gx(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmX,
         double* __restrict__ out, int64_t ld_out, double* __restrict__ part,
         int64_t part_stride, int part_row0, int M, int N, Decomp d,
         double* __restrict__ ss_out, int zero_to) {
  constexpr int BM = MT * 8 * WM, BN = NT * 8 * WN, NCW = WM * WN;
  constexpr uint32_t G_BYTES = BM * 128, X_BYTES = BN * 128, STAGE = G_BYTES + X_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  __shared__ double red[NCW];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tile, c0, c1, split;
  decode_unit(d, blockIdx.x, tile, c0, c1, split);
  const int tm = tile / d.tiles_n, tn = tile % d.tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const int nk = c1 - c0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCW) {  // producer
    if (lane == 0) {
      tma_prefetch(&tmG);
      tma_prefetch(&tmX);
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE);
        uint8_t* st = smem + s * STAGE;
        const int kx = (c0 + i) * 16;
        tma_load_2d(st, &tmG, &full[s], kx, m0);
        tma_load_2d(st + G_BYTES, &tmX, &full[s], kx, n0);
      }
    }
    return;
  }

  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, t = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ss = 0.0;
  const bool do_ss = SUMSQ && wn == 0 && tn == 0;

  for (int i = 0; i < nk; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const uint8_t* sg = smem + s * STAGE;
    const uint8_t* sx = sg + G_BYTES;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int kap = kk * 4 + t;
      double a[MT], b[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        a[mt] = lds_f64(sg + swz128_f64((wm * MT + mt) * 8 + g, kap));
        if (SUMSQ && do_ss) ss = fma(a[mt], a[mt], ss);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        b[nt] = lds_f64(sx + swz128_f64((wn * NT + nt) * 8 + g, kap));
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt], a[mt], b[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  double* o;
  int64_t ldo;
  int rbase;
  if (split < 0) {
    o = out;
    ldo = ld_out;
    rbase = 0;
  } else {
    o = part + split * part_stride;
    ldo = ld_out;
    rbase = part_row0;
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int row = m0 + (wm * MT + mt) * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int col = n0 + (wn * NT + nt) * 8 + 2 * t;
      double* p = o + (int64_t)(row - rbase) * ldo + col;
      if (col + 1 < N) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      } else if (col < N) {
        p[0] = acc[mt][nt][0];
      }
    }
    // exact-width variant: the padding columns [N, zero_to) of the output
    // (never multiplied) are stored as zeros, straight to `out`
    if (zero_to > N && wn == WN - 1 && tn == d.tiles_n - 1) {
      double* zr = out + (int64_t)row * ld_out;
      for (int col = N + 2 * t; col < zero_to; col += 8) {
        zr[col] = 0.0;
        if (col + 1 < zero_to) zr[col + 1] = 0.0;
      }
    }
  }
  if (SUMSQ) {
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
    if (threadIdx.x == 0 && tn == 0) {
      double tot = 0.0;
      for (int w = 0; w < NCW; ++w) tot += red[w];
      ss_out[blockIdx.x] = tot;
    }
  }
}

// ------------------------------------------------------------------ gtq
template <int MT, int NT, int WM, int WN, int STAGES, int MINB = 1>
__global__ void __launch_bounds__((WM * WN + 1) * 32, MINB)
    k_gtq(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmG,
          double* __restrict__ out, int64_t ld_out, double* __restrict__ part,
          int64_t part_stride, int Mk, int N, Decomp d, int zero_to) {
  constexpr int BM = MT * 8 * WM, BN = NT * 8 * WN, NCW = WM * WN;
  // Q is staged in 16-column boxes: an exact-width BM (120) stages 128
  // columns (the OOB tail is zero-filled by TMA) and multiplies BM of them
  constexpr int QBOX = (BM + 15) / 16, GBOX = BN / 16;
  static_assert(BN % 16 == 0, "G tile width must be whole 16-column boxes");
  constexpr uint32_t Q_BYTES = QBOX * 2048, G_BYTES = BN * 128, STAGE = Q_BYTES + G_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tile, c0, c1, split;
  decode_unit(d, blockIdx.x, tile, c0, c1, split);
  const int tk = tile / d.tiles_n, tn = tile % d.tiles_n;
  const int k0 = tk * BM, n0 = tn * BN;
  const int nk = c1 - c0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCW) {
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmG);
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE);
        uint8_t* st = smem + s * STAGE;
        const int y = (c0 + i) * 16;
#pragma unroll 1
        for (int b = 0; b < QBOX; ++b) tma_load_2d(st + b * 2048, &tmQ, &full[s], k0 + b * 16, y);
#pragma unroll 1
        for (int b = 0; b < GBOX; ++b)
          tma_load_2d(st + Q_BYTES + b * 2048, &tmG, &full[s], n0 + b * 16, y);
      }
    }
    return;
  }

  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, t = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int i = 0; i < nk; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const uint8_t* sq = smem + s * STAGE;
    const uint8_t* sg = sq + Q_BYTES;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rho = j + 4 * t;
      double a[MT], b[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int c = (wm * MT + mt) * 8 + g;
        a[mt] = lds_f64(sq + (c >> 4) * 2048 + swz128_f64(rho, c & 15));
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = (wn * NT + nt) * 8 + g;
        b[nt] = lds_f64(sg + (c >> 4) * 2048 + swz128_f64(rho, c & 15));
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt], a[mt], b[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  double* o = split < 0 ? out : part + split * part_stride;
  // exact-width variant: output rows [Mk, zero_to) (never multiplied) are
  // stored as zeros, straight to `out`
  if (zero_to > Mk && wm == 0 && tk == 0) {
    for (int row = Mk + g; row < zero_to; row += 8)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int col = n0 + (wn * NT + nt) * 8 + 2 * t;
        double* p = out + (int64_t)row * ld_out + col;
        if (col + 1 < N) {
          *reinterpret_cast<double2*>(p) = make_double2(0.0, 0.0);
        } else if (col < N) {
          p[0] = 0.0;
        }
      }
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int row = k0 + (wm * MT + mt) * 8 + g;
    if (row >= Mk) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int col = n0 + (wn * NT + nt) * 8 + 2 * t;
      double* p = o + (int64_t)row * ld_out + col;
      if (col + 1 < N) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      } else if (col < N) {
        p[0] = acc[mt][nt][0];
      }
    }
  }
}

// out[r][c] = sum_{s < S} part[s][r][c] for r < rows, c < cols. A block
// handles 32 consecutive entries with 8 warps splitting the S partials
// (coalesced 256-byte rows per warp), then folds the 8 warp sums in a fixed
// order: bitwise deterministic.
__global__ void __launch_bounds__(256) k_reduce_splits(double* __restrict__ out, int64_t ld,
                                                       const double* __restrict__ part,
                                                       int64_t part_stride, int S, int rows,
                                                       int cols, int lower_bm = 0,
                                                       int lower_bn = 0) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t total = (int64_t)rows * cols;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    const int64_t e = base + lane;
    double acc = 0.0;
    int64_t off = 0;
    // lower-triangular Gram: entries of skipped (strictly upper) tiles are
    // left untouched
    const bool live = e < total && (lower_bm == 0 || (int)(e % cols) / lower_bn * lower_bn <
                                                        ((int)(e / cols) / lower_bm + 1) * lower_bm);
    if (live) {
      off = (e / cols) * ld + (e % cols);
      const double* p = part + off;
#pragma unroll 4
      for (int s = grp; s < S; s += 8) acc += p[(int64_t)s * part_stride];
    }
    red[grp][lane] = acc;
    __syncthreads();
    if (grp == 0 && live) {
      double t = 0.0;
#pragma unroll
      for (int g2 = 0; g2 < 8; ++g2) t += red[g2][lane];
      out[off] = t;
    }
    __syncthreads();
  }
}

static int reduce_blocks(int64_t total) {
  int64_t b = (total + 31) / 32;
  if (b > 8 * kSMs) b = 8 * kSMs;
  return b < 1 ? 1 : (int)b;
}

// -------------------------------------------------------------- host side
namespace {

// RGSV_EXACT_WIDTH=0 turns the exact-width (k = 120) tiles off (A/B runs).
bool exact_width_enabled() {
  static const bool on = [] {
    const char* e = getenv("RGSV_EXACT_WIDTH");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// RGSV_TILE96=0 turns the 96-wide tiles (widths that are multiples of 96,
// cfg4's kp = 288) off (A/B runs).
bool tile96_enabled() {
  static const bool on = [] {
    const char* e = getenv("RGSV_TILE96");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

template <typename K>
int set_smem(K kernel, size_t bytes) {
  static thread_local const void* done[64];
  static thread_local int ndone = 0;
  for (int i = 0; i < ndone; ++i)
    if (done[i] == reinterpret_cast<const void*>(kernel)) return 0;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess)
    return RGSV_ERR_CUDA;
  if (ndone < 64) done[ndone++] = reinterpret_cast<const void*>(kernel);
  return 0;
}

// Tile-shape experiments on the cfg1 shapes (tools/gemm_ab.py), both slower
// than the configurations below: 2 CTAs/SM with a 4-stage ring (gtq 109 vs
// 99 us, gx 149 vs 90 us) and 12 DMMA warps per CTA (gtq 105, gx 111 us).
// Plan the unit list for `tiles` output tiles over `nchunks` K chunks.
Decomp plan_units(int tiles_m, int tiles_n, int nchunks, int max_split, int* units, int* S,
                  int per_sm = 1) {
  Decomp d{};
  const int tiles = tiles_m * tiles_n;
  d.tiles_n = tiles_n;
  d.nchunks = nchunks;
  const int slots = kSMs * per_sm;
  // whole-K tiles fill complete waves; the remainder (rounded out to whole
  // tile rows so split rows never overlap whole-K rows) is split along K.
  const int waves = tiles / slots;
  const int full = (waves * slots / tiles_n) * tiles_n;
  const int tail = tiles - full;
  int split = 1;
  if (tail != 0) split = slots / tail;
  if (split > max_split) split = max_split;
  if (split > nchunks / 2) split = nchunks / 2;
  if (split < 1) split = 1;
  if (split == 1 || (waves > 0 && tail > slots * 3 / 4)) {
    d.full = tiles;
    d.tail_tile0 = tiles;
    d.split = 1;
    d.cps = nchunks;
    *units = tiles;
    *S = 0;
  } else {
    d.full = full;
    d.tail_tile0 = full;
    d.split = split;
    d.cps = (nchunks + split - 1) / split;
    *units = full + tail * split;
    *S = split;
  }
  return d;
}

template <int MT, int NT, int WM, int WN, int STAGES, bool SUMSQ, int MINB = 1>
int run_gx(const GemmArgs& a, cudaStream_t st) {
  constexpr int BM = MT * 8 * WM, BN = NT * 8 * WN;
  CUtensorMap tmG, tmX;
  if (make_tmap_2d(&tmG, a.A, a.K, a.M, a.lda, 16, BM, 8)) return RGSV_ERR_CUDA;
  if (make_tmap_2d(&tmX, a.B, a.K, a.N, a.ldb, 16, BN, 8)) return RGSV_ERR_CUDA;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int nchunks = (int)((a.K + 15) / 16);
  int units, S;
  Decomp d = plan_units(tiles_m, tiles_n, nchunks, a.max_split, &units, &S, MINB);
  if (SUMSQ && tiles_n != 1) return RGSV_ERR_DIMENSION;
  int part_row0 = 0;
  if (S > 0) {
    part_row0 = (d.tail_tile0 / tiles_n) * BM;
    const size_t need = (size_t)S * (size_t)(a.M - part_row0) * a.ldc * sizeof(double);
    if (need > a.scratch_bytes) return RGSV_ERR_WORKSPACE;
  }
  const int64_t part_stride = (int64_t)(a.M - part_row0) * a.ldc;
  const size_t smem = STAGES * (BM + BN) * 128 + 2 * STAGES * 8 + 1024;
  auto kern = k_gx<MT, NT, WM, WN, STAGES, SUMSQ, MINB>;
  if (int e = set_smem(kern, smem)) return e;
  kern<<<units, (WM * WN + 1) * 32, smem, st>>>(tmG, tmX, a.C, a.ldc, a.scratch, part_stride,
                                                 part_row0, (int)a.M, (int)a.N, d, a.ss_out,
                                                 a.zero_to);
  note_launch();
  if (S > 0) {
    const int rows = (int)(a.M - part_row0);
    const int blocks = reduce_blocks((int64_t)rows * a.N);
    k_reduce_splits<<<blocks, 256, 0, st>>>(a.C + (int64_t)part_row0 * a.ldc, a.ldc, a.scratch,
                                            part_stride, S, rows, (int)a.N);
    note_launch();
  }
  if (a.ss_units) *a.ss_units = units;
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

template <int MT, int NT, int WM, int WN, int STAGES, int MINB = 1>
int run_gtq(const GemmArgs& a, cudaStream_t st) {
  constexpr int BM = MT * 8 * WM, BN = NT * 8 * WN;
  CUtensorMap tmQ, tmG;
  // Q: K rows x M cols (ld lda); G: K rows x N cols (ld ldb)
  if (make_tmap_2d(&tmQ, a.A, a.M, a.K, a.lda, 16, 16, 8)) return RGSV_ERR_CUDA;
  if (make_tmap_2d(&tmG, a.B, a.N, a.K, a.ldb, 16, 16, 8)) return RGSV_ERR_CUDA;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int nchunks = (int)((a.K + 15) / 16);
  int tiles = tiles_m * tiles_n;
  Decomp d{};
  d.tiles_n = tiles_n;
  d.nchunks = nchunks;
  // a.lower_only: only tiles touching the lower triangle (n0 < m0 + BM)
  bool lower = false;
  if (a.lower_only && tiles <= kMaxTileMap) {
    int nm = 0;
    for (int t = 0; t < tiles; ++t)
      if ((t % tiles_n) * BN < (t / tiles_n + 1) * BM) d.tmap[nm++] = (short)t;
    if (nm < tiles) {
      d.nmap = nm;
      tiles = nm;
      lower = true;
    }
  }
  int split = kSMs * MINB / tiles;
  if (split > a.max_split) split = a.max_split;
  if (split > nchunks) split = nchunks;
  if (split < 1) split = 1;
  // Long reductions (cfg2: 12500 K-chunks over 63 tiles): choose the split
  // that fills whole waves best (63 x 2 = 126 of 148 SMs -> 63 x 7 = 441 of
  // 444 slots), keeping >= 256 chunks per unit so the pipeline fill stays
  // negligible; fewer splits win ties.
  if (nchunks / 256 > split) {
    const int slots = kSMs * MINB;
    double best = (double)(tiles * split) / (double)(((tiles * split + slots - 1) / slots) * slots);
    const int smax = nchunks / 256 < a.max_split ? nchunks / 256 : a.max_split;
    for (int sp = split + 1; sp <= smax; ++sp) {
      const int u = tiles * sp;
      const double eff = (double)u / (double)(((u + slots - 1) / slots) * slots);
      if (eff > best + 0.02) {
        best = eff;
        split = sp;
      }
    }
  }
  // never more partials than the caller's scratch holds
  const size_t per_split = (size_t)a.M * a.ldc * sizeof(double);
  if (split > 1 && (size_t)split * per_split > a.scratch_bytes)
    split = per_split ? (int)(a.scratch_bytes / per_split) : 1;
  if (split < 1) split = 1;
  int units = tiles, S = 0;
  if (split == 1) {
    d.full = tiles;
    d.tail_tile0 = tiles;
    d.split = 1;
    d.cps = nchunks;
  } else {
    d.full = 0;
    d.tail_tile0 = 0;
    d.split = split;
    d.cps = (nchunks + split - 1) / split;
    units = tiles * split;
    S = split;
    const size_t need = (size_t)S * a.M * a.ldc * sizeof(double);
    if (need > a.scratch_bytes) return RGSV_ERR_WORKSPACE;
  }
  const int64_t part_stride = (int64_t)a.M * a.ldc;
  const size_t smem = STAGES * (((BM + 15) / 16) * 16 + BN) * 128 + 2 * STAGES * 8 + 1024;
  auto kern = k_gtq<MT, NT, WM, WN, STAGES, MINB>;
  if (int e = set_smem(kern, smem)) return e;
  kern<<<units, (WM * WN + 1) * 32, smem, st>>>(tmQ, tmG, a.C, a.ldc, a.scratch, part_stride,
                                                 (int)a.M, (int)a.N, d, a.zero_to);
  note_launch();
  if (S > 0) {
    const int blocks = reduce_blocks((int64_t)a.M * a.N);
    k_reduce_splits<<<blocks, 256, 0, st>>>(a.C, a.ldc, a.scratch, part_stride, S, (int)a.M,
                                            (int)a.N, lower ? BM : 0, lower ? BN : 0);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

}  // namespace

// C (M x N) = A (M x K) * B^T  with B given as N x K (both K-major).
// a.live (> 0): only the first `live` output columns can be nonzero (the
// rest of B^T is zero padding); a live width of 120 in a 128-wide output
// (cfg2's k) runs the exact-width 128 x 120 tile and zero-fills columns
// 120..127. 12 DMMA warps of 32 x 40 (3 per SM sub-partition): 5603 us at
// cfg2 vs 5894 us for 8 warps of 16 x 120 and 6126 us for the padded tile.
int gemm_gx(const GemmArgs& a0, cudaStream_t st) {
  if (a0.M <= 0 || a0.N <= 0 || a0.K <= 0) return RGSV_ERR_DIMENSION;
  if (exact_width_enabled() && (a0.N == 120 || (a0.live == 120 && a0.N == 128))) {
    GemmArgs a = a0;
    a.zero_to = a0.N;  // 128: zero-fill the padding columns
    a.N = 120;
    if (a.ss_out) return run_gx<4, 5, 4, 3, 5, true>(a, st);
    return run_gx<4, 5, 4, 3, 5, false>(a, st);
  }
  const GemmArgs& a = a0;
  if (a.ss_out) {
    if (a.N <= 16) return run_gx<2, 2, 8, 1, 6, true>(a, st);
    if (a.N <= 32) return run_gx<2, 4, 8, 1, 6, true>(a, st);
    if (a.N <= 64) return run_gx<4, 4, 4, 2, 6, true>(a, st);
    if (a.N <= 128) return run_gx<4, 8, 4, 2, 5, true>(a, st);
    return RGSV_ERR_DIMENSION;
  }
  if (a.N <= 16) return run_gx<2, 2, 8, 1, 6, false>(a, st);
  if (a.N <= 32) return run_gx<2, 4, 8, 1, 6, false>(a, st);
  if (a.N <= 64) return run_gx<4, 4, 4, 2, 6, false>(a, st);
  // widths that are whole 96-column tiles (cfg4's kp = 288 = 3 x 96; 128-wide
  // tiles would issue 384 columns): 12 DMMA warps of 32 x 32
  if (tile96_enabled() && a.N > 128 && a.N % 96 == 0) return run_gx<4, 4, 4, 3, 5, false>(a, st);
  return run_gx<4, 8, 4, 2, 5, false>(a, st);
}

// C (M x N) = A^T * B with A: K x M, B: K x N (both row-major, reduction over K rows).
// a.live (> 0): only the first `live` output rows can be nonzero (the rest
// of A's columns are zero padding); live 120 of M 128 runs the exact-width
// 120 x 64 tile (12 DMMA warps of 40 x 16, 3 per SM sub-partition) and
// zero-fills rows 120..127. Measured at cfg2: 6125 us vs 6234 us for 8 warps
// of 120 x 8 and 6579 us for the padded 128-row tile; a 9-warp 120 x 96 tile
// ran 7559 us (9 warps split 3/2/2/2 over the 4 sub-partitions).
int gemm_gtq(const GemmArgs& a0, cudaStream_t st) {
  if (a0.M <= 0 || a0.N <= 0 || a0.K <= 0) return RGSV_ERR_DIMENSION;
  if (exact_width_enabled() && a0.N >= 64 && (a0.M == 120 || (a0.live == 120 && a0.M == 128))) {
    GemmArgs a = a0;
    a.zero_to = a0.M;  // 128: zero-fill the padding rows
    a.M = 120;
    // (cfg2 G1 shape, tools/gemm_variants.py: 6 stages 5933 us; 8 stages
    //  5907 us; 12 warps of 40 x 32 spill at 128 registers: 6112 / 6092 us)
    return run_gtq<5, 2, 3, 4, 6>(a, st);
  }
  const GemmArgs& a = a0;
  // Lower-triangular Gram whose width is whole 96-tiles (cfg4's kp = 288):
  // 96 x 96 tiles, 12 DMMA warps of 24 x 32. The 6 tiles on or below the
  // diagonal are 55296 entries against 90112 for the 11 live 128 x 64 tiles.
  if (tile96_enabled() && a.lower_only && a.M == a.N && a.M >= 192 && a.M % 96 == 0)
    return run_gtq<3, 4, 4, 3, 6>(a, st);
  if (a.N <= 16 && a.M <= 16) return run_gtq<1, 1, 2, 2, 6>(a, st);
  if (a.N <= 32 && a.M <= 32) return run_gtq<2, 2, 2, 2, 6>(a, st);
  if (a.N <= 64 && a.M <= 64) return run_gtq<4, 4, 2, 2, 6>(a, st);
  if (a.M <= 16) return run_gtq<2, 4, 1, 8, 6>(a, st);
  if (a.M <= 32) return run_gtq<2, 4, 2, 4, 6>(a, st);
  if (a.M <= 64) return run_gtq<4, 4, 2, 4, 6>(a, st);
  return run_gtq<4, 4, 4, 2, 6>(a, st);
}

}  // namespace rgsv
