// FP32 GEMM passes of fp32-resident pairs (the cfg4 family) on the 5th-gen
// tensor cores: tcgen05.mma .kind::tf32 with operands staged by TMA into
// swizzled shared memory and accumulators in TMEM.
//
// Precision: "3xTF32". A TF32 product keeps 11 significant bits per
// operand, so every fp32 operand x is carried as hi + lo with hi = x as the
// tensor core reads it and lo = tf32(x - hi); the kernels accumulate
//     hi_a*hi_b + hi_a*lo_b + lo_a*hi_b          (lo_a*lo_b ~ 2^-22, dropped)
// in FP32 TMEM, i.e. fp32-level products at three TF32 MMAs each (TF32 dense
// peak 1.1 PFLOP/s => ~370 TFLOP/s of fp32-accurate work vs 37 TFLOP/s of
// FP64 DMMA). The big operand G is read in place (its hi part is G itself);
// its lo part is one extra fp32 array written by rgsv_f32_split, which also
// returns ||G||_F^2 in fp64 (core.sum_sq, core.py:115-125). The small
// operands (Omega / Qhat^T / Q) are split from fp64 by rgsv_f64_split_tf32.
//
// Shapes (m = 1e6, n = 8192, kp = 288):
//   gx : Y (M x N, fp64) = G (M x K) * X^T, X: N x K row-major   [K-major A, B]
//        the sketch G*Omega and the power step G*Qhat (rangefinder.py:115)
//   gtq: C (N x M, fp64) = Q^T G, Q: K x N, G: K x M row-major   [MN-major A, B]
//        the power step G^T Q and the projection Q^T G (engine.py:255-256);
//        the long K = rows reduction is split over CTAs (fp64 partials,
//        summed in a fixed order -> deterministic).
//
// CTA = 10 warps: warp 0 issues TMA into a `stages`-deep mbarrier ring,
// warp 1 owns TMEM and one elected lane issues the tcgen05.mma chain
// (tcgen05.commit frees a stage / hands a TMEM slot to the epilogue), warps
// 2-9 drain the accumulator slots with tcgen05.ld (warp w reads TMEM lanes
// 32*(w%4)..+31) into fp32 registers and finally store fp64.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {
namespace {

constexpr int kTileM = 128;
constexpr uint32_t kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA
constexpr uint32_t kSmemReserve = 1024 + 256;  // 1 KB alignment slack + barriers

// --- tcgen05 / TMEM wrappers --------------------------------------------------
// Shared-memory matrix descriptor (PTX ISA "matrix descriptor", sm_100):
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48),
// base offset 0, layout [61,64): 2 = 128B swizzle, 4 = 64B swizzle.
RGSV_DI uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// Instruction descriptor, kind::tf32: D f32 [4,6)=1, A/B tf32 [7,10)/[10,13)=2,
// A/B major [15]/[16] (0 = K-major, 1 = MN-major), N>>3 [17,23), M>>4 [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

RGSV_DI void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Arrive on `bar` once every previously issued tcgen05.mma of this thread has
// completed (implies tcgen05.fence::before_thread_sync).
RGSV_DI void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
RGSV_DI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
RGSV_DI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RGSV_DI void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
RGSV_DI void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns (one TMEM lane per thread).
RGSV_DI void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// L2 prefetch of a 2-D tensor tile (no shared-memory destination).
RGSV_DI void tma_prefetch_l2(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}

RGSV_DI float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// --- kernel ---------------------------------------------------------------
// The tensor core's fp32 accumulation truncates (measured: a bias linear in
// the number of accumulation steps, ~7e-9 * K relative, tools/tf32_accuracy.py).
// So TMEM holds only a short partial: every `flush` K-blocks the MMA warp
// hands the accumulator slot to the epilogue warps, which add it into fp32
// registers with round-to-nearest and free the slot; TMEM is carved into
// rotating slots so the MMAs never wait on a drain. A CTA owns one 128-row
// tile and one output chunk of <= 160 columns (a multiple of 32); wider
// outputs (cfg4: kp = 288 = 160 + 128) take two CTAs per tile, adjacent in
// the grid so the second read of the G tile hits L2. Each of the 8 epilogue
// warps owns one TMEM lane quarter (warp % 4) and half of the chunk.
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kMaxChunk = 160;
constexpr int kMaxHalf = kMaxChunk / 2;
constexpr int kMaxSlots = 4;
constexpr uint32_t kTmemCols = 512;

enum { kGX = 0, kGTQ = 1 };

struct Smem {
  uint8_t* base;
  uint64_t* full;    // TMA -> MMA, per stage
  uint64_t* empty;   // MMA -> TMA, per stage
  uint64_t* sfull;   // MMA -> epilogue, per TMEM slot
  uint64_t* sempty;  // epilogue -> MMA, per TMEM slot (kEpiWarps arrivals)
  uint32_t* tslot;
};

RGSV_DI Smem carve(uint8_t* raw, int stages, uint32_t stage_bytes) {
  Smem r;
  r.base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  r.full = reinterpret_cast<uint64_t*>(r.base + (size_t)stages * stage_bytes);
  r.empty = r.full + stages;
  r.sfull = r.empty + stages;
  r.sempty = r.sfull + kMaxSlots;
  r.tslot = reinterpret_cast<uint32_t*>(r.sempty + kMaxSlots);
  return r;
}

// MODE kGX : out (M x N, ld ldo) = G (M x K) X^T; G, X K-major (BK*4-byte
//            swizzle rows). tg/tglo boxes {BK, 128}, tbh/tbl boxes {BK, c0w}.
// MODE kGTQ: out (N x M, ld ldo) = Q^T G over rows [y*rows_per, +rows_per);
//            G (K x M), Q (K x N) MN-major: runs of 32-column boxes of BK rows
//            (128B swizzle, 32B atoms). Split y writes at out + y * split_stride.
// blockIdx.x = tile * nchunk + chunk; chunk 0 = columns [0, c0w), chunk 1 =
// [c0w, N).
template <int MODE, int BK>
__global__ void __launch_bounds__(kThreads, 1)
    k_tf32x3(const __grid_constant__ CUtensorMap tg, const __grid_constant__ CUtensorMap tglo,
             const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbl,
             double* __restrict__ out, int64_t ldo, int64_t split_stride, int M, int N, int K,
             int rows_per, int c0w, int stages, int flush, int pf) {
  constexpr bool GX = MODE == kGX;
  constexpr uint32_t SW = GX ? BK * 4 : 128;   // bytes per swizzled smem row
  constexpr uint32_t BOX = BK * 128;           // kGTQ: one 32-column box
  // K-major: 64B / 128B swizzle; MN-major tf32: 128B swizzle with 32-byte atoms
  // (the only MN-major layout tcgen05 accepts for 32-bit operands)
  constexpr uint32_t LAYOUT = GX ? (BK == 16 ? 4u : 2u) : 1u;
  extern __shared__ uint8_t smem_raw[];
  const int nchunk = N > c0w ? 2 : 1;
  const int chunk = blockIdx.x % nchunk;
  const int col0 = chunk ? c0w : 0;
  const int W = chunk ? N - c0w : c0w;  // this CTA's output columns
  const uint32_t a_bytes = GX ? kTileM * SW : 4 * BOX;
  const uint32_t b_bytes = GX ? (uint32_t)c0w * SW : (uint32_t)(c0w / 32) * BOX;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  Smem R = carve(smem_raw, stages, stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (blockIdx.x / nchunk) * kTileM;
  const int r0 = GX ? 0 : blockIdx.y * rows_per;
  const int r1 = GX ? K : min(K, r0 + rows_per);
  const int nkb = (r1 - r0 + BK - 1) / BK;
  const int ns = min(kMaxSlots, (int)(kTmemCols / c0w));
  const int ngroups = (nkb + flush - 1) / flush;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(R.full + s, 1);
      mbar_init(R.empty + s, 1);
    }
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(R.sfull + s, 1);
      mbar_init(R.sempty + s, kEpiWarps);
    }
    fence_mbar_init();
    tma_prefetch(&tg);
    tma_prefetch(&tglo);
    tma_prefetch(&tbh);
    tma_prefetch(&tbl);
  }
  if (warp == 1) tmem_alloc(R.tslot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *R.tslot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        mbar_wait(R.empty + s, ph ^ 1u);
        uint8_t* st = R.base + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(R.full + s, stage_bytes);
        const int kk = r0 + kb * BK;
        // the G tiles come from HBM: prefetch them into L2 `pf` K-blocks ahead
        // (chunk 0 of a tile only; chunk 1 re-reads them from L2)
        const int kpf = kb + pf;
        if (pf > 0 && chunk == 0 && kpf < nkb) {
          const int kq = r0 + kpf * BK;
          if (GX) {
            tma_prefetch_l2(&tg, kq, m0);
            tma_prefetch_l2(&tglo, kq, m0);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              tma_prefetch_l2(&tg, m0 + 32 * j, kq);
              tma_prefetch_l2(&tglo, m0 + 32 * j, kq);
            }
          }
        }
        if (GX) {
          tma_load_2d(st, &tg, R.full + s, kk, m0);
          tma_load_2d(st + a_bytes, &tglo, R.full + s, kk, m0);
          tma_load_2d(st + 2 * a_bytes, &tbh, R.full + s, kk, col0);
          tma_load_2d(st + 2 * a_bytes + b_bytes, &tbl, R.full + s, kk, col0);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            tma_load_2d(st + j * BOX, &tg, R.full + s, m0 + 32 * j, kk);
            tma_load_2d(st + a_bytes + j * BOX, &tglo, R.full + s, m0 + 32 * j, kk);
          }
          for (int j = 0; j < c0w / 32; ++j) {
            tma_load_2d(st + 2 * a_bytes + j * BOX, &tbh, R.full + s, col0 + 32 * j, kk);
            tma_load_2d(st + 2 * a_bytes + b_bytes + j * BOX, &tbl, R.full + s, col0 + 32 * j,
                        kk);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = idesc_tf32(kTileM, W, GX ? 0 : 1, GX ? 0 : 1);
      // descriptor strides: K-major (LBO unused, SBO = 8 rows); MN-major
      // (LBO = next 32-column box, SBO = next 4-row swizzle atom)
      const uint32_t LBO = GX ? 16u : BOX, SBO = GX ? 8 * SW : 512u;
      const uint32_t koff = GX ? 32u : 1024u;  // one MMA-K step (8 tf32)
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        const int t = kb / flush;
        const int slot = t % ns;
        const bool first = (kb % flush) == 0;
        const bool last = (kb % flush) == flush - 1 || kb == nkb - 1;
        if (first) mbar_wait(R.sempty + slot, ((uint32_t)(t / ns) & 1u) ^ 1u);
        mbar_wait(R.full + s, ph);
        tc_fence_after();
        const uint32_t a = smem_u32(R.base + (size_t)s * stage_bytes);
        const uint32_t alo = a + a_bytes, bh = a + 2 * a_bytes, bl = bh + b_bytes;
        const uint32_t td = tbase + (uint32_t)(slot * c0w);
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint32_t ko = (uint32_t)k * koff;
          const uint64_t dA = umma_desc(a + ko, LBO, SBO, LAYOUT);
          const uint64_t dAl = umma_desc(alo + ko, LBO, SBO, LAYOUT);
          const uint64_t dBh = umma_desc(bh + ko, LBO, SBO, LAYOUT);
          const uint64_t dBl = umma_desc(bl + ko, LBO, SBO, LAYOUT);
          mma_tf32(td, dA, dBh, id, (!first || k > 0) ? 1u : 0u);
          mma_tf32(td, dA, dBl, id, 1u);
          mma_tf32(td, dAl, dBh, id, 1u);
        }
        if (last) mma_commit(R.sfull + slot);
        mma_commit(R.empty + s);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;         // TMEM lane quarter of this warp
    const int h = (warp - 2) >> 2;  // which half of the chunk
    const int hw = W / 2;           // multiple of 16
    float acc[kMaxHalf];
#pragma unroll
    for (int j = 0; j < kMaxHalf; ++j) acc[j] = 0.f;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * hw);
    for (int t = 0; t < ngroups; ++t) {
      const int slot = t % ns;
      mbar_wait(R.sfull + slot, (uint32_t)(t / ns) & 1u);
      tc_fence_after();
      const uint32_t src = lane_base + (uint32_t)(slot * c0w);
#pragma unroll
      for (int j0 = 0; j0 < kMaxHalf; j0 += 16) {
        if (j0 < hw) {
          float v[16];
          tmem_ld16(src + (uint32_t)j0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[j0 + i] += v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(R.sempty + slot);
    }
    const int idx = m0 + q * 32 + lane;
    if (idx < M) {
      const int c = col0 + h * hw;
      if (GX) {
        double* dst = out + (int64_t)idx * ldo + c;
#pragma unroll
        for (int j = 0; j < kMaxHalf; j += 2)
          if (j < hw) *reinterpret_cast<double2*>(dst + j) = make_double2(acc[j], acc[j + 1]);
      } else {
        double* dst = out + (int64_t)blockIdx.y * split_stride + idx;
#pragma unroll
        for (int j = 0; j < kMaxHalf; ++j)
          if (j < hw) dst[(int64_t)(c + j) * ldo] = (double)acc[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kTmemCols);
  }
}

// ============================================================================
// gx on CTA PAIRS (tcgen05 cta_group::2): a 2-CTA cluster computes a 256-row
// tile; each CTA stages its own 128 rows of G (+ lo) and HALF of the X chunk,
// and the leader's single thread issues M = 256 MMAs that read both CTAs'
// shared memory and write both CTAs' TMEM. Per SM this halves the staged X
// bytes (52 instead of 72 KB per 32-deep K-block, 4 stages instead of 3).
// Barriers: full[] live in the leader (both CTAs' TMA bytes land there;
// count 2 = leader expect_tx + peer arrive); empty[] and sfull[] in both CTAs
// (leader's multicast commits); sempty[] in the leader (16 epilogue warps).
RGSV_DI uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
RGSV_DI void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
RGSV_DI uint32_t mapa_u32(const void* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
RGSV_DI void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// 2-SM TMA: the transaction bytes complete on the LEADER's barrier (peer bit
// of the barrier address cleared), the data lands in this CTA's smem.
RGSV_DI void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
RGSV_DI void mma_tf32_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
RGSV_DI void mma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

template <int BK>
__global__ void __launch_bounds__(kThreads, 1)
    k_tf32x3_gx2(const __grid_constant__ CUtensorMap tg, const __grid_constant__ CUtensorMap tglo,
                 const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbl,
                 double* __restrict__ out, int64_t ldo, int M, int N, int K, int c0w, int stages,
                 int flush) {
  constexpr uint32_t SW = BK * 4;
  constexpr uint32_t LAYOUT = BK == 16 ? 4u : 2u;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t rank = cta_rank();
  const int nchunk = N > c0w ? 2 : 1;
  const int pair = blockIdx.x >> 1;
  const int chunk = pair % nchunk;
  const int col0 = chunk ? c0w : 0;
  const int W = chunk ? N - c0w : c0w;   // MMA N (both CTAs' halves)
  const int hb = c0w / 2;                // staged X rows per CTA (box)
  const uint32_t a_bytes = kTileM * SW;
  const uint32_t b_bytes = (uint32_t)hb * SW;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  Smem R = carve(smem_raw, stages, stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (pair / nchunk) * 2 * kTileM + (int)rank * kTileM;
  const int xrow0 = col0 + (int)rank * (W / 2);
  const int nkb = (K + BK - 1) / BK;
  const int ns = min(kMaxSlots, (int)(kTmemCols / c0w));
  const int ngroups = (nkb + flush - 1) / flush;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(R.full + s, 2);
      mbar_init(R.empty + s, 1);
    }
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(R.sfull + s, 1);
      mbar_init(R.sempty + s, 2 * kEpiWarps);
    }
    fence_mbar_init();
    tma_prefetch(&tg);
    tma_prefetch(&tglo);
    tma_prefetch(&tbh);
    tma_prefetch(&tbl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(R.tslot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = *R.tslot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full_leader = mapa_u32(R.full, 0);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        mbar_wait(R.empty + s, ph ^ 1u);
        uint8_t* st = R.base + (size_t)s * stage_bytes;
        if (rank == 0)
          mbar_arrive_expect_tx(R.full + s, 2 * stage_bytes);
        else
          mbar_arrive_remote(full_leader + (uint32_t)s * 8u);
        const int kk = kb * BK;
        tma_load_2d_2sm(st, &tg, R.full + s, kk, m0);
        tma_load_2d_2sm(st + a_bytes, &tglo, R.full + s, kk, m0);
        tma_load_2d_2sm(st + 2 * a_bytes, &tbh, R.full + s, kk, xrow0);
        tma_load_2d_2sm(st + 2 * a_bytes + b_bytes, &tbl, R.full + s, kk, xrow0);
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      const uint32_t id = idesc_tf32(2 * kTileM, W, 0, 0);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        const int t = kb / flush;
        const int slot = t % ns;
        const bool first = (kb % flush) == 0;
        const bool last = (kb % flush) == flush - 1 || kb == nkb - 1;
        if (first) mbar_wait(R.sempty + slot, ((uint32_t)(t / ns) & 1u) ^ 1u);
        mbar_wait(R.full + s, ph);
        tc_fence_after();
        const uint32_t a = smem_u32(R.base + (size_t)s * stage_bytes);
        const uint32_t alo = a + a_bytes, bh = a + 2 * a_bytes, bl = bh + b_bytes;
        const uint32_t td = tbase + (uint32_t)(slot * c0w);
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint32_t ko = (uint32_t)k * 32u;
          const uint64_t dA = umma_desc(a + ko, 16, 8 * SW, LAYOUT);
          const uint64_t dAl = umma_desc(alo + ko, 16, 8 * SW, LAYOUT);
          const uint64_t dBh = umma_desc(bh + ko, 16, 8 * SW, LAYOUT);
          const uint64_t dBl = umma_desc(bl + ko, 16, 8 * SW, LAYOUT);
          mma_tf32_2sm(td, dA, dBh, id, (!first || k > 0) ? 1u : 0u);
          mma_tf32_2sm(td, dA, dBl, id, 1u);
          mma_tf32_2sm(td, dAl, dBh, id, 1u);
        }
        if (last) mma_commit_2sm(R.sfull + slot);
        mma_commit_2sm(R.empty + s);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int hw = W / 2;
    float acc[kMaxHalf];
#pragma unroll
    for (int j = 0; j < kMaxHalf; ++j) acc[j] = 0.f;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * hw);
    const uint32_t sempty_leader = mapa_u32(R.sempty, 0);
    for (int t = 0; t < ngroups; ++t) {
      const int slot = t % ns;
      mbar_wait(R.sfull + slot, (uint32_t)(t / ns) & 1u);
      tc_fence_after();
      const uint32_t src = lane_base + (uint32_t)(slot * c0w);
#pragma unroll
      for (int j0 = 0; j0 < kMaxHalf; j0 += 16) {
        if (j0 < hw) {
          float v[16];
          tmem_ld16(src + (uint32_t)j0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[j0 + i] += v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(sempty_leader + (uint32_t)slot * 8u);
    }
    const int idx = m0 + q * 32 + lane;
    if (idx < M) {
      double* dst = out + (int64_t)idx * ldo + col0 + h * hw;
#pragma unroll
      for (int j = 0; j < kMaxHalf; j += 2)
        if (j < hw) *reinterpret_cast<double2*>(dst + j) = make_double2(acc[j], acc[j + 1]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// out[j][i] = sum_s ws[s][j][i] in split order (deterministic).
__global__ void k_sum_splits(const double* __restrict__ ws, int S, int64_t stride, int N, int M,
                             int64_t ldw, double* __restrict__ out, int64_t ldo) {
  const int64_t total = (int64_t)N * M;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / M), i = (int)(idx % M);
    const double* p = ws + (int64_t)j * ldw + i;
    double s = 0.0;
    for (int t = 0; t < S; ++t) s += p[(int64_t)t * stride];
    out[(int64_t)j * ldo + i] = s;
  }
}

// lo = tf32(g - hi(g)), hi(g) = g as the tensor core reads it (mode 0: the
// low 13 mantissa bits dropped; mode 1: rounded to nearest); per-block fp64
// partial sums of g^2 (exact squares) for ||G||_F^2.
constexpr int kSplitBlocks = kSMs * 8;
__global__ void __launch_bounds__(256) k_split_f32(const float* __restrict__ g, int64_t ldg,
                                                   int64_t rows, int cols,
                                                   float* __restrict__ lo, int64_t ldl, int mode,
                                                   double* __restrict__ partial) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  const bool vec = ((cols & 3) == 0) && ((ldg & 3) == 0) && ((ldl & 3) == 0);
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < rows; r += (int64_t)gridDim.x * 8) {
    const float* src = g + r * ldg;
    float* dst = lo + r * ldl;
    if (vec) {
      // 4 independent 16-byte loads in flight per lane (HBM-bound pass)
      for (int c0 = lane * 4; c0 < cols; c0 += 512) {
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * 128;
          x[u] = c < cols ? __ldcs(reinterpret_cast<const float4*>(src + c))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * 128;
          float e[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
          double sq = 0.0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float h =
                mode ? tf32_rna(e[t]) : __uint_as_float(__float_as_uint(e[t]) & 0xFFFFE000u);
            sq = fma((double)e[t], (double)e[t], sq);
            e[t] = tf32_rna(e[t] - h);
          }
          acc += sq;
          if (c < cols)
            __stcs(reinterpret_cast<float4*>(dst + c), make_float4(e[0], e[1], e[2], e[3]));
        }
      }
    } else {
      for (int c = lane; c < cols; c += 32) {
        const float x = src[c];
        const float h = mode ? tf32_rna(x) : __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        acc = fma((double)x, (double)x, acc);
        dst[c] = tf32_rna(x - h);
      }
    }
  }
  __shared__ double red[8];
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

__global__ void k_sum_partials(const double* __restrict__ partial, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// hi = tf32(x), lo = tf32(x - hi) of an fp64 matrix, zero in columns
// [cols, cols_out) (padding read by the MMAs). One warp per row (grid-stride
// over rows), lanes over columns: no per-element division, coalesced.
__global__ void __launch_bounds__(256) k_split_f64(const double* __restrict__ x, int64_t ldx,
                                                   int64_t rows, int cols,
                                                   float* __restrict__ hi,
                                                   float* __restrict__ lo, int64_t ldo,
                                                   int cols_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < rows; r += (int64_t)gridDim.x * 8) {
    const double* src = x + r * ldx;
    float* ph = hi + r * ldo;
    float* pl = lo + r * ldo;
    for (int c = lane; c < cols_out; c += 32) {
      const double v = c < cols ? __ldcs(src + c) : 0.0;
      const float h = tf32_rna((float)v);
      ph[c] = h;
      pl[c] = tf32_rna((float)(v - (double)h));
    }
  }
}

// Output chunks: one MMA of N (<= 160) or two of multiples of 32.
int first_chunk(int N) {
  if (N <= kMaxChunk) return N;
  return (N / 2 + 31) / 32 * 32;
}

// Tuned on B200 at cfg4 shapes (tools/tf32_sweep.py, m = 1e6, n = 8192, N = 288):
// gx / gtq at BK 16, flush 1: 126 / 108 TFLOP/s; BK 32, flush 2: 160 / 159.
// A flush every 2 K-blocks keeps 64 K-steps (24 MMAs) in the truncating TMEM
// accumulator: relative error ~5e-7, the level of an fp32 SGEMM.
int g_bk_gx = 32;   // K-block (16: 64B swizzle rows, 32: 128B) of the gx kernel
int g_bk_gtq = 32;  // K-block (rows) of the gtq kernel
int g_rows_per_split = 8192;
int g_flush = 2;    // K-blocks accumulated in TMEM before an fp32 register flush
// L2 prefetch distance of the G tiles in K-blocks (0: off). Measured at cfg4
// (tools/tf32_sweep.py): gx 174 / 167 / 160 / 162 TFLOP/s at 0 / 2 / 4 / 8, so
// HBM latency is not the limiter; off by default (RGSV_TF32_PREFETCH).
int g_prefetch = 0;

template <int MODE, int BK>
int launch_bk(const CUtensorMap& tg, const CUtensorMap& tgl, const CUtensorMap& tbh,
              const CUtensorMap& tbl, uint32_t stage, dim3 grid, double* out, int64_t ldo,
              int64_t split_stride, int M, int N, int K, int rows_per, cudaStream_t st) {
  int stages = (int)((kSmemMax - kSmemReserve) / stage);
  if (stages > 8) stages = 8;
  if (stages < 2) return RGSV_ERR_DIMENSION;
  const uint32_t smem = (uint32_t)stages * stage + kSmemReserve;
  auto kern = k_tf32x3<MODE, BK>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return RGSV_ERR_CUDA;
  kern<<<grid, kThreads, smem, st>>>(tg, tgl, tbh, tbl, out, ldo, split_stride, M, N, K, rows_per,
                                     first_chunk(N), stages, g_flush, g_prefetch);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

template <int BK>
int launch_gx_bk(const float* g, const float* glo, int64_t ldg, const float* xh, const float* xl,
                 int64_t ldx, double* y, int64_t ldy, int M, int N, int K, cudaStream_t st) {
  constexpr int SW = BK * 4;
  const int c0w = first_chunk(N);
  CUtensorMap tg, tgl, txh, txl;
  if (make_tmap_2d_swz(&tg, g, K, M, ldg, BK, kTileM, 4, SW) ||
      make_tmap_2d_swz(&tgl, glo, K, M, ldg, BK, kTileM, 4, SW) ||
      make_tmap_2d_swz(&txh, xh, K, N, ldx, BK, c0w, 4, SW) ||
      make_tmap_2d_swz(&txl, xl, K, N, ldx, BK, c0w, 4, SW))
    return RGSV_ERR_CUDA;
  const uint32_t stage = 2u * kTileM * SW + 2u * (uint32_t)c0w * SW;
  const int tiles = (M + kTileM - 1) / kTileM * (N > c0w ? 2 : 1);
  return launch_bk<kGX, BK>(tg, tgl, txh, txl, stage, dim3(tiles), y, ldy, 0, M, N, K, K, st);
}

// 2-SM launch of gx (RGSV_TF32_2SM=1; needs N chunks whose halves are
// multiples of 8 rows).
template <int BK>
int launch_gx2_bk(const float* g, const float* glo, int64_t ldg, const float* xh,
                  const float* xl, int64_t ldx, double* y, int64_t ldy, int M, int N, int K,
                  cudaStream_t st) {
  constexpr int SW = BK * 4;
  const int c0w = first_chunk(N);
  if ((c0w / 2) % 8 || ((N - c0w) > 0 && ((N - c0w) / 2) % 8)) return RGSV_ERR_DIMENSION;
  CUtensorMap tg, tgl, txh, txl;
  if (make_tmap_2d_swz(&tg, g, K, M, ldg, BK, kTileM, 4, SW) ||
      make_tmap_2d_swz(&tgl, glo, K, M, ldg, BK, kTileM, 4, SW) ||
      make_tmap_2d_swz(&txh, xh, K, N, ldx, BK, c0w / 2, 4, SW) ||
      make_tmap_2d_swz(&txl, xl, K, N, ldx, BK, c0w / 2, 4, SW))
    return RGSV_ERR_CUDA;
  const uint32_t stage = 2u * kTileM * SW + 2u * (uint32_t)(c0w / 2) * SW;
  int stages = (int)((kSmemMax - kSmemReserve) / stage);
  if (stages > 8) stages = 8;
  if (stages < 2) return RGSV_ERR_DIMENSION;
  const uint32_t smem = (uint32_t)stages * stage + kSmemReserve;
  auto kern = k_tf32x3_gx2<BK>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return RGSV_ERR_CUDA;
  const int pairs = (M + 2 * kTileM - 1) / (2 * kTileM) * (N > c0w ? 2 : 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, tg, tgl, txh, txl, y, ldy, M, N, K, c0w, stages, g_flush) !=
      cudaSuccess)
    return RGSV_ERR_CUDA;
  note_launch();
  return 0;
}

template <int BK>
int launch_gtq_bk(const float* q, const float* ql, int64_t ldq, const float* g, const float* glo,
                  int64_t ldg, double* c, int64_t ldc, int N, int M, int K, void* scratch,
                  size_t scratch_bytes, cudaStream_t st) {
  CUtensorMap tg, tgl, tqh, tql;
  if (make_tmap_2d_swz(&tg, g, M, K, ldg, 32, BK, 4, -128) ||
      make_tmap_2d_swz(&tgl, glo, M, K, ldg, 32, BK, 4, -128) ||
      make_tmap_2d_swz(&tqh, q, N, K, ldq, 32, BK, 4, -128) ||
      make_tmap_2d_swz(&tql, ql, N, K, ldq, 32, BK, 4, -128))
    return RGSV_ERR_CUDA;
  const uint32_t box = BK * 128;
  const int c0w = first_chunk(N);
  const uint32_t stage = 2u * 4u * box + 2u * (uint32_t)(c0w / 32) * box;
  const int tiles = (M + kTileM - 1) / kTileM * (N > c0w ? 2 : 1);
  int rows_per = (g_rows_per_split + BK - 1) / BK * BK;
  int S = (K + rows_per - 1) / rows_per;
  // few column tiles and a short reduction: split finer to fill the machine
  while (S > 1 && rows_per > 4 * BK && (int64_t)tiles * S < kSMs) {
    rows_per = (rows_per / 2 + BK - 1) / BK * BK;
    S = (K + rows_per - 1) / rows_per;
  }
  if (S > 65535) return RGSV_ERR_DIMENSION;
  double* dst = c;
  int64_t ldd = ldc, stride = 0;
  if (S > 1) {
    const int64_t ldw = ((int64_t)M + 3) / 4 * 4;
    stride = (int64_t)N * ldw;
    if ((size_t)S * stride * sizeof(double) > scratch_bytes) return RGSV_ERR_WORKSPACE;
    dst = static_cast<double*>(scratch);
    ldd = ldw;
  }
  int rc = launch_bk<kGTQ, BK>(tg, tgl, tqh, tql, stage, dim3(tiles, S), dst, ldd, stride, M, N,
                               K, rows_per, st);
  if (rc) return rc;
  if (S > 1) {
    k_sum_splits<<<kSMs * 8, 256, 0, st>>>(dst, S, stride, N, M, ldd, c, ldc);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace rgsv

using namespace rgsv;

extern "C" {

int rgsv_tf32_config(int bk_gx, int bk_gtq, int rows_per_split, int flush) {
  if (flush >= 1) g_flush = flush;
  if (const char* e = getenv("RGSV_TF32_PREFETCH")) g_prefetch = atoi(e);
  if (bk_gx == 16 || bk_gx == 32) g_bk_gx = bk_gx;
  if (bk_gtq == 8 || bk_gtq == 16 || bk_gtq == 32) g_bk_gtq = bk_gtq;
  if (rows_per_split >= 64) g_rows_per_split = rows_per_split;
  return 0;
}

int rgsv_f32_split(const float* g, int64_t ldg, int64_t rows, int64_t cols, float* lo,
                   int64_t ldl, int mode, double* sumsq_out, void* ws, size_t ws_bytes,
                   void* stream) {
  if (rows < 0 || cols < 0 || cols > 0x7fffffff || ldg < cols || ldl < cols)
    return RGSV_ERR_DIMENSION;
  if (ws_bytes < kSplitBlocks * sizeof(double)) return RGSV_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(ws);
  k_split_f32<<<kSplitBlocks, 256, 0, st>>>(g, ldg, rows, (int)cols, lo, ldl, mode, part);
  note_launch();
  if (sumsq_out) {
    k_sum_partials<<<1, 1024, 0, st>>>(part, kSplitBlocks, sumsq_out);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int rgsv_f64_split_tf32(const double* x, int64_t ldx, int64_t rows, int64_t cols, float* hi,
                        float* lo, int64_t ldo, int64_t cols_out, void* stream) {
  if (rows < 0 || cols < 0 || cols_out < cols || ldo < cols_out || ldx < cols)
    return RGSV_ERR_DIMENSION;
  if (rows == 0 || cols_out == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int blocks = (int)((rows + 7) / 8);
  if (blocks > kSMs * 16) blocks = kSMs * 16;
  k_split_f64<<<blocks, 256, 0, st>>>(x, ldx, rows, (int)cols, hi, lo, ldo, (int)cols_out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

int rgsv_tf32x3_gx(const float* g, const float* glo, int64_t ldg, const float* xhi,
                   const float* xlo, int64_t ldx, double* y, int64_t ldy, int64_t M, int64_t N,
                   int64_t K, void* stream) {
  if (M < 0 || K < 1 || N < 32 || N > 2 * kMaxChunk || (N % 32) || ldg < K || ldx < K || ldy < N ||
      (ldg & 3) || (ldx & 3) || (ldy & 1) || M > 0x7fffffff || K > 0x7fffffff)
    return RGSV_ERR_DIMENSION;
  if (!aligned16(g) || !aligned16(glo) || !aligned16(xhi) || !aligned16(xlo) || !aligned16(y))
    return RGSV_ERR_DIMENSION;
  if (M == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // opt-in 2-SM variant (measured 161 vs 169 TFLOP/s for the 1-SM kernel at
  // cfg4, tools/tf32_sweep.py), read per call so tests can exercise both
  const char* e2 = getenv("RGSV_TF32_2SM");
  if (e2 && atoi(e2) == 1 && g_bk_gx == 32)
    return launch_gx2_bk<32>(g, glo, ldg, xhi, xlo, ldx, y, ldy, (int)M, (int)N, (int)K, st);
  if (g_bk_gx == 32)
    return launch_gx_bk<32>(g, glo, ldg, xhi, xlo, ldx, y, ldy, (int)M, (int)N, (int)K, st);
  return launch_gx_bk<16>(g, glo, ldg, xhi, xlo, ldx, y, ldy, (int)M, (int)N, (int)K, st);
}

int rgsv_tf32x3_gtq(const float* qhi, const float* qlo, int64_t ldq, const float* g,
                    const float* glo, int64_t ldg, double* c, int64_t ldc, int64_t N, int64_t M,
                    int64_t K, void* scratch, size_t scratch_bytes, void* stream) {
  if (M < 1 || K < 1 || N < 32 || N > 2 * kMaxChunk || (N % 32) || ldq < N || ldg < M || ldc < M ||
      (ldg & 3) || (ldq & 3) || M > 0x7fffffff || K > 0x7fffffff)
    return RGSV_ERR_DIMENSION;
  if (!aligned16(g) || !aligned16(glo) || !aligned16(qhi) || !aligned16(qlo))
    return RGSV_ERR_DIMENSION;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (g_bk_gtq == 32)
    return launch_gtq_bk<32>(qhi, qlo, ldq, g, glo, ldg, c, ldc, (int)N, (int)M, (int)K, scratch,
                             scratch_bytes, st);
  if (g_bk_gtq == 8)
    return launch_gtq_bk<8>(qhi, qlo, ldq, g, glo, ldg, c, ldc, (int)N, (int)M, (int)K, scratch,
                            scratch_bytes, st);
  return launch_gtq_bk<16>(qhi, qlo, ldq, g, glo, ldg, c, ldc, (int)N, (int)M, (int)K, scratch,
                           scratch_bytes, st);
}

}  // extern "C"
