// Shared device/host helpers for the rGSVD sm_100a kernels.
//
// FP64 math runs on the FP64 tensor pipe through mma.sync.m8n8k4.f64
// (SASS DMMA.8x8x4): ptxas rejects tcgen05.mma .kind::f64 for sm_100a, and
// DMMA is the B200's FP64 tensor-core instruction (measured 37.0 TFLOP/s
// issue peak, profiles/r01_fp64_peak.log). Operand tiles are staged
// global->shared by TMA (cp.async.bulk.tensor, SASS UTMALDG) with 128-byte
// swizzle, and handed between a producer warp and the DMMA warps through
// mbarrier full/empty rings.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define RGSV_DI __device__ __forceinline__

namespace rgsv {

constexpr int kSMs = 148;

RGSV_DI uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// D = A(8x4, row) * B(4x8, col) + D, FP64. Fragments (PTX ISA m8n8k4 .f64):
//   a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
//   c = C[lane>>2][2*(lane&3) + {0,1}].
RGSV_DI void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

RGSV_DI void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
RGSV_DI void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
RGSV_DI void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
RGSV_DI void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RGSV_DI void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

RGSV_DI void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 2-D tile load; coordinates are (inner, outer) in elements. Out-of-bounds
// parts of the box are zero-filled and still count toward complete_tx.
RGSV_DI void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Byte offset of element (row, col) inside a 1024-byte-aligned TMA box whose
// rows are 128 bytes (16 doubles) written with CU_TENSOR_MAP_SWIZZLE_128B:
// the 16-byte chunk index is XORed with row % 8.
RGSV_DI uint32_t swz128_f64(int row, int col) {
  return static_cast<uint32_t>(row * 128 + ((((col >> 1) ^ (row & 7))) << 4) + ((col & 1) << 3));
}

RGSV_DI double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rgsv

// ----------------------------------------------------------------- host side
namespace rgsv {

// Count of kernel launches issued by this library (rgsv_launch_count()).
void note_launch(int n = 1);

// Encode a 2-D row-major FP64/FP32 tensor map (inner = contiguous dim) with a
// box of box_inner x box_outer elements and 128-byte swizzle.
int make_tmap_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer,
                 uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer, int elem_bytes);
// Same with an explicit swizzle span (128, 64, 32 or 0 bytes; -128 = 128-byte
// span with 32-byte atoms, the MN-major tf32 operand layout of tcgen05).
int make_tmap_2d_swz(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer, int elem_bytes,
                     int swizzle_bytes);

}  // namespace rgsv
