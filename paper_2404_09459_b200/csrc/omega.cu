// Device generation of the reference's Gaussian test matrices (SURVEY.md
// §2b K12), bit-identical to numpy 2.3.5:
//   rng = np.random.default_rng(seed & (2^64-1)); rng.standard_normal((n, k))
// (rangefinder.py:101,112; engine.py:252-253 for seed + 1).
//
// numpy: SeedSequence(seed) -> 4 x uint64 -> PCG64 (128-bit LCG, XSL-RR
// output); standard_normal = 256-layer ziggurat consuming a VARIABLE number
// of raw draws per normal (1 on the fast path, more on the slow/tail path).
// Parallel reproduction of that sequential stream, per generator stream:
//  k_zig_attempt : every raw position p (128-bit LCG jump-ahead per thread)
//                  evaluates the attempt that would START at p: accepted?,
//                  value, raw draws consumed. Fast attempts (~99%) consume 1.
//  k_zig_walk_*  : the attempt chain, visiting only the rare "special"
//                  positions (tile-compacted lists): every tile walked in
//                  parallel from carry-in 0, then a per-stream carry pass
//                  re-walks the rare tiles entered mid-attempt; marks
//                  positions swallowed by multi-draw attempts and counts
//                  emitted normals per tile.
//  k_zig_scatter : per tile, emitted flags -> prefix -> output index; writes
//                  Omega^T (kp x ld) directly in the layout the sketch GEMM
//                  consumes (value #e of the stream is Omega[e / k][e % k]).
#include <math.h>

#include "common.cuh"
#include "rgsv_internal.h"
#include "ziggurat_tables.h"

namespace rgsv {

typedef unsigned __int128 u128;

constexpr int kZigTile = 1024;      // positions per tile
constexpr int kZigThreads = 128;    // threads per tile (8 positions each)
constexpr int kZigPerThread = kZigTile / kZigThreads;
constexpr u128 kPcgMult = ((u128)2549297995355413924ull << 64) | 4865540595714422341ull;

// ---- SeedSequence(seed).generate_state(4, uint64) (numpy bit_generator.pyx)
RGSV_DI uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}
RGSV_DI uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}
RGSV_DI void pcg64_seed(uint64_t seed, u128& state, u128& inc) {
  uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const int nent = (seed >> 32) ? 2 : 1;  // _coerce_to_uint32_array: little-endian words
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < nent ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  uint32_t hb = 0x8b51f9ddu, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  const uint64_t s0 = w[0] | ((uint64_t)w[1] << 32), s1 = w[2] | ((uint64_t)w[3] << 32);
  const uint64_t s2 = w[4] | ((uint64_t)w[5] << 32), s3 = w[6] | ((uint64_t)w[7] << 32);
  const u128 initstate = ((u128)s0 << 64) | s1, initseq = ((u128)s2 << 64) | s3;
  inc = (initseq << 1) | 1;
  state = inc;  // 0 * M + inc
  state += initstate;
  state = state * kPcgMult + inc;
}

// state after `steps` more LCG steps (binary-exponentiated affine map)
RGSV_DI u128 pcg64_advance(u128 state, u128 inc, uint64_t steps) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kPcgMult, cur_plus = inc;
  while (steps) {
    if (steps & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    steps >>= 1;
  }
  return acc_mult * state + acc_plus;
}

RGSV_DI uint64_t pcg64_out(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

RGSV_DI double raw_to_double(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

// log1p exactly as the host libm numpy calls computes it: glibc 2.39's
// fdlibm-derived __log1p, in its FMA build (the x86-64 ifunc variant picked
// on FMA-capable CPUs). GCC fuses a multiply into an add/sub only within one
// basic block, in statement order; those fusions are reproduced with __fma_rn
// and every other operation is rounded separately (__d*_rn, no contraction).
// Verified against libm on >3e5 inputs of the ziggurat tail domain by
// tools/log1p_check.py. Valid for -1 < x (the only domain used here).
RGSV_DI double log1p_glibc(double x) {
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  constexpr double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                   Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                   Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                   Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (k != 0) {
    double u = __dadd_rn(1.0, x);
    hu = __double2hiint(u);
    k = (hu >> 20) - 1023;
    c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
    c = __ddiv_rn(c, u);
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = __fma_rn(dk, ln2_lo, c);
      return __fma_rn(dk, ln2_hi, c);
    }
    const double R = __dmul_rn(hfsq, __fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z);
  const double R2 = __fma_rn(z, Lp3, Lp2);
  const double z4 = __dmul_rn(z2, z2);
  const double R3 = __fma_rn(z, Lp5, Lp4);
  const double z6 = __dmul_rn(z4, z2);
  const double R4 = __fma_rn(z, Lp7, Lp6);
  const double R = __fma_rn(z6, R4, __fma_rn(z4, R3, __fma_rn(z, Lp1, __dmul_rn(z2, R2))));
  const double t = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  const double t2 = __dadd_rn(t, __fma_rn(dk, ln2_lo, c));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, t2), f));
}

struct ZigStream {
  u128 state0;  // state before raw draw 0
  u128 inc;
};

// Per-position attempt record: consumed draws (1..), accepted flag.
// code = consumed | (accepted << 15); value stored separately.
__global__ void k_zig_seed(const uint64_t* __restrict__ seeds, int nstreams,
                           ZigStream* __restrict__ streams) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nstreams) return;
  u128 st, inc;
  pcg64_seed(seeds[s], st, inc);
  streams[s].state0 = st;
  streams[s].inc = inc;
}

__global__ void __launch_bounds__(kZigThreads) k_zig_attempt(
    const ZigStream* __restrict__ streams, int64_t P, double* __restrict__ val,
    uint16_t* __restrict__ code, int* __restrict__ tile_nspec, uint32_t* __restrict__ tile_spec) {
  const int s = blockIdx.y;
  const int64_t tile = blockIdx.x;
  const int64_t p0 = tile * kZigTile + threadIdx.x * kZigPerThread;
  const ZigStream zs = streams[s];
  double* vs = val + (int64_t)s * P;
  uint16_t* cs = code + (int64_t)s * P;
  // state after p0 + 1 steps produces raw draw p0
  u128 st = pcg64_advance(zs.state0, zs.inc, (uint64_t)p0 + 1);
  uint32_t specmask = 0;
  uint64_t raw_next = pcg64_out(st);
#pragma unroll 1
  for (int q = 0; q < kZigPerThread; ++q) {
    const int64_t p = p0 + q;
    const uint64_t r0 = raw_next;
    st = st * kPcgMult + zs.inc;  // state producing raw p + 1
    raw_next = pcg64_out(st);
    if (p >= P) continue;
    uint64_t r = r0;
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * kZigWi[idx];
    if (sign) x = -x;
    int consumed = 1, acc = 1;
    if (rabs >= kZigKi[idx]) {
      specmask |= 1u << q;
      u128 st2 = st;  // produces raw p + 1
      uint64_t rn = raw_next;
      if (idx == 0) {
        for (;;) {
          const double xx = __dmul_rn(-kZigInvR, log1p_glibc(-raw_to_double(rn)));
          st2 = st2 * kPcgMult + zs.inc;
          rn = pcg64_out(st2);
          const double yy = -log1p_glibc(-raw_to_double(rn));
          st2 = st2 * kPcgMult + zs.inc;
          rn = pcg64_out(st2);
          consumed += 2;
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
            x = ((rabs >> 8) & 1) ? -__dadd_rn(kZigR, xx) : __dadd_rn(kZigR, xx);
            break;
          }
        }
      } else {
        const double u = raw_to_double(rn);
        consumed = 2;
        // numpy's distributions.c is built without FMA: keep separate roundings
        acc = __dadd_rn(__dmul_rn(__dsub_rn(kZigFi[idx - 1], kZigFi[idx]), u), kZigFi[idx]) <
              exp(__dmul_rn(__dmul_rn(-0.5, x), x));
      }
    }
    vs[p] = x;
    cs[p] = (uint16_t)(consumed | (acc << 15));
  }
  // tile-compacted, ordered list of special offsets
  __shared__ int wcount[kZigThreads / 32];
  const int cnt = __popc(specmask);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wcount[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wcount[w];
  int pos = base + incl - cnt;
  uint32_t* ts = tile_spec + ((int64_t)s * gridDim.x + tile) * kZigTile;
  for (int q = 0; q < kZigPerThread; ++q)
    if (specmask & (1u << q)) {
      const int64_t pp = p0 + q;
      const uint32_t c = pp < P ? cs[pp] : 1u;
      ts[pos++] = (uint32_t)(threadIdx.x * kZigPerThread + q) | ((c & 0x3fffu) << 10) |
                  ((c & 0x8000u) << 16);
    }
  if (threadIdx.x == kZigThreads - 1) {
    int tot = 0;
    for (int w = 0; w < kZigThreads / 32; ++w) tot += wcount[w];
    tile_nspec[(int64_t)s * gridDim.x + tile] = tot;
  }
}

// The attempt chain through the specials is sequential only through its
// carry: how far the last attempt of tile t reaches into tile t+1 (almost
// always 0 -- a multi-draw attempt must start in the last few positions).
// So every tile is walked in parallel assuming carry-in 0 (k_zig_walk_tiles,
// one warp per (tile, stream)), and one warp per stream then runs the carry
// chain over the per-tile carry-outs, re-walking only the rare tiles whose
// actual carry-in is not 0 (k_zig_walk_fix). The result is identical to one
// sequential walk. Positions that emit nothing -- rejected starts and draws
// swallowed by multi-draw attempts -- are recorded per tile as half-open
// intervals [a, b) of tile offsets; the per-tile emit count is the tile
// length minus their total length.
constexpr int kZigMaxIv = 64;  // intervals per tile (overflow -> status bit)

// Walk tile t of stream s from carry-in `cin` (positions t0 .. t0+cin-1 are
// swallowed by the previous tile's attempt). Single thread; records in rec.
// Writes the tile's interval list / emit count; returns the carry-out.
RGSV_DI int64_t zig_walk_tile(const uint32_t* rec, int nsp, int64_t t0, int64_t t1, int64_t cin,
                              uint32_t* iv_out, int* niv_out, int* emit_out, bool* overflow) {
  int niv = 0, removed = 0;
  int64_t covered = t0 + cin;
  auto add = [&](int64_t a, int64_t b) {  // clip to this tile
    if (a < t0) a = t0;
    if (b > t1) b = t1;
    if (b <= a) return;
    const uint32_t ia = (uint32_t)(a - t0), ib = (uint32_t)(b - t0);
    if (niv < kZigMaxIv) {
      iv_out[niv++] = (ia << 16) | ib;
    } else {
      *overflow = true;
    }
    removed += (int)(ib - ia);
  };
  if (cin > 0) add(t0, covered);
  for (int i = 0; i < nsp; ++i) {
    const uint32_t r = rec[i];
    const int64_t p = t0 + (r & 1023u);
    if (p < covered) continue;  // swallowed: not an attempt start
    const int consumed = (int)((r >> 10) & 0x3fffu);
    const bool acc = (r >> 31) & 1u;
    add(acc ? p + 1 : p, p + consumed);
    covered = p + consumed;
  }
  *niv_out = niv;
  *emit_out = (int)(t1 - t0) - removed;
  return covered > t1 ? covered - t1 : 0;
}

__global__ void __launch_bounds__(32) k_zig_walk_tiles(int ntiles, int64_t P,
                                                       const int* __restrict__ tile_nspec,
                                                       const uint32_t* __restrict__ tile_spec,
                                                       int* __restrict__ tile_emit,
                                                       int* __restrict__ tile_niv,
                                                       uint32_t* __restrict__ tile_iv,
                                                       int* __restrict__ tile_cout) {
  const int t = blockIdx.x, s = blockIdx.y, lane = threadIdx.x;
  __shared__ uint32_t rec[kZigTile];
  const int64_t id = (int64_t)s * ntiles + t;
  const int nsp = tile_nspec[id];
  const uint32_t* ts = tile_spec + id * kZigTile;
  for (int i = lane; i < nsp; i += 32) rec[i] = ts[i];
  __syncwarp();
  if (lane == 0) {
    const int64_t t0 = (int64_t)t * kZigTile;
    const int64_t t1 = t0 + kZigTile < P ? t0 + kZigTile : P;
    int niv, emit;
    bool overflow = false;
    const int64_t cout = zig_walk_tile(rec, nsp, t0, t1, 0, tile_iv + id * kZigMaxIv, &niv, &emit,
                                       &overflow);
    tile_niv[id] = overflow ? -1 : niv;
    tile_emit[id] = emit;
    tile_cout[id] = (int)cout;
  }
}

__global__ void __launch_bounds__(32) k_zig_walk_fix(int ntiles, int64_t P, int64_t nvals,
                                                     const int* __restrict__ tile_nspec,
                                                     const uint32_t* __restrict__ tile_spec,
                                                     int* __restrict__ tile_emit,
                                                     int* __restrict__ tile_niv,
                                                     uint32_t* __restrict__ tile_iv,
                                                     const int* __restrict__ tile_cout,
                                                     int* __restrict__ status) {
  const int s = blockIdx.x, lane = threadIdx.x;
  __shared__ uint32_t rec[kZigTile];
  __shared__ int sh_cin;
  int64_t cin = 0, total = 0;
  bool overflow = false;
  for (int t = 0; t < ntiles; ++t) {
    const int64_t id = (int64_t)s * ntiles + t;
    if (cin > 0) {  // rare: re-walk this tile from its true carry-in
      const int nsp = tile_nspec[id];
      const uint32_t* ts = tile_spec + id * kZigTile;
      for (int i = lane; i < nsp; i += 32) rec[i] = ts[i];
      __syncwarp();
      if (lane == 0) {
        const int64_t t0 = (int64_t)t * kZigTile;
        const int64_t t1 = t0 + kZigTile < P ? t0 + kZigTile : P;
        int niv, emit;
        sh_cin = (int)zig_walk_tile(rec, nsp, t0, t1, cin, tile_iv + id * kZigMaxIv, &niv, &emit,
                                    &overflow);
        tile_niv[id] = niv;
        tile_emit[id] = emit;
      }
      __syncwarp();
      cin = sh_cin;
    } else {
      cin = tile_cout[id];
      if (tile_niv[id] < 0) overflow = true;
    }
    total += tile_emit[id];
  }
  if (lane == 0 && (total < nvals || overflow)) atomicOr(status, RGSV_ST_OMEGA_SHORT);
}

// Per tile: exclusive prefix of emit flags -> output element index e; value
// goes to Omega^T[e % k][e / k] (ld ldo) of stream s.
__global__ void __launch_bounds__(kZigThreads) k_zig_scatter(
    int64_t P, const double* __restrict__ val, const int* __restrict__ tile_emit,
    const int* __restrict__ tile_niv, const uint32_t* __restrict__ tile_iv, int64_t nvals, int k,
    double* __restrict__ out, int64_t ldo, int64_t out_stride, int64_t offset) {
  const int s = blockIdx.y;
  const int tile = blockIdx.x;
  const int ntiles = gridDim.x;
  __shared__ int64_t tbase;
  __shared__ int wcount[kZigThreads / 32];
  if (threadIdx.x == 0) {
    int64_t b = 0;
    const int* te = tile_emit + (int64_t)s * ntiles;
    for (int t = 0; t < tile; ++t) b += te[t];
    tbase = b;
  }
  __shared__ uint32_t iv[kZigMaxIv];
  __shared__ int niv;
  if (threadIdx.x == 0) niv = tile_niv[(int64_t)s * ntiles + tile];
  __syncthreads();
  for (int i = threadIdx.x; i < niv; i += blockDim.x)
    iv[i] = tile_iv[((int64_t)s * ntiles + tile) * kZigMaxIv + i];
  __syncthreads();
  const int64_t p0 = (int64_t)tile * kZigTile + threadIdx.x * kZigPerThread;
  const double* vs = val + (int64_t)s * P;
  uint32_t emask = 0;
  for (int q = 0; q < kZigPerThread; ++q) {
    const int64_t p = p0 + q;
    if (p < P) {
      const uint32_t off = (uint32_t)(threadIdx.x * kZigPerThread + q);
      bool keep = true;
      for (int i = 0; i < niv; ++i) keep &= !(off >= (iv[i] >> 16) && off < (iv[i] & 0xffffu));
      if (keep) emask |= 1u << q;
    }
  }
  const int cnt = __popc(emask);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wcount[warp] = incl;
  __syncthreads();
  int64_t e = tbase;
  for (int w = 0; w < warp; ++w) e += wcount[w];
  e += incl - cnt;
  double* o = out + (int64_t)s * out_stride;
  for (int q = 0; q < kZigPerThread; ++q) {
    if (emask & (1u << q)) {
      const int64_t f = e - offset;  // index within the requested block
      if (f >= 0 && f < nvals) o[(f % k) * ldo + f / k] = vs[p0 + q];
      ++e;
    }
  }
}

size_t omega_workspace_bytes(int nstreams, int64_t nvals) {
  // nvals counts every normal drawn, including a skipped prefix (offset)
  const int64_t P = nvals + nvals / 16 + 2 * kZigTile;
  const int64_t ntiles = (P + kZigTile - 1) / kZigTile;
  size_t b = 0;
  b += (size_t)nstreams * sizeof(ZigStream) + 256;
  b += (size_t)nstreams * P * sizeof(double) + 256;
  b += (size_t)nstreams * P * sizeof(uint16_t) + 256;
  b += (size_t)nstreams * ntiles * sizeof(int) * 4 + 1024;
  b += (size_t)nstreams * ntiles * kZigTile * sizeof(uint32_t) + 256;
  b += (size_t)nstreams * ntiles * kZigMaxIv * sizeof(uint32_t) + 256;
  return b;
}

// Generate `nstreams` Omega^T blocks (k rows x n cols, ld ldo, stride
// out_stride between streams) from seeds[] (device array) on stream st.
int omega_generate(const uint64_t* seeds, int nstreams, int64_t n, int k, double* out,
                   int64_t ldo, int64_t out_stride, int* status, void* ws, size_t ws_bytes,
                   cudaStream_t st, int64_t offset) {
  const int64_t nvals = n * (int64_t)k;
  const int64_t nall = offset + nvals;  // the stream prefix is walked, then skipped
  const int64_t P = nall + nall / 16 + 2 * kZigTile;
  const int ntiles = (int)((P + kZigTile - 1) / kZigTile);
  if (ws_bytes < omega_workspace_bytes(nstreams, nall)) return RGSV_ERR_WORKSPACE;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  ZigStream* streams = reinterpret_cast<ZigStream*>(take((size_t)nstreams * sizeof(ZigStream)));
  double* val = reinterpret_cast<double*>(take((size_t)nstreams * P * sizeof(double)));
  uint16_t* code = reinterpret_cast<uint16_t*>(take((size_t)nstreams * P * sizeof(uint16_t)));
  int* tnspec = reinterpret_cast<int*>(take((size_t)nstreams * ntiles * sizeof(int)));
  int* temit = reinterpret_cast<int*>(take((size_t)nstreams * ntiles * sizeof(int)));
  int* tniv = reinterpret_cast<int*>(take((size_t)nstreams * ntiles * sizeof(int)));
  int* tcout = reinterpret_cast<int*>(take((size_t)nstreams * ntiles * sizeof(int)));
  uint32_t* tspec =
      reinterpret_cast<uint32_t*>(take((size_t)nstreams * ntiles * kZigTile * sizeof(uint32_t)));
  uint32_t* tiv =
      reinterpret_cast<uint32_t*>(take((size_t)nstreams * ntiles * kZigMaxIv * sizeof(uint32_t)));
  k_zig_seed<<<(nstreams + 127) / 128, 128, 0, st>>>(seeds, nstreams, streams);
  note_launch();
  dim3 grid(ntiles, nstreams);
  k_zig_attempt<<<grid, kZigThreads, 0, st>>>(streams, P, val, code, tnspec, tspec);
  note_launch();
  k_zig_walk_tiles<<<grid, 32, 0, st>>>(ntiles, P, tnspec, tspec, temit, tniv, tiv, tcout);
  note_launch();
  k_zig_walk_fix<<<nstreams, 32, 0, st>>>(ntiles, P, nall, tnspec, tspec, temit, tniv, tiv, tcout,
                                          status);
  note_launch();
  k_zig_scatter<<<grid, kZigThreads, 0, st>>>(P, val, temit, tniv, tiv, nvals, k, out, ldo,
                                              out_stride, offset);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

}  // namespace rgsv
