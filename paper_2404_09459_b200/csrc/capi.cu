// extern "C" boundary (include/rgsv_b200.h) and the native pipeline driver.
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {

// defined in small.cu
int launch_stack(double* s, int64_t lds, const double* b1, int64_t ld1, int l1, const double* b2,
                 int64_t ld2, int l2, int lp, int64_t n, cudaStream_t st);
int launch_copy_block(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols,
                      int transpose, cudaStream_t st);
int launch_jacobi(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1, double* v2,
                  int64_t ld2, int nv2, int len2, double* sv2, int* nsv2, int* status,
                  cudaStream_t st);
int launch_comparative(const double* sv1, const int* nsv, const double* sv2, int64_t n, double tol,
                       double* a, double* b, double* rho, double* theta, double* p1, double* p2,
                       double* scalars, int* counts, int* status, int mode, int r_given,
                       cudaStream_t st);
int launch_sumsq(const double* a, int64_t lda, int64_t rows, int64_t cols, double* out,
                 double* part, int max_parts, cudaStream_t st);
int launch_sum(const double* part, int n, double* out, cudaStream_t st);
size_t householder_small_smem(int l);
int launch_householder_tall(double* a, int64_t lda, int m, int w, double* q, int64_t ldq,
                            double* rdiag, double* tau, int comp_count, cudaStream_t st);
int launch_jacobi_vec(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                      double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj, int ascending,
                      int* nzero, int* status, cudaStream_t st);
int launch_scale_cols(double* a, int64_t lda, int rows, int cols, const double* d,
                      cudaStream_t st);
int launch_convert_f32(const float* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
                       int64_t ldd, cudaStream_t st);
int launch_axpy(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols,
                double alpha, cudaStream_t st);
int debug_householder_profile(const double* b1, int64_t ld1, int l1, const double* b2,
                              int64_t ld2, int l2, double* q, int64_t ldq, long long* prof,
                              cudaStream_t st);
int launch_householder_small(const double* b1, int64_t ld1, int l1, const double* b2, int64_t ld2,
                             int l2, double* q, int64_t ldq, double* gwork, cudaStream_t st);

static std::atomic<long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

int make_tmap_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer,
                 uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer, int elem_bytes) {
  return make_tmap_2d_swz(out, base, inner, outer, ld_elems, box_inner, box_outer, elem_bytes,
                          128);
}

int make_tmap_2d_swz(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer, int elem_bytes,
                     int swizzle_bytes) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return RGSV_ERR_CUDA;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld_elems * elem_bytes) & 15))
    return RGSV_ERR_DIMENSION;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == -128 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                  : swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                        : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : RGSV_ERR_CUDA;
}

static inline int64_t ceil16(int64_t x) { return (x + 15) / 16 * 16; }
// Split cap of the Z^T / B = Q^T G reductions (RGSV_PROJ_SPLIT; tuning).
static int proj_split() {
  static const int v = [] {
    const char* e = getenv("RGSV_PROJ_SPLIT");
    const int x = e ? atoi(e) : 0;
    return x >= 1 ? x : kSMs;
  }();
  return v;
}
// Split cap of the tail tiles of the G X passes (RGSV_GX_SPLIT; tuning).
// cfg1 with 8 concurrent pairs: 713 / 720 / 720 pairs/s at 32 / 4 / 1 and
// 2.30 / 2.35 / 2.41 ms single-pair latency.
static int gx_split() {
  static const int v = [] {
    const char* e = getenv("RGSV_GX_SPLIT");
    const int x = e ? atoi(e) : 0;
    return x >= 1 ? x : 4;
  }();
  return v;
}
constexpr int kIntermediatePasses = 3;  // see the note in rgsv_sketch_project
static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// Upper bound of split-K partial storage for the GEMMs of one pipeline.
static size_t split_scratch_bytes(int64_t m, int64_t n, int64_t kp) {
  const int64_t ldn = ceil16(n);
  size_t a = (size_t)kSMs * kp * kp;                 // tall Gram partials
  int64_t tiles = (n + 255) / 256;
  if (tiles < 1) tiles = 1;
  size_t b = (size_t)(kSMs / tiles + 1) * kp * ldn;  // gtq projection partials
  size_t c = (size_t)kSMs * 128 * kp;                // gx tail partials
  size_t d = (size_t)32 * kp * kp + (size_t)8 * kp * ldn;  // wide gram + wide TRSM
  size_t mx = a;
  if (b > mx) mx = b;
  if (c > mx) mx = c;
  if (d > mx) mx = d;
  (void)m;
  return mx * sizeof(double) + 4096;
}

struct SketchLayout {
  size_t y, z, z2, gram, linv, rinv, rdiag, ss, tmp, scratch, total, scratch_bytes;
};

static SketchLayout sketch_layout(int64_t m, int64_t n, int k) {
  const int64_t kp = ceil16(k), ldn = ceil16(n);
  SketchLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = al256(off + bytes);
    return o;
  };
  L.y = take((size_t)m * kp * 8);
  L.z = take((size_t)kp * ldn * 8);
  L.z2 = take((size_t)kp * ldn * 8);
  L.gram = take((size_t)kp * kp * 8);
  L.linv = take((size_t)kp * kp * 8 + (size_t)kp * (kp + 1) * 8);
  L.rinv = take((size_t)kp * kp * 8);
  L.rdiag = take((size_t)kp * 8);
  L.ss = take(4096 * 8);
  L.tmp = take(64 * 8);
  L.scratch_bytes = split_scratch_bytes(m, n, kp);
  L.scratch = take(L.scratch_bytes);
  L.total = off;
  return L;
}

}  // namespace rgsv

using namespace rgsv;

extern "C" {

long long rgsv_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* rgsv_version(void) { return "rgsv_b200 0.1.0 (sm_100a, FP64 DMMA + TMA)"; }

int rgsv_device_cc(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  int ma = 0, mi = 0;
  if (cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev);
  return ma * 10 + mi;
}

size_t rgsv_omega_workspace_bytes(int nstreams, int64_t n, int k) {
  return rgsv::omega_workspace_bytes(nstreams, n * (int64_t)k);
}

int rgsv_omega_generate(const uint64_t* seeds, int nstreams, int64_t n, int k, double* out,
                        int64_t ldo, int64_t out_stride, int* status, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (nstreams < 1 || n < 1 || k < 1 || ldo < n) return RGSV_ERR_DIMENSION;
  return rgsv::omega_generate(seeds, nstreams, n, k, out, ldo, out_stride, status, workspace,
                              workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

size_t rgsv_omega_workspace_bytes_at(int nstreams, int64_t n, int k, int64_t offset) {
  return rgsv::omega_workspace_bytes(nstreams, n * (int64_t)k + offset);
}

int rgsv_omega_generate_at(const uint64_t* seeds, int nstreams, int64_t n, int k, int64_t offset,
                           double* out, int64_t ldo, int64_t out_stride, int* status,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (nstreams < 1 || n < 1 || k < 1 || ldo < n || offset < 0) return RGSV_ERR_DIMENSION;
  return rgsv::omega_generate(seeds, nstreams, n, k, out, ldo, out_stride, status, workspace,
                              workspace_bytes, reinterpret_cast<cudaStream_t>(stream), offset);
}

int rgsv_householder_qr(double* a, int64_t lda, int m, int w, double* q, int64_t ldq,
                        double* rdiag, double* tau, void* stream) {
  return launch_householder_tall(a, lda, m, w, q, ldq, rdiag, tau, 0,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_orth_complete(double* a, int64_t lda, int dim, int have, int count, double* out,
                       int64_t ldo, double* rdiag, double* tau, void* stream) {
  if (count < 1 || have < 0 || have + count > dim) return RGSV_ERR_DIMENSION;
  return launch_householder_tall(a, lda, dim, have, out, ldo, rdiag, tau, count,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_svd_vectors(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                     double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj, int ascending,
                     int* nzero, int* status, void* stream) {
  return launch_jacobi_vec(v, ldv, nv, len, acc, ldacc, sv, xn, ldx, jo, ldj, ascending, nzero,
                           status, reinterpret_cast<cudaStream_t>(stream));
}

size_t rgsv_svd_vectors_blocked_workspace_bytes(int nv) {
  return svd_vectors_blocked_workspace_bytes(nv);
}

int rgsv_svd_vectors_blocked(double* v, int64_t ldv, int nv, int len, double* acc, int64_t ldacc,
                             double* sv, double* xn, int64_t ldx, double* jo, int64_t ldj,
                             int ascending, int* nzero, int* status, void* workspace,
                             size_t workspace_bytes, void* stream) {
  if (ldv < len || ldacc < nv || ldx < len || ldj < nv) return RGSV_ERR_DIMENSION;
  if (!v || !acc || !sv || !xn || !jo || !nzero || !status) return RGSV_ERR_VALIDATION;
  return svd_vectors_blocked(v, ldv, nv, len, acc, ldacc, sv, xn, ldx, jo, ldj, ascending, nzero,
                             status, workspace, workspace_bytes,
                             reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_transpose(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols,
                   void* stream) {
  if (rows < 0 || cols < 0 || ldd < rows || lds < cols) return RGSV_ERR_DIMENSION;
  return launch_copy_block(dst, ldd, src, lds, cols, rows, 1,
                           reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_convert_f32(const float* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
                     int64_t ldd, void* stream) {
  if (rows < 0 || cols < 0 || lds < cols || ldd < cols) return RGSV_ERR_DIMENSION;
  return launch_convert_f32(src, lds, rows, cols, dst, ldd, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_scale_cols(double* a, int64_t lda, int rows, int cols, const double* d, void* stream) {
  return launch_scale_cols(a, lda, rows, cols, d, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_axpy(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols,
              double alpha, void* stream) {
  return launch_axpy(y, ldy, x, ldx, rows, cols, alpha, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- batched
namespace {
struct BatchLayout {
  size_t omega, omega_ws, omega_ws_bytes, b, mstat, total;
  int64_t kp, ldo;
};
BatchLayout batch_layout(int npairs, int64_t n, int k) {
  BatchLayout L{};
  L.kp = k <= 16 ? 16 : 32;
  L.ldo = ceil16(n);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = al256(off + bytes);
    return o;
  };
  const int nm = 2 * npairs;
  L.omega = take((size_t)nm * L.kp * L.ldo * 8);
  L.omega_ws_bytes = rgsv::omega_workspace_bytes(nm, n * (int64_t)k);
  L.omega_ws = take(L.omega_ws_bytes);
  L.b = take((size_t)nm * L.kp * L.ldo * 8);
  L.mstat = take((size_t)(nm + 16) * 4);  // + the chain launches' work counters
  L.total = off;
  return L;
}
}  // namespace

int rgsv_batch_supported(int max_rows, int64_t n, int k) {
  int cs, yrows;
  if (n > 128 || 2 * k > n || k < 1 || max_rows < k) return 0;
  return rgsv::batch_chain_plan(max_rows, (int)n, k, &cs, &yrows) == 0 ? 1 : 0;
}

size_t rgsv_batch_workspace_bytes(int npairs, int64_t n, int k) {
  return batch_layout(npairs, n, k).total;
}

int rgsv_batch_gsvd(const void* mats, int npairs, int max_rows, int64_t n, int k, int q,
                    const uint64_t* seeds, double classify_tol, double* res, int* ints,
                    double* stats, int* status, double* b_out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (npairs < 1 || k < 1 || k > 32 || n < 2 * k || n > 128 || q < 0 || max_rows < k)
    return RGSV_ERR_DIMENSION;
  if (!(classify_tol > 0.0 && classify_tol < 1e-2)) return RGSV_ERR_VALIDATION;
  BatchLayout L = batch_layout(npairs, n, k);
  if (workspace_bytes < L.total) return RGSV_ERR_WORKSPACE;
  char* ws = static_cast<char*>(workspace);
  double* om = reinterpret_cast<double*>(ws + L.omega);
  double* b = b_out ? b_out : reinterpret_cast<double*>(ws + L.b);
  int* mstat = reinterpret_cast<int*>(ws + L.mstat);
  const int nm = 2 * npairs;
  if (cudaMemsetAsync(om, 0, (size_t)nm * L.kp * L.ldo * 8, st) != cudaSuccess) return RGSV_ERR_CUDA;
  if (cudaMemsetAsync(status, 0, (size_t)npairs * 4, st) != cudaSuccess) return RGSV_ERR_CUDA;
  const int64_t res_stride = 6 * n + 4 + 2 * k;
  const int64_t mstride = L.kp * L.ldo;
  // pairs [c0, c0 + np): Omega_i for every matrix from its own stream (pair
  // j: seeds 2j, 2j + 1), the clustered chain, the per-pair small GSVD
  auto omega = [&](int c0, int np, cudaStream_t s) {
    return rgsv::omega_generate(seeds + 2 * c0, 2 * np, n, k, om + 2 * c0 * mstride, L.ldo, mstride,
                                status + c0, ws + L.omega_ws, L.omega_ws_bytes, s);
  };
  int chunk_no = 0;
  auto chain = [&](int c0, int np, cudaStream_t s) {
    int* next = mstat + nm + (chunk_no++ & 15);  // one work counter per chain launch
    return rgsv::batch_chain(static_cast<const rgsv::BatchMat*>(mats) + 2 * c0, 2 * np, max_rows,
                             (int)n, k, q, om + 2 * c0 * mstride, L.ldo, mstride,
                             b + 2 * c0 * mstride, L.ldo, mstride, stats + 4 * c0, mstat + 2 * c0,
                             next, s);
  };
  auto small = [&](int c0, int np, cudaStream_t s) {
    return rgsv::launch_batch_small(b + 2 * c0 * mstride, L.ldo, mstride, np, k, k, (int)n,
                                    classify_tol, res + c0 * res_stride, res_stride, ints + 4 * c0,
                                    status + c0, mstat + 2 * c0, s);
  };
  // Large batches run in chunks on three streams: the chain's persistent
  // clusters leave a dozen SMs idle (clusters must sit inside a GPC: 45 x 3
  // of 148 SMs at cfg3), so the Omega generation of chunk c + 1 and the small
  // GSVDs of chunk c - 1 run there while the chain of chunk c runs. The
  // results are those of the single-launch order (the kernels are the same,
  // per pair). Not taken under stream capture (the side streams are per call).
  // Chunks of >= 512 pairs (>= ~22 rounds of the 45 resident clusters each,
  // so the extra chain tails stay around 1 %).
  constexpr int kChunks = 8;
  static const int want_chunks = [] {
    const char* e = getenv("RGSV_BATCH_CHUNKS");  // tuning: 2 .. 8 (default 4)
    const int v = e ? atoi(e) : 4;
    return v >= 2 && v <= kChunks ? v : 4;
  }();
  const int chunks = npairs / 512 < want_chunks ? npairs / 512 : want_chunks;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  static const bool no_overlap = getenv("RGSV_BATCH_NO_OVERLAP") != nullptr;
  if (chunks < 2 || no_overlap ||
      cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    if (int e = omega(0, npairs, st)) return e;
    if (int e = chain(0, npairs, st)) return e;
    return small(0, npairs, st);
  }
  cudaStream_t s_om = nullptr, s_sm = nullptr, s_ch = nullptr;
  int pr_least = 0, pr_greatest = 0;
  cudaDeviceGetStreamPriorityRange(&pr_least, &pr_greatest);
  cudaEvent_t ev_fork = nullptr, ev_om[kChunks] = {}, ev_ch[kChunks] = {}, ev_join = nullptr;
  int rc = 0;
  auto ok = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == 0) rc = RGSV_ERR_CUDA;
    return e == cudaSuccess;
  };
  auto mkev = [&](cudaEvent_t* e) { return ok(cudaEventCreateWithFlags(e, cudaEventDisableTiming)); };
  // the chain runs at the highest stream priority: its clusters take the SMs
  // the filler kernels' short blocks free, not the other way round
  bool up = ok(cudaStreamCreateWithPriority(&s_om, cudaStreamNonBlocking, pr_least)) &&
            ok(cudaStreamCreateWithPriority(&s_sm, cudaStreamNonBlocking, pr_least)) &&
            ok(cudaStreamCreateWithPriority(&s_ch, cudaStreamNonBlocking, pr_greatest)) &&
            mkev(&ev_fork) && mkev(&ev_join);
  for (int c = 0; up && c < kChunks; ++c) up = mkev(&ev_om[c]) && mkev(&ev_ch[c]);
  if (up) {
    const int per = (npairs + chunks - 1) / chunks;
    ok(cudaEventRecord(ev_fork, st));  // Omega buffer and status cleared
    ok(cudaStreamWaitEvent(s_om, ev_fork, 0));
    ok(cudaStreamWaitEvent(s_sm, ev_fork, 0));
    ok(cudaStreamWaitEvent(s_ch, ev_fork, 0));
    for (int c = 0; c < chunks && rc == 0; ++c) {
      const int c0 = c * per, np = npairs - c0 < per ? npairs - c0 : per;
      if (np <= 0) break;
      if (int e = omega(c0, np, s_om)) rc = e;  // one stream: the workspace is reused in order
      ok(cudaEventRecord(ev_om[c], s_om));
    }
    for (int c = 0; c < chunks && rc == 0; ++c) {
      const int c0 = c * per, np = npairs - c0 < per ? npairs - c0 : per;
      if (np <= 0) break;
      ok(cudaStreamWaitEvent(s_ch, ev_om[c], 0));
      if (int e = chain(c0, np, s_ch)) rc = e;
      ok(cudaEventRecord(ev_ch[c], s_ch));
      ok(cudaStreamWaitEvent(s_sm, ev_ch[c], 0));
      if (rc == 0)
        if (int e = small(c0, np, s_sm)) rc = e;
    }
    ok(cudaEventRecord(ev_join, s_sm));
    ok(cudaStreamWaitEvent(st, ev_join, 0));  // s_om's work is ordered before the chains
  }
  // destroying streams / events with work in flight only defers their release
  for (int c = 0; c < kChunks; ++c) {
    if (ev_om[c]) cudaEventDestroy(ev_om[c]);
    if (ev_ch[c]) cudaEventDestroy(ev_ch[c]);
  }
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (s_ch) cudaStreamDestroy(s_ch);
  if (s_om) cudaStreamDestroy(s_om);
  if (s_sm) cudaStreamDestroy(s_sm);
  return rc;
}

size_t rgsv_sketch_workspace_bytes(int64_t m, int64_t n, int k) {
  return sketch_layout(m, n, k).total;
}

int rgsv_sketch_project(const double* g, int64_t ldg, int64_t m, int64_t n,
                        const double* omega_t, int64_t ld_omega, int k, int q, double* q_out,
                        double* b_out, int64_t ldb, double* stats, double* rdiag, int* status,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return rgsv_sketch_project_sharded(g, ldg, m, m, n, omega_t, ld_omega, k, q, q_out, b_out, ldb,
                                     stats, rdiag, status, nullptr, nullptr, workspace,
                                     workspace_bytes, stream);
}

int rgsv_sketch_project_sharded(const double* g, int64_t ldg, int64_t m, int64_t m_total,
                                int64_t n, const double* omega_t, int64_t ld_omega, int k, int q,
                                double* q_out, double* b_out, int64_t ldb, double* stats,
                                double* rdiag, int* status, rgsv_allreduce_fn allreduce,
                                void* allreduce_ctx, void* workspace, size_t workspace_bytes,
                                void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (m < 1 || n < 1 || k < 1 || q < 0 || m_total < m) return RGSV_ERR_DIMENSION;
  if (!allreduce && m_total != m) return RGSV_ERR_VALIDATION;
  if (k > m_total || k > n) return RGSV_ERR_VALIDATION;  // rangefinder.py:88-91
  Reducer red;
  red.fn = allreduce;
  red.ctx = allreduce_ctx;
  const Reducer* rp = allreduce ? &red : nullptr;
  const int64_t kp = ceil16(k), ldn = ceil16(n);
  if (kp > 512) return RGSV_ERR_DIMENSION;
  if (ldg < n || ld_omega < n || ldb < n || (ldg & 1) || (ld_omega & 1) || (ldb & 1))
    return RGSV_ERR_DIMENSION;
  SketchLayout L = sketch_layout(m, n, k);
  if (workspace_bytes < L.total) return RGSV_ERR_WORKSPACE;
  char* ws = static_cast<char*>(workspace);
  double* y = reinterpret_cast<double*>(ws + L.y);
  double* z = reinterpret_cast<double*>(ws + L.z);
  double* z2 = reinterpret_cast<double*>(ws + L.z2);
  double* gram = reinterpret_cast<double*>(ws + L.gram);
  double* linv = reinterpret_cast<double*>(ws + L.linv);
  double* rinv = reinterpret_cast<double*>(ws + L.rinv);
  double* rd_ws = reinterpret_cast<double*>(ws + L.rdiag);
  double* ss = reinterpret_cast<double*>(ws + L.ss);
  double* scratch = reinterpret_cast<double*>(ws + L.scratch);
  const size_t sb = L.scratch_bytes;

  // (1) sketch Y = G Omega, fused ||G||_F^2 (rangefinder.py:83,115)
  GemmArgs s;
  s.A = g;
  s.lda = ldg;
  s.B = omega_t;
  s.ldb = ld_omega;
  s.C = y;
  s.ldc = kp;
  s.M = m;
  s.N = kp;
  s.live = k;  // exact-width tiles where they exist (k = 120: cfg2)
  s.K = n;
  s.scratch = scratch;
  s.scratch_bytes = sb;
  s.max_split = gx_split();
  s.ss_out = ss;
  int ss_units = 0;
  s.ss_units = &ss_units;
  if (int e = gemm_gx(s, st)) return e;
  if (ss_units > 4096) return RGSV_ERR_WORKSPACE;
  if (int e = launch_sum(ss, ss_units, stats, st)) return e;
  if (int e = red(stats, 1, st)) return e;  // ||G||_F^2 over all row blocks
  // (2) Q = qr(Y).q  (rangefinder.py:119)
  double* qres = nullptr;
  // Every orthonormalisation is full shifted CholeskyQR3. (Fewer passes for
  // the intermediate bases are exact in exact arithmetic -- each pass is a
  // triangular right factor -- but measured on cfg0/cfg1 one pass inflates
  // the last Y beyond what CholeskyQR3 resolves (full-span angle 8e-5,
  // breakdowns) and two passes still miss the stage tolerances.)
  if (int e = cholqr3_tall(y, q_out, m, k, (int)kp, gram, linv, rd_ws, scratch, sb, status, &qres,
                           st, q == 0 ? 3 : kIntermediatePasses, rp, m_total))
    return e;
  for (int it = 0; it < q; ++it) {
    // Z^T = Q^T G, Qhat = qr(Z).q, Y = G Qhat, Q = qr(Y).q
    GemmArgs p;
    p.A = q_out;
    p.lda = kp;
    p.B = g;
    p.ldb = ldg;
    p.C = z;
    p.ldc = ldn;
    p.M = kp;
    p.N = n;
    p.live = k;
    p.K = m;
    p.scratch = scratch;
    p.scratch_bytes = sb;
    p.max_split = proj_split();
    if (int e = gemm_gtq(p, st)) return e;
    if (int e = red(z, kp * ldn, st)) return e;  // Z^T partials of the row blocks
    double* qt = nullptr;
    if (int e = cholqr3_wide(z, z2, n, ldn, k, (int)kp, gram, linv, rinv, rd_ws, scratch, sb,
                             status, &qt, st, kIntermediatePasses))
      return e;
    GemmArgs y2 = s;
    y2.B = qt;
    y2.ldb = ldn;
    y2.ss_out = nullptr;
    y2.ss_units = nullptr;
    if (int e = gemm_gx(y2, st)) return e;
    if (int e = cholqr3_tall(y, q_out, m, k, (int)kp, gram, linv, rd_ws, scratch, sb, status,
                             &qres, st, it == q - 1 ? 3 : kIntermediatePasses, rp, m_total))
      return e;
  }
  // (3) B = Q^T G (engine.py:255) and its energy (rangefinder.py:123)
  GemmArgs p;
  p.A = q_out;
  p.lda = kp;
  p.B = g;
  p.ldb = ldg;
  p.C = b_out;
  p.ldc = ldb;
  p.M = kp;
  p.N = n;
  p.live = k;
  p.K = m;
  p.scratch = scratch;
  p.scratch_bytes = sb;
  p.max_split = proj_split();
  if (int e = gemm_gtq(p, st)) return e;
  if (int e = red(b_out, kp * ldb, st)) return e;  // B partials -> replicated B
  if (int e = launch_sumsq(b_out, ldb, kp, n, stats + 1, ss, 1024, st)) return e;
  if (rdiag) {
    if (cudaMemcpyAsync(rdiag, rd_ws, k * sizeof(double), cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
      return RGSV_ERR_CUDA;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : RGSV_ERR_CUDA;
}

// ---------------------------------------------------------------- small GSVD
namespace {
struct SmallLayout {
  size_t s, s2, t, t2, gram, linv, rinv, rdiag, v1, v2, scratch, hh, sync, total, scratch_bytes,
      hh_bytes;
  int64_t lp, lds, kpn;
};
SmallLayout small_layout(int l1, int l2, int64_t n) {
  SmallLayout L{};
  const int64_t l = l1 + l2;
  L.lp = ceil16(l);
  L.lds = ceil16(n);
  L.kpn = ceil16(n);
  const int64_t rows = L.lp > l ? L.lp : l;
  // factor size: the wide branch (l <= n) factors lp x lp Grams, the tall
  // branch (l > n) kpn x kpn ones -- never max of both (cfg4: n = 8192, l = 576)
  const int64_t kmax = (l > n) ? L.kpn : L.lp;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = al256(off + bytes);
    return o;
  };
  L.s = take((size_t)rows * L.lds * 8);
  L.s2 = take((size_t)rows * L.lds * 8);
  L.t = take((size_t)L.lp * L.lp * 8);
  L.t2 = take((size_t)L.lp * L.lp * 8);
  L.gram = take((size_t)kmax * kmax * 8);
  L.linv = take((size_t)kmax * kmax * 8 + (size_t)kmax * (kmax + 1) * 8);
  L.rinv = take((size_t)kmax * kmax * 8);
  L.rdiag = take((size_t)kmax * 8);
  const int64_t rmax = l < L.kpn ? l : L.kpn;  // columns of the stacked Q
  L.v1 = take((size_t)(l1 + 1) * (rmax + 1) * 8);
  L.v2 = take((size_t)(l2 + 1) * (rmax + 1) * 8);
  L.scratch_bytes = split_scratch_bytes(l, n, kmax) + (size_t)kSMs * kmax * kmax * 8;
  L.scratch = take(L.scratch_bytes);
  // multi-CTA Householder of the leading l x l block (wide) or of S (tall)
  L.hh_bytes = (l <= kHhMaxRows) ? hhqr_workspace_bytes((int)l, (int)(l <= n ? l : n)) : 0;
  L.hh = take(L.hh_bytes);
  L.sync = take(bjacobi_sync_bytes());
  L.total = off;
  return L;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
// Stacked sizes l served by the multi-CTA Householder (k_hhqr) rather than
// the one-CTA register kernel, and vector counts served by the blocked
// Jacobi (k_bjacobi) rather than the one-CTA Jacobi (measured crossovers,
// DESIGN.md §4b; RGSV_HH_MIN / RGSV_BJ_MIN override them). Below 64 vectors
// the one-CTA Jacobi wins in throughput: with 8 concurrent cfg1 pairs (60
// vectors) the blocked kernel's spinning CTAs cost 736 -> 694 pairs/s.
int hh_min_l() {
  static const int v = env_int("RGSV_HH_MIN", 129);
  return v;
}
int bj_min_nv() {
  static const int v = env_int("RGSV_BJ_MIN", 64);
  return v;
}
}  // namespace

// Row-vector Jacobi dispatch: the blocked multi-CTA kernel for larger jobs.
static int jacobi_dispatch(double* v1, int64_t ld1, int nv1, int len1, double* sv1, int* nsv1,
                           double* v2, int64_t ld2, int nv2, int len2, double* sv2, int* nsv2,
                           int* status, void* sync, cudaStream_t st) {
  const int nv = nv1 > nv2 ? nv1 : nv2;
  if (sync && (nv >= bj_min_nv() || nv > 2048))
    return bjacobi(v1, ld1, nv1, len1, sv1, nsv1, v2, ld2, nv2, len2, sv2, nsv2, status, sync, st);
  return launch_jacobi(v1, ld1, nv1, len1, sv1, nsv1, v2, ld2, nv2, len2, sv2, nsv2, status, st);
}

size_t rgsv_small_gsvd_workspace_bytes(int l1, int l2, int64_t n) {
  return small_layout(l1, l2, n).total;
}

int rgsv_small_gsvd(const double* b1, int64_t ldb1, int l1, const double* b2, int64_t ldb2, int l2,
                    int64_t n, double* sv1, double* sv2, int* nsv, int* status, void* workspace,
                    size_t workspace_bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (l1 < 0 || l2 < 0 || n < 1) return RGSV_ERR_DIMENSION;
  const int l = l1 + l2;
  if (l == 0) return RGSV_ERR_RANK;  // engine.py:258-259
  SmallLayout L = small_layout(l1, l2, n);
  if (workspace_bytes < L.total) return RGSV_ERR_WORKSPACE;
  char* ws = static_cast<char*>(workspace);
  double* S = reinterpret_cast<double*>(ws + L.s);
  double* S2 = reinterpret_cast<double*>(ws + L.s2);
  double* T = reinterpret_cast<double*>(ws + L.t);
  double* T2 = reinterpret_cast<double*>(ws + L.t2);
  double* gram = reinterpret_cast<double*>(ws + L.gram);
  double* linv = reinterpret_cast<double*>(ws + L.linv);
  double* rinv = reinterpret_cast<double*>(ws + L.rinv);
  double* rdiag = reinterpret_cast<double*>(ws + L.rdiag);
  double* v1 = reinterpret_cast<double*>(ws + L.v1);
  double* v2 = reinterpret_cast<double*>(ws + L.v2);
  double* scratch = reinterpret_cast<double*>(ws + L.scratch);
  const size_t sb = L.scratch_bytes;
  void* sync = ws + L.sync;
  const int64_t lp = L.lp, lds = L.lds;

  double* Q = nullptr;
  int64_t ldq = 0;
  int r = 0;
  if (l <= n && l >= hh_min_l() && l <= kHhMaxRows) {
    // wide S: Q of the leading l x l block (= Q of S), blocked Householder
    // over many CTAs (dgeqrf + dorgqr, one cooperative launch)
    Q = T;
    ldq = lp;
    if (int e = hhqr(b1, ldb1, l1, b2, ldb2, l2, l, Q, ldq, nullptr, 0, 0, ws + L.hh, L.hh_bytes,
                     st))
      return e;
    r = l;
  } else if (l > n && l <= kHhMaxRows) {
    // tall stacked matrix (l > n): thin Q (l x n) of the Householder QR
    Q = S;
    ldq = lds;
    if (int e = hhqr(b1, ldb1, l1, b2, ldb2, l2, (int)n, Q, ldq, nullptr, 0, 0, ws + L.hh,
                     L.hh_bytes, st))
      return e;
    r = (int)n;
  } else if (l <= n && l <= 512) {
    // wide S: Householder Q of the leading l x l block (= Q of S, see
    // k_householder_small), one CTA (shared memory, or L2-resident scratch)
    Q = T;
    ldq = lp;
    if (int e = launch_householder_small(b1, ldb1, l1, b2, ldb2, l2, Q, ldq, S, st)) return e;
    r = l;
  } else if (l <= n) {
    // S = [B1; B2] (l x n, wide). S^T = P T (CholQR3 on S^T), so
    // range(S) = range(T^T) and the Q of qr(S) is the Q of qr(T^T).
    if (int e = launch_stack(S, lds, b1, ldb1, l1, b2, ldb2, l2, (int)lp, n, st)) return e;
    if (lp > kCholMaxKp) return RGSV_ERR_DIMENSION;
    double* pt = nullptr;
    if (int e = cholqr3_wide(S, S2, n, lds, l, (int)lp, gram, linv, rinv, rdiag, scratch, sb,
                             status, &pt, st))
      return e;
    // T^T = S P  (lp x lp)
    double* ssrc = (pt == S) ? S2 : S;  // the buffer not holding P^T was overwritten: rebuild S
    if (int e = launch_stack(ssrc, lds, b1, ldb1, l1, b2, ldb2, l2, (int)lp, n, st)) return e;
    GemmArgs tt;
    tt.A = ssrc;
    tt.lda = lds;
    tt.B = pt;
    tt.ldb = lds;
    tt.C = T;
    tt.ldc = lp;
    tt.M = lp;
    tt.N = lp;
    tt.K = n;
    tt.scratch = scratch;
    tt.scratch_bytes = sb;
    tt.max_split = 32;
    if (int e = gemm_gx(tt, st)) return e;
    if (int e = cholqr3_tall(T, T2, l, l, (int)lp, gram, linv, rdiag, scratch, sb, status, &Q,
                             st))
      return e;
    ldq = lp;
    r = l;
  } else {
    // tall stacked matrix (l > n): Q = qr(S).q directly
    const int64_t kpn = L.kpn;
    if (kpn > kCholMaxKp) return RGSV_ERR_DIMENSION;  // blocked Cholesky limit
    if (int e = launch_stack(S, kpn, b1, ldb1, l1, b2, ldb2, l2, l, n, st)) return e;
    // The direct method stacks the pair itself here: any stack the reference
    // accepts (sigma_min > 1e-12 sigma_max, engine.py:57) must factor, so two
    // shifted passes and two plain ones (CholeskyQR3 proper stops at
    // cond ~ 1e10 for n ~ 1000).
    if (int e = cholqr3_tall(S, S2, l, (int)n, (int)kpn, gram, linv, rdiag, scratch, sb, status,
                             &Q, st, 4, nullptr, -1, 2))
      return e;
    ldq = kpn;
    r = (int)n;
  }
  // L1 = Q[:l1, :r], L2 = Q[l1:, :r]; Jacobi on whichever side has fewer vectors
  int nv1, len1, nv2, len2;
  int64_t ld1, ld2;
  if (l1 <= r) {
    nv1 = l1; len1 = r; ld1 = r;
    if (int e = launch_copy_block(v1, ld1, Q, ldq, l1, r, 0, st)) return e;
  } else {
    nv1 = r; len1 = l1; ld1 = l1;
    if (int e = launch_copy_block(v1, ld1, Q, ldq, r, l1, 1, st)) return e;
  }
  if (l2 <= r) {
    nv2 = l2; len2 = r; ld2 = r;
    if (int e = launch_copy_block(v2, ld2, Q + (int64_t)l1 * ldq, ldq, l2, r, 0, st)) return e;
  } else {
    nv2 = r; len2 = l2; ld2 = l2;
    if (int e = launch_copy_block(v2, ld2, Q + (int64_t)l1 * ldq, ldq, r, l2, 1, st)) return e;
  }
  return jacobi_dispatch(v1, ld1, nv1, len1, sv1, nsv, v2, ld2, nv2, len2, sv2, nsv + 1, status,
                         sync, st);
}

size_t rgsv_dense_qr_workspace_bytes(int M, int N) {
  if (M < 1 || N < 1 || M > kHhMaxRows) return 0;
  return hhqr_workspace_bytes(M, N);
}

int rgsv_dense_qr(const double* a1, int64_t lda1, int m1, const double* a2, int64_t lda2,
                  int m2, int N, double* q, int64_t ldq, double* r, int64_t ldr, int phase_fix,
                  void* workspace, size_t workspace_bytes, void* stream) {
  if (m1 < 0 || m2 < 0 || N < 1 || m1 + m2 < 1 || m1 + m2 > kHhMaxRows) return RGSV_ERR_DIMENSION;
  if ((m2 > 0 && !a2) || !a1 || !q) return RGSV_ERR_VALIDATION;
  const int K = (m1 + m2) < N ? (m1 + m2) : N;
  if (ldq < K || (r && ldr < N) || (m1 > 0 && lda1 < N) || (m2 > 0 && lda2 < N))
    return RGSV_ERR_DIMENSION;
  if (!workspace || workspace_bytes < hhqr_workspace_bytes(m1 + m2, N)) return RGSV_ERR_WORKSPACE;
  return hhqr(a1, lda1, m1, a2, lda2, m2, N, q, ldq, r, ldr, phase_fix, workspace,
              workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_debug_dense_qr_profile(const double* a, int64_t lda, int M, int N, double* q,
                                void* workspace, size_t workspace_bytes, long long* prof,
                                void* stream) {
  if (M < 1 || N < 1 || M > kHhMaxRows) return RGSV_ERR_DIMENSION;
  return hhqr(a, lda, M, nullptr, 0, 0, N, q, M < N ? M : N, nullptr, 0, 0, workspace,
              workspace_bytes, reinterpret_cast<cudaStream_t>(stream), prof);
}

int rgsv_comparative(const double* sv1, const int* nsv, const double* sv2, int64_t n,
                     double classify_tol, double* alphas, double* betas, double* rho,
                     double* theta, double* p1, double* p2, double* scalars, int* counts,
                     int* status, void* stream) {
  if (n < 1) return RGSV_ERR_DIMENSION;
  if (!(classify_tol > 0.0 && classify_tol < 1e-2)) return RGSV_ERR_VALIDATION;
  return launch_comparative(sv1, nsv, sv2, n, classify_tol, alphas, betas, rho, theta, p1, p2,
                            scalars, counts, status, 0, 0, reinterpret_cast<cudaStream_t>(stream));
}

size_t rgsv_spectrum_from_l_blocks_workspace_bytes(int l1, int l2, int cols, int64_t n) {
  return al256((size_t)(l1 > 0 ? l1 : 1) * (cols + 1) * 8) +
         al256((size_t)(l2 > 0 ? l2 : 1) * (cols + 1) * 8) + al256(2 * sizeof(double) * (cols + 1)) +
         bjacobi_sync_bytes() + al256(8 * (4 * (size_t)n + 4)) + 256;
}

int rgsv_spectrum_from_l_blocks(const double* l1b, int64_t ld1, int l1, const double* l2b,
                                int64_t ld2, int l2, int cols, int64_t n, double classify_tol,
                                int branch, double* alphas, double* betas, int* counts,
                                int* status, void* workspace, size_t workspace_bytes,
                                void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (l1 < 0 || l2 < 0 || cols < 0 || n < 1 || branch < 0 || branch > 2) return RGSV_ERR_DIMENSION;
  // the singular-value counts min(l, cols) must fit the n-long spectrum
  if ((l1 > 0 && ld1 < cols) || (l2 > 0 && ld2 < cols) || (l1 < cols ? l1 : cols) > n ||
      (l2 < cols ? l2 : cols) > n)
    return RGSV_ERR_DIMENSION;
  if (!(classify_tol > 0.0 && classify_tol < 1e-2)) return RGSV_ERR_VALIDATION;
  if (workspace_bytes < rgsv_spectrum_from_l_blocks_workspace_bytes(l1, l2, cols, n))
    return RGSV_ERR_WORKSPACE;
  char* ws = static_cast<char*>(workspace);
  double* v1 = reinterpret_cast<double*>(ws);
  ws += al256((size_t)(l1 > 0 ? l1 : 1) * (cols + 1) * 8);
  double* v2 = reinterpret_cast<double*>(ws);
  ws += al256((size_t)(l2 > 0 ? l2 : 1) * (cols + 1) * 8);
  double* sv = reinterpret_cast<double*>(ws);  // sv1 | sv2 (cols + 1 each... <= min dims)
  ws += al256(2 * sizeof(double) * (cols + 1));
  void* sync = ws;
  ws += bjacobi_sync_bytes();
  double* q4 = reinterpret_cast<double*>(ws);  // rho | theta | p1 | p2 | scalars (unused here)
  ws += al256(8 * (4 * (size_t)n + 4));
  int* nsv = reinterpret_cast<int*>(ws);
  double* sv1 = sv;
  double* sv2 = sv + (cols + 1);
  // singular values of each block by one-sided Jacobi on its shorter side
  auto orient = [&](const double* b, int64_t ldb, int rows, double* v, int* nv, int* len,
                    int64_t* ld) -> int {
    if (rows == 0 || cols == 0) {
      *nv = 0;
      *len = cols > 0 ? cols : 1;
      *ld = *len;
      return 0;
    }
    if (rows <= cols) {
      *nv = rows;
      *len = cols;
      *ld = cols;
      return launch_copy_block(v, cols, b, ldb, rows, cols, 0, st);
    }
    *nv = cols;
    *len = rows;
    *ld = rows;
    return launch_copy_block(v, rows, b, ldb, cols, rows, 1, st);
  };
  int nv1, len1, nv2, len2;
  int64_t vld1, vld2;
  if (int e = orient(l1b, ld1, l1, v1, &nv1, &len1, &vld1)) return e;
  if (int e = orient(l2b, ld2, branch == 1 ? 0 : l2, v2, &nv2, &len2, &vld2)) return e;
  if (int e = jacobi_dispatch(v1, vld1, nv1, len1, sv1, nsv, v2, vld2, nv2, len2, sv2, nsv + 1,
                              status, sync, st))
    return e;
  // spectrum completion (merged / forced branch) + classification; the
  // comparative quantities the kernel also forms go to scratch
  return launch_comparative(sv1, nsv, sv2, n, classify_tol, alphas, betas, q4, q4 + n, q4 + 2 * n,
                            q4 + 3 * n, q4 + 4 * n, counts, status, branch == 0 ? 0 : branch + 2,
                            0, st);
}

int rgsv_spectrum_quantities(const double* alphas, const double* betas, int64_t n, int r,
                             double* rho, double* theta, double* p1, double* p2, double* scalars,
                             int* status, void* stream) {
  if (n < 1 || r < 0 || r > n) return RGSV_ERR_DIMENSION;
  return launch_comparative(alphas, nullptr, betas, n, 0.0, nullptr, nullptr, rho, theta, p1, p2,
                            scalars, nullptr, status, 1, r,
                            reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_entropy(const double* p, int64_t n, double* scalars, void* stream) {
  if (n < 2) return RGSV_ERR_VALIDATION;
  return launch_comparative(p, nullptr, nullptr, n, 0.0, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr, scalars, nullptr, nullptr, 2, 0,
                            reinterpret_cast<cudaStream_t>(stream));
}

size_t rgsv_svd_values_workspace_bytes(int rows, int cols) {
  return al256((size_t)rows * cols * sizeof(double)) + bjacobi_sync_bytes();
}

int rgsv_svd_values(const double* a, int64_t lda, int rows, int cols, double* sv, int* nsv,
                    int* status, void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (rows < 1 || cols < 1) return RGSV_ERR_DIMENSION;
  if (workspace_bytes < rgsv_svd_values_workspace_bytes(rows, cols)) return RGSV_ERR_WORKSPACE;
  double* v = static_cast<double*>(workspace);
  int nv, len;
  if (rows <= cols) {
    nv = rows;
    len = cols;
    if (int e = launch_copy_block(v, len, a, lda, rows, cols, 0, st)) return e;
  } else {
    nv = cols;
    len = rows;
    if (int e = launch_copy_block(v, len, a, lda, cols, rows, 1, st)) return e;
  }
  void* sync = static_cast<char*>(workspace) + al256((size_t)rows * cols * sizeof(double));
  return jacobi_dispatch(v, len, nv, len, sv, nsv, v, len, 0, len, sv, nsv + 1, status, sync, st);
}

int rgsv_gemm_gx(const double* a, int64_t lda, const double* bt, int64_t ldb, double* c,
                 int64_t ldc, int64_t M, int64_t N, int64_t K, void* scratch,
                 size_t scratch_bytes, void* stream) {
  GemmArgs g;
  g.A = a;
  g.lda = lda;
  g.B = bt;
  g.ldb = ldb;
  g.C = c;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.scratch = static_cast<double*>(scratch);
  g.scratch_bytes = scratch_bytes;
  g.max_split = 32;
  return gemm_gx(g, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_gemm_gram_lower(const double* a, int64_t lda, int64_t cols, int64_t rows, double* c,
                         int64_t ldc, void* scratch, size_t scratch_bytes, void* stream) {
  if (cols < 1 || rows < 1 || lda < cols || ldc < cols) return RGSV_ERR_DIMENSION;
  GemmArgs g;
  g.A = a;
  g.lda = lda;
  g.B = a;
  g.ldb = lda;
  g.C = c;
  g.ldc = ldc;
  g.M = cols;
  g.N = cols;
  g.K = rows;
  g.scratch = static_cast<double*>(scratch);
  g.scratch_bytes = scratch_bytes;
  g.max_split = kSMs;
  g.lower_only = 1;
  return gemm_gtq(g, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_gemm_gtq(const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                  int64_t ldc, int64_t M, int64_t N, int64_t K, void* scratch,
                  size_t scratch_bytes, void* stream) {
  GemmArgs g;
  g.A = a;
  g.lda = lda;
  g.B = b;
  g.ldb = ldb;
  g.C = c;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.scratch = static_cast<double*>(scratch);
  g.scratch_bytes = scratch_bytes;
  g.max_split = kSMs;
  return gemm_gtq(g, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_chol_inv(const double* gram, int k, int kp, int64_t shift_rows, double* linv,
                  double* rinv, double* rdiag, int* status, void* stream) {
  return chol_inv(gram, k, kp, shift_rows, linv, rinv, nullptr, rdiag, nullptr, status,
                  reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_debug_householder_profile(const double* b1, int64_t ld1, int l1, const double* b2,
                                   int64_t ld2, int l2, double* q, int64_t ldq, long long* prof,
                                   void* stream) {
  return rgsv::debug_householder_profile(b1, ld1, l1, b2, ld2, l2, q, ldq, prof,
                                         reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_debug_chol_profile(const double* gram, int k, int kp, double* linv, long long* prof,
                            int* status, void* stream) {
  return rgsv::chol_profile(gram, k, kp, linv, prof, status, reinterpret_cast<cudaStream_t>(stream));
}

int rgsv_sumsq(const double* a, int64_t lda, int64_t rows, int64_t cols, double* out,
               void* workspace, size_t workspace_bytes, void* stream) {
  if (rows < 1 || cols < 1) return RGSV_ERR_DIMENSION;
  int parts = (int)(workspace_bytes / sizeof(double));
  if (parts > 1024) parts = 1024;
  if (parts < 1) return RGSV_ERR_WORKSPACE;
  return launch_sumsq(a, lda, rows, cols, out, static_cast<double*>(workspace), parts,
                      reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
