// Collectives for the row-sharded pipeline: NCCL over
// NVLink / NVSwitch, resolved at run time.
//
// The library does not link NCCL: the process that hosts it (PyTorch, or a
// C/Go host) normally has libnccl.so.2 loaded already, and two NCCL builds
// in one process would collide on the soname. The first call dlopen()s the
// loaded copy (RTLD_NOLOAD), else the soname from the loader path.
//
// rgsv_nccl_allreduce has the rgsv_allreduce_fn signature, so a caller
// passes (rgsv_nccl_allreduce, comm) straight to rgsv_sketch_project_sharded
// and every partial (||G||^2, the k x k Grams, Z^T, B) is summed in-stream
// by NCCL; the whole sharded pair is then capturable in one CUDA graph.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "rgsv_internal.h"

namespace rgsv {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce && a.broadcast;
  });
  return a;
}

}  // namespace
}  // namespace rgsv

using namespace rgsv;

extern "C" {

int rgsv_nccl_version(void) {
  NcclApi& a = api();
  if (!a.ok || !a.get_version) return -1;
  int v = 0;
  return a.get_version(&v) == ncclSuccess ? v : -1;
}

int rgsv_nccl_get_unique_id(void* id_out) {
  NcclApi& a = api();
  if (!a.ok) return RGSV_ERR_CUDA;
  if (!id_out) return RGSV_ERR_VALIDATION;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return RGSV_ERR_CUDA;
  memcpy(id_out, &id, sizeof(id));
  return 0;
}

int rgsv_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank) {
  NcclApi& a = api();
  if (!a.ok) return RGSV_ERR_CUDA;
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return RGSV_ERR_VALIDATION;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (a.comm_init_rank(&c, nranks, uid, rank) != ncclSuccess) return RGSV_ERR_CUDA;
  *comm_out = c;
  return 0;
}

int rgsv_nccl_comm_destroy(void* comm) {
  NcclApi& a = api();
  if (!a.ok) return RGSV_ERR_CUDA;
  if (!comm) return 0;
  return a.comm_destroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? 0 : RGSV_ERR_CUDA;
}

int rgsv_nccl_allreduce(double* buf, int64_t count, void* stream, void* comm) {
  NcclApi& a = api();
  if (!a.ok) return RGSV_ERR_CUDA;
  if (count < 0 || (count > 0 && !buf) || !comm) return RGSV_ERR_VALIDATION;
  if (count == 0) return 0;
  note_launch();
  return a.all_reduce(buf, buf, (size_t)count, ncclFloat64, ncclSum,
                      static_cast<ncclComm_t>(comm),
                      reinterpret_cast<cudaStream_t>(stream)) == ncclSuccess
             ? 0
             : RGSV_ERR_CUDA;
}

int rgsv_nccl_broadcast(void* buf, int64_t bytes, int root, void* stream, void* comm) {
  NcclApi& a = api();
  if (!a.ok) return RGSV_ERR_CUDA;
  if (bytes < 0 || (bytes > 0 && !buf) || !comm || root < 0) return RGSV_ERR_VALIDATION;
  if (bytes == 0) return 0;
  note_launch();
  return a.broadcast(buf, buf, (size_t)bytes, ncclUint8, root, static_cast<ncclComm_t>(comm),
                     reinterpret_cast<cudaStream_t>(stream)) == ncclSuccess
             ? 0
             : RGSV_ERR_CUDA;
}

}  // extern "C"
