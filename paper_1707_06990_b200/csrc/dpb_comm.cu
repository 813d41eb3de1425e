// Data-parallel gradient exchange of the whole-network step:
// one NCCL communicator per GPU (one process per GPU), per-GPU BN statistics
// (the reference's semantics), and an average allreduce of the
// fp32 parameter gradients issued per block bucket on a communication stream
// as soon as that block's backward has produced them — overlapped with the
// backward of the blocks below it, joined before the step returns (so the
// caller's SGD sees averaged gradients), and capturable in the step's CUDA
// graph.
//
// NCCL is bound at run time (dlopen of libnccl.so.2, reusing the copy the
// process already loaded — e.g. torch's — when there is one), so libdpb has
// no link-time NCCL dependency and cannot pull a second NCCL into a process.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dpb.h"
#include "dpb_comm.h"
#include "dpb_internal.h"
#include "dpb_launch.h"

namespace dpb {
namespace {

// the subset of nccl.h (2.x ABI) libdpb calls
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclFloat = 7, kNcclAvg = 4 };

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);  // the NCCL already in the process
      if (api.h) break;
    }
    for (const char* n : names) {
      if (api.h) break;
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!api.h) {
      api.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* s) { return dlsym(api.h, s); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.GetErrorString)
      api.error = "libnccl.so.2 lacks the expected symbols";
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  NcclApi& n = nccl();
  return fail(DPB_NCCL_ERROR, std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "?"));
}

}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

int comm_allreduce_avg(Comm* c, float* buf, int64_t n, cudaStream_t st) {
  if (n <= 0) return DPB_OK;
  const ncclResult_t r = nccl().AllReduce(buf, buf, static_cast<size_t>(n), kNcclFloat, kNcclAvg, c->comm, st);
  return r == 0 ? DPB_OK : nccl_fail(r, "ncclAllReduce");
}

int comm_ranks(const Comm* c) { return c ? c->nranks : 1; }

}  // namespace dpb

using dpb::fail;

extern "C" {

DPB_API int dpb_comm_unique_id(uint8_t* out) {
  if (!out) return fail(DPB_CONFIG_ERROR, "null id buffer");
  dpb::NcclApi& n = dpb::nccl();
  if (!n.error.empty()) return fail(DPB_NCCL_ERROR, n.error);
  dpb::ncclUniqueId id;
  const dpb::ncclResult_t r = n.GetUniqueId(&id);
  if (r != 0) return dpb::nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, id.internal, sizeof(id.internal));
  return DPB_OK;
}

DPB_API int dpb_comm_init(int nranks, int rank, const uint8_t* id, int device, dpb_comm** out) {
  if (!out || !id) return fail(DPB_CONFIG_ERROR, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(DPB_CONFIG_ERROR, "rank outside [0, nranks)");
  dpb::NcclApi& n = dpb::nccl();
  if (!n.error.empty()) return fail(DPB_NCCL_ERROR, n.error);
  dpb::DeviceGuard dg(device);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return dpb::cuda_fail(e, "cudaSetDevice");
  auto* c = new dpb::Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  dpb::ncclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  const dpb::ncclResult_t r = n.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != 0) {
    delete c;
    return dpb::nccl_fail(r, "ncclCommInitRank");
  }
  *out = reinterpret_cast<dpb_comm*>(c);
  return DPB_OK;
}

DPB_API int dpb_comm_destroy(dpb_comm* comm) {
  if (!comm) return DPB_OK;
  auto* c = reinterpret_cast<dpb::Comm*>(comm);
  dpb::DeviceGuard dg(c->device);
  const dpb::ncclResult_t r = dpb::nccl().CommDestroy(c->comm);
  delete c;
  return r == 0 ? DPB_OK : dpb::nccl_fail(r, "ncclCommDestroy");
}

DPB_API int dpb_comm_check(dpb_comm* comm) {
  if (!comm) return fail(DPB_CONFIG_ERROR, "null communicator");
  auto* c = reinterpret_cast<dpb::Comm*>(comm);
  dpb::NcclApi& n = dpb::nccl();
  if (!n.CommGetAsyncError) return DPB_OK;
  dpb::ncclResult_t ae = 0;
  const dpb::ncclResult_t r = n.CommGetAsyncError(c->comm, &ae);
  if (r != 0) return dpb::nccl_fail(r, "ncclCommGetAsyncError");
  return ae == 0 ? DPB_OK : dpb::nccl_fail(ae, "NCCL asynchronous error");
}

}  // extern "C"
