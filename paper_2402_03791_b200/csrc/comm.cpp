// NCCL plumbing for the ZeroPP step: ZeRO-group all-gather / reduce-scatter and the
// pipeline P2P channels.  NCCL is dlopen()ed from the same libnccl.so.2 that torch
// loads (path supplied by the host), so one NCCL lives in the process.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <cuda_runtime.h>

#include "zpp_internal.h"

namespace {

typedef int ncclResult_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef void* ncclComm_t;
enum { nccl_float32 = 7, nccl_bfloat16 = 9 };
enum { nccl_sum = 0 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl g;

int nccl_err(ncclResult_t r, const char* what) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: nccl error %d (%s)", what, r, g.GetErrorString ? g.GetErrorString(r) : "?");
  return zpp::set_error(ZPP_ERR_NCCL, buf);
}

int need() { return g.h ? 0 : zpp::set_error(ZPP_ERR_NCCL, "NCCL not loaded (call zpp_nccl_load)"); }

int dt(int dtype) { return dtype == 1 ? nccl_float32 : nccl_bfloat16; }

}  // namespace

extern "C" int zpp_nccl_load(const char* path) {
  if (g.h) return ZPP_OK;
  void* h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) return zpp::set_error(ZPP_ERR_NCCL, dlerror());
#define SYM(field, name)                                                  \
  g.field = reinterpret_cast<decltype(g.field)>(dlsym(h, name));          \
  if (!g.field) return zpp::set_error(ZPP_ERR_NCCL, "missing symbol " name);
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(AllGather, "ncclAllGather");
  SYM(ReduceScatter, "ncclReduceScatter");
  SYM(AllReduce, "ncclAllReduce");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  g.h = h;
  return ZPP_OK;
}

extern "C" int zpp_nccl_unique_id(char* out128) {
  if (int rc = need()) return rc;
  ncclUniqueId id;
  ncclResult_t r = g.GetUniqueId(&id);
  if (r) return nccl_err(r, "ncclGetUniqueId");
  memcpy(out128, id.internal, 128);
  return ZPP_OK;
}

extern "C" int zpp_comm_init(const char* uid128, int nranks, int rank, void** comm) {
  if (int rc = need()) return rc;
  ncclUniqueId id;
  memcpy(id.internal, uid128, 128);
  ncclComm_t c = nullptr;
  ncclResult_t r = g.CommInitRank(&c, nranks, id, rank);
  if (r) return nccl_err(r, "ncclCommInitRank");
  *comm = c;
  return ZPP_OK;
}

extern "C" int zpp_comm_destroy(void* comm) {
  if (int rc = need()) return rc;
  ncclResult_t r = g.CommDestroy(comm);
  return r ? nccl_err(r, "ncclCommDestroy") : ZPP_OK;
}

extern "C" int zpp_allgather(void* comm, const void* send, void* recv, long long count, int dtype, uintptr_t stream) {
  if (int rc = need()) return rc;
  ncclResult_t r = g.AllGather(send, recv, (size_t)count, dt(dtype), comm, reinterpret_cast<cudaStream_t>(stream));
  return r ? nccl_err(r, "ncclAllGather") : ZPP_OK;
}

extern "C" int zpp_reduce_scatter(void* comm, const void* send, void* recv, long long count, int dtype,
                                  uintptr_t stream) {
  if (int rc = need()) return rc;
  ncclResult_t r = g.ReduceScatter(send, recv, (size_t)count, dt(dtype), nccl_sum, comm,
                                   reinterpret_cast<cudaStream_t>(stream));
  return r ? nccl_err(r, "ncclReduceScatter") : ZPP_OK;
}

extern "C" int zpp_allreduce(void* comm, const void* send, void* recv, long long count, int dtype,
                             uintptr_t stream) {
  if (int rc = need()) return rc;
  ncclResult_t r = g.AllReduce(send, recv, (size_t)count, dt(dtype), nccl_sum, comm,
                               reinterpret_cast<cudaStream_t>(stream));
  return r ? nccl_err(r, "ncclAllReduce") : ZPP_OK;
}

extern "C" int zpp_send(void* comm, const void* buf, long long count, int dtype, int peer, uintptr_t stream) {
  if (int rc = need()) return rc;
  ncclResult_t r = g.Send(buf, (size_t)count, dt(dtype), peer, comm, reinterpret_cast<cudaStream_t>(stream));
  return r ? nccl_err(r, "ncclSend") : ZPP_OK;
}

extern "C" int zpp_recv(void* comm, void* buf, long long count, int dtype, int peer, uintptr_t stream) {
  if (int rc = need()) return rc;
  ncclResult_t r = g.Recv(buf, (size_t)count, dt(dtype), peer, comm, reinterpret_cast<cudaStream_t>(stream));
  return r ? nccl_err(r, "ncclRecv") : ZPP_OK;
}
