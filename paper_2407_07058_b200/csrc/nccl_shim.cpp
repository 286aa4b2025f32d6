// nccl_shim.cpp -- the Boruvka round exchange over NVLink.
//
// libnccl.so.2 (the copy torch ships) is opened with dlopen only when a context
// is created with world > 1, so single-GPU use has no NCCL dependency.  Each
// Boruvka round, every rank holds the minimum edge key of every component over
// ITS rows; an all-reduce with ncclMin over uint64 gives every rank the global
// per-component minimum (the north star's "per-round allgather of per-component
// minimum edges", in its reduced form).  All ranks then run the identical,
// deterministic component step, so no further collective is needed.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace appd {

struct NcclApi {
  void* so = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclCommGetAsyncError) asyncError = nullptr;
};

static NcclApi g_nccl;

static bool load_nccl(std::string* err) {
  if (g_nccl.so) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* so = nullptr;
  for (const char* nm : names) {
    so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (so) break;
  }
  if (!so) {
    if (err) *err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return false;
  }
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(so, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(so, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(so, "ncclAllReduce");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(so, "ncclCommDestroy");
  g_nccl.errorString = (decltype(g_nccl.errorString))dlsym(so, "ncclGetErrorString");
  g_nccl.asyncError = (decltype(g_nccl.asyncError))dlsym(so, "ncclCommGetAsyncError");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.commDestroy) {
    if (err) *err = "libnccl.so.2 lacks a required symbol";
    return false;
  }
  g_nccl.so = so;
  return true;
}

appd_status nccl_unique_id(uint8_t out[128], std::string* err) {
  if (!load_nccl(err)) return APPD_ERR_NCCL;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) {
    if (err) *err = std::string("ncclGetUniqueId: ") + (g_nccl.errorString ? g_nccl.errorString(r) : "?");
    return APPD_ERR_NCCL;
  }
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return APPD_OK;
}

appd_status nccl_init(appd_ctx* c, const uint8_t* idbytes, int rank, int world) {
  std::string err;
  if (!load_nccl(&err)) return fail(c, APPD_ERR_NCCL, "%s", err.c_str());
  ncclUniqueId id;
  std::memcpy(&id, idbytes, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = g_nccl.commInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) {
    c->poisoned = true;
    return fail(c, APPD_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.errorString ? g_nccl.errorString(r) : "?");
  }
  c->nccl_comm = comm;
  return APPD_OK;
}

static appd_status allreduce(appd_ctx* c, u64* buf, int64_t count, ncclRedOp_t op) {
  if (!c->nccl_comm) return fail(c, APPD_ERR_NCCL, "no communicator");
  ncclResult_t r = g_nccl.allReduce(buf, buf, (size_t)count, ncclUint64, op, (ncclComm_t)c->nccl_comm, c->stream);
  if (r != ncclSuccess) {
    c->poisoned = true;
    return fail(c, APPD_ERR_NCCL, "ncclAllReduce: %s", g_nccl.errorString ? g_nccl.errorString(r) : "?");
  }
  return APPD_OK;
}

appd_status nccl_allreduce_min_u64(appd_ctx* c, u64* buf, int64_t count) { return allreduce(c, buf, count, ncclMin); }
appd_status nccl_allreduce_max_u64(appd_ctx* c, u64* buf, int64_t count) { return allreduce(c, buf, count, ncclMax); }

void nccl_destroy(appd_ctx* c) {
  if (c->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)c->nccl_comm);
  c->nccl_comm = nullptr;
}

}  // namespace appd
