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

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

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
  decltype(&ncclCommAbort) commAbort = nullptr;
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
  g_nccl.commAbort = (decltype(g_nccl.commAbort))dlsym(so, "ncclCommAbort");
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
  if (c->opt.host_allreduce) return APPD_OK;  // host exchange backend: no communicator
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

// a failed or timed-out collective: abort the communicator (peers blocked in it return
// with an error instead of hanging) and poison the context
static appd_status nccl_abort(appd_ctx* c, const char* why) {
  if (c->nccl_comm && g_nccl.commAbort) g_nccl.commAbort((ncclComm_t)c->nccl_comm);
  c->nccl_comm = nullptr;
  c->poisoned = true;
  appd_status s = fail(c, APPD_ERR_NCCL, "%s", why);
  c->nccl_aborted = true;
  return s;
}

// Wait for the context stream.  One rank, or the host exchange backend (whose callback
// blocks on the host): a plain synchronisation.  NCCL backend: poll the stream and the
// communicator's asynchronous error against the deadline opt.timeout_ms, so a dead or
// diverged peer ends the call with APPD_ERR_NCCL instead of a hang.
appd_status sync_stream(appd_ctx* c) {
  if (appd_status s = publish_flush(c)) return s;
  if (!c->coll || !c->nccl_comm) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    return e == cudaSuccess ? APPD_OK : cuda_fail(c, e, "cudaStreamSynchronize");
  }
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t limit_ms = c->opt.timeout_ms > 0 ? c->opt.timeout_ms : 300000;
  for (int spin = 0;; spin++) {
    cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) return APPD_OK;
    if (e != cudaErrorNotReady) return cuda_fail(c, e, "cudaStreamQuery");
    if (g_nccl.asyncError) {
      ncclResult_t ar = ncclSuccess;
      if (g_nccl.asyncError((ncclComm_t)c->nccl_comm, &ar) != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
        char msg[160];
        snprintf(msg, sizeof msg, "NCCL asynchronous error: %s", g_nccl.errorString ? g_nccl.errorString(ar) : "?");
        return nccl_abort(c, msg);
      }
    }
    const int64_t el = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (el > limit_ms) {
      char msg[160];
      snprintf(msg, sizeof msg, "collective wait exceeded timeout_ms = %lld (a peer rank is missing or diverged)",
               (long long)limit_ms);
      return nccl_abort(c, msg);
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// host exchange backend: device words -> pinned host -> user all-reduce -> device
static appd_status host_allreduce(appd_ctx* c, u64* buf, int64_t count, int op) {
  if (count <= 0) return APPD_OK;
  if ((int64_t)c->host_xchg.size() < count) c->host_xchg.resize(count);
  u64* h = c->host_xchg.data();
  APPD_CUDA(c, cudaMemcpyAsync(h, buf, sizeof(u64) * count, cudaMemcpyDeviceToHost, c->stream));
  APPD_CUDA(c, cudaStreamSynchronize(c->stream));
  const int32_t r = c->opt.host_allreduce(c->opt.host_allreduce_user, reinterpret_cast<uint64_t*>(h), count, op);
  if (r != 0) {
    c->poisoned = true;
    return fail(c, APPD_ERR_NCCL, "host_allreduce callback returned %d", (int)r);
  }
  APPD_CUDA(c, cudaMemcpyAsync(buf, h, sizeof(u64) * count, cudaMemcpyHostToDevice, c->stream));
  APPD_CUDA(c, cudaStreamSynchronize(c->stream));  // h is reused by the next exchange
  return APPD_OK;
}

static appd_status allreduce(appd_ctx* c, u64* buf, int64_t count, ncclRedOp_t op) {
  c->stats.collectives++;
  if (c->opt.host_allreduce) return host_allreduce(c, buf, count, op == ncclMin ? APPD_REDUCE_MIN : APPD_REDUCE_MAX);
  if (!c->nccl_comm) return fail(c, APPD_ERR_NCCL, "no communicator");
  ncclResult_t r = g_nccl.allReduce(buf, buf, (size_t)count, ncclUint64, op, (ncclComm_t)c->nccl_comm, c->stream);
  if (r != ncclSuccess) {
    char msg[160];
    snprintf(msg, sizeof msg, "ncclAllReduce: %s", g_nccl.errorString ? g_nccl.errorString(r) : "?");
    return nccl_abort(c, msg);
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
