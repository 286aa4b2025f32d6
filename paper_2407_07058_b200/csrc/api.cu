// api.cu -- the C ABI of libappd (include/appd.h) and the stage pipeline:
//   validate (a1) -> MST by Boruvka rounds (a2, a3; a8 exchange when world > 1)
//   -> sort the MST edge keys (a4) -> dendrogram: leaf order pi + heights h (a5)
//   -> fill prep: positions + sparse table (a6) -> fill (a7).
// Every step runs in this library's kernels on the context stream; the host
// only sequences them (and, in v1, runs the O(n) union-find dendrogram).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

using namespace appd;

namespace appd {

void* ws(appd_ctx* c, int slot, size_t bytes) {
  DevBuf& b = c->buf[slot];
  if (b.bytes >= bytes && b.p) return b.p;
  // cudaFree waits for the whole device: with NCCL collectives queued, wait on the stream
  // through the deadline-polled path first (a missing peer must not hang the free)
  if (b.p && c->coll && c->nccl_comm && sync_stream(c) != APPD_OK) return nullptr;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  size_t want = bytes < 256 ? 256 : bytes;
  want = (want + 4095) & ~(size_t)4095;
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return nullptr;
  }
  b.bytes = want;
  return b.p;
}

void* pinned_host(appd_ctx* c, size_t bytes) {
  if (c->pinned_bytes >= bytes && c->pinned) return c->pinned;
  if (c->pinned) cudaFreeHost(c->pinned);
  c->pinned = nullptr;
  c->pinned_bytes = 0;
  c->dend_pi = nullptr;
  c->dend_h = nullptr;
  c->have_dendrogram = false;
  size_t want = (bytes + 65535) & ~(size_t)65535;
  if (cudaHostAlloc(&c->pinned, want, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    c->pinned = nullptr;
    return nullptr;
  }
  c->pinned_bytes = want;
  return c->pinned;
}

appd_status fail(appd_ctx* c, appd_status s, const char* fmt, ...) {
  char msg[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof msg, fmt, ap);
  va_end(ap);
  // after an NCCL abort (deadline or asynchronous error) keep its status and message: a
  // caller reporting the failed step (e.g. a workspace growth that waited) is secondary
  if (c && c->nccl_aborted) return APPD_ERR_NCCL;
  if (c) c->last_error = msg;
  return s;
}

appd_status cuda_fail(appd_ctx* c, cudaError_t e, const char* where) {
  if (c) c->poisoned = true;
  return fail(c, APPD_ERR_CUDA, "CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
}

}  // namespace appd

static const char* kStatusNames[] = {"APPD_OK",
                                     "APPD_ERR_INVALID_ARGUMENT",
                                     "APPD_ERR_NONFINITE",
                                     "APPD_ERR_NOT_SYMMETRIC",
                                     "APPD_ERR_BAD_DIAGONAL",
                                     "APPD_ERR_UNSUPPORTED",
                                     "APPD_ERR_OUT_OF_MEMORY",
                                     "APPD_ERR_CUDA",
                                     "APPD_ERR_NCCL",
                                     "APPD_ERR_POISONED"};

extern "C" const char* appd_status_string(appd_status s) {
  if ((int)s < 0 || (int)s > 9) return "APPD_ERR_UNKNOWN";
  return kStatusNames[(int)s];
}

extern "C" const char* appd_version(void) { return "libappd 0.1 sm_100a"; }

extern "C" void appd_options_init(appd_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->struct_size = sizeof(appd_options);
  o->device = 0;
  o->rank = 0;
  o->world = 1;
  o->variant = APPD_VARIANT_AUTO;
  o->validate = 1;
  o->sense = 1;
  o->timing = 0;
  o->dendrogram = 0;
}

extern "C" appd_status appd_row_range_of(int64_t n, int32_t rank, int32_t world, int64_t* row0, int64_t* rows) {
  if (n < 1 || world < 1 || rank < 0 || rank >= world || !row0 || !rows) return APPD_ERR_INVALID_ARGUMENT;
  // blocks of 128 rows (the MST scan tile), split as evenly as possible
  int64_t blocks = (n + 127) / 128;
  int64_t b0 = blocks * rank / world, b1 = blocks * (rank + 1) / world;
  int64_t r0 = std::min(n, b0 * 128), r1 = std::min(n, b1 * 128);
  *row0 = r0;
  *rows = r1 - r0;
  return APPD_OK;
}

extern "C" appd_status appd_row_range(const appd_ctx* c, int64_t n, int64_t* row0, int64_t* rows) {
  if (!c) return APPD_ERR_INVALID_ARGUMENT;
  return appd_row_range_of(n, c->opt.rank, c->opt.world, row0, rows);
}

extern "C" appd_status appd_get_nccl_unique_id(uint8_t out[128]) {
  if (!out) return APPD_ERR_INVALID_ARGUMENT;
  std::string err;
  return nccl_unique_id(out, &err);
}

extern "C" appd_status appd_create(appd_ctx** out, const appd_options* opt) {
  if (!out) return APPD_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  appd_options o;
  appd_options_init(&o);
  if (opt) {
    if (opt->struct_size != sizeof(appd_options)) return APPD_ERR_INVALID_ARGUMENT;
    o = *opt;
  }
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return APPD_ERR_INVALID_ARGUMENT;
  if (o.sense != 1 && o.sense != -1) return APPD_ERR_INVALID_ARGUMENT;
  if (o.variant < 0 || o.variant > 2) return APPD_ERR_INVALID_ARGUMENT;
  if (o.metric < 0 || o.metric > 2) return APPD_ERR_INVALID_ARGUMENT;
  if (o.world > 1 && !o.nccl_unique_id && !o.host_allreduce) return APPD_ERR_INVALID_ARGUMENT;
  if (o.timeout_ms < 0 || o.list_cap < 0 || o.wide_keys < 0 || o.wide_keys > 1) return APPD_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return APPD_ERR_CUDA;
  }
  if (o.device < 0 || o.device >= ndev) return APPD_ERR_INVALID_ARGUMENT;
  appd_ctx* c = new appd_ctx();
  c->opt = o;
  c->device = o.device;
  // world 1 with an explicit communicator or host exchange runs the multi-rank path over
  // one rank (the transport exercised on one GPU; results equal the world-1 path's)
  c->coll = o.world > 1 || o.nccl_unique_id != nullptr || o.host_allreduce != nullptr;
  std::memset(&c->stats, 0, sizeof c->stats);
  c->stats.struct_size = sizeof(appd_stats);
  if (cudaSetDevice(c->device) != cudaSuccess) {
    delete c;
    return APPD_ERR_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) == cudaSuccess) c->sm_count = prop.multiProcessorCount;
  if (prop.major < 10) {
    delete c;
    return APPD_ERR_UNSUPPORTED;  // built for sm_100a only
  }
  if (o.cuda_stream) {
    c->stream = (cudaStream_t)o.cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return APPD_ERR_CUDA;
    }
    c->own_stream = true;
  }
  for (int i = 0; i < 16; i++) cudaEventCreate(&c->ev[i]);
  c->ev_ready = true;
  if (c->coll && cudaHostAlloc((void**)&c->pinned_xchg, 32 * sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    appd_destroy(c);
    return APPD_ERR_OUT_OF_MEMORY;
  }
  if (cudaHostAlloc((void**)&c->pinned_small, 64 * sizeof(unsigned), cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    appd_destroy(c);
    return APPD_ERR_OUT_OF_MEMORY;
  }
  if (cudaHostGetDevicePointer((void**)&c->pinned_small_dev, c->pinned_small, 0) != cudaSuccess) {
    cudaGetLastError();
    c->pinned_small_dev = nullptr;  // publish() falls back to copies
  }
  if (c->coll) {
    appd_status s = nccl_init(c, o.nccl_unique_id, o.rank, o.world);
    if (s != APPD_OK) {
      appd_destroy(c);
      return s;
    }
  }
  *out = c;
  return APPD_OK;
}

extern "C" appd_status appd_set_stream(appd_ctx* c, void* stream) {
  if (!c) return APPD_ERR_INVALID_ARGUMENT;
  if (c->poisoned) return APPD_ERR_POISONED;
  cudaSetDevice(c->device);
  if (stream) {
    if (c->own_stream) cudaStreamDestroy(c->stream);
    c->own_stream = false;
    c->stream = (cudaStream_t)stream;
  } else if (!c->own_stream) {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return APPD_ERR_CUDA;
    c->own_stream = true;
  }
  return APPD_OK;
}

namespace appd {
unsigned* grid_barrier_word(appd_ctx* c) {
  if (!c->gridbar) {
    if (cudaMalloc(&c->gridbar, 64) != cudaSuccess) {
      c->gridbar = nullptr;
      return nullptr;
    }
    if (cudaMemsetAsync(c->gridbar, 0, 64, c->stream) != cudaSuccess) return nullptr;
  }
  return c->gridbar;
}
}  // namespace appd

extern "C" void appd_destroy(appd_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  nccl_destroy(c);
  if (c->gridbar) cudaFree(c->gridbar);
  for (auto& b : c->buf)
    if (b.p) cudaFree(b.p);
  if (c->ev_ready)
    for (int i = 0; i < 16; i++) cudaEventDestroy(c->ev[i]);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->sev_ready)
    for (int i = 0; i < 4; i++) cudaEventDestroy(c->sev[i]);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->pinned_small) cudaFreeHost(c->pinned_small);
  if (c->pinned_xchg) cudaFreeHost(c->pinned_xchg);
  if (c->sink_host) cudaFreeHost(c->sink_host);
  cudaGetLastError();
  delete c;
}

extern "C" const char* appd_last_error(const appd_ctx* c) { return c ? c->last_error.c_str() : ""; }

extern "C" appd_status appd_error_index(const appd_ctx* c, int64_t* i, int64_t* j) {
  if (!c || !i || !j) return APPD_ERR_INVALID_ARGUMENT;
  *i = c->err_i;
  *j = c->err_j;
  return APPD_OK;
}

extern "C" appd_status appd_get_stats(const appd_ctx* c, appd_stats* s) {
  if (!c || !s || s->struct_size != sizeof(appd_stats)) return APPD_ERR_INVALID_ARGUMENT;
  *s = c->stats;
  return APPD_OK;
}

extern "C" appd_status appd_last_dendrogram(const appd_ctx* c, int32_t* pi, float* h, int64_t n) {
  if (!c || !c->have_dendrogram || c->dend_n != n) return APPD_ERR_INVALID_ARGUMENT;
  if (c->dend_on_device && n > 1) {  // GPU dendrogram: the last solve's device buffers
    cudaSetDevice(c->device);
    if (pi && cudaMemcpy(pi, c->dend_pi, sizeof(int32_t) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
      return APPD_ERR_CUDA;
    if (h && cudaMemcpy(h, c->dend_h, sizeof(float) * (n - 1), cudaMemcpyDeviceToHost) != cudaSuccess)
      return APPD_ERR_CUDA;
    return APPD_OK;
  }
  if (pi) std::memcpy(pi, c->dend_pi, sizeof(int32_t) * n);
  if (h && n > 1) std::memcpy(h, c->dend_h, sizeof(float) * (n - 1));
  return APPD_OK;
}

// ---------------------------------------------------------------------------
static appd_status check_device_ptr(appd_ctx* c, const void* p, const char* name) {
  if (!p) return fail(c, APPD_ERR_INVALID_ARGUMENT, "%s is NULL", name);
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, APPD_ERR_INVALID_ARGUMENT, "%s is not a CUDA pointer", name);
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(c, APPD_ERR_INVALID_ARGUMENT, "%s is not device memory", name);
  if (a.device != c->device) return fail(c, APPD_ERR_INVALID_ARGUMENT, "%s is on another device", name);
  return APPD_OK;
}

// Stage boundaries: CUDA events (timing) and NVTX ranges "appd:<stage>" (header-only
// NVTX3: no cost unless a profiler attaches; SURVEY §5 tracing)
static const char* kStageNames[6] = {"appd:validate", "appd:mst", "appd:sort", "appd:dendrogram", "appd:prep",
                                     "appd:fill"};
static inline void stage_event(appd_ctx* c, int idx) {
  if (c->opt.timing) cudaEventRecord(c->ev[idx], c->stream);
  if (c->nvtx_stage) nvtxRangeEnd(c->nvtx_stage);
  c->nvtx_stage = idx < 6 ? nvtxRangeStartA(kStageNames[idx]) : 0;
}
static inline void nvtx_close(appd_ctx* c) {
  if (c->nvtx_stage) nvtxRangeEnd(c->nvtx_stage);
  c->nvtx_stage = 0;
}



static float ev_ms(appd_ctx* c, int a, int b) {
  float ms = 0.0f;
  if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) {
    cudaGetLastError();
    return 0.0f;
  }
  return ms;
}

// map the three first-offender indices to a status.  Priority: any non-finite
// value first (its first occurrence in row-major order), then the first bad
// diagonal entry, then the first asymmetric pair (i < j).
static appd_status report_validation(appd_ctx* c, const u64 bad[3], int64_t n, bool points, int64_t d) {
  int which = -1;
  for (int t = 0; t < 3 && which < 0; t++)
    if (bad[t] != KEY_NONE) which = t;
  if (which < 0) return APPD_OK;
  u64 best = bad[which];
  int64_t w = points ? d : n;
  c->err_i = (int64_t)(best / (u64)w);
  c->err_j = (int64_t)(best % (u64)w);
  if (which == 0)
    return fail(c, APPD_ERR_NONFINITE, "non-finite %s at (%lld, %lld)", points ? "coordinate" : "weight",
                (long long)c->err_i, (long long)c->err_j);
  if (which == 1)
    return fail(c, APPD_ERR_BAD_DIAGONAL, "nonzero diagonal W[%lld][%lld]", (long long)c->err_i, (long long)c->err_j);
  return fail(c, APPD_ERR_NOT_SYMMETRIC, "W[%lld][%lld] != W[%lld][%lld]", (long long)c->err_i,
              (long long)c->err_j, (long long)c->err_j, (long long)c->err_i);
}

// world > 1: every rank must enter the solve with the same problem, or the ranks would
// take different branches and hang in a later collective.  One all-reduce
// (min) over the words v and ~v: v agrees on every rank iff min(v) == v and min(~v) == ~v.
static appd_status agree(appd_ctx* c, const float* X, int64_t n, int64_t d, int mode) {
  constexpr int NW = 7;
  u64 v[NW];
  v[0] = (u64)n;
  v[1] = (u64)d;
  v[2] = (u64)mode | (u64)(c->stream_out ? 1 : 0) << 8 | (u64)(c->sink ? 1 : 0) << 9 |
         (u64)(uint32_t)c->opt.world << 32;
  v[3] = (u64)(c->opt.sense + 1) | (u64)(c->opt.validate & 15) << 4 | (u64)(c->opt.metric & 15) << 8 |
         (u64)(c->opt.points_engine & 15) << 12 | (u64)(c->opt.dendrogram & 15) << 16 |
         (u64)(c->opt.variant & 15) << 20;
  v[4] = (u64)(uint32_t)c->opt.topk | (u64)(uint32_t)c->opt.finish_k << 32;
  v[5] = 0;
  v[6] = (u64)(uint32_t)c->opt.list_cap | (u64)(uint32_t)c->opt.wide_keys << 32;
  u64* dv = (u64*)ws(c, S_TMP, sizeof(u64) * 2 * NW);
  if (!dv) return fail(c, APPD_ERR_OUT_OF_MEMORY, "agreement buffer");
  if (X) {  // points mode: X is replicated, so its checksum must agree too
    appd_status s = launch_checksum_words(c, X, n * d, dv);
    if (s) return s;
    APPD_CUDA(c, cudaMemcpyAsync(c->pinned_xchg, dv, sizeof(u64), cudaMemcpyDeviceToHost, c->stream));
    APPD_SYNC(c);
    v[5] = c->pinned_xchg[0];
  }
  u64* h = c->pinned_xchg;  // 2 NW <= 32 pinned words: the copies stay inside the polled waits
  for (int i = 0; i < NW; i++) {
    h[i] = v[i];
    h[NW + i] = ~v[i];
  }
  APPD_CUDA(c, cudaMemcpyAsync(dv, h, sizeof(u64) * 2 * NW, cudaMemcpyHostToDevice, c->stream));
  appd_status s = nccl_allreduce_min_u64(c, dv, 2 * NW);
  if (s) return s;
  APPD_CUDA(c, cudaMemcpyAsync(h, dv, sizeof(u64) * 2 * NW, cudaMemcpyDeviceToHost, c->stream));
  APPD_SYNC(c);
  static const char* what[NW] = {"n", "d", "entry point / world", "options (sense, validate, metric, engine, dendrogram, variant)",
                                 "options (topk, finish_k)", "the checksum of X", "options (list_cap)"};
  for (int i = 0; i < NW; i++)
    if (h[i] != v[i] || h[NW + i] != ~v[i])
      return fail(c, APPD_ERR_INVALID_ARGUMENT, "ranks disagree on %s at solve start (this rank %llu)", what[i],
                  (unsigned long long)v[i]);
  return APPD_OK;
}

#ifdef APPD_DEV_HOOKS
// development builds, APPD_CHECK=1: the MST edges must form a spanning tree and pi must be
// a permutation (reported to stderr with the stage; the solve continues)
static void dev_check(appd_ctx* c, const char* what, const int32_t* d_eu, const int32_t* d_ev, int64_t m,
                      const int* d_pi, int64_t n) {
  static const bool on = dev_env("APPD_CHECK") != nullptr;
  if (!on) return;
  cudaStreamSynchronize(c->stream);
  std::vector<int32_t> eu(m), ev(m), pi(n);
  if (d_eu) {
    cudaMemcpy(eu.data(), d_eu, 4 * m, cudaMemcpyDeviceToHost);
    cudaMemcpy(ev.data(), d_ev, 4 * m, cudaMemcpyDeviceToHost);
    std::vector<int32_t> p(n);
    for (int64_t i = 0; i < n; i++) p[i] = (int32_t)i;
    auto find = [&](int32_t x) { while (p[x] != x) x = p[x] = p[p[x]]; return x; };
    int64_t bad = 0;
    for (int64_t e = 0; e < m; e++) {
      if (eu[e] < 0 || eu[e] >= n || ev[e] < 0 || ev[e] >= n) { bad++; continue; }
      int32_t a = find(eu[e]), b = find(ev[e]);
      if (a == b) bad++; else p[a] = b;
    }
    if (bad) fprintf(stderr, "[appd check] rank %d %s: %lld bad MST edges (n %lld)\n", c->opt.rank, what, (long long)bad, (long long)n);
  }
  if (d_pi) {
    cudaMemcpy(pi.data(), d_pi, 4 * n, cudaMemcpyDeviceToHost);
    std::vector<char> seen(n, 0);
    int64_t bad = 0;
    for (int64_t i = 0; i < n; i++) {
      if (pi[i] < 0 || pi[i] >= n || seen[pi[i]]) bad++; else seen[pi[i]] = 1;
    }
    if (bad) fprintf(stderr, "[appd check] rank %d %s: pi is not a permutation (%lld bad)\n", c->opt.rank, what, (long long)bad);
  }
}
#endif

// points mode: up to kMaxPackedPoints the edge key packs bits(d2) (31) and the pair index
// (33) into 64 bits; above it (NEXT-4, outputs beyond HBM) the wide-key path; the upper
// bound keeps every index an int32 and the pair index below 2^40
constexpr int64_t kMaxPackedPoints = 131072, kMaxPoints = 1 << 20;
constexpr int64_t kExactEngineMaxN = 2048;  // AUTO: exact FP32 engine up to here (measured)

// ---------------------------------------------------------------------------
// The Prim variant (k_prim.cu): one single-CTA launch validates the
// input, runs Prim's n - 1 steps and writes (pi, h) with the fill's preparation; the fill
// follows.  AUTO takes it below the measured crossover with Boruvka (DESIGN.md §5,
// profiles/r02/crossover.txt); it needs the whole input, so sharded weights (world > 1)
// and the streamed output always take Boruvka; points with world > 1 run it replicated.
// measured (profiles/r02/crossover.txt, whole solves): weights -- Prim wins at every n it
// fits (n <= 300: 0.08-0.14 ms against 0.32-0.39 ms); points -- Prim wins while one SM's
// O(n^2 d) distance work stays small: n = 1024 at d = 2 (0.46 vs 0.68 ms), n = 256 at
// d = 16 and d = 64, and loses at n = 2048 (d = 2), n = 1024 (d = 16), n = 512 (d = 64)
constexpr int64_t kPrimAutoMaxWeights = 300;
constexpr int64_t kPrimAutoMaxPoints = 1024, kPrimAutoMaxPointWork = 20480;  // n * (d + 8)

static bool prim_requested(const appd_ctx* c) { return c->opt.variant == APPD_VARIANT_PRIM; }

static bool want_prim(const appd_ctx* c, int64_t n, int64_t d, bool points, bool f64) {
  if (f64 || c->stream_out || c->sink || n < 2 || c->opt.wide_keys == 1) return false;
  if (!points && c->coll) return false;
  if (!prim_fits(n, d, points)) return false;
  if (prim_requested(c)) return true;
  if (c->opt.variant != APPD_VARIANT_AUTO) return false;
  if (points && c->opt.points_engine != 0) return false;
  if (!points) return n <= kPrimAutoMaxWeights;
  return n <= kPrimAutoMaxPoints && n * (d + 8) <= kPrimAutoMaxPointWork;
}

static appd_status solve_prim(appd_ctx* c, const float* W, const float* X, int64_t n, int64_t d, float* M) {
  const bool points = X != nullptr;
  const int sense = c->opt.sense;  // points too: widest paths on the exact engine or Prim
  int64_t row0, rows;
  appd_row_range_of(n, c->opt.rank, c->opt.world, &row0, &rows);
  c->stats.variant = APPD_VARIANT_PRIM;
  c->stats.dendrogram = 0;
  const int64_t m = n - 1;
  int levels = 1;
  while ((1ll << levels) <= m) levels++;
  int* pi = (int*)ws(c, S_PI, sizeof(int) * n);
  int* pos = (int*)ws(c, S_POS, sizeof(int) * n);
  int* rowpos = (int*)ws(c, S_ROWPOS, sizeof(int) * n);
  float* ST = (float*)ws(c, S_ST, sizeof(float) * m * levels);
  if (!pi || !pos || !rowpos || !ST) return fail(c, APPD_ERR_OUT_OF_MEMORY, "Prim workspace (n = %lld)", (long long)n);
  u64* bad = nullptr;
  u64* hbad = reinterpret_cast<u64*>(c->pinned_small + 40);
  if (c->opt.validate) {
    bad = (u64*)ws(c, S_VALID, 3 * sizeof(u64));
    if (!bad) return fail(c, APPD_ERR_OUT_OF_MEMORY, "validation buffer");
    APPD_CUDA(c, cudaMemsetAsync(bad, 0xFF, 3 * sizeof(u64), c->stream));
  }
  stage_event(c, 1);
  // small n: the same launch also fills M (prim_fuses_fill); rows == 0: nothing to fill
  const bool fused = prim_fuses_fill(n) && rows > 0;
  appd_status s = launch_prim(c, W, X, n, d, sense, points ? c->opt.metric : 0, bad, pi, pos, rowpos, ST, m, levels,
                              fused ? M : nullptr, row0, rows);
  if (s) return s;
  if (bad) APPD_PUBLISH(c, hbad, bad, 3 * sizeof(u64));
  for (int e = 2; e <= 4; e++) stage_event(c, e);
  const int* rows_sorted = pi;
  if (c->coll && !fused) {  // replicated Prim, this rank's rows in leaf order
    int* keys = (int*)ws(c, S_TMP, sizeof(int) * 2 * (rows + 1));
    int* rs = (int*)ws(c, S_ROWS_SORTED, sizeof(int) * (rows + 1));
    if (!keys || !rs) return fail(c, APPD_ERR_OUT_OF_MEMORY, "fill workspace");
    if ((s = launch_gather_rowpos(c, pos, row0, rows, keys, keys + rows + 1))) return s;
    if ((s = sort_pairs_i32(c, keys, rowpos, keys + rows + 1, rs, rows))) return s;
    rows_sorted = rs;
  }
  stage_event(c, 5);
  if (!fused && (s = launch_fill(c, rows_sorted, rowpos, rows, pos, ST, m, n, M, row0, sense < 0))) return s;
  stage_event(c, 6);
  APPD_SYNC(c);
  if (bad) {
    u64 hb[3];
    memcpy(hb, hbad, sizeof hb);
    if ((s = report_validation(c, hb, n, points, d))) return s;
  }
  c->dend_pi = pi;
  c->dend_h = ST;
  c->dend_on_device = true;
  c->dend_n = n;
  c->have_dendrogram = true;
  c->stats.rounds = 0;
  c->stats.fill_bytes = rows * n * 4;
  c->stats.kernel_launches = c->launches;
  if (c->opt.timing) {
    c->stats.ms_validate = ev_ms(c, 0, 1);
    c->stats.ms_mst = ev_ms(c, 1, 2);
    c->stats.ms_sort = ev_ms(c, 2, 3);
    c->stats.ms_dendrogram = ev_ms(c, 3, 4);
    c->stats.ms_prep = ev_ms(c, 4, 5);
    c->stats.ms_fill = ev_ms(c, 5, 6);
    c->stats.ms_total = ev_ms(c, 0, 6);
  }
  return APPD_OK;
}

static appd_status solve_impl(appd_ctx* c, const float* W, const float* X, int64_t n, int64_t d, float* M);

#ifdef APPD_DEV_HOOKS
namespace appd {
namespace {
struct TraceState {
  bool on = dev_env("APPD_TRACE") != nullptr;
  int depth = 0, used = 0;
  cudaEvent_t ev[1024];
  const char* site[1024];
  double host_us[1024];
  std::chrono::steady_clock::time_point t0;
};
TraceState& trace_state() {
  static TraceState t;
  return t;
}
}  // namespace
void trace_begin(appd_ctx* c) {
  TraceState& t = trace_state();
  if (!t.on || t.depth++) return;
  t.used = 0;
  t.t0 = std::chrono::steady_clock::now();
  trace_launch(c, "solve begin");
}
void trace_launch(appd_ctx* c, const char* site) {
  TraceState& t = trace_state();
  if (!t.on || t.used >= 1024) return;
  if (!t.ev[t.used]) cudaEventCreate(&t.ev[t.used]);
  cudaEventRecord(t.ev[t.used], c->stream);
  t.site[t.used] = site;
  t.host_us[t.used] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t.t0).count();
  t.used++;
}
void trace_end(appd_ctx* c) {
  TraceState& t = trace_state();
  if (!t.on || --t.depth) return;
  trace_launch(c, "solve end");
  cudaStreamSynchronize(c->stream);
  const char* base;
  for (int i = 0; i < t.used; i++) {
    float ms = 0.0f, ms0 = 0.0f;
    if (i) cudaEventElapsedTime(&ms, t.ev[i - 1], t.ev[i]);
    cudaEventElapsedTime(&ms0, t.ev[0], t.ev[i]);
    base = strrchr(t.site[i], '/');
    fprintf(stderr, "[trace] %3d host %8.1f us  gpu %8.1f us  +%7.1f us  %s\n", i, t.host_us[i], 1e3 * ms0, 1e3 * ms,
            base ? base + 1 : t.site[i]);
  }
  cudaGetLastError();
}
}  // namespace appd
#endif

// The whole pipeline (one NVTX range per call, one per stage inside)
static appd_status solve(appd_ctx* c, const float* W, const float* X, int64_t n, int64_t d, float* M) {
  nvtxRangePushA(X ? "appd_solve_points" : "appd_solve_weights");
#ifdef APPD_DEV_HOOKS
  trace_begin(c);
#endif
  const appd_status s = solve_impl(c, W, X, n, d, M);
  if (s != APPD_OK) c->npub = 0;  // queued publications of a failed solve are dropped
#ifdef APPD_DEV_HOOKS
  trace_end(c);
#endif
  nvtx_close(c);
  nvtxRangePop();
  return s;
}

// X (points) or W (weights) is a device pointer.
static appd_status solve_impl(appd_ctx* c, const float* W, const float* X, int64_t n, int64_t d, float* M) {
  const bool points = X != nullptr;
  const bool f64 = c->f64_W != nullptr;  // NEXT-3 (k_f64.cu): W and M are c->f64_W / c->f64_M
  const int sense = c->opt.sense;  // points too: widest paths on the exact engine or Prim
  int64_t row0, rows;
  appd_row_range_of(n, c->opt.rank, c->opt.world, &row0, &rows);
  std::memset(&c->stats, 0, sizeof c->stats);
  c->stats.struct_size = sizeof(appd_stats);
  c->stats.n = n;
  c->stats.d = points ? d : 0;
  c->stats.row0 = row0;
  c->stats.rows = rows;
  c->stats.variant = APPD_VARIANT_BORUVKA;
  c->launches = 0;
  c->have_dendrogram = false;
  c->err_i = c->err_j = -1;
  c->last_error.clear();
  host_mark("solve entry", true);
  if (c->coll) {
    appd_status sa = agree(c, X, n, points ? d : 0, points ? 2 : (f64 ? 3 : 1));
    if (sa) return sa;
  }
  stage_event(c, 0);
  if (n >= 2 && !f64 && want_prim(c, n, d, points, f64)) return solve_prim(c, W, X, n, d, M);
  if (prim_requested(c) && n >= 2)
    return fail(c, APPD_ERR_UNSUPPORTED,
                "variant PRIM: n = %lld does not fit one CTA (weights n <= 300; points n <= 2048 and n * (d + 3) "
                "words <= 56K), or the call needs the whole input (sharded weights, streamed output, fp64)",
                (long long)n);

  // ---- a1: validation ----
  // Points mode with the tensor-core engine: the verdict is copied asynchronously and
  // read after the engine's preparation, which synchronises anyway (deferred check).
  if (points && c->opt.metric != 0 && c->opt.points_engine == 2)
    return fail(c, APPD_ERR_UNSUPPORTED, "the tensor-core engine computes Euclidean distances only (metric = %d)",
                c->opt.metric);
  if (points && sense < 0 && c->opt.points_engine == 2)
    return fail(c, APPD_ERR_UNSUPPORTED, "the tensor-core engine finds minimum edges only (widest sense: exact engine)");
  const bool defer_validation = points && c->opt.validate && !c->coll && c->opt.points_engine != 1 &&
                                (c->opt.points_engine == 2 || n > kExactEngineMaxN) && c->opt.metric == 0 &&
                                sense > 0 && n >= 2 && n <= kMaxPackedPoints && c->opt.wide_keys != 1;
  u64* hbad = reinterpret_cast<u64*>(c->pinned_small + 40);  // 3 words, pinned
  u64* vbad = nullptr;
  if (c->opt.validate) {
    vbad = (u64*)ws(c, S_VALID, 3 * sizeof(u64));
    if (!vbad) return fail(c, APPD_ERR_OUT_OF_MEMORY, "validation buffer");
  }
  auto launch_validation = [&]() -> appd_status {
    APPD_CUDA(c, cudaMemsetAsync(vbad, 0xFF, 3 * sizeof(u64), c->stream));
    appd_status s = points ? launch_validate_points(c, X, n, d, vbad)
                    : f64  ? launch_validate_weights_f64(c, c->f64_W, n, vbad)
                           : launch_validate_weights(c, W, n, row0, rows, vbad);
    if (s) return s;
    APPD_PUBLISH(c, hbad, vbad, 3 * sizeof(u64));
    return APPD_OK;
  };
  // deferred: the tensor-core preparation validates the points itself (one launch)
  if (c->opt.validate && !defer_validation) {
    appd_status s = launch_validation();
    if (s) return s;
  }
  if (c->opt.validate && !defer_validation) {
    appd_status s;
    u64 hb[3];
    APPD_SYNC(c);
    memcpy(hb, hbad, sizeof hb);
    if (c->coll) {
      // every rank must agree on the verdict (else the others would hang in the next collective)
      u64* agree = (u64*)ws(c, S_TMP, sizeof(u64) * 3);
      if (!agree) return fail(c, APPD_ERR_OUT_OF_MEMORY, "validation buffer");
      u64* hx = c->pinned_xchg;
      memcpy(hx, hb, sizeof hb);
      APPD_CUDA(c, cudaMemcpyAsync(agree, hx, sizeof hb, cudaMemcpyHostToDevice, c->stream));
      if ((s = nccl_allreduce_min_u64(c, agree, 3))) return s;
      APPD_CUDA(c, cudaMemcpyAsync(hx, agree, sizeof hb, cudaMemcpyDeviceToHost, c->stream));
      APPD_SYNC(c);
      memcpy(hb, hx, sizeof hb);
    }
    if ((s = report_validation(c, hb, n, points, d))) return s;
  }
  stage_event(c, 1);
  host_mark("validation queued");

  if (n == 1) {
    if (c->stream_out) {
      APPD_SYNC(c);
      c->stream_out[0] = 0.0f;
    } else if (c->sink) {
      APPD_SYNC(c);
      const float zero = 0.0f;
      if (c->sink(c->sink_user, 0, 1, &zero) != 0) return fail(c, APPD_ERR_INVALID_ARGUMENT, "sink returned non-zero");
    } else if (rows > 0) {
      appd_status s = f64 ? launch_set_diag_zero_single_f64(c, c->f64_M) : launch_set_diag_zero_single(c, M);
      if (s) return s;
    }
    APPD_SYNC(c);
    c->one_pi = 0;
    c->dend_on_device = false;
    c->dend_pi = &c->one_pi;
    c->dend_h = nullptr;
    c->dend_n = 1;
    c->have_dendrogram = true;
    c->stats.kernel_launches = c->launches;
    return APPD_OK;
  }

  // ---- a2/a3: MST by Boruvka rounds ----
  // wide keys (points, n > 131072): the pair index needs more than the 33 bits beside the
  // weight; the exact engine with a two-step component reduction (k_boruvka.cu)
  const bool wide = points && (n > kMaxPackedPoints || c->opt.wide_keys == 1);
  KeySpec ks;
  ks.points = points;
  ks.shift = wide ? 63 : points ? 33 : 32;
  ks.sense = sense;
  ks.metric = points ? c->opt.metric : 0;
  int* comp = (int*)ws(c, S_COMP, sizeof(int) * n);
  u64* compbest = (u64*)ws(c, S_COMPBEST, sizeof(u64) * n);
  int* link = (int*)ws(c, S_LINK, sizeof(int) * n);
  int* parent = (int*)ws(c, S_PARENT, sizeof(int) * n);
  int* newid = (int*)ws(c, S_NEWID, sizeof(int) * (n + 1));
  int* flags = (int*)ws(c, S_FLAGS, sizeof(int) * (n + 1));
  u64* mstkeys = (u64*)ws(c, S_MSTKEYS, sizeof(u64) * n);
  u64* sorted = (u64*)ws(c, S_MSTKEYS_SORTED, sizeof(u64) * n);
  int* counters = (int*)ws(c, S_COUNTERS, sizeof(int) * 16);
  if (!comp || !compbest || !link || !parent || !newid || !flags || !mstkeys || !sorted || !counters)
    return fail(c, APPD_ERR_OUT_OF_MEMORY, "MST workspace (n = %lld)", (long long)n);
  float* XT = nullptr;
  int64_t npad = 0, dpad = 0;
  appd_status s;
  // points mode: tensor-core filter (engine 2) unless the exact engine is requested or
  // the dimension does not fit the shared-memory ring
  TcState tc;
  bool use_tc = false;
  // AUTO engine: the tensor-core filter pays off above ~2048 points; below, the symmetric
  // exact pass wins (measured, tools/engine_cmp.py: n = 2048, d = 2 / 64: 0.55 / 0.54 ms
  // exact against 0.64 / 0.64 ms tensor core; n = 4096, d = 2: 0.96 against 0.87 ms)
  const bool tc_wanted = c->opt.points_engine == 2 || (c->opt.points_engine == 0 && n > kExactEngineMaxN);
  if (points && !wide && sense > 0 && tc_wanted && c->opt.metric == 0 && n >= 2) {
    // the round state's initialisation rides on the preparation's launch
    InitList init;
    init.add(comp, n, 0, 2);
    init.add(counters, 16, 0, 0);
    init.add(compbest, n, KEY_NONE, 1);
    // no synchronisation: scale and verdict are read later
    s = tcf_prepare(c, X, n, d, &tc, &init, defer_validation ? vbad : nullptr);
    host_mark("tcf_prepare queued");
    if (s == APPD_OK) {
      use_tc = true;
      if (defer_validation) APPD_PUBLISH(c, hbad, vbad, 3 * sizeof(u64));
    } else {
      if (defer_validation) {  // the verdict decides before any fallback
        if (appd_status sl = launch_validation()) return sl;
        APPD_SYNC(c);
        u64 hb[3];
        memcpy(hb, hbad, sizeof hb);
        appd_status sv = report_validation(c, hb, n, points, d);
        if (sv) return sv;
      }
      if (s != APPD_ERR_UNSUPPORTED || c->opt.points_engine == 2) return s;
    }
    c->last_error.clear();
  }
  // read at the first synchronisation of the round loop
  bool check_first_sync = use_tc;
  c->stats.points_engine = points ? (use_tc ? 2 : 1) : 0;
  int64_t rt_begin = 0, rt_end = 0;
  if (use_tc) {
    const int64_t T = tcf_row_tiles(&tc);
    rt_begin = T * c->opt.rank / c->opt.world;
    rt_end = T * (c->opt.rank + 1) / c->opt.world;
  }
  auto ensure_xt = [&]() -> appd_status {
    if (XT) return APPD_OK;
    npad = (n + 127) / 128 * 128;
    dpad = (d + 31) / 32 * 32;
    XT = (float*)ws(c, S_XT, sizeof(float) * npad * dpad);
    if (!XT) return fail(c, APPD_ERR_OUT_OF_MEMORY, "XT workspace");
    return launch_transpose_points(c, X, n, d, XT, npad, dpad);
  };
  if (points && !use_tc && (s = ensure_xt())) return s;
  if (!use_tc) {  // (the tensor-core preparation initialised these)
    if ((s = launch_iota(c, comp, n))) return s;
    APPD_CUDA(c, cudaMemsetAsync(counters, 0, sizeof(int) * 16, c->stream));
  }
  int64_t k = n;
  int rounds = 0;
  int* hostk = reinterpret_cast<int*>(c->pinned_small + 24);  // pinned: the copies stay asynchronous
  // weights mode: round-0 candidate cache (exact per-row top-K of W)
  const int wtopk = (points || f64) ? 0 : (c->opt.topk == 0 ? 8 : (c->opt.topk < 0 ? 0 : c->opt.topk));
  u64 *f64_compw = nullptr, *f64_roww = nullptr;
  int* f64_rowj = nullptr;
  if (f64) {
    f64_compw = (u64*)ws(c, S_F64_A, sizeof(u64) * 2 * n);
    f64_roww = f64_compw ? f64_compw + n : nullptr;
    f64_rowj = (int*)ws(c, S_F64_B, sizeof(int) * n);
    if (!f64_compw || !f64_rowj) return fail(c, APPD_ERR_OUT_OF_MEMORY, "fp64 round workspace");
  }
  if (wtopk && wtopk != 4 && wtopk != 8 && wtopk != 16 && wtopk != 32)
    return fail(c, APPD_ERR_INVALID_ARGUMENT, "topk = %d (0, -1, 4, 8, 16 or 32)", c->opt.topk);
  u64* w_ckey = nullptr;
  int *w_cj = nullptr, *w_ccnt = nullptr, *w_need = nullptr, *w_list = nullptr;
  unsigned* w_count = nullptr;
  bool w_pending = false;
  if (wtopk) {
    w_ckey = (u64*)ws(c, S_TC_CKEY, sizeof(u64) * n * wtopk);
    w_cj = (int*)ws(c, S_TC_CJ, sizeof(int) * n * wtopk);
    w_ccnt = (int*)ws(c, S_TC_CCNT, sizeof(int) * n);
    w_need = (int*)ws(c, S_TC_NEED, sizeof(int) * n);
    w_list = (int*)ws(c, S_TC_ROWLIST, sizeof(int) * (n + 1));
    w_count = (unsigned*)ws(c, S_TC_CNT, 64);
    if (!w_ckey || !w_cj || !w_ccnt || !w_need || !w_list || !w_count)
      return fail(c, APPD_ERR_OUT_OF_MEMORY, "weights candidate cache");
  }
  auto w_lookup_async = [&]() -> appd_status {
    APPD_CUDA(c, cudaMemsetAsync(w_count, 0, 64, c->stream));
    appd_status s2 = launch_cache_lookup(c, (int)row0, (int)(row0 + rows), wtopk, (int)n, w_ckey, w_cj, w_ccnt, comp,
                                         compbest, w_need, w_count, w_list);
    if (s2) return s2;
    APPD_PUBLISH(c, c->pinned_small + 9, w_count, sizeof(unsigned));
    w_pending = true;
    return APPD_OK;
  };
  const int finish_k = c->opt.finish_k == 0 ? 128 : std::min(c->opt.finish_k, 128);
  bool cm_timing_pending = false, cm_status_pending = false;
  c->pinned_small[48] = 0;
  while (k > 1) {
    // ---- component-matrix finish: the contracted k-node graph's exact edge keys ----
    if (use_tc && tc.topk && rounds > 0 && finish_k > 0 && k <= finish_k) {
      tc.lookup_pending = false;  // the component matrix replaces the queued lookup
      u64* WCM = (u64*)ws(c, S_TC_WCM, sizeof(u64) * k * k);
      if (!WCM) return fail(c, APPD_ERR_OUT_OF_MEMORY, "component matrix");
      bool ovf = false;
      if (c->opt.timing >= 2) cudaEventRecord(c->ev[8], c->stream);
      if ((s = tcf_cm(c, &tc, X, comp, k, WCM, rt_begin, rt_end, &ovf, c->coll))) return s;
      if (c->coll) {  // every rank must take the same branch
        u64* flag = (u64*)ws(c, S_TMP, sizeof(u64));
        if (!flag) return fail(c, APPD_ERR_OUT_OF_MEMORY, "flag");
        u64* hx = c->pinned_xchg;
        hx[0] = ovf ? 1 : 0;
        APPD_CUDA(c, cudaMemcpyAsync(flag, hx, sizeof(u64), cudaMemcpyHostToDevice, c->stream));
        if ((s = nccl_allreduce_max_u64(c, flag, 1))) return s;
        APPD_CUDA(c, cudaMemcpyAsync(hx, flag, sizeof(u64), cudaMemcpyDeviceToHost, c->stream));
        APPD_SYNC(c);
        ovf = hx[0] != 0;
        if (!ovf && (s = nccl_allreduce_min_u64(c, WCM, k * k))) return s;
      }
      if (!ovf) {
        // Prim on the contracted graph on the device (keys are a strict order: the MST is
        // unique); its k - 1 edges are appended to mstkeys, the count checked at the end
        // (one rank: a listing overflow is detected on the device, read at the end)
        unsigned* cm_status = reinterpret_cast<unsigned*>(counters + 4);
        if ((s = launch_cm_prim(c, WCM, (int)k, mstkeys, counters, tc.counters + 1, tc.list_entries_cap, tc.cstart,
                                tc.perm, cm_status)))
          return s;
        APPD_PUBLISH(c, c->pinned_small + 48, cm_status, sizeof(unsigned));
        cm_status_pending = true;
        if (c->opt.timing >= 2) cudaEventRecord(c->ev[9], c->stream);
        cm_timing_pending = c->opt.timing != 0;  // read after the final synchronisation
        c->stats.cm_k = (int)k;
        c->stats.tcscan_launches++;
        if (!c->coll) {  // upper-triangle pass: row block rb against columns >= 512 rb
          double pairs = 0.0;
          for (int64_t rb = 0; rb * 512 < n; rb++) pairs += (double)std::min<int64_t>(512, n - rb * 512) * (n - rb * 512);
          c->stats.tcscan_flops += 2.0 * pairs * d;
        } else {
          c->stats.tcscan_flops += 2.0 * (double)(std::min<int64_t>(rt_end * 512, n) - rt_begin * 512) * n * d;
        }
        if (dev_env("APPD_DEBUG_ROUNDS"))
          fprintf(stderr, "[appd] component-matrix finish at k %lld (listing count checked at the end)\n", (long long)k);
        rounds++;
        k = 1;
        break;
      }
    }
    static const bool dbg = dev_env("APPD_DEBUG_ROUNDS") != nullptr;
    static const bool tc_verify = dev_env("APPD_TC_VERIFY") != nullptr;
    if (dbg) cudaEventRecord(c->ev[12], c->stream);
    if (!(use_tc && (tc.lookup_pending || rounds == 0)) && !w_pending && (s = launch_fill_u64(c, compbest, k, KEY_NONE)))
      return s;
    const int* cmp = rounds == 0 ? nullptr : comp;
    if (c->opt.timing >= 2) cudaEventRecord(c->ev[8], c->stream);  // per-round scan time (diagnostics)
    const int64_t l0 = c->launches;
    if (points && use_tc) {
      bool overflowed = false;
      if ((s = tcf_round(c, &tc, X, comp, rounds, k, compbest, rt_begin, rt_end, &overflowed))) return s;
      if (overflowed) {  // candidate buffer too small for this input: exact scan for this round
        if ((s = ensure_xt())) return s;
        s = launch_scan_points(c, XT, n, npad, dpad, row0, rows, cmp, compbest);
        c->stats.exact_rounds++;
      } else if (tc_verify) {  // debug: compare with the exact scan, report to stderr
        if ((s = ensure_xt())) return s;
        u64* cb2 = (u64*)ws(c, S_TMP, sizeof(u64) * k);
        if ((s = launch_fill_u64(c, cb2, k, KEY_NONE))) return s;
        if ((s = launch_scan_points(c, XT, n, npad, dpad, row0, rows, cmp, cb2))) return s;
        std::vector<u64> a(k), b(k);
        APPD_CUDA(c, cudaMemcpyAsync(a.data(), compbest, sizeof(u64) * k, cudaMemcpyDeviceToHost, c->stream));
        APPD_CUDA(c, cudaMemcpyAsync(b.data(), cb2, sizeof(u64) * k, cudaMemcpyDeviceToHost, c->stream));
        APPD_SYNC(c);
        int bad = 0;
        for (int64_t q = 0; q < k; q++)
          if (a[q] != b[q]) {
            if (bad < 5) {
              int64_t u1, v1, u2, v2;
              tri_decode(a[q] & ((1ull << 33) - 1), &u1, &v1);
              tri_decode(b[q] & ((1ull << 33) - 1), &u2, &v2);
              fprintf(stderr, "round %d comp %lld: tc (%lld,%lld) d2bits %llx  exact (%lld,%lld) d2bits %llx\n", rounds,
                      (long long)q, (long long)u1, (long long)v1, a[q] >> 33, (long long)u2, (long long)v2, b[q] >> 33);
            }
            bad++;
          }
        fprintf(stderr, "round %d: k=%lld mismatching components %d exact chunks %u fallback rows %u\n", rounds,
                (long long)k, bad, tc.h_counters[2], tc.h_counters[0]);
      }
    } else if (points && wide) {
      // per-row winners, then compw (minimum weight bits) and compbest (minimum pair index
      // among the winners of that weight), each reduced over the ranks
      u64* rowbest = (u64*)ws(c, S_WIDE_ROW, sizeof(u64) * n);
      u64* compw = (u64*)ws(c, S_WIDE_COMPW, sizeof(u64) * n);
      if (!rowbest || !compw) return fail(c, APPD_ERR_OUT_OF_MEMORY, "wide-key round workspace");
      if ((s = launch_fill_u64(c, rowbest, n, KEY_NONE))) return s;
      if ((s = launch_fill_u64(c, compw, k, KEY_NONE))) return s;
      if ((s = launch_scan_points(c, XT, n, npad, dpad, row0, rows, cmp, rowbest, true))) return s;
      if ((s = launch_wide_compw(c, rowbest, cmp, row0, row0 + rows, compw))) return s;
      if (c->coll && (s = nccl_allreduce_min_u64(c, compw, k))) return s;
      s = launch_wide_compbest(c, rowbest, cmp, row0, row0 + rows, compw, compbest);
      c->stats.exact_rounds++;
    } else if (points) {
      s = launch_scan_points(c, XT, n, npad, dpad, row0, rows, cmp, compbest);
      c->stats.exact_rounds++;
    } else if (f64) {
      s = launch_scan_weights_f64(c, c->f64_W, n, k, rounds == 0, sense, comp, f64_compw, f64_roww, f64_rowj, compbest);
    } else if (wtopk && rounds == 0) {
      s = launch_scan_weights_topk(c, W, n, row0, rows, wtopk, sense, w_ckey, w_cj, w_ccnt, compbest);
    } else if (wtopk) {
      // cached round: rows without an eligible cached key whose K-th key is below their
      // component's best are re-scanned
      if (!w_pending) {
        if ((s = w_lookup_async())) return s;
        APPD_SYNC(c);
      }
      w_pending = false;
      const unsigned cnt = c->pinned_small[9];
      c->stats.rescan_rows += cnt;
      if (cnt) c->stats.rescan_rounds++;
      s = launch_scan_weights_list(c, W, n, row0, w_list, w_count, (int)cnt, comp, compbest, sense);
    } else {
      s = launch_scan_weights(c, W, n, row0, rows, cmp, compbest, sense);
    }
    if (s) return s;
    c->stats.scan_launches += c->launches - l0;
    if (c->opt.timing >= 2) cudaEventRecord(c->ev[9], c->stream);
    host_mark("round scan queued");
    if (c->coll && (s = nccl_allreduce_min_u64(c, compbest, k))) return s;
    // the next round's cache lookup rides on this round's synchronisation (labels are
    // final): one rank, fused into the cooperative contraction when it can run
    LookupArgs la;
    bool fused_lookup = false;
    if (use_tc && tc.topk && !c->coll) {
      la.r0 = (int)tc.cache_r0;
      la.r1 = (int)tc.cache_r1;
      la.K = tc.topk;
      la.ckey = tc.ckey;
      la.cj = tc.cj;
      la.ccnt = tc.ccnt;
      la.need = tc.need;
      la.count = tc.counters + 3;
      la.list = tc.rows_list;
    } else if (wtopk && !c->coll) {
      la.r0 = (int)row0;
      la.r1 = (int)(row0 + rows);
      la.K = wtopk;
      la.ckey = w_ckey;
      la.cj = w_cj;
      la.ccnt = w_ccnt;
      la.need = w_need;
      la.count = w_count;
      la.list = w_list;
    }
    s = launch_contract(c, compbest, k, comp, n, ks.shift, link, parent, mstkeys, counters, flags, newid,
                        la.ckey ? &la : nullptr);
    if (s == APPD_ERR_UNSUPPORTED) {
      if ((s = launch_hook(c, compbest, k, comp, ks.shift, link))) return s;
      if ((s = launch_mutual(c, compbest, k, link, parent, mstkeys, counters))) return s;
      if ((s = launch_jump(c, parent, k, flags))) return s;
      if ((s = exclusive_scan_i32(c, flags, newid, k))) return s;
      if ((s = launch_relabel(c, comp, n, parent, newid))) return s;
    } else if (s) {
      return s;
    } else {
      fused_lookup = la.ckey != nullptr;
    }
    if (fused_lookup) {
      APPD_PUBLISH(c, c->pinned_small + 9, la.count, sizeof(unsigned));
      if (use_tc && tc.topk) {
        tc.lookup_pending = true;
      } else {
        w_pending = true;
      }
    } else {
      if (use_tc && tc.topk && !c->coll) {
        if ((s = launch_fill_u64(c, compbest, n, KEY_NONE))) return s;
        if ((s = tcf_lookup_async(c, &tc, comp, compbest))) return s;
      }
      if (wtopk && !c->coll) {
        if ((s = launch_fill_u64(c, compbest, n, KEY_NONE))) return s;
        if ((s = w_lookup_async())) return s;
      }
    }
    APPD_PUBLISH(c, &hostk[0], newid + (k - 1), sizeof(int));
    APPD_PUBLISH(c, &hostk[1], flags + (k - 1), sizeof(int));
    if (dbg) cudaEventRecord(c->ev[13], c->stream);
    host_mark("round queued, synchronising");
    if (fused_lookup && use_tc && tc.topk) {
      // the host waits for the round's results only; the next round's exact re-scan of the
      // flagged rows (device list and count) runs meanwhile, so the GPU does not idle while
      // the host wakes up and queues the rest of the next round
      if ((s = publish_flush(c))) return s;
      APPD_CUDA(c, cudaEventRecord(c->ev[7], c->stream));
      if ((s = tcf_speculate_rows(c, &tc, comp, compbest))) return s;
      APPD_CUDA(c, cudaEventSynchronize(c->ev[7]));
    } else {
      APPD_SYNC(c);
    }
    host_mark("round synchronised");
    if (check_first_sync) {
      check_first_sync = false;
      if (defer_validation) {  // the input verdict, queued before the engine started
        u64 hb[3];
        memcpy(hb, hbad, sizeof hb);
        appd_status sv = report_validation(c, hb, n, points, d);
        if (sv) return sv;
      }
      if (c->pinned_small[50] == 0) {  // coordinates too large for the filter: exact engine
        if (c->opt.points_engine == 2)
          return fail(c, APPD_ERR_UNSUPPORTED, "coordinates too large for the tensor-core filter");
        const int pe = c->opt.points_engine;
        c->opt.points_engine = 1;
        const appd_status s2 = solve(c, W, X, n, d, M);
        c->opt.points_engine = pe;
        return s2;
      }
    }
    if (c->opt.timing >= 2) c->stats.ms_scan += ev_ms(c, 8, 9);
    if (use_tc) {
      if (c->opt.timing && tc.scanned) {
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, c->ev[10], c->ev[11]) == cudaSuccess) c->stats.ms_tcscan += ms;
        cudaGetLastError();
      }
      c->stats.tc_candidates += (int64_t)tc.h_counters[2] * 128 + (int64_t)tc.h_counters[0] * n;
      c->stats.tc_fallback_rows += tc.h_counters[0];
      c->stats.topk = tc.topk;
      if (rounds == 0) {
        c->stats.tcscan_launches++;
        c->stats.tcscan_flops += 2.0 * (double)(std::min<int64_t>(rt_end * 512, n) - rt_begin * 512) * n * d;
        if (tc.topk) c->stats.cache_invalid_rows = tc.h_counters[0];
      } else if (!tc.topk) {
        c->stats.tcscan_launches++;
        c->stats.tcscan_flops += 2.0 * (double)(std::min<int64_t>(rt_end * 512, n) - rt_begin * 512) * n * d;
      } else if (tc.last_rescan_rows > 0) {
        c->stats.rescan_rounds++;
        c->stats.rescan_rows += tc.last_rescan_rows;
      }
      if (rounds > 0 && tc.topk && tc.scanned) {
        const int64_t blocks = c->pinned_small[8];
        c->stats.rescan_blocks += blocks;
        c->stats.tcscan_launches++;
        c->stats.tcscan_flops += 2.0 * (double)std::min<int64_t>(blocks * 512, n) * n * d;
      }
    }
    int64_t knew = (int64_t)hostk[0] + hostk[1];
    if (dbg && use_tc && rounds == 0 && tc.topk)
      fprintf(stderr, "[appd] cache build: listed (row, 32-col chunk) pairs %u\n", c->pinned_small[16]);
    if (dbg)
      fprintf(stderr, "[appd] round %d (%.3f ms): k %lld -> %lld  rescan rows %lld blocks %u  exact tiles %u fallback %u\n",
              rounds, ev_ms(c, 12, 13), (long long)k, (long long)knew, (long long)(use_tc ? tc.last_rescan_rows : 0),
              use_tc ? c->pinned_small[8] : 0u, use_tc ? tc.h_counters[2] : 0u, use_tc ? tc.h_counters[0] : 0u);
    rounds++;
    if (knew >= k || knew < 1) return fail(c, APPD_ERR_CUDA, "Boruvka made no progress (k = %lld)", (long long)k);
    k = knew;
  }
  c->stats.rounds = rounds;
  // MST edge count: checked at the final synchronisation (an internal consistency check)
  int* mst_count = reinterpret_cast<int*>(c->pinned_small + 26);
  *mst_count = -1;
  APPD_PUBLISH(c, mst_count, counters, sizeof(int));
  stage_event(c, 2);

  // ---- a4: sort the MST edge keys ascending (Kruskal order = P:L98's descending removal reversed) ----
  // only the weight bits decide the order: ties in any order are a valid Kruskal order
  // (SURVEY App. A.5), and the radix passes over the pair index would be wasted
  const int64_t m = n - 1;
  double* hw = nullptr;  // fp64: weight of each rank (k_f64.cu)
  int32_t* d_eu = (int32_t*)ws(c, S_EDGES, (sizeof(int32_t) * 2 + sizeof(float)) * m + 64);
  if (!d_eu) return fail(c, APPD_ERR_OUT_OF_MEMORY, "edge workspace");
  int32_t* d_ev = d_eu + m;
  float* d_ew = (float*)(d_ev + m);
  if (f64) {
    // the keys hold pair indices only: sort by the fp64 weights, relabel by rank
    hw = (double*)ws(c, S_F64_HW, sizeof(double) * (m + 1));
    u64* wk = (u64*)ws(c, S_F64_A, sizeof(u64) * 2 * n);
    int* ix = (int*)ws(c, S_F64_B, sizeof(int) * 2 * n);
    if (!hw || !wk || !ix) return fail(c, APPD_ERR_OUT_OF_MEMORY, "fp64 edge workspace");
    if ((s = launch_edges_f64(c, mstkeys, m, c->f64_W, n, sense, wk, wk + n, ix, ix + n, d_eu, d_ev, d_ew, hw)))
      return s;
  } else if (wide) {
    u64* key2s = (u64*)ws(c, S_WIDE_KEY2, sizeof(u64) * n);
    if (!key2s) return fail(c, APPD_ERR_OUT_OF_MEMORY, "wide-key edge workspace");
    if ((s = wide_edges(c, mstkeys, m, X, d, c->opt.metric, sense, sorted, key2s, d_eu, d_ev, d_ew))) return s;
  } else if ((s = sort_keys_u64_bits64(c, mstkeys, sorted, n - 1, ks.shift, 64))) {
    return s;
  }
  stage_event(c, 3);

  // ---- a5: dendrogram (v1: host union-find with list concatenation) ----
  // the GPU decodes the sorted keys to (u, v, w); pinned buffers keep the copies async
  if (!f64 && !wide && (s = launch_decode_edges(c, sorted, m, ks, d_eu, d_ev, d_ew))) return s;
  int levels = 1;
  while ((1ll << levels) <= m) levels++;
  const int64_t stride = m;
  int* pi = (int*)ws(c, S_PI, sizeof(int) * n);
  int* pos = (int*)ws(c, S_POS, sizeof(int) * n);
  float* ST = (float*)ws(c, S_ST, sizeof(float) * stride * levels);
  if (!pi || !pos || !ST) return fail(c, APPD_ERR_OUT_OF_MEMORY, "fill workspace");
  c->dend_n = n;
  bool pos_fused = false, rowpos_fused = false;
  if (c->opt.dendrogram != 1) {
    // v2: Prim order of the MST on the GPU (k_dendro.cu); h lands in the sparse table's level 0
#ifdef APPD_DEV_HOOKS
    dev_check(c, "edges", d_eu, d_ev, m, nullptr, n);
#endif
    // the fused tours also write pos = pi^-1 and, for a one-rank in-HBM fill, the identity
    // row positions (k_positions / k_iota folded in)
    int* rp_out = (!c->coll && !c->stream_out && !c->sink) ? (int*)ws(c, S_ROWPOS, sizeof(int) * n) : nullptr;
    if ((s = gpu_dendrogram(c, d_eu, d_ev, d_ew, n, pi, ST, pos, rp_out, &pos_fused))) return s;
    rowpos_fused = pos_fused && rp_out != nullptr;
#ifdef APPD_DEV_HOOKS
    dev_check(c, "dendrogram", nullptr, nullptr, 0, pi, n);
#endif
    c->dend_pi = pi;
    c->dend_h = ST;
    c->dend_on_device = true;
    c->stats.dendrogram = 2;
  } else {
    // v1: host union-find (Kruskal reconstruction tree); pinned buffers keep the copies async
    uint8_t* hp = (uint8_t*)pinned_host(c, 12 * (size_t)m + 8 * (size_t)n + 64);
    if (!hp) return fail(c, APPD_ERR_OUT_OF_MEMORY, "pinned host buffer");
    int32_t* h_e = (int32_t*)hp;                // eu, ev, ew (12 m bytes)
    int32_t* h_pi = (int32_t*)(hp + 12 * m);    // pi (4 n)
    float* h_h = (float*)(h_pi + n);            // h (4 (n - 1))
    APPD_CUDA(c, cudaMemcpyAsync(h_e, d_eu, 12 * (size_t)m, cudaMemcpyDeviceToHost, c->stream));
    APPD_SYNC(c);
    if ((int64_t)c->uf_scratch.size() < 8 * n) c->uf_scratch.resize(8 * n);
    host_dendrogram_uvw(h_e, h_e + m, (const float*)(h_e + 2 * m), n, h_pi, h_h, c->uf_scratch.data());
    c->dend_pi = h_pi;
    c->dend_h = h_h;
    c->dend_on_device = false;
    c->stats.dendrogram = 1;
    APPD_CUDA(c, cudaMemcpyAsync(pi, h_pi, sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    APPD_CUDA(c, cudaMemcpyAsync(ST, h_h, sizeof(float) * m, cudaMemcpyHostToDevice, c->stream));
  }
  c->have_dendrogram = !f64;  // fp64: the device h holds ranks, not weights
  stage_event(c, 4);

  // ---- a6: fill prep ----
  if (!pos_fused && (s = launch_positions(c, pi, n, pos))) return s;
  // fp64: ranks increase along the Kruskal order in either sense, so the max-combination
  const bool widest_fill = sense < 0 && !f64;
  if ((s = launch_sparse_table(c, ST, m, levels, stride, widest_fill))) return s;
  const int* rows_sorted = pi;
  int* rowpos = (int*)ws(c, S_ROWPOS, sizeof(int) * n);
  if (!rowpos) return fail(c, APPD_ERR_OUT_OF_MEMORY, "fill workspace");
  if (c->stream_out || c->sink) {
    // ---- NEXT-4: M streamed to host memory in blocks of R original rows.  Per block the
    // rows' leaf positions are gathered and sorted (the multi-rank fill path), the fill
    // writes a device block buffer (two, alternating) and copy_stream moves it to the host
    // while the next block is filled.  Sink mode: the host buffer is one of two pinned
    // staging blocks, handed to the callback once its copy is complete (while the GPU
    // fills and copies the next block).
    const int64_t R = std::min<int64_t>(c->stream_block, n);
    float* hstage = nullptr;
    if (c->sink) {
      const size_t want = sizeof(float) * 2 * (size_t)R * n;
      if (c->sink_bytes < want) {
        if (c->sink_host) cudaFreeHost(c->sink_host);
        c->sink_host = nullptr;
        c->sink_bytes = 0;
        if (cudaHostAlloc((void**)&c->sink_host, want, cudaHostAllocDefault) != cudaSuccess) {
          cudaGetLastError();
          return fail(c, APPD_ERR_OUT_OF_MEMORY, "pinned sink staging (%zu bytes)", want);
        }
        c->sink_bytes = want;
      }
      hstage = c->sink_host;
    }
    int64_t prev_b0 = -1, prev_rr = 0;
    int prev_buf = 0;
    auto drain_prev = [&]() -> appd_status {  // hand the previous block to the sink
      if (!c->sink || prev_b0 < 0) return APPD_OK;
      APPD_CUDA(c, cudaEventSynchronize(c->sev[2 + prev_buf]));
      const int64_t b0 = prev_b0;
      const int32_t r = c->sink(c->sink_user, b0, prev_rr, hstage + (size_t)prev_buf * R * n);
      prev_b0 = -1;
      if (r != 0) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamSynchronize(c->stream);
        return fail(c, APPD_ERR_INVALID_ARGUMENT, "sink returned %d at rows [%lld, %lld)", (int)r, (long long)b0,
                    (long long)(b0 + prev_rr));
      }
      return APPD_OK;
    };
    if (c->sink && cm_status_pending) {
      // the callback must never see a block that is solved again: settle a component-matrix
      // listing overflow (rare; the solve is repeated without it) before the first block
      APPD_SYNC(c);
      if (c->pinned_small[48] == 1) {
        const int fk = c->opt.finish_k;
        c->opt.finish_k = -1;
        const appd_status s2 = solve(c, W, X, n, d, M);
        c->opt.finish_k = fk;
        c->stats.cm_retries++;
        return s2;
      }
    }
    float* dblk = (float*)ws(c, S_HOST_OUT, sizeof(float) * 2 * R * n);
    int* keys = (int*)ws(c, S_TMP, sizeof(int) * 2 * (R + 1));
    int* rs = (int*)ws(c, S_ROWS_SORTED, sizeof(int) * (R + 1));
    if (!dblk || !keys || !rs) return fail(c, APPD_ERR_OUT_OF_MEMORY, "stream block buffers (%lld rows)", (long long)R);
    if (!c->copy_stream && cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(c, APPD_ERR_CUDA, "copy stream");
    if (!c->sev_ready) {
      for (int i = 0; i < 4; i++)
        if (cudaEventCreateWithFlags(&c->sev[i], cudaEventDisableTiming) != cudaSuccess)
          return fail(c, APPD_ERR_CUDA, "stream events");
      c->sev_ready = true;
    }
    stage_event(c, 5);
    int64_t blocks = 0;
    for (int64_t b0 = 0; b0 < n; b0 += R, blocks++) {
      const int64_t rr = std::min(R, n - b0);
      const int buf = (int)(blocks & 1);
      float* dst = dblk + (size_t)buf * R * n;
      if (blocks >= 2) APPD_CUDA(c, cudaStreamWaitEvent(c->stream, c->sev[2 + buf], 0));  // buffer copied out
      if ((s = launch_gather_rowpos(c, pos, b0, rr, keys, keys + rr + 1))) return s;
      if ((s = sort_pairs_i32(c, keys, rowpos, keys + rr + 1, rs, rr))) return s;
      if ((s = launch_fill(c, rs, rowpos, rr, pos, ST, stride, n, dst, b0, sense < 0))) return s;
      APPD_CUDA(c, cudaEventRecord(c->sev[buf], c->stream));
      APPD_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->sev[buf], 0));
      float* hdst = c->sink ? hstage + (size_t)buf * R * n : c->stream_out + (size_t)b0 * n;
      APPD_CUDA(c, cudaMemcpyAsync(hdst, dst, sizeof(float) * rr * n, cudaMemcpyDeviceToHost, c->copy_stream));
      APPD_CUDA(c, cudaEventRecord(c->sev[2 + buf], c->copy_stream));
      if ((s = drain_prev())) return s;
      prev_b0 = b0;
      prev_rr = rr;
      prev_buf = buf;
    }
    if ((s = drain_prev())) return s;
    APPD_CUDA(c, cudaStreamWaitEvent(c->stream, c->sev[2 + (int)((blocks - 1) & 1)], 0));  // last copy done
    if (blocks >= 2) APPD_CUDA(c, cudaStreamWaitEvent(c->stream, c->sev[2 + (int)(blocks & 1)], 0));
    stage_event(c, 6);
    APPD_SYNC(c);
    if (cm_status_pending && c->pinned_small[48] == 1) {
      const int fk = c->opt.finish_k;
      c->opt.finish_k = -1;
      const appd_status s2 = solve(c, W, X, n, d, M);
      c->opt.finish_k = fk;
      c->stats.cm_retries++;
      return s2;
    }
    if (cm_status_pending && c->pinned_small[48] != 0)
      return fail(c, APPD_ERR_CUDA, "component matrix disconnected (internal error)");
    if (*mst_count != n - 1)
      return fail(c, APPD_ERR_CUDA, "MST has %d edges, expected %lld", *mst_count, (long long)(n - 1));
    c->stats.fill_bytes = n * n * 4;
    c->stats.kernel_launches = c->launches;
    if (c->opt.timing) {
      c->stats.ms_validate = ev_ms(c, 0, 1);
      c->stats.ms_mst = ev_ms(c, 1, 2);
      c->stats.ms_sort = ev_ms(c, 2, 3);
      c->stats.ms_dendrogram = ev_ms(c, 3, 4);
      c->stats.ms_prep = ev_ms(c, 4, 5);
      c->stats.ms_fill = ev_ms(c, 5, 6);
      c->stats.ms_total = ev_ms(c, 0, 6);
    }
    return APPD_OK;
  }
  if (!c->coll) {
    if (!rowpos_fused && (s = launch_iota(c, rowpos, n))) return s;
  } else {
    int* keys = (int*)ws(c, S_TMP, sizeof(int) * 2 * (rows + 1));
    int* rs = (int*)ws(c, S_ROWS_SORTED, sizeof(int) * (rows + 1));
    if (!keys || !rs) return fail(c, APPD_ERR_OUT_OF_MEMORY, "fill workspace");
    if ((s = launch_gather_rowpos(c, pos, row0, rows, keys, keys + rows + 1))) return s;
    if ((s = sort_pairs_i32(c, keys, rowpos, keys + rows + 1, rs, rows))) return s;
    rows_sorted = rs;
  }
  stage_event(c, 5);

  // ---- a7: fill ----
  if (f64) {
    if ((s = launch_fill_f64(c, rows_sorted, rowpos, rows, pos, ST, stride, n, c->f64_M, row0, hw))) return s;
  } else if ((s = launch_fill(c, rows_sorted, rowpos, rows, pos, ST, stride, n, M, row0, sense < 0))) {
    return s;
  }
  stage_event(c, 6);
  APPD_SYNC(c);
  if (cm_status_pending && c->pinned_small[48] == 1) {
    // the component matrix's candidate list overflowed: solve again without it (rare)
    const int fk = c->opt.finish_k;
    c->opt.finish_k = -1;
    const appd_status s2 = solve(c, W, X, n, d, M);
    c->opt.finish_k = fk;
    c->stats.cm_retries++;
    return s2;
  }
  if (cm_status_pending && c->pinned_small[48] != 0)
    return fail(c, APPD_ERR_CUDA, "component matrix disconnected (internal error)");
  if (*mst_count != n - 1)
    return fail(c, APPD_ERR_CUDA, "MST has %d edges, expected %lld", *mst_count, (long long)(n - 1));
  if (cm_timing_pending) {  // the component-matrix pass's events are complete only now
    if (c->opt.timing >= 2) c->stats.ms_scan += ev_ms(c, 8, 9);
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, c->ev[10], c->ev[11]) == cudaSuccess) c->stats.ms_tcscan += ms;
    cudaGetLastError();
  }
  c->stats.fill_bytes = rows * n * (f64 ? 8 : 4);
  c->stats.kernel_launches = c->launches;
  if (c->opt.timing) {
    c->stats.ms_validate = ev_ms(c, 0, 1);
    c->stats.ms_mst = ev_ms(c, 1, 2);
    c->stats.ms_sort = ev_ms(c, 2, 3);
    c->stats.ms_dendrogram = ev_ms(c, 3, 4);
    c->stats.ms_prep = ev_ms(c, 4, 5);
    c->stats.ms_fill = ev_ms(c, 5, 6);
    c->stats.ms_total = ev_ms(c, 0, 6);
  }
  return APPD_OK;
}

static appd_status enter(appd_ctx* c) {
  if (!c) return APPD_ERR_INVALID_ARGUMENT;
  if (c->poisoned) return APPD_ERR_POISONED;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "cudaSetDevice");
  return APPD_OK;
}

extern "C" appd_status appd_solve_weights(appd_ctx* c, const float* W, int64_t n, float* M) {
  appd_status s = enter(c);
  if (s) return s;
  if (n < 1) return fail(c, APPD_ERR_INVALID_ARGUMENT, "n = %lld < 1", (long long)n);
  if (n > 92682) return fail(c, APPD_ERR_UNSUPPORTED, "weights mode supports n <= 92682 (32-bit pair index)");
  int64_t row0, rows;
  appd_row_range_of(n, c->opt.rank, c->opt.world, &row0, &rows);
  if (rows > 0 || W || M) {  // a rank that owns no rows may pass NULL blocks
    if ((s = check_device_ptr(c, W, "W"))) return s;
    if ((s = check_device_ptr(c, M, "M"))) return s;
  }
  return solve(c, W, nullptr, n, 0, M);
}

// NEXT-3: fp64 weight matrix, fp64 output (k_f64.cu).  One rank; no streaming.
extern "C" appd_status appd_solve_weights_f64(appd_ctx* c, const double* W, int64_t n, double* M) {
  appd_status s = enter(c);
  if (s) return s;
  if (n < 1) return fail(c, APPD_ERR_INVALID_ARGUMENT, "n = %lld < 1", (long long)n);
  if (n > 92682) return fail(c, APPD_ERR_UNSUPPORTED, "weights mode supports n <= 92682 (32-bit pair index)");
  if (c->coll) return fail(c, APPD_ERR_UNSUPPORTED, "appd_solve_weights_f64 runs on one rank without collectives (world = %d)", c->opt.world);
  if ((s = check_device_ptr(c, W, "W"))) return s;
  if ((s = check_device_ptr(c, M, "M"))) return s;
  if ((const void*)W == (const void*)M) return fail(c, APPD_ERR_INVALID_ARGUMENT, "W and M must not alias");
  c->f64_W = W;
  c->f64_M = M;
  float* saved = c->stream_out;
  c->stream_out = nullptr;
  s = solve(c, nullptr, nullptr, n, 0, nullptr);
  c->stream_out = saved;
  c->f64_W = nullptr;
  c->f64_M = nullptr;
  return s;
}

// NEXT-2: the paper's comparison algorithm (minimax Floyd–Warshall) on
// the GPU, k_floyd.cu.  Single rank (O(n^3); no sharding); same validation as
// appd_solve_weights; opt.sense selects minimax (+1) or widest (-1).
extern "C" appd_status appd_floyd_weights(appd_ctx* c, const float* W, int64_t n, float* M) {
  appd_status s = enter(c);
  if (s) return s;
  if (n < 1) return fail(c, APPD_ERR_INVALID_ARGUMENT, "n = %lld < 1", (long long)n);
  if (c->coll) return fail(c, APPD_ERR_UNSUPPORTED, "appd_floyd_weights runs on one rank without collectives (world = %d)", c->opt.world);
  if (n > 65536) return fail(c, APPD_ERR_UNSUPPORTED, "appd_floyd_weights: n = %lld > 65536 (O(n^3))", (long long)n);
  if ((s = check_device_ptr(c, W, "W"))) return s;
  if ((s = check_device_ptr(c, M, "M"))) return s;
  if (W == M) return fail(c, APPD_ERR_INVALID_ARGUMENT, "W and M must not alias");
  std::memset(&c->stats, 0, sizeof c->stats);
  c->stats.struct_size = sizeof(appd_stats);
  c->stats.n = n;
  c->stats.rows = n;
  c->launches = 0;
  c->have_dendrogram = false;
  c->err_i = c->err_j = -1;
  c->last_error.clear();
  stage_event(c, 0);
  if (c->opt.validate) {
    u64* bad = (u64*)ws(c, S_VALID, 3 * sizeof(u64));
    if (!bad) return fail(c, APPD_ERR_OUT_OF_MEMORY, "validation buffer");
    u64* hbad = reinterpret_cast<u64*>(c->pinned_small + 40);
    APPD_CUDA(c, cudaMemsetAsync(bad, 0xFF, 3 * sizeof(u64), c->stream));
    if ((s = launch_validate_weights(c, W, n, 0, n, bad))) return s;
    APPD_PUBLISH(c, hbad, bad, 3 * sizeof(u64));
    APPD_SYNC(c);
    u64 hb[3];
    memcpy(hb, hbad, sizeof hb);
    if ((s = report_validation(c, hb, n, false, 0))) return s;
  }
  stage_event(c, 1);
  if ((s = floyd_weights(c, W, n, M, c->opt.sense >= 0 ? 1 : -1))) return s;
  stage_event(c, 6);
  APPD_SYNC(c);
  c->stats.kernel_launches = c->launches;
  c->stats.fill_bytes = n * n * 4;
  if (c->opt.timing) {
    c->stats.ms_validate = ev_ms(c, 0, 1);
    c->stats.ms_total = ev_ms(c, 0, 6);
  }
  return APPD_OK;
}

extern "C" appd_status appd_solve_points(appd_ctx* c, const float* X, int64_t n, int64_t d, float* M) {
  appd_status s = enter(c);
  if (s) return s;
  if (n < 1 || d < 1) return fail(c, APPD_ERR_INVALID_ARGUMENT, "n = %lld, d = %lld", (long long)n, (long long)d);
  if (n > kMaxPoints) return fail(c, APPD_ERR_UNSUPPORTED, "points mode supports n <= 2^20");
  if (d > 65536) return fail(c, APPD_ERR_UNSUPPORTED, "d > 65536");
  if ((s = check_device_ptr(c, X, "X"))) return s;
  int64_t row0, rows;
  appd_row_range_of(n, c->opt.rank, c->opt.world, &row0, &rows);
  if ((rows > 0 || M) && (s = check_device_ptr(c, M, "M"))) return s;  // no rows: M may be NULL
  return solve(c, nullptr, X, n, d, M);
}

// host-buffer variants (end to end: H2D of the input and D2H of M inside the call)
static appd_status solve_host(appd_ctx* c, const float* Wh, const float* Xh, int64_t n, int64_t d, float* Mh) {
  appd_status s = enter(c);
  if (s) return s;
  if (!Mh || (!Wh && !Xh)) return fail(c, APPD_ERR_INVALID_ARGUMENT, "NULL host buffer");
  if (n < 1 || (Xh && d < 1)) return APPD_ERR_INVALID_ARGUMENT;
  int64_t row0, rows;
  appd_row_range_of(n, c->opt.rank, c->opt.world, &row0, &rows);
  size_t in_bytes = Xh ? sizeof(float) * n * d : sizeof(float) * rows * n;
  size_t out_bytes = sizeof(float) * rows * n;
  float* din = (float*)ws(c, S_HOST_IN, in_bytes);
  float* dout = (float*)ws(c, S_HOST_OUT, out_bytes);
  if (!din || !dout) return fail(c, APPD_ERR_OUT_OF_MEMORY, "device staging for host buffers");
  APPD_CUDA(c, cudaMemcpyAsync(din, Xh ? Xh : Wh, in_bytes, cudaMemcpyHostToDevice, c->stream));
  s = Xh ? solve(c, nullptr, din, n, d, dout) : solve(c, din, nullptr, n, 0, dout);
  if (s) return s;
  APPD_CUDA(c, cudaMemcpyAsync(Mh, dout, out_bytes, cudaMemcpyDeviceToHost, c->stream));
  APPD_SYNC(c);
  return APPD_OK;
}

extern "C" appd_status appd_solve_points_host(appd_ctx* c, const float* X, int64_t n, int64_t d, float* M) {
  if (c && n > kMaxPoints) return fail(c, APPD_ERR_UNSUPPORTED, "points mode supports n <= 2^20");
  if (c && d > 65536) return fail(c, APPD_ERR_UNSUPPORTED, "d > 65536");
  return solve_host(c, nullptr, X, n, d, M);
}

// NEXT-4: points mode with each row block of M handed to a host callback (n beyond host
// memory as well: 2^18 points make 256 GiB of output)
extern "C" appd_status appd_solve_points_sink(appd_ctx* c, const float* X, int64_t n, int64_t d, int64_t block_rows,
                                              int32_t (*sink)(void*, int64_t, int64_t, const float*), void* user) {
  appd_status s = enter(c);
  if (s) return s;
  if (!X || !sink) return fail(c, APPD_ERR_INVALID_ARGUMENT, "NULL X or sink");
  if (n < 1 || d < 1 || block_rows < 0) return fail(c, APPD_ERR_INVALID_ARGUMENT, "n, d, block_rows");
  if (n > kMaxPoints) return fail(c, APPD_ERR_UNSUPPORTED, "points mode supports n <= 2^20");
  if (d > 65536) return fail(c, APPD_ERR_UNSUPPORTED, "d > 65536");
  if (c->coll) return fail(c, APPD_ERR_UNSUPPORTED, "appd_solve_points_sink runs on one rank");
  const int64_t R = block_rows ? block_rows : std::max<int64_t>(128, ((int64_t)1 << 28) / n);
  float* din = (float*)ws(c, S_HOST_IN, sizeof(float) * n * d);
  if (!din) return fail(c, APPD_ERR_OUT_OF_MEMORY, "device copy of X");
  APPD_CUDA(c, cudaMemcpyAsync(din, X, sizeof(float) * n * d, cudaMemcpyHostToDevice, c->stream));
  c->sink = sink;
  c->sink_user = user;
  c->stream_block = R;
  s = solve(c, nullptr, din, n, d, nullptr);
  c->sink = nullptr;
  c->sink_user = nullptr;
  c->stream_block = 0;
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  return s;
}

// NEXT-4: points mode with M streamed to host memory in row blocks (n beyond HBM)
extern "C" appd_status appd_solve_points_stream(appd_ctx* c, const float* X, int64_t n, int64_t d, float* M,
                                                int64_t block_rows) {
  appd_status s = enter(c);
  if (s) return s;
  if (!X || !M) return fail(c, APPD_ERR_INVALID_ARGUMENT, "NULL host buffer");
  if (n < 1 || d < 1 || block_rows < 0) return fail(c, APPD_ERR_INVALID_ARGUMENT, "n, d, block_rows");
  if (n > kMaxPoints) return fail(c, APPD_ERR_UNSUPPORTED, "points mode supports n <= 2^20");
  if (d > 65536) return fail(c, APPD_ERR_UNSUPPORTED, "d > 65536");
  if (c->coll) return fail(c, APPD_ERR_UNSUPPORTED, "appd_solve_points_stream runs on one rank");
  // default block: 1 GiB of rows per buffer (two buffers), at least 128 rows
  const int64_t R = block_rows ? block_rows : std::max<int64_t>(128, ((int64_t)1 << 28) / n);
  float* din = (float*)ws(c, S_HOST_IN, sizeof(float) * n * d);
  if (!din) return fail(c, APPD_ERR_OUT_OF_MEMORY, "device copy of X");
  APPD_CUDA(c, cudaMemcpyAsync(din, X, sizeof(float) * n * d, cudaMemcpyHostToDevice, c->stream));
  c->stream_out = M;
  c->stream_block = R;
  s = solve(c, nullptr, din, n, d, nullptr);
  c->stream_out = nullptr;
  c->stream_block = 0;
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  return s;
}

extern "C" appd_status appd_solve_weights_host(appd_ctx* c, const float* W, int64_t n, float* M) {
  if (c && n > 92682) return fail(c, APPD_ERR_UNSUPPORTED, "weights mode supports n <= 92682");
  return solve_host(c, W, nullptr, n, 0, M);
}

extern "C" appd_status appd_debug_tc_gram(appd_ctx* c, const float* X, int64_t n, int64_t d, float* tc_out,
                                          float* ref_out) {
  appd_status s = enter(c);
  if (s) return s;
  if (n < 1 || d < 1) return APPD_ERR_INVALID_ARGUMENT;
  if ((s = check_device_ptr(c, X, "X"))) return s;
  return tcf_debug_gram(c, X, n, d, tc_out, ref_out);
}

extern "C" appd_status appd_points_weights(appd_ctx* c, const float* X, int64_t n, int64_t d, int64_t row0,
                                           int64_t rows, float* Wb) {
  appd_status s = enter(c);
  if (s) return s;
  if (n < 1 || d < 1 || row0 < 0 || rows < 0 || row0 + rows > n) return APPD_ERR_INVALID_ARGUMENT;
  if ((s = check_device_ptr(c, X, "X"))) return s;
  if ((s = check_device_ptr(c, Wb, "Wblock"))) return s;
  if ((s = launch_points_weights(c, X, n, d, row0, rows, Wb))) return s;
  APPD_SYNC(c);
  return APPD_OK;
}
