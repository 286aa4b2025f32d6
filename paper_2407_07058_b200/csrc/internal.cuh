// internal.cuh -- shared declarations of libappd (B200 / sm_100a).
// Nothing here is shared with oracle/ (the CPU oracle is independent).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/appd.h"

namespace appd {

typedef unsigned long long u64;

constexpr u64 KEY_NONE = ~0ULL;

// ---------------------------------------------------------------------------
// Edge keys.  A strict total order on edges is required so that Boruvka never
// forms a cycle under ties: an edge {u, v},
// u < v, is ordered by (weight, v, u).  The pair index tri(u, v) = v(v-1)/2 + u
// is monotone in (v, u), so key = wkey << shift | tri(u, v).
//   weights mode: wkey = orderable(w) (32 bits), shift 32, n <= 92682
//   points mode:  wkey = bits(d^2) (31 bits, d^2 >= +0), shift 33, n <= 131072
// Restricted to one row i, the order is "smaller weight, then smaller j", so a
// row argmin over (w, j) is consistent with the component minimum over keys.
// ---------------------------------------------------------------------------
__host__ __device__ inline uint32_t orderable(float f) {
#ifdef __CUDA_ARCH__
  uint32_t b = __float_as_uint(f);
#else
  uint32_t b;
  memcpy(&b, &f, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__host__ __device__ inline float from_orderable(uint32_t u) {
  uint32_t b = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(b);
#else
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}

__host__ __device__ inline u64 tri_index(int64_t a, int64_t b) {
  int64_t u = a < b ? a : b, v = a < b ? b : a;
  return (u64)(v * (v - 1) / 2 + u);
}

// inverse of tri_index; t < 2^33
__host__ __device__ inline void tri_decode(u64 t, int64_t* u, int64_t* v) {
  double s = sqrt(1.0 + 8.0 * (double)t);
  int64_t vv = (int64_t)((1.0 + s) * 0.5);
  while (vv * (vv - 1) / 2 > (int64_t)t) vv--;
  while ((vv + 1) * vv / 2 <= (int64_t)t) vv++;
  *v = vv;
  *u = (int64_t)t - vv * (vv - 1) / 2;
}

struct KeySpec {
  int shift;     // 32 (weights) or 33 (points)
  bool points;   // key weight is bits(d^2)
  int sense;     // +1 minimax, -1 widest (points: the weight bits through ~b & 0x7FFFFFFF)
  int metric = 0;  // points: 0 Euclidean (key = bits(d^2), weight sqrtf), 1 L1, 2 L-inf (key = bits(d))
};

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct NcclApi;  // nccl_shim.cpp

}  // namespace appd

struct appd_ctx {
  appd_options opt;
  // NEXT-3: set for the duration of appd_solve_weights_f64 (k_f64.cu)
  const double* f64_W = nullptr;
  double* f64_M = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool poisoned = false;
  std::string last_error;
  int64_t err_i = -1, err_j = -1;
  appd_stats stats;
  int64_t launches = 0;  // kernels launched in the current solve
  void* nccl_comm = nullptr;
  // the solve takes the multi-rank path (every exchange a collective): world > 1, or world 1
  // with an explicit communicator (nccl_unique_id) or host exchange (host_allreduce)
  bool coll = false;
  bool nccl_aborted = false;  // set by the NCCL abort path (the context is poisoned too)
  int sm_count = 148;
  // workspace (grown on demand)
  appd::DevBuf buf[96];
  // the last dendrogram (in the pinned host buffer)
  int32_t* dend_pi = nullptr;
  float* dend_h = nullptr;
  int64_t dend_n = 0;
  int32_t one_pi = 0;
  bool have_dendrogram = false;
  bool dend_on_device = false;      // dend_pi / dend_h are device pointers (GPU dendrogram)
  // events for stage timing
  cudaEvent_t ev[16];
  bool ev_ready = false;
  uint64_t nvtx_stage = 0;  // the open NVTX stage range (nvtxRangeId_t)
  // pinned host staging for host-buffer calls
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  unsigned* pinned_small = nullptr;  // 64 words of pinned host memory for small async reads
  // 32 pinned words for the host side of the collectives' small exchanges (agreement, verdict,
  // branch flag): a device->pageable copy would block outside the deadline-polled wait
  unsigned long long* pinned_xchg = nullptr;
  // the same words as the device sees them (mapped pinned memory): small device results are
  // published there by one kernel per synchronisation instead of one copy each (publish())
  unsigned* pinned_small_dev = nullptr;
  struct PubEntry {
    const void* src;
    unsigned* dst;
    int words;
  };
  PubEntry pub[16];
  int npub = 0;
  // word of the cooperative kernels' grid barrier (coop_grid_sync), zeroed at first use
  unsigned* gridbar = nullptr;
  std::vector<unsigned long long> host_xchg;  // host exchange backend staging (opt.host_allreduce)
  std::vector<int32_t> uf_scratch;   // host dendrogram work arrays
  // streamed output (NEXT-4, appd_solve_points_stream): M rows go to this host buffer in
  // blocks of stream_block rows, two device block buffers, copies on copy_stream
  float* stream_out = nullptr;
  int64_t stream_block = 0;
  // NEXT-4 sink (appd_solve_points_sink): blocks go through two pinned staging buffers to a
  // host callback instead of a host matrix (n beyond host memory too)
  int32_t (*sink)(void*, int64_t, int64_t, const float*) = nullptr;
  void* sink_user = nullptr;
  float* sink_host = nullptr;
  size_t sink_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t sev[4];  // filled[2], copied[2]
  bool sev_ready = false;
};

namespace appd {

// Per-device one-time setup.  cudaFuncSetAttribute and occupancy are properties of the
// current device, and one process may hold contexts on several devices (each on its own
// host thread), so every "done" flag is a per-device bit set atomically.
inline unsigned long long dev_bit(const appd_ctx* c) { return 1ull << (c->device & 63); }
inline bool needs_setup(const std::atomic<unsigned long long>& done, const appd_ctx* c) {
  return (done.load(std::memory_order_acquire) & dev_bit(c)) == 0;
}
inline void setup_done(std::atomic<unsigned long long>& done, const appd_ctx* c) {
  done.fetch_or(dev_bit(c), std::memory_order_acq_rel);
}

// Development hooks (debug prints, timing experiments, verification against the exact
// engine) read environment variables only in builds with -DAPPD_DEV_HOOKS; the product
// build never consults the environment.
#ifdef APPD_DEV_HOOKS
inline const char* dev_env(const char* name) { return getenv(name); }
#else
inline const char* dev_env(const char*) { return nullptr; }
#endif

// APPD_DEBUG_HOST=1: host-side microseconds since the solve started, at marked points
inline void host_mark(const char* what, bool reset = false) {
  static const bool on = dev_env("APPD_DEBUG_HOST") != nullptr;
  static std::chrono::steady_clock::time_point t0;
  if (!on) return;
  const auto now = std::chrono::steady_clock::now();
  if (reset) t0 = now;
  fprintf(stderr, "[host] %8.1f us  %s\n", std::chrono::duration<double, std::micro>(now - t0).count(), what);
}

// workspace slots
enum Slot {
  S_COMP = 0, S_COMPBEST, S_LINK, S_PARENT, S_NEWID, S_FLAGS, S_MSTKEYS, S_MSTKEYS_SORTED, S_COUNTERS,
  S_XT, S_PI, S_POS, S_H, S_ST, S_ROWS_SORTED, S_ROWPOS, S_TMP, S_TMP2, S_VALID, S_KEYS_TMP, S_PRIM,
  S_HOST_IN, S_HOST_OUT,
  S_TC_PART, S_TC_CENTER, S_TC_YA, S_TC_YB, S_TC_NRM, S_TC_LEN, S_TC_TML, S_TC_PERM, S_TC_SC, S_TC_KEYS,
  S_TC_CSTART, S_TC_CEND, S_TC_RS, S_TC_RE, S_TC_UB, S_TC_CAND, S_TC_CNT, S_TC_RECV, S_TC_RECC, S_TC_FALLBACK,
  S_TC_XTP, S_TC_CML, S_TC_ROWFLAG, S_TC_APPPC, S_TC_APPV, S_EDGES,
  S_TC_CKEY, S_TC_CJ, S_TC_CCNT, S_TC_NEED, S_TC_NEEDP, S_TC_BLOCKFLAG, S_TC_RBLIST, S_TC_COMPUB, S_TC_UBK,
  S_TC_THRK, S_TC_CANDCNT, S_TC_CANDK, S_TC_WCM, S_TC_ROWLIST, S_TC_XTO, S_TC_LISTA, S_TC_LISTB, S_TC_RUNS, S_DENDRO, S_TC_SEGD, S_TC_ITEMS, S_TC_ERR, S_TC_SEGERR, S_SCAN, S_TC_SCALE, S_F64_A, S_F64_B, S_F64_HW,
  S_WIDE_ROW, S_WIDE_COMPW, S_WIDE_KEY2, S_LIST_CNT, S_SORT,
  S_NSLOTS
};
static_assert(S_NSLOTS <= 96, "workspace slots");

// tensor-core filtered points scan (k_tcfilter.cu)
// the scaling of the packed operands, computed on the device from max |x - c| (no host
// round trip): y^ = fp16(scale (x - c)); maxlen bounds |y^|; s2 = scale^2; ok = 0 when the
// coordinates are too large for the filter (the solve then falls back to the exact engine)
struct TcScale {
  float scale, maxlen;
  double s2;
  int ok, pad;
};
struct TcState {
  int64_t n = 0, d = 0, npad = 0;
  int dk = 0, K = 0, stages = 0;
  float c1 = 0.0f, c2 = 0.0f, k1 = 0.0f, k2 = 0.0f, k3 = 0.0f, gamma = 0.0f;
  TcScale* dscale = nullptr;  // device
  float* center = nullptr;
  void* YA = nullptr;  // __half
  void* YB = nullptr;
  float* XTp = nullptr;  // d x npad fp32, permuted columns (exact pass)
  float *nrm = nullptr, *len = nullptr, *seg_maxlen = nullptr;
  float *err = nullptr, *seg_maxerr = nullptr;  // per-point fp16 rounding-error norms E_p
  unsigned* maxerr = nullptr;                   // max E_p (device, float bits)
  int *perm = nullptr, *sc = nullptr, *keys = nullptr, *cstart = nullptr, *cend = nullptr, *rs = nullptr,
      *re = nullptr;
  unsigned* UB = nullptr;
  unsigned* counters = nullptr;
  unsigned* h_counters = nullptr;  // pinned host copy: [0] fallback rows, [2] exact chunks
  int* fallback = nullptr;
  int* rowflag = nullptr;
  void* TM = nullptr;       // stored maxima of the scans (fp32; the cache pass: fp16 encoded, tm_store)
  void* list = nullptr;     // uint2 (row, tile) pairs that need the exact check
  unsigned list_cap = 0;
  // round-0 candidate cache (k_cache.cu); topk == 0: no cache
  int topk = 0, cap = 0;
  int64_t cache_r0 = 0, cache_r1 = 0;  // original rows whose cache this rank holds
  u64* ckey = nullptr;                 // [n][topk] exact edge keys, ascending
  int* cj = nullptr;                   // [n][topk] other endpoint (original index)
  int* ccnt = nullptr;                 // [n] entries (-1: invalid, always re-scanned)
  int* need = nullptr;                 // [n] original order: re-scan this round
  int* needp = nullptr;                // [npad] permuted order
  int* blockflag = nullptr;            // [npad / 512 + 1]; rb_list follows, then the count
  int* rb_list = nullptr;
  int* rb_count = nullptr;
  int* rows_list = nullptr;             // [n] flagged rows (original indices)
  float* XT = nullptr;                 // d x npad original-order transpose (exact row kernel)
  unsigned* lista = nullptr;           // (chunk << 17 | row) candidate entries, then sorted
  unsigned* listb = nullptr;
  unsigned list_entries_cap = 0;
  unsigned* compUB = nullptr;          // [n] component upper bound (scaled units, float bits)
  float* UBK = nullptr;                // [npad]
  float* thrK = nullptr;               // [npad]
  unsigned* cand_cnt = nullptr;        // [npad]
  u64* cand = nullptr;                 // [npad][cap]
  // per-round statistics (host)
  int64_t last_rescan_rows = 0, last_rescan_blocks = 0, invalid_rows = 0, last_list_entries = 0;
  bool scanned = false;  // this round launched the tensor-core scan (ev[10] -> ev[11] bracket it)
  bool lookup_pending = false;  // next round's cache lookup already queued (tcf_lookup_async)
  bool r0_packed = false;       // the cooperative preparation also packed round 0 (identity order)
  bool rows_spec = false;       // the next round's exact re-scan is already queued (tcf_speculate_rows)
};
appd_status tcf_speculate_rows(appd_ctx* c, TcState* st, const int* comp, u64* compbest);
// device buffers to initialise before the first round, folded into one launch
struct InitTask {
  void* p;
  int64_t count;
  u64 value;
  int kind;  // 0: fill 32-bit words with value, 1: fill 64-bit words, 2: iota (int32)
};
struct InitList {
  InitTask t[16];
  int count = 0;
  void add(void* p, int64_t count_, u64 value, int kind) { t[this->count++] = {p, count_, value, kind}; }
};
// init: buffers the caller needs initialised (done inside the preparation when it runs
// as one cooperative kernel, else by one separate launch); bad (validation, device
// u64[3], may be null): non-finite coordinates are reported there (first element index)
appd_status tcf_prepare(appd_ctx* c, const float* X, int64_t n, int64_t d, TcState* st,
                        const InitList* init = nullptr, u64* bad = nullptr);
appd_status tcf_round(appd_ctx* c, TcState* st, const float* X, const int* comp, int round, int64_t k,
                      u64* compbest, int64_t row_tile_begin, int64_t row_tile_end, bool* overflowed);

appd_status floyd_weights(appd_ctx* c, const float* W, int64_t n, float* M, int sense);
appd_status launch_cm_prim(appd_ctx* c, const u64* WCM, int k, u64* mstkeys, int* counters,
                           const unsigned* list_count, unsigned list_cap, const int* cstart, const int* perm,
                           unsigned* status);
appd_status tcf_lookup_async(appd_ctx* c, TcState* st, const int* comp, u64* compbest);
appd_status tcf_cm(appd_ctx* c, TcState* st, const float* X, const int* comp, int64_t k, u64* WCM,
                   int64_t rb_begin, int64_t rb_end, bool* listed_overflow, bool check_now);

// candidate cache (k_cache.cu)
struct ErrModel;

appd_status launch_topk_select(appd_ctx* c, int p_begin, int p_end, int n, int K, const unsigned* cnt,
                               const u64* cand, int cap, u64* ckey, int* cj, int* ccnt, u64* compbest, int* fallback,
                               unsigned* nfallback);
appd_status launch_cache_lookup(appd_ctx* c, int r0, int r1, int K, int n, const u64* ckey, const int* cj,
                                const int* ccnt, const int* comp, u64* compbest, int* need, unsigned* count,
                                int* list);
appd_status launch_rows_exact(appd_ctx* c, const float* XT, int64_t ldx, int n, int d, const int* rows,
                              const unsigned* nrows, int max_rows, const int* comp, u64* compbest);
appd_status launch_rescan_blocks(appd_ctx* c, int n, const int* perm, const int* need, int* needp, int* blockflag,
                                 int nblocks, int* list, int* count);
appd_status launch_comp_ub(appd_ctx* c, int n, int k, const u64* compbest, const TcScale* s2, const int* perm,
                           const int* needp, const unsigned* UB, const int* comp, unsigned* compUB);
int64_t tcf_row_tiles(const TcState* st);
appd_status tcf_debug_gram(appd_ctx* c, const float* X, int64_t n, int64_t d, float* tc_out, float* ref_out);

void* ws(appd_ctx* c, int slot, size_t bytes);  // grows; returns nullptr on OOM
appd_status fail(appd_ctx* c, appd_status s, const char* fmt, ...);
appd_status cuda_fail(appd_ctx* c, cudaError_t e, const char* where);

#ifdef APPD_DEV_HOOKS
#define APPD_TRACE_SYNC(c) appd::trace_launch(c, "SYNC " __FILE__ ":" APPD_STR(__LINE__))
#define APPD_TRACE_OP(c) appd::trace_launch(c, "op " __FILE__ ":" APPD_STR(__LINE__))
#else
#define APPD_TRACE_SYNC(c) \
  do {                     \
  } while (0)
#define APPD_TRACE_OP(c) \
  do {                   \
  } while (0)
#endif
#define APPD_CUDA(c, expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return appd::cuda_fail(c, _e, #expr); \
    APPD_TRACE_OP(c);                                        \
  } while (0)

#define APPD_SYNC(c)                                 \
  do {                                               \
    APPD_TRACE_SYNC(c);                              \
    appd_status _s = appd::sync_stream(c);           \
    if (_s != APPD_OK) return _s;                    \
  } while (0)

#define APPD_STR2(x) #x
#define APPD_STR(x) APPD_STR2(x)
#ifdef APPD_DEV_HOOKS
// development builds: APPD_TRACE=1 records an event after every launch and prints, per
// solve, each launch site with its host issue time and the GPU time since the previous
// event (kernel + gap), to find where the GPU idles
void trace_launch(appd_ctx* c, const char* site);
void trace_begin(appd_ctx* c);
void trace_end(appd_ctx* c);
// development builds: APPD_SYNC_EACH=1 synchronises after every launch, so an
// asynchronous fault is reported at the kernel that caused it
#define APPD_DEV_SYNC_EACH(c)                                                                    \
  do {                                                                                          \
    static const bool _each = appd::dev_env("APPD_SYNC_EACH") != nullptr;                      \
    if (_each) {                                                                                \
      cudaError_t _e2 = cudaStreamSynchronize((c)->stream);                                     \
      if (_e2 != cudaSuccess) return appd::cuda_fail(c, _e2, "kernel " __FILE__ ":" APPD_STR(__LINE__)); \
    }                                                                                           \
    appd::trace_launch(c, __FILE__ ":" APPD_STR(__LINE__));                                     \
  } while (0)
#else
#define APPD_DEV_SYNC_EACH(c) \
  do {                        \
  } while (0)
#endif
#define APPD_LAUNCHED(c)                                                                        \
  do {                                                                                          \
    (c)->launches++;                                                                            \
    cudaError_t _e = cudaGetLastError();                                                        \
    if (_e != cudaSuccess) return appd::cuda_fail(c, _e, "kernel launch " __FILE__ ":" APPD_STR(__LINE__)); \
    APPD_DEV_SYNC_EACH(c);                                                                      \
  } while (0)

#ifdef __CUDACC__
// atomicMin that first reads the current value (L2): when many threads reduce onto few
// addresses (component minima in the late rounds), most lose and skip the serialised atomic
__device__ __forceinline__ void atomic_min_lt(unsigned long long* a, unsigned long long v) {
  if (v < __ldcg(a)) atomicMin(a, v);
}
__device__ __forceinline__ void atomic_min_lt(unsigned* a, unsigned v) {
  if (v < __ldcg(a)) atomicMin(a, v);
}
// sum of blocksum[0 .. blockIdx.x) for every thread of the block: warp 0 reduces with its
// loads in flight (a serial loop over up to 147 earlier blocks was ~20 us of dependent
// L2 latency in the last block of a cooperative scan)
// Grid-wide barrier of a cooperative launch (all CTAs co-resident): thread 0 of each CTA
// adds to the counter with release semantics -- CTA 0 adds 2^31 - (G - 1), the others 1, so
// the counter's top bit flips exactly when the last CTA arrives and its low 31 bits return
// to 0 (a zeroed word serves every launch and barrier) -- then spins with acquire loads on
// the flip.  The same protocol as cooperative_groups' grid sync, without its full fences
// before and after (the release add and the acquire load order the CTA's writes and reads).
// The arrival is a fire-and-forget red.add: the generation bit it must see flip is read
// before it (this CTA has not arrived yet, so the flip cannot have happened), and that read
// overlaps the CTA's own barrier.
__device__ __forceinline__ void coop_grid_sync(unsigned* bar) {
  unsigned gen = 0;
  if (threadIdx.x == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar) : "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned inc = blockIdx.x == 0 ? (0x80000000u - (gridDim.x - 1u)) : 1u;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(inc) : "memory");
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((gen ^ cur) & 0x80000000u) == 0u);
  }
  __syncthreads();
}
// the context's barrier word (allocated and zeroed on the context's stream at first use)
unsigned* grid_barrier_word(appd_ctx* c);

__device__ __forceinline__ int blocks_before(const int* blocksum) {
  __shared__ int bb_sum;
  if (threadIdx.x < 32) {
    int s = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += 32) s += blocksum[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) bb_sum = s;
  }
  __syncthreads();
  const int r = bb_sum;
  __syncthreads();
  return r;
}
#endif

// ---- kernels (k_*.cu) ----
// validation
appd_status launch_validate_weights(appd_ctx* c, const float* W, int64_t n, int64_t row0, int64_t rows,
                                    u64* out3 /*device, 3 minima*/);
appd_status launch_validate_points(appd_ctx* c, const float* X, int64_t n, int64_t d, u64* out3);
// position-keyed 64-bit checksum of count 32-bit words (world > 1 solve-start agreement)
appd_status launch_checksum_words(appd_ctx* c, const void* x, int64_t count, u64* out);

// Boruvka
appd_status launch_scan_weights(appd_ctx* c, const float* W, int64_t n, int64_t row0, int64_t rows,
                                const int* comp, u64* compbest, int sense);
appd_status launch_scan_weights_topk(appd_ctx* c, const float* W, int64_t n, int64_t row0, int64_t rows, int K,
                                     int sense, u64* ckey, int* cj, int* ccnt, u64* compbest);
appd_status launch_scan_weights_list(appd_ctx* c, const float* W, int64_t n, int64_t row0, const int* list,
                                     const unsigned* count, int max_rows, const int* comp, u64* compbest,
                                     int sense);
appd_status launch_transpose_points(appd_ctx* c, const float* X, int64_t n, int64_t d, float* XT, int64_t npad,
                                    int64_t dpad);
appd_status launch_scan_points(appd_ctx* c, const float* XT, int64_t n, int64_t npad, int64_t dpad, int64_t row0,
                               int64_t rows, const int* comp, u64* compbest, bool wide = false);
// wide keys (points, n > 131072): per-row winners -> two-step component reduction; the MST
// edges' Kruskal order and (u, v, w) from the pair indices (k_boruvka.cu)
appd_status launch_wide_compw(appd_ctx* c, const u64* rowbest, const int* comp, int64_t r0, int64_t r1, u64* compw);
appd_status launch_wide_compbest(appd_ctx* c, const u64* rowbest, const int* comp, int64_t r0, int64_t r1,
                                 const u64* compw, u64* compbest);
appd_status wide_edges(appd_ctx* c, const u64* mstkeys, int64_t m, const float* X, int64_t d, int metric, int sense,
                       u64* key2, u64* key2_sorted, int32_t* eu, int32_t* ev, float* ew);
// Small device -> host results: queue a copy of `bytes` (a multiple of 4) from device
// memory into pinned_small; the queued copies run as ONE kernel writing the mapped host
// words, launched by the next sync_stream (a 4-byte cudaMemcpyAsync costs ~5 us of stream
// time each).  Invariant: the source must not change between publish() and that
// synchronisation (every call site publishes a value its window no longer writes).
appd_status publish(appd_ctx* c, void* host_dst, const void* dev_src, size_t bytes);
appd_status publish_flush(appd_ctx* c);
#define APPD_PUBLISH(c, dst, src, bytes)                        \
  do {                                                          \
    appd_status _p = appd::publish(c, dst, src, bytes);         \
    if (_p != APPD_OK) return _p;                               \
  } while (0)
appd_status launch_fill_u64(appd_ctx* c, u64* p, int64_t count, u64 v);
appd_status launch_iota(appd_ctx* c, int* p, int64_t count);
appd_status launch_hook(appd_ctx* c, const u64* compbest, int64_t k, const int* comp, int shift, int* link);
appd_status launch_mutual(appd_ctx* c, const u64* compbest, int64_t k, const int* link, int* parent,
                          u64* mstkeys, int* counters /*[0]=mst count*/);
appd_status launch_jump(appd_ctx* c, int* parent, int64_t k, int* flags);
appd_status launch_relabel(appd_ctx* c, int* comp, int64_t n, const int* parent, const int* newid);
// the next round's candidate-cache lookup, queued in the same cooperative launch as the
// contraction (ckey == nullptr: none): compbest[0..n) = KEY_NONE, *count = 0, then
// k_cache_lookup and k_rescan_select over rows [r0, r1)
struct LookupArgs {
  int r0 = 0, r1 = 0, K = 0;
  const u64* ckey = nullptr;
  const int* cj = nullptr;
  const int* ccnt = nullptr;
  int* need = nullptr;
  unsigned* count = nullptr;
  int* list = nullptr;
  unsigned long long* marks = nullptr;  // development builds: per-phase %globaltimer
};
// hook + mutual + jump + scan + relabel (+ the lookup) in one cooperative launch
// (APPD_ERR_UNSUPPORTED if the device cannot co-schedule it: the caller then runs the
// separate kernels)
appd_status launch_contract(appd_ctx* c, u64* compbest, int64_t k, int* comp, int64_t n, int shift, int* link,
                            int* parent, u64* mstkeys, int* counters, int* flags, int* newid,
                            const LookupArgs* look = nullptr);

// fill
appd_status launch_positions(appd_ctx* c, const int* pi, int64_t n, int* pos);
appd_status launch_sparse_table(appd_ctx* c, float* ST, int64_t m, int levels, int64_t stride, int widest);
appd_status launch_fill(appd_ctx* c, const int* rows_sorted, const int* rowpos, int64_t nrows, const int* pos,
                        const float* ST, int64_t stride, int64_t n, float* M, int64_t row0, int widest);
appd_status launch_fill_f64(appd_ctx* c, const int* rows_sorted, const int* rowpos, int64_t nrows, const int* pos,
                            const float* ST, int64_t stride, int64_t n, double* M, int64_t row0, const double* hw);
appd_status launch_validate_weights_f64(appd_ctx* c, const double* W, int64_t n, u64* out3);
appd_status launch_scan_weights_f64(appd_ctx* c, const double* W, int64_t n, int64_t k, bool round0, int sense,
                                    const int* comp, u64* compw, u64* roww, int* rowj, u64* compbest);
appd_status launch_edges_f64(appd_ctx* c, const u64* mstkeys, int64_t m, const double* W, int64_t n, int sense,
                             u64* wkey, u64* wkey_sorted, int* idx, int* idx_sorted, int32_t* eu, int32_t* ev,
                             float* ew, double* hw);
appd_status launch_set_diag_zero_single_f64(appd_ctx* c, double* M);
appd_status launch_sqrt_inplace(appd_ctx* c, float* h, int64_t m);
appd_status launch_set_diag_zero_single(appd_ctx* c, float* M);
appd_status launch_points_weights(appd_ctx* c, const float* X, int64_t n, int64_t d, int64_t row0, int64_t rows,
                                  float* Wb);
appd_status launch_gather_rowpos(appd_ctx* c, const int* pos, int64_t row0, int64_t rows, int* keys, int* vals);

// Prim variant (k_prim.cu): one persistent CTA; validation fused (bad != nullptr), then
// pi, pos, rowpos = iota and the whole sparse table over h
// (small n: M != nullptr also writes this rank's rows of the APPD in the same launch)
bool prim_fits(int64_t n, int64_t d, bool points);
bool prim_fuses_fill(int64_t n);
appd_status launch_prim(appd_ctx* c, const float* W, const float* X, int64_t n, int64_t d, int sense, int metric,
                        u64* bad, int* pi, int* pos, int* rowpos, float* ST, int64_t stride, int levels, float* M,
                        int64_t row0, int64_t rows);

// sorting (CUB)
appd_status sort_keys_u64(appd_ctx* c, const u64* in, u64* out, int64_t count);
appd_status sort_keys_u32_bits(appd_ctx* c, const unsigned* in, unsigned* out, int64_t count, int begin_bit, int end_bit);
appd_status sort_pairs_i32(appd_ctx* c, const int* kin, int* kout, const int* vin, int* vout, int64_t count);
appd_status sort_pairs_i32_bits(appd_ctx* c, const int* kin, int* kout, const int* vin, int* vout, int64_t count,
                                int end_bit);
// component labels (< 2^bits, bits <= 8) -> sorted labels sc and positions perm (stable),
// plus the label ranges cstart / cend and per position rs / re, in one cooperative launch
// (APPD_ERR_UNSUPPORTED for wider labels)
appd_status sort_components(appd_ctx* c, const int* comp, int64_t n, int bits, int* sc, int* perm, int* cstart,
                            int* cend, int* rs, int* re);
appd_status sort_keys_u64_bits64(appd_ctx* c, const u64* in, u64* out, int64_t count, int begin_bit, int end_bit);
appd_status exclusive_scan_i32(appd_ctx* c, const int* in, int* out, int64_t count);

// host dendrogram (dendrogram_host.cpp)
void host_dendrogram(const u64* sorted_keys, int64_t n, const KeySpec& ks, int32_t* pi, float* h);
void host_dendrogram_uvw(const int32_t* eu, const int32_t* ev, const float* ew, int64_t n, int32_t* pi, float* h,
                         int32_t* scratch /* 8 n */);
appd_status gpu_dendrogram(appd_ctx* c, const int32_t* eu, const int32_t* ev, const float* ew, int64_t n,
                           int32_t* pi, float* h, int* pos_out, int* rowpos_out, bool* fused_pos);
appd_status launch_decode_edges(appd_ctx* c, const u64* keys, int64_t m, const KeySpec& ks, int32_t* eu,
                                int32_t* ev, float* ew);
void* pinned_host(appd_ctx* c, size_t bytes);  // grows ctx->pinned

// NCCL (nccl_shim.cpp)
appd_status nccl_unique_id(uint8_t out[128], std::string* err);
appd_status nccl_init(appd_ctx* c, const uint8_t* id, int rank, int world);
appd_status nccl_allreduce_min_u64(appd_ctx* c, u64* buf, int64_t count);
appd_status nccl_allreduce_max_u64(appd_ctx* c, u64* buf, int64_t count);
// wait for the context stream (world > 1 NCCL: polled against opt.timeout_ms and the
// communicator's asynchronous error; the communicator is aborted on failure)
appd_status sync_stream(appd_ctx* c);
void nccl_destroy(appd_ctx* c);

}  // namespace appd
