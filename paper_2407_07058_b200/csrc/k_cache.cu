// k_cache.cu -- the per-row candidate cache of the points-mode Boruvka rounds
// ("Round 0: ... v2 keeps a top-K cache.  Round r: per row,
// first cached eligible candidate; rescan a row only if its cache is exhausted and
// its K-th key <= its component's best"; App. B measured ~2 full-pass equivalents
// instead of one pass per round).
//
// Round 0 (singletons) runs the tensor-core scan once with one maximum of G' per
// 32 columns (TM32).  For each row p:
//   k_topk_scan    the K-th largest chunk maximum gives an upper bound UBK of s^2 r
//                  for K distinct columns (each chunk's best column), hence for the
//                  row's K-th smallest exact R1 value; every chunk whose maximum meets
//                  the G' threshold of UBK (tc_common.cuh error model) is listed;
//   k_list_exact   the listed (chunk, row) pairs, sorted by chunk, are re-evaluated
//                  with the exact R1 chain (register-blocked, chunk columns and rows
//                  staged in shared memory); every column with s^2 r <= UBK is
//                  appended to the row's candidate list;
//   k_topk_select  the K smallest exact edge keys of the list are the row's cache.
// Every column not appended has s^2 r > UBK >= the K-th appended value, so the cache
// is exactly the row's K smallest keys (keys are a strict order: weight, then pair
// index).  A row whose list overflows is marked invalid (exact full-row minimum now,
// re-scan in every later round).
//
// Round r >= 1:
//   k_cache_lookup   first cached entry whose column lies in another component: that
//                    is the row's exact minimum eligible key (everything cheaper is
//                    cached and ineligible) -> atomicMin into its component;
//   k_rescan_select  a row with no eligible cached entry needs a re-scan only if its
//                    K-th key is below its component's current best (else all of its
//                    uncached edges are heavier than an edge the component already has).
#include <cfloat>
#include <vector>

#include <cooperative_groups.h>

#include "tc_common.cuh"

namespace appd {
namespace cg = cooperative_groups;

// list entries: (32-column chunk << LIST_SHIFT) | row position (n <= 2^17, chunks < 2^12)
constexpr int LIST_SHIFT = 17;
constexpr unsigned LIST_ROWMASK = (1u << LIST_SHIFT) - 1u;

// warp-aggregated append of cnt entries per lane: returns this lane's first slot
__device__ __forceinline__ unsigned warp_alloc(unsigned* counter, unsigned cnt) {
  const int lane = threadIdx.x & 31;
  unsigned incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - cnt;
}

// One pass over TM32.  A CTA of TK_PARTS warps takes 32 rows (lane = row); warp w scans
// the w-th quarter of the chunks, 32 maxima per batch with the next batch's loads in
// flight (cp.async ring), storing the maximum of every 8-chunk group (shared memory)
// and keeping the running K largest BATCH maxima (one insertion per 32 chunks).  K
// batches hold K distinct chunks, so the merged K-th largest batch maximum gK is a lower
// bound of the row's K-th largest chunk maximum.  Every group whose maximum reaches
// t = min(thr(gK), gK) is then read again (one 16-byte load, TK_RG groups per lane in
// flight): its chunks >= t are kept (shared memory) and enter the chunk-level top-K.
// Every chunk of the row's K largest is >= gK >= t, so the merged chunk-level list is
// the exact K largest, which give UBK and the listing threshold thrK >= t; the kept
// chunks passing thrK are listed.  A (row, quarter) keeping more than TK_SEL chunks reads
// its flagged groups once more; a row whose list entries do not fit is poisoned
// (cand_cnt = 2^31: invalid cache, exact full-row minimum).
constexpr int TK_PARTS = 4;
constexpr int TK_BATCH = 32;  // chunk maxima per batch (4 x 128-bit loads of fp16)
constexpr int TK_SEL = 16;    // kept chunks per (row, quarter) in shared memory
constexpr int TK_RG = 4;      // flagged groups re-read together
constexpr int TK_STAGES = 3;  // cp.async ring depth (batches; 2 in flight while one is processed)

// 16-byte asynchronous global -> shared copy (L2 only); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// packed FP32 pairs (FADD2 / FFMA2 on sm_100a): each half is the IEEE round-to-nearest
// result of the scalar operation, so the R1 chain is unchanged, at half the issue slots
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// acc + (a - b)^2 per half: sub.rn then fma.rn (the R1 step)
__device__ __forceinline__ unsigned long long f2_r1_step(unsigned long long a, unsigned long long b,
                                                         unsigned long long acc) {
  unsigned long long t, r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(a), "l"(b));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(t), "l"(acc));
  return r;
}

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// insert x into the descending list top[0..K) (branch-free network)
template <int K>
__device__ __forceinline__ void topk_insert(float (&top)[K], float x) {
#pragma unroll
  for (int t = 0; t < K; t++) {
    const float hi = fmaxf(top[t], x);
    x = fminf(top[t], x);
    top[t] = hi;
  }
}

// merge the other quarters' descending lists (shared memory) into top
template <int K>
__device__ __forceinline__ void topk_merge(float (&top)[K], const float (*stop)[K][32], int w, int lane) {
#pragma unroll
  for (int o = 0; o < TK_PARTS; o++) {
    if (o == w) continue;
    for (int t = 0; t < K; t++) {
      const float x = stop[o][t][lane];
      if (!(x > top[K - 1])) break;  // lists are descending
      topk_insert(top, x);
    }
  }
}

// 8 stored chunk values (fp16 distance estimates D', tm_store; one 16-byte piece of the
// packed table) -> floats
__device__ __forceinline__ void h8(const uint4 x, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&x);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

template <int K>
__global__ void __launch_bounds__(32 * TK_PARTS) k_topk_scan(const __half* __restrict__ TM32, int nch, int p_begin,
                                                             int p_end, const float* __restrict__ nrm,
                                                             const float* __restrict__ len, const TcScale* __restrict__ sc,
                                                             const float* __restrict__ err,
                                                             const float* __restrict__ maxerr, ErrModel em,
                                                             float* __restrict__ UBK, unsigned* __restrict__ list,
                                                             unsigned* __restrict__ count, unsigned cap,
                                                             unsigned* __restrict__ cand_cnt, int ngq) {
  extern __shared__ __align__(16) __half sgm[];   // [TK_PARTS][ngq][32] 8-chunk group minima of D' (fp16: exact)
  __shared__ float stop[TK_PARTS][K][32];         // per-quarter top-K lists for the merges
  __shared__ __half sval[TK_PARTS][TK_SEL][32];   // kept chunks: stored D' (fp16: exact)
  __shared__ unsigned short sidx[TK_PARTS][TK_SEL][32];  //   and chunk index
  __shared__ int slost[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float maxlen = sc->maxlen;
  constexpr int U8 = TK_BATCH / 8;  // 16-byte pieces per batch
  const int nch8 = (nch + 7) >> 3;
  const int g0 = (int)((int64_t)w * nch8 / TK_PARTS), g1 = (int)((int64_t)(w + 1) * nch8 / TK_PARTS);
  const int cb = 8 * g0, cend = min(nch, 8 * g1);  // this warp's chunk range (whole 8-chunk groups)
  const int nbat = (cend - cb + TK_BATCH - 1) / TK_BATCH;
  const int ng = (cend - cb + 7) / 8;               // 8-chunk groups of this quarter (<= ngq)
  __half* gm = sgm + (size_t)w * ngq * 32 + lane;   // gm[g * 32]
  // cp.async ring after the group maxima: [TK_PARTS][TK_STAGES][U8][32] uint4
  // (ngq * 32 halves per warp: a multiple of 16 bytes)
  uint4* ring = reinterpret_cast<uint4*>(sgm + (size_t)TK_PARTS * ((ngq + 1) & ~1) * 32) + (size_t)w * TK_STAGES * U8 * 32 + lane;
  for (int p0 = p_begin + 32 * blockIdx.x; p0 < p_end; p0 += 32 * gridDim.x) {
    const int p = p0 + lane;
    const bool valid = p < p_end;
    if (w == 0) slost[lane] = 0;
    const uint4* row8 = reinterpret_cast<const uint4*>(TM32 + tm32_index(0, valid ? p : p_begin, nch));
    const float ni = valid ? nrm[p] : 0.0f;  // the encoding's |y^_p|^2 (tm_low / tm_up)
    // the 8 chunks of group c .. c+7 (c a multiple of 8; chunks past cend read as +inf:
    // no eligible column)
    auto load8 = [&](int c, float (&f)[8]) {
      if (valid && c < cend) h8(__ldcs(row8 + (int64_t)(c >> 3) * 512), f);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (!valid || c + u >= cend) f[u] = INFINITY;
    };
    // ---- scan: group maxima and the top-K of group maxima.  Batches are staged by
    // cp.async into a TK_STAGES ring (each lane copies and reads only its own row's 16-byte
    // pieces, so its own wait_group orders them; no warp synchronisation)
    float top[K];
#pragma unroll
    for (int t = 0; t < K; t++) top[t] = -INFINITY;
    auto issue = [&](int b) {
      if (b < nbat) {
#pragma unroll
        for (int u = 0; u < U8; u++) {
          const int c = cb + b * TK_BATCH + 8 * u;
          const bool ok = valid && c < cend;
          cp_async16(&ring[((b % TK_STAGES) * U8 + u) * 32], row8 + (int64_t)((ok ? c : cb) >> 3) * 512, ok ? 16 : 0);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int b = 0; b < TK_STAGES - 1; b++) issue(b);
    for (int b = 0; b < nbat; b++) {
      issue(b + TK_STAGES - 1);
      cp_async_wait<TK_STAGES - 1>();
      // (rows past p_end hold zero-filled data; nothing of theirs is written)
      // the group minimum of D' (= maximum of G') in half2 arithmetic, then one decode
      float bd = INFINITY;
#pragma unroll
      for (int q = 0; q < U8; q++) {
        const uint4 x = ring[((b % TK_STAGES) * U8 + q) * 32];
        const int c = cb + b * TK_BATCH + 8 * q;
        float m;
        if (c + 8 > cend) {  // the quarter's ragged end (warp-uniform)
          float f[8];
          h8(x, f);
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (c + u >= cend) f[u] = INFINITY;
          m = fminf(fminf(fminf(f[0], f[1]), fminf(f[2], f[3])), fminf(fminf(f[4], f[5]), fminf(f[6], f[7])));
        } else {
          const __half2* hh = reinterpret_cast<const __half2*>(&x);
          const __half2 t = __hmin2(__hmin2(hh[0], hh[1]), __hmin2(hh[2], hh[3]));
          m = fminf(__low2float(t), __high2float(t));
        }
        const int g = b * (TK_BATCH / 8) + q;
        if (g < ng) gm[g * 32] = __float2half_rn(m);  // (m is an fp16 value or +inf: exact)
        bd = fminf(bd, m);
      }
      // top-K of BATCH maxima (lower bounds): K batches hold K distinct chunks
      const float bm = bd == INFINITY ? -INFINITY : tm_low(bd, ni);
      if (bm > top[K - 1]) topk_insert(top, bm);
    }
    cp_async_wait<0>();
#pragma unroll
    for (int t = 0; t < K; t++) stop[w][t][lane] = top[t];
    __syncthreads();
    topk_merge(top, stop, w, lane);
    const float gK = top[K - 1];
    float li = 0.0f, dl = 0.0f;
    if (valid) {
      li = len[p];
      dl = em_delta2(err[p], *maxerr);
    }
    // capture threshold t (fewer than K finite group maxima: every finite chunk).  The
    // top-K is of lower bounds tm_low (gK, UBK stay valid); every test against a
    // threshold takes the upper bound tm_up (the listing keeps every candidate)
    float tcap = valid ? -INFINITY : INFINITY;
    if (valid && gK > -INFINITY) tcap = fminf(gK, em_thr(em, em_upper(em, ni - 2.0f * gK, ni, li, maxlen, dl), ni, li, maxlen, dl));
    auto flagged = [&](int g) {
      const float dg = __half2float(gm[g * 32]);
      return dg < INFINITY && tm_up(dg, ni) >= tcap;
    };
    // ---- re-read the flagged groups (bit masks, ng <= 128): keep chunks >= t,
    // chunk-level top-K
    unsigned long long fm0 = 0, fm1 = 0;
    for (int g = 0; g < ng; g++) {
      if (!flagged(g)) continue;
      if (g < 64) fm0 |= 1ull << g;
      else fm1 |= 1ull << (g - 64);
    }
    int jmax = __popcll(fm0) + __popcll(fm1);
#pragma unroll
    for (int o = 16; o; o >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
#pragma unroll
    for (int t = 0; t < K; t++) top[t] = -INFINITY;
    unsigned kept = 0;
    for (int j = 0; j < jmax; j += TK_RG) {
      int gg[TK_RG];
      float vv[TK_RG][8];
#pragma unroll
      for (int r = 0; r < TK_RG; r++) {
        if (fm0) {
          gg[r] = __ffsll(fm0) - 1;
          fm0 &= fm0 - 1;
        } else if (fm1) {
          gg[r] = 63 + __ffsll(fm1);
          fm1 &= fm1 - 1;
        } else {
          gg[r] = -1;
        }
        if (gg[r] >= 0) load8(cb + 8 * gg[r], vv[r]);
        else
#pragma unroll
          for (int u = 0; u < 8; u++) vv[r][u] = INFINITY;
      }
#pragma unroll
      for (int r = 0; r < TK_RG; r++) {
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (vv[r][u] < INFINITY && tm_up(vv[r][u], ni) >= tcap) {
            if (kept < TK_SEL) {
              sval[w][kept][lane] = __float2half_rn(vv[r][u]);
              sidx[w][kept][lane] = (unsigned short)(cb + 8 * gg[r] + u);
            }
            kept++;
            const float lo = tm_low(vv[r][u], ni);
            if (lo > top[K - 1]) topk_insert(top, lo);
          }
      }
    }
    __syncthreads();  // every warp has merged the group-level lists
#pragma unroll
    for (int t = 0; t < K; t++) stop[w][t][lane] = top[t];
    __syncthreads();
    topk_merge(top, stop, w, lane);
    // fewer than K finite chunks: UBK = inf and every finite chunk is listed
    float ub = INFINITY, thr = tcap;
    if (valid && top[K - 1] > -INFINITY) {
      ub = em_upper(em, ni - 2.0f * top[K - 1], ni, li, maxlen, dl);
      thr = em_thr(em, ub, ni, li, maxlen, dl);
    }
    if (valid && w == 0) UBK[p] = ub;
    // ---- list the kept chunks passing thrK: count, one warp allocation, write
    unsigned mine = 0;
    if (kept <= TK_SEL) {
      for (unsigned t = 0; t < kept; t++) mine += tm_up(__half2float(sval[w][t][lane]), ni) >= thr;
    } else {
      for (int g = 0; g < ng; g++) {
        if (!flagged(g)) continue;
        float vv[8];
        load8(cb + 8 * g, vv);
#pragma unroll
        for (int u = 0; u < 8; u++) mine += vv[u] < INFINITY && tm_up(vv[u], ni) >= thr;
      }
    }
    unsigned slot = warp_alloc(count, mine);
    bool lost = false;
    if (kept <= TK_SEL) {
      for (unsigned t = 0; t < kept; t++)
        if (tm_up(__half2float(sval[w][t][lane]), ni) >= thr) {
          if (slot < cap) list[slot] = ((unsigned)sidx[w][t][lane] << LIST_SHIFT) | (unsigned)p;
          else lost = true;
          slot++;
        }
    } else {  // more than TK_SEL kept chunks (rare): read the flagged groups again
      for (int g = 0; g < ng; g++) {
        if (!flagged(g)) continue;
        float vv[8];
        load8(cb + 8 * g, vv);
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (vv[u] < INFINITY && tm_up(vv[u], ni) >= thr) {
            if (slot < cap) list[slot] = ((unsigned)(cb + 8 * g + u) << LIST_SHIFT) | (unsigned)p;
            else lost = true;
            slot++;
          }
      }
    }
    if (lost) slost[lane] = 1;
    __syncthreads();  // shared state reused by the next row group
    if (w == 0 && valid && slost[lane]) cand_cnt[p] = 0x80000000u;  // poisoned (cannot wrap back below the cap)
  }
}

appd_status launch_topk_scan(appd_ctx* c, int K, const __half* TM32, int nch, int p_begin, int p_end,
                             const float* nrm, const float* len, const TcScale* sc, const float* err,
                             const float* maxerr, const ErrModel& em, float* UBK, unsigned* list, unsigned* count,
                             unsigned cap, unsigned* cand_cnt) {
  const int rows = p_end - p_begin;
  if (rows <= 0) return APPD_OK;
  const int grid = std::min(c->sm_count * 16, (rows + 31) / 32);
  // 8-chunk groups per quarter: the largest quarter has ceil(ceil(nch/8)/TK_PARTS)
  const int ngq = ((nch + 7) / 8 + TK_PARTS - 1) / TK_PARTS;
  const size_t smem = sizeof(__half) * TK_PARTS * ((ngq + 1) & ~1) * 32 + sizeof(uint4) * TK_PARTS * TK_STAGES * (TK_BATCH / 8) * 32;
  if (ngq > 128) return fail(c, APPD_ERR_UNSUPPORTED, "top-K scan: %d chunks per row", nch);
#define APPD_TOPK_SCAN(KK)                                                                                     \
  do {                                                                                                         \
    static std::atomic<unsigned long long> attr_##KK{0};                                                       \
    if (needs_setup(attr_##KK, c)) {                                                                           \
      cudaFuncSetAttribute(k_topk_scan<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);          \
      setup_done(attr_##KK, c);                                                                                \
    }                                                                                                          \
    k_topk_scan<KK><<<grid, 32 * TK_PARTS, smem, c->stream>>>(TM32, nch, p_begin, p_end, nrm, len, sc, err, \
                                                              maxerr, em, UBK, list, count, cap, cand_cnt, ngq); \
  } while (0)
  switch (K) {
    case 4: APPD_TOPK_SCAN(4); break;
    case 8: APPD_TOPK_SCAN(8); break;
    case 16: APPD_TOPK_SCAN(16); break;
    case 32: APPD_TOPK_SCAN(32); break;
    default: return fail(c, APPD_ERR_INVALID_ARGUMENT, "cache length K = %d (4, 8, 16 or 32)", K);
  }
#undef APPD_TOPK_SCAN
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// Exact R1 re-check of a chunk-sorted list of (32-column chunk, row) pairs.  One CTA
// per chunk at a time (dynamic): the chunk's 32 columns are staged transposed in shared
// memory (colx[k][32]), its listed rows 128 at a time (rowx[k][128]); thread (ty, tx)
// owns a 4 x 4 micro-tile (rows 4ty.., columns 4tx..) and runs the pinned R1 chain
// with two 128-bit shared loads per 32 FP32 operations.  Positions p, q index the
// (possibly permuted) order; X is read at the original indices perm[p], perm[q].
//   MODE 0 (cache build): append every column with s^2 r <= UBK[p] to row p's list;
//   MODE 1 (component matrix): WCM[sc[p]][sc[q]] = min exact key over the pairs.
// ---------------------------------------------------------------------------

constexpr int LE_RB = 128;

__device__ __forceinline__ unsigned lower_bound_u32(const unsigned* a, unsigned n, unsigned key) {
  unsigned lo = 0, hi = n;
  while (lo < hi) {
    const unsigned mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// per chunk: first entry and number of 128-row batches (the sorted list's runs)
__global__ void k_chunk_runs(const unsigned* __restrict__ list, const unsigned* __restrict__ count, unsigned cap,
                             int nch, unsigned* __restrict__ run_lo, unsigned* __restrict__ run_nb) {
  const unsigned total = min(*count, cap);
  for (int ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nch; ch += gridDim.x * blockDim.x) {
    const unsigned lo = lower_bound_u32(list, total, (unsigned)ch << LIST_SHIFT);
    const unsigned hi = lower_bound_u32(list, total, (unsigned)(ch + 1) << LIST_SHIFT);
    run_lo[ch] = lo;
    run_nb[ch] = (hi - lo + LE_RB - 1) / LE_RB;
  }
}

// Counting sort of the list by chunk (no host-side count) in ONE cooperative launch (it
// was seven kernels, scans and memsets: 60-100 us at C4): clear, histogram, a two-array
// exclusive scan over chunk ranges per block (offsets and 128-row batch starts), item
// table (item -> chunk, first entry, rows), scatter.  The listing is emitted chunk-major
// (runs of one chunk), so the lanes of a warp mostly share a chunk: one atomic per
// distinct chunk in the warp; the lanes of one chunk take consecutive slots in lane
// order, so runs of rows listed together (one filter warp: consecutive rows, mostly one
// component) stay together and in order.
struct ListSortArgs {
  const unsigned* list;
  const unsigned* count;
  unsigned cap;
  int nch;
  unsigned *hist, *offs, *cursor, *out, *run_lo, *run_nb, *item_start;
  int4* items;
  unsigned* blocksum;  // 2 per block
  unsigned long long* marks;  // development builds (APPD_MARKS): %globaltimer per phase, CTA 0
  int aggregate;              // the listing comes in chunk runs: warp-aggregated atomics
  unsigned* cnt;              // (no runs) [nch][grid] per-CTA counts, then their offsets
  unsigned* bar;              // grid barrier word (coop_grid_sync)
};
__device__ __forceinline__ void ls_mark(const ListSortArgs& a, int i) {
  if (a.marks && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.marks[i] = t;
  }
}
__global__ void __launch_bounds__(1024) k_list_sort(const ListSortArgs a) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned total = min(*a.count, a.cap);
  ls_mark(a, 0);
  for (int64_t i = tid; i <= a.nch; i += nt) {
    a.hist[i] = 0u;
    a.cursor[i] = 0u;
  }
  coop_grid_sync(a.bar);
  ls_mark(a, 1);
  // no chunk runs (round 0: the listing is in row order, chunks at random): global atomics
  // would serialise (~23 us for 640K entries), so every CTA counts its contiguous slice of
  // the entries in shared memory and the [chunk][CTA] counts are scanned chunk-major
  extern __shared__ unsigned sh[];  // [nch] (no-runs path)
  const unsigned G = gridDim.x;
  const unsigned e_lo = (unsigned)((uint64_t)total * blockIdx.x / G), e_hi = (unsigned)((uint64_t)total * (blockIdx.x + 1) / G);
  if (a.aggregate) {
    for (unsigned e0 = (unsigned)(tid & ~31ll); e0 < total; e0 += (unsigned)nt) {  // histogram
      const unsigned e = e0 + lane;
      const unsigned ch = e < total ? a.list[e] >> LIST_SHIFT : 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, ch);
      if (e < total && lane == __ffs(peers) - 1) atomicAdd(a.hist + ch, (unsigned)__popc(peers));
    }
  } else {
    for (int i = threadIdx.x; i < a.nch; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    for (unsigned e = e_lo + threadIdx.x; e < e_hi; e += blockDim.x) atomicAdd(sh + (a.list[e] >> LIST_SHIFT), 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < a.nch; i += blockDim.x) a.cnt[(int64_t)i * G + blockIdx.x] = sh[i];
  }
  coop_grid_sync(a.bar);
  ls_mark(a, 2);
  if (!a.aggregate) {  // chunk totals, and each CTA's offset inside its chunk (a warp per chunk)
    for (int i = (int)(tid >> 5); i < a.nch; i += (int)(nt >> 5)) {
      unsigned carry = 0u, pre[8];  // the loads of up to 8 x 32 CTAs first, all in flight
#pragma unroll
      for (int u = 0; u < 8; u++) pre[u] = (u * 32u + lane < G) ? a.cnt[(int64_t)i * G + u * 32 + lane] : 0u;
      auto step = [&](unsigned v, unsigned j) {  // exclusive offsets of 32 CTAs, running carry
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (j < G) a.cnt[(int64_t)i * G + j] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      };
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u * 32u < G) step(pre[u], u * 32u + lane);
      for (unsigned j0 = 256; j0 < G; j0 += 32) step(j0 + lane < G ? a.cnt[(int64_t)i * G + j0 + lane] : 0u, j0 + lane);
      if (lane == 0) a.hist[i] = carry;
    }
    coop_grid_sync(a.bar);
  }
  // block b scans chunks [lo, hi): entries (offsets) and 128-row batches (item starts)
  __shared__ unsigned ws1[32], ws2[32];
  __shared__ unsigned carry1, carry2;
  const int Sg = (a.nch + gridDim.x - 1) / gridDim.x;
  const int lo = min(a.nch, (int)blockIdx.x * Sg), hi = min(a.nch, lo + Sg);
  if (threadIdx.x == 0) carry1 = carry2 = 0u;
  __syncthreads();
  for (int base = lo; base < hi; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const unsigned f1 = i < hi ? a.hist[i] : 0u, f2 = (f1 + LE_RB - 1) / LE_RB;
    unsigned x1 = f1, x2 = f2;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y1 = __shfl_up_sync(0xffffffffu, x1, o), y2 = __shfl_up_sync(0xffffffffu, x2, o);
      if (lane >= o) { x1 += y1; x2 += y2; }
    }
    if (lane == 31) { ws1[warp] = x1; ws2[warp] = x2; }
    __syncthreads();
    if (warp == 0) {
      unsigned w1 = lane < (int)(blockDim.x >> 5) ? ws1[lane] : 0u, w2 = lane < (int)(blockDim.x >> 5) ? ws2[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y1 = __shfl_up_sync(0xffffffffu, w1, o), y2 = __shfl_up_sync(0xffffffffu, w2, o);
        if (lane >= o) { w1 += y1; w2 += y2; }
      }
      ws1[lane] = w1;
      ws2[lane] = w2;
    }
    __syncthreads();
    if (i < hi) {
      a.offs[i] = carry1 + (warp ? ws1[warp - 1] : 0u) + x1 - f1;
      a.item_start[i] = carry2 + (warp ? ws2[warp - 1] : 0u) + x2 - f2;
      a.run_nb[i] = f2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry1 += ws1[(blockDim.x >> 5) - 1];
      carry2 += ws2[(blockDim.x >> 5) - 1];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.blocksum[2 * blockIdx.x] = carry1;
    a.blocksum[2 * blockIdx.x + 1] = carry2;
  }
  coop_grid_sync(a.bar);
  ls_mark(a, 3);
  // the sums of the earlier blocks' totals (a block-wide reduction, not a serial loop)
  if (warp == 0) {
    unsigned s1 = 0u, s2 = 0u;
    for (int b = lane; b < (int)blockIdx.x; b += 32) {
      s1 += a.blocksum[2 * b];
      s2 += a.blocksum[2 * b + 1];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      ws1[0] = s1;
      ws2[0] = s2;
    }
  }
  __syncthreads();
  const unsigned off1 = ws1[0], off2 = ws2[0];
  for (int i = lo + warp; i < hi; i += blockDim.x >> 5) {  // a warp per chunk: its item table
    const unsigned o1 = a.offs[i] + off1, o2 = a.item_start[i] + off2, h = a.hist[i], nb = a.run_nb[i];
    __syncwarp();
    if (lane == 0) {
      a.offs[i] = o1;
      a.item_start[i] = o2;
      a.run_lo[i] = o1;
    }
    for (unsigned b = lane; b < nb; b += 32) {
      const unsigned b0 = o1 + b * LE_RB;
      a.items[o2 + b] = make_int4(i, (int)b0, (int)min((unsigned)LE_RB, o1 + h - b0), 0);
    }
  }
  coop_grid_sync(a.bar);
  ls_mark(a, 4);
  if (a.aggregate) {
    for (unsigned e0 = (unsigned)(tid & ~31ll); e0 < total; e0 += (unsigned)nt) {  // scatter
      const unsigned e = e0 + lane;
      const bool ok = e < total;
      const unsigned v = ok ? a.list[e] : 0xFFFFFFFFu, ch = v >> LIST_SHIFT;
      const unsigned peers = __match_any_sync(0xffffffffu, ch);
      const int leader = __ffs(peers) - 1;
      unsigned b = 0;
      if (ok && lane == leader) b = atomicAdd(a.cursor + ch, (unsigned)__popc(peers));
      b = __shfl_sync(peers, b, leader);
      if (ok) a.out[a.offs[ch] + b + __popc(peers & ((1u << lane) - 1u))] = v;
    }
  } else {  // this CTA's slice again, cursors in shared memory from the scanned counts
    for (int i = threadIdx.x; i < a.nch; i += blockDim.x) sh[i] = a.offs[i] + a.cnt[(int64_t)i * G + blockIdx.x];
    __syncthreads();
    for (unsigned e = e_lo + threadIdx.x; e < e_hi; e += blockDim.x) {
      const unsigned v = a.list[e];
      a.out[atomicAdd(sh + (v >> LIST_SHIFT), 1u)] = v;
    }
  }
  ls_mark(a, 5);
}

appd_status launch_list_counting(appd_ctx* c, const unsigned* list, const unsigned* count, unsigned cap, int nch,
                                 unsigned* hist, unsigned* offs, unsigned* cursor, unsigned* out, unsigned* run_lo,
                                 unsigned* run_nb, unsigned* item_start, int4* items, bool aggregate) {
  unsigned* blocksum = (unsigned*)ws(c, S_SCAN, sizeof(unsigned) * 2 * (c->sm_count + 1) + 64);
  if (!blocksum) return fail(c, APPD_ERR_OUT_OF_MEMORY, "list sort workspace");
  unsigned* cnt = nullptr;
  if (!aggregate) {
    cnt = (unsigned*)ws(c, S_LIST_CNT, sizeof(unsigned) * (size_t)nch * c->sm_count + 64);
    if (!cnt) return fail(c, APPD_ERR_OUT_OF_MEMORY, "list sort counts");
  }
  ListSortArgs a{list, count, cap, nch, hist, offs, cursor, out, run_lo, run_nb, item_start, items, blocksum, nullptr,
                 aggregate ? 1 : 0, cnt, grid_barrier_word(c)};
  if (!a.bar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
  const size_t smem = aggregate ? 0 : sizeof(unsigned) * nch;
  if (smem > 64 * 1024) return fail(c, APPD_ERR_UNSUPPORTED, "list sort: %d chunks", nch);
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
    cudaFuncSetAttribute(k_list_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    setup_done(attr, c);
  }
  static const bool marks = dev_env("APPD_MARKS") != nullptr;
  if (marks) a.marks = reinterpret_cast<unsigned long long*>(ws(c, S_TMP2, 64));
  void* args[] = {&a};
  APPD_CUDA(c, cudaLaunchCooperativeKernel((const void*)k_list_sort, c->sm_count, 1024, args, smem, c->stream));
  APPD_LAUNCHED(c);
  if (marks && a.marks) {
    unsigned long long h[6];
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(h, a.marks, sizeof h, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[list_sort] clear %.1f us, hist %.1f, scan %.1f, items %.1f, scatter %.1f\n", (h[1] - h[0]) * 1e-3,
            (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3, (h[4] - h[3]) * 1e-3, (h[5] - h[4]) * 1e-3);
    std::vector<unsigned> hh(nch);
    cudaMemcpy(hh.data(), hist, sizeof(unsigned) * nch, cudaMemcpyDeviceToHost);
    unsigned mx = 0, tot = 0, big = 0;
    for (unsigned v : hh) {
      mx = std::max(mx, v);
      tot += v;
      big += v > 4096;
    }
    fprintf(stderr, "[list_sort] entries %u, chunks %d, max per chunk %u, chunks over 4096: %u\n", tot, nch, mx, big);
  }
  return APPD_OK;
}

// item table: item -> (chunk, first list entry, rows), one thread per chunk
__global__ void k_item_table(const unsigned* __restrict__ run_lo, const unsigned* __restrict__ run_nb,
                             const unsigned* __restrict__ item_start, const unsigned* __restrict__ list,
                             const unsigned* __restrict__ count, unsigned cap, int nch, int4* __restrict__ table) {
  const unsigned total = min(*count, cap);
  for (int ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nch; ch += gridDim.x * blockDim.x) {
    const unsigned lo = run_lo[ch], nb = run_nb[ch], base = item_start[ch];
    const unsigned hi = lower_bound_u32(list, total, (unsigned)(ch + 1) << LIST_SHIFT);
    for (unsigned b = 0; b < nb; b++) {
      const unsigned b0 = lo + b * LE_RB;
      table[base + b] = make_int4(ch, (int)b0, (int)min((unsigned)LE_RB, hi - b0), 0);
    }
  }
}

// Work item = (chunk, 128-row batch): item_start is the exclusive prefix of run_nb, so
// dense candidate chunks (component boundaries) spread over many CTAs.
template <int MODE>
__global__ void __launch_bounds__(256, MODE == 0 ? 5 : 4) k_list_exact(ListParams L) {
  extern __shared__ __align__(16) float sm[];
  const double s2 = MODE == 0 ? L.tsc->s2 : 0.0;
  float* colx = sm;                 // [d][32]
  float* rowx = sm + L.d * 32;      // [d][LE_RB]
  __shared__ int rowp[LE_RB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const unsigned total = min(*L.count, L.cap);
  const unsigned items = L.item_start[L.nch - 1] + L.run_nb[L.nch - 1];
  for (unsigned item = blockIdx.x; item < items; item += gridDim.x) {
    const int4 td = __ldg(L.items + item);  // (chunk, first entry, rows)
    const int ch = td.x;
    const unsigned b0 = (unsigned)td.y;
    const int nb = td.z;
    __syncthreads();  // the previous item's readers of colx / rowx / rowp are done
    const int q0 = ch * 32;
    if ((L.d & 3) == 0) {  // 16-byte loads along k, lane = column (conflict-free transposed stores)
      for (int e = threadIdx.x; e < (L.d >> 2) * 32; e += blockDim.x) {
        const int t = e & 31, k4 = e >> 5;
        const int q = q0 + t;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < L.n) v = __ldg(reinterpret_cast<const float4*>(L.X + (int64_t)(L.perm ? L.perm[q] : q) * L.d) + k4);
        colx[(4 * k4 + 0) * 32 + t] = v.x;
        colx[(4 * k4 + 1) * 32 + t] = v.y;
        colx[(4 * k4 + 2) * 32 + t] = v.z;
        colx[(4 * k4 + 3) * 32 + t] = v.w;
      }
    } else {
      for (int e = threadIdx.x; e < L.d * 32; e += blockDim.x) {
        const int k = e >> 5, t = e & 31;
        const int q = q0 + t;
        colx[e] = q < L.n ? L.X[(int64_t)(L.perm ? L.perm[q] : q) * L.d + k] : 0.0f;
      }
    }
    int oq[4], Dq[4];
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int q = q0 + 4 * tx + b;
      oq[b] = q < L.n ? (L.perm ? L.perm[q] : q) : -1;
      Dq[b] = (MODE == 1 && q < L.n) ? L.sc[q] : -1;
    }
    {
      // stage the batch's rows transposed: lane = row of a 32-row group, float4 loads; the 8
      // warps split the 4 row groups x 2 halves of k; each reads its row's list entry itself
      // (no barrier between the list read and the row loads)
      for (int g = warp; g < 2 * (LE_RB / 32); g += blockDim.x >> 5) {
        const int r = (g >> 1) * 32 + lane;
        const int p = r < nb ? (int)(__ldg(L.list + b0 + r) & LIST_ROWMASK) : -1;
        if ((g & 1) == 0) rowp[r] = p;
        const int op = p < 0 ? 0 : (L.perm ? L.perm[p] : p);
        if ((L.d & 3) == 0) {
          const float4* src = reinterpret_cast<const float4*>(L.X + (int64_t)op * L.d);
          const int kh = (L.d / 4 + 1) / 2;  // float4s in the first half of k
          const int k4a = (g & 1) ? kh : 0, k4b = (g & 1) ? L.d / 4 : kh;
          for (int k4 = k4a; k4 < k4b; k4++) {
            const float4 v = p >= 0 ? __ldg(src + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
            rowx[(4 * k4 + 0) * LE_RB + r] = v.x;
            rowx[(4 * k4 + 1) * LE_RB + r] = v.y;
            rowx[(4 * k4 + 2) * LE_RB + r] = v.z;
            rowx[(4 * k4 + 3) * LE_RB + r] = v.w;
          }
        } else if ((g & 1) == 0) {
          for (int k = 0; k < L.d; k++) rowx[k * LE_RB + r] = p >= 0 ? __ldg(L.X + (int64_t)op * L.d + k) : 0.0f;
        }
      }
      __syncthreads();
      // warp w holds rows 16 w .. 16 w + 15: skip the padding of a chunk's ragged last batch
      if (16 * warp < nb) {
      // packed pairs (FADD2 / FFMA2): rows P0 = (a0, a1), P1 = (a2, a3); columns
      // Q0 = (b0, b1), Q1 = (b2, b3) and their swaps (b1, b0), (b3, b2) built in registers.
      // P - Q gives (a0 b0, a1 b1), P - Qs gives (a0 b1, a1 b0): 16 pairs in 8 + 8 packed
      // instructions per coordinate, each half the R1 step of its pair
      unsigned long long acc2[2][2][2];  // [row pair][column pair][swapped]
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) acc2[a][b][0] = acc2[a][b][1] = 0ull;
#pragma unroll 4
      for (int k = 0; k < L.d; k++) {
        const ulonglong2 xa = *reinterpret_cast<const ulonglong2*>(rowx + k * LE_RB + 4 * ty);
        const float4 xb = *reinterpret_cast<const float4*>(colx + k * 32 + 4 * tx);
        const unsigned long long q0 = f2pack(xb.x, xb.y), q1 = f2pack(xb.z, xb.w);
        const unsigned long long s0 = f2pack(xb.y, xb.x), s1 = f2pack(xb.w, xb.z);
        acc2[0][0][0] = f2_r1_step(xa.x, q0, acc2[0][0][0]);
        acc2[0][0][1] = f2_r1_step(xa.x, s0, acc2[0][0][1]);
        acc2[0][1][0] = f2_r1_step(xa.x, q1, acc2[0][1][0]);
        acc2[0][1][1] = f2_r1_step(xa.x, s1, acc2[0][1][1]);
        acc2[1][0][0] = f2_r1_step(xa.y, q0, acc2[1][0][0]);
        acc2[1][0][1] = f2_r1_step(xa.y, s0, acc2[1][0][1]);
        acc2[1][1][0] = f2_r1_step(xa.y, q1, acc2[1][1][0]);
        acc2[1][1][1] = f2_r1_step(xa.y, s1, acc2[1][1][1]);
      }
      float acc[4][4];
#pragma unroll
      for (int pa = 0; pa < 2; pa++)
#pragma unroll
        for (int pb = 0; pb < 2; pb++) {
          f2unpack(acc2[pa][pb][0], acc[2 * pa][2 * pb], acc[2 * pa + 1][2 * pb + 1]);
          f2unpack(acc2[pa][pb][1], acc[2 * pa][2 * pb + 1], acc[2 * pa + 1][2 * pb]);
        }
      // R1 ends with sqrtf; the MST runs on d^2 (monotone, App. A.4)
      if (MODE == 0) {
        // s2 = scale^2 is a power of two, so s^2 r <= UBK  <=>  r <= UBK / s2 exactly: one
        // fp32 compare per entry against lim = rd(UBK / s2); the few passing entries append
        unsigned pass = 0;
        int op4[4];
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const int p = rowp[4 * ty + a];
          op4[a] = p < 0 ? -1 : (L.perm ? L.perm[p] : p);
          const float lim = p < 0 ? -INFINITY : __double2float_rd((double)L.UBK[p] / s2);
#pragma unroll
          for (int b = 0; b < 4; b++)
            if (acc[a][b] <= lim && oq[b] >= 0 && oq[b] != op4[a]) pass |= 1u << (4 * a + b);
        }
        if (pass) {
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++)
              if ((pass >> (4 * a + b)) & 1u) {
                const int p = rowp[4 * ty + a];
                const unsigned slot = atomicAdd(L.cnt + p, 1u);
                if (slot < (unsigned)L.ccap)
                  L.cand[(int64_t)p * L.ccap + slot] =
                      ((u64)(__float_as_uint(acc[a][b]) & 0x7FFFFFFFu) << 33) | tri_index(op4[a], oq[b]);
              }
        }
      } else {
        // component pair of each entry; the common case (one row component, one column
        // component per thread and per warp) is reduced before a single atomicMin
        int Ca[4], opa[4];
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const int p = rowp[4 * ty + a];
          Ca[a] = p >= 0 ? L.sc[p] : -1;
          opa[a] = p >= 0 ? (L.perm ? L.perm[p] : p) : -1;
        }
        u64 key[4][4];
        int cC = -2, cD = -2;
        bool uni = true;
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++) {
            const bool el = Ca[a] >= 0 && Dq[b] >= 0 && Dq[b] != Ca[a];
            key[a][b] = el ? (((u64)(__float_as_uint(acc[a][b]) & 0x7FFFFFFFu) << 33) | tri_index(opa[a], oq[b]))
                           : KEY_NONE;
            if (el) {
              if (cC == -2) { cC = Ca[a]; cD = Dq[b]; }
              else if (cC != Ca[a] || cD != Dq[b]) uni = false;
            }
          }
        u64 m = KEY_NONE;
        if (uni) {
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) m = key[a][b] < m ? key[a][b] : m;
        }
        // warp: every lane uniform on one common pair (or without entries) -> one atomic
        const bool has_pair = uni && cC >= 0;
        const unsigned hb = __ballot_sync(0xffffffffu, has_pair);
        const int src = hb ? __ffs(hb) - 1 : 0;
        const int wC = __shfl_sync(0xffffffffu, cC, src), wD = __shfl_sync(0xffffffffu, cD, src);
        const bool ok = uni && (cC < 0 || (cC == wC && cD == wD));
        if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            const u64 other = __shfl_xor_sync(0xffffffffu, m, o);
            m = other < m ? other : m;
          }
          if (lane == 0 && hb && m != KEY_NONE) atomic_min_lt(L.WCM + (int64_t)wC * L.k + wD, m);
        } else if (has_pair) {
          if (m != KEY_NONE) atomic_min_lt(L.WCM + (int64_t)cC * L.k + cD, m);
        } else if (!uni) {
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++)
              if (key[a][b] != KEY_NONE) atomic_min_lt(L.WCM + (int64_t)Ca[a] * L.k + Dq[b], key[a][b]);
        }
      }
      }  // 16 * warp < nb
      __syncthreads();
    }
  }
}

// decode the column j of pair index t given the row i
__device__ __forceinline__ int other_end(u64 t, int i) {
  const int64_t base = (int64_t)i * (i - 1) / 2;
  if ((int64_t)t >= base && (int64_t)t < base + i) return (int)((int64_t)t - base);  // j < i
  // j > i: t = j (j - 1) / 2 + i
  const u64 r = t - (u64)i;
  int64_t j = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)r)) * 0.5);
  while (j * (j - 1) / 2 > (int64_t)r) j--;
  while ((j + 1) * j / 2 <= (int64_t)r) j++;
  return (int)j;
}

// warp per row: the K smallest appended keys -> cache; round 0's row minimum ->
// compbest[row] (singletons); overflowing rows -> invalid + exact fallback list
__global__ void k_topk_select(int p_begin, int p_end, int n, int K, const unsigned* __restrict__ cnt,
                              const u64* __restrict__ cand, int cap, u64* __restrict__ ckey,
                              int* __restrict__ cj, int* __restrict__ ccnt, u64* __restrict__ compbest,
                              int* __restrict__ fallback, unsigned* __restrict__ nfallback) {
  const int warps = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rows in pairs: two rows with at most 16 candidates each are sorted together, one per
  // half warp (a 16-wide bitonic network); otherwise each row takes the whole warp
  for (int p0 = p_begin + 2 * (blockIdx.x * warps + w); p0 < p_end; p0 += 2 * gridDim.x * warps) {
    const unsigned ca = cnt[p0], cb = p0 + 1 < p_end ? cnt[p0 + 1] : 0u;
    if (ca >= 1 && ca <= 16 && cb <= 16 && ca <= (unsigned)cap && cb <= (unsigned)cap) {
      const int half = lane >> 4, hl = lane & 15;
      const int p = p0 + half;
      const unsigned c = half ? cb : ca;
      const bool live = p < p_end && c >= 1;
      u64 x = (live && hl < (int)c) ? cand[(int64_t)p * cap + hl] : KEY_NONE;
#pragma unroll
      for (int size = 2; size <= 16; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          const u64 y = __shfl_xor_sync(0xffffffffu, x, stride);
          const bool up = (hl & size) == 0;
          const bool lower = (hl & stride) == 0;
          const u64 lo = x < y ? x : y, hi = x < y ? y : x;
          x = (lower == up) ? lo : hi;
        }
      const int take = min((int)c, K);
      if (p < p_end && c == 0 && hl == 0) {  // the second row without candidates
        ccnt[p] = -1;
        fallback[atomicAdd(nfallback, 1u)] = p;
      }
      if (live && hl < take) {
        ckey[(int64_t)p * K + hl] = x;
        cj[(int64_t)p * K + hl] = other_end(x & ((1ull << 33) - 1), p);
        if (hl == 0) compbest[p] = x;
      }
      if (live && hl == 0) ccnt[p] = take;
      continue;
    }
    for (int p = p0; p < min(p0 + 2, p_end); p++) {
    const unsigned c = cnt[p];
    if (c > (unsigned)cap || c == 0) {
      if (lane == 0) {
        ccnt[p] = -1;
        fallback[atomicAdd(nfallback, 1u)] = p;
      }
      continue;
    }
    const int take = min((int)c, K);
    if (cap <= 32) {
      // one key per lane: bitonic sort across the warp, lanes 0 .. take-1 hold the answer
      u64 x = lane < (int)c ? cand[(int64_t)p * cap + lane] : KEY_NONE;
#pragma unroll
      for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          const u64 y = __shfl_xor_sync(0xffffffffu, x, stride);
          const bool up = (lane & size) == 0;  // ascending block
          const bool lower = (lane & stride) == 0;
          const u64 lo = x < y ? x : y, hi = x < y ? y : x;
          x = (lower == up) ? lo : hi;
        }
      if (lane < take) {
        ckey[(int64_t)p * K + lane] = x;
        cj[(int64_t)p * K + lane] = other_end(x & ((1ull << 33) - 1), p);
        if (lane == 0) compbest[p] = x;
      }
      if (lane == 0) ccnt[p] = take;
      continue;
    }
    u64 mine[4];  // cap <= 128
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int e = lane + 32 * u;
      mine[u] = e < (int)c ? cand[(int64_t)p * cap + e] : KEY_NONE;
    }
    for (int t = 0; t < take; t++) {
      u64 lm = mine[0];
#pragma unroll
      for (int u = 1; u < 4; u++) lm = mine[u] < lm ? mine[u] : lm;
      u64 wm = lm;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, wm, o);
        wm = other < wm ? other : wm;
      }
      // keys are unique: exactly one lane owns wm
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (mine[u] == wm) mine[u] = KEY_NONE;
      if (lane == 0) {
        ckey[(int64_t)p * K + t] = wm;
        cj[(int64_t)p * K + t] = other_end(wm & ((1ull << 33) - 1), p);
        if (t == 0) compbest[p] = wm;
      }
    }
    // a row whose list holds every other point (n - 1 <= K) is complete
    if (lane == 0) ccnt[p] = take;
    }
  }
}

// rounds >= 1: first eligible cached entry -> component minimum; rows without one
// are flagged (need = 1)
__global__ void k_cache_lookup(int r0, int r1, int K, int n, const u64* __restrict__ ckey, const int* __restrict__ cj,
                               const int* __restrict__ ccnt, const int* __restrict__ comp,
                               u64* __restrict__ compbest, int* __restrict__ need) {
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    const int c = ccnt[i];
    const int ci = comp[i];
    int flag = 1;
    if (c > 0) {
      for (int t = 0; t < c; t++) {
        const int j = cj[(int64_t)i * K + t];
        if (comp[j] != ci) {
          atomic_min_lt(compbest + ci, ckey[(int64_t)i * K + t]);
          flag = 0;
          break;
        }
      }
      // every other point cached and none eligible: the row has no eligible edge
      if (flag && c == n - 1) flag = 0;
    }
    need[i] = flag;
  }
}

// flagged rows whose K-th cached key is below the component's best need a re-scan
__global__ void k_rescan_select(int r0, int r1, int K, const u64* __restrict__ ckey, const int* __restrict__ ccnt,
                                const int* __restrict__ comp, const u64* __restrict__ compbest,
                                int* __restrict__ need, unsigned* __restrict__ count, int* __restrict__ list) {
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    if (!need[i]) continue;
    const int c = ccnt[i];
    if (c > 0 && ckey[(int64_t)i * K + (c - 1)] >= compbest[comp[i]]) {
      need[i] = 0;
      continue;
    }
    list[atomicAdd(count, 1u)] = i;
  }
}

// permuted-order row mask and the list of 512-row blocks holding flagged rows
__global__ void k_rescan_blocks(int n, const int* __restrict__ perm, const int* __restrict__ need,
                                int* __restrict__ needp, int* __restrict__ blockflag) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int f = need[perm[p]];
    needp[p] = f;
    if (f) blockflag[p / TC_ROWS] = 1;
  }
}
__global__ void k_compact_blocks(int nblocks, const int* __restrict__ blockflag, int* __restrict__ list,
                                 int* __restrict__ count) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x)
    if (blockflag[b]) list[atomicAdd(count, 1)] = b;
}

// compUB[comp] = min over flagged rows of UB (scaled units), seeded by the cached
// component minima s^2 d^2(compbest) (rounded up)
__global__ void k_comp_ub_seed(int k, const u64* __restrict__ compbest, const TcScale* __restrict__ sc,
                               unsigned* __restrict__ compUB) {
  const double s2 = sc->s2;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    const u64 key = compbest[c];
    float v = INFINITY;
    if (key != KEY_NONE) {
      const float d2 = __uint_as_float((unsigned)(key >> 33));
      const double sv = (double)d2 * s2;
      v = sv < 3.0e38 ? __double2float_ru(sv) : INFINITY;
    }
    compUB[c] = __float_as_uint(v);
  }
}
__global__ void k_comp_ub(int n, const int* __restrict__ perm, const int* __restrict__ needp,
                          const unsigned* __restrict__ UB, const int* __restrict__ comp,
                          unsigned* __restrict__ compUB) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    if (needp[p]) atomicMin(compUB + comp[perm[p]], UB[p]);
}

// ---------------------------------------------------------------------------
// Exact minimum eligible edge of a list of rows (original indices): small re-scans
// and rows whose cache overflowed.  Work item = 16 listed rows x 256 columns; each
// thread holds one column, every column value loaded once serves the 16 rows (rows in
// shared memory, staged when the row group changes); the next 8 coordinates' column
// values are loaded while the current ones are used.  A CTA takes a contiguous range
// of items (row group major) and keeps each row's best key per thread, reduced over
// the CTA only when the row group changes.  XT: d x ldx original-order transpose (zero
// padded to ldx).  comp == nullptr: singletons (eligible = j != i).
// ---------------------------------------------------------------------------
constexpr int RE_R = 16, RE_COLS = 256;
template <bool FULL>  // FULL: d % 64 == 0 (no coordinate guards in the inner loop)
__global__ void __launch_bounds__(256, 2) k_rows_exact(const float* __restrict__ XT, int64_t ldx, int n, int d,
                                                      const int* __restrict__ rows, const unsigned* __restrict__ nrows,
                                                      const int* __restrict__ comp, u64* __restrict__ compbest,
                                                      int max_rows) {
  extern __shared__ float xr[];  // [d][RE_R]
  __shared__ u64 red[8][RE_R];
  __shared__ int sri[RE_R], sci[RE_R];
  const int nr = (int)*nrows;
  if (nr > max_rows) return;  // (a speculative launch whose rows need the tensor-core pass)
  const int ngroups = (nr + RE_R - 1) / RE_R;
  const int nblk = (n + RE_COLS - 1) / RE_COLS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int KB = 64;
  const int64_t total = (int64_t)ngroups * nblk;
  const int i0 = (int)(total * blockIdx.x / gridDim.x), i1 = (int)(total * (blockIdx.x + 1) / gridDim.x);
  u64 best[RE_R];
  int g_cur = -1;
  // reduce the per-thread minima of row group g_cur over the CTA, one atomic per row
  auto flush = [&]() {
#pragma unroll
    for (int r = 0; r < RE_R; r++) {
      u64 b = best[r];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, b, o);
        b = other < b ? other : b;
      }
      if (lane == 0) red[warp][r] = b;
    }
    __syncthreads();
    if (threadIdx.x < RE_R && sri[threadIdx.x] >= 0) {
      u64 b = KEY_NONE;
      for (int w = 0; w < 8; w++) b = red[w][threadIdx.x] < b ? red[w][threadIdx.x] : b;
      if (b != KEY_NONE) atomic_min_lt(compbest + sci[threadIdx.x], b);
    }
  };
  for (int item = i0; item < i1; item++) {
    const int g = item / nblk, blk = item % nblk;
    if (g != g_cur) {
      if (g_cur >= 0) flush();
      __syncthreads();  // readers of xr / sri / red are done
      if (threadIdx.x < RE_R) {
        const int idx = g * RE_R + threadIdx.x;
        const int ri = idx < nr ? rows[idx] : -1;
        sri[threadIdx.x] = ri;
        sci[threadIdx.x] = ri >= 0 ? (comp ? comp[ri] : ri) : -1;
      }
      for (int e = threadIdx.x; e < d * RE_R; e += blockDim.x) {
        const int k = e / RE_R, r = e % RE_R;
        const int idx = g * RE_R + r;
        const int ri = idx < nr ? rows[idx] : -1;
        xr[e] = ri >= 0 ? XT[(int64_t)k * ldx + ri] : 0.0f;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < RE_R; r++) best[r] = KEY_NONE;
      g_cur = g;
    }
    unsigned long long acc2[RE_R / 2];  // rows (2 i, 2 i + 1) packed
#pragma unroll
    for (int r = 0; r < RE_R / 2; r++) acc2[r] = 0ull;
    const int j = blk * RE_COLS + threadIdx.x;
    // XT is zero padded beyond n up to ldx (a multiple of 128 >= the column blocks' end):
    // no column guard for the loads, only for the keys
    const float* xcol = XT + j;
    // the R1 chain in order k = 0, 1, ...: all KB = 64 coordinates of the column loaded at
    // once (one L2 latency per item and 64-coordinate chunk instead of one per 8)
    for (int k0 = 0; k0 < d; k0 += KB) {
      float y[KB];
      const float* src = xcol + (int64_t)k0 * ldx;
#pragma unroll
      for (int kk = 0; kk < KB; kk++) y[kk] = (FULL || k0 + kk < d) ? __ldg(src + (int64_t)kk * ldx) : 0.0f;
#pragma unroll
      for (int kk = 0; kk < KB; kk++) {
        if (!FULL && k0 + kk >= d) break;
        const unsigned long long yy = f2pack(y[kk], y[kk]);
#pragma unroll
        for (int q = 0; q < RE_R / 4; q++) {
          const ulonglong2 x4 = *reinterpret_cast<const ulonglong2*>(xr + (k0 + kk) * RE_R + 4 * q);
          acc2[2 * q] = f2_r1_step(x4.x, yy, acc2[2 * q]);
          acc2[2 * q + 1] = f2_r1_step(x4.y, yy, acc2[2 * q + 1]);
        }
      }
    }
    float acc[RE_R];
#pragma unroll
    for (int r = 0; r < RE_R / 2; r++) f2unpack(acc2[r], acc[2 * r], acc[2 * r + 1]);
    if (j < n) {
      const int cj = comp ? __ldg(comp + j) : j;
#pragma unroll
      for (int r = 0; r < RE_R; r++) {
        const int ri = sri[r];
        if (ri >= 0 && cj != sci[r]) {
          const u64 key = ((u64)(__float_as_uint(acc[r]) & 0x7FFFFFFFu) << 33) | tri_index(ri, j);
          best[r] = key < best[r] ? key : best[r];
        }
      }
    }
  }
  if (g_cur >= 0) flush();
}

appd_status launch_rows_exact(appd_ctx* c, const float* XT, int64_t ldx, int n, int d, const int* rows,
                              const unsigned* nrows, int max_rows, const int* comp, u64* compbest) {
  if (max_rows <= 0) return APPD_OK;
  const int64_t items = (int64_t)((max_rows + RE_R - 1) / RE_R) * ((n + RE_COLS - 1) / RE_COLS);
  const int grid = (int)std::min<int64_t>(items, (int64_t)c->sm_count * 2);  // persistent: 2 CTAs per SM
  const size_t smem = (size_t)d * RE_R * 4;
  if (d % 64 == 0) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_rows_exact<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_rows_exact<true><<<grid, 256, smem, c->stream>>>(XT, ldx, n, d, rows, nrows, comp, compbest, max_rows);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_rows_exact<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_rows_exact<false><<<grid, 256, smem, c->stream>>>(XT, ldx, n, d, rows, nrows, comp, compbest, max_rows);
  }
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
appd_status launch_list_exact(appd_ctx* c, int mode, const ListParams& L, unsigned* run_lo, unsigned* run_nb,
                              unsigned* item_start) {
  const size_t smem = (size_t)L.d * (32 + LE_RB) * 4;
  if (smem > 200 * 1024) return APPD_ERR_UNSUPPORTED;
  if (run_lo) {  // sorted list: runs and items from binary searches (else prepared by the caller)
    k_chunk_runs<<<(L.nch + 255) / 256, 256, 0, c->stream>>>(L.list, L.count, L.cap, L.nch, run_lo, run_nb);
    APPD_LAUNCHED(c);
    appd_status s = exclusive_scan_i32(c, (const int*)run_nb, (int*)item_start, L.nch);
    if (s) return s;
    k_item_table<<<(L.nch + 255) / 256, 256, 0, c->stream>>>(run_lo, run_nb, item_start, L.list, L.count, L.cap,
                                                            L.nch, const_cast<int4*>(L.items));
    APPD_LAUNCHED(c);
  }
  const int grid = c->sm_count * (mode == 0 ? 5 : 4);  // 5 x 40 KB of shared memory fit an SM
  // set once per device at the largest size any d needs (attribute calls cost host time)
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
    cudaFuncSetAttribute(k_list_exact<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_list_exact<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    setup_done(attr, c);
  }
  if (mode == 0) k_list_exact<0><<<grid, 256, smem, c->stream>>>(L);
  else k_list_exact<1><<<grid, 256, smem, c->stream>>>(L);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_topk_select(appd_ctx* c, int p_begin, int p_end, int n, int K, const unsigned* cnt,
                               const u64* cand, int cap, u64* ckey, int* cj, int* ccnt, u64* compbest, int* fallback,
                               unsigned* nfallback) {
  const int rows = p_end - p_begin;
  if (rows <= 0) return APPD_OK;
  const int grid = std::min(c->sm_count * 8, (rows + 7) / 8);
  k_topk_select<<<grid, 256, 0, c->stream>>>(p_begin, p_end, n, K, cnt, cand, cap, ckey, cj, ccnt, compbest,
                                             fallback, nfallback);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_cache_lookup(appd_ctx* c, int r0, int r1, int K, int n, const u64* ckey, const int* cj,
                                const int* ccnt, const int* comp, u64* compbest, int* need, unsigned* count,
                                int* list) {
  const int rows = r1 - r0;
  if (rows <= 0) return APPD_OK;
  const int grid = std::min(c->sm_count * 8, (rows + 255) / 256);
  k_cache_lookup<<<grid, 256, 0, c->stream>>>(r0, r1, K, n, ckey, cj, ccnt, comp, compbest, need);
  APPD_LAUNCHED(c);
  k_rescan_select<<<grid, 256, 0, c->stream>>>(r0, r1, K, ckey, ccnt, comp, compbest, need, count, list);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_rescan_blocks(appd_ctx* c, int n, const int* perm, const int* need, int* needp, int* blockflag,
                                 int nblocks, int* list, int* count) {
  const int grid = std::min(c->sm_count * 8, (n + 255) / 256);
  k_rescan_blocks<<<grid, 256, 0, c->stream>>>(n, perm, need, needp, blockflag);
  APPD_LAUNCHED(c);
  k_compact_blocks<<<(nblocks + 255) / 256, 256, 0, c->stream>>>(nblocks, blockflag, list, count);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_comp_ub(appd_ctx* c, int n, int k, const u64* compbest, const TcScale* s2, const int* perm,
                           const int* needp, const unsigned* UB, const int* comp, unsigned* compUB) {
  k_comp_ub_seed<<<(k + 255) / 256, 256, 0, c->stream>>>(k, compbest, s2, compUB);
  APPD_LAUNCHED(c);
  const int grid = std::min(c->sm_count * 8, (n + 255) / 256);
  k_comp_ub<<<grid, 256, 0, c->stream>>>(n, perm, needp, UB, comp, compUB);
  APPD_LAUNCHED(c);
  return APPD_OK;
}


// ===========================================================================
// Component-matrix finish (SURVEY App. B reading: "Once k_r <= ~128, one pass
// computes every row's min to every component; the contracted k x k graph then
// finishes the MST").  Points are sorted by component (labels 0..k-1, contiguous
// column ranges [cstart, cend)), and one tensor-core pass has written TM[seg][p],
// the eligible maximum of G' over each TC_TMG-column segment.
//   k_cm_rowub   CUB[C][D] = min over rows p of C of the upper bound of s^2 r from the
//                segments lying entirely inside D (an exact pair exists below it);
//   k_cm_filter  lists (p, seg) whenever a pair (p, j), j in seg and in D != C, can
//                have L <= CUB[C][D];
//   k_cm_exact   exact R1 keys of the listed segments, minimum per (C, D) by atomicMin.
// Every pair of C x D with L <= CUB[C][D] is evaluated exactly, so WCM[C][D] is the
// exact minimum key between C and D; the MST of the contracted graph (host Prim on
// k <= 128 nodes) plus the edges of the earlier rounds is the MST.
// ===========================================================================

// per 128-column segment: (first, last) component label of its real columns
__global__ void k_seg_comp(const int* __restrict__ sc, int n, int nseg, int2* __restrict__ segd) {
  for (int sg = blockIdx.x * blockDim.x + threadIdx.x; sg < nseg; sg += gridDim.x * blockDim.x) {
    const int q0 = sg * TC_TMG;
    segd[sg] = q0 < n ? make_int2(sc[q0], sc[min(q0 + TC_TMG - 1, n - 1)]) : make_int2(-1, -1);
  }
}

// segments are sorted by component: stream each row's stored maxima in order (16 loads
// in flight), keep the running maximum of the current component's full segments and
// flush its bound when the component changes
// U consecutive stored segments of one row (stride 512 floats, tm_index) from ptr; the
// first `left` of them are real, the rest -inf.  A full batch (warp-uniform) is U loads
// at immediate offsets; the lanes of invalid rows read a valid row and are masked later
template <int U>
__device__ __forceinline__ void load_segs(const float* __restrict__ ptr, int left, float (&v)[U]) {
  if (left >= U) {
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = __ldcs(ptr + u * 512);
  } else {
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = u < left ? __ldcs(ptr + u * 512) : -INFINITY;
  }
}
constexpr int CM_SPLIT = 4;  // warps per 32-row group, each over a quarter of the segments
__global__ void k_cm_rowub(CmParams P) {
  const int lane = threadIdx.x & 31;
  const float maxlen_ = P.tsc->maxlen;
  const int nseg_n = P.n / TC_TMG;  // full segments only (a partial last segment bounds nothing)
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // global warp
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int groups = (P.p_end - P.p_begin + 31) / 32;
  for (int64_t task = gw; task < (int64_t)groups * CM_SPLIT; task += nw) {
    const int p0 = P.p_begin + (int)(task / CM_SPLIT) * 32;
    const int part = (int)(task % CM_SPLIT);
    const int p = p0 + lane;
    const bool valid = p < P.p_end;
    // this row's stored maxima: segment s at tm_row[s * 512] (tm_index; one base per row,
    // immediate offsets per segment in the unrolled loads)
    const float* tm_row = P.TM + tm_index(0, min(p, P.p_end - 1), P.nseg);
    const int C = valid ? P.sc[p] : -1;
    const bool uni = __all_sync(0xffffffffu, C == __shfl_sync(0xffffffffu, C, 0));
    const float ni = valid ? P.nrm[p] : 0.0f, li = valid ? P.len[p] : 0.0f;
    const float dl = em_delta2(valid ? P.err[p] : 0.0f, *P.maxerr);
    const int smin = P.upper ? (TC_ROWS / TC_TMG) * (p0 / TC_ROWS) : 0;  // segments the scan wrote
    auto flush = [&](int D, float m) {
      float ub = (m > -INFINITY && D != C && valid) ? em_upper(P.em, ni - 2.0f * m, ni, li, maxlen_, dl) : INFINITY;
      if (uni) {  // D is warp-uniform (segment order is the same for every lane)
#pragma unroll
        for (int o = 16; o; o >>= 1) ub = fminf(ub, __shfl_xor_sync(0xffffffffu, ub, o));
        if (lane == 0 && C >= 0 && ub < INFINITY)
          atomic_min_lt(P.CUB + (int64_t)C * P.k + D, __float_as_uint(fmaxf(ub, 0.0f)));
      } else if (ub < INFINITY) {
        atomic_min_lt(P.CUB + (int64_t)C * P.k + D, __float_as_uint(fmaxf(ub, 0.0f)));
      }
    };
    constexpr int U = 16;
    const int span = (nseg_n - smin + CM_SPLIT - 1) / CM_SPLIT;
    const int sbeg = smin + part * span, send = min(nseg_n, sbeg + span);
    // runs of full segments of one component D (positions sorted by component: the full
    // segments of D are those below cend[D] / TC_TMG); straddling segments are skipped
    for (int s = sbeg; s < send;) {
      const int2 dd = P.segd[s];
      if (dd.x != dd.y) {
        s++;
        continue;
      }
      const int D = dd.x;
      const int e = max(s + 1, min(send, P.cend[D] / TC_TMG));
      float m = -INFINITY;
      for (int s0 = s; s0 < e; s0 += U) {
        float v[U];
        load_segs<U>(tm_row + (int64_t)s0 * 512, e - s0, v);
#pragma unroll
        for (int u = 0; u < U; u++) m = fmaxf(m, v[u]);
      }
      flush(D, m);
      s = e;
    }
  }
}

// one warp per 32 consecutive rows; 16 segments' loads in flight, one slot allocation
// per batch.  CUB here holds the listing thresholds T[C][D] (the host's path-pruned
// upper bounds, scaled units).  A listed segment contributes its 32-column chunks.
__global__ void k_cm_filter(CmParams P) {
  const int lane = threadIdx.x & 31;
  const float maxlen_ = P.tsc->maxlen;
  const int nseg = min(P.nseg, (P.n + TC_TMG - 1) / TC_TMG);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int groups = (P.p_end - P.p_begin + 31) / 32;
  for (int64_t task = gw; task < (int64_t)groups * CM_SPLIT; task += nw) {
    const int p0 = P.p_begin + (int)(task / CM_SPLIT) * 32;
    const int part = (int)(task % CM_SPLIT);
    const int p = p0 + lane;
    const bool valid = p < P.p_end;
    const float* tm_row = P.TM + tm_index(0, min(p, P.p_end - 1), P.nseg);
    const int C = valid ? P.sc[p] : 0;
    const float ni = valid ? P.nrm[p] : 0.0f, li = valid ? P.len[p] : 0.0f;
    const float dl = em_delta2(valid ? P.err[p] : 0.0f, *P.maxerr);
    constexpr int U = 16;
    const int smin = P.upper ? (TC_ROWS / TC_TMG) * (p0 / TC_ROWS) : 0;
    const int span = (nseg - smin + CM_SPLIT - 1) / CM_SPLIT;
    const int sbeg = smin + part * span, send = min(nseg, sbeg + span);
    // runs of segments with one threshold: the full segments of a component D (below
    // cend[D] / TC_TMG), or a single straddling segment (most permissive of its components)
    for (int s = sbeg; s < send;) {
      const int2 dd = P.segd[s];
      int e;
      float thr;
      if (dd.x == dd.y) {
        e = max(s + 1, min(send, P.cend[dd.x] / TC_TMG));
        thr = em_thr(P.em, __uint_as_float(P.CUB[(int64_t)C * P.k + dd.x]), ni, li, maxlen_, dl);
      } else {
        e = s + 1;
        float ub = 0.0f;
        for (int D = dd.x; D <= dd.y; D++)
          if (D != C) ub = fmaxf(ub, __uint_as_float(P.CUB[(int64_t)C * P.k + D]));
        thr = em_thr(P.em, ub, ni, li, maxlen_, dl);
      }
      const float thr_c = fmaxf(thr, -FLT_MAX);  // (-inf never passes: one compare per value)
      for (int s0 = s; s0 < e; s0 += U) {
        float v[U];
        load_segs<U>(tm_row + (int64_t)s0 * 512, e - s0, v);
        unsigned mask = 0;
#pragma unroll
        for (int u = 0; u < U; u++) mask |= v[u] >= thr_c ? 1u << u : 0u;
        if (!valid) mask = 0u;
        unsigned any = __reduce_or_sync(0xffffffffu, mask);
        // chunk-major emission: for each flagged segment and chunk, the warp's rows in
        // lane order (consecutive rows, mostly one component), so that the chunk runs of
        // the counting sort keep rows of one component together (k_list_exact<1>)
        while (any) {
          const int u = __ffs(any) - 1;
          any &= any - 1;
          const bool mine = (mask >> u) & 1u;
          const unsigned bal = __ballot_sync(0xffffffffu, mine);
          const int sg = s0 + u;
          const int nc = min(TC_TMG / 32, (P.n - sg * TC_TMG + 31) / 32);
          const unsigned cntw = (unsigned)__popc(bal);
          unsigned base = 0;
          if (lane == 0) base = atomicAdd(P.counters + 1, cntw * (unsigned)nc);
          base = __shfl_sync(0xffffffffu, base, 0);
          if (mine) {
            const unsigned rank = (unsigned)__popc(bal & ((1u << lane) - 1u));
            for (int t = 0; t < nc; t++) {
              const unsigned slot = base + (unsigned)t * cntw + rank;
              if (slot < P.list_cap) P.list[slot] = ((unsigned)((TC_TMG / 32) * sg + t) << LIST_SHIFT) | (unsigned)p;
            }
          }
        }
      }
      s = e;
    }
  }
}

// ---------------------------------------------------------------------------
// Contracted-graph steps of the component-matrix finish, one CTA (k <= 128 nodes, one
// thread per node).  Both are Prim's algorithm on a dense k x k matrix.
// ---------------------------------------------------------------------------
// Listing thresholds.  CUB[C][D] bounds w(C, D) from above (both directions bound the
// same w).  An MST edge (C, D) of the contracted graph satisfies w(C, D) <= the largest
// bound on the path from C to D in the MST of the bounds (cut property), so
// T = min(symmetric bound, path maximum) keeps every MST edge's minimum pair listed;
// pairs above T are not MST edges and may come out inflated.  Output T (k x k).
// warp argmin of (64-bit key, 32-bit index) pairs, smallest index among equal keys, with
// three redux.sync reductions (high word, low word among the winners, index among the
// winners) instead of a five-level shuffle tree of 64-bit pairs
__device__ __forceinline__ void warp_argmin_u64(u64& key, int& idx) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
  const bool win = hi == mhi && lo == mlo;
  const int mi = (int)__reduce_min_sync(0xffffffffu, win ? (unsigned)idx : 0xffffffffu);
  key = ((u64)mhi << 32) | mlo;
  idx = mi;
}

// (1024 threads: the k x k staging is a few loads per thread, all in flight)
__global__ void __launch_bounds__(1024) k_cm_thresholds(const unsigned* __restrict__ CUB, int k,
                                                        unsigned* __restrict__ T) {
  extern __shared__ float symb[];   // [k][k] symmetric bounds, then [k][k] path maxima
  float* pm = symb + k * k;
#pragma unroll 4
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {  // all threads stage (latency)
    const int a = e / k, b = e % k;
    symb[e] = fminf(__uint_as_float(CUB[(int64_t)a * k + b]), __uint_as_float(CUB[(int64_t)b * k + a]));
    pm[e] = 0.0f;
  }
  __syncthreads();
  // Prim from node 0 in one warp, lane l owning nodes l + 32 t (k <= 128); when node nq
  // joins through tree neighbour f with bound w, every node x already in the tree gets
  // pm[x][nq] = pm[nq][x] = max(pm[x][f], w): the path maxima of the bound MST
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool in[4];
    float key[4];
    int from[4];
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const int q = lane + 32 * t;
      in[t] = q == 0 || q >= k;
      key[t] = (q < k && q > 0) ? symb[q] : INFINITY;
      from[t] = 0;
    }
    for (int step = 1; step < k; step++) {
      // (orderable bound, node) argmin; bounds are >= 0 or +inf, so the float bits order
      u64 bv = KEY_NONE;
      int bi = 0x7fffffff;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const u64 kv = in[t] ? KEY_NONE : (((u64)__float_as_uint(key[t]) << 32) | (unsigned)(lane + 32 * t));
        if (kv < bv) { bv = kv; bi = lane + 32 * t; }
      }
      warp_argmin_u64(bv, bi);
      const int nq = bi;
      // the joining node's tree neighbour and bound, from its owner lane
      int fo = 0;
      float wo = 0.0f;
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (lane + 32 * t == nq) { fo = from[t]; wo = key[t]; in[t] = true; }
      const int f = __shfl_sync(0xffffffffu, fo, nq & 31);
      const float wq = __shfl_sync(0xffffffffu, wo, nq & 31);
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int q = lane + 32 * t;
        if (q >= k) continue;
        if (in[t] && q != nq) {  // in-tree nodes (before nq joined): path max to nq
          const float v = fmaxf(pm[q * k + f], wq);
          pm[q * k + nq] = v;
          pm[nq * k + q] = v;
        } else if (!in[t]) {
          const float wn = symb[nq * k + q];
          if (wn < key[t]) { key[t] = wn; from[t] = nq; }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int a = e / k, b = e % k;
    T[e] = __float_as_uint(a == b ? symb[e] : fminf(symb[e], pm[e]));
  }
}

// Final contracted MST: Prim on min(WCM[C][D], WCM[D][C]) (exact keys, a strict order),
// the k - 1 edge keys appended to mstkeys at counters[0]
// If the listing overflowed (*list_count > list_cap: minima may be missing) or the
// matrix is disconnected, the remaining k - 1 - added edges are placeholders of a star
// over component representatives (valid indices, largest key) so that every later
// kernel stays in bounds, and status records why (1 overflow, 2 disconnected): the host
// re-solves without the component matrix, or reports the inconsistency.
__global__ void __launch_bounds__(1024) k_cm_prim(const u64* __restrict__ WCM, int k, u64* __restrict__ mstkeys,
                                                  int* __restrict__ counters, const unsigned* __restrict__ list_count,
                                                  unsigned list_cap, const int* __restrict__ cstart,
                                                  const int* __restrict__ perm, unsigned* __restrict__ status) {
  extern __shared__ u64 wsym[];  // [k][k] symmetric minima
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {  // all threads stage (latency)
    const int a = e / k, b = e % k;
    const u64 x = WCM[(int64_t)a * k + b], y = WCM[(int64_t)b * k + a];
    wsym[e] = x < y ? x : y;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int base = counters[0];
  const bool overflow = *list_count > list_cap;
  u64 key[4];
  bool in[4];
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const int q = lane + 32 * t;
    in[t] = q == 0 || q >= k;
    key[t] = (q < k && q > 0) ? wsym[q] : KEY_NONE;
  }
  int added = 0;
  for (int step = 1; step < k; step++) {
    u64 bv = KEY_NONE;
    int bi = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < 4; t++)
      if (!in[t] && (key[t] < bv || (key[t] == bv && lane + 32 * t < bi))) { bv = key[t]; bi = lane + 32 * t; }
    warp_argmin_u64(bv, bi);
    if (bv == KEY_NONE || overflow) break;
    if (lane == 0) mstkeys[base + step - 1] = bv;
    added = step;
    if ((bi & 31) == lane) {
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (u == (bi >> 5)) in[u] = true;
    }
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const int q = lane + 32 * t;
      if (!in[t]) {
        const u64 x = wsym[bi * k + q];
        if (x < key[t]) key[t] = x;
      }
    }
  }
  if (added < k - 1) {  // placeholders: component 0 (in the tree) to every node not in it
    const int r0 = perm[cstart[0]];
    int off = base + added;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const int q = lane + 32 * t;
      const bool need = q < k && !in[t];
      const unsigned bal = __ballot_sync(0xffffffffu, need);
      if (need)
        mstkeys[off + __popc(bal & ((1u << lane) - 1u))] = (0x7F7FFFFFull << 33) | tri_index(r0, perm[cstart[q]]);
      off += __popc(bal);
    }
    if (lane == 0) *status = overflow ? 1u : 2u;
    added = k - 1;
  }
  if (lane == 0) counters[0] = base + added;
}

appd_status launch_cm_thresholds(appd_ctx* c, const unsigned* CUB, int k, unsigned* T) {
  const size_t smem = sizeof(float) * 2 * k * k;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_cm_thresholds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_cm_thresholds<<<1, 1024, smem, c->stream>>>(CUB, k, T);
  APPD_LAUNCHED(c);
  return APPD_OK;
}
appd_status launch_cm_prim(appd_ctx* c, const u64* WCM, int k, u64* mstkeys, int* counters,
                           const unsigned* list_count, unsigned list_cap, const int* cstart, const int* perm,
                           unsigned* status) {
  const size_t smem = sizeof(u64) * k * k;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_cm_prim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_cm_prim<<<1, 1024, smem, c->stream>>>(WCM, k, mstkeys, counters, list_count, list_cap, cstart, perm, status);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_seg_comp(appd_ctx* c, const int* sc, int n, int nseg, int2* segd) {
  k_seg_comp<<<(nseg + 255) / 256, 256, 0, c->stream>>>(sc, n, nseg, segd);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_cm_rowub(appd_ctx* c, const CmParams& P) {
  const int rows = P.p_end - P.p_begin;
  if (rows <= 0) return APPD_OK;
  k_cm_rowub<<<std::min(c->sm_count * 16, (rows * CM_SPLIT + 255) / 256), 256, 0, c->stream>>>(P);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_cm_filter(appd_ctx* c, const CmParams& P) {
  const int rows = P.p_end - P.p_begin;
  if (rows <= 0) return APPD_OK;
  k_cm_filter<<<std::min(c->sm_count * 16, (rows * CM_SPLIT + 255) / 256), 256, 0, c->stream>>>(P);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
