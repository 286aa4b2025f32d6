// k_boruvka.cu -- the MST stage: Boruvka rounds.
//
// P:L98 (§3) builds the MST with Prim; any MST gives the same APPD (P:L79,
// "the path between any two nodes in a minimum spanning tree (MST) is a minimax
// path", and DESIGN.md reading Q2), so the GPU uses Boruvka: each round every
// row finds its lightest edge leaving its component (a row-parallel, coalesced
// component-filtered argmin), components take the minimum over their rows, and
// the chosen edges merge components.  At most ceil(log2 n) rounds.
#include <cub/device/device_scan.cuh>

#include <cooperative_groups.h>

#include "internal.cuh"

namespace appd {
namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// weights mode: one CTA per row (grid-stride), float4 loads of W's row, the
// component labels of the columns come from L2 (n x 4 B, resident).
// Per thread: best (w, j) with strict "<" so the smallest j wins ties (columns
// are visited in increasing order per thread); then a (key) min over the CTA.
// ---------------------------------------------------------------------------
template <bool ROUND0, int SENSE>
__global__ void __launch_bounds__(256) k_scan_weights(const float* __restrict__ W, int64_t n, int64_t row0,
                                                      int64_t rows, const int* __restrict__ comp,
                                                      u64* __restrict__ compbest) {
  __shared__ u64 red[8];
  const bool vec = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t i = row0 + r;
    const float* Wr = W + r * n;
    const int ci = ROUND0 ? (int)i : comp[i];
    float bw = SENSE > 0 ? INFINITY : -INFINITY;
    int64_t bj = -1;
    if (vec) {
      const float4* W4 = reinterpret_cast<const float4*>(Wr);
      const int4* C4 = reinterpret_cast<const int4*>(comp);
      const int64_t n4 = n >> 2;
#pragma unroll 4
      for (int64_t q = threadIdx.x; q < n4; q += 256) {
        float4 w = __ldcs(W4 + q);  // streamed once per round: evict-first
        int4 cc;
        if (!ROUND0) cc = __ldg(C4 + q);
        const int64_t j = q * 4;
        float ws[4] = {w.x, w.y, w.z, w.w};
        int cs[4];
        if (!ROUND0) { cs[0] = cc.x; cs[1] = cc.y; cs[2] = cc.z; cs[3] = cc.w; }
#pragma unroll
        for (int t = 0; t < 4; t++) {
          bool elig = ROUND0 ? (j + t != i) : (cs[t] != ci);
          bool better = SENSE > 0 ? (ws[t] < bw) : (ws[t] > bw);
          if (elig && better) { bw = ws[t]; bj = j + t; }
        }
      }
    } else {
      for (int64_t j = threadIdx.x; j < n; j += 256) {
        float w = __ldcs(Wr + j);
        bool elig = ROUND0 ? (j != i) : (__ldg(comp + j) != ci);
        bool better = SENSE > 0 ? (w < bw) : (w > bw);
        if (elig && better) { bw = w; bj = j; }
      }
    }
    // row key (weight, j): weight mapped to the orderable u32 of the minimised quantity
    u64 key = KEY_NONE;
    if (bj >= 0) {
      float m = SENSE > 0 ? bw : -bw;
      m = m + 0.0f;  // -0 -> +0 (reading Q5)
      key = ((u64)orderable(m) << 32) | (u64)bj;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      u64 other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other < key ? other : key;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 k = red[0];
#pragma unroll
      for (int t = 1; t < 8; t++) k = red[t] < k ? red[t] : k;
      if (k != KEY_NONE) {
        int64_t j = (int64_t)(k & 0xFFFFFFFFull);
        u64 gkey = (k & 0xFFFFFFFF00000000ull) | tri_index(i, j);
        atomic_min_lt(compbest + ci, gkey);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// weights mode, round 0 with the candidate cache: per row the K smallest (w, j), j != i,
// exactly (the per-row order (w, j) is the global edge-key order, see above).  Each
// thread keeps a sorted local top-K of its columns (insertion only when a column beats
// its K-th), then each warp and finally warp 0 extract the CTA's K smallest.  Writes the
// cache (ckey = global keys, cj = column) and compbest[i] (singletons).
// ---------------------------------------------------------------------------
template <int K, int SENSE>
__global__ void __launch_bounds__(256) k_scan_weights_topk(const float* __restrict__ W, int64_t n, int64_t row0,
                                                         int64_t rows, u64* __restrict__ ckey, int* __restrict__ cj,
                                                         int* __restrict__ ccnt, u64* __restrict__ compbest) {
  // pass 1: per-thread minimum (columns visited in increasing j: strict '<' keeps the
  // smallest j); the K-th smallest of the 256 minima bounds the row's K-th key (they are
  // K distinct columns).  pass 2 (the row again, from L2): every key <= that bound is
  // collected; a warp sorts them (bitonic, 64 at a time) and keeps the K smallest.
  constexpr int CAP = 64;
  __shared__ u64 tmin[256];
  __shared__ u64 cand[CAP];
  __shared__ u64 tau_s;
  __shared__ int ncand;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t i = row0 + r;
    const float* Wr = W + r * n;
    auto keyof = [&](float w, int j) -> u64 {
      float m = SENSE > 0 ? w : -w;
      m = m + 0.0f;  // -0 -> +0 (reading Q5)
      return ((u64)orderable(m) << 32) | (u64)(unsigned)j;
    };
    // one float compare per element (validated input: no NaN; -0 == +0 as in the key);
    // strict '<' (widest: '>') in increasing j keeps the smallest j among equal weights,
    // so (w, j) is the thread's minimum key
    auto better = [&](float a, float b) -> bool { return SENSE > 0 ? a < b : a > b; };
    const float NOPE = SENSE > 0 ? INFINITY : -INFINITY;  // the diagonal entry never competes
    float bw = NOPE;
    int bj = -1;
    // 32-bit indices (weights mode: n <= 92682); the diagonal is not tested per element:
    // the thread whose minimum lands on it (always, for non-negative weights) re-scans its
    // own quads without it.  The full batches run without predicates.  (The scan was
    // instruction-bound at 58 % issue with 64-bit j and a per-element j != i test.)
    const int i32 = (int)i;
    auto scan4 = [&](float4 v, int j, bool skip_diag) {
      if (better(v.x, bw) && (!skip_diag || j != i32)) { bw = v.x; bj = j; }
      if (better(v.y, bw) && (!skip_diag || j + 1 != i32)) { bw = v.y; bj = j + 1; }
      if (better(v.z, bw) && (!skip_diag || j + 2 != i32)) { bw = v.z; bj = j + 2; }
      if (better(v.w, bw) && (!skip_diag || j + 3 != i32)) { bw = v.w; bj = j + 3; }
    };
    if (vec) {
      const float4* W4 = reinterpret_cast<const float4*>(Wr);
      const int n4 = (int)(n >> 2);
      int q0 = threadIdx.x;
      for (; q0 + 7 * 256 < n4; q0 += 8 * 256) {  // eight 16-byte loads in flight, then in order of j
        float4 w[8];
#pragma unroll
        for (int u = 0; u < 8; u++) w[u] = __ldcg(W4 + q0 + u * 256);
#pragma unroll
        for (int u = 0; u < 8; u++) scan4(w[u], 4 * (q0 + u * 256), false);
      }
      for (; q0 < n4; q0 += 256) scan4(__ldcg(W4 + q0), 4 * q0, false);
      if (bj == i32) {  // the diagonal won: this thread's quads again, without it
        bw = NOPE;
        bj = -1;
        for (int q = threadIdx.x; q < n4; q += 256) scan4(__ldcg(W4 + q), 4 * q, true);
      }
    } else {
      for (int j = threadIdx.x; j < (int)n; j += 256) {
        const float w = __ldcg(Wr + j);
        if (better(w, bw) && j != i32) {
          bw = w;
          bj = j;
        }
      }
    }
    const u64 mine = bj >= 0 ? keyof(bw, bj) : KEY_NONE;
    tmin[threadIdx.x] = mine;
    if (threadIdx.x == 0) ncand = 0;
    __syncthreads();
    if (warp == 0) {
      // K-th smallest of the 256 minima: 8 per lane, bitonic-sorted lane lists merged by K rounds
      u64 v[8];
#pragma unroll
      for (int t = 0; t < 8; t++) v[t] = tmin[lane * 8 + t];
#pragma unroll
      for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 7 - a; b++)
          if (v[b] > v[b + 1]) { const u64 x = v[b]; v[b] = v[b + 1]; v[b + 1] = x; }
      int h = 0;
      u64 kth = KEY_NONE;
      for (int t = 0; t < K; t++) {
        u64 head = KEY_NONE;
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (u == h) head = v[u];
        u64 best = head;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
          best = other < best ? other : best;
        }
        if (best != KEY_NONE && head == best) h++;
        kth = best;  // after K rounds: the K-th smallest (KEY_NONE if fewer than K exist)
      }
      if (lane == 0) tau_s = kth;
    }
    __syncthreads();
    const u64 tau = tau_s;
    // tau's weight as a float of the row's sense (keys are orderable(+-w) << 32 | j)
    const float tau_f = tau == KEY_NONE ? (SENSE > 0 ? INFINITY : -INFINITY)
                                        : (SENSE > 0 ? from_orderable((uint32_t)(tau >> 32))
                                                     : -from_orderable((uint32_t)(tau >> 32)));
    // pass 2: keys <= tau (a float test first; ties at tau's weight compare the full key;
    // the diagonal is excluded on that rare path)
    auto take = [&](float w, int j) {
      if (SENSE > 0 ? w <= tau_f : w >= tau_f) {
        const u64 kk = keyof(w, j);
        if (kk <= tau && j != i32) {
          const int slot = atomicAdd(&ncand, 1);
          if (slot < CAP) cand[slot] = kk;
        }
      }
    };
    auto take4 = [&](float4 v, int j) {
      take(v.x, j);
      take(v.y, j + 1);
      take(v.z, j + 2);
      take(v.w, j + 3);
    };
    if (vec) {
      const float4* W4 = reinterpret_cast<const float4*>(Wr);
      const int n4 = (int)(n >> 2);
      int q0 = threadIdx.x;
      for (; q0 + 7 * 256 < n4; q0 += 8 * 256) {
        float4 w[8];
#pragma unroll
        for (int u = 0; u < 8; u++) w[u] = __ldcs(W4 + q0 + u * 256);
#pragma unroll
        for (int u = 0; u < 8; u++) take4(w[u], 4 * (q0 + u * 256));
      }
      for (; q0 < n4; q0 += 256) take4(__ldcs(W4 + q0), 4 * q0);
    } else {
      for (int j = threadIdx.x; j < (int)n; j += 256) take(__ldcs(Wr + j), j);
    }
    __syncthreads();
    if (warp == 0) {
      const int nc = ncand;
      if (nc > CAP) {  // more than CAP keys tie below the bound: no cache for this row
        if (lane == 0) {
          ccnt[i] = -1;
          // its round-0 minimum: the smallest thread minimum
          u64 b = KEY_NONE;
          for (int t = 0; t < 256; t++) b = tmin[t] < b ? tmin[t] : b;
          if (b != KEY_NONE) compbest[i] = (b & 0xFFFFFFFF00000000ull) | tri_index(i, (int64_t)(b & 0xFFFFFFFFull));
        }
      } else {
        // bitonic sort of 64 (two per lane: lane and lane + 32)
        u64 x0 = lane < nc ? cand[lane] : KEY_NONE, x1 = lane + 32 < nc ? cand[lane + 32] : KEY_NONE;
        // sort each 32 ascending, then merge the two halves
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
          for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
            u64 y = __shfl_xor_sync(0xffffffffu, x0, stride);
            u64 lo = x0 < y ? x0 : y, hi = x0 < y ? y : x0;
            x0 = (lower == up) ? lo : hi;
            y = __shfl_xor_sync(0xffffffffu, x1, stride);
            lo = x1 < y ? x1 : y;
            hi = x1 < y ? y : x1;
            x1 = (lower == up) ? lo : hi;
          }
        // the K (<= 32) smallest of two sorted lists: lane t takes rank t by merging
        const u64 y1 = __shfl_sync(0xffffffffu, x1, 31 - lane);  // reversed second list
        u64 m = x0 < y1 ? x0 : y1;                              // bitonic sequence of the 32 smallest
#pragma unroll
        for (int stride = 16; stride > 0; stride >>= 1) {
          const u64 y = __shfl_xor_sync(0xffffffffu, m, stride);
          const bool lower = (lane & stride) == 0;
          m = lower ? (m < y ? m : y) : (m < y ? y : m);
        }
        const int take = (int)(nc < K ? nc : K);
        if (lane < take) {
          const int64_t j = (int64_t)(m & 0xFFFFFFFFull);
          const u64 g = (m & 0xFFFFFFFF00000000ull) | tri_index(i, j);
          ckey[i * K + lane] = g;
          cj[i * K + lane] = (int)j;
          if (lane == 0) compbest[i] = g;
        }
        if (lane == 0) ccnt[i] = take;
      }
    }
    __syncthreads();
  }
}

// Single-pass variant (K <= 8): ONE WARP PER ROW and one read of W.  The warp keeps
// the row's K smallest keys so far as a sorted list distributed over lanes 0..K-1, and
// its K-th as a warp-uniform threshold.  A batch is 8 float4 per lane (1024 columns);
// each lane tests its 32 values against the threshold with one float compare each
// (candidates are rare once the list is warm), and the warp inserts the few candidates
// one by one (shuffle shift of the list).  The first batch inserts the lanes' minima
// first, so that the threshold is tight at once.  Keys are (orderable(m), j), m the
// sense-adjusted weight -- the same cache as k_scan_weights_topk, whose second pass
// re-read the row from L2 and whose CTA-wide merges idled the CTA's loads.
template <int K, int SENSE>
__global__ void __launch_bounds__(256, 3) k_scan_weights_topk_w(const float* __restrict__ W, int64_t n, int64_t row0,
                                                           int64_t rows, u64* __restrict__ ckey, int* __restrict__ cj,
                                                           int* __restrict__ ccnt, u64* __restrict__ compbest) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n4 = (int)(n >> 2);  // (launched only for n % 4 == 0 and an aligned W)
  for (int64_t r = gw; r < rows; r += nw) {
    const int64_t i = row0 + r;
    const int i32 = (int)i;
    const float4* W4 = reinterpret_cast<const float4*>(W + r * n);
    u64 lk = KEY_NONE;  // lane t < K: the t-th smallest key so far
    u64 thr = KEY_NONE;
    auto insert = [&](u64 kc) {
      u64 prev = __shfl_up_sync(0xffffffffu, lk, 1);
      if (lane == 0) prev = 0ull;
      const u64 nk = prev > kc ? prev : (lk > kc ? kc : lk);
      lk = lane < K ? nk : KEY_NONE;
      thr = __shfl_sync(0xffffffffu, lk, K - 1);
    };
    for (int b0 = 0; b0 < n4; b0 += 256) {
      float m[32];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int q = b0 + u * 32 + lane;
        float4 v = make_float4(NAN, NAN, NAN, NAN);  // past the row: never a candidate
        if (q < n4) v = __ldcs(W4 + q);
        m[4 * u + 0] = SENSE > 0 ? v.x : -v.x;
        m[4 * u + 1] = SENSE > 0 ? v.y : -v.y;
        m[4 * u + 2] = SENSE > 0 ? v.z : -v.z;
        m[4 * u + 3] = SENSE > 0 ? v.w : -v.w;
      }
      if ((i32 >> 10) == (b0 >> 8)) {  // (warp-uniform) the batch with the diagonal: NaN
        const int qd = i32 >> 2;
#pragma unroll
        for (int u = 0; u < 8; u++)
#pragma unroll
          for (int c = 0; c < 4; c++)
            if (b0 + u * 32 + lane == qd && (i32 & 3) == c) m[4 * u + c] = NAN;
      }
      auto jof = [&](int e) { return 4 * (b0 + (e >> 2) * 32 + lane) + (e & 3); };
      // (-0 -> +0 in the key, reading Q5; the compares treat them as equal anyway)
      auto keyof = [&](int e) { return ((u64)orderable(m[e] + 0.0f) << 32) | (u64)(unsigned)jof(e); };
      int own = -1;  // warm-up: this lane's minimum, inserted already
      if (thr == KEY_NONE) {
        float mn = NAN;
#pragma unroll
        for (int e = 0; e < 32; e++) mn = fminf(mn, m[e]);  // (fminf skips NaN)
#pragma unroll
        for (int e = 31; e >= 0; e--)
          if (m[e] == mn) own = e;  // the smallest j among equal minima
        u64 mk = KEY_NONE;
#pragma unroll
        for (int e = 0; e < 32; e++)
          if (e == own) mk = keyof(e);
        unsigned bal = __ballot_sync(0xffffffffu, own >= 0);
        while (bal) {
          const int l = __ffs(bal) - 1;
          bal &= bal - 1;
          insert(__shfl_sync(0xffffffffu, mk, l));
        }
      }
      // candidates: m below the threshold's weight; a tie at that weight can only win if
      // the threshold's column lies in this batch or later (columns of earlier batches
      // are smaller), which is rare once the list is warm (warp-uniform test)
      const float tw = thr == KEY_NONE ? INFINITY : from_orderable((uint32_t)(thr >> 32));
      const bool tie_ok = thr == KEY_NONE || (int)(uint32_t)thr >= 4 * b0;
      unsigned mask = 0;
#pragma unroll
      for (int e = 0; e < 32; e++)
        if (m[e] < tw || (tie_ok && m[e] == tw)) mask |= 1u << e;
      if (own >= 0) mask &= ~(1u << own);
      if (__any_sync(0xffffffffu, mask != 0)) {
#pragma unroll
        for (int e = 0; e < 32; e++) {
          unsigned bal = __ballot_sync(0xffffffffu, (mask >> e) & 1u);
          const u64 ke = keyof(e);
          while (bal) {
            const int l = __ffs(bal) - 1;
            bal &= bal - 1;
            const u64 kc = __shfl_sync(0xffffffffu, ke, l);
            if (kc < thr) insert(kc);
          }
        }
      }
    }
    // the list (ascending local keys (w, j)) -> global keys; lane t writes entry t
    const unsigned valid = __ballot_sync(0xffffffffu, lk != KEY_NONE);
    if (lane < K && lk != KEY_NONE) {
      const int64_t j = (int64_t)(lk & 0xFFFFFFFFull);
      const u64 g = (lk & 0xFFFFFFFF00000000ull) | tri_index(i, j);
      ckey[i * K + lane] = g;
      cj[i * K + lane] = (int)j;
      if (lane == 0) compbest[i] = g;
    }
    if (lane == 0) ccnt[i] = __popc(valid);
  }
}

// weights mode: exact scan of a list of rows (component-filtered argmin, re-scans)
template <int SENSE>
__global__ void __launch_bounds__(256) k_scan_weights_list(const float* __restrict__ W, int64_t n, int64_t row0,
                                                         const int* __restrict__ list,
                                                         const unsigned* __restrict__ count,
                                                         const int* __restrict__ comp, u64* __restrict__ compbest) {
  __shared__ u64 red[8];
  const unsigned cnt = *count;
  for (unsigned e = blockIdx.x; e < cnt; e += gridDim.x) {
    const int64_t i = list[e];
    const float* Wr = W + (i - row0) * n;
    const int ci = comp[i];
    u64 best = KEY_NONE;
    for (int64_t j = threadIdx.x; j < n; j += 256) {
      if (__ldg(comp + j) == ci) continue;
      float m = SENSE > 0 ? __ldcs(Wr + j) : -__ldcs(Wr + j);
      m = m + 0.0f;
      const u64 loc = ((u64)orderable(m) << 32) | (u64)j;
      best = loc < best ? loc : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 b = red[0];
      for (int t = 1; t < 8; t++) b = red[t] < b ? red[t] : b;
      if (b != KEY_NONE) {
        const int64_t j = (int64_t)(b & 0xFFFFFFFFull);
        atomicMin(compbest + ci, (b & 0xFFFFFFFF00000000ull) | tri_index(i, j));
      }
    }
    __syncthreads();
  }
}

appd_status launch_scan_weights_topk(appd_ctx* c, const float* W, int64_t n, int64_t row0, int64_t rows, int K,
                                     int sense, u64* ckey, int* cj, int* ccnt, u64* compbest) {
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(rows, 1), (int64_t)c->sm_count * 8);
#define APPD_WTOPK(KK)                                                                                       \
  (sense > 0 ? (k_scan_weights_topk<KK, 1><<<grid, 256, 0, c->stream>>>(W, n, row0, rows, ckey, cj, ccnt, compbest)) \
             : (k_scan_weights_topk<KK, -1><<<grid, 256, 0, c->stream>>>(W, n, row0, rows, ckey, cj, ccnt, compbest)))
  // K <= 8: the single-pass warp-per-row kernel (8 warps per CTA)
  const int wgrid = (int)std::min<int64_t>(std::max<int64_t>((rows + 7) / 8, 1), (int64_t)c->sm_count * 8);
#define APPD_WTOPK_W(KK)                                                                                        \
  (sense > 0 ? (k_scan_weights_topk_w<KK, 1><<<wgrid, 256, 0, c->stream>>>(W, n, row0, rows, ckey, cj, ccnt, compbest)) \
             : (k_scan_weights_topk_w<KK, -1><<<wgrid, 256, 0, c->stream>>>(W, n, row0, rows, ckey, cj, ccnt, compbest)))
  const bool wv = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  switch (K) {
    case 4: if (wv) APPD_WTOPK_W(4); else APPD_WTOPK(4); break;
    case 8: if (wv) APPD_WTOPK_W(8); else APPD_WTOPK(8); break;
    case 16: APPD_WTOPK(16); break;
    case 32: APPD_WTOPK(32); break;
    default: return fail(c, APPD_ERR_INVALID_ARGUMENT, "cache length K = %d (4, 8, 16 or 32)", K);
  }
#undef APPD_WTOPK
#undef APPD_WTOPK_W
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_scan_weights_list(appd_ctx* c, const float* W, int64_t n, int64_t row0, const int* list,
                                     const unsigned* count, int max_rows, const int* comp, u64* compbest,
                                     int sense) {
  if (max_rows <= 0) return APPD_OK;
  const int grid = std::min(max_rows, c->sm_count * 8);
  if (sense > 0) k_scan_weights_list<1><<<grid, 256, 0, c->stream>>>(W, n, row0, list, count, comp, compbest);
  else k_scan_weights_list<-1><<<grid, 256, 0, c->stream>>>(W, n, row0, list, count, comp, compbest);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_scan_weights(appd_ctx* c, const float* W, int64_t n, int64_t row0, int64_t rows,
                                const int* comp, u64* compbest, int sense) {
  int grid = (int)(rows < (int64_t)c->sm_count * 8 ? rows : (int64_t)c->sm_count * 8);
  if (grid < 1) grid = 1;
  if (comp == nullptr) {
    if (sense > 0) k_scan_weights<true, 1><<<grid, 256, 0, c->stream>>>(W, n, row0, rows, comp, compbest);
    else k_scan_weights<true, -1><<<grid, 256, 0, c->stream>>>(W, n, row0, rows, comp, compbest);
  } else {
    if (sense > 0) k_scan_weights<false, 1><<<grid, 256, 0, c->stream>>>(W, n, row0, rows, comp, compbest);
    else k_scan_weights<false, -1><<<grid, 256, 0, c->stream>>>(W, n, row0, rows, comp, compbest);
  }
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// points mode: X is first transposed to XT[dpad][npad] (zero padded: a zero
// coordinate adds fmaf(0,0,acc) = acc exactly, so padding d changes nothing).
// A CTA owns 128 rows and sweeps a range of 128-column tiles; each thread owns
// an 8x8 micro-tile of squared distances, accumulated over k = 0..d-1 in order
// with the pinned R1 chain  t = x_ik - x_jk (RN), acc = fma(t, t, acc) (RN),
// written with __fsub_rn/__fmaf_rn so no contraction can change it.
// ---------------------------------------------------------------------------
__global__ void k_transpose_points(const float* __restrict__ X, int64_t n, int64_t d, float* __restrict__ XT,
                                   int64_t npad, int64_t dpad) {
  __shared__ float tile[32][33];
  int64_t i0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int64_t i = i0 + r, k = k0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < n && k < d) ? X[i * d + k] : 0.0f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    int64_t k = k0 + r, i = i0 + threadIdx.x;
    if (k < dpad && i < npad) XT[k * npad + i] = tile[threadIdx.x][r];
  }
}

appd_status launch_transpose_points(appd_ctx* c, const float* X, int64_t n, int64_t d, float* XT, int64_t npad,
                                    int64_t dpad) {
  dim3 grid((unsigned)(npad / 32), (unsigned)(dpad / 32));
  k_transpose_points<<<grid, dim3(32, 8), 0, c->stream>>>(X, n, d, XT, npad, dpad);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

constexpr int PT_BM = 128, PT_BN = 128, PT_KC = 32;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// METRIC (NEXT-3): 0 the pinned R1 chain (squared Euclidean), 1 Manhattan (acc + |t| in k
// order), 2 Chebyshev (max |t|); the zero-padded coordinates add 0 / leave the max.
template <int METRIC>
__device__ __forceinline__ float metric_step(float a, float b, float acc) {
  const float t = __fsub_rn(a, b);
  if (METRIC == 0) return __fmaf_rn(t, t, acc);
  if (METRIC == 1) return __fadd_rn(acc, fabsf(t));
  return fmaxf(acc, fabsf(t));
}

// WIDE (n > 131072, the pair index no longer fits beside the weight bits): each row's
// (bits(d2) << 32 | j) minimum goes to compbest[row] instead (the per-row winners; the
// component reduction runs in two steps, k_wide_compw / k_wide_compbest)
// SENSE -1 (widest paths): the row's LARGEST distance (smallest j on ties), keyed
// by the order-reversing map of the non-negative weight bits, ~bits & 0x7FFFFFFF (the
// same (weight, max, min) strict order, weight reversed)
__device__ __forceinline__ uint32_t sense_bits(uint32_t b, int sense) { return sense > 0 ? b : (~b & 0x7FFFFFFFu); }

template <bool ROUND0, int METRIC = 0, bool WIDE = false, int SENSE = 1>
__global__ void __launch_bounds__(256, 2)
    k_scan_points(const float* __restrict__ XT, int64_t n, int64_t npad, int dpad, int64_t row0, int64_t rows,
                  int col_tiles_per_cta, const int* __restrict__ comp, u64* __restrict__ compbest, int sym) {
  extern __shared__ __align__(16) float smem[];
  float* As = smem;                           // [2][KC][BM]
  float* Bs = smem + 2 * PT_KC * PT_BM;       // [2][KC][BN]
  int* ccol = (int*)(Bs + 2 * PT_KC * PT_BN); // [BN] component labels of the current column tile
  // sym: [16][BN] per-column best of each thread row (ty) of a tile, for the column epilogue
  u64* colbest = reinterpret_cast<u64*>(ccol + PT_BN);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t rbase = row0 + (int64_t)blockIdx.x * PT_BM;
  const int64_t total_col_tiles = npad / PT_BN;
  // sym (one rank, every row): only the column tiles ct >= this row block's own, split in
  // gridDim.y parts; the pairs of an off-diagonal tile also update their COLUMNS' rows
  const int64_t rb = blockIdx.x;
  const int64_t span = sym ? (total_col_tiles - rb + gridDim.y - 1) / gridDim.y : col_tiles_per_cta;
  const int64_t ct0 = sym ? rb + (int64_t)blockIdx.y * span : (int64_t)blockIdx.y * col_tiles_per_cta;
  int64_t ct1 = ct0 + span;
  if (ct1 > total_col_tiles) ct1 = total_col_tiles;
  if (ct0 >= ct1) return;
  const int nk = dpad / PT_KC;

  int64_t ri[8];
  int cr[8];
  float bd[8];
  int64_t bj[8];
#pragma unroll
  for (int a = 0; a < 8; a++) {
    ri[a] = rbase + ty * 8 + a;
    cr[a] = ROUND0 ? (int)ri[a] : ((ri[a] < n) ? comp[ri[a]] : -1);
    bd[a] = SENSE > 0 ? INFINITY : -INFINITY;
    bj[a] = -1;
  }

  // stage loader: chunk index s = tile_local * nk + kc
  auto load_stage = [&](int64_t s, int buf) {
    int64_t ct = ct0 + s / nk;
    int kc = (int)(s % nk);
    const float* ga = XT + (int64_t)(kc * PT_KC) * npad + rbase;
    const float* gb = XT + (int64_t)(kc * PT_KC) * npad + ct * PT_BN;
    float* sa = As + buf * PT_KC * PT_BM;
    float* sb = Bs + buf * PT_KC * PT_BN;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      int e = threadIdx.x + q * 256;  // 1024 float4 per operand
      int k = e >> 5, c4 = (e & 31) * 4;
      cp_async16(sa + k * PT_BM + c4, ga + (int64_t)k * npad + c4);
      cp_async16(sb + k * PT_BN + c4, gb + (int64_t)k * npad + c4);
    }
  };

  const int64_t nstages = (ct1 - ct0) * nk;
  load_stage(0, 0);
  cp_async_commit();
  float acc[8][8];
  for (int64_t s = 0; s < nstages; s++) {
    const int buf = (int)(s & 1);
    const int kc = (int)(s % nk);
    const int64_t ct = ct0 + s / nk;
    if (kc == 0) {
#pragma unroll
      for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 8; b++) acc[a][b] = 0.0f;
    }
    if (s + 1 < nstages) load_stage(s + 1, buf ^ 1);
    cp_async_commit();
    if (kc == 0 && !ROUND0) {
      // labels of this column tile (previous readers finished at the last __syncthreads)
      int64_t j = ct * PT_BN + (threadIdx.x & 127);
      if (threadIdx.x < 128) ccol[threadIdx.x] = (j < n) ? comp[j] : -2;
    }
    cp_async_wait<1>();
    __syncthreads();
    const float* sa = As + buf * PT_KC * PT_BM;
    const float* sb = Bs + buf * PT_KC * PT_BN;
#pragma unroll 4
    for (int k = 0; k < PT_KC; k++) {
      float4 a0 = *reinterpret_cast<const float4*>(sa + k * PT_BM + ty * 8);
      float4 a1 = *reinterpret_cast<const float4*>(sa + k * PT_BM + ty * 8 + 4);
      float4 b0 = *reinterpret_cast<const float4*>(sb + k * PT_BN + tx * 8);
      float4 b1 = *reinterpret_cast<const float4*>(sb + k * PT_BN + tx * 8 + 4);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 8; b++) acc[a][b] = metric_step<METRIC>(av[a], bv[b], acc[a][b]);
    }
    if (kc == nk - 1) {
      // epilogue of this column tile: component-filtered running argmin per row.
      // Columns are visited in increasing j per thread, so strict '<' keeps the
      // smallest j among equal distances.
#pragma unroll
      for (int b = 0; b < 8; b++) {
        int64_t j = ct * PT_BN + tx * 8 + b;
        int cj = ROUND0 ? 0 : ccol[tx * 8 + b];
#pragma unroll
        for (int a = 0; a < 8; a++) {
          bool elig = ROUND0 ? (j < n && j != ri[a]) : (cj != cr[a] && cj >= 0);
          // the first eligible column is taken even at +inf (coordinates whose squares
          // overflow): every component must choose an edge
          if (elig && (bj[a] < 0 || (SENSE > 0 ? acc[a][b] < bd[a] : acc[a][b] > bd[a]))) { bd[a] = acc[a][b]; bj[a] = j; }
        }
      }
      if (sym && ct != rb) {
        // column epilogue: each column j's best row of this tile, (weight, i) smallest, over
        // the thread's 8 rows, then over the 16 thread rows through shared memory
#pragma unroll
        for (int b = 0; b < 8; b++) {
          const int64_t j = ct * PT_BN + tx * 8 + b;
          const int cj = ROUND0 ? 0 : ccol[tx * 8 + b];
          u64 best = KEY_NONE;
#pragma unroll
          for (int a = 0; a < 8; a++) {
            const bool elig = ri[a] < n && j < n && (ROUND0 || (cj != cr[a] && cj >= 0));
            const u64 key = ((u64)sense_bits(__float_as_uint(acc[a][b]), SENSE) << 32) | (u64)ri[a];
            best = elig && key < best ? key : best;
          }
          colbest[ty * PT_BN + tx * 8 + b] = best;
        }
        __syncthreads();
        if (threadIdx.x < PT_BN) {
          u64 best = KEY_NONE;
#pragma unroll
          for (int t = 0; t < 16; t++) {
            const u64 v = colbest[t * PT_BN + threadIdx.x];
            best = v < best ? v : best;
          }
          const int64_t j = ct * PT_BN + threadIdx.x;
          if (best != KEY_NONE) {
            if (WIDE) {
              atomicMin(compbest + j, best);  // row j's winner (w, i)
            } else {
              const int64_t i = (int64_t)(best & 0xFFFFFFFFull);
              const u64 gkey = (((best >> 32) & 0x7FFFFFFFull) << 33) | tri_index(i, j);
              atomic_min_lt(compbest + (ROUND0 ? j : ccol[threadIdx.x]), gkey);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  // reduce (d2, j) over the 16 threads sharing each row (lanes differing in tx)
#pragma unroll
  for (int a = 0; a < 8; a++) {
    u64 key = bj[a] >= 0 ? (((u64)sense_bits(__float_as_uint(bd[a]), SENSE) << 32) | (u64)bj[a]) : KEY_NONE;
#pragma unroll
    for (int o = 8; o; o >>= 1) {
      u64 other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other < key ? other : key;
    }
    if (WIDE) {
      if (tx == 0 && key != KEY_NONE && ri[a] < row0 + rows && ri[a] < n) atomic_min_lt(compbest + ri[a], key);
      continue;
    }
    if (tx == 0 && key != KEY_NONE && ri[a] < row0 + rows && ri[a] < n) {
      int64_t j = (int64_t)(key & 0xFFFFFFFFull);
      u64 d2bits = (key >> 32) & 0x7FFFFFFFull;
      u64 gkey = (d2bits << 33) | tri_index(ri[a], j);
      atomic_min_lt(compbest + cr[a], gkey);
    }
  }
}

appd_status launch_scan_points(appd_ctx* c, const float* XT, int64_t n, int64_t npad, int64_t dpad, int64_t row0,
                               int64_t rows, const int* comp, u64* compbest, bool wide) {
  const size_t smem = (size_t)(2 * PT_KC * PT_BM + 2 * PT_KC * PT_BN) * 4 + PT_BN * 4 + 16 * PT_BN * 8;
  if (rows <= 0) return APPD_OK;
  // one rank holding every row: the symmetric pass (each unordered pair once)
  const int sym = (row0 == 0 && rows == n) ? 1 : 0;
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
    cudaFuncSetAttribute(k_scan_points<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<false, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<true, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<true, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_points<false, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#define APPD_ATTR_W(R0, MT, WD) \
  cudaFuncSetAttribute(k_scan_points<R0, MT, WD, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
    APPD_ATTR_W(true, 0, false); APPD_ATTR_W(false, 0, false); APPD_ATTR_W(true, 1, false);
    APPD_ATTR_W(false, 1, false); APPD_ATTR_W(true, 2, false); APPD_ATTR_W(false, 2, false);
    APPD_ATTR_W(true, 0, true); APPD_ATTR_W(false, 0, true); APPD_ATTR_W(true, 1, true);
    APPD_ATTR_W(false, 1, true); APPD_ATTR_W(true, 2, true); APPD_ATTR_W(false, 2, true);
#undef APPD_ATTR_W
    setup_done(attr, c);
  }
  int64_t row_blocks = (rows + PT_BM - 1) / PT_BM;
  int64_t col_tiles = npad / PT_BN;
  // enough CTAs for ~4 waves of 2 CTAs/SM; split the column range accordingly (sym: the
  // first row blocks hold the longest ranges and are scheduled first)
  int64_t want = (int64_t)c->sm_count * 2 * 4 * (sym ? 2 : 1);
  int64_t splits = (want + row_blocks - 1) / row_blocks;
  if (splits > col_tiles) splits = col_tiles;
  if (splits < 1) splits = 1;
  int64_t per = (col_tiles + splits - 1) / splits;
  splits = (col_tiles + per - 1) / per;
  dim3 grid((unsigned)row_blocks, (unsigned)splits);
#define APPD_SCAN_POINTS(R0, MT)                                                                               \
  (c->opt.sense > 0                                                                                           \
       ? k_scan_points<R0, MT, false, 1><<<grid, 256, smem, c->stream>>>(XT, n, npad, (int)dpad, row0, rows,  \
                                                                          (int)per, comp, compbest, sym)      \
       : k_scan_points<R0, MT, false, -1><<<grid, 256, smem, c->stream>>>(XT, n, npad, (int)dpad, row0, rows, \
                                                                           (int)per, comp, compbest, sym))
#define APPD_SCAN_POINTS_W(R0, MT)                                                                            \
  (c->opt.sense > 0                                                                                          \
       ? k_scan_points<R0, MT, true, 1><<<grid, 256, smem, c->stream>>>(XT, n, npad, (int)dpad, row0, rows,  \
                                                                         (int)per, comp, compbest, sym)      \
       : k_scan_points<R0, MT, true, -1><<<grid, 256, smem, c->stream>>>(XT, n, npad, (int)dpad, row0, rows, \
                                                                          (int)per, comp, compbest, sym))
  const int mt = c->opt.metric;
  if (wide) {
    if (comp == nullptr) {
      if (mt == 1) APPD_SCAN_POINTS_W(true, 1);
      else if (mt == 2) APPD_SCAN_POINTS_W(true, 2);
      else APPD_SCAN_POINTS_W(true, 0);
    } else {
      if (mt == 1) APPD_SCAN_POINTS_W(false, 1);
      else if (mt == 2) APPD_SCAN_POINTS_W(false, 2);
      else APPD_SCAN_POINTS_W(false, 0);
    }
  } else if (comp == nullptr) {
    if (mt == 1) APPD_SCAN_POINTS(true, 1);
    else if (mt == 2) APPD_SCAN_POINTS(true, 2);
    else APPD_SCAN_POINTS(true, 0);
  } else {
    if (mt == 1) APPD_SCAN_POINTS(false, 1);
    else if (mt == 2) APPD_SCAN_POINTS(false, 2);
    else APPD_SCAN_POINTS(false, 0);
  }
#undef APPD_SCAN_POINTS
#undef APPD_SCAN_POINTS_W
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// Wide keys (points, n > 131072: bits(d2) takes 31 bits and the pair index up to 40, more
// than 64 together).  The strict edge order (weight, max(u,v), min(u,v)) is kept by a
// two-step component reduction (SURVEY §8(a) packed-key note: "two-pass, min w first,
// then min id among the winners"): compw[C] = the minimum weight bits over C's row
// winners, then compbest[C] = the minimum pair index among the winners of that weight.
// compbest then holds the pair index alone (the contraction decodes it with shift 63).
// ---------------------------------------------------------------------------
__global__ void k_wide_compw(const u64* __restrict__ rowbest, const int* __restrict__ comp, int64_t r0, int64_t r1,
                             bool round0, u64* __restrict__ compw) {
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 rb = rowbest[i];
    if (rb != KEY_NONE) atomicMin(compw + (round0 ? i : comp[i]), rb >> 32);
  }
}

__global__ void k_wide_compbest(const u64* __restrict__ rowbest, const int* __restrict__ comp, int64_t r0,
                                int64_t r1, bool round0, const u64* __restrict__ compw, u64* __restrict__ compbest) {
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 rb = rowbest[i];
    if (rb == KEY_NONE) continue;
    const int ci = round0 ? (int)i : comp[i];
    if ((rb >> 32) == compw[ci]) atomicMin(compbest + ci, tri_index(i, (int64_t)(rb & 0xFFFFFFFFull)));
  }
}

appd_status launch_wide_compw(appd_ctx* c, const u64* rowbest, const int* comp, int64_t r0, int64_t r1, u64* compw) {
  if (r1 <= r0) return APPD_OK;
  const int grid = (int)std::min<int64_t>((r1 - r0 + 255) / 256, (int64_t)c->sm_count * 8);
  k_wide_compw<<<grid, 256, 0, c->stream>>>(rowbest, comp, r0, r1, comp == nullptr, compw);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_wide_compbest(appd_ctx* c, const u64* rowbest, const int* comp, int64_t r0, int64_t r1,
                                 const u64* compw, u64* compbest) {
  if (r1 <= r0) return APPD_OK;
  const int grid = (int)std::min<int64_t>((r1 - r0 + 255) / 256, (int64_t)c->sm_count * 8);
  k_wide_compbest<<<grid, 256, 0, c->stream>>>(rowbest, comp, r0, r1, comp == nullptr, compw, compbest);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// the MST edges of the wide keys (pair indices): key2[e] = bits(weight) << 32 | e with the
// weight recomputed from X by the same chain as the scan (R1 d2, or the L1 / L-inf
// distance), so that a radix sort over bits [32, 64) gives the Kruskal order (a4)
template <int METRIC>
__global__ void k_wide_edge_keys(const u64* __restrict__ tri, int64_t m, const float* __restrict__ X, int d,
                                 int sense, u64* __restrict__ key2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t u, v;
    tri_decode(tri[e] & ((1ull << 63) - 1), &u, &v);
    float acc = 0.0f;
    for (int k = 0; k < d; k++) {
      const float t = __fsub_rn(X[u * d + k], X[v * d + k]);
      if (METRIC == 0) acc = __fmaf_rn(t, t, acc);
      else if (METRIC == 1) acc = __fadd_rn(acc, fabsf(t));
      else acc = fmaxf(acc, fabsf(t));
    }
    key2[e] = (u64)sense_bits(__float_as_uint(acc), sense) << 32 | (u64)e;  // Kruskal order of the sense
  }
}

template <int METRIC>
__global__ void k_wide_decode(const u64* __restrict__ key2_sorted, const u64* __restrict__ tri, int64_t m, int sense,
                              int32_t* __restrict__ eu, int32_t* __restrict__ ev, float* __restrict__ ew) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    const u64 k2 = key2_sorted[p];
    int64_t u, v;
    tri_decode(tri[k2 & 0xFFFFFFFFull] & ((1ull << 63) - 1), &u, &v);
    const float w = __uint_as_float(sense_bits((uint32_t)(k2 >> 32), sense));
    eu[p] = (int32_t)u;
    ev[p] = (int32_t)v;
    ew[p] = METRIC == 0 ? __fsqrt_rn(w) : w;  // APPD(sqrtf o d2) = sqrtf o APPD(d2), App. A.4
  }
}

appd_status wide_edges(appd_ctx* c, const u64* mstkeys, int64_t m, const float* X, int64_t d, int metric, int sense,
                       u64* key2, u64* key2_sorted, int32_t* eu, int32_t* ev, float* ew) {
  if (m <= 0) return APPD_OK;
  const int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)c->sm_count * 8);
  if (metric == 1) k_wide_edge_keys<1><<<grid, 256, 0, c->stream>>>(mstkeys, m, X, (int)d, sense, key2);
  else if (metric == 2) k_wide_edge_keys<2><<<grid, 256, 0, c->stream>>>(mstkeys, m, X, (int)d, sense, key2);
  else k_wide_edge_keys<0><<<grid, 256, 0, c->stream>>>(mstkeys, m, X, (int)d, sense, key2);
  APPD_LAUNCHED(c);
  appd_status s = sort_keys_u64_bits64(c, key2, key2_sorted, m, 32, 64);
  if (s) return s;
  if (metric == 1) k_wide_decode<1><<<grid, 256, 0, c->stream>>>(key2_sorted, mstkeys, m, sense, eu, ev, ew);
  else if (metric == 2) k_wide_decode<2><<<grid, 256, 0, c->stream>>>(key2_sorted, mstkeys, m, sense, eu, ev, ew);
  else k_wide_decode<0><<<grid, 256, 0, c->stream>>>(key2_sorted, mstkeys, m, sense, eu, ev, ew);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// component step: hook, break mutual pairs, pointer-jump, compact, relabel
// ---------------------------------------------------------------------------
__global__ void k_fill_u64(u64* p, int64_t count, u64 v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
appd_status launch_fill_u64(appd_ctx* c, u64* p, int64_t count, u64 v) {
  int grid = (int)((count + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  if (grid < 1) grid = 1;
  k_fill_u64<<<grid, 256, 0, c->stream>>>(p, count, v);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// queued small results -> mapped pinned host words (one warp per entry)
struct PubArgs {
  const unsigned* src[16];
  unsigned* dst[16];
  int words[16];
  int count;
};
__global__ void k_publish(const PubArgs a) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = w; e < a.count; e += blockDim.x >> 5)
    for (int i = lane; i < a.words[e]; i += 32) a.dst[e][i] = a.src[e][i];
}
appd_status publish(appd_ctx* c, void* host_dst, const void* dev_src, size_t bytes) {
  const int64_t off = (reinterpret_cast<unsigned*>(host_dst) - c->pinned_small);
  if (!c->pinned_small_dev || off < 0 || off + (int64_t)(bytes / 4) > 64 || bytes % 4) {
    APPD_CUDA(c, cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, c->stream));
    return APPD_OK;
  }
  if (c->npub == 16) {
    appd_status s = publish_flush(c);
    if (s) return s;
  }
  c->pub[c->npub++] = {dev_src, c->pinned_small_dev + off, (int)(bytes / 4)};
  return APPD_OK;
}
appd_status publish_flush(appd_ctx* c) {
  if (c->npub == 0) return APPD_OK;
  PubArgs a;
  for (int e = 0; e < c->npub; e++) {
    a.src[e] = reinterpret_cast<const unsigned*>(c->pub[e].src);
    a.dst[e] = c->pub[e].dst;
    a.words[e] = c->pub[e].words;
  }
  a.count = c->npub;
  c->npub = 0;
  k_publish<<<1, 32 * 16, 0, c->stream>>>(a);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

__global__ void k_iota(int* p, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int)i;
}
appd_status launch_iota(appd_ctx* c, int* p, int64_t count) {
  int grid = (int)((count + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  if (grid < 1) grid = 1;
  k_iota<<<grid, 256, 0, c->stream>>>(p, count);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// link[c] = the component at the other end of c's chosen edge
__global__ void k_hook(const u64* __restrict__ compbest, int64_t k, const int* __restrict__ comp, int shift,
                       int* __restrict__ link) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= k) return;
  u64 key = compbest[c];
  if (key == KEY_NONE) { link[c] = (int)c; return; }
  int64_t u, v;
  tri_decode(key & ((1ull << shift) - 1), &u, &v);
  int cu = comp[u], cv = comp[v];
  link[c] = (cu == (int)c) ? cv : cu;
}
appd_status launch_hook(appd_ctx* c, const u64* compbest, int64_t k, const int* comp, int shift, int* link) {
  k_hook<<<(unsigned)((k + 255) / 256), 256, 0, c->stream>>>(compbest, k, comp, shift, link);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// Under a strict edge order, the only cycles among chosen edges are 2-cycles
// (c -> o -> c, the same edge).  The smaller id becomes the root; the edge is
// recorded once (by the smaller id).  Every other chosen edge is a new MST edge.
__global__ void k_mutual(const u64* __restrict__ compbest, int64_t k, const int* __restrict__ link,
                         int* __restrict__ parent, u64* __restrict__ mstkeys, int* __restrict__ counters) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= k) return;
  int o = link[c];
  if (o == (int)c) { parent[c] = (int)c; return; }
  bool mutual = link[o] == (int)c;
  if (mutual && (int)c < o) {
    parent[c] = (int)c;
  } else {
    parent[c] = o;
  }
  if (!(mutual && (int)c > o)) {
    int slot = atomicAdd(counters, 1);
    mstkeys[slot] = compbest[c];
  }
}
appd_status launch_mutual(appd_ctx* c, const u64* compbest, int64_t k, const int* link, int* parent, u64* mstkeys,
                          int* counters) {
  k_mutual<<<(unsigned)((k + 255) / 256), 256, 0, c->stream>>>(compbest, k, link, parent, mstkeys, counters);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// pointer jumping to the root; flags[c] = (c is a root)
__global__ void k_jump(int* parent, int64_t k, int* flags) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= k) return;
  int p = parent[c];
  while (true) {
    int pp = parent[p];
    if (pp == p) break;
    p = pp;
  }
  parent[c] = p;  // concurrent readers see either the old ancestor or the root
  flags[c] = (p == (int)c) ? 1 : 0;
}
appd_status launch_jump(appd_ctx* c, int* parent, int64_t k, int* flags) {
  k_jump<<<(unsigned)((k + 255) / 256), 256, 0, c->stream>>>(parent, k, flags);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

__global__ void k_relabel(int* comp, int64_t n, const int* __restrict__ parent, const int* __restrict__ newid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    comp[i] = newid[parent[comp[i]]];
}
appd_status launch_relabel(appd_ctx* c, int* comp, int64_t n, const int* parent, const int* newid) {
  int grid = (int)((n + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  k_relabel<<<grid, 256, 0, c->stream>>>(comp, n, parent, newid);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// (the radix sorts of the path: k_sort.cu)

// ---------------------------------------------------------------------------
// One Boruvka contraction in a single cooperative launch (grid-wide barriers between the
// steps of k_hook, k_mutual, k_jump, the exclusive scan of the root flags and k_relabel):
// the same operations in the same order, one launch instead of six.  newid[k] = roots.
// ---------------------------------------------------------------------------
constexpr int kContractThreads = 1024;
constexpr int64_t kContractOneMax = 1024;  // one CTA (one item per thread): CTA barriers
// development builds (APPD_MARKS): %globaltimer after each phase, CTA 0 (LookupArgs.marks)
__device__ __forceinline__ void contract_mark(const LookupArgs& la, int i) {
  if (la.marks && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    la.marks[i] = t;
  }
}
// ONE: a single CTA does it all (n, k <= kContractOneMax, where the cooperative grid would
// be one CTA anyway): every grid-wide barrier becomes a CTA barrier (C1 with Boruvka forced:
// MST 0.144 -> 0.102 ms).  At C2 (n = 4096) one CTA measured no faster than four: there the
// pointer chasing and the cache lookups' dependent loads are the bound, not the barriers.
template <bool ONE>
__device__ __forceinline__ void contract_sync(unsigned* bar) {
  if constexpr (ONE) __syncthreads();
  else coop_grid_sync(bar);
}
template <bool ONE>
__global__ void __launch_bounds__(kContractThreads) k_contract(u64* __restrict__ compbest, int k,
                                                             int* __restrict__ comp, int n, int shift,
                                                             int* __restrict__ link, int* __restrict__ parent,
                                                             u64* __restrict__ mstkeys, int* __restrict__ counters,
                                                             int* __restrict__ flags, int* __restrict__ newid,
                                                             int* __restrict__ blocksum, LookupArgs la,
                                                             unsigned* __restrict__ bar) {
  const int T = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  contract_mark(la, 0);
  // hook: the component at the other end of each component's lightest edge
  for (int c = tid; c < k; c += T) {
    const u64 key = compbest[c];
    if (key == KEY_NONE) {
      link[c] = c;
      continue;
    }
    int64_t u, v;
    tri_decode(key & ((1ull << shift) - 1), &u, &v);
    const int cu = comp[u], cv = comp[v];
    link[c] = (cu == c) ? cv : cu;
  }
  contract_sync<ONE>(bar);
  contract_mark(la, 1);
  // mutual pairs: the smaller id is the root, the shared edge is recorded once
  for (int c = tid; c < k; c += T) {
    const int o = link[c];
    if (o == c) {
      parent[c] = c;
      continue;
    }
    const bool mutual = link[o] == c;
    parent[c] = (mutual && c < o) ? c : o;
    if (!(mutual && c > o)) mstkeys[atomicAdd(counters, 1)] = compbest[c];
  }
  contract_sync<ONE>(bar);
  contract_mark(la, 2);
  // (compbest is not read after the hook and mutual phases: the next round's lookup can
  // start from KEY_NONE without a barrier of its own)
  if (la.ckey) {
    for (int i = tid; i < n; i += T) compbest[i] = KEY_NONE;
    if (tid == 0) *la.count = 0u;
  }
  // pointer jumping to the roots
  for (int c = tid; c < k; c += T) {
    int p = parent[c];
    while (true) {
      const int pp = parent[p];
      if (pp == p) break;
      p = pp;
    }
    parent[c] = p;
    flags[c] = p == c ? 1 : 0;
  }
  contract_sync<ONE>(bar);
  contract_mark(la, 3);
  // exclusive scan of the flags: block b owns [b S, (b+1) S)
  __shared__ int wsum[kContractThreads / 32];
  __shared__ int carry_s;
  const int S = (k + gridDim.x - 1) / gridDim.x;
  const int lo = min(k, (int)blockIdx.x * S), hi = min(k, lo + S);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = lo; base < hi; base += kContractThreads) {
    const int i = base + threadIdx.x;
    const int f = i < hi ? flags[i] : 0;
    int x = f;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = carry_s + (warp ? wsum[warp - 1] : 0) + x - f;
    if (i < hi) newid[i] = before;  // block-local exclusive prefix
    __syncthreads();
    if (threadIdx.x == 0) carry_s += wsum[kContractThreads / 32 - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) blocksum[blockIdx.x] = carry_s;
  contract_sync<ONE>(bar);
  contract_mark(la, 4);
  const int off = blocks_before(blocksum);
  for (int i = lo + threadIdx.x; i < hi; i += kContractThreads) newid[i] += off;
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) newid[k] = off + carry_s;
  contract_sync<ONE>(bar);
  contract_mark(la, 5);
  // relabel the points
  for (int i = tid; i < n; i += T) comp[i] = newid[parent[comp[i]]];
  if (!la.ckey) return;
  // the next round's cache lookup (k_cache_lookup, k_rescan_select) on the final labels
  contract_sync<ONE>(bar);
  contract_mark(la, 6);
  for (int i = la.r0 + tid; i < la.r1; i += T) {
    const int c = la.ccnt[i];
    const int ci = comp[i];
    int flag = 1;
    if (c > 0) {
      int t = 0;
      if (la.K == 8 && c == 8) {  // the common case: all eight labels loaded at once
        const int4* cj4 = reinterpret_cast<const int4*>(la.cj + (int64_t)i * 8);
        const int4 a = cj4[0], b = cj4[1];
        const int cc[8] = {comp[a.x], comp[a.y], comp[a.z], comp[a.w], comp[b.x], comp[b.y], comp[b.z], comp[b.w]};
        t = 8;
#pragma unroll
        for (int u = 7; u >= 0; u--)
          if (cc[u] != ci) t = u;  // the first cached entry in another component
      } else {
        while (t < c && comp[la.cj[(int64_t)i * la.K + t]] == ci) t++;
      }
      if (t < c) {
        // (most rows of a component lose: reading the current minimum first skips their
        // atomics; in the last rounds 64K rows hit a few dozen components)
        const u64 key = la.ckey[(int64_t)i * la.K + t];
        if (key < __ldcg(compbest + ci)) atomicMin(compbest + ci, key);
        flag = 0;
      }
      if (flag && c == n - 1) flag = 0;  // every other point cached, none eligible
    }
    la.need[i] = flag;
  }
  contract_sync<ONE>(bar);
  contract_mark(la, 7);
  for (int i = la.r0 + tid; i < la.r1; i += T) {
    if (!la.need[i]) continue;
    const int c = la.ccnt[i];
    if (c > 0 && la.ckey[(int64_t)i * la.K + (c - 1)] >= compbest[comp[i]]) {
      la.need[i] = 0;
      continue;
    }
    la.list[atomicAdd(la.count, 1u)] = i;
  }
}

appd_status launch_contract(appd_ctx* c, u64* compbest, int64_t k, int* comp, int64_t n, int shift, int* link,
                            int* parent, u64* mstkeys, int* counters, int* flags, int* newid, const LookupArgs* look) {
  static std::atomic<int> per_sm_plus1[64];  // 0: not yet measured on that device
  int per_sm = per_sm_plus1[c->device & 63].load() - 1;
  if (per_sm < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_contract<false>, kContractThreads, 0) != cudaSuccess)
      per_sm = 0;
    cudaGetLastError();
    per_sm_plus1[c->device & 63].store(per_sm + 1);
  }
  if (per_sm < 1) return APPD_ERR_UNSUPPORTED;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, (std::max(k, n) + kContractThreads - 1) /
                                                                                kContractThreads));
  int* blocksum = (int*)ws(c, S_SCAN, sizeof(int) * (grid + 1) + 64);
  if (!blocksum) return fail(c, APPD_ERR_OUT_OF_MEMORY, "contract workspace");
  int kk = (int)k, nn = (int)n;
  LookupArgs la = look ? *look : LookupArgs{};
  unsigned* bar = grid_barrier_word(c);
  if (!bar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
  void* args[] = {&compbest, &kk, &comp, &nn, &shift, &link, &parent, &mstkeys, &counters, &flags, &newid, &blocksum,
                  &la, &bar};
  static const bool marks = dev_env("APPD_MARKS") != nullptr;
  if (marks) la.marks = reinterpret_cast<unsigned long long*>(ws(c, S_TMP2, 128));
  if (std::max(k, n) <= kContractOneMax) {
    k_contract<true><<<1, kContractThreads, 0, c->stream>>>(compbest, kk, comp, nn, shift, link, parent, mstkeys,
                                                             counters, flags, newid, blocksum, la, bar);
    APPD_CUDA(c, cudaGetLastError());
  } else {
    APPD_CUDA(c, cudaLaunchCooperativeKernel((const void*)k_contract<false>, grid, kContractThreads, args, 0, c->stream));
  }
  c->launches++;
  if (marks && la.marks) {
    unsigned long long h[10] = {};
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(h, la.marks, sizeof h, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[contract] k %lld grid %d:", (long long)k, grid);
    for (int i = 1; i < 9 && h[i]; i++) fprintf(stderr, " %.1f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, " us\n");
    cudaMemset(la.marks, 0, 128);
  }
  return APPD_OK;
}

appd_status exclusive_scan_i32(appd_ctx* c, const int* in, int* out, int64_t count) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)count, c->stream);
  void* t = ws(c, S_TMP2, tmp + 16);
  if (!t) return fail(c, APPD_ERR_OUT_OF_MEMORY, "scan workspace");
  APPD_CUDA(c, cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)count, c->stream));
  c->launches += 2;
  return APPD_OK;
}

}  // namespace appd
