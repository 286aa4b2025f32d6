// k_cache.cu -- the per-row candidate cache of the points-mode Boruvka rounds
// ("Round 0: ... v2 keeps a top-K cache.  Round r: per row,
// first cached eligible candidate; rescan a row only if its cache is exhausted and
// its K-th key <= its component's best"; App. B measured ~2 full-pass equivalents
// instead of one pass per round).
//
// Round 0 (singletons) runs the tensor-core scan once with one maximum of G' per
// 32 columns (TM32).  For each row p:
//   k_topk_thr     the K-th largest chunk maximum gives an upper bound UBK of s^2 r
//                  for K distinct columns (each chunk's best column), hence for the
//                  row's K-th smallest exact R1 value;  thrK = the G' threshold below
//                  which no column can have L <= UBK (tc_common.cuh error model);
//   k_chunk_exact  every chunk with maximum >= thrK is re-evaluated with the exact R1
//                  chain (one CTA per chunk: the chunk's 32 columns stay in shared
//                  memory, one warp per listed row, one column per lane); every column
//                  with s^2 r <= UBK is appended to the row's candidate list;
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
#include "tc_common.cuh"

namespace appd {

// per row: UBK and the G' threshold thrK (float bits in UBK / thrK)
template <int K>
__global__ void k_topk_thr(const float* __restrict__ TM32, int64_t ld, int nch, int p_begin, int p_end,
                           const float* __restrict__ nrm, const float* __restrict__ len, float maxlen, ErrModel em,
                           float* __restrict__ UBK, float* __restrict__ thrK) {
  for (int p = p_begin + blockIdx.x * blockDim.x + threadIdx.x; p < p_end; p += gridDim.x * blockDim.x) {
    float top[K];
#pragma unroll
    for (int t = 0; t < K; t++) top[t] = -INFINITY;
    constexpr int U = 16;  // loads in flight
    for (int c = 0; c < nch; c += U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; u++) v[u] = c + u < nch ? __ldcs(TM32 + (int64_t)(c + u) * ld + p) : -INFINITY;
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (v[u] > top[K - 1]) {  // branch-free insertion into the descending list
          float x = v[u];
#pragma unroll
          for (int t = 0; t < K; t++) {
            const float hi = fmaxf(top[t], x);
            x = fminf(top[t], x);
            top[t] = hi;
          }
        }
      }
    }
    const float ni = nrm[p], li = len[p];
    float ub = INFINITY, thr = -INFINITY;
    if (top[K - 1] > -INFINITY) {
      ub = em_upper(em, ni - 2.0f * top[K - 1], ni, li, maxlen);
      thr = em_thr(em, ub, ni, li, maxlen);
    }
    UBK[p] = ub;
    thrK[p] = thr;
  }
}

struct ChunkParams {
  const float* TM32;
  int64_t ld;
  int nch;
  int p_begin, p_end;
  const float* thrK;
  const float* UBK;
  const float* X;    // n x d, original order (round 0: permuted == original)
  int n, d;
  double s2;         // scale^2 (exact power of two)
  unsigned* cnt;     // per row: appended candidates
  u64* cand;         // [row][cap]
  int cap;
  unsigned* work;    // [0]: next chunk (dynamic scheduling)
};

// One CTA per chunk (dynamic scheduling), 256 threads.  The chunk's 32 columns are
// staged transposed in shared memory (colx[k][32]); the rows that list the chunk are
// queued, then evaluated 128 at a time with the rows staged transposed as well
// (rowx[k][128]): thread (ty, tx) owns a 4 x 4 micro-tile (rows 4ty.., columns 4tx..)
// and runs the pinned R1 chain with two 128-bit shared loads per 32 FP32 operations.
constexpr int CE_WIN = 2048, CE_RB = 128, CE_QCAP = CE_WIN + CE_RB;
__global__ void __launch_bounds__(256) k_chunk_exact(ChunkParams C) {
  extern __shared__ __align__(16) float sm[];
  float* colx = sm;                  // [d][32]
  float* rowx = sm + C.d * 32;       // [d][CE_RB]
  int* queue = reinterpret_cast<int*>(rowx + C.d * CE_RB);  // [CE_QCAP]
  __shared__ int qn;
  __shared__ int chunk_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  while (true) {
    if (threadIdx.x == 0) chunk_s = (int)atomicAdd(C.work, 1u);
    __syncthreads();
    const int ch = chunk_s;
    if (ch >= C.nch) break;
    const int j0 = ch * 32;
    for (int e = threadIdx.x; e < C.d * 32; e += blockDim.x) {
      const int k = e >> 5, t = e & 31;
      const int j = j0 + t;
      colx[e] = j < C.n ? C.X[(int64_t)j * C.d + k] : 0.0f;
    }
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
    // scan the chunk's column of TM32 window by window; the queue carries over windows
    // and only full batches of CE_RB rows are evaluated until the last window
    for (int pb = C.p_begin; pb < C.p_end; pb += CE_WIN) {
      const int pe = min(C.p_end, pb + CE_WIN);
      for (int o = threadIdx.x; o < CE_WIN; o += blockDim.x) {  // warp-uniform trip count (ballot)
        const int p = pb + o;
        bool want = false;
        if (p < pe) {
          const float m = __ldcs(C.TM32 + (int64_t)ch * C.ld + p);
          want = m >= C.thrK[p] && m > -INFINITY;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, want);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&qn, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (want) queue[base + __popc(bal & ((1u << lane) - 1u))] = p;
      }
      __syncthreads();
      const int nq = qn;
      const bool last = pe >= C.p_end;
      const int nproc = last ? nq : nq / CE_RB * CE_RB;
      for (int b0 = 0; b0 < nproc; b0 += CE_RB) {
        const int nb = min(CE_RB, nproc - b0);
        // stage the batch's rows transposed: lane = row of a 32-row group, float4 loads
        for (int g = warp; g < CE_RB / 32; g += blockDim.x >> 5) {
          const int r = g * 32 + lane;
          const int p = r < nb ? queue[b0 + r] : -1;
          if ((C.d & 3) == 0) {
            const float4* src = reinterpret_cast<const float4*>(C.X + (int64_t)(p < 0 ? 0 : p) * C.d);
            for (int k4 = 0; k4 < C.d / 4; k4++) {
              const float4 v = p >= 0 ? __ldg(src + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
              rowx[(4 * k4 + 0) * CE_RB + r] = v.x;
              rowx[(4 * k4 + 1) * CE_RB + r] = v.y;
              rowx[(4 * k4 + 2) * CE_RB + r] = v.z;
              rowx[(4 * k4 + 3) * CE_RB + r] = v.w;
            }
          } else {
            for (int k = 0; k < C.d; k++) rowx[k * CE_RB + r] = p >= 0 ? __ldg(C.X + (int64_t)p * C.d + k) : 0.0f;
          }
        }
        __syncthreads();
        float acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++) acc[a][b] = 0.0f;
#pragma unroll 4
        for (int k = 0; k < C.d; k++) {
          const float4 xa = *reinterpret_cast<const float4*>(rowx + k * CE_RB + 4 * ty);
          const float4 xb = *reinterpret_cast<const float4*>(colx + k * 32 + 4 * tx);
          const float av[4] = {xa.x, xa.y, xa.z, xa.w};
          const float bv[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) {
              const float t = __fsub_rn(av[a], bv[b]);
              acc[a][b] = __fmaf_rn(t, t, acc[a][b]);
            }
        }
        // R1 ends with sqrtf; the MST runs on d^2 (monotone, App. A.4)
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const int r = 4 * ty + a;
          if (r >= nb) continue;
          const int p = queue[b0 + r];
          const double ubk = (double)C.UBK[p];
#pragma unroll
          for (int b = 0; b < 4; b++) {
            const int j = j0 + 4 * tx + b;
            if (j < C.n && j != p && (double)acc[a][b] * C.s2 <= ubk) {
              const unsigned slot = atomicAdd(C.cnt + p, 1u);
              if ((int)slot < C.cap)
                C.cand[(int64_t)p * C.cap + slot] =
                    ((u64)(__float_as_uint(acc[a][b]) & 0x7FFFFFFFu) << 33) | tri_index(p, j);
            }
          }
        }
        __syncthreads();
      }
      // keep the remainder (< CE_RB rows) at the front of the queue
      const int rem = nq - nproc;
      int carry = 0;
      if (threadIdx.x < rem) carry = queue[nproc + threadIdx.x];
      __syncthreads();
      if (threadIdx.x < rem) queue[threadIdx.x] = carry;
      if (threadIdx.x == 0) {
        if (nproc) atomicAdd(C.work + 1, (unsigned)nproc);  // statistics: listed (row, chunk)
        qn = rem;
      }
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
  for (int p = p_begin + blockIdx.x * warps + w; p < p_end; p += gridDim.x * warps) {
    const unsigned c = cnt[p];
    if ((int)c > cap || c == 0) {
      if (lane == 0) {
        ccnt[p] = -1;
        fallback[atomicAdd(nfallback, 1u)] = p;
      }
      continue;
    }
    u64 mine[4];  // cap <= 128
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int e = lane + 32 * u;
      mine[u] = e < (int)c ? cand[(int64_t)p * cap + e] : KEY_NONE;
    }
    const int take = min((int)c, K);
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
          atomicMin(compbest + ci, ckey[(int64_t)i * K + t]);
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
__global__ void k_comp_ub_seed(int k, const u64* __restrict__ compbest, double s2, unsigned* __restrict__ compUB) {
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
// and rows whose cache overflowed.  Work item = 8 listed rows x 1024 columns; each
// thread holds 4 columns, every column value loaded once serves the 8 rows (rows in
// shared memory).  XT: d x ldx original-order transpose (zero padded to ldx).
// comp == nullptr: singletons (eligible = j != i).
// ---------------------------------------------------------------------------
constexpr int RE_R = 8, RE_COLS = 1024;
__global__ void __launch_bounds__(256) k_rows_exact(const float* __restrict__ XT, int64_t ldx, int n, int d,
                                                   const int* __restrict__ rows, const unsigned* __restrict__ nrows,
                                                   const int* __restrict__ comp, u64* __restrict__ compbest) {
  extern __shared__ float xr[];  // [d][RE_R]
  __shared__ u64 red[8][RE_R];
  const int nr = (int)*nrows;
  const int ngroups = (nr + RE_R - 1) / RE_R;
  const int nblk = (n + RE_COLS - 1) / RE_COLS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int item = blockIdx.x; item < ngroups * nblk; item += gridDim.x) {
    const int g = item / nblk, blk = item % nblk;
    int ri[RE_R], ci[RE_R];
#pragma unroll
    for (int r = 0; r < RE_R; r++) {
      const int idx = g * RE_R + r;
      ri[r] = idx < nr ? rows[idx] : -1;
      ci[r] = ri[r] >= 0 ? (comp ? comp[ri[r]] : ri[r]) : -1;
    }
    __syncthreads();  // previous item's readers of xr / red are done
    for (int e = threadIdx.x; e < d * RE_R; e += blockDim.x) {
      const int k = e / RE_R, r = e % RE_R;
      xr[e] = ri[r] >= 0 ? XT[(int64_t)k * ldx + ri[r]] : 0.0f;
    }
    __syncthreads();
    float acc[RE_R][4];
#pragma unroll
    for (int r = 0; r < RE_R; r++)
#pragma unroll
      for (int u = 0; u < 4; u++) acc[r][u] = 0.0f;
    const int jb = blk * RE_COLS + threadIdx.x;
    for (int k = 0; k < d; k++) {
      float y[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int j = jb + u * 256;
        y[u] = j < n ? __ldg(XT + (int64_t)k * ldx + j) : 0.0f;
      }
      const float4 xa = *reinterpret_cast<const float4*>(xr + k * RE_R);
      const float4 xb = *reinterpret_cast<const float4*>(xr + k * RE_R + 4);
      const float xv[RE_R] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int r = 0; r < RE_R; r++)
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const float t = __fsub_rn(xv[r], y[u]);
          acc[r][u] = __fmaf_rn(t, t, acc[r][u]);
        }
    }
#pragma unroll
    for (int r = 0; r < RE_R; r++) {
      u64 best = KEY_NONE;
      if (ri[r] >= 0) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int j = jb + u * 256;
          if (j < n && (comp ? __ldg(comp + j) != ci[r] : j != ri[r])) {
            const u64 key = ((u64)(__float_as_uint(acc[r][u]) & 0x7FFFFFFFu) << 33) | tri_index(ri[r], j);
            best = key < best ? key : best;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
      }
      if (lane == 0) red[warp][r] = best;
    }
    __syncthreads();
    if (threadIdx.x < RE_R && ri[threadIdx.x] >= 0) {
      u64 best = KEY_NONE;
      for (int w = 0; w < 8; w++) best = red[w][threadIdx.x] < best ? red[w][threadIdx.x] : best;
      if (best != KEY_NONE) atomicMin(compbest + ci[threadIdx.x], best);
    }
  }
}

appd_status launch_rows_exact(appd_ctx* c, const float* XT, int64_t ldx, int n, int d, const int* rows,
                              const unsigned* nrows, int max_rows, const int* comp, u64* compbest) {
  if (max_rows <= 0) return APPD_OK;
  const int64_t items = (int64_t)((max_rows + RE_R - 1) / RE_R) * ((n + RE_COLS - 1) / RE_COLS);
  const int grid = (int)std::min<int64_t>(items, (int64_t)c->sm_count * 8);
  const size_t smem = (size_t)d * RE_R * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_rows_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_rows_exact<<<grid, 256, smem, c->stream>>>(XT, ldx, n, d, rows, nrows, comp, compbest);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
appd_status launch_topk_thr(appd_ctx* c, int K, const float* TM32, int64_t ld, int nch, int p_begin, int p_end,
                            const float* nrm, const float* len, float maxlen, const ErrModel& em, float* UBK,
                            float* thrK) {
  const int rows = p_end - p_begin;
  if (rows <= 0) return APPD_OK;
  const int grid = std::min(c->sm_count * 8, (rows + 127) / 128);
  switch (K) {
    case 4: k_topk_thr<4><<<grid, 128, 0, c->stream>>>(TM32, ld, nch, p_begin, p_end, nrm, len, maxlen, em, UBK, thrK); break;
    case 8: k_topk_thr<8><<<grid, 128, 0, c->stream>>>(TM32, ld, nch, p_begin, p_end, nrm, len, maxlen, em, UBK, thrK); break;
    case 16: k_topk_thr<16><<<grid, 128, 0, c->stream>>>(TM32, ld, nch, p_begin, p_end, nrm, len, maxlen, em, UBK, thrK); break;
    case 32: k_topk_thr<32><<<grid, 128, 0, c->stream>>>(TM32, ld, nch, p_begin, p_end, nrm, len, maxlen, em, UBK, thrK); break;
    default: return fail(c, APPD_ERR_INVALID_ARGUMENT, "cache length K = %d (4, 8, 16 or 32)", K);
  }
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_chunk_exact(appd_ctx* c, const float* TM32, int64_t ld, int nch, int p_begin, int p_end,
                               const float* thrK, const float* UBK, const float* X, int n, int d, double s2,
                               unsigned* cnt, u64* cand, int cap, unsigned* work) {
  ChunkParams C;
  C.TM32 = TM32;
  C.ld = ld;
  C.nch = nch;
  C.p_begin = p_begin;
  C.p_end = p_end;
  C.thrK = thrK;
  C.UBK = UBK;
  C.X = X;
  C.n = n;
  C.d = d;
  C.s2 = s2;
  C.cnt = cnt;
  C.cand = cand;
  C.cap = cap;
  C.work = work;
  const size_t smem = (size_t)d * (32 + CE_RB) * 4 + CE_QCAP * 4;
  if (smem > 227 * 1024) return APPD_ERR_UNSUPPORTED;
  cudaFuncSetAttribute(k_chunk_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = std::min(nch, c->sm_count * 4);
  k_chunk_exact<<<grid, 256, smem, c->stream>>>(C);
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

appd_status launch_comp_ub(appd_ctx* c, int n, int k, const u64* compbest, double s2, const int* perm,
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
// the eligible maximum of G' over each 128-column segment.
//   k_cm_rowub   CUB[C][D] = min over rows p of C of the upper bound of s^2 r from the
//                segments lying entirely inside D (an exact pair exists below it);
//   k_cm_filter  lists (p, seg) whenever a pair (p, j), j in seg and in D != C, can
//                have L <= CUB[C][D];
//   k_cm_exact   exact R1 keys of the listed segments, minimum per (C, D) by atomicMin.
// Every pair of C x D with L <= CUB[C][D] is evaluated exactly, so WCM[C][D] is the
// exact minimum key between C and D; the MST of the contracted graph (host Prim on
// k <= 128 nodes) plus the edges of the earlier rounds is the MST.
// ===========================================================================

__global__ void k_cm_rowub(CmParams P) {
  const int lane = threadIdx.x & 31;
  for (int p0 = P.p_begin + (blockIdx.x * blockDim.x + threadIdx.x) - lane; p0 < P.p_end;
       p0 += gridDim.x * blockDim.x) {
    const int p = p0 + lane;
    const bool valid = p < P.p_end;
    const int C = valid ? P.sc[p] : -1;
    const bool uni = __all_sync(0xffffffffu, C == __shfl_sync(0xffffffffu, C, 0));
    const float ni = valid ? P.nrm[p] : 0.0f, li = valid ? P.len[p] : 0.0f;
    for (int D = 0; D < P.k; D++) {
      const int s0 = (P.cstart[D] + 127) / 128, s1 = P.cend[D] / 128;  // segments inside D
      float m = -INFINITY;
      if (valid && D != C)
        for (int s = s0; s < s1; s++) m = fmaxf(m, __ldcs(P.TM + (int64_t)s * P.ld + p));
      float ub = m > -INFINITY ? em_upper(P.em, ni - 2.0f * m, ni, li, P.maxlen) : INFINITY;
      if (uni) {
#pragma unroll
        for (int o = 16; o; o >>= 1) ub = fminf(ub, __shfl_xor_sync(0xffffffffu, ub, o));
        if (lane == 0 && C >= 0 && ub < INFINITY) atomicMin(P.CUB + (int64_t)C * P.k + D, __float_as_uint(fmaxf(ub, 0.0f)));
      } else if (valid && ub < INFINITY) {
        atomicMin(P.CUB + (int64_t)C * P.k + D, __float_as_uint(fmaxf(ub, 0.0f)));
      }
    }
  }
}

// one warp per 32 consecutive rows; 8 segments' loads in flight.  CUB here holds the
// listing thresholds T[C][D] (the host's path-pruned upper bounds, scaled units).
__global__ void k_cm_filter(CmParams P) {
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int nseg = min(P.nseg, (P.n + 127) / 128);
  for (int p0 = P.p_begin + (blockIdx.x * warps + w) * 32; p0 < P.p_end; p0 += gridDim.x * warps * 32) {
    const int p = p0 + lane;
    const bool valid = p < P.p_end;
    const int C = valid ? P.sc[p] : 0;
    const float ni = valid ? P.nrm[p] : 0.0f, li = valid ? P.len[p] : 0.0f;
    int cachedD = -1;  // threshold of the last uniform segment's component (segments are sorted)
    float cachedT = 0.0f;
    constexpr int U = 8;
    for (int s0 = 0; s0 < nseg; s0 += U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; u++)
        v[u] = (valid && s0 + u < nseg) ? __ldcs(P.TM + (int64_t)(s0 + u) * P.ld + p) : -INFINITY;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int s = s0 + u;
        bool want = false;
        if (v[u] > -INFINITY) {
          const int q0 = s * 128;
          const int D0 = __ldg(P.sc + q0), D1 = __ldg(P.sc + min(q0 + 127, P.n - 1));
          float thr;
          if (D0 == D1) {
            if (D0 != cachedD) {
              cachedD = D0;
              cachedT = em_thr(P.em, __uint_as_float(P.CUB[(int64_t)C * P.k + D0]), ni, li, P.maxlen);
            }
            thr = cachedT;
          } else {  // straddling segment: the most permissive of its components
            float ub = 0.0f;
            for (int D = D0; D <= D1; D++)
              if (D != C) ub = fmaxf(ub, __uint_as_float(P.CUB[(int64_t)C * P.k + D]));
            thr = em_thr(P.em, ub, ni, li, P.maxlen);
          }
          want = v[u] >= thr;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, want);
        if (bal) {
          unsigned base = 0;
          const int leader = __ffs(bal) - 1;
          if (lane == leader) base = atomicAdd(P.counters + 1, (unsigned)__popc(bal));
          base = __shfl_sync(0xffffffffu, base, leader);
          if (want) {
            const unsigned slot = base + __popc(bal & ((1u << lane) - 1u));
            if (slot < P.list_cap) P.list[slot] = make_uint2((unsigned)p, (unsigned)s);
          }
        }
      }
    }
  }
}

__global__ void k_cm_exact(CmParams P) {
  unsigned cnt = P.counters[1];
  if (cnt > P.list_cap) cnt = P.list_cap;
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (unsigned a = blockIdx.x * warps + w; a < cnt; a += gridDim.x * warps) {
    const uint2 pt = P.list[a];
    const int p = (int)pt.x, s = (int)pt.y;
    const int C = P.sc[p];
    const int oi = P.perm[p];
    const float* xi = P.XTp + p;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const int q0 = s * 128 + lane;
    for (int kk = 0; kk < P.d; kk++) {
      const float x = __ldg(xi + (int64_t)kk * P.ld);
      const float* row = P.XTp + (int64_t)kk * P.ld + q0;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const float t = __fsub_rn(x, __ldg(row + u * 32));
        acc[u] = __fmaf_rn(t, t, acc[u]);
      }
    }
    u64 key[4];
    int Dq[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int q = q0 + u * 32;
      Dq[u] = q < P.n ? P.sc[q] : -1;
      key[u] = (Dq[u] >= 0 && Dq[u] != C)
                   ? (((u64)(__float_as_uint(acc[u]) & 0x7FFFFFFFu) << 33) | tri_index(oi, P.perm[q]))
                   : KEY_NONE;
    }
    // per component of the segment (labels are contiguous in a sorted segment)
    const int D0 = P.sc[s * 128], D1 = P.sc[min(s * 128 + 127, P.n - 1)];
    for (int D = D0; D <= D1; D++) {
      if (D == C) continue;
      u64 m = KEY_NONE;
#pragma unroll
      for (int u = 0; u < 4; u++) m = (Dq[u] == D && key[u] < m) ? key[u] : m;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, m, o);
        m = other < m ? other : m;
      }
      if (lane == 0 && m != KEY_NONE) atomicMin(P.WCM + (int64_t)C * P.k + D, m);
    }
  }
  if (lane == 0 && blockIdx.x == 0 && w == 0) atomicAdd(P.counters + 2, cnt);
}

appd_status launch_cm_rowub(appd_ctx* c, const CmParams& P) {
  const int rows = P.p_end - P.p_begin;
  if (rows <= 0) return APPD_OK;
  k_cm_rowub<<<std::min(c->sm_count * 8, (rows + 255) / 256), 256, 0, c->stream>>>(P);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

appd_status launch_cm_exact(appd_ctx* c, const CmParams& P) {
  const int rows = P.p_end - P.p_begin;
  if (rows <= 0) return APPD_OK;
  k_cm_filter<<<std::min(c->sm_count * 8, (rows + 255) / 256), 256, 0, c->stream>>>(P);
  APPD_LAUNCHED(c);
  k_cm_exact<<<c->sm_count * 16, 256, 0, c->stream>>>(P);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
