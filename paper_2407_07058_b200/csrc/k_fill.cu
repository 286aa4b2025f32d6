// k_fill.cu -- the APPD fill.
//
// Algorithm 4 writes, for each removed MST edge, its weight into every cell of
// tree1 x tree2, each cell exactly once.  Equivalently (DESIGN.md
// "leaf order"), with a leaf order pi of the single-linkage dendrogram and
// h[a] = M[pi_a][pi_{a+1}]:   M[pi_a][pi_b] = max(h[min(a,b) .. max(a,b)-1]).
//
// The fill processes a tile of rows that are consecutive in leaf order
// (positions a_0 < ... < a_{R-1}) against a block of columns in ORIGINAL order
// (so every store is a coalesced 128-bit row segment).  For a column j at
// position b:
//   b >  a_{R-1}:  M[row t][j] = max( S[t], RMQ(a_{R-1}, b) ),  S[t] = RMQ(a_t, a_{R-1})
//   b <  a_0:      M[row t][j] = max( P[t], RMQ(b, a_0) ),      P[t] = RMQ(a_0, a_t)
//   otherwise:     M = RMQ(min(a_t,b), max(a_t,b)), 0 on the diagonal (b == a_t)
// so the inner loop is one select + one max per element: the kernel is bound by
// HBM write bandwidth (n^2 * 4 bytes).  RMQ is a sparse table over h
// (ST[k][i] = max h[i .. i+2^k-1]).  Widest sense: min instead of max.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "internal.cuh"

namespace appd {
namespace cg = cooperative_groups;

__global__ void k_positions(const int* __restrict__ pi, int64_t n, int* __restrict__ pos) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    pos[pi[a]] = (int)a;
}
appd_status launch_positions(appd_ctx* c, const int* pi, int64_t n, int* pos) {
  int grid = (int)((n + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  k_positions<<<grid, 256, 0, c->stream>>>(pi, n, pos);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

__global__ void k_sqrt_inplace(float* h, int64_t m) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < m; a += (int64_t)gridDim.x * blockDim.x)
    h[a] = __fsqrt_rn(h[a]);
}
appd_status launch_sqrt_inplace(appd_ctx* c, float* h, int64_t m) {
  if (m <= 0) return APPD_OK;
  int grid = (int)((m + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  k_sqrt_inplace<<<grid, 256, 0, c->stream>>>(h, m);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// level k from level k-1 (level 0 = h, already in place)
template <bool WIDEST>
__global__ void k_st_level(float* ST, int64_t m, int64_t stride, int k) {
  const int64_t half = 1ll << (k - 1);
  const float* prev = ST + (int64_t)(k - 1) * stride;
  float* cur = ST + (int64_t)k * stride;
  const int64_t cnt = m - (1ll << k) + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    float a = prev[i], b = prev[i + half];
    cur[i] = WIDEST ? fminf(a, b) : fmaxf(a, b);
  }
}
// levels 1 .. kl (kl <= ST_LO) in one pass: a block computes level-k entries
// [i0, i0 + ST_B) for every k from level 0 [i0, i0 + ST_B + 2^kl - 1) in shared memory
constexpr int ST_LO = 8, ST_B = 2048;
template <bool WIDEST>
__global__ void __launch_bounds__(256) k_st_levels_lo(float* ST, int64_t m, int64_t stride, int kl) {
  __shared__ float buf[2][ST_B + (1 << ST_LO)];
  const float ID = WIDEST ? INFINITY : -INFINITY;
  const int64_t i0 = (int64_t)blockIdx.x * ST_B;
  int need = ST_B + (1 << kl) - 1;
  for (int i = threadIdx.x; i < need; i += blockDim.x) buf[0][i] = i0 + i < m ? ST[i0 + i] : ID;
  __syncthreads();
  for (int k = 1; k <= kl; k++) {
    const int half = 1 << (k - 1);
    need -= half;
    const float* prev = buf[(k - 1) & 1];
    float* cur = buf[k & 1];
    const int64_t cnt = m - (1ll << k) + 1;
    float* out = ST + (int64_t)k * stride;
    for (int i = threadIdx.x; i < need; i += blockDim.x) {
      const float v = WIDEST ? fminf(prev[i], prev[i + half]) : fmaxf(prev[i], prev[i + half]);
      cur[i] = v;
      if (i < ST_B && i0 + i < cnt) out[i0 + i] = v;
    }
    __syncthreads();
  }
}

// levels k0 .. levels-1 in one cooperative launch (a grid-wide barrier between levels)
template <bool WIDEST>
__global__ void __launch_bounds__(1024) k_st_levels_hi(float* ST, int64_t m, int64_t stride, int k0, int levels,
                                                       unsigned* bar) {
  for (int k = k0; k < levels; k++) {
    const int64_t half = 1ll << (k - 1);
    const float* prev = ST + (int64_t)(k - 1) * stride;
    float* cur = ST + (int64_t)k * stride;
    const int64_t cnt = m - (1ll << k) + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
      cur[i] = WIDEST ? fminf(prev[i], prev[i + half]) : fmaxf(prev[i], prev[i + half]);
    coop_grid_sync(bar);
  }
}

appd_status launch_sparse_table(appd_ctx* c, float* ST, int64_t m, int levels, int64_t stride, int widest) {
  const int kl = std::min(ST_LO, levels - 1);
  if (kl >= 1) {
    const int grid = (int)((m + ST_B - 1) / ST_B);
    if (widest) k_st_levels_lo<true><<<grid, 256, 0, c->stream>>>(ST, m, stride, kl);
    else k_st_levels_lo<false><<<grid, 256, 0, c->stream>>>(ST, m, stride, kl);
    APPD_LAUNCHED(c);
  }
  if (kl + 1 < levels) {  // the remaining levels: one cooperative launch
    int k0 = kl + 1, lv = levels;
    int64_t mm = m, st = stride;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, (m + 1023) / 1024));
    unsigned* bar = grid_barrier_word(c);
    if (!bar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
    void* args[] = {&ST, &mm, &st, &k0, &lv, &bar};
    const cudaError_t e = cudaLaunchCooperativeKernel(widest ? (const void*)k_st_levels_hi<true>
                                                              : (const void*)k_st_levels_hi<false>,
                                                       grid, 1024, args, 0, c->stream);
    if (e == cudaSuccess) {
      c->launches++;
      return APPD_OK;
    }
    cudaGetLastError();  // not co-schedulable: one launch per level
  }
  for (int k = kl + 1; k < levels; k++) {
    int64_t cnt = m - (1ll << k) + 1;
    int grid = (int)((cnt + 255) / 256);
    if (grid > c->sm_count * 8) grid = c->sm_count * 8;
    if (grid < 1) grid = 1;
    if (widest) k_st_level<true><<<grid, 256, 0, c->stream>>>(ST, m, stride, k);
    else k_st_level<false><<<grid, 256, 0, c->stream>>>(ST, m, stride, k);
    APPD_LAUNCHED(c);
  }
  return APPD_OK;
}

template <bool WIDEST>
__device__ __forceinline__ float comb(float a, float b) {
  return WIDEST ? fminf(a, b) : fmaxf(a, b);
}

// RMQ over h[l .. r-1], l < r
template <bool WIDEST>
__device__ __forceinline__ float rmq(const float* __restrict__ ST, int64_t stride, int l, int r) {
  int len = r - l;
  int k = 31 - __clz(len);
  float a = __ldg(ST + (int64_t)k * stride + l);
  float b = __ldg(ST + (int64_t)k * stride + r - (1 << k));
  return comb<WIDEST>(a, b);
}

constexpr int FILL_THREADS = 256;
constexpr int FILL_R = 128;  // max rows per tile (consecutive in leaf order; <= FILL_THREADS)

// positions spanned by one tile whose in-tile range maxima come from shared memory
constexpr int FILL_SPAN = 256, FILL_LV = 8;  // spans < FILL_SPAN: levels 0 .. FILL_LV - 1

// output store flavour (STORE: 0 streaming / evict-first st.global.cs, 1 default st.global)
template <int STORE>
__device__ __forceinline__ void fill_store4(float* dst, float4 v) {
  if (STORE == 0) __stcs(reinterpret_cast<float4*>(dst), v);
  else *reinterpret_cast<float4*>(dst) = v;
}

// OT = double (NEXT-3, k_f64.cu): the values are ranks r + 1 of the fp64 MST weights and
// the store maps each through hw[r + 1] (hw[0] = +0 for the diagonal)
template <int VEC, bool WIDEST, int STORE = 0, int RT = FILL_R, typename OT = float>
__global__ void __launch_bounds__(FILL_THREADS)
    k_fill(const int* __restrict__ rows_sorted, const int* __restrict__ rowpos, int64_t nrows,
           const int* __restrict__ pos, const float* __restrict__ ST, int64_t stride, int64_t n,
           OT* __restrict__ M, int64_t row0, const double* __restrict__ hw = nullptr) {
  __shared__ float2 sSP[FILL_R];   // (S, P) of each row: one 8-byte broadcast load per row
  __shared__ OT* sPtr[FILL_R];     // the row's first element in M
  constexpr bool F64 = sizeof(OT) == 8;
  __shared__ double2 sSPd[F64 ? FILL_R : 1];  // fp64: the weights of S and P
  __shared__ int sA[FILL_R];
  // sparse table of h over the tile's position range [aL, aR): columns whose position
  // lies inside it (the tile's own points, and other ranks' in between) need a direct
  // range maximum per element; from shared memory when the span fits
  __shared__ float sST[FILL_LV][FILL_SPAN];
  const float ID = WIDEST ? INFINITY : -INFINITY;
  const int64_t t0 = (int64_t)blockIdx.y * RT;
  int R = (int)((nrows - t0) < RT ? (nrows - t0) : RT);
  const int aL = rowpos[t0], aR = rowpos[t0 + R - 1];
  if (threadIdx.x < R) {
    int t = threadIdx.x;
    int at = rowpos[t0 + t];
    sA[t] = at;
    sPtr[t] = M + ((int64_t)rows_sorted[t0 + t] - row0) * n;
    sSP[t] = make_float2((at < aR) ? rmq<WIDEST>(ST, stride, at, aR) : ID, (at > aL) ? rmq<WIDEST>(ST, stride, aL, at) : ID);
    if constexpr (F64) sSPd[t] = make_double2(__ldg(hw + (int)fmaxf(sSP[t].x, 0.0f)), __ldg(hw + (int)fmaxf(sSP[t].y, 0.0f)));
  }
  // this thread's VEC columns
  const int64_t jbase = (int64_t)blockIdx.x * (FILL_THREADS * VEC) + (int64_t)threadIdx.x * VEC;
  int b[VEC];
  float base[VEC];
  int side[VEC];  // 0 right (use S), 1 left (use P), 2 inside
  bool any_inside = false;
#pragma unroll
  for (int q = 0; q < VEC; q++) {
    int64_t j = jbase + q;
    int bb = (j < n) ? __ldg(pos + j) : aL;
    b[q] = bb;
    if (bb > aR) { side[q] = 0; base[q] = rmq<WIDEST>(ST, stride, aR, bb); }
    else if (bb < aL) { side[q] = 1; base[q] = rmq<WIDEST>(ST, stride, bb, aL); }
    else { side[q] = 2; base[q] = ID; any_inside = true; }
  }
  const bool warp_inside = __any_sync(0xffffffffu, any_inside);
  // fp64: each value is S, P or base (or an inside range maximum): the rank comparison
  // picks which, so only the per-column weights are looked up, once
  double based[F64 ? VEC : 1];
  if constexpr (F64) {
#pragma unroll
    for (int q = 0; q < VEC; q++) based[q] = side[q] == 2 ? 0.0 : __ldg(hw + (int)fmaxf(base[q], 0.0f));
  }
  // predicate-free selection per row: v = comb(comb'(S, cS), comb'(P, cP), base) with
  // cS = +-inf (pass S / block it) by side, so no per-column predicates stay live
  const float PASS = WIDEST ? -INFINITY : INFINITY;  // comb'(x, PASS) = x
  float cS[VEC], cP[VEC];
#pragma unroll
  for (int q = 0; q < VEC; q++) {
    cS[q] = side[q] == 0 ? PASS : ID;
    cP[q] = side[q] == 1 ? PASS : ID;
  }
  const bool in_range = jbase < n;
  const int span = aR - aL;  // h[aL .. aR-1]
  const bool local = span < FILL_SPAN;  // levels k <= log2(span) < FILL_LV
  if (local) {  // the global table's levels over [aL, aR): independent loads, one barrier
    for (int k = 0; (1 << k) <= span; k++)
      for (int i = threadIdx.x; i + (1 << k) <= span; i += FILL_THREADS)
        sST[k][i] = __ldg(ST + (int64_t)k * stride + aL + i);
  }
  __syncthreads();
#pragma unroll 4
  for (int t = 0; t < R; t++) {
    const float2 SP = sSP[t];
    const float S = SP.x, P = SP.y;
    float v[VEC];
#pragma unroll
    for (int q = 0; q < VEC; q++) {
      // minimax: max(min(S, cS), min(P, cP), base); widest: min(max(S, cS), max(P, cP), base)
      const float xs = WIDEST ? fmaxf(S, cS[q]) : fminf(S, cS[q]);
      const float xp = WIDEST ? fmaxf(P, cP[q]) : fminf(P, cP[q]);
      v[q] = comb<WIDEST>(comb<WIDEST>(xs, xp), base[q]);
    }
    if (warp_inside) {
      const int at = sA[t];
#pragma unroll
      for (int q = 0; q < VEC; q++) {
        if (side[q] == 2) {
          const int bb = b[q];
          const int l = min(bb, at), r = max(bb, at);
          if (bb == at) {
            v[q] = 0.0f;
          } else if (local) {  // RMQ(l, r) from the tile's shared-memory table
            const int k = 31 - __clz(r - l);
            v[q] = comb<WIDEST>(sST[k][l - aL], sST[k][r - aL - (1 << k)]);
          } else {
            v[q] = rmq<WIDEST>(ST, stride, l, r);
          }
        }
      }
    }
    OT* dst = sPtr[t] + jbase;
    if constexpr (sizeof(OT) == 8) {
      double o[VEC];
      const double2 SPd = sSPd[t];
#pragma unroll
      for (int q = 0; q < VEC; q++) {
        if (side[q] == 2) o[q] = __ldg(hw + (int)fmaxf(v[q], 0.0f));
        else o[q] = v[q] == base[q] ? based[q] : (side[q] == 0 ? SPd.x : SPd.y);
      }
      if (VEC % 4 == 0 && in_range && jbase + VEC <= n) {  // whole 32-byte sectors per store (st.global.cs.v4.f64)
#pragma unroll
        for (int q = 0; q < VEC; q += 4)
          asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + q), "d"(o[q]), "d"(o[q + 1]),
                       "d"(o[q + 2]), "d"(o[q + 3])
                       : "memory");
      } else {
#pragma unroll
        for (int q = 0; q < VEC; q++)
          if (jbase + q < n) __stcs(reinterpret_cast<double*>(dst) + q, o[q]);
      }
    } else if (VEC == 8) {  // one 32-byte store (st.global[.cs].v8.f32, sm_100)
      if (in_range) {
        if (STORE == 0)
          asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(v[0]), "f"(v[1]),
                       "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                       : "memory");
        else
          asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(v[0]), "f"(v[1]),
                       "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                       : "memory");
      }
    } else if (VEC == 4) {
      if (in_range) fill_store4<STORE>(reinterpret_cast<float*>(dst), make_float4(v[0], v[1], v[2], v[3]));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; q++)
        if (jbase + q < n) __stcs(reinterpret_cast<float*>(dst) + q, v[q]);
    }
  }
}

// NEXT-3: fp64 output of rank-valued h (minimax sense on ranks, see k_f64.cu)
appd_status launch_fill_f64(appd_ctx* c, const int* rows_sorted, const int* rowpos, int64_t nrows, const int* pos,
                            const float* ST, int64_t stride, int64_t n, double* M, int64_t row0, const double* hw) {
  if (nrows <= 0) return APPD_OK;
  const bool even = (n % 4) == 0 && ((uintptr_t)M % 32) == 0;
  if (even) {
    // 64-row tiles (measured at n = 16384: 0.50 ms against 0.55 ms with 128-row tiles)
    dim3 g((unsigned)((n + FILL_THREADS * 8 - 1) / (FILL_THREADS * 8)), (unsigned)((nrows + 63) / 64));
    k_fill<8, false, 0, 64, double><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n,
                                                                       M, row0, hw);
  } else {
    dim3 g((unsigned)((n + FILL_THREADS - 1) / FILL_THREADS), (unsigned)((nrows + 63) / 64));
    k_fill<1, false, 0, 64, double><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n,
                                                                       M, row0, hw);
  }
  APPD_LAUNCHED(c);
  c->stats.fill_launches++;
  return APPD_OK;
}

template <int VEC, bool WIDEST>
static void fill_rt(appd_ctx* c, int rt, dim3 g, const int* rows_sorted, const int* rowpos, int64_t nrows,
                    const int* pos, const float* ST, int64_t stride, int64_t n, float* M, int64_t row0) {
  switch (rt) {
    case 128: k_fill<VEC, WIDEST, 0, 128><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0); break;
    case 64: k_fill<VEC, WIDEST, 0, 64><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0); break;
    case 32: k_fill<VEC, WIDEST, 0, 32><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0); break;
    case 16: k_fill<VEC, WIDEST, 0, 16><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0); break;
    default: k_fill<VEC, WIDEST, 0, 8><<<g, FILL_THREADS, 0, c->stream>>>(rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0); break;
  }
}

// Tile shape: VEC consecutive columns per thread (32-byte stores when n allows and every
// thread still has columns), RT rows per tile.  Large outputs: 128-row tiles; smaller ones
// shrink the tile (64, then down to 8 rows) until there are at least two waves of the 4
// resident CTAs per SM -- a small fill is latency-bound, so it needs CTAs, not long tiles
// (C1, n = 256: 60 us with four 64-row tiles of 32 busy threads each).
appd_status launch_fill(appd_ctx* c, const int* rows_sorted, const int* rowpos, int64_t nrows, const int* pos,
                        const float* ST, int64_t stride, int64_t n, float* M, int64_t row0, int widest) {
  if (nrows <= 0) return APPD_OK;
  const bool vec8 = (n % 8) == 0 && ((uintptr_t)M % 32) == 0;
  const bool vec4 = (n % 4) == 0 && ((uintptr_t)M % 16) == 0;
  // 32-byte stores by default (measured: fewer instructions per byte); APPD_FILL_VEC=4 picks 16-byte
  static const int want = dev_env("APPD_FILL_VEC") ? atoi(dev_env("APPD_FILL_VEC")) : 8;
  const int vec = (vec8 && want == 8 && n >= FILL_THREADS * 8) ? 8 : (vec4 && n >= FILL_THREADS * 4) ? 4 : 1;
  const int64_t gx = (n + FILL_THREADS * vec - 1) / (FILL_THREADS * vec);
  auto ctas = [&](int rt) { return gx * ((nrows + rt - 1) / rt); };
  const int64_t waves = (int64_t)c->sm_count * 4;
  int rt = 128;
  if (ctas(128) < 6 * waves) {
    rt = 64;
    while (rt > 8 && ctas(rt) < 2 * waves) rt /= 2;
  }
  const dim3 g((unsigned)gx, (unsigned)((nrows + rt - 1) / rt));
  if ((nrows + rt - 1) / rt > 65535) return fail(c, APPD_ERR_UNSUPPORTED, "fill grid too large");
  if (vec == 8) widest ? fill_rt<8, true>(c, rt, g, rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0)
                       : fill_rt<8, false>(c, rt, g, rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0);
  else if (vec == 4) widest ? fill_rt<4, true>(c, rt, g, rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0)
                            : fill_rt<4, false>(c, rt, g, rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0);
  else widest ? fill_rt<1, true>(c, rt, g, rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0)
              : fill_rt<1, false>(c, rt, g, rows_sorted, rowpos, nrows, pos, ST, stride, n, M, row0);
  APPD_LAUNCHED(c);
  c->stats.fill_launches++;
  return APPD_OK;
}

// rows [row0, row0+rows) of this rank: keys = positions, vals = row ids (sorted later)
__global__ void k_gather_rowpos(const int* __restrict__ pos, int64_t row0, int64_t rows, int* keys, int* vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    keys[r] = pos[row0 + r];
    vals[r] = (int)(row0 + r);
  }
}
appd_status launch_gather_rowpos(appd_ctx* c, const int* pos, int64_t row0, int64_t rows, int* keys, int* vals) {
  int grid = (int)((rows + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  if (grid < 1) grid = 1;
  k_gather_rowpos<<<grid, 256, 0, c->stream>>>(pos, row0, rows, keys, vals);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

__global__ void k_zero1(float* M) { M[0] = 0.0f; }
appd_status launch_set_diag_zero_single(appd_ctx* c, float* M) {
  k_zero1<<<1, 1, 0, c->stream>>>(M);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// K11 test hook: R1 weights of a row block, the same pinned chain as the MST scan
__global__ void k_points_weights(const float* __restrict__ X, int64_t n, int64_t d, int64_t row0, int64_t rows,
                                 float* __restrict__ Wb, int metric) {
  int64_t total = rows * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / n, j = e % n, i = row0 + r;
    float acc = 0.0f;
    for (int64_t k = 0; k < d; k++) {
      float t = __fsub_rn(X[i * d + k], X[j * d + k]);
      if (metric == 1) acc = __fadd_rn(acc, fabsf(t));      // Manhattan (NEXT-3)
      else if (metric == 2) acc = fmaxf(acc, fabsf(t));     // Chebyshev
      else acc = __fmaf_rn(t, t, acc);                      // R1
    }
    Wb[e] = (i == j) ? 0.0f : (metric == 0 ? __fsqrt_rn(acc) : acc);
  }
}
appd_status launch_points_weights(appd_ctx* c, const float* X, int64_t n, int64_t d, int64_t row0, int64_t rows,
                                  float* Wb) {
  int64_t total = rows * n;
  int grid = (int)((total + 255) / 256);
  if (grid > c->sm_count * 16) grid = c->sm_count * 16;
  if (grid < 1) grid = 1;
  k_points_weights<<<grid, 256, 0, c->stream>>>(X, n, d, row0, rows, Wb, c->opt.metric);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd

namespace appd {

// sorted MST edge keys -> endpoints and weights (the dendrogram's input)
__global__ void k_decode_edges(const u64* __restrict__ keys, int64_t m, int shift, int points, int sense, int metric,
                               int32_t* __restrict__ eu, int32_t* __restrict__ ev, float* __restrict__ ew) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const u64 key = keys[e];
    int64_t u, v;
    tri_decode(key & ((1ull << shift) - 1), &u, &v);
    const uint32_t wk = (uint32_t)(key >> shift);
    float w;
    if (points) {
      // R1: the weight is sqrtf of the squared distance; L1 / L-inf keys hold the distance
      const uint32_t b = sense > 0 ? wk : (~wk & 0x7FFFFFFFu);  // widest: the order-reversed bits
      w = metric == 0 ? __fsqrt_rn(__uint_as_float(b)) : __uint_as_float(b);
    } else {
      const float mm = from_orderable(wk);
      w = (sense > 0 ? mm : -mm) + 0.0f;
    }
    eu[e] = (int32_t)u;
    ev[e] = (int32_t)v;
    ew[e] = w;
  }
}

appd_status launch_decode_edges(appd_ctx* c, const u64* keys, int64_t m, const KeySpec& ks, int32_t* eu,
                                int32_t* ev, float* ew) {
  if (m <= 0) return APPD_OK;
  int grid = (int)((m + 255) / 256);
  if (grid > c->sm_count * 8) grid = c->sm_count * 8;
  k_decode_edges<<<grid, 256, 0, c->stream>>>(keys, m, ks.shift, ks.points ? 1 : 0, ks.sense, ks.metric, eu, ev, ew);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
