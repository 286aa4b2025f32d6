// k_tcfilter.cu -- points-mode Boruvka rounds on the 5th-gen tensor cores
// (SURVEY §8(a) row a2', "tensor cores for the -2 X^T X term of points-mode
// distance tiles").
//
// Each round needs, for every row i, its lightest edge to another component
// under the exact R1 weights.  Computing R1 for all n^2 pairs costs 2d FP32
// lane-ops per pair; instead the tensor cores (k_tcscan.cu) compute, in fp16 with
// fp32 accumulation,  G'_ij = y^_i . y^_j - |y^_j|^2 / 2  for centred, power-of-2
// scaled, fp16-rounded points y^ (the norm rides in two extra K columns), so
//     Dt_ij = |y^_i|^2 - 2 G'_ij  ~  s^2 |x_i - x_j|^2.
// A rigorous error model (tc_common.cuh) turns Dt into an upper bound
// U_ij and a lower bound L_ij of s^2 r_ij (r = the exact R1 value):
//   scan (tensor cores): UB_i = min over eligible j of U_ij; every 32-column chunk
//       whose maximum of G' meets the row's running threshold is appended;
//   exact (CUDA cores, here): each appended chunk that still meets the FINAL
//       threshold (L <= UB_i possible) is re-evaluated with the exact R1 chain.
//       Those chunks hold every candidate, hence the row's exact argmin and all of
//       its ties; the component minimum of the exact edge keys follows by atomicMin.
//       Rows whose appends did not fit the buffer are re-scanned exactly.
// Eligibility (j in another component) is cheap because the points are sorted by
// component every round: a row's ineligible columns form one contiguous range.
#include <algorithm>
#include <atomic>
#include <cmath>

#include <cooperative_groups.h>

#include "tc_common.cuh"

namespace appd {
namespace cg = cooperative_groups;

// per-row chunk buffer of the fused top-K scan (running threshold)

// ---------------------------------------------------------------------------
// preparation kernels
// ---------------------------------------------------------------------------

// per-block partial column sums (fp64), fixed partition => deterministic
// column sums in fp64, deterministic order: block b sums rows [b R, (b+1) R); thread
// slots (row lane l, dim k) with RL = 256 / d lanes (>= 1) sum rows l, l + RL, ..., then
// the lanes are added in order
// (256 threads; block index b)
__device__ __forceinline__ void center_partial_block(const float* __restrict__ X, int64_t n, int d, int rows_per_block,
                                                     int64_t b, double* __restrict__ part, double* red) {
  const int RL = d >= 256 ? 1 : 256 / d;
  const int64_t r0 = b * rows_per_block;
  const int64_t r1 = min(n, r0 + rows_per_block);
  for (int k0 = 0; k0 < d; k0 += 256) {  // d > 256: dims in slices of 256
    const int slot = threadIdx.x, l = slot / min(d, 256), k = k0 + slot % min(d, 256);
    double s = 0.0;
    if (l < RL && k < d)
#pragma unroll 8
      for (int64_t r = r0 + l; r < r1; r += RL) s += (double)__ldg(X + r * d + k);
    red[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < min(d, 256) && k0 + (int)threadIdx.x < d) {
      double t = 0.0;
      for (int q = 0; q < RL; q++) t += red[q * min(d, 256) + threadIdx.x];
      part[b * d + k0 + threadIdx.x] = t;
    }
    __syncthreads();
  }
}
__global__ void k_center_partial(const float* __restrict__ X, int64_t n, int d, int rows_per_block,
                                 double* __restrict__ part) {
  __shared__ double red[256];
  center_partial_block(X, n, d, rows_per_block, blockIdx.x, part, red);
}
// one warp per dimension: lanes sum partials b = lane, lane + 32, ..., then a fixed tree
__device__ __forceinline__ void center_final_dim(const double* __restrict__ part, int blocks, int64_t n, int d, int w,
                                                 int lane, float* __restrict__ c) {
  double s = 0.0;
#pragma unroll 8
  for (int b = lane; b < blocks; b += 32) s += part[(int64_t)b * d + w];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) c[w] = (float)(s / (double)n);
}
__global__ void k_center_final(const double* __restrict__ part, int blocks, int64_t n, int d, float* __restrict__ c) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w < d) center_final_dim(part, blocks, n, d, w, lane, c);
}
// max |x_i - c| (fp32; sets the scale only): one thread per point, block maximum, one atomic
// |x_i - c|^2 in fp32; bad: set to the element index of the first non-finite coordinate
// when one is found (validation folded into the cooperative preparation)
__device__ __forceinline__ float point_len2(const float* __restrict__ X, int64_t i, int d, const float* __restrict__ c,
                                            bool vec, u64* bad = nullptr) {
  float s = 0.0f;
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(X + i * d);
#pragma unroll 4
    for (int k = 0; k < d; k += 4) {
      const float4 v = __ldg(x4 + k / 4);
      if (bad && *bad == KEY_NONE) {
        if (!isfinite(v.x)) *bad = (u64)(i * d + k);
        else if (!isfinite(v.y)) *bad = (u64)(i * d + k + 1);
        else if (!isfinite(v.z)) *bad = (u64)(i * d + k + 2);
        else if (!isfinite(v.w)) *bad = (u64)(i * d + k + 3);
      }
      const float t0 = v.x - c[k], t1 = v.y - c[k + 1], t2 = v.z - c[k + 2], t3 = v.w - c[k + 3];
      s += t0 * t0 + t1 * t1 + t2 * t2 + t3 * t3;
    }
  } else {
    for (int k = 0; k < d; k++) {
      const float x = X[i * d + k];
      if (bad && *bad == KEY_NONE && !isfinite(x)) *bad = (u64)(i * d + k);
      const float t = x - c[k];
      s += t * t;
    }
  }
  return s;
}
// block maximum of best (non-negative) -> one atomicMax on the float bits of sqrt
__device__ __forceinline__ void block_max_sqrt(float best, unsigned* __restrict__ out) {
#pragma unroll
  for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  __shared__ float wb[32];
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int t = 0; t < (int)(blockDim.x >> 5); t++) m = fmaxf(m, wb[t]);
    atomicMax(out, __float_as_uint(sqrtf(m)));
  }
  __syncthreads();
}
__global__ void k_maxlen(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ c,
                         unsigned* __restrict__ out) {
  float best = 0.0f;
  const bool vec = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    best = fmaxf(best, point_len2(X, i, d, c, vec));
  block_max_sqrt(best, out);
}

// pack point perm[p] into the row (YA) and column (YB) operand granules:
// element (p, k) at granule p/128, byte offset g*(K/8)*128 + (k/8)*128 + r*16 + (k%8)*2
// with g = (p%128)/8, r = p%8 (K-major, no swizzle: 8-row x 16-byte core matrices).
// y^ = fp16(scale * (x - c)); K columns: [y^ (d), zero pad to dk, then
// A: 1, 1, 0..; B: hi(-|y^|^2/2), lo(-|y^|^2/2), 0..].  Padding points: A = 0,
// B augment = -65504 (never a maximum).  One thread per point, one 16-byte store per
// 8 coordinates (lanes = consecutive points: 128-byte runs per core matrix).
// one point (permuted position p; i = perm[p], or p without a permutation); xt != nullptr:
// also the transposed fp32 copy xt[k][p] (consecutive threads: consecutive p, coalesced);
// returns the point's error norm E_p
__device__ __forceinline__ float pack_point(const float* __restrict__ X, int64_t n, int d, int dk, int K,
                                            const int* __restrict__ perm, const float* __restrict__ c, float scale,
                                            bool vec, int64_t npad, int64_t p, __half* __restrict__ YA,
                                            __half* __restrict__ YB, float* __restrict__ nrm, float* __restrict__ len,
                                            float* __restrict__ err, float* __restrict__ xt) {
  {
    const int64_t gidx = p / 128;
    const int pl = (int)(p % 128), g = pl / 8, r = pl % 8;
    uint4* ga = reinterpret_cast<uint4*>(YA + gidx * 128 * K + (int64_t)g * (K / 8) * 64 + r * 8);
    uint4* gb = reinterpret_cast<uint4*>(YB + gidx * 128 * K + (int64_t)g * (K / 8) * 64 + r * 8);
    const bool real = p < n;
    const int64_t i = real ? (perm ? perm[p] : p) : 0;
    const float* xi = X + i * d;
    float s = 0.0f;
    // E^2 = |y^ - s (x - c)|^2: per coordinate e = (y^ - y) - s dt with y = s fl(x - c) and
    // dt = (x - c) - fl(x - c) exact by TwoSum; y^ - y is exact (Sterbenz: y^ = fp16(y)).
    // Only a - s dt and the squares / sum round (relative (d + 4) 2^-24 over the sum,
    // covered by the margin applied below); round-up FMAs keep the sum an upper bound.
    float e2 = 0.0f;
#pragma unroll 2
    for (int k8 = 0; k8 < dk; k8 += 8) {
      float xv[8];
      if (real && vec && k8 + 8 <= d) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(xi + k8));
        const float4 b = __ldg(reinterpret_cast<const float4*>(xi + k8 + 4));
        xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
        xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; u++) xv[u] = (real && k8 + u < d) ? __ldg(xi + k8 + u) : 0.0f;
      }
      if (xt)
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (k8 + u < d) xt[(int64_t)(k8 + u) * npad + p] = xv[u];
      __half hv[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int k = k8 + u;
        hv[u] = __float2half_rn(0.0f);
        if (real && k < d) {
          const float xk = xv[u], ck = c[k];
          const float t = __fsub_rn(xk, ck);
          const float bb = __fsub_rn(t, xk);
          const float dt = __fadd_rn(__fsub_rn(xk, __fsub_rn(t, bb)), __fsub_rn(-ck, bb));  // TwoSum error
          const float y = scale * t;
          hv[u] = __float2half_rn(y);
          const float ek = __fsub_rn(__fsub_rn(__half2float(hv[u]), y), scale * dt);
          e2 = __fmaf_ru(ek, ek, e2);
        }
        const float hf = __half2float(hv[u]);
        s = fmaf(hf, hf, s);
      }
      uint4 pk;
      pk.x = (uint32_t)__half_as_ushort(hv[0]) | ((uint32_t)__half_as_ushort(hv[1]) << 16);
      pk.y = (uint32_t)__half_as_ushort(hv[2]) | ((uint32_t)__half_as_ushort(hv[3]) << 16);
      pk.z = (uint32_t)__half_as_ushort(hv[4]) | ((uint32_t)__half_as_ushort(hv[5]) << 16);
      pk.w = (uint32_t)__half_as_ushort(hv[6]) | ((uint32_t)__half_as_ushort(hv[7]) << 16);
      ga[(k8 / 8) * 8] = pk;  // (k/8)*64 halves = 8 x 16 bytes
      gb[(k8 / 8) * 8] = pk;
    }
    // augment columns [dk, K): A = (1, 1, 0 ..), B = (hi, lo, 0 ..) of -|y^|^2 / 2
    for (int k8 = dk; k8 < K; k8 += 8) {
      uint4 a = make_uint4(0u, 0u, 0u, 0u), b = make_uint4(0u, 0u, 0u, 0u);
      if (k8 == dk) {
        if (real) {
          const uint32_t one = __half_as_ushort(__float2half_rn(1.0f));
          a.x = one | (one << 16);
          const float hn = -0.5f * s;
          const __half hi = __float2half_rn(hn);
          const __half lo = __float2half_rn(hn - __half2float(hi));
          b.x = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
        } else {
          b.x = (uint32_t)__half_as_ushort(__float2half_rn(-65504.0f));
        }
      }
      ga[(k8 / 8) * 8] = a;
      gb[(k8 / 8) * 8] = b;
    }
    nrm[p] = real ? s : 0.0f;
    len[p] = real ? sqrtf(s) : 0.0f;
    // rounded up, with a relative margin for the rounded subtraction and squares
    const float E = real ? __fsqrt_ru(__fmul_ru(e2, 1.0f + (float)(d + 8) * 0x1p-23f)) + 1e-30f : 0.0f;
    err[p] = E;
    return E;
  }
}

__global__ void k_pack(const float* __restrict__ X, int64_t n, int d, int dk, int K, const int* __restrict__ perm,
                       const float* __restrict__ c, const TcScale* __restrict__ sc, int64_t npad, __half* __restrict__ YA,
                       __half* __restrict__ YB, float* __restrict__ nrm, float* __restrict__ len,
                       float* __restrict__ err, unsigned* __restrict__ maxerr) {
  float emax = 0.0f;
  const float scale = sc->scale;
  const bool vec = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npad; p += (int64_t)gridDim.x * blockDim.x)
    emax = fmaxf(emax, pack_point(X, n, d, dk, K, perm, c, scale, vec, npad, p, YA, YB, nrm, len, err, nullptr));
  // one atomic per block for the global maximum (a single address: atomics serialise)
#pragma unroll
  for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  __shared__ float wmax[32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int t = 0; t < (int)(blockDim.x >> 5); t++) m = fmaxf(m, wmax[t]);
    if (m > 0.0f) atomicMax(maxerr, __float_as_uint(m));
  }
}

// XTp[k][p] = X[perm[p]][k]: permuted, transposed fp32 copy for coalesced exact R1 (32x32 tiles)
__global__ void k_transpose_perm(const float* __restrict__ X, int64_t n, int d, const int* __restrict__ perm,
                                 int64_t npad, float* __restrict__ XTp) {
  __shared__ float tile[32][33];
  const int64_t p0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t p = p0 + r;
    const int k = k0 + threadIdx.x;
    tile[r][threadIdx.x] = (p < n && k < d) ? X[(int64_t)perm[p] * d + k] : 0.0f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int k = k0 + r;
    const int64_t p = p0 + threadIdx.x;
    if (k < d && p < npad) XTp[(int64_t)k * npad + p] = tile[threadIdx.x][r];
  }
}

// max |y^| over each TC_TMG-column segment (one warp per segment)
__global__ void k_seg_maxlen(const float* __restrict__ len, const float* __restrict__ err, int64_t nseg,
                             float* __restrict__ seg_max, float* __restrict__ seg_maxerr) {
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int64_t g = (int64_t)blockIdx.x * warps + w; g < nseg; g += (int64_t)gridDim.x * warps) {
    float m = 0.0f, me = 0.0f;
    for (int t = lane; t < TC_TMG; t += 32) {
      m = fmaxf(m, len[g * TC_TMG + t]);
      me = fmaxf(me, err[g * TC_TMG + t]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      me = fmaxf(me, __shfl_xor_sync(0xffffffffu, me, o));
    }
    if (lane == 0) {
      seg_max[g] = m;
      seg_maxerr[g] = me;
    }
  }
}

// after sorting (comp, idx): sorted comp labels sc[p]; component ranges per permuted row
__global__ void k_comp_ranges(const int* __restrict__ sc, int64_t n, int* __restrict__ cstart,
                              int* __restrict__ cend) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = sc[p];
    if (p == 0 || sc[p - 1] != c) cstart[c] = (int)p;
    if (p == n - 1 || sc[p + 1] != c) cend[c] = (int)p + 1;
  }
}
__global__ void k_row_ranges(const int* __restrict__ sc, int64_t n, const int* __restrict__ cstart,
                             const int* __restrict__ cend, int* __restrict__ rs, int* __restrict__ re) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = sc[p];
    rs[p] = cstart[c];
    re[p] = cend[c];
  }
}

__global__ void k_gather_comp(const int* __restrict__ comp, int64_t n, int* __restrict__ keys,
                              int* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = comp[i];
    idx[i] = (int)i;
  }
}

// ---------------------------------------------------------------------------
// exact pass
// ---------------------------------------------------------------------------
struct ExactParams {
  const float* XTp;  // d x npad, permuted columns
  int64_t npad;
  int d, n;
  const int* perm;
  const float* nrm;
  const float* len;
  const float* seg_maxlen;
  const TcScale* tsc;  // device: maxlen bounds |y^|  // max |y^| over all points
  const float* err;         // E_p (permuted)
  const float* seg_maxerr;  // per segment max E
  const float* maxerr;      // max E (device)
  const int* cs;
  const int* ce;
  const unsigned* UB;
  const float* TM;  // [segment][row] eligible maximum of G'
  int nseg;         // npad / TC_TMG
  int p_begin, p_end;
  uint2* list;  // qualifying (row, tile) pairs
  unsigned list_cap;
  int* rowflag;
  int round0;
  ErrModel em;
  const int* comp;  // original-index component labels
  u64* compbest;
  unsigned* counters;  // [0] fallback rows, [1] listed tiles, [2] exact tiles evaluated
  int* fallback;
  // re-scan rounds: only rows with needp[p] are filtered, against the tighter of their
  // own bound and their component's (compUB, original-index component labels)
  const int* needp;
  const unsigned* compUB;
};

// One warp per 32 consecutive rows: every 64-column tile whose eligible maximum of G'
// meets the row's FINAL threshold (L <= UB_i possible) is listed for exact evaluation;
// those tiles hold every candidate of the row, hence its exact argmin and all ties.
// The cheap test with the largest column norm (most permissive) runs first.
__global__ void k_filter_tiles(ExactParams E) {
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int p0 = E.p_begin + (blockIdx.x * warps + w) * 32; p0 < E.p_end; p0 += gridDim.x * warps * 32) {
    const int p = p0 + lane;
    const bool valid = p < E.p_end && (!E.needp || E.needp[p]);
    if (!__any_sync(0xffffffffu, valid)) continue;
    float ub = valid ? __uint_as_float(E.UB[p]) : 0.0f;
    if (valid && E.compUB) ub = fminf(ub, __uint_as_float(E.compUB[E.comp[E.perm[p]]]));
    const float ni = valid ? E.nrm[p] : 0.0f, li = valid ? E.len[p] : 0.0f;
    const float ei = valid ? E.err[p] : 0.0f, emax = *E.maxerr;
    const float* tm_row = E.TM + tm_index(0, valid ? p : E.p_begin, E.nseg);  // segment s at tm_row[s * 512]
    const float thr_min = valid ? em_thr(E.em, ub, ni, li, E.tsc->maxlen, em_delta2(ei, emax)) : INFINITY;
    bool flagged = false;
    constexpr int U = 8;  // segments per batch: U independent coalesced loads in flight
    for (int t0 = 0; t0 < E.nseg; t0 += U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; u++)
        v[u] = (valid && t0 + u < E.nseg) ? __ldcs(tm_row + (int64_t)(t0 + u) * 512) : -INFINITY;
      bool any = false;
#pragma unroll
      for (int u = 0; u < U; u++) any |= v[u] >= thr_min && v[u] > -INFINITY;
      if (!__any_sync(0xffffffffu, any)) continue;
#pragma unroll
      for (int u = 0; u < U; u++) {
        bool want = v[u] >= thr_min && v[u] > -INFINITY;
        if (want) want = v[u] >= em_thr(E.em, ub, ni, li, E.seg_maxlen[t0 + u], em_delta2(ei, E.seg_maxerr[t0 + u]));
        const unsigned bal = __ballot_sync(0xffffffffu, want);
        if (bal) {
          unsigned base = 0;
          const int leader = __ffs(bal) - 1;
          if (lane == leader) base = atomicAdd(E.counters + 1, (unsigned)__popc(bal));
          base = __shfl_sync(0xffffffffu, base, leader);
          if (want) {
            const unsigned slot = base + __popc(bal & ((1u << lane) - 1u));
            if (slot < E.list_cap) E.list[slot] = make_uint2((unsigned)p, (unsigned)(t0 + u));
            else flagged = true;
          }
        }
      }
    }
    if (flagged) {  // list full: this row is re-scanned exactly over all columns
      E.rowflag[p] = 1;
      E.fallback[atomicAdd(E.counters, 1u)] = p;
    }
  }
}

// One warp per listed (row, tile): R1 evaluated exactly on the tile's 64 columns
// (two per lane, coalesced on XTp); the minimum edge key goes to the row's component.
__global__ void k_exact_tiles(ExactParams E) {
  unsigned cnt = E.counters[1];
  if (cnt > E.list_cap) cnt = E.list_cap;
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  unsigned done = 0;
  for (unsigned a = blockIdx.x * warps + w; a < cnt; a += gridDim.x * warps) {
    const uint2 pt = E.list[a];
    const int p = (int)pt.x, t = (int)pt.y;
    if (E.rowflag[p]) continue;  // the fallback re-scans this row completely
    done++;
    const int cs = E.round0 ? p : E.cs[p];
    const int ce = E.round0 ? p + 1 : E.ce[p];
    const int oi = E.perm[p];
    const float* xi = E.XTp + p;
    u64 key = KEY_NONE;
    constexpr int V = TC_TMG / 32;  // columns per lane, evaluated as independent chains
    float acc[V];
#pragma unroll
    for (int u = 0; u < V; u++) acc[u] = 0.0f;
    const int q0 = t * TC_TMG + lane;
    for (int k = 0; k < E.d; k++) {
      const float x = __ldg(xi + (int64_t)k * E.npad);
      const float* row = E.XTp + (int64_t)k * E.npad + q0;
#pragma unroll
      for (int u = 0; u < V; u++) {
        const float tt = __fsub_rn(x, __ldg(row + u * 32));
        acc[u] = __fmaf_rn(tt, tt, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < V; u++) {
      const int qcol = q0 + u * 32;
      if (qcol < E.n && (qcol < cs || qcol >= ce)) {
        const u64 kk = ((u64)(__float_as_uint(acc[u]) & 0x7FFFFFFFu) << 33) | tri_index(oi, E.perm[qcol]);
        key = kk < key ? kk : key;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other < key ? other : key;
    }
    if (lane == 0 && key != KEY_NONE) atomic_min_lt(E.compbest + E.comp[oi], key);
  }
  if (lane == 0 && done) atomicAdd(E.counters + 2, done);
}

// fallback: exact R1 over all eligible columns of a row (one CTA per row, 4 columns
// per thread in flight, coalesced on XTp)
__global__ void __launch_bounds__(256) k_exact_rows(ExactParams E) {
  const unsigned cnt = E.counters[0];
  __shared__ u64 red[8];
  __shared__ float xi_s[1024];
  for (unsigned f = blockIdx.x; f < cnt; f += gridDim.x) {
    const int p = E.fallback[f];
    const int cs = E.round0 ? p : E.cs[p];
    const int ce = E.round0 ? p + 1 : E.ce[p];
    const int oi = E.perm[p];
    u64 best = KEY_NONE;
    const bool xs = E.d <= 1024;  // x_i staged in shared memory (else read from global)
    if (xs)
      for (int k = threadIdx.x; k < E.d; k += blockDim.x) xi_s[k] = E.XTp[(int64_t)k * E.npad + p];
    __syncthreads();
    for (int q0 = threadIdx.x; q0 < E.n; q0 += 4 * blockDim.x) {
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int k = 0; k < E.d; k++) {
        const float x = xs ? xi_s[k] : __ldg(E.XTp + (int64_t)k * E.npad + p);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int qq = q0 + u * blockDim.x;
          const float y = qq < E.n ? __ldg(E.XTp + (int64_t)k * E.npad + qq) : 0.0f;
          const float t = __fsub_rn(x, y);
          acc[u] = __fmaf_rn(t, t, acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int qq = q0 + u * blockDim.x;
        if (qq < E.n && (qq < cs || qq >= ce)) {
          const u64 key = ((u64)(__float_as_uint(acc[u]) & 0x7FFFFFFFu) << 33) | tri_index(oi, E.perm[qq]);
          best = key < best ? key : best;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int t = 0; t < (int)(blockDim.x >> 5); t++) best = red[t] < best ? red[t] : best;
      if (best != KEY_NONE) atomic_min_lt(E.compbest + E.comp[oi], best);
    }
    __syncthreads();
  }
}

int64_t tcf_row_tiles(const TcState* st) { return st->npad / TC_ROWS; }

// ---------------------------------------------------------------------------
// host-side driver
// ---------------------------------------------------------------------------
static ErrModel error_model(const TcState* st) {
  ErrModel e;
  e.c1 = st->c1;
  e.c2 = st->c2;
  e.k1 = st->k1;
  e.k2 = st->k2;
  e.k3 = st->k3;
  e.gamma = st->gamma;
  return e;
}

// scale = 2^e with scale * max|x - c| in [2^6.5, 2^7.5): |y^|^2 < 2^15, fp16 range safe;
// fp16 rounding can lift |y^| by 2^-11 relative (plus subnormal slack): maxlen margin
__device__ __forceinline__ TcScale tc_scale_of(unsigned maxlen_bits) {
  const float ml = __uint_as_float(maxlen_bits);
  TcScale r;
  r.ok = ml < INFINITY ? 1 : 0;
  int e = 0;
  if (ml > 0.0f && r.ok) {
    e = (int)floor(7.0 - log2((double)ml) + 0.5);
    e = max(-100, min(100, e));
  }
  r.scale = (float)ldexp(1.0, e);
  r.maxlen = r.ok ? (float)((double)ml * r.scale * (1.0 + ldexp(1.0, -10)) + 1e-6) : 0.0f;
  r.s2 = (double)r.scale * (double)r.scale;
  r.pad = 0;
  return r;
}
__global__ void k_tc_scale(const unsigned* __restrict__ maxlen_bits, TcScale* __restrict__ out) {
  *out = tc_scale_of(*maxlen_bits);
}

// ---------------------------------------------------------------------------
// The whole preparation of the first round in ONE cooperative launch (it was ten kernels
// and memsets, ~100 us of a C4 solve): phase 1 per-block partial column sums (the fixed
// 64-row partition of k_center_partial: the same centre bit for bit) and the caller's
// buffer initialisations; phase 2 the centre; phase 3 max |x - c| (+ the input
// validation); phase 4 the scale, the packed operands of round 0 (identity order), the
// fp32 transpose for the exact kernels and the per-segment maxima.  Grid-wide barriers
// separate the phases.
// ---------------------------------------------------------------------------
struct PrepArgs {
  const float* X;
  int64_t n, npad;
  int d, dk, K, rpb, blocks;
  double* part;
  float* center;
  unsigned* maxlen;
  TcScale* dscale;
  __half *YA, *YB;
  float *nrm, *len, *err;
  unsigned* maxerr;
  float* xt;
  unsigned *seg_maxlen, *seg_maxerr;
  u64* bad;
  unsigned long long* dbg;  // development builds: %globaltimer after each phase (CTA 0)
  const int* perm;          // pack_tile: point at position p (nullptr: identity)
  InitList init;
  unsigned* bar;  // grid barrier word (coop_grid_sync)
};
__device__ __forceinline__ void prep_mark(const PrepArgs& a, int i) {
  if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[i] = t;
  }
}

__device__ __forceinline__ void run_init(const InitList& L, int64_t tid, int64_t nt) {
  for (int t = 0; t < L.count; t++) {
    const InitTask& T = L.t[t];
    if (T.kind == 0) {
      unsigned* p = reinterpret_cast<unsigned*>(T.p);
      for (int64_t i = tid; i < T.count; i += nt) p[i] = (unsigned)T.value;
    } else if (T.kind == 1) {
      u64* p = reinterpret_cast<u64*>(T.p);
      for (int64_t i = tid; i < T.count; i += nt) p[i] = T.value;
    } else {
      int* p = reinterpret_cast<int*>(T.p);
      for (int64_t i = tid; i < T.count; i += nt) p[i] = (int)i;
    }
  }
}

__global__ void k_init(const InitList L) {
  run_init(L, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// phase 4 body: one tile of 32 * sets points (identity order), GW warps per 32 points,
// warp w covers the 8-coordinate groups g = w % GW, w % GW + GW, ... of point lane; the
// per-group partial norms and error sums meet in shared memory (norm: fp32, any order is
// inside the error model's d 2^-24 allowance; error sum: rounded up, so an upper bound)
__device__ __forceinline__ float pack_tile(const PrepArgs& a, float scale, bool vec, int64_t p0, int G, int GW,
                                           int sets, float (*s_part)[32], float (*e_part)[32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int set = w / GW, gw = w % GW;
  const int64_t p = p0 + set * 32 + lane;
  const bool act = set < sets;
  const bool real = act && p < a.n;
  const int K = a.K, d = a.d;
  float s = 0.0f, e2 = 0.0f;
  if (act) {
    const int64_t gidx = p / 128;
    const int pl = (int)(p % 128), g8 = pl / 8, r = pl % 8;
    uint4* ga = reinterpret_cast<uint4*>(a.YA + gidx * 128 * K + (int64_t)g8 * (K / 8) * 64 + r * 8);
    uint4* gb = reinterpret_cast<uint4*>(a.YB + gidx * 128 * K + (int64_t)g8 * (K / 8) * 64 + r * 8);
    const float* xi = a.X + (real ? (a.perm ? a.perm[p] : p) : 0) * d;
    for (int g = gw; g < G; g += GW) {
      const int k8 = 8 * g;
      float xv[8];
      if (real && vec && k8 + 8 <= d) {
        const float4 u0 = __ldg(reinterpret_cast<const float4*>(xi + k8));
        const float4 u1 = __ldg(reinterpret_cast<const float4*>(xi + k8 + 4));
        xv[0] = u0.x; xv[1] = u0.y; xv[2] = u0.z; xv[3] = u0.w;
        xv[4] = u1.x; xv[5] = u1.y; xv[6] = u1.z; xv[7] = u1.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; u++) xv[u] = (real && k8 + u < d) ? __ldg(xi + k8 + u) : 0.0f;
      }
      if (a.xt)
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (k8 + u < d) a.xt[(int64_t)(k8 + u) * a.npad + p] = xv[u];
      __half hv[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int k = k8 + u;
        hv[u] = __float2half_rn(0.0f);
        if (real && k < d) {  // as pack_point: TwoSum error of the centring, exact fp16 residual
          const float xk = xv[u], ck = a.center[k];
          const float t = __fsub_rn(xk, ck);
          const float bb = __fsub_rn(t, xk);
          const float dt = __fadd_rn(__fsub_rn(xk, __fsub_rn(t, bb)), __fsub_rn(-ck, bb));
          const float y = scale * t;
          hv[u] = __float2half_rn(y);
          const float ek = __fsub_rn(__fsub_rn(__half2float(hv[u]), y), scale * dt);
          e2 = __fmaf_ru(ek, ek, e2);
        }
        const float hf = __half2float(hv[u]);
        s = fmaf(hf, hf, s);
      }
      uint4 pk;
      pk.x = (uint32_t)__half_as_ushort(hv[0]) | ((uint32_t)__half_as_ushort(hv[1]) << 16);
      pk.y = (uint32_t)__half_as_ushort(hv[2]) | ((uint32_t)__half_as_ushort(hv[3]) << 16);
      pk.z = (uint32_t)__half_as_ushort(hv[4]) | ((uint32_t)__half_as_ushort(hv[5]) << 16);
      pk.w = (uint32_t)__half_as_ushort(hv[6]) | ((uint32_t)__half_as_ushort(hv[7]) << 16);
      ga[g * 8] = pk;
      gb[g * 8] = pk;
    }
    s_part[w][lane] = s;
    e_part[w][lane] = e2;
  }
  __syncthreads();
  float E = 0.0f;
  if (act && gw == 0) {  // the set's first warp: totals, augment columns, per-point outputs
    s = 0.0f;
    e2 = 0.0f;
    for (int j = 0; j < GW; j++) {
      s += s_part[set * GW + j][lane];
      e2 = __fadd_ru(e2, e_part[set * GW + j][lane]);
    }
    const int64_t gidx = p / 128;
    const int pl = (int)(p % 128), g8 = pl / 8, r = pl % 8;
    uint4* ga = reinterpret_cast<uint4*>(a.YA + gidx * 128 * K + (int64_t)g8 * (K / 8) * 64 + r * 8);
    uint4* gb = reinterpret_cast<uint4*>(a.YB + gidx * 128 * K + (int64_t)g8 * (K / 8) * 64 + r * 8);
    for (int k8 = a.dk; k8 < K; k8 += 8) {
      uint4 ua = make_uint4(0u, 0u, 0u, 0u), ub = make_uint4(0u, 0u, 0u, 0u);
      if (k8 == a.dk) {
        if (real) {
          const uint32_t one = __half_as_ushort(__float2half_rn(1.0f));
          ua.x = one | (one << 16);
          const float hn = -0.5f * s;
          const __half hi = __float2half_rn(hn);
          const __half lo = __float2half_rn(hn - __half2float(hi));
          ub.x = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
        } else {
          ub.x = (uint32_t)__half_as_ushort(__float2half_rn(-65504.0f));
        }
      }
      ga[(k8 / 8) * 8] = ua;
      gb[(k8 / 8) * 8] = ub;
    }
    const float len = real ? sqrtf(s) : 0.0f;
    a.nrm[p] = real ? s : 0.0f;
    a.len[p] = len;
    E = real ? __fsqrt_ru(__fmul_ru(e2, 1.0f + (float)(d + 8) * 0x1p-23f)) + 1e-30f : 0.0f;
    a.err[p] = E;
    float ml = len, me = E;  // the warp's 32 points lie in one TC_TMG segment
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      ml = fmaxf(ml, __shfl_xor_sync(0xffffffffu, ml, o));
      me = fmaxf(me, __shfl_xor_sync(0xffffffffu, me, o));
    }
    if (lane == 0) {
      atomicMax(a.seg_maxlen + p / TC_TMG, __float_as_uint(ml));
      atomicMax(a.seg_maxerr + p / TC_TMG, __float_as_uint(me));
    }
  }
  __syncthreads();  // s_part / e_part are reused by the next tile
  return E;
}

__global__ void __launch_bounds__(256, 3) k_tc_prep(const PrepArgs a) {
  __shared__ double red[256];
  __shared__ float s_part[8][32], e_part[8][32];
  __shared__ float cs[1024];
  const int64_t tid = blockIdx.x * 256ll + threadIdx.x, nt = gridDim.x * 256ll;
  const int lane = threadIdx.x & 31;
  const int d = a.d;
  const bool vec = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  prep_mark(a, 0);
  // phase 1: fp64 column sums of fixed 16-row blocks, one warp per block (lanes = columns)
  for (int64_t b = tid >> 5; b < a.blocks; b += nt >> 5) {
    const int64_t r0 = b * a.rpb, r1 = min(a.n, r0 + a.rpb);
    for (int k0 = 0; k0 < d; k0 += 64) {
      const int ka = k0 + lane, kb = k0 + 32 + lane;
      double sa = 0.0, sb = 0.0;
#pragma unroll 8
      for (int64_t r = r0; r < r1; r++) {
        if (ka < d) sa += (double)__ldg(a.X + r * d + ka);
        if (kb < d) sb += (double)__ldg(a.X + r * d + kb);
      }
      if (ka < d) a.part[(int64_t)ka * a.blocks + b] = sa;  // column-major: phase 2 reads runs
      if (kb < d) a.part[(int64_t)kb * a.blocks + b] = sb;
    }
  }
  run_init(a.init, tid, nt);
  if (tid == 0) {
    *a.maxlen = 0u;
    *a.maxerr = 0u;
    if (a.bad) a.bad[0] = a.bad[1] = a.bad[2] = KEY_NONE;
  }
  prep_mark(a, 1);
  coop_grid_sync(a.bar);
  prep_mark(a, 2);
  // phase 2: the centre, one CTA per column (a fixed tree: deterministic)
  for (int k = blockIdx.x; k < d; k += gridDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int b = threadIdx.x; b < a.blocks; b += 256) s += a.part[(int64_t)k * a.blocks + b];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = 128; h; h >>= 1) {
      if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x == 0) a.center[k] = (float)(red[0] / (double)a.n);
    __syncthreads();
  }
  coop_grid_sync(a.bar);
  prep_mark(a, 3);
  const bool cs_ok = d <= 1024;  // the centre staged in shared memory
  if (cs_ok) {
    for (int k = threadIdx.x; k < d; k += 256) cs[k] = a.center[k];
    __syncthreads();
  }
  const float* cen = cs_ok ? cs : a.center;
  // phase 3: max |x - c| (fp32, sets the scale; the error model carries a 2^-10 margin)
  // and the validation: four threads per point (float4 k-steps q, q + 4, ...)
  {
    float best = 0.0f;
    u64 badi = KEY_NONE;
    const int q = (int)(tid & 3);
    for (int64_t i = tid >> 2; i < ((a.n + 7) & ~7ll); i += nt >> 2) {  // quads stay converged
      float sum = 0.0f;
      if (i < a.n) {
        if (vec) {
          const float4* x4 = reinterpret_cast<const float4*>(a.X + i * d);
#pragma unroll 4
          for (int k4 = q; k4 < d / 4; k4 += 4) {
            const float4 v = __ldg(x4 + k4);
            const int k = 4 * k4;
            if (a.bad && badi == KEY_NONE) {
              if (!isfinite(v.x)) badi = (u64)(i * d + k);
              else if (!isfinite(v.y)) badi = (u64)(i * d + k + 1);
              else if (!isfinite(v.z)) badi = (u64)(i * d + k + 2);
              else if (!isfinite(v.w)) badi = (u64)(i * d + k + 3);
            }
            const float t0 = v.x - cen[k], t1 = v.y - cen[k + 1], t2 = v.z - cen[k + 2], t3 = v.w - cen[k + 3];
            sum += t0 * t0 + t1 * t1 + t2 * t2 + t3 * t3;
          }
        } else {
          for (int k = q; k < d; k += 4) {
            const float x = a.X[i * d + k];
            if (a.bad && badi == KEY_NONE && !isfinite(x)) badi = (u64)(i * d + k);
            const float t = x - cen[k];
            sum += t * t;
          }
        }
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      best = fmaxf(best, sum);
    }
    block_max_sqrt(best, a.maxlen);
    if (badi != KEY_NONE) atomicMin(a.bad, badi);  // the smallest element index over all threads
  }
  coop_grid_sync(a.bar);
  prep_mark(a, 4);
  // phase 4: scale, packed operands, transpose, per-segment maxima
  const TcScale sc = tc_scale_of(*reinterpret_cast<volatile unsigned*>(a.maxlen));
  if (tid == 0) *a.dscale = sc;
  const int G = a.dk / 8, GW = G < 8 ? G : 8, sets = 8 / GW, PT = 32 * sets;
  float emax = 0.0f;
  for (int64_t p0 = (int64_t)blockIdx.x * PT; p0 < a.npad; p0 += (int64_t)gridDim.x * PT)
    emax = fmaxf(emax, pack_tile(a, sc.scale, vec, p0, G, GW, sets, s_part, e_part));
#pragma unroll
  for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  __shared__ float wmax[8];
  if (lane == 0) wmax[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int t = 0; t < 8; t++) m = fmaxf(m, wmax[t]);
    if (m > 0.0f) atomicMax(a.maxerr, __float_as_uint(m));
  }
  prep_mark(a, 5);
}

// the packing of a later pass (points in component order): the same tiles as phase 4 of
// k_tc_prep, the scale already on the device; seg_maxlen / seg_maxerr / maxerr zeroed
// before (k_init)
__global__ void __launch_bounds__(256, 3) k_pack_tiles(const PrepArgs a, const TcScale* __restrict__ sc) {
  __shared__ float s_part[8][32], e_part[8][32];
  const int lane = threadIdx.x & 31;
  const bool vec = (a.d & 3) == 0 && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  const float scale = sc->scale;
  const int G = a.dk / 8, GW = G < 8 ? G : 8, sets = 8 / GW, PT = 32 * sets;
  float emax = 0.0f;
  for (int64_t p0 = (int64_t)blockIdx.x * PT; p0 < a.npad; p0 += (int64_t)gridDim.x * PT)
    emax = fmaxf(emax, pack_tile(a, scale, vec, p0, G, GW, sets, s_part, e_part));
#pragma unroll
  for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  __shared__ float wmax[8];
  if (lane == 0) wmax[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int t = 0; t < 8; t++) m = fmaxf(m, wmax[t]);
    if (m > 0.0f) atomicMax(a.maxerr, __float_as_uint(m));
  }
}

// centre, scale (+ round 0's packing when cooperative), the caller's initialisations and
// the validation verdict
static appd_status launch_prepare(appd_ctx* c, const float* X, TcState* st, const InitList* init, u64* bad) {
  const int64_t n = st->n, d = st->d;
  const int rpb = 64;  // rows per partial sum (separate kernels)
  const int blocks = (int)((n + rpb - 1) / rpb);
  const int rpb_coop = 16;  // (cooperative: one warp per block)
  const int blocks_coop = (int)((n + rpb_coop - 1) / rpb_coop);
  double* part = (double*)ws(c, S_TC_PART, sizeof(double) * std::max(blocks, blocks_coop) * d);
  if (!part) return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc center");
  unsigned* maxlen = (unsigned*)(st->center + d);
  static std::atomic<unsigned long long> occ_set{0};
  static int occ[64];
  if (needs_setup(occ_set, c)) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_tc_prep, 256, 0) != cudaSuccess) o = 0;
    cudaGetLastError();
    occ[c->device & 63] = o;
    setup_done(occ_set, c);
  }
  const int per_sm = std::min(occ[c->device & 63], 4);
  InitList L;
  if (init) L = *init;
  if (per_sm >= 1 && st->topk && L.count + 8 <= 16) {
    // round 0's own initialisations ride along
    L.add(st->perm, n, 0, 2);
    L.add(st->UB, st->npad, 0x7F7F7F7Fu, 0);
    L.add(st->counters, 16, 0, 0);
    L.add(st->rowflag, n, 0, 0);
    L.add(st->cand_cnt, st->npad, 0, 0);
    L.add(st->need, n, 0, 0);
    L.add(st->seg_maxlen, st->npad / TC_TMG, 0, 0);
    L.add(st->seg_maxerr, st->npad / TC_TMG, 0, 0);
    PrepArgs a;
    a.X = X;
    a.n = n;
    a.npad = st->npad;
    a.d = (int)d;
    a.dk = st->dk;
    a.K = st->K;
    a.rpb = rpb_coop;
    a.blocks = blocks_coop;
    a.part = part;
    a.center = st->center;
    a.maxlen = maxlen;
    a.dscale = st->dscale;
    a.YA = (__half*)st->YA;
    a.YB = (__half*)st->YB;
    a.nrm = st->nrm;
    a.len = st->len;
    a.err = st->err;
    a.maxerr = st->maxerr;
    a.xt = st->XT;
    a.seg_maxlen = reinterpret_cast<unsigned*>(st->seg_maxlen);
    a.seg_maxerr = reinterpret_cast<unsigned*>(st->seg_maxerr);
    a.bad = bad;
    a.dbg = nullptr;
    a.perm = nullptr;
    a.init = L;
    a.bar = grid_barrier_word(c);
    if (!a.bar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
    static const bool times = dev_env("APPD_PREP_TIMES") != nullptr;
    if (times) a.dbg = reinterpret_cast<unsigned long long*>(ws(c, S_TMP2, 64));
    void* args[] = {&a};
    APPD_CUDA(c, cudaLaunchCooperativeKernel((const void*)k_tc_prep, c->sm_count * per_sm, 256, args, 0, c->stream));
    APPD_LAUNCHED(c);
    if (times && a.dbg) {
      unsigned long long h[6];
      cudaStreamSynchronize(c->stream);
      cudaMemcpy(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost);
      fprintf(stderr, "[prep] grid %d: phase1 %.1f us, sync %.1f, centre %.1f, maxlen %.1f, pack %.1f\n",
              c->sm_count * per_sm, (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3,
              (h[4] - h[3]) * 1e-3, (h[5] - h[4]) * 1e-3);
    }
    st->r0_packed = true;
  } else {
    if (L.count) {
      k_init<<<c->sm_count * 4, 256, 0, c->stream>>>(L);
      APPD_LAUNCHED(c);
    }
    if (bad) {
      APPD_CUDA(c, cudaMemsetAsync(bad, 0xFF, 3 * sizeof(u64), c->stream));
      appd_status s = launch_validate_points(c, X, n, d, bad);
      if (s) return s;
    }
    k_center_partial<<<blocks, 256, 0, c->stream>>>(X, n, (int)d, rpb, part);
    APPD_LAUNCHED(c);
    k_center_final<<<(unsigned)((d + 7) / 8), 256, 0, c->stream>>>(part, blocks, n, (int)d, st->center);
    APPD_LAUNCHED(c);
    APPD_CUDA(c, cudaMemsetAsync(maxlen, 0, sizeof(unsigned), c->stream));
    k_maxlen<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8), 256, 0, c->stream>>>(
        X, n, (int)d, st->center, maxlen);
    APPD_LAUNCHED(c);
    // the scale on the device (no host round trip)
    k_tc_scale<<<1, 1, 0, c->stream>>>(maxlen, st->dscale);
    APPD_LAUNCHED(c);
  }
  // its ok flag is read at the caller's next synchronisation (coordinates too large for
  // the filter: the solve falls back to the exact engine)
  APPD_PUBLISH(c, c->pinned_small + 50, &st->dscale->ok, sizeof(int));
  return APPD_OK;
}

appd_status tcf_prepare(appd_ctx* c, const float* X, int64_t n, int64_t d, TcState* st, const InitList* init,
                        u64* bad) {
  st->n = n;
  st->d = d;
  st->npad = (n + TC_ROWS - 1) / TC_ROWS * TC_ROWS;
  st->dk = (int)((d + 15) / 16 * 16);
  st->K = st->dk + 16;
  st->stages = tcf_stages(st->K);
  st->r0_packed = false;
  if (st->stages == 0) return APPD_ERR_UNSUPPORTED;
  st->center = (float*)ws(c, S_TC_CENTER, sizeof(float) * (d + 1) + 64);
  st->dscale = (TcScale*)ws(c, S_TC_SCALE, sizeof(TcScale));
  if (!st->center || !st->dscale) return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc center");
  // Error model in scaled units (tc_common.cuh):
  //  delta: each fp16 coordinate is within 2^-11 (relative, normal range) or 2^-25
  //    (absolute, subnormal) of s*(x - c); centring x - c in fp32 adds 2^-24 relative;
  //    so |(y^_i - y^_j) - s (x_i - x_j)| <= (2^-11 + 2^-20)(L + R) + 2 sqrt(d) 2^-25.
  //  eta: Dt = |y^_i|^2 - 2 G' with G' accumulated in fp32 over K terms (allowing one
  //    ulp per addition: K 2^-23 sum|terms|), the fp16 hi/lo split of -|y^_j|^2/2
  //    (2^-22 |y^_j|^2), fp32 norms of d exact products (d 2^-24 |y|^2 each) and the
  //    final subtraction (2^-24 |Dt|):
  //    |Dt - |y^_i - y^_j|^2| <= 2^-24 [4K R (L + R/2) + d (L^2 + R^2) + 4 R^2 + (L+R)^2].
  //  gamma: R1 (d fmaf steps after a 1-rounding subtraction) is within (d + 2) 2^-24
  //    of the real squared distance, relatively.
  // Each constant carries a 1% margin.
  const double u = std::ldexp(1.0, -24);
  st->c1 = (float)((std::ldexp(1.0, -11) + std::ldexp(1.0, -20)) * 1.01);
  st->c2 = (float)(2.0 * std::sqrt((double)d) * std::ldexp(1.0, -25) * 1.01 + 1e-30);
  st->k1 = (float)(4.0 * st->K * u * 1.01);
  st->k2 = (float)(d * u * 1.01);
  st->k3 = (float)(u * 1.01);
  st->gamma = (float)((d + 2.0) * u * 1.01);
  const size_t ybytes = (size_t)st->npad * st->K * 2;
  st->YA = ws(c, S_TC_YA, ybytes);
  st->YB = ws(c, S_TC_YB, ybytes);
  st->XTp = (float*)ws(c, S_TC_XTP, sizeof(float) * st->npad * d);
  st->nrm = (float*)ws(c, S_TC_NRM, sizeof(float) * st->npad);
  st->len = (float*)ws(c, S_TC_LEN, sizeof(float) * st->npad);
  st->seg_maxlen = (float*)ws(c, S_TC_TML, sizeof(float) * (st->npad / TC_TMG));
  st->err = (float*)ws(c, S_TC_ERR, sizeof(float) * st->npad + 64);
  st->seg_maxerr = (float*)ws(c, S_TC_SEGERR, sizeof(float) * (st->npad / TC_TMG) + 64);
  if (!st->err || !st->seg_maxerr) return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc error norms");
  st->maxerr = reinterpret_cast<unsigned*>(st->err + st->npad);
  st->perm = (int*)ws(c, S_TC_PERM, sizeof(int) * (n + 1));
  st->sc = (int*)ws(c, S_TC_SC, sizeof(int) * (n + 1));
  st->keys = (int*)ws(c, S_TC_KEYS, sizeof(int) * 2 * (n + 1));
  st->cstart = (int*)ws(c, S_TC_CSTART, sizeof(int) * (n + 1));
  st->cend = (int*)ws(c, S_TC_CEND, sizeof(int) * (n + 1));
  st->rs = (int*)ws(c, S_TC_RS, sizeof(int) * (n + 1));
  st->re = (int*)ws(c, S_TC_RE, sizeof(int) * (n + 1));
  st->UB = (unsigned*)ws(c, S_TC_UB, sizeof(unsigned) * st->npad);
  st->counters = (unsigned*)ws(c, S_TC_CNT, 64);
  st->h_counters = c->pinned_small;
  st->fallback = (int*)ws(c, S_TC_FALLBACK, sizeof(int) * (n + 1));
  st->rowflag = (int*)ws(c, S_TC_ROWFLAG, sizeof(int) * (n + 1));
  // cache length: option (0 = auto 16, -1 = none); the cache needs K distinct 32-column chunks
  st->topk = c->opt.topk == 0 ? 8 : (c->opt.topk < 0 ? 0 : c->opt.topk);
  if (st->topk != 0 && st->topk != 4 && st->topk != 8 && st->topk != 16 && st->topk != 32)
    return fail(c, APPD_ERR_INVALID_ARGUMENT, "topk = %d (0, -1, 4, 8, 16 or 32)", c->opt.topk);
  // TM holds 32-column maxima in the cache-building round (4x the 128-column layout)
  // (the cache pass's fp16 32-column table and the later passes' fp32 64-column tables)
  st->TM = ws(c, S_TC_APPV, std::max<int64_t>(st->topk ? sizeof(__half) * tm32_elems(st->npad) : 0,
                                             sizeof(float) * st->npad * (st->npad / TC_TMG)));
  st->list_cap = (unsigned)std::min<int64_t>(16 * n + 65536, (int64_t)1 << 30);
  st->list = ws(c, S_TC_APPPC, sizeof(uint2) * st->list_cap);
  if (st->topk) {
    st->cap = 4 * st->topk > 128 ? 128 : 4 * st->topk;
    const int64_t nb = st->npad / TC_ROWS + 1;
    st->ckey = (u64*)ws(c, S_TC_CKEY, sizeof(u64) * n * st->topk);
    st->cj = (int*)ws(c, S_TC_CJ, sizeof(int) * n * st->topk);
    st->ccnt = (int*)ws(c, S_TC_CCNT, sizeof(int) * n);
    st->need = (int*)ws(c, S_TC_NEED, sizeof(int) * n);
    st->needp = (int*)ws(c, S_TC_NEEDP, sizeof(int) * st->npad);
    st->blockflag = (int*)ws(c, S_TC_BLOCKFLAG, sizeof(int) * (2 * nb + 8));
    st->rb_list = st->blockflag ? st->blockflag + nb : nullptr;
    st->rb_count = st->blockflag ? st->blockflag + 2 * nb : nullptr;
    st->compUB = (unsigned*)ws(c, S_TC_COMPUB, sizeof(unsigned) * std::max<int64_t>(n, 2 * 128 * 128));
    st->UBK = (float*)ws(c, S_TC_UBK, sizeof(float) * st->npad);
    st->thrK = (float*)ws(c, S_TC_THRK, sizeof(float) * st->npad);
    st->cand_cnt = (unsigned*)ws(c, S_TC_CANDCNT, sizeof(unsigned) * (st->npad + 8));
    st->cand = (u64*)ws(c, S_TC_CANDK, sizeof(u64) * st->npad * st->cap);
    // every (row, chunk) pair when that is small (tiny n lists everything), else 32 per row
    const int64_t all_pairs = n * ((n + 31) / 32);
    st->list_entries_cap =
        (unsigned)std::min<int64_t>(std::max<int64_t>(32 * n + 65536, all_pairs <= (4 << 20) ? all_pairs : 0),
                                    (int64_t)1 << 31);
    if (c->opt.list_cap > 0)  // option (tests): a small capacity forces the overflow path (poisoned rows)
      st->list_entries_cap = (unsigned)c->opt.list_cap;
    st->lista = (unsigned*)ws(c, S_TC_LISTA, sizeof(unsigned) * st->list_entries_cap);
    st->listb = (unsigned*)ws(c, S_TC_LISTB, sizeof(unsigned) * st->list_entries_cap);
    if (!st->lista || !st->listb) return fail(c, APPD_ERR_OUT_OF_MEMORY, "candidate list workspace");
    st->rows_list = (int*)ws(c, S_TC_ROWLIST, sizeof(int) * (n + 1));
    st->XT = (float*)ws(c, S_TC_XTO, sizeof(float) * st->npad * d);
    if (!st->rows_list || !st->XT) return fail(c, APPD_ERR_OUT_OF_MEMORY, "candidate cache workspace");
    if (!st->ckey || !st->cj || !st->ccnt || !st->need || !st->needp || !st->blockflag || !st->compUB || !st->UBK ||
        !st->thrK || !st->cand_cnt || !st->cand)
      return fail(c, APPD_ERR_OUT_OF_MEMORY, "candidate cache workspace");
  }
  st->invalid_rows = 0;
  if (!st->YA || !st->YB || !st->XTp || !st->nrm || !st->len || !st->seg_maxlen ||
      !st->perm || !st->sc || !st->keys || !st->cstart || !st->cend || !st->rs || !st->re || !st->UB ||
      !st->counters || !st->fallback || !st->rowflag || !st->TM || !st->list)
    return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc workspace");
  return launch_prepare(c, X, st, init, bad);
}

// xt: the d x npad fp32 transpose of the packed order for the exact kernels (nullptr:
// not needed); extra: the caller's initialisations, in the same launch as the pack's own
static appd_status tcf_pack(appd_ctx* c, TcState* st, const float* X, float* xt, const InitList* extra = nullptr) {
  InitList L;
  if (extra) L = *extra;
  L.add(st->maxerr, 1, 0, 0);
  L.add(st->seg_maxlen, st->npad / TC_TMG, 0, 0);
  L.add(st->seg_maxerr, st->npad / TC_TMG, 0, 0);
  k_init<<<c->sm_count * 2, 256, 0, c->stream>>>(L);
  APPD_LAUNCHED(c);
  PrepArgs a;
  memset(&a, 0, sizeof a);
  a.X = X;
  a.n = st->n;
  a.npad = st->npad;
  a.d = (int)st->d;
  a.dk = st->dk;
  a.K = st->K;
  a.center = st->center;
  a.YA = (__half*)st->YA;
  a.YB = (__half*)st->YB;
  a.nrm = st->nrm;
  a.len = st->len;
  a.err = st->err;
  a.maxerr = st->maxerr;
  a.xt = xt;
  a.seg_maxlen = reinterpret_cast<unsigned*>(st->seg_maxlen);
  a.seg_maxerr = reinterpret_cast<unsigned*>(st->seg_maxerr);
  a.perm = st->perm;
  k_pack_tiles<<<c->sm_count * 3, 256, 0, c->stream>>>(a, st->dscale);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

static void fill_scan_params(const TcState* st, TcParams* P) {
  memset(P, 0, sizeof *P);
  P->YA = (const __half*)st->YA;
  P->YB = (const __half*)st->YB;
  P->nrm = st->nrm;
  P->len = st->len;
  P->seg_maxlen = st->seg_maxlen;
  P->err = st->err;
  P->seg_maxerr = st->seg_maxerr;
  P->cs = st->rs;
  P->ce = st->re;
  P->UB = st->UB;
  P->TM = st->TM;
  P->tm_ld = st->npad;
  P->tm_nseg = (int)(st->npad / 32);
  P->n = (int)st->n;
  P->K = st->K;
  P->stages = st->stages;
  P->col_tiles = (int)(st->npad / TC_N);
  P->em = error_model(st);
  P->seg32 = 0;
  P->rb_list = nullptr;
  P->rb_count = nullptr;
  P->upper = 0;
}

static void exact_params(const TcState* st, const TcParams& P, const int* comp, u64* compbest, int p_begin,
                         int p_end, int round0, ExactParams* E) {
  memset(E, 0, sizeof *E);
  E->XTp = st->XTp;
  E->npad = st->npad;
  E->d = (int)st->d;
  E->n = (int)st->n;
  E->perm = st->perm;
  E->nrm = st->nrm;
  E->len = st->len;
  E->seg_maxlen = st->seg_maxlen;
  E->tsc = st->dscale;
  E->err = st->err;
  E->seg_maxerr = st->seg_maxerr;
  E->maxerr = reinterpret_cast<const float*>(st->maxerr);
  E->cs = st->rs;
  E->ce = st->re;
  E->UB = st->UB;
  E->TM = static_cast<const float*>(st->TM);
  E->nseg = (int)(st->npad / TC_TMG);
  E->p_begin = p_begin;
  E->p_end = p_end;
  E->list = (uint2*)st->list;
  E->list_cap = st->list_cap;
  E->rowflag = st->rowflag;
  E->round0 = round0;
  E->em = P.em;
  E->comp = comp;
  E->compbest = compbest;
  E->counters = st->counters;
  E->fallback = st->fallback;
}

// re-scans of at most this many rows run the exact row kernel instead of a tensor-core pass
constexpr int kSmallRescan = 1024;

// filter + exact re-check of the listed (row, 128-column segment) pairs + full-row
// fallback; compbest[comp] receives the exact minimum keys
static appd_status exact_stage(appd_ctx* c, const ExactParams& E) {
  const int rows = E.p_end - E.p_begin;
  if (rows <= 0) return APPD_OK;
  k_filter_tiles<<<std::min(c->sm_count * 8, (rows + 255) / 256), 256, 0, c->stream>>>(E);
  APPD_LAUNCHED(c);
  k_exact_tiles<<<c->sm_count * 16, 256, 0, c->stream>>>(E);
  APPD_LAUNCHED(c);
  k_exact_rows<<<c->sm_count * 2, 256, 0, c->stream>>>(E);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

static int bits_for(int64_t v) {
  int b = 1;
  while ((int64_t)1 << b < v) b++;
  return b;
}

// points sorted by component (stable: by index inside a component), the permutation, and
// the component ranges: one cooperative launch for k <= 256 components, else gather, the
// library sort and two range kernels
static appd_status sort_by_component(appd_ctx* c, TcState* st, const int* comp, int64_t k, int grid_n) {
  const int64_t n = st->n;
  const int bits = bits_for(k + 1);
  appd_status s = sort_components(c, comp, n, bits, st->sc, st->perm, st->cstart, st->cend, st->rs, st->re);
  if (s != APPD_ERR_UNSUPPORTED) return s;
  k_gather_comp<<<grid_n, 256, 0, c->stream>>>(comp, n, st->keys, st->keys + n + 1);
  APPD_LAUNCHED(c);
  if ((s = sort_pairs_i32_bits(c, st->keys, st->sc, st->keys + n + 1, st->perm, n, bits))) return s;
  k_comp_ranges<<<grid_n, 256, 0, c->stream>>>(st->sc, n, st->cstart, st->cend);
  APPD_LAUNCHED(c);
  k_row_ranges<<<grid_n, 256, 0, c->stream>>>(st->sc, n, st->cstart, st->cend, st->rs, st->re);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// sort the listed (chunk << 32 | row) entries by chunk and re-check them exactly:
// mode 0 appends cache candidates, mode 1 reduces component-pair minima into WCM
static appd_status exact_list(appd_ctx* c, TcState* st, const float* X, int mode, const int* perm,
                              unsigned* count_dev, int k, u64* WCM) {
  const int nch = (int)((st->n + 31) / 32);
  appd_status s;
  unsigned cnt;
  unsigned* runs = (unsigned*)ws(c, S_TC_RUNS, sizeof(unsigned) * 6 * (nch + 2));
  if (!runs) return fail(c, APPD_ERR_OUT_OF_MEMORY, "list runs");
  unsigned *run_lo = runs, *run_nb = runs + (nch + 2), *item_start = runs + 2 * (nch + 2);
  unsigned *hist = runs + 3 * (nch + 2), *offs = runs + 4 * (nch + 2), *cursor = runs + 5 * (nch + 2);
  // counting sort by chunk on the device (no host round trip); the count is read at a
  // later synchronisation for the statistics (and the component-matrix overflow check)
  cnt = st->list_entries_cap;  // capacity bound; the kernels read the real count on the device
  APPD_PUBLISH(c, c->pinned_small + 16, count_dev, sizeof(unsigned));
  int4* items = (int4*)ws(c, S_TC_ITEMS, sizeof(int4) * ((size_t)cnt / 128 + nch + 8));
  if (!items) return fail(c, APPD_ERR_OUT_OF_MEMORY, "list items");
  if ((s = launch_list_counting(c, st->lista, count_dev, cnt, nch, hist, offs, cursor, st->listb, run_lo, run_nb,
                                item_start, items, mode == 1)))
    return s;
  ListParams L;
  memset(&L, 0, sizeof L);
  L.list = st->listb;
  L.count = count_dev;
  L.cap = cnt;
  L.nch = nch;
  L.n = (int)st->n;
  L.d = (int)st->d;
  L.X = X;
  L.perm = perm;
  L.run_lo = run_lo;
  L.run_nb = run_nb;
  L.item_start = item_start;
  L.items = items;
  L.UBK = st->UBK;
  L.tsc = st->dscale;
  L.cnt = st->cand_cnt;
  L.cand = st->cand;
  L.ccap = st->cap;
  L.sc = st->sc;
  L.k = k;
  L.WCM = WCM;
  return launch_list_exact(c, mode, L, nullptr, run_nb, item_start);
}

// Queue the exact re-scan of the next round's flagged rows BEFORE the round's host
// synchronisation (the lookup fused into the contraction left their list and count on the
// device): the GPU works while the host wakes up.  The kernel does nothing if the rows
// turn out to need the tensor-core pass (count > kSmallRescan); if the next step is the
// component matrix its result is simply not used.
appd_status tcf_speculate_rows(appd_ctx* c, TcState* st, const int* comp, u64* compbest) {
  st->rows_spec = true;
  return launch_rows_exact(c, st->XT, st->npad, (int)st->n, (int)st->d, st->rows_list, st->counters + 3, kSmallRescan,
                           comp, compbest);
}

// Queue the cache lookup of the next round (compbest must hold KEY_NONE): per-row first
// eligible cached key -> compbest, flagged rows -> rows_list; the count lands in
// pinned_small[9] at the caller's next synchronisation.
appd_status tcf_lookup_async(appd_ctx* c, TcState* st, const int* comp, u64* compbest) {
  APPD_CUDA(c, cudaMemsetAsync(st->counters, 0, 64, c->stream));
  appd_status s = launch_cache_lookup(c, (int)st->cache_r0, (int)st->cache_r1, st->topk, (int)st->n, st->ckey, st->cj,
                                      st->ccnt, comp, compbest, st->need, st->counters + 3, st->rows_list);
  if (s) return s;
  APPD_PUBLISH(c, c->pinned_small + 9, st->counters + 3, sizeof(unsigned));
  st->lookup_pending = true;
  return APPD_OK;
}

// One Boruvka round's scan: compbest[comp] = min over the component's rows of the exact
// edge key.  With the candidate cache (st->topk > 0): round 0 builds the cache on the
// tensor cores (32-column maxima) and takes every row's minimum from it; later rounds
// serve rows from the cache and re-scan (tensor cores, 128-column maxima) only the
// 512-row blocks holding rows whose cache cannot decide.  Without the cache every
// round scans all of this rank's rows.
appd_status tcf_round(appd_ctx* c, TcState* st, const float* X, const int* comp, int round, int64_t k,
                      u64* compbest, int64_t rb_begin, int64_t rb_end, bool* overflowed) {
  const int64_t n = st->n;
  const int grid_n = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
  const int T = (int)(st->npad / TC_ROWS);
  const bool cache = st->topk > 0;
  appd_status s;
  *overflowed = false;
  st->scanned = false;
  st->last_rescan_rows = 0;
  st->last_rescan_blocks = 0;
  st->h_counters[0] = st->h_counters[1] = st->h_counters[2] = 0;
  c->pinned_small[8] = 0;
  unsigned rescan_rows = 0;
  if (cache && round > 0) {
    if (!st->lookup_pending) {
      if ((s = tcf_lookup_async(c, st, comp, compbest))) return s;
      APPD_SYNC(c);
    }
    st->lookup_pending = false;  // the caller synchronised after queueing it
    const bool spec = st->rows_spec;
    st->rows_spec = false;
    rescan_rows = c->pinned_small[9];
    st->last_rescan_rows = rescan_rows;
    if (rescan_rows == 0) return APPD_OK;  // every component decided by the cache
    if (rescan_rows <= (unsigned)kSmallRescan)  // a few rows: exact FP32 rows, no permutation / tensor pass
      return spec ? APPD_OK  // already queued before the synchronisation (tcf_speculate_rows)
                  : launch_rows_exact(c, st->XT, st->npad, (int)n, (int)st->d, st->rows_list, st->counters + 3,
                                      (int)rescan_rows, comp, compbest);
  }
  const bool packed = round == 0 && st->r0_packed;  // done by the cooperative preparation
  st->r0_packed = false;
  if (round == 0) {
    if (!packed && (s = launch_iota(c, st->perm, n))) return s;
  } else {
    if ((s = sort_by_component(c, st, comp, k, grid_n))) return s;
  }
  // round 0 of the cache: the permutation is the identity, so the transpose is the
  // original-order one the exact row kernel reads
  if (!packed) {
    InitList init;  // (UB ~3.4e38: permissive)
    init.add(st->UB, st->npad, 0x7F7F7F7Fu, 0);
    init.add(st->counters, 16, 0, 0);
    init.add(st->rowflag, n, 0, 0);
    if ((s = tcf_pack(c, st, X, (cache && round == 0) ? st->XT : st->XTp, &init))) return s;
    host_mark("tcf_round: pack queued");
  }
  TcParams P;
  fill_scan_params(st, &P);
  P.round0 = round == 0;
  const int p_begin = (int)(rb_begin * TC_ROWS);
  const int p_end = (int)std::min<int64_t>(rb_end * TC_ROWS, n);
  ExactParams E;

  if (cache && round == 0) {
    // ---- cache-building scan: 32-column maxima of every row of this rank ----
    P.rb_begin = (int)rb_begin;
    P.rb_end = (int)rb_end;
    P.seg32 = 1;
    if (dev_env("APPD_TC_BENCH")) {  // debug: time the scan variants in isolation (results discarded)
      const char* names[] = {"seg64", "seg32", "", "null-epilogue", "tmem-load-only", "no-B-copies", "null+noB"};
      for (int pass : {0, 1, 3, 4, 5, 6}) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; rep++) {
          cudaEventRecord(c->ev[14], c->stream);
          if ((s = launch_tcf_scan(c, pass, P))) return s;
          cudaEventRecord(c->ev[15], c->stream);
          cudaEventSynchronize(c->ev[15]);
          float ms = 0.0f;
          cudaEventElapsedTime(&ms, c->ev[14], c->ev[15]);
          best = std::min(best, ms);
        }
        fprintf(stderr, "[appd] tc bench %-16s %.3f ms\n", names[pass], best);
      }
    }
    if (c->opt.timing) cudaEventRecord(c->ev[10], c->stream);
    if ((s = launch_tcf_scan(c, 1, P))) return s;
  host_mark("tcf_round: tc scan r0 queued");
    if (c->opt.timing) cudaEventRecord(c->ev[11], c->stream);
    st->scanned = true;
    if (p_end > p_begin) {
      const int nch = (int)(st->npad / 32);
      if (!packed) APPD_CUDA(c, cudaMemsetAsync(st->cand_cnt, 0, sizeof(unsigned) * st->npad, c->stream));
      if ((s = launch_topk_scan(c, st->topk, static_cast<const __half*>(st->TM), nch, p_begin, p_end, st->nrm, st->len,
                                st->dscale, st->err, reinterpret_cast<const float*>(st->maxerr), P.em, st->UBK,
                                st->lista, st->counters + 6,
                                st->list_entries_cap, st->cand_cnt)))
        return s;
      host_mark("tcf_round: topk scan queued");
      if ((s = exact_list(c, st, X, 0, nullptr, st->counters + 6, 0, nullptr))) return s;
  host_mark("tcf_round: exact_list queued");
      if ((s = launch_topk_select(c, p_begin, p_end, (int)n, st->topk, st->cand_cnt, st->cand, st->cap, st->ckey,
                                  st->cj, st->ccnt, compbest, st->fallback, st->counters + 0)))
        return s;
      // rows whose candidate list overflowed: exact minimum over the whole row (singletons)
      if ((s = launch_rows_exact(c, st->XT, st->npad, (int)n, (int)st->d, st->fallback, st->counters + 0,
                                 p_end - p_begin, nullptr, compbest)))
        return s;
    }
    st->cache_r0 = p_begin;
    st->cache_r1 = p_end;
    // rows outside this rank's cache are never flagged (multi-rank: need[] is read for all rows)
    if (!packed) APPD_CUDA(c, cudaMemsetAsync(st->need, 0, sizeof(int) * n, c->stream));
  } else if (cache) {
    // ---- re-scan of the blocks holding flagged rows ----
    APPD_CUDA(c, cudaMemsetAsync(st->blockflag, 0, sizeof(int) * (2 * (T + 1) + 8), c->stream));
    if ((s = launch_rescan_blocks(c, (int)n, st->perm, st->need, st->needp, st->blockflag, T, st->rb_list,
                                  st->rb_count)))
      return s;
    P.rb_list = st->rb_list;
    P.rb_count = st->rb_count;
    P.rb_begin = 0;
    P.rb_end = (int)std::min<int64_t>(T, rescan_rows);  // upper bound on the listed blocks (grid sizing)
    if (c->opt.timing) cudaEventRecord(c->ev[10], c->stream);
    if ((s = launch_tcf_scan(c, 0, P))) return s;
    if (c->opt.timing) cudaEventRecord(c->ev[11], c->stream);
    st->scanned = true;
    if ((s = launch_comp_ub(c, (int)n, (int)k, compbest, st->dscale, st->perm, st->needp, st->UB, comp, st->compUB)))
      return s;
    exact_params(st, P, comp, compbest, 0, (int)n, 0, &E);
    E.needp = st->needp;
    E.compUB = st->compUB;
    if ((s = exact_stage(c, E))) return s;
    APPD_PUBLISH(c, c->pinned_small + 8, st->rb_count, sizeof(unsigned));
  } else {
    // ---- no cache: every row of this rank ----
    P.rb_begin = (int)rb_begin;
    P.rb_end = (int)rb_end;
    if (c->opt.timing) cudaEventRecord(c->ev[10], c->stream);
    if ((s = launch_tcf_scan(c, 0, P))) return s;
    if (c->opt.timing) cudaEventRecord(c->ev[11], c->stream);
    st->scanned = true;
    exact_params(st, P, comp, compbest, p_begin, p_end, round == 0, &E);
    if ((s = exact_stage(c, E))) return s;
  }
  // statistics land in pinned memory; read after the round's stream synchronisation
  APPD_PUBLISH(c, st->h_counters, st->counters, 8 * sizeof(unsigned));
  return APPD_OK;
}

// Component-matrix finish (k_cache.cu): one tensor-core pass over this rank's rows,
// then WCM[C][D] = exact minimum edge key between components C and D (k x k, device).
// *listed_overflow is set when the candidate list overflowed (the caller then runs an
// ordinary round instead).
// check_now: synchronise and report a listing overflow here (multi-rank: every rank must
// agree before the reduction); otherwise the overflow is detected on the device by the
// contracted-graph Prim (k_cm_prim) and reported at the caller's final synchronisation
appd_status tcf_cm(appd_ctx* c, TcState* st, const float* X, const int* comp, int64_t k, u64* WCM,
                   int64_t rb_begin, int64_t rb_end, bool* listed_overflow, bool check_now) {
  const int64_t n = st->n;
  const int grid_n = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
  appd_status s;
  *listed_overflow = false;
  if ((s = sort_by_component(c, st, comp, k, grid_n))) return s;
  unsigned* CUB = st->compUB;  // k x k <= 128 x 128 words (the buffer holds n >= k^2 words or more)
  {
    InitList init;
    init.add(st->counters, 16, 0, 0);
    init.add(CUB, k * k, 0x7F7F7F7Fu, 0);  // ~3.4e38: permissive
    init.add(WCM, k * k, KEY_NONE, 1);
    if ((s = tcf_pack(c, st, X, nullptr, &init))) return s;  // the component-matrix kernels read X
  }
  TcParams P;
  fill_scan_params(st, &P);
  P.round0 = 0;
  P.rb_begin = (int)rb_begin;
  P.rb_end = (int)rb_end;
  // one rank: every unordered pair is needed from one side only -> upper-triangle pass
  P.upper = !c->coll && !dev_env("APPD_CM_FULL");
  if (c->opt.timing) cudaEventRecord(c->ev[10], c->stream);
  if ((s = launch_tcf_scan(c, 7, P))) return s;
  if (c->opt.timing) cudaEventRecord(c->ev[11], c->stream);
  CmParams C;
  memset(&C, 0, sizeof C);
  C.TM = static_cast<const float*>(st->TM);
  C.ld = st->npad;
  C.nseg = (int)(st->npad / TC_TMG);
  C.n = (int)n;
  C.k = (int)k;
  C.p_begin = (int)(rb_begin * TC_ROWS);
  C.p_end = (int)std::min<int64_t>(rb_end * TC_ROWS, n);
  C.sc = st->sc;
  C.cstart = st->cstart;
  C.cend = st->cend;
  C.nrm = st->nrm;
  C.len = st->len;
  C.seg_maxlen = st->seg_maxlen;
  C.tsc = st->dscale;
  C.err = st->err;
  C.maxerr = reinterpret_cast<const float*>(st->maxerr);
  C.em = P.em;
  C.CUB = CUB;
  C.list = st->lista;
  C.list_cap = st->list_entries_cap;
  C.counters = st->counters;
  C.XTp = st->XTp;
  C.d = (int)st->d;
  C.perm = st->perm;
  C.WCM = WCM;
  C.upper = P.upper;
  int2* segd = (int2*)ws(c, S_TC_SEGD, sizeof(int2) * (C.nseg + 1));
  if (!segd) return fail(c, APPD_ERR_OUT_OF_MEMORY, "segment descriptors");
  if ((s = launch_seg_comp(c, st->sc, (int)n, C.nseg, segd))) return s;
  C.segd = segd;
  if ((s = launch_cm_rowub(c, C))) return s;
  // listing thresholds on the device (bound MST + path maxima, k_cache.cu)
  unsigned* T = CUB + 128 * 128;
  if ((s = launch_cm_thresholds(c, CUB, (int)k, T))) return s;
  C.CUB = T;
  if ((s = launch_cm_filter(c, C))) return s;
  if ((s = exact_list(c, st, X, 1, st->perm, st->counters + 1, (int)k, WCM))) return s;
  if (check_now) {
    APPD_SYNC(c);
    st->last_list_entries = c->pinned_small[16];
    if (st->last_list_entries > st->list_entries_cap) *listed_overflow = true;
  }
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// test hook: the raw tensor-core accumulators of the first 512-row block against a
// plain FP32 dot product of the same packed fp16 operands (validates descriptors)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float packed_at(const __half* Y, int K, int64_t p, int k) {
  const int64_t gidx = p / 128;
  const int pl = (int)(p % 128), g = pl / 8, r = pl % 8;
  return __half2float(Y[gidx * 128 * K + (int64_t)g * (K / 8) * 64 + (k / 8) * 64 + r * 8 + (k % 8)]);
}

__global__ void k_ref_gram(const __half* YA, const __half* YB, int K, int64_t npad, float* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)TC_ROWS * npad;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / npad, j = e % npad;
    float s = 0.0f;
    for (int k = 0; k < K; k++) s = fmaf(packed_at(YA, K, r, k), packed_at(YB, K, j, k), s);
    out[e] = s;
  }
}

appd_status tcf_debug_gram(appd_ctx* c, const float* X, int64_t n, int64_t d, float* tc_out, float* ref_out) {
  TcState st;
  appd_status s = tcf_prepare(c, X, n, d, &st);
  if (s) return s;
  if ((s = launch_iota(c, st.perm, n))) return s;
  if ((s = tcf_pack(c, &st, X, nullptr))) return s;
  APPD_CUDA(c, cudaMemsetAsync(st.counters, 0, 64, c->stream));
  TcParams P;
  fill_scan_params(&st, &P);
  P.rb_begin = 0;
  P.rb_end = 1;
  P.round0 = 1;
  P.dump = tc_out;
  if ((s = launch_tcf_scan(c, 2, P))) return s;
  k_ref_gram<<<c->sm_count * 4, 256, 0, c->stream>>>((const __half*)st.YA, (const __half*)st.YB, st.K, st.npad,
                                                      ref_out);
  APPD_LAUNCHED(c);
  APPD_SYNC(c);
  return APPD_OK;
}

}  // namespace appd
