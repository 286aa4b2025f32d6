// k_tcfilter.cu -- points-mode Boruvka rounds on the 5th-gen tensor cores
// (SURVEY §8(a) row a2', "tensor cores for the -2 X^T X term of points-mode
// distance tiles").
//
// Each round needs, for every row i, its lightest edge to another component
// under the exact R1 weights.  Computing R1 for all n^2 pairs costs 2d FP32
// lane-ops per pair; instead the tensor cores compute, in fp16 with fp32
// accumulation,  G'_ij = y^_i . y^_j - |y^_j|^2 / 2  for centred, power-of-2
// scaled, fp16-rounded points y^ (the norm rides in two extra K columns), so
//     Dt_ij = |y^_i|^2 - 2 G'_ij  ~  s^2 |x_i - x_j|^2.
// A rigorous error model (delta, eta, gamma below) turns Dt into an
// upper bound U_ij and a lower bound L_ij of s^2 r_ij (r = the exact R1 value).
//
//   scan (tensor cores): UB_i = min over eligible j of U_ij, and, per row and
//       column range, the 16 largest 32-column chunk maxima of G' (records);
//   exact (CUDA cores): every chunk whose maximum reaches the row's threshold
//       (L <= UB_i) is re-evaluated with the exact R1 chain; these chunks hold
//       every candidate, hence the exact argmin and all its ties.  A row whose
//       records may have missed a qualifying chunk is re-scanned exactly.
// Eligibility (j in another component) is cheap because the points are sorted
// by component every round: a row's ineligible columns form one range.
//
// Scan kernel structure (persistent, one CTA per SM, 10 warps):
//   warp 0: producer -- 1-D bulk async copies (UBLKCP) of the packed fp16 operand
//           tiles into a shared-memory ring, mbarrier completion
//   warp 1: MMA issuer -- tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16
//           slices, accumulators double-buffered in TMEM (2 x 256 columns)
//   warps 2-9: epilogue -- tcgen05.ld 32x32b.x32 (software pipelined), 3-input
//           max trees (FMNMX3), per-row bound and records
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace appd {

constexpr int TC_M = 128, TC_N = 256, TC_MAX_STAGES = 8, TC_THREADS = 320, TC_REC = 16;

// Error model (scaled units).  L = |y^_i|, R = max |y^_j| over the columns considered.
//   delta = c1 (L + R) + c2       >= |(y^_i - y^_j) - s (x_i - x_j)|
//   eta   = k1 R (L + R/2) + k2 (L^2 + R^2) + k3 (4 R^2 + (L + R)^2)
//                                 >= |Dt - |y^_i - y^_j|^2|
//   gamma                         >= |r - |x_i - x_j|^2| / |x_i - x_j|^2
// Then  U = (1+gamma) (sqrt(max(Dt + eta, 0)) + delta)^2  >= s^2 r, and
//   L <= UB  is implied by  Dt <= T = (sqrt(UB / (1-gamma)) + delta)^2 + eta.
struct ErrModel {
  float c1, c2, k1, k2, k3, gamma;
};

__device__ __forceinline__ float em_delta(const ErrModel& e, float L, float R) { return e.c1 * (L + R) + e.c2; }
__device__ __forceinline__ float em_eta(const ErrModel& e, float L, float R) {
  return e.k1 * R * (L + 0.5f * R) + e.k2 * (L * L + R * R) + e.k3 * (4.0f * R * R + (L + R) * (L + R));
}
// upper bound on s^2 r for a column whose Dt is dt
__device__ __forceinline__ float em_upper(const ErrModel& e, float dt, float ni, float L, float R) {
  const float r = sqrtf(fmaxf(dt + em_eta(e, L, R), 0.0f)) + em_delta(e, L, R);
  return (1.0f + e.gamma) * r * r * (1.0f + 0x1p-18f) + 0x1p-18f * ni;
}
// G' threshold: a column can hold a candidate only if G' >= thr
__device__ __forceinline__ float em_thr(const ErrModel& e, float ub, float ni, float L, float R) {
  const float r = sqrtf(ub / (1.0f - e.gamma)) + em_delta(e, L, R);
  const float T = (r * r + em_eta(e, L, R)) * (1.0f + 0x1p-18f) + 0x1p-18f * ni;
  return 0.5f * (ni - T);
}

struct TcParams {
  const __half* YA;  // row operand granules (128 points x K, core-matrix layout)
  const __half* YB;  // column operand granules
  const float* nrm;  // |y^_p|^2 (fp32), permuted order
  const float* len;  // |y^_p|
  const float* tile_maxlen;  // max |y^_j| over each 256-column tile
  const int* cs;     // per permuted row: first position of its component
  const int* ce;     // per permuted row: one past the last position
  unsigned* UB;      // per permuted row: upper bound (float bits, >= 0)
  float* rec_v;      // per (row, column split, half): the TC_REC best chunk maxima of G'
  int* rec_c;        // ... and their 32-column chunk indices (-1 = none)
  int n;             // points
  int K;             // padded K (multiple of 16)
  int stages;        // shared-memory ring depth for the column operand
  int row_tiles_begin, row_tiles_end;  // this rank's 128-row tiles (permuted order)
  int col_tiles;     // npad / 256
  int col_splits;
  ErrModel em;
  int round0;        // singletons (eligibility = j != i)
  float* dump;       // PASS 2 (test hook) only
};

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// max of 32 values and an extra one: 16 three-input maxima (FMNMX3)
__device__ __forceinline__ float fmax33(const float (&v)[32], float x) {
  float a0 = fmax3(v[0], v[1], v[2]), a1 = fmax3(v[3], v[4], v[5]), a2 = fmax3(v[6], v[7], v[8]);
  float a3 = fmax3(v[9], v[10], v[11]), a4 = fmax3(v[12], v[13], v[14]), a5 = fmax3(v[15], v[16], v[17]);
  float a6 = fmax3(v[18], v[19], v[20]), a7 = fmax3(v[21], v[22], v[23]), a8 = fmax3(v[24], v[25], v[26]);
  float a9 = fmax3(v[27], v[28], v[29]), a10 = fmax3(v[30], v[31], x);
  float b0 = fmax3(a0, a1, a2), b1 = fmax3(a3, a4, a5), b2 = fmax3(a6, a7, a8), b3 = fmaxf(a9, a10);
  return fmaxf(fmax3(b0, b1, b2), b3);
}

template <int PASS>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tcf_scan(TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = P.K;
  const int NST = P.stages;
  const uint32_t a_bytes = TC_M * K * 2;
  const uint32_t b_bytes = TC_N * K * 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)NST * b_bytes);
  uint64_t* full = bars;          // [NST]
  uint64_t* empty = bars + NST;   // [NST]
  uint64_t* afull = bars + 2 * NST;
  uint64_t* aempty = afull + 1;
  uint64_t* tfull = aempty + 1;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; s++) { ptx::mbar_init(full + s, 1); ptx::mbar_init(empty + s, 1); }
    ptx::mbar_init(afull, 1);
    ptx::mbar_init(aempty, 1);
    for (int b = 0; b < 2; b++) { ptx::mbar_init(tfull + b, 1); ptx::mbar_init(tempty + b, 8); }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int row_tiles = P.row_tiles_end - P.row_tiles_begin;
  const int items = row_tiles * P.col_splits;
  const int per_split = (P.col_tiles + P.col_splits - 1) / P.col_splits;
  const size_t gran_bytes = (size_t)TC_M * K * 2;  // one 128-point granule

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, aph = 0;
      bool first = true;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int rt = P.row_tiles_begin + it / P.col_splits;
        const int sp = it % P.col_splits;
        const int ct0 = sp * per_split;
        const int ct1 = min(P.col_tiles, ct0 + per_split);
        if (!first) { ptx::mbar_wait(aempty, aph); aph ^= 1; }
        first = false;
        ptx::mbar_expect_tx(afull, a_bytes);
        ptx::bulk_g2s(sA, reinterpret_cast<const uint8_t*>(P.YA) + (size_t)rt * gran_bytes, a_bytes, afull);
        for (int ct = ct0; ct < ct1; ct++) {
          ptx::mbar_wait(empty + stage, ph ^ 1);
          ptx::mbar_expect_tx(full + stage, b_bytes);
          ptx::bulk_g2s(sB + stage * b_bytes, reinterpret_cast<const uint8_t*>(P.YB) + (size_t)ct * 2 * gran_bytes,
                        b_bytes, full + stage);
          if (++stage == NST) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_f16_f32(TC_M, TC_N);
      const uint32_t sbo = (uint32_t)(K / 8) * 128u;
      const uint32_t a0 = ptx::smem_u32(sA);
      const uint32_t b0 = ptx::smem_u32(sB);
      int stage = 0, buf = 0;
      uint32_t ph = 0, aph = 0, tph[2] = {0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int sp = it % P.col_splits;
        const int ct0 = sp * per_split;
        const int ct1 = min(P.col_tiles, ct0 + per_split);
        ptx::mbar_wait(afull, aph);
        aph ^= 1;
        for (int ct = ct0; ct < ct1; ct++) {
          ptx::mbar_wait(tempty + buf, tph[buf] ^ 1);
          tph[buf] ^= 1;
          ptx::mbar_wait(full + stage, ph);
          ptx::tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * TC_N);
          const uint32_t bs = b0 + stage * b_bytes;
          for (int ks = 0; ks < K / 16; ks++) {
            const uint64_t ad = ptx::sdesc(a0 + ks * 256, 128, sbo);
            const uint64_t bd = ptx::sdesc(bs + ks * 256, 128, sbo);
            ptx::mma_f16(d, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
          ptx::mma_commit(empty + stage);  // smem stage free once these MMAs complete
          ptx::mma_commit(tfull + buf);    // accumulator ready
          if (++stage == NST) { stage = 0; ph ^= 1; }
          buf ^= 1;
        }
        ptx::mma_commit(aempty);  // row operand free after the item's last MMA
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9) ----------------
    // warp w may only read TMEM lanes 32*(w%4) .. +31; two warps share each lane
    // quarter (rows) and split the 256 columns of a tile into halves of 4 chunks.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int rloc = q * 32 + lane;
    int buf = 0;
    uint32_t tph[2] = {0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int rt = P.row_tiles_begin + it / P.col_splits;
      const int sp = it % P.col_splits;
      const int ct0 = sp * per_split;
      const int ct1 = min(P.col_tiles, ct0 + per_split);
      const int p = rt * TC_M + rloc;
      const bool valid = p < P.n;
      const float ni = valid ? P.nrm[p] : 0.0f;
      const float li = valid ? P.len[p] : 0.0f;
      const int cs = valid ? (P.round0 ? p : P.cs[p]) : 0;
      const int ce = valid ? (P.round0 ? p + 1 : P.ce[p]) : 0;
      float ub = INFINITY;
      float rv[TC_REC];
      int rc[TC_REC];
#pragma unroll
      for (int s = 0; s < TC_REC; s++) { rv[s] = -INFINITY; rc[s] = -1; }

      // one chunk of 32 columns: eligible maximum, tile maximum, records
      auto process = [&](float (&v)[32], int q0, bool fast_half, float& tmax) {
        if (PASS == 2) {  // test hook: raw accumulator dump of the CTA's first item
          if (it == (int)blockIdx.x && P.dump)
#pragma unroll
            for (int t = 0; t < 32; t++) P.dump[(int64_t)rloc * P.col_tiles * TC_N + q0 + t] = v[t];
          return;
        }
        float m;
        if (fast_half) {
          m = fmax33(v, -INFINITY);
        } else {
          const bool skip = q0 >= cs && q0 + 32 <= ce;
          m = -INFINITY;
          if (!skip && valid) {
#pragma unroll
            for (int t = 0; t < 32; t++) {
              const int qq = q0 + t;
              const bool el = (qq < cs || qq >= ce) && qq < P.n;
              m = fmaxf(m, el ? v[t] : -INFINITY);
            }
          }
        }
        tmax = fmaxf(tmax, m);
        if (m > rv[TC_REC - 1]) {  // insert (value, chunk) into the descending records
          float val = m;
          int id = q0 >> 5;
#pragma unroll
          for (int s = 0; s < TC_REC; s++) {
            if (val > rv[s]) {
              const float tv = rv[s];
              const int ti = rc[s];
              rv[s] = val;
              rc[s] = id;
              val = tv;
              id = ti;
            }
          }
        }
      };

      for (int ct = ct0; ct < ct1; ct++) {
        ptx::mbar_wait(tfull + buf, tph[buf]);
        tph[buf] ^= 1;
        ptx::tc_fence_after();
        const int h0 = ct * TC_N + half * 128;  // first column of this warp's half tile
        // warp-uniform fast path: every lane's row is valid and its component range
        // misses these 128 columns, which are all real points
        const bool lane_fast = valid && (h0 + 128 <= cs || h0 >= ce) && h0 + 128 <= P.n;
        const bool fast_half = __all_sync(0xffffffffu, lane_fast);
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TC_N + half * 128);
        float tmax = -INFINITY;
        float va[32], vb[32];
        // software pipeline: the TMEM load of chunk c+1 is in flight while chunk c is processed
        ptx::tmem_ld32(tbase, va);
        ptx::tmem_ld_wait();
        ptx::reg_fence(va);
        ptx::tmem_ld32(tbase + 32, vb);
        process(va, h0, fast_half, tmax);
        ptx::tmem_ld_wait();
        ptx::reg_fence(vb);
        ptx::tmem_ld32(tbase + 64, va);
        process(vb, h0 + 32, fast_half, tmax);
        ptx::tmem_ld_wait();
        ptx::reg_fence(va);
        ptx::tmem_ld32(tbase + 96, vb);
        process(va, h0 + 64, fast_half, tmax);
        ptx::tmem_ld_wait();
        ptx::reg_fence(vb);
        process(vb, h0 + 96, fast_half, tmax);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty + buf);
        buf ^= 1;
        if (PASS == 0 && valid && tmax > -INFINITY)
          ub = fminf(ub, em_upper(P.em, ni - 2.0f * tmax, ni, li, P.tile_maxlen[ct]));
      }
      if (PASS == 0 && valid) {
        if (ub < INFINITY) atomicMin(P.UB + p, __float_as_uint(fmaxf(ub, 0.0f)));
        const int nl = P.col_splits * 2;
        const int64_t base = ((int64_t)p * nl + sp * 2 + half) * TC_REC;
#pragma unroll
        for (int s = 0; s < TC_REC; s++) {
          P.rec_v[base + s] = rv[s];
          P.rec_c[base + s] = rc[s];
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

size_t tcf_smem_bytes(int K, int stages) {
  return (size_t)TC_M * K * 2 + (size_t)stages * TC_N * K * 2 + (2 * TC_MAX_STAGES + 6) * 8 + 16;
}

// deepest ring (<= 4) that fits 227 KB of shared memory; 0 if K does not fit
int tcf_stages(int K) {
  for (int s = 4; s >= 2; s--)
    if (tcf_smem_bytes(K, s) <= 227 * 1024) return s;
  return 0;
}

appd_status launch_tcf_scan(appd_ctx* c, int pass, const TcParams& P) {
  // at least 120 KB so that exactly one CTA (and one 512-column TMEM allocation) fits per SM
  size_t smem = tcf_smem_bytes(P.K, P.stages);
  if (smem < 120 * 1024) smem = 120 * 1024;
  static int attr_done = 0;
  if (!attr_done) {
    cudaFuncSetAttribute(k_tcf_scan<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_tcf_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = 1;
  }
  const int items = (P.row_tiles_end - P.row_tiles_begin) * P.col_splits;
  int grid = c->sm_count < items ? c->sm_count : items;
  if (grid < 1) return APPD_OK;
  if (pass == 0) k_tcf_scan<0><<<grid, TC_THREADS, smem, c->stream>>>(P);
  else k_tcf_scan<2><<<1, TC_THREADS, smem, c->stream>>>(P);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// preparation kernels
// ---------------------------------------------------------------------------

// per-block partial column sums (fp64), fixed partition => deterministic
__global__ void k_center_partial(const float* __restrict__ X, int64_t n, int d, int rows_per_block,
                                 double* __restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(n, r0 + rows_per_block);
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; r++) s += (double)X[r * d + k];
    part[(int64_t)blockIdx.x * d + k] = s;
  }
}
__global__ void k_center_final(const double* __restrict__ part, int blocks, int64_t n, int d, float* __restrict__ c) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < blocks; b++) s += part[(int64_t)b * d + k];
    c[k] = (float)(s / (double)n);
  }
}
// max |x_i - c| (fp32, order independent)
__global__ void k_maxlen(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ c,
                         unsigned* __restrict__ out) {
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  float best = 0.0f;
  for (int64_t i = (int64_t)blockIdx.x * warps + w; i < n; i += (int64_t)gridDim.x * warps) {
    float s = 0.0f;
    for (int k = lane; k < d; k += 32) {
      float t = X[i * d + k] - c[k];
      s += t * t;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    best = fmaxf(best, s);
  }
  if (lane == 0) atomicMax(out, __float_as_uint(sqrtf(best)));
}

// pack point perm[p] into the row (YA) and column (YB) operand granules:
// element (p, k) at granule p/128, byte offset g*(K/8)*128 + (k/8)*128 + r*16 + (k%8)*2
// with g = (p%128)/8, r = p%8.  y^ = fp16(scale * (x - c)); K columns: [y^ (d), pad to dk,
// then A: 1, 1, 0..; B: hi(-|y^|^2/2), lo(-|y^|^2/2), 0..].  Padding points: A = 0, B aug = -65504.
__global__ void k_pack(const float* __restrict__ X, int64_t n, int d, int dk, int K, const int* __restrict__ perm,
                       const float* __restrict__ c, float scale, int64_t npad, __half* __restrict__ YA,
                       __half* __restrict__ YB, float* __restrict__ nrm, float* __restrict__ len) {
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int64_t p = (int64_t)blockIdx.x * warps + w; p < npad; p += (int64_t)gridDim.x * warps) {
    const int64_t gidx = p / 128;
    const int pl = (int)(p % 128), g = pl / 8, r = pl % 8;
    __half* ga = YA + gidx * 128 * K;
    __half* gb = YB + gidx * 128 * K;
    const bool real = p < n;
    const int64_t i = real ? perm[p] : 0;
    float s = 0.0f;
    for (int k = lane; k < dk; k += 32) {
      __half h = __float2half_rn(0.0f);
      if (real && k < d) h = __float2half_rn(scale * (X[i * d + k] - c[k]));
      const float hf = __half2float(h);
      s = fmaf(hf, hf, s);
      const int64_t off = (int64_t)g * (K / 8) * 64 + (k / 8) * 64 + r * 8 + (k % 8);  // in halves
      ga[off] = h;
      gb[off] = h;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    for (int k = dk + lane; k < K; k += 32) {
      const int64_t off = (int64_t)g * (K / 8) * 64 + (k / 8) * 64 + r * 8 + (k % 8);
      __half a = __float2half_rn(0.0f), b = __float2half_rn(0.0f);
      if (k == dk || k == dk + 1) {
        if (real) {
          a = __float2half_rn(1.0f);
          const float hn = -0.5f * s;
          const __half hi = __float2half_rn(hn);
          b = (k == dk) ? hi : __float2half_rn(hn - __half2float(hi));
        } else {
          b = (k == dk) ? __float2half_rn(-65504.0f) : __float2half_rn(0.0f);
        }
      }
      ga[off] = a;
      gb[off] = b;
    }
    if (lane == 0) {
      nrm[p] = real ? s : 0.0f;
      len[p] = real ? sqrtf(s) : 0.0f;
    }
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

// max |y^| over each 32-column chunk (the exact pass) and each 256-column tile (the scan)
__global__ void k_chunk_maxlen(const float* __restrict__ len, int64_t npad, float* __restrict__ chunk_max,
                               float* __restrict__ tile_max) {
  const int64_t t = blockIdx.x;  // one tile per block of 256 threads
  float m = len[t * TC_N + threadIdx.x];
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = m;
    chunk_max[t * 8 + (threadIdx.x >> 5)] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float x = red[0];
    for (int i = 1; i < 8; i++) x = fmaxf(x, red[i]);
    tile_max[t] = x;
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
  const float* chunk_maxlen;
  float maxlen;  // max over all points (most permissive threshold, for the overflow test)
  const int* cs;
  const int* ce;
  const unsigned* UB;
  const float* rec_v;
  const int* rec_c;
  int nl;  // record lists per row (column splits x 2)
  int p_begin, p_end;
  int round0;
  ErrModel em;
  const int* comp;  // original-index component labels
  u64* compbest;
  unsigned* counters;  // [0] fallback rows, [2] exact chunks evaluated
  int* fallback;       // permuted rows whose records may have missed a qualifying chunk
};

// One warp per row: every 32-column chunk whose recorded maximum of G' reaches the
// row's threshold holds all of the row's candidates in that chunk; the warp evaluates
// R1 exactly on those columns (one column per lane, coalesced on XTp) and keeps the
// minimum edge key.  If a record list is full and its last entry still qualifies,
// chunks beyond it may qualify too: the row goes to the exact fallback instead.
__global__ void k_exact_chunks(ExactParams E) {
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int p = E.p_begin + blockIdx.x * warps + w; p < E.p_end; p += gridDim.x * warps) {
    const float ub = __uint_as_float(E.UB[p]);
    const float ni = E.nrm[p], li = E.len[p];
    const int cs = E.round0 ? p : E.cs[p];
    const int ce = E.round0 ? p + 1 : E.ce[p];
    const int oi = E.perm[p];
    const float thr_min = em_thr(E.em, ub, ni, li, E.maxlen);
    u64 best = KEY_NONE;
    bool overflow = false;
    unsigned chunks = 0;
    for (int L = 0; L < E.nl && !overflow; L++) {
      const int64_t base = ((int64_t)p * E.nl + L) * TC_REC;
      // records are stored descending: read them one per lane, test in parallel
      const int ch_l = lane < TC_REC ? E.rec_c[base + lane] : -1;
      const float v_l = lane < TC_REC ? E.rec_v[base + lane] : -INFINITY;
      bool qual = ch_l >= 0 && v_l >= em_thr(E.em, ub, ni, li, E.chunk_maxlen[max(ch_l, 0)]);
      if (__shfl_sync(0xffffffffu, (int)(ch_l >= 0 && v_l >= thr_min), TC_REC - 1)) overflow = true;
      unsigned mask = __ballot_sync(0xffffffffu, qual);
      while (mask && !overflow) {
        const int s = __ffs(mask) - 1;
        mask &= mask - 1;
        const int ch = __shfl_sync(0xffffffffu, ch_l, s);
        chunks++;
        const int qcol = ch * 32 + lane;
        if (qcol < E.n && (qcol < cs || qcol >= ce)) {
          float acc = 0.0f;
          const float* xi = E.XTp + p;
          const float* xj = E.XTp + qcol;
          for (int k = 0; k < E.d; k++) {
            const float t = __fsub_rn(__ldg(xi + (int64_t)k * E.npad), __ldg(xj + (int64_t)k * E.npad));
            acc = __fmaf_rn(t, t, acc);
          }
          const u64 key = ((u64)(__float_as_uint(acc) & 0x7FFFFFFFu) << 33) | tri_index(oi, E.perm[qcol]);
          best = key < best ? key : best;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    if (lane == 0) {
      if (chunks) atomicAdd(E.counters + 2, chunks);
      if (overflow) {
        const unsigned slot = atomicAdd(E.counters, 1u);
        E.fallback[slot] = p;  // capacity n
      } else if (best != KEY_NONE) {
        atomicMin(E.compbest + E.comp[oi], best);
      }
    }
  }
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
      if (best != KEY_NONE) atomicMin(E.compbest + E.comp[oi], best);
    }
    __syncthreads();
  }
}

int64_t tcf_row_tiles(const TcState* st) { return st->npad / TC_M; }

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

appd_status tcf_prepare(appd_ctx* c, const float* X, int64_t n, int64_t d, TcState* st) {
  st->n = n;
  st->d = d;
  st->npad = (n + TC_N - 1) / TC_N * TC_N;
  st->dk = (int)((d + 15) / 16 * 16);
  st->K = st->dk + 16;
  st->stages = tcf_stages(st->K);
  if (st->stages == 0) return APPD_ERR_UNSUPPORTED;
  const int blocks = (int)((n + 255) / 256);
  double* part = (double*)ws(c, S_TC_PART, sizeof(double) * blocks * d);
  st->center = (float*)ws(c, S_TC_CENTER, sizeof(float) * (d + 1) + 64);
  if (!part || !st->center) return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc center");
  k_center_partial<<<blocks, 128, 0, c->stream>>>(X, n, (int)d, 256, part);
  APPD_LAUNCHED(c);
  k_center_final<<<(unsigned)((d + 127) / 128), 128, 0, c->stream>>>(part, blocks, n, (int)d, st->center);
  APPD_LAUNCHED(c);
  unsigned* maxlen = (unsigned*)(st->center + d);
  APPD_CUDA(c, cudaMemsetAsync(maxlen, 0, sizeof(unsigned), c->stream));
  k_maxlen<<<c->sm_count * 4, 256, 0, c->stream>>>(X, n, (int)d, st->center, maxlen);
  APPD_LAUNCHED(c);
  APPD_CUDA(c, cudaMemcpyAsync(c->pinned_small + 32, maxlen, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  APPD_CUDA(c, cudaStreamSynchronize(c->stream));
  float ml;
  memcpy(&ml, c->pinned_small + 32, 4);
  if (!(ml < INFINITY)) return APPD_ERR_UNSUPPORTED;  // coordinates too large for the filter
  // scale = 2^e with scale * max|y| in [2^6.5, 2^7.5): |y^|^2 < 2^15, fp16 range safe
  int e = 0;
  if (ml > 0.0f) {
    e = (int)std::floor(7.0 - std::log2((double)ml) + 0.5);
    e = std::max(-100, std::min(100, e));
  }
  st->scale = (float)std::ldexp(1.0, e);
  // fp16 rounding can lift |y^| by 2^-11 relative (plus subnormal slack)
  st->maxlen_scaled = (float)((double)ml * st->scale * (1.0 + std::ldexp(1.0, -10)) + 1e-6);
  // Error model in scaled units:
  //  delta: each fp16 coordinate is within 2^-11 (relative, normal range) or 2^-25
  //    (absolute, subnormal) of s*(x - c); centring x - c in fp32 adds 2^-24 relative;
  //    so |(y^_i - y^_j) - s (x_i - x_j)| <= (2^-11 + 2^-20)(L + R) + 2 sqrt(d) 2^-25.
  //  eta: Dt = |y^_i|^2 - 2 G' with G' accumulated in fp32 over K terms (<= K ulp-of-
  //    sum, allowing one ulp of truncation per addition: K 2^-23 sum|terms|), the fp16
  //    hi/lo split of -|y^_j|^2/2 (2^-22 |y^_j|^2), fp32 norms of d exact products
  //    (d 2^-24 |y|^2 each) and the final subtraction (2^-24 |Dt|):
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
  st->tile_maxlen = (float*)ws(c, S_TC_TML, sizeof(float) * (st->npad / TC_N));
  st->chunk_maxlen = (float*)ws(c, S_TC_CML, sizeof(float) * (st->npad / 32));
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
  if (!st->YA || !st->YB || !st->XTp || !st->nrm || !st->len || !st->tile_maxlen || !st->chunk_maxlen ||
      !st->perm || !st->sc || !st->keys || !st->cstart || !st->cend || !st->rs || !st->re || !st->UB ||
      !st->counters || !st->fallback)
    return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc workspace");
  return APPD_OK;
}

static appd_status tcf_pack(appd_ctx* c, TcState* st, const float* X) {
  const int64_t n = st->n;
  k_pack<<<c->sm_count * 8, 256, 0, c->stream>>>(X, n, (int)st->d, st->dk, st->K, st->perm, st->center, st->scale,
                                                  st->npad, (__half*)st->YA, (__half*)st->YB, st->nrm, st->len);
  APPD_LAUNCHED(c);
  dim3 tg((unsigned)(st->npad / 32), (unsigned)((st->d + 31) / 32));
  k_transpose_perm<<<tg, dim3(32, 8), 0, c->stream>>>(X, n, (int)st->d, st->perm, st->npad, st->XTp);
  APPD_LAUNCHED(c);
  k_chunk_maxlen<<<(unsigned)(st->npad / TC_N), TC_N, 0, c->stream>>>(st->len, st->npad, st->chunk_maxlen,
                                                                        st->tile_maxlen);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// one Boruvka round's scan: compbest[comp] = min over the component's rows of the exact edge key
appd_status tcf_round(appd_ctx* c, TcState* st, const float* X, const int* comp, int round, u64* compbest,
                      int64_t row_tile_begin, int64_t row_tile_end, bool* overflowed) {
  const int64_t n = st->n;
  const int grid_n = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
  appd_status s;
  if (round == 0) {
    if ((s = launch_iota(c, st->perm, n))) return s;
  } else {
    k_gather_comp<<<grid_n, 256, 0, c->stream>>>(comp, n, st->keys, st->keys + n + 1);
    APPD_LAUNCHED(c);
    if ((s = sort_pairs_i32(c, st->keys, st->sc, st->keys + n + 1, st->perm, n))) return s;
    k_comp_ranges<<<grid_n, 256, 0, c->stream>>>(st->sc, n, st->cstart, st->cend);
    APPD_LAUNCHED(c);
    k_row_ranges<<<grid_n, 256, 0, c->stream>>>(st->sc, n, st->cstart, st->cend, st->rs, st->re);
    APPD_LAUNCHED(c);
  }
  if ((s = tcf_pack(c, st, X))) return s;
  APPD_CUDA(c, cudaMemsetAsync(st->UB, 0x7F, sizeof(unsigned) * st->npad, c->stream));  // ~3.4e38
  APPD_CUDA(c, cudaMemsetAsync(st->counters, 0, 64, c->stream));
  TcParams P;
  memset(&P, 0, sizeof P);
  P.YA = (const __half*)st->YA;
  P.YB = (const __half*)st->YB;
  P.nrm = st->nrm;
  P.len = st->len;
  P.tile_maxlen = st->tile_maxlen;
  P.cs = st->rs;
  P.ce = st->re;
  P.UB = st->UB;
  P.n = (int)n;
  P.K = st->K;
  P.stages = st->stages;
  P.row_tiles_begin = (int)row_tile_begin;
  P.row_tiles_end = (int)row_tile_end;
  P.col_tiles = (int)(st->npad / TC_N);
  const int64_t rt = row_tile_end - row_tile_begin;
  int splits = (int)std::max<int64_t>(1, (c->sm_count * 4 + rt - 1) / std::max<int64_t>(rt, 1));
  if (splits > P.col_tiles) splits = P.col_tiles;
  P.col_splits = splits;
  const int nl = 2 * splits;
  P.rec_v = (float*)ws(c, S_TC_RECV, sizeof(float) * st->npad * nl * TC_REC);
  P.rec_c = (int*)ws(c, S_TC_RECC, sizeof(int) * st->npad * nl * TC_REC);
  if (!P.rec_v || !P.rec_c) return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc records");
  P.em = error_model(st);
  P.round0 = round == 0;
  P.dump = nullptr;
  if ((s = launch_tcf_scan(c, 0, P))) return s;

  ExactParams E;
  E.XTp = st->XTp;
  E.npad = st->npad;
  E.d = (int)st->d;
  E.n = (int)n;
  E.perm = st->perm;
  E.nrm = st->nrm;
  E.len = st->len;
  E.chunk_maxlen = st->chunk_maxlen;
  E.maxlen = st->maxlen_scaled;
  E.cs = st->rs;
  E.ce = st->re;
  E.UB = st->UB;
  E.rec_v = P.rec_v;
  E.rec_c = P.rec_c;
  E.nl = nl;
  E.p_begin = (int)(row_tile_begin * TC_M);
  E.p_end = (int)std::min<int64_t>(row_tile_end * TC_M, n);
  E.round0 = round == 0;
  E.em = P.em;
  E.comp = comp;
  E.compbest = compbest;
  E.counters = st->counters;
  E.fallback = st->fallback;
  const int rows = E.p_end - E.p_begin;
  if (rows > 0) {
    k_exact_chunks<<<std::min(c->sm_count * 16, (rows + 7) / 8), 256, 0, c->stream>>>(E);
    APPD_LAUNCHED(c);
    k_exact_rows<<<c->sm_count * 2, 256, 0, c->stream>>>(E);
    APPD_LAUNCHED(c);
  }
  *overflowed = false;
  // statistics land in pinned memory; read after the round's stream synchronisation
  APPD_CUDA(c, cudaMemcpyAsync(st->h_counters, st->counters, 4 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                               c->stream));
  return APPD_OK;
}

// ---------------------------------------------------------------------------
// test hook: the raw tensor-core accumulator of row tile 0 against a plain FP32
// dot product of the same packed fp16 operands (validates descriptors/layouts)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float packed_at(const __half* Y, int K, int64_t p, int k) {
  const int64_t gidx = p / 128;
  const int pl = (int)(p % 128), g = pl / 8, r = pl % 8;
  return __half2float(Y[gidx * 128 * K + (int64_t)g * (K / 8) * 64 + (k / 8) * 64 + r * 8 + (k % 8)]);
}

__global__ void k_ref_gram(const __half* YA, const __half* YB, int K, int64_t npad, float* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 128 * npad;
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
  if ((s = tcf_pack(c, &st, X))) return s;
  TcParams P;
  memset(&P, 0, sizeof P);
  P.YA = (const __half*)st.YA;
  P.YB = (const __half*)st.YB;
  P.nrm = st.nrm;
  P.len = st.len;
  P.tile_maxlen = st.tile_maxlen;
  P.n = (int)n;
  P.K = st.K;
  P.stages = st.stages;
  P.row_tiles_begin = 0;
  P.row_tiles_end = 1;
  P.col_tiles = (int)(st.npad / TC_N);
  P.col_splits = 1;
  P.round0 = 1;
  P.dump = tc_out;
  if ((s = launch_tcf_scan(c, 2, P))) return s;
  k_ref_gram<<<c->sm_count * 4, 256, 0, c->stream>>>((const __half*)st.YA, (const __half*)st.YB, st.K, st.npad,
                                                      ref_out);
  APPD_LAUNCHED(c);
  APPD_CUDA(c, cudaStreamSynchronize(c->stream));
  return APPD_OK;
}

}  // namespace appd
