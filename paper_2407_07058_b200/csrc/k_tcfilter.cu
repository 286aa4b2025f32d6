// k_tcfilter.cu -- points-mode Boruvka round on the 5th-gen tensor cores
// (SURVEY §8(a) row a2', "tensor cores for the -2 X^T X term of points-mode
// distance tiles").
//
// Each round needs, for every row i, its lightest edge to another component
// under the exact R1 weights.  Computing R1 for all n^2 pairs costs 2d FP32
// lane-ops per pair; instead the tensor cores compute, in fp16 with fp32
// accumulation, G'_ij = y^_i . y^_j - |y^_j|^2 / 2 for centred, power-of-2
// scaled, fp16-rounded points y^ (the norm rides in two extra K columns), so
//     |y^_i - y^_j|^2 = |y^_i|^2 - 2 G'_ij.
// A rigorous bound eps_ij >= |s^2 r_ij - (|y^_i|^2 - 2 G'_ij)| (fp16 rounding of
// the inputs, fp32 accumulation, R1's own rounding) gives
//   lower bound  L_ij = |y^_i|^2 - 2 G'_ij - eps_ij,  upper bound U_ij = ... + eps_ij.
// Pass A: UB_i = min_j eligible U_ij.   Pass B: every eligible j with L_ij <= UB_i
// is a candidate (this set contains the row's exact argmin, and all ties), and
// only the candidates are recomputed with the exact R1 chain.  Eligibility
// (j in another component) is cheap because the points are sorted by component
// every round: the ineligible columns of a row form one contiguous range.
//
// Kernel structure (persistent, one CTA per SM, 6 warps):
//   warp 0: producer -- 1-D bulk async copies (UBLKCP) of the packed fp16 operand
//           tiles into a 4-stage shared-memory ring, mbarrier completion
//   warp 1: MMA issuer -- tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16
//           slices, accumulators double-buffered in TMEM (2 x 256 columns)
//   warps 2-5: epilogue -- tcgen05.ld 32x32b.x32, per-row max / candidate test
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace appd {

constexpr int TC_M = 128, TC_N = 256, TC_MAX_STAGES = 8, TC_THREADS = 192;

struct TcParams {
  const __half* YA;  // row operand granules (128 points x K, core-matrix layout)
  const __half* YB;  // column operand granules
  const float* nrm;  // |y^_p|^2 (fp32), permuted order
  const float* len;  // |y^_p|
  const float* tile_maxlen;  // max |y^_j| over each 256-column tile
  const int* cs;  // per permuted row: first position of its component
  const int* ce;  // per permuted row: one past the last position
  const int* perm;  // permuted position -> original index
  unsigned* UB;  // per permuted row: upper bound (float bits, >= 0)
  uint2* cand;  // candidates (orig i, orig j)
  unsigned* cand_count;
  unsigned cand_cap;
  int* overflow;
  int n;     // points
  int K;     // padded K (multiple of 16)
  int stages;  // shared-memory ring depth for the column operand
  int row_tiles_begin, row_tiles_end;  // this rank's 128-row tiles (permuted order)
  int col_tiles;  // npad / 256
  int col_splits;
  // error model, a = |y^_i| + max_{j in T} |y^_j|:
  //   delta = c1 * a + c2 >= |(y^_i - y^_j) - s (x_i - x_j)|   (fp16 inputs, centring)
  //   eta   = c3 * a^2     >= |Dt - |y^_i - y^_j|^2|            (fp32 accumulation, norms)
  //   gamma                >= |r_ij - D_ij| / D_ij              (R1's own rounding)
  float c1, c2, c3, gamma;
  int round0;        // singletons (eligibility = j != i)
  float* dump;       // PASS 2 (test hook) only
};

__device__ __forceinline__ float fmax32(const float (&v)[32]) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = fmaxf(v[i], v[i + 16]);
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = fmaxf(a[i], a[i + 8]);
#pragma unroll
  for (int i = 0; i < 4; i++) a[i] = fmaxf(a[i], a[i + 4]);
  return fmaxf(fmaxf(a[0], a[2]), fmaxf(a[1], a[3]));
}

template <int PASS>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tcf_scan(TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = P.K;
  const int TC_STAGES = P.stages;
  const uint32_t a_bytes = TC_M * K * 2;
  const uint32_t b_bytes = TC_N * K * 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)TC_STAGES * b_bytes);
  uint64_t* full = bars;                  // [STAGES]
  uint64_t* empty = bars + TC_STAGES;     // [STAGES]
  uint64_t* afull = bars + 2 * TC_STAGES;
  uint64_t* aempty = afull + 1;
  uint64_t* tfull = aempty + 1;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; s++) { ptx::mbar_init(full + s, 1); ptx::mbar_init(empty + s, 1); }
    ptx::mbar_init(afull, 1);
    ptx::mbar_init(aempty, 1);
    for (int b = 0; b < 2; b++) { ptx::mbar_init(tfull + b, 1); ptx::mbar_init(tempty + b, 4); }
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
          if (++stage == TC_STAGES) { stage = 0; ph ^= 1; }
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
            uint64_t ad = ptx::sdesc(a0 + ks * 256, 128, sbo);
            uint64_t bd = ptx::sdesc(bs + ks * 256, 128, sbo);
            ptx::mma_f16(d, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
          ptx::mma_commit(empty + stage);  // smem stage free once these MMAs complete
          ptx::mma_commit(tfull + buf);    // accumulator ready
          if (++stage == TC_STAGES) { stage = 0; ph ^= 1; }
          buf ^= 1;
        }
        ptx::mma_commit(aempty);  // row operand free after the item's last MMA
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5: 128 rows) ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
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
      if (PASS == 1 && valid) ub = __uint_as_float(P.UB[p]);
      const int orig_i = (PASS == 1 && valid) ? P.perm[p] : 0;
      for (int ct = ct0; ct < ct1; ct++) {
        ptx::mbar_wait(tfull + buf, tph[buf]);
        tph[buf] ^= 1;
        ptx::tc_fence_after();
        const float a = li + P.tile_maxlen[ct];
        const float dl = P.c1 * a + P.c2;
        const float eta = P.c3 * a * a;
        float thr = 0.0f;
        if (PASS == 1) {
          // candidate iff its lower bound (1-gamma)(sqrt(Dt - eta) - delta)^2 <= UB_i, i.e.
          // Dt = |y^_i|^2 - 2 G' <= T = (sqrt(UB_i / (1-gamma)) + delta)^2 + eta  (+ fp32 slack)
          const float r = sqrtf(ub / (1.0f - P.gamma)) + dl;
          const float T = (r * r + eta) * (1.0f + 0x1p-18f) + 0x1p-18f * ni;
          thr = 0.5f * (ni - T);
        }
        float tmax = -INFINITY;
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TC_N);
#pragma unroll 1
        for (int c = 0; c < TC_N / 32; c++) {
          float v[32];
          ptx::tmem_ld32(tbase + c * 32, v);
          ptx::tmem_ld_wait();
          const int q0 = ct * TC_N + c * 32;
          if (PASS == 2) {  // test hook: raw accumulator dump of the CTA's first row tile
            if (it == (int)blockIdx.x && P.dump)
#pragma unroll
              for (int t = 0; t < 32; t++) P.dump[(int64_t)rloc * P.col_tiles * TC_N + q0 + t] = v[t];
            continue;
          }
          const bool skip = q0 >= cs && q0 + 32 <= ce;
          const bool fast = (q0 + 32 <= cs || q0 >= ce) && q0 + 32 <= P.n;
          const bool mask = valid && !skip && !fast;
          float m;
          if (__any_sync(0xffffffffu, mask)) {
            m = -INFINITY;
#pragma unroll
            for (int t = 0; t < 32; t++) {
              const int qq = q0 + t;
              const bool el = (qq < cs || qq >= ce) && qq < P.n;
              v[t] = el ? v[t] : -INFINITY;
              m = fmaxf(m, v[t]);
            }
          } else {
            m = fmax32(v);
          }
          if (skip || !valid) m = -INFINITY;
          if (PASS == 0) {
            tmax = fmaxf(tmax, m);
          } else {
            const bool hit = valid && m > -INFINITY && m >= thr;
            if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
              for (int t = 0; t < 32; t++) {
                const bool want = hit && v[t] >= thr && !(q0 + t >= cs && q0 + t < ce) && q0 + t < P.n;
                const unsigned bal = __ballot_sync(0xffffffffu, want);
                if (bal) {
                  unsigned base = 0;
                  const int leader = __ffs(bal) - 1;
                  if (lane == leader) base = atomicAdd(P.cand_count, (unsigned)__popc(bal));
                  base = __shfl_sync(0xffffffffu, base, leader);
                  if (want) {
                    unsigned slot = base + __popc(bal & ((1u << lane) - 1u));
                    if (slot < P.cand_cap) P.cand[slot] = make_uint2((unsigned)orig_i, (unsigned)P.perm[q0 + t]);
                    else *P.overflow = 1;
                  }
                }
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty + buf);
        buf ^= 1;
        if (PASS == 0 && tmax > -INFINITY) {
          // upper bound on s^2 r_ij for the tile's best column: (1+gamma)(sqrt(Dt + eta) + delta)^2
          const float dt = ni - 2.0f * tmax;
          const float r = sqrtf(fmaxf(dt + eta, 0.0f)) + dl;
          ub = fminf(ub, (1.0f + P.gamma) * r * r * (1.0f + 0x1p-18f) + 0x1p-18f * ni);
        }
      }
      if (PASS == 0 && valid && ub < INFINITY) atomicMin(P.UB + p, __float_as_uint(fmaxf(ub, 0.0f)));
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
    cudaFuncSetAttribute(k_tcf_scan<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_tcf_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = 1;
  }
  const int items = (P.row_tiles_end - P.row_tiles_begin) * P.col_splits;
  int grid = c->sm_count < items ? c->sm_count : items;
  if (grid < 1) return APPD_OK;
  if (pass == 0) k_tcf_scan<0><<<grid, TC_THREADS, smem, c->stream>>>(P);
  else if (pass == 1) k_tcf_scan<1><<<grid, TC_THREADS, smem, c->stream>>>(P);
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
      float hf = __half2float(h);
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
          float hn = -0.5f * s;
          __half hi = __float2half_rn(hn);
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

__global__ void k_tile_maxlen(const float* __restrict__ len, int64_t npad, float* __restrict__ out) {
  const int64_t t = blockIdx.x;
  float m = 0.0f;
  for (int j = threadIdx.x; j < TC_N; j += blockDim.x) m = fmaxf(m, len[t * TC_N + j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x / 32); i++) m = fmaxf(m, red[i]);
    out[t] = fmaxf(m, red[0]);
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

// exact R1 on every candidate, component minimum of the packed edge key
__global__ void k_exact_candidates(const float* __restrict__ X, int d, const uint2* __restrict__ cand,
                                   const unsigned* __restrict__ count, unsigned cap, const int* __restrict__ comp,
                                   u64* __restrict__ compbest) {
  unsigned cnt = *count;
  if (cnt > cap) cnt = cap;
  // one candidate per thread; the d terms in R1 order
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
    const uint2 ij = cand[e];
    const float* xi = X + (int64_t)ij.x * d;
    const float* xj = X + (int64_t)ij.y * d;
    float acc = 0.0f;
    for (int k = 0; k < d; k++) {
      float t = __fsub_rn(__ldg(xi + k), __ldg(xj + k));
      acc = __fmaf_rn(t, t, acc);
    }
    const u64 key = ((u64)(__float_as_uint(acc) & 0x7FFFFFFFu) << 33) | tri_index(ij.x, ij.y);
    atomicMin(compbest + comp[ij.x], key);
  }
}

int64_t tcf_row_tiles(const TcState* st) { return st->npad / TC_M; }

// ---------------------------------------------------------------------------
// host-side round driver for points mode on the tensor cores
// ---------------------------------------------------------------------------
appd_status tcf_prepare(appd_ctx* c, const float* X, int64_t n, int64_t d, TcState* st) {
  st->n = n;
  st->d = d;
  st->npad = (n + TC_N - 1) / TC_N * TC_N;
  st->dk = (int)((d + 15) / 16 * 16);
  st->K = st->dk + 16;
  st->stages = tcf_stages(st->K);
  if (st->stages == 0) return APPD_ERR_UNSUPPORTED;
  int blocks = (int)((n + 255) / 256);
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
  unsigned ml_bits = 0;
  APPD_CUDA(c, cudaMemcpyAsync(&ml_bits, maxlen, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  APPD_CUDA(c, cudaStreamSynchronize(c->stream));
  float ml;
  memcpy(&ml, &ml_bits, 4);
  if (!(ml < INFINITY)) return APPD_ERR_UNSUPPORTED;  // coordinates too large for the filter
  // scale = 2^e with scale * max|y| in [2^6.5, 2^7.5): |y^|^2 < 2^15, fp16 range safe
  int e = 0;
  if (ml > 0.0f) {
    double l2 = std::log2((double)ml);
    e = (int)std::floor(7.0 - l2 + 0.5);
    if (e > 100) e = 100;
    if (e < -100) e = -100;
  }
  st->scale = (float)std::ldexp(1.0, e);
  // Error model in scaled units (a = |y^_i| + |y^_j|):
  //  delta: each fp16 coordinate is within 2^-11 (relative, normal range) or 2^-25
  //    (absolute, subnormal) of s*(x - c); centring x - c in fp32 adds 2^-24 relative.
  //    |(y^_i - y^_j) - s (x_i - x_j)| <= (2^-11 + 2^-20) a + 2 sqrt(d) 2^-25.
  //  eta: Dt = |y^_i|^2 - 2 G' evaluated with fp32 accumulation of K products (each
  //    addition <= 2 ulp for the tensor-core adder), fp32 norms of d exact squares,
  //    the hi/lo fp16 split of -|y^_j|^2/2 and the final fp32 subtraction:
  //    |Dt - |y^_i - y^_j|^2| <= (4K + 2d + 16) 2^-24 a^2.
  //  gamma: R1 (d fmaf steps after an exact-to-1-ulp subtraction) is within
  //    (d + 2) 2^-24 of the real squared distance, relatively.
  st->c1 = (float)(std::ldexp(1.0, -11) + std::ldexp(1.0, -20));
  st->c2 = (float)(2.0 * std::sqrt((double)d) * std::ldexp(1.0, -25) * 1.01);
  st->c3 = (float)((4.0 * st->K + 2.0 * d + 16.0) * std::ldexp(1.0, -24) * 1.01);
  st->gamma = (float)((d + 2.0) * std::ldexp(1.0, -24) * 1.01);
  const size_t ybytes = (size_t)st->npad * st->K * 2;
  st->YA = ws(c, S_TC_YA, ybytes);
  st->YB = ws(c, S_TC_YB, ybytes);
  st->nrm = (float*)ws(c, S_TC_NRM, sizeof(float) * st->npad);
  st->len = (float*)ws(c, S_TC_LEN, sizeof(float) * st->npad);
  st->tile_maxlen = (float*)ws(c, S_TC_TML, sizeof(float) * (st->npad / TC_N));
  st->perm = (int*)ws(c, S_TC_PERM, sizeof(int) * (n + 1));
  st->sc = (int*)ws(c, S_TC_SC, sizeof(int) * (n + 1));
  st->keys = (int*)ws(c, S_TC_KEYS, sizeof(int) * 2 * (n + 1));
  st->cstart = (int*)ws(c, S_TC_CSTART, sizeof(int) * (n + 1));
  st->cend = (int*)ws(c, S_TC_CEND, sizeof(int) * (n + 1));
  st->rs = (int*)ws(c, S_TC_RS, sizeof(int) * (n + 1));
  st->re = (int*)ws(c, S_TC_RE, sizeof(int) * (n + 1));
  st->UB = (unsigned*)ws(c, S_TC_UB, sizeof(unsigned) * st->npad);
  st->cand_cap = (unsigned)std::min<int64_t>(64 * n + 4096, (int64_t)1 << 30);
  st->cand = ws(c, S_TC_CAND, sizeof(uint2) * st->cand_cap);
  st->counters = (unsigned*)ws(c, S_TC_CNT, 64);
  if (!st->YA || !st->YB || !st->nrm || !st->len || !st->tile_maxlen || !st->perm || !st->sc || !st->keys ||
      !st->cstart || !st->cend || !st->rs || !st->re || !st->UB || !st->cand || !st->counters)
    return fail(c, APPD_ERR_OUT_OF_MEMORY, "tc workspace");
  return APPD_OK;
}

// one Boruvka round's scan: compbest[comp] = min over the component's rows of the exact edge key.
// Returns APPD_ERR_UNSUPPORTED (without side effects on compbest) if the candidate buffer overflowed.
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
  k_pack<<<c->sm_count * 8, 256, 0, c->stream>>>(X, n, (int)st->d, st->dk, st->K, st->perm, st->center, st->scale,
                                                  st->npad, (__half*)st->YA, (__half*)st->YB, st->nrm, st->len);
  APPD_LAUNCHED(c);
  k_tile_maxlen<<<(unsigned)(st->npad / TC_N), 256, 0, c->stream>>>(st->len, st->npad, st->tile_maxlen);
  APPD_LAUNCHED(c);
  APPD_CUDA(c, cudaMemsetAsync(st->UB, 0x7F, sizeof(unsigned) * st->npad, c->stream));  // ~3.4e38
  APPD_CUDA(c, cudaMemsetAsync(st->counters, 0, 64, c->stream));
  TcParams P;
  P.YA = (const __half*)st->YA;
  P.YB = (const __half*)st->YB;
  P.nrm = st->nrm;
  P.len = st->len;
  P.tile_maxlen = st->tile_maxlen;
  P.cs = st->rs;
  P.ce = st->re;
  P.perm = st->perm;
  P.UB = st->UB;
  P.cand = (uint2*)st->cand;
  P.cand_count = st->counters;
  P.cand_cap = st->cand_cap;
  P.overflow = (int*)(st->counters + 4);
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
  P.c1 = st->c1;
  P.c2 = st->c2;
  P.c3 = st->c3;
  P.gamma = st->gamma;
  P.round0 = round == 0;
  P.dump = nullptr;
  if ((s = launch_tcf_scan(c, 0, P))) return s;
  if ((s = launch_tcf_scan(c, 1, P))) return s;
  unsigned h[8];
  APPD_CUDA(c, cudaMemcpyAsync(h, st->counters, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  APPD_CUDA(c, cudaStreamSynchronize(c->stream));
  st->last_candidates = h[0];
  if (h[4] != 0 || h[0] > st->cand_cap) {
    *overflowed = true;
    return APPD_OK;
  }
  *overflowed = false;
  if (h[0] > 0) {
    unsigned blocks = std::min<unsigned>((h[0] + 255) / 256, (unsigned)c->sm_count * 16);
    k_exact_candidates<<<blocks, 256, 0, c->stream>>>(X, (int)st->d, (const uint2*)st->cand, st->counters,
                                                       st->cand_cap, comp, compbest);
    APPD_LAUNCHED(c);
  }
  return APPD_OK;
}

}  // namespace appd

namespace appd {

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
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 128 * npad; e += (int64_t)gridDim.x * blockDim.x) {
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
  k_pack<<<c->sm_count * 8, 256, 0, c->stream>>>(X, n, (int)d, st.dk, st.K, st.perm, st.center, st.scale, st.npad,
                                                  (__half*)st.YA, (__half*)st.YB, st.nrm, st.len);
  APPD_LAUNCHED(c);
  TcParams P;
  memset(&P, 0, sizeof P);
  P.YA = (const __half*)st.YA;
  P.YB = (const __half*)st.YB;
  P.nrm = st.nrm;
  P.len = st.len;
  P.tile_maxlen = st.tile_maxlen;
  P.perm = st.perm;
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
