// k_tcscan.cu -- the tcgen05 scan of a points-mode Boruvka round (see k_tcfilter.cu
// for the method).  Persistent kernel, one CTA per SM, 10 warps:
//   warp 0   producer: 1-D bulk async copies (cp.async.bulk -> UBLKCP) of the packed
//            fp16 operands; the 512-row block stays resident, 256-column tiles stream
//            through a ring of shared-memory stages; mbarrier transaction counts
//   warp 1   MMA issuer (one lane): tcgen05.mma.cta_group::1.kind::f16 M=128 N=256
//            K=16 slices; per column tile the four row tiles run in turn into two
//            TMEM accumulators (2 x 256 fp32 columns); tcgen05.commit -> mbarriers
//   warps 2-9 epilogue: tcgen05.ld 32x32b.x32 (software pipelined) -> per row and
//            128-column segment the eligible maximum of G' (FMNMX3 trees), stored for
//            the exact pass, and a running upper bound UB of the row's lightest edge.
// Shared-memory traffic of an SS-mode MMA is (M + N) K 2 bytes per M N K MACs: with
// M = 128, N = 256 that is 96 B/clk at the tensor rate, below the 128 B/clk of shared
// memory; the 512-row block makes each column-operand byte read from L2 serve 512 rows.
#include <algorithm>
#include <cstdlib>

#include "tc_common.cuh"
#include "tc_ptx.cuh"

namespace appd {

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// max of 32 values: 16 three-input maxima (FMNMX3)
__device__ __forceinline__ float fmax32(const float (&v)[32]) {
  const float a0 = fmax3(v[0], v[1], v[2]), a1 = fmax3(v[3], v[4], v[5]), a2 = fmax3(v[6], v[7], v[8]);
  const float a3 = fmax3(v[9], v[10], v[11]), a4 = fmax3(v[12], v[13], v[14]), a5 = fmax3(v[15], v[16], v[17]);
  const float a6 = fmax3(v[18], v[19], v[20]), a7 = fmax3(v[21], v[22], v[23]), a8 = fmax3(v[24], v[25], v[26]);
  const float a9 = fmax3(v[27], v[28], v[29]), a10 = fmaxf(v[30], v[31]);
  const float b0 = fmax3(a0, a1, a2), b1 = fmax3(a3, a4, a5), b2 = fmax3(a6, a7, a8), b3 = fmaxf(a9, a10);
  return fmaxf(fmax3(b0, b1, b2), b3);
}

// max of 64 values: 32 three-input maxima
__device__ __forceinline__ float fmax64(const float (&v)[64]) {
  float a[22];
#pragma unroll
  for (int i = 0; i < 21; i++) a[i] = fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  a[21] = v[63];
  float b[8];
#pragma unroll
  for (int i = 0; i < 7; i++) b[i] = fmax3(a[3 * i], a[3 * i + 1], a[3 * i + 2]);
  b[7] = a[21];
  return fmaxf(fmax3(b[0], b[1], b[2]), fmax3(fmax3(b[3], b[4], b[5]), b[6], b[7]));
}

// max of 128 values: 64 three-input maxima
__device__ __forceinline__ float fmax128(const float (&v)[128]) {
  float a[43];
#pragma unroll
  for (int i = 0; i < 42; i++) a[i] = fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  a[42] = fmaxf(v[126], v[127]);
  float b[15];
#pragma unroll
  for (int i = 0; i < 14; i++) b[i] = fmax3(a[3 * i], a[3 * i + 1], a[3 * i + 2]);
  b[14] = a[42];
  const float c0 = fmax3(b[0], b[1], b[2]), c1 = fmax3(b[3], b[4], b[5]), c2 = fmax3(b[6], b[7], b[8]);
  const float c3 = fmax3(b[9], b[10], b[11]), c4 = fmax3(b[12], b[13], b[14]);
  return fmaxf(fmax3(c0, c1, c2), fmaxf(c3, c4));
}

// one warp's TC_TMG accumulator columns: a single TMEM load and a 3-input max tree
__device__ __forceinline__ void tmem_ld_seg(uint32_t taddr, float (&v)[64]) { ptx::tmem_ld64(taddr, v); }
__device__ __forceinline__ void tmem_ld_seg(uint32_t taddr, float (&v)[128]) { ptx::tmem_ld128(taddr, v); }
__device__ __forceinline__ float fmax_seg(const float (&v)[64]) { return fmax64(v); }
__device__ __forceinline__ float fmax_seg(const float (&v)[128]) { return fmax128(v); }

// eligible maximum of one 32-column chunk (row p of component range [cs, ce))
__device__ __forceinline__ float chunk_max(const float (&v)[32], bool valid, int cs, int ce, int q0, bool fast,
                                           int n) {
  if (fast) return fmax32(v);
  float m = -INFINITY;
  if (valid && !(q0 >= cs && q0 + 32 <= ce)) {
#pragma unroll
    for (int t = 0; t < 32; t++) {
      const int qq = q0 + t;
      const bool el = (qq < cs || qq >= ce) && qq < n;
      m = fmaxf(m, el ? v[t] : -INFINITY);
    }
  }
  return m;
}

// epilogue: 16 warps of 64 columns (4 lane quarters x 4 column quarters) in both
// variants (measured faster than 8 warps of 128 columns)
template <bool SEG32>
struct EpiCfg {
  static constexpr int warps = TC_EPI_WARPS;
  static constexpr int cols = TC_NA / (warps / 4);  // accumulator columns per epilogue warp
  static constexpr int threads = 32 * (2 + warps);
};

template <int PASS, bool SEG32 = false>
__global__ void __launch_bounds__(EpiCfg<SEG32>::threads, 1) k_tcf_scan(TcParams P) {
  constexpr int EPI_WARPS = EpiCfg<SEG32>::warps;
  constexpr int WCOLS = EpiCfg<SEG32>::cols;
  static_assert(SEG32 || WCOLS == TC_TMG, "stored maxima granularity");
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = P.K;
  const int NST = P.stages;
  const uint32_t gran_bytes = TC_M * K * 2;    // 128 points
  const uint32_t a_bytes = TC_RT * gran_bytes;  // 512 points
  const uint32_t b_bytes = TC_N * K * 2;        // 256 points
  uint8_t* sA = smem;
  uint8_t* sB = smem + a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)NST * b_bytes);
  uint64_t* full = bars;         // [NST]
  uint64_t* empty = bars + NST;  // [NST]
  uint64_t* afull = bars + 2 * NST;
  uint64_t* aempty = afull + 1;
  uint64_t* tfull = aempty + 1;         // [TC_NBUF]
  uint64_t* tempty = tfull + TC_NBUF;  // [TC_NBUF]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + TC_NBUF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; s++) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::mbar_init(afull, 1);
    ptx::mbar_init(aempty, 1);
    for (int b = 0; b < TC_NBUF; b++) {
      ptx::mbar_init(tfull + b, 1);
      ptx::mbar_init(tempty + b, EPI_WARPS);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int nrb = P.rb_list ? *P.rb_count : (P.rb_end - P.rb_begin);
  // Work = a sequence of column-tile units, split evenly over the persistent CTAs (at
  // most one tile of imbalance).  Plain mode: row block b's units are its col_tiles
  // tiles.  Upper mode (symmetric pass): row block rb scans only column tiles >= 2 rb;
  // blocks rb and (last - rb) are laid end to end into one virtual row of constant
  // length L, so a CTA's contiguous range touches few row blocks (one A load each).
  const int C = P.col_tiles;
  const int L = P.upper ? 2 * C - 2 * (P.rb_begin + P.rb_end - 1) : C;
  const int vrows = P.upper ? nrb / 2 : nrb;
  const int U = vrows * L + ((P.upper && (nrb & 1)) ? C - 2 * (P.rb_begin + nrb / 2) : 0);
  const int ubeg = (int)((int64_t)blockIdx.x * U / gridDim.x), uend = (int)((int64_t)(blockIdx.x + 1) * U / gridDim.x);
  // next piece (one row block, column tiles [ct0, ct1)) of this CTA's range; advances u
  auto next_piece = [&](int& u, int& rb, int& ct0, int& ct1) -> bool {
    if (u >= uend) return false;
    const int q = u / L, x = u % L;
    const int left = uend - u;
    if (!P.upper) {
      rb = P.rb_list ? __ldg(P.rb_list + q) : P.rb_begin + q;
      ct0 = x;
      ct1 = min(C, x + left);
    } else {
      const int rba = P.rb_begin + q, rbb = P.rb_end - 1 - q;
      const int la = C - 2 * rba;
      if (x < la) {
        rb = rba;
        ct0 = 2 * rba + x;
        ct1 = 2 * rba + min(la, x + left);
      } else {
        rb = rbb;
        ct0 = 2 * rbb + (x - la);
        ct1 = 2 * rbb + min(L - la, x - la + left);
      }
    }
    u += ct1 - ct0;
    return true;
  };

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, aph = 0;
      bool first = true;
      int rb, ct0, ct1;
      for (int u = ubeg; next_piece(u, rb, ct0, ct1);) {
        if (!first) {
          ptx::mbar_wait(aempty, aph);
          aph ^= 1;
        }
        first = false;
        ptx::mbar_expect_tx(afull, a_bytes);
        ptx::bulk_g2s(sA, reinterpret_cast<const uint8_t*>(P.YA) + (size_t)rb * a_bytes, a_bytes, afull);
        for (int ct = ct0; ct < ct1; ct++) {
          ptx::mbar_wait(empty + stage, ph ^ 1);
          if (PASS == 5 || PASS == 6) {  // experiment: no column-operand copies
            ptx::mbar_arrive(full + stage);
          } else {
            ptx::mbar_expect_tx(full + stage, b_bytes);
            ptx::bulk_g2s(sB + stage * b_bytes, reinterpret_cast<const uint8_t*>(P.YB) + (size_t)ct * b_bytes,
                          b_bytes, full + stage);
          }
          if (++stage == NST) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // per column tile: 8 phases (row tile r, column half hh), phase i -> TMEM buffer i % 4
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_f16_f32(TC_M, TC_NA);
      const uint32_t sbo = (uint32_t)(K / 8) * 128u;
      const uint32_t a0 = ptx::smem_u32(sA);
      const uint32_t b0 = ptx::smem_u32(sB);
      int stage = 0;
      uint32_t ph = 0, aph = 0, tph[TC_NBUF] = {};
      int rb, ct0, ct1;
      for (int u = ubeg; next_piece(u, rb, ct0, ct1);) {
        ptx::mbar_wait(afull, aph);
        aph ^= 1;
        for (int ct = ct0; ct < ct1; ct++) {
          ptx::mbar_wait(full + stage, ph);
          const uint32_t bs = b0 + stage * b_bytes;
#pragma unroll
          for (int i = 0; i < TC_RT * TC_HALVES; i++) {
            const int r = i / TC_HALVES, hh = i % TC_HALVES, b = i % TC_NBUF;
            ptx::mbar_wait(tempty + b, tph[b] ^ 1);
            tph[b] ^= 1;
            ptx::tc_fence_after();
            for (int ks = 0; ks < K / 16; ks++) {
              const uint64_t ad = ptx::sdesc(a0 + r * gran_bytes + ks * 256, 128, sbo);
              const uint64_t bd = ptx::sdesc(bs + hh * gran_bytes + ks * 256, 128, sbo);
              ptx::mma_f16(tmem + (uint32_t)(b * TC_NA), ad, bd, idesc, ks > 0 ? 1u : 0u);
            }
            ptx::mma_commit(tfull + b);  // accumulator of (row tile r, half hh) ready
          }
          ptx::mma_commit(empty + stage);  // smem stage free once these MMAs complete
          if (++stage == NST) {
            stage = 0;
            ph ^= 1;
          }
        }
        ptx::mma_commit(aempty);  // row block free after the item's last MMA
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9) ----------------
    // warp w may only read TMEM lanes 32*(w%4) .. +31: warp (q, h) reads lane quarter q
    // and 64-column half h of each 128-column accumulator; in the phases of row tile r
    // it holds a row of row tile r, so each thread owns four rows of the item.
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    uint32_t tph[TC_NBUF] = {};
    int rb, ct0, ct1;
    for (int u = ubeg; next_piece(u, rb, ct0, ct1);) {
      // lean per-row state (registers): component range and, for the bound, the best
      // maximum so far and the running upper bound.  The cache-building pass (SEG32)
      // needs no bound.  Row p = rb * 512 + r * 128 + q * 32 + lane.
      int cs[TC_RT], ce[TC_RT];
      float ub[TC_RT], gb[TC_RT], nr[TC_RT];  // nr: |y^_p|^2, the stored maxima's encoding (tm_store)
      const int pbase = rb * TC_ROWS + q * 32 + lane;
#pragma unroll
      for (int r = 0; r < TC_RT; r++) {
        const int p = pbase + r * TC_M;
        const bool valid = p < P.n;
        cs[r] = valid ? (P.round0 ? p : P.cs[p]) : 0;
        ce[r] = valid ? (P.round0 ? p + 1 : P.ce[p]) : 0;
        nr[r] = valid ? __ldg(P.nrm + p) : 0.0f;
        ub[r] = INFINITY;
        gb[r] = -INFINITY;
      }
      for (int ct = ct0; ct < ct1; ct++) {
#pragma unroll
        for (int i = 0; i < TC_RT * TC_HALVES; i++) {
          const int r = i / TC_HALVES, hh = i % TC_HALVES, b = i % TC_NBUF;
          const int h0 = ct * TC_N + hh * TC_NA + h * WCOLS;  // first column of this warp's segment
          const int seg = h0 / WCOLS;
          const int p = pbase + r * TC_M;
          const bool valid = p < P.n;
          ptx::mbar_wait(tfull + b, tph[b]);
          tph[b] ^= 1;
          ptx::tc_fence_after();
          if (PASS == 3 || PASS == 6) {  // experiment: null epilogue (MMA + producer throughput only)
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty + b);
            continue;
          }
          float v[WCOLS];
          tmem_ld_seg(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * TC_NA + h * WCOLS), v);
          ptx::tmem_ld_wait();
          ptx::reg_fence(v);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(tempty + b);  // accumulator consumed: free it early
          if (PASS == 4) {  // experiment: TMEM load only
            if (v[0] == 12345.678f && valid) static_cast<float*>(P.TM)[p] = v[WCOLS - 1];
            continue;
          }
          if (PASS == 2) {  // test hook: raw accumulators of the CTA's first item
            if (P.dump && rb == P.rb_begin) {
              const int rloc = r * TC_M + q * 32 + lane;
              for (int t = 0; t < WCOLS; t++) P.dump[(int64_t)rloc * P.col_tiles * TC_N + h0 + t] = v[t];
            }
            continue;
          }
          // warp-uniform fast path: valid rows whose component misses these real columns
          const bool fast =
              __all_sync(0xffffffffu, valid && (h0 + WCOLS <= cs[r] || h0 >= ce[r]) && h0 + WCOLS <= P.n);
          if constexpr (SEG32) {
            // 32-column maxima (the same FMNMX3 count as one tree over the segment); the
            // warp's two chunks are adjacent in the packed table: one 8-byte store
            static_assert(WCOLS == 64, "32-column pass: two chunks per epilogue warp");
            float cm[2];
#pragma unroll
            for (int c = 0; c < 2; c++) {
              float w[32];
#pragma unroll
              for (int t = 0; t < 32; t++) w[t] = v[c * 32 + t];
              cm[c] = chunk_max(w, valid, cs[r], ce[r], h0 + c * 32, fast, P.n);
            }
            if (valid)
              *reinterpret_cast<__half2*>(static_cast<__half*>(P.TM) + tm32_index(h0 / 32, p, P.tm_nseg)) =
                  __halves2half2(tm_store(cm[0], nr[r]), tm_store(cm[1], nr[r]));
          } else {
            float m;
            if (fast) {
              m = fmax_seg(v);
            } else {
              m = -INFINITY;
#pragma unroll
              for (int c = 0; c < WCOLS / 32; c++) {
                float w[32];
#pragma unroll
                for (int t = 0; t < 32; t++) w[t] = v[c * 32 + t];
                m = fmaxf(m, chunk_max(w, valid, cs[r], ce[r], h0 + c * 32, false, P.n));
              }
            }
            // eligible maximum of G' over this (row, segment); a warp's rows are
            // consecutive, so the store is coalesced ([segment][row] layout)
            if (valid) static_cast<float*>(P.TM)[tm_index(seg, p, P.col_tiles * (TC_N / TC_TMG))] = m;
            if (PASS == 0 && valid && m > gb[r]) {  // tighten the bound only when the best improves (rare)
              gb[r] = m;
              const float ni = __ldg(P.nrm + p), li = __ldg(P.len + p);
              ub[r] = fminf(ub[r], em_upper(P.em, ni - 2.0f * m, ni, li, P.seg_maxlen[seg],
                                            em_delta2(__ldg(P.err + p), P.seg_maxerr[seg])));
            }
          }
        }
      }
      if (PASS == 0 && !SEG32) {
#pragma unroll
        for (int r = 0; r < TC_RT; r++) {
          const int p = pbase + r * TC_M;
          if (p < P.n && ub[r] < INFINITY) atomicMin(P.UB + p, __float_as_uint(fmaxf(ub[r], 0.0f)));
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
  return (size_t)TC_ROWS * K * 2 + (size_t)stages * TC_N * K * 2 + (2 * TC_MAX_STAGES + 2 + 2 * TC_NBUF) * 8 + 16;
}

// deepest ring (<= TC_MAX_STAGES) that fits 227 KB of shared memory; 0 if fewer than 2 fit
int tcf_stages(int K) {
  for (int s = TC_MAX_STAGES; s >= 2; s--)
    if (tcf_smem_bytes(K, s) <= 227 * 1024) return s;
  return 0;
}

// pass 0: scan (TC_TMG-column maxima + row bound UB), 1: scan with 32-column maxima
// (cache-building round), 2: test hook (raw accumulators), 7: TC_TMG-column maxima only
// (component-matrix pass: its bounds come from k_cm_rowub).  With a row-block list the grid is sized
// for the host's upper bound P.rb_end - P.rb_begin; the kernel reads the count.
appd_status launch_tcf_scan(appd_ctx* c, int pass, const TcParams& P) {
  // at least 120 KB so that exactly one CTA (and one 512-column TMEM allocation) fits per SM
  size_t smem = tcf_smem_bytes(P.K, P.stages);
  if (smem < 120 * 1024) smem = 120 * 1024;
  static std::atomic<unsigned long long> attr_done{0};
  if (needs_setup(attr_done, c)) {
    cudaFuncSetAttribute(k_tcf_scan<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_tcf_scan<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_tcf_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_tcf_scan<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    setup_done(attr_done, c);
  }
  // column-tile units (host upper bound when the row-block list is read on the device)
  const int64_t nrb = P.rb_end - P.rb_begin;
  const int64_t units = P.upper ? (nrb + 1) / 2 * (int64_t)(2 * P.col_tiles - 2 * (P.rb_begin + P.rb_end - 1))
                                : nrb * P.col_tiles;
  int grid = (int)std::min<int64_t>(c->sm_count, units);
  if (grid < 1) return APPD_OK;
#ifdef APPD_DEV_HOOKS
  // development builds only (-DAPPD_DEV_HOOKS): pipeline experiments 3-6 (null epilogue,
  // TMEM load only, no column-operand copies) selected by APPD_TC_EXPERIMENT or pass >= 3
  static const int exp_pass = getenv("APPD_TC_EXPERIMENT") ? atoi(getenv("APPD_TC_EXPERIMENT")) : 0;
  int ep = exp_pass;
  if (pass >= 3) ep = pass;
  if (ep == 3) {
    cudaFuncSetAttribute(k_tcf_scan<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    k_tcf_scan<3><<<grid, EpiCfg<false>::threads, smem, c->stream>>>(P);
  } else if (ep == 4) {
    cudaFuncSetAttribute(k_tcf_scan<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    k_tcf_scan<4><<<grid, EpiCfg<false>::threads, smem, c->stream>>>(P);
  } else if (ep == 5) {
    cudaFuncSetAttribute(k_tcf_scan<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    k_tcf_scan<5><<<grid, EpiCfg<false>::threads, smem, c->stream>>>(P);
  } else if (ep == 6) {
    cudaFuncSetAttribute(k_tcf_scan<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    k_tcf_scan<6><<<grid, EpiCfg<false>::threads, smem, c->stream>>>(P);
  }
  if (ep >= 3 && ep <= 6) {
    APPD_LAUNCHED(c);
    return APPD_OK;
  }
#endif
  if (pass == 0) k_tcf_scan<0><<<grid, EpiCfg<false>::threads, smem, c->stream>>>(P);
  else if (pass == 1) k_tcf_scan<0, true><<<grid, EpiCfg<true>::threads, smem, c->stream>>>(P);
  else if (pass == 7) k_tcf_scan<7><<<grid, EpiCfg<false>::threads, smem, c->stream>>>(P);
  else k_tcf_scan<2><<<1, EpiCfg<false>::threads, smem, c->stream>>>(P);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
