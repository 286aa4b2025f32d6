// k_f64.cu -- NEXT-3: fp64 weight matrices ("float64").
//
// The method only compares and copies weights, so the fp64 path is the fp32
// pipeline with three changes:
//   * validation reads fp64 (same rules, reading Q5);
//   * each Borůvka round picks the per-component best edge in two steps, because an fp64
//     weight and a pair index do not fit one 64-bit key: the per-row argmin of
//     (w, j) [k_scan_weights_f64], an atomicMin of the orderable-u64 weight per component,
//     then among the rows that reach it the smallest pair index [k_pick_f64].  The order is
//     the same strict (w, max(u,v), min(u,v)) order as the fp32 path (DESIGN.md "Borůvka tie
//     order"); the component key handed to the contraction holds the pair index only;
//   * after the MST the n-1 edges are sorted by their fp64 weights and relabelled by rank:
//     the dendrogram, the sparse table and the fill then run on the ranks r+1 (exact in
//     fp32 for n-1 < 2^24; max over ranks = rank of the max weight since the sort is
//     monotone), and the fill's store maps a rank back through the table hw[r] (fp64).
// Single rank only.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace appd {

__device__ __forceinline__ u64 orderable64(double x) {
  const u64 b = (u64)__double_as_longlong(x + 0.0);  // -0 -> +0 (reading Q5)
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ---- a1: validation (the fp32 kernel's rules: finite, +-0 diagonal, symmetric after
// -0 -> +0; first offender of each kind by row-major index).  Tile pair (I, J), I <= J:
// the (I, J) tile and the transposed (J, I) tile through shared memory.
constexpr int VT64 = 64;  // 64 x 64 doubles per tile: 512-byte row segments, 32 loads in flight per thread
__global__ void __launch_bounds__(256) k_validate_f64(const double* __restrict__ W, int64_t n, int64_t T,
                                                      u64* __restrict__ out3) {
  // blockIdx.x -> (I, J), I <= J, over the T x T upper triangle (row I holds T - I pairs)
  const int64_t p = blockIdx.x;
  const double q = (double)(2 * T + 1);
  int64_t I = (int64_t)((q - sqrt(q * q - 8.0 * (double)p)) * 0.5);
  if (I < 0) I = 0;
  while (I > 0 && I * T - I * (I - 1) / 2 > p) I--;
  while ((I + 1) * T - (I + 1) * I / 2 <= p) I++;
  const int64_t J = I + (p - (I * T - I * (I - 1) / 2));
  extern __shared__ double b[];  // [VT64][VT64 + 1]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8; columns tx and tx + 32
  constexpr int RPT = VT64 / 8;                             // rows per thread
  double av[RPT][2], bv[RPT][2];
#pragma unroll
  for (int s8 = 0; s8 < RPT; s8++) {  // all loads first: tile (I, J) and tile (J, I)
    const int r = ty + 8 * s8;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int cc = tx + 32 * h;
      const int64_t ia = I * VT64 + r, ja = J * VT64 + cc, ib = J * VT64 + r, jb = I * VT64 + cc;
      av[s8][h] = (ia < n && ja < n) ? __ldcs(W + ia * n + ja) : 0.0;
      bv[s8][h] = (ib < n && jb < n) ? __ldcs(W + ib * n + jb) : 0.0;
    }
  }
#pragma unroll
  for (int s8 = 0; s8 < RPT; s8++)
#pragma unroll
    for (int h = 0; h < 2; h++) b[(ty + 8 * s8) * (VT64 + 1) + tx + 32 * h] = bv[s8][h];
  __syncthreads();
  u64 nf = KEY_NONE, dg = KEY_NONE, as = KEY_NONE;
#pragma unroll
  for (int s8 = 0; s8 < RPT; s8++) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int r = ty + 8 * s8, cc = tx + 32 * h;
      const int64_t i = I * VT64 + r, j = J * VT64 + cc;
      if (i >= n || j >= n) continue;
      const double a = av[s8][h];
      const double t = b[cc * (VT64 + 1) + r];  // W[j][i]
      const u64 ij = (u64)(i * n + j), ji = (u64)(j * n + i);
      if (!isfinite(a)) nf = min(nf, ij);
      if (!isfinite(t)) nf = min(nf, ji);
      if (i == j && a != 0.0) dg = min(dg, ij);
      if (i < j && a != t) as = min(as, ij);  // numeric != on finite values == bitwise after -0 -> +0
    }
  }
  if (!__syncthreads_or(nf != KEY_NONE || dg != KEY_NONE || as != KEY_NONE)) return;
  if (nf != KEY_NONE) atomicMin(out3 + 0, nf);
  if (dg != KEY_NONE) atomicMin(out3 + 1, dg);
  if (as != KEY_NONE) atomicMin(out3 + 2, as);
}

appd_status launch_validate_weights_f64(appd_ctx* c, const double* W, int64_t n, u64* out3) {
  const int64_t T = (n + VT64 - 1) / VT64;
  const int64_t pairs = T * (T + 1) / 2;
  if (pairs > 0x7FFFFFFFll) return fail(c, APPD_ERR_UNSUPPORTED, "fp64 validation grid");
  const size_t smem = sizeof(double) * VT64 * (VT64 + 1);
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
    cudaFuncSetAttribute(k_validate_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    setup_done(attr, c);
  }
  k_validate_f64<<<(unsigned)pairs, 256, smem, c->stream>>>(W, n, T, out3);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---- a3: one Borůvka round, step 1: per-row argmin of (w, j) over eligible columns
// (another component; round 0: j != i), one CTA per row, 16-byte loads; then the
// component's minimum orderable weight by atomicMin.
template <bool ROUND0, int SENSE>
__global__ void __launch_bounds__(256) k_scan_weights_f64(const double* __restrict__ W, int64_t n,
                                                          const int* __restrict__ comp, u64* __restrict__ compw,
                                                          u64* __restrict__ roww, int* __restrict__ rowj) {
  __shared__ u64 sw[8];
  __shared__ int sj[8];
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double* Wr = W + i * n;
    const int ci = ROUND0 ? (int)i : comp[i];
    u64 bw = KEY_NONE;
    int bj = -1;
    const bool vec = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
    if (vec) {
      const double2* W2 = reinterpret_cast<const double2*>(Wr);
      const int2* C2 = reinterpret_cast<const int2*>(comp);
#pragma unroll 4
      for (int64_t q = threadIdx.x; q < (n >> 1); q += 256) {
        const double2 w = __ldcs(W2 + q);
        int2 cc = make_int2(0, 0);
        if (!ROUND0) cc = __ldg(C2 + q);
        const int64_t j = 2 * q;
        const double ws[2] = {w.x, w.y};
        const int cs[2] = {cc.x, cc.y};
#pragma unroll
        for (int t = 0; t < 2; t++) {
          const bool elig = ROUND0 ? (j + t != i) : (cs[t] != ci);
          const u64 k = orderable64(SENSE > 0 ? ws[t] : -ws[t]);
          if (elig && k < bw) { bw = k; bj = (int)(j + t); }  // columns ascend per thread: first j wins ties
        }
      }
    } else {
      for (int64_t j = threadIdx.x; j < n; j += 256) {
        const double w = __ldcs(Wr + j);
        const bool elig = ROUND0 ? (j != i) : (__ldg(comp + j) != ci);
        const u64 k = orderable64(SENSE > 0 ? w : -w);
        if (elig && k < bw) { bw = k; bj = (int)j; }
      }
    }
    // (w, j) lexicographic minimum over the CTA
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 ow = __shfl_xor_sync(0xffffffffu, bw, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (oj >= 0 && (bj < 0 || ow < bw || (ow == bw && oj < bj))) { bw = ow; bj = oj; }
    }
    if ((threadIdx.x & 31) == 0) { sw[threadIdx.x >> 5] = bw; sj[threadIdx.x >> 5] = bj; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int t = 1; t < 8; t++)
        if (sj[t] >= 0 && (bj < 0 || sw[t] < bw || (sw[t] == bw && sj[t] < bj))) { bw = sw[t]; bj = sj[t]; }
      roww[i] = bw;
      rowj[i] = bj;
      if (bj >= 0) atomicMin(compw + ci, bw);
    }
    __syncthreads();
  }
}

// step 2: among the rows whose best weight equals their component's, the smallest pair
// index (for a fixed row the smallest j also has the smallest pair index, so this is the
// component's minimum in the strict order); the key carries the pair index only
__global__ void k_pick_f64(int64_t n, const int* __restrict__ comp, const u64* __restrict__ compw,
                           const u64* __restrict__ roww, const int* __restrict__ rowj, u64* __restrict__ compbest) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = rowj[i];
    if (j < 0) continue;
    const int ci = comp[i];
    if (roww[i] == compw[ci]) atomicMin(compbest + ci, tri_index(i, j));
  }
}

appd_status launch_scan_weights_f64(appd_ctx* c, const double* W, int64_t n, int64_t k, bool round0, int sense,
                                    const int* comp, u64* compw, u64* roww, int* rowj, u64* compbest) {
  APPD_CUDA(c, cudaMemsetAsync(compw, 0xFF, sizeof(u64) * k, c->stream));
  const int grid = (int)std::min<int64_t>(n, (int64_t)c->sm_count * 8);
  if (round0) {
    if (sense > 0) k_scan_weights_f64<true, 1><<<grid, 256, 0, c->stream>>>(W, n, comp, compw, roww, rowj);
    else k_scan_weights_f64<true, -1><<<grid, 256, 0, c->stream>>>(W, n, comp, compw, roww, rowj);
  } else {
    if (sense > 0) k_scan_weights_f64<false, 1><<<grid, 256, 0, c->stream>>>(W, n, comp, compw, roww, rowj);
    else k_scan_weights_f64<false, -1><<<grid, 256, 0, c->stream>>>(W, n, comp, compw, roww, rowj);
  }
  APPD_LAUNCHED(c);
  const int g2 = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
  k_pick_f64<<<g2, 256, 0, c->stream>>>(n, comp, compw, roww, rowj, compbest);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// ---- a4: sort the MST edges by fp64 weight and relabel them by rank ----
__global__ void k_edges_f64(const u64* __restrict__ keys, int64_t m, const double* __restrict__ W, int64_t n,
                            int sense, u64* __restrict__ wkey, int* __restrict__ idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t u, v;
    tri_decode(keys[e] & 0xFFFFFFFFull, &u, &v);
    const double w = W[u * n + v];
    wkey[e] = orderable64(sense > 0 ? w : -w);
    idx[e] = (int)e;
  }
}

// sorted position r: endpoints, rank weight r + 1 for the dendrogram, hw[r + 1] = w
// (hw[0] = +0 is the diagonal)
__global__ void k_rank_edges_f64(const u64* __restrict__ keys, const int* __restrict__ order, int64_t m,
                                 const double* __restrict__ W, int64_t n, int32_t* __restrict__ eu,
                                 int32_t* __restrict__ ev, float* __restrict__ ew, double* __restrict__ hw) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t u, v;
    tri_decode(keys[order[r]] & 0xFFFFFFFFull, &u, &v);
    eu[r] = (int32_t)u;
    ev[r] = (int32_t)v;
    ew[r] = (float)(r + 1);
    hw[r + 1] = W[u * n + v] + 0.0;
    if (r == 0) hw[0] = 0.0;
  }
}

appd_status launch_edges_f64(appd_ctx* c, const u64* mstkeys, int64_t m, const double* W, int64_t n, int sense,
                             u64* wkey, u64* wkey_sorted, int* idx, int* idx_sorted, int32_t* eu, int32_t* ev,
                             float* ew, double* hw) {
  const int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)c->sm_count * 8);
  k_edges_f64<<<grid, 256, 0, c->stream>>>(mstkeys, m, W, n, sense, wkey, idx);
  APPD_LAUNCHED(c);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, wkey, wkey_sorted, idx, idx_sorted, (int)m, 0, 64, c->stream);
  void* t = ws(c, S_KEYS_TMP, tmp + 16);
  if (!t) return fail(c, APPD_ERR_OUT_OF_MEMORY, "sort workspace");
  APPD_CUDA(c, cub::DeviceRadixSort::SortPairs(t, tmp, wkey, wkey_sorted, idx, idx_sorted, (int)m, 0, 64, c->stream));
  c->launches += 8;
  k_rank_edges_f64<<<grid, 256, 0, c->stream>>>(mstkeys, idx_sorted, m, W, n, eu, ev, ew, hw);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

__global__ void k_zero1_f64(double* M) { M[0] = 0.0; }
appd_status launch_set_diag_zero_single_f64(appd_ctx* c, double* M) {
  k_zero1_f64<<<1, 1, 0, c->stream>>>(M);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
