// tc_common.cuh -- shared pieces of the tensor-core points-mode MST scan
// (k_tcscan.cu: the tcgen05 kernel; k_tcfilter.cu: preparation, exact re-check, driver).
#pragma once
#include <cuda_fp16.h>

#include "internal.cuh"

namespace appd {

// MMA: M = 128 rows (one TMEM lane per row) x N = 256 columns x K = 16 per instruction,
// both operands from shared memory (K-major, no swizzle).  A work item keeps TC_RT = 4
// row tiles (512 rows) resident in shared memory and streams 256-column tiles of the
// column operand through a ring; TMEM holds two 256-column fp32 accumulators that the
// four row tiles of a column tile use in turn (phase r -> buffer r % 2), so the
// epilogue of one row tile overlaps the MMAs of the next.
constexpr int TC_M = 128, TC_N = 256, TC_RT = 4, TC_ROWS = TC_M * TC_RT, TC_MAX_STAGES = 6;
constexpr int TC_NA = 256;        // MMA N: accumulator width (TMEM columns per buffer)
constexpr int TC_NBUF = 2;        // TMEM accumulator buffers (TC_NBUF x TC_NA = 512 columns)
constexpr int TC_HALVES = TC_N / TC_NA;  // accumulators per (row tile, column tile)
constexpr int TC_EPI_WARPS = 16;  // 4 lane quarters x 4 column quarters of an accumulator
constexpr int TC_TMG = TC_NA / 4; // columns per epilogue warp = granularity of the stored maxima
constexpr int TC_THREADS = 32 * (2 + TC_EPI_WARPS);  // warp 0 producer, warp 1 MMA, then epilogue

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

// delta from the per-point fp16 rounding-error norms: |(y^_i - y^_j) - s (x_i - x_j)| <=
// E_i + E_j with E_p = |y^_p - s (x_p - c)| computed exactly (k_pack, double, rounded up);
// the worst case E_p <= c1 |y^_p| + c2 is what e.c1 / e.c2 bound
__device__ __forceinline__ float em_delta2(float Ei, float Ej) { return (Ei + Ej) * (1.0f + 0x1p-20f) + 1e-30f; }
__device__ __forceinline__ float em_eta(const ErrModel& e, float L, float R) {
  return e.k1 * R * (L + 0.5f * R) + e.k2 * (L * L + R * R) + e.k3 * (4.0f * R * R + (L + R) * (L + R));
}
// upper bound on s^2 r for a column whose Dt is dt
__device__ __forceinline__ float em_upper(const ErrModel& e, float dt, float ni, float L, float R, float delta) {
  const float r = sqrtf(fmaxf(dt + em_eta(e, L, R), 0.0f)) + delta;
  return (1.0f + e.gamma) * r * r * (1.0f + 0x1p-18f) + 0x1p-18f * ni;
}
// G' threshold: a column can hold a candidate (L <= ub) only if G' >= thr
__device__ __forceinline__ float em_thr(const ErrModel& e, float ub, float ni, float L, float R, float delta) {
  const float r = sqrtf(ub / (1.0f - e.gamma)) + delta;
  const float T = (r * r + em_eta(e, L, R)) * (1.0f + 0x1p-18f) + 0x1p-18f * ni;
  return 0.5f * (ni - T);
}

// Stored maxima layout, row-block major: element (segment s, row p) of a table with
// nseg segments lives at (p / 512) * nseg * 512 + s * 512 + p % 512, so the writes of
// one 512-row work item fill one contiguous region (few TLB pages) and a warp's 32
// consecutive rows stay one 128-byte line per segment.
__host__ __device__ __forceinline__ int64_t tm_index(int s, int p, int nseg) {
  return (int64_t)(p >> 9) * nseg * 512 + (int64_t)s * 512 + (p & 511);
}

// The 32-column table additionally packs 8 consecutive chunks of a row together
// (16 bytes of fp16), so a reader loads 8 chunk maxima per 128-bit access (nch rounded
// up to a multiple of 8 per 512-row block):
//   (p / 512) * nch8 * 512 + (c / 8) * 4096 + (p % 512) * 8 + c % 8
__host__ __device__ __forceinline__ int64_t tm32_index(int c, int p, int nch) {
  const int nch8 = (nch + 7) & ~7;
  return (int64_t)(p >> 9) * nch8 * 512 + (int64_t)(c >> 3) * 4096 + (p & 511) * 8 + (c & 7);
}
__host__ __device__ __forceinline__ int64_t tm32_elems(int64_t npad) {  // table size (halves)
  return npad * (((npad / 32) + 7) & ~7ll);
}

// The 32-column maxima of the cache pass are stored in fp16 (half the traffic of fp32
// for the writer and the top-K reader), as the squared-distance estimate D = |y^_i|^2 - 2 G' of the row rather than
// G' itself: D is small exactly where precision matters (near neighbours; an fp16 ulp
// of G' ~ 2^14 would be 8-16 scaled units, of D ~ 10^3 about one).  The writer rounds
// up twice (D = ni - 2m in fp32, then to fp16), so for the row's ni = |y^_i|^2:
//   tm_low(D', ni) <= m <= tm_up(D', ni)
// -- every bound derived from tm_low stays valid, and every listing test made against
// tm_up keeps every candidate.  An ineligible segment (m = -inf) is stored as +inf.
__device__ __forceinline__ __half tm_store(float m, float ni) { return __float2half_ru(__fsub_ru(ni, 2.0f * m)); }
__device__ __forceinline__ float tm_low(float D, float ni) { return 0.5f * __fsub_rd(ni, D); }
__device__ __forceinline__ float tm_up(float D, float ni) {
  // D' exceeds ni - 2m by less than one fp16 spacing (<= 2^-10 |D'|, or 2^-24) plus the
  // fp32 rounding of the subtraction (<= 2^-23 |D|)
  if (D == INFINITY) return -INFINITY;
  return 0.5f * __fadd_ru(__fsub_ru(ni, D), fmaf(fabsf(D), 0x1.1p-10f, 0x1p-23f));
}
struct TcParams {
  const __half* YA;          // row operand granules (128 points x K, core-matrix layout)
  const __half* YB;          // column operand granules
  const float* nrm;          // |y^_p|^2 (fp32), permuted order
  const float* len;          // |y^_p|
  const float* seg_maxlen;   // max |y^_j| over each TC_TMG-column segment
  const float* err;          // E_p, permuted order
  const float* seg_maxerr;   // max E_j over each TC_TMG-column segment
  const int* cs;             // per permuted row: first position of its component
  const int* ce;             // per permuted row: one past the last position
  unsigned* UB;              // per permuted row: upper bound (float bits, >= 0)
  void* TM;                  // [segment][row]: eligible maximum of G' over the TC_TMG columns (fp32), or
                             // the 32-column table of the cache pass (fp16 encoded, tm_store)
  int64_t tm_ld;             // leading dimension of TM (npad), [segment][row] layout (128-column tables)
  int tm_nseg;               // segments per row of the row-block-major 32-column table (npad / 32)
  int n;                     // points
  int K;                     // padded K (multiple of 16)
  int stages;                // shared-memory ring depth for the column operand
  int rb_begin, rb_end;      // this rank's 512-row blocks (permuted order)
  int col_tiles;             // npad / 256
  ErrModel em;
  int round0;   // singletons (eligibility = j != i)
  float* dump;  // PASS 2 (test hook) only: raw accumulator of the first item
  // TM granularity: 0 -> one maximum per TC_TMG (64) columns; 1 -> per 32 columns
  // (the cache-building round 0: 4x the maxima, 1/4 of the exact re-check work)
  int seg32;
  // optional row-block list (re-scan rounds): the *rb_count blocks of
  // rb_list[] (col_tiles units each); when null the blocks rb_begin .. rb_end-1
  const int* rb_list;
  const int* rb_count;
  // symmetric pass: row block rb scans column tiles >= 2 rb only (rb_list must be null)
  int upper;
};

struct CmParams {
  const float* TM;      // [nseg][npad]
  int64_t ld;
  int nseg;
  int n, k;
  int p_begin, p_end;
  const int* sc;        // sorted component label per position
  const int* cstart;
  const int* cend;
  const float* nrm;
  const float* len;
  const float* seg_maxlen;
  const TcScale* tsc;  // device: maxlen bounds |y^| (scaled units)
  const float* err;     // E_p (permuted order)
  const float* maxerr;  // max E over all points (device)
  ErrModel em;
  unsigned* CUB;        // [k][k] float bits
  unsigned* list;       // (32-column chunk << 17 | row) entries
  int upper;            // TM holds only segments >= 4 (p / 512) of row p (symmetric pass)
  const int2* segd;     // per segment: first and last component label of its real columns
  unsigned list_cap;
  unsigned* counters;   // [1] listed chunk entries
  const float* XTp;
  int d;
  const int* perm;
  u64* WCM;             // [k][k]
};
appd_status launch_cm_rowub(appd_ctx* c, const CmParams& P);
appd_status launch_cm_filter(appd_ctx* c, const CmParams& P);
appd_status launch_seg_comp(appd_ctx* c, const int* sc, int n, int nseg, int2* segd);
appd_status launch_cm_thresholds(appd_ctx* c, const unsigned* CUB, int k, unsigned* T);

struct ListParams {
  const unsigned* list;   // (chunk << 17 | row), sorted ascending
  const unsigned* count;  // entries (capped by cap)
  unsigned cap;
  int nch, n, d;
  const float* X;
  const int* perm;        // nullptr: identity
  const unsigned* run_lo;     // per chunk: first entry of its run in the sorted list
  const unsigned* run_nb;     // per chunk: 128-row batches
  const unsigned* item_start; // exclusive prefix of run_nb
  const int4* items;          // per work item: chunk, first list entry, rows
  // MODE 0
  const float* UBK;
  const TcScale* tsc;  // device: s2 = scale^2
  unsigned* cnt;
  u64* cand;
  int ccap;
  // MODE 1
  const int* sc;
  int k;
  u64* WCM;
};
appd_status launch_list_counting(appd_ctx* c, const unsigned* list, const unsigned* count, unsigned cap, int nch,
                                 unsigned* hist, unsigned* offs, unsigned* cursor, unsigned* out, unsigned* run_lo,
                                 unsigned* run_nb, unsigned* item_start, int4* items, bool aggregate);
appd_status launch_list_exact(appd_ctx* c, int mode, const ListParams& L, unsigned* run_lo, unsigned* run_nb,
                              unsigned* item_start);
appd_status launch_topk_scan(appd_ctx* c, int K, const __half* TM32, int nch, int p_begin, int p_end,
                             const float* nrm, const float* len, const TcScale* sc, const float* err,
                             const float* maxerr, const ErrModel& em, float* UBK, unsigned* list, unsigned* count,
                             unsigned cap, unsigned* cand_cnt);


size_t tcf_smem_bytes(int K, int stages);
int tcf_stages(int K);
appd_status launch_tcf_scan(appd_ctx* c, int pass, const TcParams& P);

}  // namespace appd
