// k_sort.cu -- radix sorts of the path.  Single-pass sorts (at most 8 key bits: the
// component labels of the tensor-core rounds, k <= 256) run as ONE cooperative launch;
// wider keys (MST edges by weight, record keys of the dendrogram, fill rows by position)
// use the library's onesweep sort, which measured as fast as a cooperative multi-pass
// version (grid barriers cost what its per-digit launches cost: ~60 us for 64K keys).
//
// The cooperative pass is three grid-wide phases of one persistent launch (one
// 1024-thread CTA per SM):
//   A  each CTA counts the digits of its contiguous segment in shared memory and writes
//      its counts to cnt[digit][CTA];
//   B  one warp per digit: exclusive scan over the CTAs, digit total;
//   C  every CTA scans the digit totals (shared memory) and scatters its segment in
//      order: the warps of a 1024-key tile take their turn, lanes with equal digits
//      ranked by __match_any_sync, so equal digits keep their input order (stable).
#include <algorithm>
#include <atomic>

#include <cub/device/device_radix_sort.cuh>

#include <cooperative_groups.h>

#include "internal.cuh"

namespace appd {
namespace cg = cooperative_groups;

namespace {

constexpr int kSortThreads = 1024;
constexpr int kMaxDigitBits = 11;  // 2048 counters per CTA (8 KB of shared memory)
constexpr int kSortCluster = 8;  // CTAs of the single-cluster sort (portable size)

template <typename K>
struct CoopSortArgs {
  const K* kin;
  K* kout;
  K* kbuf;
  const int* vin;  // nullptr: keys only
  int* vout;
  int* vbuf;
  int n, begin_bit, end_bit, passes, dbits;
  unsigned* cnt;   // [1 << dbits][G]
  unsigned* dtot;  // [1 << dbits]
  int iota_vals;   // values = input index (vin ignored)
  // optional epilogue for component labels (keys = labels, sorted): first / end position
  // of every label, and per position the range of its own label
  int *cstart, *cend, *rs, *re;
  unsigned* bar;  // grid barrier word (coop_grid_sync)
};

__device__ __forceinline__ unsigned end_bit_mask(int width, unsigned dmask) {
  return width >= 32 ? dmask : (dmask & ((1u << width) - 1u));
}

// barrier of the persistent sort: the cooperative grid, or one cluster (small sorts)
template <bool CL>
__device__ __forceinline__ void sort_sync(unsigned* bar) {
  if constexpr (CL) cg::this_cluster().sync();
  else coop_grid_sync(bar);
}

template <typename K, bool CL>
__global__ void __launch_bounds__(kSortThreads, 1) k_coop_sort(const CoopSortArgs<K> a) {
  extern __shared__ unsigned sm[];  // [ND] counts, then running scatter positions
  __shared__ unsigned part[kSortThreads / 32];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ND = 1 << a.dbits;
  const unsigned dmask = (unsigned)ND - 1u;
  const int lo = (int)((int64_t)a.n * b / G), hi = (int)((int64_t)a.n * (b + 1) / G);
  const int gwarp = (b * kSortThreads + tid) >> 5, nwarps = (G * kSortThreads) >> 5;
  for (int p = 0; p < a.passes; p++) {
    const int shift = a.begin_bit + p * a.dbits;
    // the last pass writes the output: pass p writes kout when (passes - 1 - p) is even
    K* dst = ((a.passes - 1 - p) & 1) ? a.kbuf : a.kout;
    const K* src = p == 0 ? a.kin : (((a.passes - p) & 1) ? a.kbuf : a.kout);
    int* vdst = ((a.passes - 1 - p) & 1) ? a.vbuf : a.vout;
    const int* vsrc = p == 0 ? a.vin : (((a.passes - p) & 1) ? a.vbuf : a.vout);
    // (the last pass may be narrower: bits at and above end_bit never take part)
    const unsigned pmask = end_bit_mask(a.end_bit - shift, dmask);
    auto digit = [&](K k) { return (unsigned)(k >> shift) & pmask; };
    // ---- A: this CTA's digit counts
    for (int d = tid; d < ND; d += kSortThreads) sm[d] = 0u;
    __syncthreads();
    for (int i = lo + tid; i < hi; i += kSortThreads) atomicAdd(sm + digit(src[i]), 1u);
    __syncthreads();
    for (int d = tid; d < ND; d += kSortThreads) a.cnt[(int64_t)d * G + b] = sm[d];
    sort_sync<CL>(a.bar);
    // ---- B: per digit, exclusive offsets of the CTAs and the digit total
    for (int d = gwarp; d < ND; d += nwarps) {
      unsigned carry = 0u;
      for (int j0 = 0; j0 < G; j0 += 32) {
        const int j = j0 + lane;
        const unsigned v = j < G ? a.cnt[(int64_t)d * G + j] : 0u;
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (j < G) a.cnt[(int64_t)d * G + j] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) a.dtot[d] = carry;
    }
    sort_sync<CL>(a.bar);
    // ---- C: digit bases (block scan of the totals, up to 4 per thread), then the
    // CTA's first position per digit
    {
      const int per = (ND + kSortThreads - 1) / kSortThreads;
      const int d0 = tid * per;
      unsigned loc[4], s = 0u;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        loc[u] = (u < per && d0 + u < ND) ? a.dtot[d0 + u] : 0u;
        s += loc[u];
      }
      unsigned x = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) part[warp] = x;
      __syncthreads();
      if (warp == 0) {
        unsigned w = part[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += y;
        }
        part[lane] = w;
      }
      __syncthreads();
      unsigned run = (warp ? part[warp - 1] : 0u) + x - s;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (u < per && d0 + u < ND) {
          sm[d0 + u] = run + a.cnt[(int64_t)(d0 + u) * G + b];
          run += loc[u];
        }
      __syncthreads();
    }
    // stable scatter of the segment, 1024-key tiles, warps in order
    for (int base = lo; base < hi; base += kSortThreads) {
      const int i = base + tid;
      const bool valid = i < hi;
      K key = 0;
      int val = 0;
      unsigned d = 0xFFFFFFFFu;
      if (valid) {
        key = src[i];
        d = digit(key);
        if (a.iota_vals && p == 0) val = i;
        else if (vsrc) val = vsrc[i];
      }
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      const unsigned rank = __popc(peers & ((1u << lane) - 1u));
      const int wn = min(kSortThreads, hi - base + 31) >> 5;  // warps holding keys
      for (int w = 0; w < wn; w++) {
        if (warp == w && valid) {
          unsigned pos = 0u;
          if (lane == leader) {
            pos = sm[d];
            sm[d] = pos + __popc(peers);
          }
          pos = __shfl_sync(peers, pos, leader) + rank;
          dst[pos] = key;
          if (vsrc || a.iota_vals) vdst[pos] = val;
        }
        __syncthreads();
      }
    }
    sort_sync<CL>(a.bar);
  }
  if (a.cstart) {  // label ranges (k_comp_ranges, k_row_ranges)
    const int64_t tid64 = (int64_t)b * kSortThreads + tid, nt = (int64_t)G * kSortThreads;
    for (int64_t q = tid64; q < a.n; q += nt) {
      const int cq = (int)a.kout[q];
      if (q == 0 || (int)a.kout[q - 1] != cq) a.cstart[cq] = (int)q;
      if (q == a.n - 1 || (int)a.kout[q + 1] != cq) a.cend[cq] = (int)q + 1;
    }
    sort_sync<CL>(a.bar);
    for (int64_t q = tid64; q < a.n; q += nt) {
      const int cq = (int)a.kout[q];
      a.rs[q] = a.cstart[cq];
      a.re[q] = a.cend[cq];
    }
  }
}

template <typename K>
appd_status coop_sort(appd_ctx* c, const K* kin, K* kout, const int* vin, int* vout, int64_t count, int begin_bit,
                      int end_bit, bool iota_vals = false, int* cstart = nullptr, int* cend = nullptr,
                      int* rs = nullptr, int* re = nullptr) {
  if (count <= 0) return APPD_OK;
  if (count > (int64_t)1 << 30) return fail(c, APPD_ERR_UNSUPPORTED, "sort of %lld keys", (long long)count);
  // small sorts (every CTA of one cluster holds one tile of 1024 keys): one cluster (at
  // two tiles per CTA the library sort measured faster)
  const bool cl = count >= 2048 && count <= (int64_t)kSortCluster * kSortThreads;
  // digits: up to 11 bits (fewer passes) on the grid; 8 in the cluster, where a pass over
  // a few thousand keys is dominated by its histogram of 2^bits counters
  const int maxd = cl ? 8 : kMaxDigitBits;
  const int bits = std::max(1, end_bit - begin_bit);
  const int passes = (bits + maxd - 1) / maxd;
  const int dbits = (bits + passes - 1) / passes;
  const int ND = 1 << dbits;
  const int G = cl ? kSortCluster : c->sm_count;
  const bool vals = vin || iota_vals;
  const size_t kb = (sizeof(K) * (size_t)count + 255) & ~(size_t)255, vb = vals ? (sizeof(int) * (size_t)count + 255) & ~(size_t)255 : 0;
  char* w = (char*)ws(c, S_SORT, kb + vb + sizeof(unsigned) * ((size_t)ND * G + ND) + 256);
  if (!w) return fail(c, APPD_ERR_OUT_OF_MEMORY, "sort workspace (%lld keys)", (long long)count);
  CoopSortArgs<K> a;
  a.kin = kin;
  a.kout = kout;
  a.kbuf = reinterpret_cast<K*>(w);
  a.vin = vin;
  a.vout = vout;
  a.vbuf = vals ? reinterpret_cast<int*>(w + kb) : nullptr;
  a.iota_vals = iota_vals ? 1 : 0;
  a.cstart = cstart;
  a.cend = cend;
  a.rs = rs;
  a.re = re;
  a.n = (int)count;
  a.begin_bit = begin_bit;
  a.end_bit = end_bit;
  a.passes = passes;
  a.dbits = dbits;
  a.cnt = reinterpret_cast<unsigned*>(w + kb + vb);
  a.dtot = a.cnt + (size_t)ND * G;
  a.bar = grid_barrier_word(c);
  if (!a.bar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
    cudaFuncSetAttribute(k_coop_sort<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(unsigned) << kMaxDigitBits));
    cudaFuncSetAttribute(k_coop_sort<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(unsigned) << kMaxDigitBits));
    setup_done(attr, c);
  }
  void* args[] = {&a};
  if (!cl) {
    APPD_CUDA(c, cudaLaunchCooperativeKernel((const void*)k_coop_sort<K, false>, G, kSortThreads, args,
                                             sizeof(unsigned) * (size_t)ND, c->stream));
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kSortThreads);
    cfg.dynamicSmemBytes = sizeof(unsigned) * (size_t)ND;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    APPD_CUDA(c, cudaLaunchKernelExC(&cfg, (const void*)k_coop_sort<K, true>, args));
  }
  APPD_LAUNCHED(c);
  return APPD_OK;
}

template <typename K>
appd_status lib_sort(appd_ctx* c, const K* kin, K* kout, const int* vin, int* vout, int64_t count, int begin_bit,
                     int end_bit) {
  size_t tmp = 0;
  if (vin) cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)count, begin_bit, end_bit, c->stream);
  else cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, (int)count, begin_bit, end_bit, c->stream);
  void* t = ws(c, S_KEYS_TMP, tmp + 16);
  if (!t) return fail(c, APPD_ERR_OUT_OF_MEMORY, "sort workspace");
  if (vin)
    APPD_CUDA(c, cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, (int)count, begin_bit, end_bit, c->stream));
  else
    APPD_CUDA(c, cub::DeviceRadixSort::SortKeys(t, tmp, kin, kout, (int)count, begin_bit, end_bit, c->stream));
  c->launches += 4;
  return APPD_OK;
}

template <typename K>
appd_status path_sort(appd_ctx* c, const K* kin, K* kout, const int* vin, int* vout, int64_t count, int begin_bit,
                      int end_bit) {
  // one digit pass, or a small sort (one cluster, its barriers far cheaper than the
  // library's per-pass launches): the cooperative sort; else the library's onesweep
  // From 8K to 2^17 keys the cooperative sort also takes multi-pass keys (11-bit digits: the
  // MST edges' 31 weight bits in 3 passes instead of the library's 4 launches of 8 bits);
  // below 2K keys the library's single-tile sort is the fastest
  if (end_bit - begin_bit <= kMaxDigitBits || (count >= 2048 && count <= (int64_t)kSortCluster * kSortThreads) ||
      (count > (int64_t)kSortCluster * kSortThreads && count <= (1 << 17) && end_bit - begin_bit <= 3 * kMaxDigitBits))
    return coop_sort<K>(c, kin, kout, vin, vout, count, begin_bit, end_bit);
  return lib_sort<K>(c, kin, kout, vin, vout, count, begin_bit, end_bit);
}

}  // namespace

appd_status sort_components(appd_ctx* c, const int* comp, int64_t n, int bits, int* sc, int* perm, int* cstart,
                            int* cend, int* rs, int* re) {
  if (bits > kMaxDigitBits) return APPD_ERR_UNSUPPORTED;
  return coop_sort<unsigned>(c, reinterpret_cast<const unsigned*>(comp), reinterpret_cast<unsigned*>(sc), nullptr, perm,
                             n, 0, bits, true, cstart, cend, rs, re);
}

appd_status sort_keys_u64_bits64(appd_ctx* c, const u64* in, u64* out, int64_t count, int begin_bit, int end_bit) {
  return path_sort<u64>(c, in, out, nullptr, nullptr, count, begin_bit, end_bit);
}
appd_status sort_keys_u64(appd_ctx* c, const u64* in, u64* out, int64_t count) {
  return path_sort<u64>(c, in, out, nullptr, nullptr, count, 0, 64);
}
appd_status sort_keys_u32_bits(appd_ctx* c, const unsigned* in, unsigned* out, int64_t count, int begin_bit,
                               int end_bit) {
  return path_sort<unsigned>(c, in, out, nullptr, nullptr, count, begin_bit, end_bit);
}
// (keys are non-negative on every call site: unsigned order = signed order)
appd_status sort_pairs_i32_bits(appd_ctx* c, const int* kin, int* kout, const int* vin, int* vout, int64_t count,
                                int end_bit) {
  return path_sort<unsigned>(c, reinterpret_cast<const unsigned*>(kin), reinterpret_cast<unsigned*>(kout), vin, vout,
                             count, 0, end_bit);
}
appd_status sort_pairs_i32(appd_ctx* c, const int* kin, int* kout, const int* vin, int* vout, int64_t count) {
  return path_sort<unsigned>(c, reinterpret_cast<const unsigned*>(kin), reinterpret_cast<unsigned*>(kout), vin, vout,
                             count, 0, 32);
}

}  // namespace appd
