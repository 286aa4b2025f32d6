// k_prim.cu -- the Prim variant of the MST stage.
//
// P:L98 (§3): Algorithm 4 builds the minimum spanning tree with Prim's algorithm, O(n^2):
// n - 1 steps, each adding the unvisited vertex of smallest key and relaxing every other
// key with its weight to the new vertex.  Prim's visit order pi is a leaf order of the
// single-linkage dendrogram for any tie-breaking, and the key with which
// pi_{a+1} joins is the merge height h[a] = M[pi_a][pi_{a+1}] -- so this variant emits
// (pi, h) directly: no edge sort (a4) and no dendrogram build (a5).
//
// The n steps are inherently sequential, so the variant is ONE persistent CTA (a grid- or
// cluster-wide barrier per step costs 0.2-1 us; a CTA barrier ~25 ns).  A step's cost is
// its latency chain plus the instructions every warp issues for the reduction, so the CTA
// is 4 warps -- one per SM sub-partition -- each thread owning VPT = n / 128 vertices:
//   - the input sits in shared memory: the keys of W's triangle (weights, n <= 300) or X^T
//     (points, n * d * 4 bytes <= ~200 KB).  Weights: a preceding many-CTA kernel validates
//     W (a1) and writes the triangle's keys contiguously, column by column, to global
//     memory; the Prim CTA pulls them in with ONE bulk copy (cp.async.bulk) -- one SM
//     alone would need ~10 us per pass over the n^2 elements (its 4 issue slots are the
//     limit).  Points: the CTA's 1024 threads load and validate X themselves (it is small);
//     warps 4..31 then exit (the loop synchronises on named barrier 1 of 128 threads);
//   - thread t owns the vertices u = t + s * 128, their keys in registers;
//   - per step: relax the owned keys, warp argmin with two redux.sync (the minimum key,
//     then the smallest index holding it), one __syncthreads on a double-buffered table of
//     the 4 warp winners packed as key << 32 | index, and every thread takes their minimum
//     (so no second barrier; ties go to the smallest index, as in the oracle's Prim);
//   - after the loop the CTA writes pi, pos = pi^-1, rowpos = iota and every level of the
//     sparse table over h (the fill's a6 preparation), so the fill follows directly.
// Keys are 32-bit: weights orderable(+-w) (-0 -> +0, Q5); points the bits of the
// non-negative R1 squared distance (or the L1 / L-inf distance), so u32 order = value
// order.  0xFFFFFFFF marks a visited vertex, 0xFFFFFFFE an unreached one.
#include <algorithm>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace appd {

constexpr int PRIM_THREADS = 128;            // the Prim loop: at most 4 warps
constexpr int PRIM_LOAD_THREADS = 1024;      // the load / validation phase: the whole CTA
constexpr int PRIM_LB = 4;                   // independent 16-byte loads in flight per thread
constexpr uint32_t PRIM_VISITED = 0xFFFFFFFFu, PRIM_FAR = 0xFFFFFFFEu;
constexpr int PRIM_MAX_N_WEIGHTS = 300;          // upper triangle in shared memory
constexpr size_t PRIM_SMEM_LIMIT = 225 * 1024;  // of the 227 KB opt-in maximum

enum PrimMode { PM_WEIGHTS = 0, PM_R1 = 1, PM_L1 = 2, PM_LINF = 3 };

struct PrimArgs {
  const uint32_t* keys;  // weights mode: the packed triangle keys (k_prim_pack), padded to 16 bytes
  const float* X;  // points mode: n x d
  int n, d, sense;
  u64* bad;        // validation: [nonfinite, diagonal, asymmetric] first offenders (atomicMin)
  int validate;
  int* pi;         // outputs (world 1 or replicated): leaf order, positions, identity row order
  int* pos;
  int* rowpos;
  float* ST;       // sparse table over h: levels x stride, level 0 = h
  int64_t stride;
  int levels;
  float* M;        // fused fill (small n): rows [row0, row0 + rows) of the APPD, else nullptr
  int64_t row0, rows;
  unsigned long long* dbg;  // development builds: %globaltimer at the phase boundaries (or null)
};

__device__ __forceinline__ unsigned long long prim_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t prim_key_of_weight(float w, int sense) {
  const float x = sense > 0 ? w : -w;
  return orderable(x + 0.0f);  // -0 -> +0 (Q5)
}

__device__ __forceinline__ float prim_weight_of_key(uint32_t k, int sense) {
  const float x = from_orderable(k);
  return (sense > 0 ? x : -x) + 0.0f;  // widest: -(+0) -> +0 again
}

__device__ __forceinline__ int tri_of(int a, int b) {  // a != b
  const int u = a < b ? a : b, v = a < b ? b : a;
  return v * (v - 1) / 2 + u;
}

// warp argmin of (key, idx): the minimum key, then the smallest index holding it
__device__ __forceinline__ void warp_argmin(uint32_t& key, int& idx) {
  const uint32_t m = __reduce_min_sync(0xffffffffu, key);
  idx = (int)__reduce_min_sync(0xffffffffu, key == m ? (uint32_t)idx : 0xFFFFFFFFu);
  key = m;
}

template <int NT>
__device__ __forceinline__ void prim_bar() {
  if (NT > 32) asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  else __syncwarp();
}

// NT threads run the loop: one warp (no barrier at all) up to n = 32 * VPT, else 4 warps
template <int VPT, int MODE, bool WIDEST, int NT>
__global__ void __launch_bounds__(PRIM_LOAD_THREADS, 1) k_prim(const PrimArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NW = NT / 32;
  __shared__ __align__(16) unsigned long long wbest[2][NW];
  __shared__ unsigned long long sbad[3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = A.n, d = A.d;
  float* in = reinterpret_cast<float*>(smem);  // weights: tri(n); points: X^T (d x n)
  const int in_words = MODE == PM_WEIGHTS ? (n * (n - 1) / 2 + 3) / 4 * 4 : n * d;
  int* spi = reinterpret_cast<int*>(in + in_words);
  int* spos = spi + n;
  // the sparse table over h: every level (fused fill) or two ping-pong rows of n
  float* sST = reinterpret_cast<float*>(spos + n);
  float* sh = sST;
  const bool fuse = A.M != nullptr;
  if (tid < 3) sbad[tid] = KEY_NONE;
  if (A.dbg && tid == 0) A.dbg[0] = prim_now();
  __syncthreads();

  // ---- the input into shared memory (a1 validation: weights in k_prim_pack, points here) ----
  const bool vec = (reinterpret_cast<uintptr_t>(A.X) & 15) == 0 && (d & 3) == 0;
  if (MODE == PM_WEIGHTS) {
    __shared__ __align__(8) uint64_t bar;
    const uint32_t bytes = (uint32_t)((in_words * 4 + 15) & ~15);
    if (tid == 0) {
      ptx::mbar_init(&bar, 1);
      ptx::fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      ptx::mbar_expect_tx(&bar, bytes);
      ptx::bulk_g2s(in, A.keys, bytes, &bar);
    }
    ptx::mbar_wait(&bar, 0);
  } else {
    const int total = vec ? n * d / 4 : n * d;
    for (int q = tid; q < total; q += PRIM_LOAD_THREADS) {
      float4 x4;
      const int cnt = vec ? 4 : 1;
      if (vec) x4 = __ldg(reinterpret_cast<const float4*>(A.X) + q);
      else x4.x = __ldg(A.X + q);
#pragma unroll
      for (int t = 0; t < 4; t++) {
        if (t >= cnt) break;
        const float x = t == 0 ? x4.x : t == 1 ? x4.y : t == 2 ? x4.z : x4.w;
        const int e = q * cnt + t;
        const int p = e / d, k = e - p * d;
        if (A.validate && !isfinite(x)) atomicMin(&sbad[0], (unsigned long long)e);
        in[k * n + p] = x;
      }
    }
  }
  __syncthreads();
  if (tid < 3 && A.validate && sbad[tid] != KEY_NONE) atomicMin(A.bad + tid, sbad[tid]);
  if (tid >= NT && !fuse) return;  // the loop runs on NT threads (named barrier 1 of NT, or one warp)
  if (tid < NT) {  // the other warps wait at barrier 0 for the fused fill
  if (A.dbg && tid == 0) A.dbg[1] = prim_now();

  // ---- Prim: start at vertex 0 (the oracle's R2) ----
  uint32_t key[VPT], vm[VPT];  // vm: all ones once visited (or padding), so key | vm stays visited
  int tu[VPT];                 // weights: u (u - 1) / 2, the start of the stored column u
#pragma unroll
  for (int s = 0; s < VPT; s++) {
    const int u = tid + s * NT;
    key[s] = (u < n && u != 0) ? PRIM_FAR : PRIM_VISITED;
    vm[s] = (u < n && u != 0) ? 0u : 0xFFFFFFFFu;
    const int uc = min(u, n - 1);
    tu[s] = uc * (uc - 1) / 2;
  }
  if (tid == 0) spi[0] = 0;
  int v = 0;
  for (int step = 1; step < n; step++) {
    const int par = step & 1;
    // relax every owned key against v, branch-free so the VPT updates overlap (the
    // visited / padding slots compute on a clamped index and are masked afterwards)
    uint32_t kw[VPT];
    if (MODE == PM_WEIGHTS) {
      const int base = v * (v - 1) / 2;  // column v of the stored triangle holds the u < v
      const uint32_t* ink = reinterpret_cast<const uint32_t*>(in);
#pragma unroll
      for (int s = 0; s < VPT; s++) {
        const int u = min(tid + s * NT, n - 1);
        kw[s] = ink[u < v ? base + u : tu[s] + v];  // u == v: tri(v, v) is in bounds, masked by vm
      }
    } else {
      float acc[VPT];
#pragma unroll
      for (int s = 0; s < VPT; s++) acc[s] = 0.0f;
      for (int k = 0; k < d; k++) {
        const float xv = in[k * n + v];
#pragma unroll
        for (int s = 0; s < VPT; s++) {
          const float t = __fsub_rn(in[k * n + min(tid + s * NT, n - 1)], xv);
          if (MODE == PM_R1) acc[s] = __fmaf_rn(t, t, acc[s]);
          else if (MODE == PM_L1) acc[s] = __fadd_rn(acc[s], fabsf(t));
          else acc[s] = fmaxf(acc[s], fabsf(t));
        }
      }
#pragma unroll
      // widest: the order-reversing map of the non-negative distance bits
      for (int s = 0; s < VPT; s++) kw[s] = A.sense > 0 ? __float_as_uint(acc[s]) : (~__float_as_uint(acc[s]) & 0x7FFFFFFFu);
    }
    uint32_t bk = PRIM_VISITED;
    int bi = 0;
#pragma unroll
    for (int s = 0; s < VPT; s++) {
      key[s] = min(key[s], kw[s] | vm[s]);
      const bool better = key[s] < bk;  // s ascending: ties keep the smaller index
      bk = better ? key[s] : bk;
      bi = better ? tid + s * NT : bi;
    }
    warp_argmin(bk, bi);
    if (NW > 1) {
      if (lane == 0) wbest[par][warp] = (unsigned long long)bk << 32 | (uint32_t)bi;
      prim_bar<NT>();
      unsigned long long b = wbest[par][0];
#pragma unroll
      for (int w = 1; w < NW; w++) b = min(b, wbest[par][w]);
      bk = (uint32_t)(b >> 32);
      bi = (int)(uint32_t)b;
    }
    v = bi;
    if (tid == 0) {
      spi[step] = v;
      sh[step - 1] = __uint_as_float(bk);  // the raw key; weights after the loop
    }
#pragma unroll
    for (int s = 0; s < VPT; s++)
      if (tid + s * NT == v) key[s] = vm[s] = PRIM_VISITED;
  }
  prim_bar<NT>();

  if (A.dbg && tid == 0) A.dbg[2] = prim_now();
  // ---- fill preparation (a6): pi, pos, rowpos, sparse table over h ----
  const int m = n - 1;
  for (int a = tid; a < n; a += NT) {
    const int p = spi[a];
    A.pi[a] = p;
    spos[p] = a;
    if (!fuse) {
      A.pos[p] = a;
      A.rowpos[a] = a;
    }
  }
  for (int i = tid; i < m; i += NT) {
    const uint32_t k = __float_as_uint(sh[i]);
    const uint32_t kp = A.sense > 0 ? k : (~k & 0x7FFFFFFFu);  // points: the distance bits again
    const float h = MODE == PM_WEIGHTS ? prim_weight_of_key(k, A.sense)
                    : MODE == PM_R1    ? __fsqrt_rn(__uint_as_float(kp))  // APPD(sqrtf o d2), App. A.4
                                       : __uint_as_float(kp);
    sh[i] = h;
    A.ST[i] = h;
  }
  for (int k = 1; k < A.levels; k++) {
    prim_bar<NT>();
    float* prev = fuse ? sST + (k - 1) * n : sST + ((k - 1) & 1) * n;
    float* cur = fuse ? sST + k * n : sST + (k & 1) * n;
    const int half = 1 << (k - 1), cnt = m - (1 << k) + 1;
    for (int i = tid; i < cnt; i += NT) {
      const float x = WIDEST ? fminf(prev[i], prev[i + half]) : fmaxf(prev[i], prev[i + half]);
      cur[i] = x;
      if (!fuse) A.ST[(int64_t)k * A.stride + i] = x;
    }
  }
  if (A.dbg && tid == 0) A.dbg[3] = prim_now();
  }  // tid < NT
  if (!fuse) return;
  // ---- fused fill (a7) for small n: M[i][j] = RMQ(pos i, pos j) from shared memory ----
  __syncthreads();
  // n <= 512: each pass covers 1024 / n whole rows (thread t: row t / n, column t % n)
  const int rpp = PRIM_LOAD_THREADS / n, j = tid % n, r0 = tid / n;
  if (r0 < rpp) {
    const int b = spos[j];
    for (int r = r0; r < (int)A.rows; r += rpp) {
      const int a = spos[A.row0 + r];
      float v = 0.0f;
      if (a != b) {
        const int l = min(a, b), rr = max(a, b), k = 31 - __clz(rr - l);
        const float x = sST[k * n + l], y = sST[k * n + rr - (1 << k)];
        v = WIDEST ? fminf(x, y) : fmaxf(x, y);
      }
      __stcs(A.M + (int64_t)r * n + j, v);
    }
  }
}

// Weights mode, a1 + packing: CTA i reads row i of W.  Non-finite entries and a nonzero
// diagonal are recorded at their row-major index; W[i][j] is compared with W[j][i]
// (bitwise after -0 -> +0) for j < i and the pair (j, i) recorded; and the keys of
// W[i][0..i-1] -- the stored triangle's column i, tri(j, i) = i (i - 1) / 2 + j -- are
// written contiguously.
__global__ void __launch_bounds__(256) k_prim_pack(const float* __restrict__ W, int n, int sense, int validate,
                                                   u64* __restrict__ bad, uint32_t* __restrict__ keys) {
  const int i = blockIdx.x;
  const float* Wi = W + (int64_t)i * n;
  u64 b0 = KEY_NONE, b1 = KEY_NONE, b2 = KEY_NONE;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float w = __ldg(Wi + j);
    if (validate) {
      if (!isfinite(w)) b0 = min(b0, (u64)i * n + j);
      if (j == i && (__float_as_uint(w) & 0x7FFFFFFFu) != 0) b1 = (u64)i * n + j;
    }
    if (j < i) {
      const uint32_t k = prim_key_of_weight(w, sense);
      keys[i * (i - 1) / 2 + j] = k;
      if (validate && k != prim_key_of_weight(__ldg(W + (int64_t)j * n + i), sense)) b2 = min(b2, (u64)j * n + i);
    }
  }
  if (validate) {
    if (b0 != KEY_NONE) atomicMin(bad + 0, b0);
    if (b1 != KEY_NONE) atomicMin(bad + 1, b1);
    if (b2 != KEY_NONE) atomicMin(bad + 2, b2);
  }
}

// the fused fill keeps every level of the sparse table in shared memory; up to n = 512
// (1 MiB of output: ~3 us for one SM, against ~13 us for a separate many-CTA fill whose
// tiles are a chain of dependent L2 round trips)
constexpr int64_t PRIM_FUSE_MAX_N = 512;

static int prim_levels(int64_t n) {
  int levels = 1;
  while ((1ll << levels) <= n - 1) levels++;
  return levels;
}

static size_t prim_smem(int mode, int64_t n, int64_t d, bool fuse) {
  const size_t in = mode == PM_WEIGHTS ? (size_t)((n * (n - 1) / 2 + 3) / 4 * 4) : (size_t)(n * d);
  const size_t table = fuse ? (size_t)prim_levels(n) * n : 2 * (size_t)n;
  return 4 * (in + 2 * (size_t)n + table) + 16;
}

bool prim_fuses_fill(int64_t n) { return n <= PRIM_FUSE_MAX_N; }

// can the single-CTA Prim take this problem?  (mode: 0 weights, 1 + metric points)
bool prim_fits(int64_t n, int64_t d, bool points) {
  if (n < 2 || n > 16 * PRIM_THREADS) return false;  // 16 keys per thread (64 registers at 1024 threads)
  if (!points) return n <= PRIM_MAX_N_WEIGHTS;
  return prim_smem(PM_R1, n, d, prim_fuses_fill(n)) <= PRIM_SMEM_LIMIT;
}

template <int MODE, bool WIDEST, int NT>
static void launch_prim_nt(appd_ctx* c, const PrimArgs& A, int vpt, size_t smem) {
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
#define APPD_PRIM_ATTR(V) \
  cudaFuncSetAttribute(k_prim<V, MODE, WIDEST, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PRIM_SMEM_LIMIT)
    APPD_PRIM_ATTR(1);
    APPD_PRIM_ATTR(2);
    APPD_PRIM_ATTR(4);
    APPD_PRIM_ATTR(8);
    APPD_PRIM_ATTR(16);
#undef APPD_PRIM_ATTR
    setup_done(attr, c);
  }
  switch (vpt) {
    case 1: k_prim<1, MODE, WIDEST, NT><<<1, PRIM_LOAD_THREADS, smem, c->stream>>>(A); break;
    case 2: k_prim<2, MODE, WIDEST, NT><<<1, PRIM_LOAD_THREADS, smem, c->stream>>>(A); break;
    case 4: k_prim<4, MODE, WIDEST, NT><<<1, PRIM_LOAD_THREADS, smem, c->stream>>>(A); break;
    case 8: k_prim<8, MODE, WIDEST, NT><<<1, PRIM_LOAD_THREADS, smem, c->stream>>>(A); break;
    default: k_prim<16, MODE, WIDEST, NT><<<1, PRIM_LOAD_THREADS, smem, c->stream>>>(A); break;
  }
}

// one warp (no barrier per step) while 16 keys per lane cover n, else 4 warps
template <int MODE, bool WIDEST>
static appd_status launch_prim_mode(appd_ctx* c, const PrimArgs& A, int64_t n, size_t smem) {
  const int nt = n <= 4 * 32 ? 32 : PRIM_THREADS;  // one warp only while it has few keys per lane
  int vpt = 1;
  while ((int64_t)vpt * nt < n) vpt *= 2;
  if (nt == 32) launch_prim_nt<MODE, WIDEST, 32>(c, A, vpt, smem);
  else launch_prim_nt<MODE, WIDEST, PRIM_THREADS>(c, A, vpt, smem);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

// One launch: validation (if bad != nullptr) + Prim + pi / pos / rowpos / sparse table.
appd_status launch_prim(appd_ctx* c, const float* W, const float* X, int64_t n, int64_t d, int sense, int metric,
                        u64* bad, int* pi, int* pos, int* rowpos, float* ST, int64_t stride, int levels, float* M,
                        int64_t row0, int64_t rows) {
  const bool points = X != nullptr;
  if (!prim_fits(n, d, points)) return fail(c, APPD_ERR_UNSUPPORTED, "Prim variant: n = %lld too large", (long long)n);
  PrimArgs A;
  A.keys = nullptr;
  if (!points) {
    const int64_t tw = (n * (n - 1) / 2 + 3) / 4 * 4;
    uint32_t* keys = (uint32_t*)ws(c, S_PRIM, sizeof(uint32_t) * tw + 64);
    if (!keys) return fail(c, APPD_ERR_OUT_OF_MEMORY, "Prim key triangle");
    k_prim_pack<<<(unsigned)n, 256, 0, c->stream>>>(W, (int)n, sense, bad != nullptr, bad, keys);
    APPD_LAUNCHED(c);
    A.keys = keys;
  }
  A.X = X;
  A.n = (int)n;
  A.d = points ? (int)d : 0;
  A.sense = sense;
  A.bad = bad;
  A.validate = bad != nullptr;
  A.pi = pi;
  A.pos = pos;
  A.rowpos = rowpos;
  A.ST = ST;
  A.stride = stride;
  A.levels = levels;
  A.M = (M && prim_fuses_fill(n)) ? M : nullptr;
  A.row0 = row0;
  A.rows = rows;
  A.dbg = nullptr;
#ifdef APPD_DEV_HOOKS
  static unsigned long long* dbg = nullptr;
  static unsigned long long hd[4];
  if (dev_env("APPD_PRIM_TIMES")) {
    if (!dbg) cudaMalloc(&dbg, 64);
    A.dbg = dbg;
  }
#endif
  const int mode = points ? 1 + metric : PM_WEIGHTS;
  const size_t smem = prim_smem(mode, n, d, A.M != nullptr);
  if (!points) {
    appd_status st = sense > 0 ? launch_prim_mode<PM_WEIGHTS, false>(c, A, n, smem)
                               : launch_prim_mode<PM_WEIGHTS, true>(c, A, n, smem);
#ifdef APPD_DEV_HOOKS
    if (A.dbg) {
      cudaMemcpy(hd, A.dbg, 32, cudaMemcpyDeviceToHost);
      fprintf(stderr, "[prim] n %lld weights: load %.1f us, loop %.1f us (%.1f ns/step), prep %.1f us\n", (long long)n,
              (hd[1] - hd[0]) * 1e-3, (hd[2] - hd[1]) * 1e-3, (double)(hd[2] - hd[1]) / (n - 1), (hd[3] - hd[2]) * 1e-3);
    }
#endif
    return st;
  }
  const bool widest = sense < 0;
  appd_status st = mode == PM_R1 ? (widest ? launch_prim_mode<PM_R1, true>(c, A, n, smem)
                                           : launch_prim_mode<PM_R1, false>(c, A, n, smem))
                   : mode == PM_L1 ? (widest ? launch_prim_mode<PM_L1, true>(c, A, n, smem)
                                             : launch_prim_mode<PM_L1, false>(c, A, n, smem))
                                   : (widest ? launch_prim_mode<PM_LINF, true>(c, A, n, smem)
                                             : launch_prim_mode<PM_LINF, false>(c, A, n, smem));
#ifdef APPD_DEV_HOOKS
  if (A.dbg) {
    cudaMemcpy(hd, A.dbg, 32, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[prim] n %lld d %lld: load %.1f us, loop %.1f us (%.1f ns/step), prep %.1f us\n", (long long)n,
            (long long)d, (hd[1] - hd[0]) * 1e-3, (hd[2] - hd[1]) * 1e-3,
            (double)(hd[2] - hd[1]) / (n - 1), (hd[3] - hd[2]) * 1e-3);
  }
#endif
  return st;
}

}  // namespace appd
