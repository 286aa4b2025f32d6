// k_dendro.cu -- dendrogram on the GPU: the leaf order pi and
// merge heights h from the MST, without a sequential union-find.
//
// P:L149 reads the APPD off the single-linkage dendrogram; any leaf order of it works
// (DESIGN.md "leaf order").  Prim's visit order from a root is one (SURVEY App. A.3:
// Prim never leaves a component of the threshold graph before finishing it), with
// h[a] = the key of pi_{a+1} when Prim adds it = the weight of its tree edge.  On the
// MST itself, Prim's order is a pre-order of the "record tree": rooting the MST at
// vertex 0, let val(v) be the rank (position in the ascending key order) of v's parent
// edge; the record parent of v is its nearest ancestor a with val(a) > val(v) (the
// root has val = +inf).  Visiting the record tree in pre-order with children in
// ascending val reproduces Prim's priority order: Prim finishes everything reachable
// below a weight before crossing a heavier edge, and the heavier edges on the path to v
// are exactly v's record ancestors.  (Checked against a heap-based Prim on 300 random
// trees while building this, and end to end against the oracle by the parity tests.)
//
// Steps, all data-parallel:
//   A  arcs (2 per edge) sorted by source = adjacency lists
//   B  Euler-tour successor of every arc, cut at the root
//   C  list ranking (pointer jumping) -> tour positions; the earlier arc of an edge
//      points downwards: parent and val of every vertex
//   D  nearest heavier ancestor by binary lifting (2^j-th ancestor + max val on the way)
//   E  children sorted by (record parent, val) -- the keys are laid out by val (edge
//      rank), so a stable radix sort on the record-parent bits alone gives that order
//      (2 digit passes at n = 65536 instead of 4); Euler tour of the record tree, list
//      ranking, pre-order index = 1 + down arcs before the vertex's down arc
//   F  pi[pre(v)] = v, h[a] = weight of the parent edge of pi[a+1]
#include <cooperative_groups.h>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace appd {

namespace {

__global__ void k_arcs(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev, int m,
                       int* __restrict__ src, int* __restrict__ arc) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < 2 * m; a += gridDim.x * blockDim.x) {
    const int e = a >> 1;
    src[a] = (a & 1) ? ev[e] : eu[e];
    arc[a] = a;
  }
}

// adjacency ranges of the sorted sources + inverse position of every arc
__global__ void k_adj(const int* __restrict__ ssrc, const int* __restrict__ sarc, int L, int* __restrict__ start,
                      int* __restrict__ end, int* __restrict__ posarc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const int x = ssrc[i];
    if (i == 0 || ssrc[i - 1] != x) start[x] = i;
    if (i == L - 1 || ssrc[i + 1] != x) end[x] = i + 1;
    posarc[sarc[i]] = i;
  }
}

// succ(x -> y) = the arc after (y -> x) in y's adjacency, cyclically; the tour starts
// with the root's first arc and the arc leading back into it ends the list (-1)
__global__ void k_euler_succ(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev, int m,
                             const int* __restrict__ sarc, const int* __restrict__ start,
                             const int* __restrict__ end, const int* __restrict__ posarc, int root,
                             int* __restrict__ succ, int* __restrict__ rank) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < 2 * m; a += gridDim.x * blockDim.x) {
    const int e = a >> 1;
    const int y = (a & 1) ? eu[e] : ev[e];  // head of a
    int i = posarc[a ^ 1] + 1;
    if (i == end[y]) i = start[y];
    const int s = (y == root && i == start[y]) ? -1 : sarc[i];
    succ[a] = s;
    rank[a] = s < 0 ? 0 : 1;
  }
}

// the earlier arc of each edge points from parent to child
__global__ void k_orient(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev, int m,
                         const int* __restrict__ rank, int* __restrict__ parent, int* __restrict__ val,
                         int* __restrict__ child_of) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    // larger rank (more arcs after it) = earlier in the tour
    const bool down0 = rank[2 * e] > rank[2 * e + 1];
    const int c = down0 ? ev[e] : eu[e], p = down0 ? eu[e] : ev[e];
    parent[c] = p;
    val[c] = e;
    child_of[e] = c;
  }
}

__global__ void k_lift0(const int* __restrict__ parent, const int* __restrict__ val, int n, int2* __restrict__ jm) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const int p = parent[x];
    jm[x] = make_int2(p, val[p]);
  }
}
// record parent of v: its nearest ancestor with a larger val; sort key (rpar, val)
__global__ void k_record_parent(const int2* __restrict__ jm, int levels, int n,
                                const int* __restrict__ parent, const int* __restrict__ val, int root, int sh,
                                unsigned long long* __restrict__ key) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (v == root) continue;
    const int w = val[v];
    int cur = v;
    for (int j = levels - 1; j >= 0; j--) {
      const int2 q = jm[(int64_t)j * n + cur];  // (2^j-th ancestor, max val on the way)
      if (q.y < w) cur = q.x;
    }
    const int rp = parent[cur];
    key[w] = ((unsigned long long)(unsigned)rp << sh) | (unsigned)w;  // one entry per edge rank
  }
}

// record-tree Euler tour over the sorted children S[i] = (rpar, val): arcs 2i (down
// into child i) and 2i+1 (back up); first child of x and the S index of each vertex
__global__ void k_rt_index(const unsigned long long* __restrict__ S, int m, int sh, const int* __restrict__ child_of,
                           int* __restrict__ first, int* __restrict__ sidx) {
  const unsigned long long lo = (1ull << sh) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int rp = (int)(S[i] >> sh);
    const int v = child_of[(int)(S[i] & lo)];
    sidx[v] = i;
    if (i == 0 || (int)(S[i - 1] >> sh) != rp) first[rp] = i;
  }
}
__global__ void k_rt_succ(const unsigned long long* __restrict__ S, int m, int sh, const int* __restrict__ child_of,
                          const int* __restrict__ first, const int* __restrict__ sidx, int root,
                          int* __restrict__ succ, int* __restrict__ rank) {
  const unsigned long long lo = (1ull << sh) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int rp = (int)(S[i] >> sh);
    const int v = child_of[(int)(S[i] & lo)];
    const int fc = first[v];
    const int sd = fc >= 0 ? 2 * fc : 2 * i + 1;  // into the first child, else straight back up
    int su;
    if (i + 1 < m && (int)(S[i + 1] >> sh) == rp) su = 2 * (i + 1);  // next sibling
    else su = rp == root ? -1 : 2 * sidx[rp] + 1;                    // up from the parent
    succ[2 * i] = sd;
    succ[2 * i + 1] = su;
    rank[2 * i] = 1;
    rank[2 * i + 1] = su < 0 ? 0 : 1;
  }
}

// flag[position of down arc] = 1 (positions = L - 1 - rank)
__global__ void k_down_flags(const int* __restrict__ rank, int m, int* __restrict__ flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    flag[2 * m - 1 - rank[2 * i]] = 1;
}
__global__ void k_emit(const unsigned long long* __restrict__ S, int m, int sh, const int* __restrict__ child_of,
                       const int* __restrict__ rank, const int* __restrict__ downs_before,
                       const float* __restrict__ ew, int root, int32_t* __restrict__ pi, float* __restrict__ h) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int e = (int)(S[i] & ((1ull << sh) - 1));
    const int v = child_of[e];
    const int pre = 1 + downs_before[2 * m - 1 - rank[2 * i]];
    pi[pre] = v;
    h[pre - 1] = ew[e];  // Prim's key of v: the weight of its tree edge
    if (i == 0) pi[0] = root;
  }
}

// all pointer-jumping steps in one cooperative launch (grid-wide barrier per step).
// Each thread keeps its E arcs' (succ, rank) in registers, so a step is ONE dependent
// 8-byte load of the successor's pair from the previous step's buffer (ping-pong A/B).
template <int E>
__global__ void k_rank_coop(const int* __restrict__ succ0, const int* __restrict__ rank0, int2* __restrict__ A,
                            int2* __restrict__ B, int* __restrict__ out_rank, int L, int steps, unsigned* bar) {
  const int T = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  int nx[E], rk[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int a = tid + e * T;
    nx[e] = a < L ? succ0[a] : -1;
    rk[e] = a < L ? rank0[a] : 0;
    if (a < L) A[a] = make_int2(nx[e], rk[e]);
  }
  coop_grid_sync(bar);
  for (int s = 0; s < steps; s++) {
    const int2* in = (s & 1) ? B : A;
    int2* out = (s & 1) ? A : B;
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int a = tid + e * T;
      if (a >= L) continue;
      if (nx[e] >= 0) {
        const int2 q = in[nx[e]];
        rk[e] += q.y;
        nx[e] = q.x;
      }
      out[a] = make_int2(nx[e], rk[e]);
    }
    coop_grid_sync(bar);
  }
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int a = tid + e * T;
    if (a < L) out_rank[a] = rk[e];
  }
}

// all binary-lifting levels in one cooperative launch: level j of x from level j-1 of
// its 2^(j-1)-th ancestor (own pair in registers: one dependent 8-byte load per level)
template <int E>
__global__ void k_lift_coop(int2* __restrict__ jm, int n, int levels, unsigned* bar) {
  const int T = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  int2 cur[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int x = tid + e * T;
    cur[e] = x < n ? jm[x] : make_int2(0, 0);
  }
  for (int j = 1; j < levels; j++) {
    const int2* in = jm + (size_t)(j - 1) * n;
    int2* out = jm + (size_t)j * n;
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int x = tid + e * T;
      if (x >= n) continue;
      const int2 q = in[cur[e].x];
      cur[e] = make_int2(q.x, max(cur[e].y, q.y));
      out[x] = cur[e];
    }
    coop_grid_sync(bar);
  }
}

// Barrier of the fused tours: the whole cooperative grid (one CTA per SM), or -- for
// small trees (n <= 16384) -- one thread-block cluster of kTourCluster CTAs, whose
// hardware barrier (barrier.cluster.arrive.release / wait.acquire: the CTAs' global
// writes before it are visible to the cluster after it) costs a fraction of a grid-wide
// one.  The tours are chains of ~70 barrier-separated steps on arrays of a few hundred
// KB, so at those sizes the barrier is the step.
template <bool CL>
__device__ __forceinline__ void all_sync(unsigned* bar) {
  if constexpr (CL) cg::this_cluster().sync();
  else coop_grid_sync(bar);
}

// ---------------------------------------------------------------------------
// Fused cooperative versions of the two tours (one launch each instead of 6-8):
//   k_tour1: Euler successors of the MST (k_euler_succ), list ranking, orientation
//            (k_orient + the root fix-ups), binary lifting (k_lift0 + k_lift_coop);
//   k_tour2: record-tree index and successors (k_rt_index, k_rt_succ), list ranking,
//            down flags, their exclusive scan and the outputs (k_emit).
// The same operations in the same order, separated by grid-wide barriers.
// ---------------------------------------------------------------------------
template <int E, bool CL>
__device__ __forceinline__ void pj_steps(int (&nx)[E], int (&rk)[E], int2* A, int2* B, int L, int steps, int tid,
                                         int T, unsigned* bar) {
  for (int s = 0; s < steps; s++) {
    const int2* in = (s & 1) ? B : A;
    int2* out = (s & 1) ? A : B;
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int a = tid + e * T;
      if (a >= L) continue;
      if (nx[e] >= 0) {
        const int2 q = in[nx[e]];
        rk[e] += q.y;
        nx[e] = q.x;
      }
      out[a] = make_int2(nx[e], rk[e]);
    }
    all_sync<CL>(bar);
  }
}

// exclusive prefix sum of in[0..count) into out over the whole cooperative grid: block b
// scans its contiguous segment, the block totals are added in order (grid barriers inside;
// every thread of the grid must call it)
template <bool CL>
__device__ void grid_exclusive_scan(const int* in, int* out, int count, int* blocksum, unsigned* bar) {
  __shared__ int wsum[32];
  __shared__ int carry_s;
  const int Sg = (count + gridDim.x - 1) / gridDim.x;
  const int lo_i = min(count, (int)blockIdx.x * Sg), hi_i = min(count, lo_i + Sg);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = lo_i; base < hi_i; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int f = i < hi_i ? in[i] : 0;
    int x = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    if (i < hi_i) out[i] = carry_s + (warp ? wsum[warp - 1] : 0) + x - f;
    __syncthreads();
    if (threadIdx.x == 0) carry_s += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) blocksum[blockIdx.x] = carry_s;
  all_sync<CL>(bar);
  const int off = blocks_before(blocksum);
  for (int i = lo_i + threadIdx.x; i < hi_i; i += blockDim.x) out[i] += off;
  all_sync<CL>(bar);
}

template <int E, bool CL>
__global__ void __launch_bounds__(1024) k_tour1(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev, int m,
                                                int n, int* sarc, int* start, int* end, int* posarc, int* deg,
                                                int* cursor, int* blocksum, int root, int2* A, int2* B, int* rkout,
                                                int* parent, int* val, int* child_of, int2* jm, int levels,
                                                int steps, unsigned* bar, int sh,
                                                unsigned long long* __restrict__ key) {
  const int T = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int L = 2 * m;
  // adjacency (CSR by source vertex; the order inside a list is irrelevant: the rooted
  // orientation, the only thing this tour produces, is unique)
  for (int x = tid; x < n; x += T) {
    deg[x] = 0;
    cursor[x] = 0;
  }
  all_sync<CL>(bar);
  for (int ed = tid; ed < m; ed += T) {
    atomicAdd(deg + eu[ed], 1);
    atomicAdd(deg + ev[ed], 1);
  }
  all_sync<CL>(bar);
  grid_exclusive_scan<CL>(deg, start, n, blocksum, bar);
  for (int x = tid; x < n; x += T) end[x] = start[x] + deg[x];
  for (int a = tid; a < L; a += T) {
    const int src = (a & 1) ? ev[a >> 1] : eu[a >> 1];
    const int p = start[src] + atomicAdd(cursor + src, 1);
    sarc[p] = a;
    posarc[a] = p;
  }
  all_sync<CL>(bar);
  int nx[E], rk[E];
#pragma unroll
  for (int e = 0; e < E; e++) {  // Euler successors (k_euler_succ)
    const int a = tid + e * T;
    nx[e] = -1;
    rk[e] = 0;
    if (a < L) {
      const int ed = a >> 1;
      const int y = (a & 1) ? eu[ed] : ev[ed];
      int i = posarc[a ^ 1] + 1;
      if (i == end[y]) i = start[y];
      nx[e] = (y == root && i == start[y]) ? -1 : sarc[i];
      rk[e] = nx[e] < 0 ? 0 : 1;
      A[a] = make_int2(nx[e], rk[e]);
    }
  }
  if (tid == 0) {
    val[root] = 0x7F7F7F7F;  // +inf: the root's parent edge
    parent[root] = root;
  }
  all_sync<CL>(bar);
  pj_steps<E, CL>(nx, rk, A, B, L, steps, tid, T, bar);
#pragma unroll
  for (int e = 0; e < E; e++)
    if (tid + e * T < L) rkout[tid + e * T] = rk[e];
  all_sync<CL>(bar);
  for (int ed = tid; ed < m; ed += T) {  // orientation (k_orient): the earlier arc points down
    const bool down0 = rkout[2 * ed] > rkout[2 * ed + 1];
    const int ch = down0 ? ev[ed] : eu[ed], p = down0 ? eu[ed] : ev[ed];
    parent[ch] = p;
    val[ch] = ed;
    child_of[ed] = ch;
  }
  all_sync<CL>(bar);
  int2 cur[E];
#pragma unroll
  for (int e = 0; e < E; e++) {  // lifting level 0 (k_lift0)
    const int x = tid + e * T;
    cur[e] = make_int2(0, 0);
    if (x < n) {
      const int p = parent[x];
      cur[e] = make_int2(p, val[p]);
      jm[x] = cur[e];
    }
  }
  all_sync<CL>(bar);
  for (int j = 1; j < levels; j++) {  // k_lift_coop
    const int2* in = jm + (size_t)(j - 1) * n;
    int2* out = jm + (size_t)j * n;
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int x = tid + e * T;
      if (x >= n) continue;
      const int2 q = in[cur[e].x];
      cur[e] = make_int2(q.x, max(cur[e].y, q.y));
      out[x] = cur[e];
    }
    all_sync<CL>(bar);
  }
  // record parents (k_record_parent): nearest ancestor with a larger val, by the lifting
  // levels just written; one key per edge rank
  for (int v = tid; v < n; v += T) {
    if (v == root) continue;
    const int w = val[v];
    int cur = v;
    for (int j = levels - 1; j >= 0; j--) {
      const int2 q = jm[(int64_t)j * n + cur];  // (2^j-th ancestor, max val on the way)
      if (q.y < w) cur = q.x;
    }
    key[w] = ((unsigned long long)(unsigned)parent[cur] << sh) | (unsigned)w;
  }
}

template <int E, bool CL>
__global__ void __launch_bounds__(1024) k_tour2(const unsigned long long* __restrict__ S, int m, int n, int sh,
                                                const int* __restrict__ child_of, int* first, int* sidx, int root,
                                                int2* A, int2* B, int* rkout, int* flag, int* downs, int* blocksum,
                                                const float* __restrict__ ew, int32_t* __restrict__ pi,
                                                float* __restrict__ h, int steps, unsigned* bar,
                                                int* __restrict__ pos, int* __restrict__ rowpos) {
  const int T = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int L = 2 * m;
  const unsigned long long lo = (1ull << sh) - 1;
  for (int x = tid; x < n; x += T) first[x] = -1;
  for (int q = tid; q <= L; q += T) flag[q] = 0;
  all_sync<CL>(bar);
  for (int i = tid; i < m; i += T) {  // k_rt_index
    const int rp = (int)(S[i] >> sh);
    const int v = child_of[(int)(S[i] & lo)];
    sidx[v] = i;
    if (i == 0 || (int)(S[i - 1] >> sh) != rp) first[rp] = i;
  }
  all_sync<CL>(bar);
  for (int i = tid; i < m; i += T) {  // k_rt_succ
    const int rp = (int)(S[i] >> sh);
    const int v = child_of[(int)(S[i] & lo)];
    const int fc = first[v];
    const int sd = fc >= 0 ? 2 * fc : 2 * i + 1;
    int su;
    if (i + 1 < m && (int)(S[i + 1] >> sh) == rp) su = 2 * (i + 1);
    else su = rp == root ? -1 : 2 * sidx[rp] + 1;
    A[2 * i] = make_int2(sd, 1);
    A[2 * i + 1] = make_int2(su, su < 0 ? 0 : 1);
  }
  all_sync<CL>(bar);
  int nx[E], rk[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int a = tid + e * T;
    const int2 v = a < L ? A[a] : make_int2(-1, 0);
    nx[e] = v.x;
    rk[e] = v.y;
  }
  pj_steps<E, CL>(nx, rk, A, B, L, steps, tid, T, bar);
#pragma unroll
  for (int e = 0; e < E; e++)
    if (tid + e * T < L) rkout[tid + e * T] = rk[e];
  all_sync<CL>(bar);
  for (int i = tid; i < m; i += T) flag[L - 1 - rkout[2 * i]] = 1;  // k_down_flags
  all_sync<CL>(bar);
  grid_exclusive_scan<CL>(flag, downs, L, blocksum, bar);
  for (int i = tid; i < m; i += T) {  // k_emit
    const int e = (int)(S[i] & lo);
    const int v = child_of[e];
    const int pre = 1 + downs[L - 1 - rkout[2 * i]];
    pi[pre] = v;
    h[pre - 1] = ew[e];
    if (pos) pos[v] = pre;  // (k_positions: pos = pi^-1)
    if (rowpos) rowpos[pre] = pre;
    if (i == 0) {
      pi[0] = root;
      if (pos) pos[root] = 0;
      if (rowpos) rowpos[0] = 0;
    }
  }
}

// one 1024-thread block per SM: the grid-wide barrier of every step is cheapest with
// the fewest blocks, and 148 x 1024 threads cover the 2(n-1) arcs in a few strides
constexpr int kCoopThreads = 1024;
constexpr int kTourCluster = 8;  // portable cluster size

// fused tour launch: cooperative (grid barrier) or one cluster of kTourCluster CTAs
appd_status launch_tour(appd_ctx* c, const void* fn, bool cl, int grid, void** args) {
  if (!cl) {
    APPD_CUDA(c, cudaLaunchCooperativeKernel(fn, grid, kCoopThreads, args, 0, c->stream));
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kTourCluster);
    cfg.blockDim = dim3(kCoopThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kTourCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    APPD_CUDA(c, cudaLaunchKernelExC(&cfg, fn, args));
  }
  c->launches++;
  return APPD_OK;
}
int coop_grid(appd_ctx* c, int items) {
  return std::max(1, std::min(c->sm_count, (items + kCoopThreads - 1) / kCoopThreads));
}

appd_status list_rank(appd_ctx* c, int L, int* succ0, int* rank0, int2* A, int2* B, int* out_rank) {
  int steps = 0;
  while ((1 << steps) < L) steps++;
  steps++;
  const int grid = coop_grid(c, L);
  const int E = (L + grid * kCoopThreads - 1) / (grid * kCoopThreads);
  unsigned* bar = grid_barrier_word(c);
  if (!bar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
  void* args[] = {&succ0, &rank0, &A, &B, &out_rank, &L, &steps, &bar};
  const void* fn = E <= 1 ? (const void*)k_rank_coop<1> : E <= 2 ? (const void*)k_rank_coop<2>
                 : E <= 4 ? (const void*)k_rank_coop<4> : E <= 8 ? (const void*)k_rank_coop<8> : nullptr;
  if (!fn) return fail(c, APPD_ERR_UNSUPPORTED, "GPU dendrogram: %d arcs", L);
  APPD_CUDA(c, cudaLaunchCooperativeKernel(fn, grid, kCoopThreads, args, 0, c->stream));
  c->launches++;
  return APPD_OK;
}

}  // namespace

// eu/ev/ew: MST edges in ascending key order (device); pi, h: device outputs
appd_status gpu_dendrogram(appd_ctx* c, const int32_t* eu, const int32_t* ev, const float* ew, int64_t n64,
                           int32_t* pi, float* h, int* pos_out, int* rowpos_out, bool* fused_pos) {
  if (fused_pos) *fused_pos = false;
  const int n = (int)n64, m = n - 1;
  if (n == 1) {
    APPD_CUDA(c, cudaMemsetAsync(pi, 0, sizeof(int32_t), c->stream));
    return APPD_OK;
  }
  const int L = 2 * m;
  int levels = 1;
  while ((1 << levels) < n) levels++;
  levels++;
  // workspace: int2 arrays first (8-byte aligned): lifting levels (levels x n), the two
  // pointer-jumping buffers (L each); then ints: 10 arc arrays of L (+2), 6 vertex
  // arrays of n, child_of (m); then the 64-bit record keys
  const size_t i2 = (size_t)levels * n + 2 * (size_t)L;
  const size_t ints = (size_t)10 * L + 8 * (size_t)n + 64;
  int2* w2 = (int2*)ws(c, S_DENDRO, sizeof(int2) * i2 + sizeof(int) * ints + sizeof(unsigned long long) * 2 * (size_t)m + 64);
  if (!w2) return fail(c, APPD_ERR_OUT_OF_MEMORY, "GPU dendrogram workspace");
  int2* jm = w2;
  int2* bufA = jm + (size_t)levels * n;
  int2* bufB = bufA + L;
  int* w = reinterpret_cast<int*>(bufB + L);
  int* src = w;
  int* arc = src + L;
  int* ssrc = arc + L;
  int* sarc = ssrc + L;
  int* succ0 = sarc + L;
  int* rank0 = succ0 + L;
  int* start = rank0 + L;
  int* end = start + n;
  int* posarc = end + n;  // L entries
  int* parent = posarc + L;
  int* val = parent + n;
  int* child_of = val + n;
  int* first = child_of + m;
  int* sidx = first + n;
  int* rk = sidx + n;              // L: tour ranks
  int* flag = rk + L;              // L + 1
  int* downs = flag + L + 1;       // L + 1
  unsigned long long* key = reinterpret_cast<unsigned long long*>(((uintptr_t)(downs + L + 8) + 15) & ~(uintptr_t)15);
  unsigned long long* S = key + m;
  const int gL = std::min(c->sm_count * 8, (L + 255) / 256), gn = std::min(c->sm_count * 8, (n + 255) / 256);
  const int root = 0;
  appd_status s;
  int sh = 1;
  while ((1 << sh) < n) sh++;
  int steps = 0;
  while ((1 << steps) < L) steps++;
  steps++;
  // one cluster when its threads cover the arcs in <= 4 strides, else the cooperative grid
  const bool cl = L <= kTourCluster * kCoopThreads;  // (measured: at 4 strides the grid is faster)
  const int cgrid = cl ? kTourCluster : coop_grid(c, L);
  const int cE = (L + cgrid * kCoopThreads - 1) / (cgrid * kCoopThreads);
  int* blocksum = (int*)ws(c, S_SCAN, sizeof(int) * (cgrid + 1) + 64);
  if (!blocksum) return fail(c, APPD_ERR_OUT_OF_MEMORY, "dendrogram scan workspace");
  unsigned* gbar = grid_barrier_word(c);
  if (!gbar) return fail(c, APPD_ERR_OUT_OF_MEMORY, "grid barrier word");
  if (cE <= 4) {
    // fused cooperative tours (the separate kernels below are the fallback)
    {
      // the adjacency (CSR) is built inside the tour: src / arc serve as degree / cursor
      int mm = m, nn = n, rt = root, lv = levels, st = steps, shh1 = sh;
      void* args[] = {&eu, &ev, &mm, &nn, &sarc, &start, &end, &posarc, &src, &arc, &blocksum, &rt, &bufA, &bufB,
                      &rk, &parent, &val, &child_of, &jm, &lv, &st, &gbar, &shh1, &key};
      const void* fn = cl ? (cE <= 1 ? (const void*)k_tour1<1, true> : cE <= 2 ? (const void*)k_tour1<2, true>
                                                         : (const void*)k_tour1<4, true>)
                          : (cE <= 1 ? (const void*)k_tour1<1, false> : cE <= 2 ? (const void*)k_tour1<2, false>
                                                         : (const void*)k_tour1<4, false>);
      if ((s = launch_tour(c, fn, cl, cgrid, args))) return s;
    }
    if ((s = sort_keys_u64_bits64(c, key, S, m, sh, 2 * sh))) return s;  // key[w] is in val order: a stable sort on rp
    {
      int mm = m, nn = n, shh = sh, rt = root, st = steps;
      void* args[] = {&S, &mm, &nn, &shh, &child_of, &first, &sidx, &rt, &bufA, &bufB, &rk, &flag, &downs, &blocksum,
                      &ew, &pi, &h, &st, &gbar, &pos_out, &rowpos_out};
      const void* fn = cl ? (cE <= 1 ? (const void*)k_tour2<1, true> : cE <= 2 ? (const void*)k_tour2<2, true>
                                                         : (const void*)k_tour2<4, true>)
                          : (cE <= 1 ? (const void*)k_tour2<1, false> : cE <= 2 ? (const void*)k_tour2<2, false>
                                                         : (const void*)k_tour2<4, false>);
      if ((s = launch_tour(c, fn, cl, cgrid, args))) return s;
    }
    if (fused_pos) *fused_pos = true;
    return APPD_OK;
  }
  // A: adjacency
  k_arcs<<<gL, 256, 0, c->stream>>>(eu, ev, m, src, arc);
  APPD_LAUNCHED(c);
  if ((s = sort_pairs_i32_bits(c, src, ssrc, arc, sarc, L, sh))) return s;
  k_adj<<<gL, 256, 0, c->stream>>>(ssrc, sarc, L, start, end, posarc);
  APPD_LAUNCHED(c);
  // B, C: Euler tour of the MST from the root, tour ranks
  k_euler_succ<<<gL, 256, 0, c->stream>>>(eu, ev, m, sarc, start, end, posarc, root, succ0, rank0);
  APPD_LAUNCHED(c);
  if ((s = list_rank(c, L, succ0, rank0, bufA, bufB, rk))) return s;
  // orientation: parent, val (edge rank of the parent edge), child of each edge
  APPD_CUDA(c, cudaMemsetAsync(val + root, 0x7F, sizeof(int), c->stream));  // +inf
  k_orient<<<gn, 256, 0, c->stream>>>(eu, ev, m, rk, parent, val, child_of);
  APPD_LAUNCHED(c);
  APPD_CUDA(c, cudaMemsetAsync(parent + root, 0, sizeof(int), c->stream));  // root = vertex 0 is its own parent
  // D: binary lifting, nearest heavier ancestor
  k_lift0<<<gn, 256, 0, c->stream>>>(parent, val, n, jm);
  APPD_LAUNCHED(c);
  {
    int nn = n, lv = levels;
    const int grid = coop_grid(c, n);
    const int E = (n + grid * kCoopThreads - 1) / (grid * kCoopThreads);
    const void* fn = E <= 1 ? (const void*)k_lift_coop<1> : E <= 2 ? (const void*)k_lift_coop<2>
                   : E <= 4 ? (const void*)k_lift_coop<4> : E <= 8 ? (const void*)k_lift_coop<8> : nullptr;
    if (!fn) return fail(c, APPD_ERR_UNSUPPORTED, "GPU dendrogram: n = %d", n);
    void* args[] = {&jm, &nn, &lv, &gbar};
    APPD_CUDA(c, cudaLaunchCooperativeKernel(fn, grid, kCoopThreads, args, 0, c->stream));
    c->launches++;
  }
  k_record_parent<<<gn, 256, 0, c->stream>>>(jm, levels, n, parent, val, root, sh, key);
  APPD_LAUNCHED(c);
  // E: record tree, children ascending by val
  if ((s = sort_keys_u64_bits64(c, key, S, m, sh, 2 * sh))) return s;  // key[w] is in val order: a stable sort on rp
  APPD_CUDA(c, cudaMemsetAsync(first, 0xFF, sizeof(int) * n, c->stream));
  k_rt_index<<<gn, 256, 0, c->stream>>>(S, m, sh, child_of, first, sidx);
  APPD_LAUNCHED(c);
  k_rt_succ<<<gn, 256, 0, c->stream>>>(S, m, sh, child_of, first, sidx, root, succ0, rank0);
  APPD_LAUNCHED(c);
  if ((s = list_rank(c, L, succ0, rank0, bufA, bufB, rk))) return s;
  APPD_CUDA(c, cudaMemsetAsync(flag, 0, sizeof(int) * (L + 1), c->stream));
  k_down_flags<<<gn, 256, 0, c->stream>>>(rk, m, flag);
  APPD_LAUNCHED(c);
  if ((s = exclusive_scan_i32(c, flag, downs, L))) return s;
  // F: outputs
  k_emit<<<gn, 256, 0, c->stream>>>(S, m, sh, child_of, rk, downs, ew, root, pi, h);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
