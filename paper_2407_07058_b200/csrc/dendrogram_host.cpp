// dendrogram_host.cpp -- MST edges (sorted ascending by key) -> leaf order pi and
// merge heights h (SURVEY §8(a) row a5, v1 on the host).
//
// P:L98 removes the MST edges "from large to small"; replaying that removal
// backwards is Kruskal's union order, whose merges form the single-linkage
// dendrogram ("read off the distances from the resulting dendrogram").
// Each cluster keeps its members as a linked list; merging cluster A (of u) and
// B (of v) at height w appends B's list to A's and stores w on A's old tail.
// Walking the final list gives pi, and h[a] (the value stored between pi_a and
// pi_{a+1}) is the height at which they were first joined -- the largest merge
// height between any two consecutive leaves of a cluster's contiguous block, so
// M[pi_a][pi_b] = max(h[a..b-1]).
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace appd {

static inline int32_t find_root_arr(int32_t* parent, int32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];  // path halving
    x = parent[x];
  }
  return x;
}

static inline int find_root(std::vector<int32_t>& parent, int32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];  // path halving
    x = parent[x];
  }
  return x;
}

void host_dendrogram(const u64* sorted_keys, int64_t n, const KeySpec& ks, int32_t* pi, float* h) {
  if (n == 1) { pi[0] = 0; return; }
  std::vector<int32_t> parent(n), size(n, 1), head(n), tail(n), next(n, -1);
  std::vector<float> gap(n, 0.0f);
  for (int64_t i = 0; i < n; i++) { parent[i] = (int32_t)i; head[i] = (int32_t)i; tail[i] = (int32_t)i; }
  const u64 mask = (1ull << ks.shift) - 1;
  for (int64_t e = 0; e < n - 1; e++) {
    u64 key = sorted_keys[e];
    int64_t u, v;
    tri_decode(key & mask, &u, &v);
    uint32_t wk = (uint32_t)(key >> ks.shift);
    float w;
    if (ks.points) {
      float d2;
      std::memcpy(&d2, &wk, 4);
      w = std::sqrt(d2);  // IEEE sqrt, correctly rounded = __fsqrt_rn = sqrtf (R1)
    } else {
      float m = from_orderable(wk);
      w = (ks.sense > 0 ? m : -m) + 0.0f;
    }
    int32_t ru = find_root(parent, (int32_t)u), rv = find_root(parent, (int32_t)v);
    // list(ru) then list(rv)
    next[tail[ru]] = head[rv];
    gap[tail[ru]] = w;
    int32_t nh = head[ru], nt = tail[rv];
    int32_t r = size[ru] >= size[rv] ? ru : rv;
    int32_t o = r == ru ? rv : ru;
    parent[o] = r;
    size[r] = size[ru] + size[rv];
    head[r] = nh;
    tail[r] = nt;
  }
  int32_t root = find_root(parent, 0);
  int32_t x = head[root];
  for (int64_t a = 0; a < n; a++) {
    pi[a] = x;
    if (a < n - 1) h[a] = gap[x];
    x = next[x];
  }
}

}  // namespace appd

namespace appd {

// Same merges on pre-decoded edges (u, v, w) in ascending key order, recorded as the
// Kruskal reconstruction tree (leaves 0..n-1, internal node n+e for edge e, children =
// the two clusters it joins) instead of linked lists; the leaf order is then the
// tree's in-order, computed top-down (a node's parent has a larger rank, so one pass
// over the edges in descending order places every subtree): independent stores instead
// of a dependent walk.  Union by size with path halving on one 16-byte record per
// vertex (one cache line per step).  scratch: 8 n int32.
namespace {
struct UfNode {
  int32_t parent, size, rootnode, pad;
};
inline int32_t uf_find(UfNode* a, int32_t x) {
  while (a[x].parent != x) {
    const int32_t p = a[x].parent;
    a[x].parent = a[p].parent;  // path halving
    x = a[x].parent;
  }
  return x;
}
}  // namespace

void host_dendrogram_uvw(const int32_t* eu, const int32_t* ev, const float* ew, int64_t n, int32_t* pi, float* h,
                         int32_t* scratch /* 8 n */) {
  if (n == 1) {
    pi[0] = 0;
    return;
  }
  const int64_t m = n - 1;
  UfNode* a = reinterpret_cast<UfNode*>(scratch);  // 4 n
  int32_t* kid = scratch + 4 * n;                  // 2 m: children of internal node n + e
  int32_t* lsize = scratch + 6 * n;                // m: leaves under the first child
  for (int64_t i = 0; i < n; i++) a[i] = {(int32_t)i, 1, (int32_t)i, 0};
  for (int64_t e = 0; e < m; e++) {
    const int32_t ru = uf_find(a, eu[e]), rv = uf_find(a, ev[e]);
    kid[2 * e] = a[ru].rootnode;
    kid[2 * e + 1] = a[rv].rootnode;
    lsize[e] = a[ru].size;
    const int32_t sz = a[ru].size + a[rv].size;
    const int32_t r = a[ru].size >= a[rv].size ? ru : rv, o = r == ru ? rv : ru;
    a[o].parent = r;
    a[r].size = sz;
    a[r].rootnode = (int32_t)(n + e);
  }
  // in-order offsets; the union-find records are dead, their space holds 2n - 1 offsets
  int32_t* off = scratch;
  off[n + m - 1] = 0;
  for (int64_t e = m - 1; e >= 0; e--) {
    const int32_t o = off[n + e];
    const int32_t o2 = o + lsize[e];
    off[kid[2 * e]] = o;
    off[kid[2 * e + 1]] = o2;
    h[o2 - 1] = ew[e];  // the gap between the two clusters is their merge height
  }
  for (int64_t v = 0; v < n; v++) pi[off[v]] = (int32_t)v;
}

}  // namespace appd
