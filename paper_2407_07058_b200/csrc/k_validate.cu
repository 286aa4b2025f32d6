// k_validate.cu -- ingest checks.
// A valid weight matrix is finite, has a +-0 diagonal and is bitwise symmetric
// after -0 -> +0 (reading Q5).  Each kernel records the first offender of each
// kind in row-major order as a 64-bit linear index (atomicMin); the host picks
// the earliest (ties: NONFINITE first).
#include "internal.cuh"

namespace appd {

__device__ __forceinline__ uint32_t canon_bits(float w) { return __float_as_uint(w + 0.0f); }

// 64x64 tile pairs (I,J) and (J,I), I <= J, inside the square [row0, row0+rows)^2 of
// global indices; W is the rank's row block (rows x n, first row = row0).  Both tiles
// are read with 16-byte loads (256-byte row segments), all issued before any shared-
// memory store; the transposed compare goes through padded shared memory.
constexpr int VT = 64;
__global__ void __launch_bounds__(256, 6) k_validate_square(const float* __restrict__ W, int64_t n, int64_t row0,
                                                         int64_t rows, int64_t tiles, u64* __restrict__ out3) {
  __shared__ float b[VT][VT + 1];  // the (J, I) tile; (I, J) stays in registers
  // map blockIdx.x to (I, J) with I <= J over a T x T upper triangle
  const int64_t p = blockIdx.x, T = tiles;
  // pairs before row I: f(I) = I*T - I*(I-1)/2; largest I with f(I) <= p
  double q = (double)(2 * T + 1);
  int64_t I = (int64_t)((q - sqrt(q * q - 8.0 * (double)p)) * 0.5);
  if (I < 0) I = 0;
  while (I > 0 && I * T - I * (I - 1) / 2 > p) I--;
  while ((I + 1) * T - (I + 1) * I / 2 <= p) I++;
  const int64_t J = I + (p - (I * T - I * (I - 1) / 2));
  const bool vec = ((n | row0) & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  const int c4 = threadIdx.x & 15, r0 = threadIdx.x >> 4;
  float4 va[VT / 16], vb[VT / 16];
#pragma unroll
  for (int s4 = 0; s4 < VT / 16; s4++) {
    const int r = r0 + 16 * s4;
    const int64_t li = I * VT + r, mi = J * VT + r;
    const int64_t lj = J * VT + 4 * c4, mj = I * VT + 4 * c4;
    if (vec && li < rows && lj + 3 < rows) {
      va[s4] = __ldcs(reinterpret_cast<const float4*>(W + li * n + row0 + lj));
    } else {
      va[s4].x = (li < rows && lj + 0 < rows) ? W[li * n + row0 + lj + 0] : 0.0f;
      va[s4].y = (li < rows && lj + 1 < rows) ? W[li * n + row0 + lj + 1] : 0.0f;
      va[s4].z = (li < rows && lj + 2 < rows) ? W[li * n + row0 + lj + 2] : 0.0f;
      va[s4].w = (li < rows && lj + 3 < rows) ? W[li * n + row0 + lj + 3] : 0.0f;
    }
    if (vec && mi < rows && mj + 3 < rows) {
      vb[s4] = __ldcs(reinterpret_cast<const float4*>(W + mi * n + row0 + mj));
    } else {
      vb[s4].x = (mi < rows && mj + 0 < rows) ? W[mi * n + row0 + mj + 0] : 0.0f;
      vb[s4].y = (mi < rows && mj + 1 < rows) ? W[mi * n + row0 + mj + 1] : 0.0f;
      vb[s4].z = (mi < rows && mj + 2 < rows) ? W[mi * n + row0 + mj + 2] : 0.0f;
      vb[s4].w = (mi < rows && mj + 3 < rows) ? W[mi * n + row0 + mj + 3] : 0.0f;
    }
  }
#pragma unroll
  for (int s4 = 0; s4 < VT / 16; s4++) {
    const int r = r0 + 16 * s4;
    b[r][4 * c4 + 0] = vb[s4].x;
    b[r][4 * c4 + 1] = vb[s4].y;
    b[r][4 * c4 + 2] = vb[s4].z;
    b[r][4 * c4 + 3] = vb[s4].w;
  }
  __syncthreads();
  // fast path: 32-bit tests only (non-finite: exponent all ones; asymmetric: different bits
  // unless both are zeros of either sign; bad diagonal: a non-zero on the diagonal); each
  // thread tests its own (I, J) elements (registers) against the transposed (J, I) tile
  // (shared memory, one 33 KB tile pair became one 17 KB tile: more CTAs in flight); the
  // exact first offenders are located only in a tile that has one
  const bool diag_tile = I == J;
  unsigned flag = 0;
#pragma unroll
  for (int s4 = 0; s4 < VT / 16; s4++) {
    const int r = r0 + 16 * s4;
    const float xs[4] = {va[s4].x, va[s4].y, va[s4].z, va[s4].w};
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int cc = 4 * c4 + e;
      const uint32_t bx = __float_as_uint(xs[e]), by = __float_as_uint(b[cc][r]);
      flag |= ((bx & 0x7F800000u) == 0x7F800000u) | ((by & 0x7F800000u) == 0x7F800000u);
      flag |= (bx != by) & (((bx | by) << 1) != 0u);
      if (diag_tile) flag |= (r == cc) & ((bx << 1) != 0u);
    }
  }
  if (!__syncthreads_or(flag)) return;
  // (rare: a tile pair with an offender) the (I, J) elements again from W (L2)
  u64 bad_nf = KEY_NONE, bad_diag = KEY_NONE, bad_sym = KEY_NONE;
#pragma unroll 1
  for (int s4 = 0; s4 < VT / 16; s4++) {
    const int r = r0 + 16 * s4;
#pragma unroll 1
    for (int e = 0; e < 4; e++) {
      const int cc = 4 * c4 + e;
      const int64_t li = I * VT + r, lj = J * VT + cc;
      if (li < rows && lj < rows) {
        const int64_t gi = row0 + li, gj = row0 + lj;
        const float x = W[li * n + row0 + lj];  // W[gi][gj]
        const float y = b[cc][r];  // W[gj][gi]
        const u64 idx = (u64)(gi * n + gj);
        const u64 idxT = (u64)(gj * n + gi);
        if (!isfinite(x)) bad_nf = min(bad_nf, idx);
        if (!isfinite(y)) bad_nf = min(bad_nf, idxT);
        if (gi == gj) {
          if (x != 0.0f) bad_diag = min(bad_diag, idx);
        } else if (canon_bits(x) != canon_bits(y)) {
          bad_sym = min(bad_sym, gi < gj ? idx : idxT);
        }
      }
    }
  }
  // one atomic per kind per warp
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad_nf = min(bad_nf, __shfl_xor_sync(0xffffffffu, bad_nf, o));
    bad_diag = min(bad_diag, __shfl_xor_sync(0xffffffffu, bad_diag, o));
    bad_sym = min(bad_sym, __shfl_xor_sync(0xffffffffu, bad_sym, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad_nf != KEY_NONE) atomicMin(out3 + 0, bad_nf);
    if (bad_diag != KEY_NONE) atomicMin(out3 + 1, bad_diag);
    if (bad_sym != KEY_NONE) atomicMin(out3 + 2, bad_sym);
  }
}

// finiteness of the columns outside the diagonal square (world > 1)
__global__ void k_validate_finite_rest(const float* __restrict__ W, int64_t n, int64_t row0, int64_t rows,
                                       u64* __restrict__ out3) {
  int64_t total = rows * n;
  u64 bad = KEY_NONE;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / n, j = e % n;
    if (j >= row0 && j < row0 + rows) continue;
    if (!isfinite(W[e])) bad = min(bad, (u64)((row0 + r) * n + j));
  }
  if (bad != KEY_NONE) atomicMin(out3 + 0, bad);
}

appd_status launch_validate_weights(appd_ctx* c, const float* W, int64_t n, int64_t row0, int64_t rows, u64* out3) {
  int64_t T = (rows + VT - 1) / VT;
  int64_t pairs = T * (T + 1) / 2;
  if (pairs > 0x7FFFFFFFll) return fail(c, APPD_ERR_UNSUPPORTED, "validation grid too large");
  if (pairs > 0) {
    k_validate_square<<<(unsigned)pairs, 256, 0, c->stream>>>(W, n, row0, rows, T, out3);
    APPD_LAUNCHED(c);
  }
  if (rows > 0 && rows < n) {
    k_validate_finite_rest<<<c->sm_count * 8, 256, 0, c->stream>>>(W, n, row0, rows, out3);
    APPD_LAUNCHED(c);
  }
  return APPD_OK;
}

// first non-finite coordinate (row-major element index); 16-byte loads when aligned
__global__ void k_validate_points(const float* __restrict__ X, int64_t total, u64* __restrict__ out3) {
  u64 bad = KEY_NONE;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    const float4* X4 = reinterpret_cast<const float4*>(X);
    const int64_t t4 = total >> 2;
    for (int64_t e = tid; e < t4; e += stride) {
      const float4 v = __ldcs(X4 + e);
      if (!isfinite(v.x)) bad = min(bad, (u64)(4 * e));
      else if (!isfinite(v.y)) bad = min(bad, (u64)(4 * e + 1));
      else if (!isfinite(v.z)) bad = min(bad, (u64)(4 * e + 2));
      else if (!isfinite(v.w)) bad = min(bad, (u64)(4 * e + 3));
    }
    for (int64_t e = (t4 << 2) + tid; e < total; e += stride)
      if (!isfinite(X[e])) bad = min(bad, (u64)e);
  } else {
    for (int64_t e = tid; e < total; e += stride)
      if (!isfinite(X[e])) bad = min(bad, (u64)e);
  }
  if (bad != KEY_NONE) atomicMin(out3, bad);
}

appd_status launch_validate_points(appd_ctx* c, const float* X, int64_t n, int64_t d, u64* out3) {
  int64_t total = n * d;
  int grid = (int)((total / 4 + 255) / 256);
  if (grid > c->sm_count * 16) grid = c->sm_count * 16;
  if (grid < 1) grid = 1;
  k_validate_points<<<grid, 256, 0, c->stream>>>(X, total, out3);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd

namespace appd {

// Solve-start agreement (world > 1): a position-keyed 64-bit checksum of
// the input words, sum over i of mix(i * phi + bits(x_i)) mod 2^64 (order-free to
// compute, position- and value-sensitive), so ranks holding different X disagree.
__device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) k_checksum_words(const uint32_t* __restrict__ x, int64_t count,
                                                        u64* __restrict__ out) {
  u64 acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    acc += mix64((u64)i * 0x9E3779B97F4A7C15ull + __ldg(x + i));
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

appd_status launch_checksum_words(appd_ctx* c, const void* x, int64_t count, u64* out) {
  APPD_CUDA(c, cudaMemsetAsync(out, 0, sizeof(u64), c->stream));
  if (count <= 0) return APPD_OK;
  const int grid = (int)std::min<int64_t>((count + 255) / 256, (int64_t)c->sm_count * 4);
  k_checksum_words<<<grid, 256, 0, c->stream>>>(reinterpret_cast<const uint32_t*>(x), count, out);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
