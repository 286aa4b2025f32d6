// k_floyd.cu -- NEXT-2: the paper's comparison algorithm, the minimax
// variant of Floyd–Warshall ("a modified version of the Floyd-Warshall
// algorithm", Fig. floyd: k outermost, M[i][j] = min(M[i][j],
// max(M[i][k], M[k][j])); O(n^3)), as a blocked closure over the (min, max)
// semiring on the FP32 pipe (no rounding anywhere: min and max are exact, so the result
// is bit-identical to the oracle's triple loop; no tensor cores — the semiring is not a
// multiply-add).  sense -1 (widest path) swaps min and max.
//
// Tiles of FW_T x FW_T.  For every diagonal block kb:
//   phase 1  the diagonal tile's own closure (one CTA, k sequential in shared memory);
//   phase 2  row panel (kb, J) = min(C, D (x) C) and column panel (I, kb) = min(C, C (x) D)
//            with D the closed diagonal tile: one (min, max) product each (a closed D
//            contains every path inside block kb, so one product suffices);
//   phase 3  every other tile (I, J) = min(C, A(I, kb) (x) B(kb, J)).
// Phases 2 and 3 are the same register-blocked tile product: 256 threads, an 8 x 8
// micro-tile per thread, k in chunks of 32 staged in shared memory (cp.async double
// buffer for interior tiles), and per pair of k one 3-input min over two maxima.
// The diagonal is reset to +0 at the end (reading Q3); -0 inputs read as +0 (Q5).
#include <algorithm>

#include "internal.cuh"

namespace appd {

constexpr int FW_T = 128;         // tile
constexpr int FW_KC = 32;         // k chunk staged in shared memory
constexpr int FW_AS = FW_KC + 4;  // A chunk row stride (floats): rows x k, 16-byte aligned rows
constexpr int FW_BS = FW_T + 4;   // B chunk row stride: k x columns

template <int SENSE>
__device__ __forceinline__ float fw_id() {  // identity of the "sum" (no path)
  return SENSE > 0 ? INFINITY : -INFINITY;
}
template <int SENSE>
__device__ __forceinline__ float fw_mul(float a, float b) {  // path concatenation
  return SENSE > 0 ? fmaxf(a, b) : fminf(a, b);
}
template <int SENSE>
__device__ __forceinline__ float fw_add3(float c, float x, float y) {  // choice among paths
  float r;
  if (SENSE > 0) asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(c), "f"(x), "f"(y));
  else asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(c), "f"(x), "f"(y));
  return r;
}

__device__ __forceinline__ void fw_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// M = canon(W) (-0 -> +0), all n x n
__global__ void k_fw_init(const float* __restrict__ W, int64_t total, float* __restrict__ M) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    M[e] = W[e] + 0.0f;
}
__global__ void k_fw_diag(float* __restrict__ M, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    M[i * n + i] = 0.0f;
}

// phase 1: closure of the diagonal tile kb in shared memory, k sequential
template <int SENSE>
__global__ void __launch_bounds__(1024) k_fw_phase1(float* __restrict__ M, int n, int kb) {
  extern __shared__ float fsm1[];
  float(*D)[FW_T + 1] = reinterpret_cast<float(*)[FW_T + 1]>(fsm1);  // [FW_T][FW_T + 1]
  const int o = kb * FW_T, m = min(FW_T, n - o);
  for (int e = threadIdx.x; e < FW_T * FW_T; e += blockDim.x) {
    const int i = e / FW_T, j = e % FW_T;
    D[i][j] = (i < m && j < m) ? M[(int64_t)(o + i) * n + o + j] : fw_id<SENSE>();
  }
  __syncthreads();
  for (int k = 0; k < m; k++) {
    for (int e = threadIdx.x; e < FW_T * FW_T; e += blockDim.x) {
      const int i = e / FW_T, j = e % FW_T;
      const float v = fw_mul<SENSE>(D[i][k], D[k][j]);
      D[i][j] = SENSE > 0 ? fminf(D[i][j], v) : fmaxf(D[i][j], v);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < FW_T * FW_T; e += blockDim.x) {
    const int i = e / FW_T, j = e % FW_T;
    if (i < m && j < m) M[(int64_t)(o + i) * n + o + j] = D[i][j];
  }
}

// One tile product C(I, J) = add(C, A(I, K) (x) B(K, J)) with all three tiles in M
// (the output may alias A or B: every read of the inputs precedes the first write).
// mode 0: phase 3 over (I, J), I, J != kb; mode 1: phase 2 (row panels J != kb, then
// column panels I != kb).
template <int SENSE>
__global__ void __launch_bounds__(256, 2) k_fw_tiles(float* __restrict__ M, int n, int kb, int mode) {
  extern __shared__ __align__(16) float fsm[];
  float* As = fsm;                          // [2][FW_T][FW_AS]
  float* Bs = fsm + 2 * FW_T * FW_AS;       // [2][FW_KC][FW_BS]
  const int T = (n + FW_T - 1) / FW_T;
  int I, J;
  if (mode == 0) {
    I = blockIdx.x / (T - 1);
    J = blockIdx.x % (T - 1);
    I += I >= kb;
    J += J >= kb;
  } else {
    const int t = blockIdx.x;
    if (t < T - 1) {
      I = kb;
      J = t + (t >= kb);
    } else {
      J = kb;
      I = (t - (T - 1)) + ((t - (T - 1)) >= kb);
    }
  }
  const int K = kb;
  const int r0 = I * FW_T, c0 = J * FW_T, k0 = K * FW_T;
  const int mr = min(FW_T, n - r0), mc = min(FW_T, n - c0), mk = min(FW_T, n - k0);
  const bool full = mr == FW_T && mc == FW_T && mk == FW_T && (n & 3) == 0 &&
                    (reinterpret_cast<uintptr_t>(M) & 15) == 0;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float ID = fw_id<SENSE>();

  // stage k chunk ch into buffer b
  auto stage = [&](int ch, int b) {
    float* A = As + b * FW_T * FW_AS;
    float* B = Bs + b * FW_KC * FW_BS;
    const int kc = ch * FW_KC;
    if (full) {
      for (int e = threadIdx.x; e < FW_T * (FW_KC / 4); e += 256) {  // A: 128 rows x 8 float4
        const int i = e >> 3, q = e & 7;
        fw_cp16(A + i * FW_AS + 4 * q, M + (int64_t)(r0 + i) * n + k0 + kc + 4 * q);
      }
      for (int e = threadIdx.x; e < FW_KC * (FW_T / 4); e += 256) {  // B: 32 rows x 32 float4
        const int k = e >> 5, q = e & 31;
        fw_cp16(B + k * FW_BS + 4 * q, M + (int64_t)(k0 + kc + k) * n + c0 + 4 * q);
      }
    } else {  // border tile: plain loads, the no-path identity outside the matrix
      for (int e = threadIdx.x; e < FW_T * FW_KC; e += 256) {
        const int i = e / FW_KC, k = e % FW_KC;
        A[i * FW_AS + k] = (i < mr && kc + k < mk) ? M[(int64_t)(r0 + i) * n + k0 + kc + k] : ID;
      }
      for (int e = threadIdx.x; e < FW_KC * FW_T; e += 256) {
        const int k = e / FW_T, j = e % FW_T;
        B[k * FW_BS + j] = (kc + k < mk && j < mc) ? M[(int64_t)(k0 + kc + k) * n + c0 + j] : ID;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // the thread's rows ty + 16 a and columns 4 tx + {0..3}, 64 + 4 tx + {0..3}
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; a++)
#pragma unroll
    for (int b = 0; b < 8; b++) acc[a][b] = ID;
  const int nch = (mk + FW_KC - 1) / FW_KC;
  stage(0, 0);
  for (int ch = 0; ch < nch; ch++) {
    if (ch + 1 < nch) {
      stage(ch + 1, (ch + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* A = As + (ch & 1) * FW_T * FW_AS;
    const float* B = Bs + (ch & 1) * FW_KC * FW_BS;
#pragma unroll 2
    for (int k = 0; k < FW_KC; k += 2) {
      float a0[8], a1[8];
#pragma unroll
      for (int a = 0; a < 8; a++) {
        const float2 v = *reinterpret_cast<const float2*>(A + (ty + 16 * a) * FW_AS + k);
        a0[a] = v.x;
        a1[a] = v.y;
      }
      const float4 b00 = *reinterpret_cast<const float4*>(B + k * FW_BS + 4 * tx);
      const float4 b01 = *reinterpret_cast<const float4*>(B + k * FW_BS + 64 + 4 * tx);
      const float4 b10 = *reinterpret_cast<const float4*>(B + (k + 1) * FW_BS + 4 * tx);
      const float4 b11 = *reinterpret_cast<const float4*>(B + (k + 1) * FW_BS + 64 + 4 * tx);
      const float bk0[8] = {b00.x, b00.y, b00.z, b00.w, b01.x, b01.y, b01.z, b01.w};
      const float bk1[8] = {b10.x, b10.y, b10.z, b10.w, b11.x, b11.y, b11.z, b11.w};
#pragma unroll
      for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 8; b++)
          acc[a][b] = fw_add3<SENSE>(acc[a][b], fw_mul<SENSE>(a0[a], bk0[b]), fw_mul<SENSE>(a1[a], bk1[b]));
    }
    __syncthreads();  // buffer (ch & 1) is refilled by the next iteration's stage
  }
  // C = add(C, product): read C, then write (all input reads of the tile happened above)
#pragma unroll
  for (int a = 0; a < 8; a++) {
    const int i = ty + 16 * a;
    if (i >= mr) continue;
    float* row = M + (int64_t)(r0 + i) * n + c0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int j = 64 * h + 4 * tx;
      if (full) {
        float4 cv = *reinterpret_cast<const float4*>(row + j);
        cv.x = fw_add3<SENSE>(cv.x, acc[a][4 * h + 0], acc[a][4 * h + 0]);
        cv.y = fw_add3<SENSE>(cv.y, acc[a][4 * h + 1], acc[a][4 * h + 1]);
        cv.z = fw_add3<SENSE>(cv.z, acc[a][4 * h + 2], acc[a][4 * h + 2]);
        cv.w = fw_add3<SENSE>(cv.w, acc[a][4 * h + 3], acc[a][4 * h + 3]);
        *reinterpret_cast<float4*>(row + j) = cv;
      } else {
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (j + u < mc) row[j + u] = fw_add3<SENSE>(row[j + u], acc[a][4 * h + u], acc[a][4 * h + u]);
      }
    }
  }
}

static appd_status fw_run(appd_ctx* c, float* M, int64_t n64, int sense) {
  const int n = (int)n64;
  const int T = (n + FW_T - 1) / FW_T;
  const size_t smem = sizeof(float) * (2 * FW_T * FW_AS + 2 * FW_KC * FW_BS);
  const size_t smem1 = sizeof(float) * FW_T * (FW_T + 1);
  static std::atomic<unsigned long long> attr{0};
  if (needs_setup(attr, c)) {
    cudaFuncSetAttribute(k_fw_tiles<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fw_tiles<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fw_phase1<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    cudaFuncSetAttribute(k_fw_phase1<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    setup_done(attr, c);
  }
  for (int kb = 0; kb < T; kb++) {
    if (sense > 0) k_fw_phase1<1><<<1, 1024, smem1, c->stream>>>(M, n, kb);
    else k_fw_phase1<-1><<<1, 1024, smem1, c->stream>>>(M, n, kb);
    APPD_LAUNCHED(c);
    if (T == 1) break;
    if (sense > 0) k_fw_tiles<1><<<2 * (T - 1), 256, smem, c->stream>>>(M, n, kb, 1);
    else k_fw_tiles<-1><<<2 * (T - 1), 256, smem, c->stream>>>(M, n, kb, 1);
    APPD_LAUNCHED(c);
    if (sense > 0) k_fw_tiles<1><<<(T - 1) * (T - 1), 256, smem, c->stream>>>(M, n, kb, 0);
    else k_fw_tiles<-1><<<(T - 1) * (T - 1), 256, smem, c->stream>>>(M, n, kb, 0);
    APPD_LAUNCHED(c);
  }
  return APPD_OK;
}

// W, M: device n x n; the validation verdict (same rules as appd_solve_weights) is checked
// by the caller before the closure runs
appd_status floyd_weights(appd_ctx* c, const float* W, int64_t n, float* M, int sense) {
  if ((uint64_t)n * (uint64_t)n > (1ull << 33)) return fail(c, APPD_ERR_UNSUPPORTED, "floyd: n = %lld", (long long)n);
  const int64_t total = n * n;
  int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)c->sm_count * 8);
  k_fw_init<<<grid, 256, 0, c->stream>>>(W, total, M);
  APPD_LAUNCHED(c);
  appd_status s = fw_run(c, M, n, sense);
  if (s) return s;
  k_fw_diag<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, c->stream>>>(M, n);
  APPD_LAUNCHED(c);
  return APPD_OK;
}

}  // namespace appd
