// Microbenchmark: tcgen05.mma kind::f16 SS throughput for shared-memory layouts
// (no swizzle vs 128-byte swizzle), M=128, N in {64,128,256}.  Not product code.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2407_07058_b200/csrc/tc_ptx.cuh"

using namespace appd;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int layout) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46) | ((uint64_t)layout << 61);
}

__global__ void __launch_bounds__(128, 1) k_rate(int iters, int N, int layout, int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_f16_f32(128, N);
    const uint32_t a0 = ptx::smem_u32(smem);
    const uint32_t b0 = a0 + 32768;
    // no swizzle: LBO = 128 (K halves), SBO = 1280 (8-row groups, K = 80);
    // 128B swizzle: LBO unused (16), SBO = 1024 (8 rows x 128 B)
    const uint32_t lbo = layout == 0 ? 128 : 16, sbo = layout == 0 ? 1280 : 1024;
    for (int it = 0; it < iters; it++) {
      for (int ks = 0; ks < 5; ks++) {
        const uint32_t koff = layout == 0 ? ks * 256 : (ks % 4) * 32;
        ptx::mma_f16(tmem + (it & 1) * 256, desc(a0 + koff, lbo, sbo, layout), desc(b0 + koff, lbo, sbo, layout),
                     idesc, ks > 0);
      }
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

int main1() {
  int* out;
  cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int layout : {0, 2}) {
    for (int N : {64, 128, 256}) {
      for (int w = 0; w < 2; w++) {
        cudaEventRecord(e0);
        k_rate<<<148, 128, 200 * 1024>>>(iters, N, layout, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      double macs = 148.0 * iters * 5 * 128.0 * N * 16;
      printf("layout %s N=%d: %.3f ms  %.1f TFLOP/s (fp16 dense)  cycles/mma@1.9GHz %.1f  %s\n",
             layout ? "SW128" : "NONE", N, ms, 2 * macs / ms / 1e9, ms * 1e-3 * 1.9e9 / (iters * 5.0),
             cudaGetErrorString(err));
    }
  }
  return 0;
}

// TMEM load bandwidth: warps read the 512-column allocation with tcgen05.ld 32x32b.x32
__global__ void __launch_bounds__(512, 1) k_ldtm(int iters, float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const int q = warp & 3;
  float acc = 0.0f;
  for (int it = 0; it < iters; it++) {
    float v[32];
    ptx::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(((it + warp) & 15) * 32), v);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; i++) acc += v[i];
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main2() {
  float* out;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {128, 256, 512}) {
    for (int w = 0; w < 2; w++) {
      cudaEventRecord(e0);
      k_ldtm<<<148, threads>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 148.0 * (threads / 32) * iters * 32 * 32 * 4;
    printf("LDTM %d threads/SM: %.3f ms  %.1f B/clk/SM @1.9GHz  %s\n", threads, ms,
           bytes / 148 / (ms * 1e-3 * 1.9e9), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}


// groups of 5 MMAs (N=128) into 4 rotating TMEM buffers; mode 1: commit per group;
// mode 2: commit + tcgen05.fence::after_thread_sync per group; mode 3: + try_wait on a completed barrier
__global__ void __launch_bounds__(128, 1) k_rate2(int iters, int mode, int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_f16_f32(128, 128);
    const uint32_t a0 = ptx::smem_u32(smem);
    const uint32_t b0 = a0 + 65536;
    if (mode == 3) { ptx::mbar_arrive(&bar[1]); }
    for (int it = 0; it < iters; it++) {
      if (mode == 3) ptx::mbar_wait(&bar[1], 0);
      if (mode >= 2) ptx::tc_fence_after();
      for (int ks = 0; ks < 5; ks++)
        ptx::mma_f16(tmem + (it & 3) * 128, desc(a0 + ks * 256, 128, 1280, 0), desc(b0 + ks * 256, 128, 1280, 0),
                     idesc, ks > 0);
      if (mode >= 1) ptx::mma_commit(&bar[0]);
    }
    ptx::mma_commit(&bar[0]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

int main3() {
  int* out;
  cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(k_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8000;
  for (int mode = 0; mode < 4; mode++) {
    for (int w = 0; w < 2; w++) {
      cudaEventRecord(e0);
      k_rate2<<<148, 128, 200 * 1024>>>(iters, mode, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("groups mode %d: %.3f ms  cycles/group@1.9GHz %.1f (ideal 320)  %s\n", mode, ms,
           ms * 1e-3 * 1.9e9 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
int main() { main3(); return 0; }
