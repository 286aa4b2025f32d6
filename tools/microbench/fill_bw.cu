// Write-bandwidth microbenchmark for the APPD fill's store pattern (16 GiB matrix):
// (a) linear 16-byte stores, (b) tiles of 128 rows in random order x W contiguous
// columns per CTA (the fill's shape), for W in {1024, 2048, 4096}.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_linear(float4* p, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_float4(1.f, 2.f, 3.f, 4.f));
}
__global__ void k_linear_plain(float4* p, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}
// 32-byte stores (st.global.v8.f32, sm_100)
__global__ void k_linear_v8(float* p, size_t n8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    float* q = p + 8 * i;
    asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(q), "f"(1.f), "f"(2.f), "f"(3.f),
                 "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"(8.f)
                 : "memory");
  }
}
template <int W>
__global__ void __launch_bounds__(256) k_tiles_v8(float* M, const int* rows, int n) {
  const int64_t t0 = (int64_t)blockIdx.y * 128;
  for (int t = 0; t < 128; t++) {
    float* dst = M + (int64_t)rows[t0 + t] * n + (int64_t)blockIdx.x * W + 8 * threadIdx.x;
#pragma unroll
    for (int c = 0; c < W / 2048; c++)
      asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + c * 2048), "f"(1.f),
                   "f"(2.f), "f"(3.f), "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"((float)t)
                   : "memory");
  }
}
template <int W>
__global__ void __launch_bounds__(256) k_tiles(float* M, const int* rows, int n) {
  const int64_t t0 = (int64_t)blockIdx.y * 128;
  for (int t = 0; t < 128; t++) {
    float* dst = M + (int64_t)rows[t0 + t] * n + (int64_t)blockIdx.x * W;
#pragma unroll
    for (int c = 0; c < W / 1024; c++)
      __stcs(reinterpret_cast<float4*>(dst + c * 1024) + threadIdx.x, make_float4(1.f, 2.f, 3.f, (float)t));
  }
}
// TMA bulk stores: each row segment (W floats) is written to shared memory by the CTA and
// stored by one thread with cp.async.bulk (NB segments in flight)
template <int W, int NB>
__global__ void __launch_bounds__(256) k_tiles_bulk(float* M, const int* rows, int n) {
  __shared__ __align__(128) float buf[NB][W];
  const int64_t t0 = (int64_t)blockIdx.y * 128;
  for (int t = 0; t < 128; t++) {
    const int b = t % NB;
    if (t >= NB) {
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
      __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < W / 1024; c++)
      reinterpret_cast<float4*>(buf[b] + c * 1024)[threadIdx.x] = make_float4(1.f, 2.f, 3.f, (float)t);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      float* dst = M + (int64_t)rows[t0 + t] * n + (int64_t)blockIdx.x * W;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"((uint32_t)__cvta_generic_to_shared(buf[b])), "r"(W * 4)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// persistent: grid = SMs x 4, tiles handed out in order
template <int W>
__global__ void __launch_bounds__(256) k_tiles_v8_persist(float* M, const int* rows, int n, int tiles_x, int tiles) {
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int bx = tile % tiles_x, by = tile / tiles_x;
    const int64_t t0 = (int64_t)by * 128;
    for (int t = 0; t < 128; t++) {
      float* dst = M + (int64_t)rows[t0 + t] * n + (int64_t)bx * W + 8 * threadIdx.x;
#pragma unroll
      for (int c = 0; c < W / 2048; c++)
        asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + c * 2048), "f"(1.f),
                     "f"(2.f), "f"(3.f), "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"((float)t)
                     : "memory");
    }
  }
}
template <int W>
__global__ void __launch_bounds__(256) k_tiles_v8_smem(float* M, const int* rows, int n) {
  extern __shared__ float dummy[];
  const int64_t t0 = (int64_t)blockIdx.y * 128;
  if (threadIdx.x == 0) dummy[0] = 0.f;
  for (int t = 0; t < 128; t++) {
    float* dst = M + (int64_t)rows[t0 + t] * n + (int64_t)blockIdx.x * W + 8 * threadIdx.x;
#pragma unroll
    for (int c = 0; c < W / 2048; c++)
      asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + c * 2048), "f"(1.f),
                   "f"(2.f), "f"(3.f), "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"((float)t)
                   : "memory");
  }
}
// the fill's shape with a setup of D dependent loads per CTA before its stores
template <int W, int D>
__global__ void __launch_bounds__(256) k_tiles_v8_setup(float* M, const int* rows, int n) {
  __shared__ int srow[128];
  const int64_t t0 = (int64_t)blockIdx.y * 128;
  int x = threadIdx.x + blockIdx.x * 97;
#pragma unroll
  for (int q = 0; q < D; q++) x = rows[(x * 31 + 7) & (n - 1)];
  if (threadIdx.x < 128) srow[threadIdx.x] = rows[t0 + threadIdx.x] + (x == -5 ? 1 : 0);
  __syncthreads();
  for (int t = 0; t < 128; t++) {
    float* dst = M + (int64_t)srow[t] * n + (int64_t)blockIdx.x * W + 8 * threadIdx.x;
#pragma unroll
    for (int c = 0; c < W / 2048; c++)
      asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + c * 2048), "f"(1.f),
                   "f"(2.f), "f"(3.f), "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"((float)t)
                   : "memory");
  }
}
// the same stores with varying values (hash of the element index)
template <int W>
__global__ void __launch_bounds__(256) k_tiles_v8_rand(float* M, const int* rows, int n) {
  const int64_t t0 = (int64_t)blockIdx.y * 128;
  for (int t = 0; t < 128; t++) {
    const int64_t r = rows[t0 + t];
    float* dst = M + r * n + (int64_t)blockIdx.x * W + 8 * threadIdx.x;
    unsigned h = (unsigned)(r * 2654435761u) ^ (unsigned)(blockIdx.x * W + 8 * threadIdx.x) * 40503u;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      h = h * 1664525u + 1013904223u;
      v[q] = __uint_as_float(0x3f800000u | (h >> 9));
    }
#pragma unroll
    for (int c = 0; c < W / 2048; c++)
      asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + c * 2048), "f"(v[0]),
                   "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                   : "memory");
  }
}
int main() {
  const int n = 65536;
  const size_t bytes = (size_t)n * n * 4;
  float* M;
  cudaMalloc(&M, bytes);
  std::vector<int> h(n);
  for (int i = 0; i < n; i++) h[i] = i;
  std::shuffle(h.begin(), h.end(), std::mt19937(1));
  int* rows;
  cudaMalloc(&rows, n * 4);
  cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](auto f, const char* name) {
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(a);
      f();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    printf("%-28s %.3f ms  %.2f TB/s\n", name, best, bytes / (best * 1e-3) / 1e12);
  };
  time([&] { k_linear<<<148 * 16, 256>>>((float4*)M, bytes / 16); }, "linear");
  time([&] { k_tiles<1024><<<dim3(n / 1024, n / 128), 256>>>(M, rows, n); }, "tiles 128 x 4 KB");
  time([&] { k_tiles<2048><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles 128 x 8 KB");
  time([&] { k_tiles<4096><<<dim3(n / 4096, n / 128), 256>>>(M, rows, n); }, "tiles 128 x 16 KB");
  time([&] { cudaMemsetAsync(M, 0, bytes); }, "cudaMemset");
  time([&] { k_linear_plain<<<148 * 16, 256>>>((float4*)M, bytes / 16); }, "linear plain");
  time([&] { k_linear_v8<<<148 * 16, 256>>>(M, bytes / 32); }, "linear v8 (32 B)");
  time([&] { k_tiles_v8<2048><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles v8 128 x 8 KB");
  time([&] { k_linear<<<148 * 64, 256>>>((float4*)M, bytes / 16); }, "linear (more CTAs)");
  time([&] { k_tiles_bulk<2048, 4><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles bulk 8 KB x4");
  time([&] { k_tiles_bulk<2048, 2><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles bulk 8 KB x2");
  time([&] { k_tiles_bulk<4096, 2><<<dim3(n / 4096, n / 128), 256>>>(M, rows, n); }, "tiles bulk 16 KB x2");
  time([&] { k_tiles_v8_persist<2048><<<148 * 4, 256>>>(M, rows, n, n / 2048, (n / 2048) * (n / 128)); }, "tiles v8 persistent");
  time([&] { k_tiles_v8<4096><<<dim3(n / 4096, n / 128), 256>>>(M, rows, n); }, "tiles v8 128 x 16 KB");
  // occupancy limited by dynamic shared memory: 4 / 5 / 6 CTAs per SM
  cudaFuncSetAttribute(k_tiles_v8_smem<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  time([&] { k_tiles_v8_smem<2048><<<dim3(n / 2048, n / 128), 256, 52 * 1024>>>(M, rows, n); }, "tiles v8, 4 CTAs/SM");
  time([&] { k_tiles_v8_smem<2048><<<dim3(n / 2048, n / 128), 256, 42 * 1024>>>(M, rows, n); }, "tiles v8, 5 CTAs/SM");
  time([&] { k_tiles_v8_smem<2048><<<dim3(n / 2048, n / 128), 256, 35 * 1024>>>(M, rows, n); }, "tiles v8, 6 CTAs/SM");
  time([&] { k_tiles_v8_smem<2048><<<dim3(n / 2048, n / 128), 256, 26 * 1024>>>(M, rows, n); }, "tiles v8, 8 CTAs/SM");
  time([&] { k_tiles_v8_rand<2048><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles v8, random values");
  time([&] { k_tiles_v8_setup<2048, 0><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles v8, setup 0 loads");
  time([&] { k_tiles_v8_setup<2048, 3><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles v8, setup 3 loads");
  time([&] { k_tiles_v8_setup<2048, 6><<<dim3(n / 2048, n / 128), 256>>>(M, rows, n); }, "tiles v8, setup 6 loads");
  return 0;
}
