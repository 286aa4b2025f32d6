// Microbenchmarks for design decisions (not product code):
//  1. exact-R1 distance inner loop: scalar FADD/FFMA vs packed FADD2/FFMA2
//  2. streaming write bandwidth (st.global.cs vs default, float4)
//  3. pinned host <-> device copy bandwidth
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int KD = 32;

__global__ void __launch_bounds__(256, 2) scan_scalar(float* out, int reps) {
  __shared__ float As[KD][128];
  __shared__ float Bs[KD][128];
  for (int i = threadIdx.x; i < KD * 128; i += 256) {
    (&As[0][0])[i] = (i * 0.37f) - 11.f;
    (&Bs[0][0])[i] = (i * 0.23f) - 7.f;
  }
  __syncthreads();
  int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int c = 0; c < 8; c++) acc[r][c] = 0.f;
  for (int rep = 0; rep < reps; rep++) {
#pragma unroll 4
    for (int k = 0; k < KD; k++) {
      float4 a0 = *reinterpret_cast<float4*>(&As[k][ty * 8]);
      float4 a1 = *reinterpret_cast<float4*>(&As[k][ty * 8 + 4]);
      float4 b0 = *reinterpret_cast<float4*>(&Bs[k][tx * 8]);
      float4 b1 = *reinterpret_cast<float4*>(&Bs[k][tx * 8 + 4]);
      float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int c = 0; c < 8; c++) {
          float t = __fsub_rn(a[r], b[c]);
          acc[r][c] = __fmaf_rn(t, t, acc[r][c]);
        }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int c = 0; c < 8; c++) s += acc[r][c];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

// packed: As holds duplicated row values (x,x); Bs holds negated column values
__global__ void __launch_bounds__(256, 2) scan_packed(float* out, int reps) {
  __shared__ float2 As[KD][128];   // (x_r, x_r)
  __shared__ float Bs[KD][128];    // -y_c
  for (int i = threadIdx.x; i < KD * 128; i += 256) {
    float v = (i * 0.37f) - 11.f;
    (&As[0][0])[i] = make_float2(v, v);
    (&Bs[0][0])[i] = -((i * 0.23f) - 7.f);
  }
  __syncthreads();
  int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float2 acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int c = 0; c < 4; c++) acc[r][c] = make_float2(0.f, 0.f);
  for (int rep = 0; rep < reps; rep++) {
#pragma unroll 4
    for (int k = 0; k < KD; k++) {
      float4 a01 = *reinterpret_cast<float4*>(&As[k][ty * 8]);
      float4 a23 = *reinterpret_cast<float4*>(&As[k][ty * 8 + 2]);
      float4 a45 = *reinterpret_cast<float4*>(&As[k][ty * 8 + 4]);
      float4 a67 = *reinterpret_cast<float4*>(&As[k][ty * 8 + 6]);
      float4 b0 = *reinterpret_cast<float4*>(&Bs[k][tx * 8]);
      float4 b1 = *reinterpret_cast<float4*>(&Bs[k][tx * 8 + 4]);
      float2 a[8] = {make_float2(a01.x, a01.y), make_float2(a01.z, a01.w), make_float2(a23.x, a23.y),
                     make_float2(a23.z, a23.w), make_float2(a45.x, a45.y), make_float2(a45.z, a45.w),
                     make_float2(a67.x, a67.y), make_float2(a67.z, a67.w)};
      float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                     make_float2(b1.z, b1.w)};
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
          float2 t = __fadd2_rn(a[r], b[c]);
          acc[r][c] = __ffma2_rn(t, t, acc[r][c]);
        }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int c = 0; c < 4; c++) s += acc[r][c].x + acc[r][c].y;
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

__global__ void write_cs(float4* p, size_t n4, float v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  float4 val = make_float4(v, v, v, v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) __stcs(p + i, val);
}
__global__ void write_def(float4* p, size_t n4, float v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  float4 val = make_float4(v, v, v, v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) p[i] = val;
}
// row-segment writes: each CTA writes 4KB contiguous segments of scattered rows (fill-like)
__global__ void write_rows(float4* p, int n, int rows_per_cta, const int* perm, float v) {
  // grid.x = n / rows_per_cta row tiles ; grid.y = n / 1024 column blocks
  int a0 = blockIdx.x * rows_per_cta;
  int col4 = blockIdx.y * 256 + threadIdx.x;
  float4 val = make_float4(v, v, v, v);
  size_t n4 = n / 4;
  for (int a = a0; a < a0 + rows_per_cta; a++) {
    int row = perm[a];
    __stcs(p + (size_t)row * n4 + col4, val);
  }
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d l2 %d MB smemPerBlockOptin %zu\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin);
  float* out;
  CK(cudaMalloc(&out, 148 * 64 * 256 * 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  for (int variant = 0; variant < 2; variant++) {
    int reps = 200;
    int grid = sms * 2 * 4;
    for (int w = 0; w < 2; w++) {
      cudaEventRecord(e0);
      if (variant == 0) scan_scalar<<<grid, 256>>>(out, reps);
      else scan_packed<<<grid, 256>>>(out, reps);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairk = (double)grid * 128 * 128 * KD * reps;
    printf("%s: %.3f ms, %.3f Tpair-k/s (lane-ops %.2f T/s)\n", variant ? "packed" : "scalar", ms,
           pairk / ms / 1e9, 2 * pairk / ms / 1e9);
  }
  // write bandwidth
  size_t bytes = (size_t)8 << 30;
  float4* buf;
  CK(cudaMalloc(&buf, bytes));
  size_t n4 = bytes / 16;
  for (int v = 0; v < 2; v++) {
    for (int blocks_per_sm : {4, 8, 16}) {
      float best = 1e9;
      for (int it = 0; it < 4; it++) {
        cudaEventRecord(e0);
        if (v == 0) write_cs<<<sms * blocks_per_sm, 256>>>(buf, n4, 1.f);
        else write_def<<<sms * blocks_per_sm, 256>>>(buf, n4, 1.f);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("write %s bps=%d: %.3f ms  %.1f GB/s\n", v ? "default" : "stcs", blocks_per_sm, best,
             bytes / best / 1e6);
    }
  }
  {
    int n = 45056;  // 45056^2*4 = 7.56 GiB
    int* perm;
    CK(cudaMalloc(&perm, n * 4));
    int* hp = (int*)malloc(n * 4);
    for (int i = 0; i < n; i++) hp[i] = i;
    srand(1);
    for (int i = n - 1; i > 0; i--) { int j = rand() % (i + 1); int t = hp[i]; hp[i] = hp[j]; hp[j] = t; }
    CK(cudaMemcpy(perm, hp, n * 4, cudaMemcpyHostToDevice));
    for (int rpc : {64, 128, 256}) {
      float best = 1e9;
      for (int it = 0; it < 4; it++) {
        cudaEventRecord(e0);
        write_rows<<<dim3(n / rpc, n / 1024), 256>>>(buf, n, rpc, perm, 2.f);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      double b = (double)n * n * 4;
      printf("write_rows rpc=%d: %.3f ms %.1f GB/s\n", rpc, best, b / best / 1e6);
    }
  }
  // pinned host copies
  {
    size_t hb = (size_t)16 << 30;
    void* h = nullptr;
    cudaError_t e = cudaHostAlloc(&h, hb, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      printf("pinned 16GiB alloc failed: %s\n", cudaGetErrorString(e));
      cudaGetLastError();
      hb = (size_t)4 << 30;
      CK(cudaHostAlloc(&h, hb, cudaHostAllocDefault));
    }
    size_t cb = bytes < hb ? bytes : hb;
    for (int dir = 0; dir < 2; dir++) {
      cudaEventRecord(e0);
      if (dir == 0) CK(cudaMemcpyAsync(buf, h, cb, cudaMemcpyHostToDevice));
      else CK(cudaMemcpyAsync(h, buf, cb, cudaMemcpyDeviceToHost));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s %zu MB pinned: %.2f ms %.1f GB/s\n", dir ? "D2H" : "H2D", cb >> 20, ms, cb / ms / 1e6);
    }
    printf("pinned alloc size used: %zu GiB\n", hb >> 30);
    cudaFreeHost(h);
  }
  size_t fr, tot;
  cudaMemGetInfo(&fr, &tot);
  printf("mem free %zu MiB total %zu MiB\n", fr >> 20, tot >> 20);
  return 0;
}
