// latency of warp reductions on sm_100a: dependent chains of redux.sync.min.u32 vs a
// 5-level shuffle-xor min, and bar.sync among 4 warps (clock64 per iteration)
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out, long long* cyc, int iters) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) v = __reduce_min_sync(0xffffffffu, v ^ i) + threadIdx.x;
  long long t1 = clock64();
  for (int i = 0; i < iters; i++) {
    unsigned x = v ^ i;
    for (int o = 16; o; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    v = x + threadIdx.x;
  }
  long long t2 = clock64();
  for (int i = 0; i < iters; i++) {
    unsigned m = __reduce_min_sync(0xffffffffu, v ^ i);
    v = __reduce_min_sync(0xffffffffu, (v ^ i) == m ? threadIdx.x : 0xffffffffu) + m;
  }
  long long t3 = clock64();
  __shared__ unsigned s[4];
  for (int i = 0; i < iters; i++) {
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v + i;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    v = s[(threadIdx.x >> 5) ^ 1] + 1;
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = v;
}
int main() {
  unsigned* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  for (int rep = 0; rep < 2; rep++) { k<<<1, 128>>>(o, c, 1000); cudaDeviceSynchronize(); }
  printf("cycles per iteration: redux %.1f  shfl-5 %.1f  redux-argmin(2) %.1f  bar4+sts/lds %.1f\n", c[0] / 1000.0,
         c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0);
  return 0;
}
