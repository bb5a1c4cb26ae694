// Microbenchmark: instruction-cache cold/warm cost of long straight-line code.
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__device__ __forceinline__ float body(float x0, float x1) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    x0 = __fmaf_rn(x0, 1.0001f, 0.5f);
    x1 = __fmaf_rn(x1, 0.9999f, 0.25f);
    asm volatile("" : "+f"(x0), "+f"(x1));
  }
  return x0 + x1;
}
template <int N>
__global__ void k(float* out, long long* cyc) {
  float x = threadIdx.x;
  long long t0 = clock64();
  x = body<N>(x, x + 1);
  long long t1 = clock64();
  x = body<N>(x, x + 2);   // different copy of the code (inlined again): still cold
  long long t2 = clock64();
  for (int r = 0; r < 2; ++r) x = body<N>(x, x + r);   // same code run twice: second warm
  long long t3 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  float* f; long long* c; long long h[3];
  cudaMalloc(&f, 4096); cudaMalloc(&c, 64);
  k<1024><<<1, 32>>>(f, c); cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("N=1024 (2 FFMA chains): copy1 %lld cyc, copy2 %lld cyc, loop x2 (same code) %lld cyc; ideal ~%d\n", h[0], h[1], h[2], 1024 * 5);
  k<1024><<<1, 32>>>(f, c); cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("relaunch: copy1 %lld cyc, copy2 %lld cyc, loop x2 %lld cyc\n", h[0], h[1], h[2]);
  k<256><<<148, 32>>>(f, c); cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("N=256: copy1 %lld cyc, copy2 %lld, loop x2 %lld; ideal ~%d\n", h[0], h[1], h[2], 256 * 5);
  return 0;
}
