// Microbenchmark: fp64 latency/throughput on this part (tools/micro, not product code).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dadd(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001 + 1e-9;   // DFMA chain
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_fadd(float* out, float a, int n, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fmaf_rn(x, 1.0000001f, 1e-9f);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_f2f(double* out, float a, int n, long long* cyc) {
  float x = a;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double d = (double)x; x = (float)(d * 1.0000001); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr_dfma(double* out, double a, int n) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < n; ++i) {
    x0 = x0 * 1.0000001 + 1e-9; x1 = x1 * 1.0000001 + 1e-9; x2 = x2 * 1.0000001 + 1e-9; x3 = x3 * 1.0000001 + 1e-9;
    x4 = x4 * 1.0000001 + 1e-9; x5 = x5 * 1.0000001 + 1e-9; x6 = x6 * 1.0000001 + 1e-9; x7 = x7 * 1.0000001 + 1e-9;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void thr_f2f(double* out, float a, int n) {
  double acc0 = 0, acc1 = 0;
  float x = a;
  for (int i = 0; i < n; ++i) {
    acc0 += (double)(x + (float)i);
    acc1 += (double)(x - (float)i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
}
__global__ void lat_rsqrt(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(float* out, float a, int n, long long* cyc) {
  float x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0f;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_redux(int* out, int n, long long* cyc) {
  int x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __reduce_add_sync(0xffffffffu, x) + threadIdx.x;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr_redux(int* out, int n) {
  int x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < n; ++i) {
    x0 = __reduce_add_sync(0xffffffffu, x0) ^ i; x1 = __reduce_add_sync(0xffffffffu, x1) ^ i;
    x2 = __reduce_add_sync(0xffffffffu, x2) ^ i; x3 = __reduce_add_sync(0xffffffffu, x3) ^ i;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void lat_bar(float* out, int n, long long* cyc) {
  __shared__ float s[256];
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncthreads(); x = s[(threadIdx.x + 1) & 255]; __syncthreads(); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 64);
  const int n = 4096;
  lat_dadd<<<1, 32>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  lat_dadd<<<1, 32>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cyc\n", (double)h / n);
  lat_fadd<<<1, 32>>>(f, 1.0f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cyc\n", (double)h / n);
  lat_f2f<<<1, 32>>>(d, 1.0f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("F2F.F64.F32 + DMUL + F2F.F32.F64 chain: %.2f cyc\n", (double)h / n);
  lat_rsqrt<<<1, 32>>>(d, 2.0, 256, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt(double)+1 chain: %.2f cyc\n", (double)h / 256);
  lat_shfl<<<1, 32>>>(f, 1.0f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("SHFL+FADD chain: %.2f cyc\n", (double)h / n);
  lat_bar<<<1, 256>>>(f, 1024, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("STS+BAR+LDS+BAR (256 thr): %.2f cyc\n", (double)h / 1024);
  lat_redux<<<1, 32>>>((int*)f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("REDUX.SUM dependent chain: %.2f cyc\n", (double)h / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  {
    float ms2;
    thr_redux<<<148, 512>>>((int*)d, 1024);
    cudaEventRecord(e0); thr_redux<<<148, 512>>>((int*)d, 1024); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms2, e0, e1);
    printf("REDUX throughput: %.2f warp-REDUX per clk per SM at 1.9GHz\n", 4.0 * 1024 * 148 * 16 / (ms2 * 1e-3) / 148 / 1.9e9);
  }
  int blocks = 148 * 8, thr = 256, it = 2048;
  thr_dfma<<<blocks, thr>>>(d, 1.0, it);
  cudaEventRecord(e0); thr_dfma<<<blocks, thr>>>(d, 1.0, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA throughput: %.1f GFLOP/s (%.2f DFMA/clk/SM at 1.9GHz)\n", 2.0 * 8 * it * blocks * thr / ms / 1e6,
         8.0 * it * blocks * thr / (ms * 1e-3) / 148 / 1.9e9);
  thr_f2f<<<blocks, thr>>>(d, 1.0f, it);
  cudaEventRecord(e0); thr_f2f<<<blocks, thr>>>(d, 1.0f, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("F2F.F64.F32+DADD pairs: %.2f per clk per SM at 1.9GHz\n", 2.0 * it * blocks * thr / (ms * 1e-3) / 148 / 1.9e9);
  return 0;
}
