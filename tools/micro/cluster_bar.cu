// Microbenchmark (tools/micro, not product code): the latency of one decode "phase exchange"
// inside a thread-block cluster -- every CTA writes its slice of the next activation row into
// every CTA's shared memory (distributed shared memory stores) and the cluster barrier
// (barrier.cluster.arrive.release / wait.acquire) publishes it; then every CTA reads the
// whole row back and reduces it (the next phase's norm).  Cluster sizes 8 and 16, 512 threads,
// ~200 KB of dynamic shared memory per CTA (the size a cluster-resident decode would use).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_bar cluster_bar.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t csize() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ROW floats per row (d = 1024); each CTA owns ROW / csize of them
template <int ROW>
__global__ void __launch_bounds__(512, 1) k(int iters, float* out, long long* cyc) {
  extern __shared__ __align__(16) float sm[];
  float* row = sm;   // [2][ROW] double-buffered
  __shared__ double red[16];
  const uint32_t cr = crank(), cs = csize();
  const int per = ROW / cs;
  for (int i = threadIdx.x; i < 2 * ROW; i += blockDim.x) row[i] = 1.0f;
  cbar();
  const long long t0 = clock64();
  float acc = 0.0f;
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    // "phase": reduce the whole current row (the norm of the next phase)
    double s = 0.0;
    for (int i = threadIdx.x; i < ROW; i += blockDim.x) s += (double)row[b * ROW + i] * row[b * ROW + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < 16; ++w) t += red[w];
    acc += (float)t;
    // this CTA's slice of the next row -> every CTA of the cluster
    const int n = per * (int)cs;   // (all)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int dst = i / per, j = i % per;
      const float v = 1.0f + 1e-7f * (float)(it & 7);
      st_cluster(mapa(su32(&row[(b ^ 1) * ROW + cr * per + j]), (uint32_t)dst), v);
    }
    cbar();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = acc;
    cyc[blockIdx.x] = t1 - t0;
  }
}

template <int ROW>
static void run(int cs) {
  auto kern = k<ROW>;
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  float* out;
  long long* cyc;
  cudaMalloc(&out, 64 * 4);
  cudaMalloc(&cyc, 64 * 8);
  const int iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, 10, out, cyc);
  cudaEventRecord(a);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, iters, out, cyc);
  cudaEventRecord(b);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long h[64];
  cudaMemcpy(h, cyc, cs * 8, cudaMemcpyDeviceToHost);
  printf("cluster %2d, row %d floats: %s, max active clusters %d: %.3f us per phase exchange "
         "(event), %.0f cycles (CTA 0 clock)\n",
         cs, ROW, cudaGetErrorString(e), ncl, ms * 1e3 / iters, (double)h[0] / iters);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1024>(8);
  run<1024>(16);
  run<2816>(16);
  run<2560>(16);
  return 0;
}
