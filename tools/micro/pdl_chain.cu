// Microbenchmark: per-launch cost of a dependent PDL launch chain captured in a CUDA graph
// (tools/micro, not product code).  Kernels of 147 CTAs x 512 threads, like the decode GEMV:
//   v0: griddepcontrol.wait + launch_dependents only
//   v1: + load a 4 KB row (fp32 K = 1024) and a block-wide binary64 sum (one barrier)
//   v2: v1 + every CTA writes 7 floats of the next row (the chain's real data dependency)
//   v3: v2 + a second barrier and a smem round trip (the quant step)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_go() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// v4: + the weights of the CTA bulk-copied into smem before the wait (mbarrier), waited
//     for after the reduce; v5: v4 + an L2 prefetch of 1 MB of later weights per launch
template <int V>
__global__ void __launch_bounds__(512) k(const float* __restrict__ x, float* __restrict__ y, int K,
                                         const uint8_t* __restrict__ wts) {
  __shared__ double red[16];
  __shared__ float q[4096];
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ __align__(8) uint64_t bar;
  if (V >= 4 && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(6144u) : "memory");
    for (int i = 0; i < 6; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(dyn + i * 1024)), "l"(wts + (size_t)blockIdx.x * 6144 + i * 1024), "r"(1024u),
                   "r"(su32(&bar)) : "memory");
  }
  if (V >= 5 && threadIdx.x == 32)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wts + (1 << 20) + (size_t)blockIdx.x * 8192), "r"(8192u) : "memory");
  pdl_wait();
  pdl_go();
  if (V == 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double s = 0.0;
  float v = 0.0f;
  for (int t4 = tid; t4 * 4 < K; t4 += blockDim.x) {
    const float4 a = __ldcg(reinterpret_cast<const float4*>(x) + t4);
    s += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
    v = a.x;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
  for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float r = (float)rsqrt(__shfl_sync(0xffffffffu, s, 0) / K + 1e-6);
  if (V >= 3) {
    q[tid] = v * r;
    __syncthreads();
    v = q[(tid + 1) & (blockDim.x - 1)];
  }
  if (V >= 4) {
    __syncthreads();
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
    v += (float)dyn[tid & 1023];
  }
  if (V >= 2 && tid < 7) y[blockIdx.x * 7 + tid] = v * r + 1.0f;
}

template <int V>
float run(float* a, float* b, int n, int grid = 147, int block = 512, size_t dsmem = 8192,
          const uint8_t* w = nullptr) {
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cfg.dynamicSmemBytes = dsmem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k<V>, (const float*)(i & 1 ? b : a), (i & 1 ? a : b), 1024, w);
  if (cudaStreamEndCapture(s, &g) != cudaSuccess) return -1.0f;
  cudaGraphExec_t ge;
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -1.0f;
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / (20 * n);
}

int main() {
  float *a, *b;
  cudaMalloc(&a, 1 << 20);
  cudaMalloc(&b, 1 << 20);
  cudaMemset(a, 0, 1 << 20);
  cudaMemset(b, 0, 1 << 20);
  uint8_t* w;
  cudaMalloc(&w, 4 << 20);
  cudaMemset(w, 1, 4 << 20);
  printf("PDL chain, 147 CTAs x 512 threads, us per launch:\n");
  printf("  v0 wait+trigger only           %.2f\n", run<0>(a, b, 96));
  printf("  v1 + 4KB load + block reduce   %.2f\n", run<1>(a, b, 96));
  printf("  v2 + dependent 7-float store   %.2f\n", run<2>(a, b, 96));
  printf("  v3 + 2nd barrier (quant)       %.2f\n", run<3>(a, b, 96));
  printf("  v4 + 6KB bulk-copied weights   %.2f\n", run<4>(a, b, 96, 147, 512, 8192, w));
  printf("  v4 with 100 KB dynamic smem    %.2f\n", run<4>(a, b, 96, 147, 512, 100 * 1024, w));
  printf("  v4 with 150 KB dynamic smem    %.2f\n", run<4>(a, b, 96, 147, 512, 150 * 1024, w));
  printf("  v5 + L2 prefetch               %.2f\n", run<5>(a, b, 96, 147, 512, 8192, w));
  const int gb[][2] = {{147, 256}, {74, 512}, {74, 256}, {37, 512}, {16, 512}};
  for (auto& c : gb)
    printf("  v3 grid %3d x %4d threads: %.2f  (v0 %.2f)\n", c[0], c[1], run<3>(a, b, 96, c[0], c[1]),
           run<0>(a, b, 96, c[0], c[1]));
  return 0;
}
