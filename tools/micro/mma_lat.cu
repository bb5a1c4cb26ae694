// Microbenchmark: tcgen05.mma kind::i8 (M = 128, K = 32 per instruction, operands in smem)
// throughput and issue -> commit latency for N = 64 / 128 / 256 (tools/micro, not product code).
// One CTA; groups of 4 MMAs (one 128-K k-block) each followed by a commit to an mbarrier; at
// most D groups in flight (the thread waits for group i-D before issuing group i).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2406_02528_b200/csrc/common.cuh"
using namespace tern;

template <int N, int M = 128>
__global__ void k(int groups, int depth, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint8_t* A = sm;                 // 128 x 128 u8, SW128
  uint8_t* B = sm + 16384;         // N x 128 s8, SW128
  __shared__ __align__(8) uint64_t bar[16];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) { for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (g >= depth) mbar_wait_spin(&bar[(g - depth) & 15], ((g - depth) >> 4) & 1);
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(tmem + (g & 1) * 256, umma_desc_sw128(smem_u32(A) + kk * 32), umma_desc_sw128(smem_u32(B) + kk * 32), idesc, kk != 0);
      mma_commit(&bar[g & 15]);
    }
    for (int g = groups - depth < 0 ? 0 : groups - depth; g < groups; ++g) mbar_wait_spin(&bar[g & 15], (g >> 4) & 1);
    const long long t1 = clock64();
    out[0] = t1 - t0;
    // single-group latency: issue, commit, wait
    const long long t2 = clock64();
    tc_fence_after();
    for (int kk = 0; kk < 4; ++kk)
      mma_i8(tmem, umma_desc_sw128(smem_u32(A) + kk * 32), umma_desc_sw128(smem_u32(B) + kk * 32), idesc, kk != 0);
    mma_commit(&bar[groups & 15]);
    mbar_wait_spin(&bar[groups & 15], (groups >> 4) & 1);
    out[1] = clock64() - t2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, int M = 128>
void run(long long* d) {
  cudaFuncSetAttribute(k<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  long long h[2];
  for (int depth : {2, 8}) {
    k<N, M><<<1, 128, 16384 + N * 128 + 1024>>>(64, depth, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("M=%3d N=%3d depth %d: %.0f cycles per k-block group (4 MMAs), single-group latency %lld cycles (ideal %d)\n",
           M, N, depth, (double)h[0] / 64, h[1], 4 * 128 * N / 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<64>(d);
  run<128>(d);
  run<256>(d);
  run<64, 64>(d);
  run<128, 64>(d);
  run<256, 64>(d);
  run<32>(d);
  return 0;
}
