// Microbenchmark: cycles per step of the exact MLGRU carry h = fl(fl(f*h) + b)
// for one warp over shared memory, with and without competing warps.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kC = 8, kTS = 128, kTiles = 16;

template <int MODE>
__global__ void carry(float* out, long long* cyc, int busy) {
  __shared__ float sm[3 * kTS * kC];
  float* fh = sm; float* bv = sm + kTS * kC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kTS * kC; i += blockDim.x) fh[i] = 0.5f + 1e-3f * i, bv[i] = 0.25f;
  __syncthreads();
  if (warp == 1 && lane < kC) {
    float hc = 0.f;
    long long t0 = clock64();
    for (int tile = 0; tile < kTiles; ++tile) {
      float* f = fh + lane;
      const float* b = bv + lane;
      if (MODE == 0) {
#pragma unroll 8
        for (int t = 0; t < kTS; ++t) {
          hc = __fadd_rn(__fmul_rn(f[t * kC], hc), b[t * kC]);
          f[t * kC] = hc;
        }
      } else if (MODE == 1) {
#pragma unroll
        for (int t = 0; t < kTS; ++t) {
          hc = __fadd_rn(__fmul_rn(f[t * kC], hc), b[t * kC]);
          f[t * kC] = hc;
        }
      } else if (MODE == 4) {      // separate h array, full unroll
        float* hs = f + kTS * kC * 2;   // scratch beyond bv (see smem layout)
#pragma unroll
        for (int t = 0; t < kTS; ++t) {
          hc = __fadd_rn(__fmul_rn(f[t * kC], hc), b[t * kC]);
          hs[t * kC] = hc;
        }
      } else if (MODE == 5) {      // software pipelined batches of 8 (k_scan style)
        float fa[8], ba[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) fa[u] = f[u * kC], ba[u] = b[u * kC];
#pragma unroll 1
        for (int t0 = 0; t0 < kTS; t0 += 8) {
          float fn[8], bn[8];
          const int tn = t0 + 8 < kTS ? t0 + 8 : t0;
#pragma unroll
          for (int u = 0; u < 8; ++u) fn[u] = f[(tn + u) * kC], bn[u] = b[(tn + u) * kC];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            hc = __fadd_rn(__fmul_rn(fa[u], hc), ba[u]);
            f[(t0 + u) * kC] = hc;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) fa[u] = fn[u], ba[u] = bn[u];
        }
      } else if (MODE == 6) {      // batches of 32: load all, then chain, then store all
#pragma unroll 1
        for (int t0 = 0; t0 < kTS; t0 += 32) {
          float fa[32], ba[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) fa[u] = f[(t0 + u) * kC], ba[u] = b[(t0 + u) * kC];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            hc = __fadd_rn(__fmul_rn(fa[u], hc), ba[u]);
            fa[u] = hc;
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) f[(t0 + u) * kC] = fa[u];
        }
      } else if (MODE == 2) {      // chain only, operands in registers
        float a = f[0], c = b[0];
#pragma unroll 16
        for (int t = 0; t < kTS; ++t) hc = __fadd_rn(__fmul_rn(a, hc), c);
      } else {                     // FMA chain (not exact-definition; latency reference)
        float a = f[0], c = b[0];
#pragma unroll 16
        for (int t = 0; t < kTS; ++t) hc = __fmaf_rn(a, hc, c);
      }
      __syncwarp(0xffu);
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * kC + lane] = hc;
  } else if (warp >= 2 && busy) {
    float x = threadIdx.x * 1e-3f, y = 1.0001f;
    for (int i = 0; i < busy; ++i) {
#pragma unroll 16
      for (int u = 0; u < 16; ++u) x = __fmaf_rn(x, y, 1e-7f);
    }
    out[4096 + threadIdx.x] = x;
  }
}

template <int MODE>
void run(const char* name, int busy, int threads) {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8 * 128);
  carry<MODE><<<1, threads>>>(out, cyc, busy);
  carry<MODE><<<1, threads>>>(out, cyc, busy);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s busy=%d threads=%d: %.2f cycles/step\n", name, busy, threads, (double)c / (kTS * kTiles));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int busy : {0, 2000}) {
    run<0>("smem, unroll 8", busy, 384);
    run<1>("smem, full unroll", busy, 384);
    run<4>("smem, separate h array", busy, 384);
    run<5>("smem, pipelined batch 8", busy, 384);
    run<6>("smem, batch 32 ld/chain/st", busy, 384);
    run<2>("regs, mul+add", busy, 384);
    run<3>("regs, fma", busy, 384);
  }
  return 0;
}
