// k_pack.cu -- a1: absmean ternarization + 2-bit packing (Alg. 1 weight_quant,
// PAPER.md P:344-348; readings C3, C4, C6, C7; layout: DESIGN.md "Packed weight
// layout" / tern.h).  Offline: runs once per matrix at model build.
#include "common.cuh"
#include "internal.h"

namespace tern {

constexpr int kAbsThreads = 256;
constexpr int kAbsBlocks = 512;   // fixed -> deterministic partial-sum tree

// Partial sums of |W| in binary64: block b owns elements b, b + B, b + 2B, ... per
// thread in a fixed pattern, reduced by a fixed shuffle tree.
__global__ void __launch_bounds__(kAbsThreads) k_absmean_partial(const float* __restrict__ W,
                                                                 int64_t n, double* part) {
  double s = 0.0;
  const int64_t stride = (int64_t)kAbsBlocks * kAbsThreads;
  for (int64_t i = (int64_t)blockIdx.x * kAbsThreads + threadIdx.x; i < n; i += stride) {
    float v = W[i];
    // a non-finite weight poisons the sum (caught on the host, C7)
    s += fabs((double)v);
  }
  s = warp_sum_f64(s);
  __shared__ double ws[kAbsThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kAbsThreads / 32; ++i) t += ws[i];
    part[blockIdx.x] = t;
  }
}

// m = (float)(sum / n); written to scale_out (or copied from scale_in).
__global__ void k_absmean_final(const double* part, int64_t n, const float* scale_in,
                                float* scale_out) {
  if (threadIdx.x != 0) return;
  if (scale_in) {
    *scale_out = *scale_in;
    return;
  }
  double t = 0.0;
  for (int i = 0; i < kAbsBlocks; ++i) t += part[i];
  *scale_out = (float)(t / (double)n);
}

// One thread per packed word: trits k = 16w .. 16w+15 of logical row r.
__global__ void k_pack(const float* __restrict__ W, int n, int k, int n_seg, int seg,
                       uint32_t* __restrict__ codes, int n_rows, const float* __restrict__ scale) {
  const int words_per_row = (k + 15) / 16;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * words_per_row) return;
  const int r = (int)(idx / words_per_row);
  const int w = (int)(idx % words_per_row);
  const float m = *scale;
  const float s = __fdiv_rn(1.0f, m);
  uint32_t word = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int kk = w * 16 + i;
    int e = 1;  // zero trit for the K padding
    if (kk < k) {
      float v = round_half_away(__fmul_rn(W[(int64_t)r * k + kk], s));
      v = fminf(fmaxf(v, -1.0f), 1.0f);
      e = (int)v + 1;
    }
    const int j = i & 3, f = i >> 2;
    word |= (uint32_t)e << (8 * j + 2 * f);
  }
  // K-block-major: [w/8][packed row][w%8]
  codes[((int64_t)(w >> 3) * n_rows + packed_row(seg, r, n_seg)) * 8 + (w & 7)] = word;
}

__global__ void k_codes_init(uint32_t* codes, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) codes[i] = 0x55555555u;  // every field = 1 (trit 0)
}

cudaError_t launch_codes_init(uint32_t* codes, int n_rows, int ldw, cudaStream_t s) {
  int64_t n = (int64_t)n_rows * ldw;
  k_codes_init<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(codes, n);
  return cudaGetLastError();
}

cudaError_t launch_absmean(const float* W, int64_t numel, const float* scale_in, float* scale_out,
                           double* ws, cudaStream_t s) {
  if (!scale_in) k_absmean_partial<<<kAbsBlocks, kAbsThreads, 0, s>>>(W, numel, ws);
  k_absmean_final<<<1, 32, 0, s>>>(ws, numel, scale_in, scale_out);
  return cudaGetLastError();
}

cudaError_t launch_pack_codes(const float* W, int n, int k, int n_seg, int seg, uint32_t* codes,
                              int n_rows, const float* scale, cudaStream_t s) {
  const int64_t words = (int64_t)n * ((k + 15) / 16);
  k_pack<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(W, n, k, n_seg, seg, codes, n_rows, scale);
  return cudaGetLastError();
}

size_t pack_workspace_bytes() { return sizeof(double) * kAbsBlocks; }

}  // namespace tern
