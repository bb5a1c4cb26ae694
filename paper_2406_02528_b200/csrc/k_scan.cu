// k_scan.cu -- a6: MLGRU gates + linear recurrence + output gate over time
// ("linearized ... enabling a parallel scan").
//
// The recurrence h_t = f_t h_{t-1} + (1-f_t) c_t is evaluated exactly in the
// sequential order of its definition (so h and o' are bit-identical to the
// oracle), but only the two dependent operations per step stay sequential.
// Per CTA (32 channels of one sequence, 8 warps) and time tile of 64 steps:
//   phase 1 (all warps, parallel over time): f = sigma(fhat), c = SiLU(chat),
//           b = (1-f) c  -> smem;  the next tile's loads are issued here
//   phase 2 (one warp): h = f*h + b for 64 steps (FMUL + FADD per step)
//   phase 3 (all warps, parallel over time): o' = ghat * sigma(h) -> global
// This is the "chunked parallel scan" of the transcendental work with a
// sequential carry: it keeps parity exact while spreading ~95% of the
// arithmetic over time.
#include "epilogue.cuh"

namespace tern {

constexpr int kSCh = 32;         // channels per CTA (one per lane)
constexpr int kSWarps = 8;
constexpr int kSTile = 64;       // time steps per tile
constexpr int kSPerWarp = kSTile / kSWarps;

template <typename T>
__global__ void __launch_bounds__(kSWarps * 32) k_scan(const T* __restrict__ fcg, int B, int T_,
                                                       int d, int gate, float* __restrict__ h,
                                                       T* __restrict__ oprime) {
  __shared__ float sF[kSTile][kSCh];   // f, then h after phase 2
  __shared__ float sB[kSTile][kSCh];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpb = d / kSCh;                       // channel blocks per sequence
  const int b = blockIdx.x / cpb;
  const int c0 = (blockIdx.x % cpb) * kSCh;
  const int ch = c0 + lane;
  // interleaved fused layout: per 64-channel group [64 f | 64 c | 64 g]
  const int colf = (c0 / kSegRows) * (3 * kSegRows) + (c0 % kSegRows) + lane;
  const int64_t ld = 3 * (int64_t)d;
  const T* base = fcg + (int64_t)b * T_ * ld;
  T* obase = oprime + (int64_t)b * T_ * d;

  float nf[kSPerWarp], nc[kSPerWarp], ng[kSPerWarp];
  auto load_tile = [&](int t0) {
#pragma unroll
    for (int i = 0; i < kSPerWarp; ++i) {
      const int t = t0 + warp * kSPerWarp + i;
      if (t < T_) {
        const T* p = base + (int64_t)t * ld + colf;
        nf[i] = ld_act<T>(p);
        nc[i] = ld_act<T>(p + kSegRows);
        ng[i] = ld_act<T>(p + 2 * kSegRows);
      } else {
        nf[i] = 0.0f; nc[i] = 0.0f; ng[i] = 0.0f;
      }
    }
  };

  float hc = (warp == 0) ? h[(int64_t)b * d + ch] : 0.0f;
  load_tile(0);
  for (int t0 = 0; t0 < T_; t0 += kSTile) {
    float gcur[kSPerWarp];
    // phase 1: gates, parallel over time
    float fv[kSPerWarp], bv[kSPerWarp];
#pragma unroll
    for (int i = 0; i < kSPerWarp; ++i) {
      const float f = sigmoid_vec(nf[i]);
      const float c = __fmul_rn(nc[i], sigmoid_vec(nc[i]));
      fv[i] = f;
      bv[i] = __fmul_rn(__fsub_rn(1.0f, f), c);
      gcur[i] = ng[i];
    }
#pragma unroll
    for (int i = 0; i < kSPerWarp; ++i) {
      sF[warp * kSPerWarp + i][lane] = fv[i];
      sB[warp * kSPerWarp + i][lane] = bv[i];
    }
    if (t0 + kSTile < T_) load_tile(t0 + kSTile);  // prefetch the next tile
    __syncthreads();
    // phase 2: the sequential carry (exact definition order: (f*h) + ((1-f)*c))
    if (warp == 0) {
      const int steps = min(kSTile, T_ - t0);
      if (steps == kSTile) {
#pragma unroll 8
        for (int t = 0; t < kSTile; ++t) {
          hc = __fadd_rn(__fmul_rn(sF[t][lane], hc), sB[t][lane]);
          sF[t][lane] = hc;
        }
      } else {
        for (int t = 0; t < steps; ++t) {
          hc = __fadd_rn(__fmul_rn(sF[t][lane], hc), sB[t][lane]);
          sF[t][lane] = hc;
        }
      }
    }
    __syncthreads();
    // phase 3: output gate, parallel over time
    float ov[kSPerWarp];
#pragma unroll
    for (int i = 0; i < kSPerWarp; ++i) {
      const float hv = sF[warp * kSPerWarp + i][lane];
      ov[i] = gate == TERN_GATE_SIGMOID_H ? __fmul_rn(gcur[i], sigmoid_vec(hv))
                                          : __fmul_rn(gcur[i], hv);
    }
#pragma unroll
    for (int i = 0; i < kSPerWarp; ++i) {
      const int t = t0 + warp * kSPerWarp + i;
      if (t < T_) st_act<T>(obase + (int64_t)t * d + ch, ov[i]);
    }
    __syncthreads();
  }
  if (warp == 0) h[(int64_t)b * d + ch] = hc;
}

cudaError_t launch_scan(const void* fcg, int dt, int B, int T, int d, int gate, float* h,
                        void* oprime, cudaStream_t s) {
  if (B == 0 || T == 0) return cudaSuccess;
  const int grid = B * (d / kSCh);
  if (dt == TERN_BF16)
    k_scan<__nv_bfloat16><<<grid, kSWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(fcg), B, T, d, gate, h,
        static_cast<__nv_bfloat16*>(oprime));
  else
    k_scan<float><<<grid, kSWarps * 32, 0, s>>>(static_cast<const float*>(fcg), B, T, d, gate, h,
                                                static_cast<float*>(oprime));
  return cudaGetLastError();
}

}  // namespace tern
