// k_scan.cu -- a6: MLGRU gates + linear recurrence + output gate over time
// ("linearized ... enabling a parallel scan").
//
// The recurrence h_t = f_t h_{t-1} + (1-f_t) c_t is evaluated exactly in the
// sequential order of its definition (h and o' bit-identical to the oracle);
// only its two dependent operations per step stay sequential, everything
// transcendental runs parallel over time.  One CTA = 32 channels of one
// sequence, warp-specialised and pipelined over time tiles of kTS steps:
//   warp 0 lane 0   TMA producer: 3 boxes [kTS steps x 32 ch] (f^, c^, g^ of the
//                   fused interleaved pre-activations) per tile into a kS-deep ring
//   warps 2..9      gates, phase 1 of tile i: f = sigma(f^), b = (1-f) SiLU(c^)
//                   (parallel over time, lane = channel); then phase 3 of tile
//                   i-1: o' = g^ sigma(h) (or g^ h) -> global
//   warp 1          the carry: h = f h + b over the tile's steps, in order
// so the serial carry of tile i overlaps the gate work of tiles i+1 and i-1,
// and loads run kS tiles ahead.
#include "epilogue.cuh"

namespace tern {

constexpr int kSCh = 32;                    // channels per CTA (one per lane)
constexpr int kTS = 32;                     // time steps per tile
constexpr int kS = 4;                       // ring stages
constexpr int kGateWarps = 8;
constexpr int kScanThreads = (2 + kGateWarps) * 32;
constexpr int kStepsPerGateWarp = kTS / kGateWarps;

template <typename T>
struct ScanSmem {
  T in[kS][3][kTS][kSCh];       // TMA destination: f^, c^, g^
  float fh[kS][kTS][kSCh];      // f, then h after the carry
  float bv[kS][kTS][kSCh];      // (1-f) c
  uint64_t full[kS], gated[kS], scanned[kS], empty[kS];
};

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan(const __grid_constant__ CUtensorMap tmX, int B,
                                                       int T_, int d, int gate,
                                                       float* __restrict__ h, T* __restrict__ oprime) {
  extern __shared__ __align__(128) uint8_t scan_smem[];
  ScanSmem<T>& sm = *reinterpret_cast<ScanSmem<T>*>(scan_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpb = d / kSCh;                       // channel blocks per sequence
  const int b = blockIdx.x / cpb;
  const int c0 = (blockIdx.x % cpb) * kSCh;
  // interleaved fused layout: per 64-channel group [64 f | 64 c | 64 g]
  const int colf = (c0 / kSegRows) * (3 * kSegRows) + (c0 % kSegRows);
  const int nt = (T_ + kTS - 1) / kTS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.gated[s], kGateWarps);
      mbar_init(&sm.scanned[s], 1);
      mbar_init(&sm.empty[s], kGateWarps);
    }
    fence_barrier_init();
  }
  __syncwarp();
  __syncthreads();
  pdl_wait();                 // f^c^g^ and h come from earlier kernels
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      tma_prefetch_desc(&tmX);
      const uint32_t bytes = 3u * kTS * kSCh * sizeof(T);
      for (int i = 0; i < nt; ++i) {
        const int s = i % kS;
        if (i >= kS) mbar_wait(&sm.empty[s], ((i / kS) - 1) & 1);
        mbar_arrive_expect_tx(&sm.full[s], bytes);
        const int row = b * T_ + i * kTS;
#pragma unroll
        for (int g = 0; g < 3; ++g)
          tma_load_2d(&sm.in[s][g][0][0], &tmX, &sm.full[s], colf + g * kSegRows, row);
      }
    }
  } else if (warp == 1) {
    // ---------------- the carry (exact definition order: (f*h) + ((1-f)*c))
    float hc = h[(int64_t)b * d + c0 + lane];
    for (int i = 0; i < nt; ++i) {
      const int s = i % kS;
      mbar_wait(&sm.gated[s], (i / kS) & 1);
      const int steps = min(kTS, T_ - i * kTS);
      if (steps == kTS) {
#pragma unroll 8
        for (int t = 0; t < kTS; ++t) {
          hc = __fadd_rn(__fmul_rn(sm.fh[s][t][lane], hc), sm.bv[s][t][lane]);
          sm.fh[s][t][lane] = hc;
        }
      } else {
        for (int t = 0; t < steps; ++t) {
          hc = __fadd_rn(__fmul_rn(sm.fh[s][t][lane], hc), sm.bv[s][t][lane]);
          sm.fh[s][t][lane] = hc;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.scanned[s]);
    }
    h[(int64_t)b * d + c0 + lane] = hc;
  } else {
    // ---------------- gate warps
    const int gw = warp - 2;
    T* obase = oprime + (int64_t)b * T_ * d + c0 + lane;
    auto phase1 = [&](int i) {
      const int s = i % kS;
      mbar_wait(&sm.full[s], (i / kS) & 1);
      float fv[kStepsPerGateWarp], bvv[kStepsPerGateWarp];
#pragma unroll
      for (int j = 0; j < kStepsPerGateWarp; ++j) {
        const int t = gw * kStepsPerGateWarp + j;
        const float fx = ld_act<T>(&sm.in[s][0][t][lane]);
        const float cx = ld_act<T>(&sm.in[s][1][t][lane]);
        float f, sc;
        sigmoid2(fx, cx, f, sc);
        fv[j] = f;
        bvv[j] = __fmul_rn(__fsub_rn(1.0f, f), __fmul_rn(cx, sc));   // (1-f) SiLU(c)
      }
#pragma unroll
      for (int j = 0; j < kStepsPerGateWarp; ++j) {
        const int t = gw * kStepsPerGateWarp + j;
        sm.fh[s][t][lane] = fv[j];
        sm.bv[s][t][lane] = bvv[j];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.gated[s]);
    };
    auto phase3 = [&](int i) {
      const int s = i % kS;
      mbar_wait(&sm.scanned[s], (i / kS) & 1);
      float ov[kStepsPerGateWarp];
#pragma unroll
      for (int j = 0; j < kStepsPerGateWarp; j += 2) {
        const int t = gw * kStepsPerGateWarp + j;
        const float g0 = ld_act<T>(&sm.in[s][2][t][lane]), g1 = ld_act<T>(&sm.in[s][2][t + 1][lane]);
        const float h0 = sm.fh[s][t][lane], h1 = sm.fh[s][t + 1][lane];
        if (gate == TERN_GATE_SIGMOID_H) {
          float s0, s1;
          sigmoid2(h0, h1, s0, s1);
          ov[j] = __fmul_rn(g0, s0);
          ov[j + 1] = __fmul_rn(g1, s1);
        } else {
          ov[j] = __fmul_rn(g0, h0);
          ov[j + 1] = __fmul_rn(g1, h1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);   // stage free once read
#pragma unroll
      for (int j = 0; j < kStepsPerGateWarp; ++j) {
        const int t = i * kTS + gw * kStepsPerGateWarp + j;
        if (t < T_) st_act<T>(obase + (int64_t)t * d, ov[j]);
      }
    };
    for (int i = 0; i < nt; ++i) {
      phase1(i);
      if (i > 0) phase3(i - 1);
    }
    phase3(nt - 1);
  }
}

template <typename TE>
static cudaError_t scan_go(const CUtensorMap& tm, int grid, int B, int T, int d, int gate,
                           float* h, void* oprime, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = sizeof(ScanSmem<TE>);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_scan<TE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_scan<TE>, dim3(grid), dim3(kScanThreads), smem, s, tm, B, T, d, gate, h,
                    static_cast<TE*>(oprime));
}

cudaError_t launch_scan(const void* fcg, int dt, int B, int T, int d, int gate, float* h,
                        void* oprime, cudaStream_t s) {
  if (B == 0 || T == 0) return cudaSuccess;
  const int grid = B * (d / kSCh);
  const bool bf = dt == TERN_BF16;
  const size_t es = bf ? 2 : 4;
  CUtensorMap tm;
  if (!make_map_2d(&tm, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, fcg,
                   (uint64_t)3 * d, (uint64_t)B * T, (uint64_t)3 * d * es, kSCh, kTS,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  return bf ? scan_go<__nv_bfloat16>(tm, grid, B, T, d, gate, h, oprime, s)
            : scan_go<float>(tm, grid, B, T, d, gate, h, oprime, s);
}

}  // namespace tern
