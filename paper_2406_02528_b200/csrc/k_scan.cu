// k_scan.cu -- a6: MLGRU gates + linear recurrence + output gate over time
// ("linearized ... enabling a parallel scan").
//
// The recurrence h_t = f_t h_{t-1} + (1-f_t) c_t is evaluated exactly in the
// sequential order of its definition (h and o' bit-identical to the oracle);
// only its two dependent operations per step stay sequential, everything
// transcendental runs parallel over time.  One CTA = kC (32, 16 or 8) channels of
// one sequence, warp-specialised and pipelined over time tiles of kTS = 1024/kC steps:
//   warp 0 lane 0   TMA producer: 3 boxes [kTS steps x kC ch] (f^, c^, g^ of the
//                   fused interleaved pre-activations) per tile into a kS-deep ring
//   warps 2..9      gates, phase 1 of tile i: f = sigma(f^), b = (1-f) SiLU(c^)
//                   (parallel over time and channels); then phase 3 of tile
//                   i-kLag: o' = g^ sigma(h) (or g^ h) -> global
//   warp 1          the carry: h = f h + b over the tile's steps, in order (lane = channel)
// so the serial carry of tile i overlaps the gate work of the tiles around it,
// and loads run kS tiles ahead.
#include <cstdio>
#include <type_traits>

#include "epilogue.cuh"

namespace tern {

// A tile holds kTE = 1024 (step, channel) elements: kC channels x kTS = kTE / kC
// steps.  kC = 32 (lane = channel) when the grid B*d/32 already fills the SMs; for
// small B*d the CTA narrows to 16 or 8 channels so that the gate arithmetic, which is
// what bounds a CTA here (3 exact sigmoids per element on the FP32 pipe, ~45 cycles
// per step at kC = 32), spreads over up to 4x more SMs.  The carry keeps one lane per
// channel and walks kTS steps per tile.
constexpr int kTE = 1024;
constexpr int kSShallow = 4;                // ring stages when >= 1 CTA per SM is busy
constexpr int kSDeep = 8;                   // ring stages for small grids
constexpr int kGateWarps = 8;
// 12 warps: 0 producer, 1 carry, 5 and 9 idle, the other 8 the gates.  Warp w issues
// from sub-partition w % 4, so the carry's dependent chain owns sub-partition 1 instead
// of sharing its issue slots with two busy gate warps.
constexpr int kScanThreads = 12 * 32;
__device__ __forceinline__ int gate_warp_index(int warp) {   // -1: not a gate warp
  return (warp < 2 || warp == 5 || warp == 9) ? -1 : warp - 2 - (warp > 5) - (warp > 9);
}
constexpr int kElemsPerLane = kTE / (kGateWarps * 32);   // 4

// The carry reads (f, b) of two steps as one 16-byte word and writes h of four steps as
// one: fb[(t/2)*kC + c] = (f_t, b_t, f_t+1, b_t+1), hs[(t/4)*kC + c] = (h_t .. h_t+3).
// This keeps the chain's loads and stores (1/2 + 1/2 + 1/4 per step) off its critical
// path: the loop then runs at the FMUL->FADD latency (measured, tools/micro).
template <int kC>
__device__ __forceinline__ int fb_word(int e) {   // word index of f for element e = t*kC + c
  const int t = e / kC, c = e % kC;
  return ((t >> 1) * kC + c) * 4 + (t & 1) * 2;
}
template <int kC>
__device__ __forceinline__ int h_word(int e) {
  const int t = e / kC, c = e % kC;
  return ((t >> 2) * kC + c) * 4 + (t & 3);
}

template <typename T, int kS>
struct ScanSmem {
  T in[kS][3][kTE];                         // TMA destination: f^, c^, g^ boxes [kTS][kC]
  __align__(16) float fb[kS][2 * kTE];      // (f, (1-f) c) pairs, layout above
  __align__(16) float hs[kS][kTE];          // h after the carry, layout above
  uint64_t full[kS], gated[kS], scanned[kS], empty[kS];
};

// AGG (sequence-parallel pass 1, reading C23): no outputs; the carry runs the recurrence
// from h = 0 and the running product of f, and writes the slice aggregate (A, B) to
// agg [2][B][d].
template <typename T, int kS, int kC, bool AGG = false>
__global__ void __launch_bounds__(kScanThreads) k_scan(const __grid_constant__ CUtensorMap tmX, int B,
                                                       int T_, int d, int gate,
                                                       float* __restrict__ h, T* __restrict__ oprime,
                                                       unsigned long long* prof,
                                                       float* __restrict__ agg) {
  // prof (debug, TERN_SCAN_PROF): per CTA [8] cycles: producer empty-wait, carry
  // gated-wait, carry total, gate0 full-wait, phase 1, scanned-wait, phase 3, gate0 total
  constexpr int kTS = kTE / kC;
  extern __shared__ __align__(128) uint8_t scan_smem[];
  ScanSmem<T, kS>& sm = *reinterpret_cast<ScanSmem<T, kS>*>(scan_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpb = d / kC;                         // channel blocks per sequence
  const int b = blockIdx.x / cpb;
  const int c0 = (blockIdx.x % cpb) * kC;
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
      const uint32_t bytes = 3u * kTE * sizeof(T);
      for (int i = 0; i < nt; ++i) {
        const int s = i % kS;
        if (i >= kS) {
          const long long w0 = prof ? clock64() : 0;
          mbar_wait(&sm.empty[s], ((i / kS) - 1) & 1);
          if (prof) prof[blockIdx.x * 8 + 0] += clock64() - w0;
        }
        mbar_arrive_expect_tx(&sm.full[s], bytes);
        const int row = b * T_ + i * kTS;
#pragma unroll
        for (int g = 0; g < 3; ++g)
          tma_load_2d(&sm.in[s][g][0], &tmX, &sm.full[s], colf + g * kSegRows, row);
      }
    }
  } else if (warp == 1) {
    // ---------------- the carry (exact definition order: (f*h) + ((1-f)*c))
    if (lane < kC) {
      float hc = AGG ? 0.0f : h[(int64_t)b * d + c0 + lane];
      float Ac = 1.0f;   // AGG: running product of f, left to right
      const long long c_t0 = clock64();
      long long c_w = 0;
      for (int i = 0; i < nt; ++i) {
        const int s = i % kS;
        const long long w0 = clock64();
        mbar_wait(&sm.gated[s], (i / kS) & 1);
        c_w += clock64() - w0;
        const int steps = min(kTS, T_ - i * kTS);
        const float4* __restrict__ fb4 = reinterpret_cast<const float4*>(sm.fb[s]) + lane;
        float4* __restrict__ hs4 = reinterpret_cast<float4*>(sm.hs[s]) + lane;
        if (steps == kTS) {
          // (f, b) of group g + 2 are loaded (in program order) before group g's h is
          // stored, so the shared-memory latency overlaps the dependent chain
          constexpr int kG = kTS / 4;   // groups of 4 steps
          float4 pf[kG], qf[kG];
          pf[0] = fb4[0], qf[0] = fb4[kC];
          if (kG > 1) pf[1] = fb4[2 * kC], qf[1] = fb4[3 * kC];
#pragma unroll
          for (int g = 0; g < kG; ++g) {
            if (g + 2 < kG) pf[g + 2] = fb4[(2 * g + 4) * kC], qf[g + 2] = fb4[(2 * g + 5) * kC];
            const float4 p = pf[g], q = qf[g];
            float4 o;
            o.x = __fadd_rn(__fmul_rn(p.x, hc), p.y);
            o.y = __fadd_rn(__fmul_rn(p.z, o.x), p.w);
            o.z = __fadd_rn(__fmul_rn(q.x, o.y), q.y);
            o.w = __fadd_rn(__fmul_rn(q.z, o.z), q.w);
            if (AGG) {
              Ac = __fmul_rn(__fmul_rn(__fmul_rn(__fmul_rn(Ac, p.x), p.z), q.x), q.z);
            } else {
              hs4[g * kC] = o;
            }
            hc = o.w;
          }
        } else {
          for (int t = 0; t < steps; ++t) {
            const int e = t * kC + lane;
            const float* fbw = &sm.fb[s][fb_word<kC>(e)];
            hc = __fadd_rn(__fmul_rn(fbw[0], hc), fbw[1]);
            if (AGG) Ac = __fmul_rn(Ac, fbw[0]);
            else sm.hs[s][h_word<kC>(e)] = hc;
          }
        }
        __syncwarp(kC == 32 ? 0xffffffffu : (1u << (kC & 31)) - 1u);
        if (lane == 0) mbar_arrive(&sm.scanned[s]);
      }
      if (AGG) {
        agg[(int64_t)b * d + c0 + lane] = Ac;
        agg[(int64_t)(B + b) * d + c0 + lane] = hc;
      } else {
        h[(int64_t)b * d + c0 + lane] = hc;
      }
      if (prof && lane == 0) {
        prof[blockIdx.x * 8 + 1] = c_w;
        prof[blockIdx.x * 8 + 2] = clock64() - c_t0;
      }
    }
  } else if (gate_warp_index(warp) >= 0) {
    // ---------------- gate warps: element e = (gw*4 + j)*32 + lane <-> (t = e / kC, c = e % kC)
    const int gw = gate_warp_index(warp);
    const int c = lane % kC;
    T* obase = oprime + (int64_t)b * T_ * d + c0 + c;
    const bool pr = prof && gw == 0 && lane == 0;
    long long acc[5] = {0, 0, 0, 0, 0};
    const long long g_t0 = clock64();
    auto phase1 = [&](int i) {
      const int s = i % kS;
      long long w0 = clock64();
      mbar_wait(&sm.full[s], (i / kS) & 1);
      long long w1 = clock64();
      acc[0] += w1 - w0;
      float fv[kElemsPerLane], bvv[kElemsPerLane];
#pragma unroll
      for (int j = 0; j < kElemsPerLane; ++j) {
        const int e = (gw * kElemsPerLane + j) * 32 + lane;
        const float fx = ld_act<T>(&sm.in[s][0][e]);
        const float cx = ld_act<T>(&sm.in[s][1][e]);
        float f, sc;
        sigmoid2(fx, cx, f, sc);
        fv[j] = f;
        bvv[j] = __fmul_rn(__fsub_rn(1.0f, f), __fmul_rn(cx, sc));   // (1-f) SiLU(c)
      }
#pragma unroll
      for (int j = 0; j < kElemsPerLane; ++j) {
        const int e = (gw * kElemsPerLane + j) * 32 + lane;
        *reinterpret_cast<float2*>(&sm.fb[s][fb_word<kC>(e)]) = make_float2(fv[j], bvv[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.gated[s]);
      acc[1] += clock64() - w1;
    };
    auto phase3 = [&](int i) {
      const int s = i % kS;
      long long w0 = clock64();
      mbar_wait(&sm.scanned[s], (i / kS) & 1);
      long long w1 = clock64();
      acc[2] += w1 - w0;
      if (AGG) {   // nothing to output: release the stage
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
        return;
      }
      // the gate mode and full tiles are resolved per tile, not per element
      auto out_tile = [&](auto full_c, auto sig_c) {
        constexpr bool kFull = decltype(full_c)::value, kSig = decltype(sig_c)::value;
        float ov[kElemsPerLane];
#pragma unroll
        for (int j = 0; j < kElemsPerLane; j += 2) {
          const int e = (gw * kElemsPerLane + j) * 32 + lane;
          const float g0 = ld_act<T>(&sm.in[s][2][e]), g1 = ld_act<T>(&sm.in[s][2][e + 32]);
          const float h0 = sm.hs[s][h_word<kC>(e)], h1 = sm.hs[s][h_word<kC>(e + 32)];
          if constexpr (kSig) {
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
        for (int j = 0; j < kElemsPerLane; ++j) {
          const int t = i * kTS + ((gw * kElemsPerLane + j) * 32 + lane) / kC;
          if (kFull || t < T_) st_act<T>(obase + (int64_t)t * d, ov[j]);
        }
      };
      const bool full = (i + 1) * kTS <= T_, sig = gate == TERN_GATE_SIGMOID_H;
      if (full) {
        if (sig) out_tile(std::true_type{}, std::true_type{});
        else out_tile(std::true_type{}, std::false_type{});
      } else {
        if (sig) out_tile(std::false_type{}, std::true_type{});
        else out_tile(std::false_type{}, std::false_type{});
      }
      acc[3] += clock64() - w1;
    };
    // phase 1 runs kLag tiles ahead of phase 3 so that the carry warp finds the next
    // tiles gated while the gate warps wait for it (kLag <= kS - 1: the stage phase 1
    // fills next was released by a phase 3 already issued)
    constexpr int kLag = kS >= 8 ? 4 : 1;
    for (int i = 0; i < nt; ++i) {
      phase1(i);
      if (i >= kLag) phase3(i - kLag);
    }
    for (int i = max(nt - kLag, 0); i < nt; ++i) phase3(i);
    if (pr) {
      for (int k = 0; k < 4; ++k) prof[blockIdx.x * 8 + 3 + k] = acc[k];
      prof[blockIdx.x * 8 + 7] = clock64() - g_t0;
    }
  }
}

template <typename TE, int kS, int kC, bool AGG = false>
static cudaError_t scan_go(const void* fcg, int B, int T, int d, int gate, float* h,
                           void* oprime, cudaStream_t s, float* agg = nullptr) {
  static bool attr = false;
  const size_t smem = sizeof(ScanSmem<TE, kS>);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_scan<TE, kS, kC, AGG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const bool bf = sizeof(TE) == 2;
  CUtensorMap tm;
  if (!make_map_2d(&tm, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, fcg,
                   (uint64_t)3 * d, (uint64_t)B * T, (uint64_t)3 * d * sizeof(TE), kC, kTE / kC,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  const int grid = B * (d / kC);
  static unsigned long long* dprof = nullptr;
  static const bool prof_on = getenv("TERN_SCAN_PROF") != nullptr;
  if (prof_on) {   // debug only: printed after a synchronous run
    if (!dprof) cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * 4096);
    cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * 8 * 4096, s);
  }
  cudaError_t e = launch_pdl(k_scan<TE, kS, kC, AGG>, dim3(grid), dim3(kScanThreads), smem, s, tm,
                             B, T, d, gate, h, static_cast<TE*>(oprime), prof_on ? dprof : nullptr,
                             agg);
  if (e != cudaSuccess || !prof_on || grid > 4096) return e;
  static unsigned long long hp[8 * 4096];
  cudaMemcpyAsync(hp, dprof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  double sum[8] = {0};
  for (int b = 0; b < grid; ++b)
    for (int i = 0; i < 8; ++i) sum[i] += (double)hp[b * 8 + i] / grid;
  fprintf(stderr,
          "[scan prof] B=%d T=%d d=%d kC=%d kS=%d grid=%d | per CTA cycles: prod.empty=%.0f "
          "carry.wait=%.0f carry.total=%.0f gate.full=%.0f phase1=%.0f gate.scanned=%.0f "
          "phase3=%.0f gate.total=%.0f\n",
          B, T, d, kC, kS, grid, sum[0], sum[1], sum[2], sum[3], sum[4], sum[5], sum[6], sum[7]);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- chunked scan (num_chunks > 1)
// Few long sequences (B * d / 8 CTAs do not fill the SMs, e.g. B = 1): the recurrence of
// every channel is cut into NCH = 4 contiguous time chunks [j T / 4, (j+1) T / 4) that run
// CONCURRENTLY on the 32 lanes of the carry warp (lane = chunk * 8 + channel), so each lane
// walks a quarter of the sequence ("the linear recurrence ... allows a parallel
// scan"; reading C23 fixes the composition):
//   pass A  the carry runs each chunk from h = 0 and the running product of f: the chunk
//           aggregate (A_j, B_j) with A = A f, B = f B + b (left to right);
//   compose h_in(0) = h, h_in(j+1) = A_j h_in(j) + B_j over the chunks in order (shuffles
//           within the carry warp); the state after the sequence is h_in(4);
//   pass B  the exact sequential scan of each chunk from h_in(j), with the gates' output
//           o' = g sigma(h) (or g h) -- bit-identical to the oracle's O.scan_slices(4).
// A pipeline stage holds one round: time tile r (128 steps x 8 channels) of all 4 chunks;
// the gates compute (f, (1-f) SiLU(c)) of a round in both passes (5 sigmoids per element
// in total instead of 3: the carry chain, not the gate arithmetic, bounds a CTA here).
constexpr int kChN = 4;            // chunks
constexpr int kChC = 8;            // channels per CTA
constexpr int kChTS = kTE / kChC;  // 128 steps per tile
constexpr int kChS = 2;            // ring stages (rounds)

template <typename T>
struct ChunkSmem {
  T in[kChS][kChN][3][kTE];                 // f^, c^, g^ boxes [kChTS][kChC] per chunk
  __align__(16) float fb[kChS][kChN][2 * kTE];
  __align__(16) float hs[kChS][kChN][kTE];
  uint64_t full[kChS], gated[kChS], scanned[kChS], empty[kChS];
};

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_chunked(const __grid_constant__ CUtensorMap tmX,
                                                               int B, int T_, int d, int gate,
                                                               float* __restrict__ h,
                                                               T* __restrict__ oprime) {
  extern __shared__ __align__(128) uint8_t scan_smem[];
  ChunkSmem<T>& sm = *reinterpret_cast<ChunkSmem<T>*>(scan_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpb = d / kChC;
  const int b = blockIdx.x / cpb;
  const int c0 = (blockIdx.x % cpb) * kChC;
  const int colf = (c0 / kSegRows) * (3 * kSegRows) + (c0 % kSegRows);
  // chunk j = steps [t0(j), t0(j+1)); rounds per pass = tiles of the longest chunk
  auto t0 = [&](int j) { return (int)((int64_t)j * T_ / kChN); };
  const int R = (t0(1) - t0(0) > t0(kChN) - t0(kChN - 1) ? t0(1) - t0(0) : t0(kChN) - t0(kChN - 1)) +
                kChTS - 1;
  const int nr = R / kChTS;          // rounds per pass
  const int n_seq = 2 * nr;          // pass A rounds, then pass B rounds
  auto steps_of = [&](int j, int r) {   // valid steps of chunk j's tile r
    const int left = t0(j + 1) - t0(j) - r * kChTS;
    return left < 0 ? 0 : (left > kChTS ? kChTS : left);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kChS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.gated[s], kGateWarps);
      mbar_init(&sm.scanned[s], 1);
      mbar_init(&sm.empty[s], kGateWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------- producer: one round = the r-th tile of every chunk (pass A: f^, c^;
    // pass B: f^, c^, g^); tiles past a chunk's end are not loaded
    if (lane == 0) {
      tma_prefetch_desc(&tmX);
      for (int i = 0; i < n_seq; ++i) {
        const int s = i % kChS, r = i % nr;
        const bool passB = i >= nr;
        if (i >= kChS) mbar_wait(&sm.empty[s], ((i / kChS) - 1) & 1);
        const int nbox = passB ? 3 : 2;
        int ntile = 0;
        for (int j = 0; j < kChN; ++j) ntile += steps_of(j, r) > 0;
        mbar_arrive_expect_tx(&sm.full[s], (uint32_t)(ntile * nbox * kTE * sizeof(T)));
        for (int j = 0; j < kChN; ++j) {
          if (steps_of(j, r) == 0) continue;
          const int row = b * T_ + t0(j) + r * kChTS;
          for (int g = 0; g < nbox; ++g)
            tma_load_2d(&sm.in[s][j][g][0], &tmX, &sm.full[s], colf + g * kSegRows, row);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- the carry: lane = chunk j * 8 + channel c
    const int j = lane / kChC, c = lane % kChC;
    float hc = 0.0f, Ac = 1.0f;
    for (int i = 0; i < n_seq; ++i) {
      const int s = i % kChS, r = i % nr;
      const bool passB = i >= nr;
      if (i == nr) {
        // compose the chunk aggregates in chunk order (reading C23): h_in(j) for this lane,
        // and the state after the whole sequence
        float hin = h[(int64_t)b * d + c0 + c], mine = hin;
#pragma unroll
        for (int k = 0; k < kChN; ++k) {
          const float A = __shfl_sync(0xffffffffu, Ac, k * kChC + c);
          const float Bv = __shfl_sync(0xffffffffu, hc, k * kChC + c);
          if (k == j) mine = hin;
          hin = __fadd_rn(__fmul_rn(A, hin), Bv);
        }
        if (j == 0) h[(int64_t)b * d + c0 + c] = hin;
        hc = mine;
      }
      mbar_wait(&sm.gated[s], (i / kChS) & 1);
      const int steps = steps_of(j, r);
      const float4* __restrict__ fb4 = reinterpret_cast<const float4*>(sm.fb[s][j]) + c;
      float4* __restrict__ hs4 = reinterpret_cast<float4*>(sm.hs[s][j]) + c;
      if (__all_sync(0xffffffffu, steps == kChTS)) {
        constexpr int kG = kChTS / 4;   // groups of 4 steps; (f, b) loaded 2 groups ahead
        float4 pf[kG], qf[kG];
        pf[0] = fb4[0], qf[0] = fb4[kChC];
        pf[1] = fb4[2 * kChC], qf[1] = fb4[3 * kChC];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          if (g + 2 < kG) pf[g + 2] = fb4[(2 * g + 4) * kChC], qf[g + 2] = fb4[(2 * g + 5) * kChC];
          const float4 p = pf[g], q = qf[g];
          float4 o;
          o.x = __fadd_rn(__fmul_rn(p.x, hc), p.y);
          o.y = __fadd_rn(__fmul_rn(p.z, o.x), p.w);
          o.z = __fadd_rn(__fmul_rn(q.x, o.y), q.y);
          o.w = __fadd_rn(__fmul_rn(q.z, o.z), q.w);
          if (passB) hs4[g * kChC] = o;
          else Ac = __fmul_rn(__fmul_rn(__fmul_rn(__fmul_rn(Ac, p.x), p.z), q.x), q.z);
          hc = o.w;
        }
      } else {
        for (int t = 0; t < steps; ++t) {
          const int e = t * kChC + c;
          const float* fbw = &sm.fb[s][j][fb_word<kChC>(e)];
          hc = __fadd_rn(__fmul_rn(fbw[0], hc), fbw[1]);
          if (passB) sm.hs[s][j][h_word<kChC>(e)] = hc;
          else Ac = __fmul_rn(Ac, fbw[0]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.scanned[s]);
    }
  } else if (gate_warp_index(warp) >= 0) {
    // ---------------- gate warps: element e = (gw*4 + k)*32 + lane of each chunk's tile
    const int gw = gate_warp_index(warp);
    const int cl = lane % kChC;
    T* obase = oprime + (int64_t)b * T_ * d + c0 + cl;
    auto phase1 = [&](int i) {   // (f, (1-f) SiLU(c)) of round i
      const int s = i % kChS, r = i % nr;
      mbar_wait(&sm.full[s], (i / kChS) & 1);
#pragma unroll 1
      for (int j = 0; j < kChN; ++j) {
        if (steps_of(j, r) == 0) continue;
        float fv[kElemsPerLane], bvv[kElemsPerLane];
#pragma unroll
        for (int k = 0; k < kElemsPerLane; ++k) {
          const int e = (gw * kElemsPerLane + k) * 32 + lane;
          const float fx = ld_act<T>(&sm.in[s][j][0][e]);
          const float cx = ld_act<T>(&sm.in[s][j][1][e]);
          float f, sc;
          sigmoid2(fx, cx, f, sc);
          fv[k] = f;
          bvv[k] = __fmul_rn(__fsub_rn(1.0f, f), __fmul_rn(cx, sc));   // (1-f) SiLU(c)
        }
#pragma unroll
        for (int k = 0; k < kElemsPerLane; ++k) {
          const int e = (gw * kElemsPerLane + k) * 32 + lane;
          *reinterpret_cast<float2*>(&sm.fb[s][j][fb_word<kChC>(e)]) = make_float2(fv[k], bvv[k]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.gated[s]);
    };
    auto phase3 = [&](int i) {   // pass B: o' = g sigma(h) or g h, valid steps only
      const int s = i % kChS, r = i % nr;
      mbar_wait(&sm.scanned[s], (i / kChS) & 1);
      if (i >= nr) {
        const bool sig = gate == TERN_GATE_SIGMOID_H;
#pragma unroll 1
        for (int j = 0; j < kChN; ++j) {
          const int steps = steps_of(j, r);
          if (steps == 0) continue;
          float ov[kElemsPerLane];
#pragma unroll
          for (int k = 0; k < kElemsPerLane; k += 2) {
            const int e = (gw * kElemsPerLane + k) * 32 + lane;
            const float g0 = ld_act<T>(&sm.in[s][j][2][e]), g1 = ld_act<T>(&sm.in[s][j][2][e + 32]);
            const float h0 = sm.hs[s][j][h_word<kChC>(e)], h1 = sm.hs[s][j][h_word<kChC>(e + 32)];
            if (sig) {
              float s0, s1;
              sigmoid2(h0, h1, s0, s1);
              ov[k] = __fmul_rn(g0, s0);
              ov[k + 1] = __fmul_rn(g1, s1);
            } else {
              ov[k] = __fmul_rn(g0, h0);
              ov[k + 1] = __fmul_rn(g1, h1);
            }
          }
#pragma unroll
          for (int k = 0; k < kElemsPerLane; ++k) {
            const int tl = ((gw * kElemsPerLane + k) * 32 + lane) / kChC;
            if (tl < steps) st_act<T>(obase + (int64_t)(t0(j) + r * kChTS + tl) * d, ov[k]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    };
    // phase 1 of round i runs before phase 3 of round i-1, so the carry finds a gated round
    // while the gates wait for its previous one (2 stages: round i+1 refills the stage that
    // phase 3 of round i-1 released)
    for (int i = 0; i < n_seq; ++i) {
      phase1(i);
      if (i >= 1) phase3(i - 1);
    }
    if (n_seq > 0) phase3(n_seq - 1);
  }
}

template <typename TE>
static cudaError_t scan_chunked_go(const void* fcg, int B, int T, int d, int gate, float* h,
                                   void* oprime, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = sizeof(ChunkSmem<TE>);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_scan_chunked<TE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const bool bf = sizeof(TE) == 2;
  CUtensorMap tm;
  if (!make_map_2d(&tm, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, fcg,
                   (uint64_t)3 * d, (uint64_t)B * T, (uint64_t)3 * d * sizeof(TE), kChC, kChTS,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  return launch_pdl(k_scan_chunked<TE>, dim3(B * (d / kChC)), dim3(kScanThreads), smem, s, tm, B, T, d,
                    gate, h, static_cast<TE*>(oprime));
}

static int scan_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int env_knob(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Channel width: 8 (measured best at every c2 batch: the gate arithmetic
// of a CTA is latency-bound, so 4x more, narrower CTAs win even when 32-wide ones fill
// the SMs); TERN_SCAN_KC overrides with 16 or 32.  Ring depth: deep when the grid leaves
// SMs idle (one CTA per SM then streams alone).
template <typename TE>
static cudaError_t scan_pick(const void* fcg, int B, int T, int d, int gate, float* h,
                            void* oprime, cudaStream_t s) {
  static const int kc_env = env_knob("TERN_SCAN_KC", 8);
  static const int deep_env = env_knob("TERN_SCAN_DEEP", 2);  // 0 never, 1 always, 2 auto
  const int sms = scan_num_sms();
  int kc = (kc_env == 16 || kc_env == 32) ? kc_env : 8;
  if (d % kc) kc = 8;
  const bool deep = deep_env == 1 || (deep_env == 2 && (int64_t)B * (d / kc) < sms);
#define TERN_SCAN_GO(S, C) scan_go<TE, S, C>(fcg, B, T, d, gate, h, oprime, s)
  if (deep) {
    if (kc == 8) return TERN_SCAN_GO(kSDeep, 8);
    if (kc == 16) return TERN_SCAN_GO(kSDeep, 16);
    return TERN_SCAN_GO(kSDeep, 32);
  }
  if (kc == 8) return TERN_SCAN_GO(kSShallow, 8);
  if (kc == 16) return TERN_SCAN_GO(kSShallow, 16);
  return TERN_SCAN_GO(kSShallow, 32);
#undef TERN_SCAN_GO
}

// num_chunks (tern_mlgru.num_chunks): 1 = the exact sequential scan; 4 = the chunked scan
// (reading C23); 0 = auto = 1: the chunked kernel measured SLOWER than the sequential one at
// every few-sequence shape (c2 B = 1 x 2048: 33.3 vs 21.2 us; c3 61.9 vs 31.2; c4 B = 1 x 4096:
// 180.7 vs 75.8 us, tools/scan_chunk_bench.py) -- the sequential kernel is bound by its gate
// arithmetic and pipeline, not by the carry chain, and the chunked one computes the gates of
// f and c twice (5 sigmoids per element instead of 3)
// ---------------------------------------------------------------- cross-CTA chunked scan
// num_chunks = 4 for few long sequences: the 4 slices [j T / 4, (j+1) T / 4) of a 32-channel
// group run on the 4 CTAs of one thread-block cluster (rank = slice j), so every slice has
// an SM of its own (4x the SMs of the in-CTA layout below; one CTA per SM keeps each carry
// warp's sub-partition free of other carries), and the boundary state crosses the
// cluster through distributed shared memory (reading C23):
//   pass A  gates f = sigma(f^), b = (1-f) SiLU(c^) for the whole slice into shared memory
//           (16 warps; g^ staged too), then the carry warp (lane = channel) runs the slice
//           aggregate A = A f, B = f B + b from (1, 0), left to right;
//   hop     slice j waits for h_in(j) from rank j-1 (slice 0: the state h) and sends
//           h_in(j+1) = A h_in(j) + B to rank j+1 (st.async into its shared memory,
//           completing on its mbarrier); the last slice writes the final state to h;
//   pass B  the carry scans the slice from h_in(j) over the stored (f, b), then all warps
//           form o' = g^ sigma(h) (or g^ h).
// Every operation and its order is O.scan_slices(4)'s, so the result is bit-identical to it.
constexpr int kLBC = 32;           // channels per CTA (lane = channel in the carry)
constexpr int kLBThreads = 512;    // warp 0 the carry; gates / output on the warps of
                                   // sub-partitions 1-3 (warp % 4 != 0: 12 warps), so the
                                   // carry's dependent chain has sub-partition 0 to itself
constexpr int kLBTS = 64;          // steps per pipeline tile
constexpr int kLBMaxT = 8;         // tiles per slice held in shared memory
constexpr int kLBMaxL = kLBTS * kLBMaxT;
constexpr int kLBGate = 12 * 32;   // gate / output threads

__device__ __forceinline__ uint32_t lb_mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void lb_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// shared memory (rows = steps of the slice, 32 channels each): raw f^ c^ g^ TA [3][512][32]
// (TMA, every tile issued up front), then f, b fp32 [2][512][32] (the raw f^ c^ arrays
// themselves when TA is fp32: converted in place, each element by the thread that reads it)
// (rows = the longest slice rounded up to whole tiles)
template <typename TA>
__host__ __device__ constexpr size_t lb_smem_bytes(int rows) {
  return (size_t)3 * rows * kLBC * sizeof(TA) +
         (sizeof(TA) == 4 ? 0 : (size_t)2 * rows * kLBC * sizeof(float)) + 128;
}

template <typename TA>
__global__ void __launch_bounds__(kLBThreads, 1) k_scan_lb(const __grid_constant__ CUtensorMap tmX,
                                                           int B, int T, int d, int nch, int rows,
                                                           int gate, float* h, TA* oprime,
                                                           unsigned long long* tl) {
  extern __shared__ __align__(128) float lbs[];
  __shared__ __align__(8) uint64_t full[kLBMaxT], gated[kLBMaxT], hdone[kLBMaxT], gbar, hbar;
  __shared__ __align__(16) float hin_s[kLBC];
  const int G = d / kLBC;
  const int j = blockIdx.x % nch, rem = blockIdx.x / nch, b = rem / G, cg = rem % G;
  const int s0 = (int)((int64_t)j * T / nch), s1 = (int)((int64_t)(j + 1) * T / nch);
  const int L = s1 - s0, nt = (L + kLBTS - 1) / kLBTS;
  const int kArr = rows * kLBC;
  TA* rf = reinterpret_cast<TA*>(lbs);            // raw f^, c^, g^
  TA* rc = rf + kArr;
  TA* rg = rc + kArr;
  float* F = sizeof(TA) == 4 ? reinterpret_cast<float*>(rf) : reinterpret_cast<float*>(rg + kArr);
  float* Bv = sizeof(TA) == 4 ? reinterpret_cast<float*>(rc) : F + kArr;   // f -> h, b
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = cg * kLBC;
  const int row0 = b * T + s0;                    // first row of the slice in [B*T][3d]
  const int colf = packed_row(0, c0, 3), colc = packed_row(1, c0, 3), colg = packed_row(2, c0, 3);
  constexpr uint32_t kTileBytes = kLBTS * kLBC * sizeof(TA);
  auto mark = [&](int k) {   // debug timeline (TERN_LB_TL): globaltimer per CTA and phase
    if (tl && threadIdx.x == 0) tl[(size_t)blockIdx.x * 8 + k] = gtimer();
  };
  mark(6);
  if (tid == 0) {
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < kLBMaxT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&gated[i], kLBGate / 32);
      mbar_init(&hdone[i], 1);
    }
    mbar_init(&gbar, 1);
    mbar_init(&hbar, 1);
    fence_barrier_init();
    if (j > 0) mbar_arrive_expect_tx(&hbar, kLBC * sizeof(float));
  }
  lb_cluster_sync();          // every rank's barriers armed before any st.async
  pdl_wait();                 // f^c^g^ and h come from earlier kernels
  pdl_launch_dependents();
  mark(0);
  if (tid == 32) {            // the whole slice in flight at once: f^ c^ per tile, then g^
    for (int k = 0; k < nt; ++k) {
      mbar_arrive_expect_tx(&full[k], 2 * kTileBytes);
      tma_load_2d(rf + k * kLBTS * kLBC, &tmX, &full[k], colf, row0 + k * kLBTS);
      tma_load_2d(rc + k * kLBTS * kLBC, &tmX, &full[k], colc, row0 + k * kLBTS);
    }
    if (nt > 0) {
      mbar_arrive_expect_tx(&gbar, nt * kTileBytes);
      for (int k = 0; k < nt; ++k)
        tma_load_2d(rg + k * kLBTS * kLBC, &tmX, &gbar, colg, row0 + k * kLBTS);
    }
  }
  if (warp == 0) {
    // ---- pass A carry, tile by tile behind the gates: the aggregate from (A, B) = (1, 0)
    float A = 1.0f, Bs = 0.0f;
    for (int k = 0; k < nt; ++k) {
      mbar_wait(&gated[k], 0);
      const int st1 = min(L, (k + 1) * kLBTS);
      int st = k * kLBTS;
      // groups of 8 steps, the next group's loads issued before this group's chain
      float fv[8], bv[8];
      if (st + 8 <= st1) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          fv[u] = F[(st + u) * kLBC + lane];
          bv[u] = Bv[(st + u) * kLBC + lane];
        }
      }
      for (; st + 8 <= st1; st += 8) {
        float fn[8], bn[8];
        const bool more = st + 16 <= st1;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          fn[u] = more ? F[(st + 8 + u) * kLBC + lane] : 0.0f;
          bn[u] = more ? Bv[(st + 8 + u) * kLBC + lane] : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          A = __fmul_rn(A, fv[u]);
          Bs = __fadd_rn(__fmul_rn(fv[u], Bs), bv[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          fv[u] = fn[u];
          bv[u] = bn[u];
        }
      }
      for (; st < st1; ++st) {
        const float fv = F[st * kLBC + lane];
        A = __fmul_rn(A, fv);
        Bs = __fadd_rn(__fmul_rn(fv, Bs), Bv[st * kLBC + lane]);
      }
    }
    mark(1);
    // ---- hop: h_in(j) from rank j-1 (or the state), h_in(j+1) to rank j+1 (or the state)
    const int64_t hi = (int64_t)b * d + c0 + lane;
    float hin;
    if (j == 0) {
      hin = __ldcg(h + hi);
    } else {
      mbar_wait(&hbar, 0);
      hin = hin_s[lane];
    }
    const float hout = __fadd_rn(__fmul_rn(A, hin), Bs);
    if (j + 1 < nch) {
      const uint32_t dst = lb_mapa(&hin_s[lane], (uint32_t)(j + 1));
      const uint32_t bar = lb_mapa(&hbar, (uint32_t)(j + 1));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
                   "r"(__float_as_uint(hout)), "r"(bar)
                   : "memory");
    } else {
      h[hi] = hout;   // the state after the sequence: the composition through every slice
    }
    mark(2);
    // ---- pass B carry: the exact scan of the slice from h_in(j), h over f in place, the
    // output gate following tile by tile
    float hh = hin;
    for (int k = 0; k < nt; ++k) {
      const int st1 = min(L, (k + 1) * kLBTS);
      int st = k * kLBTS;
      float fv[8], bv[8];
      if (st + 8 <= st1) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          fv[u] = F[(st + u) * kLBC + lane];
          bv[u] = Bv[(st + u) * kLBC + lane];
        }
      }
      for (; st + 8 <= st1; st += 8) {
        float fn[8], bn[8], hv[8];
        const bool more = st + 16 <= st1;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          fn[u] = more ? F[(st + 8 + u) * kLBC + lane] : 0.0f;
          bn[u] = more ? Bv[(st + 8 + u) * kLBC + lane] : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          hh = __fadd_rn(__fmul_rn(fv[u], hh), bv[u]);
          hv[u] = hh;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          F[(st + u) * kLBC + lane] = hv[u];
          fv[u] = fn[u];
          bv[u] = bn[u];
        }
      }
      for (; st < st1; ++st) {
        hh = __fadd_rn(__fmul_rn(F[st * kLBC + lane], hh), Bv[st * kLBC + lane]);
        F[st * kLBC + lane] = hh;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&hdone[k]);
    }
    mark(3);
  } else if (warp & 3) {
    // ---- gates (12 warps): tile k's f = sigma(f^), b = (1-f) SiLU(c^), in place
    const int gt = (warp - 1 - (warp >> 2)) * 32 + lane;   // 0 .. 383
    for (int k = 0; k < nt; ++k) {
      mbar_wait(&full[k], 0);
      const int e0 = k * kLBTS * kLBC, e1 = min(L, (k + 1) * kLBTS) * kLBC;
      for (int e = e0 + gt; e < e1; e += kLBGate) {
        const float fh = ld_act<TA>(rf + e), ch = ld_act<TA>(rc + e);
        float f, sc;
        sigmoid2(fh, ch, f, sc);
        F[e] = f;
        Bv[e] = __fmul_rn(__fsub_rn(1.0f, f), __fmul_rn(ch, sc));   // (1-f) SiLU(c)
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&gated[k]);
    }
    // ---- output gate, tile by tile behind the carry (a warp stores one step's 32 channels)
    if (nt > 0) mbar_wait(&gbar, 0);
    TA* obase = oprime + (int64_t)row0 * d + c0 + lane;
    const bool sig = gate == TERN_GATE_SIGMOID_H;
    for (int k = 0; k < nt; ++k) {
      mbar_wait(&hdone[k], 0);
      const int e0 = k * kLBTS * kLBC, e1 = min(L, (k + 1) * kLBTS) * kLBC;
      int e = e0 + gt;
      if (sig) {
        for (; e + kLBGate < e1; e += 2 * kLBGate) {
          float q0, q1;
          sigmoid2(F[e], F[e + kLBGate], q0, q1);
          st_act<TA>(obase + (int64_t)(e >> 5) * d, __fmul_rn(ld_act<TA>(rg + e), q0));
          st_act<TA>(obase + (int64_t)((e + kLBGate) >> 5) * d,
                     __fmul_rn(ld_act<TA>(rg + e + kLBGate), q1));
        }
        if (e < e1) {
          float q0, q1;
          sigmoid2(F[e], F[e], q0, q1);
          st_act<TA>(obase + (int64_t)(e >> 5) * d, __fmul_rn(ld_act<TA>(rg + e), q0));
        }
      } else {
        for (; e < e1; e += kLBGate)
          st_act<TA>(obase + (int64_t)(e >> 5) * d, __fmul_rn(ld_act<TA>(rg + e), F[e]));
      }
    }
  }
  mark(5);
  lb_cluster_sync();          // no rank leaves while a peer's st.async may target it
}

static bool lb_ok(int nch, int T, int d) {
  return d % kLBC == 0 && (T + nch - 1) / nch <= kLBMaxL;
}

template <typename TA>
static cudaError_t scan_lb_go(const void* fcg, int B, int T, int d, int nch, int gate, float* h,
                              void* oprime, cudaStream_t s) {
  const int rows = ((T + nch - 1) / nch + kLBTS - 1) / kLBTS * kLBTS;
  const size_t smem = lb_smem_bytes<TA>(rows);
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    e = cudaFuncSetAttribute(k_scan_lb<TA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lb_smem_bytes<TA>(kLBMaxL));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const bool bf = std::is_same<TA, __nv_bfloat16>::value;
  CUtensorMap tm;
  if (!make_map_2d(&tm, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, fcg,
                   (uint64_t)3 * d, (uint64_t)B * T, (uint64_t)3 * d * sizeof(TA), kLBC, kLBTS,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  const int grid = nch * B * (d / kLBC);
  static const char* tl_path = getenv("TERN_LB_TL");   // debug: per-CTA phase timeline
  static unsigned long long* dtl = nullptr;
  if (tl_path && !dtl) cudaMalloc(&dtl, sizeof(unsigned long long) * 8 * 65536);
  unsigned long long* tl = (tl_path && grid <= 65536) ? dtl : nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kLBThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;   // the slices of one channel group
  at[0].val.clusterDim.x = nch;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, k_scan_lb<TA>, tm, B, T, d, nch, rows, gate, h,
                         static_cast<TA*>(oprime), tl);
  if (e == cudaSuccess && tl) {
    static unsigned long long hbuf[8 * 65536];
    cudaMemcpyAsync(hbuf, tl, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    FILE* f = fopen(tl_path, "a");
    if (f) {
      fprintf(f, "launch B=%d T=%d d=%d nch=%d grid=%d\n", B, T, d, nch, grid);
      for (int i = 0; i < grid; ++i)
        fprintf(f, "%llu %llu %llu %llu %llu %llu %llu\n", hbuf[i * 8], hbuf[i * 8 + 1],
                hbuf[i * 8 + 2], hbuf[i * 8 + 3], hbuf[i * 8 + 4], hbuf[i * 8 + 5], hbuf[i * 8 + 6]);
      fclose(f);
    }
  }
  return e;
}

int scan_chunks_resolve(int num_chunks, int B, int T, int d) {
  (void)B;
  if (num_chunks == kChN && d % kChC == 0) return kChN;   // cluster kernel or the in-CTA one
  if (num_chunks == 8 && lb_ok(8, T, d)) return 8;       // cluster kernel only
  return 1;
}

cudaError_t launch_scan_chunks(const void* fcg, int dt, int B, int T, int d, int gate, float* h,
                               void* oprime, int chunks, cudaStream_t s) {
  if (B == 0 || T == 0) return cudaSuccess;
  static const int lb_on = getenv("TERN_SCAN_LB") ? atoi(getenv("TERN_SCAN_LB")) : 1;   // debug
  if ((chunks == kChN && lb_on && lb_ok(chunks, T, d)) || chunks == 8)
    return dt == TERN_BF16 ? scan_lb_go<__nv_bfloat16>(fcg, B, T, d, chunks, gate, h, oprime, s)
                           : scan_lb_go<float>(fcg, B, T, d, chunks, gate, h, oprime, s);
  if (chunks == kChN)
    return dt == TERN_BF16 ? scan_chunked_go<__nv_bfloat16>(fcg, B, T, d, gate, h, oprime, s)
                           : scan_chunked_go<float>(fcg, B, T, d, gate, h, oprime, s);
  return launch_scan(fcg, dt, B, T, d, gate, h, oprime, s);
}

cudaError_t launch_scan(const void* fcg, int dt, int B, int T, int d, int gate, float* h,
                        void* oprime, cudaStream_t s) {
  if (B == 0 || T == 0) return cudaSuccess;
  return dt == TERN_BF16 ? scan_pick<__nv_bfloat16>(fcg, B, T, d, gate, h, oprime, s)
                         : scan_pick<float>(fcg, B, T, d, gate, h, oprime, s);
}

// Sequence-parallel pass 1 (C23): the slice aggregates (A, B) of every (sequence, channel)
cudaError_t launch_scan_agg(const void* fcg, int dt, int B, int T, int d, float* agg,
                            cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  if (T == 0) {   // empty slice: the identity (A, B) = (1, 0)
    cudaError_t e = cudaMemsetAsync(agg + (size_t)B * d, 0, sizeof(float) * B * d, s);
    if (e != cudaSuccess) return e;
    return launch_fill_f32(agg, (size_t)B * d, 1.0f, s);
  }
  const bool deep = (int64_t)B * (d / 8) < scan_num_sms();
  if (dt == TERN_BF16)
    return deep ? scan_go<__nv_bfloat16, kSDeep, 8, true>(fcg, B, T, d, 0, nullptr, nullptr, s, agg)
                : scan_go<__nv_bfloat16, kSShallow, 8, true>(fcg, B, T, d, 0, nullptr, nullptr, s,
                                                             agg);
  return deep ? scan_go<float, kSDeep, 8, true>(fcg, B, T, d, 0, nullptr, nullptr, s, agg)
              : scan_go<float, kSShallow, 8, true>(fcg, B, T, d, 0, nullptr, nullptr, s, agg);
}

// Sequence-parallel composition (C23): recv [world][2][B][d] holds every rank's slice
// aggregate in rank order; h (in: the state before the sequence) becomes this rank's
// boundary state h_in(rank), hfin the state after the whole sequence h_in(world).
__global__ void k_sp_compose(const float* __restrict__ recv, int world, int rank, int64_t n,
                             float* __restrict__ h, float* __restrict__ hfin) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float hin = h[i], mine = hin;
    for (int j = 0; j < world; ++j) {
      if (j == rank) mine = hin;
      const float A = recv[(int64_t)j * 2 * n + i], Bv = recv[(int64_t)j * 2 * n + n + i];
      hin = __fadd_rn(__fmul_rn(A, hin), Bv);
    }
    h[i] = mine;
    hfin[i] = hin;
  }
}

cudaError_t launch_sp_compose(const float* recv, int world, int rank, int64_t n, float* h,
                              float* hfin, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  k_sp_compose<<<grid, 256, 0, s>>>(recv, world, rank, n, h, hfin);
  return cudaGetLastError();
}

__global__ void k_fill_f32(float* p, size_t n, float v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}
cudaError_t launch_fill_f32(float* p, size_t n, float v, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_fill_f32<<<(unsigned)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184), 256, 0, s>>>(p, n, v);
  return cudaGetLastError();
}

}  // namespace tern
