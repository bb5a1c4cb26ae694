// k_fcgscan.cu -- a4 + a6 fused for prefill: the f|c|g BitLinear GEMM
// (tcgen05.mma kind::i8, accumulators in TMEM) with the MLGRU gates, the exact
// sequential recurrence and the output gate in its epilogue (
// PAPER.md P:446-456).  The f^c^g^ pre-activations never touch HBM.
//
// Work unit = a chain: one sequence b x one 64-channel group (packed rows
// [192 g, 192 g + 192) = 64 f | 64 c | 64 g).
// A CTA walks its chain's 128-token M-tiles in time order, carrying h in the
// registers of the carry threads:
//   warp 0      TMA producer: A (int8 q rows of the tile) + B (u8 fields of the
//               group's 192 rows) per 128-wide K-block, 3-stage ring
//   warp 1      TMEM alloc + single-thread tcgen05.mma (M=128, N=192), two
//               accumulators so tile i+1's MMAs overlap tile i's epilogue
//   warps 2-9   gate warps, one per (TMEM lane quadrant q, channel half):
//               (A) thread = token row: tcgen05.ld f^,c^,g^ -> dequant (a5) ->
//               f = sigma(f^), b = (1-f) SiLU(c^), g^ -> smem, TMEM released;
//               (C) once the carry passed its 32 rows, lane = channel:
//               o' = g^ sigma(h) (or g^ h) -> global, coalesced
//   warps 10-11 carry warps (channel halves): h = f h + b over the tile's
//               rows in order, quad by quad as the gate warps deliver them
//               (bit-identical to the definition)
// mbarriers per (quad, half) pipeline the three phases across quads and
// tiles, so the serial carry overlaps the transcendental work.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "epilogue.cuh"

namespace tern {

constexpr int kFBM = 128;                 // tokens per M-tile
constexpr int kFBK = 128;                 // K-block (bytes)
constexpr int kFCW = 64;                  // channels per chain
constexpr int kFBN = 3 * kFCW;            // packed rows per chain (f|c|g)
constexpr int kFS = 3;                    // ring stages
constexpr int kFEpiWarps = 16;           // gate warps: 4 per TMEM lane quadrant
constexpr int kFThreads = (4 + kFEpiWarps) * 32;   // producer, MMA, gate warps, 2 carry
constexpr int kFQCh = kFCW / 4;          // channels per gate warp (16)
constexpr int kFPad = kFCW + 1;           // smem row stride (floats): conflict-free both ways

struct FcgScanArgs {
  int B, T, d, M, num_kb, n_rows;
  const float* deq;
  const int32_t* qsum;
  const float* scales;   // [3] f, c, g
  const float* bias;     // [3][d] or null
  float* h;              // [B][d]
  void* oprime;          // [B*T][d]
  int gate;
  int backoff;               // gate warps' wait for the carry: first sleep (ns), 0 = hinted wait
  unsigned long long* prof;  // debug (TERN_FS_PROF): [grid][8] cycles per wait site / phase
  unsigned long long* trace;   // tern_trace_enable timeline
  int nogate;                  // debug (TERN_FS_NOGATE=1): skip the gate / carry arithmetic
  unsigned long long* tl;      // debug (TERN_FS_TL=file): CTA 0 per-warp phase clocks [20][nt][8]
};

__device__ __forceinline__ void fs_tl(const FcgScanArgs& a, int warp, int i, int k) {
  if (a.tl && blockIdx.x == 0 && (threadIdx.x & 31) == 0)
    a.tl[((size_t)warp * ((a.T + 127) / 128) + i) * 8 + k] = clock64();
}

// debug: add the cycles since t0 to counter `site` of this CTA
__device__ __forceinline__ void fs_acc(const FcgScanArgs& a, int site, long long t0) {
  if (a.prof) atomicAdd(a.prof + blockIdx.x * 8 + site, (unsigned long long)(clock64() - t0));
}

struct FcgScanSmem {
  uint8_t a[kFS][kFBM * kFBK];       // 16 KB per stage (SW128)
  uint8_t b[kFS][kFBN * kFBK];       // 24 KB per stage (SW128)
  float F[kFBM][kFPad];              // f, then h
  float Bv[kFBM][kFPad];             // (1-f) SiLU(c)
  float G[kFBM][kFPad];              // g^
  uint64_t full[kFS], empty[kFS], tfull[2], tempty[2];
  uint64_t ready[4][2];              // both gate warps of (quad, half) wrote their f, b, g^
  uint64_t hdone[4][2];              // carry warp (half) finished the quad's rows
  uint64_t tmem_free;                // every gate warp is done with TMEM
  uint32_t tmem_slot;
};

__device__ __forceinline__ void epi_bar() {   // named barrier over the 8 epilogue warps
  asm volatile("bar.sync 1, %0;" ::"n"(kFEpiWarps * 32) : "memory");
}

template <typename TY>
__global__ void __launch_bounds__(kFThreads, 1)
    k_fcgscan(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const FcgScanArgs a) {
  extern __shared__ __align__(1024) uint8_t fs_raw[];
  FcgScanSmem& sm =
      *reinterpret_cast<FcgScanSmem*>(fs_raw + ((1024u - (smem_u32(fs_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = a.d / kFCW;
  const int chains = a.B * groups;
  const int nt = (a.T + kFBM - 1) / kFBM;   // M-tiles per chain
  trace_mark(a.trace, 0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kFS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], kFEpiWarps);
    }
    for (int q = 0; q < 4; ++q)
      for (int h = 0; h < 2; ++h) {
        mbar_init(&sm.ready[q][h], 2);   // the two 16-channel gate warps of the half
        mbar_init(&sm.hdone[q][h], 1);
      }
    mbar_init(&sm.tmem_free, kFEpiWarps);
    fence_barrier_init();
  }
  __syncwarp();
  if (warp == 1) tmem_alloc<512>(&sm.tmem_slot);
  static_assert(kFThreads <= 1024, "block size");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = sm.tmem_slot;
  pdl_wait();                 // q, deq, qsum and h come from earlier kernels
  pdl_launch_dependents();
  trace_mark(a.trace, 1);

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t g = 0;
      for (int ch = blockIdx.x; ch < chains; ch += gridDim.x) {
        const int b = ch / groups, grp = ch % groups;
        for (int i = 0; i < nt; ++i) {
          const int m0 = b * a.T + i * kFBM;
          for (int kb = 0; kb < a.num_kb; ++kb, ++g) {
            const int s = g % kFS;
            const long long w0 = clock64();
            if (g >= (uint32_t)kFS) mbar_wait(&sm.empty[s], ((g / kFS) - 1) & 1);
            fs_acc(a, 0, w0);
            mbar_arrive_expect_tx(&sm.full[s], kFBM * kFBK + kFBN * kFBK);
            tma_load_2d(sm.a[s], &tmA, &sm.full[s], kb * kFBK, m0);
            tma_load_2d(sm.b[s], &tmB, &sm.full[s], kb * kFBK, grp * kFBN);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      // kind::i8: D s32, A s8, B u8, both K-major, M=128, N=192
      const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(kFBN >> 3) << 17) |
                             ((uint32_t)(kFBM >> 4) << 24);
      uint32_t g = 0, it = 0;
      for (int ch = blockIdx.x; ch < chains; ch += gridDim.x) {
        for (int i = 0; i < nt; ++i, ++it) {
          const uint32_t acc = it & 1;
          const long long w1 = clock64();
          mbar_wait(&sm.tempty[acc], ((it >> 1) & 1) ^ 1);
          fs_acc(a, 1, w1);
          fs_tl(a, 1, i, 0);
          tc_fence_after();
          const uint32_t d_addr = tmem_base + acc * 256;
          for (int kb = 0; kb < a.num_kb; ++kb, ++g) {
            const int s = g % kFS;
            const long long w2 = clock64();
            mbar_wait(&sm.full[s], (g / kFS) & 1);
            fs_acc(a, 2, w2);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(sm.a[s]), b_addr = smem_u32(sm.b[s]);
#pragma unroll
            for (int kk = 0; kk < kFBK / 32; ++kk)
              mma_i8(d_addr, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                     idesc, (kb | kk) != 0);
            mma_commit(&sm.empty[s]);
          }
          mma_commit(&sm.tfull[acc]);
          fs_tl(a, 1, i, 1);
        }
      }
    }
  } else if (warp < 2 + kFEpiWarps) {
    // ---------------- gate warps (quad q, 16-channel slice cs): a 32-token x 16-channel block
    const int ew = warp - 2;
    const int quad = warp & 3;           // TMEM lanes [32 quad, 32 quad + 32)
    const int cs = ew >> 2;              // channels [16 cs, 16 cs + 16)
    const int half = cs >> 1;            // carry warp that consumes them
    const int r = quad * 32 + lane;      // token row of the tile (phase A)
    const float msf = __ldg(a.scales), msc = __ldg(a.scales + 1), msg = __ldg(a.scales + 2);
    uint32_t it = 0;
    for (int ch = blockIdx.x; ch < chains; ch += gridDim.x) {
      const int b = ch / groups, grp = ch % groups;
      const int c0 = grp * kFCW;         // first channel of the chain
      for (int i = 0; i < nt; ++i, ++it) {
        const uint32_t acc = it & 1;
        const int t0 = i * kFBM;
        const int steps = min(kFBM, a.T - t0);
        // (A) thread = token row: dequant, gates -> smem
        const long long w3 = clock64();
        fs_tl(a, warp, i, 0);
        mbar_wait(&sm.tfull[acc], (it >> 1) & 1);
        fs_tl(a, warp, i, 1);
        if (ew == 0 && lane == 0) fs_acc(a, 3, w3);
        const long long w4 = clock64();
        tc_fence_after();
        uint32_t vf[kFQCh], vc[kFQCh], vg[kFQCh];
        const uint32_t trow = tmem_base + acc * 256 + ((uint32_t)(quad * 32) << 16);
        tmem_ld16(trow + cs * kFQCh, vf);
        tmem_ld16(trow + kFCW + cs * kFQCh, vc);
        tmem_ld16(trow + 2 * kFCW + cs * kFQCh, vg);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[acc]);   // accumulator free for tile it+2
        const int row = b * a.T + t0 + r;
        const bool rv = r < steps;
        const float deq = rv ? __ldg(a.deq + row) : 0.0f;
        const int qs = rv ? __ldg(a.qsum + row) : 0;
        const float sf = __fmul_rn(deq, msf), sc = __fmul_rn(deq, msc), sg = __fmul_rn(deq, msg);
        const int cb = c0 + cs * kFQCh;
        // fp32: the bias test is resolved outside the unrolled channel loop (c2 block
        // 374 -> 367 us); bf16 keeps it inside (hoisting measured 2.4 % slower on c3 / c4)
        auto phase_a = [&](auto mode_c) {
          constexpr int kMode = decltype(mode_c)::value;   // 0 none, 1 bias, 2 run-time test
#pragma unroll
        for (int j = 0; j < kFQCh; j += 2) {
          float fh0 = __fmul_rn(i2f_small((int)vf[j] - qs), sf);
          float fh1 = __fmul_rn(i2f_small((int)vf[j + 1] - qs), sf);
          float ch0 = __fmul_rn(i2f_small((int)vc[j] - qs), sc);
          float ch1 = __fmul_rn(i2f_small((int)vc[j + 1] - qs), sc);
          float gh0 = __fmul_rn(i2f_small((int)vg[j] - qs), sg);
          float gh1 = __fmul_rn(i2f_small((int)vg[j + 1] - qs), sg);
          if (kMode == 1 || (kMode == 2 && a.bias)) {
            fh0 = __fadd_rn(fh0, __ldg(a.bias + cb + j));
            fh1 = __fadd_rn(fh1, __ldg(a.bias + cb + j + 1));
            ch0 = __fadd_rn(ch0, __ldg(a.bias + a.d + cb + j));
            ch1 = __fadd_rn(ch1, __ldg(a.bias + a.d + cb + j + 1));
            gh0 = __fadd_rn(gh0, __ldg(a.bias + 2 * a.d + cb + j));
            gh1 = __fadd_rn(gh1, __ldg(a.bias + 2 * a.d + cb + j + 1));
          }
          // R1: the unfused path stores these BitLinear outputs in the activation dtype
          fh0 = storage_round<TY>(fh0); fh1 = storage_round<TY>(fh1);
          ch0 = storage_round<TY>(ch0); ch1 = storage_round<TY>(ch1);
          gh0 = storage_round<TY>(gh0); gh1 = storage_round<TY>(gh1);
          float f0, f1, s0, s1;
          sigmoid2(fh0, fh1, f0, f1);
          sigmoid2(ch0, ch1, s0, s1);
          const int cc = cs * kFQCh + j;
          sm.F[r][cc] = f0;
          sm.F[r][cc + 1] = f1;
          sm.Bv[r][cc] = __fmul_rn(__fsub_rn(1.0f, f0), __fmul_rn(ch0, s0));   // (1-f) SiLU(c)
          sm.Bv[r][cc + 1] = __fmul_rn(__fsub_rn(1.0f, f1), __fmul_rn(ch1, s1));
          sm.G[r][cc] = gh0;
          sm.G[r][cc + 1] = gh1;
        }
        };
        if (a.nogate) {
        } else if constexpr (!std::is_same<TY, float>::value) phase_a(std::integral_constant<int, 2>{});
        else if (a.bias) phase_a(std::integral_constant<int, 1>{});
        else phase_a(std::integral_constant<int, 0>{});
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ready[quad][half]);   // carry may run these rows
        fs_tl(a, warp, i, 2);
        if (ew == 0 && lane == 0) fs_acc(a, 4, w4);
        // (C) 16 lanes per row, two rows 16 apart per instruction (their kFPad = 65 float
        // rows start 16 banks apart: conflict-free loads): o' = g^ sigma(h) for this
        // block's rows, after the carry
        const long long w5 = clock64();
        if (a.backoff) mbar_wait_backoff(&sm.hdone[quad][half], it & 1, a.backoff, 8 * a.backoff);
        else mbar_wait(&sm.hdone[quad][half], it & 1);
        if (ew == 0 && lane == 0) fs_acc(a, 5, w5);
        fs_tl(a, warp, i, 3);
        const long long w6 = clock64();
        const int cc = cs * kFQCh + (lane & 15), rsub = lane >> 4;
        TY* obase = static_cast<TY*>(a.oprime) + (int64_t)(b * a.T + t0) * a.d + c0 + cc;
        // full tiles and the gate mode are resolved outside the loop (no per-element
        // branch reconvergence)
        auto phase_c = [&](auto full_c, auto sig_c) {
          constexpr bool kFull = decltype(full_c)::value, kSig = decltype(sig_c)::value;
#pragma unroll 2
          for (int rr = 0; rr < 16; rr += 2) {
            const int t = quad * 32 + rr + 16 * rsub;   // rows t and t + 1
            const float h0 = sm.F[t][cc], h1 = sm.F[t + 1][cc];
            const float g0 = sm.G[t][cc], g1 = sm.G[t + 1][cc];
            float o0, o1;
            if constexpr (kSig) {
              float q0, q1;
              sigmoid2(h0, h1, q0, q1);
              o0 = __fmul_rn(g0, q0);
              o1 = __fmul_rn(g1, q1);
            } else {
              o0 = __fmul_rn(g0, h0);
              o1 = __fmul_rn(g1, h1);
            }
            if (kFull || t < steps) st_act<TY>(obase + (int64_t)t * a.d, o0);
            if (kFull || t + 1 < steps) st_act<TY>(obase + (int64_t)(t + 1) * a.d, o1);
          }
        };
        const bool sig = a.gate == TERN_GATE_SIGMOID_H;
        if (a.nogate) {
        } else if (steps == kFBM) {
          if (sig) phase_c(std::true_type{}, std::true_type{});
          else phase_c(std::true_type{}, std::false_type{});
        } else {
          if (sig) phase_c(std::false_type{}, std::true_type{});
          else phase_c(std::false_type{}, std::false_type{});
        }
        if (ew == 0 && lane == 0) fs_acc(a, 6, w6);
        fs_tl(a, warp, i, 4);
        // this block's smem rows are rewritten only by this warp's next phase A,
        // after the carry has finished with them (hdone above)
      }
    }
  } else {
    // ---------------- carry warps (channel half h): h = (f*h) + ((1-f)*c), in order
    const int half = warp - 2 - kFEpiWarps;
    const int cc = half * 32 + lane;
    uint32_t it = 0;
    for (int ch = blockIdx.x; ch < chains; ch += gridDim.x) {
      const int b = ch / groups, grp = ch % groups;
      const int c0 = grp * kFCW;
      float hc = a.h[(int64_t)b * a.d + c0 + cc];
      for (int i = 0; i < nt; ++i, ++it) {
        const int steps = min(kFBM, a.T - i * kFBM);
        for (int q = 0; q < 4; ++q) {
          mbar_wait(&sm.ready[q][half], it & 1);
          fs_tl(a, warp, i, 2 * q);
          const int tb = q * 32, te = min(tb + 32, steps);
          if (a.nogate) {
          } else if (te - tb == 32) {
#pragma unroll
            for (int t8 = 0; t8 < 32; t8 += 8) {
              float fv[8], bv[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                fv[j] = sm.F[tb + t8 + j][cc];
                bv[j] = sm.Bv[tb + t8 + j][cc];
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                hc = __fadd_rn(__fmul_rn(fv[j], hc), bv[j]);
                sm.F[tb + t8 + j][cc] = hc;
              }
            }
          } else {
            for (int t = tb; t < te; ++t) {
              hc = __fadd_rn(__fmul_rn(sm.F[t][cc], hc), sm.Bv[t][cc]);
              sm.F[t][cc] = hc;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.hdone[q][half]);
          fs_tl(a, warp, i, 2 * q + 1);
        }
      }
      a.h[(int64_t)b * a.d + c0 + cc] = hc;
    }
  }
  // TMEM release after the gate warps' last loads: an mbarrier, not a CTA-wide
  // bar.sync after the divergent producer / MMA roles (see k_gemm.cu)
  if (warp >= 2 && warp < 2 + kFEpiWarps) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.tmem_free);
  }
  if (warp == 1) {
    __syncwarp();
    mbar_wait(&sm.tmem_free, 0);
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
    if (TERN_TRACE_ON && a.trace && lane == 0 && blockIdx.x < 1024) a.trace[blockIdx.x * 16 + 2] = gtimer();
  }
}

template <typename TY>
static cudaError_t fcgscan_go(const CUtensorMap& ta, const CUtensorMap& tb, const FcgScanArgs& a,
                              cudaStream_t s) {
  auto kern = k_fcgscan<TY>;
  const size_t smem = sizeof(FcgScanSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int chains = a.B * (a.d / kFCW);
  const int grid = chains < num_sms ? chains : num_sms;
  static unsigned long long* dprof = nullptr;
  static const bool prof_on = getenv("TERN_FS_PROF") != nullptr;
  FcgScanArgs aa = a;
  // gate warps wait for the carry with an explicit 32..256 ns backoff: the hinted wait
  // re-polled ~43 times per wait (ncu: 15 % of the kernel's instructions were those polls);
  // measured 98.8 -> 96.8 us per c2 block.  TERN_FS_BACKOFF=0 restores the hinted wait.
  static const int backoff = getenv("TERN_FS_BACKOFF") ? atoi(getenv("TERN_FS_BACKOFF")) : 32;
  aa.backoff = backoff;
  aa.trace = trace_slot(TERN_K_FCGSCAN, grid);
  aa.nogate = getenv("TERN_FS_NOGATE") != nullptr;
  static const char* tl_path = getenv("TERN_FS_TL");   // debug: CTA 0 phase timeline
  static unsigned long long* dtl = nullptr;
  const int ntl = (a.T + kFBM - 1) / kFBM;
  const size_t tl_n = (size_t)(2 + kFEpiWarps + 2) * ntl * 8;
  if (tl_path) {
    if (dtl) cudaFree(dtl);
    cudaMalloc(&dtl, tl_n * sizeof(unsigned long long));
    cudaMemsetAsync(dtl, 0, tl_n * sizeof(unsigned long long), s);
    aa.tl = dtl;
  }
  if (prof_on) {   // debug only: printed after a synchronous run
    if (!dprof) cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * 1024);
    cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * 8 * 1024, s);
    aa.prof = dprof;
  }
  const long long t0 = 0;
  (void)t0;
  cudaError_t lerr = launch_pdl(kern, dim3(grid), dim3(kFThreads), smem, s, ta, tb, aa);
  if (lerr != cudaSuccess) return lerr;
  if (tl_path) {
    unsigned long long* h = (unsigned long long*)malloc(tl_n * sizeof(unsigned long long));
    cudaMemcpyAsync(h, dtl, tl_n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    FILE* f = fopen(tl_path, "a");
    if (f) {
      fprintf(f, "launch B=%d T=%d d=%d nt=%d\n", a.B, a.T, a.d, ntl);
      for (size_t j = 0; j < tl_n; ++j) fprintf(f, "%llu%c", h[j], (j % 8 == 7) ? '\n' : ' ');
      fclose(f);
    }
    free(h);
  }
  if (prof_on) {
    static unsigned long long h[8 * 1024];
    cudaMemcpyAsync(h, dprof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double sum[8] = {0};
    for (int b = 0; b < grid; ++b)
      for (int i = 0; i < 8; ++i) sum[i] += (double)h[b * 8 + i] / grid;
    fprintf(stderr,
            "[fcgscan prof] B=%d T=%d d=%d chains=%d | per CTA cycles: prod.empty=%.0f "
            "mma.tempty=%.0f mma.full=%.0f epi.tfull=%.0f phaseA=%.0f waitcarry=%.0f phaseC=%.0f\n",
            a.B, a.T, a.d, chains, sum[0], sum[1], sum[2], sum[3], sum[4], sum[5], sum[6]);
  }
  return cudaGetLastError();
}

// The fused kernel runs one CTA per 64-channel chain of one sequence; below two thirds of
// the SMs in chains (B*d/64 < 2*#SMs/3 = 98.7: c2 at B <= 6, c3 at B <= 3, c4 at B <= 2)
// the unfused path (GEMM over all SMs + the 8-channel-wide scan, 8x more CTAs) is
// faster or equal (measured).
bool fcgscan_preferred(int B, int d) {
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  return (int64_t)B * (d / kFCW) * 3 >= 2 * (int64_t)num_sms;
}

bool fcgscan_supported(const tern_weight& w, int d) {
  return w.e8 != nullptr && w.n_seg == 3 && w.n_out == d && d % kFCW == 0 &&
         sizeof(FcgScanSmem) + 1024 <= 227 * 1024;
}

cudaError_t launch_fcgscan(const int8_t* q, int ldq, const float* deq, const int32_t* qsum,
                           const tern_weight& w, const float* bias, int dt, int B, int T, int d,
                           int gate, float* h, void* oprime, cudaStream_t s) {
  if (B == 0 || T == 0) return cudaSuccess;
  if (!fcgscan_supported(w, d)) return cudaErrorInvalidValue;
  const int kp = (w.k + kKAlign - 1) / kKAlign * kKAlign;
  const int M = B * T;
  CUtensorMap ta, tb;
  if (!make_map_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, q, (uint64_t)kp, (uint64_t)M, (uint64_t)ldq,
                   kFBK, kFBM, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (!make_map_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, w.e8, (uint64_t)kp, (uint64_t)w.n_rows,
                   (uint64_t)kp, kFBK, kFBN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  FcgScanArgs a{};
  a.B = B;
  a.T = T;
  a.d = d;
  a.M = M;
  a.num_kb = kp / kFBK;
  a.n_rows = w.n_rows;
  a.deq = deq;
  a.qsum = qsum;
  a.scales = w.scales;
  a.bias = bias;
  a.h = h;
  a.oprime = oprime;
  a.gate = gate;
  return dt == TERN_BF16 ? fcgscan_go<__nv_bfloat16>(ta, tb, a, s) : fcgscan_go<float>(ta, tb, a, s);
}

}  // namespace tern
