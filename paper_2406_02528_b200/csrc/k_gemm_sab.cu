// k_gemm_sab.cu -- a3/a4 for decode batches (4 < M <= 256 tokens per call): the ternary
// contraction with the operands swapped so the WEIGHTS are the MMA's M = 128 operand and
// the few tokens its N (SURVEY.md Exec. summary item 7, "swap-AB"), DESIGN.md §6.
//
//   D[r][t] = sum_k e[r][k] * q[t][k]   (e = t+1 in {0,1,2} per packed row r, q int8)
//   part[slice][t][r] = D (int32, exact); k_splitk_epi then sums the K slices in order,
//   subtracts sum_k q[t][k] (sum_{+1} q - sum_{-1} q) and runs the epilogue.
//
// A decode batch streams every weight once per step while the activations are a few KB,
// so the kernel is organised around the weight stream, in its 2-bit form (0.25 B per
// weight, 4x fewer bytes than the u8 copy the prefill GEMM loads):
//   warp 0      producer: the 2-bit code span of (row tile, k-block) -- one contiguous 4 KB
//               bulk copy in the K-block-major layout -- and the q tile [NT tokens][128]
//               (TMA, 128-byte swizzle, rows beyond M zero-filled); the first stages' code
//               loads are issued before the PDL wait (weights do not depend on the
//               previous kernel)
//   warps 8-11  unpack the 2-bit fields into the u8 A tile (128 rows x 128, SW128 K-major),
//               also ahead of the dependency wait
//   warp 1      TMEM allocation + single-thread tcgen05.mma kind::i8 (A u8, B s8, M = 128,
//               N = NT), two accumulators so a tile's drain overlaps the next tile's MMAs
//   warps 4-7   drain: TMEM lane = weight row, so each token's 32 rows per warp are one
//               coalesced 128-byte store into part[slice][t][*]
// Work unit = (row tile of 128 packed rows, K slice); slices spread the few row tiles of a
// small matrix over all SMs.
//
// Status: built, bit-exact, OPT-IN (TERN_GEMM_SAB=1).  Measured slower than the default
// small-M path (u8 weight tiles, 128-wide, k_gemm.cu) on c3 B = 64 (44.7k vs 51.1k tok/s) and
// c4 B = 128 (50.8k vs 62.2k): a tcgen05.mma kind::i8 instruction costs ~116 cycles whatever
// its N up to 128 (tools/micro/mma_lat.cu: 465 cycles per 4-MMA k-block for N = 32..128, 520
// for N = 256), so with the tokens as N each weight byte costs as many MMA cycles as in the
// un-swapped kernel, and the unpack adds to the per-k-block chain.
#include <cstdio>
#include <cstdlib>

#include "epilogue.cuh"

namespace tern {

namespace {

constexpr int kSabThreads = 12 * 32;
constexpr int kSabRows = 128;   // packed weight rows per tile (MMA M)
constexpr int kSabK = 128;      // K per stage (one 128-byte swizzle row of int8)

// Code stages: 48 KB in flight per SM, most of a work unit's weights, issued before the
// dependency wait so the weight fetch overlaps the previous kernel.
// The unpack -> MMA -> release round trip (two mbarrier hand-offs and the MMAs) is long
// against a k-block's 128 MMA cycles, so the unpacked ring is deep too (measured: with 3
// stages the MMA and the unpack warps each waited ~half the kernel, TERN_SAB_PROF).
template <int NT> struct SabCfg {
  static constexpr int SC = 12;                      // code stages (4 KB each)
  static constexpr int SQ = NT >= 256 ? 3 : (NT >= 128 ? 4 : 6);   // q stages (NT x 128 B)
  static constexpr int U = NT >= 256 ? 4 : 6;        // unpacked A stages (16 KB)
  static constexpr int Q_BYTES = NT * kSabK;
  static constexpr int A_BYTES = kSabRows * kSabK;
  static constexpr int C_BYTES = kSabRows * 32;
  static constexpr int SMEM = SQ * Q_BYTES + U * A_BYTES + SC * C_BYTES + 1024 + 1024;
  static constexpr int TMEM_COLS = 2 * NT;
};

struct SabArgs {
  int M, n_rows, num_kb, n_tiles, ksplit, kb_per;
  const uint32_t* codes;   // K-block-major [num_kb][n_rows][8]
  int32_t* part;           // [ksplit][M][n_rows]
  unsigned long long* trace;   // tern_trace_enable timeline (trace build only)
  unsigned long long* prof;    // debug (TERN_SAB_PROF): [grid][8] wait cycles per site
};

// Polling mbarrier wait (no suspend hint: the hand-offs here are short and on the critical
// path) with the library's watchdog: a lost arrival traps after ~20 s instead of hanging.
__device__ __forceinline__ void spin_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, polls = 0;
  unsigned long long t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if ((++polls & 4095u) == 0) {
      const unsigned long long t = gtimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();
    }
  }
}

// spin_wait that (TERN_SAB_PROF) adds the cycles it blocked to a per-CTA site counter
__device__ __forceinline__ void swait(uint64_t* bar, uint32_t parity, unsigned long long* prof,
                                      int site) {
  if (prof == nullptr) {
    spin_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  spin_wait(bar, parity);
  atomicAdd(prof + blockIdx.x * 8 + site, (unsigned long long)(clock64() - t0));
}

template <int NT>
__global__ void __launch_bounds__(kSabThreads, 1)
    k_gemm_sab(const __grid_constant__ CUtensorMap tmQ, const SabArgs a) {
  using Cfg = SabCfg<NT>;
  extern __shared__ __align__(1024) uint8_t sab_raw[];
  uint8_t* sm = sab_raw + ((1024u - (smem_u32(sab_raw) & 1023u)) & 1023u);
  uint8_t* sQ = sm;                                   // [SQ][Q_BYTES]  (SW128)
  uint8_t* sA = sQ + Cfg::SQ * Cfg::Q_BYTES;          // [U][A_BYTES]   (SW128)
  uint8_t* sC = sA + Cfg::U * Cfg::A_BYTES;           // [SC][C_BYTES]  packed codes
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + Cfg::SC * Cfg::C_BYTES);
  uint64_t* cfull = bars;          // [SC] codes landed
  uint64_t* cempty = bars + 16;    // [SC] codes unpacked (slot free)
  uint64_t* qfull = bars + 32;     // [SQ] q tile landed
  uint64_t* qempty = bars + 40;    // [SQ] MMA done with the q tile
  uint64_t* ufull = bars + 48;     // [U] A tile unpacked
  uint64_t* uempty = bars + 56;    // [U] MMA done with the A tile
  uint64_t* tfull = bars + 64;     // [2] accumulator ready
  uint64_t* tempty = bars + 66;    // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 68);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.n_tiles * a.ksplit;
  trace_mark(a.trace, 0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    for (int s = 0; s < Cfg::SC; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 4);
    }
    for (int s = 0; s < Cfg::SQ; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 1);
    }
    for (int u = 0; u < Cfg::U; ++u) {
      mbar_init(&ufull[u], 4);
      mbar_init(&uempty[u], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // (unit, k-block) sequence of this CTA: g counts k-blocks over its units in order.  Every
  // CTA reads the same q tiles, so each walks its K range from a CTA-dependent rotation
  // (kb_at): at any moment the CTAs read different q tiles instead of all hitting the L2
  // lines of one (integer sums: the order does not change the result).
  auto unit_kb = [&](int t, int& r0, int& kb0, int& kb1) {
    const int tile = t / a.ksplit, sp = t % a.ksplit;
    r0 = tile * kSabRows;
    kb0 = sp * a.kb_per;
    kb1 = min(a.num_kb, kb0 + a.kb_per);
  };
  auto kb_at = [&](int kb0, int kb1, int j) {
    const int n = kb1 - kb0;
    return kb0 + (j + (int)(blockIdx.x % (unsigned)n)) % n;
  };

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      auto load_codes = [&](uint32_t g, int kb, int r0) {
        const int s = g % Cfg::SC;
        if (g >= (uint32_t)Cfg::SC) swait(&cempty[s], ((g / Cfg::SC) - 1) & 1, a.prof, 0);
        const uint32_t bytes = (uint32_t)min(kSabRows, a.n_rows - r0) * 32u;
        mbar_arrive_expect_tx(&cfull[s], bytes);
        bulk_load(sC + s * Cfg::C_BYTES, a.codes + ((int64_t)kb * a.n_rows + r0) * 8, bytes,
                  &cfull[s]);
      };
      // weights of the first stages before the dependency wait
      uint32_t npre = 0;
      {
        uint32_t g = 0;
        for (int t = blockIdx.x; t < total && npre < (uint32_t)Cfg::SC; t += gridDim.x) {
          int r0, kb0, kb1;
          unit_kb(t, r0, kb0, kb1);
          for (int j = 0; j < kb1 - kb0 && npre < (uint32_t)Cfg::SC; ++j, ++g, ++npre)
            load_codes(g, kb_at(kb0, kb1, j), r0);
        }
      }
      pdl_wait();   // q and its tensor comes from the previous kernel (the quant)
      uint32_t g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int r0, kb0, kb1;
        unit_kb(t, r0, kb0, kb1);
        for (int j = 0; j < kb1 - kb0; ++j, ++g) {
          const int kb = kb_at(kb0, kb1, j);
          const int sq = g % Cfg::SQ;
          if (g >= (uint32_t)Cfg::SQ) swait(&qempty[sq], ((g / Cfg::SQ) - 1) & 1, a.prof, 1);
          mbar_arrive_expect_tx(&qfull[sq], Cfg::Q_BYTES);
          tma_load_2d(sQ + sq * Cfg::Q_BYTES, &tmQ, &qfull[sq], kb * kSabK, 0);
          if (g >= npre) load_codes(g, kb, r0);
        }
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    pdl_launch_dependents();
    if (lane == 0 && a.trace && blockIdx.x < 1024) a.trace[blockIdx.x * 16 + 1] = gtimer();
    // ---------------- MMA issuer
    if (lane == 0) {
      // kind::i8 instruction descriptor: D s32, A u8 (weights e), B s8 (q), both K-major,
      // M = 128, N = NT
      const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) |
                             ((uint32_t)(kSabRows >> 4) << 24);
      uint32_t g = 0, it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const uint32_t acc = it & 1;
        swait(&tempty[acc], ((it >> 1) & 1) ^ 1, a.prof, 2);
        tc_fence_after();
        const uint32_t d_addr = tmem_base + acc * NT;
        int r0, kb0, kb1;
        unit_kb(t, r0, kb0, kb1);
        for (int j = 0; j < kb1 - kb0; ++j, ++g) {
          const int u = g % Cfg::U, sq = g % Cfg::SQ;
          swait(&ufull[u], (g / Cfg::U) & 1, a.prof, 3);
          swait(&qfull[sq], (g / Cfg::SQ) & 1, a.prof, 4);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + u * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(sQ + sq * Cfg::Q_BYTES);
#pragma unroll
          for (int kk = 0; kk < kSabK / 32; ++kk)
            mma_i8(d_addr, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                   idesc, (j | kk) != 0);
          mma_commit(&uempty[u]);
          mma_commit(&qempty[sq]);
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 8) {
    // ---------------- unpack (warps 8-11): 2-bit fields -> u8 e, SW128 K-major; needs only
    // the weights, so it runs ahead of the dependency wait
    const int tid = threadIdx.x - 256;
    const int rr0 = tid >> 3, w = tid & 7;   // word w of rows rr0 + 16 j
    uint32_t g = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int r0, kb0, kb1;
      unit_kb(t, r0, kb0, kb1);
      const int nrow = min(kSabRows, a.n_rows - r0);
      for (int j = 0; j < kb1 - kb0; ++j, ++g) {
        const int s = g % Cfg::SC, u = g % Cfg::U;
        if (g >= (uint32_t)Cfg::U) swait(&uempty[u], ((g / Cfg::U) - 1) & 1, tid == 0 ? a.prof : nullptr, 5);
        swait(&cfull[s], (g / Cfg::SC) & 1, tid == 0 ? a.prof : nullptr, 6);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(sC + s * Cfg::C_BYTES) + tid;
        uint8_t* dst = sA + u * Cfg::A_BYTES + rr0 * 128 + ((w ^ (rr0 & 7)) << 4);
#pragma unroll
        for (int j = 0; j < kSabRows / 16; ++j) {
          // rows past the matrix (ragged last tile) hold stale bytes: their D rows are
          // never stored
          const uint32_t word = rr0 + 16 * j < nrow ? src[j * 128] : 0u;
          uint4 v;
          v.x = word & 0x03030303u;
          v.y = (word >> 2) & 0x03030303u;
          v.z = (word >> 4) & 0x03030303u;
          v.w = (word >> 6) & 0x03030303u;
          *reinterpret_cast<uint4*>(dst + j * 2048) = v;
        }
        fence_proxy_async_smem();   // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {            // one arrival per unpack warp (count 4)
          mbar_arrive(&ufull[u]);
          mbar_arrive(&cempty[s]);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- drain (warps 4-7 = TMEM lane quadrants 0-3): thread = packed row
    const int quad = warp & 3;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const uint32_t acc = it & 1;
      int r0, kb0, kb1;
      unit_kb(t, r0, kb0, kb1);
      const int row = r0 + quad * 32 + lane;
      int32_t* slice = a.part + (int64_t)(t % a.ksplit) * a.M * a.n_rows;
      swait(&tfull[acc], (it >> 1) & 1, (quad == 0 && lane == 0) ? a.prof : nullptr, 7);
      tc_fence_after();
      const uint32_t trow = tmem_base + acc * NT + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < NT / 32 && c * 32 < a.M; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        tmem_ld_wait();
        if (row < a.n_rows) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int tok = c * 32 + j;
            if (tok < a.M) slice[(int64_t)tok * a.n_rows + row] = (int32_t)v[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    if (lane == 0 && a.trace && blockIdx.x < 1024) a.trace[blockIdx.x * 16 + 2] = gtimer();
  }
}

template <int NT>
cudaError_t sab_go(const CUtensorMap& tq, const SabArgs& a, cudaStream_t s) {
  using Cfg = SabCfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_sab<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int total = a.n_tiles * a.ksplit;
  const int grid = total < num_sms ? total : num_sms;
  SabArgs aa = a;
  aa.trace = TERN_TRACE_ON ? trace_slot(TERN_K_GEMM + 32, grid) : nullptr;
  static unsigned long long* dprof = nullptr;
  static const bool prof_on = getenv("TERN_SAB_PROF") != nullptr;
  if (prof_on) {   // debug only: per-site wait cycles, printed after a synchronous run
    if (!dprof) cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * 1024);
    cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * 8 * 1024, s);
    aa.prof = dprof;
  }
  cudaError_t err = launch_pdl(k_gemm_sab<NT>, dim3(grid), dim3(kSabThreads), (size_t)Cfg::SMEM, s,
                               tq, aa);
  if (err != cudaSuccess || !prof_on) return err;
  static unsigned long long h[8 * 1024];
  cudaMemcpyAsync(h, dprof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  double sum[8] = {0};
  for (int b = 0; b < grid; ++b)
    for (int i = 0; i < 8; ++i) sum[i] += (double)h[b * 8 + i] / grid;
  fprintf(stderr,
          "[sab prof] M=%d n_rows=%d kb=%d tiles=%d ks=%d NT=%d | avg wait cycles: prod.cempty=%.0f "
          "prod.qempty=%.0f mma.tempty=%.0f mma.ufull=%.0f mma.qfull=%.0f unp.uempty=%.0f "
          "unp.cfull=%.0f drain.tfull=%.0f\n",
          a.M, a.n_rows, a.num_kb, a.n_tiles, a.ksplit, NT, sum[0], sum[1], sum[2], sum[3], sum[4],
          sum[5], sum[6], sum[7]);
  return cudaSuccess;
}

}  // namespace

bool gemm_sab_supported(int M) { return M >= 1 && M <= 256; }

// int32 partials part[ks][M][n_rows] of the swap-AB contraction; *ks_out = the number of K
// slices used (the caller sums them: k_splitk_epi / k_fin).
cudaError_t launch_gemm_sab(const int8_t* q, int M, int ldq, const tern_weight& w, int32_t* part,
                            size_t part_bytes, int ks_max, int* ks_out, cudaStream_t s) {
  if (!gemm_sab_supported(M) || !part) return cudaErrorInvalidValue;
  const int kp = (w.k + kKAlign - 1) / kKAlign * kKAlign;
  const int NT = M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
  CUtensorMap tq;
  if (!make_map_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_UINT8, q, (uint64_t)kp, (uint64_t)M, (uint64_t)ldq,
                   kSabK, NT, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  SabArgs a{};
  a.M = M;
  a.n_rows = w.n_rows;
  a.num_kb = kp / kSabK;
  a.n_tiles = (w.n_rows + kSabRows - 1) / kSabRows;
  a.codes = w.codes;
  a.part = part;
  // K slices: one round of work units over the SMs
  const size_t slice = (size_t)M * w.n_rows * sizeof(int32_t);
  int ks = num_sms / a.n_tiles;
  if (ks_max > 0 && ks > ks_max) ks = ks_max;
  if (ks > a.num_kb) ks = a.num_kb;
  if ((size_t)ks * slice > part_bytes) ks = (int)(part_bytes / slice);
  if (ks < 1) return cudaErrorInvalidValue;
  a.kb_per = (a.num_kb + ks - 1) / ks;
  a.ksplit = (a.num_kb + a.kb_per - 1) / a.kb_per;
  *ks_out = a.ksplit;
  switch (NT) {
    case 32: return sab_go<32>(tq, a, s);
    case 64: return sab_go<64>(tq, a, s);
    case 128: return sab_go<128>(tq, a, s);
    default: return sab_go<256>(tq, a, s);
  }
}

}  // namespace tern
