// k_gemm.cu -- a4: prefill ternary x int8 GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulator in TMEM), DESIGN.md "Kernels / GEMM".
//
//   D[m][n] = sum_k q[m][k] * e[n][k]     (q int8 activations, e = t+1 in {0,1,2})
//   acc     = D - qsum[m]                 (= sum_{t=+1} q - sum_{t=-1} q)
//
// Per CTA: one 128 x BN output tile, K walked in 128-element blocks through an
// S-stage ring:
//   warp 4      TMA producer: A tile (int8, 128B-swizzled) + packed B tile
//               (BN rows x 8 words) -> smem, mbarrier complete_tx
//   warps 0-3   unpack: 2-bit fields -> uint8 e in the UMMA K-major SW128
//               layout (one AND per 4 values), fence.proxy.async, arrive;
//               afterwards the epilogue (tcgen05.ld -> dequant -> functor -> st)
//   warp 5      TMEM allocation + single-thread tcgen05.mma issue, commit to
//               the stage's empty barrier and finally to the accumulator barrier
#include "epilogue.cuh"

namespace tern {

constexpr int kBM = 128;
constexpr int kBK = 128;  // int8 elements = bytes = one 128B swizzle row

// Warp roles (448 threads):
//   warp 0       TMA producer            warp 1      TMEM alloc + MMA issuer
//   warps 2-5    B unpack (128 thr)      warps 6-13  epilogue (256 thr, 2 per TMEM quadrant)
// Persistent: grid = min(#tiles, #SMs), static round-robin over tiles (m-major
// so CTAs running together share A rows in L2).  Two TMEM accumulators of BN
// columns let the epilogue of tile i overlap the main loop of tile i+1.
constexpr int kGemmThreads = 448;
constexpr int kEpiWarp0 = 6;
constexpr int kEpiWarps = 8;
constexpr int kStageLd = 33;  // epilogue staging row stride (floats): conflict-free

template <int BN> struct GemmCfg {
  static constexpr int S = BN == 256 ? 3 : 4;
  static constexpr int A_BYTES = kBM * kBK;       // 16 KB
  static constexpr int BU_BYTES = BN * kBK;       // unpacked B
  static constexpr int BP_BYTES = BN * (kBK / 4); // packed B: BN rows x 8 words
  static constexpr int STAGE = A_BYTES + BU_BYTES + BP_BYTES;
  static constexpr int EPI_BYTES = kEpiWarps * 32 * kStageLd * 4;
  static constexpr int SMEM = S * STAGE + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;
};

struct GemmArgs {
  int M, n_rows, num_kb, n_tiles, m_tiles;
  const float* deq;
  const int32_t* qsum;
  Epi epi;
};

// Epilogue of one 32-column chunk held by this thread (one row): computes the
// stored values (phase A, thread = row) into the warp's staging tile, then
// writes it with row-contiguous coalesced stores (phase B, lane = column).
template <typename TY>
__device__ __forceinline__ void epi_chunk(const Epi& e, const GemmArgs& a, float* stg, int lane,
                                          int row0, int row, float deq, int qsum, int col0,
                                          const uint32_t (&v)[32], const uint32_t* vu) {
  const bool rv = row < a.M;
  const int nseg = e.n_seg;
  int out_col0;     // first output column of the chunk
  bool active = col0 < a.n_rows;
  if (e.kind == EPI_SWIGLU) {
    const int grp = col0 / 128, half = (col0 % 128) / 32;
    out_col0 = grp * 64 + half * 32;
    active = active && out_col0 < e.n_out;
  } else if (e.kind == EPI_FCG || e.kind == EPI_NONE) {
    out_col0 = col0;
  } else {
    out_col0 = (col0 / (kSegRows * nseg)) * kSegRows + (col0 % kSegRows);  // n_seg == 1: col0
  }
  if (!active) return;
  const int seg = (col0 / kSegRows) % nseg;
  const int rr0 = (col0 / (kSegRows * nseg)) * kSegRows + (col0 % kSegRows);
  // ---- optional int32 accumulator tap (parity), staged the same way
  if (e.acc) {
    int* si = reinterpret_cast<int*>(stg);
#pragma unroll
    for (int j = 0; j < 32; ++j) si[lane * kStageLd + j] = (int)v[j] - qsum;
    if (vu) {
      __syncwarp();
#pragma unroll 4
      for (int r = 0; r < 32; ++r)
        if (row0 + r < a.M && col0 + lane < a.n_rows)
          e.acc[(int64_t)(row0 + r) * e.ldacc + col0 + lane] = si[r * kStageLd + lane];
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) si[lane * kStageLd + j] = (int)vu[j] - qsum;
      __syncwarp();
#pragma unroll 4
      for (int r = 0; r < 32; ++r)
        if (row0 + r < a.M && col0 + 64 + lane < a.n_rows)
          e.acc[(int64_t)(row0 + r) * e.ldacc + col0 + 64 + lane] = si[r * kStageLd + lane];
    } else {
      __syncwarp();
#pragma unroll 4
      for (int r = 0; r < 32; ++r)
        if (row0 + r < a.M && col0 + lane < a.n_rows)
          e.acc[(int64_t)(row0 + r) * e.ldacc + col0 + lane] = si[r * kStageLd + lane];
    }
    __syncwarp();
    if (e.kind == EPI_NONE) return;
  }
  // ---- phase A: thread = row
  if (rv) {
    const float sc = __fmul_rn(deq, __ldg(e.scales + seg));
    if (e.kind == EPI_SWIGLU) {
      const float scu = __fmul_rn(deq, __ldg(e.scales + 1));
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float g = storage_round<TY>(__fmul_rn((float)((int)v[j] - qsum), sc));
        const float u = storage_round<TY>(__fmul_rn((float)((int)vu[j] - qsum), scu));
        stg[lane * kStageLd + j] = swiglu(g, u);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float o = __fmul_rn((float)((int)v[j] - qsum), sc);
        if (e.bias) o = __fadd_rn(o, __ldg(e.bias + seg * e.n_out + rr0 + j));
        stg[lane * kStageLd + j] = storage_round<TY>(o);
      }
    }
  }
  __syncwarp();
  // ---- phase B: lane = column, one coalesced row segment per store
  TY* out = static_cast<TY*>(e.out);
  const int oc = out_col0 + lane;
  const bool cv = (e.kind == EPI_SWIGLU) ? (oc < e.n_out) : (col0 + lane < a.n_rows);
  if (e.kind == EPI_RESID) {
    // all residual loads of the chunk first (they cannot be reordered past the
    // stores by the compiler), then the adds and stores
    const TY* res = static_cast<const TY*>(e.res);
    float xr[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int rw = row0 + r;
      xr[r] = (rw < a.M && cv) ? ld_act<TY>(res + (int64_t)rw * e.ldr + oc) : 0.0f;
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int rw = row0 + r;
      if (rw < a.M && cv)
        st_act<TY>(out + (int64_t)rw * e.ldo + oc, __fadd_rn(xr[r], stg[r * kStageLd + lane]));
    }
  } else {
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const int rw = row0 + r;
      if (rw < a.M && cv) st_act<TY>(out + (int64_t)rw * e.ldo + oc, stg[r * kStageLd + lane]);
    }
  }
  __syncwarp();
}

template <int BN, typename TY>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const GemmArgs a) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::S;
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sA = sm;                                   // [S][A_BYTES]
  uint8_t* sBu = sm + S * Cfg::A_BYTES;               // [S][BU_BYTES]
  uint8_t* sBp = sBu + S * Cfg::BU_BYTES;             // [S][BP_BYTES]
  float* sEpi = reinterpret_cast<float*>(sBp + S * Cfg::BP_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sEpi) + Cfg::EPI_BYTES);
  uint64_t* full = bars;            // TMA landed
  uint64_t* unpacked = bars + S;    // B unpacked
  uint64_t* empty = bars + 2 * S;   // MMA finished reading the stage
  uint64_t* tfull = bars + 3 * S;   // [2] accumulator ready
  uint64_t* tempty = bars + 3 * S + 2;  // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = a.num_kb;
  const int total = a.n_tiles * a.m_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&unpacked[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m0 = (t / a.n_tiles) * kBM, n0 = (t % a.n_tiles) * BN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % S;
          if (g >= (uint32_t)S) mbar_wait(&empty[s], ((g / S) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::BP_BYTES);
          tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * kBK, m0);
          tma_load_2d(sBp + s * Cfg::BP_BYTES, &tmB, &full[s], kb * (kBK / 16), n0);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      // kind::i8 instruction descriptor: D s32, A s8, B u8, both K-major, M=128, N=BN
      const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      uint32_t g = 0, it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const uint32_t acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_addr = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % S;
          mbar_wait(&unpacked[s], (g / S) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(sBu + s * Cfg::BU_BYTES);
#pragma unroll
          for (int kk = 0; kk < kBK / 32; ++kk)
            mma_i8(d_addr, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                   idesc, (kb | kk) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp < kEpiWarp0) {
    // ---------------- unpack (warps 2-5): 2-bit fields -> u8 e, SW128 K-major
    const int tid = threadIdx.x - 64;
    uint32_t g = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&full[s], (g / S) & 1);
        const uint32_t* bp = reinterpret_cast<const uint32_t*>(sBp + s * Cfg::BP_BYTES);
        uint8_t* bu = sBu + s * Cfg::BU_BYTES;
#pragma unroll 4
        for (int i = tid; i < BN * 8; i += 128) {
          const int row = i >> 3, w = i & 7;
          const uint32_t word = bp[i];
          uint4 v;
          v.x = word & 0x03030303u;
          v.y = (word >> 2) & 0x03030303u;
          v.z = (word >> 4) & 0x03030303u;
          v.w = (word >> 6) & 0x03030303u;
          *reinterpret_cast<uint4*>(bu + row * 128 + ((w ^ (row & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
        mbar_arrive(&unpacked[s]);
      }
    }
  } else {
    // ---------------- epilogue (warps 6-13): two warps per TMEM lane quadrant
    const int ew = warp - kEpiWarp0;
    const int quad = warp & 3;          // TMEM lanes [32*quad, 32*quad+32)
    const int half = ew >> 2;           // which half of the chunks this warp takes
    float* stg = sEpi + ew * 32 * kStageLd;
    const Epi& e = a.epi;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const uint32_t acc = it & 1;
      const int m0 = (t / a.n_tiles) * kBM, n0 = (t % a.n_tiles) * BN;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row0 = m0 + quad * 32;
      const int row = row0 + lane;
      const bool rv = row < a.M;
      const float deq = rv ? __ldg(a.deq + row) : 0.0f;
      const int qsum = rv ? __ldg(a.qsum + row) : 0;
      const uint32_t trow = tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16);
      if (e.kind == EPI_SWIGLU) {
        // pair p = (128-col group, 32-col half): gate at +0, up at +64
#pragma unroll 1
        for (int p = half; p < BN / 64; p += 2) {
          const int cb = (p >> 1) * 128 + (p & 1) * 32;
          uint32_t vg[32], vu[32];
          tmem_ld32(trow + cb, vg);
          tmem_ld32(trow + cb + 64, vu);
          tmem_ld_wait();
          epi_chunk<TY>(e, a, stg, lane, row0, row, deq, qsum, n0 + cb, vg, vu);
        }
      } else {
#pragma unroll 1
        for (int c = half; c < BN / 32; c += 2) {
          uint32_t v[32];
          tmem_ld32(trow + c * 32, v);
          tmem_ld_wait();
          epi_chunk<TY>(e, a, stg, lane, row0, row, deq, qsum, n0 + c * 32, v, nullptr);
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
  }
}

// ----------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

static bool make_map_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                        uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swz) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, typename TY>
static cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                               cudaStream_t s) {
  auto kern = k_gemm_tc<BN, TY>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GemmCfg<BN>::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int total = a.n_tiles * a.m_tiles;
  const int grid = total < num_sms ? total : num_sms;
  kern<<<grid, kGemmThreads, GemmCfg<BN>::SMEM, s>>>(ta, tb, a);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const int8_t* q, int M, int ldq, const float* deq, const int32_t* qsum,
                        const tern_weight& w, int ydt, const Epi& epi, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const int kp = (w.k + kKAlign - 1) / kKAlign * kKAlign;
  // BN = 256 when the group has whole 256-row tiles worth of work, else 128
  const int BN = (w.n_rows >= 1024 || w.n_rows % 256 == 0) ? 256 : 128;
  CUtensorMap ta, tb;
  if (!make_map_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, q, (uint64_t)kp, (uint64_t)M,
                   (uint64_t)ldq, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (!make_map_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT32, w.codes, (uint64_t)(kp / 16),
                   (uint64_t)w.n_rows, (uint64_t)w.ldw * 4, kBK / 16, BN,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  GemmArgs a{};
  a.M = M;
  a.n_rows = w.n_rows;
  a.num_kb = kp / kBK;
  a.n_tiles = (w.n_rows + BN - 1) / BN;
  a.m_tiles = (M + kBM - 1) / kBM;
  a.deq = deq;
  a.qsum = qsum;
  a.epi = epi;
  const bool yb = ydt == TERN_BF16;
  if (BN == 256)
    return yb ? gemm_launch<256, __nv_bfloat16>(ta, tb, a, s) : gemm_launch<256, float>(ta, tb, a, s);
  return yb ? gemm_launch<128, __nv_bfloat16>(ta, tb, a, s) : gemm_launch<128, float>(ta, tb, a, s);
}

}  // namespace tern
