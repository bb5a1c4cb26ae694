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

template <int BN> struct GemmCfg {
  static constexpr int S = BN == 256 ? 3 : 4;
  static constexpr int A_BYTES = kBM * kBK;       // 16 KB
  static constexpr int BU_BYTES = BN * kBK;       // unpacked B
  static constexpr int BP_BYTES = BN * (kBK / 4); // packed B: BN rows x 8 words
  static constexpr int STAGE = A_BYTES + BU_BYTES + BP_BYTES;
  static constexpr int SMEM = S * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

struct GemmArgs {
  int M, n_rows, num_kb;
  const float* deq;
  const int32_t* qsum;
  Epi epi;
};

template <int BN, typename TY>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const GemmArgs a) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::S;
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                                   // [S][A_BYTES]
  uint8_t* sBu = sm + S * Cfg::A_BYTES;               // [S][BU_BYTES]
  uint8_t* sBp = sBu + S * Cfg::BU_BYTES;             // [S][BP_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBp + S * Cfg::BP_BYTES);
  uint64_t* full = bars;            // TMA landed
  uint64_t* unpacked = bars + S;    // B unpacked
  uint64_t* empty = bars + 2 * S;   // MMA finished reading the stage
  uint64_t* accfull = bars + 3 * S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * kBM;
  const int nk = a.num_kb;

  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&unpacked[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accfull, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 4) {
    // ---------------- TMA producer
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::BP_BYTES);
        tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * kBK, m0);
        tma_load_2d(sBp + s * Cfg::BP_BYTES, &tmB, &full[s], kb * (kBK / 16), n0);
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer
    if (lane == 0) {
      // kind::i8 instruction descriptor: D s32, A s8, B u8, both K-major, M=128, N=BN
      const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % S;
        mbar_wait(&unpacked[s], (kb / S) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + s * Cfg::A_BYTES);
        const uint32_t b_addr = smem_u32(sBu + s * Cfg::BU_BYTES);
#pragma unroll
        for (int kk = 0; kk < kBK / 32; ++kk) {
          mma_i8(tmem_base, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                 idesc, (kb | kk) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accfull);
    }
  } else {
    // ---------------- unpack (warps 0-3)
    const int tid = threadIdx.x;  // 0..127
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      const uint32_t* bp = reinterpret_cast<const uint32_t*>(sBp + s * Cfg::BP_BYTES);
      uint8_t* bu = sBu + s * Cfg::BU_BYTES;
#pragma unroll 4
      for (int it = tid; it < BN * 8; it += 128) {
        const int row = it >> 3, w = it & 7;
        const uint32_t word = bp[it];
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

    // ---------------- epilogue: TMEM -> registers -> dequant -> functor -> global
    mbar_wait(accfull, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
    const bool rv = row < a.M;
    const float deq = rv ? __ldg(a.deq + row) : 0.0f;
    const int qsum = rv ? __ldg(a.qsum + row) : 0;
    const uint32_t trow = tmem_base + ((uint32_t)(warp * 32) << 16);
    const Epi& e = a.epi;
    const int nseg = e.n_seg;
    if (e.kind == EPI_SWIGLU) {
      // each 128-column group holds [64 gate | 64 up] of the same 64 channels
      for (int g = 0; g < BN / 128; ++g) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          uint32_t rg[32], ru[32];
          tmem_ld32(trow + g * 128 + half * 32, rg);
          tmem_ld32(trow + g * 128 + 64 + half * 32, ru);
          tmem_ld_wait();
          const int pcol = n0 + g * 128 + half * 32;  // packed row of the gate column
          const int grp = pcol / 128;
          const int r0 = grp * 64 + half * 32;        // logical channel of lane 0 column
          if (rv) {
            TY* out = static_cast<TY*>(e.out) + (int64_t)row * e.ldo;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int rr = r0 + j;
              const int ag = (int)rg[j] - qsum, au = (int)ru[j] - qsum;
              if (e.acc && pcol < a.n_rows) {
                e.acc[(int64_t)row * e.ldacc + pcol + j] = ag;
                e.acc[(int64_t)row * e.ldacc + pcol + 64 + j] = au;
              }
              if (rr < e.n_out) {
                const float gh = bl_out<TY>(e, ag, deq, 0, rr);
                const float uh = bl_out<TY>(e, au, deq, 1, rr);
                st_act<TY>(out + rr, swiglu(gh, uh));
              }
            }
          }
        }
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t rv32[32];
        tmem_ld32(trow + c * 32, rv32);
        tmem_ld_wait();
        const int col0 = n0 + c * 32;
        if (rv && col0 < a.n_rows) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = col0 + j;
            const int seg = (col / kSegRows) % nseg;
            const int rr = (col / (kSegRows * nseg)) * kSegRows + (col % kSegRows);
            if (col < a.n_rows && rr < e.n_out)
              epi_single<TY>(e, row, col, seg, rr, (int)rv32[j] - qsum, deq);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<BN>(tmem_base);
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
  dim3 grid((a.n_rows + BN - 1) / BN, (a.M + kBM - 1) / kBM);
  kern<<<grid, 192, GemmCfg<BN>::SMEM, s>>>(ta, tb, a);
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
  a.deq = deq;
  a.qsum = qsum;
  a.epi = epi;
  const bool yb = ydt == TERN_BF16;
  if (BN == 256)
    return yb ? gemm_launch<256, __nv_bfloat16>(ta, tb, a, s) : gemm_launch<256, float>(ta, tb, a, s);
  return yb ? gemm_launch<128, __nv_bfloat16>(ta, tb, a, s) : gemm_launch<128, float>(ta, tb, a, s);
}

}  // namespace tern
