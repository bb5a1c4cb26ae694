// k_gemm.cu -- a4: prefill ternary x int8 GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulator in TMEM), DESIGN.md "Kernels / GEMM".
//
//   D[m][n] = sum_k q[m][k] * e[n][k]     (q int8 activations, e = t+1 in {0,1,2})
//   acc     = D - qsum[m]                 (= sum_{t=+1} q - sum_{t=-1} q)
//
// Persistent, warp-specialised, one 128 x BN output tile per step:
//   warp 0      TMA producer: A tile (int8, SW128) and the B tile, either the
//               pre-expanded u8 copy (kPre: TMA SW128, no unpack) or the 2-bit
//               packed span (one bulk copy, K-block-major layout)
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue
//   warps 2-5   (packed B only) unpack 2-bit fields -> u8 e in the SW128 layout
//   warps 6-13  epilogue, two per TMEM lane quadrant: tcgen05.ld -> dequant ->
//               functor -> swizzled smem tile -> TMA bulk-tensor store
// Two TMEM accumulators let the epilogue of tile i overlap the main loop of
// tile i+1.  Shared-memory (MIO) traffic is the binding resource on this chip
// for 1-CTA tiles, which is what the pre-expanded B and the TMA-store epilogue
// minimise (measured with the TERN_GEMM_PROF counters).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "epilogue.cuh"

namespace tern {

constexpr int kBM = 128;
constexpr int kBK = 128;  // int8 elements = bytes = one 128B swizzle row
constexpr int kGemmThreads = 448;
constexpr int kEpiWarp0 = 6;
constexpr int kEpiWarps = 8;
constexpr int kEpiBuf = 4096;  // bytes of one 32x32 staging tile (fp32)
constexpr int kSmallM = 256;   // M at or below: packed B tiles (+ split-K when tiles are few)

// residual-epilogue variant (RES): ring stages and staging tiles per drain warp (the
// residual loads run kResNB - 1 chunks ahead)
#ifndef TERN_RES_S
#define TERN_RES_S 3
#endif
#ifndef TERN_RES_NB
#define TERN_RES_NB 2
#endif
constexpr int kResS = TERN_RES_S, kResNB = TERN_RES_NB;
// ring stages of the 128-wide u8 tiles (decode batches, short prefills)
#ifndef TERN_S128
#define TERN_S128 4
#endif
template <int BN, bool kPre, bool RES = false, int EW = kEpiWarps> struct GemmCfg {
  static constexpr int A_BYTES = kBM * kBK;        // 16 KB
  static constexpr int B_BYTES = BN * kBK;         // u8 B tile
  static constexpr int BP_BYTES = BN * (kBK / 4);  // packed B: BN rows x 8 words
  // TMA ring depth S, unpacked ring depth U (packed path only), epilogue
  // staging tiles per warp NB: the u8 256-wide ring takes a 4th stage (deeper
  // load pipeline) at the price of single-buffered epilogue stores -- except for the
  // residual epilogue (RES), where two staging tiles per warp let each chunk's residual
  // load be issued one chunk ahead (its HBM latency otherwise serialises the drain and
  // the MMA waits on the accumulators: TERN_GEMM_PROF mma.tempty)
  // EW = 12 drain warps (the u8 path's idle unpack warps 2-5 join the 8 drain warps) for
  // the SwiGLU epilogue, whose arithmetic (2 exact sigmoids per p) outlasts a K = 1024 tile's
  // MMAs; its staging takes the 4th ring stage
  static constexpr int S = kPre ? ((RES && BN == 256) ? kResS : (EW == 12 && BN == 256) ? 3
                                   : (BN == 128 ? TERN_S128 : 4))
                               : (BN == 256 ? 4 : 5);
  static constexpr int U = kPre ? 0 : 2;
  static constexpr int NB = (kPre && BN == 256 && RES) ? kResNB : (kPre && BN == 256) ? 1 : 2;
  static constexpr int EW0 = EW == 12 ? 2 : kEpiWarp0;   // first drain warp
  static constexpr int NG = EW / 4;                      // drain warps per TMEM lane quadrant
  static constexpr int RING = kPre ? S * (A_BYTES + B_BYTES) : S * (A_BYTES + BP_BYTES) + U * B_BYTES;
  static constexpr int EPI_BYTES = EW * NB * kEpiBuf;
  static constexpr int SMEM = RING + EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;
};

struct GemmArgs {
  int M, n_rows, num_kb, n_tiles, m_tiles;
  int ksplit, kb_per;        // split-K (small M): work unit = (tile, K slice)
  int32_t* part;             // ksplit > 1: int32 partial sums [M][n_rows], pre-zeroed
  const uint32_t* codes;     // K-block-major packed weights [num_kb][n_rows][8]
  const float* deq;
  const int32_t* qsum;
  Epi epi;
  unsigned long long* prof;  // debug (TERN_GEMM_PROF): [grid][8] wait cycles per site
  // fused quantization of A (QFuse, qctr != NULL): warps 2-5 quantize rows of qx into
  // q = the A operand (qq, ldq), deq and qsum; qctr[0] reserved, qctr[1 + b] publishes
  // 128-row block b (complete at 128)
  const void* qx;
  int qldx, qK, qmb;         // qmb = ceil(M / 128) blocks
  const float* qgain;
  float qeps;
  double qinv_k;
  int8_t* qq;
  int qldq;
  float* qdeq;
  int32_t* qqsum;
  uint32_t* qctr;
#ifdef TERN_TRACE
  unsigned long long* trace; // tern_trace_enable timeline (trace build only)
#endif
};

// mbar_wait that (in the TERN_GEMM_PROF debug mode) adds the cycles it blocked
// to a per-CTA counter for its call site.
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity, unsigned long long* prof,
                                      int site) {
  if (prof == nullptr) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  atomicAdd(prof + blockIdx.x * 8 + site, (unsigned long long)(clock64() - t0));
}

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// the staging tile added element-wise onto the global tensor (fp32 add at L2, one IEEE
// rounding per element: the residual add of EPI_RESID_RED)
__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of 16-byte chunk c of row r in a swizzled 32-row staging tile
// (fp32: 128-byte rows, SWIZZLE_128B; bf16: 64-byte rows, SWIZZLE_64B)
template <typename TY> __device__ __forceinline__ int stg_off(int r, int c);
template <> __device__ __forceinline__ int stg_off<float>(int r, int c) {
  return r * 128 + ((c ^ (r & 7)) << 4);
}
template <> __device__ __forceinline__ int stg_off<__nv_bfloat16>(int r, int c) {
  return r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
}

// write the 32 values of this thread's row into the staging tile
template <typename TY> __device__ __forceinline__ void stg_write_row(uint8_t* buf, int r, const float (&o)[32]);
template <> __device__ __forceinline__ void stg_write_row<float>(uint8_t* buf, int r, const float (&o)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(buf + stg_off<float>(r, c)) =
        make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return a | (b << 16);
}
template <> __device__ __forceinline__ void stg_write_row<__nv_bfloat16>(uint8_t* buf, int r,
                                                                          const float (&o)[32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 v;
    v.x = pack_bf16x2(o[8 * c], o[8 * c + 1]);
    v.y = pack_bf16x2(o[8 * c + 2], o[8 * c + 3]);
    v.z = pack_bf16x2(o[8 * c + 4], o[8 * c + 5]);
    v.w = pack_bf16x2(o[8 * c + 6], o[8 * c + 7]);
    *reinterpret_cast<uint4*>(buf + stg_off<__nv_bfloat16>(r, c)) = v;
  }
}
// read this thread's row of the (residual) tile back as floats
template <typename TY> __device__ __forceinline__ void stg_read_row(const uint8_t* buf, int r, float (&x)[32]);
template <> __device__ __forceinline__ void stg_read_row<float>(const uint8_t* buf, int r, float (&x)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = *reinterpret_cast<const float4*>(buf + stg_off<float>(r, c));
    x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
  }
}
template <> __device__ __forceinline__ void stg_read_row<__nv_bfloat16>(const uint8_t* buf, int r,
                                                                         float (&x)[32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 v = *reinterpret_cast<const uint4*>(buf + stg_off<__nv_bfloat16>(r, c));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[8 * c + 2 * i] = __uint_as_float(w[i] << 16);
      x[8 * c + 2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}

__device__ __forceinline__ uint32_t trow_base(uint32_t tmem_base, uint32_t acc, int BN, int quad) {
  return tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16);
}

// int32 accumulator tap (parity tests only): plain coalesced stores through a
// padded staging tile (the two staging buffers of the warp, 8 KB)
__device__ void acc_tap_chunk(const Epi& e, const GemmArgs& a, int* si, int lane, int row0,
                              int col0, int qsum, const uint32_t (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) si[lane * 32 + (j ^ lane)] = (int)v[j] - qsum;   // XOR swizzle
  __syncwarp();
  for (int r = 0; r < 32; ++r)
    if (row0 + r < a.M && col0 + lane < a.n_rows)
      e.acc[(int64_t)(row0 + r) * e.ldacc + col0 + lane] = si[r * 32 + (lane ^ r)];
  __syncwarp();
}

// ----------------------------------------------------------------- fused quantization (f3)
// a2 (RMSNorm + per-token absmax int8, readings C1-C5; DESIGN.md "Canonical
// numerics") run by the GEMM's otherwise idle warps 2-5 while the tensor cores work on
// blocks already quantized: the A operand of 128-row block b is published in qctr[1 + b]
// (a release add per finished row; the producer waits for 128 with acquire loads, then a
// generic -> async proxy fence before its TMA reads), so no standalone quant launch, no
// launch gap, and the quantization's HBM traffic overlaps the MMAs.  The arithmetic is
// k_quant's (binary64 fma sum of squares in a fixed per-warp tree order, C4; the 1-ulp
// binary64 rsqrt; fl(max|x| r) when there is no gain; IEEE divisions; round half away).
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// block until 128-row block mb of the fused quantization is published
__device__ __forceinline__ void qf_wait_block(const uint32_t* ctr, int mb) {
  const uint32_t* f = ctr + 1 + mb;
  if (ld_acquire_u32(f) >= 128u) return;
  const unsigned long long t0 = gtimer();
  while (ld_acquire_u32(f) < 128u) {
    __nanosleep(40);
    if (gtimer() - t0 > 4000000000ull) __trap();   // watchdog (4 s), as mbar_wait
  }
}
template <typename TY> __device__ __forceinline__ void qf_unpack(const uint4& u, float* v);
template <> __device__ __forceinline__ void qf_unpack<float>(const uint4& u, float* v) {
  v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
  v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
}
template <> __device__ __forceinline__ void qf_unpack<__nv_bfloat16>(const uint4& u, float* v) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
constexpr int kQfCh = 8;   // 16-byte vectors per lane per chunk of a row

// one chunk of the row (kQfCh vectors per lane, vector v = c*256 + i*32 + lane)
template <typename TY>
__device__ __forceinline__ void qf_load_chunk(const uint4* xr, bool rv, int c, int nvec, int lane,
                                              uint4 (&xv)[kQfCh]) {
#pragma unroll
  for (int i = 0; i < kQfCh; ++i) {
    const int v = c * 32 * kQfCh + i * 32 + lane;
    xv[i] = (rv && v < nvec) ? __ldg(xr + v) : make_uint4(0, 0, 0, 0);
  }
}
// quantize one loaded chunk: q bytes of vectors < nvecp (zeros beyond K = the padding)
template <typename TY>
__device__ __forceinline__ int qf_quant_chunk(const uint4 (&xv)[kQfCh], int c, int nvec, int nvecp,
                                              int lane, float r, float sc, const float* gain,
                                              int8_t* qr, bool rv) {
  constexpr int VE = 16 / sizeof(TY);
  int qs = 0;
#pragma unroll
  for (int i = 0; i < kQfCh; ++i) {
    const int v = c * 32 * kQfCh + i * 32 + lane;
    float xf[VE];
    qf_unpack<TY>(xv[i], xf);
    uint32_t pk[VE / 4];
#pragma unroll
    for (int j4 = 0; j4 < VE / 4; ++j4) {
      int qi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float y = __fmul_rn(xf[4 * j4 + j], r);
        if (gain != nullptr && v < nvec) y = __fmul_rn(y, __ldg(gain + v * VE + 4 * j4 + j));
        qi[j] = rha_int_small(__fmul_rn(y, sc));
        qs += qi[j];
      }
      pk[j4] = __byte_perm(__byte_perm(qi[0], qi[1], 0x0040), __byte_perm(qi[2], qi[3], 0x0040),
                           0x5410);
    }
    if (rv && v < nvecp) {
      if (VE == 4)
        reinterpret_cast<uint32_t*>(qr)[v] = pk[0];
      else
        reinterpret_cast<uint2*>(qr)[v] = make_uint2(pk[0], pk[VE / 4 - 1]);
    }
  }
  return qs;
}
template <typename TY>
__device__ __forceinline__ void qf_stats_chunk(const uint4 (&xv)[kQfCh], double& s0, double& s1,
                                               float& xm) {
  constexpr int VE = 16 / sizeof(TY);
#pragma unroll
  for (int i = 0; i < kQfCh; ++i) {
    float v[VE];
    qf_unpack<TY>(xv[i], v);
#pragma unroll
    for (int j = 0; j < VE; j += 2) {
      const double d0 = (double)v[j], d1 = (double)v[j + 1];
      s0 = fma(d0, d0, s0);
      s1 = fma(d1, d1, s1);
      xm = fmaxf(xm, fmaxf(fabsf(v[j]), fabsf(v[j + 1])));
    }
  }
}
template <typename TY>
__device__ __forceinline__ float qf_gain_max_chunk(const uint4 (&xv)[kQfCh], int c, int nvec, int lane,
                                                   float r, const float* gain) {
  constexpr int VE = 16 / sizeof(TY);
  float am = 0.0f;
#pragma unroll
  for (int i = 0; i < kQfCh; ++i) {
    const int v = c * 32 * kQfCh + i * 32 + lane;
    if (v >= nvec) continue;
    float xf[VE];
    qf_unpack<TY>(xv[i], xf);
#pragma unroll
    for (int j = 0; j < VE; ++j)
      am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(xf[j], r), __ldg(gain + v * VE + j))));
  }
  return am;
}

// one row by one warp, NCH chunks of kQfCh 16-byte vectors per lane (NCH == 1: the row
// stays in registers between the two passes; else the second pass reloads it, from L1/L2)
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// make this warp's stores of a finished row visible, then count the row in its block
__device__ __forceinline__ void qf_publish(uint32_t* ctr, int row, int lane) {
  fence_proxy_async_global();   // generic -> async proxy (the consumers read q by TMA)
  fence_acq_rel_gpu();
  __syncwarp();
  if (lane == 0) red_release_add(ctr + 1 + (row >> 7), 1u);
}

// One row by one warp, NCH chunks of kQfCh 16-byte vectors per lane (NCH == 1: the row
// stays in registers between the two passes; else the second pass reloads it, from L1/L2).
// The previous row of this warp is published between the passes, when its stores have
// long been issued (the fence then rarely waits).
template <typename TY, int NCH>
__device__ __forceinline__ void qf_row(const GemmArgs& a, int cur, int prev, int lane) {
  constexpr int VE = 16 / sizeof(TY);
  const int K = a.qK, nvec = K / VE, nvecp = a.num_kb * kBK / VE;
  const TY* x = static_cast<const TY*>(a.qx);
  const bool rv = cur < a.M;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)(rv ? cur : 0) * a.qldx);
  int8_t* qr = a.qq + (int64_t)(rv ? cur : 0) * a.qldq;
  double s0 = 0.0, s1 = 0.0;
  float xm = 0.0f;
  uint4 xv[kQfCh];
  qf_load_chunk<TY>(xr, rv, 0, nvec, lane, xv);
  qf_stats_chunk<TY>(xv, s0, s1, xm);
#pragma unroll 1
  for (int c = 1; c < NCH; ++c) {
    uint4 xc[kQfCh];
    qf_load_chunk<TY>(xr, rv, c, nvec, lane, xc);
    qf_stats_chunk<TY>(xc, s0, s1, xm);
  }
  double ss = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  }
  if (prev >= 0) qf_publish(a.qctr, prev, lane);
  const float r = (float)rsqrt(fma(ss, a.qinv_k, (double)a.qeps));
  float amax;
  if (a.qgain == nullptr) {
    amax = __fmul_rn(xm, r);   // max|fl(x r)| = fl(max|x| r): rounding is monotone, r > 0
  } else {
    float am = qf_gain_max_chunk<TY>(xv, 0, nvec, lane, r, a.qgain);
#pragma unroll 1
    for (int c = 1; c < NCH; ++c) {
      uint4 xc[kQfCh];
      qf_load_chunk<TY>(xr, rv, c, nvec, lane, xc);
      am = fmaxf(am, qf_gain_max_chunk<TY>(xc, c, nvec, lane, r, a.qgain));
    }
    amax = warp_max_f32(am);
  }
  const float sc = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
  int qs = 0;
  if (NCH == 1) {
    qs = qf_quant_chunk<TY>(xv, 0, nvec, nvecp, lane, r, sc, a.qgain, qr, rv);
  } else {
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      uint4 xc[kQfCh];
      qf_load_chunk<TY>(xr, rv, c, nvec, lane, xc);
      qs += qf_quant_chunk<TY>(xc, c, nvec, nvecp, lane, r, sc, a.qgain, qr, rv);
    }
  }
  qs = warp_sum_i32(qs);
  if (lane == 0 && rv) {
    a.qdeq[cur] = amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
    a.qqsum[cur] = qs;
  }
}

// warps 2-5: static row assignment, row = gw + i * GW over the grid's quant warps (in row
// order, so blocks complete in the order the tile schedule needs them; every CTA of the
// persistent grid is resident, so no warp waits on a row that cannot progress); the
// rows two ahead are prefetched into L2
template <typename TY, int NCH>
__device__ void qf_quant_loop(const GemmArgs& a, int qw, int lane) {
  const int mpad = a.qmb * 128;
  const int GW = gridDim.x * 4, gw = blockIdx.x * 4 + qw;
  const TY* x = static_cast<const TY*>(a.qx);
  const uint32_t row_bytes = (uint32_t)a.qK * sizeof(TY);
  if (lane == 0)
    for (int j = 0; j < 2; ++j)
      if (gw + j * GW < a.M) prefetch_l2_bulk(x + (int64_t)(gw + j * GW) * a.qldx, row_bytes);
  int prev = -1;
  for (int cur = gw; cur < mpad; cur += GW) {
    if (lane == 0 && cur + 2 * GW < a.M)
      prefetch_l2_bulk(x + (int64_t)(cur + 2 * GW) * a.qldx, row_bytes);
    qf_row<TY, NCH>(a, cur, prev, lane);
    prev = cur;
  }
  if (prev >= 0) qf_publish(a.qctr, prev, lane);
}
template <typename TY>
__device__ void qf_quant_warps(const GemmArgs& a, int qw, int lane) {
  constexpr int VE = 16 / sizeof(TY);
  const int nch = (a.num_kb * kBK / VE + 32 * kQfCh - 1) / (32 * kQfCh);
  switch (nch) {
    case 1: qf_quant_loop<TY, 1>(a, qw, lane); break;
    case 2: qf_quant_loop<TY, 2>(a, qw, lane); break;
    case 3: qf_quant_loop<TY, 3>(a, qw, lane); break;
    default: qf_quant_loop<TY, 4>(a, qw, lane); break;
  }
}

// QF: the fused-quantization variant (a separate instantiation, so the default kernels'
// register allocation is not shaped by the quant warps' code)
template <int BN, bool kPre, typename TY, bool RES = false, int EW = kEpiWarps, bool QF = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR,
              const GemmArgs a) {
  using Cfg = GemmCfg<BN, kPre, RES, EW>;
  static_assert(EW == 8 || (EW == 12 && kPre), "12 drain warps only on the u8 path");
  constexpr int S = Cfg::S;
  constexpr int U = Cfg::U;
  constexpr int NG = Cfg::NG;
  extern __shared__ __align__(1024) uint8_t gsm_raw[];
  // 1024-byte alignment for the swizzle atoms; offset arithmetic keeps the
  // pointer in the shared address space (no generic loads/stores)
  uint8_t* sm = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;                                                    // [S][A_BYTES]
  uint8_t* sB = sA + S * Cfg::A_BYTES;    // kPre: [S][B_BYTES]   else: [U][B_BYTES] unpacked
  uint8_t* sBp = sB + (kPre ? S : U) * Cfg::B_BYTES;                   // packed: [S][BP_BYTES]
  uint8_t* sEpi = sm + Cfg::RING;                                      // [8 warps][2][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + Cfg::EPI_BYTES);
  uint64_t* full = bars;                 // [S] TMA landed
  uint64_t* empty = bars + 8;            // [S] MMA finished with the stage
  uint64_t* unpacked = bars + 16;        // [U] B unpacked
  uint64_t* ufree = bars + 20;           // [U] MMA finished with the unpacked B
  uint64_t* tfull = bars + 24;           // [2] accumulator ready
  uint64_t* tempty = bars + 26;          // [2] accumulator drained
  constexpr int RBW = Cfg::NB > 2 ? Cfg::NB : 2;   // residual barriers per drain warp
  static_assert(28 + RBW * EW + 1 <= 64, "barrier area");
  uint64_t* rbar = bars + 28;            // [EW warps][RBW] residual tile landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28 + RBW * EW);

  const long long t_start = clock64();
#ifdef TERN_TRACE
  trace_mark(a.trace, 0);
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = a.num_kb;
  const int total = a.n_tiles * a.m_tiles * a.ksplit;
  const Epi& e = a.epi;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    if (kPre) tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmO);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int u = 0; u < U; ++u) {
      mbar_init(&unpacked[u], 128);
      mbar_init(&ufree[u], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EW);
    }
    for (int i = 0; i < RBW * EW; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // A, deq, qsum, residual come from earlier kernels: every warp but the
  // producer waits here; the producer first starts the weight (B) loads of its
  // first stages, which do not depend on them (PDL overlap with the previous
  // kernel's tail; for decode batches the weight fetch is the long pole)
  if (warp != 0) pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      auto load_b = [&](int s, int kb, int n0) {
        if (kPre) {
          tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * kBK, n0);
        } else {
          // one contiguous span (K-block-major layout); ragged last tile shorter
          const uint32_t bbytes = (uint32_t)min(BN, a.n_rows - n0) * 32u;
          bulk_load(sBp + s * Cfg::BP_BYTES, a.codes + ((int64_t)kb * a.n_rows + n0) * 8, bbytes,
                    &full[s]);
        }
      };
      auto b_bytes = [&](int n0) -> uint32_t {
        return kPre ? (uint32_t)Cfg::B_BYTES : (uint32_t)min(BN, a.n_rows - n0) * 32u;
      };
      // weights of the first unit's first S k-blocks before the dependency wait
      uint32_t npre = 0;
      if ((int)blockIdx.x < total) {
        const int t = blockIdx.x, tile = t / a.ksplit, sp = t % a.ksplit;
        const int n0 = (tile % a.n_tiles) * BN;
        const int kb0 = sp * a.kb_per, kb1 = min(nk, kb0 + a.kb_per);
        for (int kb = kb0; kb < kb1 && npre < (uint32_t)S; ++kb, ++npre) {
          mbar_expect_tx(&full[npre], b_bytes(n0));
          load_b((int)npre, kb, n0);
        }
      }
      pdl_wait();
#ifdef TERN_TRACE
      trace_mark(a.trace, 1);
#endif
      uint32_t g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int tile = t / a.ksplit, sp = t % a.ksplit;
        const int m0 = (tile / a.n_tiles) * kBM, n0 = (tile % a.n_tiles) * BN;
        const int kb1 = min(nk, (sp + 1) * a.kb_per);
        if constexpr (QF) {   // fused quantization: this tile's A rows must be published
          qf_wait_block(a.qctr, m0 >> 7);
          fence_proxy_async_global();
        }
        for (int kb = sp * a.kb_per; kb < kb1; ++kb, ++g) {
          const int s = g % S;
          if (g >= (uint32_t)S) pwait(&empty[s], ((g / S) - 1) & 1, a.prof, 0);
          if (g < npre) {   // B already in flight
            mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES);
            tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * kBK, m0);
          } else {
            mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + b_bytes(n0));
            tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * kBK, m0);
            load_b(s, kb, n0);
          }
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
        pwait(&tempty[acc], ((it >> 1) & 1) ^ 1, a.prof, 1);
        tc_fence_after();
        const uint32_t d_addr = tmem_base + acc * BN;
        const int sp = t % a.ksplit;
        const int kb0 = sp * a.kb_per, kb1 = min(nk, kb0 + a.kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % S;
          uint32_t b_addr;
          if (kPre) {
            pwait(&full[s], (g / S) & 1, a.prof, 2);
            b_addr = smem_u32(sB + s * Cfg::B_BYTES);
          } else {
            const int u = g % U;
            pwait(&unpacked[u], (g / U) & 1, a.prof, 2);
            b_addr = smem_u32(sB + u * Cfg::B_BYTES);
          }
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * Cfg::A_BYTES);
#pragma unroll
          for (int kk = 0; kk < kBK / 32; ++kk)
            mma_i8(d_addr, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                   idesc, ((kb - kb0) | kk) != 0);
          mma_commit(&empty[s]);
          if (!kPre) mma_commit(&ufree[g % U]);
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp < Cfg::EW0) {
    // ---------------- unpack (warps 2-5, packed path): 2-bit fields -> u8 e, SW128 K-major
    // (u8 path: the fused quantization of A when requested)
    if (kPre && EW == kEpiWarps) {
      if constexpr (QF) qf_quant_warps<TY>(a, warp - 2, lane);
    } else if (!kPre) {
      const int tid = threadIdx.x - 64;
      const bool pt = tid == 0;
      uint32_t g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int sp = t % a.ksplit;
        const int kb1 = min(nk, (sp + 1) * a.kb_per);
        for (int kb = sp * a.kb_per; kb < kb1; ++kb, ++g) {
          const int s = g % S, u = g % (U > 0 ? U : 1);
          if (g >= (uint32_t)U) pwait(&ufree[u], ((g / U) - 1) & 1, pt ? a.prof : nullptr, 3);
          pwait(&full[s], (g / S) & 1, pt ? a.prof : nullptr, 4);
          const uint32_t* bp = reinterpret_cast<const uint32_t*>(sBp + s * Cfg::BP_BYTES);
          uint8_t* bu = sB + u * Cfg::B_BYTES;
          // thread owns word w = tid%8 of rows tid/8 + 16 j: its swizzled 16-byte
          // chunk offset inside a row is the same for every j
          const int r0 = tid >> 3, w = tid & 7;
          const uint32_t* src = bp + tid;
          uint8_t* dst = bu + r0 * 128 + ((w ^ (r0 & 7)) << 4);
#pragma unroll
          for (int j = 0; j < BN / 16; ++j) {
            const uint32_t word = src[j * 128];
            uint4 v;
            v.x = word & 0x03030303u;
            v.y = (word >> 2) & 0x03030303u;
            v.z = (word >> 4) & 0x03030303u;
            v.w = (word >> 6) & 0x03030303u;
            *reinterpret_cast<uint4*>(dst + j * 2048) = v;
          }
          fence_proxy_async_smem();
          mbar_arrive(&unpacked[u]);
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 6-13): two warps per TMEM lane quadrant
    const int ew = warp - Cfg::EW0;
    const int quad = warp & 3;          // TMEM lanes [32*quad, 32*quad+32)
    const int half = ew >> 2;           // which of the quadrant's NG chunk streams this warp takes
    uint8_t* bufs = sEpi + ew * Cfg::NB * kEpiBuf;
    uint64_t* rb = rbar + ew * RBW;
    const bool lead = lane == 0;
    const bool legacy = e.acc != nullptr || e.kind == EPI_NONE;   // tap / parity path
    const int nseg = e.n_seg;
    const float msc0 = __ldg(e.scales), msc1 = nseg > 1 ? __ldg(e.scales + 1) : 0.0f;
    const float msc2 = nseg > 2 ? __ldg(e.scales + 2) : 0.0f;
    uint32_t it = 0, nchunk = 0;
    uint32_t rphase[2] = {0, 0};
    if (RES) {
      // residual epilogue (EPI_RESID, no taps, no split-K): chunk k of this warp (over its
      // tiles in order) reads its residual into staging buffer k % NB; the loads run NB - 1
      // chunks ahead of the compute, so their HBM latency hides behind NB - 1 chunks
      constexpr int NBR = Cfg::NB;
      // the first chunk of this warp at or after (t_, c_) (both updated to it): its tile
      // row / column
      auto chunk_at = [&](int& t_, int& c_, int& row0_, int& col0_) -> bool {
        for (; t_ < total; t_ += gridDim.x, c_ = half) {
          const int tile_ = t_ / a.ksplit;
          const int m0_ = (tile_ / a.n_tiles) * kBM, n0_ = (tile_ % a.n_tiles) * BN;
          for (; c_ < BN / 32; c_ += NG)
            if (n0_ + c_ * 32 < a.n_rows) {
              row0_ = m0_ + quad * 32;
              col0_ = n0_ + c_ * 32;
              return true;
            }
        }
        return false;
      };
      int ti = blockIdx.x, ci = half;   // issue cursor: the next chunk whose residual to load
      uint32_t nissued = 0;
      auto issue_next = [&]() {
        int nr0, nc0;
        if (chunk_at(ti, ci, nr0, nc0)) {
          const int bi = nissued % NBR;
          mbar_arrive_expect_tx(&rb[bi], 32 * 32 * sizeof(TY));
          tma_load_2d(bufs + bi * kEpiBuf, &tmR, &rb[bi], nc0, nr0);
          ++nissued;
          ci += NG;
        }
      };
      if (lead)
        for (int j = 0; j < NBR - 1; ++j) issue_next();
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const uint32_t acc = it & 1;
        const int tile = t / a.ksplit;
        const int m0 = (tile / a.n_tiles) * kBM, n0 = (tile % a.n_tiles) * BN;
        pwait(&tfull[acc], (it >> 1) & 1, (ew == 0 && lead) ? a.prof : nullptr, 5);
        tc_fence_after();
        const int row0 = m0 + quad * 32;
        const int row = row0 + lane;
        const bool rv = row < a.M;
        float deq;
        int qsum;
        if constexpr (QF) {   // deq / qsum written in this kernel: acquire, then L2 loads
          qf_wait_block(a.qctr, m0 >> 7);
          deq = rv ? __ldcg(a.deq + row) : 0.0f;
          qsum = rv ? __ldcg(a.qsum + row) : 0;
        } else {
          deq = rv ? __ldg(a.deq + row) : 0.0f;
          qsum = rv ? __ldg(a.qsum + row) : 0;
        }
        const uint32_t trow = tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
        for (int c = half; c < BN / 32; c += NG) {
          const int col0 = n0 + c * 32;
          if (col0 >= a.n_rows) continue;
          uint32_t v[32];
          tmem_ld32(trow + c * 32, v);
          const int buf = nchunk % NBR;
          uint8_t* sb = bufs + buf * kEpiBuf;
          // the residual NB - 1 chunks ahead, into the buffer of the previous chunk once
          // its store has read it
          if (lead) {
            bulk_wait_read<0>();
            issue_next();
          }
          tmem_ld_wait();
          const float sc = __fmul_rn(deq, msc0);
          float o[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float x = __fmul_rn(i2f_small((int)v[j] - qsum), sc);
            if (e.bias) x = __fadd_rn(x, __ldg(e.bias + col0 + j));
            o[j] = storage_round<TY>(x);
          }
          mbar_wait(&rb[buf], (nchunk / NBR) & 1);
          float xr[32];
          stg_read_row<TY>(sb, lane, xr);
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __fadd_rn(xr[j], o[j]);
          __syncwarp();   // all lanes read their residual rows before they are overwritten
          stg_write_row<TY>(sb, lane, o);
          fence_proxy_async_smem();
          __syncwarp();
          if (lead) {
            tma_store_2d(&tmO, sb, col0, row0);   // rows >= M / cols >= n clipped by TMA
            bulk_commit();
          }
          ++nchunk;
        }
        tc_fence_before();
        __syncwarp();
        if (lead) mbar_arrive(&tempty[acc]);
      }
    }
    for (int t = blockIdx.x; t < (RES ? 0 : total); t += gridDim.x, ++it) {
      const uint32_t acc = it & 1;
      const int tile = t / a.ksplit;
      const int m0 = (tile / a.n_tiles) * kBM, n0 = (tile % a.n_tiles) * BN;
      pwait(&tfull[acc], (it >> 1) & 1, (ew == 0 && lead) ? a.prof : nullptr, 5);
      tc_fence_after();
      const int row0 = m0 + quad * 32;
      if (a.part) {
        // split-K / finalize mode: this K slice's raw sums go to part[sp][M][n_rows]
        // (coalesced through the staging tile); k_splitk_epi sums the slices in a
        // fixed order (exact int32) and applies the epilogue
        int32_t* slice = a.part + (int64_t)(t % a.ksplit) * a.M * a.n_rows;
        int* si = reinterpret_cast<int*>(bufs);
        for (int c = half; c < BN / 32; c += NG) {
          const int col0 = n0 + c * 32;
          if (col0 >= a.n_rows) continue;
          uint32_t v[32];
          tmem_ld32(trow_base(tmem_base, acc, BN, quad) + c * 32, v);
          tmem_ld_wait();
          if (lead) bulk_wait_read<0>();   // staging tile free of pending stores
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) si[lane * 32 + (j ^ lane)] = (int)v[j];   // XOR swizzle
          __syncwarp();
          for (int r = 0; r < 32; ++r)
            if (row0 + r < a.M && col0 + lane < a.n_rows)
              slice[(int64_t)(row0 + r) * a.n_rows + col0 + lane] = si[r * 32 + (lane ^ r)];
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lead) mbar_arrive(&tempty[acc]);
        continue;
      }
      const int row = row0 + lane;
      const bool rv = row < a.M;
      float deq;
      int qsum;
      if constexpr (QF) {   // deq / qsum written in this kernel: acquire, then L2 loads
        qf_wait_block(a.qctr, m0 >> 7);
        deq = rv ? __ldcg(a.deq + row) : 0.0f;
        qsum = rv ? __ldcg(a.qsum + row) : 0;
      } else {
        deq = rv ? __ldg(a.deq + row) : 0.0f;
        qsum = rv ? __ldg(a.qsum + row) : 0;
      }
      const uint32_t trow = tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16);
      const bool swig = e.kind == EPI_SWIGLU;
      const int nch = swig ? BN / 64 : BN / 32;   // chunks (or gate/up pairs) per tile
#pragma unroll 1
      for (int c = half; c < nch; c += NG) {
        // column bookkeeping of this chunk
        int col0, out_col0;
        if (swig) {
          col0 = n0 + (c >> 1) * 128 + (c & 1) * 32;
          out_col0 = (col0 / 128) * 64 + (c & 1) * 32;
        } else {
          col0 = n0 + c * 32;
          out_col0 = e.kind == EPI_FCG ? col0 : (col0 / (kSegRows * nseg)) * kSegRows + (col0 % kSegRows);
        }
        if (col0 >= a.n_rows || (swig && out_col0 >= e.n_out)) continue;
        uint32_t v[32], vu[32];
        tmem_ld32(trow + (col0 - n0), v);
        if (swig) tmem_ld32(trow + (col0 - n0) + 64, vu);
        if (legacy) {
          tmem_ld_wait();
          int* si = reinterpret_cast<int*>(bufs);
          if (lead) bulk_wait_read<0>();   // staging buffers free of pending stores
          __syncwarp();
          if (e.acc) {
            acc_tap_chunk(e, a, si, lane, row0, col0, qsum, v);
            if (swig) acc_tap_chunk(e, a, si, lane, row0, col0 + 64, qsum, vu);
          }
          if (e.kind == EPI_NONE) continue;
        }
        const int buf = Cfg::NB == 2 ? (nchunk & 1) : 0;
        uint8_t* sb = bufs + buf * kEpiBuf;
        // the TMA store that last read this buffer (NB chunks ago) must be done
        if (lead) {
          if (Cfg::NB == 2) bulk_wait_read<1>();
          else bulk_wait_read<0>();
        }
        __syncwarp();
        const bool resid = e.kind == EPI_RESID;
        if (resid && lead) {
          mbar_arrive_expect_tx(&rb[buf], 32 * 32 * sizeof(TY));
          tma_load_2d(sb, &tmR, &rb[buf], out_col0, row0);
        }
        if (!legacy) tmem_ld_wait();
        // dequantize (a5) + functor, thread = row
        const int seg = (col0 / kSegRows) % nseg;
        const int rr0 = (col0 / (kSegRows * nseg)) * kSegRows + (col0 % kSegRows);
        const float msc = seg == 0 ? msc0 : (seg == 1 ? msc1 : msc2);
        const float sc = __fmul_rn(deq, msc);
        float o[32];
        if (swig) {
          const float scu = __fmul_rn(deq, msc1);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float g0 = storage_round<TY>(__fmul_rn(i2f_small((int)v[j] - qsum), sc));
            const float g1 = storage_round<TY>(__fmul_rn(i2f_small((int)v[j + 1] - qsum), sc));
            const float u0 = storage_round<TY>(__fmul_rn(i2f_small((int)vu[j] - qsum), scu));
            const float u1 = storage_round<TY>(__fmul_rn(i2f_small((int)vu[j + 1] - qsum), scu));
            float s0, s1;
            sigmoid2(g0, g1, s0, s1);
            o[j] = __fmul_rn(__fmul_rn(g0, s0), u0);   // SwiGLU p = SiLU(g) u
            o[j + 1] = __fmul_rn(__fmul_rn(g1, s1), u1);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float x = __fmul_rn(i2f_small((int)v[j] - qsum), sc);
            if (e.bias) x = __fadd_rn(x, __ldg(e.bias + seg * e.n_out + rr0 + j));
            o[j] = storage_round<TY>(x);
          }
        }
        if (resid) {
          mbar_wait(&rb[buf], rphase[buf]);
          rphase[buf] ^= 1;
          float xr[32];
          stg_read_row<TY>(sb, lane, xr);
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __fadd_rn(xr[j], o[j]);
          __syncwarp();   // all lanes read their residual rows before they are overwritten
        }
        stg_write_row<TY>(sb, lane, o);
        fence_proxy_async_smem();
        __syncwarp();
        if (lead) {
          // rows >= M / cols >= n clipped by TMA
          if (e.kind == EPI_RESID_RED) tma_reduce_add_2d(&tmO, sb, out_col0, row0);
          else tma_store_2d(&tmO, sb, out_col0, row0);
          bulk_commit();
        }
        ++nchunk;
      }
      tc_fence_before();
      __syncwarp();
      if (lead) mbar_arrive(&tempty[acc]);
    }
    if (lead) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
#ifdef TERN_TRACE
    if (lane == 0 && a.trace && blockIdx.x < 1024) a.trace[blockIdx.x * 16 + 2] = gtimer();
#endif
  }
  if (a.prof && threadIdx.x == 0) a.prof[blockIdx.x * 8 + 7] = clock64() - t_start;
}

// ----------------------------------------------------------------- 2-SM tiles (cta_group::2)
// A CTA pair (a cluster of 2 on one TPC) computes a 256 x 256 output tile: each CTA loads
// its own 128 rows of A (q) and its 128-row half of B (the u8 weights) per k-block, the
// leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256) reading both CTAs' shared
// memory, and the accumulator rows land in each CTA's own TMEM.  Per CTA and k-block that
// is 32 KB of TMA writes and 32 KB of MMA operand reads instead of 48 + 48 KB for a 1-CTA
// 128 x 256 tile -- shared-memory bandwidth is the binding resource of these GEMMs
// (TERN_GEMM_PROF: the MMA of a 1-CTA c2 tile takes ~3x its issue time) -- and the freed
// space buys a 6-stage ring.  Barriers: the k-block "full" barrier lives in the leader and
// counts one arrival (with its transaction bytes) per CTA, both CTAs' TMA loads complete on
// it; "empty" and "accumulator full" are signalled to both CTAs by multicast commits;
// "accumulator empty" lives in the leader and counts the 8 drain warps of both CTAs.
constexpr int k2Tile = 128 * kBK;   // A or B half-tile bytes per CTA per stage
// NB staging tiles per drain warp: 1 with a 6-stage ring, or 2 (stores overlap the next
// chunk, the residual of chunk k+1 loads during chunk k) with a 5-stage ring
template <int NB> struct Cfg2 {
  static constexpr int S = NB == 2 ? 5 : 6;
  static constexpr int SMEM = S * 2 * k2Tile + kEpiWarps * NB * kEpiBuf + 1024 + 512;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void cl_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
// TMA load into this CTA's shared memory completing on an mbarrier of the pair (the leader's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit of the pair's MMAs, arriving on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <typename TY, int NB, bool QF = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR,
               const GemmArgs a) {
  constexpr int kS2 = Cfg2<NB>::S;
  extern __shared__ __align__(1024) uint8_t gsm_raw[];
  uint8_t* sm = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;                          // [kS2][16 KB] this CTA's 128 rows of A (SW128)
  uint8_t* sB = sA + kS2 * k2Tile;           // [kS2][16 KB] this CTA's half of B (SW128)
  uint8_t* sEpi = sB + kS2 * k2Tile;         // [8 warps][NB][4 KB] staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + kEpiWarps * NB * kEpiBuf);
  uint64_t* full = bars;          // [kS2] (the leader's is the one used)
  uint64_t* empty = bars + 8;     // [kS2]
  uint64_t* tfull = bars + 16;    // [2]
  uint64_t* tempty = bars + 18;   // [2] (the leader's)
  uint64_t* rbar = bars + 20;     // [8 warps][2] residual tile landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 40);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int total = a.n_tiles * a.m_tiles;   // 256 x 256 tiles
  const int nk = a.num_kb;
  const Epi& e = a.epi;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmO);
    for (int s = 0; s < kS2; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();   // both CTAs' barriers initialised before any remote arrival
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp != 0) pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs): own A rows, own half of B
    if (lane == 0) {
      auto fullL = [&](int s) { return mapa_rank(&full[s], 0); };
      uint32_t npre = 0;
      if (cid < total) {   // weights of the first stages before the dependency wait
        const int n0 = (cid % a.n_tiles) * 256 + (int)rank * 128;
        for (int kb = 0; kb < nk && npre < (uint32_t)kS2; ++kb, ++npre) {
          cl_expect_tx(fullL((int)npre), k2Tile);
          tma_load_2d_pair(sB + npre * k2Tile, &tmB, fullL((int)npre), kb * kBK, n0);
        }
      }
      pdl_wait();
      uint32_t g = 0;
      for (int t = cid; t < total; t += ncl) {
        const int m0 = (t / a.n_tiles) * 256 + (int)rank * 128;
        const int n0 = (t % a.n_tiles) * 256 + (int)rank * 128;
        if constexpr (QF) {   // fused quantization: this CTA's 128 A rows must be published
          qf_wait_block(a.qctr, m0 >> 7);
          fence_proxy_async_global();
        }
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % kS2;
          if (g >= (uint32_t)kS2) mbar_wait(&empty[s], ((g / kS2) - 1) & 1);
          if (g < npre) {
            cl_arrive_expect_tx(fullL(s), k2Tile);
            tma_load_2d_pair(sA + s * k2Tile, &tmA, fullL(s), kb * kBK, m0);
          } else {
            cl_arrive_expect_tx(fullL(s), 2 * k2Tile);
            tma_load_2d_pair(sA + s * k2Tile, &tmA, fullL(s), kb * kBK, m0);
            tma_load_2d_pair(sB + s * k2Tile, &tmB, fullL(s), kb * kBK, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (the leader's lane 0)
    if (leader && lane == 0) {
      // kind::i8: D s32, A s8, B u8, both K-major, M = 256 (the pair), N = 256
      const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      uint32_t g = 0, it = 0;
      for (int t = cid; t < total; t += ncl, ++it) {
        const uint32_t acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_addr = tmem_base + acc * 256;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % kS2;
          mbar_wait(&full[s], (g / kS2) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * k2Tile), b_addr = smem_u32(sB + s * k2Tile);
#pragma unroll
          for (int kk = 0; kk < kBK / 32; ++kk)
            mma_i8_pair(d_addr, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                        idesc, (kb | kk) != 0);
          mma_commit_pair(&empty[s]);
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue (warps 6-13 of both CTAs): this CTA's 128 rows x 256 columns
    const int ew = warp - kEpiWarp0;
    const int quad = warp & 3;
    const int half = ew >> 2;
    uint8_t* bufs = sEpi + ew * NB * kEpiBuf;
    uint64_t* rb = rbar + ew * 2;
    const bool lead = lane == 0;
    const int nseg = e.n_seg;
    const bool swig = e.kind == EPI_SWIGLU, resid = e.kind == EPI_RESID;
    const int nch = swig ? 256 / 64 : 256 / 32;
    const float msc0 = __ldg(e.scales), msc1 = nseg > 1 ? __ldg(e.scales + 1) : 0.0f;
    const float msc2 = nseg > 2 ? __ldg(e.scales + 2) : 0.0f;
    const uint32_t temptyL = mapa_rank(&tempty[0], 0);
    // column bookkeeping of chunk c of a tile at column n0
    auto cols = [&](int n0, int c, int& col0, int& out_col0) -> bool {
      if (swig) {
        col0 = n0 + (c >> 1) * 128 + (c & 1) * 32;
        out_col0 = (col0 / 128) * 64 + (c & 1) * 32;
      } else {
        col0 = n0 + c * 32;
        out_col0 = e.kind == EPI_FCG ? col0 : (col0 / (kSegRows * nseg)) * kSegRows + (col0 % kSegRows);
      }
      return col0 < a.n_rows && !(swig && out_col0 >= e.n_out);
    };
    // the first valid chunk of this warp at or after (tile t_, chunk c_): residual coordinates
    auto next_chunk = [&](int t_, int c_, int& r0_, int& oc0_) -> bool {
      for (; t_ < total; t_ += ncl, c_ = half) {
        const int m0_ = (t_ / a.n_tiles) * 256 + (int)rank * 128, n0_ = (t_ % a.n_tiles) * 256;
        for (; c_ < nch; c_ += 2) {
          int col0_;
          if (cols(n0_, c_, col0_, oc0_)) {
            r0_ = m0_ + quad * 32;
            return true;
          }
        }
      }
      return false;
    };
    uint32_t it = 0, nchunk = 0;
    uint32_t rphase[2] = {0, 0};
    if (NB == 2 && resid && lead) {   // chunk 0's residual
      int r0_, oc0_;
      if (next_chunk(cid, half, r0_, oc0_)) {
        mbar_arrive_expect_tx(&rb[0], 32 * 32 * sizeof(TY));
        tma_load_2d(bufs, &tmR, &rb[0], oc0_, r0_);
      }
    }
    for (int t = cid; t < total; t += ncl, ++it) {
      const uint32_t acc = it & 1;
      const int m0 = (t / a.n_tiles) * 256 + (int)rank * 128, n0 = (t % a.n_tiles) * 256;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row0 = m0 + quad * 32;
      const int row = row0 + lane;
      const bool rv = row < a.M;
      float deq;
      int qsum;
      if constexpr (QF) {   // deq / qsum written in this kernel: acquire, then L2 loads
        qf_wait_block(a.qctr, m0 >> 7);
        deq = rv ? __ldcg(a.deq + row) : 0.0f;
        qsum = rv ? __ldcg(a.qsum + row) : 0;
      } else {
        deq = rv ? __ldg(a.deq + row) : 0.0f;
        qsum = rv ? __ldg(a.qsum + row) : 0;
      }
      const uint32_t trow = tmem_base + acc * 256 + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int c = half; c < nch; c += 2) {
        int col0, out_col0;
        if (!cols(n0, c, col0, out_col0)) continue;
        uint32_t v[32], vu[32];
        tmem_ld32(trow + (col0 - n0), v);
        if (swig) tmem_ld32(trow + (col0 - n0) + 64, vu);
        const int buf = NB == 2 ? (nchunk & 1) : 0;
        uint8_t* sb = bufs + buf * kEpiBuf;
        if (NB == 2 && resid) {
          // the next chunk's residual into the other buffer once its last store read it
          if (lead) {
            bulk_wait_read<0>();
            int r0_, oc0_;
            if (next_chunk(c + 2 < nch ? t : t + ncl, c + 2 < nch ? c + 2 : half, r0_, oc0_)) {
              mbar_arrive_expect_tx(&rb[buf ^ 1], 32 * 32 * sizeof(TY));
              tma_load_2d(bufs + (buf ^ 1) * kEpiBuf, &tmR, &rb[buf ^ 1], oc0_, r0_);
            }
          }
        } else {
          if (lead) {   // the store that last read this buffer (NB chunks ago) is done
            if (NB == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          if (resid && lead) {
            mbar_arrive_expect_tx(&rb[buf], 32 * 32 * sizeof(TY));
            tma_load_2d(sb, &tmR, &rb[buf], out_col0, row0);
          }
        }
        tmem_ld_wait();
        const int seg = (col0 / kSegRows) % nseg;
        const int rr0 = (col0 / (kSegRows * nseg)) * kSegRows + (col0 % kSegRows);
        const float msc = seg == 0 ? msc0 : (seg == 1 ? msc1 : msc2);
        const float sc = __fmul_rn(deq, msc);
        float o[32];
        if (swig) {
          const float scu = __fmul_rn(deq, msc1);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float g0 = storage_round<TY>(__fmul_rn(i2f_small((int)v[j] - qsum), sc));
            const float g1 = storage_round<TY>(__fmul_rn(i2f_small((int)v[j + 1] - qsum), sc));
            const float u0 = storage_round<TY>(__fmul_rn(i2f_small((int)vu[j] - qsum), scu));
            const float u1 = storage_round<TY>(__fmul_rn(i2f_small((int)vu[j + 1] - qsum), scu));
            float s0, s1;
            sigmoid2(g0, g1, s0, s1);
            o[j] = __fmul_rn(__fmul_rn(g0, s0), u0);   // SwiGLU p = SiLU(g) u
            o[j + 1] = __fmul_rn(__fmul_rn(g1, s1), u1);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float x = __fmul_rn(i2f_small((int)v[j] - qsum), sc);
            if (e.bias) x = __fadd_rn(x, __ldg(e.bias + seg * e.n_out + rr0 + j));
            o[j] = storage_round<TY>(x);
          }
        }
        if (resid) {
          mbar_wait(&rb[buf], rphase[buf]);
          rphase[buf] ^= 1;
          float xr[32];
          stg_read_row<TY>(sb, lane, xr);
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __fadd_rn(xr[j], o[j]);
          __syncwarp();
        }
        stg_write_row<TY>(sb, lane, o);
        fence_proxy_async_smem();
        __syncwarp();
        if (lead) {
          // rows >= M / cols >= n clipped by TMA
          if (e.kind == EPI_RESID_RED) tma_reduce_add_2d(&tmO, sb, out_col0, row0);
          else tma_store_2d(&tmO, sb, out_col0, row0);
          bulk_commit();
        }
        ++nchunk;
      }
      tc_fence_before();
      __syncwarp();
      if (lead) cl_arrive(temptyL + acc * 8);   // the leader's tempty[acc]
    }
    if (lead) bulk_wait<0>();
  } else if (QF && warp >= 2) {
    // ---------------- fused quantization of A (warps 2-5 of both CTAs)
    qf_quant_warps<TY>(a, warp - 2, lane);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();   // the pair is done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
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

bool make_map_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
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

template <int BN, bool kPre, typename TY, bool RES = false, int EW = kEpiWarps, bool QF = false>
static cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to,
                               const CUtensorMap& tr, const GemmArgs& a, cudaStream_t s) {
  using Cfg = GemmCfg<BN, kPre, RES, EW>;
  auto kern = k_gemm_tc<BN, kPre, TY, RES, EW, QF>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int total = a.n_tiles * a.m_tiles * a.ksplit;
  int grid = total < num_sms ? total : num_sms;
  // balanced persistent grid: with few tile waves, the fewest CTAs that keep the same number of
  // waves (c2 o-projection: 512 tiles -> 128 CTAs x 4 instead of 148 CTAs x 3..4; the makespan
  // in tiles is the same and the HBM-bound drains contend less: 38.8 -> 37.8 us).  With many
  // waves it measured slower (c2 gate|up, 20 waves: 97.2 -> 99.7 us), so only up to 8 waves.
  // TERN_GEMM_BAL=0 turns it off, 2 applies it to every grid (debug).
  static const int bal = getenv("TERN_GEMM_BAL") ? atoi(getenv("TERN_GEMM_BAL")) : 1;
  if (bal && total > num_sms && a.ksplit == 1 && a.part == nullptr) {   // not the split-K slices
    const int waves = (total + num_sms - 1) / num_sms;
    if (waves <= 8 || bal == 2) grid = (total + waves - 1) / waves;
  }
  static unsigned long long* dprof = nullptr;
  static const bool prof_on = getenv("TERN_GEMM_PROF") != nullptr;
  GemmArgs aa = a;
#ifdef TERN_TRACE
  aa.trace = trace_slot(TERN_K_GEMM, grid);
#endif
  if (prof_on) {  // debug only: per-site wait cycles, printed after a synchronous run
    if (!dprof) cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * 1024);
    cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * 8 * 1024, s);
    aa.prof = dprof;
  }
  cudaError_t lerr = launch_pdl(kern, dim3(grid), dim3(kGemmThreads), Cfg::SMEM, s, ta, tb, to, tr, aa);
  if (lerr != cudaSuccess) return lerr;
  if (prof_on) {
    static unsigned long long h[8 * 1024];
    cudaMemcpyAsync(h, dprof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double sum[8] = {0};
    for (int b = 0; b < grid; ++b)
      for (int i = 0; i < 8; ++i) sum[i] += (double)h[b * 8 + i] / grid;
    fprintf(stderr,
            "[gemm prof] M=%d n=%d K=%d BN=%d pre=%d kind=%d tiles=%d | total=%.0f prod.empty=%.0f "
            "mma.tempty=%.0f mma.B=%.0f unp.ufree=%.0f unp.full=%.0f epi.tfull=%.0f\n",
            a.M, a.n_rows, a.num_kb * 128, BN, (int)kPre, a.epi.kind, total, sum[7], sum[0],
            sum[1], sum[2], sum[3], sum[4], sum[5]);
  }
  return cudaGetLastError();
}

template <typename TY, int NB, bool QF = false>
static cudaError_t gemm2_launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to,
                                const CUtensorMap& tr, const GemmArgs& a, cudaStream_t s) {
  auto kern = k_gemm_2sm<TY, NB, QF>;
  constexpr int k2Smem = Cfg2<NB>::SMEM;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, k2Smem);
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
  int grid = 2 * total < num_sms ? 2 * total : num_sms;
  grid &= ~1;
  // balanced grid as in gemm_launch (c2 down: 256 pair tiles -> 64 pairs x 4; 54.0 -> 51.7 us)
  static const int bal = getenv("TERN_GEMM_BAL") ? atoi(getenv("TERN_GEMM_BAL")) : 1;
  if (bal && 2 * total > grid) {   // the fewest CTA pairs with the same number of tile waves
    const int pairs = grid / 2, waves = (total + pairs - 1) / pairs;
    if (waves <= 8 || bal == 2) grid = 2 * ((total + waves - 1) / waves);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = k2Smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;   // the CTA pair
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, to, tr, a);
}

template <bool kPre, typename TY>
static cudaError_t gemm_dispatch_bn(int BN, const CUtensorMap& ta, const CUtensorMap& tb,
                                    const CUtensorMap& to, const CUtensorMap& tr,
                                    const GemmArgs& a, cudaStream_t s) {
  // the residual-prefetch epilogue (GemmCfg RES) for the u8 256-wide residual GEMMs
  static const int res_on = getenv("TERN_GEMM_RES") ? atoi(getenv("TERN_GEMM_RES")) : 1;   // debug
  // (short K only: with K >= 2816 the 4th ring stage matters more -- measured c2 o 49.0 ->
  // 37.7 us, c3 o 141 -> 124 us; c2 down 57.7 -> 61.9 us with it, so down keeps S = 4)
  if (BN == 256 && kPre && res_on && a.epi.kind == EPI_RESID && a.epi.acc == nullptr &&
      a.part == nullptr && a.ksplit == 1 && a.num_kb <= 16)
    return a.qctr ? gemm_launch<256, kPre, TY, true, kEpiWarps, kPre>(ta, tb, to, tr, a, s)
                  : gemm_launch<256, kPre, TY, true>(ta, tb, to, tr, a, s);
  // (12 drain warps measured slower on c2 gate|up: 96 -> 103 us; TERN_GEMM_EW12=1 turns it on)
  static const int ew12 = getenv("TERN_GEMM_EW12") ? atoi(getenv("TERN_GEMM_EW12")) : 0;   // debug
  if constexpr (kPre) {
    if (BN == 256 && ew12 && a.epi.kind == EPI_SWIGLU && a.epi.acc == nullptr &&
        a.part == nullptr && a.ksplit == 1 && a.qctr == nullptr)
      return gemm_launch<256, true, TY, false, 12>(ta, tb, to, tr, a, s);
  }
  if (a.qctr)   // (only on the u8 path: launch_gemm's gemm_qfuse_ok requires e8)
    return BN == 256 ? gemm_launch<256, kPre, TY, false, kEpiWarps, kPre>(ta, tb, to, tr, a, s)
                     : gemm_launch<128, kPre, TY, false, kEpiWarps, kPre>(ta, tb, to, tr, a, s);
  return BN == 256 ? gemm_launch<256, kPre, TY>(ta, tb, to, tr, a, s)
                   : gemm_launch<128, kPre, TY>(ta, tb, to, tr, a, s);
}

// ----------------------------------------------------------------- split-K epilogue
// The epilogue of a split-K (or small-M) GEMM: sums the K slices' int32 partials
// in slice order (exact), then the same arithmetic as the tensor-core epilogue
// (a5 dequant, R1-R3 storage rounding, SwiGLU / MLGRU step with the paired
// sigmoid).  One thread per (row, pair of output columns or channels).
template <typename TY>
__global__ void k_splitk_epi(const int32_t* __restrict__ part, int ksplit, int M, int n_rows,
                             const float* __restrict__ deq, const int32_t* __restrict__ qsum,
                             const Epi e, unsigned long long* trace) {
  trace_mark(trace, 0);
  pdl_wait();                 // the GEMM's partial sums
  pdl_launch_dependents();
  trace_mark(trace, 1);
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool chan = e.kind == EPI_SWIGLU || e.kind == EPI_MLGRU;   // per logical channel
  const int ncol = chan ? e.n_out : (e.kind == EPI_FCG ? n_rows : e.n_out);
  const int npair = (ncol + 1) / 2;
  if (idx >= (int64_t)M * npair) {
    trace_mark(trace, 2);   // (thread 0 of the last CTA may have no pair)
    return;
  }
  const int m = (int)(idx / npair), c = (int)(idx % npair) * 2;
  const float dq = __ldg(deq + m);
  const int qs = __ldg(qsum + m);
  const int64_t sl = (int64_t)M * n_rows;
  // int32 sums over the K slices of packed columns (col, col+1) of row m, minus
  // qsum: one 8-byte load per slice (n_rows and col are even)
  const int* prow = part + (int64_t)m * n_rows;
  auto dqv = [&](int acc, int seg, int r) {
    float o = __fmul_rn(i2f_small(acc), __fmul_rn(dq, __ldg(e.scales + seg)));
    if (e.bias) o = __fadd_rn(o, __ldg(e.bias + seg * e.n_out + r));
    return storage_round<TY>(o);
  };
  TY* out = static_cast<TY*>(e.out);
  if (chan) {   // n_out even: channels c, c+1 share a 64-row group (c even)
    const int nseg = e.kind == EPI_SWIGLU ? 2 : 3;
    int2 a[3] = {make_int2(0, 0), make_int2(0, 0), make_int2(0, 0)};
    // four slices' loads issued together per round (a runtime trip count would otherwise
    // serialise one L2 round trip per slice); the sums stay in slice order (exact anyway)
    for (int k0 = 0; k0 < ksplit; k0 += 4) {
      int2 v[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int sg = 0; sg < 3; ++sg)
          v[u][sg] = (k0 + u < ksplit && sg < nseg)
                         ? __ldg(reinterpret_cast<const int2*>(prow + (k0 + u) * sl +
                                                               packed_row(sg, c, nseg)))
                         : make_int2(0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int sg = 0; sg < 3; ++sg) {
          a[sg].x += v[u][sg].x;
          a[sg].y += v[u][sg].y;
        }
    }
#pragma unroll
    for (int sg = 0; sg < 3; ++sg) {
      a[sg].x -= qs;
      a[sg].y -= qs;
    }
    const int r0 = c, r1 = c + 1;
    if (e.kind == EPI_SWIGLU) {   // p = SiLU(g) u
      const float g0 = dqv(a[0].x, 0, r0), g1 = dqv(a[0].y, 0, r1);
      const float u0 = dqv(a[1].x, 1, r0), u1 = dqv(a[1].y, 1, r1);
      float s0, s1;
      sigmoid2(g0, g1, s0, s1);
      st_act<TY>(out + (int64_t)m * e.ldo + r0, __fmul_rn(__fmul_rn(g0, s0), u0));
      st_act<TY>(out + (int64_t)m * e.ldo + r1, __fmul_rn(__fmul_rn(g1, s1), u1));
    } else {                      // MLGRU step: f, c -> h, o'
      float* hp = e.h + (int64_t)m * e.n_out;
      const float2 hv = *reinterpret_cast<const float2*>(hp + r0);
      const float f0 = dqv(a[0].x, 0, r0), f1 = dqv(a[0].y, 0, r1);
      const float c0 = dqv(a[1].x, 1, r0), c1 = dqv(a[1].y, 1, r1);
      const float g0 = dqv(a[2].x, 2, r0), g1 = dqv(a[2].y, 2, r1);
      float sf0, sf1, sc0, sc1;
      sigmoid2(f0, c0, sf0, sc0);
      sigmoid2(f1, c1, sf1, sc1);
      const float h0 = __fadd_rn(__fmul_rn(sf0, hv.x),
                                 __fmul_rn(__fsub_rn(1.0f, sf0), __fmul_rn(c0, sc0)));
      const float h1 = __fadd_rn(__fmul_rn(sf1, hv.y),
                                 __fmul_rn(__fsub_rn(1.0f, sf1), __fmul_rn(c1, sc1)));
      float o0, o1;
      if (e.gate == TERN_GATE_SIGMOID_H) {
        float q0, q1;
        sigmoid2(h0, h1, q0, q1);
        o0 = __fmul_rn(g0, q0);
        o1 = __fmul_rn(g1, q1);
      } else {
        o0 = __fmul_rn(g0, h0);
        o1 = __fmul_rn(g1, h1);
      }
      *reinterpret_cast<float2*>(hp + r0) = make_float2(h0, h1);
      st_act<TY>(out + (int64_t)m * e.ldo + r0, o0);
      st_act<TY>(out + (int64_t)m * e.ldo + r1, o1);
    }
    trace_mark(trace, 2);
    return;
  }
  // one segment or the interleaved f|c|g columns: columns c, c+1 (c even)
  int2 a = make_int2(0, 0);
  for (int k0 = 0; k0 < ksplit; k0 += 4) {   // four slices' loads in flight per round
    int2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = k0 + u < ksplit ? __ldg(reinterpret_cast<const int2*>(prow + (k0 + u) * sl + c))
                             : make_int2(0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a.x += v[u].x;
      a.y += v[u].y;
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int col = c + j;
    if (col >= ncol) break;
    int seg = 0, r = col;
    if (e.kind == EPI_FCG) {   // col is the packed row
      seg = (col / kSegRows) % e.n_seg;
      r = (col / (kSegRows * e.n_seg)) * kSegRows + (col % kSegRows);
      if (r >= e.n_out) continue;
    }
    float o = dqv((j == 0 ? a.x : a.y) - qs, seg, r);
    if (e.kind == EPI_RESID)
      o = __fadd_rn(ld_act<TY>(static_cast<const TY*>(e.res) + (int64_t)m * e.ldr + r), o);
    else if (e.kind == EPI_RESID_RED)   // the residual is already in place
      o = __fadd_rn(ld_act<TY>(out + (int64_t)m * e.ldo + r), o);
    st_act<TY>(out + (int64_t)m * e.ldo + (e.kind == EPI_FCG ? col : r), o);
  }
  trace_mark(trace, 2);
}

int g_gemm_sab = getenv("TERN_GEMM_SAB") ? (atoi(getenv("TERN_GEMM_SAB")) != 0) : 0;
int g_gemm_2sm = getenv("TERN_GEMM_2SM") ? (atoi(getenv("TERN_GEMM_2SM")) != 0) : 1;

// the split-K / finalize decision of launch_gemm (small M, few tiles)
static bool gemm_finalize(int M, const tern_weight& w, const Epi& epi, int32_t* part,
                          size_t part_bytes, int tiles, int num_kb, int num_sms, bool ks_req) {
  const size_t slice = (size_t)M * w.n_rows * sizeof(int32_t);
  return ks_req || epi.kind == EPI_MLGRU ||
         (part && part_bytes >= slice && epi.kind != EPI_NONE && w.n_rows % 2 == 0 &&
          epi.acc == nullptr && tiles * 2 <= num_sms && num_kb >= 2);
}

static int gemm_bn(int M, const tern_weight& w, int nsm) {
  static const int bn_force = getenv("TERN_GEMM_BN") ? atoi(getenv("TERN_GEMM_BN")) : 0;   // debug
  int BN = (w.n_rows >= 1024 || w.n_rows % 256 == 0) ? 256 : 128;
  // small M (decode batches): narrower tiles so the weight rows spread over more SMs
  if (M <= kSmallM) BN = 128;
  // few 256-wide tiles (a short prefill, e.g. one 2048-token sequence: the N = 1024 GEMMs
  // have 64 tiles for 148 SMs): 128-wide tiles double the CTAs that work while still one
  // wave (measured c2 B = 1 x 2048: 103.5 -> 98.5 us per block; the same switch where it
  // makes two waves -- c3's 128-tile GEMMs -- cost c3 B = 1 170 -> 188 us)
  const int t256 = ((M + kBM - 1) / kBM) * ((w.n_rows + 255) / 256);
  if (BN == 256 && 2 * t256 <= nsm) BN = 128;
  if (bn_force == 128 || bn_force == 256) BN = bn_force;
  return BN;
}

static int sm_count() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

// fused quantization: opt-in (tern_set_qfuse; measured slower than quant + GEMM)
int g_qfuse_on = getenv("TERN_QFUSE") ? (atoi(getenv("TERN_QFUSE")) != 0) : 0;

bool gemm_qfuse_ok(int M, const tern_weight& w, const Epi& epi, int32_t* part, size_t part_bytes) {
  if (!g_qfuse_on || M <= kSmallM || w.e8 == nullptr || epi.acc != nullptr) return false;
  if (epi.kind == EPI_NONE || epi.kind == EPI_MLGRU) return false;
  const int nsm = sm_count();
  const int BN = gemm_bn(M, w, nsm);
  const int kp = (w.k + kKAlign - 1) / kKAlign * kKAlign;
  const int tiles = ((w.n_rows + BN - 1) / BN) * ((M + kBM - 1) / kBM);
  return !gemm_finalize(M, w, epi, part, part_bytes, tiles, kp / kBK, nsm, false);
}

cudaError_t launch_gemm(const int8_t* q, int M, int ldq, const float* deq, const int32_t* qsum,
                        const tern_weight& w, int ydt, const Epi& epi, cudaStream_t s,
                        int32_t* part, size_t part_bytes, int* ks_out, const QFuse* qf) {
  if (M <= 0) return cudaSuccess;
  if (qf && (ks_out || !gemm_qfuse_ok(M, w, epi, part, part_bytes))) {
    // not a fusable shape: the standalone quantization first
    cudaError_t qe = launch_quant(qf->x, ydt, M, w.k, qf->ldx, qf->gain, qf->eps,
                                  const_cast<int8_t*>(q), ldq, const_cast<float*>(deq),
                                  const_cast<int32_t*>(qsum), nullptr, nullptr, s);
    if (qe != cudaSuccess) return qe;
    qf = nullptr;
  }
  const int kp = (w.k + kKAlign - 1) / kKAlign * kKAlign;
  const int BN = gemm_bn(M, w, sm_count());
  // the u8 copy halves shared-memory traffic when the tensor cores are the limit
  // (large M); for decode batches the weight bytes are, and the 2-bit codes are 4x fewer
  // small M: the u8 copy too (TMA only, no smem unpack on the critical path:
  // measured faster for decode batches than the 4x smaller 2-bit codes)
  static const int small_pre = getenv("TERN_SMALLM_PRE") ? atoi(getenv("TERN_SMALLM_PRE")) : 1;   // debug
  const bool pre = w.e8 != nullptr && (M > kSmallM || small_pre);
  const bool yb = ydt == TERN_BF16;
  const size_t ys = yb ? 2 : 4;
  const CUtensorMapDataType ydtype = yb ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUtensorMapSwizzle yswz = yb ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUtensorMap ta, tb, to, tr;
  memset(&tb, 0, sizeof(tb));
  memset(&to, 0, sizeof(to));
  memset(&tr, 0, sizeof(tr));
  if (!make_map_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, q, (uint64_t)kp, (uint64_t)M,
                   (uint64_t)ldq, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (pre && !make_map_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, w.e8, (uint64_t)kp,
                          (uint64_t)w.n_rows, (uint64_t)kp, kBK, BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (epi.kind != EPI_NONE) {
    const int ncols = epi.kind == EPI_FCG ? w.n_rows : epi.n_out;
    if (!make_map_2d(&to, ydtype, epi.out, (uint64_t)ncols, (uint64_t)M, (uint64_t)epi.ldo * ys,
                     32, 32, yswz))
      return cudaErrorInvalidValue;
    if (epi.kind == EPI_RESID &&
        !make_map_2d(&tr, ydtype, epi.res, (uint64_t)epi.n_out, (uint64_t)M,
                     (uint64_t)epi.ldr * ys, 32, 32, yswz))
      return cudaErrorInvalidValue;
  }
  GemmArgs a{};
  a.M = M;
  a.n_rows = w.n_rows;
  a.codes = w.codes;
  a.num_kb = kp / kBK;
  a.n_tiles = (w.n_rows + BN - 1) / BN;
  a.m_tiles = (M + kBM - 1) / kBM;
  a.deq = deq;
  a.qsum = qsum;
  a.epi = epi;
  a.ksplit = 1;
  a.kb_per = a.num_kb;
  if (qf) {   // fused quantization of A (only on the paths below that take it)
    a.qx = qf->x;
    a.qldx = qf->ldx;
    a.qK = w.k;
    a.qmb = (M + 127) / 128;
    a.qgain = qf->gain;
    a.qeps = qf->eps;
    a.qinv_k = 1.0 / (double)w.k;
    a.qq = const_cast<int8_t*>(q);
    a.qldq = ldq;
    a.qdeq = const_cast<float*>(deq);
    a.qqsum = const_cast<int32_t*>(qsum);
    a.qctr = qf->ctr;
  }
  // split-K / finalize mode when the tiles cannot fill the SMs (decode batches,
  // small M) or the epilogue is the MLGRU step (decode T = 1 above the GEMV
  // limit): K slices write int32 partials, k_splitk_epi sums them exactly and
  // runs the epilogue
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = a.n_tiles * a.m_tiles;
  const size_t slice = (size_t)M * w.n_rows * sizeof(int32_t);
  // (the split-K epilogue reads column pairs: even n_rows, true for every fused group)
  const bool finalize = gemm_finalize(M, w, epi, part, part_bytes, tiles, a.num_kb, num_sms,
                                      ks_out != nullptr);
  // decode batches, opt-in (TERN_GEMM_SAB=1; measured slower, k_gemm_sab.cu): the swap-AB
  // kernel streams the 2-bit codes (weights as the MMA's M operand, tokens as N) into int32
  // K-slice partials
  if (g_gemm_sab && M <= kSmallM && gemm_sab_supported(M) && part && part_bytes >= slice &&
      epi.acc == nullptr && (epi.kind != EPI_NONE || ks_out) && w.n_rows % 2 == 0) {
    int ks = 0;
    const int ks_max = (ks_out && *ks_out > 0) ? *ks_out : 0;
    cudaError_t err = launch_gemm_sab(q, M, ldq, w, part, part_bytes, ks_max, &ks, s);
    if (err != cudaSuccess) return err;
    if (ks_out) {   // partials only: the caller finalizes (k_fin.cu)
      *ks_out = ks;
      return cudaSuccess;
    }
    return launch_splitk_epi(part, ks, M, w.n_rows, deq, qsum, epi, ydt, s);
  }
  if (finalize) {
    if (!part || part_bytes < slice) return cudaErrorInvalidValue;
    int ks = num_sms / tiles;   // one round of work units over the SMs
    if (ks_out && *ks_out > 0 && ks > *ks_out) ks = *ks_out;
    if (ks < 1) ks = 1;
    // the slices' int32 partials cost L2 traffic (ks * M * n * 4 bytes): few, long K
    // slices -- except for very small M, where that traffic is negligible
    static const int ks_env = getenv("TERN_KS_CAP") ? atoi(getenv("TERN_KS_CAP")) : 0;   // debug
    const int ks_cap = ks_env > 0 ? ks_env : (M <= 64 ? 16 : 4);
    if (ks > ks_cap) ks = ks_cap;
    if (ks > a.num_kb) ks = a.num_kb;
    if ((size_t)ks * slice > part_bytes) ks = (int)(part_bytes / slice);
    a.kb_per = (a.num_kb + ks - 1) / ks;
    a.ksplit = (a.num_kb + a.kb_per - 1) / a.kb_per;
    a.part = part;
    cudaError_t err = pre ? (yb ? gemm_dispatch_bn<true, __nv_bfloat16>(BN, ta, tb, to, tr, a, s)
                                : gemm_dispatch_bn<true, float>(BN, ta, tb, to, tr, a, s))
                          : (yb ? gemm_dispatch_bn<false, __nv_bfloat16>(BN, ta, tb, to, tr, a, s)
                                : gemm_dispatch_bn<false, float>(BN, ta, tb, to, tr, a, s));
    if (err != cudaSuccess) return err;
    if (ks_out) {   // partials only: the caller finalizes (k_fin.cu)
      *ks_out = a.ksplit;
      return cudaSuccess;
    }
    const bool chan = epi.kind == EPI_SWIGLU || epi.kind == EPI_MLGRU;
    const int ncol = chan ? epi.n_out : (epi.kind == EPI_FCG ? w.n_rows : epi.n_out);
    const int64_t n = (int64_t)M * ((ncol + 1) / 2);
    const unsigned grid = (unsigned)((n + 255) / 256);
    const int32_t* pc = part;
    unsigned long long* tr = trace_slot(TERN_K_GEMM + 16, (int)grid);
    if (yb)
      return launch_pdl(k_splitk_epi<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, pc, a.ksplit, M,
                        w.n_rows, deq, qsum, epi, tr);
    return launch_pdl(k_splitk_epi<float>, dim3(grid), dim3(256), 0, s, pc, a.ksplit, M, w.n_rows,
                      deq, qsum, epi, tr);
  }
  // large M with the u8 weight copy and a long K loop: 256 x 256 tiles on CTA pairs
  // (k_gemm_2sm; measured: c2 down 57.5 -> 55.5 us, c3 gate|up 538 -> 508, c3 down 253 -> 220;
  // short-K GEMMs stay on single CTAs: c2 gate|up (K = 1024) 96 -> 108 us on pairs, and the
  // short residual GEMMs take the residual-prefetch variant)
  static const int kb2 = getenv("TERN_GEMM_2SM_KB") ? atoi(getenv("TERN_GEMM_2SM_KB")) : 16;  // debug
  static const int res2 = getenv("TERN_GEMM_2SM_RESID") ? atoi(getenv("TERN_GEMM_2SM_RESID")) : 0;  // debug
  const bool res_short = epi.kind == EPI_RESID && a.num_kb <= 16 && !res2;
  if (pre && BN == 256 && g_gemm_2sm && epi.acc == nullptr && epi.kind != EPI_NONE &&
      a.num_kb >= kb2 && !res_short && M > kSmallM) {
    CUtensorMap tb2;
    if (!make_map_2d(&tb2, CU_TENSOR_MAP_DATA_TYPE_UINT8, w.e8, (uint64_t)kp, (uint64_t)w.n_rows,
                     (uint64_t)kp, kBK, 128, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    GemmArgs a2 = a;
    a2.m_tiles = (M + 255) / 256;
    static const int nb2 = getenv("TERN_GEMM_2SM_NB") ? atoi(getenv("TERN_GEMM_2SM_NB")) : 2;  // debug
    if (a2.qctr)
      return yb ? gemm2_launch<__nv_bfloat16, 2, true>(ta, tb2, to, tr, a2, s)
                : gemm2_launch<float, 2, true>(ta, tb2, to, tr, a2, s);
    if (nb2 == 1)
      return yb ? gemm2_launch<__nv_bfloat16, 1>(ta, tb2, to, tr, a2, s)
                : gemm2_launch<float, 1>(ta, tb2, to, tr, a2, s);
    return yb ? gemm2_launch<__nv_bfloat16, 2>(ta, tb2, to, tr, a2, s)
              : gemm2_launch<float, 2>(ta, tb2, to, tr, a2, s);
  }
  if (pre)
    return yb ? gemm_dispatch_bn<true, __nv_bfloat16>(BN, ta, tb, to, tr, a, s)
              : gemm_dispatch_bn<true, float>(BN, ta, tb, to, tr, a, s);
  return yb ? gemm_dispatch_bn<false, __nv_bfloat16>(BN, ta, tb, to, tr, a, s)
            : gemm_dispatch_bn<false, float>(BN, ta, tb, to, tr, a, s);
}

cudaError_t launch_splitk_epi(const int32_t* part, int ks, int M, int n_rows, const float* deq,
                              const int32_t* qsum, const Epi& epi, int ydt, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const bool chan = epi.kind == EPI_SWIGLU || epi.kind == EPI_MLGRU;
  const int ncol = chan ? epi.n_out : (epi.kind == EPI_FCG ? n_rows : epi.n_out);
  const int64_t n = (int64_t)M * ((ncol + 1) / 2);
  const unsigned grid = (unsigned)((n + 255) / 256);
  unsigned long long* tr = trace_slot(TERN_K_GEMM + 16, (int)grid);
  if (ydt == TERN_BF16)
    return launch_pdl(k_splitk_epi<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, part, ks, M,
                      n_rows, deq, qsum, epi, tr);
  return launch_pdl(k_splitk_epi<float>, dim3(grid), dim3(256), 0, s, part, ks, M, n_rows, deq,
                    qsum, epi, tr);
}

// ----------------------------------------------------------------- u8 expansion (kPre B)
// e8[r][k] = 2-bit field of trit k of packed row r (e = t+1), k < Kp.
__global__ void k_expand(const uint32_t* __restrict__ codes, int n_rows, int kp,
                         uint8_t* __restrict__ e8) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one word
  const int words = kp / 16;
  if (idx >= (int64_t)n_rows * words) return;
  const int r = (int)(idx / words), w = (int)(idx % words);
  const uint32_t word = codes[((int64_t)(w >> 3) * n_rows + r) * 8 + (w & 7)];
  uint4 v;
  v.x = word & 0x03030303u;
  v.y = (word >> 2) & 0x03030303u;
  v.z = (word >> 4) & 0x03030303u;
  v.w = (word >> 6) & 0x03030303u;
  *reinterpret_cast<uint4*>(e8 + (int64_t)r * kp + w * 16) = v;
}

cudaError_t launch_expand(const tern_weight& w, uint8_t* e8, cudaStream_t s) {
  const int kp = w.ldw * 16;
  const int64_t n = (int64_t)w.n_rows * (kp / 16);
  k_expand<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w.codes, w.n_rows, kp, e8);
  return cudaGetLastError();
}

}  // namespace tern
