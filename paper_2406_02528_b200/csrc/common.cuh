// common.cuh -- device helpers shared by the libtern kernels (sm_100a only).
//
// Numerics: every float op is written as an
// explicit IEEE round-to-nearest intrinsic (__fmul_rn, __fadd_rn, ...), and the
// library is built with -fmad=false, so no a*b+c is contracted except where
// __fmaf_rn is written.  These are independent re-implementations of the
// specification; nothing here is shared with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "internal.h"

#ifndef __CUDACC__
#error "CUDA only"
#endif

namespace tern {


// ----------------------------------------------------------------- numerics
// Canonical exp (reading C12): x = k ln2 + r, k = rint(x*log2e), two-constant
// Cody-Waite reduction, degree-7 Taylor polynomial in Horner form with fma,
// then multiply by 2^k.  Constants are the binary32 values in DESIGN.md.
__device__ __forceinline__ float exp_c(float x) {
  // branch-free (selects only), so unrolled element loops keep their ILP
  const float k = rintf(__fmul_rn(x, 0x1.715476p+0f));
  float r = __fmaf_rn(-k, 0x1.62e400p-1f, x);
  r = __fmaf_rn(-k, 0x1.7f7d1cp-20f, r);
  float p = 0x1.a01a02p-13f;
  p = __fmaf_rn(p, r, 0x1.6c16c2p-10f);
  p = __fmaf_rn(p, r, 0x1.111112p-7f);
  p = __fmaf_rn(p, r, 0x1.555556p-5f);
  p = __fmaf_rn(p, r, 0x1.555556p-3f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  int ki = (int)k;
  const bool big = ki > 127;
  p = big ? __fmul_rn(p, 2.0f) : p;
  ki = big ? ki - 1 : ki;
  ki = max(min(ki, 127), -126);   // in-range x never needs the clamp
  float res = __fmul_rn(p, __int_as_float((ki + 127) << 23));
  res = x >= 0x1.62e430p+6f ? __int_as_float(0x7f800000) : res;
  res = x < -0x1.5d589ep+6f ? 0.0f : res;
  return x != x ? x : res;
}

// Correctly rounded 1/d for d >= 1 (== IEEE __fdiv_rn(1, d)) without the
// division's special-case scaffolding: MUFU reciprocal estimate + one Newton
// correction with an exact FMA residual.  d >= 2^120 (results near the
// subnormal range) and NaN take the IEEE path.  Equality with __fdiv_rn is
// checked exhaustively over all mantissas by tern_selftest (GPU test).
__device__ __forceinline__ float rcp_ge1(float d) {
  if (!(d < 0x1p120f)) return __fdiv_rn(1.0f, d);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  const float e = __fmaf_rn(-d, r, 1.0f);
  return __fmaf_rn(r, e, r);
}

// sigma(x) = 1/(1+exp(-x)); the reciprocal is the correctly rounded one.
__device__ __forceinline__ float sigmoid_c(float x) {
  return rcp_ge1(__fadd_rn(1.0f, exp_c(-x)));
}
// SiLU tau(x) = x sigma(x).
__device__ __forceinline__ float silu_c(float x) { return __fmul_rn(x, sigmoid_c(x)); }

// Fast reciprocal of d >= 1: MUFU estimate + one Newton step with an exact
// FMA residual; equal to IEEE 1/d for 1 <= d < 2^126 (tern_selftest 0 checks
// every mantissa of every exponent), 0 for d >= 2^126 (flush-to-zero).
__device__ __forceinline__ float rcp_fast(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  const float e = __fmaf_rn(-d, r, 1.0f);
  return __fmaf_rn(r, e, r);
}

// a = a*b + c on two lanes at once (FFMA2, sm_100); FMA only -- an explicit
// f32x2 mul+add pair could be contracted by ptxas, so none is written.
__device__ __forceinline__ void fma2(float& a0, float& a1, float b0, float b1, float c0, float c1) {
  unsigned long long A, B, Cc, D;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(Cc) : "f"(c0), "f"(c1));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(Cc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(D));
}

// Two sigmoids for vectorised loops (scan, SwiGLU epilogue): exp_c's exact
// operation sequence with the FMAs paired on FFMA2, no branches, no range
// selects and no conversion-pipe instructions (domain |x| < 2^21; the
// activations here are dequantized BitLinear outputs, |x| < 127*K*deq*m).  Equal bit for bit to sigmoid_c (IEEE 1/(1+exp_c(-x))) whenever
// that result is a normal number (>= 2^-126, i.e. x > -87.3); below it returns
// 0 instead of a subnormal (< 1.2e-38): far inside every tolerance and
// quantizing identically downstream.  Checked over 2^24 points by
// tern_selftest 2.
__device__ __forceinline__ void sigmoid2(float x0, float x1, float& s0, float& s1) {
  const float y0 = -x0, y1 = -x1;
  // rint(y log2e) with the 1.5*2^23 magic constant (exact round-to-nearest-even
  // for |z| < 2^22, the same value rintf gives) -- no FRND / F2I (conversion
  // pipe: 16/clk/SM); the integer k is read from the magic sum's bits
  const float z0 = __fmul_rn(y0, 0x1.715476p+0f), z1 = __fmul_rn(y1, 0x1.715476p+0f);
  const float m0 = __fadd_rn(z0, 12582912.0f), m1 = __fadd_rn(z1, 12582912.0f);
  const float k0 = __fsub_rn(m0, 12582912.0f), k1 = __fsub_rn(m1, 12582912.0f);
  const int ik0 = __float_as_int(m0) - 0x4B400000, ik1 = __float_as_int(m1) - 0x4B400000;
  float r0 = -k0, r1 = -k1;
  fma2(r0, r1, 0x1.62e400p-1f, 0x1.62e400p-1f, y0, y1);       // y - k ln2_hi
  float t0 = -k0, t1 = -k1;
  fma2(t0, t1, 0x1.7f7d1cp-20f, 0x1.7f7d1cp-20f, r0, r1);     // - k ln2_lo
  r0 = t0; r1 = t1;
  float p0 = 0x1.a01a02p-13f, p1 = 0x1.a01a02p-13f;
  fma2(p0, p1, r0, r1, 0x1.6c16c2p-10f, 0x1.6c16c2p-10f);
  fma2(p0, p1, r0, r1, 0x1.111112p-7f, 0x1.111112p-7f);
  fma2(p0, p1, r0, r1, 0x1.555556p-5f, 0x1.555556p-5f);
  fma2(p0, p1, r0, r1, 0x1.555556p-3f, 0x1.555556p-3f);
  fma2(p0, p1, r0, r1, 0.5f, 0.5f);
  fma2(p0, p1, r0, r1, 1.0f, 1.0f);
  fma2(p0, p1, r0, r1, 1.0f, 1.0f);
  // p * 2^k with k clamped to the normal exponents: k >= 128 (exp overflows)
  // then gives d ~ 2^127 whose reciprocal flushes to 0 = 1/inf; k <= -127
  // gives d == 1 exactly, as the true tiny exp would.
  const int i0 = max(min(ik0, 127), -126), i1 = max(min(ik1, 127), -126);
  const float e0 = __fmul_rn(p0, __int_as_float((i0 + 127) << 23));
  const float e1 = __fmul_rn(p1, __int_as_float((i1 + 127) << 23));
  s0 = rcp_fast(__fadd_rn(1.0f, e0));
  s1 = rcp_fast(__fadd_rn(1.0f, e1));
}

// round half away from zero (reading C3), exact for any finite float.
__device__ __forceinline__ float round_half_away(float v) {
  float t = truncf(v);
  if (fabsf(__fsub_rn(v, t)) >= 0.5f) t = __fadd_rn(t, copysignf(1.0f, v));
  return t;
}

// The same for |v| < 2^22 without the conversion pipe (truncf is an FRND, and
// the float->int that follows an F2I, both on the 16/clk/SM conversion unit):
// v + 1.5*2^23 rounds to nearest even; a tie (|v - r| == 0.5, exact) is moved
// away from zero.  Equal to round_half_away on that range (tern_selftest 3).
__device__ __forceinline__ float round_half_away_small(float v) {
  const float r = __fsub_rn(__fadd_rn(v, 12582912.0f), 12582912.0f);
  return fabsf(__fsub_rn(v, r)) == 0.5f ? __fadd_rn(v, copysignf(0.5f, v)) : r;
}
// integral float |r| < 2^22 -> int, also on the FP32 pipe
__device__ __forceinline__ int int_of_integral(float r) {
  return __float_as_int(__fadd_rn(r, 12582912.0f)) - 0x4B400000;
}
// int_of_integral(round_half_away_small(v)) in fewer instructions, for |v| < 2^22:
// w = v + copysign(1/2, v) rounded toward zero, then w's integer part (toward zero) from the
// bits of w + copysign(1.5 * 2^23, v), also rounded toward zero.  Exact: rounding toward zero
// never steps over an integer (integers are floats), so trunc(fl_rz(v +- 1/2)) ==
// trunc(v +- 1/2) == round half away from zero (checked for every such float: tern_selftest 4)
__device__ __forceinline__ int rha_int_small(float v) {
  const uint32_t sg = __float_as_uint(v) & 0x80000000u;
  const float w = __fadd_rz(v, __uint_as_float(sg | 0x3f000000u));
  const uint32_t b = __float_as_uint(__fadd_rz(w, __uint_as_float(sg | 0x4B400000u)));
  return sg ? (int)(0xCB400000u - b) : (int)(b - 0x4B400000u);
}

// bf16 storage rounding (R0-R3): round to nearest even and widen back.
__device__ __forceinline__ float bf16r(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}

template <typename T> __device__ __forceinline__ float ld_act(const T* p);
template <> __device__ __forceinline__ float ld_act<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_act<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
// L2-coherent load (bypasses L1) of data written by an earlier grid in a PDL chain
template <typename T> __device__ __forceinline__ float ld_act_cg(const T* p);
template <> __device__ __forceinline__ float ld_act_cg<float>(const float* p) { return __ldcg(p); }
template <> __device__ __forceinline__ float ld_act_cg<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __uint_as_float((uint32_t)__ldcg(reinterpret_cast<const unsigned short*>(p)) << 16);
}
template <typename T> __device__ __forceinline__ void st_act(T* p, float v);
template <> __device__ __forceinline__ void st_act<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void st_act<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}
// value as it will be stored (identity for fp32, bf16 rounding for bf16)
template <typename T> __device__ __forceinline__ float storage_round(float v);
template <> __device__ __forceinline__ float storage_round<float>(float v) { return v; }
template <> __device__ __forceinline__ float storage_round<__nv_bfloat16>(float v) { return bf16r(v); }

// packed row index of (segment s, logical row r) in a fused group
__device__ __forceinline__ int packed_row(int s, int r, int n_seg) {
  return (r / kSegRows) * (n_seg * kSegRows) + s * kSegRows + (r % kSegRows);
}

// Exact int -> float for |v| < 2^22 without the conversion pipe (I2F runs at
// 16/clk/SM): add the integer to the bits of 1.5*2^23, subtract 1.5*2^23.
// acc - qsum of a BitLinear is bounded by 127*K < 2^21.
__device__ __forceinline__ float i2f_small(int v) {
  return __fsub_rn(__int_as_float(0x4B400000 + v), 12582912.0f);
}

// ----------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------- int dot
// dp4a with unsigned 8-bit weight fields and signed 8-bit activations.
__device__ __forceinline__ int dp4a_us(uint32_t a_u8x4, uint32_t b_s8x4, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8x4), "r"(b_s8x4), "r"(c));
  return d;
}

// ----------------------------------------------------------------- PTX: mbarrier / TMA / tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  // "memory": keeps the read in program order with barriers and memory ops
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
  return t;
}
// Device timeline (tern_trace_enable): thread 0 of CTA b < 1024 records the
// %globaltimer at mark 0 (start), 1 (dependency wait released), 2 (end).
// Compiled in only with -DTERN_TRACE (python -m paper_2406_02528_b200.build
// --trace): the marks cost ~2% of a prefill step even when disabled.
#ifdef TERN_TRACE
#define TERN_TRACE_ON 1
__device__ __forceinline__ void trace_mark(unsigned long long* tr, int mark) {
  if (tr != nullptr && threadIdx.x == 0 && blockIdx.x < 1024) tr[blockIdx.x * 16 + mark] = gtimer();
}
#else
#define TERN_TRACE_ON 0
__device__ __forceinline__ void trace_mark(unsigned long long*, int) {}
#endif
// Adds to the expected transaction bytes of the current phase without arriving.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Polling wait without a suspend-time hint (short waits on the critical path).
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// Waits for the phase with the given parity.  try_wait carries a suspend-time
// hint, so a waiting warp sleeps until the phase completes (or the hint
// elapses) instead of spinning on the issue slots its CTA's busy warps need.
// A watchdog turns a lost arrival (a pipeline bug) into a trap after ~20 s of
// %globaltimer instead of a silent hang.
#ifndef TERN_MBAR_HINT
#define TERN_MBAR_HINT 0x989680   // suspend-time hint (ns); 0: plain try_wait polling
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, polls = 0;
  unsigned long long t0 = 0;
  do {
#if TERN_MBAR_HINT
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"((uint32_t)TERN_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
#endif
    if (!done && (++polls & 1023u) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();
    }
  } while (!done);
}
// Waits with an explicit exponential sleep instead of the suspend hint: for warps that
// wait long while other warps of their sub-partition compute (k_fcgscan's gate warps
// waiting for the carry), the hinted try_wait re-polls on every barrier event of the CTA
// (~40 polls per wait measured), and the polls take the busy warps' issue slots.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity,
                                                  uint32_t ns0 = 32, uint32_t ns_max = 256) {
  uint32_t done = 0, ns = ns0;
  unsigned long long t0 = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
    ns = ns < ns_max ? 2 * ns : ns_max;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t0 == 0) t0 = t;
    else if (t - t0 > 20000000000ull) __trap();   // watchdog, as mbar_wait
  }
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// 1-D bulk async copy global -> shared, completing on an mbarrier (TMA engine).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Programmatic dependent launch: let the next grid in the stream start, and
// wait until the previous grid's results are visible.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Host: launch with programmatic dependent launch allowed (the kernel must
// call pdl_wait() before touching data produced by earlier kernels, and may
// call pdl_launch_dependents() to let the next one start its prologue).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, int8 x uint8 -> int32 (kind::i8), one thread issues.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 columns of 32-bit from TMEM; thread i gets lane (base+i), cols [col, col+32)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 columns of 32-bit from TMEM; thread i gets lane (base+i), cols [col, col+16)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, 8-row
// atoms of 1024 B (SBO = 1024), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

}  // namespace tern
