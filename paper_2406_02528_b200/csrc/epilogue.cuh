// epilogue.cuh -- a5 dequantization + the fused per-element functors shared by
// the decode GEMV and the tcgen05 GEMM.
//   dequant: O = (float)acc * (deq * m_seg) [+ b]
//   R1 rounding of every BitLinear output in bf16 mode, R2 of o' and p, R3 of
//   the residual stream.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace tern {

__device__ __forceinline__ float dequant(int acc, float deq, float mseg) {
  return __fmul_rn((float)acc, __fmul_rn(deq, mseg));
}

// BitLinear output value for (segment seg, logical row r), R1-rounded for TY.
template <typename TY>
__device__ __forceinline__ float bl_out(const Epi& e, int acc, float deq, int seg, int r) {
  float o = dequant(acc, deq, __ldg(e.scales + seg));
  if (e.bias) o = __fadd_rn(o, __ldg(e.bias + seg * e.n_out + r));
  return storage_round<TY>(o);
}

// Same with the segment's scale already in a register.
template <typename TY>
__device__ __forceinline__ float bl_val(const Epi& e, int acc, float deq, float mseg, int seg, int r) {
  float o = dequant(acc, deq, mseg);
  if (e.bias) o = __fadd_rn(o, __ldg(e.bias + seg * e.n_out + r));
  return storage_round<TY>(o);
}

// One recurrence step of the MLGRU with the same op order as the
// sequential definition: h' = (f*h) + ((1-f)*c).
__device__ __forceinline__ float mlgru_step(float f, float h, float c) {
  const float a = __fmul_rn(f, h);
  const float om = __fsub_rn(1.0f, f);
  const float b = __fmul_rn(om, c);
  return __fadd_rn(a, b);
}
__device__ __forceinline__ float mlgru_out(float g, float h, int gate) {
  return gate == TERN_GATE_SIGMOID_H ? __fmul_rn(g, sigmoid_c(h)) : __fmul_rn(g, h);
}
// GLU gate: p = SiLU(g) * u
__device__ __forceinline__ float swiglu(float g, float u) { return __fmul_rn(silu_c(g), u); }

// Element epilogue for the kinds that need one segment (STORE, RESID, FCG).
// col = packed row index of the accumulator, r/seg its logical coordinates.
template <typename TY>
__device__ __forceinline__ void epi_single(const Epi& e, int m, int col, int seg, int r, int acc,
                                           float deq) {
  if (e.acc) e.acc[(int64_t)m * e.ldacc + col] = acc;
  if (e.kind == EPI_NONE) return;
  const float o = bl_out<TY>(e, acc, deq, seg, r);
  TY* out = static_cast<TY*>(e.out);
  if (e.kind == EPI_STORE) {
    st_act<TY>(out + (int64_t)m * e.ldo + r, o);
  } else if (e.kind == EPI_RESID) {
    const float x = ld_act<TY>(static_cast<const TY*>(e.res) + (int64_t)m * e.ldr + r);
    st_act<TY>(out + (int64_t)m * e.ldo + r, __fadd_rn(x, o));
  } else {  // EPI_FCG: keep the interleaved column order
    st_act<TY>(out + (int64_t)m * e.ldo + col, o);
  }
}

}  // namespace tern
