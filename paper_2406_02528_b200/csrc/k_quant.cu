// k_quant.cu -- a2: fused RMSNorm + per-token absmax int8 quantization
// (Alg. 1 rms_norm_fwd + activation_quant; Eq. 1 P:501-505;
// readings C1-C5, C7).  The row is held in registers, so the activation is read
// from HBM exactly once (the point of the fused design).  HBM-bound:
// reads K*sizeof(x), writes roundup(K,128) bytes + 12 B per row.
//
// TPR threads per row (32..256) so that every thread holds at most NV 16-byte
// vectors: small register tiles keep occupancy (and bytes in flight) high.
// Element loops are branch-free (out-of-row vectors are predicated to zero,
// which also produces the zero padding up to Kp); sum(x^2) accumulates in
// binary64 with explicit fma (C4), partials combined in a fixed order.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace tern {

constexpr int kQThreads = 256;

template <typename TX> struct QVec;
template <> struct QVec<float> {
  static constexpr int N = 4;
  __device__ static void unpack(const uint4& u, float* v) {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
    v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
  }
};
template <> struct QVec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void unpack(const uint4& u, float* v) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

__device__ __forceinline__ uint4 ldg_stream_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// sum over the WPR warps of one row (every thread of the row gets the total)
template <int RPC, int WPR>
__device__ __forceinline__ double row_sum_d(double v, double (*red)[WPR], int rloc, int wr, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (WPR > 1) {
    __syncthreads();
    if (lane == 0) red[rloc][wr] = v;
    __syncthreads();
    v = red[rloc][0];
#pragma unroll
    for (int i = 1; i < WPR; ++i) v += red[rloc][i];
  }
  return v;
}
template <int RPC, int WPR>
__device__ __forceinline__ float row_max_f(float v, float (*red)[WPR], int rloc, int wr, int lane) {
  v = warp_max_f32(v);
  if (WPR > 1) {
    __syncthreads();
    if (lane == 0) red[rloc][wr] = v;
    __syncthreads();
    v = red[rloc][0];
#pragma unroll
    for (int i = 1; i < WPR; ++i) v = fmaxf(v, red[rloc][i]);
  }
  return v;
}

// Centred norm + quant of the thread's share of one row (reading C22):
//   mu = (float)(sum x / K), var = sum (x - mu)^2 / K (binary64; x - mu exact),
//   r = (float)(1 / sqrt(var + eps)), y = ((x - mu) r) w, then absmax quant.
// Padding elements (v >= nvec) take no part in the moments and quantize to 0.
template <typename TX, int TPR, int NV>
__device__ __forceinline__ void centred_row(const uint4 (&xv)[NV], bool rv, int row, int t, int lane,
                                            int wr, int rloc, int nvec, int nvecp, int K,
                                            const float* __restrict__ gain, float eps,
                                            int8_t* __restrict__ q, int ldq, float* __restrict__ deq,
                                            int32_t* __restrict__ qsum, float* __restrict__ inv_rms,
                                            float* __restrict__ absmax,
                                            double (*red_d)[TPR / 32], float (*red_f)[TPR / 32],
                                            int (*red_i)[TPR / 32]) {
  constexpr int VE = QVec<TX>::N;
  constexpr int WPR = TPR / 32;
  constexpr int RPC = kQThreads / TPR;
  double sx = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float v[VE];
    QVec<TX>::unpack(xv[i], v);   // zeros outside the row
#pragma unroll
    for (int j = 0; j < VE; ++j) sx += (double)v[j];
  }
  sx = row_sum_d<RPC, WPR>(sx, red_d, rloc, wr, lane);
  const float mu = (float)(sx / (double)K);
  double sv = 0.0;
  float dm = 0.0f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = t + i * TPR;
    float xf[VE];
    QVec<TX>::unpack(xv[i], xf);
    if (v < nvec) {
#pragma unroll
      for (int j = 0; j < VE; ++j) {
        const double dd = (double)xf[j] - (double)mu;
        sv = fma(dd, dd, sv);
        dm = fmaxf(dm, fabsf(__fsub_rn(xf[j], mu)));
      }
    }
  }
  sv = row_sum_d<RPC, WPR>(sv, red_d, rloc, wr, lane);
  const float r = (float)(1.0 / sqrt(sv / (double)K + (double)eps));
  float amax;
  if (gain == nullptr) {
    amax = __fmul_rn(row_max_f<RPC, WPR>(dm, red_f, rloc, wr, lane), r);   // monotone, r > 0
  } else {
    float am = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int v = t + i * TPR;
      float xf[VE];
      QVec<TX>::unpack(xv[i], xf);
      if (v < nvec) {
#pragma unroll
        for (int j = 0; j < VE; ++j)
          am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(__fsub_rn(xf[j], mu), r), __ldg(gain + v * VE + j))));
      }
    }
    amax = row_max_f<RPC, WPR>(am, red_f, rloc, wr, lane);
  }
  const float sc = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
  int8_t* qr = q + (int64_t)(rv ? row : 0) * ldq;
  int qs = 0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = t + i * TPR;
    float xf[VE];
    QVec<TX>::unpack(xv[i], xf);
    uint32_t pk[VE / 4];
#pragma unroll
    for (int j4 = 0; j4 < VE / 4; ++j4) {
      int qi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        qi[j] = 0;
        if (v < nvec) {
          float y = __fmul_rn(__fsub_rn(xf[4 * j4 + j], mu), r);
          if (gain) y = __fmul_rn(y, __ldg(gain + v * VE + 4 * j4 + j));
          qi[j] = rha_int_small(__fmul_rn(y, sc));
        }
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
  qs = warp_sum_i32(qs);
  if (WPR > 1) {
    __syncthreads();
    if (lane == 0) red_i[rloc][wr] = qs;
    __syncthreads();
    qs = red_i[rloc][0];
#pragma unroll
    for (int i = 1; i < WPR; ++i) qs += red_i[rloc][i];
  }
  if (t == 0 && rv) {
    deq[row] = amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
    qsum[row] = qs;
    if (inv_rms) inv_rms[row] = r;
    if (absmax) absmax[row] = amax;
  }
}

// TPR threads per row, NV vectors per thread; CTA = kQThreads/TPR rows.
// CENT: the centred norm of Alg. 1 (reading C22; gain checked at
// run time, row bounds always checked).
template <typename TX, int TPR, int NV, bool GAIN, bool FULL, bool CENT = false>
__global__ void __launch_bounds__(kQThreads) k_quant(const TX* __restrict__ x, int M, int K, int ldx,
                                                     const float* __restrict__ gain, float eps,
                                                     double inv_k, int8_t* __restrict__ q, int ldq,
                                                     float* __restrict__ deq,
                                                     int32_t* __restrict__ qsum,
                                                     float* __restrict__ inv_rms,
                                                     float* __restrict__ absmax,
                                                     unsigned long long* trace, int rev) {
  trace_mark(trace, 0);
  constexpr int VE = QVec<TX>::N;
  constexpr int WPR = TPR / 32;                 // warps per row
  constexpr int RPC = kQThreads / TPR;          // rows per CTA
  __shared__ double red_d[RPC][WPR];
  __shared__ float red_f[RPC][WPR];
  __shared__ int red_i[RPC][WPR];
  const int lane = threadIdx.x & 31;
  const int rloc = threadIdx.x / TPR, t = threadIdx.x % TPR, wr = t >> 5;
  // rev: the CTAs walk the rows from the last to the first.  The producing kernel wrote the rows
  // in ascending order and x is larger than what L2 keeps, so the LAST rows are the ones still
  // resident; reading in the producer's order would evict them just before they are needed.
  const int row_f = blockIdx.x * RPC + rloc;
  const bool rv = row_f < M;
  const int row = rev ? M - 1 - row_f : row_f;
  const int nvec = K / VE, nvecp = ((K + kKAlign - 1) / kKAlign * kKAlign) / VE;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)(rv ? row : 0) * ldx);
  pdl_wait();                 // x is the previous kernel's output
  pdl_launch_dependents();
  trace_mark(trace, 1);

  uint4 xv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = t + i * TPR;
    // FULL: the row is exactly TPR*NV vectors (no bounds checks at all)
    xv[i] = (FULL ? rv : (rv && v < nvec)) ? ldg_stream_v4(xr + v) : make_uint4(0, 0, 0, 0);
  }
  if (CENT) {
    centred_row<TX, TPR, NV>(xv, rv, row, t, lane, wr, rloc, nvec, nvecp, K, gain, eps, q, ldq, deq,
                             qsum, inv_rms, absmax, red_d, red_f, red_i);
    trace_mark(trace, 2);
    return;
  }
  double s0 = 0.0, s1 = 0.0;
  float xm = 0.0f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float v[VE];
    QVec<TX>::unpack(xv[i], v);
#pragma unroll
    for (int j = 0; j < VE; j += 2) {
      const double d0 = (double)v[j], d1 = (double)v[j + 1];
      s0 = fma(d0, d0, s0);
      s1 = fma(d1, d1, s1);
      xm = fmaxf(xm, fmaxf(fabsf(v[j]), fabsf(v[j + 1])));
    }
  }
  double ss = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  }
  if (WPR > 1) {
    if (lane == 0) { red_d[rloc][wr] = ss; red_f[rloc][wr] = xm; }
    __syncthreads();
    ss = red_d[rloc][0];
    xm = red_f[rloc][0];
#pragma unroll
    for (int i = 1; i < WPR; ++i) { ss += red_d[rloc][i]; xm = fmaxf(xm, red_f[rloc][i]); }
  }
  const float r = (float)rsqrt(fma(ss, inv_k, (double)eps));
  float amax;
  if (!GAIN) {
    // max|fl(x r)| = fl(max|x| r): rounding is monotone and r > 0
    amax = __fmul_rn(xm, r);
  } else {
    float am = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int v = t + i * TPR;
      float xf[VE];
      QVec<TX>::unpack(xv[i], xf);
      const float4* g4 = reinterpret_cast<const float4*>(gain + (v < nvec ? v : 0) * VE);
#pragma unroll
      for (int j = 0; j < VE; j += 4) {
        const float4 g = __ldg(g4 + j / 4);
        am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(xf[j], r), g.x)));
        am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(xf[j + 1], r), g.y)));
        am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(xf[j + 2], r), g.z)));
        am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(xf[j + 3], r), g.w)));
      }
    }
    am = warp_max_f32(am);
    if (WPR > 1) {
      __syncthreads();   // red_f of the first round has been read
      if (lane == 0) red_f[rloc][wr] = am;
      __syncthreads();
      am = red_f[rloc][0];
#pragma unroll
      for (int i = 1; i < WPR; ++i) am = fmaxf(am, red_f[rloc][i]);
    }
    amax = am;
  }
  const float sc = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
  int8_t* qr = q + (int64_t)(rv ? row : 0) * ldq;
  int qs = 0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = t + i * TPR;
    float xf[VE];
    QVec<TX>::unpack(xv[i], xf);   // zeros outside the row -> q = 0 (the padding)
    uint32_t pk[VE / 4];
#pragma unroll
    for (int j4 = 0; j4 < VE / 4; ++j4) {
      float g[4] = {1.0f, 1.0f, 1.0f, 1.0f};
      if (GAIN) {
        const float4 gg = __ldg(reinterpret_cast<const float4*>(gain + (v < nvec ? v : 0) * VE) + j4);
        g[0] = gg.x; g[1] = gg.y; g[2] = gg.z; g[3] = gg.w;
      }
      int qi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float y = __fmul_rn(xf[4 * j4 + j], r);
        if (GAIN) y = __fmul_rn(y, g[j]);
        // |y*sc| <= 127(1+2^-23), so the clamp to [-128,127] (C5) never acts
        qi[j] = rha_int_small(__fmul_rn(y, sc));
        qs += qi[j];
      }
      // low bytes of the four ints -> one word (two byte permutes)
      pk[j4] = __byte_perm(__byte_perm(qi[0], qi[1], 0x0040), __byte_perm(qi[2], qi[3], 0x0040),
                           0x5410);
    }
    if (FULL ? rv : (rv && v < nvecp)) {
      if (VE == 4)
        reinterpret_cast<uint32_t*>(qr)[v] = pk[0];
      else
        reinterpret_cast<uint2*>(qr)[v] = make_uint2(pk[0], pk[VE / 4 - 1]);
    }
  }
  qs = warp_sum_i32(qs);
  if (WPR > 1) {
    if (lane == 0) red_i[rloc][wr] = qs;
    __syncthreads();
    qs = red_i[rloc][0];
#pragma unroll
    for (int i = 1; i < WPR; ++i) qs += red_i[rloc][i];
  }
  if (t == 0 && rv) {
    deq[row] = amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
    qsum[row] = qs;
    if (inv_rms) inv_rms[row] = r;
    if (absmax) absmax[row] = amax;
  }
  trace_mark(trace, 2);
}

template <typename TX, int TPR, int NV>
static void quant_go(const TX* x, int m, int k, int ldx, const float* gain, float eps, int8_t* q,
                     int ldq, float* deq, int32_t* qsum, float* inv_rms, float* absmax,
                     cudaStream_t s, int norm) {
  constexpr int RPC = kQThreads / TPR;
  const int grid = (m + RPC - 1) / RPC;
  const double inv_k = 1.0 / (double)k;
  const bool full = k == TPR * NV * QVec<TX>::N;   // then also k == Kp
  static const int rev_env = getenv("TERN_QUANT_REV") ? atoi(getenv("TERN_QUANT_REV")) : 1;   // debug
  const int rev = rev_env && m > 256;   // prefill-sized inputs only
  auto kern = norm == TERN_NORM_CENTERED
                  ? k_quant<TX, TPR, NV, false, false, true>
                  : (gain ? k_quant<TX, TPR, NV, true, false>
                          : (full ? k_quant<TX, TPR, NV, false, true> : k_quant<TX, TPR, NV, false, false>));
  launch_pdl(kern, dim3(grid), dim3(kQThreads), 0, s, x, m, k, ldx, gain, eps, inv_k, q, ldq, deq,
             qsum, inv_rms, absmax, trace_slot(TERN_K_QUANT, grid), rev);
}

template <typename TX, int TPR>
static void quant_nv(int nv, const TX* x, int m, int k, int ldx, const float* gain, float eps,
                     int8_t* q, int ldq, float* deq, int32_t* qsum, float* inv_rms, float* absmax,
                     cudaStream_t s, int norm) {
  // exactly as many register vectors as the row needs: predicated-off slots of
  // the fully unrolled loops still cost issue slots, and this kernel is issue-bound
  switch (nv) {
    case 1: case 2: quant_go<TX, TPR, 2>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
    case 3: quant_go<TX, TPR, 3>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
    case 4: quant_go<TX, TPR, 4>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
    case 5: quant_go<TX, TPR, 5>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
    case 6: quant_go<TX, TPR, 6>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
    case 7: quant_go<TX, TPR, 7>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
    default: quant_go<TX, TPR, 8>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm); break;
  }
}

template <typename TX>
static cudaError_t quant_dispatch(const TX* x, int m, int k, int ldx, const float* gain, float eps,
                                  int8_t* q, int ldq, float* deq, int32_t* qsum, float* inv_rms,
                                  float* absmax, cudaStream_t s, int norm) {
  const int kp = (k + kKAlign - 1) / kKAlign * kKAlign;
  const int nvp = kp / QVec<TX>::N;   // vectors per (padded) row
  // few rows (decode batches): latency-bound, so spread each row over 256
  // threads (<= 4 vectors each) instead of maximising per-thread work
  if (m <= 256 && nvp > 64 && nvp <= 256 * 4) {
    quant_nv<TX, 256>((nvp + 255) / 256, x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm);
    return cudaGetLastError();
  }
  // smallest threads-per-row with <= NVMAX vectors per thread (8; debug knob TERN_QUANT_NVMAX)
  static const int nvmax_env = getenv("TERN_QUANT_NVMAX") ? atoi(getenv("TERN_QUANT_NVMAX")) : 8;
  const int nvmax = (nvmax_env >= 2 && nvmax_env <= 8) ? nvmax_env : 8;
  // bf16 rows of 2048 (c3's d): two warps per row, 4 vectors each, measured faster than one warp
  // with 8 (57.3 -> 54.0 us per launch at 32768 rows); fp32 rows and K = 5632 measured slower so
  if (sizeof(TX) == 2 && nvp == 256 && nvmax == 8)
    quant_nv<TX, 64>(4, x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm);
  else if (nvp <= 32 * nvmax)
    quant_nv<TX, 32>((nvp + 31) / 32, x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm);
  else if (nvp <= 64 * nvmax)
    quant_nv<TX, 64>((nvp + 63) / 64, x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm);
  else if (nvp <= 128 * nvmax)
    quant_nv<TX, 128>((nvp + 127) / 128, x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm);
  else if (nvp <= 256 * 8)
    quant_nv<TX, 256>((nvp + 255) / 256, x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_quant(const void* x, int xdt, int m, int k, int ldx, const float* gain,
                         float eps, int8_t* q, int ldq, float* deq, int32_t* qsum, float* inv_rms,
                         float* absmax, cudaStream_t s, int norm, uint32_t* zero, int nzero) {
  // (QFuse, opt-in: the block's fused-quantization counters zeroed ahead of its GEMMs -- a
  // memset node, not a side job of the kernel, which would cost it registers)
  if (zero != nullptr && nzero > 0) {
    const cudaError_t ze = cudaMemsetAsync(zero, 0, sizeof(uint32_t) * (size_t)nzero, s);
    if (ze != cudaSuccess) return ze;
  }
  if (m == 0) return cudaSuccess;
  if (xdt == TERN_BF16)
    return quant_dispatch(static_cast<const __nv_bfloat16*>(x), m, k, ldx, gain, eps, q, ldq, deq,
                          qsum, inv_rms, absmax, s, norm);
  return quant_dispatch(static_cast<const float*>(x), m, k, ldx, gain, eps, q, ldq, deq, qsum,
                        inv_rms, absmax, s, norm);
}

}  // namespace tern
