// k_quant.cu -- a2: fused RMSNorm + per-token absmax int8 quantization
// (Alg. 1 rms_norm_fwd + activation_quant; Eq. 1 P:501-505;
// readings C1-C5, C7).  One CTA per row, the row held in registers, so the
// activation is read from HBM exactly once (the point of the fused design,
// P:391).  HBM-bound: reads K*sizeof(x), writes roundup(K,128) bytes + 12 B.
#include "common.cuh"
#include "internal.h"

namespace tern {

constexpr int kQThreads = 128;

template <typename TX> struct Vec4;
template <> struct Vec4<float> {
  __device__ static void load(const float* p, float (&v)[4]) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
};
template <> struct Vec4<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float (&v)[4]) {
    uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    v[0] = __uint_as_float(t.x << 16);
    v[1] = __uint_as_float(t.x & 0xffff0000u);
    v[2] = __uint_as_float(t.y << 16);
    v[3] = __uint_as_float(t.y & 0xffff0000u);
  }
};

// Deterministic block reductions: fixed shuffle tree, then warp partials summed
// in warp order by every thread.
template <int NW>
__device__ __forceinline__ double block_sum_f64(double v, double* red) {
  v = warp_sum_f64(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}
template <int NW>
__device__ __forceinline__ float block_max_f32(float v, float* red) {
  v = warp_max_f32(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int i = 0; i < NW; ++i) t = fmaxf(t, red[i]);
  return t;
}
template <int NW>
__device__ __forceinline__ int block_sum_i32(int v, int* red) {
  v = warp_sum_i32(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}

// NCH = max number of 4-element chunks per thread (compile-time register tile).
template <typename TX, int NCH>
__global__ void __launch_bounds__(kQThreads) k_quant(const TX* __restrict__ x, int K, int ldx,
                                                     const float* __restrict__ gain, float eps,
                                                     int8_t* __restrict__ q, int ldq,
                                                     float* __restrict__ deq,
                                                     int32_t* __restrict__ qsum,
                                                     float* __restrict__ inv_rms,
                                                     float* __restrict__ absmax) {
  constexpr int NW = kQThreads / 32;
  __shared__ double red_d[NW];
  __shared__ float red_f[NW];
  __shared__ int red_i[NW];
  const int row = blockIdx.x;
  const TX* xr = x + (int64_t)row * ldx;
  const int nc = K >> 2;  // K % 16 == 0
  float v[NCH][4];
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = threadIdx.x + i * kQThreads;
    if (c < nc) {
      Vec4<TX>::load(xr + 4 * c, v[i]);
    } else {
      v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) ss += (double)v[i][j] * (double)v[i][j];
  }
  ss = block_sum_f64<NW>(ss, red_d);
  const float r = (float)(1.0 / sqrt(ss / (double)K + (double)eps));
  float a = 0.0f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = threadIdx.x + i * kQThreads;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float y = __fmul_rn(v[i][j], r);
      if (gain && c < nc) y = __fmul_rn(y, __ldg(gain + 4 * c + j));
      v[i][j] = y;
      a = fmaxf(a, fabsf(y));
    }
  }
  a = block_max_f32<NW>(a, red_f);
  const float s = a > 0.0f ? __fdiv_rn(127.0f, a) : 0.0f;
  int8_t* qr = q + (int64_t)row * ldq;
  const int ncp = ((K + kKAlign - 1) / kKAlign * kKAlign) >> 2;
  int qs = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = threadIdx.x + i * kQThreads;
    if (c < ncp) {
      uint32_t packed = 0;
      if (c < nc && a > 0.0f) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // |y*s| <= 127(1+2^-23), so the clamp to [-128,127] (C5) never acts
          const int qi = (int)round_half_away(__fmul_rn(v[i][j], s));
          qs += qi;
          packed |= ((uint32_t)qi & 0xffu) << (8 * j);
        }
      }
      reinterpret_cast<uint32_t*>(qr)[c] = packed;
    }
  }
  qs = block_sum_i32<NW>(qs, red_i);
  if (threadIdx.x == 0) {
    deq[row] = a > 0.0f ? __fdiv_rn(a, 127.0f) : 0.0f;
    qsum[row] = qs;
    if (inv_rms) inv_rms[row] = r;
    if (absmax) absmax[row] = a;
  }
}

// Warp-per-row variant for K <= 32*4*NV: no block-level barriers at all; 8 rows
// per 256-thread CTA.  Same arithmetic, reductions in a fixed shuffle order.
template <typename TX, int NV>
__global__ void __launch_bounds__(256) k_quant_warp(const TX* __restrict__ x, int M, int K,
                                                    int ldx, const float* __restrict__ gain,
                                                    float eps, int8_t* __restrict__ q, int ldq,
                                                    float* __restrict__ deq,
                                                    int32_t* __restrict__ qsum,
                                                    float* __restrict__ inv_rms,
                                                    float* __restrict__ absmax) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  const TX* xr = x + (int64_t)row * ldx;
  const int nc = K >> 2;
  float v[NV][4];
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nc) {
      Vec4<TX>::load(xr + 4 * c, v[i]);
    } else {
      v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) ss += (double)v[i][j] * (double)v[i][j];
  }
  ss = warp_sum_f64(ss);
  const float r = (float)(1.0 / sqrt(ss / (double)K + (double)eps));
  float a = 0.0f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float y = __fmul_rn(v[i][j], r);
      if (gain && c < nc) y = __fmul_rn(y, __ldg(gain + 4 * c + j));
      v[i][j] = y;
      a = fmaxf(a, fabsf(y));
    }
  }
  a = warp_max_f32(a);
  const float s = a > 0.0f ? __fdiv_rn(127.0f, a) : 0.0f;
  int8_t* qr = q + (int64_t)row * ldq;
  const int ncp = ((K + kKAlign - 1) / kKAlign * kKAlign) >> 2;
  int qs = 0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < ncp) {
      uint32_t packed = 0;
      if (c < nc && a > 0.0f) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // |y*s| <= 127(1+2^-23), so the clamp to [-128,127] (C5) never acts
          const int qi = (int)round_half_away(__fmul_rn(v[i][j], s));
          qs += qi;
          packed |= ((uint32_t)qi & 0xffu) << (8 * j);
        }
      }
      reinterpret_cast<uint32_t*>(qr)[c] = packed;
    }
  }
  qs = warp_sum_i32(qs);
  if (lane == 0) {
    deq[row] = a > 0.0f ? __fdiv_rn(a, 127.0f) : 0.0f;
    qsum[row] = qs;
    if (inv_rms) inv_rms[row] = r;
    if (absmax) absmax[row] = a;
  }
}

template <typename TX>
static cudaError_t quant_dispatch(const TX* x, int m, int k, int ldx, const float* gain, float eps,
                                  int8_t* q, int ldq, float* deq, int32_t* qsum, float* inv_rms,
                                  float* absmax, cudaStream_t s) {
  const int kp = (k + kKAlign - 1) / kKAlign * kKAlign;
  const int chunks = kp / 4;
  const int nch = (chunks + kQThreads - 1) / kQThreads;
  const int nv = (chunks + 31) / 32;
  const int g8 = (m + 7) / 8;
#define TERN_QW(N)                                                                            \
  k_quant_warp<TX, N><<<g8, 256, 0, s>>>(x, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, \
                                         absmax)
  if (nv <= 8) { TERN_QW(8); return cudaGetLastError(); }
  if (nv <= 16) { TERN_QW(16); return cudaGetLastError(); }
  if (nv <= 24) { TERN_QW(24); return cudaGetLastError(); }
#undef TERN_QW
#define TERN_Q(N)                                                                              \
  k_quant<TX, N><<<m, kQThreads, 0, s>>>(x, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, \
                                         absmax)
  if (nch <= 2) TERN_Q(2);
  else if (nch <= 4) TERN_Q(4);
  else if (nch <= 8) TERN_Q(8);
  else if (nch <= 14) TERN_Q(14);
  else if (nch <= 32) TERN_Q(32);
  else return cudaErrorInvalidValue;
#undef TERN_Q
  return cudaGetLastError();
}

cudaError_t launch_quant(const void* x, int xdt, int m, int k, int ldx, const float* gain,
                         float eps, int8_t* q, int ldq, float* deq, int32_t* qsum, float* inv_rms,
                         float* absmax, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  if (xdt == TERN_BF16)
    return quant_dispatch(static_cast<const __nv_bfloat16*>(x), m, k, ldx, gain, eps, q, ldq, deq,
                          qsum, inv_rms, absmax, s);
  return quant_dispatch(static_cast<const float*>(x), m, k, ldx, gain, eps, q, ldq, deq, qsum,
                        inv_rms, absmax, s);
}

}  // namespace tern
