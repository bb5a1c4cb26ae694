// k_fxp.cu -- fixed-point W8A16 numerics of the paper's Loihi 2 deployment
// ("Implementation Details on Intel Loihi 2",
// P:707-723 "Fixed-Point Implementation Details"; readings F1-F5 in DESIGN.md §3b).
//
// All five are integer kernels bound by HBM: grids are sized to the SM count, loads
// are 16-byte vectors where the layout allows, reductions are warp shuffles plus one
// shared-memory stage.  The look-up tables (9 sigmoid points, 24 inverse-sqrt seeds)
// are formed on the host in binary64 from their definitions and passed by value as
// kernel parameters (constant bank), so no launch depends on a prior table upload.
// Nothing here divides (shifts, multiplies, the two tables), as on the neurocores.
#include <cmath>
#include <cstdint>

#include <cuda_bf16.h>

#include "internal.h"

namespace tern {

constexpr int kFxThreads = 256;
constexpr int kFxXexp = 6;    // F3: sigmoid inputs in Q6
constexpr int kFxYexp = 15;   // F3: sigmoid outputs in Q15
constexpr int kFxNsig = 8;    // F3: N_sigma (9 points x = 0..8)

struct SigLut { int32_t y[kFxNsig + 1]; };
struct RsqLut { uint32_t g[24]; };

static int fx_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
static int fx_grid(int64_t work, int per_cta) {
  const int64_t want = (work + per_cta - 1) / per_cta;
  const int64_t cap = (int64_t)fx_sms() * 8;
  return (int)(want < 1 ? 1 : want < cap ? want : cap);
}

// ---------------------------------------------------------------- shared device pieces
__device__ __forceinline__ int64_t fx_rha_shift(int64_t v, int s) {   // round(v / 2^s), half away
  if (s == 0) return v;
  const uint64_t a = v < 0 ? (uint64_t)(-v) : (uint64_t)v;
  const uint64_t r = (a + (1ull << (s - 1))) >> s;
  return v < 0 ? -(int64_t)r : (int64_t)r;
}

// F3: Q6 -> Q15 sigma through the 9-point table, linear interpolation with a floor
// (the tables are read from shared memory: lanes index them divergently, which the
// constant bank would serialise)
__device__ __forceinline__ int32_t fx_sigmoid(int32_t x, const int32_t* __restrict__ L) {
  const uint32_t a = x < 0 ? 0u - (uint32_t)x : (uint32_t)x;
  int32_t y;
  if (a >= (uint32_t)(kFxNsig << kFxXexp)) {
    y = L[kFxNsig];
  } else {
    const int i = (int)(a >> kFxXexp);
    const int32_t fr = (int32_t)(a & ((1u << kFxXexp) - 1));
    const int32_t y0 = L[i], y1 = L[i + 1];
    y = y0 + (((y1 - y0) * fr) >> kFxXexp);   // (y1 - y0) * fr < 2^15 * 2^6: no overflow
  }
  return x < 0 ? (1 << kFxYexp) - y : y;
}

// F4: 1/sqrt(v 2^e) = y 2^ey, v > 0
__device__ __forceinline__ void fx_inv_sqrt(uint64_t v, int e, const uint32_t* __restrict__ L,
                                            uint32_t& y_out, int& ey_out) {
  const int p = 63 - __clzll((long long)v);
  uint64_t m = p >= 30 ? v >> (p - 30) : v << (30 - p);
  int E = e + p;
  if (E & 1) {
    m <<= 1;
    E -= 1;
  }
  const int k = (int)((m - (1ull << 30)) >> 27);
  uint64_t y = L[k];
#pragma unroll
  for (int it = 0; it < 5; ++it) {
    const uint64_t y2 = (y * y) >> 30;
    const uint64_t my2 = (m * y2) >> 30;
    y = (y * (3ull * (1ull << 30) - my2)) >> 31;
  }
  y_out = (uint32_t)y;
  ey_out = -30 - E / 2;   // E even
}

__device__ __forceinline__ uint32_t fx_warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------- F1 norm scales
// one CTA: max|w| -> e = round(log2 max) - shift without a logarithm: max = f 2^p with
// f in [1/2, 1) (frexpf, exact); log2 max = p + log2 f rounds to p when f >= 2^-1/2,
// else p - 1 (no float lies within 1e-8 of 2^-1/2, so the binary64 constant decides).
__global__ void __launch_bounds__(1024) k_fxp_scales(const float* __restrict__ w, int n, int shift,
                                                     int8_t* __restrict__ wq, int32_t* e_out,
                                                     int32_t* status) {
  __shared__ uint32_t red[32];
  __shared__ int se, sst;
  uint32_t mx = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mx = max(mx, __float_as_uint(fabsf(w[i])));
  mx = fx_warp_max_u32(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    v = fx_warp_max_u32(v);
    if (threadIdx.x == 0) {
      const float m = __uint_as_float(v);
      int st = 0, e = 0;
      if (!(m > 0.0f) || v >= 0x7f800000u) {
        st = 2;   // zero vector or non-finite
      } else {
        int p;
        const float f = frexpf(m, &p);
        e = ((double)f >= 0.70710678118654752440 ? p : p - 1) - shift;
      }
      se = e;
      sst = st;
      *status = st;
      *e_out = e;
    }
  }
  __syncthreads();
  if (sst) return;
  const int e = se;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = roundf(ldexpf(w[i], -e));   // exact scaling, then half away
    wq[i] = (int8_t)v;                          // |v| <= round(2^(6.5)) = 91 for shift <= 6
  }
}

// ---------------------------------------------------------------- F2 activations
template <typename T>
__device__ __forceinline__ float fx_ld(const T* p, int64_t i) {
  if constexpr (sizeof(T) == 4) return reinterpret_cast<const float*>(p)[i];
  else return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

template <typename T>
__global__ void __launch_bounds__(kFxThreads) k_fxp_absmax(const T* __restrict__ x, int64_t n,
                                                           uint32_t* __restrict__ mx_out) {
  __shared__ uint32_t red[kFxThreads / 32];
  uint32_t mx = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int kV = 16 / sizeof(T);   // elements per 16-byte vector
  const int64_t nv = (reinterpret_cast<uintptr_t>(x) & 15) ? 0 : n / kV;
  for (int64_t i = tid; i < nv; i += stride) {
    const int4 raw = __ldg(reinterpret_cast<const int4*>(x) + i);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int k = 0; k < kV; ++k) mx = max(mx, __float_as_uint(fabsf(fx_ld<T>(e, k))));
  }
  for (int64_t i = nv * kV + tid; i < n; i += stride)
    mx = max(mx, __float_as_uint(fabsf(fx_ld<T>(x, i))));
  mx = fx_warp_max_u32(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = threadIdx.x < kFxThreads / 32 ? red[threadIdx.x] : 0u;
    v = fx_warp_max_u32(v);
    if (threadIdx.x == 0) atomicMax(mx_out, v);   // non-negative floats order as their bits
  }
}

// the smallest e with round(max / 2^e) <= 32767 (every CTA derives it from the same max)
__device__ __forceinline__ int fx_act_exponent(uint32_t bits) {
  const float m = __uint_as_float(bits);
  if (!(m > 0.0f)) return 0;
  int p;
  frexpf(m, &p);
  int e = p - 16;
  while (roundf(ldexpf(m, -e)) > 32767.0f) ++e;
  while (roundf(ldexpf(m, -(e - 1))) <= 32767.0f) --e;
  return e;
}

template <typename T>
__global__ void __launch_bounds__(kFxThreads) k_fxp_quant_act(const T* __restrict__ x, int64_t n,
                                                              const uint32_t* __restrict__ mx,
                                                              int16_t* __restrict__ q,
                                                              int32_t* __restrict__ e_out) {
  const int e = fx_act_exponent(*mx);
  if (blockIdx.x == 0 && threadIdx.x == 0) *e_out = e;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float sc = ldexpf(1.0f, -e);   // x 2^-e is exact as a product with 2^-e ...
  constexpr int kV = 16 / sizeof(T);
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(q)) & 15) == 0 &&
                   e > -126 && e < 126;   // ... while 2^-e is a normal float
  const int64_t nv = vec ? n / kV : 0;
  for (int64_t i = tid; i < nv; i += stride) {
    const int4 raw = __ldg(reinterpret_cast<const int4*>(x) + i);
    const T* el = reinterpret_cast<const T*>(&raw);
    int16_t o[kV];
#pragma unroll
    for (int k = 0; k < kV; ++k) o[k] = (int16_t)roundf(__fmul_rn(fx_ld<T>(el, k), sc));
    if constexpr (kV == 8) {
      *reinterpret_cast<int4*>(q + i * kV) = *reinterpret_cast<const int4*>(o);
    } else {
      *reinterpret_cast<int2*>(q + i * kV) = *reinterpret_cast<const int2*>(o);
    }
  }
  for (int64_t i = nv * kV + tid; i < n; i += stride)
    q[i] = (int16_t)roundf(ldexpf(fx_ld<T>(x, i), -e));
}

// ---------------------------------------------------------------- F3 / F4 elementwise
__global__ void __launch_bounds__(kFxThreads) k_fxp_sigmoid(const int32_t* __restrict__ x, int64_t n,
                                                            int32_t* __restrict__ y,
                                                            const SigLut Lp) {
  __shared__ int32_t L[kFxNsig + 1];
  if (threadIdx.x <= kFxNsig) L[threadIdx.x] = Lp.y[threadIdx.x];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n >> 2;
  const int4* x4 = reinterpret_cast<const int4*>(x);
  int4* y4 = reinterpret_cast<int4*>(y);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const int4 v = __ldg(x4 + i);
    y4[i] = make_int4(fx_sigmoid(v.x, L), fx_sigmoid(v.y, L), fx_sigmoid(v.z, L),
                      fx_sigmoid(v.w, L));
  }
  for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = fx_sigmoid(x[i], L);
}

__global__ void __launch_bounds__(kFxThreads) k_fxp_inv_sqrt(const uint64_t* __restrict__ v,
                                                             const int32_t* __restrict__ e,
                                                             int64_t n, uint32_t* __restrict__ y,
                                                             int32_t* __restrict__ ey,
                                                             const RsqLut Lp) {
  __shared__ uint32_t L[24];
  if (threadIdx.x < 24) L[threadIdx.x] = Lp.g[threadIdx.x];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t vi = __ldg(reinterpret_cast<const unsigned long long*>(v) + i);
    if (vi == 0) {   // outside the domain (v > 0): defined as y = 0, ey = 0
      y[i] = 0;
      ey[i] = 0;
      continue;
    }
    uint32_t yi;
    int ei;
    fx_inv_sqrt(vi, __ldg(e + i), L, yi, ei);
    y[i] = yi;
    ey[i] = ei;
  }
}

// ---------------------------------------------------------------- F5 RMSNorm (Eq. 1)
// One CTA per row: the row is staged in shared memory as int16 (one HBM read), the int64
// sum of squares and the int64 max |t| are block reductions, the output is written once.
__device__ __forceinline__ int64_t fx_block_sum_i64(int64_t v, int64_t* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int64_t s = 0;
#pragma unroll
  for (int w = 0; w < kFxThreads / 32; ++w) s += red[w];
  return s;
}
__device__ __forceinline__ int64_t fx_block_max_i64(int64_t v, int64_t* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int64_t s = 0;
#pragma unroll
  for (int w = 0; w < kFxThreads / 32; ++w) s = max(s, red[w]);
  return s;
}

__global__ void __launch_bounds__(kFxThreads) k_fxp_rmsnorm(const int16_t* __restrict__ xq,
                                                            const int32_t* __restrict__ ex_dev,
                                                            const int8_t* __restrict__ wq, int ew,
                                                            double eps, int64_t sd, int rows, int d,
                                                            int16_t* __restrict__ out,
                                                            int32_t* __restrict__ eo,
                                                            const RsqLut Lp) {
  extern __shared__ __align__(16) int16_t row_s[];
  __shared__ int64_t red[kFxThreads / 32];
  __shared__ uint32_t L[24];
  if (threadIdx.x < 24) L[threadIdx.x] = Lp.g[threadIdx.x];
  __syncthreads();
  const int ex = *ex_dev;
  // eps_q = round(d eps 2^(-2 ex - k2)) in binary64 (F5), on the even grid 2^k2 of the sum:
  // k2 = 0 unless the activations are so small that eps_q would exceed 2^60 (reading F5b)
  int k2 = 0;
  while (round(ldexp(__dmul_rn((double)d, eps), -2 * ex - k2)) > 0x1p60) k2 += 2;
  const int64_t eps_q = (int64_t)round(ldexp(__dmul_rn((double)d, eps), -2 * ex - k2));
  const bool vec = (d & 7) == 0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int16_t* x = xq + (int64_t)r * d;
    int64_t S = 0;
    if (vec) {   // 8 int16 per 16-byte load
      const int4* x4 = reinterpret_cast<const int4*>(x);
      int4* s4 = reinterpret_cast<int4*>(row_s);
      for (int i = threadIdx.x; i < d / 8; i += kFxThreads) {
        const int4 v = __ldg(x4 + i);
        s4[i] = v;
        const int32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int32_t lo = (int16_t)(w[k] & 0xffff), hi = w[k] >> 16;
          S += (int64_t)(lo * lo) + (int64_t)(hi * hi);   // each square < 2^30
        }
      }
    } else {
      for (int i = threadIdx.x; i < d; i += kFxThreads) {
        const int32_t v = x[i];
        row_s[i] = (int16_t)v;
        S += (int64_t)(v * v);
      }
    }
    S = fx_block_sum_i64(S, red);
    const uint64_t D = (uint64_t)fx_rha_shift(S, k2) + (uint64_t)eps_q;
    int16_t* o = out + (int64_t)r * d;
    if (D == 0) {
      for (int i = threadIdx.x; i < d; i += kFxThreads) o[i] = 0;
      if (threadIdx.x == 0) eo[r] = 0;
      continue;
    }
    uint32_t yq;
    int ey;
    fx_inv_sqrt(D, k2, L, yq, ey);
    const int64_t rsd = (int64_t)(((uint64_t)yq * (uint64_t)sd) >> 16);
    int64_t tmax = 0;
    for (int i = threadIdx.x; i < d; i += kFxThreads) {
      int64_t t = (int64_t)(row_s[i] * (int32_t)__ldg(wq + i)) * rsd;
      tmax = max(tmax, t < 0 ? -t : t);
    }
    tmax = fx_block_max_i64(tmax, red);
    int s = 0;
    while (fx_rha_shift(tmax, s) > 32767) ++s;
    for (int i = threadIdx.x; i < d; i += kFxThreads)
      o[i] = (int16_t)fx_rha_shift((int64_t)(row_s[i] * (int32_t)__ldg(wq + i)) * rsd, s);
    if (threadIdx.x == 0) eo[r] = s + ew + ey;
    __syncthreads();   // row_s is rewritten by the next row
  }
}

// Fast path for d = 256 NV (NV <= 12; c2-c4 widths 1024, 2048, 2560, 2816): one WARP per
// row, the row in registers (NV 16-byte vectors per lane), reductions by shuffles only,
// the gains staged once per CTA in shared memory.  Same arithmetic as k_fxp_rmsnorm.
constexpr int kFxWarpRows = 8;   // warps (rows in flight) per CTA
template <int NV>
__global__ void __launch_bounds__(kFxWarpRows * 32) k_fxp_rmsnorm_warp(
    const int16_t* __restrict__ xq, const int32_t* __restrict__ ex_dev,
    const int8_t* __restrict__ wq, int ew, double eps, int64_t sd, int rows,
    int16_t* __restrict__ out, int32_t* __restrict__ eo, const RsqLut Lp) {
  constexpr int d = NV * 256;
  __shared__ __align__(16) int8_t w_s[d];
  __shared__ uint32_t L[24];
  if (threadIdx.x < 24) L[threadIdx.x] = Lp.g[threadIdx.x];
  for (int i = threadIdx.x; i < d / 16; i += blockDim.x)
    reinterpret_cast<int4*>(w_s)[i] = __ldg(reinterpret_cast<const int4*>(wq) + i);
  __syncthreads();
  const int ex = *ex_dev;
  int k2 = 0;   // F5b (as k_fxp_rmsnorm)
  while (round(ldexp(__dmul_rn((double)d, eps), -2 * ex - k2)) > 0x1p60) k2 += 2;
  const int64_t eps_q = (int64_t)round(ldexp(__dmul_rn((double)d, eps), -2 * ex - k2));
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * kFxWarpRows + (threadIdx.x >> 5);
  for (int r = wid; r < rows; r += gridDim.x * kFxWarpRows) {
    const int4* x4 = reinterpret_cast<const int4*>(xq + (int64_t)r * d);
    int4 v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = __ldg(x4 + lane + 32 * j);
    int64_t S = 0;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {   // two squares (each <= 2^30) per uint32, then widen
        const int32_t lo = (int16_t)(w4[k] & 0xffff), hi = w4[k] >> 16;
        S += (int64_t)((uint32_t)(lo * lo) + (uint32_t)(hi * hi));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    const uint64_t D = (uint64_t)fx_rha_shift(S, k2) + (uint64_t)eps_q;
    int16_t* orow = out + (int64_t)r * d;
    if (D == 0) {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        reinterpret_cast<int4*>(orow)[lane + 32 * j] = make_int4(0, 0, 0, 0);
      if (lane == 0) eo[r] = 0;
      continue;
    }
    uint32_t yq;
    int ey;
    fx_inv_sqrt(D, k2, L, yq, ey);
    const int64_t rsd = (int64_t)(((uint64_t)yq * (uint64_t)sd) >> 16);
    // x * w per element (|.| < 2^22, int32), then the int64 product with rsd
    int32_t xw[NV][8];
    int64_t tmax = 0;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int2 wv = *reinterpret_cast<const int2*>(w_s + (lane + 32 * j) * 8);
      const int32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int32_t xv = (int16_t)((w4[k >> 1] >> ((k & 1) * 16)) & 0xffff);
        const int32_t wk = (int8_t)(((k < 4 ? wv.x : wv.y) >> ((k & 3) * 8)) & 0xff);
        xw[j][k] = xv * wk;
        const int32_t a = xw[j][k] < 0 ? -xw[j][k] : xw[j][k];
        tmax = max(tmax, (int64_t)a);
      }
    }
    // max |t| = max |x w| * rsd (rsd > 0): one int64 product instead of d
    tmax *= rsd;
#pragma unroll
    for (int o = 16; o; o >>= 1) tmax = max(tmax, (int64_t)__shfl_xor_sync(0xffffffffu, tmax, o));
    int s = 0;
    while (fx_rha_shift(tmax, s) > 32767) ++s;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      int32_t o8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o8[k] = (int32_t)fx_rha_shift((int64_t)xw[j][k] * rsd, s);
      int4 ov;
      ov.x = (o8[0] & 0xffff) | (o8[1] << 16);
      ov.y = (o8[2] & 0xffff) | (o8[3] << 16);
      ov.z = (o8[4] & 0xffff) | (o8[5] << 16);
      ov.w = (o8[6] & 0xffff) | (o8[7] << 16);
      reinterpret_cast<int4*>(orow)[lane + 32 * j] = ov;
    }
    if (lane == 0) eo[r] = s + ew + ey;
  }
}

// ---------------------------------------------------------------- F6 W8A16 BitLinear
// int16 rows -> two s8 digit planes for the int8 tensor cores: a = 256 hi + lo' + 128 with
// hi = a >> 8 in [-128, 127] and lo' = (a & 255) - 128 in [-128, 127]; pads (k >= K) are
// 0 in both planes (their ternary codes are 0, so nothing is lost); per-row digit sums are
// the GEMM's q-sum corrections.  One warp per row.
__global__ void __launch_bounds__(256) k_fxp_split(const int16_t* __restrict__ a, int m, int k,
                                                    int ldq, int8_t* __restrict__ hi,
                                                    int8_t* __restrict__ lo,
                                                    int32_t* __restrict__ qs_hi,
                                                    int32_t* __restrict__ qs_lo) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= m) return;
  const int16_t* ar = a + (int64_t)r * k;
  int8_t* hr = hi + (int64_t)r * ldq;
  int8_t* lr = lo + (int64_t)r * ldq;
  int32_t sh = 0, sl = 0;
  for (int c = lane * 4; c < ldq; c += 128) {   // 4 columns per lane: one 32-bit store each
    uint32_t ph = 0, pl = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int32_t h = 0, l = 0;
      if (c + j < k) {
        const int32_t v = ar[c + j];
        h = v >> 8;                  // arithmetic: floor(v / 256)
        l = (v & 255) - 128;
      }
      sh += h;
      sl += l;
      ph |= (uint32_t)(h & 255) << (8 * j);
      pl |= (uint32_t)(l & 255) << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(hr + c) = ph;
    *reinterpret_cast<uint32_t*>(lr + c) = pl;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sh += __shfl_xor_sync(0xffffffffu, sh, o);
    sl += __shfl_xor_sync(0xffffffffu, sl, o);
  }
  if (lane == 0) {
    qs_hi[r] = sh;
    qs_lo[r] = sl;
  }
}

// a row of K ones (pads 0) and its sum: contracting it gives each output's sum_k t[n][k]
__global__ void k_fxp_ones(int8_t* __restrict__ ones, int k, int ldq, int32_t* __restrict__ qs) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ldq; c += gridDim.x * blockDim.x)
    ones[c] = c < k ? 1 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *qs = k;
}

// (bq, eb) = F1([beta], shift 6) on the device: the same frexp rule as k_fxp_scales
__device__ __forceinline__ void fx_beta(float beta, int& bq, int& eb) {
  int p;
  const float f = frexpf(fabsf(beta), &p);
  eb = ((double)f >= 0.70710678118654752440 ? p : p - 1) - 6;
  bq = (int)roundf(ldexpf(beta, -eb));
}

// acc = 256 acc_hi + acc_lo + 128 rowsum (exact), p = acc bq, per-row int16 requantization
__global__ void __launch_bounds__(kFxThreads) k_fxp_combine(
    const int32_t* __restrict__ acc_hi, const int32_t* __restrict__ acc_lo, int ldacc,
    const int32_t* __restrict__ rowsum, const float* __restrict__ scale, int n, int m,
    const int32_t* __restrict__ en, int16_t* __restrict__ y, int ldy, int32_t* __restrict__ ey) {
  __shared__ int64_t red[kFxThreads / 32];
  int bq, eb;
  fx_beta(__ldg(scale), bq, eb);
  for (int r = blockIdx.x; r < m; r += gridDim.x) {
    const int32_t* h = acc_hi + (int64_t)r * ldacc;
    const int32_t* l = acc_lo + (int64_t)r * ldacc;
    int64_t pmax = 0;
    for (int c = threadIdx.x; c < n; c += kFxThreads) {
      const int64_t acc = 256 * (int64_t)h[c] + l[c] + 128 * (int64_t)__ldg(rowsum + c);
      const int64_t pv = acc * bq;
      pmax = max(pmax, pv < 0 ? -pv : pv);
    }
    pmax = fx_block_max_i64(pmax, red);
    int s = 0;
    while (fx_rha_shift(pmax, s) > 32767) ++s;
    int16_t* yr = y + (int64_t)r * ldy;
    for (int c = threadIdx.x; c < n; c += kFxThreads) {
      const int64_t acc = 256 * (int64_t)h[c] + l[c] + 128 * (int64_t)__ldg(rowsum + c);
      yr[c] = (int16_t)fx_rha_shift(acc * bq, s);
    }
    if (threadIdx.x == 0) ey[r] = s + en[r] + eb;
    __syncthreads();   // red is reused by the next row
  }
}

// ---------------------------------------------------------------- host side
static SigLut sig_lut() {   // F3: y_i = floor(sigma(i) 2^15), sigma in binary64
  SigLut L;
  for (int i = 0; i <= kFxNsig; ++i)
    L.y[i] = (int32_t)std::floor(std::ldexp(1.0 / (1.0 + std::exp(-(double)i)), kFxYexp));
  return L;
}
static RsqLut rsq_lut() {   // F4: seeds 1/sqrt(1 + (k + 1/2)/8) in Q30, k = 0..23
  RsqLut L;
  for (int k = 0; k < 24; ++k)
    L.g[k] = (uint32_t)std::llround(std::ldexp(1.0, 30) / std::sqrt(1.0 + (k + 0.5) / 8.0));
  return L;
}

cudaError_t launch_fxp_scales(const float* w, int n, int shift, int8_t* wq, int32_t* e,
                              int32_t* status, cudaStream_t s) {
  k_fxp_scales<<<1, 1024, 0, s>>>(w, n, shift, wq, e, status);
  return cudaGetLastError();
}

cudaError_t launch_fxp_quant_act(const void* x, int dt, int64_t n, int16_t* q, int32_t* e,
                                 uint32_t* ws, cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(ws, 0, sizeof(uint32_t), s);
  if (err != cudaSuccess) return err;
  const int grid = fx_grid(n, kFxThreads * 8);
  if (dt == TERN_BF16) {
    k_fxp_absmax<__nv_bfloat16><<<grid, kFxThreads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), n, ws);
    k_fxp_quant_act<__nv_bfloat16><<<grid, kFxThreads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), n, ws, q, e);
  } else {
    k_fxp_absmax<float><<<grid, kFxThreads, 0, s>>>(static_cast<const float*>(x), n, ws);
    k_fxp_quant_act<float><<<grid, kFxThreads, 0, s>>>(static_cast<const float*>(x), n, ws, q, e);
  }
  return cudaGetLastError();
}

cudaError_t launch_fxp_sigmoid(const int32_t* x, int64_t n, int32_t* y, cudaStream_t s) {
  static const SigLut L = sig_lut();
  if (n == 0) return cudaSuccess;
  k_fxp_sigmoid<<<fx_grid(n, kFxThreads * 16), kFxThreads, 0, s>>>(x, n, y, L);
  return cudaGetLastError();
}

cudaError_t launch_fxp_inv_sqrt(const uint64_t* v, const int32_t* e, int64_t n, uint32_t* y,
                                int32_t* ey, cudaStream_t s) {
  static const RsqLut L = rsq_lut();
  if (n == 0) return cudaSuccess;
  k_fxp_inv_sqrt<<<fx_grid(n, kFxThreads * 8), kFxThreads, 0, s>>>(v, e, n, y, ey, L);
  return cudaGetLastError();
}

cudaError_t launch_fxp_rmsnorm(const int16_t* xq, const int32_t* ex, const int8_t* wq, int ew,
                               double eps, int rows, int d, int16_t* out, int32_t* eo,
                               cudaStream_t s) {
  static const RsqLut L = rsq_lut();
  if (rows == 0) return cudaSuccess;
  const int64_t sd = std::llround(std::ldexp(std::sqrt((double)d), 16));   // sqrt(d) in Q16
  const size_t smem = ((size_t)d * sizeof(int16_t) + 15) / 16 * 16;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_fxp_rmsnorm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (d % 256 == 0 && d <= 12 * 256 && ((reinterpret_cast<uintptr_t>(wq) |
                                           reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    const int want = (rows + kFxWarpRows - 1) / kFxWarpRows;
    const int grid = want < fx_sms() * 8 ? want : fx_sms() * 8;
#define TERN_FXW(NV)                                                                         \
  case NV:                                                                                   \
    k_fxp_rmsnorm_warp<NV><<<grid, kFxWarpRows * 32, 0, s>>>(xq, ex, wq, ew, eps, sd, rows, \
                                                              out, eo, L);                  \
    return cudaGetLastError();
    switch (d / 256) {
      TERN_FXW(1) TERN_FXW(2) TERN_FXW(3) TERN_FXW(4) TERN_FXW(5) TERN_FXW(6)
      TERN_FXW(7) TERN_FXW(8) TERN_FXW(9) TERN_FXW(10) TERN_FXW(11) TERN_FXW(12)
    }
#undef TERN_FXW
  }
  const int grid = rows < fx_sms() * 8 ? rows : fx_sms() * 8;
  k_fxp_rmsnorm<<<grid, kFxThreads, smem, s>>>(xq, ex, wq, ew, eps, sd, rows, d, out, eo, L);
  return cudaGetLastError();
}

cudaError_t launch_fxp_split(const int16_t* a, int m, int k, int ldq, int8_t* hi, int8_t* lo,
                             int32_t* qs_hi, int32_t* qs_lo, int8_t* ones, int32_t* qs_ones,
                             cudaStream_t s) {
  k_fxp_ones<<<(ldq + 255) / 256, 256, 0, s>>>(ones, k, ldq, qs_ones);
  if (m > 0) k_fxp_split<<<(m + 7) / 8, 256, 0, s>>>(a, m, k, ldq, hi, lo, qs_hi, qs_lo);
  return cudaGetLastError();
}

cudaError_t launch_fxp_combine(const int32_t* acc_hi, const int32_t* acc_lo, int ldacc,
                               const int32_t* rowsum, const float* scale, int n, int m,
                               const int32_t* en, int16_t* y, int ldy, int32_t* ey,
                               cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int grid = m < fx_sms() * 4 ? m : fx_sms() * 4;
  k_fxp_combine<<<grid, kFxThreads, 0, s>>>(acc_hi, acc_lo, ldacc, rowsum, scale, n, m, en, y,
                                            ldy, ey);
  return cudaGetLastError();
}

}  // namespace tern
