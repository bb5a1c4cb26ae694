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
__device__ __forceinline__ int32_t fx_sigmoid(int32_t x, const SigLut& L) {
  const uint32_t a = x < 0 ? 0u - (uint32_t)x : (uint32_t)x;
  int32_t y;
  if (a >= (uint32_t)(kFxNsig << kFxXexp)) {
    y = L.y[kFxNsig];
  } else {
    const int i = (int)(a >> kFxXexp);
    const int32_t fr = (int32_t)(a & ((1u << kFxXexp) - 1));
    const int32_t y0 = L.y[i], y1 = L.y[i + 1];
    y = y0 + (((y1 - y0) * fr) >> kFxXexp);   // (y1 - y0) * fr < 2^15 * 2^6: no overflow
  }
  return x < 0 ? (1 << kFxYexp) - y : y;
}

// F4: 1/sqrt(v 2^e) = y 2^ey, v > 0
__device__ __forceinline__ void fx_inv_sqrt(uint64_t v, int e, const RsqLut& L, uint32_t& y_out,
                                            int& ey_out) {
  const int p = 63 - __clzll((long long)v);
  uint64_t m = p >= 30 ? v >> (p - 30) : v << (30 - p);
  int E = e + p;
  if (E & 1) {
    m <<= 1;
    E -= 1;
  }
  const int k = (int)((m - (1ull << 30)) >> 27);
  uint64_t y = L.g[k];
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
  if constexpr (sizeof(T) == 4) return __ldg(reinterpret_cast<const float*>(p) + i);
  else return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

template <typename T>
__global__ void __launch_bounds__(kFxThreads) k_fxp_absmax(const T* __restrict__ x, int64_t n,
                                                           uint32_t* __restrict__ mx_out) {
  __shared__ uint32_t red[kFxThreads / 32];
  uint32_t mx = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
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
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    q[i] = (int16_t)roundf(ldexpf(fx_ld<T>(x, i), -e));
}

// ---------------------------------------------------------------- F3 / F4 elementwise
__global__ void __launch_bounds__(kFxThreads) k_fxp_sigmoid(const int32_t* __restrict__ x, int64_t n,
                                                            int32_t* __restrict__ y,
                                                            const SigLut L) {
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
                                                             const RsqLut L) {
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
                                                            const RsqLut L) {
  extern __shared__ __align__(16) int16_t row_s[];
  __shared__ int64_t red[kFxThreads / 32];
  const int ex = *ex_dev;
  // eps_q = round(d eps 2^(-2 ex)) in binary64 (F5): the same operations as the definition
  // (clamped to 2^60 so S + eps_q stays in 64 bits for tiny activations)
  const double eps_d = round(ldexp(__dmul_rn((double)d, eps), -2 * ex));
  const int64_t eps_q = eps_d > 0x1p60 ? (1ll << 60) : (int64_t)eps_d;
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
    const uint64_t D = (uint64_t)S + (uint64_t)eps_q;
    int16_t* o = out + (int64_t)r * d;
    if (D == 0) {
      for (int i = threadIdx.x; i < d; i += kFxThreads) o[i] = 0;
      if (threadIdx.x == 0) eo[r] = 0;
      continue;
    }
    uint32_t yq;
    int ey;
    fx_inv_sqrt(D, 0, L, yq, ey);
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
  const int grid = rows < fx_sms() * 8 ? rows : fx_sms() * 8;
  k_fxp_rmsnorm<<<grid, kFxThreads, smem, s>>>(xq, ex, wq, ew, eps, sd, rows, d, out, eo, L);
  return cudaGetLastError();
}

}  // namespace tern
