// k_bwd.cu -- SURVEY 8(f) f4(iii): Alg. 1 BackwardPass of one
// BitLinear with the straight-through estimator, readings B1-B6:
//
//   dY = dO x W~^T                      W~ = t m_w, the forward's ternary weight  (B1)
//   dX = rms_norm_bwd(dY, X, mu, r)     (B4/B5; mu = 0 for the RMSNorm)
//   dW = dO^T x Y~                      Y~ = q deq, the forward's activation     (B2)
//   db = sum over tokens of dO
//
// The forward's r, q, deq are recomputed by the forward's own quantizer (k_quant, B3).
// The two contractions are dense, so they run on the tensor cores (k_bwd_mma,
// tcgen05.mma kind::f16, bf16 operands, fp32 accumulators in TMEM): the fp32 operand is
// split into bf16 hi + lo parts laid side by side along K (hi = bf16(v), lo = bf16(v - hi),
// |v - hi - lo| <= 2^-16 |v|), the exact operand (the trits, the int8 q) is read twice, so
// one GEMM over K' = 2K gives the fp32-accurate product (B7).  Operands are K-major bf16
// rows prepared by small transpose kernels; the long dW contraction (over the tokens) is
// split over K with fp32 partials summed in slice order.  The CUDA-core fp32 GEMM
// (k_bwd_gemm) stays as the reference path (tern_set_bwd_tc(0)).  Sums run in a fixed
// order (no atomics), so results are deterministic.
#include "common.cuh"
#include "internal.h"

namespace tern {

constexpr int kBT = 128;   // output tile (rows and columns)
constexpr int kBKc = 16;   // contraction step
constexpr int kBwdThreads = 256;

// A operand: fp32, either row-major [I][Kc] (lda) or transposed storage [Kc][I] (lda)
// B operand: [Kc][J] bytes (ldb): u8 fields e (value e - 1) or int8 q scaled by bscale[k]
template <bool A_T, bool B_Q>
__global__ void __launch_bounds__(kBwdThreads)
    k_bwd_gemm(const float* __restrict__ A, int lda, const uint8_t* __restrict__ Bm, int ldb,
               const float* __restrict__ bscale, const float* __restrict__ alpha, int I, int J,
               int Kc, float* __restrict__ Cm, int ldc) {
  __shared__ __align__(16) float As[2][kBKc][kBT];
  __shared__ __align__(16) float Bs[2][kBKc][kBT];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = blockIdx.y * kBT, j0 = blockIdx.x * kBT;
  pdl_wait();
  pdl_launch_dependents();
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0f;

  float ra[8];   // staged A values of this thread (next k-step)
  float rb[8];   // staged B values
  auto load = [&](int k0) {
    if (!A_T) {
      // rows i0 + tid/2, k0 + (tid&1)*8 .. +8
      const int r = tid >> 1, c = (tid & 1) * 8;
      const int gi = i0 + r;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int gk = k0 + c + u;
        ra[u] = (gi < I && gk < Kc) ? __ldg(A + (int64_t)gi * lda + gk) : 0.0f;
      }
    } else {
      // k row k0 + tid/16, i columns (tid&15)*8 .. +8
      const int kr = tid >> 4, c = (tid & 15) * 8;
      const int gk = k0 + kr;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int gi = i0 + c + u;
        ra[u] = (gk < Kc && gi < I) ? __ldg(A + (int64_t)gk * lda + gi) : 0.0f;
      }
    }
    const int kr = tid >> 4, c = (tid & 15) * 8;
    const int gk = k0 + kr;
    const float sc = (B_Q && gk < Kc) ? __ldg(bscale + gk) : 1.0f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int gj = j0 + c + u;
      float v = 0.0f;
      if (gk < Kc && gj < J) {
        const uint8_t b = __ldg(Bm + (int64_t)gk * ldb + gj);
        v = B_Q ? __fmul_rn((float)(int8_t)b, sc) : (float)((int)b - 1);
      }
      rb[u] = v;
    }
  };
  auto store = [&](int buf) {
    if (!A_T) {
      const int r = tid >> 1, c = (tid & 1) * 8;
#pragma unroll
      for (int u = 0; u < 8; ++u) As[buf][c + u][r] = ra[u];
    } else {
      const int kr = tid >> 4, c = (tid & 15) * 8;
#pragma unroll
      for (int u = 0; u < 8; ++u) As[buf][kr][c + u] = ra[u];
    }
    const int kr = tid >> 4, c = (tid & 15) * 8;
#pragma unroll
    for (int u = 0; u < 8; ++u) Bs[buf][kr][c + u] = rb[u];
  };

  const int nk = (Kc + kBKc - 1) / kBKc;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * kBKc);   // global loads in flight during the FMAs
#pragma unroll
    for (int kk = 0; kk < kBKc; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = __fmaf_rn(a[x], b[y], acc[x][y]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
  const float al = alpha ? __ldg(alpha) : 1.0f;
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int gi = i0 + (x < 4 ? ty * 4 + x : 64 + ty * 4 + x - 4);
    if (gi >= I) continue;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const int gj = j0 + (y < 4 ? tx * 4 + y : 64 + tx * 4 + y - 4);
      if (gj < J) Cm[(int64_t)gi * ldc + gj] = __fmul_rn(acc[x][y], al);
    }
  }
}

// rms_norm_bwd of one row per CTA, binary64 sums (B4-B6):
//   dsig = sum dY (x - mu) (-1/2) r^3;  dmu = sum(-r dY) + dsig mean(x - mu)  (centred only)
//   dX = r dY + 2 dsig (x - mu) / K + dmu / K
__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}
// 4 consecutive activation values (vector v of the row) as floats: fp32 or bf16 storage
template <typename TX> __device__ __forceinline__ float4 ld4(const TX* row, int v);
template <> __device__ __forceinline__ float4 ld4<float>(const float* row, int v) {
  return __ldg(reinterpret_cast<const float4*>(row) + v);
}
template <> __device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* row, int v) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(row) + v);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}

// NV float4 vectors of x and dY per thread held in registers (K <= 1024 NV), one read of each
template <int NV, typename TX>
__global__ void __launch_bounds__(kBwdThreads)
    k_bwd_norm(const TX* __restrict__ x, const float* __restrict__ dY, const float* __restrict__ r,
               int K, int centred, float* __restrict__ dX) {
  __shared__ double red[kBwdThreads / 32];
  const int row = blockIdx.x;
  const TX* xr = x + (int64_t)row * K;
  const float4* dyr = reinterpret_cast<const float4*>(dY + (int64_t)row * K);
  const int nv = K / 4;
  pdl_wait();
  pdl_launch_dependents();
  float4 xv[NV], gv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = threadIdx.x + i * kBwdThreads;
    xv[i] = v < nv ? ld4<TX>(xr, v) : make_float4(0.f, 0.f, 0.f, 0.f);
    gv[i] = v < nv ? __ldg(dyr + v) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float mu = 0.0f;
  if (centred) {
    double sx = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      sx += ((double)xv[i].x + (double)xv[i].y) + ((double)xv[i].z + (double)xv[i].w);
    mu = (float)(block_sum_d(sx, red) / (double)K);
  }
  double sdx = 0.0, sdy = 0.0, sxc = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = threadIdx.x + i * kBwdThreads;
    if (v >= nv) continue;
    const float xs[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
    const float gs[4] = {gv[i].x, gv[i].y, gv[i].z, gv[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double xc = (double)xs[j] - (double)mu, g = (double)gs[j];
      sdx = fma(g, xc, sdx);
      sdy += g;
      sxc += xc;
    }
  }
  sdx = block_sum_d(sdx, red);
  const double rd = (double)__ldg(r + row);
  const double dsig = sdx * -0.5 * rd * rd * rd;
  double dmu = 0.0;
  if (centred) {
    sdy = block_sum_d(sdy, red);
    sxc = block_sum_d(sxc, red);
    dmu = -rd * sdy + dsig * (sxc / (double)K);
  }
  const double c1 = 2.0 * dsig / (double)K, c0 = dmu / (double)K;
  float4* dxr = reinterpret_cast<float4*>(dX + (int64_t)row * K);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = threadIdx.x + i * kBwdThreads;
    if (v >= nv) continue;
    const float xs[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
    const float gs[4] = {gv[i].x, gv[i].y, gv[i].z, gv[i].w};
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o[j] = (float)(rd * (double)gs[j] + c1 * ((double)xs[j] - (double)mu) + c0);
    dxr[v] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// the same with one warp per row (K <= 128 NV: 32 lanes x NV float4 each of x and dY): shuffle
// reductions only, no block barriers, 8 rows per CTA
template <int NV, typename TX>
__global__ void __launch_bounds__(256)
    k_bwd_norm_w(const TX* __restrict__ x, const float* __restrict__ dY, const float* __restrict__ r,
                 int M, int K, int centred, float* __restrict__ dX) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_wait();
  pdl_launch_dependents();
  if (row >= M) return;
  const TX* xr = x + (int64_t)row * K;
  const float4* dyr = reinterpret_cast<const float4*>(dY + (int64_t)row * K);
  const int nv = K / 4;
  float4 xv[NV], gv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = lane + i * 32;
    xv[i] = v < nv ? ld4<TX>(xr, v) : make_float4(0.f, 0.f, 0.f, 0.f);
    gv[i] = v < nv ? __ldg(dyr + v) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float mu = 0.0f;
  if (centred) {
    double sx = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      sx += ((double)xv[i].x + (double)xv[i].y) + ((double)xv[i].z + (double)xv[i].w);
    mu = (float)(warp_sum_f64(sx) / (double)K);
  }
  double sdx = 0.0, sdy = 0.0, sxc = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (lane + i * 32 >= nv) continue;
    const float xs[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
    const float gs[4] = {gv[i].x, gv[i].y, gv[i].z, gv[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double xc = (double)xs[j] - (double)mu, g = (double)gs[j];
      sdx = fma(g, xc, sdx);
      sdy += g;
      sxc += xc;
    }
  }
  sdx = warp_sum_f64(sdx);
  const double rd = (double)__ldg(r + row);
  const double dsig = sdx * -0.5 * rd * rd * rd;
  double dmu = 0.0;
  if (centred) {
    sdy = warp_sum_f64(sdy);
    sxc = warp_sum_f64(sxc);
    dmu = -rd * sdy + dsig * (sxc / (double)K);
  }
  const double c1 = 2.0 * dsig / (double)K, c0 = dmu / (double)K;
  float4* dxr = reinterpret_cast<float4*>(dX + (int64_t)row * K);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = lane + i * 32;
    if (v >= nv) continue;
    const float xs[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
    const float gs[4] = {gv[i].x, gv[i].y, gv[i].z, gv[i].w};
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o[j] = (float)(rd * (double)gs[j] + c1 * ((double)xs[j] - (double)mu) + c0);
    dxr[v] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

template <typename TX>
static cudaError_t launch_bwd_norm(const TX* x, const float* dY, const float* r, int m, int k,
                                   int centred, float* dX, cudaStream_t s) {
  // rows up to 1024 elements: a warp per row (registers, shuffles); longer rows: a CTA per row
  const unsigned gw = (unsigned)((m + 7) / 8);
  if (k <= 512) return launch_pdl(k_bwd_norm_w<4, TX>, dim3(gw), dim3(256), 0, s, x, dY, r, m, k, centred, dX);
  if (k <= 1024) return launch_pdl(k_bwd_norm_w<8, TX>, dim3(gw), dim3(256), 0, s, x, dY, r, m, k, centred, dX);
  const int nv = (k / 4 + kBwdThreads - 1) / kBwdThreads;   // float4 vectors per thread
  if (nv <= 1) return launch_pdl(k_bwd_norm<1, TX>, dim3(m), dim3(kBwdThreads), 0, s, x, dY, r, k, centred, dX);
  if (nv <= 2) return launch_pdl(k_bwd_norm<2, TX>, dim3(m), dim3(kBwdThreads), 0, s, x, dY, r, k, centred, dX);
  if (nv <= 4) return launch_pdl(k_bwd_norm<4, TX>, dim3(m), dim3(kBwdThreads), 0, s, x, dY, r, k, centred, dX);
  if (nv <= 8) return launch_pdl(k_bwd_norm<8, TX>, dim3(m), dim3(kBwdThreads), 0, s, x, dY, r, k, centred, dX);
  return launch_pdl(k_bwd_norm<16, TX>, dim3(m), dim3(kBwdThreads), 0, s, x, dY, r, k, centred, dX);
}

// db[n] = sum over the M tokens of dO[m][n]: 32 columns per CTA, 8 warps over the rows, the
// warps' partials combined in warp order
__global__ void __launch_bounds__(kBwdThreads)
    k_bwd_colsum(const float* __restrict__ dO, int M, int N, float* __restrict__ db) {
  __shared__ float part[8][32];
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + l;
  pdl_wait();
  pdl_launch_dependents();
  float s = 0.0f;
  if (n < N)
    for (int m = w; m < M; m += 8) s = __fadd_rn(s, __ldg(dO + (int64_t)m * N + n));
  part[w][l] = s;
  __syncthreads();
  if (w == 0 && n < N) {
    float t = part[0][l];
    for (int i = 1; i < 8; ++i) t = __fadd_rn(t, part[i][l]);
    db[n] = t;
  }
}


// ----------------------------------------------------------------- tensor-core path (B7)
constexpr int kMmaThreads = 192;   // warp 0 TMA, warp 1 MMA, warps 2-5 drain (TMEM quadrants)
constexpr int kBwdS = 4;           // ring stages
constexpr int kBwdKB = 64;         // bf16 elements per k-block (one 128-byte swizzle row)

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// C[i][j] (+ over the k-blocks [kb0, kb1) of this z-slice) = sum_k A[i][k] B[j][k], A and B
// K-major bf16 (TMA SW128), B's k-block index taken modulo nkb_b (the exact operand read
// for both halves of the hi | lo split).  ksplit == 1: out = alpha * C; else the slice's raw
// sums go to part[z][I][J].
template <int BN>
__global__ void __launch_bounds__(kMmaThreads, 1)
    k_bwd_mma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              int I, int J, int nkb, int nkb_b, int kb_per, const float* __restrict__ alpha,
              float* __restrict__ out, int ldo, float* __restrict__ part) {
  constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128;
  extern __shared__ __align__(1024) uint8_t bsm_raw[];
  uint8_t* sm = bsm_raw + ((1024u - (smem_u32(bsm_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;
  uint8_t* sB = sA + kBwdS * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kBwdS * B_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + kBwdS;
  uint64_t* tfull = bars + 2 * kBwdS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kBwdS + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.y * 128, j0 = blockIdx.x * BN, z = blockIdx.z;
  const int kb0 = z * kb_per, kb1 = min(nkb, kb0 + kb_per);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kBwdS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  if (warp == 0) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % kBwdS;
        if (g >= (uint32_t)kBwdS) mbar_wait(&empty[s], ((g / kBwdS) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * kBwdKB, i0);
        tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], (kb % nkb_b) * kBwdKB, j0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::f16: D f32 (1 << 4), A bf16 (1 << 7), B bf16 (1 << 10), both K-major, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      uint32_t g = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % kBwdS;
        mbar_wait(&full[s], (g / kBwdS) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + s * A_BYTES), b_addr = smem_u32(sB + s * B_BYTES);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)   // K = 16 bf16 = 32 bytes per MMA
          mma_bf16(tmem_base, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                   idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
  } else {
    const int quad = warp & 3;   // TMEM lanes [32 quad, 32 quad + 32)
    mbar_wait(tfull, 0);
    tc_fence_after();
    const float al = (part == nullptr && alpha) ? __ldg(alpha) : 1.0f;
    const bool empty_slice = kb1 <= kb0;
    // the ring is idle once the accumulator is complete: each drain warp stages 32 x 32
    // chunks there (row = lane), then writes them out row by row (128 contiguous bytes per
    // store instruction)
    float* stg = reinterpret_cast<float*>(sm) + (warp - 2) * 32 * 33;
    const int r0 = i0 + quad * 32;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 32; ++t)
        stg[lane * 33 + t] = empty_slice ? 0.0f : __fmul_rn(__uint_as_float(v[t]), al);
      __syncwarp();
      const int jc = j0 + c * 32 + lane;
      if (jc < J) {
        for (int r = 0; r < 32 && r0 + r < I; ++r) {
          float* dst = part ? part + ((int64_t)z * I + r0 + r) * J : out + (int64_t)(r0 + r) * ldo;
          dst[jc] = stg[r * 33 + lane];
        }
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<BN>(tmem_base);
  }
}

// out[i][j] = alpha * sum over the ks slices (in order) of part[z][i][j]
__global__ void k_bwd_reduce(const float* __restrict__ part, int ks, int64_t n, int J, int ldo,
                             const float* __restrict__ alpha, float* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  pdl_launch_dependents();
  if (e >= n) return;
  float s = __ldg(part + e);
  for (int z = 1; z < ks; ++z) s = __fadd_rn(s, __ldg(part + (int64_t)z * n + e));
  const float al = alpha ? __ldg(alpha) : 1.0f;
  out[(e / J) * ldo + e % J] = __fmul_rn(s, al);
}

__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(__fsub_rn(v, __bfloat162float(hi)));
}
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat16 ha, la, hb, lb;
  split_bf16(a, ha, la);
  split_bf16(b, hb, lb);
  hi = (uint32_t)__bfloat16_as_ushort(ha) | ((uint32_t)__bfloat16_as_ushort(hb) << 16);
  lo = (uint32_t)__bfloat16_as_ushort(la) | ((uint32_t)__bfloat16_as_ushort(lb) << 16);
}

// dO [m][n] fp32 -> Ady [m][2 np] = [hi | lo] (np = roundup(n, 64), zero padded),
// Adw [n][2 mp] = [hi | lo] of the transposed dO' = dO deq[m] (mp = roundup(m, 64)), and
// the column sums of this CTA's 64 rows, dbp[blockIdx.y][n] (rows in order); 64 x 64 tiles
// through shared memory, column pairs per thread (bf16x2 stores)
template <typename TD>
__global__ void __launch_bounds__(256)
    k_bwd_prep_do(const TD* __restrict__ dO, const float* __restrict__ deq, int m, int n,
                  int np, int mp, uint32_t* __restrict__ Ady, uint32_t* __restrict__ Adw,
                  float* __restrict__ dbp) {
  __shared__ float t[64][65];
  __shared__ float cs[8][64];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;   // 8 groups
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  pdl_wait();
  pdl_launch_dependents();
  {
    const int c = n0 + 2 * lane;   // this thread's column pair
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = grp * 8 + i, mm = m0 + r;
      float2 v = make_float2(0.0f, 0.0f);
      if (mm < m) {
        const TD* src = dO + (int64_t)mm * n + c;
        if (c + 1 < n && (n & 1) == 0) {
          if constexpr (sizeof(TD) == 4) {
            v = __ldg(reinterpret_cast<const float2*>(src));
          } else {
            const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(src));
            v = make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
          }
        } else {
          if (c < n) v.x = ld_act<TD>(src);
          if (c + 1 < n) v.y = ld_act<TD>(src + 1);
        }
      }
      if (mm < m && c < np) {
        uint32_t hi, lo;
        split2(v.x, v.y, hi, lo);
        Ady[((int64_t)mm * 2 * np + c) >> 1] = hi;
        Ady[((int64_t)mm * 2 * np + np + c) >> 1] = lo;
      }
      s0 = __fadd_rn(s0, v.x);
      s1 = __fadd_rn(s1, v.y);
      const float d = mm < m ? __ldg(deq + mm) : 0.0f;
      t[r][2 * lane] = __fmul_rn(v.x, d);
      t[r][2 * lane + 1] = __fmul_rn(v.y, d);
    }
    cs[grp][2 * lane] = s0;
    cs[grp][2 * lane + 1] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 64 && n0 + threadIdx.x < n) {
    float s = cs[0][threadIdx.x];
    for (int g = 1; g < 8; ++g) s = __fadd_rn(s, cs[g][threadIdx.x]);
    dbp[(int64_t)blockIdx.y * n + n0 + threadIdx.x] = s;
  }
  // transposed: row pair 2 lane of the tile, columns grp*8 .. +8
  const int mm = m0 + 2 * lane;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = grp * 8 + i, nn = n0 + c;
    if (nn < n && mm < mp) {
      uint32_t hi, lo;
      split2(t[2 * lane][c], t[2 * lane + 1][c], hi, lo);
      Adw[((int64_t)nn * 2 * mp + mm) >> 1] = hi;
      Adw[((int64_t)nn * 2 * mp + mp + mm) >> 1] = lo;
    }
  }
}

// db[n] = sum over the row blocks (in order) of dbp[b][n]: 32 columns per CTA, warp w sums
// the blocks w, w + 8, ... in order, the 8 warp partials are combined in warp order
__global__ void __launch_bounds__(256)
    k_bwd_dbsum(const float* __restrict__ dbp, int nb, int n, float* __restrict__ db) {
  __shared__ float ps[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  pdl_wait();
  pdl_launch_dependents();
  float s = 0.0f;
  if (c < n)
#pragma unroll 4
    for (int b = w; b < nb; b += 8) s = __fadd_rn(s, __ldg(dbp + (int64_t)b * n + c));
  ps[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < n) {
    float t = ps[0][lane];
    for (int i = 1; i < 8; ++i) t = __fadd_rn(t, ps[i][lane]);
    db[c] = t;
  }
}

// the exact operands, transposed to K-major bf16 (64 x 64 tiles): Tt [k][np] = e8[n][j] - 1
// (the trits of W~ without the scale) and Qt [k][mp] = q[m][j]; rows beyond `rows` are zero
__global__ void __launch_bounds__(256)
    k_bwd_prep_t(const uint8_t* __restrict__ src, int rows, int cols, int lds, int rows_p,
                 int is_e8, uint32_t* __restrict__ dst) {
  __shared__ float t[64][65];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  pdl_wait();
  pdl_launch_dependents();
  {
    const int cq = threadIdx.x & 15, rg = threadIdx.x >> 4;   // 4 columns, 16 row groups
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rg * 4 + i, rr = r0 + r;
      uint32_t w = 0;
      const int c = c0 + 4 * cq;
      if (rr < rows && c < cols) w = __ldg(reinterpret_cast<const uint32_t*>(src + (int64_t)rr * lds + c));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t b = (w >> (8 * j)) & 0xffu;
        float v = is_e8 ? (float)((int)b - 1) : (float)(int8_t)b;
        t[r][4 * cq + j] = (rr < rows && c + j < cols) ? v : 0.0f;
      }
    }
  }
  __syncthreads();
  const int rr = r0 + 2 * lane;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = grp * 8 + i, cc = c0 + c;
    if (cc < cols && rr < rows_p) {
      const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(t[2 * lane][c]));
      const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(t[2 * lane + 1][c]));
      dst[((int64_t)cc * rows_p + rr) >> 1] = lo | (hi << 16);
    }
  }
}

int g_bwd_tc = 1;   // tern_set_bwd_tc

static int bwd_sms() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

// C[I][J] = alpha * sum_{k < 2 kp_half} A[i][k] B[j][k mod kp_half], A [I][2 kp_half], B [J][kp_half]
// hi_only: the fp32 operand is exactly bf16 (lo = 0), so only the hi half is contracted
static cudaError_t bwd_mma(const __nv_bfloat16* A, const __nv_bfloat16* B, int I, int J,
                           int kp_half, const float* alpha, float* out, int ldo, float* part,
                           size_t part_floats, cudaStream_t s, bool hi_only = false) {
  constexpr int BN = 256;
  CUtensorMap ta, tb;
  if (!make_map_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, A, (uint64_t)2 * kp_half, (uint64_t)I,
                   (uint64_t)2 * kp_half * 2, kBwdKB, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, B, (uint64_t)kp_half, (uint64_t)J,
                   (uint64_t)kp_half * 2, kBwdKB, BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int nkb_b = kp_half / kBwdKB, nkb = hi_only ? nkb_b : 2 * nkb_b;
  const int tiles = ((I + 127) / 128) * ((J + BN - 1) / BN);
  // split the contraction when the tiles cannot fill the SMs (dW: few tiles, long K)
  int ks = 1;
  const int nsm = bwd_sms();
  if (tiles < nsm && part) {
    ks = nsm / tiles;
    if (ks > nkb / 8) ks = nkb / 8;
    if ((size_t)ks * I * J > part_floats) ks = (int)(part_floats / ((size_t)I * J));
    if (ks < 1) ks = 1;
  }
  const int kb_per = (nkb + ks - 1) / ks;
  ks = (nkb + kb_per - 1) / kb_per;
  constexpr int smem = kBwdS * (128 * 128 + BN * 128) + 1024 + 256;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_bwd_mma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaError_t e = launch_pdl(k_bwd_mma<BN>, dim3((J + BN - 1) / BN, (I + 127) / 128, ks),
                             dim3(kMmaThreads), (size_t)smem, s, ta, tb, I, J, nkb, nkb_b, kb_per,
                             alpha, out, ldo, ks > 1 ? part : (float*)nullptr);
  if (e != cudaSuccess || ks == 1) return e;
  const int64_t n = (int64_t)I * J;
  return launch_pdl(k_bwd_reduce, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
                    (const float*)part, ks, n, J, ldo, alpha, out);
}

static size_t al256(size_t b) { return (b + 255) / 256 * 256; }
static int rup64(int v) { return (v + 63) / 64 * 64; }

// workspace: q, deq, qsum, r, dY (fp32 [m][k]); the tensor-core path adds Ady [m][2 np],
// Adw [n][2 mp], Tt [k][np], Qt [k][mp] (bf16) and the dW slice partials
struct BwdWs {
  size_t q, deq, qsum, r, dy, ady, adw, tt, qt, dbp, part, part_floats, total;
};
static BwdWs bwd_ws(int m, int k, int n) {
  BwdWs w{};
  const size_t kp = (size_t)((k + kKAlign - 1) / kKAlign * kKAlign);
  const size_t np = rup64(n), mp = rup64(m);
  size_t o = 0;
  w.q = o; o += al256((size_t)m * kp);
  w.deq = o; o += al256((size_t)m * 4);
  w.qsum = o; o += al256((size_t)m * 4);
  w.r = o; o += al256((size_t)m * 4);
  w.dy = o; o += al256((size_t)m * k * 4);
  w.ady = o; o += al256((size_t)m * 2 * np * 2);
  w.adw = o; o += al256((size_t)n * 2 * mp * 2);
  w.tt = o; o += al256((size_t)k * np * 2);
  w.qt = o; o += al256((size_t)k * mp * 2);
  w.dbp = o; o += al256((size_t)(mp / 64) * n * 4);
  // split-K slices exist only while tiles * ks <= the SM count, and I x J <= tiles x 128 x 256,
  // so SMs x 128 x 256 floats always hold them (19 MB on 148 SMs, whatever the shape)
  int nsm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess || nsm < 148) {
    cudaGetLastError();   // no device (CPU host query): the B200 count
    nsm = 148;
  }
  w.part_floats = (size_t)nsm * 128 * 256;
  w.part = o; o += al256(w.part_floats * 4);
  w.total = o;
  return w;
}

size_t bwd_workspace(int m, int k, int n) { return bwd_ws(m, k, n).total; }

cudaError_t launch_bitlinear_bwd(const void* xv, int dt, int m, int k, const tern_weight& w,
                                 float eps, int norm, const void* dOv, float* dX, float* dW,
                                 float* db, void* ws, cudaStream_t s) {
  const bool bf = dt == TERN_BF16;   // (bf16 x and dO: the tensor-core path only, checked by the API)
  const float* x = static_cast<const float*>(xv);
  const float* dO = static_cast<const float*>(dOv);
  const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(xv);
  const __nv_bfloat16* dOb = static_cast<const __nv_bfloat16*>(dOv);
  if (m == 0) return cudaSuccess;
  const int kp = (k + kKAlign - 1) / kKAlign * kKAlign;
  const int n = w.n_out;
  const BwdWs L = bwd_ws(m, k, n);
  char* base = static_cast<char*>(ws);
  int8_t* q = reinterpret_cast<int8_t*>(base + L.q);
  float* deq = reinterpret_cast<float*>(base + L.deq);
  int32_t* qsum = reinterpret_cast<int32_t*>(base + L.qsum);
  float* r = reinterpret_cast<float*>(base + L.r);
  float* dY = reinterpret_cast<float*>(base + L.dy);
  // the forward's r, q, deq (B3)
  cudaError_t e = launch_quant(xv, dt, m, k, k, nullptr, eps, q, kp, deq, qsum, r, nullptr, s,
                               norm);
  if (e != cudaSuccess) return e;
  if (g_bwd_tc) {
    const int np = rup64(n), mp = rup64(m);
    auto* Ady = reinterpret_cast<__nv_bfloat16*>(base + L.ady);
    auto* Adw = reinterpret_cast<__nv_bfloat16*>(base + L.adw);
    auto* Tt = reinterpret_cast<__nv_bfloat16*>(base + L.tt);
    auto* Qt = reinterpret_cast<__nv_bfloat16*>(base + L.qt);
    float* part = reinterpret_cast<float*>(base + L.part);
    float* dbp = reinterpret_cast<float*>(base + L.dbp);
    const dim3 gp((np + 63) / 64, (mp + 63) / 64);
    e = bf ? launch_pdl(k_bwd_prep_do<__nv_bfloat16>, gp, dim3(256), 0, s, dOb, (const float*)deq,
                        m, n, np, mp, reinterpret_cast<uint32_t*>(Ady),
                        reinterpret_cast<uint32_t*>(Adw), dbp)
           : launch_pdl(k_bwd_prep_do<float>, gp, dim3(256), 0, s, dO, (const float*)deq, m, n,
                        np, mp, reinterpret_cast<uint32_t*>(Ady), reinterpret_cast<uint32_t*>(Adw),
                        dbp);
    if (e != cudaSuccess) return e;
    if (db) {
      e = launch_pdl(k_bwd_dbsum, dim3((n + 31) / 32), dim3(256), 0, s, (const float*)dbp,
                     mp / 64, n, db);
      if (e != cudaSuccess) return e;
    }
    e = launch_pdl(k_bwd_prep_t, dim3((k + 63) / 64, (np + 63) / 64), dim3(256), 0, s, w.e8, n, k,
                   kp, np, 1, reinterpret_cast<uint32_t*>(Tt));
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_bwd_prep_t, dim3((k + 63) / 64, (mp + 63) / 64), dim3(256), 0, s,
                   reinterpret_cast<const uint8_t*>(q), m, k, kp, mp, 0,
                   reinterpret_cast<uint32_t*>(Qt));
    if (e != cudaSuccess) return e;
    // dY [m][k] = (dO_hi | dO_lo) x (T | T)^T * m_w
    e = bwd_mma(Ady, Tt, m, k, np, w.scales, dY, k, part, L.part_floats, s, bf);
    if (e != cudaSuccess) return e;
    e = bf ? launch_bwd_norm(xb, dY, r, m, k, norm == TERN_NORM_CENTERED ? 1 : 0, dX, s)
           : launch_bwd_norm(x, dY, r, m, k, norm == TERN_NORM_CENTERED ? 1 : 0, dX, s);
    if (e != cudaSuccess) return e;
    // dW [n][k] = (dO'^T_hi | dO'^T_lo) x (q^T | q^T)^T
    e = bwd_mma(Adw, Qt, n, k, mp, nullptr, dW, k, part, L.part_floats, s);
    if (e != cudaSuccess) return e;
  } else {
    // dY = dO x W~^T: I = m tokens, J = k inputs, contraction over the n output rows of e8
    e = launch_pdl(k_bwd_gemm<false, false>, dim3((k + kBT - 1) / kBT, (m + kBT - 1) / kBT),
                   dim3(kBwdThreads), 0, s, dO, n, w.e8, kp, (const float*)nullptr, w.scales, m, k,
                   n, dY, k);
    if (e != cudaSuccess) return e;
    e = launch_bwd_norm(x, dY, r, m, k, norm == TERN_NORM_CENTERED ? 1 : 0, dX, s);
    if (e != cudaSuccess) return e;
    // dW = dO^T x Y~: I = n output rows, J = k inputs, contraction over the m tokens
    e = launch_pdl(k_bwd_gemm<true, true>, dim3((k + kBT - 1) / kBT, (n + kBT - 1) / kBT),
                   dim3(kBwdThreads), 0, s, dO, n, reinterpret_cast<const uint8_t*>(q), kp,
                   (const float*)deq, (const float*)nullptr, n, k, m, dW, k);
    if (e != cudaSuccess) return e;
  }
  if (db && !g_bwd_tc)
    e = launch_pdl(k_bwd_colsum, dim3((n + 31) / 32), dim3(kBwdThreads), 0, s, dO, m, n, db);
  return e;
}

}  // namespace tern
