// k_bwd.cu -- SURVEY 8(f) f4(iii): Alg. 1 BackwardPass of one
// BitLinear with the straight-through estimator, readings B1-B6:
//
//   dY = dO x W~^T                      W~ = t m_w, the forward's ternary weight  (B1)
//   dX = rms_norm_bwd(dY, X, mu, r)     (B4/B5; mu = 0 for the RMSNorm)
//   dW = dO^T x Y~                      Y~ = q deq, the forward's activation     (B2)
//   db = sum over tokens of dO
//
// The forward's r, q, deq are recomputed by the forward's own quantizer (k_quant, B3).
// The two contractions run on CUDA cores in fp32 (k_bwd_gemm): a 128 x 128 output tile per
// CTA, 8 x 8 per thread, operands staged through double-buffered shared memory; the
// ternary operand of dY is read from the weight's u8 copy (e = t + 1) and the int8
// activation of dW is scaled by deq as it is staged.  Sums run in a fixed order (no
// atomics), so results are deterministic.
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
__global__ void __launch_bounds__(kBwdThreads)
    k_bwd_norm(const float* __restrict__ x, const float* __restrict__ dY, const float* __restrict__ r,
               int K, int centred, float* __restrict__ dX) {
  __shared__ double red[kBwdThreads / 32];
  const int row = blockIdx.x;
  const float* xr = x + (int64_t)row * K;
  const float* dyr = dY + (int64_t)row * K;
  pdl_wait();
  pdl_launch_dependents();
  float mu = 0.0f;
  if (centred) {
    double sx = 0.0;
    for (int j = threadIdx.x; j < K; j += kBwdThreads) sx += (double)__ldg(xr + j);
    mu = (float)(block_sum_d(sx, red) / (double)K);
  }
  double sdx = 0.0, sdy = 0.0, sxc = 0.0;
  for (int j = threadIdx.x; j < K; j += kBwdThreads) {
    const double xc = (double)__ldg(xr + j) - (double)mu;
    const double g = (double)__ldg(dyr + j);
    sdx = fma(g, xc, sdx);
    sdy += g;
    sxc += xc;
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
  for (int j = threadIdx.x; j < K; j += kBwdThreads) {
    const double xc = (double)__ldg(xr + j) - (double)mu;
    dX[(int64_t)row * K + j] = (float)(rd * (double)__ldg(dyr + j) + c1 * xc + c0);
  }
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

size_t bwd_workspace(int m, int k, int n) {
  (void)n;
  const size_t kp = (size_t)((k + kKAlign - 1) / kKAlign * kKAlign);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  return al((size_t)m * kp) + 3 * al((size_t)m * 4) + al((size_t)m * k * 4);
}

cudaError_t launch_bitlinear_bwd(const float* x, int m, int k, const tern_weight& w, float eps,
                                 int norm, const float* dO, float* dX, float* dW, float* db,
                                 void* ws, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int kp = (k + kKAlign - 1) / kKAlign * kKAlign;
  const int n = w.n_out;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  char* p = static_cast<char*>(ws);
  int8_t* q = reinterpret_cast<int8_t*>(p);
  p += al((size_t)m * kp);
  float* deq = reinterpret_cast<float*>(p);
  p += al((size_t)m * 4);
  int32_t* qsum = reinterpret_cast<int32_t*>(p);
  p += al((size_t)m * 4);
  float* r = reinterpret_cast<float*>(p);
  p += al((size_t)m * 4);
  float* dY = reinterpret_cast<float*>(p);
  // the forward's r, q, deq (B3)
  cudaError_t e = launch_quant(x, TERN_F32, m, k, k, nullptr, eps, q, kp, deq, qsum, r, nullptr, s,
                               norm);
  if (e != cudaSuccess) return e;
  // dY = dO x W~^T: I = m tokens, J = k inputs, contraction over the n output rows of e8
  e = launch_pdl(k_bwd_gemm<false, false>, dim3((k + kBT - 1) / kBT, (m + kBT - 1) / kBT),
                 dim3(kBwdThreads), 0, s, dO, n, w.e8, kp, (const float*)nullptr, w.scales, m, k,
                 n, dY, k);
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_bwd_norm, dim3(m), dim3(kBwdThreads), 0, s, x, (const float*)dY,
                 (const float*)r, k, norm == TERN_NORM_CENTERED ? 1 : 0, dX);
  if (e != cudaSuccess) return e;
  // dW = dO^T x Y~: I = n output rows, J = k inputs, contraction over the m tokens
  e = launch_pdl(k_bwd_gemm<true, true>, dim3((k + kBT - 1) / kBT, (n + kBT - 1) / kBT),
                 dim3(kBwdThreads), 0, s, dO, n, reinterpret_cast<const uint8_t*>(q), kp,
                 (const float*)deq, (const float*)nullptr, n, k, m, dW, k);
  if (e != cudaSuccess) return e;
  if (db)
    e = launch_pdl(k_bwd_colsum, dim3((n + 31) / 32), dim3(kBwdThreads), 0, s, dO, m, n, db);
  return e;
}

}  // namespace tern
