// k_selftest.cu -- device self-checks of numerics shortcuts used by the kernels
// (exposed as tern_selftest for the GPU test suite).
//   0: rcp_fast(d) == __fdiv_rn(1, d) for every mantissa of every exponent
//      0..125 (d in [1, 2^126)), and rcp_ge1 likewise
//   1: sigmoid_c(x) == 1/(1+exp_c(-x)) with IEEE division over a dense x sweep
//   2: sigmoid2 (the paired vector sigmoid) == the same, except that results
//      below 2^-126 may be 0, over the same sweep
//   3: the conversion-free round half away from zero (and int extraction)
#include "common.cuh"

namespace tern {

__global__ void k_selftest_rcp(unsigned long long* bad) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;  // mantissa
  if (m >= (1u << 23)) return;
  unsigned long long nb = 0;
  for (int ex = 0; ex <= 125; ++ex) {
    const float d = __uint_as_float(((uint32_t)(ex + 127) << 23) | m);
    const uint32_t ref = __float_as_uint(__fdiv_rn(1.0f, d));
    nb += __float_as_uint(rcp_fast(d)) != ref;
    nb += __float_as_uint(rcp_ge1(d)) != ref;
  }
  if (nb) atomicAdd(bad, nb);
}

__global__ void k_selftest_sigmoid2(unsigned long long* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // pairs of the 2^24 points
  const float x0 = -96.0f + (float)(2 * i) * (192.0f / 16777216.0f);
  const float x1 = -96.0f + (float)(2 * i + 1) * (192.0f / 16777216.0f);
  float a0, a1;
  sigmoid2(x0, x1, a0, a1);
  const float b0 = __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_c(-x0)));
  const float b1 = __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_c(-x1)));
  unsigned long long nb = 0;
  nb += __float_as_uint(a0) != __float_as_uint(b0) && !(b0 < 0x1p-126f && a0 == 0.0f);
  nb += __float_as_uint(a1) != __float_as_uint(b1) && !(b1 < 0x1p-126f && a1 == 0.0f);
  if (nb) atomicAdd(bad, nb);
}

__global__ void k_selftest_sigmoid(unsigned long long* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // 2^24 points in [-96, 96)
  const float x = -96.0f + (float)i * (192.0f / 16777216.0f);
  const float a = sigmoid_c(x);
  const float b = __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_c(-x)));
  if (__float_as_uint(a) != __float_as_uint(b) && !(a != a && b != b)) atomicAdd(bad, 1ull);
}

// 3: round_half_away_small == round_half_away and int_of_integral == (int)
//    for every float with |v| < 2^22 (both signs, exponent fields 0..148)
__global__ void k_selftest_rha(unsigned long long* bad) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;  // mantissa
  if (m >= (1u << 23)) return;
  unsigned long long nb = 0;
  for (uint32_t ex = 0; ex <= 148; ++ex)
    for (uint32_t sg = 0; sg < 2; ++sg) {
      const float v = __uint_as_float((sg << 31) | (ex << 23) | m);
      const float a = round_half_away_small(v), b = round_half_away(v);
      nb += __float_as_uint(a) != __float_as_uint(b) && !(a == 0.0f && b == 0.0f);
      nb += int_of_integral(b) != (int)b;
    }
  if (nb) atomicAdd(bad, nb);
}

// 4: rha_int_small == int_of_integral(round_half_away(v)) for every float with |v| < 2^22
__global__ void k_selftest_rha_int(unsigned long long* bad) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;  // mantissa
  if (m >= (1u << 23)) return;
  unsigned long long nb = 0;
  for (uint32_t ex = 0; ex <= 148; ++ex)
    for (uint32_t sg = 0; sg < 2; ++sg) {
      const float v = __uint_as_float((sg << 31) | (ex << 23) | m);
      nb += rha_int_small(v) != int_of_integral(round_half_away(v));
    }
  if (nb) atomicAdd(bad, nb);
}

cudaError_t launch_selftest(int which, unsigned long long* bad, int* exps, int n_exp,
                            cudaStream_t s) {
  (void)exps;
  (void)n_exp;
  if (which == 0) {
    k_selftest_rcp<<<(1 << 23) / 256, 256, 0, s>>>(bad);
  } else if (which == 1) {
    k_selftest_sigmoid<<<(1 << 24) / 256, 256, 0, s>>>(bad);
  } else if (which == 2) {
    k_selftest_sigmoid2<<<(1 << 23) / 256, 256, 0, s>>>(bad);
  } else if (which == 3) {
    k_selftest_rha<<<(1 << 23) / 256, 256, 0, s>>>(bad);
  } else {
    k_selftest_rha_int<<<(1 << 23) / 256, 256, 0, s>>>(bad);
  }
  return cudaGetLastError();
}

}  // namespace tern
