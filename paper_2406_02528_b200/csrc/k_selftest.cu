// k_selftest.cu -- device self-checks of numerics shortcuts used by the kernels
// (exposed as tern_selftest for the GPU test suite).
//   0: rcp_ge1(d) == __fdiv_rn(1, d) for every mantissa at several exponents
//   1: sigmoid_c(x) == 1/(1+exp_c(-x)) with IEEE division over a dense x sweep
#include "common.cuh"

namespace tern {

__global__ void k_selftest_rcp(const int* exps, int n_exp, unsigned long long* bad) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;  // mantissa
  if (m >= (1u << 23)) return;
  unsigned long long nb = 0;
  for (int i = 0; i < n_exp; ++i) {
    const float d = __uint_as_float(((uint32_t)(exps[i] + 127) << 23) | m);
    nb += __float_as_uint(rcp_ge1(d)) != __float_as_uint(__fdiv_rn(1.0f, d));
  }
  if (nb) atomicAdd(bad, nb);
}

__global__ void k_selftest_sigmoid(unsigned long long* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // 2^24 points in [-96, 96)
  const float x = -96.0f + (float)i * (192.0f / 16777216.0f);
  const float a = sigmoid_c(x);
  const float b = __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_c(-x)));
  if (__float_as_uint(a) != __float_as_uint(b) && !(a != a && b != b)) atomicAdd(bad, 1ull);
}

cudaError_t launch_selftest(int which, unsigned long long* bad, int* exps, int n_exp,
                            cudaStream_t s) {
  if (which == 0) {
    k_selftest_rcp<<<(1 << 23) / 256, 256, 0, s>>>(exps, n_exp, bad);
  } else {
    k_selftest_sigmoid<<<(1 << 24) / 256, 256, 0, s>>>(bad);
  }
  return cudaGetLastError();
}

}  // namespace tern
