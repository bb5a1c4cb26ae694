// k_shard.cu -- output-feature sharding helper: an
// all-gather of the ranks' [M][cs] output slices lands rank-major
// ([world][M][cs]); the next BitLinear needs token-major rows [M][world*cs].
// One 16-byte vector per thread.
#include "common.cuh"

namespace tern {

__global__ void k_unshard(const uint4* __restrict__ g, int world, int M, int vcs,
                          uint4* __restrict__ full) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // index into full
  const int64_t n = (int64_t)M * world * vcs;
  if (i >= n) return;
  const int64_t m = i / ((int64_t)world * vcs);
  const int rem = (int)(i - m * world * vcs);
  const int r = rem / vcs, j = rem - r * vcs;
  full[i] = g[((int64_t)r * M + m) * vcs + j];
}

cudaError_t launch_unshard(const void* gathered, int dt, int world, int M, int cs, void* full,
                           cudaStream_t s) {
  const int es = dt == TERN_BF16 ? 2 : 4;
  const int vcs = cs * es / 16;   // cs % 16 == 0 (checked by the caller)
  const int64_t n = (int64_t)M * world * vcs;
  if (n == 0) return cudaSuccess;
  k_unshard<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(static_cast<const uint4*>(gathered), world,
                                                        M, vcs, static_cast<uint4*>(full));
  return cudaGetLastError();
}

}  // namespace tern
