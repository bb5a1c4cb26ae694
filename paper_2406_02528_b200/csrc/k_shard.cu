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


// ----------------------------------------------------------------------------
// the sharded BitLinear input gathered as int8 codes.
// Rank r holds the slice x_r = x[:, r*cs : (r+1)*cs] of every row.  The row's
// norm needs whole-row moments, so each rank contributes binary64 partials
// ("rounds", each one small all-gather), every rank combines the world's
// partials in rank order (so all ranks hold identical mu, r, amax), quantizes
// its own slice, and only the int8 codes (+ an int32 partial q-sum per row)
// are all-gathered -- 2x (bf16) / 4x (fp32) fewer bytes than the activations.
//   RMSNorm (C1):  round 0: (sum x^2, max|x|)      [+ round 1: max|(x r) w| with a gain]
//   centred (C22): round 0: (sum x, -)  round 1: (sum (x-mu)^2, max|x-mu|)  [+ round 2 gain]
// Row scalars from the rounds gathered so far; st_k = [world][M][2] doubles.
struct SliceNorm {
  const void* x;      // slice [M][ldx]
  int ldx, M, cs, K, dt, rank, world, cent;
  const float* gain;  // full-row gain [K] or null
  float eps;
  const double* st0;  // gathered rounds (null when not yet available)
  const double* st1;
  const double* st2;
};

template <typename TX>
__device__ __forceinline__ float ld_x(const void* p, int64_t i) {
  return ld_act<TX>(static_cast<const TX*>(p) + i);
}

// combine the world's partials of row m in rank order
__device__ __forceinline__ double comb_sum(const double* st, int world, int M, int m, int j) {
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += st[((int64_t)r * M + m) * 2 + j];
  return s;
}
__device__ __forceinline__ double comb_max(const double* st, int world, int M, int m, int j) {
  double v = 0.0;
  for (int r = 0; r < world; ++r) v = fmax(v, st[((int64_t)r * M + m) * 2 + j]);
  return v;
}

// row scalars (mu, r, amax) once the rounds they need are gathered
struct RowScal {
  float mu, r, amax;
};
__device__ __forceinline__ RowScal row_scalars(const SliceNorm& a, int m, int upto) {
  RowScal o{0.0f, 0.0f, 0.0f};
  const int base = a.cent ? 1 : 0;   // round holding (sum sq, max)
  if (a.cent) {
    if (upto < 1) return o;
    o.mu = (float)(comb_sum(a.st0, a.world, a.M, m, 0) / (double)a.K);
  }
  if (upto <= base) return o;
  const double* sq = a.cent ? a.st1 : a.st0;
  const double ss = comb_sum(sq, a.world, a.M, m, 0);
  o.r = a.cent ? (float)(1.0 / sqrt(ss / (double)a.K + (double)a.eps))
               : (float)rsqrt(fma(ss, 1.0 / (double)a.K, (double)a.eps));
  if (a.gain == nullptr) {
    o.amax = __fmul_rn((float)comb_max(sq, a.world, a.M, m, 1), o.r);
  } else if (upto > base + 1) {
    o.amax = (float)comb_max(a.cent ? a.st2 : a.st1, a.world, a.M, m, 1);
  }
  return o;
}

// partials of round `rnd` for this rank's slice: one warp per row
template <typename TX>
__global__ void k_slice_stats(const SliceNorm a, int rnd, double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.M) return;
  const int m = warp;
  const RowScal rs = row_scalars(a, m, rnd);
  const int base = a.cent ? 1 : 0;
  double s = 0.0;
  float mx = 0.0f;
  for (int j = lane; j < a.cs; j += 32) {
    const float x = ld_x<TX>(a.x, (int64_t)m * a.ldx + j);
    const float d = a.cent ? __fsub_rn(x, rs.mu) : x;
    if (a.cent && rnd == 0) {
      s += (double)x;
    } else if (rnd == base) {
      const double dd = a.cent ? (double)x - (double)rs.mu : (double)x;
      s = fma(dd, dd, s);
      mx = fmaxf(mx, fabsf(d));
    } else {   // gain round: max |((x - mu) r) w|
      mx = fmaxf(mx, fabsf(__fmul_rn(__fmul_rn(d, rs.r), __ldg(a.gain + a.rank * a.cs + j))));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    out[(int64_t)m * 2 + 0] = s;
    out[(int64_t)m * 2 + 1] = (double)mx;
  }
}

// quantize this rank's slice with the combined row scalars: codes [M][cs] then
// the row q-sum partials [M] (int32) behind them (one send buffer); deq [M]
template <typename TX>
// codes to q [M][ldq] (zero padded from cs to ldq), q-sum partials to qs_out [M]
__global__ void k_slice_quant(const SliceNorm a, int rounds, int8_t* __restrict__ q, int ldq,
                              int32_t* __restrict__ qs_out, float* __restrict__ deq) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.M) return;
  const int m = warp;
  const RowScal rs = row_scalars(a, m, rounds);
  const float sc = rs.amax > 0.0f ? __fdiv_rn(127.0f, rs.amax) : 0.0f;
  int qs = 0;
  for (int j = lane; j < a.cs; j += 32) {
    int qi = 0;
    if (rs.amax > 0.0f) {
      const float x = ld_x<TX>(a.x, (int64_t)m * a.ldx + j);
      float y = __fmul_rn(a.cent ? __fsub_rn(x, rs.mu) : x, rs.r);
      if (a.gain) y = __fmul_rn(y, __ldg(a.gain + a.rank * a.cs + j));
      qi = int_of_integral(round_half_away_small(__fmul_rn(y, sc)));   // |y sc| <= 127 (C5)
    }
    q[(int64_t)m * ldq + j] = (int8_t)qi;
    qs += qi;
  }
  for (int j = a.cs + lane; j < ldq; j += 32) q[(int64_t)m * ldq + j] = 0;
  qs = warp_sum_i32(qs);
  if (lane == 0) {
    qs_out[m] = qs;
    deq[m] = rs.amax > 0.0f ? __fdiv_rn(rs.amax, 127.0f) : 0.0f;   // identical on every rank
  }
}

// gathered [world][M*cs codes | M q-sums] -> token-major codes [M][ldq] (zero
// padded to ldq) and q-sums [M]
__global__ void k_unshard_q(const int8_t* __restrict__ g, int world, int M, int cs, int8_t* q,
                            int ldq, int32_t* __restrict__ qsum) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // element of q
  const int64_t n = (int64_t)M * ldq;
  const int64_t per = (int64_t)M * cs + 4 * (int64_t)M;   // bytes per rank
  if (i < n) {
    const int m = (int)(i / ldq), k = (int)(i % ldq);
    int8_t v = 0;
    if (k < world * cs) {
      const int r = k / cs, j = k - r * cs;
      v = g[r * per + (int64_t)m * cs + j];
    }
    q[i] = v;
  }
  if (i < M) {
    int s = 0;
    for (int r = 0; r < world; ++r)
      s += reinterpret_cast<const int32_t*>(g + r * per + (int64_t)M * cs)[i];
    qsum[i] = s;
  }
}

static SliceNorm slice_norm(const void* x, int ldx, int M, int cs, int world, int rank, int dt,
                            const float* gain, float eps, int norm) {
  SliceNorm a{};
  a.x = x;
  a.ldx = ldx;
  a.M = M;
  a.cs = cs;
  a.K = cs * world;
  a.dt = dt;
  a.rank = rank;
  a.world = world;
  a.cent = norm == TERN_NORM_CENTERED;
  a.gain = gain;
  a.eps = eps;
  return a;
}

int slice_rounds(int norm, bool gain) { return (norm == TERN_NORM_CENTERED ? 2 : 1) + (gain ? 1 : 0); }

cudaError_t launch_slice_stats(const void* x, int ldx, int M, int cs, int world, int rank, int dt,
                               const float* gain, float eps, int norm, const double* const* st,
                               int rnd, double* out, cudaStream_t s) {
  SliceNorm a = slice_norm(x, ldx, M, cs, world, rank, dt, gain, eps, norm);
  a.st0 = st[0];
  a.st1 = st[1];
  a.st2 = st[2];
  const unsigned grid = (unsigned)((M * 32 + 255) / 256);
  if (dt == TERN_BF16) k_slice_stats<__nv_bfloat16><<<grid, 256, 0, s>>>(a, rnd, out);
  else k_slice_stats<float><<<grid, 256, 0, s>>>(a, rnd, out);
  return cudaGetLastError();
}

cudaError_t launch_slice_quant(const void* x, int ldx, int M, int cs, int world, int rank, int dt,
                               const float* gain, float eps, int norm, const double* const* st,
                               int8_t* q, int ldq, int32_t* qs_out, float* deq, cudaStream_t s) {
  SliceNorm a = slice_norm(x, ldx, M, cs, world, rank, dt, gain, eps, norm);
  a.st0 = st[0];
  a.st1 = st[1];
  a.st2 = st[2];
  const int rounds = slice_rounds(norm, gain != nullptr);
  const unsigned grid = (unsigned)((M * 32 + 255) / 256);
  if (dt == TERN_BF16) k_slice_quant<__nv_bfloat16><<<grid, 256, 0, s>>>(a, rounds, q, ldq, qs_out, deq);
  else k_slice_quant<float><<<grid, 256, 0, s>>>(a, rounds, q, ldq, qs_out, deq);
  return cudaGetLastError();
}

cudaError_t launch_unshard_q(const int8_t* gathered, int world, int M, int cs, int8_t* q, int ldq,
                             int32_t* qsum, cudaStream_t s) {
  const int64_t n = (int64_t)M * ldq;
  const int64_t nt = n > M ? n : M;
  k_unshard_q<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(gathered, world, M, cs, q, ldq, qsum);
  return cudaGetLastError();
}

}  // namespace tern
