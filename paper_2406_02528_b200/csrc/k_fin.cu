// k_fin.cu -- batched-decode finalize (4 < B <= 256, T = 1): one CTA per token
// row turns the split-K GEMM's int32 K-slice partials into the BitLinear's
// output (a5 dequant + the MLGRU step a6 / SwiGLU a7 / residual a8 epilogue)
// AND, because the CTA holds the whole output row, immediately applies the
// NEXT BitLinear's fused RMSNorm + absmax int8 quantization (a2) to it.  A
// decode phase is then GEMM + finalize (two launches) instead of quant + GEMM
// + epilogue, and the quantization never re-reads its input from memory.
// DESIGN.md "Kernels / batched decode".
//
// Arithmetic: the epilogue is k_splitk_epi's (slices summed in order, exact
// int32; the paired sigmoid), the quantization k_quant's (binary64 sum of
// squares, rsqrt, round half away from zero, C1-C5), applied to the output as
// stored (R1-R3 rounded), so results equal the three-kernel path bit for bit.
#include "epilogue.cuh"

namespace tern {

constexpr int kFinThreads = 512;
constexpr int kFinWarps = kFinThreads / 32;

struct FinArgs {
  const int32_t* part;   // [ks][M][n_rows]
  int ks, M, n_rows;
  const float* deq;      // this BitLinear's activation scales [M]
  const int32_t* qsum;   // and q sums [M]
  Epi e;                 // MLGRU / SWIGLU / RESID / STORE, out row stride e.ldo
  // next BitLinear's quantization of the output row (nq == nullptr: none)
  const float* ngain;
  float neps;
  double ninv_k;
  int8_t* nq;
  int nldq, nkp;
  float* ndeq;
  int32_t* nqsum;
  int nnorm;             // tern_norm_mode of the next BitLinear
  unsigned long long* trace;
};

// NP channel pairs per thread (pair p = tid + j*512 holds channels 2p, 2p+1)
template <typename TY, int NP>
__global__ void __launch_bounds__(kFinThreads, 1) k_fin(const FinArgs a) {
  __shared__ double red_d[kFinWarps];
  __shared__ float red_f[kFinWarps];
  __shared__ int red_i[kFinWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = blockIdx.x;
  const Epi& e = a.e;
  const int n = e.n_out, npair = n >> 1, nseg = e.n_seg;
  // constants before the dependency wait
  const float sc0 = __ldg(e.scales), sc1 = nseg > 1 ? __ldg(e.scales + 1) : 0.0f;
  const float sc2 = nseg > 2 ? __ldg(e.scales + 2) : 0.0f;
  trace_mark(a.trace, 0);
  pdl_wait();   // the GEMM's partials
  pdl_launch_dependents();
  trace_mark(a.trace, 1);
  const float dq = __ldg(a.deq + m);
  const int qs = __ldg(a.qsum + m);
  const float s0 = __fmul_rn(dq, sc0), s1 = __fmul_rn(dq, sc1), s2 = __fmul_rn(dq, sc2);
  const int64_t sl = (int64_t)a.M * a.n_rows;
  const int32_t* prow = a.part + (int64_t)m * a.n_rows;
  // every load first (partials of all K slices, state, residual): independent
  // requests in flight together instead of one L2 round trip per channel pair
  int2 av[NP][3];
  float2 pv[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int p = tid + j * kFinThreads;
    av[j][0] = av[j][1] = av[j][2] = make_int2(0, 0);
    pv[j] = make_float2(0.0f, 0.0f);
    if (p >= npair) continue;
    const int c = 2 * p;   // channels c, c+1 (same 64-row group: c even)
    if (e.kind == EPI_MLGRU) {
      pv[j] = __ldcg(reinterpret_cast<const float2*>(e.h + (int64_t)m * n + c));
    } else if (e.kind == EPI_RESID) {
      const TY* rp = static_cast<const TY*>(e.res) + (int64_t)m * e.ldr + c;
      pv[j] = make_float2(ld_act_cg<TY>(rp), ld_act_cg<TY>(rp + 1));
    }
  }
  for (int k = 0; k < a.ks; ++k) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int p = tid + j * kFinThreads;
      if (p >= npair) continue;
      const int c = 2 * p;
#pragma unroll
      for (int sg = 0; sg < 3; ++sg) {
        if (sg < nseg) {
          const int col = nseg == 1 ? c : packed_row(sg, c, nseg);
          const int2 v = __ldcg(reinterpret_cast<const int2*>(prow + k * sl + col));
          av[j][sg].x += v.x;
          av[j][sg].y += v.y;
        }
      }
    }
  }
  auto dqv = [&](int acc, float s, int seg, int r) {
    float o = __fmul_rn(i2f_small(acc - qs), s);
    if (e.bias) o = __fadd_rn(o, __ldg(e.bias + seg * n + r));
    return storage_round<TY>(o);
  };
  TY* out = static_cast<TY*>(e.out) + (int64_t)m * e.ldo;
  float y[2 * NP];
  double ss0 = 0.0, ss1 = 0.0;
  float ym = 0.0f;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int p = tid + j * kFinThreads;
    y[2 * j] = y[2 * j + 1] = 0.0f;
    if (p >= npair) continue;
    const int c = 2 * p;
    float o0, o1;
    if (e.kind == EPI_MLGRU) {
      const float fh0 = dqv(av[j][0].x, s0, 0, c), fh1 = dqv(av[j][0].y, s0, 0, c + 1);
      const float ch0 = dqv(av[j][1].x, s1, 1, c), ch1 = dqv(av[j][1].y, s1, 1, c + 1);
      const float gh0 = dqv(av[j][2].x, s2, 2, c), gh1 = dqv(av[j][2].y, s2, 2, c + 1);
      float sf0, sf1, sc0v, sc1v;
      sigmoid2(fh0, ch0, sf0, sc0v);
      sigmoid2(fh1, ch1, sf1, sc1v);
      const float h0 = __fadd_rn(__fmul_rn(sf0, pv[j].x),
                                 __fmul_rn(__fsub_rn(1.0f, sf0), __fmul_rn(ch0, sc0v)));
      const float h1 = __fadd_rn(__fmul_rn(sf1, pv[j].y),
                                 __fmul_rn(__fsub_rn(1.0f, sf1), __fmul_rn(ch1, sc1v)));
      if (e.gate == TERN_GATE_SIGMOID_H) {
        float q0, q1;
        sigmoid2(h0, h1, q0, q1);
        o0 = __fmul_rn(gh0, q0);
        o1 = __fmul_rn(gh1, q1);
      } else {
        o0 = __fmul_rn(gh0, h0);
        o1 = __fmul_rn(gh1, h1);
      }
      *reinterpret_cast<float2*>(e.h + (int64_t)m * n + c) = make_float2(h0, h1);
    } else if (e.kind == EPI_SWIGLU) {   // p = SiLU(g) u
      const float gv0 = dqv(av[j][0].x, s0, 0, c), gv1 = dqv(av[j][0].y, s0, 0, c + 1);
      const float uv0 = dqv(av[j][1].x, s1, 1, c), uv1 = dqv(av[j][1].y, s1, 1, c + 1);
      float q0, q1;
      sigmoid2(gv0, gv1, q0, q1);
      o0 = __fmul_rn(__fmul_rn(gv0, q0), uv0);
      o1 = __fmul_rn(__fmul_rn(gv1, q1), uv1);
    } else {   // RESID / STORE (one segment)
      o0 = dqv(av[j][0].x, s0, 0, c);
      o1 = dqv(av[j][0].y, s0, 0, c + 1);
      if (e.kind == EPI_RESID) {
        o0 = __fadd_rn(pv[j].x, o0);
        o1 = __fadd_rn(pv[j].y, o1);
      }
    }
    // the stored values (R1-R3 rounded) are the next BitLinear's input
    o0 = storage_round<TY>(o0);
    o1 = storage_round<TY>(o1);
    st_act<TY>(out + c, o0);
    st_act<TY>(out + c + 1, o1);
    y[2 * j] = o0;
    y[2 * j + 1] = o1;
    const double d0 = (double)o0, d1 = (double)o1;
    ss0 = fma(d0, d0, ss0);
    ss1 = fma(d1, d1, ss1);
    ym = fmaxf(ym, fmaxf(fabsf(o0), fabsf(o1)));
  }
  if (a.nq == nullptr) {
    trace_mark(a.trace, 2);
    return;
  }
  // ---------------- the next BitLinear's RMSNorm + absmax int8 quant of this row
  const bool cent = a.nnorm == TERN_NORM_CENTERED;
  float mu = 0.0f;   // centred norm (Alg. 1, reading C22): moments of y - mu
  if (cent) {
    double sx = 0.0;
#pragma unroll
    for (int j = 0; j < 2 * NP; ++j) sx += (double)y[j];   // zeros outside the row
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
    if (lane == 0) red_d[warp] = sx;
    __syncthreads();
    sx = red_d[0];
#pragma unroll
    for (int i = 1; i < kFinWarps; ++i) sx += red_d[i];
    mu = (float)(sx / (double)n);
    __syncthreads();   // red_d is reused below
    ss0 = ss1 = 0.0;
    ym = 0.0f;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if (tid + j * kFinThreads < npair) {
        const double d0 = (double)y[2 * j] - (double)mu, d1 = (double)y[2 * j + 1] - (double)mu;
        ss0 = fma(d0, d0, ss0);
        ss1 = fma(d1, d1, ss1);
        ym = fmaxf(ym, fmaxf(fabsf(__fsub_rn(y[2 * j], mu)), fabsf(__fsub_rn(y[2 * j + 1], mu))));
      }
    }
  }
  double ss = ss0 + ss1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    ym = fmaxf(ym, __shfl_xor_sync(0xffffffffu, ym, o));
  }
  if (lane == 0) { red_d[warp] = ss; red_f[warp] = ym; }
  __syncthreads();
  ss = red_d[0];
  ym = red_f[0];
#pragma unroll
  for (int i = 1; i < kFinWarps; ++i) { ss += red_d[i]; ym = fmaxf(ym, red_f[i]); }
  const float r = cent ? (float)(1.0 / sqrt(ss / (double)n + (double)a.neps))
                       : (float)rsqrt(fma(ss, a.ninv_k, (double)a.neps));
  float amax;
  if (a.ngain == nullptr) {
    amax = __fmul_rn(ym, r);   // rounding is monotone and r > 0
  } else {
    float am = 0.0f;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int p = tid + j * kFinThreads;
      if (p < npair) {
        const float2 g = __ldg(reinterpret_cast<const float2*>(a.ngain) + p);
        am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(__fsub_rn(y[2 * j], mu), r), g.x)));
        am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(__fsub_rn(y[2 * j + 1], mu), r), g.y)));
      }
    }
    am = warp_max_f32(am);
    __syncthreads();   // red_f of the first round has been read
    if (lane == 0) red_f[warp] = am;
    __syncthreads();
    am = red_f[0];
#pragma unroll
    for (int i = 1; i < kFinWarps; ++i) am = fmaxf(am, red_f[i]);
    amax = am;
  }
  const float sc = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
  int8_t* qr = a.nq + (int64_t)m * a.nldq;
  int qsum = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int p = tid + j * kFinThreads;
    if (p < npair) {
      float v0 = __fmul_rn(__fsub_rn(y[2 * j], mu), r), v1 = __fmul_rn(__fsub_rn(y[2 * j + 1], mu), r);
      if (a.ngain) {
        const float2 g = __ldg(reinterpret_cast<const float2*>(a.ngain) + p);
        v0 = __fmul_rn(v0, g.x);
        v1 = __fmul_rn(v1, g.y);
      }
      // |v*sc| <= 127(1+2^-23): the clamp to [-128,127] (C5) never acts
      const int q0 = int_of_integral(round_half_away_small(__fmul_rn(v0, sc)));
      const int q1 = int_of_integral(round_half_away_small(__fmul_rn(v1, sc)));
      qsum += q0 + q1;
      *reinterpret_cast<uint16_t*>(qr + 2 * p) = (uint16_t)((q0 & 0xff) | ((q1 & 0xff) << 8));
    }
  }
  for (int k = n + 2 * tid; k < a.nkp; k += 2 * kFinThreads)   // zero padding up to Kp
    *reinterpret_cast<uint16_t*>(qr + k) = 0;
  qsum = warp_sum_i32(qsum);
  __syncthreads();
  if (lane == 0) red_i[warp] = qsum;
  __syncthreads();
  if (tid == 0) {
    int t = red_i[0];
#pragma unroll
    for (int i = 1; i < kFinWarps; ++i) t += red_i[i];
    a.nqsum[m] = t;
    a.ndeq[m] = amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
  }
  trace_mark(a.trace, 2);
}

template <typename TY>
static cudaError_t fin_go(const FinArgs& a, cudaStream_t s) {
  const int np = (a.e.n_out / 2 + kFinThreads - 1) / kFinThreads;
  if (np <= 2) return launch_pdl(k_fin<TY, 2>, dim3(a.M), dim3(kFinThreads), 0, s, a);
  if (np <= 4) return launch_pdl(k_fin<TY, 4>, dim3(a.M), dim3(kFinThreads), 0, s, a);
  if (np <= 8) return launch_pdl(k_fin<TY, 8>, dim3(a.M), dim3(kFinThreads), 0, s, a);
  return cudaErrorInvalidValue;
}

bool fin_supported(int n_out) { return n_out % 2 == 0 && n_out / 2 <= 8 * kFinThreads; }

cudaError_t launch_fin(const int32_t* part, int ks, int M, int n_rows, const float* deq,
                       const int32_t* qsum, const Epi& e, int ydt, const float* ngain, float neps,
                       int8_t* nq, int nldq, float* ndeq, int32_t* nqsum, cudaStream_t s,
                       int nnorm) {
  if (M <= 0) return cudaSuccess;
  if (!fin_supported(e.n_out)) return cudaErrorInvalidValue;
  if (e.kind != EPI_MLGRU && e.kind != EPI_SWIGLU && e.kind != EPI_RESID && e.kind != EPI_STORE)
    return cudaErrorInvalidValue;
  FinArgs a{};
  a.part = part;
  a.ks = ks;
  a.M = M;
  a.n_rows = n_rows;
  a.deq = deq;
  a.qsum = qsum;
  a.e = e;
  a.ngain = ngain;
  a.neps = neps;
  a.ninv_k = 1.0 / (double)e.n_out;
  a.nq = nq;
  a.nldq = nldq;
  a.nkp = (e.n_out + kKAlign - 1) / kKAlign * kKAlign;
  a.ndeq = ndeq;
  a.nqsum = nqsum;
  a.nnorm = nnorm;
  a.trace = trace_slot(TERN_K_FIN, M);
  return ydt == TERN_BF16 ? fin_go<__nv_bfloat16>(a, s) : fin_go<float>(a, s);
}

}  // namespace tern
