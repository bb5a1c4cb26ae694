// k_gemv.cu -- a3: decode-time ternary GEMV (M <= 8 tokens) with the fused
// RMSNorm+quant prologue (a2) and the block's epilogues (a5-a8), DESIGN.md
// "Kernels / decode GEMV".
//
// A decode step is a chain of 4 dependent BitLinears per block, so
// each launch is latency-bound at batch 1 and HBM-bound on the packed weights
// at large models; the kernel is organised around its critical path:
//  * before griddepcontrol.wait (PDL) every thread loads its share of the
//    CTA's packed weights into REGISTERS (16-byte non-temporal loads), so the
//    weight fetch overlaps the previous kernel (weights do not depend on it);
//  * right after the wait: the input row(s) and, for the epilogue, the state
//    h / residual are loaded at once; the row's RMSNorm + absmax int8 quant is
//    recomputed per CTA (no extra launch or grid sync) with two block barriers;
//    sum(x^2) in double-float (common.cuh, reading C4), one thread finishes it
//    in binary64;
//  * dot: lanes split K in 64-trit chunks, warps split rows; each 2-bit field
//    e = t+1 is isolated with one AND and fed to dp4a (u8 x s8):
//        sum_k e_k q_k = acc + sum_k q_k  ->  acc = (sum) - qsum
//    (field f carries e*4^f; the exact sum is shifted back);
//  * epilogue per (token, channel): dequantization (a5), then the MLGRU step
//    with the state update (a6), SwiGLU (a7) or the residual add (a8).
// CTA = `ch` logical channels of every segment of the group, so f, c and g
// (or gate and up) of the same channels meet in one CTA.
#include <cstdio>
#include <cstdlib>

#include "epilogue.cuh"

namespace tern {

constexpr int kGThreads = 512;
// Per-dot-lane q sums folded into the quant step (fp32 rows) or recomputed by
// every warp from the q row (bf16 rows): measured c2 (fp32) decode 2391 -> 2451
// tok/s with the fold, c4 (bf16) 1005 -> 888 -- kept per activation type.
template <typename TX> struct LqFold { static constexpr bool on = sizeof(TX) == 4; };
constexpr int kGWarps = kGThreads / 32;
// 16-byte activation vectors per thread per row (register tile of the prologue)
// (2 vectors cover every config row: fp32 K <= 4096, bf16 K <= 8192; a deeper
// tile only adds predicated-off registers -- 4 made the bf16 kernel spill)
template <int MM> struct GNVX { static constexpr int v = 2; };

struct GemvArgs {
  const void* x;
  int ldx, K, Kp, M;
  const float* gain;
  float eps;
  const uint32_t* codes;
  int n_rows, n_out, n_seg, ch;
  int sw_stride;  // words between consecutive K-blocks of a segment in smem
  double inv_k;  // 1/K (binary64)
  int norm;      // tern_norm_mode of the input row
  int ld_at;     // debug knob TERN_GEMV_LD_AT: where launch_dependents fires (0: after the
                 // wait, 1: after the quant, 2: at the end)
  int strip;     // debug knob TERN_GEMV_STRIP (timing experiments only, wrong results):
                 // 1 skip the dot, 2 skip the epilogue math, 4 skip the quant
  Epi epi;
  QuantTaps taps;
  const uint8_t* pf;         // L2 prefetch hint: a later launch's packed weights
  size_t pf_bytes;
  unsigned long long* prof;  // debug (TERN_GEMV_PROF): [grid][8] clock64 per phase
  unsigned long long* trace; // tern_trace_enable: [grid][8] globaltimer (start, released, end, smid, phases)
};

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint4 ldg_stream16(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 16 bytes of activations -> floats
template <typename TX> struct XVec;
template <> struct XVec<float> {
  static constexpr int N = 4;
  __device__ static void unpack(const uint4& u, float* v) {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
    v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
  }
};
template <> struct XVec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void unpack(const uint4& u, float* v) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

// dot of one 16-byte weight chunk (4 words = 64 trits) with 64 int8 activations
__device__ __forceinline__ int chunk_dot(const uint4& w, const int8_t* q) {
  const uint4* qv = reinterpret_cast<const uint4*>(q);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  int s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 a = qv[k];
    // field f of word k holds trits 4f..4f+3 of its 16, i.e. q bytes [4f, 4f+4)
    const int f0 = dp4a_us(ws[k] & 0x03030303u, a.x, 0);
    const int f1 = dp4a_us(ws[k] & 0x0C0C0C0Cu, a.y, 0);
    const int f2 = dp4a_us(ws[k] & 0x30303030u, a.z, 0);
    const int f3 = dp4a_us(ws[k] & 0xC0C0C0C0u, a.w, 0);
    s += f0 + (f1 >> 2) + (f2 >> 4) + (f3 >> 6);   // each term is an exact multiple
  }
  return s;
}

__device__ __forceinline__ uint32_t* sw_words(uint8_t* smem) { return reinterpret_cast<uint32_t*>(smem); }

// sum over the 32 lanes, result in every lane
__device__ __forceinline__ int warp_allsum_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- phase pieces
// (shared by the one-BitLinear kernel k_gemv and the whole-stack persistent
// kernel k_stack_decode)

// Warp 0: bulk-copy unit's packed weights into dst (completing on bar), or with
// l2_only just pull them into L2.  In the K-block-major layout the unit's rows
// of one segment within one 64-row group are one contiguous span per K-block.
// Smem: [seg][kb] blocks of ch rows x 8 words, block stride SW words (SW = 8 mod
// 32: conflict-free dot reads).  A unit without rows arrives with 0 bytes.
__device__ __forceinline__ void gemv_issue(const GemvArgs& a, int unit, uint32_t* dst,
                                           uint64_t* bar, int lane, bool l2_only) {
  const int nkb = a.Kp >> 7, SW = a.sw_stride;
  const int r0 = unit * a.ch, r1 = min(r0 + a.ch, a.n_out);   // logical rows [r0, r1)
  if (!l2_only && lane == 0)
    mbar_arrive_expect_tx(bar, r1 > r0 ? (uint32_t)(a.n_seg * nkb * (r1 - r0) * 32) : 0u);
  if (r1 <= r0) return;
  __syncwarp();
  const int g0 = r0 >> 6, g1 = (r1 - 1) >> 6;   // 64-row groups touched (<= 2)
  const int nparts = a.n_seg == 1 ? 1 : g1 - g0 + 1;
  const int nspan = a.n_seg * nkb * nparts;
  for (int sp = lane; sp < nspan; sp += 32) {
    const int part = sp % nparts, t = sp / nparts;
    const int kb = t % nkb, sg = t / nkb;
    int a0r = r0, a1r = r1;
    if (a.n_seg > 1) {
      const int gb = (g0 + part) << 6;
      a0r = max(r0, gb);
      a1r = min(r1, gb + 64);
    }
    const int pr = a.n_seg == 1 ? a0r : packed_row(sg, a0r, a.n_seg);
    const uint32_t* src = a.codes + ((int64_t)kb * a.n_rows + pr) * 8;
    const uint32_t bytes = (uint32_t)(a1r - a0r) * 32u;
    if (l2_only)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    else
      bulk_load(dst + (sg * nkb + kb) * SW + (a0r - r0) * 8, src, bytes, bar);
  }
}

// Epilogue operands: lane m of warp w owns token m of channels w, w+16, w+32,
// w+48 (state h or residual).
template <typename TY>
__device__ __forceinline__ void gemv_pre(const GemvArgs& a, int unit, int warp, int lane,
                                         float (&pre)[4]) {
  const Epi& e = a.epi;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pre[j] = 0.0f;
    const int i = warp + j * kGWarps, rr = unit * a.ch + i;
    if (lane < a.M && i < a.ch && rr < a.n_out) {
      if (e.kind == EPI_MLGRU) pre[j] = __ldcg(e.h + (int64_t)lane * e.n_out + rr);
      if (e.kind == EPI_RESID)
        pre[j] = ld_act_cg<TY>(static_cast<const TY*>(e.res) + (int64_t)lane * e.ldr + rr);
    }
  }
}

#define GPROF(i)                                                                   \
  if (a.prof && tid == 0 && (i) < 8) a.prof[blockIdx.x * 8 + (i)] = clock64() - pt0; \
  if (a.trace && tid == 0 && (i) >= 2) a.trace[blockIdx.x * 16 + 3 + (i)] = gtimer();

// From the input rows to the stored outputs: fused RMSNorm + int8 quant of the
// M rows (a2), wait for the weights (bar, parity), dot (a3) and epilogue.
// CENT: Alg. 1's centred norm (reading C22) instead of RMSNorm (compile-time,
// so the default path carries none of its code).
template <int MM, typename TX, typename TY, bool CENT>
__device__ __forceinline__ void gemv_run(const GemvArgs& a, int unit, const uint32_t* swd,
                                         int8_t* qs, uint64_t* wbar, uint32_t parity,
                                         const float (&msc)[3], const float (&pre)[4],
                                         double (*red_d)[kGWarps], float (*red_m)[kGWarps],
                                         int (*lq_s)[kGWarps][32], long long pt0) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Epi& e = a.epi;
  const int nkb = a.Kp >> 7;
  const int SW = a.sw_stride;
  // per-lane sums of the q bytes each dot lane will visit (filled by the quant
  // step below; every block barrier before the first use orders the zeroing)
  if (LqFold<TX>::on) {
#pragma unroll
    for (int m = 0; m < MM; ++m) lq_s[m][warp][lane] = 0;
  }
  // ---------------- prologue: fused RMSNorm + int8 quant (a2) of the M rows.
  // x in registers (kGNVX 16-byte vectors per thread per row); sum(x^2) in
  // binary64 (C4), max|x|; one block barrier for the partials, every warp then
  // finishes the reduction itself.
  constexpr int VE = XVec<TX>::N;
  const int nvec = a.K / VE, nvecp = a.Kp / VE;
  constexpr int kGNVX = GNVX<MM>::v;
  uint4 xv[MM][kGNVX];
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    const uint4* src =
        reinterpret_cast<const uint4*>(static_cast<const TX*>(a.x) + (int64_t)m * a.ldx);
#pragma unroll
    for (int i = 0; i < kGNVX; ++i) {
      const int v = tid + i * kGThreads;
      xv[m][i] = (m < a.M && v < nvec) ? __ldcg(src + v) : make_uint4(0, 0, 0, 0);
    }
  }
  // centred norm (Alg. 1, reading C22): the row mean first, then the moments
  // are taken of x - mu (exact in binary64); mu = 0 leaves the RMSNorm path
  float mu[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) mu[m] = 0.0f;
  constexpr bool cent = CENT;
  if (cent) {
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      double sx = 0.0;
#pragma unroll
      for (int i = 0; i < kGNVX; ++i) {
        float v[VE];
        XVec<TX>::unpack(xv[m][i], v);   // zeros outside the row
#pragma unroll
        for (int j = 0; j < VE; ++j) sx += (double)v[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
      if (lane == 0) red_d[m][warp] = sx;
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      double sx = lane < kGWarps ? red_d[m][lane] : 0.0;
#pragma unroll
      for (int o = kGWarps / 2; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
      mu[m] = (float)(__shfl_sync(0xffffffffu, sx, 0) / (double)a.K);
    }
    __syncthreads();   // red_d is reused below
  }
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    double s0 = 0.0, s1 = 0.0;
    float xmax = 0.0f;
#pragma unroll
    for (int i = 0; i < kGNVX; ++i) {
      float v[VE];
      XVec<TX>::unpack(xv[m][i], v);
      if (cent) {
        const bool in = tid + i * kGThreads < nvec;   // padding takes no part in the moments
#pragma unroll
        for (int j = 0; j < VE; j += 2) {
          const double d0 = in ? (double)v[j] - (double)mu[m] : 0.0;
          const double d1 = in ? (double)v[j + 1] - (double)mu[m] : 0.0;
          s0 = fma(d0, d0, s0);
          s1 = fma(d1, d1, s1);
          if (in)
            xmax = fmaxf(xmax, fmaxf(fabsf(__fsub_rn(v[j], mu[m])), fabsf(__fsub_rn(v[j + 1], mu[m]))));
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < VE; j += 2) {
        const double d0 = (double)v[j], d1 = (double)v[j + 1];
        s0 = fma(d0, d0, s0);
        s1 = fma(d1, d1, s1);
        xmax = fmaxf(xmax, fmaxf(fabsf(v[j]), fabsf(v[j + 1])));
      }
    }
    double sd = s0 + s1;
    if (m == 0) { GPROF(2) }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sd += __shfl_xor_sync(0xffffffffu, sd, o);
      xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    }
    if (m == 0) { GPROF(3) }
    if (lane == 0) { red_d[m][warp] = sd; red_m[m][warp] = xmax; }
  }
  __syncthreads();
  GPROF(4)
  float rinv[MM], amax[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    // every warp: lanes 0..15 take one partial each, tree over 16
    double sd = lane < kGWarps ? red_d[m][lane] : 0.0;
    float xm = lane < kGWarps ? red_m[m][lane] : 0.0f;
#pragma unroll
    for (int o = kGWarps / 2; o > 0; o >>= 1) {
      sd += __shfl_xor_sync(0xffffffffu, sd, o);
      xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
    }
    sd = __shfl_sync(0xffffffffu, sd, 0);
    xm = __shfl_sync(0xffffffffu, xm, 0);
    rinv[m] = cent ? (float)(1.0 / sqrt(sd / (double)a.K + (double)a.eps))
                   : (float)rsqrt(fma(sd, a.inv_k, (double)a.eps));
    // max|fl(x r)| = fl(max|x| r): rounding is monotone and r > 0
    amax[m] = __fmul_rn(xm, rinv[m]);
  }
  if (a.gain) {   // with a gain the max is taken over y = (x r) g: one more round
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      float am = 0.0f;
#pragma unroll
      for (int i = 0; i < kGNVX; ++i) {
        const int v = tid + i * kGThreads;
        float xf[VE];
        XVec<TX>::unpack(xv[m][i], xf);
#pragma unroll
        for (int j = 0; j < VE; ++j)
          if (v < nvec)
            am = fmaxf(am, fabsf(__fmul_rn(__fmul_rn(CENT ? __fsub_rn(xf[j], mu[m]) : xf[j], rinv[m]),
                                           __ldg(a.gain + v * VE + j))));
      }
      am = warp_max_f32(am);
      __syncthreads();   // everyone has read red_m above
      if (lane == 0) red_m[m][warp] = am;
      __syncthreads();
      am = lane < kGWarps ? red_m[m][lane] : 0.0f;
      am = warp_max_f32(am);
      amax[m] = am;
    }
  }
  GPROF(5)
  // quantize own elements: q = round(y * 127/amax), half away from zero (C3, C5)
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    const float sc = amax[m] > 0.0f ? __fdiv_rn(127.0f, amax[m]) : 0.0f;
    int8_t* qrow = qs + m * a.Kp;
    int tq = 0;   // this thread's q bytes, all in the 16-byte word range of one dot lane
#pragma unroll
    for (int i = 0; i < kGNVX; ++i) {
      const int v = tid + i * kGThreads;
      if (v < nvecp) {
        uint32_t pk[VE / 4];
#pragma unroll
        for (int j4 = 0; j4 < VE / 4; ++j4) pk[j4] = 0;
        if (v < nvec && amax[m] > 0.0f) {
          float xf[VE];
          XVec<TX>::unpack(xv[m][i], xf);
#pragma unroll
          for (int j = 0; j < VE; ++j) {
            float y = __fmul_rn(CENT ? __fsub_rn(xf[j], mu[m]) : xf[j], rinv[m]);
            if (a.gain) y = __fmul_rn(y, __ldg(a.gain + v * VE + j));
            // |y*sc| <= 127(1+2^-23), so the clamp to [-128,127] (C5) never acts
            const int qi = int_of_integral(round_half_away_small(__fmul_rn(y, sc)));
            tq += qi;
            pk[j >> 2] |= ((uint32_t)qi & 0xffu) << (8 * (j & 3));
          }
        }
        if (VE == 4)
          *reinterpret_cast<uint32_t*>(qrow + v * 4) = pk[0];
        else
          *reinterpret_cast<uint2*>(qrow + v * 8) = make_uint2(pk[0], pk[VE / 4 - 1]);
      }
    }
    // vector v holds q bytes [v*VE, v*VE+VE) of word v*VE/16, read by dot lane
    // (v*VE/16) % 32 -- the same lane for all of this thread's vectors; the
    // 16/VE threads sharing a lane within the warp are adjacent
    constexpr int G = 16 / VE;   // threads per dot lane in a warp (4 fp32, 2 bf16)
    if (LqFold<TX>::on) {
#pragma unroll
      for (int o = 1; o < G; o <<= 1) tq += __shfl_xor_sync(0xffffffffu, tq, o);
      if ((lane & (G - 1)) == 0) lq_s[m][warp][(tid / G) & 31] = tq;   // one writer per entry
    }
  }
  float deq[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) deq[m] = amax[m] > 0.0f ? __fdiv_rn(amax[m], 127.0f) : 0.0f;
  if (unit == 0 && tid < a.M) {
#pragma unroll
    for (int m = 0; m < MM; ++m)
      if (m == tid) {
        if (a.taps.deq) a.taps.deq[m] = deq[m];
        if (a.taps.inv_rms) a.taps.inv_rms[m] = rinv[m];
        if (a.taps.absmax) a.taps.absmax[m] = amax[m];
      }
  }
  __syncthreads();            // q rows visible
  if (a.ld_at == 1) pdl_launch_dependents();
  mbar_wait(wbar, parity);    // weights landed (long since, in a PDL chain)
  GPROF(6)
  if (unit == 0 && a.taps.q) {
    for (int m = 0; m < a.M; ++m)
      for (int k = tid * 16; k < a.Kp; k += kGThreads * 16)
        *reinterpret_cast<uint4*>(a.taps.q + (int64_t)m * a.taps.ldq + k) =
            *reinterpret_cast<const uint4*>(qs + m * a.Kp + k);
  }

  // ---------------- dot + epilogue: warp w owns channels w, w+16, ... with all
  // their segments (f,c,g / gate,up); lanes split the row's 32-bit words
  // (16 trits x 16 q bytes; consecutive lanes -> consecutive words, no bank
  // conflicts).  sum e*q - sum q = sum t*q: each lane starts from minus
  // the sum of the q bytes it will visit, so no per-row q sum is needed.
  const int W = a.Kp >> 4;   // words per row
  int lq[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) lq[m] = 0;
  if (LqFold<TX>::on) {
#pragma unroll
    for (int m = 0; m < MM; ++m)
#pragma unroll
      for (int w = 0; w < kGWarps; ++w) lq[m] += lq_s[m][w][lane];
  } else {
    for (int w = lane; w < W; w += 32) {
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const uint4 qv = *reinterpret_cast<const uint4*>(qs + m * a.Kp + w * 16);
        lq[m] = dp4a_us(0x01010101u, qv.x, lq[m]);
        lq[m] = dp4a_us(0x01010101u, qv.y, lq[m]);
        lq[m] = dp4a_us(0x01010101u, qv.z, lq[m]);
        lq[m] = dp4a_us(0x01010101u, qv.w, lq[m]);
      }
    }
  }
  TY* out = static_cast<TY*>(e.out);
  // MM == 1 and a warp owning >= 2 channels: channels j and j+1 share the q
  // loads and their dot chains interleave (the c3/c4 gate|up phases have up to
  // 3 channels per warp); results parked in accn[] for the second channel
  int accn[3] = {0, 0, 0};
  bool have_next = false;
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int i = warp + j * kGWarps;
    if (i >= a.ch) break;
    const int rr = unit * a.ch + i;
    int acc[3] = {0, 0, 0};
    if (have_next) {
#pragma unroll
      for (int sgi = 0; sgi < 3; ++sgi) acc[sgi] = accn[sgi];
      have_next = false;
    } else {
      const int i2 = i + kGWarps;
      const bool two = MM == 1 && j < 3 && i2 < a.ch;
      int part[3][MM], part2[3];
#pragma unroll
      for (int sgi = 0; sgi < 3; ++sgi) {
        part2[sgi] = -lq[0];
#pragma unroll
        for (int m = 0; m < MM; ++m) part[sgi][m] = -lq[m];
      }
      for (int w = lane; w < W; w += 32) {
        uint4 qv[MM];
#pragma unroll
        for (int m = 0; m < MM; ++m) qv[m] = *reinterpret_cast<const uint4*>(qs + m * a.Kp + w * 16);
#pragma unroll
        for (int sgi = 0; sgi < 3; ++sgi) {
          if (sgi < a.n_seg) {
            const uint32_t* wrow = swd + (sgi * nkb + (w >> 3)) * SW + (w & 7);
            const uint32_t wd = wrow[i * 8];
#pragma unroll
            for (int m = 0; m < MM; ++m) {
              const int f0 = dp4a_us(wd & 0x03030303u, qv[m].x, 0);
              const int f1 = dp4a_us(wd & 0x0C0C0C0Cu, qv[m].y, 0);
              const int f2 = dp4a_us(wd & 0x30303030u, qv[m].z, 0);
              const int f3 = dp4a_us(wd & 0xC0C0C0C0u, qv[m].w, 0);
              part[sgi][m] += f0 + (f1 >> 2) + (f2 >> 4) + (f3 >> 6);   // exact multiples
            }
            if (two) {
              const uint32_t wd2 = wrow[i2 * 8];
              const int f0 = dp4a_us(wd2 & 0x03030303u, qv[0].x, 0);
              const int f1 = dp4a_us(wd2 & 0x0C0C0C0Cu, qv[0].y, 0);
              const int f2 = dp4a_us(wd2 & 0x30303030u, qv[0].z, 0);
              const int f3 = dp4a_us(wd2 & 0xC0C0C0C0u, qv[0].w, 0);
              part2[sgi] += f0 + (f1 >> 2) + (f2 >> 4) + (f3 >> 6);
            }
          }
        }
      }
      // all-reduce, then lane m keeps token m's accumulators
#pragma unroll
      for (int sgi = 0; sgi < 3; ++sgi) {
        if (sgi < a.n_seg) {
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            const int v = warp_allsum_i32(part[sgi][m]);
            if (lane == m) acc[sgi] = v;
          }
          if (two) {
            const int v = warp_allsum_i32(part2[sgi]);
            if (lane == 0) accn[sgi] = v;
          }
        }
      }
      have_next = two;
    }
    if (j == 0) { GPROF(7) }
    if (rr >= a.n_out || lane >= a.M) continue;
    const int m = lane;
    float dq = deq[0];
#pragma unroll
    for (int mm = 1; mm < MM; ++mm)
      if (m == mm) dq = deq[mm];
    const float pv = j == 0 ? pre[0] : (j == 1 ? pre[1] : (j == 2 ? pre[2] : pre[3]));
    if (e.acc) {
      for (int sg = 0; sg < a.n_seg; ++sg)
        e.acc[(int64_t)m * e.ldacc + (a.n_seg == 1 ? rr : packed_row(sg, rr, a.n_seg))] =
            sg == 0 ? acc[0] : (sg == 1 ? acc[1] : acc[2]);
    }
    if (e.kind == EPI_MLGRU) {
      const float fh = bl_val<TY>(e, acc[0], dq, msc[0], 0, rr);
      const float chh = bl_val<TY>(e, acc[1], dq, msc[1], 1, rr);
      const float gh = bl_val<TY>(e, acc[2], dq, msc[2], 2, rr);
      const float f = sigmoid_c(fh);
      const float cc = silu_c(chh);
      const float h = mlgru_step(f, pv, cc);
      e.h[(int64_t)m * e.n_out + rr] = h;
      st_act<TY>(out + (int64_t)m * e.ldo + rr, mlgru_out(gh, h, e.gate));
    } else if (e.kind == EPI_SWIGLU) {
      const float gh = bl_val<TY>(e, acc[0], dq, msc[0], 0, rr);
      const float uh = bl_val<TY>(e, acc[1], dq, msc[1], 1, rr);
      st_act<TY>(out + (int64_t)m * e.ldo + rr, swiglu(gh, uh));
    } else if (e.kind == EPI_RESID) {
      const float o = bl_val<TY>(e, acc[0], dq, msc[0], 0, rr);
      st_act<TY>(out + (int64_t)m * e.ldo + rr, __fadd_rn(pv, o));
    } else if (e.kind == EPI_STORE || e.kind == EPI_FCG) {
      for (int sg = 0; sg < a.n_seg; ++sg) {
        const float o = bl_val<TY>(e, sg == 0 ? acc[0] : (sg == 1 ? acc[1] : acc[2]), dq,
                                   sg == 0 ? msc[0] : (sg == 1 ? msc[1] : msc[2]), sg, rr);
        const int col = e.kind == EPI_FCG ? packed_row(sg, rr, a.n_seg) : rr;
        st_act<TY>(out + (int64_t)m * e.ldo + col, o);
      }
    }
  }
  GPROF(9)
}

// ---------------------------------------------------------------- lean batch-1 kernel
// The batch-1 decode phase (c2 / c4 B = 1, the paper's generate workload P:241): one token,
// RMSNorm without a gain, no taps.  The arithmetic is gemv_run's bit for bit (binary64
// sum of squares rounded once to r, C4; round half away, C3; Σ e q − Σ q).  A
// phase is a few microseconds of latency-bound work on every SM, and with 16 warps per CTA
// the SM sub-partitions' issue slots are the binding resource, so the kernel spends as few
// warp-instructions as it can after the dependency wait (measured):
//   * only the warps that hold part of the x row take part in the norm and the quant;
//   * warp reductions of the max and of the integer sums are single REDUX instructions
//     (max |x| compares float bits: order-preserving for non-negative floats);
//   * the dot keeps one accumulator per 2-bit field (sum_f dp4a(w & mask_f, q_f)): the
//     field scales 4^f are divided out once per lane and channel instead of once per word (exact:
//     every term of field f is a multiple of 4^f) -- 2 instructions per 4 trits;
//   * the epilogue runs lane-parallel: lane j finishes the warp's j-th channel;
//   * compact code (no per-M unrolling, no gain / centred / tap / profiling paths).
template <typename TX, typename TY>
__global__ void __launch_bounds__(kGThreads) k_gemv1(const GemvArgs a) {
  extern __shared__ __align__(128) uint8_t g_smem[];
  int8_t* qs = reinterpret_cast<int8_t*>(g_smem + (size_t)a.n_seg * (a.Kp >> 7) * a.sw_stride * 4);
  __shared__ double red_d[kGWarps];
  __shared__ unsigned red_m[kGWarps];
  __shared__ int red_q[kGWarps];
  __shared__ float sh_amax;
  __shared__ __align__(8) uint64_t wbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = blockIdx.x;
  if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 0] = gtimer();
  if (warp == 0) {   // this CTA's packed weights -> smem (bulk copies; independent of the chain)
    if (lane == 0) {
      mbar_init(&wbar, 1);
      fence_barrier_init();
    }
    __syncwarp();
    gemv_issue(a, unit, sw_words(g_smem), &wbar, lane, false);
  }
  if (a.pf && tid == 32) {   // L2 prefetch of this CTA's share of a later launch's weights
    const size_t chunk = ((a.pf_bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
    const size_t off = chunk * blockIdx.x;
    if (off < a.pf_bytes) {
      const size_t n = a.pf_bytes - off < chunk ? a.pf_bytes - off : chunk;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf + off), "r"((uint32_t)n)
                   : "memory");
    }
  }
  const Epi& e = a.epi;
  // epilogue operands of this warp's channels: lane j <-> channel warp + 16 j (j < 4)
  const int ich = warp + lane * kGWarps, rch = unit * a.ch + ich;
  const bool own = lane < 4 && ich < a.ch && rch < a.n_out;
  float msc[3];
#pragma unroll
  for (int sg = 0; sg < 3; ++sg) msc[sg] = sg < a.n_seg ? __ldg(e.scales + sg) : 0.0f;
  pdl_wait();
  if (a.ld_at == 0) pdl_launch_dependents();
  if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 1] = gtimer();
  float pre = 0.0f;
  // (trace marks, tid 0: 9 x loaded, 10 norm done, 5 q row ready, 6 first dot loop,
  //  7 its sums, 8 all dots, 2 epilogue done)
  if (own && e.kind == EPI_MLGRU) pre = __ldcg(e.h + rch);
  if (own && e.kind == EPI_RESID) pre = ld_act_cg<TY>(static_cast<const TY*>(e.res) + rch);
  // ---- x -> registers, binary64 sum of squares and max |x| (a2, C4): warps holding data
  constexpr int VE = XVec<TX>::N;
  const int nvec = a.K / VE, nvecp = a.Kp / VE;
  const int nwx = (nvecp + 31) >> 5 < kGWarps ? (nvecp + 31) >> 5 : kGWarps;   // data warps
  const bool xw = warp < nwx;
  uint4 xv[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  if (xw) {
    const uint4* src = static_cast<const uint4*>(a.x);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int v = tid + i * kGThreads;
      if (v < nvec) xv[i] = __ldcg(src + v);
    }
    double s0 = 0.0, s1 = 0.0;
    float xm = 0.0f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      float v[VE];
      XVec<TX>::unpack(xv[i], v);
#pragma unroll
      for (int j = 0; j < VE; j += 2) {
        s0 = fma((double)v[j], (double)v[j], s0);
        s1 = fma((double)v[j + 1], (double)v[j + 1], s1);
        xm = fmaxf(xm, fmaxf(fabsf(v[j]), fabsf(v[j + 1])));
      }
    }
    double sd = s0 + s1;
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 9] = gtimer();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
    const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(xm));
    if (lane == 0) {
      red_d[warp] = sd;
      red_m[warp] = mb;
    }
  }
  __syncthreads();
  int tq = 0;
  if (xw) {
    double sd = lane < nwx ? red_d[lane] : 0.0;
#pragma unroll
    for (int o = kGWarps / 2; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
    sd = __shfl_sync(0xffffffffu, sd, 0);
    const unsigned mb = __reduce_max_sync(0xffffffffu, lane < nwx ? red_m[lane] : 0u);
    const float rinv = (float)rsqrt(fma(sd, a.inv_k, (double)a.eps));
    // max|fl(x r)| = fl(max|x| r): rounding is monotone and r > 0
    const float amax = __fmul_rn(__uint_as_float(mb), rinv);
    if (tid == 0) sh_amax = amax;
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 10] = gtimer();
    // quantize own elements: q = round(x r * 127/amax), half away from zero (C3, C5)
    const float sc = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int v = tid + i * kGThreads;
      if (v < nvecp && !(a.strip & 4)) {
        uint32_t pk[VE / 4];
#pragma unroll
        for (int j4 = 0; j4 < VE / 4; ++j4) pk[j4] = 0;
        if (v < nvec && amax > 0.0f) {
          float xf[VE];
          XVec<TX>::unpack(xv[i], xf);
#pragma unroll
          for (int j = 0; j < VE; ++j) {
            // |y*sc| <= 127(1+2^-23), so the clamp to [-128,127] (C5) never acts
            const int qi =
                int_of_integral(round_half_away_small(__fmul_rn(__fmul_rn(xf[j], rinv), sc)));
            tq += qi;
            pk[j >> 2] |= ((uint32_t)qi & 0xffu) << (8 * (j & 3));
          }
        }
        if (VE == 4)
          *reinterpret_cast<uint32_t*>(qs + v * 4) = pk[0];
        else
          *reinterpret_cast<uint2*>(qs + v * 8) = make_uint2(pk[0], pk[VE / 4 - 1]);
      }
    }
    tq = __reduce_add_sync(0xffffffffu, tq);
    if (lane == 0) red_q[warp] = tq;
  }
  __syncthreads();            // q row, q-sum partials and amax visible
  if (a.ld_at == 1) pdl_launch_dependents();
  if (warp >= a.ch) return;   // no channel for this warp (nothing else to do)
  mbar_wait(&wbar, 0);        // weights landed (long since, in a PDL chain)
  if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 5] = gtimer();
  const int qsum = __reduce_add_sync(0xffffffffu, lane < nwx ? red_q[lane] : 0);
  // ---- dot (a3): warp w owns channels w, w+16, ... with all their segments; lanes split
  // the row's 32-bit words (16 trits x 16 q bytes each)
  const int W = a.Kp >> 4, nkb = a.Kp >> 7, SW = a.sw_stride;
  const uint32_t* swd = sw_words(g_smem);
  int accl[3] = {0, 0, 0};   // lane j: channel warp + 16 j
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int i = warp + j * kGWarps;
    if (i >= a.ch) break;
    int pf[3][4];
#pragma unroll
    for (int sg = 0; sg < 3; ++sg)
#pragma unroll
      for (int f = 0; f < 4; ++f) pf[sg][f] = 0;
#pragma unroll 2
    for (int w = lane; w < ((a.strip & 1) ? 0 : W); w += 32) {
      const uint4 qv = *reinterpret_cast<const uint4*>(qs + w * 16);
      const uint32_t* wrow = swd + (w >> 3) * SW + (w & 7) + i * 8;
#pragma unroll
      for (int sg = 0; sg < 3; ++sg) {
        if (sg < a.n_seg) {
          const uint32_t wd = wrow[sg * nkb * SW];
          // field f of the word holds trits 4f..4f+3, i.e. q bytes [4f, 4f+4), times 4^f
          pf[sg][0] = dp4a_us(wd & 0x03030303u, qv.x, pf[sg][0]);
          pf[sg][1] = dp4a_us(wd & 0x0C0C0C0Cu, qv.y, pf[sg][1]);
          pf[sg][2] = dp4a_us(wd & 0x30303030u, qv.z, pf[sg][2]);
          pf[sg][3] = dp4a_us(wd & 0xC0C0C0C0u, qv.w, pf[sg][3]);
        }
      }
    }
    if (a.trace && tid == 0 && j == 0) a.trace[blockIdx.x * 16 + 6] = gtimer();
#pragma unroll
    for (int sg = 0; sg < 3; ++sg) {
      if (sg < a.n_seg) {
        // sum e q over the row: every term of the lane's field-f sum is a multiple of 4^f,
        // so the shifts are exact per lane; one REDUX per segment
        const int t = __reduce_add_sync(0xffffffffu, pf[sg][0] + (pf[sg][1] >> 2) +
                                                         (pf[sg][2] >> 4) + (pf[sg][3] >> 6));
        if (lane == j) accl[sg] = t - qsum;   // sum e q - sum q = sum t q
      }
    }
    if (a.trace && tid == 0 && j == 0) a.trace[blockIdx.x * 16 + 7] = gtimer();
  }
  if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 8] = gtimer();
  if (!own) return;
  // ---- epilogue (a5-a8), lane-parallel over the warp's channels
  const float amax = sh_amax;
  const float deq = amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
  TY* out = static_cast<TY*>(e.out);
  const int rr = rch;
  if (a.strip & 2) {
    st_act<TY>(out + rr, (float)accl[0]);
  } else if (e.kind == EPI_MLGRU) {
    const float fh = bl_val<TY>(e, accl[0], deq, msc[0], 0, rr);
    const float chh = bl_val<TY>(e, accl[1], deq, msc[1], 1, rr);
    const float gh = bl_val<TY>(e, accl[2], deq, msc[2], 2, rr);
    const float h = mlgru_step(sigmoid_c(fh), pre, silu_c(chh));
    e.h[rr] = h;
    st_act<TY>(out + rr, mlgru_out(gh, h, e.gate));
  } else if (e.kind == EPI_SWIGLU) {
    const float gh = bl_val<TY>(e, accl[0], deq, msc[0], 0, rr);
    const float uh = bl_val<TY>(e, accl[1], deq, msc[1], 1, rr);
    st_act<TY>(out + rr, swiglu(gh, uh));
  } else if (e.kind == EPI_RESID) {
    st_act<TY>(out + rr, __fadd_rn(pre, bl_val<TY>(e, accl[0], deq, msc[0], 0, rr)));
  } else {   // EPI_STORE / EPI_FCG
    for (int sg = 0; sg < a.n_seg; ++sg) {
      const float o = bl_val<TY>(e, sg == 0 ? accl[0] : (sg == 1 ? accl[1] : accl[2]), deq,
                                 sg == 0 ? msc[0] : (sg == 1 ? msc[1] : msc[2]), sg, rr);
      st_act<TY>(out + (e.kind == EPI_FCG ? packed_row(sg, rr, a.n_seg) : rr), o);
    }
  }
  if (a.trace && lane == 0 && warp == 0) a.trace[blockIdx.x * 16 + 2] = gtimer();
}

// One BitLinear per launch (PDL chain of launches).
template <int MM, typename TX, typename TY, bool CENT>
__global__ void __launch_bounds__(kGThreads) k_gemv(const GemvArgs a) {
  extern __shared__ __align__(128) uint8_t g_smem[];
  int8_t* qs = reinterpret_cast<int8_t*>(g_smem + (size_t)a.n_seg * (a.Kp >> 7) * a.sw_stride * 4);  // [MM][Kp]
  __shared__ double red_d[MM][kGWarps];
  __shared__ float red_m[MM][kGWarps];
  __shared__ int lq_s[MM][kGWarps][32];
  __shared__ __align__(8) uint64_t wbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = blockIdx.x;
  long long pt0 = 0;
  if (a.prof) pt0 = clock64();
  if (a.trace && tid == 0) {
    a.trace[blockIdx.x * 16 + 0] = gtimer();
    a.trace[blockIdx.x * 16 + 3] = clock64();
  }
  // packed weights -> smem with the TMA engine (bulk copies; the LSU pipe stays
  // free for the running kernel's critical path)
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&wbar, 1);
      fence_barrier_init();
    }
    __syncwarp();
    gemv_issue(a, unit, sw_words(g_smem), &wbar, lane, false);
  }
  // L2 prefetch of this CTA's share of a later launch's weights (HBM-resident
  // stacks: the weight stream runs ahead of the dependency chain)
  if (a.pf && tid == 32) {
    const size_t chunk = ((a.pf_bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
    const size_t off = chunk * blockIdx.x;
    if (off < a.pf_bytes) {
      const size_t n = a.pf_bytes - off < chunk ? a.pf_bytes - off : chunk;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf + off), "r"((uint32_t)n)
                   : "memory");
    }
  }
  // dequantization scales are constants: load them before the wait too
  float msc[3];
#pragma unroll
  for (int sg = 0; sg < 3; ++sg) msc[sg] = sg < a.n_seg ? __ldg(a.epi.scales + sg) : 0.0f;
  GPROF(0)
  pdl_wait();
  // let the next kernel start its weight prefetch only now: earlier triggers
  // let grids two launches ahead occupy SM slots and delay this grid's CTAs
  if (a.ld_at == 0) pdl_launch_dependents();
  GPROF(1)
  if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 1] = gtimer();
  float pre[4];
  gemv_pre<TY>(a, unit, warp, lane, pre);
  gemv_run<MM, TX, TY, CENT>(a, unit, sw_words(g_smem), qs, &wbar, 0, msc, pre, red_d, red_m, lq_s,
                             pt0);
  if (a.trace) {
    __syncthreads();
    if (tid == 0) {
      a.trace[blockIdx.x * 16 + 2] = gtimer();
      a.trace[blockIdx.x * 16 + 4] = clock64();
    }
  }
}
#undef GPROF

// ---------------------------------------------------------------- f2: whole stack
// One decode step through every block in ONE persistent launch:
// one CTA per SM, all co-resident (cooperative launch); the 4 dependent
// BitLinear phases of each block are separated by grid-wide barriers instead
// of kernel boundaries.  While phase p runs, the TMA engine already copies
// phase p+1's weight slice into the other shared-memory buffer and phase p+2's
// slice is prefetched into L2, so the weight stream runs ahead of the chain.
// The arithmetic of a phase is gemv_run's, bit for bit.
struct StackPhase {
  const void* x;          // input rows [M][K]
  const void* res;        // residual [M][n_out] (RESID)
  void* out;              // output [M][n_out]
  float* h;               // MLGRU state [M][n_out]
  const uint32_t* codes;  // packed weight group
  const float* scales;    // [n_seg]
  const float* gain;      // [K] or null
  const float* bias;      // [n_seg*n_out] or null
  int K, n_rows, n_out, ch, sw_stride, kind, n_seg, gate;
  float eps;
  int norm;
};
constexpr int kStackMaxPhases = 128;   // 32 blocks per launch (kernel parameter space)
constexpr size_t kStackTraceStride = 1024 * 16;   // = one k_gemv trace slot (kTraceCtas * 16)
struct StackArgs {
  int n_phase, M, buf_words, pad_;
  unsigned* bar;   // grid barrier: [0] counter (zero at launch), [64 + cta] flags
  int bar_mode;    // grid_wait
  unsigned epoch;  // flags (mode 2): phase p of this launch is complete at epoch + p + 1
  unsigned long long* trace;   // tern_trace_enable: one k_gemv-layout slot per phase
  StackPhase ph[kStackMaxPhases];
};

__device__ __forceinline__ GemvArgs stack_args(const StackPhase& s, int M) {
  GemvArgs a{};
  a.x = s.x;
  a.ldx = s.K;
  a.K = s.K;
  a.Kp = (s.K + kKAlign - 1) / kKAlign * kKAlign;
  a.M = M;
  a.gain = s.gain;
  a.eps = s.eps;
  a.codes = s.codes;
  a.n_rows = s.n_rows;
  a.n_out = s.n_out;
  a.n_seg = s.n_seg;
  a.ch = s.ch;
  a.sw_stride = s.sw_stride;
  a.inv_k = 1.0 / (double)s.K;
  a.norm = s.norm;
  a.epi.kind = s.kind;
  a.epi.n_out = s.n_out;
  a.epi.n_seg = s.n_seg;
  a.epi.scales = s.scales;
  a.epi.bias = s.bias;
  a.epi.out = s.out;
  a.epi.ldo = s.n_out;
  a.epi.res = s.res;
  a.epi.ldr = s.n_out;
  a.epi.h = s.h;
  a.epi.gate = s.gate;
  return a;
}

// Grid barrier between phases.  bar_mode (debug knob TERN_STACK_BAR):
//  0: one counter, red.release add / ld.acquire polling by thread 0
//  1: one counter, red.release add / relaxed polling + one acquire fence
//  2: one flag word per CTA (st.release of the phase number), warp 0 polls all
//     flags with relaxed loads, then one acquire fence
__device__ __forceinline__ void grid_arrive(unsigned* bar, int mode, unsigned phase_done) {
  if (mode == 2) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 64 + blockIdx.x), "r"(phase_done)
                 : "memory");
  } else {
    if (mode == 0) __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  }
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void watchdog(uint32_t& polls, unsigned long long& t0) {
  if ((++polls & 1023u) == 0) {   // a lost arrival traps instead of hanging the GPU
    const unsigned long long t = gtimer();
    if (t0 == 0) t0 = t;
    else if (t - t0 > 20000000000ull) __trap();
  }
}
// mode 0/1: called by thread 0; mode 2: called by warp 0
__device__ __forceinline__ void grid_wait(const unsigned* bar, int mode, unsigned target_count,
                                          unsigned phase, int lane) {
  uint32_t polls = 0;
  unsigned long long t0 = 0;
  if (mode == 0) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if ((int)(v - target_count) >= 0) break;
      watchdog(polls, t0);
    }
  } else if (mode == 1) {
    while ((int)(ld_relaxed(bar) - target_count) < 0) watchdog(polls, t0);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  } else {
    const unsigned G = gridDim.x;
    while (true) {
      bool ok = true;
      for (unsigned i = lane; i < G; i += 32) ok &= (int)(ld_relaxed(bar + 64 + i) - phase) >= 0;
      if (__all_sync(0xffffffffu, ok)) break;
      watchdog(polls, t0);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
}

template <int MM, typename TX, typename TY>
__global__ void __launch_bounds__(kGThreads, 1) k_stack_decode(const __grid_constant__ StackArgs sa) {
  extern __shared__ __align__(128) uint8_t g_smem[];
  uint32_t* const wb0 = sw_words(g_smem);   // weight buffers: wb0 + (p & 1) * buf_words
  int8_t* qs = reinterpret_cast<int8_t*>(g_smem + (size_t)sa.buf_words * 8);
  __shared__ double red_d[MM][kGWarps];
  __shared__ float red_m[MM][kGWarps];
  __shared__ int lq_s[MM][kGWarps][32];
  __shared__ __align__(8) uint64_t wbar[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = blockIdx.x;
  const unsigned G = gridDim.x;
  if (tid == 0) {
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) gemv_issue(stack_args(sa.ph[0], sa.M), unit, wb0, &wbar[0], lane, false);
#pragma unroll 1
  for (int p = 0; p < sa.n_phase; ++p) {
    GemvArgs a = stack_args(sa.ph[p], sa.M);
    if (sa.trace) {
      a.trace = sa.trace + (size_t)p * kStackTraceStride;
      if (tid == 0) {
        a.trace[blockIdx.x * 16 + 0] = gtimer();
        a.trace[blockIdx.x * 16 + 3] = clock64();
      }
    }
    // weights run ahead: p+1 into the other buffer (free: phase p-1 ended with a
    // block barrier), p+2 into L2
    if (p + 1 < sa.n_phase && warp == 0) {
      fence_proxy_async_smem();
      gemv_issue(stack_args(sa.ph[p + 1], sa.M), unit, wb0 + ((p + 1) & 1) * sa.buf_words,
                 &wbar[(p + 1) & 1], lane, false);
    }
    if (p + 2 < sa.n_phase && warp == 1)
      gemv_issue(stack_args(sa.ph[p + 2], sa.M), unit, nullptr, nullptr, lane, true);
    float msc[3];
#pragma unroll
    for (int sg = 0; sg < 3; ++sg) msc[sg] = sg < a.n_seg ? __ldg(a.epi.scales + sg) : 0.0f;
    // h and the residual were written at least two phases ago: safe before the barrier
    float pre[4];
    gemv_pre<TY>(a, unit, warp, lane, pre);
    if (p > 0) {
      if (sa.bar_mode == 2 ? warp == 0 : tid == 0)
        grid_wait(sa.bar, sa.bar_mode, (unsigned)p * G, sa.epoch + (unsigned)p, lane);
      __syncthreads();
    }
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16 + 1] = gtimer();
    if (unit * a.ch < a.n_out) {
      if (a.norm == TERN_NORM_CENTERED)
        gemv_run<MM, TX, TY, true>(a, unit, wb0 + (p & 1) * sa.buf_words, qs, &wbar[p & 1],
                                   (uint32_t)(p >> 1) & 1u, msc, pre, red_d, red_m, lq_s, 0);
      else
        gemv_run<MM, TX, TY, false>(a, unit, wb0 + (p & 1) * sa.buf_words, qs, &wbar[p & 1],
                                    (uint32_t)(p >> 1) & 1u, msc, pre, red_d, red_m, lq_s, 0);
    }
    __syncthreads();
    if (a.trace && tid == 0) {
      a.trace[blockIdx.x * 16 + 2] = gtimer();
      a.trace[blockIdx.x * 16 + 4] = clock64();
    }
    if (p + 1 < sa.n_phase && tid == 0) grid_arrive(sa.bar, sa.bar_mode, sa.epoch + (unsigned)p + 1);
  }
}

// ----------------------------------------------------------------- device trace (debug)
constexpr int kTraceLaunches = 1024, kTraceCtas = 1024;
static unsigned long long* g_trace = nullptr;
static bool g_trace_on = false;
static int g_trace_seq = 0;
static int g_trace_units[kTraceLaunches];

void gemv_trace_enable(int on) {
  if (on && !g_trace) {
    if (cudaMalloc(&g_trace, sizeof(unsigned long long) * kTraceLaunches * kTraceCtas * 16) != cudaSuccess) {
      g_trace = nullptr;
      return;
    }
  }
  g_trace_on = on && g_trace;
  g_trace_seq = 0;
  if (g_trace_on)   // unwritten marks read as 0 (tools/decode_trace.py prints them as '-')
    cudaMemset(g_trace, 0, sizeof(unsigned long long) * kTraceLaunches * kTraceCtas * 16);
}

unsigned long long* trace_slot(int kind, int ctas) {
  if (!g_trace_on) return nullptr;
  const int slot = g_trace_seq % kTraceLaunches;
  g_trace_units[slot] = (ctas < kTraceCtas ? ctas : kTraceCtas) | (kind << 20);
  ++g_trace_seq;
  return g_trace + (size_t)slot * kTraceCtas * 16;
}

int gemv_trace_collect(unsigned long long* out, int max_launches) {
  const int n = g_trace_seq < kTraceLaunches ? g_trace_seq : kTraceLaunches;
  if (!out || !g_trace) return n;
  const int m = n < max_launches ? n : max_launches;
  cudaDeviceSynchronize();
  for (int i = 0; i < m; ++i) {
    out[(size_t)i * (kTraceCtas * 16 + 1)] = (unsigned long long)g_trace_units[i];
    cudaMemcpy(out + (size_t)i * (kTraceCtas * 16 + 1) + 1, g_trace + (size_t)i * kTraceCtas * 16,
               sizeof(unsigned long long) * kTraceCtas * 16, cudaMemcpyDeviceToHost);
  }
  return m;
}

// smem words between K-blocks of one segment: ch rows x 8 words, padded to 8 mod 32
static int gemv_sw_stride(int ch) { return ch * 8 + ((8 - ch * 8) % 32 + 32) % 32; }
// dynamic shared memory of one CTA: weights and q rows
static size_t gemv_smem(int MM, int n_seg, int ch, int Kp) {
  return (size_t)n_seg * (Kp / 128) * gemv_sw_stride(ch) * 4 + (size_t)MM * Kp;
}

template <int MM, typename TX, typename TY>
static cudaError_t gemv_launch(const GemvArgs& a, int units, cudaStream_t s) {
  const size_t smem = gemv_smem(MM, a.n_seg, a.ch, a.Kp);
  const bool cent = a.norm == TERN_NORM_CENTERED;
  auto kern = cent ? k_gemv<MM, TX, TY, true> : k_gemv<MM, TX, TY, false>;
  static size_t smem_set[2] = {48 * 1024, 48 * 1024};
  if (smem > smem_set[cent]) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    smem_set[cent] = 200 * 1024;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static unsigned long long* dprof = nullptr;
  static const bool prof_on = getenv("TERN_GEMV_PROF") != nullptr;
  GemvArgs aa = a;
  if (g_trace_on && units <= kTraceCtas) {
    const int slot = g_trace_seq % kTraceLaunches;
    aa.trace = g_trace + (size_t)slot * kTraceCtas * 16;
    g_trace_units[slot] = units | (TERN_K_GEMV << 20);
    ++g_trace_seq;
  }
  if (prof_on) {  // debug only: per-phase clocks, printed after a synchronous run
    if (!dprof) cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * 4096);
    cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * 8 * 4096, s);
    aa.prof = dprof;
  }
  cudaError_t err = cudaLaunchKernelEx(&cfg, kern, aa);
  if (prof_on) {
    static unsigned long long h[8 * 4096];
    cudaMemcpyAsync(h, dprof, sizeof(unsigned long long) * 8 * units, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double sum[8] = {0}, mx[8] = {0};
    for (int b = 0; b < units; ++b)
      for (int i = 0; i < 7; ++i) {
        sum[i] += (double)h[b * 8 + i] / units;
        mx[i] = fmax(mx[i], (double)h[b * 8 + i]);
      }
    fprintf(stderr,
            "[gemv prof] M=%d K=%d n_out=%d n_seg=%d ch=%d units=%d | cycles avg: "
            "wload %.0f pdlwait %.0f sq %.0f r %.0f quant %.0f dot %.0f end %.0f (max end %.0f)\n",
            a.M, a.K, a.n_out, a.n_seg, a.ch, units, sum[0], sum[1],
            sum[2], sum[3], sum[4], sum[5], sum[6], mx[6]);
  }
  return err;
}

// the lean batch-1 kernel: M = 1, RMSNorm without a gain, no taps (TERN_GEMV_LEAN=0: off)
static bool gemv_lean_ok(const GemvArgs& a) {
  static const bool on = !getenv("TERN_GEMV_LEAN") || atoi(getenv("TERN_GEMV_LEAN")) != 0;
  return on && a.M == 1 && a.gain == nullptr && a.norm == TERN_NORM_RMS && a.prof == nullptr &&
         a.taps.q == nullptr && a.taps.deq == nullptr && a.taps.inv_rms == nullptr &&
         a.taps.absmax == nullptr && a.epi.acc == nullptr && a.epi.kind != EPI_NONE;
}

template <typename TX, typename TY>
static cudaError_t gemv1_launch(const GemvArgs& a, int units, cudaStream_t s) {
  const size_t smem = gemv_smem(1, a.n_seg, a.ch, a.Kp);
  auto kern = k_gemv1<TX, TY>;
  static size_t smem_set = 48 * 1024;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    smem_set = 200 * 1024;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GemvArgs aa = a;
  if (g_trace_on && units <= kTraceCtas) {
    const int slot = g_trace_seq % kTraceLaunches;
    aa.trace = g_trace + (size_t)slot * kTraceCtas * 16;
    g_trace_units[slot] = units | (TERN_K_GEMV << 20);
    ++g_trace_seq;
  }
  return cudaLaunchKernelEx(&cfg, kern, aa);
}

template <typename TX, typename TY>
static cudaError_t gemv_dispatch_m(const GemvArgs& a, int units, cudaStream_t s) {
  if (gemv_lean_ok(a)) return gemv1_launch<TX, TY>(a, units, s);
  if (a.M <= 1) return gemv_launch<1, TX, TY>(a, units, s);
  if (a.M <= 2) return gemv_launch<2, TX, TY>(a, units, s);
  return gemv_launch<4, TX, TY>(a, units, s);
}

bool gemv_supported(int M, int K, int xdt) {
  const int ve = xdt == TERN_BF16 ? 8 : 4;
  if (M < 1 || M > kGemvMaxM) return false;
  const int nvx = M <= 2 ? GNVX<2>::v : GNVX<4>::v;
  return K <= nvx * kGThreads * ve;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_gemv(const void* x, int xdt, int ydt, int M, int K, int ldx, const float* gain,
                        float eps, const tern_weight& w, const Epi& epi, const QuantTaps* taps,
                        cudaStream_t s, const void* pf, size_t pf_bytes, int norm) {
  if (M <= 0) return cudaSuccess;
  if (!gemv_supported(M, K, xdt)) return cudaErrorInvalidValue;
  GemvArgs a{};
  a.x = x;
  a.ldx = ldx;
  a.K = K;
  a.inv_k = 1.0 / (double)K;
  a.norm = norm;
  static const int ld_at = getenv("TERN_GEMV_LD_AT") ? atoi(getenv("TERN_GEMV_LD_AT")) : 0;
  static const int strip = getenv("TERN_GEMV_STRIP") ? atoi(getenv("TERN_GEMV_STRIP")) : 0;
  a.ld_at = ld_at;
  a.strip = strip;
  a.Kp = (K + kKAlign - 1) / kKAlign * kKAlign;
  a.M = M;
  a.gain = gain;
  a.eps = eps;
  a.codes = w.codes;
  a.n_rows = w.n_rows;
  a.n_out = w.n_out;
  a.n_seg = w.n_seg;
  const int MMt = M <= 1 ? 1 : (M <= 2 ? 2 : 4);
  // channels per CTA: one CTA per SM (the per-SM work is balanced and every
  // SM streams its share of the weights), bounded by shared memory and by
  // one thread per (token, channel) in the epilogue
  int ch = (w.n_out + num_sms() - 1) / num_sms();
  while (ch > 1 && (gemv_smem(MMt, w.n_seg, ch, a.Kp) > 160 * 1024 || ch > 4 * kGWarps)) --ch;
  if (gemv_smem(MMt, w.n_seg, ch, a.Kp) > 200 * 1024) return cudaErrorInvalidValue;
  a.ch = ch;
  a.sw_stride = gemv_sw_stride(ch);
  a.epi = epi;
  if (taps) a.taps = *taps;
  a.pf = static_cast<const uint8_t*>(pf);
  a.pf_bytes = pf ? (pf_bytes & ~size_t(15)) : 0;
  if (a.pf_bytes == 0) a.pf = nullptr;
  const int units = (w.n_out + ch - 1) / ch;
  const bool xb = xdt == TERN_BF16, yb = ydt == TERN_BF16;
  if (xb && yb) return gemv_dispatch_m<__nv_bfloat16, __nv_bfloat16>(a, units, s);
  if (xb) return gemv_dispatch_m<__nv_bfloat16, float>(a, units, s);
  if (yb) return gemv_dispatch_m<float, __nv_bfloat16>(a, units, s);
  return gemv_dispatch_m<float, float>(a, units, s);
}

// ---------------------------------------------------------------- f2 host side
template <int MM, typename T>
static cudaError_t stack_launch(const StackArgs& sa, int grid, size_t smem, cudaStream_t s) {
  auto kern = k_stack_decode<MM, T, T>;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (grid barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, sa);
}

bool stack_decode_plan(const StackPhaseDesc* ph, int n, int M, int xdt, size_t* smem_out) {
  if (n <= 0 || M < 1 || M > kGemvMaxM) return false;
  const int G = num_sms();
  const int MMt = M <= 1 ? 1 : (M <= 2 ? 2 : 4);
  size_t buf = 0;
  int kp_max = 0;
  for (int i = 0; i < n; ++i) {
    const tern_weight& w = ph[i].w;
    if (!gemv_supported(M, ph[i].K, xdt)) return false;
    const int ch = (w.n_out + G - 1) / G;
    if (ch > 4 * kGWarps) return false;   // epilogue: <= 4 channels per warp
    const int Kp = (ph[i].K + kKAlign - 1) / kKAlign * kKAlign;
    kp_max = Kp > kp_max ? Kp : kp_max;
    const size_t b = (size_t)w.n_seg * (Kp / 128) * gemv_sw_stride(ch) * 4;
    buf = b > buf ? b : buf;
  }
  const size_t smem = 2 * buf + (size_t)MMt * kp_max;
  if (smem > 200 * 1024) return false;
  if (smem_out) *smem_out = smem;
  return true;
}

cudaError_t launch_stack_decode(const StackPhaseDesc* ph, int n, int M, int xdt, unsigned* bar,
                                cudaStream_t s) {
  size_t smem = 0;
  if (!stack_decode_plan(ph, n, M, xdt, &smem)) return cudaErrorNotSupported;
  const int G = num_sms();
  for (int c0 = 0; c0 < n; c0 += kStackMaxPhases) {
    const int cn = n - c0 < kStackMaxPhases ? n - c0 : kStackMaxPhases;
    thread_local StackArgs sa;   // large: keep it off the host stack
    sa = StackArgs{};
    sa.n_phase = cn;
    sa.M = M;
    sa.bar = bar;
    sa.trace = nullptr;
    if (g_trace_on && G <= kTraceCtas && cn <= kTraceLaunches) {
      if (g_trace_seq % kTraceLaunches + cn > kTraceLaunches) g_trace_seq += kTraceLaunches - g_trace_seq % kTraceLaunches;
      const int slot = g_trace_seq % kTraceLaunches;
      sa.trace = g_trace + (size_t)slot * kTraceCtas * 16;
      for (int i = 0; i < cn; ++i) g_trace_units[slot + i] = G | (TERN_K_STACK << 20);
      g_trace_seq += cn;
    }
    size_t buf = 0;
    int kp_max = 0;
    for (int i = 0; i < cn; ++i) {
      const StackPhaseDesc& d = ph[c0 + i];
      StackPhase& q = sa.ph[i];
      q.x = d.x;
      q.res = d.res;
      q.out = d.out;
      q.h = d.h;
      q.codes = d.w.codes;
      q.scales = d.w.scales;
      q.gain = d.gain;
      q.bias = d.bias;
      q.K = d.K;
      q.n_rows = d.w.n_rows;
      q.n_out = d.w.n_out;
      q.n_seg = d.w.n_seg;
      q.ch = (d.w.n_out + G - 1) / G;
      q.sw_stride = gemv_sw_stride(q.ch);
      q.kind = d.kind;
      q.gate = d.gate;
      q.eps = d.eps;
      q.norm = d.norm;
      const int Kp = (d.K + kKAlign - 1) / kKAlign * kKAlign;
      kp_max = Kp > kp_max ? Kp : kp_max;
      const size_t b = (size_t)q.n_seg * (Kp / 128) * q.sw_stride * 4;
      buf = b > buf ? b : buf;
    }
    sa.buf_words = (int)(buf / 4);
    const int MMt = M <= 1 ? 1 : (M <= 2 ? 2 : 4);
    const size_t sm = 2 * buf + (size_t)MMt * kp_max;
    static const int bar_mode = getenv("TERN_STACK_BAR") ? atoi(getenv("TERN_STACK_BAR")) : 1;
    sa.bar_mode = bar_mode;
    // flags: zeroed with the counter, so every launch counts phases from 0
    sa.epoch = 0;
    cudaError_t e = cudaMemsetAsync(bar, 0, (64 + (size_t)G) * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    const bool b16 = xdt == TERN_BF16;
    if (MMt == 1) e = b16 ? stack_launch<1, __nv_bfloat16>(sa, G, sm, s) : stack_launch<1, float>(sa, G, sm, s);
    else if (MMt == 2) e = b16 ? stack_launch<2, __nv_bfloat16>(sa, G, sm, s) : stack_launch<2, float>(sa, G, sm, s);
    else e = b16 ? stack_launch<4, __nv_bfloat16>(sa, G, sm, s) : stack_launch<4, float>(sa, G, sm, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tern
