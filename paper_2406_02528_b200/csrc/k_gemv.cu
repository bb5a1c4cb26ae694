// k_gemv.cu -- a3: decode-time ternary GEMV (M <= 8 tokens), HBM-bound on the
// packed weights.
//
//  * before griddepcontrol.wait (PDL) one thread starts bulk async copies of
//    the CTA's packed weight rows into shared memory, so the weight fetch
//    overlaps the previous kernel's tail (weights do not depend on it);
//  * prologue: every CTA re-computes the fused RMSNorm + absmax int8 quantization
//    of the M input rows (a2) into shared memory, in a fixed
//    reduction order, so no extra launch or grid sync is needed;
//  * main loop: packed weights are streamed with coalesced 32-bit non-caching
//    loads; the 2-bit fields e = t+1 are isolated with one AND each and fed to
//    dp4a (u8 x s8) against the int8 activations:
//        sum_k e_k q_k = acc + sum_k q_k  ->  acc = (sum) - qsum
//    four field accumulators per token are recombined exactly
//    (field f carries a factor 4^f);
//  * epilogue: dequantization (a5) and the fused functors (MLGRU step with the
//    state update, SwiGLU, residual add) per (token, channel).
// Work unit = `ch` logical channels of every segment of the group, so a CTA
// owns f, c and g (or gate and up) of the same channels.
#include "epilogue.cuh"

namespace tern {

constexpr int kGThreads = 256;
constexpr int kGWarps = kGThreads / 32;
constexpr int kGMaxPT = 28;  // prologue register tile: K <= 28*256 = 7168

struct GemvArgs {
  const void* x;
  int ldx, K, Kp, M;
  const float* gain;
  float eps;
  const uint32_t* codes;
  int n_rows, n_out, n_seg, ch, ksplit;
  Epi epi;
  QuantTaps taps;
};

__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int MM, typename TX, typename TY>
__global__ void __launch_bounds__(kGThreads) k_gemv(const GemvArgs a) {
  extern __shared__ __align__(128) uint8_t g_smem[];
  const int R = a.n_seg * a.ch;
  const int nkb = a.Kp / kKAlign;
  const int slot = a.ch * 8 + 8;   // words per (segment, K-block) slot, padded vs bank conflicts
  uint32_t* sW = reinterpret_cast<uint32_t*>(g_smem);         // [n_seg][nkb][slot] words
  int8_t* qs = reinterpret_cast<int8_t*>(g_smem + a.n_seg * nkb * slot * 4);   // [MM][Kp]
  int* accs = reinterpret_cast<int*>(qs + MM * a.Kp);               // [MM][R]
  __shared__ __align__(8) uint64_t wbar;
  __shared__ float s_deq[MM];
  __shared__ int s_qsum[MM];
  __shared__ double red_d[kGWarps];
  __shared__ float red_f[kGWarps];
  __shared__ int red_i[kGWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int unit = blockIdx.x;

  // ---------------- weight prefetch (independent of the previous kernel)
  if (tid == 0) {
    mbar_init(&wbar, 1);
    fence_barrier_init();
    fence_proxy_async_smem();
    // the unit's rows of one segment are consecutive packed rows, so each
    // (segment, K-block) is one contiguous span of vcnt*32 bytes
    const int vcnt = min(a.ch, a.n_out - unit * a.ch);
    mbar_arrive_expect_tx(&wbar, (uint32_t)(a.n_seg * nkb * vcnt * 32));
    for (int sg = 0; sg < a.n_seg; ++sg) {
      const int p0 = packed_row(sg, unit * a.ch, a.n_seg);
      for (int kb = 0; kb < nkb; ++kb)
        bulk_load(sW + (sg * nkb + kb) * slot, a.codes + ((int64_t)kb * a.n_rows + p0) * 8,
                  (uint32_t)vcnt * 32u, &wbar);
    }
  }
  pdl_launch_dependents();
  pdl_wait();

  for (int i = tid; i < MM * R; i += kGThreads) accs[i] = 0;

  // ---------------- prologue: fused RMSNorm + quantization (a2) per row
  for (int m = 0; m < MM; ++m) {
    int8_t* qrow = qs + m * a.Kp;
    if (m >= a.M) {
      for (int k = tid; k < a.Kp; k += kGThreads) qrow[k] = 0;
      if (tid == 0) { s_deq[m] = 0.0f; s_qsum[m] = 0; }
      continue;
    }
    const TX* xr = static_cast<const TX*>(a.x) + (int64_t)m * a.ldx;
    const int npt = (a.K + kGThreads - 1) / kGThreads;   // uniform: skips unused slots
    float v[kGMaxPT];
    double ss = 0.0;
    float xmax = 0.0f;
#pragma unroll
    for (int i = 0; i < kGMaxPT; ++i) {
      v[i] = 0.0f;
      if (i < npt) {
        const int k = tid + i * kGThreads;
        v[i] = k < a.K ? ld_act<TX>(xr + k) : 0.0f;
        ss += (double)v[i] * (double)v[i];
        xmax = fmaxf(xmax, fabsf(v[i]));
      }
    }
    // one reduction round for sum(x^2) and max|x|: without a gain,
    // max|x*r| = fl(max|x| * r) exactly (rounding is monotone)
    ss = warp_sum_f64(ss);
    xmax = warp_max_f32(xmax);
    if (lane == 0) { red_d[warp] = ss; red_f[warp] = xmax; }
    __syncthreads();
    double tot = 0.0;
    xmax = 0.0f;
#pragma unroll
    for (int i = 0; i < kGWarps; ++i) { tot += red_d[i]; xmax = fmaxf(xmax, red_f[i]); }
    const float r = (float)(1.0 / sqrt(tot / (double)a.K + (double)a.eps));
    float amax;
    if (a.gain == nullptr) {
      amax = __fmul_rn(xmax, r);
#pragma unroll
      for (int i = 0; i < kGMaxPT; ++i)
        if (i < npt) v[i] = __fmul_rn(v[i], r);
    } else {
      amax = 0.0f;
#pragma unroll
      for (int i = 0; i < kGMaxPT; ++i) {
        if (i < npt) {
          const int k = tid + i * kGThreads;
          float y = __fmul_rn(v[i], r);
          if (k < a.K) y = __fmul_rn(y, __ldg(a.gain + k));
          v[i] = y;
          amax = fmaxf(amax, fabsf(y));
        }
      }
      amax = warp_max_f32(amax);
      __syncthreads();
      if (lane == 0) red_f[warp] = amax;
      __syncthreads();
      amax = 0.0f;
#pragma unroll
      for (int i = 0; i < kGWarps; ++i) amax = fmaxf(amax, red_f[i]);
    }
    const float s = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
    int qsum = 0;
#pragma unroll
    for (int i = 0; i < kGMaxPT; ++i) {
      const int k = tid + i * kGThreads;
      if (i <= npt && k < a.Kp) {
        int qi = 0;
        if (k < a.K && amax > 0.0f) {
          // |v*s| <= 127 (1+2^-23) always, so the clamp to [-128,127] (C5) is inert
          const float t = round_half_away(__fmul_rn(v[i], s));
          qi = (int)t;
        }
        qsum += qi;
        qrow[k] = (int8_t)qi;
      }
    }
    qsum = warp_sum_i32(qsum);
    if (lane == 0) red_i[warp] = qsum;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int i = 0; i < kGWarps; ++i) t += red_i[i];
      s_qsum[m] = t;
      s_deq[m] = amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
      if (blockIdx.x == 0) {
        if (a.taps.deq) a.taps.deq[m] = s_deq[m];
        if (a.taps.inv_rms) a.taps.inv_rms[m] = r;
        if (a.taps.absmax) a.taps.absmax[m] = amax;
      }
    }
    __syncthreads();  // red_* reused by the next row
  }
  if (blockIdx.x == 0 && a.taps.q) {
    for (int m = 0; m < a.M; ++m)
      for (int k = tid; k < a.Kp; k += kGThreads)
        a.taps.q[(int64_t)m * a.taps.ldq + k] = qs[m * a.Kp + k];
  }

  // ---------------- main loop: (row quad, K slice) items per warp
  mbar_wait(&wbar, 0);
  const int nwords = a.Kp >> 4;
  const int nquads = (R + 3) >> 2;
  const int items = nquads * a.ksplit;
  const int wslice = (nwords + a.ksplit - 1) / a.ksplit;
  for (int it = warp; it < items; it += kGWarps) {
    const int quad = it / a.ksplit, ks = it % a.ksplit;
    const int w0 = ks * wslice;
    const int w1 = min(nwords, w0 + wslice);
    const uint32_t* wrow[4];
    bool valid[4];
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) {
      const int j = quad * 4 + qd;
      const int seg = j / a.ch, i = j % a.ch;
      const int rr = unit * a.ch + i;
      valid[qd] = (j < R) && (rr < a.n_out);
      wrow[qd] = sW + (valid[qd] ? (seg * nkb * slot + i * 8) : 0);
    }
    int acc[4][MM];
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
#pragma unroll
      for (int m = 0; m < MM; ++m) acc[qd][m] = 0;
    for (int w = w0 + lane; w < w1; w += 32) {
      uint32_t wd[4];
#pragma unroll
      const int wo = (w >> 3) * slot + (w & 7);   // (K-block, word) inside the slot
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) wd[qd] = valid[qd] ? wrow[qd][wo] : 0x55555555u;
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const uint4 qv = *reinterpret_cast<const uint4*>(qs + m * a.Kp + w * 16);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          // field f carries e*4^f; fold 4^f back after the reduction
          int f0 = dp4a_us(wd[qd] & 0x03030303u, qv.x, 0);
          int f1 = dp4a_us(wd[qd] & 0x0C0C0C0Cu, qv.y, 0);
          int f2 = dp4a_us(wd[qd] & 0x30303030u, qv.z, 0);
          int f3 = dp4a_us(wd[qd] & 0xC0C0C0C0u, qv.w, 0);
          acc[qd][m] += f0 + (f1 >> 2) + (f2 >> 4) + (f3 >> 6);
        }
      }
    }
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const int t = warp_sum_i32(acc[qd][m]);
        if (lane == 0 && valid[qd]) atomicAdd(&accs[m * R + quad * 4 + qd], t);
      }
  }
  __syncthreads();

  // ---------------- epilogue per (token, channel)
  const Epi& e = a.epi;
  for (int idx = tid; idx < MM * a.ch; idx += kGThreads) {
    const int m = idx / a.ch, i = idx % a.ch;
    const int rr = unit * a.ch + i;
    if (m >= a.M || rr >= a.n_out) continue;
    const float deq = s_deq[m];
    const int* am = accs + m * R;
    if (e.acc) {
      for (int sg = 0; sg < a.n_seg; ++sg)
        e.acc[(int64_t)m * e.ldacc + packed_row(sg, rr, a.n_seg)] = am[sg * a.ch + i] - s_qsum[m];
    }
    TY* out = static_cast<TY*>(e.out);
    if (e.kind == EPI_MLGRU) {
      const float fh = bl_out<TY>(e, am[i] - s_qsum[m], deq, 0, rr);
      const float chh = bl_out<TY>(e, am[a.ch + i] - s_qsum[m], deq, 1, rr);
      const float gh = bl_out<TY>(e, am[2 * a.ch + i] - s_qsum[m], deq, 2, rr);
      const float f = sigmoid_c(fh);
      const float c = silu_c(chh);
      float* hp = e.h + (int64_t)m * e.n_out + rr;
      const float h = mlgru_step(f, *hp, c);
      *hp = h;
      st_act<TY>(out + (int64_t)m * e.ldo + rr, mlgru_out(gh, h, e.gate));
    } else if (e.kind == EPI_SWIGLU) {
      const float gh = bl_out<TY>(e, am[i] - s_qsum[m], deq, 0, rr);
      const float uh = bl_out<TY>(e, am[a.ch + i] - s_qsum[m], deq, 1, rr);
      st_act<TY>(out + (int64_t)m * e.ldo + rr, swiglu(gh, uh));
    } else if (e.kind != EPI_NONE) {
      Epi e1 = e;
      e1.acc = nullptr;
      epi_single<TY>(e1, m, rr, 0, rr, am[i] - s_qsum[m], deq);
    }
  }
}

template <int MM, typename TX, typename TY>
static cudaError_t gemv_launch(const GemvArgs& a, int units, cudaStream_t s) {
  const int R = a.n_seg * a.ch;
  const size_t smem = (size_t)a.n_seg * (a.Kp / kKAlign) * (a.ch * 8 + 8) * 4 + (size_t)MM * a.Kp +
                      (size_t)MM * R * sizeof(int);
  auto kern = k_gemv<MM, TX, TY>;
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
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename TX, typename TY>
static cudaError_t gemv_dispatch_m(const GemvArgs& a, int units, cudaStream_t s) {
  if (a.M <= 1) return gemv_launch<1, TX, TY>(a, units, s);
  if (a.M <= 2) return gemv_launch<2, TX, TY>(a, units, s);
  if (a.M <= 4) return gemv_launch<4, TX, TY>(a, units, s);
  return gemv_launch<8, TX, TY>(a, units, s);
}

cudaError_t launch_gemv(const void* x, int xdt, int ydt, int M, int K, int ldx, const float* gain,
                        float eps, const tern_weight& w, const Epi& epi, const QuantTaps* taps,
                        cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (M > 8 || K > kGMaxPT * kGThreads) return cudaErrorInvalidValue;
  GemvArgs a{};
  a.x = x;
  a.ldx = ldx;
  a.K = K;
  a.Kp = (K + kKAlign - 1) / kKAlign * kKAlign;
  a.M = M;
  a.gain = gain;
  a.eps = eps;
  a.codes = w.codes;
  a.n_rows = w.n_rows;
  a.n_out = w.n_out;
  a.n_seg = w.n_seg;
  // channels per CTA: enough CTAs to cover the SMs about twice
  int ch = 32;
  while (ch > 4 && (w.n_out + ch - 1) / ch < 296) ch >>= 1;
  if (w.n_seg == 3 && ch > 8) ch = 8;
  a.ch = ch;
  const int nquads = (w.n_seg * ch + 3) / 4;
  int ksplit = 1;
  while (nquads * ksplit < kGWarps && ksplit < 8) ksplit <<= 1;
  a.ksplit = ksplit;
  a.epi = epi;
  if (taps) a.taps = *taps;
  const int units = (w.n_out + ch - 1) / ch;
  const bool xb = xdt == TERN_BF16, yb = ydt == TERN_BF16;
  if (xb && yb) return gemv_dispatch_m<__nv_bfloat16, __nv_bfloat16>(a, units, s);
  if (xb) return gemv_dispatch_m<__nv_bfloat16, float>(a, units, s);
  if (yb) return gemv_dispatch_m<float, __nv_bfloat16>(a, units, s);
  return gemv_dispatch_m<float, float>(a, units, s);
}

}  // namespace tern
