/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle of the MatMul-free LM
 * block forward pass (arxiv 2406.02528).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  It shares no code, header, table or constant generator with the
 * CUDA path in paper_2406_02528_b200/ and never includes or links it.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n (section named
 * beside it); "C<k>" = a reading listed in DESIGN.md section "Readings".
 *
 * Conventions:
 *   - every float operation is one IEEE binary32 operation, round to nearest
 *     even; this file is built with -O2 -ffp-contract=off, no fast-math, so
 *     the compiler never fuses a*b+c except where fmaf() is written;
 *   - round() in the paper ("round then clamp") is round half away
 *     from zero (C3) == C99 roundf();
 *   - sums of squares / absolute values accumulate in binary64 in index order
 *     (C4) and are rounded once to binary32;
 *   - exp is the canonical exp_c specified in DESIGN.md (C12), written out
 *     below from that specification;
 *   - bf16 storage points R0..R3 round to nearest even (C13).
 *
 * Loops run in the order the paper's equations are written; OpenMP is used
 * only across independent rows / (sequence, channel) pairs, each of which is
 * reduced sequentially, so results do not depend on the thread count.
 *
 * Parity status per function: all functions are pinned by tests in
 * tests/test_oracle_pins.py (the fixed-point orc_fxp_* section by
 * tests/test_fxp_oracle.py; the bf16 rounding points R1-R3 by its test_bf16_*
 * pins against torch's RNE) except the composed end-to-end block values,
 * which the paper never prints ("parity unpinned" for orc_block values;
 * they are pinned only through their pinned parts and invariants).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_DEGENERATE 2
#define ORC_ERR_OVERFLOW 5

/* ------------------------------------------------------------------------ */
/* threading                                                                 */
/* ------------------------------------------------------------------------ */
void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
int orc_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* scalar primitives                                                         */
/* ------------------------------------------------------------------------ */

/* bf16 storage rounding (C13): round a binary32 to the nearest bfloat16
 * (ties to even) and return it widened back to binary32.  NaN passes. */
float orc_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return x;
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  u &= 0xffff0000u;
  memcpy(&x, &u, 4);
  return x;
}

/* "round then clamp" of Alg. 1; round half away from zero
 * (C3) is exactly C99 roundf. */
static float rha(float v) { return roundf(v); }

/* Canonical exp_c (C12): range reduction
 * x = k ln2 + r with k = rint(x log2e), Cody-Waite two-constant reduction
 * with fmaf, degree-7 Taylor polynomial in Horner form with fmaf, then
 * scaling by 2^k.  Constants are the binary32 values listed in DESIGN.md. */
float orc_exp(float x) {
  if (x != x) return x;
  if (x >= 0x1.62e430p+6f) return INFINITY;   /* >= ln(FLT_MAX) */
  if (x < -0x1.5d589ep+6f) return 0.0f;       /* <  ln(FLT_MIN) */
  float k = rintf(x * 0x1.715476p+0f);         /* log2(e) */
  float r = fmaf(-k, 0x1.62e400p-1f, x);       /* ln2_hi  */
  r = fmaf(-k, 0x1.7f7d1cp-20f, r);            /* ln2_lo  */
  float p = 0x1.a01a02p-13f;                   /* 1/5040 */
  p = fmaf(p, r, 0x1.6c16c2p-10f);             /* 1/720  */
  p = fmaf(p, r, 0x1.111112p-7f);              /* 1/120  */
  p = fmaf(p, r, 0x1.555556p-5f);              /* 1/24   */
  p = fmaf(p, r, 0x1.555556p-3f);              /* 1/6    */
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  int ki = (int)k;
  if (ki > 127) { p = p * 2.0f; ki -= 1; }
  return p * ldexpf(1.0f, ki);
}

/* logistic sigmoid sigma(x) = 1/(1+e^{-x}) */
float orc_sigmoid(float x) { return 1.0f / (1.0f + orc_exp(-x)); }

/* SiLU tau(x) = x * sigma(x) ("tau is the SiLU activation") */
float orc_silu(float x) { return x * orc_sigmoid(x); }

void orc_exp_arr(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = orc_exp(x[i]);
}
void orc_sigmoid_arr(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = orc_sigmoid(x[i]);
}
void orc_bf16_arr(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = orc_bf16(x[i]);
}

/* ------------------------------------------------------------------------ */
/* a1: weight_quant (Alg. 1), absmean ternarization                */
/* ------------------------------------------------------------------------ */

/* m = mean(|W|) over the whole matrix (one scale per matrix, C6), summed in
 * binary64 in index order and rounded once to binary32 (C4).
 * Returns ORC_ERR_DEGENERATE for an all-zero or non-finite W (C7). */
int orc_absmean(const float* W, int64_t n, float* m_out) {
  if (n <= 0) return ORC_ERR_ARG;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(W[i])) return ORC_ERR_DEGENERATE;
    s += fabs((double)W[i]);
  }
  float m = (float)(s / (double)n);
  if (!(m > 0.0f) || !isfinite(m)) return ORC_ERR_DEGENERATE;
  *m_out = m;
  return ORC_OK;
}

/* s = 1/mean|W|;  W~ = round(s W) clamped to [-1,1]   (the listing's
 * "sX" is read as "sW", C6).  The dequantized weight is t * m ("* 1/s"). */
void orc_ternarize(const float* W, int64_t n, float m, int8_t* t) {
  float s = 1.0f / m;
  for (int64_t i = 0; i < n; ++i) {
    float v = rha(W[i] * s);
    if (v > 1.0f) v = 1.0f;
    if (v < -1.0f) v = -1.0f;
    t[i] = (int8_t)v;
  }
}

/* Zero fraction of a ternary matrix ("unstructured sparsity"). */
double orc_zero_fraction(const int8_t* t, int64_t n) {
  int64_t z = 0;
  for (int64_t i = 0; i < n; ++i) z += (t[i] == 0);
  return n > 0 ? (double)z / (double)n : 0.0;
}

/* Decoder of the GPU packing layout, written from its specification in
 * DESIGN.md "Packed weight layout" (not from the CUDA code):
 *   trit k of a row lives in word k/16 of that row, byte j = k%4, bit field
 *   f = (k%16)/4 at bits [8j+2f, 8j+2f+1]; the field holds e = t + 1 in
 *   {0,1,2}; storage is K-block-major: word w of packed row r is at index
 *   ((w/8) * n_rows + r) * 8 + w%8 (8 words = one K-block of 128 trits).
 * Rows of fused groups are interleaved in groups of seg_rows:
 *   packed row of (segment s, logical row r) =
 *     (r / seg_rows) * (n_seg * seg_rows) + s * seg_rows + r % seg_rows.
 * Returns ORC_ERR_ARG if a field holds the unused value 3. */
int64_t orc_packed_row(int64_t s, int64_t r, int64_t n_seg, int64_t seg_rows) {
  return (r / seg_rows) * (n_seg * seg_rows) + s * seg_rows + (r % seg_rows);
}
int orc_unpack_row(const uint32_t* codes, int64_t n_rows, int64_t r, int k, int8_t* t) {
  for (int kk = 0; kk < k; ++kk) {
    int64_t widx = kk / 16;
    uint32_t w = codes[((widx / 8) * n_rows + r) * 8 + widx % 8];
    int j = kk % 4, f = (kk % 16) / 4;
    uint32_t e = (w >> (8 * j + 2 * f)) & 3u;
    if (e == 3u) return ORC_ERR_ARG;
    t[kk] = (int8_t)((int)e - 1);
  }
  return ORC_OK;
}
/* Unpack segment s (n logical rows) of a packed group into t[n][k]. */
int orc_unpack_segment(const uint32_t* codes, int64_t n_rows, int n, int k, int n_seg, int s,
                       int seg_rows, int8_t* t) {
  for (int r = 0; r < n; ++r) {
    int64_t pr = orc_packed_row(s, r, n_seg, seg_rows);
    int rc = orc_unpack_row(codes, n_rows, pr, k, t + (int64_t)r * k);
    if (rc) return rc;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* a2: RMSNorm (Eq. 1, read as the mean form C1) and               */
/*     activation_quant (Alg. 1, per token C2)                     */
/* ------------------------------------------------------------------------ */

/* Norm variant: 0 = RMSNorm as read in C1 (default);
 * 1 = the centred form of Alg. 1 rms_norm_fwd, reading C22.
 * Process-wide setting of the oracle (test infrastructure). */
static int g_norm_mode = 0;
void orc_set_norm_mode(int mode) { g_norm_mode = mode; }
int orc_get_norm_mode(void) { return g_norm_mode; }

/* RMSNorm(x; w, eps) = x / sqrt(eps + mean(x^2)) * w   (C1).
 * r = 1/sqrt(mean(x^2) + eps) computed in binary64, rounded to binary32;
 * y_j = (x_j * r) * w_j  in binary32.  gain == NULL means w = 1.
 *
 * Centred form (Alg. 1: mu, sigma^2 = mean(X), variance(X);
 * r = 1/sqrt(sigma^2 + eps); Y = r (X - mu)), reading C22:
 *   mu      = (float)( sum_j x_j / K )              sum in binary64, index order
 *   sigma^2 = sum_j (x_j - mu)^2 / K                binary64 (x_j - mu is exact there)
 *   r       = (float)( 1 / sqrt(sigma^2 + eps) )    binary64, rounded once
 *   y_j     = ((x_j - mu) * r) * w_j                every step binary32 */
float orc_rmsnorm(const float* x, int K, const float* gain, float eps, float* y) {
  if (g_norm_mode == 1) {
    double sx = 0.0;
    for (int j = 0; j < K; ++j) sx += (double)x[j];
    const float mu = (float)(sx / (double)K);
    double sv = 0.0;
    for (int j = 0; j < K; ++j) {
      const double dj = (double)x[j] - (double)mu;
      sv += dj * dj;
    }
    const double var = sv / (double)K;
    float r = (float)(1.0 / sqrt(var + (double)eps));
    for (int j = 0; j < K; ++j) {
      float v = (x[j] - mu) * r;
      if (gain) v = v * gain[j];
      y[j] = v;
    }
    return r;
  }
  double ss = 0.0;
  for (int j = 0; j < K; ++j) ss += (double)x[j] * (double)x[j];
  double ms = ss / (double)K;
  float r = (float)(1.0 / sqrt(ms + (double)eps));
  for (int j = 0; j < K; ++j) {
    float v = x[j] * r;
    if (gain) v = v * gain[j];
    y[j] = v;
  }
  return r;
}

/* activation_quant: s = 127/max|y|, q = round(s y) clamped to
 * [-128,127]; the dequantization factor is 1/s, carried as deq = max|y|/127.
 * An all-zero row gives q = 0 and deq = 0 (C7). Returns max|y|. */
float orc_act_quant(const float* y, int K, int8_t* q, float* deq) {
  float a = 0.0f;
  for (int j = 0; j < K; ++j) {
    float v = fabsf(y[j]);
    if (v > a) a = v;
  }
  if (a == 0.0f) {
    for (int j = 0; j < K; ++j) q[j] = 0;
    *deq = 0.0f;
    return a;
  }
  float s = 127.0f / a;
  for (int j = 0; j < K; ++j) {
    float v = rha(y[j] * s);
    if (v > 127.0f) v = 127.0f;
    if (v < -128.0f) v = -128.0f;
    q[j] = (int8_t)v;
  }
  *deq = a / 127.0f;
  return a;
}

/* Fused norm + quant of M rows of X[M][K] (Alg. 1 rms_norm_fwd, P:325-334,
 * with the C1 reading).  Outputs q[M][K], deq[M], inv_rms[M], absmax[M]. */
int orc_quant_rows(const float* X, int M, int K, const float* gain, float eps, int8_t* q,
                   float* deq, float* inv_rms, float* absmax) {
  if (M < 0 || K <= 0) return ORC_ERR_ARG;
  int bad = 0;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    float* y = (float*)malloc(sizeof(float) * (size_t)K);
    if (!y) { bad = 1; continue; }
    float r = orc_rmsnorm(X + (int64_t)i * K, K, gain, eps, y);
    float a = orc_act_quant(y, K, q + (int64_t)i * K, &deq[i]);
    if (inv_rms) inv_rms[i] = r;
    if (absmax) absmax[i] = a;
    free(y);
  }
  return bad ? ORC_ERR_ARG : ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* a3/a4: ternary accumulation, literally  sum_{W=+1} x - sum_{W=-1} x  */
/* ------------------------------------------------------------------------ */
int64_t orc_tern_dot(const int8_t* t, const int8_t* q, int K) {
  int64_t plus = 0, minus = 0;
  for (int j = 0; j < K; ++j) {
    if (t[j] == 1) plus += q[j];
    else if (t[j] == -1) minus += q[j];
  }
  return plus - minus;
}

/* acc[M][N] = q[M][K] (*) t[N][K]^T  (int32; errors if a sum leaves int32) */
int orc_tern_matmul(const int8_t* q, int M, int K, const int8_t* t, int N, int32_t* acc) {
  int bad = 0;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i)
    for (int n = 0; n < N; ++n) {
      int64_t a = orc_tern_dot(t + (int64_t)n * K, q + (int64_t)i * K, K);
      if (a > INT32_MAX || a < INT32_MIN) bad = 1;
      acc[(int64_t)i * N + n] = (int32_t)a;
    }
  return bad ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* BitLinear forward (Alg. 1 forward_pass):                        */
/*   O = Y~ (*) W~ + b, Y~ = act_quant(RMSNorm(X)), dequantized by            */
/*   (1/s_a) * mean|W|  ("* 1/s", "* 1/s").                        */
/*   O_n = (float)acc_n * (deq * m)  [+ b_n]; in bf16 mode O is rounded to     */
/*   bf16 (R1).                                                               */
/* Optional taps: q_out[M][K], acc_out[M][N], deq_out[M].                      */
/* ------------------------------------------------------------------------ */
int orc_bitlinear(const float* X, int M, int K, const float* gain, float eps, const int8_t* t,
                  int N, float m_w, const float* bias, int bf16, float* O, int8_t* q_out,
                  int32_t* acc_out, float* deq_out) {
  if (M < 0 || K <= 0 || N <= 0) return ORC_ERR_ARG;
  int bad = 0;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    float* y = (float*)malloc(sizeof(float) * (size_t)K);
    int8_t* q = (int8_t*)malloc((size_t)K);
    if (!y || !q) { bad = ORC_ERR_ARG; free(y); free(q); continue; }
    float deq;
    orc_rmsnorm(X + (int64_t)i * K, K, gain, eps, y);
    orc_act_quant(y, K, q, &deq);
    float sc = deq * m_w;
    for (int n = 0; n < N; ++n) {
      int64_t a = orc_tern_dot(t + (int64_t)n * K, q, K);
      if (a > INT32_MAX || a < INT32_MIN) bad = ORC_ERR_OVERFLOW;
      float o = (float)a * sc;
      if (bias) o = o + bias[n];
      if (bf16) o = orc_bf16(o);
      O[(int64_t)i * N + n] = o;
      if (acc_out) acc_out[(int64_t)i * N + n] = (int32_t)a;
    }
    if (q_out) memcpy(q_out + (int64_t)i * K, q, (size_t)K);
    if (deq_out) deq_out[i] = deq;
    free(y);
    free(q);
  }
  return bad;
}

/* ------------------------------------------------------------------------ */
/* a6: MLGRU elementwise part:                                    */
/*   f_t = sigma(fhat_t), c_t = tau(chat_t), h_t = f_t h_{t-1} + (1-f_t) c_t, */
/*   o'_t = g_t * sigma(h_t)   (gate_mode 0)                           */
/*   o'_t = g_t * h_t          (gate_mode 1, BASELINE config 0 literal, C8)   */
/* Sequential over t per channel; h_0 = H (0 at prefill start).         */
/* Arrays are [B][T][d]; H is [B][d] in/out.  bf16 mode rounds o' (R2).       */
/* ------------------------------------------------------------------------ */

/* one recurrence step, h' = f*h + (1-f)*c, each product / sum one binary32 op */
static float scan_step(float f, float h, float c) {
  float a = f * h;
  float om = 1.0f - f;
  float b = om * c;
  return a + b;
}

/* Plain sequential scan of raw gates: h_t = f_t h_{t-1} + (1-f_t) c_t */
void orc_scan_seq(const float* f, const float* c, int T, float h0, float* h_out) {
  float h = h0;
  for (int t = 0; t < T; ++t) {
    h = scan_step(f[t], h, c[t]);
    h_out[t] = h;
  }
}

/* Self-check only (not the definition): chunked scan composing pairs
 * (a_t, b_t) = (f_t, (1-f_t) c_t) with (a2,b2) o (a1,b1) = (a1 a2, a2 b1 + b2)
 * (S:197).  Within a chunk the pairs are composed left to right; chunk
 * aggregates are then applied to the carried state. */
void orc_scan_chunked(const float* f, const float* c, int T, int chunk, float h0, float* h_out) {
  if (chunk <= 0) chunk = T > 0 ? T : 1;
  float h = h0;
  for (int s = 0; s < T; s += chunk) {
    int e = s + chunk < T ? s + chunk : T;
    /* local prefix of the chunk from state 0 with running products */
    float A = 1.0f, Bv = 0.0f;
    for (int t = s; t < e; ++t) {
      float a = f[t];
      float b = (1.0f - f[t]) * c[t];
      /* (a,b) o (A,Bv) */
      A = A * a;
      Bv = a * Bv + b;
      h_out[t] = A * h + Bv;
    }
    h = h_out[e - 1];
  }
}

/* Sequence-parallel scan ("a multi-GPU sequence-parallel scan (carry
 * exchange) is the long-context variant"; reading C23 in DESIGN.md).  The T steps are cut
 * into W contiguous slices [j T / W, (j+1) T / W).  Each slice's aggregate is the
 * left-to-right composition of its pairs (a, b) = (f, (1-f) c),
 *   A = A a,  Bv = a Bv + b   (from A = 1, Bv = 0; i.e. the recurrence from h = 0),
 * the boundary states compose in slice order, h_in(0) = H, h_in(j+1) = A_j h_in(j) + Bv_j,
 * each slice is then scanned sequentially from its h_in, and the final state is the
 * composition through every slice, h_in(W).  W = 1 is the sequential scan. */
static int g_scan_slices = 1;
void orc_set_scan_slices(int w) { g_scan_slices = w >= 1 ? w : 1; }
int orc_get_scan_slices(void) { return g_scan_slices; }

void orc_scan_seqpar(const float* f, const float* c, int T, int W, float h0, float* h_out,
                     float* h_final) {
  float hin = h0;
  for (int j = 0; j < W; ++j) {
    const int s0 = (int)((int64_t)j * T / W), s1 = (int)((int64_t)(j + 1) * T / W);
    float A = 1.0f, Bv = 0.0f;
    for (int t = s0; t < s1; ++t) {
      A = A * f[t];
      Bv = scan_step(f[t], Bv, c[t]);
    }
    float h = hin;
    for (int t = s0; t < s1; ++t) {
      h = scan_step(f[t], h, c[t]);
      h_out[t] = h;
    }
    hin = A * hin + Bv;
  }
  *h_final = hin;
}

static int orc_mlgru_scan_sp(const float* fhat, const float* chat, const float* ghat, int B, int T,
                             int d, int gate_mode, int bf16, float* H, float* oprime, int W) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int ch = 0; ch < d; ++ch) {
      float hin = H[(int64_t)b * d + ch];
      for (int j = 0; j < W; ++j) {
        const int s0 = (int)((int64_t)j * T / W), s1 = (int)((int64_t)(j + 1) * T / W);
        float A = 1.0f, Bv = 0.0f, h = hin;
        for (int t = s0; t < s1; ++t) {
          int64_t i = ((int64_t)b * T + t) * d + ch;
          float f = orc_sigmoid(fhat[i]);
          float c = orc_silu(chat[i]);
          A = A * f;
          Bv = scan_step(f, Bv, c);
          h = scan_step(f, h, c);
          float o = gate_mode == 0 ? ghat[i] * orc_sigmoid(h) : ghat[i] * h;
          if (bf16) o = orc_bf16(o);
          oprime[i] = o;
        }
        hin = A * hin + Bv;
      }
      H[(int64_t)b * d + ch] = hin;
    }
  return ORC_OK;
}

int orc_mlgru_scan(const float* fhat, const float* chat, const float* ghat, int B, int T, int d,
                   int gate_mode, int bf16, float* H, float* oprime) {
  if (B < 0 || T < 0 || d <= 0) return ORC_ERR_ARG;
  if (g_scan_slices > 1)
    return orc_mlgru_scan_sp(fhat, chat, ghat, B, T, d, gate_mode, bf16, H, oprime, g_scan_slices);
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int ch = 0; ch < d; ++ch) {
      float h = H[(int64_t)b * d + ch];
      for (int t = 0; t < T; ++t) {
        int64_t i = ((int64_t)b * T + t) * d + ch;
        float f = orc_sigmoid(fhat[i]);
        float c = orc_silu(chat[i]);
        h = scan_step(f, h, c);
        float o = gate_mode == 0 ? ghat[i] * orc_sigmoid(h) : ghat[i] * h;
        if (bf16) o = orc_bf16(o);
        oprime[i] = o;
      }
      H[(int64_t)b * d + ch] = h;
    }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* MLGRU token mixer, one call = B sequences of T tokens.         */
/* f,c,g,o BitLinears each preceded by their RMSNorm; f,c,g share the */
/* input and gain_x (C10).  Biases optional (C11).                            */
/* Taps (optional, [B][T][d]): fhat, chat, ghat, oprime.                      */
/* ------------------------------------------------------------------------ */
typedef struct {
  const int8_t *tf, *tc, *tg, *to;   /* [d][d] each, row = output channel */
  float mf, mc, mg, mo;              /* mean|W| per matrix */
  const float *bf, *bc, *bg, *bo;    /* [d] or NULL */
  const float *gain_x, *gain_o;      /* [d] or NULL (= ones) */
} orc_mlgru_w;

typedef struct {
  const int8_t *tg, *tu, *td;        /* [l][d], [l][d], [d][l] */
  float mg, mu, md;
  const float *gain_x, *gain_p;      /* [d], [l] or NULL */
} orc_glu_w;

int orc_mlgru(const orc_mlgru_w* w, const float* X, int B, int T, int d, float eps,
              int gate_mode, int bf16, float* H, float* O, float* fhat, float* chat,
              float* ghat, float* oprime) {
  int64_t n = (int64_t)B * T * d;
  int M = B * T;
  float* F = fhat ? fhat : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* C = chat ? chat : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* G = ghat ? ghat : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* P = oprime ? oprime : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  int rc = 0;
  rc |= orc_bitlinear(X, M, d, w->gain_x, eps, w->tf, d, w->mf, w->bf, bf16, F, 0, 0, 0);
  rc |= orc_bitlinear(X, M, d, w->gain_x, eps, w->tc, d, w->mc, w->bc, bf16, C, 0, 0, 0);
  rc |= orc_bitlinear(X, M, d, w->gain_x, eps, w->tg, d, w->mg, w->bg, bf16, G, 0, 0, 0);
  rc |= orc_mlgru_scan(F, C, G, B, T, d, gate_mode, bf16, H, P);
  rc |= orc_bitlinear(P, M, d, w->gain_o, eps, w->to, d, w->mo, w->bo, bf16, O, 0, 0, 0);
  if (!fhat) free(F);
  if (!chat) free(C);
  if (!ghat) free(G);
  if (!oprime) free(P);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* a7: GLU channel mixer: g = x(*)W_g, u = x(*)W_u,               */
/* p = tau(g) * u, d = p (*) W_d.  No biases.  bf16 rounds p (R2). */
/* Taps (optional): ghat, uhat [M][l], p [M][l].                               */
/* ------------------------------------------------------------------------ */
/* GLU gating p = tau(g) * u elementwise; bf16 mode rounds p (R2). */
void orc_swiglu_arr(const float* g, const float* u, int64_t n, int bf16, float* p) {
  for (int64_t i = 0; i < n; ++i) {
    float v = orc_silu(g[i]) * u[i];
    p[i] = bf16 ? orc_bf16(v) : v;
  }
}

int orc_glu(const orc_glu_w* w, const float* X, int M, int d, int l, float eps, int bf16,
            float* O, float* ghat, float* uhat, float* p) {
  int64_t n = (int64_t)M * l;
  float* G = ghat ? ghat : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* U = uhat ? uhat : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* Pp = p ? p : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  int rc = 0;
  rc |= orc_bitlinear(X, M, d, w->gain_x, eps, w->tg, l, w->mg, 0, bf16, G, 0, 0, 0);
  rc |= orc_bitlinear(X, M, d, w->gain_x, eps, w->tu, l, w->mu, 0, bf16, U, 0, 0, 0);
  orc_swiglu_arr(G, U, n, bf16, Pp);
  rc |= orc_bitlinear(Pp, M, l, w->gain_p, eps, w->td, d, w->md, 0, bf16, O, 0, 0, 0);
  if (!ghat) free(G);
  if (!uhat) free(U);
  if (!p) free(Pp);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* a8: block = token mixer + channel mixer with residuals (C9):        */
/*   x1 = x + MLGRU(x);  y = x1 + GLU(x1)   (bf16 mode rounds x1 and y, R3)   */
/* X, Y: [B][T][d]; H: [B][d] in/out.  Taps: x1 [B][T][d] (optional).          */
/* ------------------------------------------------------------------------ */
int orc_block(const orc_mlgru_w* mw, const orc_glu_w* gw, const float* X, int B, int T, int d,
              int l, float eps, int gate_mode, int bf16, float* H, float* Y, float* x1_tap) {
  int64_t n = (int64_t)B * T * d;
  int M = B * T;
  float* O = (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* X1 = x1_tap ? x1_tap : (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  float* D = (float*)malloc(sizeof(float) * (size_t)(n ? n : 1));
  int rc = orc_mlgru(mw, X, B, T, d, eps, gate_mode, bf16, H, O, 0, 0, 0, 0);
  for (int64_t i = 0; i < n; ++i) {
    float v = X[i] + O[i];
    X1[i] = bf16 ? orc_bf16(v) : v;
  }
  rc |= orc_glu(gw, X1, M, d, l, eps, bf16, D, 0, 0, 0);
  for (int64_t i = 0; i < n; ++i) {
    float v = X1[i] + D[i];
    Y[i] = bf16 ? orc_bf16(v) : v;
  }
  free(O);
  free(D);
  if (!x1_tap) free(X1);
  return rc;
}

/* ======================================================================== */
/* Fixed-point W8A16 numerics of the Loihi 2 deployment (*/
/* PAPER.md P:499-518 "Implementation Details on Intel Loihi 2"    */
/* Appendix "Fixed-Point Implementation Details").  Readings F1-F5 in        */
/* DESIGN.md.  Integer arithmetic only, except where a reading says a       */
/* constant is formed in binary64.                                           */
/* ======================================================================== */

/* round half away from zero of an exact rational v / 2^s, s >= 0 (F2, F5) */
static int64_t rha_shift(int64_t v, int s) {
  if (s == 0) return v;
  const uint64_t a = v < 0 ? (uint64_t)(-v) : (uint64_t)v;
  const uint64_t r = (a + ((uint64_t)1 << (s - 1))) >> s;
  return v < 0 ? -(int64_t)r : (int64_t)r;
}

/* F1 -- norm-scale quantization: w_q = round(w / s_w),
 * s_w = 2^(round(log2(max|w|)) - shift).  The paper's literal form is shift = 0
 * (then |w_q| <= 1); shift = 6 uses the int8 range (|w_q| <= 91).  round() is
 * half away from zero (C3); log2 is evaluated in binary64. */
int orc_fxp_scales(const float* w, int n, int shift, int8_t* wq, int* e_out) {
  if (n <= 0 || shift < 0 || shift > 6) return ORC_ERR_ARG;
  float mx = 0.0f;
  for (int i = 0; i < n; ++i) {
    const float a = fabsf(w[i]);
    if (a > mx) mx = a;
  }
  if (!(mx > 0.0f) || !isfinite(mx)) return ORC_ERR_DEGENERATE;
  const int e = (int)round(log2((double)mx)) - shift;
  for (int i = 0; i < n; ++i) {
    const double v = round(ldexp((double)w[i], -e));   /* w / 2^e is exact */
    if (v > 127.0 || v < -127.0) return ORC_ERR_OVERFLOW;
    wq[i] = (int8_t)v;
  }
  *e_out = e;
  return ORC_OK;
}

/* F2 -- dynamic 16-bit activation quantization, P:508 ("quantization scales
 * for the activations are computed for each batch individually"), with a
 * power-of-two scale ("bit-shift operations"): e = the smallest integer
 * with round(max|x| / 2^e) <= 32767; q = round(x / 2^e).  An all-zero tensor
 * gets e = 0. */
int orc_fxp_quant_act(const float* x, int64_t n, int16_t* q, int* e_out) {
  if (n < 0) return ORC_ERR_ARG;
  float mx = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    const float a = fabsf(x[i]);
    if (!isfinite(a)) return ORC_ERR_ARG;
    if (a > mx) mx = a;
  }
  int e = 0;
  if (mx > 0.0f) {
    int p;
    frexp((double)mx, &p);            /* mx in [2^(p-1), 2^p) */
    e = p - 16;                       /* mx / 2^e in [2^15, 2^16): too big ... */
    while (round(ldexp((double)mx, -e)) > 32767.0) ++e;
    while (round(ldexp((double)mx, -(e - 1))) <= 32767.0) --e;   /* ... smallest e */
  }
  for (int64_t i = 0; i < n; ++i) q[i] = (int16_t)round(ldexp((double)x[i], -e));
  *e_out = e;
  return ORC_OK;
}

/* F3 -- sigmoid LUT: x_fxp = round(x 2^x_exp), x_exp = 6; LUT of
 * N_sigma + 1 = 9 points x_i = i 2^x_exp (i = 0..8, i.e. x = 0, 1, ..., 8),
 * y_i = floor(sigma(i) 2^y_exp), y_exp = 15, sigma in binary64; piecewise
 * linear interpolation between adjacent points with a floor; inputs beyond
 * the last point take y_8; negative inputs via sigma(-x) = 1 - sigma(x), i.e.
 * 2^y_exp - y(|x|). */
#define ORC_FXP_XEXP 6
#define ORC_FXP_YEXP 15
#define ORC_FXP_NSIG 8
int32_t orc_fxp_sigmoid(int32_t x) {
  int32_t lut[ORC_FXP_NSIG + 1];
  for (int i = 0; i <= ORC_FXP_NSIG; ++i)
    lut[i] = (int32_t)floor(ldexp(1.0 / (1.0 + exp(-(double)i)), ORC_FXP_YEXP));
  const int64_t a = x < 0 ? -(int64_t)x : (int64_t)x;
  int32_t y;
  if (a >= ((int64_t)ORC_FXP_NSIG << ORC_FXP_XEXP)) {
    y = lut[ORC_FXP_NSIG];
  } else {
    const int i = (int)(a >> ORC_FXP_XEXP);
    const int64_t fr = a - ((int64_t)i << ORC_FXP_XEXP);
    y = lut[i] + (int32_t)(((int64_t)(lut[i + 1] - lut[i]) * fr) >> ORC_FXP_XEXP);
  }
  return x < 0 ? (1 << ORC_FXP_YEXP) - y : y;
}
void orc_fxp_sigmoid_arr(const int32_t* x, int32_t* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = orc_fxp_sigmoid(x[i]);
}

/* F4 -- inverse square root, P:722-723 ("treats the input as an integer
 * paired with a fixed exponent, uses a LUT with 24 values to produce an
 * initial guess ... refined using five iterations of the Newton-Raphson
 * method, all in a fixed-point format").  Input v 2^e with v > 0.  Normalise
 * to m 2^E, m in [1, 4) held as Q30 (m_q = m 2^30), E even; the 24 LUT values
 * are 1/sqrt of the centres of the 24 intervals [1 + k/8, 1 + (k+1)/8) that
 * tile [1, 4): g_k = round(2^30 / sqrt(1 + (k + 1/2)/8)) (binary64); then five
 * Newton steps y <- y (3 - m y^2) / 2 in Q30 with truncating shifts:
 *   y <- (y * (3*2^30 - ((m_q * ((y*y) >> 30)) >> 30))) >> 31.
 * Result: 1/sqrt(v 2^e) = y 2^(ey), ey = -30 - E/2. */
int orc_fxp_inv_sqrt(uint64_t v, int e, uint32_t* y_out, int* ey_out) {
  if (v == 0) return ORC_ERR_ARG;
  int p = 63;
  while (!((v >> p) & 1)) --p;                     /* v in [2^p, 2^(p+1)) */
  uint64_t m = p >= 30 ? v >> (p - 30) : v << (30 - p);   /* [2^30, 2^31); drops low bits */
  int E = e + p;
  if (E & 1) {                                     /* make the exponent even */
    m <<= 1;
    E -= 1;
  }
  const int k = (int)((m - ((uint64_t)1 << 30)) >> 27);   /* (m - 1) * 8 in [0, 24) */
  uint64_t y = (uint64_t)llround(ldexp(1.0, 30) / sqrt(1.0 + (k + 0.5) / 8.0));
  for (int it = 0; it < 5; ++it) {
    const uint64_t y2 = (y * y) >> 30;
    const uint64_t my2 = (m * y2) >> 30;
    y = (y * ((uint64_t)3 * ((uint64_t)1 << 30) - my2)) >> 31;
  }
  *y_out = (uint32_t)y;
  *ey_out = -30 - E / 2;
  return ORC_OK;
}
int orc_fxp_inv_sqrt_arr(const uint64_t* v, const int32_t* e, int64_t n, uint32_t* y,
                         int32_t* ey) {
  for (int64_t i = 0; i < n; ++i) {
    int t;
    const int rc = orc_fxp_inv_sqrt(v[i], e[i], &y[i], &t);
    if (rc) return rc;
    ey[i] = t;
  }
  return ORC_OK;
}

/* F5 -- RMSNorm of Eq. 1 in fixed point with eps = 1e-3,
 * read with the mean over the d channels (C1; the printed Eq. 1 omits 1/d):
 *   y_i = x_i / sqrt(eps + (1/d) sum_j x_j^2) * w_i
 * with x_i = xq_i 2^ex (int16, F2) and w_i = wq_i 2^ew (int8, F1).  Since
 *   1/sqrt(eps + S 2^(2ex)/d) = sqrt(d) 2^(-ex) / sqrt(S + eps_q),
 * S = sum xq_j^2 (int64, exact) and eps_q = round(d eps 2^(-2ex)) (binary64,
 * half away; 0 when eps underflows -- the paper's reason for eps = 1e-3),
 * the row computes (yq, ey) = inv_sqrt(S + eps_q, 0) (F4).  For activations so
 * small that round(d eps 2^(-2ex)) > 2^60 the sum is formed on a coarser even
 * grid 2^(2k) instead, with the smallest k for which it fits (reading F5b):
 *   D = rha(S / 2^(2k)) + round(d eps 2^(-2ex-2k)),  (yq, ey) = inv_sqrt(D, 2k),
 * which is the same value to 2^-60 relative (F4 keeps 31 bits of it); k = 0 is
 * the formula above.  Then
 * rsd = (yq * sd) >> 16 with sd = round(sqrt(d) 2^16) (binary64), then
 * t_i = xq_i * wq_i * rsd (int64, real value t_i 2^(ew + ey)), and stores
 * out_i = round(t_i / 2^s) (half away) with the smallest s >= 0 for which
 * every |out_i| <= 32767: output exponent eo = s + ew + ey per row.
 * A row with S + eps_q = 0 (all zero, eps underflowed) outputs zeros, eo = 0. */
int orc_fxp_rmsnorm(const int16_t* xq, int ex, const int8_t* wq, int ew, int rows, int d,
                    double eps, int16_t* out, int32_t* eo) {
  if (rows < 0 || d <= 0 || d > 65536 || !(eps >= 0.0)) return ORC_ERR_ARG;
  int k2 = 0;                                      /* the even grid 2^k2 of D (F5b) */
  while (round(ldexp((double)d * eps, -2 * ex - k2)) > 0x1p60) k2 += 2;
  const int64_t eps_q = (int64_t)round(ldexp((double)d * eps, -2 * ex - k2));
  const int64_t sd = (int64_t)llround(ldexp(sqrt((double)d), 16));
  for (int r = 0; r < rows; ++r) {
    const int16_t* x = xq + (int64_t)r * d;
    int16_t* o = out + (int64_t)r * d;
    int64_t S = 0;
    for (int j = 0; j < d; ++j) S += (int64_t)x[j] * x[j];
    const uint64_t D = (uint64_t)rha_shift(S, k2) + (uint64_t)eps_q;
    if (D == 0) {
      for (int j = 0; j < d; ++j) o[j] = 0;
      eo[r] = 0;
      continue;
    }
    uint32_t yq;
    int ey;
    orc_fxp_inv_sqrt(D, k2, &yq, &ey);
    const int64_t rsd = (int64_t)(((uint64_t)yq * (uint64_t)sd) >> 16);
    int64_t tmax = 0;
    for (int j = 0; j < d; ++j) {
      int64_t t = (int64_t)x[j] * wq[j] * rsd;
      if (t < 0) t = -t;
      if (t > tmax) tmax = t;
    }
    int s = 0;
    while (rha_shift(tmax, s) > 32767) ++s;
    for (int j = 0; j < d; ++j) o[j] = (int16_t)rha_shift((int64_t)x[j] * wq[j] * rsd, s);
    eo[r] = s + ew + ey;
  }
  return ORC_OK;
}

/* F6 -- a BitLinear in W8A16 ("8-bit weights and 16-bit activations"; the
 * ternary weights need no further quantization): F5's RMSNorm of the int16 input,
 * the ternary contraction of the int16 normalised activations (exact, int64 here; it
 * fits int32 for K <= 65535), the matrix scale beta quantized like the norm scales (F1
 * with shift 6 applied to the scalar beta), and the output requantized per row to int16
 * with the smallest fitting exponent (as in F5):
 *   (yn, en) = F5(xq, ex, gq, eg, eps);  acc[r][n] = sum_k t[n][k] yn[r][k];
 *   (bq, eb) = F1([beta], 6);  p = acc bq;  y = round(p / 2^s) (half away),
 *   ey[r] = s + en[r] + eb. */
int orc_fxp_bitlinear(const int16_t* xq, int ex, const int8_t* gq, int eg, double eps,
                      const int8_t* t, float beta, int M, int K, int N, int16_t* y, int32_t* ey) {
  if (M < 0 || K <= 0 || K > 65535 || N <= 0) return ORC_ERR_ARG;
  int8_t bq;
  int eb;
  int rc = orc_fxp_scales(&beta, 1, 6, &bq, &eb);
  if (rc) return rc;
  int16_t* yn = (int16_t*)malloc(sizeof(int16_t) * ((size_t)M * K + 1));
  int32_t* en = (int32_t*)malloc(sizeof(int32_t) * ((size_t)M + 1));
  int64_t* p = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  if (!yn || !en || !p) {
    free(yn);
    free(en);
    free(p);
    return ORC_ERR_ARG;
  }
  rc = orc_fxp_rmsnorm(xq, ex, gq, eg, M, K, eps, yn, en);
  for (int r = 0; r < M && rc == ORC_OK; ++r) {
    int64_t pmax = 0;
    for (int n = 0; n < N; ++n) {
      int64_t acc = 0;
      for (int k = 0; k < K; ++k) acc += (int64_t)t[(int64_t)n * K + k] * yn[(int64_t)r * K + k];
      p[n] = acc * bq;
      const int64_t a = p[n] < 0 ? -p[n] : p[n];
      if (a > pmax) pmax = a;
    }
    int s = 0;
    while (rha_shift(pmax, s) > 32767) ++s;
    for (int n = 0; n < N; ++n) y[(int64_t)r * N + n] = (int16_t)rha_shift(p[n], s);
    ey[r] = s + en[r] + eb;
  }
  free(yn);
  free(en);
  free(p);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* f4(iii): Alg. 1 BackwardPass of one BitLinear, straight-       */
/* through estimator.  Readings:                       */
/*   B1  "dY = dO x W^T": W is the ternarized weight the forward      */
/*       multiplied by, W~ = t m (the straight-through estimator passes the   */
/*       gradient of the quantizers through unchanged);                       */
/*   B2  "dW = dO^T x Y~" is [n_out][k_in], the latent weight's       */
/*       layout; Y~ = q deq (the forward's dequantized activation, a5);       */
/*   B3  mu, sigma^2, r "loaded" are the forward's own values,        */
/*       recomputed here with the forward's arithmetic (orc_rmsnorm);         */
/*   B4  rms_norm_bwd literally for the centred norm (norm = 1,   */
/*       reading C22); for the default RMSNorm (norm = 0, C1) mu is the       */
/*       constant 0, so the d mu term is absent: dX = r dY + 2 dsigma^2 X/N;  */
/*   B5  mean(X - mu) in d mu is as printed (the textbook factor -2   */
/*       multiplies the same mean, which is 0 up to rounding);                */
/*   B6  no gain (Alg. 1 has none); every sum in binary64, index order; the  */
/*       outputs are binary64 (the oracle's precision).                       */
/* Inputs: X [M][K] fp32, t [N][K] int8 trits with scale m_w (the forward's   */
/* W~ = t m_w), dO [M][N] fp32.  Outputs: dX [M][K], dW [N][K], db [N]        */
/* (db may be NULL), all double.                                              */
/* ------------------------------------------------------------------------ */
int orc_bitlinear_bwd(const float* X, int M, int K, const int8_t* t, int N, float m_w, float eps,
                      int norm, const float* dO, double* dX, double* dW, double* db) {
  if (M < 0 || K <= 0 || N <= 0 || (norm != 0 && norm != 1)) return ORC_ERR_ARG;
  const int saved = g_norm_mode;
  g_norm_mode = norm;
  double* Yt = (double*)malloc(sizeof(double) * ((size_t)M * K + 1));   /* Y~ = q deq, exact */
  if (!Yt) { g_norm_mode = saved; return ORC_ERR_ARG; }
  int bad = 0;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    const float* x = X + (int64_t)i * K;
    float* y = (float*)malloc(sizeof(float) * (size_t)K);
    int8_t* q = (int8_t*)malloc((size_t)K);
    double* dY = (double*)malloc(sizeof(double) * (size_t)K);
    if (!y || !q || !dY) { bad = 1; free(y); free(q); free(dY); continue; }
    /* forward recompute (B3): r from rms_norm_fwd, Y~ from activation_quant */
    const float r = orc_rmsnorm(x, K, NULL, eps, y);
    float deq;
    orc_act_quant(y, K, q, &deq);
    for (int j = 0; j < K; ++j) Yt[(int64_t)i * K + j] = (double)q[j] * (double)deq;
    float mu = 0.0f;
    if (norm == 1) {
      double sx = 0.0;
      for (int j = 0; j < K; ++j) sx += (double)x[j];
      mu = (float)(sx / (double)K);
    }
    /* dY = dO x W~^T (B1) */
    for (int j = 0; j < K; ++j) {
      double s = 0.0;
      for (int n = 0; n < N; ++n)
        s += (double)dO[(int64_t)i * N + n] * ((double)t[(int64_t)n * K + j] * (double)m_w);
      dY[j] = s;
    }
    /* rms_norm_bwd (B4/B5) */
    const double rd = (double)r;
    double dsig = 0.0;
    for (int j = 0; j < K; ++j) dsig += dY[j] * ((double)x[j] - (double)mu) * -0.5 * rd * rd * rd;
    double dmu = 0.0;
    if (norm == 1) {
      double s1 = 0.0, s2 = 0.0;
      for (int j = 0; j < K; ++j) {
        s1 += -rd * dY[j];
        s2 += (double)x[j] - (double)mu;
      }
      dmu = s1 + dsig * (s2 / (double)K);
    }
    for (int j = 0; j < K; ++j)
      dX[(int64_t)i * K + j] = rd * dY[j] + 2.0 * dsig * ((double)x[j] - (double)mu) / (double)K +
                               dmu / (double)K;
    free(y);
    free(q);
    free(dY);
  }
  g_norm_mode = saved;
  if (!bad) {
    /* dW = dO^T x Y~ (B2): dW[n][j] = sum_m dO[m][n] Y~[m][j] */
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N; ++n)
      for (int j = 0; j < K; ++j) {
        double s = 0.0;
        for (int i = 0; i < M; ++i)
          s += (double)dO[(int64_t)i * N + n] * Yt[(int64_t)i * K + j];
        dW[(int64_t)n * K + j] = s;
      }
    /* db = sum(dO) over tokens */
    if (db)
      for (int n = 0; n < N; ++n) {
        double s = 0.0;
        for (int i = 0; i < M; ++i) s += (double)dO[(int64_t)i * N + n];
        db[n] = s;
      }
  }
  free(Yt);
  return bad ? ORC_ERR_ARG : ORC_OK;
}
