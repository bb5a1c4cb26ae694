/*
 * tern.h -- C ABI of libtern.so, a B200 (sm_100a) implementation of the
 * forward pass of the MatMul-free LM block (arxiv 2406.02528).
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; C<k> = a reading of
 * the paper listed in DESIGN.md "Readings"; DESIGN.md sections are named.
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA memory)
 *    unless a comment says "host".  The caller owns every buffer, including
 *    the workspace; the library never allocates device memory.
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream), performs no host synchronisation (except tern_pack,
 *    see below) and no allocation, and is therefore CUDA-graph capturable.
 *  - Arguments are validated before anything is launched; a call that
 *    returns an error has had no side effect.  A call with no tokens (B*T or
 *    m == 0) is a no-op returning TERN_OK; its buffers may then be NULL.  Checked: NULL pointers, sizes
 *    <= 0, K and leading dimensions not multiples of 16 elements, pointers
 *    not 16-byte aligned, workspace too small, device not sm_100.
 *  - Errors are returned as tern_status; tern_last_error() gives a
 *    thread-local message.  Asynchronous kernel faults surface at the next
 *    synchronisation, as in CUDA.  Nothing aborts and nothing throws.
 *  - Activations are row-major [rows][ld] in tern_dtype; fp32 scales;
 *    the recurrent state h is always fp32 [B][d] (C13).
 *  - Numerics follow DESIGN.md "Canonical numerics" exactly (round half
 *    away from zero C3, binary64 sums of squares C4, canonical exp C12,
 *    bf16 storage points R0-R3), so integer results (int8 activations,
 *    int32 accumulators, ternary codes) reproduce the CPU oracle bit for bit
 *    given the same fp32 scales.
 *  - y must not alias x.  h is updated in place.  Concurrent calls must use
 *    disjoint h and workspace buffers.
 */
#ifndef TERN_H
#define TERN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define TERN_ABI_VERSION 1

typedef struct CUstream_st* tern_stream; /* == cudaStream_t */

typedef enum {
  TERN_OK = 0,
  TERN_ERR_INVALID_ARG = 1,  /* bad pointer / size / alignment / workspace       */
  TERN_ERR_DEGENERATE = 2,   /* tern_pack: mean|W| == 0 or W non-finite (C7)       */
  TERN_ERR_UNSUPPORTED = 3,  /* shape or device this build does not handle        */
  TERN_ERR_CUDA = 4          /* a CUDA runtime error; text in tern_last_error()    */
} tern_status;

typedef enum { TERN_F32 = 0, TERN_BF16 = 1 } tern_dtype;

/* MLGRU output gate (C8): o' = g * sigma(h) as written in P:452 / P:661, or
 * o' = g * h as written in BASELINE.json configs[0]. */
typedef enum { TERN_GATE_SIGMOID_H = 0, TERN_GATE_LINEAR_H = 1 } tern_gate_mode;
/* The norm in front of every BitLinear:
 *   TERN_NORM_RMS      = 0: y = x r w, r = 1/sqrt(mean(x^2) + eps)   (Eq. 1, reading C1; default)
 *   TERN_NORM_CENTERED = 1: y = (x - mu) r w, r = 1/sqrt(var(x) + eps)  (Alg. 1, C22)
 * with mu = (float)(sum x / K) and var = sum (x - mu)^2 / K in binary64. */
typedef enum { TERN_NORM_RMS = 0, TERN_NORM_CENTERED = 1 } tern_norm_mode;

int tern_abi_version(void);
/* Thread-local text of the last error (host pointer, valid until the next call). */
const char* tern_last_error(void);

/* ------------------------------------------------------------------------
 * Packed ternary weights (a1).  DESIGN.md "Packed weight layout":
 *   trit t in {-1,0,+1} is stored as the 2-bit field e = t + 1;
 *   16 trits per uint32 word: trit k is in word k/16 of its row, byte k%4,
 *   bits [2f, 2f+1] of that byte with f = (k%16)/4;
 *   K-block-major storage: codes[Kp/128][n_rows][8] -- word j of packed row
 *   r in K-block b (trits 128b+16j .. 128b+16j+15) is at ((b*n_rows)+r)*8+j,
 *   so one K-block of any run of rows is contiguous (one bulk copy per tile);
 *   Kp = roundup(k, 128), ldw = Kp/16 words per row; trits in the padding
 *   k..Kp-1 are 0 (field 1).
 * A fused group of n_seg matrices of n_out rows each (f|c|g: 3, gate|up: 2)
 * interleaves rows in groups of seg_rows (64):
 *   packed row of (segment s, row r) = (r/64)*(n_seg*64) + s*64 + r%64,
 *   n_rows = roundup(n_out, 64) * n_seg (rows of a ragged last group are
 *   padding and produce outputs that are never stored).
 * One fp32 dequantization scale mean|W| per segment (one per matrix, C6).
 * ------------------------------------------------------------------------ */
typedef struct {
  const uint32_t* codes;  /* device [Kp/128][n_rows][8] (K-block-major, see above) */
  const float* scales;    /* device [n_seg]: mean|W| of each source matrix         */
  int32_t n_out;          /* logical output rows per segment                       */
  int32_t k;              /* logical input features                                */
  int32_t ldw;            /* words per packed row, == roundup(k,128)/16            */
  int32_t n_seg;          /* 1, 2 or 3                                             */
  int32_t n_rows;         /* packed rows = roundup(n_out,64)*n_seg (n_seg>1) or n_out */
  const uint8_t* e8;      /* optional device [n_rows][Kp] u8 copy of the fields e=t+1
                             (tern_expand); when set, the prefill GEMM loads it with TMA
                             instead of unpacking the 2-bit codes in shared memory; NULL
                             = unpack in shared memory (4x less memory)             */
} tern_weight;

/* Number of packed rows and words per row for a group (host helper). */
int32_t tern_packed_rows(int32_t n_out, int32_t n_seg);
int32_t tern_packed_ldw(int32_t k);

/* Fill the n_rows*ldw words of codes with the zero trit (field value 1).
 * Call once on a fresh buffer before tern_pack. */
tern_status tern_codes_init(uint32_t* codes, int32_t n_rows, int32_t ldw, tern_stream stream);

/* Bytes of workspace tern_pack needs for an [n][k] matrix. */
size_t tern_pack_workspace(int32_t n, int32_t k);

/* a1: absmean ternarization + packing (Alg. 1 weight_quant):
 *   m = mean|W| (binary64 sum, rounded once to fp32, C4) or *scale_in,
 *   s = 1/m, t = clamp(round(s*W), -1, 1) with round half away from zero.
 * W: device fp32 [n][k] row-major (the latent weight of ONE matrix).
 * scale_in: device pointer to one float, or NULL to compute mean|W|.
 * Writes segment seg_idx of the group into codes (see layout above; n_rows =
 * tern_packed_rows(n, n_seg) rows of the whole group) and the
 * scale to scale_out[0] (device).  This offline call synchronises `stream`
 * to check the scale: returns TERN_ERR_DEGENERATE if m == 0 or is not finite
 * (S:39).  ws: device workspace of tern_pack_workspace(n,k) bytes. */
tern_status tern_pack(const float* W, int32_t n, int32_t k, const float* scale_in, int32_t n_seg,
                      int32_t seg_idx, uint32_t* codes, int32_t n_rows, float* scale_out, void* ws,
                      size_t ws_bytes, tern_stream stream);

/* Expand the 2-bit codes of w into the u8 copy e8[n_rows][Kp] (field values
 * e = t+1) used by the prefill GEMM's TMA path; e8 must hold n_rows*Kp bytes. */
tern_status tern_expand(const tern_weight* w, uint8_t* e8, tern_stream stream);

/* ------------------------------------------------------------------------
 * a2: fused RMSNorm + per-token absmax int8 quantization (Alg. 1
 * rms_norm_fwd + activation_quant, Eq. 1, readings C1,
 * C2, C3, C4, C5, C7):
 *   r = (float)(1/sqrt(mean_fp64(x^2) + eps)); y = (x*r)*gain;
 *   a = max|y|; q = clamp(round(y*(127/a)), -128, 127); deq = a/127;
 *   a == 0 gives q = 0 and deq = 0.
 * x: [m][ldx] of xdt; gain: [k] fp32 or NULL (ones).
 * Outputs: q int8 [m][ldq] (ldq >= roundup(k,128); columns k..ldq-1 are
 * written as 0), deq [m], qsum [m] = sum_j q_j (int32), and optionally
 * inv_rms [m] and absmax [m] (NULL to skip).
 * ------------------------------------------------------------------------ */
tern_status tern_quant(const void* x, tern_dtype xdt, int32_t m, int32_t k, int32_t ldx,
                       const float* gain, float eps, int8_t* q, int32_t ldq, float* deq,
                       int32_t* qsum, float* inv_rms, float* absmax, tern_stream stream);

/* Optional parity taps of bitlinear_fwd; any pointer may be NULL. */
typedef struct {
  int8_t* q;        /* [m][ldq] quantized activations                       */
  int32_t ldq;
  int32_t* acc;     /* [m][ldacc] int32 ternary accumulators, packed-row order */
  int32_t ldacc;
  float* deq;       /* [m] absmax/127                                         */
  float* inv_rms;   /* [m]                                                    */
  float* absmax;    /* [m]                                                    */
} tern_bl_taps;

/* Workspace bytes for bitlinear_fwd on m rows of k features.  For
 * 4 < m <= 256 it includes room for split-K int32 partials (38.8 MB), which
 * lets the GEMM spread few output tiles over all SMs; a smaller workspace
 * (>= the m*Kp + 512-byte base) is accepted and runs without split-K. */
size_t tern_bitlinear_workspace(int32_t m, int32_t k);

/* a2-a5: BitLinear forward (Alg. 1 forward_pass):
 *   acc_n = sum_{t=+1} q - sum_{t=-1} q  (int32)
 *   y_n = (float)acc_n * (deq * m_seg) [+ bias_n]
 * rounded to bf16 when ydt == TERN_BF16 (R1).
 * w must have n_seg == 1.  y: [m][ldy] of ydt, ldy >= w->n_out.
 * m <= tern_get_gemv_max_m() (and K within the GEMV's register tile: fp32
 * K <= 4096, bf16 K <= 8192) runs the decode GEMV (norm+quant fused in its
 * prologue); larger m runs tern_quant + the tcgen05 int8 GEMM. */
tern_status bitlinear_fwd(const void* x, tern_dtype xdt, int32_t m, int32_t k, int32_t ldx,
                          const float* gain, float eps, const tern_weight* w, const float* bias,
                          void* y, tern_dtype ydt, int32_t ldy, const tern_bl_taps* taps, void* ws,
                          size_t ws_bytes, tern_stream stream);

/* a3/a4 on pre-quantized activations (parity entry point):
 * acc[m][ldacc] = q (*) W~ over all packed rows (int32, exact). */
tern_status tern_contract(const int8_t* q, int32_t m, int32_t ldq, const int32_t* qsum,
                          const tern_weight* w, int32_t* acc, int32_t ldacc, tern_stream stream);

/* ------------------------------------------------------------------------
 * a6: MLGRU gates + recurrence + output gate:
 *   f = sigma(fhat), c = SiLU(chat), h_t = f*h_{t-1} + (1-f)*c, h_0 = h,
 *   o' = ghat * sigma(h_t) (gate = TERN_GATE_SIGMOID_H) or ghat * h_t.
 * fcg: [B*T][3d] pre-activations in the fused interleaved order
 *      (per 64-channel group: 64 f | 64 c | 64 g), dtype dt;
 * h:   fp32 [B][d] in/out; oprime: [B*T][d] dtype dt (bf16 rounds o', R2).
 * Exact sequential recurrence per channel (bit-identical to the oracle);
 * the transcendental work is spread over time within each CTA. d % 64 == 0.
 * ------------------------------------------------------------------------ */
tern_status tern_mlgru_scan(const void* fcg, tern_dtype dt, int32_t B, int32_t T, int32_t d,
                            tern_gate_mode gate, float* h, void* oprime, tern_stream stream);

/* ------------------------------------------------------------------------
 * Mixers and block.  Weight groups: fcg = {W_f, W_c, W_g} (n_seg 3, d->d),
 * o = W_o (d->d), gu = {W_gate, W_up} (n_seg 2, d->l), down = W_down (l->d).
 * Gains: NULL = ones.  Biases (C11) optional; the GLU has none.
 * Each BitLinear normalizes its own input; f, c and g share theirs
 * (C10), as do gate and up.
 * ------------------------------------------------------------------------ */
typedef struct {
  tern_weight fcg, o;
  const float *gain_x, *gain_o;     /* [d], [d]                */
  const float *bias_fcg;            /* [3][d] (f, c, g) or NULL */
  const float *bias_o;              /* [d] or NULL              */
  tern_gate_mode gate;
  float eps;
  tern_norm_mode norm;              /* of both BitLinears' inputs (0: RMSNorm) */
  /* Prefill scan over time ("parallel scan"; reading C23): 1 = the exact sequential
   * recurrence (bit-identical to the definition); 4 = the chunked scan: each channel's
   * sequence is cut into 4 contiguous chunks [j T/4, (j+1) T/4) scanned concurrently
   * from their composed boundary states (chunk aggregates A = prod f, B = the recurrence
   * from 0, composed in order) -- equal to the oracle's 4-slice composition
   * (O.scan_slices(4)) and within reading S4's tolerance of the sequential scan; 8 = the
   * same with 8 chunks (O.scan_slices(8)).  With d % 32 == 0 and ceil(T / chunks) <= 512
   * the chunks of a 32-channel group run on the CTAs of one thread-block cluster, handing
   * the boundary state on through distributed shared memory; otherwise 4 runs on one CTA
   * per 8 channels (d % 8 == 0) and 8 falls back to the exact scan.  0 = auto, currently 1
   * (DESIGN.md §6 has the measured comparison).  Other values: TERN_ERR_UNSUPPORTED.
   * tern_mlgru_chunks() reports the resolved value. */
  int32_t num_chunks;
} tern_mlgru;

/* The scan chunk count mlgru_fwd / block_prefill will use for B sequences of T tokens
 * (host helper; resolves num_chunks = 0). */
int32_t tern_mlgru_chunks(const tern_mlgru* p, int32_t B, int32_t T, int32_t d);

typedef struct {
  tern_weight gu, down;
  const float *gain_x, *gain_p;     /* [d], [l] */
  float eps;
  tern_norm_mode norm;              /* of both BitLinears' inputs (0: RMSNorm) */
} tern_glu;

/* Output-feature sharding of a block over `world` ranks (BASELINE.json
 * configs[3,4]).  Rank r holds the rows of every
 * BitLinear for its channel slice: f, c, g, o and down rows [r*ds, (r+1)*ds)
 * with ds = d/world, gate and up rows [r*ls, (r+1)*ls) with ls = l/world, each
 * packed with the FULL matrix's mean|W| scale (tern_pack's scale_in).  Its
 * state h is [B][ds].  Before every BitLinear the input row is gathered whole
 * (the row norm and the contraction need all K), so each block calls `ag`
 * four times on `stream`: o', x1, p and y.  ag(ctx, send, recv,
 * bytes_per_rank, stream) must place the world equal chunks, in rank order,
 * at recv (a torch.distributed / NCCL all-gather into a tensor) and return 0;
 * it is called from inside block_prefill / block_decode (also during CUDA
 * graph capture).  Outputs are bit-identical to world = 1: gathers move
 * values unchanged, int32 sums are exact and every norm sees the full row.
 * Requires ds % 64 == 0 and ls % 16 == 0.  world <= 1: no sharding. */
typedef int (*tern_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes_per_rank,
                                 tern_stream stream);
/* Sum of `count` int32 over the ranks into recv (recv may equal send), on
 * `stream`; 0 = ok (a torch.distributed / NCCL all_reduce).  Exact. */
typedef int (*tern_allreduce_fn)(void* ctx, const int32_t* send, int32_t* recv, size_t count,
                                 tern_stream stream);
typedef struct {
  int32_t rank, world;
  tern_allgather_fn ag;
  void* ctx;
  /* 1 = on the tensor-core path (B*T > gemv_max_m) the o',
   * x1 and p gathers move int8 codes instead of activations: each rank sends
   * binary64 partials of the row moments (one small gather per round: 1 for
   * RMSNorm, 2 centred, +1 with a gain), every rank combines them in rank
   * order, quantizes its own slice and the codes (+ int32 partial q-sums) are
   * gathered -- 2x (bf16) / 4x (fp32) fewer bytes.  The summation order of the
   * moments differs from world = 1, so results equal the oracle (and world = 1)
   * except in the rare fp64-boundary cases of reading C4.  The block output y
   * is still gathered whole.  0 (default): gather activations. */
  int32_t gather_q;
  /* SURVEY 8(f) f1(ii), Megatron pairing: 1 = f|c|g and gate|up stay
   * column-parallel (output rows [r*ds..), [r*ls..) as above) but W_o and
   * W_down are ROW-parallel: rank r holds their input columns [r*ds, (r+1)*ds)
   * and [r*ls, (r+1)*ls) for all d outputs (tern_weight k = ds / ls, n_out =
   * d, packed with the full matrix's scale).  Each of o' and p then stays a
   * local slice: its row moments are exchanged (as with gather_q), every rank
   * quantizes its slice, multiplies it by its weight columns into int32
   * partials of all d outputs, and `ar` sums them exactly -- 2 collectives of
   * activations per block instead of 4, and x1 / y come out whole on every
   * rank.  Requires ar; always the tensor-core path. */
  int32_t megatron;
  tern_allreduce_fn ar;
} tern_shard;

typedef struct {
  tern_mlgru mix;
  tern_glu ch;
  int32_t d, l;       /* full widths (also when sharded) */
  tern_shard shard;   /* zero-initialise for an unsharded block */
  /* optional (may be NULL): the tern_block decoded right after this one.  The
   * decode GEMVs then prefetch its f|c|g and o weights into L2 while this
   * block's channel mixer runs (each GEMV also prefetches the weights two
   * launches ahead inside the block), so HBM-resident stacks stream weights
   * ahead of the dependency chain.  A hint only: results do not change. */
  const void* next_block;
} tern_block;

/* Workspace bytes for mlgru_fwd / glu_fwd / block_* on B sequences x T tokens. */
size_t tern_mlgru_workspace(const tern_mlgru* p, int32_t B, int32_t T, int32_t d, tern_dtype dt);
size_t tern_glu_workspace(const tern_glu* p, int32_t m, int32_t d, int32_t l, tern_dtype dt);
size_t tern_block_workspace(const tern_block* b, int32_t B, int32_t T, tern_dtype dt);

/* Byte offsets of the block's intermediates inside its workspace, valid after
 * block_prefill / block_decode returns on the stream (parity taps):
 *   fcg [B*T][3d], oprime [B*T][d], x1 [B*T][d], p [B*T][l], all dtype dt
 *   (sharded blocks: fcg of the rank's channels; oprime, x1, p gathered whole).
 *   fp32 prefill with more than 256 tokens writes x1 into y instead and adds the channel
 *   mixer onto it in place (TMA reduce-add), so the x1 tap is not written there. */
typedef struct {
  size_t fcg, oprime, x1, p;
} tern_block_taps;
tern_status tern_block_ws_layout(const tern_block* b, int32_t B, int32_t T, tern_dtype dt,
                                 tern_block_taps* out /* host */);

/* MLGRU token mixer: out = o_t for x [B][T][d] (no residual). */
tern_status mlgru_fwd(const tern_mlgru* p, const void* x, void* out, tern_dtype dt, int32_t B,
                      int32_t T, int32_t d, float* h, void* ws, size_t ws_bytes,
                      tern_stream stream);

/* GLU channel mixer: out = d_t for x [m][d] (no residual). */
tern_status glu_fwd(const tern_glu* p, const void* x, void* out, tern_dtype dt, int32_t m,
                    int32_t d, int32_t l, void* ws, size_t ws_bytes, tern_stream stream);

/* a8: block prefill, x1 = x + MLGRU(x), y = x1 + GLU(x1) (C9), over
 * B sequences of T tokens starting from state h (0 at a fresh prefill,
 * P:456); h holds h_T afterwards.  bf16 rounds x1 and y (R3). */
tern_status block_prefill(const tern_block* b, const void* x, void* y, tern_dtype dt, int32_t B,
                          int32_t T, float* h, void* ws, size_t ws_bytes, tern_stream stream);

/* a8/a9: one decode step (T = 1) continuing state h. B <= gemv_max_m runs
 * four GEMV launches (norm+quant fused into each prologue, the MLGRU step
 * and SwiGLU fused into epilogues); larger B runs the prefill path with T=1. */
tern_status block_decode(const tern_block* b, const void* x, void* y, tern_dtype dt, int32_t B,
                         float* h, void* ws, size_t ws_bytes, tern_stream stream);

/* a9 + SURVEY 8(f) f2: one decode step (T = 1) through a whole stack of L
 * blocks in ONE persistent launch: x [B][d] -> y [B][d], states h[i] ([B][d]
 * fp32, device) of block i continued in place ("fall-through
 * mode").  Same arithmetic as L block_decode calls chained through their
 * outputs, bit for bit; the 4L dependent BitLinear phases are separated by
 * grid-wide barriers in one cooperative kernel (one CTA per SM) instead of
 * kernel launches, and each phase's weight slice is copied into shared memory
 * while the previous phase runs.
 *   blocks: host array of L unsharded blocks with equal d and l (next_block is
 *           ignored); h: host array of L device pointers; x, y device, y != x.
 *   ws: tern_stack_decode_workspace bytes (device, 16-byte aligned), owned by
 *       the caller; concurrent calls need disjoint ws.
 * Returns TERN_ERR_UNSUPPORTED (no side effects) when B > 4, a block is
 * sharded, d or l exceed the decode GEMV register tile, or a phase's weight
 * slice does not fit shared memory: use block_decode then.  B == 0 is a no-op.
 * CUDA-graph capturable (a 4-byte memset + one kernel per 32 blocks). */
size_t tern_stack_decode_workspace(const tern_block* blocks, int32_t L, int32_t B, tern_dtype dt);
tern_status stack_decode(const tern_block* blocks, int32_t L, const void* x, void* y,
                         tern_dtype dt, int32_t B, float* const* h, void* ws, size_t ws_bytes,
                         tern_stream stream);

/* ------------------------------------------------------------------------
 * Alg. 1 BackwardPass of one BitLinear
 * with the straight-through estimator; readings B1-B6:
 *   dY = dO x W~^T        W~ = t * scale, the ternary weight the forward used (B1)
 *   dX = rms_norm_bwd(dY, X, mu, sigma^2, r)                      (B4, B5)
 *        dsig = sum_j dY_j (x_j - mu) (-1/2) r^3
 *        dmu  = sum_j (-r dY_j) + dsig * mean(x - mu)   (norm = TERN_NORM_CENTERED only;
 *               TERN_NORM_RMS has mu = 0 and no dmu term)
 *        dX_j = r dY_j + 2 dsig (x_j - mu) / k + dmu / k
 *   dW = dO^T x Y~        Y~ = q * deq, the forward's quantized activation (B2)
 *   db = sum over the m tokens of dO
 * mu, r, q, deq are the forward's (recomputed from x with the forward's own quantizer,
 * B3); no gain (Alg. 1 has none).  Arguments (device pointers, caller-owned):
 *   x  [m][k] of dt (fp32, or bf16 widened exactly -- the bf16 configs; bf16 needs the
 *   tensor-core path), row-major, the forward input;  w: one segment (n_seg = 1) with its
 *   u8 copy e8 (tern_expand);  dO [m][n_out] of dt;  outputs fp32 dX [m][k], dW [n_out][k] (the
 *   latent weight's layout), db [n_out] (NULL = skip), all fp32;  ws >=
 *   bitlinear_bwd_workspace(m, k, n_out) bytes, 16-byte aligned.  m == 0 writes dW = 0
 *   and db = 0.  Deterministic sums (no atomics).
 * Errors: TERN_ERR_INVALID_ARG (null pointers, k % 16 != 0, n_seg != 1, no e8, small
 * ws, bad norm), all checked before any launch; asynchronous faults as elsewhere. */
size_t bitlinear_bwd_workspace(int32_t m, int32_t k, int32_t n_out);
/* 1 (default): the backward's two contractions on the tensor cores (bf16 hi + lo split of
 * the fp32 operand, reading B7); 0: fp32 CUDA-core GEMMs (the reference path). */
void tern_set_bwd_tc(int32_t on);
int32_t tern_get_bwd_tc(void);
tern_status bitlinear_bwd(const void* x, tern_dtype dt, int32_t m, int32_t k, const tern_weight* w,
                          float eps, int32_t norm, const void* dO, float* dX, float* dW, float* db,
                          void* ws, size_t ws_bytes, tern_stream stream);

/* ------------------------------------------------------------------------
 * Measurement hooks (bench.py roofline): while enabled, every kernel launch
 * made by this library on a non-capturing stream is bracketed by two CUDA
 * events recorded on that same stream, with its shape.  tern_profile_collect
 * synchronises those events, copies up to `max` records into `out` (host
 * array; NULL just counts) and returns the number of records; records are
 * kept until the next tern_profile_enable(1).  Not for use in production.
 * ------------------------------------------------------------------------ */
typedef enum { TERN_K_QUANT = 0, TERN_K_GEMV = 1, TERN_K_GEMM = 2, TERN_K_SCAN = 3,
               TERN_K_FCGSCAN = 4, TERN_K_STACK = 5, TERN_K_FIN = 6,
               TERN_K_GEMM_QF = 7 /* GEMM with the a2 quantization of its A fused in */
             } tern_kernel_id;
typedef struct {
  int32_t kernel;   /* tern_kernel_id                                        */
  int32_t epi;      /* epilogue kind (GEMV/GEMM) or gate mode (scan)         */
  int32_t m;        /* rows (tokens); scan: B*T                              */
  int32_t n;        /* GEMV/GEMM: packed weight rows; scan: d; quant: 0;
                       stack: blocks                                          */
  int32_t k;        /* input features                                        */
  int32_t n_seg;    /* weight segments                                       */
  int32_t dtype;    /* activation dtype (tern_dtype)                         */
  float ms;         /* elapsed device time between the two events            */
} tern_prof_rec;
void tern_profile_enable(int32_t on);
int32_t tern_profile_collect(tern_prof_rec* out, int32_t max);

/* Device-side timeline of kernel launches (debug; works inside CUDA graphs):
 * while enabled, each launch made on the host gets a trace slot (up to 1024
 * launches, then the slots wrap) in which thread 0 of every CTA (the first
 * 1024) records the %globaltimer (ns) at its start, when its dependency wait
 * (griddepcontrol.wait / grid barrier) released, and at its end; decode GEMV
 * CTAs add their SM id, clocks and intermediate phase marks.
 * tern_trace_collect synchronises the device and copies up to max_launches
 * records to out (host), each 1 + 1024*16 uint64: [0] = CTA count | (kernel
 * << 20) (tern_kernel_id; the split-K epilogue is TERN_K_GEMM + 16), then per
 * CTA {start, released, end, ...}; returns the number of launches recorded
 * (out == NULL just counts).  Replaying a captured graph overwrites the slots
 * assigned at capture time.  Only the decode GEMV records in the default
 * build; the other kernels' marks are compiled into the debug variant
 * libtern_trace.so (build.py --trace). */
void tern_trace_enable(int32_t on);
int32_t tern_trace_collect(uint64_t* out, int32_t max_launches);

/* ------------------------------------------------------------------------
 * Sequence-parallel prefill (the long-context variant; reading
 * C23 in DESIGN.md).  The T tokens of every sequence are cut into `world`
 * contiguous slices [r T/world, (r+1) T/world); rank r runs
 * block_prefill_sp on its slice x [B][T_local][d] with the state h [B][d]
 * the whole sequence starts from (identical on every rank).  Per block, the
 * MLGRU scan exchanges ONE all-gather of 2 B d floats per rank -- the slice
 * aggregates (A = prod f, B = the recurrence from 0, composed left to right,
 * S:197) -- each rank composes the earlier ranks' aggregates in rank order into
 * its boundary state, scans its slice exactly from it, and h leaves holding
 * the state after the WHOLE sequence (the composition through every slice,
 * the same on all ranks).  Everything else in the block is token-local.  The
 * result equals the oracle's W-slice scan (O.scan_slices) bit for bit; with
 * world = 1 it equals block_prefill.  T_local may be 0 (a rank with no
 * tokens still joins the exchange; x, y may then be NULL).  The block must
 * not be output-sharded.  ag is called once per block on `stream`.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t rank, world;
  tern_allgather_fn ag;
  void* ctx;
} tern_seqpar;
size_t tern_block_prefill_sp_workspace(const tern_block* b, int32_t B, int32_t T_local,
                                       tern_dtype dt, int32_t world);
tern_status block_prefill_sp(const tern_block* b, const void* x, void* y, tern_dtype dt,
                             int32_t B, int32_t T_local, float* h, const tern_seqpar* sp,
                             void* ws, size_t ws_bytes, tern_stream stream);

/* ------------------------------------------------------------------------
 * Fixed-point W8A16 numerics of the paper's Loihi 2 deployment (SURVEY 8(f)
 * f4(ii); readings F1-F5 in DESIGN.md §3b).
 * Integers in, integers out, a value v with exponent e meaning v * 2^e.
 * Asynchronous on `stream` unless stated; device pointers unless stated.
 * ------------------------------------------------------------------------ */
/* F1: norm gains w [n] (fp32) -> wq [n] (int8) and the exponent e
 * (written to *e_host) with w ~ wq 2^e, 2^e = 2^(round(log2 max|w|) - shift),
 * round half away; shift 0 is the printed formula (|wq| <= 1), shift 6 uses
 * the int8 range (|wq| <= 91).  0 <= shift <= 6.  ws: device scratch >= 16
 * bytes, 16-byte aligned.  Synchronous (an offline weight-preparation step);
 * TERN_ERR_DEGENERATE if max|w| is 0 or not finite (wq then untouched). */
tern_status tern_fxp_scales(const float* w, int32_t n, int32_t shift, int8_t* wq, int32_t* e_host,
                            void* ws, tern_stream stream);
/* F2: dynamic 16-bit activation quantization of x [n] (fp32 or bf16,
 * finite) with ONE power-of-two exponent for the tensor: *e (device int32) =
 * the smallest e with round(max|x| / 2^e) <= 32767, q = round(x / 2^e) (half
 * away) int16 [n].  An all-zero x gives e = 0.  ws: device scratch >= 16
 * bytes, 16-byte aligned (the max).  n == 0: no-op. */
tern_status tern_fxp_quant_act(const void* x, tern_dtype dt, int64_t n, int16_t* q, int32_t* e,
                               void* ws, tern_stream stream);
/* F3: LUT sigmoid, x [n] int32 in Q6 (x_exp = 6) -> y [n] int32
 * in Q15 (y_exp = 15): 9 points x = 0..8 holding floor(sigma(i) 2^15), linear
 * interpolation with a floor, |x| >= 8 -> the last point, sigma(-x) = 2^15 -
 * sigma(x).  x, y 16-byte aligned. */
tern_status tern_fxp_sigmoid(const int32_t* x, int64_t n, int32_t* y, tern_stream stream);
/* F4: 1/sqrt(v 2^e) ~ y 2^ey for v [n] (uint64, > 0) and e [n]
 * (int32): 24-entry seed table over [1, 4) + five Newton steps in Q30.
 * y [n] uint32 (Q30 mantissa in (2^29, 2^30]), ey [n] int32.  v == 0 is
 * outside the domain and gives y = 0, ey = 0.  v 8-byte aligned. */
tern_status tern_fxp_inv_sqrt(const uint64_t* v, const int32_t* e, int64_t n, uint32_t* y,
                              int32_t* ey, tern_stream stream);
/* F5 (Eq. 1; eps = 1e-3 P:510): RMSNorm of int16 rows xq
 * [rows][d] with exponent *ex (device int32, e.g. from tern_fxp_quant_act)
 * and int8 gains wq [d] with exponent ew (host, from tern_fxp_scales):
 * out [rows][d] int16 and eo [rows] int32 (one exponent per row, the
 * smallest that fits).  Integer sum of squares, eps on its grid
 * (round(d eps 2^(-2 ex)), clamped to 2^60), F4 for the inverse square root,
 * sqrt(d) in Q16.  1 <= d <= 65536; xq 16-byte aligned. */
tern_status tern_fxp_rmsnorm(const int16_t* xq, const int32_t* ex, const int8_t* wq, int32_t ew,
                             double eps, int32_t rows, int32_t d, int16_t* out, int32_t* eo,
                             tern_stream stream);

/* F6: a BitLinear in W8A16.  xq [m][k] int16 with exponent *ex
 * (device int32), norm gains gq [k] int8 with exponent eg (host), eps (1e-3):
 *   (yn, en) = tern_fxp_rmsnorm(xq)            (per-row exponents en)
 *   acc[r][n] = sum_k t[n][k] yn[r][k]          (exact; on the int8 tensor
 *     cores as 256 (W hi) + (W lo') + 128 sum_k t[n][k], hi = yn >> 8,
 *     lo' = (yn & 255) - 128, both s8: one GEMM over 2m + 1 operand rows,
 *     the last a row of ones)
 *   (bq, eb) = F1(w->scales[0], shift 6);  y = round(acc bq / 2^s) int16
 *   with the smallest fitting s per row, ey[r] = s + en[r] + eb.
 * w: n_seg == 1, w->k == k <= 65535.  y [m][ldy] int16, ldy >= n_out; ey [m].
 * xq and ws 16-byte aligned; ws_bytes >= tern_fxp_bitlinear_workspace(m, k,
 * w->n_rows).  m == 0: no-op. */
size_t tern_fxp_bitlinear_workspace(int32_t m, int32_t k, int32_t n_rows);
tern_status tern_fxp_bitlinear(const int16_t* xq, const int32_t* ex, int32_t m, int32_t k,
                               const int8_t* gq, int32_t eg, double eps, const tern_weight* w,
                               int16_t* y, int32_t ldy, int32_t* ey, void* ws, size_t ws_bytes,
                               tern_stream stream);

/* Device self-check of the numerics shortcuts the kernels take (test use):
 * which = 0: the FMA-corrected reciprocals used by the sigmoids equal IEEE
 * 1/d for every mantissa of every exponent 0..125 (d in [1, 2^126));
 * which = 1: sigmoid equals 1/(1+exp_c(-x)) with IEEE division at 2^24
 * points in [-96, 96);
 * which = 2: the paired vector sigmoid of the scan / SwiGLU epilogue equals
 * the same except that results below 2^-126 may be 0;
 * which = 3: the conversion-free round half away from zero used by every
 * quantizer (and its integer extraction) equals the reference for every
 * float with |v| < 2^22;
 * which = 4: the round-toward-zero form of it (k_quant's) equals the same. 
 * Synchronous; writes the mismatch count to *mismatches (host).  ws: device
 * scratch of >= 64 bytes. */
tern_status tern_selftest(int32_t which, void* ws, uint64_t* mismatches);

/* Norm variant used by tern_quant and bitlinear_fwd (process-wide, host;
 * default TERN_NORM_RMS).  Mixers and blocks take theirs from tern_mlgru.norm
 * and tern_glu.norm.  Not thread-safe to change while calls are in flight. */
void tern_set_norm_mode(tern_norm_mode mode);
tern_norm_mode tern_get_norm_mode(void);

/* Tuning knob (host): largest m sent to the decode GEMV (default 4, max 4;
 * 0 forces the tensor-core path everywhere).  Not thread-safe to change
 * while calls are in flight. */
void tern_set_gemv_max_m(int32_t m);
/* Tuning knob (host): how prefill runs the f|c|g BitLinear and the MLGRU scan.
 * 2 always as one fused kernel (k_fcgscan; needs the e8 weight copy and
 * d % 64 == 0); 0 never: GEMM + tern_mlgru_scan (then the f^c^g^ tap of
 * tern_block_ws_layout is written); 1 (default) fused when its 64-channel
 * chains fill at least two thirds of the SMs (3*B*d/64 >= 2*#SMs), else
 * unfused, whose scan spreads 8 channels per CTA.  Results are identical.  Values outside
 * 0..2 are clamped. */
void tern_set_fused_scan(int32_t mode);
int32_t tern_get_fused_scan(void);
int32_t tern_get_gemv_max_m(void);
/* Tuning knob (host): 1 runs decode steps with gemv_max_m < B <= 256 as, per
 * BitLinear, a split-K GEMM writing int32 partials plus one row-wise finalize
 * that applies the epilogue and quantizes the row for the next BitLinear
 * (9 launches per block); 0 (default, measured faster on c3) runs quant +
 * GEMM + epilogue per BitLinear.  Results are identical. */
void tern_set_batched_fin(int32_t on);
int32_t tern_get_batched_fin(void);
/* Tuning knob (host): 1 runs the contraction of 4 < M <= 256 token calls that have a
 * split-K workspace (decode batches) with the swap-AB kernel (weights as the MMA's
 * 128-row operand, streamed as 2-bit codes and unpacked in shared memory; tokens as N);
 * 0 (default, measured faster on c3 B = 64 and c4 B = 128) with the u8-tile GEMM.
 * Results are identical (integer sums).  Initial value: env TERN_GEMM_SAB, else 0. */
void tern_set_gemm_sab(int32_t on);
int32_t tern_get_gemm_sab(void);
/* Tuning knob (host): 1 (default) runs large-M GEMMs with the u8 weight copy and K >= 2048
 * on CTA pairs (tcgen05.mma.cta_group::2, 256 x 256 tiles, k_gemm_2sm); 0 always on single
 * CTAs (128 x 256 tiles).  Results are identical.  Initial value: env TERN_GEMM_2SM, else 1. */
void tern_set_gemm_2sm(int32_t on);
int32_t tern_get_gemm_2sm(void);
/* Tuning knob (host): 1 fuses the RMSNorm + int8 quantization (a2) of the
 * o, gate|up and down BitLinears' inputs into their prefill GEMMs (block_prefill, mlgru_fwd,
 * glu_fwd with M > 256 tokens): the GEMM's warps 2-5 quantize rows in order and publish
 * 128-row blocks through counters in the block workspace, the TMA producer waits for a
 * block before loading it; no standalone quant launch.  Bit-identical results; default 0
 * (measured slower than quant + GEMM on B200: DESIGN.md section 6). */
void tern_set_qfuse(int32_t on);
int32_t tern_get_qfuse(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* TERN_H */
