// internal.h -- launch interfaces between the C ABI (api.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tern.h"

namespace tern {

constexpr int kSegRows = 64;  // interleave group of fused weight segments
constexpr int kKAlign = 128;  // K padding of packed rows / quantized activations

// Epilogue applied to int32 accumulators (shared by the GEMV and the GEMM).
enum EpiKind : int {
  EPI_STORE = 0,   // y[m][r] = R1(dequant + bias)                      (n_seg == 1)
  EPI_RESID = 1,   // y[m][r] = R3(res[m][r] + R1(dequant + bias))       (n_seg == 1)
  EPI_FCG = 2,     // y[m][packed row] = R1(dequant + bias)  (interleaved pre-activations)
  EPI_MLGRU = 3,   // decode: f,c,g -> h update -> o'[m][r]              (n_seg == 3, GEMV)
  EPI_SWIGLU = 4,  // p[m][r] = R2(SiLU(R1 g) * R1 u)                    (n_seg == 2)
  EPI_NONE = 5,    // accumulators only (tap)
  EPI_RESID_RED = 6  // fp32: y[m][r] += R1(dequant + bias) in place (y holds the residual;
                     // TMA reduce-add in the tensor-core GEMMs, one IEEE fp32 add = EPI_RESID's)
};

struct Epi {
  int kind;
  int n_out, n_seg;
  const float* scales;   // [n_seg] mean|W|
  const float* bias;     // [n_seg*n_out] or null
  void* out;             // output activations (dtype of the kernel)
  int ldo;
  const void* res;       // residual input, same dtype as out
  int ldr;
  float* h;              // MLGRU state [M][n_out] fp32
  int gate;              // tern_gate_mode
  int32_t* acc;          // optional int32 accumulator tap [M][ldacc] (packed rows)
  int ldacc;
};

struct QuantTaps {
  int8_t* q;
  int ldq;
  float* deq;
  float* inv_rms;
  float* absmax;
};

// host: 2-D TMA descriptor (inner = contiguous dim), 128-B L2 promotion (k_gemm.cu)
bool make_map_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                 uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                 CUtensorMapSwizzle swz);

// a1
cudaError_t launch_codes_init(uint32_t* codes, int n_rows, int ldw, cudaStream_t s);
cudaError_t launch_absmean(const float* W, int64_t numel, const float* scale_in, float* scale_out,
                           double* ws, cudaStream_t s);
cudaError_t launch_pack_codes(const float* W, int n, int k, int n_seg, int seg, uint32_t* codes,
                              int n_rows, const float* scale, cudaStream_t s);
size_t pack_workspace_bytes();
// a2
cudaError_t launch_quant(const void* x, int xdt, int m, int k, int ldx, const float* gain,
                         float eps, int8_t* q, int ldq, float* deq, int32_t* qsum, float* inv_rms,
                         float* absmax, cudaStream_t s, int norm = TERN_NORM_RMS,
                         uint32_t* zero = nullptr, int nzero = 0);
// a2 fused into the consuming GEMM (f3; k_gemm.cu "fused quantization"): the GEMM's idle
// warps 2-5 run the RMSNorm + absmax quantization of x row by row (rows taken
// in a static order), publishing each finished 128-row block in ctr[1 + block]; the TMA
// producer waits for a block before loading its A tiles.  ctr must be zero at launch
// ([1 + ceil(M/128)] words; block_ws region qf, zeroed ahead of the block's first quant launch).
struct QFuse {
  const void* x;
  int ldx;
  const float* gain;   // NULL = ones
  float eps;
  uint32_t* ctr;
};
extern int g_qfuse_on;   // tern_set_qfuse
constexpr int kQfAreas = 3;   // o, gate|up, down (one counter area per fused GEMM of a block)
inline int qf_words(int M) { return 1 + (M + 127) / 128; }
// a3 (decode GEMV, norm+quant prologue fused): x [M][ldx] -> epilogue
constexpr int kGemvMaxM = 4;
bool gemv_supported(int M, int K, int xdt);   // M <= kGemvMaxM and K within the register tile
// pf / pf_bytes: optional L2 prefetch of a later launch's packed weights
cudaError_t launch_gemv(const void* x, int xdt, int ydt, int M, int K, int ldx, const float* gain,
                        float eps, const tern_weight& w, const Epi& epi, const QuantTaps* taps,
                        cudaStream_t s, const void* pf = nullptr, size_t pf_bytes = 0,
                        int norm = TERN_NORM_RMS);
// swap-AB tcgen05 contraction for decode batches (k_gemm_sab.cu): int32 partials
// part[ks][M][n_rows] from the 2-bit codes; *ks_out = slices used
bool gemm_sab_supported(int M);
extern int g_gemm_sab;   // tern_set_gemm_sab
extern int g_gemm_2sm;   // tern_set_gemm_2sm
cudaError_t launch_gemm_sab(const int8_t* q, int M, int ldq, const tern_weight& w, int32_t* part,
                            size_t part_bytes, int ks_max, int* ks_out, cudaStream_t s);
cudaError_t launch_splitk_epi(const int32_t* part, int ks, int M, int n_rows, const float* deq,
                              const int32_t* qsum, const Epi& e, int ydt, cudaStream_t s);
// a4 (tcgen05 int8 GEMM): q [M][ldq] -> epilogue
// part: optional int32 scratch [M][n_rows] enabling split-K for small M (nullptr: never);
// with part, decode batches (M <= 256) take the swap-AB kernel above
// ks_out: partials only (part required): the K-slice count is returned and no
// epilogue runs (launch_fin finalizes); *ks_out > 0 on entry caps the count
cudaError_t launch_gemm(const int8_t* q, int M, int ldq, const float* deq, const int32_t* qsum,
                        const tern_weight& w, int ydt, const Epi& epi, cudaStream_t s,
                        int32_t* part = nullptr, size_t part_bytes = 0, int* ks_out = nullptr,
                        const QFuse* qf = nullptr);
// f4(iii) Alg. 1 backward (k_bwd.cu); g_bwd_tc: tensor-core contractions (tern_set_bwd_tc)
extern int g_bwd_tc;
size_t bwd_workspace(int m, int k, int n);
cudaError_t launch_bitlinear_bwd(const void* x, int dt, int m, int k, const tern_weight& w,
                                 float eps, int norm, const void* dO, float* dX, float* dW,
                                 float* db, void* ws, cudaStream_t s);
// whether launch_gemm runs a QFuse request inside the GEMM (else it launches k_quant first)
bool gemm_qfuse_ok(int M, const tern_weight& w, const Epi& epi, int32_t* part, size_t part_bytes);
// batched decode: one CTA per row sums the ks partial slices [ks][M][n_rows],
// applies e (MLGRU / SWIGLU / RESID / STORE) and, when nq is set, the next
// BitLinear's RMSNorm + int8 quant of the stored output row (gain ngain, eps
// neps) into nq [M][nldq], ndeq, nqsum (which may alias deq / qsum)
bool fin_supported(int n_out);
cudaError_t launch_fin(const int32_t* part, int ks, int M, int n_rows, const float* deq,
                       const int32_t* qsum, const Epi& e, int ydt, const float* ngain, float neps,
                       int8_t* nq, int nldq, float* ndeq, int32_t* nqsum, cudaStream_t s,
                       int nnorm = TERN_NORM_RMS);
// f2: whole-stack decode step in one persistent cooperative launch.  A phase
// is one decode BitLinear with its epilogue (MLGRU / SWIGLU / RESID / STORE),
// contiguous rows (ld = K for x, n_out for out/res/h).
struct StackPhaseDesc {
  const void* x;
  const void* res;
  void* out;
  float* h;
  tern_weight w;
  const float* gain;
  const float* bias;
  float eps;
  int kind, gate, K, norm;
};
bool stack_decode_plan(const StackPhaseDesc* ph, int n, int M, int xdt, size_t* smem);
// bar: one zeroed-per-launch u32 grid-barrier counter (device); returns
// cudaErrorNotSupported when the plan does not fit (stack_decode_plan false)
cudaError_t launch_stack_decode(const StackPhaseDesc* ph, int n, int M, int xdt, unsigned* bar,
                                cudaStream_t s);
// debug timeline (globaltimer per CTA, tern_trace_enable): a slot for one launch
// of `ctas` CTAs of kernel `kind` (tern_kernel_id), or nullptr when tracing is off
unsigned long long* trace_slot(int kind, int ctas);
// debug timeline of GEMV launches (globaltimer per CTA), see tern_trace_enable
void gemv_trace_enable(int on);
int gemv_trace_collect(unsigned long long* out, int max_launches);
cudaError_t launch_selftest(int which, unsigned long long* bad, int* exps, int n_exp,
                            cudaStream_t s);
cudaError_t launch_expand(const tern_weight& w, uint8_t* e8, cudaStream_t s);
// sharding: full[m][r*cs + j] = gathered[r][m][j]
cudaError_t launch_unshard(const void* gathered, int dt, int world, int M, int cs, void* full,
                           cudaStream_t s);
// f1(i): sharded BitLinear input gathered as int8 codes (k_shard.cu).  st: the
// gathered stat rounds so far ([world][M][2] doubles each, null if absent)
int slice_rounds(int norm, bool gain);
cudaError_t launch_slice_stats(const void* x, int ldx, int M, int cs, int world, int rank, int dt,
                               const float* gain, float eps, int norm, const double* const* st,
                               int rnd, double* out, cudaStream_t s);
cudaError_t launch_slice_quant(const void* x, int ldx, int M, int cs, int world, int rank, int dt,
                               const float* gain, float eps, int norm, const double* const* st,
                               int8_t* q, int ldq, int32_t* qs_out, float* deq, cudaStream_t s);
// (launch_splitk_epi, above: the split-K epilogue on its own -- sums ks int32 slices
// part[ks][M][n_rows] and applies e; also f1(ii), after the all-reduce of a row-parallel
// GEMM's partials)
cudaError_t launch_unshard_q(const int8_t* gathered, int world, int M, int cs, int8_t* q, int ldq,
                             int32_t* qsum, cudaStream_t s);
// a4 + a6 fused (prefill): f|c|g GEMM with the MLGRU scan in its epilogue
bool fcgscan_supported(const tern_weight& w, int d);
cudaError_t launch_fcgscan(const int8_t* q, int ldq, const float* deq, const int32_t* qsum,
                           const tern_weight& w, const float* bias, int dt, int B, int T, int d,
                           int gate, float* h, void* oprime, cudaStream_t s);
// a6
bool fcgscan_preferred(int B, int d);
// sequence-parallel scan (C23): slice aggregates, boundary-state composition
cudaError_t launch_scan_agg(const void* fcg, int dt, int B, int T, int d, float* agg,
                            cudaStream_t s);
cudaError_t launch_sp_compose(const float* recv, int world, int rank, int64_t n, float* h,
                              float* hfin, cudaStream_t s);
cudaError_t launch_fill_f32(float* p, size_t n, float v, cudaStream_t s);
// k_fxp.cu: fixed-point W8A16 numerics (f4(ii))
cudaError_t launch_fxp_scales(const float* w, int n, int shift, int8_t* wq, int32_t* e,
                              int32_t* status, cudaStream_t s);
cudaError_t launch_fxp_quant_act(const void* x, int dt, int64_t n, int16_t* q, int32_t* e,
                                 uint32_t* ws, cudaStream_t s);
cudaError_t launch_fxp_sigmoid(const int32_t* x, int64_t n, int32_t* y, cudaStream_t s);
cudaError_t launch_fxp_inv_sqrt(const uint64_t* v, const int32_t* e, int64_t n, uint32_t* y,
                                int32_t* ey, cudaStream_t s);
cudaError_t launch_fxp_split(const int16_t* a, int m, int k, int ldq, int8_t* hi, int8_t* lo,
                             int32_t* qs_hi, int32_t* qs_lo, int8_t* ones, int32_t* qs_ones,
                             cudaStream_t s);
cudaError_t launch_fxp_combine(const int32_t* acc_hi, const int32_t* acc_lo, int ldacc,
                               const int32_t* rowsum, const float* scale, int n, int m,
                               const int32_t* en, int16_t* y, int ldy, int32_t* ey,
                               cudaStream_t s);
cudaError_t launch_fxp_rmsnorm(const int16_t* xq, const int32_t* ex, const int8_t* wq, int ew,
                               double eps, int rows, int d, int16_t* out, int32_t* eo,
                               cudaStream_t s);
// chunked prefill scan (tern_mlgru.num_chunks, reading C23): resolve 0 = auto to 1 or 4
int scan_chunks_resolve(int num_chunks, int B, int T, int d);
cudaError_t launch_scan_chunks(const void* fcg, int dt, int B, int T, int d, int gate, float* h,
                               void* oprime, int chunks, cudaStream_t s);
cudaError_t launch_scan(const void* fcg, int dt, int B, int T, int d, int gate, float* h,
                        void* oprime, cudaStream_t s);

}  // namespace tern
