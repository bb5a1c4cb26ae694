// api.cu -- the C ABI of libtern.so (include/tern.h): argument validation,
// workspace carve-up and the launch sequences of the block (DESIGN.md
// "Boundary").  Every check runs before the first launch, so a failing call
// has no side effects.  No allocation, no host sync (except tern_pack).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace tern;

namespace {

thread_local std::string g_err;
int g_gemv_max_m = kGemvMaxM;
int g_fused_scan = 1;
int g_batched_fin = 0;   // tern_set_batched_fin
// fp32 block prefill: x1 is written into y and the channel mixer's down projection is added
// onto it in place (EPI_RESID_RED, TMA reduce-add) -- no residual tile loads in its drain
int g_resid_red = getenv("TERN_RESID_RED") ? (atoi(getenv("TERN_RESID_RED")) != 0) : 1;
int g_norm_mode = TERN_NORM_RMS;   // tern_set_norm_mode (tern_quant, bitlinear_fwd)
constexpr int kSplitKMaxM = 256;

tern_status fail(tern_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

tern_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return TERN_OK;
  return fail(TERN_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define TRY_CUDA(expr, where)                              \
  do {                                                     \
    tern_status _st = cuda_status((expr), (where));        \
    if (_st != TERN_OK) return _st;                        \
  } while (0)
#define CHECK(cond, ...)                                   \
  do {                                                     \
    if (!(cond)) return fail(TERN_ERR_INVALID_ARG, __VA_ARGS__); \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
int kpad(int k) { return (k + kKAlign - 1) / kKAlign * kKAlign; }
size_t dsize(tern_dtype dt) { return dt == TERN_BF16 ? 2 : 4; }
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
bool valid_dt(tern_dtype dt) { return dt == TERN_F32 || dt == TERN_BF16; }

// device must be sm_100 (B200); cached per device
tern_status check_device() {
  static int cached[64];
  static std::once_flag once;
  std::call_once(once, [] { memset(cached, 0, sizeof(cached)); });
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(TERN_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  if (dev < 0 || dev >= 64) return fail(TERN_ERR_UNSUPPORTED, "device index %d", dev);
  if (cached[dev] == 0) {
    int maj = 0, mnr = 0;
    cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev);
    cached[dev] = (maj == 10 && mnr == 0) ? 1 : -1;
  }
  if (cached[dev] < 0) return fail(TERN_ERR_UNSUPPORTED, "libtern needs an sm_100 (B200) device");
  return TERN_OK;
}

tern_status check_weight(const tern_weight* w, int k, int n_seg, const char* name) {
  CHECK(w, "%s: null weight", name);
  CHECK(w->codes && aligned16(w->codes), "%s: codes null or not 16-byte aligned", name);
  CHECK(w->scales, "%s: null scales", name);
  CHECK(w->k == k, "%s: weight k=%d but input has %d features", name, w->k, k);
  CHECK(w->n_seg == n_seg, "%s: n_seg=%d, expected %d", name, w->n_seg, n_seg);
  CHECK(w->n_out > 0, "%s: n_out must be > 0", name);
  CHECK(w->n_rows == tern_packed_rows(w->n_out, w->n_seg), "%s: n_rows=%d inconsistent", name,
        w->n_rows);
  CHECK(w->ldw == kpad(k) / 16, "%s: ldw=%d must be %d", name, w->ldw, kpad(k) / 16);
  CHECK(w->e8 == nullptr || aligned16(w->e8), "%s: e8 not 16-byte aligned", name);
  return TERN_OK;
}

// ----------------------------------------------------------------- profiling hooks
struct ProfRec {
  cudaEvent_t a, b;
  tern_prof_rec meta;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_ev_pool;

cudaEvent_t prof_event() {
  if (!g_ev_pool.empty()) {
    cudaEvent_t e = g_ev_pool.back();
    g_ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// RAII: records an event before and after the launches in its scope.
struct Prof {
  bool on = false;
  ProfRec r{};
  cudaStream_t s;
  Prof(int kernel, int epi, int m, int n, int k, int n_seg, int dtype, cudaStream_t st) : s(st) {
    if (!g_prof_on) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    r.a = prof_event();
    r.b = prof_event();
    r.meta = tern_prof_rec{kernel, epi, m, n, k, n_seg, dtype, 0.0f};
    on = r.a && r.b && cudaEventRecord(r.a, st) == cudaSuccess;
  }
  ~Prof() {
    if (!on) return;
    cudaEventRecord(r.b, s);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back(r);
  }
};

size_t codes_bytes(const tern_weight& w) { return (size_t)w.n_rows * w.ldw * 4; }

Epi make_epi(int kind, const tern_weight& w, const float* bias, void* out, int ldo) {
  Epi e{};
  e.kind = kind;
  e.n_out = w.n_out;
  e.n_seg = w.n_seg;
  e.scales = w.scales;
  e.bias = bias;
  e.out = out;
  e.ldo = ldo;
  return e;
}

struct BlockWs {
  size_t q, deq, qsum, qf, fcg, oprime, x1, p, sout, gbuf, stl, stg, qsend, qgath, accb, part,
      part_bytes, total;
};
// world > 1 adds the rank's local outputs [M][max(ds,ls)] and the gather
// target [world][M][max(ds,ls)] (M > 1 gathers are then unshuffled to [M][width])
BlockWs block_ws(int32_t M, int32_t d, int32_t l, int32_t fcg_rows, tern_dtype dt,
                 int32_t world = 1, bool mega = false) {
  BlockWs w{};
  size_t off = 0;
  const int kq = kpad(d > l ? d : l);
  w.q = off; off += al256((size_t)M * kq);
  w.deq = off; off += al256((size_t)M * 4);
  w.qsum = off; off += al256((size_t)M * 4);
  // fused-quantization counters (QFuse): one area per fused GEMM of the block (o, gate|up,
  // down), zeroed ahead of the block's first quant launch (QFuse mode only)
  w.qf = off; off += al256((size_t)kQfAreas * qf_words(M) * 4);
  w.fcg = off; off += al256((size_t)M * fcg_rows * dsize(dt));
  w.oprime = off; off += al256((size_t)M * d * dsize(dt));
  w.x1 = off; off += al256((size_t)M * d * dsize(dt));
  w.p = off; off += al256((size_t)M * (l > 0 ? l : 1) * dsize(dt));
  w.sout = w.gbuf = w.stl = w.stg = w.qsend = w.qgath = off;
  if (world > 1) {
    const size_t cs = (size_t)((d > l ? d : l) / world);
    w.sout = off; off += al256((size_t)M * cs * dsize(dt));
    w.gbuf = off; off += al256((size_t)world * M * cs * dsize(dt));
    // int8-code gathers (tern_shard.gather_q): moment partials and code slices
    w.stl = off; off += al256((size_t)M * 16);
    w.stg = off; off += 3 * al256((size_t)world * M * 16);
    w.qsend = off; off += al256((size_t)M * cs + 4 * (size_t)M);
    w.qgath = off; off += al256((size_t)world * ((size_t)M * cs + 4 * (size_t)M));
  }
  // Megatron pairing: int32 partials of all d outputs + the q-sum partials,
  // all-reduced together
  w.accb = off;
  if (world > 1 && mega) off += al256(((size_t)M * d + (size_t)M) * 4);
  // split-K partial sums for small M (decode batches above the GEMV limit)
  w.part = off;
  w.part_bytes = 0;
  if (M <= kSplitKMaxM) {
    size_t rows = (size_t)fcg_rows;
    const size_t gu_rows = 2 * (((size_t)(l > 0 ? l : 1) + 63) / 64 * 64);
    if (gu_rows > rows) rows = gu_rows;
    if ((size_t)d > rows) rows = (size_t)d;
    // split-K slices: ksplit * tiles <~ 2 * SMs, so slices * M * rows <= 2*148*128*256
    size_t pb = (size_t)M * rows * 4 * 8;
    const size_t cap = (size_t)2 * 148 * 128 * 256 * 4;
    if (pb < cap) pb = cap;
    w.part_bytes = al256(pb);
    off += w.part_bytes;
  }
  w.total = off;
  return w;
}

template <typename T> T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// one BitLinear on the tensor-core path: quant (a2) then GEMM (a4+a5+functor)
tern_status bl_tc(const void* x, tern_dtype xdt, int M, int K, int ldx, const float* gain,
                  float eps, const tern_weight& w, tern_dtype ydt, const Epi& epi, int8_t* q,
                  int ldq, float* deq, int32_t* qsum, float* inv_rms, float* absmax,
                  cudaStream_t s, int32_t* part = nullptr, size_t part_bytes = 0,
                  int norm = TERN_NORM_RMS, uint32_t* zero = nullptr, int nzero = 0) {
  {
    Prof p(TERN_K_QUANT, 0, M, 0, K, 0, xdt, s);
    TRY_CUDA(launch_quant(x, xdt, M, K, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax, s, norm,
                          zero, nzero),
             "quant");
  }
  Prof p(TERN_K_GEMM, epi.kind, M, w.n_rows, w.k, w.n_seg, ydt, s);
  TRY_CUDA(launch_gemm(q, M, ldq, deq, qsum, w, ydt, epi, s, part, part_bytes), "gemm");
  return TERN_OK;
}

// The same BitLinear with the a2 quantization fused into the GEMM (f3, k_gemm.cu "fused
// quantization") when the shape takes the large-M tensor-core path and the norm is the
// RMSNorm; ctr = a zeroed QFuse counter area.  Otherwise quant + GEMM as bl_tc.
tern_status bl_tc_qf(const void* x, tern_dtype dt, int M, int K, const float* gain, float eps,
                     const tern_weight& w, const Epi& epi, int8_t* q, int ldq, float* deq,
                     int32_t* qsum, uint32_t* ctr, cudaStream_t s, int32_t* part,
                     size_t part_bytes, int norm) {
  if (ctr == nullptr || norm != TERN_NORM_RMS || !gemm_qfuse_ok(M, w, epi, part, part_bytes))
    return bl_tc(x, dt, M, K, K, gain, eps, w, dt, epi, q, ldq, deq, qsum, nullptr, nullptr, s,
                 part, part_bytes, norm);
  QFuse qf{x, K, gain, eps, ctr};
  Prof p(TERN_K_GEMM_QF, epi.kind, M, w.n_rows, w.k, w.n_seg, dt, s);
  TRY_CUDA(launch_gemm(q, M, ldq, deq, qsum, w, dt, epi, s, part, part_bytes, nullptr, &qf),
           "gemm + fused quant");
  return TERN_OK;
}

int block_world(const tern_block* b) { return b->shard.world > 1 ? b->shard.world : 1; }

tern_status check_block(const tern_block* b) {
  CHECK(b, "null block");
  const int d = b->d, l = b->l;
  CHECK(d > 0 && d % 64 == 0, "d=%d must be a positive multiple of 64", d);
  CHECK(l > 0 && l % 16 == 0, "l=%d must be a positive multiple of 16", l);
  const int world = block_world(b);
  if (world > 1) {
    CHECK(b->shard.ag, "sharded block: null all-gather callback");
    CHECK(b->shard.rank >= 0 && b->shard.rank < world, "shard rank %d of %d", b->shard.rank, world);
    CHECK(d % (64 * world) == 0 && l % (16 * world) == 0,
          "sharded block: d/world=%d must be a multiple of 64 and l/world=%d of 16", d / world,
          l / world);
  }
  const int ds = d / world, ls = l / world;
  tern_status st;
  if ((st = check_weight(&b->mix.fcg, d, 3, "fcg")) != TERN_OK) return st;
  const bool mega_w = world > 1 && b->shard.megatron;
  if ((st = check_weight(&b->mix.o, mega_w ? ds : d, 1, "o")) != TERN_OK) return st;
  if ((st = check_weight(&b->ch.gu, d, 2, "gate|up")) != TERN_OK) return st;
  if ((st = check_weight(&b->ch.down, mega_w ? ls : l, 1, "down")) != TERN_OK) return st;
  const bool mega = world > 1 && b->shard.megatron;
  CHECK(!mega || b->shard.ar, "Megatron-paired block: null all-reduce callback");
  CHECK(b->mix.fcg.n_out == ds, "MLGRU f|c|g weights must be d -> d/world");
  CHECK(b->ch.gu.n_out == ls, "GLU gate|up weights must be d -> l/world");
  if (mega) {   // row-parallel o and down: input columns of this rank, all d outputs
    CHECK(b->mix.o.n_out == d && b->mix.o.k == ds, "Megatron o must be d/world -> d");
    CHECK(b->ch.down.n_out == d && b->ch.down.k == ls, "Megatron down must be l/world -> d");
  } else {
    CHECK(b->mix.o.n_out == ds, "MLGRU o weights must be d -> d/world");
    CHECK(b->ch.down.n_out == ds, "GLU down weights must be l -> d/world");
  }
  CHECK(b->mix.gate == TERN_GATE_SIGMOID_H || b->mix.gate == TERN_GATE_LINEAR_H, "bad gate mode");
  if (b->mix.num_chunks != 0 && b->mix.num_chunks != 1 && b->mix.num_chunks != 4 &&
      b->mix.num_chunks != 8)
    return fail(TERN_ERR_UNSUPPORTED, "num_chunks=%d (0, 1, 4 or 8)", b->mix.num_chunks);
  CHECK(b->mix.eps > 0 && b->ch.eps > 0, "eps must be > 0");
  CHECK((b->mix.norm == TERN_NORM_RMS || b->mix.norm == TERN_NORM_CENTERED) &&
            (b->ch.norm == TERN_NORM_RMS || b->ch.norm == TERN_NORM_CENTERED),
        "bad norm mode");
  return TERN_OK;
}

}  // namespace

extern "C" {

int tern_abi_version(void) { return TERN_ABI_VERSION; }

tern_status tern_selftest(int32_t which, void* ws, uint64_t* mismatches) {
  CHECK(ws && mismatches && aligned16(ws) && which >= 0 && which <= 4, "tern_selftest: args");
  tern_status st = check_device();
  if (st) return st;
  static const int exps[11] = {0, 1, 2, 5, 10, 20, 40, 60, 80, 100, 119};
  unsigned long long* bad = static_cast<unsigned long long*>(ws);
  int* dexp = reinterpret_cast<int*>(static_cast<char*>(ws) + 16);
  TRY_CUDA(cudaMemset(bad, 0, 8), "selftest memset");
  TRY_CUDA(cudaMemcpy(dexp, exps, sizeof(exps), cudaMemcpyHostToDevice), "selftest h2d");
  TRY_CUDA(launch_selftest(which, bad, dexp, 11, 0), "selftest");
  unsigned long long h = 0;
  TRY_CUDA(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost), "selftest d2h");
  *mismatches = h;
  return TERN_OK;
}

void tern_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (on) {
    for (auto& r : g_prof) {
      g_ev_pool.push_back(r.a);
      g_ev_pool.push_back(r.b);
    }
    g_prof.clear();
  }
  g_prof_on = on != 0;
}

void tern_trace_enable(int32_t on) { gemv_trace_enable(on); }
int32_t tern_trace_collect(uint64_t* out, int32_t max_launches) {
  return gemv_trace_collect(reinterpret_cast<unsigned long long*>(out), max_launches);
}

int32_t tern_profile_collect(tern_prof_rec* out, int32_t max) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  int32_t n = 0;
  for (auto& r : g_prof) {
    if (out && n < max) {
      cudaEventSynchronize(r.b);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, r.a, r.b);
      out[n] = r.meta;
      out[n].ms = ms;
    }
    ++n;
  }
  return out ? (n < max ? n : max) : n;
}
const char* tern_last_error(void) { return g_err.c_str(); }
void tern_set_fused_scan(int32_t mode) { g_fused_scan = mode < 0 ? 0 : mode > 2 ? 2 : mode; }
int32_t tern_get_fused_scan(void) { return g_fused_scan; }
void tern_set_gemv_max_m(int32_t m) { g_gemv_max_m = m < 0 ? 0 : (m > kGemvMaxM ? kGemvMaxM : m); }
int32_t tern_get_gemv_max_m(void) { return g_gemv_max_m; }
void tern_set_batched_fin(int32_t on) { g_batched_fin = on ? 1 : 0; }
void tern_set_gemm_sab(int32_t on) { g_gemm_sab = on ? 1 : 0; }
void tern_set_gemm_2sm(int32_t on) { g_gemm_2sm = on ? 1 : 0; }
void tern_set_qfuse(int32_t on) { g_qfuse_on = on ? 1 : 0; }
void tern_set_bwd_tc(int32_t on) { g_bwd_tc = on ? 1 : 0; }
int32_t tern_get_bwd_tc(void) { return g_bwd_tc; }
int32_t tern_get_qfuse(void) { return g_qfuse_on; }
int32_t tern_get_gemm_2sm(void) { return g_gemm_2sm; }
int32_t tern_get_gemm_sab(void) { return g_gemm_sab; }
void tern_set_norm_mode(tern_norm_mode mode) {
  g_norm_mode = mode == TERN_NORM_CENTERED ? TERN_NORM_CENTERED : TERN_NORM_RMS;
}
tern_norm_mode tern_get_norm_mode(void) { return (tern_norm_mode)g_norm_mode; }
int32_t tern_get_batched_fin(void) { return g_batched_fin; }

int32_t tern_packed_rows(int32_t n_out, int32_t n_seg) {
  if (n_seg <= 1) return n_out;
  return (n_out + kSegRows - 1) / kSegRows * kSegRows * n_seg;
}
int32_t tern_packed_ldw(int32_t k) { return kpad(k) / 16; }

tern_status tern_codes_init(uint32_t* codes, int32_t n_rows, int32_t ldw, tern_stream stream) {
  CHECK(codes && n_rows > 0 && ldw > 0, "tern_codes_init: bad arguments");
  tern_status st = check_device();
  if (st) return st;
  TRY_CUDA(launch_codes_init(codes, n_rows, ldw, (cudaStream_t)stream), "codes_init");
  return TERN_OK;
}

tern_status tern_expand(const tern_weight* w, uint8_t* e8, tern_stream stream) {
  CHECK(w && e8 && aligned16(e8), "tern_expand: null/misaligned pointer");
  tern_status st = check_weight(w, w->k, w->n_seg, "tern_expand");
  if (st) return st;
  if ((st = check_device()) != TERN_OK) return st;
  TRY_CUDA(launch_expand(*w, e8, (cudaStream_t)stream), "expand");
  return TERN_OK;
}

size_t tern_pack_workspace(int32_t n, int32_t k) {
  (void)n; (void)k;
  return pack_workspace_bytes() + 256;
}

tern_status tern_pack(const float* W, int32_t n, int32_t k, const float* scale_in, int32_t n_seg,
                      int32_t seg_idx, uint32_t* codes, int32_t n_rows, float* scale_out, void* ws,
                      size_t ws_bytes, tern_stream stream) {
  CHECK(W && codes && scale_out && ws, "tern_pack: null pointer");
  CHECK(n > 0 && k > 0, "tern_pack: n=%d k=%d must be > 0", n, k);
  CHECK(n_seg >= 1 && n_seg <= 3 && seg_idx >= 0 && seg_idx < n_seg, "tern_pack: bad segment");
  CHECK(n_rows == tern_packed_rows(n, n_seg), "tern_pack: n_rows=%d, expected %d", n_rows,
        tern_packed_rows(n, n_seg));
  CHECK(ws_bytes >= tern_pack_workspace(n, k), "tern_pack: workspace too small");
  CHECK(aligned16(ws), "tern_pack: workspace not 16-byte aligned");
  tern_status st = check_device();
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  double* part = static_cast<double*>(ws);
  float* scratch = reinterpret_cast<float*>(static_cast<char*>(ws) + pack_workspace_bytes());
  TRY_CUDA(launch_absmean(W, (int64_t)n * k, scale_in, scratch, part, s), "absmean");
  float m = 0.0f;
  TRY_CUDA(cudaMemcpyAsync(&m, scratch, sizeof(float), cudaMemcpyDeviceToHost, s), "scale d2h");
  TRY_CUDA(cudaStreamSynchronize(s), "tern_pack sync");
  if (!(m > 0.0f) || !(m < __FLT_MAX__))
    return fail(TERN_ERR_DEGENERATE, "tern_pack: mean|W| = %g (all-zero or non-finite W)", m);
  TRY_CUDA(cudaMemcpyAsync(scale_out, scratch, sizeof(float), cudaMemcpyDeviceToDevice, s),
           "scale copy");
  TRY_CUDA(launch_pack_codes(W, n, k, n_seg, seg_idx, codes, n_rows, scratch, s), "pack");
  return TERN_OK;
}

tern_status tern_quant(const void* x, tern_dtype xdt, int32_t m, int32_t k, int32_t ldx,
                       const float* gain, float eps, int8_t* q, int32_t ldq, float* deq,
                       int32_t* qsum, float* inv_rms, float* absmax, tern_stream stream) {
  CHECK(x && q && deq && qsum, "tern_quant: null pointer");
  CHECK(valid_dt(xdt), "tern_quant: bad dtype");
  CHECK(m >= 0 && k > 0 && k % 16 == 0, "tern_quant: m=%d k=%d (k must be a multiple of 16)", m, k);
  CHECK(k <= 32 * 128 * 4, "tern_quant: k=%d too large", k);
  CHECK(ldx >= k && ldx % 16 == 0 && aligned16(x), "tern_quant: ldx/alignment");
  CHECK(ldq >= kpad(k) && ldq % 16 == 0 && aligned16(q), "tern_quant: ldq must be >= %d", kpad(k));
  CHECK(eps > 0, "tern_quant: eps must be > 0");
  tern_status st = check_device();
  if (st) return st;
  TRY_CUDA(launch_quant(x, xdt, m, k, ldx, gain, eps, q, ldq, deq, qsum, inv_rms, absmax,
                        (cudaStream_t)stream, g_norm_mode),
           "quant");
  return TERN_OK;
}

size_t bitlinear_ws_base(int32_t m, int32_t k) {
  return al256((size_t)m * kpad(k)) + 2 * al256((size_t)m * 4);
}
constexpr size_t kBlPartBytes = (size_t)2 * 148 * 128 * 256 * 4;   // split-K partials
size_t tern_bitlinear_workspace(int32_t m, int32_t k) {
  const bool splitk = m > kGemvMaxM && m <= kSplitKMaxM;
  return bitlinear_ws_base(m, k) + (splitk ? kBlPartBytes : 0);
}

tern_status bitlinear_fwd(const void* x, tern_dtype xdt, int32_t m, int32_t k, int32_t ldx,
                          const float* gain, float eps, const tern_weight* w, const float* bias,
                          void* y, tern_dtype ydt, int32_t ldy, const tern_bl_taps* taps, void* ws,
                          size_t ws_bytes, tern_stream stream) {
  CHECK(valid_dt(xdt) && valid_dt(ydt), "bitlinear_fwd: bad dtype");
  CHECK(m >= 0 && k > 0 && k % 16 == 0, "bitlinear_fwd: m=%d k=%d", m, k);
  if (m == 0) return TERN_OK;   // no tokens: a no-op
  CHECK(x && y, "bitlinear_fwd: null x/y");
  CHECK(ldx >= k && ldx % 16 == 0 && aligned16(x), "bitlinear_fwd: ldx/alignment");
  tern_status st = check_weight(w, k, 1, "bitlinear_fwd");
  if (st) return st;
  CHECK(ldy >= w->n_out && ldy % 16 == 0 && aligned16(y), "bitlinear_fwd: ldy/alignment");
  CHECK(eps > 0, "bitlinear_fwd: eps must be > 0");
  const bool gemv = m <= g_gemv_max_m && gemv_supported(m, k, xdt);
  if (taps) {
    CHECK(!taps->q || taps->ldq >= kpad(k), "bitlinear_fwd: taps ldq");
    CHECK(!taps->acc || taps->ldacc >= w->n_rows, "bitlinear_fwd: taps ldacc");
  }
  if (!gemv) {
    CHECK(ws && aligned16(ws) && ws_bytes >= bitlinear_ws_base(m, k),
          "bitlinear_fwd: workspace too small (%zu < %zu)", ws_bytes, bitlinear_ws_base(m, k));
    CHECK(k <= 16384, "bitlinear_fwd: k too large");
  }
  st = check_device();
  if (st) return st;
  if (m == 0) return TERN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  Epi e = make_epi(EPI_STORE, *w, bias, y, ldy);
  if (taps && taps->acc) {
    e.acc = taps->acc;
    e.ldacc = taps->ldacc;
  }
  if (gemv) {
    QuantTaps qt{};
    if (taps) {
      qt.q = taps->q; qt.ldq = taps->ldq; qt.deq = taps->deq;
      qt.inv_rms = taps->inv_rms; qt.absmax = taps->absmax;
    }
    Prof pr(TERN_K_GEMV, e.kind, m, w->n_rows, k, 1, xdt, s);
    TRY_CUDA(launch_gemv(x, xdt, ydt, m, k, ldx, gain, eps, *w, e, &qt, s, nullptr, 0, g_norm_mode),
             "gemv");
    return TERN_OK;
  }
  int8_t* q = (taps && taps->q) ? taps->q : static_cast<int8_t*>(ws);
  const int ldq = (taps && taps->q) ? taps->ldq : kpad(k);
  float* deq = (taps && taps->deq) ? taps->deq : at<float>(ws, al256((size_t)m * kpad(k)));
  int32_t* qsum = at<int32_t>(ws, al256((size_t)m * kpad(k)) + al256((size_t)m * 4));
  // split-K partials behind the base workspace when the caller provided them
  const size_t base = bitlinear_ws_base(m, k);
  int32_t* part = nullptr;
  size_t part_bytes = 0;
  if (m <= kSplitKMaxM && ws_bytes >= base + kBlPartBytes && !(taps && taps->acc)) {
    part = at<int32_t>(ws, base);
    part_bytes = ws_bytes - base;
  }
  return bl_tc(x, xdt, m, k, ldx, gain, eps, *w, ydt, e, q, ldq, deq, qsum,
               taps ? taps->inv_rms : nullptr, taps ? taps->absmax : nullptr, s, part, part_bytes,
               g_norm_mode);
}

size_t bitlinear_bwd_workspace(int32_t m, int32_t k, int32_t n) {
  if (m <= 0 || k <= 0 || n <= 0) return 0;
  return bwd_workspace(m, k, n);
}

tern_status bitlinear_bwd(const void* x, tern_dtype dt, int32_t m, int32_t k, const tern_weight* w,
                          float eps, int32_t norm, const void* dO, float* dX, float* dW, float* db,
                          void* ws, size_t ws_bytes, tern_stream stream) {
  CHECK(valid_dt(dt), "bitlinear_bwd: bad dtype");
  CHECK(dt == TERN_F32 || g_bwd_tc, "bitlinear_bwd: bf16 inputs need the tensor-core path");
  CHECK(m >= 0 && k > 0 && k % 16 == 0, "bitlinear_bwd: m=%d k=%d", m, k);
  CHECK(norm == TERN_NORM_RMS || norm == TERN_NORM_CENTERED, "bitlinear_bwd: norm=%d", norm);
  tern_status st = check_weight(w, k, 1, "bitlinear_bwd");
  if (st) return st;
  CHECK(w->e8 != nullptr, "bitlinear_bwd: the weight's u8 copy e8 is required (tern_expand)");
  CHECK(eps > 0, "bitlinear_bwd: eps must be > 0");
  CHECK(dW, "bitlinear_bwd: null dW");
  if (m == 0) {   // no tokens: dW = 0, db = 0
    TRY_CUDA(cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)w->n_out * k, (cudaStream_t)stream),
             "bwd zero dW");
    if (db) TRY_CUDA(cudaMemsetAsync(db, 0, sizeof(float) * w->n_out, (cudaStream_t)stream), "bwd zero db");
    return TERN_OK;
  }
  CHECK(x && dO && dX, "bitlinear_bwd: null pointer");
  CHECK(aligned16(x) && aligned16(dX) && aligned16(dO), "bitlinear_bwd: x, dO, dX must be 16-byte aligned");
  CHECK(k <= 32 * 128 * 4, "bitlinear_bwd: k=%d too large", k);
  CHECK(ws && aligned16(ws) && ws_bytes >= bwd_workspace(m, k, w->n_out),
        "bitlinear_bwd: workspace too small (%zu < %zu)", ws_bytes, bwd_workspace(m, k, w->n_out));
  st = check_device();
  if (st) return st;
  TRY_CUDA(launch_bitlinear_bwd(x, dt, m, k, *w, eps, norm, dO, dX, dW, db, ws,
                                (cudaStream_t)stream),
           "bitlinear_bwd");
  return TERN_OK;
}

tern_status tern_contract(const int8_t* q, int32_t m, int32_t ldq, const int32_t* qsum,
                          const tern_weight* w, int32_t* acc, int32_t ldacc, tern_stream stream) {
  CHECK(q && qsum && acc && w, "tern_contract: null pointer");
  CHECK(m >= 0, "tern_contract: m < 0");
  tern_status st = check_weight(w, w ? w->k : 0, w ? w->n_seg : 1, "tern_contract");
  if (st) return st;
  CHECK(ldq >= kpad(w->k) && ldq % 16 == 0 && aligned16(q), "tern_contract: ldq");
  CHECK(ldacc >= w->n_rows, "tern_contract: ldacc < n_rows");
  st = check_device();
  if (st) return st;
  Epi e = make_epi(EPI_NONE, *w, nullptr, nullptr, 0);
  e.acc = acc;
  e.ldacc = ldacc;
  // deq is unused by EPI_NONE; pass qsum as a harmless readable pointer
  TRY_CUDA(launch_gemm(q, m, ldq, reinterpret_cast<const float*>(qsum), qsum, *w, TERN_F32, e,
                       (cudaStream_t)stream),
           "gemm");
  return TERN_OK;
}

// ---------------------------------------------------------------- fixed point (f4(ii))
tern_status tern_fxp_scales(const float* w, int32_t n, int32_t shift, int8_t* wq, int32_t* e_host,
                            void* ws, tern_stream stream) {
  CHECK(w && wq && e_host && ws, "tern_fxp_scales: null pointer");
  CHECK(n > 0 && shift >= 0 && shift <= 6, "tern_fxp_scales: n=%d shift=%d", n, shift);
  CHECK(aligned16(ws), "tern_fxp_scales: workspace not 16-byte aligned");
  tern_status st = check_device();
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* dev = static_cast<int32_t*>(ws);   // [0] e, [1] status
  TRY_CUDA(launch_fxp_scales(w, n, shift, wq, dev, dev + 1, s), "fxp_scales");
  int32_t h[2] = {0, 0};
  TRY_CUDA(cudaMemcpyAsync(h, dev, sizeof(h), cudaMemcpyDeviceToHost, s), "fxp_scales d2h");
  TRY_CUDA(cudaStreamSynchronize(s), "fxp_scales sync");
  if (h[1]) return fail(TERN_ERR_DEGENERATE, "tern_fxp_scales: max|w| is 0 or not finite");
  *e_host = h[0];
  return TERN_OK;
}

tern_status tern_fxp_quant_act(const void* x, tern_dtype dt, int64_t n, int16_t* q, int32_t* e,
                               void* ws, tern_stream stream) {
  CHECK(valid_dt(dt), "tern_fxp_quant_act: bad dtype");
  CHECK(n >= 0, "tern_fxp_quant_act: n=%lld", (long long)n);
  if (n == 0) return TERN_OK;
  CHECK(x && q && e && ws, "tern_fxp_quant_act: null pointer");
  CHECK(aligned16(ws), "tern_fxp_quant_act: workspace not 16-byte aligned");
  tern_status st = check_device();
  if (st) return st;
  TRY_CUDA(launch_fxp_quant_act(x, dt, n, q, e, static_cast<uint32_t*>(ws), (cudaStream_t)stream),
           "fxp_quant_act");
  return TERN_OK;
}

tern_status tern_fxp_sigmoid(const int32_t* x, int64_t n, int32_t* y, tern_stream stream) {
  CHECK(n >= 0, "tern_fxp_sigmoid: n=%lld", (long long)n);
  if (n == 0) return TERN_OK;
  CHECK(x && y && aligned16(x) && aligned16(y), "tern_fxp_sigmoid: null or unaligned pointer");
  tern_status st = check_device();
  if (st) return st;
  TRY_CUDA(launch_fxp_sigmoid(x, n, y, (cudaStream_t)stream), "fxp_sigmoid");
  return TERN_OK;
}

tern_status tern_fxp_inv_sqrt(const uint64_t* v, const int32_t* e, int64_t n, uint32_t* y,
                              int32_t* ey, tern_stream stream) {
  CHECK(n >= 0, "tern_fxp_inv_sqrt: n=%lld", (long long)n);
  if (n == 0) return TERN_OK;
  CHECK(v && e && y && ey, "tern_fxp_inv_sqrt: null pointer");
  CHECK((reinterpret_cast<uintptr_t>(v) & 7u) == 0, "tern_fxp_inv_sqrt: v not 8-byte aligned");
  tern_status st = check_device();
  if (st) return st;
  TRY_CUDA(launch_fxp_inv_sqrt(v, e, n, y, ey, (cudaStream_t)stream), "fxp_inv_sqrt");
  return TERN_OK;
}

tern_status tern_fxp_rmsnorm(const int16_t* xq, const int32_t* ex, const int8_t* wq, int32_t ew,
                             double eps, int32_t rows, int32_t d, int16_t* out, int32_t* eo,
                             tern_stream stream) {
  CHECK(rows >= 0 && d >= 1 && d <= 65536, "tern_fxp_rmsnorm: rows=%d d=%d", rows, d);
  CHECK(eps >= 0.0 && eps < 1e30, "tern_fxp_rmsnorm: eps=%g", eps);
  if (rows == 0) return TERN_OK;
  CHECK(xq && ex && wq && out && eo, "tern_fxp_rmsnorm: null pointer");
  CHECK(aligned16(xq), "tern_fxp_rmsnorm: xq not 16-byte aligned");
  tern_status st = check_device();
  if (st) return st;
  TRY_CUDA(launch_fxp_rmsnorm(xq, ex, wq, ew, eps, rows, d, out, eo, (cudaStream_t)stream),
           "fxp_rmsnorm");
  return TERN_OK;
}

// W8A16 BitLinear (F6) workspace: the normalised rows and their exponents, then ONE int8
// operand of 2m + 1 rows for the tcgen05 GEMM -- the m high-digit rows, the m low-digit
// rows and a row of ones (its product is sum_k t[n][k]) -- with their q-sums, and the
// int32 accumulators of all 2m + 1 rows: one GEMM launch for the whole contraction
struct FxpBlWs {
  size_t yn, en, a, qs, acc, total;
};
static FxpBlWs fxp_bl_ws(int m, int k, int n_rows) {
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t ldq = (size_t)kpad(k), rows = 2 * (size_t)m + 1;
  FxpBlWs L;
  size_t o = 0;
  L.yn = o; o += up((size_t)m * k * 2 + 16);
  L.en = o; o += up((size_t)m * 4 + 4);
  L.a = o; o += up(rows * ldq + 16);
  L.qs = o; o += up(rows * 4);
  L.acc = o; o += up(rows * n_rows * 4);
  L.total = o;
  return L;
}

size_t tern_fxp_bitlinear_workspace(int32_t m, int32_t k, int32_t n_rows) {
  if (m < 0 || k <= 0 || n_rows <= 0) return 0;
  return fxp_bl_ws(m, k, n_rows).total;
}

tern_status tern_fxp_bitlinear(const int16_t* xq, const int32_t* ex, int32_t m, int32_t k,
                               const int8_t* gq, int32_t eg, double eps, const tern_weight* w,
                               int16_t* y, int32_t ldy, int32_t* ey, void* ws, size_t ws_bytes,
                               tern_stream stream) {
  CHECK(m >= 0 && k >= 1 && k <= 65535, "tern_fxp_bitlinear: m=%d k=%d", m, k);
  CHECK(eps >= 0.0 && eps < 1e30, "tern_fxp_bitlinear: eps=%g", eps);
  tern_status st = check_weight(w, k, 1, "tern_fxp_bitlinear");
  if (st) return st;
  if (m == 0) return TERN_OK;
  CHECK(xq && ex && gq && y && ey && ws, "tern_fxp_bitlinear: null pointer");
  CHECK(aligned16(xq) && aligned16(ws), "tern_fxp_bitlinear: xq / ws not 16-byte aligned");
  CHECK(ldy >= w->n_out, "tern_fxp_bitlinear: ldy=%d < n_out=%d", ldy, w->n_out);
  const FxpBlWs L = fxp_bl_ws(m, k, w->n_rows);
  CHECK(ws_bytes >= L.total, "tern_fxp_bitlinear: workspace %zu < %zu", ws_bytes, L.total);
  st = check_device();
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  char* b = static_cast<char*>(ws);
  int16_t* yn = reinterpret_cast<int16_t*>(b + L.yn);
  int32_t* en = reinterpret_cast<int32_t*>(b + L.en);
  int8_t* a = reinterpret_cast<int8_t*>(b + L.a);
  int32_t* qs = reinterpret_cast<int32_t*>(b + L.qs);
  int32_t* acc = reinterpret_cast<int32_t*>(b + L.acc);
  const int ldq = kpad(k);
  const size_t nr = (size_t)w->n_rows;
  TRY_CUDA(launch_fxp_rmsnorm(xq, ex, gq, eg, eps, m, k, yn, en, s), "fxp_bitlinear norm");
  TRY_CUDA(launch_fxp_split(yn, m, k, ldq, a, a + (size_t)m * ldq, qs, qs + m,
                            a + (size_t)2 * m * ldq, qs + 2 * m, s),
           "fxp_bitlinear split");
  // the exact int8 x ternary contraction of all 2m + 1 rows (EPI_NONE: int32 out)
  Epi e = make_epi(EPI_NONE, *w, nullptr, nullptr, 0);
  e.acc = acc;
  e.ldacc = w->n_rows;
  TRY_CUDA(launch_gemm(a, 2 * m + 1, ldq, reinterpret_cast<const float*>(qs), qs, *w, TERN_F32, e,
                       s),
           "fxp_bitlinear gemm");
  TRY_CUDA(launch_fxp_combine(acc, acc + (size_t)m * nr, w->n_rows, acc + (size_t)2 * m * nr,
                              w->scales, w->n_out, m, en, y, ldy, ey, s),
           "fxp_bitlinear combine");
  return TERN_OK;
}

tern_status tern_mlgru_scan(const void* fcg, tern_dtype dt, int32_t B, int32_t T, int32_t d,
                            tern_gate_mode gate, float* h, void* oprime, tern_stream stream) {
  CHECK(fcg && h && oprime, "tern_mlgru_scan: null pointer");
  CHECK(valid_dt(dt), "tern_mlgru_scan: bad dtype");
  CHECK(B >= 0 && T >= 0 && d > 0 && d % 64 == 0, "tern_mlgru_scan: B=%d T=%d d=%d", B, T, d);
  CHECK(gate == TERN_GATE_SIGMOID_H || gate == TERN_GATE_LINEAR_H, "tern_mlgru_scan: gate");
  tern_status st = check_device();
  if (st) return st;
  Prof pr(TERN_K_SCAN, gate, B * T, d, d, 3, dt, (cudaStream_t)stream);
  TRY_CUDA(launch_scan(fcg, dt, B, T, d, gate, h, oprime, (cudaStream_t)stream), "scan");
  return TERN_OK;
}

size_t tern_mlgru_workspace(const tern_mlgru* p, int32_t B, int32_t T, int32_t d, tern_dtype dt) {
  const int rows = p ? p->fcg.n_rows : 3 * d;
  return block_ws(B * T, d, 0, rows, dt).total;
}
size_t tern_glu_workspace(const tern_glu* p, int32_t m, int32_t d, int32_t l, tern_dtype dt) {
  (void)p;
  return block_ws(m, d, l, 0, dt).total;
}
size_t tern_block_workspace(const tern_block* b, int32_t B, int32_t T, tern_dtype dt) {
  if (!b) return 0;
  return block_ws(B * T, b->d, b->l, b->mix.fcg.n_rows, dt, block_world(b),
                   b->shard.megatron != 0).total;
}

tern_status tern_block_ws_layout(const tern_block* b, int32_t B, int32_t T, tern_dtype dt,
                                 tern_block_taps* out) {
  CHECK(b && out, "tern_block_ws_layout: null pointer");
  BlockWs w = block_ws(B * T, b->d, b->l, b->mix.fcg.n_rows, dt, block_world(b),
                   b->shard.megatron != 0);
  out->fcg = w.fcg;
  out->oprime = w.oprime;
  out->x1 = w.x1;
  out->p = w.p;
  return TERN_OK;
}

namespace {

// token mixer: x [M][d] -> out (o, or x1 = x + o when resid), state h
// L2 prefetch hints for the two GEMVs of a mixer (decode): weights of later launches
struct PfPlan {
  const void* p[2] = {nullptr, nullptr};
  size_t n[2] = {0, 0};
};

// Sequence-parallel prefill (C23): this rank holds tokens [rank T/world, ...) of every
// sequence; the scan's boundary state comes from the other ranks' slice aggregates.
struct SeqPar {
  int rank = 0, world = 1;
  tern_allgather_fn ag = nullptr;
  void* ctx = nullptr;
  float *send = nullptr, *recv = nullptr, *hfin = nullptr;   // [2][B][d], [world][2][B][d], [B][d]
};

tern_status run_mlgru(const tern_mlgru& p, const void* x, void* out, bool resid, tern_dtype dt,
                      int B, int T, int d, float* h, void* ws, const BlockWs& L, cudaStream_t s,
                      const PfPlan& pf = PfPlan(), const SeqPar* sp = nullptr) {
  const int M = B * T;
  void* op = at<char>(ws, L.oprime);
  if (sp) {
    // pass 1 on the f^c^g^ of this slice, exchange, compose, pass 2 = the exact scan of
    // the slice from its boundary state; the state after the block is the composition
    // through every slice (identical on all ranks)
    int8_t* q = at<int8_t>(ws, L.q);
    float* deq = at<float>(ws, L.deq);
    int32_t* qsum = at<int32_t>(ws, L.qsum);
    void* fcg = at<char>(ws, L.fcg);
    const int ldq = kpad(d);
    if (T > 0) {
      Epi e1 = make_epi(EPI_FCG, p.fcg, p.bias_fcg, fcg, p.fcg.n_rows);
      tern_status st = bl_tc(x, dt, M, d, d, p.gain_x, p.eps, p.fcg, dt, e1, q, ldq, deq, qsum,
                             nullptr, nullptr, s, at<int32_t>(ws, L.part), L.part_bytes, p.norm);
      if (st) return st;
    }
    TRY_CUDA(launch_scan_agg(fcg, dt, B, T, d, sp->send, s), "seqpar aggregates");
    const size_t per = (size_t)2 * B * d * sizeof(float);
    if (sp->ag(sp->ctx, sp->send, sp->recv, per, (tern_stream)s) != 0)
      return fail(TERN_ERR_CUDA, "block_prefill_sp: all-gather callback failed");
    TRY_CUDA(launch_sp_compose(sp->recv, sp->world, sp->rank, (int64_t)B * d, h, sp->hfin, s),
             "seqpar compose");
    if (T > 0) {
      Prof pr(TERN_K_SCAN, p.gate, B * T, d, d, 3, dt, s);
      TRY_CUDA(launch_scan(fcg, dt, B, T, d, p.gate, h, op, s), "scan");
    }
    TRY_CUDA(cudaMemcpyAsync(h, sp->hfin, sizeof(float) * B * d, cudaMemcpyDeviceToDevice, s),
             "seqpar state");
    if (T == 0) return TERN_OK;
    Epi e2 = make_epi(resid ? EPI_RESID : EPI_STORE, p.o, p.bias_o, out, d);
    e2.res = x;
    e2.ldr = d;
    return bl_tc(op, dt, M, d, d, p.gain_o, p.eps, p.o, dt, e2, q, ldq, deq, qsum, nullptr,
                 nullptr, s, at<int32_t>(ws, L.part), L.part_bytes, p.norm);
  }
  if (T == 1 && B <= g_gemv_max_m && gemv_supported(B, d, dt)) {
    Epi e1 = make_epi(EPI_MLGRU, p.fcg, p.bias_fcg, op, d);
    e1.h = h;
    e1.gate = p.gate;
    {
      Prof pr(TERN_K_GEMV, e1.kind, B, p.fcg.n_rows, d, 3, dt, s);
      TRY_CUDA(launch_gemv(x, dt, dt, B, d, d, p.gain_x, p.eps, p.fcg, e1, nullptr, s, pf.p[0],
                           pf.n[0], p.norm),
               "gemv fcg");
    }
    Epi e2 = make_epi(resid ? EPI_RESID : EPI_STORE, p.o, p.bias_o, out, d);
    e2.res = x;
    e2.ldr = d;
    Prof pr(TERN_K_GEMV, e2.kind, B, p.o.n_rows, d, 1, dt, s);
    TRY_CUDA(launch_gemv(op, dt, dt, B, d, d, p.gain_o, p.eps, p.o, e2, nullptr, s, pf.p[1], pf.n[1],
                         p.norm),
             "gemv o");
    return TERN_OK;
  }
  int8_t* q = at<int8_t>(ws, L.q);
  float* deq = at<float>(ws, L.deq);
  int32_t* qsum = at<int32_t>(ws, L.qsum);
  void* fcg = at<char>(ws, L.fcg);
  const int ldq = kpad(d);
  // QFuse counter areas of this block's fused GEMMs (o, gate|up, down): the first quant
  // launch below zeroes them
  uint32_t* qf0 = at<uint32_t>(ws, L.qf);
  const int nqf = g_qfuse_on ? kQfAreas * qf_words(M) : 0;
  // the prefill scan: sequential (1) or chunked over time (4, 8; tern_mlgru.num_chunks)
  const int chunks = T > 1 ? scan_chunks_resolve(p.num_chunks, B, T, d) : 1;
  // the fused kernel walks each sequence's 128-token tiles; short sequences (decode
  // steps with B > gemv_max_m) take GEMM + scan instead
  if (T == 1 && L.part_bytes > 0) {
    // decode step above the GEMV limit: the MLGRU step runs in the GEMM's
    // split-K epilogue (no f^c^g^ round trip, no scan launch)
    Epi e1 = make_epi(EPI_MLGRU, p.fcg, p.bias_fcg, op, d);
    e1.h = h;
    e1.gate = p.gate;
    tern_status st = bl_tc(x, dt, M, d, d, p.gain_x, p.eps, p.fcg, dt, e1, q, ldq, deq, qsum,
                           nullptr, nullptr, s, at<int32_t>(ws, L.part), L.part_bytes, p.norm);
    if (st) return st;
  } else if (T >= 64 && fcgscan_supported(p.fcg, d) && chunks == 1 &&
             (g_fused_scan == 2 || (g_fused_scan == 1 && fcgscan_preferred(B, d)))) {
    // a4 + a6 fused: f^c^g^ stay on chip (k_fcgscan.cu)
    {
      Prof pr(TERN_K_QUANT, 0, M, 0, d, 0, dt, s);
      TRY_CUDA(launch_quant(x, dt, M, d, d, p.gain_x, p.eps, q, ldq, deq, qsum, nullptr, nullptr, s,
                            p.norm, qf0, nqf),
               "quant");
    }
    Prof pr(TERN_K_FCGSCAN, p.gate, M, p.fcg.n_rows, d, 3, dt, s);
    TRY_CUDA(launch_fcgscan(q, ldq, deq, qsum, p.fcg, p.bias_fcg, dt, B, T, d, p.gate, h, op, s),
             "fcgscan");
  } else {
    Epi e1 = make_epi(EPI_FCG, p.fcg, p.bias_fcg, fcg, p.fcg.n_rows);
    tern_status st = bl_tc(x, dt, M, d, d, p.gain_x, p.eps, p.fcg, dt, e1, q, ldq, deq, qsum,
                           nullptr, nullptr, s, at<int32_t>(ws, L.part), L.part_bytes, p.norm,
                           qf0, nqf);
    if (st) return st;
    Prof pr(TERN_K_SCAN, p.gate, B * T, d, d, 3, dt, s);
    TRY_CUDA(launch_scan_chunks(fcg, dt, B, T, d, p.gate, h, op, chunks, s), "scan");
  }
  Epi e2 = make_epi(resid ? EPI_RESID : EPI_STORE, p.o, p.bias_o, out, d);
  e2.res = x;
  e2.ldr = d;
  // o' is quantized inside the o GEMM (counter area 0, zeroed by the quant of x above)
  return bl_tc_qf(op, dt, M, d, p.gain_o, p.eps, p.o, e2, q, ldq, deq, qsum, qf0, s,
                  at<int32_t>(ws, L.part), L.part_bytes, p.norm);
}

// channel mixer: x [M][d] -> out (d, or y = x + d when resid)
// in_place: x is `out` (the block's x1 written into y), the residual added in place
tern_status run_glu(const tern_glu& p, const void* x, void* out, bool resid, tern_dtype dt, int M,
                    int d, int l, void* ws, const BlockWs& L, cudaStream_t s,
                    const PfPlan& pf = PfPlan(), bool qf_ready = false, bool in_place = false) {
  void* pp = at<char>(ws, L.p);
  Epi e1 = make_epi(EPI_SWIGLU, p.gu, nullptr, pp, l);
  Epi e2 = make_epi(in_place ? EPI_RESID_RED : (resid ? EPI_RESID : EPI_STORE), p.down, nullptr,
                    out, d);
  e2.res = in_place ? nullptr : x;
  e2.ldr = d;
  if (M <= g_gemv_max_m && gemv_supported(M, d, dt) && gemv_supported(M, l, dt)) {
    {
      Prof pr(TERN_K_GEMV, e1.kind, M, p.gu.n_rows, d, 2, dt, s);
      TRY_CUDA(launch_gemv(x, dt, dt, M, d, d, p.gain_x, p.eps, p.gu, e1, nullptr, s, pf.p[0],
                           pf.n[0], p.norm),
               "gemv gu");
    }
    Prof pr(TERN_K_GEMV, e2.kind, M, p.down.n_rows, l, 1, dt, s);
    TRY_CUDA(launch_gemv(pp, dt, dt, M, l, l, p.gain_p, p.eps, p.down, e2, nullptr, s, pf.p[1],
                         pf.n[1], p.norm),
             "gemv down");
    return TERN_OK;
  }
  int8_t* q = at<int8_t>(ws, L.q);
  float* deq = at<float>(ws, L.deq);
  int32_t* qsum = at<int32_t>(ws, L.qsum);
  // QFuse counter areas 1 (gate|up) and 2 (down); qf_ready: zeroed by the token mixer's
  // first quant launch (block prefill), else by the quant of x here
  uint32_t* qf0 = at<uint32_t>(ws, L.qf);
  const int qw = qf_words(M);
  tern_status st = qf_ready
      ? bl_tc_qf(x, dt, M, d, p.gain_x, p.eps, p.gu, e1, q, kpad(d), deq, qsum, qf0 + qw, s,
                 at<int32_t>(ws, L.part), L.part_bytes, p.norm)
      : bl_tc(x, dt, M, d, d, p.gain_x, p.eps, p.gu, dt, e1, q, kpad(d), deq, qsum, nullptr,
              nullptr, s, at<int32_t>(ws, L.part), L.part_bytes, p.norm, qf0,
              g_qfuse_on ? kQfAreas * qw : 0);
  if (st) return st;
  return bl_tc_qf(pp, dt, M, l, p.gain_p, p.eps, p.down, e2, q, kpad(l), deq, qsum, qf0 + 2 * qw,
                  s, at<int32_t>(ws, L.part), L.part_bytes, p.norm);
}

// one BitLinear on either path (decode GEMV with its fused prologue, or quant + GEMM)
tern_status bitlinear_any(bool gemv, const void* x, tern_dtype dt, int M, int K, const float* gain,
                          float eps, const tern_weight& w, const Epi& e, void* ws, const BlockWs& L,
                          cudaStream_t s, int norm) {
  if (gemv) {
    Prof pr(TERN_K_GEMV, e.kind, M, w.n_rows, K, w.n_seg, dt, s);
    TRY_CUDA(launch_gemv(x, dt, dt, M, K, K, gain, eps, w, e, nullptr, s, nullptr, 0, norm), "gemv");
    return TERN_OK;
  }
  return bl_tc(x, dt, M, K, K, gain, eps, w, dt, e, at<int8_t>(ws, L.q), kpad(K),
               at<float>(ws, L.deq), at<int32_t>(ws, L.qsum), nullptr, nullptr, s,
               at<int32_t>(ws, L.part), L.part_bytes, norm);
}

// gather the ranks' [M][cs] slices into full [M][world*cs] rows
tern_status shard_gather(const tern_shard& sh, const void* send, void* full, int M, int cs,
                         tern_dtype dt, void* ws, const BlockWs& L, cudaStream_t s) {
  const size_t bytes = (size_t)M * cs * dsize(dt);
  void* dst = M == 1 ? full : at<char>(ws, L.gbuf);
  const int rc = sh.ag(sh.ctx, send, dst, bytes, (tern_stream)s);
  if (rc != 0) return fail(TERN_ERR_CUDA, "all-gather callback failed (%d)", rc);
  if (M > 1) TRY_CUDA(launch_unshard(dst, dt, sh.world, M, cs, full, s), "unshard");
  return TERN_OK;
}

// f1(i): gather the next BitLinear's input as int8 codes (tern_shard.gather_q):
// x_r [M][cs] this rank's slice (activations) -> q [M][kpad(K)], deq, qsum
tern_status shard_gather_q(const tern_shard& sh, const void* x_r, int M, int cs, const float* gain,
                           float eps, int norm, tern_dtype dt, void* ws, const BlockWs& L,
                           cudaStream_t s) {
  const int world = sh.world, K = cs * world;
  double* stl = at<double>(ws, L.stl);
  const double* st[3] = {nullptr, nullptr, nullptr};
  const int rounds = slice_rounds(norm, gain != nullptr);
  for (int rnd = 0; rnd < rounds; ++rnd) {
    TRY_CUDA(launch_slice_stats(x_r, cs, M, cs, world, sh.rank, dt, gain, eps, norm, st, rnd, stl,
                                s),
             "slice stats");
    double* g = at<double>(ws, L.stg + (size_t)rnd * al256((size_t)world * M * 16));
    const int rc = sh.ag(sh.ctx, stl, g, (size_t)M * 16, (tern_stream)s);
    if (rc != 0) return fail(TERN_ERR_CUDA, "all-gather callback failed (%d)", rc);
    st[rnd] = g;
  }
  int8_t* send = at<int8_t>(ws, L.qsend);
  TRY_CUDA(launch_slice_quant(x_r, cs, M, cs, world, sh.rank, dt, gain, eps, norm, st, send, cs,
                              reinterpret_cast<int32_t*>(send + (size_t)M * cs),
                              at<float>(ws, L.deq), s),
           "slice quant");
  const size_t per = (size_t)M * cs + 4 * (size_t)M;
  const int rc = sh.ag(sh.ctx, send, at<int8_t>(ws, L.qgath), per, (tern_stream)s);
  if (rc != 0) return fail(TERN_ERR_CUDA, "all-gather callback failed (%d)", rc);
  TRY_CUDA(launch_unshard_q(at<int8_t>(ws, L.qgath), world, M, cs, at<int8_t>(ws, L.q), kpad(K),
                            at<int32_t>(ws, L.qsum), s),
           "unshard q");
  return TERN_OK;
}

// GEMM on the gathered codes (the quant already happened per slice)
tern_status gemm_q(int M, int K, const tern_weight& w, tern_dtype dt, const Epi& e, void* ws,
                   const BlockWs& L, cudaStream_t s) {
  Prof pr(TERN_K_GEMM, e.kind, M, w.n_rows, K, w.n_seg, dt, s);
  TRY_CUDA(launch_gemm(at<int8_t>(ws, L.q), M, kpad(K), at<float>(ws, L.deq),
                       at<int32_t>(ws, L.qsum), w, dt, e, s, at<int32_t>(ws, L.part), L.part_bytes),
           "gemm");
  return TERN_OK;
}

// f1(ii): a row-parallel BitLinear: x_r [M][cs] this rank's slice of the input
// -> moments exchanged, slice quantized, int32 partials of all n outputs
// (minus nothing: the q-sum partials ride along) -> all-reduce -> epilogue e
tern_status rowpar_bitlinear(const tern_shard& sh, const void* x_r, int M, int cs,
                             const float* gain, float eps, int norm, const tern_weight& w,
                             const Epi& e, tern_dtype dt, void* ws, const BlockWs& L,
                             cudaStream_t s) {
  const int world = sh.world, n = w.n_out;
  double* stl = at<double>(ws, L.stl);
  const double* st[3] = {nullptr, nullptr, nullptr};
  const int rounds = slice_rounds(norm, gain != nullptr);
  for (int rnd = 0; rnd < rounds; ++rnd) {
    TRY_CUDA(launch_slice_stats(x_r, cs, M, cs, world, sh.rank, dt, gain, eps, norm, st, rnd, stl,
                                s),
             "slice stats");
    double* g = at<double>(ws, L.stg + (size_t)rnd * al256((size_t)world * M * 16));
    const int rc = sh.ag(sh.ctx, stl, g, (size_t)M * 16, (tern_stream)s);
    if (rc != 0) return fail(TERN_ERR_CUDA, "all-gather callback failed (%d)", rc);
    st[rnd] = g;
  }
  int32_t* acc = at<int32_t>(ws, L.accb);        // [M][n] partials, then [M] q sums
  int32_t* qs_r = acc + (size_t)M * n;
  int8_t* q = at<int8_t>(ws, L.q);
  TRY_CUDA(launch_slice_quant(x_r, cs, M, cs, world, sh.rank, dt, gain, eps, norm, st, q, kpad(cs),
                              qs_r, at<float>(ws, L.deq), s),
           "slice quant");
  int ks = 1;   // one K slice: the partials go straight to the all-reduce
  {
    Prof pr(TERN_K_GEMM, EPI_NONE, M, w.n_rows, cs, 1, dt, s);
    Epi ge = make_epi(EPI_NONE, w, nullptr, nullptr, 0);
    TRY_CUDA(launch_gemm(q, M, kpad(cs), at<float>(ws, L.deq), qs_r, w, dt, ge, s, acc,
                         (size_t)M * n * 4, &ks),
             "gemm (row-parallel partials)");
  }
  const int rc = sh.ar(sh.ctx, acc, acc, (size_t)M * n + (size_t)M, (tern_stream)s);
  if (rc != 0) return fail(TERN_ERR_CUDA, "all-reduce callback failed (%d)", rc);
  TRY_CUDA(launch_splitk_epi(acc, 1, M, n, at<float>(ws, L.deq), qs_r, e, dt, s), "epilogue");
  return TERN_OK;
}

// a8 with output-feature sharding (tern.h tern_shard): 4 gathers per block
tern_status run_block_sharded(const tern_block& b, const void* x, void* y, tern_dtype dt, int B,
                              int T, float* h, void* ws, const BlockWs& L, cudaStream_t s) {
  const tern_shard& sh = b.shard;
  const int M = B * T, d = b.d, l = b.l, ds = d / sh.world, ls = l / sh.world;
  const size_t es = dsize(dt);
  const tern_mlgru& mx = b.mix;
  const tern_glu& gl = b.ch;
  const bool gv = T == 1 && B <= g_gemv_max_m && gemv_supported(B, d, dt) &&
                  gemv_supported(B, l, dt);
  void* sout = at<char>(ws, L.sout);
  void* op = at<char>(ws, L.oprime);
  void* x1 = at<char>(ws, L.x1);
  void* pf = at<char>(ws, L.p);
  tern_status st;
  // token mixer on this rank's channels: f, c, g -> (scan) -> o'_r
  if (gv) {
    Epi e1 = make_epi(EPI_MLGRU, mx.fcg, mx.bias_fcg, sout, ds);
    e1.h = h;
    e1.gate = mx.gate;
    if ((st = bitlinear_any(true, x, dt, M, d, mx.gain_x, mx.eps, mx.fcg, e1, ws, L, s, mx.norm))) return st;
  } else {
    void* fcg = at<char>(ws, L.fcg);
    Epi e1 = make_epi(EPI_FCG, mx.fcg, mx.bias_fcg, fcg, mx.fcg.n_rows);
    if ((st = bitlinear_any(false, x, dt, M, d, mx.gain_x, mx.eps, mx.fcg, e1, ws, L, s, mx.norm))) return st;
    Prof pr(TERN_K_SCAN, mx.gate, M, ds, ds, 3, dt, s);
    TRY_CUDA(launch_scan(fcg, dt, B, T, ds, mx.gate, h, sout, s), "scan");
  }
  if (sh.megatron) {
    // f1(ii): o and down row-parallel; o' and p never leave the rank, x1 and y
    // are produced whole on every rank by the all-reduced epilogues
    if ((st = rowpar_bitlinear(sh, sout, M, ds, mx.gain_o, mx.eps, mx.norm, mx.o,
                               [&] {
                                 Epi e2 = make_epi(EPI_RESID, mx.o, mx.bias_o, x1, d);
                                 e2.res = x;
                                 e2.ldr = d;
                                 return e2;
                               }(),
                               dt, ws, L, s)))
      return st;
    Epi e3 = make_epi(EPI_SWIGLU, gl.gu, nullptr, sout, ls);
    if ((st = bitlinear_any(false, x1, dt, M, d, gl.gain_x, gl.eps, gl.gu, e3, ws, L, s, gl.norm)))
      return st;
    Epi e4 = make_epi(EPI_RESID, gl.down, nullptr, y, d);
    e4.res = x1;
    e4.ldr = d;
    return rowpar_bitlinear(sh, sout, M, ls, gl.gain_p, gl.eps, gl.norm, gl.down, e4, dt, ws, L, s);
  }
  if (sh.gather_q && !gv) {
    // f1(i): o', x1 and p cross the ranks as int8 codes; x1 stays a local slice
    void* x1r = x1;   // [M][ds]
    if ((st = shard_gather_q(sh, sout, M, ds, mx.gain_o, mx.eps, mx.norm, dt, ws, L, s))) return st;
    Epi e2 = make_epi(EPI_RESID, mx.o, mx.bias_o, x1r, ds);
    e2.res = static_cast<const char*>(x) + (size_t)sh.rank * ds * es;
    e2.ldr = d;
    if ((st = gemm_q(M, d, mx.o, dt, e2, ws, L, s))) return st;
    if ((st = shard_gather_q(sh, x1r, M, ds, gl.gain_x, gl.eps, gl.norm, dt, ws, L, s))) return st;
    Epi e3 = make_epi(EPI_SWIGLU, gl.gu, nullptr, sout, ls);
    if ((st = gemm_q(M, d, gl.gu, dt, e3, ws, L, s))) return st;
    if ((st = shard_gather_q(sh, sout, M, ls, gl.gain_p, gl.eps, gl.norm, dt, ws, L, s))) return st;
    Epi e4 = make_epi(EPI_RESID, gl.down, nullptr, sout, ds);
    e4.res = x1r;
    e4.ldr = ds;
    if ((st = gemm_q(M, l, gl.down, dt, e4, ws, L, s))) return st;
    return shard_gather(sh, sout, y, M, ds, dt, ws, L, s);
  }
  if ((st = shard_gather(sh, sout, op, M, ds, dt, ws, L, s))) return st;
  // o: x1_r = x[:, r] + o'(*)W_o[r]
  Epi e2 = make_epi(EPI_RESID, mx.o, mx.bias_o, sout, ds);
  e2.res = static_cast<const char*>(x) + (size_t)sh.rank * ds * es;
  e2.ldr = d;
  if ((st = bitlinear_any(gv, op, dt, M, d, mx.gain_o, mx.eps, mx.o, e2, ws, L, s, mx.norm))) return st;
  if ((st = shard_gather(sh, sout, x1, M, ds, dt, ws, L, s))) return st;
  // channel mixer: p_r = SiLU(g_r) u_r, then y_r = x1[:, r] + p(*)W_d[r]
  Epi e3 = make_epi(EPI_SWIGLU, gl.gu, nullptr, sout, ls);
  if ((st = bitlinear_any(gv, x1, dt, M, d, gl.gain_x, gl.eps, gl.gu, e3, ws, L, s, gl.norm))) return st;
  if ((st = shard_gather(sh, sout, pf, M, ls, dt, ws, L, s))) return st;
  Epi e4 = make_epi(EPI_RESID, gl.down, nullptr, sout, ds);
  e4.res = static_cast<const char*>(x1) + (size_t)sh.rank * ds * es;
  e4.ldr = d;
  if ((st = bitlinear_any(gv, pf, dt, M, l, gl.gain_p, gl.eps, gl.down, e4, ws, L, s, gl.norm))) return st;
  return shard_gather(sh, sout, y, M, ds, dt, ws, L, s);
}

// a8 decode step for gemv_max_m < B <= kSplitKMaxM: per BitLinear one split-K
// tcgen05 GEMM writing int32 partials and one row-wise finalize (k_fin.cu) that
// applies the epilogue and quantizes its output row for the next BitLinear, so
// only the block input needs a quant launch (9 launches per block)
bool batched_decode_ok(const tern_block& b, int B, int T, const BlockWs& L) {
  return T == 1 && B > g_gemv_max_m && B <= kSplitKMaxM && L.part_bytes > 0 &&
         fin_supported(b.d) && fin_supported(b.l) && g_batched_fin;
}

tern_status run_block_decode_batched(const tern_block& b, const void* x, void* y, tern_dtype dt,
                                     int B, float* h, void* ws, const BlockWs& L, cudaStream_t s) {
  const int d = b.d, l = b.l;
  const tern_mlgru& mx = b.mix;
  const tern_glu& gl = b.ch;
  int8_t* q = at<int8_t>(ws, L.q);
  float* deq = at<float>(ws, L.deq);
  int32_t* qsum = at<int32_t>(ws, L.qsum);
  int32_t* part = at<int32_t>(ws, L.part);
  void* op = at<char>(ws, L.oprime);
  void* x1 = at<char>(ws, L.x1);
  void* pp = at<char>(ws, L.p);
  {
    Prof pr(TERN_K_QUANT, 0, B, 0, d, 0, dt, s);
    TRY_CUDA(launch_quant(x, dt, B, d, d, mx.gain_x, mx.eps, q, kpad(d), deq, qsum, nullptr,
                          nullptr, s, mx.norm),
             "quant");
  }
  // one phase: GEMM partials, then finalize (+ the next BitLinear's quant)
  auto phase = [&](const tern_weight& w, int K, const Epi& e, const float* ngain, float neps,
                   bool nquant, int nnorm) -> tern_status {
    int ks = 1;
    {
      Prof pr(TERN_K_GEMM, EPI_NONE, B, w.n_rows, K, w.n_seg, dt, s);
      Epi ge = make_epi(EPI_NONE, w, nullptr, nullptr, 0);
      TRY_CUDA(launch_gemm(q, B, kpad(K), deq, qsum, w, dt, ge, s, part, L.part_bytes, &ks),
               "gemm (partials)");
    }
    Prof pr(TERN_K_FIN, e.kind, B, w.n_rows, K, w.n_seg, dt, s);
    TRY_CUDA(launch_fin(part, ks, B, w.n_rows, deq, qsum, e, dt, ngain, neps,
                        nquant ? q : nullptr, kpad(e.n_out), deq, qsum, s, nnorm),
             "finalize");
    return TERN_OK;
  };
  tern_status st;
  Epi e1 = make_epi(EPI_MLGRU, mx.fcg, mx.bias_fcg, op, d);
  e1.h = h;
  e1.gate = mx.gate;
  if ((st = phase(mx.fcg, d, e1, mx.gain_o, mx.eps, true, mx.norm))) return st;
  Epi e2 = make_epi(EPI_RESID, mx.o, mx.bias_o, x1, d);
  e2.res = x;
  e2.ldr = d;
  if ((st = phase(mx.o, d, e2, gl.gain_x, gl.eps, true, gl.norm))) return st;
  Epi e3 = make_epi(EPI_SWIGLU, gl.gu, nullptr, pp, l);
  if ((st = phase(gl.gu, d, e3, gl.gain_p, gl.eps, true, gl.norm))) return st;
  Epi e4 = make_epi(EPI_RESID, gl.down, nullptr, y, d);
  e4.res = x1;
  e4.ldr = d;
  return phase(gl.down, l, e4, nullptr, 0.0f, false, TERN_NORM_RMS);
}

tern_status check_act(const void* x, const void* y, const void* ws, size_t ws_bytes, size_t need,
                      tern_dtype dt, const char* name) {
  CHECK(x && y, "%s: null x/y", name);
  CHECK(aligned16(x) && aligned16(y), "%s: x/y not 16-byte aligned", name);
  CHECK(x != y, "%s: y must not alias x", name);
  CHECK(valid_dt(dt), "%s: bad dtype", name);
  CHECK(ws && aligned16(ws) && ws_bytes >= need, "%s: workspace too small (%zu < %zu)", name,
        ws_bytes, need);
  return TERN_OK;
}

}  // namespace

int32_t tern_mlgru_chunks(const tern_mlgru* p, int32_t B, int32_t T, int32_t d) {
  if (!p || B < 1 || T < 2 || d < 1) return 1;
  if (p->num_chunks != 0 && p->num_chunks != 1 && p->num_chunks != 4 && p->num_chunks != 8)
    return 0;
  return tern::scan_chunks_resolve(p->num_chunks, B, T, d);
}

tern_status mlgru_fwd(const tern_mlgru* p, const void* x, void* out, tern_dtype dt, int32_t B,
                      int32_t T, int32_t d, float* h, void* ws, size_t ws_bytes,
                      tern_stream stream) {
  CHECK(p, "mlgru_fwd: null params");
  CHECK(B >= 0 && T >= 0 && d > 0 && d % 64 == 0, "mlgru_fwd: B=%d T=%d d=%d", B, T, d);
  if (B * T == 0) return TERN_OK;   // no tokens: a no-op
  CHECK(h, "mlgru_fwd: null state");
  tern_status st;
  if ((st = check_weight(&p->fcg, d, 3, "fcg")) != TERN_OK) return st;
  if ((st = check_weight(&p->o, d, 1, "o")) != TERN_OK) return st;
  CHECK(p->fcg.n_out == d && p->o.n_out == d, "mlgru_fwd: weights must be d x d");
  CHECK(p->eps > 0, "mlgru_fwd: eps");
  CHECK(p->norm == TERN_NORM_RMS || p->norm == TERN_NORM_CENTERED, "mlgru_fwd: bad norm mode");
  if (p->num_chunks != 0 && p->num_chunks != 1 && p->num_chunks != 4 && p->num_chunks != 8)
    return fail(TERN_ERR_UNSUPPORTED, "mlgru_fwd: num_chunks=%d (0, 1, 4 or 8)", p->num_chunks);
  BlockWs L = block_ws(B * T, d, 0, p->fcg.n_rows, dt);
  if ((st = check_act(x, out, ws, ws_bytes, L.total, dt, "mlgru_fwd")) != TERN_OK) return st;
  if ((st = check_device()) != TERN_OK) return st;
  if (B * T == 0) return TERN_OK;
  return run_mlgru(*p, x, out, false, dt, B, T, d, h, ws, L, (cudaStream_t)stream);
}

tern_status glu_fwd(const tern_glu* p, const void* x, void* out, tern_dtype dt, int32_t m,
                    int32_t d, int32_t l, void* ws, size_t ws_bytes, tern_stream stream) {
  CHECK(p, "glu_fwd: null params");
  CHECK(m >= 0 && d > 0 && d % 16 == 0 && l > 0 && l % 16 == 0, "glu_fwd: m=%d d=%d l=%d", m, d, l);
  if (m == 0) return TERN_OK;   // no tokens: a no-op
  tern_status st;
  if ((st = check_weight(&p->gu, d, 2, "gate|up")) != TERN_OK) return st;
  if ((st = check_weight(&p->down, l, 1, "down")) != TERN_OK) return st;
  CHECK(p->gu.n_out == l && p->down.n_out == d, "glu_fwd: weights must be d->l, l->d");
  CHECK(p->eps > 0, "glu_fwd: eps");
  CHECK(p->norm == TERN_NORM_RMS || p->norm == TERN_NORM_CENTERED, "glu_fwd: bad norm mode");
  BlockWs L = block_ws(m, d, l, 0, dt);
  if ((st = check_act(x, out, ws, ws_bytes, L.total, dt, "glu_fwd")) != TERN_OK) return st;
  if ((st = check_device()) != TERN_OK) return st;
  if (m == 0) return TERN_OK;
  return run_glu(*p, x, out, false, dt, m, d, l, ws, L, (cudaStream_t)stream);
}

static tern_status block_run(const tern_block* b, const void* x, void* y, tern_dtype dt, int32_t B,
                             int32_t T, float* h, void* ws, size_t ws_bytes, tern_stream stream,
                             const char* name) {
  tern_status st = check_block(b);
  if (st) return st;
  CHECK(B >= 0 && T >= 0, "%s: B=%d T=%d", name, B, T);
  CHECK(valid_dt(dt), "%s: bad dtype", name);
  if (B * T == 0) return TERN_OK;   // no tokens: a no-op (buffers may be empty / NULL)
  CHECK(h, "%s: null state", name);
  BlockWs L = block_ws(B * T, b->d, b->l, b->mix.fcg.n_rows, dt, block_world(b),
                   b->shard.megatron != 0);
  if ((st = check_act(x, y, ws, ws_bytes, L.total, dt, name)) != TERN_OK) return st;
  if ((st = check_device()) != TERN_OK) return st;
  if (B * T == 0) return TERN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (block_world(b) > 1) return run_block_sharded(*b, x, y, dt, B, T, h, ws, L, s);
  if (batched_decode_ok(*b, B, T, L)) return run_block_decode_batched(*b, x, y, dt, B, h, ws, L, s);
  void* x1 = at<char>(ws, L.x1);
  // weight-stream prefetch (decode GEMVs): the token mixer pulls this block's
  // channel-mixer weights into L2, the channel mixer the next block's token mixer
  PfPlan pm, pg;
  if (T == 1) {
    pm.p[0] = b->ch.gu.codes;
    pm.n[0] = codes_bytes(b->ch.gu);
    pm.p[1] = b->ch.down.codes;
    pm.n[1] = codes_bytes(b->ch.down);
    if (b->next_block) {
      const tern_block* nb = static_cast<const tern_block*>(b->next_block);
      pg.p[0] = nb->mix.fcg.codes;
      pg.n[0] = codes_bytes(nb->mix.fcg);
      pg.p[1] = nb->mix.o.codes;
      pg.n[1] = codes_bytes(nb->mix.o);
    }
  }
  // fp32 prefill on the tensor-core path: x1 goes into y and the down projection is added
  // onto it in place (EPI_RESID_RED)
  const bool red = g_resid_red && dt == TERN_F32 && T > 1 && B * T > kSplitKMaxM &&
                   b->mix.norm == TERN_NORM_RMS;
  if (red) x1 = y;
  if ((st = run_mlgru(b->mix, x, x1, true, dt, B, T, b->d, h, ws, L, s, pm)) != TERN_OK) return st;
  // prefill: the token mixer's quant of x zeroed the gate|up counters (QFuse)
  return run_glu(b->ch, x1, y, true, dt, B * T, b->d, b->l, ws, L, s, pg, T > 1, red);
}

// ---------------------------------------------------------------- sequence-parallel prefill
static size_t sp_extra(int B, int d, int world) {
  return al256((size_t)2 * B * d * 4) + al256((size_t)world * 2 * B * d * 4) +
         al256((size_t)B * d * 4);
}

size_t tern_block_prefill_sp_workspace(const tern_block* b, int32_t B, int32_t T_local,
                                       tern_dtype dt, int32_t world) {
  if (!b || B < 0 || T_local < 0 || world < 1) return 0;
  return block_ws(B * (T_local > 0 ? T_local : 1), b->d, b->l, b->mix.fcg.n_rows, dt).total +
         sp_extra(B, b->d, world);
}

tern_status block_prefill_sp(const tern_block* b, const void* x, void* y, tern_dtype dt,
                             int32_t B, int32_t T_local, float* h, const tern_seqpar* sp,
                             void* ws, size_t ws_bytes, tern_stream stream) {
  tern_status st = check_block(b);
  if (st) return st;
  CHECK(sp && sp->ag, "block_prefill_sp: null seqpar / all-gather");
  CHECK(sp->world >= 1 && sp->rank >= 0 && sp->rank < sp->world, "block_prefill_sp: rank %d of %d",
        sp->rank, sp->world);
  CHECK(block_world(b) == 1, "block_prefill_sp: the block must not be output-sharded");
  CHECK(B >= 1 && T_local >= 0, "block_prefill_sp: B=%d T_local=%d", B, T_local);
  CHECK(valid_dt(dt), "block_prefill_sp: bad dtype");
  CHECK(h && ws && aligned16(ws), "block_prefill_sp: null state or unaligned workspace");
  const int Tq = T_local > 0 ? T_local : 1;
  BlockWs L = block_ws(B * Tq, b->d, b->l, b->mix.fcg.n_rows, dt);
  const size_t need = L.total + sp_extra(B, b->d, sp->world);
  CHECK(ws_bytes >= need, "block_prefill_sp: workspace %zu < %zu", ws_bytes, need);
  if (T_local > 0) {
    CHECK(x && y && aligned16(x) && aligned16(y), "block_prefill_sp: x / y null or unaligned");
  }
  if ((st = check_device()) != TERN_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  SeqPar P;
  P.rank = sp->rank;
  P.world = sp->world;
  P.ag = sp->ag;
  P.ctx = sp->ctx;
  char* base = static_cast<char*>(ws) + L.total;
  P.send = reinterpret_cast<float*>(base);
  P.recv = reinterpret_cast<float*>(base + al256((size_t)2 * B * b->d * 4));
  P.hfin = reinterpret_cast<float*>(base + al256((size_t)2 * B * b->d * 4) +
                                    al256((size_t)sp->world * 2 * B * b->d * 4));
  void* x1 = at<char>(ws, L.x1);
  if ((st = run_mlgru(b->mix, x, x1, true, dt, B, T_local, b->d, h, ws, L, s, PfPlan(), &P)) !=
      TERN_OK)
    return st;
  if (T_local == 0) return TERN_OK;
  return run_glu(b->ch, x1, y, true, dt, B * T_local, b->d, b->l, ws, L, s);
}

tern_status block_prefill(const tern_block* b, const void* x, void* y, tern_dtype dt, int32_t B,
                          int32_t T, float* h, void* ws, size_t ws_bytes, tern_stream stream) {
  return block_run(b, x, y, dt, B, T, h, ws, ws_bytes, stream, "block_prefill");
}

tern_status block_decode(const tern_block* b, const void* x, void* y, tern_dtype dt, int32_t B,
                         float* h, void* ws, size_t ws_bytes, tern_stream stream) {
  return block_run(b, x, y, dt, B, 1, h, ws, ws_bytes, stream, "block_decode");
}

// ----------------------------------------------------------------- f2: stack decode
namespace {
struct StackWs {
  size_t bar, a, x1, p, xb, total;
};
StackWs stack_ws(int B, int d, int l, tern_dtype dt) {
  StackWs w{};
  size_t off = 0;
  w.bar = off; off += al256((64 + 1024) * 4);   // grid barrier counter + per-CTA flags
  w.a = off; off += al256((size_t)B * d * dsize(dt));    // o'
  w.x1 = off; off += al256((size_t)B * d * dsize(dt));   // x1 = x + o
  w.p = off; off += al256((size_t)B * l * dsize(dt));    // p = SiLU(g) u
  w.xb = off; off += al256((size_t)B * d * dsize(dt));   // block outputs between blocks
  w.total = off;
  return w;
}

// the 4 phases of every block; buffers: a block's input is x (block 0) or xb,
// its output xb (y for the last); xb can be both because the down phase that
// overwrites it runs two grid barriers after its last reader (the o phase)
std::vector<StackPhaseDesc> stack_phases(const tern_block* blocks, int L, const void* x, void* y,
                                         float* const* h, void* ws, const StackWs& W) {
  std::vector<StackPhaseDesc> ph;
  ph.reserve((size_t)4 * L);
  void* a = at<char>(ws, W.a);
  void* x1 = at<char>(ws, W.x1);
  void* p = at<char>(ws, W.p);
  void* xb = at<char>(ws, W.xb);
  for (int i = 0; i < L; ++i) {
    const tern_block& b = blocks[i];
    const void* xin = i == 0 ? x : xb;
    void* xout = i == L - 1 ? y : xb;
    StackPhaseDesc f{xin, nullptr, a, h[i], b.mix.fcg, b.mix.gain_x, b.mix.bias_fcg, b.mix.eps,
                     EPI_MLGRU, (int)b.mix.gate, b.d, (int)b.mix.norm};
    StackPhaseDesc o{a, xin, x1, nullptr, b.mix.o, b.mix.gain_o, b.mix.bias_o, b.mix.eps,
                     EPI_RESID, 0, b.d, (int)b.mix.norm};
    StackPhaseDesc g{x1, nullptr, p, nullptr, b.ch.gu, b.ch.gain_x, nullptr, b.ch.eps,
                     EPI_SWIGLU, 0, b.d, (int)b.ch.norm};
    StackPhaseDesc dn{p, x1, xout, nullptr, b.ch.down, b.ch.gain_p, nullptr, b.ch.eps,
                      EPI_RESID, 0, b.l, (int)b.ch.norm};
    ph.push_back(f);
    ph.push_back(o);
    ph.push_back(g);
    ph.push_back(dn);
  }
  return ph;
}

tern_status check_stack(const tern_block* blocks, int32_t L, int32_t B, tern_dtype dt,
                        const char* name) {
  CHECK(blocks && L > 0, "%s: null blocks or L=%d", name, L);
  CHECK(B >= 0, "%s: B=%d", name, B);
  CHECK(valid_dt(dt), "%s: bad dtype", name);
  tern_status st;
  for (int i = 0; i < L; ++i) {
    if ((st = check_block(&blocks[i])) != TERN_OK) return st;
    CHECK(blocks[i].d == blocks[0].d && blocks[i].l == blocks[0].l, "%s: block %d widths differ",
          name, i);
  }
  return TERN_OK;
}
}  // namespace

size_t tern_stack_decode_workspace(const tern_block* blocks, int32_t L, int32_t B, tern_dtype dt) {
  if (!blocks || L <= 0 || B < 0) return 0;
  return stack_ws(B, blocks[0].d, blocks[0].l, dt).total;
}

tern_status stack_decode(const tern_block* blocks, int32_t L, const void* x, void* y,
                         tern_dtype dt, int32_t B, float* const* h, void* ws, size_t ws_bytes,
                         tern_stream stream) {
  tern_status st = check_stack(blocks, L, B, dt, "stack_decode");
  if (st) return st;
  if (B == 0) return TERN_OK;   // no tokens: a no-op
  CHECK(h, "stack_decode: null state array");
  for (int i = 0; i < L; ++i) CHECK(h[i], "stack_decode: null state of block %d", i);
  const StackWs W = stack_ws(B, blocks[0].d, blocks[0].l, dt);
  if ((st = check_act(x, y, ws, ws_bytes, W.total, dt, "stack_decode")) != TERN_OK) return st;
  for (int i = 0; i < L; ++i)
    if (block_world(&blocks[i]) > 1)
      return fail(TERN_ERR_UNSUPPORTED, "stack_decode: block %d is sharded", i);
  if ((st = check_device()) != TERN_OK) return st;
  std::vector<StackPhaseDesc> ph = stack_phases(blocks, L, x, y, h, ws, W);
  if (!stack_decode_plan(ph.data(), (int)ph.size(), B, dt, nullptr))
    return fail(TERN_ERR_UNSUPPORTED, "stack_decode: B=%d d=%d l=%d outside the persistent plan", B,
                blocks[0].d, blocks[0].l);
  Prof pr(TERN_K_STACK, 0, B, L, blocks[0].d, 0, dt, (cudaStream_t)stream);
  TRY_CUDA(launch_stack_decode(ph.data(), (int)ph.size(), B, dt, at<unsigned>(ws, W.bar),
                               (cudaStream_t)stream),
           "stack_decode");
  return TERN_OK;
}

}  // extern "C"
