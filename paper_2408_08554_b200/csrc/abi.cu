// abi.cu -- the C-ABI (include/abq_cuda.h): argument validation in the
// reference's order and wording, error state, and dispatch to the sm_100a
// kernels.  No CPU compute path exists here: every numeric result is produced
// by a CUDA kernel; if the device is missing the call fails with ABQ_ERR_CUDA.
#include <algorithm>
#include <climits>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace abq_dev {

// ---- state -----------------------------------------------------------------
std::string& last_error() {
  static thread_local std::string s;
  return s;
}

int fail(int status, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  last_error() = buf;
  return status;
}

uint64_t& launch_counter() {
  static thread_local uint64_t n = 0;
  return n;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

// per-thread, per-device scratch for synchronous status reporting
static unsigned long long* scratch_words() {
  static thread_local unsigned long long* ptr[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!ptr[dev]) {
    if (cudaMalloc(&ptr[dev], 8 * sizeof(unsigned long long)) != cudaSuccess) {
      cudaGetLastError();
      ptr[dev] = nullptr;
    }
  }
  return ptr[dev];
}

static int g_gemv_variant = ABQ_GEMV_AUTO;

// ---- kernels implemented in the other translation units --------------------
int run_quantize(const void* x, int x_dtype, size_t rows, size_t cols, const QuantParams& qp,
                 const double* ca, const double* cb, uint8_t* codes, uint64_t* planes,
                 unsigned nplanes, double* scales, int32_t* zps, int64_t* rowsums,
                 unsigned long long* bad, unsigned long long* range, cudaStream_t st);
int run_bitpack(const uint8_t* codes, size_t rows, size_t cols, unsigned bits, uint64_t* planes,
                unsigned long long* bad, cudaStream_t st);
int run_unpack(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, uint8_t* codes,
               cudaStream_t st);
int run_code_rowsums(const uint8_t* codes, size_t rows, size_t cols, int64_t* out, cudaStream_t st);
int run_dequantize(const uint8_t* codes, size_t rows, size_t cols, const double* scales, const int32_t* zps,
                   int per_tensor, double* out, cudaStream_t st);
int run_plane_rowsums(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, int64_t* out,
                      cudaStream_t st);
template <typename Acc>
int run_zero_point_correct(const Acc* acc, size_t m, size_t n, const int64_t* ra, const int64_t* cb,
                           const int32_t* za, const int32_t* zb, size_t k, Acc* out, cudaStream_t st);
int run_bmma(const uint64_t* a, size_t m, unsigned a_plane, const uint64_t* bt, size_t n,
             unsigned b_plane, size_t k, int32_t* out, cudaStream_t st);
int run_gemm_popc(const uint64_t* A, unsigned p, size_t m, const uint64_t* W, unsigned q, size_t n,
                  size_t k, bool wide, const EpiParams& e, cudaStream_t st, int token_tile = 0);
size_t frag_words(unsigned q, size_t n, size_t k);
size_t imma_ws_bytes(size_t n, size_t k);
bool imma_supported(size_t m, size_t k);
bool dec_supported(unsigned q, size_t n, size_t k, size_t m);
int run_gemv_dec_qact(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m, const uint32_t* codes,
                      const double* s_a, const int32_t* z_a, const long long* rowsum, const QuantParams& qp,
                      const EpiParams& e, cudaStream_t st, const DecNext* nx);
size_t qact_codes_bytes(size_t m, size_t k);
int run_stage_in(void* dst, const void* src, size_t bytes, cudaStream_t st);
bool qact_supported(size_t m, size_t k);
int run_rmsnorm_quant(const __half* x, const __half* gain, float eps, size_t m, size_t k, const QuantParams& qp,
                      __half* y_out, uint32_t* codes, double* s_a, int32_t* z_a, long long* rowsum,
                      unsigned long long* err, cudaStream_t st);
int run_silu_mul_quant(const __half* gate, const __half* up, size_t m, size_t k, const QuantParams& qp,
                       __half* y_out, uint32_t* codes, double* s_a, int32_t* z_a, long long* rowsum,
                       unsigned long long* err, cudaStream_t st);
unsigned long long*& trace_buffer();
int run_prepack_frag(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* frag,
                     cudaStream_t st);
int run_gemv_imma_planes(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m,
                         const uint64_t* a_planes, unsigned p, const EpiParams& e, cudaStream_t st);
int run_gemv_dec(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m, const void* x, int x_dtype,
                 const QuantParams& qp, const EpiParams& e, void* ws, unsigned long long* bad_out,
                 cudaStream_t st, const DecNext* nx);

// successor-layer hint of a weights block (abq_weights.next), for the decode GEMV
static const DecNext* next_of(const abq_weights* w, DecNext* buf) {
  const abq_weights* n = w->next;
  if (!n || !n->frag || n->q < 1 || n->q > 8 || n->n == 0 || n->k == 0) return nullptr;
  *buf = DecNext{n->frag, n->q, n->n, n->k};
  return buf;
}

int run_gemm_bmma(const uint64_t* a, unsigned p, size_t m, const uint64_t* w, unsigned q, size_t n, size_t k,
                  int32_t* out, cudaStream_t st);
size_t tc_words(unsigned q, size_t n, size_t k);
int run_prepack_tc(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* out,
                   cudaStream_t st);
bool gemm_tc_supported(size_t k);
int run_gemm_tc(const uint32_t* wtc, unsigned q, size_t n, size_t k, const uint8_t* act, size_t m,
                const EpiParams& e, cudaStream_t st, unsigned long long* bad_word = nullptr,
                unsigned long long* bad_out = nullptr, bool pdl = false, unsigned* sk_flags = nullptr,
                uint32_t* sk_part = nullptr, EnginePlan plan = EnginePlan{0, 0});
size_t tc_sk_flag_bytes(size_t n, size_t k);
int& gemm_schedule();
size_t tc_sk_part_bytes(size_t m, size_t n, size_t k);
int run_tile_codes(const uint8_t* src, size_t m, size_t k, uint8_t* dst, cudaStream_t st);
int run_act_quant(const void* x, int x_dtype, size_t m, size_t k, int mt, const QuantParams& qp,
                  uint32_t* out, int row_ld, double* s_a, int32_t* z_a, long long* rowsum,
                  unsigned long long* bad_word, cudaStream_t st);

// decode GEMV on the tensor pipe: weights prepacked, M <= 8 tokens.  API path
// (activation planes given, abq_linear_planes): gemv_imma_kernel
static bool use_imma(const abq_weights* w, size_t m, size_t k) {
  return w->frag != nullptr && m >= 1 && m <= 8 && imma_supported(m, k) &&
         g_gemv_variant != ABQ_GEMV_POPC;
}
// serving path (abq_linear, activations quantized on the fly): gemv_dec_kernel
static bool use_dec(const abq_weights* w, size_t m, size_t k) {
  return w->frag != nullptr && dec_supported(w->q, w->n, k, m) && g_gemv_variant != ABQ_GEMV_POPC;
}
// prefill GEMM on tcgen05: weights prepacked (tc planes), M >= 9 tokens
// (prefill-only weights -- no frag layout resident -- serve small m here too)
static bool use_tc(const abq_weights* w, size_t m, size_t k, bool wide) {
  return w->tc != nullptr && (m >= 9 || w->frag == nullptr) && !wide && gemm_tc_supported(k) &&
         g_gemv_variant != ABQ_GEMV_POPC;
}

// ---- shared validation -----------------------------------------------------
static bool fits_int32_host(unsigned p, unsigned q, size_t k) {
  unsigned log_k = 0;
  while ((size_t{1} << log_k) < k + 1) ++log_k;
  return p + q + log_k <= 31;
}

static bool tile_valid_host(const abq_tile_config& t, unsigned p, unsigned q) {
  if (t.WK != 128) return false;
  if (t.BK != 128 && t.BK != 256 && t.BK != 384 && t.BK != 512) return false;
  if (t.BK % t.WK != 0) return false;
  if (t.BM == 0 || t.BN == 0 || t.WM == 0 || t.WN == 0) return false;
  if (t.WM % 8 != 0 || t.WN % 8 != 0) return false;
  const double warps = (double(t.BM) * p / double(t.WM)) * (double(t.BN) * q / double(t.WN));
  return warps >= 1.0 && warps <= 32.0;
}

static unsigned levels_of(const abq_quant_spec& s) {
  return s.scheme == ABQ_BALANCED ? (1u << s.bits) + 1u : (1u << s.bits);
}
static unsigned planes_of(const abq_quant_spec& s) {
  const unsigned L = levels_of(s);
  unsigned p = 0;
  while ((1u << p) < L) ++p;
  return p;
}

// QuantSpec::validate (quantizer.hpp:61-70) + passthrough rejection (quantizer.hpp:150)
static int validate_spec(const abq_quant_spec* s) {
  if (!s) return fail(ABQ_ERR_VALUE, "quantize: null QuantSpec");
  const bool passthrough = s->bits >= 16;
  if (s->bits < 1 || (s->bits > 8 && !passthrough))
    return fail(ABQ_ERR_VALUE, "QuantSpec: bits must be in [1,8] (or >=16 for passthrough)");
  if (s->scheme == ABQ_BALANCED && s->bits > 7 && !passthrough)
    return fail(ABQ_ERR_VALUE,
                "QuantSpec: balanced codes reach 2^bits and must fit one byte, so bits <= 7");
  if (!(s->alpha > 0.0 && s->alpha <= 1.0)) return fail(ABQ_ERR_VALUE, "QuantSpec: alpha must be in (0,1]");
  if (!(s->beta > 0.0 && s->beta <= 1.0)) return fail(ABQ_ERR_VALUE, "QuantSpec: beta must be in (0,1]");
  if (s->scheme < 0 || s->scheme > 2) return fail(ABQ_ERR_VALUE, "QuantSpec: unknown scheme");
  if (s->granularity < 0 || s->granularity > 2) return fail(ABQ_ERR_VALUE, "QuantSpec: unknown granularity");
  if (passthrough) return fail(ABQ_ERR_VALUE, "quantize: passthrough spec cannot be materialized");
  return ABQ_OK;
}

static QuantParams params_of(const abq_quant_spec& s) {
  QuantParams qp;
  qp.bits = s.bits;
  qp.scheme = s.scheme;
  qp.per_tensor = s.granularity == ABQ_PER_TENSOR;
  qp.alpha = s.alpha;
  qp.beta = s.beta;
  qp.levels = levels_of(s);
  return qp;
}

static int check_device() {
  static thread_local bool ok = false;  // a device, once seen, stays
  if (ok) return ABQ_OK;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(ABQ_ERR_CUDA, "abq: no CUDA device available (%s); the engine has no CPU path",
                cudaGetErrorString(e));
  }
  ok = true;
  return ABQ_OK;
}

static int sync_read(unsigned long long* dev_word, cudaStream_t st, unsigned long long* out) {
  ABQ_CUDA_TRY(cudaMemcpyAsync(out, dev_word, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  ABQ_CUDA_TRY(cudaStreamSynchronize(st));
  return ABQ_OK;
}

static void add_stats(abq_gemm_stats* stats, const abq_tile_config& t, size_t m, size_t n,
                      unsigned p, unsigned q) {
  if (!stats) return;
  // gemm.hpp:108-115: one block tile per (BM rows, BN cols); p*q plane pairs per tile
  const uint64_t tiles = uint64_t((m + t.BM - 1) / t.BM) * uint64_t((n + t.BN - 1) / t.BN);
  stats->block_tiles += tiles;
  stats->plane_pair_products += tiles * p * q;
}

// tcgen05 GEMM from packed activation planes: recombine the activation planes
// to u8 codes (unpack kernel), tile them into the GEMM operand layout and,
// when no tc-layout weights are resident, re-lay the ABQP weight planes out
// for the GEMM, in stream-ordered scratch.
static int gemm_tc_from_planes(const uint64_t* a, unsigned p, size_t m, const uint64_t* w_planes,
                               const uint32_t* wtc, unsigned q, size_t n, size_t k,
                               const EpiParams& e, cudaStream_t s, EnginePlan plan = EnginePlan{0, 0}) {
  uint8_t* codes = nullptr;
  ABQ_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&codes), m * k + tc_act_bytes(m, k), s));
  uint8_t* tiled = codes + m * k;  // 16-B aligned: k % 16 == 0
  int st = run_unpack(a, p, m, k, codes, s);
  if (!st) st = run_tile_codes(codes, m, k, tiled, s);
  uint32_t* tmp = nullptr;
  if (!st && !wtc) {
    cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&tmp), tc_words(q, n, k) * 4, s);
    if (err != cudaSuccess) st = fail(ABQ_ERR_CUDA, "gemm_tc: scratch: %s", cudaGetErrorString(err));
    if (!st) st = run_prepack_tc(w_planes, q, n, k, tmp, s);
    wtc = tmp;
  }
  // the stream-K schedule needs its (zeroed) flags and partial tiles
  unsigned* flags = nullptr;
  uint32_t* part = nullptr;
  if (!st && plan.schedule == ABQ_GEMM_STREAM_K) {
    cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&flags), tc_sk_flag_bytes(n, k), s);
    if (err == cudaSuccess) err = cudaMemsetAsync(flags, 0, tc_sk_flag_bytes(n, k), s);
    if (err == cudaSuccess) err = cudaMallocAsync(reinterpret_cast<void**>(&part), tc_sk_part_bytes(m, n, k), s);
    if (err != cudaSuccess) st = fail(ABQ_ERR_CUDA, "gemm_tc: stream-K scratch: %s", cudaGetErrorString(err));
  }
  if (!st) st = run_gemm_tc(wtc, q, n, k, tiled, m, e, s, nullptr, nullptr, false, flags, part, plan);
  if (flags) cudaFreeAsync(flags, s);
  if (part) cudaFreeAsync(part, s);
  cudaFreeAsync(codes, s);
  if (tmp) cudaFreeAsync(tmp, s);
  return st;
}

static EpiParams raw_epi(void* out, size_t n, bool wide) {
  EpiParams e{};
  e.mode = wide ? EPI_ACC_I64 : EPI_ACC_I32;
  e.out = out;
  e.ldo = static_cast<long long>(n);
  return e;
}

}  // namespace abq_dev

using namespace abq_dev;

static int epi_mode_of(int out_kind, int* mode) {
  switch (out_kind) {
    case ABQ_OUT_F64: *mode = EPI_F64; return ABQ_OK;
    case ABQ_OUT_F16: *mode = EPI_F16; return ABQ_OK;
    case ABQ_OUT_F32: *mode = EPI_F32; return ABQ_OK;
    case ABQ_OUT_CORR_I64: *mode = EPI_CORR_I64; return ABQ_OK;
    default: return fail(ABQ_ERR_VALUE, "linear: unknown out_kind %d", out_kind);
  }
}

static int check_qact(const abq_qact* out, const abq_quant_spec* spec, size_t m, size_t k, const char* who) {
  int st = validate_spec(spec);
  if (st) return st;
  if (spec->granularity == ABQ_PER_TENSOR)
    return fail(ABQ_ERR_VALUE, "%s: per-token activation spec required (the ReQuant is fused per token)", who);
  if (!out || !out->codes || !out->scales || !out->zero_points || !out->rowsums)
    return fail(ABQ_ERR_VALUE, "%s: output buffers missing", who);
  if (out->m != m || out->k != k) return fail(ABQ_ERR_SHAPE, "%s: output shape differs from the input", who);
  if (!qact_supported(m, k))
    return fail(ABQ_ERR_VALUE, "%s: m <= 8 tokens, K %% 8 == 0 and K <= 16384 required (m=%zu, K=%zu)", who, m, k);
  if (out->bits != spec->bits) return fail(ABQ_ERR_VALUE, "%s: out->bits differs from the spec", who);
  return check_device();
}

template <typename Launch>
static int producer_call(int64_t* err_index, size_t k, cudaStream_t s, Launch&& launch) {
  unsigned long long* sc = nullptr;
  unsigned long long* err = reinterpret_cast<unsigned long long*>(err_index);
  if (!err) {
    sc = scratch_words();
    if (!sc) return fail(ABQ_ERR_CUDA, "producer: cannot allocate device scratch");
    ABQ_CUDA_TRY(cudaMemsetAsync(sc, 0xFF, 8, s));
    err = sc;
  }
  int st = launch(err);
  if (st || err_index) return st;
  unsigned long long b = 0;
  if ((st = sync_read(sc, s, &b))) return st;
  if (b != ~0ull) return fail(ABQ_ERR_VALUE, "quantize: non-finite element at (%llu,%llu)", b / k, b % k);
  return ABQ_OK;
}

extern "C" {

const char* abq_last_error(void) { return last_error().c_str(); }
int abq_version(void) { return 1; }
uint64_t abq_launch_count(void) { return launch_counter(); }

int abq_fits_int32(unsigned p, unsigned q, size_t k) { return fits_int32_host(p, q, k) ? 1 : 0; }

int abq_tile_valid(const abq_tile_config* tile, unsigned p, unsigned q) {
  return tile && tile_valid_host(*tile, p, q) ? 1 : 0;
}

abq_tile_config abq_default_tile(unsigned p, unsigned q) {
  abq_tile_config t;
  t.BM = 64;
  t.BN = 64;
  t.BK = 512;
  t.WM = 32 * p;
  t.WN = 32 * q;
  t.WK = 128;
  return t;
}

int abq_padding_redundancy(size_t m, unsigned p, size_t mma_m, double* out) {
  if (m == 0 || p == 0 || mma_m == 0)
    return fail(ABQ_ERR_VALUE, "padding_redundancy: arguments must be positive");
  const size_t expanded = p * m;
  const size_t padded = (expanded + mma_m - 1) / mma_m * mma_m;
  *out = double(padded - expanded) / double(padded);
  return ABQ_OK;
}

unsigned abq_spec_levels(const abq_quant_spec* spec) { return spec ? levels_of(*spec) : 0u; }
unsigned abq_spec_planes(const abq_quant_spec* spec) { return spec ? planes_of(*spec) : 0u; }

int abq_set_gemv_variant(int variant) {
  if (variant < ABQ_GEMV_AUTO || variant > ABQ_GEMV_RECOMB)
    return fail(ABQ_ERR_VALUE, "abq_set_gemv_variant: unknown variant %d", variant);
  g_gemv_variant = variant;
  return ABQ_OK;
}
int abq_get_gemv_variant(void) { return g_gemv_variant; }

int abq_set_gemm_schedule(int schedule) {
  if (schedule < ABQ_GEMM_AUTO || schedule > ABQ_GEMM_STREAM_K)
    return fail(ABQ_ERR_VALUE, "abq_set_gemm_schedule: unknown schedule %d", schedule);
  gemm_schedule() = schedule;
  return ABQ_OK;
}
int abq_get_gemm_schedule(void) { return gemm_schedule(); }

// ---- producer-fused ReQuant (producer.cu) ----------------------------------
size_t abq_qact_codes_bytes(size_t m, size_t k) { return qact_codes_bytes(m, k); }

int abq_rmsnorm_quant(const void* x, const void* gain, float eps, size_t m, size_t k, const abq_quant_spec* spec,
                      void* y_out, const abq_qact* out, int64_t* err_index, void* stream) {
  int st = check_qact(out, spec, m, k, "rmsnorm_quant");
  if (st) return st;
  if (!x || !gain) return fail(ABQ_ERR_VALUE, "rmsnorm_quant: null input");
  if (!(eps >= 0.0f)) return fail(ABQ_ERR_VALUE, "rmsnorm_quant: eps must be >= 0");
  const QuantParams qp = params_of(*spec);
  cudaStream_t s = as_stream(stream);
  return producer_call(err_index, k, s, [&](unsigned long long* err) {
    return run_rmsnorm_quant(static_cast<const __half*>(x), static_cast<const __half*>(gain), eps, m, k, qp,
                             static_cast<__half*>(y_out), out->codes, out->scales, out->zero_points,
                             reinterpret_cast<long long*>(out->rowsums), err, s);
  });
}

int abq_silu_mul_quant(const void* gate, const void* up, size_t m, size_t k, const abq_quant_spec* spec,
                       void* y_out, const abq_qact* out, int64_t* err_index, void* stream) {
  int st = check_qact(out, spec, m, k, "silu_mul_quant");
  if (st) return st;
  if (!gate || !up) return fail(ABQ_ERR_VALUE, "silu_mul_quant: null input");
  const QuantParams qp = params_of(*spec);
  cudaStream_t s = as_stream(stream);
  return producer_call(err_index, k, s, [&](unsigned long long* err) {
    return run_silu_mul_quant(static_cast<const __half*>(gate), static_cast<const __half*>(up), m, k, qp,
                              static_cast<__half*>(y_out), out->codes, out->scales, out->zero_points,
                              reinterpret_cast<long long*>(out->rowsums), err, s);
  });
}

int abq_stage_in(void* dst, const void* src_host, size_t bytes, void* stream) {
  if (!dst || !src_host) return fail(ABQ_ERR_VALUE, "stage_in: null buffer");
  int st = check_device();
  if (st) return st;
  return run_stage_in(dst, src_host, bytes, as_stream(stream));
}

int abq_linear_qact(const abq_qact* act, const abq_weights* w, void* y, int out_kind, void* stream) {
  if (!act || !w) return fail(ABQ_ERR_VALUE, "linear_qact: null argument");
  if (act->k != w->k) return fail(ABQ_ERR_SHAPE, "quantized_linear: inner dimensions differ");
  if (!w->frag) return fail(ABQ_ERR_VALUE, "linear_qact: weights lack the decode (frag) layout");
  if (!dec_supported(w->q, w->n, act->k, act->m))
    return fail(ABQ_ERR_VALUE, "linear_qact: decode GEMV does not cover m=%zu n=%zu K=%zu", act->m, w->n, act->k);
  if (act->bits < 1 || act->bits > 8) return fail(ABQ_ERR_VALUE, "linear_qact: activation bits must be in [1,8]");
  int mode = 0, st = epi_mode_of(out_kind, &mode);
  if (st) return st;
  if ((st = check_device())) return st;
  EpiParams e{};
  e.mode = mode;
  e.out = y;
  e.ldo = static_cast<long long>(w->n);
  e.s_b = w->scales;
  e.sb_stride = w->per_tensor ? 0 : 1;
  e.z_b = w->zero_points;
  e.zb_stride = w->per_tensor ? 0 : 1;
  e.colsum_b = w->colsums;
  e.k = static_cast<long long>(act->k);
  QuantParams qp{};
  qp.bits = act->bits;
  DecNext nb;
  return run_gemv_dec_qact(w->frag, w->q, w->n, act->k, act->m, act->codes, act->scales, act->zero_points,
                           reinterpret_cast<const long long*>(act->rowsums), qp, e, as_stream(stream),
                           next_of(w, &nb));
}

int abq_set_tuning(const char* key, long long value) {
  if (!key) return fail(ABQ_ERR_VALUE, "abq_set_tuning: null key");
  DecTuning& t = dec_tuning();
  const std::string k(key);
  if (k == "dec_pre_kb" && value >= -1) t.pre_kb = static_cast<int>(value);
  else if (k == "dec_ring_kb" && value >= 0) t.ring_kb = static_cast<int>(value);
  else if (k == "dec_pdl") t.pdl = value != 0;
  else if (k == "dec_pace_ns" && value >= 0) t.pace_ns = static_cast<int>(value);
  else if (k == "dec_grid_balanced") t.grid_balanced = value != 0;
  else if (k == "tc_dbg") t.tc_dbg = static_cast<int>(value);
  else if (k == "tc_tt" && value >= 0) t.tc_tt = static_cast<int>(value);
  else if (k == "tc_pre" && value >= 0) t.tc_pre = static_cast<int>(value);
  else if (k == "tc_sk_ctas" && value >= 2 && value <= 64) t.tc_sk_ctas = static_cast<int>(value);
  else if (k == "dec_next_kb" && value >= 0) t.next_kb = static_cast<int>(value);
  else if (k == "dec_next_min_kb" && value >= 0) t.next_min_kb = static_cast<int>(value);
  else if (k == "dec_next_at" && value >= 1 && value <= 100) t.next_at = static_cast<int>(value);
  else if (k == "dec_l2_plain") t.l2_plain = value != 0;
  else if (k == "dec_dbg_nostream") t.dbg_nostream = value != 0;
  else if (k == "reset") t = DecTuning{};
  else return fail(ABQ_ERR_VALUE, "abq_set_tuning: unknown key or bad value '%s'=%lld", key, value);
  return ABQ_OK;
}

int abq_set_trace_buffer(void* dev_words) {
  trace_buffer() = static_cast<unsigned long long*>(dev_words);
  return ABQ_OK;
}

// ---- quantizer -------------------------------------------------------------
int abq_quantize(const void* x, int x_dtype, size_t rows, size_t cols, const abq_quant_spec* spec,
                 const double* comp_a, const double* comp_b, uint8_t* codes, double* scales,
                 int32_t* zero_points, void* stream) {
  int st = validate_spec(spec);
  if (st) return st;
  if ((comp_a == nullptr) != (comp_b == nullptr))
    return fail(ABQ_ERR_SHAPE, "quantize: compensation pair does not match matrix shape");
  if ((st = check_device())) return st;
  unsigned long long* sc = scratch_words();
  if (!sc) return fail(ABQ_ERR_CUDA, "quantize: cannot allocate device scratch");
  cudaStream_t s = as_stream(stream);
  st = run_quantize(x, x_dtype, rows, cols, params_of(*spec), comp_a, comp_b, codes, nullptr, 0,
                    scales, zero_points, nullptr, sc, sc + 1, s);
  if (st) return st;
  unsigned long long bad = 0;
  if ((st = sync_read(sc, s, &bad))) return st;
  if (bad != ~0ull)
    return fail(ABQ_ERR_VALUE, "quantize: non-finite element at (%llu,%llu)", bad / cols, bad % cols);
  return ABQ_OK;
}

int abq_quant_pack_act(const void* x, int x_dtype, size_t m, size_t k, const abq_quant_spec* spec,
                       uint64_t* planes, double* scales, int32_t* zero_points, int64_t* rowsums,
                       uint8_t* codes, int64_t* err_index, void* stream) {
  int st = validate_spec(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  unsigned long long* sc = scratch_words();
  if (!sc) return fail(ABQ_ERR_CUDA, "quant_pack_act: cannot allocate device scratch");
  cudaStream_t s = as_stream(stream);
  unsigned long long* bad = err_index ? reinterpret_cast<unsigned long long*>(err_index) : sc;
  st = run_quantize(x, x_dtype, m, k, params_of(*spec), nullptr, nullptr, codes, planes,
                    planes_of(*spec), scales, zero_points, rowsums, bad, sc + 1, s);
  if (st || err_index) return st;
  unsigned long long b = 0;
  if ((st = sync_read(sc, s, &b))) return st;
  if (b != ~0ull)
    return fail(ABQ_ERR_VALUE, "quantize: non-finite element at (%llu,%llu)", b / k, b % k);
  return ABQ_OK;
}

// ---- bit planes ------------------------------------------------------------
int abq_bitpack(const uint8_t* codes, size_t rows, size_t cols, unsigned bits, uint64_t* planes,
                void* stream) {
  if (bits < 1 || bits > 8) return fail(ABQ_ERR_VALUE, "bitpack: plane count must be in [1,8]");
  int st = check_device();
  if (st) return st;
  unsigned long long* sc = scratch_words();
  if (!sc) return fail(ABQ_ERR_CUDA, "bitpack: cannot allocate device scratch");
  cudaStream_t s = as_stream(stream);
  if ((st = run_bitpack(codes, rows, cols, bits, planes, sc, s))) return st;
  unsigned long long bad = 0;
  if ((st = sync_read(sc, s, &bad))) return st;
  if (bad != ~0ull) {
    uint8_t c = 0;
    ABQ_CUDA_TRY(cudaMemcpy(&c, codes + bad, 1, cudaMemcpyDeviceToHost));
    return fail(ABQ_ERR_VALUE, "bitpack: code %d at (%llu,%llu) needs more than %u planes", int(c),
                bad / cols, bad % cols, bits);
  }
  return ABQ_OK;
}

int abq_unpack(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, uint8_t* codes,
               void* stream) {
  int st = check_device();
  if (st) return st;
  return run_unpack(planes, bits, rows, cols, codes, as_stream(stream));
}

int abq_gemm_btc(const uint64_t* a, unsigned p, size_t m, size_t a_k, const uint64_t* bt, unsigned q,
                 size_t n, size_t b_k, int32_t* out, void* stream) {
  if (a_k != b_k) return fail(ABQ_ERR_SHAPE, "gemm_btc: shared K dimension differs");
  if (!fits_int32_host(p, q, a_k))
    return fail(ABQ_ERR_OVERFLOW, "gemm_btc: p+q+ceil(log2(K+1)) = %u+%u+log2(%zu+1) exceeds 31", p, q, a_k);
  int st = check_device();
  if (st) return st;
  return run_gemm_bmma(a, p, m, bt, q, n, a_k, out, as_stream(stream));
}

int abq_bmma(const uint64_t* a, unsigned a_planes, size_t m, unsigned a_plane, const uint64_t* bt,
             unsigned b_planes, size_t n, unsigned b_plane, size_t k, int32_t* out, void* stream) {
  if (a_plane >= a_planes || b_plane >= b_planes)
    return fail(ABQ_ERR_VALUE, "bmma: plane index out of range");
  int st = check_device();
  if (st) return st;
  return run_bmma(a, m, a_plane, bt, n, b_plane, k, out, as_stream(stream));
}

// ---- engine ----------------------------------------------------------------
// TileConfig -> sm_100a engine schedule (the reference's
// tile, gemm.hpp:19-59, picks the CPU block / warp tiling).  BM (activation
// rows per block) caps the token tile: the tcgen05 GEMM's UMMA N (16..256) or
// the AND+popcount kernel's token block (1..8); BK (k depth per block) selects
// the k-split: BK == 128 -> stream-K over all SMs (CTAs share a row-tile's
// k-range), deeper -> one CTA per 128-channel row-tile.  Results never depend
// on it (tile transparency, test_bitkernel.cpp:104-115); time does, so the
// reference's autotune over tile candidates times different kernels.
static EnginePlan plan_of(const abq_tile_config* t) {
  EnginePlan pl{0, ABQ_GEMM_AUTO};
  if (!t) return pl;
  int tt = 1;
  while (tt * 2 <= static_cast<int>(std::min<size_t>(t->BM, 256))) tt *= 2;
  pl.token_tile = tt;
  pl.schedule = t->BK <= 128 ? ABQ_GEMM_STREAM_K : ABQ_GEMM_CLASSIC;
  return pl;
}

static int gemm_common(const char* name, const uint64_t* a, unsigned p, size_t m, size_t a_k,
                       const uint64_t* bt, unsigned q, size_t n, size_t b_k,
                       const abq_tile_config* tile, bool wide, bool check_overflow, void* out,
                       abq_gemm_stats* stats, void* stream) {
  if (a_k != b_k) return fail(ABQ_ERR_SHAPE, "%s: shared K dimension differs", name);
  if (tile) {
    if (!tile_valid_host(*tile, p, q))
      return fail(ABQ_ERR_VALUE,
                  "TileConfig invalid for p=%u q=%u: BM=%zu BN=%zu BK=%zu WM=%zu WN=%zu WK=%zu", p, q,
                  tile->BM, tile->BN, tile->BK, tile->WM, tile->WN, tile->WK);
  }
  if (check_overflow && !fits_int32_host(p, q, a_k))
    return fail(ABQ_ERR_OVERFLOW,
                "%s: p+q+ceil(log2(K+1)) = %u+%u+log2(%zu+1) exceeds 31; use gemm_arbitrary_wide",
                name, p, q, a_k);
  if (p < 1 || p > 8 || q < 1 || q > 8) return fail(ABQ_ERR_VALUE, "%s: plane counts must be in [1,8]", name);
  int st = check_device();
  if (st) return st;
  if (m * n > 0 && a_k == 0) {
    // K == 0: every sum is empty
    ABQ_CUDA_TRY(cudaMemsetAsync(out, 0, m * n * (wide ? 8 : 4), as_stream(stream)));
  } else if (m >= 16 && !wide && gemm_tc_supported(a_k) && g_gemv_variant != ABQ_GEMV_POPC) {
    // prefill-shaped: recombined planes on tcgen05 (weights re-laid out per call)
    st = gemm_tc_from_planes(a, p, m, bt, nullptr, q, n, a_k, raw_epi(out, n, wide), as_stream(stream),
                             plan_of(tile));
    if (st) return st;
  } else {
    st = run_gemm_popc(a, p, m, bt, q, n, a_k, wide, raw_epi(out, n, wide), as_stream(stream),
                       plan_of(tile).token_tile);
    if (st) return st;
  }
  if (tile) add_stats(stats, *tile, m, n, p, q);
  return ABQ_OK;
}

int abq_tile_engine_plan(const abq_tile_config* tile, int* token_tile, int* schedule) {
  if (!tile || !token_tile || !schedule) return fail(ABQ_ERR_VALUE, "tile_engine_plan: null argument");
  const EnginePlan pl = plan_of(tile);
  *token_tile = pl.token_tile;
  *schedule = pl.schedule;
  return ABQ_OK;
}

int abq_gemm_arbitrary(const uint64_t* a, unsigned p, size_t m, size_t a_k, const uint64_t* bt,
                       unsigned q, size_t n, size_t b_k, const abq_tile_config* tile, int32_t* out,
                       abq_gemm_stats* stats, void* stream) {
  abq_tile_config def = abq_default_tile(p, q);
  return gemm_common("gemm_arbitrary", a, p, m, a_k, bt, q, n, b_k, tile ? tile : &def, false, true,
                     out, stats, stream);
}

int abq_gemm_arbitrary_wide(const uint64_t* a, unsigned p, size_t m, size_t a_k,
                            const uint64_t* bt, unsigned q, size_t n, size_t b_k,
                            const abq_tile_config* tile, int64_t* out, abq_gemm_stats* stats,
                            void* stream) {
  abq_tile_config def = abq_default_tile(p, q);
  return gemm_common("gemm_arbitrary_wide", a, p, m, a_k, bt, q, n, b_k, tile ? tile : &def, true,
                     false, out, stats, stream);
}

int abq_gemm_naive(const uint64_t* a, unsigned p, size_t m, size_t a_k, const uint64_t* bt,
                   unsigned q, size_t n, size_t b_k, int32_t* out, void* stream) {
  // gemm.hpp:213-231: no tile and no overflow guard (int32 wraps like the reference would)
  return gemm_common("gemm_naive", a, p, m, a_k, bt, q, n, b_k, nullptr, false, false, out, nullptr,
                     stream);
}

int abq_zero_point_correct_i32(const int32_t* acc, size_t m, size_t n, const int64_t* rowsum_a,
                               const int64_t* colsum_b, const int32_t* z_a, const int32_t* z_b,
                               size_t k, int32_t* out, void* stream) {
  int st = check_device();
  if (st) return st;
  return run_zero_point_correct<int32_t>(acc, m, n, rowsum_a, colsum_b, z_a, z_b, k, out,
                                         as_stream(stream));
}

int abq_zero_point_correct_i64(const int64_t* acc, size_t m, size_t n, const int64_t* rowsum_a,
                               const int64_t* colsum_b, const int32_t* z_a, const int32_t* z_b,
                               size_t k, int64_t* out, void* stream) {
  int st = check_device();
  if (st) return st;
  return run_zero_point_correct<int64_t>(acc, m, n, rowsum_a, colsum_b, z_a, z_b, k, out,
                                         as_stream(stream));
}

int abq_code_rowsums(const uint8_t* codes, size_t rows, size_t cols, int64_t* out, void* stream) {
  int st = check_device();
  if (st) return st;
  return run_code_rowsums(codes, rows, cols, out, as_stream(stream));
}

int abq_dequantize(const uint8_t* codes, size_t rows, size_t cols, const double* scales,
                   const int32_t* zero_points, int per_tensor, double* out, void* stream) {
  int st = check_device();
  if (st) return st;
  return run_dequantize(codes, rows, cols, scales, zero_points, per_tensor, out, as_stream(stream));
}

int abq_plane_rowsums(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, int64_t* out,
                      void* stream) {
  int st = check_device();
  if (st) return st;
  return run_plane_rowsums(planes, bits, rows, cols, out, as_stream(stream));
}

size_t abq_weights_frag_bytes(unsigned q, size_t n, size_t k) { return frag_words(q, n, k) * 4; }

int abq_weights_prepack(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* frag,
                        void* stream) {
  if (q < 1 || q > 8) return fail(ABQ_ERR_VALUE, "weights_prepack: plane count must be in [1,8]");
  int st = check_device();
  if (st) return st;
  return run_prepack_frag(planes, q, n, k, frag, as_stream(stream));
}

size_t abq_weights_tc_bytes(unsigned q, size_t n, size_t k) { return tc_words(q, n, k) * 4; }

int abq_weights_prepack_tc(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* tc,
                           void* stream) {
  if (q < 1 || q > 8) return fail(ABQ_ERR_VALUE, "weights_prepack_tc: plane count must be in [1,8]");
  int st = check_device();
  if (st) return st;
  return run_prepack_tc(planes, q, n, k, tc, as_stream(stream));
}

// ---- fused linear ----------------------------------------------------------

int abq_linear_planes(const abq_act* act, const abq_weights* w, void* y, int out_kind,
                      void* stream) {
  if (!act || !w) return fail(ABQ_ERR_VALUE, "quantized_linear: null operand");
  if (act->k != w->k) return fail(ABQ_ERR_SHAPE, "quantized_linear: inner dimensions differ");
  if (act->p < 1 || act->p > 8 || w->q < 1 || w->q > 8)
    return fail(ABQ_ERR_VALUE, "quantized_linear: plane counts must be in [1,8]");
  int mode = 0;
  int st = epi_mode_of(out_kind, &mode);
  if (st) return st;
  if ((st = check_device())) return st;
  EpiParams e{};
  e.mode = mode;
  e.out = y;
  e.ldo = static_cast<long long>(w->n);
  e.s_a = act->scales;
  e.sa_stride = act->per_tensor ? 0 : 1;
  e.z_a = act->zero_points;
  e.za_stride = act->per_tensor ? 0 : 1;
  e.rowsum_a = act->rowsums;
  e.s_b = w->scales;
  e.sb_stride = w->per_tensor ? 0 : 1;
  e.z_b = w->zero_points;
  e.zb_stride = w->per_tensor ? 0 : 1;
  e.colsum_b = w->colsums;
  e.k = static_cast<long long>(act->k);
  const bool wide = !fits_int32_host(act->p, w->q, act->k);
  if (use_imma(w, act->m, act->k))
    return run_gemv_imma_planes(w->frag, w->q, w->n, act->k, act->m, act->planes, act->p, e,
                                as_stream(stream));
  if (use_tc(w, act->m, act->k, wide))
    return gemm_tc_from_planes(act->planes, act->p, act->m, w->planes, w->tc, w->q, w->n, act->k, e,
                               as_stream(stream));
  if (!w->planes)
    return fail(ABQ_ERR_VALUE,
                "quantized_linear: no resident weight layout serves m=%zu (the decode layout covers m <= 8, "
                "the prefill layout m >= 1; the ABQP planes were dropped)", act->m);
  return run_gemm_popc(act->planes, act->p, act->m, w->planes, w->q, w->n, act->k, wide, e,
                       as_stream(stream));
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

size_t abq_linear_workspace_bytes(size_t m, size_t n, size_t k, unsigned act_planes) {
  // [gacc + gcnt for the stream-K decode GEMV][stream-K GEMM flags][ReQuant report word, 256 B][act planes][s_a][z_a]
  // [rowsum_a][range 256 B][tiled u8 act codes for the tcgen05 GEMM][row-major u8 codes m x k]
  // [stream-K GEMM partial tiles]; everything before the act planes depends on n, k only
  return align256(imma_ws_bytes(n, k)) + align256(tc_sk_flag_bytes(n, k)) + 256 +
         align256(size_t(act_planes) * m * wpr_of(k) * 8) + align256(m * 8) + align256(m * 4) +
         align256(m * 8) + 256 + align256(tc_act_bytes(m, k)) + align256(m * k) +
         align256(tc_sk_part_bytes(std::min<size_t>(m, 256), n, k));
  // (the stream-K partial tiles are sized for min(m, 256) tokens: the GEMM only
  // runs stream-K up to 256 tokens, and the total must not shrink as m grows,
  // so a workspace sized for max_m serves every m <= max_m)
}

int abq_linear(const void* x, int x_dtype, size_t m, size_t k, const abq_quant_spec* act_spec,
               const abq_weights* w, void* y, int out_kind, void* workspace, size_t workspace_bytes,
               int64_t* err_index, void* stream) {
  int st = validate_spec(act_spec);
  if (st) return st;
  if (!w) return fail(ABQ_ERR_VALUE, "quantized_linear: null weights");
  if (k != w->k) return fail(ABQ_ERR_SHAPE, "quantized_linear: inner dimensions differ");
  const unsigned p = planes_of(*act_spec);
  const size_t need = abq_linear_workspace_bytes(m, w->n, k, p);
  if (workspace_bytes < need)
    return fail(ABQ_ERR_VALUE, "linear: workspace too small (%zu < %zu)", workspace_bytes, need);
  int mode = 0;
  if ((st = epi_mode_of(out_kind, &mode))) return st;
  if ((st = check_device())) return st;
  char* ws = static_cast<char*>(workspace);
  void* ws_imma = ws;
  ws += align256(imma_ws_bytes(w->n, k));
  unsigned* sk_flags = reinterpret_cast<unsigned*>(ws);
  ws += align256(tc_sk_flag_bytes(w->n, k));
  // zero between calls; at an offset independent of m (the regions after it
  // move with m and hold data of earlier calls)
  unsigned long long* bad_word = reinterpret_cast<unsigned long long*>(ws);
  ws += 256;
  uint64_t* planes = reinterpret_cast<uint64_t*>(ws);
  ws += align256(size_t(p) * m * wpr_of(k) * 8);
  double* sa = reinterpret_cast<double*>(ws);
  ws += align256(m * 8);
  int32_t* za = reinterpret_cast<int32_t*>(ws);
  ws += align256(m * 4);
  int64_t* ra = reinterpret_cast<int64_t*>(ws);
  ws += align256(m * 8);
  unsigned long long* range = reinterpret_cast<unsigned long long*>(ws);
  unsigned long long* sc = nullptr;
  if (!err_index) {
    sc = scratch_words();
    if (!sc) return fail(ABQ_ERR_CUDA, "linear: cannot allocate device scratch");
  }
  unsigned long long* bad = err_index ? reinterpret_cast<unsigned long long*>(err_index) : sc;
  cudaStream_t s = as_stream(stream);
  if (use_dec(w, m, k)) {
    // single launch: ReQuant prologue + tensor-pipe plane GEMV + fused epilogue
    EpiParams e{};
    e.mode = mode;
    e.out = y;
    e.ldo = static_cast<long long>(w->n);
    e.s_b = w->scales;
    e.sb_stride = w->per_tensor ? 0 : 1;
    e.z_b = w->zero_points;
    e.zb_stride = w->per_tensor ? 0 : 1;
    e.colsum_b = w->colsums;
    e.k = static_cast<long long>(k);
    const QuantParams qp = params_of(*act_spec);
    DecNext nb;
    st = run_gemv_dec(w->frag, w->q, w->n, k, m, x, x_dtype, qp, e, ws_imma, bad, s, next_of(w, &nb));
    if (st) return st;
  } else if (use_tc(w, m, k, !fits_int32_host(p, w->q, k))) {
    // ReQuant straight to u8 codes (K1), then the tcgen05 GEMM with the fused epilogue
    uint8_t* codes = reinterpret_cast<uint8_t*>(range + 32);  // tiled operand
    uint8_t* rowmajor = codes + align256(tc_act_bytes(m, k));
    uint32_t* sk_part = reinterpret_cast<uint32_t*>(rowmajor + align256(m * k));
    // per-token (or few-token per-tensor) ReQuant: one CTA per token, PDL into the GEMM
    const bool fast_k1 = act_spec->granularity != ABQ_PER_TENSOR || m <= 8;
    if (fast_k1) {
      st = run_act_quant(x, x_dtype, m, k, 1, params_of(*act_spec), reinterpret_cast<uint32_t*>(codes),
                         tc_act_groups(static_cast<long long>(m)), sa, za, reinterpret_cast<long long*>(ra),
                         bad_word, s);
    } else {
      st = run_quantize(x, x_dtype, m, k, params_of(*act_spec), nullptr, nullptr, rowmajor, nullptr, p, sa,
                        za, ra, bad, range, s);
      if (!st) st = run_tile_codes(rowmajor, m, k, codes, s);
    }
    if (st) return st;
    EpiParams e{};
    e.mode = mode;
    e.out = y;
    e.ldo = static_cast<long long>(w->n);
    e.s_a = sa;
    e.sa_stride = fast_k1 || act_spec->granularity != ABQ_PER_TENSOR ? 1 : 0;
    e.z_a = za;
    e.za_stride = e.sa_stride;
    e.rowsum_a = ra;
    e.s_b = w->scales;
    e.sb_stride = w->per_tensor ? 0 : 1;
    e.z_b = w->zero_points;
    e.zb_stride = w->per_tensor ? 0 : 1;
    e.colsum_b = w->colsums;
    e.k = static_cast<long long>(k);
    st = run_gemm_tc(w->tc, w->q, w->n, k, codes, m, e, s, fast_k1 ? bad_word : nullptr,
                     fast_k1 ? bad : nullptr, fast_k1, sk_flags, sk_part);
    if (st) return st;
  } else {
    st = run_quantize(x, x_dtype, m, k, params_of(*act_spec), nullptr, nullptr, nullptr, planes, p, sa,
                      za, ra, bad, range, s);
    if (st) return st;
    abq_act act{planes, p, m, k, sa, za, ra, act_spec->granularity == ABQ_PER_TENSOR};
    if ((st = abq_linear_planes(&act, w, y, out_kind, stream))) return st;
  }
  if (err_index) return ABQ_OK;
  unsigned long long b = 0;
  if ((st = sync_read(sc, s, &b))) return st;
  if (b != ~0ull)
    return fail(ABQ_ERR_VALUE, "quantize: non-finite element at (%llu,%llu)", b / k, b % k);
  return ABQ_OK;
}

int abq_linear_host(const void* x_host, int x_dtype, size_t m, size_t k, void* x_stage,
                    const abq_quant_spec* act_spec, const abq_weights* w, void* y_host, int out_kind,
                    void* workspace, size_t workspace_bytes, int64_t* err_index, void* stream) {
  if (!x_host || !x_stage || !y_host) return fail(ABQ_ERR_VALUE, "linear_host: null buffer");
  const size_t esize = x_dtype == ABQ_F16 ? 2 : x_dtype == ABQ_F32 ? 4 : 8;
  int st = check_device();
  if (st) return st;
  if ((st = run_stage_in(x_stage, x_host, m * k * esize, as_stream(stream)))) return st;
  return abq_linear(x_stage, x_dtype, m, k, act_spec, w, y_host, out_kind, workspace, workspace_bytes, err_index,
                    stream);
}

}  // extern "C"
