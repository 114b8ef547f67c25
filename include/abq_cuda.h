/*
 * abq_cuda.h -- C-ABI of the B200-native ABQ-LLM bit-plane quantized matmul
 * engine (libabq_cuda.so, built from paper_2408_08554_b200/csrc for sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (/root/reference/proj, header-only C++20) exposes it as inline C++
 * functions in namespace abq; each entry point below cites the function it
 * replaces.  The C++ mirror with the reference's exact signatures and
 * exception classes lives in include/abq/ and forwards here.
 *
 * Conventions (identical to the reference):
 *   - operand a = activation codes (M x K, p = act planes), bt = weight codes
 *     stored transposed (N x K, q = weight planes)   gemm.hpp:181-185
 *   - bit planes in the ABQP layout: [plane][row][word], u64 words,
 *     words_per_row = ceil(K/64), bit c of a row = bit (c%64) of word (c/64),
 *     LSB-first, tail bits zero                       bitplane.hpp:15-44, io.hpp:102-124
 *   - FP64 quantizer with round-half-away-from-zero   quantizer.hpp:146-213
 *
 * Rules of the ABI: plain pointers and sizes only.  All array pointers are
 * DEVICE pointers (cudaMalloc / torch CUDA storage) unless stated otherwise;
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Every entry point returns an abq_status; on failure abq_last_error()
 * returns a thread-local message shaped like the reference's exception text.
 * Entry points that the reference can fail on with data-dependent errors
 * (code range, non-finite input) synchronise `stream` to report them, exactly
 * where the reference would throw; the *_async variants instead record the
 * first offending flat index into a caller-provided device word.
 */
#ifndef ABQ_CUDA_H_
#define ABQ_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: the C-ABI image of the reference exception hierarchy
 * core.hpp:13-36 (Error > ShapeError / ValueError / OverflowError / IoError). */
typedef enum {
  ABQ_OK = 0,
  ABQ_ERR_SHAPE = 1,    /* abq::ShapeError */
  ABQ_ERR_VALUE = 2,    /* abq::ValueError */
  ABQ_ERR_OVERFLOW = 3, /* abq::OverflowError */
  ABQ_ERR_IO = 4,       /* abq::IoError */
  ABQ_ERR_CUDA = 5      /* launch / device failure (abq::Error) */
} abq_status;

/* quantizer.hpp:14-15 */
typedef enum { ABQ_ASYMMETRIC = 0, ABQ_SYMMETRIC = 1, ABQ_BALANCED = 2 } abq_scheme;
typedef enum { ABQ_PER_TENSOR = 0, ABQ_PER_CHANNEL = 1, ABQ_PER_TOKEN = 2 } abq_granularity;

/* element types of float inputs / outputs */
typedef enum { ABQ_F16 = 0, ABQ_F64 = 1, ABQ_F32 = 2 } abq_dtype;

/* QuantSpec  quantizer.hpp:37-71.  balance_scale is applied by the caller to
 * x before quantization (toyblock.hpp:228-234), as in the reference. */
typedef struct {
  unsigned bits;   /* [1,8]; balanced <= 7 */
  int scheme;      /* abq_scheme */
  int granularity; /* abq_granularity */
  double alpha;    /* (0,1] max-side clip */
  double beta;     /* (0,1] min-side clip */
} abq_quant_spec;

/* TileConfig  gemm.hpp:19-48 (validated exactly like the reference; the GPU
 * kernels choose their own sm_100a tiling, results are tile-invariant). */
typedef struct {
  size_t BM, BN, BK, WM, WN, WK;
} abq_tile_config;

/* GemmStats  gemm.hpp:61-64 (accumulated, never reset, like the reference) */
typedef struct {
  uint64_t block_tiles;
  uint64_t plane_pair_products;
} abq_gemm_stats;

/* Device-resident, offline-packed weights (the reference
 * re-packs weights on every quantized_linear call, gemm.hpp:274-278).
 * planes: ABQP [q][n][words_per_row]; scales/zero_points: n entries
 * (per-channel) or 1 (per-tensor); colsums[n] = code_rowsums(wt.codes). */
typedef struct abq_weights_s {
  const uint64_t* planes;
  unsigned q;
  size_t n, k;
  const double* scales;
  const int32_t* zero_points;
  const int64_t* colsums;
  int per_tensor;
  /* optional fragment-major copy of the planes for the tensor-pipe decode
   * GEMV (abq_weights_prepack); NULL = AND+popcount kernels only */
  const uint32_t* frag;
  /* optional tcgen05-GEMM copy of the planes (abq_weights_prepack_tc) used
   * for M >= 9 tokens; NULL = no prefill tensor-core path */
  const uint32_t* tc;
  /* optional successor-layer hint: the weights the caller runs NEXT on this
   * stream (a decode step's layer order is static).  In the decode GEMV's
   * tail, once a CTA's own weights have landed, it prefetches the first
   * KB of its share of next->frag into L2 (HBM otherwise idles while the
   * grid finishes and the next launch's CTAs start); NULL = no hint.  Results
   * never depend on it. */
  const struct abq_weights_s* next;
} abq_weights;

/* Activation-side metadata produced by abq_quant_pack_act (per-token or
 * per-tensor scales / zero points, code row sums). */
typedef struct {
  const uint64_t* planes; /* [p][m][words_per_row] */
  unsigned p;
  size_t m, k;
  const double* scales;
  const int32_t* zero_points;
  const int64_t* rowsums;
  int per_tensor;
} abq_act;

/* ---- library / errors ---------------------------------------------------- */
const char* abq_last_error(void);
int abq_version(void);
/* Number of kernel launches this thread issued through the library so far
 * (bench.py reports it as gpu_launches). */
uint64_t abq_launch_count(void);

/* ---- scalar helpers (host-only, no device work) --------------------------- */
/* fits_int32  gemm.hpp:73-77 */
int abq_fits_int32(unsigned p, unsigned q, size_t k);
/* TileConfig::valid  gemm.hpp:24-32 */
int abq_tile_valid(const abq_tile_config* tile, unsigned p, unsigned q);
/* default_tile  gemm.hpp:51-59 */
abq_tile_config abq_default_tile(unsigned p, unsigned q);
/* padding_redundancy  tune.hpp:17-23 (ABQ_ERR_VALUE on non-positive args) */
int abq_padding_redundancy(size_t m, unsigned p, size_t mma_m, double* out);
/* QuantSpec::levels / planes  quantizer.hpp:49-59 */
unsigned abq_spec_levels(const abq_quant_spec* spec);
unsigned abq_spec_planes(const abq_quant_spec* spec);

/* ---- L1: quantizer ------------------------------------------------------- */
/* quantize  quantizer.hpp:146-213.  x: rows x cols (x_dtype F16 / F32 / F64).
 * comp_a[rows] / comp_b[cols] may both be NULL (no compensation pair).
 * scales / zero_points: 1 (per-tensor) or rows entries.  Synchronous error
 * check (ValueError with "(i,j)" for non-finite input, quantizer.hpp:131-140). */
int abq_quantize(const void* x, int x_dtype, size_t rows, size_t cols, const abq_quant_spec* spec,
                 const double* comp_a, const double* comp_b, uint8_t* codes, double* scales,
                 int32_t* zero_points, void* stream);

/* K1: ReQuant + BitPacking of activations, fused: x -> act planes + per-row
 * scale / zero point + code row sums (quantizer.hpp:146-213 -> bitplane.hpp:47-64
 * -> gemm.hpp:256-261).  `codes` may be NULL.  If err_index is non-NULL the
 * call is asynchronous: the first non-finite flat index (or -1, all bits set,
 * when every element is finite) is written there; otherwise the call
 * synchronises and reports ValueError. */
int abq_quant_pack_act(const void* x, int x_dtype, size_t m, size_t k, const abq_quant_spec* spec,
                       uint64_t* planes, double* scales, int32_t* zero_points, int64_t* rowsums,
                       uint8_t* codes, int64_t* err_index, void* stream);

/* ---- L2: bit planes ------------------------------------------------------ */
/* bitpack  bitplane.hpp:47-64 (ValueError "code c at (i,j) needs more than b planes") */
int abq_bitpack(const uint8_t* codes, size_t rows, size_t cols, unsigned bits, uint64_t* planes,
                void* stream);
/* unpack  bitplane.hpp:66-76 */
int abq_unpack(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, uint8_t* codes,
               void* stream);
/* bmma  bitplane.hpp:81-96 (one plane pair, AND + popcount) */
int abq_bmma(const uint64_t* a, unsigned a_planes, size_t m, unsigned a_plane, const uint64_t* bt,
             unsigned b_planes, size_t n, unsigned b_plane, size_t k, int32_t* out, void* stream);

/* ---- L3: engine ---------------------------------------------------------- */
/* TileConfig -> sm_100a engine schedule used by gemm_arbitrary(_wide)
 * (SURVEY.md 8f-3): BM caps the token tile (tcgen05 UMMA N 16..256, or the
 * AND+popcount kernel's token block 1..8) -- written to *token_tile as the
 * largest power of two <= min(BM, 256); BK == 128 selects the stream-K
 * schedule (CTAs share each 128-channel row-tile's k-range), deeper BK one CTA
 * per row-tile -- *schedule = ABQ_GEMM_STREAM_K / ABQ_GEMM_CLASSIC.  Results
 * are identical for every valid tile; run time is not. */
int abq_tile_engine_plan(const abq_tile_config* tile, int* token_tile, int* schedule);
/* gemm_arbitrary  gemm.hpp:185-198: validation order ShapeError (K differs),
 * ValueError (tile), OverflowError (fits_int32).  a_k / b_k are the two
 * operands' cols. */
int abq_gemm_arbitrary(const uint64_t* a, unsigned p, size_t m, size_t a_k, const uint64_t* bt,
                       unsigned q, size_t n, size_t b_k, const abq_tile_config* tile, int32_t* out,
                       abq_gemm_stats* stats, void* stream);
/* gemm_arbitrary_wide  gemm.hpp:201-209 (int64 accumulators) */
int abq_gemm_arbitrary_wide(const uint64_t* a, unsigned p, size_t m, size_t a_k,
                            const uint64_t* bt, unsigned q, size_t n, size_t b_k,
                            const abq_tile_config* tile, int64_t* out, abq_gemm_stats* stats,
                            void* stream);
/* gemm_btc: the same plane GEMM as gemm_arbitrary (gemm.hpp:94-146, int32
 * accumulators) on the b1 tensor-core path (mma.sync m16n8k256 .b1 and.popc),
 * kept as the measured comparator of the tcgen05 recombination GEMM; (p, q) in
 * {(4,4), (8,8), (8,2), (8,4), (4,8), (2,2)}.  Validation as gemm_arbitrary. */
int abq_gemm_btc(const uint64_t* a, unsigned p, size_t m, size_t a_k, const uint64_t* bt, unsigned q,
                 size_t n, size_t b_k, int32_t* out, void* stream);
/* gemm_naive  gemm.hpp:213-231 */
int abq_gemm_naive(const uint64_t* a, unsigned p, size_t m, size_t a_k, const uint64_t* bt,
                   unsigned q, size_t n, size_t b_k, int32_t* out, void* stream);
/* zero_point_correct  gemm.hpp:235-254 (int64 arithmetic, Acc output) */
int abq_zero_point_correct_i32(const int32_t* acc, size_t m, size_t n, const int64_t* rowsum_a,
                               const int64_t* colsum_b, const int32_t* z_a, const int32_t* z_b,
                               size_t k, int32_t* out, void* stream);
int abq_zero_point_correct_i64(const int64_t* acc, size_t m, size_t n, const int64_t* rowsum_a,
                               const int64_t* colsum_b, const int32_t* z_a, const int32_t* z_b,
                               size_t k, int64_t* out, void* stream);
/* code_rowsums  gemm.hpp:256-261 */
int abq_code_rowsums(const uint8_t* codes, size_t rows, size_t cols, int64_t* out, void* stream);
/* dequantize  quantizer.hpp:243-254: out[i][j] = (code - z[g]) * step[g] in FP64,
 * g = 0 (per_tensor) or i (per-row granularities).  Validation (code range,
 * parameter counts) is the caller's, as QuantizedTensor::validate. */
int abq_dequantize(const uint8_t* codes, size_t rows, size_t cols, const double* scales,
                   const int32_t* zero_points, int per_tensor, double* out, void* stream);

/* K5: colsum_b of packed weights from their planes (= code_rowsums(wt.codes),
 * gemm.hpp:278): colsum[j] = sum_t 2^t popc(W_t[j]). */
int abq_plane_rowsums(const uint64_t* planes, unsigned bits, size_t rows, size_t cols,
                      int64_t* out, void* stream);

/* K5: offline re-layout of ABQP weight planes into the fragment-major plane
 * layout consumed by the decode GEMV on the int8 tensor pipe: [row-tile of 16]
 * [k-block of 256][plane][lane][4 x u32] -- same bits, same byte count (rows
 * padded to 16, K to 256 with zero bits). */
size_t abq_weights_frag_bytes(unsigned q, size_t n, size_t k);
int abq_weights_prepack(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* frag,
                        void* stream);
/* K5 for the prefill GEMM: ABQP planes -> [row-tile 128][k-block 128][plane]
 * [row][4 x u32] (bit 8b+c of word j <-> k = 32j + 4c + b), the layout the
 * tcgen05 kernel rebuilds u8 codes from. */
size_t abq_weights_tc_bytes(unsigned q, size_t n, size_t k);
int abq_weights_prepack_tc(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* tc,
                           void* stream);

/* Fused engine linear on packed operands (K2/K3 + K4):
 *   y[i][j] = s_a[i] * s_b[j] * corrected[i][j]        gemm.hpp:266-307
 * out_kind selects what is written:
 *   ABQ_OUT_F64  double, bit-identical to the reference's Mat (API parity)
 *   ABQ_OUT_F16  fp16 = round-to-nearest of the same double (perf mode)
 *   ABQ_OUT_F32  float = round-to-nearest of the same double
 *   ABQ_OUT_CORR_I64  the int64 zero-point-corrected accumulator */
typedef enum {
  ABQ_OUT_F64 = 1,
  ABQ_OUT_F16 = 0,
  ABQ_OUT_F32 = 2,
  ABQ_OUT_CORR_I64 = 3
} abq_out_kind;
int abq_linear_planes(const abq_act* act, const abq_weights* w, void* y, int out_kind,
                      void* stream);

/* One-call engine linear from float activations (K1 + K2/K3 + K4): the
 * device-resident equivalent of quantize(act) + quantized_linear
 * (toyblock.hpp:240-242).  workspace >= abq_linear_workspace_bytes(m,n,k,p)
 * and must be ZERO-FILLED before its first use (the engine leaves it zeroed).
 * err_index (device, may be NULL => synchronous check) as in abq_quant_pack_act.
 * With w->frag set and m <= 8 this is ONE kernel launch (ReQuant in the
 * prologue, tensor-pipe plane GEMV, fused epilogue). */
size_t abq_linear_workspace_bytes(size_t m, size_t n, size_t k, unsigned act_planes);
int abq_linear(const void* x, int x_dtype, size_t m, size_t k, const abq_quant_spec* act_spec,
               const abq_weights* w, void* y, int out_kind, void* workspace,
               size_t workspace_bytes, int64_t* err_index, void* stream);

/* ---- producer-fused ReQuant for decode --------------------
 * The op that produces a decode linear's input -- RMSNorm (toyblock.hpp:257,
 * 267) or SiLU(gate) * up (toyblock.hpp:274-275) -- quantizes its own fp16
 * output per token (quantizer.hpp:146-213, same codes / s_a / z_a / row sums as
 * abq_quant_pack_act on that output) straight into the decode GEMV's code
 * layout; abq_linear_qact consumes it, so every projection that reads the same
 * activations (q/k/v, gate/up) shares one ReQuant.  m <= 8 tokens, per-token
 * asymmetric / symmetric / balanced spec, K % 8 == 0, K <= 16384.
 * err_index (device int64, may be NULL => synchronous check): the caller sets
 * it to -1; the smallest flat index of a non-finite output element is written
 * (atomic min), -1 stays when every element is finite. */
typedef struct {
  uint32_t* codes;      /* abq_qact_codes_bytes(m, k) bytes, device */
  double* scales;       /* [m] s_a */
  int32_t* zero_points; /* [m] z_a */
  int64_t* rowsums;     /* [m] code row sums */
  size_t m, k;
  unsigned bits;        /* activation bits the codes were made with */
} abq_qact;
size_t abq_qact_codes_bytes(size_t m, size_t k);
/* y = fp16(gain * fp16(x * rsqrt(mean(x^2) + eps))), x / gain / y_out fp16 [m][k] / [k]
 * (LLaMA RMSNorm); y_out may be NULL. */
int abq_rmsnorm_quant(const void* x, const void* gain, float eps, size_t m, size_t k,
                      const abq_quant_spec* spec, void* y_out, const abq_qact* out, int64_t* err_index,
                      void* stream);
/* y = fp16(fp16(silu(gate)) * up), fp16 [m][k]; y_out may be NULL. */
int abq_silu_mul_quant(const void* gate, const void* up, size_t m, size_t k, const abq_quant_spec* spec,
                       void* y_out, const abq_qact* out, int64_t* err_index, void* stream);
/* decode linear on producer-quantized activations (w->frag required): one
 * GEMV launch, no ReQuant phases on its critical path. */
int abq_linear_qact(const abq_qact* act, const abq_weights* w, void* y, int out_kind, void* stream);

/* ---- end-to-end serving with host buffers ----------------------------------
 * abq_stage_in: device dst <- pinned host src (read over PCIe by a kernel
 * through the UVA address; 16-B aligned), PDL-chained: the loads are issued as
 * soon as the kernel starts (overlapping the previous kernel), the stores after
 * griddepcontrol.wait, so a following engine linear starts streaming its
 * weights early and only its activation read waits for the copy.  The engine
 * linears accept pinned host memory as their output y (the epilogue writes the
 * result over PCIe): one H2D kernel + one linear per step, no copy nodes. */
int abq_stage_in(void* dst, const void* src_host, size_t bytes, void* stream);
/* abq_stage_in(x_stage <- x_host) + abq_linear(x_stage -> y_host) in one call
 * (x_host / y_host pinned host memory, x_stage an m*k device buffer): the
 * end-to-end serving step on host buffers. */
int abq_linear_host(const void* x_host, int x_dtype, size_t m, size_t k, void* x_stage,
                    const abq_quant_spec* act_spec, const abq_weights* w, void* y_host, int out_kind,
                    void* workspace, size_t workspace_bytes, int64_t* err_index, void* stream);

/* ---- kernel selection (decode GEMV variants) -------------- */
typedef enum {
  ABQ_GEMV_AUTO = 0,
  ABQ_GEMV_POPC = 1,   /* bit-serial AND + popcount over p x q plane pairs */
  ABQ_GEMV_RECOMB = 2  /* plane -> u8 recombination in registers + IMMA */
} abq_gemv_variant;
int abq_set_gemv_variant(int variant);
int abq_get_gemv_variant(void);

/* prefill GEMM schedule (tcgen05 path, m >= 9): one CTA per 128-channel row
 * tile, or stream-K over all SMs (CTAs share (row-tile, k-block) units and
 * hand partial tiles to the tile's finisher).  Results are identical; the
 * GPU-side counterpart of the reference's tile choice, picked by
 * abq.autotune_linear.  Process-global, like engine_threads (gemm.hpp:81-84). */
typedef enum {
  ABQ_GEMM_AUTO = 0,
  ABQ_GEMM_CLASSIC = 1,
  ABQ_GEMM_STREAM_K = 2
} abq_gemm_schedule;
int abq_set_gemm_schedule(int schedule);
int abq_get_gemm_schedule(void);

/* Launch-planning knobs for sweeps and tools (results never depend on them;
 * the defaults are the measured best): "dec_pre_kb" (decode GEMV weight-ring
 * KB issued before the activations are awaited, default 64), "dec_ring_kb"
 * (ring cap, 0 = whole CTA share), "dec_pdl" (0/1), "tc_dbg" (prefill GEMM
 * experiment switches, tools/trace_gemm.py), "tc_tt" (prefill token-tile cap),
 * "dec_pace_ns" (decode producer-warp slot spacing), "reset".  Returns ABQ_ERR_VALUE
 * for an unknown key. */
int abq_set_tuning(const char* key, long long value);

/* Profiling hook (phase stamps, [grid][64] u64 per launch, NULL = off).  The
 * stamps are compiled only into the trace build of the library
 * (make -C paper_2408_08554_b200/csrc TRACE=1 -> libabq_cuda_trace.so, loaded by
 * tools/trace_*.py via ABQ_LIB); in the product library this is a no-op. */
int abq_set_trace_buffer(void* dev_words);

#ifdef __cplusplus
}
#endif

#endif /* ABQ_CUDA_H_ */
