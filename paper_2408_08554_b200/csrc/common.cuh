// common.cuh -- shared helpers for the sm_100a ABQ engine (error state,
// launch accounting, epilogue parameters, small device utilities).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "abq_cuda.h"

namespace abq_dev {

// ---- host-side error state (thread-local, C-ABI abq_last_error) -----------
std::string& last_error();

// Process-wide launch-planning knobs, set through abq_set_tuning (tools and
// sweeps only; the defaults are the measured best).  Results never depend on them.
struct DecTuning {
  int pre_kb = -1;   // decode GEMV: weight-ring KB issued before the activations are awaited (-1 = auto)
  int ring_kb = 0;   // decode GEMV: ring size cap in KB (0 = the CTA's whole share when it fits)
  int pdl = 1;       // decode GEMV: programmatic dependent launch
  int pace_ns = 0;   // decode GEMV: producer-warp slot spacing while awaiting activations (0 = auto)
  int grid_balanced = 0;  // decode GEMV: fewer CTAs, all with the same row-tile count
  int tc_dbg = 0;    // prefill GEMM: experiment switches (tools/trace_gemm.py), 0 in production
  int tc_tt = 0;     // prefill GEMM: token-tile cap for the serving path (0 = by M)
  int tc_pre = 0;    // prefill GEMM: weight stages requested before the PDL wait (0 = the whole ring)
  int tc_sk_ctas = 2;  // prefill GEMM stream-K: CTAs per row-tile (grid = min(SMs, this x row-tiles))
  int next_kb = 64;  // decode GEMV: KB per CTA of the successor layer prefetched into L2 in the tail (0 = off)
  int next_min_kb = 128;  // ... only when this layer's per-CTA weight share is at least this long
  int next_at = 100;      // ... issued once this percentage of the CTA's share has landed
  int l2_plain = 0;  // decode GEMV: weight TMA without the L2 evict-first hint
  int dbg_nostream = 0;  // decode GEMV, TRACE build only: no weight stream (timing experiment, results invalid)
};
DecTuning& dec_tuning();

// the layer the caller runs next (abq_weights.next): its decode-layout weights
// are prefetched into L2 in this layer's tail
struct DecNext {
  const uint32_t* frag;
  unsigned q;
  size_t n, k;
};

// engine schedule picked from a TileConfig (abi.cu plan_of): token-tile cap
// (0 = by M) and the prefill GEMM schedule (ABQ_GEMM_*, 0 = auto)
struct EnginePlan {
  int token_tile;
  int schedule;
};
int fail(int status, const char* fmt, ...);
uint64_t& launch_counter();
int num_sms();

#define ABQ_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::abq_dev::fail(ABQ_ERR_CUDA, "%s: CUDA error %s (%s:%d)", __func__,   \
                             cudaGetErrorString(_e), __FILE__, __LINE__);           \
  } while (0)

// checks the launch that was just issued and counts it
#define ABQ_LAUNCHED()                                                              \
  do {                                                                              \
    ++::abq_dev::launch_counter();                                                  \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess)                                                          \
      return ::abq_dev::fail(ABQ_ERR_CUDA, "%s: launch failed: %s (%s:%d)", __func__, \
                             cudaGetErrorString(_e), __FILE__, __LINE__);           \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline size_t wpr_of(size_t cols) { return (cols + 63) / 64; }

// "Code slices": the prepacked weight layouts store the q-bit weight codes
// split into power-of-two-wide slices (the binary decomposition of q, widest
// first: 7 = 4 + 2 + 1), slice i holding code bits [slice_off(q,i),
// slice_off + slice_width).  A w-bit slice packs 32/w fields per u32 word as
// (8/w) groups of 4 byte lanes -- bits [8b + w*s, 8b + w*s + w) -- so the
// kernels widen it to byte codes with one shift and one mask per group,
// ((x >> w*s) & ((2^w - 1) * 0x01010101)), instead of one shift + merge per
// bit plane.  Same byte count as the ABQP planes; q = 1 is exactly a plane.
__host__ __device__ constexpr int slice_count(int q) { return (q & 1) + ((q >> 1) & 1) + ((q >> 2) & 1) + (q >> 3); }
__host__ __device__ constexpr int slice_width(int q, int i) {
  int seen = 0;
  for (int b = 3; b >= 0; --b)
    if (q & (1 << b)) {
      if (seen == i) return 1 << b;
      ++seen;
    }
  return 0;
}
__host__ __device__ constexpr int slice_off(int q, int i) {
  int off = 0;
  for (int j = 0; j < i; ++j) off += slice_width(q, j);
  return off;
}
// slice holding code bit `bit`
__host__ __device__ constexpr int slice_of_bit(int q, int bit) {
  int i = 0;
  while (slice_off(q, i) + slice_width(q, i) <= bit) ++i;
  return i;
}

// u8 activation codes of the tcgen05 GEMM, "tiled": [k-block of 128][token
// group of 8][16-k chunk][token % 8][16 B].  A tile of TT tokens x 128 k is
// one contiguous TT * 128-byte run (one TMA bulk copy) that is directly a UMMA
// K-major no-swizzle operand (core matrices 8 tokens x 16 B).  Groups are
// allocated for m rounded up to 256 tokens so that every token tile is in
// bounds; codes past K (to the 128 multiple) are zero.
__host__ __device__ inline int tc_act_groups(long long m) { return static_cast<int>(((m + 255) / 256) * 32); }
__host__ __device__ inline size_t tc_act_offset(long long tok, long long k, int groups) {
  return ((static_cast<size_t>(k >> 7) * groups + static_cast<size_t>(tok >> 3)) * 8 + ((k >> 4) & 7)) * 128 +
         (tok & 7) * 16 + (k & 15);
}
inline size_t tc_act_bytes(size_t m, size_t k) {
  return static_cast<size_t>(tc_act_groups(static_cast<long long>(m))) * 8 * ((k + 127) / 128) * 128;
}

// Kernel parameters live in constant bank 0 and are fetched through the
// constant cache on first use.  Kernels that start a TMA stream of ~200 KB per
// SM must touch their parameter block BEFORE the stream: a constant-cache miss
// issued behind it waits microseconds for the SM's memory queue to drain.
// One warp reads one word per 32 B of the block and consumes it.
template <typename T>
__device__ __forceinline__ void warm_param_block(const T& params, int lane) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&params);
  constexpr int kWords = static_cast<int>(sizeof(T) / 4);
  for (int i = lane * 8; i < kWords; i += 256) {
    const uint32_t v = w[i];
    asm volatile("" ::"r"(v));
  }
}

// QuantSpec as the kernels see it (quantizer.hpp:37-71)
struct QuantParams {
  unsigned bits;
  int scheme;
  int per_tensor;
  double alpha;
  double beta;
  unsigned levels;  // QuantSpec::levels
};

// ---- fused epilogue (K4): bit reduction result -> zero-point correction ->
// dequant, gemm.hpp:235-254 and 292-306 --------------------------------------
enum EpiMode : int {
  EPI_ACC_I32 = 0,   // raw acc (gemm_arbitrary)
  EPI_ACC_I64 = 1,   // raw acc (gemm_arbitrary_wide)
  EPI_F64 = 2,       // s_a*s_b*corrected, IEEE double (API parity)
  EPI_F16 = 3,       // same double rounded to fp16
  EPI_F32 = 4,       // same double rounded to fp32
  EPI_CORR_I64 = 5,  // corrected accumulator
};

struct EpiParams {
  int mode;
  void* out;
  long long ldo;
  const double* s_a;
  int sa_stride;
  const int32_t* z_a;
  int za_stride;
  const int64_t* rowsum_a;
  const double* s_b;
  int sb_stride;
  const int32_t* z_b;
  int zb_stride;
  const int64_t* colsum_b;
  long long k;
};

// epilogue with the activation-side values already in hand (sa, za, rowsum of
// token i), used by kernels that computed them on chip.
__device__ __forceinline__ void epi_store_v(const EpiParams& e, long long i, long long j,
                                            long long acc, double sa, long long za, long long ra) {
  const long long o = i * e.ldo + j;
  if (e.mode == EPI_ACC_I32) {
    static_cast<int32_t*>(e.out)[o] = static_cast<int32_t>(acc);
    return;
  }
  if (e.mode == EPI_ACC_I64) {
    static_cast<int64_t*>(e.out)[o] = acc;
    return;
  }
  // corrected = acc - z_a*colsum_b - z_b*rowsum_a + K*z_a*z_b   (int64, gemm.hpp:248-250)
  const long long zb = e.z_b[j * e.zb_stride];
  const long long corr = acc - za * e.colsum_b[j] - zb * ra + e.k * za * zb;
  if (e.mode == EPI_CORR_I64) {
    static_cast<int64_t*>(e.out)[o] = corr;
    return;
  }
  // s_a[i] * s_b[j] * corrected, left to right, no contraction (gemm.hpp:298)
  const double y = __dmul_rn(__dmul_rn(sa, e.s_b[j * e.sb_stride]), static_cast<double>(corr));
  if (e.mode == EPI_F64)
    static_cast<double*>(e.out)[o] = y;
  else if (e.mode == EPI_F16)
    static_cast<__half*>(e.out)[o] = __double2half(y);
  else
    static_cast<float*>(e.out)[o] = __double2float_rn(y);
}

__device__ __forceinline__ void epi_store(const EpiParams& e, long long i, long long j,
                                          long long acc) {
  if (e.mode == EPI_ACC_I32 || e.mode == EPI_ACC_I64) {
    epi_store_v(e, i, j, acc, 0.0, 0, 0);
    return;
  }
  epi_store_v(e, i, j, acc, e.s_a[i * e.sa_stride], e.z_a[i * e.za_stride], e.rowsum_a[i]);
}

// ---- ordered-key encoding so that atomicMin/Max on u64 orders doubles -----
__device__ __forceinline__ unsigned long long dkey(double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

}  // namespace abq_dev
