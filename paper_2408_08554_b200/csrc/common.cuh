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
