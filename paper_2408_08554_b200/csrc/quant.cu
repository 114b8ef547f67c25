// quant.cu -- K1 (activation ReQuant + BitPacking), bitpack / unpack, row
// sums, plane row sums, zero-point correction and bmma kernels for sm_100a.
//
// Reference semantics restated here (paths relative to /root/reference/proj):
//   quantize            include/abq/quantizer.hpp:146-213 (FP64, round half away)
//   bitpack / unpack    include/abq/bitplane.hpp:47-76     ([plane][row][word] LSB-first)
//   bmma                include/abq/bitplane.hpp:81-96
//   code_rowsums        include/abq/gemm.hpp:256-261
//   zero_point_correct  include/abq/gemm.hpp:235-254
//
// Bit-exactness notes: every FP64 operation of the reference is issued as an
// explicit round-to-nearest intrinsic (__dmul_rn / __dadd_rn / __dsub_rn /
// IEEE '/'), so ptxas can never contract a multiply-add into an FMA; CUDA's
// round() is round-half-away-from-zero like std::round.  fp16 -> double is
// exact, min / max are order-free.
#include <cfloat>

#include <math_constants.h>

#include "common.cuh"
#include "quant_dev.cuh"

namespace abq_dev {


// ---- per-tensor range (grid-wide) + non-finite detection ------------------
template <typename T>
__global__ void tensor_range_kernel(const T* __restrict__ x, size_t rows, size_t cols,
                                    const double* ca, const double* cb,
                                    unsigned long long* range /*[2]: min key, max key*/,
                                    unsigned long long* bad_index) {
  double lo = CUDART_INF, hi = -CUDART_INF;
  const size_t total = rows * cols;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t i = idx / cols, j = idx % cols;
    const double raw = load_as_double(x, idx);
    if (!isfinite(raw)) atomicMin(bad_index, static_cast<unsigned long long>(idx));
    const double v = ca ? __dadd_rn(raw, __dmul_rn(ca[i], cb[j])) : raw;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  __shared__ double s_lo[32], s_hi[32];
  lo = warp_min(lo);
  hi = warp_max(hi);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    lo = lane < nw ? s_lo[lane] : CUDART_INF;
    hi = lane < nw ? s_hi[lane] : -CUDART_INF;
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0) {
      atomicMin(&range[0], dkey(lo));
      atomicMax(&range[1], dkey(hi));
    }
  }
}

// ---- K1: one CTA per row: range -> (step, z) -> codes -> planes / rowsum ---
// planes written byte-wise: byte g of a plane row covers elements 8g..8g+7
// (little-endian u64 words, LSB-first), tail bytes up to wpr*8 are zeroed.
template <typename T>
__global__ void __launch_bounds__(256)
    quant_rows_kernel(const T* __restrict__ x, size_t rows, size_t cols, QuantParams qp,
                      const double* __restrict__ ca, const double* __restrict__ cb,
                      const unsigned long long* __restrict__ tensor_range,
                      uint8_t* __restrict__ codes, uint8_t* __restrict__ planes_bytes,
                      unsigned nplanes, double* __restrict__ scales,
                      int32_t* __restrict__ zero_points, int64_t* __restrict__ rowsums,
                      unsigned long long* __restrict__ bad_index) {
  __shared__ double s_lo[32], s_hi[32];
  __shared__ long long s_sum[32];
  __shared__ double s_step;
  __shared__ int s_z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t wpr = (cols + 63) / 64;
  const size_t row_bytes = wpr * 8;
  const size_t groups = (cols + 7) / 8;
  const double top = static_cast<double>(qp.levels - 1);

  for (size_t i = blockIdx.x; i < rows; i += gridDim.x) {
    if (!qp.per_tensor) {
      double lo = CUDART_INF, hi = -CUDART_INF;
      for (size_t j = threadIdx.x; j < cols; j += blockDim.x) {
        const double raw = load_as_double(x, i * cols + j);
        if (!isfinite(raw)) atomicMin(bad_index, static_cast<unsigned long long>(i * cols + j));
        const double v = ca ? __dadd_rn(raw, __dmul_rn(ca[i], cb[j])) : raw;
        lo = fmin(lo, v);
        hi = fmax(hi, v);
      }
      lo = warp_min(lo);
      hi = warp_max(hi);
      if (lane == 0) {
        s_lo[warp] = lo;
        s_hi[warp] = hi;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) {
          lo = fmin(lo, s_lo[w]);
          hi = fmax(hi, s_hi[w]);
        }
        lo = fmin(lo, s_lo[0]);
        hi = fmax(hi, s_hi[0]);
        double step;
        int z;
        group_params(qp, lo, hi, &step, &z);
        s_step = step;
        s_z = z;
        scales[i] = step;
        zero_points[i] = z;
      }
    } else if (threadIdx.x == 0) {
      double step;
      int z;
      group_params(qp, dkey_inv(tensor_range[0]), dkey_inv(tensor_range[1]), &step, &z);
      s_step = step;
      s_z = z;
      if (i == 0) {
        scales[0] = step;
        zero_points[0] = z;
      }
    }
    __syncthreads();
    const double step = s_step;
    const double zd = static_cast<double>(s_z);
    long long rsum = 0;
    for (size_t g = threadIdx.x; g < row_bytes; g += blockDim.x) {
      unsigned pbytes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (g < groups) {
        const size_t j0 = g * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const size_t j = j0 + e;
          if (j < cols) {
            const unsigned c = quant_code(value_at(x, cols, i, j, ca, cb), step, zd, top);
            rsum += c;
            if (codes) codes[i * cols + j] = static_cast<uint8_t>(c);
#pragma unroll
            for (int s = 0; s < 8; ++s) pbytes[s] |= ((c >> s) & 1u) << e;
          }
        }
      }
      if (planes_bytes)
        for (unsigned s = 0; s < nplanes; ++s)
          planes_bytes[(static_cast<size_t>(s) * rows + i) * row_bytes + g] =
              static_cast<uint8_t>(pbytes[s]);
    }
    if (rowsums) {
      rsum = warp_sum(rsum);
      if (lane == 0) s_sum[warp] = rsum;
      __syncthreads();
      if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < nw; ++w) t += s_sum[w];
        rowsums[i] = t;
      }
    }
    __syncthreads();
  }
}

// ---- bitpack of u8 codes (bitplane.hpp:47-64) ------------------------------
__global__ void bitpack_kernel(const uint8_t* __restrict__ codes, size_t rows, size_t cols,
                               unsigned bits, uint8_t* __restrict__ planes_bytes,
                               unsigned long long* __restrict__ bad_index) {
  const size_t row_bytes = ((cols + 63) / 64) * 8;
  const size_t total = rows * row_bytes;
  const unsigned max_code = bits >= 8 ? 255u : ((1u << bits) - 1u);
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t i = idx / row_bytes, g = idx % row_bytes;
    unsigned pb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const size_t j = g * 8 + e;
      if (j < cols) {
        const unsigned c = codes[i * cols + j];
        if (c > max_code) atomicMin(bad_index, static_cast<unsigned long long>(i * cols + j));
#pragma unroll
        for (int s = 0; s < 8; ++s) pb[s] |= ((c >> s) & 1u) << e;
      }
    }
    for (unsigned s = 0; s < bits; ++s)
      planes_bytes[(static_cast<size_t>(s) * rows + i) * row_bytes + g] = static_cast<uint8_t>(pb[s]);
  }
}

// ---- unpack (bitplane.hpp:66-76) ------------------------------------------
__global__ void unpack_kernel(const uint64_t* __restrict__ planes, unsigned bits, size_t rows,
                              size_t cols, uint8_t* __restrict__ codes) {
  const size_t wpr = (cols + 63) / 64;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < rows * cols;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t i = idx / cols, j = idx % cols;
    unsigned c = 0;
    for (unsigned s = 0; s < bits; ++s)
      c |= static_cast<unsigned>((planes[(static_cast<size_t>(s) * rows + i) * wpr + j / 64] >> (j % 64)) & 1u) << s;
    codes[idx] = static_cast<uint8_t>(c);
  }
}

// ---- code_rowsums (gemm.hpp:256-261): one warp per row --------------------
__global__ void code_rowsums_kernel(const uint8_t* __restrict__ codes, size_t rows, size_t cols,
                                    int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t i = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += warps) {
    long long s = 0;
    for (size_t j = lane; j < cols; j += 32) s += codes[i * cols + j];
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
}

// ---- plane row sums: sum_t 2^t popc(P_t[row]) = code row sum ---------------
__global__ void plane_rowsums_kernel(const uint64_t* __restrict__ planes, unsigned bits, size_t rows,
                                     size_t cols, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const size_t wpr = (cols + 63) / 64;
  const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t i = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += warps) {
    long long s = 0;
    for (unsigned t = 0; t < bits; ++t) {
      const uint64_t* r = planes + (static_cast<size_t>(t) * rows + i) * wpr;
      long long c = 0;
      for (size_t w = lane; w < wpr; w += 32) c += __popcll(r[w]);
      s += c << t;
    }
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
}

// ---- zero_point_correct (gemm.hpp:235-254) ---------------------------------
template <typename Acc>
__global__ void zero_point_correct_kernel(const Acc* __restrict__ acc, size_t m, size_t n,
                                          const int64_t* __restrict__ rowsum_a,
                                          const int64_t* __restrict__ colsum_b,
                                          const int32_t* __restrict__ z_a,
                                          const int32_t* __restrict__ z_b, long long k,
                                          Acc* __restrict__ out) {
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < m * n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t i = idx / n, j = idx % n;
    const long long v = static_cast<long long>(acc[idx]) - static_cast<long long>(z_a[i]) * colsum_b[j] -
                        static_cast<long long>(z_b[j]) * rowsum_a[i] +
                        k * static_cast<long long>(z_a[i]) * static_cast<long long>(z_b[j]);
    out[idx] = static_cast<Acc>(v);
  }
}

// ---- bmma: one plane pair (bitplane.hpp:81-96) -----------------------------
__global__ void bmma_kernel(const uint64_t* __restrict__ a, size_t m, unsigned a_plane,
                            const uint64_t* __restrict__ bt, size_t n, unsigned b_plane,
                            size_t wpr, int32_t* __restrict__ out) {
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < m * n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t i = idx / n, j = idx % n;
    const uint64_t* ra = a + (static_cast<size_t>(a_plane) * m + i) * wpr;
    const uint64_t* rb = bt + (static_cast<size_t>(b_plane) * n + j) * wpr;
    int acc = 0;
    for (size_t w = 0; w < wpr; ++w) acc += __popcll(ra[w] & rb[w]);
    out[idx] = acc;
  }
}

// ============================================================================
// host launchers (called from abi.cu)
// ============================================================================
static int grid_for(size_t work, int block) {
  size_t g = (work + block - 1) / block;
  size_t cap = static_cast<size_t>(num_sms()) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

template <typename T>
static int launch_quant(const T* x, size_t rows, size_t cols, const QuantParams& qp,
                        const double* ca, const double* cb, uint8_t* codes, uint64_t* planes,
                        unsigned nplanes, double* scales, int32_t* zps, int64_t* rowsums,
                        unsigned long long* bad, unsigned long long* range, cudaStream_t st) {
  if (qp.per_tensor) {
    tensor_range_kernel<T><<<grid_for(rows * cols, 256), 256, 0, st>>>(x, rows, cols, ca, cb,
                                                                      range, bad);
    ABQ_LAUNCHED();
  }
  const int grid = static_cast<int>(rows < static_cast<size_t>(num_sms()) * 8 ? rows : num_sms() * 8);
  quant_rows_kernel<T><<<grid > 0 ? grid : 1, 256, 0, st>>>(
      x, rows, cols, qp, ca, cb, range, codes, reinterpret_cast<uint8_t*>(planes), nplanes,
      scales, zps, rowsums, bad);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

// status/range init: bad = UINT64_MAX; range = {min key = max, max key = 0}
__global__ void scratch_init_kernel(unsigned long long* bad, unsigned long long* range) {
  *bad = ~0ull;
  if (range) {
    range[0] = ~0ull;
    range[1] = 0ull;
  }
}

int run_quantize(const void* x, int x_dtype, size_t rows, size_t cols, const QuantParams& qp,
                 const double* ca, const double* cb, uint8_t* codes, uint64_t* planes,
                 unsigned nplanes, double* scales, int32_t* zps, int64_t* rowsums,
                 unsigned long long* bad, unsigned long long* range, cudaStream_t st) {
  scratch_init_kernel<<<1, 1, 0, st>>>(bad, qp.per_tensor ? range : nullptr);
  ABQ_LAUNCHED();
  if (rows == 0 || cols == 0) {
    // reference: empty range -> lo=+inf, hi=-inf per group (no elements); rows==0 has no groups
    return ABQ_OK;
  }
  switch (x_dtype) {
    case ABQ_F16:
      return launch_quant(static_cast<const __half*>(x), rows, cols, qp, ca, cb, codes, planes,
                          nplanes, scales, zps, rowsums, bad, range, st);
    case ABQ_F32:
      return launch_quant(static_cast<const float*>(x), rows, cols, qp, ca, cb, codes, planes,
                          nplanes, scales, zps, rowsums, bad, range, st);
    case ABQ_F64:
      return launch_quant(static_cast<const double*>(x), rows, cols, qp, ca, cb, codes, planes,
                          nplanes, scales, zps, rowsums, bad, range, st);
    default:
      return fail(ABQ_ERR_VALUE, "quantize: unsupported input dtype %d", x_dtype);
  }
}

int run_bitpack(const uint8_t* codes, size_t rows, size_t cols, unsigned bits, uint64_t* planes,
                unsigned long long* scratch, cudaStream_t st) {
  scratch_init_kernel<<<1, 1, 0, st>>>(scratch, nullptr);
  ABQ_LAUNCHED();
  const size_t work = rows * wpr_of(cols) * 8;
  if (work == 0) return ABQ_OK;
  bitpack_kernel<<<grid_for(work, 256), 256, 0, st>>>(codes, rows, cols, bits,
                                                      reinterpret_cast<uint8_t*>(planes), scratch);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

int run_unpack(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, uint8_t* codes,
               cudaStream_t st) {
  if (rows * cols == 0) return ABQ_OK;
  unpack_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(planes, bits, rows, cols, codes);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

int run_code_rowsums(const uint8_t* codes, size_t rows, size_t cols, int64_t* out, cudaStream_t st) {
  if (rows == 0) return ABQ_OK;
  code_rowsums_kernel<<<grid_for(rows * 32, 256), 256, 0, st>>>(codes, rows, cols, out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

// ---- dequantize  quantizer.hpp:243-254: out = (code - z) * step (FP64, RN) ---
__global__ void dequantize_kernel(const uint8_t* __restrict__ codes, size_t rows, size_t cols,
                                  const double* __restrict__ scales, const int32_t* __restrict__ zps,
                                  int per_tensor, double* __restrict__ out) {
  const size_t total = rows * cols, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const size_t g = per_tensor ? 0 : idx / cols;
    out[idx] = __dmul_rn(__dsub_rn(static_cast<double>(codes[idx]), static_cast<double>(zps[g])), scales[g]);
  }
}

int run_dequantize(const uint8_t* codes, size_t rows, size_t cols, const double* scales, const int32_t* zps,
                   int per_tensor, double* out, cudaStream_t st) {
  if (rows == 0 || cols == 0) return ABQ_OK;
  dequantize_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(codes, rows, cols, scales, zps, per_tensor, out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

int run_plane_rowsums(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, int64_t* out,
                      cudaStream_t st) {
  if (rows == 0) return ABQ_OK;
  plane_rowsums_kernel<<<grid_for(rows * 32, 256), 256, 0, st>>>(planes, bits, rows, cols, out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <typename Acc>
int run_zero_point_correct(const Acc* acc, size_t m, size_t n, const int64_t* ra, const int64_t* cb,
                           const int32_t* za, const int32_t* zb, size_t k, Acc* out, cudaStream_t st) {
  if (m * n == 0) return ABQ_OK;
  zero_point_correct_kernel<Acc><<<grid_for(m * n, 256), 256, 0, st>>>(
      acc, m, n, ra, cb, za, zb, static_cast<long long>(k), out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}
template int run_zero_point_correct<int32_t>(const int32_t*, size_t, size_t, const int64_t*,
                                             const int64_t*, const int32_t*, const int32_t*, size_t,
                                             int32_t*, cudaStream_t);
template int run_zero_point_correct<int64_t>(const int64_t*, size_t, size_t, const int64_t*,
                                             const int64_t*, const int32_t*, const int32_t*, size_t,
                                             int64_t*, cudaStream_t);

int run_bmma(const uint64_t* a, size_t m, unsigned a_plane, const uint64_t* bt, size_t n,
             unsigned b_plane, size_t k, int32_t* out, cudaStream_t st) {
  if (m * n == 0) return ABQ_OK;
  bmma_kernel<<<grid_for(m * n, 256), 256, 0, st>>>(a, m, a_plane, bt, n, b_plane, wpr_of(k), out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

}  // namespace abq_dev
