// quant_dev.cuh -- device-side restatement of the reference quantizer math
// (quantizer.hpp:146-213), shared by the standalone K1 kernels and the fused
// GEMV prologue.  Every FP64 operation is an explicit round-to-nearest
// intrinsic or IEEE division, so no FMA contraction can change a result;
// round() is half-away-from-zero like std::round (core.hpp:145).
#pragma once

#include <math_constants.h>

#include "common.cuh"

namespace abq_dev {

template <typename T>
__device__ __forceinline__ double load_as_double(const T* p, size_t idx);
template <>
__device__ __forceinline__ double load_as_double<__half>(const __half* p, size_t idx) {
  return static_cast<double>(__half2float(p[idx]));
}
template <>
__device__ __forceinline__ double load_as_double<float>(const float* p, size_t idx) {
  return static_cast<double>(p[idx]);
}
template <>
__device__ __forceinline__ double load_as_double<double>(const double* p, size_t idx) {
  return p[idx];
}

// value after the optional compensation pair: v = x + a[i]*b[j]  (quantizer.hpp:161-166)
template <typename T>
__device__ __forceinline__ double value_at(const T* x, size_t cols, size_t i, size_t j,
                                           const double* ca, const double* cb) {
  double v = load_as_double(x, i * cols + j);
  if (ca) v = __dadd_rn(v, __dmul_rn(ca[i], cb[j]));
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// step and zero point of one axis group (quantizer.hpp:169-201)
__device__ __forceinline__ void group_params(const QuantParams& qp, double lo_raw, double hi_raw,
                                             double* step_out, int* z_out) {
  const double lo = __dmul_rn(qp.beta, lo_raw);
  const double hi = __dmul_rn(qp.alpha, hi_raw);
  double step;
  int z;
  if (qp.scheme == ABQ_ASYMMETRIC) {
    if (hi == lo) {
      step = 1.0;
      z = 0;
    } else {
      step = __dsub_rn(hi, lo) / static_cast<double>(qp.levels - 1);
      double zz = round(-lo / step);
      const double top = static_cast<double>(qp.levels - 1);
      zz = zz < 0.0 ? 0.0 : (top < zz ? top : zz);
      z = static_cast<int>(zz);
    }
  } else {
    const double alo = fabs(lo), ahi = fabs(hi);
    const double amax = alo < ahi ? ahi : alo;
    const int half = 1 << (qp.bits - 1);
    if (amax == 0.0) {
      step = 1.0;
      z = 0;
    } else {
      if (qp.scheme == ABQ_BALANCED)
        step = amax / static_cast<double>(half);
      else
        step = qp.bits == 1 ? amax : amax / static_cast<double>(half - 1);
      z = half;
    }
  }
  *step_out = step;
  *z_out = z;
}

// code = clamp(round(v/step) + z, 0, L-1)  (quantizer.hpp:205-210)
__device__ __forceinline__ unsigned quant_code(double v, double step, double z, double top) {
  double c = __dadd_rn(round(v / step), z);
  c = c < 0.0 ? 0.0 : (top < c ? top : c);
  return static_cast<unsigned>(c);
}

// Same result as quant_code, with the IEEE division replaced by a multiply by
// the reciprocal except near rounding ties.  q1 = RN(v * RN(1/step)) is within
// a few ulp of RN(v/step); round() only changes value across half-integers, so
// whenever q1 is farther than a generous 2^-44 relative band from the nearest
// n + 1/2 both quotients round to the same integer.  Inside the band the exact
// IEEE quotient is used.  (Bit-exactness is tested against the reference on
// every quantizer case, tests/test_gpu_parity.py.)
__device__ __forceinline__ unsigned quant_code_fast(double v, double step, double inv_step,
                                                    double z, double top) {
  double q = __dmul_rn(v, inv_step);
  const double f = floor(q);
  const double d = fabs(__dsub_rn(__dsub_rn(q, f), 0.5));
  if (d <= fmax(fabs(q), 1.0) * 5.6843418860808015e-14) q = v / step;  // 2^-44
  double c = __dadd_rn(round(q), z);
  c = c < 0.0 ? 0.0 : (top < c ? top : c);
  return static_cast<unsigned>(c);
}

// RN32(1/step) for quant_code_f32, or NaN (forcing its exact path) where the
// fp32 reciprocal would lose precision (denormal) or overflow.
__device__ __forceinline__ float f32_reciprocal(double step) {
  return step > 0x1p-100 && step < 0x1p100 ? static_cast<float>(1.0 / step) : CUDART_NAN_F;
}

// Same bound via the fp32 reciprocal of RN32(step) (no FP64 division on the
// prologue's critical path): inv32 is within (1 + 2^-24)^2 - 1 < 2^-22.9 of
// 1/step, so q = RN32(v * inv32) in quant_code_f32 / quant_codes8_f16 is within
// |q| * 2^-22.3 of v/step, still inside their 2^-21 tie band.
__device__ __forceinline__ float f32_reciprocal_fast(double step) {
  return step > 0x1p-100 && step < 0x1p100 ? __frcp_rn(__double2float_rn(step)) : CUDART_NAN_F;
}

// group_params plus inv32 = f32_reciprocal_fast(step), with the asymmetric
// zero point z = clamp(round(RN64(-lo / step))) taken from the fp32 quotient
// qz = RN32(RN32(-lo) * inv32) -- within |qz| * 2^-21.9 of -lo/step -- whenever
// qz is farther than max(|qz|, 1) * 2^-20 from the nearest n + 1/2 (then both
// round to rint(qz)); otherwise, and for |qz| >= 2^22, by the IEEE quotient.
// One FP64 division (step) on the prologue's critical path instead of three.
// the rare paths out of line (small inline code).  Results are returned BY
// VALUE: an out-of-line callee writing through pointers puts the caller's
// variables in local memory, and a local-memory miss behind the SM's TMA weight
// stream is a full L2 round trip on the critical path.
struct StepZ {
  double step;
  int z;
};
static __device__ __noinline__ StepZ group_params_ool(QuantParams qp, double lo_raw, double hi_raw) {
  StepZ r;
  group_params(qp, lo_raw, hi_raw, &r.step, &r.z);
  return r;
}
static __device__ __noinline__ double round_div_ool(double a, double b) { return round(a / b); }

__device__ __forceinline__ void group_params_fast(const QuantParams& qp, double lo_raw, double hi_raw,
                                                  double* step_out, int* z_out, float* inv_out) {
  if (qp.scheme != ABQ_ASYMMETRIC) {
    const StepZ r = group_params_ool(qp, lo_raw, hi_raw);
    *step_out = r.step;
    *z_out = r.z;
    *inv_out = f32_reciprocal_fast(r.step);
    return;
  }
  const double lo = __dmul_rn(qp.beta, lo_raw);
  const double hi = __dmul_rn(qp.alpha, hi_raw);
  if (hi == lo) {
    *step_out = 1.0;
    *z_out = 0;
    *inv_out = 1.0f;
    return;
  }
  const double step = __dsub_rn(hi, lo) / static_cast<double>(qp.levels - 1);
  const float inv32 = f32_reciprocal_fast(step);
  const float q = __fmul_rn(__double2float_rn(-lo), inv32);
  const float t = __fadd_rn(q, 12582912.0f);  // 1.5 * 2^23
  const float r = __fsub_rn(t, 12582912.0f);
  const float d = __fsub_rn(0.5f, fabsf(__fsub_rn(q, r)));
  double zz = (fabsf(q) < 4194304.0f && d > fmaxf(fabsf(q), 1.0f) * 9.5367431640625e-07f)  // 2^22, 2^-20
                  ? static_cast<double>(r)
                  : round_div_ool(-lo, step);
  const double top = static_cast<double>(qp.levels - 1);
  zz = zz < 0.0 ? 0.0 : (top < zz ? top : zz);
  *step_out = step;
  *z_out = static_cast<int>(zz);
  *inv_out = inv32;
}

// Same result as quant_code for a value exactly representable in fp32 (fp16 /
// fp32 activations without a compensation pair), on the fp32 pipe.
// q = RN32(v * RN32(1/step)) is within |q| * 2^-22.9 of the reference's
// RN64(v / step); round() only changes value across half-integers, so when q is
// farther than |q| * 2^-21 from the nearest n + 1/2 both round to the same
// integer r, which is then rint(q) (magic-number add, no conversion unit).
// Otherwise -- or for |q| >= 2^22 -- the exact FP64 path decides.
// z, top: integers in [0, 255] (group_params clamps the zero point).
__device__ __forceinline__ unsigned quant_code_f32(float v, double step, float inv32, int z, int top) {
  const float q = __fmul_rn(v, inv32);
  const float t = __fadd_rn(q, 12582912.0f);  // 1.5 * 2^23: rint(q) in the low mantissa bits
  const float r = __fsub_rn(t, 12582912.0f);
  const float d = __fsub_rn(0.5f, fabsf(__fsub_rn(q, r)));  // distance to the nearest n + 1/2
  if (!(fabsf(q) < 4194304.0f && d > fmaxf(fabsf(q), 1.0f) * 4.76837158203125e-07f))  // 2^22, 2^-21
    return quant_code(static_cast<double>(v), step, static_cast<double>(z), static_cast<double>(top));
  const int c = (__float_as_int(t) - 0x4B400000) + z;
  return static_cast<unsigned>(c < 0 ? 0 : (c > top ? top : c));
}

// Exact code of an fp16 value x whose fp32 quotient estimate q = RN32(x RN32(1/step))
// lies in the tie band, without the FP64 division: |q| is within the band
// (< 1/4 for |q| < 2^19) of h = floor(|q|) + 1/2, so round(RN64(|x|/step)) is
// floor(|q|) + 1 iff RN64(|x|/step) >= h.  With r = RN(|x| - h step) (one FMA,
// sign exact): r >= 0 => |x|/step >= h.  Else D = h step - |x| > 0 and
// RN64(|x|/step) = h iff |x|/step is above the midpoint of h and its double
// predecessor h - u, i.e. D < T = (u/2) step (T exact: u is a power of two):
// RN(D) < T => yes, RN(D) > T => no; RN(D) == T (or |q| >= 2^19) is left to
// the division (*ok = false).  code = clamp(sign(x) * mag + z, 0, top), as
// quant_code (quantizer.hpp:205-209: round half away from zero, then + z).
__device__ __forceinline__ int quant_code_tie(float xf, float q, double step, int z, int top, bool* ok) {
  const float qa = fabsf(q);
  if (!(qa < 524288.0f)) {
    *ok = false;
    return 0;
  }
  const double n = floor(static_cast<double>(qa)), h = n + 0.5;
  const double r = __fma_rn(-h, step, fabs(static_cast<double>(xf)));
  int mag = static_cast<int>(n) + 1;
  if (r < 0.0) {
    const double u = h - __longlong_as_double(__double_as_longlong(h) - 1);
    const double T = __dmul_rn(__dmul_rn(u, 0.5), step), d = -r;
    if (d > T) mag -= 1;
    else if (!(d < T)) {
      *ok = false;
      return 0;
    }
  }
  const int c = (xf < 0.0f ? -mag : mag) + z;
  return c < 0 ? 0 : (c > top ? top : c);
}

// In-band elements (mask bit e of band) of a vector replaced by their exact
// codes (quant_code_tie inline; the FP64 division out of line only where that
// cannot decide).  Rare: about one element per 4096-wide token at 8-bit codes.
__device__ __forceinline__ uint3 quant_codes8_ties(const uint4& xv, double step, float inv32, int z, int top,
                                                   uint32_t band, uint32_t w0, uint32_t w1);

// Eight fp16 activations (one 16-byte vector) -> eight u8 codes (two words,
// element e in byte e%4 of word e/4), all on the fp32 pipe.  Elements inside
// the tie band of quant_code_f32 (mask bit e) are then replaced by their exact
// FP64 codes out of line, one FP64 division per flagged element: the band is
// ~2^-21 |q| wide, so at 8-bit codes about one element per 4096-wide token
// falls in it, and recomputing the whole vector cost that warp ~8 divisions on
// the critical path of every CTA.  Returns {word 0, word 1, code sum}, by value
// (a pointer argument would put the words in local memory).
static __device__ __noinline__ uint3 quant_codes8_patch(uint4 xv, double step, int z, int top, uint32_t band,
                                                        uint32_t w0, uint32_t w1) {
  const __half* hv = reinterpret_cast<const __half*>(&xv);
#pragma unroll 1
  for (int e = 0; e < 8; ++e) {
    if (!((band >> e) & 1u)) continue;
    const unsigned c = quant_code(static_cast<double>(__half2float(hv[e])), step, static_cast<double>(z),
                                  static_cast<double>(top));
    const uint32_t sh = 8u * static_cast<uint32_t>(e & 3), m = ~(0xFFu << sh);
    if (e < 4) w0 = (w0 & m) | (c << sh);
    else w1 = (w1 & m) | (c << sh);
  }
  uint32_t sum = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) sum += ((w0 >> (8 * b)) & 0xFFu) + ((w1 >> (8 * b)) & 0xFFu);
  return make_uint3(w0, w1, sum);
}
__device__ __forceinline__ uint3 quant_codes8_ties(const uint4& xv, double step, float inv32, int z, int top,
                                                   uint32_t band, uint32_t w0, uint32_t w1) {
  uint32_t slow = 0;
#pragma unroll 1
  for (uint32_t b = band; b; b &= b - 1u) {
    const int e = __ffs(static_cast<int>(b)) - 1;
    const uint32_t wd = (e >> 1) == 0 ? xv.x : (e >> 1) == 1 ? xv.y : (e >> 1) == 2 ? xv.z : xv.w;
    const float xf = __half2float(__ushort_as_half(static_cast<unsigned short>(wd >> (16 * (e & 1)))));
    bool ok = true;
    const uint32_t c = static_cast<uint32_t>(quant_code_tie(xf, __fmul_rn(xf, inv32), step, z, top, &ok));
    if (!ok) {
      slow |= 1u << e;
      continue;
    }
    const uint32_t sh = 8u * static_cast<uint32_t>(e & 3), m = ~(0xFFu << sh);
    if (e < 4) w0 = (w0 & m) | (c << sh);
    else w1 = (w1 & m) | (c << sh);
  }
  if (slow) return quant_codes8_patch(xv, step, z, top, slow, w0, w1);
  uint32_t sum = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) sum += ((w0 >> (8 * b)) & 0xFFu) + ((w1 >> (8 * b)) & 0xFFu);
  return make_uint3(w0, w1, sum);
}
__device__ __forceinline__ int quant_codes8_f16(const uint4& xv, double step, float inv32, int z, int top,
                                                uint32_t* w0, uint32_t* w1) {
  const __half2* h2 = reinterpret_cast<const __half2*>(&xv);
  int c[8];
  uint32_t band = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __half22float2(h2[e]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float v = h ? f.y : f.x;
      const float q = __fmul_rn(v, inv32);
      const float t = __fadd_rn(q, 12582912.0f);
      const float r = __fsub_rn(t, 12582912.0f);
      const float d = __fsub_rn(0.5f, fabsf(__fsub_rn(q, r)));
      const bool in = fabsf(q) < 4194304.0f && d > fmaxf(fabsf(q), 1.0f) * 4.76837158203125e-07f;
      band |= (in ? 0u : 1u) << (2 * e + h);
      const int ci = (__float_as_int(t) - 0x4B400000) + z;
      c[2 * e + h] = ci < 0 ? 0 : (ci > top ? top : ci);
    }
  }
  *w0 = static_cast<uint32_t>(c[0]) | (static_cast<uint32_t>(c[1]) << 8) | (static_cast<uint32_t>(c[2]) << 16) |
        (static_cast<uint32_t>(c[3]) << 24);
  *w1 = static_cast<uint32_t>(c[4]) | (static_cast<uint32_t>(c[5]) << 8) | (static_cast<uint32_t>(c[6]) << 16) |
        (static_cast<uint32_t>(c[7]) << 24);
  if (band) {
    const uint3 r = quant_codes8_ties(xv, step, inv32, z, top, band, *w0, *w1);
    *w0 = r.x;
    *w1 = r.y;
    return static_cast<int>(r.z);
  }
  return c[0] + c[1] + c[2] + c[3] + c[4] + c[5] + c[6] + c[7];
}

// Asymmetric per-token zero point and reciprocal step for the CODES, on the
// fp32 pipe (the exact FP64 step -- s_a for the epilogue -- is computed off the
// critical path): step32 = RN32(RN32(hi - lo) RN32(1/(L-1))), inv32 =
// RN32(1/step32) is within (1 + 2^-24)^4 - 1 < 2^-21.99 of 1/step; codes with
// it stay within 5 * 2^-24 < 2^-21 (the tie band) of v/step, and the zero point
// qz = RN32(-lo inv32) within 2^-21.6 < 2^-20 (its band here).  Returns false
// (caller takes group_params_fast) for other schemes, alpha or beta != 1, a
// zero point inside its band, or a step outside the normal range.
__device__ __forceinline__ bool codes_params_f32(const QuantParams& qp, float lo, float hi, float* inv_out,
                                                 int* z_out) {
  if (qp.scheme != ABQ_ASYMMETRIC || qp.alpha != 1.0 || qp.beta != 1.0) return false;
  if (hi == lo) {  // degenerate range: step 1, zero point 0 (quantizer.hpp:176-178)
    *inv_out = 1.0f;
    *z_out = 0;
    return true;
  }
  const float step32 = __fmul_rn(__fsub_rn(hi, lo), __frcp_rn(static_cast<float>(qp.levels - 1)));
  if (!(step32 > 0x1p-100f && step32 < 0x1p100f)) return false;
  const float inv32 = __frcp_rn(step32);
  const float q = __fmul_rn(-lo, inv32);
  const float t = __fadd_rn(q, 12582912.0f);
  const float d = __fsub_rn(0.5f, fabsf(__fsub_rn(q, __fsub_rn(t, 12582912.0f))));
  if (!(fabsf(q) < 4194304.0f && d > fmaxf(fabsf(q), 1.0f) * 9.5367431640625e-07f)) return false;  // 2^22, 2^-20
  const int top = static_cast<int>(qp.levels - 1), zi = __float_as_int(t) - 0x4B400000;
  *inv_out = inv32;
  *z_out = zi < 0 ? 0 : (zi > top ? top : zi);
  return true;
}

// Per-token form of the quant_codes8_f16 test: with Qmax >= |q| for every
// element of the token (band_threshold), |q - rint(q)| < thr = 0.5 - max(Qmax,
// 1) 2^-21 implies the element is outside the tie band of quant_code_f32, so
// one compare per element replaces the per-element band arithmetic.
__device__ __forceinline__ float band_threshold(float lo, float hi, float inv32) {
  const float qmax = __fmul_ru(fmaxf(fabsf(lo), fabsf(hi)), __fmul_ru(inv32, 1.0000010f));  // >= every |q|
  return qmax < 4194304.0f ? 0.5f - fmaxf(qmax, 1.0f) * 4.76837158203125e-07f : -1.0f;  // -1: all exact
}
__device__ __forceinline__ int quant_codes8_f16_band(const uint4& xv, double step, float inv32, float thr, int z,
                                                     int top, uint32_t* w0, uint32_t* w1) {
  const __half2* h2 = reinterpret_cast<const __half2*>(&xv);
  int c[8];
  uint32_t band = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __half22float2(h2[e]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float q = __fmul_rn(h ? f.y : f.x, inv32);
      const float t = __fadd_rn(q, 12582912.0f);  // 1.5 * 2^23: rint(q) in the low mantissa bits
      band |= (fabsf(__fsub_rn(q, __fsub_rn(t, 12582912.0f))) < thr ? 0u : 1u) << (2 * e + h);
      const int ci = (__float_as_int(t) - 0x4B400000) + z;
      c[2 * e + h] = ci < 0 ? 0 : (ci > top ? top : ci);
    }
  }
  *w0 = static_cast<uint32_t>(c[0]) | (static_cast<uint32_t>(c[1]) << 8) | (static_cast<uint32_t>(c[2]) << 16) |
        (static_cast<uint32_t>(c[3]) << 24);
  *w1 = static_cast<uint32_t>(c[4]) | (static_cast<uint32_t>(c[5]) << 8) | (static_cast<uint32_t>(c[6]) << 16) |
        (static_cast<uint32_t>(c[7]) << 24);
  if (band) {  // rare: exact codes of the flagged elements only
    const uint3 r = quant_codes8_ties(xv, step, inv32, z, top, band, *w0, *w1);
    *w0 = r.x;
    *w1 = r.y;
    return static_cast<int>(r.z);
  }
  return c[0] + c[1] + c[2] + c[3] + c[4] + c[5] + c[6] + c[7];
}

// nonzero iff one of the eight fp16 values is Inf or NaN (exponent all ones)
__device__ __forceinline__ uint32_t f16x8_nonfinite(const uint4& v) {
  const uint32_t m = 0x7C007C00u;
  auto one = [&](uint32_t w) {
    const uint32_t e = w & m;
    return static_cast<uint32_t>((e & 0xFFFFu) == 0x7C00u) | static_cast<uint32_t>((e >> 16) == 0x7C00u);
  };
  return one(v.x) | one(v.y) | one(v.z) | one(v.w);
}

}  // namespace abq_dev
