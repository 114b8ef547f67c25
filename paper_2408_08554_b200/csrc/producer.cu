// producer.cu -- ReQuant fused into the ops that PRODUCE a decode linear's
// input (the reference's quant_linear re-quantizes the output
// of rmsnorm / silu(gate) * up, toyblock.hpp:220-245 and 252-282):
//
//   rmsnorm_quant_kernel   x (fp16) -> y = fp16(gain * fp16(x * rsqrt(mean(x^2) + eps)))
//   silu_mul_quant_kernel  gate, up (fp16) -> y = fp16(fp16(silu(gate)) * up)
//
// and, in the same kernel, the per-token ReQuant of y (quantizer.hpp:146-213,
// FP64 semantics, the same code path as the fused GEMV prologue: exact range
// in the ordered-int image of fp32, one FP64 division, fp32 codes with an
// exact FP64 tie path) written straight into the decode GEMV's B-fragment
// code layout + s_a / z_a / code row sums.  The consuming GEMV
// (abq_linear_qact) then starts its main loop right after copying the codes:
// no range / step / code phases on its critical path, and one producer feeds
// every projection that reads the same activations (q/k/v, gate/up).
//
// One CTA per token, kProdThreads threads, the row kept in registers.
#include <math_constants.h>

#include <algorithm>

#include "common.cuh"
#include "gemv_frag.cuh"
#include "quant_dev.cuh"

namespace abq_dev {

constexpr int kProdThreads = 256;
constexpr int kProdNV = 8;  // 16-byte vectors of 8 fp16 per thread: K <= 8 * 8 * 256 = 16384

// the decode GEMV's token tile for m tokens (gemv_dec.cu dec_mt)
static inline int qact_mt(size_t m) { return m <= 1 ? 1 : m <= 2 ? 2 : m <= 4 ? 4 : 8; }

struct ProdSmem {
  float red[kProdThreads / 32];
  int lo[kProdThreads / 32], hi[kProdThreads / 32];
  int sum[kProdThreads / 32];
};

// ReQuant of the CTA's token row held in registers (v[r] = elements
// 8 (tid + r T) .. +7) into the B-fragment code layout; writes s_a / z_a /
// rowsum of the token.  Non-finite elements: atomicMin of the flat index.
__device__ void requant_row_f16(const uint4 (&v)[kProdNV], int nvec, int k, int tok, int mt, int kpad,
                                const QuantParams& qp, uint32_t* codes, double* s_a, int32_t* z_a,
                                long long* rowsum, unsigned long long* err, ProdSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto ord = [](float f) {
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7FFFFFFF;
  };
  auto unord = [](int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); };
  int lo = 0x7FFFFFFF, hi = static_cast<int>(0x80000000u);
  uint32_t bad = 0;
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    if (tid + r * kProdThreads >= nvec) break;
    bad |= f16x8_nonfinite(v[r]);
    const __half2* h2 = reinterpret_cast<const __half2*>(&v[r]);
    __half2 mn = h2[0], mx = h2[0];
#pragma unroll
    for (int e = 1; e < 4; ++e) {
      mn = __hmin2(mn, h2[e]);
      mx = __hmax2(mx, h2[e]);
    }
    lo = min(lo, min(ord(__low2float(mn)), ord(__high2float(mn))));
    hi = max(hi, max(ord(__low2float(mx)), ord(__high2float(mx))));
  }
  if (bad && err) {
#pragma unroll
    for (int r = 0; r < kProdNV; ++r) {
      const int idx = tid + r * kProdThreads;
      if (idx >= nvec) break;
      const __half* h = reinterpret_cast<const __half*>(&v[r]);
      for (int e = 0; e < 8; ++e)
        if (!isfinite(__half2float(h[e])))
          atomicMin(err, static_cast<unsigned long long>(tok) * k + static_cast<unsigned long long>(idx) * 8 + e);
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane == 0) {
    sm.lo[warp] = lo;
    sm.hi[warp] = hi;
  }
  __syncthreads();
  int l2 = lane < kProdThreads / 32 ? sm.lo[lane] : 0x7FFFFFFF;
  int h2 = lane < kProdThreads / 32 ? sm.hi[lane] : static_cast<int>(0x80000000u);
  l2 = __reduce_min_sync(0xffffffffu, l2);
  h2 = __reduce_max_sync(0xffffffffu, h2);
  double step = 0.0;
  int z = 0;
  float inv32 = 0.0f;
  group_params_fast(qp, unord(l2), unord(h2), &step, &z, &inv32);
  if (tid == 0) {
    s_a[tok] = step;
    z_a[tok] = z;
  }
  const int topi = static_cast<int>(qp.levels - 1);
  const int tb = tok / mt, i = tok % mt;
  uint32_t* dst = codes + static_cast<size_t>(tb) * mt * kpad / 4;
  int rsum = 0;
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    const int idx = tid + r * kProdThreads;
    if (idx >= nvec) break;
    uint32_t w0, w1;
    rsum += quant_codes8_f16(v[r], step, inv32, z, topi, &w0, &w1);
    dst[act_frag_index(2 * idx, i, mt)] = w0;
    dst[act_frag_index(2 * idx + 1, i, mt)] = w1;
  }
  for (int g4 = k / 4 + tid; g4 < kpad / 4; g4 += kProdThreads) dst[act_frag_index(g4, i, mt)] = 0u;
  rsum = __reduce_add_sync(0xffffffffu, rsum);  // <= 255 * 16384 < 2^31
  if (lane == 0) sm.sum[warp] = rsum;
  __syncthreads();
  if (tid == 0) {
    long long s = 0;
    for (int w = 0; w < kProdThreads / 32; ++w) s += sm.sum[w];
    rowsum[tok] = s;
  }
}

__global__ void __launch_bounds__(kProdThreads) rmsnorm_quant_kernel(
    const __half* __restrict__ x, const __half* __restrict__ gain, float eps, int k, int mt, int kpad,
    QuantParams qp, __half* __restrict__ y_out, uint32_t* __restrict__ codes, double* __restrict__ s_a,
    int32_t* __restrict__ z_a, long long* __restrict__ rowsum, unsigned long long* __restrict__ err) {
  __shared__ ProdSmem sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tok = blockIdx.x;
  const int nvec = k >> 3;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // x may come from the previous kernel
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(tok) * k);
  uint4 v[kProdNV];
  float ss = 0.0f;
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    const int idx = tid + r * kProdThreads;
    v[r] = idx < nvec ? __ldg(xr + idx) : make_uint4(0u, 0u, 0u, 0u);
  }
  // the consumers (GEMV launches) may start streaming their weights now
  asm volatile("griddepcontrol.launch_dependents;");
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    const __half2* h2 = reinterpret_cast<const __half2*>(&v[r]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h2[e]);
      ss = fmaf(f.x, f.x, ss);
      ss = fmaf(f.y, f.y, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) sm.red[warp] = ss;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int w = 0; w < kProdThreads / 32; ++w) tot += sm.red[w];
  const float rstd = rsqrtf(tot / static_cast<float>(k) + eps);
  const uint4* gr = reinterpret_cast<const uint4*>(gain);
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    const int idx = tid + r * kProdThreads;
    if (idx >= nvec) break;
    const uint4 gv = __ldg(gr + idx);
    __half2* h2 = reinterpret_cast<__half2*>(&v[r]);
    const __half2* g2 = reinterpret_cast<const __half2*>(&gv);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h2[e]);
      const __half2 nrm = __floats2half2_rn(f.x * rstd, f.y * rstd);  // hidden.to(fp16)
      h2[e] = __hmul2(g2[e], nrm);                                   // weight * hidden
    }
    if (y_out) reinterpret_cast<uint4*>(y_out + static_cast<size_t>(tok) * k)[idx] = v[r];
  }
  requant_row_f16(v, nvec, k, tok, mt, kpad, qp, codes, s_a, z_a, rowsum, err, sm);
}

__global__ void __launch_bounds__(kProdThreads) silu_mul_quant_kernel(
    const __half* __restrict__ gate, const __half* __restrict__ up, int k, int mt, int kpad, QuantParams qp,
    __half* __restrict__ y_out, uint32_t* __restrict__ codes, double* __restrict__ s_a, int32_t* __restrict__ z_a,
    long long* __restrict__ rowsum, unsigned long long* __restrict__ err) {
  __shared__ ProdSmem sm;
  const int tid = threadIdx.x, tok = blockIdx.x;
  const int nvec = k >> 3;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint4* gr = reinterpret_cast<const uint4*>(gate + static_cast<size_t>(tok) * k);
  const uint4* ur = reinterpret_cast<const uint4*>(up + static_cast<size_t>(tok) * k);
  uint4 v[kProdNV], u[kProdNV];
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    const int idx = tid + r * kProdThreads;
    v[r] = idx < nvec ? __ldg(gr + idx) : make_uint4(0u, 0u, 0u, 0u);
    u[r] = idx < nvec ? __ldg(ur + idx) : make_uint4(0u, 0u, 0u, 0u);
  }
  asm volatile("griddepcontrol.launch_dependents;");
#pragma unroll
  for (int r = 0; r < kProdNV; ++r) {
    const int idx = tid + r * kProdThreads;
    if (idx >= nvec) break;
    __half2* h2 = reinterpret_cast<__half2*>(&v[r]);
    const __half2* u2 = reinterpret_cast<const __half2*>(&u[r]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 g = __half22float2(h2[e]);
      const __half2 s = __floats2half2_rn(g.x / (1.0f + __expf(-g.x)), g.y / (1.0f + __expf(-g.y)));  // silu, fp16
      h2[e] = __hmul2(s, u2[e]);
    }
    if (y_out) reinterpret_cast<uint4*>(y_out + static_cast<size_t>(tok) * k)[idx] = v[r];
  }
  requant_row_f16(v, nvec, k, tok, mt, kpad, qp, codes, s_a, z_a, rowsum, err, sm);
}

// ---- stage-in of host activations (end-to-end serving path) --------------------
// dst (device) <- src (pinned host memory, read over PCIe through its UVA
// address): the loads are issued first, then griddepcontrol.wait (the previous
// kernel in the stream may still read dst), then the stores.  PDL: launched
// early, the PCIe read latency overlaps the previous kernel's tail.
__global__ void __launch_bounds__(256) stage_in_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                       size_t n16, unsigned char* __restrict__ dst_tail,
                                                       const unsigned char* __restrict__ src_tail, int tail) {
  asm volatile("griddepcontrol.launch_dependents;");
  constexpr int R = 4;
  const size_t base = static_cast<size_t>(blockIdx.x) * 256 * R + threadIdx.x;
  uint4 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const size_t i = base + static_cast<size_t>(r) * 256;
    if (i < n16) v[r] = src[i];
  }
  unsigned char t = 0;
  const bool has_tail = blockIdx.x == 0 && static_cast<int>(threadIdx.x) < tail;
  if (has_tail) t = src_tail[threadIdx.x];
  asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const size_t i = base + static_cast<size_t>(r) * 256;
    if (i < n16) dst[i] = v[r];
  }
  if (has_tail) dst_tail[threadIdx.x] = t;
}

// ---- host ---------------------------------------------------------------------
size_t qact_codes_bytes(size_t m, size_t k) {
  const size_t mt = static_cast<size_t>(qact_mt(m));
  const size_t kpad = (k + kKBlock - 1) / kKBlock * kKBlock;
  return (m + mt - 1) / mt * mt * kpad;
}

bool qact_supported(size_t m, size_t k) { return m >= 1 && m <= 8 && k >= 8 && k % 8 == 0 && k <= 8 * kProdNV * kProdThreads; }

static int launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelExC(&cfg, fn, args);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "producer launch: %s", cudaGetErrorString(err));
  ABQ_LAUNCHED();
  return ABQ_OK;
}

int run_stage_in(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return ABQ_OK;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15)
    return fail(ABQ_ERR_VALUE, "stage_in: 16-byte aligned buffers required");
  size_t n16 = bytes / 16;
  int tail = static_cast<int>(bytes - n16 * 16);
  uint4* d = static_cast<uint4*>(dst);
  const uint4* s = static_cast<const uint4*>(src);
  unsigned char* dt = static_cast<unsigned char*>(dst) + n16 * 16;
  const unsigned char* stl = static_cast<const unsigned char*>(src) + n16 * 16;
  const unsigned grid = static_cast<unsigned>(std::max<size_t>(1, (n16 + 1023) / 1024));
  void* args[] = {&d, &s, &n16, &dt, &stl, &tail};
  return launch_pdl(reinterpret_cast<const void*>(stage_in_kernel), dim3(grid), dim3(256), args, st);
}

int run_rmsnorm_quant(const __half* x, const __half* gain, float eps, size_t m, size_t k, const QuantParams& qp,
                      __half* y_out, uint32_t* codes, double* s_a, int32_t* z_a, long long* rowsum,
                      unsigned long long* err, cudaStream_t st) {
  if (m == 0) return ABQ_OK;
  int ik = static_cast<int>(k), mt = qact_mt(m), kpad = static_cast<int>((k + kKBlock - 1) / kKBlock * kKBlock);
  void* args[] = {&x, &gain, &eps, &ik, &mt, &kpad, const_cast<QuantParams*>(&qp), &y_out, &codes, &s_a, &z_a,
                  &rowsum, &err};
  return launch_pdl(reinterpret_cast<const void*>(rmsnorm_quant_kernel), dim3(static_cast<unsigned>(m)),
                    dim3(kProdThreads), args, st);
}

int run_silu_mul_quant(const __half* gate, const __half* up, size_t m, size_t k, const QuantParams& qp,
                       __half* y_out, uint32_t* codes, double* s_a, int32_t* z_a, long long* rowsum,
                       unsigned long long* err, cudaStream_t st) {
  if (m == 0) return ABQ_OK;
  int ik = static_cast<int>(k), mt = qact_mt(m), kpad = static_cast<int>((k + kKBlock - 1) / kKBlock * kKBlock);
  void* args[] = {&gate, &up, &ik, &mt, &kpad, const_cast<QuantParams*>(&qp), &y_out, &codes, &s_a, &z_a,
                  &rowsum, &err};
  return launch_pdl(reinterpret_cast<const void*>(silu_mul_quant_kernel), dim3(static_cast<unsigned>(m)),
                    dim3(kProdThreads), args, st);
}

}  // namespace abq_dev
