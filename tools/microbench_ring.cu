// Throughput of the decode-GEMV consumer loop in isolation: one CTA per SM
// (or two), a producer warp streaming W bytes per CTA through a ring of S
// slots (8 units of 2 KB = 16 KB per slot, 1-D TMA bulk copies) from a buffer
// that is either L2-resident (small, re-read) or HBM-streamed (large), and NW
// consumer warps doing, per unit, nothing / the LDS only / LDS + W4 raw-mask
// IMMAs.  Prints bytes per clock per SM and us per CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbring tools/microbench_ring.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NW, int UPW>
__global__ void __launch_bounds__((NW + 1) * 32) ring_kernel(const uint8_t* src, size_t wrap, int units, int S, int mode,
                                                              unsigned long long* out) {
  constexpr int UPS = 8, UB = 2048, SB = UPS * UB * UPW, NG = NW / UPS;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t sacc[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nsl = units / (UPS * UPW);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(UPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long t0 = clock64();
  const uint8_t* base = src + (blockIdx.x * (size_t)units * UB) % wrap;
  if (warp == NW) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nsl; ++i) {
        if (i >= S) wait_par(&empty[s], ph ^ 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(SB));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + s * SB)),
                     "l"(base + (size_t)i * SB), "r"(SB), "r"(sa(&full[s])) : "memory");
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
    return;
  }
  const int grp = warp / UPS, wi = warp % UPS;
  int acc[2][4] = {};
  uint32_t x = 0;
  int s = grp;
  uint32_t ph = 0;
  const uint32_t ring_lane = sa(sm) + wi * UB * UPW + lane * 16;
  for (int i = grp; i < nsl; i += NG) {
    wait_par(&full[s], ph);
    for (int uu = 0; uu < UPW; ++uu)
    if (mode >= 1) {
      uint4 w[4];
      const uint32_t a = ring_lane + s * SB + uu * UB;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[t].x), "=r"(w[t].y), "=r"(w[t].z), "=r"(w[t].w) : "r"(a + t * 512));
      if (mode == 1) {
#pragma unroll
        for (int t = 0; t < 4; ++t) x ^= w[t].x ^ w[t].y ^ w[t].z ^ w[t].w;
      } else if (mode == 4) {  // CUDA-core dot products: raw nibble fields x activation words
        uint32_t d[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int Q = 0; Q < 4; ++Q)
#pragma unroll
          for (int f = 0; f < 2; ++f) {
            const uint32_t m = 0x0F0F0F0Fu << (4 * f);
            const uint32_t a0 = x + Q * 2 + f, a1 = x ^ (Q * 2 + f);
            d[2 * f + 0] = __dp4a(w[Q].x & m, a0, d[2 * f + 0]);
            d[2 * f + 1] = __dp4a(w[Q].y & m, a0, d[2 * f + 1]);
            d[2 * f + 0] = __dp4a(w[Q].z & m, a1, d[2 * f + 0]);
            d[2 * f + 1] = __dp4a(w[Q].w & m, a1, d[2 * f + 1]);
          }
        acc[0][0] += d[0] + (d[2] >> 4);
        acc[0][1] += d[1] + (d[3] >> 4);
      } else {
#pragma unroll
        for (int Q = 0; Q < 4; ++Q)
#pragma unroll
          for (int f = 0; f < 2; ++f) {
            const uint32_t m = 0x0F0F0F0Fu << (4 * f);
            imma(acc[f], w[Q].x & m, w[Q].y & m, w[Q].z & m, w[Q].w & m, x + Q, x + f);
          }
        if (mode == 3) {  // per-unit row-tile flush: combine the fields, shared atomics, zero
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t v = (uint32_t)acc[0][r] + ((uint32_t)acc[1][r] >> 4);
            acc[0][r] = acc[1][r] = 0;
            if ((lane & 3) == 0 && (r & 1) == 0) atomicAdd(&sacc[(lane >> 2) + 8 * (r >> 1)], v);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    s += NG;
    if (s >= S) { s -= S; ph ^= 1u; }
  }
  const long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (x == 0x1234567u && acc[0][0] == 7 && acc[1][1] == 3) out[1000] = x + sacc[lane & 15];
}

template <int NW, int UPW = 1>
void run(const uint8_t* buf, size_t wrap, int units, int S, int mode, int ctas, unsigned long long* out, const char* tag) {
  const size_t smem = (size_t)S * 16384 * UPW;
  cudaFuncSetAttribute(ring_kernel<NW, UPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ring_kernel<NW, UPW><<<ctas, (NW + 1) * 32, smem>>>(buf, wrap, units, S, mode, out);
  cudaEventRecord(e0);
  const int R = 20;
  for (int r = 0; r < R; ++r) ring_kernel<NW, UPW><<<ctas, (NW + 1) * 32, smem>>>(buf, wrap, units, S, mode, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[296];
  cudaMemcpy(h, out, ctas * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < ctas; ++i) cyc += h[i];
  cyc /= ctas;
  const double bytes = (double)units * 2048;
  printf("%-5s UPW=%d NW=%2d S=%2d mode=%d ctas=%d: %6.1f B/clk per CTA (%.2f us CTA, %.2f us/launch, %.0f GB/s)  %s\n", tag, UPW, NW, S, mode,
         ctas, bytes / cyc, cyc / 1965.0, ms * 1e3 / R, bytes * ctas / (ms * 1e-3 / R) * 1e-9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = 1ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* out;
  cudaMalloc(&out, 8 * 2048);
  const int units = 75 * 16;  // 2.4 MB per CTA: long enough to measure the steady state
  for (int l2 = 1; l2 >= 1; --l2) {
    const size_t wrap = l2 ? (size_t)units * 2048 * 8 : big;  // L2: 8 CTAs' worth re-read by all
    const char* tag = l2 ? "L2" : "HBM";
    for (int mode = 1; mode < 5; ++mode) {
      if (mode == 3) continue;
      run<16, 1>(buf, wrap, units, 8, mode, sms, out, tag);
      run<16, 2>(buf, wrap, units, 4, mode, sms, out, tag);
      run<16, 4>(buf, wrap, units, 2, mode, sms, out, tag);
      run<8, 2>(buf, wrap, units, 6, mode, sms, out, tag);
      run<8, 4>(buf, wrap, units, 3, mode, sms, out, tag);
    }
  }
  return 0;
}
