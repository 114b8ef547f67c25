// Throughput of the decode-GEMV unit body on sm_100a with operands resident in
// shared memory (no TMA waits): q=4 weight planes merged into u8 codes
// (shift + LOP3 per plane-register) + one IMMA m16n8k32 per k32 chunk.
// Variants isolate the ALU work and the IMMA work.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbg tools/microbench_gemv_body.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int MODE>  // 0 full, 1 ALU only (xor into acc), 2 IMMA only (raw words)
__global__ void __launch_bounds__(512, 1) body(int units, int* out) {
  __shared__ uint4 ws[16][4][32];
  __shared__ uint2 bs[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 4 * 32; i += blockDim.x)
    (&ws[0][0][0])[i] = make_uint4(i * 2654435761u, i * 40503u, i ^ 0x5bd1e995u, i * 97u);
  for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) (&bs[0][0])[i] = make_uint2(i * 3u, i * 7u);
  __syncthreads();
  int acc[4] = {0, 0, 0, 0};
  for (int u = 0; u < units; ++u) {
    uint4 w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) w[t] = ws[(warp + u) & 15][t][lane];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint2 b = bs[c][lane];
      uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      if (MODE != 2) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int tb = 4 + t;
          const uint32_t m = 0x01010101u << tb;
          if (tb >= c) {
            a0 |= (w[t].x << (tb - c)) & m; a1 |= (w[t].y << (tb - c)) & m;
            a2 |= (w[t].z << (tb - c)) & m; a3 |= (w[t].w << (tb - c)) & m;
          } else {
            const uint32_t f = 1u << (32 - (c - tb));
            a0 |= __umulhi(w[t].x, f) & m; a1 |= __umulhi(w[t].y, f) & m;
            a2 |= __umulhi(w[t].z, f) & m; a3 |= __umulhi(w[t].w, f) & m;
          }
        }
      } else {
        a0 = w[c & 3].x; a1 = w[c & 3].y; a2 = w[c & 3].z; a3 = w[c & 3].w;
      }
      if (MODE == 1) {
        acc[0] ^= a0 + b.x; acc[1] ^= a1 + b.y; acc[2] ^= a2; acc[3] ^= a3;
      } else {
        imma(acc, a0, a1, a2, a3, b.x, b.y);
      }
    }
  }
  if ((acc[0] ^ acc[1] ^ acc[2] ^ acc[3]) == 0x12345) out[0] = 1;
}

template <int MODE>
void run(const char* name, int warps_per_cta, int* out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int units = 2000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  body<MODE><<<sms, warps_per_cta * 32>>>(units, out);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  body<MODE><<<sms, warps_per_cta * 32>>>(units, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double units_per_sm = double(units) * warps_per_cta;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-10s warps=%2d  %.1f cycles/unit/SM  -> q=4 bytes/clk/SM %.1f  (%.1f us)\n", name, warps_per_cta,
         cyc / units_per_sm, 2048.0 * units_per_sm / cyc, ms * 1e3);
}

int main() {
  int* out; cudaMalloc(&out, 4);
  for (int w : {8, 16}) {
    run<0>("full", w, out);
    run<1>("alu-only", w, out);
    run<2>("imma-only", w, out);
  }
  return 0;
}
