// Pure compute rate of the decode-GEMV inner body with the weights already
// in shared memory (no TMA, no barriers): NW warps per CTA, one CTA per SM,
// each warp loops over 2 KB units (W4 raw-mask fields x IMMA m16n8k32, or
// x DP4A), optional per-unit row-tile flush.  Reports bytes/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbcomp tools/microbench_compute.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32) comp(int iters, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];  // 64 units of 2 KB
  __shared__ uint32_t sacc[64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 512; i += NW * 32) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (tid < 64) sacc[tid] = 0;
  __syncthreads();
  int acc[2][4] = {};
  uint32_t dacc[4] = {};
  const uint32_t b0 = lane * 77u, b1 = lane * 13u;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int unit = (warp + it * NW) & 63;
    const uint4* p = reinterpret_cast<const uint4*>(sm + unit * 2048) + lane;
    uint4 w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) w[t] = p[t * 32];
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int Q = 0; Q < 4; ++Q)
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const uint32_t m = 0x0F0F0F0Fu << (4 * f);
          imma(acc[f], w[Q].x & m, w[Q].y & m, w[Q].z & m, w[Q].w & m, b0 + Q, b1 + f);
        }
      if (MODE == 2) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t v = (uint32_t)acc[0][r] + ((uint32_t)acc[1][r] >> 4);
          acc[0][r] = acc[1][r] = 0;
          if ((lane & 3) == 0 && (r & 1) == 0) atomicAdd(&sacc[(lane >> 2) + 8 * (r >> 1)], v);
        }
      }
    } else {
#pragma unroll
      for (int Q = 0; Q < 4; ++Q)
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const uint32_t m = 0x0F0F0F0Fu << (4 * f);
          dacc[2 * f] = __dp4a(w[Q].x & m, b0 + Q, dacc[2 * f]);
          dacc[2 * f + 1] = __dp4a(w[Q].y & m, b1 + Q, dacc[2 * f + 1]);
          dacc[2 * f] = __dp4a(w[Q].z & m, b0 ^ Q, dacc[2 * f]);
          dacc[2 * f + 1] = __dp4a(w[Q].w & m, b1 ^ Q, dacc[2 * f + 1]);
        }
    }
  }
  const long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc[0][0] == 7 && acc[1][2] == 9 && dacc[0] == 3 && dacc[3] == 5) out[2000] = sacc[lane];
}

template <int NW, int MODE>
void run(int sms, unsigned long long* out, const char* name) {
  const int iters = 2000;
  cudaFuncSetAttribute(comp<NW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  comp<NW, MODE><<<sms, NW * 32, 131072>>>(iters, out);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  printf("%-26s NW=%2d: %6.1f B/clk/SM  (%5.0f cycles per unit per warp)  %s\n", name, NW, 2048.0 * iters * NW / c,
         c / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, 8 * 4096);
  run<4, 0>(sms, out, "IMMA raw-mask");
  run<8, 0>(sms, out, "IMMA raw-mask");
  run<16, 0>(sms, out, "IMMA raw-mask");
  run<32, 0>(sms, out, "IMMA raw-mask");
  run<8, 2>(sms, out, "IMMA raw-mask + flush");
  run<16, 2>(sms, out, "IMMA raw-mask + flush");
  run<32, 2>(sms, out, "IMMA raw-mask + flush");
  run<8, 1>(sms, out, "DP4A raw-mask");
  run<16, 1>(sms, out, "DP4A raw-mask");
  run<32, 1>(sms, out, "DP4A raw-mask");
  return 0;
}
